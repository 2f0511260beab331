"""Pin the CPU oracle (oracle/) and the host-side restatements to the reference's
own outputs (tests/golden/*.json, made by tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

import opgen
import oracle
from oracle.migrate import OracleMigrationManager
from paper_2604_12171_b200 import events, fabric


def test_fingerprints_match_reference(golden):
    g = golden("fingerprints.json")
    for parts, value in g["hashes"]:
        assert events.stable_hash(*parts) == value
        assert oracle.stable_hash(*parts) == value
    for seed, vals in g["payloads"]:
        for pos, v in zip((0, 1, 2, 3, 17, 511, 2047), vals):
            assert events.payload_fingerprint(seed, pos) == v
            assert oracle.payload(seed, pos) == v
    seed = events.stable_hash("r0000", 0)
    assert [oracle.payload(seed, p) for p in range(4)] == g["engine_r0000_g0"]
    # SURVEY Appendix A known answers
    assert g["engine_r0000_g0"] == [77374864552834275, 4641851620854602396,
                                    9206328377156370517, 4547433096603362830]
    assert g["addresses_gpu3"] == [0x300000000000, 0x300000200000, 0x300000400000,
                                   0x300000600000]


def test_expansion_is_word_splitmix():
    fp = 0x1234_5678_9ABC_DEF0
    cell = oracle.expand_cell(fp, 2, 64)
    words = np.frombuffer(cell, dtype=np.uint64)
    for w in range(8):
        assert int(words[w]) == int(oracle.lib().or_expand_word(fp, 2, w))
    assert oracle.expand_cell(fp, 2, 64) != oracle.expand_cell(fp, 3, 64)


@pytest.mark.parametrize("seed", range(40))
def test_oracle_replays_reference_kv_sequences(golden, seed):
    case = golden("kv_sequences.json")[seed]
    p = case["params"]
    st = oracle.OracleStore(p["gpu_id"], p["k"], p["s"], p["capacity"], p["groups"])
    excs = (oracle.KvError, ValueError)
    for i, op in enumerate(opgen.kv_ops(seed)):
        assert opgen.apply_op(st, op, excs) == case["results"][i], (i, op)
        assert opgen.light_state(st) + [st.occupied] == case["lights"][i], (i, op)
    assert opgen.full_state(st) == case["final"]
    assert hashlib.sha256(repr(st.state_digest()).encode()).hexdigest() == case["digest_sha"]


class _OracleNS:
    EventScheduler = events.EventScheduler
    EventTrace = events.EventTrace
    CommFabric = fabric.CommFabric
    FabricConfig = fabric.FabricConfig

    @staticmethod
    def KvStore(gpu_id, k, s, cap, resident_groups=()):
        return oracle.OracleStore(gpu_id, k, s, cap, resident_groups)

    MigrationManager = OracleMigrationManager


@pytest.mark.parametrize("seed", range(80))
def test_oracle_replays_reference_migrations(golden, seed):
    case = golden("migration_cases.json")[seed]
    res = opgen.run_migration_case(_OracleNS, case["case"])
    want = dict(case["result"])
    want.pop("drained")
    assert res == want
