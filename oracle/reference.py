"""The REFERENCE itself (pipeshift, CPython) staged for timing -- TEST / BASELINE
INFRASTRUCTURE ONLY (bench.py's reference arm and cpu_baseline, tools/).

`stage()` is the committed recipe: it copies the reference package
/root/reference/pkg/src/pipeshift (and its packaged scenario) unmodified into the
git-ignored oracle/_ref/, which travels to the GPU box with the repo snapshot (gpurun
ships untracked files), so the reference's own CPU path can be timed on the box's
host cores.  /root/reference exists only in the dev container; nothing here reads it
at run time on the box.  No reference source is committed.

The timers follow SURVEY §8(d) "CPU baseline": bounded samples of the bench workload
(Llama-3-8B shape: 4096-B token-layer cells, 16-token blocks, k = 4, 2048-token
requests, migrating groups 2-3 of a PP2 stage), scaled per unit.  The reference moves
8-byte fingerprints, not KV bytes, so its byte rates are "KV-equivalent" (cells x 4096 B).
"""

from __future__ import annotations

import os
import platform
import shutil
import subprocess
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
REFERENCE_SRC = Path("/root/reference/pkg/src/pipeshift")
REFERENCE_SCENARIO = Path("/root/reference/pkg/scenarios/heterogeneous_shift.yaml")
REFERENCE_TESTS = Path("/root/reference/pkg/tests")

CELL = 4096          # token_kv_bytes_per_layer of the Llama-3 shapes
K, S, CTX = 4, 16, 2048
SRC_GROUPS, MIG_GROUPS = (0, 1, 2, 3), (2, 3)
MIG_LAYERS = set(range(9, 17))   # groups 2, 3 at k = 4: the PP2 -> 4 migrating layers


def stage(force: bool = False) -> Path | None:
    """Copy the unmodified reference package into oracle/_ref/ (dev container only)."""
    if not REFERENCE_SRC.is_dir():
        return REF_DIR if (REF_DIR / "pipeshift" / "__init__.py").exists() else None
    dst = REF_DIR / "pipeshift"
    stale = force or not dst.exists() or any(
        not (dst / p.name).exists() or p.stat().st_mtime > (dst / p.name).stat().st_mtime
        for p in REFERENCE_SRC.glob("*.py"))
    if stale:
        if dst.exists():
            shutil.rmtree(dst)
        shutil.copytree(REFERENCE_SRC, dst, ignore=shutil.ignore_patterns("__pycache__"))
        (REF_DIR / "scenarios").mkdir(parents=True, exist_ok=True)
        if REFERENCE_SCENARIO.exists():
            shutil.copy2(REFERENCE_SCENARIO, REF_DIR / "scenarios" / REFERENCE_SCENARIO.name)
    # the reference's own test modules, unmodified: tests/test_gpu_reference_own_suites.py
    # runs them against this package's data plane through the maintainer shim
    tdst = REF_DIR / "tests"
    if REFERENCE_TESTS.is_dir() and (force or not tdst.exists() or any(
            not (tdst / p.name).exists() or p.stat().st_mtime > (tdst / p.name).stat().st_mtime
            for p in REFERENCE_TESTS.glob("*.py"))):
        if tdst.exists():
            shutil.rmtree(tdst)
        shutil.copytree(REFERENCE_TESTS, tdst, ignore=shutil.ignore_patterns("__pycache__"))
    return REF_DIR


def available() -> bool:
    return (REF_DIR / "pipeshift" / "__init__.py").exists()


def pipeshift():
    """Import the staged reference (oracle/_ref/pipeshift)."""
    if not available():
        raise RuntimeError("reference not staged: run oracle.reference.stage() in the dev container")
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import pipeshift as ps  # noqa: PLC0415
    return ps


def host_info() -> dict:
    cpu = ""
    try:
        cpu = next(l.split(":", 1)[1].strip() for l in
                   subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()
                   if l.startswith("Model name"))
    except Exception:
        pass
    return {"cpu": cpu, "nproc": os.cpu_count(), "python": platform.python_version()}


def _payloads(ps, rid: str, g: int, start: int, n: int) -> list[int]:
    # PipelineEngine._payloads (engine.py:252-261) for positions start..start+n-1
    seed = ps.events.stable_hash(rid, g)
    return [((seed * 0x9E3779B97F4A7C15 + p * 0xBF58476D1CE4E5B9) & ((1 << 63) - 1))
            for p in range(start, start + n)]


class BulkRound:
    """One bench step on the reference: MigrationManager.start_migration of the PP2 -> 4
    pair (seed every live cell of groups 2-3, migrator.py:170-183) + the event loop until
    the bulk patch is drained, sent and applied (migrator.py:208-273, 93-132), over a
    source stage holding n_req requests x 2048 tokens in groups 0-3."""

    def __init__(self, n_req: int) -> None:
        ps = self.ps = pipeshift()
        from pipeshift import kvstore  # noqa: PLC0415
        self.n_req = n_req
        self.cap = n_req * (CTX // S) + 8
        self.src = kvstore.KvStore(1, K, S, self.cap, resident_groups=set(SRC_GROUPS))
        for i in range(n_req):
            for g in SRC_GROUPS:
                self.src.append(f"r{i:04d}", g, CTX, _payloads(ps, f"r{i:04d}", g, 0, CTX))
        self.cells = n_req * CTX * len(MIG_GROUPS) * K

    def run(self) -> float:
        ps = self.ps
        from pipeshift import events, kvstore, migrator  # noqa: PLC0415
        sched, trace = events.EventScheduler(), events.EventTrace()
        fab = ps.CommFabric(sched, trace, [1, 2], ps.FabricConfig())
        dst = kvstore.KvStore(2, K, S, self.cap, resident_groups=set(MIG_GROUPS))
        mgr = migrator.MigrationManager(sched, trace, fab, {1: self.src, 2: dst},
                                        token_kv_bytes=CELL, k=K)
        t0 = time.perf_counter()
        mgr.start_migration({(1, 2): MIG_LAYERS})
        sched.run(until=60.0)
        dt = time.perf_counter() - t0
        assert mgr.lag(2) == 0 and len(dst.snapshot_group(MIG_GROUPS[0])) == self.n_req
        return dt


def time_steady(n_req: int = 64, rounds: int = 20) -> dict:
    """Steady patch rounds on the reference after the bulk round: every round appends the
    decode pattern -- one new token per request in each of the stage's groups
    (engine.py:377-404) -- notifies the migration (on_kv_written, migrator.py:190-197) and
    runs the event loop until the round's patch is drained, sent and applied."""
    ps = pipeshift()
    from pipeshift import events, kvstore, migrator  # noqa: PLC0415
    b = BulkRound.__new__(BulkRound)
    b.ps, b.n_req = ps, n_req
    b.cap = n_req * (CTX // S + 2) + 8
    b.src = kvstore.KvStore(1, K, S, b.cap, resident_groups=set(SRC_GROUPS))
    for i in range(n_req):
        for g in SRC_GROUPS:
            b.src.append(f"r{i:04d}", g, CTX, _payloads(ps, f"r{i:04d}", g, 0, CTX))
    sched, trace = events.EventScheduler(), events.EventTrace()
    fab = ps.CommFabric(sched, trace, [1, 2], ps.FabricConfig())
    dst = kvstore.KvStore(2, K, S, b.cap, resident_groups=set(MIG_GROUPS))
    mgr = migrator.MigrationManager(sched, trace, fab, {1: b.src, 2: dst}, token_kv_bytes=CELL, k=K)
    mgr.start_migration({(1, 2): MIG_LAYERS})
    sched.run(until=60.0)
    dt = 0.0
    for r in range(rounds):
        pos = CTX + r
        t0 = time.perf_counter()
        for i in range(n_req):
            for g in SRC_GROUPS:
                b.src.append(f"r{i:04d}", g, 1, _payloads(ps, f"r{i:04d}", g, pos, 1))
                mgr.on_kv_written(1, f"r{i:04d}", g, pos, 1)
        sched.run(until=sched.now + 1.0)
        dt += time.perf_counter() - t0
        assert mgr.lag(2) == 0
    cells = n_req * len(MIG_GROUPS) * K
    return {"requests": n_req, "cells_per_round": cells, "rounds": rounds,
            "us_per_round": round(dt / rounds * 1e6, 1),
            "kv_equivalent_gbs": round(cells * CELL * rounds / dt / 1e9, 4),
            "note": "includes the stage's append of the round's tokens (all 4 groups)"}


def time_append(n_req: int = 64) -> dict:
    from pipeshift import kvstore  # noqa: PLC0415
    ps = pipeshift()
    st = kvstore.KvStore(1, K, S, n_req * (CTX // S) + 8, resident_groups=set(SRC_GROUPS))
    pays = {(i, g): _payloads(ps, f"r{i:04d}", g, 0, CTX) for i in range(n_req) for g in SRC_GROUPS}
    t0 = time.perf_counter()
    for (i, g), p in pays.items():
        st.append(f"r{i:04d}", g, CTX, p)
    dt = time.perf_counter() - t0
    cells = n_req * len(SRC_GROUPS) * CTX * K
    return {"tokens": n_req * len(SRC_GROUPS) * CTX, "cells": cells, "seconds": round(dt, 3),
            "cells_per_s": round(cells / dt), "kv_equivalent_gbs": round(cells * CELL / dt / 1e9, 4)}


def time_resize(n_blocks: int = 33344) -> dict:
    """compact + resize (kvstore.py:247-282) at the bench source store's block count."""
    from pipeshift import kvstore  # noqa: PLC0415
    pipeshift()
    st = kvstore.KvStore(1, K, S, n_blocks, resident_groups={0, 1})
    for i in range(240):
        st.append(f"r{i:04d}", 0, CTX, [0] * CTX)
    for i in range(0, 240, 4):
        st.free_request(f"r{i:04d}")
    t0 = time.perf_counter()
    st.compact()
    st.resize(int(n_blocks * 0.8))
    dt = time.perf_counter() - t0
    return {"blocks_from": n_blocks, "blocks_to": int(n_blocks * 0.8), "ms": round(dt * 1e3, 3)}


def time_scenario() -> dict:
    ps = pipeshift()
    path = REF_DIR / "scenarios" / REFERENCE_SCENARIO.name
    if not path.exists():
        return {"error": "packaged scenario not staged"}
    sc = ps.load_scenario(str(path))
    t0 = time.perf_counter()
    ps.run_scenario(sc, seed=0)
    return {"scenario": path.name, "seed": 0, "seconds": round(time.perf_counter() - t0, 2)}
