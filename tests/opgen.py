"""Seeded KvStore / migration op sequences shared by the golden-fixture generator
(tests/golden/make_golden.py, runs the reference) and the parity tests (run the
oracle and the GPU store).  Pure Python, no reference import."""

from __future__ import annotations

import random

from paper_2604_12171_b200.events import stable_hash


def payload(rid: str, group: int, pos: int) -> int:
    return stable_hash(rid, group, pos)


def wpayload(rid: str, group: int, pos: int) -> int:
    return stable_hash("w", rid, group, pos)


def kv_store_params(seed: int) -> dict:
    rng = random.Random(seed * 7919 + 1)
    k = rng.choice([1, 2, 4])
    s = rng.choice([4, 8, 16])
    groups = sorted(rng.sample(range(6), rng.randint(1, 3)))
    return {"gpu_id": rng.randint(1, 4), "k": k, "s": s, "capacity": rng.randint(8, 40),
            "groups": groups}


def kv_ops(seed: int, n_ops: int = 80) -> list[dict]:
    """Random append / write_slots / free / compact / resize / drop / add ops."""
    rng = random.Random(seed)
    p = kv_store_params(seed)
    groups = list(p["groups"])
    extra = [g for g in range(6) if g not in groups]
    reqs = [f"r{i}" for i in range(7)]
    ops: list[dict] = []
    for _ in range(n_ops):
        x = rng.random()
        rid = rng.choice(reqs)
        if x < 0.45:
            ops.append({"op": "append", "rid": rid, "g": rng.choice(groups),
                        "n": rng.randint(0, 3 * p["s"])})
        elif x < 0.55:
            g = rng.choice(groups)
            top = rng.randint(1, 4 * p["s"])
            pos = sorted(rng.sample(range(top), rng.randint(1, min(top, 12))))
            ops.append({"op": "write_slots", "rid": rid, "g": g, "pos": pos})
        elif x < 0.68:
            ops.append({"op": "free", "rid": rid})
        elif x < 0.78:
            ops.append({"op": "compact"})
        elif x < 0.9:
            ops.append({"op": "resize", "n": rng.randint(0, p["capacity"] + 12)})
        elif x < 0.95 and len(groups) > 1:
            g = rng.choice(groups)
            ops.append({"op": "drop", "groups": [g]})
            groups.remove(g)
            extra.append(g)
        elif extra:
            g = rng.choice(extra)
            ops.append({"op": "add_group", "g": g})
            extra.remove(g)
            groups.append(g)
        else:
            ops.append({"op": "compact"})
    return ops


def apply_op(store, op: dict, exc_types: tuple) -> str:
    """Apply one op to a KvStore-like object; returns a result tag."""
    kind = op["op"]
    try:
        if kind == "append":
            rid, g, n = op["rid"], op["g"], op["n"]
            start = store.tables[rid].written.get(g, 0) if rid in store.tables else 0
            slots = store.append(rid, g, n, [payload(rid, g, start + i) for i in range(n)])
            return "ok:" + ",".join(f"{s.block_id}/{s.offset}" for s in slots)
        if kind == "write_slots":
            rid, g = op["rid"], op["g"]
            store.write_slots(rid, g, [(q, wpayload(rid, g, q)) for q in op["pos"]])
            return "ok"
        if kind == "free":
            stats = store.free_request(op["rid"])
            return "ok:" + repr(sorted(stats.items()))
        if kind == "compact":
            return f"ok:{store.compact()}"
        if kind == "resize":
            store.resize(op["n"])
            return "ok"
        if kind == "drop":
            return f"ok:{store.drop_layer_groups(op['groups'])}"
        if kind == "add_group":
            store.resident_groups |= {op["g"]}
            return "ok"
    except exc_types as e:  # noqa: PERF203
        return "err:" + type(e).__name__
    raise ValueError(kind)


def light_state(store) -> list:
    return [store.capacity_blocks, store.used_blocks, store.free_blocks,
            round(store.effective_utilization(), 12)]


def full_state(store) -> dict:
    tables = {}
    for rid in sorted(store.tables):
        t = store.tables[rid]
        tables[rid] = {"chain": [b.block_id for b in t.chain],
                       "written": sorted([int(g), int(w)] for g, w in t.written.items())}
    checks = {}
    for rid in sorted(store.tables):
        for g, w in sorted(store.tables[rid].written.items()):
            vals = []
            for pos in range(w):
                try:
                    vals.append(int(store.read_checksum(rid, g, pos)))
                except Exception:  # holes left by sparse write_slots
                    vals.append(None)
            checks[f"{rid}|{g}"] = vals
    return {"blocks": [[b.block_id, b.state] for b in store.blocks], "tables": tables,
            "checksums": checks, "resident": sorted(store.resident_groups),
            "light": light_state(store)}


def migration_case(seed: int) -> dict:
    """A two-store migration scenario: fill, start, writes/frees during migration."""
    rng = random.Random(seed + 424242)
    k = rng.choice([1, 2, 4])
    s = rng.choice([4, 8, 16])
    src_groups = [0, 1, 2]
    mig_groups = sorted(rng.sample(src_groups, rng.randint(1, 2)))
    layers = sorted(layer for g in mig_groups for layer in range(g * k + 1, g * k + k + 1))
    fills = []
    for i in range(rng.randint(1, 5)):
        rid = f"q{i}"
        for g in src_groups:
            fills.append((rid, g, rng.randint(1, 3 * s)))
    events = []
    t = 0.0
    for _ in range(rng.randint(2, 10)):
        t += rng.uniform(0.0002, 0.004)
        x = rng.random()
        rid = f"q{rng.randint(0, 6)}"
        if x < 0.7:
            events.append({"t": t, "op": "write", "rid": rid, "g": rng.choice(src_groups),
                           "n": rng.randint(1, s + 3)})
        else:
            events.append({"t": t, "op": "free", "rid": rid})
    return {"k": k, "s": s, "src_groups": src_groups, "dst_groups": [5],
            "layers": layers, "fills": fills, "events": events,
            "capacity": rng.randint(40, 80), "drain_period": rng.choice([1e-3, 2e-3, 1e-2]),
            "streaming": rng.random() < 0.85}


def run_migration_case(ns, case: dict, store_kwargs: dict | None = None) -> dict:
    """Drive one migration_case through a pipeshift-like namespace ``ns``
    (attributes KvStore, MigrationManager, EventScheduler, EventTrace, CommFabric,
    FabricConfig).  Returns the observable results compared bit-exactly."""
    import hashlib

    kw = store_kwargs or {}
    sched = ns.EventScheduler()
    trace = ns.EventTrace()
    fabric = ns.CommFabric(sched, trace, [1, 2], ns.FabricConfig())
    k, s = case["k"], case["s"]
    src = ns.KvStore(1, k, s, case["capacity"], resident_groups=case["src_groups"], **kw)
    dst = ns.KvStore(2, k, s, case["capacity"], resident_groups=case["dst_groups"], **kw)
    mgr = ns.MigrationManager(sched, trace, fabric, {1: src, 2: dst}, token_kv_bytes=8 * 1024,
                              k=k, drain_period=case["drain_period"])
    for rid, g, n in case["fills"]:
        start = src.tables[rid].written.get(g, 0) if rid in src.tables else 0
        src.append(rid, g, n, [payload(rid, g, start + i) for i in range(n)])
    mig_groups = sorted({(layer - 1) // k for layer in case["layers"]})
    dst.resident_groups |= set(mig_groups)
    mgr.start_migration({(1, 2): set(case["layers"])}, streaming=case["streaming"])

    def make(ev):
        def fire():
            rid = ev["rid"]
            if ev["op"] == "write":
                g, n = ev["g"], ev["n"]
                start = src.tables[rid].written.get(g, 0) if rid in src.tables else 0
                try:
                    src.append(rid, g, n, [payload(rid, g, start + i) for i in range(n)])
                except Exception:
                    return
                mgr.on_kv_written(1, rid, g, start, n)
            else:
                src.free_request(rid)
                mgr.on_request_freed(rid)
        return fire

    for ev in case["events"]:
        sched.at(ev["t"], make(ev))
    sched.run(until=5.0)
    pauses: list = []
    mgr.final_sync_all(pauses.append)
    sched.run(until=10.0)
    recv = mgr.receivers[(1, 2)]
    return {
        "src": {str(g): {r: list(v) for r, v in src.snapshot_group(g).items()} for g in mig_groups},
        "dst": {str(g): {r: list(v) for r, v in dst.snapshot_group(g).items()} for g in mig_groups},
        "t_sched": mgr.counters.t_sched.get(2, 0),
        "t_applied": mgr.counters.t_applied.get(2, 0),
        "applied_log": [list(x) for x in recv.applied_cells_log],
        "pauses": pauses,
        "trace_sha": hashlib.sha256(trace.to_jsonl().encode()).hexdigest(),
        "n_events": len(trace),
        "dst_light": light_state(dst),
        "src_light": light_state(src),
    }
