"""Time the REFERENCE (pipeshift, CPython) on this container's CPU at the bench shape.

    python tools/time_reference.py        -> profiles/reference_cpu_r1.json

The reference cannot travel to the GPU box (only this container has /root/reference),
so bench.py's reference arm times the oracle port there; this records the reference's
own CPU path beside it (SURVEY §8d "CPU baseline"): single-threaded CPython, bounded
samples of the bench workload (Llama-3-8B shape, 16-token blocks, k = 4, 2048-token
requests), scaled per unit:
  - KvStore.append cells/s (kvstore.py:163-199);
  - one bulk migration round, MigrationManager.start_migration + scheduler.run
    (migrator.py:170-273), in cells/s and "KV-equivalent" GB/s (cells x 4096 B; the
    reference moves 8-byte fingerprints, not KV bytes);
  - compact + resize at the bench's block count (kvstore.py:247-282);
  - the packaged heterogeneous_shift scenario, whole run wall time.
"""

from __future__ import annotations

import json
import platform
import subprocess
import sys
import time
from pathlib import Path

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
ROOT = Path(__file__).resolve().parents[1]

import pipeshift  # noqa: E402
from pipeshift import events, kvstore, migrator  # noqa: E402

CELL = 4096          # token_kv_bytes_per_layer of the Llama-3 shapes
K, S, CTX = 4, 16, 2048


def payloads(rid, g, start, n):
    seed = events.stable_hash(rid, g)
    return [((seed * 0x9E3779B97F4A7C15 + p * 0xBF58476D1CE4E5B9) & ((1 << 63) - 1))
            for p in range(start, start + n)]


def time_append(n_req=64):
    st = kvstore.KvStore(1, K, S, n_req * (CTX // S) + 8, resident_groups={0, 1, 2, 3})
    pays = {(i, g): payloads(f"r{i:04d}", g, 0, CTX) for i in range(n_req) for g in range(4)}
    t0 = time.perf_counter()
    for (i, g), p in pays.items():
        st.append(f"r{i:04d}", g, CTX, p)
    dt = time.perf_counter() - t0
    cells = n_req * 4 * CTX * K
    return {"tokens": n_req * 4 * CTX, "cells": cells, "seconds": round(dt, 3),
            "cells_per_s": round(cells / dt), "kv_equivalent_gbs": round(cells * CELL / dt / 1e9, 4)}


def time_bulk_round(n_req=64):
    sched, trace = events.EventScheduler(), events.EventTrace()
    fab = pipeshift.CommFabric(sched, trace, [1, 2], pipeshift.FabricConfig())
    cap = n_req * (CTX // S) + 8
    src = kvstore.KvStore(1, K, S, cap, resident_groups={0, 1, 2, 3})
    dst = kvstore.KvStore(2, K, S, cap, resident_groups={2, 3})
    mgr = migrator.MigrationManager(sched, trace, fab, {1: src, 2: dst}, token_kv_bytes=CELL, k=K)
    for i in range(n_req):
        for g in range(4):
            src.append(f"r{i:04d}", g, CTX, payloads(f"r{i:04d}", g, 0, CTX))
    layers = set(range(9, 17))     # groups 2, 3: the PP2 -> 4 migrating layers
    t0 = time.perf_counter()
    mgr.start_migration({(1, 2): layers})
    sched.run(until=60.0)
    dt = time.perf_counter() - t0
    cells = n_req * 2 * CTX * K
    assert mgr.lag(2) == 0
    return {"keys": n_req * 2 * CTX, "cells": cells, "seconds": round(dt, 3),
            "cells_per_s": round(cells / dt), "kv_equivalent_gbs": round(cells * CELL / dt / 1e9, 4),
            "note": "wall time of start_migration + the event loop until the bulk patch is applied"}


def time_resize():
    n_blocks = 33344                 # the bench source store's capacity
    st = kvstore.KvStore(1, K, S, n_blocks, resident_groups={0, 1})
    for i in range(0, 240):
        st.append(f"r{i:04d}", 0, CTX, [0] * CTX)
    for i in range(0, 240, 4):
        st.free_request(f"r{i:04d}")
    t0 = time.perf_counter()
    st.compact()
    st.resize(int(n_blocks * 0.8))
    dt = time.perf_counter() - t0
    return {"blocks_from": n_blocks, "blocks_to": int(n_blocks * 0.8), "seconds": round(dt, 4)}


def time_scenario():
    sc = pipeshift.load_scenario("/root/reference/pkg/scenarios/heterogeneous_shift.yaml")
    t0 = time.perf_counter()
    pipeshift.run_scenario(sc, seed=0)
    return {"scenario": "heterogeneous_shift.yaml", "seed": 0,
            "seconds": round(time.perf_counter() - t0, 2)}


def time_simulations():
    """The golden runs of tests/golden/simulations.json on the reference (same builders
    as tests/golden/make_golden.py)."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    from pipeshift.simulation import Simulation
    from scenarios import hetero_scenario
    from test_coordinator import C_B, fig3_scenario

    runs = {"fig3_seed5": (fig3_scenario(triggers=[(0.02, C_B)], num_requests=4, rate=500.0), 5),
            "hetero_c10_seed123": (hetero_scenario(rate=7.0, n=40), 123),
            "hetero_n60_seed7": (hetero_scenario(rate=7.0, n=60), 7)}
    out = {}
    for name, (scen, seed) in runs.items():
        t0 = time.perf_counter()
        sim = Simulation(scen, seed=seed)
        sim.scheduler.run(until=600.0)
        out[name] = {"seconds": round(time.perf_counter() - t0, 3), "events": len(sim.trace)}
    return out


def main():
    cpu = ""
    try:
        cpu = next(l.split(":", 1)[1].strip() for l in
                   subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()
                   if l.startswith("Model name"))
    except Exception:
        pass
    out = {"what": "reference pipeshift (CPython, 1 thread) timed in the dev container",
           "cpu": cpu, "python": platform.python_version(), "cores_used": 1,
           "append": time_append(), "bulk_round": time_bulk_round(), "resize": time_resize(),
           "scenario": time_scenario(), "simulations": time_simulations()}
    path = ROOT / "profiles" / "reference_cpu_r1.json"
    path.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
