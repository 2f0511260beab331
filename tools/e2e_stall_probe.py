"""Probe for the intermittent host stall in bench.py's `e2e` leg: runs the e2e loop
(measure_e2e_api) repeatedly on the bench rig, alone and right after the legs that run
before it in bench.py (resize, act_hop), and prints each run's ms/step, slowest host
step and that step's phases (free / append / push / d2h).  Writes gpurun_out/e2e_stall.json.

    python tools/e2e_stall_probe.py [--steps 20] [--reps 4]
"""

import argparse
import gc
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--reps", type=int, default=4)
    args = ap.parse_args()

    import torch

    import bench
    from paper_2604_12171_b200.perf import PatchRig, Workload

    torch.cuda.set_device(0)
    wl = Workload(batch=256, ctx=2048)
    stream = torch.cuda.Stream()
    rig = PatchRig(wl, device=0)
    for i in range(wl.batch):
        rig.registry.handle(f"api{i:04d}")
    rig.use_stream(stream.cuda_stream)
    rig.fill()
    gc.collect()
    gc.freeze()
    rig.bulk_round()
    torch.cuda.synchronize()

    runs = []

    def e2e(tag):
        r = bench.measure_e2e_api(rig, stream, torch, wl, args.steps, 1)
        row = {"tag": tag, "gbs": r["value"], "ms_per_step": r["ms_per_step"],
               "host_step_ms_max": r["host_step_ms_max"], "phases": r["host_step_phases_ms"], "staging": r["staging"],
               "vmm": rig.src.vmm_stats() if hasattr(rig.src, "vmm_stats") else None}
        runs.append(row)
        print(json.dumps(row), flush=True)

    for rep in range(args.reps):
        e2e(f"alone{rep}")
    # bench.py's order: resize (drops the migrating groups once), act_hop, then e2e
    t0 = time.perf_counter()
    bench.measure_resize(rig, stream, torch, wl)
    runs.append({"tag": "resize", "ms": round((time.perf_counter() - t0) * 1e3, 1)})
    for rep in range(args.reps):
        e2e(f"after_resize{rep}")
    for rep in range(args.reps):
        bench.measure_act_hop(torch)
        e2e(f"after_act{rep}")
    os.makedirs(ROOT / "gpurun_out", exist_ok=True)
    (ROOT / "gpurun_out" / "e2e_stall.json").write_text(json.dumps(runs, indent=1))


if __name__ == "__main__":
    main()
