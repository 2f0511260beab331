#!/usr/bin/env python3
"""Benchmark of the live PP-reconfiguration data path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one KV-patch round of BASELINE configs[1] (Llama-3-8B shape, PP2->4,
16-token blocks, k=4): every live cell of the two migrating layer groups of
B=256 requests x 2048 tokens is marked dirty, drained (K3 scan/compact) and
pushed into the destination's paged pools (fused K4 gather -> K5 scatter).
`value` is KV-patch GB/s (KvPatch.payload_bytes per second, inputs resident);
`e2e` is the same round through the C-ABI with the KV arriving from pinned host
memory each step.  Extra keys report switch pause, resize latency and
paged-attention decode tokens/s.  Under torchrun every rank runs its own pair on
its own GPU (weak scaling, no data-path collective); timing is max over ranks.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import time

import numpy as np
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"]
HBM_FALLBACK_GBS = 6650.0
NVLINK_GBS = 900.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-sweep", action="store_true")
    ap.add_argument("--skip-c3", action="store_true")
    ap.add_argument("--skip-c2", action="store_true")
    ap.add_argument("--only-step", action="store_true",
                    help="time the KV-patch step only (for the ncu launch list of the step)")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--ctx", type=int, default=2048)
    return ap.parse_args()


# ------------------------------------------------------------------------------ dist
def dist_init(n: int):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    return rank, world


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------------------ clocks
class Clocks:
    """SM clock + throttle reasons sampled through NVML every 5 ms while the timed
    region runs (a thread; nvidia-smi's startup is longer than a short timed region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None
        self._stop = None
        self._th = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return self
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                         pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
                except Exception:
                    pass
                self._stop.wait(0.005)

        self._th = threading.Thread(target=run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        if self._th is not None:
            self._stop.set()
            self._th.join()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"],
                    "samples": 0}
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(m for m, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml"}


# ------------------------------------------------------------------------------ CPU legs
def cpu_patch_rate(wl, seconds: float = 12.0, n_req: int = 8) -> dict:
    """The oracle PORT (oracle/oracle.c, the reference's _drain + PatchReceiver._apply
    restated in C, moving real KV bytes) on all host cores: KV-patch GB/s of a bounded
    sample of the same workload (n_req requests x ctx tokens x the migrating groups).
    Reported as `cpu_baseline_port`, beside the reference itself."""
    import numpy as np

    import oracle
    from paper_2604_12171_b200.events import stable_hash

    threads = os.cpu_count() or 1
    blocks = n_req * wl.blocks_per_req + 8
    G = len(wl.src_groups)
    src = oracle.OracleStore(1, wl.k, wl.s, blocks, wl.src_groups, num_groups=G,
                             cell_bytes=wl.cell_bytes)
    dst = oracle.OracleStore(2, wl.k, wl.s, blocks, wl.mig_groups, num_groups=G,
                             cell_bytes=wl.cell_bytes)
    for i in range(n_req):
        for g in wl.mig_groups:
            seed = stable_hash(f"r{i:04d}", g)
            src.append(f"r{i:04d}", g, wl.ctx, [oracle.payload(seed, p) for p in range(wl.ctx)])
    dirty = oracle.OracleDirty()
    rank = src.reg.rank()
    sample_bytes = n_req * wl.ctx * len(wl.mig_groups) * wl.k * wl.cell_bytes
    rounds, t_total = 0, 0.0
    while t_total < seconds or rounds < 2:
        t0 = time.perf_counter()
        for i in range(n_req):
            h = src.reg.handle(f"r{i:04d}")
            for g in wl.mig_groups:
                dirty.mark(h, g, 0, wl.ctx)
        keys, cells = dirty.patch_round(src, dst, rank, wl.k, threads)
        t_total += time.perf_counter() - t0
        rounds += 1
        assert keys == n_req * wl.ctx * len(wl.mig_groups)
    gbs = sample_bytes * rounds / t_total / 1e9
    return {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"{rounds} rounds x {n_req} requests x {wl.ctx} tokens x "
                      f"{len(wl.mig_groups)} groups x k={wl.k} x {wl.cell_bytes} B "
                      f"({sample_bytes / 1e9:.2f} GB/round), oracle/oracle.c with {threads} threads",
            "seconds": round(t_total, 2)}


REF_SAMPLE_REQS = 64   # requests per reference step: 1/4 of the B = 256 workload


def reference_rate(wl, steps: int, warmup: int, n_req: int = REF_SAMPLE_REQS) -> dict:
    """The reference itself (pipeshift from oracle/_ref, staged by oracle/reference.py's
    recipe) on the host: each step is one bulk KV-patch round of the bench pair --
    MigrationManager.start_migration + the event loop until the patch is applied
    (migrator.py:170-273, 93-132) -- over a bounded sample of the workload (n_req of the
    B requests x ctx tokens, groups 2-3 of 0-3, k = 4).  CPython is single-threaded: 1
    core.  The reference moves 8-byte fingerprints per cell; GB/s is KV-equivalent
    (cells x 4096 B), the unit of our arm."""
    from oracle import reference as R

    assert (wl.ctx, wl.k, wl.s, wl.cell_bytes) == (R.CTX, R.K, R.S, R.CELL)
    rnd = R.BulkRound(n_req)
    for _ in range(warmup):
        rnd.run()
    secs = [rnd.run() for _ in range(steps)]
    total = sum(secs)
    gbs = rnd.cells * R.CELL * steps / total / 1e9
    return {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "reference",
            "sample": f"{n_req} of the {wl.batch} requests per step ({n_req} x {wl.ctx} tokens x "
                      f"{len(wl.mig_groups)} groups x k={wl.k} = {rnd.cells} cells, "
                      f"{rnd.cells * R.CELL / 1e9:.2f} GB KV-equivalent); pipeshift (oracle/_ref), "
                      f"CPython 1 thread; the reference moves 8-B fingerprints, bytes are "
                      f"KV-equivalent (cells x {R.CELL} B)",
            "steps": steps, "seconds": round(total, 2),
            "ms_per_step_sample": round(total / steps * 1e3, 2),
            "sample_bytes": int(rnd.cells * R.CELL),
            "host": R.host_info()}


def run_reference(args, wl, rank: int, world: int) -> None:
    if rank != 0:
        return
    K, W = args.steps, args.warmup
    from oracle import reference as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not staged (run "
                          "__graft_entry__.build() in the dev container)"}), flush=True)
        return
    cb = reference_rate(wl, K, W)
    extras = {"append": R.time_append(16), "compact_resize": R.time_resize(),
              # the steady patch rounds and the full packaged scenario too
              "steady_round": R.time_steady(64, 20), "scenario": R.time_scenario()}
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "GB/s",
        "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": cb["ms_per_step_sample"],
        # the rate is measured on a bounded sample of the step's workload (cpu_baseline.sample):
        # ms_per_step is the sample's, and these are the bytes it moved
        "sample_bytes_per_step": cb.get("sample_bytes"),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic", "config": config_of(wl, world),
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_extras": extras,
    }
    print(json.dumps(line), flush=True)


def guarded(name: str, fn):
    """Run one extra measurement; a failure (e.g. a smaller GPU out of memory for the C3
    fill) is recorded in the line instead of losing the whole bench line."""
    try:
        return fn()
    except Exception as e:  # noqa: BLE001 - reported, not swallowed
        import traceback
        traceback.print_exc(file=sys.stderr)
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def profile_traffic(kernel: str, n_q: int | None = None, wl=None):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` at this bench's
    shape, from the committed ncu capture (profiles/traffic_r2.json, tools/gpu_r2.sh; r1 before it existed);
    None when the run's shape is not the captured one (B = 256, ctx = 2048)."""
    if wl is not None and (wl.batch, wl.ctx) != (256, 2048):
        return None
    path = ROOT / "profiles" / "traffic_r2.json"
    if not path.exists():
        path = ROOT / "profiles" / "traffic_r1.json"
    try:
        rows = json.loads(path.read_text())
    except Exception:
        return None
    for r in rows:
        if r.get("kernel") == kernel and r.get("n_q") == n_q:
            return r.get("dram_bytes")
    return None


def config_of(wl, world: int) -> dict:
    name = wl.name if (wl.batch, wl.ctx) == (256, 2048) else \
        f"llama3-8b PP2->4: one migrating pair (layers 9-16), B={wl.batch}, ctx={wl.ctx}"
    return {"workload": name, "model_shape": "llama-3-8b (32L, 32q/8kv x 128, bf16)",
            "pp_change": "2->4", "migrating_layers": "9-16 (groups 2,3)",
            "stacking_k": wl.k, "tokens_per_block": wl.s, "batch": wl.batch, "ctx": wl.ctx,
            "kv_bytes_per_token_layer": wl.cell_bytes,
            "bytes_per_step": wl.payload_bytes,
            "l2": f"inputs ({wl.payload_bytes / 1e9:.1f} GB per step) exceed the 126 MB L2; "
                  "no flush needed",
            "parallelism": (f"ring of {world} cross-process pairs (rank r -> r+1, one per GPU)"
                            if world > 1 else "1 pair on one GPU")}


# ------------------------------------------------------------------------------ GPU legs
def main() -> None:
    args = parse()
    rank, world = dist_init(args.gpus)
    from paper_2604_12171_b200.perf import Workload

    wl = Workload(batch=args.batch, ctx=args.ctx)
    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return

    import torch

    from paper_2604_12171_b200 import _native as N
    from paper_2604_12171_b200.perf import PatchRig, read_peaks

    dev = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    lib = N.lib()
    peaks = read_peaks(ROOT / "MEASURED_PEAKS.json")
    hbm_peak = float(peaks.get("hbm_gbs", HBM_FALLBACK_GBS))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"

    # ---- C3 first, on a clean GPU: 70B-shape stage with HBM pre-filled by KV (~160 GB
    # peak), live shrink with K6 relocation, patch of the leaving groups, drop, grow
    shared_gpu = world > max(torch.cuda.device_count(), 1) and not args.only_step
    if shared_gpu:
        # ranks sharing a GPU (a one-GPU box under torchrun): the legs sized for a whole
        # GPU's HBM (configs[2]'s 160 GB pre-fill, the 8B-shape decoders) cannot fit N times
        # over, so the line is the bulk round and the e2e round (the ring's), as
        # `--only-step` plus e2e
        args.only_step = True
        if rank == 0:
            print(f"[bench] {world} ranks on {torch.cuda.device_count()} GPU(s): bulk round "
                  "+ e2e only", file=sys.stderr)
    if args.only_step:
        skip_e2e = args.skip_e2e
        args.skip_c3 = args.skip_c2 = args.skip_sweep = args.skip_e2e = args.skip_cpu = True
        if shared_gpu:
            args.skip_e2e = skip_e2e
    c3 = None
    if not args.skip_c3 and rank == 0:
        from paper_2604_12171_b200.perf import c3_live_resize
        c3 = guarded("c3_live_resize", lambda: c3_live_resize(dev))
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    barrier(world)

    stream = torch.cuda.Stream(device=dev)
    rig = PatchRig(wl, device=dev)
    # the e2e requests get their handles now, in the same order on every rank: across a
    # cross-process pair the rows carry the sender's handles and the receiver frees by its
    # own, so both registries must agree (later rank-0-only legs register other names)
    for i in range(wl.batch):
        rig.registry.handle(f"api{i:04d}")
    rig.use_stream(stream.cuda_stream)
    rig.fill()
    # the host block manager's mirror is millions of small objects: collect once and freeze
    # them, so a cyclic-GC pass cannot land inside a wall-clock measurement below
    gc.collect()
    gc.freeze()
    K, W = args.steps, args.warmup
    # N > 1: a ring of cross-process pairs, rank r -> r+1 over the imported peer pools
    # (NVLink stores); N = 1: the pair's destination is a second store on this GPU
    ring = None
    if world > 1:
        from paper_2604_12171_b200.dist import RingPair
        ring = RingPair(rig, rank, world, f"bench-{os.environ.get('MASTER_PORT', '0')}")
        ring.use_stream(stream.cuda_stream)
    stepper = ring if ring is not None else rig

    # ---- value_cold: the first bulk round of a reconfiguration, into a destination with no
    # chains yet (the receiver reserves every block on the host while the copy runs).  As in
    # the reference's Phase 3 (coordinator.py:203-230) the destination's incoming groups are
    # mapped before StartKVMigration: the wait for the background mapping is reported apart
    tm0 = time.perf_counter()
    map_wait_ms = rig.dst.prepare_wait() if ring is None else 0.0
    map_wait_ms = (time.perf_counter() - tm0) * 1e3
    torch.cuda.synchronize()
    tc0 = time.perf_counter()
    cold_keys, _ = stepper.bulk_round()
    torch.cuda.synchronize()
    cold_ms = allmax((time.perf_counter() - tc0) * 1e3, world)
    assert cold_keys == wl.batch * wl.ctx * len(wl.mig_groups)
    value_cold = {"value": round(world * wl.payload_bytes / (cold_ms / 1e3) / 1e9, 2),
                  "unit": "GB/s", "ms": round(cold_ms, 3),
                  "phase3_map_wait_ms": round(map_wait_ms, 3),
                  "note": "first bulk round into empty destination chains (wall clock: seed, "
                          "host block reservation pipelined with K3 + push); the incoming "
                          "groups' pools are mapped first (Phase 3, phase3_map_wait_ms); "
                          "`value` is the warm re-push"}

    # ---- value: bulk KV-patch rounds, everything resident in HBM
    for _ in range(W):
        stepper.bulk_round()
    torch.cuda.synchronize()
    N.check(lib.pl_timing_reset())
    N.check(lib.pl_timing_enable(1))
    barrier(world)
    launches0 = N.launch_count()
    with Clocks(dev) as clocks:
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        keys_total = 0
        for _ in range(K):
            keys, cells = stepper.bulk_round()
            keys_total += keys
        t1.record(stream)
        torch.cuda.synchronize()
    launches = N.launch_count() - launches0
    N.check(lib.pl_timing_enable(0))
    ms = t0.elapsed_time(t1)
    ms = allmax(ms, world)
    barrier(world)
    assert keys_total == K * wl.batch * wl.ctx * len(wl.mig_groups)
    value = world * K * wl.payload_bytes / (ms / 1e3) / 1e9
    push_ms, push_n = N.timing("patch_push")
    drain_ms, drain_n = N.timing("drain")
    push_avg = push_ms / max(push_n, 1)
    if ring is None:
        # algorithmic HBM bytes of one push launch: payload read + write + 2 x 8 B fp
        alg_bytes = 2 * wl.payload_bytes + 2 * 8 * wl.batch * wl.ctx * len(wl.mig_groups)
        bound, peak, psrc, traffic = "hbm", hbm_peak, peak_src, profile_traffic("push_batched_kernel", None, wl)
    elif world <= torch.cuda.device_count():
        # bytes each GPU sends over NVLink per launch (it receives as many concurrently)
        alg_bytes = wl.payload_bytes + 8 * wl.batch * wl.ctx * len(wl.mig_groups)
        bound, peak, psrc, traffic = "nvlink", NVLINK_GBS, "nominal 900 GB/s per direction", None
    else:
        # ranks share a GPU (functional run of the ring on a smaller box): HBM-bound
        alg_bytes = 2 * wl.payload_bytes + 2 * 8 * wl.batch * wl.ctx * len(wl.mig_groups)
        bound, peak, psrc, traffic = "hbm (ranks share one GPU)", hbm_peak, peak_src, None
    achieved = alg_bytes / (push_avg / 1e3) / 1e9
    roofline = {"kernel": "push_batched_kernel (K4 gather -> K5 scatter fused, batched resolve)",
                "bound": bound, "achieved": round(achieved, 1), "peak": peak,
                "peak_source": psrc, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "alg_bytes_per_launch": alg_bytes,
                "avg_launch_ms": round(push_avg, 4),
                "share_of_step": round(push_ms / ms, 4) if ms else None,
                "drain_ms_per_step": round(drain_ms / max(K, 1), 4)}

    pause = c2 = decode = decode_70b = wstage = resize = act_hop = None
    if not args.only_step:
        # ---- switch pause (data-path part): residual patch after one decode round + barrier
        pause = guarded("switch_pause", lambda: measure_switch_pause(rig, stream, torch, wl))

        # ---- C2 timeline: live migration on a side stream under steady decode
        if not args.skip_c2:
            from paper_2604_12171_b200.perf import c2_live
            c2 = guarded("c2_live", lambda: c2_live(rig, stream))

        # ---- paged-attention decode over the source stage (16 layers): the 8B shape
        # (GQA 4) and the 70B shape (64 q heads over the same 8 KV heads x 128, GQA 8)
        decode = guarded("decode", lambda: measure_decode(rig, stream, torch, wl, hbm_peak, K, W))
        decode_70b = guarded("decode_70b", lambda: measure_decode(rig, stream, torch, wl, hbm_peak,
                                                                     K, W, n_q=64))

        # ---- AddLayerWeights on the copy engine: the 8 migrating layers' weights
        wstage = guarded("weight_stage", lambda: measure_weight_stage(rig, stream, torch, wl, dev))

        # ---- resize latency: post-commit cleanup on the source (drop, shrink, regrow)
        resize = guarded("resize", lambda: measure_resize(rig, stream, torch, wl))

        # ---- K7 activation hop through the stage ring
        act_hop = guarded("act_hop", lambda: measure_act_hop(torch))

    # ---- e2e: KV arrives from pinned host memory every step, result read back
    e2e = e2e_kv = None
    if not args.skip_e2e:
        e2e = guarded("e2e", lambda: measure_e2e_api(rig, stream, torch, wl, K, world, ring))
        if e2e and "ms_per_step" in e2e:
            # the step's device work is three passes over the payload: K1 writes the cells,
            # the push reads and writes them -- the HBM bound of the whole e2e step
            # (ranks sharing one GPU share its HBM: their bytes add up on it)
            per_gpu = world // max(torch.cuda.device_count(), 1) if shared_gpu else 1
            e2e["hbm_bytes_per_step"] = 3 * wl.payload_bytes * per_gpu
            e2e["hbm_bound_ms"] = round(3 * wl.payload_bytes * per_gpu / (hbm_peak * 1e9) * 1e3, 3)
            e2e["hbm_frac"] = round(e2e["hbm_bound_ms"] / e2e["ms_per_step"], 4)
    if ring is not None:
        ring.close()
    if not args.skip_e2e and not shared_gpu:
        # a heavier variant: the real 17 GB of KV bytes stream from pinned host memory
        e2e_kv = guarded("e2e_real_kv", lambda: measure_e2e(rig, stream, torch, wl, K, world))
    rig.destroy()
    if ring is not None:
        ring.dst.close()

    # ---- configs[1] live with real stage compute: the 8B-shaped decoder (bf16 GEMMs, K1/K2
    # over the stage stores) under a PP 2 -> 4 reconfiguration switched by the reference's
    # lag < tau test, against a static run (tokens must be equal)
    c2_model = c4_model = None
    if not args.skip_c2 and rank == 0:
        c2_model = guarded("c2_model", lambda: measure_c2_model(wl))
        c4_model = guarded("c4_model", lambda: measure_c4_model(wl))

    # ---- C5: dirty-rate x block-size sweep and concurrent pairs (configs[4], 1 GPU); after
    # the e2e legs, so their store churn (dozens of pools created and released) cannot
    # overlap the headline measurement
    sweep = pairs = None
    if not args.skip_sweep and rank == 0:
        from paper_2604_12171_b200.perf import c5_sweep
        sweep = guarded("c5_sweep", lambda: c5_sweep(dev))
        from paper_2604_12171_b200.perf import c5_pairs
        pairs = guarded("c5_pairs", lambda: c5_pairs(dev))

    if rank != 0:
        return
    cpu = cpu_port = None
    if not args.skip_cpu:
        from oracle import reference as R
        # the reference itself (pipeshift, 1 core) ~15 s, and the 16-thread C port beside it
        cpu = guarded("cpu_baseline", lambda: reference_rate(wl, 10, 1)) if R.available() else None
        cpu_port = guarded("cpu_baseline_port", lambda: cpu_patch_rate(wl))
    # the driver keeps the TAIL of stdout: the bulky per-point sweeps go first, the headline
    # extras (decode, pause, live timeline, resize incl. background mapping) last
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(ms / K, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": config_of(wl, world),
        "c5_sweep": sweep,
        "c5_pairs": pairs,
        "e2e_real_kv_from_host": e2e_kv,
        "weight_stage": wstage,
        "c3_live_resize": c3,
        "c2_live": c2,
        "c2_model": c2_model,
        "c4_model": c4_model,
        "resize": resize,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "cpu_baseline_port": cpu_port,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "value_cold": value_cold,
        "switch_pause_ms": pause,
        "act_hop": act_hop,
        "decode": decode,
        "decode_70b_shape": decode_70b,
        "tail": tail_summary(c2_model, c3, resize, decode, decode_70b, pause, value_cold,
                             hbm_peak, act_hop, sweep, c4_model),
    }
    print(json.dumps(line), flush=True)


def tail_summary(c2, c3, resize, decode, decode_70b, pause, value_cold, hbm_peak,
                 act_hop=None, sweep=None, c4=None) -> dict:
    """The headline extras in one small object at the very end of the line."""
    def get(d, *path):
        for p in path:
            if not isinstance(d, dict) or p not in d:
                return None
            d = d[p]
        return d

    out = {"value_cold_gbs": get(value_cold, "value"),
           "decode_8b": {"tokens_per_s": get(decode, "tokens_per_s"),
                         "hbm_frac": get(decode, "roofline", "frac")},
           "decode_70b_shape": {"tokens_per_s": get(decode_70b, "tokens_per_s"),
                                "hbm_frac": get(decode_70b, "roofline", "frac")},
           "switch_pause_data_path_ms": get(pause, "median"),
           "act_hop_us": {k: get(act_hop, k, "us_per_hop") for k in ("8b", "70b")}}
    if isinstance(sweep, list):
        # steady rounds of the C5 sweep at 16-token blocks: wall vs kernel time
        # (hbm_frac: the round's kernels' algorithmic HBM bytes -- payload read + write --
        # per kernel second, over the measured copy peak)
        out["c5_steady_16tok"] = {
            r["dirty"]: {"wall_us": round(r["ms"] * 1e3, 1),
                         "kernel_us": round(r["kernel_ms"] * 1e3, 1),
                         "hbm_frac": round(r["kernel_hbm_gbs"] / hbm_peak, 3)
                         if r.get("kernel_hbm_gbs") else None}
            for r in sweep if r.get("tokens_per_block") == 16}
    if isinstance(c2, dict) and "error" not in c2:
        out["c2_model_8b_live"] = {k: c2.get(k) for k in (
            "tokens_equal_static", "tpot_ms_static", "tpot_ms_before", "tpot_ms_during",
            "tpot_ms_after", "switch_step", "pause") if k in c2}
        out["c2_model_8b_live"]["bulk_gbs"] = get(c2, "bulk", "gbs")
    if isinstance(c4, dict) and "error" not in c4:
        out["c4_model_8b_uneven"] = {k: c4.get(k) for k in (
            "tokens_equal_static", "tpot_ms_static", "tpot_ms_before", "tpot_ms_during",
            "tpot_ms_after", "switch_step", "pause") if k in c4}
        out["c4_model_8b_uneven"]["bulk_gbs"] = get(c4, "bulk", "gbs")
    if isinstance(resize, dict) and "error" not in resize:
        out["resize_full_ms"] = {k: resize.get(k) for k in (
            "drop_groups_full_ms", "shrink_full_ms", "grow_warm_full_ms", "grow_cold_full_ms")}
        out["resize_critical_path_ms"] = {k: resize.get(k) for k in (
            "drop_groups_ms", "shrink_ms", "grow_warm_ms", "grow_cold_ms")}
    if isinstance(c3, dict) and "error" not in c3:
        out["c3_70b"] = {k: c3.get(k) for k in (
            "phase2_shrink_full_ms", "map_incoming_group_full_ms", "grow_full_ms",
            "phase2_shrink_ms", "map_incoming_group_ms", "grow_ms")}
        out["c3_70b"]["bulk_patch_gbs"] = get(c3, "bulk_patch", "gbs")
    return out


def measure_c2_model(wl, steps: int = 40, reconfig_at: int = 8, run_dir: str | None = None) -> dict:
    """BASELINE configs[1] with the 8B-shaped decoder (paper_2604_12171_b200/model8b.py):
    B = 256 requests at 2048 prefilled positions decode greedily for `steps` steps; the
    live run starts the PP 2 -> 4 reconfiguration (layers 9-16: GPU 1 -> 3, 25-32: 2 -> 4)
    after step `reconfig_at` and switches at the first per-step poll with lag < tau = 50
    cells.  TPOT = wall ms per decode step (one token for every request), before / while
    migrating / after the switch, and for the static run; the pause split into draining
    the in-flight step, the residual round, and barrier + switch."""
    import gc

    import torch

    from paper_2604_12171_b200.engine import compute_metrics
    from paper_2604_12171_b200.events import EventTrace
    from paper_2604_12171_b200.model8b import run_live, summarize

    gc.collect()
    torch.cuda.empty_cache()
    kw = dict(batch=wl.batch, ctx=wl.ctx, steps=steps, reconfig_at=reconfig_at)
    static = run_live(live=False, **kw)
    tr = EventTrace()
    live = run_live(live=True, trace=tr, **kw)
    s = summarize(live, static)
    s["trace_metrics"] = compute_metrics(tr).as_row()   # reference schema (engine.py:112-184)
    if run_dir:   # trace.jsonl / metrics.csv / summary.json in the reference runner's schema
        from paper_2604_12171_b200 import outputs
        outputs.write_run(run_dir, tr, "configs[1]:pp2->pp4 (8B shape)", 0, mode="perf", stages=4)
    c = s.pop("commit") or {}
    s["pause"] = {k: c.get(k) for k in ("pause_ms", "drain_ms", "residual_ms",
                                        "barrier_and_switch_ms", "residual_cells", "lag_at_poll")}
    s["lag_polls"] = s["lag_polls"][:12]
    s["note"] = ("all 4 stage stores on one GPU (distinct on hardware); bf16 GEMMs via cuBLAS, "
                 "K1 + K2 + the patch engine are this repo's kernels; patch rounds on a "
                 "lowest-priority side stream; TPOT includes the greedy token read-back")
    return s


def measure_c4_model(wl, steps: int = 40, reconfig_at: int = 8, run_dir: str | None = None) -> dict:
    """BASELINE configs[3] with the 8B-shaped decoder: 8 stage stores (one GPU here, one GPU
    each on hardware), an even split (4 layers per stage, k = 2) re-split live into the
    generation-heavy uneven split 2/4/4/6/6/4/4/2 -- six pairs migrate at once, stages 2, 3,
    6, 7 both send and receive -- under decode at B requests x ctx prefilled positions;
    switch at the first per-step poll with lag < tau = 50.  TPOT before / while migrating /
    after, the pause split, and the tokens against the static run.  (TTFT needs prefill,
    which this decode-only stage model does not run; configs[3]'s TTFT/TPOT trace metrics
    come from the 8-process tiny-model run, tools/c4_live.py.)"""
    import gc

    import torch

    from paper_2604_12171_b200.engine import compute_metrics
    from paper_2604_12171_b200.events import EventTrace
    from paper_2604_12171_b200.model8b import EVEN8, UNEVEN8, run_live, summarize

    gc.collect()
    torch.cuda.empty_cache()
    kw = dict(batch=wl.batch, ctx=wl.ctx, steps=steps, reconfig_at=reconfig_at, src=EVEN8,
              dst=UNEVEN8, k=2)
    static = run_live(live=False, **kw)
    tr = EventTrace()
    live = run_live(live=True, trace=tr, **kw)
    s = summarize(live, static)
    s["trace_metrics"] = compute_metrics(tr).as_row()   # reference schema (engine.py:112-184)
    if run_dir:   # trace.jsonl / metrics.csv / summary.json in the reference runner's schema
        from paper_2604_12171_b200 import outputs
        outputs.write_run(run_dir, tr, "configs[3]:even8->uneven8 (8B shape)", 0, mode="perf",
                          stages=8)
    c = s.pop("commit") or {}
    s["pause"] = {k: c.get(k) for k in ("pause_ms", "drain_ms", "residual_ms",
                                        "barrier_and_switch_ms", "residual_cells", "lag_at_poll")}
    s["lag_polls"] = s["lag_polls"][:12]
    s["split"] = {"from": [len(v) for _, v in sorted(EVEN8.items())],
                  "to": [len(v) for _, v in sorted(UNEVEN8.items())], "k": 2}
    s["note"] = ("8 stage stores on one GPU (distinct on hardware); bf16 GEMMs via cuBLAS, "
                 "K1 + K2 + the patch engine are this repo's kernels; six pairs patch on one "
                 "lowest-priority side stream; TPOT includes the greedy token read-back")
    torch.cuda.empty_cache()
    return s


def measure_act_hop(torch, hops: int = 200) -> dict:
    """K7: one stage-to-stage activation hop through an activation ring (csrc/act.cu) at
    decode batch B = 256: 2 MiB (8B shape, d = 4096 bf16) and 4 MiB (70B shape, d = 8192).
    Here both stages are in this process on one GPU, so a hop is two HBM copies (into the
    receiver's slot, out of it); across GPUs the first one is an NVLink write.  Device time
    from the first send to the last receive (events), and the host time per send + recv."""
    from paper_2604_12171_b200.dist import ActRing

    out = {}
    for name, d in (("8b", 4096), ("70b", 8192)):
        nbytes = 256 * d * 2
        owner = ActRing.create(torch.cuda.current_device(), nbytes, n_slots=4)
        tx = ActRing.open(torch.cuda.current_device(), owner.export())
        a, b = torch.cuda.Stream(), torch.cuda.Stream()
        x = torch.randn(256, d, device="cuda").to(torch.bfloat16)
        y = torch.empty_like(x)
        torch.cuda.synchronize()
        for _ in range(8):
            tx.send(x, a.cuda_stream)
            owner.recv(y, b.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(a)
        t0 = time.perf_counter()
        for _ in range(hops):
            tx.send(x, a.cuda_stream)
            owner.recv(y, b.cuda_stream)
        host_us = (time.perf_counter() - t0) / hops * 1e6
        e1.record(b)
        torch.cuda.synchronize()
        assert torch.equal(x, y)
        us = e0.elapsed_time(e1) * 1e3 / hops
        out[name] = {"bytes": nbytes, "us_per_hop": round(us, 2),
                     "gbs": round(nbytes / us / 1e3, 1),
                     "hbm_gbs": round(4 * nbytes / us / 1e3, 1),
                     "host_us_per_hop": round(host_us, 2)}
        tx.close()
        owner.close()
    out["note"] = ("one process, one GPU: hop = copy into the receiver's slot + copy out "
                   "(hbm_gbs counts both copies' read + write); the stages' streams are "
                   "ordered by interprocess events, no host sync")
    return out


def measure_switch_pause(rig, stream, torch, wl) -> dict:
    """After the bulk copy converged: one decode round writes B tokens into every
    group (K1 fused with the dirty mark), then the switch: pause -> drain the
    compute stream -> final residual patch -> barrier -> switch -> resume."""
    from paper_2604_12171_b200 import _native as N
    from paper_2604_12171_b200.perf import append_batch
    from paper_2604_12171_b200.events import stable_hash

    rig.bulk_round()
    torch.cuda.synchronize()
    reqs, groups, counts, seeds = [], [], [], []
    for i, h in enumerate(rig.handles):
        for g in wl.src_groups:
            reqs.append(h)
            groups.append(g)
            counts.append(1)
            seeds.append(stable_hash(f"r{i:04d}", g))
    samples = []
    for _ in range(5):
        append_batch(rig.src, reqs, groups, counts, seeds, mark=True)
        t0 = time.perf_counter()          # pause_admission
        stream.synchronize()              # pipeline drained (in-flight writes done)
        keys, cells = rig.patch.push(rig.dst, rig.registry.rank())   # final sync
        stream.synchronize()              # barrier: residual applied on the destination
        samples.append((time.perf_counter() - t0) * 1e3)
        assert keys == wl.batch * len(wl.mig_groups)
    return {"median": round(statistics.median(samples), 4), "max": round(max(samples), 4),
            "residual_cells": wl.batch * len(wl.mig_groups) * wl.k,
            "residual_bytes": wl.batch * len(wl.mig_groups) * wl.k * wl.cell_bytes,
            "note": "data-path part of the pause (drain of queued writes + residual patch + "
                    "barrier); excludes pipeline drain of model compute"}


def measure_decode(rig, stream, torch, wl, hbm_peak, K, W, n_q=None) -> dict:
    import ctypes as C

    from paper_2604_12171_b200 import _native as N

    lib = N.lib()
    B = wl.batch
    n_q = n_q or wl.n_q
    rows = torch.tensor(rig.handles, dtype=torch.int32, device="cuda")
    ctx_now = wl.ctx
    ctx = torch.full((B,), ctx_now, dtype=torch.int32, device="cuda")
    q = torch.randn(B, n_q, wl.head_dim, dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(q)
    torch.cuda.synchronize()   # q/rows/ctx come from torch's stream; decode runs on `stream`
    layers = [(g, j) for g in wl.src_groups for j in range(wl.k)]

    def step():
        for g, j in layers:
            N.check(lib.pl_paged_attn_decode(rig.src._h, g, j, C.c_void_p(q.data_ptr()),
                                             C.c_void_p(out.data_ptr()),
                                             C.c_void_p(rows.data_ptr()),
                                             C.c_void_p(ctx.data_ptr()), B, n_q, wl.n_kv,
                                             wl.head_dim, wl.head_dim ** -0.5, ctx_now,
                                             C.c_void_p(stream.cuda_stream)))

    for _ in range(W):
        step()
    torch.cuda.synchronize()
    N.check(lib.pl_timing_reset())
    N.check(lib.pl_timing_enable(1))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(K):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    N.check(lib.pl_timing_enable(0))
    ms = e0.elapsed_time(e1) / K
    attn_ms, attn_n = N.timing("paged_attn")
    per_launch = attn_ms / max(attn_n, 1)
    kv_bytes_layer = B * ctx_now * wl.cell_bytes
    q_bytes = 2 * B * n_q * wl.head_dim * 2
    achieved = (kv_bytes_layer + q_bytes) / (per_launch / 1e3) / 1e9
    return {"tokens_per_s": round(B / (ms / 1e3), 1), "ms_per_step": round(ms, 4),
            "layers_per_step": len(layers), "batch": B, "ctx": ctx_now, "n_q": n_q,
            "n_kv": wl.n_kv, "head_dim": wl.head_dim,
            "roofline": {"kernel": "paged_attn_mma_kernel<128,8> (TMA 128B-swizzled ring, "
                                   "mma.sync bf16, +combine)", "bound": "hbm",
                         "traffic": profile_traffic("paged_attn_mma", n_q, wl),
                         "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(achieved / hbm_peak, 4),
                         "alg_bytes_per_launch": kv_bytes_layer + q_bytes,
                         "avg_launch_ms": round(per_launch, 4)}}


def measure_weight_stage(rig, stream, torch, wl, dev) -> dict:
    """Stage the weights of the migrating layers (8 x 0.436 GB for the 8B shape, SURVEY
    §8 sizes) from pinned host memory on the low-priority copy stream, alone and while
    the stage keeps decoding on its compute stream (inference must not yield)."""
    from paper_2604_12171_b200.staging import LayerWeightStager

    layer_bytes = 436 * 1000 * 1000
    n_layers = len(wl.mig_groups) * wl.k
    host = {l: {"w": torch.empty(layer_bytes, dtype=torch.uint8, pin_memory=True)}
            for l in range(n_layers)}
    for l in host:
        host[l]["w"].fill_(l)
    st = LayerWeightStager(dev, host)
    st.stage_layers(range(n_layers))   # warm-up: device buffers allocated once
    st.wait()
    st.evict_layers(range(n_layers))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.stage_layers(range(n_layers))
    st.wait()
    ms_alone = (time.perf_counter() - t0) * 1e3
    st.evict_layers(range(n_layers))
    torch.cuda.synchronize()
    # decode alone vs decode while staging
    dec = lambda: measure_decode(rig, stream, torch, wl, 1.0, 5, 1)["ms_per_step"]  # noqa: E731
    d_alone = dec()
    t0 = time.perf_counter()
    st.stage_layers(range(n_layers))
    d_during = dec()
    still = st.staging_active()
    st.wait()
    ms_overlap = (time.perf_counter() - t0) * 1e3
    st.evict_layers(range(n_layers))
    total = n_layers * layer_bytes
    return {"layers": n_layers, "bytes": total, "ms": round(ms_alone, 2),
            "gbs": round(total / ms_alone / 1e6, 2),
            "decode_ms_per_step_alone": d_alone, "decode_ms_per_step_during_stage": d_during,
            "stage_ms_with_decode": round(ms_overlap, 2), "stage_still_running_after_decode": still,
            "note": "pinned host -> HBM, cudaMemcpyAsync in 64 MiB chunks on a lowest-priority "
                    "stream (copy engine); decode runs on its own stream"}


def measure_e2e_api(rig, stream, torch, wl, K, world, ring=None) -> dict:
    """The bulk round through the reference-facing call shape with host buffers: every
    step the B requests' migrating groups are appended with host payload arrays
    (KvStore.append(rid, group, n, payloads), kvstore.py:163-199, batched into one
    pl_store_append_batch_payloads: one H2D of the fingerprints, K1 expands them into the
    cells and sets the dirty bits), then drained and pushed (MigrationStream pump ->
    PatchReceiver, one pl_patch_push), and the device's drained-key count is read back
    (D2H, asynchronously: the host prepares step i+1 while the device runs step i).
    Timed wall-clock over K steps, host<->device copies included; every step's result
    is checked after the final sync."""
    from paper_2604_12171_b200.events import stable_hash
    from paper_2604_12171_b200.perf import append_batch_payloads, engine_payloads

    names = [f"api{i:04d}" for i in range(wl.batch)]
    handles = [rig.registry.handle(n) for n in names]
    reqs = [h for h in handles for _ in wl.mig_groups]
    groups = [g for _ in handles for g in wl.mig_groups]
    counts = [wl.ctx] * len(reqs)
    host = np.concatenate([engine_payloads(stable_hash(n, g), wl.ctx) for n in names
                           for g in wl.mig_groups])
    results = torch.zeros(K + 1, dtype=torch.int64, pin_memory=True)

    # N > 1: the round is the ring's cross-process one (rank r -> r + 1 over the imported
    # peer pools), as for `value`; the receiving store is ring.dst
    recv_store = ring.dst if ring is not None else rig.dst
    sender = ring.tx.patch if ring is not None else rig.patch

    phases = []   # host ms per step: free, append (H2D + K1), push, D2H enqueue
    # the receiving stage's host work runs on its own thread, as it would in its own
    # process on its own GPU (ctypes drops the GIL for the call; the two stores share no
    # host state); joined before the push, which reserves on the receiver
    from concurrent.futures import ThreadPoolExecutor
    receiver = ThreadPoolExecutor(max_workers=1)

    def one_step(i):
        p0 = time.perf_counter()
        # the previous step's requests leave both stages
        recv_free = receiver.submit(recv_store.free_requests, names)
        rig.src.free_requests(names)
        p1 = time.perf_counter()
        assert append_batch_payloads(rig.src, reqs, groups, counts, host, mark=True) == len(reqs)
        recv_free.result()
        p2 = time.perf_counter()
        if ring is None:
            keys, _ = rig.patch.push(rig.dst, rig.registry.rank())
        else:
            ring.tx.begin()
            ring.rx.serve_rows()
            keys, _ = ring.tx.finish()
            ring.rx.serve_ack()
        p3 = time.perf_counter()
        # D2H of the step's result (drained-key count), enqueued behind the push; the host
        # goes on preparing the next step while the device works (a pipelined driver)
        N.check(N.lib().pl_patch_device_drained_async(
            sender.h, C.c_void_p(results.data_ptr() + 8 * i)))
        phases.append((p1 - p0, p2 - p1, p3 - p2, time.perf_counter() - p3))
        return keys

    import ctypes as C

    from paper_2604_12171_b200 import _native as N
    if ring is not None:
        N.check(N.lib().pl_patch_set_active(rig.patch.h, 0))   # only the ring pair marks
    for i in range(wl.batch):   # room: the bulk requests leave both stages
        # MigrationStream.on_request_freed (migrator.py:199-204): writes still marked for a
        # finished request (earlier legs' decode appends) are dropped, not shipped
        for p in {id(rig.patch): rig.patch, id(sender): sender}.values():
            p.discard_request(f"r{i:04d}", rig.registry)
        rig.src.free_request(f"r{i:04d}")
        recv_store.free_request(f"r{i:04d}")
    try:
        one_step(K)
        torch.cuda.synchronize()
        # a host sync point after the warm-up: staging rings it outgrew are freed here
        rig.src.sync()
        recv_store.sync()
        # no cyclic-GC pass inside the wall-clock region (earlier legs leave many objects)
        gc.collect()
        gc.disable()
        phases.clear()
        st0 = [st.staging_stats() for st in (rig.src, recv_store)]
        t0 = time.perf_counter()
        marks = []
        for i in range(K):
            keys = one_step(i)
            marks.append(time.perf_counter())
        stream.synchronize()
        torch.cuda.synchronize()
        sec = time.perf_counter() - t0
        st1 = [st.staging_stats() for st in (rig.src, recv_store)]
        last_push = sender.last_push_stats() if hasattr(sender, "last_push_stats") else None
    finally:
        gc.enable()
        receiver.shutdown()
        if ring is not None:
            N.check(N.lib().pl_patch_set_active(rig.patch.h, 1))
    sec = allmax(sec, world)
    expect = wl.batch * wl.ctx * len(wl.mig_groups)
    assert keys == expect and all(int(x) == expect for x in results[:K]), results[:K]
    rig.src.free_requests(names)
    recv_store.free_requests(names)
    return {"value": round(world * K * wl.payload_bytes / sec / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": int(host.nbytes + 16 * len(reqs)),
            "d2h_bytes_per_step": 8, "ms_per_step": round(sec / K * 1e3, 3),
            # host time between consecutive step calls returning (the device runs ahead or
            # behind; a stall anywhere in the loop shows up here as one long step)
            "host_step_ms_max": round(max(b - a for a, b in zip([t0] + marks, marks)) * 1e3, 3),
            # the slowest step's host phases: free, append (H2D + K1 enqueue), push, D2H
            "host_step_phases_ms": dict(zip(("free", "append", "push", "d2h"), (
                round(x * 1e3, 3) for x in max(phases, key=sum)))),
            # the last step's push, host phases (ms): snapshot, receiver reservation, table
            # flush, K3 / copy enqueue (pl_patch_last_push_stats)
            "last_push_phases_ms": last_push,
            # H2D staging rings of the sending / receiving store over the timed steps
            "staging": {name: {"ring_mb": round(b["ring_bytes"] / 2**20, 1),
                               "outgrows": b["outgrows"] - a["outgrows"],
                               "retire_waits": b["retire_waits"] - a["retire_waits"],
                               "wait_ms": round((b["wait_ns"] - a["wait_ns"]) / 1e6, 3)}
                        for name, a, b in zip(("src", "dst"), st0, st1)},
            "path": "host payload fingerprints -> pl_store_append_batch_payloads (K1 expand + "
                    "mark) -> pl_patch_push (K3 + fused K4/K5) -> D2H drained count "
                    "(pipelined: step i+1 is prepared on the host while step i runs)"
                    + ("; N > 1: the ring's cross-process round (rank r -> r + 1), as `value`"
                       if ring is not None else "")}


def measure_e2e(rig, stream, torch, wl, K, world) -> dict:
    """The bulk round through the C-ABI with host buffers: each step the migrating
    groups' KV of all B requests streams from pinned host memory (H2D, chunked and
    double-buffered), is appended by K1 with the fused dirty mark, then drained and
    pushed; the device drained count is read back (D2H)."""
    from paper_2604_12171_b200 import _native as N
    from paper_2604_12171_b200.perf import append_batch
    from paper_2604_12171_b200.events import stable_hash

    per_req = wl.ctx * wl.k * wl.cell_bytes          # one (request, group)
    chunk_reqs = 16
    chunk_bytes = chunk_reqs * len(wl.mig_groups) * per_req
    host = torch.empty(chunk_bytes, dtype=torch.uint8, pin_memory=True)
    host.random_(0, 255)
    dev = [torch.empty(chunk_bytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    copy_stream = torch.cuda.Stream()
    done_copy = [torch.cuda.Event() for _ in range(2)]
    done_use = [torch.cuda.Event() for _ in range(2)]
    result = torch.empty(1, dtype=torch.int64, pin_memory=True)
    e2e_names = [f"e2e{i:04d}" for i in range(wl.batch)]
    handles = [rig.registry.handle(n) for n in e2e_names]

    def one_step():
        for n in e2e_names:   # the previous step's requests leave both stages
            rig.src.free_request(n)
            rig.dst.free_request(n)
        for c0 in range(0, wl.batch, chunk_reqs):
            b = (c0 // chunk_reqs) % 2
            copy_stream.wait_event(done_use[b])
            with torch.cuda.stream(copy_stream):
                dev[b].copy_(host, non_blocking=True)
                done_copy[b].record(copy_stream)
            stream.wait_event(done_copy[b])
            reqs, groups, counts, seeds = [], [], [], []
            for i in range(c0, min(c0 + chunk_reqs, wl.batch)):
                for g in wl.mig_groups:
                    reqs.append(handles[i])
                    groups.append(g)
                    counts.append(wl.ctx)
                    seeds.append(stable_hash(e2e_names[i], g))
            append_batch(rig.src, reqs, groups, counts, seeds, kv_dev=dev[b].data_ptr(), mark=True)
            done_use[b].record(stream)
        keys, _ = rig.patch.push(rig.dst, rig.registry.rank())
        # D2H of the step's result: the device's drained-key count
        result[0] = rig.patch.device_drained()
        return keys

    # the e2e requests need room: the bulk requests leave both stages first
    for i in range(wl.batch):
        rig.src.free_request(f"r{i:04d}")
        rig.dst.free_request(f"r{i:04d}")
    one_step()
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()
    try:
        t0 = time.perf_counter()
        for _ in range(K):
            keys = one_step()
            stream.synchronize()
        sec = time.perf_counter() - t0
    finally:
        gc.enable()
    sec = allmax(sec, world)
    assert keys == wl.batch * wl.ctx * len(wl.mig_groups)
    for n in e2e_names:
        rig.src.free_request(n)
        rig.dst.free_request(n)
    return {"value": round(world * K * wl.payload_bytes / sec / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": (wl.batch // chunk_reqs) * chunk_bytes,
            "d2h_bytes_per_step": 8, "ms_per_step": round(sec / K * 1e3, 2)}


def measure_resize(rig, stream, torch, wl) -> dict:
    """Post-commit cleanup on the source stage (coordinator.py:340-354): drop the groups
    that left, compact + shrink to a smaller budget, then grow back; wall ms each.

    The *_ms figures are the critical path of each call (host block manager, K6 moves,
    block-table remap, VMM map of new chunks).  Physical reclaim of retired chunks runs
    on the store's reclaimer thread (vmm.cu); `reclaim_ms` is how long forcing it to
    finish took afterwards (memory back with the driver), reported beside it.  A grow
    inside the grace period re-takes the still-mapped tail (`grow_warm_ms`); a grow
    after the reclaim maps fresh chunks from the driver: the capacity is published at once
    (`grow_cold_ms`) and the tail is mapped on the reclaimer thread
    (`grow_cold_background_ms`: until that mapping is done)."""
    st = rig.src
    out = {}

    def vdelta(a, b):
        return {k: b[k] - a[k] for k in ("tail_reused_chunks", "cache_reused_chunks",
                                         "created_chunks")}

    torch.cuda.synchronize()
    st.reclaim()
    t0 = time.perf_counter()
    freed = st.drop_layer_groups(list(wl.mig_groups))
    out["drop_groups_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    out["drop_pending_reclaim_bytes"] = st.vmm_stats()["pending_reclaim_bytes"]
    out["drop_reclaim_ms"] = round(st.reclaim(), 3)
    # resize latency = compact + VMM unmap/map + K6, i.e. until the physical
    # memory is back with the driver (unmap forced now instead of after the grace period)
    out["drop_groups_full_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    # free a quarter of the requests so the shrink must relocate live tail blocks
    for i in range(0, wl.batch, 4):
        st.free_request(f"r{i:04d}")
    cap = st.capacity_blocks
    target = max(st.used_blocks + 16, int(cap * 0.8))
    st.sync()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.compact()
    st.resize(target)
    st.sync()
    out["shrink_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    out["shrink_stats"] = st.last_resize_stats()
    v0 = st.vmm_stats()
    t0 = time.perf_counter()
    st.resize(cap)
    st.sync()
    out["grow_warm_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    out["grow_warm_full_ms"] = round((time.perf_counter() - t0) * 1e3 + st.prepare_wait(), 3)
    v1 = st.vmm_stats()
    out["grow_warm_stats"] = {**st.last_resize_stats(), **vdelta(v0, v1)}
    # the shrink again, now timed until its tail is unmapped (full latency)
    t0 = time.perf_counter()
    st.compact()
    st.resize(target)
    st.sync()
    out["reclaim_ms"] = round(st.reclaim(), 3)
    out["shrink_full_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    v2 = st.vmm_stats()
    t0 = time.perf_counter()
    st.resize(cap)
    st.sync()
    out["grow_cold_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    # the new tail is mapped by the reclaimer thread (lazy grow); time until it is done
    out["grow_cold_background_ms"] = round((time.perf_counter() - t0) * 1e3 + st.prepare_wait(), 3)
    out["grow_cold_full_ms"] = out["grow_cold_background_ms"]
    out["grow_cold_stats"] = {**st.last_resize_stats(), **vdelta(v2, st.vmm_stats())}
    out["blocks"] = {"from": cap, "to": target, "live": st.used_blocks}
    out["tokens_freed_by_drop"] = freed
    out["note"] = ("*_full_ms = SURVEY 8(d) resize latency: until the VMM unmap/map is done "
                   "(physical memory returned / mapped); *_ms without 'full' = the critical "
                   "path of the call (unmap/map run on the store's reclaimer thread)")
    return out


if __name__ == "__main__":
    main()
