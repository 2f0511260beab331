"""Phase times of one cross-process ring round (bench.py --gpus N topology); run under
torchrun.  Two ranks may share one GPU (functional timing of the control path).
Bulk rounds (every live cell re-seeded) first, then steady decode-pattern rounds (one
new token per request and migrating group): the control of a steady round is the host
time around the push -- drain rows + post, the receiver's reservation + reply, the
sender's push enqueue + "applied" -- against the push's device time."""
import faulthandler, json, os, sys, time
faulthandler.dump_traceback_later(float(os.environ.get("PROBE_DUMP_S", "1e9")), exit=True)
sys.path.insert(0, '.')
import numpy as np
import torch
import torch.distributed as dist
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
dev = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
torch.cuda.set_device(dev)
from paper_2604_12171_b200.perf import PatchRig, Workload
from paper_2604_12171_b200.dist import RingPair
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rig = PatchRig(Workload(batch=batch), device=dev)
s = torch.cuda.Stream()
rig.use_stream(s.cuda_stream)
rig.fill()
ring = RingPair(rig, rank, world, f"probe-{os.environ.get('MASTER_PORT')}")
ring.use_stream(s.cuda_stream)
names = ["seed", "begin(drain rows+send)", "serve_rows(recv+reserve+reply)", "finish(push+ack)", "serve_ack"]
for it in range(5):
    dist.barrier()
    t = [time.perf_counter()]
    ring.tx.seed(); t.append(time.perf_counter())
    ring.tx.begin(); t.append(time.perf_counter())
    ring.rx.serve_rows(); t.append(time.perf_counter())
    ring.tx.finish(); t.append(time.perf_counter())
    ring.rx.serve_ack(); t.append(time.perf_counter())
    if rank == 0 and it >= 2:
        print("bulk  ", " | ".join(f"{n} {1e3*(b-a):.3f}" for n, a, b in zip(names, t, t[1:])), f"total {1e3*(t[-1]-t[0]):.3f} ms", flush=True)
torch.cuda.synchronize()
# steady decode-pattern rounds: position ctx + i of every request in both migrating groups
wl = rig.wl
reqs = [h for h in rig.handles for _ in wl.mig_groups]
groups = [g for _ in rig.handles for g in wl.mig_groups]
ctrl, pushes, walls = [], [], []
for i in range(40):
    starts = [wl.ctx - 1 - (i % 8)] * len(reqs)          # rewrite of existing tail positions
    ring.tx.patch.mark_batch(reqs, groups, starts, [1] * len(reqs))
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    ring.tx.begin()
    t1 = time.perf_counter()
    ring.rx.serve_rows()
    t2 = time.perf_counter()
    ring.tx.finish()
    t3 = time.perf_counter()
    ring.rx.serve_ack()
    t4 = time.perf_counter()
    ring.dst.sync(); rig.src.sync()
    t5 = time.perf_counter()
    if i >= 5:
        ctrl.append((t4 - t0) * 1e6)
        walls.append((t5 - t0) * 1e6)
        pushes.append(((t1 - t0) * 1e6, (t2 - t1) * 1e6, (t3 - t2) * 1e6, (t4 - t3) * 1e6))
if rank == 0:
    p = np.median(np.array(pushes), axis=0)
    print(json.dumps({"steady_keys_per_round": len(reqs),
                      "control_us_median": round(float(np.median(ctrl)), 1),
                      "wall_us_median": round(float(np.median(walls)), 1),
                      "phases_us": {"begin": round(p[0], 1), "serve_rows": round(p[1], 1),
                                    "finish": round(p[2], 1), "serve_ack": round(p[3], 1)}}), flush=True)
ring.close()
dist.destroy_process_group()
