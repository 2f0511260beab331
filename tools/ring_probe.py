"""Phase times of one cross-process ring round (bench.py --gpus N topology); run under
torchrun.  Two ranks may share one GPU (functional timing of the control path)."""
import os, sys, time
sys.path.insert(0, '.')
import torch
import torch.distributed as dist
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
dev = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
torch.cuda.set_device(dev)
from paper_2604_12171_b200.perf import PatchRig, Workload
from paper_2604_12171_b200.dist import RingPair
rig = PatchRig(Workload(batch=int(sys.argv[1]) if len(sys.argv) > 1 else 64), device=dev)
s = torch.cuda.Stream()
rig.use_stream(s.cuda_stream)
rig.fill()
ring = RingPair(rig, rank, world, f"probe-{os.environ.get('MASTER_PORT')}")
ring.use_stream(s.cuda_stream)
for it in range(5):
    dist.barrier()
    t = [time.perf_counter()]
    ring.tx.seed(); t.append(time.perf_counter())
    ring.tx.begin(); t.append(time.perf_counter())
    ring.rx.serve_rows(); t.append(time.perf_counter())
    ring.tx.finish(); t.append(time.perf_counter())
    ring.rx.serve_ack(); t.append(time.perf_counter())
    if rank == 0 and it >= 2:
        names = ["seed", "begin(drain rows+send)", "serve_rows(recv+reserve+reply)", "finish(push+sync+ack)", "serve_ack"]
        print(" | ".join(f"{n} {1e3*(b-a):.2f}" for n, a, b in zip(names, t, t[1:])), f"total {1e3*(t[-1]-t[0]):.2f} ms", flush=True)
ring.close()
dist.destroy_process_group()
