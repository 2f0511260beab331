"""BASELINE configs[3] machinery on one GPU: 8 stage processes (16-layer tiny Llama), an
even split re-split live into an uneven one mid-decode.  Rank 0 records the run's trace
in the reference schema and writes trace.jsonl / metrics.csv / summary.json (outputs.py)
to gpurun_out/c4_live_run/; prints compute_metrics and the decode-step latency before /
during / after the switch.  The 8 processes share one B200, so the latencies show the
mechanism (pause, interference), not 8-GPU pipeline timings."""
import json
import multiprocessing as mp
import os
import socket
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")


def stage(rank, world, port, prefix, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import dist_workers as W
    from paper_2604_12171_b200.engine import compute_metrics
    from paper_2604_12171_b200.events import EventTrace
    from paper_2604_12171_b200.llama import (DistStagedLlama, LlamaConfig, generate_dist,
                                              init_weights, step_latency_around_switch)
    cfg = LlamaConfig(n_layers=16)
    m = DistStagedLlama(cfg, init_weights(cfg, 1), W.CONF_EVEN8, rank, channel_prefix=prefix)
    prompts = [[(7 * b + i) % 1000 for i in range(40 + 9 * b)] for b in range(8)]
    tr = EventTrace() if rank == 0 else None
    generate_dist(m, prompts, [2 * b for b in range(8)], 48, reconfig=(40, W.CONF_UNEVEN8),
                  switch_at=60, trace=tr)
    if rank == 0:
        from paper_2604_12171_b200 import outputs
        outputs.write_run("gpurun_out/c4_live_run", tr, "configs[3]:even8->uneven8", 0,
                          mode="perf", stages=8)
        q.put(("main", {"metrics": compute_metrics(tr).as_row(),
                        "steps": step_latency_around_switch(tr), "events": len(tr), "stages": 8,
                        "note": "8 stage processes share one B200: mechanism (pause, "
                                "interference), not 8-GPU pipeline timings"}))
    q.put(("phases", rank, {"pause": getattr(m, "switch_phases_ms", None),
                            "post_commit": getattr(m, "post_commit_ms", None)}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=stage, args=(r, 8, port, f"c4-{os.getpid()}", q)) for r in range(8)]
    for p in ps:
        p.start()
    res, phases = None, {}
    for _ in range(9):
        msg = q.get(timeout=600)
        if msg[0] == "main":
            res = msg[1]
        else:
            phases[msg[1]] = msg[2]
    for p in ps:
        p.join(timeout=120)
    # every rank's share of the pause (weight gate, residual round) and of the post-commit
    # cleanup after it (pair teardown, drop + evict)
    res["switch_phases_ms_by_rank"] = {r: phases[r] for r in sorted(phases)}
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/c4_live.json", "w"), indent=1)
    print(json.dumps(res, indent=1))
