"""Stage processes of tests/test_gpu_dist_llama.py: ranks on cuda:0; activations move
device to device through the K7 rings (csrc/act.cu; gloo only carries the step's token
ids and the lag all-reduce), KV patches through the cross-process push; the stage
compute runs in exact mode so the tokens can be compared with the CPU oracle."""

import os

PROMPTS = [[3, 17, 400, 9, 77], [5] * 12, list(range(100, 123)), [1000, 2, 2, 2, 999, 64, 31, 8]]
JOINS = [0, 2, 5, 9]
N_GEN = 24
CONF_A = {1: [1, 2], 2: [3, 4]}          # PP2 on GPUs 1-2, GPU 3 idle (zero-layer extension)
CONF_B = {1: [1], 2: [2, 3], 3: [4]}     # PP3 (BASELINE configs[0])


def stage(rank, world, port, prefix, q, live):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2604_12171_b200.llama import (DistStagedLlama, LlamaConfig, generate_dist,
                                                  init_weights)
        cfg = LlamaConfig()
        m = DistStagedLlama(cfg, init_weights(cfg, 0), CONF_A, rank, channel_prefix=prefix,
                            exact=True)
        outs = generate_dist(m, PROMPTS, JOINS, N_GEN,
                             reconfig=(10, CONF_B) if live else None,
                             switch_at=("converged" if live == "converged" else 20) if live else None)
        q.put((rank, outs, sorted(m.store.resident_groups),
               {"mode": m.link.mode, "host_staged": m.link.host_staged,
                "sent_bytes": m.link.sent_bytes}))
        dist.barrier()
        m.close()
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, "error", traceback.format_exc()))


# BASELINE configs[3] shape on 8 stage processes: 16-layer tiny model, an even split
# (2 layers per GPU) re-split live into an uneven, generation-heavy one
CONF_EVEN8 = {g: [2 * g - 1, 2 * g] for g in range(1, 9)}
CONF_UNEVEN8 = {1: [1], 2: [2, 3], 3: [4, 5], 4: [6, 7, 8], 5: [9, 10, 11], 6: [12, 13],
                7: [14, 15], 8: [16]}


def stage8(rank, world, port, prefix, q, live):
    try:
        import time

        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2604_12171_b200.llama import (DistStagedLlama, LlamaConfig, generate_dist,
                                                  init_weights)
        cfg = LlamaConfig(n_layers=16)
        m = DistStagedLlama(cfg, init_weights(cfg, 1), CONF_EVEN8, rank, channel_prefix=prefix,
                            exact=True)
        t0 = time.perf_counter()
        outs = generate_dist(m, PROMPTS, JOINS, N_GEN,
                             reconfig=(8, CONF_UNEVEN8) if live else None,
                             switch_at=16 if live else None)
        q.put((rank, outs, sorted(m.store.resident_groups), time.perf_counter() - t0,
               {"mode": m.link.mode, "host_staged": m.link.host_staged,
                "sent_bytes": m.link.sent_bytes}))
        dist.barrier()
        m.close()
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, "error", traceback.format_exc()))
