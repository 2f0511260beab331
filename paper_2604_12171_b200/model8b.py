"""BASELINE configs[1] live with real stage compute (SURVEY §8f-2 at the 8B shape).

A Llama-3-8B-shaped decoder (32 layers, d = 4096, 32 q / 8 KV heads x 128, SwiGLU
14336, vocab 128256, bf16 random-init weights) runs greedy decode over B = 256 requests
whose KV (2048 prefilled positions each, 16-token blocks, k = 4 layers per group) lives
in the paged stores of its pipeline stages, while a live PP 2 -> 4 reconfiguration moves
layers 9-16 (GPU 1 -> 3) and 25-32 (GPU 2 -> 4):

  - per layer: RMSNorm, QKV / O / MLP projections (bf16 tensor-core GEMMs, cuBLAS via
    torch: library GEMMs for the dense parts), RoPE, then the KV path of this repo --
    K1 appends the new token's cells into the layer group of the stage's store with the
    fused dirty mark (engine.py:377-404, migrator.py:190-197; the group's other layers are
    written with pl_store_write_layer as they are produced), K2 decodes over the store's
    block table;
  - reconfiguration (coordinator.py:203-338): the destinations map the arriving groups,
    every pair seeds its live cells and pushes them (bulk) on a lowest-priority side
    stream, then one patch round per decode step; the coordinator polls the reference's
    safe-switch test every step -- lag = cells written but not yet applied on the
    destination (t_sched - t_applied, migrator.py:74-90, 341-348) < tau = 50 -- and
    commits: pause admission, drain the in-flight step, residual round (final sync),
    barrier, switch ownership, resume; the sources drop the groups that left
    (coordinator.py:340-354).
All stages share one GPU here (stage stores are distinct, as distinct GPUs would hold
them); on hardware each stage's store is on its own GPU and the push crosses NVLink.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass
from math import ceil

import numpy as np

from . import _native as N
from .events import stable_hash
from .kvstore import KvStore, RequestRegistry
from .perf import NativePatch, append_batch


@dataclass(frozen=True)
class Shape8B:
    n_layers: int = 32
    d: int = 4096
    n_q: int = 32
    n_kv: int = 8
    head_dim: int = 128
    ffn: int = 14336
    vocab: int = 128256
    theta: float = 500000.0
    eps: float = 1e-5
    k: int = 4
    s: int = 16

    @property
    def cell_bytes(self) -> int:
        return 2 * self.n_kv * self.head_dim * 2

    @property
    def groups(self) -> int:
        return self.n_layers // self.k


PP2 = {1: list(range(1, 17)), 2: list(range(17, 33)), 3: [], 4: []}
PP4 = {1: list(range(1, 9)), 3: list(range(9, 17)), 2: list(range(17, 25)), 4: list(range(25, 33))}


def _split(sizes: list[int]) -> dict[int, list[int]]:
    out, l = {}, 1
    for g, n in enumerate(sizes, start=1):
        out[g] = list(range(l, l + n))
        l += n
    return out


# BASELINE configs[3] at the 8B shape (SURVEY §8(d) C4 scaled to 32 layers, k = 2): an even
# 8-stage split re-split live into a generation-heavy uneven one; six pairs migrate
# (1->2, 2->3, 3->4, 6->5, 7->6, 8->7), stages 2, 3, 6, 7 both send and receive
EVEN8 = _split([4] * 8)
UNEVEN8 = _split([2, 4, 4, 6, 6, 4, 4, 2])


def _vp(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


class Pipeline8B:
    """The stages of one PP config on one GPU; stage g's KV in its own store (gpu id g)."""

    def __init__(self, config: dict[int, list[int]], batch: int = 256, ctx: int = 2048,
                 max_steps: int = 64, device: int = 0, seed: int = 0,
                 shape: Shape8B = Shape8B()) -> None:
        import torch

        self.torch = torch
        self.sh = sh = shape
        self.B, self.ctx0 = batch, ctx
        self.device = device
        self.dev = torch.device("cuda", device)
        self.stream = torch.cuda.Stream(device=device)
        lo, _ = torch.cuda.Stream.priority_range()
        self.side = torch.cuda.Stream(device=device, priority=lo)   # patch rounds
        self.registry = RequestRegistry()
        self.rids = [f"r{i:04d}" for i in range(batch)]
        self.handles = [self.registry.handle(r) for r in self.rids]
        self.owner = {l: g for g, ls in config.items() for l in ls}
        cap = batch * (ceil((ctx + max_steps) / sh.s) + 1) + 64
        self.stores: dict[int, KvStore] = {}
        for g in sorted(config):
            groups = sorted({(l - 1) // sh.k for l in config[g]})
            st = KvStore(g, sh.k, sh.s, cap, groups, num_groups=sh.groups,
                         cell_bytes=sh.cell_bytes, device=device, registry=self.registry)
            N.check(N.lib().pl_store_set_stream(st._h, C.c_void_p(self.stream.cuda_stream)))
            self.stores[g] = st
        self._init_weights(seed)
        self.pos = [ctx] * batch                 # next position of every request
        self.rows = torch.tensor(self.handles, dtype=torch.int32, device=self.dev)
        self.patches: dict[tuple[int, int], NativePatch] = {}
        self.moving: dict[tuple[int, int], list[int]] = {}
        self.inflight: list = []                 # (event, cells) of pushes not yet applied
        self.patched_cells = 0

    # ------------------------------------------------------------------ weights, KV fill
    def _init_weights(self, seed: int) -> None:
        torch, sh = self.torch, self.sh
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)

        def mat(i, o):
            w = torch.randn(i, o, generator=g, device=self.dev, dtype=torch.float32)
            return (w * (1.0 / i ** 0.5)).to(torch.bfloat16)

        qkv = (sh.n_q + 2 * sh.n_kv) * sh.head_dim
        self.w = {"embed": torch.randn(sh.vocab, sh.d, generator=g, device=self.dev).to(torch.bfloat16),
                  "final_norm": torch.ones(sh.d, device=self.dev),
                  "lm_head": mat(sh.d, sh.vocab)}
        for l in range(sh.n_layers):
            self.w[l] = {"attn_norm": 1 + 0.1 * torch.randn(sh.d, generator=g, device=self.dev),
                         "wqkv": mat(sh.d, qkv), "wo": mat(sh.n_q * sh.head_dim, sh.d),
                         "mlp_norm": 1 + 0.1 * torch.randn(sh.d, generator=g, device=self.dev),
                         "w13": mat(sh.d, 2 * sh.ffn), "w2": mat(sh.ffn, sh.d)}
        inv = 1.0 / (sh.theta ** (torch.arange(0, sh.head_dim, 2, device=self.dev,
                                               dtype=torch.float64) / sh.head_dim))
        self.inv_freq = inv

    def fill(self, seed: int = 1, chunk: int = 16) -> None:
        """Prefilled context: ctx positions of every request in every resident group,
        seeded random bf16 K/V written by K1 (the same bytes for the same seed)."""
        torch, sh = self.torch, self.sh
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        with torch.cuda.stream(self.stream):
            for gpu, st in sorted(self.stores.items()):
                for grp in sorted(st.resident_groups):
                    for c0 in range(0, self.B, chunk):
                        hs = self.handles[c0:c0 + chunk]
                        kv = torch.randn(len(hs) * self.ctx0, sh.k, sh.cell_bytes // 2,
                                         generator=g, device=self.dev).to(torch.bfloat16)
                        append_batch(st, hs, [grp] * len(hs), [self.ctx0] * len(hs),
                                     [stable_hash(self.rids[c0 + i], grp) for i in range(len(hs))],
                                     kv_dev=kv.data_ptr())
        self.stream.synchronize()

    # ------------------------------------------------------------------ decode
    def _rms(self, x, w):
        x32 = x.float()
        return (x32 * torch_rsqrt(x32, self.sh.eps) * w).to(self.torch.bfloat16)

    def order(self) -> list[int]:
        first: dict[int, int] = {}
        for layer, gpu in self.owner.items():
            first[gpu] = min(first.get(gpu, layer), layer)
        return sorted(first, key=first.get)

    def step(self, tokens, in_step_rounds: bool = False) -> "object":
        """One decode step of every request (token ids [B] on device) -> next tokens [B].

        With `in_step_rounds`, each migrating pair's patch round is enqueued as soon as
        the step has written the last layer of the pair's groups (MigrationStream.pump on
        on_kv_written, migrator.py:190-197, 208-225): the round then overlaps the rest of
        the step's compute instead of trailing it."""
        torch, sh, B = self.torch, self.sh, self.B
        pos_t = torch.tensor(self.pos, dtype=torch.int32, device=self.dev)
        ctx_t = pos_t + 1
        ang = pos_t.double()[:, None] * self.inv_freq[None, :]
        cos, sin = ang.cos().float()[:, None, :], ang.sin().float()[:, None, :]
        max_ctx = max(self.pos) + 1
        kvbuf = torch.zeros(B, sh.k, sh.cell_bytes // 2, dtype=torch.bfloat16, device=self.dev)
        out = torch.empty(B, sh.n_q, sh.head_dim, dtype=torch.bfloat16, device=self.dev)
        x = self.w["embed"][tokens].float()
        half = sh.head_dim // 2
        lib = N.lib()
        keep = []

        def rope(t):
            t1, t2 = t[..., :half], t[..., half:]
            return torch.cat([t1 * cos - t2 * sin, t2 * cos + t1 * sin], dim=-1)

        for gpu in self.order():
            st = self.stores[gpu]
            for l in sorted(l for l, g in self.owner.items() if g == gpu):
                w = self.w[l - 1]
                grp, j = (l - 1) // sh.k, (l - 1) % sh.k
                h = self._rms(x, w["attn_norm"])
                qkv = (h @ w["wqkv"]).float()
                q = rope(qkv[:, : sh.n_q * sh.head_dim].view(B, sh.n_q, sh.head_dim))
                kk = rope(qkv[:, sh.n_q * sh.head_dim:(sh.n_q + sh.n_kv) * sh.head_dim]
                          .view(B, sh.n_kv, sh.head_dim))
                vv = qkv[:, (sh.n_q + sh.n_kv) * sh.head_dim:]
                cell = torch.cat([kk.reshape(B, -1), vv], dim=1).to(torch.bfloat16)
                qb = q.to(torch.bfloat16).contiguous()
                if j == 0:
                    # KvStore.append of the group for the new token (blocks, fingerprint,
                    # fused dirty mark): layer 0's cell now, layers 1..k-1 as produced
                    kvbuf[:, 0] = cell
                    done = append_batch(st, self.handles, [grp] * B, [1] * B,
                                        [stable_hash(r, grp) for r in self.rids],
                                        kv_dev=kvbuf.data_ptr(), mark=True)
                    assert done == B
                    keep.append(kvbuf)
                    kvbuf = torch.zeros_like(kvbuf)
                else:
                    N.check(lib.pl_store_write_layer(st._h, grp, j, _vp(self.rows), _vp(pos_t), B,
                                                     _vp(cell), sh.cell_bytes,
                                                     C.c_void_p(self.stream.cuda_stream)))
                    keep.append(cell)
                N.check(lib.pl_paged_attn_decode(st._h, grp, j, _vp(qb), _vp(out), _vp(self.rows),
                                                 _vp(ctx_t), B, sh.n_q, sh.n_kv, sh.head_dim,
                                                 sh.head_dim ** -0.5, max_ctx,
                                                 C.c_void_p(self.stream.cuda_stream)))
                keep.append(qb)
                x = x + (out.view(B, -1) @ w["wo"]).float()
                h = self._rms(x, w["mlp_norm"])
                a = h @ w["w13"]
                x = x + ((torch.nn.functional.silu(a[:, : sh.ffn]) * a[:, sh.ffn:]) @ w["w2"]).float()
                if in_step_rounds:
                    for pair, layers in self.moving.items():
                        if l == max(layers):
                            self.pump(pairs=[pair])
        logits = self._rms(x, self.w["final_norm"]) @ self.w["lm_head"]
        for i in range(B):
            self.pos[i] += 1
        self._keep = keep
        return logits.argmax(-1)

    # ------------------------------------------------------------------ live reconfiguration
    def start_reconfig(self, target: dict[int, list[int]], before_bulk=None) -> dict:
        """Phase 3: destinations map the arriving groups, every pair seeds all live cells
        of its groups (MigrationStream.start) and pushes them on the side stream (bulk)."""
        sh = self.sh
        new_owner = {l: g for g, ls in target.items() for l in ls}
        moves: dict[tuple[int, int], list[int]] = {}
        for l in sorted(self.owner):
            if self.owner[l] != new_owner[l]:
                moves.setdefault((self.owner[l], new_owner[l]), []).append(l)
        self.target = new_owner
        # Phase 3 (coordinator.py:205-206): the destinations map the arriving groups' pools
        # (reclaimer thread, overlapped with AddLayerWeights on hardware, weights.py:103-125);
        # the bulk patch starts once they are mapped
        t0 = time.perf_counter()
        for (src, dst), layers in sorted(moves.items()):
            self.stores[dst].resident_groups |= {(l - 1) // sh.k for l in layers}
        for (src, dst) in sorted(moves):
            self.stores[dst].prepare_wait()
        self.map_ms = round((time.perf_counter() - t0) * 1e3, 3)
        for (src, dst), layers in sorted(moves.items()):
            groups = sorted({(l - 1) // sh.k for l in layers})
            p = NativePatch(self.stores[src], groups, sh.k)
            p.set_stream(self.side.cuda_stream)
            self.patches[(src, dst)] = p
            self.moving[(src, dst)] = layers
            p.seed()
        if before_bulk is not None:
            before_bulk()
        return self.pump()

    def pump(self, pairs=None) -> dict:
        """One patch round per pair (MigrationStream.pump -> _drain -> _send_patch ->
        PatchReceiver.receive): K3 + fused K4/K5 on the side stream; the round's cells
        count as applied once its event has completed."""
        torch = self.torch
        rank = self.registry.rank()
        keys_total = cells_total = 0
        for pair, p in self.patches.items():
            if pairs is not None and pair not in pairs:
                continue
            keys, cells = p.push(self.stores[pair[1]], rank)
            keys_total += keys
            cells_total += cells
        ev = torch.cuda.Event()
        ev.record(self.side)
        self.inflight.append((ev, cells_total))
        self.patched_cells += cells_total
        return {"keys": keys_total, "cells": cells_total, "event": ev,
                "host_phases_ms": {f"{a}->{b}": p.last_push_stats()
                                   for (a, b), p in self.patches.items()}}

    def lag(self) -> int:
        """t_sched - t_applied in cells over every destination (migrator.py:74-90): cells
        marked and not yet drained, plus drained cells whose push has not completed."""
        self.inflight = [(e, c) for e, c in self.inflight if not e.query()]
        pending = sum(c for _, c in self.inflight)
        return pending + sum(p.dirty_keys() * self.sh.k for p in self.patches.values())

    def switch(self) -> dict:
        """Phase 5 from the pause on: drain the in-flight step, final sync (residual round),
        barrier (the residual is applied on every destination), switch ownership, and the
        post-commit cleanup on the sources (drop the groups that left)."""
        t0 = time.perf_counter()
        self.stream.synchronize()                  # pipeline drained
        t1 = time.perf_counter()
        res = self.pump()                          # final sync: residual round
        t2 = time.perf_counter()
        self.side.synchronize()                    # barrier: applied everywhere
        for (src, dst) in self.patches:
            self.stores[dst].sync()
        t3 = time.perf_counter()
        for (src, dst), layers in self.moving.items():
            for l in layers:
                self.owner[l] = dst
        t4 = time.perf_counter()                   # resume admission here
        for p in self.patches.values():
            p.close()
        for (src, dst), layers in self.moving.items():
            self.stores[src].drop_layer_groups(sorted({(l - 1) // self.sh.k for l in layers}))
        self.patches.clear()
        self.moving.clear()
        self.inflight.clear()
        ms = lambda a, b: round((b - a) * 1e3, 4)  # noqa: E731
        return {"pause_ms": ms(t0, t4), "drain_ms": ms(t0, t1), "residual_ms": ms(t1, t3),
                "residual_enqueue_ms": ms(t1, t2), "barrier_and_switch_ms": ms(t3, t4),
                "residual_cells": res["cells"],
                "cleanup_ms_after_resume": ms(t4, time.perf_counter())}

    def close(self) -> None:
        for p in self.patches.values():
            p.close()
        for st in self.stores.values():
            st.close()
        self.stores.clear()


def torch_rsqrt(x32, eps):
    return (x32.pow(2).mean(-1, keepdim=True) + eps).rsqrt()


def run_live(batch: int = 256, ctx: int = 2048, steps: int = 40, reconfig_at: int = 8,
             live: bool = True, tau: int = 50, device: int = 0, seed: int = 0,
             src: dict | None = None, dst: dict | None = None, k: int = 4,
             trace=None) -> dict:
    """Greedy decode for `steps` steps over the stages of `src` (default PP2, k = 4); with
    `live`, the reconfiguration to `dst` (default PP4: configs[1]; EVEN8 -> UNEVEN8 at k = 2
    is configs[3]) starts after step `reconfig_at` and commits at the first poll with
    lag < tau.  Returns the tokens of every step and the timeline (per-step TPOT, phases,
    pause breakdown).  `trace` (an events.EventTrace) receives the run in the reference's
    trace schema with wall-clock times (the engine's request / decode-step events, the
    coordinator's reconfigure / convergence / commit-pause events), so
    engine.compute_metrics and outputs.write_run apply; requests arrive with their
    prefilled context, so TTFT is the first decode step."""
    import torch

    src, dst = src or PP2, dst or PP4
    pipe = Pipeline8B(src, batch, ctx, max_steps=steps + 4, device=device, seed=seed,
                      shape=Shape8B(k=k))
    pipe.fill()
    tokens = torch.arange(batch, device=pipe.dev, dtype=torch.long) * 7 % pipe.sh.vocab
    out = {"tokens": [], "step_ms": [], "phase": [], "lag": []}
    phase = "before"
    commit = None
    bulk = None
    t_run = time.perf_counter()

    def emit(kind, at=None, actor="engine", **payload):
        if trace is not None:
            trace.emit((at if at is not None else time.perf_counter()) - t_run, actor, kind,
                       **payload)

    for rid in pipe.rids:
        emit("request_arrival", id=rid, input_len=ctx, output_len=steps)
    with torch.cuda.stream(pipe.stream):
        for t in range(steps):
            if phase == "migrating":
                lag = pipe.lag()                   # the safe-switch poll (once per step)
                out["lag"].append(lag)
                emit("convergence_check", actor="coordinator", lag=lag, tau=tau)
                if lag < tau:
                    tp = time.perf_counter()
                    emit("commit_pause_start", at=tp, actor="coordinator")
                    commit = {"step": t, "lag_at_poll": lag, **pipe.switch()}
                    emit("commit_pause_end", at=tp + commit["pause_ms"] / 1e3, actor="coordinator")
                    emit("reconfigure_end", actor="coordinator", outcome="success")
                    phase = "after"
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            th = time.perf_counter()
            e0.record(pipe.stream)
            # while migrating, every pair's round is enqueued inside the step right after
            # the pair's last source layer (overlapping the rest of the step), so the
            # next step's poll sees the lag the reference's poll would (migrator.py:74-90)
            nxt = pipe.step(tokens, in_step_rounds=(phase == "migrating"))
            e1.record(pipe.stream)
            tok_host = nxt.cpu()                   # greedy: the next inputs come back
            host_ms = (time.perf_counter() - th) * 1e3
            out["tokens"].append(tok_host.tolist())
            out["step_ms"].append((e0, e1, host_ms))
            out["phase"].append(phase)
            emit("decode_step", step=t, batch=batch, ms=round(host_ms, 4))
            for rid in pipe.rids:
                if t == 0:
                    emit("first_token", id=rid)
                if t == steps - 1:
                    emit("request_done", id=rid)
            tokens = nxt
            if live and t == reconfig_at:
                emit("reconfigure_start", actor="coordinator",
                     target={str(g): ls for g, ls in sorted(dst.items())})
                tb = time.perf_counter()
                b0 = torch.cuda.Event(enable_timing=True)
                r = pipe.start_reconfig(dst, before_bulk=lambda: b0.record(pipe.side))
                b1 = torch.cuda.Event(enable_timing=True)
                b1.record(pipe.side)
                bulk = {"cells": r["cells"], "bytes": r["cells"] * pipe.sh.cell_bytes,
                        "phase3_map_ms": pipe.map_ms,
                        "host_enqueue_ms": round((time.perf_counter() - tb) * 1e3 - pipe.map_ms, 3),
                        "host_phases_ms": r["host_phases_ms"], "events": (b0, b1)}
                emit("migration_seeded", actor="coordinator", cells=r["cells"])
                phase = "migrating"
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_run
    step_ms = [a.elapsed_time(b) for a, b, _ in out["step_ms"]]
    host_ms = [h for _, _, h in out["step_ms"]]
    res = {"tokens": out["tokens"], "step_ms": [round(x, 4) for x in step_ms],
           "step_wall_ms": [round(x, 4) for x in host_ms], "phase": out["phase"],
           "lag_polls": out["lag"], "wall_s": round(wall, 3), "commit": commit,
           "config_end": {g: ls for g, ls in sorted(
               {g: sorted(l for l, o in pipe.owner.items() if o == g) for g in pipe.stores}.items())}}
    if bulk is not None:
        b0, b1 = bulk.pop("events")
        bulk["device_ms"] = round(b0.elapsed_time(b1), 3)
        bulk["gbs"] = round(bulk["bytes"] / bulk["device_ms"] / 1e6, 1)
        res["bulk"] = bulk
    pipe.close()
    del pipe
    torch.cuda.empty_cache()
    return res


def summarize(live: dict, static: dict) -> dict:
    """TPOT (device ms per decode step = per generated token of every request) before,
    while migrating, after; the switch step and pause; tokens vs the static run."""
    def med(xs):
        return round(float(np.median(xs)), 4) if xs else None

    by = {p: [m for m, ph in zip(live["step_wall_ms"], live["phase"]) if ph == p]
          for p in ("before", "migrating", "after")}
    dev = {p: [m for m, ph in zip(live["step_ms"], live["phase"]) if ph == p]
           for p in ("before", "migrating", "after")}
    return {"tokens_equal_static": live["tokens"] == static["tokens"],
            "steps": len(live["tokens"]),
            "tpot_ms_before": med(by["before"]), "tpot_ms_during": med(by["migrating"]),
            "tpot_ms_after": med(by["after"]),
            "tpot_ms_static": med(static["step_wall_ms"]),
            "device_step_ms": {p: med(v) for p, v in dev.items()},
            "steps_per_phase": {p: len(v) for p, v in by.items()},
            "switch_step": (live["commit"] or {}).get("step"),
            "lag_polls": live["lag_polls"],
            "commit": live["commit"], "bulk": live.get("bulk"),
            "config_end": live["config_end"]}
