"""Real stage compute over the live-reconfigurable KV path.

The reference's engine step is a cost model (engine.py:335-351); this module runs
an actual Llama decoder whose KV lives in the paged stores of the pipeline
stages, so decode load during a live reconfiguration is real and the generated
token ids can be checked:

  - every layer's K/V of the new token is written by K1 into the store of the
    stage that owns the layer, fused with the dirty mark of any migration
    patch streaming that layer (engine.py:377-404, migrator.py:190-197);
  - attention is K2 over that store's block table;
  - dense layers (projections, MLP, LM head) are plain fp32 GEMMs (cuBLAS via
    torch, plumbing), embeddings/argmax are torch ops;
  - a live PP reconfiguration moves layers between stages while decode keeps
    running: bulk copy, one patch round per decode step, residual patch at the
    switch, then the layer's owner flips and the source drops the group
    (coordinator.py:232-354).  Bit-exact KV movement means the token stream is
    identical to a run without the reconfiguration.

Stages are stores (one per pipeline GPU id); on one physical GPU they share the
device and run in stage order on one stream.  The layer -> group map uses
stacking factor k = 1 (group = layer - 1), as in BASELINE configs[0].
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .events import stable_hash
from .kvstore import KvStore, RequestRegistry
from .perf import NativePatch, append_batch


@dataclass(frozen=True)
class LlamaConfig:
    """Tiny Llama-style model of BASELINE configs[0] / SURVEY §8d C1."""
    n_layers: int = 4
    d_model: int = 256
    n_q: int = 4
    n_kv: int = 2
    head_dim: int = 64
    ffn: int = 512
    vocab: int = 1024
    rope_theta: float = 10000.0
    eps: float = 1e-5

    @property
    def cell_bytes(self) -> int:
        return 2 * self.n_kv * self.head_dim * 2


def init_weights(cfg: LlamaConfig, seed: int = 0) -> dict[str, np.ndarray]:
    """Random-init fp32 weights (numpy, seeded), scaled so activations stay O(1)."""
    rng = np.random.default_rng(seed)

    def mat(i, o, gain=1.0):
        return (rng.standard_normal((i, o)) * gain / np.sqrt(i)).astype(np.float32)

    d, hq, hkv = cfg.d_model, cfg.n_q * cfg.head_dim, cfg.n_kv * cfg.head_dim
    w = {"embed": rng.standard_normal((cfg.vocab, d)).astype(np.float32)}
    for li in range(cfg.n_layers):
        w[f"l{li}.attn_norm"] = (1 + 0.1 * rng.standard_normal(d)).astype(np.float32)
        w[f"l{li}.wq"] = mat(d, hq, 2.0)
        w[f"l{li}.wk"] = mat(d, hkv, 2.0)
        w[f"l{li}.wv"] = mat(d, hkv)
        w[f"l{li}.wo"] = mat(hq, d)
        w[f"l{li}.mlp_norm"] = (1 + 0.1 * rng.standard_normal(d)).astype(np.float32)
        w[f"l{li}.w1"] = mat(d, cfg.ffn)
        w[f"l{li}.w3"] = mat(d, cfg.ffn)
        w[f"l{li}.w2"] = mat(cfg.ffn, d)
    w["final_norm"] = (1 + 0.1 * rng.standard_normal(d)).astype(np.float32)
    w["lm_head"] = mat(d, cfg.vocab, 4.0)
    return w


def _vp(t):
    return C.c_void_p(t.data_ptr())


def _vp_stream(stream):
    return C.c_void_p(stream.cuda_stream)


def pipeline_order(owner: dict[int, int]) -> list[int]:
    """GPUs that hold layers, in pipeline order (by their first layer); a GPU with no
    layers (the zero-layer extension) is not a stage."""
    first: dict[int, int] = {}
    for layer, gpu in owner.items():
        first[gpu] = min(first.get(gpu, layer), layer)
    return sorted(first, key=first.get)


def layer_moves(owner: dict[int, int], target: dict[int, list[int]]) -> dict[tuple[int, int], list[int]]:
    """M_mig of a reconfiguration (cluster.py:238-270, diff_configs): for every layer whose
    owner changes, the (src, dst) pair it moves over; pairs and layers sorted."""
    new_owner = {l: g for g, ls in target.items() for l in ls}
    if sorted(new_owner) != sorted(owner):
        raise ValueError("target must place every layer exactly once")
    moves: dict[tuple[int, int], list[int]] = {}
    for layer in sorted(owner):
        if owner[layer] != new_owner[layer]:
            moves.setdefault((owner[layer], new_owner[layer]), []).append(layer)
    return dict(sorted(moves.items()))


def rope_tables(pos, head_dim: int, theta: float) -> tuple[np.ndarray, np.ndarray]:
    """Exact mode's RoPE cos/sin [B, D/2] (float64, numpy) for positions pos [B]."""
    inv = 1.0 / (theta ** (np.arange(0, head_dim, 2, dtype=np.float64) / head_dim))
    ang = np.asarray(pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.ascontiguousarray(np.cos(ang)), np.ascontiguousarray(np.sin(ang))


class LlamaCompute:
    """The math of one decode step, layer by layer, over whichever store owns a layer.

    Two numerics modes share the KV path (K1 writes into the paged stores, attention over
    their block tables):
      - default: fp32 dense layers (cuBLAS via torch), K2 tensor-core attention (bf16);
      - exact=True: every op a deterministic fp64 kernel of csrc/exact.cu (sequential fma
        dot products, fixed exp), bit-identical to the CPU oracle (oracle/llama_exact.c),
        so generated token ids are checked exactly; same bf16 rounding points (K, V, q,
        attention output)."""

    def __init__(self, cfg: LlamaConfig, weights: dict[str, np.ndarray], device: int,
                 registry: RequestRegistry, stream, layers=None, exact: bool = False) -> None:
        """`layers` (1-based, default all): which layers' weights go to the device now;
        the embedding, final norm and LM head always do."""
        import torch

        self.torch = torch
        self.cfg = cfg
        self.registry = registry
        self.stream = stream
        self.exact = exact
        self.act_dtype = torch.float64 if exact else torch.float32
        dev = torch.device("cuda", device)
        keep = None if layers is None else {f"l{l - 1}" for l in layers}

        def wanted(k: str) -> bool:   # per-layer keys are "l<i>.<name>"
            return keep is None or "." not in k or k.split(".", 1)[0] in keep

        self.w = {k: self.to_device(v, dev) for k, v in weights.items() if wanted(k)}

    def to_device(self, v, dev):
        t = self.torch.from_numpy(np.asarray(v)) if isinstance(v, np.ndarray) else v
        return t.to(device=dev, dtype=self.act_dtype)

    def begin(self, rids: list, positions: list[int], device) -> dict:
        """Per-step state: request rows, context lengths after this token, RoPE tables."""
        torch, c = self.torch, self.cfg
        handles = [self.registry.handle(r) for r in rids]
        if self.exact:
            cos, sin = rope_tables(positions, c.head_dim, c.rope_theta)
            ctx_host = [p + 1 for p in positions]
            return {"rids": rids, "handles": handles, "ctx_host": ctx_host,
                    "ctx": torch.tensor(ctx_host, dtype=torch.int32, device=device),
                    "rows": torch.tensor(handles, dtype=torch.int32, device=device),
                    "cos": torch.from_numpy(cos).to(device), "sin": torch.from_numpy(sin).to(device)}
        pos = torch.tensor(positions, device=device)
        inv = 1.0 / (c.rope_theta ** (torch.arange(0, c.head_dim, 2, device=device,
                                                   dtype=torch.float64) / c.head_dim))
        ang = pos[:, None].double() * inv[None, :]
        ctx_host = [p + 1 for p in positions]
        return {"rids": rids, "handles": handles, "ctx_host": ctx_host,
                "ctx": torch.tensor(ctx_host, dtype=torch.int32, device=device),
                "rows": torch.tensor(handles, dtype=torch.int32, device=device),
                "cos": ang.cos().float()[:, None, :], "sin": ang.sin().float()[:, None, :],
                "out": torch.empty(len(rids), c.n_q, c.head_dim, dtype=torch.bfloat16,
                                   device=device)}

    def _rmsnorm(self, x, g):
        if self.exact:
            out = self.torch.empty_like(x)
            N.check(N.lib().pl_exact_rmsnorm(_vp(x), _vp(g), _vp(out), x.shape[0], x.shape[1],
                                             float(self.cfg.eps), _vp_stream(self.stream)))
            return out
        var = x.double().pow(2).mean(-1, keepdim=True)
        return (x / (var + self.cfg.eps).sqrt()).float() * g

    def _gemv(self, x, w, resid=None):
        """exact mode: out = resid + x @ w, sequential fma chains (pl_exact_gemv)"""
        out = self.torch.empty(x.shape[0], w.shape[1], dtype=self.torch.float64, device=x.device)
        N.check(N.lib().pl_exact_gemv(_vp(x), _vp(w), _vp(resid) if resid is not None else None,
                                      _vp(out), x.shape[0], x.shape[1], w.shape[1],
                                      _vp_stream(self.stream)))
        return out

    def embed(self, tokens):
        return self.w["embed"][tokens]

    def head(self, x):
        if self.exact:
            return self._gemv(self._rmsnorm(x, self.w["final_norm"]), self.w["lm_head"])
        return self._rmsnorm(x, self.w["final_norm"]) @ self.w["lm_head"]

    def _layer_exact(self, li: int, x, st: KvStore, sc: dict):
        """Exact mode of layer(): the same K1 write / paged attention, deterministic fp64."""
        torch, c, w = self.torch, self.cfg, self.w
        B = len(sc["rids"])
        lib, stream = N.lib(), _vp_stream(self.stream)
        h = self._rmsnorm(x, w[f"l{li}.attn_norm"])
        q = self._gemv(h, w[f"l{li}.wq"])
        k = self._gemv(h, w[f"l{li}.wk"])
        v = self._gemv(h, w[f"l{li}.wv"])
        q_r = torch.empty_like(q)
        kv = torch.empty(B, 2 * c.n_kv * c.head_dim, dtype=torch.bfloat16, device=x.device)
        N.check(lib.pl_exact_rope_pack(_vp(q), _vp(k), _vp(v), _vp(sc["cos"]), _vp(sc["sin"]),
                                       _vp(q_r), _vp(kv), B, c.n_q, c.n_kv, c.head_dim, stream))
        seeds = [stable_hash(r, li) for r in sc["rids"]]
        done = append_batch(st, sc["handles"], [li] * B, [1] * B, seeds, kv_dev=kv.data_ptr(),
                            mark=True)
        assert done == B
        att = torch.empty_like(q_r)
        N.check(lib.pl_exact_attn_decode(st._h, li, 0, _vp(q_r), _vp(att), _vp(sc["rows"]),
                                         _vp(sc["ctx"]), B, c.n_q, c.n_kv, c.head_dim,
                                         float(c.head_dim) ** -0.5, max(sc["ctx_host"]), stream))
        x = self._gemv(att, w[f"l{li}.wo"], x)
        h = self._rmsnorm(x, w[f"l{li}.mlp_norm"])
        a = self._gemv(h, w[f"l{li}.w1"])
        g = self._gemv(h, w[f"l{li}.w3"])
        m = torch.empty_like(a)
        N.check(lib.pl_exact_silu_mul(_vp(a), _vp(g), _vp(m), a.numel(), stream))
        x = self._gemv(m, w[f"l{li}.w2"], x)
        sc.setdefault("keep", []).append((kv, q_r, att))  # alive until the stream consumed them
        return x

    def layer(self, li: int, x, st: KvStore, sc: dict):
        """Layer li (0-based): K/V of the new tokens into `st` by K1 (fused dirty mark),
        K2 attention over `st`'s block table, then the dense parts."""
        if self.exact:
            return self._layer_exact(li, x, st, sc)
        torch, c, w = self.torch, self.cfg, self.w
        B = len(sc["rids"])
        cos, sin, out = sc["cos"], sc["sin"], sc["out"]

        def rope(t):
            t1, t2 = t[..., : c.head_dim // 2], t[..., c.head_dim // 2:]
            return torch.cat([t1 * cos - t2 * sin, t2 * cos + t1 * sin], dim=-1)

        h = self._rmsnorm(x, w[f"l{li}.attn_norm"])
        q = rope((h @ w[f"l{li}.wq"]).view(B, c.n_q, c.head_dim)).to(torch.bfloat16)
        k = rope((h @ w[f"l{li}.wk"]).view(B, c.n_kv, c.head_dim))
        v = (h @ w[f"l{li}.wv"]).view(B, c.n_kv, c.head_dim)
        # cell = [K: n_kv x D][V: n_kv x D] bf16, one per (request, layer)
        kv = torch.cat([k.reshape(B, -1), v.reshape(B, -1)], dim=1).to(torch.bfloat16).contiguous()
        seeds = [stable_hash(r, li) for r in sc["rids"]]
        done = append_batch(st, sc["handles"], [li] * B, [1] * B, seeds, kv_dev=kv.data_ptr(),
                            mark=True)
        assert done == B
        N.check(N.lib().pl_paged_attn_decode(
            st._h, li, 0, C.c_void_p(q.data_ptr()), C.c_void_p(out.data_ptr()),
            C.c_void_p(sc["rows"].data_ptr()), C.c_void_p(sc["ctx"].data_ptr()), B, c.n_q,
            c.n_kv, c.head_dim, c.head_dim ** -0.5, max(sc["ctx_host"]),
            C.c_void_p(self.stream.cuda_stream)))
        x = x + out.float().view(B, -1) @ w[f"l{li}.wo"]
        h = self._rmsnorm(x, w[f"l{li}.mlp_norm"])
        a = h @ w[f"l{li}.w1"]
        x = x + (torch.nn.functional.silu(a) * (h @ w[f"l{li}.w3"])) @ w[f"l{li}.w2"]
        sc.setdefault("keep", []).append((kv, q))  # alive until the stream consumed them
        return x


class StagedLlama:
    """A Llama decoder split into pipeline stages, each stage's KV in its own store."""

    def __init__(self, cfg: LlamaConfig, weights: dict[str, np.ndarray],
                 config: dict[int, list[int]], device: int = 0, tokens_per_block: int = 16,
                 capacity_blocks: int = 256, registry: RequestRegistry | None = None,
                 exact: bool = False) -> None:
        import torch

        self.torch = torch
        self.cfg = cfg
        self.device = device
        self.s = tokens_per_block
        self.capacity = capacity_blocks
        self.registry = registry or RequestRegistry()
        # one non-default stream for the whole stage loop: torch ops, K1, K2 and the patch
        # rounds are ordered by it (callers run model code under `with model.on_stream()`)
        self.stream = torch.cuda.Stream(device=device)
        self.compute = LlamaCompute(cfg, weights, device, self.registry, self.stream,
                                    exact=exact)
        self.stores: dict[int, KvStore] = {}
        self.owner: dict[int, int] = {}          # layer (1-based) -> gpu id
        for gpu, layers in config.items():
            self._store(gpu, [l - 1 for l in layers])
            for l in layers:
                self.owner[l] = gpu
        assert sorted(self.owner) == list(range(1, cfg.n_layers + 1)), "every layer needs a stage"
        self.pos: dict = {}                      # rid -> tokens written (context length)
        self.patches: dict[tuple[int, int], NativePatch] = {}
        self.moving: dict[tuple[int, int], list[int]] = {}   # pair -> layers
        self.patched_bytes = 0

    # ---------------------------------------------------------------- stores
    def _store(self, gpu: int, groups: list[int]) -> KvStore:
        st = self.stores.get(gpu)
        if st is None:
            st = KvStore(gpu, 1, self.s, self.capacity, groups, num_groups=self.cfg.n_layers,
                         cell_bytes=self.cfg.cell_bytes, device=self.device,
                         registry=self.registry)
            N.check(N.lib().pl_store_set_stream(st._h, C.c_void_p(self.stream.cuda_stream)))
            self.stores[gpu] = st
        return st

    def on_stream(self):
        return self.torch.cuda.stream(self.stream)

    def config(self) -> dict[int, list[int]]:
        out: dict[int, list[int]] = {}
        for l, g in sorted(self.owner.items()):
            out.setdefault(g, []).append(l)
        return out

    # ---------------------------------------------------------------- decode
    def step(self, rids: list, tokens) -> "object":
        """One decode step for requests `rids` (token ids on device, [B]) -> fp32 logits
        [B, vocab].  Each request's new token lands at its current context length."""
        sc = self.compute.begin(rids, [self.pos.get(r, 0) for r in rids], tokens.device)
        x = self.compute.embed(tokens)
        for li in range(self.cfg.n_layers):
            x = self.compute.layer(li, x, self.stores[self.owner[li + 1]], sc)
        for r in rids:
            self.pos[r] = self.pos.get(r, 0) + 1
        return self.compute.head(x)

    def free(self, rid) -> None:
        """Request finished: its KV leaves every stage (engine.py:420-430); a migrating
        pair drops its dirty keys (DirtyBitmap.discard_request, migrator.py:43-48)."""
        h = self.registry.find(rid)
        for p in self.patches.values():
            if h is not None:
                out = C.c_int64()
                N.check(N.lib().pl_patch_discard_request(p.h, h, C.byref(out)))
        for st in self.stores.values():
            st.free_request(rid)
        self.pos.pop(rid, None)

    # ---------------------------------------------------------------- live reconfiguration
    def start_reconfig(self, target: dict[int, list[int]]) -> dict[tuple[int, int], list[int]]:
        """Phase 3 (coordinator.py:224-230): for every layer whose owner changes, the
        destination stage maps the layer's pool, a patch engine per (src, dst) pair seeds
        all live cells of its layers and pushes them (bulk copy); from now on K1 marks
        every new cell of those layers dirty."""
        new_owner = {l: g for g, ls in target.items() for l in ls}
        moves = layer_moves(self.owner, target)
        for (src, dst), layers in moves.items():
            d = self._store(dst, [])
            d.resident_groups |= {l - 1 for l in layers}
            p = NativePatch(self.stores[src], [l - 1 for l in layers], 1)
            self.patches[(src, dst)] = p
            self.moving[(src, dst)] = layers
            p.seed()
        self.target = new_owner
        self.pump()
        return moves

    def pump(self) -> int:
        """One patch round per migrating pair (MigrationStream.pump -> _drain ->
        _send_patch -> receive, migrator.py:208-273): drain the dirty cells (K3) and push
        them into the destination's pools (K4+K5).  Returns the cells moved."""
        cells_total = 0
        rank = self.registry.rank()
        for (src, dst), p in self.patches.items():
            keys, cells = p.push(self.stores[dst], rank)
            cells_total += cells
            self.patched_bytes += cells * self.cfg.cell_bytes
        return cells_total

    def lag(self) -> int:
        """Dirty keys not yet drained, over every pair (the converged() test's t_sched -
        t_applied, migrator.py:341-348, once the in-flight patch has been applied)."""
        return sum(p.dirty_keys() for p in self.patches.values())

    def switch(self) -> int:
        """Phase 5 (coordinator.py:275-338): with decode paused between steps, the residual
        patch of every pair is applied, layer ownership flips to the target, and the
        sources drop the layers that left (post-commit cleanup, coordinator.py:340-354)."""
        residual = self.pump()
        for (src, dst), layers in self.moving.items():
            for l in layers:
                self.owner[l] = dst
        self._leaving = dict(self.moving)
        self._closing = dict(self.patches)
        self.patches.clear()
        self.moving.clear()
        return residual

    def post_commit(self) -> None:
        """After the pause (Coordinator._post_commit_cleanup, coordinator.py:340-354, runs
        after commit_pause_end): the pairs' patch engines close and the sources drop the
        layers that left."""
        for p in getattr(self, "_closing", {}).values():
            p.close()
        for (src, dst), layers in getattr(self, "_leaving", {}).items():
            self.stores[src].drop_layer_groups([l - 1 for l in layers])
        self._closing, self._leaving = {}, {}


def generate(model: StagedLlama, prompts: list[list[int]], joins: list[int], n_gen: int,
             reconfig: tuple[int, dict] | None = None, switch_at: int | str | None = None,
             record: list | None = None, trace=None, tau: int = 50) -> list[list[int]]:
    """Greedy decode of len(prompts) requests that join at steps `joins`, one token per
    request per step (prompt tokens are fed one at a time).  `reconfig` = (step, target
    config) starts a live reconfiguration after that step; `switch_at` commits it (a step,
    or "converged": at the first step whose lag -- cells written since the last patch
    round -- is below `tau`, the reference's dirty-set threshold).
    `record` (optional) receives (rids, tokens, positions, logits) per step; `trace`
    (an events.EventTrace) receives the run's events in the reference's trace schema with
    wall-clock times, so engine.compute_metrics gives TTFT/TPOT (engine.py:112-184)."""
    torch = model.torch

    def step(rids, toks, poss):
        tok_t = torch.tensor(toks, dtype=torch.long, device=f"cuda:{model.device}")
        logits = model.step(rids, tok_t)
        nxt = logits.argmax(-1).tolist()
        if record is not None:
            record.append((rids, toks, poss, logits.cpu().numpy()))
        return nxt

    with model.on_stream():
        return _drive(model, step, prompts, joins, n_gen, reconfig, switch_at, trace,
                      lambda: bool(model.patches), tau)


def _drive(model, step, prompts, joins, n_gen, reconfig, switch_at, trace, migrating,
           tau: int = 50):
    import time

    t_start = time.perf_counter()

    def emit(kind, **payload):
        if trace is not None:
            trace.emit(time.perf_counter() - t_start, "engine", kind, **payload)

    B = len(prompts)
    outs: list[list[int]] = [[] for _ in range(B)]
    t = 0
    while any(len(o) < n_gen for o in outs):
        act = [b for b in range(B) if joins[b] <= t and len(outs[b]) < n_gen]
        for b in act:
            if t == joins[b]:
                emit("request_arrival", id=f"seq{b}", input_len=len(prompts[b]), output_len=n_gen)
        if act:
            toks, poss = [], []
            for b in act:
                p = t - joins[b]
                toks.append(prompts[b][p] if p < len(prompts[b]) else outs[b][-1])
                poss.append(p)
            t_step = time.perf_counter()
            nxt = step([f"seq{b}" for b in act], toks, poss)
            emit("decode_step", step=t, batch=len(act),
                 ms=round((time.perf_counter() - t_step) * 1e3, 4))
            for b, p, n in zip(act, poss, nxt):
                if p >= len(prompts[b]) - 1:
                    outs[b].append(int(n))
                    if len(outs[b]) == 1:
                        emit("first_token", id=f"seq{b}")
                    if len(outs[b]) == n_gen:
                        emit("request_done", id=f"seq{b}")
        converged = False
        if reconfig is not None and t == reconfig[0]:
            emit("reconfigure_start", target={str(k): v for k, v in reconfig[1].items()})
            model.start_reconfig(reconfig[1])
            emit("migration_seeded")
        elif migrating():
            # the safe-switch test (migrator.py:341-348, tau = 50 cells by default,
            # scenario.py:82): cells written since the last round and not yet patched
            lag = model.lag()
            emit("convergence_check", lag=lag, tau=tau)
            if switch_at == "converged" and lag < tau:
                converged = True
            else:
                model.pump()
                emit("patch_round")
        if converged or (switch_at is not None and t == switch_at):
            emit("commit_pause_start")
            model.switch()
            emit("commit_pause_end")
            # post-commit cleanup after the pause, as the reference orders it
            # (coordinator.py:326-334: commit_pause_end, resume, _post_commit_cleanup)
            model.post_commit()
            emit("reconfigure_end", outcome="success")
        t += 1
    return outs


# ======================================================================================
# One process per stage GPU: activations over a torch.distributed group
# (StageLink, K7), KV patches over the cross-process push (dist.PatchSender/Receiver).
class DistStagedLlama:
    """This rank's stage of a pipeline whose stages are processes.  Every rank runs the
    same step schedule; stage i receives the hidden states from the previous stage,
    runs its layers over its own store and sends them on; the last stage's greedy tokens
    are broadcast so every rank knows the next inputs."""

    def __init__(self, cfg: LlamaConfig, weights: dict[str, np.ndarray],
                 config: dict[int, list[int]], rank: int, device: int = 0,
                 tokens_per_block: int = 16, capacity_blocks: int = 256,
                 registry: RequestRegistry | None = None, channel_prefix: str = "pl",
                 group=None, exact: bool = False, act_mode: str | None = None) -> None:
        import torch

        from .dist import StageLink

        self.torch = torch
        self.cfg = cfg
        self.rank = rank
        self.gpu = rank + 1                       # pipeline GPU id of this process
        self.device = device
        self.prefix = channel_prefix
        self.group = group
        self.registry = registry or RequestRegistry()
        self.stream = torch.cuda.Stream(device=device)
        self.link = StageLink(group, mode=act_mode, prefix=channel_prefix, device=device)
        self.owner = {l: g for g, ls in config.items() for l in ls}
        own_layers = [l for l, g in self.owner.items() if g == self.gpu]
        self.compute = LlamaCompute(cfg, weights, device, self.registry, self.stream,
                                    layers=own_layers, exact=exact)
        # every layer's weights sit in pinned host memory; arriving layers are staged on
        # a copy engine during the migration and gate the switch (coordinator.py:239-240)
        from .staging import LayerWeightStager

        host = {}
        for l in range(1, cfg.n_layers + 1):
            pre = f"l{l - 1}."
            host[l] = {k: torch.from_numpy(v).pin_memory() for k, v in weights.items()
                       if k.startswith(pre)}
        self.stager = LayerWeightStager(device, host,
                                        is_layer_committed=lambda l: self.owner.get(l) == self.gpu)
        mine = [l - 1 for l, g in self.owner.items() if g == self.gpu]
        self.store = KvStore(self.gpu, 1, tokens_per_block, capacity_blocks, mine,
                             num_groups=cfg.n_layers, cell_bytes=cfg.cell_bytes, device=device,
                             registry=self.registry)
        N.check(N.lib().pl_store_set_stream(self.store._h, C.c_void_p(self.stream.cuda_stream)))
        self.pos: dict = {}
        self.senders: dict = {}
        self.receivers: dict = {}
        self.moving: dict = {}

    def on_stream(self):
        return self.torch.cuda.stream(self.stream)

    def close(self) -> None:
        """Release the activation rings and the closed pairs' patch engines (after every
        rank finished stepping)."""
        from .dist import reap_patches

        self.stream.synchronize()
        reap_patches()
        self.link.close()

    def _order(self) -> list[int]:
        return pipeline_order(self.owner)

    def step_tokens(self, rids: list, tokens: list[int]) -> list[int]:
        torch, c = self.torch, self.cfg
        dev = torch.device("cuda", self.device)
        order = self._order()
        B = len(rids)
        sc = self.compute.begin(rids, [self.pos.get(r, 0) for r in rids], dev)
        nxt = torch.empty(B, dtype=torch.long)
        if self.gpu in order:
            i = order.index(self.gpu)
            if i == 0:
                x = self.compute.embed(torch.tensor(tokens, dtype=torch.long, device=dev))
            else:
                if self.link.host_staged:
                    self.stream.synchronize()
                # device path: the stage's stream waits for the previous stage's copy
                x = self.link.recv((B, c.d_model), self.compute.act_dtype, order[i - 1] - 1, dev)
            for l in sorted(l for l, g in self.owner.items() if g == self.gpu):
                x = self.compute.layer(l - 1, x, self.store, sc)
            if i + 1 < len(order):
                if self.link.host_staged:
                    self.stream.synchronize()
                self.link.send(x, order[i + 1] - 1)
            else:
                nxt = self.compute.head(x).argmax(-1).cpu()
        self.link.dist.broadcast(nxt, order[-1] - 1, group=self.group)
        for r in rids:
            self.pos[r] = self.pos.get(r, 0) + 1
        return [int(t) for t in nxt]

    # ---------------------------------------------------------------- live reconfiguration
    def _pairs(self):
        return sorted(self.moving)

    def start_reconfig(self, target: dict[int, list[int]]) -> None:
        from .dist import Channel, PatchReceiver, PatchSender, reap_patches

        reap_patches()   # engines of an earlier reconfiguration's pairs
        new_owner = {l: g for g, ls in target.items() for l in ls}
        moves = layer_moves(self.owner, target)
        self.moving = moves
        self.target = new_owner
        arriving = [l for (src, dst), ls in moves.items() if dst == self.gpu for l in ls]
        if arriving:
            self.stager.stage_layers(arriving)
        # channels are set up in one global pair order on every rank (no wait cycles)
        for (src, dst) in self._pairs():
            groups = [l - 1 for l in moves[(src, dst)]]
            name = f"{self.prefix}-{src}-{dst}"
            if dst == self.gpu:
                self.receivers[(src, dst)] = PatchReceiver(self.store, groups,
                                                           Channel(name, server=True))
            elif src == self.gpu:
                tx = PatchSender(self.store, groups, 1, Channel(name, server=False),
                                 self.registry.rank)
                tx.seed()
                self.senders[(src, dst)] = tx
        self.pump()

    def pump(self) -> None:
        for pair in self._pairs():
            if pair in self.senders:
                self.senders[pair].round()
            elif pair in self.receivers:
                assert self.receivers[pair].serve()

    def lag(self) -> int:
        """Dirty cells not yet patched, summed over every pair of every rank (all ranks
        take the same switch decision)."""
        import torch

        mine = sum(tx.dirty_keys() for tx in self.senders.values())
        t = torch.tensor([mine], dtype=torch.int64)
        if self.link.backend == "nccl":
            t = t.cuda(self.device)
        self.link.dist.all_reduce(t, group=self.group)
        return int(t.item())

    def switch(self) -> None:
        t0 = time.perf_counter()
        # the commit waits for the arriving layers' weights (coordinator.py:239-240)
        self.stager.wait()
        self.stager.make_current_wait(self.stream)
        for (src, dst), layers in self.moving.items():
            if dst == self.gpu:
                for l in layers:
                    self.compute.w.update({k: t.to(self.compute.act_dtype)
                                           for k, t in self.stager.resident[l].items()})
        t1 = time.perf_counter()
        self.pump()                     # residual patch of every pair
        t2 = time.perf_counter()
        # the residual is applied on every destination once each receiver's stream waits on
        # its sender's push (serve_ack, device-side); ownership flips and decode resumes.
        # Tearing the pairs down (sync + unmap of the imported pools) and dropping the
        # leaving groups is post-commit cleanup (post_commit, after commit_pause_end).
        for (src, dst), layers in self.moving.items():
            for l in layers:
                self.owner[l] = dst
        self._leaving = dict(self.moving)
        self.moving = {}
        self.switch_phases_ms = {"weights": round((t1 - t0) * 1e3, 3),
                                 "residual_round": round((t2 - t1) * 1e3, 3)}

    def post_commit(self) -> None:
        """Coordinator._post_commit_cleanup (coordinator.py:340-354), after the pause: every
        pair closes (one global pair order on every rank), the sources drop the groups and
        evict the weights of the layers that left."""
        t2 = time.perf_counter()
        close_detail = {}
        for pair in sorted(getattr(self, "_leaving", {})):
            if pair in self.senders:
                tx = self.senders.pop(pair)
                tx.close()
                close_detail[f"{pair[0]}->{pair[1]}"] = getattr(tx, "close_phases_ms", None)
            elif pair in self.receivers:
                tr = time.perf_counter()
                assert not self.receivers.pop(pair).serve()
                close_detail[f"{pair[0]}->{pair[1]} rx"] = round((time.perf_counter() - tr) * 1e3, 3)
        t3 = time.perf_counter()
        t_drop = 0.0
        for (src, dst), layers in getattr(self, "_leaving", {}).items():
            if src == self.gpu:
                td = time.perf_counter()
                self.store.drop_layer_groups([l - 1 for l in layers])
                t_drop += time.perf_counter() - td
                # the leaving layers' weights go too (post-commit evict, coordinator.py:340-354)
                for l in layers:
                    for k in [k for k in self.compute.w if k.startswith(f"l{l - 1}.")]:
                        del self.compute.w[k]
                self.stager.evict_layers([l for l in layers if l in self.stager.resident])
        self._leaving = {}
        ms = lambda a, b: round((b - a) * 1e3, 3)  # noqa: E731
        # after the pause: pair teardown (close handshake, sync, unmap), drop + evict
        self.post_commit_ms = {"pair_close": ms(t2, t3), "drop_evict": ms(t3, time.perf_counter()),
                               "drop": round(t_drop * 1e3, 3),
                               "close_detail": close_detail}


def step_latency_around_switch(trace) -> dict:
    """Median decode-step latency before the reconfiguration, while it migrates, and after
    the switch (TPOT across the switch), plus the pause."""
    phase, out = "before", {"before": [], "migrating": [], "after": []}
    pause = 0.0
    t0 = None
    for ev in trace:
        if ev.kind == "reconfigure_start":
            phase = "migrating"
        elif ev.kind == "commit_pause_start":
            t0 = ev.time
        elif ev.kind == "commit_pause_end":
            pause += ev.time - t0
            phase = "after"
        elif ev.kind == "decode_step":
            out[phase].append(ev.payload["ms"])
    res = {k: (round(float(np.median(v)), 4) if v else None) for k, v in out.items()}
    res["steps"] = {k: len(v) for k, v in out.items()}
    res["pause_ms"] = round(pause * 1e3, 4)
    return res


def generate_dist(model: DistStagedLlama, prompts: list[list[int]], joins: list[int], n_gen: int,
                  reconfig: tuple[int, dict] | None = None,
                  switch_at: int | str | None = None, trace=None,
                  tau: int = 50) -> list[list[int]]:
    """generate() with the stages in separate processes; every rank returns the tokens
    (pass `trace` on one rank to record the run's events)."""
    with model.on_stream():
        return _drive(model, lambda rids, toks, poss: model.step_tokens(rids, toks), prompts,
                      joins, n_gen, reconfig, switch_at, trace, lambda: bool(model.moving), tau)
