"""numpy oracle of the tiny Llama decode -- TEST INFRASTRUCTURE ONLY.

The reference has no model (engine.py:343-347 is a cost model), so generated
token ids are "parity unpinned" against it; this oracle pins
them to the textbook Llama decoder (RMSNorm, RoPE rotate-half, GQA attention,
SwiGLU MLP) evaluated in fp32 with exactly the roundings the device path applies:
K, V, q rounded to bf16 before attention (the paged cells and K2's operands are
bf16) and the attention output rounded to bf16 (K2 writes bf16).  Weights are an
explicit input, shared with the GPU run.
"""

from __future__ import annotations

import numpy as np

from .attention import bf16_to_f32, decode_attention, f32_to_bf16


def bf16_round(x: np.ndarray) -> np.ndarray:
    return bf16_to_f32(f32_to_bf16(x))


def rmsnorm(x: np.ndarray, w: np.ndarray, eps: float) -> np.ndarray:
    var = (x.astype(np.float64) ** 2).mean(-1, keepdims=True)
    return (x / np.sqrt(var + eps)).astype(np.float32) * w


def rope(x: np.ndarray, pos: np.ndarray, theta: float) -> np.ndarray:
    """x [B, H, D] rotated by the positions pos [B] (rotate-half convention)."""
    D = x.shape[-1]
    inv = 1.0 / (theta ** (np.arange(0, D, 2, dtype=np.float64) / D))
    ang = pos[:, None].astype(np.float64) * inv[None, :]             # [B, D/2]
    cos = np.cos(ang).astype(np.float32)[:, None, :]
    sin = np.sin(ang).astype(np.float32)[:, None, :]
    x1, x2 = x[..., : D // 2], x[..., D // 2:]
    return np.concatenate([x1 * cos - x2 * sin, x2 * cos + x1 * sin], axis=-1)


class OracleLlama:
    """Per-sequence KV lists (bf16-rounded fp32) and one decode step at a time."""

    def __init__(self, cfg, weights: dict) -> None:
        self.cfg = cfg
        self.w = weights
        self.k: dict = {}   # (seq, layer) -> list of [n_kv, D]
        self.v: dict = {}

    def step(self, seqs: list, tokens: np.ndarray, pos: np.ndarray) -> np.ndarray:
        """tokens [B] at positions pos [B] -> logits [B, vocab] (fp32)."""
        c, w = self.cfg, self.w
        B = len(seqs)
        x = w["embed"][tokens].astype(np.float32)
        for li in range(c.n_layers):
            h = rmsnorm(x, w[f"l{li}.attn_norm"], c.eps)
            q = (h @ w[f"l{li}.wq"]).reshape(B, c.n_q, c.head_dim)
            k = (h @ w[f"l{li}.wk"]).reshape(B, c.n_kv, c.head_dim)
            v = (h @ w[f"l{li}.wv"]).reshape(B, c.n_kv, c.head_dim)
            q = bf16_round(rope(q, pos, c.rope_theta))
            k = bf16_round(rope(k, pos, c.rope_theta))
            v = bf16_round(v)
            ks, vs = [], []
            for b, sq in enumerate(seqs):
                self.k.setdefault((sq, li), []).append(k[b])
                self.v.setdefault((sq, li), []).append(v[b])
                ks.append(np.stack(self.k[(sq, li)]))
                vs.append(np.stack(self.v[(sq, li)]))
            att = bf16_round(decode_attention(q, ks, vs, c.head_dim ** -0.5))
            x = x + att.reshape(B, -1) @ w[f"l{li}.wo"]
            h = rmsnorm(x, w[f"l{li}.mlp_norm"], c.eps)
            a = h @ w[f"l{li}.w1"]
            x = x + ((a / (1.0 + np.exp(-a))) * (h @ w[f"l{li}.w3"])) @ w[f"l{li}.w2"]
        return rmsnorm(x, w["final_norm"], c.eps) @ w["lm_head"]


# ======================================================================================
# Exact mode: the same decode step with every operation's order and rounding fixed
# (llama_exact.c), which the GPU's exact mode (csrc/exact.cu) reproduces bit for bit.
def rope_tables(pos: np.ndarray, head_dim: int, theta: float) -> tuple[np.ndarray, np.ndarray]:
    """cos/sin [B, D/2] (float64) for positions pos [B]: the tables both sides consume."""
    inv = 1.0 / (theta ** (np.arange(0, head_dim, 2, dtype=np.float64) / head_dim))
    ang = np.asarray(pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.ascontiguousarray(np.cos(ang)), np.ascontiguousarray(np.sin(ang))


class ExactOracleLlama:
    """Greedy decode in the exact arithmetic of llama_exact.c: fp64 logits, bit-identical
    to the GPU's exact mode; per-sequence KV as bf16-valued doubles."""

    def __init__(self, cfg, weights: dict) -> None:
        from . import lib
        self.L = lib()
        self.cfg = cfg
        self.w = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in weights.items()}
        self.k: dict = {}   # (seq, layer) -> list of [n_kv, D]
        self.v: dict = {}

    @staticmethod
    def _p(a):
        import ctypes as C
        return C.c_void_p(a.ctypes.data) if a is not None else None

    def _gemv(self, x, w, resid=None):
        B, I = x.shape
        O = w.shape[1]
        out = np.empty((B, O), dtype=np.float64)
        self.L.or_ex_gemv(self._p(x), self._p(w), self._p(resid), self._p(out), B, I, O)
        return out

    def _rmsnorm(self, x, g):
        out = np.empty_like(x)
        self.L.or_ex_rmsnorm(self._p(x), self._p(g), self._p(out), x.shape[0], x.shape[1],
                             float(self.cfg.eps))
        return out

    def step(self, seqs: list, tokens, pos) -> np.ndarray:
        """tokens [B] at positions pos [B] -> logits [B, vocab] (float64)."""
        c, w = self.cfg, self.w
        B, D = len(seqs), c.head_dim
        cos, sin = rope_tables(np.asarray(pos), D, c.rope_theta)
        x = np.ascontiguousarray(w["embed"][np.asarray(tokens)])
        for li in range(c.n_layers):
            h = self._rmsnorm(x, w[f"l{li}.attn_norm"])
            q = self._gemv(h, w[f"l{li}.wq"])
            k = self._gemv(h, w[f"l{li}.wk"])
            v = self._gemv(h, w[f"l{li}.wv"])
            self.L.or_ex_rope(self._p(q), self._p(cos), self._p(sin), B, c.n_q, D, 1)
            self.L.or_ex_rope(self._p(k), self._p(cos), self._p(sin), B, c.n_kv, D, 1)
            v = np.vectorize(self.L.or_bf16_round, otypes=[np.float64])(v)
            q, k, v = (a.reshape(B, -1, D) for a in (q, k, v))
            att = np.empty((B, c.n_q, D), dtype=np.float64)
            for b, sq in enumerate(seqs):
                self.k.setdefault((sq, li), []).append(k[b].copy())
                self.v.setdefault((sq, li), []).append(v[b].copy())
                ks = np.ascontiguousarray(np.stack(self.k[(sq, li)]))
                vs = np.ascontiguousarray(np.stack(self.v[(sq, li)]))
                n = ks.shape[0]
                scratch = np.empty(n, dtype=np.float64)
                qb = np.ascontiguousarray(q[b])
                ob = np.empty((c.n_q, D), dtype=np.float64)
                self.L.or_ex_attn(self._p(qb), self._p(ks), self._p(vs), n, c.n_q, c.n_kv, D,
                                  float(D) ** -0.5, self._p(scratch), self._p(ob))
                att[b] = ob
            x = self._gemv(np.ascontiguousarray(att.reshape(B, -1)), w[f"l{li}.wo"], x)
            h = self._rmsnorm(x, w[f"l{li}.mlp_norm"])
            a = self._gemv(h, w[f"l{li}.w1"])
            g = self._gemv(h, w[f"l{li}.w3"])
            m = np.empty_like(a)
            self.L.or_ex_silu_mul(self._p(a), self._p(g), self._p(m), a.size)
            x = self._gemv(m, w[f"l{li}.w2"], x)
        return self._gemv(self._rmsnorm(x, w["final_norm"]), w["lm_head"])

    def generate(self, prompts: list[list[int]], joins: list[int], n_gen: int) -> list[list[int]]:
        """The schedule of paper_2604_12171_b200.llama.generate (one token per active
        request per step, prompts fed one token at a time), greedy (first max)."""
        B = len(prompts)
        outs: list[list[int]] = [[] for _ in range(B)]
        t = 0
        while any(len(o) < n_gen for o in outs):
            act = [b for b in range(B) if joins[b] <= t and len(outs[b]) < n_gen]
            if act:
                toks, poss = [], []
                for b in act:
                    p = t - joins[b]
                    toks.append(prompts[b][p] if p < len(prompts[b]) else outs[b][-1])
                    poss.append(p)
                logits = self.step([f"seq{b}" for b in act], toks, poss)
                for b, p, row in zip(act, poss, logits):
                    if p >= len(prompts[b]) - 1:
                        outs[b].append(int(np.argmax(row)))
            t += 1
        return outs
