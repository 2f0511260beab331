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
