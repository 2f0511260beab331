"""fp32 numpy oracle of paged-attention decode -- TEST INFRASTRUCTURE ONLY.

The reference has no attention (decode is the cost model at engine.py:343-347),
so this is the new oracle SURVEY.md §8c asks for ("parity unpinned" against
the reference; pinned instead to the textbook definition softmax(q k^T * scale) v
with GQA head mapping q_head -> q_head // (n_q / n_kv)).  It reads K/V through
the same block tables the kernel uses, gathering token rows from an explicit
pool array laid out like the device units.
"""

from __future__ import annotations

import numpy as np


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """round-to-nearest-even fp32 -> bf16 bit pattern"""
    u = np.asarray(x, dtype=np.float32).view(np.uint32)
    rounding = ((u >> 16) & 1) + 0x7FFF
    return ((u + rounding) >> 16).astype(np.uint16)


def decode_attention(q: np.ndarray, k: list[np.ndarray], v: list[np.ndarray],
                     scale: float, with_atol: bool = False):
    """q [B, n_q, D] fp32; k[b], v[b] [ctx_b, n_kv, D] fp32 -> out [B, n_q, D] fp32.

    with_atol: also the elementwise absolute slack of a bf16 kernel, 2^-7 * E_p[|v|]
    (the softmax-weighted mean of |v| per output element): the kernel rounds P to bf16
    (2^-9 relative per weight, in numerator and denominator), which moves an output by
    up to ~2^-8 * E_p[|v|] whatever the output's own magnitude (cancellation), and
    rounds the output to bf16 (2^-9 relative, inside the 2e-2 relative term)."""
    B, n_q, D = q.shape
    out = np.zeros((B, n_q, D), dtype=np.float32)
    atol = np.zeros((B, n_q, D), dtype=np.float32)
    for b in range(B):
        kb, vb = k[b], v[b]
        if kb.shape[0] == 0:
            continue
        n_kv = kb.shape[1]
        group = n_q // n_kv
        for h in range(n_q):
            kv = h // group
            s = (kb[:, kv, :] @ q[b, h]) * np.float32(scale)
            s = s - s.max()
            p = np.exp(s.astype(np.float64)).astype(np.float32)
            out[b, h] = (p[:, None] * vb[:, kv, :]).sum(0) / p.sum()
            atol[b, h] = 2.0 ** -7 * (p[:, None] * np.abs(vb[:, kv, :])).sum(0) / p.sum()
    return (out, atol) if with_atol else out


def gather_paged(pool: np.ndarray, unit_bytes: int, fp_bytes: int, s: int, layer: int,
                 table: list[int], ctx: int, n_kv: int, D: int) -> tuple[np.ndarray, np.ndarray]:
    """K, V [ctx, n_kv, D] (bf16 bits) of one sequence from a byte pool of units."""
    cell = 2 * n_kv * D * 2
    ks, vs = [], []
    for t in range(ctx):
        base = table[t // s] * unit_bytes + fp_bytes + (layer * s + t % s) * cell
        row = pool[base: base + cell].view(np.uint16)
        ks.append(row[: n_kv * D].reshape(n_kv, D))
        vs.append(row[n_kv * D:].reshape(n_kv, D))
    if not ks:
        z = np.zeros((0, n_kv, D), np.uint16)
        return z, z
    return np.stack(ks), np.stack(vs)
