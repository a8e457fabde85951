"""CPU oracle (test infrastructure only) — per-kernel numpy restatements.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module, and only as the checker.  The product path never imports it.

The reference (arxiv 2603.12831 `hybridserve`) pins no numerics: its layer is
a cost charge, "a symbolic computation trace substitutes for numerical
correctness" (reference SPEC.md:8).  What it does pin is the module sequence
of one layer, QKV -> Attn -> Proj -> ResidualAdd -> MLP -> ResidualAdd
(reference pkg/src/hybridserve/engine.py:56), decode attention over ctx+1
tokens (engine.py:675,740) and causal chunked prefill over
pairwise_units (scheduling.py:127-133).  The arithmetic of each module is the
standard Llama block (RMSNorm, rotate-half RoPE, GQA attention, SwiGLU); its
restatement here is pinned against HF transformers' LlamaModel with the same
weights (tests/golden/hf_tiny_*.npz, made by oracle/gen_hf_golden.py).
"""

from __future__ import annotations

import numpy as np


def to_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bfloat16 (round-to-nearest-even), as float32."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = rounded.astype(np.uint32).view(np.float32)
    # keep NaN payloads NaN
    return np.where(np.isnan(a), a, out).reshape(a.shape)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 (already bf16-valued) -> uint16 bit patterns."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def rope_tables(max_pos: int, head_dim: int, theta: float) -> tuple[np.ndarray, np.ndarray]:
    """cos/sin tables [max_pos, head_dim/2]: HF LlamaRotaryEmbedding's
    inverse frequencies theta^(-2i/hd) and angles pos * inv, both evaluated in
    float64 and rounded to fp32 once (HF rounds the inverse frequency to fp32
    first; at the 9k-32k positions of long BE contexts that alone moves the
    angle by ~5e-4 rad, far above the fp32 validation bound)."""
    half = head_dim // 2
    inv = 1.0 / (float(theta) ** (np.arange(0, head_dim, 2, dtype=np.float64) / head_dim))
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :half]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def apply_rope(x: np.ndarray, pos: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """x: [rows, heads, hd] fp32, pos: [rows] -> rotate-half RoPE."""
    half = x.shape[-1] // 2
    c = cos[pos][:, None, :]
    s = sin[pos][:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1).astype(np.float32)


def rmsnorm(h: np.ndarray, w: np.ndarray, eps: float) -> np.ndarray:
    """fp32 RMSNorm of the fp32 residual stream, result rounded to bf16."""
    h64 = h.astype(np.float64)
    inv = 1.0 / np.sqrt((h64 * h64).mean(axis=-1, keepdims=True) + eps)
    return to_bf16((h64 * inv * w.astype(np.float64)).astype(np.float32))


def gemm(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """x [t, k] @ w[n, k]^T with fp64 accumulation -> fp32."""
    return (x.astype(np.float64, copy=False) @ w.astype(np.float64, copy=False).T).astype(
        np.float32)


def silu_mul(gate_up: np.ndarray, ffn: int) -> np.ndarray:
    g = gate_up[..., :ffn].astype(np.float64)
    u = gate_up[..., ffn:].astype(np.float64)
    return to_bf16((g / (1.0 + np.exp(-g)) * u).astype(np.float32))


def attention_rows(q: np.ndarray, k: np.ndarray, v: np.ndarray, n_kv: int,
                   mask: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray]:
    """GQA softmax attention.

    q: [nq_rows, n_q, hd]; k, v: [n_keys, n_kv, hd]; mask: [nq_rows, n_keys]
    (True = attend).  Returns (out [nq_rows, n_q, hd] fp32, lse [nq_rows, n_q]
    natural log).
    """
    n_q, hd = q.shape[1], q.shape[2]
    group = n_q // n_kv
    kx = np.repeat(k.astype(np.float64), group, axis=1)  # [keys, n_q, hd]
    vx = np.repeat(v.astype(np.float64), group, axis=1)
    s = np.einsum("rhd,khd->rhk", q.astype(np.float64), kx) / np.sqrt(hd)
    if mask is not None:
        s = np.where(mask[:, None, :], s, -np.inf)
    m = s.max(axis=-1, keepdims=True)
    p = np.exp(s - m)
    l_ = p.sum(axis=-1, keepdims=True)
    out = np.einsum("rhk,khd->rhd", p / l_, vx)
    lse = (m + np.log(l_))[..., 0]
    return out.astype(np.float32), lse.astype(np.float32)


def decode_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, n_kv: int):
    """One decode row: q [n_q, hd] over ctx+1 keys k/v [keys, n_kv, hd]."""
    o, lse = attention_rows(q[None], k, v, n_kv)
    return o[0], lse[0]


def prefill_attention(q: np.ndarray, pos: np.ndarray, k: np.ndarray, v: np.ndarray, n_kv: int):
    """Causal chunk: query rows at absolute positions `pos` over keys 0..max(pos)."""
    keys = np.arange(k.shape[0])
    mask = keys[None, :] <= pos[:, None]
    return attention_rows(q, k, v, n_kv, mask)


def lse_merge(parts: np.ndarray, lse: np.ndarray) -> np.ndarray:
    """parts [P, n_q, hd] (normalised), lse [P, n_q] -> merged [n_q, hd]."""
    m = lse.max(axis=0)
    w = np.exp(lse.astype(np.float64) - m)
    return ((w[..., None] * parts.astype(np.float64)).sum(0) / w.sum(0)[..., None]).astype(
        np.float32)


def argmax_first(logits: np.ndarray) -> np.ndarray:
    """Greedy token per row, lowest index on ties (numpy semantics)."""
    return np.argmax(logits, axis=-1).astype(np.int32)
