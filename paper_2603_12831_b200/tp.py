"""Tensor parallelism of the serving step (BASELINE config 4: Llama-3-70B,
TP=8 over NVLink, BE attention piggybacked on 8 NUMA-pinned CPU pools).

The reference charges TP as one collective cost per layer, gamma
(engine.py:944, LatencyModelSet.gamma latency.py:141-147, profiles.py:234).
Here it is real: every rank holds a Megatron-style shard of each layer

  * QKV and gate/up column-parallel (a rank owns n_q/W query heads, n_kv/W
    KV heads and ffn/W MLP columns),
  * O and down row-parallel (their partial sums are all-reduced),
  * embedding, norms and LM head replicated,

and the two all-reduces per layer are fused into the residual-add + RMSNorm
launches (libhs `tp_add_norm`): each rank publishes its local split-K sum and
reads its peers' straight from their HBM over NVLink P2P (CUDA IPC), summing
in rank order so the residual stream -- and therefore every greedy token --
is bit-identical on all ranks.  Attention Piggybacking is head-sharded: each
rank ships its own heads' q/k/v to its own CPU pool and merges its own heads'
results, so no collective is added for it.

A group is one process per rank (one GPU each); the ranks exchange their
IPC handles through torch.distributed (`open_group`) and then run identical
engines (the scheduler is deterministic), so every rank issues the same
hs_layer sequence with the same row counts.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import replace

import numpy as np

from .errors import ConfigError
from .models import TransformerConfig

HANDLE_BYTES = 128


def shard_config(cfg: TransformerConfig, world: int) -> TransformerConfig:
    """Per-rank dimensions of a `world`-way tensor-parallel shard."""
    if world < 1 or cfg.n_q % world or cfg.n_kv % world or cfg.ffn % world:
        raise ConfigError(f"{cfg.name}: heads ({cfg.n_q}/{cfg.n_kv}) and ffn ({cfg.ffn}) must "
                          f"divide by the tensor-parallel degree {world}")
    if world == 1:
        return cfg
    return replace(cfg, name=f"{cfg.name}-tp{world}", n_q=cfg.n_q // world,
                   n_kv=cfg.n_kv // world, ffn=cfg.ffn // world, tp=world)


def shard_weights(w: dict, cfg: TransformerConfig, rank: int, world: int) -> dict:
    """Rank `rank`'s shard of full-model weights in libhs' host format
    (bf16 bit patterns / fp32 norms, [out][in] matrices)."""
    hd = cfg.head_dim
    nq, nkv, f = cfg.n_q // world, cfg.n_kv // world, cfg.ffn // world
    q0, k0 = rank * nq * hd, rank * nkv * hd
    kb, vb = cfg.n_q * hd, cfg.n_q * hd + cfg.n_kv * hd

    def qkv(m):
        return np.ascontiguousarray(np.concatenate(
            [m[q0:q0 + nq * hd], m[kb + k0:kb + k0 + nkv * hd], m[vb + k0:vb + k0 + nkv * hd]]))

    def gate_up(m):
        g0 = rank * f
        return np.ascontiguousarray(np.concatenate([m[g0:g0 + f], m[cfg.ffn + g0:cfg.ffn + g0 + f]]))

    out = {k: w[k] for k in ("embed", "lm_head", "final_norm", "norm_in", "norm_post")}
    out["qkv"] = [qkv(m) for m in w["qkv"]]
    out["o"] = [np.ascontiguousarray(m[:, q0:q0 + nq * hd]) for m in w["o"]]
    out["gate_up"] = [gate_up(m) for m in w["gate_up"]]
    out["down"] = [np.ascontiguousarray(m[:, rank * f:(rank + 1) * f]) for m in w["down"]]
    return out


def _bind(lib) -> None:
    lib.hs_tp_export.argtypes = [C.c_void_p, C.c_void_p]
    lib.hs_tp_open.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    for f in (lib.hs_tp_export, lib.hs_tp_open):
        f.restype = C.c_int


def open_group(ctx, rank: int, world: int, group=None) -> None:
    """Form a TP group across processes (one rank per GPU): every rank's IPC
    handles are all-gathered over torch.distributed (any backend)."""
    import torch.distributed as dist

    from . import _lib

    lib = ctx.lib
    _bind(lib)
    mine = C.create_string_buffer(HANDLE_BYTES)
    _lib.check(lib.hs_tp_export(ctx.h, mine), "hs_tp_export")
    gathered = [None] * world
    dist.all_gather_object(gathered, mine.raw, group=group)
    blob = b"".join(gathered)
    _lib.check(lib.hs_tp_open(ctx.h, rank, world, C.c_char_p(blob)), "hs_tp_open")
