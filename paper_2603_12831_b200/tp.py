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


# ---------------------------------------------------------------- live mode
#
# A live TP group has one planner: rank 0 runs the LiveEngine and its
# context is wrapped in a MirrorContext that forwards every state-changing
# libhs call to the followers (one message per iteration over
# torch.distributed); the followers replay the calls on their own shard
# contexts.  The merge decisions need no message at all: with device-polled
# merges every rank's controller reads all ranks' completion tags (shared
# host segments, hs_pg_share_tags) and merges an item only once every rank's
# CPU pool has finished its heads, so the ranks take identical decisions on
# identical FIFOs -- the per-layer agreement a live group needs.  The
# fused all-reduce keeps the residual streams (and the tokens) bit-identical.

# calls that change device or replica state, in the order rank 0 issued them
# (cpu_submit only occurs with host-decided merges, which a live group cannot
# use on GPUs: rank 0 alone would see its own pool's completions)
_MIRRORED = ("set_page_table", "host_kv_reserve", "host_kv_release", "iter_begin", "layer",
             "pg_inject", "pg_stop", "pg_iter", "pg_enable", "iter_end_async", "swap_async",
             "cpu_submit", "sync")


def share_tags(ctx, rank: int, world: int, prefix: str, group=None) -> None:
    """Merge agreement across a TP group (hs_pg_share_tags, two phases
    around a barrier).  The context must have device-polled merges on."""
    import torch.distributed as dist

    ctx.pg_share_tags(prefix, rank, world, 0)
    dist.barrier(group=group)
    ctx.pg_share_tags(prefix, rank, world, 1)
    dist.barrier(group=group)


class MirrorContext:
    """Rank 0's HsContext, recording the state-changing calls for the
    followers (`flush` ships them; `swap_done` turning true is recorded as a
    wait, so a follower never uses pages its own copy has not landed)."""

    def __init__(self, ctx, group=None):
        self._ctx, self._group = ctx, group
        self._cmds: list = []

    def __getattr__(self, name):
        attr = getattr(self._ctx, name)
        if name not in _MIRRORED:
            return attr

        def call(*a, **kw):
            self._cmds.append((name, a, kw))
            return attr(*a, **kw)

        return call

    def swap_done(self, ticket: int) -> bool:
        done = self._ctx.swap_done(ticket)
        if done:
            self._cmds.append(("swap_wait", (ticket,), {}))
        return done

    def flush(self, stop: bool = False) -> None:
        import torch.distributed as dist

        msg = [(self._cmds, stop)]
        self._cmds = []
        dist.broadcast_object_list(msg, src=0, group=self._group)


def follow(ctx, group=None, on_iteration=None) -> int:
    """A follower rank: replay rank 0's calls on this rank's shard context
    until rank 0 stops; `on_iteration(ticket)` after each replayed
    iteration end.  Returns the number of iterations replayed."""
    import time

    import torch.distributed as dist

    n = 0
    ctx.anchor()  # iteration completion times are reported relative to it
    while True:
        msg = [None]
        dist.broadcast_object_list(msg, src=0, group=group)
        cmds, stop = msg[0]
        for name, a, kw in cmds:
            if name == "swap_wait":
                while not ctx.swap_done(a[0]):
                    time.sleep(5e-5)
                continue
            out = getattr(ctx, name)(*a, **kw)
            if name == "iter_end_async":
                n += 1
                if on_iteration:
                    on_iteration(out)
        if stop:
            return n
