"""Host runtime of the B200 step: the libhs context wrapper and `CudaStep`,
the LayerStep that executes the engine's schedule on the GPU.

`CudaStep` turns the engine's events into libhs calls:

  Engine._start_iteration  -> begin_iteration: rows of the BatchPlan (decodes
                              first, then chunk tokens), split-K decode work
                              items, prefill tiles, logit rows   (hs_iter_begin)
  Engine._run_layer        -> layer: carry / merge / restart rows  (hs_layer)
  Engine._on_layer_done(L) -> end_iteration: greedy tokens back   (hs_iter_end)
  Engine._maybe_start_host -> cpu_service: host attention of the work items
                              (hs_cpu_attend)
  swap-out / resume / preempt / complete -> page + host-KV management

References: engine.py:879-1047 (iteration), 402-508 (swaps), 512-560 (CPU
service) of pkg/src/hybridserve.  There is no CPU fallback: without libhs
and an sm_100 device the constructor raises.
"""

from __future__ import annotations

import ctypes as C
import zlib
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .engine import (
    MERGE_CHAIN,
    MERGE_INJECT,
    MERGE_TOKEN_END,
    MERGE_TOKEN_NEXT,
    LayerStep,
)
from .errors import ScenarioError
from .models import TransformerConfig

PAGE = _lib.PAGE_TOKENS
_IP = C.POINTER(C.c_int)


class HsModelCfg(C.Structure):
    _fields_ = [("d_model", C.c_int), ("n_layers", C.c_int), ("n_q", C.c_int),
                ("n_kv", C.c_int), ("head_dim", C.c_int), ("ffn", C.c_int), ("vocab", C.c_int),
                ("rope_theta", C.c_float), ("norm_eps", C.c_float)]


class HsRtCfg(C.Structure):
    _fields_ = [("max_rows", C.c_int), ("max_slots", C.c_int), ("kv_pages", C.c_int),
                ("max_pages_per_req", C.c_int), ("max_pos", C.c_int), ("max_chunks", C.c_int),
                ("cpu_threads", C.c_int), ("host_kv_bytes", C.c_int64), ("device", C.c_int),
                ("cpu_list", _IP), ("n_cpu_list", C.c_int), ("precision", C.c_int)]

PRECISIONS = {"bf16": 0, "fp32": 1}  # HS_PREC_BF16 / HS_PREC_FP32 (include/hs.h)


class HsIterDesc(C.Structure):
    _fields_ = [("n_rows", C.c_int), ("n_decode", C.c_int), ("row_slot", _IP),
                ("row_pos", _IP), ("row_token", _IP), ("n_chunks", C.c_int), ("chunks", _IP),
                ("row_chunk_begin", _IP), ("n_tiles", C.c_int), ("tiles", _IP),
                ("n_logit_rows", C.c_int), ("logit_rows", _IP)]


class HsLayerDesc(C.Structure):
    _fields_ = [("layer", C.c_int), ("n_carry", C.c_int), ("carry_slot", _IP),
                ("carry_pos", _IP), ("n_merge", C.c_int), ("merge_slot", _IP),
                ("n_restart", C.c_int), ("restart_idx", _IP), ("restart_pos", _IP),
                ("merge_tag", _IP)]


def result_tag(ctx: int, layer: int) -> int:
    """HS_RESULT_TAG(ctx, layer) of include/hs.h: the completion tag a CPU
    worker publishes after writing a work item's result row."""
    v = ((ctx << 8) | layer) & 0xFFFFFFFF
    return v - (1 << 32) if v >= 1 << 31 else v


W_EMBED, W_LM_HEAD, W_FINAL_NORM, W_QKV, W_O, W_GATE_UP, W_DOWN, W_NORM_IN, W_NORM_POST = range(9)

_CTX_SIGS = {
    "hs_create": [C.POINTER(HsModelCfg), C.POINTER(HsRtCfg), C.POINTER(C.c_void_p)],
    "hs_destroy": [C.c_void_p],
    "hs_set_weight": [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_size_t],
    "hs_init_weights": [C.c_void_p, C.c_uint64, C.c_float],
    "hs_set_page_table": [C.c_void_p, C.c_int, _IP, C.c_int],
    "hs_host_kv_reserve": [C.c_void_p, C.c_int, C.c_int],
    "hs_host_kv_release": [C.c_void_p, C.c_int],
    "hs_host_kv_ptr": [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), _IP],
    "hs_swap_out": [C.c_void_p, C.c_int, C.c_int],
    "hs_swap_in": [C.c_void_p, C.c_int, C.c_int],
    "hs_iter_begin": [C.c_void_p, C.POINTER(HsIterDesc)],
    "hs_layer": [C.c_void_p, C.POINTER(HsLayerDesc)],
    "hs_iter_end": [C.c_void_p, _IP, C.c_int],
    "hs_cpu_attend": [C.c_void_p, _IP, _IP, _IP, C.c_int],
    "hs_sync": [C.c_void_p],
    "hs_keep_logits": [C.c_void_p, C.c_int],
    "hs_read_logits": [C.c_void_p, C.c_void_p, C.c_int],
    "hs_iter_logits": [C.c_void_p, C.c_int, C.c_void_p, C.c_int],
    "hs_read_ship": [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t],
    "hs_read_result": [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t],
    "hs_read_residual": [C.c_void_p, C.c_int, C.c_void_p],
    "hs_cpu_submit": [C.c_void_p, _IP, _IP, _IP, C.c_int],
    "hs_cpu_poll": [C.c_void_p, _IP, _IP, C.c_void_p, C.c_int],
    "hs_cpu_in_flight": [C.c_void_p],
    "hs_swap_out_async": [C.c_void_p, C.c_int, C.c_int, _IP],
    "hs_swap_in_async": [C.c_void_p, C.c_int, C.c_int, _IP],
    "hs_swap_done": [C.c_void_p, C.c_int],
    "hs_anchor": [C.c_void_p],
    "hs_iter_end_async": [C.c_void_p, _IP],
    "hs_iter_poll": [C.c_void_p, C.c_int, _IP, C.c_int, C.POINTER(C.c_double)],
    "hs_iter_ntokens": [C.c_void_p, C.c_int],
    "hs_mark": [C.c_void_p],
    "hs_wait_mark": [C.c_void_p, C.c_int],
    "hs_timer": [C.c_void_p],
    "hs_timer_elapsed": [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_float)],
    # device-polled merges
    "hs_pg_enable": [C.c_void_p, C.c_int],
    "hs_pg_inject": [C.c_void_p, _IP, _IP, _IP, C.c_int],
    "hs_pg_stop": [C.c_void_p, _IP, _IP, C.c_int],
    "hs_pg_iter": [C.c_void_p, C.c_int, _IP, C.c_int],
    "hs_pg_log": [C.c_void_p, C.c_int, _IP, C.c_int],
    "hs_pg_share_tags": [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.c_int],
    # remote CPU hosts (cpu_host.py)
    "hs_cpu_host_connect": [C.c_void_p, C.c_int, C.c_char_p, C.c_int],
    "hs_cpu_place": [C.c_void_p, C.c_int, C.c_int, C.c_int],
    "hs_cpu_remote_stats": [C.c_void_p, C.c_int, C.POINTER(C.c_int64)],
    "hs_cpu_fetch_async": [C.c_void_p, C.c_int, C.c_int],
    "hs_cpu_fetch_done": [C.c_void_p, C.c_int],
}
_NONNEG_RETURNS = {"hs_cpu_fetch_done", "hs_iter_end", "hs_cpu_poll", "hs_cpu_in_flight", "hs_swap_done", "hs_mark",
                   "hs_timer", "hs_iter_poll", "hs_iter_ntokens", "hs_pg_log"}
_lib._SIGNATURES.update(_CTX_SIGS)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_IP)


def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


@dataclass
class RuntimeConfig:
    max_rows: int = 1024
    max_slots: int = 256
    kv_pages: int = 1024
    max_pages_per_req: int = 256
    max_pos: int = 16384
    max_chunks: int = 4096
    cpu_threads: int = 8
    host_kv_bytes: int = 1 << 30
    device: int = 0
    cpu_list: tuple = ()  # the replica's CPU-attention cores (replicas.core_set)
    # "bf16" serving datapath, or "fp32" validation datapath (fp32 weights,
    # activations, KV, piggyback mailboxes and host attention; SIMT kernels)
    precision: str = "bf16"
    # remote CPU hosts 1..n of the scenario's cluster: (addr, port) of each
    # running `cpu_host` server, connected at context creation
    remote_hosts: tuple = ()


class HsContext:
    """Owns one libhs context (one GPU replica)."""

    def __init__(self, model: TransformerConfig, rt: RuntimeConfig):
        lib = _lib.load()
        for name, argtypes in _CTX_SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = C.c_int
        lib.hs_stream.argtypes = [C.c_void_p]
        lib.hs_stream.restype = C.c_void_p
        lib.hs_cpu_busy_seconds.argtypes = [C.c_void_p]
        lib.hs_cpu_busy_seconds.restype = C.c_double
        lib.hs_wall_seconds.argtypes = []
        lib.hs_wall_seconds.restype = C.c_double
        lib.hs_launch_count.argtypes = []
        lib.hs_launch_count.restype = C.c_ulonglong
        lib.hs_profile.argtypes = [C.c_void_p, C.c_int]
        lib.hs_profile.restype = C.c_int
        lib.hs_profile_read.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int]
        lib.hs_profile_read.restype = C.c_int
        _lib.require_device()
        self.lib = lib
        self.model = model
        self.rt = rt
        mc = HsModelCfg(model.d_model, model.n_layers, model.n_q, model.n_kv, model.head_dim,
                        model.ffn, model.vocab, model.rope_theta, model.norm_eps)
        cpus = np.asarray(rt.cpu_list or [], np.int32)
        if rt.precision not in PRECISIONS:
            from .errors import ConfigError

            raise ConfigError(f"precision {rt.precision!r} (choose from {sorted(PRECISIONS)})")
        rc = HsRtCfg(rt.max_rows, rt.max_slots, rt.kv_pages, rt.max_pages_per_req, rt.max_pos,
                     rt.max_chunks, rt.cpu_threads, rt.host_kv_bytes, rt.device,
                     cpus.ctypes.data_as(_IP) if len(cpus) else None, len(cpus),
                     PRECISIONS[rt.precision])
        h = C.c_void_p()
        _lib.check(lib.hs_create(C.byref(mc), C.byref(rc), C.byref(h)), "hs_create")
        self.h = h
        self._tok = np.zeros(2 * rt.max_rows, np.int32)
        self.remote_host_ids: set[int] = set()
        for i, (addr, port) in enumerate(getattr(rt, "remote_hosts", ()) or (), start=1):
            self.cpu_host_connect(i, addr, port)

    def close(self) -> None:
        if self.h:
            self.lib.hs_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _call(self, name: str, *args) -> int:
        rc = getattr(self.lib, name)(self.h, *args)
        if rc > 0 and name in _NONNEG_RETURNS:
            return rc
        if rc != 0:
            _lib.check(rc if rc > 0 else -rc, name)
        return rc

    @property
    def stream(self) -> int:
        return self.lib.hs_stream(self.h)

    # weights
    def set_weight(self, kind: int, layer: int, arr: np.ndarray) -> None:
        a = np.ascontiguousarray(arr)
        self._call("hs_set_weight", kind, layer, a.ctypes.data_as(C.c_void_p), a.nbytes)

    def init_weights(self, seed: int, std: float = 0.02) -> None:
        self._call("hs_init_weights", seed, std)

    def load_weights(self, w: dict) -> None:
        """w: numpy weights (bf16 bit patterns as uint16 for matrices, or
        fp32 matrices for the fp32 datapath; fp32 norms): embed, lm_head,
        final_norm, and per-layer lists."""
        self.set_weight(W_EMBED, 0, w["embed"])
        self.set_weight(W_LM_HEAD, 0, w["lm_head"])
        self.set_weight(W_FINAL_NORM, 0, w["final_norm"])
        for l in range(self.model.n_layers):
            self.set_weight(W_QKV, l, w["qkv"][l])
            self.set_weight(W_O, l, w["o"][l])
            self.set_weight(W_GATE_UP, l, w["gate_up"][l])
            self.set_weight(W_DOWN, l, w["down"][l])
            self.set_weight(W_NORM_IN, l, w["norm_in"][l])
            self.set_weight(W_NORM_POST, l, w["norm_post"][l])

    def set_page_table(self, slot: int, pages) -> None:
        p = _i32(pages)
        self._call("hs_set_page_table", slot, _ip(p), len(p))

    def host_kv_reserve(self, slot: int, cap: int) -> None:
        self._call("hs_host_kv_reserve", slot, cap)

    def host_kv_release(self, slot: int) -> None:
        self._call("hs_host_kv_release", slot)

    def swap_out(self, slot: int, tokens: int) -> None:
        self._call("hs_swap_out", slot, tokens)

    def swap_in(self, slot: int, tokens: int) -> None:
        self._call("hs_swap_in", slot, tokens)

    def iter_begin(self, rows_slot, rows_pos, rows_tok, n_decode, chunks, chunk_begin, tiles,
                   logit_rows) -> None:
        self._keep = [_i32(rows_slot), _i32(rows_pos), _i32(rows_tok),
                      _i32(chunks).reshape(-1), _i32(chunk_begin), _i32(tiles).reshape(-1),
                      _i32(logit_rows)]
        s, p, t, ch, cb, ti, lr = self._keep
        d = HsIterDesc(len(s), n_decode, _ip(s), _ip(p), _ip(t), len(ch) // 5, _ip(ch), _ip(cb),
                       len(ti) // 4, _ip(ti), len(lr), _ip(lr))
        self._call("hs_iter_begin", C.byref(d))

    def layer(self, layer: int, carry_slot, carry_pos, merge_slot, restart_idx, restart_pos,
              merge_tag=None):
        cs, cp, ms, ri, rp = (_i32(carry_slot), _i32(carry_pos), _i32(merge_slot),
                              _i32(restart_idx), _i32(restart_pos))
        mt = _i32(merge_tag) if merge_tag is not None else None
        d = HsLayerDesc(layer, len(cs), _ip(cs), _ip(cp), len(ms), _ip(ms), len(ri), _ip(ri),
                        _ip(rp), _ip(mt) if mt is not None else None)
        self._call("hs_layer", C.byref(d))

    def iter_end(self) -> np.ndarray:
        n = self.lib.hs_iter_end(self.h, _ip(self._tok), len(self._tok))
        if n < 0:
            _lib.check(-n if n < 0 else n, "hs_iter_end")
        return self._tok[:n].copy()

    def cpu_attend(self, slots, layers, ctxs) -> None:
        s, l, c = _i32(slots), _i32(layers), _i32(ctxs)
        self._call("hs_cpu_attend", _ip(s), _ip(l), _ip(c), len(s))

    def sync(self) -> None:
        self._call("hs_sync")

    # live mode
    def cpu_submit(self, slots, layers, ctxs) -> None:
        s, l, c = _i32(slots), _i32(layers), _i32(ctxs)
        self._call("hs_cpu_submit", _ip(s), _ip(l), _ip(c), len(s))

    def cpu_poll(self, max_items: int = 4096):
        s = np.zeros(max_items, np.int32)
        l = np.zeros(max_items, np.int32)
        n = self._call("hs_cpu_poll", _ip(s), _ip(l), None, max_items)
        return s[:n], l[:n]

    def cpu_host_connect(self, host: int, addr: str, port: int) -> None:
        self._call("hs_cpu_host_connect", host, addr.encode(), int(port))
        self.remote_host_ids.add(host)

    def cpu_place(self, slot: int, host: int, tokens: int) -> None:
        """Moves the slot's host KV (its first `tokens` tokens) to CPU host
        `host` (0 = this replica's own host)."""
        self._call("hs_cpu_place", slot, host, tokens)

    def cpu_fetch_async(self, slot: int, tokens: int) -> None:
        self._call("hs_cpu_fetch_async", slot, tokens)

    def cpu_fetch_done(self, slot: int) -> bool:
        return self._call("hs_cpu_fetch_done", slot) == 1

    def remote_stats(self, host: int) -> dict:
        out = (C.c_int64 * 4)()
        self._call("hs_cpu_remote_stats", host, out)
        return dict(zip(("items", "put_bytes", "get_bytes", "result_bytes"), list(out)))

    def cpu_busy_seconds(self) -> float:
        return self.lib.hs_cpu_busy_seconds(self.h)

    def swap_async(self, slot: int, tokens: int, out: bool) -> int:
        t = C.c_int(0)
        self._call("hs_swap_out_async" if out else "hs_swap_in_async", slot, tokens, C.byref(t))
        return t.value

    def swap_done(self, ticket: int) -> bool:
        return self._call("hs_swap_done", ticket) == 1

    def anchor(self) -> None:
        self._call("hs_anchor")

    def iter_end_async(self) -> int:
        t = C.c_int(0)
        self._call("hs_iter_end_async", C.byref(t))
        return t.value

    def iter_poll(self, ticket: int):
        """(tokens, done_ms after the anchor) once finished, else None."""
        ms = C.c_double(0)
        rc = self._call("hs_iter_poll", ticket, _ip(self._tok), len(self._tok), C.byref(ms))
        if rc == 0:
            return None
        n = self._call("hs_iter_ntokens", ticket)
        return self._tok[:n].copy(), ms.value

    def mark(self) -> int:
        return self._call("hs_mark")

    def wait_mark(self, mark_id: int) -> None:
        self._call("hs_wait_mark", mark_id)

    def timer(self) -> int:
        return self._call("hs_timer")

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float(0)
        self._call("hs_timer_elapsed", a, b, C.byref(ms))
        return ms.value

    # device-polled merges (include/hs.h, piggyback.cu)
    def pg_enable(self, on: bool = True) -> None:
        self._call("hs_pg_enable", int(on))

    def pg_inject(self, slots, ctxs, lefts) -> None:
        s, c, l_ = _i32(slots), _i32(ctxs), _i32(lefts)
        if len(s):
            self._call("hs_pg_inject", _ip(s), _ip(c), _ip(l_), len(s))

    def pg_stop(self, slots, flags) -> None:
        s, f = _i32(slots), _i32(flags)
        if len(s):
            self._call("hs_pg_stop", _ip(s), _ip(f), len(s))

    def pg_iter(self, cap: int, bounds, inject_bound: int) -> None:
        b = _i32(bounds)
        self._call("hs_pg_iter", cap, _ip(b), inject_bound)

    def pg_share_tags(self, prefix: str, rank: int, world: int, phase: int) -> None:
        self._call("hs_pg_share_tags", prefix.encode(), rank, world, phase)

    def pg_log(self, ticket: int) -> list[list[tuple[int, int]]]:
        """Per layer (1..L): [(slot, flags)] decided by the device."""
        if not hasattr(self, "_pg_buf"):
            self._pg_buf = np.zeros(self.model.n_layers * (1 + 2 * 1024), np.int32)
        n = self._call("hs_pg_log", ticket, _ip(self._pg_buf), len(self._pg_buf))
        out, k = [], 0
        buf = self._pg_buf[:n].tolist()
        for _ in range(self.model.n_layers):
            cnt = buf[k]
            out.append([(buf[k + 1 + 2 * i], buf[k + 2 + 2 * i]) for i in range(cnt)])
            k += 1 + 2 * cnt
        return out

    def keep_logits(self, on: bool = True) -> None:
        self._call("hs_keep_logits", int(on))

    def read_logits(self, rows: int) -> np.ndarray:
        out = np.zeros((rows, self.model.vocab), np.float32)
        self._call("hs_read_logits", out.ctypes.data_as(C.c_void_p), rows)
        return out

    def iter_logits(self, ticket: int, rows: int) -> np.ndarray:
        out = np.zeros((rows, self.model.vocab), np.float32)
        if rows:
            self._call("hs_iter_logits", ticket, out.ctypes.data_as(C.c_void_p), rows)
        return out


def prompt_tokens(req_id: str, length: int, vocab: int, seed: int = 0) -> np.ndarray:
    """Synthetic prompt ids: uniform in [0, vocab) from a per-request seed."""
    rng = np.random.default_rng((zlib.crc32(req_id.encode()) << 8) ^ seed)
    return rng.integers(0, vocab, size=length, dtype=np.int64).astype(np.int32)


SMALL_KV_PAGE_HEADS = 2048  # below this much KV (x 64 tokens x 1 head) a launch is latency-bound
MIN_SMALL_CHUNK = 16        # pages per chunk then (1024 tokens)


def decode_chunks(ctxs: list[int], n_kv: int, target_ctas: int = 296, max_pages: int = 64):
    """Split-K work list for decode attention (K1): each decode row's KV
    pages are cut into near-equal chunks, the chunk size being the smallest
    that keeps chunks x KV heads within one wave of `target_ctas` (2 CTAs
    per SM x 148 SMs), so the launch has no tail wave of short chunks.
    Rows longer than `max_pages` pages always split (bounded merge fan-in).
    A small batch of short rows (at most SMALL_KV_PAGE_HEADS page-heads of
    KV, every row within MIN_SMALL_CHUNK pages) is bound by latency, not HBM:
    its rows are then not split and skip the combine (measured on B200, 8B
    geometry, in-stream: 2 x 700 ctx 11.6 -> 8.7 us, 8 x 700 11.1 -> 9.5 us,
    16 x 700 14.2 -> 11.8 us; longer rows lose when left whole, e.g. 4 x 2000
    13.2 -> 16.5 us at 16-page chunks; tools/probe_decode.py)."""
    pages = [(c + PAGE - 1) // PAGE for c in ctxs]
    total = sum(pages)
    per = max(1, min(max_pages, -(-total * n_kv // target_ctas))) if total else 1
    while per < max_pages and n_kv * sum(-(-n // per) for n in pages) > target_ctas:
        per += 1
    if total and total * n_kv <= SMALL_KV_PAGE_HEADS and max(pages) <= MIN_SMALL_CHUNK:
        per = max(per, max(pages))
    chunks, begin = [], [0]
    for r, (c, n) in enumerate(zip(ctxs, pages)):
        k = max(1, -(-n // per))
        for i in range(k):
            chunks.append((r, -1, i * n // k, (i + 1) * n // k, c))
        begin.append(len(chunks))
    return chunks, begin


class PagePool:
    """Free list of 64-token KV pages; per-slot page lists."""

    def __init__(self, n_pages: int):
        self.free = list(range(n_pages - 1, -1, -1))
        self.owned: dict[int, list[int]] = {}

    def ensure(self, slot: int, tokens: int) -> bool:
        """Grow the slot's pages to hold `tokens`; True if the list changed."""
        have = self.owned.setdefault(slot, [])
        need = (tokens + PAGE - 1) // PAGE
        if need <= len(have):
            return False
        if need - len(have) > len(self.free):
            raise ScenarioError(f"KV page pool exhausted (slot {slot} needs {need} pages)")
        while len(have) < need:
            have.append(self.free.pop())
        return True

    def release(self, slot: int) -> None:
        for p in reversed(self.owned.pop(slot, [])):
            self.free.append(p)


class CudaStep(LayerStep):
    """Executes the engine's schedule on the B200 through libhs."""

    def __init__(self, model: TransformerConfig, rt: Optional[RuntimeConfig] = None,
                 weights: Optional[dict] = None, weight_seed: int = 0, prompt_seed: int = 0,
                 keep_logits: bool = False, ctx=None):
        self.model = model
        self.rt = rt or RuntimeConfig()
        # `ctx` lets the CPU test suite drive the host logic against a
        # recording stand-in (tests/fake_device.py); serving always builds
        # the libhs context
        self.ctx = ctx if ctx is not None else HsContext(model, self.rt)
        if weights is not None:
            self.ctx.load_weights(weights)
        elif ctx is None:  # a caller-built context already holds its weights
            self.ctx.init_weights(weight_seed)
        self.keep = keep_logits
        if keep_logits:
            self.ctx.keep_logits(True)
        self.prompt_seed = prompt_seed
        self.pages = PagePool(self.rt.kv_pages)
        self.slots: dict[str, int] = {}
        self.free_slots = list(range(self.rt.max_slots - 1, -1, -1))
        self.generated: dict[str, list[int]] = {}
        self.prompts: dict[str, np.ndarray] = {}
        self._dirty: set[int] = set()
        self._carry: list[tuple[int, int]] = []
        self._logit_reqs: list[str] = []
        self._merge_L: list[str] = []
        self.last_logits: Optional[np.ndarray] = None
        self.last_token_reqs: list[str] = []
        self.last_tokens: Optional[np.ndarray] = None
        self.iterations = 0
        self._pending_release: list[str] = []
        self._tags: dict[str, int] = {}  # completion tag of each request's outstanding result
        self.remote_slots: dict[int, int] = {}  # slot -> remote CPU host holding its KV
        self.remote_colocated = 0  # offloads to a remote host id with no server connected
        # host<->device bytes moved by the step (metadata, tokens, piggyback rows)
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    # -- bookkeeping --------------------------------------------------------

    def attach(self, engine) -> None:
        self.engine = engine
        if engine.layers != self.model.n_layers:
            raise ScenarioError(
                f"scenario has {engine.layers} layers but transformer {self.model.name} has "
                f"{self.model.n_layers}")

    def slot_of(self, rid: str) -> int:
        s = self.slots.get(rid)
        if s is None:
            if not self.free_slots:
                raise ScenarioError("out of request slots (raise RuntimeConfig.max_slots)")
            s = self.slots[rid] = self.free_slots.pop()
        return s

    def tokens_of(self, req) -> np.ndarray:
        """Prompt ids followed by generated ids (for recompute rebuilds)."""
        need = req.prompt_len + req.rebuild_tokens
        if need > req.prompt_len and len(self.generated.get(req.id, [])) < req.rebuild_tokens:
            self.drain()  # tokens of in-flight iterations are needed now
        p = self.prompts.get(req.id)
        if p is None:
            p = self.prompts[req.id] = prompt_tokens(req.id, req.prompt_len, self.model.vocab,
                                                     self.prompt_seed)
        gen = self.generated.get(req.id, [])
        return np.concatenate([p, np.asarray(gen, np.int32)]) if gen else p

    def _ensure(self, slot: int, tokens: int) -> None:
        if self.pages.ensure(slot, tokens):
            self._dirty.add(slot)

    def _flush_pages(self) -> None:
        for s in sorted(self._dirty):
            self.ctx.set_page_table(s, self.pages.owned.get(s, []))
        self._dirty.clear()

    # -- LayerStep ---------------------------------------------------------------

    def begin_iteration(self, plan) -> None:
        eng = self.engine
        self._release_pending()
        slots, pos, toks = [], [], []
        dec_ctx = []
        logit_rows = []
        self._logit_reqs = []
        for rid in plan.ls_decode + plan.be_decode_gpu:
            r = eng.requests[rid]
            s = self.slot_of(rid)
            self._ensure(s, r.ctx + 1)
            logit_rows.append(len(slots))
            self._logit_reqs.append(rid)
            slots.append(s)
            pos.append(r.ctx)
            toks.append(-1)
            dec_ctx.append(r.ctx + 1)
        n_dec = len(slots)
        tiles = []
        for rid, q in plan.ls_prefill_chunks + plan.be_prefill_chunks:
            r = eng.requests[rid]
            s = self.slot_of(rid)
            done = r.prefill_done
            self._ensure(s, done + q)
            seq = self.tokens_of(r)
            row0 = len(slots)
            for j in range(0, q, 64):
                tiles.append((s, row0 + j, done + j, min(64, q - j)))
            slots += [s] * q
            pos += list(range(done, done + q))
            toks += seq[done:done + q].tolist()
            if done + q >= r.prefill_target and r.rebuild_tokens == 0:
                logit_rows.append(len(slots) - 1)
                self._logit_reqs.append(rid)
        chunks, begin = decode_chunks(dec_ctx, self.model.n_kv)
        chunks = [(row, slots[row], p0, p1, c) for row, _, p0, p1, c in chunks]
        self.h2d_bytes += 4 * (4 * len(slots) + 5 * len(chunks) + len(begin) + 4 * len(tiles)
                               + 2 * len(logit_rows))
        self.h2d_bytes += 4 * sum(len(self.pages.owned.get(s_, [])) for s_ in self._dirty)
        self._flush_pages()
        self.ctx.iter_begin(slots, pos, toks, n_dec, chunks, begin, tiles, logit_rows)
        self._carry = []
        self._merge_L = []

    def layer(self, layer: int, merges) -> None:
        eng = self.engine
        carry = list(self._carry)
        merge_slots, merge_ids, restart_idx, restart_pos, next_carry = [], [], [], [], []
        merge_tags = []
        for item, outcome in merges:
            r = eng.requests[item.req_id]
            s = self.slot_of(item.req_id)
            if outcome == MERGE_INJECT:
                carry.append((s, r.ctx, item.req_id))
                continue
            if outcome == MERGE_CHAIN:
                next_carry.append((s, r.ctx, item.req_id))
            elif outcome == MERGE_TOKEN_NEXT:
                restart_idx.append(len(merge_slots))
                restart_pos.append(r.ctx)
            merge_slots.append(s)
            merge_ids.append(item.req_id)
            merge_tags.append(self._tags.pop(item.req_id))
        # the device checks every merged row's completion tag before use
        self.ctx.layer(layer, [c[0] for c in carry], [c[1] for c in carry], merge_slots,
                       restart_idx, restart_pos, merge_tags)
        shipped = [c[2] for c in carry] + [merge_ids[i] for i in restart_idx]
        m = self.model
        self.h2d_bytes += 4 * (4 * len(carry) + len(merge_slots) + 4 * len(restart_idx))
        self.h2d_bytes += len(merge_slots) * m.result_bytes       # host result rows (PCIe reads)
        self.d2h_bytes += len(shipped) * m.ship_bytes             # q|k|v rows (PCIe writes)
        self._carry = next_carry
        if layer == self.model.n_layers:
            self._merge_L = merge_ids
        return shipped

    def end_iteration(self, plan) -> None:
        toks = self.ctx.iter_end()
        reqs = self._logit_reqs + self._merge_L
        if len(toks) != len(reqs):
            raise RuntimeError(f"libhs returned {len(toks)} tokens for {len(reqs)} rows")
        self.d2h_bytes += 4 * len(toks)
        for rid, t in zip(reqs, toks):
            self.generated.setdefault(rid, []).append(int(t))
        self.last_token_reqs = reqs
        self.last_tokens = toks
        if self.keep and len(reqs):
            self.last_logits = self.ctx.read_logits(len(reqs))
        self.iterations += 1

    def cpu_service(self, host_id: int, items) -> None:
        for it in items:
            self._tags[it.req_id] = result_tag(it.ctx_tokens, it.layer)
        self.ctx.cpu_attend([self.slot_of(it.req_id) for it in items], [it.layer for it in items],
                            [it.ctx_tokens for it in items])

    def swap_out_done(self, req) -> None:
        s = self.slot_of(req.id)
        self.ctx.host_kv_reserve(s, req.prompt_len + req.output_len + 1)
        self.ctx.swap_out(s, req.kv_held)
        self.pages.release(s)
        self._dirty.add(s)
        self._place(req, s, req.kv_held)

    def _place(self, req, slot: int, tokens: int) -> None:
        """The engine offloaded `req` to CPU host `req.swap_dest`
        (_distribute_offload, reference engine.py:402-419): a remote host
        (>= 1) receives the context that just landed in the slot's host
        region and services the request's work items from now on."""
        # the hook runs inside _finish_swap_out before kv_place takes the host
        dest = getattr(req, "swap_dest", None)
        host = dest if isinstance(dest, int) else (
            req.kv_place if isinstance(req.kv_place, int) else 0)
        if host <= 0:
            return
        if host in getattr(self.ctx, "remote_host_ids", ()):
            self.ctx.cpu_place(slot, host, tokens)
            self.remote_slots[slot] = host
        else:  # no server runs for that host: it is co-located with host 0
            self.remote_colocated += 1

    def _unplace(self, slot: int, tokens: int) -> None:
        """Swap-in from a remote host: its KV comes back into the slot's
        host region first."""
        if self.remote_slots.pop(slot, 0):
            self.ctx.cpu_place(slot, 0, tokens)

    def resumed_on_gpu(self, req) -> None:
        s = self.slot_of(req.id)
        self._ensure(s, req.ctx)
        self._flush_pages()
        self._unplace(s, req.ctx)
        self.ctx.swap_in(s, req.ctx)
        self.ctx.host_kv_release(s)

    def preempted(self, req) -> None:
        s = self.slot_of(req.id)
        self.pages.release(s)
        self._dirty.add(s)

    def released(self, req) -> None:
        # a chain can complete inside _run_layer(L) before this layer's rows
        # (which still read the slot's residual) are launched: free the slot
        # once the iteration is over
        self._pending_release.append(req.id)

    def _release_pending(self) -> None:
        for rid in self._pending_release:
            self._tags.pop(rid, None)
            s = self.slots.pop(rid, None)
            if s is None:
                continue
            self.pages.release(s)
            self.remote_slots.pop(s, None)
            self.ctx.host_kv_release(s)
            self._dirty.discard(s)
            self.free_slots.append(s)
        self._pending_release.clear()

    def drain(self) -> None:
        """Synchronous steps have no iterations in flight."""

    def finish(self) -> None:
        self.ctx.sync()
        self._release_pending()


class LiveCudaStep(CudaStep):
    """CudaStep for LiveEngine: asynchronous CPU service and swaps, launch
    pacing and per-iteration device timing (CUDA events).

    device_merges=True: the piggyback merge decisions are taken by the GPU
    (hs_pg_*, include/hs.h): layers are launched without row lists, shipped
    work items reach the CPU pool through the device's work ring, and each
    finished iteration hands its decision log to the engine (payload
    "pg_log": per layer [(request id, flags)])."""

    def __init__(self, *args, device_merges: bool = False, **kw):
        super().__init__(*args, **kw)
        self.device_merges = device_merges
        if device_merges:
            self.ctx.pg_enable(True)
        self._marks: list[int] = []
        self.last_device_ms = 0.0
        self.swap_out_tickets: dict[int, str] = {}
        # swap-ins from remote hosts: ticket -> (slot, tokens, DMA ticket once fetched)
        self._fetches: dict[int, tuple] = {}
        self._fetch_seq = 0
        self._inflight: list[tuple[int, list[str], object]] = []  # (ticket, reqs, payload)
        # iterations finished by a blocking drain() (a recompute rebuild
        # needing their tokens) that the engine has not resolved yet: handed
        # out first by the next poll_iterations()
        self._drained: list = []
        self.anchor_wall = 0.0
        # per finished iteration, in order: (request ids, greedy tokens, logits
        # or None) -- the realised token stream, kept when trace_tokens is set
        self.trace_tokens = False
        self.token_log: list[tuple[list[str], np.ndarray, Optional[np.ndarray]]] = []

    def set_anchor(self, wall: float) -> None:
        """Device events are reported relative to this host time."""
        self.ctx.anchor()
        self.anchor_wall = wall

    def pg_begin(self, cap: int, bounds, inject_bound: int, injections=(), stops=()) -> None:
        """Device-polled merges, per iteration after begin_iteration: new
        chains [(request id, ctx, tokens left)], stop-flag changes [(request
        id, flag)], this iteration's cap and the launch bounds."""
        if injections:
            self.ctx.pg_inject([self.slot_of(r) for r, _, _ in injections],
                               [c for _, c, _ in injections], [n for _, _, n in injections])
        if stops:
            self.ctx.pg_stop([self.slot_of(r) for r, _ in stops], [int(f) for _, f in stops])
        self.h2d_bytes += 16 * (len(injections) + len(stops)) + 4 * len(bounds)
        self.ctx.pg_iter(cap, bounds, inject_bound)

    def layer(self, layer: int, merges):
        if self.device_merges:
            self.ctx.layer(layer, [], [], [], [], [])
            shipped = []
        else:
            shipped = super().layer(layer, merges)
        self._marks.append(self.ctx.mark())
        if len(self._marks) > 64:
            del self._marks[:-16]
        return shipped

    def pace(self, lag: int) -> None:
        """Block until at most `lag` launched layers are still queued."""
        if len(self._marks) > lag:
            self.ctx.wait_mark(self._marks[-lag - 1])

    def end_iteration(self, plan, payload=None) -> None:
        """Queue the token readback; the iteration completes asynchronously."""
        ticket = self.ctx.iter_end_async()
        flush = getattr(self.ctx, "flush", None)
        if flush is not None:  # TP group leader: ship this iteration's calls to the followers
            flush()
        reqs = list(self._logit_reqs) if self.device_merges else self._logit_reqs + self._merge_L
        self._inflight.append((ticket, reqs, payload))
        self.iterations += 1

    def reset(self, timeout_s: float = 60.0) -> None:
        """Quiesce the replica (in-flight iterations, CPU items, swaps) and
        release every request slot, so a new engine can be attached to the
        same context (weights and arenas are kept)."""
        import time

        self._poll(block=True)
        self._drained = []
        t0 = time.perf_counter()
        while self.ctx.lib.hs_cpu_in_flight(self.ctx.h) > 0:
            if time.perf_counter() - t0 > timeout_s:
                raise RuntimeError("reset: CPU-attention items still in flight")
            time.sleep(1e-3)
        self.ctx.cpu_poll()
        self.ctx.sync()
        if getattr(self, "device_merges", False):
            self.ctx.pg_enable(True)  # drop the device's queued items
        for s in list(self.slots.values()):
            self.pages.release(s)
            self.ctx.host_kv_release(s)
            self._dirty.add(s)
        self._flush_pages()
        self.slots.clear()
        self.remote_slots.clear()
        self._fetches.clear()
        self.free_slots = list(range(self.rt.max_slots - 1, -1, -1))
        for d in (self.generated, self.prompts, self._tags):
            d.clear()
        self._pending_release.clear()
        self._carry, self._merge_L, self._logit_reqs = [], [], []
        self.token_log.clear()

    def iterations_in_flight(self) -> int:
        return len(self._inflight) + len(self._drained)

    def drain(self) -> None:
        """Finish every in-flight iteration (their tokens are recorded); the
        records stay queued for the engine's next poll_iterations()."""
        self._drained += self._poll(block=True)

    def poll_iterations(self, block: bool = False):
        """Finished iterations in order: [(payload, t_done_wall, tokens)]."""
        out, self._drained = self._drained, []
        return out + self._poll(block)

    def _poll(self, block: bool):
        out = []
        while self._inflight:
            ticket, reqs, payload = self._inflight[0]
            res = self.ctx.iter_poll(ticket)
            if res is None:
                if not block:
                    break
                self.ctx.wait_mark(self._marks[-1]) if self._marks else self.ctx.sync()
                continue
            toks, ms = res
            self._inflight.pop(0)
            if self.device_merges:
                # the device's decisions; the chains merged at the last layer
                # own the token rows after the plan's logit rows (the rest of
                # the launch bound is padding)
                by_slot = {s: rid for rid, s in self.slots.items()}
                log = [[(by_slot[s], f) for s, f in recs] for recs in self.ctx.pg_log(ticket)]
                reqs = list(reqs) + [rid for rid, _ in log[-1]]
                if len(toks) < len(reqs):
                    raise RuntimeError(f"libhs returned {len(toks)} tokens for {len(reqs)} rows")
                toks = toks[:len(reqs)]
                if payload is not None:
                    payload["pg_log"] = log
                # piggyback traffic the device moved: every merged result row
                # (H2D), every shipped q|k|v row (D2H): chains carried into the
                # next layer, injections, restarts
                m = self.model
                n_res = sum(1 for recs in log for _, f in recs if not f & 1)
                n_ship = (sum(1 for recs in log[:-1] for _, f in recs if not f & 1)
                          + sum(1 for recs in log for _, f in recs if f & 3))
                self.h2d_bytes += n_res * m.result_bytes
                self.d2h_bytes += n_ship * m.ship_bytes
            elif len(toks) != len(reqs):
                raise RuntimeError(f"libhs returned {len(toks)} tokens for {len(reqs)} rows")
            if self.trace_tokens:
                lg = self.ctx.iter_logits(ticket, len(toks)) if self.keep else None
                self.token_log.append((list(reqs), toks.copy(), lg))
            self.d2h_bytes += 4 * len(toks)
            for rid, t in zip(reqs, toks):
                self.generated.setdefault(rid, []).append(int(t))
            out.append((payload, self.anchor_wall + ms / 1e3, toks))
        return out

    def cpu_submit(self, items) -> None:
        for it in items:
            self._tags[it.req_id] = result_tag(it.ctx_tokens, it.layer)
        self.ctx.cpu_submit([self.slot_of(it.req_id) for it in items],
                            [it.layer for it in items], [it.ctx_tokens for it in items])

    def cpu_poll(self):
        slots, layers = self.ctx.cpu_poll()
        if not len(slots):
            return []
        by_slot = {s: rid for rid, s in self.slots.items()}
        return [(by_slot[int(s)], int(l)) for s, l in zip(slots, layers)]

    def swap_out_async(self, req) -> int:
        s = self.slot_of(req.id)
        self.ctx.host_kv_reserve(s, req.prompt_len + req.output_len + 1)
        return self.ctx.swap_async(s, req.kv_held, out=True)

    def swap_in_async(self, req) -> int:
        s = self.slot_of(req.id)
        self._ensure(s, req.ctx)
        self._flush_pages()
        if self.remote_slots.pop(s, 0):
            # from a remote host: the KV comes back over the network first
            # (without blocking the engine), then the DMA is issued by
            # swap_done; fetch tickets are negative
            self.ctx.cpu_fetch_async(s, req.ctx)
            self._fetch_seq -= 1
            self._fetches[self._fetch_seq] = (s, req.ctx, None)
            return self._fetch_seq
        return self.ctx.swap_async(s, req.ctx, out=False)

    def swap_done(self, ticket: int) -> bool:
        if ticket in self._fetches:
            s, n, dma = self._fetches[ticket]
            if dma is None:
                if not self.ctx.cpu_fetch_done(s):
                    return False
                self._fetches[ticket] = (s, n, self.ctx.swap_async(s, n, out=False))
                return False
            if self.ctx.swap_done(dma):
                del self._fetches[ticket]
                return True
            return False
        return self.ctx.swap_done(ticket)

    def swap_out_done(self, req) -> None:
        s = self.slot_of(req.id)
        self.pages.release(s)
        self._dirty.add(s)
        self._place(req, s, req.kv_held)

    def resumed_on_gpu(self, req) -> None:
        s = self.slot_of(req.id)
        self.remote_slots.pop(s, None)
        self.ctx.host_kv_release(s)

    def cpu_service(self, host_id: int, items) -> None:
        raise AssertionError("live mode submits work items asynchronously")
