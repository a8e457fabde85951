"""Profiler on real kernels: fit the scheduler's latency models to the B200.

The reference fits its models against synthetic profiles
(pkg/src/hybridserve/latency.py:355-398).  Here the same three families are
fitted to device timings of the libhs kernels of one layer:

* dense: Alg. 1 (`build_dense_table`, latency.py:200-259) with a probe that
  times the real Dense modules (QKV, O, gate-up, down GEMMs + epilogues);
  measured latencies are made monotone (running max) before tabulation so
  timing noise cannot create spurious ladder steps;
* decode attention: least squares of Eq. 3 over (context tokens, requests);
* prefill attention: least squares of Eq. 2 over pairwise units.

The result is a LatencyModelSet (serialised with model_set_to_dict, the
reference's models.json schema) that LiveEngine budgets against.
"""

from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np

from .latency import (
    LatencyModelSet,
    build_dense_table,
    comm_models_for,
    fit_decode_attn,
    fit_prefill_attn,
    model_set_from_dict,
    model_set_to_dict,
)
from .profiles import DeviceClass
from .scheduling import pairwise_units


def _probe(ctx, name: str, *args, reps: int = 5) -> float:
    lib = ctx.lib
    fn = getattr(lib, name)
    fn.argtypes = [C.c_void_p] + [C.c_int] * (len(args) + 1) + [C.POINTER(C.c_float)]
    fn.restype = C.c_int
    us = C.c_float(0)
    rc = fn(ctx.h, *args, reps, C.byref(us))
    if rc:
        from . import _lib

        _lib.check(rc, name)
    return float(us.value)


def calibrate(ctx, cluster, max_batch: int = 8192, max_ctx: int = 16384,
              dense_threshold_us: float | None = None, seed: int = 0,
              log=None) -> LatencyModelSet:
    """Probe the context's kernels and fit the model set.  Clobbers page
    tables: run before serving."""
    max_batch = min(max_batch, ctx.rt.max_rows)
    memo: dict[int, float] = {}

    def dense(n: int) -> float:
        if n not in memo:
            memo[n] = _probe(ctx, "hs_probe_dense", n)
        return memo[n]

    # monotone envelope of the measured curve
    def dense_mono(n: int) -> float:
        best = dense(n)
        for m_ in memo:
            if m_ < n:
                best = max(best, memo[m_])
        return best

    if dense_threshold_us is None:
        dense_threshold_us = max(2.0, 0.05 * dense(1))
    table, diag = build_dense_table(dense_mono, 1, max_batch, threshold=dense_threshold_us)
    if log:
        log(f"dense: {diag.probe_calls} probes, {diag.n_segments} segments, "
            f"d(1)={dense(1):.1f}us d({max_batch})={dense(max_batch):.1f}us")

    rng = np.random.default_rng(seed)
    da = []
    for _ in range(24):
        g = int(rng.integers(1, 65))
        c = int(rng.integers(64, max_ctx // 2))
        c = min(c, (ctx.rt.max_pages_per_req * 64) - 1, (ctx.rt.kv_pages * 64) // g - 1)
        if c < 2:
            continue
        da.append((float(g * c), g, _probe(ctx, "hs_probe_decode", g, c)))
    da_model, _ = fit_decode_attn(da)
    pa = []
    for _ in range(16):
        q = int(rng.integers(16, min(4096, ctx.rt.max_rows)))
        done = int(rng.integers(0, max_ctx // 2))
        done = min(done, ctx.rt.max_pages_per_req * 64 - q - 1)
        pa.append((pairwise_units(done, q), _probe(ctx, "hs_probe_prefill", q, done)))
    pa_model, _ = fit_prefill_attn(pa)
    if pa_model.per_unit < 0:
        pa_model = type(pa_model)(0.0, pa_model.base)
    if log:
        log(f"decode attn: {da_model}; prefill attn: {pa_model}")
    return LatencyModelSet(DeviceClass.GPU, pa_model, da_model, table, comm_models_for(cluster))


def save(models: LatencyModelSet, path: Path, meta: dict | None = None) -> None:
    doc = {"sets": {"GPU": model_set_to_dict(models)}, "meta": meta or {}}
    path.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")


def load(path: Path) -> LatencyModelSet:
    return model_set_from_dict(json.loads(Path(path).read_text())["sets"]["GPU"])
