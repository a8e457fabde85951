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
    DecodeAttnModel,
    LatencyModelSet,
    PrefillAttnModel,
    build_dense_table,
    comm_models_for,
    fit_decode_attn,
    fit_prefill_attn,
    model_set_from_dict,
    model_set_to_dict,
    predict_decode_attn,
    predict_dense,
    predict_prefill_attn,
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
    da = decode_samples(ctx, rng, 32, max_ctx)
    da_model = fit_decode_attn_nonneg(da)
    pa = prefill_samples(ctx, rng, 32, max_ctx)
    pa_model = fit_prefill_attn_nonneg(pa)
    if log:
        log(f"decode attn: {da_model}; prefill attn: {pa_model}")
    return LatencyModelSet(DeviceClass.GPU, pa_model, da_model, table, comm_models_for(cluster))


def decode_samples(ctx, rng, n: int, max_ctx: int) -> list[tuple[float, int, float]]:
    """(context tokens, requests, us) of the decode-attention kernel at
    random batch shapes (Eq. 3's regressors)."""
    out = []
    for _ in range(n):
        g = int(rng.integers(1, 65))
        c = int(rng.integers(64, max_ctx // 2))
        c = min(c, (ctx.rt.max_pages_per_req * 64) - 1, (ctx.rt.kv_pages * 64) // g - 1)
        if c < 2:
            continue
        out.append((float(g * c), g, _probe(ctx, "hs_probe_decode", g, c)))
    return out


def prefill_samples(ctx, rng, n: int, max_ctx: int) -> list[tuple[float, float]]:
    """(pairwise units, us) of the chunked-prefill kernel (Eq. 2)."""
    out = []
    for _ in range(n):
        q = int(rng.integers(16, min(4096, ctx.rt.max_rows)))
        done = int(rng.integers(0, max_ctx // 2))
        done = min(done, ctx.rt.max_pages_per_req * 64 - q - 1)
        out.append((pairwise_units(done, q), _probe(ctx, "hs_probe_prefill", q, done)))
    return out


def nnls(design: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Least squares with non-negative coefficients, exact for the 2-3
    regressors of Eq. 2/3: the best unconstrained solution over every
    support subset whose coefficients are all >= 0.  A latency model must not
    credit a request or a token with negative time (the reference's plain
    lstsq, latency.py:162-186, can: on B200 the fitted per-request decode
    term came out at -0.035 us)."""
    k = design.shape[1]
    best, best_err = np.zeros(k), float(np.sum(y * y))
    for mask in range(1, 1 << k):
        cols = [j for j in range(k) if mask >> j & 1]
        coef, *_ = np.linalg.lstsq(design[:, cols], y, rcond=None)
        if np.any(coef < 0):
            continue
        err = float(np.sum((design[:, cols] @ coef - y) ** 2))
        if err < best_err:
            best = np.zeros(k)
            best[cols] = coef
            best_err = err
    return best


def _rel_nnls(design: np.ndarray, y: np.ndarray) -> np.ndarray:
    """NNLS on relative residuals (rows scaled by 1/y): the scheduler's
    budget test is relative to the SLO, and short kernels dominate the
    sample count, so a fit in absolute microseconds would trade their
    accuracy for the long ones'."""
    w = 1.0 / np.maximum(y, 1e-6)
    return nnls(design * w[:, None], y * w)


def fit_decode_attn_nonneg(samples) -> DecodeAttnModel:
    fit_decode_attn(samples)  # the reference's degeneracy checks
    a = np.asarray(samples, dtype=float)
    c = _rel_nnls(np.column_stack([a[:, 0], a[:, 1], np.ones(len(a))]), a[:, 2])
    return DecodeAttnModel(float(c[0]), float(c[1]), float(c[2]))


def _rel_l1_line(x: np.ndarray, y: np.ndarray) -> tuple[float, float]:
    """y ~ a*x + b (a, b >= 0) minimising the mean relative error
    |a*x + b - y| / y -- the accuracy the paper reports.
    An L1 optimum of a two-parameter line passes through two samples (or
    one, with a or b at its bound), so the candidates are enumerated."""
    cands = [(0.0, float(np.median(y)))]
    for i in range(len(x)):
        if x[i] > 0:
            cands.append((float(y[i] / x[i]), 0.0))
        cands.append((0.0, float(y[i])))
        for j in range(i + 1, len(x)):
            if x[j] != x[i]:
                a = (y[j] - y[i]) / (x[j] - x[i])
                b = y[i] - a * x[i]
                if a >= 0 and b >= 0:
                    cands.append((float(a), float(b)))
    err = [float(np.mean(np.abs(a * x + b - y) / y)) for a, b in cands]
    return cands[int(np.argmin(err))]


def fit_prefill_attn_nonneg(samples) -> PrefillAttnModel:
    """Eq. 2 (linear in pairwise units) fitted for the mean relative error:
    the kernel's time steps with its tile waves at short chunks, which a
    least-squares line (even on relative residuals) pays for with the many
    short samples."""
    fit_prefill_attn(samples)
    a = np.asarray(samples, dtype=float)
    keep = a[:, 1] > 0
    per_unit, base = _rel_l1_line(a[keep, 0], a[keep, 1])
    return PrefillAttnModel(per_unit, base)


def accuracy(ctx, models: LatencyModelSet, seed: int = 1, n: int = 12,
             max_ctx: int = 16384, max_batch: int = 4096) -> dict:
    """Held-out accuracy of the fitted models against fresh kernel timings,
    in the paper's form: mean and 90th-percentile
    accuracy, 1 - |predicted - measured| / measured, per model family."""
    rng = np.random.default_rng(seed)
    fam = {}
    dn = [int(x) for x in rng.integers(1, min(max_batch, ctx.rt.max_rows), n)]
    fam["dense"] = [(predict_dense(models.dense, x), _probe(ctx, "hs_probe_dense", x)) for x in dn]
    fam["decode_attn"] = [(predict_decode_attn(models.decode_attn, c, g), us)
                          for c, g, us in decode_samples(ctx, rng, n, max_ctx)]
    fam["prefill_attn"] = [(predict_prefill_attn(models.prefill_attn, u), us)
                           for u, us in prefill_samples(ctx, rng, n, max_ctx)]
    out = {}
    for k, pairs in fam.items():
        acc = np.array([1.0 - abs(p - m) / m for p, m in pairs if m > 0])
        out[k] = {"mean": float(acc.mean()), "p90": float(np.percentile(acc, 10)),
                  "samples": len(acc)}
    return out


def save(models: LatencyModelSet, path: Path, meta: dict | None = None) -> None:
    doc = {"sets": {"GPU": model_set_to_dict(models)}, "meta": meta or {}}
    path.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")


def load(path: Path) -> LatencyModelSet:
    return model_set_from_dict(json.loads(Path(path).read_text())["sets"]["GPU"])
