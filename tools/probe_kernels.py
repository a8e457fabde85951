"""Micro-timing of the libhs kernels on Llama-3-8B shapes (CUDA events on the
launching stream, L2 flushed between reps).  Prints one JSON line per case.

    python tools/probe_kernels.py [--quick]
"""

from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200 import _lib  # noqa: E402

PEAKS = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()) \
    if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else \
    {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def p(t):
    return C.c_void_p(t.data_ptr())


def timed(fn, reps=20, flush=None):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


def main():
    quick = "--quick" in sys.argv
    dev = torch.device("cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    shapes = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096),
              "down": (4096, 14336)}
    toks = [1, 16, 64, 256] if quick else [1, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]
    for name, (n, k) in shapes.items():
        w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
        wb = torch.empty_like(w)
        _lib.call("hs_op_relayout_blocked", p(w), p(wb), n, k, stream)
        for t in toks:
            x = torch.randn(t, k, device=dev).to(torch.bfloat16)
            part = torch.empty(16 * t * n, dtype=torch.float32, device=dev)
            used = C.c_int(0)

            def run():
                _lib.call("hs_op_gemm_bf16", p(x), t, k, p(w), n, k, p(part), 16, C.byref(used),
                          stream)

            sec = timed(run, flush=flush)

            def run_b():
                _lib.call("hs_op_gemm_bf16_blocked", p(x), t, k, p(wb), n, k, p(part), 16,
                          C.byref(used), stream)

            sec_b = timed(run_b, flush=flush)
            flops = 2.0 * t * n * k
            bytes_ = 2.0 * n * k + 2.0 * t * k + 4.0 * used.value * t * n
            print(json.dumps({"kernel": "gemm", "shape": name, "tokens": t, "splits": used.value,
                              "us": sec * 1e6, "us_blocked": sec_b * 1e6,
                              "gbs_blocked": (2.0 * n * k + 2.0 * t * k) / sec_b / 1e9,
                              "tflops": flops / sec / 1e12,
                              "gbs": bytes_ / sec / 1e9,
                              "hbm_frac": bytes_ / sec / 1e9 / PEAKS["hbm_gbs"],
                              "tensor_frac": flops / sec / 1e12 / PEAKS["bf16_tflops"]}),
                  flush=True)
    # decode attention: 8B geometry, batch of g requests at ctx c
    n_q, n_kv, hd, layers = 32, 8, 128, 1
    for g, ctx in ([(16, 1024), (64, 2048)] if quick else
                   [(1, 1024), (16, 512), (16, 2048), (64, 1024), (64, 4096), (128, 2048)]):
        npg = (ctx + 63) // 64
        pages = g * npg
        pool = torch.randn(layers * pages * 2 * n_kv * 64 * hd, device=dev).to(torch.bfloat16)
        pt = torch.arange(pages, dtype=torch.int32, device=dev).reshape(g, npg)
        q = torch.randn(g, n_q * hd, device=dev).to(torch.bfloat16)
        chunk = max(1, -(-g * npg * n_kv // 296))
        ch, beg = [], [0]
        for r in range(g):
            for p0 in range(0, npg, chunk):
                ch.append((r, r, p0, min(npg, p0 + chunk), ctx))
            beg.append(len(ch))
        dch = torch.tensor(ch, dtype=torch.int32, device=dev)
        dbeg = torch.tensor(beg, dtype=torch.int32, device=dev)
        op = torch.empty(len(ch) * n_q * hd, device=dev)
        lp = torch.empty(len(ch) * n_q, device=dev)
        out = torch.empty(g, n_q * hd, dtype=torch.bfloat16, device=dev)

        def run_dec():
            _lib.call("hs_op_decode_attention", p(pool), layers, pages, n_kv, hd, 0, p(q),
                      n_q * hd, n_q, p(pt), npg, p(dch), len(ch), p(op), p(lp), stream)
            _lib.call("hs_op_decode_combine", p(op), p(lp), p(dbeg), g, n_q, n_kv, hd, p(out),
                      n_q * hd, C.c_void_p(0), stream)

        sec = timed(run_dec, flush=flush)
        bytes_ = g * ctx * 2 * n_kv * hd * 2
        print(json.dumps({"kernel": "decode_attn", "g": g, "ctx": ctx, "chunks": len(ch),
                          "us": sec * 1e6, "gbs": bytes_ / sec / 1e9,
                          "hbm_frac": bytes_ / sec / 1e9 / PEAKS["hbm_gbs"]}), flush=True)


if __name__ == "__main__":
    main()
