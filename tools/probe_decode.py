"""Decode attention (K1 with the fused K2 combine) on Llama-3-8B geometry at
serving-like batches, chunked exactly as the runtime does
(runtime.decode_chunks).  Two timings: one launch between events (L2
flushed), and 32 back-to-back launches (one per layer, different layers of
the pool) like the step issues them.  Algorithmic bytes = sum(ctx) * 4 KiB."""
import ctypes as C
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200 import _lib  # noqa: E402
from paper_2603_12831_b200 import runtime  # noqa: E402
from paper_2603_12831_b200.runtime import decode_chunks  # noqa: E402

if os.environ.get("HS_NO_SMALL"):  # compare against chunking without the small-batch rule
    runtime.SMALL_KV_PAGE_HEADS = 0

_lib.load()
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
HBM = 6555.5


def p(t):
    return C.c_void_p(t.data_ptr())


def ev_time(fn, reps=10):
    ts = []
    for i in range(reps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


n_q, n_kv, hd, layers = 32, 8, 128, 32
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
cases = [(8, 700), (16, 700), (24, 700), (32, 700), (16, 2000), (8, 9000), (64, 2048),
         (128, 2048)]
TARGET = int(sys.argv[1]) if len(sys.argv) > 1 else 296  # decode_chunks target CTAs
if len(sys.argv) > 2:
    cases = [tuple(int(v) for v in c.split("x")) for c in sys.argv[2:]]
for g, ctx in cases:
    npg = (ctx + 63) // 64
    pages = g * npg
    pool = torch.empty(layers * pages * 2 * n_kv * 64 * hd, dtype=torch.bfloat16, device=dev)
    pool.normal_()
    pt = torch.arange(pages, dtype=torch.int32, device=dev).reshape(g, npg)
    q = torch.randn(g, n_q * hd, device=dev).to(torch.bfloat16)
    chunks, begin = decode_chunks([ctx] * g, n_kv, target_ctas=TARGET)
    ch = torch.tensor([[r, r, a, b, c] for r, _, a, b, c in chunks], dtype=torch.int32,
                      device=dev)
    beg = torch.tensor(begin, dtype=torch.int32, device=dev)
    op = torch.empty(len(chunks) * n_q * hd, device=dev)
    lp = torch.empty(len(chunks) * n_q, device=dev)
    cnt = torch.zeros(g * n_kv, dtype=torch.int32, device=dev)
    out = torch.empty(g, n_q * hd, dtype=torch.bfloat16, device=dev)

    def one(layer=0):
        _lib.call("hs_op_decode_attention_fused", p(pool), layers, pages, n_kv, hd, layer, p(q),
                  n_q * hd, n_q, p(pt), npg, p(ch), len(chunks), g, p(beg), p(op), p(lp), p(cnt),
                  p(out), n_q * hd, st)

    def stream32():
        for l_ in range(layers):
            one(l_)

    us1 = ev_time(one)
    us32 = ev_time(stream32, reps=5) / layers
    by = g * ctx * 2 * n_kv * hd * 2
    print(json.dumps({"target": TARGET, "g": g, "ctx": ctx, "ctas": len(chunks) * n_kv,
                      "pages_per_chunk": max(b - a for _, _, a, b, _ in chunks),
                      "us_single": round(us1, 2), "us_in_stream": round(us32, 2),
                      "frac_single": round(by / us1 / 1e3 / HBM, 3),
                      "frac_in_stream": round(by / us32 / 1e3 / HBM, 3)}), flush=True)
    del pool
