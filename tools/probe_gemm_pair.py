"""K3 at prefill-sized batches: the 1-SM stream-K kernel (hs_op_gemm_bf16)
against the CTA-pair kernel (hs_op_gemm_bf16_pair) on the Llama-3-8B layer
shapes, one launch between events with L2 flushed (median of 10), plus the
bf16 tensor fraction against MEASURED_PEAKS.json.

    python tools/probe_gemm_pair.py [tokens ...]
"""
import ctypes as C
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200 import _lib  # noqa: E402

_lib.load()
ROOT = Path(__file__).resolve().parent.parent
peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
PEAK = peaks.get("bf16_tflops", 1590.0)
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
p = lambda a: C.c_void_p(a.data_ptr())  # noqa: E731
SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}


def timed(fn, reps=10):
    ts = []
    for _ in range(reps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts = sorted(ts[2:])
    return ts[len(ts) // 2]


for t in [int(a) for a in sys.argv[1:]] or [256, 512, 1024]:
    for name, (n, k) in SHAPES.items():
        w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
        x = torch.randn(t, k, device=dev).to(torch.bfloat16)
        part = torch.empty(16 * t * n, dtype=torch.float32, device=dev)
        used = C.c_int(0)
        row = {"tokens": t, "gemm": name}
        for op in ("hs_op_gemm_bf16", "hs_op_gemm_bf16_pair"):
            us = timed(lambda: _lib.call(op, p(x), t, k, p(w), n, k, p(part), 16, C.byref(used), None))
            tf = 2.0 * t * n * k / (us * 1e-6) / 1e12
            key = "pair" if op.endswith("pair") else "one_sm"
            row[key + "_us"] = round(us, 2)
            row[key + "_frac"] = round(tf / PEAK, 3)
            row[key + "_planes"] = used.value
        print(json.dumps(row), flush=True)
        del w, x, part
