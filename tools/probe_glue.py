"""Isolated glue-kernel bandwidth (C-ABI ops on torch buffers, CUDA events,
L2 flushed): SiLU*up and residual-add-norm over split-K planes vs a torch
copy of the same bytes."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200 import _lib  # noqa: E402

_lib.load()
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def p(t):
    return C.c_void_p(t.data_ptr())


def timed(fn, reps=10):
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
    ts.sort()
    return ts[len(ts) // 2]


ffn, d = 14336, 4096
for rows in (16, 64, 256, 512):
    for splits in (1, 2, 3):
        part = torch.randn(splits * rows * 2 * ffn, device=dev)
        act = torch.empty(rows, ffn, dtype=torch.bfloat16, device=dev)
        us = timed(lambda: _lib.call("hs_op_silu_mul", p(part), splits, rows, ffn, p(act), ffn,
                                     None))
        by = part.numel() * 4 + act.numel() * 2
        dst = torch.empty_like(part)
        us_cp = timed(lambda: dst.copy_(part))
        print(f"silu rows {rows:4d} splits {splits}: {us:7.1f} us {by / us / 1e3:7.0f} GB/s | "
              f"torch copy of the planes {us_cp:7.1f} us "
              f"{2 * part.numel() * 4 / us_cp / 1e3:7.0f} GB/s", flush=True)
        del part, dst
for rows in (16, 64, 512):
    splits = 4
    part = torch.randn(splits * rows * d, device=dev)
    h = torch.randn(rows * d, device=dev)
    w = torch.ones(d, device=dev)
    out = torch.empty(rows, d, dtype=torch.bfloat16, device=dev)
    us = timed(lambda: _lib.call("hs_op_residual_add_norm", p(part), splits, rows, d, p(h), p(w),
                                 C.c_float(1e-5), p(out), d, None))
    by = part.numel() * 4 + 2 * h.numel() * 4 + out.numel() * 2
    print(f"addnorm rows {rows:4d} splits {splits}: {us:7.1f} us {by / us / 1e3:7.0f} GB/s",
          flush=True)
