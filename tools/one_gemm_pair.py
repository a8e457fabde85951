"""Launch one GEMM shape with the 1-SM or the CTA-pair kernel a few times
(for ncu captures): python tools/one_gemm_pair.py n k tokens [pair|one]"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200 import _lib  # noqa: E402

n, k, t = (int(x) for x in sys.argv[1:4])
op = "hs_op_gemm_bf16_pair" if (sys.argv[4] if len(sys.argv) > 4 else "pair") == "pair" else "hs_op_gemm_bf16"
dev = torch.device("cuda")
w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
x = torch.randn(t, k, device=dev).to(torch.bfloat16)
part = torch.empty(16 * t * n, dtype=torch.float32, device=dev)
used = C.c_int(0)
p = lambda a: C.c_void_p(a.data_ptr())  # noqa: E731
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(4):
    flush.zero_()
    _lib.call(op, p(x), t, k, p(w), n, k, p(part), 16, C.byref(used), None)
torch.cuda.synchronize()
print("planes", used.value)
