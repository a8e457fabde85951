"""Plain vs fused-epilogue GEMMs of one Llama-3-8B layer (device us)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200.models import get_transformer  # noqa: E402
from paper_2603_12831_b200.runtime import HsContext, RuntimeConfig  # noqa: E402

ctx = HsContext(get_transformer("llama3-8b"), RuntimeConfig(max_rows=512, max_slots=8, kv_pages=64,
                                                            max_pages_per_req=8, max_pos=64,
                                                            max_chunks=64, cpu_threads=1,
                                                            host_kv_bytes=0))
ctx.init_weights(0)
fn = ctx.lib.hs_probe_gemm
fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]
for which, name in enumerate(["qkv", "o", "gate_up", "down"]):
    for n in (1, 16, 32, 64, 128):
        r = []
        for fused in (0, 1):
            us = C.c_float()
            assert fn(ctx.h, which, n, fused, 20, C.byref(us)) == 0
            r.append(us.value)
        print(f"{name:8s} n={n:4d} plain {r[0]:7.1f} us   fused {r[1]:7.1f} us")
