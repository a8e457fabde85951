"""One GEMM of Llama-3-8B layer 0 between events: planes path vs the fused
cluster-split path (hs_probe_gemm), per projection and batch size."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200.models import get_transformer  # noqa: E402
from paper_2603_12831_b200.runtime import HsContext, RuntimeConfig  # noqa: E402

ctx = HsContext(get_transformer("llama3-8b"),
                RuntimeConfig(max_rows=512, max_slots=8, kv_pages=64, max_pages_per_req=8,
                              max_pos=128, max_chunks=64, cpu_threads=1, host_kv_bytes=0))
ctx.init_weights(0)
fn = ctx.lib.hs_probe_gemm
fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]
MB = {0: 50.3, 1: 33.6, 2: 234.9, 3: 117.4}
for n in [int(a) for a in sys.argv[1:]] or (8, 32):
    for w, name in enumerate(("qkv", "o", "gate_up", "down")):
        out = []
        for fused in (0, 1):
            us = C.c_float()
            rc = fn(ctx.h, w, n, fused, 9, C.byref(us))
            out.append(f"{us.value:7.1f}" if rc == 0 else "  n/a  ")
        print(f"n={n:3d} {name:8s} planes {out[0]} us  fused {out[1]} us  "
              f"(HBM floor {MB[w] / 6.55:.1f} us)", flush=True)
