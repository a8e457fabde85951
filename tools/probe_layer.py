"""Per-layer device time of the dense part of Llama-3-8B as hs_layer issues
it, 32 layers back to back (weights streamed from HBM, no events between
launches): each op alone, the GEMMs, the glue kernels, all of it.  The
GEMM-only time against the 66.5 us roofline (436 MB / 6555 GB/s) is the
in-stream streaming efficiency."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200.models import get_transformer  # noqa: E402
from paper_2603_12831_b200.runtime import HsContext, RuntimeConfig  # noqa: E402

ctx = HsContext(get_transformer("llama3-8b"), RuntimeConfig(max_rows=1024, max_slots=8, kv_pages=64,
                                                            max_pages_per_req=8, max_pos=128,
                                                            max_chunks=64, cpu_threads=1,
                                                            host_kv_bytes=0))
ctx.init_weights(0)
fn = ctx.lib.hs_probe_dense_mode
fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]
OPS = ["qkv", "rope", "o", "addnorm1", "gate_up", "silu", "down", "addnorm2"]


def t(n, mode):
    us = C.c_float()
    assert fn(ctx.h, n, mode, 32, 7, C.byref(us)) == 0, ctx.lib.hs_last_error()
    return us.value


for n in [int(a) for a in sys.argv[1:]] or (1, 16, 32, 64, 128, 256, 512):
    ops = {name: t(n, 1 << b) for b, name in enumerate(OPS)}
    g, e, a = t(n, 0x55), t(n, 0xAA), t(n, 0xFF)
    print(f"n={n:4d} " + " ".join(f"{k} {v:6.1f}" for k, v in ops.items())
          + f" | gemms {g:6.1f} glue {e:6.1f} layer {a:6.1f} us (gemm roofline frac "
          f"{66.5 / g:.2f})", flush=True)
