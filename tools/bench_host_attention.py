"""Single-thread throughput of the C1 host attention kernel (hs_host_attention:
all KV heads of one item, Llama-3-8B geometry), no GPU needed.

    python tools/bench_host_attention.py [keys] [impl 1=AVX-512-BF16 2=AVX2] [reps]
"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200 import _lib  # noqa: E402

keys = int(sys.argv[1]) if len(sys.argv) > 1 else 9000
impl = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
n_q, n_kv, hd = 32, 8, 128
lib = _lib.load()
rng = np.random.default_rng(0)
q = rng.integers(0x3c00, 0x3f00, n_q * hd, dtype=np.uint16)
k = rng.integers(0x3c00, 0x3f00, n_kv * keys * hd, dtype=np.uint16)
v = rng.integers(0x3c00, 0x3f00, n_kv * keys * hd, dtype=np.uint16)
out = np.zeros(n_q * hd, np.uint16)
lse = np.zeros(n_q, np.float32)
P = C.c_void_p
ts = []
for i in range(reps + 2):
    t = time.perf_counter()
    _lib.check(lib.hs_host_attention(q.ctypes.data_as(P), k.ctypes.data_as(P), v.ctypes.data_as(P),
                                     keys, n_q, n_kv, hd, out.ctypes.data_as(P),
                                     lse.ctypes.data_as(P), impl), "hs_host_attention")
    ts.append(time.perf_counter() - t)
dt = float(np.median(ts[2:]))
by = 2 * n_kv * keys * hd * 2
print(f"impl {impl} keys {keys}: {dt * 1e3:.2f} ms per item-layer, {by / dt / 1e9:.2f} GB/s single thread")
