"""Diagnostic for K6 (attn_prefill_tc.cu) built with HS_NVCC_DEFS=-DHS_K6_TRACE:
one 1024-token chunk after 31,744 context tokens, then the SM-clock stamps
of CTA (0, 0)'s page handoffs (softmax S-ready / P-done, MMA-thread P-seen,
P.V issued, S(i+2) issued, refill done), as medians over pages 16..111 in
cycles.  Usage: HS_NVCC_DEFS=-DHS_K6_TRACE python tools/debug_k6_trace.py"""
import ctypes as C
import dataclasses
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200 import _build  # noqa: E402

_build.build(force=True)
from paper_2603_12831_b200 import profiler  # noqa: E402
from paper_2603_12831_b200.models import get_transformer  # noqa: E402
from paper_2603_12831_b200.runtime import HsContext, RuntimeConfig  # noqa: E402

m = dataclasses.replace(get_transformer("llama3-8b"), n_layers=1)
ctx = HsContext(m, RuntimeConfig(max_rows=4096, max_slots=8, kv_pages=600, max_pages_per_req=580,
                                 max_pos=37000, max_chunks=4096, cpu_threads=1, host_kv_bytes=0))
ctx.init_weights(0)
us = profiler._probe(ctx, "hs_probe_prefill", 1024, 31744, reps=3)
buf = (C.c_longlong * (8 * 128))()
assert ctx.lib.hs_debug_k6_trace(buf) == 0
t = np.array(list(buf), dtype=np.int64).reshape(8, 128).astype(np.float64)
names = ["s_ready", "p_done_t0", "mma_p_seen_t0", "mma_p_seen_t1", "pv_issued",
         "s2_issued", "refill_done", "p_done_t1"]
pg = slice(16, 112)
d = lambda a, b, sh=0: np.median(t[b][pg.start + sh:pg.stop + sh] - t[a][pg])  # noqa: E731
print(f"kernel {us:.1f} us; per page (median cycles):")
print("  page period (s_ready i -> i+1):", d(0, 0, 1))
print("  softmax t0 (s_ready -> p_done):", d(0, 1))
print("  t1 p_done - t0 p_done:", d(1, 7))
print("  p_done t0 -> MMA sees t0:", d(1, 2))
print("  MMA sees t0 -> sees t1:", d(2, 3))
print("  sees t1 -> PV issued:", d(3, 4))
print("  PV issued -> S(i+2) issued:", d(4, 5))
print("  S(i+2) issued -> refill done:", d(5, 6))
print("  S(i+2) issued -> softmax sees S(i+2):", d(5, 0, 2))
print("  refill done -> MMA sees P(i+1) t0:", d(6, 2, 1))
