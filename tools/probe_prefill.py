"""K6 chunked-prefill attention on Llama-3-8B geometry: device time of one
layer's launch (hs_probe_prefill: one request, q chunk tokens after `done`
context tokens) and its tensor throughput, 4 * n_q * hd flops per attended
pair (pairwise_units, reference scheduling.py:127-133).

    python tools/probe_prefill.py [config]      (HS_PREFILL_MMA=1: warp-MMA kernel)
"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200 import profiler  # noqa: E402
from paper_2603_12831_b200.models import get_transformer  # noqa: E402
from paper_2603_12831_b200.runtime import HsContext, RuntimeConfig  # noqa: E402
from paper_2603_12831_b200.scheduling import pairwise_units  # noqa: E402
import dataclasses  # noqa: E402

m = dataclasses.replace(get_transformer(sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"), n_layers=1)
ctx = HsContext(m, RuntimeConfig(max_rows=4096, max_slots=8, kv_pages=600, max_pages_per_req=580,
                                 max_pos=37000, max_chunks=4096, cpu_threads=1, host_kv_bytes=0))
ctx.init_weights(0)
peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()) \
    if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else {}
kern = "warp-mma" if os.environ.get("HS_PREFILL_MMA") else "tcgen05"
for q, done in ((64, 0), (256, 0), (512, 0), (512, 1536), (2048, 0), (512, 8192), (1024, 31744)):
    us = profiler._probe(ctx, "hs_probe_prefill", q, done, reps=10)
    fl = 4.0 * m.n_q * m.head_dim * pairwise_units(done, q)
    tf = fl / (us * 1e-6) / 1e12
    print(json.dumps({"kernel": kern, "q": q, "done": done, "us": round(us, 2),
                      "tflops": round(tf, 1),
                      "frac_of_bf16_peak": round(tf / peak.get("bf16_tflops", 1590.0), 3)}))
