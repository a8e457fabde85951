"""Host CPU-attention throughput (the C1 worker pool) on Llama-3-8B shapes:
n items x (ctx+1) keys, all layers' KV in the pinned host arena."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200.models import get_transformer  # noqa: E402
from paper_2603_12831_b200.runtime import HsContext, RuntimeConfig  # noqa: E402

m = get_transformer("llama3-8b")
ctx_len = int(sys.argv[1]) if len(sys.argv) > 1 else 9000
n_items = int(sys.argv[2]) if len(sys.argv) > 2 else 32
threads = int(sys.argv[3]) if len(sys.argv) > 3 else 14
cap = ctx_len + 64
per_req = cap * m.n_layers * 2 * m.n_kv * m.head_dim * 2
rt = RuntimeConfig(max_rows=64, max_slots=n_items + 1, kv_pages=64, max_pages_per_req=8,
                   max_pos=256, max_chunks=64, cpu_threads=threads,
                   host_kv_bytes=per_req * n_items + (1 << 20))
ctx = HsContext(m, rt)
for s in range(n_items):
    ctx.host_kv_reserve(s, cap)
slots = np.arange(n_items, dtype=np.int32)
for layer in (1, 2):  # first touch of the arena pages, then timed
    t = time.perf_counter()
    ctx.cpu_attend(slots, np.full(n_items, layer, np.int32), np.full(n_items, ctx_len, np.int32))
    dt = time.perf_counter() - t
bytes_ = n_items * (ctx_len + 1) * 2 * m.n_kv * m.head_dim * 2
print(f"cpu attention: {n_items} items x ctx {ctx_len}, {threads} threads: {dt*1e3:.1f} ms, "
      f"{bytes_ / dt / 1e9:.1f} GB/s KV read, {n_items / dt:.0f} item-layers/s")
