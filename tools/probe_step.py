"""Device time of whole serving iterations of Llama-3-8B issued straight
through the C ABI (no engine, no Python planning between layers): B LS
decode rows at context `ctx` plus M piggyback merges and M chain carries
per layer, N iterations back to back between two events.  Compared with the
live bench's iteration_ms_p50 it separates kernel time from host-induced
GPU idle.

    python tools/probe_step.py [B] [ctx] [M] [N] [config]

(config llama3-70b-tp8: one rank's shard of config 4, the exchange with the
other ranks left out -- its per-rank compute.)
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_12831_b200.models import get_transformer  # noqa: E402
from paper_2603_12831_b200.runtime import (HsContext, RuntimeConfig,  # noqa: E402
                                           decode_chunks)

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
CTX = int(sys.argv[2]) if len(sys.argv) > 2 else 700
M = int(sys.argv[3]) if len(sys.argv) > 3 else 0
N = int(sys.argv[4]) if len(sys.argv) > 4 else 50
m = get_transformer(sys.argv[5] if len(sys.argv) > 5 else "llama3-8b")
npg = (CTX + 64) // 64
ctx = HsContext(m, RuntimeConfig(max_rows=1024, max_slots=B + M + 8, kv_pages=(B + M) * npg + 8,
                                 max_pages_per_req=npg, max_pos=CTX + 64, max_chunks=4096,
                                 cpu_threads=1, host_kv_bytes=0))
ctx.init_weights(0)
for s in range(B + M):
    ctx.set_page_table(s, list(range(s * npg, (s + 1) * npg)))
rows = list(range(B))
chunks, begin = decode_chunks([CTX + 1] * B, m.n_kv)
chunks = [(r, r, a, b, c) for r, _, a, b, c in chunks]
msl = list(range(B, B + M))


T = {"begin": 0.0, "layer": 0.0, "end": 0.0}


def iteration():
    a = time.perf_counter()
    ctx.iter_begin(rows, [CTX] * B, [-1] * B, B, chunks, begin, [], rows)
    b = time.perf_counter()
    for layer in range(1, m.n_layers + 1):
        carry = msl if layer > 1 else []
        ctx.layer(layer, carry, [CTX] * len(carry), msl, [], [])
    c = time.perf_counter()
    t = ctx.iter_end_async()
    T["begin"] += b - a
    T["layer"] += c - b
    T["end"] += time.perf_counter() - c
    return t


for _ in range(3):
    iteration()
ctx.sync()
for k in T:
    T[k] = 0.0
t0 = ctx.timer()
w0 = time.perf_counter()
for _ in range(N):
    iteration()
w1 = time.perf_counter()
t1 = ctx.timer()
ctx.sync()
w2 = time.perf_counter()
ms = ctx.elapsed_ms(t0, t1) / N
# every weight byte once per iteration (layers + LM head) at the measured HBM rate
roof = (m.params_per_layer * m.n_layers + m.vocab * m.d_model) * 2 / 6549.8e9 * 1e3
print(f"B={B} ctx={CTX} M={M}: device {ms:.3f} ms/iter; host issue {(w1 - w0) * 1e3 / N:.3f} "
      f"ms/iter; wall {(w2 - w0) * 1e3 / N:.3f} ms/iter; weight roofline {roof:.2f} ms "
      f"(frac {roof / ms:.2f}); host us: begin {T['begin'] * 1e6 / N:.1f}, per layer "
      f"{T['layer'] * 1e6 / N / m.n_layers:.1f}, end {T['end'] * 1e6 / N:.1f}", flush=True)
# device-only: a spin kernel holds the stream while the host issues two
# iterations (the staging ring lets the host run two ahead), so the events
# bracket pure device time
import torch  # noqa: E402

ext = torch.cuda.ExternalStream(ctx.lib.hs_stream(ctx.h))
dev = []
for _ in range(8):
    with torch.cuda.stream(ext):
        torch.cuda._sleep(30_000_000)
    a = ctx.timer()
    iteration()
    iteration()
    b = ctx.timer()
    ctx.sync()
    dev.append(ctx.elapsed_ms(a, b) / 2)
dev.sort()
print(f"   device-only (host ahead): {dev[len(dev) // 2]:.3f} ms/iter", flush=True)
ctx.close()
