"""Device-polled piggyback merges (csrc/piggyback.cu; north star item 3):
the GPU takes the reference's merge decision -- the output FIFO head-run
with head.layer == layer, at most `cap` per layer, plus layer-1 injections
(pkg/src/hybridserve/engine.py:861-919) -- from the CPU workers' completion
tags, and continues / restarts / ends chains as _process_merge does
(engine.py:982-1022).

GPU: on a deterministic schedule (a BE backlog resident in host DRAM, no
arrivals, no swaps; after every layer the host waits until the CPU pool has
finished everything shipped so far, so every shipped result is complete
before its merge slot) the host-decided and the device-decided modes take
identical merges, layer by layer, and emit the same tokens.
"""

import collections
import copy
import sys
import time
from pathlib import Path

import numpy as np
import pytest

from oracle.scenarios import APPENDIX_B
from oracle.serve_oracle import device_weights, make_weights


def _sync_step_cls():
    from paper_2603_12831_b200.runtime import LiveCudaStep

    class SyncStep(LiveCudaStep):
        """Every layer runs to completion and the CPU pool drains before the
        next launch (no timing in the decisions)."""

        def layer(self, layer, merges):
            shipped = super().layer(layer, merges)
            return shipped

        def settle(self):
            self.ctx.sync()
            time.sleep(0.003)  # the pool's dispatcher picks up published items
            t0 = time.perf_counter()
            while self.ctx.lib.hs_cpu_in_flight(self.ctx.h) > 0:
                if time.perf_counter() - t0 > 30:
                    raise RuntimeError("CPU pool did not drain")
                time.sleep(1e-4)

    return SyncStep


def _deterministic_run(device_merges: bool, n_be: int = 12, iterations: int = 160, fake=None):
    from paper_2603_12831_b200.live import LiveEngine
    from paper_2603_12831_b200.models import TRANSFORMERS
    from paper_2603_12831_b200.runtime import RuntimeConfig
    from paper_2603_12831_b200.scenario import scenario_from_dict
    from paper_2603_12831_b200.state import SimRequest
    from paper_2603_12831_b200.workload import RequestSpec, ServiceClass

    cfg = TRANSFORMERS["tiny"]
    w = make_weights(cfg, 0)
    rt = RuntimeConfig(max_rows=512, max_slots=64, kv_pages=64, max_pages_per_req=16,
                       max_pos=2048, max_chunks=512, cpu_threads=4, host_kv_bytes=128 << 20)
    kw = {"ctx": fake(cfg, rt)} if fake else {"weights": device_weights(w), "keep_logits": True}
    step = _sync_step_cls()(cfg, rt, device_merges=device_merges, **kw)
    step.trace_tokens = True
    doc = copy.deepcopy(APPENDIX_B)
    doc["profiles"]["cluster"]["gpu_kv_capacity"] = 1  # BE stays in host DRAM
    doc["profiles"]["cluster"]["max_piggyback_per_layer"] = 4  # the cap binds
    eng = LiveEngine(scenario_from_dict(doc, "det"), step=step, pace_layers=64, batch_trace=True)
    rng = np.random.default_rng(7)
    for i in range(n_be):
        p, o = int(rng.integers(100, 300)), int(rng.integers(8, 16))
        r = SimRequest(RequestSpec(f"BE-{i:03d}", ServiceClass.BE, p, o, 0.0))
        eng.requests[r.id] = r
        r.admitted, r.phase, r.prefill_done, r.tokens_out = True, "decode", p, 1
        r.token_times = [0.0]
        r.first_token_time = 0.0
        need = r.prompt_len + r.output_len - r.tokens_out + 1
        eng.kv.alloc_host(0, need)
        r.swap_reserved, r.kv_place, r.kv_held = need, 0, r.ctx
        step.ctx.host_kv_reserve(step.slot_of(r.id), r.prompt_len + r.output_len + 1)
        eng._inject(r)
    orig_layer = step.layer

    def layer(l, merges):
        out = orig_layer(l, merges)
        if not device_merges:
            eng._submit_shipped(out)
            out = []
        step.settle()
        return out

    step.layer = layer

    def after(_n):
        eng.drain()
        step.settle()

    eng.run_live(max_iterations=iterations, arrivals=collections.deque(), idle_exit=True,
                 on_iteration=after)
    step.finish()
    merges = [[(l, list(m)) for l, m, _ in it["layers"] if m] for it in eng.batch_trace]
    return eng, step, merges


def test_device_and_host_merges_agree_on_the_fake_device():
    """The host replay of device decisions (LiveEngine device mode) against
    the Python model of the controller (tests/fake_device.py)."""
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from fake_device import FakeHsContext, FakePgContext

    eh, _, mh = _deterministic_run(False, fake=lambda c, r: FakeHsContext(c, r, cpu_ms=0.3))
    ed, _, md = _deterministic_run(True, fake=lambda c, r: FakePgContext(c, r, cpu_ms=0.3))
    assert eh.counters["merges"] > 100, eh.counters
    for k in ("merges", "injections", "be_tokens_cpu", "tokens_total", "iterations"):
        assert eh.counters[k] == ed.counters[k], (k, eh.counters[k], ed.counters[k])
    assert mh == md


@pytest.mark.gpu
def test_device_and_host_merges_agree(cuda):
    eh, sh, mh = _deterministic_run(False)
    ed, sd, md = _deterministic_run(True)
    assert eh.counters["merges"] > 100 and eh.counters["be_tokens_cpu"] > 10, eh.counters
    for k in ("merges", "injections", "be_tokens_cpu", "tokens_total", "iterations"):
        assert eh.counters[k] == ed.counters[k], (k, eh.counters[k], ed.counters[k])
    assert mh == md
    # the same tokens (up to near-ties of the two launch shapes' rounding)
    th = [(tuple(r), tuple(t)) for r, t, _ in sh.token_log]
    td = [(tuple(r), tuple(t)) for r, t, _ in sd.token_log]
    assert [r for r, _ in th] == [r for r, _ in td]
    same = sum(a == b for (_, x), (_, y) in zip(th, td) for a, b in zip(x, y))
    total = sum(len(x) for _, x in th)
    assert same >= 0.97 * total, (same, total)
    print(f"merges {eh.counters['merges']} identical in both modes; tokens {same}/{total}")
