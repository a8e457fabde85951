"""CPU tests of the live serving host path (`LiveEngine` + `LiveCudaStep`)
against a recording stand-in for libhs (tests/fake_device.py): the
asynchronous CPU pool, swaps on the copy stream, pipelined iterations and
pacing, with wall-clock completions and randomised CPU latencies.  Checks the
reference's conservation rules end to end (every request completes with its
output length, KV and residual bookkeeping return to zero, every slot is
released) — reference pkg/src/hybridserve/engine.py:200-216 (complete),
402-508 (swaps), 512-560 (CPU service), 879-1047 (iterations).
"""

import copy
import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent))

from fake_device import FakeHsContext, FakePgContext  # noqa: E402

from oracle.scenarios import APPENDIX_B  # noqa: E402


def _run(kv_tokens, seed, pace_layers=1, pace_tail=0, cpu_ms=0.5, device_merges=False):
    from paper_2603_12831_b200.live import LiveEngine
    from paper_2603_12831_b200.models import TRANSFORMERS
    from paper_2603_12831_b200.runtime import LiveCudaStep, RuntimeConfig
    from paper_2603_12831_b200.scenario import scenario_from_dict

    cfg = TRANSFORMERS["tiny"]
    rt = RuntimeConfig(max_rows=1024, max_slots=64, kv_pages=256, max_pages_per_req=16,
                       max_pos=2048, max_chunks=1024, cpu_threads=4, host_kv_bytes=256 << 20)
    fake = (FakePgContext if device_merges else FakeHsContext)(cfg, rt, iter_ms=0.25,
                                                               cpu_ms=cpu_ms, rng_seed=seed)
    step = LiveCudaStep(cfg, rt, ctx=fake, device_merges=device_merges)
    doc = copy.deepcopy(APPENDIX_B)
    doc["profiles"]["cluster"]["gpu_kv_capacity"] = kv_tokens
    eng = LiveEngine(scenario_from_dict(doc, "live"), step=step, pace_layers=pace_layers,
                     pace_tail=pace_tail)
    n = eng.run_live(horizon_s=30.0)
    step.finish()
    return eng, step, fake, n


@pytest.mark.parametrize("device_merges", [False, True])
@pytest.mark.parametrize("seed,pace", [(0, (1, 0)), (1, (2, 1)), (2, (1, 0))])
def test_live_engine_serves_every_request(seed, pace, device_merges):
    eng, step, fake, n = _run(1600, seed, *pace, device_merges=device_merges)
    c = eng.counters
    assert not eng.stalled
    assert c["tokens_total"] == sum(r.output_len for r in eng.requests.values())
    assert all(r.phase == "done" and r.tokens_out == r.output_len for r in eng.requests.values())
    # the asynchronous machinery was exercised
    assert c["swap_out_done"] > 0 and c["merges"] > 0 and c["be_tokens_cpu"] > 0
    assert c["swap_out_started"] == c["swap_out_done"]
    # conservation: queues drained, KV returned, residuals consumed, slots free
    assert not eng.queues.output and not eng.pending_injections and not eng._order
    assert eng.kv.gpu_used == 0 and eng.kv.host_used == [0]
    assert not any(eng.residuals.outstanding(r) for r in eng.requests)
    assert not step.slots and len(step.free_slots) == step.rt.max_slots
    assert not fake.host_kv
    if device_merges:  # the device's FIFO drained in step with the host mirror
        assert not fake.fifo and not fake.inj and fake.merged_total == c["merges"] - c["injections"]
        assert fake.bound_binding == 0
    # every token time was patched to its iteration's device completion
    for r in eng.requests.values():
        assert r.token_times == sorted(r.token_times)
    assert all("end" in rec for rec in eng.iteration_log)


def test_live_engine_reports_a_wedged_policy():
    """Appendix B's 1000-token GPU KV budget can be filled by LS requests
    alone on the wall clock (two decodes + one partial prefill); the policy
    then has nothing to swap out.  The live engine must detect it (the
    reference's event loop just runs out of events) instead of spinning to
    the horizon."""
    import time

    t = time.perf_counter()
    stalled = 0
    for seed in range(3):
        eng, _, _, _ = _run(1000, seed)
        stalled += eng.stalled
        if eng.stalled:
            assert eng.kv.gpu_used == eng.kv.gpu_capacity
    assert time.perf_counter() - t < 25.0
    assert stalled >= 1
