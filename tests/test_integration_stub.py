"""The INTEGRATION.md stub (integration/hybridserve_b200.py) is runnable.

CPU: over the UNMODIFIED reference engine (/root/reference, when present) with
a recording stand-in for libhs: the reference's own simulation is unchanged
(identical counters and report to a plain reference run) while every
iteration, layer, merge, CPU service and swap reaches the device boundary
with valid arguments.  GPU: the same stub over this repository's restatement
of the engine (the reference is not on the GPU box) on the real libhs emits
exactly the tokens of the CudaStep-driven engine on the same schedule.
"""

import copy
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(Path(__file__).resolve().parent))
REF = Path("/root/reference/pkg/src")

from oracle.scenarios import APPENDIX_B  # noqa: E402


def _rt():
    from paper_2603_12831_b200.runtime import RuntimeConfig

    return RuntimeConfig(max_rows=2048, max_slots=64, kv_pages=256, max_pages_per_req=16,
                         max_pos=2048, max_chunks=1024, cpu_threads=2, host_kv_bytes=64 << 20)


@pytest.mark.skipif(not REF.exists(), reason="reference package not present on this host")
def test_stub_over_the_unmodified_reference():
    from fake_device import FakeHsContext

    sys.path.insert(0, str(REF))
    try:
        import hybridserve.engine as ref_engine
        from hybridserve.scenario import scenario_from_dict as ref_scenario
    finally:
        sys.path.remove(str(REF))
    from integration.hybridserve_b200 import engine_class
    from paper_2603_12831_b200.models import TRANSFORMERS
    from paper_2603_12831_b200.runtime import CudaStep

    doc = copy.deepcopy(APPENDIX_B)
    doc["horizon_s"] = 2.0
    plain = ref_engine.Engine(ref_scenario(doc)).run()
    rt = _rt()
    fake = FakeHsContext(TRANSFORMERS["tiny"], rt)
    dev = CudaStep(TRANSFORMERS["tiny"], rt, ctx=fake)
    eng = engine_class(ref_engine.Engine)(ref_scenario(doc), model="tiny", rt=rt, device=dev)
    rep = eng.run()
    assert rep.counters == plain.counters
    assert rep.to_json() == plain.to_json()
    c = rep.counters
    assert fake.calls["iter_begin"] == c["iterations"]
    assert fake.calls["layer"] == c["iterations"] * doc["profiles"]["cluster"]["layers"]
    assert fake.calls["iter_end"] == c["iterations"]
    assert c["merges"] > 0 and fake.calls["cpu_attend"] > 0 and fake.calls["swap"] > 0
    # every token of the run came back through hs_iter_end
    assert sum(len(v) for v in dev.generated.values()) == c["tokens_total"]


@pytest.mark.gpu
def test_stub_emits_the_cudastep_tokens(cuda):
    from integration.hybridserve_b200 import engine_class
    from oracle.serve_oracle import device_weights, make_weights
    from paper_2603_12831_b200.engine import Engine
    from paper_2603_12831_b200.models import TRANSFORMERS
    from paper_2603_12831_b200.runtime import CudaStep
    from paper_2603_12831_b200.scenario import scenario_from_dict

    cfg = TRANSFORMERS["tiny"]
    w = device_weights(make_weights(cfg, 0))
    doc = copy.deepcopy(APPENDIX_B)
    doc["horizon_s"] = 1.3
    ref_step = CudaStep(cfg, _rt(), weights=w)
    r1 = Engine(scenario_from_dict(doc, "a"), step=ref_step).run()
    ref_step.finish()
    eng = engine_class(Engine)(scenario_from_dict(doc, "b"), model="tiny", rt=_rt(), weights=w)
    r2 = eng.run()
    assert r1.counters == r2.counters
    assert eng.device.generated == ref_step.generated
    assert sum(len(v) for v in ref_step.generated.values()) > 500
