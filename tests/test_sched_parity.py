"""Control-plane parity: the product engine reproduces the reference
simulator's decisions bit-for-bit on every recorded scenario
(tests/golden/sched_*.json.gz, generated from the unmodified reference by
oracle/gen_sched_golden.py): every BatchPlan, every per-layer merge, the
fitted latency models, counters, the full report, and digests of the audit,
event and layer-start logs."""

import copy
import gzip
import hashlib
import json

import pytest

from oracle.scenarios import SCENARIOS
from paper_2603_12831_b200.engine import Engine
from paper_2603_12831_b200.latency import model_set_to_dict
from paper_2603_12831_b200.scenario import scenario_from_dict


def _digest(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True).encode()).hexdigest()


def _plan_record(plan) -> dict:
    return {
        "ls_decode": list(plan.ls_decode),
        "ls_prefill_chunks": [[r, q] for r, q in plan.ls_prefill_chunks],
        "be_prefill_chunks": [[r, q] for r, q in plan.be_prefill_chunks],
        "be_decode_gpu": list(plan.be_decode_gpu),
        "be_offload_cpu": list(plan.be_offload_cpu),
        "swap_back_in": list(plan.swap_back_in),
        "piggyback_per_layer": {str(k): v for k, v in sorted(plan.piggyback_per_layer.items())},
        "loads": list(plan.loads),
    }


def _load(golden_dir, name):
    with gzip.open(golden_dir / f"sched_{name}.json.gz", "rt") as fh:
        return json.load(fh)


def run_product(doc, name):
    eng = Engine(scenario_from_dict(copy.deepcopy(doc), name))
    plans = []
    orig = eng._plan

    def wrapped():
        p = orig()
        plans.append(_plan_record(p))
        return p

    eng._plan = wrapped
    report = eng.run()
    return eng, report, plans


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_engine_bit_exact_against_reference(golden_dir, name):
    gold = _load(golden_dir, name)
    assert gold["doc"] == json.loads(json.dumps(SCENARIOS[name]))
    eng, report, plans = run_product(gold["doc"], name)
    assert model_set_to_dict(eng.models) == gold["models"]
    assert len(plans) == len(gold["plans"])
    for i, (mine, ref) in enumerate(zip(plans, gold["plans"])):
        assert mine == ref, f"plan {i} differs"
    merges = [[e["t"], e["request"], e["layer"], e["source"]] for e in eng.events
              if e["kind"] == "merge"]
    assert merges == gold["merges"]
    assert dict(sorted(report.counters.items())) == gold["counters"]
    assert json.loads(report.to_json()) == gold["report"]
    assert _digest(eng.audit) == gold["audit_sha"]
    assert _digest(eng.events) == gold["events_sha"]
    assert _digest([list(x) for x in eng.layer_start_log]) == gold["layer_start_sha"]


def test_appendix_b_golden_values(golden_dir):
    """SURVEY.md Appendix B numbers for the config-1 fixture."""
    gold = _load(golden_dir, "appendix_b")
    c = gold["counters"]
    assert c["iterations"] == 6099 and c["merges"] == 40 and c["injections"] == 2
    assert c["swap_out_done"] == 2 and c["swap_in_done"] == 2 and c["be_tokens_cpu"] == 19
    assert c["tokens_total"] == 6280 and c["residual_puts"] == c["residual_gets"] == 38
    r = gold["report"]
    assert r["ttft_attainment"] == 1.0 and r["tpot_attainment"] == 1.0
    assert abs(r["be_decode_tput"] - 244.35) < 1e-9
