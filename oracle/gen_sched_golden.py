"""Golden-vector generator for the control plane (test infrastructure only).

Runs the UNMODIFIED reference simulator (`hybridserve`, imported read-only
from /root/reference/pkg/src; this script only runs in the dev container
where the reference is mounted) on the scenarios in SCENARIOS and records
what pins the hot path's inputs:

* every BatchPlan returned by Engine._plan (reference engine.py:577-805),
* per-layer merges (the `merge` events, engine.py:902-919),
* counters, the report JSON and the audit log,
* SHA-256 digests of the full event log and layer_start_log.

Output: tests/golden/sched_<name>.json.gz.  The product engine is then
required to reproduce all of it bit-for-bit (tests/test_sched_parity.py).

Usage:  python oracle/gen_sched_golden.py
"""

from __future__ import annotations

import copy
import gzip
import hashlib
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF_SRC = Path("/root/reference/pkg/src")
OUT = ROOT / "tests" / "golden"

sys.path.insert(0, str(ROOT))
from oracle.scenarios import SCENARIOS  # noqa: E402


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


def run_reference(doc: dict, name: str, inject=None) -> dict:
    os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
    sys.dont_write_bytecode = True
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    from hybridserve.engine import Engine
    from hybridserve.scenario import scenario_from_dict

    eng = Engine(scenario_from_dict(copy.deepcopy(doc), name))
    plans = []
    orig = eng._plan

    def wrapped():
        plan = orig()
        plans.append(_plan_record(plan))
        return plan

    eng._plan = wrapped
    report = eng.run()
    merges = [[e["t"], e["request"], e["layer"], e["source"]] for e in eng.events
              if e["kind"] == "merge"]
    return {
        "name": name,
        "doc": doc,
        "plans": plans,
        "merges": merges,
        "counters": dict(sorted(report.counters.items())),
        "report": json.loads(report.to_json()),
        "audit_sha": _digest(eng.audit),
        "audit_len": len(eng.audit),
        "events_sha": _digest(eng.events),
        "events_len": len(eng.events),
        "layer_start_sha": _digest([list(x) for x in eng.layer_start_log]),
        "layer_starts": len(eng.layer_start_log),
        "models": _models_doc(eng.models),
    }


def _models_doc(models) -> dict:
    from hybridserve.latency import model_set_to_dict

    return model_set_to_dict(models)


def main() -> None:
    if not REF_SRC.exists():
        raise SystemExit("reference not mounted; golden vectors are generated in the dev container")
    OUT.mkdir(parents=True, exist_ok=True)
    for name, doc in SCENARIOS.items():
        rec = run_reference(doc, name)
        path = OUT / f"sched_{name}.json.gz"
        with gzip.open(path, "wt") as fh:
            json.dump(rec, fh, sort_keys=True)
        print(f"{name}: plans={len(rec['plans'])} merges={len(rec['merges'])} "
              f"events={rec['events_len']} -> {path.name} ({path.stat().st_size // 1024} KiB)")


if __name__ == "__main__":
    main()
