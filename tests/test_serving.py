"""End-to-end serving parity (config 1: tiny Llama, 8 LS + 32 BE, the
Appendix B schedule with swap-out/in, injections and piggyback merges).

The engine replays the reference's schedule (bit-exact, test_sched_parity)
while a LayerStep executes the numerics.  `TeeStep` drives libhs
(`CudaStep`) and the numpy oracle (`OracleStep`) in lockstep and compares,
per iteration, every produced token and its logits (relative error bound
2e-2, the north star's bf16 tolerance).  Greedy tokens must agree except at
genuine near-ties (top-2 logit gap below the observed logit error), where the
oracle is teacher-forced onto the GPU's token so the sequences stay aligned.
"""

import copy

import numpy as np
import pytest

from oracle.scenarios import APPENDIX_B
from oracle.serve_oracle import OracleStep, device_weights, make_weights
from oracle.tee import TeeStep
from paper_2603_12831_b200.engine import Engine
from paper_2603_12831_b200.models import TRANSFORMERS
from paper_2603_12831_b200.scenario import scenario_from_dict

LOGIT_REL_TOL = 2e-2


def _prompt_fn(vocab):
    from paper_2603_12831_b200.runtime import prompt_tokens

    return lambda rid, n: prompt_tokens(rid, n, vocab, 0)


def test_oracle_step_runs_appendix_b_schedule():
    """CPU-only: the oracle LayerStep consumes the full Appendix-B event
    stream (chains, swaps, injections) and emits every token the engine
    counts."""
    cfg = TRANSFORMERS["tiny"]
    ora = OracleStep(cfg, make_weights(cfg, 0), _prompt_fn(cfg.vocab))
    doc = copy.deepcopy(APPENDIX_B)
    doc["horizon_s"] = 1.35  # first swap-outs at ~1.26 s
    eng = Engine(scenario_from_dict(doc, "b"), step=ora)
    report = eng.run()
    produced = sum(len(v) for v in ora.generated.values())
    assert produced == report.counters["tokens_total"]
    assert report.counters["merges"] > 0 and report.counters["be_tokens_cpu"] > 0
    assert report.counters["injections"] > 0


@pytest.mark.gpu
def test_cuda_step_matches_oracle_on_appendix_b(cuda):
    from paper_2603_12831_b200.runtime import CudaStep, RuntimeConfig

    cfg = TRANSFORMERS["tiny"]
    w = make_weights(cfg, 0)
    rt = RuntimeConfig(max_rows=2048, max_slots=64, kv_pages=256, max_pages_per_req=16,
                       max_pos=2048, max_chunks=1024, cpu_threads=4, host_kv_bytes=256 << 20)
    gpu = CudaStep(cfg, rt, weights=device_weights(w), keep_logits=True)
    ora = OracleStep(cfg, w, _prompt_fn(cfg.vocab))
    tee = TeeStep(gpu, ora)
    eng = Engine(scenario_from_dict(copy.deepcopy(APPENDIX_B), "appendix_b"), step=tee)
    report = eng.run()
    c = report.counters
    assert c["merges"] == 40 and c["swap_out_done"] == 2 and c["be_tokens_cpu"] == 19
    assert tee.compared == c["tokens_total"] == 6280
    assert not tee.bad, tee.bad[:5]
    assert tee.max_rel < LOGIT_REL_TOL, tee.max_rel
    # random-init logits are flat (std ~0.3 over 1024 ids): near-ties where
    # the top-2 gap is below twice the measured logit error occur at ~1 %
    assert tee.ties <= 0.05 * tee.compared
    print(f"compared={tee.compared} max_rel={tee.max_rel:.2e} ties={tee.ties}")
