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


class TeeStep:
    def __init__(self, gpu, ora):
        self.gpu, self.ora = gpu, ora
        self.max_rel = 0.0
        self.compared = 0
        self.ties = 0
        self.bad: list = []

    def attach(self, engine):
        self.gpu.attach(engine)
        self.ora.attach(engine)

    def begin_iteration(self, plan):
        self.gpu.begin_iteration(plan)
        self.ora.begin_iteration(plan)

    def layer(self, layer, merges):
        self.gpu.layer(layer, merges)
        self.ora.layer(layer, merges)

    def end_iteration(self, plan):
        self.gpu.end_iteration(plan)
        mark = len(self.ora.logit_log)
        before = {rid: len(v) for rid, v in self.ora.generated.items()}
        self.ora.end_iteration(plan)
        ora_logits = {}
        # chain tokens were emitted during layer L, batch tokens just now
        for rid, lg in self.ora.logit_log[-(len(self.gpu.last_token_reqs)):]:
            ora_logits[rid] = lg
        logits = self.gpu.last_logits
        for i, (rid, tok) in enumerate(zip(self.gpu.last_token_reqs, self.gpu.last_tokens)):
            ref = ora_logits[rid]
            got = logits[i]
            rel = float(np.abs(got - ref).max() / np.abs(ref).max())
            self.max_rel = max(self.max_rel, rel)
            self.compared += 1
            ora_tok = self.ora.generated[rid][-1]
            if int(tok) != ora_tok:
                top2 = np.sort(ref)[-2:]
                gap = float(top2[1] - top2[0]) / float(np.abs(ref).max())
                if gap <= 2 * rel + 1e-6:
                    self.ties += 1
                    self.ora.force_token(rid, int(tok))
                else:
                    self.bad.append((rid, int(tok), ora_tok, gap, rel))
        del mark, before

    def cpu_service(self, host_id, items):
        self.gpu.cpu_service(host_id, items)
        self.ora.cpu_service(host_id, items)

    def swap_out_done(self, req):
        self.gpu.swap_out_done(req)

    def resumed_on_gpu(self, req):
        self.gpu.resumed_on_gpu(req)

    def preempted(self, req):
        self.gpu.preempted(req)

    def released(self, req):
        self.gpu.released(req)

    def finish(self):
        self.gpu.finish()


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
