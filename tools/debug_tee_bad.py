"""Diagnostic: run the Appendix-B tee (tests/test_serving.py) and print every
row whose logits miss the oracle by more than 2e-2, with its iteration and
whether it was a piggyback-chain row.  Usage: python tools/debug_tee_bad.py [runs]"""

import copy
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.scenarios import APPENDIX_B  # noqa: E402
from oracle.serve_oracle import OracleStep, device_weights, make_weights  # noqa: E402
from oracle.tee import TeeStep  # noqa: E402
from paper_2603_12831_b200.engine import Engine  # noqa: E402
from paper_2603_12831_b200.models import TRANSFORMERS  # noqa: E402
from paper_2603_12831_b200.runtime import CudaStep, RuntimeConfig, prompt_tokens  # noqa: E402
from paper_2603_12831_b200.scenario import scenario_from_dict  # noqa: E402


class LogTee(TeeStep):
    def __init__(self, gpu, ora):
        super().__init__(gpu, ora)
        self.rows = []

    def end_iteration(self, plan):
        before = self.max_rel
        self.max_rel = 0.0
        n_chain = len(self.gpu._merge_L)
        reqs = list(self.gpu.last_token_reqs)
        super().end_iteration(plan)
        if self.max_rel > 2e-2:
            ora = {rid: lg for rid, lg in self.ora.logit_log[-len(reqs):]}
            for i, rid in enumerate(reqs):
                ref = ora[rid]
                got = self.gpu.last_logits[i]
                rel = float(np.abs(got - ref).max() / np.abs(ref).max())
                if rel > 2e-2:
                    self.rows.append((self.iterations - 1, rid, i >= len(reqs) - n_chain,
                                      round(rel, 3), bool(np.isfinite(got).all()),
                                      float(np.abs(got).max()), float(np.abs(ref).max())))
        self.max_rel = max(before, self.max_rel)


def run():
    cfg = TRANSFORMERS["tiny"]
    w = make_weights(cfg, 0)
    rt = RuntimeConfig(max_rows=2048, max_slots=64, kv_pages=256, max_pages_per_req=16,
                       max_pos=2048, max_chunks=1024, cpu_threads=4, host_kv_bytes=256 << 20)
    gpu = CudaStep(cfg, rt, weights=device_weights(w), keep_logits=True)
    ora = OracleStep(cfg, w, lambda rid, n: prompt_tokens(rid, n, cfg.vocab, 0))
    tee = LogTee(gpu, ora)
    eng = Engine(scenario_from_dict(copy.deepcopy(APPENDIX_B), "appendix_b"), step=tee)
    eng.run()
    gpu.finish()
    return tee


if __name__ == "__main__":
    for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
        t = run()
        print(f"run {k}: max_rel={t.max_rel:.3e} bad={len(t.bad)} ties={t.ties} "
              f"n_bad_rows={len(t.rows)}", flush=True)
        for r in t.rows[:12]:
            print("   ", r, flush=True)
