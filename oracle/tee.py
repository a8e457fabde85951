"""Lockstep comparison of the libhs step against the numpy oracle (test
infrastructure only): drives both LayerSteps with the same engine events and
compares, per iteration, every greedy token and its logits.  Near-ties (top-2
logit gap within twice the measured logit error) teacher-force the oracle
onto the GPU's token so the sequences stay aligned."""

import numpy as np


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
