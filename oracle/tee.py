"""Lockstep comparison of the libhs step against the numpy oracle (test
infrastructure only): drives both LayerSteps with the same engine events and
compares, per iteration, every greedy token and its logits.  The oracle is
teacher-forced onto the GPU's tokens (OracleStep.teacher: chain tokens before
the oracle's layer L, whose restart embeds the token; batch tokens before its
end of iteration), so a near-tie flip -- the GPU's token within twice the
measured logit error of the oracle's argmax -- does not fork the sequences;
any other disagreement is reported in `bad`."""

import numpy as np


class TeeStep:
    def __init__(self, gpu, ora):
        self.gpu, self.ora = gpu, ora
        self.max_rel = 0.0
        self.compared = 0
        self.ties = 0
        self.bad: list = []
        self.iterations = 0
        self.tie_iterations: list[int] = []  # iteration index of every near-tie

    def attach(self, engine):
        self.gpu.attach(engine)
        self.ora.attach(engine)

    def begin_iteration(self, plan):
        self.gpu.begin_iteration(plan)
        self.ora.begin_iteration(plan)

    def layer(self, layer, merges):
        self.gpu.layer(layer, merges)
        if layer == self.gpu.model.n_layers and merges:
            # chain tokens of this layer: the GPU's choice (the oracle's layer
            # L also embeds the token for the chain's restart)
            toks = self.gpu.ctx.iter_end()
            reqs = self.gpu._logit_reqs + self.gpu._merge_L
            chain = set(self.gpu._merge_L)
            self.ora.teacher.update({r: int(t) for r, t in zip(reqs, toks) if r in chain})
        self.ora.layer(layer, merges)

    def end_iteration(self, plan):
        self.gpu.end_iteration(plan)
        mark = len(self.ora.logit_log)
        before = {rid: len(v) for rid, v in self.ora.generated.items()}
        n_batch = len(self.gpu.last_token_reqs) - len(self.gpu._merge_L)
        self.ora.teacher.update({r: int(t) for r, t in zip(self.gpu.last_token_reqs[:n_batch],
                                                           self.gpu.last_tokens[:n_batch])})
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
            ora_tok = int(np.argmax(ref))
            if int(tok) != ora_tok:
                gap = float(ref[ora_tok] - ref[int(tok)]) / float(np.abs(ref).max())
                if gap <= 2 * rel + 1e-6:
                    self.ties += 1
                    self.tie_iterations.append(self.iterations)
                else:
                    self.bad.append((rid, int(tok), ora_tok, gap, rel))
        del mark, before
        self.iterations += 1

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
