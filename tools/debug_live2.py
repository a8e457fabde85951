"""Debug: bisect the live-path mismatch. argv[1] in {base, syncpool, syncswap, both}."""
import sys, os, collections
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from paper_2603_12831_b200 import runtime as RT
from oracle import replay as R

mode = sys.argv[1]
if mode in ("syncpool", "both"):
    def cpu_submit(self, items):
        for it in items:
            self._tags[it.req_id] = RT.result_tag(it.ctx_tokens, it.layer)
        self.ctx.cpu_attend([self.slot_of(it.req_id) for it in items], [it.layer for it in items],
                            [it.ctx_tokens for it in items])
        self.__dict__.setdefault("_fake_done", []).extend((it.req_id, it.layer) for it in items)
    def cpu_poll(self):
        out = self.__dict__.get("_fake_done", [])
        self._fake_done = []
        return out
    RT.LiveCudaStep.cpu_submit = cpu_submit
    RT.LiveCudaStep.cpu_poll = cpu_poll
if mode in ("syncswap", "both"):
    def swap_out_async(self, req):
        s = self.slot_of(req.id)
        self.ctx.host_kv_reserve(s, req.prompt_len + req.output_len + 1)
        self.ctx.swap_out(s, req.kv_held)
        return -1
    def swap_in_async(self, req):
        s = self.slot_of(req.id)
        self._ensure(s, req.ctx)
        self._flush_pages()
        self.ctx.swap_in(s, req.ctx)
        return -2
    def swap_done(self, t):
        return True
    RT.LiveCudaStep.swap_out_async = swap_out_async
    RT.LiveCudaStep.swap_in_async = swap_in_async
    RT.LiveCudaStep.swap_done = swap_done
from test_live_parity import _live_run
from paper_2603_12831_b200.runtime import prompt_tokens
cfg, w, eng, step, n = _live_run(1, 0)
c = eng.counters
st = R.replay(eng.batch_trace, step.token_log, cfg, w, lambda rid, k: prompt_tokens(rid, k, cfg.vocab, 0))
print(mode, "iters", n, "merges", c["merges"], "cpu_tok", c["be_tokens_cpu"], "swaps", c["swap_out_done"], c["swap_in_done"],
      "compared", st.compared, "ties", st.ties, "bad", len(st.bad), "max_rel", round(st.max_rel, 4),
      "bad reqs", collections.Counter(b[0] for b in st.bad).most_common(5))
