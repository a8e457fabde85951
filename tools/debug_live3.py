"""Debug: detail of the first bad token in sync-pool/sync-swap live mode."""
import sys, os, collections
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
sys.argv = [sys.argv[0], "both"]
exec(open("tools/debug_live2.py").read().split("from test_live_parity import _live_run")[0])
from paper_2603_12831_b200 import runtime as RT
slot_log = []
_orig_slot_of = RT.CudaStep.slot_of
def slot_of(self, rid):
    new = rid not in self.slots
    s = _orig_slot_of(self, rid)
    if new:
        slot_log.append((self.iterations, rid, s))
    return s
RT.CudaStep.slot_of = slot_of
_orig_rel = RT.CudaStep._release_pending
def _release_pending(self):
    for rid in self._pending_release:
        if rid in self.slots:
            slot_log.append((self.iterations, rid, -self.slots[rid] - 1))
    return _orig_rel(self)
RT.CudaStep._release_pending = _release_pending
from test_live_parity import _live_run
from oracle import replay as R
from paper_2603_12831_b200.runtime import prompt_tokens
cfg, w, eng, step, n = _live_run(1, 0)
st = R.replay(eng.batch_trace, step.token_log, cfg, w, lambda rid, k: prompt_tokens(rid, k, cfg.vocab, 0))
print("bad", len(st.bad), "compared", st.compared)
first = {}
for b in st.bad:
    first.setdefault(b[0], b)
order = sorted(first.values(), key=lambda b: b[4])
print("first bads:", [(b[0], b[4]) for b in order])
rid, k = order[0][0], order[0][4]
print("slot history of", rid, [x for x in slot_log if x[1] == rid])
myslots = {x[2] for x in slot_log if x[1] == rid}
print("all users of its slot(s):", [x for x in slot_log if abs(x[2]) in myslots or (-x[2]-1) in myslots])
for i in range(max(0, k - 8), k + 1):
    it = eng.batch_trace[i]
    p = it["plan"]
    print(f"it {i}: dec {len(p['ls_decode'])}+{p['be_decode_gpu']} chunks {p['ls_prefill_chunks']} {p['be_prefill_chunks']}")
    for layer, merges, snap in it["layers"]:
        if merges:
            print(f"    L{layer}:", [(r, o, snap[r][0]) for r, o in merges])
    reqs, toks, lg = step.token_log[i]
    print("    tokens:", list(zip(reqs, toks.tolist())))
r = eng.requests[rid]
print(rid, "prompt", r.prompt_len, "out", r.output_len, "placements", r.placement_log)
