"""Debug: live run of config 1 + oracle replay; per-token mismatch report."""
import sys, os, collections
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from test_live_parity import _live_run
from oracle import replay as R
from paper_2603_12831_b200.runtime import prompt_tokens

pace = int(sys.argv[1]) if len(sys.argv) > 1 else 1
tail = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg, w, eng, step, n = _live_run(pace, tail)
print("counters", {k: v for k, v in eng.counters.items() if v})
# annotate which tokens are chain tokens
chain_tok = set()
for i, it in enumerate(eng.batch_trace):
    for layer, merges, snap in it["layers"]:
        if layer == cfg.n_layers:
            for rid, o in merges:
                chain_tok.add((i, rid))
orig = R.ReplayStats
bad_detail = []
class S(orig):
    pass
# monkeypatch replay loop to record iteration index of bad tokens
st = R.replay(eng.batch_trace, step.token_log, cfg, w, lambda rid, k: prompt_tokens(rid, k, cfg.vocab, 0))
print("compared", st.compared, "ties", st.ties, "bad", len(st.bad), "max_rel", st.max_rel)
# locate bad tokens by iteration
idx = {}
for i, (reqs, toks, lg) in enumerate(step.token_log):
    for rid in reqs:
        idx.setdefault(rid, []).append(i)
byreq = collections.Counter(b[0] for b in st.bad)
print("bad by request", byreq.most_common(12))
for rid, _ in byreq.most_common(4):
    r = eng.requests[rid]
    print(rid, r.cls, "prompt", r.prompt_len, "out", r.output_len, "placements", r.placement_log[:6])
    its = idx.get(rid, [])
    kinds = ["chain" if (i, rid) in chain_tok else "batch" for i in its]
    print("   token iterations/kinds", list(zip(its, kinds))[:40])
first = {}
for b in st.bad:
    first.setdefault(b[0], b[4])
print("first bad iteration per request:", sorted(first.items(), key=lambda x: x[1])[:20])
for rid, k in sorted(first.items(), key=lambda x: x[1])[:6]:
    kind = "chain" if (k, rid) in chain_tok else "batch"
    # merges of this rid up to k
    hist = []
    for i, it in enumerate(eng.batch_trace[:k + 1]):
        for layer, merges, snap in it["layers"]:
            for r2, o in merges:
                if r2 == rid:
                    hist.append((i, layer, o, snap[rid][0]))
        if rid in it["snap"]:
            hist.append((i, "row", it["snap"][rid]))
    print(rid, "first bad at", k, kind, "history tail", hist[-12:])
