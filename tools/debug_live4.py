"""Debug: compare GPU ship/result rows of every piggyback item with the oracle replay."""
import sys, os, collections, ctypes as C
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from types import SimpleNamespace
from paper_2603_12831_b200 import runtime as RT
from oracle import llama_ops as O
rows = {}
def cpu_submit(self, items):
    for it in items:
        self._tags[it.req_id] = RT.result_tag(it.ctx_tokens, it.layer)
    slots = [self.slot_of(it.req_id) for it in items]
    m = self.model
    ships = []
    for s in slots:
        b = np.zeros(m.qkv_dim, np.uint16)
        self.ctx._call("hs_read_ship", s, b.ctypes.data_as(C.c_void_p), b.nbytes)
        ships.append(O.from_bf16_bits(b))
    self.ctx.cpu_attend(slots, [it.layer for it in items], [it.ctx_tokens for it in items])
    for it, s, sh in zip(items, slots, ships):
        b = np.zeros(m.n_q * m.head_dim, np.uint16)
        self.ctx._call("hs_read_result", s, b.ctypes.data_as(C.c_void_p), b.nbytes)
        rows[(it.req_id, it.layer, it.ctx_tokens)] = (sh, O.from_bf16_bits(b), s)
    self.__dict__.setdefault("_fake_done", []).extend((it.req_id, it.layer) for it in items)
def cpu_poll(self):
    out = self.__dict__.get("_fake_done", [])
    self._fake_done = []
    return out
RT.LiveCudaStep.cpu_submit = cpu_submit
RT.LiveCudaStep.cpu_poll = cpu_poll
from test_live_parity import _live_run
from oracle.serve_oracle import OracleStep
from oracle.replay import _Engine
from paper_2603_12831_b200.runtime import prompt_tokens
cfg, w, eng, step, n = _live_run(1, 0)
ora = OracleStep(cfg, w, lambda rid, k: prompt_tokens(rid, k, cfg.vocab, 0))
e2 = _Engine(cfg.n_layers); ora.attach(e2)
def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-9))
nq = cfg.n_q * cfg.head_dim
worst_ship = worst_res = 0.0
reported = 0
for k_it, (it, (reqs, toks, lg)) in enumerate(zip(eng.batch_trace, step.token_log)):
    e2.update(it["snap"]); plan = SimpleNamespace(**it["plan"])
    ora.begin_iteration(plan); n_log = len(ora.logit_log)
    for layer, merges, snap in it["layers"]:
        e2.update(snap); items = []
        for rid, outcome in merges:
            if outcome != "inject":
                lay0, pos, q, kk, vv = ora.ship[rid]
                key = (rid, lay0 + 1, pos)
                ora.cpu_service(0, [SimpleNamespace(req_id=rid, layer=lay0 + 1, ctx_tokens=pos)])
                if key in rows:
                    sh, res, slot = rows[key]
                    oship = np.concatenate([q.reshape(-1), kk.reshape(-1), vv.reshape(-1)])
                    rs, rr = rel(sh, oship), rel(res, ora.result[rid])
                    worst_ship, worst_res = max(worst_ship, rs), max(worst_res, rr)
                    if (rs > 2e-2 or rr > 2e-2) and reported < 12:
                        reported += 1
                        print(f"it {k_it} L{layer} {rid} slot {slot} item {key}: ship rel {rs:.3e} (q {rel(sh[:nq], q.reshape(-1)):.2e} k {rel(sh[nq:nq+cfg.n_kv*cfg.head_dim], kk.reshape(-1)):.2e} v {rel(sh[nq+cfg.n_kv*cfg.head_dim:], vv.reshape(-1)):.2e}) result rel {rr:.3e}")
                else:
                    print("missing gpu rows for", key)
            items.append((SimpleNamespace(req_id=rid, layer=layer), outcome))
        ora.layer(layer, items)
    ora.end_iteration(plan)
    for rid, tok in zip(reqs, toks):
        ora.force_token(rid, int(tok))
print("worst ship", worst_ship, "worst result", worst_res)
