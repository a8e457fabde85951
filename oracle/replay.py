"""Replay of a live run's realised schedule through the CPU oracle (test
infrastructure only; never imported by the product).

`LiveEngine(batch_trace=True)` records, per iteration, the plan's rows, every
layer's merges with their outcomes and the request state each call saw;
`LiveCudaStep(trace_tokens=True)` records the greedy tokens (and logits) the
GPU produced.  `replay()` drives `OracleStep` through exactly that schedule —
the same LayerStep calls the virtual-clock engine would make (reference
pkg/src/hybridserve/engine.py:879-1047) — and compares every token.  The CPU
service of a merged work item is evaluated just before its merge: a chain has
at most one item in flight (engine.py:982-1022), so its shipped q/k/v is
still the one the host worker attended.  The oracle is teacher-forced onto
the GPU's token (OracleStep.teacher, set before the iteration runs, so a
chain's restart at layer L embeds the GPU's token too), so a near-tie flip
does not fork the two sequences.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np

from oracle.serve_oracle import OracleStep


class _Req:
    __slots__ = ("id", "ctx", "prompt_len", "output_len", "prefill_done", "rebuild_tokens",
                 "phase")

    @property
    def prefill_target(self) -> int:
        return self.prompt_len + self.rebuild_tokens


class _Engine:
    def __init__(self, layers: int):
        self.layers = layers
        self.requests: dict[str, _Req] = {}

    def update(self, snap: dict) -> None:
        for rid, (ctx, p, o, done, rebuild, phase) in snap.items():
            r = self.requests.get(rid)
            if r is None:
                r = self.requests[rid] = _Req()
                r.id = rid
            r.ctx, r.prompt_len, r.output_len = ctx, p, o
            r.prefill_done, r.rebuild_tokens, r.phase = done, rebuild, phase


@dataclass
class ReplayStats:
    compared: int = 0
    ties: int = 0
    max_rel: float = 0.0
    logits_compared: int = 0
    merges: int = 0
    bad: list = field(default_factory=list)


def replay(trace: list[dict], token_log: list, cfg, weights: dict, prompt_fn,
           tie_tol: float = 2e-2) -> ReplayStats:
    """Oracle replay of `trace` (LiveEngine.batch_trace) against the GPU's
    `token_log` (LiveCudaStep.token_log, same iteration order)."""
    if len(trace) != len(token_log):
        raise AssertionError(f"{len(trace)} traced iterations, {len(token_log)} token records")
    eng = _Engine(cfg.n_layers)
    ora = OracleStep(cfg, weights, prompt_fn)
    ora.attach(eng)
    st = ReplayStats()
    for k_it, (it, (reqs, toks, logits)) in enumerate(zip(trace, token_log)):
        eng.update(it["snap"])
        plan = SimpleNamespace(**it["plan"])
        ora.teacher = {rid: int(t) for rid, t in zip(reqs, toks)}
        ora.begin_iteration(plan)
        n_log = len(ora.logit_log)
        for layer, merges, snap in it["layers"]:
            eng.update(snap)
            items = []
            for rid, outcome in merges:
                if outcome != "inject":
                    lay0, pos = ora.ship[rid][:2]
                    ora.cpu_service(0, [SimpleNamespace(req_id=rid, layer=lay0 + 1,
                                                        ctx_tokens=pos)])
                items.append((SimpleNamespace(req_id=rid, layer=layer), outcome))
            st.merges += len(items)
            ora.layer(layer, items)
        ora.end_iteration(plan)
        emitted = ora.logit_log[n_log:]
        # chain tokens (emitted during layer L) come after the batch rows on
        # the GPU; order the oracle's emissions the same way
        by_rid = {rid: lg for rid, lg in emitted}
        if sorted(by_rid) != sorted(reqs):
            raise AssertionError(f"token rows differ: gpu {sorted(reqs)} oracle {sorted(by_rid)}")
        for i, (rid, tok) in enumerate(zip(reqs, toks)):
            ref = by_rid[rid]
            scale = float(np.abs(ref).max())
            if logits is not None:
                rel = float(np.abs(logits[i] - ref).max() / scale)
                st.max_rel = max(st.max_rel, rel)
                st.logits_compared += 1
            st.compared += 1
            ora_tok = int(np.argmax(ref))
            if int(tok) != ora_tok:
                # the GPU's choice must be a near-tie of the oracle's logits
                gap = float(ref[ora_tok] - ref[int(tok)]) / scale
                if gap <= tie_tol:
                    st.ties += 1
                else:
                    st.bad.append((rid, int(tok), ora_tok, gap, k_it))
        if ora.teacher:
            raise AssertionError(f"GPU tokens without an oracle emission: {ora.teacher}")
    return st
