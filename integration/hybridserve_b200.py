"""The integration a `hybridserve` maintainer adds to the reference package
(INTEGRATION.md): `B200Engine` subclasses the reference's own
`hybridserve.engine.Engine` and turns the cost it charges into real work on
the B200 through libhs's C ABI, at the reference's hook sites:

  _start_iteration  (engine.py:879-900)  -> hs_iter_begin  (the BatchPlan rows)
  _run_layer        (engine.py:921-950)  -> hs_layer       (carry / merge / restart rows)
  _process_merge    (engine.py:991-1022) -> the layer's merged rows and their outcome
  _commit_iteration (engine.py:1024-1047)-> hs_iter_end    (greedy tokens)
  _maybe_start_host (engine.py:529-544)  -> hs_cpu_attend  (host attention of the items)
  _finish_swap_out / _maybe_resume_on_gpu / _preempt_recompute / _complete
                    (engine.py:383-508)  -> host KV, swaps, page and slot release

The reference's event loop, scheduler, queues, residual store and request
API run unchanged; this module only observes them and issues the device
work.  The row bookkeeping (slots, 64-token pages, split-K decode chunks,
prefill tiles, completion tags) is libhs's Python binding,
`paper_2603_12831_b200.runtime.CudaStep`, which a maintainer vendors next to
`libhs.so`.  Everything crosses the boundary as plain int32 arrays and
pointers (include/hs.h).

Usage (with the reference importable as `hybridserve`):

    from integration.hybridserve_b200 import B200Engine
    report = B200Engine(scenario, model="tiny").run()
    report.counters, engine.device.generated   # tokens per request
"""

from __future__ import annotations

from typing import Optional

from paper_2603_12831_b200.engine import (
    MERGE_CHAIN,
    MERGE_INJECT,
    MERGE_TOKEN_END,
    MERGE_TOKEN_NEXT,
)
from paper_2603_12831_b200.models import get_transformer
from paper_2603_12831_b200.runtime import CudaStep, RuntimeConfig


def engine_class(base):
    """B200Engine over `base` (the reference's hybridserve.engine.Engine, or
    any class with the same hook sites)."""

    class B200Engine(base):
        def __init__(self, scenario, model: str = "tiny", rt: Optional[RuntimeConfig] = None,
                     weights: Optional[dict] = None, device=None, **kw):
            super().__init__(scenario, **kw)
            cfg = get_transformer(model)
            # libhs context + row bookkeeping (CudaStep is only the adapter
            # here: the reference engine drives it through the hooks below)
            self.device = device or CudaStep(cfg, rt or RuntimeConfig(), weights=weights)
            self.device.attach(self)
            self._merges: list = []

        # -- iteration / layer ------------------------------------------------
        def _start_iteration(self, plan) -> None:        # engine.py:879
            self._plan_rows = plan
            self._began = False
            super()._start_iteration(plan)

        def _run_layer(self) -> None:                    # engine.py:921
            it = self._iter
            if it.layer == 1 and not self._began:
                self.device.begin_iteration(it.plan)   # hs_iter_begin
                self._began = True
            self._merges = []
            super()._run_layer()                       # consumes merges, charges time
            self.device.layer(it.layer, self._merges)  # hs_layer

        def _process_merge(self, item, layer, qkv_done, layer_end):  # engine.py:991
            req = self.requests[item.req_id]
            injected = req.chain_state == "inject"
            out = super()._process_merge(item, layer, qkv_done, layer_end)
            if injected:
                outcome = MERGE_INJECT
            elif layer < self.layers:
                outcome = MERGE_CHAIN
            else:  # the chain continued with its next token iff it re-entered QKV(1)
                outcome = MERGE_TOKEN_NEXT if req.chain_state == "input" else MERGE_TOKEN_END
            self._merges.append((item, outcome))
            return out

        def _commit_iteration(self, plan) -> None:       # engine.py:1024
            self.device.end_iteration(plan)            # hs_iter_end: greedy tokens
            super()._commit_iteration(plan)

        # -- CPU service -------------------------------------------------------
        def _maybe_start_host(self, host_id: int) -> None:  # engine.py:529
            host = self.hosts[host_id]
            items = [] if host.busy else list(self.queues.input[host_id])
            super()._maybe_start_host(host_id)
            if items and self.hosts[host_id].busy:
                self.device.cpu_service(host_id, items)  # hs_cpu_attend

        # -- KV placement ------------------------------------------------------
        def _finish_swap_out(self, req) -> None:         # engine.py:437
            self.device.swap_out_done(req)             # hs_host_kv_reserve + hs_swap_out
            super()._finish_swap_out(req)

        def _maybe_resume_on_gpu(self, req) -> None:     # engine.py:478
            was = req.kv_place
            super()._maybe_resume_on_gpu(req)
            if was != "gpu" and req.kv_place == "gpu":
                self.device.resumed_on_gpu(req)        # hs_swap_in + hs_host_kv_release

        def _preempt_recompute(self, req) -> None:       # engine.py:499
            super()._preempt_recompute(req)
            self.device.preempted(req)

        def _complete(self, req, time: float) -> None:   # engine.py:383
            super()._complete(req, time)
            self.device.released(req)

        def run(self, *a, **kw):
            rep = super().run(*a, **kw)
            self.device.finish()
            return rep

    return B200Engine


def reference_engine():
    """B200Engine over the unmodified reference (hybridserve on sys.path)."""
    from hybridserve.engine import Engine

    return engine_class(Engine)
