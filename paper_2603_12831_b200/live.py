"""Live serving: the engine on the wall clock with real asynchronous work.

`LiveEngine` keeps every planning rule and state transition of `Engine`
(and therefore of the reference, pkg/src/hybridserve/engine.py) and changes
only where time comes from:

* iterations run on the B200 (`LiveCudaStep`); layer l is launched once the
  GPU is at most one layer behind, so the merges consumed at its start are
  the results that have *really* arrived (the reference's FIFO head-run
  semantics, engine.py:902-919, evaluated at launch time);
* work items are submitted to the CPU-attention pool behind a CUDA event of
  the layer that shipped their q/k/v, and completions enter the output FIFO
  in completion order (engine.py:512-560);
* KV swaps run on the copy stream; a swap-in starts once the request's chain
  is idle so every token's KV is on the host (engine.py:456-497);
* token times are CUDA-synchronised wall-clock stamps, so LS TPOT
  attainment and BE tokens/s are measured, not charged.

The virtual-time call sites are rerouted through `_push`, so the base-class
code paths are reused unchanged.
"""

from __future__ import annotations

import time
from collections import deque
from typing import Callable, Optional

from .engine import (
    EV_LAYER_DONE,
    EV_RESULT,
    EV_SERVICE_DONE,
    EV_SWAP_DONE,
    EV_WORKITEM,
    MERGE_TOKEN_END,
    MERGE_TOKEN_NEXT,
    Engine,
)
from .state import IterationState, ResultItem, SimRequest, WorkItem
from .workload import build_requests


class LiveEngine(Engine):
    def __init__(self, scenario, models=None, step=None, pace_layers: int = 1,
                 pace_tail: int = 0, batch_trace: bool = False):
        super().__init__(scenario, models=models, step=step)
        # device-polled merges (step.device_merges): the GPU takes every merge
        # decision; the engine replays the bookkeeping from each finished
        # iteration's decision log, in the device's order
        self.device_merges = bool(getattr(step, "device_merges", False))
        self._pg_inj: deque = deque()        # injections handed to the device, not yet taken
        self._pg_stop: dict[str, bool] = {}  # stop flag last sent per chain
        self._pg_enq: list = []              # work items enqueued by the merge being replayed
        self._pg_bucket: list = []           # chain items the next layer ships
        # realised batch composition, per iteration: the plan's rows, every
        # layer's merges with their outcomes, and the request state each call
        # saw (the replay input of the oracle; cf. the reference's decision
        # audit and module traces, engine.py:305-319, 975-980)
        self.batch_trace: Optional[list[dict]] = [] if batch_trace else None
        self.t0 = time.perf_counter()
        self.pace_layers = pace_layers
        # the last `pace_tail` layers of an iteration are launched without
        # waiting for the GPU, so the queue holds enough work to cover the
        # host's planning of the next iteration (merge decisions of those
        # layers are made that much earlier)
        self.pace_tail = pace_tail
        self._unshipped: dict[str, object] = {}   # WorkItems awaiting their ship launch
        self._submitted: dict[str, object] = {}   # WorkItems in the CPU pool
        # results enter the output FIFO in submission order (a reorder
        # buffer): the reference services a host queue as one batch whose
        # results arrive together in item order (engine.py:546-554), which the
        # FIFO head-run merge rule (engine.py:902-919) relies on
        self._order: deque = deque()
        self._finished: set[str] = set()
        self._pg_done = self._pg_merged = 0  # device mode: CPU completions polled / merged
        self._swaps: dict[int, tuple[str, str]] = {}
        self._swapin_wait: set[str] = set()
        self._collect: Optional[list] = None  # tokens emitted by the iteration being launched
        self._dirty = True
        self.iteration_log: list[dict] = []
        self._last_done = None
        # host-time accounting (seconds): planning, layer issue, waiting on
        # the GPU in pace(); the bench reports it to tell host- from GPU-bound
        self.host_s = {"plan": 0.0, "issue": 0.0, "pace_wait": 0.0}
        self.stalled = False

    def clock(self) -> float:
        return time.perf_counter() - self.t0

    # -- rerouted virtual-time actions -----------------------------------------

    def _push(self, t: float, kind: str, payload) -> None:
        if kind == EV_WORKITEM:
            if self.device_merges:
                self._pg_enq.append(payload)
                return
            self._unshipped[payload.req_id] = payload
        elif kind == EV_SWAP_DONE:
            rid, direction = payload
            req = self.requests[rid]
            if direction == "out":
                self._swaps[self.step.swap_out_async(req)] = (rid, "out")
            else:
                self._swapin_wait.add(rid)
        elif kind in (EV_LAYER_DONE, EV_SERVICE_DONE, EV_RESULT):
            raise AssertionError(f"{kind} is not scheduled in live mode")
        else:
            super()._push(t, kind, payload)

    def _emit_token(self, req: SimRequest, t: float) -> None:
        super()._emit_token(req, t)
        if self._collect is not None:
            # stamped with the iteration's device completion time once known
            self._collect.append((req, len(req.token_times) - 1))

    def _complete(self, req: SimRequest, t: float) -> None:
        super()._complete(req, t)
        if self._collect is not None:
            self._collect.append((req, -1))

    def _snap(self, rids) -> dict:
        out = {}
        for rid in rids:
            r = self.requests[rid]
            out[rid] = (r.ctx, r.prompt_len, r.output_len, r.prefill_done, r.rebuild_tokens,
                        r.phase)
        return out

    # -- async completions ---------------------------------------------------------

    def _poll_async(self) -> None:
        now = self.clock()
        for rid, layer in self.step.cpu_poll():
            if self.device_merges:
                # a hint that the device has something to merge (the device
                # decides from the completion tags themselves).  Counted, not
                # matched against the host mirror: a completion can be polled
                # before the replay of the iteration that shipped the item
                # reaches the mirror, and a dropped hint would leave the
                # engine idle with a merge waiting on the device.
                self._pg_done += 1
                self._dirty = True
                continue
            self._finished.add(rid)
        while not self.device_merges and self._order and self._order[0].req_id in self._finished:
            item = self._order.popleft()
            rid = item.req_id
            self._finished.discard(rid)
            self._submitted.pop(rid)
            self.now = now
            if self.opts.record_traces:
                self.traces.setdefault(rid, []).append((item.layer, "Attn", "CPU"))
            self._on_result(ResultItem(rid, item.layer, now, item.enq_seq))
            self._dirty = True
        for ticket in [t for t in self._swaps if self.step.swap_done(t)]:
            rid, direction = self._swaps.pop(ticket)
            self.now = now
            req = self.requests[rid]
            if direction == "out":
                self._finish_swap_out(req)
            else:
                self._finish_swap_in(req)
            self._dirty = True
        for rid in list(self._swapin_wait):
            req = self.requests[rid]
            if req.phase == "done" or req.swap_state != "in_transfer":
                self._swapin_wait.discard(rid)
                continue
            if req.chain_state in ("none", "inject"):
                self._swapin_wait.discard(rid)
                self._swaps[self.step.swap_in_async(req)] = (rid, "in")

    def _submit_shipped(self, req_ids) -> None:
        items = [self._unshipped.pop(rid) for rid in req_ids]
        if not items:
            return
        self.step.cpu_submit(items)
        for it in items:
            self._submitted[it.req_id] = it
            self._order.append(it)
            self.queues.input_enq += 1
            self.queues.input_deq += 1
            self._log("workitem_enq", request=it.req_id, layer=it.layer, host=0)

    # -- iterations -------------------------------------------------------------------

    def _live_iteration(self, plan) -> bool:
        cap = self._merge_cap(plan.loads)
        pending = (self.queues.output or self.pending_injections
                   or (self.device_merges and (self._pg_inj or self._pg_done > self._pg_merged)))
        has_work = (plan.ls_decode or plan.ls_prefill_chunks or plan.be_prefill_chunks
                    or plan.be_decode_gpu or (cap > 0 and pending))
        if not has_work:
            return False
        self.gpu_busy = True
        self.counters["iterations"] += 1
        it = IterationState(plan=plan, merge_cap=cap, start=self.now, layer=1, merges_total=0,
                            merge_layers={})
        self._iter = it
        self._collect = []
        trace = None
        if self.batch_trace is not None:
            rows = [r for r in plan.ls_decode + plan.be_decode_gpu] + \
                   [r for r, _ in plan.ls_prefill_chunks + plan.be_prefill_chunks]
            trace = {"plan": {"ls_decode": list(plan.ls_decode),
                              "be_decode_gpu": list(plan.be_decode_gpu),
                              "ls_prefill_chunks": list(plan.ls_prefill_chunks),
                              "be_prefill_chunks": list(plan.be_prefill_chunks)},
                     "snap": self._snap(rows), "layers": []}
            self.batch_trace.append(trace)
        self.step.begin_iteration(plan)
        if self.device_merges:
            self._pg_begin(cap)
        ctx_sum = {"ls_ctx": sum(self.requests[r].ctx for r in plan.ls_decode),
                   "be_gpu_ctx": sum(self.requests[r].ctx for r in plan.be_decode_gpu),
                   "merge_ctx": 0}
        for layer in range(1, self.layers + 1):
            it.layer = layer
            tail = layer > self.layers - self.pace_tail
            t_w = time.perf_counter()
            self.step.pace(self.pace_tail if tail else self.pace_layers)
            t_i = time.perf_counter()
            self.host_s["pace_wait"] += t_i - t_w
            self._poll_async()
            self.now = start = self.clock()
            if self.device_merges:
                self.step.layer(layer, [])
                self.host_s["issue"] += time.perf_counter() - t_i
                continue
            merged = self._consume_merges(layer, cap)
            if merged:
                ctx_sum["merge_ctx"] += sum(self.requests[i.req_id].ctx for i in merged)
                it.merges_total += len(merged)
                it.merge_layers[layer] = len(merged)
                self.counters["merges"] += len(merged)
            outcomes = [(item, self._process_merge(item, layer, start, start))
                        for item in merged]
            if trace is not None:
                trace["layers"].append((layer, [(i.req_id, o) for i, o in outcomes],
                                        self._snap([i.req_id for i in merged])))
            self._submit_shipped(self.step.layer(layer, outcomes))
            self.host_s["issue"] += time.perf_counter() - t_i
            if self.opts.record_layer_times:
                self.layer_start_log.append((it.start, layer, start))
        # Pipelined: queue the token readback and commit now; the host plans
        # the next iteration while this one runs.  Token times are patched to
        # the iteration's device completion time when it is polled.
        rec = {"start": it.start, "decodes": len(plan.ls_decode) + len(plan.be_decode_gpu),
               "ls_decodes": len(plan.ls_decode), "be_gpu_decodes": len(plan.be_decode_gpu),
               "chunk_tokens": sum(q for _, q in plan.ls_prefill_chunks + plan.be_prefill_chunks),
               "be_chunk_tokens": sum(q for _, q in plan.be_prefill_chunks),
               "merges": it.merges_total, "batch_tokens": plan.loads.batch_tokens,
               "marks": self._collect, **ctx_sum}
        if self.device_merges:
            rec["trace"] = trace
        self.step.end_iteration(plan, payload=rec)
        self._iter = None
        self.gpu_busy = False
        self.now = self.clock()
        self._commit_iteration(plan)
        self._collect = None
        rec["chain_tokens"] = sum(1 for r, i in rec["marks"] if i >= 0 and r.cls.value == "BE")
        self.iteration_log.append(rec)
        self._dirty = True
        self._resolve_iterations()
        return True

    def _resolve_iterations(self, block: bool = False) -> None:
        for rec, t_done, _ in self.step.poll_iterations(block=block):
            if self.device_merges:
                self._pg_replay(rec, t_done)
            for req, idx in rec.pop("marks"):
                if idx < 0:
                    req.completion = t_done
                    continue
                req.token_times[idx] = t_done
                if idx == 0:
                    req.first_token_time = t_done
            rec["end"] = t_done
            rec["device_ms"] = (t_done - self._last_done) * 1e3 if self._last_done else None
            self._last_done = t_done

    # -- device-polled merges ----------------------------------------------------------

    def _runnable(self) -> bool:
        if self.device_merges and (self._pg_inj or self._pg_done > self._pg_merged):
            return True
        return super()._runnable()

    def _enqueue_workitem(self, req: SimRequest, layer: int, time_: float) -> None:
        if not self.device_merges:
            return super()._enqueue_workitem(req, layer, time_)
        # the device ships the item; a swap-in directive takes effect at the
        # chain's next token boundary on the device (the stop flag), not at
        # the ship of its last layer (engine.py:319-320)
        item = WorkItem(req.id, layer, req.ctx, next(self._seq), time_)
        req.chain_state = "input"
        req.chain_layer = layer
        self._pg_enq.append(item)

    def _pg_begin(self, cap: int) -> None:
        """Hand new chains and stop-flag changes to the device, then this
        iteration's cap and launch bounds."""
        inj = []
        while self.pending_injections:
            item = self.pending_injections.popleft()
            r = self.requests[item.req_id]
            inj.append((r.id, r.ctx, r.output_len - r.tokens_out))
            r.chain_state = "device"  # owned by the device until the log says otherwise
            self._pg_inj.append(item)
        stops = []
        for r in self._live():
            if r.chain_state == "none" or not isinstance(r.kv_place, int):
                continue
            want = r.swap_state in ("in_pending", "in_transfer", "in_done")
            if want != self._pg_stop.get(r.id, False):
                stops.append((r.id, want))
                self._pg_stop[r.id] = want
        bounds = self._pg_bounds(cap, len(self._pg_inj) - len(inj))
        self.step.pg_begin(cap, bounds, min(cap, len(self._pg_inj)), inj, stops)

    def _pg_bounds(self, cap: int, injected_before: int) -> list[int]:
        """Launch bound of each layer's merges: the chains that can be at that
        layer.  A chain advances at most one layer per iteration (its item
        merged at layer x ships at x+1 and needs another iteration), so one
        whose item the host mirror shows at layer m can be merged this
        iteration only at m .. m+lag, lag = iterations launched but not yet
        replayed; a chain injected in one of those (its first item is layer 1)
        at 1 .. lag."""
        L = self.layers
        lag = self.step.iterations_in_flight()
        cnt = [0] * (L + 1)
        for w in self._order:
            for k in range(min(lag, L - 1) + 1):
                cnt[(w.layer - 1 + k) % L + 1] += 1
        for _ in range(injected_before):  # taken at layer 1 of an earlier iteration at best
            for k in range(min(lag, L)):
                cnt[k % L + 1] += 1
        return [min(cap, c) for c in cnt[1:]]

    def _pg_ship(self, items) -> None:
        for w in items:
            self._order.append(w)
            self._submitted[w.req_id] = w
            self.queues.input_enq += 1
            self.queues.input_deq += 1

    def _pg_boundary(self, item: ResultItem, t: float, flags: int) -> str:
        """Layer-L merge as the device took it (engine.py:1005-1021): the
        token is emitted; the chain restarted on the device unless it is done
        or was stopped by a swap-in directive."""
        req = self.requests[item.req_id]
        self.residuals.get(req.id, self.layers)
        req.chain_state = "none"
        req.kv_held += 1
        self._emit_token(req, t)
        self.counters["be_tokens_cpu"] += 1
        if req.tokens_out >= req.output_len:
            if flags & 2:
                raise AssertionError(f"device restarted finished chain {req.id}")
            self._pg_stop.pop(req.id, None)
            self._complete(req, t)
            return MERGE_TOKEN_END
        if flags & 2:
            if req.swap_state == "in_pending":
                # the directive reached the device after this boundary: the
                # chain runs one more token, whose KV the swap-in must also
                # hold on the GPU (the directive reserved ctx + 1 tokens)
                if self.kv.alloc_gpu(1):
                    req.gpu_reserved += 1
                else:
                    self._cancel_swap_in(req)
            self._chain_qkv(req, 1, t)
            return MERGE_TOKEN_NEXT
        self._pg_stop.pop(req.id, None)
        if req.swap_state == "in_pending":
            self._start_swap_in(req, t)
        elif req.swap_state in ("in_transfer", "in_done"):
            self._maybe_resume_on_gpu(req)
        else:  # the directive was withdrawn after the device stopped the chain
            self._inject(req)
        return MERGE_TOKEN_END

    def _pg_replay(self, rec: dict, t: float) -> None:
        """Apply one finished iteration's device decisions (hs_pg_log) to the
        engine state, layer by layer, with the reference's merge semantics;
        items enter the host mirror of the FIFO in the device's ship order."""
        log = rec.pop("pg_log", None)
        trace = rec.pop("trace", None)
        if log is None:
            return
        self.now = t
        L = self.layers
        merges = chain_tokens = merge_ctx = 0
        self._pg_bucket = []
        for layer, recs in enumerate(log, 1):
            self._pg_ship(self._pg_bucket)  # this layer's carries (merged at layer-1)
            self._pg_bucket = []
            same, outcomes = [], []
            for rid, flags in recs:
                req = self.requests[rid]
                if flags & 1:
                    item = self._pg_inj.popleft()
                    if item.req_id != rid:
                        raise AssertionError(f"device injected {rid}, host expected {item.req_id}")
                    self.counters["injections"] += 1
                    req.chain_state = "inject"
                    out = self._process_merge(item, 1, t, t)
                else:
                    w = self._order.popleft()
                    if w.req_id != rid or w.layer != layer:
                        raise AssertionError(f"device merged {rid} at layer {layer}, host FIFO "
                                             f"head is {w.req_id} at layer {w.layer}")
                    self._submitted.pop(rid, None)
                    self._pg_merged += 1
                    self.queues.output_enq += 1
                    self.queues.output_deq += 1
                    req.chain_state = "output"
                    item = ResultItem(rid, layer, t, w.enq_seq)
                    merge_ctx += req.ctx
                    if layer < L:
                        out = self._process_merge(item, layer, t, t)
                    else:
                        out = self._pg_boundary(item, t, flags)
                        chain_tokens += 1
                outcomes.append((rid, out))
                for w in self._pg_enq:
                    (self._pg_bucket if w.layer == layer + 1 else same).append(w)
                self._pg_enq = []
            self._pg_ship(same)  # injections (layer 1) / restarts (layer L)
            if recs:
                merges += len(recs)
                self.counters["merges"] += len(recs)
            if trace is not None:
                trace["layers"].append((layer, outcomes, self._snap([r for r, _ in recs])))
        rec["merges"] = merges
        rec["chain_tokens"] = chain_tokens
        rec["merge_ctx"] = merge_ctx
        self._dirty = True

    # -- main loop ------------------------------------------------------------------------

    def admit_specs(self, specs) -> deque:
        q = deque()
        for spec in specs:
            req = SimRequest(spec)
            self.requests[req.id] = req
            q.append(req)
        return q

    def run_live(self, max_iterations: Optional[int] = None, horizon_s: Optional[float] = None,
                 on_iteration: Optional[Callable[[int], None]] = None,
                 arrivals: Optional[deque] = None, idle_exit: bool = True) -> int:
        """Serve until `max_iterations`, the horizon, or (idle_exit) no work
        is left.  Returns the number of iterations run."""
        if self.step.anchor_wall == 0.0:
            self.step.set_anchor(self.clock())
        if arrivals is None:
            arrivals = self.admit_specs(build_requests(self.scenario.workload,
                                                       horizon_s or self.scenario.horizon_s))
        n = 0
        horizon = horizon_s if horizon_s is not None else float("inf")
        while True:
            self.now = self.clock()
            if self.now > horizon or (max_iterations is not None and n >= max_iterations):
                break
            while arrivals and arrivals[0].arrival <= self.now:
                self._on_arrival(arrivals.popleft())
                self._dirty = True
            self._poll_async()
            self._resolve_iterations()
            if self._dirty and self._runnable():
                self._dirty = False
                t_p = time.perf_counter()
                plan = self._plan()
                self.host_s["plan"] += time.perf_counter() - t_p
                if self._live_iteration(plan):
                    n += 1
                    if on_iteration:
                        on_iteration(n)
                    continue
            quiet = (not arrivals and not self._submitted and not self._swaps
                     and not self._swapin_wait and not self._pg_inj)
            if idle_exit and quiet and not self._runnable():
                break
            if quiet and not self._dirty and not self.step.iterations_in_flight():
                # the last plan had no work and nothing can change the state
                # any more (no arrival, CPU item, swap or iteration pending):
                # the policy is wedged, e.g. GPU KV held by partial prefills
                # (the reference's event loop simply runs out of events here,
                # engine.py:1065-1088)
                self.stalled = True
                break
            time.sleep(2e-5)
        self._resolve_iterations(block=True)
        return n

    def drain(self) -> None:
        self._resolve_iterations(block=True)

    def stall_report(self) -> dict:
        """Diagnostic for a stalled run: every unfinished request's state and
        the KV accounting."""
        reqs = {r.id: (r.phase, r.chain_state, r.swap_state, r.kv_place, r.ctx, r.kv_held,
                       r.gpu_reserved, r.swap_reserved, r.tokens_out, r.output_len)
                for r in self.requests.values() if r.phase not in ("done", "rejected")}
        return {"gpu_used": self.kv.gpu_used, "gpu_capacity": self.kv.gpu_capacity,
                "host_used": list(self.kv.host_used), "pending_injections": len(self.pending_injections),
                "pg": (len(self._pg_inj), len(self._pg_enq), self._pg_done, self._pg_merged,
                       len(self._order)),
                "reqs": reqs}
