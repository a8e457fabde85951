"""Serving engine: the deterministic event loop around the per-layer step.

One GPU stream executes batch plans layer by layer; CPU hosts service BE
attention work items and return results through one FIFO output queue;
transfers and KV swaps run asynchronously and never block the GPU timeline.
Offloaded BE requests advance as piggyback chains: a work item carries one
layer's q/k/v to a CPU host, the result returns through the output queue,
and a later iteration merges it at the same layer's post-attention Dense,
which also runs the next layer's QKV and ships the next work item
(reference pkg/src/hybridserve/engine.py:1-19, §3.2).

Two things are plugged in:

* the *clock*: layer durations come from the device profile
  (`probe_dense`/`probe_attention`, the virtual clock that keeps every
  scheduling decision bit-comparable with the reference), and
* the *step* (`LayerStep`, optional): the executor of the real numerics.
  `runtime.CudaStep` runs each layer on the B200 through libhs with exactly
  the rows the reference's `_run_layer` would charge for (engine.py:921-950),
  mirrors every residual put/get into device memory, ships BE q/k/v to the
  host CPU-attention pool and merges the host results.

Without a step the engine is a drop-in for the reference simulator; with a
step it is a replay of that schedule on real kernels.  `live.LiveEngine`
replaces the virtual clock by the device clock.
"""

from __future__ import annotations

import heapq
import itertools
from collections import deque
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import IntegrityFault, ScenarioError
from .latency import LatencyModelSet, fit_model_set
from .metrics import RequestRecord, SimReport, build_report
from .planner import PlannerMixin
from .profiles import Phase, probe_attention, probe_dense
from .scenario import EngineOptions, Scenario
from .scheduling import SchedulerState, SloConfig, admit_ls
from .state import (
    CpuHost,
    CpuQueues,
    IterationState,
    KvManager,
    ResidualStore,
    ResultItem,
    SimRequest,
    WorkItem,
)
from .workload import ServiceClass, build_requests

US = 1e-6
MODULE_SEQUENCE = ("QKV", "Attn", "Proj", "ResidualAdd", "MLP", "ResidualAdd")
_CALIBRATION_CORES = 24

EV_ARRIVAL = "arrival"
EV_LAYER_DONE = "gpu_layer_done"
EV_WORKITEM = "workitem_arrival"
EV_SERVICE_DONE = "cpu_service_done"
EV_RESULT = "result_arrival"
EV_SWAP_DONE = "swap_done"

# outcome of one piggyback merge, reported to the step
MERGE_INJECT = "inject"          # fresh token enters: QKV(1) only, ship
MERGE_CHAIN = "chain"            # Proj+MLP at l, QKV(l+1), ship
MERGE_TOKEN_NEXT = "token_next"  # Proj+MLP at L, token, QKV(1) of the next token, ship
MERGE_TOKEN_END = "token_end"    # Proj+MLP at L, token; chain stops (done / swap-in)


class LayerStep:
    """Executor interface the engine drives (no-op = pure virtual clock)."""

    def attach(self, engine: "Engine") -> None: ...
    def begin_iteration(self, plan) -> None: ...
    def layer(self, layer: int, merges: list[tuple[ResultItem, str]]) -> None: ...
    def end_iteration(self, plan) -> None: ...
    def cpu_service(self, host_id: int, items: list[WorkItem]) -> None: ...
    def swap_out_done(self, req: SimRequest) -> None: ...
    def resumed_on_gpu(self, req: SimRequest) -> None: ...
    def preempted(self, req: SimRequest) -> None: ...
    def released(self, req: SimRequest) -> None: ...
    def finish(self) -> None: ...


class Engine(PlannerMixin):
    def __init__(self, scenario: Scenario, models: Optional[LatencyModelSet] = None,
                 inject_missing_residual: Optional[tuple[str, int]] = None,
                 step: Optional[LayerStep] = None):
        self.scenario = scenario
        self.opts: EngineOptions = scenario.engine
        self.slo: SloConfig = scenario.slo
        self.cluster = scenario.cluster
        self.gpu = scenario.gpu_profile
        self.cpu = scenario.cpu_profile
        self.layers = scenario.cluster.layers
        if models is None:
            models, _ = fit_model_set(self.gpu, self.cluster, seed=scenario.seed)
        self.models = models
        self.now = 0.0
        self._heap: list = []
        self._seq = itertools.count()
        self.requests: dict[str, SimRequest] = {}
        self.queues = CpuQueues(self.cluster.cpu_hosts)
        self.residuals = ResidualStore(fault=inject_missing_residual)
        self.kv = KvManager(self.cluster.gpu_kv_capacity, self.cluster.cpu_mem_tokens,
                            self.cluster.cpu_hosts)
        speed = self.cluster.cpu_cores_per_host / _CALIBRATION_CORES * self.opts.cpu_speed_factor
        self.hosts = [CpuHost(id=h, speed=speed) for h in range(self.cluster.cpu_hosts)]
        self.pending_injections: deque[ResultItem] = deque()
        self.gpu_busy = False
        self._iter: Optional[IterationState] = None
        self.counters: dict[str, int] = dict.fromkeys(
            ("arrivals", "ls_admitted", "ls_rejected", "iterations", "tokens_total",
             "be_tokens_cpu", "merges", "injections", "swap_out_started", "swap_out_done",
             "swap_in_started", "swap_in_done", "swap_in_cancelled", "evictions",
             "ls_decode_deferrals", "offload_parked", "preemptions"), 0)
        self.events: list[dict] = []
        self.audit: list[dict] = []
        self.traces: dict[str, list[tuple[int, str, str]]] = {}
        self.trace_steps: dict[str, list[str]] = {}
        self.layer_start_log: list[tuple[float, int, float]] = []
        self._noise_rng = (np.random.default_rng(scenario.seed + 1000)
                           if self.opts.apply_noise else None)
        self.step = step or LayerStep()
        self.step.attach(self)

    # -- plumbing -----------------------------------------------------------

    def _push(self, time: float, kind: str, payload) -> None:
        heapq.heappush(self._heap, (time, next(self._seq), kind, payload))

    def _log(self, kind: str, **fields) -> None:
        if self.opts.record_events:
            self.events.append({"t": self.now, "kind": kind, **fields})

    def _audit(self, op: str, request: str, lhs: float, rhs: float, outcome) -> None:
        self.audit.append({"time": self.now, "op": op, "request": request, "lhs_us": lhs,
                           "rhs_us": rhs, "outcome": outcome})

    def _dense_us(self, n: int) -> float:
        return probe_dense(self.gpu, n, self._noise_rng) if n > 0 else 0.0

    def _gamma_us(self, n: int) -> float:
        return self.models.gamma(n)

    def _link_us(self, host: int, tokens: float) -> float:
        alpha, beta = self.cluster.pcie if host == 0 else self.cluster.network
        return alpha + beta * tokens if tokens > 0 else 0.0

    @staticmethod
    def _req_host(req: SimRequest) -> int:
        return req.kv_place if isinstance(req.kv_place, int) else 0

    def _live(self) -> list[SimRequest]:
        return [r for r in self.requests.values() if r.phase in ("prefill", "decode")]

    # -- request lifecycle ----------------------------------------------------

    def _on_arrival(self, req: SimRequest) -> None:
        self.counters["arrivals"] += 1
        if req.prompt_len + 1 > self.cluster.gpu_kv_capacity:
            raise ScenarioError(
                f"request {req.id}: prompt of {req.prompt_len} tokens exceeds the "
                f"GPU KV capacity of {self.cluster.gpu_kv_capacity}")
        if req.cls == ServiceClass.LS:
            if self.scenario.policy in ("omniserve", "gpu_only"):
                d = admit_ls(req.view(), self._ls_state(), self.models, self.slo)
                self._audit("admit_ls", req.id, d.lhs_us, d.rhs_us,
                            "admit" if d.admitted else "reject")
                if not d.admitted:
                    req.phase = "rejected"
                    self.counters["ls_rejected"] += 1
                    self._log("reject", request=req.id)
                    return
            self.counters["ls_admitted"] += 1
        req.admitted = True
        req.phase = "prefill"
        req.kv_place = "gpu"
        req.placement_log.append((self.now, "gpu"))
        self._log("admit", request=req.id)

    def _ls_state(self) -> SchedulerState:
        live = self._live()
        return SchedulerState(
            prefill=[r.view() for r in live if r.cls == ServiceClass.LS and r.phase == "prefill"],
            decode=[r.view() for r in live if r.cls == ServiceClass.LS and r.phase == "decode"])

    def _emit_token(self, req: SimRequest, time: float) -> None:
        req.tokens_out += 1
        req.token_times.append(time)
        if req.first_token_time is None:
            req.first_token_time = time
        self.counters["tokens_total"] += 1

    def _complete(self, req: SimRequest, time: float) -> None:
        req.phase = "done"
        req.completion = time
        if self.residuals.outstanding(req.id):
            raise IntegrityFault(f"request {req.id} completed with residuals outstanding", req.id)
        if req.kv_place == "gpu":
            self.kv.free_gpu(req.kv_held)
        elif isinstance(req.kv_place, int):
            self.kv.free_host(req.kv_place, req.swap_reserved)
        if req.gpu_reserved:
            self.kv.free_gpu(req.gpu_reserved)
        req.kv_held = req.gpu_reserved = req.swap_reserved = 0
        req.swap_state = "none"
        self._log("complete", request=req.id, tokens=req.tokens_out)
        self.step.released(req)

    # -- offload / swaps --------------------------------------------------------

    def _distribute_offload(self, req: SimRequest) -> Optional[int]:
        """Local host while it has room for the lifetime reservation, else the
        least-loaded remote (ties: lowest id)."""
        need = req.kv_held + (req.output_len - req.tokens_out) + 1
        if self.kv.host_free(0) >= need:
            host = 0
        else:
            fits = [h for h in range(1, self.cluster.cpu_hosts) if self.kv.host_free(h) >= need]
            if not fits:
                return None
            host = min(fits, key=lambda h: (self.kv.host_used[h], h))
        self.kv.alloc_host(host, need)
        req.swap_reserved = need
        return host

    def _start_swap_out(self, req: SimRequest) -> bool:
        host = self._distribute_offload(req)
        if host is None:
            self.counters["offload_parked"] += 1
            return False
        req.swap_state = "out"
        req.swap_dest = host
        self.counters["swap_out_started"] += 1
        self._log("swap_out_start", request=req.id, host=host, tokens=req.kv_held)
        self._push(self.now + self._link_us(host, req.kv_held) * US, EV_SWAP_DONE, (req.id, "out"))
        return True

    def _finish_swap_out(self, req: SimRequest) -> None:
        host = req.swap_dest
        self.step.swap_out_done(req)  # copies the pages to host `swap_dest`, then frees them
        req.swap_dest = None
        self.kv.free_gpu(req.kv_held)
        req.kv_place = host
        req.swap_state = "none"
        req.placement_log.append((self.now, f"cpu{host}"))
        self.counters["swap_out_done"] += 1
        self._log("swap_out_done", request=req.id, host=host)
        self._inject(req)

    def _inject(self, req: SimRequest) -> None:
        self.pending_injections.append(ResultItem(req.id, 1, self.now, next(self._seq)))
        req.chain_state = "inject"
        req.chain_layer = 1

    def _start_swap_in(self, req: SimRequest, start_time: float) -> None:
        req.swap_state = "in_transfer"
        tokens = req.kv_held + 1
        host = self._req_host(req)
        self.counters["swap_in_started"] += 1
        self._log("swap_in_start", request=req.id, host=host, tokens=tokens, start=start_time)
        self._push(start_time + self._link_us(host, tokens) * US, EV_SWAP_DONE, (req.id, "in"))

    def _finish_swap_in(self, req: SimRequest) -> None:
        if req.phase == "done":
            return
        self.kv.free_host(self._req_host(req), req.swap_reserved)
        req.swap_reserved = 0
        req.swap_state = "in_done"
        self.counters["swap_in_done"] += 1
        self._log("swap_in_done", request=req.id)
        self._maybe_resume_on_gpu(req)

    def _maybe_resume_on_gpu(self, req: SimRequest) -> None:
        if req.swap_state == "in_done" and req.chain_state == "none" and req.phase == "decode":
            req.kv_place = "gpu"
            req.swap_state = "none"
            req.placement_log.append((self.now, "gpu"))
            held = req.ctx
            if held < req.gpu_reserved:
                self.kv.free_gpu(req.gpu_reserved - held)
            req.kv_held = held
            req.gpu_reserved = 0
            self.step.resumed_on_gpu(req)

    def _cancel_swap_in(self, req: SimRequest) -> None:
        req.swap_state = "none"
        if req.gpu_reserved:
            self.kv.free_gpu(req.gpu_reserved)
            req.gpu_reserved = 0
        self.counters["swap_in_cancelled"] += 1
        self._log("swap_in_cancelled", request=req.id)

    def _preempt_recompute(self, req: SimRequest) -> None:
        self.kv.free_gpu(req.kv_held)
        req.kv_held = 0
        req.phase = "prefill"
        req.rebuild_tokens = max(0, req.tokens_out - 1)
        req.prefill_done = 0
        self.counters["preemptions"] += 1
        self._log("preempt", request=req.id)
        self.step.preempted(req)

    # -- CPU attention service -----------------------------------------------

    def _enqueue_workitem(self, req: SimRequest, layer: int, time: float) -> None:
        item = WorkItem(req.id, layer, req.ctx, next(self._seq), time)
        req.chain_state = "input"
        req.chain_layer = layer
        self._push(time, EV_WORKITEM, item)
        # delayed swap-in: the final layer's q/k/v leaving the GPU means the
        # last token's KV now exists for every layer
        if layer == self.layers and req.swap_state == "in_pending":
            self._start_swap_in(req, time)

    def _on_workitem(self, item: WorkItem) -> None:
        host = self._req_host(self.requests[item.req_id])
        self.queues.input[host].append(item)
        self.queues.input_enq += 1
        self._log("workitem_enq", request=item.req_id, layer=item.layer, host=host)
        self._maybe_start_host(host)

    def _maybe_start_host(self, host_id: int) -> None:
        host = self.hosts[host_id]
        q = self.queues.input[host_id]
        if host.busy or not q:
            return
        items = list(q)
        q.clear()
        self.queues.input_deq += len(items)
        host.busy = True
        load = sum(it.ctx_tokens + 1 for it in items)
        dur = probe_attention(self.cpu, Phase.DECODE, load, len(items), self._noise_rng) / host.speed
        self.step.cpu_service(host_id, items)
        self._log("cpu_service_start", host=host_id, items=len(items))
        self._push(self.now + dur * US, EV_SERVICE_DONE, (host_id, items))

    def _on_service_done(self, host_id: int, items: list[WorkItem]) -> None:
        self.hosts[host_id].busy = False
        for it in items:
            if self.opts.record_traces:
                self.traces.setdefault(it.req_id, []).append((it.layer, "Attn", "CPU"))
            ready = self.now + self._link_us(host_id, self.cluster.result_payload_tokens) * US
            self._push(ready, EV_RESULT, ResultItem(it.req_id, it.layer, ready, it.enq_seq))
        self._log("cpu_service_done", host=host_id, items=len(items))
        self._maybe_start_host(host_id)

    def _on_result(self, item: ResultItem) -> None:
        self.queues.output.append(item)
        self.queues.output_enq += 1
        self.requests[item.req_id].chain_state = "output"
        self._log("result_enq", request=item.req_id, layer=item.layer)

    def _runnable(self) -> bool:
        if self.queues.output or self.pending_injections:
            return True
        for r in self._live():
            if r.phase == "prefill":
                return True
            if r.phase == "decode" and r.kv_place == "gpu" and r.swap_state == "none":
                return True
        return False

    # -- iteration execution ---------------------------------------------------

    def _start_iteration(self, plan) -> None:
        cap = self._merge_cap(plan.loads)
        has_work = (plan.ls_decode or plan.ls_prefill_chunks or plan.be_prefill_chunks
                    or plan.be_decode_gpu
                    or (cap > 0 and (self.queues.output or self.pending_injections)))
        if not has_work:
            return  # directives only
        self.gpu_busy = True
        self.counters["iterations"] += 1
        self._iter = IterationState(plan=plan, merge_cap=cap, start=self.now, layer=1,
                                    merges_total=0, merge_layers={})
        self.step.begin_iteration(plan)
        self._run_layer()

    def _consume_merges(self, layer: int, cap: int) -> list[ResultItem]:
        """FIFO head-run of results for this layer (head-of-line blocking),
        then layer-1 injections, at most `cap` in total."""
        taken: list[ResultItem] = []
        out = self.queues.output
        while len(taken) < cap and out and out[0].layer == layer:
            item = out.popleft()
            self.queues.output_deq += 1
            self._log("merge", request=item.req_id, layer=layer, source="queue")
            taken.append(item)
        if layer == 1:
            while len(taken) < cap and self.pending_injections:
                item = self.pending_injections.popleft()
                self.counters["injections"] += 1
                self._log("merge", request=item.req_id, layer=1, source="inject")
                taken.append(item)
        return taken

    def _layer_charge_us(self, loads, n_merged: int, decodes: int) -> tuple[float, float]:
        """(dense, total) µs of one layer on the virtual clock
        (engine.py:931-945; the accumulation order is part of parity)."""
        n_l = loads.batch_tokens + n_merged
        dense = self._dense_us(n_l)
        dur = dense
        if loads.prefill_units > 0:
            dur += probe_attention(self.gpu, Phase.PREFILL, loads.prefill_units,
                                   rng=self._noise_rng)
        if decodes > 0:
            dur += probe_attention(self.gpu, Phase.DECODE, loads.attn_tokens, decodes,
                                   rng=self._noise_rng)
        dur += self.cluster.merge_cost_per_result * n_merged
        dur += self._gamma_us(n_l)
        return dense, dur

    def _run_layer(self) -> None:
        it = self._iter
        start = self.now
        merged = self._consume_merges(it.layer, it.merge_cap)
        if merged:
            it.merges_total += len(merged)
            it.merge_layers[it.layer] = len(merged)
            self.counters["merges"] += len(merged)
        decodes = len(it.plan.ls_decode) + len(it.plan.be_decode_gpu)
        dense, dur = self._layer_charge_us(it.plan.loads, len(merged), decodes)
        qkv_done = start + self.opts.qkv_time_fraction * dense * US
        layer_end = start + dur * US
        outcomes = [(item, self._process_merge(item, it.layer, qkv_done, layer_end))
                    for item in merged]
        self.step.layer(it.layer, outcomes)
        if self.opts.record_layer_times:
            self.layer_start_log.append((it.start, it.layer, start))
        self._push(layer_end, EV_LAYER_DONE, it.layer)

    def _on_layer_done(self, layer: int) -> None:
        it = self._iter
        if it.layer < self.layers:
            it.layer += 1
            self._run_layer()
            return
        plan = it.plan
        self._log("iteration", start=it.start, end=self.now,
                  decodes=len(plan.ls_decode) + len(plan.be_decode_gpu),
                  chunk_tokens=sum(q for _, q in plan.ls_prefill_chunks + plan.be_prefill_chunks),
                  merges=it.merges_total, prefill_units=plan.loads.prefill_units,
                  attn_tokens=plan.loads.attn_tokens, batch_tokens=plan.loads.batch_tokens,
                  merge_layers={str(k): v for k, v in sorted(it.merge_layers.items())})
        self._iter = None
        self.gpu_busy = False
        self.step.end_iteration(plan)
        self._commit_iteration(plan)

    def _chain_qkv(self, req: SimRequest, layer: int, time: float) -> None:
        """Residual save + QKV of the chain's next layer, then ship q/k/v."""
        self.residuals.put(req.id, layer)
        if self.opts.record_traces:
            self.traces.setdefault(req.id, []).append((layer, "QKV", "GPU"))
        self._enqueue_workitem(
            req, layer, time + self._link_us(self._req_host(req),
                                             self.cluster.qkv_payload_tokens) * US)

    def _process_merge(self, item: ResultItem, layer: int, qkv_done: float,
                       layer_end: float) -> str:
        req = self.requests[item.req_id]
        if req.chain_state == "inject":
            self._chain_qkv(req, 1, qkv_done)
            return MERGE_INJECT
        self.residuals.get(req.id, layer)
        if self.opts.record_traces:
            tr = self.traces.setdefault(req.id, [])
            tr += [(layer, "Proj", "GPU"), (layer, "ResidualAdd", "GPU"), (layer, "MLP", "GPU"),
                   (layer, "ResidualAdd", "GPU")]
        if layer < self.layers:
            self._chain_qkv(req, layer + 1, layer_end)
            return MERGE_CHAIN
        req.chain_state = "none"
        req.kv_held += 1  # written on the host inside the lifetime reservation
        self._emit_token(req, layer_end)
        self.counters["be_tokens_cpu"] += 1
        if self.opts.record_traces:
            self.trace_steps.setdefault(req.id, []).append("token")
        if req.tokens_out >= req.output_len:
            self._complete(req, layer_end)
            return MERGE_TOKEN_END
        if req.swap_state == "in_pending":
            self._start_swap_in(req, layer_end)
            return MERGE_TOKEN_END
        if req.swap_state in ("in_transfer", "in_done"):
            self._maybe_resume_on_gpu(req)
            return MERGE_TOKEN_END
        self._chain_qkv(req, 1, layer_end)
        return MERGE_TOKEN_NEXT

    def _commit_iteration(self, plan) -> None:
        end = self.now
        for rid in plan.ls_decode + plan.be_decode_gpu:
            req = self.requests[rid]
            if req.phase != "decode":
                continue
            self._emit_token(req, end)
            if self.opts.record_traces:
                self._trace_gpu_pass(rid, "token")
            if req.tokens_out >= req.output_len:
                self._complete(req, end)
        for rid, q in plan.ls_prefill_chunks + plan.be_prefill_chunks:
            req = self.requests[rid]
            req.prefill_done += q
            if self.opts.record_traces:
                self._trace_gpu_pass(rid, "chunk")
            if req.prefill_done >= req.prefill_target:
                req.phase = "decode"
                if req.rebuild_tokens:
                    req.rebuild_tokens = 0  # context rebuilt; no new token
                else:
                    self._emit_token(req, end)  # prefill completion emits token 1
                if req.tokens_out >= req.output_len:
                    self._complete(req, end)

    def _trace_gpu_pass(self, rid: str, step: str) -> None:
        tr = self.traces.setdefault(rid, [])
        for layer in range(1, self.layers + 1):
            tr += [(layer, m, "GPU") for m in MODULE_SEQUENCE]
        self.trace_steps.setdefault(rid, []).append(step)

    # -- main loop ---------------------------------------------------------------

    def _dispatch(self, kind: str, payload) -> None:
        if kind == EV_ARRIVAL:
            self._on_arrival(self.requests[payload])
        elif kind == EV_LAYER_DONE:
            self._on_layer_done(payload)
        elif kind == EV_WORKITEM:
            self._on_workitem(payload)
        elif kind == EV_SERVICE_DONE:
            self._on_service_done(*payload)
        elif kind == EV_RESULT:
            self._on_result(payload)
        elif kind == EV_SWAP_DONE:
            rid, direction = payload
            req = self.requests[rid]
            if direction == "out":
                self._finish_swap_out(req)
            else:
                self._finish_swap_in(req)

    def run(self, specs=None) -> SimReport:
        """Simulate to the horizon.  `specs` replaces the scenario's generated
        trace (a replica's share of a routed trace, replicas.route)."""
        horizon = self.scenario.horizon_s
        if specs is None:
            specs = build_requests(self.scenario.workload, horizon)
        for spec in specs:
            req = SimRequest(spec)
            self.requests[req.id] = req
            self._push(spec.arrival_time, EV_ARRIVAL, req.id)
        while self._heap:
            time, _, kind, payload = heapq.heappop(self._heap)
            if time > horizon:
                break
            self.now = time
            self._dispatch(kind, payload)
            if not self.gpu_busy and self._runnable():
                self._start_iteration(self._plan())
        self.step.finish()
        return self.report()

    def report(self) -> SimReport:
        records = sorted((self._record(r) for r in self.requests.values()),
                         key=lambda r: (r.arrival, r.id))
        c = self.counters
        c["input_queue_enq"] = self.queues.input_enq
        c["input_queue_deq"] = self.queues.input_deq
        c["output_queue_enq"] = self.queues.output_enq
        c["output_queue_deq"] = self.queues.output_deq
        c["residual_puts"] = self.residuals.puts
        c["residual_gets"] = self.residuals.gets
        echo = {"name": self.scenario.name, "model": self.scenario.model,
                "policy": self.scenario.policy, "seed": self.scenario.seed,
                "horizon_s": self.scenario.horizon_s}
        return build_report(records, self.slo, self.scenario.horizon_s, c, echo)

    @staticmethod
    def _record(req: SimRequest) -> RequestRecord:
        return RequestRecord(id=req.id, cls=req.cls, prompt_len=req.prompt_len,
                             output_len=req.output_len, arrival=req.arrival,
                             admitted=req.admitted, first_token_time=req.first_token_time,
                             token_times=list(req.token_times), completion=req.completion,
                             prefill_tokens_done=req.prefill_done,
                             placements=list(req.placement_log))


def run(scenario: Scenario, models: Optional[LatencyModelSet] = None,
        inject_missing_residual: Optional[tuple[str, int]] = None,
        step: Optional[LayerStep] = None) -> SimReport:
    return Engine(scenario, models=models, inject_missing_residual=inject_missing_residual,
                  step=step).run()


# -- trace verification ----------------------------------------------------------


def reference_trace(n_passes: int, layers: int) -> list[tuple[int, str]]:
    """Module sequence of a GPU-only execution with n_passes full passes."""
    return [(layer, m) for _ in range(n_passes) for layer in range(1, layers + 1)
            for m in MODULE_SEQUENCE]


@dataclass(frozen=True)
class TraceDivergence:
    request_id: str
    index: int
    expected: Optional[tuple]
    actual: Optional[tuple]


def verify_trace(engine: Engine) -> list[TraceDivergence]:
    """Every BE request's executed module sequence must equal a GPU-only
    pass structure; devices may differ only on Attn entries."""
    out: list[TraceDivergence] = []
    for rid in sorted(engine.traces):
        if engine.requests[rid].cls != ServiceClass.BE:
            continue
        got = engine.traces[rid]
        want = reference_trace(len(engine.trace_steps.get(rid, [])), engine.layers)
        for i in range(max(len(want), len(got))):
            w = want[i] if i < len(want) else None
            g = got[i] if i < len(got) else None
            if w is None or g is None:
                out.append(TraceDivergence(rid, i, w, g))
                continue
            layer, module, device = g
            if (layer, module) != w or (module != "Attn" and device != "GPU"):
                out.append(TraceDivergence(rid, i, w, g))
    return out
