"""Per-iteration batch planning (the dynamic batching-control policy).

`PlannerMixin._plan_budgeted` produces the BatchPlan + Loads the B200 step
executes.  It restates the reference planner stage by stage
(pkg/src/hybridserve/engine.py:577-850) — eviction under LS KV pressure,
LS decodes, LS chunks, BE chunks under the reserved share while piggyback
work waits, BE decode placement (GPU vs offload), swap-back-in directives,
advisory per-layer piggyback budgets — keeping every accumulation order so
the plans are bit-identical (tests/test_sched_parity.py).
"""

from __future__ import annotations

from collections import deque

from .scheduling import (
    BatchPlan,
    BePlacement,
    Loads,
    SchedulerState,
    be_decode_admit,
    chunk_prefill_budget,
    headroom_baseline_plan,
    max_piggyback_count,
    pairwise_units,
    piggyback_budget,
)
from .workload import ServiceClass

_LS, _BE = ServiceClass.LS, ServiceClass.BE
LS_PROTECT_MARGIN = 256  # tokens BE allocations leave free (engine.py:629)
LS_PREFILL_PRESSURE_CAP = 4096  # engine.py:641-643


class _Acc:
    """Running load accumulators of the batch being planned."""

    __slots__ = ("units", "attn", "reqs", "tokens")

    def __init__(self):
        self.units = 0.0
        self.attn = 0.0
        self.reqs = 0
        self.tokens = 0

    def loads(self) -> Loads:
        return Loads(self.units, self.attn, self.reqs, self.tokens)

    def add_decode(self, ctx: int) -> None:
        self.attn += ctx + 1
        self.reqs += 1
        self.tokens += 1

    def add_chunk(self, done: int, q: int) -> None:
        self.units += pairwise_units(done, q)
        self.tokens += q


class PlannerMixin:
    def _ordered(self, reqs):
        return sorted(reqs, key=lambda r: (r.arrival, r.id))

    def _plan(self) -> BatchPlan:
        if self.scenario.policy == "headroom":
            return self._plan_headroom()
        return self._plan_budgeted()

    def _be_slot_exists(self, req, ls_protect: int, offload_allowed: bool) -> bool:
        """BE prefill start gate: workspace for the whole prompt now, and a
        lifetime home somewhere (engine.py:582-596)."""
        room = self.kv.gpu_free - ls_protect
        if room < req.prompt_len + 1:
            return False
        lifetime = req.prompt_len + req.output_len + 1
        if room >= lifetime:
            return True
        return offload_allowed and any(
            self.kv.host_free(h) >= lifetime for h in range(self.cluster.cpu_hosts))

    # -- stages ------------------------------------------------------------

    def _evict_for_ls(self, ls_decode, ls_prefill, be_prefill, be_resident, offload_allowed):
        pressure = len(ls_decode) + min(sum(r.remaining_prompt for r in ls_prefill),
                                        LS_PREFILL_PRESSURE_CAP)
        if pressure <= self.kv.gpu_free:
            return be_prefill
        expected_free = self.kv.gpu_free
        victims = list(reversed(be_resident)) + [r for r in reversed(be_prefill) if r.kv_held > 0]
        for v in victims:
            if pressure <= expected_free:
                break
            if v.phase == "decode" and offload_allowed and self._start_swap_out(v):
                expected_free += v.kv_held
                be_resident.remove(v)
            else:
                expected_free += v.kv_held
                self._preempt_recompute(v)
                if v in be_resident:
                    be_resident.remove(v)
                    be_prefill = self._ordered(be_prefill + [v])
            self.counters["evictions"] += 1
        return be_prefill

    def _plan_budgeted(self) -> BatchPlan:
        plan = BatchPlan()
        offload_allowed = self.scenario.policy in ("omniserve", "no_admission_control")
        live = self._live()
        ls_decode = self._ordered([r for r in live if r.cls == _LS and r.phase == "decode"
                                   and r.kv_place == "gpu"])
        ls_prefill = self._ordered([r for r in live if r.cls == _LS and r.phase == "prefill"])
        be_prefill = self._ordered([r for r in live if r.cls == _BE and r.phase == "prefill"])
        be_resident = self._ordered([r for r in live if r.cls == _BE and r.phase == "decode"
                                     and r.kv_place == "gpu" and r.swap_state == "none"])
        be_offloaded = self._ordered([r for r in live if r.cls == _BE and r.phase == "decode"
                                      and isinstance(r.kv_place, int)])
        acc = _Acc()
        ls_protect = len(ls_decode) + LS_PROTECT_MARGIN
        ls_reserve = ls_protect + sum(r.output_len - r.tokens_out for r in ls_decode)

        be_prefill = self._evict_for_ls(ls_decode, ls_prefill, be_prefill, be_resident,
                                        offload_allowed)
        for r in list(ls_decode):
            if not self.kv.alloc_gpu(1):
                self.counters["ls_decode_deferrals"] += 1
                continue
            r.kv_held += 1
            acc.add_decode(r.ctx)
            plan.ls_decode.append(r.id)

        piggyback_waiting = bool(self.queues.output or self.pending_injections)
        for r in ls_prefill:
            if self.kv.gpu_free <= 0:
                break
            budget = self.slo.decode_layer_budget_us - self._gamma_us(
                acc.tokens + r.remaining_prompt)
            q = chunk_prefill_budget(r.prefill_done, r.prefill_target, acc.loads(), self.models,
                                     budget)
            q = min(q, self.kv.gpu_free)
            self._audit("chunk_prefill", r.id, float(r.remaining_prompt), budget, q)
            if q <= 0:
                continue
            self._take_chunk(r, q, acc)
            plan.ls_prefill_chunks.append((r.id, q))
        for r in be_prefill:
            if self.kv.gpu_free - ls_protect <= 0:
                break
            if (r.prefill_done == 0 and r.rebuild_tokens == 0
                    and not self._be_slot_exists(r, ls_protect, offload_allowed)):
                continue
            base = (self.slo.reserved_decode_layer_budget_us if piggyback_waiting
                    else self.slo.decode_layer_budget_us)
            budget = base - self._gamma_us(acc.tokens + r.remaining_prompt)
            q = chunk_prefill_budget(r.prefill_done, r.prefill_target, acc.loads(), self.models,
                                     budget)
            q = min(q, self.kv.gpu_free - ls_protect)
            self._audit("chunk_prefill_be", r.id, float(r.remaining_prompt), budget, q)
            if q <= 0:
                continue
            self._take_chunk(r, q, acc)
            plan.be_prefill_chunks.append((r.id, q))

        for r in be_resident:
            d = be_decode_admit(r.ctx, acc.loads(), self.models, self.slo,
                                self.kv.gpu_free + r.kv_held)
            self._audit("be_decode", r.id, d.lhs_us, d.rhs_us, d.placement.value)
            if (d.placement == BePlacement.ON_GPU and self.kv.gpu_free > ls_reserve
                    and self.kv.alloc_gpu(1)):
                r.kv_held += 1
                acc.add_decode(r.ctx)
                plan.be_decode_gpu.append(r.id)
            elif offload_allowed and self._start_swap_out(r):
                plan.be_offload_cpu.append(r.id)

        if offload_allowed:
            self._plan_swap_ins(plan, acc, be_offloaded, ls_reserve)

        ready: dict[int, int] = {}
        for item in self.queues.output:
            ready[item.layer] = ready.get(item.layer, 0) + 1
        if self.pending_injections:
            ready[1] = ready.get(1, 0) + len(self.pending_injections)
        loads = acc.loads()
        if ready:
            plan.piggyback_per_layer = piggyback_budget(
                ready, loads, self.models, self.slo, self.cluster.max_piggyback_per_layer)
        plan.loads = loads
        return plan

    def _take_chunk(self, r, q: int, acc: _Acc) -> None:
        self.kv.alloc_gpu(q)
        r.kv_held += q
        acc.add_chunk(r.prefill_done, q)

    def _plan_swap_ins(self, plan, acc: _Acc, be_offloaded, ls_reserve: int) -> None:
        """Swap-back-in directives; their loads go to shadow accumulators that
        only sequence later directives (engine.py:749-791)."""
        sh_attn, sh_reqs, sh_tokens = acc.attn, acc.reqs, acc.tokens
        for r in be_offloaded:
            if r.swap_state != "in_pending":
                continue
            d = be_decode_admit(r.ctx, Loads(acc.units, sh_attn, sh_reqs, sh_tokens), self.models,
                                self.slo, r.ctx)
            if d.placement == BePlacement.ON_GPU:
                sh_attn += r.ctx + 1
                sh_reqs += 1
                sh_tokens += 1
            else:
                self._cancel_swap_in(r)
        for r in be_offloaded:
            if r.swap_state != "none" or r.phase != "decode":
                continue
            d = be_decode_admit(r.ctx, Loads(acc.units, sh_attn, sh_reqs, sh_tokens), self.models,
                                self.slo, self.kv.gpu_free - 1 - ls_reserve)
            if d.placement != BePlacement.ON_GPU or not self.kv.alloc_gpu(r.ctx + 1):
                continue
            r.gpu_reserved = r.ctx + 1
            r.swap_state = "in_pending"
            sh_attn += r.ctx + 1
            sh_reqs += 1
            sh_tokens += 1
            plan.swap_back_in.append(r.id)
            self._log("swap_in_directive", request=r.id)
            if not self.opts.delayed_swap_in or r.chain_state in ("none", "inject"):
                if r.chain_state == "inject":
                    self.pending_injections = deque(
                        i for i in self.pending_injections if i.req_id != r.id)
                    r.chain_state = "none"
                self._start_swap_in(r, self.now)

    def _plan_headroom(self) -> BatchPlan:
        live = self._live()
        state = SchedulerState(
            prefill=[r.view() for r in self._ordered([x for x in live if x.phase == "prefill"])],
            decode=[r.view() for r in self._ordered([x for x in live if x.phase == "decode"])])
        plan = headroom_baseline_plan(state, self.scenario.headroom_frac,
                                      self.cluster.gpu_kv_capacity,
                                      self.opts.headroom_chunk_tokens)
        acc = _Acc()
        kept: set[str] = set()
        for rid in plan.ls_decode + plan.be_decode_gpu:
            r = self.requests[rid]
            if not self.kv.alloc_gpu(1):
                self.counters["ls_decode_deferrals"] += 1
                continue
            r.kv_held += 1
            kept.add(rid)
            acc.add_decode(r.ctx)
        plan.ls_decode = [x for x in plan.ls_decode if x in kept]
        plan.be_decode_gpu = [x for x in plan.be_decode_gpu if x in kept]
        for chunks in (plan.ls_prefill_chunks, plan.be_prefill_chunks):
            kept_chunks = []
            for rid, q in chunks:
                r = self.requests[rid]
                q = min(q, self.kv.gpu_free)
                if q <= 0:
                    continue
                self._take_chunk(r, q, acc)
                kept_chunks.append((rid, q))
            chunks[:] = kept_chunks
        plan.loads = acc.loads()
        return plan

    def _merge_cap(self, loads: Loads) -> int:
        """One piggyback cap per iteration, computed whenever any chain is in
        flight (engine.py:861-877)."""
        in_flight = (bool(self.queues.output) or bool(self.pending_injections)
                     or any(r.chain_state != "none" for r in self.requests.values()
                            if r.phase == "decode" and isinstance(r.kv_place, int)))
        if not in_flight:
            return 0
        return max_piggyback_count(loads, self.models, self.slo,
                                   self.cluster.max_piggyback_per_layer)
