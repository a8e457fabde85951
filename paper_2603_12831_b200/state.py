"""Runtime bookkeeping of the serving engine: request state, the residual
store, CPU queues and token-granular KV accounting.

Semantics follow the reference engine (pkg/src/hybridserve/engine.py:68-247);
on the real path the *data* behind these records lives in libhs (device
residual rows indexed by request slot, paged KV, pinned piggyback mailboxes)
while these host records keep the integrity checks and the scheduler view.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass
from typing import Optional

from .errors import IntegrityFault
from .scheduling import RequestPhase, RequestView
from .workload import RequestSpec


class SimRequest:
    """Live state of one request (reference engine.py:68-130)."""

    __slots__ = (
        "id", "cls", "prompt_len", "output_len", "arrival", "admitted", "phase", "prefill_done",
        "tokens_out", "token_times", "first_token_time", "completion", "kv_place", "kv_held",
        "gpu_reserved", "swap_reserved", "chain_state", "chain_layer", "swap_state", "swap_dest",
        "rebuild_tokens", "placement_log",
    )

    def __init__(self, spec: RequestSpec):
        self.id = spec.id
        self.cls = spec.cls
        self.prompt_len = spec.prompt_len
        self.output_len = spec.output_len
        self.arrival = spec.arrival_time
        self.admitted = False
        self.phase = "queued"  # queued | prefill | decode | done | rejected
        self.prefill_done = 0
        self.tokens_out = 0
        self.token_times: list[float] = []
        self.first_token_time: Optional[float] = None
        self.completion: Optional[float] = None
        self.kv_place: Optional[object] = None  # "gpu" or a host index
        self.kv_held = 0
        self.gpu_reserved = 0
        self.swap_reserved = 0
        self.chain_state = "none"  # none | inject | input | output
        self.chain_layer = 0
        self.swap_state = "none"  # none | out | in_pending | in_transfer | in_done
        self.swap_dest: Optional[int] = None
        self.rebuild_tokens = 0
        self.placement_log: list[tuple[float, str]] = []

    @property
    def ctx(self) -> int:
        """KV tokens of the context, excluding the token being generated."""
        if self.phase == "prefill":
            return self.prefill_done
        return self.prompt_len + max(0, self.tokens_out - 1)

    @property
    def prefill_target(self) -> int:
        return self.prompt_len + self.rebuild_tokens

    @property
    def remaining_prompt(self) -> int:
        return self.prefill_target - self.prefill_done

    def view(self) -> RequestView:
        in_prefill = self.phase == "prefill"
        return RequestView(
            id=self.id, cls=self.cls, prompt_len=self.prefill_target,
            done_tokens=self.prefill_done if in_prefill else self.ctx,
            arrival_time=self.arrival,
            phase=RequestPhase.PREFILL if in_prefill else RequestPhase.DECODE,
        )


class ResidualStore:
    """Skip-connection rows of offloaded chains keyed by (request, layer);
    written once, read once (reference engine.py:133-161).  The optional
    fault drops exactly one write to exercise IntegrityFault detection."""

    def __init__(self, fault: Optional[tuple[str, int]] = None):
        self._held: dict[tuple[str, int], int] = {}
        self._fault = fault
        self.puts = 0
        self.gets = 0

    def put(self, req_id: str, layer: int, size: int = 1) -> bool:
        key = (req_id, layer)
        if self._fault == key:
            self._fault = None
            return False  # dropped write
        if key in self._held:
            raise IntegrityFault(f"residual already stored for {key}", req_id, layer)
        self._held[key] = size
        self.puts += 1
        return True

    def get(self, req_id: str, layer: int) -> int:
        key = (req_id, layer)
        if key not in self._held:
            raise IntegrityFault(f"residual missing for {key}", req_id, layer)
        self.gets += 1
        return self._held.pop(key)

    def outstanding(self, req_id: str) -> int:
        return sum(1 for (r, _) in self._held if r == req_id)


@dataclass
class WorkItem:
    req_id: str
    layer: int
    ctx_tokens: int
    enq_seq: int
    enq_time: float


@dataclass
class ResultItem:
    req_id: str
    layer: int
    ready_time: float
    enq_seq: int


class CpuQueues:
    """Per-host input FIFOs + the single output FIFO drained by merges."""

    def __init__(self, n_hosts: int):
        self.input: list[deque[WorkItem]] = [deque() for _ in range(n_hosts)]
        self.output: deque[ResultItem] = deque()
        self.input_enq = self.input_deq = self.output_enq = self.output_deq = 0


class KvManager:
    """Token-granular KV accounting for the GPU cache and each CPU host."""

    def __init__(self, gpu_capacity: int, host_capacity: int, n_hosts: int):
        self.gpu_capacity = gpu_capacity
        self.gpu_used = 0
        self.host_capacity = host_capacity
        self.host_used = [0] * n_hosts

    @property
    def gpu_free(self) -> int:
        return self.gpu_capacity - self.gpu_used

    def alloc_gpu(self, tokens: int) -> bool:
        if tokens > self.gpu_free:
            return False
        self.gpu_used += tokens
        return True

    def free_gpu(self, tokens: int) -> None:
        self.gpu_used -= tokens
        if self.gpu_used < 0:
            raise IntegrityFault("GPU KV accounting went negative")

    def host_free(self, host: int) -> int:
        return self.host_capacity - self.host_used[host]

    def alloc_host(self, host: int, tokens: int) -> bool:
        if tokens > self.host_free(host):
            return False
        self.host_used[host] += tokens
        return True

    def free_host(self, host: int, tokens: int) -> None:
        self.host_used[host] -= tokens
        if self.host_used[host] < 0:
            raise IntegrityFault("CPU KV accounting went negative")


@dataclass
class CpuHost:
    id: int
    speed: float
    busy: bool = False


@dataclass
class IterationState:
    plan: object
    merge_cap: int
    start: float
    layer: int
    merges_total: int
    merge_layers: dict[int, int]
