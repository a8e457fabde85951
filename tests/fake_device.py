"""A recording stand-in for `runtime.HsContext` (test infrastructure).

It lets the CPU suite run `LiveEngine` + `LiveCudaStep` — the live serving
host logic the bench measures (asynchronous CPU pool, asynchronous swaps,
pipelined iterations, pacing) — without a GPU: every libhs call is checked
for argument sanity and answered on the wall clock with configurable
latencies.  Tokens are deterministic functions of the request slot.  No
numerics: the GPU parity of the same path is tests/test_live_parity.py.
"""

from __future__ import annotations

import time

import numpy as np


class FakeLib:
    def __init__(self):
        self.launches = 0

    def hs_launch_count(self):
        return self.launches

    def hs_cpu_in_flight(self, _h):
        return 0


class FakeHsContext:
    def __init__(self, model, rt, iter_ms=0.3, cpu_ms=1.0, swap_ms=2.0, rng_seed=0):
        self.model, self.rt = model, rt
        self.iter_s, self.cpu_s, self.swap_s = iter_ms / 1e3, cpu_ms / 1e3, swap_ms / 1e3
        self.rng = np.random.default_rng(rng_seed)
        self.lib = FakeLib()
        self.h = object()
        self.t_anchor = time.perf_counter()
        self.busy_until = 0.0      # device time (wall) the queued work finishes
        self.marks: list[float] = []
        self.iters: list[tuple[float, int]] = []   # (done time, tokens)
        self.cpu: list[tuple[float, int, int]] = []  # (done, slot, layer)
        self.cpu_in_flight = 0
        self.swaps: list[float] = []
        self.host_kv: dict[int, int] = {}
        self.pages: dict[int, int] = {}
        self._rows_logit = 0
        self._merge_last = 0
        self.calls = {"iter_begin": 0, "layer": 0, "cpu_submit": 0, "swap": 0, "merged": 0}
        self.max_rows_seen = 0

    # device queue model: work is serial on one stream
    def _enqueue(self, dur: float) -> float:
        now = time.perf_counter()
        self.busy_until = max(self.busy_until, now) + dur
        return self.busy_until

    def load_weights(self, w):
        pass

    def init_weights(self, seed, std=0.02):
        pass

    def keep_logits(self, on=True):
        pass

    def set_page_table(self, slot, pages):
        assert 0 <= slot < self.rt.max_slots
        assert len(pages) <= self.rt.max_pages_per_req, (slot, len(pages))
        self.pages[slot] = len(pages)

    def host_kv_reserve(self, slot, cap):
        assert 0 <= slot < self.rt.max_slots and cap > 0
        assert slot not in self.host_kv, ("slot already holds a host KV region", slot)
        self.host_kv[slot] = cap

    def host_kv_release(self, slot):
        self.host_kv.pop(slot, None)

    def iter_begin(self, rows_slot, rows_pos, rows_tok, n_decode, chunks, chunk_begin, tiles,
                   logit_rows):
        n = len(rows_slot)
        assert n <= self.rt.max_rows and n_decode <= n
        assert len(chunk_begin) == n_decode + 1
        for s, p in zip(rows_slot, rows_pos):
            assert 0 <= s < self.rt.max_slots and 0 <= p < self.rt.max_pos
            assert p < 64 * self.pages.get(s, 0), ("row beyond its pages", s, p)
        self.max_rows_seen = max(self.max_rows_seen, n)
        self._rows_logit = len(logit_rows)
        self._rows = n
        self.calls["iter_begin"] += 1

    def layer(self, layer, carry_slot, carry_pos, merge_slot, restart_idx, restart_pos,
              merge_tag=None):
        assert 1 <= layer <= self.model.n_layers
        for s in list(carry_slot) + list(merge_slot):
            assert 0 <= s < self.rt.max_slots
        for s in merge_slot:
            assert s in self.host_kv, ("merge of a request without host KV", s)
        assert merge_tag is None or len(merge_tag) == len(merge_slot)
        if layer == self.model.n_layers:
            self._merge_last = len(merge_slot)
        self.calls["layer"] += 1
        self.calls["merged"] += len(merge_slot) + len(carry_slot)
        self.lib.launches += 9
        self._enqueue(self.iter_s / self.model.n_layers)

    def mark(self) -> int:
        self.marks.append(self.busy_until)
        return len(self.marks) - 1

    def wait_mark(self, mark_id):
        t = self.marks[mark_id]
        while time.perf_counter() < t:
            time.sleep(1e-5)

    def sync(self):
        while time.perf_counter() < self.busy_until:
            time.sleep(1e-5)

    def anchor(self):
        self.t_anchor = time.perf_counter()

    def iter_end_async(self) -> int:
        self.iters.append((self.busy_until, self._rows_logit + self._merge_last))
        self._merge_last = 0
        return len(self.iters) - 1

    # synchronous (replay) entry points
    def iter_end(self):
        n = self._rows_logit + self._merge_last
        self._merge_last = 0
        self.calls["iter_end"] = self.calls.get("iter_end", 0) + 1
        return np.arange(n, dtype=np.int32) % max(self.model.vocab, 1)

    def cpu_attend(self, slots, layers, ctxs):
        for s, l, c in zip(slots, layers, ctxs):
            assert s in self.host_kv and 1 <= l <= self.model.n_layers
            assert 0 < c + 1 <= self.host_kv[s], ("ctx beyond the host reservation", s, c)
        self.calls["cpu_attend"] = self.calls.get("cpu_attend", 0) + len(slots)

    def swap_out(self, slot, tokens):
        assert slot in self.host_kv and 0 < tokens <= self.host_kv[slot]
        self.calls["swap"] += 1

    def swap_in(self, slot, tokens):
        assert slot in self.host_kv and tokens > 0
        assert tokens <= 64 * self.pages.get(slot, 0), ("swap-in beyond the slot's pages", slot)
        self.calls["swap"] += 1

    def iter_poll(self, ticket):
        done, n = self.iters[ticket]
        if time.perf_counter() < done:
            return None
        toks = np.arange(n, dtype=np.int32) % max(self.model.vocab, 1)
        return toks, (done - self.t_anchor) * 1e3

    def iter_logits(self, ticket, rows):
        return np.zeros((rows, self.model.vocab), np.float32)

    def cpu_submit(self, slots, layers, ctxs):
        self.calls["cpu_submit"] += 1
        for s, l, c in zip(slots, layers, ctxs):
            assert s in self.host_kv, ("CPU item without host KV", s)
            assert 1 <= l <= self.model.n_layers
            assert 0 < c + 1 <= self.host_kv[s], ("ctx beyond the host reservation", s, c)
            jitter = self.rng.uniform(0.5, 1.5)
            # the item starts once the ship layer has run on the device
            self.cpu.append((self.busy_until + self.cpu_s * jitter, int(s), int(l)))
            self.cpu_in_flight += 1

    def cpu_poll(self, max_items=4096):
        now = time.perf_counter()
        done = sorted([c for c in self.cpu if c[0] <= now])[:max_items]
        self.cpu = [c for c in self.cpu if c not in done]
        self.cpu_in_flight -= len(done)
        return (np.array([d[1] for d in done], np.int32), np.array([d[2] for d in done], np.int32))

    def cpu_busy_seconds(self):
        return 0.0

    def swap_async(self, slot, tokens, out):
        assert 0 <= slot < self.rt.max_slots and tokens > 0
        if out:
            assert slot in self.host_kv
        self.calls["swap"] += 1
        self.swaps.append(max(self.busy_until, time.perf_counter()) + self.swap_s)
        return len(self.swaps) - 1

    def swap_done(self, ticket) -> bool:
        return time.perf_counter() >= self.swaps[ticket]

    def timer(self):
        return 0

    def elapsed_ms(self, a, b):
        return 0.0

    def close(self):
        pass


class FakePgContext(FakeHsContext):
    """FakeHsContext with device-polled merges: a Python model of the
    controller kernel of csrc/piggyback.cu (FIFO head-run from completion
    times, layer-1 injections, carries, restarts, stop flags, decision log)
    executed when each layer is launched."""

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        self.pg_on = False
        self.fifo: list[list[int]] = []      # [slot, layer, ctx, ready_time]
        self.inj: list[int] = []
        self.slot_ctx: dict[int, int] = {}
        self.slot_left: dict[int, int] = {}
        self.slot_stop: dict[int, int] = {}
        self.prev: list[int] = []
        self.cap = 0
        self.bounds: list[int] = []
        self.inj_bound = 0
        self.logs: dict[int, list] = {}
        self._log: list = []
        self._n_logit = 0
        self.merged_total = 0
        self.bound_binding = 0

    def pg_enable(self, on=True):
        self.pg_on = bool(on)

    def pg_inject(self, slots, ctxs, lefts):
        for s, c, l_ in zip(slots, ctxs, lefts):
            assert l_ >= 1 and s in self.host_kv and c + l_ <= self.host_kv[s]
            self.inj.append(int(s))
            self.slot_ctx[int(s)] = int(c)
            self.slot_left[int(s)] = int(l_)
            self.slot_stop[int(s)] = 0

    def pg_stop(self, slots, flags):
        for s, f in zip(slots, flags):
            self.slot_stop[int(s)] = int(f)

    def pg_iter(self, cap, bounds, inject_bound):
        self.cap, self.bounds, self.inj_bound = cap, [min(b, cap) for b in bounds], min(inject_bound, cap)
        self._log = []

    def iter_begin(self, *a, **kw):
        super().iter_begin(*a, **kw)
        self._n_logit = self._rows_logit

    def layer(self, layer, carry_slot, carry_pos, merge_slot, restart_idx, restart_pos,
              merge_tag=None):
        if not self.pg_on:
            return super().layer(layer, carry_slot, carry_pos, merge_slot, restart_idx,
                                 restart_pos, merge_tag)
        L = self.model.n_layers
        now = time.perf_counter()
        m_max = self.bounds[layer - 1]
        c_max = self.inj_bound if layer == 1 else self.bounds[layer - 2]
        k = 0
        while k < min(self.cap, m_max) and k < len(self.fifo):
            e = self.fifo[k]
            if e[1] != layer or e[3] > now:
                break
            k += 1
        # the host's launch bound must never be what stops the head-run
        ku = 0
        while ku < min(self.cap, len(self.fifo)) and self.fifo[ku][1] == layer and self.fifo[ku][3] <= now:
            ku += 1
        self.bound_binding += ku > k
        taken, self.fifo = self.fifo[:k], self.fifo[k:]
        n_inj = min(len(self.inj), self.cap - k, c_max) if layer == 1 else 0
        inj, self.inj = self.inj[:n_inj], self.inj[n_inj:]
        carries = inj if layer == 1 else self.prev[:c_max]
        ship_t = self._enqueue(self.iter_s / L)
        for s in carries:
            self._push_item(s, layer, ship_t)
        recs = []
        restarts = 0
        if layer < L:
            self.prev = [e[0] for e in taken]
            recs = [(e[0], 0) for e in taken]
        else:
            self.prev = []
            for e in taken:
                s = e[0]
                self.slot_left[s] -= 1
                self.slot_ctx[s] += 1
                if self.slot_left[s] > 0 and not self.slot_stop.get(s, 0):
                    self._push_item(s, 1, ship_t)
                    recs.append((s, 2))
                    restarts += 1
                else:
                    recs.append((s, 4))
            self._merge_last = m_max
        recs += [(s, 1) for s in inj]
        self.merged_total += len(taken)
        self._log.append(recs)
        self.calls["layer"] += 1
        self.lib.launches += 10

    def _push_item(self, s, layer, ship_t):
        """A shipped work item: FIFO entry + its CPU completion time."""
        ready = ship_t + self.cpu_s * self.rng.uniform(0.5, 1.5)
        assert s in self.host_kv and self.slot_ctx[s] + 1 <= self.host_kv[s]
        self.fifo.append([s, layer, self.slot_ctx[s], ready])
        self.cpu.append((ready, s, layer))
        self.cpu_in_flight += 1

    def iter_end_async(self):
        t = super().iter_end_async()
        self.logs[t] = self._log
        return t

    def pg_log(self, ticket):
        return self.logs.pop(ticket)
