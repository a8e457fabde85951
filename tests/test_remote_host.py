"""Remote CPU hosts (reference engine.py:329-331, 402-419,
529-560): a request offloaded to host h >= 1 has its KV and its per-layer
work items serviced by a separate `cpu_host` process over TCP.

CPU tests drive the server's wire protocol directly against the numpy
oracle (HELLO / PUT / ATTEND / GET / FREE / BYE, csrc/cpu_remote.cpp).  The
GPU test runs the Appendix-B schedule with the local host full -- as the
reference's own `test_remote_transfer_charged_on_network` does -- so every
offload lands on remote hosts, and compares the served tokens and logits
with the oracle."""

import copy
import socket
import struct

import numpy as np
import pytest

from oracle import llama_ops as O
from paper_2603_12831_b200.models import TRANSFORMERS

HELLO, PUT, ATTEND, GET, FREE, BYE, RESULT, KV, ERR, PUT_ROWS, KV_ROWS = range(1, 12)


def _hdr(op, slot=0, a=0, b=0):
    return struct.pack("<4i", op, slot, a, b)


def _recv(s, n):
    buf = bytearray()
    while len(buf) < n:
        chunk = s.recv(n - len(buf))
        if not chunk:
            raise ConnectionError("server closed the connection")
        buf += chunk
    return bytes(buf)


def _hello(s, cfg):
    dims = np.array([cfg.d_model, cfg.n_layers, cfg.n_q, cfg.n_kv, cfg.head_dim, cfg.ffn,
                     cfg.vocab], np.int32)
    s.sendall(_hdr(HELLO, 0, 2, len(dims)) + dims.tobytes())
    return struct.unpack("<4i", _recv(s, 16))


@pytest.fixture(scope="module")
def host():
    from paper_2603_12831_b200 import cpu_host

    h = cpu_host.spawn(TRANSFORMERS["tiny"], threads=2, max_slots=16)
    yield h
    h.stop()
    assert h.proc.returncode == 0


def test_remote_host_attends_like_the_oracle(host):
    cfg = TRANSFORMERS["tiny"]
    L, nkv, nq, hd = cfg.n_layers, cfg.n_kv, cfg.n_q, cfg.head_dim
    rng = np.random.default_rng(0)
    cap, ctx, slot = 96, 70, 5
    # the replica's host region [layers][2][n_kv][cap][hd]; only ctx tokens travel
    region = O.to_bf16(rng.standard_normal((L, 2, nkv, cap, hd)).astype(np.float32))
    with socket.create_connection((host.addr, host.port)) as s:
        assert _hello(s, cfg)[0] == HELLO
        # a placement: the header, then the rows in two chunks
        rows = O.bf16_bits(region[:, :, :, :ctx]).reshape(L * 2 * nkv, ctx * hd)
        s.sendall(_hdr(PUT, slot, ctx, cap) + _hdr(PUT_ROWS, slot, 0, 3) + rows[:3].tobytes()
                  + _hdr(PUT_ROWS, slot, 3, len(rows) - 3) + rows[3:].tobytes())
        kv = region.copy()
        for step, layer in enumerate((2, 1, 2)):  # two tokens at layer 2, one at layer 1
            c = ctx + (1 if step == 2 else 0)
            q = O.to_bf16(rng.standard_normal((nq, hd)).astype(np.float32))
            k = O.to_bf16(rng.standard_normal((nkv, hd)).astype(np.float32))
            v = O.to_bf16(rng.standard_normal((nkv, hd)).astype(np.float32))
            ship = np.concatenate([q.ravel(), k.ravel(), v.ravel()])
            s.sendall(_hdr(ATTEND, slot, layer, c) + O.bf16_bits(ship).tobytes())
            h = struct.unpack("<4i", _recv(s, 16))
            assert h == (RESULT, slot, layer, c)
            got = O.from_bf16_bits(np.frombuffer(_recv(s, nq * hd * 2), np.uint16)).reshape(nq, hd)
            kv[layer - 1, 0, :, c] = k
            kv[layer - 1, 1, :, c] = v
            K = kv[layer - 1, 0, :, :c + 1].transpose(1, 0, 2)
            V = kv[layer - 1, 1, :, :c + 1].transpose(1, 0, 2)
            ref, _ = O.decode_attention(q, K, V, nkv)
            err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-6)
            assert err < 1.5e-2, (step, err)
        # GET returns the context with the appended tokens (swap-in from the host)
        s.sendall(_hdr(GET, slot, ctx + 2))
        rows, n_rows = {}, L * 2 * nkv
        while len(rows) < n_rows:  # KV_ROWS chunks (slot, first row, rows)
            op, sl, r0, nr = struct.unpack("<4i", _recv(s, 16))
            assert op == KV_ROWS and sl == slot and r0 == len(rows), (op, sl, r0, nr)
            for r in range(r0, r0 + nr):
                rows[r] = np.frombuffer(_recv(s, (ctx + 2) * hd * 2), np.uint16)
        back = np.stack([rows[r] for r in range(n_rows)]).reshape(L, 2, nkv, ctx + 2, hd)
        want = O.bf16_bits(kv[:, :, :, :ctx + 2])
        # layer 1 got one appended token (position ctx); its position ctx+1 is unwritten
        assert np.array_equal(back[:, :, :, :ctx], want[:, :, :, :ctx])
        assert np.array_equal(back[1, :, :, ctx:ctx + 2], want[1, :, :, ctx:ctx + 2])
        assert np.array_equal(back[0, :, :, ctx], want[0, :, :, ctx])
        s.sendall(_hdr(FREE, slot) + _hdr(BYE, 0, 0))


def test_remote_host_rejects_bad_requests(host):
    cfg = TRANSFORMERS["tiny"]
    import dataclasses

    with socket.create_connection((host.addr, host.port)) as s:  # wrong geometry
        h = _hello(s, dataclasses.replace(cfg, n_kv=cfg.n_kv * 2))
        assert h[0] == ERR and h[2] == 1  # HS_E_CONFIG
    with socket.create_connection((host.addr, host.port)) as s:  # item for a slot without KV
        assert _hello(s, cfg)[0] == HELLO
        ship = np.zeros(cfg.qkv_dim, np.uint16)
        s.sendall(_hdr(ATTEND, 3, 1, 0) + ship.tobytes())
        h = struct.unpack("<4i", _recv(s, 16))
        assert h[0] == ERR and h[2] == 2  # HS_E_INTEGRITY


def test_remote_hosts_start_and_stop():
    from paper_2603_12831_b200 import cpu_host

    with cpu_host.RemoteHosts(TRANSFORMERS["tiny"], 2, threads=1, max_slots=4) as rh:
        ports = [h.port for h in rh.hosts]
        assert len(set(ports)) == 2 and all(p > 0 for p in ports)
    assert all(h.proc.returncode == 0 for h in rh.hosts)


def _remote_doc():
    from oracle.scenarios import APPENDIX_B

    doc = copy.deepcopy(APPENDIX_B)
    doc["profiles"]["cluster"]["cpu_hosts"] = 3
    return doc


def test_engine_offloads_to_remote_hosts_when_local_is_full():
    """The schedule the GPU test serves: every offload on a remote host."""
    from paper_2603_12831_b200.engine import Engine
    from paper_2603_12831_b200.scenario import scenario_from_dict

    doc = _remote_doc()
    doc["horizon_s"] = 3.0
    eng = Engine(scenario_from_dict(doc, "remote"))
    eng.kv.host_used[0] = eng.kv.host_capacity
    rep = eng.run()
    hosts = [e["host"] for e in eng.events if e["kind"] == "swap_out_start"]
    assert hosts and all(h >= 1 for h in hosts)
    assert rep.counters["be_tokens_cpu"] > 0 and rep.counters["merges"] > 0


@pytest.mark.gpu
def test_cuda_step_with_remote_hosts_matches_oracle(cuda):
    from oracle.serve_oracle import OracleStep, device_weights, make_weights
    from oracle.tee import TeeStep
    from paper_2603_12831_b200 import cpu_host
    from paper_2603_12831_b200.engine import Engine
    from paper_2603_12831_b200.runtime import CudaStep, RuntimeConfig, prompt_tokens
    from paper_2603_12831_b200.scenario import scenario_from_dict

    cfg = TRANSFORMERS["tiny"]
    w = make_weights(cfg, 0)
    with cpu_host.RemoteHosts(cfg, 2, threads=2, max_slots=64) as rh:
        rt = RuntimeConfig(max_rows=2048, max_slots=64, kv_pages=256, max_pages_per_req=16,
                           max_pos=2048, max_chunks=1024, cpu_threads=2, host_kv_bytes=64 << 20)
        rt.remote_hosts = tuple((h.addr, h.port) for h in rh.hosts)
        gpu = CudaStep(cfg, rt, weights=device_weights(w), keep_logits=True)
        ora = OracleStep(cfg, w, lambda rid, n: prompt_tokens(rid, n, cfg.vocab, 0))
        tee = TeeStep(gpu, ora)
        eng = Engine(scenario_from_dict(_remote_doc(), "remote"), step=tee)
        eng.kv.host_used[0] = eng.kv.host_capacity  # local host full: offloads go remote
        report = eng.run()
        c = report.counters
        stats = [gpu.ctx.remote_stats(h) for h in (1, 2)]
        gpu.ctx.close()
    items = sum(s["items"] for s in stats)
    assert c["swap_out_done"] >= 1 and c["swap_in_done"] >= 1 and c["be_tokens_cpu"] > 0
    assert items > 0 and sum(s["put_bytes"] for s in stats) > 0
    assert sum(s["get_bytes"] for s in stats) > 0  # swap-in fetched the KV back
    assert gpu.remote_colocated == 0
    assert tee.compared == c["tokens_total"] > 0
    assert not tee.bad, tee.bad[:5]
    assert tee.max_rel < 2e-2, tee.max_rel
    print(f"remote items={items} compared={tee.compared} max_rel={tee.max_rel:.2e} {stats}")


@pytest.mark.gpu
@pytest.mark.parametrize("device_merges", [False, True])
def test_live_engine_with_remote_hosts_matches_oracle_replay(cuda, device_merges):
    """The live path (asynchronous pool, device-polled merges) with every
    offloaded request on a remote host: work items relayed from the event /
    the device's work ring, results completed by the relay; the realised
    schedule replayed through the oracle."""
    from oracle.replay import replay
    from paper_2603_12831_b200 import cpu_host
    from paper_2603_12831_b200.live import LiveEngine
    from paper_2603_12831_b200.runtime import LiveCudaStep, RuntimeConfig, prompt_tokens
    from paper_2603_12831_b200.scenario import scenario_from_dict

    from oracle.serve_oracle import device_weights, make_weights

    cfg = TRANSFORMERS["tiny"]
    w = make_weights(cfg, 0)
    dev_w = device_weights(w)
    for attempt in range(3):
        with cpu_host.RemoteHosts(cfg, 2, threads=2, max_slots=64) as rh:
            rt = RuntimeConfig(max_rows=2048, max_slots=64, kv_pages=256, max_pages_per_req=16,
                               max_pos=2048, max_chunks=1024, cpu_threads=2,
                               host_kv_bytes=256 << 20)
            rt.remote_hosts = tuple((h.addr, h.port) for h in rh.hosts)
            step = LiveCudaStep(cfg, rt, weights=dev_w, keep_logits=True,
                                device_merges=device_merges)
            step.trace_tokens = True
            doc = _remote_doc()
            doc["profiles"]["cluster"]["gpu_kv_capacity"] = 1600  # as tests/test_live_parity.py
            eng = LiveEngine(scenario_from_dict(doc, "live_remote"), step=step, batch_trace=True)
            eng.kv.host_used[0] = eng.kv.host_capacity
            n = eng.run_live(horizon_s=30.0)
            step.finish()
            stats = [step.ctx.remote_stats(h) for h in (1, 2)]
            print("host processes:", [h.proc.poll() for h in rh.hosts])
            step.ctx.close()
        if not eng.stalled:
            break
        print("policy wedge, rerun:", n)
    c = eng.counters
    assert not eng.stalled and c["tokens_total"] == 6280, (n, c)
    assert c["swap_out_done"] > 0 and c["be_tokens_cpu"] > 0 and c["merges"] > 0, c
    assert sum(s["items"] for s in stats) > 0 and step.remote_colocated == 0, stats
    st = replay(eng.batch_trace, step.token_log, cfg, w,
                lambda rid, k: prompt_tokens(rid, k, cfg.vocab, 0))
    assert st.merges == c["merges"]
    assert st.compared == c["tokens_total"]
    assert not st.bad, st.bad[:5]
    assert st.max_rel < 2e-2, st.max_rel
    print(f"live remote: iterations={n} tokens={st.compared} merges={st.merges} {stats}")


def test_remote_host_streams_fetches_between_results(host):
    """A fetch (GET) of a long context streams in chunks; an item of another
    slot sent right behind it is answered between the chunks instead of
    after the whole context."""
    cfg = TRANSFORMERS["tiny"]
    L, nkv, nq, hd = cfg.n_layers, cfg.n_kv, cfg.n_q, cfg.head_dim
    rng = np.random.default_rng(1)
    big, small, ctx, cap = 7, 8, 40000, 40100  # 5 MB per row: one row per chunk
    n_rows = L * 2 * nkv
    with socket.create_connection((host.addr, host.port)) as s:
        assert _hello(s, cfg)[0] == HELLO
        region = rng.integers(0, 1 << 14, (n_rows, ctx * hd)).astype(np.uint16)
        s.sendall(_hdr(PUT, big, ctx, cap) + _hdr(PUT_ROWS, big, 0, n_rows) + region.tobytes())
        s.sendall(_hdr(PUT, small, 10, 64) + _hdr(PUT_ROWS, small, 0, n_rows)
                  + np.zeros((n_rows, 10 * hd), np.uint16).tobytes())
        ship = np.zeros(cfg.qkv_dim, np.uint16)
        # the swap-in pattern: the fetch, its FREE right behind it, then an item
        s.sendall(_hdr(GET, big, ctx) + _hdr(FREE, big) + _hdr(ATTEND, small, 1, 10)
                  + ship.tobytes())
        got, order = {}, []
        while len(got) < n_rows or "result" not in order:
            op, sl, a, b = struct.unpack("<4i", _recv(s, 16))
            if op == RESULT:
                assert (sl, a, b) == (small, 1, 10)
                _recv(s, nq * hd * 2)
                order.append("result")
                continue
            assert op == KV_ROWS and sl == big
            for r in range(a, a + b):
                got[r] = np.frombuffer(_recv(s, ctx * hd * 2), np.uint16)
            order.append("rows")
        assert all(np.array_equal(got[r], region[r]) for r in range(n_rows))
        assert order.index("result") < len(order) - 1, order  # not behind the whole context
        s.sendall(_hdr(FREE, small) + _hdr(BYE, 0, 0))
