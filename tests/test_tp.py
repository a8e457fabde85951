"""Tensor parallelism (config 4's TP path).

CPU: the Megatron sharding of `tp.shard_weights` reproduces the full layer
(column-parallel QKV / gate-up, row-parallel O / down whose partial sums add
up to the unsharded projection).  GPU: a TP=2 group of two processes (the
deployment shape: one rank per process, exchange buffers shared through CUDA
IPC handles all-gathered over torch.distributed/gloo; here both ranks sit on
the test box's one GPU) serves the Appendix-B schedule; rank 0 runs in
lockstep with the full-model numpy oracle (every token and its logits as for
TP=1) and both ranks must emit identical tokens.
"""

import copy

import numpy as np
import pytest

from oracle import llama_ops as O
from oracle.scenarios import APPENDIX_B
from oracle.serve_oracle import OracleStep, device_weights, make_weights
from oracle.tee import TeeStep
from paper_2603_12831_b200 import tp
from paper_2603_12831_b200.engine import Engine
from paper_2603_12831_b200.errors import ConfigError
from paper_2603_12831_b200.models import TRANSFORMERS
from paper_2603_12831_b200.scenario import scenario_from_dict


def test_shard_config_dims():
    cfg = TRANSFORMERS["tiny"]
    s = tp.shard_config(cfg, 2)
    assert (s.n_q, s.n_kv, s.ffn, s.d_model, s.vocab, s.tp) == (2, 1, 384, 256, 1024, 2)
    assert tp.shard_config(cfg, 1) is cfg
    with pytest.raises(ConfigError):
        tp.shard_config(cfg, 3)


@pytest.mark.parametrize("world", [2])
def test_sharded_layer_equals_full_layer(world):
    cfg = TRANSFORMERS["tiny"]
    w = make_weights(cfg, 0)
    rng = np.random.default_rng(1)
    x = O.to_bf16(rng.standard_normal((5, cfg.d_model)).astype(np.float32))
    hd = cfg.head_dim
    full_qkv = O.gemm(x, w["qkv"][0])
    full_gu = O.gemm(x, w["gate_up"][0])
    attn = O.to_bf16(rng.standard_normal((5, cfg.n_q * hd)).astype(np.float32))
    act = O.to_bf16(rng.standard_normal((5, cfg.ffn)).astype(np.float32))
    o_sum = np.zeros((5, cfg.d_model))
    down_sum = np.zeros((5, cfg.d_model))
    sc = tp.shard_config(cfg, world)
    for r in range(world):
        ws = tp.shard_weights(w, cfg, r, world)
        q = O.gemm(x, ws["qkv"][0])
        nq, nk = sc.n_q * hd, sc.n_kv * hd
        np.testing.assert_array_equal(q[:, :nq], full_qkv[:, r * nq:(r + 1) * nq])
        kb = cfg.n_q * hd
        np.testing.assert_array_equal(q[:, nq:nq + nk], full_qkv[:, kb + r * nk:kb + (r + 1) * nk])
        vb = kb + cfg.n_kv * hd
        np.testing.assert_array_equal(q[:, nq + nk:], full_qkv[:, vb + r * nk:vb + (r + 1) * nk])
        gu = O.gemm(x, ws["gate_up"][0])
        f = sc.ffn
        np.testing.assert_array_equal(gu[:, :f], full_gu[:, r * f:(r + 1) * f])
        np.testing.assert_array_equal(gu[:, f:], full_gu[:, cfg.ffn + r * f:cfg.ffn + (r + 1) * f])
        o_sum += O.gemm(attn[:, r * nq:(r + 1) * nq], ws["o"][0])
        down_sum += O.gemm(act[:, r * f:(r + 1) * f], ws["down"][0])
        assert ws["embed"] is w["embed"] and ws["lm_head"] is w["lm_head"]
    np.testing.assert_allclose(o_sum, O.gemm(attn, w["o"][0]), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(down_sum, O.gemm(act, w["down"][0]), rtol=1e-5, atol=1e-6)


def _ipc_rank(rank, world, port, horizon, q):
    """One TP rank in its own process: shard context, IPC handle exchange
    over gloo, the Appendix-B schedule (rank 0 against the full oracle)."""
    import os

    import torch.distributed as dist

    from paper_2603_12831_b200.runtime import CudaStep, RuntimeConfig, prompt_tokens

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = TRANSFORMERS["tiny"]
        w = make_weights(cfg, 0)
        rt = RuntimeConfig(max_rows=2048, max_slots=64, kv_pages=256, max_pages_per_req=16,
                           max_pos=2048, max_chunks=1024, cpu_threads=2, host_kv_bytes=64 << 20)
        step = CudaStep(tp.shard_config(cfg, world), rt,
                        weights=tp.shard_weights(device_weights(w), cfg, rank, world),
                        keep_logits=rank == 0)
        tp.open_group(step.ctx, rank, world)
        doc = copy.deepcopy(APPENDIX_B)
        doc["horizon_s"] = horizon
        tee = None
        if rank == 0:
            ora = OracleStep(cfg, w, lambda rid, n: prompt_tokens(rid, n, cfg.vocab, 0))
            tee = TeeStep(step, ora)
        report = Engine(scenario_from_dict(doc, f"tp{rank}"), step=tee or step).run()
        stats = (tee.compared, tee.max_rel, tee.ties, tee.bad[:5]) if tee else None
        q.put((rank, dict(report.counters), {k: list(v) for k, v in step.generated.items()},
               stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_tp2_two_processes_match_full_oracle(cuda):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_rank, args=(r, 2, port, 1.3, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        rank, counters, gen, stats = q.get(timeout=900)
        out[rank] = (counters, gen, stats)
    for p in procs:
        p.join(timeout=60)
    assert [p.exitcode for p in procs] == [0, 0], [p.exitcode for p in procs]
    (c0, g0, st), (c1, g1, _) = out[0], out[1]
    assert c0 == c1 and c0["merges"] > 0 and c0["injections"] > 0
    diverged = [k for k in g0 if g0[k] != g1.get(k)]
    assert not diverged, diverged[:5]  # bit-identical residual streams -> identical tokens
    compared, max_rel, ties, bad = st
    assert compared == c0["tokens_total"] > 0
    assert not bad, bad
    assert max_rel < 2e-2, max_rel
    print(f"tp2: compared={compared} max_rel={max_rel:.2e} ties={ties}")


def _live_rank(rank, world, port, q, device_merges=True, max_iterations=300):
    """One rank of a live TP group: rank 0 plans (LiveEngine, device-polled
    merges, its context mirrored to the follower), rank 1 replays rank 0's
    calls; both ranks' controllers read both ranks' completion tags."""
    import os

    import torch.distributed as dist

    from paper_2603_12831_b200.live import LiveEngine
    from paper_2603_12831_b200.runtime import HsContext, LiveCudaStep, RuntimeConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = TRANSFORMERS["tiny"]
        w = make_weights(cfg, 0)
        sc = tp.shard_config(cfg, world)
        # slow time-shared iterations let arrivals pile up into large prefill
        # batches: room for every row the 1600-token KV budget admits
        rt = RuntimeConfig(max_rows=2048, max_slots=64, kv_pages=256, max_pages_per_req=16,
                           max_pos=2048, max_chunks=1024, cpu_threads=2,
                           host_kv_bytes=128 << 20)
        ctx = HsContext(sc, rt)
        ctx.load_weights(tp.shard_weights(device_weights(w), cfg, rank, world))
        tp.open_group(ctx, rank, world)
        if device_merges:
            ctx.pg_enable(True)
            tp.share_tags(ctx, rank, world, f"/hs_tp_test_{port}")
        if rank == 0:
            mirror = tp.MirrorContext(ctx)
            step = LiveCudaStep(sc, rt, ctx=mirror, device_merges=device_merges)
            step.ctx.keep_logits(True)
            step.keep = True
            step.trace_tokens = True
            doc = copy.deepcopy(APPENDIX_B)
            doc["profiles"]["cluster"]["gpu_kv_capacity"] = 1600
            eng = LiveEngine(scenario_from_dict(doc, "tp_live"), step=step, pace_layers=64,
                             pace_tail=0, batch_trace=True)
            # two processes time-share the test box's one GPU (every fused
            # all-reduce waits for a context switch): a bounded run
            n = eng.run_live(horizon_s=40.0, max_iterations=max_iterations)
            step.finish()
            mirror.flush(stop=True)
            q.put((0, dict(eng.counters), eng.batch_trace,
                   [(r, t.tolist(), lg) for r, t, lg in step.token_log], n, eng.stalled))
        else:
            toks = []

            def grab(ticket):
                import time

                while True:
                    res = ctx.iter_poll(ticket)
                    if res is not None:
                        toks.append(res[0].tolist())
                        return
                    time.sleep(5e-5)

            n = tp.follow(ctx, on_iteration=grab)
            q.put((1, n, toks))
        ctx.close()
    except Exception:  # report at once instead of leaving the parent waiting
        import traceback

        q.put((rank, "error", traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_live_tp2_device_merges_agree_and_match_oracle(cuda):
    """Live TP=2 (config 4's path): one planner, merges decided on both
    ranks' devices from both ranks' completion tags.  Both ranks emit
    identical tokens, and rank 0's realised schedule replayed through the
    full-model oracle matches (logits within 2e-2)."""
    import socket

    import torch.multiprocessing as mp

    from oracle.replay import replay
    from paper_2603_12831_b200.runtime import prompt_tokens

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_live_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        msg = q.get(timeout=1500)
        assert msg[1] != "error", msg[2]
        out[msg[0]] = msg[1:]
    for p in procs:
        p.join(timeout=60)
    assert [p.exitcode for p in procs] == [0, 0], [p.exitcode for p in procs]
    counters, trace, token_log, n0, stalled = out[0]
    n1, toks1 = out[1]
    assert not stalled and counters["tokens_total"] > 300, counters
    assert counters["merges"] > 0 and counters["be_tokens_cpu"] > 0
    assert n1 == n0 == len(token_log)
    for (reqs, t0, _), t1 in zip(token_log, toks1):  # rank 1's rows: same, plus padding
        assert t1[:len(t0)] == t0
    cfg = TRANSFORMERS["tiny"]
    w = make_weights(cfg, 0)
    tl = [(r, np.asarray(t, np.int32), lg) for r, t, lg in token_log]
    st = replay(trace, tl, cfg, w, lambda rid, k: prompt_tokens(rid, k, cfg.vocab, 0))
    assert st.compared == counters["tokens_total"]
    assert not st.bad, st.bad[:5]
    assert st.max_rel < 2e-2, st.max_rel
    print(f"live tp2: iterations={n0} tokens={st.compared} merges={counters['merges']} "
          f"max_rel={st.max_rel:.2e} ties={st.ties}")


def _mirror_rank(rank, world, port, q):
    """CPU: the live-TP call mirroring over gloo against recording libhs
    stand-ins (tests/fake_device.py)."""
    import os
    import sys
    from pathlib import Path

    import torch.distributed as dist

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from fake_device import FakePgContext

    from paper_2603_12831_b200.live import LiveEngine
    from paper_2603_12831_b200.runtime import LiveCudaStep, RuntimeConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    except Exception:
        import traceback

        q.put((rank, "error", traceback.format_exc(), None, None))
        raise
    try:
        sc = tp.shard_config(TRANSFORMERS["tiny"], world)
        rt = RuntimeConfig(max_rows=1024, max_slots=64, kv_pages=256, max_pages_per_req=16,
                           max_pos=2048, max_chunks=1024, cpu_threads=2, host_kv_bytes=1 << 20)
        # host-decided merges: the stand-ins cannot share completion tags across
        # processes, so the follower's fake replays rank 0's merge lists (the
        # device-decided agreement itself is the GPU test above)
        fake = FakePgContext(sc, rt, iter_ms=0.25, cpu_ms=0.5, rng_seed=rank)
        if rank == 0:
            mirror = tp.MirrorContext(fake)
            step = LiveCudaStep(sc, rt, ctx=mirror)
            doc = copy.deepcopy(APPENDIX_B)
            # 2400 GPU KV tokens: BE requests still swap out (13 swap-outs in
            # tests/test_live_host.py's run of this budget) but the LS load alone
            # cannot fill it -- with 1600 the mirrored run, slower per
            # iteration under a loaded host, hit the policy's wall-clock wedge
            doc["profiles"]["cluster"]["gpu_kv_capacity"] = 2400
            eng = LiveEngine(scenario_from_dict(doc, "mirror"), step=step, pace_layers=1)
            eng.run_live(horizon_s=30.0)
            step.finish()
            mirror.flush(stop=True)
            if eng.stalled:  # the reference policy's wall-clock wedge (test_live_host.py)
                q.put((0, "error", "policy wedge", None, None))
                return
            q.put((0, dict(fake.calls), sorted(fake.pages.items()), len(fake.iters),
                   eng.counters["tokens_total"]))
        else:
            n = tp.follow(fake)
            q.put((1, dict(fake.calls), sorted(fake.pages.items()), n, None))
    except Exception:
        import traceback

        q.put((rank, "error", traceback.format_exc(), None, None))
        raise
    finally:
        dist.destroy_process_group()


def test_live_tp_mirror_replays_every_call():
    """The follower of a live TP group replays exactly the state-changing
    calls of the planning rank: the same iterations, layers, page tables,
    swaps and host-KV reservations (two gloo ranks on CPU)."""
    import queue
    import socket

    import torch.multiprocessing as mp

    def attempt():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        procs = [ctx.Process(target=_mirror_rank, args=(r, 2, port, q)) for r in range(2)]
        for p in procs:
            p.start()
        out, err = {}, None
        try:
            for _ in procs:
                msg = q.get(timeout=120)
                if msg[1] == "error":
                    err = msg[2]
                    break
                out[msg[0]] = msg[1:]
        except queue.Empty:
            err = "no result within 120 s"
        for p in procs:
            p.join(timeout=30 if err is None else 5)
            if p.is_alive():
                p.kill()
        if err is None and [p.exitcode for p in procs] != [0, 0]:
            err = f"exit codes {[p.exitcode for p in procs]}"
        return out, err

    # a wall-clock run of two spawned ranks (gloo rendezvous on a fresh port):
    # retried, with the reason printed, on an environmental failure or the
    # reference policy's wall-clock wedge (a policy property, not the mirror)
    out, err = attempt()
    for _ in range(2):
        if err is None:
            break
        print("mirror run failed, retrying:", err)
        out, err = attempt()
    assert err is None, err
    calls0, pages0, iters0, tokens = out[0]
    calls1, pages1, iters1, _ = out[1]
    assert tokens > 1000
    assert iters0 == iters1 > 100
    for k in ("iter_begin", "layer", "swap", "cpu_submit", "merged"):
        assert calls0[k] == calls1[k], (k, calls0[k], calls1[k])
    assert calls0["swap"] > 0
    assert pages0 == pages1
