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
