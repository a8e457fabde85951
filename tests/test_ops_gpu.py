"""Per-kernel parity: each libhs kernel (through the C ABI) against the numpy
oracle on the same seeded inputs.  Tolerances: fp32 outputs of bf16 GEMMs
1e-4 of the output scale; bf16 outputs 1.5e-2 of the output scale (one bf16
rounding of values in [-scale, scale] plus fp32 accumulation order)."""

import ctypes as C

import numpy as np
import pytest

from oracle import llama_ops as O

pytestmark = pytest.mark.gpu


_KEEP: list = []  # device buffers must outlive the asynchronous kernels that use them


def _t(x, dev, dtype=None):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    t = t.to(dev)
    _KEEP.append(t)
    return t


@pytest.fixture(autouse=True)
def _release_buffers():
    yield
    _KEEP.clear()


def _p(t):
    return C.c_void_p(t.data_ptr())


def _bf16_np(rng, shape, scale=1.0):
    return O.to_bf16((rng.standard_normal(shape) * scale).astype(np.float32))


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize(
    "tokens,n,k",
    [(1, 128, 64), (5, 256, 256), (16, 512, 4096), (17, 6144, 4096), (37, 1024, 1024),
     (64, 384, 512), (100, 256, 1024), (200, 384, 512), (300, 256, 128), (513, 128, 256)],
)
def test_gemm_tcgen05(cuda, tokens, n, k):
    import torch
    from paper_2603_12831_b200 import _lib

    rng = np.random.default_rng(tokens * 7 + n + k)
    x = _bf16_np(rng, (tokens, k))
    w = _bf16_np(rng, (n, k), 0.05)
    xd, wd = _t(x, cuda, torch.bfloat16), _t(w, cuda, torch.bfloat16)
    max_splits = 16
    part = torch.zeros(max_splits * tokens * n, dtype=torch.float32, device=cuda)
    out = torch.zeros(tokens * n, dtype=torch.float32, device=cuda)
    used = C.c_int(0)
    _lib.call("hs_op_gemm_bf16", _p(xd), tokens, k, _p(wd), n, k, _p(part), max_splits,
              C.byref(used), None)
    _lib.call("hs_op_splitk_reduce", _p(part), used.value, tokens, n, _p(out), None)
    torch.cuda.synchronize()
    ref = O.gemm(x, w)
    assert _rel(out.cpu().numpy().reshape(tokens, n), ref) < 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("tokens,n,k", [(256, 256, 256), (300, 512, 512), (512, 768, 1024),
                                        (1024, 1024, 4096), (700, 6144, 4096)])
def test_gemm_cta_pair(cuda, tokens, n, k):
    """K3 on CTA pairs (tcgen05.mma.cta_group::2) against the oracle; the
    partial planes sum to the product."""
    import torch
    from paper_2603_12831_b200 import _lib

    rng = np.random.default_rng(tokens * 5 + n + k)
    x = _bf16_np(rng, (tokens, k))
    w = _bf16_np(rng, (n, k), 0.05)
    xd, wd = _t(x, cuda, torch.bfloat16), _t(w, cuda, torch.bfloat16)
    max_splits = 16
    part = torch.full((max_splits * tokens * n,), float("nan"), dtype=torch.float32, device=cuda)
    out = torch.zeros(tokens * n, dtype=torch.float32, device=cuda)
    used = C.c_int(0)
    _lib.call("hs_op_gemm_bf16_pair", _p(xd), tokens, k, _p(wd), n, k, _p(part), max_splits,
              C.byref(used), None)
    _lib.call("hs_op_splitk_reduce", _p(part), used.value, tokens, n, _p(out), None)
    torch.cuda.synchronize()
    ref = O.gemm(x, w)
    assert _rel(out.cpu().numpy().reshape(tokens, n), ref) < 1e-4, used.value


def _make_pool(rng, layers, pages, n_kv, hd):
    pool = _bf16_np(rng, (layers, pages, 2, n_kv, 64, hd))
    return pool


def _gather_kv(pool, layer, page_list, ctx):
    # -> k, v: [ctx, n_kv, hd]
    blocks = pool[layer, page_list]  # [np, 2, n_kv, 64, hd]
    k = blocks[:, 0].transpose(0, 2, 1, 3).reshape(-1, pool.shape[3], pool.shape[5])[:ctx]
    v = blocks[:, 1].transpose(0, 2, 1, 3).reshape(-1, pool.shape[3], pool.shape[5])[:ctx]
    return k, v


@pytest.mark.parametrize("n_q,n_kv,hd", [(4, 2, 64), (32, 8, 128), (8, 1, 128), (4, 4, 128)])
@pytest.mark.parametrize("chunk_pages", [1, 3, 16])
def test_decode_attention_split_k(cuda, n_q, n_kv, hd, chunk_pages):
    import torch
    from paper_2603_12831_b200 import _lib

    rng = np.random.default_rng(n_q * 31 + hd + chunk_pages)
    layers, pages = 2, 48
    pool = _make_pool(rng, layers, pages, n_kv, hd)
    ctxs = [1, 63, 64, 65, 200, 700]
    max_pages = 12
    perm = rng.permutation(pages)
    pt = np.zeros((len(ctxs), max_pages), np.int32)
    cursor = 0
    for r, c in enumerate(ctxs):
        npg = (c + 63) // 64
        pt[r, :npg] = perm[cursor:cursor + npg]
        cursor += npg
    q = _bf16_np(rng, (len(ctxs), n_q, hd))
    layer = 1
    chunks, begin = [], [0]
    for r, c in enumerate(ctxs):
        npg = (c + 63) // 64
        for p0 in range(0, npg, chunk_pages):
            chunks.append((r, r, p0, min(npg, p0 + chunk_pages), c))
        begin.append(len(chunks))
    chunks = np.array(chunks, np.int32)
    dpool = _t(pool, cuda, torch.bfloat16)
    dq = _t(q, cuda, torch.bfloat16)
    dpt = _t(pt, cuda)
    dch = _t(chunks, cuda)
    dbeg = _t(np.array(begin, np.int32), cuda)
    opart = torch.zeros(len(chunks) * n_q * hd, dtype=torch.float32, device=cuda)
    lpart = torch.zeros(len(chunks) * n_q, dtype=torch.float32, device=cuda)
    out = torch.zeros(len(ctxs), n_q * hd, dtype=torch.bfloat16, device=cuda)
    lse = torch.zeros(len(ctxs) * n_q, dtype=torch.float32, device=cuda)
    _lib.call("hs_op_decode_attention", _p(dpool), layers, pages, n_kv, hd, layer, _p(dq),
              n_q * hd, n_q, _p(dpt), max_pages, _p(dch), len(chunks), _p(opart), _p(lpart), None)
    _lib.call("hs_op_decode_combine", _p(opart), _p(lpart), _p(dbeg), len(ctxs), n_q, n_kv, hd,
              _p(out), n_q * hd, _p(lse), None)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy().reshape(len(ctxs), n_q, hd)
    got_lse = lse.cpu().numpy().reshape(len(ctxs), n_q)
    for r, c in enumerate(ctxs):
        k, v = _gather_kv(pool, layer, pt[r, :(c + 63) // 64], c)
        ref, ref_lse = O.decode_attention(q[r], k, v, n_kv)
        assert _rel(got[r], ref) < 1.5e-2, (r, c)
        assert np.abs(got_lse[r] - ref_lse).max() < 2e-2


@pytest.mark.parametrize("n_q,n_kv,hd", [(4, 2, 64), (32, 8, 128)])
@pytest.mark.parametrize("done,q_len", [(0, 1), (0, 64), (0, 100), (130, 37), (64, 200)])
def test_prefill_attention_causal(cuda, n_q, n_kv, hd, done, q_len):
    _prefill_case(cuda, n_q, n_kv, hd, done, q_len)


# the tcgen05 kernel's GQA packings (G = 1, 4, 8 query heads per KV head:
# 13B, 8B, 70B-TP8), the two-Q-tile CTAs of large chunks (>= 2/3 of the SMs
# busy) and a longer context
@pytest.mark.parametrize("n_q,n_kv,hd,done,q_len", [
    (40, 40, 128, 70, 130), (8, 1, 128, 100, 300), (16, 2, 128, 0, 129),
    (32, 8, 128, 0, 832), (32, 8, 128, 64, 900), (32, 8, 128, 3000, 200)])
def test_prefill_attention_gqa_and_two_tile(cuda, n_q, n_kv, hd, done, q_len):
    _prefill_case(cuda, n_q, n_kv, hd, done, q_len)


def _prefill_case(cuda, n_q, n_kv, hd, done, q_len):
    import torch
    from paper_2603_12831_b200 import _lib

    rng = np.random.default_rng(done * 13 + q_len + hd)
    layers = 1
    total = done + q_len
    npg = (total + 63) // 64
    pages = max(16, npg + 2)
    pool = _make_pool(rng, layers, pages, n_kv, hd)
    max_pages = max(8, npg)
    pt = np.zeros((2, max_pages), np.int32)
    pt[1, :npg] = rng.permutation(pages)[:npg]
    slot = 1
    q = _bf16_np(rng, (q_len, n_q, hd))
    tiles = np.array([(slot, r0, done + r0, min(64, q_len - r0)) for r0 in range(0, q_len, 64)],
                     np.int32)
    dpool = _t(pool, cuda, torch.bfloat16)
    dq = _t(q, cuda, torch.bfloat16)
    out = torch.zeros(q_len, n_q * hd, dtype=torch.bfloat16, device=cuda)
    _lib.call("hs_op_prefill_attention", _p(dpool), layers, pages, n_kv, hd, 0, _p(dq), n_q * hd,
              n_q, _p(_t(pt, cuda)), max_pages, _p(_t(tiles, cuda)), len(tiles), _p(out),
              n_q * hd, None)
    torch.cuda.synchronize()
    k, v = _gather_kv(pool, 0, pt[1, :npg], total)
    ref, _ = O.prefill_attention(q, np.arange(done, total), k, v, n_kv)
    got = out.float().cpu().numpy().reshape(q_len, n_q, hd)
    assert _rel(got, ref) < 1.5e-2


def test_qkv_rope_scatter_and_ship(cuda):
    import torch
    from paper_2603_12831_b200 import _lib

    rng = np.random.default_rng(5)
    n_q, n_kv, hd, layers, pages = 8, 2, 128, 2, 6
    n_tot = (n_q + 2 * n_kv) * hd
    rows, splits = 5, 3
    part = rng.standard_normal((splits, rows, n_tot)).astype(np.float32)
    pos = np.array([0, 5, 63, 64, 130], np.int32)
    slot = np.array([0, 1, 2, 3, 1], np.int32)
    mode = np.array([0, 0, 1, 0, 1], np.int32)
    cos, sin = O.rope_tables(256, hd, 500000.0)
    pt = np.array([[0, 1, 2], [3, 4, 5], [0, 0, 0], [2, 1, 0]], np.int32)
    pool = np.zeros((layers, pages, 2, n_kv, 64, hd), np.float32)
    dpool = _t(pool, cuda, torch.bfloat16)
    qbuf = torch.zeros(rows, n_q * hd, dtype=torch.bfloat16, device=cuda)
    ship = torch.zeros(4, n_tot, dtype=torch.bfloat16, device=cuda)
    _lib.call("hs_op_qkv_rope_scatter", _p(_t(part, cuda)), splits, rows, n_q, n_kv, hd,
              _p(_t(cos, cuda)), _p(_t(sin, cuda)), _p(_t(pos, cuda)), _p(_t(slot, cuda)),
              _p(_t(mode, cuda)), _p(qbuf), n_q * hd, _p(dpool), layers, pages, 1,
              _p(_t(pt, cuda)), 3, _p(ship), n_tot, None)
    torch.cuda.synchronize()
    full = part.sum(0)
    q = O.apply_rope(full[:, : n_q * hd].reshape(rows, n_q, hd), pos, cos, sin)
    k = O.apply_rope(full[:, n_q * hd:(n_q + n_kv) * hd].reshape(rows, n_kv, hd), pos, cos, sin)
    v = full[:, (n_q + n_kv) * hd:].reshape(rows, n_kv, hd)
    gq = qbuf.float().cpu().numpy().reshape(rows, n_q, hd)
    gpool = dpool.float().cpu().numpy()
    gship = ship.float().cpu().numpy()
    for r in range(rows):
        if mode[r] == 0:
            assert np.allclose(gq[r], O.to_bf16(q[r]), atol=1e-6, rtol=0)
            page = pt[slot[r], pos[r] // 64]
            assert np.allclose(gpool[1, page, 0, :, pos[r] % 64], O.to_bf16(k[r]), atol=1e-6)
            assert np.allclose(gpool[1, page, 1, :, pos[r] % 64], O.to_bf16(v[r]), atol=1e-6)
        else:
            row = np.concatenate([q[r].ravel(), k[r].ravel(), v[r].ravel()])
            assert np.allclose(gship[slot[r]], O.to_bf16(row), atol=1e-6)


def test_norms_embed_silu_argmax_merge(cuda):
    import torch
    from paper_2603_12831_b200 import _lib

    rng = np.random.default_rng(9)
    rows, d, vocab, ffn, splits = 6, 256, 1000, 384, 2
    emb = _bf16_np(rng, (vocab, d))
    tok = rng.integers(0, vocab, rows).astype(np.int32)
    h = torch.zeros(rows * d, dtype=torch.float32, device=cuda)
    _lib.call("hs_op_embed", _p(_t(tok, cuda)), rows, _p(_t(emb, cuda, torch.bfloat16)), d,
              _p(h), None)
    torch.cuda.synchronize()
    assert np.array_equal(h.cpu().numpy().reshape(rows, d), emb[tok])

    w = (1.0 + 0.1 * rng.standard_normal(d)).astype(np.float32)
    out = torch.zeros(rows, d, dtype=torch.bfloat16, device=cuda)
    _lib.call("hs_op_rmsnorm", _p(h), rows, d, _p(_t(w, cuda)), C.c_float(1e-5), _p(out), d, None)
    part = rng.standard_normal((splits, rows, d)).astype(np.float32)
    out2 = torch.zeros(rows, d, dtype=torch.bfloat16, device=cuda)
    _lib.call("hs_op_residual_add_norm", _p(_t(part, cuda)), splits, rows, d, _p(h),
              _p(_t(w, cuda)), C.c_float(1e-5), _p(out2), d, None)
    torch.cuda.synchronize()
    assert _rel(out.float().cpu().numpy(), O.rmsnorm(emb[tok], w, 1e-5)) < 1e-2
    h2 = emb[tok] + part.sum(0)
    assert np.allclose(h.cpu().numpy().reshape(rows, d), h2, atol=1e-5)
    assert _rel(out2.float().cpu().numpy(), O.rmsnorm(h2, w, 1e-5)) < 1e-2

    gu = rng.standard_normal((splits, rows, 2 * ffn)).astype(np.float32)
    act = torch.zeros(rows, ffn, dtype=torch.bfloat16, device=cuda)
    _lib.call("hs_op_silu_mul", _p(_t(gu, cuda)), splits, rows, ffn, _p(act), ffn, None)
    torch.cuda.synchronize()
    assert _rel(act.float().cpu().numpy(), O.silu_mul(gu.sum(0), ffn)) < 1e-2

    lg = rng.standard_normal((splits, rows, vocab)).astype(np.float32)
    lg[:, 2, 17] = 50.0  # tie between index 17 and 400 on row 2
    lg[:, 2, 400] = 50.0
    toks = torch.zeros(rows, dtype=torch.int32, device=cuda)
    logits = torch.zeros(rows * vocab, dtype=torch.float32, device=cuda)
    _lib.call("hs_op_argmax", _p(_t(lg, cuda)), splits, rows, vocab, _p(toks), _p(logits), None)
    torch.cuda.synchronize()
    ref_logits = lg.sum(0)
    assert np.allclose(logits.cpu().numpy().reshape(rows, vocab), ref_logits, atol=1e-5)
    assert np.array_equal(toks.cpu().numpy(), O.argmax_first(ref_logits))

    n_q, hd, n_parts = 4, 64, 3
    parts = _bf16_np(rng, (rows, n_parts, n_q * hd))
    lse = rng.standard_normal((rows, n_parts, n_q)).astype(np.float32)
    mo = torch.zeros(rows, n_q * hd, dtype=torch.bfloat16, device=cuda)
    _lib.call("hs_op_lse_merge", _p(_t(parts, cuda, torch.bfloat16)), _p(_t(lse, cuda)), n_parts,
              rows, n_q, hd, n_q * hd, n_parts * n_q * hd, _p(mo), n_q * hd, None)
    torch.cuda.synchronize()
    got = mo.float().cpu().numpy().reshape(rows, n_q, hd)
    for r in range(rows):
        ref = O.lse_merge(parts[r].reshape(n_parts, n_q, hd), lse[r])
        assert _rel(got[r], ref) < 1.5e-2


@pytest.mark.parametrize("tokens,n,k", [(1, 128, 64), (16, 6144, 4096), (77, 384, 512),
                                        (300, 256, 1024)])
def test_gemm_tcgen05_blocked_weights(cuda, tokens, n, k):
    """Same GEMM with weights pre-tiled [n/128][k/64][128][64] (4-D TMA map)."""
    import torch
    from paper_2603_12831_b200 import _lib

    rng = np.random.default_rng(tokens + n)
    x = _bf16_np(rng, (tokens, k))
    w = _bf16_np(rng, (n, k), 0.05)
    xd, wd = _t(x, cuda, torch.bfloat16), _t(w, cuda, torch.bfloat16)
    wb = torch.empty_like(wd)
    _lib.call("hs_op_relayout_blocked", _p(wd), _p(wb), n, k, None)
    part = torch.zeros(16 * tokens * n, dtype=torch.float32, device=cuda)
    out = torch.zeros(tokens * n, dtype=torch.float32, device=cuda)
    used = C.c_int(0)
    _lib.call("hs_op_gemm_bf16_blocked", _p(xd), tokens, k, _p(wb), n, k, _p(part), 16,
              C.byref(used), None)
    _lib.call("hs_op_splitk_reduce", _p(part), used.value, tokens, n, _p(out), None)
    torch.cuda.synchronize()
    assert _rel(out.cpu().numpy().reshape(tokens, n), O.gemm(x, w)) < 1e-4


@pytest.mark.parametrize("n_q,n_kv,hd", [(32, 8, 128), (4, 2, 64)])
@pytest.mark.parametrize("chunk_pages", [1, 4, 64])
def test_decode_attention_fused_combine(cuda, n_q, n_kv, hd, chunk_pages):
    """K1 with K2 fused into the last CTA per (row, KV head); run twice to
    check the self-resetting counters."""
    import torch
    from paper_2603_12831_b200 import _lib

    rng = np.random.default_rng(11 + chunk_pages)
    layers, pages = 1, 64
    pool = _make_pool(rng, layers, pages, n_kv, hd)
    ctxs = [1, 64, 65, 300, 1100]
    max_pages = 20
    perm = rng.permutation(pages)
    pt = np.zeros((len(ctxs), max_pages), np.int32)
    cur = 0
    for r, c in enumerate(ctxs):
        npg = (c + 63) // 64
        pt[r, :npg] = perm[cur:cur + npg]
        cur += npg
    q = _bf16_np(rng, (len(ctxs), n_q, hd))
    chunks, begin = [], [0]
    for r, c in enumerate(ctxs):
        npg = (c + 63) // 64
        for p0 in range(0, npg, chunk_pages):
            chunks.append((r, r, p0, min(npg, p0 + chunk_pages), c))
        begin.append(len(chunks))
    dpool, dq = _t(pool, cuda, torch.bfloat16), _t(q, cuda, torch.bfloat16)
    dpt, dch = _t(pt, cuda), _t(np.array(chunks, np.int32), cuda)
    dbeg = _t(np.array(begin, np.int32), cuda)
    cnt = torch.zeros(len(ctxs) * n_kv, dtype=torch.int32, device=cuda)
    opart = torch.zeros(len(chunks) * n_q * hd, dtype=torch.float32, device=cuda)
    lpart = torch.zeros(len(chunks) * n_q, dtype=torch.float32, device=cuda)
    for _ in range(2):
        out = torch.zeros(len(ctxs), n_q * hd, dtype=torch.bfloat16, device=cuda)
        _lib.call("hs_op_decode_attention_fused", _p(dpool), layers, pages, n_kv, hd, 0, _p(dq),
                  n_q * hd, n_q, _p(dpt), max_pages, _p(dch), len(chunks), len(ctxs), _p(dbeg),
                  _p(opart),
                  _p(lpart), _p(cnt), _p(out), n_q * hd, None)
        torch.cuda.synchronize()
        got = out.float().cpu().numpy().reshape(len(ctxs), n_q, hd)
        for r, c in enumerate(ctxs):
            k, v = _gather_kv(pool, 0, pt[r, :(c + 63) // 64], c)
            ref, _ = O.decode_attention(q[r], k, v, n_kv)
            assert _rel(got[r], ref) < 1.5e-2, (r, c)
    assert int(cnt.abs().sum().item()) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("rows,d,splits", [(33, 4096, 3), (300, 256, 1), (64, 5120, 16),
                                           (8, 4096, 0)])
def test_residual_add_norm_row_and_cluster_forms(cuda, rows, d, splits):
    """Both launch forms of K4 (8-CTA cluster per row for <= 32 rows, one CTA
    per row above) against the fp64 oracle."""
    import torch
    from paper_2603_12831_b200 import _lib

    rng = np.random.default_rng(rows + d)
    h0 = rng.standard_normal((rows, d)).astype(np.float32)
    w = (1.0 + 0.1 * rng.standard_normal(d)).astype(np.float32)
    part = rng.standard_normal((max(splits, 1), rows, d)).astype(np.float32)
    h = _t(h0, cuda)
    out = torch.zeros(rows, d, dtype=torch.bfloat16, device=cuda)
    _lib.call("hs_op_residual_add_norm", _p(_t(part, cuda)), splits, rows, d, _p(h),
              _p(_t(w, cuda)), C.c_float(1e-5), _p(out), d, None)
    torch.cuda.synchronize()
    h2 = h0 + (part.sum(0) if splits else 0.0)
    assert np.allclose(h.cpu().numpy().reshape(rows, d), h2, atol=1e-4)
    assert _rel(out.float().cpu().numpy(), O.rmsnorm(h2, w, 1e-5)) < 1e-2


@pytest.mark.gpu
@pytest.mark.parametrize("rows,ffn,splits", [(1, 14336, 7), (129, 768, 2), (40, 13824, 16)])
def test_silu_mul_shapes(cuda, rows, ffn, splits):
    import torch
    from paper_2603_12831_b200 import _lib

    rng = np.random.default_rng(rows + ffn)
    gu = rng.standard_normal((splits, rows, 2 * ffn)).astype(np.float32)
    act = torch.zeros(rows, ffn, dtype=torch.bfloat16, device=cuda)
    _lib.call("hs_op_silu_mul", _p(_t(gu, cuda)), splits, rows, ffn, _p(act), ffn, None)
    torch.cuda.synchronize()
    assert _rel(act.float().cpu().numpy(), O.silu_mul(gu.sum(0), ffn)) < 1e-2


@pytest.mark.gpu
@pytest.mark.parametrize("ctxs", [[9000, 700, 9001], [32768, 1]])
def test_decode_attention_long_context(cuda, ctxs):
    """K1+K2 at the bench's and config 5's context lengths, split exactly as
    the runtime splits them (runtime.decode_chunks).  Logical pages map onto
    a small physical pool with repeats, so 32k-token rows stay cheap to build
    while every page load goes through the page table."""
    import torch
    from paper_2603_12831_b200 import _lib
    from paper_2603_12831_b200.runtime import decode_chunks

    n_q, n_kv, hd = 32, 8, 128
    rng = np.random.default_rng(sum(ctxs))
    pages = 96
    pool = _make_pool(rng, 1, pages, n_kv, hd)
    max_pages = max((c + 63) // 64 for c in ctxs)
    pt = rng.integers(0, pages, size=(len(ctxs), max_pages)).astype(np.int32)
    q = _bf16_np(rng, (len(ctxs), n_q, hd))
    chunks, begin = decode_chunks(ctxs, n_kv)
    chunks = np.array([(r, r, p0, p1, c) for r, _, p0, p1, c in chunks], np.int32)
    dpool, dq = _t(pool, cuda, torch.bfloat16), _t(q, cuda, torch.bfloat16)
    dpt, dch = _t(pt, cuda), _t(chunks, cuda)
    dbeg = _t(np.array(begin, np.int32), cuda)
    cnt = torch.zeros(len(ctxs) * n_kv, dtype=torch.int32, device=cuda)
    opart = torch.zeros(len(chunks) * n_q * hd, dtype=torch.float32, device=cuda)
    lpart = torch.zeros(len(chunks) * n_q, dtype=torch.float32, device=cuda)
    out = torch.zeros(len(ctxs), n_q * hd, dtype=torch.bfloat16, device=cuda)
    _lib.call("hs_op_decode_attention_fused", _p(dpool), 1, pages, n_kv, hd, 0, _p(dq),
              n_q * hd, n_q, _p(dpt), max_pages, _p(dch), len(chunks), len(ctxs), _p(dbeg),
              _p(opart),
              _p(lpart), _p(cnt), _p(out), n_q * hd, None)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy().reshape(len(ctxs), n_q, hd)
    for r, c in enumerate(ctxs):
        k, v = _gather_kv(pool, 0, pt[r, :(c + 63) // 64], c)
        ref, _ = O.decode_attention(q[r], k, v, n_kv)
        assert _rel(got[r], ref) < 1.5e-2, (r, c, _rel(got[r], ref))
