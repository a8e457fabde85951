"""C1 host attention (CPU, no GPU needed): AVX-512-BF16 and AVX2 paths of
the piggyback CPU worker against the numpy oracle, incl. ragged key counts
(tile tails of 1..15 keys) and every GQA group size used by the configs."""

import ctypes as C

import numpy as np
import pytest

from oracle import llama_ops as O


def _run(q, k, v, n_q, n_kv, hd, impl):
    from paper_2603_12831_b200 import _lib

    lib = _lib.load()
    qb, kb, vb = (np.ascontiguousarray(O.bf16_bits(x)) for x in (q, k, v))
    out = np.zeros(n_q * hd, np.uint16)
    lse = np.zeros(n_q, np.float32)
    rc = lib.hs_host_attention(qb.ctypes.data_as(C.c_void_p), kb.ctypes.data_as(C.c_void_p),
                               vb.ctypes.data_as(C.c_void_p), k.shape[1], n_q, n_kv, hd,
                               out.ctypes.data_as(C.c_void_p), lse.ctypes.data_as(C.c_void_p),
                               impl)
    _lib.check(rc, "hs_host_attention")
    return O.from_bf16_bits(out).reshape(n_q, hd), lse


def _has_avx512bf16() -> bool:
    try:
        return "avx512_bf16" in open("/proc/cpuinfo").read()
    except OSError:
        return False


@pytest.mark.parametrize("impl", [1, 2])
@pytest.mark.parametrize("n_q,n_kv,hd", [(32, 8, 128), (4, 2, 64), (40, 40, 128), (8, 1, 128)])
@pytest.mark.parametrize("keys", [1, 15, 16, 17, 63, 300])
def test_host_attention_matches_oracle(impl, n_q, n_kv, hd, keys):
    if impl == 1 and not _has_avx512bf16():
        pytest.skip("no AVX-512-BF16 on this host")
    rng = np.random.default_rng(keys * 7 + n_q + impl)
    q = O.to_bf16(rng.standard_normal((n_q, hd)).astype(np.float32))
    k = O.to_bf16(rng.standard_normal((n_kv, keys, hd)).astype(np.float32))
    v = O.to_bf16(rng.standard_normal((n_kv, keys, hd)).astype(np.float32))
    got, lse = _run(q, k, v, n_q, n_kv, hd, impl)
    ref, ref_lse = O.decode_attention(q, k.transpose(1, 0, 2), v.transpose(1, 0, 2), n_kv)
    err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-6)
    assert err < 1.5e-2, err
    assert np.abs(lse - ref_lse).max() < 1e-2


def test_host_attention_without_amx_matches_oracle():
    """The vdpbf16ps QK^T path (hosts without AMX, or HS_CPU_AMX=0) in a fresh
    process, since the AMX choice is made once per process."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    if not _has_avx512bf16():
        pytest.skip("no AVX-512-BF16 on this host")
    root = Path(__file__).resolve().parent.parent
    code = (
        "import numpy as np, sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')\n"
        "from test_cpu_attention import _run\n"
        "from oracle import llama_ops as O\n"
        "rng = np.random.default_rng(3)\n"
        "q = O.to_bf16(rng.standard_normal((32, 128)).astype(np.float32))\n"
        "k = O.to_bf16(rng.standard_normal((8, 301, 128)).astype(np.float32))\n"
        "v = O.to_bf16(rng.standard_normal((8, 301, 128)).astype(np.float32))\n"
        "got, _ = _run(q, k, v, 32, 8, 128, 1)\n"
        "ref, _ = O.decode_attention(q, k.transpose(1, 0, 2), v.transpose(1, 0, 2), 8)\n"
        "print(float(np.abs(got - ref).max() / np.abs(ref).max()))\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**os.environ, "HS_CPU_AMX": "0"}, timeout=120)
    assert out.returncode == 0, out.stderr
    assert float(out.stdout.strip().splitlines()[-1]) < 1.5e-2


@pytest.mark.parametrize("impl", [1, 2])
@pytest.mark.parametrize("keys", [9000, 32769])
def test_host_attention_long_context(impl, keys):
    """C1 at the bench's BE context (~9k keys, AMX QK^T + prefetch path) and at
    config 5's 32k-token prompts, Llama-3-8B geometry."""
    if impl == 1 and not _has_avx512bf16():
        pytest.skip("no AVX-512-BF16 on this host")
    n_q, n_kv, hd = 32, 8, 128
    rng = np.random.default_rng(keys + impl)
    q = O.to_bf16((rng.standard_normal((n_q, hd)) * 0.3).astype(np.float32))
    k = O.to_bf16(rng.standard_normal((n_kv, keys, hd)).astype(np.float32))
    v = O.to_bf16(rng.standard_normal((n_kv, keys, hd)).astype(np.float32))
    got, lse = _run(q, k, v, n_q, n_kv, hd, impl)
    ref, ref_lse = O.decode_attention(q, k.transpose(1, 0, 2), v.transpose(1, 0, 2), n_kv)
    err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-6)
    assert err < 1.5e-2, err
    assert np.abs(lse - ref_lse).max() < 1e-2
