"""The CPU oracle itself is pinned before it is trusted:
* its Llama arithmetic against HF transformers' LlamaForCausalLM (golden
  logits in tests/golden/hf_tiny.npz, oracle/gen_hf_golden.py);
* its bf16-rounding mode stays within the north-star 2e-2 of the fp32 mode;
* the per-op restatements against closed-form identities."""

import numpy as np
import pytest

from oracle import llama_ops as O
from oracle.serve_oracle import OracleModel, make_weights
from paper_2603_12831_b200.models import TRANSFORMERS


@pytest.fixture(scope="module")
def tiny():
    cfg = TRANSFORMERS["tiny"]
    return cfg, make_weights(cfg, seed=0)


def test_oracle_matches_hf_transformers_llama(golden_dir, tiny):
    cfg, w = tiny
    g = np.load(golden_dir / "hf_tiny.npz")
    ours = OracleModel(cfg, w, bf16_points=False).forward(g["tokens"])
    ref = g["logits"].astype(np.float64)
    rel = np.abs(ours - ref).max() / np.abs(ref).max()
    assert rel < 1e-4, rel
    assert np.array_equal(ours.argmax(-1), ref.argmax(-1))


def test_bf16_rounding_points_within_north_star_bound(golden_dir, tiny):
    cfg, w = tiny
    g = np.load(golden_dir / "hf_tiny.npz")
    lo = OracleModel(cfg, w, bf16_points=True).forward(g["tokens"])
    ref = g["logits"]
    rel = np.abs(lo - ref).max(axis=-1) / np.abs(ref).max(axis=-1)
    assert rel.max() < 2e-2, rel.max()


def test_bf16_rounding_is_round_to_nearest_even():
    x = np.array([1.0, 1.00390625, 1.01171875, -2.5, 3.0e-39, np.inf], np.float32)
    r = O.to_bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == 1.015625 and r[3] == -2.5
    assert np.isinf(r[5])
    b = O.bf16_bits(np.array([1.0, -2.0], np.float32))
    assert list(b) == [0x3F80, 0xC000]
    assert np.array_equal(O.from_bf16_bits(b), np.array([1.0, -2.0], np.float32))


def test_lse_merge_equals_full_softmax():
    rng = np.random.default_rng(3)
    n_q, hd, keys = 4, 64, 300
    q = rng.standard_normal((1, n_q, hd)).astype(np.float32)
    k = rng.standard_normal((keys, 2, hd)).astype(np.float32)
    v = rng.standard_normal((keys, 2, hd)).astype(np.float32)
    full, lse_full = O.attention_rows(q, k, v, 2)
    parts, lses = [], []
    for a, b in [(0, 100), (100, 250), (250, 300)]:
        o, l_ = O.attention_rows(q, k[a:b], v[a:b], 2)
        parts.append(o[0])
        lses.append(l_[0])
    merged = O.lse_merge(np.stack(parts), np.stack(lses))
    assert np.allclose(merged, full[0], atol=1e-5)
    m = np.max(lses, axis=0)
    assert np.allclose(m + np.log(np.exp(np.array(lses) - m).sum(0)), lse_full[0], atol=1e-5)


def test_rope_tables_rotate_pairs():
    cos, sin = O.rope_tables(64, 8, 10000.0)
    x = np.random.default_rng(1).standard_normal((3, 2, 8)).astype(np.float32)
    pos = np.array([0, 5, 63])
    y = O.apply_rope(x, pos, cos, sin)
    assert np.allclose(y[0], x[0])  # position 0 is the identity
    assert np.allclose(np.linalg.norm(y, axis=-1), np.linalg.norm(x, axis=-1), atol=1e-5)
