"""fp32 validation datapath (north star: "logits within ... 1e-4 in an fp32
validation mode where greedy tokens must also match over the first 64
steps").

libhs runs with hs_rt_cfg.precision = HS_PREC_FP32: fp32 weights,
activations, paged KV, piggyback mailboxes, host KV and CPU attention, SIMT
fp32 kernels on the device (csrc/step_f32.cu).  The oracle runs the same
schedule with no bf16 rounding points (float64 arithmetic, fp32 storage).
Config 1 (tiny Llama, the Appendix-B schedule through the first swap-outs,
injections and piggyback merges) is compared token by token: logits within
1e-4 relative, and every greedy token of the first 64 iterations identical.
The 2-layer Llama-3-8B-shaped run is in test_serving_8b.py.
"""

import copy

import pytest

from oracle.scenarios import APPENDIX_B
from oracle.serve_oracle import OracleStep, device_weights, make_weights
from oracle.tee import TeeStep

LOGIT_REL_TOL_FP32 = 1e-4


@pytest.mark.gpu
def test_fp32_datapath_matches_oracle_on_appendix_b(cuda):
    from paper_2603_12831_b200.engine import Engine
    from paper_2603_12831_b200.models import TRANSFORMERS
    from paper_2603_12831_b200.runtime import CudaStep, RuntimeConfig, prompt_tokens
    from paper_2603_12831_b200.scenario import scenario_from_dict

    cfg = TRANSFORMERS["tiny"]
    w = make_weights(cfg, 0, bf16=False)
    rt = RuntimeConfig(max_rows=2048, max_slots=64, kv_pages=256, max_pages_per_req=16,
                       max_pos=2048, max_chunks=1024, cpu_threads=4, host_kv_bytes=256 << 20,
                       precision="fp32")
    gpu = CudaStep(cfg, rt, weights=device_weights(w, fp32=True), keep_logits=True)
    ora = OracleStep(cfg, w, lambda rid, k: prompt_tokens(rid, k, cfg.vocab, 0),
                     bf16_points=False)
    tee = TeeStep(gpu, ora)
    doc = copy.deepcopy(APPENDIX_B)
    doc["horizon_s"] = 1.4  # past the first swap-outs, injections and merges
    report = Engine(scenario_from_dict(doc, "fp32"), step=tee).run()
    c = report.counters
    assert c["merges"] > 0 and c["injections"] > 0 and c["be_tokens_cpu"] > 0, c
    assert tee.iterations >= 64
    assert tee.compared == c["tokens_total"]
    assert not tee.bad, tee.bad[:5]
    assert tee.max_rel < LOGIT_REL_TOL_FP32, tee.max_rel
    assert not [i for i in tee.tie_iterations if i < 64], tee.tie_iterations
    assert tee.ties == 0, tee.tie_iterations
    print(f"fp32: iterations={tee.iterations} tokens={tee.compared} merges={c['merges']} "
          f"max_rel={tee.max_rel:.2e}")


def test_fp32_oracle_has_no_bf16_rounding():
    """CPU: the oracle's fp32 mode keeps unrounded fp32 weights and values."""
    import numpy as np

    from oracle.serve_oracle import OracleModel
    from paper_2603_12831_b200.models import TRANSFORMERS

    cfg = TRANSFORMERS["tiny"]
    w = make_weights(cfg, 0, bf16=False)
    bits = w["qkv"][0].view(np.uint32) & 0xFFFF
    assert (bits != 0).mean() > 0.9  # not bf16-representable
    m = OracleModel(cfg, w, bf16_points=False)
    q, k, v = m.qkv(np.ones((1, cfg.d_model), np.float32), 0, np.array([3]))
    assert ((q.view(np.uint32) & 0xFFFF) != 0).any()
