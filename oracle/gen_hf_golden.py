"""Pins the oracle's Llama arithmetic against HF transformers (test
infrastructure only).  Builds transformers.LlamaForCausalLM with the tiny
config and the oracle's synthetic weights, runs one fp32 causal forward and
stores tokens + logits in tests/golden/hf_tiny.npz.  The check itself
(tests/test_oracle.py) needs only numpy.

Usage: python oracle/gen_hf_golden.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle.serve_oracle import make_weights  # noqa: E402
from paper_2603_12831_b200.models import TRANSFORMERS  # noqa: E402


def main() -> None:
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    cfg = TRANSFORMERS["tiny"]
    w = make_weights(cfg, seed=0)
    hf_cfg = LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.d_model,
                         intermediate_size=cfg.ffn, num_hidden_layers=cfg.n_layers,
                         num_attention_heads=cfg.n_q, num_key_value_heads=cfg.n_kv,
                         head_dim=cfg.head_dim, rms_norm_eps=cfg.norm_eps,
                         rope_theta=cfg.rope_theta, max_position_embeddings=4096,
                         tie_word_embeddings=False, attention_bias=False, mlp_bias=False)
    model = LlamaForCausalLM(hf_cfg).float().eval()
    sd = model.state_dict()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))  # noqa: E731
    sd["model.embed_tokens.weight"] = t(w["embed"])
    sd["lm_head.weight"] = t(w["lm_head"])
    sd["model.norm.weight"] = t(w["final_norm"])
    nq, nk = cfg.n_q * cfg.head_dim, cfg.n_kv * cfg.head_dim
    for l in range(cfg.n_layers):
        p = f"model.layers.{l}."
        qkv = w["qkv"][l]
        sd[p + "self_attn.q_proj.weight"] = t(qkv[:nq])
        sd[p + "self_attn.k_proj.weight"] = t(qkv[nq:nq + nk])
        sd[p + "self_attn.v_proj.weight"] = t(qkv[nq + nk:])
        sd[p + "self_attn.o_proj.weight"] = t(w["o"][l])
        sd[p + "mlp.gate_proj.weight"] = t(w["gate_up"][l][:cfg.ffn])
        sd[p + "mlp.up_proj.weight"] = t(w["gate_up"][l][cfg.ffn:])
        sd[p + "mlp.down_proj.weight"] = t(w["down"][l])
        sd[p + "input_layernorm.weight"] = t(w["norm_in"][l])
        sd[p + "post_attention_layernorm.weight"] = t(w["norm_post"][l])
    model.load_state_dict(sd)
    toks = np.random.default_rng(7).integers(0, cfg.vocab, 48)
    with torch.no_grad():
        logits = model(torch.from_numpy(toks)[None]).logits[0].double().numpy()
    out = ROOT / "tests" / "golden" / "hf_tiny.npz"
    np.savez_compressed(out, tokens=toks.astype(np.int32), logits=logits.astype(np.float32),
                        weight_seed=0)
    print(f"wrote {out} ({out.stat().st_size // 1024} KiB), transformers "
          f"{__import__('transformers').__version__}")


if __name__ == "__main__":
    main()
