"""Transformer configurations the B200 step executes (BASELINE.json configs).

The reference names models only through cost profiles ("34B"/"70B",
pkg/src/hybridserve/profiles.py:216-252); the product runs the real layer,
so the architecture is named here: Llama blocks (RMSNorm, rotate-half RoPE,
GQA attention, SwiGLU MLP).  Weights are synthetic (random init), as the
north star prescribes.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class TransformerConfig:
    name: str
    d_model: int
    n_layers: int
    n_q: int
    n_kv: int
    head_dim: int
    ffn: int
    vocab: int
    rope_theta: float = 500000.0
    norm_eps: float = 1e-5
    tp: int = 1  # tensor-parallel shard this config describes (per-GPU dims)

    @property
    def qkv_dim(self) -> int:
        return (self.n_q + 2 * self.n_kv) * self.head_dim

    @property
    def params_per_layer(self) -> int:
        d = self.d_model
        return self.qkv_dim * d + d * self.n_q * self.head_dim + 3 * self.ffn * d

    @property
    def kv_bytes_per_token_layer(self) -> int:
        return 2 * self.n_kv * self.head_dim * 2

    @property
    def ship_bytes(self) -> int:  # piggyback D2H per item per layer
        return self.qkv_dim * 2

    @property
    def result_bytes(self) -> int:  # piggyback H2D per item per layer
        return self.n_q * self.head_dim * 2


TRANSFORMERS: dict[str, TransformerConfig] = {
    # config 1: "tiny Llama (2 layers, d=256, 4 heads)"; n_kv=2 exercises GQA
    "tiny": TransformerConfig("tiny", 256, 2, 4, 2, 64, 768, 1024, rope_theta=10000.0),
    "llama3-8b": TransformerConfig("llama3-8b", 4096, 32, 32, 8, 128, 14336, 128256),
    "llama2-13b": TransformerConfig("llama2-13b", 5120, 40, 40, 40, 128, 13824, 32000,
                                    rope_theta=10000.0),
    # Llama-3-70B (config 4) and its per-GPU shard under 8-way tensor
    # parallelism (tp.shard_config: 8 q heads, 1 KV head, ffn 3584 per rank;
    # embedding and LM head replicated)
    "llama3-70b": TransformerConfig("llama3-70b", 8192, 80, 64, 8, 128, 28672, 128256),
    "llama3-70b-tp8": TransformerConfig("llama3-70b-tp8", 8192, 80, 8, 1, 128, 3584, 128256,
                                        tp=8),
}


def get_transformer(name: str) -> TransformerConfig:
    try:
        return TRANSFORMERS[name]
    except KeyError:
        from .errors import ConfigError

        raise ConfigError(f"unknown transformer {name!r} (choose from {sorted(TRANSFORMERS)})")
