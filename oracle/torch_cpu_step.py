"""CPU baseline of the serving step (baseline infrastructure only; never
imported by the product): one serving iteration of the Llama-3-8B step on
the host cores in torch bf16, restated from the same module sequence as the
numpy oracle (reference pkg/src/hybridserve/engine.py:56, QKV -> Attn ->
Proj -> ResidualAdd -> MLP -> ResidualAdd, over the concatenated LS + BE
rows of engine.py:921-950) -- the SURVEY §7 `TorchCpuStep`, tuned for speed
rather than bit-tracking:

* weights bf16 [out][in] (`F.linear`, oneDNN / AMX on the host), all layers
  distinct, so every iteration streams the full 16 GB like the GPU step;
* LS decode rows attend over their own KV (ctx ~700); piggyback BE rows
  attend over host-resident KV (ctx ~9000, the CPU attention of
  engine.py:529-560), every row its own KV buffer;
* LM head + greedy argmax for every token-producing row (engine.py:1024-1047).

`bench.py --impl reference` times whole iterations of this class on the
box's host cores (all of them) and reports BE tokens/s, ms per iteration and
the weight stream's achieved GB/s.
"""

from __future__ import annotations

import time

import torch
import torch.nn.functional as F


class TorchCpuStep:
    def __init__(self, cfg, n_ls: int, ls_ctx: int, n_be_gpu: int, n_merge: int, be_ctx: int,
                 threads: int, seed: int = 0):
        torch.set_num_threads(threads)
        self.cfg = cfg
        self.threads = threads
        self.n_ls, self.n_be_gpu, self.n_merge = n_ls, n_be_gpu, n_merge
        g = torch.Generator().manual_seed(seed)
        d, hd = cfg.d_model, cfg.head_dim

        def mat(n, k):
            return (torch.randn(n, k, generator=g, dtype=torch.float32) * 0.02).to(torch.bfloat16)

        self.layers = [{"qkv": mat(cfg.qkv_dim, d), "o": mat(d, cfg.n_q * hd),
                        "gu": mat(2 * cfg.ffn, d), "down": mat(d, cfg.ffn)}
                       for _ in range(cfg.n_layers)]
        self.embed = mat(cfg.vocab, d)
        self.lm_head = mat(cfg.vocab, d)
        self.weight_bytes = 2 * (cfg.params_per_layer * cfg.n_layers + cfg.vocab * d)

        # per-row KV [n_kv, keys, hd] for two alternating layer slots (> L3:
        # every layer's attention reads its bytes from DRAM)
        def kv(n, keys):
            return [(torch.randn(n, cfg.n_kv, keys, hd, generator=g).to(torch.bfloat16),
                     torch.randn(n, cfg.n_kv, keys, hd, generator=g).to(torch.bfloat16))
                    for _ in range(2)]

        self.kv_gpu_rows = kv(max(n_ls, 1), max(ls_ctx, 1))  # LS decodes
        self.ls_ctx = ls_ctx
        self.kv_be = kv(max(n_merge, 1), be_ctx) if n_merge else None
        self.kv_be_res = kv(n_be_gpu, be_ctx) if n_be_gpu else None
        self.tokens = torch.randint(0, cfg.vocab, (n_ls + n_be_gpu + n_merge,), generator=g)
        self.kv_bytes = 0
        for grp, n, keys in ((self.kv_gpu_rows, n_ls, ls_ctx), (self.kv_be_res, n_be_gpu, be_ctx),
                             (self.kv_be, n_merge, be_ctx)):
            if grp is not None:
                self.kv_bytes += n * 2 * cfg.n_kv * keys * hd * 2 * cfg.n_layers

    def _norm(self, x):
        x32 = x.float()
        return (x32 * torch.rsqrt(x32.pow(2).mean(-1, keepdim=True) + self.cfg.norm_eps)).to(
            torch.bfloat16)

    def _attend(self, q, k, v):
        # q [rows, n_q, hd] over k/v [rows, n_kv, keys, hd] (GQA)
        out = F.scaled_dot_product_attention(q.unsqueeze(2), k, v, enable_gqa=True)
        return out.squeeze(2)

    @torch.inference_mode()
    def iteration(self) -> dict:
        """One serving iteration; returns timing and work."""
        c = self.cfg
        t0 = time.perf_counter()
        rows = self.n_ls + self.n_be_gpu + self.n_merge
        x = self.embed[self.tokens].float()
        nq, hd = c.n_q * c.head_dim, c.head_dim
        for li, w in enumerate(self.layers):
            qkv = F.linear(self._norm(x), w["qkv"])
            q = qkv[:, :nq].reshape(rows, c.n_q, hd)
            outs = []
            a, b = self.n_ls, self.n_ls + self.n_be_gpu
            k, v = self.kv_gpu_rows[li & 1]
            outs.append(self._attend(q[:a], k[:a, :, :self.ls_ctx], v[:a, :, :self.ls_ctx]))
            if self.n_be_gpu:
                kb, vb = self.kv_be_res[li & 1]
                outs.append(self._attend(q[a:b], kb, vb))
            if self.n_merge:
                kb, vb = self.kv_be[li & 1]
                outs.append(self._attend(q[b:], kb, vb))
            attn = torch.cat(outs).reshape(rows, nq)
            x = x + F.linear(attn, w["o"]).float()
            gu = F.linear(self._norm(x), w["gu"])
            act = (F.silu(gu[:, :c.ffn].float()) * gu[:, c.ffn:].float()).to(torch.bfloat16)
            x = x + F.linear(act, w["down"]).float()
        logits = F.linear(self._norm(x), self.lm_head)
        toks = logits.float().argmax(-1)
        dt = time.perf_counter() - t0
        return {"s": dt, "tokens": toks, "weight_gbs": self.weight_bytes / dt / 1e9,
                "kv_gbs": self.kv_bytes / dt / 1e9, "be_tokens": self.n_be_gpu + self.n_merge}
