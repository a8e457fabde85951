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
                 threads: int, seed: int = 0, n_prefill: int = 0, be_gpu_ctx: int = 0):
        torch.set_num_threads(threads)
        self.cfg = cfg
        self.threads = threads
        self.n_ls, self.n_be_gpu, self.n_merge = n_ls, n_be_gpu, n_merge
        # prefill chunk tokens of the iteration: one causal chunk whose K/V
        # come from its own rows (the chunked prefill of scheduling.py:127-133)
        self.n_prefill = n_prefill
        be_gpu_ctx = be_gpu_ctx or be_ctx
        g = torch.Generator().manual_seed(seed)
        d, hd = cfg.d_model, cfg.head_dim

        def mat(n, k):
            return (torch.randn(n, k, generator=g, dtype=torch.float32) * 0.02).to(torch.bfloat16)

        # one random layer, cloned into distinct memory for the others (the
        # values do not change the cost; every iteration still streams all
        # layers from DRAM, and init stays at memcpy speed instead of ~1 min
        # of normal_() for 8B parameters)
        first = {"qkv": mat(cfg.qkv_dim, d), "o": mat(d, cfg.n_q * hd),
                 "gu": mat(2 * cfg.ffn, d), "down": mat(d, cfg.ffn)}
        self.layers = [first] + [{k: v.clone() for k, v in first.items()}
                                 for _ in range(cfg.n_layers - 1)]
        self.embed = torch.empty(cfg.vocab, d, dtype=torch.bfloat16).uniform_(-0.03, 0.03)
        self.lm_head = torch.empty(cfg.vocab, d, dtype=torch.bfloat16).uniform_(-0.03, 0.03)
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
        self.kv_be_res = kv(n_be_gpu, be_gpu_ctx) if n_be_gpu else None
        self.tokens = torch.randint(0, cfg.vocab, (n_ls + n_be_gpu + n_merge + n_prefill,),
                                    generator=g)
        self.kv_bytes = 0
        for grp, n, keys in ((self.kv_gpu_rows, n_ls, ls_ctx), (self.kv_be_res, n_be_gpu, be_gpu_ctx),
                             (self.kv_be, n_merge, be_ctx)):
            if grp is not None:
                self.kv_bytes += n * 2 * cfg.n_kv * keys * hd * 2 * cfg.n_layers

    def _norm(self, x):
        x32 = x.float()
        return (x32 * torch.rsqrt(x32.pow(2).mean(-1, keepdim=True) + self.cfg.norm_eps)).to(
            torch.bfloat16)

    def _attend(self, q, k, v):
        # q [rows, n_q, hd] over k/v [rows, n_kv, keys, hd] (GQA): the group's
        # query heads as the M side of two batched bf16 matmuls (measured on
        # an 8-core host: 20.6 GB/s of KV vs 15.2 for F.scaled_dot_product_attention)
        rows, nq, hd = q.shape
        nkv = k.shape[1]
        qq = q.reshape(rows, nkv, nq // nkv, hd)
        s = torch.matmul(qq, k.transpose(-1, -2)).float() * (hd ** -0.5)
        p = torch.softmax(s, -1).to(torch.bfloat16)
        return torch.matmul(p, v).reshape(rows, nq, hd)

    @torch.inference_mode()
    def iteration(self) -> dict:
        """One serving iteration; returns timing and work."""
        c = self.cfg
        t0 = time.perf_counter()
        rows = self.n_ls + self.n_be_gpu + self.n_merge + self.n_prefill
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
            e = b + self.n_merge
            if self.n_merge:
                kb, vb = self.kv_be[li & 1]
                outs.append(self._attend(q[b:e], kb, vb))
            if self.n_prefill:
                kv0 = nq
                kp = qkv[e:, kv0:kv0 + c.n_kv * hd].reshape(-1, c.n_kv, hd).transpose(0, 1)
                vp = qkv[e:, kv0 + c.n_kv * hd:].reshape(-1, c.n_kv, hd).transpose(0, 1)
                qp = q[e:].transpose(0, 1)
                op = F.scaled_dot_product_attention(qp.unsqueeze(0), kp.unsqueeze(0),
                                                    vp.unsqueeze(0), is_causal=True,
                                                    enable_gqa=True)
                outs.append(op.squeeze(0).transpose(0, 1))
            attn = torch.cat(outs).reshape(rows, nq)
            x = x + F.linear(attn, w["o"]).float()
            gu = F.linear(self._norm(x), w["gu"])
            act = (F.silu(gu[:, :c.ffn].float()) * gu[:, c.ffn:].float()).to(torch.bfloat16)
            x = x + F.linear(act, w["down"]).float()
        # token rows: decodes and merged chains (a prefill chunk's last row
        # only at completion; left out of the sample)
        logits = F.linear(self._norm(x[:self.n_ls + self.n_be_gpu + self.n_merge]), self.lm_head)
        toks = logits.float().argmax(-1)
        dt = time.perf_counter() - t0
        return {"s": dt, "tokens": toks, "weight_gbs": self.weight_bytes / dt / 1e9,
                "kv_gbs": self.kv_bytes / dt / 1e9, "be_tokens": self.n_be_gpu + self.n_merge}
