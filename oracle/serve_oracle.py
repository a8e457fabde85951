"""CPU oracle of the serving step (test infrastructure only; never imported by
the product).  It implements the LayerStep interface request by request in
numpy, independently of libhs' row layout:

* batch rows (decodes over ctx+1 keys, causal chunk prefill) run the Llama
  block at each layer (module sequence QKV -> Attn -> Proj -> ResidualAdd ->
  MLP -> ResidualAdd, reference pkg/src/hybridserve/engine.py:56);
* Attention Piggybacking chains follow the reference dataflow
  (engine.py:982-1022, §3.2): an injected token runs QKV(1) and
  ships q/k/v; the host appends k/v and attends over ctx+1 keys; the merge at
  layer l fetches the residual saved before QKV(l), runs Proj+MLP(l), saves
  the residual and ships QKV(l+1); at the last layer the token is emitted and
  the next token's QKV(1) ships.

Precision mirrors the product's rounding points (bf16 weights, bf16 normed
activations / q,k,v / attention outputs / MLP activation, fp32 residual
stream and logits) with float64 arithmetic in between, so logits agree to
~1e-3 and the 2e-2 north-star bound has headroom.  The arithmetic of each
module is pinned against HF transformers' Llama (tests/golden/hf_tiny.npz).
"""

from __future__ import annotations

import numpy as np

from oracle import llama_ops as O


class OracleModel:
    """fp32 (bf16-valued) weights + the per-row Llama block."""

    def __init__(self, cfg, weights: dict, bf16_points: bool = True):
        self.cfg = cfg
        # float64 copies of the (bf16-valued) weights: exact, and cast once
        self.w = {k: ([x.astype(np.float64) for x in v] if isinstance(v, list)
                      else v.astype(np.float64)) for k, v in weights.items()}
        self.cos, self.sin = O.rope_tables(32768, cfg.head_dim, cfg.rope_theta)
        # round at the product's bf16 points, or stay fp32/fp64 throughout
        # (the mode pinned against HF transformers)
        self.r = O.to_bf16 if bf16_points else (lambda x: np.asarray(x, np.float32))

    def _norm(self, h, w):
        h64 = h.astype(np.float64)
        inv = 1.0 / np.sqrt((h64 * h64).mean(axis=-1, keepdims=True) + self.cfg.norm_eps)
        return self.r((h64 * inv * w.astype(np.float64)).astype(np.float32))

    def qkv(self, h: np.ndarray, layer: int, pos: np.ndarray):
        """h [rows, d] fp32 residual -> bf16 (q [rows,n_q,hd], k, v [rows,n_kv,hd])."""
        c = self.cfg
        xn = self._norm(h, self.w["norm_in"][layer])
        y = O.gemm(xn, self.w["qkv"][layer])
        nq, nk, hd = c.n_q * c.head_dim, c.n_kv * c.head_dim, c.head_dim
        q = O.apply_rope(y[:, :nq].reshape(-1, c.n_q, hd), pos, self.cos, self.sin)
        k = O.apply_rope(y[:, nq:nq + nk].reshape(-1, c.n_kv, hd), pos, self.cos, self.sin)
        v = y[:, nq + nk:].reshape(-1, c.n_kv, hd)
        return self.r(q), self.r(k), self.r(v)

    def post_attention(self, h: np.ndarray, attn: np.ndarray, layer: int) -> np.ndarray:
        """Proj + ResidualAdd + MLP + ResidualAdd; attn [rows, n_q*hd] bf16."""
        c = self.cfg
        h = (h.astype(np.float64) + O.gemm(attn, self.w["o"][layer])).astype(np.float32)
        xn2 = self._norm(h, self.w["norm_post"][layer])
        gu = O.gemm(xn2, self.w["gate_up"][layer]).astype(np.float64)
        g, u = gu[:, :c.ffn], gu[:, c.ffn:]
        act = self.r((g / (1.0 + np.exp(-g)) * u).astype(np.float32))
        return (h.astype(np.float64) + O.gemm(act, self.w["down"][layer])).astype(np.float32)

    def logits(self, h: np.ndarray) -> np.ndarray:
        return O.gemm(self._norm(h, self.w["final_norm"]), self.w["lm_head"])

    def attend(self, q, k, v, pos):
        """q [rows,n_q,hd] at positions pos over keys k/v [keys,n_kv,hd]."""
        hi = int(pos.max()) + 1
        out, _ = O.attention_rows(q, k[:hi], v[:hi], self.cfg.n_kv,
                                  np.arange(hi)[None, :] <= pos[:, None])
        return self.r(out.reshape(len(pos), -1))

    def forward(self, toks) -> np.ndarray:
        """Plain causal forward of one sequence -> logits of every position."""
        toks = np.asarray(toks)
        pos = np.arange(len(toks))
        h = self.embed(toks)
        for li in range(self.cfg.n_layers):
            q, k, v = self.qkv(h, li, pos)
            h = self.post_attention(h, self.attend(q, k, v, pos), li)
        return self.logits(h)

    def embed(self, toks) -> np.ndarray:
        return self.w["embed"][np.asarray(toks)].astype(np.float32)


class OracleStep:
    """LayerStep restatement (duck-typed; see paper_2603_12831_b200.engine)."""

    def __init__(self, cfg, weights: dict, prompt_fn, bf16_points: bool = True):
        self.cfg = cfg
        # bf16_points=False: the fp32 validation datapath (no bf16 roundings)
        self.m = OracleModel(cfg, weights, bf16_points)
        self.prompt_fn = prompt_fn  # (req_id, length) -> int32 ids
        self.kv: dict[str, np.ndarray] = {}
        self.resid: dict[str, np.ndarray] = {}
        self.ship: dict[str, tuple] = {}
        self.result: dict[str, np.ndarray] = {}
        self.last_token: dict[str, int] = {}
        self.generated: dict[str, list[int]] = {}
        self.pending: dict[str, tuple] = {}  # chains waiting for QKV(l+1)
        self.logit_log: list[tuple[str, np.ndarray]] = []
        self.forced = 0
        # teacher forcing known in advance (replays of a recorded run): the
        # token to emit for a request, used instead of the oracle's argmax --
        # also for a chain's restart, which embeds the token inside layer L
        self.teacher: dict[str, int] = {}

    # -- helpers --------------------------------------------------------------
    def attach(self, engine):
        self.engine = engine

    def _kv(self, rid: str) -> np.ndarray:
        if rid not in self.kv:
            r = self.engine.requests[rid]
            cap = r.prompt_len + r.output_len + 2
            c = self.cfg
            self.kv[rid] = np.zeros((c.n_layers, 2, cap, c.n_kv, c.head_dim), np.float32)
        return self.kv[rid]

    def _seq(self, r) -> np.ndarray:
        p = self.prompt_fn(r.id, r.prompt_len)
        g = self.generated.get(r.id, [])
        return np.concatenate([p, np.asarray(g, np.int32)]) if g else p

    def _attend(self, rid, layer, q, pos):
        """q [rows, n_q, hd] at positions pos over the request's KV[0..pos]."""
        kv = self._kv(rid)[layer]
        return self.m.attend(q, kv[0], kv[1], pos)

    def _ship_qkv(self, rid, layer, h_row, pos):
        q, k, v = self.m.qkv(h_row[None], layer, np.array([pos]))
        self.ship[rid] = (layer, pos, q[0], k[0], v[0])

    # -- LayerStep --------------------------------------------------------------
    def begin_iteration(self, plan):
        eng = self.engine
        self.groups = []  # (rid, kind, positions, h)
        for rid in plan.ls_decode + plan.be_decode_gpu:
            r = eng.requests[rid]
            h = self.m.embed([self.last_token[rid]])
            self.groups.append([rid, "decode", np.array([r.ctx]), h])
        for rid, q in plan.ls_prefill_chunks + plan.be_prefill_chunks:
            r = eng.requests[rid]
            done = r.prefill_done
            toks = self._seq(r)[done:done + q]
            final = done + q >= r.prefill_target and r.rebuild_tokens == 0
            self.groups.append([rid, "final" if final else "chunk",
                                np.arange(done, done + q), self.m.embed(toks)])
        self.chain_tokens: list[tuple[str, np.ndarray]] = []

    def layer(self, layer, merges):
        L = self.cfg.n_layers
        li = layer - 1
        if self.groups:
            # rows are independent through the dense modules: one GEMM per
            # module over all groups, attention per request
            sizes = [len(g[2]) for g in self.groups]
            h_all = np.concatenate([g[3] for g in self.groups])
            pos_all = np.concatenate([g[2] for g in self.groups])
            q, k, v = self.m.qkv(h_all, li, pos_all)
            attn, o = [], 0
            for g, n in zip(self.groups, sizes):
                rid, pos = g[0], g[2]
                kv = self._kv(rid)
                kv[li, 0, pos] = k[o:o + n]
                kv[li, 1, pos] = v[o:o + n]
                attn.append(self._attend(rid, li, q[o:o + n], pos))
                o += n
            h_all = self.m.post_attention(h_all, np.concatenate(attn), li)
            o = 0
            for g, n in zip(self.groups, sizes):
                g[3] = h_all[o:o + n]
                o += n
        for item, outcome in merges:
            rid = item.req_id
            if outcome == "inject":
                h = self.m.embed([self.last_token[rid]])[0]
                self.resid[rid] = h
                self._ship_qkv(rid, 0, h, self.engine.requests[rid].ctx)
                continue
            h = self.resid.pop(rid)
            h = self.m.post_attention(h[None], self.result.pop(rid)[None], li)[0]
            if outcome == "chain":
                self.resid[rid] = h
                self._ship_qkv(rid, li + 1, h, self.engine.requests[rid].ctx)
                continue
            lg = self.m.logits(h[None])[0]
            self.chain_tokens.append((rid, lg))
            tok = int(O.argmax_first(lg[None])[0])
            self._emit(rid, tok, lg)
            if outcome == "token_next":
                h1 = self.m.embed([self.last_token[rid]])[0]
                self.resid[rid] = h1
                self._ship_qkv(rid, 0, h1, self.engine.requests[rid].ctx)

    def _emit(self, rid, tok, lg):
        if rid in self.teacher:
            forced = self.teacher.pop(rid)
            self.forced += forced != tok
            tok = forced
        self.last_token[rid] = tok
        self.generated.setdefault(rid, []).append(tok)
        self.logit_log.append((rid, lg))

    def end_iteration(self, plan):
        for rid, kind, pos, h in self.groups:
            if kind == "chunk":
                continue
            lg = self.m.logits(h[-1:])[0]
            self._emit(rid, int(O.argmax_first(lg[None])[0]), lg)

    def force_token(self, rid: str, tok: int) -> None:
        """Teacher forcing for near-tie argmax flips (see tests)."""
        if self.last_token.get(rid) != tok:
            self.forced += 1
            self.last_token[rid] = tok
            self.generated[rid][-1] = tok

    def cpu_service(self, host_id, items):
        for it in items:
            layer, pos, q, k, v = self.ship.pop(it.req_id)
            assert layer == it.layer - 1 and pos == it.ctx_tokens, (layer, pos, it)
            kv = self._kv(it.req_id)
            kv[layer, 0, pos] = k
            kv[layer, 1, pos] = v
            self.result[it.req_id] = self._attend(it.req_id, layer, q[None], np.array([pos]))[0]

    def swap_out_done(self, req): ...
    def resumed_on_gpu(self, req): ...
    def preempted(self, req):
        pass  # KV is rebuilt by the re-prefill (positions overwritten)
    def released(self, req): ...
    def finish(self): ...


def make_weights(cfg, seed: int = 0, std: float = 0.02, bf16: bool = True) -> dict:
    """Synthetic Llama weights: N(0, std) rounded to bf16 (or kept fp32 for
    the fp32 validation datapath); norm gains 1 + 0.1 N(0,1) in fp32 so the
    norm weights are exercised."""
    rng = np.random.default_rng(seed)
    d, L = cfg.d_model, cfg.n_layers

    def mat(n, k):
        m = (rng.standard_normal((n, k)) * std).astype(np.float32)
        return O.to_bf16(m) if bf16 else m

    def gain():
        return (1.0 + 0.1 * rng.standard_normal(d)).astype(np.float32)

    w = {"embed": mat(cfg.vocab, d), "lm_head": mat(cfg.vocab, d), "final_norm": gain(),
         "qkv": [], "o": [], "gate_up": [], "down": [], "norm_in": [], "norm_post": []}
    for _ in range(L):
        w["qkv"].append(mat(cfg.qkv_dim, d))
        w["o"].append(mat(d, cfg.n_q * cfg.head_dim))
        w["gate_up"].append(mat(2 * cfg.ffn, d))
        w["down"].append(mat(d, cfg.ffn))
        w["norm_in"].append(gain())
        w["norm_post"].append(gain())
    return w


def device_weights(w: dict, fp32: bool = False) -> dict:
    """Same weights in libhs' host format: bf16 bit patterns (or fp32
    matrices for the fp32 datapath), fp32 norms."""
    if fp32:
        return w
    out = {}
    for k, v in w.items():
        if isinstance(v, list):
            out[k] = [O.bf16_bits(x) if x.ndim == 2 else x for x in v]
        else:
            out[k] = O.bf16_bits(v) if v.ndim == 2 else v
    return out
