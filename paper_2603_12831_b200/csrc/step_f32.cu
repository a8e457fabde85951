// fp32 validation datapath of the serving step (hs_rt_cfg.precision ==
// HS_PREC_FP32).
//
// The north star pins numerics twice: logits within 2e-2 of the oracle in
// bf16, and within 1e-4 -- with greedy tokens identical over the first 64
// steps -- in an fp32 validation mode.  This file is that mode: the same
// layer as hs_layer() (reference pkg/src/hybridserve/engine.py:921-1022: the
// module sequence QKV -> Attn -> Proj -> ResidualAdd -> MLP -> ResidualAdd of
// engine.py:56 over the batch rows, the piggyback carry / merge / restart
// rows, the LM head and greedy token) with every tensor in fp32: weights,
// normed activations, q/k/v, the paged KV pool, the piggyback ship / result
// mailboxes and the host KV the CPU pool attends over.  The kernels are
// plain SIMT fp32 (fp32 FMAs, no tensor-core rounding): this mode exists to
// be exact, not fast, and it runs on the device like the serving path -- it
// is not a CPU fallback.
//
// Row layout per call (as in step.cu): rows [0, B) batch rows, [B, B+C)
// carry rows (QKV only, shipped), merged rows [B, B+M) after attention.
#include <math_constants.h>

#include <algorithm>

#include "hs_common.cuh"
#include "hs_ctx.h"

namespace hs {
namespace {

constexpr int kTokBlock = 8;  // token rows per warp in the fp32 GEMM

// y[t][n] = sum_k x[t][k] * w[n][k]: one warp per (feature, 8-token block);
// lanes stride k by float4, each keeps 8 fp32 partial sums, warp tree sum.
__global__ void __launch_bounds__(256)
    gemm_f32_kernel(const float* __restrict__ x, int ldx, int tokens,
                    const float* __restrict__ w, int n_out, int k, float* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = blockIdx.x * 8 + warp;
  const int t0 = blockIdx.y * kTokBlock;
  if (n >= n_out) return;
  const int nt = min(kTokBlock, tokens - t0);
  float acc[kTokBlock];
#pragma unroll
  for (int j = 0; j < kTokBlock; ++j) acc[j] = 0.f;
  const float* wr = w + static_cast<size_t>(n) * k;
  for (int kk = lane * 4; kk < k; kk += 128) {
    const float4 wv = *reinterpret_cast<const float4*>(wr + kk);
#pragma unroll
    for (int j = 0; j < kTokBlock; ++j) {
      if (j < nt) {
        const float4 xv =
            *reinterpret_cast<const float4*>(x + static_cast<size_t>(t0 + j) * ldx + kk);
        acc[j] = fmaf(wv.x, xv.x, acc[j]);
        acc[j] = fmaf(wv.y, xv.y, acc[j]);
        acc[j] = fmaf(wv.z, xv.z, acc[j]);
        acc[j] = fmaf(wv.w, xv.w, acc[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kTokBlock; ++j)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
  if (lane < nt) {
    float v = acc[0];
#pragma unroll
    for (int j = 1; j < kTokBlock; ++j)
      if (lane == j) v = acc[j];
    y[static_cast<size_t>(t0 + lane) * n_out + n] = v;
  }
}

int gemm_f32(const float* x, int ldx, int tokens, const float* w, int n_out, int k, float* y,
             cudaStream_t st) {
  if (tokens <= 0) return HS_OK;
  if (k % 4 || ldx % 4) return HS_E_CONFIG;
  dim3 grid((n_out + 7) / 8, (tokens + kTokBlock - 1) / kTokBlock);
  return launch_pdl(gemm_f32_kernel, grid, dim3(256), 0, st, x, ldx, tokens, w, n_out, k, y);
}

__global__ void embed_f32_kernel(const int* __restrict__ tok, const float* __restrict__ emb,
                                 int d, float* __restrict__ h) {
  pdl_wait();
  pdl_trigger();
  const float* src = emb + static_cast<size_t>(tok[blockIdx.x]) * d;
  float* dst = h + static_cast<size_t>(blockIdx.x) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = src[i];
}

// block sum of a double over 256 threads
__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];
  __syncthreads();
  return t;
}

// Per row r: hn = (row source) + y[r] (y may be null); h[r] = hn; the put
// rows also store hn into the residual store; out[r] = RMSNorm(hn) * w.
// Row sources and puts follow RowIo (the residual get / put of merged rows).
__global__ void __launch_bounds__(256)
    add_norm_f32_kernel(const float* __restrict__ y, int d, float* __restrict__ h,
                        const float* __restrict__ w, float eps, float* __restrict__ out, RowIo io) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[8];
  const int r = blockIdx.x;
  const float* src = io.row_src(h, r, d);
  float* hr = h + static_cast<size_t>(r) * d;
  float* put = io.row_put(r, d);
  double ss = 0.0;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float v = y ? src[i] + y[static_cast<size_t>(r) * d + i] : src[i];
    hr[i] = v;
    if (put) put[i] = v;
    ss += static_cast<double>(v) * v;
  }
  ss = block_sum(ss, red);
  const float inv = static_cast<float>(1.0 / sqrt(ss / d + eps));
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    out[static_cast<size_t>(r) * d + i] = hr[i] * inv * w[i];
}

int add_norm_f32(const float* y, int rows, int d, float* h, const float* w, float eps, float* out,
                 cudaStream_t st, const RowIo& io = RowIo{}) {
  if (rows <= 0) return HS_OK;
  return launch_pdl(add_norm_f32_kernel, dim3(rows), dim3(256), 0, st, y, d, h, w, eps, out, io);
}

// QKV epilogue: rotate-half RoPE of q and k heads, then per row
//   batch row:  q -> fq[r], k/v -> the request's fp32 KV page at row_pos
//   carry row:  q|k|v -> the slot's fp32 ship mailbox (piggyback D2H,
//               engine.py:982-989)
// and rows past the QKV rows gather merged host results (result mailbox ->
// fattn[B + i]) behind their completion tags, as in the bf16 step.
struct RopeArgs {
  const float* y;
  int rows, n_batch, n_q, n_kv, hd;
  const float *cos, *sin;
  const int *row_pos, *row_slot, *carry_pos, *carry_slot;
  float* q;
  float* pool;
  KvGeom g;
  int layer;
  const int* page_table;
  int pt_stride;
  float* ship;
  const float* result;
  const int* merge_slot;
  int n_merge;
  float* attn_merged;  // fattn + B * nqh
  const int* expect;
  const unsigned* tags;
  unsigned* fault;
  int layer1;
};

__global__ void __launch_bounds__(256) rope_f32_kernel(RopeArgs a) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const int nqh = a.n_q * a.hd, qkv_n = (a.n_q + 2 * a.n_kv) * a.hd;
  if (r >= a.rows) {  // merged row: the host attention result
    const int i = r - a.rows;
    const int slot = a.merge_slot[i];
    if (a.expect) {
      __shared__ int ok;
      if (threadIdx.x == 0) {
        unsigned tag;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(tag) : "l"(a.tags + slot) : "memory");
        ok = tag == static_cast<unsigned>(a.expect[i]);
        if (!ok) {
          a.fault[1] = slot;
          a.fault[2] = a.layer1;
          a.fault[3] = tag;
          __threadfence_system();
          atomicExch(a.fault, 1u);
        }
      }
      __syncthreads();
      if (!ok) return;
    }
    const float* src = a.result + static_cast<size_t>(slot) * nqh;
    float* dst = a.attn_merged + static_cast<size_t>(i) * nqh;
    for (int e = threadIdx.x; e < nqh; e += blockDim.x) dst[e] = src[e];
    return;
  }
  const bool batch = r < a.n_batch;
  const int pos = batch ? a.row_pos[r] : a.carry_pos[r - a.n_batch];
  const int slot = batch ? a.row_slot[r] : a.carry_slot[r - a.n_batch];
  const int half = a.hd / 2;
  const float* src = a.y + static_cast<size_t>(r) * qkv_n;
  // one thread per (head, rotation pair); v heads copy both halves
  for (int t = threadIdx.x; t < (a.n_q + 2 * a.n_kv) * half; t += blockDim.x) {
    const int head = t / half, j = t % half;
    const float x1 = src[head * a.hd + j], x2 = src[head * a.hd + half + j];
    float y1 = x1, y2 = x2;
    if (head < a.n_q + a.n_kv) {
      const float c = a.cos[static_cast<size_t>(pos) * half + j];
      const float s = a.sin[static_cast<size_t>(pos) * half + j];
      y1 = x1 * c - x2 * s;
      y2 = x2 * c + x1 * s;
    }
    float* dst;
    if (!batch) {
      dst = a.ship + static_cast<size_t>(slot) * qkv_n + head * a.hd;
    } else if (head < a.n_q) {
      dst = a.q + static_cast<size_t>(r) * nqh + head * a.hd;
    } else {
      const int kv = head < a.n_q + a.n_kv ? 0 : 1;
      const int kh = head - a.n_q - kv * a.n_kv;
      const int phys = a.page_table[static_cast<size_t>(slot) * a.pt_stride + pos / kPageTokens];
      dst = a.pool + (kv_row(a.g, a.layer, phys, kv, kh) + pos % kPageTokens) * a.hd;
    }
    dst[j] = y1;
    dst[half + j] = y2;
  }
}

// Attention of batch row r, query head h over the request's keys [0, pos]:
// decode rows (pos = ctx, ctx+1 keys, engine.py:675) and causal chunk rows
// alike.  Flash-style over 128-key tiles: warps score keys (lanes split the
// head dim), then thread e < hd accumulates output feature e.
__global__ void __launch_bounds__(128)
    attn_f32_kernel(const float* __restrict__ q, int n_q, int n_kv, int hd,
                    const float* __restrict__ pool, KvGeom g, int layer,
                    const int* __restrict__ page_table, int pt_stride,
                    const int* __restrict__ row_pos, const int* __restrict__ row_slot,
                    float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  constexpr int kTile = 128;
  __shared__ float qs[128];
  __shared__ float sc[kTile];
  __shared__ float red[4];
  const int r = blockIdx.x, h = blockIdx.y;
  const int kvh = h / (n_q / n_kv);
  const int pos = row_pos[r], slot = row_slot[r];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* qr = q + static_cast<size_t>(r) * n_q * hd + h * hd;
  for (int e = threadIdx.x; e < hd; e += blockDim.x) qs[e] = qr[e];
  __syncthreads();
  const float scale = rsqrtf(static_cast<float>(hd));
  float m = -CUDART_INF_F, l = 0.f, acc = 0.f;
  const int* pt = page_table + static_cast<size_t>(slot) * pt_stride;
  for (int t0 = 0; t0 <= pos; t0 += kTile) {
    const int nt = min(kTile, pos + 1 - t0);
    for (int j = warp; j < nt; j += 4) {
      const int key = t0 + j;
      const float* kr = pool + (kv_row(g, layer, pt[key / kPageTokens], 0, kvh) +
                                key % kPageTokens) * hd;
      float dot = 0.f;
      for (int e = lane; e < hd; e += 32) dot = fmaf(qs[e], kr[e], dot);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (lane == 0) sc[j] = dot * scale;
    }
    __syncthreads();
    // tile max
    float tm = -CUDART_INF_F;
    for (int j = threadIdx.x; j < nt; j += blockDim.x) tm = fmaxf(tm, sc[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
    if (lane == 0) red[warp] = tm;
    __syncthreads();
    tm = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    const float mn = fmaxf(m, tm);
    const float corr = expf(m - mn);
    l *= corr;
    acc *= corr;
    for (int j = 0; j < nt; ++j) {
      const float p = expf(sc[j] - mn);
      l += p;
      if (threadIdx.x < hd) {
        const int key = t0 + j;
        const float* vr = pool + (kv_row(g, layer, pt[key / kPageTokens], 1, kvh) +
                                  key % kPageTokens) * hd;
        acc = fmaf(p, vr[threadIdx.x], acc);
      }
    }
    m = mn;
    __syncthreads();  // sc / red reused by the next tile
  }
  if (threadIdx.x < hd) out[static_cast<size_t>(r) * n_q * hd + h * hd + threadIdx.x] = acc / l;
}

__global__ void silu_f32_kernel(const float* __restrict__ gu, int ffn, float* __restrict__ act) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.y;
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= ffn) return;
  const float g = gu[static_cast<size_t>(r) * 2 * ffn + f];
  const float u = gu[static_cast<size_t>(r) * 2 * ffn + ffn + f];
  act[static_cast<size_t>(r) * ffn + f] = g / (1.f + expf(-g)) * u;
}

}  // namespace
}  // namespace hs

#define RCF(x)                                                                             \
  do {                                                                                     \
    const int rc_ = (x);                                                                   \
    if (rc_ != HS_OK)                                                                      \
      return hs::set_error(rc_, "%s:%d %s: %s", __FILE__, __LINE__, #x,                    \
                           cudaGetErrorString(cudaGetLastError()));                        \
  } while (0)

int layer_f32(hs_ctx* c, const hs_layer_desc* d, const LayerRows& lr) {
  const ModelCfg& m = c->m;
  const int l = d->layer - 1;
  const int B = c->B, C = d->n_carry, M = d->n_merge, R = d->n_restart;
  const bool last = d->layer == m.layers;
  const int NL = last ? c->n_logit + M : 0;
  const int d_ = m.d, nqh = m.n_q * m.hd, qkv_n = m.qkv_n();
  cudaStream_t st = c->st;
  float* y = c->part;  // GEMM output [rows][n] (one plane)
  float* result_d = reinterpret_cast<float*>(c->result_d);
  float* ship_d = reinterpret_cast<float*>(c->ship_d);
  if (l == 0) {
    RCF(select_tokens(c->it_tok, c->it_slot, B, lr.carry_slot, c->last_token, B + C, c->tok, st));
    if (B + C > 0)
      RCF(launch_pdl(embed_f32_kernel, dim3(B + C), dim3(256), 0, st, c->tok, c->fw_embed, d_,
                     c->h));
    RCF(scatter_rows_f32(c->h + static_cast<size_t>(B) * d_, lr.carry_slot, C, d_, c->resid, st));
    RCF(add_norm_f32(nullptr, B + C, d_, c->h, c->n_in[0], m.eps, c->fx, st));
  }
  // QKV + RoPE / KV write / ship, and the merged rows' host results
  RCF(gemm_f32(c->fx, d_, B + C, c->fw_qkv[l], qkv_n, d_, y, st));
  RopeArgs ra{};
  ra.y = y;
  ra.rows = B + C;
  ra.n_batch = B;
  ra.n_q = m.n_q;
  ra.n_kv = m.n_kv;
  ra.hd = m.hd;
  ra.cos = c->rope_cos;
  ra.sin = c->rope_sin;
  ra.row_pos = c->it_pos;
  ra.row_slot = c->it_slot;
  ra.carry_pos = lr.carry_pos;
  ra.carry_slot = lr.carry_slot;
  ra.q = c->fq;
  ra.pool = c->kv_f32;
  ra.g = c->geom;
  ra.layer = l;
  ra.page_table = c->page_table;
  ra.pt_stride = c->r.max_pages_per_req;
  ra.ship = ship_d;
  ra.result = result_d;
  ra.merge_slot = lr.merge_slot;
  ra.n_merge = M;
  ra.attn_merged = c->fattn + static_cast<size_t>(B) * nqh;
  ra.expect = lr.merge_tag;
  ra.tags = c->tag_d;
  ra.fault = c->fault_d;
  ra.layer1 = d->layer;
  if (B + C + M > 0) RCF(launch_pdl(rope_f32_kernel, dim3(B + C + M), dim3(256), 0, st, ra));
  if (B > 0)
    RCF(launch_pdl(attn_f32_kernel, dim3(B, m.n_q), dim3(128), 0, st, c->fq, m.n_q, m.n_kv, m.hd,
                   c->kv_f32, c->geom, l, c->page_table, c->r.max_pages_per_req, c->it_pos,
                   c->it_slot, c->fattn));
  const int N = B + M;
  // Proj + ResidualAdd (+ the merged rows' residual get) + RMSNorm
  RCF(gemm_f32(c->fattn, nqh, N, c->fw_o[l], d_, nqh, y, st));
  RowIo io;
  io.src = c->resid;
  io.src_idx = M ? lr.merge_slot : nullptr;
  io.src_from = B;
  RCF(add_norm_f32(y, N, d_, c->h, c->n_post[l], m.eps, c->fx2, st, io));
  // MLP + ResidualAdd + the next layer's input norm (or the final norm);
  // chains merged here store their residual for the next layer's merge
  RCF(gemm_f32(c->fx2, d_, N, c->fw_gu[l], 2 * m.ffn, d_, y, st));
  if (N > 0)
    RCF(launch_pdl(silu_f32_kernel, dim3((m.ffn + 255) / 256, N), dim3(256), 0, st, y, m.ffn,
                   c->fact));
  RCF(gemm_f32(c->fact, m.ffn, N, c->fw_down[l], d_, m.ffn, y, st));
  RowIo io2;
  if (!last && M) {
    io2.put = c->resid;
    io2.put_idx = lr.merge_slot;
    io2.put_from = B;
  }
  RCF(add_norm_f32(y, N, d_, c->h, last ? c->w_final : c->n_in[l + 1], m.eps, c->fx, st, io2));
  if (!last) return HS_OK;
  // LM head + greedy token (engine.py:1005-1013, 1024-1047)
  RCF(gather_rows_f32(c->fx, lr.logit_rows, NL, d_, c->flin, st));
  RCF(gemm_f32(c->flin, d_, NL, c->fw_lm, m.vocab, d_, y, st));
  RCF(argmax_rows(y, Planes(1), NL, m.vocab, c->tok_out, c->keep_logits ? c->logits : nullptr, st));
  RCF(scatter_tokens(c->tok_out, lr.logit_slots, NL, c->last_token, st));
  c->n_tok_out = NL;
  c->merges_L = M;
  // chains continuing with their next token: embed, residual put, QKV(1), ship
  if (R > 0) {
    RCF(select_tokens(nullptr, nullptr, 0, lr.restart_slot, c->last_token, R, c->tok, st));
    RCF(launch_pdl(embed_f32_kernel, dim3(R), dim3(256), 0, st, c->tok, c->fw_embed, d_, c->hr));
    RCF(scatter_rows_f32(c->hr, lr.restart_slot, R, d_, c->resid, st));
    RCF(add_norm_f32(nullptr, R, d_, c->hr, c->n_in[0], m.eps, c->fxr, st));
    RCF(gemm_f32(c->fxr, d_, R, c->fw_qkv[0], qkv_n, d_, y, st));
    RopeArgs rr = ra;
    rr.rows = R;
    rr.n_batch = 0;
    rr.carry_pos = lr.restart_pos;
    rr.carry_slot = lr.restart_slot;
    rr.layer = 0;
    rr.n_merge = 0;
    rr.expect = nullptr;
    RCF(launch_pdl(rope_f32_kernel, dim3(R), dim3(256), 0, st, rr));
  }
  return HS_OK;
}
