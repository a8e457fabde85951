// K4/K5/K8/K9 and the split-K epilogues: the bandwidth-bound glue of one
// transformer layer.  Every kernel here reads the fp32 split-K partials the
// tcgen05 GEMM wrote and fuses the reduction with the operation that follows
// the projection (RoPE + KV-page scatter + piggyback ship after QKV;
// residual add + RMSNorm after O-proj / down-proj; SiLU*up after gate-up;
// greedy argmax after the LM head).
#include <math_constants.h>

#include <algorithm>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  float t = 0.f;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

// ---------------------------------------------------------------- embedding
__global__ void embed_kernel(const int* __restrict__ tokens, const bf16* __restrict__ emb, int d,
                             float* __restrict__ h) {
  const int r = blockIdx.x;
  const bf16* src = emb + static_cast<size_t>(tokens[r]) * d;
  float* dst = h + static_cast<size_t>(r) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = __bfloat162float(src[i]);
}

int embed_gather(const int* tokens, int rows, const bf16* emb, int d, float* h, cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  embed_kernel<<<rows, 256, 0, st>>>(tokens, emb, d, h);
  return launched();
}

// ---------------------------------------------------------------- RMSNorm
__global__ void rmsnorm_kernel(const float* __restrict__ h, int d, const float* __restrict__ w,
                               float eps, bf16* __restrict__ out, int ld_out) {
  __shared__ float red[32];
  const int r = blockIdx.x;
  const float* x = h + static_cast<size_t>(r) * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss += x[i] * x[i];
  const float inv = rsqrtf(block_sum(ss, red) / d + eps);
  bf16* o = out + static_cast<size_t>(r) * ld_out;
  for (int i = threadIdx.x; i < d; i += blockDim.x) o[i] = __float2bfloat16(x[i] * inv * w[i]);
}

int rmsnorm_rows(const float* h, int rows, int d, const float* w, float eps, bf16* out, int ld_out,
                 cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  rmsnorm_kernel<<<rows, 256, 0, st>>>(h, d, w, eps, out, ld_out);
  return launched();
}

// ---------------------------------------------------------------- split-K
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int splits, size_t total,
                                     float* __restrict__ out) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += part[k * total + i];
    out[i] = s;
  }
}

int splitk_reduce(const float* part, int splits, int rows, int n, float* out, cudaStream_t st) {
  const size_t total = static_cast<size_t>(rows) * n;
  if (!total) return HS_OK;
  const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, size_t(148 * 16)));
  splitk_reduce_kernel<<<blocks, 256, 0, st>>>(part, splits, total, out);
  return launched();
}

// h += sum_s part[s]; out = rmsnorm(h) * w   (out may be null)
__global__ void residual_add_norm_kernel(const float* __restrict__ part, int splits, int rows,
                                         int d, float* __restrict__ h, const float* __restrict__ w,
                                         float eps, bf16* __restrict__ out, int ld_out) {
  __shared__ float red[32];
  const int r = blockIdx.x;
  float* x = h + static_cast<size_t>(r) * d;
  const size_t plane = static_cast<size_t>(rows) * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float v = x[i];
    for (int k = 0; k < splits; ++k) v += part[k * plane + static_cast<size_t>(r) * d + i];
    x[i] = v;
    ss += v * v;
  }
  if (!out) return;
  const float inv = rsqrtf(block_sum(ss, red) / d + eps);
  bf16* o = out + static_cast<size_t>(r) * ld_out;
  for (int i = threadIdx.x; i < d; i += blockDim.x) o[i] = __float2bfloat16(x[i] * inv * w[i]);
}

int residual_add_norm(const float* part, int splits, int rows, int d, float* h, const float* w,
                      float eps, bf16* out, int ld_out, cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  residual_add_norm_kernel<<<rows, 256, 0, st>>>(part, splits, rows, d, h, w, eps, out, ld_out);
  return launched();
}

// ---------------------------------------------------------------- QKV epilogue
// Per row: reduce split-K partials of [q | k | v], rotate q and k
// (rotate-half RoPE from precomputed fp32 tables), then
//   mode 0: q -> qbuf row, k/v -> the request's KV page at position pos
//   mode 1: q/k/v -> the request's piggyback ship slot (pinned host memory,
//           mapped into the device address space: the D2H of Attention
//           Piggybacking, reference engine.py:982-989 _chain_qkv)
//   mode 2: q -> qbuf row, k/v -> ship slot (GPU attention of a row whose KV
//           lives on the host is not used; reserved)
__global__ void qkv_rope_scatter_kernel(const float* __restrict__ part, int splits, int rows,
                                        int n_q, int n_kv, int hd,
                                        const float* __restrict__ rope_cos,
                                        const float* __restrict__ rope_sin,
                                        const int* __restrict__ row_pos,
                                        const int* __restrict__ row_slot,
                                        const int* __restrict__ row_mode, bf16* __restrict__ qbuf,
                                        int q_row_stride, bf16* __restrict__ kv_pool, KvGeom geom,
                                        int layer, const int* __restrict__ page_table,
                                        int pt_stride, bf16* __restrict__ ship, int ship_stride) {
  const int r = blockIdx.x;
  const int n_tot = (n_q + 2 * n_kv) * hd;
  const size_t plane = static_cast<size_t>(rows) * n_tot;
  const float* src = part + static_cast<size_t>(r) * n_tot;
  const int pos = row_pos[r], slot = row_slot[r], mode = row_mode[r];
  const int half = hd / 2;
  const float* cs = rope_cos + static_cast<size_t>(pos) * half;
  const float* sn = rope_sin + static_cast<size_t>(pos) * half;
  bf16* kpage = nullptr;
  bf16* vpage = nullptr;
  if (mode == 0) {
    const int phys = page_table[static_cast<size_t>(slot) * pt_stride + pos / kPageTokens];
    const int t = pos % kPageTokens;
    kpage = kv_pool + (kv_row(geom, layer, phys, 0, 0) + t) * hd;
    vpage = kv_pool + (kv_row(geom, layer, phys, 1, 0) + t) * hd;
  }
  bf16* shp = mode == 1 ? ship + static_cast<size_t>(slot) * ship_stride : nullptr;
  // rotated pairs: q heads then k heads
  const int n_pairs = (n_q + n_kv) * half;
  for (int p = threadIdx.x; p < n_pairs; p += blockDim.x) {
    const int head = p / half, i = p % half;
    const int base = head * hd;
    float x1 = 0.f, x2 = 0.f;
    for (int k = 0; k < splits; ++k) {
      x1 += src[k * plane + base + i];
      x2 += src[k * plane + base + i + half];
    }
    const float c = cs[i], s = sn[i];
    const bf16 y1 = __float2bfloat16(x1 * c - x2 * s);
    const bf16 y2 = __float2bfloat16(x2 * c + x1 * s);
    if (mode == 1) {
      shp[base + i] = y1;
      shp[base + i + half] = y2;
    } else if (head < n_q) {
      bf16* qd = qbuf + static_cast<size_t>(r) * q_row_stride + base;
      qd[i] = y1;
      qd[i + half] = y2;
    } else {
      // kv page row for head kh: rows of one (page, kv, head) block are
      // contiguous; heads are 64 rows apart
      const int kh = head - n_q;
      bf16* kd = kpage + static_cast<size_t>(kh) * kPageTokens * hd;
      kd[i] = y1;
      kd[i + half] = y2;
    }
  }
  // v heads (no rotation)
  const int vbase = (n_q + n_kv) * hd;
  for (int e = threadIdx.x; e < n_kv * hd; e += blockDim.x) {
    float x = 0.f;
    for (int k = 0; k < splits; ++k) x += src[k * plane + vbase + e];
    const bf16 y = __float2bfloat16(x);
    if (mode == 1) {
      shp[vbase + e] = y;
    } else {
      const int kh = e / hd, i = e % hd;
      vpage[static_cast<size_t>(kh) * kPageTokens * hd + i] = y;
    }
  }
}

int qkv_rope_scatter(const float* part, int splits, int rows, int n_q, int n_kv, int head_dim,
                     const float* rope_cos, const float* rope_sin, const int* row_pos,
                     const int* row_slot, const int* row_mode, bf16* qbuf, int q_row_stride,
                     bf16* kv_pool, const KvGeom& g, int layer, const int* page_table,
                     int pt_stride, bf16* ship, int ship_stride, cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  qkv_rope_scatter_kernel<<<rows, 256, 0, st>>>(part, splits, rows, n_q, n_kv, head_dim, rope_cos,
                                                rope_sin, row_pos, row_slot, row_mode, qbuf,
                                                q_row_stride, kv_pool, g, layer, page_table,
                                                pt_stride, ship, ship_stride);
  return launched();
}

// ---------------------------------------------------------------- SwiGLU
__global__ void silu_mul_kernel(const float* __restrict__ part, int splits, int rows, int ffn,
                                bf16* __restrict__ act, int ld_act) {
  const size_t plane = static_cast<size_t>(rows) * 2 * ffn;
  const size_t total = static_cast<size_t>(rows) * ffn;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = idx / ffn, i = idx % ffn;
    const float* src = part + r * 2 * ffn;
    float gt = 0.f, up = 0.f;
    for (int k = 0; k < splits; ++k) {
      gt += src[k * plane + i];
      up += src[k * plane + ffn + i];
    }
    const float s = gt / (1.f + __expf(-gt));
    act[r * ld_act + i] = __float2bfloat16(s * up);
  }
}

int silu_mul(const float* part, int splits, int rows, int ffn, bf16* act, int ld_act,
             cudaStream_t st) {
  const size_t total = static_cast<size_t>(rows) * ffn;
  if (!total) return HS_OK;
  const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, size_t(148 * 16)));
  silu_mul_kernel<<<blocks, 256, 0, st>>>(part, splits, rows, ffn, act, ld_act);
  return launched();
}

// ---------------------------------------------------------------- greedy argmax
__global__ void argmax_kernel(const float* __restrict__ part, int splits, int rows, int vocab,
                              int* __restrict__ tokens, float* __restrict__ logits_out) {
  __shared__ float sv[32];
  __shared__ int si[32];
  const int r = blockIdx.x;
  const size_t plane = static_cast<size_t>(rows) * vocab;
  const float* src = part + static_cast<size_t>(r) * vocab;
  float best = -CUDART_INF_F;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < vocab; i += blockDim.x) {
    float v = 0.f;
    for (int k = 0; k < splits; ++k) v += src[k * plane + i];
    if (logits_out) logits_out[static_cast<size_t>(r) * vocab + i] = v;
    if (v > best || (v == best && i < bi)) {
      best = v;
      bi = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    for (int i = 1; i < nw; ++i)
      if (sv[i] > best || (sv[i] == best && si[i] < bi)) {
        best = sv[i];
        bi = si[i];
      }
    tokens[r] = bi;
  }
}

int argmax_rows(const float* part, int splits, int rows, int vocab, int* tokens, float* logits_out,
                cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  argmax_kernel<<<rows, 512, 0, st>>>(part, splits, rows, vocab, tokens, logits_out);
  return launched();
}

// ---------------------------------------------------------------- LSE merge
// Combines n_parts partial attention outputs (bf16, each normalised) with
// their natural-log LSEs into one bf16 output row: the merge step of
// Attention Piggybacking for host-computed partials (K2 on the piggyback
// path).  parts: [row][part][n_q*hd] (strides given), lse: [row][part][n_q].
template <int HD>
__global__ void lse_merge_kernel(const bf16* __restrict__ parts, const float* __restrict__ lse,
                                 int n_parts, int rows, int n_q, int part_stride,
                                 int row_stride_parts, bf16* __restrict__ out,
                                 int out_row_stride) {
  const int pair = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pair >= rows * n_q) return;
  const int r = pair / n_q, h = pair % n_q;
  const float* ls = lse + static_cast<size_t>(r) * n_parts * n_q;
  float mx = -CUDART_INF_F;
  for (int p = 0; p < n_parts; ++p) mx = fmaxf(mx, ls[p * n_q + h]);
  const float mu = mx == -CUDART_INF_F ? 0.f : mx;
  constexpr int PER = HD / 32;
  float acc[PER] = {};
  float ws = 0.f;
  for (int p = 0; p < n_parts; ++p) {
    const float w = __expf(ls[p * n_q + h] - mu);
    ws += w;
    const bf16* src =
        parts + static_cast<size_t>(r) * row_stride_parts + static_cast<size_t>(p) * part_stride +
        h * HD;
#pragma unroll
    for (int j = 0; j < PER; ++j) acc[j] += w * __bfloat162float(src[lane + 32 * j]);
  }
  const float inv = ws > 0.f ? 1.f / ws : 0.f;
  bf16* dst = out + static_cast<size_t>(r) * out_row_stride + h * HD;
#pragma unroll
  for (int j = 0; j < PER; ++j) dst[lane + 32 * j] = __float2bfloat16(acc[j] * inv);
}

int lse_merge_rows(const bf16* parts, const float* lse, int n_parts, int rows, int n_q,
                   int head_dim, int part_stride, int row_stride_parts, bf16* out,
                   int out_row_stride, cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  const int blocks = (rows * n_q + 3) / 4;
  if (head_dim == 128)
    lse_merge_kernel<128><<<blocks, 128, 0, st>>>(parts, lse, n_parts, rows, n_q, part_stride,
                                                  row_stride_parts, out, out_row_stride);
  else if (head_dim == 64)
    lse_merge_kernel<64><<<blocks, 128, 0, st>>>(parts, lse, n_parts, rows, n_q, part_stride,
                                                 row_stride_parts, out, out_row_stride);
  else
    return HS_E_CONFIG;
  return launched();
}

}  // namespace hs
