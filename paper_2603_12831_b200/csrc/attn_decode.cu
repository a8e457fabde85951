// K1 + K2: split-K paged flash-decoding over the GPU-resident KV pool.
//
// One CTA per (chunk of KV pages of one request, KV head).  KV pages
// ([64 tokens x head_dim] per head) are staged into shared memory by TMA
// (cp.async.bulk.tensor, SWIZZLE_128B boxes of 64 x 64) through a 3-stage
// mbarrier pipeline.  The GQA group of query heads that share the KV head
// forms the M=16 side of warp-level bf16 MMAs (QK^T and PV); the softmax is
// online per warp with quad shuffles, and the 4 warps (16 tokens of each
// page apiece) are merged through shared memory at the end.  Each CTA
// writes a normalised partial output and its log-sum-exp; decode_combine
// (K2) LSE-merges the partials of a request before the O projection.
//
// This is the work the reference charges as
// probe_attention(gpu, DECODE, attn_tokens, g) in Engine._run_layer
// (reference pkg/src/hybridserve/engine.py:939-942; loads accumulate ctx+1
// per decode at engine.py:675,740).  The kernel is HBM-bound: it reads
// sum(ctx+1) * 2 * n_kv * head_dim * 2 bytes per layer; the tensor-core
// instruction used for the tiny GQA tiles is irrelevant to that bound.
#include <math_constants.h>

#include <cooperative_groups.h>

#include <cstdlib>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace cg = cooperative_groups;

namespace hs {

#ifndef HS_DEC_STAGES
#define HS_DEC_STAGES 3
#endif
constexpr int kDecStages = HS_DEC_STAGES;
constexpr int kDecThreads = 128;

int make_kv_map(CUtensorMap* map, const bf16* pool, const KvGeom& g) {
  const uint64_t rows = static_cast<uint64_t>(g.layers) * g.pages * 2 * g.n_kv * kPageTokens;
  return make_map_2d_bf16(map, pool, g.head_dim, rows, static_cast<uint64_t>(g.head_dim) * 2, 64,
                          kPageTokens);
}

// WG warp groups of 4 warps: with WG = 2 the groups take alternate pages of
// the chunk (one CTA per SM for small batches, where the page loop's
// latency, not HBM, bounds the launch), with twice the stages in flight.
// CL > 1 (whole rows, small launches): the CL CTAs of a cluster split the
// chunk's pages into contiguous ranges and rank 0 LSE-merges their
// normalised partials through distributed shared memory.
template <int HD, int WG, int CL>
__global__ void __launch_bounds__(kDecThreads * WG, WG == 1 ? 2 : 1)
    decode_attn_kernel(const __grid_constant__ CUtensorMap kv_map, KvGeom geom, int layer,
                       const bf16* __restrict__ q, int q_row_stride, int n_q,
                       const int* __restrict__ page_table, int pt_stride,
                       const DecodeChunk* __restrict__ chunks, float* __restrict__ o_part,
                       float* __restrict__ lse_part, float scale_log2,
                       const int* __restrict__ row_chunk_begin, int* __restrict__ counters,
                       bf16* __restrict__ out, int out_row_stride) {
  constexpr int kBoxBytes = kPageTokens * 128;
  constexpr int kHalf = (HD / 64) * kBoxBytes;  // K (or V) of one page
  constexpr int kStageBytes = 2 * kHalf;
  constexpr int NT = HD / 8;   // output n-tiles
  constexpr int KS = HD / 16;  // k-steps over head_dim

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kStages = kDecStages * WG;
  constexpr int kThreads = kDecThreads * WG;
  constexpr int kWarps = 4 * WG;
  __shared__ uint64_t full[kStages];
  __shared__ float sm_m[kWarps][16], sm_l[kWarps][16];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int crank = CL > 1 ? static_cast<int>(blockIdx.x % CL) : 0;  // rank in the x-cluster
  const DecodeChunk ch = chunks[CL > 1 ? blockIdx.x / CL : blockIdx.x];
  const int kvh = blockIdx.y;
  const int G = n_q / geom.n_kv;
  // this CTA's pages: the chunk, or its crank-th contiguous range
  const int cpages = ch.page_end - ch.page_begin;
  const int cper = (cpages + CL - 1) / CL;
  const int p_lo = min(cpages, crank * cper);
  const int npages = min(cpages, p_lo + cper) - p_lo;
  const int page0 = ch.page_begin + p_lo;
  const int* pt = page_table + static_cast<size_t>(ch.slot) * pt_stride + page0;

  // the chunk's page ids, read once: the refill of a stage then issues its
  // TMA at once instead of waiting on a dependent global load per page (the
  // page table was uploaded ahead of the iteration: safe before the PDL wait)
  constexpr int kPtCache = 64;
  __shared__ int pt_s[kPtCache];
  for (int i = threadIdx.x; i < min(npages, kPtCache); i += kThreads) pt_s[i] = pt[i];
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&kv_map);
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int i) {
    const int s = i % kStages;
    const int phys = i < kPtCache ? pt_s[i] : pt[i];
    uint8_t* dst = smem + s * kStageBytes;
    mbar_expect_tx(&full[s], kStageBytes);
    const int rk = static_cast<int>(kv_row(geom, layer, phys, 0, kvh));
    const int rv = static_cast<int>(kv_row(geom, layer, phys, 1, kvh));
#pragma unroll
    for (int b = 0; b < HD / 64; ++b) {
      tma_load_2d(dst + b * kBoxBytes, &kv_map, &full[s], b * 64, rk);
      tma_load_2d(dst + kHalf + b * kBoxBytes, &kv_map, &full[s], b * 64, rv);
    }
  };
  // Before the previous kernel's results are visible (PDL): only pages that
  // cannot hold this layer's new token (position ctx-1, written by the QKV
  // epilogue just before) are safe to stream; the chunk list and the page
  // table were uploaded ahead of the iteration.
  const int safe = max(0, min(npages, (ch.ctx - 1) / kPageTokens - page0));
  const int first = min(kStages, npages);
  if (threadIdx.x == 0)
    for (int i = 0; i < min(first, safe); ++i) issue(i);
  pdl_enter();  // q and the new token's K/V are visible from here on
  if (threadIdx.x == 0)
    for (int i = min(first, safe); i < first; ++i) issue(i);

  // Q fragments (A operand, rows = query heads of this GQA group)
  uint32_t qa[KS][4];
  {
    const bf16* qrow = q + static_cast<size_t>(ch.row) * q_row_stride;
    const int h0 = kvh * G + g, h1 = kvh * G + g + 8;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int d0 = ks * 16 + tig * 2;
      uint32_t z = 0;
      qa[ks][0] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + h0 * HD + d0) : z;
      qa[ks][1] = g + 8 < G ? *reinterpret_cast<const uint32_t*>(qrow + h1 * HD + d0) : z;
      qa[ks][2] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + h0 * HD + d0 + 8) : z;
      qa[ks][3] = g + 8 < G ? *reinterpret_cast<const uint32_t*>(qrow + h1 * HD + d0 + 8) : z;
    }
  }

  float o[NT][4];
#pragma unroll
  for (int i = 0; i < NT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F, l0 = 0.f, l1 = 0.f;
  const int tb = (warp & 3) * 16;  // this warp's 16 tokens inside every page
  const int wg = warp >> 2;         // pages wg, wg + WG, ... are this group's

  for (int i0 = 0; i0 < npages; i0 += WG) {
   const int i = i0 + wg;
   if (i < npages) {
    const int s = i % kStages;
    mbar_wait(&full[s], (i / kStages) & 1);
    const int tok0 = (page0 + i) * kPageTokens + tb;
    if (tok0 < ch.ctx) {  // warp-uniform
      const uint32_t kbase = smem_u32(smem + s * kStageBytes);
      const uint32_t vbase = kbase + kHalf;
      float sc[2][4];
#pragma unroll
      for (int n = 0; n < 2; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
      {
        const int mi = lane >> 3, r = lane & 7;
        const int row = tb + (mi >> 1) * 8 + r;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(swz_addr(kbase, row, ks * 2 + (mi & 1)), b0, b1, b2, b3);
          mma_bf16_16816(sc[0], qa[ks], b0, b1);
          mma_bf16_16816(sc[1], qa[ks], b2, b3);
        }
      }
      // scale, mask, online softmax (rows g and g+8)
      float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        const int t = tok0 + n * 8 + tig * 2;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool ok = (t + (e & 1)) < ch.ctx;
          sc[n][e] = ok ? sc[n][e] * scale_log2 : -CUDART_INF_F;
        }
        mx0 = fmaxf(mx0, fmaxf(sc[n][0], sc[n][1]));
        mx1 = fmaxf(mx1, fmaxf(sc[n][2], sc[n][3]));
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      const float mu0 = mn0 == -CUDART_INF_F ? 0.f : mn0;
      const float mu1 = mn1 == -CUDART_INF_F ? 0.f : mn1;
      const float a0 = exp2f(m0 - mu0), a1 = exp2f(m1 - mu1);
      m0 = mn0;
      m1 = mn1;
      float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        sc[n][0] = exp2f(sc[n][0] - mu0);
        sc[n][1] = exp2f(sc[n][1] - mu0);
        sc[n][2] = exp2f(sc[n][2] - mu1);
        sc[n][3] = exp2f(sc[n][3] - mu1);
        rs0 += sc[n][0] + sc[n][1];
        rs1 += sc[n][2] + sc[n][3];
      }
      l0 = l0 * a0 + rs0;
      l1 = l1 * a1 + rs1;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        o[nt][0] *= a0;
        o[nt][1] *= a0;
        o[nt][2] *= a1;
        o[nt][3] *= a1;
      }
      uint32_t pa[4];
      pa[0] = pack_bf16x2(sc[0][0], sc[0][1]);
      pa[1] = pack_bf16x2(sc[0][2], sc[0][3]);
      pa[2] = pack_bf16x2(sc[1][0], sc[1][1]);
      pa[3] = pack_bf16x2(sc[1][2], sc[1][3]);
      {
        const int mi = lane >> 3, r = lane & 7;
        const int row = tb + (mi & 1) * 8 + r;
#pragma unroll
        for (int j = 0; j < NT / 2; ++j) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(swz_addr(vbase, row, 2 * j + (mi >> 1)), b0, b1, b2, b3);
          mma_bf16_16816(o[2 * j], pa, b0, b1);
          mma_bf16_16816(o[2 * j + 1], pa, b2, b3);
        }
      }
    }
   }
    __syncthreads();  // every warp is done with its stage
    if (threadIdx.x == 0)
      for (int j = i0 + kStages; j < i0 + kStages + WG && j < npages; ++j) issue(j);
  }

  // quad-reduce the row sums
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  if (tig == 0) {
    sm_m[warp][g] = m0;
    sm_m[warp][g + 8] = m1;
    sm_l[warp][g] = l0;
    sm_l[warp][g + 8] = l1;
  }
  __syncthreads();
  // cross-warp merge: rescale each warp's O to the common max, sum in smem
  float M0 = -CUDART_INF_F, M1 = -CUDART_INF_F;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    M0 = fmaxf(M0, sm_m[w][g]);
    M1 = fmaxf(M1, sm_m[w][g + 8]);
  }
  const float Mu0 = M0 == -CUDART_INF_F ? 0.f : M0, Mu1 = M1 == -CUDART_INF_F ? 0.f : M1;
  const float f0 = exp2f(m0 - Mu0), f1 = exp2f(m1 - Mu1);
  // [4 warps][16 rows][HD + 8]: the pad spreads the 8 row groups of a warp
  // over different banks
  constexpr int SO = HD + 8;
  float* so = reinterpret_cast<float*>(smem);
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int d = nt * 8 + tig * 2;
    *reinterpret_cast<float2*>(&so[(warp * 16 + g) * SO + d]) = make_float2(o[nt][0] * f0, o[nt][1] * f0);
    *reinterpret_cast<float2*>(&so[(warp * 16 + g + 8) * SO + d]) =
        make_float2(o[nt][2] * f1, o[nt][3] * f1);
  }
  __syncthreads();
  if constexpr (CL > 1) {
    // this CTA's normalised partial [G][HD] and its LSE (log2 units), then
    // rank 0 merges the cluster's partials out of the peers' shared memory
    float* s_o = so + kWarps * 16 * SO;
    __shared__ float s_lse[16];
    for (int idx = threadIdx.x; idx < G * HD; idx += kThreads) {
      const int r = idx / HD, d = idx % HD;
      float Mr = -CUDART_INF_F;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) Mr = fmaxf(Mr, sm_m[w][r]);
      const float Mur = Mr == -CUDART_INF_F ? 0.f : Mr;
      float L = 0.f, acc = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        L += sm_l[w][r] * exp2f(sm_m[w][r] - Mur);
        acc += so[(w * 16 + r) * SO + d];
      }
      s_o[idx] = L > 0.f ? acc / L : 0.f;
      if (d == 0) s_lse[r] = L > 0.f ? Mur + log2f(L) : -CUDART_INF_F;
    }
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    if (crank == 0) {
      for (int idx = threadIdx.x; idx < G * HD; idx += kThreads) {
        const int r = idx / HD, d = idx % HD;
        float lk[CL];
        float mx = -CUDART_INF_F;
#pragma unroll
        for (int k = 0; k < CL; ++k) {
          lk[k] = *cluster.map_shared_rank(&s_lse[r], k);
          mx = fmaxf(mx, lk[k]);
        }
        const float mu = mx == -CUDART_INF_F ? 0.f : mx;
        float ws = 0.f, acc = 0.f;
#pragma unroll
        for (int k = 0; k < CL; ++k) {
          const float w = exp2f(lk[k] - mu);
          ws += w;
          acc += w * *cluster.map_shared_rank(&s_o[idx], k);
        }
        out[static_cast<size_t>(ch.row) * out_row_stride + (kvh * G + r) * HD + d] =
            __float2bfloat16(ws > 0.f ? acc / ws : 0.f);
      }
    }
    cluster.sync();  // the peers' shared memory stays alive until rank 0 is done
    return;
  }
  const int base = (blockIdx.x * geom.n_kv + kvh) * G;
  const int c_lo = out ? row_chunk_begin[ch.row] : 0;
  const int n_row_chunks = out ? row_chunk_begin[ch.row + 1] - c_lo : 0;
  if (out && n_row_chunks == 1) {  // whole row in this CTA: normalise and store
    for (int idx = threadIdx.x; idx < G * HD; idx += kThreads) {
      const int r = idx / HD, d = idx % HD;
      float Mr = -CUDART_INF_F;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) Mr = fmaxf(Mr, sm_m[w][r]);
      const float Mur = Mr == -CUDART_INF_F ? 0.f : Mr;
      float L = 0.f, acc = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        L += sm_l[w][r] * exp2f(sm_m[w][r] - Mur);
        acc += so[(w * 16 + r) * SO + d];
      }
      out[static_cast<size_t>(ch.row) * out_row_stride + (kvh * G + r) * HD + d] =
          __float2bfloat16(L > 0.f ? acc / L : 0.f);
    }
    return;
  }
  for (int idx = threadIdx.x; idx < G * HD; idx += kThreads) {
    const int r = idx / HD, d = idx % HD;
    float Mr = -CUDART_INF_F;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) Mr = fmaxf(Mr, sm_m[w][r]);
    const float Mur = Mr == -CUDART_INF_F ? 0.f : Mr;
    float L = 0.f, acc = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      L += sm_l[w][r] * exp2f(sm_m[w][r] - Mur);
      acc += so[(w * 16 + r) * SO + d];
    }
    o_part[static_cast<size_t>(base + r) * HD + d] = L > 0.f ? acc / L : 0.f;
    if (d == 0)
      lse_part[base + r] = L > 0.f ? (Mur + log2f(L)) * 0.69314718055994530942f : -CUDART_INF_F;
  }
  if (!out) return;
  // fused K2: the last CTA of this (row, KV head) merges the row's chunks
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(&counters[ch.row * geom.n_kv + kvh], 1);
    s_last = prev == n_row_chunks - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // every chunk's LSE of this (row, KV head) into smem with independent
  // loads, per-head weights, then the weighted sum with 4 loads in flight
  float* s_w = reinterpret_cast<float*>(smem);  // [n_row_chunks][G]
  float* s_inv = s_w + n_row_chunks * G;        // [G]
  for (int i = threadIdx.x; i < n_row_chunks * G; i += kThreads) {
    const int c = c_lo + i / G, r = i % G;
    s_w[i] = __ldcg(&lse_part[(c * geom.n_kv + kvh) * G + r]);
  }
  __syncthreads();
  if (threadIdx.x < G) {
    const int r = threadIdx.x;
    float mx = -CUDART_INF_F;
    for (int c = 0; c < n_row_chunks; ++c) mx = fmaxf(mx, s_w[c * G + r]);
    const float mu = mx == -CUDART_INF_F ? 0.f : mx;
    float ws = 0.f;
    for (int c = 0; c < n_row_chunks; ++c) {
      const float w = __expf(s_w[c * G + r] - mu);
      s_w[c * G + r] = w;
      ws += w;
    }
    s_inv[r] = ws > 0.f ? 1.f / ws : 0.f;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * HD; idx += kThreads) {
    const int r = idx / HD, d = idx % HD;
    const float* src = o_part + (static_cast<size_t>(c_lo * geom.n_kv + kvh) * G + r) * HD + d;
    const size_t cstride = static_cast<size_t>(geom.n_kv) * G * HD;
    float acc = 0.f;
    int c = 0;
    for (; c + 4 <= n_row_chunks; c += 4) {
      const float v0 = __ldcg(src + c * cstride), v1 = __ldcg(src + (c + 1) * cstride),
                  v2 = __ldcg(src + (c + 2) * cstride), v3 = __ldcg(src + (c + 3) * cstride);
      acc += s_w[c * G + r] * v0;
      acc += s_w[(c + 1) * G + r] * v1;
      acc += s_w[(c + 2) * G + r] * v2;
      acc += s_w[(c + 3) * G + r] * v3;
    }
    for (; c < n_row_chunks; ++c) acc += s_w[c * G + r] * __ldcg(src + c * cstride);
    out[static_cast<size_t>(ch.row) * out_row_stride + (kvh * G + r) * HD + d] =
        __float2bfloat16(acc * s_inv[r]);
  }
  if (threadIdx.x == 0) counters[ch.row * geom.n_kv + kvh] = 0;  // ready for the next launch
}

// K2: merge the split partials of each (row, query head).  One warp per pair.
template <int HD>
__global__ void decode_combine_kernel(const float* __restrict__ o_part,
                                      const float* __restrict__ lse_part,
                                      const int* __restrict__ row_chunk_begin, int rows, int n_q,
                                      int n_kv, bf16* __restrict__ out, int out_row_stride,
                                      float* __restrict__ lse_out) {
  pdl_enter();  // dependent data of the previous kernel is visible
  const int pair = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pair >= rows * n_q) return;
  const int row = pair / n_q, h = pair % n_q;
  const int G = n_q / n_kv;
  const int kvh = h / G, gi = h % G;
  const int c0 = row_chunk_begin[row], c1 = row_chunk_begin[row + 1];
  float mx = -CUDART_INF_F;
  for (int c = c0; c < c1; ++c) mx = fmaxf(mx, lse_part[(c * n_kv + kvh) * G + gi]);
  const float mu = mx == -CUDART_INF_F ? 0.f : mx;
  constexpr int PER = HD / 32;
  float acc[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) acc[j] = 0.f;
  float wsum = 0.f;
  for (int c = c0; c < c1; ++c) {
    const int idx = (c * n_kv + kvh) * G + gi;
    const float w = __expf(lse_part[idx] - mu);
    wsum += w;
    const float* src = o_part + static_cast<size_t>(idx) * HD;
#pragma unroll
    for (int j = 0; j < PER; ++j) acc[j] += w * src[lane + 32 * j];
  }
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
  bf16* dst = out + static_cast<size_t>(row) * out_row_stride + h * HD;
#pragma unroll
  for (int j = 0; j < PER; ++j) dst[lane + 32 * j] = __float2bfloat16(acc[j] * inv);
  if (lse_out && lane == 0) lse_out[pair] = wsum > 0.f ? mu + logf(wsum) : -CUDART_INF_F;
}

template <int HD, int WG, int CL = 1>
static int launch_decode_wg(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
                            int q_row_stride, int n_q, const int* pt, int pt_stride,
                            const DecodeChunk* chunks, int n_chunks, float* o_part,
                            float* lse_part, cudaStream_t st, const int* row_chunk_begin,
                            int* counters, bf16* out, int out_row_stride) {
  constexpr int kStageBytes = 2 * (HD / 64) * kPageTokens * 128;
  constexpr int kSmem = kDecStages * WG * kStageBytes + 1024;
  static_assert(4 * WG * 16 * (HD + 8) * 4 + 16 * HD * 4 <= kDecStages * WG * kStageBytes,
                "merge scratch must fit");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_attn_kernel<HD, WG, CL>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    attr = true;
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(HD));
  dim3 grid(n_chunks * CL, g.n_kv);
  if (CL > 1)
    return launch_pdl_cluster(decode_attn_kernel<HD, WG, CL>, dim3(grid), dim3(kDecThreads * WG),
                              kSmem, st, CL, kv_map, g, layer, q, q_row_stride, n_q, pt,
                              pt_stride, chunks, o_part, lse_part, scale_log2, row_chunk_begin,
                              counters, out, out_row_stride);
  return launch_pdl(decode_attn_kernel<HD, WG, CL>, dim3(grid), dim3(kDecThreads * WG), kSmem, st,
                    kv_map, g, layer, q, q_row_stride, n_q, pt, pt_stride, chunks, o_part,
                    lse_part, scale_log2, row_chunk_begin, counters, out, out_row_stride);
}

// Two warp groups per CTA when the launch is at most one CTA per SM (small
// batches, latency-bound page loops); one group otherwise (HS_DEC_WG=1/2
// forces it, tuning knob).
template <int HD>
static int launch_decode(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
                         int q_row_stride, int n_q, const int* pt, int pt_stride,
                         const DecodeChunk* chunks, int n_chunks, float* o_part, float* lse_part,
                         cudaStream_t st, const int* row_chunk_begin = nullptr,
                         int* counters = nullptr, bf16* out = nullptr, int out_row_stride = 0,
                         bool rows_whole = false) {
  static const int forced = [] {
    const char* e = getenv("HS_DEC_WG");
    return e ? atoi(e) : 0;
  }();
  static const int cl_max = [] {
    const char* e = getenv("HS_DEC_CLUSTER");
    return e ? atoi(e) : 4;
  }();
  // whole rows of a launch that leaves SMs idle: a cluster per chunk
  const int ctas = n_chunks * g.n_kv;
  if (out && rows_whole && !forced) {
    if (cl_max >= 4 && 4 * ctas <= 148)
      return launch_decode_wg<HD, 2, 4>(kv_map, g, layer, q, q_row_stride, n_q, pt, pt_stride,
                                        chunks, n_chunks, o_part, lse_part, st, row_chunk_begin,
                                        counters, out, out_row_stride);
    if (cl_max >= 2 && 2 * ctas <= 148)
      return launch_decode_wg<HD, 2, 2>(kv_map, g, layer, q, q_row_stride, n_q, pt, pt_stride,
                                        chunks, n_chunks, o_part, lse_part, st, row_chunk_begin,
                                        counters, out, out_row_stride);
  }
  const bool two = forced ? forced == 2 : ctas <= 148;
  if (two)
    return launch_decode_wg<HD, 2>(kv_map, g, layer, q, q_row_stride, n_q, pt, pt_stride, chunks,
                                   n_chunks, o_part, lse_part, st, row_chunk_begin, counters, out,
                                   out_row_stride);
  return launch_decode_wg<HD, 1>(kv_map, g, layer, q, q_row_stride, n_q, pt, pt_stride, chunks,
                                 n_chunks, o_part, lse_part, st, row_chunk_begin, counters, out,
                                 out_row_stride);
}

int decode_attention(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
                     int q_row_stride, int n_q, const int* page_table, int pt_stride,
                     const DecodeChunk* chunks, int n_chunks, float* o_part, float* lse_part,
                     cudaStream_t st) {
  if (n_chunks <= 0) return HS_OK;
  if (n_q % g.n_kv || n_q / g.n_kv > 16) return HS_E_CONFIG;
  if (g.head_dim == 128)
    return launch_decode<128>(kv_map, g, layer, q, q_row_stride, n_q, page_table, pt_stride,
                              chunks, n_chunks, o_part, lse_part, st);
  if (g.head_dim == 64)
    return launch_decode<64>(kv_map, g, layer, q, q_row_stride, n_q, page_table, pt_stride, chunks,
                             n_chunks, o_part, lse_part, st);
  return HS_E_CONFIG;
}

int decode_attention_fused(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
                           int q_row_stride, int n_q, const int* page_table, int pt_stride,
                           const DecodeChunk* chunks, int n_chunks, const int* row_chunk_begin,
                           float* o_part, float* lse_part, int* counters, bf16* out,
                           int out_row_stride, cudaStream_t st, bool rows_whole) {
  if (n_chunks <= 0) return HS_OK;
  if (n_q % g.n_kv || n_q / g.n_kv > 16) return HS_E_CONFIG;
  if (g.head_dim == 128)
    return launch_decode<128>(kv_map, g, layer, q, q_row_stride, n_q, page_table, pt_stride,
                              chunks, n_chunks, o_part, lse_part, st, row_chunk_begin, counters,
                              out, out_row_stride, rows_whole);
  if (g.head_dim == 64)
    return launch_decode<64>(kv_map, g, layer, q, q_row_stride, n_q, page_table, pt_stride, chunks,
                             n_chunks, o_part, lse_part, st, row_chunk_begin, counters, out,
                             out_row_stride, rows_whole);
  return HS_E_CONFIG;
}

int decode_combine(const float* o_part, const float* lse_part, const int* row_chunk_begin,
                   int rows, int n_q, int n_kv, int head_dim, bf16* out, int out_row_stride,
                   float* lse_out, cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  const int blocks = (rows * n_q + 3) / 4;
  if (head_dim == 128)
    return launch_pdl(decode_combine_kernel<128>, dim3(blocks), dim3(128), 0, st, o_part,
                      lse_part, row_chunk_begin, rows, n_q, n_kv, out, out_row_stride, lse_out);
  if (head_dim == 64)
    return launch_pdl(decode_combine_kernel<64>, dim3(blocks), dim3(128), 0, st, o_part, lse_part,
                      row_chunk_begin, rows, n_q, n_kv, out, out_row_stride, lse_out);
  return HS_E_CONFIG;
}

}  // namespace hs
