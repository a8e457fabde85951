// K6: causal chunked-prefill attention over the paged KV pool -- the
// warp-MMA (mma.sync) version, kept as the A/B baseline of the tcgen05
// kernel in attn_prefill_tc.cu (HS_PREFILL_MMA=1 selects it).
//
// One CTA per (tile of <= 64 query tokens of one request, query head); warp w
// owns query rows 16w..16w+15.  The chunk's own K/V were scattered into the
// pool by the QKV epilogue, so every key (context and chunk) is read through
// the same TMA page path as decode.  Flash-attention-2 style online softmax
// with bf16 warp MMAs and fp32 accumulators.
//
// This is the work the reference charges as
// probe_attention(gpu, PREFILL, prefill_units) (reference
// pkg/src/hybridserve/engine.py:935-938), with prefill_units =
// pairwise_units(done, q) = q*(2*done+q+1)/2 attended pairs
// (scheduling.py:127-133).
#include <math_constants.h>

#include <cstdlib>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

constexpr int kPreStages = 2;
constexpr int kPreThreads = 128;

template <int HD>
__global__ void __launch_bounds__(kPreThreads)
    prefill_attn_kernel(const __grid_constant__ CUtensorMap kv_map, KvGeom geom, int layer,
                        const bf16* __restrict__ q, int q_row_stride, int n_q,
                        const int* __restrict__ page_table, int pt_stride,
                        const PrefillTile* __restrict__ tiles, bf16* __restrict__ out,
                        int out_row_stride, float scale_log2) {
  pdl_wait();  // dependent data of the previous kernel is visible
  pdl_trigger();
  constexpr int kBoxBytes = kPageTokens * 128;
  constexpr int kHalf = (HD / 64) * kBoxBytes;
  constexpr int kStageBytes = 2 * kHalf;
  constexpr int NT = HD / 8;
  constexpr int KS = HD / 16;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kPreStages];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const PrefillTile tile = tiles[blockIdx.x];
  const int h = blockIdx.y;
  const int G = n_q / geom.n_kv;
  const int kvh = h / G;
  const int kv_len = tile.pos0 + tile.nq;  // causal limit of the tile
  const int npages = (kv_len + kPageTokens - 1) / kPageTokens;
  const int* pt = page_table + static_cast<size_t>(tile.slot) * pt_stride;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&kv_map);
    for (int s = 0; s < kPreStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int i) {
    const int s = i % kPreStages;
    const int phys = pt[i];
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
  if (threadIdx.x == 0)
    for (int i = 0; i < min(kPreStages, npages); ++i) issue(i);

  // query rows of this warp: r0 = 16w + g, r1 = r0 + 8
  const int r0 = warp * 16 + g, r1 = r0 + 8;
  const int p0 = tile.pos0 + r0, p1 = tile.pos0 + r1;  // absolute positions
  const bool v0 = r0 < tile.nq, v1 = r1 < tile.nq;
  uint32_t qa[KS][4];
  {
    const bf16* q0 = q + static_cast<size_t>(tile.q_row + r0) * q_row_stride + h * HD;
    const bf16* q1 = q + static_cast<size_t>(tile.q_row + r1) * q_row_stride + h * HD;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int d0 = ks * 16 + tig * 2;
      qa[ks][0] = v0 ? *reinterpret_cast<const uint32_t*>(q0 + d0) : 0u;
      qa[ks][1] = v1 ? *reinterpret_cast<const uint32_t*>(q1 + d0) : 0u;
      qa[ks][2] = v0 ? *reinterpret_cast<const uint32_t*>(q0 + d0 + 8) : 0u;
      qa[ks][3] = v1 ? *reinterpret_cast<const uint32_t*>(q1 + d0 + 8) : 0u;
    }
  }
  float o[NT][4];
#pragma unroll
  for (int i = 0; i < NT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F, l0 = 0.f, l1 = 0.f;
  const int warp_last_pos = tile.pos0 + min(warp * 16 + 15, tile.nq - 1);

  for (int i = 0; i < npages; ++i) {
    const int s = i % kPreStages;
    mbar_wait(&full[s], (i / kPreStages) & 1);
    const int kbase_tok = i * kPageTokens;
    if (warp * 16 < tile.nq && kbase_tok <= warp_last_pos) {  // warp-uniform
      const uint32_t kbase = smem_u32(smem + s * kStageBytes);
      const uint32_t vbase = kbase + kHalf;
      float sc[8][4];
#pragma unroll
      for (int n = 0; n < 8; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
      const int mi = lane >> 3, rr = lane & 7;
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // pairs of key n-tiles (16 keys)
        const int row = np * 16 + (mi >> 1) * 8 + rr;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(swz_addr(kbase, row, ks * 2 + (mi & 1)), b0, b1, b2, b3);
          mma_bf16_16816(sc[2 * np], qa[ks], b0, b1);
          mma_bf16_16816(sc[2 * np + 1], qa[ks], b2, b3);
        }
      }
      float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        const int kp = kbase_tok + n * 8 + tig * 2;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = kp + (e & 1);
          const bool ok = (e < 2) ? (v0 && key <= p0) : (v1 && key <= p1);
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
      for (int n = 0; n < 8; ++n) {
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
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {  // 16 keys per k-step
        uint32_t pa[4];
        pa[0] = pack_bf16x2(sc[2 * kk][0], sc[2 * kk][1]);
        pa[1] = pack_bf16x2(sc[2 * kk][2], sc[2 * kk][3]);
        pa[2] = pack_bf16x2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
        pa[3] = pack_bf16x2(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
        const int row = kk * 16 + (mi & 1) * 8 + rr;
#pragma unroll
        for (int j = 0; j < NT / 2; ++j) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(swz_addr(vbase, row, 2 * j + (mi >> 1)), b0, b1, b2, b3);
          mma_bf16_16816(o[2 * j], pa, b0, b1);
          mma_bf16_16816(o[2 * j + 1], pa, b2, b3);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && i + kPreStages < npages) issue(i + kPreStages);
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  bf16* o0 = out + static_cast<size_t>(tile.q_row + r0) * out_row_stride + h * HD;
  bf16* o1 = out + static_cast<size_t>(tile.q_row + r1) * out_row_stride + h * HD;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int d = nt * 8 + tig * 2;
    if (v0) *reinterpret_cast<uint32_t*>(o0 + d) = pack_bf16x2(o[nt][0] * inv0, o[nt][1] * inv0);
    if (v1) *reinterpret_cast<uint32_t*>(o1 + d) = pack_bf16x2(o[nt][2] * inv1, o[nt][3] * inv1);
  }
}

template <int HD>
static int launch_prefill(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
                          int q_row_stride, int n_q, const int* pt, int pt_stride,
                          const PrefillTile* tiles, int n_tiles, bf16* out, int out_row_stride,
                          cudaStream_t st) {
  constexpr int kSmem = kPreStages * 2 * (HD / 64) * kPageTokens * 128 + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(prefill_attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSmem);
    attr = true;
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(HD));
  dim3 grid(n_tiles, n_q);
  return launch_pdl(prefill_attn_kernel<HD>, dim3(grid), dim3(kPreThreads), kSmem, st, kv_map, g, layer, q, q_row_stride, n_q, pt, pt_stride, tiles, out, out_row_stride,
      scale_log2);
}

// HS_PREFILL_MMA=1 (probe knob, read once): the warp-MMA kernel below
// instead of the tcgen05 one (attn_prefill_tc.cu), for A/B measurements.
static bool use_warp_mma() {
  static const bool v = [] {
    const char* e = std::getenv("HS_PREFILL_MMA");
    return e && std::atoi(e) != 0;
  }();
  return v;
}

int prefill_attention(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
                      int q_row_stride, int n_q, const int* page_table, int pt_stride,
                      const PrefillTile* tiles, int n_tiles, bf16* out, int out_row_stride,
                      cudaStream_t st) {
  if (n_tiles <= 0) return HS_OK;
  if (!use_warp_mma() && n_q % g.n_kv == 0 && n_q / g.n_kv <= 8)
    return prefill_attention_tc(kv_map, g, layer, q, q_row_stride, n_q, page_table, pt_stride,
                                tiles, n_tiles, out, out_row_stride, st);
  if (n_q % g.n_kv) return HS_E_CONFIG;
  if (g.head_dim == 128)
    return launch_prefill<128>(kv_map, g, layer, q, q_row_stride, n_q, page_table, pt_stride,
                               tiles, n_tiles, out, out_row_stride, st);
  if (g.head_dim == 64)
    return launch_prefill<64>(kv_map, g, layer, q, q_row_stride, n_q, page_table, pt_stride, tiles,
                              n_tiles, out, out_row_stride, st);
  return HS_E_CONFIG;
}

}  // namespace hs
