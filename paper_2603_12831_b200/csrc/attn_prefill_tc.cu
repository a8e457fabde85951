// K6 on the 5th-generation tensor cores: causal chunked-prefill attention
// over the paged KV pool with tcgen05.mma, TMEM accumulators and TMA-staged
// KV pages.
//
// The reference charges this work as probe_attention(gpu, PREFILL,
// prefill_units) with prefill_units = pairwise_units(done, q) =
// q*(2*done+q+1)/2 attended (query, key) pairs
// (pkg/src/hybridserve/engine.py:935-938, scheduling.py:127-133): 4*n_q*hd
// flops per pair, the step's only tensor-bound attention.
//
// One CTA per (block of query tokens of one prefill tile, KV head).  The
// MMA rows pack every query head of the KV head's GQA group: row = token * G
// + g (G = n_q / n_kv), so each KV page is read once per group instead of
// once per query head; a CTA holds NT = 1 or 2 Q tiles of 128 rows (2 when
// the launch still fills every SM: two tiles share each staged page, half
// the KV traffic per flop).  Keys go in blocks of 128 (two KV pages staged
// side by side by TMA).  Per key block j and Q tile t:
//
//   S_j = Q_t K_j^T    tcgen05.mma M=128 N=128 K=hd into the tile's 128 TMEM
//                      columns (A = Q K-major smem, B = the two K pages)
//   P_j = exp2(S_j*scale - m), one TMEM lane (row) per thread of the tile's
//         four warps (one FFMA + one MUFU.EX2 per score, the row sum over
//         the fp32 P), written back as bf16 pairs into the first 64 of those
//         columns (tcgen05.st)
//   O_t += P_j V_j     tcgen05.mma M=128 N=hd K=128 with A = P read from
//                      TMEM and B = the V pages (MN-major), accumulated in
//                      TMEM; then S_{j+1} of the same tile is issued into the
//                      same columns (MMAs run in issue order)
//
// The two tiles alternate on the tensor pipe: while one tile's warps run
// the softmax of block j, the other tile's P.V and next S execute (N = 128
// S tiles run the tensor pipe at full rate; N = 64 ran at half).  The
// running max m only moves when a row's max grows by more than 2^8 (lazy
// rescaling): P <= 256 stays exact enough in bf16 and O in TMEM is rescaled
// (tcgen05.ld / st) only on those rare blocks.  The last warp issues the TMA
// loads (2-stage ring of 128-key blocks) and, from one thread, every MMA.
// One CTA per SM (192 KB of shared memory, 512 TMEM columns).
#include <math_constants.h>

#include <algorithm>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

#ifdef HS_K6_TRACE
// diagnostic build only (HS_NVCC_DEFS=-DHS_K6_TRACE): SM clock stamps of the
// page handoffs of CTA (0, 0), read back with hs_debug_k6_trace
__device__ long long g_k6_trace[8][128];
#define K6T(ev, i)                                                              \
  do {                                                                          \
    if (blockIdx.x == 0 && blockIdx.y == 0 && (i) < 128) g_k6_trace[ev][i] = clock64(); \
  } while (0)
#else
#define K6T(ev, i) \
  do {             \
  } while (0)
#endif

namespace {

constexpr int kTcStages = 2;   // 128-key blocks of K and V in flight (64 KB each at hd 128)
constexpr int kBlkKeys = 128;  // keys per S tile (two KV pages): N = 128 per S MMA
constexpr int kMaxTiles = 2;            // Q tiles of 128 rows sharing each KV page
constexpr int kTcSoftmaxThreads = 128;  // per tile: warps 4t..4t+3, one TMEM lane (row) each
constexpr int kRows = 128;              // MMA M
constexpr float kRescaleLog2 = 8.0f;    // lazy-rescale threshold (P <= 2^8)

// TMEM columns with NT tiles: S of tile t (128 fp32 columns, later P_j as 64
// columns of bf16 pairs), then O (NT x 128)
template <int NT>
__host__ __device__ constexpr int s_col(int t) { return t * kBlkKeys; }
template <int NT>
__host__ __device__ constexpr int o_col(int t) { return NT * 128 + t * 128; }
template <int NT>
constexpr int kTmemCols = NT * 256;

// MN-major SWIZZLE_128B operand (the V page as staged by TMA: keys are
// rows of 128 B holding 64 hd elements): LBO = byte distance between
// 64-element chunks along N (the next TMA box), SBO = 1024 B between
// 8-key groups along K.
__device__ __forceinline__ uint64_t umma_desc_mn128(uint32_t smem_addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

// one MUFU.EX2 (subnormal results flush to 0, far below bf16 P's resolution)
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 32 lanes x 16 columns, no wait (batch several, then tmem_wait_ld)
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]: the A operand (M = 128 lanes x K = 16,
// bf16 pairs in 8 consecutive 32-bit columns) read from tensor memory
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

template <int HD, int NT>
__global__ void __launch_bounds__(NT * kTcSoftmaxThreads + 32, 1)
    prefill_attn_tc_kernel(const __grid_constant__ CUtensorMap kv_map, KvGeom geom, int layer,
                           const bf16* __restrict__ q, int q_row_stride, int n_q,
                           const int* __restrict__ page_table, int pt_stride,
                           const PrefillTile* __restrict__ tiles, int blocks_per_tile,
                           bf16* __restrict__ out, int out_row_stride, float scale_log2) {
  constexpr int kBox = kPageTokens * 128;          // one [64 keys][64 el] SW128 box
  constexpr int kChunk = kBlkKeys * 128;           // [128 keys][64 el]: two pages of a chunk
  constexpr int kKvBytes = (HD / 64) * kChunk;     // K or V of one key block
  constexpr int kStageBytes = 2 * kKvBytes;
  constexpr int kQBytes = (HD / 64) * kRows * 128;  // one Q tile
  constexpr int kKSteps = HD / 16;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                   // [tile][kQBytes]
  uint8_t* sKV = sQ + NT * kQBytes;     // [stage][K | V][chunk][128 keys][128 B]
  __shared__ uint64_t kv_full[kTcStages], kv_empty[kTcStages];
  __shared__ uint64_t s_full[NT], p_full[NT], o_full[NT];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const PrefillTile tile = tiles[blockIdx.x / blocks_per_tile];
  const int kvh = blockIdx.y;
  const int G = n_q / geom.n_kv;
  const int T = min(kPageTokens, NT * kRows / G);     // tokens per block
  const int t0 = (blockIdx.x % blocks_per_tile) * T;      // first token of the block
  const int nt = min(T, tile.nq - t0);                    // tokens of this block
  if (nt <= 0) return;                                    // (uniform per CTA)
  const int n_tiles = (nt * G + kRows - 1) / kRows;       // Q tiles with rows (1 or 2)
  const int last_pos = tile.pos0 + t0 + nt - 1;
  const int npages = last_pos / kPageTokens + 1;
  const int nblk = (npages + 1) / 2;                      // 128-key blocks
  const int* pt = page_table + static_cast<size_t>(tile.slot) * pt_stride;
  const int mma_warp = NT * 4;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&kv_map);
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < NT; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], kTcSoftmaxThreads);
      mbar_init(&o_full[t], 1);
    }
    fence_mbar_init();
  }
  if (warp == mma_warp) tmem_alloc<kTmemCols<NT>>(&tmem_base_sh);
  pdl_wait();  // q (QKV epilogue) and this layer's K/V pages are written
  pdl_trigger();

  // softmax threads: tile qt, row (TMEM lane) r; block row = qt*128 + r is
  // token t0 + row/G of head kvh*G + row%G
  const int qt = warp >> 2, r = threadIdx.x & (kRows - 1);
  const int brow = threadIdx.x;
  const int tok = brow / G, gh = brow % G;
  const bool valid = warp < mma_warp && tok < nt;
  const int pos = tile.pos0 + t0 + tok;
  if (warp < mma_warp && qt < n_tiles) {  // Q row -> smem, K-major SWIZZLE_128B
    const bf16* src = q + static_cast<size_t>(tile.q_row + t0 + tok) * q_row_stride +
                      static_cast<size_t>(kvh * G + gh) * HD;
    uint8_t* dq = sQ + qt * kQBytes;
#pragma unroll
    for (int c = 0; c < HD / 8; ++c) {
      uint4 v = valid ? reinterpret_cast<const uint4*>(src)[c] : make_uint4(0, 0, 0, 0);
      const int kb = c >> 3, cc = c & 7;
      *reinterpret_cast<uint4*>(dq + kb * (kRows * 128) + r * 128 + ((cc ^ (r & 7)) << 4)) = v;
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == mma_warp) {
    if (lane == 0) {
      // key block j = pages 2j and 2j+1 (an odd tail repeats its last page:
      // those keys are masked, the data only has to be finite)
      auto issue = [&](int j) {
        const int s = j % kTcStages;
        uint8_t* dst = sKV + s * kStageBytes;
        mbar_expect_tx(&kv_full[s], kStageBytes);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int phys = pt[min(2 * j + h, npages - 1)];
          const int rk = static_cast<int>(kv_row(geom, layer, phys, 0, kvh));
          const int rv = static_cast<int>(kv_row(geom, layer, phys, 1, kvh));
#pragma unroll
          for (int b = 0; b < HD / 64; ++b) {
            tma_load_2d(dst + b * kChunk + h * kBox, &kv_map, &kv_full[s], b * 64, rk);
            tma_load_2d(dst + kKvBytes + b * kChunk + h * kBox, &kv_map, &kv_full[s], b * 64, rv);
          }
        }
      };
      for (int j = 0; j < min(kTcStages, nblk); ++j) issue(j);
      const uint32_t id_s = umma_idesc_bf16(kRows, kBlkKeys);
      const uint32_t id_o = umma_idesc_bf16(kRows, HD) | (1u << 16);  // B (V) MN-major
      // S_j = Q_t K_j^T (M=128, N=128 keys) into tile t's S columns; the
      // previous block's P.V (reading P from those columns) was issued first
      auto mma_s = [&](int j, int t) {
        const int s = j % kTcStages;
        mbar_wait(&kv_full[s], (j / kTcStages) & 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(sKV + s * kStageBytes);
        const uint32_t q_base = smem_u32(sQ + t * kQBytes);
#pragma unroll
        for (int kk = 0; kk < kKSteps; ++kk) {
          const uint32_t off_a = (kk >> 2) * (kRows * 128) + (kk & 3) * 32;
          const uint32_t off_b = (kk >> 2) * kChunk + (kk & 3) * 32;
          umma_bf16(tmem + s_col<NT>(t), umma_desc_k128(q_base + off_a),
                    umma_desc_k128(k_base + off_b), id_s, kk > 0);
        }
        umma_commit(&s_full[t]);
      };
      for (int t = 0; t < n_tiles; ++t) mma_s(0, t);
      for (int j = 0; j < nblk; ++j) {
        const int s = j % kTcStages;
        const uint32_t v_base = smem_u32(sKV + s * kStageBytes + kKvBytes);
        for (int t = 0; t < n_tiles; ++t) {
          mbar_wait(&p_full[t], j & 1);  // P_j in TMEM, O rescaled if needed
          tc_fence_after();
          K6T(2 + t, j);
          const uint32_t p_tmem = tmem + s_col<NT>(t);  // P_j: bf16 pairs, 64 columns
#pragma unroll
          for (int kk = 0; kk < kBlkKeys / 16; ++kk)  // O += P_j V_j (16 keys per step)
            umma_bf16_ts(tmem + o_col<NT>(t), p_tmem + kk * 8,
                         umma_desc_mn128(v_base + kk * 2048, kChunk), id_o, (j | kk) != 0);
          if (j + 1 == nblk) umma_commit(&o_full[t]);
          if (t == n_tiles - 1) umma_commit(&kv_empty[s]);  // after every P_j V_j
          // this tile's next S (the other tile's softmax runs meanwhile)
          if (j + 1 < nblk) mma_s(j + 1, t);
        }
        K6T(4, j);
        if (j + kTcStages < nblk) {
          mbar_wait(&kv_empty[s], (j / kTcStages) & 1);  // K_j, V_j consumed
          issue(j + kTcStages);
        }
        K6T(6, j);
      }
    }
  } else if (qt < n_tiles) {
    // softmax: thread = TMEM lane = MMA row of tile qt
    const uint32_t t_row = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    float m = -CUDART_INF_F, l = 0.f;
    for (int j = 0; j < nblk; ++j) {
      // S_j done implies the previous P.V is done too (MMAs complete in order)
      mbar_wait(&s_full[qt], j & 1);
      tc_fence_after();
      if (threadIdx.x == 0) K6T(0, j);
      float sv[kBlkKeys];
      {
        uint32_t rr[8][16];
#pragma unroll
        for (int c = 0; c < 8; ++c) tmem_ld16_nw(t_row + s_col<NT>(qt) + c * 16, rr[c]);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
          for (int e = 0; e < 16; ++e) sv[c * 16 + e] = __uint_as_float(rr[c][e]);
      }
      const int kbase = j * kBlkKeys;
      if (!(valid && kbase + kBlkKeys - 1 <= pos)) {  // diagonal block / padding row
#pragma unroll
        for (int k = 0; k < kBlkKeys; ++k)
          if (!(valid && kbase + k <= pos)) sv[k] = -CUDART_INF_F;
      }
      // row max of the raw scores (the scale is positive: it commutes)
      float mx4[4] = {-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F};
#pragma unroll
      for (int k = 0; k < kBlkKeys; ++k) mx4[k & 3] = fmaxf(mx4[k & 3], sv[k]);
      const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * scale_log2;
      // lazy rescale: move m only when the row max outgrows it by 2^8
      const bool grow = mx > m + kRescaleLog2;
      const float m_new = grow ? mx : m;
      const float alpha = grow ? exp2f(m - m_new) : 1.f;  // 0 on the first block
      m = m_new;
      const float mu = m == -CUDART_INF_F ? 0.f : m;
      if (j > 0 && __any_sync(0xffffffffu, grow)) {  // O *= alpha (warp-collective)
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) {
          uint32_t rr[16];
          tmem_ld16_nw(t_row + o_col<NT>(qt) + c * 16, rr);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) rr[e] = __float_as_uint(__uint_as_float(rr[e]) * alpha);
          tmem_st16(t_row + o_col<NT>(qt) + c * 16, rr);
        }
      }
      // P_j = 2^(s * scale - m) as bf16 pairs into the first 64 S columns:
      // one FFMA and one MUFU.EX2 per score, the row sum over the fp32 P
      const float nmu = -mu;
      float rs4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < kBlkKeys / 32; ++c) {
        uint32_t pw[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float a = ex2_ftz(fmaf(sv[c * 32 + 2 * e], scale_log2, nmu));
          const float b = ex2_ftz(fmaf(sv[c * 32 + 2 * e + 1], scale_log2, nmu));
          rs4[e & 3] += a + b;
          pw[e] = pack_bf16x2(a, b);
        }
        tmem_st16(t_row + s_col<NT>(qt) + c * 16, pw);
      }
      tmem_wait_st();
      const float rs = (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
      l = l * alpha + rs;
      tc_fence_before();
      if (threadIdx.x == 0) K6T(1, j);
      if (threadIdx.x == kRows) K6T(7, j);
      mbar_arrive(&p_full[qt]);
    }
    mbar_wait(&o_full[qt], 0);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    bf16* dst = out + static_cast<size_t>(tile.q_row + t0 + tok) * out_row_stride +
                static_cast<size_t>(kvh * G + gh) * HD;
#pragma unroll
    for (int c = 0; c < HD / 16; ++c) {
      uint32_t rr[16];
      tmem_ld16_nw(t_row + o_col<NT>(qt) + c * 16, rr);
      tmem_wait_ld();
      if (valid) {
        uint4 w0, w1;
        w0.x = pack_bf16x2(__uint_as_float(rr[0]) * inv, __uint_as_float(rr[1]) * inv);
        w0.y = pack_bf16x2(__uint_as_float(rr[2]) * inv, __uint_as_float(rr[3]) * inv);
        w0.z = pack_bf16x2(__uint_as_float(rr[4]) * inv, __uint_as_float(rr[5]) * inv);
        w0.w = pack_bf16x2(__uint_as_float(rr[6]) * inv, __uint_as_float(rr[7]) * inv);
        w1.x = pack_bf16x2(__uint_as_float(rr[8]) * inv, __uint_as_float(rr[9]) * inv);
        w1.y = pack_bf16x2(__uint_as_float(rr[10]) * inv, __uint_as_float(rr[11]) * inv);
        w1.z = pack_bf16x2(__uint_as_float(rr[12]) * inv, __uint_as_float(rr[13]) * inv);
        w1.w = pack_bf16x2(__uint_as_float(rr[14]) * inv, __uint_as_float(rr[15]) * inv);
        reinterpret_cast<uint4*>(dst)[2 * c] = w0;
        reinterpret_cast<uint4*>(dst)[2 * c + 1] = w1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == mma_warp) {
    tc_fence_after();
    tmem_free<kTmemCols<NT>>(tmem);
  }
}

template <int HD, int NT>
int launch_tc_nt(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
                 int q_row_stride, int n_q, const int* pt, int pt_stride,
                 const PrefillTile* tiles, int n_tiles, bf16* out, int out_row_stride,
                 cudaStream_t st) {
  constexpr int kSmem = NT * (HD / 64) * kRows * 128 +
                        kTcStages * 2 * (HD / 64) * kBlkKeys * 128 + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(prefill_attn_tc_kernel<HD, NT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    attr = true;
  }
  const int G = n_q / g.n_kv;
  const int T = std::min(kPageTokens, NT * kRows / G);
  const int blocks_per_tile = (kPageTokens + T - 1) / T;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(HD));
  return launch_pdl(prefill_attn_tc_kernel<HD, NT>, dim3(n_tiles * blocks_per_tile, g.n_kv),
                    dim3(NT * kTcSoftmaxThreads + 32), kSmem, st, kv_map, g, layer, q,
                    q_row_stride, n_q, pt, pt_stride, tiles, blocks_per_tile, out,
                    out_row_stride, scale_log2);
}

// Two Q tiles per CTA halve the KV traffic per flop, but only pay while the
// launch still covers most SMs (one CTA per SM: 225 KB smem, 512 TMEM cols;
// measured at 32k context: 128 two-tile CTAs 1088 us vs 256 one-tile 1146)
template <int HD>
int launch_tc(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
              int q_row_stride, int n_q, const int* pt, int pt_stride, const PrefillTile* tiles,
              int n_tiles, bf16* out, int out_row_stride, cudaStream_t st) {
  const int G = n_q / g.n_kv;
  const int bpt2 = (kPageTokens + std::min(kPageTokens, 2 * kRows / G) - 1) /
                   std::min(kPageTokens, 2 * kRows / G);
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (3 * n_tiles * bpt2 * g.n_kv >= 2 * sms)
    return launch_tc_nt<HD, 2>(kv_map, g, layer, q, q_row_stride, n_q, pt, pt_stride, tiles,
                               n_tiles, out, out_row_stride, st);
  return launch_tc_nt<HD, 1>(kv_map, g, layer, q, q_row_stride, n_q, pt, pt_stride, tiles,
                             n_tiles, out, out_row_stride, st);
}

}  // namespace

// tcgen05 K6 (GQA groups of <= 128 / 16 query heads share a CTA's KV pages)
int prefill_attention_tc(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
                         int q_row_stride, int n_q, const int* page_table, int pt_stride,
                         const PrefillTile* tiles, int n_tiles, bf16* out, int out_row_stride,
                         cudaStream_t st) {
  if (n_tiles <= 0) return HS_OK;
  if (n_q % g.n_kv || n_q / g.n_kv > kRows / 16) return HS_E_CONFIG;
  if (g.head_dim == 128)
    return launch_tc<128>(kv_map, g, layer, q, q_row_stride, n_q, page_table, pt_stride, tiles,
                          n_tiles, out, out_row_stride, st);
  if (g.head_dim == 64)
    return launch_tc<64>(kv_map, g, layer, q, q_row_stride, n_q, page_table, pt_stride, tiles,
                         n_tiles, out, out_row_stride, st);
  return HS_E_CONFIG;
}

}  // namespace hs

#ifdef HS_K6_TRACE
extern "C" __attribute__((visibility("default"))) int hs_debug_k6_trace(long long* host) {
  return cudaMemcpyFromSymbol(host, hs::g_k6_trace, sizeof(hs::g_k6_trace)) == cudaSuccess ? 0 : 1;
}
#endif
