// K3: layer-wise-batched Dense GEMM on 5th-gen tensor cores.
//
//   out[split][t][n] = sum_{k in split} X[t][k] * W[n][k]      (fp32 partials)
//
// "Swap-AB" orientation: the weight matrix is the UMMA A operand (M = 128
// output features per CTA tile) and the token rows are the B operand
// (N = BN tokens, 16..256).  Serving batches are mostly a few dozen rows, so
// weights dominate HBM traffic; putting them on the M side keeps every CTA
// streaming 128-row weight tiles while the token tile is only as wide as the
// batch.  Split-K over grid.z fills all 148 SMs when N/128 alone cannot.
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator +
// single-thread tcgen05.mma issuer, warps 2..5 = epilogue (tcgen05.ld from
// TMEM lane quarter warp%4 -> coalesced fp32 stores).
//
// Replaces the cost-oracle charge probe_dense() (reference
// pkg/src/hybridserve/profiles.py:132-143) with real QKV / O / gate-up / down
// projections ("QKV + proj + MLP", profiles.py:135).
#include <cudaTypedefs.h>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

constexpr int kGemmThreads = 192;
constexpr int kTileM = 128;  // output features per CTA tile
constexpr int kTileK = 64;   // one 128-byte swizzle atom of bf16

template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN <= 16 ? 6 : (BN <= 32 ? 5 : 4);
  static constexpr int kABytes = kTileM * kTileK * 2;
  static constexpr int kBBytes = BN * kTileK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kAccCols = BN < 32 ? 32 : BN;        // one accumulator
  static constexpr int kTmemCols = 2 * kAccCols;            // double-buffered
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

// Stream-K work split.  The GEMM is `tiles` output tiles (128 features x BN
// tokens) of `kb` k-blocks each: U = tiles * kb units.  CTA c of G owns the
// contiguous units [start(c), start(c+1)) — tile-aligned when there are at
// least G tiles — so every CTA streams the same number of weight bytes in a
// single wave.  A tile whose k-range spans several CTAs gets one fp32
// partial plane per CTA (plane = c - first owner of the tile); the CTA that
// finishes a tile zero-fills the tile's unused planes, so consumers always
// sum exactly `planes` planes and the result is deterministic.
struct StreamK {
  int tiles, kb, G, aligned;
  __host__ __device__ long long start(int c) const {
    if (aligned) return (static_cast<long long>(c) * tiles / G) * kb;
    return static_cast<long long>(c) * tiles * kb / G;
  }
  __host__ __device__ int owner(long long u) const {  // largest c with start(c) <= u
    int lo = 0, hi = G - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (start(mid) <= u) lo = mid; else hi = mid - 1;
    }
    return lo;
  }
};

// kBlocked: weights pre-tiled as [N/128][K/64][128][64] so every 16 KB TMA
// box is one contiguous run of HBM (row-major weights make each box 128
// scattered 128-byte segments).
template <int BN, bool kBlocked>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap map_w,
                        const __grid_constant__ CUtensorMap map_x, float* __restrict__ out,
                        int n_out, int tokens, StreamK sk, int planes) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;  // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_tiles = n_out / kTileM;
  const long long u_begin = sk.start(blockIdx.x), u_end = sk.start(blockIdx.x + 1);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrival per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();  // dependents may be scheduled; they wait for our completion

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      // walk the CTA's unit range; weights never depend on the previous
      // kernel, so the first stages' weight tiles go out before the PDL wait
      int i = 0;
      bool waited = false;
      int pre = 0;
      for (long long u = u_begin; u < u_end; ++u, ++i) {
        const int t = static_cast<int>(u / sk.kb), k = static_cast<int>(u % sk.kb);
        const int n0 = (t % n_tiles) * kTileM, t0 = (t / n_tiles) * BN;
        const int s = i % C::kStages;
        const uint32_t ph = (i / C::kStages) & 1;
        if (i < C::kStages) {
          mbar_expect_tx(&full[s], C::kStageBytes);
          if (kBlocked)
            tma_load_4d_hint(sA + s * C::kABytes, &map_w, &full[s], 0, 0, k, n0 / kTileM, pol);
          else
            tma_load_2d_hint(sA + s * C::kABytes, &map_w, &full[s], k * kTileK, n0, pol);
          ++pre;
          continue;
        }
        if (!waited) {
          pdl_wait();
          waited = true;
          long long v = u_begin;
          for (int j = 0; j < pre; ++j, ++v) {
            const int tj = static_cast<int>(v / sk.kb), kj = static_cast<int>(v % sk.kb);
            tma_load_2d(sB + j * C::kBBytes, &map_x, &full[j], kj * kTileK, (tj / n_tiles) * BN);
          }
        }
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], C::kStageBytes);
        if (kBlocked)
          tma_load_4d_hint(sA + s * C::kABytes, &map_w, &full[s], 0, 0, k, n0 / kTileM, pol);
        else
          tma_load_2d_hint(sA + s * C::kABytes, &map_w, &full[s], k * kTileK, n0, pol);
        tma_load_2d(sB + s * C::kBBytes, &map_x, &full[s], k * kTileK, t0);
      }
      if (!waited) {
        pdl_wait();
        long long v = u_begin;
        for (int j = 0; j < pre; ++j, ++v) {
          const int tj = static_cast<int>(v / sk.kb), kj = static_cast<int>(v % sk.kb);
          tma_load_2d(sB + j * C::kBBytes, &map_x, &full[j], kj * kTileK, (tj / n_tiles) * BN);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(kTileM, BN);
      int i = 0, seg = 0;
      for (long long u = u_begin; u < u_end; ++seg) {
        const int t = static_cast<int>(u / sk.kb);
        const long long seg_end = min(u_end, static_cast<long long>(t + 1) * sk.kb);
        const int acc = seg & 1;
        const uint32_t tacc = tmem + acc * C::kAccCols;
        mbar_wait(&tempty[acc], ((seg >> 1) & 1) ^ 1);  // epilogue drained this buffer
        tc_fence_after();
        for (int first = 1; u < seg_end; ++u, ++i, first = 0) {
          const int s = i % C::kStages;
          mbar_wait(&full[s], (i / C::kStages) & 1);
          tc_fence_after();
          const uint64_t a = umma_desc_k128(smem_u32(sA + s * C::kABytes));
          const uint64_t b = umma_desc_k128(smem_u32(sB + s * C::kBBytes));
#pragma unroll
          for (int k = 0; k < kTileK / 16; ++k)
            umma_bf16(tacc, a + 2 * k, b + 2 * k, idesc, (first && k == 0) ? 0u : 1u);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int n_local = q * 32 + lane;
    pdl_wait();  // `out` may still be read by the previous kernel
    int seg = 0;
    for (long long u = u_begin; u < u_end; ++seg) {
      const int t = static_cast<int>(u / sk.kb);
      const long long t_first = static_cast<long long>(t) * sk.kb;
      const long long seg_end = min(u_end, t_first + sk.kb);
      const int acc = seg & 1;
      const int c_first = sk.owner(t_first);
      const int plane = static_cast<int>(blockIdx.x) - c_first;
      const bool tile_done = seg_end == t_first + sk.kb;  // this CTA finishes the tile
      const int used = tile_done ? plane + 1 : 0;
      const int n = (t % n_tiles) * kTileM + n_local;
      const int t0 = (t / n_tiles) * BN;
      mbar_wait(&tfull[acc], (seg >> 1) & 1);
      tc_fence_after();
      float* o = out + static_cast<size_t>(plane) * tokens * n_out + n;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        if (t0 + c >= tokens) break;
        float v[16];
        tmem_ld16(tmem + acc * C::kAccCols + (static_cast<uint32_t>(q * 32) << 16) + c, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int tt = t0 + c + j;
          if (tt < tokens) o[static_cast<size_t>(tt) * n_out] = v[j];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      // zero the planes no CTA covers for this tile
      for (int p = used; tile_done && p < planes; ++p) {
        float* z = out + static_cast<size_t>(p) * tokens * n_out + n;
        for (int tt = t0; tt < min(tokens, t0 + BN); ++tt) z[static_cast<size_t>(tt) * n_out] = 0.f;
      }
      u = seg_end;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<C::kTmemCols>(tmem);
  }
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int make_map_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  auto fn = encode_fn();
  if (!fn) return HS_E_CUDA;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? HS_OK : HS_E_CUDA;
}

int gemm_pick_bn(int tokens) {
  if (tokens <= 16) return 16;
  if (tokens <= 32) return 32;
  if (tokens <= 64) return 64;
  if (tokens <= 128) return 128;
  return 256;
}

static StreamK plan_streamk(int n_out, int k, int tokens, int bn, int G) {
  StreamK sk;
  sk.tiles = (n_out / kTileM) * ((tokens + bn - 1) / bn);
  sk.kb = k / kTileK;
  sk.G = G;
  // tile-aligned (no partial planes) once every CTA gets >= 4 whole tiles
  sk.aligned = sk.tiles >= 4 * G;
  return sk;
}

static int streamk_planes(const StreamK& sk) {
  int worst = 1;
  for (int t = 0; t < sk.tiles; ++t) {
    const int a = sk.owner(static_cast<long long>(t) * sk.kb);
    const int b = sk.owner(static_cast<long long>(t + 1) * sk.kb - 1);
    worst = max(worst, b - a + 1);
  }
  return worst;
}

// CTAs of one wave (148 SMs x resident CTAs), capped by the work and by the
// number of partial planes the caller can hold.
static StreamK choose_streamk(int n_out, int k, int tokens, int bn, int max_planes, int* planes) {
  const int per_sm = bn <= 64 ? 2 : 1;
  const int tiles = (n_out / kTileM) * ((tokens + bn - 1) / bn);
  const int units = tiles * (k / kTileK);
  int G = min(148 * per_sm, units);
  // at least ~4 k-blocks per CTA so the pipeline amortises its prologue
  G = max(1, min(G, max(tiles, units / 4)));
  for (;;) {
    StreamK sk = plan_streamk(n_out, k, tokens, bn, G);
    const int p = streamk_planes(sk);
    if (p <= max_planes || G == 1) {
      *planes = p;
      return sk;
    }
    G = max(1, G * max_planes / (p + 1));
  }
}

int gemm_pick_splits(int n_out, int k, int tokens, int bn, int max_splits) {
  int planes = 1;
  choose_streamk(n_out, k, tokens, bn, max_splits, &planes);
  return planes;
}

template <int BN, bool kBlocked>
static int launch_bn(const CUtensorMap& mw, const CUtensorMap& mx, float* out, int n_out,
                     int tokens, const StreamK& sk, int planes, cudaStream_t st) {
  using C = GemmCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN, kBlocked>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sk.G);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, gemm_bf16_tn_kernel<BN, kBlocked>, mw, mx, out, n_out, tokens, sk,
                     planes);
  return launched();
}

// `max_planes`: partial planes the output buffer holds; the planes actually
// written (all of them, zero-filled where unused) are returned in *planes.
template <bool kBlocked>
static int launch_any(const CUtensorMap& mw, const CUtensorMap& mx, int bn, float* out, int n_out,
                      int tokens, const StreamK& sk, int planes, cudaStream_t st) {
  switch (bn) {
    case 16: return launch_bn<16, kBlocked>(mw, mx, out, n_out, tokens, sk, planes, st);
    case 32: return launch_bn<32, kBlocked>(mw, mx, out, n_out, tokens, sk, planes, st);
    case 64: return launch_bn<64, kBlocked>(mw, mx, out, n_out, tokens, sk, planes, st);
    case 128: return launch_bn<128, kBlocked>(mw, mx, out, n_out, tokens, sk, planes, st);
    case 256: return launch_bn<256, kBlocked>(mw, mx, out, n_out, tokens, sk, planes, st);
  }
  return HS_E_CONFIG;
}

int gemm_launch(const CUtensorMap& mw, const CUtensorMap& mx, int bn, float* out, int n_out,
                int tokens, int k, int max_planes, cudaStream_t st, int* planes, bool blocked) {
  *planes = 1;
  if (tokens <= 0) return HS_OK;
  if (n_out % kTileM || k % kTileK) return HS_E_CONFIG;
  const StreamK sk = choose_streamk(n_out, k, tokens, bn, max_planes, planes);
  return blocked ? launch_any<true>(mw, mx, bn, out, n_out, tokens, sk, *planes, st)
                 : launch_any<false>(mw, mx, bn, out, n_out, tokens, sk, *planes, st);
}

// Row-major [n][k] -> blocked [n/128][k/64][128][64] (one thread per 16 B).
__global__ void relayout_blocked_kernel(const bf16* __restrict__ src, bf16* __restrict__ dst,
                                        int n, int k) {
  const size_t chunks = static_cast<size_t>(n) * k / 8;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < chunks;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t e = i * 8;
    const int row = static_cast<int>(e / k), col = static_cast<int>(e % k);
    const size_t o = ((static_cast<size_t>(row / kTileM) * (k / kTileK) + col / kTileK) * kTileM +
                      row % kTileM) * kTileK + col % kTileK;
    *reinterpret_cast<int4*>(dst + o) = *reinterpret_cast<const int4*>(src + e);
  }
}

int relayout_blocked(const bf16* src, bf16* dst, int n, int k, cudaStream_t st) {
  if (n % kTileM || k % kTileK) return HS_E_CONFIG;
  relayout_blocked_kernel<<<148 * 8, 256, 0, st>>>(src, dst, n, k);
  return launched();
}

int make_weight_map_blocked(CUtensorMap* map, const bf16* w, int n_out, int k) {
  auto fn = encode_fn();
  if (!fn) return HS_E_CUDA;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(kTileK), static_cast<cuuint64_t>(kTileM),
                        static_cast<cuuint64_t>(k / kTileK), static_cast<cuuint64_t>(n_out / kTileM)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(kTileK) * 2,
                           static_cast<cuuint64_t>(kTileK) * kTileM * 2,
                           static_cast<cuuint64_t>(kTileK) * kTileM * 2 * (k / kTileK)};
  cuuint32_t box[4] = {kTileK, kTileM, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<bf16*>(w), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? HS_OK : HS_E_CUDA;
}

int make_weight_map(CUtensorMap* map, const bf16* w, int n_out, int k) {
  return make_map_2d_bf16(map, w, k, n_out, static_cast<uint64_t>(k) * 2, kTileK, kTileM);
}

int make_act_map(CUtensorMap* map, const bf16* x, int rows, int k, int ld, int bn) {
  return make_map_2d_bf16(map, x, k, rows, static_cast<uint64_t>(ld) * 2, kTileK, bn);
}

}  // namespace hs
