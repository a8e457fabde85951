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

#include <algorithm>
#include <cstdlib>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

constexpr int kGemmThreads = 192;
constexpr int kTileM = 128;  // output features per CTA tile
constexpr int kTileK = 64;   // one 128-byte swizzle atom of bf16

#ifndef HS_GEMM_ST16
#define HS_GEMM_ST16 4
#endif
#ifndef HS_GEMM_ST32
#define HS_GEMM_ST32 4
#endif
template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN <= 16 ? HS_GEMM_ST16 : (BN <= 32 ? HS_GEMM_ST32 : 4);
  static constexpr int kABytes = kTileM * kTileK * 2;
  static constexpr int kBBytes = BN * kTileK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kAccCols = BN < 32 ? 32 : BN;        // one accumulator
  static constexpr int kTmemCols = 2 * kAccCols;            // double-buffered
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

// Stream-K work split (StreamK, hs_internal.h).  A tile whose k-range spans
// several CTAs gets one fp32 partial plane per CTA (plane = c - first owner
// of the tile); the CTA that finishes a tile zero-fills the tile's unused
// planes, so consumers always sum exactly `planes` planes and the result is
// deterministic.

// kBlocked: weights pre-tiled as [N/128][K/64][128][64] so every 16 KB TMA
// box is one contiguous run of HBM (row-major weights make each box 128
// scattered 128-byte segments).
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Apply the fused epilogue to 16 token columns `v` of output feature row n
// (all 32 lanes of the warp call this together: the pairings shuffle).
template <int Epi>
__device__ __forceinline__ void epi_apply(const EpiParams& ep, int n, int lane, int t0c,
                                          int tokens, float (&v)[16]) {
  if constexpr (Epi == EPI_RESID) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int tt = t0c + j;
      if (tt < tokens) ep.h[static_cast<size_t>(tt) * ep.ld_h + n] += v[j];
    }
  } else if constexpr (Epi == EPI_SILU) {
    // rows interleaved in 32-row groups: lanes 0-15 gate, 16-31 up of the
    // same 16 features (weights permuted by permute_rows_gate_up)
    const int f = 16 * (n >> 5) + lane;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float up = __shfl_xor_sync(0xffffffffu, v[j], 16);
      const int tt = t0c + j;
      if (lane < 16 && tt < tokens) {
        const float g = v[j];
        ep.act[static_cast<size_t>(tt) * ep.ld_act + f] =
            __float2bfloat16(g / (1.f + __expf(-g)) * up);
      }
    }
  } else if constexpr (Epi == EPI_QKV) {
    // rotate-half pairs (i, i+hd/2) sit in adjacent rows (permute_rows_qkv)
    const int hd = ep.hd, half = hd / 2;
    const int head = n / hd, p = n % hd, jj = p >> 1;
    const bool odd = p & 1;
    const bool rotate = head < ep.n_q + ep.n_kv;
    const int f = odd ? jj + half : jj;  // original feature inside the head
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float partner = __shfl_xor_sync(0xffffffffu, v[j], 1);
      const int tt = t0c + j;
      if (tt >= tokens) continue;
      const bool batch = tt < ep.n_batch;
      const int slot = batch ? ep.row_slot[tt] : ep.carry_slot[tt - ep.n_batch];
      if (slot < 0) continue;  // padding carry row (device-polled merges)
      const int pos = batch ? ep.row_pos[tt] : ep.carry_pos[tt - ep.n_batch];
      float y = v[j];
      if (rotate) {
        const float c = ep.rope_cos[static_cast<size_t>(pos) * half + jj];
        const float sn = ep.rope_sin[static_cast<size_t>(pos) * half + jj];
        const float x1 = odd ? partner : v[j], x2 = odd ? v[j] : partner;
        y = odd ? x2 * c + x1 * sn : x1 * c - x2 * sn;
      }
      bf16* dst;
      if (!batch) {
        dst = ep.ship + static_cast<size_t>(slot) * ep.ship_stride + head * hd;
      } else if (head < ep.n_q) {
        dst = ep.qbuf + static_cast<size_t>(tt) * ep.q_row_stride + head * hd;
      } else {
        const int kv = head < ep.n_q + ep.n_kv ? 0 : 1;
        const int kh = head - ep.n_q - kv * ep.n_kv;
        const int phys = ep.page_table[static_cast<size_t>(slot) * ep.pt_stride + pos / 64];
        dst = ep.kv_pool + (kv_row(ep.geom, ep.layer, phys, kv, kh) + pos % 64) * hd;
      }
      dst[f] = __float2bfloat16(y);
    }
  }
}

template <int BN, bool kBlocked, int Epi>
__global__ void __launch_bounds__(kGemmThreads, 2)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap map_w,
                        const __grid_constant__ CUtensorMap map_x, float* __restrict__ out,
                        int n_out, int tokens, StreamK sk, int planes, EpiParams ep) {
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
    __shared__ int s_last;
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
      const int n = (t % n_tiles) * kTileM + n_local;
      const int t0 = (t / n_tiles) * BN;
      const uint32_t tbase = tmem + acc * C::kAccCols + (static_cast<uint32_t>(q * 32) << 16);
      mbar_wait(&tfull[acc], (seg >> 1) & 1);
      tc_fence_after();
      const int n_seg = Epi == EPI_PLANES ? 1 : sk.owner(t_first + sk.kb - 1) - c_first + 1;
      bool fix = true;
      if (Epi == EPI_PLANES || n_seg > 1) {
        // publish this segment's fp32 partial plane
        float* o = out + static_cast<size_t>(plane) * tokens * n_out + n;
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
          if (t0 + c >= tokens) break;
          float v[16];
          tmem_ld16(tbase + c, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int tt = t0 + c + j;
            if (tt < tokens) o[static_cast<size_t>(tt) * n_out] = v[j];
          }
        }
        if (Epi == EPI_PLANES) {
          fix = false;
          // zero the planes no CTA covers for this tile (planes = 0: the
          // consumers read per-tile plane counts instead, see Planes)
          for (int p = tile_done ? plane + 1 : planes; p < planes; ++p) {
            float* z = out + static_cast<size_t>(p) * tokens * n_out + n;
            for (int tt = t0; tt < min(tokens, t0 + BN); ++tt) z[static_cast<size_t>(tt) * n_out] = 0.f;
          }
        } else {
          // stream-K fixup: the CTA whose segment completes last applies the
          // epilogue to the sum of all segments (per-tile semaphore)
          __threadfence();
          epi_bar();
          if (threadIdx.x == 64) s_last = atomicAdd(&ep.tile_sem[t], 1) == n_seg - 1;
          epi_bar();
          fix = s_last;
          if (fix) __threadfence();
        }
      }
      if constexpr (Epi != EPI_PLANES) {
        if (fix) {
#pragma unroll 1
          for (int c = 0; c < BN; c += 16) {
            if (t0 + c >= tokens) break;
            float v[16];
            tmem_ld16(tbase + c, v);
            // other segments' partials, 2 planes of loads in flight at a time
            for (int p0 = 0; p0 < n_seg; p0 += 2) {
              float w[2][16];
#pragma unroll
              for (int pp = 0; pp < 2; ++pp) {
                const int p = p0 + pp;
                const float* o = out + static_cast<size_t>(p) * tokens * n_out + n;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                  const int tt = t0 + c + j;
                  w[pp][j] = (p < n_seg && p != plane && tt < tokens)
                                 ? __ldcg(o + static_cast<size_t>(tt) * n_out) : 0.f;
                }
              }
#pragma unroll
              for (int pp = 0; pp < 2; ++pp)
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] += w[pp][j];
            }
            epi_apply<Epi>(ep, n, lane, t0 + c, tokens, v);
          }
          if (n_seg > 1 && threadIdx.x == 64) ep.tile_sem[t] = 0;  // ready for the next launch
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
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

// HS_GEMM_MAX_BN (tuning knob, read once): cap on the token-tile width.
static int max_bn() {
  static const int cap = [] {
    const char* e = getenv("HS_GEMM_MAX_BN");
    const int v = e ? atoi(e) : 256;
    return (v == 16 || v == 32 || v == 64 || v == 128) ? v : 256;
  }();
  return cap;
}

int gemm_pick_bn(int tokens) {
  int bn = 256;
  if (tokens <= 16) bn = 16;
  else if (tokens <= 32) bn = 32;
  else if (tokens <= 64) bn = 64;
  else if (tokens <= 128) bn = 128;
  return std::min(bn, max_bn());
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
static StreamK choose_streamk_uncached(int n_out, int k, int tokens, int bn, int max_planes,
                                      int* planes) {
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

// The schedule is a pure function of the shape; the step asks for the same
// few shapes every layer, so plans are memoised (host issue cost: the plane
// count walks every tile).  Per thread: each replica's engine thread issues.
static StreamK choose_streamk(int n_out, int k, int tokens, int bn, int max_planes, int* planes) {
  HProf hp(HP_PLAN);
  struct Entry {
    int n_out, k, tokens, bn, max_planes, planes;
    StreamK sk;
  };
  constexpr int kWays = 256;
  thread_local Entry cache[kWays];
  thread_local bool init = false;
  if (!init) {
    for (auto& e : cache) e.n_out = -1;
    init = true;
  }
  const unsigned h = (static_cast<unsigned>(n_out) * 2654435761u) ^ (static_cast<unsigned>(k) * 40503u) ^
                     (static_cast<unsigned>(tokens) * 97u) ^ (static_cast<unsigned>(bn) << 7) ^
                     (static_cast<unsigned>(max_planes) << 13);
  Entry& e = cache[(h ^ (h >> 11)) % kWays];
  if (e.n_out == n_out && e.k == k && e.tokens == tokens && e.bn == bn &&
      e.max_planes == max_planes) {
    *planes = e.planes;
    return e.sk;
  }
  const StreamK sk = choose_streamk_uncached(n_out, k, tokens, bn, max_planes, planes);
  e = Entry{n_out, k, tokens, bn, max_planes, *planes, sk};
  return sk;
}

int gemm_pick_splits(int n_out, int k, int tokens, int bn, int max_splits) {
  int planes = 1;
  choose_streamk(n_out, k, tokens, bn, max_splits, &planes);
  return planes;
}

template <int BN, bool kBlocked, int Epi>
static int launch_bn(const CUtensorMap& mw, const CUtensorMap& mx, float* out, int n_out,
                     int tokens, const StreamK& sk, int planes, const EpiParams& ep,
                     cudaStream_t st) {
  using C = GemmCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN, kBlocked, Epi>,
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
  HProf hp(HP_LAUNCH);
  cudaLaunchKernelEx(&cfg, gemm_bf16_tn_kernel<BN, kBlocked, Epi>, mw, mx, out, n_out, tokens,
                     sk, planes, ep);
  return launched();
}

// `max_planes`: partial planes the output buffer holds; the planes actually
// written (all of them, zero-filled where unused) are returned in *planes.
template <bool kBlocked, int Epi>
static int launch_any(const CUtensorMap& mw, const CUtensorMap& mx, int bn, float* out, int n_out,
                      int tokens, const StreamK& sk, int planes, const EpiParams& ep,
                      cudaStream_t st) {
  switch (bn) {
    case 16: return launch_bn<16, kBlocked, Epi>(mw, mx, out, n_out, tokens, sk, planes, ep, st);
    case 32: return launch_bn<32, kBlocked, Epi>(mw, mx, out, n_out, tokens, sk, planes, ep, st);
    case 64: return launch_bn<64, kBlocked, Epi>(mw, mx, out, n_out, tokens, sk, planes, ep, st);
    case 128: return launch_bn<128, kBlocked, Epi>(mw, mx, out, n_out, tokens, sk, planes, ep, st);
    case 256: return launch_bn<256, kBlocked, Epi>(mw, mx, out, n_out, tokens, sk, planes, ep, st);
  }
  return HS_E_CONFIG;
}

int gemm_launch_planes(const CUtensorMap& mw, const CUtensorMap& mx, int bn, float* out, int n_out,
                       int tokens, int k, int max_planes, cudaStream_t st, Planes* planes) {
  *planes = Planes(1);
  if (tokens <= 0) return HS_OK;
  if (n_out % kTileM || k % kTileK) return HS_E_CONFIG;
  int n = 1;
  const StreamK sk = choose_streamk(n_out, k, tokens, bn, max_planes, &n);
  planes->n = n;
  planes->sk = sk;
  planes->n_tiles = n_out / kTileM;
  planes->bn = bn;
  const EpiParams ep{};
  return launch_any<false, EPI_PLANES>(mw, mx, bn, out, n_out, tokens, sk, 0, ep, st);
}

int gemm_launch(const CUtensorMap& mw, const CUtensorMap& mx, int bn, float* out, int n_out,
                int tokens, int k, int max_planes, cudaStream_t st, int* planes, bool blocked) {
  *planes = 1;
  if (tokens <= 0) return HS_OK;
  if (n_out % kTileM || k % kTileK) return HS_E_CONFIG;
  const StreamK sk = choose_streamk(n_out, k, tokens, bn, max_planes, planes);
  const EpiParams ep{};
  return blocked ? launch_any<true, EPI_PLANES>(mw, mx, bn, out, n_out, tokens, sk, *planes, ep, st)
                 : launch_any<false, EPI_PLANES>(mw, mx, bn, out, n_out, tokens, sk, *planes, ep, st);
}

int gemm_launch_fused(const CUtensorMap& mw, const CUtensorMap& mx, int bn, float* scratch,
                      int n_out, int tokens, int k, int max_planes, int epi, const EpiParams& ep,
                      cudaStream_t st) {
  if (tokens <= 0) return HS_OK;
  if (n_out % kTileM || k % kTileK) return HS_E_CONFIG;
  int planes = 1;
  const StreamK sk = choose_streamk(n_out, k, tokens, bn, max_planes, &planes);
  switch (epi) {
    case EPI_RESID:
      return launch_any<false, EPI_RESID>(mw, mx, bn, scratch, n_out, tokens, sk, planes, ep, st);
    case EPI_SILU:
      return launch_any<false, EPI_SILU>(mw, mx, bn, scratch, n_out, tokens, sk, planes, ep, st);
    case EPI_QKV:
      return launch_any<false, EPI_QKV>(mw, mx, bn, scratch, n_out, tokens, sk, planes, ep, st);
  }
  return HS_E_CONFIG;
}

// Row permutations that put each fused epilogue's operand pair in one warp:
//   gate-up: 32-row groups [16 gate rows | 16 up rows] of the same features
//   qkv:     inside every head, rows (2j, 2j+1) = features (j, j + hd/2)
__global__ void permute_rows_kernel(const bf16* __restrict__ src, bf16* __restrict__ dst,
                                    int rows, int k, int kind, int a, int b) {
  const int p = blockIdx.x;  // destination row
  int o;
  if (kind == 0) {  // gate-up: a = ffn
    const int blk = p / 32, i = p % 32;
    o = i < 16 ? 16 * blk + i : a + 16 * blk + (i - 16);
  } else {  // qkv: a = head_dim
    const int head = p / a, r = p % a;
    o = head * a + ((r & 1) ? (r >> 1) + a / 2 : (r >> 1));
  }
  const int4* s = reinterpret_cast<const int4*>(src + static_cast<size_t>(o) * k);
  int4* d = reinterpret_cast<int4*>(dst + static_cast<size_t>(p) * k);
  for (int i = threadIdx.x; i < k / 8; i += blockDim.x) d[i] = s[i];
}

int permute_rows(const bf16* src, bf16* dst, int rows, int k, int kind, int a, cudaStream_t st) {
  return launch_pdl(permute_rows_kernel, dim3(rows), dim3(128), 0, st, src, dst, rows, k, kind, a,
                    0);
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
