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
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap map_w,
                        const __grid_constant__ CUtensorMap map_x, float* __restrict__ out,
                        int n_out, int tokens, int kb_per_split, int kb_total) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * kTileM;
  const int t0 = blockIdx.y * BN;
  const int split = blockIdx.z;
  const int kb0 = split * kb_per_split;
  const int kb1 = min(kb_total, kb0 + kb_per_split);
  const int nkb = kb1 - kb0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::kStages;
        const uint32_t ph = (i / C::kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], C::kStageBytes);
        tma_load_2d_hint(sA + s * C::kABytes, &map_w, &full[s], (kb0 + i) * kTileK, n0, pol);
        tma_load_2d(sB + s * C::kBBytes, &map_x, &full[s], (kb0 + i) * kTileK, t0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(kTileM, BN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::kStages;
        const uint32_t ph = (i / C::kStages) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint64_t a = umma_desc_k128(smem_u32(sA + s * C::kABytes));
        const uint64_t b = umma_desc_k128(smem_u32(sB + s * C::kBBytes));
#pragma unroll
        for (int k = 0; k < kTileK / 16; ++k) {
          // +32 bytes along K inside the 128B swizzle atom = +2 in the
          // 16-byte start-address field
          umma_bf16(tmem, a + 2 * k, b + 2 * k, idesc, (i | k) != 0);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(tfull);
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int n = n0 + q * 32 + lane;
    float* o = out + static_cast<size_t>(split) * tokens * n_out + n;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      if (t0 + c >= tokens) break;
      float v[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
      if (n < n_out) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int t = t0 + c + j;
          if (t < tokens) o[static_cast<size_t>(t) * n_out] = v[j];
        }
      }
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

int gemm_pick_splits(int n_out, int k, int tokens, int bn, int max_splits) {
  const int tiles = (n_out / kTileM) * ((tokens + bn - 1) / bn);
  const int kb_total = k / kTileK;
  const int per_sm = bn <= 64 ? 2 : 1;
  const int target = 148 * per_sm;
  int splits = (target + tiles - 1) / tiles;
  splits = min(splits, max(1, kb_total / 4));
  splits = max(1, min(splits, max_splits));
  const int kbps = (kb_total + splits - 1) / splits;
  return (kb_total + kbps - 1) / kbps;
}

template <int BN>
static int launch_bn(const CUtensorMap& mw, const CUtensorMap& mx, float* out, int n_out,
                     int tokens, int k, int splits, cudaStream_t st) {
  using C = GemmCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::kSmemBytes);
    attr_set = true;
  }
  const int kb_total = k / kTileK;
  const int kbps = (kb_total + splits - 1) / splits;
  dim3 grid(n_out / kTileM, (tokens + BN - 1) / BN, splits);
  gemm_bf16_tn_kernel<BN><<<grid, kGemmThreads, C::kSmemBytes, st>>>(mw, mx, out, n_out, tokens,
                                                                    kbps, kb_total);
  return launched();
}

int gemm_launch(const CUtensorMap& mw, const CUtensorMap& mx, int bn, float* out, int n_out,
                int tokens, int k, int splits, cudaStream_t st) {
  if (tokens <= 0) return HS_OK;
  if (n_out % kTileM || k % kTileK) return HS_E_CONFIG;
  switch (bn) {
    case 16: return launch_bn<16>(mw, mx, out, n_out, tokens, k, splits, st);
    case 32: return launch_bn<32>(mw, mx, out, n_out, tokens, k, splits, st);
    case 64: return launch_bn<64>(mw, mx, out, n_out, tokens, k, splits, st);
    case 128: return launch_bn<128>(mw, mx, out, n_out, tokens, k, splits, st);
    case 256: return launch_bn<256>(mw, mx, out, n_out, tokens, k, splits, st);
  }
  return HS_E_CONFIG;
}

int make_weight_map(CUtensorMap* map, const bf16* w, int n_out, int k) {
  return make_map_2d_bf16(map, w, k, n_out, static_cast<uint64_t>(k) * 2, kTileK, kTileM);
}

int make_act_map(CUtensorMap* map, const bf16* x, int rows, int k, int ld, int bn) {
  return make_map_2d_bf16(map, x, k, rows, static_cast<uint64_t>(ld) * 2, kTileK, bn);
}

}  // namespace hs
