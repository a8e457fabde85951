// K3 for prefill-sized batches on CTA pairs: the swap-AB stream-K GEMM of
// gemm_tcgen05.cu issued as tcgen05.mma.cta_group::2 (M = 256 weight rows,
// N = 256 tokens per pair tile).
//
//   out[plane][t][n] = sum_{k in segment} X[t][k] * W[n][k]      (fp32 partials)
//
// Each CTA of a pair stages its own 128 weight rows and HALF of the token
// tile (128 tokens); the MMA reads both CTAs' shared memory, so a pipeline
// stage is 32 KB per CTA instead of 48 (six stages in flight instead of
// four) and every token tile is read from L2 once per pair instead of once
// per CTA.  The leader CTA (rank 0) owns the full barriers (both CTAs' TMA
// loads signal it, `.cta_group::2`), issues every MMA and multicasts its
// commits to both CTAs' empty / accumulator-full barriers; both CTAs drain
// their half of the accumulator (TMEM lanes = their weight rows) and report
// to the leader's accumulator-empty barrier.
//
// Stream-K over pair tiles (256 features x 256 tokens): the partial planes
// have the same layout as the 1-SM kernel's, with Planes::tile_m = 256.
// Used from 256 batch rows up (gemm_pick_2sm), where the 1-SM kernel is
// bound by its four-stage pipeline; reference charge: probe_dense,
// pkg/src/hybridserve/profiles.py:132-143.
#include <algorithm>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

namespace {

constexpr int kThreads2 = 192;  // warp 0 TMA, warp 1 TMEM + MMA, warps 2-5 epilogue
constexpr int kPairM = 256;     // weight rows per pair tile
constexpr int kHalfM = 128;     // per CTA
constexpr int kK2 = 64;         // one SW128 atom of bf16
constexpr int kBN2 = 256;       // tokens per pair tile
constexpr int kStages2 = 6;
constexpr int kABytes2 = kHalfM * kK2 * 2;          // 16 KB
constexpr int kBBytes2 = (kBN2 / 2) * kK2 * 2;      // 16 KB: this CTA's half of the tokens
constexpr int kStageBytes2 = kABytes2 + kBBytes2;
constexpr int kAccCols2 = kBN2;                     // fp32 accumulator columns
constexpr int kTmemCols2 = 2 * kAccCols2;           // double-buffered: 512
constexpr int kSmem2 = kStages2 * kStageBytes2 + 1024 + 256;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// shared::cluster address of `p` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
// TMA load into this CTA's shared memory, completing on the mbarrier at the
// shared::cluster address `bar` (the leader's)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar,
                                                 int32_t c0, int32_t c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this offset in both CTAs once the MMAs issued so
// far have completed
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   bar_cluster_addr)
               : "memory");
}

__global__ void __launch_bounds__(kThreads2, 1)
    gemm_bf16_2sm_kernel(const __grid_constant__ CUtensorMap map_w,
                         const __grid_constant__ CUtensorMap map_x, float* __restrict__ out,
                         int n_out, int tokens, StreamK sk, int planes) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages2 * kABytes2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages2 * kStageBytes2);
  uint64_t* empty = full + kStages2;
  uint64_t* tfull = empty + kStages2;  // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int worker = static_cast<int>(blockIdx.x >> 1);
  const int n_tiles = n_out / kPairM;
  const long long u_begin = sk.start(worker), u_end = sk.start(worker + 1);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < kStages2; ++s) {
      mbar_init(&full[s], 1);   // leader: its producer's arrive + both CTAs' bytes
      mbar_init(&empty[s], 1);  // the leader's multicast commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // leader: 4 epilogue warps of each CTA
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(kTmemCols2)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the leader's barriers exist before any peer TMA / arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      // weights first (independent of the previous kernel), tokens after the
      // PDL wait; every load completes on the leader's full barrier
      int i = 0, pre = 0;
      bool waited = false;
      for (long long u = u_begin; u < u_end; ++u, ++i) {
        const int t = static_cast<int>(u / sk.kb), k = static_cast<int>(u % sk.kb);
        const int n0 = (t % n_tiles) * kPairM + static_cast<int>(rank) * kHalfM;
        const int t0 = (t / n_tiles) * kBN2 + static_cast<int>(rank) * (kBN2 / 2);
        const int s = i % kStages2;
        const uint32_t ph = (i / kStages2) & 1;
        const uint32_t fb = map_rank(&full[s], 0);
        if (i < kStages2) {
          if (leader) mbar_expect_tx(&full[s], 2 * kStageBytes2);
          tma_load_2d_pair(sA + s * kABytes2, &map_w, fb, k * kK2, n0, pol_w);
          ++pre;
          continue;
        }
        if (!waited) {
          pdl_wait();
          waited = true;
          long long v = u_begin;
          for (int j = 0; j < pre; ++j, ++v) {
            const int tj = static_cast<int>(v / sk.kb), kj = static_cast<int>(v % sk.kb);
            tma_load_2d_pair(sB + j * kBBytes2, &map_x, map_rank(&full[j], 0), kj * kK2,
                             (tj / n_tiles) * kBN2 + static_cast<int>(rank) * (kBN2 / 2), pol_x);
          }
        }
        mbar_wait(&empty[s], ph ^ 1);
        if (leader) mbar_expect_tx(&full[s], 2 * kStageBytes2);
        tma_load_2d_pair(sA + s * kABytes2, &map_w, fb, k * kK2, n0, pol_w);
        tma_load_2d_pair(sB + s * kBBytes2, &map_x, fb, k * kK2, t0, pol_x);
      }
      if (!waited) {
        pdl_wait();
        long long v = u_begin;
        for (int j = 0; j < pre; ++j, ++v) {
          const int tj = static_cast<int>(v / sk.kb), kj = static_cast<int>(v % sk.kb);
          tma_load_2d_pair(sB + j * kBBytes2, &map_x, map_rank(&full[j], 0), kj * kK2,
                           (tj / n_tiles) * kBN2 + static_cast<int>(rank) * (kBN2 / 2), pol_x);
        }
      }
    }
  } else if (warp == 1) {
    // the whole warp walks the loop (descriptors stay warp-uniform, in the
    // uniform datapath); one elected lane issues
    if (leader) {
      constexpr uint32_t idesc = umma_idesc_bf16(kPairM, kBN2);
      int i = 0, seg = 0;
      for (long long u = u_begin; u < u_end; ++seg) {
        const int t = static_cast<int>(u / sk.kb);
        const long long seg_end = min(u_end, static_cast<long long>(t + 1) * sk.kb);
        const int acc = seg & 1;
        const uint32_t tacc = tmem + acc * kAccCols2;
        mbar_wait(&tempty[acc], ((seg >> 1) & 1) ^ 1);  // both CTAs drained this buffer
        tc_fence_after();
        for (int first = 1; u < seg_end; ++u, ++i, first = 0) {
          const int s = i % kStages2;
          mbar_wait(&full[s], (i / kStages2) & 1);
          tc_fence_after();
          const uint64_t a = umma_desc_k128(smem_u32(sA + s * kABytes2));
          const uint64_t b = umma_desc_k128(smem_u32(sB + s * kBBytes2));
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < kK2 / 16; ++k)
              umma_bf16_pair(tacc, a + 2 * k, b + 2 * k, idesc, (first && k == 0) ? 0u : 1u);
            umma_commit_pair(&empty[s]);
          }
          __syncwarp();
        }
        if (elect_one()) umma_commit_pair(&tfull[acc]);
        __syncwarp();
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int n_local = static_cast<int>(rank) * kHalfM + q * 32 + lane;
    const uint32_t te0 = map_rank(&tempty[0], 0), te1 = map_rank(&tempty[1], 0);
    pdl_wait();  // `out` may still be read by the previous kernel
    int seg = 0;
    for (long long u = u_begin; u < u_end; ++seg) {
      const int t = static_cast<int>(u / sk.kb);
      const long long t_first = static_cast<long long>(t) * sk.kb;
      const long long seg_end = min(u_end, t_first + sk.kb);
      const int acc = seg & 1;
      const int c_first = sk.owner(t_first);
      const int plane = worker - c_first;
      const bool tile_done = seg_end == t_first + sk.kb;
      const int n = (t % n_tiles) * kPairM + n_local;
      const int t0 = (t / n_tiles) * kBN2;
      const uint32_t tbase = tmem + acc * kAccCols2 + (static_cast<uint32_t>(q * 32) << 16);
      mbar_wait(&tfull[acc], (seg >> 1) & 1);
      tc_fence_after();
      float* o = out + static_cast<size_t>(plane) * tokens * n_out + n;
#pragma unroll 1
      for (int c = 0; c < kBN2; c += 16) {
        if (t0 + c >= tokens) break;
        float v[16];
        tmem_ld16(tbase + c, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int tt = t0 + c + j;
          if (tt < tokens) o[static_cast<size_t>(tt) * n_out] = v[j];
        }
      }
      // uniform plane count (op-level API): zero the planes no worker covers
      for (int p = tile_done ? plane + 1 : planes; p < planes; ++p) {
        float* z = out + static_cast<size_t>(p) * tokens * n_out + n;
        for (int tt = t0; tt < min(tokens, t0 + kBN2); ++tt) z[static_cast<size_t>(tt) * n_out] = 0.f;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(acc ? te1 : te0);
      u = seg_end;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no peer arrive / MMA operand read targets this CTA any more
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols2)
                 : "memory");
  }
}

StreamK plan_pairs(int n_out, int k, int tokens, int max_planes, int* planes_out) {
  const int tiles = (n_out / kPairM) * ((tokens + kBN2 - 1) / kBN2);
  const int kb = k / kK2;
  const int units = tiles * kb;
  int G = std::min(74, units);
  G = std::max(1, std::min(G, std::max(tiles, units / 4)));
  for (;;) {
    StreamK sk;
    sk.tiles = tiles;
    sk.kb = kb;
    sk.G = G;
    sk.aligned = tiles >= 4 * G;
    int worst = 1;
    for (int t = 0; t < tiles; ++t) {
      const int a = sk.owner(static_cast<long long>(t) * kb);
      const int b = sk.owner(static_cast<long long>(t + 1) * kb - 1);
      worst = std::max(worst, b - a + 1);
    }
    if (worst <= max_planes || G == 1) {
      *planes_out = worst;
      return sk;
    }
    G = std::max(1, G * max_planes / (worst + 1));
  }
}

}  // namespace

bool gemm_pair_ok(int n_out, int k, int tokens) {
  static const bool on = [] {
    const char* e = getenv("HS_GEMM_2SM");
    return !e || atoi(e) != 0;
  }();
  return on && tokens >= kBN2 && n_out % kPairM == 0 && k % kK2 == 0;
}

// mx: the activation map with 128-token boxes (half of a pair tile).
// uniform_planes: zero-fill to a uniform plane count (op API), else the
// consumers read per-tile counts (Planes with tile_m = 256).
int gemm_launch_pair(const CUtensorMap& mw, const CUtensorMap& mx_half, float* out, int n_out,
                     int tokens, int k, int max_planes, bool uniform_planes, cudaStream_t st,
                     Planes* planes) {
  int n = 1;
  const StreamK sk = plan_pairs(n_out, k, tokens, max_planes, &n);
  planes->n = n;
  planes->sk = sk;
  planes->n_tiles = n_out / kPairM;
  planes->bn = kBN2;
  planes->tile_m = kPairM;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_bf16_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2);
    attr = true;
  }
  return launch_pdl_cluster(gemm_bf16_2sm_kernel, dim3(2 * sk.G), dim3(kThreads2), kSmem2, st, 2,
                            mw, mx_half, out, n_out, tokens, sk, uniform_planes ? n : 0);
}

}  // namespace hs
