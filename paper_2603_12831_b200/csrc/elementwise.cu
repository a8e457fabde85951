// K4/K5/K8/K9 and the split-K epilogues: the bandwidth-bound glue of one
// transformer layer.  Every kernel here reads the fp32 split-K partials the
// tcgen05 GEMM wrote and fuses the reduction with the operation that follows
// the projection (RoPE + KV-page scatter + piggyback ship after QKV;
// residual add + RMSNorm after O-proj / down-proj; SiLU*up after gate-up;
// greedy argmax after the LM head).
#include <math_constants.h>

#include <algorithm>

#include <cooperative_groups.h>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace cg = cooperative_groups;

namespace hs {

constexpr int kMaxSplits = 16;

// Sums of `splits` fp32 split-K planes at p (plane stride in floats), plane 0
// first (a fixed order: results are bit-reproducible).
__device__ __forceinline__ void add4(float4& a, const float4& v) {
  a.x += v.x;
  a.y += v.y;
  a.z += v.z;
  a.w += v.w;
}

__device__ __forceinline__ float4 ld4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

// Every plane's load in flight at once (one memory round trip for up to
// kMaxSplits planes), summed plane 0 first.
__device__ __forceinline__ float4 sum_planes4_all(const float* __restrict__ p, size_t plane,
                                                  int splits) {
  float4 v[kMaxSplits];
#pragma unroll
  for (int k = 0; k < kMaxSplits; ++k)
    if (k < splits) v[k] = ld4(p + k * plane);
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int k = 0; k < kMaxSplits; ++k)
    if (k < splits) add4(a, v[k]);
  return a;
}

// two streams at once (gate and up of SwiGLU): twice the loads in flight
__device__ __forceinline__ void sum_planes4x2(const float* __restrict__ p,
                                              const float* __restrict__ q, size_t plane,
                                              int splits, float4& a, float4& b) {
  a = make_float4(0.f, 0.f, 0.f, 0.f);
  b = a;
  int k = 0;
  for (; k + 2 <= splits; k += 2) {
    const float4 p0 = ld4(p + k * plane), p1 = ld4(p + (k + 1) * plane);
    const float4 q0 = ld4(q + k * plane), q1 = ld4(q + (k + 1) * plane);
    add4(a, p0);
    add4(a, p1);
    add4(b, q0);
    add4(b, q1);
  }
  if (k < splits) {
    add4(a, ld4(p + k * plane));
    add4(b, ld4(q + k * plane));
  }
}

__device__ __forceinline__ float2 sum_planes2(const float* __restrict__ p, size_t plane,
                                              int splits) {
  float2 a = make_float2(0.f, 0.f);
  int k = 0;
  for (; k + 4 <= splits; k += 4) {
    float2 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldg(reinterpret_cast<const float2*>(p + (k + j) * plane));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      a.x += v[j].x;
      a.y += v[j].y;
    }
  }
  for (; k < splits; ++k) {
    const float2 v = __ldg(reinterpret_cast<const float2*>(p + k * plane));
    a.x += v.x;
    a.y += v.y;
  }
  return a;
}

__device__ __forceinline__ float sum_planes1(const float* __restrict__ p, size_t plane,
                                             int splits) {
  float a = 0.f;
  int k = 0;
  for (; k + 4 <= splits; k += 4) {
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldg(p + (k + j) * plane);
#pragma unroll
    for (int j = 0; j < 4; ++j) a += v[j];
  }
  for (; k < splits; ++k) a += __ldg(p + k * plane);
  return a;
}

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
  pdl_enter();  // dependent data of the previous kernel is visible
  const int r = blockIdx.x;
  const bf16* src = emb + static_cast<size_t>(tokens[r]) * d;
  float* dst = h + static_cast<size_t>(r) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = __bfloat162float(src[i]);
}

int embed_gather(const int* tokens, int rows, const bf16* emb, int d, float* h, cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  return launch_pdl(embed_kernel, dim3(rows), dim3(256), 0, st, tokens, emb, d, h);
}

// ---------------------------------------------------------------- RMSNorm
// (the residual_add_norm kernels with no partials to add; defined below)
int rmsnorm_rows(const float* h, int rows, int d, const float* w, float eps, bf16* out, int ld_out,
                 cudaStream_t st) {
  return residual_add_norm(nullptr, 0, rows, d, const_cast<float*>(h), w, eps, out, ld_out, st);
}

// ---------------------------------------------------------------- split-K
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int splits, size_t total,
                                     float* __restrict__ out) {
  pdl_enter();  // dependent data of the previous kernel is visible
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
  return launch_pdl(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, st, part, splits, total, out);
}

// h += sum_s part[s]; out = rmsnorm(h) * w   (out may be null)
// One 8-CTA thread-block cluster per row: each CTA owns d/8 columns, the
// row's sum of squares is reduced through distributed shared memory, so a
// handful of rows still spreads over 8x as many SMs.
constexpr int kNormCluster = 8;

__global__ void __cluster_dims__(kNormCluster, 1, 1) __launch_bounds__(256)
    residual_add_norm_kernel(const float* __restrict__ part, Planes splits, int rows, int d,
                             float* __restrict__ h, const float* __restrict__ w, float eps,
                             bf16* __restrict__ out, int ld_out, RowIo io) {
  pdl_enter();  // dependent data of the previous kernel is visible
  __shared__ float red[32];
  __shared__ float ssq_all[kNormCluster];
  cg::cluster_group cluster = cg::this_cluster();
  const int r = blockIdx.y;
  const int rank = static_cast<int>(cluster.block_rank());
  const int cols = d / kNormCluster;  // multiple of 4
  const int c0 = rank * cols;
  float* x = h + static_cast<size_t>(r) * d + c0;
  const float* xin = io.row_src(h, r, d) + c0;
  float* put = io.row_put(r, d);
  const bool write = splits.n > 0 || xin != x;
  const size_t plane = static_cast<size_t>(rows) * d;
  const float* pp = part + static_cast<size_t>(r) * d + c0;
  float ss = 0.f;
  for (int i = threadIdx.x * 4; i < cols; i += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(xin + i);
    if (splits.n > 0) {
      const float4 a = sum_planes4_all(pp + i, plane, splits.count(r, c0 + i));
      v.x += a.x;
      v.y += a.y;
      v.z += a.z;
      v.w += a.w;
    }
    if (write) *reinterpret_cast<float4*>(x + i) = v;
    if (put) *reinterpret_cast<float4*>(put + c0 + i) = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  if (!out) return;
  ss = block_sum(ss, red);
  // push this CTA's partial into every rank's slot table, one cluster
  // barrier, then each rank sums the table in rank order (no remote reads
  // after the barrier, so no second barrier to keep shared memory alive)
  if (threadIdx.x < kNormCluster) *cluster.map_shared_rank(&ssq_all[rank], threadIdx.x) = ss;
  cluster.sync();
  float total = 0.f;
#pragma unroll
  for (int k = 0; k < kNormCluster; ++k) total += ssq_all[k];
  const float inv = rsqrtf(total / d + eps);
  bf16* o = out + static_cast<size_t>(r) * ld_out + c0;
  const float* wp = w + c0;
  for (int i = threadIdx.x * 4; i < cols; i += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(x + i);
    const float4 g = *reinterpret_cast<const float4*>(wp + i);
    uint2 pk;
    pk.x = pack_bf16x2(v.x * inv * g.x, v.y * inv * g.y);
    pk.y = pack_bf16x2(v.z * inv * g.z, v.w * inv * g.w);
    *reinterpret_cast<uint2*>(o + i) = pk;
  }
}

// Tensor-parallel form: h = (io source | h) + sum over ranks (rank order) of
// each rank's local split-K sum, then the same cluster RMSNorm.  The
// dependents are released only after every peer has published, so a
// PDL-launched successor never occupies SMs a peer context still needs.
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __cluster_dims__(kNormCluster, 1, 1) __launch_bounds__(256)
    tp_add_norm_kernel(const float* __restrict__ part, Planes splits, int rows, int d,
                       float* __restrict__ h, const float* __restrict__ w, float eps,
                       bf16* __restrict__ out, int ld_out, RowIo io, TpPeers peers,
                       unsigned epoch) {
  pdl_wait();
  __shared__ float red[32];
  __shared__ float ssq_cta;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int cols = d / kNormCluster;
  const int c0 = rank * cols;
  const int par = epoch & 1;
  const size_t plane = static_cast<size_t>(rows) * d;
  // a fixed grid loops over the rows (every rank's grid is small enough to
  // be resident next to its peers' even when a group shares one device)
  for (int r = blockIdx.y; r < rows; r += gridDim.y) {
    const float* pp = part + static_cast<size_t>(r) * d + c0;
    const size_t xoff = par * peers.xbuf_par + static_cast<size_t>(r) * d + c0;
    const size_t foff = par * peers.flag_par + static_cast<size_t>(r) * kNormCluster + rank;
    // 1. publish this rank's partial of these columns
    float* mine = peers.xbuf[peers.me] + xoff;
    for (int i = threadIdx.x * 4; i < cols; i += blockDim.x * 4)
      *reinterpret_cast<float4*>(mine + i) = sum_planes4_all(pp + i, plane, splits.count(r, c0 + i));
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      st_release_sys(peers.flag[peers.me] + foff, epoch);
      // 2. wait for every peer's partial of the same columns
      // a peer that never publishes fails the launch after 20 s instead of
      // hanging the device (time-sliced peers on one GPU may take a while)
      uint64_t t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (int p = 0; p < peers.world; ++p) {
        while (static_cast<int>(ld_acquire_sys(peers.flag[p] + foff) - epoch) < 0) {
          __nanosleep(256);
          uint64_t now;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
          if (now - t0 > 20000000000ull) __trap();
        }
      }
    }
    __syncthreads();
    // 3. h = source + sum of all ranks' partials in rank order
    float* x = h + static_cast<size_t>(r) * d + c0;
    const float* xin = io.row_src(h, r, d) + c0;
    float* put = io.row_put(r, d);
    float ss = 0.f;
    for (int i = threadIdx.x * 4; i < cols; i += blockDim.x * 4) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int p = 0; p < peers.world; ++p)
        add4(a, __ldcv(reinterpret_cast<const float4*>(peers.xbuf[p] + xoff + i)));
      float4 v = *reinterpret_cast<const float4*>(xin + i);
      add4(v, a);
      *reinterpret_cast<float4*>(x + i) = v;
      if (put) *reinterpret_cast<float4*>(put + c0 + i) = v;
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    ss = block_sum(ss, red);
    if (threadIdx.x == 0) ssq_cta = ss;
    cluster.sync();
    float total = 0.f;
#pragma unroll
    for (int k = 0; k < kNormCluster; ++k) total += *cluster.map_shared_rank(&ssq_cta, k);
    cluster.sync();
    const float inv = rsqrtf(total / d + eps);
    bf16* o = out + static_cast<size_t>(r) * ld_out + c0;
    const float* wp = w + c0;
    for (int i = threadIdx.x * 4; i < cols; i += blockDim.x * 4) {
      const float4 v = *reinterpret_cast<const float4*>(x + i);
      const float4 g = *reinterpret_cast<const float4*>(wp + i);
      uint2 pk;
      pk.x = pack_bf16x2(v.x * inv * g.x, v.y * inv * g.y);
      pk.y = pack_bf16x2(v.z * inv * g.z, v.w * inv * g.w);
      *reinterpret_cast<uint2*>(o + i) = pk;
    }
  }
  // dependents are released only once every peer has published (no
  // PDL-launched successor may take SMs a peer context still needs)
  pdl_trigger();
}

int tp_add_norm(const float* part, const Planes& splits, int rows, int d, float* h, const float* w,
                float eps, bf16* out, int ld_out, cudaStream_t st, const RowIo& io,
                const TpPeers& peers, unsigned epoch) {
  if (rows <= 0) return HS_OK;
  if (d % (4 * kNormCluster) || splits.n > kMaxSplits || splits.n < 1 || peers.world < 1 ||
      peers.world > kMaxTp)
    return HS_E_CONFIG;
  constexpr int kTpRowCtas = 32;  // clusters per rank (rows are looped over)
  dim3 grid(kNormCluster, std::min(rows, kTpRowCtas));
  const int threads = std::min(256, ((d / kNormCluster / 4) + 31) / 32 * 32);
  return launch_pdl(tp_add_norm_kernel, dim3(grid), dim3(threads), 0, st, part, splits, rows, d,
                    h, w, eps, out, ld_out, io, peers, epoch);
}

// Many rows: one 256-thread CTA per row holding the row in registers (up to
// kRowVec float4 per thread, d <= 8192), no cluster barriers.
constexpr int kRowVec = 8;

__global__ void __launch_bounds__(256)
    residual_add_norm_rows_kernel(const float* __restrict__ part, Planes splits, int rows, int d,
                                  float* __restrict__ h, const float* __restrict__ w, float eps,
                                  bf16* __restrict__ out, int ld_out, RowIo io) {
  pdl_enter();
  __shared__ float red[32];
  const int r = blockIdx.x;
  float* x = h + static_cast<size_t>(r) * d;
  const float* xin = io.row_src(h, r, d);
  float* put = io.row_put(r, d);
  const bool write = splits.n > 0 || xin != x;
  const size_t plane = static_cast<size_t>(rows) * d;
  const float* pp = part + static_cast<size_t>(r) * d;
  // planes outer, the row's vectors inner: kRowVec loads in flight per plane
  float4 v[kRowVec];
  int cnt[kRowVec];
#pragma unroll
  for (int k = 0; k < kRowVec; ++k) {
    v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int i = (threadIdx.x + k * 256) * 4;
    cnt[k] = i < d ? splits.count(r, i) : 0;
  }
  for (int s = 0; s < splits.n; ++s) {
    const float* ps = pp + s * plane;
    float4 t[kRowVec];
#pragma unroll
    for (int k = 0; k < kRowVec; ++k) {
      const int i = (threadIdx.x + k * 256) * 4;
      if (s < cnt[k]) t[k] = ld4(ps + i);
    }
#pragma unroll
    for (int k = 0; k < kRowVec; ++k)
      if (s < cnt[k]) add4(v[k], t[k]);
  }
  // h += sum of the planes (the same association as the cluster form)
#pragma unroll
  for (int k = 0; k < kRowVec; ++k) {
    const int i = (threadIdx.x + k * 256) * 4;
    if (i < d) {
      float4 hv = *reinterpret_cast<const float4*>(xin + i);
      add4(hv, v[k]);
      v[k] = hv;
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kRowVec; ++k) {
    const int i = (threadIdx.x + k * 256) * 4;
    if (i < d) {
      if (write) *reinterpret_cast<float4*>(x + i) = v[k];
      if (put) *reinterpret_cast<float4*>(put + i) = v[k];
      ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
    }
  }
  if (!out) return;
  const float inv = rsqrtf(block_sum(ss, red) / d + eps);
  bf16* o = out + static_cast<size_t>(r) * ld_out;
#pragma unroll
  for (int k = 0; k < kRowVec; ++k) {
    const int i = (threadIdx.x + k * 256) * 4;
    if (i < d) {
      const float4 g = *reinterpret_cast<const float4*>(w + i);
      uint2 pk;
      pk.x = pack_bf16x2(v[k].x * inv * g.x, v[k].y * inv * g.y);
      pk.y = pack_bf16x2(v[k].z * inv * g.z, v[k].w * inv * g.w);
      *reinterpret_cast<uint2*>(o + i) = pk;
    }
  }
}

// up to this many rows the 8-CTA cluster form (one float4 column group per
// thread, every plane in flight) beats a CTA per row
constexpr int kClusterRowsMax = 64;

int residual_add_norm(const float* part, const Planes& splits, int rows, int d, float* h,
                      const float* w, float eps, bf16* out, int ld_out, cudaStream_t st,
                      const RowIo& io) {
  if (rows <= 0) return HS_OK;
  if (d % (4 * kNormCluster) || splits.n > kMaxSplits) return HS_E_CONFIG;
  if (rows > kClusterRowsMax && d <= 4 * 256 * kRowVec)
    return launch_pdl(residual_add_norm_rows_kernel, dim3(rows), dim3(256), 0, st, part, splits,
                      rows, d, h, w, eps, out, ld_out, io);
  dim3 grid(kNormCluster, rows);
  const int threads = std::min(256, ((d / kNormCluster / 4) + 31) / 32 * 32);
  return launch_pdl(residual_add_norm_kernel, dim3(grid), dim3(threads), 0, st, part, splits, rows,
                    d, h, w, eps, out, ld_out, io);
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
// grid (feature blocks, rows), 256 threads; each thread owns two rotation
// pairs (j, j+1) of one head: one float4 (permuted layout, pairs adjacent) or
// two float2 loads per split plane, bf16x2 stores of both halves.  q and k
// heads are rotated, v heads copied.
__global__ void __launch_bounds__(256)
    qkv_rope_scatter_kernel(const float* __restrict__ part, Planes splits, int rows, int n_q,
                            int n_kv, int hd, const float* __restrict__ rope_cos,
                            const float* __restrict__ rope_sin, const int* __restrict__ row_pos,
                            const int* __restrict__ row_slot, const int* __restrict__ row_mode,
                            int n_batch, const int* __restrict__ carry_pos,
                            const int* __restrict__ carry_slot, bf16* __restrict__ qbuf,
                            int q_row_stride, bf16* __restrict__ kv_pool, KvGeom geom, int layer,
                            const int* __restrict__ page_table, int pt_stride,
                            bf16* __restrict__ ship, int ship_stride, int permuted, RowCopy rc) {
  pdl_enter();  // dependent data of the previous kernel is visible
  const int r = blockIdx.y;
  if (r >= rows) {  // merged rows: host attention result -> attention buffer
    const int i = r - rows;
    // device-polled merges: padding rows (negative slot) are not consumed
    if (rc.idx[i] < 0) return;
    if (rc.expect) {
      // every CTA copying part of the row acquires the row's completion tag
      // itself (the acquire orders this CTA's row loads after the worker's
      // release); a row whose tag does not match is not consumed
      __shared__ int ok;
      if (threadIdx.x == 0) {
        const int slot = rc.idx[i];
        unsigned tag;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(tag) : "l"(rc.tags + slot) : "memory");
        ok = tag == static_cast<unsigned>(rc.expect[i]);
        if (!ok && blockIdx.x == 0) {
          rc.fault[1] = slot;
          rc.fault[2] = rc.layer;
          rc.fault[3] = tag;
          __threadfence_system();
          atomicExch(rc.fault, 1u);
        }
      }
      __syncthreads();
      if (!ok) return;
    }
    const uint4* src = reinterpret_cast<const uint4*>(rc.src + static_cast<size_t>(rc.idx[i]) * rc.src_stride);
    uint4* dst = reinterpret_cast<uint4*>(rc.dst + static_cast<size_t>(i) * rc.dst_stride);
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < rc.width / 8; v += gridDim.x * blockDim.x)
      dst[v] = src[v];
    return;
  }
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int quarter = hd / 4, half = hd / 2;
  const int heads = n_q + 2 * n_kv;
  if (t >= heads * quarter) return;
  const int head = t / quarter, j = 2 * (t % quarter);
  const int n_tot = heads * hd;
  const size_t plane = static_cast<size_t>(rows) * n_tot;
  const int base = head * hd;
  const float* src = part + static_cast<size_t>(r) * n_tot + base;
  // rows [0, n_batch) come from the iteration's row arrays (mode 0 = KV
  // page scatter, or per-row modes when given); rows beyond are carry rows
  // shipped to the host (mode 1)
  const bool batch = r < n_batch;
  const int pos = batch ? row_pos[r] : carry_pos[r - n_batch];
  const int slot = batch ? row_slot[r] : carry_slot[r - n_batch];
  const int mode = batch ? (row_mode ? row_mode[r] : 0) : 1;
  if (slot < 0) return;  // padding carry row (device-polled merges): nothing shipped
  float a1, a2, b1, b2;  // (x1, x2) of pairs j and j+1
  const int np = splits.count(r, base);
  if (permuted) {  // feature i of the head in row 2i, feature i + hd/2 in row 2i+1
    const float4 v = sum_planes4_all(src + 2 * j, plane, np);
    a1 = v.x, a2 = v.y, b1 = v.z, b2 = v.w;
  } else {
    const float2 lo = sum_planes2(src + j, plane, np);
    const float2 hi = sum_planes2(src + half + j, plane, np);
    a1 = lo.x, b1 = lo.y, a2 = hi.x, b2 = hi.y;
  }
  float y1a = a1, y2a = a2, y1b = b1, y2b = b2;
  if (head < n_q + n_kv) {  // rotate q and k heads
    const float2 c = *reinterpret_cast<const float2*>(rope_cos + static_cast<size_t>(pos) * half + j);
    const float2 s = *reinterpret_cast<const float2*>(rope_sin + static_cast<size_t>(pos) * half + j);
    y1a = a1 * c.x - a2 * s.x;
    y2a = a2 * c.x + a1 * s.x;
    y1b = b1 * c.y - b2 * s.y;
    y2b = b2 * c.y + b1 * s.y;
  }
  bf16* dst;
  if (mode == 1) {
    dst = ship + static_cast<size_t>(slot) * ship_stride + base;
  } else if (head < n_q) {
    dst = qbuf + static_cast<size_t>(r) * q_row_stride + base;
  } else {
    const int kv = head < n_q + n_kv ? 0 : 1;
    const int kh = head - n_q - kv * n_kv;
    const int phys = page_table[static_cast<size_t>(slot) * pt_stride + pos / kPageTokens];
    dst = kv_pool + (kv_row(geom, layer, phys, kv, kh) + pos % kPageTokens) * hd;
  }
  *reinterpret_cast<uint32_t*>(dst + j) = pack_bf16x2(y1a, y1b);
  *reinterpret_cast<uint32_t*>(dst + half + j) = pack_bf16x2(y2a, y2b);
}

int qkv_rope_scatter(const float* part, const Planes& splits, int rows, int n_q, int n_kv,
                     int head_dim,
                     const float* rope_cos, const float* rope_sin, const int* row_pos,
                     const int* row_slot, const int* row_mode, int n_batch, const int* carry_pos,
                     const int* carry_slot, bf16* qbuf, int q_row_stride, bf16* kv_pool,
                     const KvGeom& g, int layer, const int* page_table, int pt_stride, bf16* ship,
                     int ship_stride, cudaStream_t st, int permuted, const RowCopy& rc) {
  if (rows + rc.n <= 0) return HS_OK;
  if (splits.n > kMaxSplits || head_dim % 8 || q_row_stride % 2 || ship_stride % 2 ||
      (rc.n && (rc.width % 8 || rc.src_stride % 8 || rc.dst_stride % 8)))
    return HS_E_CONFIG;
  const int threads = (n_q + 2 * n_kv) * head_dim / 4;
  dim3 grid((threads + 255) / 256, rows + rc.n);
  return launch_pdl(qkv_rope_scatter_kernel, grid, dim3(256), 0, st, part, splits, rows, n_q, n_kv,
                    head_dim, rope_cos, rope_sin, row_pos, row_slot, row_mode, n_batch, carry_pos,
                    carry_slot, qbuf, q_row_stride, kv_pool, g, layer, page_table, pt_stride, ship,
                    ship_stride, permuted, rc);
}

// ---------------------------------------------------------------- SwiGLU
// grid (feature blocks, rows); each thread 4 consecutive features: float4
// loads of gate and up from every split plane, one 8-byte bf16 store.
__global__ void __launch_bounds__(256)
    silu_mul_kernel(const float* __restrict__ part, Planes splits, int rows, int ffn,
                    bf16* __restrict__ act, int ld_act, int permuted) {
  pdl_enter();  // dependent data of the previous kernel is visible
  const int r = blockIdx.y;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i >= ffn) return;
  const size_t plane = static_cast<size_t>(rows) * 2 * ffn;
  const float* src = part + static_cast<size_t>(r) * 2 * ffn;
  // permuted: 32-row groups [16 gate | 16 up] of the same features
  const int gi = permuted ? 32 * (i >> 4) + (i & 15) : i;
  const int ui = permuted ? gi + 16 : ffn + i;
  float4 g, u;
  sum_planes4x2(src + gi, src + ui, plane, splits.count(r, gi), g, u);
  auto f = [](float gt, float up) { return gt / (1.f + __expf(-gt)) * up; };
  uint2 pk;
  pk.x = pack_bf16x2(f(g.x, u.x), f(g.y, u.y));
  pk.y = pack_bf16x2(f(g.z, u.z), f(g.w, u.w));
  *reinterpret_cast<uint2*>(act + static_cast<size_t>(r) * ld_act + i) = pk;
}

int silu_mul(const float* part, const Planes& splits, int rows, int ffn, bf16* act, int ld_act,
             cudaStream_t st, int permuted) {
  if (rows <= 0 || ffn <= 0) return HS_OK;
  if (ffn % 16 || ld_act % 4 || splits.n > kMaxSplits) return HS_E_CONFIG;
  dim3 grid((ffn / 4 + 255) / 256, rows);
  return launch_pdl(silu_mul_kernel, grid, dim3(256), 0, st, part, splits, rows, ffn, act, ld_act,
                    permuted);
}

// ---------------------------------------------------------------- greedy argmax
// One 8-CTA cluster per row; each CTA scans a vocab slice, the cluster picks
// the best (value, lowest index) through distributed shared memory.
constexpr int kArgCluster = 8;

__device__ __forceinline__ void better(float& bv, int& bi, float v, int i) {
  if (v > bv || (v == bv && i < bi)) {
    bv = v;
    bi = i;
  }
}

__global__ void __cluster_dims__(kArgCluster, 1, 1) __launch_bounds__(512)
    argmax_kernel(const float* __restrict__ part, Planes splits, int rows, int vocab,
                  int* __restrict__ tokens, float* __restrict__ logits_out) {
  pdl_enter();  // dependent data of the previous kernel is visible
  __shared__ float sv[32];
  __shared__ int si[32];
  __shared__ float cta_v;
  __shared__ int cta_i;
  cg::cluster_group cluster = cg::this_cluster();
  const int r = blockIdx.y;
  const int rank = static_cast<int>(cluster.block_rank());
  const int per = (vocab + kArgCluster - 1) / kArgCluster;
  const int lo = rank * per, hi = min(vocab, lo + per);
  const size_t plane = static_cast<size_t>(rows) * vocab;
  const float* src = part + static_cast<size_t>(r) * vocab;
  float best = -CUDART_INF_F;
  int bi = 0x7fffffff;
  if ((vocab & 3) == 0) {
    // float4 columns, kArgVec per thread with every load of a plane in flight
    // (planes summed plane 0 first, as sum_planes1 does)
    constexpr int kArgVec = 8;
    const int n4 = vocab / 4, per4 = (n4 + kArgCluster - 1) / kArgCluster;
    const int lo4 = rank * per4, hi4 = min(n4, lo4 + per4);
    for (int base = lo4; base < hi4; base += kArgVec * blockDim.x) {
      float4 acc[kArgVec];
#pragma unroll
      for (int j = 0; j < kArgVec; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      int cnt[kArgVec];
#pragma unroll
      for (int j = 0; j < kArgVec; ++j) {
        const int i4 = base + j * blockDim.x + threadIdx.x;
        cnt[j] = i4 < hi4 ? splits.count(r, 4 * i4) : 0;
      }
      for (int sp = 0; sp < splits.n; ++sp) {
        float4 t[kArgVec];
#pragma unroll
        for (int j = 0; j < kArgVec; ++j) {
          const int i4 = base + j * blockDim.x + threadIdx.x;
          if (sp < cnt[j]) t[j] = ld4(src + sp * plane + 4 * i4);
        }
#pragma unroll
        for (int j = 0; j < kArgVec; ++j)
          if (sp < cnt[j]) add4(acc[j], t[j]);
      }
#pragma unroll
      for (int j = 0; j < kArgVec; ++j) {
        const int i4 = base + j * blockDim.x + threadIdx.x;
        if (i4 >= hi4) continue;
        if (logits_out)
          *reinterpret_cast<float4*>(logits_out + static_cast<size_t>(r) * vocab + 4 * i4) = acc[j];
        better(best, bi, acc[j].x, 4 * i4);
        better(best, bi, acc[j].y, 4 * i4 + 1);
        better(best, bi, acc[j].z, 4 * i4 + 2);
        better(best, bi, acc[j].w, 4 * i4 + 3);
      }
    }
  } else {
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const float v = sum_planes1(src + i, plane, splits.count(r, i));
      if (logits_out) logits_out[static_cast<size_t>(r) * vocab + i] = v;
      better(best, bi, v, i);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    better(best, bi, __shfl_xor_sync(0xffffffffu, best, o), __shfl_xor_sync(0xffffffffu, bi, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) better(best, bi, sv[k], si[k]);
    cta_v = best;
    cta_i = bi;
  }
  cluster.sync();
  if (rank == 0 && threadIdx.x == 0) {
    float v = cta_v;
    int idx = cta_i;
    for (int k = 1; k < kArgCluster; ++k)
      better(v, idx, *cluster.map_shared_rank(&cta_v, k), *cluster.map_shared_rank(&cta_i, k));
    tokens[r] = idx;
  }
  cluster.sync();
}

int argmax_rows(const float* part, const Planes& splits, int rows, int vocab, int* tokens,
                float* logits_out,
                cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  if (splits.n > kMaxSplits) return HS_E_CONFIG;
  dim3 grid(kArgCluster, rows);
  return launch_pdl(argmax_kernel, dim3(grid), dim3(512), 0, st, part, splits, rows, vocab, tokens, logits_out);
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
  pdl_enter();  // dependent data of the previous kernel is visible
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
    return launch_pdl(lse_merge_kernel<128>, dim3(blocks), dim3(128), 0, st, parts, lse, n_parts,
                      rows, n_q, part_stride, row_stride_parts, out, out_row_stride);
  if (head_dim == 64)
    return launch_pdl(lse_merge_kernel<64>, dim3(blocks), dim3(128), 0, st, parts, lse, n_parts,
                      rows, n_q, part_stride, row_stride_parts, out, out_row_stride);
  return HS_E_CONFIG;
}

}  // namespace hs
