// Internal launcher declarations shared by the libhs translation units.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/hs.h"

typedef __nv_bfloat16 bf16;

namespace hs {

// every kernel launch site returns through launched(): counts the launch
// (the bench's gpu_launches) and reports a launch error as HS_E_CUDA
extern unsigned long long g_launches;
// host-side issue profiler (HS_HOST_PROF=1): nanoseconds per section,
// printed by hs_destroy
extern int g_hprof_on;
extern double g_hprof_ns[8];
extern unsigned long long g_hprof_n[8];
double hprof_now_ns();
struct HProf {
  int sec;
  double t0;
  explicit HProf(int s) : sec(s), t0(g_hprof_on ? hprof_now_ns() : 0.0) {}
  ~HProf() {
    if (g_hprof_on) {
      g_hprof_ns[sec] += hprof_now_ns() - t0;
      g_hprof_n[sec] += 1;
    }
  }
};
enum { HP_LAYER = 0, HP_PACK = 1, HP_PLAN = 2, HP_LAUNCH = 3, HP_BEGIN = 4, HP_END = 5 };
inline int launched() {
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 4;
}

// Launch with programmatic stream serialization: the kernel may be scheduled
// while its predecessor drains; every libhs kernel begins with
// griddepcontrol.wait (pdl_wait) before touching dependent memory and
// triggers its own dependents right away.
template <typename... KArgs, typename... Args>
inline int launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HProf hp(HP_LAUNCH);
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  return launched();
}

// Same, as clusters of `cluster_x` CTAs along x (distributed shared memory).
template <typename... KArgs, typename... Args>
inline int launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster_x;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  HProf hp(HP_LAUNCH);
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  return launched();
}

// ---- KV pool geometry (used by GEMM epilogues and attention) ----
struct KvGeom {
  int layers, pages, n_kv, head_dim;
};
__host__ __device__ inline int64_t kv_row(const KvGeom& g, int layer, int page, int kv, int head) {
  return ((((int64_t)layer * g.pages + page) * 2 + kv) * g.n_kv + head) * 64;
}

// ---- GEMM stream-K schedule (gemm_tcgen05.cu) ----
// The GEMM is `tiles` output tiles (128 features x BN tokens) of `kb`
// k-blocks each: U = tiles * kb units.  CTA c of G owns the contiguous units
// [start(c), start(c+1)) -- tile-aligned when there are at least 4G tiles.
struct StreamK {
  int tiles, kb, G, aligned;
  __host__ __device__ long long start(int c) const {
    if (aligned) return (static_cast<long long>(c) * tiles / G) * kb;
    return static_cast<long long>(c) * tiles * kb / G;
  }
  // largest c with start(c) <= u, in closed form (start is floor(c*X/G)
  // scaled, so c*X < (x+1)*G); checked against a binary search over the
  // whole range of shapes
  __host__ __device__ int owner(long long u) const {
    const unsigned long long num = aligned ? (static_cast<unsigned long long>(u / kb) + 1) * G - 1
                                           : (static_cast<unsigned long long>(u) + 1) * G - 1;
    const unsigned long long den = aligned ? tiles : static_cast<unsigned long long>(tiles) * kb;
    // 32-bit division when it fits (every serving shape): the glue kernels
    // call this on their critical path
    const unsigned long long c = (num >> 32) == 0 && (den >> 32) == 0
                                     ? static_cast<unsigned>(num) / static_cast<unsigned>(den)
                                     : num / den;
    return static_cast<int>(c < static_cast<unsigned long long>(G - 1) ? c : G - 1);
  }
};

// ---- split-K partial planes of a GEMM launch, as its consumers see them:
// `n` planes at most; with a stream-K map (sk.G > 0) the planes of tile t
// (BN token rows x 128 features) are only the ones its segments wrote, so
// the GEMM zero-fills nothing and consumers read no empty planes.  A plain
// int converts to a uniform count (caller-written planes, op-level API).
struct Planes {
  int n = 1;
  StreamK sk{0, 0, 0, 0};
  int n_tiles = 0, bn = 0;
  int tile_m = 128;  // features per tile (256: the CTA-pair kernel, gemm_2sm.cu)
  Planes() = default;
  Planes(int uniform) : n(uniform) {}  // NOLINT(runtime/explicit)
  __host__ __device__ int count(int row, int feat) const {
    if (sk.G <= 0) return n;
    const int t = (row / bn) * n_tiles + feat / tile_m;
    const long long a = static_cast<long long>(t) * sk.kb;
    return sk.owner(a + sk.kb - 1) - sk.owner(a) + 1;
  }
};

// ---- GEMM fused epilogues (stream-K fixup, gemm_tcgen05.cu) ----
enum { EPI_PLANES = 0, EPI_RESID = 1, EPI_SILU = 2, EPI_QKV = 3 };
struct EpiParams {
  int* tile_sem;  // per-tile semaphores (zeroed once; self-resetting)
  // EPI_RESID: h[t][n] += y
  float* h;
  int ld_h;
  // EPI_SILU: act[t][f] = silu(gate) * up (weights permuted, see permute_rows)
  bf16* act;
  int ld_act;
  // EPI_QKV: RoPE + KV-page scatter (rows < n_batch) / piggyback ship (carry rows)
  const float* rope_cos;
  const float* rope_sin;
  const int* row_pos;
  const int* row_slot;
  int n_batch;
  const int* carry_pos;
  const int* carry_slot;
  bf16* qbuf;
  int q_row_stride;
  bf16* kv_pool;
  KvGeom geom;
  int layer;
  const int* page_table;
  int pt_stride;
  bf16* ship;
  int ship_stride;
  int n_q, n_kv, hd;
};
int gemm_launch_fused(const CUtensorMap& mw, const CUtensorMap& mx, int bn, float* scratch,
                      int n_out, int tokens, int k, int max_planes, int epi, const EpiParams& ep,
                      cudaStream_t st);
int permute_rows(const bf16* src, bf16* dst, int rows, int k, int kind, int a, cudaStream_t st);

// ---- TMA maps / GEMM (gemm_tcgen05.cu) ----
int make_map_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
int make_weight_map(CUtensorMap* map, const bf16* w, int n_out, int k);
int make_act_map(CUtensorMap* map, const bf16* x, int rows, int k, int ld, int bn);
int gemm_pick_bn(int tokens);
int gemm_pick_splits(int n_out, int k, int tokens, int bn, int max_splits);
// Persistent stream-K GEMM; writes `*planes` (<= max_planes) fp32 partial
// planes [planes][tokens][n_out] whose sum is the product.
// step-level launch: per-tile planes, no zero fill (consumers take `Planes`)
// CTA-pair GEMM (gemm_2sm.cu) for >= 256 token rows: same partial-plane
// output; mx_half is the activation map with 128-token boxes.
bool gemm_pair_ok(int n_out, int k, int tokens);
int gemm_launch_pair(const CUtensorMap& mw, const CUtensorMap& mx_half, float* out, int n_out,
                     int tokens, int k, int max_planes, bool uniform_planes, cudaStream_t st,
                     Planes* planes);
int gemm_launch_planes(const CUtensorMap& mw, const CUtensorMap& mx, int bn, float* out, int n_out,
                       int tokens, int k, int max_planes, cudaStream_t st, Planes* planes);
int gemm_launch(const CUtensorMap& mw, const CUtensorMap& mx, int bn, float* out, int n_out,
                int tokens, int k, int max_planes, cudaStream_t st, int* planes,
                bool blocked = false);
// weights pre-tiled [n/128][k/64][128][64] (see gemm_tcgen05.cu)
int relayout_blocked(const bf16* src, bf16* dst, int n, int k, cudaStream_t st);
int make_weight_map_blocked(CUtensorMap* map, const bf16* w, int n_out, int k);

// ---- KV pool: [layers][pages][2 (K,V)][n_kv][64 tokens][head_dim] bf16 ----
int make_kv_map(CUtensorMap* map, const bf16* pool, const KvGeom& g);

// ---- attention (attn_decode.cu / attn_prefill.cu) ----
struct DecodeChunk {
  int row;         // decode row (index into q / output)
  int slot;        // request slot (page-table row)
  int page_begin;  // first logical page of this chunk
  int page_end;    // one past last logical page
  int ctx;         // valid kv tokens of the request (context + new token)
};
int decode_attention(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
                     int q_row_stride, int n_q, const int* page_table, int pt_stride,
                     const DecodeChunk* chunks, int n_chunks, float* o_part, float* lse_part,
                     cudaStream_t st);
// Fused variant: the last CTA of each (row, KV head) LSE-merges the row's
// chunks (self-resetting counters [rows * n_kv], zero-initialised) and writes
// the bf16 output; single-chunk rows are written directly.  rows_whole (every
// row is one chunk): a small launch splits each chunk's pages over a cluster
// of CTAs merged through distributed shared memory.
int decode_attention_fused(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
                           int q_row_stride, int n_q, const int* page_table, int pt_stride,
                           const DecodeChunk* chunks, int n_chunks, const int* row_chunk_begin,
                           float* o_part, float* lse_part, int* counters, bf16* out,
                           int out_row_stride, cudaStream_t st, bool rows_whole = false);
int decode_combine(const float* o_part, const float* lse_part, const int* row_chunk_begin,
                   int rows, int n_q, int n_kv, int head_dim, bf16* out, int out_row_stride,
                   float* lse_out, cudaStream_t st);

struct PrefillTile {
  int slot;   // request slot
  int q_row;  // first row of this tile in q / output
  int pos0;   // absolute position of the tile's first query token
  int nq;     // query rows in this tile (<= 64)
};
int prefill_attention(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
                      int q_row_stride, int n_q, const int* page_table, int pt_stride,
                      const PrefillTile* tiles, int n_tiles, bf16* out, int out_row_stride,
                      cudaStream_t st);
// tcgen05 / TMEM version (attn_prefill_tc.cu): GQA groups share KV pages
int prefill_attention_tc(const CUtensorMap& kv_map, const KvGeom& g, int layer, const bf16* q,
                         int q_row_stride, int n_q, const int* page_table, int pt_stride,
                         const PrefillTile* tiles, int n_tiles, bf16* out, int out_row_stride,
                         cudaStream_t st);

// ---- elementwise (elementwise.cu) ----
int embed_gather(const int* tokens, int rows, const bf16* emb, int d, float* h, cudaStream_t st);
int rmsnorm_rows(const float* h, int rows, int d, const float* w, float eps, bf16* out, int ld_out,
                 cudaStream_t st);
int splitk_reduce(const float* part, int splits, int rows, int n, float* out, cudaStream_t st);
// Row indirections of the add-norm (the piggyback residual store,
// engine.py:982-1004): rows >= src_from start from src[src_idx[r - src_from]]
// instead of h[r] (residual get); rows >= put_from also store their new h
// into put[put_idx[r - put_from]] (residual put).  Zero = plain rows.
struct RowIo {
  const float* src = nullptr;
  const int* src_idx = nullptr;
  int src_from = 0;
  float* put = nullptr;
  const int* put_idx = nullptr;
  int put_from = 0;
  __device__ __forceinline__ const float* row_src(const float* h, int r, int d) const {
    // a negative index is a padding row (device-polled merges): its own row
    const int i = (src_idx && r >= src_from) ? src_idx[r - src_from] : -1;
    return i >= 0 ? src + static_cast<size_t>(i) * d : h + static_cast<size_t>(r) * d;
  }
  __device__ __forceinline__ float* row_put(int r, int d) const {
    const int i = (put_idx && r >= put_from) ? put_idx[r - put_from] : -1;
    return i >= 0 ? put + static_cast<size_t>(i) * d : nullptr;
  }
};
// n rows gathered dst[i] = src[idx[i]] (bf16, width multiple of 8): the host
// attention results of merged rows, folded into the RoPE launch
struct RowCopy {
  const bf16* src = nullptr;
  int src_stride = 0;
  const int* idx = nullptr;
  int n = 0;
  bf16* dst = nullptr;
  int dst_stride = 0;
  int width = 0;
  // completion check (optional): row i is consumed only after its slot's
  // tag (written by the CPU worker after the result) equals expect[i];
  // a mismatch is recorded in fault[0..3] = {1, slot, layer, tag seen}
  const int* expect = nullptr;
  const unsigned* tags = nullptr;
  unsigned* fault = nullptr;
  int layer = 0;
};
int residual_add_norm(const float* part, const Planes& splits, int rows, int d, float* h, const float* w,
                      float eps, bf16* out, int ld_out, cudaStream_t st, const RowIo& io = RowIo{});

// ---- tensor parallelism: the all-reduce of a row-parallel projection fused
// into its residual-add + RMSNorm (elementwise.cu).  Every rank publishes its
// local partial rows into its own exchange buffer and raises a per-(row,
// column block) flag; peers read the partials straight from that memory
// (NVLink P2P through CUDA IPC, or the same device for a single-process
// group) once the flag shows the exchange's epoch, and all ranks sum them in
// rank order, so the new residual stream is bit-identical on every rank.
constexpr int kMaxTp = 8;
struct TpPeers {
  float* xbuf[kMaxTp];      // each rank's exchange buffer [2][max_rows][d] fp32
  unsigned* flag[kMaxTp];   // each rank's flags [2][max_rows * 8]
  int world = 1, me = 0;
  size_t xbuf_par = 0;      // floats per parity
  size_t flag_par = 0;      // flags per parity
};
int tp_add_norm(const float* part, const Planes& splits, int rows, int d, float* h, const float* w,
                float eps, bf16* out, int ld_out, cudaStream_t st, const RowIo& io,
                const TpPeers& peers, unsigned epoch);
// rows [0, n_batch): row_* arrays (row_mode may be null = all KV-scatter);
// rows [n_batch, rows): carry_* arrays, shipped to the host mailbox
int qkv_rope_scatter(const float* part, const Planes& splits, int rows, int n_q, int n_kv, int head_dim,
                     const float* rope_cos, const float* rope_sin, const int* row_pos,
                     const int* row_slot, const int* row_mode, int n_batch, const int* carry_pos,
                     const int* carry_slot, bf16* qbuf, int q_row_stride, bf16* kv_pool,
                     const KvGeom& g, int layer, const int* page_table, int pt_stride, bf16* ship,
                     int ship_stride, cudaStream_t st, int permuted = 0,
                     const RowCopy& rc = RowCopy{});
int silu_mul(const float* part, const Planes& splits, int rows, int ffn, bf16* act, int ld_act,
             cudaStream_t st, int permuted = 0);
int argmax_rows(const float* part, const Planes& splits, int rows, int vocab, int* tokens, float* logits_out,
                cudaStream_t st);
int lse_merge_rows(const bf16* parts, const float* lse, int n_parts, int rows, int n_q,
                   int head_dim, int part_stride, int row_stride_parts, bf16* out,
                   int out_row_stride, cudaStream_t st);

}  // namespace hs
