// Row-routing kernels of the piggyback step: token selection, residual-store
// get/put (reference ResidualStore, engine.py:133-161), merged-row gathers
// from the host result mailboxes (the H2D half of Attention Piggybacking,
// engine.py:556-560 -> 991-1003), last-token scatter after the LM head, and
// KV swap between the paged pool and the host KV arena (engine.py:421-508).
#include "hs_common.cuh"
#include "hs_internal.h"
#include "hs_step.h"

namespace hs {

// rows < n_batch: tok = row_token >= 0 ? row_token : last_token[row_slot];
// rows >= n_batch (carry rows): tok = last_token[carry_slot]
__global__ void select_tokens_kernel(const int* __restrict__ row_token,
                                     const int* __restrict__ row_slot, int n_batch,
                                     const int* __restrict__ carry_slot,
                                     const int* __restrict__ last_token, int rows,
                                     int* __restrict__ tok) {
  pdl_wait();  // dependent data of the previous kernel is visible
  pdl_trigger();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  if (r >= n_batch) {  // a negative slot is a padding row (device-polled merges)
    const int cs = carry_slot[r - n_batch];
    tok[r] = cs >= 0 ? last_token[cs] : 0;
    return;
  }
  const int t = row_token[r];
  tok[r] = t >= 0 ? t : last_token[row_slot[r]];
}

// dst[r] = src[idx[r]]  (fp32 rows of width d)
__global__ void gather_rows_f32_kernel(const float* __restrict__ src, const int* __restrict__ idx,
                                       int d, float* __restrict__ dst) {
  pdl_wait();  // dependent data of the previous kernel is visible
  pdl_trigger();
  const int r = blockIdx.x;
  if (idx[r] < 0) return;  // padding row
  const float4* s = reinterpret_cast<const float4*>(src + static_cast<size_t>(idx[r]) * d);
  float4* o = reinterpret_cast<float4*>(dst + static_cast<size_t>(r) * d);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) o[i] = s[i];
}

// dst[idx[r]] = src[r]
__global__ void scatter_rows_f32_kernel(const float* __restrict__ src, const int* __restrict__ idx,
                                        int d, float* __restrict__ dst) {
  pdl_wait();  // dependent data of the previous kernel is visible
  pdl_trigger();
  const int r = blockIdx.x;
  if (idx[r] < 0) return;  // padding row
  const float4* s = reinterpret_cast<const float4*>(src + static_cast<size_t>(r) * d);
  float4* o = reinterpret_cast<float4*>(dst + static_cast<size_t>(idx[r]) * d);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) o[i] = s[i];
}

// bf16 rows (width w elements, multiple of 8): dst[r] = src_base + idx[r]*src_stride
__global__ void gather_rows_bf16_kernel(const bf16* __restrict__ src, int src_stride,
                                        const int* __restrict__ idx, int w, bf16* __restrict__ dst,
                                        int dst_stride) {
  pdl_wait();  // dependent data of the previous kernel is visible
  pdl_trigger();
  const int r = blockIdx.x;
  const int4* s = reinterpret_cast<const int4*>(src + static_cast<size_t>(idx[r]) * src_stride);
  int4* o = reinterpret_cast<int4*>(dst + static_cast<size_t>(r) * dst_stride);
  for (int i = threadIdx.x; i < w / 8; i += blockDim.x) o[i] = s[i];
}

__global__ void scatter_tokens_kernel(const int* __restrict__ tok, const int* __restrict__ slot,
                                      int n, int* __restrict__ last_token) {
  pdl_wait();  // dependent data of the previous kernel is visible
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && slot[i] >= 0) last_token[slot[i]] = tok[i];
}

// Swap: copy `tokens` KV entries of one request between its pool pages and
// a host KV region laid out [layers][2][n_kv][cap][hd] (mapped pinned
// memory, written/read by the SMs over PCIe).
template <bool kToHost>
__global__ void kv_swap_kernel(bf16* __restrict__ pool, KvGeom g, const int* __restrict__ pages,
                               int tokens, bf16* __restrict__ host, int cap) {
  pdl_wait();  // dependent data of the previous kernel is visible
  pdl_trigger();
  // grid.x = layers*2*n_kv, grid.y = token tiles of 64
  const int lkh = blockIdx.x;
  const int h = lkh % g.n_kv;
  const int kv = (lkh / g.n_kv) % 2;
  const int layer = lkh / (2 * g.n_kv);
  const int tile = blockIdx.y;
  const int t0 = tile * kPageTokens;
  if (t0 >= tokens) return;
  const int nt = min(kPageTokens, tokens - t0);
  bf16* dev = pool + kv_row(g, layer, pages[tile], kv, h) * g.head_dim;
  bf16* hst = host + ((static_cast<size_t>(layer) * 2 + kv) * g.n_kv + h) * cap * g.head_dim +
              static_cast<size_t>(t0) * g.head_dim;
  const int n16 = nt * g.head_dim / 8;
  for (int i = threadIdx.x; i < n16; i += blockDim.x) {
    if (kToHost)
      reinterpret_cast<int4*>(hst)[i] = reinterpret_cast<const int4*>(dev)[i];
    else
      reinterpret_cast<int4*>(dev)[i] = reinterpret_cast<const int4*>(hst)[i];
  }
}

// ------------------------------------------------------------------ launchers
int select_tokens(const int* row_token, const int* row_slot, int n_batch, const int* carry_slot,
                  const int* last_token, int rows, int* tok, cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  return launch_pdl(select_tokens_kernel, dim3((rows + 127) / 128), dim3(128), 0, st, row_token, row_slot, n_batch, carry_slot, last_token, rows, tok);
}

int gather_rows_f32(const float* src, const int* idx, int rows, int d, float* dst,
                    cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  return launch_pdl(gather_rows_f32_kernel, dim3(rows), dim3(256), 0, st, src, idx, d, dst);
}

int scatter_rows_f32(const float* src, const int* idx, int rows, int d, float* dst,
                     cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  return launch_pdl(scatter_rows_f32_kernel, dim3(rows), dim3(256), 0, st, src, idx, d, dst);
}

int gather_rows_bf16(const bf16* src, int src_stride, const int* idx, int rows, int w, bf16* dst,
                     int dst_stride, cudaStream_t st) {
  if (rows <= 0) return HS_OK;
  return launch_pdl(gather_rows_bf16_kernel, dim3(rows), dim3(128), 0, st, src, src_stride, idx, w, dst, dst_stride);
}

int scatter_tokens(const int* tok, const int* slot, int n, int* last_token, cudaStream_t st) {
  if (n <= 0) return HS_OK;
  return launch_pdl(scatter_tokens_kernel, dim3((n + 127) / 128), dim3(128), 0, st, tok, slot, n, last_token);
}

int kv_swap(bool to_host, bf16* pool, const KvGeom& g, const int* pages, int tokens, bf16* host,
            int cap, cudaStream_t st) {
  if (tokens <= 0) return HS_OK;
  dim3 grid(g.layers * 2 * g.n_kv, (tokens + kPageTokens - 1) / kPageTokens);
  if (to_host)
    return launch_pdl(kv_swap_kernel<true>, grid, dim3(256), 0, st, pool, g, pages, tokens, host,
                      cap);
  return launch_pdl(kv_swap_kernel<false>, grid, dim3(256), 0, st, pool, g, pages, tokens, host,
                    cap);
}

}  // namespace hs
