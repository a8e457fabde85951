// extern "C" op-level entry points (include/hs.h) over the internal launchers.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <ctime>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {
thread_local char g_last_error[512] = {0};
unsigned long long g_launches = 0;
int g_hprof_on = [] {
  const char* e = getenv("HS_HOST_PROF");
  return e && e[0] == '1' ? 1 : 0;
}();
double g_hprof_ns[8] = {0};
unsigned long long g_hprof_n[8] = {0};
double hprof_now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e9 + ts.tv_nsec;
}

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}

static int cuda_status(int rc, const char* what) {
  if (rc == HS_OK) return HS_OK;
  if (rc == HS_E_CUDA) {
    cudaError_t e = cudaGetLastError();
    return set_error(HS_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
  }
  return set_error(rc, "%s: invalid configuration", what);
}
}  // namespace hs

using namespace hs;

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

const char* hs_version(void) { return "libhs 0.1 sm_100a"; }

int hs_last_error(char* buf, int cap) {
  const int n = static_cast<int>(strlen(g_last_error));
  if (buf && cap > 0) {
    strncpy(buf, g_last_error, cap - 1);
    buf[cap - 1] = 0;
  }
  return n;
}

unsigned long long hs_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int hs_device_ok(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return p.major == 10 ? 1 : 0;
}

int hs_op_gemm_bf16(const void* x, int tokens, int ldx, const void* w, int n_out, int k,
                    float* out_partial, int max_splits, int* splits_used, void* stream) {
  if (tokens < 0 || n_out % 128 || k % 64 || ldx < k || max_splits < 1)
    return set_error(HS_E_CONFIG, "gemm: bad shape tokens=%d n=%d k=%d ldx=%d", tokens, n_out, k,
                     ldx);
  if (tokens == 0) {
    if (splits_used) *splits_used = 1;
    return HS_OK;
  }
  const int bn = gemm_pick_bn(tokens);
  CUtensorMap mw, mx;
  if (make_weight_map(&mw, static_cast<const bf16*>(w), n_out, k) != HS_OK ||
      make_act_map(&mx, static_cast<const bf16*>(x), tokens, k, ldx, bn) != HS_OK)
    return set_error(HS_E_CUDA, "gemm: cuTensorMapEncodeTiled failed");
  int planes = 1;
  const int rc = gemm_launch(mw, mx, bn, out_partial, n_out, tokens, k, max_splits, S(stream),
                             &planes);
  if (splits_used) *splits_used = planes;
  return cuda_status(rc, "gemm");
}

int hs_op_gemm_bf16_pair(const void* x, int tokens, int ldx, const void* w, int n_out, int k,
                         float* out_partial, int max_splits, int* splits_used, void* stream) {
  if (tokens < 256 || n_out % 256 || k % 64 || ldx < k || max_splits < 1)
    return set_error(HS_E_CONFIG, "gemm_pair: bad shape tokens=%d n=%d k=%d ldx=%d", tokens,
                     n_out, k, ldx);
  CUtensorMap mw, mx;
  if (make_weight_map(&mw, static_cast<const bf16*>(w), n_out, k) != HS_OK ||
      make_act_map(&mx, static_cast<const bf16*>(x), tokens, k, ldx, 128) != HS_OK)
    return set_error(HS_E_CUDA, "gemm_pair: cuTensorMapEncodeTiled failed");
  Planes planes;
  const int rc = gemm_launch_pair(mw, mx, out_partial, n_out, tokens, k, max_splits, true,
                                  S(stream), &planes);
  if (splits_used) *splits_used = planes.n;
  return cuda_status(rc, "gemm_pair");
}

int hs_op_relayout_blocked(const void* w, void* w_blocked, int n, int k, void* stream) {
  return cuda_status(relayout_blocked(static_cast<const bf16*>(w), static_cast<bf16*>(w_blocked),
                                      n, k, S(stream)),
                     "relayout_blocked");
}

int hs_op_gemm_bf16_blocked(const void* x, int tokens, int ldx, const void* w_blocked, int n_out,
                            int k, float* out_partial, int max_splits, int* splits_used,
                            void* stream) {
  if (tokens < 0 || n_out % 128 || k % 64 || ldx < k || max_splits < 1)
    return set_error(HS_E_CONFIG, "gemm: bad shape tokens=%d n=%d k=%d", tokens, n_out, k);
  if (tokens == 0) {
    if (splits_used) *splits_used = 1;
    return HS_OK;
  }
  const int bn = gemm_pick_bn(tokens);
  CUtensorMap mw, mx;
  if (make_weight_map_blocked(&mw, static_cast<const bf16*>(w_blocked), n_out, k) != HS_OK ||
      make_act_map(&mx, static_cast<const bf16*>(x), tokens, k, ldx, bn) != HS_OK)
    return set_error(HS_E_CUDA, "gemm: cuTensorMapEncodeTiled failed");
  int planes = 1;
  const int rc = gemm_launch(mw, mx, bn, out_partial, n_out, tokens, k, max_splits, S(stream),
                             &planes, true);
  if (splits_used) *splits_used = planes;
  return cuda_status(rc, "gemm_blocked");
}

int hs_op_splitk_reduce(const float* part, int splits, int rows, int n, float* out,
                        void* stream) {
  return cuda_status(splitk_reduce(part, splits, rows, n, out, S(stream)), "splitk_reduce");
}

int hs_op_decode_attention(const void* kv_pool, int layers, int pages, int n_kv, int head_dim,
                           int layer, const void* q, int q_row_stride, int n_q,
                           const int* page_table, int pt_stride, const int* chunks, int n_chunks,
                           float* o_part, float* lse_part, void* stream) {
  KvGeom g{layers, pages, n_kv, head_dim};
  CUtensorMap m;
  if (make_kv_map(&m, static_cast<const bf16*>(kv_pool), g) != HS_OK)
    return set_error(HS_E_CUDA, "decode: kv map encode failed");
  return cuda_status(
      decode_attention(m, g, layer, static_cast<const bf16*>(q), q_row_stride, n_q, page_table,
                       pt_stride, reinterpret_cast<const DecodeChunk*>(chunks), n_chunks, o_part,
                       lse_part, S(stream)),
      "decode_attention");
}

int hs_op_decode_attention_fused(const void* kv_pool, int layers, int pages, int n_kv,
                                 int head_dim, int layer, const void* q, int q_row_stride, int n_q,
                                 const int* page_table, int pt_stride, const int* chunks,
                                 int n_chunks, int rows, const int* row_chunk_begin, float* o_part,
                                 float* lse_part, int* counters, void* out, int out_row_stride,
                                 void* stream) {
  KvGeom g{layers, pages, n_kv, head_dim};
  CUtensorMap m;
  if (make_kv_map(&m, static_cast<const bf16*>(kv_pool), g) != HS_OK)
    return set_error(HS_E_CUDA, "decode: kv map encode failed");
  return cuda_status(
      decode_attention_fused(m, g, layer, static_cast<const bf16*>(q), q_row_stride, n_q,
                             page_table, pt_stride, reinterpret_cast<const DecodeChunk*>(chunks),
                             n_chunks, row_chunk_begin, o_part, lse_part, counters,
                             static_cast<bf16*>(out), out_row_stride, S(stream), n_chunks == rows),
      "decode_attention_fused");
}

int hs_op_decode_combine(const float* o_part, const float* lse_part, const int* row_chunk_begin,
                         int rows, int n_q, int n_kv, int head_dim, void* out,
                         int out_row_stride, float* lse_out, void* stream) {
  return cuda_status(decode_combine(o_part, lse_part, row_chunk_begin, rows, n_q, n_kv, head_dim,
                                    static_cast<bf16*>(out), out_row_stride, lse_out, S(stream)),
                     "decode_combine");
}

int hs_op_prefill_attention(const void* kv_pool, int layers, int pages, int n_kv, int head_dim,
                            int layer, const void* q, int q_row_stride, int n_q,
                            const int* page_table, int pt_stride, const int* tiles, int n_tiles,
                            void* out, int out_row_stride, void* stream) {
  KvGeom g{layers, pages, n_kv, head_dim};
  CUtensorMap m;
  if (make_kv_map(&m, static_cast<const bf16*>(kv_pool), g) != HS_OK)
    return set_error(HS_E_CUDA, "prefill: kv map encode failed");
  return cuda_status(
      prefill_attention(m, g, layer, static_cast<const bf16*>(q), q_row_stride, n_q, page_table,
                        pt_stride, reinterpret_cast<const PrefillTile*>(tiles), n_tiles,
                        static_cast<bf16*>(out), out_row_stride, S(stream)),
      "prefill_attention");
}

int hs_op_embed(const int* tokens, int rows, const void* emb, int d, float* h, void* stream) {
  return cuda_status(embed_gather(tokens, rows, static_cast<const bf16*>(emb), d, h, S(stream)),
                     "embed");
}

int hs_op_rmsnorm(const float* h, int rows, int d, const float* w, float eps, void* out,
                  int ld_out, void* stream) {
  return cuda_status(rmsnorm_rows(h, rows, d, w, eps, static_cast<bf16*>(out), ld_out, S(stream)),
                     "rmsnorm");
}

int hs_op_residual_add_norm(const float* part, int splits, int rows, int d, float* h,
                            const float* w, float eps, void* out, int ld_out, void* stream) {
  return cuda_status(residual_add_norm(part, splits, rows, d, h, w, eps, static_cast<bf16*>(out),
                                       ld_out, S(stream)),
                     "residual_add_norm");
}

int hs_op_qkv_rope_scatter(const float* part, int splits, int rows, int n_q, int n_kv,
                           int head_dim, const float* rope_cos, const float* rope_sin,
                           const int* row_pos, const int* row_slot, const int* row_mode,
                           void* qbuf, int q_row_stride, void* kv_pool, int layers, int pages,
                           int layer, const int* page_table, int pt_stride, void* ship,
                           int ship_stride, void* stream) {
  KvGeom g{layers, pages, n_kv, head_dim};
  return cuda_status(
      qkv_rope_scatter(part, splits, rows, n_q, n_kv, head_dim, rope_cos, rope_sin, row_pos,
                       row_slot, row_mode, rows, nullptr, nullptr, static_cast<bf16*>(qbuf),
                       q_row_stride,
                       static_cast<bf16*>(kv_pool), g, layer, page_table, pt_stride,
                       static_cast<bf16*>(ship), ship_stride, S(stream)),
      "qkv_rope_scatter");
}

int hs_op_silu_mul(const float* part, int splits, int rows, int ffn, void* act, int ld_act,
                   void* stream) {
  return cuda_status(silu_mul(part, splits, rows, ffn, static_cast<bf16*>(act), ld_act, S(stream)),
                     "silu_mul");
}

int hs_op_argmax(const float* part, int splits, int rows, int vocab, int* tokens,
                 float* logits_out, void* stream) {
  return cuda_status(argmax_rows(part, splits, rows, vocab, tokens, logits_out, S(stream)),
                     "argmax");
}

int hs_op_lse_merge(const void* parts, const float* lse, int n_parts, int rows, int n_q,
                    int head_dim, int part_stride, int row_stride_parts, void* out,
                    int out_row_stride, void* stream) {
  return cuda_status(lse_merge_rows(static_cast<const bf16*>(parts), lse, n_parts, rows, n_q,
                                    head_dim, part_stride, row_stride_parts,
                                    static_cast<bf16*>(out), out_row_stride, S(stream)),
                     "lse_merge");
}

}  // extern "C"
