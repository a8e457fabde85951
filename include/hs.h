/*
 * libhs — C ABI of the B200-native OmniServe serving step.
 *
 * The reference (arxiv 2603.12831, package `hybridserve`) has no FFI: its
 * "device" is the pure-Python cost oracle
 *   probe_dense(profile, n, rng)                 pkg/src/hybridserve/profiles.py:132-143
 *   probe_attention(profile, phase, c, g, rng)   pkg/src/hybridserve/profiles.py:146-169
 * called from Engine._run_layer (pkg/src/hybridserve/engine.py:921-950), with
 * the CPU attention service in Engine._maybe_start_host / _on_service_done /
 * _on_result (engine.py:529-560) and the residual store in ResidualStore
 * (engine.py:133-161).  libhs replaces those charges with real work; every
 * entry point below names the reference site it stands in for.  The
 * reference-side ctypes binding a maintainer would add is in INTEGRATION.md.
 *
 * Conventions: plain pointers and sizes only; `stream` is a cudaStream_t
 * passed as void* (NULL = legacy default stream).  Every function returns an
 * int status; no exception crosses the ABI.  Status -> reference exception:
 *   HS_E_CONFIG    -> ConfigError          (errors.py:4)
 *   HS_E_INTEGRITY -> IntegrityFault       (errors.py:12-18)
 *   HS_E_CAPACITY  -> ScenarioError        (errors.py:21)
 *   HS_E_CUDA      -> RuntimeError
 * Details of the most recent failure on the calling thread: hs_last_error().
 */
#ifndef HS_H_
#define HS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define HS_OK 0
#define HS_E_CONFIG 1
#define HS_E_INTEGRITY 2
#define HS_E_CAPACITY 3
#define HS_E_CUDA 4

#define HS_PAGE_TOKENS 64

/* ---------------------------------------------------------------- library */
const char* hs_version(void);
/* Copies the calling thread's last error message; returns its length. */
int hs_last_error(char* buf, int cap);
/* 1 if a CUDA device of compute capability 10.x is visible. */
int hs_device_ok(void);

/* -------------------------------------------------------------- op level
 * Single-kernel entry points over caller-owned device buffers.  They are the
 * building blocks of hs_layer() below and are exported so parity tests can
 * check each kernel against the CPU oracle in isolation.
 */

/* K3 Dense (probe_dense, profiles.py:132-143): fp32 split-K partials
 * out[s][t][n] = sum_{k in split s} x[t][k] * w[n][k]  (bf16 in, tcgen05).
 * n_out % 128 == 0, k % 64 == 0.  *splits_used <= max_splits. */
int hs_op_gemm_bf16(const void* x, int tokens, int ldx, const void* w, int n_out, int k,
                    float* out_partial, int max_splits, int* splits_used, void* stream);
/* out[t][n] = sum_s part[s][t][n] */
int hs_op_splitk_reduce(const float* part, int splits, int rows, int n, float* out,
                        void* stream);

/* KV pool: [layers][pages][2][n_kv][64][head_dim] bf16 (one TMA-able tensor). */
/* K1 decode attention (probe_attention DECODE, engine.py:939-942).
 * chunks: device int32[n_chunks][5] = {row, slot, page_begin, page_end, ctx}.
 * o_part: [n_chunks][n_q][head_dim] fp32, lse_part: [n_chunks][n_q] fp32. */
int hs_op_decode_attention(const void* kv_pool, int layers, int pages, int n_kv, int head_dim,
                           int layer, const void* q, int q_row_stride, int n_q,
                           const int* page_table, int pt_stride, const int* chunks, int n_chunks,
                           float* o_part, float* lse_part, void* stream);
/* K2: LSE-merge the chunks of each row (row_chunk_begin: int32[rows+1]). */
int hs_op_decode_combine(const float* o_part, const float* lse_part, const int* row_chunk_begin,
                         int rows, int n_q, int n_kv, int head_dim, void* out,
                         int out_row_stride, float* lse_out, void* stream);
/* K6 chunked causal prefill (probe_attention PREFILL, engine.py:935-938).
 * tiles: device int32[n_tiles][4] = {slot, q_row, pos0, nq<=64}. */
int hs_op_prefill_attention(const void* kv_pool, int layers, int pages, int n_kv, int head_dim,
                            int layer, const void* q, int q_row_stride, int n_q,
                            const int* page_table, int pt_stride, const int* tiles, int n_tiles,
                            void* out, int out_row_stride, void* stream);
/* K8 embedding gather: h[r][:] = emb[tokens[r]][:] (fp32 residual stream). */
int hs_op_embed(const int* tokens, int rows, const void* emb, int d, float* h, void* stream);
/* K4 RMSNorm: out = bf16(h * rsqrt(mean(h^2)+eps) * w). */
int hs_op_rmsnorm(const float* h, int rows, int d, const float* w, float eps, void* out,
                  int ld_out, void* stream);
/* h += sum_s part[s]; out = RMSNorm(h)*w if out != NULL ("ResidualAdd",
 * engine.py:56). */
int hs_op_residual_add_norm(const float* part, int splits, int rows, int d, float* h,
                            const float* w, float eps, void* out, int ld_out, void* stream);
/* K5 QKV epilogue: split-K reduce, rotate-half RoPE, then per row
 * mode 0 -> q to qbuf, k/v to the row's KV page at row_pos;
 * mode 1 -> q|k|v to ship[row_slot] (piggyback D2H, engine.py:982-989). */
int hs_op_qkv_rope_scatter(const float* part, int splits, int rows, int n_q, int n_kv,
                           int head_dim, const float* rope_cos, const float* rope_sin,
                           const int* row_pos, const int* row_slot, const int* row_mode,
                           void* qbuf, int q_row_stride, void* kv_pool, int layers, int pages,
                           int layer, const int* page_table, int pt_stride, void* ship,
                           int ship_stride, void* stream);
/* SwiGLU: act = silu(gate) * up from split-K partials of [gate | up]. */
int hs_op_silu_mul(const float* part, int splits, int rows, int ffn, void* act, int ld_act,
                   void* stream);
/* K9 greedy argmax over split-K LM-head partials (lowest index on ties);
 * logits_out (fp32 [rows][vocab]) may be NULL. */
int hs_op_argmax(const float* part, int splits, int rows, int vocab, int* tokens,
                 float* logits_out, void* stream);
/* K2 on the piggyback path: merge n_parts normalised partials (bf16) with
 * natural-log LSEs into one bf16 row per (row, head). */
int hs_op_lse_merge(const void* parts, const float* lse, int n_parts, int rows, int n_q,
                    int head_dim, int part_stride, int row_stride_parts, void* out,
                    int out_row_stride, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* HS_H_ */
