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
/* number of kernels libhs has launched in this process */
unsigned long long hs_launch_count(void);

/* C1 on the calling thread: decode attention of one row (q [n_q][hd] bf16)
 * over K/V [n_kv][n_keys][hd] bf16 -> out [n_q][hd] bf16, lse [n_q] (natural
 * log, may be NULL).  impl: 0 = best available, 1 = AVX-512-BF16, 2 = AVX2.
 * Pure host code (no device needed). */
int hs_host_attention(const void* q, const void* k, const void* v, int n_keys, int n_q, int n_kv,
                      int head_dim, void* out, float* lse, int impl);

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
/* Same product on CTA pairs (tcgen05.mma.cta_group::2, 256 weight rows x
 * 256 tokens per pair tile; the step uses it from 256 rows up).
 * tokens >= 256, n_out % 256 == 0, k % 64 == 0. */
int hs_op_gemm_bf16_pair(const void* x, int tokens, int ldx, const void* w, int n_out, int k,
                         float* out_partial, int max_splits, int* splits_used, void* stream);
/* Same product with the weights pre-tiled [n/128][k/64][128][64] (each
 * 16 KB TMA box contiguous in HBM); hs_op_relayout_blocked converts. */
int hs_op_relayout_blocked(const void* w, void* w_blocked, int n, int k, void* stream);
int hs_op_gemm_bf16_blocked(const void* x, int tokens, int ldx, const void* w_blocked, int n_out,
                            int k, float* out_partial, int max_splits, int* splits_used,
                            void* stream);
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
/* K1+K2 fused: the last CTA of each (row, KV head) merges the row's chunks
 * and writes out[row] (bf16); counters: int32[rows * n_kv], zeroed once
 * (the kernel resets them).  rows: decode rows of the list; when every row
 * is one chunk (n_chunks == rows) a small launch splits each row's pages
 * over a thread-block cluster merged in distributed shared memory. */
int hs_op_decode_attention_fused(const void* kv_pool, int layers, int pages, int n_kv,
                                 int head_dim, int layer, const void* q, int q_row_stride, int n_q,
                                 const int* page_table, int pt_stride, const int* chunks,
                                 int n_chunks, int rows, const int* row_chunk_begin, float* o_part,
                                 float* lse_part, int* counters, void* out, int out_row_stride,
                                 void* stream);
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

/* ------------------------------------------------------------ step level
 * One context per GPU replica.  It owns the weights, the paged KV pool, the
 * device residual store (ResidualStore, engine.py:133-161), the pinned
 * piggyback mailboxes (one q|k|v ship row and one result row per request
 * slot: a chain has at most one item in flight, engine.py:982-1022), the
 * pinned host KV arena of offloaded requests and the CPU-attention pool.
 */
typedef struct hs_ctx hs_ctx;

typedef struct {
  int d_model, n_layers, n_q, n_kv, head_dim, ffn, vocab;
  float rope_theta, norm_eps;
} hs_model_cfg;

typedef struct {
  int max_rows;          /* batch tokens + piggyback rows entering one layer   */
  int max_slots;         /* concurrent requests                                 */
  int kv_pages;          /* 64-token pages in the GPU KV pool                   */
  int max_pages_per_req; /* page-table width                                    */
  int max_pos;           /* RoPE table length                                   */
  int max_chunks;        /* split-K decode-attention work items per layer       */
  int cpu_threads;       /* CPU attention workers of this replica               */
  int64_t host_kv_bytes; /* pinned host KV arena (offloaded BE requests)        */
  int device;
  /* the replica's CPU-attention core set (NUMA node of `device`, split among
     the GPUs on that node; "private queues, equal CPU share").
     Workers are pinned to these cores and the pinned host arenas are
     first-touched from them.  NULL / 0 = no pinning. */
  const int* cpu_list;
  int n_cpu_list;
  /* HS_PREC_BF16: the serving datapath (bf16 weights / activations / KV, fp32
     accumulation and residual stream, tcgen05 GEMMs).  HS_PREC_FP32: the
     validation datapath (north star: logits within 1e-4 of the fp32 oracle,
     greedy tokens identical over the first 64 steps) -- fp32 weights,
     activations, KV pool, piggyback mailboxes, host KV and CPU attention,
     SIMT kernels on the same device; probes and tensor parallelism are
     bf16-only. */
  int precision;
} hs_rt_cfg;
#define HS_PREC_BF16 0
#define HS_PREC_FP32 1

enum {
  HS_W_EMBED = 0, HS_W_LM_HEAD = 1, HS_W_FINAL_NORM = 2, HS_W_QKV = 3, HS_W_O = 4,
  HS_W_GATE_UP = 5, HS_W_DOWN = 6, HS_W_NORM_IN = 7, HS_W_NORM_POST = 8
};

/* Engine.__init__ (engine.py:251-298) device side. */
int hs_create(const hs_model_cfg* model, const hs_rt_cfg* rt, hs_ctx** out);
int hs_destroy(hs_ctx* ctx);
void* hs_stream(hs_ctx* ctx);

/* Tensor parallelism (config 4; the reference folds it into gamma,
 * engine.py:944 / latency.py:141-147).  Each rank's context holds its shard
 * (q/kv heads and ffn columns; O and down row-parallel); the two all-reduces
 * per layer are fused into the residual-add + RMSNorm launches and read the
 * peers' partials over NVLink P2P.  Multi-process: every rank exports its
 * exchange handles (HS_TP_HANDLE_BYTES), the caller all-gathers them (e.g.
 * torch.distributed over gloo) and passes all ranks' handles in rank order to
 * hs_tp_open.  Every rank must then issue the same sequence of hs_layer
 * calls with the same row counts (identical, deterministic engines). */
#define HS_TP_HANDLE_BYTES 128
int hs_tp_export(hs_ctx* ctx, void* handles /* HS_TP_HANDLE_BYTES */);
int hs_tp_open(hs_ctx* ctx, int rank, int world, const void* all_handles /* world x 128 */);
/* bf16 matrices [out][in] (qkv rows: q heads, k heads, v heads; gate_up
 * rows: gate then up), fp32 norm vectors.  Layer is 0-based. */
int hs_set_weight(hs_ctx* ctx, int kind, int layer, const void* host, size_t bytes);
/* synthetic N(0, std) bf16 weights generated on the device, norms = 1 */
int hs_init_weights(hs_ctx* ctx, uint64_t seed, float std);
/* page ids of a request slot (KvManager token accounting, engine.py:194-230) */
int hs_set_page_table(hs_ctx* ctx, int slot, const int* pages, int n);

/* host KV of offloaded requests (_distribute_offload, engine.py:402-419) */
int hs_host_kv_reserve(hs_ctx* ctx, int slot, int cap_tokens);
int hs_host_kv_release(hs_ctx* ctx, int slot);
int hs_host_kv_ptr(hs_ctx* ctx, int slot, void** host_ptr, int* cap_tokens);
/* one-shot KV transfer of `tokens` entries (swap-out / swap-in,
 * engine.py:421-508): GPU pages of the slot <-> its host region */
int hs_swap_out(hs_ctx* ctx, int slot, int tokens);
int hs_swap_in(hs_ctx* ctx, int slot, int tokens);

/* Iteration (BatchPlan) descriptor; rows = decodes first, then chunk tokens. */
typedef struct {
  int n_rows, n_decode;
  const int* row_slot;   /* [n_rows] */
  const int* row_pos;    /* [n_rows] absolute position of the row's token */
  const int* row_token;  /* [n_rows] token id, or -1 = the slot's last generated token */
  int n_chunks;
  const int* chunks;          /* [n_chunks][5] decode split-K work items */
  const int* row_chunk_begin; /* [n_decode+1] */
  int n_tiles;
  const int* tiles;      /* [n_tiles][4] prefill tiles */
  int n_logit_rows;
  const int* logit_rows; /* rows producing a token at the last layer */
} hs_iter_desc;

/* Per-layer piggyback descriptor (_consume_merges + _process_merge,
 * engine.py:902-1022). */
typedef struct {
  int layer;             /* 1-based */
  int n_carry;           /* QKV(layer)-only rows shipped to the host: layer 1 =
                            injected fresh tokens, else chains merged at layer-1 */
  const int* carry_slot;
  const int* carry_pos;
  int n_merge;           /* host results merged at this layer (Proj + MLP) */
  const int* merge_slot;
  int n_restart;         /* last layer: merged chains continuing with the next
                            token (embed + QKV(1) + ship) */
  const int* restart_idx;  /* indices into merge_slot */
  const int* restart_pos;
  const int* merge_tag;  /* optional (NULL = unchecked): the completion tag each
                            merged result must carry, HS_RESULT_TAG(ctx, layer)
                            of its work item; the device verifies it before
                            consuming the row and hs_iter_end / hs_iter_poll
                            report a mismatch as HS_E_INTEGRITY */
} hs_layer_desc;
/* completion tag a CPU worker publishes (release) after writing a work
 * item's result row: item context length and 1-based layer */
#define HS_RESULT_TAG(ctx, layer) ((int)(((unsigned)(ctx) << 8) | (unsigned)(layer)))

int hs_iter_begin(hs_ctx* ctx, const hs_iter_desc* desc);
/* Engine._run_layer (engine.py:921-950) on the device. */
int hs_layer(hs_ctx* ctx, const hs_layer_desc* desc);
/* Waits for the iteration; copies its greedy tokens (logit rows, then the
 * chains merged at the last layer) and returns their count. */
int hs_iter_end(hs_ctx* ctx, int* tokens_out, int n);
/* CPU attention service of n work items (slot, 1-based layer, ctx):
 * appends each item's new k/v to the host KV and writes the attention
 * result row into the slot's result mailbox (engine.py:529-560). */
int hs_cpu_attend(hs_ctx* ctx, const int* slots, const int* layers, const int* ctxs, int n);
/* Waits for the compute stream and the swap copy stream. */
int hs_sync(hs_ctx* ctx);

/* ------------------------------------------------------------ live mode
 * Asynchronous counterparts used by the wall-clock engine: the GPU never
 * waits on the host.  Work items shipped by the last hs_layer() call are
 * submitted behind a CUDA event; worker threads (pinned to this replica's
 * cores) service them and append completions to a FIFO (the reference's
 * output queue, engine.py:181-191,556-560).  Swaps run on a low-priority
 * copy stream (pack + one 2D DMA); hs_swap_done polls a ticket. */
int hs_cpu_submit(hs_ctx* ctx, const int* slots, const int* layers, const int* ctxs, int n);
int hs_cpu_poll(hs_ctx* ctx, int* slots, int* layers, double* t_done, int max);
int hs_cpu_in_flight(hs_ctx* ctx);
double hs_cpu_busy_seconds(hs_ctx* ctx);
double hs_wall_seconds(void);
int hs_swap_out_async(hs_ctx* ctx, int slot, int tokens, int* ticket);
int hs_swap_in_async(hs_ctx* ctx, int slot, int tokens, int* ticket);
/* 1 = done, 0 = in flight */
int hs_swap_done(hs_ctx* ctx, int ticket);

/* ------------------------------------------------------- remote CPU hosts
 * The reference's cluster has `cpu_hosts` CPU hosts: host 0 is the GPU's
 * own (PCIe), hosts 1.. are remote (network link, engine.py:329-331); a
 * request is offloaded to the local host while its memory lasts, else to
 * the least loaded remote host (_distribute_offload, engine.py:402-419),
 * and its work items are serviced there (engine.py:529-560).
 *
 * hs_cpu_host_serve runs a remote host: a blocking TCP server that owns the
 * KV of the requests placed on it and runs the host attention kernel for
 * every client replica (one slot namespace per connection).  It prints
 * "HS_CPU_HOST_READY port=<p>" once listening (port 0: any free port) and
 * returns after a client's shutdown request.  No GPU is needed.
 *
 * A replica connects each remote host id once (hs_cpu_host_connect) and
 * places a slot's KV on it after the swap-out landed in the slot's host
 * region (hs_cpu_place(slot, host, ctx tokens): the context is streamed to
 * the remote host, and from then on the slot's work items -- hs_cpu_attend
 * and hs_cpu_submit alike, device-polled ones included -- are relayed there
 * in FIFO order and their results written into the slot's result mailbox
 * with the same completion tag as a local item).  hs_cpu_place(slot, 0,
 * tokens) fetches the KV back into the region (before a swap-in); releasing
 * the region frees the remote copy.  bf16 datapath only. */
int hs_cpu_host_serve(const hs_model_cfg* model, const char* bind_addr, int port, int threads,
                      int max_slots);
int hs_cpu_host_connect(hs_ctx* ctx, int host, const char* addr, int port);
int hs_cpu_place(hs_ctx* ctx, int slot, int host, int tokens);
/* Live swap-in from a remote host without blocking the engine: queue the
 * fetch of the slot's KV into its host region (and the host's free), then
 * poll hs_cpu_fetch_done (1 = landed, the slot is local again; 0 = in
 * flight) before the swap-in DMA. */
int hs_cpu_fetch_async(hs_ctx* ctx, int slot, int tokens);
int hs_cpu_fetch_done(hs_ctx* ctx, int slot);
/* [4]: work items relayed, KV bytes placed, KV bytes fetched back, result bytes */
int hs_cpu_remote_stats(hs_ctx* ctx, int host, int64_t* stats);
/* Pipelined iterations: hs_iter_end_async queues the token readback and an
 * event and returns at once (the host plans the next iteration while this
 * one runs); hs_iter_poll returns 1 with the tokens and the completion time
 * in ms after the last hs_anchor() once the iteration has finished. */
int hs_anchor(hs_ctx* ctx);
int hs_iter_end_async(hs_ctx* ctx, int* ticket);
int hs_iter_poll(hs_ctx* ctx, int ticket, int* tokens_out, int n, double* done_ms);
int hs_iter_ntokens(hs_ctx* ctx, int ticket);
/* ------------------------------------------------- device-polled merges
 * The piggyback merge decision taken by the GPU (north star item 3; the
 * reference's _consume_merges / _merge_cap, engine.py:861-919, and the chain
 * continuation of _process_merge, engine.py:982-1022).  With hs_pg_enable(1)
 * the output FIFO of work items lives on the device: at the head of every
 * hs_layer a controller kernel reads the CPU workers' completion tags
 * (ld.acquire.sys) and merges the ready head-run whose layer matches, at
 * most `cap` rows; chains merged at layer l are carried into QKV(l+1) and
 * shipped; at the last layer every merged chain emits its token and
 * restarts unless it is done or stopped.  Shipped items reach the CPU pool
 * through a work ring in mapped host memory (no host submission).  The
 * hs_layer_desc row lists are ignored in this mode (only `layer` is read).
 * Per iteration:
 *   hs_iter_begin(...); hs_pg_iter(cap, merge_bound[n_layers], inject_bound);
 *   hs_layer(l) for l = 1..L; hs_iter_end_async(&ticket);
 *   once finished: hs_iter_poll(ticket, tokens...) -- the tokens of the
 *   plan's logit rows, then one row per merge_bound[L] entry of which the
 *   first (merged chains at L) are valid -- and hs_pg_log(ticket, ...).
 * Bounds are the launch sizes (padding rows cost compute, not correctness);
 * the device never merges more than the bound.
 * hs_pg_log output, per layer 1..L: count n, then n records (slot, flags);
 * flags 1 = injection taken at layer 1 (carry), 2 = chain restarted with its
 * next token at layer L, 4 = chain ended at layer L (done or stopped), 0 =
 * merged and carried into the next layer.  Returns the number of ints. */
/* on = 1 on an enabled context drops every queued item and injection (a new
 * engine takes over the replica) */
int hs_pg_enable(hs_ctx* ctx, int on);
/* fresh chains entering at layer 1 (engine.py:437-454 _inject): context
 * length and tokens still to generate (>= 1), in injection order */
int hs_pg_inject(hs_ctx* ctx, const int* slots, const int* ctx_tokens, const int* tokens_left,
                 int n);
/* swap-in directive at the chain's next token boundary (engine.py:489-494) */
int hs_pg_stop(hs_ctx* ctx, const int* slots, const int* stop, int n);
int hs_pg_iter(hs_ctx* ctx, int cap, const int* merge_bound, int inject_bound);
int hs_pg_log(hs_ctx* ctx, int ticket, int* out, int n);
/* Tensor-parallel groups: the ranks agree on every merge.  Phase 0 moves this
 * rank's completion tags into the POSIX shared-memory segment
 * "<prefix>.<rank>" (rank 0 also creates "<prefix>.dec"); after a barrier
 * across the group, phase 1 maps the peers' segments.  Rank 0's controller
 * then merges an item only once every rank's CPU pool has finished its heads
 * of it and publishes each layer's decision in "<prefix>.dec"; the other
 * ranks' controllers apply that decision (one snapshot of the tags for the
 * whole group).  The ranks must issue identical calls. */
int hs_pg_share_tags(hs_ctx* ctx, const char* prefix, int rank, int world, int phase);
/* stream marks for launch pacing, and timing events (CUDA events on the
 * compute stream; elapsed in ms between two timer ids) */
int hs_mark(hs_ctx* ctx);
int hs_wait_mark(hs_ctx* ctx, int id);
int hs_timer(hs_ctx* ctx);
int hs_timer_elapsed(hs_ctx* ctx, int a, int b, float* ms);
/* Per-kernel-class device time and algorithmic work of the launches made
 * while profiling is on (CUDA events around each launch).  classes:
 * 0 = Dense GEMMs, 1 = decode attention (K1+K2), 2 = prefill attention,
 * 3 = whole hs_layer spans (device time from a layer's first to last kernel).
 * stats[c] = {launches, milliseconds, bytes, flops}. */
int hs_profile(hs_ctx* ctx, int on);
int hs_profile_read(hs_ctx* ctx, double* stats /* [4][4] */, int reset);
/* Profiler probes on the context's own buffers and layer-0 weights (device
 * microseconds, median of reps): Dense modules over n rows; decode attention
 * of g requests with ctx keys each; causal prefill of q new tokens after
 * `done` tokens of context (the seam of build_dense_table, latency.py:200). */
int hs_probe_dense(hs_ctx* ctx, int n, int reps, float* us);
/* one layer-0 GEMM (which: 0 qkv, 1 o, 2 gate-up, 3 down), plain partial
 * planes (fused = 0) or with its fused stream-K epilogue (fused = 1) */
/* dense part of `layers` consecutive layers as hs_layer issues it; mode =
   op bitmask (0 QKV GEMM, 1 RoPE/KV/ship, 2 O GEMM, 3 add-norm, 4 gate-up
   GEMM, 5 SiLU, 6 down GEMM, 7 add-norm); *us = median per-layer us */
int hs_probe_dense_mode(hs_ctx* ctx, int n, int mode, int layers, int reps, float* us);
/* the 4 Dense GEMMs of all layers at n rows back to back (PDL chain intact)
 * between one event pair on the step stream: median us per launch and the
 * algorithmic bytes per launch (bench roofline) */
int hs_probe_gemm_stream(hs_ctx* ctx, int n, int reps, float* us, double* bytes);
/* PCIe rate of the piggyback mailboxes: dir 0 SM stores to the mapped ship
 * mailbox, 1 SM loads from the mapped result mailbox, 2/3 the same bytes by
 * the copy engine (D2H/H2D); `rows` items; median us and bytes moved */
int hs_probe_pcie(hs_ctx* ctx, int dir, int rows, int reps, float* us, double* bytes);
int hs_probe_gemm(hs_ctx* ctx, int which, int n, int fused, int reps, float* us);
int hs_probe_decode(hs_ctx* ctx, int g, int ctx_len, int reps, float* us);
int hs_probe_prefill(hs_ctx* ctx, int q, int done, int reps, float* us);

/* test taps */
int hs_keep_logits(hs_ctx* ctx, int on);
int hs_read_logits(hs_ctx* ctx, float* host, int rows);
/* logits of a pipelined iteration (hs_iter_end_async ticket; hs_keep_logits on) */
int hs_iter_logits(hs_ctx* ctx, int ticket, float* host, int rows);
int hs_read_ship(hs_ctx* ctx, int slot, void* host, size_t bytes);
int hs_read_result(hs_ctx* ctx, int slot, void* host, size_t bytes);
int hs_read_residual(hs_ctx* ctx, int slot, float* host);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* HS_H_ */
