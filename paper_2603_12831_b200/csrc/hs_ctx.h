// The serving-step context (one per GPU replica), shared by the bf16 step
// (step.cu) and the fp32 validation datapath (step_f32.cu).
#pragma once

#include <atomic>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "hs_internal.h"
#include "hs_step.h"

namespace hs {

inline constexpr int kBns[5] = {16, 32, 64, 128, 256};
inline int bn_index(int bn) {
  for (int i = 0; i < 5; ++i)
    if (kBns[i] == bn) return i;
  return 4;
}

struct ActBuf {  // a bf16 activation buffer with one TMA map per token-tile width
  bf16* p = nullptr;
  int rows = 0, k = 0;
  CUtensorMap maps[5];
};

struct HostRegion {
  size_t offset = 0;  // bytes into the arena
  int cap = 0;        // tokens
  bool used = false;
};

// Device-polled piggyback merges (piggyback.cu): the output FIFO of work
// items lives on the device, the merge decision of every layer is taken by
// a controller kernel from the CPU workers' completion tags, and the shipped
// items reach the CPU pool through a work ring in mapped host memory.
struct PgDev {
  int Q = 0;                  // FIFO / work-ring capacity (entries)
  int Qi = 0;                 // injection-ring capacity
  int* q = nullptr;           // FIFO [Q][3]: slot, layer (1-based), ctx
  int* inj = nullptr;         // injection ring [Qi]: slot
  int* st = nullptr;          // counters, see PG_* below
  int* slot_ctx = nullptr;    // [max_slots] the chain's current context length
  int* slot_left = nullptr;   // [max_slots] tokens still to generate, this one included
  int* slot_stop = nullptr;   // [max_slots] 1 = end the chain at its next token boundary
  int* prev = nullptr;        // [max_rows] slots merged at the previous layer
  int* lists = nullptr;       // per-layer row lists written by the controller
  int* it_logit_slots = nullptr;  // [max_rows] the iteration's logit-row slots
  int* work_d = nullptr;      // work ring [Q][4] (slot, layer, ctx, seq), mapped host
  int* work_tail_d = nullptr; // published entries (mapped host)
  int* log_d = nullptr;       // per-iteration decision log (mapped host)
  const unsigned* tags = nullptr;  // completion tags (mapped host)
  // tensor-parallel group: every rank's completion tags (shared host
  // segments); an item is ready once all ranks' CPU pools finished it
  const unsigned* peer_tags[8] = {};
  int n_peer = 0;
  // TP group: rank 0's controller publishes each layer's decision (merged
  // count, injections) into a shared ring; the followers' controllers take
  // it from there, so every rank applies one snapshot of the tags
  int* dec = nullptr;         // [kDecRing][4]: seq, k, n_inj, pad (mapped, shared)
  int dec_role = 0;           // 0 = single rank, 1 = publishes, 2 = follows
  int list_cap = 0;           // entries per list in `lists`
  int log_stride = 0;         // ints per iteration in the log
};
enum { PG_HEAD = 0, PG_TAIL = 1, PG_PUB = 2, PG_INJ_HEAD = 3, PG_INJ_TAIL = 4, PG_PREV_N = 5,
       PG_SEQ = 6, PG_STATE_INTS = 8 };
constexpr int kDecRing = 64;

// device pointers of one hs_layer call's row lists (packed staging run)
struct LayerRows {
  const int *carry_slot, *carry_pos, *merge_slot, *restart_slot, *restart_pos, *logit_rows,
      *logit_slots, *merge_tag;
};

}  // namespace hs

using namespace hs;

struct hs_ctx {
  ModelCfg m{};
  hs_rt_cfg r{};
  cudaStream_t st = nullptr;
  KvGeom geom{};
  // fp32 validation datapath (hs_rt_cfg.precision == HS_PREC_FP32, step_f32.cu):
  // fp32 weights, activations, KV pool, piggyback mailboxes and host KV;
  // SIMT kernels instead of the bf16 tcgen05/TMA ones
  bool fp32 = false;
  int kv_elem = 2;  // bytes per KV / mailbox element (2 bf16, 4 fp32)
  float *fw_embed = nullptr, *fw_lm = nullptr;
  std::vector<float*> fw_qkv, fw_o, fw_gu, fw_down;
  float *fx = nullptr, *fx2 = nullptr, *fattn = nullptr, *fact = nullptr, *fq = nullptr,
        *flin = nullptr, *fxr = nullptr;
  float* kv_f32 = nullptr;  // [layers][pages][2][n_kv][64][hd] fp32 (aliases kv_pool)
  // weights
  bf16 *w_embed = nullptr, *w_lm = nullptr;
  float* w_final = nullptr;
  std::vector<bf16*> w_qkv, w_o, w_gu, w_down;
  std::vector<float*> n_in, n_post;
  std::vector<CUtensorMap> m_qkv, m_o, m_gu, m_down;
  CUtensorMap m_lm{};
  // kv
  bf16* kv_pool = nullptr;
  CUtensorMap m_kv{};
  int* page_table = nullptr;
  // activations
  float* h = nullptr;      // residual stream [max_rows][d]
  float* hr = nullptr;     // restart rows [max_rows][d]
  ActBuf xn, xn2, attn, act, lin, xr;
  bf16* qbuf = nullptr;
  float* part = nullptr;
  size_t part_floats = 0;
  float *o_part = nullptr, *lse_part = nullptr;
  float* resid = nullptr;  // device residual store [max_slots][d]
  int* last_token = nullptr;
  int* tok = nullptr;
  int* tok_out = nullptr;
  float *rope_cos = nullptr, *rope_sin = nullptr;
  float* logits = nullptr;  // optional debug copy of the last LM-head logits
  bool keep_logits = false;
  float* logit_ring = nullptr;  // pinned [kIterRing][2*max_rows][vocab]: logits of async iterations
  // metadata (device) and pinned staging
  int* dm = nullptr;   // iteration + layer metadata
  int* hm = nullptr;   // pinned staging (two halves), mapped
  int* hm_d = nullptr;  // its device alias (zero-copy layer metadata)
  size_t meta_ints = 0;
  int stage_half = 0;
  size_t stage_pos = 0;
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  // iteration state; pointers into the packed per-iteration device block
  int B = 0, D = 0, n_chunks = 0, n_tiles = 0, n_logit = 0, n_tok_out = 0, merges_L = 0;
  int* dm_iter = nullptr;   // packed iteration metadata (one upload per iteration)
  int* dm_layer = nullptr;  // packed layer metadata (one upload per layer)
  size_t iter_cap = 0, layer_cap = 0;
  const int *it_slot = nullptr, *it_pos = nullptr, *it_tok = nullptr, *it_chunks = nullptr,
            *it_cbeg = nullptr, *it_tiles = nullptr;
  std::vector<int> h_logit_rows, h_logit_slots;  // host copies (layer-L gather lists)
  int* dec_counters = nullptr;
  int* tile_sem = nullptr;  // stream-K fixup semaphores of the fused GEMMs
  // tensor parallelism (hs_tp_*): this rank's exchange buffer and flags, the
  // group's pointers, the exchange counter and the IPC mappings to close
  int tp_world = 1, tp_rank = 0;
  float* tp_xbuf = nullptr;
  unsigned* tp_flag = nullptr;
  TpPeers tp{};
  unsigned tp_epoch = 0;
  std::vector<void*> tp_opened;
  int* tokens_pinned = nullptr;
  // piggyback mailboxes (pinned, mapped)
  bf16 *ship_h = nullptr, *ship_d = nullptr, *result_h = nullptr, *result_d = nullptr;
  // completion tags of the result mailbox (one per slot, written by the CPU
  // workers) and the device fault record (hs_layer_desc.merge_tag checks)
  unsigned *tag_h = nullptr, *tag_d = nullptr, *fault_h = nullptr, *fault_d = nullptr;
  // host KV arena (pinned, mapped)
  bf16 *hkv_h = nullptr, *hkv_d = nullptr;
  size_t hkv_bytes = 0;
  std::vector<HostRegion> regions;
  std::vector<std::pair<size_t, size_t>> free_list;  // (offset, bytes)
  ThreadPool* pool = nullptr;
  std::vector<int> cpus;  // the replica's CPU-attention core set (empty: unpinned)
  CpuService* cpu = nullptr;
  // remote CPU hosts (cpu_remote.cpp): relay per host id (index 0 = this
  // replica's own host, unused) and the host each slot's KV lives on
  std::vector<RemoteHost*> remotes;
  std::unique_ptr<std::atomic<int>[]> slot_host;
  // live swap-ins from a remote host: the slot's pending fetch (host, done flag)
  std::map<int, std::pair<int, std::shared_ptr<std::atomic<int>>>> fetches;
  // swaps: copy stream + contiguous staging for pack/unpack around one 2D DMA
  cudaStream_t copy_st = nullptr;
  bf16* swap_stage = nullptr;
  size_t swap_stage_elems = 0;
  std::map<int, cudaEvent_t> swap_ev;
  int next_ticket = 1;
  // asynchronous iteration completion: ring of pinned token buffers + events
  static constexpr int kIterRing = 8;
  int* tok_ring = nullptr;  // pinned [kIterRing][2*max_rows]
  cudaEvent_t iter_ev[kIterRing] = {};
  int iter_n[kIterRing] = {};
  int next_iter = 0;
  cudaEvent_t anchor = nullptr;
  // marks (pacing) and timing events on the compute stream
  std::vector<cudaEvent_t> marks, timers;
  int next_mark = 0, next_timer = 0;
  // per-kernel-class profiling (class, start, stop, bytes, flops)
  bool prof_on = false;
  struct Rec { int cls; cudaEvent_t a, b; double bytes, flops; };
  std::vector<Rec> prof_pending;
  std::vector<cudaEvent_t> prof_free;
  double prof_stats[4][4] = {};
  double dec_kv_tokens = 0, pre_units = 0, pre_kv_tokens = 0;
  // device-polled piggyback merges (piggyback.cu)
  bool pg_on = false;
  PgDev pg{};
  int* pg_work_h = nullptr;   // host side of the work ring / tail / log
  int* pg_tail_h = nullptr;
  int* pg_log_h = nullptr;
  int* pg_logit_h = nullptr;  // [kIterRing][max_rows] logit-row slots per iteration (mapped)
  int* pg_logit_d = nullptr;
  int* pg_ops_h = nullptr;    // admin-op staging ring (mapped)
  int* pg_ops_d = nullptr;
  cudaEvent_t pg_op_ev[8] = {};
  int pg_op_next = 0;
  int pg_cap = 0;             // this iteration's per-layer merge cap
  int pg_inj_bound = 0;       // host bound on the layer-1 injections taken
  std::vector<int> pg_bound;  // host bound on the merges of each layer
  int pg_iter_slot = 0;       // ring slot of the iteration being issued
  // TP groups: this rank's tags moved into a POSIX shm segment (shared with
  // the peers) and the peers' segments mapped here
  std::vector<std::pair<void*, size_t>> pg_shm;  // mapped segments (own first)
  std::string pg_shm_own;                        // names to unlink on destroy
  std::string pg_shm_dec;
  unsigned* pg_tag_alloc = nullptr;              // the original cudaHostAlloc tags
};

// the fp32 validation datapath of hs_layer (step_f32.cu); called after the
// row lists are packed, with the same row semantics as the bf16 layer
int layer_f32(hs_ctx* c, const hs_layer_desc* d, const hs::LayerRows& rows);

namespace hs {
// device-polled piggyback merges (piggyback.cu)
int pg_alloc(hs_ctx* c);
void pg_free(hs_ctx* c);
// launches the layer's controller; fills `rows` with its device lists and
// the host bounds of the carry / merge / restart counts
int pg_control(hs_ctx* c, int layer, hs::LayerRows* rows, int* n_carry, int* n_merge,
               int* n_restart);
int pg_publish(hs_ctx* c);
int ctx_cpu_service(hs_ctx* c);  // starts the CPU-attention pool if needed (step.cu)
}  // namespace hs
