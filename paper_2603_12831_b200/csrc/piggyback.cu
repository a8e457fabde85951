// Device-polled Attention Piggybacking: the merge decision on the GPU.
//
// The reference consumes the piggyback output FIFO at the start of every
// layer: the head-run of results with head.layer == layer, at most `cap`
// per layer (one cap computed per iteration), plus layer-1 injections of
// fresh chains (Engine._consume_merges / _merge_cap,
// pkg/src/hybridserve/engine.py:861-919), and every merged chain continues
// with QKV of its next layer, shipped to the host (_chain_qkv /
// _process_merge, engine.py:982-1022).  In this mode that FIFO lives in HBM
// and a one-warp controller kernel at the head of each layer takes the
// decision itself:
//
//   * a work item is "in the output FIFO" once the CPU worker has published
//     its completion tag HS_RESULT_TAG(ctx, layer) (release) after the result
//     row; the controller reads the tags of the FIFO head with
//     ld.acquire.sys, 32 candidates per warp ballot, and takes the ready
//     prefix whose layer matches, bounded by the cap;
//   * the merged rows, the carries (chains merged at the previous layer, or
//     the injections taken at layer 1) and, at the last layer, the restarts
//     (chains whose next token is due and not stopped by a swap-in
//     directive) are written as the layer's row lists; rows up to the host's
//     launch bounds are padding (slot -1: no ship, no residual put, no tag);
//   * every item shipped by a layer is pushed to the FIFO tail; the next
//     controller (or the publish at the end of the last layer) copies the
//     entries whose rows have landed into the work ring in mapped host
//     memory and releases its tail, which the CPU pool's dispatcher polls;
//   * each layer's decisions are logged per iteration (mapped host memory)
//     so the host engine replays its bookkeeping in the same order.
//
// The host never sits between a completion and its merge: no host poll, no
// host decision, no per-layer host<->device round trip.
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "hs_common.cuh"
#include "hs_internal.h"
#include "hs_step.h"

#include "hs_ctx.h"

namespace hs {

namespace {

constexpr int kLogRecords = 512;  // merge + injection records per layer in the log
constexpr int kOpBufs = 8;        // admin-op staging buffers (ring)
constexpr int kOpInts = 4096;     // ints per admin-op buffer

#define PG_CK(x)                                                                           \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      return set_error(HS_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x,                  \
                       cudaGetErrorString(e_));                                            \
  } while (0)

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct ListPtrs {
  int *carry_slot, *carry_pos, *merge_slot, *merge_tag, *restart_slot, *restart_pos,
      *logit_slots;
};

__host__ __device__ inline ListPtrs lists_of(const PgDev& p) {
  ListPtrs l;
  const int n = p.list_cap;
  l.carry_slot = p.lists;
  l.carry_pos = l.carry_slot + n;
  l.merge_slot = l.carry_pos + n;
  l.merge_tag = l.merge_slot + n;
  l.restart_slot = l.merge_tag + n;
  l.restart_pos = l.restart_slot + n;
  l.logit_slots = l.restart_pos + n;  // 2n
  return l;
}

// Copy the FIFO entries [pub, tail) into the host work ring and release the
// new tail (their rows were written by kernels that completed before this
// one started: griddepcontrol.wait).
__device__ void publish_entries(const PgDev& p, int lane) {
  const int pub = p.st[PG_PUB], tail = p.st[PG_TAIL];
  for (int i = pub + lane; i < tail; i += 32) {
    const int* e = p.q + static_cast<size_t>(i % p.Q) * 3;
    int* w = p.work_d + static_cast<size_t>(i % p.Q) * 4;
    w[0] = e[0];
    w[1] = e[1];
    w[2] = e[2];
    w[3] = i;
  }
  __syncwarp();
  if (lane == 0 && tail != pub) {
    __threadfence_system();
    st_release_sys(p.work_tail_d, tail);
    p.st[PG_PUB] = tail;
  }
}

__global__ void pg_publish_kernel(PgDev p) {
  pdl_wait();
  pdl_trigger();
  publish_entries(p, threadIdx.x);
}

// admin ops staged by the host, in stream order: {0, slot, ctx, left} =
// inject a fresh chain (layer-1 entry); {1, slot, stop, 0} = stop flag;
// {2, 0, 0, 0} = drop everything queued
__global__ void pg_admin_kernel(PgDev p, const int* ops, int n) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  int tail = p.st[PG_INJ_TAIL];
  for (int i = 0; i < n; ++i) {
    const int* o = ops + 4 * i;
    const int slot = o[1];
    if (o[0] == 0) {
      p.inj[tail % p.Qi] = slot;
      ++tail;
      p.slot_ctx[slot] = o[2];
      p.slot_left[slot] = o[3];
      p.slot_stop[slot] = 0;
    } else if (o[0] == 1) {
      p.slot_stop[slot] = o[2];
    } else {  // flush: every queued item and injection is dropped (a new engine)
      p.st[PG_HEAD] = p.st[PG_TAIL];
      p.st[PG_INJ_HEAD] = tail;
      p.st[PG_PREV_N] = 0;
    }
  }
  p.st[PG_INJ_TAIL] = tail;
}

// One warp.  layer is 1-based; c_max / m_max are the host's launch bounds
// for the carry / merge rows of this layer (padding beyond the decision).
__global__ void pg_control_kernel(PgDev p, int layer, int n_layers, int cap, int c_max, int m_max,
                                  int n_logit, int log_slot) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x;
  publish_entries(p, lane);
  __syncwarp();
  const ListPtrs L = lists_of(p);
  const int head = p.st[PG_HEAD], tail = p.st[PG_TAIL];
  // FIFO head-run at this layer (engine.py:902-911): ready prefix, layer match
  const int limit = min(cap, m_max);
  const int avail = min(tail - head, limit);
  int k = 0;
  while (k < limit) {
    const int i = k + lane;
    bool ok = false;
    if (i < avail) {
      const int* e = p.q + static_cast<size_t>((head + i) % p.Q) * 3;
      if (e[1] == layer) {
        const unsigned want = static_cast<unsigned>(HS_RESULT_TAG(e[2], layer));
        ok = ld_acquire_sys(p.tags + e[0]) == want;
        // a TP group merges an item only once every rank's pool finished
        // its heads: all ranks read the same tags, take the same decision
        for (int r = 0; r < p.n_peer; ++r) ok = ok && ld_acquire_sys(p.peer_tags[r] + e[0]) == want;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    const int run = m == 0xffffffffu ? 32 : __ffs(~m) - 1;
    k += run;
    if (run < 32) break;
  }
  k = min(k, limit);
  // layer-1 injections fill the rest of the cap (engine.py:912-918)
  const int inj_head = p.st[PG_INJ_HEAD];
  int n_inj = layer == 1 ? max(0, min(min(p.st[PG_INJ_TAIL] - inj_head, cap - k), c_max)) : 0;
  if (p.dec_role) {
    // TP group: one snapshot of the tags for every rank.  Rank 0 publishes
    // its decision (taken over all ranks' tags) for this layer; the others
    // apply it (their FIFOs are identical: same calls, same decisions)
    const int seq = p.st[PG_SEQ] + 1;
    int* slot = p.dec + (seq % kDecRing) * 4;
    if (p.dec_role == 1) {
      if (lane == 0) {
        slot[1] = k;
        slot[2] = n_inj;
        __threadfence_system();
        st_release_sys(slot, seq);
      }
    } else {
      int got = 0;
      if (lane == 0) {
        const long long t0 = clock64();
        for (;;) {
          int v;
          asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(slot) : "memory");
          if (v == seq) break;
          if (clock64() - t0 > 40000000000LL) __trap();  // ~20 s: the leader is gone
          __nanosleep(200);
        }
        got = 1;
      }
      __syncwarp();
      (void)got;
      k = *reinterpret_cast<volatile int*>(slot + 1);
      n_inj = *reinterpret_cast<volatile int*>(slot + 2);
    }
    __syncwarp();
    if (lane == 0) p.st[PG_SEQ] = seq;
  }
  const int n_prev = layer == 1 ? 0 : min(p.st[PG_PREV_N], c_max);
  const int n_carry = layer == 1 ? n_inj : n_prev;
  const bool last = layer == n_layers;
  __syncwarp();
  // row lists (padding: slot -1)
  for (int i = lane; i < m_max; i += 32) {
    if (i < k) {
      const int* e = p.q + static_cast<size_t>((head + i) % p.Q) * 3;
      L.merge_slot[i] = e[0];
      L.merge_tag[i] = HS_RESULT_TAG(e[2], layer);
    } else {
      L.merge_slot[i] = -1;
      L.merge_tag[i] = 0;
    }
    if (last) L.logit_slots[n_logit + i] = i < k ? L.merge_slot[i] : -1;
  }
  if (last)
    for (int i = lane; i < n_logit; i += 32) L.logit_slots[i] = p.it_logit_slots[i];
  for (int i = lane; i < c_max; i += 32) {
    int slot = -1;
    if (i < n_carry) slot = layer == 1 ? p.inj[(inj_head + i) % p.Qi] : p.prev[i];
    L.carry_slot[i] = slot;
    L.carry_pos[i] = slot >= 0 ? p.slot_ctx[slot] : 0;
  }
  __syncwarp();
  if (lane == 0) {
    int t = tail;
    // this layer's carries are shipped by its QKV launch: FIFO items (slot,
    // layer, ctx) in ship order
    for (int i = 0; i < n_carry; ++i) {
      int* e = p.q + static_cast<size_t>(t % p.Q) * 3;
      e[0] = L.carry_slot[i];
      e[1] = layer;
      e[2] = L.carry_pos[i];
      ++t;
    }
    int* log = p.log_d + static_cast<size_t>(log_slot) * p.log_stride +
               static_cast<size_t>(layer - 1) * (1 + 2 * kLogRecords);
    log[0] = k + n_inj;
    int nr = 0;
    for (int i = 0; i < k; ++i) {
      const int slot = L.merge_slot[i];
      int flags = 0;
      if (last) {
        // the chain's token is emitted (engine.py:1005-1016); it continues
        // with the next token unless it is done or a swap-in stops it
        const int left = p.slot_left[slot] - 1;
        p.slot_left[slot] = left;
        const int ctx = p.slot_ctx[slot] + 1;
        p.slot_ctx[slot] = ctx;
        if (left > 0 && !p.slot_stop[slot]) {
          L.restart_slot[nr] = slot;
          L.restart_pos[nr] = ctx;
          int* e = p.q + static_cast<size_t>(t % p.Q) * 3;
          e[0] = slot;
          e[1] = 1;
          e[2] = ctx;
          ++t;
          ++nr;
          flags = 2;
        } else {
          flags = 4;
        }
      } else {
        p.prev[i] = slot;
      }
      log[1 + 2 * i] = slot;
      log[2 + 2 * i] = flags;
    }
    for (int i = 0; i < n_inj; ++i) {
      log[1 + 2 * (k + i)] = L.carry_slot[i];
      log[2 + 2 * (k + i)] = 1;
    }
    if (last)
      for (int i = nr; i < m_max; ++i) {
        L.restart_slot[i] = -1;
        L.restart_pos[i] = 0;
      }
    p.st[PG_PREV_N] = last ? 0 : k;
    p.st[PG_HEAD] = head + k;
    p.st[PG_TAIL] = t;
    p.st[PG_INJ_HEAD] = inj_head + n_inj;
    __threadfence_system();
  }
}

}  // namespace

int pg_alloc(hs_ctx* c) {
  if (c->pg.q) return HS_OK;
  PgDev& p = c->pg;
  const hs_rt_cfg& r = c->r;
  p.Q = 2 * r.max_slots + 64;
  p.Qi = 2 * r.max_slots + 64;
  p.list_cap = r.max_rows;
  p.log_stride = c->m.layers * (1 + 2 * kLogRecords);
  const int S = r.max_slots;
  size_t ints = static_cast<size_t>(p.Q) * 3 + p.Qi + PG_STATE_INTS + 3 * static_cast<size_t>(S) +
                r.max_rows + 8 * static_cast<size_t>(p.list_cap);
  int* base = nullptr;
  if (cudaMalloc(&base, ints * sizeof(int)) != cudaSuccess)
    return set_error(HS_E_CUDA, "device-polled merges: allocation failed");
  if (cudaMemsetAsync(base, 0, ints * sizeof(int), c->st) != cudaSuccess)
    return set_error(HS_E_CUDA, "device-polled merges: clear failed");
  p.q = base;
  p.inj = p.q + static_cast<size_t>(p.Q) * 3;
  p.st = p.inj + p.Qi;
  p.slot_ctx = p.st + PG_STATE_INTS;
  p.slot_left = p.slot_ctx + S;
  p.slot_stop = p.slot_left + S;
  p.prev = p.slot_stop + S;
  p.lists = p.prev + r.max_rows;
  const size_t host_ints = static_cast<size_t>(p.Q) * 4 + 16 +
                           static_cast<size_t>(hs_ctx::kIterRing) * p.log_stride +
                           static_cast<size_t>(hs_ctx::kIterRing) * r.max_rows +
                           static_cast<size_t>(kOpBufs) * kOpInts;
  int* h = nullptr;
  if (cudaHostAlloc(&h, host_ints * sizeof(int), cudaHostAllocMapped) != cudaSuccess)
    return set_error(HS_E_CUDA, "device-polled merges: pinned allocation failed");
  std::memset(h, 0, host_ints * sizeof(int));
  c->pg_work_h = h;
  c->pg_tail_h = h + static_cast<size_t>(p.Q) * 4;
  c->pg_log_h = c->pg_tail_h + 16;
  c->pg_logit_h = c->pg_log_h + static_cast<size_t>(hs_ctx::kIterRing) * p.log_stride;
  c->pg_ops_h = c->pg_logit_h + static_cast<size_t>(hs_ctx::kIterRing) * r.max_rows;
  int* hd = nullptr;
  if (cudaHostGetDevicePointer(&hd, h, 0) != cudaSuccess)
    return set_error(HS_E_CUDA, "device-polled merges: mapped pointer");
  p.work_d = hd;
  p.work_tail_d = hd + static_cast<size_t>(p.Q) * 4;
  p.log_d = p.work_tail_d + 16;
  c->pg_logit_d = p.log_d + static_cast<size_t>(hs_ctx::kIterRing) * p.log_stride;
  c->pg_ops_d = c->pg_logit_d + static_cast<size_t>(hs_ctx::kIterRing) * r.max_rows;
  p.tags = c->tag_d;
  if (cudaDeviceSynchronize() != cudaSuccess)
    return set_error(HS_E_CUDA, "device-polled merges: init");
  return HS_OK;
}

void pg_free(hs_ctx* c) {
  for (auto& seg : c->pg_shm) {
    cudaHostUnregister(seg.first);
    munmap(seg.first, seg.second);
  }
  c->pg_shm.clear();
  if (!c->pg_shm_own.empty()) shm_unlink(c->pg_shm_own.c_str());
  c->pg_shm_own.clear();
  if (!c->pg_shm_dec.empty()) shm_unlink(c->pg_shm_dec.c_str());
  c->pg_shm_dec.clear();
  if (c->pg_tag_alloc) {  // the context frees its own allocation
    c->tag_h = c->pg_tag_alloc;
    c->pg_tag_alloc = nullptr;
  }
  if (c->pg.q) cudaFree(c->pg.q);
  if (c->pg_work_h) cudaFreeHost(c->pg_work_h);
  c->pg = PgDev{};
  for (auto& e : c->pg_op_ev)
    if (e) cudaEventDestroy(e), e = nullptr;
  c->pg_work_h = c->pg_tail_h = c->pg_log_h = c->pg_logit_h = c->pg_logit_d = nullptr;
  c->pg_ops_h = c->pg_ops_d = nullptr;
}

int pg_control(hs_ctx* c, int layer, LayerRows* rows, int* n_carry, int* n_merge,
               int* n_restart) {
  const int L = c->m.layers;
  const int l0 = layer - 1;
  if (static_cast<int>(c->pg_bound.size()) != L)
    return set_error(HS_E_CONFIG, "device-polled merges: hs_pg_iter not called for this iteration");
  const int m_max = std::min({c->pg_bound[l0], c->pg_cap, kLogRecords});
  const int c_max = layer == 1 ? std::min(c->pg_inj_bound, kLogRecords)
                               : std::min({c->pg_bound[l0 - 1], c->pg_cap, kLogRecords});
  if (m_max + c->n_logit > c->pg.list_cap || c_max > c->pg.list_cap)
    return set_error(HS_E_CAPACITY, "device-polled merges: bounds exceed max_rows");
  PgDev p = c->pg;
  p.it_logit_slots = c->pg_logit_d + static_cast<size_t>(c->pg_iter_slot) * c->r.max_rows;
  if (launch_pdl(pg_control_kernel, dim3(1), dim3(32), 0, c->st, p, layer, L, c->pg_cap, c_max,
                 m_max, c->n_logit, c->pg_iter_slot))
    return set_error(HS_E_CUDA, "pg_control launch: %s", cudaGetErrorString(cudaGetLastError()));
  const ListPtrs lp = lists_of(c->pg);
  rows->carry_slot = lp.carry_slot;
  rows->carry_pos = lp.carry_pos;
  rows->merge_slot = lp.merge_slot;
  rows->merge_tag = lp.merge_tag;
  rows->restart_slot = lp.restart_slot;
  rows->restart_pos = lp.restart_pos;
  rows->logit_slots = lp.logit_slots;
  rows->logit_rows = nullptr;
  *n_carry = c_max;
  *n_merge = m_max;
  *n_restart = layer == L ? m_max : 0;
  return HS_OK;
}

int pg_publish(hs_ctx* c) {
  if (launch_pdl(pg_publish_kernel, dim3(1), dim3(32), 0, c->st, c->pg))
    return set_error(HS_E_CUDA, "pg_publish launch: %s", cudaGetErrorString(cudaGetLastError()));
  return HS_OK;
}

}  // namespace hs

// ------------------------------------------------------------------ C ABI
using namespace hs;

namespace {
// Admin ops travel through a small ring of pinned buffers read in place by
// the kernel; a buffer is reused once the launch that read it (kOpBufs calls
// ago) has executed, so staging never waits on the stream in steady state.
int stage_ops(hs_ctx* c, const std::vector<int>& ops) {
  for (size_t off = 0; off < ops.size(); off += kOpInts) {
    const size_t n = std::min<size_t>(kOpInts, ops.size() - off);
    const int b = c->pg_op_next++ % kOpBufs;
    if (c->pg_op_ev[b]) PG_CK(cudaEventSynchronize(c->pg_op_ev[b]));
    else PG_CK(cudaEventCreateWithFlags(&c->pg_op_ev[b], cudaEventDisableTiming));
    int* h = c->pg_ops_h + static_cast<size_t>(b) * kOpInts;
    std::memcpy(h, ops.data() + off, n * sizeof(int));
    const int* d = c->pg_ops_d + static_cast<size_t>(b) * kOpInts;
    if (launch_pdl(pg_admin_kernel, dim3(1), dim3(32), 0, c->st, c->pg, d, static_cast<int>(n / 4)))
      return set_error(HS_E_CUDA, "device-polled merges: admin launch");
    PG_CK(cudaEventRecord(c->pg_op_ev[b], c->st));
  }
  return HS_OK;
}
}  // namespace

int hs_pg_enable(hs_ctx* c, int on) {
  if (!on) {
    c->pg_on = false;
    return HS_OK;
  }
  if (c->fp32) return set_error(HS_E_CONFIG, "device-polled merges: bf16 datapath only");
  if (c->pg_on) return stage_ops(c, {2, 0, 0, 0});  // re-enable: drop the queued items
  if (int rc = pg_alloc(c)) return rc;
  if (int rc = ctx_cpu_service(c)) return rc;
  cpu_service_attach_ring(c->cpu, c->pg_work_h, c->pg_tail_h, c->pg.Q);
  c->pg_on = true;
  return HS_OK;
}

int hs_pg_inject(hs_ctx* c, const int* slots, const int* ctx_tokens, const int* tokens_left,
                 int n) {
  if (!c->pg_on) return set_error(HS_E_CONFIG, "device-polled merges are off");
  std::vector<int> ops;
  for (int i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= c->r.max_slots || ctx_tokens[i] < 0 ||
        ctx_tokens[i] + tokens_left[i] >= c->r.max_pos || tokens_left[i] < 1)
      return set_error(HS_E_CONFIG, "inject %d: slot %d ctx %d left %d out of range", i, slots[i],
                       ctx_tokens[i], tokens_left[i]);
    if (c->regions[slots[i]].cap < ctx_tokens[i] + tokens_left[i])
      return set_error(HS_E_CONFIG, "inject: slot %d host KV holds %d tokens, chain needs %d",
                       slots[i], c->regions[slots[i]].cap, ctx_tokens[i] + tokens_left[i]);
    ops.insert(ops.end(), {0, slots[i], ctx_tokens[i], tokens_left[i]});
  }
  return stage_ops(c, ops);
}

int hs_pg_stop(hs_ctx* c, const int* slots, const int* stop, int n) {
  if (!c->pg_on) return set_error(HS_E_CONFIG, "device-polled merges are off");
  std::vector<int> ops;
  for (int i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= c->r.max_slots)
      return set_error(HS_E_CONFIG, "stop %d: slot %d out of range", i, slots[i]);
    ops.insert(ops.end(), {1, slots[i], stop[i] ? 1 : 0, 0});
  }
  return stage_ops(c, ops);
}

int hs_pg_iter(hs_ctx* c, int cap, const int* merge_bound, int inject_bound) {
  if (!c->pg_on) return set_error(HS_E_CONFIG, "device-polled merges are off");
  const int L = c->m.layers;
  if (cap < 0 || inject_bound < 0) return set_error(HS_E_CONFIG, "negative cap / bound");
  c->pg_cap = cap;
  c->pg_inj_bound = std::min(inject_bound, cap);
  c->pg_bound.assign(merge_bound, merge_bound + L);
  for (int& b : c->pg_bound) b = std::max(0, std::min(b, cap));
  c->pg_iter_slot = c->next_iter % hs_ctx::kIterRing;
  // the iteration's logit-row slots (the controller of the last layer
  // appends the merged chains' slots after them), read in place from mapped
  // memory; the ring slot's previous iteration has finished (hs_iter_end_async)
  if (c->n_logit > 0)
    std::memcpy(c->pg_logit_h + static_cast<size_t>(c->pg_iter_slot) * c->r.max_rows,
                c->h_logit_slots.data(), c->n_logit * sizeof(int));
  return HS_OK;
}

int hs_pg_log(hs_ctx* c, int ticket, int* out, int n) {
  if (!c->pg_log_h) return -set_error(HS_E_CONFIG, "device-polled merges were never enabled");
  if (ticket < c->next_iter - hs_ctx::kIterRing || ticket >= c->next_iter)
    return -set_error(HS_E_CONFIG, "iteration ticket %d out of window", ticket);
  const int slot = ticket % hs_ctx::kIterRing;
  if (cudaEventQuery(c->iter_ev[slot]) != cudaSuccess)
    return -set_error(HS_E_CONFIG, "iteration %d has not finished", ticket);
  const volatile int* log = c->pg_log_h + static_cast<size_t>(slot) * c->pg.log_stride;
  int k = 0;
  for (int l = 0; l < c->m.layers; ++l) {
    const volatile int* e = log + static_cast<size_t>(l) * (1 + 2 * kLogRecords);
    const int cnt = e[0];
    if (k + 1 + 2 * cnt > n) return -set_error(HS_E_CAPACITY, "log buffer too small");
    out[k++] = cnt;
    for (int i = 0; i < 2 * cnt; ++i) out[k++] = e[1 + i];
  }
  return k;
}

// Tensor-parallel agreement on the merge decision: phase 0 moves this rank's
// completion tags into the shared segment "<prefix>.<rank>"; after a barrier
// across the group, phase 1 maps every peer's segment, so each rank's
// controller reads all ranks' tags and they take identical decisions.
int hs_pg_share_tags(hs_ctx* c, const char* prefix, int rank, int world, int phase) {
  if (!c->pg_on) return set_error(HS_E_CONFIG, "device-polled merges are off");
  if (world < 1 || world > 8 || rank < 0 || rank >= world)
    return set_error(HS_E_CONFIG, "rank %d of %d out of range", rank, world);
  const size_t bytes = static_cast<size_t>(c->r.max_slots) * sizeof(unsigned);
  auto map_seg = [&](const std::string& name, bool create, void** out) -> int {
    const int fd = shm_open(name.c_str(), create ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
    if (fd < 0) return set_error(HS_E_CONFIG, "shm_open %s failed", name.c_str());
    if (create && ftruncate(fd, static_cast<off_t>(bytes)) != 0) {
      close(fd);
      return set_error(HS_E_CONFIG, "ftruncate %s failed", name.c_str());
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) return set_error(HS_E_CONFIG, "mmap %s failed", name.c_str());
    if (cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) !=
        cudaSuccess) {
      munmap(p, bytes);
      return set_error(HS_E_CUDA, "cudaHostRegister %s failed", name.c_str());
    }
    c->pg_shm.emplace_back(p, bytes);
    *out = p;
    return HS_OK;
  };
  const std::string base = std::string(prefix) + ".";
  const size_t dec_bytes = static_cast<size_t>(kDecRing) * 4 * sizeof(int);
  auto map_dec = [&](bool create) -> int {
    const std::string name = base + "dec";
    const int fd = shm_open(name.c_str(), create ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
    if (fd < 0) return set_error(HS_E_CONFIG, "shm_open %s failed", name.c_str());
    if (create && ftruncate(fd, static_cast<off_t>(dec_bytes)) != 0) {
      close(fd);
      return set_error(HS_E_CONFIG, "ftruncate %s failed", name.c_str());
    }
    void* p = mmap(nullptr, dec_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) return set_error(HS_E_CONFIG, "mmap %s failed", name.c_str());
    if (create) std::memset(p, 0, dec_bytes);
    if (cudaHostRegister(p, dec_bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) !=
        cudaSuccess) {
      munmap(p, dec_bytes);
      return set_error(HS_E_CUDA, "cudaHostRegister %s failed", name.c_str());
    }
    c->pg_shm.emplace_back(p, dec_bytes);
    if (create) c->pg_shm_dec = name;
    PG_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->pg.dec), p, 0));
    c->pg.dec_role = create ? 1 : 2;
    return HS_OK;
  };
  if (phase == 0 && world > 1 && rank == 0)
    if (int rc = map_dec(true)) return rc;
  if (phase == 1 && world > 1 && rank != 0)
    if (int rc = map_dec(false)) return rc;
  if (phase == 0) {
    PG_CK(cudaDeviceSynchronize());
    void* p = nullptr;
    c->pg_shm_own = base + std::to_string(rank);
    if (int rc = map_seg(c->pg_shm_own, true, &p)) return rc;
    std::memcpy(p, c->tag_h, bytes);  // the current tags (all retracted at start)
    c->pg_tag_alloc = c->tag_h;
    c->tag_h = static_cast<unsigned*>(p);
    PG_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->tag_d), p, 0));
    c->pg.tags = c->tag_d;
    return HS_OK;
  }
  int n = 0;
  for (int r = 0; r < world; ++r) {
    if (r == rank) continue;
    void* p = nullptr;
    if (int rc = map_seg(base + std::to_string(r), false, &p)) return rc;
    unsigned* d = nullptr;
    PG_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), p, 0));
    c->pg.peer_tags[n++] = d;
  }
  c->pg.n_peer = n;
  return HS_OK;
}
