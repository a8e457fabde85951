// The serving-step context: one per GPU replica.
//
// Owns the model weights, the paged KV pool, the device residual store, the
// pinned (mapped) piggyback mailboxes, the pinned host KV arena of offloaded
// requests and the CPU-attention worker pool, and launches one transformer
// layer over the concatenated LS+BE rows per hs_layer() call.  This is the
// real work behind Engine._run_layer (reference
// pkg/src/hybridserve/engine.py:921-950):
//
//   rows [0, B)        batch rows of the iteration plan (decodes, chunk tokens)
//   rows [B, B+C)      carry rows: QKV(l) of piggyback chains, shipped D2H
//                      (layer 1: injected fresh tokens, engine.py:995-998;
//                       l > 1: chains merged at l-1, engine.py:1002-1004)
//   rows [B, B+M)      merged rows: host attention results entering
//                      Proj + ResidualAdd + MLP + ResidualAdd at layer l
//                      (engine.py:999-1001), residual fetched from the store
//
// All launches go to one stream; nothing here blocks on the host except
// hs_iter_end (token readback) and hs_cpu_attend (replay-mode service).
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <new>
#include <vector>

#include "hs_common.cuh"
#include "hs_internal.h"
#include "hs_step.h"

#include "hs_ctx.h"

namespace {

// ---- metadata offsets (ints) inside dm / staging ----
struct MetaLayout {
  size_t row_slot, row_pos, row_token, row_mode, chunks, row_chunk_begin, tiles, logit_rows,
      logit_slot, merge_slot, restart_slot, restart_pos, restart_token, restart_mode, total;
};

MetaLayout layout_of(const hs_rt_cfg& r) {
  MetaLayout L{};
  size_t o = 0;
  const size_t R = r.max_rows;
  L.row_slot = o; o += R;
  L.row_pos = o; o += R;
  L.row_token = o; o += R;
  L.row_mode = o; o += R;
  L.chunks = o; o += static_cast<size_t>(r.max_chunks) * 5;
  L.row_chunk_begin = o; o += R + 1;
  L.tiles = o; o += R * 4;
  L.logit_rows = o; o += R;
  L.logit_slot = o; o += R;
  L.merge_slot = o; o += R;
  L.restart_slot = o; o += R;
  L.restart_pos = o; o += R;
  L.restart_token = o; o += R;
  L.restart_mode = o; o += R;
  L.total = o;
  return L;
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      return set_error(HS_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x,                  \
                       cudaGetErrorString(e_));                                            \
  } while (0)

#define RC(x)                                                                              \
  do {                                                                                     \
    int rc_ = (x);                                                                         \
    if (rc_ != HS_OK) {                                                                    \
      if (rc_ == HS_E_CUDA)                                                                \
        return set_error(HS_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x,                \
                         cudaGetErrorString(cudaGetLastError()));                          \
      return set_error(rc_, "%s:%d %s failed", __FILE__, __LINE__, #x);                    \
    }                                                                                      \
  } while (0)

// Every device buffer starts zeroed: memory recycled from a context freed
// earlier in the process holds that context's bytes (NaN patterns included),
// and masked attention tails multiply P = 0 into whatever V holds.
template <typename T>
int dalloc(T** p, size_t n) {
  const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
  CK(cudaMalloc(reinterpret_cast<void**>(p), bytes));
  CK(cudaMemset(*p, 0, bytes));
  // cudaMemset runs on the legacy stream, which does not order against the
  // context's non-blocking streams: finish it before anything can use p
  CK(cudaDeviceSynchronize());
  return HS_OK;
}

// Host-to-device copy ordered on the context stream and complete on return
// (a pageable cudaMemcpy can return before its DMA has landed, and the
// legacy stream it uses does not order against the non-blocking streams).
int h2d(hs_ctx* c, void* dst, const void* src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->st));
  CK(cudaStreamSynchronize(c->st));
  return HS_OK;
}

int make_act(ActBuf& a, int rows, int k) {
  RC(dalloc(&a.p, static_cast<size_t>(rows) * k));
  a.rows = rows;
  a.k = k;
  for (int i = 0; i < 5; ++i)
    if (make_act_map(&a.maps[i], a.p, rows, k, k, kBns[i]) != HS_OK)
      return set_error(HS_E_CUDA, "activation map encode failed");
  return HS_OK;
}

cudaEvent_t prof_event(hs_ctx* c) {
  if (!c->prof_free.empty()) {
    cudaEvent_t e = c->prof_free.back();
    c->prof_free.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {  // records a start event now and a stop event on destruction
  hs_ctx* c;
  int cls;
  double bytes, flops;
  cudaEvent_t a = nullptr;
  ProfScope(hs_ctx* c_, int cls_, double bytes_, double flops_)
      : c(c_), cls(cls_), bytes(bytes_), flops(flops_) {
    if (c->prof_on) {
      a = prof_event(c);
      cudaEventRecord(a, c->st);
    }
  }
  ~ProfScope() {
    if (!a) return;
    cudaEvent_t b = prof_event(c);
    cudaEventRecord(b, c->st);
    c->prof_pending.push_back({cls, a, b, bytes, flops});
  }
};

int prof_collect(hs_ctx* c) {
  if (c->prof_pending.empty()) return HS_OK;
  CK(cudaEventSynchronize(c->prof_pending.back().b));
  for (auto& r : c->prof_pending) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    double* st = c->prof_stats[r.cls];
    st[0] += 1;
    st[1] += ms;
    st[2] += r.bytes;
    st[3] += r.flops;
    c->prof_free.push_back(r.a);
    c->prof_free.push_back(r.b);
  }
  c->prof_pending.clear();
  return HS_OK;
}

// GEMM over `tokens` rows of an activation buffer against a cached weight map.
int gemm(hs_ctx* c, const CUtensorMap& mw, const ActBuf& x, int tokens, int n_out, int k,
         Planes* planes_out) {
  if (tokens <= 0) {
    *planes_out = Planes(1);
    return HS_OK;
  }
  // algorithmic traffic: weights + bf16 activations in + bf16 result out
  ProfScope ps(c, 0, 2.0 * n_out * k + 2.0 * tokens * k + 2.0 * tokens * n_out,
               2.0 * tokens * n_out * k);
  const int bn = gemm_pick_bn(tokens);
  const size_t per_split = static_cast<size_t>(tokens) * n_out;
  const int cap = static_cast<int>(std::min<size_t>(16, c->part_floats / per_split));
  if (cap < 1) return set_error(HS_E_CAPACITY, "split-K buffer too small for %d x %d", tokens, n_out);
  if (gemm_pair_ok(n_out, k, tokens))  // prefill-sized batches: CTA pairs
    return gemm_launch_pair(mw, x.maps[bn_index(128)], c->part, n_out, tokens, k, cap, false,
                            c->st, planes_out);
  return gemm_launch_planes(mw, x.maps[bn_index(bn)], bn, c->part, n_out, tokens, k, cap, c->st,
                            planes_out);
}

// GEMM with an epilogue fused into its stream-K fixup (no partial planes
// leave the kernel); the split-K buffer is scratch for multi-segment tiles.
int gemm_fused(hs_ctx* c, const CUtensorMap& mw, const ActBuf& x, int tokens, int n_out, int k,
               int epi, const EpiParams& ep) {
  if (tokens <= 0) return HS_OK;
  const int bn = gemm_pick_bn(tokens);
  const size_t per_split = static_cast<size_t>(tokens) * n_out;
  const int cap = static_cast<int>(std::min<size_t>(16, c->part_floats / per_split));
  if (cap < 1) return set_error(HS_E_CAPACITY, "split-K buffer too small for %d x %d", tokens, n_out);
  ProfScope ps(c, 0, 2.0 * n_out * k + 2.0 * tokens * k + 2.0 * tokens * n_out,
               2.0 * tokens * n_out * k);
  return gemm_launch_fused(mw, x.maps[bn_index(bn)], bn, c->part, n_out, tokens, k, cap, epi, ep,
                           c->st);
}

// A fused epilogue pays a serial fixup that reads every other K-segment of
// the tile; beyond a few segments the parallel glue kernel is faster.
constexpr int kFuseMaxSegments = 1;  // measured: a fixup on the critical path loses at small M

bool fuse_ok(hs_ctx* c, int tokens, int n_out, int k) {
  if (tokens <= 0) return true;  // nothing to launch either way
  const int bn = gemm_pick_bn(tokens);
  const size_t per_split = static_cast<size_t>(tokens) * n_out;
  const int cap = static_cast<int>(std::min<size_t>(16, c->part_floats / per_split));
  return gemm_pick_splits(n_out, k, tokens, bn, cap) <= kFuseMaxSegments;
}

EpiParams epi_base(hs_ctx* c) {
  EpiParams ep{};
  ep.tile_sem = c->tile_sem;
  ep.h = c->h;
  ep.ld_h = c->m.d;
  ep.act = c->act.p;
  ep.ld_act = c->m.ffn;
  ep.rope_cos = c->rope_cos;
  ep.rope_sin = c->rope_sin;
  ep.qbuf = c->qbuf;
  ep.q_row_stride = c->m.n_q * c->m.hd;
  ep.kv_pool = c->kv_pool;
  ep.geom = c->geom;
  ep.page_table = c->page_table;
  ep.pt_stride = c->r.max_pages_per_req;
  ep.ship = c->ship_d;
  ep.ship_stride = c->m.qkv_n();
  ep.n_q = c->m.n_q;
  ep.n_kv = c->m.n_kv;
  ep.hd = c->m.hd;
  return ep;
}

int* stage(hs_ctx* c, size_t n) {
  // pinned staging ring: half per iteration, guarded by the event of the
  // iteration that last used it
  const size_t half = c->meta_ints;
  if (c->stage_pos + n > half) return nullptr;
  int* p = c->hm + c->stage_half * half + c->stage_pos;
  c->stage_pos += n;
  return p;
}

int upload(hs_ctx* c, size_t dst_off, const int* src, size_t n) {
  if (n == 0) return HS_OK;
  int* s = stage(c, n);
  if (!s) return set_error(HS_E_CAPACITY, "metadata staging overflow");
  std::memcpy(s, src, n * sizeof(int));
  CK(cudaMemcpyAsync(c->dm + dst_off, s, n * sizeof(int), cudaMemcpyHostToDevice, c->st));
  return HS_OK;
}

int upload_fill(hs_ctx* c, size_t dst_off, int value, size_t n) {
  if (n == 0) return HS_OK;
  int* s = stage(c, n);
  if (!s) return set_error(HS_E_CAPACITY, "metadata staging overflow");
  for (size_t i = 0; i < n; ++i) s[i] = value;
  CK(cudaMemcpyAsync(c->dm + dst_off, s, n * sizeof(int), cudaMemcpyHostToDevice, c->st));
  return HS_OK;
}

// Packs several int arrays into one pinned staging run and ships them with a
// single cudaMemcpyAsync into a device block; returns device pointers.
// With dev == nullptr the kernels read the staging run itself through its
// mapped device alias (zero-copy: no copy node between two PDL launches).
struct Packer {
  hs_ctx* c;
  int* host = nullptr;
  int* dev;
  size_t n = 0, cap;
  bool zero_copy;
  Packer(hs_ctx* c_, int* dev_, size_t cap_) : c(c_), dev(dev_), cap(cap_), zero_copy(!dev_) {}
  bool reserve(size_t total) {
    host = stage(c, total);
    cap = total;
    if (host && zero_copy) dev = c->hm_d + (host - c->hm);
    return host != nullptr;
  }
  const int* add(const int* src, size_t cnt) {
    const int* d = dev + n;
    if (cnt) std::memcpy(host + n, src, cnt * sizeof(int));
    n += cnt;
    return d;
  }
  const int* fill(int v, size_t cnt) {
    const int* d = dev + n;
    for (size_t i = 0; i < cnt; ++i) host[n + i] = v;
    n += cnt;
    return d;
  }
  int flush(cudaStream_t st) {
    if (n == 0 || zero_copy) return HS_OK;
    CK(cudaMemcpyAsync(dev, host, n * sizeof(int), cudaMemcpyHostToDevice, st));
    return HS_OK;
  }
};

// deterministic N(0, std) weights from a counter hash (splitmix64 + Box-Muller)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void init_normal_kernel(bf16* w, size_t n, uint64_t seed, float std) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint64_t a = mix64(seed ^ (i * 2 + 0x1234567ull));
    const uint64_t b = mix64(a ^ 0xA5A5A5A5DEADBEEFull);
    const float u1 = (static_cast<float>(a >> 40) + 1.0f) * (1.0f / 16777217.0f);
    const float u2 = static_cast<float>(b >> 40) * (1.0f / 16777216.0f);
    const float z = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
    w[i] = __float2bfloat16(z * std);
  }
}

__global__ void init_normal_f32_kernel(float* w, size_t n, uint64_t seed, float std) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint64_t a = mix64(seed ^ (i * 2 + 0x1234567ull));
    const uint64_t b = mix64(a ^ 0xA5A5A5A5DEADBEEFull);
    const float u1 = (static_cast<float>(a >> 40) + 1.0f) * (1.0f / 16777217.0f);
    const float u2 = static_cast<float>(b >> 40) * (1.0f / 16777216.0f);
    w[i] = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2) * std;
  }
}

__global__ void fill_f32_kernel(float* p, size_t n, float v) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

int rope_init(hs_ctx* c) {
  const int half = c->m.hd / 2;
  std::vector<float> cs(static_cast<size_t>(c->r.max_pos) * half), sn(cs.size());
  // inverse frequencies and angles in float64 (rounded to fp32 once, at the
  // table): at the 9k-32k positions of BE contexts an fp32 inverse
  // frequency alone would put ~5e-4 rad of error into the angle
  std::vector<double> inv(half);
  for (int i = 0; i < half; ++i)
    inv[i] = 1.0 / std::pow(static_cast<double>(c->m.theta), 2.0 * i / c->m.hd);
  for (int p = 0; p < c->r.max_pos; ++p)
    for (int i = 0; i < half; ++i) {
      const double a = static_cast<double>(p) * inv[i];
      cs[static_cast<size_t>(p) * half + i] = static_cast<float>(std::cos(a));
      sn[static_cast<size_t>(p) * half + i] = static_cast<float>(std::sin(a));
    }
  RC(dalloc(&c->rope_cos, cs.size()));
  RC(dalloc(&c->rope_sin, sn.size()));
  RC(h2d(c, c->rope_cos, cs.data(), cs.size() * 4));
  RC(h2d(c, c->rope_sin, sn.data(), sn.size() * 4));
  return HS_OK;
}

int build_maps(hs_ctx* c) {
  const ModelCfg& m = c->m;
  c->m_qkv.resize(m.layers);
  c->m_o.resize(m.layers);
  c->m_gu.resize(m.layers);
  c->m_down.resize(m.layers);
  for (int l = 0; l < m.layers; ++l) {
    if (make_weight_map(&c->m_qkv[l], c->w_qkv[l], m.qkv_n(), m.d) ||
        make_weight_map(&c->m_o[l], c->w_o[l], m.d, m.n_q * m.hd) ||
        make_weight_map(&c->m_gu[l], c->w_gu[l], 2 * m.ffn, m.d) ||
        make_weight_map(&c->m_down[l], c->w_down[l], m.d, m.ffn))
      return set_error(HS_E_CUDA, "weight map encode failed");
  }
  if (make_weight_map(&c->m_lm, c->w_lm, m.vocab, m.d))
    return set_error(HS_E_CUDA, "lm head map encode failed");
  return HS_OK;
}

void free_all(hs_ctx* c) {
  // stop and join the CPU-attention workers first: an in-flight work item
  // reads the ship mailbox and host KV and writes the result mailbox / tags
  // the remote relays complete items into the CPU service: stop them first
  for (auto* r : c->remotes)
    if (r) remote_destroy(r);
  c->remotes.clear();
  if (c->cpu) destroy_cpu_service(c->cpu);
  c->cpu = nullptr;
  pg_free(c);
  auto F = [](void* p) {
    if (p) cudaFree(p);
  };
  F(c->w_embed);
  F(c->w_lm);
  F(c->w_final);
  for (auto p : c->w_qkv) F(p);
  for (auto p : c->w_o) F(p);
  for (auto p : c->w_gu) F(p);
  for (auto p : c->w_down) F(p);
  for (auto p : c->n_in) F(p);
  for (auto p : c->n_post) F(p);
  if (!c->fp32) F(c->kv_pool);
  F(c->kv_f32);
  F(c->fw_embed);
  F(c->fw_lm);
  for (auto* v : {&c->fw_qkv, &c->fw_o, &c->fw_gu, &c->fw_down})
    for (auto p : *v) F(p);
  for (float* p : {c->fx, c->fx2, c->fattn, c->fact, c->fq, c->flin, c->fxr}) F(p);
  F(c->page_table);
  F(c->h);
  F(c->hr);
  for (ActBuf* a : {&c->xn, &c->xn2, &c->attn, &c->act, &c->lin, &c->xr}) F(a->p);
  F(c->qbuf);
  F(c->part);
  F(c->o_part);
  F(c->lse_part);
  F(c->resid);
  F(c->last_token);
  F(c->tok);
  F(c->tok_out);
  F(c->rope_cos);
  F(c->rope_sin);
  F(c->logits);
  F(c->dm);
  F(c->dm_iter);
  F(c->dm_layer);
  F(c->dec_counters);
  F(c->tile_sem);
  if (c->hm) cudaFreeHost(c->hm);
  if (c->tokens_pinned) cudaFreeHost(c->tokens_pinned);
  if (c->ship_h) cudaFreeHost(c->ship_h);
  if (c->result_h) cudaFreeHost(c->result_h);
  if (c->tag_h) cudaFreeHost(c->tag_h);
  if (c->fault_h) cudaFreeHost(c->fault_h);
  if (c->hkv_h) cudaFreeHost(c->hkv_h);
  for (auto& e : c->stage_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : c->marks) cudaEventDestroy(e);
  for (auto e : c->iter_ev)
    if (e) cudaEventDestroy(e);
  if (c->anchor) cudaEventDestroy(c->anchor);
  if (c->tok_ring) cudaFreeHost(c->tok_ring);
  if (c->logit_ring) cudaFreeHost(c->logit_ring);
  for (auto e : c->prof_free) cudaEventDestroy(e);
  for (auto& r : c->prof_pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c->timers) cudaEventDestroy(e);
  for (auto& kv : c->swap_ev) cudaEventDestroy(kv.second);
  F(c->swap_stage);
  if (c->copy_st) cudaStreamDestroy(c->copy_st);
  if (c->st) cudaStreamDestroy(c->st);
  delete c->pool;
}

// Pins the calling thread to `cpus` for its lifetime so that pages it
// first-touches (cudaHostAlloc pins and zero-fills them) land on that NUMA
// node under the default local-allocation policy.
struct AffinityScope {
  cpu_set_t saved;
  bool active = false;
  explicit AffinityScope(const std::vector<int>& cpus) {
    if (cpus.empty() || pthread_getaffinity_np(pthread_self(), sizeof(saved), &saved)) return;
    cpu_set_t set;
    CPU_ZERO(&set);
    for (int cpu : cpus) CPU_SET(cpu, &set);
    active = pthread_setaffinity_np(pthread_self(), sizeof(set), &set) == 0;
  }
  ~AffinityScope() {
    if (active) pthread_setaffinity_np(pthread_self(), sizeof(saved), &saved);
  }
};

int create(const hs_model_cfg* mc, const hs_rt_cfg* rc, hs_ctx* c) {
  ModelCfg& m = c->m;
  m = ModelCfg{mc->d_model, mc->n_layers, mc->n_q, mc->n_kv, mc->head_dim, mc->ffn, mc->vocab,
               mc->rope_theta, mc->norm_eps};
  c->r = *rc;
  const hs_rt_cfg& r = c->r;
  if (r.precision != HS_PREC_BF16 && r.precision != HS_PREC_FP32)
    return set_error(HS_E_CONFIG, "precision %d unknown", r.precision);
  c->fp32 = r.precision == HS_PREC_FP32;
  c->kv_elem = c->fp32 ? 4 : 2;
  m.fp32 = c->fp32;
  if (m.d % 128 || m.ffn % 128 || m.vocab % 128 || (m.hd != 64 && m.hd != 128) ||
      m.n_q % m.n_kv || m.n_q / m.n_kv > 16 || (m.n_q * m.hd) % 64 || m.qkv_n() % 128)
    return set_error(HS_E_CONFIG, "model dims unsupported (d/ffn/vocab %% 128, hd 64|128, G<=16)");
  if (r.max_rows < 1 || r.max_slots < 1 || r.kv_pages < 1 || r.max_pages_per_req < 1 ||
      r.max_pos < 1 || r.max_chunks < 1)
    return set_error(HS_E_CONFIG, "runtime capacities must be >= 1");
  CK(cudaSetDevice(r.device));
  CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  // weights (matrices bf16 [out][in], or fp32 in the validation datapath)
  const size_t d = m.d;
  RC(dalloc(&c->w_final, d));
  c->n_in.assign(m.layers, nullptr);
  c->n_post.assign(m.layers, nullptr);
  for (int l = 0; l < m.layers; ++l) {
    RC(dalloc(&c->n_in[l], d));
    RC(dalloc(&c->n_post[l], d));
  }
  if (c->fp32) {
    RC(dalloc(&c->fw_embed, static_cast<size_t>(m.vocab) * d));
    RC(dalloc(&c->fw_lm, static_cast<size_t>(m.vocab) * d));
    for (auto* v : {&c->fw_qkv, &c->fw_o, &c->fw_gu, &c->fw_down}) v->assign(m.layers, nullptr);
    for (int l = 0; l < m.layers; ++l) {
      RC(dalloc(&c->fw_qkv[l], static_cast<size_t>(m.qkv_n()) * d));
      RC(dalloc(&c->fw_o[l], d * m.n_q * m.hd));
      RC(dalloc(&c->fw_gu[l], 2 * static_cast<size_t>(m.ffn) * d));
      RC(dalloc(&c->fw_down[l], d * m.ffn));
    }
  } else {
    RC(dalloc(&c->w_embed, static_cast<size_t>(m.vocab) * d));
    RC(dalloc(&c->w_lm, static_cast<size_t>(m.vocab) * d));
    c->w_qkv.assign(m.layers, nullptr);
    c->w_o.assign(m.layers, nullptr);
    c->w_gu.assign(m.layers, nullptr);
    c->w_down.assign(m.layers, nullptr);
    for (int l = 0; l < m.layers; ++l) {
      RC(dalloc(&c->w_qkv[l], static_cast<size_t>(m.qkv_n()) * d));
      RC(dalloc(&c->w_o[l], d * m.n_q * m.hd));
      RC(dalloc(&c->w_gu[l], 2 * static_cast<size_t>(m.ffn) * d));
      RC(dalloc(&c->w_down[l], d * m.ffn));
    }
    RC(build_maps(c));
  }
  // kv pool
  c->geom = KvGeom{m.layers, r.kv_pages, m.n_kv, m.hd};
  const size_t pool_elems =
      static_cast<size_t>(m.layers) * r.kv_pages * 2 * m.n_kv * kPageTokens * m.hd;
  if (c->fp32) {
    RC(dalloc(&c->kv_f32, pool_elems));
    c->kv_pool = reinterpret_cast<bf16*>(c->kv_f32);  // swaps move it as bytes
  } else {
    RC(dalloc(&c->kv_pool, pool_elems));
    if (make_kv_map(&c->m_kv, c->kv_pool, c->geom)) return set_error(HS_E_CUDA, "kv map failed");
  }
  // zero the pool: the attention kernels multiply the masked tail of a page
  // (P = 0) into V, and 0 x NaN is NaN -- recycled device memory can hold any
  // bit pattern where no token has been written yet
  CK(cudaMemset(c->kv_pool, 0, pool_elems * (c->fp32 ? sizeof(float) : sizeof(bf16))));
  RC(dalloc(&c->page_table, static_cast<size_t>(r.max_slots) * r.max_pages_per_req));
  CK(cudaMemset(c->page_table, 0, static_cast<size_t>(r.max_slots) * r.max_pages_per_req * 4));
  // activations
  const size_t R = r.max_rows;
  RC(dalloc(&c->h, R * d));
  RC(dalloc(&c->hr, R * d));
  if (c->fp32) {
    for (float** p : {&c->fx, &c->fx2, &c->flin, &c->fxr}) RC(dalloc(p, R * d));
    RC(dalloc(&c->fattn, R * m.n_q * m.hd));
    RC(dalloc(&c->fq, R * m.n_q * m.hd));
    RC(dalloc(&c->fact, R * m.ffn));
  } else {
    RC(make_act(c->xn, r.max_rows, m.d));
    RC(make_act(c->xn2, r.max_rows, m.d));
    RC(make_act(c->attn, r.max_rows, m.n_q * m.hd));
    RC(make_act(c->act, r.max_rows, m.ffn));
    RC(make_act(c->lin, r.max_rows, m.d));
    RC(make_act(c->xr, r.max_rows, m.d));
    RC(dalloc(&c->qbuf, R * m.n_q * m.hd));
  }
  const size_t widest = std::max<size_t>(std::max<size_t>(2 * m.ffn, m.vocab), m.qkv_n());
  c->part_floats = std::max<size_t>(R * widest, static_cast<size_t>(16) * 64 * widest);
  RC(dalloc(&c->part, c->part_floats));
  RC(dalloc(&c->o_part, static_cast<size_t>(r.max_chunks) * m.n_q * m.hd));
  RC(dalloc(&c->lse_part, static_cast<size_t>(r.max_chunks) * m.n_q));
  RC(dalloc(&c->resid, static_cast<size_t>(r.max_slots) * d));
  RC(dalloc(&c->last_token, r.max_slots));
  CK(cudaMemset(c->last_token, 0, r.max_slots * 4));
  RC(dalloc(&c->tok, R));
  RC(dalloc(&c->tok_out, 2 * R));
  RC(rope_init(c));
  // metadata
  c->meta_ints = layout_of(r).total + 16 * R * (m.layers + 2);
  RC(dalloc(&c->dm, layout_of(r).total));
  c->iter_cap = 3 * R + 5 * static_cast<size_t>(r.max_chunks) + (R + 1) + 4 * R + 16;
  c->layer_cap = 9 * R + 16;
  RC(dalloc(&c->dm_iter, c->iter_cap));
  RC(dalloc(&c->dm_layer, c->layer_cap));
  RC(dalloc(&c->dec_counters, R * m.n_kv));
  {
    const size_t max_n = std::max<size_t>(std::max<size_t>(m.qkv_n(), 2 * m.ffn),
                                          std::max<size_t>(m.d, m.vocab));
    const size_t tiles = (max_n / 128) * ((R + 15) / 16);
    RC(dalloc(&c->tile_sem, tiles));
    CK(cudaMemset(c->tile_sem, 0, tiles * sizeof(int)));
  }
  CK(cudaMemset(c->dec_counters, 0, R * m.n_kv * sizeof(int)));
  // host allocations below are first-touched on the replica's NUMA node
  c->cpus.assign(r.cpu_list, r.cpu_list + (r.cpu_list ? r.n_cpu_list : 0));
  c->r.cpu_list = nullptr;  // the caller's array is not retained
  for (int cpu : c->cpus)
    if (cpu < 0 || cpu >= CPU_SETSIZE) return set_error(HS_E_CONFIG, "cpu_list entry %d invalid", cpu);
  AffinityScope near(c->cpus);
  CK(cudaHostAlloc(reinterpret_cast<void**>(&c->hm), 2 * c->meta_ints * sizeof(int),
                   cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->hm_d), c->hm, 0));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&c->tokens_pinned), 2 * R * sizeof(int),
                   cudaHostAllocDefault));
  for (auto& e : c->stage_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // piggyback mailboxes: pinned host memory mapped into the device space
  const size_t ship_elems = static_cast<size_t>(r.max_slots) * m.qkv_n();
  const size_t res_elems = static_cast<size_t>(r.max_slots) * m.n_q * m.hd;
  CK(cudaHostAlloc(reinterpret_cast<void**>(&c->ship_h), ship_elems * c->kv_elem,
                   cudaHostAllocMapped));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&c->result_h), res_elems * c->kv_elem,
                   cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->ship_d), c->ship_h, 0));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->result_d), c->result_h, 0));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&c->tag_h), r.max_slots * sizeof(unsigned),
                   cudaHostAllocMapped));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&c->fault_h), 4 * sizeof(unsigned), cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->tag_d), c->tag_h, 0));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->fault_d), c->fault_h, 0));
  std::memset(c->tag_h, 0xff, r.max_slots * sizeof(unsigned));
  std::memset(c->fault_h, 0, 4 * sizeof(unsigned));
  // host KV arena
  c->regions.assign(r.max_slots, HostRegion{});
  if (r.host_kv_bytes > 0) {
    c->hkv_bytes = static_cast<size_t>(r.host_kv_bytes);
    CK(cudaHostAlloc(reinterpret_cast<void**>(&c->hkv_h), c->hkv_bytes, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->hkv_d), c->hkv_h, 0));
    c->free_list.push_back({0, c->hkv_bytes});
  }
  c->pool = new ThreadPool(std::max(0, r.cpu_threads - 1), c->cpus);
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK(cudaStreamCreateWithPriority(&c->copy_st, cudaStreamNonBlocking, lo));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&c->tok_ring),
                   sizeof(int) * hs_ctx::kIterRing * 2 * r.max_rows, cudaHostAllocDefault));
  for (auto& e : c->iter_ev) CK(cudaEventCreate(&e));
  CK(cudaEventCreate(&c->anchor));
  c->marks.resize(64);
  c->timers.resize(8192);
  for (auto& e : c->marks) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : c->timers) CK(cudaEventCreate(&e));
  // legacy-stream memsets/copies above vs the non-blocking streams
  CK(cudaDeviceSynchronize());
  return HS_OK;
}

bf16* host_region(hs_ctx* c, int slot) {
  return reinterpret_cast<bf16*>(reinterpret_cast<uint8_t*>(c->hkv_h) + c->regions[slot].offset);
}

// mailbox rows of a slot (bf16 rows, or fp32 rows in the validation datapath)
bf16* ship_row(hs_ctx* c, int slot) {
  return reinterpret_cast<bf16*>(reinterpret_cast<uint8_t*>(c->ship_h) +
                                 static_cast<size_t>(slot) * c->m.qkv_n() * c->kv_elem);
}
bf16* result_row(hs_ctx* c, int slot) {
  return reinterpret_cast<bf16*>(reinterpret_cast<uint8_t*>(c->result_h) +
                                 static_cast<size_t>(slot) * c->m.n_q * c->m.hd * c->kv_elem);
}
size_t region_bytes(const hs_ctx* c, int cap_tokens) {
  return static_cast<size_t>(cap_tokens) * c->m.layers * 2 * c->m.n_kv * c->m.hd * c->kv_elem;
}
// the pool / host-region geometry in bf16 units (an fp32 head row is two
// bf16-sized halves per element: the swap kernels move bytes)
KvGeom swap_geom(const hs_ctx* c) {
  KvGeom g = c->geom;
  g.head_dim = g.head_dim * c->kv_elem / 2;
  return g;
}

// A result row is complete: publish its tag (release: the row's bytes are
// visible to a reader that acquires the tag, the device included).
void publish_tag(hs_ctx* c, int slot, int ctx, int layer) {
  reinterpret_cast<std::atomic<unsigned>*>(c->tag_h + slot)
      ->store(static_cast<unsigned>(HS_RESULT_TAG(ctx, layer)), std::memory_order_release);
}

// The slot's previous completion tag no longer stands for a result in the
// mailbox (a new work item of the slot is being serviced).
void retract_tag(hs_ctx* c, int slot) {
  reinterpret_cast<std::atomic<unsigned>*>(c->tag_h + slot)->store(0xffffffffu, std::memory_order_relaxed);
}

// Integrity faults the kernels recorded (a merged result whose completion
// tag did not match): HS_E_INTEGRITY, the reference's IntegrityFault.
int check_device_faults(hs_ctx* c) {
  volatile unsigned* f = c->fault_h;
  if (!f[0]) return HS_OK;
  const unsigned slot = f[1], layer = f[2], seen = f[3];
  f[0] = 0;
  return set_error(HS_E_INTEGRITY,
                   "piggyback result of slot %u merged at layer %u before it was complete "
                   "(completion tag 0x%x)", slot, layer, seen);
}

// the CPU host a slot's KV lives on (0 = this replica's own host)
int slot_host_of(hs_ctx* c, int slot) {
  return c->slot_host ? c->slot_host[slot].load(std::memory_order_acquire) : 0;
}

int ensure_cpu_service(hs_ctx* c) {
  if (c->cpu) return HS_OK;
  if (c->r.cpu_threads <= 0) return set_error(HS_E_CONFIG, "no CPU attention threads configured");
  c->cpu = make_cpu_service(c->m, c->r.cpu_threads, c->cpus);
  cpu_service_bind(
      c->cpu, [c](int s) { return ship_row(c, s); }, [c](int s) { return result_row(c, s); },
      [c](int s) { return host_region(c, s); }, [c](int s) { return c->regions[s].cap; },
      [c](int s, int ctx, int layer) { publish_tag(c, s, ctx, layer); },
      [c](int s) { retract_tag(c, s); });
  cpu_service_route(c->cpu, [c](int s, int layer, int ctx, cudaEvent_t ev,
                                std::function<void()> done) {
    const int h = slot_host_of(c, s);
    if (h <= 0) return false;
    remote_attend(c->remotes[h], s, layer, ctx, ev, ship_row(c, s), result_row(c, s),
                  [c, s] { retract_tag(c, s); }, std::move(done));
    return true;
  });
  return HS_OK;
}

// Asynchronous one-shot KV transfer on the copy stream:
//   out: pool pages -> pack (HBM) -> one 2D DMA into the host region
//   in:  one 2D DMA into staging -> unpack into the slot's (new) pages
// ordered after everything already queued on the compute stream.
int swap_async(hs_ctx* c, int slot, int tokens, bool to_host, int* ticket) {
  if (slot < 0 || slot >= c->r.max_slots) return set_error(HS_E_CONFIG, "slot out of range");
  HostRegion& hr = c->regions[slot];
  if (!hr.used) return set_error(HS_E_INTEGRITY, "slot %d has no host KV region", slot);
  if (tokens > hr.cap) return set_error(HS_E_CAPACITY, "swap of %d tokens exceeds region", tokens);
  const ModelCfg& m = c->m;
  const KvGeom sg = swap_geom(c);
  const size_t rows = static_cast<size_t>(m.layers) * 2 * m.n_kv;
  const size_t need = rows * tokens * sg.head_dim;
  if (need > c->swap_stage_elems) {
    CK(cudaStreamSynchronize(c->copy_st));
    if (c->swap_stage) CK(cudaFree(c->swap_stage));
    c->swap_stage = nullptr;
    RC(dalloc(&c->swap_stage, need));
    c->swap_stage_elems = need;
  }
  cudaEvent_t dep, done;
  CK(cudaEventCreateWithFlags(&dep, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  CK(cudaEventRecord(dep, c->st));
  CK(cudaStreamWaitEvent(c->copy_st, dep, 0));
  CK(cudaEventDestroy(dep));
  const int* pages = c->page_table + static_cast<size_t>(slot) * c->r.max_pages_per_req;
  bf16* host = host_region(c, slot);
  const size_t w = static_cast<size_t>(tokens) * sg.head_dim * 2;
  const size_t host_pitch = static_cast<size_t>(hr.cap) * sg.head_dim * 2;
  if (to_host) {
    RC(kv_swap(true, c->kv_pool, sg, pages, tokens, c->swap_stage, tokens, c->copy_st));
    if (tokens > 0)
      CK(cudaMemcpy2DAsync(host, host_pitch, c->swap_stage, w, w, rows, cudaMemcpyDeviceToHost,
                           c->copy_st));
  } else {
    if (tokens > 0)
      CK(cudaMemcpy2DAsync(c->swap_stage, w, host, host_pitch, w, rows, cudaMemcpyHostToDevice,
                           c->copy_st));
    RC(kv_swap(false, c->kv_pool, sg, pages, tokens, c->swap_stage, tokens, c->copy_st));
  }
  CK(cudaEventRecord(done, c->copy_st));
  *ticket = c->next_ticket++;
  c->swap_ev[*ticket] = done;
  return HS_OK;
}

int kv_swap_pages(hs_ctx* c, int slot, int tokens, bool to_host) {
  if (slot < 0 || slot >= c->r.max_slots) return set_error(HS_E_CONFIG, "slot out of range");
  HostRegion& hr = c->regions[slot];
  if (!hr.used) return set_error(HS_E_INTEGRITY, "slot %d has no host KV region", slot);
  if (tokens > hr.cap) return set_error(HS_E_CAPACITY, "swap of %d tokens exceeds region", tokens);
  const int* pages = c->page_table + static_cast<size_t>(slot) * c->r.max_pages_per_req;
  bf16* host = reinterpret_cast<bf16*>(reinterpret_cast<uint8_t*>(c->hkv_d) + hr.offset);
  RC(kv_swap(to_host, c->kv_pool, swap_geom(c), pages, tokens, host, hr.cap, c->st));
  CK(cudaStreamSynchronize(c->st));
  return HS_OK;
}

}  // namespace

namespace hs {
int ctx_cpu_service(hs_ctx* c) { return ensure_cpu_service(c); }
}  // namespace hs

namespace {
template <typename F>
int time_reps(hs_ctx* c, int reps, F&& body, float* us) {
  if (c->fp32) return set_error(HS_E_CONFIG, "probes time the bf16 serving datapath only");
  std::vector<float> ts;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < reps + 2; ++i) {
    CK(cudaEventRecord(a, c->st));
    RC(body());
    CK(cudaEventRecord(b, c->st));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (i >= 2) ts.push_back(ms * 1000.f);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  std::sort(ts.begin(), ts.end());
  *us = ts[ts.size() / 2];
  return HS_OK;
}

int probe_pages(hs_ctx* c, int g, int tokens) {
  const int per = (tokens + kPageTokens - 1) / kPageTokens;
  if (per > c->r.max_pages_per_req || g > c->r.max_slots)
    return set_error(HS_E_CAPACITY, "probe exceeds page table");
  std::vector<int> pt(per);
  for (int s = 0; s < g; ++s) {
    for (int i = 0; i < per; ++i) pt[i] = (s * per + i) % c->r.kv_pages;
    RC(h2d(c, c->page_table + static_cast<size_t>(s) * c->r.max_pages_per_req, pt.data(),
                  per * 4));
  }
  return HS_OK;
}
}  // namespace

extern "C" {

int hs_create(const hs_model_cfg* m, const hs_rt_cfg* r, hs_ctx** out) {
  if (!m || !r || !out) return set_error(HS_E_CONFIG, "null argument");
  hs_ctx* c = new (std::nothrow) hs_ctx();
  if (!c) return set_error(HS_E_CAPACITY, "out of host memory");
  const int rc = create(m, r, c);
  if (rc != HS_OK) {
    free_all(c);
    delete c;
    return rc;
  }
  *out = c;
  return HS_OK;
}

int hs_destroy(hs_ctx* c) {
  if (!c) return HS_OK;
  if (g_hprof_on) {
    static const char* names[6] = {"layer", "pack", "plan", "launch", "iter_begin", "iter_end"};
    for (int i = 0; i < 6; ++i)
      if (g_hprof_n[i])
        fprintf(stderr, "[hs host] %-10s n=%8llu  %8.2f us/call  %10.1f ms total\n", names[i],
                g_hprof_n[i], g_hprof_ns[i] / g_hprof_n[i] / 1e3, g_hprof_ns[i] / 1e6);
  }
  cudaStreamSynchronize(c->st);
  free_all(c);
  delete c;
  return HS_OK;
}

void* hs_stream(hs_ctx* c) { return c ? c->st : nullptr; }

int hs_set_weight(hs_ctx* c, int kind, int layer, const void* host, size_t bytes) {
  const ModelCfg& m = c->m;
  const size_t d = m.d;
  void* dst = nullptr;
  size_t want = 0;
  const bool per_layer = kind >= HS_W_QKV;
  if (per_layer && (layer < 0 || layer >= m.layers))
    return set_error(HS_E_CONFIG, "layer %d out of range", layer);
  switch (kind) {
    case HS_W_EMBED: dst = c->w_embed; want = static_cast<size_t>(m.vocab) * d * 2; break;
    case HS_W_LM_HEAD: dst = c->w_lm; want = static_cast<size_t>(m.vocab) * d * 2; break;
    case HS_W_FINAL_NORM: dst = c->w_final; want = d * 4; break;
    case HS_W_QKV: dst = c->w_qkv[layer]; want = static_cast<size_t>(m.qkv_n()) * d * 2; break;
    case HS_W_O: dst = c->w_o[layer]; want = d * m.n_q * m.hd * 2; break;
    case HS_W_GATE_UP: dst = c->w_gu[layer]; want = 2 * static_cast<size_t>(m.ffn) * d * 2; break;
    case HS_W_DOWN: dst = c->w_down[layer]; want = d * m.ffn * 2; break;
    case HS_W_NORM_IN: dst = c->n_in[layer]; want = d * 4; break;
    case HS_W_NORM_POST: dst = c->n_post[layer]; want = d * 4; break;
    default: return set_error(HS_E_CONFIG, "unknown weight kind %d", kind);
  }
  if (c->fp32 && kind != HS_W_FINAL_NORM && kind != HS_W_NORM_IN && kind != HS_W_NORM_POST) {
    // validation datapath: fp32 matrices in the caller's [out][in] order
    float* fdst = nullptr;
    switch (kind) {
      case HS_W_EMBED: fdst = c->fw_embed; break;
      case HS_W_LM_HEAD: fdst = c->fw_lm; break;
      case HS_W_QKV: fdst = c->fw_qkv[layer]; break;
      case HS_W_O: fdst = c->fw_o[layer]; break;
      case HS_W_GATE_UP: fdst = c->fw_gu[layer]; break;
      default: fdst = c->fw_down[layer]; break;
    }
    if (bytes != 2 * want)
      return set_error(HS_E_CONFIG, "fp32 weight %d: %zu bytes, want %zu", kind, bytes, 2 * want);
    RC(h2d(c, fdst, host, bytes));
    return HS_OK;
  }
  if (bytes != want) return set_error(HS_E_CONFIG, "weight %d: %zu bytes, want %zu", kind, bytes, want);
  if (kind == HS_W_QKV || kind == HS_W_GATE_UP) {
    // rows reordered for the fused epilogues (see permute_rows)
    bf16* tmp = nullptr;
    CK(cudaMalloc(reinterpret_cast<void**>(&tmp), bytes));
    RC(h2d(c, tmp, host, bytes));
    const int rows = kind == HS_W_QKV ? m.qkv_n() : 2 * m.ffn;
    const int rc = permute_rows(tmp, static_cast<bf16*>(dst), rows, m.d,
                                kind == HS_W_QKV ? 1 : 0, kind == HS_W_QKV ? m.hd : m.ffn, c->st);
    CK(cudaStreamSynchronize(c->st));
    cudaFree(tmp);
    if (rc != HS_OK) return set_error(HS_E_CUDA, "weight permutation failed");
    return HS_OK;
  }
  RC(h2d(c, dst, host, bytes));
  return HS_OK;
}

int hs_init_weights(hs_ctx* c, uint64_t seed, float std) {
  const ModelCfg& m = c->m;
  const size_t d = m.d;
  uint64_t s = seed * 0x100000001B3ull + 17;
  auto init = [&](bf16* p, size_t n) {
    init_normal_kernel<<<148 * 8, 256, 0, c->st>>>(p, n, s, std);
    s = s * 6364136223846793005ull + 1442695040888963407ull;
  };
  auto ones = [&](float* p, size_t n) { fill_f32_kernel<<<64, 256, 0, c->st>>>(p, n, 1.0f); };
  if (c->fp32) {
    auto initf = [&](float* p, size_t n) {
      init_normal_f32_kernel<<<148 * 8, 256, 0, c->st>>>(p, n, s, std);
      s = s * 6364136223846793005ull + 1442695040888963407ull;
    };
    initf(c->fw_embed, static_cast<size_t>(m.vocab) * d);
    initf(c->fw_lm, static_cast<size_t>(m.vocab) * d);
    ones(c->w_final, d);
    for (int l = 0; l < m.layers; ++l) {
      initf(c->fw_qkv[l], static_cast<size_t>(m.qkv_n()) * d);
      initf(c->fw_o[l], d * m.n_q * m.hd);
      initf(c->fw_gu[l], 2 * static_cast<size_t>(m.ffn) * d);
      initf(c->fw_down[l], d * m.ffn);
      ones(c->n_in[l], d);
      ones(c->n_post[l], d);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->st));
    return HS_OK;
  }
  init(c->w_embed, static_cast<size_t>(m.vocab) * d);
  init(c->w_lm, static_cast<size_t>(m.vocab) * d);
  ones(c->w_final, d);
  for (int l = 0; l < m.layers; ++l) {
    init(c->w_qkv[l], static_cast<size_t>(m.qkv_n()) * d);
    init(c->w_o[l], d * m.n_q * m.hd);
    init(c->w_gu[l], 2 * static_cast<size_t>(m.ffn) * d);
    init(c->w_down[l], d * m.ffn);
    ones(c->n_in[l], d);
    ones(c->n_post[l], d);
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->st));
  return HS_OK;
}

int hs_set_page_table(hs_ctx* c, int slot, const int* pages, int n) {
  if (slot < 0 || slot >= c->r.max_slots || n < 0 || n > c->r.max_pages_per_req)
    return set_error(HS_E_CONFIG, "page table row out of range (slot %d, %d pages)", slot, n);
  for (int i = 0; i < n; ++i)
    if (pages[i] < 0 || pages[i] >= c->r.kv_pages)
      return set_error(HS_E_CONFIG, "page id %d out of range", pages[i]);
  int* s = stage(c, n);
  if (!s) return set_error(HS_E_CAPACITY, "metadata staging overflow");
  std::memcpy(s, pages, n * sizeof(int));
  CK(cudaMemcpyAsync(c->page_table + static_cast<size_t>(slot) * c->r.max_pages_per_req, s,
                     n * sizeof(int), cudaMemcpyHostToDevice, c->st));
  return HS_OK;
}

int hs_keep_logits(hs_ctx* c, int on) {
  c->keep_logits = on != 0;
  const size_t per_iter = static_cast<size_t>(2 * c->r.max_rows) * c->m.vocab;
  if (c->keep_logits && !c->logits) RC(dalloc(&c->logits, per_iter));
  if (c->keep_logits && !c->logit_ring)
    CK(cudaHostAlloc(reinterpret_cast<void**>(&c->logit_ring),
                     sizeof(float) * hs_ctx::kIterRing * per_iter, cudaHostAllocDefault));
  return HS_OK;
}

int hs_iter_logits(hs_ctx* c, int ticket, float* host, int rows) {
  if (!c->logit_ring) return set_error(HS_E_CONFIG, "logits not kept (hs_keep_logits)");
  if (ticket < c->next_iter - hs_ctx::kIterRing || ticket >= c->next_iter)
    return set_error(HS_E_CONFIG, "iteration ticket %d out of window", ticket);
  const int slot = ticket % hs_ctx::kIterRing;
  if (rows > c->iter_n[slot]) return set_error(HS_E_CONFIG, "only %d logit rows", c->iter_n[slot]);
  CK(cudaEventSynchronize(c->iter_ev[slot]));
  const size_t per_iter = static_cast<size_t>(2 * c->r.max_rows) * c->m.vocab;
  std::memcpy(host, c->logit_ring + slot * per_iter, sizeof(float) * rows * c->m.vocab);
  return HS_OK;
}

int hs_read_logits(hs_ctx* c, float* host, int rows) {
  if (!c->logits) return set_error(HS_E_CONFIG, "logits not kept (hs_keep_logits)");
  if (rows > c->n_tok_out) return set_error(HS_E_CONFIG, "only %d logit rows", c->n_tok_out);
  CK(cudaStreamSynchronize(c->st));
  CK(cudaMemcpy(host, c->logits, static_cast<size_t>(rows) * c->m.vocab * 4,
                cudaMemcpyDeviceToHost));
  return HS_OK;
}

int hs_host_kv_reserve(hs_ctx* c, int slot, int cap_tokens) {
  if (slot < 0 || slot >= c->r.max_slots) return set_error(HS_E_CONFIG, "slot out of range");
  HostRegion& hr = c->regions[slot];
  if (hr.used) return set_error(HS_E_INTEGRITY, "slot %d already holds a host KV region", slot);
  const size_t bytes = region_bytes(c, cap_tokens);
  for (size_t i = 0; i < c->free_list.size(); ++i) {
    auto& f = c->free_list[i];
    if (f.second >= bytes) {
      hr.offset = f.first;
      hr.cap = cap_tokens;
      hr.used = true;
      f.first += bytes;
      f.second -= bytes;
      if (f.second == 0) c->free_list.erase(c->free_list.begin() + i);
      return HS_OK;
    }
  }
  return set_error(HS_E_CAPACITY, "host KV arena exhausted (%zu bytes requested)", bytes);
}

int hs_host_kv_release(hs_ctx* c, int slot) {
  if (slot < 0 || slot >= c->r.max_slots) return set_error(HS_E_CONFIG, "slot out of range");
  HostRegion& hr = c->regions[slot];
  if (!hr.used) return HS_OK;
  if (const int h = slot_host_of(c, slot); h > 0) {
    // the relay may still read the region (a queued PUT): drain it first
    remote_free(c->remotes[h], slot);
    c->slot_host[slot].store(0, std::memory_order_release);
    if (!remote_flush_puts(c->remotes[h], slot))
      return set_error(HS_E_CUDA, "remote CPU host %d: connection failed", h);
  }
  // the slot's last completion tag stands for nothing any more: a later
  // occupant's item with the same (ctx, layer) must not read as complete.
  // Retracted in stream order: a merge of the slot's last result that the
  // host already launched (pipelined iterations) still checks its tag first.
  if (cudaMemsetAsync(c->tag_d + slot, 0xff, sizeof(unsigned), c->st) != cudaSuccess)
    return set_error(HS_E_CUDA, "host_kv_release: tag retract");
  const size_t bytes = region_bytes(c, hr.cap);
  c->free_list.push_back({hr.offset, bytes});
  std::sort(c->free_list.begin(), c->free_list.end());
  std::vector<std::pair<size_t, size_t>> merged;
  for (auto& f : c->free_list) {
    if (!merged.empty() && merged.back().first + merged.back().second == f.first)
      merged.back().second += f.second;
    else
      merged.push_back(f);
  }
  c->free_list.swap(merged);
  hr = HostRegion{};
  return HS_OK;
}

int hs_host_kv_ptr(hs_ctx* c, int slot, void** host_ptr, int* cap) {
  if (slot < 0 || slot >= c->r.max_slots || !c->regions[slot].used)
    return set_error(HS_E_CONFIG, "slot %d has no host KV region", slot);
  *host_ptr = reinterpret_cast<uint8_t*>(c->hkv_h) + c->regions[slot].offset;
  *cap = c->regions[slot].cap;
  return HS_OK;
}

int hs_swap_out(hs_ctx* c, int slot, int tokens) { return kv_swap_pages(c, slot, tokens, true); }
int hs_swap_in(hs_ctx* c, int slot, int tokens) { return kv_swap_pages(c, slot, tokens, false); }

int hs_iter_begin(hs_ctx* c, const hs_iter_desc* d) {
  HProf hp_begin(HP_BEGIN);
  const hs_rt_cfg& r = c->r;
  if (d->n_rows < 0 || d->n_rows > r.max_rows || d->n_decode > d->n_rows ||
      d->n_chunks > r.max_chunks || d->n_logit_rows > d->n_rows || d->n_tiles > r.max_rows)
    return set_error(HS_E_CAPACITY, "iteration exceeds capacities (rows %d, chunks %d)", d->n_rows,
                     d->n_chunks);
  // every batch row writes its K/V into the slot's pages at row_pos and is
  // rotated with the RoPE table row row_pos
  for (int i = 0; i < d->n_rows; ++i) {
    if (d->row_slot[i] < 0 || d->row_slot[i] >= r.max_slots)
      return set_error(HS_E_CONFIG, "row %d: slot %d out of range", i, d->row_slot[i]);
    if (d->row_pos[i] < 0 || d->row_pos[i] >= r.max_pos ||
        d->row_pos[i] / kPageTokens >= r.max_pages_per_req)
      return set_error(HS_E_CONFIG, "row %d: position %d outside max_pos %d / page table", i,
                       d->row_pos[i], r.max_pos);
  }
  // switch pinned staging halves: everything staged into the current half is
  // enqueued before this event; the new half may be rewritten once the
  // copies staged into it last time have executed
  CK(cudaEventRecord(c->stage_ev[c->stage_half], c->st));
  c->stage_half ^= 1;
  CK(cudaEventSynchronize(c->stage_ev[c->stage_half]));
  c->stage_pos = 0;
  const MetaLayout L = layout_of(r);
  c->B = d->n_rows;
  c->D = d->n_decode;
  c->n_chunks = d->n_chunks;
  c->n_tiles = d->n_tiles;
  c->n_logit = d->n_logit_rows;
  c->n_tok_out = 0;
  c->merges_L = 0;
  {
    const size_t total = 3 * static_cast<size_t>(d->n_rows) + 5 * static_cast<size_t>(d->n_chunks) +
                         (d->n_chunks ? d->n_decode + 1 : 0) + 4 * static_cast<size_t>(d->n_tiles);
    if (total > c->iter_cap) return set_error(HS_E_CAPACITY, "iteration metadata too large");
    Packer pk(c, c->dm_iter, total);
    if (!pk.reserve(total)) return set_error(HS_E_CAPACITY, "metadata staging overflow");
    c->it_slot = pk.add(d->row_slot, d->n_rows);
    c->it_pos = pk.add(d->row_pos, d->n_rows);
    c->it_tok = pk.add(d->row_token, d->n_rows);
    c->it_chunks = pk.add(d->chunks, static_cast<size_t>(d->n_chunks) * 5);
    c->it_cbeg = pk.add(d->row_chunk_begin, d->n_chunks ? d->n_decode + 1 : 0);
    c->it_tiles = pk.add(d->tiles, static_cast<size_t>(d->n_tiles) * 4);
    RC(pk.flush(c->st));
  }
  c->h_logit_rows.assign(d->logit_rows, d->logit_rows + d->n_logit_rows);
  c->h_logit_slots.resize(d->n_logit_rows);
  for (int i = 0; i < d->n_logit_rows; ++i) c->h_logit_slots[i] = d->row_slot[d->logit_rows[i]];
  c->dec_kv_tokens = 0;
  for (int r = 0; r < d->n_decode && d->n_chunks; ++r)
    c->dec_kv_tokens += d->chunks[static_cast<size_t>(d->row_chunk_begin[r]) * 5 + 4];
  c->pre_units = 0;
  c->pre_kv_tokens = 0;
  for (int t = 0; t < d->n_tiles; ++t) {
    const double pos0 = d->tiles[t * 4 + 2], nq = d->tiles[t * 4 + 3];
    c->pre_units += nq * pos0 + nq * (nq + 1) / 2;
    c->pre_kv_tokens += pos0 + nq;
  }
  return HS_OK;
}

// HS_SKIP (probe knob, read once): bit mask of layer launches to leave out
// so tools/probe_step.py can measure each kernel's in-stream cost by
// ablation -- 1 RoPE, 2 decode attention, 4 add-norm after O, 8 SiLU,
// 16 add-norm after down, 32/64/128/256 the QKV/O/gate-up/down GEMMs.
// Results are garbage with any bit set; never set in serving.
static int skip_mask() {
  static const int m = [] {
    const char* e = getenv("HS_SKIP");
    return e ? atoi(e) : 0;
  }();
  return m;
}

int hs_layer(hs_ctx* c, const hs_layer_desc* d) {
  HProf hp_layer(HP_LAYER);
  const int skip = skip_mask();
  const ModelCfg& m = c->m;
  const hs_rt_cfg& r = c->r;
  const MetaLayout L = layout_of(r);
  const int l = d->layer - 1;  // 0-based
  const int B = c->B;
  const bool last = d->layer == m.layers;
  const bool tp = c->tp_world > 1;  // row-parallel O / down: fused all-reduce
  if (l < 0 || l >= m.layers) return set_error(HS_E_CONFIG, "layer %d out of range", d->layer);
  const bool dev_merges = c->pg_on;  // merge decision taken on the device (piggyback.cu)
  if (dev_merges && c->fp32)
    return set_error(HS_E_CONFIG, "device-polled merges: bf16 datapath only");
  int C = d->n_carry, M = d->n_merge, R = d->n_restart;
  if (!dev_merges) {
    if (B + C > r.max_rows || B + M > r.max_rows || d->n_restart > M)
      return set_error(HS_E_CAPACITY, "layer rows exceed max_rows");
    for (int i = 0; i < C; ++i)
      if (d->carry_pos[i] < 0 || d->carry_pos[i] >= r.max_pos || d->carry_slot[i] < 0 ||
          d->carry_slot[i] >= r.max_slots)
        return set_error(HS_E_CONFIG, "carry row %d: slot %d / position %d out of range", i,
                         d->carry_slot[i], d->carry_pos[i]);
    for (int i = 0; i < M; ++i)
      if (d->merge_slot[i] < 0 || d->merge_slot[i] >= r.max_slots)
        return set_error(HS_E_CONFIG, "merge row %d: slot %d out of range", i, d->merge_slot[i]);
    for (int i = 0; i < d->n_restart; ++i)
      if (d->restart_idx[i] < 0 || d->restart_idx[i] >= M || d->restart_pos[i] < 0 ||
          d->restart_pos[i] >= r.max_pos)
        return set_error(HS_E_CONFIG, "restart row %d: index %d / position %d out of range", i,
                         d->restart_idx[i], d->restart_pos[i]);
  }
  int* dm = c->dm;
  cudaStream_t st = c->st;
  const int d_ = m.d, nqh = m.n_q * m.hd;
  Planes sp(1);
  ProfScope whole(c, 3, 0.0, 0.0);  // the layer's span on the device
  const int *carry_slot = nullptr, *carry_pos = nullptr, *merge_slot = nullptr,
            *restart_slot = nullptr, *restart_pos = nullptr, *logit_rows = nullptr,
            *logit_slots = nullptr, *merge_tag = nullptr;
  int NL = 0;
  if (dev_merges) {
    // the controller takes this layer's FIFO head-run from the completion
    // tags and writes the row lists (padding rows: slot -1); C / M / R are
    // the host bounds the launches are sized for
    LayerRows lr{};
    RC(pg_control(c, d->layer, &lr, &C, &M, &R));
    if (B + C > r.max_rows || B + M > r.max_rows)
      return set_error(HS_E_CAPACITY, "layer rows exceed max_rows (device-polled bounds)");
    carry_slot = lr.carry_slot, carry_pos = lr.carry_pos, merge_slot = lr.merge_slot;
    restart_slot = lr.restart_slot, restart_pos = lr.restart_pos, merge_tag = lr.merge_tag;
    logit_slots = lr.logit_slots;
    NL = last ? c->n_logit + M : 0;
    if (NL) {
      std::vector<int> lrows(NL);
      for (int i = 0; i < NL; ++i) lrows[i] = i < c->n_logit ? c->h_logit_rows[i] : B + (i - c->n_logit);
      Packer pk(c, nullptr, 0);
      if (static_cast<size_t>(NL) > c->layer_cap || !pk.reserve(NL))
        return set_error(HS_E_CAPACITY, "metadata staging overflow");
      logit_rows = pk.add(lrows.data(), NL);
    }
  } else {
    NL = last ? c->n_logit + M : 0;
    // one packed staging run: carry slots/pos, merge slots, restart slots/pos
    // and, at the last layer, the LM-head gather rows and their slots; the
    // kernels read it in place from pinned host memory (a few hundred bytes)
    Packer pk(c, nullptr, 0);
    const bool tagged = d->merge_tag != nullptr;
    const size_t total = 2 * static_cast<size_t>(C) + M + 2 * static_cast<size_t>(R) + 2 * NL +
                         (tagged ? M : 0);
    if (total > c->layer_cap) return set_error(HS_E_CAPACITY, "layer metadata too large");
    if (total && !pk.reserve(total)) return set_error(HS_E_CAPACITY, "metadata staging overflow");
    std::vector<int> rslot(R), lrows(NL), lslots(NL);
    for (int i = 0; i < R; ++i) rslot[i] = d->merge_slot[d->restart_idx[i]];
    for (int i = 0; i < NL; ++i) {
      const bool batch = i < c->n_logit;
      lrows[i] = batch ? c->h_logit_rows[i] : B + (i - c->n_logit);
      lslots[i] = batch ? c->h_logit_slots[i] : d->merge_slot[i - c->n_logit];
    }
    carry_slot = total ? pk.add(d->carry_slot, C) : nullptr;
    carry_pos = total ? pk.add(d->carry_pos, C) : nullptr;
    merge_slot = total ? pk.add(d->merge_slot, M) : nullptr;
    restart_slot = total ? pk.add(rslot.data(), R) : nullptr;
    restart_pos = total ? pk.add(d->restart_pos, R) : nullptr;
    logit_rows = total ? pk.add(lrows.data(), NL) : nullptr;
    logit_slots = total ? pk.add(lslots.data(), NL) : nullptr;
    merge_tag = tagged && M ? pk.add(d->merge_tag, M) : nullptr;
    if (total) {
      HProf hp(HP_PACK);
      RC(pk.flush(st));
    }
  }
  if (c->fp32)
    return layer_f32(c, d, LayerRows{carry_slot, carry_pos, merge_slot, restart_slot, restart_pos,
                                      logit_rows, logit_slots, merge_tag});
  if (l == 0) {
    // embed batch rows (+ injected chains: fresh token from last_token)
    RC(select_tokens(c->it_tok, c->it_slot, B, carry_slot, c->last_token, B + C, c->tok, st));
    RC(embed_gather(c->tok, B + C, c->w_embed, d_, c->h, st));
    // residual put for injections (reference _chain_qkv(req, 1), engine.py:997)
    RC(scatter_rows_f32(c->h + static_cast<size_t>(B) * d_, carry_slot, C, d_, c->resid, st));
    RC(rmsnorm_rows(c->h, B + C, d_, c->n_in[0], m.eps, c->xn.p, d_, st));
  }
  // QKV over batch + carry rows with RoPE, KV-page scatter and the piggyback
  // ship fused into the GEMM epilogue
  EpiParams ep = epi_base(c);
  bool gathered = false;  // host results already copied by the RoPE launch
  ep.layer = l;
  ep.row_pos = c->it_pos;
  ep.row_slot = c->it_slot;
  ep.n_batch = B;
  ep.carry_pos = carry_pos;
  ep.carry_slot = carry_slot;
  if (fuse_ok(c, B + C, m.qkv_n(), d_)) {
    RC(gemm_fused(c, c->m_qkv[l], c->xn, B + C, m.qkv_n(), d_, EPI_QKV, ep));
  } else {
    if (!(skip & 32)) RC(gemm(c, c->m_qkv[l], c->xn, B + C, m.qkv_n(), d_, &sp));
    // + merged rows: host attention results into the attention buffer
    RowCopy rc{c->result_d, nqh, merge_slot, M, c->attn.p + static_cast<size_t>(B) * nqh, nqh,
               nqh, merge_tag, c->tag_d, c->fault_d, d->layer};
    if (!(skip & 1))
      RC(qkv_rope_scatter(c->part, sp, B + C, m.n_q, m.n_kv, m.hd, c->rope_cos, c->rope_sin,
                          c->it_pos, c->it_slot, nullptr, B, carry_pos, carry_slot, c->qbuf, nqh,
                          c->kv_pool, c->geom, l, c->page_table, r.max_pages_per_req, c->ship_d,
                          m.qkv_n(), st, 1, rc));
    gathered = true;
  }
  // attention of batch rows (K1 with the K2 merge fused into its last CTA)
  {
  ProfScope pd(c, 1, c->dec_kv_tokens * 2.0 * m.n_kv * m.hd * 2.0 + 4.0 * c->D * nqh,
               4.0 * c->dec_kv_tokens * nqh);
  if (!(skip & 2))
  RC(decode_attention_fused(c->m_kv, c->geom, l, c->qbuf, nqh, m.n_q, c->page_table,
                            r.max_pages_per_req, reinterpret_cast<const DecodeChunk*>(c->it_chunks),
                            c->n_chunks, c->it_cbeg, c->o_part, c->lse_part, c->dec_counters,
                            c->attn.p, nqh, st, c->n_chunks == c->D));
  }
  {
  ProfScope pp(c, 2, c->pre_kv_tokens * 2.0 * m.n_kv * m.hd * 2.0, 4.0 * c->pre_units * nqh);
  RC(prefill_attention(c->m_kv, c->geom, l, c->qbuf, nqh, m.n_q, c->page_table,
                       r.max_pages_per_req, reinterpret_cast<const PrefillTile*>(c->it_tiles),
                       c->n_tiles, c->attn.p, nqh, st));
  }
  // merged rows: host attention result (+ completion check), when no RoPE
  // launch carried it
  if (!gathered && M > 0) {
    RowCopy rc{c->result_d, nqh, merge_slot, M, c->attn.p + static_cast<size_t>(B) * nqh, nqh,
               nqh, merge_tag, c->tag_d, c->fault_d, d->layer};
    RC(qkv_rope_scatter(nullptr, 1, 0, m.n_q, m.n_kv, m.hd, nullptr, nullptr, nullptr, nullptr,
                        nullptr, 0, nullptr, nullptr, nullptr, nqh, nullptr, c->geom, l, nullptr, 0,
                        nullptr, m.qkv_n(), st, 1, rc));
  }
  const int N = B + M;
  // Proj + ResidualAdd + RMSNorm (residual add fused into the GEMM when the
  // tiles have few K-segments)
  if (tp) {
    RC(gemm(c, c->m_o[l], c->attn, N, d_, nqh, &sp));
    RowIo io;
    io.src = c->resid;
    io.src_idx = M ? merge_slot : nullptr;
    io.src_from = B;
    RC(tp_add_norm(c->part, sp, N, d_, c->h, c->n_post[l], m.eps, c->xn2.p, d_, st, io, c->tp,
                   ++c->tp_epoch));
  } else if (fuse_ok(c, N, d_, nqh)) {
    RC(gather_rows_f32(c->resid, merge_slot, M, d_, c->h + static_cast<size_t>(B) * d_, st));
    RC(gemm_fused(c, c->m_o[l], c->attn, N, d_, nqh, EPI_RESID, ep));
    RC(rmsnorm_rows(c->h, N, d_, c->n_post[l], m.eps, c->xn2.p, d_, st));
  } else {
    if (!(skip & 64)) RC(gemm(c, c->m_o[l], c->attn, N, d_, nqh, &sp));
    // merged rows start from their stored residual (the residual get)
    RowIo io;
    io.src = c->resid;
    io.src_idx = M ? merge_slot : nullptr;
    io.src_from = B;
    if (!(skip & 4))
      RC(residual_add_norm(c->part, sp, N, d_, c->h, c->n_post[l], m.eps, c->xn2.p, d_, st, io));
  }
  // MLP: SiLU*up, down + ResidualAdd, then the next layer's input norm (or the
  // final norm)
  if (!tp && fuse_ok(c, N, 2 * m.ffn, d_)) {
    RC(gemm_fused(c, c->m_gu[l], c->xn2, N, 2 * m.ffn, d_, EPI_SILU, ep));
  } else {
    if (!(skip & 128)) RC(gemm(c, c->m_gu[l], c->xn2, N, 2 * m.ffn, d_, &sp));
    if (!(skip & 8)) RC(silu_mul(c->part, sp, N, m.ffn, c->act.p, m.ffn, st, 1));
  }
  const float* w_next = last ? c->w_final : c->n_in[l + 1];
  bool put = false;  // residual put for the chains' next layer (engine.py:985)
  if (tp) {
    RC(gemm(c, c->m_down[l], c->act, N, d_, m.ffn, &sp));
    RowIo io;
    if (!last && M) {
      io.put = c->resid;
      io.put_idx = merge_slot;
      io.put_from = B;
      put = true;
    }
    RC(tp_add_norm(c->part, sp, N, d_, c->h, w_next, m.eps, c->xn.p, d_, st, io, c->tp,
                   ++c->tp_epoch));
  } else if (fuse_ok(c, N, d_, m.ffn)) {
    RC(gemm_fused(c, c->m_down[l], c->act, N, d_, m.ffn, EPI_RESID, ep));
    RC(rmsnorm_rows(c->h, N, d_, w_next, m.eps, c->xn.p, d_, st));
  } else {
    if (!(skip & 256)) RC(gemm(c, c->m_down[l], c->act, N, d_, m.ffn, &sp));
    RowIo io;
    if (!last && M) {
      io.put = c->resid;
      io.put_idx = merge_slot;
      io.put_from = B;
      put = true;
    }
    if (!(skip & 16))
      RC(residual_add_norm(c->part, sp, N, d_, c->h, w_next, m.eps, c->xn.p, d_, st, io));
  }
  if (!last) {
    if (!put)
      RC(scatter_rows_f32(c->h + static_cast<size_t>(B) * d_, merge_slot, M, d_, c->resid, st));
    return HS_OK;
  }
  // ---- final layer: LM head + greedy token for decode / finishing-prefill
  // rows and for every chain completing a token (engine.py:1005-1013, 1024-1047)
  RC(gather_rows_bf16(c->xn.p, d_, logit_rows, NL, d_, c->lin.p, d_, st));
  RC(gemm(c, c->m_lm, c->lin, NL, m.vocab, d_, &sp));
  RC(argmax_rows(c->part, sp, NL, m.vocab, c->tok_out, c->keep_logits ? c->logits : nullptr, st));
  RC(scatter_tokens(c->tok_out, logit_slots, NL, c->last_token, st));
  c->n_tok_out = NL;
  c->merges_L = M;
  // chains continuing with the next token: embed, residual put, QKV(1), ship
  if (R > 0) {
    RC(select_tokens(nullptr, nullptr, 0, restart_slot, c->last_token, R, c->tok, st));
    RC(embed_gather(c->tok, R, c->w_embed, d_, c->hr, st));
    RC(scatter_rows_f32(c->hr, restart_slot, R, d_, c->resid, st));
    RC(rmsnorm_rows(c->hr, R, d_, c->n_in[0], m.eps, c->xr.p, d_, st));
    EpiParams er = epi_base(c);
    er.layer = 0;
    er.n_batch = 0;
    er.carry_pos = restart_pos;
    er.carry_slot = restart_slot;
    if (fuse_ok(c, R, m.qkv_n(), d_)) {
      RC(gemm_fused(c, c->m_qkv[0], c->xr, R, m.qkv_n(), d_, EPI_QKV, er));
    } else {
      RC(gemm(c, c->m_qkv[0], c->xr, R, m.qkv_n(), d_, &sp));
      RC(qkv_rope_scatter(c->part, sp, R, m.n_q, m.n_kv, m.hd, c->rope_cos, c->rope_sin, nullptr,
                          nullptr, nullptr, 0, restart_pos, restart_slot, c->qbuf, nqh,
                          c->kv_pool, c->geom, 0, c->page_table, r.max_pages_per_req, c->ship_d,
                          m.qkv_n(), st, 1));
    }
  }
  // device-polled merges: the work items shipped by this layer (carries and
  // restarts) become visible to the CPU pool once their rows have landed
  if (dev_merges) RC(pg_publish(c));
  return HS_OK;
}

// ---- tensor parallelism ---------------------------------------------------
static int tp_alloc(hs_ctx* c) {
  if (c->tp_xbuf) return HS_OK;
  const size_t R = c->r.max_rows, d = c->m.d;
  c->tp.xbuf_par = R * d;
  c->tp.flag_par = R * 8;
  CK(cudaMalloc(&c->tp_xbuf, 2 * c->tp.xbuf_par * sizeof(float)));
  CK(cudaMalloc(&c->tp_flag, 2 * c->tp.flag_par * sizeof(unsigned)));
  CK(cudaMemset(c->tp_flag, 0, 2 * c->tp.flag_par * sizeof(unsigned)));
  CK(cudaDeviceSynchronize());
  return HS_OK;
}

int hs_tp_export(hs_ctx* c, void* handles) {
  RC(tp_alloc(c));
  cudaIpcMemHandle_t hx, hf;
  CK(cudaIpcGetMemHandle(&hx, c->tp_xbuf));
  CK(cudaIpcGetMemHandle(&hf, c->tp_flag));
  std::memcpy(handles, &hx, sizeof(hx));
  std::memcpy(static_cast<char*>(handles) + HS_TP_HANDLE_BYTES / 2, &hf, sizeof(hf));
  return HS_OK;
}

int hs_tp_open(hs_ctx* c, int rank, int world, const void* all_handles) {
  if (c->fp32) return set_error(HS_E_CONFIG, "tensor parallelism runs the bf16 datapath only");
  if (world < 1 || world > kMaxTp || rank < 0 || rank >= world)
    return set_error(HS_E_CONFIG, "tensor-parallel rank %d of %d out of range", rank, world);
  RC(tp_alloc(c));
  for (int p = 0; p < world; ++p) {
    if (p == rank) {
      c->tp.xbuf[p] = c->tp_xbuf;
      c->tp.flag[p] = c->tp_flag;
      continue;
    }
    const char* h = static_cast<const char*>(all_handles) + static_cast<size_t>(p) * HS_TP_HANDLE_BYTES;
    cudaIpcMemHandle_t hx, hf;
    std::memcpy(&hx, h, sizeof(hx));
    std::memcpy(&hf, h + HS_TP_HANDLE_BYTES / 2, sizeof(hf));
    void *px = nullptr, *pf = nullptr;
    CK(cudaIpcOpenMemHandle(&px, hx, cudaIpcMemLazyEnablePeerAccess));
    CK(cudaIpcOpenMemHandle(&pf, hf, cudaIpcMemLazyEnablePeerAccess));
    c->tp_opened.push_back(px);
    c->tp_opened.push_back(pf);
    c->tp.xbuf[p] = static_cast<float*>(px);
    c->tp.flag[p] = static_cast<unsigned*>(pf);
  }
  c->tp.world = world;
  c->tp.me = rank;
  c->tp_world = world;
  c->tp_rank = rank;
  return HS_OK;
}

// Count-returning entry points (hs_iter_end, hs_iter_poll, hs_mark,
// hs_timer, hs_swap_done) report errors as the negated status code.
int hs_iter_end(hs_ctx* c, int* tokens_out, int n) {
  const int rc = [&]() -> int {
    if (n < c->n_tok_out)
      return set_error(HS_E_CONFIG, "token buffer too small (%d < %d)", n, c->n_tok_out);
    if (c->n_tok_out > 0)
      CK(cudaMemcpyAsync(c->tokens_pinned, c->tok_out, c->n_tok_out * sizeof(int),
                         cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    RC(prof_collect(c));
    RC(check_device_faults(c));
    if (c->n_tok_out > 0) std::memcpy(tokens_out, c->tokens_pinned, c->n_tok_out * sizeof(int));
    return HS_OK;
  }();
  return rc ? -rc : c->n_tok_out;
}

int hs_anchor(hs_ctx* c) {
  CK(cudaEventRecord(c->anchor, c->st));
  CK(cudaEventSynchronize(c->anchor));
  return HS_OK;
}

int hs_iter_end_async(hs_ctx* c, int* ticket) {
  const int id = c->next_iter;
  const int slot = id % hs_ctx::kIterRing;
  if (id >= hs_ctx::kIterRing) {  // the ring slot must have been consumed
    const cudaError_t e = cudaEventQuery(c->iter_ev[slot]);
    if (e == cudaErrorNotReady) CK(cudaEventSynchronize(c->iter_ev[slot]));
  }
  int* dst = c->tok_ring + static_cast<size_t>(slot) * 2 * c->r.max_rows;
  if (c->n_tok_out > 0)
    CK(cudaMemcpyAsync(dst, c->tok_out, c->n_tok_out * sizeof(int), cudaMemcpyDeviceToHost,
                       c->st));
  if (c->keep_logits && c->logit_ring && c->n_tok_out > 0)
    CK(cudaMemcpyAsync(c->logit_ring + slot * static_cast<size_t>(2 * c->r.max_rows) * c->m.vocab,
                       c->logits, sizeof(float) * c->n_tok_out * c->m.vocab,
                       cudaMemcpyDeviceToHost, c->st));
  CK(cudaEventRecord(c->iter_ev[slot], c->st));
  c->iter_n[slot] = c->n_tok_out;
  *ticket = id;
  c->next_iter = id + 1;
  return HS_OK;
}

// 1 = done (tokens copied, *done_ms = completion time after the anchor), 0 = running
int hs_iter_poll(hs_ctx* c, int ticket, int* tokens_out, int n, double* done_ms) {
  int ready = 0;
  const int rc = [&]() -> int {
    if (ticket < c->next_iter - hs_ctx::kIterRing || ticket >= c->next_iter)
      return set_error(HS_E_CONFIG, "iteration ticket %d out of window", ticket);
    const int slot = ticket % hs_ctx::kIterRing;
    const cudaError_t e = cudaEventQuery(c->iter_ev[slot]);
    if (e == cudaErrorNotReady) return HS_OK;
    if (e != cudaSuccess) return set_error(HS_E_CUDA, "iteration: %s", cudaGetErrorString(e));
    if (n < c->iter_n[slot]) return set_error(HS_E_CONFIG, "token buffer too small");
    RC(check_device_faults(c));
    std::memcpy(tokens_out, c->tok_ring + static_cast<size_t>(slot) * 2 * c->r.max_rows,
                c->iter_n[slot] * sizeof(int));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->anchor, c->iter_ev[slot]));
    *done_ms = ms;
    ready = 1;
    return HS_OK;
  }();
  return rc ? -rc : ready;
}

int hs_iter_ntokens(hs_ctx* c, int ticket) {
  return c->iter_n[ticket % hs_ctx::kIterRing];
}

int hs_cpu_attend(hs_ctx* c, const int* slots, const int* layers, const int* ctxs, int n) {
  CK(cudaStreamSynchronize(c->st));  // the shipped q/k/v rows have landed
  const ModelCfg& m = c->m;
  for (int i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= c->r.max_slots || !c->regions[slots[i]].used)
      return set_error(HS_E_INTEGRITY, "work item for slot %d without host KV", slots[i]);
    if (ctxs[i] >= c->regions[slots[i]].cap)
      return set_error(HS_E_CAPACITY, "host KV of slot %d full (ctx %d)", slots[i], ctxs[i]);
    if (layers[i] < 1 || layers[i] > m.layers)
      return set_error(HS_E_CONFIG, "work item layer %d out of range", layers[i]);
    if (ctxs[i] < 0 || ctxs[i] >= c->r.max_pos)
      return set_error(HS_E_CONFIG, "work item ctx %d outside [0, max_pos)", ctxs[i]);
  }
  for (int i = 0; i < n; ++i) retract_tag(c, slots[i]);
  // items of slots placed on remote hosts go to their relays first and are
  // serviced there while the local pool runs
  std::vector<int> local;
  std::vector<char> used_host(c->remotes.size(), 0);
  for (int i = 0; i < n; ++i) {
    const int h = slot_host_of(c, slots[i]);
    if (h <= 0) {
      local.push_back(i);
      continue;
    }
    used_host[h] = 1;
    remote_attend(c->remotes[h], slots[i], layers[i], ctxs[i], nullptr, ship_row(c, slots[i]),
                  result_row(c, slots[i]), nullptr, nullptr);
  }
  const int nl = static_cast<int>(local.size());
  c->pool->parallel_for(nl * m.n_kv, [&](int task) {
    const int i = local[task / m.n_kv], h = task % m.n_kv;
    const int s = slots[i];
    cpu_attend_head(m, ship_row(c, s), host_region(c, s), c->regions[s].cap, layers[i] - 1,
                    ctxs[i], h, result_row(c, s), nullptr);
  });
  for (size_t h = 1; h < used_host.size(); ++h)
    if (used_host[h] && !remote_quiesce(c->remotes[h]))
      return set_error(HS_E_CUDA, "remote CPU host %zu: connection failed", h);
  for (int i = 0; i < n; ++i) publish_tag(c, slots[i], ctxs[i], layers[i]);
  return HS_OK;
}

int hs_mark(hs_ctx* c) {
  const int id = c->next_mark++;
  const cudaError_t e = cudaEventRecord(c->marks[id % c->marks.size()], c->st);
  return e == cudaSuccess ? id : -set_error(HS_E_CUDA, "hs_mark: %s", cudaGetErrorString(e));
}

int hs_wait_mark(hs_ctx* c, int id) {
  if (id < 0 || id < c->next_mark - static_cast<int>(c->marks.size())) return HS_OK;
  CK(cudaEventSynchronize(c->marks[id % c->marks.size()]));
  return HS_OK;
}

int hs_timer(hs_ctx* c) {
  const int id = c->next_timer++;
  const cudaError_t e = cudaEventRecord(c->timers[id % c->timers.size()], c->st);
  return e == cudaSuccess ? id : -set_error(HS_E_CUDA, "hs_timer: %s", cudaGetErrorString(e));
}

int hs_timer_elapsed(hs_ctx* c, int a, int b, float* ms) {
  const int n = static_cast<int>(c->timers.size());
  if (a < c->next_timer - n || b < c->next_timer - n)
    return set_error(HS_E_CONFIG, "timer %d/%d recycled", a, b);
  CK(cudaEventSynchronize(c->timers[b % n]));
  CK(cudaEventElapsedTime(ms, c->timers[a % n], c->timers[b % n]));
  return HS_OK;
}

int hs_profile(hs_ctx* c, int on) {
  c->prof_on = on != 0;
  return HS_OK;
}

int hs_profile_read(hs_ctx* c, double* stats, int reset) {
  RC(prof_collect(c));
  std::memcpy(stats, c->prof_stats, sizeof(c->prof_stats));
  if (reset) std::memset(c->prof_stats, 0, sizeof(c->prof_stats));
  return HS_OK;
}

int hs_probe_dense(hs_ctx* c, int n, int reps, float* us) {
  const ModelCfg& m = c->m;
  if (n < 1 || n > c->r.max_rows) return set_error(HS_E_CONFIG, "probe rows out of range");
  const int d_ = m.d, nqh = m.n_q * m.hd;
  return time_reps(c, reps, [&]() -> int {
    Planes sp;
    EpiParams ep = epi_base(c);
    RC(gemm(c, c->m_qkv[0], c->xn, n, m.qkv_n(), d_, &sp));  // (+ a RoPE epilogue in the layer)
    RC(gemm_fused(c, c->m_o[0], c->attn, n, d_, nqh, EPI_RESID, ep));
    RC(rmsnorm_rows(c->h, n, d_, c->n_post[0], m.eps, c->xn2.p, d_, c->st));
    RC(gemm_fused(c, c->m_gu[0], c->xn2, n, 2 * m.ffn, d_, EPI_SILU, ep));
    RC(gemm_fused(c, c->m_down[0], c->act, n, d_, m.ffn, EPI_RESID, ep));
    RC(rmsnorm_rows(c->h, n, d_, c->n_in[0], m.eps, c->xn.p, d_, c->st));
    return HS_OK;
  }, us);
}

// The four Dense GEMMs of every layer at n rows, back to back on the step's
// stream (PDL chain intact, weights streamed from HBM: 16 GB per pass >> L2)
// between one pair of events, on the live activation buffers; results go to
// the split-K scratch only, so a running serving context is not disturbed.
// *us = median time per launch, *bytes = algorithmic bytes per launch.
int hs_probe_gemm_stream(hs_ctx* c, int n, int reps, float* us, double* bytes) {
  const ModelCfg& m = c->m;
  if (n < 1 || n > c->r.max_rows) return set_error(HS_E_CONFIG, "probe rows out of range");
  const int d_ = m.d, nqh = m.n_q * m.hd;
  const double per_layer = 2.0 * (static_cast<double>(m.qkv_n()) * d_ + static_cast<double>(d_) * nqh +
                                  2.0 * m.ffn * d_ + static_cast<double>(d_) * m.ffn) +
                           2.0 * n * (d_ + m.qkv_n() + nqh + d_ + d_ + 2.0 * m.ffn + m.ffn + d_);
  int err = time_reps(c, reps, [&]() -> int {
    Planes s;
    for (int l = 0; l < m.layers; ++l) {
      RC(gemm(c, c->m_qkv[l], c->xn, n, m.qkv_n(), d_, &s));
      RC(gemm(c, c->m_o[l], c->attn, n, d_, nqh, &s));
      RC(gemm(c, c->m_gu[l], c->xn2, n, 2 * m.ffn, d_, &s));
      RC(gemm(c, c->m_down[l], c->act, n, d_, m.ffn, &s));
    }
    return HS_OK;
  }, us);
  *us /= 4 * m.layers;
  *bytes = per_layer / 4;
  return err;
}

// PCIe rate of the piggyback exchange: `rows` items moved between HBM and the
// pinned host mailboxes, median over reps (events on the step stream).
//   dir 0: SM stores into the mapped ship mailbox (q|k|v rows, the D2H of
//          the step's RoPE/ship launch);  dir 1: SM loads from the mapped
//          result mailbox (the H2D gather of host attention results);
//   dir 2 / 3: the same bytes by the copy engine (cudaMemcpyAsync D2H / H2D).
int hs_probe_pcie(hs_ctx* c, int dir, int rows, int reps, float* us, double* bytes) {
  const ModelCfg& m = c->m;
  if (rows < 1 || rows > c->r.max_slots || rows > static_cast<int>(c->layer_cap))
    return set_error(HS_E_CONFIG, "probe rows out of range");
  const int qkv = m.qkv_n(), nqh = m.n_q * m.hd;
  std::vector<int> ident(rows);
  for (int i = 0; i < rows; ++i) ident[i] = i;
  RC(h2d(c, c->dm_layer, ident.data(), rows * sizeof(int)));
  bf16* scratch = reinterpret_cast<bf16*>(c->part);
  const int w = (dir == 0 || dir == 2) ? qkv : nqh;
  *bytes = 2.0 * rows * w;
  return time_reps(c, reps, [&]() -> int {
    switch (dir) {
      case 0: return gather_rows_bf16(scratch, w, c->dm_layer, rows, w, c->ship_d, w, c->st);
      case 1: return gather_rows_bf16(c->result_d, w, c->dm_layer, rows, w, scratch, w, c->st);
      case 2:
        CK(cudaMemcpyAsync(c->ship_h, scratch, static_cast<size_t>(*bytes), cudaMemcpyDeviceToHost, c->st));
        return HS_OK;
      default:
        CK(cudaMemcpyAsync(scratch, c->result_h, static_cast<size_t>(*bytes), cudaMemcpyHostToDevice, c->st));
        return HS_OK;
    }
  }, us);
}

// The dense part of `layers` consecutive layers exactly as hs_layer issues it
// on the unfused path (QKV GEMM + RoPE/KV/ship, O GEMM + residual-add-norm,
// gate-up GEMM + SiLU, down GEMM + residual-add-norm), back to back with no
// events in between.  `mode` selects the ops (bit list below); the per-layer
// time of each subset shows how much of the layer is launch/ramp overhead
// rather than streaming.
int hs_probe_dense_mode(hs_ctx* c, int n, int mode, int layers, int reps, float* us) {
  const ModelCfg& m = c->m;
  if (n < 1 || n > c->r.max_rows) return set_error(HS_E_CONFIG, "probe rows out of range");
  if (layers < 1 || layers > m.layers) return set_error(HS_E_CONFIG, "probe layers out of range");
  const int d_ = m.d, nqh = m.n_q * m.hd;
  // op bits: 0 QKV GEMM, 1 RoPE/KV/ship, 2 O GEMM, 3 residual-add-norm,
  // 4 gate-up GEMM, 5 SiLU, 6 down GEMM, 7 residual-add-norm
  auto on = [mode](int b) { return (mode >> b) & 1; };
  // every row a carry row of slot 0 at position 0 (page-table row 0 valid)
  RC(probe_pages(c, 1, 64));
  CK(cudaMemsetAsync(c->dm_layer, 0, 2 * static_cast<size_t>(n) * sizeof(int), c->st));
  const int* cslot = c->dm_layer;
  const int* cpos = c->dm_layer + n;
  auto planes = [&](int n_out, int k) {
    return std::max(1, gemm_pick_splits(n_out, k, n, gemm_pick_bn(n), 16));
  };
  const int s_qkv = planes(m.qkv_n(), d_), s_o = planes(d_, nqh), s_gu = planes(2 * m.ffn, d_),
            s_dn = planes(d_, m.ffn);
  int err = time_reps(c, reps, [&]() -> int {
    Planes s, pq(s_qkv), po(s_o), pg(s_gu), pd(s_dn);
    for (int l = 0; l < layers; ++l) {
      if (on(0)) RC(gemm(c, c->m_qkv[l], c->xn, n, m.qkv_n(), d_, &pq));
      if (on(1))
        RC(qkv_rope_scatter(c->part, pq, n, m.n_q, m.n_kv, m.hd, c->rope_cos, c->rope_sin,
                            nullptr, nullptr, nullptr, 0, cpos, cslot, c->qbuf, nqh, c->kv_pool,
                            c->geom, l, c->page_table, c->r.max_pages_per_req, c->ship_d,
                            m.qkv_n(), c->st, 1));
      if (on(2)) RC(gemm(c, c->m_o[l], c->attn, n, d_, nqh, &po));
      if (on(3))
        RC(residual_add_norm(c->part, po, n, d_, c->h, c->n_post[l], m.eps, c->xn2.p, d_, c->st));
      if (on(4)) RC(gemm(c, c->m_gu[l], c->xn2, n, 2 * m.ffn, d_, &pg));
      if (on(5)) RC(silu_mul(c->part, pg, n, m.ffn, c->act.p, m.ffn, c->st, 1));
      if (on(6)) RC(gemm(c, c->m_down[l], c->act, n, d_, m.ffn, &pd));
      if (on(7))
        RC(residual_add_norm(c->part, pd, n, d_, c->h, c->n_in[l], m.eps, c->xn.p, d_, c->st));
    }
    return HS_OK;
  }, us);
  *us /= layers;
  return err;
}

// one GEMM of layer 0: which 0=qkv 1=o 2=gate_up 3=down; fused 0=planes 1=fused epilogue
int hs_probe_gemm(hs_ctx* c, int which, int n, int fused, int reps, float* us) {
  const ModelCfg& m = c->m;
  if (n < 1 || n > c->r.max_rows) return set_error(HS_E_CONFIG, "probe rows out of range");
  const int d_ = m.d, nqh = m.n_q * m.hd;
  EpiParams ep = epi_base(c);
  // QKV epilogue as a pure ship of n carry rows (slot 0, position 0)
  CK(cudaMemsetAsync(c->dm_layer, 0, 2 * static_cast<size_t>(n) * sizeof(int), c->st));
  ep.n_batch = 0;
  ep.carry_slot = c->dm_layer;
  ep.carry_pos = c->dm_layer + n;
  return time_reps(c, reps, [&]() -> int {
    Planes sp;
    switch (which) {
      case 0:
        return fused ? gemm_fused(c, c->m_qkv[0], c->xn, n, m.qkv_n(), d_, EPI_QKV, ep)
                     : gemm(c, c->m_qkv[0], c->xn, n, m.qkv_n(), d_, &sp);
      case 1:
        return fused ? gemm_fused(c, c->m_o[0], c->attn, n, d_, nqh, EPI_RESID, ep)
                     : gemm(c, c->m_o[0], c->attn, n, d_, nqh, &sp);
      case 2:
        return fused ? gemm_fused(c, c->m_gu[0], c->xn2, n, 2 * m.ffn, d_, EPI_SILU, ep)
                     : gemm(c, c->m_gu[0], c->xn2, n, 2 * m.ffn, d_, &sp);
      default:
        return fused ? gemm_fused(c, c->m_down[0], c->act, n, d_, m.ffn, EPI_RESID, ep)
                     : gemm(c, c->m_down[0], c->act, n, d_, m.ffn, &sp);
    }
  }, us);
}

int hs_probe_decode(hs_ctx* c, int g, int ctx_len, int reps, float* us) {
  const ModelCfg& m = c->m;
  if (g < 1 || g > c->r.max_rows) return set_error(HS_E_CONFIG, "probe rows out of range");
  RC(probe_pages(c, g, ctx_len));
  const int per = (ctx_len + kPageTokens - 1) / kPageTokens;
  // the runtime's chunking (runtime.decode_chunks): smallest chunk keeping
  // one wave of 296 CTAs, rows split into near-equal chunks
  int chunk = std::max(1, std::min(64, (g * per * m.n_kv + 295) / 296));
  while (chunk < 64 && m.n_kv * g * ((per + chunk - 1) / chunk) > 296) ++chunk;
  if (g * per * m.n_kv <= 2048 && per <= 16) chunk = std::max(chunk, per);  // small: rows unsplit
  const int k = std::max(1, (per + chunk - 1) / chunk);
  std::vector<int> ch, beg{0};
  for (int r = 0; r < g; ++r) {
    for (int i = 0; i < k; ++i) ch.insert(ch.end(), {r, r, i * per / k, (i + 1) * per / k, ctx_len});
    beg.push_back(static_cast<int>(ch.size() / 5));
  }
  if (static_cast<int>(ch.size() / 5) > c->r.max_chunks)
    return set_error(HS_E_CAPACITY, "probe exceeds max_chunks");
  const MetaLayout L = layout_of(c->r);
  RC(h2d(c, c->dm + L.chunks, ch.data(), ch.size() * 4));
  RC(h2d(c, c->dm + L.row_chunk_begin, beg.data(), beg.size() * 4));
  const int nch = static_cast<int>(ch.size() / 5), nqh = m.n_q * m.hd;
  return time_reps(c, reps, [&]() -> int {
    RC(decode_attention(c->m_kv, c->geom, 0, c->qbuf, nqh, m.n_q, c->page_table,
                        c->r.max_pages_per_req,
                        reinterpret_cast<const DecodeChunk*>(c->dm + L.chunks), nch, c->o_part,
                        c->lse_part, c->st));
    RC(decode_combine(c->o_part, c->lse_part, c->dm + L.row_chunk_begin, g, m.n_q, m.n_kv, m.hd,
                      c->attn.p, nqh, nullptr, c->st));
    return HS_OK;
  }, us);
}

int hs_probe_prefill(hs_ctx* c, int q, int done, int reps, float* us) {
  const ModelCfg& m = c->m;
  if (q < 1 || q > c->r.max_rows) return set_error(HS_E_CONFIG, "probe rows out of range");
  RC(probe_pages(c, 1, done + q));
  std::vector<int> tiles;
  for (int j = 0; j < q; j += 64) tiles.insert(tiles.end(), {0, j, done + j, std::min(64, q - j)});
  const MetaLayout L = layout_of(c->r);
  RC(h2d(c, c->dm + L.tiles, tiles.data(), tiles.size() * 4));
  const int nt = static_cast<int>(tiles.size() / 4), nqh = m.n_q * m.hd;
  return time_reps(c, reps, [&]() -> int {
    return prefill_attention(c->m_kv, c->geom, 0, c->qbuf, nqh, m.n_q, c->page_table,
                             c->r.max_pages_per_req,
                             reinterpret_cast<const PrefillTile*>(c->dm + L.tiles), nt, c->attn.p,
                             nqh, c->st);
  }, us);
}

int hs_swap_out_async(hs_ctx* c, int slot, int tokens, int* ticket) {
  return swap_async(c, slot, tokens, true, ticket);
}

int hs_swap_in_async(hs_ctx* c, int slot, int tokens, int* ticket) {
  return swap_async(c, slot, tokens, false, ticket);
}

int hs_swap_done(hs_ctx* c, int ticket) {
  auto it = c->swap_ev.find(ticket);
  if (it == c->swap_ev.end()) return -set_error(HS_E_CONFIG, "unknown swap ticket %d", ticket);
  const cudaError_t e = cudaEventQuery(it->second);
  if (e == cudaErrorNotReady) return 0;
  if (e != cudaSuccess) return -set_error(HS_E_CUDA, "swap: %s", cudaGetErrorString(e));
  cudaEventDestroy(it->second);
  c->swap_ev.erase(it);
  return 1;
}

int hs_cpu_submit(hs_ctx* c, const int* slots, const int* layers, const int* ctxs, int n) {
  RC(ensure_cpu_service(c));
  for (int i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= c->r.max_slots || !c->regions[slots[i]].used)
      return set_error(HS_E_INTEGRITY, "work item for slot %d without host KV", slots[i]);
    if (ctxs[i] >= c->regions[slots[i]].cap)
      return set_error(HS_E_CAPACITY, "host KV of slot %d full (ctx %d)", slots[i], ctxs[i]);
    if (layers[i] < 1 || layers[i] > c->m.layers)
      return set_error(HS_E_CONFIG, "work item layer %d out of range", layers[i]);
    if (ctxs[i] < 0 || ctxs[i] >= c->r.max_pos)
      return set_error(HS_E_CONFIG, "work item ctx %d outside [0, max_pos)", ctxs[i]);
  }
  return cpu_service_submit(c->cpu, c->st, slots, layers, ctxs, n);
}

int hs_cpu_poll(hs_ctx* c, int* slots, int* layers, double* t_done, int max) {
  if (!c->cpu) return 0;
  return cpu_service_poll(c->cpu, slots, layers, t_done, max);
}

int hs_cpu_in_flight(hs_ctx* c) { return c->cpu ? cpu_service_in_flight(c->cpu) : 0; }

double hs_cpu_busy_seconds(hs_ctx* c) { return c->cpu ? cpu_service_busy(c->cpu) : 0.0; }

double hs_wall_seconds(void) { return wall_seconds(); }

int hs_cpu_host_connect(hs_ctx* c, int host, const char* addr, int port) {
  if (host < 1 || host > 4096 || !addr) return set_error(HS_E_CONFIG, "remote host id %d", host);
  if (static_cast<int>(c->remotes.size()) <= host) c->remotes.resize(host + 1, nullptr);
  if (c->remotes[host]) return set_error(HS_E_CONFIG, "remote host %d already connected", host);
  if (!c->slot_host) {
    c->slot_host.reset(new std::atomic<int>[c->r.max_slots]);
    for (int s = 0; s < c->r.max_slots; ++s) c->slot_host[s].store(0);
  }
  RC(ensure_cpu_service(c));
  RemoteHost* r = remote_connect(c->m, addr, port);
  if (!r) return HS_E_CONFIG;  // remote_connect set the message
  c->remotes[host] = r;
  return HS_OK;
}

int hs_cpu_place(hs_ctx* c, int slot, int host, int tokens) {
  if (slot < 0 || slot >= c->r.max_slots) return set_error(HS_E_CONFIG, "slot out of range");
  if (host < 0 || (host > 0 && (host >= static_cast<int>(c->remotes.size()) || !c->remotes[host])))
    return set_error(HS_E_CONFIG, "CPU host %d is not connected to this replica", host);
  HostRegion& hr = c->regions[slot];
  if (!hr.used) return set_error(HS_E_INTEGRITY, "slot %d has no host KV region", slot);
  if (tokens < 0 || tokens > hr.cap)
    return set_error(HS_E_CAPACITY, "placement of %d tokens exceeds the region", tokens);
  const int cur = slot_host_of(c, slot);
  if (cur == host) return HS_OK;
  if (cur > 0) {  // back from a remote host: its KV (with every appended token) into the region
    const bool ok = remote_get(c->remotes[cur], slot, tokens, host_region(c, slot), hr.cap);
    remote_free(c->remotes[cur], slot);
    c->slot_host[slot].store(0, std::memory_order_release);
    if (!ok) return set_error(HS_E_CUDA, "remote CPU host %d: connection failed", cur);
  }
  if (host > 0) {
    remote_put(c->remotes[host], slot, tokens, host_region(c, slot), hr.cap);
    c->slot_host[slot].store(host, std::memory_order_release);
  }
  return HS_OK;
}

int hs_cpu_fetch_async(hs_ctx* c, int slot, int tokens) {
  if (slot < 0 || slot >= c->r.max_slots) return set_error(HS_E_CONFIG, "slot out of range");
  HostRegion& hr = c->regions[slot];
  if (!hr.used) return set_error(HS_E_INTEGRITY, "slot %d has no host KV region", slot);
  if (tokens < 0 || tokens > hr.cap)
    return set_error(HS_E_CAPACITY, "fetch of %d tokens exceeds the region", tokens);
  const int cur = slot_host_of(c, slot);
  if (cur <= 0) return set_error(HS_E_CONFIG, "slot %d is not on a remote host", slot);
  if (c->fetches.count(slot)) return set_error(HS_E_CONFIG, "slot %d: fetch in flight", slot);
  auto flag = std::make_shared<std::atomic<int>>(0);
  remote_get_async(c->remotes[cur], slot, tokens, host_region(c, slot), hr.cap, flag);
  remote_free(c->remotes[cur], slot);
  c->fetches[slot] = {cur, flag};
  return HS_OK;
}

int hs_cpu_fetch_done(hs_ctx* c, int slot) {
  auto it = c->fetches.find(slot);
  if (it == c->fetches.end()) return -set_error(HS_E_CONFIG, "slot %d: no fetch in flight", slot);
  if (it->second.second->load(std::memory_order_acquire)) {
    c->slot_host[slot].store(0, std::memory_order_release);
    c->fetches.erase(it);
    return 1;
  }
  if (remote_failed(c->remotes[it->second.first]))
    return -set_error(HS_E_CUDA, "remote CPU host %d: connection failed", it->second.first);
  return 0;
}

int hs_cpu_remote_stats(hs_ctx* c, int host, int64_t* out) {
  if (host < 1 || host >= static_cast<int>(c->remotes.size()) || !c->remotes[host])
    return set_error(HS_E_CONFIG, "CPU host %d is not connected", host);
  std::memcpy(out, remote_stats(c->remotes[host]), 4 * sizeof(int64_t));
  return HS_OK;
}

int hs_sync(hs_ctx* c) {
  CK(cudaStreamSynchronize(c->st));
  if (c->copy_st) CK(cudaStreamSynchronize(c->copy_st));
  return HS_OK;
}

int hs_read_ship(hs_ctx* c, int slot, void* host, size_t bytes) {
  CK(cudaStreamSynchronize(c->st));
  if (slot < 0 || slot >= c->r.max_slots || bytes != static_cast<size_t>(c->m.qkv_n()) * c->kv_elem)
    return set_error(HS_E_CONFIG, "ship row: slot %d / %zu bytes", slot, bytes);
  std::memcpy(host, ship_row(c, slot), bytes);
  return HS_OK;
}

int hs_read_result(hs_ctx* c, int slot, void* host, size_t bytes) {
  CK(cudaStreamSynchronize(c->st));
  if (slot < 0 || slot >= c->r.max_slots ||
      bytes != static_cast<size_t>(c->m.n_q) * c->m.hd * c->kv_elem)
    return set_error(HS_E_CONFIG, "result row: slot %d / %zu bytes", slot, bytes);
  std::memcpy(host, result_row(c, slot), bytes);
  return HS_OK;
}

int hs_read_residual(hs_ctx* c, int slot, float* host) {
  CK(cudaStreamSynchronize(c->st));
  CK(cudaMemcpy(host, c->resid + static_cast<size_t>(slot) * c->m.d, c->m.d * 4,
                cudaMemcpyDeviceToHost));
  return HS_OK;
}

}  // extern "C"
