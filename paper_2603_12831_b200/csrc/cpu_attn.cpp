// C1: BE decode attention on host cores (the CPU side of Attention
// Piggybacking).  The reference charges it as
// probe_attention(cpu, DECODE, sum(ctx+1), n) / host.speed
// (pkg/src/hybridserve/engine.py:529-544); here it is computed: the shipped
// q/k/v row of an offloaded request is read from its pinned mailbox, the new
// token's k/v is appended to the request's host KV, and q attends over the
// ctx+1 host entries.  One task per (work item, KV head) so the GQA group
// shares every K/V row it streams from host DRAM.
#include <immintrin.h>
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "hs_step.h"

namespace hs {

// ---------------------------------------------------------------- thread pool
ThreadPool::ThreadPool(int n, const std::vector<int>& cpus) {
  for (int i = 0; i < n; ++i) {
    workers_.emplace_back([this, i] { loop(i); });
    if (!cpus.empty()) {
      cpu_set_t set;
      CPU_ZERO(&set);
      CPU_SET(cpus[i % cpus.size()], &set);
      pthread_setaffinity_np(workers_.back().native_handle(), sizeof(set), &set);
    }
  }
}

ThreadPool::~ThreadPool() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}

void ThreadPool::loop(int) {
  uint64_t seen = 0;
  for (;;) {
    const std::function<void(int)>* body;
    int n;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      // a call the caller finished alone before this worker woke: body_ is
      // already cleared (the caller clears it under the lock before it
      // returns).  Joining it would race the next call's reset of next_.
      if (!body_) continue;
      body = body_;
      n = n_;
      ++active_;
    }
    for (int i = next_.fetch_add(1); i < n; i = next_.fetch_add(1)) (*body)(i);
    {
      std::lock_guard<std::mutex> g(mu_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }
}

void ThreadPool::parallel_for(int n, const std::function<void(int)>& body) {
  if (n <= 0) return;
  if (workers_.empty() || n == 1) {
    for (int i = 0; i < n; ++i) body(i);
    return;
  }
  {
    std::lock_guard<std::mutex> g(mu_);
    body_ = &body;
    n_ = n;
    next_.store(0);
    ++gen_;
  }
  cv_.notify_all();
  for (int i = next_.fetch_add(1); i < n; i = next_.fetch_add(1)) body(i);
  std::unique_lock<std::mutex> lk(mu_);
  done_cv_.wait(lk, [&] { return active_ == 0 && next_.load() >= n; });
  body_ = nullptr;
}

// ---------------------------------------------------------------- kernels
static inline float bf2f(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t f2bf(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x7FFFFFu)) return static_cast<uint16_t>(u >> 16);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// 8 bf16 -> 8 fp32 (AVX2)
static inline __m256 load8_bf16(const uint16_t* p) {
  __m128i h = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p));
  return _mm256_castsi256_ps(_mm256_slli_epi32(_mm256_cvtepu16_epi32(h), 16));
}

static inline float hsum8(__m256 v) {
  __m128 lo = _mm256_castps256_ps128(v), hi = _mm256_extractf128_ps(v, 1);
  lo = _mm_add_ps(lo, hi);
  lo = _mm_add_ps(lo, _mm_movehl_ps(lo, lo));
  lo = _mm_add_ss(lo, _mm_shuffle_ps(lo, lo, 1));
  return _mm_cvtss_f32(lo);
}

constexpr int kMaxGroup = 16;
constexpr int kMaxHd = 128;
constexpr int kTile = 256;  // keys per softmax tile (online softmax across tiles)

// One (item, kv head): G query heads over ctx+1 keys.
static void attend_head(const ModelCfg& m, const uint16_t* q, const uint16_t* K,
                        const uint16_t* V, int n_keys, uint16_t* out, float* lse) {
  const int G = m.n_q / m.n_kv, hd = m.hd;
  const float scale = 1.0f / std::sqrt(static_cast<float>(hd));
  alignas(32) float qf[kMaxGroup][kMaxHd];
  alignas(32) float acc[kMaxGroup][kMaxHd];
  float mx[kMaxGroup], den[kMaxGroup];
  alignas(32) float s[kMaxGroup][kTile];
  for (int g = 0; g < G; ++g) {
    for (int i = 0; i < hd; ++i) qf[g][i] = bf2f(q[g * hd + i]) * scale;
    for (int i = 0; i < hd; ++i) acc[g][i] = 0.f;
    mx[g] = -INFINITY;
    den[g] = 0.f;
  }
  for (int t0 = 0; t0 < n_keys; t0 += kTile) {
    const int nt = std::min(kTile, n_keys - t0);
    float tmax[kMaxGroup];
    for (int g = 0; g < G; ++g) tmax[g] = -INFINITY;
    for (int t = 0; t < nt; ++t) {
      const uint16_t* kr = K + static_cast<size_t>(t0 + t) * hd;
      __m256 kv[kMaxHd / 8];
      for (int c = 0; c < hd / 8; ++c) kv[c] = load8_bf16(kr + 8 * c);
      for (int g = 0; g < G; ++g) {
        __m256 a = _mm256_setzero_ps();
        for (int c = 0; c < hd / 8; ++c) a = _mm256_fmadd_ps(_mm256_load_ps(&qf[g][8 * c]), kv[c], a);
        const float v = hsum8(a);
        s[g][t] = v;
        tmax[g] = std::max(tmax[g], v);
      }
    }
    for (int g = 0; g < G; ++g) {
      const float nm = std::max(mx[g], tmax[g]);
      const float corr = std::exp(mx[g] - nm);
      den[g] *= corr;
      for (int i = 0; i < hd; ++i) acc[g][i] *= corr;
      mx[g] = nm;
      float sum = 0.f;
      for (int t = 0; t < nt; ++t) {
        s[g][t] = std::exp(s[g][t] - nm);
        sum += s[g][t];
      }
      den[g] += sum;
    }
    for (int t = 0; t < nt; ++t) {
      const uint16_t* vr = V + static_cast<size_t>(t0 + t) * hd;
      __m256 vv[kMaxHd / 8];
      for (int c = 0; c < hd / 8; ++c) vv[c] = load8_bf16(vr + 8 * c);
      for (int g = 0; g < G; ++g) {
        const __m256 p = _mm256_set1_ps(s[g][t]);
        for (int c = 0; c < hd / 8; ++c)
          _mm256_store_ps(&acc[g][8 * c],
                          _mm256_fmadd_ps(p, vv[c], _mm256_load_ps(&acc[g][8 * c])));
      }
    }
  }
  for (int g = 0; g < G; ++g) {
    const float inv = 1.f / den[g];
    for (int i = 0; i < hd; ++i) out[g * hd + i] = f2bf(acc[g][i] * inv);
    if (lse) lse[g] = mx[g] + std::log(den[g]);
  }
}

void attend_group_avx512(int G, int hd, const uint16_t* q, const uint16_t* K, const uint16_t* V,
                         int n_keys, uint16_t* out, float* lse);
bool cpu_has_avx512bf16();

// AVX-512-BF16 when the host has it (cpu_attn_avx512.cpp), else AVX2/FMA.
static void attend_dispatch(const ModelCfg& m, const uint16_t* q, const uint16_t* K,
                            const uint16_t* V, int n_keys, uint16_t* out, float* lse,
                            bool allow_avx512 = true) {
  const int G = m.n_q / m.n_kv;
  if (allow_avx512 && cpu_has_avx512bf16() && (m.hd == 64 || m.hd == 128) && G <= 16)
    attend_group_avx512(G, m.hd, q, K, V, n_keys, out, lse);
  else
    attend_head(m, q, K, V, n_keys, out, lse);
}

// fp32 validation datapath: same layout in fp32 elements, exact float64 sums
void cpu_attend_head_f32(const ModelCfg& m, const float* ship, float* host_kv, int cap, int layer,
                         int ctx, int h, float* out_row) {
  const int hd = m.hd, G = m.n_q / m.n_kv;
  const float* k_new = ship + static_cast<size_t>(m.n_q) * hd + static_cast<size_t>(h) * hd;
  const float* v_new = ship + static_cast<size_t>(m.n_q + m.n_kv) * hd + static_cast<size_t>(h) * hd;
  float* K = host_kv + ((static_cast<size_t>(layer) * 2 + 0) * m.n_kv + h) * cap * hd;
  float* V = host_kv + ((static_cast<size_t>(layer) * 2 + 1) * m.n_kv + h) * cap * hd;
  std::memcpy(K + static_cast<size_t>(ctx) * hd, k_new, hd * sizeof(float));
  std::memcpy(V + static_cast<size_t>(ctx) * hd, v_new, hd * sizeof(float));
  const int n = ctx + 1;
  std::vector<double> sc(n), acc(hd);
  const double scale = 1.0 / std::sqrt(static_cast<double>(hd));
  for (int g = 0; g < G; ++g) {
    const float* q = ship + static_cast<size_t>(h * G + g) * hd;
    double mx = -1e300;
    for (int j = 0; j < n; ++j) {
      const float* k = K + static_cast<size_t>(j) * hd;
      double dot = 0.0;
      for (int e = 0; e < hd; ++e) dot += static_cast<double>(q[e]) * k[e];
      sc[j] = dot * scale;
      mx = std::max(mx, sc[j]);
    }
    double l = 0.0;
    std::fill(acc.begin(), acc.end(), 0.0);
    for (int j = 0; j < n; ++j) {
      const double p = std::exp(sc[j] - mx);
      l += p;
      const float* v = V + static_cast<size_t>(j) * hd;
      for (int e = 0; e < hd; ++e) acc[e] += p * v[e];
    }
    float* o = out_row + static_cast<size_t>(h * G + g) * hd;
    for (int e = 0; e < hd; ++e) o[e] = static_cast<float>(acc[e] / l);
  }
}

void cpu_attend_head(const ModelCfg& m, const bf16* ship_row, bf16* host_kv, int cap, int layer,
                     int ctx, int h, bf16* out_row, float* lse_out) {
  if (m.fp32) {
    cpu_attend_head_f32(m, reinterpret_cast<const float*>(ship_row),
                        reinterpret_cast<float*>(host_kv), cap, layer, ctx, h,
                        reinterpret_cast<float*>(out_row));
    return;
  }
  const int hd = m.hd, G = m.n_q / m.n_kv;
  const uint16_t* ship = reinterpret_cast<const uint16_t*>(ship_row);
  const uint16_t* q = ship + static_cast<size_t>(h) * G * hd;
  const uint16_t* k_new = ship + static_cast<size_t>(m.n_q) * hd + static_cast<size_t>(h) * hd;
  const uint16_t* v_new =
      ship + static_cast<size_t>(m.n_q + m.n_kv) * hd + static_cast<size_t>(h) * hd;
  uint16_t* base = reinterpret_cast<uint16_t*>(host_kv);
  uint16_t* K = base + ((static_cast<size_t>(layer) * 2 + 0) * m.n_kv + h) * cap * hd;
  uint16_t* V = base + ((static_cast<size_t>(layer) * 2 + 1) * m.n_kv + h) * cap * hd;
  std::memcpy(K + static_cast<size_t>(ctx) * hd, k_new, hd * 2);
  std::memcpy(V + static_cast<size_t>(ctx) * hd, v_new, hd * 2);
  attend_dispatch(m, q, K, V, ctx + 1,
                  reinterpret_cast<uint16_t*>(out_row) + static_cast<size_t>(h) * G * hd,
                  lse_out ? lse_out + h * G : nullptr);
}

void cpu_attend_one(const ModelCfg& m, const bf16* ship_row, bf16* host_kv, int cap, int layer,
                    int ctx, bf16* out_row, float* lse_out) {
  for (int h = 0; h < m.n_kv; ++h)
    cpu_attend_head(m, ship_row, host_kv, cap, layer, ctx, h, out_row, lse_out);
}

}  // namespace hs

using namespace hs;

extern "C" int hs_host_attention(const void* q, const void* k, const void* v, int n_keys, int n_q,
                                 int n_kv, int head_dim, void* out, float* lse, int impl) {
  if (n_keys < 1 || n_q % n_kv || n_q / n_kv > 16 || (head_dim != 64 && head_dim != 128))
    return set_error(HS_E_CONFIG, "host attention: unsupported shape");
  if (impl == 1 && !cpu_has_avx512bf16())
    return set_error(HS_E_CONFIG, "host attention: no AVX-512-BF16 on this CPU");
  ModelCfg m{};
  m.n_q = n_q;
  m.n_kv = n_kv;
  m.hd = head_dim;
  const int G = n_q / n_kv;
  for (int h = 0; h < n_kv; ++h) {
    const size_t kv_off = static_cast<size_t>(h) * n_keys * head_dim;
    const uint16_t* qh = static_cast<const uint16_t*>(q) + static_cast<size_t>(h) * G * head_dim;
    uint16_t* oh = static_cast<uint16_t*>(out) + static_cast<size_t>(h) * G * head_dim;
    attend_dispatch(m, qh, static_cast<const uint16_t*>(k) + kv_off,
                    static_cast<const uint16_t*>(v) + kv_off, n_keys, oh, lse ? lse + h * G : nullptr,
                    impl != 2);
  }
  return HS_OK;
}
