// C1 fast path: BE decode attention on AVX-512-BF16 host cores.
//
// QK^T: on AMX-BF16 tiles where the CPU and kernel allow it (K rows loaded
// as tile rows straight from the host KV, Q^T packed once), else vdpbf16ps
// on the bf16 q and K rows (32 MACs per instruction) with the per-key
// partial vectors of a 16-key tile transpose-reduced into one 16-lane score
// vector.  PV: two keys at a time, their V rows interleaved
// (unpacklo/hi_epi16) into bf16 pairs and multiplied by the pair of softmax
// weights with vdpbf16ps — the same bf16 rounding of P the GPU kernel uses.
// Online softmax across tiles with a vectorised exp2.  Layout: one request's
// K (or V) for one layer and KV head is contiguous [keys][hd] (host KV arena,
// DESIGN.md §4).
#include <immintrin.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "hs_step.h"

#define HS_AVX512 __attribute__((target("avx512f,avx512bw,avx512vl,avx512dq,avx512bf16")))
#define HS_AMX \
  __attribute__((target("avx512f,avx512bw,avx512vl,avx512dq,avx512bf16,amx-tile,amx-bf16")))

namespace hs {

namespace {

HS_AVX512 inline __m512 exp2_ps(__m512 x) {
  // 2^x = 2^n * 2^f, f in [-0.5, 0.5]; degree-6 minimax polynomial
  x = _mm512_max_ps(x, _mm512_set1_ps(-126.f));
  const __m512 n = _mm512_roundscale_ps(x, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
  const __m512 f = _mm512_sub_ps(x, n);
  __m512 p = _mm512_set1_ps(1.5353362e-4f);
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.3398874e-3f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(9.6180573e-3f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(5.5503324e-2f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(2.4022652e-1f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(6.9314718e-1f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.0f));
  const __m512i e = _mm512_slli_epi32(_mm512_add_epi32(_mm512_cvtps_epi32(n), _mm512_set1_epi32(127)), 23);
  return _mm512_mul_ps(p, _mm512_castsi512_ps(e));
}

// v[t] (16 vectors of 16 partial sums) -> r[t] = sum of v[t]'s lanes.
HS_AVX512 inline __m512 transpose_reduce16(const __m512* v) {
  __m512 w[8], x[4], y[2];
  for (int k = 0; k < 8; ++k)
    w[k] = _mm512_add_ps(_mm512_shuffle_f32x4(v[2 * k], v[2 * k + 1], 0x44),
                         _mm512_shuffle_f32x4(v[2 * k], v[2 * k + 1], 0xEE));
  for (int k = 0; k < 4; ++k)
    x[k] = _mm512_add_ps(_mm512_shuffle_f32x4(w[2 * k], w[2 * k + 1], 0x88),
                         _mm512_shuffle_f32x4(w[2 * k], w[2 * k + 1], 0xDD));
  for (int k = 0; k < 2; ++k)
    y[k] = _mm512_add_ps(_mm512_shuffle_ps(x[2 * k], x[2 * k + 1], 0x88),
                         _mm512_shuffle_ps(x[2 * k], x[2 * k + 1], 0xDD));
  const __m512 z = _mm512_add_ps(_mm512_shuffle_ps(y[0], y[1], 0x88),
                                 _mm512_shuffle_ps(y[0], y[1], 0xDD));
  // lane 4i+j of z holds key i+4j: permute to key order
  const __m512i idx = _mm512_setr_epi32(0, 4, 8, 12, 1, 5, 9, 13, 2, 6, 10, 14, 3, 7, 11, 15);
  return _mm512_permutexvar_ps(idx, z);
}

inline uint16_t f2bf_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

constexpr int kMaxG = 16;

// acc[g][c] += sum over the tile's key pairs of P(pair) x V(pair) for GN
// heads of chunk c (32 dims), accumulators in registers.
template <int GN>
HS_AVX512 inline void pv_tile(const uint16_t* V, int hd, int t0, int nt, int c,
                              const uint32_t (*ppair)[8], float (*acc_lo)[4][16],
                              float (*acc_hi)[4][16]) {
  __m512 lo[GN], hi[GN];
  for (int j = 0; j < GN; ++j) {
    lo[j] = _mm512_load_ps(acc_lo[j][c]);
    hi[j] = _mm512_load_ps(acc_hi[j][c]);
  }
  for (int k = 0; 2 * k < nt; ++k) {
    const uint16_t* va = V + static_cast<size_t>(t0 + 2 * k) * hd + 32 * c;
    const __m512i a = _mm512_loadu_si512(va);
    const __m512i b = 2 * k + 1 < nt ? _mm512_loadu_si512(va + hd) : _mm512_setzero_si512();
    const __m512bh ul = reinterpret_cast<__m512bh>(_mm512_unpacklo_epi16(a, b));
    const __m512bh uh = reinterpret_cast<__m512bh>(_mm512_unpackhi_epi16(a, b));
    for (int j = 0; j < GN; ++j) {
      const __m512bh pp = reinterpret_cast<__m512bh>(_mm512_set1_epi32(static_cast<int>(ppair[j][k])));
      lo[j] = _mm512_dpbf16_ps(lo[j], ul, pp);
      hi[j] = _mm512_dpbf16_ps(hi[j], uh, pp);
    }
  }
  for (int j = 0; j < GN; ++j) {
    _mm512_store_ps(acc_lo[j][c], lo[j]);
    _mm512_store_ps(acc_hi[j][c], hi[j]);
  }
}

}  // namespace

// ---- AMX for QK^T: S^T[16 keys][G] = K[16 keys][hd] . Q^T, the K rows
// loaded as tile rows straight from the host KV (no repacking), Q^T packed
// once per call in the VNNI pair layout.  tmm0 = K chunk (16 x 32 bf16),
// tmm2 = scores (16 x G fp32), tmm4..7 = Q^T chunks (16 pairs x G).
// AMX needs the process's permission for the tile state (Linux
// ARCH_REQ_XCOMP_PERM); without it, or on CPUs without AMX-BF16, QK^T stays
// on vdpbf16ps (HS_CPU_AMX=0 forces that too).
bool amx_ready() {
  static const bool ok = [] {
    const char* e = getenv("HS_CPU_AMX");
    if (e && e[0] == '0') return false;
    unsigned a, b, c, d;
    __asm__ __volatile__("cpuid" : "=a"(a), "=b"(b), "=c"(c), "=d"(d) : "a"(7), "c"(0));
    const bool has = ((d >> 22) & 1) && ((d >> 24) & 1);  // AMX-BF16, AMX-TILE
    if (!has) return false;
    constexpr long kArchReqXcompPerm = 0x1023, kXfeatureXtiledata = 18;
    return syscall(SYS_arch_prctl, kArchReqXcompPerm, kXfeatureXtiledata) == 0;
  }();
  return ok;
}

struct alignas(64) TileCfg {
  uint8_t palette, start_row, reserved[14];
  uint16_t colsb[16];
  uint8_t rows[16];
};

HS_AMX inline void amx_config(int G) {
  thread_local int configured_g = -1;
  if (configured_g == G) return;
  TileCfg cfg{};
  cfg.palette = 1;
  cfg.rows[0] = 16;
  cfg.colsb[0] = 64;  // K chunk: 16 keys x 32 bf16
  cfg.rows[2] = 16;
  cfg.colsb[2] = static_cast<uint16_t>(4 * G);  // scores: 16 keys x G fp32
  for (int t = 4; t < 8; ++t) {
    cfg.rows[t] = 16;  // 32 dims as 16 bf16 pairs
    cfg.colsb[t] = static_cast<uint16_t>(4 * G);
  }
  _tile_loadconfig(&cfg);
  configured_g = G;
}

// scores[16][G] (fp32) of keys [t0, t0 + 16) over the C = hd/32 chunks;
// keys past n_keys come from the zero-padded `tail` copy.
HS_AMX inline void amx_scores(const uint16_t* K, int hd, int C, int t0, int nt, const uint16_t* tail,
                              float* scores, int G) {
  const uint16_t* base = nt == 16 ? K + static_cast<size_t>(t0) * hd : tail;
  _tile_zero(2);
  _tile_loadd(0, base, hd * 2);
  _tile_dpbf16ps(2, 0, 4);
  if (C > 1) {
    _tile_loadd(0, base + 32, hd * 2);
    _tile_dpbf16ps(2, 0, 5);
  }
  if (C > 2) {
    _tile_loadd(0, base + 64, hd * 2);
    _tile_dpbf16ps(2, 0, 6);
    _tile_loadd(0, base + 96, hd * 2);
    _tile_dpbf16ps(2, 0, 7);
  }
  _tile_stored(2, scores, 4 * G);
}

// q: [G][hd] bf16 (one GQA group), K/V: [n_keys][hd] bf16 -> out [G][hd] bf16,
// lse [G] (natural log, optional).  hd in {64, 128}.
HS_AMX void attend_group_avx512(int G, int hd, const uint16_t* q, const uint16_t* K,
                                   const uint16_t* V, int n_keys, uint16_t* out, float* lse) {
  const int C = hd / 32;  // 32-bf16 chunks per row
  const float scale_log2 = 1.4426950408889634f / std::sqrt(static_cast<float>(hd));
  __m512bh qb[kMaxG][4];
  for (int g = 0; g < G; ++g)
    for (int c = 0; c < C; ++c)
      qb[g][c] = reinterpret_cast<__m512bh>(_mm512_loadu_si512(q + g * hd + 32 * c));
  alignas(64) float acc_lo[kMaxG][4][16], acc_hi[kMaxG][4][16];
  std::memset(acc_lo, 0, sizeof(acc_lo));
  std::memset(acc_hi, 0, sizeof(acc_hi));
  float m[kMaxG], den[kMaxG];
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    den[g] = 0.f;
  }
  __m512 part[kMaxG][16];
  __m512 raw[kMaxG];
  alignas(64) uint32_t ppair[kMaxG][8];
  // AMX: Q^T chunks in the VNNI pair layout, loaded once into tmm4..7
  const bool amx = amx_ready();
  alignas(64) uint16_t qv[4][16][32];
  alignas(64) uint16_t tail[16 * 128];
  alignas(64) float sc[16 * kMaxG];
  if (amx) {
    amx_config(G);
    std::memset(qv, 0, sizeof(qv));
    for (int c = 0; c < C; ++c)
      for (int r = 0; r < 16; ++r)
        for (int g = 0; g < G; ++g) {
          qv[c][r][2 * g] = q[g * hd + 32 * c + 2 * r];
          qv[c][r][2 * g + 1] = q[g * hd + 32 * c + 2 * r + 1];
        }
    _tile_loadd(4, qv[0], 64);
    _tile_loadd(5, qv[1], 64);
    _tile_loadd(6, qv[2], 64);
    _tile_loadd(7, qv[3], 64);
  }
  const __m512i lane = _mm512_setr_epi32(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15);
  // software prefetch of the K/V rows pf_tiles 16-key tiles ahead: one
  // host core's hardware prefetchers alone leave DRAM latency exposed
  // (B200 box, 14 workers, 32 x 9000 ctx: 103 GB/s without, 129 GB/s with
  // 2 tiles + AMX QK^T; HS_CPU_PF tunes it, 0 = off)
  static const int pf_tiles = [] {
    const char* e = getenv("HS_CPU_PF");
    return e ? atoi(e) : 2;
  }();
  const size_t row_bytes = static_cast<size_t>(hd) * 2;
  for (int t0 = 0; t0 < n_keys; t0 += 16) {
    const int nt = n_keys - t0 < 16 ? n_keys - t0 : 16;
    if (pf_tiles > 0) {
      const int tp = t0 + 16 * pf_tiles;
      if (tp < n_keys) {
        const int np = n_keys - tp < 16 ? n_keys - tp : 16;
        const char* kp = reinterpret_cast<const char*>(K + static_cast<size_t>(tp) * hd);
        const char* vp = reinterpret_cast<const char*>(V + static_cast<size_t>(tp) * hd);
        for (size_t off = 0; off < np * row_bytes; off += 64) {
          _mm_prefetch(kp + off, _MM_HINT_T0);
          _mm_prefetch(vp + off, _MM_HINT_T0);
        }
      }
    }
    // ---- scores of 16 keys for every head of the group
    if (amx) {
      if (nt < 16) {
        std::memset(tail, 0, sizeof(tail));
        std::memcpy(tail, K + static_cast<size_t>(t0) * hd, static_cast<size_t>(nt) * hd * 2);
      }
      amx_scores(K, hd, C, t0, nt, tail, sc, G);
      const __m512i idx = _mm512_mullo_epi32(lane, _mm512_set1_epi32(G));
      for (int g = 0; g < G; ++g)
        raw[g] = _mm512_i32gather_ps(_mm512_add_epi32(idx, _mm512_set1_epi32(g)), sc, 4);
    } else {
      for (int t = 0; t < 16; ++t) {
        if (t < nt) {
          const uint16_t* kr = K + static_cast<size_t>(t0 + t) * hd;
          __m512bh kc[4];
          for (int c = 0; c < C; ++c)
            kc[c] = reinterpret_cast<__m512bh>(_mm512_loadu_si512(kr + 32 * c));
          for (int g = 0; g < G; ++g) {
            __m512 a = _mm512_dpbf16_ps(_mm512_setzero_ps(), qb[g][0], kc[0]);
            for (int c = 1; c < C; ++c) a = _mm512_dpbf16_ps(a, qb[g][c], kc[c]);
            part[g][t] = a;
          }
        } else {
          for (int g = 0; g < G; ++g) part[g][t] = _mm512_setzero_ps();
        }
      }
      for (int g = 0; g < G; ++g) raw[g] = transpose_reduce16(part[g]);
    }
    const __mmask16 valid = static_cast<__mmask16>((1u << nt) - 1u);
    for (int g = 0; g < G; ++g) {
      __m512 s = _mm512_mul_ps(raw[g], _mm512_set1_ps(scale_log2));
      s = _mm512_mask_blend_ps(valid, _mm512_set1_ps(-INFINITY), s);
      const float tmax = _mm512_reduce_max_ps(s);
      const float nm = m[g] > tmax ? m[g] : tmax;
      const float corr = std::exp2(m[g] - nm);
      m[g] = nm;
      const __m512 p = _mm512_maskz_mov_ps(valid, exp2_ps(_mm512_sub_ps(s, _mm512_set1_ps(nm))));
      den[g] = den[g] * corr + _mm512_reduce_add_ps(p);
      if (corr != 1.f) {
        const __m512 cv = _mm512_set1_ps(corr);
        for (int c = 0; c < C; ++c) {
          _mm512_store_ps(acc_lo[g][c], _mm512_mul_ps(_mm512_load_ps(acc_lo[g][c]), cv));
          _mm512_store_ps(acc_hi[g][c], _mm512_mul_ps(_mm512_load_ps(acc_hi[g][c]), cv));
        }
      }
      // P as bf16 pairs (key 2k, key 2k+1)
      const __m256bh pb = _mm512_cvtneps_pbh(p);
      _mm256_store_si256(reinterpret_cast<__m256i*>(ppair[g]), reinterpret_cast<__m256i>(pb));
    }
    // ---- PV, two keys at a time: per 32-dim chunk, up to four heads'
    // accumulators stay in registers across the tile's key pairs
    for (int c = 0; c < C; ++c)
      for (int g0 = 0; g0 < G; g0 += 4) {
        switch (G - g0 < 4 ? G - g0 : 4) {
          case 1: pv_tile<1>(V, hd, t0, nt, c, ppair + g0, acc_lo + g0, acc_hi + g0); break;
          case 2: pv_tile<2>(V, hd, t0, nt, c, ppair + g0, acc_lo + g0, acc_hi + g0); break;
          case 3: pv_tile<3>(V, hd, t0, nt, c, ppair + g0, acc_lo + g0, acc_hi + g0); break;
          default: pv_tile<4>(V, hd, t0, nt, c, ppair + g0, acc_lo + g0, acc_hi + g0); break;
        }
      }
  }
  // un-permute: acc_lo[c] lane 4L+j -> dim 32c + 8L + j, acc_hi -> +4
  for (int g = 0; g < G; ++g) {
    const float inv = 1.f / den[g];
    for (int c = 0; c < C; ++c)
      for (int L = 0; L < 4; ++L)
        for (int j = 0; j < 4; ++j) {
          out[g * hd + 32 * c + 8 * L + j] = f2bf_rne(acc_lo[g][c][4 * L + j] * inv);
          out[g * hd + 32 * c + 8 * L + 4 + j] = f2bf_rne(acc_hi[g][c][4 * L + j] * inv);
        }
    if (lse) lse[g] = (m[g] + std::log2(den[g])) * 0.69314718055994530942f;
  }
}

bool cpu_has_avx512bf16() {
  static const int ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                        __builtin_cpu_supports("avx512bf16");
  return ok;
}

}  // namespace hs
