// Internal declarations of the serving-step context (step.cu, cpu_attn.cpp).
#pragma once

#include <atomic>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "hs_internal.h"

namespace hs {

int select_tokens(const int* row_token, const int* row_slot, int n_batch, const int* carry_slot,
                  const int* last_token, int rows, int* tok, cudaStream_t st);
int gather_rows_f32(const float* src, const int* idx, int rows, int d, float* dst,
                    cudaStream_t st);
int scatter_rows_f32(const float* src, const int* idx, int rows, int d, float* dst,
                     cudaStream_t st);
int gather_rows_bf16(const bf16* src, int src_stride, const int* idx, int rows, int w, bf16* dst,
                     int dst_stride, cudaStream_t st);
int scatter_tokens(const int* tok, const int* slot, int n, int* last_token, cudaStream_t st);
int kv_swap(bool to_host, bf16* pool, const KvGeom& g, const int* pages, int tokens, bf16* host,
            int cap, cudaStream_t st);

int set_error(int code, const char* fmt, ...);

// ---------------------------------------------------------------- CPU pool
// Fixed set of worker threads running parallel_for bodies (the BE
// CPU-attention service, reference engine.py:529-554; §4 uses an
// OpenMP pool per GPU).  Workers are pinned to `cpus` when given.
class ThreadPool {
 public:
  explicit ThreadPool(int n, const std::vector<int>& cpus = {});
  ~ThreadPool();
  int size() const { return static_cast<int>(workers_.size()) + 1; }
  // runs body(i) for i in [0, n) on the pool plus the calling thread
  void parallel_for(int n, const std::function<void(int)>& body);

 private:
  void loop(int id);
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* body_ = nullptr;
  int n_ = 0;
  std::atomic<int> next_{0};
  int active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct ModelCfg {
  int d, layers, n_q, n_kv, hd, ffn, vocab;
  float theta, eps;
  bool fp32 = false;  // validation datapath: fp32 mailboxes, host KV and CPU attention
  int qkv_n() const { return (n_q + 2 * n_kv) * hd; }
};

// Host-side decode attention for one offloaded request and one layer:
// appends the new token's k/v at position ctx of the request's host KV
// ([layers][2][n_kv][cap][hd] bf16) and attends q over ctx+1 entries.
void cpu_attend_head(const ModelCfg& m, const bf16* ship_row, bf16* host_kv, int cap, int layer,
                     int ctx, int h, bf16* out_row, float* lse_out);
// fp32 validation datapath: the same over fp32 rows / host KV (float64 sums)
void cpu_attend_head_f32(const ModelCfg& m, const float* ship_row, float* host_kv, int cap,
                         int layer, int ctx, int h, float* out_row);
void cpu_attend_one(const ModelCfg& m, const bf16* ship_row, bf16* host_kv, int cap, int layer,
                    int ctx, bf16* out_row, float* lse_out);

// asynchronous CPU-attention service (cpu_pool.cpp)
class CpuService;
CpuService* make_cpu_service(const ModelCfg& m, int threads, const std::vector<int>& cpus);
void destroy_cpu_service(CpuService* s);
void cpu_service_bind(CpuService* s, std::function<bf16*(int)> ship, std::function<bf16*(int)> res,
                      std::function<bf16*(int)> kv, std::function<int(int)> cap,
                      std::function<void(int, int, int)> publish,
                      std::function<void(int)> retract);
int cpu_service_submit(CpuService* s, cudaStream_t st, const int* slots, const int* layers,
                       const int* ctxs, int n);
int cpu_service_poll(CpuService* s, int* slots, int* layers, double* t_done, int max);
// device-polled merges: the pool takes its work items from a ring the GPU
// publishes into (mapped host memory: [Q][4] slot, layer, ctx, seq + tail)
void cpu_service_attach_ring(CpuService* s, const int* ring, const int* tail, int Q);
int cpu_service_in_flight(CpuService* s);
void cpu_service_route(
    CpuService* s,
    std::function<bool(int, int, int, cudaEvent_t, std::function<void()>)> route);

// remote CPU hosts (cpu_remote.cpp): one TCP relay per remote host; every
// op is sent in FIFO order by the relay's sender thread
class RemoteHost;
RemoteHost* remote_connect(const ModelCfg& m, const char* addr, int port);
void remote_destroy(RemoteHost* r);
// the slot's context (first ctx tokens of a [layers][2][n_kv][cap][hd] region) moves to the host
void remote_put(RemoteHost* r, int slot, int ctx, const bf16* region, int cap);
void remote_attend(RemoteHost* r, int slot, int layer, int ctx, cudaEvent_t ev, const bf16* ship,
                   bf16* result, std::function<void()> before_send, std::function<void()> done);
// blocking: the host's copy (with every appended token) lands in the region
bool remote_get(RemoteHost* r, int slot, int ctx, bf16* region, int cap);
bool remote_flush_puts(RemoteHost* r, int slot);
// non-blocking fetch (a live swap-in): `flag` becomes 1 once the KV landed
void remote_get_async(RemoteHost* r, int slot, int ctx, bf16* region, int cap,
                      std::shared_ptr<std::atomic<int>> flag);
bool remote_failed(RemoteHost* r);  // no PUT of the slot reads its region any more
void remote_free(RemoteHost* r, int slot);
bool remote_quiesce(RemoteHost* r);  // false once the connection failed
const int64_t* remote_stats(RemoteHost* r);
double cpu_service_busy(CpuService* s);
double wall_seconds();

}  // namespace hs
