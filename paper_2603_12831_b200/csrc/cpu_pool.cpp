// Asynchronous CPU-attention service (live mode).
//
// The GPU writes a chain's q/k/v row into its pinned mailbox inside hs_layer;
// hs_cpu_submit records a CUDA event behind those writes and queues one task
// per (work item, KV head).  Worker threads wait for the event, append the
// new k/v to the request's host KV, attend over ctx+1 keys and write the
// result mailbox; when every head of an item is done the item is appended to
// the completion FIFO that hs_cpu_poll drains.  This is the per-host input
// queue -> CPU service -> output queue path of the reference
// (pkg/src/hybridserve/engine.py:181-191, 512-560) with real workers instead
// of a charged service time; the GPU never waits on it (results are merged
// only once polled, engine.py:902-919).
#include <chrono>
#include <cstring>
#include <deque>
#include <thread>

#include "hs_step.h"

namespace hs {

struct CpuItem {
  int slot, layer, ctx;
  int ev;             // index into the event pool
  int heads_left;
  double t_submit;
};

struct CpuTask {
  int item;  // index into items_
  int head;
};

class CpuService {
 public:
  CpuService(const ModelCfg& m, int n_threads, int n_events, const std::vector<int>& cpus)
      : m_(m) {
    events_.resize(n_events);
    ev_refs_.assign(n_events, 0);
    for (auto& e : events_) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    for (int i = 0; i < n_threads; ++i) {
      threads_.emplace_back([this] { loop(); });
      if (!cpus.empty()) {
        cpu_set_t set;
        CPU_ZERO(&set);
        CPU_SET(cpus[i % cpus.size()], &set);
        pthread_setaffinity_np(threads_.back().native_handle(), sizeof(set), &set);
      }
    }
  }

  ~CpuService() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    if (dispatcher_.joinable()) dispatcher_.join();
    for (auto& t : threads_) t.join();
    for (auto& e : events_) cudaEventDestroy(e);
  }

  // mailboxes / KV resolution provided by the context
  std::function<bf16*(int slot)> ship_row, result_row, host_kv;
  std::function<void(int slot, int ctx, int layer)> publish;
  std::function<void(int slot)> retract;  // the slot's previous completion tag is void
  std::function<int(int slot)> host_cap;
  // remote CPU hosts (cpu_remote.cpp): hands the item to the relay of the
  // slot's remote host and returns true, or returns false for a local slot.
  // `done` completes the item from the relay's receiver thread.
  std::function<bool(int slot, int layer, int ctx, cudaEvent_t ev, std::function<void()> done)>
      route;

  int submit(cudaStream_t st, const int* slots, const int* layers, const int* ctxs, int n) {
    if (n <= 0) return HS_OK;
    int ev;
    {
      std::unique_lock<std::mutex> lk(mu_);
      // find a free event (all of its previous items finished)
      ev = -1;
      for (int k = 0; k < static_cast<int>(events_.size()); ++k) {
        const int e = (next_ev_ + k) % events_.size();
        if (ev_refs_[e] == 0) {
          ev = e;
          break;
        }
      }
      if (ev < 0) return set_error(HS_E_CAPACITY, "cpu service: event pool exhausted");
      next_ev_ = (ev + 1) % events_.size();
      ev_refs_[ev] = n;
    }
    if (cudaEventRecord(events_[ev], st) != cudaSuccess) {
      std::lock_guard<std::mutex> g(mu_);
      ev_refs_[ev] = 0;  // not handed to any item
      return set_error(HS_E_CUDA, "cpu service: event record failed");
    }
    const double now = wall();
    {
      std::lock_guard<std::mutex> g(mu_);
      for (int i = 0; i < n; ++i) {
        in_flight_ += 1;
        if (to_remote(slots[i], layers[i], ctxs[i], ev)) continue;
        const int idx = static_cast<int>(items_.size());
        items_.push_back(CpuItem{slots[i], layers[i], ctxs[i], ev, m_.n_kv, now});
        for (int h = 0; h < m_.n_kv; ++h) tasks_.push_back(CpuTask{idx, h});
      }
    }
    cv_.notify_all();
    return HS_OK;
  }

  // Device-polled merges: work items arrive through a ring the GPU publishes
  // into (entries written, then the tail released after the rows landed);
  // a dispatcher thread turns new entries into tasks.  No CUDA events.
  void attach_ring(const int* ring, const int* tail, int Q) {
    std::lock_guard<std::mutex> g(mu_);
    if (dispatcher_.joinable()) return;
    ring_ = ring;
    ring_tail_ = tail;
    ring_q_ = Q;
    ring_next_ = __atomic_load_n(tail, __ATOMIC_ACQUIRE);
    dispatcher_ = std::thread([this] { dispatch(); });
  }

  int poll(int* slots, int* layers, double* t_done, int max) {
    std::lock_guard<std::mutex> g(mu_);
    int k = 0;
    while (k < max && !done_.empty()) {
      const auto d = done_.front();
      done_.pop_front();
      slots[k] = std::get<0>(d);
      layers[k] = std::get<1>(d);
      if (t_done) t_done[k] = std::get<2>(d);
      ++k;
    }
    return k;
  }

  int in_flight() {
    std::lock_guard<std::mutex> g(mu_);
    return in_flight_;
  }

  double busy_seconds() const { return busy_ns_.load() * 1e-9; }

  static double wall() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
  }

 private:
  // called with mu_ held; the relay's completion takes mu_ from its own thread
  bool to_remote(int slot, int layer, int ctx, int ev) {
    if (!route) return false;
    return route(slot, layer, ctx, ev >= 0 ? events_[ev] : nullptr, [this, slot, layer, ctx, ev] {
      std::lock_guard<std::mutex> g(mu_);
      publish(slot, ctx, layer);
      done_.emplace_back(slot, layer, wall());
      if (ev >= 0) --ev_refs_[ev];
      --in_flight_;
    });
  }

  void dispatch() {
    int idle = 0;
    for (;;) {
      {
        std::lock_guard<std::mutex> g(mu_);
        if (stop_) return;
      }
      const int tail = __atomic_load_n(ring_tail_, __ATOMIC_ACQUIRE);
      if (tail == ring_next_) {
        if (++idle < 256) {
          __builtin_ia32_pause();
        } else {
          std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
        continue;
      }
      idle = 0;
      const double now = wall();
      {
        std::lock_guard<std::mutex> g(mu_);
        for (int i = ring_next_; i != tail; ++i) {
          const int* e = ring_ + static_cast<size_t>(i % ring_q_) * 4;
          ++in_flight_;
          if (to_remote(e[0], e[1], e[2], -1)) continue;
          const int idx = static_cast<int>(items_.size());
          items_.push_back(CpuItem{e[0], e[1], e[2], -1, m_.n_kv, now});
          for (int h = 0; h < m_.n_kv; ++h) tasks_.push_back(CpuTask{idx, h});
        }
      }
      ring_next_ = tail;
      cv_.notify_all();
    }
  }

  void loop() {
    for (;;) {
      CpuTask t;
      CpuItem it;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !tasks_.empty(); });
        if (stop_) return;
        t = tasks_.front();
        tasks_.pop_front();
        it = items_[t.item];
      }
      if (it.ev >= 0) cudaEventSynchronize(events_[it.ev]);  // the shipped row has landed
      // the slot's previous result was consumed before this item's ship
      // launch (stream order): retract its tag so the device cannot take a
      // stale tag for this item's result (every head does it before the
      // item's publish below)
      retract(it.slot);
      const auto t0 = std::chrono::steady_clock::now();
      cpu_attend_head(m_, ship_row(it.slot), host_kv(it.slot), host_cap(it.slot), it.layer - 1,
                      it.ctx, t.head, result_row(it.slot), nullptr);
      busy_ns_ += std::chrono::duration_cast<std::chrono::nanoseconds>(
                      std::chrono::steady_clock::now() - t0)
                      .count();
      std::lock_guard<std::mutex> g(mu_);
      CpuItem& ref = items_[t.item];
      if (--ref.heads_left == 0) {
        // every head's result row is written (the mutex orders the other
        // workers' writes before this point): publish the completion tag
        // the device checks before merging the row
        publish(ref.slot, ref.ctx, ref.layer);
        done_.emplace_back(ref.slot, ref.layer, wall());
        if (ref.ev >= 0) --ev_refs_[ref.ev];
        --in_flight_;
        // compact the item table once everything queued so far is finished
        if (in_flight_ == 0 && tasks_.empty()) items_.clear();
      }
    }
  }

  ModelCfg m_;
  std::vector<std::thread> threads_;
  std::vector<cudaEvent_t> events_;
  std::vector<int> ev_refs_;
  int next_ev_ = 0;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<CpuTask> tasks_;
  std::vector<CpuItem> items_;
  std::deque<std::tuple<int, int, double>> done_;
  int in_flight_ = 0;
  bool stop_ = false;
  std::atomic<int64_t> busy_ns_{0};
  std::thread dispatcher_;
  const int* ring_ = nullptr;
  const int* ring_tail_ = nullptr;
  int ring_q_ = 0, ring_next_ = 0;
};

CpuService* make_cpu_service(const ModelCfg& m, int threads, const std::vector<int>& cpus) {
  return new CpuService(m, threads, 1024, cpus);
}
void destroy_cpu_service(CpuService* s) { delete s; }
void cpu_service_bind(CpuService* s, std::function<bf16*(int)> ship, std::function<bf16*(int)> res,
                      std::function<bf16*(int)> kv, std::function<int(int)> cap,
                      std::function<void(int, int, int)> publish,
                      std::function<void(int)> retract) {
  s->ship_row = std::move(ship);
  s->result_row = std::move(res);
  s->host_kv = std::move(kv);
  s->host_cap = std::move(cap);
  s->publish = std::move(publish);
  s->retract = std::move(retract);
}
void cpu_service_route(
    CpuService* s,
    std::function<bool(int, int, int, cudaEvent_t, std::function<void()>)> route) {
  s->route = std::move(route);
}
int cpu_service_submit(CpuService* s, cudaStream_t st, const int* slots, const int* layers,
                       const int* ctxs, int n) {
  return s->submit(st, slots, layers, ctxs, n);
}
int cpu_service_poll(CpuService* s, int* slots, int* layers, double* t_done, int max) {
  return s->poll(slots, layers, t_done, max);
}
int cpu_service_in_flight(CpuService* s) { return s->in_flight(); }
void cpu_service_attach_ring(CpuService* s, const int* ring, const int* tail, int Q) {
  s->attach_ring(ring, tail, Q);
}
double cpu_service_busy(CpuService* s) { return s->busy_seconds(); }
double wall_seconds() { return CpuService::wall(); }

}  // namespace hs
