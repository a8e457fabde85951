// Remote CPU hosts: BE decode attention on a host other than the GPU's own.
//
// The reference models a cluster with `cpu_hosts` CPU hosts: host 0 is the
// GPU's local host (reached over PCIe), hosts 1.. are remote (reached over
// the network, alpha/beta of cluster.network; engine.py:329-331).  A request
// is offloaded to the local host while its memory lasts, else to the least
// loaded remote host (engine.py:402-419), and from then on its per-layer
// work items travel GPU -> local host -> network -> remote host and the
// results travel back (engine.py:529-560 with the link charge of its host).
//
// Here a remote host is a separate process (`hs_cpu_host_serve`, launched by
// paper_2603_12831_b200/cpu_host.py) that owns the KV of the requests placed
// on it and runs the same host attention kernel (cpu_attend_head).  The
// GPU's replica keeps one TCP connection per remote host; a sender thread
// forwards, in FIFO order, KV placements (the swapped-out context), work
// items (the shipped q|k|v row, once the device wrote it) and KV fetches
// (swap-in from a remote host); a receiver thread writes each result row
// into the slot's result mailbox and completes the item exactly like a
// local worker would (completion tag, then the output FIFO).
//
// Wire format: a 16-byte header {op, slot, a, b} followed by the payload.
//   PUT    slot, a=ctx tokens, b=cap     (allocates the slot's KV)
//   PUT_ROWS slot, a=first row, b=rows  + that many of the [layers][2][n_kv]
//          rows, ctx*hd each (a placement streams in chunks, so other
//          slots' items and fetches are not stuck behind a 1 GB context)
//   ATTEND slot, a=layer (1-based), b=ctx  + one q|k|v row ((n_q+2n_kv)*hd)
//   GET    slot, a=ctx  -> KV_ROWS replies (slot, a=first row, b=rows + the
//          rows), streamed in chunks between the RESULTs of later items
//   FREE   slot
//   HELLO  a=byte width of an element, + hs_model_cfg ints -> HELLO reply
//   BYE    a=1: also stop the server
//   RESULT slot, a=layer, b=ctx  + n_q*hd row (the attention output)
//   ERR    a=code, + message bytes (b)
#include <arpa/inet.h>
#include <execinfo.h>
#include <signal.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <sys/socket.h>
#include <unistd.h>

#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <deque>
#include <map>
#include <memory>

#include "hs_step.h"

namespace hs {

namespace {

enum : int32_t {
  RM_HELLO = 1, RM_PUT = 2, RM_ATTEND = 3, RM_GET = 4, RM_FREE = 5, RM_BYE = 6,
  RM_RESULT = 7, RM_ERR = 9, RM_PUT_ROWS = 10, RM_KV_ROWS = 11  // 8: retired
};

struct RmHdr {
  int32_t op, slot, a, b;
};
static_assert(sizeof(RmHdr) == 16, "wire header");

bool send_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t k = ::send(fd, c, n, MSG_NOSIGNAL);
    if (k < 0 && errno == EINTR) continue;
    if (k <= 0) return false;
    c += k;
    n -= static_cast<size_t>(k);
  }
  return true;
}

bool recv_all(int fd, void* p, size_t n) {
  char* c = static_cast<char*>(p);
  while (n) {
    const ssize_t k = ::recv(fd, c, n, 0);
    if (k < 0 && errno == EINTR) continue;
    if (k <= 0) return false;
    c += k;
    n -= static_cast<size_t>(k);
  }
  return true;
}

bool send_hdr(int fd, int32_t op, int32_t slot, int32_t a, int32_t b) {
  const RmHdr h{op, slot, a, b};
  return send_all(fd, &h, sizeof h);
}

void set_nodelay(int fd) {
  int one = 1;
  setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
}

size_t kv_row_elems(const ModelCfg& m) { return static_cast<size_t>(2) * m.layers * m.n_kv; }

int model_ints(const ModelCfg& m, int32_t* out) {
  out[0] = m.d;
  out[1] = m.layers;
  out[2] = m.n_q;
  out[3] = m.n_kv;
  out[4] = m.hd;
  out[5] = m.ffn;
  out[6] = m.vocab;
  return 7;
}

}  // namespace

// ------------------------------------------------------------ client side

struct RemoteOp {
  int32_t op, slot, a, b;
  cudaEvent_t ev = nullptr;          // ATTEND: the shipped row has landed once this fires
  const bf16* src = nullptr;         // PUT: local region; ATTEND: ship row
  int src_cap = 0;
  bf16* dst = nullptr;               // ATTEND: result row; GET: local region
  int dst_cap = 0;
  std::function<void()> before_send;  // ATTEND: retract the slot's previous tag
  std::function<void()> done;         // ATTEND / GET: called by the receiver
};

class RemoteHost {
 public:
  RemoteHost(const ModelCfg& m, int fd) : m_(m), fd_(fd) {
    sender_ = std::thread([this] { send_loop(); });
    receiver_ = std::thread([this] { recv_loop(); });
  }

  ~RemoteHost() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    sender_.join();
    ::shutdown(fd_, SHUT_RDWR);  // unblocks the receiver
    receiver_.join();
    ::close(fd_);
  }

  void push(RemoteOp op) {
    {
      std::lock_guard<std::mutex> g(mu_);
      if (op.op == RM_PUT) ++puts_of_slot_[op.slot];
      q_.push_back(std::move(op));
    }
    cv_.notify_all();
  }

  // waits until no queued or streaming PUT of `slot` still reads its local region
  bool flush_puts(int slot) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] {
      auto it = puts_of_slot_.find(slot);
      return failed_ || it == puts_of_slot_.end() || it->second == 0;
    });
    return !failed_;
  }

  // waits for the reply of the op whose `done` flag is `flag`
  bool wait_flag(const std::atomic<bool>& flag) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return failed_ || flag.load(); });
    return !failed_;
  }

  // waits until every queued op has been sent (and every reply received)
  bool quiesce() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] {
      return failed_ || (q_.empty() && attends_.empty() && gets_.empty() && !sending_ &&
                         !put_active_);
    });
    return !failed_;
  }

  bool failed() {
    std::lock_guard<std::mutex> g(mu_);
    return failed_;
  }

  int64_t stats[4] = {0, 0, 0, 0};  // items, put bytes, get bytes, result bytes

 private:
  void fail() {
    std::lock_guard<std::mutex> g(mu_);
    failed_ = true;
    cv_.notify_all();
  }

  // Sender: ops leave in FIFO order per slot, but a placement (PUT) streams
  // in chunks and the other slots' ops overtake it between chunks.  An op of
  // a slot with a PUT in flight or queued ahead of it waits.
  void send_loop() {
    const size_t rows_total = kv_row_elems(m_);
    RemoteOp put;  // the placement being streamed (put_active_)
    size_t put_row = 0;
    bool alternate = false;  // a chunk goes next (control ops cannot starve a placement)
    for (;;) {
      RemoteOp op;
      bool chunk = false;
      size_t r0 = 0, nr = 0;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !q_.empty() || put_active_; });
        if (q_.empty() && !put_active_) {  // stop_ with nothing left to send
          send_hdr(fd_, RM_BYE, 0, 0, 0);
          return;
        }
        int pick = -1;
        blocked_.clear();
        if (put_active_ && alternate) goto stream_chunk;
        if (put_active_) blocked_.push_back(put.slot);
        for (size_t i = 0; i < q_.size(); ++i) {
          const bool b = std::find(blocked_.begin(), blocked_.end(), q_[i].slot) != blocked_.end();
          if (q_[i].op == RM_PUT) {
            if (!b && !put_active_ && pick < 0) {  // start the oldest startable placement
              pick = static_cast<int>(i);
              break;
            }
            blocked_.push_back(q_[i].slot);
            continue;
          }
          if (!b) {
            pick = static_cast<int>(i);
            break;
          }
        }
        if (pick >= 0) {
          op = std::move(q_[pick]);
          q_.erase(q_.begin() + pick);
          if (op.op == RM_PUT) {
            put = op;
            put_row = 0;
            put_active_ = true;
          }
        } else {  // every queued op waits for the placement in flight: stream its next chunk
        stream_chunk:
          chunk = true;
          const size_t row_bytes = static_cast<size_t>(put.a) * m_.hd * sizeof(bf16);
          nr = std::max<size_t>(1, (size_t(4) << 20) / std::max<size_t>(row_bytes, 1));
          r0 = put_row;
          nr = std::min(nr, rows_total - r0);
          put_row += nr;
        }
        sending_ = true;
        alternate = put_active_ && !chunk;
      }
      bool ok = true;
      static const bool trace = std::getenv("HS_CPU_HOST_TRACE") != nullptr;
      if (trace)
        std::fprintf(stderr, "hs remote host: send op %d slot %d\n", chunk ? RM_PUT_ROWS : op.op,
                     chunk ? put.slot : op.slot);
      if (chunk) {
        ok = send_hdr(fd_, RM_PUT_ROWS, put.slot, static_cast<int32_t>(r0),
                      static_cast<int32_t>(nr));
        const size_t row = static_cast<size_t>(put.a) * m_.hd;
        for (size_t r = r0; ok && r < r0 + nr; ++r)
          if (row) ok = send_all(fd_, put.src + r * put.src_cap * m_.hd, row * sizeof(bf16));
        stats[1] += static_cast<int64_t>(nr * row * sizeof(bf16));
      } else {
        if (op.ev) cudaEventSynchronize(op.ev);
        if (op.before_send) op.before_send();
        const bool reply = op.op == RM_ATTEND || op.op == RM_GET;
        if (reply) {  // registered before the request leaves: the receiver may see it at once
          std::lock_guard<std::mutex> g(mu_);
          (op.op == RM_ATTEND ? attends_ : gets_).push_back(op);
        }
        ok = send_hdr(fd_, op.op, op.slot, op.a, op.b);
        if (ok && op.op == RM_ATTEND) {
          ok = send_all(fd_, op.src, static_cast<size_t>(m_.qkv_n()) * sizeof(bf16));
          stats[0] += 1;
        }
      }
      {
        std::lock_guard<std::mutex> g(mu_);
        sending_ = false;
        if (chunk && put_row >= rows_total) {  // placement complete
          put_active_ = false;
          --puts_of_slot_[put.slot];
        } else if (!chunk && op.op == RM_PUT && rows_total == 0) {
          put_active_ = false;
          --puts_of_slot_[op.slot];
        }
        if (!ok) failed_ = true;
      }
      cv_.notify_all();
      if (!ok) {
        std::fprintf(stderr, "hs remote host: send of op %d (slot %d) failed (%s)\n",
                     chunk ? RM_PUT_ROWS : op.op, chunk ? put.slot : op.slot,
                     std::strerror(errno));
        return;
      }
    }
  }

  // Receiver: RESULTs arrive in the order of the ATTENDs, KV_ROWS chunks in
  // the order of the GETs (one streaming at a time), the two interleaved.
  void recv_loop() {
    const size_t rows_total = kv_row_elems(m_);
    for (;;) {
      RmHdr h;
      if (!recv_all(fd_, &h, sizeof h)) {
        std::lock_guard<std::mutex> g(mu_);
        if (!attends_.empty() || !gets_.empty() || !q_.empty()) failed_ = true;
        cv_.notify_all();
        return;
      }
      const bool result = h.op == RM_RESULT;
      RemoteOp op;
      {
        std::lock_guard<std::mutex> g(mu_);
        std::deque<RemoteOp>& fifo = result ? attends_ : gets_;
        if ((h.op != RM_RESULT && h.op != RM_KV_ROWS) || fifo.empty()) {
          if (h.op == RM_ERR) {
            std::vector<char> msg(static_cast<size_t>(std::max(0, h.b)) + 1, 0);
            recv_all(fd_, msg.data(), static_cast<size_t>(std::max(0, h.b)));
            std::fprintf(stderr, "hs remote host: error %d: %s\n", h.a, msg.data());
          } else {
            std::fprintf(stderr, "hs remote host: unexpected message %d (slot %d, %d, %d)\n",
                         h.op, h.slot, h.a, h.b);
          }
          failed_ = true;
          cv_.notify_all();
          return;
        }
        op = fifo.front();  // popped once handled: quiesce() waits for it
      }
      bool ok = false, finished = false;
      if (result && h.slot == op.slot && h.a == op.a && h.b == op.b) {
        const size_t bytes = static_cast<size_t>(m_.n_q) * m_.hd * sizeof(bf16);
        ok = recv_all(fd_, op.dst, bytes);
        stats[3] += static_cast<int64_t>(bytes);
        finished = true;
      } else if (!result && h.slot == op.slot && h.a >= 0 && h.b >= 0 &&
                 static_cast<size_t>(h.a) + h.b <= rows_total) {
        const size_t row = static_cast<size_t>(op.a) * m_.hd;
        ok = true;
        for (int r = h.a; ok && r < h.a + h.b; ++r)
          if (row) ok = recv_all(fd_, op.dst + static_cast<size_t>(r) * op.dst_cap * m_.hd,
                                 row * sizeof(bf16));
        stats[2] += static_cast<int64_t>(h.b * row * sizeof(bf16));
        finished = static_cast<size_t>(h.a) + h.b == rows_total;
      }
      if (!ok) {
        fail();
        return;
      }
      if (!finished) continue;
      if (op.done) op.done();
      {
        std::lock_guard<std::mutex> g(mu_);
        (result ? attends_ : gets_).pop_front();
      }
      cv_.notify_all();
    }
  }

  ModelCfg m_;
  int fd_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<RemoteOp> q_, attends_, gets_;  // sent ops awaiting their reply
  bool sending_ = false, stop_ = false, failed_ = false, put_active_ = false;
  std::map<int, int> puts_of_slot_;  // queued or streaming placements per slot
  std::vector<int> blocked_;         // send_loop scratch
  std::thread sender_, receiver_;
};

RemoteHost* remote_connect(const ModelCfg& m, const char* addr, int port) {
  if (m.fp32) {
    set_error(HS_E_CONFIG, "remote CPU hosts serve the bf16 datapath only");
    return nullptr;
  }
  const int fd = ::socket(AF_INET, SOCK_STREAM, 0);
  if (fd < 0) {
    set_error(HS_E_CONFIG, "socket: %s", std::strerror(errno));
    return nullptr;
  }
  sockaddr_in sa{};
  sa.sin_family = AF_INET;
  sa.sin_port = htons(static_cast<uint16_t>(port));
  if (inet_pton(AF_INET, addr, &sa.sin_addr) != 1 ||
      ::connect(fd, reinterpret_cast<sockaddr*>(&sa), sizeof sa) != 0) {
    set_error(HS_E_CONFIG, "connect %s:%d: %s", addr, port, std::strerror(errno));
    ::close(fd);
    return nullptr;
  }
  set_nodelay(fd);
  int32_t dims[8];
  const int nd = model_ints(m, dims);
  RmHdr h;
  if (!send_hdr(fd, RM_HELLO, 0, static_cast<int32_t>(sizeof(bf16)), nd) ||
      !send_all(fd, dims, nd * sizeof(int32_t)) || !recv_all(fd, &h, sizeof h) ||
      h.op != RM_HELLO) {
    set_error(HS_E_CONFIG, "remote host %s:%d rejected the model", addr, port);
    ::close(fd);
    return nullptr;
  }
  return new RemoteHost(m, fd);
}

void remote_destroy(RemoteHost* r) { delete r; }

void remote_put(RemoteHost* r, int slot, int ctx, const bf16* region, int cap) {
  RemoteOp op{RM_PUT, slot, ctx, cap};
  op.src = region;
  op.src_cap = cap;
  r->push(std::move(op));
}

void remote_attend(RemoteHost* r, int slot, int layer, int ctx, cudaEvent_t ev, const bf16* ship,
                   bf16* result, std::function<void()> before_send, std::function<void()> done) {
  RemoteOp op{RM_ATTEND, slot, layer, ctx};
  op.ev = ev;
  op.src = ship;
  op.dst = result;
  op.before_send = std::move(before_send);
  op.done = std::move(done);
  r->push(std::move(op));
}

bool remote_get(RemoteHost* r, int slot, int ctx, bf16* region, int cap) {
  RemoteOp op{RM_GET, slot, ctx, 0};
  op.dst = region;
  op.dst_cap = cap;
  auto flag = std::make_shared<std::atomic<bool>>(false);
  op.done = [flag] { flag->store(true); };
  r->push(std::move(op));
  return r->wait_flag(*flag);  // the receiver notifies after done()
}

bool remote_flush_puts(RemoteHost* r, int slot) { return r->flush_puts(slot); }

void remote_get_async(RemoteHost* r, int slot, int ctx, bf16* region, int cap,
                      std::shared_ptr<std::atomic<int>> flag) {
  RemoteOp op{RM_GET, slot, ctx, 0};
  op.dst = region;
  op.dst_cap = cap;
  op.done = [flag] { flag->store(1, std::memory_order_release); };
  r->push(std::move(op));
}

bool remote_failed(RemoteHost* r) { return r->failed(); }

void remote_free(RemoteHost* r, int slot) { r->push(RemoteOp{RM_FREE, slot, 0, 0}); }

bool remote_quiesce(RemoteHost* r) { return r->quiesce(); }

const int64_t* remote_stats(RemoteHost* r) { return r->stats; }

// ------------------------------------------------------------ server side

namespace {

struct ServerSlot {
  std::vector<bf16> kv;
  int cap = 0;
  int put_ctx = 0;  // tokens per row of the placement being received
};

// a crashing host process says where before it dies (it runs unattended)
void fatal_signal(int sig) {
  void* frames[48];
  const int n = backtrace(frames, 48);
  char msg[64];
  const int len = std::snprintf(msg, sizeof msg, "hs cpu host: fatal signal %d\n", sig);
  if (write(2, msg, len) < 0) {}
  backtrace_symbols_fd(frames, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}

// one client connection (one GPU replica): its own slot namespace
bool serve_client(int fd, const ModelCfg& m, ThreadPool& pool, std::mutex& pool_mu,
                  int max_slots, bool* shutdown) {
  set_nodelay(fd);
  std::vector<ServerSlot> slots(static_cast<size_t>(max_slots));
  std::vector<bf16> ship(static_cast<size_t>(m.qkv_n())), out(static_cast<size_t>(m.n_q) * m.hd);
  RmHdr cur{};
  static const bool trace = std::getenv("HS_CPU_HOST_TRACE") != nullptr;
  auto err = [&](int code, const char* msg) {
    std::fprintf(stderr, "hs cpu host: %s (op %d slot %d a %d b %d)\n", msg, cur.op, cur.slot,
                 cur.a, cur.b);
    const int n = static_cast<int>(std::strlen(msg));
    send_hdr(fd, RM_ERR, 0, code, n);
    send_all(fd, msg, n);
    return false;
  };
  // the fetch being streamed back (one at a time, in GET order): its rows go
  // out in ~4 MB chunks whenever no request is waiting on the socket, so the
  // RESULTs of later items are not held behind a multi-GB context
  std::deque<RmHdr> gets;  // slot, a = ctx
  std::vector<int> freeing;  // FREEs waiting for their slot's fetch to go out
  size_t get_row = 0;
  const size_t rows_total = kv_row_elems(m);
  auto stream_chunk = [&]() -> bool {
    const RmHdr g = gets.front();
    const ServerSlot& sl = slots[g.slot];
    const size_t row = static_cast<size_t>(g.a) * m.hd;
    size_t nr = std::max<size_t>(1, (size_t(4) << 20) / std::max<size_t>(row * sizeof(bf16), 1));
    nr = std::min(nr, rows_total - get_row);
    if (!send_hdr(fd, RM_KV_ROWS, g.slot, static_cast<int32_t>(get_row), static_cast<int32_t>(nr)))
      return false;
    for (size_t r = get_row; r < get_row + nr; ++r)
      if (row && !send_all(fd, sl.kv.data() + r * sl.cap * m.hd, row * sizeof(bf16))) return false;
    get_row += nr;
    if (get_row == rows_total) {
      gets.pop_front();
      get_row = 0;
      // deferred FREEs of slots with no fetch left
      for (size_t i = 0; i < freeing.size();) {
        bool pending = false;
        for (const RmHdr& q : gets) pending |= q.slot == freeing[i];
        if (pending) {
          ++i;
          continue;
        }
        slots[freeing[i]] = ServerSlot{};
        freeing.erase(freeing.begin() + i);
      }
    }
    return true;
  };
  // a request touching a slot whose fetch is still streaming: finish it first
  auto drain_gets_of = [&](int slot) -> bool {
    for (;;) {
      bool pending = false;
      for (const RmHdr& g : gets) pending |= g.slot == slot;
      if (!pending) return true;
      if (!stream_chunk()) return false;
    }
  };
  for (;;) {
    while (!gets.empty()) {  // stream while no request is waiting
      pollfd pf{fd, POLLIN, 0};
      if (::poll(&pf, 1, 0) > 0) break;
      if (!stream_chunk()) return false;
    }
    RmHdr h;
    if (!recv_all(fd, &h, sizeof h)) return true;  // client went away
    cur = h;
    // a FREE right behind its slot's fetch (the usual swap-in) is deferred
    // until the stream is out; any other request on that slot drains it
    if (h.op == RM_FREE && h.slot >= 0 && h.slot < max_slots) {
      bool streaming = false;
      for (const RmHdr& g : gets) streaming |= g.slot == h.slot;
      if (streaming) {
        freeing.push_back(h.slot);
        continue;
      }
    }
    if (h.op != RM_HELLO && h.op != RM_BYE && h.slot >= 0 && h.slot < max_slots &&
        !drain_gets_of(h.slot))
      return false;
    if (trace) std::fprintf(stderr, "hs cpu host: op %d slot %d a %d b %d\n", h.op, h.slot, h.a, h.b);
    const bool slot_ok = h.slot >= 0 && h.slot < max_slots;
    switch (h.op) {
      case RM_HELLO: {
        int32_t dims[16] = {0}, mine[8];
        if (h.b < 0 || h.b > 16 || !recv_all(fd, dims, h.b * sizeof(int32_t))) return false;
        const int nd = model_ints(m, mine);
        if (h.a != static_cast<int32_t>(sizeof(bf16)) || h.b != nd ||
            std::memcmp(dims, mine, nd * sizeof(int32_t)) != 0)
          return err(HS_E_CONFIG, "model geometry mismatch");
        send_hdr(fd, RM_HELLO, 0, 0, 0);
        break;
      }
      case RM_PUT: {
        if (!slot_ok || h.a < 0 || h.b < h.a) return err(HS_E_CONFIG, "bad PUT");
        ServerSlot& s = slots[h.slot];
        s.cap = h.b;
        s.put_ctx = h.a;
        s.kv.assign(kv_row_elems(m) * static_cast<size_t>(s.cap) * m.hd, bf16{});
        break;
      }
      case RM_PUT_ROWS: {
        if (!slot_ok || slots[h.slot].cap == 0 || h.a < 0 || h.b < 0 ||
            static_cast<size_t>(h.a) + h.b > kv_row_elems(m))
          return err(HS_E_CONFIG, "bad PUT_ROWS");
        ServerSlot& s = slots[h.slot];
        const size_t row = static_cast<size_t>(s.put_ctx) * m.hd;
        for (int r = h.a; r < h.a + h.b; ++r)
          if (row && !recv_all(fd, s.kv.data() + static_cast<size_t>(r) * s.cap * m.hd,
                               row * sizeof(bf16)))
            return false;
        break;
      }
      case RM_ATTEND: {
        if (!recv_all(fd, ship.data(), ship.size() * sizeof(bf16))) return false;
        if (!slot_ok || slots[h.slot].cap == 0) return err(HS_E_INTEGRITY, "item without KV");
        ServerSlot& s = slots[h.slot];
        if (h.a < 1 || h.a > m.layers || h.b < 0 || h.b >= s.cap)
          return err(HS_E_CAPACITY, "item outside the slot's KV");
        {
          std::lock_guard<std::mutex> g(pool_mu);
          pool.parallel_for(m.n_kv, [&](int head) {
            cpu_attend_head(m, ship.data(), s.kv.data(), s.cap, h.a - 1, h.b, head, out.data(),
                            nullptr);
          });
        }
        if (!send_hdr(fd, RM_RESULT, h.slot, h.a, h.b) ||
            !send_all(fd, out.data(), out.size() * sizeof(bf16)))
          return false;
        break;
      }
      case RM_GET: {
        if (!slot_ok || slots[h.slot].cap < h.a || h.a < 0) return err(HS_E_CONFIG, "bad GET");
        gets.push_back(h);
        break;
      }
      case RM_FREE:
        if (slot_ok) slots[h.slot] = ServerSlot{};
        break;
      case RM_BYE:
        while (!gets.empty())
          if (!stream_chunk()) return false;
        *shutdown = h.a == 1;
        return true;
      default:
        return err(HS_E_CONFIG, "unknown op");
    }
  }
}

}  // namespace

}  // namespace hs

extern "C" {

// Serves remote-host CPU attention until a client sends BYE(1).  Prints
// "HS_CPU_HOST_READY port=<p>" on stdout once listening (port 0 = any).
__attribute__((visibility("default"))) int hs_cpu_host_serve(const hs_model_cfg* mc,
                                                             const char* bind_addr, int port,
                                                             int threads, int max_slots) {
  using namespace hs;
  if (!mc || threads < 1 || max_slots < 1) return set_error(HS_E_CONFIG, "bad server config");
  for (int sig : {SIGSEGV, SIGBUS, SIGILL, SIGFPE, SIGABRT}) signal(sig, fatal_signal);
  ModelCfg m{mc->d_model, mc->n_layers, mc->n_q,      mc->n_kv,    mc->head_dim,
             mc->ffn,     mc->vocab,    mc->rope_theta, mc->norm_eps};
  const int lfd = ::socket(AF_INET, SOCK_STREAM, 0);
  if (lfd < 0) return set_error(HS_E_CONFIG, "socket: %s", std::strerror(errno));
  int one = 1;
  setsockopt(lfd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof one);
  sockaddr_in sa{};
  sa.sin_family = AF_INET;
  sa.sin_port = htons(static_cast<uint16_t>(port));
  if (inet_pton(AF_INET, bind_addr ? bind_addr : "127.0.0.1", &sa.sin_addr) != 1 ||
      ::bind(lfd, reinterpret_cast<sockaddr*>(&sa), sizeof sa) != 0 || ::listen(lfd, 8) != 0) {
    ::close(lfd);
    return set_error(HS_E_CONFIG, "bind/listen: %s", std::strerror(errno));
  }
  socklen_t len = sizeof sa;
  getsockname(lfd, reinterpret_cast<sockaddr*>(&sa), &len);
  std::printf("HS_CPU_HOST_READY port=%d\n", ntohs(sa.sin_port));
  std::fflush(stdout);
  ThreadPool pool(threads - 1);
  std::mutex pool_mu;
  std::atomic<bool> shutdown{false};
  std::vector<std::thread> clients;
  while (!shutdown.load()) {
    const int fd = ::accept(lfd, nullptr, nullptr);
    if (fd < 0) {
      if (errno == EINTR) continue;
      break;
    }
    clients.emplace_back([&, fd] {
      bool stop = false;
      if (!serve_client(fd, m, pool, pool_mu, max_slots, &stop))
        std::fprintf(stderr, "hs cpu host: connection dropped (%s)\n", std::strerror(errno));
      ::close(fd);
      if (stop) {
        shutdown = true;
        ::shutdown(lfd, SHUT_RDWR);  // unblocks accept()
      }
    });
  }
  for (auto& t : clients) t.join();
  ::close(lfd);
  return HS_OK;
}

}  // extern "C"
