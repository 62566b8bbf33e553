// wire.cpp — the framed DGDS wire protocol in front of the GPU draft server
// (reference: proj/include/rollsim/dgds_wire.hpp:12-28, proj/src/dgds_wire.cpp).
//
// Frames are a 4-byte big-endian payload length + payload; a payload starts with
// an op tag (0x01 update_cst, 0x02 fetch_cst, 0x03 register_group, reply = tag
// | 0x80, 0x7F error + message). Replies are byte-identical to the reference's
// serve_payload for the same server state.
//
// B200-first service: a reader thread per connection decodes frames and hands
// them to ONE dispatcher thread, which folds every update_cst waiting at that
// moment (one per connection: clients keep one request in flight, dgds_wire.hpp:56)
// into a single dgds_update_batch — one append-kernel launch instead of one per
// request — then answers each connection. Per-connection order is unchanged;
// requests of different connections are concurrent in the reference too.
#include <arpa/inet.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <future>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/dgds_b200.h"
#include "kernels.h"

namespace {

constexpr uint8_t kOpUpdate = 0x01, kOpFetch = 0x02, kOpRegister = 0x03, kOpReply = 0x80, kOpError = 0x7F;

struct Writer {  // detail::ByteWriter (bytes.hpp): big-endian
  std::vector<uint8_t> b;
  void u8(uint8_t v) { b.push_back(v); }
  void be(uint64_t v, int bytes) {
    for (int s = 8 * (bytes - 1); s >= 0; s -= 8) b.push_back(static_cast<uint8_t>(v >> s));
  }
  void str(const std::string& s) {
    be(s.size(), 2);
    b.insert(b.end(), s.begin(), s.end());
  }
};

struct Reader {  // detail::ByteReader: throws "truncated record" like the reference
  const uint8_t* p;
  const uint8_t* end;
  uint64_t be(int bytes) {
    if (end - p < bytes) throw std::out_of_range("truncated record");
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v = (v << 8) | *p++;
    return v;
  }
  std::string str() {
    const uint64_t n = be(2);
    if (static_cast<uint64_t>(end - p) < n) throw std::out_of_range("truncated record");
    std::string s(reinterpret_cast<const char*>(p), n);
    p += n;
    return s;
  }
};

std::vector<uint8_t> error_reply(const std::string& msg) {
  Writer w;
  w.u8(kOpError);
  w.str(msg);
  return w.b;
}

struct UpdateReq {
  std::string gid;
  int32_t rid;
  uint64_t prev;
  std::vector<int32_t> toks;
};

UpdateReq decode_update(Reader& r) {
  UpdateReq u;
  u.gid = r.str();
  u.rid = static_cast<int32_t>(static_cast<uint32_t>(r.be(4)));
  u.prev = r.be(8);
  const uint64_t n = r.be(4);
  if (static_cast<uint64_t>(r.end - r.p) / 4 < n) throw std::out_of_range("truncated record");
  u.toks.resize(n);
  for (uint64_t i = 0; i < n; ++i) u.toks[i] = static_cast<int32_t>(static_cast<uint32_t>(r.be(4)));
  return u;
}

std::vector<uint8_t> update_reply(const dgds_update_reply& rep) {
  Writer w;
  w.u8(kOpUpdate | kOpReply);
  w.u8(rep.ok ? 1 : 0);
  w.be(rep.version, 8);
  w.be(rep.acked_tokens, 8);
  return w.b;
}

int32_t intern(dgds_server* s, const std::string& gid) {
  int32_t h = -1;
  if (dgds_intern(s, gid.data(), gid.size(), &h) != DGDS_OK) throw std::runtime_error(dgds_last_error());
  return h;
}

void check(int rc) {
  if (rc == DGDS_OK) return;
  if (rc == DGDS_EINVAL) throw std::invalid_argument(dgds_last_error());
  throw std::runtime_error(dgds_last_error());
}

// One update_cst per request, applied as ONE batch in arrival order. A request the
// reference rejects with an exception gets that error reply after the effects the
// reference makes before throwing (dgds.cpp:39-48, cst.cpp:118-128): the group is
// auto-registered / refreshed, the stream created, and a prev_token_count mismatch is
// an ordinary ok=false reply (the tokens are never inspected then). A negative token
// after valid ones is the documented divergence: the reference inserts the prefix
// before throwing; here the record is rejected whole.
void serve_updates(dgds_server* s, std::vector<UpdateReq*>& reqs, double now, std::vector<std::vector<uint8_t>*>& out) {
  std::vector<int32_t> hs, rids;
  std::vector<uint64_t> prevs, offs{0};
  std::vector<int32_t> toks;
  std::vector<size_t> idx;
  std::vector<char> neg_token;
  for (size_t i = 0; i < reqs.size(); ++i) {
    UpdateReq& u = *reqs[i];
    int32_t h;
    try {
      h = intern(s, u.gid);
      if (u.rid < 0) {
        check(dgds_touch_group(s, h, now));
        throw std::invalid_argument("request_id must be nonnegative");
      }
    } catch (const std::exception& e) {
      *out[i] = error_reply(e.what());
      continue;
    }
    bool neg = false;
    for (int32_t t : u.toks) neg = neg || t < 0;
    hs.push_back(h);
    rids.push_back(u.rid);
    prevs.push_back(u.prev);
    if (!neg) toks.insert(toks.end(), u.toks.begin(), u.toks.end());  // else: an empty record (touch + stream)
    offs.push_back(toks.size());
    idx.push_back(i);
    neg_token.push_back(neg ? 1 : 0);
  }
  if (idx.empty()) return;
  std::vector<dgds_update_reply> rep(idx.size());
  const int rc = dgds_update_batch(s, static_cast<int64_t>(idx.size()), hs.data(), rids.data(), prevs.data(),
                                   offs.data(), toks.data(), now, rep.data());
  for (size_t k = 0; k < idx.size(); ++k) {
    std::vector<uint8_t>& o = *out[idx[k]];
    if (rc != DGDS_OK) o = error_reply(dgds_last_error());
    else if (neg_token[k] && rep[k].ok) o = error_reply("negative token");
    else o = update_reply(rep[k]);
  }
}

std::vector<uint8_t> serve_fetch(dgds_server* s, Reader& r, double now) {
  const uint64_t n = r.be(4);
  std::vector<int32_t> hs;
  std::vector<uint64_t> cached;
  for (uint64_t i = 0; i < n; ++i) {
    hs.push_back(intern(s, r.str()));
    cached.push_back(r.be(8));
  }
  std::vector<dgds_fetch_reply> rep(n);
  const uint8_t* blobs = nullptr;
  if (n) check(dgds_fetch_cst(s, static_cast<int64_t>(n), hs.data(), cached.data(), now, rep.data(), &blobs));
  Writer w;
  w.u8(kOpFetch | kOpReply);
  w.be(n, 4);
  for (const auto& x : rep) {
    w.u8(static_cast<uint8_t>(x.kind));
    w.be(x.version, 8);
    w.be(x.blob_len, 4);
    if (x.blob_len) w.b.insert(w.b.end(), blobs + x.blob_off, blobs + x.blob_off + x.blob_len);
  }
  return w.b;
}

std::vector<uint8_t> serve_register(dgds_server* s, Reader& r, double now) {
  const std::string gid = r.str();
  const uint32_t ttl = static_cast<uint32_t>(r.be(4));
  check(dgds_register_group(s, intern(s, gid), static_cast<double>(ttl), now));
  Writer w;
  w.u8(kOpRegister | kOpReply);
  w.u8(1);
  return w.b;
}

// Serve a run of payloads in order, batching consecutive updates (serve_payload, dgds_wire.cpp:103-143).
void serve_run(dgds_server* s, const std::vector<const std::vector<uint8_t>*>& payloads, double now,
               std::vector<std::vector<uint8_t>>& replies) {
  replies.assign(payloads.size(), {});
  std::vector<UpdateReq> ups(payloads.size());
  std::vector<UpdateReq*> batch;
  std::vector<std::vector<uint8_t>*> batch_out;
  auto flush = [&] {
    if (!batch.empty()) serve_updates(s, batch, now, batch_out);
    batch.clear();
    batch_out.clear();
  };
  for (size_t i = 0; i < payloads.size(); ++i) {
    Reader r{payloads[i]->data(), payloads[i]->data() + payloads[i]->size()};
    try {
      const uint8_t op = static_cast<uint8_t>(r.be(1));
      if (op == kOpUpdate) {
        ups[i] = decode_update(r);
        batch.push_back(&ups[i]);
        batch_out.push_back(&replies[i]);
        continue;
      }
      flush();
      if (op == kOpFetch) replies[i] = serve_fetch(s, r, now);
      else if (op == kOpRegister) replies[i] = serve_register(s, r, now);
      else replies[i] = error_reply("unknown op tag " + std::to_string(op));
    } catch (const std::exception& e) {
      replies[i] = error_reply(e.what());
    }
  }
  flush();
}

bool read_all(int fd, uint8_t* p, size_t n) {
  while (n > 0) {
    const ssize_t r = ::read(fd, p, n);
    if (r == 0) return false;
    if (r < 0) throw std::runtime_error("socket read failed");
    p += r;
    n -= static_cast<size_t>(r);
  }
  return true;
}

void write_all(int fd, const uint8_t* p, size_t n) {
  while (n > 0) {
    const ssize_t w = ::write(fd, p, n);
    if (w <= 0) throw std::runtime_error("socket write failed");
    p += w;
    n -= static_cast<size_t>(w);
  }
}

bool read_frame(int fd, std::vector<uint8_t>& payload) {
  uint8_t len[4];
  if (!read_all(fd, len, 4)) return false;
  const uint32_t n = (uint32_t(len[0]) << 24) | (uint32_t(len[1]) << 16) | (uint32_t(len[2]) << 8) | uint32_t(len[3]);
  if (n > (1u << 30)) throw std::runtime_error("frame too large");
  payload.resize(n);
  if (n > 0 && !read_all(fd, payload.data(), n)) throw std::runtime_error("truncated frame");
  return true;
}

void write_frame(int fd, const std::vector<uint8_t>& payload) {
  std::vector<uint8_t> f(4 + payload.size());
  const uint32_t n = static_cast<uint32_t>(payload.size());
  f[0] = static_cast<uint8_t>(n >> 24);
  f[1] = static_cast<uint8_t>(n >> 16);
  f[2] = static_cast<uint8_t>(n >> 8);
  f[3] = static_cast<uint8_t>(n);
  std::memcpy(f.data() + 4, payload.data(), payload.size());
  write_all(fd, f.data(), f.size());
}

}  // namespace

struct dgds_wire_service {
  dgds_server* s = nullptr;
  int listen_fd = -1;
  int port = 0;
  std::atomic<bool> stopping{false};       // accept + readers
  std::atomic<bool> dispatch_stop{false};  // the dispatcher, after every reader is gone
  std::thread accept_thread, dispatch_thread;
  std::mutex conn_mu;
  std::vector<std::thread> conns;
  std::vector<int> conn_fds;
  struct Req {
    std::vector<uint8_t> payload;
    std::promise<std::vector<uint8_t>> reply;
  };
  std::mutex qmu;
  std::condition_variable qcv;
  std::deque<Req*> q;
  std::chrono::steady_clock::time_point start = std::chrono::steady_clock::now();
  std::atomic<uint64_t> requests{0}, batches{0};

  double now() const { return std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count(); }

  void dispatch_loop() {
    while (true) {
      std::vector<Req*> run;
      {
        std::unique_lock<std::mutex> lk(qmu);
        qcv.wait(lk, [&] { return dispatch_stop.load() || !q.empty(); });
        if (q.empty() && dispatch_stop.load()) return;
        run.assign(q.begin(), q.end());
        q.clear();
      }
      std::vector<const std::vector<uint8_t>*> pl;
      for (Req* r : run) pl.push_back(&r->payload);
      std::vector<std::vector<uint8_t>> replies;
      serve_run(s, pl, now(), replies);
      requests += run.size();
      batches += 1;
      for (size_t i = 0; i < run.size(); ++i) run[i]->reply.set_value(std::move(replies[i]));
    }
  }

  void handle(int fd) {
    try {
      std::vector<uint8_t> payload;
      while (!stopping.load() && read_frame(fd, payload)) {
        Req r;
        r.payload = std::move(payload);
        auto fut = r.reply.get_future();
        {
          std::lock_guard<std::mutex> lk(qmu);
          q.push_back(&r);
        }
        qcv.notify_one();
        write_frame(fd, fut.get());
        payload.clear();
      }
    } catch (const std::exception&) {
      // connection torn down
    }
    ::close(fd);
  }

  void accept_loop() {
    while (!stopping.load()) {
      const int fd = ::accept(listen_fd, nullptr, nullptr);
      if (fd < 0) {
        if (stopping.load()) break;
        continue;
      }
      int one = 1;
      ::setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
      std::lock_guard<std::mutex> lk(conn_mu);
      conn_fds.push_back(fd);
      conns.emplace_back([this, fd] { handle(fd); });
    }
  }
};

extern "C" {

int dgds_wire_serve_payload(dgds_server* s, const uint8_t* payload, uint64_t len, double now, uint8_t* out,
                            uint64_t cap, uint64_t* out_len) {
  if (!s || (!payload && len) || !out_len) return dgds::set_error(DGDS_EINVAL, "null argument");
  std::vector<uint8_t> p(payload, payload + len);
  std::vector<std::vector<uint8_t>> replies;
  serve_run(s, {&p}, now, replies);
  *out_len = replies[0].size();
  if (replies[0].size() > cap) return dgds::set_error(DGDS_EBUFFER, "reply buffer too small");
  if (!replies[0].empty()) std::memcpy(out, replies[0].data(), replies[0].size());
  return DGDS_OK;
}

int dgds_wire_service_start(dgds_server* s, int32_t port, dgds_wire_service** out, int32_t* bound_port) {
  if (!s || !out) return dgds::set_error(DGDS_EINVAL, "null argument");
  auto* w = new dgds_wire_service();
  w->s = s;
  w->listen_fd = ::socket(AF_INET, SOCK_STREAM, 0);
  if (w->listen_fd < 0) {
    delete w;
    return dgds::set_error(DGDS_ESTATE, "cannot create listening socket");
  }
  int one = 1;
  ::setsockopt(w->listen_fd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof(one));
  sockaddr_in addr{};
  addr.sin_family = AF_INET;
  addr.sin_addr.s_addr = htonl(INADDR_LOOPBACK);
  addr.sin_port = htons(static_cast<uint16_t>(port));
  if (::bind(w->listen_fd, reinterpret_cast<sockaddr*>(&addr), sizeof(addr)) != 0 || ::listen(w->listen_fd, 64) != 0) {
    ::close(w->listen_fd);
    delete w;
    return dgds::set_error(DGDS_ESTATE, "cannot bind draft service port " + std::to_string(port));
  }
  socklen_t alen = sizeof(addr);
  ::getsockname(w->listen_fd, reinterpret_cast<sockaddr*>(&addr), &alen);
  w->port = ntohs(addr.sin_port);
  w->dispatch_thread = std::thread([w] { w->dispatch_loop(); });
  w->accept_thread = std::thread([w] { w->accept_loop(); });
  if (bound_port) *bound_port = w->port;
  *out = w;
  return DGDS_OK;
}

int dgds_wire_service_stats(dgds_wire_service* w, uint64_t* requests, uint64_t* batches) {
  if (!w) return dgds::set_error(DGDS_EINVAL, "null argument");
  if (requests) *requests = w->requests.load();
  if (batches) *batches = w->batches.load();
  return DGDS_OK;
}

int dgds_wire_service_stop(dgds_wire_service* w) {
  if (!w) return DGDS_OK;
  w->stopping.store(true);
  ::shutdown(w->listen_fd, SHUT_RDWR);
  ::close(w->listen_fd);
  if (w->accept_thread.joinable()) w->accept_thread.join();
  {
    std::lock_guard<std::mutex> lk(w->conn_mu);
    for (int fd : w->conn_fds) ::shutdown(fd, SHUT_RDWR);  // unblock readers
  }
  for (auto& t : w->conns)  // the dispatcher still answers requests in flight
    if (t.joinable()) t.join();
  w->dispatch_stop.store(true);
  w->qcv.notify_all();
  if (w->dispatch_thread.joinable()) w->dispatch_thread.join();
  delete w;
  return DGDS_OK;
}

}  // extern "C"
