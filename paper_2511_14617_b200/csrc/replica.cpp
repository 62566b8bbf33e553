// replica.cpp — replica sync and memory reclamation: GDX1 delta / full-snapshot blobs
// (GroupDraftIndex::delta_since / full_snapshot / apply_blob / compact_log, cst.cpp:233-329;
// DraftServer::fetch_cst, dgds.cpp:53-97), and the same-capacity rebuild + history-arena
// compaction that returns the memory of dropped and expired groups (dgds.cpp:25-34,99-128).
#include "server_internal.h"

namespace dgds_host {

constexpr uint8_t kBlobDelta = 1, kBlobFull = 2;

size_t blob_preamble_bytes(const std::string& gid) { return 4 + 1 + 2 + gid.size() + 8 + 8 + 4; }

void put_be(uint8_t*& p, uint64_t v, int bytes) {
  for (int b = bytes - 1; b >= 0; --b) *p++ = static_cast<uint8_t>(v >> (8 * b));
}

void write_preamble(uint8_t* p, uint8_t kind, const std::string& gid, uint64_t from, uint64_t to, uint32_t n) {
  *p++ = 'G';
  *p++ = 'D';
  *p++ = 'X';
  *p++ = '1';
  *p++ = kind;
  put_be(p, gid.size(), 2);
  std::memcpy(p, gid.data(), gid.size());
  p += gid.size();
  put_be(p, from, 8);
  put_be(p, to, 8);
  put_be(p, n, 4);
}

struct BlobReader {  // detail::ByteReader (bytes.hpp) over a caller buffer
  const uint8_t* p;
  const uint8_t* end;
  bool ok = true;
  uint64_t get(int bytes) {
    if (end - p < bytes) {
      ok = false;
      p = end;
      return 0;
    }
    uint64_t v = 0;
    for (int b = 0; b < bytes; ++b) v = (v << 8) | *p++;
    return v;
  }
  std::string str() {
    const uint64_t n = get(2);
    if (!ok || static_cast<uint64_t>(end - p) < n) {
      ok = false;
      return {};
    }
    std::string s(reinterpret_cast<const char*>(p), n);
    p += n;
    return s;
  }
};

int compact_history(dgds_server* s) {
  std::vector<dgds::CopyPiece> pcs;
  uint64_t live = 0;
  for (auto& g : s->groups) {
    if (!g.alive) continue;
    for (LogRec& e : g.log) {
      pcs.push_back(dgds::CopyPiece{e.off, live, e.len, 0});
      e.off = live;
      live += e.len;
    }
  }
  const uint64_t cap = std::max<uint64_t>(1ull << 20, live + live / 2);
  int32_t* nb = nullptr;
  if (cudaMalloc(&nb, cap * sizeof(int32_t)) != cudaSuccess) return fail(DGDS_ENOMEM, "history arena allocation failed");
  if (!pcs.empty()) {
    if (int rc = s->d_blob_pieces.ensure(pcs.size() * sizeof(dgds::CopyPiece))) return rc;
    DGDS_CUDA(cudaMemcpyAsync(s->d_blob_pieces.p, pcs.data(), pcs.size() * sizeof(dgds::CopyPiece),
                              cudaMemcpyHostToDevice, s->st));
    DGDS_CUDA(dgds::launch_copy_pieces(static_cast<const dgds::CopyPiece*>(s->d_blob_pieces.p),
                                       static_cast<int64_t>(pcs.size()), s->d_hist, nb, s->st));
  }
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  cudaFree(s->d_hist);
  s->d_hist = nb;
  s->T.hist = nb;
  s->hist_cap = cap;
  s->T.hist_cap = cap;
  s->hist_used = live;
  s->dead_hist_tokens = 0;
  return DGDS_OK;
}

// Pack the live streams' token extents (moved and retired extents are dropped) and rewrite
// the device stream table. Runs after the rebuild, so no entry names a retired stream.
int compact_streams(dgds_server* s) {
  std::vector<dgds::CopyPiece> pcs;
  std::vector<dgds::StreamInfo> rows(s->stream_cap, dgds::StreamInfo{0, 0, 0});
  uint64_t live = 0;
  for (auto& g : s->groups) {
    if (!g.alive) continue;
    g.streams.for_each([&](int32_t, StreamRec& r) {
      const uint64_t nc = r.stored ? (std::max<uint64_t>(64, r.stored + r.stored / 4) + 7) / 8 * 8 : 0;
      if (r.stored) pcs.push_back(dgds::CopyPiece{r.sh_base, live, static_cast<uint32_t>(r.stored), 0});
      r.sh_base = live;
      r.sh_cap = nc;
      rows[r.slot] = dgds::StreamInfo{live, static_cast<uint32_t>(r.stored), g.root};
      live += nc;
    });
  }
  const uint64_t cap = std::max<uint64_t>(1ull << 20, live + live / 2);
  if (cap >= (1ull << 32)) return fail(DGDS_ENOMEM, "stream-history arena exceeds 2^32 tokens");
  int32_t* nb = nullptr;
  if (cudaMalloc(&nb, cap * sizeof(int32_t)) != cudaSuccess) return fail(DGDS_ENOMEM, "stream-history allocation failed");
  if (!pcs.empty()) {
    if (int rc = s->d_blob_pieces.ensure(pcs.size() * sizeof(dgds::CopyPiece))) return rc;
    DGDS_CUDA(cudaMemcpyAsync(s->d_blob_pieces.p, pcs.data(), pcs.size() * sizeof(dgds::CopyPiece),
                              cudaMemcpyHostToDevice, s->st));
    DGDS_CUDA(dgds::launch_copy_pieces(static_cast<const dgds::CopyPiece*>(s->d_blob_pieces.p),
                                       static_cast<int64_t>(pcs.size()), s->d_shist, nb, s->st));
  }
  DGDS_CUDA(cudaMemcpyAsync(s->T.sinfo, rows.data(), rows.size() * sizeof(dgds::StreamInfo), cudaMemcpyHostToDevice,
                            s->st));
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  cudaFree(s->d_shist);
  s->d_shist = nb;
  s->T.shist = nb;
  s->shist_cap = cap;
  s->T.shist_cap = cap;
  s->shist_used = live;
  s->dead_shist_tokens = 0;
  return DGDS_OK;
}

int compact_memory(dgds_server* s) {
  // planned-but-unlaunched device updates hold arena offsets and have not written their tokens
  if (s->plans_made != s->plans_launched) return fail(DGDS_ESTATE, "memory compaction with update plans outstanding");
  materialize_logs(s);
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  if (int rc = rebuild(s, s->T.cap)) return rc;
  if (int rc = compact_history(s)) return rc;
  if (int rc = compact_streams(s)) return rc;
  s->compactions += 1;
  return DGDS_OK;
}

// after explicit retirements: compact once retired groups hold > 40% of the history
int maybe_compact(dgds_server* s) {
  if (s->dead_hist_tokens < (1ull << 12) || s->dead_hist_tokens * 10 < s->hist_used * 4) return DGDS_OK;
  return compact_memory(s);
}

}  // namespace dgds_host

using namespace dgds_host;

extern "C" {

int dgds_fetch_cst(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* cached, double now,
                   dgds_fetch_reply* rep, const uint8_t** blobs) {
  if (!s || n < 0 || (n > 0 && (!handles || !cached || !rep || !blobs))) return fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  // a planned-but-unlaunched device update has bumped versions but not yet written its tokens
  if (s->plans_made != s->plans_launched) return fail(DGDS_ESTATE, "fetch_cst with update plans outstanding");
  materialize_logs(s);  // pending plans' history-log records first
  DGDS_CUDA(cudaSetDevice(s->p.device));
  for (int64_t i = 0; i < n; ++i)
    if (int rc = check_handle(s, handles[i])) return rc;
  std::vector<dgds::BlobPiece> pieces;
  struct Pre {
    int64_t i;
    uint8_t kind;
    uint64_t from, to;
    uint32_t count;
  };
  std::vector<Pre> pre;
  uint64_t total = 0;
  for (int64_t i = 0; i < n; ++i) {
    GroupRec& g = s->groups[handles[i]];
    dgds_fetch_reply& r = rep[i];
    r = dgds_fetch_reply{};
    if (!live_entry(s, g, now)) {  // lazy expiry erases it (dgds.cpp:25-34)
      r.kind = DGDS_FETCH_UNKNOWN_GROUP;
      continue;
    }
    g.expires = now + g.ttl;
    const uint64_t cur = g.version, c = cached[i];
    r.version = cur;
    if (c == cur && c != 0) {
      r.kind = DGDS_FETCH_UP_TO_DATE;
      continue;
    }
    if (c == cur) {  // both 0: nothing appended yet, the reference answers UpToDate too
      r.kind = DGDS_FETCH_UP_TO_DATE;
      continue;
    }
    const bool delta = c != 0 && c < cur && c >= g.log_floor;  // else Full (stale, fresh or compacted)
    const uint64_t base = (total + 7) & ~7ull;
    uint64_t pos = base + blob_preamble_bytes(g.gid);
    if (delta) {
      const size_t first = g.delta_base + static_cast<size_t>(c - g.log_floor);
      for (size_t k = first; k < g.log.size(); ++k) {
        const LogRec& e = g.log[k];
        pos += 16;
        pieces.push_back(dgds::BlobPiece{e.off, pos, e.start, e.len, static_cast<uint32_t>(e.rid), 1, 0});
        pos += 4ull * e.len;
      }
      pre.push_back(Pre{i, kBlobDelta, c, cur, static_cast<uint32_t>(g.log.size() - first)});
    } else {
      // std::map order: request id ascending; a stream's tokens are its log entries in order
      std::vector<std::pair<int32_t, uint64_t>> st;  // (rid, stored)
      g.streams.for_each([&](int32_t rid, StreamRec& sr) { st.emplace_back(rid, sr.stored); });
      std::sort(st.begin(), st.end());
      std::vector<uint32_t> order(g.log.size());
      for (size_t k = 0; k < order.size(); ++k) order[k] = static_cast<uint32_t>(k);
      std::stable_sort(order.begin(), order.end(),
                       [&](uint32_t a, uint32_t b) { return g.log[a].rid < g.log[b].rid; });
      size_t o = 0;
      for (const auto& [rid, stored] : st) {
        pos += 12;
        while (o < order.size() && g.log[order[o]].rid < rid) ++o;  // (no stream without a record)
        bool first = true;
        for (; o < order.size() && g.log[order[o]].rid == rid; ++o) {
          const LogRec& e = g.log[order[o]];
          pieces.push_back(dgds::BlobPiece{e.off, pos, stored, e.len, static_cast<uint32_t>(rid), first ? 2u : 0u, 0});
          first = false;
          pos += 4ull * e.len;
        }
        if (first) pieces.push_back(dgds::BlobPiece{0, pos, 0, 0, static_cast<uint32_t>(rid), 2, 0});  // empty stream
      }
      pre.push_back(Pre{i, kBlobFull, 0, cur, static_cast<uint32_t>(st.size())});
    }
    r.kind = delta ? DGDS_FETCH_DELTA : DGDS_FETCH_FULL;
    r.blob_off = base;
    r.blob_len = pos - base;
    total = pos;
  }
  if (total == 0) {
    *blobs = static_cast<const uint8_t*>(s->h_blob.p);
    return DGDS_OK;
  }
  if (int rc = s->d_blob.ensure(total)) return rc;
  if (int rc = s->h_blob.ensure(total)) return rc;
  if (!pieces.empty()) {
    if (int rc = s->d_blob_pieces.ensure(pieces.size() * sizeof(dgds::BlobPiece))) return rc;
    DGDS_CUDA(cudaMemcpyAsync(s->d_blob_pieces.p, pieces.data(), pieces.size() * sizeof(dgds::BlobPiece),
                              cudaMemcpyHostToDevice, s->st));
    DGDS_CUDA(dgds::launch_blob_fill(static_cast<const dgds::BlobPiece*>(s->d_blob_pieces.p),
                                     static_cast<int64_t>(pieces.size()), s->d_hist,
                                     static_cast<uint8_t*>(s->d_blob.p), s->st));
  }
  DGDS_CUDA(cudaMemcpyAsync(s->h_blob.p, s->d_blob.p, total, cudaMemcpyDeviceToHost, s->st));
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  uint8_t* hb = static_cast<uint8_t*>(s->h_blob.p);
  for (const Pre& p : pre) {
    const GroupRec& g = s->groups[handles[p.i]];
    write_preamble(hb + rep[p.i].blob_off, p.kind, g.gid, p.from, p.to, p.count);
  }
  *blobs = hb;
  return DGDS_OK;
}

int dgds_compact_group(dgds_server* s, int32_t h, uint64_t before_version) {  // dgds.cpp:153-158, cst.cpp:324-329
  if (!s) return fail(DGDS_EINVAL, "null server");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  materialize_logs(s);  // pending plans' history-log records first
  if (int rc = check_handle(s, h)) return rc;
  GroupRec& g = s->groups[h];
  if (!g.alive) return DGDS_OK;
  const uint64_t floor = std::min(before_version, g.version);
  if (floor <= g.log_floor) return DGDS_OK;
  g.delta_base += static_cast<size_t>(floor - g.log_floor);  // the entries stay: full snapshots need them
  g.log_floor = floor;
  return DGDS_OK;
}

int dgds_apply_blob(dgds_server* s, int32_t h, const uint8_t* blob, uint64_t len, double now, uint64_t* version) {
  if (!s || (!blob && len)) return fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  materialize_logs(s);  // pending plans' history-log records first
  if (int rc = check_handle(s, h)) return rc;
  GroupRec& g = s->groups[h];
  BlobReader r{blob, blob + len};
  char magic[4];
  for (char& c : magic) c = static_cast<char>(r.get(1));
  if (!r.ok || std::memcmp(magic, "GDX1", 4) != 0) return fail(DGDS_EBLOB, "bad draft blob magic");
  const uint8_t kind = static_cast<uint8_t>(r.get(1));
  const std::string gid = r.str();
  if (!r.ok) return fail(DGDS_EBLOB, "truncated record");
  if (gid != g.gid) return fail(DGDS_EBLOB, "draft blob for group " + gid + " applied to " + g.gid);
  const uint64_t from = r.get(8), to = r.get(8);
  if (!r.ok) return fail(DGDS_EBLOB, "truncated record");
  if (!live_entry(s, g, now)) {  // a replica starts empty (version 0)
    if (int rc = create_group(s, g, s->p.default_ttl_seconds, now)) return rc;
  }
  g.expires = now + g.ttl;
  std::vector<int32_t> rids, toks;
  std::vector<uint64_t> prevs, offs{0};
  auto read_tokens = [&](uint64_t cnt) -> bool {
    if (static_cast<uint64_t>(r.end - r.p) / 4 < cnt) {
      r.ok = false;
      return false;
    }
    for (uint64_t k = 0; k < cnt; ++k) toks.push_back(static_cast<int32_t>(static_cast<uint32_t>(r.get(4))));
    return true;
  };
  if (kind == kBlobDelta) {
    if (from != g.version)
      return fail(DGDS_EBLOB, "delta expects replica at version " + std::to_string(from) + ", replica is at " +
                                  std::to_string(g.version));
    const uint64_t cnt = r.get(4);
    // entries apply in order; like the reference, stop at the first one out of order
    std::unordered_map<int32_t, uint64_t> stored;
    bool bad = false;
    for (uint64_t k = 0; k < cnt && r.ok; ++k) {
      const int32_t rid = static_cast<int32_t>(static_cast<uint32_t>(r.get(4)));
      const uint64_t start = r.get(8);
      const uint64_t n = r.get(4);
      if (!r.ok || !read_tokens(n)) break;
      auto it = stored.find(rid);
      if (it == stored.end()) {
        const StreamRec* sr = g.streams.find(rid);
        it = stored.emplace(rid, sr ? sr->stored : 0).first;
      }
      if (start != it->second) {  // append() would reply ok=false (checked before its empty-token return)
        toks.resize(offs.back());
        bad = true;
        break;
      }
      it->second += n;
      rids.push_back(rid);
      prevs.push_back(start);
      offs.push_back(toks.size());
    }
    if (!r.ok && !bad) return fail(DGDS_EBLOB, "truncated record");
    std::vector<int32_t> hs(rids.size(), h);
    std::vector<dgds_update_reply> rep(rids.size());
    if (!rids.empty()) {
      if (int rc = update_batch_locked(s, static_cast<int64_t>(rids.size()), hs.data(), rids.data(), prevs.data(),
                                       offs.data(), toks.data(), now, rep.data()))
        return rc;
    }
    if (bad) return fail(DGDS_EBLOB, "delta entry out of order during apply");
    if (g.version != to) return fail(DGDS_EBLOB, "delta apply ended at unexpected version");
  } else if (kind == kBlobFull) {
    const uint64_t cnt = r.get(4);
    for (uint64_t k = 0; k < cnt && r.ok; ++k) {
      rids.push_back(static_cast<int32_t>(static_cast<uint32_t>(r.get(4))));
      const uint64_t n = r.get(8);
      if (!r.ok || !read_tokens(n)) break;
      prevs.push_back(0);
      offs.push_back(toks.size());
    }
    if (!r.ok) return fail(DGDS_EBLOB, "truncated record");
    // replace the replica: a fresh root, no streams, no history (cst.cpp:300-318)
    const double ttl = g.ttl;
    retire_group(s, g);
    if (int rc = create_group(s, g, ttl, now)) return rc;
    std::vector<int32_t> hs(rids.size(), h);
    std::vector<dgds_update_reply> rep(rids.size());
    if (!rids.empty()) {
      if (int rc = update_batch_locked(s, static_cast<int64_t>(rids.size()), hs.data(), rids.data(), prevs.data(),
                                       offs.data(), toks.data(), now, rep.data()))
        return rc;
    }
    g.version = to;  // a restored replica owns no history older than the snapshot
    g.delta_base = g.log.size();
    g.log_floor = to;
  } else {
    return fail(DGDS_EBLOB, "unknown draft blob kind");
  }
  if (version) *version = g.version;
  return DGDS_OK;
}

int dgds_compact_memory(dgds_server* s) {
  if (!s) return fail(DGDS_EINVAL, "null server");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  materialize_logs(s);  // pending plans' history-log records first
  DGDS_CUDA(cudaSetDevice(s->p.device));
  return compact_memory(s);
}

int dgds_get_memory_stats(dgds_server* s, dgds_memory_stats* out) {
  if (!s || !out) return fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  uint64_t used = 0;
  if (int rc = read_used(s, &used)) return rc;
  s->used_ub = used;
  out->slots = s->T.cap;
  out->used_slots = used;
  out->history_capacity = s->hist_cap;
  out->history_tokens = s->hist_used;
  out->dead_history_tokens = s->dead_hist_tokens;
  out->compactions = s->compactions;
  return DGDS_OK;
}

}  // extern "C"
