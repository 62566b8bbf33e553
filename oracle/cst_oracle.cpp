// cst_oracle.cpp — CPU restatement of the reference DGDS hot path.
//
// TEST INFRASTRUCTURE ONLY (see oracle/Makefile). This is the checker the GPU
// parity tests compare against; it is never linked into or called by the
// product library. Parity of this restatement with the reference itself is
// pinned by tests/test_oracle.py against (a) the SPEC known-answer examples,
// (b) golden fixtures generated from the compiled reference
// (oracle/make_golden.py -> tests/golden/), and (c) live randomized
// differential runs against oracle/_ref/libdgds_ref.so when it is present.
//
// The restatement is deliberately NOT the reference's node/edge-map trie: it
// keys every window by its token CONTENT. The reference trie
// (proj/src/cst.cpp:86-116) stores, for every contiguous window of length
// <= max_pattern_len + max_spec_len inside one request stream, a node whose
// count is the number of occurrences of that window; children of a window w
// are the windows w·t that occurred. A content-keyed table has exactly the same
// observable state (counts and child sets), so speculate() below — which follows
// proj/src/cst.cpp:153-228 step by step — must return identical results.

#include <algorithm>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "oracle_capi.h"

namespace {

thread_local std::string g_err;

using Seq = std::vector<int32_t>;

struct Window {
  uint32_t count = 0;
  Seq next;  // distinct continuation tokens (child set), insertion order irrelevant
};

std::string key_of(const int32_t* p, size_t n) { return std::string(reinterpret_cast<const char*>(p), n * 4); }

// validate_args: proj/src/cst.cpp:18-25
void check_args(const orc_args& a) {
  if (a.pattern_lookup_min < 1 || a.pattern_lookup_min > a.pattern_lookup_max)
    throw std::invalid_argument("speculation args: need 1 <= pattern_lookup_min <= pattern_lookup_max");
  if (a.max_spec_tokens < 0) throw std::invalid_argument("speculation args: max_spec_tokens must be >= 0");
  if (a.top_k < 1) throw std::invalid_argument("speculation args: top_k must be >= 1");
  if (a.min_step_freq < 0.0) throw std::invalid_argument("speculation args: min_step_freq must be >= 0");
  if (a.min_support < 0) throw std::invalid_argument("speculation args: min_support must be >= 0");
}

struct Cand {
  Seq toks;
  double score;
  int64_t support;
};

// candidate_before: proj/src/cst.cpp:29-33 (score desc, support desc, tokens lexicographic asc)
bool before(const Cand& a, const Cand& b) {
  if (a.score != b.score) return a.score > b.score;
  if (a.support != b.support) return a.support > b.support;
  return a.toks < b.toks;
}

struct Index {
  int lim_pattern = 8, lim_spec = 16;
  uint64_t version = 0;
  std::unordered_map<std::string, Window> windows;  // content key -> window
  Window root;                                      // the empty context (node 0 in the reference)
  std::map<int, Seq> streams;                       // request_id -> stored tokens

  int depth_cap() const { return lim_pattern + lim_spec; }  // cst.cpp:106-107

  Window* find(const int32_t* p, size_t n) {
    if (n == 0) return &root;
    auto it = windows.find(key_of(p, n));
    return it == windows.end() ? nullptr : &it->second;
  }
  const Window* find(const int32_t* p, size_t n) const { return const_cast<Index*>(this)->find(p, n); }

  // insert_token (cst.cpp:105-116): every window of length <= depth cap that
  // ends at the new token gains one occurrence; a window seen for the first
  // time becomes a child of its prefix window (ensure_child, cst.cpp:90-103).
  void push_token(Seq& s, int32_t t) {
    s.push_back(t);
    const size_t end = s.size();
    const size_t lmax = std::min<size_t>(static_cast<size_t>(depth_cap()), end);
    for (size_t len = 1; len <= lmax; ++len) {
      const int32_t* w = s.data() + (end - len);
      Window& win = windows[key_of(w, len)];
      if (win.count++ == 0) {
        Window* parent = find(w, len - 1);
        parent->next.push_back(t);
      }
    }
  }

  // append (cst.cpp:118-133): gap check, empty append, insert, version bump.
  void append(int rid, uint64_t prev, const int32_t* toks, uint64_t n, int32_t* ok, uint64_t* ver,
              uint64_t* acked) {
    if (rid < 0) throw std::invalid_argument("request_id must be nonnegative");
    Seq& s = streams[rid];  // a mismatched append still creates the stream (cst.cpp:121)
    if (prev != s.size()) {
      *ok = 0;
      *ver = version;
      *acked = s.size();
      return;
    }
    if (n == 0) {
      *ok = 1;
      *ver = version;
      *acked = s.size();
      return;
    }
    for (uint64_t i = 0; i < n; ++i) {
      if (toks[i] < 0) throw std::invalid_argument("negative token");
      push_token(s, toks[i]);
    }
    ++version;
    *ok = 1;
    *ver = version;
    *acked = s.size();
  }

  // speculate (cst.cpp:153-228), with the work counters of SURVEY.md §8(d).
  std::vector<Cand> speculate(const int32_t* pat, size_t plen, const orc_args& a, orc_qstats* st) const {
    check_args(a);
    orc_qstats local{};
    orc_qstats& S = st ? *st : local;
    S = orc_qstats{};
    const int pmax = std::min(a.pattern_lookup_max, lim_pattern);  // cst.cpp:156-158
    const int smax = std::min(a.max_spec_tokens, lim_spec);
    if (plen == 0 || a.pattern_lookup_min > pmax) return {};

    // Longest admissible suffix (cst.cpp:160-178): the first length whose
    // whole walk from the root succeeds wins; no shorter fallback afterwards.
    Seq ctx;
    const Window* locus = nullptr;
    for (int len = std::min<int>(pmax, static_cast<int>(plen)); len >= a.pattern_lookup_min; --len) {
      const int32_t* suf = pat + (plen - len);
      bool ok = true;
      for (int i = 1; i <= len; ++i) {
        ++S.suffix_lookups;
        if (!find(suf, i)) {
          ok = false;
          break;
        }
      }
      if (ok) {
        ctx.assign(suf, suf + len);
        locus = find(suf, len);
        break;
      }
    }
    if (!locus) return {};

    struct Path {
      Seq ctx;  // matched suffix + drafted tokens: identifies the trie node
      double score;
      int64_t support;
      Seq toks;
    };
    auto pbefore = [](const Path& x, const Path& y) {
      if (x.score != y.score) return x.score > y.score;
      if (x.support != y.support) return x.support > y.support;
      return x.toks < y.toks;
    };
    std::vector<Path> beam{Path{ctx, 1.0, static_cast<int64_t>(locus->count), {}}};
    std::vector<Cand> finals;
    for (int depth = 0; depth < smax && !beam.empty(); ++depth) {  // cst.cpp:196-221
      std::vector<Path> pool;
      for (Path& p : beam) {
        const Window* w = find(p.ctx.data(), p.ctx.size());
        ++S.expansions;
        S.children += static_cast<int64_t>(w->next.size());
        S.child_sectors += (8 * static_cast<int64_t>(w->next.size()) + 31) / 32;
        bool grew = false;
        for (int32_t t : w->next) {
          Seq c = p.ctx;
          c.push_back(t);
          const int64_t cnt = find(c.data(), c.size())->count;
          const double step = static_cast<double>(cnt) / static_cast<double>(w->count);
          if (step < a.min_step_freq || cnt < a.min_support) continue;
          Path q{std::move(c), p.score * step, cnt, p.toks};
          q.toks.push_back(t);
          pool.push_back(std::move(q));
          grew = true;
        }
        // a path is final only when it has no qualifying child (cst.cpp:213-214)
        if (!grew && !p.toks.empty()) finals.push_back(Cand{p.toks, p.score, p.support});
      }
      if (static_cast<int>(pool.size()) > a.top_k) {  // cst.cpp:216-219
        std::sort(pool.begin(), pool.end(), pbefore);
        pool.resize(static_cast<size_t>(a.top_k));
      }
      beam.swap(pool);
    }
    for (Path& p : beam)
      if (!p.toks.empty()) finals.push_back(Cand{p.toks, p.score, p.support});
    std::sort(finals.begin(), finals.end(), before);  // cst.cpp:225-227
    if (static_cast<int>(finals.size()) > a.top_k) finals.resize(static_cast<size_t>(a.top_k));
    S.cands = static_cast<int64_t>(finals.size());
    for (const auto& f : finals) S.cand_tokens += static_cast<int64_t>(f.toks.size());
    return finals;
  }
};

// speculate_oracle (cst.cpp:386-453): brute-force rescans of explicit sequences.
int64_t count_occ(const std::vector<Seq>& seqs, const Seq& w) {  // scan_count, cst.cpp:336-352
  int64_t n = 0;
  for (const Seq& s : seqs)
    for (size_t i = 0; i + w.size() <= s.size(); ++i)
      if (std::equal(w.begin(), w.end(), s.begin() + static_cast<long>(i))) ++n;
  return n;
}

std::vector<std::pair<int32_t, int64_t>> continuations(const std::vector<Seq>& seqs, const Seq& w) {
  std::vector<std::pair<int32_t, int64_t>> out;  // scan_continuations, cst.cpp:355-382
  for (const Seq& s : seqs)
    for (size_t i = 0; i + w.size() + 1 <= s.size(); ++i) {
      if (!std::equal(w.begin(), w.end(), s.begin() + static_cast<long>(i))) continue;
      int32_t t = s[i + w.size()];
      auto it = std::find_if(out.begin(), out.end(), [&](auto& e) { return e.first == t; });
      if (it == out.end())
        out.emplace_back(t, 1);
      else
        ++it->second;
    }
  return out;
}

std::vector<Cand> brute(const std::vector<Seq>& seqs, const int32_t* pat, size_t plen, const orc_args& a) {
  check_args(a);
  if (plen == 0) return {};
  Seq m;
  int64_t mc = 0;
  for (int len = std::min<int>(a.pattern_lookup_max, static_cast<int>(plen)); len >= a.pattern_lookup_min; --len) {
    Seq suf(pat + (plen - len), pat + plen);
    int64_t n = count_occ(seqs, suf);
    if (n > 0) {
      m = suf;
      mc = n;
      break;
    }
  }
  if (mc == 0) return {};
  struct P {
    Seq ctx;
    double score;
    int64_t support;
    Seq toks;
  };
  std::vector<P> beam{P{m, 1.0, mc, {}}};
  std::vector<Cand> finals;
  for (int d = 0; d < a.max_spec_tokens && !beam.empty(); ++d) {
    std::vector<P> pool;
    for (P& p : beam) {
      bool grew = false;
      for (auto [t, cnt] : continuations(seqs, p.ctx)) {
        double step = static_cast<double>(cnt) / static_cast<double>(p.support);
        if (step < a.min_step_freq || cnt < a.min_support) continue;
        P q{p.ctx, p.score * step, cnt, p.toks};
        q.ctx.push_back(t);
        q.toks.push_back(t);
        pool.push_back(std::move(q));
        grew = true;
      }
      if (!grew && !p.toks.empty()) finals.push_back(Cand{p.toks, p.score, p.support});
    }
    if (static_cast<int>(pool.size()) > a.top_k) {
      std::sort(pool.begin(), pool.end(), [](const P& x, const P& y) {
        return before(Cand{x.toks, x.score, x.support}, Cand{y.toks, y.score, y.support});
      });
      pool.resize(static_cast<size_t>(a.top_k));
    }
    beam.swap(pool);
  }
  for (P& p : beam)
    if (!p.toks.empty()) finals.push_back(Cand{p.toks, p.score, p.support});
  std::sort(finals.begin(), finals.end(), before);
  if (static_cast<int>(finals.size()) > a.top_k) finals.resize(static_cast<size_t>(a.top_k));
  return finals;
}

int emit(const std::vector<Cand>& c, orc_cands* out) {
  out->n = 0;
  for (const Cand& d : c) {
    if (out->n >= out->k_cap || static_cast<int>(d.toks.size()) > out->s_cap) {
      g_err = "candidate buffer too small";
      return -1;
    }
    const int i = out->n++;
    std::memcpy(out->tokens + static_cast<size_t>(i) * out->s_cap, d.toks.data(), d.toks.size() * 4);
    out->lens[i] = static_cast<int32_t>(d.toks.size());
    out->scores[i] = d.score;
    out->supports[i] = d.support;
  }
  return 0;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

void* orc_index_new(const char*, int32_t max_pattern_len, int32_t max_spec_len) {
  if (max_pattern_len < 1 || max_spec_len < 0) {  // cst.cpp:79-84
    g_err = "draft index limits out of range";
    return nullptr;
  }
  auto* ix = new Index;
  ix->lim_pattern = max_pattern_len;
  ix->lim_spec = max_spec_len;
  return ix;
}

void orc_index_free(void* idx) { delete static_cast<Index*>(idx); }

int orc_index_append(void* idx, int32_t rid, uint64_t prev, const int32_t* toks, uint64_t n, int32_t* ok,
                     uint64_t* version, uint64_t* acked) {
  return guarded([&] {
    static_cast<Index*>(idx)->append(rid, prev, toks, n, ok, version, acked);
    return 0;
  });
}

int orc_index_speculate(const void* idx, const int32_t* pat, uint64_t plen, const orc_args* args, orc_cands* out) {
  return guarded([&] { return emit(static_cast<const Index*>(idx)->speculate(pat, plen, *args, nullptr), out); });
}

int orc_index_speculate_stats(const void* idx, const int32_t* pat, uint64_t plen, const orc_args* args,
                              orc_cands* out, orc_qstats* stats) {
  return guarded([&] { return emit(static_cast<const Index*>(idx)->speculate(pat, plen, *args, stats), out); });
}

uint64_t orc_index_version(const void* idx) { return static_cast<const Index*>(idx)->version; }
uint64_t orc_index_node_count(const void* idx) {
  return static_cast<const Index*>(idx)->windows.size() + 1;  // + root, as nodes_.size() (cst.cpp:83)
}
uint64_t orc_index_stored_tokens(const void* idx, int32_t rid) {
  const auto& m = static_cast<const Index*>(idx)->streams;
  auto it = m.find(rid);
  return it == m.end() ? 0 : it->second.size();
}

int orc_oracle_speculate(const int32_t* toks, const uint64_t* offsets, uint64_t nseq, const int32_t* pat,
                         uint64_t plen, const orc_args* args, orc_cands* out) {
  return guarded([&] {
    std::vector<Seq> seqs(nseq);
    for (uint64_t i = 0; i < nseq; ++i) seqs[i].assign(toks + offsets[i], toks + offsets[i + 1]);
    return emit(brute(seqs, pat, plen, *args), out);
  });
}

// Verification + draft length (proj/src/engine.cpp:78-85 and :115-143).
int32_t orc_draft_len(int32_t sd_enabled, int32_t adaptive, int32_t cap, int32_t budget, int32_t n_running) {
  if (!sd_enabled) return 0;
  int32_t d = adaptive ? std::min(cap, budget / n_running) : cap;
  return std::max(d, 0);
}

void orc_verify(const int32_t* cand_tokens, const int32_t* cand_lens, int32_t ncand, int32_t s_cap,
                const int32_t* truth_next, int32_t truth_left, int32_t limit, int32_t* drafted, int32_t* accepted,
                int32_t* emitted) {
  int32_t dr = 0, acc = 0;
  for (int32_t c = 0; c < ncand; ++c) {
    dr += cand_lens[c];
    int32_t cap = std::min(cand_lens[c], truth_left);
    int32_t m = 0;
    while (m < cap && cand_tokens[static_cast<size_t>(c) * s_cap + m] == truth_next[m]) ++m;
    acc = std::max(acc, m);
  }
  const int32_t em = std::min(acc + 1, limit);
  *drafted = dr;
  *accepted = em - 1;
  *emitted = em;
}

}  // extern "C"
