// host_query.cpp — the query paths of the server: host-buffer batches (staged on the
// host workers behind dgds_speculate_submit, two result slots, compaction + PCIe copy-out
// into mapped pinned memory), the device / record / segmented / zero-copy engine APIs,
// reply-record compaction, and host-buffer verification (cst.cpp:153-228, engine.cpp:115-143).
#include "server_internal.h"

namespace {
// K2a -> K2b queue of queries whose locus is a node: one entry per query of the launch.
int set_cplx(dgds_server* s, dgds::QueryLaunch& L) {
  if (int rc = s->d_cplx.ensure(std::max<int64_t>(1, L.n) * sizeof(dgds::CplxRec))) return rc;
  L.cplx = static_cast<dgds::CplxRec*>(s->d_cplx.p);
  L.cplx_count = s->d_cplx_count;
  return DGDS_OK;
}
}  // namespace

namespace dgds_host {

// One host-buffer query batch: its results live in the mapped pinned block of its slot
// (valid until the batch submitted kQSlots later reuses the slot).
struct HostResult {
  int64_t n = 0, ncand = 0, ntok = 0;
  const int64_t* cand_off = nullptr;  // [n + 1]
  const dgds::CandMeta* meta = nullptr;  // [ncand], candidate_before order within a query
  const int64_t* tok_off = nullptr;   // [ncand + 1]
  const int32_t* tokens = nullptr;    // [ntok]
  const int32_t* verify = nullptr;    // [3][n] drafted | accepted | emitted, or null
};

// Stage queries [j0, j1) of chunk b (chunk-relative) into its pinned block: pattern rows are
// built in cache, then streamed out with non-temporal stores. With idx, query i of the batch
// reads row idx[i] of the caller's pattern / truth / limit arrays (a cluster owner's share of
// a batch, staged without an intermediate gather); handles are always the batch's own.
// Returns the first query of the range with a bad handle (>= ng) or decreasing offsets, or -1.
int64_t stage_rows(const QInBlock& b, char* hb, int64_t j0, int64_t j1, int32_t P, int64_t ng, const int32_t* handles,
                   const int64_t* idx, const uint64_t* pat_offs, const int32_t* patterns, const int32_t* truth,
                   int32_t truth_stride, const int32_t* truth_left, const int32_t* limit, bool verify) {
  if (j0 >= j1) return -1;
  int64_t bad = -1;
  const int64_t q0 = b.q0 + j0, m = j1 - j0;
  int32_t* hl = reinterpret_cast<int32_t*>(hb + b.o_len);
  int32_t* hp = reinterpret_cast<int32_t*>(hb + b.o_pat);
  thread_local std::vector<int32_t> lens, rows, tr, tl, lm;
  lens.resize(m);
  rows.assign(static_cast<size_t>(m) * P, 0);
  for (int64_t j = j0; j < j1; ++j) {
    const int64_t i = b.q0 + j, r = idx ? idx[i] : i;
    const int32_t hd = handles[i];
    if ((hd < 0 || hd >= ng || pat_offs[r + 1] < pat_offs[r]) && bad < 0) bad = i;
    const uint64_t L = pat_offs[r + 1] - pat_offs[r];
    lens[j - j0] = static_cast<int32_t>(std::min<uint64_t>(L, 0x7FFFFFFF));
    const uint64_t keep = std::min<uint64_t>(L, static_cast<uint64_t>(P));
    const int32_t* src = patterns + pat_offs[r + 1] - keep;
    int32_t* dst = rows.data() + (j - j0) * P;
    for (uint64_t k = 0; k < keep; ++k) dst[k] = src[k];
  }
  nt_copy(hl + j0, lens.data(), m * 4);
  nt_copy(hp + j0 * P, rows.data(), rows.size() * 4);
  nt_copy(hb + j0 * 4, handles + q0, m * 4);
  if (verify) {
    const int32_t *vtr = truth + q0 * truth_stride, *vtl = truth_left + q0, *vlm = limit + q0;
    if (idx) {
      tr.resize(static_cast<size_t>(m) * truth_stride);
      tl.resize(m);
      lm.resize(m);
      for (int64_t j = 0; j < m; ++j) {
        const int64_t r = idx[q0 + j];
        std::memcpy(tr.data() + j * truth_stride, truth + r * truth_stride, truth_stride * 4);
        tl[j] = truth_left[r];
        lm[j] = limit[r];
      }
      vtr = tr.data();
      vtl = tl.data();
      vlm = lm.data();
    }
    nt_copy(hb + b.o_tr + static_cast<size_t>(j0) * truth_stride * 4, vtr, static_cast<size_t>(m) * truth_stride * 4);
    nt_copy(hb + b.o_tl + j0 * 4, vtl, m * 4);
    nt_copy(hb + b.o_lm + j0 * 4, vlm, m * 4);
  }
  _mm_sfence();  // streaming stores globally visible before the copy is issued
  return bad;
}

// Issue the H2D of every chunk of the pending batch (from the worker that staged last).
// The batch's H2D, one copy per chunk block (per-row copies queued by each stager measured
// slower: many small copies from several threads), from the worker that staged last; then the
// per-chunk events the query launches wait on.
cudaError_t issue_h2d(dgds_server* s) {
  dgds_server::PendingQuery& pq = s->pq;
  dgds_server::QSlot& slot = s->qslot[pq.ticket % dgds_server::kQSlots];
  char* h = static_cast<char*>(slot.hq.p);
  char* d = static_cast<char*>(slot.dq.p);
  cudaError_t e = cudaSetDevice(s->p.device);
  for (int c = 0; c < pq.nch && e == cudaSuccess; ++c) {
    const QInBlock& b = pq.blk[c];
    if (s->h2d_kernel) {  // the GPU pulls the mapped staging block
      dgds::CopyOutRegions Rin{};
      Rin.n = 1;
      Rin.total_idx[0] = -1;
      Rin.begin_idx[0] = -1;
      Rin.fixed_bytes[0] = static_cast<int64_t>(b.bytes);
      Rin.src[0] = h + b.base;
      Rin.dst[0] = d + b.base;
      // a narrow grid: enough reads in flight for PCIe, SMs left to the append kernel running beside it
      e = dgds::launch_copy_out(nullptr, Rin, Rin.fixed_bytes[0], s->copy_st, s->h2d_blocks);
    } else {
      e = cudaMemcpyAsync(d + b.base, h + b.base, b.bytes, cudaMemcpyHostToDevice, s->copy_st);
    }
    if (e == cudaSuccess) e = cudaEventRecord(s->ev_h2d[c], s->copy_st);
  }
  return e;
}

// Check the arguments, then stage (and validate handles / offsets) on the worker pool without
// waiting: the caller's next host work (typically the next tick's dgds_update_batch planning)
// overlaps the staging. The worker that stages last issues the H2D and launches the kernels;
// any later call that touches the device first joins it (flush_pending), so every batch sees
// exactly the updates launched before it. Caller holds s->mu.
int speculate_submit(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                     const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride, const int32_t* truth,
                     int32_t truth_stride, const int32_t* truth_left, const int32_t* limit, bool verify,
                     uint64_t* ticket, const int64_t* idx = nullptr) {
  PhaseClock pc("speculate_submit");
  if (int rc = flush_pending(s)) return rc;
  const int64_t nargs = args_stride ? n : 1;
  int32_t max_k = 1, max_s = 1;
  for (int64_t i = 0; i < nargs; ++i) {
    const dgds_spec_args& a = args[(idx && args_stride ? idx[i] : i) * args_stride];
    if (int rc = check_args(a)) return rc;
    max_k = std::max(max_k, a.top_k);
    max_s = std::max(max_s, std::min(a.max_spec_tokens, s->p.max_spec_len));
  }
  if (verify && (!truth || !truth_left || !limit || truth_stride < 0))
    return fail(DGDS_EINVAL, "verify needs truth inputs");
  pc.mark("args");
  const int32_t P = s->p.max_pattern_len;  // only the last max_pattern_len tokens can matter
  dgds_server::PendingQuery& pq = s->pq;
  // optional chunks of the batch (DGDS_Q_CHUNKS): chunk c's copy-out beside chunk c+1's query
  int nch = n >= 32768 ? s->q_chunks : 1;
  const int64_t per = static_cast<int64_t>(align_up((n + nch - 1) / nch, 256));
  nch = static_cast<int>((n + per - 1) / per);
  size_t in_all = 0;
  for (int c = 0; c < nch; ++c) {  // per-chunk block: handles | pat_len | patterns | args | truth | truth_left | limit
    QInBlock& b = pq.blk[c];
    b.q0 = c * per;
    b.m = std::min<int64_t>(per, n - b.q0);
    b.base = in_all;
    b.o_len = align_up(b.m * 4, 256);
    b.o_pat = align_up(b.o_len + b.m * 4, 256);
    b.o_args = align_up(b.o_pat + static_cast<size_t>(b.m) * P * 4, 256);
    b.o_tr = align_up(b.o_args + (args_stride ? b.m : 1) * sizeof(dgds_spec_args), 256);
    b.o_tl = align_up(b.o_tr + (verify ? static_cast<size_t>(b.m) * truth_stride * 4 : 0), 256);
    b.o_lm = align_up(b.o_tl + (verify ? b.m * 4 : 0), 256);
    b.bytes = align_up(b.o_lm + (verify ? b.m * 4 : 0), 16);  // the copy-in kernel moves 16-B units
    in_all = align_up(b.base + b.bytes, 256);
  }
  const uint64_t tk = s->last_ticket + 1;
  dgds_server::QSlot& slot = s->qslot[tk % dgds_server::kQSlots];
  DGDS_CUDA(cudaEventSynchronize(slot.done));  // the slot's previous batch is complete
  slot.ticket = 0;  // its results are gone from here on
  pc.mark("slot_wait");
  // device outputs (internal strides) + compaction scratch; mapped result block
  const int32_t K = max_k, Sx = max_s;
  const int64_t nk = static_cast<int64_t>(n) * K;
  QOutLayout& o = pq.out;
  o.sc = 0;
  o.sp = align_up(o.sc + nk * 8, 256);
  o.nc = align_up(o.sp + nk * 8, 256);
  o.ln = align_up(o.nc + n * 4, 256);
  o.tk = align_up(o.ln + nk * 4, 256);
  o.v = align_up(o.tk + static_cast<size_t>(nk) * Sx * 4, 256);
  o.bs = align_up(o.v + (verify ? static_cast<size_t>(n) * 12 : 0), 256);
  o.tot = align_up(o.bs + static_cast<size_t>((per + 255) / 256) * 16, 256);
  o.cmeta = align_up(o.tot + static_cast<size_t>(nch) * 16, 256);
  o.ctoff = align_up(o.cmeta + nk * sizeof(dgds::CandMeta), 256);
  o.ccoff = align_up(o.ctoff + nk * 8, 256);
  o.ctok = align_up(o.ccoff + (n + 1) * 8, 256);
  const size_t dev_total = o.ctok + static_cast<size_t>(nk) * Sx * 4;
  slot.h_coff = 256;  // totals | cand_off | verify | meta | tok_off | tokens
  slot.h_v = align_up(slot.h_coff + (n + 1) * 8, 256);
  slot.h_meta = align_up(slot.h_v + (verify ? n * 12 : 0), 256);
  slot.h_toff = align_up(slot.h_meta + nk * sizeof(dgds::CandMeta), 256);
  slot.h_tok = align_up(slot.h_toff + (nk + 1) * 8, 256);
  if (int rc = slot.hq.ensure(in_all)) return rc;
  if (int rc = slot.dq.ensure(in_all)) return rc;
  if (int rc = slot.dout.ensure(dev_total)) return rc;
  if (int rc = slot.ho.ensure(slot.h_tok + static_cast<size_t>(nk) * Sx * 4)) return rc;
  char* h = static_cast<char*>(slot.hq.p);
  for (int c = 0; c < nch; ++c) {  // args: tiny, copied here
    const QInBlock& b = pq.blk[c];
    auto* ha = reinterpret_cast<dgds_spec_args*>(h + b.base + b.o_args);
    if (!args_stride) ha[0] = args[0];
    else
      for (int64_t j = 0; j < b.m; ++j) ha[j] = args[(idx ? idx[b.q0 + j] : b.q0 + j) * args_stride];
  }
  pq.n = n;
  pq.nch = nch;
  pq.K = K;
  pq.Sx = Sx;
  pq.args_stride = args_stride;
  pq.truth_stride = truth_stride;
  pq.verify = verify;
  pq.ticket = tk;
  pq.h2d_err = cudaSuccess;
  pq.handles = handles;
  pq.ng = static_cast<int64_t>(s->groups.size());
  pq.stager_launch = !s->profiling;  // LaunchTimer state belongs to the caller's thread
  pq.launched = false;
  pq.launch_rc = DGDS_OK;
  slot.ticket = tk;
  slot.err = DGDS_OK;
  slot.n = n;
  slot.verify = verify;
  s->last_ticket = tk;
  *ticket = tk;
  // stage (and validate) on the workers; tasks cover [0, n) and split at chunk boundaries. An
  // asynchronous stage uses a few workers: it overlaps the caller's next host work, which
  // would otherwise be starved of memory bandwidth.
  WorkerPool& pool = s->workers();
  const bool async = s->async_stage && n >= 8192 && pool.threads() > 1;
  const int tasks = n < 8192 ? 1 : async ? std::min(s->stage_tasks, pool.threads() - 1) : 4 * pool.threads();
  const int64_t span = (n + tasks - 1) / tasks;
  const int64_t ng = static_cast<int64_t>(s->groups.size());
  pq.left.store(tasks);
  pq.bad.store(INT64_MAX);
  auto job = [s, h, span, n, per, P, ng, handles, idx, pat_offs, patterns, truth, truth_stride, truth_left, limit,
              verify](int t) {
    const int64_t i0 = t * span, i1 = std::min<int64_t>(n, i0 + span);
    int64_t first_bad = INT64_MAX;
    for (int64_t i = i0; i < i1;) {
      const int c = static_cast<int>(i / per);
      const QInBlock& b = s->pq.blk[c];
      const int64_t e = std::min<int64_t>(i1, b.q0 + b.m);
      const int64_t bad = stage_rows(b, h + b.base, i - b.q0, e - b.q0, P, ng, handles, idx, pat_offs, patterns, truth,
                                     truth_stride, truth_left, limit, verify);
      if (bad >= 0 && bad < first_bad) first_bad = bad;
      i = e;
    }
    if (first_bad != INT64_MAX) {
      int64_t cur = s->pq.bad.load();
      while (first_bad < cur && !s->pq.bad.compare_exchange_weak(cur, first_bad)) {
      }
    }
    if (s->pq.left.fetch_sub(1) == 1 && s->pq.bad.load() == INT64_MAX) {  // the last stager
      PhaseClock lpc("stager_launch");
      dgds_server::PendingQuery& q = s->pq;  // (nothing is launched for an invalid batch)
      if (q.h2d_err == cudaSuccess) q.h2d_err = issue_h2d(s);
      lpc.mark("h2d");
      if (q.h2d_err == cudaSuccess && q.stager_launch) {
        q.launch_rc = launch_batch(s, false);
        lpc.mark("launch");
        if (q.launch_rc) q.launch_msg = dgds_last_error();
        q.launched = true;
      }
    }
  };
  pq.active = true;
  if (async) {
    pool.post(tasks, job);  // a bad handle / offset is reported by the batch's wait
  } else {
    pool.run(tasks, job);
    if (pq.bad.load() != INT64_MAX) {  // staged here: report at submit, nothing was queued
      const int64_t i = pq.bad.load();
      pq.active = false;
      slot.ticket = 0;
      s->last_ticket = tk - 1;
      if (int rc = check_handle(s, handles[i])) return rc;
      return fail(DGDS_EINVAL, "pattern offsets must be nondecreasing");
    }
  }
  pc.mark("post");
  return DGDS_OK;
}

// Launch a staged batch's kernels (its H2D issued): query (+ verify), compaction, copy-out.
// Run by the worker that staged last, or by flush_pending when that worker could not (profiling
// timers are main-thread state). Reads server state that every main-thread mutation of it
// (root table, index table, stream and history arrays) first flushes, i.e. joins the worker.
int launch_batch(dgds_server* s, bool timed) {
  dgds_server::PendingQuery& pq = s->pq;
  dgds_server::QSlot& slot = s->qslot[pq.ticket % dgds_server::kQSlots];
  const QOutLayout& o = pq.out;
  const int64_t n = pq.n;
  const int32_t K = pq.K, Sx = pq.Sx, P = s->p.max_pattern_len;
  const bool verify = pq.verify;
  const int nch = pq.nch;
  char* d = static_cast<char*>(slot.dq.p);
  char* dout = static_cast<char*>(slot.dout.p);
  char* ho = static_cast<char*>(slot.ho.p);
  long long* d_bs = reinterpret_cast<long long*>(dout + o.bs);
  long long* d_tot = reinterpret_cast<long long*>(dout + o.tot);  // [chunk][candidates, tokens], cumulative
  auto* d_meta = reinterpret_cast<dgds::CandMeta*>(dout + o.cmeta);
  auto* d_toff = reinterpret_cast<int64_t*>(dout + o.ctoff);
  auto* d_coff = reinterpret_cast<int64_t*>(dout + o.ccoff);
  int32_t* d_ctok = reinterpret_cast<int32_t*>(dout + o.ctok);
  int32_t* d_v = reinterpret_cast<int32_t*>(dout + o.v);
  for (int c = 0; c < nch; ++c) {
    const QInBlock& b = pq.blk[c];
    const char* db = d + b.base;
    const int64_t q0 = b.q0, m = b.m;
    DGDS_CUDA(cudaStreamWaitEvent(s->st, s->ev_h2d[c], 0));
    dgds::QueryLaunch L{};
    L.T = s->T;
    L.root_of = s->d_root_of;
    L.n_handles = static_cast<int32_t>(s->root_of_cap);
    L.n = m;
    L.handles = reinterpret_cast<const int32_t*>(db);
    L.pat_len = reinterpret_cast<const int32_t*>(db + b.o_len);
    L.patterns = reinterpret_cast<const int32_t*>(db + b.o_pat);
    L.pat_stride = P;
    L.args = reinterpret_cast<const dgds_spec_args*>(db + b.o_args);
    L.args_stride = pq.args_stride ? 1 : 0;
    L.k_stride = K;
    L.s_stride = Sx;
    dgds::soa_strides(L);
    L.scores = reinterpret_cast<double*>(dout + o.sc) + q0 * K;
    L.supports = reinterpret_cast<int64_t*>(dout + o.sp) + q0 * K;
    L.n_cands = reinterpret_cast<int32_t*>(dout + o.nc) + q0;
    L.lens = reinterpret_cast<int32_t*>(dout + o.ln) + q0 * K;
    L.tokens = reinterpret_cast<int32_t*>(dout + o.tk) + q0 * K * Sx;
    L.err_flag = s->d_err;
    L.stat_part = s->d_stat_part;
  if (int rc = set_cplx(s, L)) return rc;
    if (verify) {
      L.truth = reinterpret_cast<const int32_t*>(db + b.o_tr);
      L.truth_stride = pq.truth_stride;
      L.truth_left = reinterpret_cast<const int32_t*>(db + b.o_tl);
      L.limit = reinterpret_cast<const int32_t*>(db + b.o_lm);
      L.v_drafted = d_v + q0;
      L.v_accepted = d_v + n + q0;
      L.v_emitted = d_v + 2 * n + q0;
    }
    if (timed) {
      LaunchTimer lt(s, 1, s->st);
      DGDS_CUDA(dgds::launch_query(L, K, Sx, s->st));
    } else {
      DGDS_CUDA(dgds::launch_query(L, K, Sx, s->st));
    }
    DGDS_CUDA(dgds::launch_compact(m, K, Sx, L.n_cands, L.lens, L.scores, L.supports, L.tokens, d_bs, d_tot + 2 * c,
                                   d_meta, d_ctok, d_coff + q0, d_toff, c ? d_tot + 2 * (c - 1) : nullptr, s->st));
    DGDS_CUDA(cudaEventRecord(s->ev_cmp[c], s->st));
    DGDS_CUDA(cudaStreamWaitEvent(s->out_st, s->ev_cmp[c], 0));
    dgds::CopyOutRegions R{};
    auto region = [&](const void* src, char* dst, int tot, int begin, int elem, int64_t fixed) {
      const int i = R.n++;
      R.src[i] = static_cast<const char*>(src);
      R.dst[i] = dst;
      R.total_idx[i] = tot;
      R.begin_idx[i] = begin;
      R.elem_bytes[i] = elem;
      R.fixed_bytes[i] = fixed;
    };
    const int tc = 2 * c, tb = c ? 2 * (c - 1) : -1;
    region(d_coff + q0, ho + slot.h_coff + q0 * 8, -1, -1, 0, m * 8);
    if (verify)
      for (int k = 0; k < 3; ++k)
        region(d_v + k * n + q0, ho + slot.h_v + (k * n + q0) * 4, -1, -1, 0, m * 4);
    region(d_meta, ho + slot.h_meta, tc, tb, sizeof(dgds::CandMeta), 0);
    region(d_toff, ho + slot.h_toff, tc, tb, 8, 0);
    region(d_ctok, ho + slot.h_tok, tc + 1, c ? tb + 1 : -1, 4, 0);
    if (c == nch - 1) region(d_tot + tc, ho, -1, -1, 0, 16);
    DGDS_CUDA(dgds::launch_copy_out(d_tot, R, m * K * static_cast<int64_t>(sizeof(dgds::CandMeta) + 8 + Sx * 4),
                                    s->out_st, nch > 1 ? s->out_blocks : 592));
  }
  DGDS_CUDA(cudaEventRecord(slot.done, s->out_st));  // after st's work (out_st waited on it)
  return DGDS_OK;
}

// Completes the pending batch: joins its staging workers and, unless the last of them did,
// launches its kernels. Runs before any later call on the server touches the device.
// Caller holds s->mu.
int flush_pending(dgds_server* s) {
  dgds_server::PendingQuery& pq = s->pq;
  if (!pq.active) return DGDS_OK;
  PhaseClock pc("flush_pending");
  s->workers().join();
  pq.active = false;
  pc.mark("join");
  dgds_server::QSlot& slot = s->qslot[pq.ticket % dgds_server::kQSlots];
  if (pq.bad.load() != INT64_MAX) {  // reported by the batch's wait, not by the call that flushed
    const int64_t i = pq.bad.load();
    const int32_t hd = pq.handles[i];
    slot.err = DGDS_EINVAL;
    slot.err_msg = (hd < 0 || hd >= pq.ng) ? "bad group handle" : "pattern offsets must be nondecreasing";
    return DGDS_OK;
  }
  if (pq.h2d_err.load() != cudaSuccess) return fail(DGDS_ECUDA, cudaGetErrorString(pq.h2d_err.load()));
  if (pq.launched) {
    if (pq.launch_rc) return fail(pq.launch_rc, pq.launch_msg);
    return DGDS_OK;
  }
  const int rc = launch_batch(s, true);
  pc.mark("launch");
  return rc;
}

// Waits for a submitted batch and describes its results. Caller holds s->mu.
int speculate_finish(dgds_server* s, uint64_t ticket, HostResult* r) {
  if (ticket == 0 || ticket > s->last_ticket) return fail(DGDS_EINVAL, "unknown query ticket");
  if (s->pq.active && s->pq.ticket == ticket)  // waiting on the batch still being staged
    if (int rc = flush_pending(s)) return rc;
  {
    const dgds_server::QSlot& sl = s->qslot[ticket % dgds_server::kQSlots];
    if (sl.ticket == ticket && sl.err) return fail(sl.err, sl.err_msg);
  }
  dgds_server::QSlot& slot = s->qslot[ticket % dgds_server::kQSlots];
  if (slot.ticket != ticket) return fail(DGDS_EINVAL, "query ticket expired (its result slot was reused)");
  DGDS_CUDA(cudaEventSynchronize(slot.done));
  char* ho = static_cast<char*>(slot.ho.p);
  const int64_t n = slot.n;
  r->n = n;
  r->ncand = reinterpret_cast<const long long*>(ho)[0];
  r->ntok = reinterpret_cast<const long long*>(ho)[1];
  auto* coff = reinterpret_cast<int64_t*>(ho + slot.h_coff);
  auto* toff = reinterpret_cast<int64_t*>(ho + slot.h_toff);
  coff[n] = r->ncand;
  toff[r->ncand] = r->ntok;
  r->cand_off = coff;
  r->meta = reinterpret_cast<const dgds::CandMeta*>(ho + slot.h_meta);
  r->tok_off = toff;
  r->tokens = reinterpret_cast<const int32_t*>(ho + slot.h_tok);
  r->verify = slot.verify ? reinterpret_cast<const int32_t*>(ho + slot.h_v) : nullptr;
  s->last_d2h_bytes =
      16 + (n + 1) * 8 + (slot.verify ? n * 12 : 0) + r->ncand * (sizeof(dgds::CandMeta) + 8) + r->ntok * 4;
  return DGDS_OK;
}

int speculate_host(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                   const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride, const int32_t* truth,
                   int32_t truth_stride, const int32_t* truth_left, const int32_t* limit, bool verify,
                   HostResult* r, const int64_t* idx = nullptr) {
  uint64_t t = 0;
  if (int rc = speculate_submit(s, n, handles, pat_offs, patterns, args, args_stride, truth, truth_stride,
                                truth_left, limit, verify, &t, idx))
    return rc;
  PhaseClock pc("speculate_wait");
  return speculate_finish(s, t, r);
}

void fill_view(const HostResult& r, dgds_result_view* out);

// dgds_speculate_verify_view over rows idx[0..n) of the caller's arrays (handles: n server
// handles, one per query): a cluster owner's share of a batch (cluster.cpp).
int speculate_view_indexed(dgds_server* s, int64_t n, const int64_t* idx, const int32_t* handles,
                           const uint64_t* pat_offs, const int32_t* patterns, const dgds_spec_args* args,
                           int64_t args_stride, const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                           const int32_t* limit, dgds_result_view* out) {
  *out = dgds_result_view{};
  if (n == 0) return DGDS_OK;
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc = flush_pending(s)) return rc;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  HostResult r;
  if (int rc = speculate_host(s, n, handles, pat_offs, patterns, args, args_stride, truth, truth_stride, truth_left,
                              limit, truth != nullptr, &r, idx))
    return rc;
  fill_view(r, out);
  return DGDS_OK;
}

void fill_view(const HostResult& r, dgds_result_view* out) {
  out->n_queries = r.n;
  out->n_cands = r.ncand;
  out->n_tokens = r.ntok;
  out->cand_off = r.cand_off;
  out->cands = reinterpret_cast<const dgds_cand_meta*>(r.meta);
  out->tok_off = r.tok_off;
  out->tokens = r.tokens;
  if (r.verify) {
    out->drafted = r.verify;
    out->accepted = r.verify + r.n;
    out->emitted = r.verify + 2 * r.n;
  }
}

static int speculate_records_impl(dgds_server* s, int64_t n, const int32_t* d_records,
                                  const dgds_query_record_layout* lay, const dgds_spec_args* d_args,
                                  int64_t args_stride, int32_t max_top_k, int32_t max_spec, int32_t* d_replies,
                                  int32_t n_seg, int64_t seg_rows, const int32_t* d_seg_count,
                                  int32_t* const* seg_out, int32_t origin_field, dgds_query_stats* d_stats,
                                  void* stream) {
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (n == 0) return DGDS_OK;
  if (!lay || !d_records || !d_args || (!d_replies && !seg_out)) return fail(DGDS_EINVAL, "null argument");
  if (max_top_k < 1 || max_top_k > DGDS_MAX_TOP_K) return fail(DGDS_EUNSUPPORTED, "max_top_k out of range");
  if (max_spec <= 0 || max_spec > s->p.max_spec_len) max_spec = std::max(1, s->p.max_spec_len);
  const dgds_query_record_layout& y = *lay;
  if (y.rec_words < 1 || y.reply_words < 1 || (y.reply_words & 1) || (y.off_scores & 1) || (y.off_supports & 1))
    return fail(DGDS_EINVAL, "bad record layout (reply words and 8-byte fields must be even)");
  if (y.rec_words - y.off_pattern < s->p.max_pattern_len)
    return fail(DGDS_EINVAL, "query record pattern field shorter than max_pattern_len");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  StreamJoin join(s, stream);
  dgds::QueryLaunch L{};
  L.T = s->T;
  L.root_of = s->d_root_of;
  L.n_handles = static_cast<int32_t>(s->root_of_cap);
  L.n = n;
  L.handles = d_records + y.off_handle;
  L.pat_len = d_records + y.off_pat_len;
  L.patterns = d_records + y.off_pattern;
  L.pat_stride = y.rec_words;
  L.args = d_args;
  L.args_stride = args_stride;
  L.k_stride = max_top_k;
  L.s_stride = max_spec;
  L.in_qstride = y.rec_words;
  L.rec_words_out = y.reply_words;
  L.rec_out = d_replies;
  if (seg_out) {
    L.seg_rows = seg_rows;
    L.seg_count = d_seg_count;
    if (origin_field >= 0) L.seg_origin = d_records + origin_field;
    for (int i = 0; i < n_seg; ++i) L.seg_out[i] = seg_out[i];
  }
  L.off_nc = y.off_n_cands;
  L.off_len = y.off_lens;
  L.off_sc = y.off_scores;
  L.off_sp = y.off_supports;
  L.off_tk = y.off_tokens;
  L.off_v = y.off_verify;
  if (y.off_verify >= 0) {
    L.truth = d_records + y.off_truth;
    L.truth_stride = y.rec_words;
    L.truth_left = d_records + y.off_truth_left;
    L.limit = d_records + y.off_limit;
  }
  L.stats = d_stats;
  L.err_flag = s->d_err;
  L.stat_part = s->d_stat_part;
  if (int rc = set_cplx(s, L)) return rc;
  L.dbg = s->d_dbg;
  {
    LaunchTimer lt(s, 1, join.stream());
    DGDS_CUDA(dgds::launch_query(L, max_top_k, max_spec, join.stream()));
  }
  return DGDS_OK;
}

}  // namespace dgds_host

using namespace dgds_host;

extern "C" {

int dgds_speculate_verify_batch(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                                const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride,
                                const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                                const int32_t* limit, dgds_candidates* out, dgds_verify_out* vout) {
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (n == 0) return DGDS_OK;
  if (!out) return fail(DGDS_EINVAL, "null output");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  {
    const int64_t nargs = args_stride ? n : 1;
    int32_t max_k = 1, max_s = 1;
    for (int64_t i = 0; i < nargs; ++i) {
      if (int rc = check_args(args[i * args_stride])) return rc;
      max_k = std::max(max_k, args[i * args_stride].top_k);
      max_s = std::max(max_s, std::min(args[i * args_stride].max_spec_tokens, s->p.max_spec_len));
    }
    if (out->k_stride < max_k || out->s_stride < max_s)
      return fail(DGDS_EBUFFER, "candidate buffer strides too small");
  }
  HostResult r;
  if (int rc = speculate_host(s, n, handles, pat_offs, patterns, args, args_stride, truth, truth_stride, truth_left,
                              limit, vout != nullptr, &r))
    return rc;
  PhaseClock pc("scatter");
  // scatter into the caller's strided buffers, in parallel chunks (per-query offsets are known)
  WorkerPool& pool = s->workers();
  const int tasks = n >= 8192 ? 4 * pool.threads() : 1;
  const int64_t chunk = (n + tasks - 1) / tasks;
  pool.run(tasks, [&](int t) {
    const int64_t q0 = t * chunk, q1 = std::min<int64_t>(n, q0 + chunk);
    for (int64_t q = q0; q < q1; ++q) {
      const int64_t c0 = r.cand_off[q], c1 = r.cand_off[q + 1];
      out->n_cands[q] = static_cast<int32_t>(c1 - c0);
      for (int64_t c = c0; c < c1; ++c) {
        const int64_t di = q * out->k_stride + (c - c0);
        const dgds::CandMeta& m = r.meta[c];
        out->lens[di] = m.len;
        out->scores[di] = m.score;
        out->supports[di] = m.support;
        std::memcpy(out->tokens + di * out->s_stride, r.tokens + r.tok_off[c], m.len * 4);
      }
    }
    if (vout && q0 < q1) {
      std::memcpy(vout->drafted + q0, r.verify + q0, (q1 - q0) * 4);
      std::memcpy(vout->accepted + q0, r.verify + n + q0, (q1 - q0) * 4);
      std::memcpy(vout->emitted + q0, r.verify + 2 * n + q0, (q1 - q0) * 4);
    }
  });
  return DGDS_OK;
}

int dgds_speculate_verify_view(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                               const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride,
                               const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                               const int32_t* limit, dgds_result_view* out) {
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (!out) return fail(DGDS_EINVAL, "null output");
  *out = dgds_result_view{};
  if (n == 0) return DGDS_OK;
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  HostResult r;
  if (int rc = speculate_host(s, n, handles, pat_offs, patterns, args, args_stride, truth, truth_stride, truth_left,
                              limit, truth != nullptr, &r))
    return rc;
  fill_view(r, out);
  return DGDS_OK;
}

int dgds_speculate_submit(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                          const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride,
                          const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                          const int32_t* limit, uint64_t* ticket) {
  if (!s || !ticket) return fail(DGDS_EINVAL, "null argument");
  if (n <= 0) return fail(DGDS_EINVAL, "submit needs a non-empty batch");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  return speculate_submit(s, n, handles, pat_offs, patterns, args, args_stride, truth, truth_stride, truth_left,
                          limit, truth != nullptr, ticket);
}

int dgds_speculate_wait(dgds_server* s, uint64_t ticket, dgds_result_view* out) {
  if (!s || !out) return fail(DGDS_EINVAL, "null argument");
  *out = dgds_result_view{};
  std::lock_guard<std::mutex> lk(s->mu);
  // host state only: no flush
  DGDS_CUDA(cudaSetDevice(s->p.device));
  HostResult r;
  if (int rc = speculate_finish(s, ticket, &r)) return rc;
  fill_view(r, out);
  return DGDS_OK;
}

int dgds_replies_submit(dgds_server* s, int64_t n, const int32_t* d_replies, const dgds_query_record_layout* lay,
                        int32_t max_top_k, int32_t max_spec, void* stream, uint64_t* ticket) {
  if (!s || !lay || !d_replies || !ticket) return fail(DGDS_EINVAL, "null argument");
  if (n <= 0) return fail(DGDS_EINVAL, "submit needs a non-empty batch");
  if (max_top_k < 1 || max_top_k > DGDS_MAX_TOP_K) return fail(DGDS_EUNSUPPORTED, "max_top_k out of range");
  if (max_spec < 1) return fail(DGDS_EINVAL, "max_spec must be >= 1");
  const dgds_query_record_layout& y = *lay;
  if (y.reply_words < 1 || (y.reply_words & 1) || (y.off_scores & 1) || (y.off_supports & 1))
    return fail(DGDS_EINVAL, "bad record layout (reply words and 8-byte fields must be even)");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc = flush_pending(s)) return rc;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  StreamJoin join(s, stream);
  const cudaStream_t js = join.stream();
  const uint64_t tk = s->last_ticket + 1;
  dgds_server::QSlot& slot = s->qslot[tk % dgds_server::kQSlots];
  DGDS_CUDA(cudaEventSynchronize(slot.done));  // the slot's previous batch is complete
  slot.ticket = 0;
  const bool verify = y.off_verify >= 0;
  const int32_t K = max_top_k, Sx = max_spec;
  const int64_t nk = n * K;
  // device: block sums | totals | meta | tok_off | cand_off | tokens | verify [3][n]
  const int64_t nblk = (n + 255) / 256;
  const size_t o_bs = 0;
  const size_t o_tot = align_up(o_bs + static_cast<size_t>(nblk) * 16, 256);
  const size_t o_cmeta = align_up(o_tot + 16, 256);
  const size_t o_ctoff = align_up(o_cmeta + nk * sizeof(dgds::CandMeta), 256);
  const size_t o_ccoff = align_up(o_ctoff + nk * 8, 256);
  const size_t o_ctok = align_up(o_ccoff + (n + 1) * 8, 256);
  const size_t o_v = align_up(o_ctok + static_cast<size_t>(nk) * Sx * 4, 256);
  const size_t dev_total = o_v + (verify ? n * 12 : 0);
  slot.h_coff = 256;  // totals | cand_off | verify | meta | tok_off | tokens
  slot.h_v = align_up(slot.h_coff + (n + 1) * 8, 256);
  slot.h_meta = align_up(slot.h_v + (verify ? n * 12 : 0), 256);
  slot.h_toff = align_up(slot.h_meta + nk * sizeof(dgds::CandMeta), 256);
  slot.h_tok = align_up(slot.h_toff + (nk + 1) * 8, 256);
  if (int rc = slot.dout.ensure(dev_total)) return rc;
  if (int rc = slot.ho.ensure(slot.h_tok + static_cast<size_t>(nk) * Sx * 4)) return rc;
  char* dout = static_cast<char*>(slot.dout.p);
  char* ho = static_cast<char*>(slot.ho.p);
  long long* d_bs = reinterpret_cast<long long*>(dout + o_bs);
  long long* d_tot = reinterpret_cast<long long*>(dout + o_tot);
  auto* d_meta = reinterpret_cast<dgds::CandMeta*>(dout + o_cmeta);
  auto* d_toff = reinterpret_cast<int64_t*>(dout + o_ctoff);
  auto* d_coff = reinterpret_cast<int64_t*>(dout + o_ccoff);
  int32_t* d_ctok = reinterpret_cast<int32_t*>(dout + o_ctok);
  int32_t* d_v = reinterpret_cast<int32_t*>(dout + o_v);
  dgds::CmpIn in{};  // reply records: int32 fields at stride reply_words, 8-byte fields at reply_words / 2
  in.n_cands = d_replies + y.off_n_cands;
  in.qs_nc = y.reply_words;
  in.lens = d_replies + y.off_lens;
  in.qs_len = y.reply_words;
  in.scores = reinterpret_cast<const double*>(d_replies + y.off_scores);
  in.qs_sc = y.reply_words / 2;
  in.supports = reinterpret_cast<const int64_t*>(d_replies + y.off_supports);
  in.qs_sp = y.reply_words / 2;
  in.tokens = d_replies + y.off_tokens;
  in.qs_tok = y.reply_words;
  in.cs_tok = max_spec;
  in.verify = verify ? d_replies + y.off_verify : nullptr;
  in.qs_v = y.reply_words;
  DGDS_CUDA(dgds::launch_compact_in(n, in, d_bs, d_tot, d_meta, d_ctok, d_coff, d_toff, verify ? d_v : nullptr,
                                    nullptr, js));
  // the copy-out (PCIe-bound) runs on out_st, so the caller's stream moves on
  DGDS_CUDA(cudaEventRecord(s->ev_cmp[0], js));
  DGDS_CUDA(cudaStreamWaitEvent(s->out_st, s->ev_cmp[0], 0));
  dgds::CopyOutRegions R{};
  auto region = [&](const void* src, char* dst, int tot, int elem, int64_t fixed) {
    const int i = R.n++;
    R.src[i] = static_cast<const char*>(src);
    R.dst[i] = dst;
    R.total_idx[i] = tot;
    R.begin_idx[i] = -1;
    R.elem_bytes[i] = elem;
    R.fixed_bytes[i] = fixed;
  };
  region(d_coff, ho + slot.h_coff, -1, 0, n * 8);
  if (verify) region(d_v, ho + slot.h_v, -1, 0, n * 12);
  region(d_meta, ho + slot.h_meta, 0, sizeof(dgds::CandMeta), 0);
  region(d_toff, ho + slot.h_toff, 0, 8, 0);
  region(d_ctok, ho + slot.h_tok, 1, 4, 0);
  region(d_tot, ho, -1, 0, 16);
  DGDS_CUDA(dgds::launch_copy_out(d_tot, R, nk * static_cast<int64_t>(sizeof(dgds::CandMeta) + 8 + Sx * 4),
                                  s->out_st));
  DGDS_CUDA(cudaEventRecord(slot.done, s->out_st));
  slot.ticket = tk;
  slot.n = n;
  slot.verify = verify;
  slot.err = DGDS_OK;
  s->last_ticket = tk;
  *ticket = tk;
  return DGDS_OK;
}

int dgds_speculate_batch(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                         const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride,
                         dgds_candidates* out) {
  return dgds_speculate_verify_batch(s, n, handles, pat_offs, patterns, args, args_stride, nullptr, 0, nullptr,
                                     nullptr, out, nullptr);
}

int dgds_decode_step_device(dgds_server* s, int64_t n, const int32_t* d_handles, const int32_t* d_ctx,
                            int32_t ctx_stride, const int32_t* d_generated, const int32_t* d_limit,
                            const int32_t* d_truth, int32_t truth_stride, const int32_t* d_truth_left,
                            const dgds_spec_args* args, const dgds_spec_policy* policy,
                            const int32_t* d_draft_len, int32_t draft_len, const dgds_candidates* d_out,
                            const dgds_verify_out* d_vout, int32_t* d_next_draft_len, int64_t* d_totals,
                            void* stream) {
  if (!s || !args || !policy || !d_vout || !d_truth || !d_truth_left || !d_limit || !d_generated || !d_ctx ||
      !d_handles)
    return fail(DGDS_EINVAL, "null argument");
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (n == 0) return DGDS_OK;
  if (int rc = check_args(dgds_spec_args{0, args->pattern_lookup_max, args->pattern_lookup_min, 1,
                                         args->min_step_freq, args->min_support}))
    return rc;
  const int32_t k = std::max(1, policy->multi_path_k);
  if (k > DGDS_MAX_TOP_K) return fail(DGDS_EUNSUPPORTED, "multi_path_k above DGDS_MAX_TOP_K");
  if (ctx_stride < s->p.max_pattern_len) return fail(DGDS_EINVAL, "ctx_stride must be >= max_pattern_len");
  if (d_out && (d_out->k_stride < k || d_out->s_stride < 1)) return fail(DGDS_EBUFFER, "bad output strides");
  const int32_t max_spec = std::max(1, std::min(std::max(policy->per_request_cap, 1), s->p.max_spec_len));
  if (truth_stride < max_spec) return fail(DGDS_EINVAL, "truth_stride below the draft length cap");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  StreamJoin join(s, stream);
  if (int rc = s->d_step_args.ensure(sizeof(dgds_spec_args))) return rc;
  DGDS_CUDA(cudaMemcpyAsync(s->d_step_args.p, args, sizeof(dgds_spec_args), cudaMemcpyHostToDevice, join.stream()));
  dgds::QueryLaunch L{};
  L.T = s->T;
  L.root_of = s->d_root_of;
  L.n_handles = static_cast<int32_t>(s->root_of_cap);
  L.n = n;
  L.handles = d_handles;
  L.pat_len = nullptr;
  L.patterns = d_ctx;
  L.pat_stride = ctx_stride;
  L.args = static_cast<const dgds_spec_args*>(s->d_step_args.p);
  L.args_stride = 0;
  if (d_out) {
    L.k_stride = d_out->k_stride;
    L.s_stride = d_out->s_stride;
    dgds::soa_strides(L);
    L.n_cands = d_out->n_cands;
    L.lens = d_out->lens;
    L.scores = d_out->scores;
    L.supports = d_out->supports;
    L.tokens = d_out->tokens;
  } else {
    L.k_stride = k;
    L.s_stride = max_spec;
  }
  L.in_qstride = 1;
  L.v_qstride = 1;
  L.truth = d_truth;
  L.truth_stride = truth_stride;
  L.truth_left = d_truth_left;
  L.limit = d_limit;
  L.v_drafted = d_vout->drafted;
  L.v_accepted = d_vout->accepted;
  L.v_emitted = d_vout->emitted;
  L.err_flag = s->d_err;
  L.stat_part = s->d_stat_part;
  if (int rc = set_cplx(s, L)) return rc;
  L.engine = 1;
  L.draft_len = draft_len;
  L.draft_len_dev = d_draft_len;
  L.gen = d_generated;
  L.policy = *policy;
  L.step_acc = s->d_step_acc;
  L.next_draft_len = d_next_draft_len;
  L.step_totals = reinterpret_cast<long long*>(d_totals);
  {
    LaunchTimer lt(s, 1, join.stream());
    DGDS_CUDA(dgds::launch_query(L, k, max_spec, join.stream()));
  }
  return DGDS_OK;
}

int dgds_speculate_device(dgds_server* s, int64_t n, const int32_t* d_handles, const int32_t* d_pat_len,
                          const int32_t* d_patterns, int32_t pat_stride, const dgds_spec_args* d_args,
                          int64_t args_stride, int32_t max_top_k, int32_t max_spec, const dgds_candidates* d_out,
                          const int32_t* d_truth, int32_t truth_stride, const int32_t* d_truth_left,
                          const int32_t* d_limit, const dgds_verify_out* d_vout, dgds_query_stats* d_stats,
                          void* stream) {
  if (max_spec <= 0 || max_spec > s->p.max_spec_len) max_spec = std::max(1, s->p.max_spec_len);
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (n == 0) return DGDS_OK;
  if (max_top_k < 1 || max_top_k > DGDS_MAX_TOP_K) return fail(DGDS_EUNSUPPORTED, "max_top_k out of range");
  if (pat_stride < s->p.max_pattern_len) return fail(DGDS_EINVAL, "pat_stride must be >= max_pattern_len");
  if (d_out && (d_out->k_stride < max_top_k || d_out->s_stride < 1)) return fail(DGDS_EBUFFER, "bad output strides");
  if (d_vout && (!d_truth || !d_truth_left || !d_limit)) return fail(DGDS_EINVAL, "verify needs truth inputs");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  StreamJoin join(s, stream);
  dgds::QueryLaunch L{};
  L.T = s->T;
  L.root_of = s->d_root_of;
  L.n_handles = static_cast<int32_t>(s->root_of_cap);
  L.n = n;
  L.handles = d_handles;
  L.pat_len = d_pat_len;
  L.patterns = d_patterns;
  L.pat_stride = pat_stride;
  L.args = d_args;
  L.args_stride = args_stride;
  if (d_out) {
    L.k_stride = d_out->k_stride;
    L.s_stride = d_out->s_stride;
    dgds::soa_strides(L);
    L.n_cands = d_out->n_cands;
    L.lens = d_out->lens;
    L.scores = d_out->scores;
    L.supports = d_out->supports;
    L.tokens = d_out->tokens;
  }
  L.in_qstride = 1;
  L.v_qstride = 1;
  if (d_vout) {
    L.truth = d_truth;
    L.truth_stride = truth_stride;
    L.truth_left = d_truth_left;
    L.limit = d_limit;
    L.v_drafted = d_vout->drafted;
    L.v_accepted = d_vout->accepted;
    L.v_emitted = d_vout->emitted;
  }
  L.stats = d_stats;
  L.err_flag = s->d_err;
  L.stat_part = s->d_stat_part;
  if (int rc = set_cplx(s, L)) return rc;
  L.dbg = s->d_dbg;
  {
    LaunchTimer lt(s, 1, join.stream());
    DGDS_CUDA(dgds::launch_query(L, max_top_k, max_spec, join.stream()));
  }
  return DGDS_OK;
}

int dgds_speculate_records(dgds_server* s, int64_t n, const int32_t* d_records, const dgds_query_record_layout* lay,
                           const dgds_spec_args* d_args, int64_t args_stride, int32_t max_top_k, int32_t max_spec,
                           int32_t* d_replies, dgds_query_stats* d_stats, void* stream) {
  return speculate_records_impl(s, n, d_records, lay, d_args, args_stride, max_top_k, max_spec, d_replies, 0, 0,
                                nullptr, nullptr, -1, d_stats, stream);
}

int dgds_speculate_records_seg(dgds_server* s, int32_t n_seg, int64_t seg_rows, const int32_t* d_records,
                               const int32_t* d_seg_count, const dgds_query_record_layout* lay,
                               const dgds_spec_args* d_args, int64_t args_stride, int32_t max_top_k,
                               int32_t max_spec, int32_t* const* seg_out, int32_t origin_field,
                               dgds_query_stats* d_stats, void* stream) {
  if (n_seg < 1 || n_seg > dgds::kMaxSegments || seg_rows < 0) return fail(DGDS_EINVAL, "bad segment shape");
  if (lay && origin_field >= lay->rec_words) return fail(DGDS_EINVAL, "origin field outside the record");
  if (!d_seg_count || !seg_out) return fail(DGDS_EINVAL, "null argument");
  for (int i = 0; i < n_seg; ++i)
    if (!seg_out[i]) return fail(DGDS_EINVAL, "null segment output");
  return speculate_records_impl(s, static_cast<int64_t>(n_seg) * seg_rows, d_records, lay, d_args, args_stride,
                                max_top_k, max_spec, nullptr, n_seg, seg_rows, d_seg_count, seg_out, origin_field,
                                d_stats, stream);
}

int dgds_verify_batch(dgds_server* s, int64_t n, const dgds_candidates* c, const int32_t* truth, int32_t truth_stride,
                      const int32_t* truth_left, const int32_t* limit, dgds_verify_out* out) {
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (n == 0) return DGDS_OK;
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  const int K = c->k_stride, Sx = c->s_stride;
  const size_t o_ln = align_up(n * 4, 256);
  const size_t o_tk = align_up(o_ln + n * K * 4, 256);
  const size_t o_tr = align_up(o_tk + static_cast<size_t>(n) * K * Sx * 4, 256);
  const size_t o_tl = align_up(o_tr + static_cast<size_t>(n) * truth_stride * 4, 256);
  const size_t o_lm = align_up(o_tl + n * 4, 256);
  const size_t in_total = o_lm + n * 4;
  char* h = nullptr;
  cudaEvent_t ev_free = nullptr;
  if (int rc = next_stage(s, in_total, &h, &ev_free)) return rc;
  if (int rc = s->d_stage.ensure(in_total)) return rc;
  if (int rc = s->h_out.ensure(n * 12)) return rc;
  if (int rc = s->d_out.ensure(n * 12)) return rc;
  std::memcpy(h, c->n_cands, n * 4);
  std::memcpy(h + o_ln, c->lens, n * K * 4);
  std::memcpy(h + o_tk, c->tokens, static_cast<size_t>(n) * K * Sx * 4);
  std::memcpy(h + o_tr, truth, static_cast<size_t>(n) * truth_stride * 4);
  std::memcpy(h + o_tl, truth_left, n * 4);
  std::memcpy(h + o_lm, limit, n * 4);
  char* d = static_cast<char*>(s->d_stage.p);
  int32_t* dv = static_cast<int32_t*>(s->d_out.p);
  DGDS_CUDA(cudaMemcpyAsync(d, h, in_total, cudaMemcpyHostToDevice, s->st));
  DGDS_CUDA(cudaEventRecord(ev_free, s->st));
  DGDS_CUDA(dgds::launch_verify(n, K, Sx, reinterpret_cast<const int32_t*>(d), reinterpret_cast<const int32_t*>(d + o_ln),
                                reinterpret_cast<const int32_t*>(d + o_tk), reinterpret_cast<const int32_t*>(d + o_tr),
                                truth_stride, reinterpret_cast<const int32_t*>(d + o_tl),
                                reinterpret_cast<const int32_t*>(d + o_lm), dv, dv + n, dv + 2 * n, s->st));
  DGDS_CUDA(cudaMemcpyAsync(s->h_out.p, dv, n * 12, cudaMemcpyDeviceToHost, s->st));
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  const int32_t* hv = static_cast<const int32_t*>(s->h_out.p);
  std::memcpy(out->drafted, hv, n * 4);
  std::memcpy(out->accepted, hv + n, n * 4);
  std::memcpy(out->emitted, hv + 2 * n, n * 4);
  return DGDS_OK;
}

int dgds_batch_speculate_zc(dgds_server* s, int64_t n, const int32_t* d_handles, const int64_t* d_pat_end,
                            const int32_t* d_pat_len, const int32_t* d_pattern_buffer, const int64_t* d_out_offsets,
                            int32_t* d_output_buffer, const dgds_query_record_layout* lay,
                            const dgds_spec_args* d_args, int64_t args_stride, int32_t max_top_k, int32_t max_spec,
                            dgds_query_stats* d_stats, void* stream) {
  if (!s || n < 0) return fail(DGDS_EINVAL, "bad batch");
  if (n == 0) return DGDS_OK;
  if (!d_handles || !d_pat_end || !d_pat_len || !d_pattern_buffer || !d_out_offsets || !d_output_buffer || !lay ||
      !d_args)
    return fail(DGDS_EINVAL, "null argument");
  if (max_top_k < 1 || max_top_k > DGDS_MAX_TOP_K) return fail(DGDS_EUNSUPPORTED, "max_top_k out of range");
  if (max_spec <= 0 || max_spec > s->p.max_spec_len) max_spec = std::max(1, s->p.max_spec_len);
  const dgds_query_record_layout& y = *lay;
  if (y.reply_words < 1 || (y.off_scores & 1) || (y.off_supports & 1))
    return fail(DGDS_EINVAL, "bad reply layout (8-byte fields must be even)");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  StreamJoin join(s, stream);
  dgds::QueryLaunch L{};
  L.T = s->T;
  L.root_of = s->d_root_of;
  L.n_handles = static_cast<int32_t>(s->root_of_cap);
  L.n = n;
  L.handles = d_handles;
  L.pat_len = d_pat_len;
  L.patterns = d_pattern_buffer;
  L.pat_end = d_pat_end;
  L.pat_stride = 0x7FFFFFFF;  // the pattern is read in place: no row clamp
  L.in_qstride = 1;
  L.args = d_args;
  L.args_stride = args_stride;
  L.k_stride = max_top_k;
  L.s_stride = max_spec;
  L.rec_words_out = y.reply_words;
  L.rec_out = d_output_buffer;
  L.out_off = d_out_offsets;
  L.off_nc = y.off_n_cands;
  L.off_len = y.off_lens;
  L.off_sc = y.off_scores;
  L.off_sp = y.off_supports;
  L.off_tk = y.off_tokens;
  L.off_v = -1;  // the engine verifies with the target model
  L.stats = d_stats;
  L.err_flag = s->d_err;
  L.stat_part = s->d_stat_part;
  if (int rc = set_cplx(s, L)) return rc;
  L.dbg = s->d_dbg;
  {
    LaunchTimer lt(s, 1, join.stream());
    DGDS_CUDA(dgds::launch_query(L, max_top_k, max_spec, join.stream()));
  }
  return DGDS_OK;
}

}  // extern "C"
