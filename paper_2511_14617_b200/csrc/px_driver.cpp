// px_driver.cpp — the routed multi-GPU tick loop in C++ (dgds_px_driver_*, include/dgds_b200.h).
//
// One rank of the owner-routed draft service: every tick the rank sends its
// queries to their owners' slabs (dgds_px_send), serves the queries it owns (K2 + fused K3,
// replies stored straight into the senders' reply slab: dgds_speculate_records_seg), and
// applies the append records routed to it — the reference's shard routing (dgds.cpp:10-51)
// over NVLink peer memory. The loop keeps bench_multi.py's pipeline, minus the interpreter:
//
//   side stream   appends of tick s+1 -> owners, then their metadata rows D2H (event ev_meta)
//   side_q stream queries of tick s+1 -> owners, once tick s's replies are home (ev_rep)
//   planner       the server's planner thread plans tick s+1's appends as its metadata lands
//   main stream   K2(s) ... K1(s) [plan s] -> K2(s+1) -> K1(s+1) ...
//
// Slab parities are reused only after a round trip proves the readers finished: a tick's
// sends wait for the replies of the previous tick (ev_rep), which the owners produced after
// their K1 of the tick before (the last reader of the parity).
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "../../include/dgds_b200.h"

namespace dgds {
int set_error(int code, const std::string& msg);  // server.cpp
}

struct dgds_px_driver {
  dgds_server* s = nullptr;
  dgds_px* px = nullptr;
  int32_t world = 1, rank = 0, q_origin = -1, max_top_k = 1, max_spec = 1;
  dgds_px_channel_desc q{}, rep{}, a{};
  dgds_query_record_layout layout{};
  const dgds_spec_args* d_args = nullptr;
  int32_t* d_overflow = nullptr;
  std::vector<dgds_px_tick> ticks;
  cudaStream_t main = nullptr, side = nullptr, side_q = nullptr;
  cudaEvent_t ev_rep[2] = {nullptr, nullptr}, ev_meta[2] = {nullptr, nullptr};
  int32_t* h_meta[2] = {nullptr, nullptr};  // [world * a.rows][5] leading words of the routed rows
  int32_t* h_cnt[2] = {nullptr, nullptr};   // [world] rows per sender
  std::vector<void*> bases;
  std::vector<int32_t*> seg_out[2];  // reply destinations per peer, by parity
  std::map<int64_t, int> inflight;   // tick -> metadata buffer
  std::map<int64_t, uint64_t> plans;  // tick -> planner job
  std::vector<char> q_sent;
  int64_t run_until = 0, plan_until = 0;
  dgds_query_stats* d_stats = nullptr;
};

namespace {

#define PXD_CUDA(x)                                                                         \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) return dgds::set_error(DGDS_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

char* at(dgds_px_driver* d, int peer, uint64_t off) { return static_cast<char*>(d->bases[peer]) + off; }

int route_appends(dgds_px_driver* d, int64_t s) {
  if (s >= static_cast<int64_t>(d->ticks.size()) || d->inflight.count(s)) return DGDS_OK;
  const dgds_px_tick& t = d->ticks[s];
  const int k = static_cast<int>(s % 2);
  const uint64_t seq = static_cast<uint64_t>(s) + 1;
  if (s > 0) PXD_CUDA(cudaStreamWaitEvent(d->side, d->ev_rep[(s - 1) % 2], 0));
  if (int rc = dgds_px_send(d->px, t.n_a, t.a_owner, t.a, d->a.words, d->a.rows, d->a.slab_off[seq % 2],
                            d->a.count_off[seq % 2], d->a.flag_off, seq, 1, -1, nullptr, d->d_overflow, d->side))
    return rc;
  if (int rc = dgds_px_wait(d->px, d->a.flag_off, seq, d->side)) return rc;
  // metadata columns of every row (one 2-D copy) and the per-sender counts
  PXD_CUDA(cudaMemcpy2DAsync(d->h_meta[k], 20, at(d, d->rank, d->a.slab_off[seq % 2]), d->a.words * 4, 20,
                             static_cast<size_t>(d->world) * d->a.rows, cudaMemcpyDeviceToHost, d->side));
  PXD_CUDA(cudaMemcpyAsync(d->h_cnt[k], at(d, d->rank, d->a.count_off[seq % 2]), 4 * d->world,
                           cudaMemcpyDeviceToHost, d->side));
  PXD_CUDA(cudaEventRecord(d->ev_meta[k], d->side));
  d->inflight[s] = k;
  return DGDS_OK;
}

int send_queries(dgds_px_driver* d, int64_t s) {
  if (s >= static_cast<int64_t>(d->ticks.size()) || d->q_sent[s]) return DGDS_OK;
  const dgds_px_tick& t = d->ticks[s];
  const uint64_t seq = static_cast<uint64_t>(s) + 1;
  if (s > 0) PXD_CUDA(cudaStreamWaitEvent(d->side_q, d->ev_rep[(s - 1) % 2], 0));
  if (int rc = dgds_px_send(d->px, t.n_q, t.q_owner, t.q, d->q.words, d->q.rows, d->q.slab_off[seq % 2],
                            d->q.count_off[seq % 2], d->q.flag_off, seq, 0, d->q_origin, nullptr, d->d_overflow,
                            d->side_q))
    return rc;
  d->q_sent[s] = 1;
  return DGDS_OK;
}

int submit_plan(dgds_px_driver* d, int64_t s, int k) {
  uint64_t job = 0;
  const uint64_t seq = static_cast<uint64_t>(s) + 1;
  if (int rc = dgds_update_plan_routed_async(d->s, d->ev_meta[k], d->world, d->a.rows, d->h_cnt[k], d->h_meta[k], 5,
                                             reinterpret_cast<const int32_t*>(at(d, d->rank, d->a.slab_off[seq % 2])),
                                             d->a.words, 0.0, &job))
    return rc;
  d->plans[s] = job;
  return DGDS_OK;
}

// Tick s, first half (engine.cpp:88-143): queries (+ fused verification) on the current index.
int q_part(dgds_px_driver* d, int64_t s) {
  if (int rc = route_appends(d, s)) return rc;  // normally in flight since the previous tick
  if (int rc = send_queries(d, s)) return rc;
  const uint64_t seq = static_cast<uint64_t>(s) + 1;
  if (int rc = dgds_px_wait(d->px, d->q.flag_off, seq, d->main)) return rc;
  if (int rc = dgds_speculate_records_seg(d->s, d->world, d->q.rows,
                                          reinterpret_cast<const int32_t*>(at(d, d->rank, d->q.slab_off[seq % 2])),
                                          reinterpret_cast<const int32_t*>(at(d, d->rank, d->q.count_off[seq % 2])),
                                          &d->layout, d->d_args, 0, d->max_top_k, d->max_spec,
                                          d->seg_out[seq % 2].data(), d->q_origin, d->d_stats, d->main))
    return rc;
  if (int rc = dgds_px_signal(d->px, d->rep.flag_off, seq, d->main)) return rc;
  if (int rc = dgds_px_wait(d->px, d->rep.flag_off, seq, d->main)) return rc;  // this rank's replies are home
  PXD_CUDA(cudaEventRecord(d->ev_rep[s % 2], d->main));
  return DGDS_OK;
}

// Tick s, second half (engine.cpp:144-161): the appends of the tick's emitted tokens, planned
// on the planner thread as their metadata arrived, launched after the tick's queries; then
// tick s+1's queries are enqueued, so the GPU has work while the next plan is made.
int a_part(dgds_px_driver* d, int64_t s) {
  auto it = d->inflight.find(s);
  if (it == d->inflight.end()) return dgds::set_error(DGDS_ESTATE, "tick appends were not routed");
  const int k = it->second;
  d->inflight.erase(it);
  if (!d->plans.count(s))  // the planner is FIFO: tick s is planned before tick s+1
    if (int rc = submit_plan(d, s, k)) return rc;
  if (int rc = route_appends(d, s + 1)) return rc;
  auto nx = d->inflight.find(s + 1);
  if (s + 1 < d->plan_until && nx != d->inflight.end() && !d->plans.count(s + 1))
    if (int rc = submit_plan(d, s + 1, nx->second)) return rc;
  if (int rc = send_queries(d, s + 1)) return rc;
  int64_t nrej = 0;
  dgds_update_plan* plan = nullptr;
  const uint64_t job = d->plans[s];
  d->plans.erase(s);
  if (int rc = dgds_update_plan_take(d->s, job, &nrej, &plan)) return rc;
  if (nrej) return dgds::set_error(DGDS_ESTATE, "routed append out of order");
  PXD_CUDA(cudaStreamWaitEvent(d->main, d->ev_meta[k], 0));  // K1 reads the slab rows delivered on side
  if (int rc = dgds_update_launch(d->s, plan, d->main)) return rc;
  if (s + 1 < d->run_until) return q_part(d, s + 1);
  return DGDS_OK;
}

}  // namespace

extern "C" {

int dgds_px_driver_create(dgds_server* s, dgds_px* px, int32_t world, int32_t rank, const dgds_px_channel_desc* q,
                          const dgds_px_channel_desc* rep, const dgds_px_channel_desc* a, int32_t q_origin_word,
                          const dgds_query_record_layout* layout, const dgds_spec_args* d_args, int32_t max_top_k,
                          int32_t max_spec, int32_t* d_overflow, const dgds_px_tick* ticks, int64_t n_ticks,
                          void* main_stream, dgds_px_driver** out) {
  if (!s || !px || !q || !rep || !a || !layout || !d_args || !d_overflow || !out || (n_ticks > 0 && !ticks) ||
      world < 1 || rank < 0 || rank >= world || n_ticks < 0)
    return dgds::set_error(DGDS_EINVAL, "bad px driver arguments");
  if (a->words < 6 || q_origin_word < 0 || q_origin_word >= q->words || !rep->shared)
    return dgds::set_error(DGDS_EINVAL, "px driver: append rows need 6+ words, queries an origin word, replies a "
                                        "shared slab");
  *out = nullptr;
  auto d = new dgds_px_driver();
  d->s = s;
  d->px = px;
  d->world = world;
  d->rank = rank;
  d->q = *q;
  d->rep = *rep;
  d->a = *a;
  d->q_origin = q_origin_word;
  d->layout = *layout;
  d->d_args = d_args;
  d->max_top_k = max_top_k;
  d->max_spec = max_spec;
  d->d_overflow = d_overflow;
  d->ticks.assign(ticks, ticks + n_ticks);
  d->q_sent.assign(n_ticks, 0);
  d->main = static_cast<cudaStream_t>(main_stream);
  auto fail_out = [&](int rc) {
    dgds_px_driver_destroy(d);
    return rc;
  };
  d->bases.resize(world);
  for (int p = 0; p < world; ++p)
    if (int rc = dgds_px_region(px, p, &d->bases[p])) return fail_out(rc);
  for (int par = 0; par < 2; ++par) {
    d->seg_out[par].resize(world);
    for (int p = 0; p < world; ++p)
      d->seg_out[par][p] = reinterpret_cast<int32_t*>(at(d, p, rep->slab_off[par]));
  }
  cudaError_t e = cudaStreamCreateWithFlags(&d->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&d->side_q, cudaStreamNonBlocking);
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
    e = cudaEventCreateWithFlags(&d->ev_rep[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_meta[k], cudaEventDisableTiming);
    if (e == cudaSuccess)
      e = cudaHostAlloc(reinterpret_cast<void**>(&d->h_meta[k]), static_cast<size_t>(world) * a->rows * 20 + 64,
                        cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&d->h_cnt[k]), 4 * world + 64, cudaHostAllocDefault);
  }
  if (e != cudaSuccess) return fail_out(dgds::set_error(DGDS_ECUDA, std::string("px driver: ") + cudaGetErrorString(e)));
  *out = d;
  return DGDS_OK;
}

int dgds_px_driver_run(dgds_px_driver* d, int64_t first, int64_t last, int64_t plan_to, dgds_query_stats* d_stats) {
  if (!d || first < 0 || last > static_cast<int64_t>(d->ticks.size()) || first >= last)
    return dgds::set_error(DGDS_EINVAL, "bad tick range");
  d->run_until = last;
  d->plan_until = plan_to > 0 ? plan_to : last;
  d->d_stats = d_stats;
  if (int rc = q_part(d, first)) return rc;
  for (int64_t s = first; s < last; ++s)
    if (int rc = a_part(d, s)) return rc;
  return DGDS_OK;
}

int dgds_px_driver_destroy(dgds_px_driver* d) {
  if (!d) return DGDS_OK;
  if (d->side) cudaStreamSynchronize(d->side);
  if (d->side_q) cudaStreamSynchronize(d->side_q);
  // planned ahead but not run: their records are accepted (stream counts advanced), so they are
  // launched, keeping the index consistent with the bookkeeping
  for (auto& kv : d->plans) {
    int64_t nrej = 0;
    dgds_update_plan* p = nullptr;
    if (dgds_update_plan_take(d->s, kv.second, &nrej, &p) == DGDS_OK && p) {
      cudaStreamWaitEvent(d->main, d->ev_meta[kv.first % 2], 0);
      dgds_update_launch(d->s, p, d->main);
    }
  }
  if (d->main) cudaStreamSynchronize(d->main);
  for (int k = 0; k < 2; ++k) {
    if (d->ev_rep[k]) cudaEventDestroy(d->ev_rep[k]);
    if (d->ev_meta[k]) cudaEventDestroy(d->ev_meta[k]);
    if (d->h_meta[k]) cudaFreeHost(d->h_meta[k]);
    if (d->h_cnt[k]) cudaFreeHost(d->h_cnt[k]);
  }
  if (d->side) cudaStreamDestroy(d->side);
  if (d->side_q) cudaStreamDestroy(d->side_q);
  delete d;
  return DGDS_OK;
}

}  // extern "C"
