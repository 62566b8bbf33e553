"""End-to-end throughput of the N-GPU cluster API (dgds_cluster_*: one process, one shard per GPU,
host buffers in and out) on C2-shaped ticks:

  python tools/cluster_bench.py N [weak|strong] [ticks]

weak: the C2 group set replicated N times (per-GPU work fixed); strong: C2 sharded over N GPUs.
Per tick: one 16-token record per stream (dgds_cluster_update_batch) + 65,536 x N (weak) or 65,536
(strong) R1 queries with fused verification (dgds_cluster_speculate_verify_batch), wall time
around the whole tick (the host splits by owner, one host thread per GPU runs its batch).
Reported in profiles/, not a bench.py line (bench.py's N>1 runs are one process per GPU).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14617_b200 import dgds as D  # noqa: E402
from paper_2511_14617_b200.workload import CONFIGS, generate_workload, group_id  # noqa: E402


def proc_stats():
    """Process minor/major faults and summed thread context switches (/proc), for the timed ticks."""
    f = open("/proc/self/stat").read().rsplit(")", 1)[1].split()
    r = {"minflt": int(f[7]), "majflt": int(f[9]), "vol_cs": 0, "invol_cs": 0}
    for t in os.listdir("/proc/self/task"):
        try:
            for line in open("/proc/self/task/%s/status" % t):
                if line.startswith("voluntary_ctxt_switches"):
                    r["vol_cs"] += int(line.split()[1])
                elif line.startswith("nonvoluntary_ctxt_switches"):
                    r["invol_cs"] += int(line.split()[1])
        except OSError:
            pass
    return r


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    mode = sys.argv[2] if len(sys.argv) > 2 else "weak"
    ticks = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    cfg = CONFIGS["C2"]
    tr = generate_workload(cfg)
    reps = N if mode == "weak" else 1
    G, R = cfg.num_groups, cfg.group_size
    gids = [("%s" % group_id(g)) + ("" if k == 0 else "/r%d" % k) for k in range(reps) for g in range(G)]
    S = len(gids) * R
    base = np.tile(np.arange(G * R), reps)  # trace stream of each cluster stream
    lens = tr.lengths[base]
    pre = (lens * 0.5).astype(np.int64) // 16 * 16
    c = D.DraftCluster(D.DgdsParams(), devices=list(range(N)),
                       expected_nodes=int(pre.sum() * 3 // N) + (1 << 20), expected_streams=S // N + 1024)
    h_of_stream = np.repeat(c.group_handles(gids), R).astype(np.int32)
    rid = np.tile(np.arange(R, dtype=np.int32), len(gids))
    L = D.lib()
    pos = np.zeros(S, np.int64)
    t0 = time.time()
    while (pos < pre).any():
        live = np.nonzero(pos < pre)[0]
        ns = np.minimum(128, pre[live] - pos[live])
        offs = np.zeros(len(live) + 1, np.uint64)
        offs[1:] = np.cumsum(ns)
        idx = np.repeat(tr.offsets[base[live]] + pos[live], ns) + (
            np.arange(int(offs[-1])) - np.repeat(offs[:-1].astype(np.int64), ns))
        toks = np.ascontiguousarray(tr.tokens[idx], np.int32)
        rep = np.zeros(len(live), D.DraftServer.REPLY_DTYPE)
        D.check(L.dgds_cluster_update_batch(c._h, len(live), D._ptr(h_of_stream[live]), D._ptr(rid[live]),
                                            D._ptr(pos[live].astype(np.uint64)), D._ptr(offs), D._ptr(toks), 0.0,
                                            D._ptr(rep)))
        pos[live] += ns
    prefill_s = time.time() - t0
    Q = 65536 * (N if mode == "weak" else 1)
    rng = np.random.default_rng(3)
    args = D.args_array([D.SpeculationArgs(8, 6, 1, 4, 0.25, 1)])
    K, SP = 4, 8

    def make_tick():
        live = np.nonzero(pos < lens)[0]
        ns = np.minimum(16, lens[live] - pos[live])
        offs = np.zeros(len(live) + 1, np.uint64)
        offs[1:] = np.cumsum(ns)
        idx = np.repeat(tr.offsets[base[live]] + pos[live], ns) + (
            np.arange(int(offs[-1])) - np.repeat(offs[:-1].astype(np.int64), ns))
        app = (live, pos[live].astype(np.uint64), offs, np.ascontiguousarray(tr.tokens[idx], np.int32))
        pos[live] += ns
        st = rng.integers(0, S, Q)
        st = st[pre[st] >= 7]
        qp = 6 + (rng.random(len(st)) * (pre[st] - 6 + 1)).astype(np.int64)
        qb = tr.offsets[base[st]] + qp
        pats = np.stack([tr.tokens[qb - 6 + j] for j in range(6)], 1).astype(np.int32).reshape(-1)
        poff = np.arange(0, 6 * len(st) + 1, 6, dtype=np.uint64)
        tl = (lens[st] - qp).astype(np.int32)
        tru = np.zeros((len(st), SP), np.int32)
        for j in range(SP):
            ok = j < tl
            tru[ok, j] = tr.tokens[(qb + j)[ok]]
        return app, (h_of_stream[st].copy(), poff, pats, tru, tl), (h_of_stream[live].copy(), rid[live].copy())

    WARM = 8  # lets the per-owner staging buffers reach their steady capacity
    work = [make_tick() for _ in range(ticks + WARM)]
    nc_tot = 0
    nmax = max(len(t[1][0]) for t in work)
    out = D.CandidateBatch(nmax, K, SP)  # reused: fresh pages would fault inside the timed ticks
    dr, ac, em = (np.zeros(nmax, np.int32) for _ in range(3))
    vo = D._lib.VerifyOut(D._ptr(dr), D._ptr(ac), D._ptr(em))
    reps = np.zeros(S, D.DraftServer.REPLY_DTYPE)

    phase = [0.0, 0.0]

    def run(t):
        nonlocal nc_tot
        (live, prev, offs, toks), (qh, poff, pats, tru, tl) = t[0], t[1]
        hs, rs = t[2]
        ta = time.perf_counter()
        D.check(L.dgds_cluster_update_batch(c._h, len(live), D._ptr(hs), D._ptr(rs),
                                            D._ptr(prev), D._ptr(offs), D._ptr(toks), 0.0, D._ptr(reps)))
        n = len(qh)
        tb = time.perf_counter()
        D.check(L.dgds_cluster_speculate_verify_batch(c._h, n, D._ptr(qh), D._ptr(poff), D._ptr(pats), D._ptr(args), 0,
                                                      D._ptr(tru), SP, D._ptr(tl), D._ptr(tl), D.C.byref(out.c()),
                                                      D.C.byref(vo)))
        phase[0] += tb - ta
        phase[1] += time.perf_counter() - tb
        nc_tot += int(out.n_cands[:n].sum())
        return n, int(offs[-1])

    for t in work[:WARM]:
        run(t)
    phase[:] = [0.0, 0.0]
    pst0 = proc_stats()
    t0 = time.perf_counter()
    nq = ntok = 0
    for t in work[WARM:]:
        a, b = run(t)
        nq += a
        ntok += b
    dt = time.perf_counter() - t0
    pst1 = proc_stats()
    print(json.dumps({"tool": "cluster_bench", "n_gpus": N, "mode": mode, "ticks": ticks, "queries_per_tick": Q,
                      "e2e_queries_per_s": nq / dt, "e2e_append_tokens_per_s": ntok / dt,
                      "ms_per_tick": 1e3 * dt / ticks,
                      "update_ms": 1e3 * phase[0] / ticks, "query_ms": 1e3 * phase[1] / ticks, "prefill_s": prefill_s,
                      "proc": {k: pst1[k] - pst0[k] for k in pst0}, "groups": len(gids),
                      "path": "dgds_cluster_update_batch + dgds_cluster_speculate_verify_batch, host buffers, serial "
                              "ticks, one process"}))
    c.close()


if __name__ == "__main__":
    main()
