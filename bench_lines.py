"""Extra bench lines (keys of bench.py's JSON line), device-timed like the headline:

  c5_sweep      engine-shaped ticks on the C4 (Kimi-K2-shaped) trace: B running requests, each
                appending its next 16-token record and issuing ONE draft query whose pattern is
                its own context's last 6 tokens (Instance::decode_step, engine.cpp:88-107), for
                B in 1K..16K (BASELINE.json configs[4]);
  c3_adaptive   the C3 (Qwen2-VL-72B-shaped) trace, every live request per tick, per-request
                draft length from the adaptive policy d = min(cap 8, budget 4096 / n_running),
                spec_len = min(d, limit - 1) (engine.cpp:78-85,95), top-1;
  c2_full       the C2 index with every response fully appended (R1 as BASELINE.md defines
                it), R1 queries only (nothing is left to append).

Each line reports device throughput and the roofline of both kernel groups (append =
k_stage + K1 + K1b, query = K2a + K2b) from the server's per-launch CUDA events, with the same
algorithmic-byte definitions as the headline.
"""
from __future__ import annotations

import ctypes as C
import gc
import time

import numpy as np

REC = 16


def build_index(cfg_name, prefill, device, extra_tokens_per_stream=0, seed=1234, num_groups=None):
    """Server + untimed prefill of the first `prefill` of every response (16-token records).
    num_groups: a larger group set of the same shape (the generator draws each group from its own
    substream, so the first groups are the config's own)."""
    import dataclasses

    from paper_2511_14617_b200.dgds import DgdsParams, DraftServer
    from paper_2511_14617_b200.workload import CONFIGS, generate_workload, group_id
    cfg = CONFIGS[cfg_name]
    if num_groups:
        cfg = dataclasses.replace(cfg, num_groups=num_groups)
    tr = generate_workload(cfg)
    G, R = cfg.num_groups, cfg.group_size
    S = G * R
    pre = (tr.lengths * prefill).astype(np.int64) // REC * REC if prefill < 1.0 else tr.lengths.astype(np.int64)
    idx_tokens = int(pre.sum()) + S * extra_tokens_per_stream
    srv = DraftServer(DgdsParams(), device=device, expected_nodes=min(idx_tokens * 3, 1_900_000_000),
                      expected_streams=S)
    gids = [group_id(g) for g in range(G)]
    handles = np.repeat(srv.group_handles(gids), R).astype(np.int32)
    rids = np.tile(np.arange(R, dtype=np.int32), G)
    pos = np.zeros(S, np.int64)
    t0 = time.time()
    while True:
        live = np.nonzero(pos < pre)[0]
        if len(live) == 0:
            break
        n_rec = np.minimum((pre[live] - pos[live] + REC - 1) // REC, 8)
        rs = np.repeat(live, n_rec)
        k_in = np.arange(len(rs)) - np.repeat(np.cumsum(n_rec) - n_rec, n_rec)
        starts = pos[rs] + k_in * REC
        ns = np.minimum(REC, pre[rs] - starts)
        offs = np.zeros(len(ns) + 1, np.uint64)
        offs[1:] = np.cumsum(ns)
        idx = np.repeat(tr.offsets[rs] + starts, ns) + (np.arange(int(offs[-1])) - np.repeat(offs[:-1].astype(np.int64), ns))
        rep = srv.update_arrays(handles[rs], rids[rs], starts.astype(np.uint64), offs, tr.tokens[idx], 0.0)
        assert rep["ok"].all()
        pos[live] += np.minimum(pre[live] - pos[live], 8 * REC)
    return dict(tr=tr, srv=srv, handles=handles, rids=rids, pos=pos, S=S, G=G, R=R, prefill_s=time.time() - t0)


def append_alg_bytes(start, n, D=24):
    start = np.asarray(start, np.int64)
    n = np.asarray(n, np.int64)
    keep = n > 0
    lo, hi, n = start[keep] + 1, start[keep] + n[keep], n[keep]
    top = np.minimum(hi, D)
    ramp = np.where(lo <= D, (lo + top) * (top - lo + 1) // 2, 0)
    flat = np.where(hi > D, (hi - np.maximum(lo, D + 1) + 1) * D, 0)
    return int((4 * n + 64 * (ramp + flat)).sum())


def run_ticks(ix, ticks, warmup, dev, peak):
    """ticks: list of dicts (device inputs prepared beforehand) with keys
    app (None or dict h, r, prev, offs, d_tok, alg, ntok), q (dict h, pl, pat, tru, tl, lim, args, stride,
    n, K, S). Times the ticks after `warmup` of them with CUDA events on the server stream."""
    import torch

    from paper_2511_14617_b200 import _lib
    srv = ix["srv"]
    L = _lib.lib()
    sstream = srv.cuda_stream
    ext = torch.cuda.ExternalStream(sstream, device=dev)
    Kmax = max(t["q"]["K"] for t in ticks)
    Smax = max(t["q"]["S"] for t in ticks)
    Qmax = max(t["q"]["n"] for t in ticks)
    out = dict(nc=torch.zeros(Qmax, dtype=torch.int32, device=dev),
               ln=torch.zeros(Qmax * Kmax, dtype=torch.int32, device=dev),
               sc=torch.zeros(Qmax * Kmax, dtype=torch.float64, device=dev),
               sp=torch.zeros(Qmax * Kmax, dtype=torch.int64, device=dev),
               tk=torch.zeros(Qmax * Kmax * Smax, dtype=torch.int32, device=dev),
               v=torch.zeros((3, Qmax), dtype=torch.int32, device=dev))
    d_stats = torch.zeros(8, dtype=torch.int64, device=dev)
    cand = _lib.Candidates(Kmax, Smax, out["nc"].data_ptr(), out["ln"].data_ptr(), out["sc"].data_ptr(),
                           out["sp"].data_ptr(), out["tk"].data_ptr())
    vo = _lib.VerifyOut(out["v"][0].data_ptr(), out["v"][1].data_ptr(), out["v"][2].data_ptr())

    def step(t, stats):
        a, q = t["app"], t["q"]
        if a is not None:
            srv.update_device(a["h"], a["r"], a["prev"], a["offs"], a["d_tok"].data_ptr(), 0.0, sstream)
        _lib.check(L.dgds_speculate_device(
            srv.handle, q["n"], C.c_void_p(q["h"].data_ptr()), C.c_void_p(q["pl"].data_ptr()),
            C.c_void_p(q["pat"].data_ptr()), 8, C.c_void_p(q["args"].data_ptr()), q["stride"], q["K"], q["S"],
            C.byref(cand), C.c_void_p(q["tru"].data_ptr()), q["S"], C.c_void_p(q["tl"].data_ptr()),
            C.c_void_p(q["lim"].data_ptr()), C.byref(vo), C.c_void_p(d_stats.data_ptr()) if stats else None,
            C.c_void_p(sstream)))

    torch.cuda.synchronize()
    for t in ticks[:warmup]:
        step(t, False)
    torch.cuda.synchronize()
    prof = _lib.Profile()
    _lib.check(L.dgds_profile_enable(srv.handle, 1))
    _lib.check(L.dgds_profile_read(srv.handle, C.byref(prof), 1))
    gc.collect()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(ext)
    for t in ticks[warmup:]:
        step(t, True)
    e1.record(ext)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    _lib.check(L.dgds_profile_read(srv.handle, C.byref(prof), 1))
    _lib.check(L.dgds_profile_enable(srv.handle, 0))
    K = len(ticks) - warmup
    nq = sum(t["q"]["n"] for t in ticks[warmup:])
    ntok = sum(t["app"]["ntok"] for t in ticks[warmup:] if t["app"] is not None)
    a_alg = sum(t["app"]["alg"] for t in ticks[warmup:] if t["app"] is not None)
    q_alg = int(d_stats[7].item())
    T = ms / 1e3
    res = {"ticks": K, "ms_per_tick": ms / K, "queries_per_s": nq / T, "queries_per_tick": nq / K,
           "append_tokens_per_s": ntok / T if ntok else None}
    if prof.query_ms > 0:
        ach = q_alg / (prof.query_ms / 1e3) / 1e9
        res["roofline_query"] = {"achieved": ach, "frac": ach / peak, "avg_launch_ms": prof.query_ms / max(1, K),
                                 "alg_bytes_per_tick": q_alg / K}
    if prof.append_ms > 0 and a_alg:
        ach = a_alg / (prof.append_ms / 1e3) / 1e9
        res["roofline_append"] = {"achieved": ach, "frac": ach / peak, "avg_launch_ms": prof.append_ms / max(1, K),
                                  "alg_bytes_per_tick": a_alg / K}
    return res


def _query_inputs(tr, st, qpos, dev, args_rows, stride, K, S, handles):
    import torch
    n = len(st)
    base = tr.offsets[st] + qpos
    pat = np.zeros((n, 8), np.int32)
    for j in range(6):
        ok = qpos - 6 + j >= 0
        pat[ok, j] = tr.tokens[(base - 6 + j)[ok]]
    pl = np.minimum(qpos, 6).astype(np.int32)
    # patterns shorter than 6 (a context of fewer tokens) sit at the row's end
    for short in np.nonzero(pl < 6)[0]:
        k = pl[short]
        pat[short, :k] = tr.tokens[base[short] - k:base[short]]
    tl = (tr.lengths[st] - qpos).astype(np.int32)
    tru = np.zeros((n, S), np.int32)
    for j in range(S):
        ok = j < tl
        tru[ok, j] = tr.tokens[(base + j)[ok]]
    return dict(h=torch.from_numpy(handles[st]).to(dev), pl=torch.from_numpy(pl).to(dev),
                pat=torch.from_numpy(pat).to(dev), tru=torch.from_numpy(tru).to(dev), tl=torch.from_numpy(tl).to(dev),
                lim=torch.from_numpy(tl).to(dev), args=torch.from_numpy(args_rows.view(np.uint8).copy()).to(dev),
                stride=stride, n=n, K=K, S=S)


def _append_inputs(tr, live, pos, handles, rids, dev):
    import torch
    ns = np.minimum(REC, tr.lengths[live] - pos[live])
    keep = ns > 0
    live, ns = live[keep], ns[keep]
    offs = np.zeros(len(live) + 1, np.uint64)
    offs[1:] = np.cumsum(ns)
    idx = np.repeat(tr.offsets[live] + pos[live], ns) + (np.arange(int(offs[-1])) - np.repeat(offs[:-1].astype(np.int64), ns))
    a = dict(h=handles[live], r=rids[live], prev=pos[live].astype(np.uint64), offs=offs,
             d_tok=torch.from_numpy(tr.tokens[idx]).to(dev), alg=append_alg_bytes(pos[live], ns), ntok=int(offs[-1]))
    pos[live] += ns
    return a


def c5_sweep(dev, device, peak, Bs=(1024, 2048, 4096, 8192, 16384), ticks=40, warmup=5, seed=5):
    """Engine-shaped ticks on the C4-shaped trace at 50% prefill: B running requests. C4 has 8,192
    streams, so the trace is the C4 shape with 1,024 groups (16,384 streams; its first 512 groups are
    C4's own) to reach B = 16K."""
    from paper_2511_14617_b200.dgds import SpeculationArgs, args_array
    ix = build_index("C4", 0.5, device, extra_tokens_per_stream=REC * (ticks + warmup) * 2, num_groups=1024)
    tr, rng = ix["tr"], np.random.default_rng(seed)
    args = args_array([SpeculationArgs(8, 6, 1, 4, 0.25, 1)])
    rows = []
    for B in Bs:
        live_all = np.nonzero(ix["pos"] + REC * (ticks + warmup) <= tr.lengths)[0]
        if len(live_all) < B:  # short responses: take the longest-remaining ones
            live_all = np.argsort(ix["pos"] - tr.lengths)[:B]
        run = np.sort(rng.choice(live_all, size=min(B, len(live_all)), replace=False))
        tk = []
        for _ in range(ticks + warmup):
            app = _append_inputs(tr, run, ix["pos"], ix["handles"], ix["rids"], dev)
            q = _query_inputs(tr, run, ix["pos"][run].copy(), dev, args, 0, 4, 8, ix["handles"])
            tk.append(dict(app=app, q=q))
        r = run_ticks(ix, tk, warmup, dev, peak)
        r["running_requests"] = int(len(run))
        rows.append(r)
        del tk
    entries, nodes = ix["srv"].entry_count(), ix["srv"].node_count()
    ix["srv"].close()
    return {"workload": "C4-shaped trace (1024 groups x 16, <=64K tokens, V 163840; the first 512 groups are C4) at 50% "
                        "prefill on ONE GPU; per tick "
                        "each of B running requests appends its next 16-token record and issues one query "
                        "(pattern = its own context's last 6 tokens, top-4, draft 8, fused verify)",
            "index_entries": entries, "index_nodes": nodes, "points": rows}


def c3_adaptive(dev, device, peak, ticks=60, warmup=5):
    """C3 trace at 50% prefill; each tick every live request appends and queries with its
    adaptive draft length (engine.cpp:78-85,95)."""
    from paper_2511_14617_b200.dgds import SpeculationArgs, args_array, draft_len
    ix = build_index("C3", 0.5, device, extra_tokens_per_stream=REC * (ticks + warmup))
    tr = ix["tr"]
    tk = []
    ds = []
    for _ in range(ticks + warmup):
        live = np.nonzero(ix["pos"] < tr.lengths)[0]
        d = draft_len(True, True, 8, 4096, len(live))
        app = _append_inputs(tr, live, ix["pos"], ix["handles"], ix["rids"], dev)
        q_pos = ix["pos"][live].copy()  # the context after this tick's record
        limit = tr.lengths[live] - q_pos
        spec = np.minimum(d, np.maximum(limit - 1, 0))
        args = args_array([SpeculationArgs(int(x), 6, 1, 1, 0.25, 1) for x in spec])
        q = _query_inputs(tr, live, q_pos, dev, args, 1, 1, 8, ix["handles"])
        tk.append(dict(app=app, q=q))
        ds.append(d)
    r = run_ticks(ix, tk, warmup, dev, peak)
    r["draft_len_range"] = [int(min(ds)), int(max(ds))]
    r["index_entries"] = ix["srv"].entry_count()
    ix["srv"].close()
    r["workload"] = ("C3 trace (128 groups x 8, <=16K tokens, V 152064) at 50% prefill; per tick every live request "
                     "appends its next record and queries with spec_len = min(d, limit-1), d = min(8, 4096/n_running)"
                     ", top-1")
    return r


def c2_full(dev, device, peak, Q=65536, ticks=40, warmup=5, seed=9):
    """C2 with every response fully appended (R1); R1 queries only."""
    from paper_2511_14617_b200.dgds import SpeculationArgs, args_array
    ix = build_index("C2", 1.0, device)
    tr, rng = ix["tr"], np.random.default_rng(seed)
    args = args_array([SpeculationArgs(8, 6, 1, 4, 0.25, 1)])
    pool = np.nonzero(ix["pos"] >= 7)[0]
    tk = []
    for _ in range(ticks + warmup):
        st = pool[rng.integers(0, len(pool), Q)]
        qpos = 6 + (rng.random(Q) * (ix["pos"][st] - 6 + 1)).astype(np.int64)
        qpos = np.minimum(qpos, ix["pos"][st])
        tk.append(dict(app=None, q=_query_inputs(tr, st, qpos, dev, args, 0, 4, 8, ix["handles"])))
    r = run_ticks(ix, tk, warmup, dev, peak)
    r["index_entries"] = ix["srv"].entry_count()
    r["index_nodes"] = ix["srv"].node_count()
    r["index_slots"] = ix["srv"].index_slots()
    r["index_gb"] = r["index_slots"] * 32 / 1e9
    r["prefill_s"] = ix["prefill_s"]
    ix["srv"].close()
    r["workload"] = ("C2 with every response fully appended (R1, BASELINE.md); 65,536 R1 queries per tick, top-4, "
                     "draft 8, fused verify")
    return r
