"""GPU parity at the measured scale: the bench's C2 workload (and C3 / C4 samples) built on the
GPU and in the compiled reference (oracle/_ref: the reference GroupDraftIndex, many groups
driven in bulk on host threads), then ~50K draft queries compared bit-exactly (tokens, order,
IEEE score bits, supports, candidate counts) together with the fused verification
(drafted / accepted / emitted, engine.cpp:115-143) and the trie node counts. Streaming ticks
(one 16-token record per stream) follow the prefill, so K1's conversions, riders and walks are
checked at steady state, not only on a cold build.
"""
import dataclasses

import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_14617_b200 import dgds as D
from paper_2511_14617_b200.workload import CONFIGS, generate_workload, group_id

pytestmark = pytest.mark.gpu

REC = 16


def _records(tr, R, lo, hi):
    """16-token records covering positions [lo, hi) of every stream, round-robin by record."""
    S = len(lo)
    n_rec = np.maximum(0, (hi - lo + REC - 1) // REC)
    recs = []
    k = 0
    while True:
        live = np.nonzero(n_rec > k)[0]
        if len(live) == 0:
            break
        st = live
        starts = lo[st] + k * REC
        ns = np.minimum(REC, hi[st] - starts)
        recs.append((st, starts, ns))
        k += 1
    st = np.concatenate([r[0] for r in recs]) if recs else np.zeros(0, np.int64)
    starts = np.concatenate([r[1] for r in recs]) if recs else np.zeros(0, np.int64)
    ns = np.concatenate([r[2] for r in recs]) if recs else np.zeros(0, np.int64)
    offs = np.zeros(len(ns) + 1, np.uint64)
    offs[1:] = np.cumsum(ns)
    idx = np.repeat(tr.offsets[st] + starts, ns) + (np.arange(int(offs[-1])) - np.repeat(offs[:-1].astype(np.int64), ns))
    return st, starts, offs, tr.tokens[idx].astype(np.int32)


def _append_both(srv, gs, tr, R, handles, lo, hi, chunk=200_000):
    st, starts, offs, toks = _records(tr, R, lo, hi)
    group = (st // R).astype(np.int32)
    rid = (st % R).astype(np.int32)
    ok, ver, ack = gs.append(group, rid, starts.astype(np.uint64), offs, toks)
    # the GPU gets the same records in the same order, in batches of ~chunk records
    for a in range(0, len(st), chunk):
        b = min(len(st), a + chunk)
        o = offs[a:b + 1] - offs[a]
        rep = srv.update_arrays(handles[st[a:b]], rid[a:b], starts[a:b].astype(np.uint64), o,
                                toks[int(offs[a]):int(offs[b])], 0.0)
        assert (rep["ok"] == ok[a:b]).all() and (rep["version"] == ver[a:b]).all() and (rep["acked"] == ack[a:b]).all()
    return len(st)


def _queries(tr, R, indexed, n, rng, plen=6):
    S = len(indexed)
    pool = np.nonzero(indexed >= plen + 1)[0]
    st = pool[rng.integers(0, len(pool), n)]
    pos = plen + (rng.random(n) * (indexed[st] - plen + 1)).astype(np.int64)
    pos = np.minimum(pos, indexed[st])
    pats = np.stack([tr.tokens[tr.offsets[s] + p - plen:tr.offsets[s] + p] for s, p in zip(st, pos)]).astype(np.int32)
    return st, pos, pats


def _compare(srv, gs, tr, R, handles, st, pos, pats, spec, top_k, lim_spec=16):
    n = len(st)
    k_cap = int(top_k.max())
    s_cap = int(min(spec.max(), lim_spec))
    oa = (O.OrcArgs * n)()
    for i in range(n):
        oa[i] = O.make_args(int(spec[i]), 6, 1, int(top_k[i]))
    pat_offs = np.arange(n + 1, dtype=np.uint64) * pats.shape[1]
    nc, ln, sc, sp, tk = gs.speculate((st // R).astype(np.int32), pat_offs, pats.reshape(-1), oa, k_cap, s_cap)
    # GPU: host batch API with fused verification against the stream's true continuation
    args = D.args_array([D.SpeculationArgs(int(spec[i]), 6, 1, int(top_k[i])) for i in range(n)])
    truth = np.zeros((n, s_cap), np.int32)
    tl = np.zeros(n, np.int32)
    for i, (s, p) in enumerate(zip(st, pos)):
        t = tr.stream(s)[p:p + s_cap]
        truth[i, :len(t)] = t
        tl[i] = tr.lengths[s] - p
    v = srv.speculate_view(handles[st], pat_offs, pats.reshape(-1), args, 1, truth=truth, truth_left=tl, limit=tl)
    got_nc = np.diff(v.cand_off)
    assert (got_nc == nc).all(), "candidate counts differ: %d queries" % int((got_nc != nc).sum())
    c0 = v.cand_off[:-1]
    mism = 0
    for j in range(k_cap):
        has = nc > j
        ci = (c0 + j)[has]
        assert (v.cands["len"][ci] == ln[has, j]).all()
        assert (v.cands["score"][ci].view(np.uint64) == sc[has, j].view(np.uint64)).all()
        assert (v.cands["support"][ci] == sp[has, j]).all()
        for q, c in zip(np.nonzero(has)[0], ci):
            L = ln[q, j]
            mism += int((v.tokens[v.tok_off[c]:v.tok_off[c] + L] != tk[q, j, :L]).any())
    assert mism == 0, "%d candidates with different tokens" % mism
    # fused verification == engine.cpp:115-143 restated over the reference's candidates
    dr = (ln * (np.arange(k_cap)[None, :] < nc[:, None])).sum(1)
    acc = np.zeros(n, np.int64)
    for j in range(k_cap):
        cap = np.minimum(ln[:, j], tl)
        m = np.zeros(n, np.int64)
        run = nc > j
        for i in range(s_cap):
            run = run & (i < cap) & (tk[:, j, i] == truth[:, i])
            m += run
        acc = np.maximum(acc, m)
    em = np.minimum(acc + 1, tl)
    assert (v.drafted == dr).all() and (v.emitted == em).all() and (v.accepted == em - 1).all()
    return int(nc.sum())


def _run(cfg_name, ngroups, prefill, n_queries, ticks, top_k_fn, spec_fn, seed):
    base = CONFIGS[cfg_name]
    cfg = dataclasses.replace(base, num_groups=ngroups)  # the first groups of the trace, bit-identical
    tr = generate_workload(cfg)
    R = cfg.group_size
    S = tr.num_streams
    gids = [group_id(g) for g in range(ngroups)]
    gs = O.reference().group_set(gids)
    lens = tr.lengths.astype(np.int64)
    pre = (lens * prefill).astype(np.int64) // REC * REC
    srv = D.DraftServer(D.DgdsParams(), device=0, expected_nodes=int(pre.sum()) * 3, expected_streams=S)
    handles = np.repeat(srv.group_handles(gids), R).astype(np.int32)
    _append_both(srv, gs, tr, R, handles, np.zeros(S, np.int64), pre)
    assert srv.node_count() == gs.node_count()
    assert srv.device_error() == 0
    rng = np.random.default_rng(seed)
    indexed = pre.copy()
    total = 0
    for t in range(ticks + 1):
        if t > 0:  # one record per stream, then queries over everything indexed so far
            nxt = np.minimum(indexed + REC, lens)
            _append_both(srv, gs, tr, R, handles, indexed, nxt)
            indexed = nxt
            assert srv.node_count() == gs.node_count()
        n = n_queries if t == 0 else n_queries // 4
        st, pos, pats = _queries(tr, R, indexed, n, rng)
        total += _compare(srv, gs, tr, R, handles, st, pos, pats, spec_fn(rng, n), top_k_fn(rng, n))
    assert srv.device_error() == 0
    srv.close()
    return total


def test_c2_scale_parity():
    """32 of C2's 256 groups (V 163,840) at 50% prefill, 50,000 queries top-4 draft 8, then 3 ticks."""
    cands = _run("C2", 32, 0.5, 50_000, 3, lambda r, n: np.full(n, 4), lambda r, n: np.full(n, 8), 11)
    assert cands > 50_000


def test_c3_adaptive_draft_len_parity():
    """16 of C3's 128 groups (128x8 shape, V 152,064); per-request max_spec_tokens = d_r of the
    adaptive policy (engine.cpp:78-85: min(cap 8, budget 4096 / n_running)) for n_running drawn
    over a decaying batch, top-1 (AdaptiveSpecPolicy k = 1)."""
    def spec(rng, n):
        running = rng.integers(256, 8192, n)
        return np.array([D.draft_len(True, True, 8, 4096, int(x)) for x in running])
    cands = _run("C3", 16, 0.6, 30_000, 2, lambda r, n: np.ones(n, np.int64), spec, 12)
    assert cands > 10_000


def test_c4_full_streams_parity():
    """4 of C4's 512 groups (16 responses up to 64K tokens) fully appended (R1 as BASELINE.md
    defines it), top-4: long streams exercise extent growth and deep counts."""
    cands = _run("C4", 4, 1.0, 20_000, 0, lambda r, n: np.full(n, 4), lambda r, n: np.full(n, 8), 13)
    assert cands > 20_000
