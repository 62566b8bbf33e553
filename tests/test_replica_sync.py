"""Replica sync: GDX1 delta / full-snapshot blobs and fetch_cst.

- byte-exact blobs: the same operation sequence on the compiled reference DraftServer
  and on ours gives identical (kind, version, blob bytes) for every cached version
  (cst.cpp:233-269, dgds.cpp:53-97), including compaction, expiry, empty streams;
- cross-apply: our blobs restore a reference GroupDraftIndex replica, reference blobs
  restore a GPU replica (cst.cpp:271-321); both answer queries like the source;
- the reference's error behaviour of apply_blob.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_14617_b200 import dgds as D

pytestmark = pytest.mark.gpu


def keys(cs):
    return [c.key() for c in cs]


class RefServer:
    def __init__(self, ref, ttl=600.0):
        self.ref = ref
        self.h = ref.L.orc_ref_server_new(1, 0.0, 16, ttl, 8, 16)

    def update(self, g, r, p, toks, now):
        import ctypes as C
        ok, v, a = C.c_int32(), C.c_uint64(), C.c_uint64()
        arr = np.asarray(toks, np.int32)
        assert self.ref.L.orc_ref_server_update(self.h, g.encode(), r, p, arr.ctypes.data_as(C.POINTER(C.c_int32)),
                                                len(arr), now, C.byref(ok), C.byref(v), C.byref(a)) == 0
        return D.UpdateReply(bool(ok.value), v.value, a.value)

    def fetch(self, g, cached, now):
        return self.ref.server_fetch(self.h, g, cached, now)

    def __del__(self):
        self.ref.L.orc_ref_server_free(self.h)


def _ops(seed, groups=("ga", "gb", "gc"), n_ops=160, vocab=12):
    rng = np.random.default_rng(seed)
    stored = {}
    t = 0.0
    for _ in range(n_ops):
        g = groups[int(rng.integers(len(groups)))]
        r = int(rng.integers(5))
        have = stored.get((g, r), 0)
        kind = rng.random()
        if kind < 0.08:
            prev = have + 3  # out of order: rejected, but creates the stream (cst.cpp:121)
        else:
            prev = have
        n = int(rng.integers(0, 20))
        toks = rng.integers(0, vocab, n).tolist()
        if prev == have:
            stored[(g, r)] = have + n
        t += float(rng.random())
        yield g, r, prev, toks, t


@pytest.mark.parametrize("seed", [1, 2])
def test_fetch_blobs_byte_identical(reference, seed):
    if reference is None:
        pytest.skip("oracle/_ref not built")
    rs = RefServer(reference)
    s = D.DraftServer(D.DgdsParams(shard_count=1), expected_nodes=1 << 16)
    versions = {}
    for k, (g, r, prev, toks, now) in enumerate(_ops(seed)):
        assert s.update_cst(g, r, prev, toks, now) == rs.update(g, r, prev, toks, now)
        versions.setdefault(g, []).append(s.group_version(g))
        if k % 23 == 22:  # checkpoint: every cached version, plus compaction
            for gg, vs in versions.items():
                cur = vs[-1]
                for cached in sorted({0, 1, cur // 2, max(0, cur - 1), cur, cur + 5}):
                    got = s.fetch_cst([gg], [cached], now)[0]
                    kind, ver, blob = rs.fetch(gg, cached, now)
                    assert (got.kind, got.version, got.blob) == (kind, ver, blob), (gg, cached, cur)
            if k % 46 == 45 and "ga" in versions:
                s.compact_group("ga", versions["ga"][-1] // 2)
                reference.server_compact(rs.h, "ga", versions["ga"][-1] // 2)
    # unknown and expired groups
    assert s.fetch_cst(["nope"], [0], 1.0)[0].kind == D.FetchKind.UnknownGroup
    got = s.fetch_cst(["ga"], [0], 1e6)[0]
    kind, ver, blob = rs.fetch("ga", 0, 1e6)
    assert (got.kind, got.version, got.blob) == (kind, ver, blob) == (D.FetchKind.UnknownGroup, 0, b"")


def test_blobs_cross_apply_and_replica_queries(reference):
    if reference is None:
        pytest.skip("oracle/_ref not built")
    from paper_2511_14617_b200.workload import CONFIGS, generate_workload
    tr = generate_workload(CONFIGS["C1"])
    src = D.DraftServer(D.DgdsParams(), expected_nodes=1 << 21)
    rep_gpu = D.DraftServer(D.DgdsParams(), expected_nodes=1 << 21)  # a GPU-resident replica
    ref_idx = reference.index(group_id="g00000")                       # a reference replica
    args = D.SpeculationArgs(8, 6, 1, 4, 0.25, 1)
    oargs = O.make_args(8, 6, 1, 4, 0.25, 1)
    rng = np.random.default_rng(7)
    pos = [0] * 16
    cached_gpu = cached_ref = 0
    for rnd in range(6):
        for _ in range(40):  # appends on the source
            r = int(rng.integers(16))
            n = int(rng.integers(1, 200))
            t = tr.stream(r)[pos[r]:pos[r] + n]
            if len(t):
                assert src.update_cst("g00000", r, pos[r], t, 0.0).ok
                pos[r] += len(t)
        if rnd == 3:
            src.compact_group("g00000", src.group_version("g00000"))  # forces Full for both replicas
        for who in ("gpu", "ref"):
            cached = cached_gpu if who == "gpu" else cached_ref
            f = src.fetch_cst(["g00000"], [cached], 0.0)[0]
            expect_kind = D.FetchKind.Full if cached == 0 or rnd == 3 else D.FetchKind.Delta
            assert f.kind == expect_kind, (rnd, who)
            if who == "gpu":
                cached_gpu = rep_gpu.apply_blob("g00000", f.blob)
                assert cached_gpu == f.version
            else:
                cached_ref = reference.index_apply_blob(ref_idx, f.blob)
                assert cached_ref == f.version
        # the three indexes answer identically
        for _ in range(60):
            r = int(rng.integers(16))
            p = int(rng.integers(1, max(2, pos[r])))
            pat = tr.stream(r)[max(0, p - 6):p]
            want = keys(src.speculate("g00000", pat, args))
            assert keys(rep_gpu.speculate("g00000", pat, args)) == want
            assert keys(ref_idx.speculate(pat, oargs)) == want
        # reference replica -> blob -> GPU replica matches too (full snapshot of the reference)
        snap = reference.index_full_snapshot(ref_idx)
        fresh = D.DraftServer(D.DgdsParams(), expected_nodes=1 << 21)
        assert fresh.apply_blob("g00000", snap) == cached_ref
        assert fresh.fetch_cst(["g00000"], [0], 0.0)[0].blob == snap  # and re-serialises byte-identically


def test_apply_blob_errors_match_reference(reference):
    if reference is None:
        pytest.skip("oracle/_ref not built")
    src = D.DraftServer(D.DgdsParams(), expected_nodes=1 << 16)
    src.update_cst("g1", 0, 0, [1, 2, 3, 4], 0.0)
    v1 = src.group_version("g1")
    src.update_cst("g1", 1, 0, [1, 2, 5], 0.0)
    full = src.fetch_cst(["g1"], [0], 0.0)[0].blob
    delta = src.fetch_cst(["g1"], [v1], 0.0)[0].blob
    rep = D.DraftServer(D.DgdsParams(), expected_nodes=1 << 16)
    ref_idx = reference.index(group_id="g1")
    cases = [
        (b"XDX1" + full[4:], "bad draft blob magic"),
        (full[:-3], "truncated"),
        (delta, "delta expects replica at version 1, replica is at 0"),
        (full[:4] + b"\x09" + full[5:], "unknown draft blob kind"),
    ]
    for blob, msg in cases:
        with pytest.raises(RuntimeError, match=msg):
            rep.apply_blob("g1", blob)
        with pytest.raises(Exception):
            reference.index_apply_blob(ref_idx, blob)
    other = D.DraftServer(D.DgdsParams(), expected_nodes=1 << 16)
    with pytest.raises(RuntimeError, match="draft blob for group g1 applied to g2"):
        other.apply_blob("g2", full)
    assert rep.apply_blob("g1", full) == src.group_version("g1")
    assert rep.fetch_cst(["g1"], [0], 0.0)[0].blob == full


def test_device_and_routed_updates_keep_replica_logs():
    """Device-buffer updates (dgds_update_batch_device) and two-phase routed updates
    (dgds_update_plan_routed, or the planner thread's _async / _take, then dgds_update_launch;
    the next plan is made before the previous launch) append their history-log records after
    the K1 launch. fetch_cst blobs (full and
    delta) stay byte-identical to a host-path twin fed the same records."""
    import ctypes as C
    import torch
    from paper_2511_14617_b200 import _lib
    dev = torch.device("cuda:0")
    L = _lib.lib()
    host = D.DraftServer(D.DgdsParams(), expected_nodes=1 << 16)
    devs = D.DraftServer(D.DgdsParams(), expected_nodes=1 << 16)
    routed = D.DraftServer(D.DgdsParams(), expected_nodes=1 << 16)
    rng = np.random.default_rng(12)
    groups = ["ga", "gb", "gc"]
    stored = {}
    RW = 5 + 16  # routed row: handle, rid, prev lo, prev hi, count, 16 tokens
    pending = None  # routed plan made but not yet launched
    versions = {}
    for rnd in range(8):
        gids, rids, prevs, toks = [], [], [], []
        for _ in range(int(rng.integers(4, 30))):
            g = groups[int(rng.integers(3))]
            r = int(rng.integers(4))
            t = rng.integers(0, 9, int(rng.integers(1, 17))).tolist()
            if any(g == a and r == b for a, b in zip(gids, rids)):
                continue  # one record per stream per batch keeps the twins' batches identical
            gids.append(g)
            rids.append(r)
            prevs.append(stored.get((g, r), 0))
            toks.append(t)
            stored[(g, r)] = stored.get((g, r), 0) + len(t)
        now = float(rnd)
        rh = host.update_batch(gids, rids, prevs, toks, now)
        # device-buffer path
        hd = devs.group_handles(gids)
        offs = np.zeros(len(toks) + 1, np.uint64)
        offs[1:] = np.cumsum([len(t) for t in toks])
        d_tok = torch.tensor(np.concatenate(toks).astype(np.int32), device=dev)
        rd = devs.update_device(hd, np.array(rids, np.int32), np.array(prevs, np.uint64), offs, d_tok.data_ptr(), now)
        assert [(x.ok, x.version, x.acked_tokens) for x in rh] == [(bool(a), int(b), int(c)) for a, _, b, c in rd]
        # routed path: plan this round; launch the previous round's plan after it
        hr = routed.group_handles(gids)
        n = len(gids)
        meta = np.zeros((n, 5), np.int32)
        rows = np.zeros((n, RW), np.int32)
        for i in range(n):
            meta[i] = [hr[i], rids[i], prevs[i] & 0xFFFFFFFF, prevs[i] >> 32, len(toks[i])]
            rows[i, :5] = meta[i]
            rows[i, 5:5 + len(toks[i])] = toks[i]
        d_rows = torch.from_numpy(rows).to(dev)
        counts = np.array([n], np.int32)
        nrej = C.c_int64()
        plan = C.c_void_p()
        if rnd % 2:  # the server's planner thread (dgds_update_plan_routed_async / _take)
            job = C.c_uint64()
            _lib.check(L.dgds_update_plan_routed_async(routed.handle, None, 1, n, counts.ctypes.data,
                                                       meta.ctypes.data, 5, C.c_void_p(d_rows.data_ptr()), RW, now,
                                                       C.byref(job)))
            _lib.check(L.dgds_update_plan_take(routed.handle, job.value, C.byref(nrej), C.byref(plan)))
        else:
            _lib.check(L.dgds_update_plan_routed(routed.handle, 1, n, counts.ctypes.data, meta.ctypes.data, 5,
                                                 C.c_void_p(d_rows.data_ptr()), RW, now, C.byref(nrej),
                                                 C.byref(plan)))
        assert nrej.value == 0
        if pending is not None:
            _lib.check(L.dgds_update_launch(routed.handle, pending[0], None))
        pending = (plan, d_rows)
        for g in set(gids):
            versions.setdefault(g, []).append(host.group_version(g))
        if rnd % 3 == 2:
            _lib.check(L.dgds_update_launch(routed.handle, pending[0], None))
            pending = None
            torch.cuda.synchronize()
            for g in groups:
                if g not in versions:
                    continue
                for cached in sorted({0, versions[g][0], versions[g][-1] // 2}):
                    want = host.fetch_cst([g], [cached], now)[0]
                    for other in (devs, routed):
                        got = other.fetch_cst([g], [cached], now)[0]
                        assert (got.kind, got.version, got.blob) == (want.kind, want.version, want.blob), (g, cached)
