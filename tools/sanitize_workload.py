"""A small workload that launches every sm_100a kernel of the library, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; logs in profiles/r2_sanitizer_*.log):

  k_stage, k_append (K1), k_walks (K1b)       several append batches incl. extent growth
  k_query modes 0 / 1 / 2 (K2a, K2b, K3)     host API, device API with fused verify + counters
  decode step                                 dgds_decode_step_device
  k_rebuild_*, k_remap_active, k_node_count   a forced growth rebuild, drop + compaction
  k_blob_fill, k_copy_pieces                  fetch_cst blobs, memory compaction
  k_px_* (peer exchange)                      two ranks in one process on one GPU
Results are checked against the CPU restatement so a sanitizer run is also a parity run.
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402
from paper_2511_14617_b200 import _lib  # noqa: E402
from paper_2511_14617_b200 import dgds as D  # noqa: E402
from paper_2511_14617_b200.workload import WorkloadConfig, generate_workload  # noqa: E402


def main():
    import torch
    tr = generate_workload(WorkloadConfig(num_groups=3, group_size=4, location=300.0, scale=0.3,
                                          pattern_similarity=0.8, vocab_size=40, max_tokens=600, seed=3))
    s = D.DraftServer(D.DgdsParams(), device=0, expected_nodes=256, expected_streams=8)  # small: rebuilds
    ref = {g: O.restatement().index("g%05d" % g) for g in range(3)}
    pos = np.zeros(tr.num_streams, np.int64)
    for rnd in range(12):  # a few records per stream per batch
        gids, rids, prevs, toks = [], [], [], []
        for st in range(tr.num_streams):
            g, r = divmod(st, 4)
            n = int(min(7 + rnd, tr.lengths[st] - pos[st]))
            if n <= 0:
                continue
            t = tr.stream(st)[pos[st]:pos[st] + n]
            gids.append("g%05d" % g)
            rids.append(r)
            prevs.append(int(pos[st]))
            toks.append(t)
            ref[g].append(r, int(pos[st]), t)
            pos[st] += n
        reps = s.update_batch(gids, rids, prevs, toks, 0.0)
        assert all(x.ok for x in reps)
    rng = np.random.default_rng(1)
    qg, qp, exp = [], [], []
    for _ in range(300):
        st = int(rng.integers(0, tr.num_streams))
        p = int(rng.integers(1, pos[st] + 1))
        pat = tr.stream(st)[max(0, p - 6):p]
        qg.append("g%05d" % (st // 4))
        qp.append(pat)
        exp.append([c.key() for c in ref[st // 4].speculate(pat, O.make_args(8, 6, 1, 4))])
    got = s.speculate_batch(qg, qp, D.SpeculationArgs(8, 6, 1, 4))
    assert [[c.key() for c in x] for x in got] == exp
    assert s.node_count() == sum(r.node_count for r in ref.values())
    # device API with fused verify and counters
    dev = torch.device("cuda:0")
    n = len(qg)
    h = torch.from_numpy(s.group_handles(qg).astype(np.int32)).to(dev)
    pl = torch.tensor([len(p) for p in qp], dtype=torch.int32, device=dev)
    pat = np.zeros((n, 8), np.int32)
    for i, p in enumerate(qp):
        pat[i, :len(p)] = p
    d_pat = torch.from_numpy(pat).to(dev)
    d_args = torch.from_numpy(D.args_array([D.SpeculationArgs(8, 6, 1, 4)]).view(np.uint8)).to(dev)
    K, S = 4, 8
    out = [torch.zeros(n, dtype=torch.int32, device=dev), torch.zeros(n * K, dtype=torch.int32, device=dev),
           torch.zeros(n * K, dtype=torch.float64, device=dev), torch.zeros(n * K, dtype=torch.int64, device=dev),
           torch.zeros(n * K * S, dtype=torch.int32, device=dev)]
    tru = torch.zeros((n, S), dtype=torch.int32, device=dev)
    tl = torch.full((n,), 5, dtype=torch.int32, device=dev)
    v = torch.zeros((3, n), dtype=torch.int32, device=dev)
    stats = torch.zeros(8, dtype=torch.int64, device=dev)
    cand = _lib.Candidates(K, S, *[x.data_ptr() for x in out])
    vo = _lib.VerifyOut(v[0].data_ptr(), v[1].data_ptr(), v[2].data_ptr())
    p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    cs = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(_lib.lib().dgds_speculate_device(s.handle, n, p(h), p(pl), p(d_pat), 8, p(d_args), 0, K, S,
                                                C.byref(cand), p(tru), S, p(tl), p(tl), C.byref(vo), p(stats), cs))
    # decode step on the device
    gen = pl.clone()
    pol = _lib.SpecPolicy(1, 1, 64, 8, 2, 0)
    sa = _lib.SpecArgs(0, 6, 1, 1, 0.25, 1)
    d_next = torch.zeros(1, dtype=torch.int32, device=dev)
    tot = torch.zeros(4, dtype=torch.int64, device=dev)
    _lib.check(_lib.lib().dgds_decode_step_device(s.handle, n, p(h), p(d_pat), 8, p(gen), p(tl), p(tru), S, p(tl),
                                                  C.byref(sa), C.byref(pol), None, 4, C.byref(cand), C.byref(vo),
                                                  p(d_next), p(tot), cs))
    torch.cuda.synchronize()
    # replica blobs, drop + compaction
    s.fetch_cst(["g00000", "g00001"], [0, 0], 0.0)
    s.drop_group("g00002")
    s.compact_memory()
    got = s.speculate_batch(qg[:50], qp[:50], D.SpeculationArgs(8, 6, 1, 4))
    for i in range(50):
        if qg[i] != "g00002":
            assert [c.key() for c in got[i]] == exp[i]
    assert s.device_error() == 0
    s.close()
    # peer exchange (two ranks in one process): the exchange kernels
    from paper_2511_14617_b200.peer import PeerExchange
    pxs = PeerExchange.local_group(2, 0, {"q": (64, 21)})
    for px in pxs:
        px.set_timeout(5.0)
    recs = [torch.randint(0, 100, (40, 21), dtype=torch.int32, device=dev) for _ in range(2)]
    owners = [torch.randint(0, 2, (40,), dtype=torch.int32, device=dev) for _ in range(2)]
    for r in range(2):
        pxs[r].send("q", owners[r], recs[r], 1, stable=True)
    for r in range(2):
        pxs[r].wait("q", 1)
    torch.cuda.synchronize()
    for px in pxs:
        assert px.overflow.item() == 0
        px.close()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
