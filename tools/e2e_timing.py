"""Break down the host-buffer (e2e) path: python prep, update_batch, speculate_verify_batch."""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14617_b200 import _lib
from paper_2511_14617_b200.dgds import DgdsParams, DraftServer, SpeculationArgs, args_array, CandidateBatch
from paper_2511_14617_b200.workload import CONFIGS, generate_workload, group_id

cfg = CONFIGS["C2"]
tr = generate_workload(cfg)
S = cfg.num_groups * cfg.group_size
srv = DraftServer(DgdsParams(), expected_nodes=200_000_000, expected_streams=S)
hs = np.repeat(srv.group_handles([group_id(g) for g in range(cfg.num_groups)]), cfg.group_size).astype(np.int32)
rid = np.tile(np.arange(cfg.group_size, dtype=np.int32), cfg.num_groups)
pos = np.zeros(S, np.int64)
L = _lib.lib()
Q, kq, dl = 65536, 4, 8
rng = np.random.default_rng(0)
sp_args = args_array([SpeculationArgs(dl, 6, 1, kq, 0.25, 1)])
cb = CandidateBatch(Q, kq, dl)
dr = np.zeros(Q, np.int32); ac = np.zeros(Q, np.int32); em = np.zeros(Q, np.int32)
vo = _lib.VerifyOut(dr.ctypes.data, ac.ctypes.data, em.ctypes.data)
for step in range(12):
    t0 = time.perf_counter()
    live = np.nonzero(pos < tr.lengths)[0]
    ns = np.minimum(64, tr.lengths[live] - pos[live])
    offs = np.zeros(len(live) + 1, np.uint64); offs[1:] = np.cumsum(ns)
    g0 = tr.offsets[live] + pos[live]
    idx = np.repeat(g0, ns) + (np.arange(int(offs[-1])) - np.repeat(offs[:-1].astype(np.int64), ns))
    toks = np.ascontiguousarray(tr.tokens[idx]); prev = pos[live].astype(np.uint64)
    st = rng.integers(0, S, Q); st = st[pos[st] + ns.max() > 8][:Q]
    st = np.resize(st, Q); qp = np.maximum(6, (rng.random(Q) * np.maximum(pos[st], 7)).astype(np.int64))
    qp = np.minimum(qp, np.maximum(pos[st], 6))
    base = tr.offsets[st] + qp
    pat = np.stack([tr.tokens[base - 6 + j] for j in range(6)], 1).astype(np.int32).reshape(-1)
    poff = np.arange(0, 6 * Q + 1, 6, dtype=np.uint64)
    tl = np.maximum(1, (tr.lengths[st] - qp)).astype(np.int32)
    tru = np.zeros((Q, dl), np.int32)
    qh = hs[st].copy()
    t1 = time.perf_counter()
    srv.update_arrays(hs[live], rid[live], prev, offs, toks, 0.0)
    t2 = time.perf_counter()
    if os.environ.get("E2E_VIEW"):
        v = _lib.ResultView()
        _lib.check(L.dgds_speculate_verify_view(srv.handle, Q, qh.ctypes.data, poff.ctypes.data, pat.ctypes.data,
                                                 sp_args.ctypes.data, 0, tru.ctypes.data, dl, tl.ctypes.data,
                                                 tl.ctypes.data, C.byref(v)))
    else:
        _lib.check(L.dgds_speculate_verify_batch(srv.handle, Q, qh.ctypes.data, poff.ctypes.data, pat.ctypes.data,
                                                  sp_args.ctypes.data, 0, tru.ctypes.data, dl, tl.ctypes.data,
                                                  tl.ctypes.data, C.byref(cb.c()), C.byref(vo)))
    t3 = time.perf_counter()
    pos[live] += ns
    print(f"step {step}: prep {1e3*(t1-t0):.2f} ms  update {1e3*(t2-t1):.2f} ms ({len(live)} recs, {int(offs[-1])} tok)  "
          f"speculate_verify {1e3*(t3-t2):.2f} ms")
