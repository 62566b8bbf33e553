"""Per-warp K1 timing distribution on the C2 bench step (DGDS_APPEND_DBG=1): is the
append launch set by the median warp chain or by a tail?"""
import ctypes as C, os, sys
import numpy as np
os.environ["DGDS_APPEND_DBG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_14617_b200 import _lib
from paper_2511_14617_b200.dgds import DgdsParams, DraftServer
from paper_2511_14617_b200.workload import CONFIGS, generate_workload, group_id

cfg = CONFIGS["C2"]
tr = generate_workload(cfg)
S = cfg.num_groups * cfg.group_size
srv = DraftServer(DgdsParams(), expected_nodes=600_000_000, expected_streams=S)
hs = np.repeat(srv.group_handles([group_id(g) for g in range(cfg.num_groups)]), cfg.group_size).astype(np.int32)
rid = np.tile(np.arange(cfg.group_size, dtype=np.int32), cfg.num_groups)
pos = np.zeros(S, np.int64)
pre = (tr.lengths * 0.5).astype(np.int64) // 16 * 16


def tick(cap, n_tok):
    live = np.nonzero(pos < cap)[0]
    ns = np.minimum(n_tok, cap[live] - pos[live])
    offs = np.zeros(len(live) + 1, np.uint64); offs[1:] = np.cumsum(ns)
    g0 = tr.offsets[live] + pos[live]
    idx = np.repeat(g0, ns) + (np.arange(int(offs[-1])) - np.repeat(offs[:-1].astype(np.int64), ns))
    srv.update_arrays(hs[live], rid[live], pos[live].astype(np.uint64), offs, np.ascontiguousarray(tr.tokens[idx]), 0.0)
    pos[live] += ns
    return len(live)


while (pos < pre).any():
    tick(pre, 128)
for _ in range(4):
    nw = tick(tr.lengths, 16)
    torch.cuda.synchronize()
    out = np.zeros((65536, 2), np.uint64)
    _lib.check(_lib.lib().dgds_debug_append_timing(srv.handle, out.ctypes.data, 65536))
    t = out[:nw]
    t0 = t[:, 0].min()
    dur = (t[:, 1] - t[:, 0]) / 1e3
    end = (t[:, 1] - t0) / 1e3
    print(f"warps {nw}: chain us median {np.median(dur):.1f} p90 {np.percentile(dur, 90):.1f} p99 {np.percentile(dur, 99):.1f} "
          f"max {dur.max():.1f}; start spread {(t[:, 0].max() - t0) / 1e3:.1f} us; kernel span {end.max():.1f} us")
