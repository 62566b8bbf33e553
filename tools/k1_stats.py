"""Append-path counters on the C2 bench tick (DGDS_K1_STATS=1): claims, leaves, conversions,
rider matches, K1b events and walk lengths per 16-token tick of all 4,096 streams."""
import ctypes as C, os, sys
import numpy as np
os.environ["DGDS_K1_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_14617_b200 import _lib
from paper_2511_14617_b200.dgds import DgdsParams, DraftServer
from paper_2511_14617_b200.workload import CONFIGS, generate_workload, group_id

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
tr = generate_workload(cfg)
S = cfg.num_groups * cfg.group_size
srv = DraftServer(DgdsParams(), expected_nodes=int(tr.tokens.size) * 2, expected_streams=S)
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
    return int(offs[-1])


def stats():
    out = np.zeros(8, np.uint64)
    _lib.check(_lib.lib().dgds_debug_dump(srv.handle, 6, out.ctypes.data, out.nbytes))
    return out.astype(np.int64)


while (pos < pre).any():
    tick(pre, 128)
base = stats()
for _ in range(4):
    a = stats()
    ntok = tick(tr.lengths, 16)
    torch.cuda.synchronize()
    d = stats() - a
    print(f"tick of {ntok} tokens: claims {d[0]} ({d[0]/ntok:.2f}/token), leaves {d[1]}, conversions {d[2]}, rider "
          f"matches {d[3]}, events {d[4]}, walk steps {d[5]} (longest so far {stats()[6]}), walks {d[7]}")
print("entries", srv.entry_count(), "nodes", srv.node_count())
