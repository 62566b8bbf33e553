"""Per-query phase timing of the query kernel (debug hook dgds_debug_query_timing).

  python tools/phase_timing.py C2      # bench.py's step on config C2, prints phase cycles
Profiling aid only (tools/), not part of the product or the bench contract.
"""
import contextlib
import ctypes as C
import io
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
extra = sys.argv[2:]
sys.argv = ["bench.py", "--steps", "3", "--warmup", "1", "--no-cpu-baseline", "--e2e-steps", "0", "--config", cfg] + extra
import bench  # noqa: E402
import paper_2511_14617_b200.dgds as D  # noqa: E402
from paper_2511_14617_b200 import _lib  # noqa: E402

L = _lib.lib()
L.dgds_debug_query_timing.argtypes = [C.c_void_p, C.c_void_p]
q = int(sys.argv[sys.argv.index("--queries") + 1]) if "--queries" in sys.argv else 65536
buf = torch.zeros((q, 8), dtype=torch.int64, device="cuda:0")
state = {"set": False}
_orig = D.DraftServer.update_device


def upd(self, *a, **k):
    if not state["set"]:
        L.dgds_debug_query_timing(self.handle, C.c_void_p(buf.data_ptr()))
        state["set"] = True
    return _orig(self, *a, **k)


D.DraftServer.update_device = upd
f = io.StringIO()
with contextlib.redirect_stdout(f):
    bench.main()
d0 = json.loads(f.getvalue().strip().splitlines()[-1])
print(cfg, "query ms %.4f append ms %.4f nodes %d value %.1f M q/s" % (
    d0["roofline_query"]["avg_launch_ms"], d0["roofline_append"]["avg_launch_ms"], d0["config"]["index_nodes"],
    d0["value"] / 1e6))
torch.cuda.synchronize()
d = buf.cpu().numpy()
d = d[d[:, 0] > 0]
for i, name in enumerate(["phaseA_cyc", "phaseB_cyc", "out_cyc", "depth_it", "child_it", "merge_it", "winner", "nf"]):
    v = d[:, i]
    print(f"{name:12s} mean {v.mean():10.1f} p50 {np.percentile(v, 50):10.1f} p90 {np.percentile(v, 90):10.1f} "
          f"max {v.max()}")
cx = d[d[:, 3] > 0]  # phase B ran: the branching queries (K2b)
print("branching queries:", len(cx), "of", len(d))
for i, name in enumerate(["phaseA_cyc", "phaseB_cyc", "out_cyc", "depth_it", "child_it", "merge_it", "winner", "nf"]):
    v = cx[:, i]
    print(f"  {name:12s} mean {v.mean():10.1f} p50 {np.percentile(v, 50):10.1f} p90 {np.percentile(v, 90):10.1f} "
          f"p99 {np.percentile(v, 99):10.1f} max {v.max()}")
