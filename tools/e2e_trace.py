"""Device timeline of the host-buffer (e2e) tick: update_batch + speculate_verify_view, under the
torch profiler (CUPTI sees our kernels and copies). Writes gpurun_out/e2e_trace.json and prints
the last tick's events."""
import ctypes as C, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14617_b200 import _lib
from paper_2511_14617_b200.dgds import DgdsParams, DraftServer, SpeculationArgs, args_array
from paper_2511_14617_b200.workload import CONFIGS, generate_workload, group_id

cfg = CONFIGS["C2"]
tr = generate_workload(cfg)
S = cfg.num_groups * cfg.group_size
srv = DraftServer(DgdsParams(), expected_nodes=600_000_000, expected_streams=S)
hs = np.repeat(srv.group_handles([group_id(g) for g in range(cfg.num_groups)]), cfg.group_size).astype(np.int32)
rid = np.tile(np.arange(cfg.group_size, dtype=np.int32), cfg.group_size and cfg.num_groups)
pos = np.zeros(S, np.int64)
L = _lib.lib()
Q, kq, dl, rt = 65536, 4, 8, 16
rng = np.random.default_rng(0)
sp_args = args_array([SpeculationArgs(dl, 6, 1, kq, 0.25, 1)])
v = _lib.ResultView()


def tick(n_tok):
    live = np.nonzero(pos < tr.lengths)[0]
    ns = np.minimum(n_tok, tr.lengths[live] - pos[live])
    offs = np.zeros(len(live) + 1, np.uint64); offs[1:] = np.cumsum(ns)
    g0 = tr.offsets[live] + pos[live]
    idx = np.repeat(g0, ns) + (np.arange(int(offs[-1])) - np.repeat(offs[:-1].astype(np.int64), ns))
    toks = np.ascontiguousarray(tr.tokens[idx]); prev = pos[live].astype(np.uint64)
    st = rng.integers(0, S, Q)
    qp = np.maximum(6, (rng.random(Q) * np.maximum(pos[st], 7)).astype(np.int64))
    qp = np.minimum(qp, np.maximum(pos[st], 6))
    base = tr.offsets[st] + qp
    pat = np.stack([tr.tokens[base - 6 + j] for j in range(6)], 1).astype(np.int32).reshape(-1)
    poff = np.arange(0, 6 * Q + 1, 6, dtype=np.uint64)
    tl = np.maximum(1, (tr.lengths[st] - qp)).astype(np.int32)
    tru = np.zeros((Q, dl), np.int32)
    qh = hs[st].copy()
    srv.update_arrays(hs[live], rid[live], prev, offs, toks, 0.0)
    _lib.check(L.dgds_speculate_verify_view(srv.handle, Q, qh.ctypes.data, poff.ctypes.data, pat.ctypes.data,
                                            sp_args.ctypes.data, 0, tru.ctypes.data, dl, tl.ctypes.data,
                                            tl.ctypes.data, C.byref(v)))
    pos[live] += ns


for _ in range(16):  # prefill-ish: 16 x 128 tokens
    tick(128)
for _ in range(3):
    tick(rt)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as p:
    for _ in range(3):
        tick(rt)
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
p.export_chrome_trace("gpurun_out/e2e_trace.json")
t = json.load(open("gpurun_out/e2e_trace.json"))
ev = [e for e in t["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset", "cuda_runtime")]
ev.sort(key=lambda e: e["ts"])
gpu = [e for e in ev if e.get("cat") != "cuda_runtime"]
t0 = gpu[-16]["ts"] if len(gpu) > 16 else gpu[0]["ts"]
for e in [x for x in ev if x["ts"] >= t0 - 2000]:
    kind = "GPU" if e.get("cat") != "cuda_runtime" else "cpu"
    print(f"{kind} {e['ts'] - t0:9.1f} {e['dur']:8.1f} {e['ts'] - t0 + e['dur']:9.1f} s{e['args'].get('stream', '')} {e['name'][:60]}")
