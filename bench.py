"""Benchmark of the DGDS hot path (BASELINE.json metric: draft queries/s and
appended tokens/s, % of HBM roofline).

One STEP is one draft-server tick on synthetic grouped-rollout traffic of the
chosen config (default C2 Moonlight-shaped):
  * append phase: the next 16-token record (DraftClient flush size,
    dgds.hpp:21) of every stream that still has tokens;
  * query phase: Q draft queries (R1 regime: pattern = the 6 tokens before a
    random position of a random stream's indexed prefix), top-4 / draft 8,
    with fused verification against the stream's ground truth.
The index is prefilled (untimed) with the first half of every response.

  python bench.py [--gpus N --steps K --warmup W]      # our sm_100a path
  python bench.py --impl reference ...                 # reference CPU arm (oracle/_ref)

Prints ONE JSON line on rank 0. Multi-GPU: torchrun, one rank per GPU; groups
are owned by fnv1a64(group_id) % N (dgds.cpp:10-14) and every rank's queries
and appends are routed to the owner with NCCL all-to-all.
"""
from __future__ import annotations

import argparse
import ctypes as C
import gc
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_CONFIG = "C2"
# Measured random 32-B access ceiling of this pool's B200 (tools/chase.cu,
# profiles/r1_microbench.md): 36.1 G accesses/s = 1155 GB/s of useful sectors.
RANDOM_CEILING_GBS = 1155.0
# dram__bytes_read.sum + dram__bytes_write.sum per launch, from one `ncu --set full` capture of
# the same command (profiles/r2_summary.md); a capture constant, not measured in this run.
QUERY_TRAFFIC = {"value": 63374336 + 1956864 + 28820736 + 26624,
                 "source": "capture constant: ncu --set full prof_query_r2f (K2a + K2b, read + write), profiles/r2_summary.md"}
APPEND_TRAFFIC = {"value": 903936 + 24150272 + 882944 + 4275200 + 512,
                  "source": "capture constant: ncu --set full prof_append_r2e (k_stage + K1 + K1b, read + write), "
                            "profiles/r2_summary.md"}
CONFIG_NAMES = {
    "C1": "single group 16 x 4K, vocab 32K",
    "C2": "Moonlight-shaped 256 groups x 16 responses <=32K tokens, vocab 163840",
    "C3": "Qwen2-VL-72B-shaped 128 groups x 8 responses, 16K, vocab 152064",
    "C4": "Kimi-K2-shaped long-CoT 512 groups x 16 responses <=64K, vocab 163840",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIG_NAMES))
    ap.add_argument("--queries", type=int, default=65536, help="draft queries per step (per rank)")
    ap.add_argument("--record-tokens", type=int, default=16)
    ap.add_argument("--top-k", type=int, default=4)
    ap.add_argument("--draft-len", type=int, default=8)
    ap.add_argument("--prefill", type=float, default=0.5)
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-groups", type=int, default=0,
                    help="groups in the bounded CPU sample (0: 8 per host thread, at most all)")
    ap.add_argument("--no-lines", action="store_true", help="skip the c5_sweep / c3_adaptive / c2_full lines")
    ap.add_argument("--cpu-steps", type=int, default=8)
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: replicate the config's group set per GPU (weak) or shard it (strong, e.g. C4)")
    ap.add_argument("--route", default="px", choices=["px", "nccl"],
                    help="N>1 owner routing: NVLink peer-memory exchange fused into the kernels (px) "
                         "or NCCL all_to_all_single (nccl, the library baseline)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML, sampled from a thread)

class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            if os.environ.get("DGDS_NO_CLOCKS") == "1":  # debug only: a run without clock samples is invalid
                raise RuntimeError("clock sampling disabled")
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.002)

    def __enter__(self):
        # the timed region runs without the cyclic GC (a collection is a multi-ms host stall,
        # and at N>1 one rank's stall holds every rank at the next exchange); callers collect
        # before their barrier, so the ranks enter the region together
        gc.disable()
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()
            self._sample()  # the region's last state (its end event is already recorded and synced)
        gc.enable()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def append_alg_bytes(start: np.ndarray, n: np.ndarray, D: int = 24) -> int:
    """B_app = 4 + 64 * min(D, t+1) per token at stream position t (vectorised)."""
    start = np.asarray(start, np.int64)
    n = np.asarray(n, np.int64)
    keep = n > 0
    lo, hi, n = start[keep] + 1, start[keep] + n[keep], n[keep]  # t+1 ranges over lo..hi
    top = np.minimum(hi, D)
    ramp = np.where(lo <= D, (lo + top) * (top - lo + 1) // 2, 0)
    flat = np.where(hi > D, (hi - np.maximum(lo, D + 1) + 1) * D, 0)
    return int((4 * n + 64 * (ramp + flat)).sum())


# ---------------------------------------------------------------------------
# synthetic schedule shared by both arms

class Schedule:
    def __init__(self, args, cfg_name, rank=0):
        from paper_2511_14617_b200.workload import CONFIGS, generate_workload, group_id
        self.cfg = CONFIGS[cfg_name]
        t0 = time.time()
        self.tr = generate_workload(self.cfg)
        self.gen_s = time.time() - t0
        self.G, self.R = self.cfg.num_groups, self.cfg.group_size
        self.S = self.G * self.R
        self.gids = [group_id(g) for g in range(self.G)]
        lens = self.tr.lengths
        self.prefill = (lens * args.prefill).astype(np.int64) // args.record_tokens * args.record_tokens
        self.rt = args.record_tokens
        self.rng = np.random.default_rng(args.seed + 7919 * rank)

    def queries(self, q, streams=None):
        """R1 queries: random stream, random position in [6, prefill]."""
        pool = np.arange(self.S) if streams is None else np.asarray(streams)
        pool = pool[self.prefill[pool] >= 7]
        st = pool[self.rng.integers(0, len(pool), q)]
        pos = 6 + (self.rng.random(q) * (self.prefill[st] - 6 + 1)).astype(np.int64)
        pos = np.minimum(pos, self.prefill[st])
        return st.astype(np.int64), pos


# ---------------------------------------------------------------------------
# reference CPU arm

def ref_lib():
    from oracle import oracle as O
    R = O.reference()
    if R is None:
        return None, "oracle/_ref/libdgds_ref.so not built (reference sources unavailable at build time)"
    return R, None


_BENCH_CFG = None


def bench_cfg_type():
    global _BENCH_CFG
    if _BENCH_CFG is None:
        from oracle.oracle import OrcArgs

        class BenchCfg(C.Structure):
            _fields_ = [("threads", C.c_int32), ("n_streams", C.c_int32), ("group_size", C.c_int32),
                        ("steps", C.c_int32), ("record_tokens", C.c_int32), ("queries_per_step", C.c_int32),
                        ("max_pattern_len", C.c_int32), ("max_spec_len", C.c_int32), ("pad_", C.c_int32),
                        ("args", OrcArgs)]
        _BENCH_CFG = BenchCfg
    return _BENCH_CFG


def run_reference_cpu(args, sched: Schedule, n_groups: int, steps: int, q_per_step: int, threads: int):
    """Reference GroupDraftIndex, thread-per-shard over `threads` host cores, on the
    first n_groups groups of the same trace. Returns per-phase rates."""
    from oracle import oracle as O
    R, why = ref_lib()
    if R is None:
        raise RuntimeError(why)
    L = R.L
    BenchCfg = bench_cfg_type()
    if not hasattr(L, "_bench_set"):
        L.orc_ref_bench.argtypes = [C.POINTER(BenchCfg), C.POINTER(C.c_char_p), C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p]
        L._bench_set = True
    ng = min(n_groups, sched.G)
    S = ng * sched.R
    tr = sched.tr
    toks = np.ascontiguousarray(tr.tokens[:tr.offsets[S]], np.int32)
    offs = np.ascontiguousarray(tr.offsets[:S + 1], np.int64)
    pre = np.ascontiguousarray(sched.prefill[:S], np.int64)
    rng = np.random.default_rng(args.seed + 1)
    pool = np.nonzero(pre >= 7)[0]
    qs = pool[rng.integers(0, len(pool), steps * q_per_step)].astype(np.int32)
    qp = (6 + (rng.random(len(qs)) * (pre[qs] - 6 + 1)).astype(np.int64))
    qp = np.minimum(qp, pre[qs]).astype(np.int64)
    gids = (C.c_char_p * ng)(*[g.encode() for g in sched.gids[:ng]])
    cfg = BenchCfg(threads, S, sched.R, steps, sched.rt, q_per_step, 8, 16, 0,
                   O.make_args(args.draft_len, 6, 1, args.top_k, 0.25, 1))
    out = np.zeros(2 + 4 * steps, np.float64)
    rc = L.orc_ref_bench(C.byref(cfg), gids, toks.ctypes.data, offs.ctypes.data, pre.ctypes.data, qs.ctypes.data,
                         qp.ctypes.data, out.ctypes.data)
    if rc != 0:
        raise RuntimeError(L.orc_last_error().decode())
    per = out[2:].reshape(steps, 4)
    app_s, app_t, q_s, q_n = per[:, 0].sum(), per[:, 1].sum(), per[:, 2].sum(), per[:, 3].sum()
    return {"prefill_s": out[0], "prefill_tokens": out[1], "append_s": app_s, "append_tokens": app_t,
            "query_s": q_s, "queries": q_n, "step_s": app_s + q_s, "groups": ng, "streams": S}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_sample_groups(args, sched) -> int:
    """Whole groups in the bounded CPU sample: 8 per host thread (thread-per-shard balance), or
    --cpu-groups, at most the whole trace."""
    threads = os.cpu_count() or 1
    return min(args.cpu_groups or 8 * threads, sched.G)


def main_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    R, why = ref_lib()
    cfg_name = args.config
    if R is None:
        print(json.dumps({"impl": "reference", "unavailable": why}))
        return
    sched = Schedule(args, cfg_name)
    threads = os.cpu_count() or 1
    # step = the same tick as our arm, on a bounded sample of whole groups; queries
    # scale with the sample so the queries:appended-tokens mix matches
    ng = cpu_sample_groups(args, sched)
    frac = ng / sched.G
    q = max(1, int(args.queries * frac))
    r = run_reference_cpu(args, sched, ng, args.steps + args.warmup, q, threads)
    qps = r["queries"] / r["step_s"]
    line = {
        "impl": "reference", "metric": "draft_queries_per_s", "value": qps, "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * r["step_s"] / (args.steps + args.warmup), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "i32+f64", "data": "synthetic",
        "append_tokens_per_s": r["append_tokens"] / r["step_s"],
        "query_phase_qps": r["queries"] / r["query_s"], "append_phase_tokens_per_s": r["append_tokens"] / r["append_s"],
        "config": {"workload": f"{cfg_name}: {CONFIG_NAMES[cfg_name]}", "queries_per_step": q,
                   "record_tokens": args.record_tokens, "top_k": args.top_k, "draft_len": args.draft_len,
                   "prefill": args.prefill, "sample_groups": ng},
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "reference",
                         "sample": f"{ng} of {sched.G} groups ({r['streams']} streams), prefill "
                                   f"{int(r['prefill_tokens'])} tokens, {args.steps + args.warmup} steps of "
                                   f"{q} queries + 1 record/stream; {cpu_model()}"},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# our arm

def main_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2511_14617_b200 import _lib
    from paper_2511_14617_b200.dgds import ARGS_DTYPE, DgdsParams, DraftServer, SpeculationArgs, args_array

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("NCCL_DEBUG", "WARN")  # stdout carries exactly one JSON line
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import datetime
        # short collective timeout: a failing rank must not leave its peers spinning on the box
        dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=120))
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    if world > 1:
        from bench_multi import run_multi  # routed multi-GPU step
        return run_multi(args, world, rank, local, dev)

    sched = Schedule(args, args.config)
    tr = sched.tr
    S = sched.S
    # ---- server + untimed prefill (host API, 16-token records, round-robin) ----
    idx_tokens = int(sched.prefill.sum()) + S * args.record_tokens * (args.steps + args.warmup + 2 * args.e2e_steps + 4)
    # table entries: ~1.8 per token on these traces (nodes seen twice + leaves), sized with headroom
    srv = DraftServer(DgdsParams(), device=local, expected_nodes=min(idx_tokens * 3, 1_900_000_000),
                      expected_streams=S)
    handles_of_stream = np.repeat(srv.group_handles(sched.gids), sched.R).astype(np.int32)
    rid_of_stream = np.tile(np.arange(sched.R, dtype=np.int32), sched.G)
    t0 = time.time()
    chunk = 8 * args.record_tokens
    pos = np.zeros(S, np.int64)
    while True:
        live = np.nonzero(pos < sched.prefill)[0]
        if len(live) == 0:
            break
        n_rec = np.minimum((sched.prefill[live] - pos[live] + args.record_tokens - 1) // args.record_tokens, 8)
        recs_stream = np.repeat(live, n_rec)
        k_in = np.arange(len(recs_stream)) - np.repeat(np.cumsum(n_rec) - n_rec, n_rec)
        starts = pos[recs_stream] + k_in * args.record_tokens
        ns = np.minimum(args.record_tokens, sched.prefill[recs_stream] - starts)
        offs = np.zeros(len(ns) + 1, np.uint64)
        offs[1:] = np.cumsum(ns)
        g0 = tr.offsets[recs_stream] + starts
        idx = np.repeat(g0, ns) + (np.arange(int(offs[-1])) - np.repeat(offs[:-1].astype(np.int64), ns))
        rep = srv.update_arrays(handles_of_stream[recs_stream], rid_of_stream[recs_stream], starts.astype(np.uint64),
                                offs, tr.tokens[idx], 0.0)
        assert rep["ok"].all()
        pos[live] += np.minimum(sched.prefill[live] - pos[live], chunk)
    torch.cuda.synchronize()
    prefill_s = time.time() - t0

    # ---- per-step inputs, resident in HBM before timing ----
    K, W = args.steps, args.warmup
    Q = args.queries
    kq, dl = args.top_k, args.draft_len
    sp_args = args_array([SpeculationArgs(dl, 6, 1, kq, 0.25, 1)])
    d_args = torch.from_numpy(sp_args.view(np.uint8).copy()).to(dev)
    steps_in = []
    spos = pos.copy()
    for s in range(W + K):
        live = np.nonzero(spos < tr.lengths)[0]
        ns = np.minimum(args.record_tokens, tr.lengths[live] - spos[live])
        offs = np.zeros(len(live) + 1, np.uint64)
        offs[1:] = np.cumsum(ns)
        g0 = tr.offsets[live] + spos[live]
        idx = np.repeat(g0, ns) + (np.arange(int(offs[-1])) - np.repeat(offs[:-1].astype(np.int64), ns))
        d_tok = torch.from_numpy(tr.tokens[idx]).to(dev)
        app = dict(h=handles_of_stream[live], r=rid_of_stream[live], prev=spos[live].astype(np.uint64), offs=offs,
                   d_tok=d_tok, alg=append_alg_bytes(spos[live], ns), ntok=int(offs[-1]))
        spos[live] += ns
        st, qpos = sched.queries(Q)
        pat = np.zeros((Q, 8), np.int32)
        tru = np.zeros((Q, dl), np.int32)
        base = tr.offsets[st] + qpos
        for j in range(6):
            pat[:, j] = tr.tokens[base - 6 + j]
        tl = (tr.lengths[st] - qpos).astype(np.int32)
        for j in range(dl):
            ok = j < tl
            tru[ok, j] = tr.tokens[(base + j)[ok]]
        qd = dict(h=torch.from_numpy(handles_of_stream[st]).to(dev),
                  pl=torch.full((Q,), 6, dtype=torch.int32, device=dev),
                  pat=torch.from_numpy(pat).to(dev), tru=torch.from_numpy(tru).to(dev),
                  tl=torch.from_numpy(tl).to(dev), lim=torch.from_numpy(tl).to(dev))
        steps_in.append((app, qd))
    out = dict(nc=torch.zeros(Q, dtype=torch.int32, device=dev), ln=torch.zeros(Q * kq, dtype=torch.int32, device=dev),
               sc=torch.zeros(Q * kq, dtype=torch.float64, device=dev),
               sp=torch.zeros(Q * kq, dtype=torch.int64, device=dev),
               tk=torch.zeros(Q * kq * dl, dtype=torch.int32, device=dev),
               v=torch.zeros((3, Q), dtype=torch.int32, device=dev))
    d_stats = torch.zeros(8, dtype=torch.int64, device=dev)
    cand = _lib.Candidates(kq, dl, out["nc"].data_ptr(), out["ln"].data_ptr(), out["sc"].data_ptr(),
                           out["sp"].data_ptr(), out["tk"].data_ptr())
    vo = _lib.VerifyOut(out["v"][0].data_ptr(), out["v"][1].data_ptr(), out["v"][2].data_ptr())
    L = _lib.lib()
    sstream = srv.cuda_stream
    ext = torch.cuda.ExternalStream(sstream, device=dev)

    def step(s, stats):
        app, qd = steps_in[s]
        # on the server's own stream (dgds_cuda_stream): no cross-stream joins per call
        srv.update_device(app["h"], app["r"], app["prev"], app["offs"], app["d_tok"].data_ptr(), 0.0, sstream)
        _lib.check(L.dgds_speculate_device(
            srv.handle, Q, C.c_void_p(qd["h"].data_ptr()), C.c_void_p(qd["pl"].data_ptr()),
            C.c_void_p(qd["pat"].data_ptr()), 8, C.c_void_p(d_args.data_ptr()), 0, kq, dl, C.byref(cand),
            C.c_void_p(qd["tru"].data_ptr()), dl, C.c_void_p(qd["tl"].data_ptr()), C.c_void_p(qd["lim"].data_ptr()),
            C.byref(vo), C.c_void_p(d_stats.data_ptr()) if stats else None, C.c_void_p(sstream)))

    torch.cuda.synchronize()  # inputs were built on torch's stream; the steps run on the server's
    for s in range(W):
        step(s, False)
    torch.cuda.synchronize()
    prof = _lib.Profile()
    _lib.check(L.dgds_profile_enable(srv.handle, 1))
    _lib.check(L.dgds_profile_read(srv.handle, C.byref(prof), 1))
    d_stats.zero_()
    gc.collect()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    tp = None
    if os.environ.get("DGDS_DEVICE_TRACE"):  # debug only: device timeline of the timed steps (numbers then invalid)
        from torch.profiler import ProfilerActivity, profile
        tp = profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA])
        tp.__enter__()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        kl0 = L.dgds_kernel_launches()
        e0.record(ext)
        for s in range(W, W + K):
            step(s, True)
        e1.record(ext)
        kl1 = L.dgds_kernel_launches()
        torch.cuda.synchronize()
        w1 = time.perf_counter()
    if tp is not None:
        tp.__exit__(None, None, None)
        os.makedirs("gpurun_out", exist_ok=True)
        tp.export_chrome_trace("gpurun_out/device_trace.json")
    dev_ms = e0.elapsed_time(e1)
    _lib.check(L.dgds_profile_read(srv.handle, C.byref(prof), 1))
    _lib.check(L.dgds_profile_enable(srv.handle, 0))
    st_ = d_stats.cpu().numpy()
    app_tok = sum(steps_in[s][0]["ntok"] for s in range(W, W + K))
    app_alg = sum(steps_in[s][0]["alg"] for s in range(W, W + K))
    q_alg = int(st_[7])
    T = dev_ms / 1e3
    qps = Q * K / T
    peak, peak_kind = peaks()
    q_ach = q_alg / (prof.query_ms / 1e3) / 1e9 if prof.query_ms > 0 else 0.0
    a_ach = app_alg / (prof.append_ms / 1e3) / 1e9 if prof.append_ms > 0 else 0.0
    dom_q = prof.query_ms >= prof.append_ms
    roof_q = {"kernel": "query: k_query K2a + K2b (+K3 fused)", "bound": "hbm", "achieved": q_ach, "peak": peak,
              "unit": "GB/s", "frac": q_ach / peak, "frac_random_ceiling": q_ach / RANDOM_CEILING_GBS,
              "traffic": QUERY_TRAFFIC["value"], "traffic_source": QUERY_TRAFFIC["source"],
              "alg_bytes_per_launch": q_alg / K,
              "avg_launch_ms": prof.query_ms / max(1, prof.query_launches), "peak_kind": peak_kind}
    roof_a = {"kernel": "append: k_stage + k_append (K1) + k_walks (K1b)", "bound": "hbm", "achieved": a_ach,
              "peak": peak, "unit": "GB/s", "frac": a_ach / peak, "frac_random_ceiling": a_ach / RANDOM_CEILING_GBS,
              "traffic": APPEND_TRAFFIC["value"], "traffic_source": APPEND_TRAFFIC["source"],
              "alg_bytes_per_launch": app_alg / K,
              "avg_launch_ms": prof.append_ms / max(1, prof.append_launches), "peak_kind": peak_kind}
    nodes = srv.node_count()
    entries = srv.entry_count()
    slots = srv.index_slots()

    # ---- e2e: same tick through the host C ABI (host buffers, H2D/D2H inside) ----
    e2e = None
    if args.e2e_steps > 0:
        WE = 2  # warm-up steps per mode: both result slots' pinned buffers reach their steady size
        E = args.e2e_steps + WE

        def make_steps(count):
            out = []
            for _ in range(count):
                live = np.nonzero(spos < tr.lengths)[0]
                ns = np.minimum(args.record_tokens, tr.lengths[live] - spos[live])
                offs = np.zeros(len(live) + 1, np.uint64)
                offs[1:] = np.cumsum(ns)
                g0 = tr.offsets[live] + spos[live]
                idx = np.repeat(g0, ns) + (np.arange(int(offs[-1])) - np.repeat(offs[:-1].astype(np.int64), ns))
                toks = np.ascontiguousarray(tr.tokens[idx])
                prev = spos[live].astype(np.uint64)
                spos[live] += ns
                st, qpos = sched.queries(Q)
                base = tr.offsets[st] + qpos
                pat = np.stack([tr.tokens[base - 6 + j] for j in range(6)], 1).astype(np.int32).reshape(-1)
                poff = np.arange(0, 6 * Q + 1, 6, dtype=np.uint64)
                tl = (tr.lengths[st] - qpos).astype(np.int32)
                tru = np.zeros((Q, dl), np.int32)
                for j in range(dl):
                    ok = j < tl
                    tru[ok, j] = tr.tokens[(base + j)[ok]]
                out.append((np.ascontiguousarray(handles_of_stream[live]), np.ascontiguousarray(rid_of_stream[live]),
                            prev, offs, toks.astype(np.int32, copy=False), handles_of_stream[st].copy(), poff, pat,
                            tru, tl))
            return out

        view = _lib.ResultView()
        em_sum = [0]
        last = C.c_uint64()
        ticket = C.c_uint64()

        reply_buf = np.zeros(len(handles_of_stream), srv.REPLY_DTYPE)  # reused by every tick

        def update(hs_):
            (h, r, prev, offs, toks) = hs_[:5]
            _lib.check(L.dgds_update_batch(srv.handle, len(h), h.ctypes.data, r.ctypes.data, prev.ctypes.data,
                                           offs.ctypes.data, toks.ctypes.data, 0.0, reply_buf.ctypes.data))

        def submit(hs_):
            (qh, poff, pat, tru, tl) = hs_[5:]
            _lib.check(L.dgds_speculate_submit(srv.handle, Q, qh.ctypes.data, poff.ctypes.data, pat.ctypes.data,
                                               sp_args.ctypes.data, 0, tru.ctypes.data, dl, tl.ctypes.data,
                                               tl.ctypes.data, C.byref(ticket)))
            return int(ticket.value)

        def consume(t):
            # compact results (CSR) in the server's pinned block; the step reads every emitted count
            _lib.check(L.dgds_speculate_wait(srv.handle, t, C.byref(view)))
            em_sum[0] += int(np.ctypeslib.as_array(C.cast(view.emitted, C.POINTER(C.c_int32)), shape=(Q,)).sum())
            _lib.check(L.dgds_last_transfer(srv.handle, C.byref(last)))
            return int(last.value)

        def h2d_bytes(hs_):
            # bytes actually staged: tokens + segment table (32 B/record) + pieces (16 B/record);
            # patterns (8 int32 rows), pattern lengths, handles, truth rows, truth_left, limit, args
            return hs_[4].nbytes + len(hs_[0]) * (32 + 16) + Q * (4 + 4 + 8 * 4 + dl * 4 + 4 + 4) + 32

        def run(steps, pipelined):
            """serial: update, query, read results, next tick. pipelined: tick s+1's host work
            (update plan + K1 launch, query staging + launch) is issued before tick s's results
            are read, so it overlaps tick s's device work (two result slots)."""
            d2h, pend = 0, None
            for hs_ in steps:
                update(hs_)
                t = submit(hs_)
                if not pipelined:
                    d2h += consume(t)
                    continue
                if pend is not None:
                    d2h += consume(pend)
                pend = t
            if pend is not None:
                d2h += consume(pend)
            return d2h

        res = {}
        tp = None
        for mode in ("serial", "pipelined"):
            steps = make_steps(E)
            run(steps[:WE], mode == "pipelined")
            torch.cuda.synchronize()
            if mode == "pipelined" and os.environ.get("DGDS_E2E_TRACE"):  # debug only (numbers then invalid)
                from torch.profiler import ProfilerActivity, profile
                tp = profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA])
                tp.__enter__()
            gc.collect()
            gc.disable()  # like the device-timed region: no cyclic-GC pause inside the timed ticks
            t0 = time.perf_counter()
            d2h = run(steps[WE:], mode == "pipelined")
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            gc.enable()
            n_e = len(steps) - WE
            res[mode] = {"value": Q * n_e / (t1 - t0), "unit": "queries/s",
                         "h2d_bytes_per_step": sum(h2d_bytes(x) for x in steps[WE:]) // n_e,
                         "d2h_bytes_per_step": d2h // n_e, "steps": n_e,
                         "append_tokens_per_s": sum(x[4].size for x in steps[WE:]) / (t1 - t0)}
        if tp is not None:
            tp.__exit__(None, None, None)
            os.makedirs("gpurun_out", exist_ok=True)
            tp.export_chrome_trace("gpurun_out/e2e_bench_trace.json")
        e2e = dict(res["pipelined"])
        e2e["path"] = ("per tick: dgds_update_batch + dgds_speculate_submit, then dgds_speculate_wait on the "
                       "previous tick's ticket (host buffers in, compact pinned results out; every emitted count "
                       "read); the next tick's host work overlaps this tick's device work")
        e2e["serial"] = res["serial"]
        e2e["serial"]["path"] = "per tick: dgds_update_batch + dgds_speculate_submit + dgds_speculate_wait"

    # ---- CPU baseline (reference, bounded sample, all host cores) ----
    cpu = None
    if not args.no_cpu_baseline:
        try:
            ng = cpu_sample_groups(args, sched)
            qn = max(1, int(Q * ng / sched.G))
            threads = os.cpu_count() or 1
            r = run_reference_cpu(args, sched, ng, args.cpu_steps, qn, threads)
            cpu = {"value": r["queries"] / r["step_s"], "unit": "queries/s", "cores": threads, "kind": "reference",
                   "append_tokens_per_s": r["append_tokens"] / r["step_s"],
                   "query_phase_qps": r["queries"] / r["query_s"],
                   "append_phase_tokens_per_s": r["append_tokens"] / r["append_s"],
                   "sample": f"{ng}/{sched.G} groups, {args.cpu_steps} steps x ({qn} queries + 1 record/stream), "
                             f"thread-per-shard reference GroupDraftIndex; {cpu_model()}"}
        except Exception as e:  # the reported baseline must never break our own line
            cpu = {"value": None, "unit": "queries/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    line = {
        "metric": "draft_queries_per_s", "value": qps, "unit": "queries/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": dev_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "i32+f64", "data": "synthetic",
        "append_tokens_per_s": app_tok / T,
        "query_phase_qps": Q * K / (prof.query_ms / 1e3) if prof.query_ms else None,
        "append_phase_tokens_per_s": app_tok / (prof.append_ms / 1e3) if prof.append_ms else None,
        "config": {"workload": f"{args.config}: {CONFIG_NAMES[args.config]}", "queries_per_step": Q,
                   "append_records_per_step": int(np.mean([len(steps_in[s][0]['h']) for s in range(W, W + K)])),
                   "append_tokens_per_step": app_tok / K, "record_tokens": args.record_tokens, "top_k": kq,
                   "draft_len": dl, "regime": "R1 built index (prefix prefilled) + streaming appends",
                   "prefill": args.prefill, "prefill_s": prefill_s, "index_nodes": nodes,
                   "index_entries": entries, "index_slots": slots, "index_load": entries / slots,
                   "l2": "inputs larger than L2 (index of %.1f GB, 126 MB L2); per-step inputs distinct"
                         % (slots * 32 / 1e9), "parallelism": "single GPU"},
        "roofline": roof_q if dom_q else roof_a,
        "roofline_query": roof_q, "roofline_append": roof_a,
        "cpu_baseline": cpu, "e2e": e2e,
        # our kernels enqueued in the timed region (k_stage + K1 + K1b + K2a + K2b per tick;
        # K2 folds its counters in its last block)
        "gpu_launches": int(kl1 - kl0),
        "wall_ms_per_step": 1e3 * (w1 - w0) / K,
        "clocks": clk.summary(),
    }
    srv.close()
    # ---- extra lines: engine-shaped C5 sweep on C4, C3 with adaptive draft length, C2 full index ----
    if not args.no_lines:
        import bench_lines
        torch.cuda.synchronize()
        gc.collect()
        for key, fn in (("c5_sweep", bench_lines.c5_sweep), ("c3_adaptive", bench_lines.c3_adaptive),
                        ("c2_full", bench_lines.c2_full)):
            try:
                line[key] = fn(dev, local, peak)
            except Exception as e:  # an extra line must never break the headline
                line[key] = {"unavailable": repr(e)}
            gc.collect()
            torch.cuda.empty_cache()
    print(json.dumps(line))


def main():
    args = parse()
    if args.impl == "reference":
        main_reference(args)
    else:
        main_b200(args)


if __name__ == "__main__":
    main()
