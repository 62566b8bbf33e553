"""Summarise a torch-profiler chrome trace of bench_multi's timed ticks: per-stream GPU events
of the last few ticks (start offset, duration), to locate gaps between K2, K1 and the exchange
kernels. Usage: python tools/trace_ticks.py gpurun_out/trace_r0.json [n_events]"""
import json
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
ev = json.load(open(path))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
gpu.sort(key=lambda e: e["ts"])
gpu = gpu[-n:]
t0 = gpu[0]["ts"]
for e in gpu:
    print(f"{e['ts'] - t0:9.1f} {e['dur']:7.1f} s{e.get('tid')} {e['name'][:70]}")
