"""Time the peer-exchange send kernels in one process (two local ranks on cuda:0).
Usage: python tools/px_bench.py [n_records] [words] [iters]"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14617_b200.peer import PeerExchange

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
W = int(sys.argv[2]) if len(sys.argv) > 2 else 21
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 50
dev = torch.device("cuda:0")
cap = int(1.5 * n / 2) + 512
pxs = PeerExchange.local_group(2, 0, {"q": (cap, W)})
rec = torch.randint(0, 1 << 20, (n, W), dtype=torch.int32, device=dev)
own = torch.randint(0, 2, (n,), dtype=torch.int32, device=dev)
seq = 0
for _ in range(5):
    seq += 1
    for r in range(2):
        pxs[r].send("q", own, rec, seq, want_slot=False)
    for r in range(2):
        pxs[r].wait("q", seq)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    seq += 1
    pxs[0].send("q", own, rec, seq, want_slot=False)
    pxs[1].send("q", own, rec, seq, want_slot=False)
    pxs[0].wait("q", seq)
    pxs[1].wait("q", seq)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters / 2
print(f"n={n} words={W}: {1e3 * ms:.1f} us per send+wait ({n * W * 4 / ms / 1e6:.1f} GB/s of rows)")
