import torch, time
for mb in (0.25, 1, 5, 20, 64):
    n = int(mb * (1 << 20))
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20
    e0.record()
    for _ in range(20): h.copy_(d, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    t2 = e0.elapsed_time(e1) / 20
    hp = torch.empty(n, dtype=torch.uint8); hp.fill_(1)
    torch.cuda.synchronize(); w0 = time.perf_counter()
    for _ in range(5): d.copy_(hp)
    torch.cuda.synchronize(); t3 = (time.perf_counter() - w0) / 5
    print(f"{mb:6} MB  H2D pinned {n/t/1e6:7.1f} GB/s  D2H pinned {n/t2/1e6:7.1f} GB/s  H2D pageable {n/t3/1e9:6.1f} GB/s")
