"""Multi-GPU step of bench.py (torchrun, one rank per GPU, NCCL).

Weak scaling: for N ranks the config's group set is replicated N times (256*N
C2-shaped groups, same seed, so groups 0..255 are exactly C2), every rank owns
the groups with fnv1a64(group_id) % N == rank (dgds.cpp:10-14) and produces the
traffic of the streams s with s % N == rank: per step one 16-token record per
produced stream plus Q draft queries, exactly the N=1 per-rank work. Records
are routed to their owners with NCCL all-to-all (paper_2511_14617_b200/
routing.py); the owner runs K1 / K2+K3 and the replies return through the
inverse all-to-all. Timing: CUDA events on the step stream, max over ranks.
"""
from __future__ import annotations

import ctypes as C
import gc
import json
import os
import time
from dataclasses import replace

import numpy as np
import torch
import torch.distributed as dist

APP_W = 21  # append record: [local handle, request id, prev lo, prev hi, n, tokens[16]]
QRY_W = 21  # query record: [local handle, pat_len, pattern[8], truth_left, limit, truth[8], pad]


def _gpu_local_cpus(local):
    """CPUs local to visible GPU `local` (NVML affinity), or None."""
    try:
        import pynvml
        pynvml.nvmlInit()
        uuid = str(torch.cuda.get_device_properties(local).uuid)
        h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        words = (os.cpu_count() + 63) // 64
        mask = pynvml.nvmlDeviceGetCpuAffinity(h, words)
        return {64 * w + b for w, m in enumerate(mask) for b in range(64) if (m >> b) & 1}
    except Exception:
        return None


def _pin_rank_cores(world, local):
    """Give each rank its own slice of the host cores (threads created later inherit it), so
    the ranks' host paths do not preempt each other (the tick waits on every rank's host).
    The slice is taken from the cores local to the rank's GPU (NVML affinity; ranks whose GPUs
    share those cores split them), so its pinned staging and host round trips stay on-socket."""
    try:
        cores = sorted(os.sched_getaffinity(0))
        near = [_gpu_local_cpus(g) for g in range(world)]
        if all(n is not None for n in near):
            mine = sorted(set(cores) & near[local])
            peers = [g for g in range(world) if near[g] == near[local]]  # ranks on the same CPU set
            per = len(mine) // len(peers)
            if per >= 2:
                k = peers.index(local)
                os.sched_setaffinity(0, set(mine[k * per:(k + 1) * per]))
                return
        per = len(cores) // world
        if per >= 2:
            os.sched_setaffinity(0, set(cores[local * per:(local + 1) * per]))
    except (AttributeError, OSError):
        pass


def run_multi(args, world, rank, local, dev):
    # The tick loop hands work between the main thread and the planner thread every tick; with
    # the default 5 ms GIL switch interval a hand-off could wait behind the other thread's
    # bytecode (measured: fewer slow runs at 0.1 ms)
    import sys
    sys.setswitchinterval(float(os.environ.get("DGDS_SWITCH_INTERVAL", "0.0001")))
    # measured on a 4-GPU box: pinning each rank to 8 cores cost 10-15% at N=4 (0.347-0.368 vs
    # 0.313-0.317 ms per tick unpinned), so it is opt-in
    if os.environ.get("DGDS_PIN_CORES", "0") == "1":
        _pin_rank_cores(world, local)
        if os.environ.get("DGDS_TICK_TRACE") == "1":
            print(f"rank {local} cores {sorted(os.sched_getaffinity(0))} near {sorted(_gpu_local_cpus(local) or [])[:4]}...",
                  flush=True)
    from bench import CONFIG_NAMES, RANDOM_CEILING_GBS, ClockSampler, append_alg_bytes, peaks
    from paper_2511_14617_b200 import _lib
    from paper_2511_14617_b200.dgds import DgdsParams, DraftServer, SpeculationArgs, args_array, shard_of_group
    from paper_2511_14617_b200.peer import PeerExchange, speculate_routed
    from paper_2511_14617_b200.routing import PaddedRouter, cuda_unpack
    from paper_2511_14617_b200.workload import CONFIGS, generate_workload, group_id

    base = CONFIGS[args.config]
    strong = args.scaling == "strong"
    # weak: the group set is replicated N times (per-GPU work fixed); strong: the config's own
    # group set is sharded over the N GPUs (total work fixed; e.g. C4, the Kimi-K2 shape, which
    # does not fit one GPU)
    cfg = base if strong else replace(base, num_groups=base.num_groups * world)
    tr = generate_workload(cfg)
    G, R = cfg.num_groups, cfg.group_size
    S = G * R
    rt = args.record_tokens
    assert rt <= 16, "records carry at most 16 tokens"
    owner_g = np.array([shard_of_group(group_id(g), world) for g in range(G)], np.int64)
    mine = np.nonzero(owner_g == rank)[0]
    local_h = np.zeros(G, np.int32)
    for o in range(world):
        gs = np.nonzero(owner_g == o)[0]
        local_h[gs] = np.arange(len(gs), dtype=np.int32)
    prefill = (tr.lengths * args.prefill).astype(np.int64) // rt * rt
    my_streams = (mine[:, None] * R + np.arange(R)[None, :]).reshape(-1)
    K, W = args.steps, args.warmup
    Q, kq, dl = args.queries, args.top_k, args.draft_len
    if strong:
        Q = max(1, Q // world)  # the config's query batch, split over the ranks
    E = max(0, args.e2e_steps)
    assert dl <= 8, "query records carry 8 truth tokens"
    idx_tokens = int(prefill[my_streams].sum()) + len(my_streams) * rt * (K + W + E) * world
    srv = DraftServer(DgdsParams(), device=local, expected_nodes=min(idx_tokens * 24, 1_900_000_000),
                      expected_streams=len(my_streams))
    h = srv.group_handles([group_id(int(g)) for g in mine])
    assert (h == np.arange(len(mine))).all()

    # ---- untimed prefill of the owned groups ----
    pos = np.zeros(S, np.int64)
    chunk = 8 * rt
    live_set = my_streams
    while True:
        live = live_set[pos[live_set] < prefill[live_set]]
        if len(live) == 0:
            break
        n_rec = np.minimum((prefill[live] - pos[live] + rt - 1) // rt, 8)
        rs = np.repeat(live, n_rec)
        k_in = np.arange(len(rs)) - np.repeat(np.cumsum(n_rec) - n_rec, n_rec)
        starts = pos[rs] + k_in * rt
        ns = np.minimum(rt, prefill[rs] - starts)
        offs = np.zeros(len(ns) + 1, np.uint64)
        offs[1:] = np.cumsum(ns)
        g0 = tr.offsets[rs] + starts
        idx = np.repeat(g0, ns) + (np.arange(int(offs[-1])) - np.repeat(offs[:-1].astype(np.int64), ns))
        rep = srv.update_arrays(local_h[rs // R], (rs % R).astype(np.int32), starts.astype(np.uint64), offs,
                                tr.tokens[idx], 0.0)
        assert rep["ok"].all()
        pos[live] += np.minimum(prefill[live] - pos[live], chunk)
    pos = prefill.copy()  # every rank knows every stream's prefix length

    # owner-side algorithmic append bytes of every tick (the records of the owned streams,
    # whoever produces them), computed here so no bookkeeping runs inside the timed region
    own_alg = []
    pos_own = prefill.copy()
    for s in range(W + K + E):
        live_o = my_streams[pos_own[my_streams] < tr.lengths[my_streams]]
        ns_o = np.minimum(rt, tr.lengths[live_o] - pos_own[live_o])
        own_alg.append(append_alg_bytes(pos_own[live_o], ns_o))
        pos_own[live_o] += ns_o

    # ---- per-step inputs of this rank (the streams it produces), resident in HBM ----
    produced = np.arange(rank, S, world)
    rng = np.random.default_rng(args.seed + 7919 * rank)
    steps_in = []
    for s in range(W + K + E):
        live = produced[pos[produced] < tr.lengths[produced]]
        ns = np.minimum(rt, tr.lengths[live] - pos[live])
        rec = np.zeros((len(live), APP_W), np.int32)
        rec[:, 0] = local_h[live // R]
        rec[:, 1] = live % R
        rec[:, 2] = (pos[live] & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
        rec[:, 3] = (pos[live] >> 32).astype(np.int32)
        rec[:, 4] = ns
        for j in range(16):
            ok = j < ns
            rec[ok, 5 + j] = tr.tokens[tr.offsets[live[ok]] + pos[live[ok]] + j]
        alg = append_alg_bytes(pos[live], ns)
        pos[live] += ns
        pool = produced[prefill[produced] >= 7]
        st = pool[rng.integers(0, len(pool), Q)]
        qp = np.minimum(6 + (rng.random(Q) * (prefill[st] - 6 + 1)).astype(np.int64), prefill[st])
        qr = np.zeros((Q, QRY_W), np.int32)
        qr[:, 0] = local_h[st // R]
        qr[:, 1] = 6
        b0 = tr.offsets[st] + qp
        for j in range(6):
            qr[:, 2 + j] = tr.tokens[b0 - 6 + j]
        tl = (tr.lengths[st] - qp).astype(np.int32)
        qr[:, 10] = tl
        qr[:, 11] = tl
        for j in range(dl):
            ok = j < tl
            qr[ok, 12 + j] = tr.tokens[(b0 + j)[ok]]
        steps_in.append(dict(app=torch.from_numpy(rec).to(dev), app_owner=torch.from_numpy(owner_g[live // R]).to(
            device=dev, dtype=torch.int32), q=torch.from_numpy(qr).to(dev),
            q_owner=torch.from_numpy(owner_g[st // R]).to(device=dev, dtype=torch.int32), alg=alg,
            ntok=int(ns.sum())))

    router = PaddedRouter(world)
    capq = int(1.5 * Q / world) + 512
    capa = int(1.5 * len(produced) / world) + 64
    sp_args = torch.from_numpy(args_array([SpeculationArgs(dl, 6, 1, kq, 0.25, 1)]).view(np.uint8).copy()).to(dev)
    L = _lib.lib()
    d_stats = torch.zeros(8, dtype=torch.int64, device=dev)
    app_alg_owner = [0]
    overflow = torch.zeros((), dtype=torch.bool, device=dev)
    side = torch.cuda.Stream(dev)
    side_q = torch.cuda.Stream(dev)  # early query sends (px)
    q_sent = set()
    ev_side = torch.cuda.Event()  # spin-waited: blocking events cost 1-3 ms of wakeup per tick here
    meta_h = torch.empty((world * capa, 5), dtype=torch.int32).pin_memory()
    mq = world * capq
    # reply record: n_cands | lens[k] | pad | scores[k] f64 | supports[k] i64 | tokens[k][dl] | verify[3] | pad
    off_sc = 2 + kq - (kq % 2)
    off_sp = off_sc + 2 * kq
    off_tk = off_sp + 2 * kq
    off_v = off_tk + kq * dl
    rep_w = (off_v + 3 + 1) // 2 * 2
    layout = _lib.RecordLayout(QRY_W, 0, 1, 2, 10, 11, 12, rep_w, 0, 1, off_sc, off_sp, off_tk, off_v)
    replies = torch.zeros((mq, rep_w), dtype=torch.int32, device=dev)
    prof_host = {}
    dbg = os.environ.get("DGDS_MULTI_BREAKDOWN") == "1"  # device-synchronised phases (debug)
    host_t = os.environ.get("DGDS_MULTI_HOSTTIME") == "1"  # host time per phase, no syncs (debug)

    def mark(name, t0):
        if not (dbg or host_t):
            return t0
        if dbg:
            torch.cuda.synchronize()
        t1 = time.perf_counter()
        prof_host[name] = prof_host.get(name, 0.0) + t1 - t0
        if name == "route_cur":
            prof_host.setdefault("route_cur_each_us", []).append(round(1e6 * (t1 - t0)))
        return t1

    # Append records of a tick are routed one tick AHEAD (side stream, double-buffered):
    # the owner's O(records) host bookkeeping then overlaps the previous tick's GPU work.
    meta_bufs = [meta_h, torch.empty_like(meta_h).pin_memory()]
    cnt_bufs = [torch.zeros(world, dtype=torch.int32).pin_memory() for _ in range(2)]
    ev_bufs = [ev_side, torch.cuda.Event()]
    ev_rep = [torch.cuda.Event(), torch.cuda.Event()]
    inflight = {}
    use_px = args.route == "px"
    if use_px:
        # NVLink peer-memory exchange: q rows -> owners, replies -> senders, append rows -> owners
        # replies land in a shared slab in query order: the query record's pad word carries its index
        px = PeerExchange(world, rank, local, {"q": (capq, QRY_W), "rep": (Q, rep_w, "shared"),
                                               "a": (capa, APP_W)})
        rep_view = {p: px.slab("rep", p) for p in (1, 2)}  # parity 1, 0

    def route_appends(s):
        if s >= len(steps_in) or s in inflight:
            return
        inp = steps_in[s]
        k = s % 2
        if "ready" in inp:  # e2e: the inputs were copied in on the main stream
            side.wait_event(inp["ready"])
        if use_px:
            seq = s + 1
            with torch.cuda.stream(side):
                # this parity was last read by the owners' K1 of tick s-2; their replies of tick s-1
                # (queued after that K1 on their streams) prove it is free
                if s > 0:
                    side.wait_event(ev_rep[(s - 1) % 2])
                px.send("a", inp["app_owner"], inp["app"], seq, stable=True, want_slot=False, stream=side)
                px.wait("a", seq, stream=side)
                # metadata columns of every row (one 2-D DMA) and the per-sender counts
                _lib.check(L.dgds_copy_rows_d2h(C.c_void_p(meta_bufs[k].data_ptr()), 20,
                                                C.c_void_p(px.slab_ptr("a", seq)), APP_W * 4, 20, world * capa,
                                                C.c_void_p(side.cuda_stream)))
                _lib.check(L.dgds_copy_rows_d2h(C.c_void_p(cnt_bufs[k].data_ptr()), 4 * world,
                                                C.c_void_p(px.counts_ptr("a", seq)), 4 * world, 4 * world, 1,
                                                C.c_void_p(side.cuda_stream)))
                ev_bufs[k].record(side)
            inflight[s] = (None, None, k)
            return
        # step inputs are resident before the timed region, so the side stream needs no
        # dependency on the main stream: the next tick's exchange can run under this tick's kernels
        with torch.cuda.stream(side):
            ra, st_a = router.forward(inp["app_owner"], inp["app"], capa)
            meta_bufs[k].copy_(ra[:, :5], non_blocking=True)
            ev_bufs[k].record(side)
        ra.record_stream(torch.cuda.current_stream(dev))  # K1 reads the tokens on the main stream
        inflight[s] = (ra, st_a[1], k)

    def send_queries(s):
        """Queries of tick s go to their owners as soon as the replies of tick s-1 are home
        (the point where an engine knows its next patterns), overlapping the owners' K1 of
        tick s-1. The owner's slab parity of tick s was last read by its K2 of tick s-2."""
        if not use_px or s >= len(steps_in) or s in q_sent:
            return
        inp = steps_in[s]
        with torch.cuda.stream(side_q):
            if "ready" in inp:
                side_q.wait_event(inp["ready"])
            if s > 0:
                side_q.wait_event(ev_rep[(s - 1) % 2])
            px.send("q", inp["q_owner"], inp["q"], s + 1, origin_word=QRY_W - 1, want_slot=False, stream=side_q)
        q_sent.add(s)

    plans = {}  # tick -> plan, or a future of one (planned on a helper thread)
    planner = None
    if use_px:
        from concurrent.futures import ThreadPoolExecutor
        planner = ThreadPoolExecutor(max_workers=1)  # ctypes and event waits release the GIL
    run_until = [0]  # ticks < run_until[0] run in the current loop (their queries may be issued ahead)
    # ticks < plan_until[0] may be planned ahead (host bookkeeping of their routed appends): the
    # warm-up plans the first timed tick, so the timed region starts with a full pipeline, as
    # every later tick does; a tick that will not run is never planned
    plan_until = [0]

    native_planner = use_px and os.environ.get("DGDS_NATIVE_PLANNER", "1") == "1"

    def submit_plan(s, k):
        """Tick s's routed plan, made off the main thread: the server's C++ planner thread
        (waits for the metadata event, no GIL), or the Python helper thread."""
        if native_planner:
            job = C.c_uint64()
            _lib.check(L.dgds_update_plan_routed_async(
                srv.handle, C.c_void_p(ev_bufs[k].cuda_event), world, capa, C.c_void_p(cnt_bufs[k].data_ptr()),
                C.c_void_p(meta_bufs[k].data_ptr()), 5, C.c_void_p(px.slab_ptr("a", s + 1)), APP_W, 0.0,
                C.byref(job)))
            return job.value
        return planner.submit(make_plan, s, k)

    def take_plan(h):
        if not native_planner:
            return h.result()
        nrej = C.c_int64()
        plan = C.c_void_p()
        _lib.check(L.dgds_update_plan_take(srv.handle, h, C.byref(nrej), C.byref(plan)))
        if nrej.value:
            raise RuntimeError("routed append out of order")
        return plan

    def make_plan(s, k):
        """Host half of tick s's appends (dgds_update_plan_routed): waits for the tick's routed
        metadata, does the bookkeeping, returns the plan to launch after tick s's queries."""
        ev_bufs[k].synchronize()
        nrej = C.c_int64()
        plan = C.c_void_p()
        _lib.check(L.dgds_update_plan_routed(srv.handle, world, capa, C.c_void_p(cnt_bufs[k].data_ptr()),
                                             C.c_void_p(meta_bufs[k].data_ptr()), 5,
                                             C.c_void_p(px.slab_ptr("a", s + 1)), APP_W, 0.0, C.byref(nrej),
                                             C.byref(plan)))
        if nrej.value:
            raise RuntimeError("routed append out of order")
        return plan

    def q_part(s, stats):
        """Tick s, first half (engine.cpp:88-143): draft queries (+ fused verify) on the current index."""
        nonlocal overflow
        inp = steps_in[s]
        main = torch.cuda.current_stream(dev)
        t0 = mark("start", time.perf_counter())
        route_appends(s)  # normally already in flight since the previous tick
        t0 = mark("route_cur", t0)
        seq, k = s + 1, s % 2
        if use_px:
            # (1)+(2) queries stored into the owners' slabs; the owner's K2+K3 stores each reply
            # straight into its sender's reply slab; (3) gather into query order
            send_queries(s)  # normally already sent during the previous tick
            t0 = mark("q_fwd", t0)
            speculate_routed(srv, px, "q", "rep", seq, layout, sp_args, kq, dl, d_stats if stats else None, main,
                             origin_field=QRY_W - 1)
            t0 = mark("q_kernel", t0)
            px.wait("rep", seq, stream=main)
            back = rep_view[2 - seq % 2]  # [Q, rep_w] in query order, no gather
            ev_rep[k].record(main)
            t0 = mark("q_rev", t0)
        else:
            if "ready" in inp:  # e2e: inputs copied in on the copy stream
                main.wait_event(inp["ready"])
            # (1) queries -> owners (static splits, no host sync)
            rq, st_q = router.forward(inp["q_owner"], inp["q"], capq)
            t0 = mark("q_fwd", t0)
            # (2) owner: K2 + fused K3 straight from the received query records into reply records
            _lib.check(L.dgds_speculate_records(srv.handle, mq, C.c_void_p(rq.data_ptr()), C.byref(layout),
                                                C.c_void_p(sp_args.data_ptr()), 0, kq, dl,
                                                C.c_void_p(replies.data_ptr()),
                                                C.c_void_p(d_stats.data_ptr()) if stats else None,
                                                C.c_void_p(main.cuda_stream)))
            t0 = mark("q_kernel", t0)
            back, ovq = router.reverse(replies, st_q)
            overflow = overflow | ovq
            t0 = mark("q_rev", t0)
        return back

    def a_part(s, stats, pipeline=False):
        """Tick s, second half (engine.cpp:144-161): the appends of the tick's emitted tokens,
        planned on the host during the previous tick (px), launched after the tick's queries.
        With pipeline, tick s+1's queries are enqueued before tick s+1 is planned, so the GPU
        has work queued while the host plans. Returns tick s+1's reply view when enqueued."""
        nonlocal overflow
        main = torch.cuda.current_stream(dev)
        t0 = time.perf_counter()
        ra, ova, k = inflight.pop(s)
        if use_px:
            # tick s+1's exchanges first: they need only tick s's replies (ev_rep), and their kernels
            # get SMs before K1 fills them; the helper thread plans tick s+1 as its metadata lands
            if s not in plans:  # the planner is FIFO: tick s must be planned before tick s+1
                plans[s] = submit_plan(s, k)
            route_appends(s + 1)
            if s + 1 < plan_until[0] and (s + 1) in inflight and (s + 1) not in plans:
                plans[s + 1] = submit_plan(s + 1, inflight[s + 1][2])
            send_queries(s + 1)
            t0 = mark("route_next", t0)
            plan = take_plan(plans.pop(s))
            t0 = mark("meta_np", t0)
            main.wait_event(ev_bufs[k])  # K1 reads the slab rows delivered on the side stream
            _lib.check(L.dgds_update_launch(srv.handle, plan, C.c_void_p(main.cuda_stream)))
            if stats:
                app_alg_owner[0] += own_alg[s]
            t0 = mark("append_call", t0)
            nxt = None
            if pipeline and s + 1 < run_until[0]:
                nxt = q_part(s + 1, stats)
            mark("send_next", t0)
            return nxt
        ev_bufs[k].synchronize()
        t0 = mark("meta_wait", t0)
        meta = meta_bufs[k].numpy()
        rows = np.nonzero(meta[:, 0] >= 0)[0]
        if len(rows):
            m = meta[rows]
            n = m[:, 4].astype(np.uint64)
            prev = m[:, 2].view(np.uint32).astype(np.uint64) | (m[:, 3].astype(np.uint64) << np.uint64(32))
            starts = rows.astype(np.uint64) * np.uint64(APP_W) + np.uint64(5)
            main.wait_event(ev_bufs[k])
            rep = srv.update_device_strided(m[:, 0].copy(), m[:, 1].copy(), prev, starts, n, ra.data_ptr(), 0.0,
                                            main.cuda_stream)
            if not rep["ok"].all():
                raise RuntimeError("routed append out of order")
        if stats:
            app_alg_owner[0] += own_alg[s]
        overflow = overflow | ova
        t0 = mark("append_call", t0)
        route_appends(s + 1)  # the next tick's appends (NCCL route), one tick ahead
        mark("route_next", t0)
        return None

    tick_ev = [] if os.environ.get("DGDS_TICK_TRACE") == "1" else None  # debug: per-tick device times

    # The px tick loop runs in C++ (dgds_px_driver_*, csrc/px_driver.cpp) unless
    # DGDS_PX_DRIVER=python: same pipeline, no interpreter on the per-tick critical path.
    native_driver = use_px and os.environ.get("DGDS_PX_DRIVER", "native") == "native"
    drv = None
    if native_driver:
        from paper_2511_14617_b200.peer import TickDriver
        n_drv = W + K  # the device-resident ticks; the e2e loop below runs in Python after a sync
        drv = TickDriver(srv, px, layout, sp_args, kq, dl,
                         [(steps_in[i]["q_owner"], steps_in[i]["q"], steps_in[i]["app_owner"], steps_in[i]["app"])
                          for i in range(n_drv)], QRY_W - 1, stream=torch.cuda.current_stream(dev))

    def run_ticks(a, b, stats, plan_to=None):
        """Ticks [a, b) back to back, pipelined (px) or in order (nccl); ticks < plan_to (default b)
        may be planned ahead."""
        if native_driver:
            drv.run(a, b, plan_to or 0, d_stats if stats else None)
            return None
        run_until[0] = b
        plan_until[0] = b if plan_to is None else plan_to
        back = q_part(a, stats)
        for s in range(a, b):
            if tick_ev is not None and stats:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(torch.cuda.current_stream(dev))
                tick_ev.append(ev)
            nxt = a_part(s, stats, pipeline=use_px)
            if not use_px and s + 1 < b:
                nxt = q_part(s + 1, stats)
            back = nxt if nxt is not None else back
        return back

    run_ticks(0, W, False, plan_to=W + 1)  # the first timed tick is planned during the warm-up
    torch.cuda.synchronize()
    prof = _lib.Profile()
    _lib.check(L.dgds_profile_enable(srv.handle, 1))
    _lib.check(L.dgds_profile_read(srv.handle, C.byref(prof), 1))
    d_stats.zero_()
    px_l0 = px.status()[1] if use_px else 0
    gc.collect()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tp = None
    if os.environ.get("DGDS_TORCH_PROFILE"):  # debug only: a timeline of the timed steps (numbers then invalid)
        from torch.profiler import ProfilerActivity, profile
        tp = profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA])
        tp.__enter__()
    with ClockSampler(local) as clk:
        kl0 = L.dgds_kernel_launches()
        e0.record()
        run_ticks(W, W + K, True)
        e1.record()
        kl1 = L.dgds_kernel_launches()
        torch.cuda.synchronize()
    if tp is not None:
        tp.__exit__(None, None, None)
        os.makedirs("gpurun_out", exist_ok=True)
        tp.export_chrome_trace(f"gpurun_out/trace_r{rank}.json")
        if rank == 0:
            print(tp.key_averages().table(sort_by="cuda_time_total", row_limit=22), flush=True)
            print(tp.key_averages().table(sort_by="cpu_time_total", row_limit=22), flush=True)
    if tick_ev:
        print(f"rank {rank} tick us:", [round(1e3 * tick_ev[i].elapsed_time(tick_ev[i + 1]))
                                        for i in range(len(tick_ev) - 1)], flush=True)
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    T = ms.item() / 1e3
    _lib.check(L.dgds_profile_read(srv.handle, C.byref(prof), 1))
    # our launches in the timed region: K1 + K2/K3 (server profile), plus the routing kernels —
    # px send/wait/signal (counted by the exchange)
    route_launches = (px.status()[1] - px_l0) if use_px else 0
    tot = torch.tensor([sum(steps_in[s]["ntok"] for s in range(W, W + K)), int(d_stats[7].item()),
                        app_alg_owner[0], prof.query_ms * 1e3, prof.append_ms * 1e3,
                        (kl1 - kl0) + route_launches], dtype=torch.float64,
                       device=dev)
    dist.all_reduce(tot)
    ntok_all, q_alg_all, a_alg_all, qus_all, aus_all, launches_all = tot.tolist()

    # ---- e2e: the same routed step with pinned host inputs copied in and replies read back ----
    e2e = None
    if E > 0:
        host_in = [{k: (v.cpu().pin_memory() if torch.is_tensor(v) else v) for k, v in steps_in[s].items()}
                   for s in range(W + K, W + K + E)]
        h2d = sum(x["app"].nbytes + x["app_owner"].nbytes + x["q"].nbytes + x["q_owner"].nbytes for x in host_in)
        cp = torch.cuda.Stream(dev)  # input H2D beside the kernels
        main = torch.cuda.current_stream(dev)
        keys = ("app", "app_owner", "q", "q_owner")
        # device input sets and pinned reply buffers, double-buffered and allocated up front (an
        # allocation inside the loop is a device-synchronising cudaMalloc / cudaHostAlloc)
        d_sets = [{k: torch.empty((max(x[k].shape[0] for x in host_in),) + tuple(host_in[0][k].shape[1:]),
                                  dtype=host_in[0][k].dtype, device=dev) for k in keys} for _ in range(2)]
        ev_in_free = [torch.cuda.Event(), torch.cuda.Event()]
        emitted = [0]
        tickets = {}
        view = _lib.ResultView()
        last = C.c_uint64()

        def issue_inputs(j):
            buf = d_sets[j % 2]
            with torch.cuda.stream(cp):
                if j >= 2:  # set j%2 was read by tick j-2's exchanges, all done before its K1 was queued
                    cp.wait_event(ev_in_free[j % 2])
                d_in = {}
                for k in keys:
                    v = buf[k][:host_in[j][k].shape[0]]
                    v.copy_(host_in[j][k], non_blocking=True)
                    d_in[k] = v
                d_in["ready"] = torch.cuda.Event()
                d_in["ready"].record(cp)
            steps_in.append(d_in)

        def d2h_replies(j, back):
            # the tick's reply records, compacted on the main stream right after its reply wait (the
            # owners' replies of tick j+2 reuse this slab parity only after that stream passes tick
            # j+1's reply wait), then copied out over PCIe into the server's next result slot
            tk = C.c_uint64()
            _lib.check(L.dgds_replies_submit(srv.handle, back.shape[0], C.c_void_p(back.data_ptr()),
                                             C.byref(layout), kq, dl, C.c_void_p(main.cuda_stream), C.byref(tk)))
            tickets[j] = int(tk.value)

        def consume(j):
            _lib.check(L.dgds_speculate_wait(srv.handle, tickets.pop(j), C.byref(view)))
            emitted[0] += int(np.ctypeslib.as_array(C.cast(view.emitted, C.POINTER(C.c_int32)), shape=(Q,)).sum())
            _lib.check(L.dgds_last_transfer(srv.handle, C.byref(last)))
            return int(last.value)

        warm = torch.zeros((Q, rep_w), dtype=torch.int32, device=dev)  # both result slots reach their size
        for j in range(2):
            d2h_replies(-1 - j, warm)
            consume(-1 - j)
        emitted[0] = 0
        gc.collect()
        dist.barrier()
        torch.cuda.synchronize()
        gc.disable()  # no cyclic-GC pause inside the timed ticks
        t0 = time.perf_counter()
        d2h = 0
        base_s = len(steps_in)
        run_until[0] = base_s + E
        plan_until[0] = base_s + E
        # pipelined like the single-GPU e2e loop: tick j+1's inputs, exchanges and queries are
        # queued before tick j's replies are read on the host
        issue_inputs(0)
        d2h_replies(0, q_part(base_s, False))
        e2e_trace = [] if os.environ.get("DGDS_MULTI_E2E_TRACE") == "1" else None  # host µs per phase (debug)
        for j in range(E):
            ta = time.perf_counter()
            if j + 1 < E:
                issue_inputs(j + 1)
            tb = time.perf_counter()
            nxt = a_part(base_s + j, False, pipeline=use_px)
            ev_in_free[j % 2].record(main)  # after tick j's K1 was queued behind its exchanges
            if not use_px and j + 1 < E:
                nxt = q_part(base_s + j + 1, False)
            tc = time.perf_counter()
            if nxt is not None:
                d2h_replies(j + 1, nxt)
            td = time.perf_counter()
            d2h += consume(j)
            if e2e_trace is not None:
                e2e_trace.append([round(1e6 * x) for x in (tb - ta, tc - tb, td - tc, time.perf_counter() - td)])
        if e2e_trace is not None:
            print(f"rank {rank} e2e inputs|a_part|d2h|consume us:", e2e_trace, flush=True)
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device=dev)
        gc.enable()
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": world * Q * E / dt.item(), "unit": "queries/s", "h2d_bytes_per_step": h2d // E,
               "d2h_bytes_per_step": d2h // E, "steps": E,
               "path": ("routed ticks, pinned host records in (copy stream); each tick's reply records compacted "
                        "into a CSR result view in pinned memory (dgds_replies_submit / dgds_speculate_wait), every "
                        "emitted count read; tick j+1 is queued before tick j's replies are read")}

    if dbg or host_t:
        print(f"rank {rank} breakdown (s, all steps):",
              dict({k: (round(v, 4) if isinstance(v, float) else v) for k, v in prof_host.items()
                    if k != "route_cur_each_us"}, rank=rank, cores=sorted(os.sched_getaffinity(0))), flush=True)
    if use_px:
        timed_out, _ = px.status()
        if timed_out:
            raise RuntimeError("peer exchange wait timed out: results of this run are invalid")
        overflow = px.overflow.bool()
    if bool(overflow.item()):
        raise RuntimeError("routing capacity overflow: results of this run are invalid")
    if rank == 0:
        peak, peak_kind = peaks()
        # sums over ranks of bytes and of launch time: their ratio is the per-GPU rate
        q_ach = q_alg_all / (qus_all / 1e6) / 1e9 if qus_all else 0.0
        a_ach = a_alg_all / (aus_all / 1e6) / 1e9 if aus_all else 0.0
        dom_q = qus_all >= aus_all
        roof = lambda kern, ach, alg, us, n: {  # noqa: E731
            "kernel": kern, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "frac_random_ceiling": ach / RANDOM_CEILING_GBS, "traffic": None, "alg_bytes_per_launch": alg / max(1, n),
            "avg_launch_ms": us / 1e3 / max(1, n), "peak_kind": peak_kind, "per_gpu": True}
        line = {
            "metric": "draft_queries_per_s", "value": world * Q * K / T, "unit": "queries/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": 1e3 * T / K, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "i32+f64", "data": "synthetic",
            "append_tokens_per_s": ntok_all / T,
            "config": {"workload": f"{args.config}: {CONFIG_NAMES[args.config]} " + (
                           f"(group set sharded over {world} GPUs)" if strong else f"(group set replicated x{world})"),
                       "queries_per_step": world * Q, "queries_per_rank": Q, "record_tokens": rt, "top_k": kq,
                       "draft_len": dl, "prefill": args.prefill, "groups": G,
                       "routing": ("fnv1a64(gid) % N owner; NVLink peer-memory exchange: k_px_send stores rows "
                                   "into the owner's slab, K2+K3 stores replies into the sender's slab (no collectives)"
                                   if use_px else
                                   "fnv1a64(gid) % N owner; NCCL all_to_all_single (counts, payload, replies)"),
                       "tick_loop": ("C++ dgds_px_driver (csrc/px_driver.cpp)" if native_driver else
                                     "Python (bench_multi.py)"),
                       "l2": ("inputs larger than L2 (per-GPU index = 1/N of the config's index)" if strong else
                              "inputs larger than L2 (per-GPU index ~ the N=1 index)"),
                       "parallelism": f"group-sharded dp{world}"},
            "roofline": roof("k_query (K2+K3)", q_ach, q_alg_all, qus_all, K * world) if dom_q else roof(
                "k_append (K1)", a_ach, a_alg_all, aus_all, K * world),
            "roofline_query": roof("k_query (K2+K3)", q_ach, q_alg_all, qus_all, K * world),
            "roofline_append": roof("k_append (K1)", a_ach, a_alg_all, aus_all, K * world),
            "cpu_baseline": None, "e2e": e2e, "gpu_launches": int(launches_all), "clocks": clk.summary(),
        }
        print(json.dumps(line))
    dist.barrier()
    torch.cuda.synchronize()
    if planner is not None:
        planner.shutdown(wait=True)
    if drv is not None:
        drv.close()
    if use_px:
        px.close()  # every rank is past its last exchange (barrier above)
    srv.close()
    dist.barrier()
    dist.destroy_process_group()
