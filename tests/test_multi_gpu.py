"""Multi-GPU parity (N-GPU outputs identical to the CPU oracle).

Two processes, one GPU each, connected by the NVLink peer exchange (dgds_px_*):
every rank produces the 16-token records of its streams and the draft queries of
its requests for groups of BOTH owners (fnv1a64(gid) % 2, dgds.cpp:10-14).
Records reach their owner with a stable send, the owner applies them
(dgds_update_batch_routed). Queries reach their owner stamped with their index,
and the owner's K2+K3 stores each reply straight into the sender's reply slab.
Every reply must equal the CPU restatement oracle fed the same appends.
Skipped on fewer than two GPUs.
"""
from __future__ import annotations

import ctypes as C
import os
import socket
import traceback
from dataclasses import replace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

APP_W, QRY_W, RW = 21, 21, 58
KQ, DL = 4, 8


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _decode(row):
    nc = int(row[0])
    out = []
    for c in range(nc):
        L = int(row[1 + c])
        sc = row[6 + 2 * c:8 + 2 * c].copy().view(np.float64)[0]
        sp = row[14 + 2 * c:16 + 2 * c].copy().view(np.int64)[0]
        out.append((tuple(int(x) for x in row[22 + c * DL:22 + c * DL + L]), np.float64(sc).view(np.uint64).item(),
                    int(sp)))
    return out


def _worker(rank, world, port, errfile):
    try:
        _run(rank, world, port)
    except Exception:
        with open(errfile + f".{rank}", "w") as f:
            f.write(traceback.format_exc())
        raise


def _run(rank, world, port):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    from oracle import oracle as O
    from paper_2511_14617_b200 import _lib
    from paper_2511_14617_b200 import dgds as D
    from paper_2511_14617_b200.peer import PeerExchange, speculate_routed
    from paper_2511_14617_b200.workload import CONFIGS, generate_workload, group_id

    cfg = replace(CONFIGS["C1"], num_groups=8, group_size=4, location=400.0, max_tokens=400, vocab_size=40)
    tr = generate_workload(cfg)
    G, R = cfg.num_groups, cfg.group_size
    S = G * R
    owner_g = np.array([D.shard_of_group(group_id(g), world) for g in range(G)], np.int32)
    assert len(set(owner_g.tolist())) == world, "both ranks must own groups"
    local_h = np.zeros(G, np.int32)
    for o in range(world):
        gs = np.nonzero(owner_g == o)[0]
        local_h[gs] = np.arange(len(gs), dtype=np.int32)
    srv = D.DraftServer(D.DgdsParams(), device=rank, expected_nodes=1 << 20, expected_streams=S)
    mine = np.nonzero(owner_g == rank)[0]
    assert (srv.group_handles([group_id(int(g)) for g in mine]) == np.arange(len(mine))).all()

    Q = 1500
    capa, capq = S, Q
    px = PeerExchange(world, rank, rank, {"a": (capa, APP_W), "q": (capq, QRY_W), "rep": (Q, RW, "shared")})
    px.set_timeout(20.0)
    L = _lib.lib()
    pos = np.zeros(S, np.int64)
    produced = np.arange(rank, S, world)
    oracle_lib = O.restatement()
    oidx = {g: oracle_lib.index(group_id=group_id(g)) for g in range(G)}
    meta = torch.zeros((world * capa, 5), dtype=torch.int32).pin_memory()
    cnt = torch.zeros(world, dtype=torch.int32).pin_memory()
    seq = 0
    while (pos < tr.lengths).any():
        seq += 1
        live = produced[pos[produced] < tr.lengths[produced]]
        rec = np.zeros((max(1, len(live)), APP_W), np.int32)
        own = np.full(len(rec), -1, np.int32)
        for i, s in enumerate(live):
            n = int(min(16, tr.lengths[s] - pos[s]))
            rec[i, :5] = [local_h[s // R], s % R, pos[s] & 0xFFFFFFFF, pos[s] >> 32, n]
            rec[i, 5:5 + n] = tr.stream(s)[pos[s]:pos[s] + n]
            own[i] = owner_g[s // R]
        px.send("a", torch.from_numpy(own).to(dev), torch.from_numpy(rec).to(dev), seq, stable=True,
                want_slot=False)
        px.wait("a", seq)
        meta.copy_(px.slab("a", seq)[:, :5])
        cnt.copy_(px.counts("a", seq))
        torch.cuda.synchronize()
        nrej = C.c_int64()
        _lib.check(L.dgds_update_batch_routed(srv.handle, world, capa, C.c_void_p(cnt.data_ptr()),
                                              C.c_void_p(meta.data_ptr()), 5, C.c_void_p(px.slab_ptr("a", seq)),
                                              APP_W, 0.0, C.byref(nrej), None))
        assert nrej.value == 0
        # every rank advances every stream (all know the schedule) and feeds the oracle
        for s in range(S):
            if pos[s] < tr.lengths[s]:
                n = int(min(16, tr.lengths[s] - pos[s]))
                assert oidx[s // R].append(s % R, int(pos[s]), tr.stream(s)[pos[s]:pos[s] + n])[0]
                pos[s] += n
        torch.cuda.synchronize()
        dist.barrier()

    # draft queries for streams of every group, routed to their owners
    rng = np.random.default_rng(100 + rank)
    st = rng.integers(0, S, Q)
    qp = np.array([rng.integers(1, tr.lengths[s]) for s in st])
    plen = rng.integers(0, 9, Q)
    qr = np.zeros((Q, QRY_W), np.int32)
    pats = []
    for i, (s, p, L_) in enumerate(zip(st, qp, plen)):
        pat = tr.stream(s)[max(0, p - L_):p]
        pats.append(pat)
        qr[i, 0] = local_h[s // R]
        qr[i, 1] = len(pat)
        qr[i, 2:2 + len(pat)] = pat  # the pattern field starts at word 2 (<= max_pattern_len words)
        truth = tr.stream(s)[p:p + DL]
        qr[i, 10] = qr[i, 11] = tr.lengths[s] - p
        qr[i, 12:12 + len(truth)] = truth
    q_own = owner_g[st // R].astype(np.int32)
    args = D.SpeculationArgs(DL, 6, 1, KQ, 0.1, 1)
    d_args = torch.from_numpy(D.args_array([args]).view(np.uint8)).to(dev)
    lay = _lib.RecordLayout(QRY_W, 0, 1, 2, 10, 11, 12, RW, 0, 1, 6, 14, 22, 54)
    qseq = 1
    px.send("q", torch.from_numpy(q_own).to(dev), torch.from_numpy(qr).to(dev), qseq, origin_word=QRY_W - 1,
            want_slot=False)
    speculate_routed(srv, px, "q", "rep", qseq, lay, d_args, KQ, DL, origin_field=QRY_W - 1)
    px.wait("rep", qseq)
    torch.cuda.synchronize()
    back = px.slab("rep", qseq)[:Q].cpu().numpy()
    assert px.status()[0] is False and px.overflow.item() == 0
    oargs = O.make_args(DL, 6, 1, KQ, 0.1, 1)
    bad = 0
    drafted_total = 0
    for i in range(Q):
        exp = [c.key() for c in oidx[st[i] // R].speculate(pats[i], oargs)]
        got = _decode(back[i])
        if got != exp:
            bad += 1
        drafted_total += len(got)
        # verification (engine.cpp:115-143) against the record's truth
        acc = 0
        for c in got:
            m = 0
            while m < min(len(c[0]), qr[i, 10]) and c[0][m] == qr[i, 12 + m]:
                m += 1
            acc = max(acc, m)
        em = min(acc + 1, qr[i, 11])
        assert (back[i, 54], back[i, 55], back[i, 56]) == (sum(len(c[0]) for c in got), em - 1, em), i
    assert bad == 0, f"rank {rank}: {bad} of {Q} replies differ from the oracle"
    assert drafted_total > Q // 2
    dist.barrier()
    px.close()
    srv.close()
    dist.destroy_process_group()


def test_two_gpu_routed_parity(tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp
    errfile = str(tmp_path / "err")
    try:
        mp.spawn(_worker, args=(2, _free_port(), errfile), nprocs=2, join=True)
    except Exception:
        msgs = [open(errfile + f".{r}").read() for r in range(2) if os.path.exists(errfile + f".{r}")]
        raise AssertionError("\n".join(msgs) or "worker failed")


def _driver_worker(rank, world, port, errfile):
    try:
        _run_driver(rank, world, port)
    except Exception:
        with open(errfile + f".{rank}", "w") as f:
            f.write(traceback.format_exc())
        raise


def _run_driver(rank, world, port):
    """The C++ tick loop (dgds_px_driver_*): T routed ticks of appends + queries enqueued in one
    call; the replies of the last two ticks (still in their slab parities) must equal the oracle
    fed every earlier tick's appends, i.e. each tick's queries saw exactly the ticks before it."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    from oracle import oracle as O
    from paper_2511_14617_b200 import _lib
    from paper_2511_14617_b200 import dgds as D
    from paper_2511_14617_b200.peer import PeerExchange, TickDriver
    from paper_2511_14617_b200.workload import CONFIGS, generate_workload, group_id

    cfg = replace(CONFIGS["C1"], num_groups=8, group_size=4, location=400.0, max_tokens=400, vocab_size=40)
    tr = generate_workload(cfg)
    G, R = cfg.num_groups, cfg.group_size
    S = G * R
    owner_g = np.array([D.shard_of_group(group_id(g), world) for g in range(G)], np.int32)
    local_h = np.zeros(G, np.int32)
    for o in range(world):
        gs = np.nonzero(owner_g == o)[0]
        local_h[gs] = np.arange(len(gs), dtype=np.int32)
    srv = D.DraftServer(D.DgdsParams(), device=rank, expected_nodes=1 << 20, expected_streams=S)
    mine = np.nonzero(owner_g == rank)[0]
    assert (srv.group_handles([group_id(int(g)) for g in mine]) == np.arange(len(mine))).all()
    Q, T = 600, 12
    px = PeerExchange(world, rank, rank, {"a": (S, APP_W), "q": (Q, QRY_W), "rep": (Q, RW, "shared")})
    px.set_timeout(20.0)
    ora = O.restatement()
    oidx = {g: ora.index(group_id=group_id(g)) for g in range(G)}
    oargs = O.make_args(DL, 6, 1, KQ, 0.1, 1)
    rng = np.random.default_rng(300 + rank)
    produced = np.arange(rank, S, world)
    pos = np.zeros(S, np.int64)
    keep, expected = [], {}
    for t in range(T):
        # queries of tick t see the appends of ticks < t (K2 of a tick runs before its K1)
        st = rng.choice(np.nonzero(pos >= 2)[0], Q) if t > 0 else rng.integers(0, S, Q)
        qr = np.zeros((Q, QRY_W), np.int32)
        pats = []
        for i, s_ in enumerate(st):
            p = int(rng.integers(0, pos[s_] + 1))
            pat = tr.stream(s_)[max(0, p - int(rng.integers(0, 9))):p]
            pats.append(pat)
            truth = tr.stream(s_)[p:p + DL]
            qr[i, 0], qr[i, 1] = local_h[s_ // R], len(pat)
            qr[i, 2:2 + len(pat)] = pat
            qr[i, 10] = qr[i, 11] = max(1, tr.lengths[s_] - p)
            qr[i, 12:12 + len(truth)] = truth
        if t >= T - 2:
            expected[t] = [[c.key() for c in oidx[s_ // R].speculate(pat, oargs)] for s_, pat in zip(st, pats)]
        live = [s_ for s_ in range(S) if pos[s_] < tr.lengths[s_]]
        mine_live = [s_ for s_ in live if s_ % world == rank]
        rec = np.zeros((max(1, len(mine_live)), APP_W), np.int32)
        own = np.full(len(rec), -1, np.int32)
        for i, s_ in enumerate(mine_live):
            n = int(min(16, tr.lengths[s_] - pos[s_]))
            rec[i, :5] = [local_h[s_ // R], s_ % R, pos[s_] & 0xFFFFFFFF, pos[s_] >> 32, n]
            rec[i, 5:5 + n] = tr.stream(s_)[pos[s_]:pos[s_] + n]
            own[i] = owner_g[s_ // R]
        for s_ in live:  # every rank feeds the oracle every stream (the schedule is known to all)
            n = int(min(16, tr.lengths[s_] - pos[s_]))
            assert oidx[s_ // R].append(s_ % R, int(pos[s_]), tr.stream(s_)[pos[s_]:pos[s_] + n])[0]
            pos[s_] += n
        tensors = [torch.from_numpy(x).to(dev) for x in (owner_g[st // R].astype(np.int32), qr, own, rec)]
        keep.append(tensors)
    lay = _lib.RecordLayout(QRY_W, 0, 1, 2, 10, 11, 12, RW, 0, 1, 6, 14, 22, 54)
    d_args = torch.from_numpy(D.args_array([D.SpeculationArgs(DL, 6, 1, KQ, 0.1, 1)]).view(np.uint8)).to(dev)
    drv = TickDriver(srv, px, lay, d_args, KQ, DL, keep, QRY_W - 1)
    drv.run(0, T - 3, T - 2)  # a first run that plans ahead
    drv.run(T - 3, T)
    torch.cuda.synchronize()
    assert px.status()[0] is False and px.overflow.item() == 0
    for t in (T - 2, T - 1):
        back = px.slab("rep", t + 1)[:Q].cpu().numpy()
        bad = [i for i in range(Q) if _decode(back[i]) != expected[t][i]]
        assert not bad, f"rank {rank} tick {t}: {len(bad)} of {Q} replies differ from the oracle (first {bad[0]})"
    assert sum(int(r[0]) for r in back) > Q // 2
    dist.barrier()
    drv.close()
    assert srv.node_count() == sum(oidx[int(g)].node_count for g in mine)
    dist.barrier()
    px.close()
    srv.close()
    dist.destroy_process_group()


def test_two_gpu_native_tick_driver(tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp
    errfile = str(tmp_path / "err")
    try:
        mp.spawn(_driver_worker, args=(2, _free_port(), errfile), nprocs=2, join=True)
    except Exception:
        msgs = [open(errfile + f".{r}").read() for r in range(2) if os.path.exists(errfile + f".{r}")]
        raise AssertionError("\n".join(msgs) or "worker failed")


def test_cluster_on_two_gpus(restatement):
    """dgds_cluster_* with one shard per GPU (devices 0 and 1): the same differential as the
    one-GPU cluster test, so groups really live on different devices."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import test_gpu_parity as T
    T.test_cluster_routes_by_shard_and_matches_oracle(restatement, (0, 1))
