"""Staggered engine replay over the GPU draft server.

The reference declares the engine seam ``SpeculationSource`` (engine.hpp:67-74)
but ships no adapter; this module is that adapter plus the decode loop it
serves, restating ``Instance::decode_step`` (engine.cpp:69-167) for the draft
path only: the draft-length policy (:78-85), query construction (:88-113),
verification (:115-143, run on the GPU by dgds_verify_batch) and emission
(:147-161) into a DraftClient-style append buffer that flushes a stream once
``append_batch_tokens`` are pending (DraftClient::note_tokens / push_stream,
dgds.cpp:193-217). With fetch_period 0 the client answers from fresh
server-side state, which is what the GPU server returns.

Request r of every group is admitted at step r*stagger.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np

from .dgds import ARGS_DTYPE, DgdsParams, DraftServer, SpeculationArgs
from .workload import Trace, group_id


@dataclass
class ReplayConfig:
    stagger: int = 256
    append_batch_tokens: int = 16
    batch_token_budget: int = 64   # AdaptiveSpecPolicy (engine.hpp:28-33)
    per_request_cap: int = 8
    adaptive: bool = True
    multi_path_k: int = 1
    args: SpeculationArgs = None   # lookup bounds / cutoffs; max_spec_tokens and top_k set per step
    max_steps: int = 1 << 30
    t_base: float = 0.030          # StepTimeModel (engine.hpp:18-23)
    t_tok: float = 40e-6


class _ClientBuffer:
    """DraftClient pending-stream bookkeeping (dgds.hpp:146-150, dgds.cpp:193-217)."""

    def __init__(self, server: DraftServer, batch_tokens: int):
        self.server = server
        self.batch = batch_tokens
        self.pending = {}

    def note(self, gid: str, rid: int, toks: np.ndarray, out: list):
        if len(toks) == 0:
            return
        ps = self.pending.setdefault((gid, rid), [[], 0])
        ps[0].extend(int(t) for t in toks)
        if len(ps[0]) - ps[1] >= self.batch:
            out.append((gid, rid, ps))

    def push(self, flushes: list, now: float):
        # one batched update per step, in the order the reference would issue them
        while flushes:
            gids = [f[0] for f in flushes]
            rids = [f[1] for f in flushes]
            prevs = [f[2][1] for f in flushes]
            toks = [f[2][0][f[2][1]:] for f in flushes]
            reps = self.server.update_batch(gids, rids, prevs, toks, now)
            again = []
            for f, rep in zip(flushes, reps):
                ps = f[2]
                if rep.ok:
                    ps[1] = rep.acked_tokens
                elif ps[1] < rep.acked_tokens <= len(ps[0]):
                    ps[1] = rep.acked_tokens
                elif rep.acked_tokens < ps[1]:
                    ps[1] = rep.acked_tokens
                else:
                    raise RuntimeError("draft append resync cannot make progress for group " + f[0])
                if ps[1] < len(ps[0]):
                    again.append(f)
            flushes = again


def replay(trace: Trace, cfg: ReplayConfig, server: DraftServer = None, record: bool = True):
    """Returns (step_batch[list], records[N,4] of slot/drafted/accepted/emitted, n_queries)."""
    args = cfg.args or SpeculationArgs()
    G, R = trace.cfg.num_groups, trace.cfg.group_size
    if server is None:
        server = DraftServer(DgdsParams(append_batch_tokens=cfg.append_batch_tokens, fetch_period=0.0),
                             expected_nodes=max(1 << 16, int(trace.tokens.size) * 24))
    client = _ClientBuffer(server, cfg.append_batch_tokens)
    gids = [group_id(g) for g in range(G)]
    n = G * R
    lens = trace.lengths.astype(np.int64)
    offs = trace.offsets
    generated = np.zeros(n, np.int64)
    state = np.zeros(n, np.int8)  # 0 pending, 1 running, 2 finished
    running: List[int] = []
    step_batch, recs = [], []
    nq = 0
    now = 0.0
    step = 0
    finished = 0
    pmax, pmin = args.pattern_lookup_max, args.pattern_lookup_min
    k = max(1, cfg.multi_path_k)
    while finished < n and step < cfg.max_steps:
        for s in range(n):  # admission in (group, request) order, like the reference loop
            if state[s] == 0 and (s % R) * cfg.stagger == step:
                state[s] = 1
                running.append(s)
        if not running:
            step += 1
            step_batch.append(0)
            continue
        nr = len(running)
        d = max(min(cfg.per_request_cap, cfg.batch_token_budget // nr) if cfg.adaptive else cfg.per_request_cap, 0)
        run = np.asarray(running, np.int64)
        rem = lens[run] - generated[run]
        limit = rem  # chunk budget = whole response, so remaining_chunk == remaining_truth
        spec_len = np.minimum(d, limit - 1)
        pat_len = np.minimum(pmax, generated[run])
        use = (d > 0) & (spec_len > 0) & (pat_len >= pmin)
        qi = np.nonzero(use)[0]
        S = max(1, min(cfg.per_request_cap, server.params.max_spec_len))
        n_c = np.zeros(nr, np.int32)
        c_len = np.zeros(nr * k, np.int32)
        c_tok = np.zeros(nr * k * S, np.int32)
        if len(qi):
            nq += len(qi)
            pats, a = [], np.zeros(len(qi), ARGS_DTYPE)
            for j, i in enumerate(qi):
                s = int(run[i])
                g0 = offs[s] + generated[s]
                pats.append(trace.tokens[g0 - pat_len[i]:g0])
                a[j] = (spec_len[i], pmax, pmin, k, args.min_step_freq, args.min_support)
            poff = np.zeros(len(qi) + 1, np.uint64)
            poff[1:] = np.cumsum([len(p) for p in pats])
            flat = np.concatenate(pats).astype(np.int32)
            handles = server.group_handles(gids[int(run[i]) // R] for i in qi)
            cb = server.speculate_arrays(handles, poff, flat, a, 1)
            for j, i in enumerate(qi):
                nc = int(cb.n_cands[j])
                n_c[i] = nc
                for c in range(nc):
                    L = int(cb.lens[j * cb.k + c])
                    c_len[i * k + c] = L
                    c_tok[(i * k + c) * S:(i * k + c) * S + L] = cb.tokens[(j * cb.k + c) * cb.s:(j * cb.k + c) * cb.s + L]
        # verification on the GPU (engine.cpp:115-143)
        from .dgds import CandidateBatch
        vb = CandidateBatch(nr, k, S)
        vb.n_cands[:] = n_c
        vb.lens[:] = c_len
        vb.tokens[:] = c_tok
        truth = np.zeros((nr, S), np.int32)
        for i in range(nr):
            s = int(run[i])
            g0 = offs[s] + generated[s]
            m = min(S, int(rem[i]))
            truth[i, :m] = trace.tokens[g0:g0 + m]
        drafted, accepted, emitted = server.verify_batch(vb, truth, rem.astype(np.int32), limit.astype(np.int32))
        if record:
            step_batch.append(nr)
            for i in range(nr):
                recs.append((int(run[i] // R) * R + int(run[i] % R), int(drafted[i]), int(accepted[i]),
                             int(emitted[i])))
        duration = cfg.t_base + cfg.t_tok * float(np.sum(1 + drafted.astype(np.int64)))
        flushes = []
        for i in range(nr):
            s = int(run[i])
            e = int(emitted[i])
            g0 = offs[s] + generated[s]
            client.note(gids[s // R], s % R, trace.tokens[g0:g0 + e], flushes)
            generated[s] += e
        client.push(flushes, now)
        now += duration
        keep = []
        for s in running:
            if generated[s] >= lens[s]:
                state[s] = 2
                finished += 1
            else:
                keep.append(s)
        running = keep
        step += 1
    return step_batch, np.asarray(recs, np.int64).reshape(-1, 4), nq


def replay_device(trace: Trace, cfg: ReplayConfig, server: DraftServer = None, feedback: int = 0):
    """The same staggered replay with each decode step's draft path on the device
    (dgds_decode_step_device): the draft length d, per-request spec_len / pat_len / no-query rule,
    the queries and the verification all run in the step's kernels. The host keeps the request
    states and the append buffer. Returns (step_batch, records, d_sequence, device_next_d, admitted)
    where device_next_d[i] is the step kernel's d for step i+1 (exact when step i+1 admitted nobody)."""
    import ctypes as C

    import torch

    from . import _lib
    args = cfg.args or SpeculationArgs()
    G, R = trace.cfg.num_groups, trace.cfg.group_size
    if server is None:
        server = DraftServer(DgdsParams(append_batch_tokens=cfg.append_batch_tokens, fetch_period=0.0),
                             expected_nodes=max(1 << 16, int(trace.tokens.size) * 3))
    client = _ClientBuffer(server, cfg.append_batch_tokens)
    gids = [group_id(g) for g in range(G)]
    n = G * R
    lens = trace.lengths.astype(np.int64)
    offs = trace.offsets
    generated = np.zeros(n, np.int64)
    state = np.zeros(n, np.int8)
    running: List[int] = []
    step_batch, recs, ds, dev_next, admitted = [], [], [], [], []
    now, step, finished = 0.0, 0, 0
    k = max(1, cfg.multi_path_k)
    P = server.params
    S = max(1, min(cfg.per_request_cap, P.max_spec_len))
    W = P.max_pattern_len
    dev = torch.device("cuda", server.device)
    pol = _lib.SpecPolicy(1, 1 if cfg.adaptive else 0, cfg.batch_token_budget, cfg.per_request_cap, k, feedback)
    sa = _lib.SpecArgs(0, args.pattern_lookup_max, args.pattern_lookup_min, 1, args.min_step_freq, args.min_support)
    d_next = torch.zeros(1, dtype=torch.int32, device=dev)
    handles_all = server.group_handles(gids)
    L = _lib.lib()
    while finished < n and step < cfg.max_steps:
        adm = 0
        for s in range(n):
            if state[s] == 0 and (s % R) * cfg.stagger == step:
                state[s] = 1
                running.append(s)
                adm += 1
        if not running:
            step += 1
            step_batch.append(0)
            continue
        nr = len(running)
        d = max(min(cfg.per_request_cap, cfg.batch_token_budget // nr) if cfg.adaptive else cfg.per_request_cap, 0)
        ds.append(d)
        admitted.append(adm)
        run = np.asarray(running, np.int64)
        rem = (lens[run] - generated[run]).astype(np.int32)
        ctx = np.zeros((nr, W), np.int32)
        truth = np.zeros((nr, S), np.int32)
        for i in range(nr):
            s = int(run[i])
            g0 = offs[s] + generated[s]
            c = int(min(generated[s], W))
            ctx[i, :c] = trace.tokens[g0 - c:g0]
            m = min(S, int(rem[i]))
            truth[i, :m] = trace.tokens[g0:g0 + m]
        t = {name: torch.from_numpy(np.ascontiguousarray(x)).to(dev) for name, x in (
            ("h", handles_all[run // R].astype(np.int32)), ("ctx", ctx), ("gen", generated[run].astype(np.int32)),
            ("lim", rem), ("tru", truth), ("tl", rem))}
        v = torch.zeros((3, nr), dtype=torch.int32, device=dev)
        vo = _lib.VerifyOut(v[0].data_ptr(), v[1].data_ptr(), v[2].data_ptr())
        p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
        _lib.check(L.dgds_decode_step_device(server.handle, nr, p(t["h"]), p(t["ctx"]), W, p(t["gen"]), p(t["lim"]),
                                             p(t["tru"]), S, p(t["tl"]), C.byref(sa), C.byref(pol), None, d, None,
                                             C.byref(vo), p(d_next), None, C.c_void_p(server.cuda_stream)))
        torch.cuda.synchronize()
        drafted, accepted, emitted = (x.cpu().numpy() for x in v)
        dev_next.append(int(d_next.item()))
        step_batch.append(nr)
        for i in range(nr):
            recs.append((int(run[i] // R) * R + int(run[i] % R), int(drafted[i]), int(accepted[i]), int(emitted[i])))
        duration = cfg.t_base + cfg.t_tok * float(np.sum(1 + drafted.astype(np.int64)))
        flushes = []
        for i in range(nr):
            s = int(run[i])
            e = int(emitted[i])
            g0 = offs[s] + generated[s]
            client.note(gids[s // R], s % R, trace.tokens[g0:g0 + e], flushes)
            generated[s] += e
        client.push(flushes, now)
        now += duration
        keep = []
        for s in running:
            if generated[s] >= lens[s]:
                state[s] = 2
                finished += 1
            else:
                keep.append(s)
        running = keep
        step += 1
    return step_batch, np.asarray(recs, np.int64).reshape(-1, 4), ds, dev_next, admitted
