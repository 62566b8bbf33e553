"""ctypes loaders for the CPU checkers under oracle/ — TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs. The product package never imports this module.

* :func:`restatement` -> our C++ restatement (oracle/liboracle.so, cst_oracle.cpp)
* :func:`reference`   -> the reference sources compiled in place
  (oracle/_ref/libdgds_ref.so via ref_capi.cpp), or ``None`` when absent.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libdgds_ref.so")


class OrcArgs(C.Structure):
    """rollsim::SpeculationArgs (proj/include/rollsim/cst.hpp:16-23)."""

    _fields_ = [
        ("max_spec_tokens", C.c_int32),
        ("pattern_lookup_max", C.c_int32),
        ("pattern_lookup_min", C.c_int32),
        ("top_k", C.c_int32),
        ("min_step_freq", C.c_double),
        ("min_support", C.c_int64),
    ]


class OrcCands(C.Structure):
    _fields_ = [
        ("tokens", C.POINTER(C.c_int32)),
        ("lens", C.POINTER(C.c_int32)),
        ("scores", C.POINTER(C.c_double)),
        ("supports", C.POINTER(C.c_int64)),
        ("k_cap", C.c_int32),
        ("s_cap", C.c_int32),
        ("n", C.c_int32),
    ]


class OrcQStats(C.Structure):
    _fields_ = [
        ("suffix_lookups", C.c_int64),
        ("expansions", C.c_int64),
        ("children", C.c_int64),
        ("child_sectors", C.c_int64),
        ("cand_tokens", C.c_int64),
        ("cands", C.c_int64),
    ]


class OrcWcfg(C.Structure):
    _fields_ = [
        ("num_groups", C.c_int32),
        ("group_size", C.c_int32),
        ("length_family", C.c_int32),
        ("vocab_size", C.c_int32),
        ("location", C.c_double),
        ("scale", C.c_double),
        ("group_correlation", C.c_double),
        ("noise_base", C.c_double),
        ("pattern_similarity", C.c_double),
        ("prompt_mean", C.c_double),
        ("prompt_spread", C.c_double),
        ("max_tokens", C.c_int32),
        ("pad_", C.c_int32),
        ("seed", C.c_uint64),
    ]


class OrcReplayCfg(C.Structure):
    _fields_ = [
        ("stagger_steps", C.c_int32),
        ("append_batch_tokens", C.c_int32),
        ("batch_token_budget", C.c_int32),
        ("per_request_cap", C.c_int32),
        ("adaptive_enabled", C.c_int32),
        ("multi_path_k", C.c_int32),
        ("max_pattern_len", C.c_int32),
        ("max_spec_len", C.c_int32),
        ("max_steps", C.c_int32),
        ("pad_", C.c_int32),
        ("args", OrcArgs),
    ]


def make_args(max_spec_tokens=8, pattern_lookup_max=6, pattern_lookup_min=1, top_k=1,
              min_step_freq=0.25, min_support=1) -> OrcArgs:
    return OrcArgs(max_spec_tokens, pattern_lookup_max, pattern_lookup_min, top_k,
                   float(min_step_freq), int(min_support))


@dataclass(frozen=True)
class Candidate:
    tokens: tuple
    score: float
    support: int

    def key(self):
        """Bit-exact comparison key (score as its raw IEEE-754 pattern)."""
        return (self.tokens, np.float64(self.score).view(np.uint64).item(), self.support)


class OracleError(RuntimeError):
    pass


def _i32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


class _Lib:
    def __init__(self, path: str):
        self.path = path
        L = C.CDLL(path)
        self.L = L
        L.orc_last_error.restype = C.c_char_p
        L.orc_index_new.restype = C.c_void_p
        L.orc_index_new.argtypes = [C.c_char_p, C.c_int32, C.c_int32]
        L.orc_index_free.argtypes = [C.c_void_p]
        L.orc_index_append.argtypes = [C.c_void_p, C.c_int32, C.c_uint64, C.POINTER(C.c_int32), C.c_uint64,
                                       C.POINTER(C.c_int32), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.orc_index_speculate.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_uint64, C.POINTER(OrcArgs),
                                          C.POINTER(OrcCands)]
        L.orc_index_speculate_stats.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_uint64,
                                                C.POINTER(OrcArgs), C.POINTER(OrcCands), C.POINTER(OrcQStats)]
        L.orc_index_version.restype = C.c_uint64
        L.orc_index_version.argtypes = [C.c_void_p]
        L.orc_index_node_count.restype = C.c_uint64
        L.orc_index_node_count.argtypes = [C.c_void_p]
        L.orc_index_stored_tokens.restype = C.c_uint64
        L.orc_index_stored_tokens.argtypes = [C.c_void_p, C.c_int32]
        L.orc_oracle_speculate.argtypes = [C.POINTER(C.c_int32), C.POINTER(C.c_uint64), C.c_uint64,
                                           C.POINTER(C.c_int32), C.c_uint64, C.POINTER(OrcArgs),
                                           C.POINTER(OrcCands)]

    def err(self):
        return OracleError(self.L.orc_last_error().decode())

    def index(self, group_id="g", max_pattern_len=8, max_spec_len=16) -> "Index":
        return Index(self, group_id, max_pattern_len, max_spec_len)

    def oracle_speculate(self, sequences, pattern, args: OrcArgs):
        """speculate_oracle (proj/src/cst.cpp:386-453)."""
        offs = np.zeros(len(sequences) + 1, dtype=np.uint64)
        for i, s in enumerate(sequences):
            offs[i + 1] = offs[i] + len(s)
        flat = np.ascontiguousarray(np.concatenate([np.asarray(s, np.int32) for s in sequences])
                                    if sequences else np.zeros(0, np.int32), dtype=np.int32)
        pat = np.ascontiguousarray(pattern, dtype=np.int32)
        out, bufs = _cands(args)
        rc = self.L.orc_oracle_speculate(
            _i32p(flat), offs.ctypes.data_as(C.POINTER(C.c_uint64)), len(sequences), _i32p(pat), len(pat),
            C.byref(args), C.byref(out))
        if rc != 0:
            raise self.err()
        return _read(out, bufs)


def _cands(args: OrcArgs, s_cap=None):
    k = max(1, int(args.top_k))
    s = max(1, int(s_cap if s_cap is not None else max(args.max_spec_tokens, 1)))
    toks = np.zeros(k * s, np.int32)
    lens = np.zeros(k, np.int32)
    scores = np.zeros(k, np.float64)
    sup = np.zeros(k, np.int64)
    out = OrcCands(_i32p(toks), _i32p(lens), scores.ctypes.data_as(C.POINTER(C.c_double)),
                   sup.ctypes.data_as(C.POINTER(C.c_int64)), k, s, 0)
    return out, (toks, lens, scores, sup, s)


def _read(out: OrcCands, bufs):
    toks, lens, scores, sup, s = bufs
    res = []
    for i in range(out.n):
        res.append(Candidate(tuple(int(x) for x in toks[i * s:i * s + lens[i]]), float(scores[i]), int(sup[i])))
    return res


class Index:
    """GroupDraftIndex (proj/include/rollsim/cst.hpp:42-138) behind the oracle C ABI."""

    def __init__(self, lib: _Lib, group_id, max_pattern_len, max_spec_len):
        self.lib = lib
        self.h = lib.L.orc_index_new(group_id.encode(), max_pattern_len, max_spec_len)
        if not self.h:
            raise lib.err()
        self.max_spec_len = max_spec_len

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.orc_index_free(self.h)
            self.h = None

    def append(self, request_id, prev_token_count, tokens):
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        ok = C.c_int32()
        ver = C.c_uint64()
        ack = C.c_uint64()
        rc = self.lib.L.orc_index_append(self.h, request_id, prev_token_count, _i32p(t), len(t), C.byref(ok),
                                         C.byref(ver), C.byref(ack))
        if rc != 0:
            raise self.lib.err()
        return bool(ok.value), int(ver.value), int(ack.value)

    def speculate(self, pattern, args: OrcArgs):
        pat = np.ascontiguousarray(pattern, dtype=np.int32)
        out, bufs = _cands(args, max(1, min(int(args.max_spec_tokens), self.max_spec_len)))
        rc = self.lib.L.orc_index_speculate(self.h, _i32p(pat), len(pat), C.byref(args), C.byref(out))
        if rc != 0:
            raise self.lib.err()
        return _read(out, bufs)

    def speculate_stats(self, pattern, args: OrcArgs):
        pat = np.ascontiguousarray(pattern, dtype=np.int32)
        out, bufs = _cands(args, max(1, min(int(args.max_spec_tokens), self.max_spec_len)))
        st = OrcQStats()
        rc = self.lib.L.orc_index_speculate_stats(self.h, _i32p(pat), len(pat), C.byref(args), C.byref(out),
                                                  C.byref(st))
        if rc != 0:
            raise self.lib.err()
        return _read(out, bufs), st

    @property
    def version(self):
        return int(self.lib.L.orc_index_version(self.h))

    @property
    def node_count(self):
        return int(self.lib.L.orc_index_node_count(self.h))

    def stored_tokens(self, rid):
        return int(self.lib.L.orc_index_stored_tokens(self.h, rid))


class RefLib(_Lib):
    """Extra entry points only the compiled reference exports (server, workload, replay)."""

    def __init__(self, path):
        super().__init__(path)
        L = self.L
        L.orc_ref_shard_of_group.argtypes = [C.c_char_p, C.c_int32]
        L.orc_ref_fnv1a64.restype = C.c_uint64
        L.orc_ref_fnv1a64.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_ref_server_new.restype = C.c_void_p
        L.orc_ref_server_new.argtypes = [C.c_int32, C.c_double, C.c_int32, C.c_double, C.c_int32, C.c_int32]
        L.orc_ref_server_free.argtypes = [C.c_void_p]
        L.orc_ref_server_update.argtypes = [C.c_void_p, C.c_char_p, C.c_int32, C.c_uint64, C.POINTER(C.c_int32),
                                            C.c_uint64, C.c_double, C.POINTER(C.c_int32),
                                            C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.orc_ref_server_speculate.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_int32), C.c_uint64,
                                               C.POINTER(OrcArgs), C.POINTER(OrcCands)]
        L.orc_ref_server_register.argtypes = [C.c_void_p, C.c_char_p, C.c_double, C.c_double]
        L.orc_ref_server_drop.argtypes = [C.c_void_p, C.c_char_p]
        L.orc_ref_server_sweep.argtypes = [C.c_void_p, C.c_double]
        L.orc_ref_server_has_group.argtypes = [C.c_void_p, C.c_char_p]
        L.orc_ref_server_group_version.restype = C.c_uint64
        L.orc_ref_server_group_version.argtypes = [C.c_void_p, C.c_char_p]
        L.orc_ref_server_shard_group_count.restype = C.c_uint64
        L.orc_ref_server_shard_group_count.argtypes = [C.c_void_p, C.c_int32]
        L.orc_ref_server_fetch.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64, C.c_double, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_uint64), C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.orc_ref_server_compact.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64]
        L.orc_index_full_snapshot.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.orc_index_delta_since.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int32), C.c_void_p, C.c_uint64,
                                            C.POINTER(C.c_uint64)]
        L.orc_index_apply_blob.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.orc_index_compact.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_ref_wire_serve.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_double, C.c_void_p, C.c_uint64,
                                         C.POINTER(C.c_uint64)]
        L.orc_ref_tcp_new.restype = C.c_void_p
        L.orc_ref_tcp_new.argtypes = [C.c_char_p, C.c_int32]
        L.orc_ref_tcp_free.argtypes = [C.c_void_p]
        L.orc_ref_tcp_update.argtypes = [C.c_void_p, C.c_char_p, C.c_int32, C.c_uint64, C.POINTER(C.c_int32),
                                         C.c_uint64, C.POINTER(C.c_int32), C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint64)]
        L.orc_ref_tcp_fetch.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_uint64), C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.orc_ref_tcp_register.argtypes = [C.c_void_p, C.c_char_p, C.c_double]
        L.orc_ref_service_new.restype = C.c_void_p
        L.orc_ref_service_new.argtypes = [C.c_int32]
        L.orc_ref_service_port.argtypes = [C.c_void_p]
        L.orc_ref_service_free.argtypes = [C.c_void_p]
        L.orc_ref_workload_new.restype = C.c_void_p
        L.orc_ref_workload_new.argtypes = [C.POINTER(OrcWcfg)]
        L.orc_ref_workload_free.argtypes = [C.c_void_p]
        L.orc_ref_workload_num_groups.argtypes = [C.c_void_p]
        L.orc_ref_workload_group_id.restype = C.c_char_p
        L.orc_ref_workload_group_id.argtypes = [C.c_void_p, C.c_int32]
        L.orc_ref_workload_prompt_len.argtypes = [C.c_void_p, C.c_int32]
        L.orc_ref_workload_group_size.argtypes = [C.c_void_p, C.c_int32]
        L.orc_ref_workload_output_len.restype = C.c_int64
        L.orc_ref_workload_output_len.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        L.orc_ref_workload_output.restype = C.POINTER(C.c_int32)
        L.orc_ref_workload_output.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        L.orc_ref_workload_fingerprint.restype = C.c_uint64
        L.orc_ref_workload_fingerprint.argtypes = [C.c_void_p]
        L.orc_ref_gset_new.restype = C.c_void_p
        L.orc_ref_gset_new.argtypes = [C.c_int32, C.POINTER(C.c_char_p), C.c_int32, C.c_int32]
        L.orc_ref_gset_free.argtypes = [C.c_void_p]
        L.orc_ref_gset_append.argtypes = [C.c_void_p, C.c_int64] + [C.c_void_p] * 5 + [C.c_int32] + [C.c_void_p] * 3
        L.orc_ref_gset_speculate.argtypes = ([C.c_void_p, C.c_int64] + [C.c_void_p] * 4 + [C.c_int32, C.c_int32,
                                                                                          C.c_int32]
                                             + [C.c_void_p] * 5)
        L.orc_ref_gset_node_count.restype = C.c_uint64
        L.orc_ref_gset_node_count.argtypes = [C.c_void_p]
        L.orc_ref_replay.restype = C.c_int64
        L.orc_ref_replay.argtypes = [C.c_void_p, C.POINTER(OrcReplayCfg), C.POINTER(C.c_int32), C.c_int64,
                                     C.POINTER(C.c_int32), C.c_int64, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_uint64)]

    def shard_of_group(self, gid: str, n: int) -> int:
        return int(self.L.orc_ref_shard_of_group(gid.encode(), n))

    # ---- many GroupDraftIndex objects in bulk (scale parity tests) ----
    def group_set(self, gids, max_pattern_len=8, max_spec_len=16) -> "GroupSet":
        return GroupSet(self, gids, max_pattern_len, max_spec_len)

    # ---- replica sync (GDX1 blobs) ----
    def _blob_call(self, fn, *args):
        cap = 1 << 16
        while True:
            buf = C.create_string_buffer(cap)
            ln = C.c_uint64()
            rc = fn(*args, buf, cap, C.byref(ln))
            if rc == -2:
                cap = int(ln.value)
                continue
            if rc != 0:
                raise self.err()
            return buf.raw[:ln.value]

    def server_fetch(self, srv, gid: str, cached: int, now: float):
        """DraftServer::fetch_cst for one group -> (kind, version, blob bytes)."""
        kind, ver = C.c_int32(), C.c_uint64()
        blob = self._blob_call(lambda b, c, l: self.L.orc_ref_server_fetch(srv, gid.encode(), cached, now,
                                                                           C.byref(kind), C.byref(ver), b, c, l))
        return int(kind.value), int(ver.value), blob

    def wire_serve(self, srv, payload: bytes, now: float) -> bytes:
        """wire::serve_payload (dgds_wire.cpp:103-143)."""
        buf = C.create_string_buffer(bytes(payload), max(1, len(payload)))
        return self._blob_call(lambda b, c, l: self.L.orc_ref_wire_serve(srv, buf, len(payload), now, b, c, l))

    def server_compact(self, srv, gid: str, before: int):
        if self.L.orc_ref_server_compact(srv, gid.encode(), before) != 0:
            raise self.err()

    def index_full_snapshot(self, idx) -> bytes:
        return self._blob_call(lambda b, c, l: self.L.orc_index_full_snapshot(idx.h, b, c, l))

    def index_delta_since(self, idx, since: int):
        avail = C.c_int32()
        blob = self._blob_call(lambda b, c, l: self.L.orc_index_delta_since(idx.h, since, C.byref(avail), b, c, l))
        return blob if avail.value else None

    def index_apply_blob(self, idx, blob: bytes) -> int:
        ver = C.c_uint64()
        buf = C.create_string_buffer(bytes(blob), len(blob))
        if self.L.orc_index_apply_blob(idx.h, buf, len(blob), C.byref(ver)) != 0:
            raise self.err()
        return int(ver.value)

    def index_compact(self, idx, before: int):
        if self.L.orc_index_compact(idx.h, before) != 0:
            raise self.err()

    def workload(self, **cfg):
        """generate_workload (proj/src/workload.cpp:51-103) -> (group_ids, prompt_lens, outputs)."""
        c = wcfg(**cfg)
        h = self.L.orc_ref_workload_new(C.byref(c))
        if not h:
            raise self.err()
        try:
            ids, plens, outs = [], [], []
            for g in range(self.L.orc_ref_workload_num_groups(h)):
                ids.append(self.L.orc_ref_workload_group_id(h, g).decode())
                plens.append(self.L.orc_ref_workload_prompt_len(h, g))
                gs = []
                for i in range(self.L.orc_ref_workload_group_size(h, g)):
                    n = self.L.orc_ref_workload_output_len(h, g, i)
                    p = self.L.orc_ref_workload_output(h, g, i)
                    gs.append(np.ctypeslib.as_array(p, shape=(n,)).copy())
                outs.append(gs)
            fp = int(self.L.orc_ref_workload_fingerprint(h))
        finally:
            self.L.orc_ref_workload_free(h)
        return ids, plens, outs, fp

    def replay(self, cfg: dict, replay: OrcReplayCfg, step_cap=1 << 20, rec_cap=1 << 24):
        c = wcfg(**cfg)
        h = self.L.orc_ref_workload_new(C.byref(c))
        if not h:
            raise self.err()
        try:
            sb = np.zeros(step_cap, np.int32)
            rec = np.zeros(4 * rec_cap, np.int32)
            nrec = C.c_int64()
            nq = C.c_uint64()
            steps = self.L.orc_ref_replay(h, C.byref(replay), _i32p(sb), step_cap, _i32p(rec), rec_cap,
                                          C.byref(nrec), C.byref(nq))
            if steps < 0:
                raise self.err()
        finally:
            self.L.orc_ref_workload_free(h)
        return sb[:steps].copy(), rec[:4 * nrec.value].reshape(-1, 4).copy(), int(nq.value)


class GroupSet:
    """The reference GroupDraftIndex for many groups, appended and queried in bulk on host
    threads split by group (oracle/ref_capi.cpp orc_ref_gset_*). TEST INFRASTRUCTURE ONLY."""

    def __init__(self, lib: "RefLib", gids, max_pattern_len, max_spec_len):
        import numpy as np
        self.lib, self.np = lib, np
        arr = (C.c_char_p * len(gids))(*[g.encode() for g in gids])
        self.h = lib.L.orc_ref_gset_new(len(gids), arr, max_pattern_len, max_spec_len)
        if not self.h:
            raise OracleError(lib.err())
        self.threads = os.cpu_count() or 8

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.orc_ref_gset_free(self.h)
            self.h = None

    def append(self, group, rid, prev, offs, tokens):
        np = self.np
        n = len(group)
        group, rid = np.ascontiguousarray(group, np.int32), np.ascontiguousarray(rid, np.int32)
        prev, offs = np.ascontiguousarray(prev, np.uint64), np.ascontiguousarray(offs, np.uint64)
        tokens = np.ascontiguousarray(tokens, np.int32)
        ok = np.zeros(n, np.int32)
        ver = np.zeros(n, np.uint64)
        ack = np.zeros(n, np.uint64)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        if self.lib.L.orc_ref_gset_append(self.h, n, p(group), p(rid), p(prev), p(offs), p(tokens), self.threads,
                                          p(ok), p(ver), p(ack)):
            raise OracleError(self.lib.err())
        return ok, ver, ack

    def speculate(self, group, pat_offs, pats, args, k_cap, s_cap):
        """args: one OrcArgs per query (ctypes array). Returns n_cands, lens, scores, supports, tokens
        shaped [n], [n,k], [n,k], [n,k], [n,k,s]."""
        np = self.np
        n = len(group)
        group = np.ascontiguousarray(group, np.int32)
        pat_offs = np.ascontiguousarray(pat_offs, np.uint64)
        pats = np.ascontiguousarray(pats, np.int32)
        nc = np.zeros(n, np.int32)
        ln = np.zeros((n, k_cap), np.int32)
        sc = np.zeros((n, k_cap), np.float64)
        sp = np.zeros((n, k_cap), np.int64)
        tk = np.zeros((n, k_cap, s_cap), np.int32)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        if self.lib.L.orc_ref_gset_speculate(self.h, n, p(group), p(pat_offs), p(pats), C.cast(args, C.c_void_p),
                                             self.threads, k_cap, s_cap, p(nc), p(ln), p(sc), p(sp), p(tk)):
            raise OracleError(self.lib.err())
        return nc, ln, sc, sp, tk

    def node_count(self) -> int:
        return int(self.lib.L.orc_ref_gset_node_count(self.h))


def wcfg(num_groups=1, group_size=16, length_family=0, vocab_size=32000, location=4096.0, scale=0.0,
         group_correlation=1.0, noise_base=0.5, pattern_similarity=0.8, prompt_mean=512.0,
         prompt_spread=128.0, max_tokens=4096, seed=7) -> OrcWcfg:
    return OrcWcfg(num_groups, group_size, length_family, vocab_size, location, scale, group_correlation,
                   noise_base, pattern_similarity, prompt_mean, prompt_spread, max_tokens, 0, seed)


_cache = {}


def build():
    """Compile the checkers (make -C oracle). The reference part only builds when /root/reference exists."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def restatement() -> _Lib:
    if "o" not in _cache:
        if not os.path.exists(LIB_ORACLE):
            build()
        _cache["o"] = _Lib(LIB_ORACLE)
    return _cache["o"]


def reference():
    """The compiled reference, or None when it was never built (no /root/reference here)."""
    if "r" not in _cache:
        _cache["r"] = RefLib(LIB_REF) if os.path.exists(LIB_REF) else None
    return _cache["r"]
