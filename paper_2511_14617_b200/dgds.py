"""Python mirror of the reference draft-server interface over the B200 C ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/rollsim/dgds.hpp:18-162, cst.hpp:16-32,
engine.hpp:28-33) so the parity tests read like the reference's own contract
(SPEC.md:107-264): ``update_cst`` returns an :class:`UpdateReply` (an
out-of-order append is a value, not an error), ``speculate`` returns a list of
:class:`DraftCandidate` in ``candidate_before`` order, invalid arguments raise
``ValueError`` (the reference's ``std::invalid_argument``).

Every call runs on the GPU through libdgds_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib


@dataclass
class SpeculationArgs:
    """rollsim::SpeculationArgs (cst.hpp:16-23)."""

    max_spec_tokens: int = 8
    pattern_lookup_max: int = 6
    pattern_lookup_min: int = 1
    top_k: int = 1
    min_step_freq: float = 0.25
    min_support: int = 1

    def c(self) -> _lib.SpecArgs:
        return _lib.SpecArgs(self.max_spec_tokens, self.pattern_lookup_max, self.pattern_lookup_min, self.top_k,
                             float(self.min_step_freq), int(self.min_support))


ARGS_DTYPE = np.dtype([("max_spec_tokens", "<i4"), ("pattern_lookup_max", "<i4"), ("pattern_lookup_min", "<i4"),
                       ("top_k", "<i4"), ("min_step_freq", "<f8"), ("min_support", "<i8")])


def args_array(args: Sequence[SpeculationArgs]) -> np.ndarray:
    a = np.zeros(len(args), ARGS_DTYPE)
    for i, x in enumerate(args):
        a[i] = (x.max_spec_tokens, x.pattern_lookup_max, x.pattern_lookup_min, x.top_k, x.min_step_freq,
                x.min_support)
    return a


@dataclass(frozen=True)
class DraftCandidate:
    """rollsim::DraftCandidate (cst.hpp:25-29)."""

    tokens: tuple
    score: float
    support: int

    def key(self):
        """Bit-exact comparison key (score as its raw IEEE-754 bit pattern)."""
        return (self.tokens, np.float64(self.score).view(np.uint64).item(), self.support)


class FetchKind:  # dgds.hpp:31
    UpToDate, Delta, Full, UnknownGroup = 0, 1, 2, 3


@dataclass(frozen=True)
class FetchReply:  # dgds.hpp:33-37
    kind: int
    version: int
    blob: bytes


@dataclass(frozen=True)
class UpdateReply:
    """rollsim::UpdateReply (dgds.hpp:39-43)."""

    ok: bool
    version: int
    acked_tokens: int


@dataclass
class DgdsParams:
    """rollsim::DgdsParams (dgds.hpp:18-24) incl. GroupDraftIndex::Limits (cst.hpp:44-47)."""

    shard_count: int = 1
    fetch_period: float = 0.2
    append_batch_tokens: int = 16
    default_ttl_seconds: float = 600.0
    max_pattern_len: int = 8
    max_spec_len: int = 16


@dataclass
class SpecQuery:
    """rollsim::SpecQuery (dgds.hpp:118-122)."""

    group_id: str
    pattern: Sequence[int]
    args: SpeculationArgs = field(default_factory=SpeculationArgs)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def shard_of_group(group_id: str, shard_count: int) -> int:
    """shard_of_group (dgds.cpp:10-14): fnv1a64(group_id) % shard_count."""
    if shard_count < 1:
        raise ValueError("shard_count must be >= 1")
    b = group_id.encode()
    return int(lib().dgds_shard_of_group(b, len(b), shard_count))


def fnv1a64(data: bytes) -> int:
    return int(lib().dgds_fnv1a64(data, len(data)))


def draft_len(sd_enabled: bool, adaptive: bool, per_request_cap: int, batch_token_budget: int, n_running: int) -> int:
    """Instance::decode_step draft-length policy (engine.cpp:78-85)."""
    return int(lib().dgds_draft_len(int(sd_enabled), int(adaptive), per_request_cap, batch_token_budget, n_running))


class DraftServer:
    """GPU-resident rollsim::DraftServer (dgds.hpp:51-91) on one CUDA device."""

    def __init__(self, params: Optional[DgdsParams] = None, device: int = 0, expected_nodes: int = 0,
                 expected_streams: int = 0):
        self.params = params or DgdsParams()
        p = self.params
        cp = _lib.Params(p.shard_count, p.append_batch_tokens, p.fetch_period, p.default_ttl_seconds,
                         p.max_pattern_len, p.max_spec_len, device, 0, expected_nodes, expected_streams)
        h = C.c_void_p()
        check(lib().dgds_create(C.byref(cp), C.byref(h)))
        self._h = h
        self._handles = {}
        self.device = device

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            flags = 0
            if os.environ.get("DGDS_ASSERT_CLEAN"):  # test runs: device error flags must stay clear
                out = C.c_int32()
                check(lib().dgds_device_error(self._h, C.byref(out)))
                flags = out.value
            lib().dgds_destroy(self._h)
            self._h = None
            if flags:
                raise RuntimeError("device error flags 0x%x at close (dgds_device_error)" % flags)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def cuda_stream(self) -> int:
        return int(lib().dgds_cuda_stream(self._h) or 0)

    # ---- group identity -------------------------------------------------
    def group_handle(self, group_id: str) -> int:
        h = self._handles.get(group_id)
        if h is None:
            b = group_id.encode()
            out = C.c_int32()
            check(lib().dgds_intern(self._h, b, len(b), C.byref(out)))
            h = self._handles[group_id] = out.value
        return h

    def group_handles(self, group_ids: Iterable[str]) -> np.ndarray:
        return np.fromiter((self.group_handle(g) for g in group_ids), dtype=np.int32)

    # ---- DraftServer API ----------------------------------------------------
    def register_group(self, group_id: str, ttl_seconds: float, now: float):
        check(lib().dgds_register_group(self._h, self.group_handle(group_id), float(ttl_seconds), float(now)))

    def drop_group(self, group_id: str):
        check(lib().dgds_drop_group(self._h, self.group_handle(group_id)))

    def sweep_expired(self, now: float):
        check(lib().dgds_sweep_expired(self._h, float(now)))

    def has_group(self, group_id: str) -> bool:
        out = C.c_int32()
        check(lib().dgds_has_group(self._h, self.group_handle(group_id), C.byref(out)))
        return bool(out.value)

    def group_version(self, group_id: str) -> int:
        out = C.c_uint64()
        check(lib().dgds_group_version(self._h, self.group_handle(group_id), C.byref(out)))
        return int(out.value)

    def stored_tokens(self, group_id: str, request_id: int) -> int:
        out = C.c_uint64()
        check(lib().dgds_stored_tokens(self._h, self.group_handle(group_id), request_id, C.byref(out)))
        return int(out.value)

    def shard_count(self) -> int:
        return self.params.shard_count

    def shard_group_count(self, shard: int) -> int:
        out = C.c_uint64()
        check(lib().dgds_shard_group_count(self._h, shard, C.byref(out)))
        return int(out.value)

    def node_count(self) -> int:
        out = C.c_uint64()
        check(lib().dgds_node_count(self._h, C.byref(out)))
        return int(out.value)

    def entry_count(self) -> int:
        """Table entries in use (nodes with count >= 2 and leaves)."""
        out = C.c_uint64()
        check(lib().dgds_entry_count(self._h, C.byref(out)))
        return out.value

    def device_error(self) -> int:
        """Reads and clears the device error flags (0 = clean); see dgds_device_error."""
        out = C.c_int32()
        check(lib().dgds_device_error(self._h, C.byref(out)))
        return out.value

    def batch_speculate_zc(self, d_handles, d_pat_end, d_pat_len, d_pattern_buffer, d_out_offsets,
                           d_output_buffer, layout, d_args, args_stride: int, max_top_k: int, max_spec: int,
                           d_stats=None, stream: int = 0) -> None:
        """The paper's zero-copy batch_speculate: device tensors in, reply records
        written into the engine's output buffer at d_out_offsets (dgds_batch_speculate_zc)."""
        p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        check(lib().dgds_batch_speculate_zc(self._h, int(d_handles.shape[0]), p(d_handles), p(d_pat_end),
                                            p(d_pat_len), p(d_pattern_buffer), p(d_out_offsets), p(d_output_buffer),
                                            C.byref(layout), p(d_args), args_stride, max_top_k, max_spec,
                                            p(d_stats) if d_stats is not None else None,
                                            C.c_void_p(stream or None)))

    # ---- replica sync (GDX1 blobs, cst.cpp:233-329; fetch_cst, dgds.cpp:53-97) ----
    def fetch_cst(self, group_ids: Sequence[str], cached_versions: Sequence[int], now: float) -> List[FetchReply]:
        """DraftServer::fetch_cst: per group UpToDate / Delta / Full / UnknownGroup with the
        reference's byte-exact blob."""
        if len(group_ids) != len(cached_versions):
            raise ValueError("fetch_cst: group_ids and draft_cache_infos must have equal length")
        n = len(group_ids)
        if n == 0:
            return []
        hs = np.ascontiguousarray(self.group_handles(group_ids), np.int32)
        cv = np.ascontiguousarray(cached_versions, np.uint64)
        reps = (_lib.FetchReply * n)()
        base = C.c_void_p()
        check(lib().dgds_fetch_cst(self._h, n, _ptr(hs), _ptr(cv), float(now), reps, C.byref(base)))
        out = []
        for r in reps:
            blob = C.string_at(base.value + r.blob_off, r.blob_len) if r.blob_len else b""
            out.append(FetchReply(int(r.kind), int(r.version), blob))
        return out

    def compact_group(self, group_id: str, before_version: int):
        check(lib().dgds_compact_group(self._h, self.group_handle(group_id), int(before_version)))

    def apply_blob(self, group_id: str, blob: bytes, now: float = 0.0) -> int:
        """GroupDraftIndex::apply_blob on this server's copy of the group (a GPU replica)."""
        v = C.c_uint64()
        buf = C.create_string_buffer(bytes(blob), len(blob))
        check(lib().dgds_apply_blob(self._h, self.group_handle(group_id), buf, len(blob), float(now), C.byref(v)))
        return int(v.value)

    def compact_memory(self):
        """Reclaim retired groups' slots (same-capacity rebuild) and history (dgds_compact_memory)."""
        check(lib().dgds_compact_memory(self._h))

    def memory_stats(self) -> dict:
        m = _lib.MemoryStats()
        check(lib().dgds_get_memory_stats(self._h, C.byref(m)))
        return {k: int(getattr(m, k)) for k, _ in m._fields_}

    def index_slots(self) -> int:
        out = C.c_uint64()
        check(lib().dgds_index_slots(self._h, C.byref(out)))
        return int(out.value)

    def update_cst(self, group_id: str, request_id: int, prev_token_count: int, new_tokens: Sequence[int],
                   now: float) -> UpdateReply:
        return self.update_batch([group_id], [request_id], [prev_token_count], [new_tokens], now)[0]

    def update_batch(self, group_ids, request_ids, prev_counts, token_lists, now: float) -> List[UpdateReply]:
        """n update_cst calls in call order (dgds.cpp:36-51)."""
        handles = self.group_handles(group_ids)
        toks = [np.asarray(t, dtype=np.int64) for t in token_lists]
        offs = np.zeros(len(toks) + 1, np.uint64)
        offs[1:] = np.cumsum([len(t) for t in toks]) if toks else []
        flat = np.concatenate(toks).astype(np.int32) if toks and offs[-1] else np.zeros(0, np.int32)
        if any((t < 0).any() or (t > 0x7FFFFFFF).any() for t in toks):
            raise ValueError("negative token")
        rep = self.update_arrays(handles, np.asarray(request_ids, np.int32), np.asarray(prev_counts, np.uint64),
                                 offs, flat, now)
        return [UpdateReply(bool(r["ok"]), int(r["version"]), int(r["acked"])) for r in rep]

    REPLY_DTYPE = np.dtype([("ok", "<i4"), ("pad", "<i4"), ("version", "<u8"), ("acked", "<u8")])

    def update_arrays(self, handles: np.ndarray, request_ids: np.ndarray, prev_counts: np.ndarray,
                      tok_offsets: np.ndarray, tokens: np.ndarray, now: float) -> np.ndarray:
        """Array form of update_batch (host buffers); returns the reply records."""
        n = len(handles)
        handles = np.ascontiguousarray(handles, np.int32)
        request_ids = np.ascontiguousarray(request_ids, np.int32)
        prev_counts = np.ascontiguousarray(prev_counts, np.uint64)
        tok_offsets = np.ascontiguousarray(tok_offsets, np.uint64)
        tokens = np.ascontiguousarray(tokens, np.int32)
        rep = np.zeros(n, self.REPLY_DTYPE)
        check(lib().dgds_update_batch(self._h, n, _ptr(handles), _ptr(request_ids), _ptr(prev_counts),
                                      _ptr(tok_offsets), _ptr(tokens), float(now), _ptr(rep)))
        return rep

    def update_device(self, handles: np.ndarray, request_ids: np.ndarray, prev_counts: np.ndarray,
                      tok_offsets: np.ndarray, d_tokens_ptr: int, now: float, stream: int = 0) -> np.ndarray:
        """Host metadata + device token payload (zero-copy append)."""
        n = len(handles)
        handles = np.ascontiguousarray(handles, np.int32)
        request_ids = np.ascontiguousarray(request_ids, np.int32)
        prev_counts = np.ascontiguousarray(prev_counts, np.uint64)
        tok_offsets = np.ascontiguousarray(tok_offsets, np.uint64)
        rep = np.zeros(n, self.REPLY_DTYPE)
        check(lib().dgds_update_batch_device(self._h, n, _ptr(handles), _ptr(request_ids), _ptr(prev_counts),
                                             _ptr(tok_offsets), C.c_void_p(d_tokens_ptr), float(now), _ptr(rep),
                                             C.c_void_p(stream or None)))
        return rep

    def update_device_strided(self, handles: np.ndarray, request_ids: np.ndarray, prev_counts: np.ndarray,
                              tok_starts: np.ndarray, tok_counts: np.ndarray, d_tokens_ptr: int, now: float,
                              stream: int = 0) -> np.ndarray:
        """Host metadata + device tokens at d_tokens[tok_starts[i] ..+ tok_counts[i]] (routed records)."""
        n = len(handles)
        handles = np.ascontiguousarray(handles, np.int32)
        request_ids = np.ascontiguousarray(request_ids, np.int32)
        prev_counts = np.ascontiguousarray(prev_counts, np.uint64)
        tok_starts = np.ascontiguousarray(tok_starts, np.uint64)
        tok_counts = np.ascontiguousarray(tok_counts, np.uint64)
        rep = np.zeros(n, self.REPLY_DTYPE)
        check(lib().dgds_update_batch_device_strided(self._h, n, _ptr(handles), _ptr(request_ids), _ptr(prev_counts),
                                                     _ptr(tok_starts), _ptr(tok_counts), C.c_void_p(d_tokens_ptr),
                                                     float(now), _ptr(rep), C.c_void_p(stream or None)))
        return rep

    def speculate(self, group_id: str, pattern: Sequence[int], args: SpeculationArgs) -> List[DraftCandidate]:
        """DraftServer::speculate (dgds.cpp:130-138)."""
        return self.speculate_batch([group_id], [pattern], [args])[0]

    def batch_speculate(self, queries: Sequence[SpecQuery], now: float = 0.0) -> List[List[DraftCandidate]]:
        """DraftClient::batch_speculate with fetch_period 0 (dgds.cpp:274-292): fresh, server-side answers."""
        return self.speculate_batch([q.group_id for q in queries], [q.pattern for q in queries],
                                    [q.args for q in queries])

    def speculate_batch(self, group_ids, patterns, args) -> List[List[DraftCandidate]]:
        n = len(group_ids)
        if n == 0:
            return []
        handles = self.group_handles(group_ids)
        pats = [np.asarray(p, dtype=np.int64) for p in patterns]
        offs = np.zeros(n + 1, np.uint64)
        offs[1:] = np.cumsum([len(p) for p in pats])
        flat = (np.concatenate(pats) if offs[-1] else np.zeros(0, np.int64))
        flat = np.clip(flat, -(1 << 31), (1 << 31) - 1).astype(np.int32)
        if isinstance(args, SpeculationArgs):
            arr, stride = args_array([args]), 0
        else:
            arr, stride = args_array(list(args)), 1
        res = self.speculate_arrays(handles, offs, flat, arr, stride)
        return res.to_lists()

    def speculate_arrays(self, handles: np.ndarray, pat_offsets: np.ndarray, patterns: np.ndarray,
                         args: np.ndarray, args_stride: int) -> "CandidateBatch":
        n = len(handles)
        handles = np.ascontiguousarray(handles, np.int32)
        pat_offsets = np.ascontiguousarray(pat_offsets, np.uint64)
        patterns = np.ascontiguousarray(patterns, np.int32)
        args = np.ascontiguousarray(args, ARGS_DTYPE)
        a = args if args_stride else args[:1]
        k = max(1, int(a["top_k"].max())) if len(a) else 1
        s = max(1, int(np.minimum(a["max_spec_tokens"], self.params.max_spec_len).max())) if len(a) else 1
        out = CandidateBatch(n, k, s)
        check(lib().dgds_speculate_batch(self._h, n, _ptr(handles), _ptr(pat_offsets), _ptr(patterns), _ptr(args),
                                         args_stride, C.byref(out.c())))
        return out

    def speculate_view(self, handles: np.ndarray, pat_offsets: np.ndarray, patterns: np.ndarray, args: np.ndarray,
                       args_stride: int, truth: Optional[np.ndarray] = None, truth_left: Optional[np.ndarray] = None,
                       limit: Optional[np.ndarray] = None) -> "ResultView":
        """Batch query (+ fused verification when `truth` is given) returning compact per-query
        candidate lists as zero-copy views of the server's pinned result block
        (dgds_speculate_verify_view) — valid until the second-next host query batch on this server
        (two result slots)."""
        n = len(handles)
        handles = np.ascontiguousarray(handles, np.int32)
        pat_offsets = np.ascontiguousarray(pat_offsets, np.uint64)
        patterns = np.ascontiguousarray(patterns, np.int32)
        args = np.ascontiguousarray(args, ARGS_DTYPE)
        v = _lib.ResultView()
        if truth is not None:
            truth = np.ascontiguousarray(truth, np.int32).reshape(n, -1)
            tl = np.ascontiguousarray(truth_left, np.int32)
            lm = np.ascontiguousarray(limit, np.int32)
            check(lib().dgds_speculate_verify_view(self._h, n, _ptr(handles), _ptr(pat_offsets), _ptr(patterns),
                                                   _ptr(args), args_stride, _ptr(truth), truth.shape[1], _ptr(tl),
                                                   _ptr(lm), C.byref(v)))
        else:
            check(lib().dgds_speculate_verify_view(self._h, n, _ptr(handles), _ptr(pat_offsets), _ptr(patterns),
                                                   _ptr(args), args_stride, None, 0, None, None, C.byref(v)))
        return ResultView(v)

    def speculate_submit(self, handles: np.ndarray, pat_offsets: np.ndarray, patterns: np.ndarray, args: np.ndarray,
                         args_stride: int, truth: Optional[np.ndarray] = None,
                         truth_left: Optional[np.ndarray] = None, limit: Optional[np.ndarray] = None) -> int:
        """Asynchronous speculate_view (dgds_speculate_submit): validates, starts staging and
        returns a ticket for speculate_wait. Two batches can be in flight. The input arrays are
        read asynchronously; this object keeps them alive until the ticket is waited on."""
        n = len(handles)
        handles = np.ascontiguousarray(handles, np.int32)
        pat_offsets = np.ascontiguousarray(pat_offsets, np.uint64)
        patterns = np.ascontiguousarray(patterns, np.int32)
        args = np.ascontiguousarray(args, ARGS_DTYPE)
        t = _lib._U64()
        if truth is not None:
            truth = np.ascontiguousarray(truth, np.int32).reshape(n, -1)
            tl = np.ascontiguousarray(truth_left, np.int32)
            lm = np.ascontiguousarray(limit, np.int32)
            check(lib().dgds_speculate_submit(self._h, n, _ptr(handles), _ptr(pat_offsets), _ptr(patterns),
                                              _ptr(args), args_stride, _ptr(truth), truth.shape[1], _ptr(tl),
                                              _ptr(lm), C.byref(t)))
        else:
            check(lib().dgds_speculate_submit(self._h, n, _ptr(handles), _ptr(pat_offsets), _ptr(patterns),
                                              _ptr(args), args_stride, None, 0, None, None, C.byref(t)))
            tl = lm = None
        tk = int(t.value)
        inflight = self.__dict__.setdefault("_inflight", {})
        for old in [k for k in inflight if k <= tk - 2]:  # their slots are reused: inputs long read
            del inflight[old]
        inflight[tk] = (handles, pat_offsets, patterns, args, truth, tl, lm)
        return tk

    def speculate_wait(self, ticket: int) -> "ResultView":
        """Results of a submitted batch (zero-copy views, valid until two batches later)."""
        v = _lib.ResultView()
        check(lib().dgds_speculate_wait(self._h, ticket, C.byref(v)))
        self.__dict__.get("_inflight", {}).pop(ticket, None)
        return ResultView(v)

    def verify_batch(self, cands: "CandidateBatch", truth: np.ndarray, truth_left: np.ndarray, limit: np.ndarray):
        """Instance::decode_step verification (engine.cpp:115-143) on the GPU."""
        n = cands.n
        truth = np.ascontiguousarray(truth, np.int32).reshape(n, -1)
        tl = np.ascontiguousarray(truth_left, np.int32)
        lm = np.ascontiguousarray(limit, np.int32)
        dr = np.zeros(n, np.int32)
        ac = np.zeros(n, np.int32)
        em = np.zeros(n, np.int32)
        vo = _lib.VerifyOut(_ptr(dr), _ptr(ac), _ptr(em))
        check(lib().dgds_verify_batch(self._h, n, C.byref(cands.c()), _ptr(truth), truth.shape[1], _ptr(tl), _ptr(lm),
                                      C.byref(vo)))
        return dr, ac, em


CAND_META_DTYPE = np.dtype([("score", np.float64), ("support", np.int64), ("len", np.int32),
                            ("reserved", np.int32)])


def _as_np(ptr: Optional[int], n: int, ctype, dtype=None) -> Optional[np.ndarray]:
    if not ptr:
        return None if dtype is None and ctype is None else np.zeros(0, dtype or np.int32)
    a = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(n,))
    return a.view(dtype) if dtype is not None else a


class ResultView:
    """dgds_result_view as numpy arrays over the server's pinned block (no copy).
    candidates of query q: cands[cand_off[q]:cand_off[q + 1]]; tokens of candidate c:
    tokens[tok_off[c]:tok_off[c + 1]]."""

    def __init__(self, v: _lib.ResultView):
        n, m, t = v.n_queries, v.n_cands, v.n_tokens
        self.n = n
        self.cand_off = _as_np(v.cand_off, n + 1, C.c_int64) if n else np.zeros(1, np.int64)
        raw = _as_np(v.cands, m * CAND_META_DTYPE.itemsize, C.c_uint8) if m else np.zeros(0, np.uint8)
        self.cands = raw.view(CAND_META_DTYPE)
        self.tok_off = _as_np(v.tok_off, m + 1, C.c_int64) if n else np.zeros(1, np.int64)
        self.tokens = _as_np(v.tokens, t, C.c_int32) if t else np.zeros(0, np.int32)
        self.drafted = _as_np(v.drafted, n, C.c_int32) if v.drafted else None
        self.accepted = _as_np(v.accepted, n, C.c_int32) if v.accepted else None
        self.emitted = _as_np(v.emitted, n, C.c_int32) if v.emitted else None

    def candidates(self, q: int) -> List[DraftCandidate]:
        out = []
        for c in range(int(self.cand_off[q]), int(self.cand_off[q + 1])):
            toks = tuple(int(x) for x in self.tokens[self.tok_off[c]:self.tok_off[c + 1]])
            out.append(DraftCandidate(toks, float(self.cands["score"][c]), int(self.cands["support"][c])))
        return out


class CandidateBatch:
    """Caller-owned candidate buffers (dgds_candidates)."""

    def __init__(self, n: int, k_stride: int, s_stride: int):
        self.n, self.k, self.s = n, k_stride, s_stride
        self.n_cands = np.zeros(n, np.int32)
        self.lens = np.zeros(n * k_stride, np.int32)
        self.scores = np.zeros(n * k_stride, np.float64)
        self.supports = np.zeros(n * k_stride, np.int64)
        self.tokens = np.zeros(n * k_stride * s_stride, np.int32)
        self._c = None

    def c(self) -> _lib.Candidates:
        if self._c is None:
            self._c = _lib.Candidates(self.k, self.s, _ptr(self.n_cands), _ptr(self.lens), _ptr(self.scores),
                                      _ptr(self.supports), _ptr(self.tokens))
        return self._c

    def query(self, q: int) -> List[DraftCandidate]:
        res = []
        for c in range(int(self.n_cands[q])):
            i = q * self.k + c
            L = int(self.lens[i])
            t = self.tokens[i * self.s:i * self.s + L]
            res.append(DraftCandidate(tuple(int(x) for x in t), float(self.scores[i]), int(self.supports[i])))
        return res

    def to_lists(self) -> List[List[DraftCandidate]]:
        return [self.query(q) for q in range(self.n)]


class DraftCluster:
    """N GPUs behind one draft server (dgds_cluster_*): group g lives on GPU fnv1a64(g) % n, the
    reference's shard_of_group (dgds.cpp:10-14); batch calls split by owner and run the GPUs
    concurrently, returning results in call order."""

    def __init__(self, params: Optional[DgdsParams] = None, devices: Sequence[int] = (0,), expected_nodes: int = 0,
                 expected_streams: int = 0):
        self.params = params or DgdsParams()
        p = self.params
        cp = _lib.Params(p.shard_count, p.append_batch_tokens, p.fetch_period, p.default_ttl_seconds,
                         p.max_pattern_len, p.max_spec_len, 0, 0, expected_nodes, expected_streams)
        devs = (C.c_int32 * len(devices))(*devices)
        h = C.c_void_p()
        check(lib().dgds_cluster_create(C.byref(cp), len(devices), devs, C.byref(h)))
        self._h = h
        self._handles = {}

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().dgds_cluster_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def size(self) -> int:
        return int(lib().dgds_cluster_size(self._h))

    def group_handles(self, group_ids: Iterable[str]) -> np.ndarray:
        out = []
        for g in group_ids:
            h = self._handles.get(g)
            if h is None:
                v = C.c_int32()
                b = g.encode()
                check(lib().dgds_cluster_intern(self._h, b, len(b), C.byref(v)))
                h = self._handles[g] = v.value
            out.append(h)
        return np.asarray(out, np.int32)

    def owner(self, group_id: str) -> int:
        v = C.c_int32()
        check(lib().dgds_cluster_owner(self._h, int(self.group_handles([group_id])[0]), C.byref(v)))
        return v.value

    def update_batch(self, group_ids, request_ids, prev_counts, token_lists, now: float) -> List[UpdateReply]:
        n = len(group_ids)
        if n == 0:
            return []
        handles = self.group_handles(group_ids)
        toks = [np.asarray(t, dtype=np.int64) for t in token_lists]
        offs = np.zeros(n + 1, np.uint64)
        offs[1:] = np.cumsum([len(t) for t in toks])
        flat = np.concatenate(toks).astype(np.int32) if offs[-1] else np.zeros(0, np.int32)
        rids = np.ascontiguousarray(request_ids, np.int32)
        prev = np.ascontiguousarray(prev_counts, np.uint64)
        rep = np.zeros(n, DraftServer.REPLY_DTYPE)
        check(lib().dgds_cluster_update_batch(self._h, n, _ptr(handles), _ptr(rids), _ptr(prev), _ptr(offs),
                                              _ptr(flat), float(now), _ptr(rep)))
        return [UpdateReply(bool(r["ok"]), int(r["version"]), int(r["acked"])) for r in rep]

    def speculate_batch(self, group_ids, patterns, args) -> List[List[DraftCandidate]]:
        n = len(group_ids)
        if n == 0:
            return []
        handles = self.group_handles(group_ids)
        pats = [np.asarray(p, dtype=np.int64) for p in patterns]
        offs = np.zeros(n + 1, np.uint64)
        offs[1:] = np.cumsum([len(p) for p in pats])
        flat = (np.concatenate(pats) if offs[-1] else np.zeros(0, np.int64)).astype(np.int32)
        if isinstance(args, SpeculationArgs):
            arr, stride = args_array([args]), 0
        else:
            arr, stride = args_array(list(args)), 1
        a = arr if stride else arr[:1]
        k = max(1, int(a["top_k"].max()))
        s = max(1, int(np.minimum(a["max_spec_tokens"], self.params.max_spec_len).max()))
        out = CandidateBatch(n, k, s)
        check(lib().dgds_cluster_speculate_verify_batch(self._h, n, _ptr(handles), _ptr(offs), _ptr(flat), _ptr(arr),
                                                        stride, None, 0, None, None, C.byref(out.c()), None))
        return out.to_lists()

    def node_count(self) -> int:
        out = C.c_uint64()
        check(lib().dgds_cluster_node_count(self._h, C.byref(out)))
        return int(out.value)

    def group_version(self, group_id: str) -> int:
        out = C.c_uint64()
        check(lib().dgds_cluster_group_version(self._h, int(self.group_handles([group_id])[0]), C.byref(out)))
        return int(out.value)
