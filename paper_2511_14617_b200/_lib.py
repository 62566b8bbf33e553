"""ctypes binding of libdgds_b200.so (the C ABI in include/dgds_b200.h).

The library is the only implementation: if it is missing or no CUDA device is
present, the calls fail loudly — there is no CPU fallback path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DGDS_LIB_VARIANT=<name> loads a test-only build variant (build.py VARIANTS), e.g. hash10
LIB_PATH = os.path.join(HERE, "libdgds_b200%s.so" % ("_" + os.environ["DGDS_LIB_VARIANT"]
                                                       if os.environ.get("DGDS_LIB_VARIANT") else ""))

DGDS_OK = 0
DGDS_EINVAL = -1
DGDS_ECUDA = -2
DGDS_ENOMEM = -3
DGDS_EUNSUPPORTED = -4
DGDS_EBUFFER = -5
DGDS_ESTATE = -6
DGDS_EBLOB = -7
MAX_DEPTH = 32
MAX_TOP_K = 32


class Params(C.Structure):
    _fields_ = [
        ("shard_count", C.c_int32),
        ("append_batch_tokens", C.c_int32),
        ("fetch_period", C.c_double),
        ("default_ttl_seconds", C.c_double),
        ("max_pattern_len", C.c_int32),
        ("max_spec_len", C.c_int32),
        ("device", C.c_int32),
        ("reserved0", C.c_int32),
        ("expected_nodes", C.c_uint64),
        ("expected_streams", C.c_uint64),
    ]


class SpecArgs(C.Structure):
    _fields_ = [
        ("max_spec_tokens", C.c_int32),
        ("pattern_lookup_max", C.c_int32),
        ("pattern_lookup_min", C.c_int32),
        ("top_k", C.c_int32),
        ("min_step_freq", C.c_double),
        ("min_support", C.c_int64),
    ]


class UpdateReplyC(C.Structure):
    _fields_ = [("ok", C.c_int32), ("reserved0", C.c_int32), ("version", C.c_uint64), ("acked_tokens", C.c_uint64)]


class Candidates(C.Structure):
    _fields_ = [
        ("k_stride", C.c_int32),
        ("s_stride", C.c_int32),
        ("n_cands", C.c_void_p),
        ("lens", C.c_void_p),
        ("scores", C.c_void_p),
        ("supports", C.c_void_p),
        ("tokens", C.c_void_p),
    ]


class SpecPolicy(C.Structure):  # dgds_spec_policy (AdaptiveSpecPolicy, engine.hpp:28-33)
    _fields_ = [("sd_enabled", C.c_int32), ("adaptive", C.c_int32), ("batch_token_budget", C.c_int32),
                ("per_request_cap", C.c_int32), ("multi_path_k", C.c_int32), ("feedback", C.c_int32)]


class VerifyOut(C.Structure):
    _fields_ = [("drafted", C.c_void_p), ("accepted", C.c_void_p), ("emitted", C.c_void_p)]


class ResultView(C.Structure):
    _fields_ = [("n_queries", C.c_int64), ("n_cands", C.c_int64), ("n_tokens", C.c_int64),
                ("cand_off", C.c_void_p), ("cands", C.c_void_p), ("tok_off", C.c_void_p), ("tokens", C.c_void_p),
                ("drafted", C.c_void_p), ("accepted", C.c_void_p), ("emitted", C.c_void_p)]


class FetchReply(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("version", C.c_uint64), ("blob_off", C.c_uint64),
                ("blob_len", C.c_uint64)]


class MemoryStats(C.Structure):
    _fields_ = [("slots", C.c_uint64), ("used_slots", C.c_uint64), ("history_capacity", C.c_uint64),
                ("history_tokens", C.c_uint64), ("dead_history_tokens", C.c_uint64), ("compactions", C.c_uint64)]


class QueryStats(C.Structure):
    _fields_ = [
        ("queries", C.c_uint64),
        ("pattern_tokens", C.c_uint64),
        ("suffix_lookups", C.c_uint64),
        ("expansions", C.c_uint64),
        ("child_sectors", C.c_uint64),
        ("cands", C.c_uint64),
        ("cand_tokens", C.c_uint64),
        ("algorithmic_bytes", C.c_uint64),
    ]


class PxChannelDesc(C.Structure):  # dgds_px_channel_desc
    _fields_ = [("rows", C.c_int32), ("words", C.c_int32), ("shared", C.c_int32), ("pad", C.c_int32),
                ("flag_off", C.c_uint64), ("count_off", C.c_uint64 * 2), ("slab_off", C.c_uint64 * 2)]


class PxTick(C.Structure):  # dgds_px_tick
    _fields_ = [("n_q", C.c_int64), ("n_a", C.c_int64), ("q_owner", C.c_void_p), ("q", C.c_void_p),
                ("a_owner", C.c_void_p), ("a", C.c_void_p)]


class RecordLayout(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("rec_words", "off_handle", "off_pat_len", "off_pattern", "off_truth_left",
                                         "off_limit", "off_truth", "reply_words", "off_n_cands", "off_lens",
                                         "off_scores", "off_supports", "off_tokens", "off_verify")]


class Profile(C.Structure):
    _fields_ = [("append_launches", C.c_uint64), ("query_launches", C.c_uint64), ("append_ms", C.c_double),
                ("query_ms", C.c_double)]


class WorkloadCfg(C.Structure):
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
        ("reserved0", C.c_int32),
        ("seed", C.c_uint64),
    ]


class DgdsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"dgds error {code}: {msg}")
        self.code = code


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_U64 = C.c_uint64
_D = C.c_double

EXPORTS = {
    "dgds_last_error": (C.c_char_p, []),
    "dgds_version_string": (C.c_char_p, []),
    "dgds_fnv1a64": (_U64, [_P, C.c_size_t]),
    "dgds_shard_of_group": (_I32, [C.c_char_p, C.c_size_t, _I32]),
    "dgds_create": (C.c_int, [C.POINTER(Params), C.POINTER(_P)]),
    "dgds_destroy": (C.c_int, [_P]),
    "dgds_cuda_stream": (_P, [_P]),
    "dgds_intern": (C.c_int, [_P, C.c_char_p, C.c_size_t, C.POINTER(_I32)]),
    "dgds_register_group": (C.c_int, [_P, _I32, _D, _D]),
    "dgds_drop_group": (C.c_int, [_P, _I32]),
    "dgds_sweep_expired": (C.c_int, [_P, _D]),
    "dgds_has_group": (C.c_int, [_P, _I32, C.POINTER(_I32)]),
    "dgds_group_version": (C.c_int, [_P, _I32, C.POINTER(_U64)]),
    "dgds_stored_tokens": (C.c_int, [_P, _I32, _I32, C.POINTER(_U64)]),
    "dgds_shard_group_count": (C.c_int, [_P, _I32, C.POINTER(_U64)]),
    "dgds_node_count": (C.c_int, [_P, C.POINTER(_U64)]),
    "dgds_entry_count": (C.c_int, [_P, C.POINTER(_U64)]),
    "dgds_device_error": (C.c_int, [_P, C.POINTER(C.c_int32)]),
    "dgds_index_slots": (C.c_int, [_P, C.POINTER(_U64)]),
    "dgds_update_batch": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P, _D, _P]),
    "dgds_update_batch_device": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P, _D, _P, _P]),
    "dgds_update_batch_device_strided": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P, _P, _D, _P, _P]),
    "dgds_speculate_batch": (C.c_int, [_P, _I64, _P, _P, _P, _P, _I64, C.POINTER(Candidates)]),
    "dgds_cluster_create": (C.c_int, [_P, C.c_int32, _P, C.POINTER(_P)]),
    "dgds_cluster_destroy": (C.c_int, [_P]),
    "dgds_cluster_size": (C.c_int32, [_P]),
    "dgds_cluster_server": (_P, [_P, C.c_int32]),
    "dgds_cluster_intern": (C.c_int, [_P, C.c_char_p, C.c_size_t, C.POINTER(C.c_int32)]),
    "dgds_cluster_owner": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int32)]),
    "dgds_cluster_register_group": (C.c_int, [_P, C.c_int32, C.c_double, C.c_double]),
    "dgds_cluster_drop_group": (C.c_int, [_P, C.c_int32]),
    "dgds_cluster_sweep_expired": (C.c_int, [_P, C.c_double]),
    "dgds_cluster_has_group": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int32)]),
    "dgds_cluster_group_version": (C.c_int, [_P, C.c_int32, C.POINTER(_U64)]),
    "dgds_cluster_stored_tokens": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(_U64)]),
    "dgds_cluster_shard_group_count": (C.c_int, [_P, C.c_int32, C.POINTER(_U64)]),
    "dgds_cluster_node_count": (C.c_int, [_P, C.POINTER(_U64)]),
    "dgds_cluster_update_batch": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P, C.c_double, _P]),
    "dgds_cluster_speculate_verify_batch": (C.c_int, [_P, _I64, _P, _P, _P, _P, _I64, _P, _I32, _P, _P,
                                                      C.POINTER(Candidates), _P]),
    "dgds_decode_step_device": (C.c_int, [_P, _I64, _P, _P, _I32, _P, _P, _P, _I32, _P, C.POINTER(SpecArgs),
                                          C.POINTER(SpecPolicy), _P, _I32, C.POINTER(Candidates),
                                          C.POINTER(VerifyOut), _P, _P, _P]),
    "dgds_speculate_device": (C.c_int, [_P, _I64, _P, _P, _P, _I32, _P, _I64, _I32, _I32, C.POINTER(Candidates), _P,
                                        _I32,
                                        _P, _P, C.POINTER(VerifyOut), _P, _P]),
    "dgds_speculate_verify_batch": (C.c_int, [_P, _I64, _P, _P, _P, _P, _I64, _P, _I32, _P, _P,
                                              C.POINTER(Candidates), C.POINTER(VerifyOut)]),
    "dgds_profile_enable": (C.c_int, [_P, _I32]),
    "dgds_last_transfer": (C.c_int, [_P, C.POINTER(_U64)]),
    "dgds_debug_query_timing": (C.c_int, [_P, _P]),
    "dgds_profile_read": (C.c_int, [_P, C.POINTER(Profile), _I32]),
    "dgds_verify_batch": (C.c_int, [_P, _I64, C.POINTER(Candidates), _P, _I32, _P, _P, C.POINTER(VerifyOut)]),
    "dgds_draft_len": (_I32, [_I32, _I32, _I32, _I32, _I32]),
    "dgds_route_pack": (C.c_int, [_I64, _I32, _P, _P, _I32, _P, _P, _P, _P]),
    "dgds_route_unpack": (C.c_int, [_I64, _P, _I32, _P, _P, _P]),
    "dgds_route_pack_padded": (C.c_int, [_I64, _I32, _P, _P, _I32, _I64, _P, _P, _P, _P]),
    "dgds_speculate_records": (C.c_int, [_P, _I64, _P, C.POINTER(RecordLayout), _P, _I64, _I32, _I32, _P, _P, _P]),
    "dgds_batch_speculate_zc": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P, _P, C.POINTER(RecordLayout), _P, _I64, _I32,
                                          _I32, _P, _P]),
    "dgds_debug_append_timing": (C.c_int, [_P, _P, _I64]),
    "dgds_debug_dump": (C.c_int, [_P, C.c_int32, _P, _U64]),
    "dgds_compact_memory": (C.c_int, [_P]),
    "dgds_get_memory_stats": (C.c_int, [_P, C.POINTER(MemoryStats)]),
    "dgds_touch_group": (C.c_int, [_P, _I32, C.c_double]),
    "dgds_wire_serve_payload": (C.c_int, [_P, _P, _U64, C.c_double, _P, _U64, C.POINTER(_U64)]),
    "dgds_wire_service_start": (C.c_int, [_P, _I32, C.POINTER(C.c_void_p), C.POINTER(_I32)]),
    "dgds_wire_service_stats": (C.c_int, [_P, C.POINTER(_U64), C.POINTER(_U64)]),
    "dgds_wire_service_stop": (C.c_int, [_P]),
    "dgds_fetch_cst": (C.c_int, [_P, _I64, _P, _P, C.c_double, C.POINTER(FetchReply), C.POINTER(C.c_void_p)]),
    "dgds_compact_group": (C.c_int, [_P, _I32, _U64]),
    "dgds_apply_blob": (C.c_int, [_P, _I32, _P, _U64, C.c_double, C.POINTER(_U64)]),
    "dgds_update_batch_routed": (C.c_int, [_P, _I32, _I64, _P, _P, _I32, _P, _I32, C.c_double, C.POINTER(_I64),
                                           _P]),
    "dgds_update_plan_routed": (C.c_int, [_P, _I32, _I64, _P, _P, _I32, _P, _I32, C.c_double, C.POINTER(_I64),
                                          C.POINTER(C.c_void_p)]),
    "dgds_update_launch": (C.c_int, [_P, _P, _P]),
    "dgds_update_plan_routed_async": (C.c_int, [_P, _P, _I32, _I64, _P, _P, _I32, _P, _I32, C.c_double,
                                                C.POINTER(_U64)]),
    "dgds_update_plan_take": (C.c_int, [_P, _U64, C.POINTER(_I64), C.POINTER(_P)]),
    "dgds_copy_rows_d2h": (C.c_int, [_P, _I64, _P, _I64, _I64, _I64, _P]),
    "dgds_speculate_verify_view": (C.c_int, [_P, _I64, _P, _P, _P, _P, _I64, _P, _I32, _P, _P, C.POINTER(ResultView)]),
    "dgds_speculate_submit": (C.c_int, [_P, _I64, _P, _P, _P, _P, _I64, _P, _I32, _P, _P, C.POINTER(_U64)]),
    "dgds_speculate_wait": (C.c_int, [_P, _U64, C.POINTER(ResultView)]),
    "dgds_replies_submit": (C.c_int, [_P, _I64, _P, C.POINTER(RecordLayout), _I32, _I32, _P, C.POINTER(_U64)]),
    "dgds_speculate_records_seg": (C.c_int, [_P, _I32, _I64, _P, _P, C.POINTER(RecordLayout), _P, _I64, _I32, _I32,
                                             C.POINTER(C.c_void_p), _I32, _P, _P]),
    "dgds_px_create": (C.c_int, [_I32, _I32, _I32, _U64, C.POINTER(C.c_void_p), _P]),
    "dgds_px_connect": (C.c_int, [_P, _P]),
    "dgds_px_connect_local": (C.c_int, [C.POINTER(C.c_void_p), _I32]),
    "dgds_px_region": (C.c_int, [_P, _I32, C.POINTER(C.c_void_p)]),
    "dgds_px_send": (C.c_int, [_P, _I64, _P, _P, _I32, _I64, _U64, _U64, _U64, _U64, _I32, _I32, _P, _P, _P]),
    "dgds_px_wait": (C.c_int, [_P, _U64, _U64, _P]),
    "dgds_px_signal": (C.c_int, [_P, _U64, _U64, _P]),
    "dgds_px_status": (C.c_int, [_P, C.POINTER(_I32), C.POINTER(_U64)]),
    "dgds_px_set_timeout": (C.c_int, [_P, _U64]),
    "dgds_px_destroy": (C.c_int, [_P]),
    "dgds_kernel_launches": (_U64, []),
    "dgds_px_driver_create": (C.c_int, [_P, _P, _I32, _I32, _P, _P, _P, _I32, _P, _P, _I32, _I32, _P, _P, _I64, _P,
                                        C.POINTER(C.c_void_p)]),
    "dgds_px_driver_run": (C.c_int, [_P, _I64, _I64, _I64, _P]),
    "dgds_px_driver_destroy": (C.c_int, [_P]),
}

_lib = None


def lib():
    """Load libdgds_b200.so (building it first if this checkout has nvcc and no .so)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from . import build as _b

            _b.build(variant=os.environ.get("DGDS_LIB_VARIANT") or None)
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc == DGDS_OK:
        return
    msg = lib().dgds_last_error().decode(errors="replace")
    if rc == DGDS_EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    raise DgdsError(rc, msg)
