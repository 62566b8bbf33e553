"""Synthetic grouped-rollout traces (generate_workload, proj/src/workload.cpp:51-103).

Generated natively by a tools library (tools/workload/workload_gen.cpp -> libdgds_workload.so,
separate from the draft-server library) so the GPU box can build the exact reference inputs
without the reference. The config table is BASELINE.md §3.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, asdict

import numpy as np

import os

from . import _lib

_WL = None


def lib():
    """tools/workload/libdgds_workload.so (built with the library by build.py)."""
    global _WL
    if _WL is None:
        from . import build as _b
        path = _b.WORKLOAD_LIB
        if not os.path.exists(path):
            _b.build_workload()
        L = C.CDLL(path)
        L.dgds_generate_workload.restype = C.c_int
        L.dgds_generate_workload.argtypes = [C.POINTER(_lib.WorkloadCfg), C.c_void_p, C.c_void_p, C.c_void_p]
        _WL = L
    return _WL


def _check(rc):
    if rc != 0:
        raise ValueError("invalid workload configuration")


@dataclass(frozen=True)
class WorkloadConfig:
    """rollsim::WorkloadConfig + LengthModel + PromptLenModel (workload.hpp:19-41)."""

    num_groups: int = 16
    group_size: int = 8
    length_family: int = 0  # 0 lognormal, 1 pareto
    location: float = 1000.0
    scale: float = 1.0
    group_correlation: float = 0.9
    noise_base: float = 0.5
    pattern_similarity: float = 0.5
    vocab_size: int = 50000
    max_tokens: int = 8192
    prompt_mean: float = 512.0
    prompt_spread: float = 128.0
    seed: int = 0

    def c(self) -> _lib.WorkloadCfg:
        return _lib.WorkloadCfg(self.num_groups, self.group_size, self.length_family, self.vocab_size,
                                self.location, self.scale, self.group_correlation, self.noise_base,
                                self.pattern_similarity, self.prompt_mean, self.prompt_spread, self.max_tokens, 0,
                                self.seed)


# BASELINE.md §3 / SURVEY.md §8(d): seed 7, rho_pat 0.8.
CONFIGS = {
    "C1": WorkloadConfig(num_groups=1, group_size=16, location=4096.0, scale=0.0, group_correlation=1.0,
                         pattern_similarity=0.8, vocab_size=32000, max_tokens=4096, seed=7),
    "C2": WorkloadConfig(num_groups=256, group_size=16, location=8192.0, scale=0.8, group_correlation=0.9,
                         pattern_similarity=0.8, vocab_size=163840, max_tokens=32768, seed=7),
    "C3": WorkloadConfig(num_groups=128, group_size=8, location=8192.0, scale=0.6, group_correlation=0.9,
                         pattern_similarity=0.8, vocab_size=152064, max_tokens=16384, seed=7),
    "C4": WorkloadConfig(num_groups=512, group_size=16, location=16384.0, scale=0.8, group_correlation=0.9,
                         pattern_similarity=0.8, vocab_size=163840, max_tokens=65536, seed=7),
}
CONFIG_TOTAL_TOKENS = {"C1": 65536, "C2": 43_694_591, "C3": 9_029_385, "C4": 167_396_311}


def group_id(g: int) -> str:
    return "g%05d" % g  # workload.cpp:61-63


class Trace:
    """Flattened trace: stream s = g*group_size + i holds tokens[offsets[s]:offsets[s+1]]."""

    def __init__(self, cfg: WorkloadConfig, lengths, prompt_lens, tokens):
        self.cfg = cfg
        self.lengths = lengths
        self.prompt_lens = prompt_lens
        self.tokens = tokens
        self.offsets = np.zeros(len(lengths) + 1, np.int64)
        np.cumsum(lengths, out=self.offsets[1:])

    @property
    def num_streams(self):
        return len(self.lengths)

    def stream(self, s: int) -> np.ndarray:
        return self.tokens[self.offsets[s]:self.offsets[s + 1]]

    def group_ids(self):
        return [group_id(g) for g in range(self.cfg.num_groups)]


def lengths_only(cfg: WorkloadConfig):
    n = cfg.num_groups * cfg.group_size
    lengths = np.zeros(n, np.int64)
    plens = np.zeros(cfg.num_groups, np.int32)
    c = cfg.c()
    _check(lib().dgds_generate_workload(C.byref(c), lengths.ctypes.data_as(C.c_void_p),
                                            plens.ctypes.data_as(C.c_void_p), None))
    return lengths, plens


def generate_workload(cfg: WorkloadConfig) -> Trace:
    lengths, plens = lengths_only(cfg)
    tokens = np.zeros(int(lengths.sum()), np.int32)
    c = cfg.c()
    _check(lib().dgds_generate_workload(C.byref(c), lengths.ctypes.data_as(C.c_void_p),
                                            plens.ctypes.data_as(C.c_void_p), tokens.ctypes.data_as(C.c_void_p)))
    return Trace(cfg, lengths, plens, tokens)
