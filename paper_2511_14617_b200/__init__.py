"""B200-native Distributed Grouped Draft Server (Seer, arXiv 2511.14617) hot path.

Per-prompt-group counted suffix index on the GPU: batched append, batched
multi-path draft query and fused verification, behind the reference
draft-server interface. See DESIGN.md and include/dgds_b200.h.
"""
from .dgds import (DgdsParams, DraftCandidate, DraftServer, SpecQuery, SpeculationArgs, UpdateReply, draft_len,
                   fnv1a64, shard_of_group)
from .workload import CONFIGS, WorkloadConfig, generate_workload

__all__ = ["DgdsParams", "DraftCandidate", "DraftServer", "SpecQuery", "SpeculationArgs", "UpdateReply", "draft_len",
           "fnv1a64", "shard_of_group", "CONFIGS", "WorkloadConfig", "generate_workload"]
