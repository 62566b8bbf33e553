"""Owner routing of draft-server traffic across GPUs (one process per GPU).

Groups are owned by ``fnv1a64(group_id) % world`` — the reference's own
``shard_of_group`` (proj/src/dgds.cpp:10-14). A rank's append records and
draft queries go to the owning rank with an all-to-all over NCCL
(``torch.distributed``): the fixed-size records are bucketed by owner
(``dgds_route_pack``, stable), the per-owner counts are exchanged, then the
payloads; replies come back through the inverse all-to-all and are scattered
into the original order (``dgds_route_unpack``).

``Router`` is backend-agnostic: with CUDA tensors it uses the sm_100a
pack/unpack kernels; the CPU/gloo tests inject a host packer to check the
exchange protocol itself.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist

from . import _lib


def cuda_pack(owner: torch.Tensor, records: torch.Tensor, world: int) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Stable bucketing of [n, w] int32 records by owner on the GPU (k_route_*)."""
    n, w = records.shape
    out = torch.empty_like(records)
    counts = torch.empty(world, dtype=torch.int64, device=records.device)
    perm = torch.empty(n, dtype=torch.int64, device=records.device)
    stream = torch.cuda.current_stream(records.device).cuda_stream
    _lib.check(_lib.lib().dgds_route_pack(n, world, C.c_void_p(owner.data_ptr()), C.c_void_p(records.data_ptr()), w,
                                          C.c_void_p(out.data_ptr()), C.c_void_p(counts.data_ptr()),
                                          C.c_void_p(perm.data_ptr()), C.c_void_p(stream)))
    return out, counts, perm


def cuda_unpack(packed: torch.Tensor, perm: torch.Tensor) -> torch.Tensor:
    """out[i] = packed[perm[i]] for i < len(perm), on the GPU (k_route_gather)."""
    n, w = perm.shape[0], packed.shape[1]
    out = torch.empty((n, w), dtype=packed.dtype, device=packed.device)
    stream = torch.cuda.current_stream(packed.device).cuda_stream
    _lib.check(_lib.lib().dgds_route_unpack(n, C.c_void_p(packed.data_ptr()), w, C.c_void_p(perm.data_ptr()),
                                            C.c_void_p(out.data_ptr()), C.c_void_p(stream)))
    return out


class Router:
    """One exchange round: records of every rank -> their owners -> replies back."""

    def __init__(self, world: int, group=None, pack: Optional[Callable] = None, unpack: Optional[Callable] = None):
        self.world = world
        self.group = group
        self.pack = pack or cuda_pack
        self.unpack = unpack or cuda_unpack

    def forward(self, owner: torch.Tensor, records: torch.Tensor):
        """Send record i to rank owner[i]. Returns (received [m, w], state for `reverse`)."""
        packed, counts, perm = self.pack(owner, records, self.world)
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts, group=self.group)
        send_splits = counts.tolist()
        recv_splits = recv_counts.tolist()
        received = records.new_empty((sum(recv_splits), records.shape[1]))
        dist.all_to_all_single(received, packed, recv_splits, send_splits, group=self.group)
        return received, (perm, send_splits, recv_splits)

    def reverse(self, replies: torch.Tensor, state) -> torch.Tensor:
        """Return one reply row per received record to its sender, in the sender's original order."""
        perm, send_splits, recv_splits = state
        back = replies.new_empty((sum(send_splits), replies.shape[1]))
        dist.all_to_all_single(back, replies.contiguous(), send_splits, recv_splits, group=self.group)
        return self.unpack(back, perm)


def cuda_pack_padded(owner: torch.Tensor, records: torch.Tensor, world: int, cap: int):
    """Stable bucketing straight into the fixed-capacity send layout (k_route_*_padded):
    returns ([world*cap, w] with empty rows = -1, slot row of each record, overflow flag)."""
    n, w = records.shape
    out = torch.empty((world * cap, w), dtype=records.dtype, device=records.device)
    slot = torch.empty(n, dtype=torch.int64, device=records.device)
    overflow = torch.zeros(1, dtype=torch.int32, device=records.device)
    stream = torch.cuda.current_stream(records.device).cuda_stream
    _lib.check(_lib.lib().dgds_route_pack_padded(n, world, C.c_void_p(owner.data_ptr()),
                                                 C.c_void_p(records.data_ptr()), w, cap, C.c_void_p(out.data_ptr()),
                                                 C.c_void_p(slot.data_ptr()), C.c_void_p(overflow.data_ptr()),
                                                 C.c_void_p(stream)))
    return out, slot, overflow


class PaddedRouter:
    """Fixed-capacity exchange: every rank sends `cap` rows to every rank, so the
    split sizes are static and no host synchronisation is needed. Empty rows are
    -1 (an invalid group handle: the query kernel answers it with nothing, the
    append path skips it). Overflow (> cap records for one owner) is reported as
    a device flag."""

    def __init__(self, world: int, group=None, pack_padded: Optional[Callable] = None,
                 unpack: Optional[Callable] = None):
        self.world = world
        self.group = group
        self.pack_padded = pack_padded or cuda_pack_padded
        self.unpack = unpack or cuda_unpack

    def forward(self, owner: torch.Tensor, records: torch.Tensor, cap: int):
        send, slot, overflow = self.pack_padded(owner, records, self.world, cap)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=self.group)
        return recv, (slot, overflow)

    def reverse(self, replies: torch.Tensor, state):
        slot, overflow = state
        back = torch.empty_like(replies)
        dist.all_to_all_single(back, replies.contiguous(), group=self.group)
        return self.unpack(back, slot), overflow
