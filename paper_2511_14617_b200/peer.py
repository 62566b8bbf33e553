"""Owner routing over NVLink peer memory (one process per GPU) — no collectives.

The reference routes a group's traffic to shard ``fnv1a64(gid) % N``
(proj/src/dgds.cpp:10-14). Here each rank owns one device region that every
other rank maps through CUDA IPC (``dgds_px_*`` in include/dgds_b200.h). A
*channel* is a double-buffered slab per receiver, ``[parity][sender][rows][words]``
int32, plus per-sender counts and a monotone sequence flag:

- ``send``  scatters records into their owners' slabs (stores over NVLink) and
  publishes counts + ``flag = seq`` (k_px_send_*);
- ``wait``  makes later kernels on the stream see every sender's exchange ``seq``;
- ``signal`` publishes ``flag = seq`` after kernels that wrote into peers' slabs
  (the query kernel writes its reply records straight into the sender's reply
  slab, ``dgds_speculate_records_seg``).

Parity ``seq % 2`` selects the slab; a sender may rewrite a parity only after a
round trip proves the receiver finished reading it (bench_multi.py keeps that
order).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import torch

from . import _lib

_ALIGN = 256


class _DevArray:
    """__cuda_array_interface__ wrapper: a torch view of raw device memory."""

    def __init__(self, ptr: int, shape: Tuple[int, ...], typestr: str):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def _view(ptr: int, shape: Tuple[int, ...], typestr: str, device: torch.device) -> torch.Tensor:
    return torch.as_tensor(_DevArray(ptr, shape, typestr), device=device)


@dataclass
class Channel:
    name: str
    rows: int            # rows per sender in one slab (shared: rows of the whole slab)
    words: int           # int32 words per row
    flag_off: int
    count_off: Tuple[int, int]
    slab_off: Tuple[int, int]
    shared: bool = False  # one [rows][words] slab that every sender addresses by row


def _layout(world: int, spec: Dict[str, tuple]) -> Tuple[Dict[str, Channel], int]:
    off = 0
    chans = {}
    heads = {}
    for name in spec:  # headers first: flags (8 B per sender) and two parities of counts
        flag = off
        off += 8 * world
        c0 = off
        off += 4 * world
        c1 = off
        off += 4 * world
        off = (off + 63) // 64 * 64
        heads[name] = (flag, (c0, c1))
    off = (off + _ALIGN - 1) // _ALIGN * _ALIGN
    for name, sp in spec.items():
        rows, words = sp[0], sp[1]
        shared = len(sp) > 2 and sp[2] == "shared"
        slabs = []
        for _ in range(2):
            slabs.append(off)
            off += ((1 if shared else world) * rows * words * 4 + _ALIGN - 1) // _ALIGN * _ALIGN
        chans[name] = Channel(name, rows, words, heads[name][0], heads[name][1], (slabs[0], slabs[1]), shared)
    return chans, off


class PeerExchange:
    """One rank's end of the NVLink exchange. ``channels`` maps name -> (rows per sender, words)
    or (rows, words, "shared") for a slab that senders address by row (replies in query order)."""

    def __init__(self, world: int, rank: int, device: int, channels: Dict[str, Tuple[int, int]], group=None,
                 connect: bool = True):
        self.world, self.rank = world, rank
        self.device = torch.device("cuda", device)
        self.ch, self.bytes = _layout(world, channels)
        L = _lib.lib()
        h = C.c_void_p()
        self._handle = C.create_string_buffer(64)
        _lib.check(L.dgds_px_create(device, world, rank, self.bytes, C.byref(h), self._handle))
        self.h = h
        self.overflow = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._bases: Optional[List[int]] = None
        self._seg_ptrs: Dict[Tuple[str, int], C.Array] = {}
        if connect and world > 1:
            import torch.distributed as dist
            hs = [None] * world
            dist.all_gather_object(hs, self._handle.raw, group=group)
            _lib.check(L.dgds_px_connect(self.h, b"".join(hs)))

    @staticmethod
    def local_group(world: int, device: int, channels: Dict[str, Tuple[int, int]]) -> List["PeerExchange"]:
        """All `world` ranks in this process (tests on one GPU)."""
        pxs = [PeerExchange(world, r, device, channels, connect=False) for r in range(world)]
        arr = (C.c_void_p * world)(*[p.h.value for p in pxs])
        _lib.check(_lib.lib().dgds_px_connect_local(arr, world))
        return pxs

    # ---- addresses ----
    def bases(self) -> List[int]:
        if self._bases is None:
            out = []
            for p in range(self.world):
                b = C.c_void_p()
                _lib.check(_lib.lib().dgds_px_region(self.h, p, C.byref(b)))
                out.append(b.value)
            self._bases = out
        return self._bases

    def slab_ptr(self, ch: str, seq: int) -> int:
        return self.bases()[self.rank] + self.ch[ch].slab_off[seq % 2]

    def counts_ptr(self, ch: str, seq: int) -> int:
        return self.bases()[self.rank] + self.ch[ch].count_off[seq % 2]

    def slab(self, ch: str, seq: int) -> torch.Tensor:
        """This rank's received rows of exchange `seq`: [world * rows, words] (sender-major)."""
        c = self.ch[ch]
        rows = c.rows if c.shared else self.world * c.rows
        return _view(self.bases()[self.rank] + c.slab_off[seq % 2], (rows, c.words), "<i4", self.device)

    def counts(self, ch: str, seq: int) -> torch.Tensor:
        c = self.ch[ch]
        return _view(self.bases()[self.rank] + c.count_off[seq % 2], (self.world,), "<i4", self.device)

    def seg_out(self, ch: str, seq: int) -> C.Array:
        """Per peer p: where this rank's rows start in p's slab of `ch` (reply destinations)."""
        key = (ch, seq % 2)
        if key not in self._seg_ptrs:
            c = self.ch[ch]
            mine = 0 if c.shared else 4 * self.rank * c.rows * c.words
            self._seg_ptrs[key] = (C.c_void_p * self.world)(*[b + c.slab_off[seq % 2] + mine for b in self.bases()])
        return self._seg_ptrs[key]

    # ---- exchange ----
    def send(self, ch: str, owner: torch.Tensor, records: torch.Tensor, seq: int, stable: bool = False,
             slot: Optional[torch.Tensor] = None, origin_word: int = -1, want_slot: bool = True,
             stream=None) -> Optional[torch.Tensor]:
        """Rows to their owners' slabs of exchange `seq`. Returns the slot map
        (owner * rows + row, -1 if dropped) unless want_slot is False; origin_word >= 0 stamps
        each delivered row with its index here (replies then come back in this order)."""
        c = self.ch[ch]
        n = records.shape[0]
        assert records.dtype == torch.int32 and records.is_contiguous() and records.shape[1] == c.words
        assert owner.dtype == torch.int32 and owner.is_contiguous() and owner.shape[0] == n
        if slot is None and want_slot:
            slot = torch.empty(n, dtype=torch.int64, device=self.device)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _lib.check(_lib.lib().dgds_px_send(self.h, n, C.c_void_p(owner.data_ptr()), C.c_void_p(records.data_ptr()),
                                           c.words, c.rows, c.slab_off[seq % 2], c.count_off[seq % 2], c.flag_off,
                                           seq, 1 if stable else 0, origin_word,
                                           C.c_void_p(slot.data_ptr()) if slot is not None else None,
                                           C.c_void_p(self.overflow.data_ptr()), C.c_void_p(st.cuda_stream)))
        return slot

    def wait(self, ch: str, seq: int, stream=None) -> None:
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _lib.check(_lib.lib().dgds_px_wait(self.h, self.ch[ch].flag_off, seq, C.c_void_p(st.cuda_stream)))

    def signal(self, ch: str, seq: int, stream=None) -> None:
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _lib.check(_lib.lib().dgds_px_signal(self.h, self.ch[ch].flag_off, seq, C.c_void_p(st.cuda_stream)))

    def status(self) -> Tuple[bool, int]:
        t, n = _lib._I32(), _lib._U64()
        _lib.check(_lib.lib().dgds_px_status(self.h, C.byref(t), C.byref(n)))
        return bool(t.value), int(n.value)

    def set_timeout(self, seconds: float) -> None:
        _lib.check(_lib.lib().dgds_px_set_timeout(self.h, int(seconds * 1e9)))

    def close(self) -> None:
        if self.h:
            _lib.lib().dgds_px_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def speculate_routed(srv, px: PeerExchange, q_ch: str, rep_ch: str, seq: int, layout, d_args: torch.Tensor,
                     max_top_k: int, max_spec: int, stats: Optional[torch.Tensor] = None, stream=None,
                     origin_field: int = -1) -> None:
    """Owner side of a routed query exchange: K2 + fused K3 over the received query rows of
    exchange `seq`, replies stored straight into each sender's `rep_ch` slab (at the row the
    sender stamped into `origin_field` when >= 0, for a shared reply slab), then signalled."""
    c = px.ch[q_ch]
    st = stream if stream is not None else torch.cuda.current_stream(px.device)
    px.wait(q_ch, seq, st)
    _lib.check(_lib.lib().dgds_speculate_records_seg(
        srv.handle, px.world, c.rows, C.c_void_p(px.slab_ptr(q_ch, seq)),
        C.c_void_p(px.counts_ptr(q_ch, seq)), C.byref(layout), C.c_void_p(d_args.data_ptr()), 0, max_top_k,
        max_spec, px.seg_out(rep_ch, seq), origin_field, C.c_void_p(stats.data_ptr()) if stats is not None else None,
        C.c_void_p(st.cuda_stream)))
    px.signal(rep_ch, seq, st)


class TickDriver:
    """The routed tick loop in C++ (``dgds_px_driver_*``, csrc/px_driver.cpp) for one rank.

    ``ticks`` is a list of (q_owner, q_records, a_owner, a_records) device tensors, one per tick
    (int32, contiguous; query rows carry ``q_origin_word``, append rows the layout
    handle | request id | prev lo | prev hi | count | tokens). ``run(first, last)`` enqueues
    ticks [first, last) on ``stream``: queries to their owners, the owner's K2 + K3 with replies
    into the senders' shared ``rep`` slab, appends to their owners planned on the server's
    planner thread and launched after each tick's queries."""

    def __init__(self, srv, px: PeerExchange, layout, d_args: torch.Tensor, max_top_k: int, max_spec: int,
                 ticks: Sequence[Tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]],
                 q_origin_word: int, stream=None, q: str = "q", rep: str = "rep", a: str = "a"):
        L = _lib.lib()
        self._keep = [t for tick in ticks for t in tick]  # the driver reads them until it is destroyed
        descs = [self._desc(px.ch[n]) for n in (q, rep, a)]
        arr = (_lib.PxTick * len(ticks))(*[_lib.PxTick(qr.shape[0], ar.shape[0], qo.data_ptr(), qr.data_ptr(),
                                                       ao.data_ptr(), ar.data_ptr()) for qo, qr, ao, ar in ticks])
        st = stream if stream is not None else torch.cuda.current_stream(px.device)
        self.h = C.c_void_p()
        _lib.check(L.dgds_px_driver_create(srv.handle, px.h, px.world, px.rank, C.byref(descs[0]), C.byref(descs[1]),
                                           C.byref(descs[2]), q_origin_word, C.byref(layout),
                                           C.c_void_p(d_args.data_ptr()), max_top_k, max_spec,
                                           C.c_void_p(px.overflow.data_ptr()), arr, len(ticks),
                                           C.c_void_p(st.cuda_stream), C.byref(self.h)))

    @staticmethod
    def _desc(c: Channel):
        d = _lib.PxChannelDesc()
        d.rows, d.words, d.shared, d.flag_off = c.rows, c.words, 1 if c.shared else 0, c.flag_off
        d.count_off[0], d.count_off[1] = c.count_off
        d.slab_off[0], d.slab_off[1] = c.slab_off
        return d

    def run(self, first: int, last: int, plan_to: int = 0, stats: Optional[torch.Tensor] = None) -> None:
        """Ticks [first, last); ticks < plan_to (0: last) may be planned ahead."""
        _lib.check(_lib.lib().dgds_px_driver_run(self.h, first, last, plan_to,
                                                 C.c_void_p(stats.data_ptr()) if stats is not None else None))

    def close(self) -> None:
        """Launches any tick planned ahead but not run, then frees the driver."""
        if self.h:
            _lib.check(_lib.lib().dgds_px_driver_destroy(self.h))
            self.h = C.c_void_p()

