"""Framed DGDS wire protocol (reference: proj/include/rollsim/dgds_wire.hpp:12-28).

``WireService`` runs the B200 server behind the protocol (csrc/wire.cpp: reader
thread per connection, one dispatcher that applies every waiting update_cst as
one batch). ``WireClient`` is a blocking client with the reference
``TcpTransport`` semantics (one request in flight, 0x7F replies raise). The
``encode_*`` / ``decode_*`` helpers are the reference's record layouts.
"""
from __future__ import annotations

import ctypes as C
import socket
import struct
import threading
from typing import List, Sequence, Tuple

from . import _lib
from .dgds import FetchReply, UpdateReply

OP_UPDATE, OP_FETCH, OP_REGISTER, OP_REPLY, OP_ERROR = 0x01, 0x02, 0x03, 0x80, 0x7F


def _str(s: str) -> bytes:
    b = s.encode()
    return struct.pack(">H", len(b)) + b


def encode_update_request(group_id: str, request_id: int, prev_token_count: int, tokens: Sequence[int]) -> bytes:
    return (bytes([OP_UPDATE]) + _str(group_id) + struct.pack(">IQI", request_id & 0xFFFFFFFF, prev_token_count,
                                                               len(tokens))
            + struct.pack(f">{len(tokens)}i", *tokens))


def encode_fetch_request(group_ids: Sequence[str], cached_versions: Sequence[int]) -> bytes:
    out = bytes([OP_FETCH]) + struct.pack(">I", len(group_ids))
    for g, v in zip(group_ids, cached_versions):
        out += _str(g) + struct.pack(">Q", v)
    return out


def encode_register_request(group_id: str, ttl_seconds: int) -> bytes:
    return bytes([OP_REGISTER]) + _str(group_id) + struct.pack(">I", ttl_seconds)


def frame(payload: bytes) -> bytes:
    return struct.pack(">I", len(payload)) + payload


class WireError(RuntimeError):
    pass


def _check_reply(reply: bytes, op: int) -> memoryview:
    if reply and reply[0] == OP_ERROR:
        n = struct.unpack(">H", reply[1:3])[0]
        raise WireError("draft server error: " + reply[3:3 + n].decode())
    if not reply or reply[0] != (op | OP_REPLY):
        raise WireError("unexpected reply tag")
    return memoryview(reply)[1:]


def decode_update_reply(reply: bytes) -> UpdateReply:
    m = _check_reply(reply, OP_UPDATE)
    ok, ver, acked = struct.unpack(">BQQ", m[:17])
    return UpdateReply(bool(ok), ver, acked)


def decode_fetch_reply(reply: bytes) -> List[FetchReply]:
    m = _check_reply(reply, OP_FETCH)
    n = struct.unpack(">I", m[:4])[0]
    p = 4
    out = []
    for _ in range(n):
        kind, ver, blen = struct.unpack(">BQI", m[p:p + 13])
        p += 13
        out.append(FetchReply(kind, ver, bytes(m[p:p + blen])))
        p += blen
    return out


class WireClient:
    """Blocking client over TCP (TcpTransport, dgds_wire.cpp:176-250)."""

    def __init__(self, host: str, port: int):
        self.sock = socket.create_connection((host, port))
        self.sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
        self.lock = threading.Lock()

    def _recv(self, n: int) -> bytes:
        buf = bytearray()
        while len(buf) < n:
            chunk = self.sock.recv(n - len(buf))
            if not chunk:
                raise WireError("draft server closed connection")
            buf += chunk
        return bytes(buf)

    def round_trip(self, payload: bytes) -> bytes:
        with self.lock:
            self.sock.sendall(frame(payload))
            n = struct.unpack(">I", self._recv(4))[0]
            return self._recv(n)

    def update_cst(self, group_id, request_id, prev_token_count, tokens) -> UpdateReply:
        return decode_update_reply(self.round_trip(encode_update_request(group_id, request_id, prev_token_count,
                                                                         list(tokens))))

    def fetch_cst(self, group_ids, cached_versions) -> List[FetchReply]:
        return decode_fetch_reply(self.round_trip(encode_fetch_request(group_ids, cached_versions)))

    def register_group(self, group_id, ttl_seconds):
        _check_reply(self.round_trip(encode_register_request(group_id, int(ttl_seconds))), OP_REGISTER)

    def close(self):
        self.sock.close()


class WireService:
    """The GPU draft server behind the framed protocol on 127.0.0.1 (dgds_wire_service_*)."""

    def __init__(self, server, port: int = 0):
        self.server = server
        h = C.c_void_p()
        p = _lib._I32()
        _lib.check(_lib.lib().dgds_wire_service_start(server.handle, port, C.byref(h), C.byref(p)))
        self.h, self.port = h, int(p.value)

    def stats(self) -> Tuple[int, int]:
        r, b = _lib._U64(), _lib._U64()
        _lib.check(_lib.lib().dgds_wire_service_stats(self.h, C.byref(r), C.byref(b)))
        return int(r.value), int(b.value)

    def stop(self):
        if self.h:
            _lib.lib().dgds_wire_service_stop(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.stop()


def serve_payload(server, payload: bytes, now: float) -> bytes:
    """wire::serve_payload on the B200 server: one request payload -> reply payload."""
    cap = 1 << 16
    while True:
        out = C.create_string_buffer(cap)
        n = _lib._U64()
        buf = C.create_string_buffer(bytes(payload), max(1, len(payload)))
        rc = _lib.lib().dgds_wire_serve_payload(server.handle, buf, len(payload), float(now), out, cap, C.byref(n))
        if rc == _lib.DGDS_EBUFFER:
            cap = int(n.value)
            continue
        _lib.check(rc)
        return out.raw[:n.value]
