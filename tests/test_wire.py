"""Framed wire service (dgds_wire.hpp:12-28, dgds_wire.cpp:103-332).

- serve_payload: replies byte-identical to the reference's for the same request
  sequence, errors included (unknown op, truncated record, negative token, bad TTL);
- the reference's own TcpTransport client against our GPU service gives the replies
  it gets from the reference TcpDraftService;
- concurrent clients: the dispatcher folds waiting update_cst frames into batches, and
  the final state equals the sequential reference.
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import pytest

from paper_2511_14617_b200 import dgds as D
from paper_2511_14617_b200 import wire as W

pytestmark = pytest.mark.gpu


def _ref_server(ref):
    return ref.L.orc_ref_server_new(1, 0.0, 16, 600.0, 8, 16)


def test_serve_payload_byte_identical(reference):
    if reference is None:
        pytest.skip("oracle/_ref not built")
    rs = _ref_server(reference)
    s = D.DraftServer(D.DgdsParams(), expected_nodes=1 << 16)
    rng = np.random.default_rng(3)
    stored = {}
    payloads = []
    for k in range(300):
        g = f"g{int(rng.integers(3))}"
        r = int(rng.integers(4))
        op = rng.random()
        if op < 0.6:
            have = stored.get((g, r), 0)
            prev = have if rng.random() > 0.1 else have + 2
            toks = rng.integers(0, 9, int(rng.integers(0, 12))).tolist()
            if rng.random() < 0.03:
                toks.insert(0, -5)  # negative token (first: the reference inserts no prefix before throwing)
            rid = r if rng.random() > 0.02 else -1  # u32 0xFFFFFFFF -> negative request id
            payloads.append(W.encode_update_request(g, rid, prev, toks))
            if prev == have and -5 not in toks and rid >= 0:
                stored[(g, r)] = have + len(toks)
        elif op < 0.8:
            ids = [f"g{int(x)}" for x in rng.integers(0, 4, int(rng.integers(1, 4)))]
            payloads.append(W.encode_fetch_request(ids, [int(x) for x in rng.integers(0, 30, len(ids))]))
        elif op < 0.9:
            payloads.append(W.encode_register_request(f"g{int(rng.integers(4))}", int(rng.integers(0, 3)) * 300))
        else:
            payloads.append([bytes([0x09]), b"", W.encode_update_request("g0", 0, 0, [1, 2])[:9]][k % 3])
    for k, p in enumerate(payloads):
        now = float(k)
        assert W.serve_payload(s, p, now) == reference.wire_serve(rs, p, now), (k, p[:16])
    reference.L.orc_ref_server_free(rs)


def _ref_tcp(ref, port):
    t = ref.L.orc_ref_tcp_new(b"127.0.0.1", port)
    assert t, ref.err()
    return t


def _tcp_update(ref, t, g, r, p, toks):
    ok, v, a = C.c_int32(), C.c_uint64(), C.c_uint64()
    arr = np.asarray(toks, np.int32)
    rc = ref.L.orc_ref_tcp_update(t, g.encode(), r, p, arr.ctypes.data_as(C.POINTER(C.c_int32)), len(arr),
                                  C.byref(ok), C.byref(v), C.byref(a))
    return ("err", ref.err().args[0]) if rc else (ok.value, v.value, a.value)


def _tcp_fetch(ref, t, g, cached):
    kind, ver = C.c_int32(), C.c_uint64()
    blob = ref._blob_call(lambda b, c, l: ref.L.orc_ref_tcp_fetch(t, g.encode(), cached, C.byref(kind),
                                                                  C.byref(ver), b, c, l))
    return kind.value, ver.value, blob


def test_reference_tcp_client_against_gpu_service(reference):
    if reference is None:
        pytest.skip("oracle/_ref not built")
    s = D.DraftServer(D.DgdsParams(), expected_nodes=1 << 16)
    rsv = reference.L.orc_ref_service_new(0)
    with W.WireService(s) as svc:
        ours = _ref_tcp(reference, svc.port)
        theirs = _ref_tcp(reference, reference.L.orc_ref_service_port(rsv))
        rng = np.random.default_rng(9)
        pos = {}
        for k in range(200):
            g, r = f"grp{int(rng.integers(2))}", int(rng.integers(3))
            if rng.random() < 0.7:
                prev = pos.get((g, r), 0)
                toks = rng.integers(0, 7, int(rng.integers(1, 10))).tolist()
                a = _tcp_update(reference, ours, g, r, prev, toks)
                b = _tcp_update(reference, theirs, g, r, prev, toks)
                assert a == b, k
                pos[(g, r)] = prev + len(toks)
            elif rng.random() < 0.8:
                cached = int(rng.integers(0, 20))
                assert _tcp_fetch(reference, ours, g, cached) == _tcp_fetch(reference, theirs, g, cached), k
            else:
                assert reference.L.orc_ref_tcp_register(ours, g.encode(), 600.0) == 0
                assert reference.L.orc_ref_tcp_register(theirs, g.encode(), 600.0) == 0
        reference.L.orc_ref_tcp_free(ours)
        reference.L.orc_ref_tcp_free(theirs)
    reference.L.orc_ref_service_free(rsv)


def test_concurrent_clients_are_batched(reference):
    if reference is None:
        pytest.skip("oracle/_ref not built")
    s = D.DraftServer(D.DgdsParams(), expected_nodes=1 << 20)
    rng = np.random.default_rng(5)
    n_clients, rounds = 8, 60
    seqs = [rng.integers(0, 50, rounds * 16).astype(np.int32) for _ in range(n_clients)]
    errors = []
    with W.WireService(s) as svc:
        def run(c):
            try:
                cl = W.WireClient("127.0.0.1", svc.port)
                for k in range(rounds):
                    rep = cl.update_cst("shared", c, k * 16, seqs[c][k * 16:(k + 1) * 16].tolist())
                    assert rep.ok and rep.acked_tokens == (k + 1) * 16
                cl.close()
            except Exception as e:  # pragma: no cover - surfaced below
                errors.append(e)
        th = [threading.Thread(target=run, args=(c,)) for c in range(n_clients)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errors, errors
        requests, batches = svc.stats()
        assert requests == n_clients * rounds and batches < requests  # folded into batches
        snap = W.WireClient("127.0.0.1", svc.port).fetch_cst(["shared"], [0])[0]
    idx = reference.index(group_id="shared")
    for c in range(n_clients):
        assert idx.append(c, 0, seqs[c])[0]
    want = reference.index_full_snapshot(idx)
    # version counts appends (rounds per client), the reference index had one append per stream
    assert snap.kind == D.FetchKind.Full and snap.version == n_clients * rounds
    assert snap.blob[:4] == b"GDX1"
    hdr = 4 + 1 + 2 + len("shared")
    assert snap.blob[hdr + 16:] == want[hdr + 16:]  # same streams, same tokens (after from/to)
