"""Sequential CPU model of the compressed-index append (k_stage + K1 + K1b walks).

Debug aid: runs the same per-lane algorithm as kernels.cu on one interleaving
(segments one after another, events after all segments) and expands the
compressed index into the full trie (window -> count) to compare with a
brute-force window count. Not used by the product or the tests.
"""
import random
import sys
from collections import Counter


def brute(streams, D):
    c = Counter()
    for s in streams:
        for t in range(len(s)):
            for L in range(1, min(D, t + 1) + 1):
                c[tuple(s[t - L + 1:t + 1])] += 1
    return c


class Model:
    def __init__(self, D):
        self.D = D
        self.slots = {}  # (parent, token) -> dict(id, count(occ-1), occ=(stream, depth, pos))
        self.byid = {}
        self.next_id = 1
        self.hist = {}  # stream -> tokens
        self.active = {}  # stream -> [32]
        self.ov = {}
        self.events = []

    def add(self, parent, tok, occ, inc=1):
        """add_window: returns (id, created, converted, displaced occ)."""
        k = (parent, tok)
        e = self.slots.get(k)
        if e is None:
            e = dict(id=self.next_id, count=inc - 1, occ=occ if inc == 1 else (occ[0], occ[1], "mark"), key=k)
            self.next_id += 1
            self.slots[k] = e
            self.byid[e["id"]] = e
            return e["id"], True, False, None
        old = e["count"]
        e["count"] += inc
        if e["occ"][2] != "mark" and old == 0:
            d = e["occ"]
            e["occ"] = (d[0], d[1], "mark")
            return e["id"], False, True, d
        return e["id"], False, False, None

    def append_batch(self, recs, order=None):
        """recs: list of (stream, tokens) in call order; one segment per stream."""
        segs = {}
        for s, toks in recs:
            segs.setdefault(s, []).extend(toks)
        start = {s: len(self.hist.get(s, [])) for s in segs}
        for s, toks in segs.items():  # k_stage
            self.hist.setdefault(s, []).extend(toks)
            self.active.setdefault(s, [0] * 32)
            self.ov.setdefault(s, [0] * 32)
        items = list(segs.items())
        if order:
            random.Random(order).shuffle(items)
        D = self.D
        for s, toks in items:  # K1, one segment at a time
            len0 = start[s]
            a = [self.active[s][l] if (l < D and l < len0) else 0 for l in range(32)]
            for l in range(32):
                o = self.ov[s][l]
                if o:
                    self.ov[s][l] = 0
                    if l < D and l < len0:
                        a[l] = o
            rider = [None] * 32  # (stream, pos)
            ln = len0
            for t in toks:
                newsize = min(D, ln + 1)
                na = [0] * 32
                nr = [None] * 32
                for l in range(newsize):
                    parent = ("root", 0) if l == 0 else a[l - 1]
                    if parent == 0:
                        continue
                    prd = rider[l - 1] if l > 0 else None
                    inc = 1
                    if prd is not None:
                        rs, rp = prd
                        if rp + 1 < len(self.hist[rs]) and self.hist[rs][rp + 1] == t:
                            inc = 2
                        else:
                            self.events.append((parent, l, rs, rp))
                    id_, created, conv, d = self.add(parent, t, (s, l + 1, ln), inc)
                    if not created or inc == 2:
                        na[l] = id_
                        if inc == 2:
                            nr[l] = (prd[0], prd[1] + 1)
                        if conv:
                            if nr[l] is None:
                                nr[l] = (d[0], d[2])
                            else:
                                self.events.append((id_, l + 1, d[0], d[2]))
                for l in range(32):
                    if nr[l] is not None and l + 1 >= D:
                        nr[l] = None
                a, rider = na, nr
                ln += 1
            for l in range(32):
                if rider[l] is not None:
                    self.events.append((a[l], l + 1, rider[l][0], rider[l][1]))
            for l in range(32):
                if l < D and l < ln:
                    self.active[s][l] = a[l]
        # K1b
        evs, self.events = self.events, []
        for ev in evs:
            self.walk(*ev)

    def walk(self, id_, depth, stream, pos):
        stk = []
        cur = (id_, depth, stream, pos)
        rider = None
        while True:
            cid, d, s, p0 = cur
            L = len(self.hist[s])
            p = p0 + 1
            if p == L:
                self.ov[s][d - 1] = cid
            if rider is not None and rider[1] + 1 >= len(self.hist[rider[0]]):
                self.ov[rider[0]][d - 1] = cid
                rider = None
            if d < self.D and p < L:
                x = self.hist[s][p]
                inc = 1
                if rider is not None:
                    if self.hist[rider[0]][rider[1] + 1] == x:
                        inc = 2
                    else:
                        stk.append((cid, d, rider[0], rider[1]))
                        rider = None
                nid, created, conv, dd = self.add(cid, x, (s, d + 1, p), inc)
                if not created or inc == 2:
                    if inc == 2:
                        rider = (rider[0], rider[1] + 1)
                    if conv:
                        if rider is None:
                            rider = (dd[0], dd[2])
                        else:
                            stk.append((nid, d + 1, dd[0], dd[2]))
                    cur = (nid, d + 1, s, p)
                    continue
            elif rider is not None and d < self.D:
                stk.append((cid, d, rider[0], rider[1]))
            rider = None
            if not stk:
                break
            cur = stk.pop()

    def expand(self):
        """window tuple -> count, from entries and the implicit chains below leaves."""
        out = Counter()

        def window(e):
            toks = []
            while True:
                toks.append(e["key"][1])
                par = e["key"][0]
                if isinstance(par, tuple):
                    return tuple(reversed(toks))
                e = self.byid[par]

        for e in self.slots.values():
            w = window(e)
            out[w] += e["count"] + 1
            if e["count"] == 0 and e["occ"][2] != "mark":
                s, d, p = e["occ"]
                h = self.hist[s]
                k = 1
                while d + k <= self.D and p + k < len(h):
                    out[w + tuple(h[p + 1:p + k + 1])] += 1
                    k += 1
        return out


def s_root(s):
    return 0  # one group


def check(streams, D, rec=4, batch_all=True, order=None):
    m = Model(D)
    recs = []
    for r, s in enumerate(streams):
        for p in range(0, len(s), rec):
            recs.append((p, r, s[p:p + rec]))
    recs.sort(key=lambda x: x[0])
    if batch_all:
        m.append_batch([(r, t) for _, r, t in recs], order)
    else:
        for _, r, t in recs:
            m.append_batch([(r, t)])
    got = m.expand()
    exp = brute(streams, D)
    return got == exp, got, exp


if __name__ == "__main__":
    bad = 0
    for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 200):
        rng = random.Random(seed)
        ns = rng.randint(1, 4)
        streams = [[rng.randrange(rng.randint(2, 5)) for _ in range(rng.randint(1, 40))] for _ in range(ns)]
        for ball in (True, False):
            ok, got, exp = check(streams, D=rng.choice([3, 5, 24]), batch_all=ball, order=seed)
            if not ok:
                bad += 1
                if bad < 3:
                    diff = {k: (got.get(k), exp.get(k)) for k in set(got) | set(exp) if got.get(k) != exp.get(k)}
                    print("seed", seed, ball, streams, list(diff.items())[:5])
    print("bad", bad)
