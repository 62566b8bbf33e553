"""Debug: small randomized cases, GPU vs restatement, first mismatch printed (with node counts)."""
import sys, random, faulthandler, time
faulthandler.dump_traceback_later(100, exit=True)
sys.path.insert(0, ".")
from oracle import oracle as O
from paper_2511_14617_b200 import dgds as D

def case(seed, nstreams=2, length=12, vocab=3, batch_all=False):
    rng = random.Random(seed)
    s = D.DraftServer(D.DgdsParams(max_pattern_len=8, max_spec_len=16), device=0)
    ref = O.restatement().index("g")
    toks = [[rng.randrange(vocab) for _ in range(length)] for _ in range(nstreams)]
    recs = []
    for r in range(nstreams):
        for p in range(0, length, 4):
            recs.append((r, p, toks[r][p:p + 4]))
    rng.shuffle(recs)
    recs.sort(key=lambda x: x[1])  # keep per-stream order
    batches = [recs] if batch_all else [[x] for x in recs]
    for b in batches:
        reps = s.update_batch(["g"] * len(b), [x[0] for x in b], [x[1] for x in b], [x[2] for x in b], 0.0)
        for x in b:
            ref.append(x[0], x[1], x[2])
    t1 = time.time()
    err = s.device_error()
    print("  device_error %.2fs" % (time.time() - t1), flush=True)
    if err:
        print("device error flags", err, "streams", toks, flush=True)
    nc = s.node_count(); rc = ref.node_count
    bad = []
    pats = []
    for r in range(nstreams):
        for p in range(1, length + 1):
            for L in (1, 2, 3, 6):
                if p - L < 0: continue
                pats.append(toks[r][p - L:p])
    a = D.SpeculationArgs(8, 6, 1, 4, 0.0, 1)
    gots = s.speculate_batch(["g"] * len(pats), pats, a)
    for pat, g in zip(pats, gots):
        got = [c.key() for c in g]
        exp = [c.key() for c in ref.speculate(pat, O.make_args(8, 6, 1, 4, 0.0, 1))]
        if got != exp:
            bad.append((pat, got, exp))
    s.close()
    return nc, rc, bad, toks

cfgs = [(2, 12, 3), (3, 40, 4), (4, 120, 8), (4, 400, 64)]
if len(sys.argv) > 2:
    cfgs = [tuple(int(x) for x in sys.argv[2].split(","))]
for (ns, ln, voc) in cfgs:
  for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    for ball in (False, True):
        faulthandler.dump_traceback_later(60, exit=True)
        t0 = time.time()
        print("case", ns, ln, voc, seed, ball, flush=True)
        nc, rc, bad, toks = case(seed, nstreams=ns, length=ln, vocab=voc, batch_all=ball)
        print("  %.2fs" % (time.time() - t0), flush=True)
        if nc != rc or bad:
            print("cfg", ns, ln, voc, "seed", seed, "batch_all", ball, "nodes gpu", nc, "ref", rc, "streams", toks if ln < 50 else "")
            for b in bad[:3]:
                print("  pat", b[0], "\n   got", b[1], "\n   exp", b[2])
            sys.exit(1)
print("all ok")
