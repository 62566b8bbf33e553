"""Generate the golden fixtures under tests/golden/ from the COMPILED REFERENCE.

TEST INFRASTRUCTURE ONLY. Needs oracle/_ref/libdgds_ref.so (built from
/root/reference by oracle/Makefile), so it runs in the build container, not on
the GPU box; the JSON it writes is committed and travels.

  python oracle/make_golden.py            # all fixtures
  python oracle/make_golden.py --quick    # skip the large-trace fingerprints

Fixtures:
  spec_kats.json       SPEC.md known-answer examples, answered by the reference
  random_cases.json    randomized append/query schedules (AC1-style)
  c1_queries.json      config C1 (1 x 16 x 4096, V 32000, rho_pat 0.8) R1 queries, k=1 and k=4
  replay_small.json    staggered engine replay through reference Instance/DraftClient
  workload_fp.json     sha256 of reference generate_workload traces for C1..C4
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys
from dataclasses import asdict

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def cands_json(cs):
    return [{"tokens": list(c.tokens), "score_bits": np.float64(c.score).view(np.uint64).item(),
             "score": c.score, "support": c.support} for c in cs]


def args_json(a: O.OrcArgs):
    return {"max_spec_tokens": a.max_spec_tokens, "pattern_lookup_max": a.pattern_lookup_max,
            "pattern_lookup_min": a.pattern_lookup_min, "top_k": a.top_k, "min_step_freq": a.min_step_freq,
            "min_support": a.min_support}


def random_cases(R, n_cases=400, seed=2511):
    rng = random.Random(seed)
    cases = []
    for _ in range(n_cases):
        V = rng.randint(2, 8)
        nreq = rng.randint(1, 4)
        lim = rng.choice([(8, 16), (8, 16), (8, 16), (2, 3), (3, 5), (4, 4)])
        ix = R.index("g", *lim)
        stored = [0] * nreq
        appends = []
        for _ in range(rng.randint(1, 14)):
            r = rng.randrange(nreq)
            n = rng.randint(0, 6)
            toks = [rng.randrange(V) for _ in range(n)]
            prev = stored[r] if rng.random() < 0.88 else rng.randint(0, 30)
            ok, ver, acked = ix.append(r, prev, toks)
            if ok:
                stored[r] += n
            appends.append({"request_id": r, "prev": prev, "tokens": toks,
                            "reply": {"ok": ok, "version": ver, "acked": acked}})
        queries = []
        for _ in range(6):
            a = O.make_args(rng.randint(0, 16), 1, 1, rng.randint(1, 4), rng.choice([0.0, 0.1, 0.25, 0.5]),
                            rng.choice([0, 1, 2, 3]))
            a.pattern_lookup_max = rng.randint(1, 8)
            a.pattern_lookup_min = rng.randint(1, a.pattern_lookup_max)
            pat = [rng.randrange(V) for _ in range(rng.randint(0, 9))]
            queries.append({"pattern": pat, "args": args_json(a), "expect": cands_json(ix.speculate(pat, a))})
        cases.append({"limits": list(lim), "appends": appends, "queries": queries, "node_count": ix.node_count,
                      "version": ix.version})
    return cases


def spec_kats(R):
    """SPEC.md:132-134,141-143,150-152 + SURVEY.md §8(c) edge semantics, answered by the reference."""
    out = []

    def run(name, lim, appends, pattern, args):
        ix = R.index("g", *lim)
        reps = [ix.append(r, p, t) for (r, p, t) in appends]
        out.append({"name": name, "limits": list(lim),
                    "appends": [{"request_id": r, "prev": p, "tokens": t} for (r, p, t) in appends],
                    "replies": [list(x) for x in reps], "pattern": pattern, "args": args_json(args),
                    "expect": cands_json(ix.speculate(pattern, args))})

    A = O.make_args
    run("single_seq_unique", (8, 16), [(1, 0, [1, 2, 3])], [2], A(8, 6, 1, 1))
    run("unique_continuation", (8, 16), [(1, 0, [1, 2, 3, 4, 5])], [2, 3], A(8, 6, 1, 1))
    run("symmetric_split", (8, 16), [(1, 0, [1, 2, 3]), (2, 0, [1, 2, 4])], [1, 2], A(8, 6, 1, 2))
    run("isolation_no_fallback", (8, 16), [(1, 0, [1, 2]), (2, 0, [2, 9])], [1, 2], A(8, 6, 1, 1))
    run("out_of_order", (8, 16), [(1, 0, [1, 2]), (1, 5, [3])], [1], A(8, 6, 1, 1))
    run("empty_append", (8, 16), [(1, 0, []), (1, 0, [4, 5])], [4], A(8, 6, 1, 1))
    run("absent_pattern", (8, 16), [(1, 0, [1, 2, 3])], [7], A(8, 6, 1, 1))
    run("max_spec_zero", (8, 16), [(1, 0, [1, 2, 3])], [1], A(0, 6, 1, 1))
    run("limits_clamp", (2, 3), [(1, 0, [1, 2, 3, 4, 5, 6, 7, 8, 9])], [2, 3], A(8, 6, 1, 1))
    run("end_of_stream_dilution", (8, 16), [(1, 0, [5, 6]), (2, 0, [5, 6, 7])], [5, 6], A(8, 6, 1, 1))
    run("five_way_split_pruned", (8, 16),
        [(r, 0, [1, 10 + r]) for r in range(5)], [1], A(8, 6, 1, 4))
    run("lookup_min_above_max", (8, 16), [(1, 0, [1, 2, 3])], [1, 2], A(8, 6, 6, 1))
    run("min_support_2", (8, 16), [(1, 0, [1, 2, 1, 3, 1, 2])], [1], A(8, 6, 1, 2, 0.0, 2))
    return out


def c1_queries(R, n=1500, seed=99):
    cfg = dict(num_groups=1, group_size=16, location=4096.0, scale=0.0, group_correlation=1.0,
               pattern_similarity=0.8, vocab_size=32000, max_tokens=4096, seed=7)
    ids, plens, outs, fp = R.workload(**cfg)
    ix = R.index(ids[0], 8, 16)
    streams = outs[0]
    # R1 build: 16-token records, round-robin request order
    pos = [0] * len(streams)
    while any(p < len(s) for p, s in zip(pos, streams)):
        for r, s in enumerate(streams):
            if pos[r] < len(s):
                t = s[pos[r]:pos[r] + 16]
                ok, _, _ = ix.append(r, pos[r], t)
                assert ok
                pos[r] += len(t)
    rng = random.Random(seed)
    qs = []
    for i in range(n):
        r = rng.randrange(len(streams))
        p = rng.randint(6, len(streams[r]) - 1)
        k = 1 if i % 2 == 0 else 4
        a = O.make_args(8, 6, 1, k, 0.25, 1)
        pat = [int(x) for x in streams[r][p - 6:p]]
        qs.append({"stream": r, "pos": p, "top_k": k, "expect": cands_json(ix.speculate(pat, a))})
    return {"config": cfg, "node_count": ix.node_count, "version": ix.version, "queries": qs}


def replay_small(R):
    cfgs = []
    for (ng, gs, loc, rho, stagger, k, budget, adaptive, abt) in [
        (2, 4, 300.0, 0.8, 32, 1, 64, 1, 16),
        (1, 6, 200.0, 0.9, 16, 4, 4096, 1, 1),
        (3, 3, 150.0, 0.7, 8, 2, 8, 0, 4),
    ]:
        wc = dict(num_groups=ng, group_size=gs, location=loc, scale=0.3, group_correlation=0.9,
                  pattern_similarity=rho, vocab_size=50, max_tokens=512, seed=11)
        rc = O.OrcReplayCfg(stagger, abt, budget, 8, adaptive, k, 8, 16, 100000, 0, O.make_args(8, 6, 1, 1))
        steps, rec, nq = R.replay(wc, rc)
        cfgs.append({"workload": wc, "stagger": stagger, "append_batch_tokens": abt, "batch_token_budget": budget,
                     "per_request_cap": 8, "adaptive": adaptive, "multi_path_k": k,
                     "args": args_json(O.make_args(8, 6, 1, 1)), "steps": steps.tolist(),
                     "records": rec.tolist(), "queries": nq})
    return cfgs


def workload_fp(R, names):
    from paper_2511_14617_b200.workload import CONFIGS
    out = {}
    for name in names:
        ids, plens, outs, fp = R.workload(**asdict(CONFIGS[name]))
        h = hashlib.sha256()
        lens = []
        for g in outs:
            for s in g:
                h.update(np.ascontiguousarray(s, np.int32).tobytes())
                lens.append(len(s))
        out[name] = {"sha256": h.hexdigest(), "total_tokens": int(sum(lens)), "prompt_lens_head": plens[:8],
                     "ref_trace_fingerprint": fp}
        del outs
    return out


def main():
    R = O.reference()
    if R is None:
        raise SystemExit("oracle/_ref/libdgds_ref.so missing: run make -C oracle (needs /root/reference)")
    os.makedirs(GOLD, exist_ok=True)
    quick = "--quick" in sys.argv

    def dump(name, obj):
        with open(os.path.join(GOLD, name), "w") as f:
            json.dump(obj, f, separators=(",", ":"))
        print("wrote", name, os.path.getsize(os.path.join(GOLD, name)))

    dump("spec_kats.json", spec_kats(R))
    dump("random_cases.json", random_cases(R))
    dump("c1_queries.json", c1_queries(R))
    dump("replay_small.json", replay_small(R))
    dump("workload_fp.json", workload_fp(R, ["C1", "C3"] if quick else ["C1", "C2", "C3", "C4"]))


if __name__ == "__main__":
    main()
