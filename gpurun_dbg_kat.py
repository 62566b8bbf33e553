import sys, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import load_golden
from paper_2511_14617_b200 import dgds as D
def gkeys(e): return [(tuple(x["tokens"]), x["score"], x["support"]) for x in e]
for kat in load_golden("spec_kats.json"):
    s = D.DraftServer(D.DgdsParams(max_pattern_len=kat["limits"][0], max_spec_len=kat["limits"][1]))
    gid = "kat-" + kat["name"]
    reps = [s.update_cst(gid, a["request_id"], a["prev"], a["tokens"], 0.0) for a in kat["appends"]]
    a = kat["args"]
    got = s.speculate(gid, kat["pattern"], D.SpeculationArgs(a["max_spec_tokens"], a["pattern_lookup_max"], a["pattern_lookup_min"], a["top_k"], a["min_step_freq"], a["min_support"]))
    ok = [(c.tokens, c.score, c.support) for c in got] == gkeys(kat["expect"])
    print(kat["name"], "OK" if ok else "FAIL", [(c.tokens, c.score, c.support) for c in got], gkeys(kat["expect"]), s.node_count())
