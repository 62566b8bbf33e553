import sys, faulthandler, time
faulthandler.dump_traceback_later(40, exit=True)
sys.path.insert(0, ".")
from oracle import oracle as O
from paper_2511_14617_b200 import dgds as D
streams = [[0, 2, 2, 0, 1, 2, 1, 2, 2, 0, 2, 0], [1, 1, 2, 0, 0, 2, 1, 2, 2, 1, 1, 2]]
s = D.DraftServer(D.DgdsParams(max_pattern_len=8, max_spec_len=16), device=0)
recs = []
for r in range(2):
    for p in range(0, 12, 4):
        recs.append((p, r, streams[r][p:p + 4]))
recs.sort(key=lambda x: x[0])
print("update", flush=True)
if len(sys.argv) > 1:
    recs = recs[:int(sys.argv[1])]
reps = s.update_batch(["g"] * len(recs), [x[1] for x in recs], [x[0] for x in recs], [x[2] for x in recs], 0.0)
print("replies", [(r.ok, r.version, r.acked_tokens) for r in reps], flush=True)
print("entries", s.entry_count(), flush=True)
print("err", s.device_error(), flush=True)
print("nodes", s.node_count(), flush=True)
import numpy as np, ctypes as C
from paper_2511_14617_b200 import _lib
cap = s.index_slots()
buf = np.zeros((cap, 8), np.uint32)
_lib.check(_lib.lib().dgds_debug_dump(s.handle, 0, buf.ctypes.data_as(C.c_void_p), buf.nbytes))
si = np.zeros((4, 4), np.uint32)
_lib.check(_lib.lib().dgds_debug_dump(s.handle, 1, si.ctypes.data_as(C.c_void_p), si.nbytes))
print("sinfo", si)
ev = np.zeros((64, 6), np.uint32)
_lib.check(_lib.lib().dgds_debug_dump(s.handle, 5, ev.ctypes.data_as(C.c_void_p), ev.nbytes))
print("events", ev[:20])
sh = np.zeros(160, np.int32)
_lib.check(_lib.lib().dgds_debug_dump(s.handle, 4, sh.ctypes.data_as(C.c_void_p), sh.nbytes))
print("shist", sh)
occ = np.nonzero(buf[:, 0])[0]
byid = {}
for i in occ:
    byid[i + 1] = buf[i]
def window(i):
    toks = []
    while True:
        e = byid[i]
        toks.append(int(e[1]))
        if e[0] > 0xFFBFFFFF:
            return tuple(reversed(toks))
        if int(e[0]) not in byid:
            return ("BADPARENT", int(e[0])) + tuple(reversed(toks))
        i = int(e[0])
wins = {}
for i in occ:
    e = buf[i]
    w = window(i + 1)
    print(i + 1, "parent", int(e[0]), "tok", int(e[1]), "occ s", int(e[2]) & 0xFFFFFF, "d", (int(e[2]) >> 24) + 1, "pos", int(e[3]), "cnt", int(e[4]) + 1, "fc", int(e[5]), "h", hex(int(e[6])), "ns", int(e[7]), "win", w)
    wins.setdefault(w, []).append(i + 1)
print("duplicates", {k: v for k, v in wins.items() if len(v) > 1})
