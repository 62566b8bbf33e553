"""Top source lines of an ncu report by warp-stall samples and instructions executed.

  python tools/ncu_hot.py gpurun_out/prof_query.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ix = {}
for i, k in enumerate(hdr):
    ix.setdefault(k, i)
lines = []
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr) or not r[0]:
        continue
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]])
        ins = int(r[ix["Instructions Executed"]])
    except ValueError:
        continue
    lines.append((s, ins, int(r[0]), r[1].strip()[:110]))
tot = sum(x[0] for x in lines) or 1
toti = sum(x[1] for x in lines) or 1
print(f"total stall samples {tot}, warp instructions {toti}")
for s, ins, ln, src in sorted(lines, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% {100*ins/toti:5.1f}%i  L{ln:<5d} {src}")
