"""Top warp-stall SASS instructions of an ncu capture (run here, CPU side).

    python tools/ncu_hot.py <rep.ncu-rep> [N]
Prints the N instructions with the most stall samples, with the stall reason
columns that dominate, plus a coarse per-opcode summary.
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr_i]
body = [r for r in rows[hdr_i + 1:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") or "Stall" in c and "Sampling" not in c]
tot = sum(int(r[si]) for r in body)
print("total samples", tot, "instructions", len(body))
idx = {r[0]: k for k, r in enumerate(body)}
top = sorted(body, key=lambda r: -int(r[si]))[:n]
for r in top:
    k = idx[r[0]]
    prev = body[k - 1][1].strip() if k > 0 else ""
    print(f"{int(r[si]):6d} {100*int(r[si])/tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:70]:70s} | prev: {prev[:50]}")
ops = Counter()
for r in body:
    op = r[1].strip().split()[0] if r[1].strip() else "?"
    if op.startswith("@"):
        op = r[1].strip().split()[1]
    ops[op.split(".")[0]] += int(r[si])
print("by opcode:", [(o, round(100 * v / tot, 1)) for o, v in ops.most_common(15)])
