"""Attribute ncu warp-stall samples to CUDA source lines (CPU side).

    python tools/ncu_lines.py <rep.ncu-rep> <lib.so> <mangled-kernel> [N] [kernel-regex]
Extracts the kernel's cubin from the .so, maps SASS offsets to file:line with
nvdisasm --print-line-info (needs -lineinfo), and sums the per-instruction
samples of the ncu source page per line.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, lib, kern = sys.argv[1:4]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
kfilter = ["-k", f"regex:{sys.argv[5]}"] if len(sys.argv) > 5 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kfilter,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[hi + 1:] if len(r) == len(h)]
base = int(body[0][0], 16)
samples = {int(r[0], 16) - base: int(r[si]) for r in body}

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
line_of = {}
for f in os.listdir(tmp):
    dis = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, f)], capture_output=True,
                         text=True).stdout
    sec = f".text.{kern}:"
    if sec not in dis:
        continue
    part = dis.split(sec, 1)[1].split("//---------------------", 1)[0]
    cur = None
    for l in part.splitlines():
        m = re.search(r'line (\d+)', l)
        if "//## File" in l:
            fm = re.search(r'File "([^"]+)", line (\d+)', l)
            if fm:
                cur = f"{os.path.basename(fm.group(1))}:{fm.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            line_of[int(m.group(1), 16)] = cur
    break
agg = collections.Counter()
for off, s in samples.items():
    agg[line_of.get(off, "?")] += s
tot = sum(samples.values())
print("total samples", tot)
for k, v in agg.most_common(n):
    print(f"{v:7d} {100 * v / tot:5.1f}%  {k}")
