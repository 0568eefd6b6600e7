"""Print SASS of the kernels whose (mangled) name contains a substring.
    python tools/sass_fn.py <lib.so> <substring> [--grep REGEX] [--count REGEX]"""
import re
import subprocess
import sys

lib, sub = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", out)
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    if sub not in name:
        continue
    lines = b.split("\n")
    if "--count" in sys.argv:
        pat = re.compile(sys.argv[sys.argv.index("--count") + 1])
        print(name[:90], len([l for l in lines if pat.search(l)]), "of", len(lines))
    elif "--grep" in sys.argv:
        pat = re.compile(sys.argv[sys.argv.index("--grep") + 1])
        print("==", name)
        for l in lines:
            if pat.search(l):
                print(l.strip()[:120])
    else:
        print("==", name)
        print("\n".join(lines))
