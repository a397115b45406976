"""Dump the SASS of one kernel (substring match) from a .so and count the
instructions of the phase-2 loop (between the VOTE.ANY ... !P0 refill and
its backward branch).  Usage: python tools/sass_loop.py LIB SUBSTR"""
import re
import subprocess
import sys

lib, sub = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", txt)[1:]:
    name = f.split("\n")[0]
    if sub not in name:
        continue
    lines = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", l).strip() for l in f.split("\n")
             if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
    print(name, "total", len(lines))
    out = sys.argv[3] if len(sys.argv) > 3 else None
    if out:
        open(out, "w").write("\n".join(lines))
    from collections import Counter
    ops = Counter(l.split()[1].split(".")[0] if not l.split()[1].startswith("@") else l.split()[2].split(".")[0] for l in lines if len(l.split()) > 1)
    print(ops.most_common(25))
    break
