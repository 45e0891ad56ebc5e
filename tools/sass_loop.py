"""Instruction mix of the hottest loop (smallest backward-branch loop with
>= 64 FFMA2) of one kernel in the built library: python tools/sass_loop.py <mangled-substring>"""
import collections
import re
import subprocess
import sys

lib = sys.argv[2] if len(sys.argv) > 2 else "paper_1409_7474_b200/_lib/liblse_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
f, body = False, []
for line in sass.split("\n"):
    if "Function : " in line:
        f = sys.argv[1] in line
        continue
    if f:
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            body.append((int(m.group(1), 16), m.group(2).strip()))
best = None
for a, t in body:
    m = re.search(r"BRA (0x[0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        loop = [x for x in body if int(m.group(1), 16) <= x[0] <= a]
        n2 = sum("FFMA2" in x[1] for x in loop)
        if n2 >= 64 and (best is None or len(loop) < len(best[1])):
            best = (n2, loop)
if best:
    c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for _, t in best[1])
    print(len(best[1]), "instructions in the loop")
    for k, v in c.most_common(30):
        print(f"{v:5d} {k}")
spills = sum(1 for _, t in body if t.startswith(("STL", "LDL")) or " STL" in t or " LDL" in t)
print("local ld/st instructions in the function:", spills)
