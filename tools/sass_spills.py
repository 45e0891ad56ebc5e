"""List the local-memory (STL/LDL) instructions of one kernel in the built
library with the source line each belongs to (static view; pair with ncu's
per-instruction execution counts to see which ones run per unit)."""
import re
import subprocess
import sys
import tempfile

import os
lib = os.path.abspath(sys.argv[1])
fn = sys.argv[2]                     # mangled-name substring
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=d, check=True, capture_output=True)
    import glob
    cub = glob.glob(f"{d}/*.cubin")[0]
    out = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if ".section" in l and ".text." in l and fn in l)
end = next(i for i in range(start + 1, len(lines)) if ".section" in lines[i])
cur = ""
for l in lines[start:end]:
    m = re.search(r'line (\d+)', l)
    if l.strip().startswith("//## File"):
        cur = " <- ".join(re.findall(r'line (\d+)', l))
        continue
    if re.search(r'\b(STL|LDL)', l):
        addr = re.search(r'/\*([0-9a-f]+)\*/', l).group(1)
        print(f"{addr:>6s}  {l.split('*/')[-1].strip():40s}  {cur}")
