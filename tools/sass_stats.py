"""Per-kernel SASS statistics of libvqc.so (run here, no GPU):
local-memory traffic (spills), FP64 ops, shuffles, shared-memory ops."""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2404_06314_b200/_lib/libvqc.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)[1:]
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    ops = Counter()
    for line in f.split("\n"):
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
        if m:
            ops[m.group(2)] += 1
    total = sum(ops.values())
    keys = ["DFMA", "DMUL", "DADD", "LDS", "STS", "LDL", "STL", "LDG", "STG", "SHFL", "BRX", "BAR"]
    print(f"{name[:60]:60s} total={total:6d} " + " ".join(f"{k}={ops.get(k, 0)}" for k in keys))
