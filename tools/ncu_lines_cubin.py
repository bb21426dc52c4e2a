"""Attribute ncu SASS stall samples of a JIT kernel to source lines using the
cached cubin (line info from NVRTC -lineinfo).

    python tools/ncu_lines_cubin.py <sass.csv> <cubin> <kernel-name> [column]
"""
import collections
import csv
import re
import subprocess
import sys

sass_csv, cubin, kname = sys.argv[1], sys.argv[2], sys.argv[3]
column = sys.argv[4] if len(sys.argv) > 4 else "Warp Stall Sampling (All Samples)"
rows = list(csv.reader(open(sass_csv)))
hdr, body = None, []
for r in rows:
    if r and r[0] == "Kernel Name":
        if hdr:
            break
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr:
        body.append(r)
ci, ai, ei = hdr.index(column), hdr.index("Address"), hdr.index("Instructions Executed")
samples = {}
for r in body:
    try:
        samples[int(r[ai], 16)] = (float(r[ci] or 0), float(r[ei] or 0))
    except ValueError:
        pass
base = min(samples)
dis = subprocess.run(["nvdisasm", "-g", "-fun", kname, cubin], capture_output=True, text=True).stdout
if not dis:
    dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
    parts = re.split(r"\n\s*\.text\.(\S+):", dis)
    dis = next(parts[i + 1] for i in range(1, len(parts), 2) if parts[i] == kname)
cur, a2l = None, {}
for line in dis.split("\n"):
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m and cur:
        a2l[int(m.group(1), 16)] = cur
agg, ex = collections.Counter(), collections.Counter()
tot = sum(v[0] for v in samples.values()) or 1.0
etot = sum(v[1] for v in samples.values()) or 1.0
for a, (s, e) in samples.items():
    ln = a2l.get(a - base, "?")
    agg[ln] += s
    ex[ln] += e
for ln, s in agg.most_common(40):
    print(f"{s / tot * 100:5.1f}% stall {ex[ln] / etot * 100:5.1f}% exec  {ln}")
