"""Attribute ncu SASS-level stall samples to source lines (run here).

    python tools/ncu_lines.py <report.ncu-rep> <kernel-substring> [lib.so]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kname = sys.argv[1], sys.argv[2]
lib = sys.argv[3] if len(sys.argv) > 3 else "paper_2404_06314_b200/_lib/libvqc.so"
column = sys.argv[4] if len(sys.argv) > 4 else "Warp Stall Sampling (All Samples)"
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]
if column == "?":
    print("\n".join(hdr))
    sys.exit(0)
if column not in hdr:  # substring match (e.g. "long_sb")
    column = next(h for h in hdr if column.lower() in h.lower())
samples = {}
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        samples[int(d["Address"], 16)] = (float(d[column] or 0), d["Source"])
    except ValueError:
        pass
if samples:
    base = min(samples)
    samples = {a - base: v for a, v in samples.items()}
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.startswith("engine") and f.endswith(".cubin") and "scheduler" not in f][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
parts = re.split(r"\n\s*\.text\.(\S+):", dis)
addr2line = {}
for i in range(1, len(parts), 2):
    if kname not in parts[i]:
        continue
    cur = None
    for line in parts[i + 1].split("\n"):
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
        if m and cur:
            addr2line[int(m.group(1), 16)] = cur
    break
agg = {}
tot = 0.0
for a, (s, _) in samples.items():
    line = addr2line.get(a, "?")
    agg[line] = agg.get(line, 0.0) + s
    tot += s
src_cache = {}
for line, s in sorted(agg.items(), key=lambda x: -x[1])[:40]:
    f, _, n = line.partition(":")
    text = ""
    for root in ("paper_2404_06314_b200/csrc", "include"):
        p = os.path.join(root, f)
        if os.path.exists(p):
            src_cache.setdefault(p, open(p).read().split("\n"))
            text = src_cache[p][int(n) - 1].strip()[:90] if n.isdigit() else ""
    print(f"{100 * s / tot:5.1f}%  {line:22s} {text}")
