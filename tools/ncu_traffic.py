"""Summarise an ncu --csv launch list (gpu__time_duration.sum and optionally
dram__bytes_read.sum / dram__bytes_write.sum) per kernel class.

    python tools/ncu_traffic.py launches.csv [--rows R] [--out traffic.json]

Kernel classes: vqc_jit_pf* / k_pass<.,0> -> pass_forward, vqc_jit_pa* /
k_pass<.,2> -> pass_adjoint, k_smem / vqc_jit_s* -> smem, others by name.
"""
import argparse
import csv
import io
import json
import re

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--out", default="")
a = ap.parse_args()
text = open(a.csv).read()
start = text.find('"ID"')
rows = list(csv.reader(io.StringIO(text[start:])))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
idi = hdr.index("ID")


def klass(name: str) -> str:
    if name.startswith("vqc_jit_pf") or re.search(r"k_pass<\d+, 0>", name):
        return "pass_forward"
    if name.startswith("vqc_jit_pa") or re.search(r"k_pass<\d+, 2>", name):
        return "pass_adjoint"
    if name.startswith("vqc_jit_s") or "k_smem" in name:
        return "smem_fwd_adjoint"
    m = re.search(r"vqc::(\w+)", name)
    return m.group(1) if m else name.split("(")[0][:40]


launch = {}
for r in rows[1:]:
    if len(r) <= vi:
        continue
    d = launch.setdefault(r[idi], {"kernel": r[ki]})
    try:
        d[r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:
        pass
agg = {}
for d in launch.values():
    c = klass(d["kernel"])
    g = agg.setdefault(c, {"launches": 0, "time_ns": 0.0, "dram_bytes": 0.0})
    g["launches"] += 1
    g["time_ns"] += d.get("gpu__time_duration.sum", 0.0)
    g["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot_t = sum(g["time_ns"] for g in agg.values()) or 1.0
out = {"source": a.csv, "rows": a.rows, "kernels": {}}
for c, g in sorted(agg.items(), key=lambda x: -x[1]["time_ns"]):
    e = {"launches": g["launches"], "share": g["time_ns"] / tot_t, "avg_us": g["time_ns"] / g["launches"] / 1e3}
    if g["dram_bytes"] > 0:
        e["dram_bytes_per_launch"] = g["dram_bytes"] / g["launches"]
        e["dram_gbs"] = g["dram_bytes"] / g["time_ns"]
        if a.rows:
            e["dram_bytes_per_sample"] = g["dram_bytes"] / a.rows
    out["kernels"][c] = e
    print(f"{c:22s} launches {g['launches']:5d} share {e['share']:.3f} avg {e['avg_us']:9.1f} us"
          + (f"  dram/launch {e.get('dram_bytes_per_launch', 0)/1e6:8.1f} MB  {e.get('dram_gbs', 0):7.1f} GB/s" if g["dram_bytes"] else ""))
if a.out:
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
