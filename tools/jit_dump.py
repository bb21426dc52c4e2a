"""Dump / compile (CPU-side, NVRTC) the JIT source a plan would build.

    python tools/jit_dump.py --config 4 [--compile] [--out /tmp/cfg4.cu]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2404_06314_b200 import configs, native  # noqa: E402
from paper_2404_06314_b200.engine import WrtLayout, encoding_set  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--compile", action="store_true")
ap.add_argument("--out", default="")
a = ap.parse_args()
spec = configs.CONFIGS[a.config]
circ, obs, wrt = configs.build(spec, configs.native_api())
compiled = circ.compiled()
layout = WrtLayout.build(compiled, wrt)
off, size = compiled.offsets[encoding_set(circ).name]
src, secs = native.jit_source(compiled, layout.wrt_col, off, size, compile=a.compile)
if a.out:
    with open(a.out, "w") as fh:
        fh.write(src)
print(f"cfg{a.config}: source {len(src)} bytes, {src.count(chr(10))} lines"
      + (f", NVRTC compile {secs:.2f} s" if secs is not None else ""))
