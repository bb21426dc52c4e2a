"""Print the lowered device program of a BASELINE config (CPU, via the test simulator library).

    python tools/dump_program.py --config 3 [--tile 11] [--reg-slots 4]
"""
import argparse
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_06314_b200 import configs  # noqa: E402
from paper_2404_06314_b200.engine import WrtLayout  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--tile", type=int, default=11)
ap.add_argument("--reg-slots", type=int, default=4)
a = ap.parse_args()
so = os.path.join(ROOT, "tests", "native", "_build", "libvqcsim.so")
subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-o", so,
                os.path.join(ROOT, "tests", "native", "program_sim.cpp"),
                os.path.join(ROOT, "paper_2404_06314_b200", "csrc", "scheduler.cpp")], check=True)
lib = ctypes.CDLL(so)
I, F = ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double)
spec = configs.CONFIGS[a.config]
circ, obs, wrt = configs.build(spec, configs.native_api())
c = circ.compiled()
lay = WrtLayout.build(c, wrt)
arrs = [np.ascontiguousarray(x) for x in (c.kinds, c.q0, c.q1, c.coeff, c.f_offs, c.f_idx, lay.wrt_col)]
lib.sim_dump(spec.n, ctypes.c_int64(len(c.kinds)), arrs[0].ctypes.data_as(I), arrs[1].ctypes.data_as(I),
             arrs[2].ctypes.data_as(I), arrs[3].ctypes.data_as(F), arrs[4].ctypes.data_as(I),
             arrs[5].ctypes.data_as(I), ctypes.c_int64(c.total_params), arrs[6].ctypes.data_as(I),
             a.tile, 12, a.reg_slots)
