"""Run one config's fwd+adjoint (VJP) a few times — a short command for ncu.

    python tools/profile_one.py --config 3 --rows 512 --reps 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_06314_b200 import configs, native  # noqa: E402
from paper_2404_06314_b200.engine import BatchEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--rows", type=int, default=512)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--mode", default="vjp", choices=("vjp", "jacobian", "forward"))
a = ap.parse_args()
spec = configs.CONFIGS[a.config]
circ, obs, wrt = configs.build(spec, configs.native_api())
x, w = configs.inputs_and_weights(spec, batch=a.rows)
eng = BatchEngine(device="cuda:0")
dev = torch.device("cuda:0")
plan, layout = eng.plans.get(circ, obs, wrt, dev)
flat = eng.base_flat(circ, {"w": w})
B, M, C = len(x), len(obs), layout.n_cols
d_x = torch.from_numpy(x).to(dev)
d_w = torch.from_numpy(flat).to(dev)
up = torch.ones((B, M), dtype=torch.float64, device=dev)
e = torch.empty((B, M), dtype=torch.float64, device=dev)
rows = torch.empty((B, C), dtype=torch.float64, device=dev)
vs = torch.empty((C,), dtype=torch.float64, device=dev)
jac = torch.empty((B, M, C), dtype=torch.float64, device=dev)
mode = {"vjp": native.VQC_MODE_VJP, "jacobian": native.VQC_MODE_JACOBIAN,
        "forward": native.VQC_MODE_FORWARD}[a.mode]
ws = torch.empty(max(1, plan.workspace_bytes(B, mode)), dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
for _ in range(a.reps):
    if a.mode == "vjp":
        plan.adjoint(d_x, d_w, up, e, None, rows, vs, ws, st)
    elif a.mode == "jacobian":
        plan.adjoint(d_x, d_w, None, e, jac, None, None, ws, st)
    else:
        plan.forward(d_x, d_w, e, ws, st)
torch.cuda.synchronize()
print(plan.describe(), float(e.sum()))
