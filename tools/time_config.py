"""Quick device timing of one config (VJP fwd+adjoint) with per-kernel split.

    python tools/time_config.py --config 4 [--rows N] [--reps 3]
Env knobs read by libvqc: VQC_REG_SLOTS, VQC_TILE_QUBITS, VQC_STATE_BUDGET_MB.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_06314_b200 import configs, native  # noqa: E402
from paper_2404_06314_b200.engine import BatchEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
spec = configs.CONFIGS[a.config]
rows = a.rows or spec.batch
circ, obs, wrt = configs.build(spec, configs.native_api())
x, w = configs.inputs_and_weights(spec, batch=rows)
eng = BatchEngine(device="cuda:0", precision=os.environ.get("VQC_PRECISION", "complex128"))
dev = torch.device("cuda:0")
plan, layout = eng.plans.get(circ, obs, wrt, dev)
flat = eng.base_flat(circ, {"w": w})
B, M, C = len(x), len(obs), layout.n_cols
d_x, d_w = torch.from_numpy(x).to(dev), torch.from_numpy(flat).to(dev)
up = torch.ones((B, M), dtype=torch.float64, device=dev)
e = torch.empty((B, M), dtype=torch.float64, device=dev)
vs = torch.empty((C,), dtype=torch.float64, device=dev)
ws = torch.empty(plan.workspace_bytes(B, native.VQC_MODE_VJP), dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
plan.adjoint(d_x, d_w, up, e, None, None, vs, ws, st)
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
native.profile_enable(True)
t0.record()
for _ in range(a.reps):
    plan.adjoint(d_x, d_w, up, e, None, None, vs, ws, st)
t1.record()
torch.cuda.synchronize()
prof = native.profile_report()
ms = t0.elapsed_time(t1) / a.reps
F = configs.flops_per_sample(spec) * B
print(json.dumps({"config": a.config, "rows": B, "ms": round(ms, 3), "samples_per_s": round(B / ms * 1e3, 1),
                  "frac_fp64": round(F / (ms * 1e-3) / 37.1e12, 4), "precision": eng.precision,
                  "env": {k: os.environ.get(k) for k in ("VQC_REG_SLOTS", "VQC_TILE_QUBITS", "VQC_STATE_BUDGET_MB")},
                  "kernels": {k: [round(v[0] / a.reps, 3), v[1] // a.reps] for k, v in prof.items()},
                  "plan": json.loads(plan.describe())}))
