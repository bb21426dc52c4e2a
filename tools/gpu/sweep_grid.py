"""Qubits x depth sweep of the GPU module (forward + backward device time), CSV
with the reference's columns plus samples/s; the headline metric's axes.

    python tools/gpu/sweep_grid.py gpurun_out/sweep_grid.csv
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_06314_b200.sweep import run_sweep, write_csv  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep_grid.csv"
pts = []
# batch sized so every point moves a comparable number of amplitudes
for q, batch in ((4, 16384), (6, 16384), (8, 16384), (10, 8192), (12, 4096), (14, 2048), (16, 1024), (18, 256), (20, 64)):
    pts += run_sweep([q], [2, 4, 8], [batch], repeats=3, device="cuda:0")

for p in pts:
    print(p.qubits, p.depth, p.batch, f"{p.batch / p.total[0]:.4g} samples/s", f"fwd {p.forward[0]*1e3:.3f} ms bwd {p.backward[0]*1e3:.3f} ms")
write_csv(pts, out, seed=0, note="B200, device-timed forward + backward of QuantumModule (reuploading ansatz, per-qubit <Z>), tools/gpu/sweep_grid.py")
