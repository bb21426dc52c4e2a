import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_06314_b200.sweep import run_sweep  # noqa: E402
for q, b in ((4, 16384), (8, 16384), (10, 8192), (12, 4096)):
    for p in run_sweep([q], [8], [b], repeats=3, device="cuda:0"):
        print(p.qubits, p.depth, p.batch, f"{p.batch / p.total[0]:.4g} samples/s", f"fwd {p.forward[0]*1e3:.3f} ms bwd {p.backward[0]*1e3:.3f} ms")
