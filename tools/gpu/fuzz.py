"""Random-circuit fuzz of the default GPU paths against the CPU oracle.

    python tools/gpu/fuzz.py [seconds] [first_seed]
Random gate lists over every gate kind (tests/test_gpu_parity._rand_circuit),
1-15 qubits, Z-only or general Pauli observables (Z-only above 12 qubits),
Jacobian mode; prints the worst relative error per size and fails above 1e-10
(VQC_PRECISION=complex64: 1e-5).
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ.setdefault("VQC_JIT_CACHE", "0")   # every circuit is new anyway

from conftest import close, oracle_batch  # noqa: E402
from test_gpu_parity import _pauli_obs, _rand_circuit, _z_obs  # noqa: E402

from paper_2404_06314_b200 import BatchEngine, BatchRequest  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
prec = os.environ.get("VQC_PRECISION", "complex128")
tol = 1e-10 if prec == "complex128" else 1e-5
eng = BatchEngine(precision=prec)
worst, count = {}, 0
t0 = time.time()
while time.time() - t0 < budget:
    rng = np.random.default_rng(50_000 + seed)
    n = int(rng.integers(1, 16))
    circ, tr = _rand_circuit(rng, n, int(rng.integers(5, 40 + 6 * n)))
    general = n <= 12 and rng.random() < 0.5
    obs = (_pauli_obs if general else _z_obs)(rng, n, int(rng.integers(1, 5)))
    x = rng.uniform(-2, 2, (int(rng.integers(1, 9)), 4))
    wrt = ("a", "b", "s")
    e_ref, j_ref = oracle_batch(circ, obs, tr, x, wrt)
    res = eng.run_batch(BatchRequest(circ, obs, tr, x, wrt=wrt))
    err = max([close(res.expectations, e_ref)] + [close(res.gradients[k], j_ref[k]) for k in wrt])
    worst[n] = max(worst.get(n, 0.0), err)
    if err >= tol:
        print(f"FAIL seed {seed}: n={n} general={general} err={err:.3e}")
        sys.exit(1)
    seed += 1
    count += 1
    eng.plans._plans.clear()   # free the plan (device tables, JIT modules stay cached per source)
print(f"{count} circuits, worst relative error per qubit count:",
      {n: f"{e:.1e}" for n, e in sorted(worst.items())})
