"""Small workloads for compute-sanitizer (one tool per gpurun call):

    compute-sanitizer --tool memcheck  python tools/sanitize_case.py
    compute-sanitizer --tool racecheck python tools/sanitize_case.py

Covers the on-chip JIT kernel (cfg2, VJP and Jacobian modes), the
interpreter kernels (VQC_JIT=0 in a second plan set), and a 13-qubit HBM
plan (ping-pong JIT pass kernels, forward + VJP adjoint) in complex128 and
complex64. Rows are few: the tools slow kernels down by orders of magnitude.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_06314_b200 import configs  # noqa: E402
from paper_2404_06314_b200.engine import BatchEngine, BatchRequest  # noqa: E402


def run(eng, circ, obs, w, x, wrt):
    r = eng.run_batch(BatchRequest(circ, obs, w, x, wrt=wrt))
    f = eng.run_batch(BatchRequest(circ, obs, w, x))
    return float(np.abs(r.expectations - f.expectations).max())


def main():
    dev = "cuda:0"
    out = {}
    spec = configs.CONFIGS[2]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=int(os.environ.get("SAN_ROWS", "8")))
    out["cfg2"] = run(BatchEngine(device=dev), circ, obs, {"w": w}, x, wrt)
    # VJP through the module (the autograd path)
    from paper_2404_06314_b200.module import QuantumModule
    mod = QuantumModule(circ, obs, "x", ["w"], device=dev)
    xt = torch.from_numpy(x).to(dev).requires_grad_(True)
    mod(xt).sum().backward()
    # 13-qubit HBM plan (random circuit with every gate kind)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    from test_gpu_parity import _rand_circuit, _z_obs
    rng = np.random.default_rng(13)
    c13, tr = _rand_circuit(rng, 13, 60)
    o13 = _z_obs(rng, 13, 2)
    x13 = rng.uniform(-2, 2, (2, 4))
    for prec in ("complex128", "complex64"):
        out["n13_" + prec] = run(BatchEngine(device=dev, precision=prec), c13, o13, tr, x13, ("a", "b", "s"))
    torch.cuda.synchronize()
    print(out)


if __name__ == "__main__":
    main()
