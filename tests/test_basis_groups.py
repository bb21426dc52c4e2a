"""General X/Y Pauli observables on HBM plans (n > 12) via per-pattern basis
rotation (engine.basis_groups / basis_circuit).

CPU: the identity <psi|P|psi> = Sum_groups <U_g psi| Z_g |U_g psi> and the
matching Jacobians are checked with the oracle (which evaluates general Pauli
strings directly, _kernels.py:155-217) on random circuits and observables.
GPU: run_batch on 13- and 14-qubit circuits with X/Y observables vs the oracle.
"""

import numpy as np
import pytest

from conftest import close, oracle_batch

TOL = 1e-10


def _random(seed, n, n_gates=40):
    from paper_2404_06314_b200.ir import AngleExpression, Circuit, Gate, GateKind, ParameterSet
    from paper_2404_06314_b200.observables import Observable
    rng = np.random.default_rng(seed)
    sets = (ParameterSet("s", 3, "encoding"), ParameterSet("w", 5, "trainable"))
    pool = [("s", i) for i in range(3)] + [("w", i) for i in range(5)]
    gates = []
    for _ in range(n_gates):
        k = int(rng.integers(5))
        if k < 3:
            refs = [pool[int(rng.integers(len(pool)))]]
            gates.append(Gate(GateKind(k), (int(rng.integers(n)),),
                              AngleExpression(float(rng.uniform(-2, 2)), tuple(refs))))
        elif k == 3:
            a, b = rng.permutation(n)[:2]
            gates.append(Gate(GateKind.CNOT, (int(a), int(b))))
        else:
            gates.append(Gate(GateKind.H, (int(rng.integers(n)),)))
    circ = Circuit(n, tuple(gates), sets)
    obs = []
    for _ in range(3):
        terms = tuple((float(rng.uniform(-2, 2)),
                       "".join("IXYZ"[int(rng.integers(4))] for _ in range(n)))
                      for _ in range(int(rng.integers(1, 4))))
        obs.append(Observable(terms))
    w = rng.uniform(-1.5, 1.5, 5)
    x = rng.uniform(-1.5, 1.5, (4, 3))
    return circ, obs, w, x


def test_basis_groups_partition_terms():
    from paper_2404_06314_b200.engine import basis_groups
    from paper_2404_06314_b200.observables import Observable
    obs = [Observable(((1.0, "XZI"), (2.0, "ZZI"))), Observable(((3.0, "IYX"),))]
    groups = dict(basis_groups(obs, 3))
    assert set(groups) == {"X--", "---", "-YX"}
    assert groups["X--"][0].terms == ((1.0, "ZZI"),)
    assert groups["X--"][1].terms == ((0.0, "III"),)
    assert groups["-YX"][1].terms == ((3.0, "IZZ"),)
    assert all(o.is_z_only for _, g in groups.items() for o in g)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_basis_rotation_identity_with_oracle(oracle_mod, seed):
    from paper_2404_06314_b200.engine import basis_circuit, basis_groups
    circ, obs, w, x = _random(seed, 4)
    e_ref, j_ref = oracle_batch(circ, obs, {"w": w}, x, ("w", "s"))
    e_sum = np.zeros_like(e_ref)
    j_sum = {k: np.zeros_like(v) for k, v in j_ref.items()}
    for pattern, group in basis_groups(obs, 4):
        e, j = oracle_batch(basis_circuit(circ, pattern), group, {"w": w}, x, ("w", "s"))
        e_sum += e
        for k in j_sum:
            j_sum[k] += j[k]
    assert close(e_sum, e_ref) < TOL
    for k in j_ref:
        assert close(j_sum[k], j_ref[k]) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("n,seed", [(13, 0), (14, 1)])
def test_gpu_xy_observables_on_hbm_plans(n, seed):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200.engine import BatchEngine, BatchRequest
    circ, obs, w, x = _random(seed, n, n_gates=60)
    e_ref, j_ref = oracle_batch(circ, obs, {"w": w}, x, ("w", "s"))
    res = BatchEngine(device="cuda:0").run_batch(
        BatchRequest(circ, obs, {"w": w}, x, wrt=("w", "s")))
    assert close(res.expectations, e_ref) < TOL
    for k in j_ref:
        assert close(res.gradients[k], j_ref[k]) < TOL
    fwd = BatchEngine(device="cuda:0").run_batch(BatchRequest(circ, obs, {"w": w}, x))
    assert close(fwd.expectations, e_ref) < TOL


@pytest.mark.gpu
def test_gpu_module_autograd_xy_on_hbm_plans():
    """QuantumModule.forward / autograd and .backward with X/Y observables at
    n = 13: per-group QuantumFunction nodes summed, vs the oracle."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200.module import QuantumModule
    circ, obs, w, x = _random(2, 13, n_gates=50)
    mod = QuantumModule(circ, obs, "s", ["w"], seed=0, device="cuda:0")
    with torch.no_grad():
        mod.values["w"].copy_(torch.from_numpy(w))
    xt = torch.from_numpy(x).cuda().requires_grad_(True)
    out = mod(xt)
    up = np.random.default_rng(1).normal(size=out.shape)
    out.backward(torch.from_numpy(up).cuda())
    e_ref, j_ref = oracle_batch(circ, obs, {"w": w}, x, ("w", "s"))
    assert close(out.detach().cpu().numpy(), e_ref) < TOL
    assert close(mod.values["w"].grad.cpu().numpy(), np.einsum("bm,bmp->p", up, j_ref["w"])) < TOL
    assert close(xt.grad.cpu().numpy(), np.einsum("bm,bmf->bf", up, j_ref["s"])) < TOL
    vjp = mod.backward(x, up)
    assert close(vjp["w"], np.einsum("bm,bmp->p", up, j_ref["w"])) < TOL
