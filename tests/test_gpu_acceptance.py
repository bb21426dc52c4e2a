"""The reference's acceptance protocols, pointed at the GPU engine.

The reference pins its gradient path with agreement suites run against its
own CPU backends (/root/reference/pkg/tests/test_acceptance.py:57-87, the
50-circuit gradient-oracle suite; test_gradients.py:223-257, three-way
agreement; test_batch.py:107-132, batch invariance and single-row identity;
test_model.py:133-166, VJP == Jacobian slices and the finite-difference
check of the contraction). The same protocols run here through this
package's public API (``gradients``, ``BatchEngine``, ``QuantumModule``) on
libvqc.so, with the reference's tolerances, plus a 1e-10 comparison of every
adjoint result with the CPU oracle.
"""

import numpy as np
import pytest

from conftest import close, oracle_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    return "cuda:0"


def _z_obs(n, count):
    from paper_2404_06314_b200.observables import parse_observable
    return [parse_observable("".join("Z" if q == i % n else "I" for q in range(n)))
            for i in range(count)]


def _reuploading(rng, n, d, m):
    """Re-uploading ansatz with n - 1 features (encoding angles lambda*s,
    s shared across layers) and M single-Z observables."""
    from paper_2404_06314_b200.ir import build_reuploading_ansatz
    circ = build_reuploading_ansatz(n, d, num_features=max(1, n - 1))
    binding = {"s": rng.uniform(-1.0, 1.0, circ.set_named("s").size),
               "theta": rng.uniform(0.0, 2 * np.pi, circ.set_named("theta").size),
               "lambda": rng.uniform(0.5, 1.5, circ.set_named("lambda").size)}
    return circ, binding, _z_obs(n, m)


def _oracle_single(circ, binding, obs, wrt):
    """Oracle Jacobian for one full binding (encoding row = binding['s'])."""
    trainable = {k: v for k, v in binding.items() if k != "s"}
    e, jac = oracle_batch(circ, obs, trainable, binding["s"][None, :], wrt)
    return e[0], {k: v[0] for k, v in jac.items()}


def test_gradient_oracle_suite_50_circuits(cuda):
    """adjoint == param-shift (1e-9), both == finite differences (1e-5) over
    50 random re-uploading circuits, n in [2, 8], d in [1, 4], M in [1, 8];
    adjoint == CPU oracle at 1e-10."""
    from paper_2404_06314_b200 import gradients as G
    from paper_2404_06314_b200.engine import BatchEngine
    eng = BatchEngine(device=cuda)
    rng = np.random.default_rng(1234)
    wrt = ("theta", "lambda", "s")
    worst = {"shift": 0.0, "fd": 0.0, "oracle": 0.0}
    for case in range(50):
        n, d, m = int(rng.integers(2, 9)), int(rng.integers(1, 5)), int(rng.integers(1, 9))
        circ, binding, obs = _reuploading(rng, n, d, m)
        adj = G.adjoint_gradients(circ, binding, obs, wrt, engine=eng)
        shift = G.parameter_shift_gradients(circ, binding, obs, wrt, engine=eng)
        fd = G.finite_difference_gradients(circ, binding, obs, wrt, h=1e-4, engine=eng)
        e_ref, j_ref = _oracle_single(circ, binding, obs, wrt)
        worst["oracle"] = max(worst["oracle"], close(adj.expectations, e_ref))
        for k in wrt:
            worst["shift"] = max(worst["shift"], np.abs(adj.gradients[k] - shift.gradients[k]).max())
            worst["fd"] = max(worst["fd"], np.abs(adj.gradients[k] - fd.gradients[k]).max(),
                              np.abs(shift.gradients[k] - fd.gradients[k]).max())
            worst["oracle"] = max(worst["oracle"], close(adj.gradients[k], j_ref[k]))
        assert worst["shift"] <= 1e-9, (case, worst)
        assert worst["fd"] <= 1e-5, (case, worst)
        assert worst["oracle"] <= 1e-10, (case, worst)


def test_three_way_agreement_general_observables(cuda):
    """Random gate mixes (every reference gate kind, 0-2 factor expressions,
    shared references) with general X/Y/Z observables, n in [2, 3]."""
    from test_basis_groups import _random

    from paper_2404_06314_b200 import gradients as G
    from paper_2404_06314_b200.engine import BatchEngine
    eng = BatchEngine(device=cuda)
    for seed in range(15):
        n = 2 + seed % 2
        circ, obs, w, x = _random(100 + seed, n, n_gates=2 + seed)
        binding = {"s": x[0], "w": w}
        wrt = ("w", "s")
        adj = G.adjoint_gradients(circ, binding, obs, wrt, engine=eng)
        shift = G.parameter_shift_gradients(circ, binding, obs, wrt, engine=eng)
        fd = G.finite_difference_gradients(circ, binding, obs, wrt, engine=eng)
        for k in wrt:
            assert np.abs(adj.gradients[k] - shift.gradients[k]).max(initial=0.0) <= 1e-9
            assert np.abs(adj.gradients[k] - fd.gradients[k]).max(initial=0.0) <= 1e-5


def test_analytic_anchors(cuda):
    """<Z> = cos(theta), d<Z>/dtheta = -sin(theta) for RX(theta)|0> at four
    angles, adjoint and param-shift, 1e-12."""
    from paper_2404_06314_b200 import gradients as G
    from paper_2404_06314_b200.engine import BatchEngine
    from paper_2404_06314_b200.ir import AngleExpression, Circuit, Gate, GateKind, ParameterSet
    eng = BatchEngine(device=cuda)
    circ = Circuit(1, (Gate(GateKind.RX, (0,), AngleExpression(1.0, (("theta", 0),))),),
                   (ParameterSet("theta", 1),))
    z = _z_obs(1, 1)
    for theta in (0.0, 0.3, np.pi / 2, np.pi):
        for fn in (G.adjoint_gradients, G.parameter_shift_gradients):
            r = fn(circ, {"theta": np.array([theta])}, z, ["theta"], engine=eng)
            assert abs(r.expectations[0] - np.cos(theta)) <= 1e-12
            assert abs(r.gradients["theta"][0, 0] + np.sin(theta)) <= 1e-12


def test_batch_rows_independent_and_single_row_identity(cuda):
    """Each row of a batch equals the same row run alone (bitwise) and the
    single-binding adjoint call on that row (1e-12), for every method."""
    from paper_2404_06314_b200 import gradients as G
    from paper_2404_06314_b200.engine import BatchEngine, BatchRequest
    eng = BatchEngine(device=cuda)
    rng = np.random.default_rng(7)
    circ, binding, obs = _reuploading(rng, 5, 2, 3)
    trainable = {k: v for k, v in binding.items() if k != "s"}
    x = rng.uniform(-1, 1, (6, circ.set_named("s").size))
    wrt = ("theta", "lambda", "s")
    for method in ("adjoint", "param-shift", "spsa"):
        full = eng.run_batch(BatchRequest(circ, obs, trainable, x, method=method, wrt=wrt, seed=9))
        for b in (0, 5):
            one = eng.run_batch(BatchRequest(circ, obs, trainable, x[b:b + 1], method=method,
                                             wrt=wrt, seed=9, row_offset=b))
            assert np.array_equal(one.expectations[0], full.expectations[b])
            for k in wrt:
                assert np.array_equal(one.gradients[k][0], full.gradients[k][b])
    full = eng.run_batch(BatchRequest(circ, obs, trainable, x, wrt=wrt))
    direct = G.adjoint_gradients(circ, dict(trainable, s=x[0]), obs, wrt, engine=eng)
    assert close(full.expectations[0], direct.expectations) <= 1e-12
    for k in wrt:
        assert close(full.gradients[k][0], direct.gradients[k]) <= 1e-12


def test_module_vjp_equals_jacobian_slices_and_fd(cuda):
    """QuantumModule.backward with a one-hot upstream equals the matching
    Jacobian slice (1e-14 abs in the reference; 1e-12 here: the VJP seeds one
    combined bra), and a random-upstream contraction matches central
    differences of sum(upstream * forward) (1e-4)."""
    import torch

    from paper_2404_06314_b200.ir import build_reuploading_ansatz
    from paper_2404_06314_b200.module import QuantumModule
    rng = np.random.default_rng(3)
    circ = build_reuploading_ansatz(3, 1, num_features=3)
    mod = QuantumModule(circ, _z_obs(3, 2), "s", ["theta", "lambda"], seed=1, device=cuda)
    x = rng.uniform(-1, 1, (2, 3))
    full = mod.jacobians(x)
    for b in range(2):
        for i in range(2):
            up = np.zeros((2, 2))
            up[b, i] = 1.0
            g = mod.backward(x, up)
            for k in ("theta", "lambda"):
                assert np.abs(g[k] - full.gradients[k][b, i]).max() <= 1e-12
    x4 = rng.uniform(-1, 1, (4, 3))
    up = rng.normal(size=(4, 2))
    g = mod.backward(x4, up)
    h = 1e-5

    def loss():
        with torch.no_grad():
            return float(np.sum(up * mod(x4).cpu().numpy()))

    for k in ("theta", "lambda"):
        p = mod.values[k]
        for j in range(p.numel()):
            old = float(p[j])
            with torch.no_grad():
                p[j] = old + h
            fp = loss()
            with torch.no_grad():
                p[j] = old - h
            fm = loss()
            with torch.no_grad():
                p[j] = old
            assert abs(g[k][j] - (fp - fm) / (2 * h)) <= 1e-4
