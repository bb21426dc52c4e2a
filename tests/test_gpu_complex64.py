"""complex64 mode (north star: "1e-5 for an optional complex64 mode").

Plans created with precision "complex64" evolve single-precision states in
JIT kernels built with VQC_C64; angles, fused-block matrices, inner-product
reductions, expectations and gradients stay float64. Every check compares
with the complex128 reference results (goldens made by the reference
itself, or the oracle pinned to them) at |gpu - ref| <= 1e-5 * max(1, |ref|).
"""

import ast
import os

import numpy as np
import pytest

from conftest import GOLDEN, close, oracle_batch

pytestmark = pytest.mark.gpu
TOL64 = 1e-5


@pytest.fixture(scope="module")
def eng():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200.engine import BatchEngine
    return BatchEngine(device="cuda:0", precision="complex64")


def _req(circ, obs, w, x, wrt):
    from paper_2404_06314_b200.engine import BatchRequest
    return BatchRequest(circ, obs, w, x, wrt=wrt)


@pytest.mark.parametrize("cfg_id", [1, 2, 3, 4, 5])
def test_configs_vs_reference_goldens(eng, cfg_id):
    """Expectations, Jacobians (run_batch) and the VJP (upstream = ones) on
    the golden rows of every BASELINE config."""
    import torch

    from paper_2404_06314_b200 import configs, native
    g = np.load(os.path.join(GOLDEN, f"cfg{cfg_id}.npz"))
    spec = configs.CONFIGS[cfg_id]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x = g["x_rows"]
    res = eng.run_batch(_req(circ, obs, {"w": g["w"]}, x, wrt))
    assert close(res.expectations, g["expect"]) < TOL64
    assert close(res.gradients["w"], g["jac_w"]) < TOL64
    if "jac_x" in g.files:
        assert close(res.gradients["x"], g["jac_x"]) < TOL64
    plan, layout = eng.plans.get(circ, obs, wrt, eng.device)
    assert '"precision": "complex64"' in plan.describe()
    dev = eng.device
    B, M = len(x), len(obs)
    flat = eng.base_flat(circ, {"w": g["w"]})
    rows = torch.empty((B, layout.n_cols), dtype=torch.float64, device=dev)
    vsum = torch.empty((layout.n_cols,), dtype=torch.float64, device=dev)
    ws = torch.empty(plan.workspace_bytes(B, native.VQC_MODE_VJP), dtype=torch.uint8, device=dev)
    plan.adjoint(torch.from_numpy(x).to(dev), torch.from_numpy(flat).to(dev),
                 torch.ones((B, M), dtype=torch.float64, device=dev), None, None, rows, vsum, ws,
                 torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    P = spec.num_weights
    assert close(vsum.cpu().numpy()[:P], g["vjp_w"]) < TOL64 * max(1.0, B / 8)
    if "vjp_x_rows" in g.files:
        assert close(rows.cpu().numpy()[:, P:], g["vjp_x_rows"]) < TOL64


def _random_cases():
    path = os.path.join(GOLDEN, "random.npz")
    return list(range(int(np.load(path)["count"]))) if os.path.exists(path) else []


@pytest.mark.parametrize("idx", _random_cases()[::3])
def test_random_circuits_vs_reference(eng, idx):
    """Reference-generated random circuits (every gate kind, products of
    parameters, Z and general X/Y/Z Pauli sums)."""
    from paper_2404_06314_b200 import ir
    from paper_2404_06314_b200.observables import Observable
    g = np.load(os.path.join(GOLDEN, "random.npz"))
    p = f"c{idx}_"
    circ = ir.circuit_from_dict(ast.literal_eval(str(g[p + "doc"])))
    obs = [Observable(t) for t in ast.literal_eval(str(g[p + "obs"]))]
    trainable = {"theta": g[p + "theta"], "lam": g[p + "lam"]}
    res = eng.run_batch(_req(circ, obs, trainable, g[p + "inputs"], ("theta", "lam", "s")))
    assert close(res.expectations, g[p + "expect"]) < TOL64
    for name in ("theta", "lam", "s"):
        assert close(res.gradients[name], g[p + "jac_" + name]) < TOL64


@pytest.mark.parametrize("n", [1, 4, 9, 12, 13, 15])
def test_random_with_cz_vs_oracle(eng, n):
    from test_gpu_parity import _rand_circuit, _z_obs
    rng = np.random.default_rng(700 + n)
    circ, trainable = _rand_circuit(rng, n, 30 + 4 * n)
    obs = _z_obs(rng, n, 3)
    x = rng.uniform(-2, 2, (5, 4))
    wrt = ("a", "b", "s")
    e_ref, j_ref = oracle_batch(circ, obs, trainable, x, wrt)
    res = eng.run_batch(_req(circ, obs, trainable, x, wrt))
    assert close(res.expectations, e_ref) < TOL64
    for k in wrt:
        assert close(res.gradients[k], j_ref[k]) < TOL64


def test_module_autograd_and_degenerate(eng):
    """QuantumModule(precision='complex64') autograd vs the oracle; an empty
    circuit and an empty batch keep their shapes."""
    import torch

    from paper_2404_06314_b200 import configs
    from paper_2404_06314_b200.ir import Circuit, ParameterSet
    from paper_2404_06314_b200.module import QuantumModule
    from paper_2404_06314_b200.observables import parse_observable
    spec = configs.CONFIGS[2]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=48)
    mod = QuantumModule(circ, obs, "x", ["w"], device="cuda:0", precision="complex64")
    with torch.no_grad():
        mod.values["w"].copy_(torch.from_numpy(w))
    xt = torch.from_numpy(x).to("cuda:0").requires_grad_(True)
    up = np.random.default_rng(0).normal(size=(48, len(obs)))
    out = mod(xt)
    out.backward(torch.from_numpy(up).to("cuda:0"))
    e_ref, j_ref = oracle_batch(circ, obs, {"w": w}, x, ("w", "x"))
    assert close(out.detach().cpu().numpy(), e_ref) < TOL64
    assert close(mod.values["w"].grad.cpu().numpy(), np.einsum("bm,bmp->p", up, j_ref["w"])) < 48 * TOL64
    assert close(xt.grad.cpu().numpy(), np.einsum("bm,bmf->bf", up, j_ref["x"])) < TOL64
    empty = Circuit(3, (), (ParameterSet("s", 2, "encoding"),))
    r = eng.run_batch(_req(empty, [parse_observable("ZII"), parse_observable("IIZ")], {},
                           np.zeros((3, 2)), ("s",)))
    assert np.array_equal(r.expectations, np.ones((3, 2)))
    assert r.gradients["s"].shape == (3, 2, 2) and not r.gradients["s"].any()
    r0 = eng.run_batch(_req(circ, obs, {"w": w}, np.zeros((0, spec.n)), wrt))
    assert r0.expectations.shape == (0, len(obs))
