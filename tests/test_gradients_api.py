"""Single-binding gradient API (reference gradients.py:204-283) on the GPU
engine vs the oracle; tolerances follow the reference's agreement suite
(test_gradients.py:223-257: shift vs adjoint 1e-9, FD 1e-5)."""

import numpy as np
import pytest

from conftest import close, lowered

TOL = 1e-10


def _case(seed=0, n=4):
    from test_basis_groups import _random
    circ, obs, w, x = _random(seed, n)
    return circ, obs, {"s": x[0], "w": w}


def _oracle(oracle_mod, circ, obs, binding, wrt):
    from paper_2404_06314_b200.engine import WrtLayout
    comp = circ.compiled()
    layout = WrtLayout.build(comp, wrt)
    flat = comp.flat_values(binding)
    e, j = oracle_mod.run_batch(lowered(circ, obs), flat, 0, 0, np.zeros((1, 0)), layout.wrt_col)
    return e[0], j[0], layout, flat


def test_argument_validation():
    from paper_2404_06314_b200 import gradients as G
    circ, obs, b = _case()
    with pytest.raises(ValueError, match="c must be > 0"):
        G.spsa_gradients(circ, b, obs, ("w",), c=0.0)
    with pytest.raises(ValueError, match="samples must be >= 1"):
        G.spsa_gradients(circ, b, obs, ("w",), samples=0)
    with pytest.raises(ValueError, match="step h must be > 0"):
        G.finite_difference_gradients(circ, b, obs, ("w",), h=-1.0)
    with pytest.raises(ValueError, match="binding does not match"):
        G.adjoint_gradients(circ, {"w": b["w"]}, obs, ("w",))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1])
def test_gpu_single_binding_methods(oracle_mod, seed):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200 import gradients as G
    circ, obs, b = _case(seed)
    wrt = ("w", "s")
    e_ref, j_ref, layout, flat = _oracle(oracle_mod, circ, obs, b, wrt)
    split = lambda j: {n: j[:, lo:hi] for n, lo, hi in layout.slices}  # noqa: E731
    adj = G.adjoint_gradients(circ, b, obs, wrt)
    assert close(adj.expectations, e_ref) < TOL
    for k, v in split(j_ref).items():
        assert close(adj.gradients[k], v) < TOL
    ps = G.parameter_shift_gradients(circ, b, obs, wrt)
    for k, v in split(j_ref).items():
        assert np.abs(ps.gradients[k] - v).max() < 1e-9
    fd = G.finite_difference_gradients(circ, b, obs, wrt)
    for k, v in split(j_ref).items():
        assert np.abs(fd.gradients[k] - v).max() < 1e-5
    sp = G.spsa_gradients(circ, b, obs, wrt, c=0.01, samples=3, seed=7)
    e_o, j_o = oracle_mod.spsa_row(lowered(circ, obs), flat, layout.flat_of_col, 0.01, 3,
                                   np.random.default_rng(7))
    assert close(sp.expectations, e_o) < TOL
    for k, v in split(j_o).items():
        assert close(sp.gradients[k], v) < TOL
    empty = G.adjoint_gradients(circ, b, [], wrt)
    assert empty.expectations.shape == (0,) and empty.gradients["w"].shape == (0, 5)


@pytest.mark.gpu
def test_gpu_spsa_fd_xy_observables_hbm_plan(oracle_mod):
    """SPSA and finite differences with X/Y strings at n = 13 (HBM plans are
    Z-only at the ABI): both must take the basis-group split like run_batch."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200 import gradients as G
    circ, obs, b = _case(3, n=13)
    assert not all(o.is_z_only for o in obs)
    wrt = ("w", "s")
    e_ref, j_ref, layout, flat = _oracle(oracle_mod, circ, obs, b, wrt)
    split = lambda j: {n: j[:, lo:hi] for n, lo, hi in layout.slices}  # noqa: E731
    fd = G.finite_difference_gradients(circ, b, obs, wrt)
    assert close(fd.expectations, e_ref) < TOL
    for k, v in split(j_ref).items():
        assert np.abs(fd.gradients[k] - v).max() < 1e-5
    sp = G.spsa_gradients(circ, b, obs, wrt, c=0.01, samples=2, seed=4)
    e_o, j_o = oracle_mod.spsa_row(lowered(circ, obs), flat, layout.flat_of_col, 0.01, 2,
                                   np.random.default_rng(4))
    assert close(sp.expectations, e_o) < TOL
    for k, v in split(j_o).items():
        assert close(sp.gradients[k], v) < TOL


@pytest.mark.gpu
def test_gpu_spsa_row_offset_slices_bitwise():
    """run_batch(method='spsa') on two row slices with matching row_offset
    concatenates to the full-batch result bit for bit (rank sharding)."""
    import dataclasses

    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200 import configs
    from paper_2404_06314_b200.engine import BatchEngine, BatchRequest
    spec = configs.CONFIGS[2]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=10)
    eng = BatchEngine(device="cuda:0")
    req = BatchRequest(circ, obs, {"w": w}, x, method="spsa", wrt=wrt, seed=9, spsa_samples=2)
    full = eng.run_batch(req)
    a = eng.run_batch(dataclasses.replace(req, inputs=x[:4]))
    b = eng.run_batch(dataclasses.replace(req, inputs=x[4:], row_offset=4))
    assert np.array_equal(np.concatenate([a.expectations, b.expectations]), full.expectations)
    for k in full.gradients:
        assert np.array_equal(np.concatenate([a.gradients[k], b.gradients[k]]), full.gradients[k])
