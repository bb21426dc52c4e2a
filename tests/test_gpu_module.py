"""QuantumModule (torch.nn.Module + autograd node) on the GPU vs the oracle,
mirroring the reference's model tests (test_model.py: VJP == Jacobian
slices, finite-difference check, construction-order initialisation)."""

import numpy as np
import pytest

from conftest import close, oracle_batch

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    return torch


def _module(spec_id, seed=7):
    from paper_2404_06314_b200 import configs
    from paper_2404_06314_b200.module import QuantumModule
    spec = configs.CONFIGS[spec_id]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    return spec, circ, obs, QuantumModule(circ, obs, "x", ["w"], seed=seed, device="cuda:0")


@pytest.mark.parametrize("cfg_id", [1, 2, 3])
def test_autograd_matches_oracle(torch, cfg_id):
    from paper_2404_06314_b200 import configs
    spec, circ, obs, mod = _module(cfg_id)
    x, _ = configs.inputs_and_weights(spec, batch=min(spec.batch, 96))
    w = mod.parameter_values()["w"]
    xt = torch.from_numpy(x).cuda().requires_grad_(True)
    out = mod(xt)
    rng = np.random.default_rng(cfg_id)
    up = rng.normal(size=out.shape)
    out.backward(torch.from_numpy(up).cuda())
    e_ref, j_ref = oracle_batch(circ, obs, {"w": w}, x, ("w", "x"))
    assert close(out.detach().cpu().numpy(), e_ref) < TOL
    assert close(mod.values["w"].grad.cpu().numpy(), np.einsum("bm,bmp->p", up, j_ref["w"])) < TOL
    assert close(xt.grad.cpu().numpy(), np.einsum("bm,bmf->bf", up, j_ref["x"])) < TOL


def test_autograd_hbm_plan_matches_oracle(torch):
    """cfg4 (16 qubits: HBM passes, separate forward / adjoint schedules) through
    the autograd node with a row-dependent upstream."""
    from paper_2404_06314_b200 import configs
    spec, circ, obs, mod = _module(4)
    x, _ = configs.inputs_and_weights(spec, batch=4)
    w = mod.parameter_values()["w"]
    xt = torch.from_numpy(x).cuda().requires_grad_(True)
    out = mod(xt)
    up = np.random.default_rng(4).normal(size=out.shape)
    out.backward(torch.from_numpy(up).cuda())
    e_ref, j_ref = oracle_batch(circ, obs, {"w": w}, x, ("w", "x"))
    assert close(out.detach().cpu().numpy(), e_ref) < TOL
    assert close(mod.values["w"].grad.cpu().numpy(), np.einsum("bm,bmp->p", up, j_ref["w"])) < TOL
    assert close(xt.grad.cpu().numpy(), np.einsum("bm,bmf->bf", up, j_ref["x"])) < TOL


def test_reference_style_backward_and_jacobians(torch):
    # model.py:644-662: backward == einsum over the Jacobian slices
    from paper_2404_06314_b200 import configs
    spec, circ, obs, mod = _module(2)
    x, _ = configs.inputs_and_weights(spec, batch=40)
    up = np.random.default_rng(1).normal(size=(40, len(obs)))
    vjp = mod.backward(x, up)
    jac = mod.jacobians(x)
    assert jac.expectations.shape == (40, 8) and jac.gradients["w"].shape == (40, 8, 64)
    assert close(vjp["w"], np.einsum("bm,bmp->p", up, jac.gradients["w"])) < TOL
    with pytest.raises(ValueError, match="upstream shape"):
        mod.backward(x, up[:, :3])


def test_finite_difference(torch):
    # test_model.py:146-166: directional FD check of the contraction
    from paper_2404_06314_b200 import configs
    spec, circ, obs, mod = _module(1)
    x, _ = configs.inputs_and_weights(spec, batch=8)
    up = np.random.default_rng(2).normal(size=(8, 1))
    g = mod.backward(x, up)["w"]
    d = np.random.default_rng(3).normal(size=g.shape)
    h = 1e-5
    w0 = mod.values["w"].detach().clone()

    def f(wv):
        with torch.no_grad():
            mod.values["w"].copy_(wv)
            return float((mod(x).cpu().numpy() * up).sum())

    fd = (f(w0 + h * torch.from_numpy(d).cuda()) - f(w0 - h * torch.from_numpy(d).cuda())) / (2 * h)
    f(w0)
    assert abs(fd - g @ d) < 1e-6


def test_initialisation_order_and_seed(torch):
    # model.py:72-96: sets drawn in declared order from one default_rng(seed)
    _, _, _, mod = _module(3, seed=11)
    ref = np.random.default_rng(11).uniform(0, 2 * np.pi, 288)
    np.testing.assert_array_equal(mod.parameter_values()["w"], ref)


def test_optimizer_step_reduces_loss(torch):
    from paper_2404_06314_b200 import configs
    spec, circ, obs, mod = _module(2, seed=0)
    x, _ = configs.inputs_and_weights(spec, batch=64)
    target = torch.zeros((64, 8), dtype=torch.float64, device="cuda")
    opt = torch.optim.SGD(mod.parameters(), lr=0.05)
    losses = []
    for _ in range(5):
        opt.zero_grad()
        loss = ((mod(x) - target) ** 2).mean()
        loss.backward()
        opt.step()
        losses.append(float(loss.detach()))
    assert losses[-1] < losses[0]


def test_nccl_world_size_1_allreduce(torch):
    """Single-process NCCL group: the sharded path's collective is a no-op sum."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2404_06314_b200 import parallel
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        _, _, _, mod = _module(1)
        out = mod(np.zeros((4, 4)))
        out.sum().backward()
        before = mod.values["w"].grad.clone()
        parallel.allreduce_module_grads(mod)
        assert torch.equal(before, mod.values["w"].grad)
    finally:
        dist.destroy_process_group()


def test_hybrid_module_matches_reference_semantics(torch):
    """HybridModule (model.py:152-222): oracle-built reference of its backward."""
    from paper_2404_06314_b200 import configs
    from paper_2404_06314_b200.module import HybridModule
    spec, circ, obs, qmod = _module(2, seed=3)
    hyb = HybridModule(5, qmod, 3, seed=9)
    rng = np.random.default_rng(4)
    x = rng.normal(size=(12, 5))
    up = rng.normal(size=(12, 3))
    g = hyb.backward(x, up)
    # reference math (model.py:720-742) with oracle Jacobians
    Wp = hyb.pre_weight.detach().cpu().numpy()
    bp = hyb.pre_bias.detach().cpu().numpy()
    Wq = hyb.post_weight.detach().cpu().numpy()
    pre = x @ Wp.T + bp
    ang = np.pi * np.tanh(pre)
    w = qmod.parameter_values()["w"]
    q, jac = oracle_batch(circ, obs, {"w": w}, ang, ("w", "x"))
    d_q = up @ Wq
    d_ang = np.einsum("bm,bmf->bf", d_q, jac["x"])
    d_pre = d_ang * np.pi * (1.0 - np.tanh(pre) ** 2)
    ref = {"post.weight": up.T @ q, "post.bias": up.sum(0), "w": np.einsum("bm,bmp->p", d_q, jac["w"]),
           "pre.weight": d_pre.T @ x, "pre.bias": d_pre.sum(0)}
    for k, v in ref.items():
        assert close(g[k], v) < TOL, k
    with pytest.raises(ValueError, match="single-qubit"):
        from paper_2404_06314_b200 import parse_observable
        from paper_2404_06314_b200.module import QuantumModule
        bad = QuantumModule(circ, [parse_observable("ZZ" + "I" * 6)], "x", ["w"], device="cuda:0")
        HybridModule(5, bad, 3)
