"""Classifier training (training.py) pinned to the reference's own training
run (tests/golden/training.npz, made by make_golden.py from
vqckit.train_classifier with its Adam, lr 0.05 / lambda 0.01).

CPU: the torch loop over an oracle-backed module (test infrastructure: the
oracle's Jacobian as the autograd backward) must reproduce the reference's
epoch records and final parameters. GPU: the same loop on QuantumModule,
whose backward is the VJP adjoint kernel."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN, oracle_batch

TOL = 1e-9


def _golden():
    return np.load(os.path.join(GOLDEN, "training.npz"))


def _problem():
    from paper_2404_06314_b200.ir import build_reuploading_ansatz
    from paper_2404_06314_b200.observables import Observable
    g = _golden()
    f, y = g["features"], g["labels"]
    circuit = build_reuploading_ansatz(4, 2, num_features=4)
    obs = [Observable(((2.0, "ZIII"),)), Observable(((2.0, "IZII"),))]
    return g, ((f[:32], y[:32]), (f[32:40], y[32:40])), circuit, obs


class _OracleFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, theta, lam, mod):
        vals = {"theta": theta.numpy(), "lambda": lam.numpy()}
        e, jac = oracle_batch(mod.circuit, mod.obs, vals, x.numpy(), ("theta", "lambda"))
        ctx.jac = jac
        return torch.from_numpy(e)

    @staticmethod
    def backward(ctx, up):
        u = up.numpy()
        return (None, torch.from_numpy(np.einsum("bm,bmp->p", u, ctx.jac["theta"])),
                torch.from_numpy(np.einsum("bm,bmp->p", u, ctx.jac["lambda"])), None)


class OracleModule(torch.nn.Module):
    """Same construction and draw order as QuantumModule, on the CPU oracle."""

    def __init__(self, circuit, obs, seed):
        super().__init__()
        from paper_2404_06314_b200.module import Constant, Uniform
        rng = np.random.default_rng(seed)
        self.circuit, self.obs, self.num_outputs = circuit, obs, len(obs)
        th = Uniform().draw(rng, circuit.set_named("theta").size)
        la = Constant(1.0).draw(rng, circuit.set_named("lambda").size)
        self.theta = torch.nn.Parameter(torch.from_numpy(th))
        self.lam = torch.nn.Parameter(torch.from_numpy(la))
        self.values = {"theta": self.theta, "lambda": self.lam}

    def forward(self, x):
        return _OracleFn.apply(x, self.theta, self.lam, self)


def _run(module):
    from paper_2404_06314_b200.training import set_rates, train_classifier
    _, (train, test), _, _ = _problem()
    opt = torch.optim.Adam(set_rates(module, 0.05, {"lambda": 0.01}))
    return train_classifier(module, train, test, epochs=3, batch_size=8, optimizer=opt, seed=3)


def _check(recs, theta, lam):
    g = _golden()
    assert np.abs(np.array([r.loss for r in recs]) - g["loss"]).max() < TOL
    assert np.array_equal(np.array([r.metric for r in recs]), g["metric"])
    assert np.abs(theta - g["theta"]).max() < TOL
    assert np.abs(lam - g["lam"]).max() < TOL


def test_training_with_oracle_module_matches_reference(oracle_mod):
    _, _, circuit, obs = _problem()
    mod = OracleModule(circuit, obs, seed=11)
    recs = _run(mod)
    _check(recs, mod.theta.detach().numpy(), mod.lam.detach().numpy())


def test_set_rates_and_shape_errors():
    from paper_2404_06314_b200.training import set_rates, train_classifier
    _, (train, test), circuit, obs = _problem()
    mod = OracleModule(circuit, obs, seed=0)
    groups = set_rates(mod, 0.1, {"lambda": 0.5})
    assert [(g["name"], g["lr"]) for g in groups] == [("theta", 0.1), ("lambda", 0.5)]
    with pytest.raises(ValueError, match="unknown parameter sets"):
        set_rates(mod, 0.1, {"nope": 1.0})
    mod.num_outputs = 1
    with pytest.raises(ValueError, match="outputs but the labels need 2 classes"):
        train_classifier(mod, train, test, 1, 8, torch.optim.SGD(mod.parameters(), lr=0.1))


@pytest.mark.gpu
def test_gpu_training_matches_reference():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200.module import Constant, QuantumModule, Uniform
    _, _, circuit, obs = _problem()
    mod = QuantumModule(circuit, obs, "s", [("theta", Uniform()), ("lambda", Constant(1.0))],
                        seed=11, device="cuda:0")
    recs = _run(mod)
    vals = mod.parameter_values()
    _check(recs, vals["theta"], vals["lambda"])
