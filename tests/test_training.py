"""train_classifier + SGD / Adam (training.py:59-94, optim.py:13-66) against
the reference's own training run (tests/golden/training.npz, made by
make_golden.py from vqckit.train_classifier).

CPU: the loop driven by an oracle-backed module (test infrastructure) must
reproduce the reference's records and final parameters. GPU: the same loop on
this package's QuantumModule (VJP adjoint on libvqc.so)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, oracle_batch

TOL = 1e-9


def _golden():
    return np.load(os.path.join(GOLDEN, "training.npz"))


def _problem():
    from paper_2404_06314_b200.ir import build_reuploading_ansatz
    from paper_2404_06314_b200.observables import Observable
    from paper_2404_06314_b200.training import ArrayDataset
    g = _golden()
    ds = ArrayDataset(g["features"], g["labels"], np.arange(32), np.arange(32, 40), 2)
    circuit = build_reuploading_ansatz(4, 2, num_features=4)
    obs = [Observable(((2.0, "ZIII"),)), Observable(((2.0, "IZII"),))]
    return g, ds, circuit, obs


class OracleModule:
    """Reference-style module (numpy, live parameter arrays) over the oracle."""

    def __init__(self, circuit, obs, seed):
        from paper_2404_06314_b200.module import Constant, Uniform
        rng = np.random.default_rng(seed)
        self.circuit, self.obs = circuit, obs
        self.params = {"theta": Uniform().draw(rng, circuit.set_named("theta").size),
                       "lambda": Constant(1.0).draw(rng, circuit.set_named("lambda").size)}
        self.num_outputs, self.encoding_size = len(obs), 4

    def parameters(self):
        return self.params

    def forward(self, x):
        return oracle_batch(self.circuit, self.obs, self.params, x, ())[0]

    def backward(self, x, upstream, method=None):
        _, jac = oracle_batch(self.circuit, self.obs, self.params, x, ("theta", "lambda"))
        return {n: np.einsum("bm,bmp->p", upstream, j) for n, j in jac.items()}


def _run(module):
    from paper_2404_06314_b200.training import Adam, train_classifier
    opt = Adam(lr=0.05, per_set={"lambda": 0.01})
    return train_classifier(_problem()[1], module, epochs=3, batch_size=8, optimizer=opt, seed=3)


def test_optimizers_match_formulas():
    from paper_2404_06314_b200.training import SGD, Adam
    p = {"a": np.array([1.0, -2.0])}
    g = {"a": np.array([0.5, 0.25])}
    SGD(lr=0.1, per_set={"a": 0.2}).step(p, g)
    assert np.allclose(p["a"], [0.9, -2.05])
    p = {"a": np.array([1.0])}
    Adam(lr=0.1).step(p, {"a": np.array([3.0])})
    assert np.allclose(p["a"], [0.9], atol=1e-7)        # first Adam step = lr * sign
    with pytest.raises(ValueError, match="gradient shape"):
        SGD().step({"a": np.zeros(2)}, {"a": np.zeros(3)})


def test_training_with_oracle_module_matches_reference(oracle_mod):
    g, _, circuit, obs = _problem()
    mod = OracleModule(circuit, obs, seed=11)
    recs = _run(mod)
    assert np.abs(np.array([r.loss for r in recs]) - g["loss"]).max() < TOL
    assert np.array_equal(np.array([r.metric for r in recs]), g["metric"])
    assert np.abs(mod.params["theta"] - g["theta"]).max() < TOL
    assert np.abs(mod.params["lambda"] - g["lam"]).max() < TOL


def test_shape_errors():
    from paper_2404_06314_b200.training import SGD, train_classifier
    g, ds, circuit, obs = _problem()
    mod = OracleModule(circuit, obs[:1], seed=0)
    mod.num_outputs = 1
    with pytest.raises(ValueError, match="outputs but the dataset has 2 classes"):
        train_classifier(ds, mod, 1, 8, SGD())


@pytest.mark.gpu
def test_gpu_training_matches_reference():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200.module import Constant, QuantumModule, Uniform
    g, _, circuit, obs = _problem()
    mod = QuantumModule(circuit, obs, "s", [("theta", Uniform()), ("lambda", Constant(1.0))],
                        seed=11, device="cuda:0")
    recs = _run(mod)
    assert np.abs(np.array([r.loss for r in recs]) - g["loss"]).max() < TOL
    assert np.array_equal(np.array([r.metric for r in recs]), g["metric"])
    vals = mod.parameter_values()
    assert np.abs(vals["theta"] - g["theta"]).max() < TOL
    assert np.abs(vals["lambda"] - g["lam"]).max() < TOL


def _reinforce(policy):
    from paper_2404_06314_b200.training import SGD, CartPoleEnv, train_reinforce
    return train_reinforce(CartPoleEnv(), policy, episodes_per_epoch=2, epochs=3,
                           optimizer=SGD(lr=0.05), seed=9)


def _check_reinforce(recs, theta, lam):
    g = np.load(os.path.join(GOLDEN, "reinforce.npz"))
    assert np.array_equal(np.array([r.metric for r in recs]), g["metric"])   # episode returns
    assert np.array_equal(np.array([r.loss for r in recs]), g["loss"])
    assert np.abs(theta - g["theta"]).max() < TOL
    assert np.abs(lam - g["lam"]).max() < TOL


def test_cartpole_env_contract():
    from paper_2404_06314_b200.training import CartPoleEnv
    env = CartPoleEnv()
    with pytest.raises(RuntimeError, match="reset"):
        env.step(0)
    s = env.reset(seed=1)
    assert s.shape == (4,) and np.all(np.abs(s) <= 0.05)
    with pytest.raises(ValueError, match="action must be 0 or 1"):
        env.step(2)
    steps = 0
    done = False
    while not done:
        _, r, done = env.step(1)
        steps += 1
        assert r == 1.0
    assert 1 <= steps < 500       # always pushing right drops the pole


def test_reinforce_with_oracle_module_matches_reference(oracle_mod):
    from paper_2404_06314_b200.ir import build_reuploading_ansatz
    from paper_2404_06314_b200.observables import Observable
    circuit = build_reuploading_ansatz(4, 2, num_features=4)
    obs = [Observable(((3.0, "ZIII"),)), Observable(((3.0, "IZII"),))]
    mod = OracleModule(circuit, obs, seed=5)
    recs = _reinforce(mod)
    _check_reinforce(recs, mod.params["theta"], mod.params["lambda"])


@pytest.mark.gpu
def test_gpu_reinforce_matches_reference():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200.training import cartpole_policy
    policy = cartpole_policy(depth=2, seed=5, device="cuda:0")
    recs = _reinforce(policy)
    vals = policy.parameter_values()
    _check_reinforce(recs, vals["theta"], vals["lambda"])
