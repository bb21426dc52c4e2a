"""Classifier training on the GPU path.

Mirrors the reference's softmax classifier loop and optimizers
(vqckit/training.py:22-94, optim.py:13-66): same shuffling (one
``default_rng(seed)``, a permutation per epoch), same loss, the same
logit-space upstream ``(softmax - onehot) / B`` contracted through
``QuantumModule.backward`` (here one VJP-seeded adjoint launch sequence on the
GPU), and the same per-set-rate SGD / Adam updates on float64 parameter
dicts. Works with any module exposing ``forward``, ``backward``,
``parameter_values`` / ``values`` (this package's ``QuantumModule``) or a
reference-style module whose ``parameters()`` returns live arrays.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass

import numpy as np


@dataclass
class EpochRecord:
    epoch: int
    loss: float
    metric: float  # accuracy for the classifier


@dataclass
class ArrayDataset:
    """The reference's ``Dataset`` shape (datasets.py:16-31): features (N, F),
    integer labels, train / test index arrays."""

    features: np.ndarray
    labels: np.ndarray
    train_idx: np.ndarray
    test_idx: np.ndarray
    num_classes: int

    @property
    def num_features(self) -> int:
        return self.features.shape[1]

    def train(self):
        return self.features[self.train_idx], self.labels[self.train_idx]

    def test(self):
        return self.features[self.test_idx], self.labels[self.test_idx]


def write_training_log(records, path) -> None:
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(["epoch", "loss", "metric"])
        for r in records:
            writer.writerow([r.epoch, repr(r.loss), repr(r.metric)])


def softmax(logits: np.ndarray) -> np.ndarray:
    z = np.exp(logits - logits.max(axis=-1, keepdims=True))
    return z / z.sum(axis=-1, keepdims=True)


def one_hot(labels: np.ndarray, num_classes: int) -> np.ndarray:
    out = np.zeros((len(labels), num_classes))
    out[np.arange(len(labels)), labels] = 1.0
    return out


def cross_entropy(probs: np.ndarray, labels: np.ndarray) -> float:
    picked = probs[np.arange(len(labels)), labels]
    return float(-np.mean(np.log(np.clip(picked, 1e-12, None))))


class SGD:
    """p -= rate(set) * grad (optim.py:13-30)."""

    def __init__(self, lr: float = 0.01, per_set: dict | None = None):
        self.lr = float(lr)
        self.per_set = dict(per_set or {})
        self.step_count = 0

    def rate(self, name: str) -> float:
        return self.per_set.get(name, self.lr)

    def step(self, params: dict, grads: dict) -> None:
        self.step_count += 1
        for name, grad in grads.items():
            p = params[name]
            _check(name, p, grad)
            p -= self.rate(name) * grad


class Adam:
    """Bias-corrected Adam with per-set rates (optim.py:33-66)."""

    def __init__(self, lr: float = 0.001, per_set: dict | None = None,
                 beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8):
        self.lr = float(lr)
        self.per_set = dict(per_set or {})
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.step_count = 0
        self._m: dict = {}
        self._v: dict = {}

    def rate(self, name: str) -> float:
        return self.per_set.get(name, self.lr)

    def step(self, params: dict, grads: dict) -> None:
        self.step_count += 1
        t = self.step_count
        for name, grad in grads.items():
            p = params[name]
            _check(name, p, grad)
            if name not in self._m:
                self._m[name] = np.zeros_like(p)
                self._v[name] = np.zeros_like(p)
            m, v = self._m[name], self._v[name]
            m *= self.beta1
            m += (1 - self.beta1) * grad
            v *= self.beta2
            v += (1 - self.beta2) * np.square(grad)
            m_hat = m / (1 - self.beta1 ** t)
            v_hat = v / (1 - self.beta2 ** t)
            p -= self.rate(name) * m_hat / (np.sqrt(v_hat) + self.eps)


def _check(name, p, grad):
    if p.shape != np.shape(grad):
        raise ValueError(f"{name}: gradient shape {np.shape(grad)} "
                         f"does not match parameter shape {p.shape}")


def _numpy(a) -> np.ndarray:
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.asarray(a, np.float64)


def _forward(module, x) -> np.ndarray:
    import torch
    with torch.no_grad():
        return _numpy(module.forward(x))


def _params(module) -> dict:
    if hasattr(module, "parameter_values"):
        return module.parameter_values()
    return module.parameters()      # reference modules: live arrays


def _store(module, params: dict) -> None:
    values = getattr(module, "values", None)
    if values is None or not hasattr(module, "parameter_values"):
        return                      # live arrays were updated in place
    import torch
    with torch.no_grad():
        for name, p in params.items():
            values[name].copy_(torch.from_numpy(p))


def accuracy(module, features, labels) -> float:
    probs = softmax(_forward(module, features))
    return float(np.mean(probs.argmax(axis=1) == labels))


def train_classifier(dataset, module, epochs: int, batch_size: int, optimizer,
                     seed: int = 0, method: str | None = None,
                     log=None) -> list[EpochRecord]:
    """Minibatch softmax / cross-entropy training (training.py:59-94)."""
    if module.num_outputs != dataset.num_classes:
        raise ValueError(f"module has {module.num_outputs} outputs but the "
                         f"dataset has {dataset.num_classes} classes")
    if module.encoding_size != dataset.num_features:
        raise ValueError(f"module encodes {module.encoding_size} features "
                         f"but the dataset has {dataset.num_features}")
    rng = np.random.default_rng(seed)
    train_x, train_y = dataset.train()
    test_x, test_y = dataset.test()
    records = []
    for epoch in range(epochs):
        order = rng.permutation(len(train_y))
        losses = []
        for lo in range(0, len(order), batch_size):
            idx = order[lo:lo + batch_size]
            xb, yb = train_x[idx], train_y[idx]
            probs = softmax(_forward(module, xb))
            losses.append(cross_entropy(probs, yb))
            upstream = (probs - one_hot(yb, dataset.num_classes)) / len(idx)
            grads = module.backward(xb, upstream, method=method)
            params = _params(module)
            optimizer.step(params, grads)
            _store(module, params)
        record = EpochRecord(epoch, float(np.mean(losses)), accuracy(module, test_x, test_y))
        records.append(record)
        if log is not None:
            log(record)
    return records


# -- REINFORCE on cart-pole (training.py:97-193, cartpole.py) -------------------

# classic cart-pole constants (cartpole.py:11-23): g, masses, pole half-length,
# push force, Euler step, termination limits, episode cap
CARTPOLE = dict(gravity=9.8, m_cart=1.0, m_pole=0.1, half_len=0.5, force=10.0, dt=0.02,
                angle_limit=12.0 * np.pi / 180.0, x_limit=2.4, max_steps=500)


def cartpole_derivatives(state, push: float, c=CARTPOLE):
    """(x_acc, theta_acc) of the frictionless cart-pole under a horizontal push."""
    _, _, th, th_dot = state
    m_tot = c["m_cart"] + c["m_pole"]
    ml = c["m_pole"] * c["half_len"]
    cos_t, sin_t = np.cos(th), np.sin(th)
    tmp = (push + ml * th_dot ** 2 * sin_t) / m_tot
    th_acc = (c["gravity"] * sin_t - cos_t * tmp) / (
        c["half_len"] * (4.0 / 3.0 - c["m_pole"] * cos_t ** 2 / m_tot))
    return tmp - ml * th_acc * cos_t / m_tot, th_acc


class CartPoleEnv:
    """State (x, x_dot, theta, theta_dot); action 0 pushes left, 1 right;
    reward 1 per step survived. Same reset draws and Euler update order as
    the reference environment (cartpole.py:26-68)."""

    def __init__(self, seed: int | None = None):
        self._rng = np.random.default_rng(seed)
        self.state = np.zeros(4)
        self.steps = 0
        self.terminated = True

    def reset(self, seed: int | None = None) -> np.ndarray:
        if seed is not None:
            self._rng = np.random.default_rng(seed)
        self.state = self._rng.uniform(-0.05, 0.05, 4)
        self.steps, self.terminated = 0, False
        return self.state.copy()

    def step(self, action: int):
        if self.terminated:
            raise RuntimeError("step() called on a terminated episode; call reset() first")
        if action not in (0, 1):
            raise ValueError(f"action must be 0 or 1, got {action}")
        c = CARTPOLE
        x_acc, th_acc = cartpole_derivatives(self.state, c["force"] if action == 1 else -c["force"])
        x, x_dot, th, th_dot = self.state
        # positions advance with the old velocities, then velocities update
        self.state = np.array([x + c["dt"] * x_dot, x_dot + c["dt"] * x_acc,
                               th + c["dt"] * th_dot, th_dot + c["dt"] * th_acc])
        self.steps += 1
        self.terminated = bool(abs(self.state[0]) > c["x_limit"]
                               or abs(self.state[2]) > c["angle_limit"]
                               or self.steps >= c["max_steps"])
        return self.state.copy(), 1.0, self.terminated


def cartpole_policy(depth: int = 3, seed: int | None = None, logit_scale: float = 3.0,
                    device=None):
    """4-qubit re-uploading policy, one scaled Z observable per action
    (training.py:99-117), as a GPU QuantumModule."""
    from .ir import build_reuploading_ansatz
    from .module import Constant, QuantumModule, Uniform
    from .observables import Observable
    circuit = build_reuploading_ansatz(4, depth, num_features=4)
    obs = [Observable(((logit_scale, "ZIII"),)), Observable(((logit_scale, "IZII"),))]
    return QuantumModule(circuit, obs, "s", [("theta", Uniform()), ("lambda", Constant(1.0))],
                         seed=seed, device=device)


def encode_state(state: np.ndarray) -> np.ndarray:
    return np.arctan(state)


def returns_to_go(rewards, discount: float) -> np.ndarray:
    out = np.empty(len(rewards))
    acc = 0.0
    for t in range(len(rewards) - 1, -1, -1):
        acc = rewards[t] + discount * acc
        out[t] = acc
    return out


def sample_episode(env, policy, rng, reset_seed: int):
    """One rollout: per step a batch-1 forward, then rng.choice over the
    softmax (training.py:134-151)."""
    state = env.reset(seed=reset_seed)
    states, actions, rewards, probs_all = [], [], [], []
    done = False
    while not done:
        enc = encode_state(state)
        probs = softmax(_forward(policy, enc[None, :])[0])
        action = int(rng.choice(len(probs), p=probs))
        states.append(enc)
        actions.append(action)
        probs_all.append(probs)
        state, reward, done = env.step(action)
        rewards.append(reward)
    return (np.asarray(states), np.asarray(actions, np.int64), np.asarray(rewards),
            np.asarray(probs_all))


def train_reinforce(env, policy, episodes_per_epoch: int, epochs: int, optimizer,
                    discount: float = 0.99, seed: int = 0, log=None) -> list[EpochRecord]:
    """REINFORCE without baseline (training.py:154-193): the epoch's visited
    states go through ONE batched VJP with upstream
    (onehot(action) - softmax) * return-to-go / episodes, negated for the
    descending optimizer."""
    if policy.num_outputs < 2:
        raise ValueError("policy needs one observable per action")
    rng = np.random.default_rng(seed)
    records = []
    for epoch in range(epochs):
        states, ups, returns = [], [], []
        for _ in range(episodes_per_epoch):
            reset_seed = int(rng.integers(0, 2 ** 31))
            s, a, r, p = sample_episode(env, policy, rng, reset_seed)
            ups.append((one_hot(a, policy.num_outputs) - p) * returns_to_go(r, discount)[:, None])
            states.append(s)
            returns.append(r.sum())
        ascent = policy.backward(np.concatenate(states),
                                 np.concatenate(ups) / episodes_per_epoch)
        params = _params(policy)
        optimizer.step(params, {n: -g for n, g in ascent.items()})
        _store(policy, params)
        mean_return = float(np.mean(returns))
        record = EpochRecord(epoch, -mean_return, mean_return)
        records.append(record)
        if log is not None:
            log(record)
    return records


# -- dataset helpers (datasets.py:47-66, 106-125) --------------------------------

Dataset = ArrayDataset


def split_indices(n: int, seed: int, test_fraction: float = 0.2):
    """Sorted, disjoint train / test indices from one seeded permutation."""
    order = np.random.default_rng(seed).permutation(n)
    n_test = int(round(n * test_fraction))
    return np.sort(order[n_test:]), np.sort(order[:n_test])


def from_arrays(features, labels, seed: int = 0, test_fraction: float = 0.2) -> ArrayDataset:
    features = np.asarray(features, dtype=np.float64)
    labels = np.asarray(labels)
    if np.any(labels != labels.astype(np.int64)):
        raise ValueError("labels must be integers")
    labels = labels.astype(np.int64)
    if np.any(labels < 0):
        raise ValueError("labels must be non-negative")
    classes = int(labels.max()) + 1 if len(labels) else 0
    tr, te = split_indices(len(labels), seed, test_fraction)
    return ArrayDataset(features, labels, tr, te, classes)


def synthetic_blobs(samples_per_class: int = 60, num_features: int = 4, num_classes: int = 2,
                    separation: float = 3.0, noise: float = 0.5, seed: int = 0,
                    test_fraction: float = 0.2) -> ArrayDataset:
    """One Gaussian blob per class around a random direction scaled to
    ``separation``; draws: centres first, then each class's noise in order."""
    rng = np.random.default_rng(seed)
    centers = rng.normal(size=(num_classes, num_features))
    centers = centers / np.linalg.norm(centers, axis=1, keepdims=True) * separation
    feats = np.concatenate([centers[c] + noise * rng.normal(size=(samples_per_class, num_features))
                            for c in range(num_classes)])
    labels = np.repeat(np.arange(num_classes, dtype=np.int64), samples_per_class)
    return from_arrays(feats, labels, seed=seed, test_fraction=test_fraction)


def load_dataset(path, seed: int = 0, test_fraction: float = 0.2) -> ArrayDataset:
    """Text table -> dataset (datasets.py:69-103): comma- or whitespace-
    separated, '#' comments and blank lines skipped, an optional non-numeric
    header as the first content row, last column = integer label."""
    rows, width, seen_content = [], None, False
    with open(path) as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            fields = line.split(",") if "," in line else line.split()
            try:
                values = [float(f) for f in fields]
            except ValueError as exc:
                if not seen_content:          # header row
                    seen_content = True
                    continue
                raise ValueError(f"{path}:{lineno}: malformed row") from exc
            seen_content = True
            if width is None:
                width = len(values)
                if width < 2:
                    raise ValueError(f"{path}:{lineno}: need at least one feature column "
                                     "and one label column")
            elif len(values) != width:
                raise ValueError(f"{path}:{lineno}: expected {width} columns, "
                                 f"got {len(values)}")
            if values[-1] != int(values[-1]):
                raise ValueError(f"{path}:{lineno}: unknown label {values[-1]!r} "
                                 "(labels must be integers)")
            rows.append(values)
    if not rows:
        raise ValueError(f"{path}: no data rows")
    data = np.asarray(rows)
    return from_arrays(data[:, :-1], data[:, -1], seed, test_fraction)
