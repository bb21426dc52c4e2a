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
