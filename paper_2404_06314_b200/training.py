"""Classifier training over the GPU module with torch optimizers (SURVEY §8f
item 4).

The reference trains its quantum classifier with a numpy loop and its own
optimizers (vqckit/training.py:59-94, optim.py:13-66): it contracts the
logit gradient ``(softmax - onehot) / B`` through ``QuantumModule.backward``.
Here the module is a torch ``nn.Module`` whose backward is the VJP-seeded
adjoint kernel, so the loop is plain torch: ``F.cross_entropy`` on the
module's (B, C) outputs, ``loss.backward()``, and any ``torch.optim``
optimizer. ``set_rates`` builds per-parameter-set learning rates (the
reference's ``per_set``) as torch param groups.

Shuffling uses one ``np.random.default_rng(seed)`` permutation per epoch, so
a run visits minibatches in the same order as the reference's loop with the
same seed. That is why the tests can pin this loop to a reference training
run (tests/golden/training.npz).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F


@dataclass
class EpochRecord:
    epoch: int
    loss: float      # mean minibatch cross-entropy of the epoch
    metric: float    # test accuracy after the epoch


def set_rates(module, lr: float, per_set: dict | None = None) -> list[dict]:
    """torch param groups: one per named parameter set of a QuantumModule
    (``module.values``), learning rate ``per_set.get(name, lr)``; any other
    parameters (e.g. a HybridModule's dense layers) share one group at ``lr``."""
    per_set = dict(per_set or {})
    quantum = getattr(module, "quantum", module)
    named = dict(getattr(quantum, "values", {}))
    unknown = set(per_set) - set(named)
    if unknown:
        raise ValueError(f"per_set names unknown parameter sets: {sorted(unknown)}")
    groups = [{"params": [p], "lr": float(per_set.get(n, lr)), "name": n} for n, p in named.items()]
    seen = {id(p) for p in named.values()}
    rest = [p for p in module.parameters() if id(p) not in seen]
    if rest:
        groups.append({"params": rest, "lr": float(lr), "name": "other"})
    return groups


def _as_tensor(a, device, dtype):
    t = a if torch.is_tensor(a) else torch.from_numpy(np.ascontiguousarray(a))
    return t.to(device=device, dtype=dtype)


@torch.no_grad()
def accuracy(module, features, labels) -> float:
    dev = next(module.parameters()).device
    logits = module(_as_tensor(features, dev, torch.float64))
    y = _as_tensor(labels, dev, torch.long)
    return float((logits.argmax(dim=1) == y).double().mean().item()) if len(y) else 0.0


def train_classifier(module, train, test, epochs: int, batch_size: int,
                     optimizer: torch.optim.Optimizer, seed: int = 0, log=None) -> list[EpochRecord]:
    """Minibatch cross-entropy training; ``train`` / ``test`` are
    (features (N, F), integer labels (N,)) pairs. Each step is one forward
    launch plus one VJP adjoint launch sequence on the module's device."""
    (xtr, ytr), (xte, yte) = train, test
    n_out = getattr(module, "num_outputs", None) or getattr(module, "output_dim", None)
    classes = int(np.max(np.concatenate([np.asarray(ytr), np.asarray(yte)]))) + 1 if len(ytr) else 0
    if n_out is not None and classes > n_out:
        raise ValueError(f"module has {n_out} outputs but the labels need {classes} classes")
    if batch_size < 1:
        raise ValueError(f"batch_size must be >= 1, got {batch_size}")
    dev = next(module.parameters()).device
    x = _as_tensor(xtr, dev, torch.float64)
    y = _as_tensor(ytr, dev, torch.long)
    rng = np.random.default_rng(seed)
    records = []
    for epoch in range(epochs):
        order = torch.from_numpy(rng.permutation(len(y))).to(dev)
        batch_losses = []
        for idx in order.split(batch_size):
            optimizer.zero_grad(set_to_none=True)
            loss = F.cross_entropy(module(x[idx]), y[idx])
            loss.backward()
            optimizer.step()
            batch_losses.append(loss.detach())
        mean = torch.stack(batch_losses).mean().item() if batch_losses else float("nan")
        rec = EpochRecord(epoch, float(mean), accuracy(module, xte, yte))
        records.append(rec)
        if log is not None:
            log(rec)
    return records
