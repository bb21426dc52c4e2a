"""The five BASELINE.json workloads as circuits + seeded synthetic inputs.

Shapes follow BASELINE.json ``configs`` and SURVEY §8(d): sets ``x``
(encoding, n) then ``w`` (trainable, P); per layer and qubit the encoding
rotation ENC(x[q]) then the trainable rotations in listed order (each takes
the next ``w`` index), then the entanglers. Inputs: ``rng =
default_rng(1000 + id)``, ``x = rng.uniform(-pi, pi, (B, n))`` first, then the
weights. There is no public dataset for this path; these seeded draws are
the benchmark inputs.

``build(cfg, api)`` is duck-typed over an IR namespace (this package's
``ir``/``observables``, or the reference's ``vqckit`` for golden generation,
which needs ``cz_decompose=True`` because the reference has no CZ gate:
CZ(c,t) = H(t) CNOT(c,t) H(t)).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ConfigSpec:
    cfg_id: int
    n: int
    layers: int
    batch: int
    enc: str               # "RX" | "RY"
    trainable: tuple       # rotation kinds per qubit per layer
    entangler: str         # "cnot_ring" | "cz_chain" | "cz_all"
    observables: str       # "zzzz" | "per_qubit" | "sum_z" | "z0z1"
    weights: str           # "uniform" | "normal"
    wrt_inputs: bool

    @property
    def num_weights(self) -> int:
        return self.n * self.layers * len(self.trainable)

    @property
    def name(self) -> str:
        return (f"cfg{self.cfg_id}_{self.n}q_L{self.layers}_B{self.batch}_"
                f"{self.entangler}")


CONFIGS = {
    1: ConfigSpec(1, 4, 2, 32, "RX", ("RY", "RZ"), "cnot_ring", "zzzz", "uniform", True),
    2: ConfigSpec(2, 8, 4, 1024, "RX", ("RY", "RZ"), "cz_chain", "per_qubit", "normal", True),
    3: ConfigSpec(3, 12, 8, 4096, "RY", ("RX", "RY", "RZ"), "cnot_ring", "sum_z", "uniform", False),
    4: ConfigSpec(4, 16, 10, 16384, "RX", ("RY", "RZ"), "cnot_ring", "per_qubit", "uniform", True),
    5: ConfigSpec(5, 22, 6, 512, "RY", ("RX", "RY", "RZ"), "cz_all", "z0z1", "uniform", False),
}


def entangler_pairs(spec: ConfigSpec) -> list[tuple[str, int, int]]:
    n = spec.n
    if spec.entangler == "cnot_ring":
        return [("CNOT", q, (q + 1) % n) for q in range(n)] if n > 1 else []
    if spec.entangler == "cz_chain":
        return [("CZ", q, q + 1) for q in range(n - 1)]
    if spec.entangler == "cz_all":
        return [("CZ", i, j) for i in range(n) for j in range(i + 1, n)]
    raise ValueError(spec.entangler)


def observable_terms(spec: ConfigSpec) -> list[list[tuple[float, str]]]:
    n = spec.n

    def z(qs):
        return "".join("Z" if q in qs else "I" for q in range(n))

    if spec.observables == "zzzz":
        return [[(1.0, z(range(n)))]]
    if spec.observables == "per_qubit":
        return [[(1.0, z((q,)))] for q in range(n)]
    if spec.observables == "sum_z":
        return [[(1.0, z((q,))) for q in range(n)]]
    if spec.observables == "z0z1":
        return [[(1.0, z((0, 1)))]]
    raise ValueError(spec.observables)


def build(spec: ConfigSpec, api, cz_decompose: bool = False):
    """(circuit, observables, wrt) built from ``api``'s IR classes."""
    GK = api.GateKind
    gates = []
    widx = 0
    for _ in range(spec.layers):
        for q in range(spec.n):
            gates.append(api.Gate(GK[spec.enc], (q,), api.AngleExpression(1.0, (("x", q),))))
            for kind in spec.trainable:
                gates.append(api.Gate(GK[kind], (q,), api.AngleExpression(1.0, (("w", widx),))))
                widx += 1
        for kind, a, b in entangler_pairs(spec):
            if kind == "CZ" and cz_decompose:
                gates += [api.Gate(GK.H, (b,)), api.Gate(GK.CNOT, (a, b)), api.Gate(GK.H, (b,))]
            else:
                gates.append(api.Gate(GK[kind], (a, b)))
    sets = (api.ParameterSet("x", spec.n, "encoding"),
            api.ParameterSet("w", spec.num_weights, "trainable"))
    circuit = api.Circuit(spec.n, tuple(gates), sets)
    observables = [api.Observable(tuple(terms)) for terms in observable_terms(spec)]
    wrt = ("w", "x") if spec.wrt_inputs else ("w",)
    return circuit, observables, wrt


def inputs_and_weights(spec: ConfigSpec, batch: int | None = None):
    """Seeded synthetic data: x (B, n) ~ U(-pi, pi) drawn first, then w."""
    rng = np.random.default_rng(1000 + spec.cfg_id)
    x = rng.uniform(-np.pi, np.pi, (spec.batch, spec.n))
    if spec.weights == "normal":
        w = rng.normal(0.0, 1.0, spec.num_weights)
    else:
        w = rng.uniform(0.0, 2 * np.pi, spec.num_weights)
    if batch is not None:
        x = x[:batch]
    return x, w


def native_api():
    """This package's IR namespace for ``build``."""
    from types import SimpleNamespace

    from . import ir, observables
    return SimpleNamespace(GateKind=ir.GateKind, Gate=ir.Gate, AngleExpression=ir.AngleExpression,
                           ParameterSet=ir.ParameterSet, Circuit=ir.Circuit,
                           Observable=observables.Observable)


def flops_per_sample(spec: ConfigSpec, K: int = 1) -> float:
    """SURVEY §8(d) algorithmic FP64 flops per sample:
    F = 2^n [6R + 6R(1+K) + 4 Rn K]; K = 1 (VJP) or M (Jacobian)."""
    R = spec.n * spec.layers * (1 + len(spec.trainable))
    Rn = R if spec.wrt_inputs else spec.n * spec.layers * len(spec.trainable)
    return float(2 ** spec.n) * (6 * R + 6 * R * (1 + K) + 4 * Rn * K)


def hbm_bytes_per_sample(spec: ConfigSpec, K: int = 1) -> float:
    """SURVEY §8(d) modelled HBM floor (n >= 13): 16·2^n·L·(2 + 2(1+K))."""
    if spec.n <= 12:
        return 0.0
    return 16.0 * 2 ** spec.n * spec.layers * (2 + 2 * (1 + K))
