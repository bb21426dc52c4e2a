"""Single-binding gradient API (gradients.py:204-283 of the reference):
``adjoint_gradients``, ``parameter_shift_gradients``, ``spsa_gradients`` and
``finite_difference_gradients`` for one full binding (every set, encoding
included), returning ``GradientResult(expectations (M,), {set: (M, size)})``.

All four run on the GPU engine as a batch of one row: adjoint through
``vqc_adjoint``, the others as forward launches over the angle circuit
(engine._run_shifted / device_row_angles). SPSA draws from
``default_rng(seed)`` itself, as the reference does for a single binding.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .engine import (BatchEngine, BatchRequest, WrtLayout, angle_circuit, default_engine,
                     device_row_angles)
from .ir import Circuit, ParameterSet, validate_binding
from .observables import ObservablePack

DEFAULT_SPSA_C = 0.01
DEFAULT_SPSA_SAMPLES = 1
DEFAULT_FD_STEP = 1e-4
_ENC = "__binding_row__"


@dataclass
class GradientResult:
    """Expectations (M,) plus per-set gradient arrays of shape (M, set.size)."""

    expectations: np.ndarray
    gradients: dict


def _as_batch(circuit: Circuit, binding, observables, wrt, engine):
    """(engine, one-row request, layout). The whole binding becomes the
    trainable values of a circuit whose sets are all trainable plus an empty
    encoding set appended last (flat offsets unchanged)."""
    validate_binding(circuit, binding)
    ObservablePack.from_observables(list(observables), circuit.num_qubits)
    sets = tuple(ParameterSet(s.name, s.size, "trainable") for s in circuit.parameter_sets)
    cached = circuit.__dict__.get("_single_binding")
    if cached is None:
        cached = Circuit(circuit.num_qubits, circuit.gates,
                         sets + (ParameterSet(_ENC, 0, "encoding"),))
        object.__setattr__(circuit, "_single_binding", cached)
    layout = WrtLayout.build(cached.compiled(), wrt)
    req = BatchRequest(cached, list(observables),
                       {s.name: np.asarray(binding[s.name], np.float64) for s in sets},
                       np.zeros((1, 0)), wrt=tuple(wrt))
    return engine or default_engine(), req, layout


def _result(expect, grad, layout) -> GradientResult:
    return GradientResult(np.asarray(expect, np.float64).reshape(-1),
                          {n: np.ascontiguousarray(grad[:, lo:hi]) for n, lo, hi in layout.slices})


def _empty(layout) -> GradientResult:
    return _result(np.zeros(0), np.zeros((0, layout.n_cols)), layout)


def _batch_result(res, layout) -> GradientResult:
    grad = (np.concatenate([res.gradients[n] for n, _, _ in layout.slices], axis=-1)[0]
            if layout.slices else np.zeros((res.expectations.shape[1], 0)))
    return _result(res.expectations[0], grad, layout)


def adjoint_gradients(circuit: Circuit, binding, observables, wrt,
                      engine: BatchEngine | None = None) -> GradientResult:
    """Reverse-sweep gradients (gradients.py:204-220)."""
    eng, req, layout = _as_batch(circuit, binding, observables, wrt, engine)
    if not req.observables:
        return _empty(layout)
    return _batch_result(eng.run_batch(req), layout)


def parameter_shift_gradients(circuit: Circuit, binding, observables, wrt,
                              engine: BatchEngine | None = None) -> GradientResult:
    """+-pi/2 shift rule per gate occurrence (gradients.py:223-240)."""
    eng, req, layout = _as_batch(circuit, binding, observables, wrt, engine)
    if not req.observables:
        return _empty(layout)
    req.method = "param-shift"
    return _batch_result(eng.run_batch(req), layout)


def spsa_gradients(circuit: Circuit, binding, observables, wrt, c: float = DEFAULT_SPSA_C,
                   samples: int = DEFAULT_SPSA_SAMPLES, seed: int = 0,
                   engine: BatchEngine | None = None) -> GradientResult:
    """Rademacher-direction estimate, rng = default_rng(seed) (gradients.py:243-266)."""
    if c <= 0:
        raise ValueError(f"perturbation magnitude c must be > 0, got {c}")
    if samples < 1:
        raise ValueError(f"samples must be >= 1, got {samples}")
    eng, req, layout = _as_batch(circuit, binding, observables, wrt, engine)
    if not req.observables:
        return _empty(layout)
    req.method, req.spsa_c, req.spsa_samples = "spsa", c, samples
    flat = eng.base_flat(req.circuit, req.trainable_values)
    if layout.n_cols == 0:
        return _batch_result(eng.run_batch(req), layout)
    if isinstance(seed, (int, np.integer)) and 0 <= int(seed) < 2 ** 64:
        draws = {"single_seed": int(seed)}       # native draws (vqc_spsa_signs)
    else:                                        # anything else default_rng accepts
        draws = {"rng_for_row": lambda b: np.random.default_rng(seed)}
    e, g = eng._run_shifted(req, req.circuit, req.observables, layout, flat, req.inputs, **draws)
    return _result(e[0], g[0], layout)


def finite_difference_gradients(circuit: Circuit, binding, observables, wrt,
                                h: float = DEFAULT_FD_STEP,
                                engine: BatchEngine | None = None) -> GradientResult:
    """Central differences per requested entry (gradients.py:269-283): the
    1 + 2C perturbed flats are one forward launch over the angle circuit."""
    import torch
    if h <= 0:
        raise ValueError(f"step h must be > 0, got {h}")
    eng, req, layout = _as_batch(circuit, binding, observables, wrt, engine)
    if not req.observables:
        return _empty(layout)
    comp = req.circuit.compiled()
    flat = eng.base_flat(req.circuit, req.trainable_values)
    C = layout.n_cols
    flats = np.repeat(flat[None], 1 + 2 * C, 0)
    for col, p in enumerate(layout.flat_of_col):
        flats[1 + 2 * col, p] = flat[p] + h
        flats[2 + 2 * col, p] = flat[p] - h
    _, rot = angle_circuit(req.circuit)
    ang = device_row_angles(comp, torch.from_numpy(flats).to(eng.device), rot)
    e = eng.forward_angle_rows(req.circuit, req.observables, ang)   # (1+2C, M)
    grad = np.empty((len(req.observables), C))
    for col in range(C):
        grad[:, col] = (e[1 + 2 * col] - e[2 + 2 * col]) / (2.0 * h)
    return _result(e[0], grad, layout)
