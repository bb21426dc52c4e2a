"""TEST INFRASTRUCTURE — the CPU oracle's Python face (not product code).

Loads ``oracle/_build/liborc.so`` (``oracle/vqc_oracle.c``, a plain-C
restatement of the reference kernels in vqckit/_kernels.py) through ctypes and
exposes the reference's flat-array semantics:

* ``run_batch``  — batch.py:147-217 (``BatchEngine.run_batch``, adjoint
  method): (B, M) expectations and the (B, M, n_cols) Jacobian, rows split
  over threads exactly as batch.py:54-72 does.
* ``evolve``     — circuit.py:229-245 (one forward evolution).
* ``apply_gate`` — statevector.py:404-420.
* ``expval``     — _kernels.py:182-198.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU arms import this.
The lowered arrays it consumes follow circuit.py:168-216 (CompiledCircuit)
and observables.py:132-167 (ObservablePack).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liborc.so")
_lib = None

_I64P = ctypes.POINTER(ctypes.c_int64)
_F64P = ctypes.POINTER(ctypes.c_double)


class _OrcProblem(ctypes.Structure):
    _fields_ = [
        ("n_qubits", ctypes.c_int64), ("n_gates", ctypes.c_int64),
        ("kinds", _I64P), ("q0", _I64P), ("q1", _I64P), ("gen_axis", _I64P),
        ("coeff", _F64P), ("f_offs", _I64P), ("f_idx", _I64P),
        ("total_params", ctypes.c_int64),
        ("n_obs", ctypes.c_int64), ("term_offs", _I64P), ("t_coeffs", _F64P),
        ("t_xmask", _I64P), ("t_smask", _I64P), ("t_phases", _F64P),
    ]


def build() -> str:
    """Compile the oracle with its Makefile (gcc, OpenMP) if needed."""
    if not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH)
            < os.path.getmtime(os.path.join(_HERE, "vqc_oracle.c"))):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.orc_run_batch.restype = ctypes.c_int
        _lib.orc_run_batch.argtypes = [
            ctypes.POINTER(_OrcProblem), _F64P, ctypes.c_int64, ctypes.c_int64,
            _F64P, ctypes.c_int64, _I64P, ctypes.c_int64, ctypes.c_int,
            _F64P, _F64P]
        _lib.orc_evolve.restype = None
        _lib.orc_evolve.argtypes = [ctypes.POINTER(_OrcProblem), _F64P, _F64P]
        _lib.orc_apply_gate.restype = None
        _lib.orc_apply_gate.argtypes = [_F64P, ctypes.c_int, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_double, ctypes.c_int]
        _lib.orc_expval_terms.restype = None
        _lib.orc_expval_terms.argtypes = [_F64P, ctypes.c_int, _F64P, _I64P, _I64P,
                                          _F64P, ctypes.c_int64, ctypes.c_int64, _F64P]
    return _lib


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t):
    return a.ctypes.data_as(t)


@dataclass
class Lowered:
    """Reference-layout arrays: CompiledCircuit + ObservablePack."""

    n_qubits: int
    kinds: np.ndarray
    q0: np.ndarray
    q1: np.ndarray
    gen_axis: np.ndarray
    coeff: np.ndarray
    f_offs: np.ndarray
    f_idx: np.ndarray
    total_params: int
    term_offs: np.ndarray
    t_coeffs: np.ndarray
    t_xmask: np.ndarray
    t_smask: np.ndarray
    t_phases: np.ndarray   # (T, 2) float64 re/im

    def __post_init__(self):
        self.kinds, self.q0, self.q1 = _i64(self.kinds), _i64(self.q0), _i64(self.q1)
        self.gen_axis, self.f_offs, self.f_idx = (_i64(self.gen_axis), _i64(self.f_offs),
                                                  _i64(self.f_idx))
        self.coeff = _f64(self.coeff)
        self.term_offs, self.t_xmask, self.t_smask = (_i64(self.term_offs),
                                                      _i64(self.t_xmask), _i64(self.t_smask))
        self.t_coeffs = _f64(self.t_coeffs)
        ph = np.asarray(self.t_phases)
        if np.iscomplexobj(ph):
            ph = np.stack([ph.real, ph.imag], axis=-1)
        self.t_phases = _f64(ph.reshape(-1, 2))

    @property
    def n_obs(self) -> int:
        return len(self.term_offs) - 1

    def struct(self) -> _OrcProblem:
        return _OrcProblem(
            self.n_qubits, len(self.kinds), _p(self.kinds, _I64P), _p(self.q0, _I64P),
            _p(self.q1, _I64P), _p(self.gen_axis, _I64P), _p(self.coeff, _F64P),
            _p(self.f_offs, _I64P), _p(self.f_idx, _I64P), self.total_params,
            self.n_obs, _p(self.term_offs, _I64P), _p(self.t_coeffs, _F64P),
            _p(self.t_xmask, _I64P), _p(self.t_smask, _I64P), _p(self.t_phases, _F64P))


def run_batch(low: Lowered, base_flat, enc_off: int, enc_size: int, inputs,
              wrt_col, threads: int | None = None):
    """batch.py:147-217 semantics; returns (expect (B,M), jac (B,M,n_cols))."""
    inputs = _f64(np.asarray(inputs, np.float64).reshape(len(inputs), enc_size))
    base_flat = _f64(base_flat)
    wrt_col = _i64(wrt_col)
    n_cols = int(wrt_col.max(initial=-1)) + 1
    B, M = inputs.shape[0], low.n_obs
    expect = np.zeros((B, M))
    jac = np.zeros((B, M, n_cols))
    if threads is None:
        threads = os.cpu_count() or 1
    prob = low.struct()
    rc = lib().orc_run_batch(ctypes.byref(prob), _p(base_flat, _F64P), enc_off, enc_size,
                             _p(inputs, _F64P), B, _p(wrt_col, _I64P), n_cols,
                             int(threads), _p(expect, _F64P), _p(jac, _F64P))
    if rc < 0:
        raise ValueError(f"batch input {-1 - rc} failed: imaginary expectation")
    return expect, jac


def evolve(low: Lowered, flat) -> np.ndarray:
    flat = _f64(flat)
    out = np.zeros(2 << low.n_qubits)
    prob = low.struct()
    lib().orc_evolve(ctypes.byref(prob), _p(flat, _F64P), _p(out, _F64P))
    return out.view(np.complex128)


def apply_gate(state: np.ndarray, kind: int, q0: int, q1: int = 0, angle: float = 0.0,
               adjoint: bool = False) -> np.ndarray:
    st = np.ascontiguousarray(state, dtype=np.complex128).copy()
    n = int(np.log2(st.shape[0]))
    lib().orc_apply_gate(st.view(np.float64).ctypes.data_as(_F64P), n, kind, q0, q1,
                         float(angle), int(adjoint))
    return st


def expval(state: np.ndarray, coeffs, x_masks, sign_masks, phases) -> complex:
    st = np.ascontiguousarray(state, dtype=np.complex128)
    n = int(np.log2(st.shape[0]))
    coeffs, xm, sm = _f64(coeffs), _i64(x_masks), _i64(sign_masks)
    ph = np.asarray(phases)
    if np.iscomplexobj(ph):
        ph = np.stack([ph.real, ph.imag], axis=-1)
    ph = _f64(ph.reshape(-1, 2))
    out = np.zeros(2)
    lib().orc_expval_terms(st.view(np.float64).ctypes.data_as(_F64P), n, _p(coeffs, _F64P),
                           _p(xm, _I64P), _p(sm, _I64P), _p(ph, _F64P), 0, len(coeffs),
                           _p(out, _F64P))
    return complex(out[0], out[1])


def vjp(upstream: np.ndarray, jac: np.ndarray) -> np.ndarray:
    """model.py:141-142 / engine_server.py:135-136 contraction, per row."""
    return np.einsum("bm,bmp->bp", upstream, jac)


# -- shift-rule and SPSA gradients (gradients.py:121-201), small cases only ----

def _angles(low: Lowered, flat) -> np.ndarray:
    """compute_angles (_kernels.py:128-134): coefficient first, factors in order."""
    out = np.zeros(len(low.kinds))
    for g in range(len(low.kinds)):
        a = low.coeff[g]
        for t in range(low.f_offs[g], low.f_offs[g + 1]):
            a *= flat[low.f_idx[t]]
        out[g] = a
    return out


def _run_angles(low: Lowered, angles) -> np.ndarray:
    """run_program on explicit per-gate angles (circuit.py:229-245)."""
    st = np.zeros(1 << low.n_qubits, np.complex128)
    st[0] = 1.0
    for g in range(len(low.kinds)):
        st = apply_gate(st, int(low.kinds[g]), int(low.q0[g]), int(low.q1[g]), float(angles[g]))
    return st


def _pack_expectations(low: Lowered, st) -> np.ndarray:
    """pack_expectations (gradients.py:84-99)."""
    out = np.empty(low.n_obs)
    for m in range(low.n_obs):
        lo, hi = low.term_offs[m], low.term_offs[m + 1]
        out[m] = expval(st, low.t_coeffs[lo:hi], low.t_xmask[lo:hi], low.t_smask[lo:hi],
                        np.asarray(low.t_phases).reshape(-1, 2)[lo:hi]).real
    return out


def param_shift_row(low: Lowered, flat, wrt_col):
    """param_shift_flat (gradients.py:137-160) for one row: (expect (M,), grad (M, n_cols))."""
    flat = np.asarray(flat, np.float64)
    n_cols = int(np.max(wrt_col, initial=-1)) + 1
    angles = _angles(low, flat)
    expect = _pack_expectations(low, _run_angles(low, angles))
    grad = np.zeros((low.n_obs, n_cols))
    for g in range(len(low.kinds)):
        if low.gen_axis[g] < 0:
            continue
        lo, hi = low.f_offs[g], low.f_offs[g + 1]
        partials = []
        for t in range(lo, hi):                       # _occurrence_partials (121-134)
            col = wrt_col[low.f_idx[t]]
            if col < 0:
                continue
            partial = low.coeff[g]
            for u in range(lo, hi):
                if u != t:
                    partial *= flat[low.f_idx[u]]
            partials.append((int(col), float(partial)))
        if not partials:
            continue
        base = angles[g]
        angles[g] = base + 0.5 * np.pi
        f_plus = _pack_expectations(low, _run_angles(low, angles))
        angles[g] = base - 0.5 * np.pi
        f_minus = _pack_expectations(low, _run_angles(low, angles))
        angles[g] = base
        occ = 0.5 * (f_plus - f_minus)
        for col, partial in partials:
            grad[:, col] += occ * partial
    return expect, grad


def spsa_row(low: Lowered, flat, flat_of_col, c: float, samples: int, rng):
    """spsa_flat (gradients.py:180-201) for one row; ``rng`` is the row's
    default_rng(mix_seed(seed, b)) (batch.py:197)."""
    flat = np.array(flat, np.float64)
    idx = np.asarray(flat_of_col, np.int64)
    expect = _pack_expectations(low, _run_angles(low, _angles(low, flat)))
    grad = np.zeros((low.n_obs, len(idx)))
    base = flat[idx].copy()
    for _ in range(samples):
        delta = rng.integers(0, 2, size=len(idx)).astype(np.float64)
        delta = 2.0 * delta - 1.0
        flat[idx] = base + c * delta
        f_plus = _pack_expectations(low, _run_angles(low, _angles(low, flat)))
        flat[idx] = base - c * delta
        f_minus = _pack_expectations(low, _run_angles(low, _angles(low, flat)))
        flat[idx] = base
        grad += np.outer(f_plus - f_minus, 1.0 / (2.0 * c * delta))
    grad /= samples
    return expect, grad
