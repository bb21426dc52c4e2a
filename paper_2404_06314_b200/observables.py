"""Pauli-sum observables (reference: vqckit/observables.py, statevector.py:105-128).

An observable is a real-weighted sum of Pauli strings; character k acts on
qubit k. ``pack_observables`` produces the reference's ObservablePack layout
(observables.py:132-167) for ``vqc_plan_create``. The GPU path evaluates
Z strings (x_mask == 0); strings with X/Y letters are rejected at plan time.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def pauli_masks(pauli_string: str) -> tuple[int, int, complex]:
    """(x_mask, sign_mask, i^{#Y}) with P|b> = phase (-1)^{popcount(b & sign)} |b ^ x>."""
    x_mask = sign_mask = n_y = 0
    for q, letter in enumerate(pauli_string):
        bit = 1 << q
        if letter == "I":
            continue
        if letter == "X":
            x_mask |= bit
        elif letter == "Y":
            x_mask |= bit
            sign_mask |= bit
            n_y += 1
        elif letter == "Z":
            sign_mask |= bit
        else:
            raise ValueError(f"invalid Pauli letter {letter!r} in {pauli_string!r}")
    return x_mask, sign_mask, 1j ** (n_y % 4)


@dataclass(frozen=True)
class Observable:
    terms: tuple[tuple[float, str], ...]

    def __post_init__(self):
        terms = tuple((float(c), str(p)) for c, p in self.terms)
        object.__setattr__(self, "terms", terms)
        if not terms:
            raise ValueError("observable needs at least one term")
        width = len(terms[0][1])
        for _, string in terms:
            if len(string) != width:
                raise ValueError(f"inconsistent Pauli string lengths: {string!r} vs length {width}")
            pauli_masks(string)

    @property
    def num_qubits(self) -> int:
        return len(self.terms[0][1])

    @property
    def is_z_only(self) -> bool:
        return all(set(s) <= {"I", "Z"} for _, s in self.terms)


def parse_observable(text: str) -> Observable:
    """``"0.5*ZZI + IIZ"`` style text (observables.py:70-92)."""
    terms = []
    for raw in text.split("+"):
        term = raw.strip()
        if not term:
            raise ValueError(f"empty term in observable {text!r}")
        coeff, string = 1.0, term
        if "*" in term:
            head, _, string = term.partition("*")
            try:
                coeff = float(head.strip())
            except ValueError as exc:
                raise ValueError(f"bad coefficient in term {term!r}") from exc
            string = string.strip()
        if not string or any(ch not in "IXYZ" for ch in string):
            raise ValueError(f"bad Pauli string in term {term!r}")
        terms.append((coeff, string))
    if len({len(s) for _, s in terms}) > 1:
        raise ValueError(f"inconsistent string lengths in {text!r}")
    return Observable(tuple(terms))


def z_observable(num_qubits: int, qubits, coeff: float = 1.0) -> Observable:
    """coeff * prod_{q in qubits} Z_q as a one-term observable."""
    chars = ["I"] * num_qubits
    for q in qubits:
        chars[q] = "Z"
    return Observable(((coeff, "".join(chars)),))


@dataclass(frozen=True, eq=False)
class ObservablePack:
    """M observables as contiguous term arrays (observables.py:132-167)."""

    num_obs: int
    num_qubits: int
    term_offs: np.ndarray
    coeffs: np.ndarray
    x_masks: np.ndarray
    sign_masks: np.ndarray
    phases: np.ndarray  # (T, 2) float64: re, im of i^{#Y}

    @staticmethod
    def from_observables(observables, num_qubits: int) -> "ObservablePack":
        observables = list(observables)
        offs = [0]
        coeffs, xm, sm, ph = [], [], [], []
        for obs in observables:
            if obs.num_qubits != num_qubits:
                raise ValueError(f"observable on {obs.num_qubits} qubits does not match "
                                 f"{num_qubits}-qubit circuit")
            for c, string in obs.terms:
                x, s, p = pauli_masks(string)
                coeffs.append(c)
                xm.append(x)
                sm.append(s)
                ph.append((p.real, p.imag))
            offs.append(len(coeffs))
        return ObservablePack(
            len(observables), num_qubits, np.asarray(offs, np.int64),
            np.asarray(coeffs, np.float64), np.asarray(xm, np.int64), np.asarray(sm, np.int64),
            np.asarray(ph, np.float64).reshape(-1, 2))
