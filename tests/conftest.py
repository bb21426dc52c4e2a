"""Shared test helpers. The CPU oracle (oracle/) is the checker here."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs libvqc.so kernels)")


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.build()
    return oracle


def lowered(circuit, observables):
    """Oracle input (reference array layout) from this package's compiler."""
    from oracle.oracle import Lowered
    from paper_2404_06314_b200.observables import ObservablePack
    c = circuit.compiled()
    pack = ObservablePack.from_observables(observables, circuit.num_qubits)
    return Lowered(c.num_qubits, c.kinds, c.q0, c.q1, c.gen_axis, c.coeff, c.f_offs, c.f_idx,
                   c.total_params, pack.term_offs, pack.coeffs, pack.x_masks, pack.sign_masks,
                   pack.phases)


def oracle_batch(circuit, observables, trainable, inputs, wrt, threads=None):
    """batch.py semantics via the oracle: (expect (B,M), {set: (B,M,size)})."""
    from oracle import oracle
    from paper_2404_06314_b200.engine import WrtLayout, encoding_set
    comp = circuit.compiled()
    enc = encoding_set(circuit)
    binding = dict(trainable)
    binding[enc.name] = np.zeros(enc.size)
    base = comp.flat_values(binding)
    layout = WrtLayout.build(comp, wrt)
    off, size = comp.offsets[enc.name]
    expect, jac = oracle.run_batch(lowered(circuit, observables), base, off, size,
                                   np.asarray(inputs, np.float64).reshape(len(inputs), size),
                                   layout.wrt_col, threads)
    return expect, {n: jac[:, :, lo:hi] for n, lo, hi in layout.slices}


def close(a, b, tol=1e-10):
    """|a - b| <= tol * max(1, |b|) elementwise (SURVEY §8c parity protocol)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    err = np.abs(a - b) / np.maximum(1.0, np.abs(b))
    return float(err.max(initial=0.0))
