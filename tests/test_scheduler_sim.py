"""CPU check of the circuit -> device-program lowering (scheduler.cpp).

tests/native/program_sim.cpp interprets the emitted pass/segment/op program
semantically on a full state (test infrastructure, no GPU) and asserts the
structural invariants the sm_100a kernels rely on. Results must match the
oracle: reordering only commuting gates leaves outputs unchanged up to
rounding. Small tiles force the multi-pass (HBM-mode) schedule at small n.
"""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, close, oracle_batch

from paper_2404_06314_b200 import configs
from paper_2404_06314_b200.engine import WrtLayout, encoding_set
from paper_2404_06314_b200.observables import Observable, ObservablePack

_NATIVE = os.path.join(ROOT, "tests", "native")
_SO = os.path.join(_NATIVE, "_build", "libvqcsim.so")
_I64P = ctypes.POINTER(ctypes.c_int64)
_F64P = ctypes.POINTER(ctypes.c_double)


@pytest.fixture(scope="module")
def sim():
    srcs = [os.path.join(_NATIVE, "program_sim.cpp"),
            os.path.join(ROOT, "paper_2404_06314_b200", "csrc", "scheduler.cpp")]
    hdrs = [os.path.join(ROOT, "paper_2404_06314_b200", "csrc", f)
            for f in ("scheduler.h", "program.h")]
    if not os.path.exists(_SO) or any(os.path.getmtime(s) > os.path.getmtime(_SO) for s in srcs + hdrs):
        os.makedirs(os.path.dirname(_SO), exist_ok=True)
        subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-o", _SO, *srcs], check=True)
    lib = ctypes.CDLL(_SO)
    lib.sim_run.restype = ctypes.c_int
    return lib


def run_sim(lib, circuit, observables, flat, wrt, tile_qubits=11, smem_max=12, upstream=None, reg_slots=4):
    c = circuit.compiled()
    pack = ObservablePack.from_observables(observables, circuit.num_qubits)
    layout = WrtLayout.build(c, wrt)
    M = len(observables)
    K = 1 if upstream is not None else M
    expect = np.zeros(max(M, 1))
    grad = np.zeros((max(K, 1), max(layout.n_cols, 1)))
    stats = np.zeros(4, np.int64)
    err = ctypes.create_string_buffer(256)
    arrs = [np.ascontiguousarray(a, dtype=t) for a, t in (
        (c.kinds, np.int64), (c.q0, np.int64), (c.q1, np.int64), (c.coeff, np.float64),
        (c.f_offs, np.int64), (c.f_idx if len(c.f_idx) else [0], np.int64),
        (layout.wrt_col if len(layout.wrt_col) else [-1], np.int64),
        (pack.term_offs, np.int64), (pack.coeffs if len(pack.coeffs) else [0.0], np.float64),
        (pack.sign_masks if len(pack.sign_masks) else [0], np.int64),
        (flat if len(flat) else [0.0], np.float64))]
    up = None if upstream is None else np.ascontiguousarray(upstream, np.float64)
    rc = lib.sim_run(
        circuit.num_qubits, ctypes.c_int64(len(c.kinds)), arrs[0].ctypes.data_as(_I64P),
        arrs[1].ctypes.data_as(_I64P), arrs[2].ctypes.data_as(_I64P), arrs[3].ctypes.data_as(_F64P),
        arrs[4].ctypes.data_as(_I64P), arrs[5].ctypes.data_as(_I64P), ctypes.c_int64(c.total_params),
        arrs[6].ctypes.data_as(_I64P), tile_qubits, smem_max, reg_slots, M, arrs[7].ctypes.data_as(_I64P),
        arrs[8].ctypes.data_as(_F64P), arrs[9].ctypes.data_as(_I64P), arrs[10].ctypes.data_as(_F64P),
        None if up is None else up.ctypes.data_as(_F64P), expect.ctypes.data_as(_F64P),
        grad.ctypes.data_as(_F64P), stats.ctypes.data_as(_I64P), err, 256)
    if rc != 0:
        raise AssertionError(err.value.decode())
    return expect[:M], grad[:K, :layout.n_cols], stats, layout


def _flat_row(circuit, trainable, x_row):
    enc = encoding_set(circuit)
    b = dict(trainable)
    b[enc.name] = np.asarray(x_row, np.float64)
    return circuit.compiled().flat_values(b)


@pytest.mark.parametrize("cfg_id", [1, 2, 3, 4])
@pytest.mark.parametrize("tile", [None, 6])
@pytest.mark.parametrize("reg_slots", [4, 5])
def test_configs(sim, cfg_id, tile, reg_slots):
    spec = configs.CONFIGS[cfg_id]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=2)
    e_ref, j_ref = oracle_batch(circ, obs, {"w": w}, x, wrt)
    kw = {} if tile is None else {"tile_qubits": tile, "smem_max": min(tile, spec.n - 1)}
    kw["reg_slots"] = reg_slots
    for b in range(len(x)):
        flat = _flat_row(circ, {"w": w}, x[b])
        e, jac, stats, layout = run_sim(sim, circ, obs, flat, wrt, **kw)
        assert close(e, e_ref[b]) < 1e-12
        full = np.concatenate([j_ref[n][b] for n, _, _ in layout.slices], axis=1)
        assert close(jac, full) < 1e-12
        u = np.linspace(-1, 1, len(obs))
        _, vjp, _, _ = run_sim(sim, circ, obs, flat, wrt, upstream=u, **kw)
        assert close(vjp[0], u @ full) < 1e-12


def _random(rng, n, n_gates):
    from paper_2404_06314_b200.ir import AngleExpression, Circuit, Gate, GateKind, ParameterSet
    sets = (ParameterSet("s", 3, "encoding"), ParameterSet("a", 4), ParameterSet("b", 2))
    pool = [(s.name, i) for s in sets for i in range(s.size)]
    gates = []
    for _ in range(n_gates):
        kind = list(GateKind)[int(rng.integers(7))]
        if kind.num_qubits == 2 and n < 2:
            kind = GateKind.RZ
        if kind.num_qubits == 2:
            a, b = rng.permutation(n)[:2]
            gates.append(Gate(kind, (int(a), int(b))))
        elif kind.is_rotation:
            refs = []
            for _ in range(int(rng.integers(0, 4))):
                r = pool[int(rng.integers(len(pool)))]
                if r not in refs:
                    refs.append(r)
            gates.append(Gate(kind, (int(rng.integers(n)),),
                              AngleExpression(float(rng.uniform(-2, 2)), tuple(refs))))
        else:
            gates.append(Gate(kind, (int(rng.integers(n)),)))
    circ = Circuit(n, tuple(gates), sets)
    obs = [Observable(((float(rng.uniform(-1, 1)),
                        "".join("Z" if rng.random() < 0.5 else "I" for _ in range(n))),
                       (0.5, "Z" + "I" * (n - 1))))
           for _ in range(2)]
    return circ, obs, {"a": rng.uniform(-2, 2, 4), "b": rng.uniform(-2, 2, 2)}


@pytest.mark.parametrize("n", list(range(1, 11)))
@pytest.mark.parametrize("tile", [4, 6, 11])
@pytest.mark.parametrize("reg_slots", [3, 4, 5])
def test_random_circuits(sim, n, tile, reg_slots):
    if tile <= 3 or (tile < n and tile < 4):
        pytest.skip("tile too small")
    if tile < reg_slots + 2 and tile < n:
        pytest.skip("tile too small for the register slots")
    rng = np.random.default_rng(1000 * n + tile)
    for rep in range(2):
        circ, obs, tr = _random(rng, n, int(rng.integers(0, 60)))
        x = rng.uniform(-2, 2, (1, 3))
        wrt = ("a", "s", "b")
        e_ref, j_ref = oracle_batch(circ, obs, tr, x, wrt)
        flat = _flat_row(circ, tr, x[0])
        smem_max = 12 if tile >= n else min(tile, n - 1)
        e, jac, _, layout = run_sim(sim, circ, obs, flat, wrt, tile_qubits=min(tile, n),
                                    smem_max=smem_max, reg_slots=reg_slots)
        assert close(e, e_ref[0]) < 1e-12
        full = np.concatenate([j_ref[k][0] for k, _, _ in layout.slices], axis=1)
        assert close(jac, full) < 1e-12


def test_schedule_is_compact_for_cfg4(sim):
    """The HBM schedule must not degenerate to a pass per gate."""
    spec = configs.CONFIGS[4]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=1)
    flat = _flat_row(circ, {"w": w}, x[0])
    _, _, stats, _ = run_sim(sim, circ, obs, flat, wrt)
    passes, segments = int(stats[0]), int(stats[1])
    assert passes <= 3 * spec.layers, passes
    assert segments <= 8 * spec.layers * 3, segments


def test_pass_splitting_of_whole_state_tiles(sim, monkeypatch):
    """Whole-state tiles (n <= 12 on the pass kernels) cut passes of more than
    VQC_PASS_SEGMENTS segments into several passes over the same qubits (a
    bound on the JIT compile time of deep circuits): same results, more
    passes, every structural invariant still checked by the simulator."""
    spec = configs.CONFIGS[3]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=1)
    e_ref, j_ref = oracle_batch(circ, obs, {"w": w}, x, wrt)
    flat = _flat_row(circ, {"w": w}, x[0])
    kw = {"tile_qubits": 12, "smem_max": 7, "reg_slots": 3}
    _, _, stats_one, _ = run_sim(sim, circ, obs, flat, wrt, **kw)
    monkeypatch.setenv("VQC_PASS_SEGMENTS", "5")
    e, jac, stats_cut, layout = run_sim(sim, circ, obs, flat, wrt, **kw)
    assert stats_one[0] == 1 and stats_cut[0] > 4          # passes
    full = np.concatenate([j_ref[n][0] for n, _, _ in layout.slices], axis=1)
    assert close(e, e_ref[0]) < 1e-12 and close(jac, full) < 1e-12
