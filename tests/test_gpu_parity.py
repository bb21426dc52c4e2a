"""GPU parity: libvqc.so (through the C ABI) vs the oracle / reference goldens.

Tolerance (BASELINE north star, complex128): |gpu - ref| <= 1e-10 * max(1, |ref|).
"""

import ast
import os

import numpy as np
import pytest

from conftest import GOLDEN, close, oracle_batch

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2404_06314_b200 import build
    build.build()
    return torch


def _engine():
    from paper_2404_06314_b200 import BatchEngine
    return BatchEngine()


def _request(circ, obs, w, x, wrt):
    from paper_2404_06314_b200 import BatchRequest
    return BatchRequest(circ, obs, w, x, wrt=wrt)


def _golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} missing")
    return np.load(path)


@pytest.mark.parametrize("cfg_id", [1, 2, 3, 4, 5])
def test_config_golden_jacobian(torch_cuda, cfg_id):
    """Per-row expectations and Jacobians on the golden rows (reference run_batch)."""
    from paper_2404_06314_b200 import configs
    g = _golden(f"cfg{cfg_id}.npz")
    spec = configs.CONFIGS[cfg_id]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    res = _engine().run_batch(_request(circ, obs, {"w": g["w"]}, g["x_rows"], wrt))
    assert close(res.expectations, g["expect"]) < TOL
    assert close(res.gradients["w"], g["jac_w"]) < TOL
    if "jac_x" in g:
        assert close(res.gradients["x"], g["jac_x"]) < TOL
    fwd = _engine().run_batch(_request(circ, obs, {"w": g["w"]}, g["x_rows"], ()))
    assert close(fwd.expectations, g["expect_fwd"]) < TOL


@pytest.mark.parametrize("cfg_id", [1, 2, 3, 4, 5])
def test_config_golden_vjp(torch_cuda, cfg_id):
    """VJP mode (upstream = ones) through vqc_adjoint vs the reference einsum."""
    torch = torch_cuda
    from paper_2404_06314_b200 import configs
    g = _golden(f"cfg{cfg_id}.npz")
    spec = configs.CONFIGS[cfg_id]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    eng = _engine()
    plan, layout = eng.plans.get(circ, obs, wrt, eng.device)
    x = g["x_rows"]
    B, M = len(x), len(obs)
    dev = eng.device
    flat = eng.base_flat(circ, {"w": g["w"]})
    d_x = torch.from_numpy(x).to(dev)
    d_w = torch.from_numpy(flat).to(dev)
    up = torch.ones((B, M), dtype=torch.float64, device=dev)
    rows = torch.empty((B, layout.n_cols), dtype=torch.float64, device=dev)
    vsum = torch.empty((layout.n_cols,), dtype=torch.float64, device=dev)
    expect = torch.empty((B, M), dtype=torch.float64, device=dev)
    from paper_2404_06314_b200 import native
    ws = torch.empty(plan.workspace_bytes(B, native.VQC_MODE_VJP), dtype=torch.uint8, device=dev)
    plan.adjoint(d_x, d_w, up, expect, None, rows, vsum, ws, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert close(expect.cpu().numpy(), g["expect"]) < TOL
    name_cols = {n: (lo, hi) for n, lo, hi in layout.slices}
    lo, hi = name_cols["w"]
    assert close(vsum.cpu().numpy()[lo:hi], g["vjp_w"]) < TOL
    if "vjp_x_rows" in g:
        lo, hi = name_cols["x"]
        assert close(rows.cpu().numpy()[:, lo:hi], g["vjp_x_rows"]) < TOL


def _vjp_device(torch, eng, circ, obs, wrt, w, x, up):
    """vqc_adjoint in VJP mode on device buffers: (expect, per-row VJP rows, summed VJP)."""
    from paper_2404_06314_b200 import native
    plan, layout = eng.plans.get(circ, obs, wrt, eng.device)
    dev = eng.device
    B, M = len(x), len(obs)
    flat = eng.base_flat(circ, w if isinstance(w, dict) else {"w": w})
    d_x, d_w = torch.from_numpy(x).to(dev), torch.from_numpy(flat).to(dev)
    d_up = torch.from_numpy(np.ascontiguousarray(up)).to(dev)
    rows = torch.empty((B, layout.n_cols), dtype=torch.float64, device=dev)
    vsum = torch.empty((layout.n_cols,), dtype=torch.float64, device=dev)
    expect = torch.empty((B, M), dtype=torch.float64, device=dev)
    ws = torch.empty(plan.workspace_bytes(B, native.VQC_MODE_VJP), dtype=torch.uint8, device=dev)
    plan.adjoint(d_x, d_w, d_up, expect, None, rows, vsum, ws, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return expect.cpu().numpy(), rows.cpu().numpy(), vsum.cpu().numpy()


@pytest.mark.parametrize("cfg_id", [1, 2, 3])
def test_config_full_batch_vs_oracle(torch_cuda, cfg_id):
    """SURVEY §8(c) protocol: the FULL batch of cfg1-3 (cfg3: 4096 rows, so
    every CTA index of the on-chip kernel, rows 4032-4095 included) in
    Jacobian mode and in VJP mode with a row-dependent upstream, against the
    oracle (itself pinned to the reference goldens)."""
    torch = torch_cuda
    from paper_2404_06314_b200 import configs
    spec = configs.CONFIGS[cfg_id]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec)
    e_ref, j_ref = oracle_batch(circ, obs, {"w": w}, x, wrt)
    eng = _engine()
    res = eng.run_batch(_request(circ, obs, {"w": w}, x, wrt))
    assert res.expectations.shape == (spec.batch, len(obs))
    assert close(res.expectations, e_ref) < TOL
    for k in wrt:
        assert close(res.gradients[k], j_ref[k]) < TOL
    hi = slice(spec.batch - 64, spec.batch)   # the last CTAs of the launch
    for k in wrt:
        assert close(res.gradients[k][hi], j_ref[k][hi]) < TOL
    up = np.random.default_rng(cfg_id).normal(size=(spec.batch, len(obs)))
    e, rows, vsum = _vjp_device(torch, eng, circ, obs, wrt, w, x, up)
    ref_rows = np.concatenate([np.einsum("bm,bmp->bp", up, j_ref[k]) for k in wrt], axis=1)
    assert close(e, e_ref) < TOL
    assert close(rows, ref_rows) < TOL
    assert close(vsum, ref_rows.sum(axis=0)) < 1e-10 * max(1.0, np.abs(ref_rows).sum(axis=0).max())


def test_combined_observable_vjp_matches_reference_call(torch_cuda):
    """The VJP kernel (one bra seeded with sum_m O_m psi) equals the
    reference's own VJP-equivalent call, run_batch with one combined
    observable (goldens comb_*, cfg2 and cfg4)."""
    torch = torch_cuda
    from paper_2404_06314_b200 import configs
    for cfg_id in (2, 4):
        g = _golden(f"cfg{cfg_id}.npz")
        if "comb_vjp_w" not in g.files:
            pytest.skip("goldens predate the combined-observable fixtures")
        spec = configs.CONFIGS[cfg_id]
        circ, obs, wrt = configs.build(spec, configs.native_api())
        x = g["x_rows"]
        e, rows, vsum = _vjp_device(torch, _engine(), circ, obs, wrt, g["w"], x,
                                    np.ones((len(x), len(obs))))
        P = spec.num_weights
        assert close(e.sum(axis=1), g["comb_expect"][:, 0]) < TOL
        assert close(vsum[:P], g["comb_vjp_w"]) < TOL
        assert close(rows[:, P:], g["comb_vjp_x_rows"]) < TOL


def _random_cases():
    path = os.path.join(GOLDEN, "random.npz")
    if not os.path.exists(path):
        return []
    g = np.load(path)
    return list(range(int(g["count"])))


@pytest.mark.parametrize("idx", _random_cases())
def test_random_circuits_vs_reference(torch_cuda, idx):
    """Random circuits over RX RY RZ CNOT H X, shared/product parameters, Pauli sums."""
    from paper_2404_06314_b200 import ir
    from paper_2404_06314_b200.observables import Observable
    g = np.load(os.path.join(GOLDEN, "random.npz"))
    p = f"c{idx}_"
    circ = ir.circuit_from_dict(ast.literal_eval(str(g[p + "doc"])))
    obs = [Observable(t) for t in ast.literal_eval(str(g[p + "obs"]))]
    trainable = {"theta": g[p + "theta"], "lam": g[p + "lam"]}
    res = _engine().run_batch(_request(circ, obs, trainable, g[p + "inputs"], ("theta", "lam", "s")))
    assert close(res.expectations, g[p + "expect"]) < TOL
    for name in ("theta", "lam", "s"):
        assert close(res.gradients[name], g[p + "jac_" + name]) < TOL


def _rand_circuit(rng, n, n_gates, with_cz=True):
    from paper_2404_06314_b200.ir import AngleExpression, Circuit, Gate, GateKind, ParameterSet
    sets = (ParameterSet("s", 4, "encoding"), ParameterSet("a", 5), ParameterSet("b", 3))
    pool = [(s.name, i) for s in sets for i in range(s.size)]
    kinds = list(GateKind) if with_cz else [k for k in GateKind if k != GateKind.CZ]
    gates = []
    for _ in range(n_gates):
        kind = kinds[int(rng.integers(len(kinds)))]
        if kind.num_qubits == 2 and n < 2:
            kind = GateKind.H
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
    trainable = {"a": rng.uniform(-2, 2, 5), "b": rng.uniform(-2, 2, 3)}
    return circ, trainable


def _z_obs(rng, n, m):
    from paper_2404_06314_b200.observables import Observable
    out = []
    for _ in range(m):
        terms = []
        for _ in range(int(rng.integers(1, 4))):
            terms.append((float(rng.uniform(-2, 2)),
                          "".join("Z" if rng.random() < 0.4 else "I" for _ in range(n))))
        out.append(Observable(tuple(terms)))
    return out


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8, 11, 12, 13, 14, 15])
def test_random_with_cz_vs_oracle(torch_cuda, n):
    """All gate kinds incl. CZ; n spans the on-chip (<=12) and HBM-pass (>=13) paths."""
    rng = np.random.default_rng(100 + n)
    circ, trainable = _rand_circuit(rng, n, 30 + 4 * n)
    obs = _z_obs(rng, n, 3)
    x = rng.uniform(-2, 2, (5, 4))
    wrt = ("a", "b", "s")
    e_ref, j_ref = oracle_batch(circ, obs, trainable, x, wrt)
    res = _engine().run_batch(_request(circ, obs, trainable, x, wrt))
    assert close(res.expectations, e_ref) < TOL
    for k in wrt:
        assert close(res.gradients[k], j_ref[k]) < TOL


def _pauli_obs(rng, n, m):
    from paper_2404_06314_b200.observables import Observable
    out = []
    for _ in range(m):
        terms = []
        for _ in range(int(rng.integers(1, 4))):
            terms.append((float(rng.uniform(-2, 2)), "".join("IXYZ"[int(rng.integers(4))] for _ in range(n))))
        out.append(Observable(tuple(terms)))
    return out


@pytest.mark.parametrize("n", [8, 9, 10, 11, 12])
def test_whole_state_tile_general_observables(torch_cuda, n):
    """8 <= n <= 12 run the pass kernels on one tile holding the whole state
    (n <= 10: forward and adjoint in one kernel; 11, 12: separate 4-slot
    forward kernel, 256 / 512-thread CTAs with thread-group barriers): general
    X/Y/Z strings, Jacobians and a VJP with a row-dependent upstream."""
    rng = np.random.default_rng(700 + n)
    circ, trainable = _rand_circuit(rng, n, 40 + 4 * n)
    obs = _pauli_obs(rng, n, 3)
    x = rng.uniform(-2, 2, (6, 4))
    wrt = ("a", "b", "s")
    e_ref, j_ref = oracle_batch(circ, obs, trainable, x, wrt)
    res = _engine().run_batch(_request(circ, obs, trainable, x, wrt))
    assert close(res.expectations, e_ref) < TOL
    for k in wrt:
        assert close(res.gradients[k], j_ref[k]) < TOL
    up = rng.uniform(-1, 1, (len(x), len(obs)))
    e, rows, vsum = _vjp_device(torch_cuda, _engine(), circ, obs, wrt, trainable, x, up)
    ref_rows = np.concatenate([np.einsum("bm,bmp->bp", up, j_ref[k]) for k in wrt], axis=1)
    assert close(e, e_ref) < TOL
    assert close(rows, ref_rows) < TOL
    assert close(vsum, ref_rows.sum(axis=0)) < 1e-10 * max(1.0, np.abs(ref_rows).sum(axis=0).max())


@pytest.mark.parametrize("n", [4, 5, 6, 7])
@pytest.mark.parametrize("pad", ["8", "0"])
def test_small_circuits_padded_and_on_chip(torch_cuda, monkeypatch, n, pad):
    """4-7 qubit circuits are planned on 8 qubits by default (idle qubits stay
    in |0>, pass kernels); VQC_PAD_QUBITS=0 keeps them on the on-chip JIT
    kernels. Both against the oracle, general observables."""
    monkeypatch.setenv("VQC_PAD_QUBITS", pad)
    rng = np.random.default_rng(900 + n)
    circ, trainable = _rand_circuit(rng, n, 30 + 4 * n)
    obs = _pauli_obs(rng, n, 3)
    x = rng.uniform(-2, 2, (37, 4))
    wrt = ("a", "b", "s")
    e_ref, j_ref = oracle_batch(circ, obs, trainable, x, wrt)
    res = _engine().run_batch(_request(circ, obs, trainable, x, wrt))
    assert close(res.expectations, e_ref) < TOL
    for k in wrt:
        assert close(res.gradients[k], j_ref[k]) < TOL
    up = rng.uniform(-1, 1, (len(x), len(obs)))
    e, rows, vsum = _vjp_device(torch_cuda, _engine(), circ, obs, wrt, trainable, x, up)
    ref_rows = np.concatenate([np.einsum("bm,bmp->bp", up, j_ref[k]) for k in wrt], axis=1)
    assert close(e, e_ref) < TOL and close(rows, ref_rows) < TOL


@pytest.mark.parametrize("n", [9, 12])
def test_on_chip_jit_kernels_kept_by_knob(torch_cuda, monkeypatch, n):
    """VQC_SMEM_MAX_QUBITS=12 keeps 8-12 qubit plans on the on-chip JIT kernels
    (several samples per CTA / thread pairs), the default before the pass
    kernels took them over."""
    monkeypatch.setenv("VQC_SMEM_MAX_QUBITS", "12")
    rng = np.random.default_rng(800 + n)
    circ, trainable = _rand_circuit(rng, n, 30 + 4 * n)
    obs = _pauli_obs(rng, n, 2)
    x = rng.uniform(-2, 2, (4, 4))
    wrt = ("a", "b", "s")
    e_ref, j_ref = oracle_batch(circ, obs, trainable, x, wrt)
    res = _engine().run_batch(_request(circ, obs, trainable, x, wrt))
    assert close(res.expectations, e_ref) < TOL
    for k in wrt:
        assert close(res.gradients[k], j_ref[k]) < TOL


@pytest.mark.parametrize("n,jit", [(9, "0"), (12, "0"), (13, "0"), (14, "0"), (9, "1"), (13, "1")])
def test_kernel_paths_vs_oracle(torch_cuda, monkeypatch, n, jit):
    """The prebuilt interpreter (VQC_JIT=0: op-decoding kernels, 4-slot thread
    pairs) and the JIT with every variant forced (VQC_JIT=1), on the same
    random circuits as the default path."""
    monkeypatch.setenv("VQC_JIT", jit)
    rng = np.random.default_rng(300 + n)
    circ, trainable = _rand_circuit(rng, n, 30 + 4 * n)
    obs = _z_obs(rng, n, 2)
    x = rng.uniform(-2, 2, (4, 4))
    wrt = ("a", "b", "s")
    e_ref, j_ref = oracle_batch(circ, obs, trainable, x, wrt)
    res = _engine().run_batch(_request(circ, obs, trainable, x, wrt))
    assert close(res.expectations, e_ref) < TOL
    for k in wrt:
        assert close(res.gradients[k], j_ref[k]) < TOL


@pytest.mark.parametrize("knobs", [{"VQC_ADJ_DUAL": "0", "VQC_REG_SLOTS": "4"}, {"VQC_SMEM_DUAL": "1"},
                                   {"VQC_FWD_TILE": "12"}, {"VQC_GROUP_SYNC": "0"}, {"VQC_DIRECT_IO": "1"},
                                   {"VQC_DIRECT_IO": "1", "VQC_DIO_LINES": "2"}, {"VQC_FORCED_LOW": "2"},
                                   {"VQC_FOLD_THREAD_TARGETS": "0"}])
def test_schedule_variants_cfg4_rows(torch_cuda, monkeypatch, knobs):
    """Alternative schedules and kernel variants kept behind knobs
    (thread-pair 4-slot adjoint, dual on-chip adjoint, 12-qubit forward
    tiles, CTA barriers with per-segment CTA reductions, sweep ends
    exchanging registers with HBM directly, 64-byte HBM chunks, CNOT folds on
    register targets only) agree with the reference golden rows."""
    from paper_2404_06314_b200 import configs
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    cfg = 4 if "VQC_SMEM_DUAL" not in knobs else 3
    g = _golden(f"cfg{cfg}.npz")
    spec = configs.CONFIGS[cfg]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    res = _engine().run_batch(_request(circ, obs, {"w": g["w"]}, g["x_rows"], wrt))
    assert close(res.expectations, g["expect"]) < TOL
    assert close(res.gradients["w"], g["jac_w"]) < TOL


@pytest.mark.parametrize("cfg", [2, 3])
def test_whole_state_tile_cut_into_passes(torch_cuda, monkeypatch, cfg):
    """VQC_PASS_SEGMENTS cuts a whole-state tile's single pass into several
    (the compile-time bound for deep circuits, default 48 segments): cfg2
    (forward and adjoint sweeps in one program, 8 qubits) and cfg3 (separate
    forward program, 12 qubits) on 3-segment passes against the goldens."""
    from paper_2404_06314_b200 import configs
    monkeypatch.setenv("VQC_PASS_SEGMENTS", "3")
    g = _golden(f"cfg{cfg}.npz")
    spec = configs.CONFIGS[cfg]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    eng = _engine()
    res = eng.run_batch(_request(circ, obs, {"w": g["w"]}, g["x_rows"], wrt))
    plan, _ = eng.plans.get(circ, obs, tuple(wrt), eng.device)
    import json
    assert json.loads(plan.describe())["passes"] > 2
    assert close(res.expectations, g["expect"]) < TOL
    for k in wrt:
        assert close(res.gradients[k], g["jac_" + k]) < TOL


@pytest.mark.parametrize("n", [9, 13])
@pytest.mark.parametrize("terms", [7, 70])
def test_many_term_observables(torch_cuda, n, terms):
    """Z-string observables are compile-time constants of the observing pass
    up to 64 terms; beyond that (70 here) the kernels read them from shared
    memory. Both against the oracle, Jacobians and a row-dependent VJP."""
    from paper_2404_06314_b200.observables import Observable
    rng = np.random.default_rng(1000 + n + terms)
    circ, trainable = _rand_circuit(rng, n, 30 + 4 * n)
    def zterms(k):
        return tuple((float(rng.uniform(-2, 2)), "".join("Z" if rng.random() < 0.4 else "I" for _ in range(n)))
                     for _ in range(k))
    obs = [Observable(zterms(terms)), Observable(zterms(2))]
    x = rng.uniform(-2, 2, (5, 4))
    wrt = ("a", "b", "s")
    e_ref, j_ref = oracle_batch(circ, obs, trainable, x, wrt)
    res = _engine().run_batch(_request(circ, obs, trainable, x, wrt))
    assert close(res.expectations, e_ref) < TOL
    for k in wrt:
        assert close(res.gradients[k], j_ref[k]) < TOL
    up = rng.uniform(-1, 1, (len(x), len(obs)))
    e, rows, _ = _vjp_device(torch_cuda, _engine(), circ, obs, wrt, trainable, x, up)
    ref_rows = np.concatenate([np.einsum("bm,bmp->bp", up, j_ref[k]) for k in wrt], axis=1)
    assert close(e, e_ref) < TOL and close(rows, ref_rows) < TOL


def test_hbm_chunking_is_bitwise_invariant(torch_cuda, monkeypatch):
    """Row chunking (state budget) must not change any per-row result."""
    from paper_2404_06314_b200 import configs
    spec = configs.CONFIGS[4]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=6)
    a = _engine().run_batch(_request(circ, obs, {"w": w}, x, wrt))
    monkeypatch.setenv("VQC_STATE_BUDGET_MB", "4")   # forces 1-2 rows per chunk
    b = _engine().run_batch(_request(circ, obs, {"w": w}, x, wrt))
    np.testing.assert_array_equal(a.expectations, b.expectations)
    for k in a.gradients:
        np.testing.assert_array_equal(a.gradients[k], b.gradients[k])


def test_determinism(torch_cuda):
    from paper_2404_06314_b200 import configs
    spec = configs.CONFIGS[3]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=300)
    eng = _engine()
    a = eng.run_batch(_request(circ, obs, {"w": w}, x, wrt))
    b = eng.run_batch(_request(circ, obs, {"w": w}, x, wrt))
    np.testing.assert_array_equal(a.expectations, b.expectations)
    np.testing.assert_array_equal(a.gradients["w"], b.gradients["w"])


def test_degenerate_shapes(torch_cuda):
    """Empty batch and M = 0 keep their dims (batch.py:464-468)."""
    from paper_2404_06314_b200 import configs
    spec = configs.CONFIGS[1]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec)
    eng = _engine()
    r = eng.run_batch(_request(circ, obs, {"w": w}, x[:0], wrt))
    assert r.expectations.shape == (0, 1) and r.gradients["w"].shape == (0, 1, 16)
    r = eng.run_batch(_request(circ, [], {"w": w}, x[:3], wrt))
    assert r.expectations.shape == (3, 0) and r.gradients["x"].shape == (3, 0, 4)


def test_more_rows_than_one_grid_holds(torch_cuda):
    """Pass kernels index rows with the grid's y dimension: a call of more
    than 65535 rows runs in row chunks. Rows on both sides of the chunk
    boundary equal the same inputs evaluated in a small batch (batch
    invariance, reference tests/test_batch.py:107-132)."""
    from paper_2404_06314_b200 import configs
    spec = configs.CONFIGS[2]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=64)
    eng = _engine()
    small = eng.run_batch(_request(circ, obs, {"w": w}, x, ("x",)))
    B = 65535 + 700
    big = eng.run_batch(_request(circ, obs, {"w": w}, np.tile(x, (B // 64 + 1, 1))[:B], ("x",)))
    assert big.expectations.shape == (B, len(obs))
    for lo in (0, 65535 - 31, B - 64):
        idx = np.arange(lo, lo + 64) % 64
        assert np.array_equal(big.expectations[lo:lo + 64], small.expectations[idx])
        assert np.array_equal(big.gradients["x"][lo:lo + 64], small.gradients["x"][idx])


def test_more_rows_than_one_grid_holds_hbm_plan(torch_cuda):
    """The same on an HBM plan: a forward-only call of a 13-qubit circuit
    keeps one 128 KiB state per row, so the 16 GiB state budget alone would
    allow 131072 rows per launch; rows beyond the grid limit go to the next
    chunk."""
    rng = np.random.default_rng(77)
    circ, tr = _rand_circuit(rng, 13, 30)
    obs = _z_obs(rng, 13, 2)
    x = rng.uniform(-2, 2, (64, 4))
    eng = _engine()
    small = eng.run_batch(_request(circ, obs, tr, x, ()))
    B = 65535 + 200
    big = eng.run_batch(_request(circ, obs, tr, np.tile(x, (B // 64 + 1, 1))[:B], ()))
    assert big.expectations.shape == (B, 2)
    for lo in (0, 65535 - 31, B - 64):
        assert np.array_equal(big.expectations[lo:lo + 64], small.expectations[np.arange(lo, lo + 64) % 64])


def test_failing_input_reports_index(torch_cuda):
    """Per-row failure reporting (reference tests/test_batch.py:196-209): the
    reference wraps a failing row's exception in BatchInputError(index); on
    the GPU a row fails when its inputs or outputs are not finite."""
    from paper_2404_06314_b200 import BatchInputError, configs
    spec = configs.CONFIGS[2]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=6)
    x = x.copy()
    x[4, 1] = np.nan
    with pytest.raises(BatchInputError, match="input 4") as ei:
        _engine().run_batch(_request(circ, obs, {"w": w}, x, wrt))
    assert ei.value.index == 4
    x[4, 1] = 0.5
    wbad = w.copy()
    wbad[3] = np.inf          # every row's outputs are NaN: the first one is reported
    with pytest.raises(BatchInputError, match="input 0"):
        _engine().run_batch(_request(circ, obs, {"w": wbad}, x, wrt))
    res = _engine().run_batch(_request(circ, obs, {"w": w}, x, wrt))
    assert np.isfinite(res.expectations).all()


def test_xy_observables_on_chip(torch_cuda):
    """General Pauli strings (observables.py:70-92) on the on-chip path."""
    from paper_2404_06314_b200 import configs, parse_observable
    spec = configs.CONFIGS[2]
    circ, _, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=16)
    obs = [parse_observable("0.5*XZYIIIII + -1.2*IIIIYYXZ + 0.3*ZIIIIIII"),
           parse_observable("YIIIIIIY"), parse_observable("IIXIIIII + 2*IIIZIIII")]
    e_ref, j_ref = oracle_batch(circ, obs, {"w": w}, x, wrt)
    res = _engine().run_batch(_request(circ, obs, {"w": w}, x, wrt))
    assert close(res.expectations, e_ref) < TOL
    for k in wrt:
        assert close(res.gradients[k], j_ref[k]) < TOL


def test_xy_observables_on_hbm_path(torch_cuda):
    """cfg4 (16 qubits, HBM plans) with X / Y observables: run_batch splits
    the terms per X/Y pattern onto basis-rotated Z-basis plans."""
    from paper_2404_06314_b200 import configs, parse_observable
    spec = configs.CONFIGS[4]
    circ, _, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=2)
    obs = [parse_observable("X" + "I" * 15), parse_observable("I" * 3 + "Y" + "Z" + "I" * 11)]
    e_ref, j_ref = oracle_batch(circ, obs, {"w": w}, x, wrt)
    res = _engine().run_batch(_request(circ, obs, {"w": w}, x, wrt))
    assert close(res.expectations, e_ref) < TOL
    for k in wrt:
        assert close(res.gradients[k], j_ref[k]) < TOL


def test_no_gates_circuit(torch_cuda):
    from paper_2404_06314_b200.ir import Circuit, ParameterSet
    from paper_2404_06314_b200 import parse_observable
    for n in (3, 14):
        circ = Circuit(n, (), (ParameterSet("s", 1, "encoding"), ParameterSet("t", 1)))
        obs = [parse_observable("Z" + "I" * (n - 1))]
        res = _engine().run_batch(_request(circ, obs, {"t": np.zeros(1)}, np.zeros((2, 1)), ("t",)))
        np.testing.assert_array_equal(res.expectations, np.ones((2, 1)))
        np.testing.assert_array_equal(res.gradients["t"], np.zeros((2, 1, 1)))


def test_max_qubits_24(torch_cuda):
    """Largest register the reference allows (statevector.py:21)."""
    from paper_2404_06314_b200.ir import AngleExpression, Circuit, Gate, GateKind, ParameterSet
    from paper_2404_06314_b200.observables import z_observable
    n = 24
    gates = [Gate(GateKind.RY, (q,), AngleExpression(1.0, (("s", q % 2),))) for q in range(n)]
    gates += [Gate(GateKind.CNOT, (q, q + 1)) for q in range(n - 1)]
    gates += [Gate(GateKind.RX, (q,), AngleExpression(0.5, (("t", q % 3),))) for q in (0, 12, 23)]
    circ = Circuit(n, tuple(gates), (ParameterSet("s", 2, "encoding"), ParameterSet("t", 3)))
    obs = [z_observable(n, (0,)), z_observable(n, (23,)), z_observable(n, (5, 17))]
    x = np.array([[0.3, -1.1]])
    t = np.array([0.2, 0.9, -0.4])
    e_ref, j_ref = oracle_batch(circ, obs, {"t": t}, x, ("t", "s"))
    res = _engine().run_batch(_request(circ, obs, {"t": t}, x, ("t", "s")))
    assert close(res.expectations, e_ref) < TOL
    for k in ("t", "s"):
        assert close(res.gradients[k], j_ref[k]) < TOL


def test_host_abi_matches_device_abi(torch_cuda):
    """vqc_run_batch_host (numpy in/out) == the device-pointer path."""
    from paper_2404_06314_b200 import configs
    g = _golden("cfg2.npz")
    spec = configs.CONFIGS[2]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    eng = _engine()
    plan, layout = eng.plans.get(circ, obs, wrt, eng.device)
    flat = eng.base_flat(circ, {"w": g["w"]})
    x = g["x_rows"]
    e, jac, _, _ = plan.run_batch_host(x, flat, jacobian=True)
    assert close(e, g["expect"]) < TOL
    lo, hi = [(a, b) for n, a, b in layout.slices if n == "w"][0]
    assert close(jac[:, :, lo:hi], g["jac_w"]) < TOL
    up = np.ones((len(x), len(obs)))
    e2, _, rows, vsum = plan.run_batch_host(x, flat, upstream=up)
    assert close(vsum[lo:hi], g["vjp_w"]) < TOL
