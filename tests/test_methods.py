"""param-shift and SPSA (gradients.py:137-201, batch.py:193-201).

CPU: the oracle's restatement is pinned against reference goldens
(tests/golden/methods.npz, made by make_golden.py from vqckit's run_batch) and
against the oracle's own adjoint Jacobian (the reference's three-way agreement,
test_gradients.py:223-257); the host helpers of the GPU path (angle circuit,
per-row angles) are checked without a GPU.
GPU: BatchEngine.run_batch(method="param-shift" | "spsa") runs the shifted
evaluations as batched forward launches and must match the goldens.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, close, lowered, oracle_batch

TOL = 1e-10


def _golden():
    return np.load(os.path.join(GOLDEN, "methods.npz"))


def _setup(cfg_id):
    from paper_2404_06314_b200 import configs
    spec = configs.CONFIGS[cfg_id]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec)
    return circ, obs, wrt, x, w


def _flats(circ, w, xs):
    comp = circ.compiled()
    off, size = comp.offsets["x"]
    flat = comp.flat_values({"w": w, "x": np.zeros(size)})
    flats = np.repeat(flat[None], len(xs), 0)
    flats[:, off:off + size] = xs
    return flats


def _stack(g, cfg_id, name, wrt):
    return np.concatenate([g[f"cfg{cfg_id}_{name}_jac_{k}"] for k in wrt], axis=-1)


@pytest.mark.parametrize("cfg_id,rows", [(1, 4), (2, 2)])
def test_oracle_param_shift_matches_reference(oracle_mod, cfg_id, rows):
    from paper_2404_06314_b200.engine import WrtLayout
    g = _golden()
    circ, obs, wrt, x, w = _setup(cfg_id)
    low = lowered(circ, obs)
    layout = WrtLayout.build(circ.compiled(), wrt)
    ref = _stack(g, cfg_id, "ps", wrt)
    for b, flat in enumerate(_flats(circ, w, x[:rows])):
        e, j = oracle_mod.param_shift_row(low, flat, layout.wrt_col)
        assert close(e, g[f"cfg{cfg_id}_ps_expect"][b]) < TOL
        assert close(j, ref[b]) < TOL


@pytest.mark.parametrize("cfg_id,rows", [(1, 4), (2, 2)])
def test_oracle_spsa_matches_reference(oracle_mod, cfg_id, rows):
    from paper_2404_06314_b200.engine import WrtLayout, mix_seed
    g = _golden()
    circ, obs, wrt, x, w = _setup(cfg_id)
    low = lowered(circ, obs)
    layout = WrtLayout.build(circ.compiled(), wrt)
    ref = _stack(g, cfg_id, "spsa", wrt)
    seed, c, k = int(g["spsa_seed"]), float(g["spsa_c"]), int(g["spsa_samples"])
    for b, flat in enumerate(_flats(circ, w, x[:rows])):
        rng = np.random.default_rng(mix_seed(seed, b))
        e, j = oracle_mod.spsa_row(low, flat, layout.flat_of_col, c, k, rng)
        assert close(e, g[f"cfg{cfg_id}_spsa_expect"][b]) < TOL
        assert close(j, ref[b]) < TOL


def test_param_shift_agrees_with_adjoint(oracle_mod):
    """Shift rule is exact for exp(-i theta P / 2) gates: param-shift == adjoint
    Jacobian (test_gradients.py:223-257 uses 1e-9)."""
    g = _golden()
    circ, obs, wrt, x, w = _setup(2)
    _, jac = oracle_batch(circ, obs, {"w": w}, x[:8], wrt)
    adj = np.concatenate([jac[k] for k in wrt], axis=-1)
    assert np.abs(_stack(g, 2, "ps", wrt) - adj).max() < 1e-9


def test_spsa_is_a_directional_derivative():
    """Each SPSA sample is (f+ - f-) / (2c delta) = (J . delta) / delta up to
    O(c^2): rebuild the estimate from the adjoint Jacobian and the row's
    deltas (rng = default_rng(mix_seed(seed, b)), batch.py:197)."""
    from paper_2404_06314_b200.engine import WrtLayout, mix_seed
    g = _golden()
    circ, obs, wrt, x, w = _setup(1)
    _, jac = oracle_batch(circ, obs, {"w": w}, x[:4], wrt)
    adj = np.concatenate([jac[k] for k in wrt], axis=-1)
    layout = WrtLayout.build(circ.compiled(), wrt)
    seed, k = int(g["spsa_seed"]), int(g["spsa_samples"])
    spsa = _stack(g, 1, "spsa", wrt)
    for b in range(4):
        rng = np.random.default_rng(mix_seed(seed, b))
        est = np.zeros_like(adj[b])
        for _ in range(k):
            d = 2.0 * rng.integers(0, 2, size=layout.n_cols).astype(np.float64) - 1.0
            est += np.outer(adj[b] @ d, 1.0 / d)
        # third-order term: c^2/6 * D^3 f[delta, delta, delta] over 20 columns
        assert np.abs(spsa[b] - est / k).max() < 2e-3


def test_native_spsa_signs_match_numpy():
    """vqc_spsa_signs (host C++: SeedSequence + PCG64 + bounded draws) is bit
    for bit numpy's default_rng(mix_seed(seed, row)).integers(0, 2, size=C)
    per sample (batch.py:197, gradients.py:180-201), for one- and two-word
    entropies, odd draw counts (the 32-bit half-word buffer carries over
    between samples) and negative / oversized seeds (mix_seed wraps mod 2^64)."""
    from paper_2404_06314_b200 import native
    from paper_2404_06314_b200.engine import mix_seed
    for seed in (0, 1, 20240406, 2**32 - 1, 2**32, 2**40 + 3, 2**64 - 1, -5, 2**70 + 9):
        for row0 in (0, 7, 100000):
            for K, C in ((1, 1), (1, 7), (3, 5), (2, 64)):
                got = native.spsa_signs(seed, row0, 5, K, C)
                assert got.shape == (5, K, C) and got.dtype == np.int8
                for r in range(5):
                    rng = np.random.default_rng(mix_seed(seed, row0 + r))
                    for k in range(K):
                        want = 2.0 * rng.integers(0, 2, size=C).astype(np.float64) - 1.0
                        assert np.array_equal(got[r, k].astype(np.float64), want), (seed, row0, r, k)
    # single-binding form: every row from default_rng(seed) itself
    for seed in (0, 3, 2**33 + 1):
        got = native.spsa_signs(seed, 0, 2, 3, 9, per_row_seed=False)
        rng = np.random.default_rng(seed)
        want = np.stack([2.0 * rng.integers(0, 2, size=9).astype(np.float64) - 1.0 for _ in range(3)])
        assert np.array_equal(got[0].astype(np.float64), want)
        assert np.array_equal(got[1], got[0])
    assert native.spsa_signs(1, 0, 0, 1, 4).shape == (0, 1, 4)


def test_angle_circuit_host_helpers(oracle_mod):
    """angle_circuit keeps gates and makes rotation r read angles[r]; row_angles
    equals the reference's compute_angles (oracle restatement)."""
    from paper_2404_06314_b200.engine import angle_circuit, row_angles
    circ, obs, wrt, x, w = _setup(2)
    ac, rot = angle_circuit(circ)
    assert angle_circuit(circ)[0] is ac
    comp, acomp = circ.compiled(), ac.compiled()
    assert np.array_equal(comp.kinds, acomp.kinds) and np.array_equal(comp.q0, acomp.q0)
    assert acomp.offsets == {"angles": (0, len(rot))}
    flats = _flats(circ, w, x[:3])
    ang = row_angles(comp, flats, rot)
    low = lowered(circ, obs)
    for b in range(3):
        ref = oracle_mod._angles(low, flats[b])
        assert np.array_equal(ang[b], ref[rot])
    # evolving the angle circuit on those angles == evolving the source circuit
    st_src = oracle_mod.evolve(low, flats[0])
    st_ang = oracle_mod.evolve(lowered(ac, obs), ang[0])
    assert np.abs(st_src - st_ang).max() < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["param-shift", "spsa"])
@pytest.mark.parametrize("cfg_id", [1, 2])
def test_gpu_methods_match_reference(cfg_id, method):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200.engine import BatchEngine, BatchRequest
    g = _golden()
    circ, obs, wrt, x, w = _setup(cfg_id)
    rows = int(g[f"cfg{cfg_id}_rows"])
    name = "ps" if method == "param-shift" else "spsa"
    kw = {}
    if method == "spsa":
        kw = dict(seed=int(g["spsa_seed"]), spsa_c=float(g["spsa_c"]),
                  spsa_samples=int(g["spsa_samples"]))
    res = BatchEngine(device="cuda:0").run_batch(
        BatchRequest(circ, obs, {"w": w}, x[:rows], method=method, wrt=wrt, **kw))
    assert close(res.expectations, g[f"cfg{cfg_id}_{name}_expect"]) < TOL
    for k in wrt:
        assert close(res.gradients[k], g[f"cfg{cfg_id}_{name}_jac_{k}"]) < TOL


@pytest.mark.gpu
def test_gpu_param_shift_chunked_equals_adjoint():
    """Chunked shift evaluations (several forward launches) on an HBM-mode
    circuit agree with the adjoint path."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200 import engine as eng
    circ, obs, wrt, x, w = _setup(4)
    e = eng.BatchEngine(device="cuda:0")
    adj = e.run_batch(eng.BatchRequest(circ, obs, {"w": w}, x[:3], wrt=wrt))
    old = eng.SHIFT_CHUNK_ROWS
    eng.SHIFT_CHUNK_ROWS = 1000          # 1 row per chunk (961 evaluations per row)
    try:
        ps = e.run_batch(eng.BatchRequest(circ, obs, {"w": w}, x[:3], method="param-shift",
                                          wrt=wrt))
    finally:
        eng.SHIFT_CHUNK_ROWS = old
    assert close(ps.expectations, adj.expectations) < TOL
    for k in wrt:
        assert np.abs(ps.gradients[k] - adj.gradients[k]).max() < 1e-9


@pytest.mark.gpu
def test_gpu_module_backward_param_shift_equals_adjoint():
    """QuantumModule.backward(method="param-shift") takes the reference's
    Jacobian + einsum route (model.py:140-142) and equals the adjoint VJP."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200.module import QuantumModule
    circ, obs, wrt, x, w = _setup(2)
    mod = QuantumModule(circ, obs, "x", ["w"], seed=3, device="cuda:0")
    up = np.random.default_rng(0).normal(size=(6, len(obs)))
    adj = mod.backward(x[:6], up)
    ps = mod.backward(x[:6], up, method="param-shift")
    assert np.abs(adj["w"] - ps["w"]).max() < 1e-9


def test_device_row_angles_equal_host_on_cpu_tensors():
    """device_row_angles (torch gather path used by SPSA) == row_angles bit for
    bit; run on CPU tensors here, the GPU tests cover the CUDA placement."""
    import torch
    from paper_2404_06314_b200.engine import angle_circuit, device_row_angles, row_angles
    from paper_2404_06314_b200.ir import build_reuploading_ansatz
    circ = build_reuploading_ansatz(3, 2, num_features=3)   # lambda * s products
    comp = circ.compiled()
    _, rot = angle_circuit(circ)
    flats = np.random.default_rng(0).normal(size=(5, comp.total_params))
    host = row_angles(comp, flats, rot)
    dev = device_row_angles(comp, torch.from_numpy(flats), rot).numpy()
    assert np.array_equal(host, dev)
