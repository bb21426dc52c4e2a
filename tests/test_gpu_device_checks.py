"""Device bounds checks (VQC_CHECKS=1): the JIT units of the plan are built
with VQC_DEVICE_CHECKS, which range-checks every shared-memory tile address
of the register loads / stores and the observe step, every global state
index of the tile loads / stores, and every gradient-slot output; a failure
fails the call. compute-sanitizer is closed on this pool, so this is the
memcheck stand-in; run on all five configs (both precisions) and random
circuits on every kernel family, results must equal the unchecked run
bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(monkeypatch, checks, circ, obs, w, x, wrt, precision):
    from paper_2404_06314_b200.engine import BatchEngine, BatchRequest
    monkeypatch.setenv("VQC_CHECKS", "1" if checks else "0")
    eng = BatchEngine(device="cuda:0", precision=precision)   # fresh plan cache
    r = eng.run_batch(BatchRequest(circ, obs, w, x, wrt=wrt))
    plan, _ = eng.plans.get(circ, obs, wrt, eng.device)
    return r, plan


@pytest.mark.parametrize("precision", ["complex128", "complex64"])
@pytest.mark.parametrize("cfg_id", [1, 2, 3, 4, 5])
def test_configs_under_device_checks(monkeypatch, cfg_id, precision):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200 import configs
    spec = configs.CONFIGS[cfg_id]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=min(spec.batch, 3 if cfg_id == 5 else 16))
    ref, _ = _run(monkeypatch, False, circ, obs, {"w": w}, x, wrt, precision)
    chk, plan = _run(monkeypatch, True, circ, obs, {"w": w}, x, wrt, precision)
    assert '"jit": true' in plan.describe()
    assert np.array_equal(chk.expectations, ref.expectations)
    for k in wrt:
        assert np.array_equal(chk.gradients[k], ref.gradients[k])


@pytest.mark.parametrize("n", [2, 5, 9, 12, 13, 14])
def test_random_circuits_under_device_checks(monkeypatch, n):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from test_gpu_parity import _rand_circuit, _z_obs
    rng = np.random.default_rng(900 + n)
    circ, tr = _rand_circuit(rng, n, 30 + 4 * n)
    obs = _z_obs(rng, n, 2)
    x = rng.uniform(-2, 2, (3, 4))
    from conftest import close
    ref, _ = _run(monkeypatch, False, circ, obs, tr, x, ("a", "b", "s"), "complex128")
    chk, _ = _run(monkeypatch, True, circ, obs, tr, x, ("a", "b", "s"), "complex128")
    assert close(chk.expectations, ref.expectations) < 1e-12   # n < 4: interpreter vs JIT
    for k in ("a", "b", "s"):
        assert close(chk.gradients[k], ref.gradients[k]) < 1e-12
