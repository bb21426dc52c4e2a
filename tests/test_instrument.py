"""Sweep counters (instrument.py) and expression_partial (circuit.py:150-165)."""

import numpy as np
import pytest


def test_counters_unit():
    from paper_2404_06314_b200.instrument import SweepCounters
    c = SweepCounters()
    c.add_forward(3)
    c.add_reverse(ket=2, bra=5)
    assert c.snapshot() == (3, 2, 5)
    c.reset()
    assert c.snapshot() == (0, 0, 0)


def test_expression_partial():
    from paper_2404_06314_b200.ir import AngleExpression, expression_partial
    e = AngleExpression(1.5, (("lam", 0), ("s", 2)))
    b = {"lam": np.array([2.0]), "s": np.array([0.0, 0.0, -3.0])}
    assert expression_partial(e, ("lam", 0), b) == 1.5 * -3.0
    assert expression_partial(e, ("s", 2), b) == 1.5 * 2.0
    assert expression_partial(e, ("s", 1), b) == 0.0
    with pytest.raises(ValueError, match="unresolved"):
        expression_partial(e, ("s", 2), {"s": b["s"]})


@pytest.mark.gpu
def test_gpu_sweep_structure():
    """Adjoint Jacobian: B forward + B ket + B*M bra sweeps; param-shift:
    B * (1 + 2S) forward sweeps and no reverse sweeps."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200 import configs
    from paper_2404_06314_b200.engine import BatchEngine, BatchRequest
    from paper_2404_06314_b200.instrument import sweep_counters
    spec = configs.CONFIGS[2]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=4)
    eng = BatchEngine(device="cuda:0")
    sweep_counters.reset()
    eng.run_batch(BatchRequest(circ, obs, {"w": w}, x, wrt=wrt))
    assert sweep_counters.snapshot() == (4, 4, 4 * len(obs))
    sweep_counters.reset()
    eng.run_batch(BatchRequest(circ, obs, {"w": w}, x, method="param-shift", wrt=wrt))
    n_rot = sum(g.expr is not None for g in circ.gates)
    assert sweep_counters.snapshot() == (4 * (1 + 2 * n_rot), 0, 0)
