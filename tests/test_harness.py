"""Sweep harness (bench.py:24-178 layout) on the GPU engine: host logic on
CPU, one timed sweep point on the GPU."""

import numpy as np
import pytest


def test_materialize_recipe():
    """One default_rng(seed): trainable sets U(0, 2pi) in declaration order,
    then inputs U(-1, 1) (bench.py:63-81)."""
    from paper_2404_06314_b200.harness import BenchConfig, materialize
    circ, obs, train, x = materialize(BenchConfig(qubits=3, depth=2, batch=5, seed=4))
    rng = np.random.default_rng(4)
    theta = rng.uniform(0.0, 2.0 * np.pi, 12)
    lam = rng.uniform(0.0, 2.0 * np.pi, 6)
    assert list(train) == ["theta", "lambda"]
    assert np.array_equal(train["theta"], theta) and np.array_equal(train["lambda"], lam)
    assert np.array_equal(x, rng.uniform(-1.0, 1.0, (5, 3)))
    assert [o.terms[0][1] for o in obs] == ["ZII", "IZI", "IIZ"]


def test_default_observables_cycle():
    from paper_2404_06314_b200.harness import default_observables
    assert [o.terms[0][1] for o in default_observables(2, 3)] == ["ZI", "IZ", "ZI"]


def test_csv_round_trip(tmp_path):
    from paper_2404_06314_b200.harness import (CSV_COLUMNS, BenchConfig, BenchRecord,
                                               read_csv, write_csv)
    rec = BenchRecord(BenchConfig(qubits=4, depth=2, batch=8), (0.1, 0.05, 0.2),
                      (0.3, 0.2, 0.4), (0.4, 0.25, 0.6), {"note": 1.5})
    path = tmp_path / "sweep.csv"
    write_csv([rec], path, seed=7)
    text = path.read_text().splitlines()
    assert text[0] == "# seed=7" and text[1] == "# note=1.5"
    rows = read_csv(path)
    assert list(rows[0]) == CSV_COLUMNS
    assert rows[0]["qubits"] == "4" and float(rows[0]["backward_min"]) == 0.2
    with pytest.raises(ValueError, match="repeats"):
        BenchConfig(repeats=0)


@pytest.mark.gpu
def test_gpu_sweep_point(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200.harness import read_csv, run_sweep, write_csv
    recs = run_sweep([4, 8], [2], batch=64, repeats=2)
    assert len(recs) == 2 and all(r.total[0] > 0 for r in recs)
    write_csv(recs, tmp_path / "s.csv", seed=0)
    assert [r["qubits"] for r in read_csv(tmp_path / "s.csv")] == ["4", "8"]
