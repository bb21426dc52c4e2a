"""Timing sweep (sweep.py): CSV layout on CPU, one timed point on the GPU."""

import pytest


def test_csv_round_trip(tmp_path):
    from paper_2404_06314_b200.sweep import CSV_COLUMNS, SweepPoint, read_csv, speedups, write_csv
    p = SweepPoint(4, 2, 8, (0.1, 0.05, 0.2), (0.3, 0.2, 0.4), (0.4, 0.25, 0.6))
    path = tmp_path / "sweep.csv"
    write_csv([p], path, seed=7, note="b200")
    text = path.read_text().splitlines()
    assert text[0] == "# seed=7" and text[1] == "# b200"
    rows = read_csv(path)
    assert tuple(rows[0]) == CSV_COLUMNS
    assert rows[0]["qubits"] == "4" and float(rows[0]["backward_min"]) == 0.2
    cpu = [dict(rows[0], total="4.0")]
    assert speedups(rows, cpu).tolist() == [10.0]


@pytest.mark.gpu
def test_gpu_sweep_point(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2404_06314_b200.sweep import read_csv, run_sweep, write_csv
    pts = run_sweep([4, 8], [2], [64], repeats=2, device="cuda:0")
    assert len(pts) == 2 and all(p.total[0] > 0 for p in pts)
    write_csv(pts, tmp_path / "s.csv", seed=0)
    assert [r["qubits"] for r in read_csv(tmp_path / "s.csv")] == ["4", "8"]
    with pytest.raises(ValueError, match="repeats"):
        run_sweep([4], [1], [4], repeats=0, device="cuda:0")
