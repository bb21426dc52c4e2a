"""Checkpoints (model.py:227-269) and dataset helpers (datasets.py:47-125):
host logic, CPU only."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN


def test_synthetic_blobs_match_reference():
    from paper_2404_06314_b200.training import synthetic_blobs
    g = np.load(os.path.join(GOLDEN, "blobs.npz"))
    ds = synthetic_blobs(samples_per_class=10, num_features=3, num_classes=3, seed=4)
    for k in ("features", "labels", "train_idx", "test_idx"):
        assert np.array_equal(getattr(ds, k), g[k]), k
    assert ds.num_classes == 3 and ds.num_features == 3


def test_from_arrays_validation():
    from paper_2404_06314_b200.training import from_arrays
    with pytest.raises(ValueError, match="integers"):
        from_arrays(np.zeros((2, 1)), [0.5, 1])
    with pytest.raises(ValueError, match="non-negative"):
        from_arrays(np.zeros((2, 1)), [0, -1])


def _module():
    from paper_2404_06314_b200 import build_reuploading_ansatz, z_observable
    from paper_2404_06314_b200.module import QuantumModule
    c = build_reuploading_ansatz(2, 1, 2)
    return QuantumModule(c, [z_observable(2, [0]), z_observable(2, [1])], "s",
                         ["theta", "lambda"], seed=0, device="cpu")


def test_checkpoint_round_trip(tmp_path):
    import torch
    from paper_2404_06314_b200.module import HybridModule, load_checkpoint, save_checkpoint
    mod = _module()
    path = tmp_path / "q.json"
    save_checkpoint(mod, path)
    before = mod.parameter_values()
    with torch.no_grad():
        mod.values["theta"].add_(1.0)
    load_checkpoint(mod, path)
    after = mod.parameter_values()
    assert all(np.array_equal(before[k], after[k]) for k in before)
    doc = json.loads(path.read_text())
    assert list(doc) == ["sets"] and list(doc["sets"]) == ["theta", "lambda"]

    hyb = HybridModule(3, _module(), 2, seed=1)
    hpath = tmp_path / "h.json"
    save_checkpoint(hyb, hpath)
    w0 = hyb.pre_weight.detach().clone()
    with torch.no_grad():
        hyb.pre_weight.zero_()
    load_checkpoint(hyb, hpath)
    assert torch.equal(hyb.pre_weight.detach(), w0)
    assert set(json.loads(hpath.read_text())) == {"sets", "pre", "post"}


def test_checkpoint_errors(tmp_path):
    from paper_2404_06314_b200.module import load_checkpoint
    mod = _module()
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"sets": {"nope": [1.0]}}))
    with pytest.raises(ValueError, match="not in module"):
        load_checkpoint(mod, bad)
    bad.write_text(json.dumps({"sets": {"theta": [1.0]}}))
    with pytest.raises(ValueError, match="has shape"):
        load_checkpoint(mod, bad)


def test_load_dataset_matches_reference():
    """tests/golden/toy_table.csv (comment, header, blank line) loaded by the
    reference -> toy_table.npz."""
    from paper_2404_06314_b200.training import load_dataset
    g = np.load(os.path.join(GOLDEN, "toy_table.npz"))
    ds = load_dataset(os.path.join(GOLDEN, "toy_table.csv"), seed=2, test_fraction=0.4)
    for k in ("features", "labels", "train_idx", "test_idx"):
        assert np.array_equal(getattr(ds, k), g[k]), k


@pytest.mark.parametrize("text,match", [
    ("1,2\n3,x\n", "malformed row"),
    ("1\n", "at least one feature"),
    ("1,2,0\n1,1\n", "expected 3 columns"),
    ("1,0.5\n", "unknown label"),
    ("# only comments\n\n", "no data rows"),
])
def test_load_dataset_errors(tmp_path, text, match):
    from paper_2404_06314_b200.training import load_dataset
    p = tmp_path / "t.csv"
    p.write_text(text)
    with pytest.raises(ValueError, match=match):
        load_dataset(p)
