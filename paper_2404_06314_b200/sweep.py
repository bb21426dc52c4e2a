"""Paper-style timing sweeps on the GPU module.

The paper's figures time a QNN layer's forward and backward over grids of
qubits, depth and batch size. The reference's runner does that with
wall-clock timers around its CPU batch calls and writes a CSV
(vqckit/bench.py:24-27 columns, 110-190). This module times the same
quantity the way a torch user sees it on the GPU:

* forward: ``QuantumModule(x)`` (one ``vqc_forward`` launch sequence);
* backward: ``out.backward(upstream)`` (the VJP adjoint kernels, per-row
  input gradients plus the batch-summed weight gradients).

Each repeat is timed with CUDA events on the current stream. Inputs stay
resident on the device. The CSV keeps the reference's column names, so the
reference's plotting reads these files; the ``threads`` column is 0 (no
host threads do the work).
"""

from __future__ import annotations

import csv
import itertools
import statistics
from dataclasses import dataclass

import numpy as np
import torch

from .ir import build_reuploading_ansatz
from .observables import z_observable

CSV_COLUMNS = ("qubits", "depth", "batch", "observables", "method", "threads",
               "forward", "forward_min", "forward_max",
               "backward", "backward_min", "backward_max",
               "total", "total_min", "total_max")


@dataclass(frozen=True)
class SweepPoint:
    qubits: int
    depth: int
    batch: int
    forward: tuple[float, float, float]    # mean, min, max seconds
    backward: tuple[float, float, float]
    total: tuple[float, float, float]

    def row(self) -> dict:
        out = {"qubits": self.qubits, "depth": self.depth, "batch": self.batch,
               "observables": self.qubits, "method": "adjoint", "threads": 0}
        for name in ("forward", "backward", "total"):
            mean, lo, hi = getattr(self, name)
            out.update({name: mean, f"{name}_min": lo, f"{name}_max": hi})
        return out


def _summary(xs) -> tuple[float, float, float]:
    return statistics.fmean(xs), min(xs), max(xs)


def time_point(qubits: int, depth: int, batch: int, repeats: int = 5, seed: int = 0,
               device="cuda") -> SweepPoint:
    """Forward / backward seconds of one re-uploading QNN layer (the reference
    ansatz, one <Z_q> output per qubit), weights and inputs seeded."""
    from .module import QuantumModule
    if repeats < 1:
        raise ValueError(f"repeats must be >= 1, got {repeats}")
    circuit = build_reuploading_ansatz(qubits, depth, qubits)
    obs = [z_observable(qubits, (q,)) for q in range(qubits)]
    mod = QuantumModule(circuit, obs, "s", ["theta", "lambda"], seed=seed, device=device)
    dev = mod.flat_weights().device
    gen = torch.Generator(device="cpu").manual_seed(seed)
    x = (2 * torch.rand((batch, qubits), generator=gen, dtype=torch.float64) - 1).to(dev)
    x.requires_grad_(True)
    up = torch.ones((batch, qubits), dtype=torch.float64, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    fwd, bwd = [], []
    for rep in range(repeats + 1):           # repeat 0 builds plans / JIT: untimed
        a, b, c = ev(), ev(), ev()
        a.record()
        out = mod(x)
        b.record()
        out.backward(up)
        c.record()
        torch.cuda.synchronize(dev)
        if rep:
            fwd.append(a.elapsed_time(b) * 1e-3)
            bwd.append(b.elapsed_time(c) * 1e-3)
        mod.zero_grad(set_to_none=True)
        x.grad = None
    return SweepPoint(qubits, depth, batch, _summary(fwd), _summary(bwd),
                      _summary([f + g for f, g in zip(fwd, bwd)]))


def run_sweep(qubits, depths, batches, repeats: int = 5, seed: int = 0, device="cuda",
              echo=None) -> list[SweepPoint]:
    points = []
    for q, d, b in itertools.product(qubits, depths, batches):
        p = time_point(q, d, b, repeats, seed, device)
        points.append(p)
        if echo is not None:
            echo(f"q={q} d={d} B={b}: forward {p.forward[0] * 1e3:.3f} ms, "
                 f"backward {p.backward[0] * 1e3:.3f} ms")
    return points


def write_csv(points, path, seed: int, note: str | None = None) -> None:
    """Comment lines (seed, optional note) then one row per point."""
    with open(path, "w", newline="") as fh:
        fh.write(f"# seed={seed}\n")
        if note:
            fh.write(f"# {note}\n")
        w = csv.DictWriter(fh, fieldnames=CSV_COLUMNS)
        w.writeheader()
        for p in points:
            w.writerow({k: (repr(v) if isinstance(v, float) else v) for k, v in p.row().items()})


def read_csv(path) -> list[dict]:
    with open(path) as fh:
        return list(csv.DictReader(line for line in fh if not line.startswith("#")))


def speedups(gpu_rows, cpu_rows) -> np.ndarray:
    """total(cpu) / total(gpu) for rows matched on (qubits, depth, batch)."""
    key = lambda r: (int(r["qubits"]), int(r["depth"]), int(r["batch"]))  # noqa: E731
    cpu = {key(r): float(r["total"]) for r in cpu_rows}
    return np.array([cpu[key(r)] / float(r["total"]) for r in gpu_rows if key(r) in cpu])
