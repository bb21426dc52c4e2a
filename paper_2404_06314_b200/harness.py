"""Paper-style timing sweeps on the GPU engine.

Same configuration knobs, input recipe and CSV layout as the reference's
benchmark runner (vqckit/bench.py:24-60 config + columns, 63-81 inputs,
110-160 timing, 163-178 CSV), so sweeps over qubits / depth / batch
(the paper's Fig. 1/2 and Table I shapes) produce files the reference's
tooling reads. Each timed call is a full ``BatchEngine.run_batch`` with host
arrays in and out (the reference's timed region); the GPU work is synchronous
inside it because results come back as numpy arrays.
"""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass, field

import numpy as np

from .engine import BatchEngine, BatchRequest
from .ir import build_reuploading_ansatz, load_circuit
from .observables import Observable, parse_observable

CSV_COLUMNS = ["qubits", "depth", "batch", "observables", "method", "threads",
               "forward", "forward_min", "forward_max",
               "backward", "backward_min", "backward_max",
               "total", "total_min", "total_max"]


@dataclass
class BenchConfig:
    qubits: int = 12
    depth: int = 3
    batch: int = 48
    observables: int | None = None      # default: one Z per qubit
    method: str = "adjoint"
    repeats: int = 10
    seed: int = 0
    circuit_file: str | None = None
    observable_texts: tuple = ()
    spsa_samples: int = 2000
    spsa_c: float = 0.01

    def __post_init__(self):
        if self.repeats < 1:
            raise ValueError(f"repeats must be >= 1, got {self.repeats}")

    @property
    def num_observables(self) -> int:
        if self.observable_texts:
            return len(self.observable_texts)
        return self.observables if self.observables is not None else self.qubits


def default_observables(num_qubits: int, count: int) -> list:
    """Z on qubit i mod n for i < count."""
    return [Observable(((1.0, "".join("Z" if q == i % num_qubits else "I"
                                      for q in range(num_qubits))),))
            for i in range(count)]


def materialize(config: BenchConfig):
    """(circuit, observables, trainable values, inputs): one default_rng(seed)
    draws every trainable set U(0, 2pi) in declaration order, then the inputs
    U(-1, 1) (bench.py:63-81)."""
    circuit = (load_circuit(config.circuit_file) if config.circuit_file
               else build_reuploading_ansatz(config.qubits, config.depth, config.qubits))
    if config.observable_texts:
        observables = [parse_observable(t) for t in config.observable_texts]
    else:
        m = config.observables if config.observables is not None else circuit.num_qubits
        observables = default_observables(circuit.num_qubits, m)
    rng = np.random.default_rng(config.seed)
    trainable = {s.name: rng.uniform(0.0, 2.0 * np.pi, s.size)
                 for s in circuit.sets_with_role("trainable")}
    enc = circuit.sets_with_role("encoding")
    if len(enc) != 1:
        raise ValueError("benchmark circuit needs exactly one encoding set")
    inputs = rng.uniform(-1.0, 1.0, (config.batch, enc[0].size))
    return circuit, observables, trainable, inputs


def _stats(times) -> tuple:
    return float(np.mean(times)), float(np.min(times)), float(np.max(times))


@dataclass
class BenchRecord:
    config: BenchConfig
    forward: tuple        # (mean, min, max) seconds
    backward: tuple
    total: tuple
    extras: dict = field(default_factory=dict)

    def csv_row(self) -> list:
        c = self.config
        # "threads" column: the GPU engine has none; 1 keeps the file readable
        return [c.qubits, c.depth, c.batch, c.num_observables, c.method, 1,
                *(repr(v) for v in self.forward), *(repr(v) for v in self.backward),
                *(repr(v) for v in self.total)]


def run_bench(config: BenchConfig, engine: BatchEngine | None = None, echo=print) -> BenchRecord:
    engine = engine or BatchEngine()
    circuit, observables, trainable, inputs = materialize(config)
    wrt = tuple(s.name for s in circuit.sets_with_role("trainable"))

    def req(sets):
        return BatchRequest(circuit, observables, trainable, inputs, method=config.method,
                            wrt=sets, seed=config.seed,
                            spsa_samples=max(1, config.spsa_samples // 10),
                            spsa_c=config.spsa_c)

    fwd_req, bwd_req = req(()), req(wrt)
    engine.run_batch(fwd_req)             # plan build + JIT outside the timers
    engine.run_batch(bwd_req)
    fwd, bwd = [], []
    for _ in range(config.repeats):
        t0 = time.perf_counter()
        engine.run_batch(fwd_req)
        t1 = time.perf_counter()
        engine.run_batch(bwd_req)
        t2 = time.perf_counter()
        fwd.append(t1 - t0)
        bwd.append(t2 - t1)
    rec = BenchRecord(config, _stats(fwd), _stats(bwd),
                      _stats([a + b for a, b in zip(fwd, bwd)]))
    if echo is not None:
        echo(f"q={config.qubits} d={config.depth} B={config.batch}: forward "
             f"{rec.forward[0]:.6f}s backward {rec.backward[0]:.6f}s")
    return rec


def run_sweep(qubits, depths, batch: int, engine: BatchEngine | None = None, **kw) -> list:
    engine = engine or BatchEngine()
    return [run_bench(BenchConfig(qubits=q, depth=d, batch=batch, **kw), engine)
            for q in qubits for d in depths]


def write_csv(records, path, seed: int) -> None:
    """Comment header with the seed (and extras), then CSV_COLUMNS rows."""
    with open(path, "w", newline="") as fh:
        fh.write(f"# seed={seed}\n")
        for rec in records:
            for key, value in rec.extras.items():
                fh.write(f"# {key}={value!r}\n")
        writer = csv.writer(fh)
        writer.writerow(CSV_COLUMNS)
        for rec in records:
            writer.writerow(rec.csv_row())


def read_csv(path) -> list:
    with open(path) as fh:
        return list(csv.DictReader(line for line in fh if not line.startswith("#")))
