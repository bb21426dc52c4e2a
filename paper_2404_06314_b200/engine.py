"""GPU batch engine: drop-in for the reference's ``BatchEngine.run_batch``.

Reference: vqckit/batch.py:54-217 (split, request/result types, validation,
degenerate shapes) and gradients.py:46-81 (WrtLayout). Where the reference
fans rows out over a thread pool and runs one numba sweep per gate per row,
this engine hands the whole batch to libvqc.so in one call per direction.
Row partitioning across GPUs reuses ``split_workload`` (parallel.py).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from . import native
from .ir import Circuit
from .observables import Observable, ObservablePack

METHODS = ("adjoint", "param-shift", "spsa")
GPU_METHODS = ("adjoint",)
_MASK64 = (1 << 64) - 1


def split_workload(batch_size: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous ranges covering [0, batch_size); the first
    ``batch_size - parts*floor(batch_size/parts)`` take one extra row
    (batch.py:54-72). Used for GPU (rank) sharding."""
    if batch_size < 0:
        raise ValueError(f"batch_size must be >= 0, got {batch_size}")
    if parts < 1:
        raise ValueError(f"threads must be >= 1, got {parts}")
    base, extra = divmod(batch_size, parts)
    out, start = [], 0
    for t in range(parts):
        stop = start + base + (1 if t < extra else 0)
        out.append((start, stop))
        start = stop
    return out


def mix_seed(seed: int, index: int) -> int:
    """splitmix64 step (batch.py:75-81): per-row seeds independent of sharding."""
    z = (int(seed) + (index + 1) * 0x9E3779B97F4A7C15) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


@dataclass(frozen=True, eq=False)
class WrtLayout:
    """Output-column layout of the requested sets (gradients.py:46-81)."""

    wrt_col: np.ndarray                        # flat index -> column or -1
    slices: tuple[tuple[str, int, int], ...]   # (set, lo, hi) columns
    flat_of_col: np.ndarray

    @property
    def n_cols(self) -> int:
        return len(self.flat_of_col)

    @staticmethod
    def build(compiled, wrt) -> "WrtLayout":
        wrt = list(wrt)
        if len(set(wrt)) != len(wrt):
            raise ValueError(f"duplicate set names in wrt: {wrt}")
        wrt_col = np.full(compiled.total_params, -1, np.int64)
        slices, flat_of_col = [], []
        for name in wrt:
            if name not in compiled.offsets:
                raise ValueError(f"unknown parameter set {name!r} in wrt")
            off, size = compiled.offsets[name]
            lo = len(flat_of_col)
            wrt_col[off:off + size] = np.arange(lo, lo + size)
            flat_of_col.extend(range(off, off + size))
            slices.append((name, lo, lo + size))
        return WrtLayout(wrt_col, tuple(slices), np.asarray(flat_of_col, np.int64))


@dataclass
class BatchRequest:
    circuit: Circuit
    observables: list
    trainable_values: dict
    inputs: np.ndarray                  # (B, encoding size)
    method: str = "adjoint"
    wrt: tuple = ()
    threads: int | None = None          # accepted for API parity; unused on the GPU
    seed: int = 0
    spsa_c: float = 0.01
    spsa_samples: int = 1


@dataclass
class BatchResult:
    expectations: np.ndarray            # (B, M)
    gradients: dict = field(default_factory=dict)   # set -> (B, M, size)


class BatchInputError(RuntimeError):
    """A row failed; carries its index (batch.py:104-109)."""

    def __init__(self, index: int, cause: Exception):
        super().__init__(f"batch input {index} failed: {cause}")
        self.index = index


def encoding_set(circuit: Circuit):
    enc = circuit.sets_with_role("encoding")
    if len(enc) != 1:
        raise ValueError(f"batched evaluation needs exactly one encoding set, "
                         f"circuit has {len(enc)}")
    return enc[0]


def _device(device):
    import torch
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the vqc GPU path has no CPU fallback")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


class PlanCache:
    """(circuit, observables, wrt, device) -> native.Plan."""

    def __init__(self):
        self._plans: dict = {}
        self._lock = threading.Lock()

    def get(self, circuit: Circuit, observables, wrt: tuple, device):
        key = (circuit, tuple(observables), tuple(wrt), str(device))
        with self._lock:
            plan = self._plans.get(key)
            if plan is None:
                compiled = circuit.compiled()
                pack = ObservablePack.from_observables(observables, circuit.num_qubits)
                layout = WrtLayout.build(compiled, wrt)
                enc = encoding_set(circuit)
                off, size = compiled.offsets[enc.name]
                plan = (native.Plan(compiled, pack, layout.wrt_col, off, size, device), layout)
                self._plans[key] = plan
            return plan


class Workspace:
    """Grow-only device scratch buffer (torch caching allocator underneath)."""

    def __init__(self):
        self._buf = None

    def get(self, nbytes: int, device):
        import torch
        if nbytes <= 0:
            return None
        if self._buf is None or self._buf.numel() < nbytes or self._buf.device != device:
            self._buf = torch.empty(int(nbytes), dtype=torch.uint8, device=device)
        return self._buf


class BatchEngine:
    """GPU replacement for vqckit's BatchEngine (batch.py:120-217)."""

    def __init__(self, threads: int | None = None, device=None):
        if threads is not None and threads < 1:
            raise ValueError(f"threads must be >= 1, got {threads}")
        self.threads = threads
        self._device_arg = device
        self.plans = PlanCache()
        self.workspace = Workspace()

    @property
    def device(self):
        return _device(self._device_arg)

    def close(self) -> None:
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def base_flat(self, circuit: Circuit, trainable_values: dict) -> np.ndarray:
        trainable = {s.name for s in circuit.sets_with_role("trainable")}
        given = set(trainable_values)
        if given != trainable:
            raise ValueError(f"trainable_values must cover exactly {sorted(trainable)}, "
                             f"got {sorted(given)}")
        compiled = circuit.compiled()
        enc = encoding_set(circuit)
        binding = {k: np.asarray(v, np.float64) for k, v in trainable_values.items()}
        binding[enc.name] = np.zeros(enc.size)
        return compiled.flat_values(binding)

    def run_batch(self, request: BatchRequest) -> BatchResult:
        import torch

        circuit = request.circuit
        if request.method not in METHODS:
            raise ValueError(f"unknown method {request.method!r}; expected one of {METHODS}")
        if request.method not in GPU_METHODS:
            raise NotImplementedError(f"method {request.method!r} is not on the GPU path "
                                      "(adjoint only)")
        enc = encoding_set(circuit)
        inputs = np.asarray(request.inputs, dtype=np.float64)
        if inputs.ndim != 2 or inputs.shape[1] != enc.size:
            raise ValueError(f"inputs must have shape (B, {enc.size}), got {inputs.shape}")
        observables = list(request.observables)
        ObservablePack.from_observables(observables, circuit.num_qubits)  # dimension checks
        layout = WrtLayout.build(circuit.compiled(), request.wrt)
        flat = self.base_flat(circuit, request.trainable_values)
        B, M, C = inputs.shape[0], len(observables), layout.n_cols
        if B == 0 or M == 0:
            grad = np.zeros((B, M, C))
            return BatchResult(np.empty((B, M)),
                               {n: np.ascontiguousarray(grad[:, :, lo:hi])
                                for n, lo, hi in layout.slices})
        dev = self.device
        plan, _ = self.plans.get(circuit, observables, tuple(request.wrt), dev)
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev)
            d_in = torch.from_numpy(inputs).to(dev)
            d_w = torch.from_numpy(flat).to(dev)
            expect = torch.empty((B, M), dtype=torch.float64, device=dev)
            if C == 0:
                ws = self.workspace.get(plan.workspace_bytes(B, native.VQC_MODE_FORWARD), dev)
                plan.forward(d_in, d_w, expect, ws, stream.cuda_stream)
                jac = None
            else:
                ws = self.workspace.get(plan.workspace_bytes(B, native.VQC_MODE_JACOBIAN), dev)
                jac = torch.empty((B, M, C), dtype=torch.float64, device=dev)
                plan.adjoint(d_in, d_w, None, expect, jac, None, None, ws, stream.cuda_stream)
            expect_h = expect.cpu().numpy()
            jac_h = jac.cpu().numpy() if jac is not None else np.zeros((B, M, 0))
        return BatchResult(expect_h, {n: np.ascontiguousarray(jac_h[:, :, lo:hi])
                                      for n, lo, hi in layout.slices})


_default: BatchEngine | None = None


def default_engine() -> BatchEngine:
    global _default
    if _default is None:
        _default = BatchEngine()
    return _default


def run_batch(request: BatchRequest) -> BatchResult:
    return default_engine().run_batch(request)
