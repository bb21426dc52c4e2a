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
GPU_METHODS = METHODS
_MASK64 = (1 << 64) - 1
# rows of angle vectors per forward launch in the shift/SPSA paths (bounds the
# (rows, R) f64 input block and the (rows, M) result block)
SHIFT_CHUNK_ROWS = 1 << 18


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
    row_offset: int = 0                 # global index of row 0 (rank shards: SPSA seeds)


@dataclass
class BatchResult:
    expectations: np.ndarray            # (B, M)
    gradients: dict = field(default_factory=dict)   # set -> (B, M, size)


class BatchInputError(RuntimeError):
    """A row failed; carries its index (batch.py:104-109)."""

    def __init__(self, index: int, cause: Exception):
        super().__init__(f"batch input {index} failed: {cause}")
        self.index = index


def _check_rows(values: np.ndarray, row_offset: int, what: str) -> None:
    """Per-row failure reporting (batch.py:196-202). The reference wraps
    whatever a row's worker raises in ``BatchInputError(index)``; a GPU row
    cannot raise, so a row fails when its inputs or its expectations are not
    finite, and the first such row is reported by its global index."""
    rows = values.reshape(values.shape[0], -1)
    bad = ~np.isfinite(rows).all(axis=1)
    if bad.any():
        b = int(np.argmax(bad))
        raise BatchInputError(row_offset + b, FloatingPointError(f"non-finite {what}"))


def encoding_set(circuit: Circuit):
    enc = circuit.sets_with_role("encoding")
    if len(enc) != 1:
        raise ValueError(f"batched evaluation needs exactly one encoding set, "
                         f"circuit has {len(enc)}")
    return enc[0]


def angle_circuit(circuit: Circuit):
    """The circuit with every rotation's angle made a direct input: one
    encoding set ``angles`` of size R, rotation r = 1.0 * angles[r]. Running
    it forward on rows of per-gate angles is how the shift / SPSA methods
    batch their shifted evaluations onto the GPU forward kernel. Returns
    (circuit, rotation gate indices); cached on the source circuit."""
    from .ir import AngleExpression, Gate, ParameterSet
    cached = circuit.__dict__.get("_angle_circuit")
    if cached is None:
        rot = [g for g, gate in enumerate(circuit.gates) if gate.expr is not None]
        slot = {g: r for r, g in enumerate(rot)}
        gates = tuple(
            Gate(gate.kind, gate.qubits, AngleExpression(1.0, (("angles", slot[g]),)))
            if gate.expr is not None else gate
            for g, gate in enumerate(circuit.gates))
        ac = Circuit(circuit.num_qubits, gates,
                     (ParameterSet("angles", len(rot), "encoding"),))
        cached = (ac, np.asarray(rot, np.int64))
        object.__setattr__(circuit, "_angle_circuit", cached)
    return cached


def row_angles(compiled, flats: np.ndarray, rot: np.ndarray) -> np.ndarray:
    """angle_g = coeff_g * prod factors (compute_angles, _kernels.py:128-134)
    for every row of ``flats`` (rows, total_params) -> (rows, R), factors
    multiplied in declaration order like the reference."""
    out = np.empty((flats.shape[0], len(rot)))
    for r, g in enumerate(rot):
        a = np.full(flats.shape[0], compiled.coeff[g])
        for t in range(compiled.f_offs[g], compiled.f_offs[g + 1]):
            a = a * flats[:, compiled.f_idx[t]]
        out[:, r] = a
    return out


def device_row_angles(compiled, flats, rot: np.ndarray):
    """``row_angles`` on a device tensor of flat rows: factors gathered per
    rotation and multiplied left to right after the coefficient; ragged
    factor lists are padded with an all-ones column (x * 1.0 is exact)."""
    import torch
    P = flats.shape[1]
    nf = [int(compiled.f_offs[g + 1] - compiled.f_offs[g]) for g in rot]
    width = max(nf, default=0)
    gather = np.full((len(rot), width), P, np.int64)
    for r, g in enumerate(rot):
        gather[r, :nf[r]] = compiled.f_idx[compiled.f_offs[g]:compiled.f_offs[g + 1]]
    ext = torch.cat([flats, torch.ones_like(flats[:, :1])], dim=1)
    d_gather = torch.from_numpy(gather).to(flats.device)
    a = torch.from_numpy(compiled.coeff[rot].copy()).to(flats.device)[None, :].expand(
        flats.shape[0], -1)
    for k in range(width):
        a = a * ext[:, d_gather[:, k]]
    return a.contiguous()


SMEM_MAX_QUBITS = 12     # on-chip plans take any Pauli string (engine.cu kSmemMaxQubits)


def basis_groups(observables, num_qubits: int):
    """Split every observable's terms by their X/Y pattern. Returns
    [(pattern, [Observable per m])]: pattern[q] is "X", "Y" or "-", and each
    group's observables are Z strings (X/Y -> Z; an observable with no term in
    the group gets a zero-weight identity term, so Sum_groups == original)."""
    groups: dict = {}
    for m, obs in enumerate(observables):
        for coeff, string in obs.terms:
            pat = "".join(ch if ch in "XY" else "-" for ch in string.upper())
            zs = "".join("Z" if ch in "XYZ" else "I" for ch in string.upper())
            groups.setdefault(pat, [[] for _ in observables])[m].append((coeff, zs))
    ident = "I" * num_qubits
    return [(pat, [Observable(tuple(t) if t else ((0.0, ident),)) for t in per_m])
            for pat, per_m in groups.items()]


def basis_circuit(circuit: Circuit, pattern: str) -> Circuit:
    """The circuit followed by the constant basis change U with U^dag Z U = P
    per qubit: H for X, RX(pi/2) for Y (e^{i pi X/4} Z e^{-i pi X/4} = Y).
    Constant-angle rotations carry no factors, so no gradient columns."""
    from .ir import AngleExpression, Gate, GateKind
    extra = []
    for q, ch in enumerate(pattern):     # Pauli char k acts on qubit k
        if ch == "X":
            extra.append(Gate(GateKind.H, (q,)))
        elif ch == "Y":
            extra.append(Gate(GateKind.RX, (q,), AngleExpression(0.5 * np.pi, ())))
    return Circuit(circuit.num_qubits, circuit.gates + tuple(extra), circuit.parameter_sets)


def _device(device):
    import torch
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the vqc GPU path has no CPU fallback")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


class PlanCache:
    """(circuit, observables, wrt, device, precision) -> native.Plan."""

    def __init__(self, precision: str = "complex128"):
        if precision not in native.PRECISIONS:
            raise ValueError(f"precision must be one of {tuple(native.PRECISIONS)}, got {precision!r}")
        self.precision = precision
        self._plans: dict = {}
        self._lock = threading.Lock()

    def get(self, circuit: Circuit, observables, wrt: tuple, device):
        key = (circuit, tuple(observables), tuple(wrt), str(device), self.precision)
        with self._lock:
            plan = self._plans.get(key)
            if plan is None:
                compiled = circuit.compiled()
                pack = ObservablePack.from_observables(observables, circuit.num_qubits)
                layout = WrtLayout.build(compiled, wrt)
                enc = encoding_set(circuit)
                off, size = compiled.offsets[enc.name]
                plan = (native.Plan(compiled, pack, layout.wrt_col, off, size, device,
                                    self.precision), layout)
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
    """GPU replacement for vqckit's BatchEngine (batch.py:120-217).

    ``precision``: "complex128" (the reference's state type, default) or
    "complex64" (single-precision states, float64 angles, reductions and
    outputs; matches the reference to 1e-5)."""

    def __init__(self, threads: int | None = None, device=None, precision: str = "complex128"):
        if threads is not None and threads < 1:
            raise ValueError(f"threads must be >= 1, got {threads}")
        self.threads = threads
        self._device_arg = device
        self.precision = precision
        self.plans = PlanCache(precision)
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
        _check_rows(inputs, request.row_offset, "input")
        if circuit.num_qubits > SMEM_MAX_QUBITS and not all(o.is_z_only for o in observables):
            return self._run_basis_groups(request, observables, layout, B, M, C)
        dev = self.device
        if C > 0 and request.method != "adjoint":
            expect_h, grad_h = self._run_shifted(request, circuit, observables, layout,
                                                 flat, inputs)
            return BatchResult(expect_h, {n: np.ascontiguousarray(grad_h[:, :, lo:hi])
                                          for n, lo, hi in layout.slices})
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
        _check_rows(expect_h, request.row_offset, "expectation (non-finite parameters?)")
        return BatchResult(expect_h, {n: np.ascontiguousarray(jac_h[:, :, lo:hi])
                                      for n, lo, hi in layout.slices})


    def _run_basis_groups(self, request, observables, layout, B, M, C) -> BatchResult:
        """X/Y Pauli strings on HBM plans (n > 12): one Z-basis run per X/Y
        pattern over the basis-rotated circuit; expectations and Jacobians
        are sums over groups (expectations are linear in the observable)."""
        import dataclasses
        expect = np.zeros((B, M))
        grads = {n: np.zeros((B, M, hi - lo)) for n, lo, hi in layout.slices}
        cache = request.circuit.__dict__.setdefault("_basis_circuits", {})
        for pattern, group_obs in basis_groups(observables, request.circuit.num_qubits):
            if pattern not in cache:
                cache[pattern] = basis_circuit(request.circuit, pattern)
            res = self.run_batch(dataclasses.replace(request, circuit=cache[pattern],
                                                     observables=group_obs))
            expect += res.expectations
            for n in grads:
                grads[n] += res.gradients[n]
        return BatchResult(expect, grads)

    def forward_angle_rows(self, circuit: Circuit, observables, angles: np.ndarray,
                           as_tensor: bool = False) -> np.ndarray:
        """Expectations (rows, M) of ``circuit`` with per-row rotation angles
        (rows, R): one GPU forward launch sequence over ``angle_circuit``.
        X/Y strings on HBM plans (n > 12) run one Z-basis launch per basis
        group over the angle circuit followed by its constant basis change
        (the same split as ``run_batch``)."""
        ac, _ = angle_circuit(circuit)
        if circuit.num_qubits > SMEM_MAX_QUBITS and not all(o.is_z_only for o in observables):
            cache = ac.__dict__.setdefault("_basis_circuits", {})
            total = None
            for pattern, group_obs in basis_groups(observables, circuit.num_qubits):
                if pattern not in cache:
                    cache[pattern] = basis_circuit(ac, pattern)
                e = self._forward_rows(cache[pattern], group_obs, angles, as_tensor)
                total = e if total is None else total + e
            return total
        return self._forward_rows(ac, observables, angles, as_tensor)

    def _forward_rows(self, ac: Circuit, observables, angles, as_tensor: bool = False):
        import torch
        dev = self.device
        plan, _ = self.plans.get(ac, observables, (), dev)
        rows, M = angles.shape[0], len(observables)
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev)
            d_in = (angles.contiguous() if torch.is_tensor(angles)
                    else torch.from_numpy(np.ascontiguousarray(angles)).to(dev))
            d_w = torch.zeros(max(1, angles.shape[1]), dtype=torch.float64, device=dev)
            expect = torch.empty((rows, M), dtype=torch.float64, device=dev)
            ws = self.workspace.get(plan.workspace_bytes(rows, native.VQC_MODE_FORWARD), dev)
            plan.forward(d_in, d_w, expect, ws, stream.cuda_stream)
            return expect if as_tensor else expect.cpu().numpy()

    def _run_shifted(self, request, circuit, observables, layout, flat, inputs,
                     rng_for_row=None, single_seed=None):
        """param-shift (gradients.py:137-160) and SPSA (gradients.py:180-201)
        as batched GPU forward evaluations. Each row's shifted / perturbed
        evaluations become extra rows of per-gate angles (computed on the host
        in the reference's arithmetic order), so a chunk of B rows is one
        forward call over B*(1+2S) angle rows. SPSA draws its directions
        natively (vqc_spsa_signs, bit for bit numpy's per-row generators) and
        forms its estimate on the device in the reference's accumulation
        order; param-shift's differences and chain rule through the angle
        expressions run on the device too (one FP64 matrix product sums the
        terms of a column)."""
        import torch
        compiled = circuit.compiled()
        enc = encoding_set(circuit)
        off, size = compiled.offsets[enc.name]
        _, rot = angle_circuit(circuit)
        B, M, C = inputs.shape[0], len(observables), layout.n_cols
        expect = np.empty((B, M))
        grad = np.zeros((B, M, C))
        f_offs, f_idx, wrt_col = compiled.f_offs, compiled.f_idx, layout.wrt_col
        if request.method == "param-shift":
            # rotation slots with a requested factor (row-independent) and,
            # per slot, (column, factor positions of the other factors)
            shifted, partials = [], []
            for r, g in enumerate(rot):
                terms = []
                for t in range(f_offs[g], f_offs[g + 1]):
                    col = wrt_col[f_idx[t]]
                    if col >= 0:
                        terms.append((int(col), [f_idx[u] for u in range(f_offs[g], f_offs[g + 1])
                                                 if u != t]))
                if terms:
                    shifted.append(r)
                    partials.append((g, terms))
            per_row = 1 + 2 * len(shifted)
            # flattened (slot, column, coefficient, other factors) terms for the
            # device-side chain rule: other-factor lists padded with an index
            # one past the flat vector (a column of ones)
            t_slot = [s for s, (_, terms) in enumerate(partials) for _ in terms]
            t_col = [col for _, terms in partials for col, _ in terms]
            t_coeff = [float(compiled.coeff[g]) for g, terms in partials for _ in terms]
            t_others = [others for _, terms in partials for _, others in terms]
            width = max([len(o) for o in t_others], default=0)
            t_pad = [list(o) + [flat.shape[0]] * (width - len(o)) for o in t_others]
        else:
            if request.spsa_samples < 1:
                raise ValueError(f"spsa_samples must be >= 1, got {request.spsa_samples}")
            per_row = 1 + 2 * request.spsa_samples
        step = max(1, SHIFT_CHUNK_ROWS // per_row)
        for lo in range(0, B, step):
            hi = min(B, lo + step)
            n = hi - lo
            flats = np.repeat(flat[None], n, 0)
            flats[:, off:off + size] = inputs[lo:hi]
            if request.method == "param-shift":
                # base angles on the host (n, R); the 1+2S shifted copies are
                # built on the device: same IEEE adds as base[r] +/- pi/2
                base = torch.from_numpy(row_angles(compiled, flats, rot)).to(self.device)
                rows = base[:, None, :].repeat(1, per_row, 1)           # (n, 1+2S, R)
                if shifted:
                    j = torch.arange(len(shifted), device=base.device) * 2 + 1
                    r = torch.as_tensor(shifted, device=base.device)
                    rows[:, j, r] = base[:, r] + 0.5 * np.pi
                    rows[:, j + 1, r] = base[:, r] - 0.5 * np.pi
                e = self.forward_angle_rows(circuit, observables, rows.view(n * per_row, -1),
                                            as_tensor=True).view(n, per_row, M)
                expect[lo:hi] = e[:, 0].cpu().numpy()
                if t_slot:
                    # occurrence values 0.5 (f+ - f-) per shifted slot, the
                    # partial of each term's angle expression w.r.t. its
                    # requested factor (coefficient times the other factors),
                    # and the sum over the terms of a column as one FP64
                    # matrix product with the 0/1 term-to-column matrix
                    dev = e.device
                    occ = 0.5 * (e[:, 1::2] - e[:, 2::2])                           # (n, S, M)
                    partial = torch.tensor(t_coeff, dtype=torch.float64, device=dev).repeat(n, 1)
                    if width:
                        ext = torch.cat([torch.from_numpy(flats).to(dev),
                                         torch.ones((n, 1), dtype=torch.float64, device=dev)], 1)
                        pad = torch.tensor(t_pad, dtype=torch.int64, device=dev)    # (T, width)
                        for u in range(width):
                            partial = partial * ext[:, pad[:, u]]
                    contrib = occ[:, torch.tensor(t_slot, device=dev)] * partial[:, :, None]   # (n, T, M)
                    onehot = torch.zeros((len(t_col), C), dtype=torch.float64, device=dev)
                    onehot[torch.arange(len(t_col), device=dev), torch.tensor(t_col, device=dev)] = 1.0
                    grad[lo:hi] = torch.matmul(contrib.transpose(1, 2), onehot).cpu().numpy()  # (n, M, C)
            else:
                K, c, idx = request.spsa_samples, request.spsa_c, layout.flat_of_col
                if single_seed is not None:
                    # single-binding form: default_rng(seed) itself for every row
                    deltas = native.spsa_signs(single_seed, 0, n, K, C, per_row_seed=False
                                               ).astype(np.float64)
                elif rng_for_row is None:
                    # the reference's per-row generators (default_rng(mix_seed(seed,
                    # global row)), batch.py:197) and draws, natively on the host
                    deltas = native.spsa_signs(request.seed, request.row_offset + lo, n, K, C
                                               ).astype(np.float64)
                else:
                    deltas = np.empty((n, K, C))
                    for i in range(n):
                        rng = rng_for_row(lo + i)
                        for k in range(K):
                            d = rng.integers(0, 2, size=C).astype(np.float64)
                            deltas[i, k] = 2.0 * d - 1.0
                # perturbed flats and their angles on the device (same IEEE
                # ops as the reference: base +/- (c * delta), then coeff * f1 * f2 ...)
                d_flats = torch.from_numpy(flats).to(self.device)
                d_idx = torch.from_numpy(idx).to(self.device)
                d_delta = torch.from_numpy(deltas).to(self.device)      # (n, K, C)
                d_cd = c * d_delta
                pf = d_flats[:, None, :].repeat(1, per_row, 1)          # (n, 1+2K, P)
                base = d_flats[:, None, d_idx]
                pf[:, 1::2][:, :, d_idx] = base + d_cd
                pf[:, 2::2][:, :, d_idx] = base - d_cd
                ang = device_row_angles(compiled, pf.view(n * per_row, -1), rot)
                e = self.forward_angle_rows(circuit, observables, ang, as_tensor=True).view(n, per_row, M)
                # the estimate on the device: the reference's elementwise IEEE
                # operations in its accumulation order (no fused multiply-add)
                d_inv = 1.0 / ((2.0 * c) * d_delta)
                g_acc = torch.zeros((n, M, C), dtype=torch.float64, device=self.device)
                for k in range(K):
                    diff = e[:, 1 + 2 * k] - e[:, 2 + 2 * k]                # (n, M)
                    g_acc += diff[:, :, None] * d_inv[:, k][:, None, :]
                expect[lo:hi] = e[:, 0].cpu().numpy()
                grad[lo:hi] = (g_acc / K).cpu().numpy()
        return expect, grad


_default: BatchEngine | None = None


def default_engine() -> BatchEngine:
    global _default
    if _default is None:
        _default = BatchEngine()
    return _default


def run_batch(request: BatchRequest) -> BatchResult:
    return default_engine().run_batch(request)
