"""QuantumModule (torch.nn.Module) + the autograd node over libvqc.so.

Reference: vqckit/model.py:27-142 — initializers, construction-order
parameter sets drawn from one ``default_rng(seed)``, ``forward`` /
``jacobians`` / ``backward``. The reference's autograd node is the TypeScript
``QuantumLayer`` (frontend/src/autograd.ts:78-123, engine_server.py:102-139):
forward saves the inputs; backward returns the per-set VJP plus the optional
input gradient. ``QuantumFunction`` is that node as a torch.autograd.Function:

* forward  -> ``vqc_forward``: (B, M) expectations;
* backward -> ``vqc_adjoint`` in VJP mode: one fused forward + adjoint sweep
  seeded with sum_m u[b,m] O_m (2 reverse state sweeps instead of the
  reference's M+1), giving the per-row input gradient and the batch-summed
  weight gradient.

API note: ``torch.nn.Module.parameters()`` keeps torch semantics (optimizers
need it); the reference's ``parameters()`` dict is ``values`` /
``parameter_values()`` here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import native
from .engine import BatchEngine, BatchRequest, BatchResult, encoding_set

TWO_PI = 2.0 * np.pi


@dataclass(frozen=True)
class Uniform:
    lo: float = 0.0
    hi: float = TWO_PI

    def draw(self, rng, size):
        return rng.uniform(self.lo, self.hi, size)


@dataclass(frozen=True)
class Constant:
    value: float = 1.0

    def draw(self, rng, size):
        return np.full(size, float(self.value))


@dataclass(frozen=True)
class Normal:
    mean: float = 0.0
    stddev: float = 1.0

    def draw(self, rng, size):
        return rng.normal(self.mean, self.stddev, size)


class QuantumFunction(torch.autograd.Function):
    """(inputs (B,F), flat (P,)) -> expectations (B,M) with adjoint backward."""

    @staticmethod
    def forward(ctx, inputs, flat, module, group=None):
        dev = inputs.device
        plan = module._plan(with_inputs=False, group=group)
        B = inputs.shape[0]
        expect = torch.empty((B, module.num_outputs), dtype=torch.float64, device=dev)
        if B > 0 and module.num_outputs > 0:
            ws = module._engine.workspace.get(plan.workspace_bytes(B, native.VQC_MODE_FORWARD), dev)
            with torch.cuda.device(dev):   # launches go to the plan's device context
                plan.forward(inputs, flat, expect, ws, torch.cuda.current_stream(dev).cuda_stream)
        ctx.module, ctx.group = module, group
        ctx.save_for_backward(inputs, flat)
        return expect

    @staticmethod
    def backward(ctx, grad_out):
        inputs, flat = ctx.saved_tensors
        module = ctx.module
        need_x = ctx.needs_input_grad[0]
        plan = module._plan(with_inputs=need_x, group=ctx.group)
        dev = inputs.device
        B = inputs.shape[0]
        upstream = grad_out.contiguous().to(torch.float64)
        rows = torch.empty((B, plan.num_cols), dtype=torch.float64, device=dev)
        vsum = torch.empty((plan.num_cols,), dtype=torch.float64, device=dev)
        ws = module._engine.workspace.get(plan.workspace_bytes(B, native.VQC_MODE_VJP), dev)
        with torch.cuda.device(dev):
            plan.adjoint(inputs, flat, upstream, None, None, rows, vsum, ws,
                         torch.cuda.current_stream(dev).cuda_stream)
        grad_flat = torch.zeros_like(flat)
        cols = module._trainable_cols
        grad_flat[module._trainable_flat] = vsum[:cols]
        grad_x = rows[:, cols:] if need_x else None
        return grad_x, grad_flat, None, None


class QuantumModule(torch.nn.Module):
    """Trainable multi-observable quantum model over one encoding set.

    Construction mirrors model.py:60-97: ``trainable`` is an ordered sequence
    of set names or (name, initializer) pairs; unlisted initializers default
    to Uniform[0, 2pi); values are drawn in that order from one
    ``np.random.default_rng(seed)``. ``precision="complex64"`` evolves
    single-precision states (float64 angles, reductions and outputs; within
    1e-5 of the complex128 reference).
    """

    def __init__(self, circuit, observables, encoding_set: str, trainable,
                 seed: int | None = None, threads: int | None = None,
                 method: str = "adjoint", device=None, precision: str = "complex128"):
        super().__init__()
        self.circuit = circuit
        self.observables = list(observables)
        self.method = method
        enc = circuit.set_named(encoding_set)
        if enc.role != "encoding":
            raise ValueError(f"set {encoding_set!r} has role {enc.role!r}, "
                             "expected an encoding set")
        self.encoding_set = encoding_set
        specs = []
        for item in trainable:
            if isinstance(item, str):
                specs.append((item, Uniform(0.0, TWO_PI)))
            else:
                name, init = item
                specs.append((str(name), init))
        names = [n for n, _ in specs]
        if len(set(names)) != len(names):
            raise ValueError(f"parameter set declared twice: {names}")
        missing = {s.name for s in circuit.sets_with_role("trainable")} - set(names)
        if missing:
            raise ValueError(f"trainable sets not configured: {sorted(missing)}")
        for n in names:
            if circuit.set_named(n).role != "trainable":
                raise ValueError(f"set {n!r} is not trainable")
        self.trainable_specs = tuple(specs)
        rng = np.random.default_rng(seed)
        self._engine = BatchEngine(threads, device=device, precision=precision)
        dev = self._engine.device
        self._params = torch.nn.ParameterList()
        for n, init in specs:
            vals = np.asarray(init.draw(rng, circuit.set_named(n).size), np.float64)
            self._params.append(torch.nn.Parameter(torch.from_numpy(vals.copy()).to(dev)))
        compiled = circuit.compiled()
        self._enc_off, self._enc_size = compiled.offsets[encoding_set]
        flat_idx = []
        for n in names:
            off, size = compiled.offsets[n]
            flat_idx.extend(range(off, off + size))
        self._trainable_flat = torch.as_tensor(flat_idx, dtype=torch.long, device=dev)
        self._trainable_cols = len(flat_idx)
        self._total = compiled.total_params

    # -- reference-shaped accessors --------------------------------------------
    @property
    def values(self) -> dict:
        return {n: p for (n, _), p in zip(self.trainable_specs, self._params)}

    def parameter_values(self) -> dict:
        return {n: p.detach().cpu().numpy().copy() for n, p in self.values.items()}

    @property
    def num_outputs(self) -> int:
        return len(self.observables)

    @property
    def encoding_size(self) -> int:
        return self.circuit.set_named(self.encoding_set).size

    def trainable_names(self) -> tuple[str, ...]:
        return tuple(n for n, _ in self.trainable_specs)

    # -- plumbing ----------------------------------------------------------------
    def _plan(self, with_inputs: bool, group=None):
        wrt = self.trainable_names() + ((self.encoding_set,) if with_inputs else ())
        circ, obs = ((self.circuit, self.observables) if group is None
                     else self._basis_groups()[group])
        plan, _ = self._engine.plans.get(circ, obs, wrt, self._engine.device)
        return plan

    def _basis_groups(self):
        """None when the plan takes the observables directly; for X/Y Pauli
        strings on HBM plans (n > 12) the [(basis circuit, Z observables)]
        split of engine.basis_groups, whose outputs sum to the original."""
        if "_groups" not in self.__dict__:
            from .engine import SMEM_MAX_QUBITS, basis_circuit, basis_groups
            groups = None
            if (self.circuit.num_qubits > SMEM_MAX_QUBITS
                    and not all(o.is_z_only for o in self.observables)):
                groups = [(basis_circuit(self.circuit, pat), obs)
                          for pat, obs in basis_groups(self.observables, self.circuit.num_qubits)]
            self.__dict__["_groups"] = groups
        return self.__dict__["_groups"]

    def flat_weights(self) -> torch.Tensor:
        """Flat parameter vector in declaration order, encoding slot zeroed."""
        dev = self._engine.device
        parts = {n: p for n, p in self.values.items()}
        chunks = []
        for s in self.circuit.parameter_sets:
            if s.name in parts:
                chunks.append(parts[s.name])
            else:
                chunks.append(torch.zeros(s.size, dtype=torch.float64, device=dev))
        if not chunks:
            return torch.zeros(0, dtype=torch.float64, device=dev)
        return torch.cat(chunks)

    def _as_inputs(self, inputs) -> torch.Tensor:
        dev = self._engine.device
        if not torch.is_tensor(inputs):
            inputs = torch.from_numpy(np.atleast_2d(np.asarray(inputs, np.float64)))
        if inputs.dim() == 1:
            inputs = inputs.unsqueeze(0)
        if inputs.dim() != 2 or inputs.shape[1] != self.encoding_size:
            raise ValueError(f"inputs must have shape (B, {self.encoding_size}), "
                             f"got {tuple(inputs.shape)}")
        return inputs.to(device=dev, dtype=torch.float64).contiguous()

    # -- API ---------------------------------------------------------------------
    def forward(self, inputs) -> torch.Tensor:
        """(B, M) expectations; differentiable w.r.t. weights and inputs."""
        x, flat = self._as_inputs(inputs), self.flat_weights()
        groups = self._basis_groups()
        if groups is None:
            return QuantumFunction.apply(x, flat, self, None)
        out = QuantumFunction.apply(x, flat, self, 0)
        for g in range(1, len(groups)):
            out = out + QuantumFunction.apply(x, flat, self, g)
        return out

    def jacobians(self, inputs, method: str | None = None, wrt=None,
                  threads: int | None = None) -> BatchResult:
        """Raw (B, M) expectations and (B, M, set.size) gradients (model.py:644-649)."""
        wrt = self.trainable_names() if wrt is None else tuple(wrt)
        x = self._as_inputs(inputs).cpu().numpy()
        req = BatchRequest(self.circuit, self.observables, self.parameter_values(), x,
                           method=method or self.method, wrt=wrt, threads=threads)
        return self._engine.run_batch(req)

    def backward(self, inputs, upstream, method: str | None = None,
                 threads: int | None = None) -> dict:
        """sum_{b,m} upstream[b,m] d<O_m>(x_b)/dp per trainable set (model.py:651-662).

        Computed as one VJP-seeded adjoint sweep rather than the reference's
        full Jacobian followed by an einsum."""
        x = self._as_inputs(inputs)
        up = np.asarray(upstream.detach().cpu() if torch.is_tensor(upstream) else upstream,
                        dtype=np.float64)
        expected = (x.shape[0], self.num_outputs)
        if up.shape != expected:
            raise ValueError(f"upstream shape {up.shape} does not match forward output {expected}")
        if (method or self.method) != "adjoint":
            # shift / SPSA: the reference's Jacobian + einsum (model.py:140-142)
            res = self.jacobians(x, method=method, threads=threads)
            return {n: np.einsum("bm,bmp->p", up, t) for n, t in res.gradients.items()}
        dev = self._engine.device
        B = x.shape[0]
        groups = self._basis_groups()
        host = None
        for g in (range(len(groups)) if groups is not None else (None,)):
            plan = self._plan(with_inputs=False, group=g)
            vsum = torch.zeros(plan.num_cols, dtype=torch.float64, device=dev)
            if B > 0 and self.num_outputs > 0:
                d_up = torch.from_numpy(np.ascontiguousarray(up)).to(dev)
                ws = self._engine.workspace.get(plan.workspace_bytes(B, native.VQC_MODE_VJP), dev)
                with torch.no_grad(), torch.cuda.device(dev):
                    plan.adjoint(x, self.flat_weights().detach(), d_up, None, None, None, vsum,
                                 ws, torch.cuda.current_stream(dev).cuda_stream)
            part = vsum.cpu().numpy()
            host = part if host is None else host + part
        out, col = {}, 0
        for n in self.trainable_names():
            size = self.circuit.set_named(n).size
            out[n] = host[col:col + size].copy()
            col += size
        return out


def _single_qubit(obs) -> bool:
    return all(sum(ch != "I" for ch in string) <= 1 for _, string in obs.terms)


class HybridModule(torch.nn.Module):
    """Dense pre-layer -> pi*tanh squash -> QuantumModule -> dense post-layer.

    Mirrors model.py:152-222 (same initialisation order and bounds from one
    ``default_rng(seed)``; single-qubit observables required). Gradients flow
    through QuantumFunction, i.e. the quantum core's input gradient comes from
    the same VJP-seeded adjoint sweep as its weight gradient.
    """

    def __init__(self, input_dim: int, quantum: QuantumModule, output_dim: int, seed: int | None = None):
        super().__init__()
        for obs in quantum.observables:
            if not _single_qubit(obs):
                raise ValueError("hybrid quantum core must use single-qubit observables")
        self.input_dim = int(input_dim)
        self.output_dim = int(output_dim)
        self.quantum = quantum
        enc, m = quantum.encoding_size, quantum.num_outputs
        rng = np.random.default_rng(seed)
        bp = 1.0 / np.sqrt(max(1, input_dim))
        bq = 1.0 / np.sqrt(max(1, m))
        dev = quantum._engine.device

        def param(a):
            return torch.nn.Parameter(torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(dev))

        self.pre_weight = param(rng.uniform(-bp, bp, (enc, input_dim)))
        self.pre_bias = param(rng.uniform(-bp, bp, enc))
        self.post_weight = param(rng.uniform(-bq, bq, (output_dim, m)))
        self.post_bias = param(rng.uniform(-bq, bq, output_dim))

    def forward(self, inputs) -> torch.Tensor:
        x = inputs if torch.is_tensor(inputs) else torch.from_numpy(np.atleast_2d(np.asarray(inputs, np.float64)))
        x = x.to(device=self.pre_weight.device, dtype=torch.float64)
        if x.dim() != 2 or x.shape[1] != self.input_dim:
            raise ValueError(f"inputs must have shape (B, {self.input_dim}), got {tuple(x.shape)}")
        angles = torch.pi * torch.tanh(x @ self.pre_weight.T + self.pre_bias)
        return self.quantum(angles) @ self.post_weight.T + self.post_bias

    def backward(self, inputs, upstream) -> dict:
        """Gradients of sum(upstream * forward) per weight block (model.py:720-742)."""
        up = torch.as_tensor(np.asarray(upstream.detach().cpu() if torch.is_tensor(upstream) else upstream,
                                        dtype=np.float64), device=self.pre_weight.device)
        n = np.atleast_2d(np.asarray(inputs.detach().cpu() if torch.is_tensor(inputs) else inputs)).shape[0]
        if tuple(up.shape) != (n, self.output_dim):
            raise ValueError(f"upstream shape {tuple(up.shape)} does not match (B, {self.output_dim})")
        named = {"pre.weight": self.pre_weight, "pre.bias": self.pre_bias,
                 "post.weight": self.post_weight, "post.bias": self.post_bias}
        named.update(self.quantum.values)
        for p in named.values():
            p.grad = None
        out = self.forward(inputs)
        out.backward(up)
        return {k: v.grad.detach().cpu().numpy().copy() for k, v in named.items()}
