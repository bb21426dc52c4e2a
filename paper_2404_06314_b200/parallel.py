"""Batch sharding across the GPUs of one node.

The reference parallelises a batch over worker threads with a static
contiguous split (batch.py:54-72, 182-212): rows are independent, every
worker writes disjoint rows, results are bit-identical for any thread count.
Here the same split distributes rows over ranks (one process per GPU,
torch.distributed); each rank runs its rows through libvqc.so and the only
exchange is one all-reduce (sum) of the batch-summed weight gradient — the
data-parallel step BASELINE config 4/5 name. Per-row outputs (expectations,
input gradients, Jacobian rows) stay on their rank unless gathered.

The functions take the per-shard compute as a callable so the sharding and
reduction logic is testable on CPU with the gloo backend.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .engine import split_workload


@dataclass
class ShardResult:
    rows: tuple[int, int]          # [lo, hi) global rows of this rank
    expectations: np.ndarray       # (hi - lo, M)
    vjp_rows: np.ndarray           # (hi - lo, n_cols) per-row VJP (input gradients live here)
    vjp_sum: np.ndarray            # (n_cols,) summed over ALL ranks after the all-reduce


def shard_rows(batch: int, world: int, rank: int) -> tuple[int, int]:
    """This rank's contiguous row range (batch.py:54-72 split over ranks)."""
    return split_workload(batch, world)[rank]


def allreduce_sum(vec, group=None):
    """Sum a 1-D gradient vector over ranks in place (one collective).

    numpy input goes through a CPU tensor (gloo); torch CUDA tensors go
    straight to NCCL.
    """
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return vec
    if isinstance(vec, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(vec))
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t.numpy()
    dist.all_reduce(vec, op=dist.ReduceOp.SUM, group=group)
    return vec


def sharded_vjp(inputs: np.ndarray, upstream: np.ndarray,
                compute: Callable[[np.ndarray, np.ndarray], tuple[np.ndarray, np.ndarray, np.ndarray]],
                rank: int, world: int, group=None) -> ShardResult:
    """Run this rank's rows through ``compute(x_rows, u_rows) -> (expect, vjp_rows, vjp_sum)``
    and all-reduce the weight-gradient sum."""
    lo, hi = shard_rows(inputs.shape[0], world, rank)
    expect, rows, vsum = compute(inputs[lo:hi], upstream[lo:hi])
    vsum = allreduce_sum(np.array(vsum, dtype=np.float64, copy=True), group)
    return ShardResult((lo, hi), expect, rows, vsum)


def gather_rows(local: np.ndarray, batch: int, world: int, group=None) -> np.ndarray:
    """All-gather per-row outputs into the full (batch, ...) array on every rank."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or world == 1:
        return local
    ranges = split_workload(batch, world)
    width = local.shape[1:] if local.ndim > 1 else ()
    pad_rows = max(hi - lo for lo, hi in ranges)
    buf = np.zeros((pad_rows, *width))
    buf[: local.shape[0]] = local
    t = torch.from_numpy(buf)
    outs = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    return np.concatenate([o.numpy()[: hi - lo] for o, (lo, hi) in zip(outs, ranges)], axis=0)


def allreduce_module_grads(module, group=None) -> None:
    """Sum every parameter's .grad over ranks with a single flattened
    collective (QuantumModule weights after a sharded backward)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    grads = [p.grad for p in module.parameters() if p.grad is not None]
    if not grads:
        return
    flat = torch.cat([g.reshape(-1) for g in grads])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    off = 0
    for g in grads:
        g.copy_(flat[off: off + g.numel()].view_as(g))
        off += g.numel()


def sharded_run_batch(request, run: Callable, rank: int, world: int, group=None,
                      gather: bool = True):
    """``run_batch`` semantics over ranks for any method: this rank evaluates
    its contiguous rows (``row_offset`` keeps SPSA's per-row seeds global, as
    the reference's worker threads do, batch.py:197), then expectations and
    Jacobians are all-gathered in row order. ``run(request) -> BatchResult``
    is the per-rank engine call (``BatchEngine.run_batch`` on this rank's GPU)."""
    import dataclasses

    from .engine import BatchResult

    inputs = np.asarray(request.inputs, np.float64)
    B = inputs.shape[0]
    lo, hi = shard_rows(B, world, rank)
    local = run(dataclasses.replace(request, inputs=inputs[lo:hi],
                                    row_offset=request.row_offset + lo))
    if not gather:
        return local
    M = local.expectations.shape[1]
    expect = gather_rows(local.expectations, B, world, group)
    grads = {}
    for name, g in local.gradients.items():
        flat = gather_rows(g.reshape(g.shape[0], -1), B, world, group)
        grads[name] = np.ascontiguousarray(flat.reshape(B, M, -1))
    return BatchResult(expect, grads)
