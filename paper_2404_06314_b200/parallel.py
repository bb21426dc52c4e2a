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


def _comm_device(group=None):
    """Where collective buffers live: the current CUDA device under NCCL
    (NCCL only moves device memory), host memory under gloo."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _active(group=None) -> bool:
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1


def allreduce_sum(vec, group=None):
    """Sum a 1-D gradient vector over ranks (one collective). torch tensors
    are reduced in place on their own device; numpy arrays are staged through
    a tensor on the backend's device and returned as a new array."""
    import torch
    import torch.distributed as dist

    if not _active(group):
        return vec
    if isinstance(vec, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(vec, np.float64)).to(_comm_device(group))
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t.cpu().numpy()
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
    """All-gather per-row outputs into the full (batch, ...) array on every
    rank. Shards may be empty (batch < world, batch == 0): every rank sends a
    buffer padded to the largest shard (at least one row)."""
    import torch
    import torch.distributed as dist

    if not _active(group) or world == 1:
        return local
    ranges = split_workload(batch, world)
    width = tuple(local.shape[1:])
    pad_rows = max(1, max(hi - lo for lo, hi in ranges))
    buf = np.zeros((pad_rows, *width))
    buf[: local.shape[0]] = local
    t = torch.from_numpy(buf).to(_comm_device(group))
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    parts = [o.cpu().numpy()[: hi - lo] for o, (lo, hi) in zip(outs, ranges)]
    return np.concatenate(parts, axis=0).reshape(batch, *width)


def allreduce_module_grads(module, group=None) -> None:
    """Sum every parameter's .grad over ranks with a single flattened
    collective (QuantumModule weights after a sharded backward)."""
    import torch
    import torch.distributed as dist

    if not _active(group):
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

    from .engine import BatchInputError

    inputs = np.asarray(request.inputs, np.float64)
    B = inputs.shape[0]
    lo, hi = shard_rows(B, world, rank)
    # a failing row (BatchInputError, batch.py:196-202) must fail every rank:
    # the lowest failing global index is agreed on before anyone leaves, or
    # the other ranks would wait in the gather below
    failed, cause = -1, None
    local = None
    try:
        local = run(dataclasses.replace(request, inputs=inputs[lo:hi],
                                        row_offset=request.row_offset + lo))
    except BatchInputError as exc:
        failed, cause = exc.index, exc.__cause__ or exc
    if _active(group) and world > 1:
        import torch
        import torch.distributed as dist
        big = np.iinfo(np.int64).max
        t = torch.tensor([failed if failed >= 0 else big], dtype=torch.int64, device=_comm_device(group))
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        first = int(t.item())
        if first != big:
            raise BatchInputError(first, cause if failed == first else RuntimeError("row failed on another rank"))
    elif failed >= 0:
        raise BatchInputError(failed, cause)
    if not gather:
        return local
    expect = gather_rows(local.expectations, B, world, group)
    grads = {}
    for name, g in local.gradients.items():
        # explicit widths: numpy cannot infer -1 for a zero-row shard
        rows, m, size = g.shape
        flat = gather_rows(g.reshape(rows, m * size), B, world, group)
        grads[name] = np.ascontiguousarray(flat.reshape(B, m, size))
    return BatchResult(expect, grads)
