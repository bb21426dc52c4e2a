"""Multi-rank sharding on CPU (gloo, world_size 2): the row split, the single
weight-gradient all-reduce and the row gather give the single-process result.

The per-shard compute here is the CPU oracle (test infrastructure), standing in
for libvqc.so, so the host-side data-parallel logic is exercised without GPUs.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import oracle_batch


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    from paper_2404_06314_b200 import configs
    spec = configs.CONFIGS[2]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=13)   # odd: uneven shards
    rng = np.random.default_rng(3)
    up = rng.normal(size=(13, len(obs)))
    return circ, obs, wrt, x, w, up


def _oracle_compute(circ, obs, wrt, w):
    def compute(x_rows, u_rows):
        e, jac = oracle_batch(circ, obs, {"w": w}, x_rows, wrt, threads=1)
        full = np.concatenate([jac[n] for n in wrt], axis=2)          # (b, M, cols)
        rows = np.einsum("bm,bmp->bp", u_rows, full)
        return e, rows, rows.sum(axis=0)
    return compute


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from paper_2404_06314_b200 import parallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        circ, obs, wrt, x, w, up = _problem()
        res = parallel.sharded_vjp(x, up, _oracle_compute(circ, obs, wrt, w), rank, world)
        rows = parallel.gather_rows(res.vjp_rows, x.shape[0], world)
        exp = parallel.gather_rows(res.expectations, x.shape[0], world)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), vsum=res.vjp_sum, rows=rows, exp=exp,
                 lo=res.rows[0], hi=res.rows[1])
    finally:
        dist.destroy_process_group()


def test_split_matches_reference_rule():
    from paper_2404_06314_b200.parallel import shard_rows
    # batch.py:54-72: first B - T*floor(B/T) ranges take one extra row
    assert [shard_rows(10, 4, r) for r in range(4)] == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert [shard_rows(2, 4, r) for r in range(4)] == [(0, 1), (1, 2), (2, 2), (2, 2)]


@pytest.mark.timeout(300)
def test_world_size_2_gloo(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    circ, obs, wrt, x, w, up = _problem()
    e_ref, rows_ref, sum_ref = _oracle_compute(circ, obs, wrt, w)(x, up)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        np.testing.assert_allclose(d["vsum"], sum_ref, rtol=1e-12, atol=1e-13)
        np.testing.assert_array_equal(d["rows"], rows_ref)   # per-row results are bitwise
        np.testing.assert_array_equal(d["exp"], e_ref)
    lo0, hi0 = np.load(tmp_path / "r0.npz")["lo"], np.load(tmp_path / "r0.npz")["hi"]
    assert (int(lo0), int(hi0)) == (0, 7)


def _spsa_run(circ, obs, wrt):
    """CPU stand-in for BatchEngine.run_batch(method="spsa"): the oracle's
    SPSA per row with the engine's seeding rule mix_seed(seed, row_offset + b)."""
    from oracle import oracle
    from paper_2404_06314_b200.engine import BatchResult, WrtLayout, mix_seed
    from conftest import lowered

    def run(req):
        comp = circ.compiled()
        layout = WrtLayout.build(comp, wrt)
        off, size = comp.offsets["x"]
        flat = comp.flat_values({"w": req.trainable_values["w"], "x": np.zeros(size)})
        low = lowered(circ, obs)
        B = req.inputs.shape[0]
        e = np.zeros((B, len(obs)))
        j = np.zeros((B, len(obs), layout.n_cols))
        for b in range(B):
            f = flat.copy()
            f[off:off + size] = req.inputs[b]
            rng = np.random.default_rng(mix_seed(req.seed, req.row_offset + b))
            e[b], j[b] = oracle.spsa_row(low, f, layout.flat_of_col, req.spsa_c,
                                         req.spsa_samples, rng)
        return BatchResult(e, {n: j[:, :, lo:hi] for n, lo, hi in layout.slices})
    return run


def _spsa_problem():
    from paper_2404_06314_b200 import configs
    from paper_2404_06314_b200.engine import BatchRequest
    spec = configs.CONFIGS[1]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=7)
    req = BatchRequest(circ, obs, {"w": w}, x, method="spsa", wrt=wrt, seed=5, spsa_samples=2)
    return circ, obs, wrt, req


def _spsa_worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from paper_2404_06314_b200 import parallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        circ, obs, wrt, req = _spsa_problem()
        res = parallel.sharded_run_batch(req, _spsa_run(circ, obs, wrt), rank, world)
        np.savez(os.path.join(out_dir, f"s{rank}.npz"), exp=res.expectations,
                 **{f"g_{k}": v for k, v in res.gradients.items()})
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_run_batch_spsa_seeds_are_global(tmp_path):
    """Sharded SPSA == single-process SPSA bit for bit: each rank seeds its
    rows with the GLOBAL row index (row_offset), then rows are gathered."""
    world = 2
    mp.start_processes(_spsa_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    circ, obs, wrt, req = _spsa_problem()
    full = _spsa_run(circ, obs, wrt)(req)
    for r in range(world):
        d = np.load(tmp_path / f"s{r}.npz")
        np.testing.assert_array_equal(d["exp"], full.expectations)
        for k in wrt:
            np.testing.assert_array_equal(d[f"g_{k}"], full.gradients[k])


def _tiny_run(req):
    """Per-rank stand-in with the engine's output shapes: (b, M) and (b, M, size)."""
    from paper_2404_06314_b200.engine import BatchResult
    x = np.asarray(req.inputs)
    b = x.shape[0]
    e = np.stack([x.sum(axis=1), x[:, 0] if b else np.zeros(0)], axis=1) if b else np.zeros((0, 2))
    g = np.repeat(x[:, None, :], 2, axis=1) + req.row_offset
    return BatchResult(e, {"x": g})


def _empty_worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from paper_2404_06314_b200 import parallel
    from paper_2404_06314_b200.engine import BatchRequest
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for B in (1, 0):
            x = np.arange(3.0 * B).reshape(B, 3)
            req = BatchRequest(None, [], {}, x)
            res = parallel.sharded_run_batch(req, _tiny_run, rank, world)
            np.savez(os.path.join(out_dir, f"e{B}_{rank}.npz"), exp=res.expectations,
                     g=res.gradients["x"])
        v = parallel.allreduce_sum(np.array([1.0, 2.0]))
        np.save(os.path.join(out_dir, f"v{rank}.npy"), v)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_run_batch_empty_shards(tmp_path):
    """B < world (a rank gets no rows) and B == 0 must not hang or raise."""
    world = 2
    mp.start_processes(_empty_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    for B in (1, 0):
        x = np.arange(3.0 * B).reshape(B, 3)
        from paper_2404_06314_b200.engine import BatchRequest
        full = _tiny_run(BatchRequest(None, [], {}, x))
        for r in range(world):
            d = np.load(tmp_path / f"e{B}_{r}.npz")
            assert d["exp"].shape == (B, 2) and d["g"].shape == (B, 2, 3)
            np.testing.assert_array_equal(d["exp"], full.expectations)
            np.testing.assert_array_equal(d["g"], full.gradients["x"])
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"v{r}.npy"), [2.0, 4.0])


def _failing_run(req):
    """Stand-in engine call that fails like BatchEngine.run_batch: the first
    row whose inputs are not finite, reported by its global index."""
    from paper_2404_06314_b200.engine import _check_rows
    _check_rows(np.asarray(req.inputs, np.float64), req.row_offset, "input")
    return _tiny_run(req)


def _failure_worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from paper_2404_06314_b200 import parallel
    from paper_2404_06314_b200.engine import BatchInputError, BatchRequest
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = np.arange(21.0).reshape(7, 3)
        x[5, 1] = np.nan                      # row 5 lives on rank 1 only
        got = -1
        try:
            parallel.sharded_run_batch(BatchRequest(None, [], {}, x), _failing_run, rank, world)
        except BatchInputError as exc:
            got = exc.index
        # the group is still usable: nobody was left waiting in a collective
        v = parallel.allreduce_sum(np.array([1.0]))
        np.save(os.path.join(out_dir, f"f{rank}.npy"), np.array([got, v[0]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_run_batch_row_failure_reaches_every_rank(tmp_path):
    """A row that fails on one rank raises BatchInputError(global index) on
    every rank (batch.py:196-202), and no rank hangs in the gather."""
    world = 2
    mp.start_processes(_failure_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"f{r}.npy"), [5.0, 2.0])
