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
