"""CPU checks of the host side of the row-partitioned path (no GPU): slab generation and the
torchrun bootstrap, with two gloo ranks.

* every rank's host slab (aggmg_generate_*_rows) concatenates to the one-GPU generator
  matrix, for even and uneven partitions (the inputs aggmg_dist_matrix_from_host takes);
* bench.py's weak-scaling grid and rank bootstrap (unique-id broadcast over torch.distributed,
  even row partition, rank-order gather) work across two processes."""
import os
import socket

import numpy as np
import pytest

from paper_1403_1649_b200 import aggmg as M
from paper_1403_1649_b200 import dist as D


def concat(parts):
    ro = [np.zeros(1, dtype=np.int64)]
    cols, vals, base = [], [], 0
    for p in parts:
        ro.append(p.row_offsets[1:] + base)
        base += p.nnz
        cols.append(p.col_indices)
        vals.append(p.values)
    return np.concatenate(ro), np.concatenate(cols), np.concatenate(vals)


@pytest.mark.parametrize("kind,dims,grid", [("poisson", 2, (13, 9, 1)), ("poisson", 3, (7, 6, 5)),
                                            ("jump27", 3, (6, 5, 7))])
def test_host_slabs_concatenate_to_the_global_matrix(kind, dims, grid):
    nx, ny, nz = grid
    b = M.b200()
    full = (b.generate_jump27(nx, ny, nz, 1e6, 2) if kind == "jump27"
            else b.generate_poisson(dims, nx, ny, nz))
    n = full.n_rows
    for part in ([0, n], [0, n // 2, n], [0, 1, n // 3, n // 3, n]):
        slabs = [D.host_rows(kind, part[r], part[r + 1] - part[r], nx, ny, nz, dims=dims,
                             jump=1e6, block=2) for r in range(len(part) - 1)]
        for s in slabs:
            assert s.n_cols == n
        ro, ci, va = concat(slabs)
        assert np.array_equal(ro, full.row_offsets)
        assert np.array_equal(ci, full.col_indices)
        assert np.array_equal(va.view(np.uint64), full.values.view(np.uint64))


def test_host_slab_range_errors():
    with pytest.raises(M.Error, match="row range"):
        D.host_rows("poisson", 100, 50, 5, 5, 5)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q):
    import torch.distributed as tdist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    # bootstrap exactly as bench.run_dist does (a stand-in id: no GPU / NCCL here)
    obj = [bytes(range(128)) if rank == 0 else None]
    tdist.broadcast_object_list(obj, src=0)
    dims, nx, ny, nz = 3, 6, 5, 4
    gx, gy, gz = bench.world_grid_dims(dims, nx, ny, nz, world)
    n = gx * gy * gz
    r0, r1 = n * rank // world, n * (rank + 1) // world
    slab = D.host_rows("poisson", r0, r1 - r0, gx, gy, gz, dims=3)
    gathered = [None] * world
    tdist.all_gather_object(gathered, (r0, r1, slab.row_offsets, slab.col_indices, slab.values,
                                       obj[0]))
    tdist.destroy_process_group()
    if rank == 0:
        q.put((gx, gy, gz, gathered))


def test_two_gloo_ranks_bootstrap_and_slabs():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gx, gy, gz, gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert (gx, gy, gz) == (12, 5, 4)  # weak scaling: x doubled first
    assert gathered[0][0] == 0 and gathered[0][1] == gathered[1][0] and gathered[1][1] == 12 * 5 * 4
    assert gathered[1][5] == bytes(range(128))  # the id rank 0 broadcast
    full = M.b200().generate_poisson(3, gx, gy, gz)
    parts = [M.SparseMatrix(g[1] - g[0], full.n_cols, g[2], g[3], g[4]) for g in gathered]
    ro, ci, va = concat(parts)
    assert np.array_equal(ro, full.row_offsets)
    assert np.array_equal(ci, full.col_indices)
    assert np.array_equal(va, full.values)
