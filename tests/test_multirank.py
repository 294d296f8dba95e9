"""Multi-rank decomposition on CPU (gloo, world size 2 and 4).

Every rank runs the oracle on its C tile with its A row block and B column
block, exchanges the clearance maxima through the same grid / group / MAX
reduction code the GPU path uses (paper_2602_02549_b200.dist), and finishes
the emulation with the reduced maxima.  The gathered tiles must equal the
single-process result bit for bit — the property the 8-GPU run relies on.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_02549_b200 import dist as pdist

M, K, N_, NMOD = 24, 40, 18, 14


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, phi, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    A = O.gen_matrix(M, K, phi, O.derive_seed(3, 0, 0))
    B = O.gen_matrix(K, N_, phi, O.derive_seed(3, 0, 1))
    tile = pdist.tile_of(rank, world, M, N_)
    rows, cols = pdist.make_groups(dist, world)
    Ab, Bb = A[tile.rows], B[:, tile.cols]
    local = O.os_ii(Ab, Bb, NMOD, want_cmax=True)
    rmax, cmax = pdist.reduce_maxima_host(dist, tile, rows, cols, local.inter["cmax_row"].copy(),
                                          local.inter["cmax_col"].copy())
    res = O.os_ii(Ab, Bb, NMOD, ext_cmax_row=rmax, ext_cmax_col=cmax)
    np.save(os.path.join(out_dir, f"tile{rank}.npy"), res.C)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,phi", [(2, 0.0), (2, 2.0), (4, 1.0)])
def test_tiled_equals_single(tmp_path, world, phi):
    mp.start_processes(_worker, args=(world, _port(), phi, str(tmp_path)), nprocs=world, join=True,
                       start_method="fork")
    from oracle import oracle as O
    A = O.gen_matrix(M, K, phi, O.derive_seed(3, 0, 0))
    B = O.gen_matrix(K, N_, phi, O.derive_seed(3, 0, 1))
    full = O.os_ii(A, B, NMOD).C
    Cg = np.empty_like(full)
    for rank in range(world):
        t = pdist.tile_of(rank, world, M, N_)
        Cg[t.rows, t.cols] = np.load(tmp_path / f"tile{rank}.npy")
    assert Cg.tobytes() == full.tobytes()


def test_without_exchange_differs():
    """Sanity: skipping the exchange changes the scaling (it is not a no-op)."""
    from oracle import oracle as O
    A = O.gen_matrix(M, K, 2.0, O.derive_seed(3, 0, 0))
    B = O.gen_matrix(K, N_, 2.0, O.derive_seed(3, 0, 1))
    full = O.os_ii(A, B, NMOD, keep_intermediates=True)
    t = pdist.tile_of(0, 2, M, N_)
    part = O.os_ii(A[t.rows], B[:, t.cols], NMOD, keep_intermediates=True)
    assert not np.array_equal(part.inter["nu"], full.inter["nu"])


def test_grid_shapes():
    assert pdist.grid_shape(8) == (2, 4) and pdist.grid_shape(4) == (2, 2) and pdist.grid_shape(2) == (2, 1)
    tiles = [pdist.tile_of(r, 8, 100, 37) for r in range(8)]
    cover = np.zeros((100, 37), dtype=int)
    for t in tiles:
        cover[t.rows, t.cols] += 1
    assert (cover == 1).all()
