"""The per-process multi-GPU path of bench.py --gpus N on real kernels:
dist.tile_of / make_groups / max_reduce_hook driving oz2g_gemm's reduce hook
from inside the device pipeline.  NCCL cannot place two ranks on one GPU, so
the ranks here share cuda:0 and reduce with gloo (which all-reduces CUDA
tensors through the host); the hook, the groups, the tiles and the device
kernels are exactly the ones the NCCL run uses.  The gathered C tiles must
equal the single-process result bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_02549_b200 import dist as pdist

M, K, N_, NMOD = 300, 96, 260, 14


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, phi, out_dir, shape=(M, K, N_), host=False):
    import torch
    import paper_2602_02549_b200 as oz
    from oracle import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    m, k, n = shape
    A = O.gen_matrix(m, k, phi, O.derive_seed(5, 0, 0))
    B = O.gen_matrix(k, n, phi, O.derive_seed(5, 0, 1))
    tile = pdist.tile_of(rank, world, m, n)
    rows, cols = pdist.make_groups(dist, world)
    hook = pdist.max_reduce_hook(dist, tile, rows, cols, dev)
    Ah = np.ascontiguousarray(A[tile.rows])
    Bh = np.ascontiguousarray(B[:, tile.cols])
    if host:  # host arrays: the pipelined upload path, exponents after the all-reduce
        C = oz.os_ii(Ah, Bh, NMOD, reduce_maxima=hook).C
    else:
        C = oz.os_ii(torch.from_numpy(Ah).to(dev), torch.from_numpy(Bh).to(dev), NMOD, reduce_maxima=hook).C.cpu().numpy()
    np.save(os.path.join(out_dir, f"tile{rank}.npy"), C)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,phi", [(2, 1.0), (4, 2.0)])
def test_hook_tiles_equal_single(cuda, oracle, tmp_path, world, phi):
    mp.start_processes(_worker, args=(world, _port(), phi, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    A = oracle.gen_matrix(M, K, phi, oracle.derive_seed(5, 0, 0))
    B = oracle.gen_matrix(K, N_, phi, oracle.derive_seed(5, 0, 1))
    full = oracle.os_ii(A, B, NMOD).C
    Cg = np.empty_like(full)
    for rank in range(world):
        t = pdist.tile_of(rank, world, M, N_)
        Cg[t.rows, t.cols] = np.load(tmp_path / f"tile{rank}.npy")
    assert np.array_equal(Cg.view(np.uint64), full.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2])
def test_hook_host_pipeline(cuda, oracle, tmp_path, world):
    """Host arrays with a reduce hook: tiles of >= 2048 rows upload in chunks
    that overlap the scans and clearance products, then the maxima are
    all-reduced before the exponents — same C as the single process."""
    shape = (4608, 64, 600)
    mp.start_processes(_worker, args=(world, _port(), 1.0, str(tmp_path), shape, True), nprocs=world, join=True,
                       start_method="spawn")
    m, k, n = shape
    A = oracle.gen_matrix(m, k, 1.0, oracle.derive_seed(5, 0, 0))
    B = oracle.gen_matrix(k, n, 1.0, oracle.derive_seed(5, 0, 1))
    full = oracle.os_ii(A, B, NMOD).C
    Cg = np.empty_like(full)
    for rank in range(world):
        t = pdist.tile_of(rank, world, m, n)
        Cg[t.rows, t.cols] = np.load(tmp_path / f"tile{rank}.npy")
    assert np.array_equal(Cg.view(np.uint64), full.view(np.uint64))
