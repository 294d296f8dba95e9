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


def _worker(rank, world, port, phi, out_dir):
    import torch
    import paper_2602_02549_b200 as oz
    from oracle import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    A = O.gen_matrix(M, K, phi, O.derive_seed(5, 0, 0))
    B = O.gen_matrix(K, N_, phi, O.derive_seed(5, 0, 1))
    tile = pdist.tile_of(rank, world, M, N_)
    rows, cols = pdist.make_groups(dist, world)
    hook = pdist.max_reduce_hook(dist, tile, rows, cols, dev)
    Ab = torch.from_numpy(np.ascontiguousarray(A[tile.rows])).to(dev)
    Bb = torch.from_numpy(np.ascontiguousarray(B[:, tile.cols])).to(dev)
    C = oz.os_ii(Ab, Bb, NMOD, reduce_maxima=hook).C
    np.save(os.path.join(out_dir, f"tile{rank}.npy"), C.cpu().numpy())
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
