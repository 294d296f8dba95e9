"""The library-driven NCCL path (csrc/comm.cpp, oz2g_gemm_dist).

CPU (no GPU needed):
  * oz2g_dist_layout: for 1, 2, 4, 8 ranks the 1-D shards assemble into the
    tile blocks the way comm.cpp gathers them — the A shards of a grid row,
    in row-comm order, are its A row block; the B shards of a grid column, in
    column-comm order and interleaved by panels, are its B column block;
  * the same assembly over torch.distributed gloo, world 2 and 4: all-gather
    in row / column groups, then the oracle on each tile with the max-reduced
    clearance maxima — the gathered C equals the single-process C bit for bit.
GPU (one device, so world size 1 — NCCL refuses two ranks on one GPU): the
NCCL communicator (init, ncclCommSplit, all-gathers, MAX all-reduce) runs
inside oz2g_gemm_dist and its tile equals os_ii bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_02549_b200 import dist as pdist


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_layout_assembles_tiles(world):
    m, n = 16 * world, 8 * world
    R, C = pdist.grid_shape(world)
    lays = [pdist.layout(world, q, m, n) for q in range(world)]
    for q, t in enumerate(lays):
        assert (t["R"], t["C"], t["r"], t["c"]) == (R, C, q // C, q % C)
        tt = pdist.tile_of(q, world, m, n)
        assert (t["rows"], t["cols"]) == (tt.rows, tt.cols)
        # row comm of grid row r: ranks r*C + c, c = 0..C-1, in order of c
        rows = np.concatenate([np.arange(m)[lays[t["r"] * C + c]["a_shard"]] for c in range(C)])
        assert np.array_equal(rows, np.arange(m)[t["rows"]])
        # column comm of grid column c: ranks r*C + c, r = 0..R-1, panels in order of r
        cols = np.concatenate([np.arange(n)[lays[r * C + t["c"]]["b_shard"]] for r in range(R)])
        assert np.array_equal(cols, np.arange(n)[t["cols"]])


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


M, K, N_, NMOD = 32, 40, 16, 14


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    A = O.gen_matrix(M, K, 1.0, O.derive_seed(5, 0, 0))
    B = O.gen_matrix(K, N_, 1.0, O.derive_seed(5, 0, 1))
    lay = pdist.layout(world, rank, M, N_)
    R, C = lay["R"], lay["C"]
    rows_g, cols_g = pdist.make_groups(dist, world)
    # what the rank holds: its 1-D shards only
    a_sh = torch.from_numpy(np.ascontiguousarray(A[lay["a_shard"]]))
    b_sh = torch.from_numpy(np.ascontiguousarray(B[:, lay["b_shard"]]))
    # the gathers of comm.cpp: A in the row group, B in the column group + panel interleave
    a_parts = [torch.empty_like(a_sh) for _ in range(C)]
    dist.all_gather(a_parts, a_sh, group=rows_g[lay["r"]])
    b_parts = [torch.empty_like(b_sh) for _ in range(R)]
    dist.all_gather(b_parts, b_sh, group=cols_g[lay["c"]])
    Ab = torch.cat(a_parts, 0).numpy()
    Bb = torch.cat(b_parts, 1).numpy()
    assert np.array_equal(Ab, A[lay["rows"]]) and np.array_equal(Bb, B[:, lay["cols"]])
    tile = pdist.tile_of(rank, world, M, N_)
    local = O.os_ii(Ab, Bb, NMOD, want_cmax=True)
    rmax, cmax = pdist.reduce_maxima_host(dist, tile, rows_g, cols_g, local.inter["cmax_row"].copy(),
                                          local.inter["cmax_col"].copy())
    res = O.os_ii(Ab, Bb, NMOD, ext_cmax_row=rmax, ext_cmax_col=cmax)
    np.save(os.path.join(out_dir, f"tile{rank}.npy"), res.C)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_assembly_equals_single(tmp_path, world):
    mp.start_processes(_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True, start_method="fork")
    from oracle import oracle as O
    A = O.gen_matrix(M, K, 1.0, O.derive_seed(5, 0, 0))
    B = O.gen_matrix(K, N_, 1.0, O.derive_seed(5, 0, 1))
    full = O.os_ii(A, B, NMOD).C
    Cg = np.empty_like(full)
    for rank in range(world):
        t = pdist.tile_of(rank, world, M, N_)
        Cg[t.rows, t.cols] = np.load(tmp_path / f"tile{rank}.npy")
    assert np.array_equal(Cg.view(np.uint64), full.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("dt,overlap,m", [(torch.float64, 1, 640), (torch.float32, 1, 640), (torch.float64, 0, 640),
                                          (torch.float64, 1, 642), (torch.float64, 1, 4100)])
def test_nccl_world1(cuda, oracle, dt, overlap, m):
    """NCCL path at world size 1: with "dist_pipeline" A arrives in four row
    chunks (ncclBroadcast each, ragged last chunk for m = 642) under the
    chunked scans; without it the blocks are all-gathered first."""
    import paper_2602_02549_b200 as oz
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_port())
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("gloo", rank=0, world_size=1)
    prev = oz.get_option("dist_pipeline")
    oz.set_option("dist_pipeline", overlap)
    try:
        comm = pdist.NativeComm(dist, 1, 0)
        k, n = 300, 520
        npdt = np.float64 if dt == torch.float64 else np.float32
        A = oracle.gen_matrix(m, k, 1.0, 91, npdt)
        B = oracle.gen_matrix(k, n, 1.0, 92, npdt)
        ref = oracle.os_ii(A, B, 14).C
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        for tiles in (False, True):
            out = torch.empty((m, n), dtype=dt, device="cuda")
            comm.gemm(dA, dB, 14, m, n, out, tiles=tiles)
            bits = np.uint64 if npdt == np.float64 else np.uint32
            assert np.array_equal(out.cpu().numpy().view(bits), ref.view(bits)), tiles
        # a strided shard (lda > k) goes through the same gather
        big = torch.zeros((m, k + 7), dtype=dt, device="cuda")
        big[:, :k] = dA
        out = torch.empty((m, n), dtype=dt, device="cuda")
        comm.gemm(big[:, :k], dB, 14, m, n, out)
        assert np.array_equal(out.cpu().numpy(), ref)
        with pytest.raises(oz.DomainError):
            bad = dA.clone()
            bad[3] = 0
            comm.gemm(bad, dB, 14, m, n, out)
        comm.close()
    finally:
        oz.set_option("dist_pipeline", prev)
        if own:
            dist.destroy_process_group()
