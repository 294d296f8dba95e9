"""Multi-GPU decomposition of one emulated GEMM.

C is tiled 2-D over the ranks of one node (R x Cc grid: 2 -> 2x1, 4 -> 2x2,
8 -> 2x4).  Rank (r, c) holds the row block r of A (all of k) and the column
block c of B (all of k) and produces the C tile (r, c); no output reduction is
needed.  The only exchange is the max-reduction of the clearance-product
maxima: mu_i needs the maximum over ALL columns of row i of C̄ (scaling.hpp:
175-183), nu_j over ALL rows (scaling.hpp:184-192).  Each rank computes the
maxima of its tile, then all-reduces (MAX) the row maxima over the ranks of
its grid row and the column maxima over the ranks of its grid column — the
callback the C ABI exposes between the clearance product and the scaling
exponents (oz2g.h, oz2g_reduce_maxima_fn).  With that step the tiled result is
bit-identical to the single-GPU (and the reference's) result.
"""
from __future__ import annotations

from dataclasses import dataclass


def grid_shape(world: int) -> tuple[int, int]:
    return {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (2, 4)}.get(world, (world, 1))


@dataclass
class Tile:
    rank: int
    r: int
    c: int
    R: int
    C: int
    rows: slice
    cols: slice


def tile_of(rank: int, world: int, m: int, n: int) -> Tile:
    R, Cc = grid_shape(world)
    r, c = rank // Cc, rank % Cc
    mb, nb = -(-m // R), -(-n // Cc)
    return Tile(rank, r, c, R, Cc, slice(min(m, r * mb), min(m, (r + 1) * mb)),
                slice(min(n, c * nb), min(n, (c + 1) * nb)))


def make_groups(dist, world: int):
    """Row / column process groups; every rank must call this (same order)."""
    R, Cc = grid_shape(world)
    rows = [dist.new_group([rr * Cc + cc for cc in range(Cc)]) for rr in range(R)]
    cols = [dist.new_group([rr * Cc + cc for rr in range(R)]) for cc in range(Cc)]
    return rows, cols


class _DevArray:
    """__cuda_array_interface__ view of a raw int32 device buffer (no copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<i4", "data": (ptr, False),
                                         "version": 3, "strides": None}


def max_reduce_hook(dist, tile: Tile, row_groups, col_groups, device):
    """The oz2g_reduce_maxima_fn for torch.distributed (NCCL on CUDA pointers)."""
    import torch

    def hook(row_ptr, m, col_ptr, n, stream):
        if m and tile.C > 1:
            dist.all_reduce(torch.as_tensor(_DevArray(row_ptr, m), device=device), op=dist.ReduceOp.MAX,
                            group=row_groups[tile.r])
        if n and tile.R > 1:
            dist.all_reduce(torch.as_tensor(_DevArray(col_ptr, n), device=device), op=dist.ReduceOp.MAX,
                            group=col_groups[tile.c])

    return hook


def reduce_maxima_host(dist, tile: Tile, row_groups, col_groups, cmax_row, cmax_col):
    """Same reduction on host int32 arrays (gloo); used by the CPU tests."""
    import torch
    tr = torch.from_numpy(cmax_row)
    tc = torch.from_numpy(cmax_col)
    if tile.C > 1:
        dist.all_reduce(tr, op=dist.ReduceOp.MAX, group=row_groups[tile.r])
    if tile.R > 1:
        dist.all_reduce(tc, op=dist.ReduceOp.MAX, group=col_groups[tile.c])
    return tr.numpy(), tc.numpy()


# ---------------------------------------------------------------------------
# Native path: NCCL driven by the library (csrc/comm.cpp, oz2g_gemm_dist).
# ---------------------------------------------------------------------------
def layout(world: int, rank: int, m: int, n: int) -> dict:
    """The tile and 1-D shard ranges of `rank` (oz2g_dist_layout): A rows
    [q m/P, (q+1) m/P) and the B columns of shard c*R + r are what the rank
    holds before a call; its C tile is (rows, cols)."""
    import ctypes as C

    from . import _lib
    t = _lib.DistTile()
    if _lib.load().oz2g_dist_layout(int(world), int(rank), int(m), int(n), C.byref(t)) != 0:
        raise ValueError("oz2g_dist_layout: bad arguments")
    return {"R": t.R, "C": t.C, "r": t.r, "c": t.c,
            "rows": slice(t.row0, t.row0 + t.rows), "cols": slice(t.col0, t.col0 + t.cols),
            "a_shard": slice(t.a_shard_row0, t.a_shard_row0 + t.a_shard_rows),
            "b_shard": slice(t.b_shard_col0, t.b_shard_col0 + t.b_shard_cols)}


class NativeComm:
    """The library's communicator (world + row / column NCCL comms).  Every
    rank constructs it collectively; the NCCL unique id travels over the
    given torch.distributed process group (any backend)."""

    def __init__(self, dist, world: int, rank: int, group=None):
        import ctypes as C

        from . import _lib
        L = _lib.load()
        self._L = L
        buf = (C.c_ubyte * 128)()
        if rank == 0 and L.oz2g_comm_unique_id(buf) != 0:
            raise RuntimeError(L.oz2g_comm_last_error().decode())
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0, group=group)
        idb = (C.c_ubyte * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        if L.oz2g_comm_init(idb, int(world), int(rank), C.byref(h)) != 0:
            raise RuntimeError(L.oz2g_comm_last_error().decode())
        self.handle = h
        self.world, self.rank = world, rank

    def gemm(self, A, B, n_moduli: int, m: int, n: int, out, tiles: bool = False, timing: bool = False):
        """This rank's C tile of os_ii(A_global, B_global, n_moduli): A, B are
        the rank's shards (default) or its row / column blocks (tiles=True),
        CUDA tensors; `out` the tile (rows x cols, row-major)."""
        import ctypes as C

        import torch

        from . import _lib
        from .emulate import _EXC, CudaError
        prec = _lib.OZ2G_FP64 if A.dtype == torch.float64 else _lib.OZ2G_FP32
        k = A.shape[1]
        flags = (_lib.OZ2G_DIST_TILES if tiles else _lib.OZ2G_DIST_SHARDS) | (_lib.OZ2G_TIMING if timing else 0)
        diag = _lib.Diag()
        stream = torch.cuda.current_stream(A.device).cuda_stream
        rc = self._L.oz2g_gemm_dist(prec, int(m), int(n), int(k), A.data_ptr(), A.stride(0), B.data_ptr(),
                                    B.stride(0), out.data_ptr(), out.stride(0), int(n_moduli), flags,
                                    C.c_void_p(int(stream)), self.handle, C.byref(diag))
        if rc != 0:
            raise _EXC.get(rc, CudaError)(self._L.oz2g_comm_last_error().decode())
        return diag

    def close(self):
        if self.handle:
            self._L.oz2g_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass
