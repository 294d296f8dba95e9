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
