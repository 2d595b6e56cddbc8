"""CPU, world_size 2 over gloo: the host logic of the multi-GPU path
(paper_2512_08321_b200/dist.py) — tile grid, the accurate-mode MAX exchange of
bound maxima, operand scatter and tile gather.  The per-tile GPU compute is
replaced here by the oracle / torch CPU matmul (checkers only)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_08321_b200.dist import TileGrid, TileGroups, gather_tiles, reduce_bound_maxima, \
    scatter_operands


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(fn, world, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def test_tile_grid():
    assert [(g.R, g.C) for g in map(TileGrid.for_world, (1, 2, 4, 8))] == \
        [(1, 1), (1, 2), (2, 2), (2, 4)]
    g = TileGrid.for_world(8)
    cover = np.zeros((1000, 999), int)
    for r in range(8):
        i0, i1 = g.rows(1000, r)
        j0, j1 = g.cols(999, r)
        cover[i0:i1, j0:j1] += 1
    assert np.all(cover == 1)
    assert g.row_members(1) == [4, 5, 6, 7] and g.col_members(2) == [2, 6]


def _accurate_exchange(rank, world, R, C):
    from oracle import ozaki2 as orc
    grid = TileGrid(R, C)
    groups = TileGroups(grid, rank)
    m, n, k, N = 24, 30, 40, 13
    a = orc.gen_matrix(m, k, 2.0, 70)
    b = orc.gen_matrix(k, n, 2.0, 71)
    a[5] = 0  # a dead row
    i0, i1 = grid.rows(m, rank)
    j0, j1 = grid.cols(n, rank)
    pf, pa, delta = orc.scale_thresholds(orc.pick_moduli(N).P)
    # local bound product of this tile (what crtg_accurate_partial computes)
    _, _, bound = orc.accurate_exps(orc._split(a[i0:i1]), orc._split(b[:, j0:j1]), pa, delta)
    row_max = torch.from_numpy(bound.max(axis=1).astype(np.int32))
    col_max = torch.from_numpy(bound.max(axis=0).astype(np.int32))
    reduce_bound_maxima(row_max, col_max, groups)
    _, _, full = orc.accurate_exps(orc._split(a), orc._split(b), pa, delta)
    assert np.array_equal(row_max.numpy(), full.max(axis=1)[i0:i1].astype(np.int32))
    assert np.array_equal(col_max.numpy(), full.max(axis=0)[j0:j1].astype(np.int32))
    # identical exponents to the single-process accurate scaling
    mu, nu = orc.exponents(a, b, N, "accurate")

    def fin(mx, peak, bar):
        mx = mx.astype(np.float64)
        dead = (mx <= 0) | (peak == 0)
        lb = orc.log2_up(np.where(dead, 1.0, mx)).astype(np.float64)
        g = np.floor(orc.f32_down(float(pa) - float(delta) * lb)).astype(np.int64)
        return np.clip(np.where(dead, 1023, bar + g), -1023, 1023)

    bar_mu, _, _ = orc.bound_operands(orc._split(a[i0:i1]), 1)
    bar_nu, _, _ = orc.bound_operands(orc._split(b[:, j0:j1]), 0)
    peak_a = orc._peak(orc._split(a[i0:i1]), 1)
    peak_b = orc._peak(orc._split(b[:, j0:j1]), 0)
    assert np.array_equal(fin(row_max.numpy(), peak_a, bar_mu), mu[i0:i1])
    assert np.array_equal(fin(col_max.numpy(), peak_b, bar_nu), nu[j0:j1])


@pytest.mark.parametrize("R,C", [(1, 2), (2, 1)])
def test_accurate_bound_exchange_gloo(R, C):
    _run(_accurate_exchange, 2, R, C)


def _scatter_gather(rank, world, two_level):
    grid = TileGrid.for_world(world)
    groups = TileGroups(grid, rank) if two_level else None
    m, n, k = 9, 14, 11
    rng = np.random.default_rng(3)
    a = b = None
    if rank == 0:
        a = torch.from_numpy(rng.integers(-9, 9, (m, k)) + 1j * rng.integers(-9, 9, (m, k)))
        b = torch.from_numpy(rng.integers(-9, 9, (k, n)) + 1j * rng.integers(-9, 9, (k, n)))
    a_loc, b_loc = scatter_operands(a, b, grid, rank, m, n, k, torch.complex128, "cpu",
                                    groups=groups)
    i0, i1 = grid.rows(m, rank)
    j0, j1 = grid.cols(n, rank)
    assert a_loc.shape == (i1 - i0, k) and b_loc.shape == (k, j1 - j0)
    c = gather_tiles(a_loc @ b_loc, grid, rank, m, n)
    if rank == 0:
        assert torch.equal(c, a @ b)


def test_scatter_gather_gloo():
    _run(_scatter_gather, 2, False)


def test_scatter_two_level_gloo():
    # 2 x 2 grid: root -> row / column leaders -> broadcasts over grid rows / columns
    _run(_scatter_gather, 4, True)
