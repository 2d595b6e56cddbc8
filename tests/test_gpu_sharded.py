"""GPU: the multi-GPU building blocks on one device.  Two (or four) output
tiles are computed separately through the staged C-ABI (local bound maxima ->
MAX exchange -> injected exponents), and the assembled product must be
bit-identical to the single-call emulation (fast and accurate mode)."""

import numpy as np
import pytest

from oracle import ozaki2 as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("mode,prec,R,C", [("accurate", "double", 1, 2), ("accurate", "double", 2, 2),
                                          ("accurate", "single", 2, 1), ("fast", "double", 2, 2)])
def test_tiles_assemble_bitwise(mode, prec, R, C):
    import paper_2512_08321_b200 as crt
    from paper_2512_08321_b200 import dist as d
    m, n, k = 300, 260, 500
    a = torch.from_numpy(orc.gen_matrix(m, k, 1.5, 80, prec)).cuda()
    b = torch.from_numpy(orc.gen_matrix(k, n, 1.5, 81, prec)).cuda()
    cfg = crt.EmuConfig(precision=prec, domain="complex", mode=mode)
    full = crt.emulate_gemm_complex(a, b, cfg)
    grid = d.TileGrid(R, C)
    tiles = {}
    parts = {}
    for rank in range(grid.world):
        i0, i1 = grid.rows(m, rank)
        j0, j1 = grid.cols(n, rank)
        a_loc, b_loc = a[i0:i1].contiguous(), b[:, j0:j1].contiguous()
        if mode == "fast":
            tiles[rank] = crt.run_complex(a_loc, b_loc, cfg)
        else:
            parts[rank] = (a_loc, b_loc, d.accurate_partial(a_loc, b_loc, cfg))
    if mode == "accurate":
        # the exchange: MAX over grid rows / columns (what NCCL all_reduce does)
        for rank, (_, _, p) in parts.items():
            r, c = grid.coords(rank)
            p["row_max"] = torch.stack([parts[q][2]["row_max"] for q in grid.row_members(r)]).amax(0)
            p["col_max"] = torch.stack([parts[q][2]["col_max"] for q in grid.col_members(c)]).amax(0)
        for rank, (a_loc, b_loc, p) in parts.items():
            mu, nu = d.accurate_exponents(p, cfg)
            tiles[rank] = d.tile_with_exponents(a_loc, b_loc, mu, nu, cfg)
    out = torch.empty_like(full)
    for rank, t in tiles.items():
        i0, i1 = grid.rows(m, rank)
        j0, j1 = grid.cols(n, rank)
        out[i0:i1, j0:j1] = t
    assert torch.equal(out.view(torch.float64 if prec == "double" else torch.float32),
                       full.view(torch.float64 if prec == "double" else torch.float32))
