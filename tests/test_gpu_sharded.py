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


# ----------------------------------------------- the distributed driver, end to end
def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _dist_entry(rank, world, port, backend, mode, shape, q):
    import os

    import torch.distributed as dist

    import paper_2512_08321_b200 as crt
    from paper_2512_08321_b200 import dist as d
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", rank % ndev)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, k = shape
        a = b = None
        if rank == 0:
            a = torch.from_numpy(orc.gen_matrix(m, k, 2.0, 90)).to(dev)
            b = torch.from_numpy(orc.gen_matrix(k, n, 2.0, 91)).to(dev)
        cfg = crt.EmuConfig(domain="complex", mode=mode, num_moduli=14)
        grid = d.TileGrid.for_world(world)
        emu = d.ShardedEmulator(cfg, grid, rank)
        groups = emu.groups or (d.TileGroups(grid, rank) if world > 2 else None)
        a_loc, b_loc = d.scatter_operands(a, b, grid, rank, m, n, k, torch.complex128, dev,
                                          groups=groups)
        c_loc = emu.tile(a_loc, b_loc)
        c = d.gather_tiles(c_loc, grid, rank, m, n)
        if rank == 0:
            full = crt.emulate_gemm_complex(a, b, cfg)
            q.put(bool(torch.equal(c.view(torch.float64), full.view(torch.float64))))
    finally:
        dist.destroy_process_group()


def _spawn(world, backend, mode, shape):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_dist_entry, args=(world, _free_port(), backend, mode, shape, q),
                       nprocs=world, join=True, start_method="spawn")
    return q.get(timeout=10)


@pytest.mark.parametrize("mode", ["fast", "accurate"])
def test_sharded_product_nccl_single_rank(mode):
    """The NCCL code path on the device (world size 1): scatter, tile (accurate:
    the MAX all-reduce over NCCL), gather -> bitwise the single-call product."""
    assert _spawn(1, "nccl", mode, (600, 520, 700))


@pytest.mark.parametrize("mode", ["fast", "accurate"])
def test_sharded_product_two_ranks_one_gpu(mode):
    """Two ranks sharing one GPU over gloo (device tensors staged through the
    host): the real multi-rank exchange -- scatter, MAX all-reduce of the bound
    maxima, grouped gather -- bitwise the single-call product."""
    assert _spawn(2, "gloo", mode, (600, 520, 700))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs (NCCL over NVLink)")
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_product_nccl_multi_gpu(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    assert _spawn(world, "nccl", "accurate", (1100, 900, 800))
