"""Multi-GPU emulated ZGEMM/CGEMM by output tiles of C.

One process per GPU (torch.distributed, NCCL over NVLink on the box; gloo in
the CPU tests).  World size W is laid out as an R x C grid of output tiles
(1x1, 1x2, 2x2, 2x4, ...): rank (r, c) holds the A row-block A[I_r, :] and the
B column-block B[:, J_c] and computes C[I_r, J_c].

* Fast mode needs no collective on the data path: mu_i depends only on row i of
  A over the full k, nu_j only on column j of B (reference scaling.py:174-213),
  so a tile is bit-identical to the same block of the single-GPU product.
* Accurate mode has exactly one exchange: mu_i = f(max_j bound_ij) is global in
  j (scaling.py:260-271).  Each rank computes the bound-GEMM maxima of its tile
  (`crtg_accurate_partial`), all-reduces the row maxima (MAX, int32) over the
  ranks of its grid row and the column maxima over its grid column, then every
  rank derives identical exponents (`crtg_accurate_exponents`) and runs the
  pipeline with them (`crtg_gemm_complex_exps`).
* Inputs/outputs move with point-to-point NCCL send/recv from/to a root rank
  (`scatter_operands`, `gather_tiles`); benchmarks time compute with operands
  already resident, as the driver's weak-scaling contract asks.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native as nat
from .config import EmuConfig
from .errors import DomainError
from .moduli import device_constants


@dataclass(frozen=True)
class TileGrid:
    """R x C grid of output tiles over `world` ranks, rank = r * C + c."""

    R: int
    C: int

    @classmethod
    def for_world(cls, world: int) -> "TileGrid":
        if world < 1:
            raise ValueError("world size must be positive")
        r = 1 << (int(math.log2(world)) // 2)
        while world % r:
            r //= 2
        return cls(r, world // r)

    @property
    def world(self) -> int:
        return self.R * self.C

    def coords(self, rank: int):
        return divmod(rank, self.C)

    @staticmethod
    def split(extent: int, parts: int, idx: int):
        """Balanced contiguous split: part idx of [0, extent)."""
        base, rem = divmod(extent, parts)
        lo = idx * base + min(idx, rem)
        return lo, lo + base + (1 if idx < rem else 0)

    def rows(self, m: int, rank: int):
        return self.split(m, self.R, self.coords(rank)[0])

    def cols(self, n: int, rank: int):
        return self.split(n, self.C, self.coords(rank)[1])

    def row_members(self, r: int):
        return [r * self.C + c for c in range(self.C)]

    def col_members(self, c: int):
        return [r * self.C + c for r in range(self.R)]


class TileGroups:
    """Process groups of every grid row and column (created collectively)."""

    def __init__(self, grid: TileGrid, rank: int):
        self.grid = grid
        self.rank = rank
        r, c = grid.coords(rank)
        self.row_group = None
        self.col_group = None
        # new_group must be called by every rank for every group, in order
        for rr in range(grid.R):
            g = dist.new_group(grid.row_members(rr))
            if rr == r:
                self.row_group = g
        for cc in range(grid.C):
            g = dist.new_group(grid.col_members(cc))
            if cc == c:
                self.col_group = g


def reduce_bound_maxima(row_max: torch.Tensor, col_max: torch.Tensor,
                        groups: TileGroups) -> None:
    """In place: MAX-all-reduce the tile's bound-product row maxima over its grid
    row and the column maxima over its grid column (the accurate-mode exchange)."""
    if groups.grid.C > 1:
        dist.all_reduce(row_max, op=dist.ReduceOp.MAX, group=groups.row_group)
    if groups.grid.R > 1:
        dist.all_reduce(col_max, op=dist.ReduceOp.MAX, group=groups.col_group)


def _staged() -> bool:
    """gloo moves CPU tensors only: device tensors are staged through the host
    (CPU tests / several ranks sharing one GPU); NCCL sends device memory."""
    return dist.get_backend() == "gloo"


def _send(t: torch.Tensor, dst: int) -> None:
    dist.send(t.cpu() if (_staged() and t.is_cuda) else t, dst)


def _isend_op(t: torch.Tensor, dst: int):
    return dist.P2POp(dist.isend, t.cpu() if (_staged() and t.is_cuda) else t, dst)


def _recv(t: torch.Tensor, src: int) -> None:
    if _staged() and t.is_cuda:
        buf = torch.empty(t.shape, dtype=t.dtype)
        dist.recv(buf, src)
        t.copy_(buf)
    else:
        dist.recv(t, src)


def scatter_operands(a, b, grid: TileGrid, rank: int, m: int, n: int, k: int,
                     dtype, device, root: int = 0, groups: "TileGroups | None" = None):
    """Root distributes A[I_r,:] and B[:,J_c]; returns the local blocks (contiguous,
    on `device`).

    With `groups` (R x C > 2 ranks): two levels, so the root sends each block
    ONCE — A's row-block r goes to the row leader (r, 0) and B's column-block c
    to the column leader (0, c), which broadcast it over their grid row / column
    (NVSwitch: every rank has full bandwidth to every peer, so the broadcasts of
    different groups run side by side).  Root egress ~ |A| + |B| instead of
    R*C*(|A|/R + |B|/C).  Without groups: one point-to-point send per rank."""
    i0, i1 = grid.rows(m, rank)
    j0, j1 = grid.cols(n, rank)
    r_me, c_me = grid.coords(rank)
    if groups is None or grid.world <= 2:
        if rank == root:
            ops = []
            for dst in range(grid.world):
                di0, di1 = grid.rows(m, dst)
                dj0, dj1 = grid.cols(n, dst)
                ablk = a[di0:di1].contiguous().to(device)
                bblk = b[:, dj0:dj1].contiguous().to(device)
                if dst == root:
                    a_loc, b_loc = ablk, bblk
                else:
                    ops += [_isend_op(ablk, dst), _isend_op(bblk, dst)]
            _batched(ops)  # all peers' blocks leave the root concurrently
            return a_loc, b_loc
        a_loc = torch.empty((i1 - i0, k), dtype=dtype, device=device)
        b_loc = torch.empty((k, j1 - j0), dtype=dtype, device=device)
        _recv(a_loc, root)
        _recv(b_loc, root)
        return a_loc, b_loc
    a_lead = grid.row_members(r_me)[0]   # (r, 0)
    b_lead = grid.col_members(c_me)[0]   # (0, c)
    a_loc = b_loc = None
    # level 1: root -> leaders (one block each)
    if rank == root:
        ops = []
        for r in range(grid.R):
            di0, di1 = grid.rows(m, grid.row_members(r)[0])
            blk = a[di0:di1].contiguous().to(device)
            if grid.row_members(r)[0] == root:
                a_loc = blk
            else:
                ops.append(_isend_op(blk, grid.row_members(r)[0]))
        for c in range(grid.C):
            dj0, dj1 = grid.cols(n, grid.col_members(c)[0])
            blk = b[:, dj0:dj1].contiguous().to(device)
            if grid.col_members(c)[0] == root:
                b_loc = blk
            else:
                ops.append(_isend_op(blk, grid.col_members(c)[0]))
        _batched(ops)
    if a_loc is None:
        a_loc = torch.empty((i1 - i0, k), dtype=dtype, device=device)
        if rank == a_lead:
            _recv(a_loc, root)
    if b_loc is None:
        b_loc = torch.empty((k, j1 - j0), dtype=dtype, device=device)
        if rank == b_lead:
            _recv(b_loc, root)
    # level 2: leaders broadcast over their grid row / column
    if grid.C > 1:
        _bcast(a_loc, a_lead, groups.row_group)
    if grid.R > 1:
        _bcast(b_loc, b_lead, groups.col_group)
    return a_loc, b_loc


def _bcast(t: torch.Tensor, src: int, group) -> None:
    if _staged() and t.is_cuda:
        buf = t.cpu()
        dist.broadcast(buf, src, group=group)
        t.copy_(buf)
    else:
        dist.broadcast(t, src, group=group)


def _batched(ops) -> None:
    """Post point-to-point ops together (one NCCL group: the transfers to / from
    different peers run concurrently over NVSwitch) and wait for all of them."""
    if not ops:
        return
    for w in dist.batch_isend_irecv(ops):
        w.wait()


def gather_tiles(c_loc: torch.Tensor, grid: TileGrid, rank: int, m: int, n: int,
                 root: int = 0):
    """Every rank sends its C tile to root; root posts all receives at once
    (grouped) and returns the assembled C."""
    if rank != root:
        _send(c_loc.contiguous(), root)
        return None
    out = torch.empty((m, n), dtype=c_loc.dtype, device=c_loc.device)
    staged = _staged() and c_loc.is_cuda
    ops, bufs = [], []
    for src in range(grid.world):
        i0, i1 = grid.rows(m, src)
        j0, j1 = grid.cols(n, src)
        if src == root:
            out[i0:i1, j0:j1] = c_loc
            continue
        buf = torch.empty((i1 - i0, j1 - j0), dtype=c_loc.dtype,
                          device="cpu" if staged else c_loc.device)
        ops.append(dist.P2POp(dist.irecv, buf, src))
        bufs.append(((i0, i1, j0, j1), buf))
    _batched(ops)
    for (i0, i1, j0, j1), buf in bufs:
        out[i0:i1, j0:j1].copy_(buf)
    return out


def _prec(cfg: EmuConfig, dtype) -> int:
    p = nat.SINGLE if cfg.precision == "single" else nat.DOUBLE
    return p | (16 if dtype == torch.complex64 else 0)


def accurate_partial(a_loc: torch.Tensor, b_loc: torch.Tensor, cfg: EmuConfig) -> dict:
    """Local half of accurate scaling for one tile (crtg_accurate_partial):
    bound-product row/column maxima plus the row/column-local bars and absmax."""
    dev = a_loc.device
    m, k = a_loc.shape
    n = b_loc.shape[1]
    nmod = cfg.resolved_moduli
    lib = nat.load()
    prec = _prec(cfg, a_loc.dtype)
    ws = torch.empty(lib.crtg_workspace_size(prec, nat.ACCURATE, m, n, k, nmod, n),
                     dtype=torch.uint8, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    out = dict(row_max=torch.empty(m, **i32), col_max=torch.empty(n, **i32),
               bar_mu=torch.empty(m, **i32), bar_nu=torch.empty(n, **i32),
               row_abs=torch.empty(m, dtype=torch.float64, device=dev),
               col_abs=torch.empty(n, dtype=torch.float64, device=dev),
               diag=torch.zeros(nat.DIAG_LEN, dtype=torch.int64, device=dev))
    nat.call("crtg_accurate_partial", prec, m, n, k, a_loc.data_ptr(), a_loc.stride(0),
             b_loc.data_ptr(), b_loc.stride(0), ctypes.byref(device_constants(nmod)),
             ws.data_ptr(), ws.numel(), out["row_max"].data_ptr(), out["col_max"].data_ptr(),
             out["bar_mu"].data_ptr(), out["bar_nu"].data_ptr(), out["row_abs"].data_ptr(),
             out["col_abs"].data_ptr(), out["diag"].data_ptr(),
             torch.cuda.current_stream(dev).cuda_stream)
    return out


def accurate_exponents(part: dict, cfg: EmuConfig):
    """Exponents from the (reduced) maxima of `accurate_partial` (crtg_accurate_exponents)."""
    dev = part["row_max"].device
    consts = device_constants(cfg.resolved_moduli)
    stream = torch.cuda.current_stream(dev).cuda_stream
    mu = torch.empty_like(part["row_max"])
    nu = torch.empty_like(part["col_max"])
    diag = part["diag"]
    nat.call("crtg_accurate_exponents", mu.numel(), part["row_max"].data_ptr(),
             part["row_abs"].data_ptr(), part["bar_mu"].data_ptr(), ctypes.byref(consts),
             mu.data_ptr(), diag.data_ptr() + 8 * nat.DIAG_CLAMPED_MU, stream)
    nat.call("crtg_accurate_exponents", nu.numel(), part["col_max"].data_ptr(),
             part["col_abs"].data_ptr(), part["bar_nu"].data_ptr(), ctypes.byref(consts),
             nu.data_ptr(), diag.data_ptr() + 8 * nat.DIAG_CLAMPED_NU, stream)
    d = diag.cpu().tolist()
    if d[2] or d[3]:
        raise DomainError("matrix entries must be finite")
    return mu, nu


def tile_with_exponents(a_loc, b_loc, mu, nu, cfg: EmuConfig, sync_check: bool = True):
    """C tile from injected exponents (crtg_gemm_complex_exps)."""
    dev = a_loc.device
    m, k = a_loc.shape
    n = b_loc.shape[1]
    nmod = cfg.resolved_moduli
    lib = nat.load()
    prec = _prec(cfg, a_loc.dtype)
    ws = torch.empty(lib.crtg_workspace_size(prec, nat.FAST, m, n, k, nmod, cfg.n_block),
                     dtype=torch.uint8, device=dev)
    odt = torch.complex64 if cfg.precision == "single" else torch.complex128
    out = torch.empty((m, n), dtype=odt, device=dev)
    diag = torch.zeros(nat.DIAG_LEN, dtype=torch.int64, device=dev)
    nat.call("crtg_gemm_complex_exps", prec, m, n, k, a_loc.data_ptr(), a_loc.stride(0),
             b_loc.data_ptr(), b_loc.stride(0), out.data_ptr(), out.stride(0),
             ctypes.byref(device_constants(nmod)), cfg.n_block, mu.data_ptr(), nu.data_ptr(),
             ws.data_ptr(), ws.numel(), diag.data_ptr(), 1 if sync_check else 0,
             torch.cuda.current_stream(dev).cuda_stream)
    return out


class ShardedEmulator:
    """Computes this rank's tile C[I_r, J_c] of an emulated complex product."""

    def __init__(self, cfg: EmuConfig, grid: TileGrid | None = None, rank: int | None = None):
        self.cfg = cfg
        self.rank = dist.get_rank() if rank is None else rank
        self.grid = grid or TileGrid.for_world(dist.get_world_size())
        self.groups = TileGroups(self.grid, self.rank) if cfg.mode == "accurate" else None

    def tile(self, a_loc: torch.Tensor, b_loc: torch.Tensor, sync_check: bool = True):
        from .emulate import run_complex
        if a_loc.dtype != b_loc.dtype:
            a_loc, b_loc = a_loc.to(torch.complex128), b_loc.to(torch.complex128)
        if self.cfg.mode == "fast":
            return run_complex(a_loc, b_loc, self.cfg, sync_check=sync_check)
        part = accurate_partial(a_loc, b_loc, self.cfg)
        reduce_bound_maxima(part["row_max"], part["col_max"], self.groups)
        mu, nu = accurate_exponents(part, self.cfg)
        return tile_with_exponents(a_loc, b_loc, mu, nu, self.cfg, sync_check)
