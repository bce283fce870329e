"""Snapshots of device slabs in the reference's formats (pkg/src/expmhd/snapshot.py).

Binary ``.mhd25``: 96-byte little-endian header, then the state cell-major
``(nx, ny, 8)``.  The field-major -> cell-major transpose runs on the GPU
(``emhd_cells_pack``); because x is the outermost axis of the cell-major block, every x-slab
owns ONE contiguous byte range of the file (offset ``96 + 64 * x_offset * ny``), so slab ranks
write and read their own rows in parallel with no gather.  Files are byte-identical to the
reference writer's (tests/golden/snapshot_recon16x12.mhd25).

``write_snapshot_csv`` is the reference's small-grid text twin: the state is copied to the
host and formatted exactly as the reference does (repr of Python floats).
"""

import os
import struct

import numpy as np
import torch

from . import _native as N
from . import device as D
from .mhd import NVARS, Grid2D, MhdParams, _diag_ctx

MAGIC = b"MHD25\x00"
VERSION = 1
_HEADER = struct.Struct("<6sHII4dd4d8x")      # snapshot.py:33
HEADER_SIZE = _HEADER.size

class SnapshotFormatError(ValueError):
    """Malformed snapshot file (snapshot.py:39-40)."""


def _header(grid, time, params):
    return _HEADER.pack(MAGIC, VERSION, grid.nx, grid.ny, grid.x_lo, grid.x_hi, grid.y_lo,
                        grid.y_hi, float(time), params.gamma, params.mu, params.eta, params.kappa)


def _shape_check(U, grid, nx_local):
    shape = tuple(int(s) for s in U.shape)
    if shape != (NVARS, nx_local, grid.ny):
        raise ValueError(f"state shape {shape} does not match grid "
                         f"({NVARS}, {grid.nx}, {grid.ny})")


def _bc_for(layout):
    from .mhd import BoundaryPolicy
    bx = "periodic" if layout is None else ("periodic" if layout.bc_lo == "external" else layout.bc_lo)
    return BoundaryPolicy(bx, "periodic")


def write_snapshot(path, U, grid, time, params, layout=None, comm=None):
    """Write a binary field snapshot (snapshot.py:43-57).

    ``U``: the (8, nx, ny) state, or with ``layout`` this rank's (8, nx_local, ny) slab, on
    the device (or host, copied up).  Every rank of the layout calls this; rank 0 writes the
    header and sizes the file, each rank then writes its own cell-major rows.
    """
    f = _diag_ctx(grid, _bc_for(layout), layout, comm)
    L = f.layout
    if not isinstance(U, torch.Tensor):
        U = np.asarray(U, dtype=float)
    _shape_check(U, grid, L.nx_local)
    u = D.to_device(U).reshape(-1)
    ncell = L.nx_local * grid.ny
    cells = torch.empty(ncell * NVARS, dtype=D.F64, device=D.device())
    N.check(f.ctx.lib.emhd_cells_pack(f.ctx.sync_stream(), D.ptr(u), ncell, D.ptr(cells)), "cells_pack")
    host = torch.empty(cells.numel(), dtype=D.F64, pin_memory=True)
    host.copy_(cells, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    body = host.numpy().astype("<f8", copy=False).tobytes()
    size = HEADER_SIZE + NVARS * 8 * grid.nx * grid.ny
    if L.rank == 0:
        with open(path, "wb") as fh:
            fh.write(_header(grid, time, params))
            fh.truncate(size)
    f.comm.barrier()
    fd = os.open(path, os.O_WRONLY)
    try:
        os.pwrite(fd, body, HEADER_SIZE + NVARS * 8 * L.x_offset * grid.ny)
    finally:
        os.close(fd)
    f.comm.barrier()


def _parse_header(path, raw):
    """Header fields of a .mhd25 file, validated with the reference's messages (:62-76)."""
    if len(raw) < HEADER_SIZE:
        raise SnapshotFormatError(f"{path}: truncated header")
    fields = _HEADER.unpack(raw[:HEADER_SIZE])
    if fields[0] != MAGIC:
        raise SnapshotFormatError(f"{path}: bad magic {fields[0]!r}")
    if fields[1] != VERSION:
        raise SnapshotFormatError(f"{path}: unsupported version {fields[1]}")
    nx, ny = fields[2], fields[3]
    grid = Grid2D(nx, ny, *fields[4:8])
    gamma, mu, eta, kappa = fields[9:13]
    return grid, fields[8], MhdParams(mu=mu, eta=eta, kappa=kappa, gamma=gamma)


def read_snapshot(path, layout=None, comm=None):
    """Read a binary snapshot (snapshot.py:60-80); returns (U, grid, time, params).

    U is a device tensor (8, nx, ny), or with ``layout`` this rank's (8, nx_local, ny) rows,
    read straight from the rank's byte range and transposed back on the GPU.
    """
    with open(path, "rb") as fh:
        grid, time, params = _parse_header(path, fh.read(HEADER_SIZE))
        values = (os.fstat(fh.fileno()).st_size - HEADER_SIZE) // 8
        if values * 8 + HEADER_SIZE != os.fstat(fh.fileno()).st_size or values != grid.n_dof:
            raise SnapshotFormatError(f"{path}: expected {grid.n_dof} values, found {values}")
        if layout is not None and (layout.nx_global, layout.ny) != (grid.nx, grid.ny):
            raise ValueError(f"{path}: grid {grid.nx}x{grid.ny} does not match the slab layout")
        f = _diag_ctx(grid, _bc_for(layout), layout, comm)
        L = f.layout
        ncell = L.nx_local * grid.ny
        fh.seek(HEADER_SIZE + NVARS * 8 * L.x_offset * grid.ny)
        body = np.frombuffer(fh.read(ncell * NVARS * 8), dtype="<f8")
    cells = torch.from_numpy(body.astype(np.float64)).to(D.device())
    U = torch.empty(ncell * NVARS, dtype=D.F64, device=D.device())
    N.check(f.ctx.lib.emhd_cells_unpack(f.ctx.sync_stream(), D.ptr(cells), ncell, D.ptr(U)),
            "cells_unpack")
    return U.view(NVARS, L.nx_local, grid.ny), grid, time, params


def _csv_lines(U, grid, time, params):
    yield f"# MHD25 csv time={time!r} nx={grid.nx} ny={grid.ny}"
    yield f"# domain=[{grid.x_lo!r},{grid.x_hi!r}]x[{grid.y_lo!r},{grid.y_hi!r}]"
    yield (f"# gamma={params.gamma!r} mu={params.mu!r} eta={params.eta!r} "
           f"kappa={params.kappa!r}")
    yield "x,y,rho,mx,my,mz,Bx,By,Bz,e"
    xc, yc = grid.cell_centers()
    cells = np.moveaxis(U, 0, -1)                 # (nx, ny, 8) view
    for i, xi in enumerate(xc.tolist()):
        for j, yj in enumerate(yc.tolist()):
            # Python floats: repr round-trips exactly (the reference's formatting)
            yield ",".join(map(repr, [xi, yj] + cells[i, j].tolist()))


def write_snapshot_csv(path, U, grid, time, params):
    """The CSV alternative of the snapshot (snapshot.py:83-99): small grids, one rank."""
    U = D.to_host(U) if isinstance(U, torch.Tensor) else np.asarray(U, dtype=float)
    with open(path, "w") as fh:
        fh.write("\n".join(_csv_lines(U.reshape(NVARS, grid.nx, grid.ny), grid, time, params)) + "\n")
