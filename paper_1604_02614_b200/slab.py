"""x-slab domain decomposition: placement, halo exchange and reductions.

The reference is single-process; this is the B200 build's own
spatial decomposition.  Rank r owns global rows
[x_offset, x_offset + nx_local) of all 8 fields.  x is periodic in every
benchmark configuration, so interior slab edges form a ring; non-periodic
outer edges are filled by the rank itself from the boundary policy.

Halo buffers use the C ABI layout [side][field][row][ny]: side 0 holds the two
rows below local row 0 (global rows x_offset-2, x_offset-1), side 1 the two
rows above local row nx_local-1.  Exchange is point-to-point through
torch.distributed (NCCL on GPUs, gloo in the CPU tests); the reductions are
SUM / MAX all-reduces of a few doubles per Arnoldi pass.
"""

from dataclasses import dataclass

import torch
import torch.distributed as dist

NF = 8
EXTERNAL = "external"


@dataclass(frozen=True)
class SlabLayout:
    nx_global: int
    ny: int
    rank: int
    size: int
    nx_local: int
    x_offset: int
    bc_lo: str          # boundary policy name, or "external" (halo from a neighbour)
    bc_hi: str
    lo_neighbor: int    # rank sending our side-0 halo (-1: none)
    hi_neighbor: int

    @property
    def distributed(self):
        return self.size > 1

    @property
    def n_local(self):
        return NF * self.nx_local * self.ny


def split_rows(nx, size):
    """Balanced contiguous row ranges: (counts, offsets)."""
    base, extra = divmod(nx, size)
    counts = [base + (1 if r < extra else 0) for r in range(size)]
    offs = [sum(counts[:r]) for r in range(size)]
    return counts, offs


def make_layout(nx_global, ny, bc_x, rank=0, size=1):
    """Slab placement of rank `rank` of `size` for an x-policy `bc_x`."""
    if size < 1 or not (0 <= rank < size):
        raise ValueError("bad rank / size")
    counts, offs = split_rows(nx_global, size)
    if min(counts) < 2:
        raise ValueError(f"{nx_global} rows cannot be split over {size} ranks (>= 2 rows each)")
    if size == 1:
        return SlabLayout(nx_global, ny, 0, 1, nx_global, 0, bc_x, bc_x, -1, -1)
    periodic = bc_x == "periodic"
    lo_nb = (rank - 1) % size if (periodic or rank > 0) else -1
    hi_nb = (rank + 1) % size if (periodic or rank < size - 1) else -1
    bc_lo = EXTERNAL if lo_nb >= 0 else bc_x
    bc_hi = EXTERNAL if hi_nb >= 0 else bc_x
    return SlabLayout(nx_global, ny, rank, size, counts[rank], offs[rank], bc_lo, bc_hi, lo_nb, hi_nb)


class Comm:
    """Halo exchange and small all-reduces for one slab layout."""

    def __init__(self, layout, group=None):
        self.layout = layout
        self.group = group

    def exchange(self, sendbuf, recvbuf):
        """sendbuf[0] = our two lowest rows, sendbuf[1] = our two highest rows.

        After the call recvbuf[0] holds the lo neighbour's two highest rows and
        recvbuf[1] the hi neighbour's two lowest rows.
        """
        L = self.layout
        if not L.distributed:
            return recvbuf
        s = sendbuf.view(2, -1)
        r = recvbuf.view(2, -1)
        # Two ordered phases so that P2P matching (in posting order per peer
        # pair, no tags) stays correct when lo and hi neighbour coincide (P=2):
        # phase 1 shifts top rows upwards, phase 2 bottom rows downwards.
        ops = []
        if L.hi_neighbor >= 0:
            ops.append(dist.P2POp(dist.isend, s[1].contiguous(), L.hi_neighbor, self.group))
        if L.lo_neighbor >= 0:
            ops.append(dist.P2POp(dist.irecv, r[0], L.lo_neighbor, self.group))
        if L.lo_neighbor >= 0:
            ops.append(dist.P2POp(dist.isend, s[0].contiguous(), L.lo_neighbor, self.group))
        if L.hi_neighbor >= 0:
            ops.append(dist.P2POp(dist.irecv, r[1], L.hi_neighbor, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return recvbuf

    def allreduce_sum(self, t):
        if self.layout.distributed:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def allreduce_max(self, t):
        if self.layout.distributed:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def allreduce_min(self, t):
        if self.layout.distributed:
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return t

    def barrier(self):
        if self.layout.distributed:
            dist.barrier(group=self.group)


def halo_shape(ny):
    return (2, NF, 2, ny)


def pack_edges_torch(x_local, nx_local, ny):
    """Host-logic twin of emhd_pack_edges for CPU tests (no arithmetic)."""
    U = x_local.view(NF, nx_local, ny)
    out = torch.empty(halo_shape(ny), dtype=x_local.dtype, device=x_local.device)
    out[0] = U[:, 0:2, :]
    out[1] = U[:, nx_local - 2:nx_local, :]
    return out


class PushHalo:
    """Symmetric-memory halo buffer of one slab rank plus its neighbours' peer pointers.

    The producer of the Arnoldi vector w (``emhd_update_push``) stores its edge rows straight
    into the neighbours' buffers over NVLink, replacing the per-iteration P2P halo exchange;
    the norm all-reduce that follows orders those stores before the neighbours' next stencil,
    and the dot-product all-reduces of the next iteration order the neighbours' reads before
    the following overwrite (one buffer suffices).  ``PushHalo.create`` returns None (callers
    keep the NCCL exchange) unless every rank of the group set it up.
    """

    def __init__(self, buf, lo_ptr, hi_ptr, handle):
        self.buf, self.lo_ptr, self.hi_ptr, self._handle = buf, lo_ptr, hi_ptr, handle

    @staticmethod
    def create(layout, comm):
        import os
        if not layout.distributed or os.environ.get("EMHD_PUSH_HALO", "1") == "0":
            return None
        if not dist.is_initialized() or dist.get_backend(comm.group) != "nccl":
            return None
        group = comm.group if comm.group is not None else dist.group.WORLD
        n = 2 * NF * 2 * layout.ny
        dev = torch.device("cuda", torch.cuda.current_device())

        def agree(ok):
            t = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=comm.group)
            return t.item() == 1.0

        buf = None
        try:
            import torch.distributed._symmetric_memory as symm_mem
            buf = symm_mem.empty(n, dtype=torch.float64, device=dev)
            buf.zero_()
            ok = True
        except Exception:
            ok = False
        if not agree(ok):
            return None
        try:
            if hasattr(symm_mem, "enable_symm_mem_for_group"):
                try:
                    symm_mem.enable_symm_mem_for_group(group.group_name)
                except Exception:
                    pass
            hdl = symm_mem.rendezvous(buf, group)
            lo = hi = None
            if layout.lo_neighbor >= 0:
                lo = hdl.get_buffer(layout.lo_neighbor, (n,), torch.float64, 0)
            if layout.hi_neighbor >= 0:
                hi = hdl.get_buffer(layout.hi_neighbor, (n,), torch.float64, 0)
            ok = True
        except Exception:
            ok = False
        if not agree(ok):
            return None
        torch.cuda.synchronize()
        dist.barrier(group=comm.group)
        return PushHalo(buf.view(halo_shape(layout.ny)), None if lo is None else lo.data_ptr(),
                        None if hi is None else hi.data_ptr(), (hdl, lo, hi))
