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

import numpy as np
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
        # any EXTERNAL side: halos come from a neighbour (a rank may be its own neighbour: the
        # periodic ring of one, used to exercise the slab path on a single GPU)
        return self.size > 1 or self.lo_neighbor >= 0 or self.hi_neighbor >= 0

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


def make_ring_layout(nx, ny):
    """One rank owning a periodic x-ring with itself as both neighbours: every slab-path code
    path (EXTERNAL boundaries, halo exchange, all-reduces) on one GPU, bit-identical to the
    periodic single-domain result."""
    return SlabLayout(nx, ny, 0, 1, nx, 0, EXTERNAL, EXTERNAL, 0, 0)


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
        if L.size == 1:                       # ring of one: this rank is both neighbours
            r[0].copy_(s[1])
            r[1].copy_(s[0])
            return recvbuf
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
        if self.layout.size > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def allreduce_max(self, t):
        if self.layout.size > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def allreduce_min(self, t):
        if self.layout.size > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return t

    def barrier(self):
        if self.layout.size > 1:
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


class NativeComm(Comm):
    """Slab collectives issued by libemhd itself (emhd_comm_init_nccl / _host).

    Once attached to the rank's context, the Arnoldi driver keeps its one C call per iteration
    on slab ranks: the dot and norm all-reduces are stream-ordered NCCL collectives issued from
    C (no host sync, no Python between kernels) and the halo of the vector a stencil perturbs is
    exchanged on a second stream while the stencil's interior rows run.  ``transport``:
    ``"nccl"`` (one process per GPU; the two 128-byte unique ids travel by a torch.distributed
    broadcast) or ``"host"`` (several ranks on one GPU; collectives stage through pinned host
    memory and this object's torch.distributed group — gloo in the tests).
    """

    native = True

    def __init__(self, layout, group=None, transport="nccl"):
        super().__init__(layout, group)
        if transport not in ("nccl", "host"):
            raise ValueError("transport must be 'nccl' or 'host'")
        self.transport = transport
        self.ctx = None
        self._cb = None

    def attach(self, ctx):
        """Collective over the group: create this rank's communicator inside ``ctx``."""
        import ctypes
        from . import _native as N
        L = self.layout
        if self.transport == "nccl":
            ids = None
            if L.rank == 0:
                a, b = ctypes.create_string_buffer(128), ctypes.create_string_buffer(128)
                N.check(ctx.lib.emhd_nccl_unique_id(a), "nccl_unique_id")
                N.check(ctx.lib.emhd_nccl_unique_id(b), "nccl_unique_id")
                ids = [a.raw, b.raw]
            if L.size > 1:
                box = [ids]
                src = 0 if self.group is None else dist.get_global_rank(self.group, 0)
                dist.broadcast_object_list(box, src=src, group=self.group)
                ids = box[0]
            N.check(ctx.lib.emhd_comm_init_nccl(ctx.h, L.size, L.rank, L.lo_neighbor, L.hi_neighbor,
                                                ids[0], ids[1]), "comm_init_nccl")
        else:
            def ar(user, buf, n, op):
                try:
                    t = torch.from_numpy(np.ctypeslib.as_array(buf, shape=(n,)))
                    red = {0: dist.ReduceOp.SUM, 2: dist.ReduceOp.MAX, 3: dist.ReduceOp.MIN}[op]
                    if L.size > 1:
                        dist.all_reduce(t, op=red, group=self.group)
                    return 0
                except Exception:
                    return 1

            def ex(user, send, recv, n_side):
                try:
                    s_ = torch.from_numpy(np.ctypeslib.as_array(send, shape=(2 * n_side,))).clone()
                    r_ = torch.from_numpy(np.ctypeslib.as_array(recv, shape=(2 * n_side,)))
                    if L.size == 1:           # ring of one: my top rows are my lo halo
                        r_[:n_side].copy_(s_[n_side:])
                        r_[n_side:].copy_(s_[:n_side])
                    else:
                        Comm.exchange(self, s_, r_)
                    return 0
                except Exception:
                    return 1
            self._cb = (N.HostAllreduceFn(ar), N.HostExchangeFn(ex))     # keep the thunks alive
            N.check(ctx.lib.emhd_comm_init_host(ctx.h, L.size, L.rank, L.lo_neighbor, L.hi_neighbor,
                                                self._cb[0], self._cb[1], None), "comm_init_host")
        self.ctx = ctx

    def _c(self, t, op):
        from . import _native as N
        if self.ctx is None or not t.is_cuda:
            return None
        N.check(self.ctx.lib.emhd_allreduce(self.ctx.sync_stream(), t.data_ptr(), t.numel(), op),
                "allreduce")
        return t

    def allreduce_sum(self, t):
        from . import _native as N
        return self._c(t, N.OP_SUM) if t.is_cuda and self.ctx is not None else super().allreduce_sum(t)

    def allreduce_max(self, t):
        from . import _native as N
        return self._c(t, N.OP_MAX) if t.is_cuda and self.ctx is not None else super().allreduce_max(t)

    def allreduce_min(self, t):
        from . import _native as N
        return self._c(t, N.OP_MIN) if t.is_cuda and self.ctx is not None else super().allreduce_min(t)

    def barrier(self):
        if self.layout.size > 1:
            dist.barrier(group=self.group)
