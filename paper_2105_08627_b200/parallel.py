"""Multi-GPU paths of SURVEY 8(e).

(1) Port sharding: one RHS per port, ports p = rank (mod world).

Each rank owns a replicated libsvh handle on its GPU, solves its ports through
``svh_solve_columns`` (C-ABI) and the admittance columns are all-gathered over
the process group -- the only collective of the solve.  Y -> Z -> L/R is done
by ``svh_y_to_zl`` in libsvh.  The partition / gather / assembly logic is
independent of the solver so it can be exercised with gloo on CPU.

(2) Slab-decomposed matvec (``SlabMatvec``): for a grid too large for one GPU or
strong scaling, rank r holds the y-slab r*Kyl <= y < (r+1)*Kyl; one product is
svh_slab_forward -> all-to-all -> svh_slab_middle -> all-to-all ->
svh_slab_backward (C-ABI; every FFT pass runs in libsvh).  The all-to-all moves
the x-transformed current once per direction (2 Kt points per component in
total, the minimum for a 3-D FFT transpose).  ``virtual_ranks`` runs all P slabs
in one process on one GPU with the exchange done by device copies (the path the
single-GPU tests exercise; NCCL cannot place two ranks on one GPU).
"""
from __future__ import annotations

import numpy as np


def my_ports(n_ports: int, rank: int, world: int):
    """Ports solved by this rank (round robin, p = rank mod world)."""
    return [p for p in range(n_ports) if p % world == rank]


def gather_columns(local_cols, sel, n_ports: int, group=None):
    """All-gather admittance columns.

    local_cols: complex array (n_ports, len(sel)) -- column j is port sel[j].
    Returns the full complex (n_ports, n_ports) Y with Y[:, p] = column of port p.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    per = (n_ports + world - 1) // world
    buf = torch.zeros(per, n_ports + 1, 2, dtype=torch.float64)
    for j, p in enumerate(sel):
        buf[j, 0, 0] = float(p)
        buf[j, 0, 1] = 1.0          # slot used
        buf[j, 1:, 0] = torch.from_numpy(np.ascontiguousarray(local_cols[:, j].real))
        buf[j, 1:, 1] = torch.from_numpy(np.ascontiguousarray(local_cols[:, j].imag))
    backend = dist.get_backend(group)
    if backend == "nccl":
        buf = buf.cuda()
    out = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    Y = np.zeros((n_ports, n_ports), dtype=np.complex128)
    seen = np.zeros(n_ports, dtype=bool)
    for t in out:
        t = t.cpu().numpy()
        for j in range(per):
            if t[j, 0, 1] == 1.0:
                p = int(t[j, 0, 0])
                assert not seen[p], "port solved twice"
                seen[p] = True
                Y[:, p] = t[j, 1:, 0] + 1j * t[j, 1:, 1]
    assert seen.all(), "port not solved"
    return Y


def solve_sharded(handle, ports, group=None):
    """Distributed svh_solve: returns dict(Y, Z, L, R, stats) identical on every rank."""
    import torch.distributed as dist
    from . import svh

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    P = len(ports)
    sel = my_ports(P, rank, world)
    if sel:
        cols, stats, code = handle.solve_columns(ports, sel)
    else:
        cols, stats, code = np.zeros((P, 0), dtype=np.complex128), {}, 0
    Y = gather_columns(cols, sel, P, group)
    Z, L, R = svh.y_to_zl(Y, handle.freq)
    return dict(Y=Y, Z=Z, L=L, R=R, stats=stats, code=code, ports_local=sel)


def slab_exchange(send, recv, P, group=None):
    """The all-to-all of the slab matvec: chunk p of ``send`` goes to rank p, chunk s of
    ``recv`` comes from rank s (equal chunks).  NCCL (NVLink) moves device buffers directly,
    ordered on the current stream (no host synchronisation); a gloo group stages them through
    host memory (the multi-process tests on one GPU)."""
    import torch.distributed as dist
    assert send.numel() % P == 0 and recv.numel() == send.numel()
    if dist.get_backend(group) == "nccl" or not send.is_cuda:
        dist.all_to_all_single(recv, send, group=group)
        return
    hs = send.cpu()
    hr = hs.new_empty(hs.shape)
    dist.all_to_all_single(hr, hs, group=group)
    recv.copy_(hr)


def virtual_exchange(sends, recvs):
    """In-process all-to-all between P virtual ranks: recv[r] chunk s = send[s] chunk r."""
    P = len(sends)
    for r in range(P):
        rc = recvs[r].view(P, -1)
        for s_ in range(P):
            rc[s_].copy_(sends[s_].view(P, -1)[r])


class SlabMatvec:
    """Slab-decomposed Eq. 9 product on lattice-layout slabs [nrhs][5][Kz][Kyl][Kx].

    ``rank``/``P`` with a process group: one slab per process (torch.distributed).
    ``virtual_ranks`` (P > 1, no group): all slabs of one process, exchange by copies.
    """

    def __init__(self, handle, P, rank=0, group=None):
        self.h, self.P, self.rank, self.group = handle, int(P), int(rank), group
        self.Kyl, self.Nxl, self.chunk, self.per_rhs = handle.slab_sizes(self.P)

    def _buffers(self, nrhs, device):
        import torch
        n = nrhs * self.per_rhs
        return (torch.empty(n, dtype=torch.complex64, device=device),
                torch.empty(n, dtype=torch.complex64, device=device))

    def matvec(self, I_slab, green_only=False):
        """This rank's slab of Z.I (collective over the group)."""
        import torch
        I_slab = I_slab.contiguous()
        nrhs = I_slab.shape[0]
        send, recv = self._buffers(nrhs, I_slab.device)
        out = torch.empty_like(I_slab)
        # libsvh launches on the current stream; the collectives are ordered after it (NCCL) or
        # synchronise through the host copy (gloo)
        self.h.slab_forward(self.rank, self.P, I_slab, send)
        slab_exchange(send, recv, self.P, self.group)
        self.h.slab_middle(self.rank, self.P, recv, send, nrhs)
        slab_exchange(send, recv, self.P, self.group)
        self.h.slab_backward(self.rank, self.P, recv, I_slab, out, green_only)
        return out

    def matvec_virtual(self, I_grid, green_only=False):
        """All P slabs in this process: I_grid [nrhs][5][Kz][Ky][Kx] -> Z.I (same layout)."""
        import torch
        P, Kyl = self.P, self.Kyl
        nrhs = I_grid.shape[0]
        slabs = [I_grid[:, :, :, r * Kyl:(r + 1) * Kyl, :].contiguous() for r in range(P)]
        bufs = [self._buffers(nrhs, I_grid.device) for _ in range(P)]
        sends, recvs = [b[0] for b in bufs], [b[1] for b in bufs]
        for r in range(P):
            self.h.slab_forward(r, P, slabs[r], sends[r])
        virtual_exchange(sends, recvs)
        for r in range(P):
            self.h.slab_middle(r, P, recvs[r], sends[r], nrhs)
        virtual_exchange(sends, recvs)
        out = torch.empty_like(I_grid)
        for r in range(P):
            o = torch.empty_like(slabs[r])
            self.h.slab_backward(r, P, recvs[r], slabs[r], o, green_only)
            out[:, :, :, r * Kyl:(r + 1) * Kyl, :] = o
        return out


class P2PSlabMatvec:
    """Fused-exchange slab matvec (SURVEY 8(e)(2) fused variant): svh_slab_forward_p2p /
    svh_slab_middle_p2p store each destination's chunk straight into the peer's receive buffer
    over NVLink peer memory (CUDA IPC) and synchronise with stream memory operations -- no
    all-to-all, no local send buffer, no host synchronisation.  The process group is used once,
    at construction, to exchange the 64-byte IPC handles (all_gather_object)."""

    def __init__(self, handle, nrhs, group=None):
        import torch.distributed as dist
        from . import svh
        self.h, self.group = handle, group
        self.P, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.Kyl, self.Nxl, self.chunk, self.per_rhs = handle.slab_sizes(self.P)
        self.nrhs = int(nrhs)
        nb = self.nrhs * self.per_rhs * 8
        self.own = [svh.ipc_alloc(nb), svh.ipc_alloc(nb), svh.ipc_alloc(2 * self.P * 4)]   # recv1, recv2, flags
        handles = [None] * self.P
        dist.all_gather_object(handles, [hd for _, hd in self.own], group=group)
        self.peer = []          # [buffer kind][peer rank] -> device pointer in this process
        self.opened = []
        for k in range(3):
            row = []
            for p in range(self.P):
                if p == self.rank:
                    row.append(self.own[k][0])
                else:
                    ptr = svh.ipc_open(handles[p][k])
                    self.opened.append(ptr)
                    row.append(ptr)
            self.peer.append(row)
        self.epoch = 0
        dist.barrier(group=group)

    def matvec(self, I_slab, green_only=False):
        """This rank's slab of Z.I ([nrhs][5][Kz][Kyl][Kx]); every rank calls it the same number
        of times (collective by construction)."""
        import torch
        I_slab = I_slab.contiguous()
        assert I_slab.shape[0] == self.nrhs
        self.epoch += 1
        out = torch.empty_like(I_slab)
        self.h.slab_forward_p2p(self.rank, self.P, I_slab, self.peer[0], self.peer[2], self.epoch)
        self.h.slab_middle_p2p(self.rank, self.P, self.own[0][0], self.peer[1], self.peer[2], self.epoch, self.nrhs)
        self.h.slab_backward(self.rank, self.P, self.own[1][0], I_slab, out, green_only)
        return out

    def close(self):
        """Collective: unmap the peers' buffers and free this rank's (after a barrier, so no
        peer still writes into them)."""
        import torch
        import torch.distributed as dist
        from . import svh
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        for p in self.opened:
            svh.ipc_close(p)
        dist.barrier(group=self.group)
        for ptr, _ in self.own:
            svh.ipc_free(ptr)
        self.opened, self.own = [], []

