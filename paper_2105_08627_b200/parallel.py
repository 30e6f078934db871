"""Multi-GPU port sharding: one RHS per port, ports p = rank (mod world).

Each rank owns a replicated libsvh handle on its GPU, solves its ports through
``svh_solve_columns`` (C-ABI) and the admittance columns are all-gathered over
the process group -- the only collective of the solve.  Y -> Z -> L/R is done
by ``svh_y_to_zl`` in libsvh.  The partition / gather / assembly logic is
independent of the solver so it can be exercised with gloo on CPU.
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
