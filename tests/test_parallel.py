"""Multi-process (gloo, world_size 2, CPU) tests of the port-sharding layer and the
host-side Y -> Z -> L post-processing of libsvh (no GPU needed)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_08627_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, P, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = np.random.default_rng(seed)
    Y = g.standard_normal((P, P)) + 1j * g.standard_normal((P, P))
    sel = parallel.my_ports(P, rank, world)
    cols = Y[:, sel]
    full = parallel.gather_columns(cols, sel, P)
    q.put((rank, sel, np.array_equal(full, Y)))
    dist.destroy_process_group()


@pytest.mark.parametrize("P,world", [(5, 2), (16, 2), (1, 2)])
def test_gather_columns_gloo(P, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    owned = sorted(sum([r[1] for r in res], []))
    assert owned == list(range(P))          # every port solved exactly once
    assert all(r[2] for r in res)           # identical Y on every rank


def test_my_ports_partition():
    for P in range(1, 20):
        for world in (1, 2, 3, 8):
            allp = sorted(sum([parallel.my_ports(P, r, world) for r in range(world)], []))
            assert allp == list(range(P))


def test_y_to_zl_host():
    """svh_y_to_zl (C-ABI, host only) inverts Y and splits L/R (reading G13)."""
    from paper_2105_08627_b200 import svh
    g = np.random.default_rng(0)
    Y = g.standard_normal((4, 4)) + 1j * g.standard_normal((4, 4)) + 4 * np.eye(4)
    f = 3e9
    Z, L, R = svh.y_to_zl(Y, f)
    assert np.allclose(Z @ Y, np.eye(4), atol=1e-12)
    assert np.allclose(L, Z.imag / (2 * np.pi * f)) and np.allclose(R, Z.real)
    with pytest.raises(svh.SvhError):
        svh.y_to_zl(np.zeros((2, 2)), f)


def _slab_worker(rank, world, port, q):
    """Each rank fills its send buffer with (src rank, dest chunk, index) tags; after the
    all-to-all chunk s of recv must hold rank s's chunk addressed to this rank."""
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    chunk = 6
    send = torch.zeros(world * chunk, dtype=torch.complex64)
    for p in range(world):
        for i in range(chunk):
            send[p * chunk + i] = complex(100 * rank + p, i)
    recv = torch.empty_like(send)
    parallel.slab_exchange(send, recv, world)
    ok = all(recv[s * chunk + i] == complex(100 * s + rank, i) for s in range(world) for i in range(chunk))
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_exchange_gloo(world):
    """SURVEY 8(e)(2) slab transpose: the NCCL/gloo all-to-all routes chunk p of rank r's
    send buffer to chunk r of rank p's recv buffer, as svh_slab_* lay them out."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_virtual_exchange_matches_all_to_all():
    """The single-process exchange used by the virtual-slab GPU tests is the same routing."""
    import torch
    P, chunk = 4, 3
    sends = [torch.tensor([complex(100 * r + p, i) for p in range(P) for i in range(chunk)], dtype=torch.complex64)
             for r in range(P)]
    recvs = [torch.empty_like(s) for s in sends]
    parallel.virtual_exchange(sends, recvs)
    for r in range(P):
        for s in range(P):
            for i in range(chunk):
                assert recvs[r][s * chunk + i] == complex(100 * s + r, i)
