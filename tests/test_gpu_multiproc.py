"""Multi-process paths of SURVEY 8(e) through libsvh, 2 ranks on one GPU over gloo (the
collectives are CPU-staged; every kernel of a rank is independent of the other rank's, so
sharing one GPU is safe).

* Port sharding (8(e)(1)): parallel.solve_sharded on 2 ranks returns the admittance matrix
  of the single-process svh_solve BIT FOR BIT (north star: "L from 8-GPU RHS sharding must
  equal the 1-GPU L bit for bit") -- every reduction of the solve has a batch-independent
  order, so a port's arithmetic does not depend on which ports share its batch.
* Slab-decomposed matvec (8(e)(2)): parallel.SlabMatvec.matvec with one y-slab per rank and
  the two all-to-alls through the process group equals the single-GPU svh_matvec_grid.
"""
import os
import socket

import numpy as np
import pytest

import svh_inputs

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _three_port_case():
    mat = np.zeros((3, 8, 16), np.uint8)
    mat[0, :, :] = 1
    mat[2, 1:3, 1:15] = 1
    mat[2, 5:7, 1:15] = 1
    mat[1, 1:3, 14:15] = 1
    mat[1, 5:7, 14:15] = 1
    g = [(0, -1, (0, 0, 0), (1, 8, 1))]
    ports = [{"plus": [(0, -1, (1, 1, 2), (2, 3, 3))], "minus": g},
             {"plus": [(0, -1, (1, 5, 2), (2, 7, 3))], "minus": g},
             {"plus": [(0, +1, (15, 0, 0), (16, 8, 1))], "minus": g}]
    return dict(mat_id=mat, dx=0.25e-6, materials=[(1.7e7, 90e-9)], freq=10e9, ports=ports)


def _solve_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    from paper_2105_08627_b200 import parallel, svh
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    case = _three_port_case()
    with svh.setup_case(case, tucker_tol=0.0, rre=1e-7) as h:
        res = parallel.solve_sharded(h, case["ports"])
    q.put((rank, res["Y"], res["L"], res["ports_local"]))
    dist.destroy_process_group()


def test_sharded_solve_bitwise_equals_single(svh_lib):
    import torch.multiprocessing as mp
    case = _three_port_case()
    with svh_lib.setup_case(case, tucker_tol=0.0, rre=1e-7) as h:
        single = h.solve(case["ports"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_solve_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    owned = sorted(sum([list(r[3]) for r in res], []))
    assert owned == [0, 1, 2]
    for r in res:
        assert np.array_equal(r[1], single["Y"]), np.max(np.abs(r[1] - single["Y"]))
        assert np.array_equal(r[2], single["L"])


def test_batch_independent_port_solve(svh_lib):
    """The arithmetic behind the bitwise claim: solving port p alone (svh_solve_columns with one
    column) gives bitwise the column of the batched 3-port solve."""
    case = _three_port_case()
    with svh_lib.setup_case(case, tucker_tol=0.0, rre=1e-7) as h:
        full = h.solve(case["ports"])
        for p in range(3):
            cols, _, code = h.solve_columns(case["ports"], [p])
            assert code == 0
            assert np.array_equal(cols[:, 0], full["Y"][:, p]), p


def _slab_worker(rank, world, port, shape, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    from oracle.lattice import Lattice
    from paper_2105_08627_b200 import svh
    from paper_2105_08627_b200.parallel import SlabMatvec
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    case = svh_inputs.layered(shape)
    lat = Lattice(case["mat_id"])
    I = svh_inputs.currents(lat.K, 2, seed=31)
    g = np.zeros((2, 5) + case["mat_id"].shape, dtype=np.complex64)
    c = lat.coords
    g[:, :, c[:, 2], c[:, 1], c[:, 0]] = I
    with svh.setup_case(case) as h:
        sm = SlabMatvec(h, world, rank=rank)
        mine = torch.from_numpy(g[:, :, :, rank * sm.Kyl:(rank + 1) * sm.Kyl, :].copy()).cuda()
        out = sm.matvec(mine).cpu().numpy()
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("shape", [(40, 64, 6), (40, 8, 40)])
def test_slab_matvec_two_processes(svh_lib, shape):
    import torch
    import torch.multiprocessing as mp
    from oracle.lattice import Lattice
    case = svh_inputs.layered(shape)
    lat = Lattice(case["mat_id"])
    I = svh_inputs.currents(lat.K, 2, seed=31)
    g = np.zeros((2, 5) + case["mat_id"].shape, dtype=np.complex64)
    c = lat.coords
    g[:, :, c[:, 2], c[:, 1], c[:, 0]] = I
    with svh_lib.setup_case(case) as h:
        whole = h.matvec_grid(torch.from_numpy(g).cuda()).cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, shape, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    Kyl = shape[1] // 2
    got = np.concatenate([res[0], res[1]], axis=3)
    assert got.shape == whole.shape
    assert np.linalg.norm(got - whole) <= 1e-6 * np.linalg.norm(whole)
    del Kyl


def _p2p_worker(rank, world, port, shape, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    from oracle.lattice import Lattice
    from paper_2105_08627_b200 import svh
    from paper_2105_08627_b200.parallel import P2PSlabMatvec, SlabMatvec
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    case = svh_inputs.layered(shape)
    lat = Lattice(case["mat_id"])
    outs = []
    with svh.setup_case(case) as h:
        sm = P2PSlabMatvec(h, 2)
        staged = SlabMatvec(h, world, rank=rank)
        for it in range(3):     # several products: epochs advance, the two buffers alternate roles
            I = svh_inputs.currents(lat.K, 2, seed=40 + it)
            g = np.zeros((2, 5) + case["mat_id"].shape, dtype=np.complex64)
            c = lat.coords
            g[:, :, c[:, 2], c[:, 1], c[:, 0]] = I
            mine = torch.from_numpy(g[:, :, :, rank * sm.Kyl:(rank + 1) * sm.Kyl, :].copy()).cuda()
            outs.append((sm.matvec(mine).cpu().numpy(), staged.matvec(mine).cpu().numpy()))
        sm.close()
    q.put((rank, outs))
    dist.destroy_process_group()


@pytest.mark.parametrize("shape", [(40, 64, 6), (24, 16, 20)])
def test_p2p_slab_matvec_two_processes(svh_lib, shape):
    """Fused-exchange slab matvec (peer-memory stores + stream flag waits):
    bitwise equal to the collective-staged slab path (same kernels, same data) and equal to the
    single-GPU product, over three consecutive products."""
    import torch
    import torch.multiprocessing as mp
    from oracle.lattice import Lattice
    case = svh_inputs.layered(shape)
    lat = Lattice(case["mat_id"])
    wholes = []
    with svh_lib.setup_case(case) as h:
        for it in range(3):
            I = svh_inputs.currents(lat.K, 2, seed=40 + it)
            g = np.zeros((2, 5) + case["mat_id"].shape, dtype=np.complex64)
            c = lat.coords
            g[:, :, c[:, 2], c[:, 1], c[:, 0]] = I
            wholes.append(h.matvec_grid(torch.from_numpy(g).cuda()).cpu().numpy())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, 2, port, shape, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for it in range(3):
        for r in range(2):
            assert np.array_equal(res[r][it][0], res[r][it][1]), (it, r)
        got = np.concatenate([res[0][it][0], res[1][it][0]], axis=3)
        assert np.linalg.norm(got - wholes[it]) <= 1e-6 * np.linalg.norm(wholes[it])
