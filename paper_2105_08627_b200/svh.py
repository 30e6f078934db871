"""Thin Python binding of libsvh (include/svh.h) -- argument marshalling only.

Every step of the hot path runs in libsvh's CUDA kernels; torch is used only for
device memory and streams.  There is no CPU fallback: if libsvh.so is missing
or no CUDA device is present the calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsvh.so")

SVH_OK = 0
ERRORS = {-1: "SVH_EINVAL", -2: "SVH_ENOMEM", -3: "SVH_ECUDA", -4: "SVH_ENCCL", -5: "SVH_ENOCONV",
          -6: "SVH_EOPENPORT", -7: "SVH_ECACHE"}


class SvhError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class Grid(ctypes.Structure):
    _fields_ = [("kx", ctypes.c_int32), ("ky", ctypes.c_int32), ("kz", ctypes.c_int32), ("dx_m", ctypes.c_double)]


class Material(ctypes.Structure):
    _fields_ = [("sigma_n_S_per_m", ctypes.c_double), ("lambda_L_m", ctypes.c_double)]


class FaceRect(ctypes.Structure):
    _fields_ = [("axis", ctypes.c_int32), ("side", ctypes.c_int32), ("lo", ctypes.c_int32 * 3),
                ("hi", ctypes.c_int32 * 3)]


class Port(ctypes.Structure):
    _fields_ = [("n_plus", ctypes.c_int32), ("plus", ctypes.POINTER(FaceRect)),
                ("n_minus", ctypes.c_int32), ("minus", ctypes.POINTER(FaceRect))]


class Opts(ctypes.Structure):
    _fields_ = [("tucker_tol", ctypes.c_double), ("restart", ctypes.c_int32), ("rre", ctypes.c_double),
                ("inner_tol", ctypes.c_double), ("inner_maxit", ctypes.c_int32), ("max_iters", ctypes.c_int32),
                ("rhs_chunk", ctypes.c_int32), ("verbose", ctypes.c_int32), ("kernel_cache", ctypes.c_char_p),
                ("plan", ctypes.c_int32), ("precision", ctypes.c_int32), ("schur_solver", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("total_iterations", ctypes.c_int32),
                ("inner_iterations", ctypes.c_int32), ("converged", ctypes.c_int32), ("final_rre", ctypes.c_double),
                ("t_setup_s", ctypes.c_double), ("t_solve_s", ctypes.c_double), ("t_matvec_s", ctypes.c_double),
                ("t_precond_s", ctypes.c_double), ("ranks", (ctypes.c_int32 * 3) * 7),
                ("compression_ratio", ctypes.c_double), ("t_precond_setup_s", ctypes.c_double),
                ("precond_bytes", ctypes.c_double), ("schur_solver", ctypes.c_int32),
                ("amg_levels", ctypes.c_int32), ("amg_op_complexity", ctypes.c_double)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "ranks"}
        d["ranks"] = [[self.ranks[q][a] for a in range(3)] for q in range(7)]
        return d


_lib = None


def lib():
    """Load libsvh.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -m paper_2105_08627_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.svh_default_opts.argtypes = [ctypes.POINTER(Opts)]
        L.svh_default_opts.restype = None
        L.svh_setup.argtypes = [ctypes.POINTER(Grid), ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(Material), i32,
                                dbl, ctypes.POINTER(Opts), i32, ctypes.POINTER(vp)]
        L.svh_set_frequency.argtypes = [vp, dbl]
        L.svh_unknowns.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.svh_embedding.argtypes = [vp, ctypes.POINTER(i32)]
        L.svh_plan_info.argtypes = [vp, ctypes.POINTER(i64)]
        vpp = ctypes.POINTER(vp)
        L.svh_ipc_alloc.argtypes = [ctypes.c_size_t, vpp, ctypes.c_char_p]
        L.svh_ipc_free.argtypes = [vp]
        L.svh_ipc_open.argtypes = [ctypes.c_char_p, vpp]
        L.svh_ipc_close.argtypes = [vp]
        L.svh_slab_forward_p2p.argtypes = [vp, i32, i32, vp, vpp, vpp, ctypes.c_uint32, i32, vp]
        L.svh_slab_middle_p2p.argtypes = [vp, i32, i32, vp, vpp, vpp, ctypes.c_uint32, i32, vp]
        L.svh_matvec_z.argtypes = [vp, vp, vp, i32, i32, vp]
        L.svh_matvec_plan.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(ctypes.c_float),
                                      ctypes.POINTER(ctypes.c_float)]
        L.svh_slab_sizes.argtypes = [vp, i32, ctypes.POINTER(i64)]
        L.svh_matvec_host.argtypes = [vp, vp, vp, i32, i32, i32, vp]
        L.svh_kernel_cache_build.argtypes = [ctypes.c_char_p, ctypes.POINTER(i32), dbl, i32]
        L.svh_slab_forward.argtypes = [vp, i32, i32, vp, vp, i32, vp]
        L.svh_slab_middle.argtypes = [vp, i32, i32, vp, vp, i32, vp]
        L.svh_slab_backward.argtypes = [vp, i32, i32, vp, vp, vp, i32, i32, vp]
        L.svh_matvec.argtypes = [vp, vp, vp, i32, i32, vp]
        L.svh_matvec_grid.argtypes = [vp, vp, vp, i32, i32, vp]
        L.svh_apply_system.argtypes = [vp, vp, vp, i32, vp]
        dp = ctypes.POINTER(ctypes.c_double)
        L.svh_solve.argtypes = [vp, ctypes.POINTER(Port), i32, dp, dp, dp, dp, ctypes.POINTER(Stats)]
        L.svh_solve_columns.argtypes = [vp, ctypes.POINTER(Port), i32, ctypes.POINTER(i32), i32, dp,
                                        ctypes.POINTER(Stats)]
        L.svh_get_kernels.argtypes = [vp, dp]
        L.svh_y_to_zl.argtypes = [dp, i32, dbl, dp, dp, dp]
        L.svh_profile_enable.argtypes = [vp, i32]
        L.svh_profile_read.argtypes = [vp, dp, ctypes.POINTER(i64), i32]
        L.svh_get_stats.argtypes = [vp, ctypes.POINTER(Stats)]
        L.svh_destroy.argtypes = [vp]
        L.svh_destroy.restype = None
        L.svh_last_error.restype = ctypes.c_char_p
        L.svh_launch_count.restype = i64
        for name in ("svh_kernel_cache_build", "svh_matvec_host", "svh_slab_sizes", "svh_slab_forward", "svh_slab_middle", "svh_slab_backward",
                     "svh_setup", "svh_set_frequency", "svh_unknowns", "svh_embedding", "svh_plan_info", "svh_matvec",
                     "svh_matvec_grid", "svh_apply_system", "svh_solve", "svh_solve_columns", "svh_get_kernels",
                     "svh_get_stats", "svh_profile_enable", "svh_profile_read", "svh_y_to_zl", "svh_matvec_plan",
                     "svh_ipc_alloc", "svh_ipc_free", "svh_ipc_open", "svh_ipc_close", "svh_slab_forward_p2p",
                     "svh_slab_middle_p2p", "svh_matvec_z"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


EXPORTED = ("svh_default_opts", "svh_setup", "svh_set_frequency", "svh_unknowns", "svh_embedding", "svh_plan_info",
            "svh_kernel_cache_build", "svh_matvec_host", "svh_slab_sizes", "svh_slab_forward", "svh_slab_middle",
            "svh_slab_backward",
            "svh_matvec",
            "svh_matvec_grid", "svh_apply_system", "svh_solve", "svh_solve_columns", "svh_get_kernels",
            "svh_get_stats", "svh_profile_enable", "svh_profile_read", "svh_y_to_zl", "svh_matvec_plan",
            "svh_ipc_alloc", "svh_ipc_free", "svh_ipc_open", "svh_ipc_close", "svh_slab_forward_p2p",
            "svh_slab_middle_p2p", "svh_matvec_z", "svh_destroy",
            "svh_last_error", "svh_launch_count")


def _check(code):
    if code != SVH_OK:
        raise SvhError(code, lib().svh_last_error().decode())


def y_to_zl(Y, freq):
    """svh_y_to_zl: Z = Y^-1, L = Im Z / omega, R = Re Z (host, in libsvh)."""
    Y = np.asarray(Y, dtype=np.complex128)
    P = Y.shape[0]
    Yi = np.empty(2 * P * P)
    Yi[0::2] = Y.real.ravel()
    Yi[1::2] = Y.imag.ravel()
    Z = np.zeros(2 * P * P)
    L = np.zeros(P * P)
    R = np.zeros(P * P)
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    _check(lib().svh_y_to_zl(dp(Yi), P, float(freq), dp(Z), dp(L), dp(R)))
    return (Z[0::2] + 1j * Z[1::2]).reshape(P, P), L.reshape(P, P), R.reshape(P, P)


def launch_count() -> int:
    return int(lib().svh_launch_count())


def _ptr_array(ptrs):
    return (ctypes.c_void_p * len(ptrs))(*[ctypes.c_void_p(int(p)) for p in ptrs])


def ipc_alloc(nbytes):
    """svh_ipc_alloc: a zeroed device buffer and its 64-byte CUDA IPC handle -> (ptr, handle)."""
    p = ctypes.c_void_p()
    hd = ctypes.create_string_buffer(64)
    _check(lib().svh_ipc_alloc(int(nbytes), ctypes.byref(p), hd))
    return int(p.value), bytes(hd.raw)


def ipc_open(handle):
    p = ctypes.c_void_p()
    _check(lib().svh_ipc_open(bytes(handle), ctypes.byref(p)))
    return int(p.value)


def ipc_close(ptr):
    _check(lib().svh_ipc_close(ctypes.c_void_p(int(ptr))))


def ipc_free(ptr):
    _check(lib().svh_ipc_free(ctypes.c_void_p(int(ptr))))


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def make_ports(ports):
    """Python port dicts (svh_inputs convention) -> ctypes array (keeps buffers alive)."""
    keep = []
    arr = (Port * max(1, len(ports)))()
    for i, p in enumerate(ports):
        lists = []
        for key in ("plus", "minus"):
            rects = p[key]
            ra = (FaceRect * max(1, len(rects)))()
            for j, (axis, side, lo, hi) in enumerate(rects):
                ra[j].axis = axis
                ra[j].side = side
                for d in range(3):
                    ra[j].lo[d] = int(lo[d])
                    ra[j].hi[d] = int(hi[d])
            keep.append(ra)
            lists.append((len(rects), ra))
        arr[i].n_plus, arr[i].plus = lists[0][0], ctypes.cast(lists[0][1], ctypes.POINTER(FaceRect))
        arr[i].n_minus, arr[i].minus = lists[1][0], ctypes.cast(lists[1][1], ctypes.POINTER(FaceRect))
    keep.append(arr)
    return arr, keep


class Handle:
    """svh_setup ... svh_destroy.  Mirrors the C-ABI names."""

    def __init__(self, mat_id, dx, materials, freq, tucker_tol=0.0, device=0, **opts):
        L = lib()
        mat = np.ascontiguousarray(np.asarray(mat_id, dtype=np.uint8))
        kz, ky, kx = mat.shape
        g = Grid(kx, ky, kz, float(dx))
        mats = (Material * len(materials))(*[Material(float(s), float(l)) for s, l in materials])
        o = Opts()
        L.svh_default_opts(ctypes.byref(o))
        o.tucker_tol = float(tucker_tol)
        for k, v in opts.items():
            setattr(o, k, v.encode() if isinstance(v, str) else v)
        h = ctypes.c_void_p()
        _check(L.svh_setup(ctypes.byref(g), mat.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), mats,
                           len(materials), float(freq), ctypes.byref(o), int(device), ctypes.byref(h)))
        self._h = h
        self.device = device
        self.freq = float(freq)
        self.tucker = tucker_tol > 0
        self.shape = (kz, ky, kx)
        K, M = ctypes.c_int64(), ctypes.c_int64()
        _check(L.svh_unknowns(h, ctypes.byref(K), ctypes.byref(M)))
        self.K, self.M = K.value, M.value
        self.N = 5 * self.K + self.M
        n3 = (ctypes.c_int32 * 3)()
        _check(L.svh_embedding(h, n3))
        self.embedding = tuple(n3)
        info = (ctypes.c_int64 * 4)()
        _check(L.svh_plan_info(h, info))
        # non-empty (y, z) rows and z planes: the pruned passes touch only these
        self.rows_nonempty, self.planes_nonempty = int(info[0]), int(info[1])

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            lib().svh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- API
    def set_frequency(self, freq):
        _check(lib().svh_set_frequency(self._h, float(freq)))
        self.freq = float(freq)

    def matvec(self, I, out=None, green_only=False, stream=None):
        """I: torch complex64 cuda tensor [nrhs, 5, K] (or [5, K])."""
        import torch
        squeeze = I.dim() == 2
        Ib = I.unsqueeze(0) if squeeze else I
        assert Ib.dtype == torch.complex64 and Ib.is_cuda and Ib.shape[1:] == (5, self.K)
        Ib = Ib.contiguous()
        o = torch.empty_like(Ib) if out is None else out
        _check(lib().svh_matvec(self._h, ctypes.c_void_p(Ib.data_ptr()), ctypes.c_void_p(o.data_ptr()),
                                Ib.shape[0], int(green_only), _stream_ptr(stream)))
        return o[0] if squeeze and out is None else o

    def matvec_z(self, I, out=None, green_only=False, stream=None):
        """svh_matvec_z: the complex128 build (handle set up with precision=1); I: complex128
        [nrhs][5][K] (or [5][K]) on the device."""
        import torch
        Ib = I.unsqueeze(0) if I.dim() == 2 else I
        assert Ib.dtype == torch.complex128 and Ib.is_cuda and Ib.shape[1:] == (5, self.K)
        Ib = Ib.contiguous()
        o = torch.empty_like(Ib) if out is None else out
        _check(lib().svh_matvec_z(self._h, ctypes.c_void_p(Ib.data_ptr()), ctypes.c_void_p(o.data_ptr()),
                                  Ib.shape[0], int(green_only), _stream_ptr(stream)))
        return o if I.dim() == 3 else o[0]

    def matvec_host(self, I_host, out_host, green_only=False, chunk=0, stream=None):
        """End-to-end product on host tensors (complex64 [nrhs, 5, K], pinned for overlap):
        H2D / passes / D2H pipelined by libsvh; returns when out_host is filled."""
        import torch
        assert I_host.dtype == torch.complex64 and not I_host.is_cuda and I_host.is_contiguous()
        assert out_host.shape == I_host.shape and out_host.dtype == torch.complex64 and not out_host.is_cuda
        _check(lib().svh_matvec_host(self._h, ctypes.c_void_p(I_host.data_ptr()), ctypes.c_void_p(out_host.data_ptr()),
                                     I_host.shape[0], int(green_only), int(chunk), _stream_ptr(stream)))
        return out_host

    def matvec_grid(self, I, out=None, green_only=False, stream=None):
        """I: torch complex64 cuda tensor [nrhs, 5, kz, ky, kx]."""
        import torch
        assert I.dtype == torch.complex64 and I.is_cuda and tuple(I.shape[1:]) == (5,) + self.shape
        I = I.contiguous()
        o = torch.empty_like(I) if out is None else out
        _check(lib().svh_matvec_grid(self._h, ctypes.c_void_p(I.data_ptr()), ctypes.c_void_p(o.data_ptr()),
                                     I.shape[0], int(green_only), _stream_ptr(stream)))
        return o

    # -- slab-decomposed matvec; orchestration in parallel.SlabMatvec
    def slab_sizes(self, P):
        """(Kyl, Nxl, elements per peer chunk per RHS, send/recv elements per RHS)."""
        out = (ctypes.c_int64 * 4)()
        _check(lib().svh_slab_sizes(self._h, int(P), out))
        return tuple(int(v) for v in out)

    def slab_forward(self, rank, P, I_slab, send, stream=None):
        _check(lib().svh_slab_forward(self._h, int(rank), int(P), ctypes.c_void_p(I_slab.data_ptr()),
                                      ctypes.c_void_p(send.data_ptr()), I_slab.shape[0], _stream_ptr(stream)))

    def slab_middle(self, rank, P, recv, send, nrhs, stream=None):
        _check(lib().svh_slab_middle(self._h, int(rank), int(P), ctypes.c_void_p(recv.data_ptr()),
                                     ctypes.c_void_p(send.data_ptr()), int(nrhs), _stream_ptr(stream)))

    def slab_forward_p2p(self, rank, P, I_slab, recv1_peers, flag_peers, epoch, stream=None):
        """Fused-exchange forward step: pass A, chunks stored into the peers' recv1 buffers (raw
        device pointers, indexed by rank), flag slot 0 = epoch, stream wait for every peer."""
        _check(lib().svh_slab_forward_p2p(self._h, int(rank), int(P), ctypes.c_void_p(I_slab.data_ptr()),
                                          _ptr_array(recv1_peers), _ptr_array(flag_peers), int(epoch),
                                          I_slab.shape[0], _stream_ptr(stream)))

    def slab_middle_p2p(self, rank, P, recv1, recv2_peers, flag_peers, epoch, nrhs, stream=None):
        _check(lib().svh_slab_middle_p2p(self._h, int(rank), int(P), ctypes.c_void_p(int(recv1)),
                                         _ptr_array(recv2_peers), _ptr_array(flag_peers), int(epoch), int(nrhs),
                                         _stream_ptr(stream)))

    def slab_backward(self, rank, P, recv, I_slab, out, green_only=False, stream=None):
        """recv: a device tensor or a raw device pointer (int, e.g. an svh_ipc_alloc buffer)."""
        recv = recv if isinstance(recv, int) else recv.data_ptr()
        _check(lib().svh_slab_backward(self._h, int(rank), int(P), ctypes.c_void_p(recv),
                                       ctypes.c_void_p(I_slab.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                       I_slab.shape[0], int(green_only), _stream_ptr(stream)))

    def apply_system(self, x, out=None, stream=None):
        import torch
        xb = x.unsqueeze(0) if x.dim() == 1 else x
        assert xb.dtype == torch.complex64 and xb.is_cuda and xb.shape[1] == self.N
        xb = xb.contiguous()
        o = torch.empty_like(xb) if out is None else out
        _check(lib().svh_apply_system(self._h, ctypes.c_void_p(xb.data_ptr()), ctypes.c_void_p(o.data_ptr()),
                                      xb.shape[0], _stream_ptr(stream)))
        return o[0] if x.dim() == 1 and out is None else o

    def solve(self, ports):
        P = len(ports)
        arr, keep = make_ports(ports)
        Z = np.zeros(2 * P * P)
        Lm = np.zeros(P * P)
        R = np.zeros(P * P)
        Y = np.zeros(2 * P * P)
        st = Stats()
        dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
        code = lib().svh_solve(self._h, arr, P, dp(Z), dp(Lm), dp(R), dp(Y), ctypes.byref(st))
        if code not in (SVH_OK, -5):
            _check(code)
        del keep
        return dict(Z=(Z[0::2] + 1j * Z[1::2]).reshape(P, P), L=Lm.reshape(P, P), R=R.reshape(P, P),
                    Y=(Y[0::2] + 1j * Y[1::2]).reshape(P, P), stats=st.as_dict(), code=code)

    def solve_columns(self, ports, sel):
        P = len(ports)
        arr, keep = make_ports(ports)
        sel = np.ascontiguousarray(np.asarray(sel, dtype=np.int32))
        Y = np.zeros(2 * P * max(1, sel.size))
        st = Stats()
        code = lib().svh_solve_columns(self._h, arr, P, sel.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                       sel.size, Y.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                       ctypes.byref(st))
        if code not in (SVH_OK, -5):
            _check(code)
        del keep
        Yc = (Y[0::2] + 1j * Y[1::2])[: P * sel.size].reshape(sel.size, P).T  # column j = port sel[j]
        return Yc, st.as_dict(), code

    def kernels(self):
        kz, ky, kx = self.shape
        out = np.zeros((7, kz, ky, kx))
        _check(lib().svh_get_kernels(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def profile(self, on=True):
        _check(lib().svh_profile_enable(self._h, int(on)))

    def profile_read(self, reset=True):
        """Per-record device ms and launch counts: [0:5] = P5 passes A..E, [5] = whole P3s products."""
        ms = np.zeros(6)
        n = np.zeros(6, dtype=np.int64)
        _check(lib().svh_profile_read(self._h, ms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                      n.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(reset)))
        return ms, n

    def matvec_plan(self):
        """(plan of the last matvec chunk: 3 = P3s / 5 = P5, P5 ms, P3s ms of the last auto-selection)."""
        p, a, b = ctypes.c_int32(), ctypes.c_float(), ctypes.c_float()
        _check(lib().svh_matvec_plan(self._h, ctypes.byref(p), ctypes.byref(a), ctypes.byref(b)))
        return int(p.value), float(a.value), float(b.value)

    def stats(self):
        st = Stats()
        _check(lib().svh_get_stats(self._h, ctypes.byref(st)))
        return st.as_dict()


def kernel_cache_build(path, nmax, tol=1e-10, device=0):
    """Algorithm 2 install stage (svh_kernel_cache_build): Tucker-compressed unit-voxel kernels on
    the offset domain nmax = (Nx, Ny, Nz), written to `path`; use with setup(kernel_cache=path)."""
    n = (ctypes.c_int32 * 3)(*[int(v) for v in nmax])
    _check(lib().svh_kernel_cache_build(str(path).encode(), n, float(tol), int(device)))


def setup_case(case, tucker_tol=None, device=0, **opts):
    """Build a Handle from an svh_inputs case dict."""
    tol = case.get("tucker_tol", 0.0) if tucker_tol is None else tucker_tol
    return Handle(case["mat_id"], case["dx"], case["materials"], case["freq"], tucker_tol=tol, device=device,
                  **opts)


