"""Algorithm 2: install-time Tucker cache of the Toeplitz kernels and the setup
that restores a grid's kernels from it.  Parity: the restored kernels match
the direct quadrature within the cache tolerance, the matvec built on them matches the fp64
oracle (north-star bar), and a cache smaller than the grid is refused (SVH_ECACHE)."""
import numpy as np
import pytest

import svh_inputs
from oracle.lattice import Lattice
from oracle.operator import matvec_direct

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cache_file(tmp_path_factory, svh_lib):
    p = tmp_path_factory.mktemp("svxt") / "kernels.svxt"
    svh_lib.kernel_cache_build(p, (48, 40, 12), tol=1e-10)
    return p


@pytest.mark.parametrize("shape", [(24, 20, 6), (48, 40, 12), (7, 33, 3)])
def test_restored_kernels_vs_quadrature(svh_lib, cache_file, shape):
    case = svh_inputs.random_fill(shape, fill=0.6, seed=sum(shape))
    with svh_lib.setup_case(case) as h:
        direct = h.kernels()
    with svh_lib.setup_case(case, kernel_cache=str(cache_file)) as h:
        cached = h.kernels()
    # Alg. 1 bounds the Frobenius error of each weighted tensor on the big domain by tol; the
    # trimmed block inherits the absolute error, so compare relative to each kernel's norm
    for q in range(7):
        err = np.linalg.norm(cached[q] - direct[q]) / np.linalg.norm(direct[q])
        assert err < 1e-8, (q, err)


def test_cached_matvec_vs_oracle(svh_lib, cache_file):
    import torch
    case = svh_inputs.layered((40, 36, 10))
    lat = Lattice(case["mat_id"])
    I = svh_inputs.currents(lat.K, 2, seed=41)
    w = 2 * np.pi * case["freq"]
    with svh_lib.setup_case(case, kernel_cache=str(cache_file)) as h:
        for go in (True, False):
            got = h.matvec(torch.from_numpy(I.astype(np.complex64)).cuda(), green_only=go).cpu().numpy()
            ref = matvec_direct(lat, case["materials"], w, case["dx"], I, green_only=go)
            for r in range(2):
                assert np.linalg.norm(got[r] - ref[r]) / np.linalg.norm(ref[r]) < 1e-5


def test_cache_too_small_is_refused(svh_lib, cache_file):
    case = svh_inputs.random_fill((49, 8, 4), fill=0.5, seed=1)
    with pytest.raises(svh_lib.SvhError, match="smaller than the grid"):
        svh_lib.setup_case(case, kernel_cache=str(cache_file))


def test_not_a_cache_is_refused(svh_lib, tmp_path):
    bad = tmp_path / "bad.svxt"
    bad.write_bytes(b"NOPE" + bytes(64))
    case = svh_inputs.random_fill((8, 8, 4), fill=0.5, seed=1)
    with pytest.raises(svh_lib.SvhError, match="not an SVXT"):
        svh_lib.setup_case(case, kernel_cache=str(bad))


def test_cache_file_layout_and_crc(svh_lib, cache_file):
    """The SVXT layout of SPEC S:236: magic, u32 version, f64 tol, u64 N_max[3], u32 block
    count, per block a 2-byte tag and u64 ranks, f64 factors + core, trailing CRC-32 (zlib) of
    every preceding byte."""
    import struct
    import zlib
    b = open(cache_file, "rb").read()
    assert b[:4] == b"SVXT"
    ver, tol = struct.unpack_from("<Id", b, 4)
    nmax = struct.unpack_from("<3Q", b, 16)
    (nblk,) = struct.unpack_from("<I", b, 40)
    assert (ver, nmax, nblk) == (2, (48, 40, 12), 7) and tol == 1e-10
    pos = 44
    for tag in (b"00", b"1x", b"1y", b"1z", b"2x", b"2y", b"2z"):
        assert b[pos:pos + 2] == tag
        d = struct.unpack_from("<3Q", b, pos + 2)
        pos += 2 + 24 + 8 * (sum(n * r for n, r in zip(nmax, d)) + d[0] * d[1] * d[2])
    assert pos == len(b) - 4
    assert struct.unpack_from("<I", b, pos)[0] == zlib.crc32(b[:pos])


def test_corrupt_cache_is_refused(svh_lib, cache_file, tmp_path):
    """One flipped payload byte fails the CRC-32 (SPEC S:214 'checksum mismatch')."""
    b = bytearray(open(cache_file, "rb").read())
    b[len(b) // 2] ^= 0x40
    bad = tmp_path / "flipped.svxt"
    bad.write_bytes(bytes(b))
    case = svh_inputs.random_fill((8, 8, 4), fill=0.5, seed=1)
    with pytest.raises(svh_lib.SvhError, match="checksum"):
        svh_lib.setup_case(case, kernel_cache=str(bad))
