"""Pins for oracle/tucker.py (Algorithm 1, Eq. 10-11) -- CPU only."""
import numpy as np
import pytest

from oracle import kernels, tucker


def test_mode_product_properties():
    """Eq. 11: identity factor leaves T unchanged; all-ones row sums a mode (SPEC examples);
    (T x_i A) x_i B = T x_i (B A); products on different modes commute."""
    g = np.random.default_rng(0)
    T = g.standard_normal((3, 4, 5))
    for m in range(3):
        assert np.allclose(tucker.mode_product(T, np.eye(T.shape[m]), m), T)
    ones = np.ones((2, 2, 2))
    s = tucker.mode_product(ones, np.ones((1, 2)), 0)
    assert s.shape == (1, 2, 2) and np.all(s == 2)
    A, B = g.standard_normal((6, 4)), g.standard_normal((2, 6))
    assert np.allclose(tucker.mode_product(tucker.mode_product(T, A, 1), B, 1), tucker.mode_product(T, B @ A, 1))
    C, D = g.standard_normal((7, 3)), g.standard_normal((2, 5))
    assert np.allclose(tucker.mode_product(tucker.mode_product(T, C, 0), D, 2),
                       tucker.mode_product(tucker.mode_product(T, D, 2), C, 0))
    # one explicit entry (definition): V[v, j, k] = sum_i T[i, j, k] F[v, i]
    V = tucker.mode_product(T, C, 0)
    assert abs(V[4, 2, 3] - sum(T[i, 2, 3] * C[4, i] for i in range(3))) < 1e-13


def test_rank_one_and_constructed():
    """SPEC tucker examples: u(x)v(x)w -> ranks (1,1,1) exact; C0 x_i F_i with orthonormal
    factors (core 2x3x4) -> ranks (2,3,4) at tol 1e-10, exact reconstruction."""
    g = np.random.default_rng(1)
    u, v, w = g.standard_normal(5), g.standard_normal(6), g.standard_normal(7)
    T = np.einsum("i,j,k->ijk", u, v, w)
    C, F = tucker.tucker_svd(T, 1e-10)
    assert C.shape == (1, 1, 1)
    assert np.allclose(tucker.reconstruct(C, F), T, atol=1e-13 * np.abs(T).max())
    C0 = g.standard_normal((2, 3, 4))
    Fs = [np.linalg.qr(g.standard_normal((n, r)))[0] for n, r in [(8, 2), (9, 3), (10, 4)]]
    T = tucker.reconstruct(C0, Fs)
    C, F = tucker.tucker_svd(T, 1e-10)
    assert C.shape == (2, 3, 4)
    assert np.linalg.norm(tucker.reconstruct(C, F) - T) < 1e-12 * np.linalg.norm(T)
    for Fi in F:
        assert np.allclose(Fi.T @ Fi, np.eye(Fi.shape[1]), atol=1e-12)


@pytest.mark.parametrize("tol", [1e-4, 1e-6, 1e-8])
def test_kernel_compression_within_tol(tol):
    """Alg. 1 guarantee ||O - O_hat||_F <= tol ||O||_F on a real kernel (K0, 24^3 offsets),
    with a compression far below dense (P:91 'Tucker compressible')."""
    n = 24
    offs = np.array([(x, y, z) for x in range(n) for y in range(n) for z in range(n)])
    K0 = kernels.seven_kernels(offs)[:, 0].reshape(n, n, n)
    O = tucker.weighted_toeplitz(K0)
    C, F = tucker.tucker_svd(O, tol)
    err = np.linalg.norm(tucker.reconstruct(C, F) - O) / np.linalg.norm(O)
    assert err <= tol
    assert C.size + sum(f.size for f in F) < 0.3 * O.size   # 24^3 is small; CR grows with Kt


def test_weighted_toeplitz_equals_circulant_and_spectrum_error():
    """Reading G8, pinned with numpy FFT: the relative Frobenius error of a truncated
    Tucker representation is the same for the weighted Toeplitz tensor, the embedded
    circulant and its 3-D DFT (Parseval), and the mode-wise ranks coincide."""
    K = (6, 5, 4)
    offs = np.array([(x, y, z) for x in range(K[0]) for y in range(K[1]) for z in range(K[2])])
    K1x = kernels.seven_kernels(offs)[:, 1].reshape(K)      # odd along x
    N = (12, 10, 8)
    circ = tucker.embed_circulant(K1x, N, odd=(True, False, False))
    O = tucker.weighted_toeplitz(K1x)
    assert np.isclose(np.linalg.norm(O), np.linalg.norm(circ), rtol=1e-13)
    spec = np.fft.fftn(circ)
    assert np.isclose(np.linalg.norm(spec), np.sqrt(np.prod(N)) * np.linalg.norm(circ), rtol=1e-12)
    # rank-truncate the Toeplitz representation, embed -> same error in circulant and spectrum
    C, F = tucker.tucker_svd(O, 1e-3)
    Oh = tucker.reconstruct(C, F)
    w = [np.where(np.arange(k) == 0, 1.0, np.sqrt(2.0)) for k in K]
    Th = Oh / (w[0][:, None, None] * w[1][None, :, None] * w[2][None, None, :])
    circ_h = tucker.embed_circulant(Th, N, odd=(True, False, False))
    e_t = np.linalg.norm(Oh - O) / np.linalg.norm(O)
    e_c = np.linalg.norm(circ_h - circ) / np.linalg.norm(circ)
    e_s = np.linalg.norm(np.fft.fftn(circ_h) - spec) / np.linalg.norm(spec)
    assert abs(e_t - e_c) < 1e-12 and abs(e_c - e_s) < 1e-12
    # mode ranks of the weighted Toeplitz tensor == numerical ranks of the circulant unfoldings
    for i in range(3):
        s_t = np.linalg.svd(tucker.unfold(O, i), compute_uv=False)
        s_c = np.linalg.svd(tucker.unfold(circ, i), compute_uv=False)
        assert np.allclose(np.sort(s_t)[::-1][:K[i]], np.sort(s_c)[::-1][:K[i]], rtol=1e-10, atol=1e-14)


def test_ranks_nearly_constant_with_size():
    """the maximum multilinear rank stays nearly constant as Kt grows (<= 3 apart)."""
    ranks = []
    for n in (12, 24):
        offs = np.array([(x, y, z) for x in range(n) for y in range(n) for z in range(n)])
        K0 = kernels.seven_kernels(offs)[:, 0].reshape(n, n, n)
        C, F = tucker.tucker_svd(tucker.weighted_toeplitz(K0), 1e-6)
        ranks.append(max(C.shape))
    assert abs(ranks[0] - ranks[1]) <= 3, ranks


def test_embed_circulant_odd_sign_pinned():
    """Reading G7 for an odd kernel, pinned to values the parity assumption does not produce:
    every entry of the embedding of K1x (odd along x, even along y, z) equals the kernel
    integrated directly at the SIGNED offset m (oracle quadrature at negative m_x), and the
    circulant product reproduces the direct linear convolution y_l = sum_k K1x(l - k) I_k
     -- a flipped sign or a transposed offset fails both."""
    K = (4, 3, 2)
    N = (8, 6, 4)
    offs = np.array([(x, y, z) for x in range(K[0]) for y in range(K[1]) for z in range(K[2])])
    K1x = kernels.seven_kernels(offs)[:, 1].reshape(K)
    circ = tucker.embed_circulant(K1x, N, odd=(True, False, False))
    signed = np.array([(x, y, z) for x in range(-K[0] + 1, K[0]) for y in range(-K[1] + 1, K[1])
                       for z in range(-K[2] + 1, K[2])])
    direct = kernels.seven_kernels(signed)[:, 1]
    for m, val in zip(signed, direct):
        assert np.isclose(circ[m[0] % N[0], m[1] % N[1], m[2] % N[2]], val, rtol=1e-12, atol=1e-16)
    assert np.any(direct < 0) and np.any(direct > 0)
    # the spectrum of an x-odd, y/z-even real sequence is purely imaginary
    spec = np.fft.fftn(circ)
    assert np.max(np.abs(spec.real)) < 1e-13 * np.max(np.abs(spec.imag))
    # circulant product == direct linear convolution over the grid
    rng = np.random.default_rng(3)
    I = rng.standard_normal(K) + 1j * rng.standard_normal(K)
    pad = np.zeros(N, dtype=complex)
    pad[:K[0], :K[1], :K[2]] = I
    y_fft = np.fft.ifftn(np.fft.fftn(pad) * spec)[:K[0], :K[1], :K[2]]
    table = {tuple(m): v for m, v in zip(signed, direct)}
    y_dir = np.zeros(K, dtype=complex)
    for l in np.ndindex(*K):
        for k in np.ndindex(*K):
            y_dir[l] += table[(l[0] - k[0], l[1] - k[1], l[2] - k[2])] * I[k]
    assert np.allclose(y_fft, y_dir, rtol=1e-12, atol=1e-15)
