"""Oracle: Tucker decomposition of the interaction tensors.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Eq. 10: O = C x1 F1 x2 F2 x3 F3.
* Eq. 11: i-mode product V = C x_i F, V[.., v, ..] = sum_i' C[.., i', ..] F[v, i'].
* Algorithm 1: for each mode, SVD of the mode-i unfolding of O,
  truncation at tol/sqrt(3), F_i = U_i, C = C x_i F_i^*.
  Reading G9: "index of maximum (normalized) value smaller than tol/sqrt(3)"
  is taken as the tail-energy rule sqrt(sum_{k>d} s_k^2)/||O||_F <= tol/sqrt(3),
  which guarantees ||O - O_hat||_F <= tol ||O||_F.  The SVD is numpy's direct
  SVD (not a Gram eigendecomposition, which cannot resolve s_k < sqrt(eps) s_1).
  Reading G10: F^* is the conjugate transpose.
* Reading G8: the circulant embedding and the DFT act mode-wise, so the Tucker
  ranks / relative Frobenius error of the embedded circulant (and of its
  spectrum) equal those of the Toeplitz tensor weighted by 1 at offset 0 and
  sqrt(2) elsewhere on every axis.  ``weighted_toeplitz`` builds that tensor.
"""
from __future__ import annotations

import numpy as np


def mode_product(T, F, mode: int):
    """Eq. 11: result[..., v, ...] = sum_i T[..., i, ...] F[v, i] along axis ``mode`` (0-based)."""
    Tm = np.moveaxis(T, mode, 0)
    out = np.tensordot(F, Tm, axes=([1], [0]))
    return np.moveaxis(out, 0, mode)


def unfold(T, mode: int):
    """Mode-i unfolding: rows indexed by the i-th index (D_i x prod of the others)."""
    return np.moveaxis(T, mode, 0).reshape(T.shape[mode], -1)


def truncation_rank(s, norm_o, tol):
    """Reading G9: smallest d with sqrt(sum_{k>d} s_k^2) <= tol/sqrt(3) * ||O||_F (d >= 1)."""
    tail = np.sqrt(np.maximum(np.cumsum((s ** 2)[::-1])[::-1], 0.0))   # tail[k] = ||s[k:]||
    thr = tol / np.sqrt(3.0) * norm_o
    for d in range(1, len(s) + 1):
        if d == len(s) or tail[d] <= thr:
            return d
    return len(s)


def tucker_svd(O, tol):
    """Algorithm 1. Returns (core, [F1, F2, F3])."""
    O = np.asarray(O)
    norm_o = np.linalg.norm(O.ravel())
    C = O.copy()
    F = []
    for i in range(3):
        U, s, _ = np.linalg.svd(unfold(O, i), full_matrices=False)   # line 5-6
        d = truncation_rank(s, norm_o, tol) if norm_o > 0 else 1        # line 7
        Fi = U[:, :d]
        F.append(Fi)
        C = mode_product(C, Fi.conj().T, i)                              # line 8
    return C, F


def reconstruct(C, F):
    """Eq. 10."""
    out = C
    for i in range(3):
        out = mode_product(out, F[i], i)
    return out


def weighted_toeplitz(T):
    """Reading G8: T (non-negative offsets, axes ordered as given) times 1 / sqrt(2) weights."""
    W = T.copy()
    for ax in range(3):
        w = np.full(T.shape[ax], np.sqrt(2.0))
        w[0] = 1.0
        shape = [1, 1, 1]
        shape[ax] = -1
        W = W * w.reshape(shape)
    return W


def embed_circulant(T, N, odd):
    """Circulant embedding (reading G7) of a non-negative-offset tensor with per-axis parity.

    T: (K1, K2, K3) values at m >= 0; N: embedding extents (>= 2K-1); odd[ax] True if the
    kernel is odd along that axis (T(-m) = -T(m) on that axis).  Index m -> m, -m -> N - m.
    """
    K = T.shape
    full = np.zeros(tuple(N))
    for idx in np.ndindex(*K):
        for signs in np.ndindex(2, 2, 2):
            m = [idx[a] * (1 if signs[a] == 0 else -1) for a in range(3)]
            if any(signs[a] == 1 and idx[a] == 0 for a in range(3)):
                continue
            val = T[idx]
            for a in range(3):
                if signs[a] == 1 and odd[a]:
                    val = -val
            full[tuple(m[a] % N[a] for a in range(3))] = val
    return full
