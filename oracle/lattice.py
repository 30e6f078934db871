"""Oracle: voxel lattice, face nodes and the incidence matrix A.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Domain of Kx x Ky x Kz voxels of edge dx, K non-empty voxels.
* Each non-empty voxel has 6 nodes at its face centres; shared faces are one
  node; M = number of unique nodes; N = 5K + M.
* A (M x 5K) is the incidence matrix of Eq. 7.  Its entries are
  deferred to [18] by the paper; reading G1/G12: A[r, (b,k)] is the
  outward flux of basis f^b_k through face r, with the G1 normalisation making
  it dimensionless (current in amperes).  Per basis (derived by integrating
  Eq. 4-6 over each face):
      f^x: -1 at -x face, +1 at +x face (same for y, z)
      f^2D: +1/2 at both x faces, -1/2 at both y faces
      f^3D: +1/2 at both x faces, +1/2 at both y faces, -1 at both z faces
  An interior face row sums the contributions of its two voxels.

Conventions shared with the public API (stated in include/svh.h):
  mat_id has shape (Kz, Ky, Kx) (x fastest); 0 = empty.
  Voxels are enumerated in flat x-fastest order of occupied cells.
  Nodes: x-faces, then y-faces, then z-faces; within a family, flat order over
  the face lattice (x-faces lattice (Kz, Ky, Kx+1), x fastest, etc.), keeping
  faces adjacent to at least one non-empty voxel.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

# flux of each basis (component order x, y, z, 2D, 3D) through the
# (-face, +face) of each axis; rows: basis, cols: (axis, side)
FLUX = {
    "x": {0: (-1.0, +1.0)},
    "y": {1: (-1.0, +1.0)},
    "z": {2: (-1.0, +1.0)},
    "2D": {0: (+0.5, +0.5), 1: (-0.5, -0.5)},
    "3D": {0: (+0.5, +0.5), 1: (+0.5, +0.5), 2: (-1.0, -1.0)},
}
BASES = ("x", "y", "z", "2D", "3D")


class Lattice:
    """Occupied voxels and unique face nodes of a voxel grid."""

    def __init__(self, mat_id):
        mat_id = np.asarray(mat_id)
        if mat_id.ndim != 3:
            raise ValueError("mat_id must be (Kz, Ky, Kx)")
        self.mat_id = mat_id
        self.Kz, self.Ky, self.Kx = mat_id.shape
        occ = mat_id != 0
        self.occ = occ
        kk, jj, ii = np.nonzero(occ)           # C order => x fastest
        self.coords = np.stack([ii, jj, kk], axis=1).astype(np.int64)  # (K,3) as (x,y,z)
        self.K = self.coords.shape[0]
        if self.K == 0:
            raise ValueError("zero non-empty voxels")
        self.voxel_mat = mat_id[kk, jj, ii]
        # face lattices: face (axis a) index along a runs 0..K_a (face between cells i-1, i)
        self.face_index = []   # per axis: array over face lattice, -1 if not a node
        next_id = 0
        for a in range(3):
            shp = [self.Kz, self.Ky, self.Kx]
            shp[2 - a] += 1
            # face i along axis a has cell i on its + side and cell i-1 on its - side
            # lo[..i..] = occ[..i-1..] (zero at i = 0); hi[..i..] = occ[..i..] (zero at i = K_a)
            lo = np.pad(occ, [(1, 0) if d == 2 - a else (0, 0) for d in range(3)])
            hi = np.pad(occ, [(0, 1) if d == 2 - a else (0, 0) for d in range(3)])
            present = lo | hi
            idx = -np.ones(shp, dtype=np.int64)
            n = int(present.sum())
            idx[present] = np.arange(next_id, next_id + n)
            next_id += n
            self.face_index.append(idx)
        self.M = next_id
        self.N = 5 * self.K + self.M

    def face_node(self, axis: int, cell_xyz, side: int):
        """Node id of the face of voxel cell_xyz (K,3) on the given side (-1/+1) of axis."""
        c = np.asarray(cell_xyz).copy()
        if side > 0:
            c[..., axis] += 1
        return self.face_index[axis][c[..., 2], c[..., 1], c[..., 0]]

    def incidence(self):
        """A as scipy CSR, shape (M, 5K); columns component-major."""
        rows, cols, vals = [], [], []
        ar = np.arange(self.K)
        for bi, b in enumerate(BASES):
            for axis, (fm, fp) in FLUX[b].items():
                for side, f in ((-1, fm), (+1, fp)):
                    rows.append(self.face_node(axis, self.coords, side))
                    cols.append(bi * self.K + ar)
                    vals.append(np.full(self.K, f))
        A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(self.M, 5 * self.K))
        return A.tocsr()  # duplicates (none within a column) summed per row entry
