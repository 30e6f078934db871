"""SuperVoxHenry fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct restatement of what the
paper (arXiv 2105.08627, /root/reference/PAPER.md, cited as ``P:<line>``)
computes.  It exists only to check the CUDA path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2105_08627_b200``) never imports it, and it imports nothing from the
product path: the two share no code, headers, tables or constants.  Seeded
inputs come from ``svh_inputs`` (geometry + random numbers only, no method
arithmetic).

Modules
-------
kernels   Galerkin interaction integrals of the PWC/PWL voxel bases
          (Eq. 4-6, App. A, App. B).
lattice   voxel enumeration, face nodes, incidence matrix A.
operator  two-fluid local term (Eq. 3, 22-23), dense Z (Eq. 8) and the direct
          matrix-free product Z.I that Eq. 9 accelerates.
solve     saddle system Eq. 7 with port potentials, dense LU, Y -> Z -> L.
tucker    Algorithm 1 (Tucker-SVD / HOSVD) and Eq. 10-11.

Parity status per function is listed in DESIGN.md ("Oracle pins").
"""
