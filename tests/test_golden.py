"""Pins of the oracle against values the paper prints (tests/golden/, each file cites its source)."""
import json
import os

import numpy as np

from oracle import kernels

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _canonical(triple):
    # the source/test profile pair of an axis integrates to the same reduced kernel up to the
    # parity s -> -s (W01(s) = W10(-s)), so (a, b) and (b, a) are one Toeplitz tensor
    return tuple(tuple(sorted(p)) for p in triple)


def test_table2_storage_is_seven_kernels():
    """Table II: 112 B per voxel = 7 complex-double Toeplitz tensors.  The oracle's
    expansion of the 25 blocks of Eq. 8 must reduce to exactly 7 distinct reduced integrals
    (a dropped or extra term in the basis dot products would change the count)."""
    g = json.load(open(os.path.join(GOLDEN, "table2_toeplitz_memory.json")))
    per_voxel = [mb * 2 ** 20 / (L / g["dx_um"]) ** 3 for L, mb in zip(g["edge_um"], g["memory_MB"])]
    assert np.allclose(per_voxel, 112.0, atol=0.01)
    classes = {_canonical(tr) for tr in kernels.all_triples()}
    assert len(classes) == 7
    assert 7 * 16 == round(per_voxel[0])
    # and the zero blocks of Eq. 8: (x,y), (x,z), (y,z), (z,2D) and transposes
    for b, a in [("x", "y"), ("x", "z"), ("y", "z"), ("z", "2D")]:
        assert kernels.block_terms(b, a) == [] and kernels.block_terms(a, b) == []
