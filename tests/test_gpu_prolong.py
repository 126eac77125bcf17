"""Device one-level prolongation (ksb_prolong) vs the oracle's SpaceHierarchy::prolong, bit for bit.

The reference transfers the warm start with the step prolongation matrix (proj/src/fespace.cpp:35-56,76-84;
proj/src/driver.cpp:367-371). Hierarchy: a coarse box, one uniform refinement, two adaptive refinements with
seeded marks (bisection chains, so some new vertices have new parents).
"""
import numpy as np
import pytest

import paper_2103_02824_b200 as kb
from oracle import OMesh, Oracle

pytestmark = pytest.mark.gpu


def hierarchy(ctx):
    h = kb.Hierarchy()
    orc = Oracle([[1.0, 0.0, 0.0, 0.0]], n_pairs=1)
    a, b = kb.Mesh.box([-3.0] * 3, [3.0] * 3, 3), OMesh.box([-3.0] * 3, [3.0] * 3, 3)
    h.push(a)
    orc.push(b)
    a, b = a.uniform_refine(), b.uniform_refine()
    h.push(a)
    orc.push(b)
    rng = np.random.default_rng(7)
    for _ in range(2):
        marks = np.sort(rng.choice(a.n_tets, 40, replace=False)).astype(np.int32)
        a, b = a.adapt_refine(marks), b.adapt_refine(marks)
        h.push(a)
        orc.push(b)
    return h, orc


def test_prolong_full_and_interior_bitexact(ctx):
    h, orc = hierarchy(ctx)
    rng = np.random.default_rng(11)
    for lev in range(1, h.n_levels):
        L, P = kb.Level(ctx, h, lev), kb.Level(ctx, h, lev - 1)
        # full vertex layout, 3 columns (ld 4)
        x = rng.standard_normal((P.n, 4))
        y = ctx.empty((L.n, 4))
        L.prolong(ctx.to_device(x), y, False, False, ncols=3)
        ref = orc.prolong(x[:, :3], lev - 1, lev)
        assert np.array_equal(y.download()[:, :3], ref), lev
        # interior blocks (zero trace), 2 columns
        pi, li = P.index("interior"), L.index("interior")
        full = np.zeros((P.n, 2))
        full[pi] = rng.standard_normal((P.ni, 2))
        z = ctx.empty((L.ni, 2))
        L.prolong(ctx.to_device(np.ascontiguousarray(full[pi])), z, True, True)
        assert np.array_equal(z.download(), orc.prolong(full, lev - 1, lev)[li]), lev
        L.close()
        P.close()


def test_prolong_level0_is_an_error(ctx):
    h, _ = hierarchy(ctx)
    L = kb.Level(ctx, h, 0)
    x = ctx.empty((L.n,))
    with pytest.raises(kb.KsbError, match="hierarchy"):
        L.prolong(x, x, False, False)
