"""Standard multilevel correction (the reference's comparison method) on the device vs the oracle.

driver::solve_level_mlc (proj/src/driver.cpp:200-302) on the correction-test fixture
(proj/tests/test_correction.cpp:25-55): Z=2 nucleus, two orbitals, coarse box + one uniform refinement (and an
adaptive variant), warm start = the oracle's coarse SCF prolonged to the fine level. Tolerances as the north star:
eigenvalues 1e-8 relative, orbitals / density / Hartree potential 1e-6 relative L2 after sign alignment.
"""
import numpy as np
import pytest

import paper_2103_02824_b200 as kb
from paper_2103_02824_b200.driver import run, solve_level_mlc

from test_gpu_correction import ATOMS, Case, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("xc,hartree,adapt", [("lda", True, 0), ("lda", True, 2), ("none", False, 0)])
def test_solve_level_mlc_matches_oracle(ctx, xc, hartree, adapt):
    c = Case(ctx, xc=xc, hartree=hartree, adapt=adapt)
    lam = c.lam.copy()
    Phi = c.dev(c.phi_block(c.orb))
    w = c.dev(c.w)
    rho = ctx.empty((c.L.n,))
    res = solve_level_mlc(c.L, lam, Phi, w, tol_outer=1e-6, level=c.lev, rho=rho, tol_linear=1e-12)
    lo, oo, wo, ro, do = c.orc.solve_level_mlc(c.lev, c.lam, c.orb, c.w, tol_outer=1e-6, tol_linear=1e-12)
    assert res.outer_iterations == len(do)
    assert np.abs(lam - lo).max() <= 1e-8 * np.abs(lo).max(), (lam, lo)
    P = Phi.download()
    sgn = np.sign(np.sum(P * oo[c.interior], axis=0))
    assert rel(P * sgn, oo[c.interior]) < 1e-6
    assert rel(rho.download(), ro) < 1e-6
    if hartree:
        assert rel(w.download(), wo) < 1e-6
    else:
        assert not np.any(w.download())
    np.testing.assert_allclose(res.deltas, do, rtol=1e-5)


def test_mlc_sweep_needs_begin(ctx):
    c = Case(ctx)
    Phi = c.dev(c.phi_block(c.orb))
    with pytest.raises(kb.KsbError, match="before mlc_begin"):
        c.L.mlc_sweep(c.lam.copy(), Phi)
    # a correction step in between invalidates a begun MLC level (it reuses the work buffers)
    w = c.dev(c.w)
    c.L.mlc_begin(c.lam.copy(), Phi, w, tol_linear=1e-12)
    c.L.correction_step(c.lam.copy(), c.dev(c.phi_block(c.orb)), c.dev(c.w), tol_linear=1e-12)
    with pytest.raises(kb.KsbError, match="before mlc_begin"):
        c.L.mlc_sweep(c.lam.copy(), Phi)


def test_run_standard_mlc_mode(ctx):
    """driver::run with Mode::standard_mlc (proj/src/driver.cpp:381-384): coarse SCF, then MLC levels"""
    log = run(ctx, ATOMS, n_pairs=1, occupancy=2.0, xc="lda", box=5.0, n_coarse=4, max_levels=3, refine="uniform",
              mode="standard_mlc", tol_linear=1e-10)
    assert not log.aborted, log.abort_reason
    assert len(log.records) == 3
    assert all(r.outer_iterations >= 1 for r in log.records[1:])
    assert all(np.isfinite(r.lambdas).all() and np.isfinite(r.energy).all() for r in log.records)
