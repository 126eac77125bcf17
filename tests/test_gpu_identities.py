"""Identity tests of the device path that do not go through the oracle (the reference's own test strategy,
SURVEY.md §4): ledger nesting identities (proj/tests/test_correction.cpp:322-355), zero right-hand side
(:86-114), and bitwise determinism of reruns (the reference's results are independent of worker count;
proj/src/driver.cpp:475-507 -- here: fixed-order reductions, no floating-point atomics)."""
import numpy as np
import pytest

from test_gpu_correction import Case, rel

pytestmark = pytest.mark.gpu


def coarse_to_fine(c, U):
    """phi = P(0 -> level) U for coarse interior coefficient columns U (n_H x k); composite prolongation rows"""
    col, val = c.h.prolongation(c.lev)
    n0 = c.h.meshes[0].n_vertices
    ci = np.nonzero(~c.h.meshes[0].array("on_boundary").astype(bool))[0]
    full0 = np.zeros((n0, U.shape[1]))
    full0[ci] = U
    out = np.zeros((col.shape[0], U.shape[1]))
    for k in range(4):
        m = col[:, k] >= 0
        out[m] += val[m, k, None] * full0[col[m, k]]
    return out


@pytest.mark.parametrize("adapt", [0, 2])
def test_ledger_nesting_identities(ctx, adapt):
    """phi_tilde = P u: P^T M phi = M_H u, P^T S phi = C_H u, phi^T M phi = u^T M_H u, phi^T S phi = u^T C_H u"""
    c = Case(ctx, adapt=adapt)
    nh = c.L.nH
    U = np.random.default_rng(4).standard_normal((nh, c.N))
    phi = coarse_to_fine(c, U)
    zero = np.zeros(c.L.n)
    c.L.prepare_blocks(c.dev(c.phi_block(phi)), c.dev(zero), c.dev(zero), c.dev(zero))
    MH, CH = c.L.blocks("M_H"), c.L.blocks("C_H")
    assert np.abs(MH - MH.T).max() <= 1e-13 * np.abs(MH).max()
    for name in ("A_H1", "A_H3", "A_H4"):
        A = c.L.blocks(name)
        assert np.abs(A - A.T).max() <= 1e-13 * max(np.abs(A).max(), 1e-300), name
    Ah4 = c.L.blocks("A_h4")
    for i in range(c.N):
        assert np.abs(Ah4[i] - Ah4[i].T).max() <= 1e-13 * np.abs(Ah4[i]).max()
    cHh, dphi = c.L.blocks("c_Hh"), c.L.blocks("d_phi")
    gam, zet = c.L.blocks("gamma"), c.L.blocks("zeta_phi")
    for i in range(c.N):
        u = U[:, i]
        assert rel(cHh[i], MH @ u) < 1e-10
        assert rel(dphi[i], CH @ u) < 1e-10
        assert abs(gam[i] - u @ MH @ u) <= 1e-10 * abs(u @ MH @ u)
        assert abs(zet[i] - u @ CH @ u) <= 1e-10 * abs(u @ CH @ u)


def test_zero_orbital_gives_zero_correction(ctx):
    """bvp_orbital with phi = 0: the right-hand side vanishes and the solve returns exactly 0"""
    c = Case(ctx)
    vxc = c.orc.xc_potential(c.orc.density(c.orb))
    Phi = np.array(c.phi_block(c.orb))
    Phi[:, 1] = 0.0
    PhiT = ctx.empty((c.L.ni, c.N))
    att, its, _ = c.L.outer_solve(c.dev(c.w), c.dev(vxc), c.lam, c.dev(Phi), PhiT, tol_linear=1e-12)
    out = PhiT.download()
    assert np.all(out[:, 1] == 0.0) and its[1] == 0 and att[1] == -1
    assert np.linalg.norm(out[:, 0]) > 0


def test_correction_step_is_bitwise_deterministic(ctx):
    c = Case(ctx)
    res = []
    for _ in range(2):
        lam = c.lam.copy()
        Phi, w = c.dev(c.phi_block(c.orb)), c.dev(c.w)
        lg = c.L.correction_step(lam, Phi, w, tol_linear=1e-12)
        res.append((lam, Phi.download(), w.download(), lg["inner_iterations"], lg["delta"]))
    a, b = res
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1], b[1])
    assert np.array_equal(a[2], b[2])
    assert a[3] == b[3] and a[4] == b[4]
