"""The reference's exact SGS preconditioner on the device (CgOptions::precond = 1, sgs.cu): parity mode.

EllipticSolver::apply_sgs + pcg (proj/src/solver.cpp:50-111) against the oracle's restatement (precond 0 = SGS):
* multi-column PCG on a refined and on an adaptive level, unshifted and shifted (A + sigma M, the level-shift
  ladder's operator, proj/src/correction.cpp:50-61): identical iteration counts, solutions within 1e-9;
* a whole correction step in SGS mode on the LiH adaptive fixture (tests/test_gpu_adaptive.py): the shift-ladder
  attempts and every orbital's CG iteration count identical to the oracle's, which runs the reference algorithm.
"""
import numpy as np
import pytest

import paper_2103_02824_b200 as kb
from oracle import OMesh, Oracle

from test_gpu_adaptive import LIH, near_marks

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def hierarchy(adaptive):
    atoms = np.array([[2.0, 0.31, -0.17, 0.05], [1.0, -1.6, 1.1, 0.4]])
    h = kb.Hierarchy()
    orc = Oracle(atoms, n_pairs=1)
    a, b = kb.Mesh.box([-6.0] * 3, [6.0] * 3, 6), OMesh.box([-6.0] * 3, [6.0] * 3, 6)
    h.push(a)
    orc.push(b)
    a, b = a.uniform_refine(), b.uniform_refine()
    h.push(a)
    orc.push(b)
    if adaptive:
        marks = near_marks(b.array("xyz"), b.array("tets"), atoms.tolist(), 2.0)
        a, b = a.adapt_refine(marks), b.adapt_refine(marks)
        h.push(a)
        orc.push(b)
    return atoms, h, orc, h.n_levels - 1


@pytest.mark.parametrize("adaptive", [False, True])
def test_sgs_pcg_matches_oracle(ctx, adaptive):
    atoms, h, orc, lev = hierarchy(adaptive)
    L = kb.Level(ctx, h, lev)
    # 1/2 S + M_ext + 4 M: positive definite (the Z = 2 well binds at -2)
    L.assemble(kb.MAT_USER0, c_s=0.5, c_m=4.0, potential=(kb.POT_COULOMB, atoms))
    op = orc.operator(lev, c_s=0.5, c_m=4.0, potential=(0, atoms), precond=0)  # oracle precond 0 = SGS
    B = np.random.default_rng(5).standard_normal((L.ni, 3))
    B[:, 1] = 0.0
    X, st = L.cg_solve_host(kb.MAT_USER0, B, 3, opts=L.cg_options(tol=1e-10, precond=1))
    Xo, sto = op.pcg(B, tol=1e-10)
    for j in range(3):
        assert st[j].converged and sto[j]["converged"]
        assert st[j].iterations == sto[j]["iterations"], (j, st[j].iterations, sto[j]["iterations"])
    assert st[1].iterations == 0 and np.all(X[:, 1] == 0.0)
    assert rel(X, Xo) <= 1e-9
    # the Jacobi production path takes more iterations to the same solution
    Xj, stj = L.cg_solve_host(kb.MAT_USER0, B, 3, opts=L.cg_options(tol=1e-10))
    assert rel(Xj, Xo) <= 1e-8 and stj[0].iterations > st[0].iterations
    L.close()


def test_sgs_shifted_operator(ctx):
    """A + sigma_j M per column (the shift ladder's dual-value operator) with an indefinite A: the unshifted SGS-PCG
    breaks down at the same iteration as the oracle's, the shifted ones converge in the same number of steps"""
    atoms, h, orc, lev = hierarchy(True)
    L = kb.Level(ctx, h, lev)
    L.assemble(kb.MAT_USER0, c_s=0.5, potential=(kb.POT_COULOMB, atoms))  # a_op = 1/2 S + M_ext: indefinite
    L.assemble(kb.MAT_USER0 + 1, c_m=1.0)
    sig = np.array([0.0, 3.0, 12.0])
    B = np.random.default_rng(9).standard_normal((L.ni, 3))
    X, st = L.cg_solve_host(kb.MAT_USER0, B, 3, opts=L.cg_options(tol=1e-10, precond=1), shift_mat=kb.MAT_USER0 + 1,
                            sigma=sig)
    for j, s in enumerate(sig):
        op = orc.operator(lev, c_s=0.5, c_m=s, potential=(0, atoms), precond=0)
        Xo, sto = op.pcg(B[:, j:j + 1], tol=1e-10)
        assert bool(st[j].breakdown) == bool(sto[0]["breakdown"]), j
        assert bool(st[j].converged) == bool(sto[0]["converged"]), j
        assert st[j].iterations == sto[0]["iterations"], (j, st[j].iterations, sto[0]["iterations"])
        if sto[0]["converged"]:
            assert rel(X[:, j], Xo[:, 0]) <= 1e-9
    L.close()


def test_correction_step_sgs_mode_matches_oracle_logs(ctx):
    atoms, N = LIH, 2
    h = kb.Hierarchy()
    orc = Oracle(atoms, n_pairs=N, occ=2.0, xc="lda")
    a, b = kb.Mesh.box([-8.0] * 3, [8.0] * 3, 8), OMesh.box([-8.0] * 3, [8.0] * 3, 8)
    h.push(a)
    orc.push(b)
    a, b = a.uniform_refine(), b.uniform_refine()
    h.push(a)
    orc.push(b)
    marks = near_marks(b.array("xyz"), b.array("tets"), atoms, 2.5)
    a, b = a.adapt_refine(marks), b.adapt_refine(marks)
    h.push(a)
    orc.push(b)
    lev = 2
    L = kb.Level(ctx, h, lev)
    L.set_system(atoms, n_pairs=N, occupancy=2.0, xc="lda")
    L.level_ops()
    it = L.index("interior")
    lam0, orb0, w0, _ = orc.coarse_scf(tol=1e-8, mixing=0.3)
    orb = orc.prolong(orb0, 0, lev)
    w = orc.prolong(w0, 0, lev)[:, 0]
    blk = np.ascontiguousarray(orb[it])
    Phi, dw = ctx.to_device(blk), ctx.to_device(w)
    lam_g, lam_o, orb_o, w_o = lam0.copy(), lam0.copy(), orb.copy(), w.copy()
    for outer in range(2):
        lg = L.correction_step(lam_g, Phi, dw, ld=N, precond=1)
        lam_o, orb_o, w_o, lo = orc.correction_step(lev, lam_o, orb_o, w_o)
        assert lg["attempts"] == lo["attempts"], outer
        assert lg["iterations"] == lo["cg_iterations"], (outer, lg["iterations"], lo["cg_iterations"])
        assert lg["hartree_iterations"] == lo["hartree_iterations"], outer
        assert np.abs(lam_g - lam_o).max() <= 1e-8 * np.abs(lam_o).max()
    P = Phi.download()
    O = orb_o[it]
    assert rel(2.0 * (P ** 2).sum(1), 2.0 * (O ** 2).sum(1)) <= 1e-6
    assert rel(dw.download(), w_o) <= 1e-6
    L.close()
