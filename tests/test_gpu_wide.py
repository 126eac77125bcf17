"""Many-orbital variants of the correction-step kernels vs the CPU oracle.

The cfg4/cfg5 orbital counts (N = 21, 120) switch several kernels to their wide forms: the interleaved SpMM with
a column tail mask (N not a multiple of the lane-group width), the staged orbital-parallel projection (N >= 8),
the warp-per-tet squared-density load (N >= 32) and the one-warp-per-eigenvalue multisection (N * nev >= 4 * SMs).
Orbitals here are seeded smooth fields (zero on the boundary) on the reference's correction-test fixture
(proj/tests/test_correction.cpp:25-55); identities checked are the same as tests/test_gpu_correction.py's.
"""
import numpy as np
import pytest

import paper_2103_02824_b200 as kb
from oracle import OMesh, Oracle

pytestmark = pytest.mark.gpu

ATOMS = [[2.0, 0.31, -0.17, 0.05]]


class Wide:
    def __init__(self, ctx, N, hartree=True, xc="lda"):
        self.h = kb.Hierarchy()
        self.orc = Oracle(ATOMS, n_pairs=N, occ=1.0, xc=xc, hartree=hartree, xc_on=xc != "none")
        a, b = kb.Mesh.box([-5.0] * 3, [5.0] * 3, 4), OMesh.box([-5.0] * 3, [5.0] * 3, 4)
        self.h.push(a)
        self.orc.push(b)
        a, b = a.uniform_refine(), b.uniform_refine()
        self.h.push(a)
        self.orc.push(b)
        self.lev = 1
        self.L = kb.Level(ctx, self.h, self.lev)
        self.L.set_system(ATOMS, n_pairs=N, occupancy=1.0, xc=xc, hartree=hartree, xc_on=xc != "none")
        self.L.level_ops()
        self.ctx, self.N = ctx, N
        self.interior = self.L.index("interior")
        xyz = a.array("xyz")
        rng = np.random.default_rng(1000 + N)
        u = (xyz + 5.0) / 10.0  # unit cube coordinates; sin(pi k u) vanishes on the boundary
        orb = np.zeros((self.L.n, N))
        for i in range(N):
            k = rng.integers(1, 4, 3)
            orb[:, i] = np.prod(np.sin(np.pi * k * u), axis=1) * rng.uniform(0.5, 1.5)
        self.orb = orb
        self.lam = np.sort(rng.uniform(-1.0, -0.2, N))

    def dev(self, a):
        return self.ctx.to_device(np.ascontiguousarray(a))


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("N", [12, 21, 40])
def test_wide_sqload_and_blocks(ctx, N):
    c = Wide(ctx, N)
    Phi = c.dev(c.orb[c.interior])
    sq = ctx.empty(c.L.ni)
    c.L.sqload(Phi, sq)
    assert rel(sq.download(), c.orc.sqload(c.lev, c.orb)[c.interior]) < 1e-13
    rho_o = c.orc.density(c.orb)
    vxc_o = c.orc.xc_potential(rho_o)
    bc_o = c.orc.boundary_values(c.lev, c.orc.moments(c.lev, rho_o))
    wt_o, _ = c.orc.hartree_exact(c.lev, c.orb, bc_o, tol=1e-12)
    bnd = np.setdiff1d(np.arange(c.L.n), c.interior)
    ell = np.zeros(c.L.n)
    ell[bnd] = bc_o[bnd]
    c.L.prepare_blocks(Phi, c.dev(wt_o - ell), c.dev(ell), c.dev(vxc_o))
    B = c.orc.prepare_blocks(c.lev, c.orb, wt_o, vxc_o, bc_o)
    for name in ["A_H1", "A_H3", "A_H4", "A_h4", "b_H1", "b_H3", "b_H4", "rhs", "c_Hh", "d_phi", "beta1", "beta3",
                 "beta4", "gamma", "zeta_phi"]:
        g, o = c.L.blocks(name), B.get(name)
        assert g.shape == o.shape, name
        assert np.abs(g - o).max() <= 1e-11 * max(1e-300, np.abs(o).max()), name


@pytest.mark.parametrize("N", [12, 21, 40])
def test_wide_outer_solve(ctx, N):
    """orbital block BVP: tail-masked interleaved SpMM (N = 12: 4x4 lanes of 16; 21 odd; 40: 16x4 of 64)"""
    c = Wide(ctx, N)
    rho_o = c.orc.density(c.orb)
    vxc_o = c.orc.xc_potential(rho_o)
    w = np.zeros(c.L.n)
    ld = N + (N & 1)  # device blocks keep an even leading dimension; odd N carries one pad column
    Phi = np.zeros((c.L.ni, ld))
    Phi[:, :N] = c.orb[c.interior]
    PhiT = ctx.empty((c.L.ni, ld))
    att, its, md = c.L.outer_solve(c.dev(w), c.dev(vxc_o), c.lam, c.dev(Phi), PhiT, tol_linear=1e-12)
    ph_o, att_o, its_o, sig_o = c.orc.outer_solve(c.lev, w, vxc_o, c.lam, c.orb, tol=1e-12)
    assert list(att) == list(att_o)
    assert rel(PhiT.download()[:, :N], ph_o[c.interior]) < 1e-8


def test_wide_inner_sweep_many_eigenvalues(ctx):
    """N = 40 orbitals on n_H = 27: nev = 28, 1120 (orbital, k) multisection items -> one warp per eigenvalue.
    Hartree off, so the inner iteration is a single sweep on both sides (proj/src/correction.cpp:360)."""
    N = 40
    c = Wide(ctx, N, hartree=False, xc="none")
    zero = np.zeros(c.L.n)
    c.L.prepare_blocks(c.dev(c.orb[c.interior]), c.dev(zero), c.dev(zero), c.dev(zero))
    g = c.L.inner_scf(c.lam)
    B = c.orc.prepare_blocks(c.lev, c.orb, zero, zero, zero, hartree_on=False)
    o = B.inner_scf(c.lam)
    assert g["iterations"] == o["iterations"] == 1
    assert np.abs(g["lambda_"] - o["lambda_"]).max() <= 1e-9 * np.abs(o["lambda_"]).max()
    assert rel(g["theta2"], o["theta2"]) < 1e-7
    assert rel(g["phi_H"], o["phi_H"]) < 1e-7


def test_prepare_blocks_gemm_form_matches_per_tet_kernel(ctx):
    """The aggregated projection (KSB_PROJ_GEMM=1: per-chunk coefficient sums, FP64 DMMA products) gives the same
    ledger as the per-tet kernel (itself pinned to the oracle's prepare_blocks, proj/src/correction.cpp:148-150,
    173-194) on a refined level, N = 40"""
    import os

    import numpy as np

    import paper_2103_02824_b200 as kb

    atoms = [[2.0, 0.31, -0.17, 0.05]]
    N = 40
    h = kb.Hierarchy()
    a = kb.Mesh.box([-5.0] * 3, [5.0] * 3, 4)
    h.push(a)
    for _ in range(2):
        a = a.uniform_refine()
        h.push(a)
    L = kb.Level(ctx, h, 2)
    L.set_system(atoms, n_pairs=N)
    L.level_ops()
    it = L.index("interior")
    rng = np.random.default_rng(17)
    orb = np.zeros((L.n, N))
    orb[it] = rng.standard_normal((L.ni, N))
    wt = np.zeros(L.n)
    wt[it] = rng.standard_normal(L.ni)
    ell = np.sin(np.arange(L.n) * 0.1)
    vxc = -np.abs(np.cos(np.arange(L.n) * 0.07))
    out = {}
    for g in ("0", "1"):
        os.environ["KSB_PROJ_GEMM"] = g
        try:
            L.prepare_blocks(ctx.to_device(np.ascontiguousarray(orb[it])), ctx.to_device(wt), ctx.to_device(ell),
                             ctx.to_device(vxc))
            out[g] = {k: L.blocks(k) for k in ("A_h4", "rhs", "b_H1", "b_H3", "b_H4", "c_Hh", "d_phi", "beta1", "beta3",
                                               "beta4", "gamma", "zeta_phi")}
        finally:
            os.environ.pop("KSB_PROJ_GEMM", None)
    for k in out["0"]:
        x, y = out["1"][k], out["0"][k]
        assert np.linalg.norm(x - y) <= 1e-11 * max(np.linalg.norm(y), 1e-300), k
    L.close()
