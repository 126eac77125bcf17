"""K-ASM / K-SpMM / multi-RHS CG through the C-ABI vs the CPU oracle."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2103_02824_b200 as kb
from oracle import OMesh, Oracle

pytestmark = pytest.mark.gpu

ATOMS = np.array([[2.0, 0.31, -0.17, 0.05], [1.0, -0.6, 0.4, 0.9]])
GAUSS = np.array([[3.0, 0.8, 0.2, -0.1, 0.3], [1.5, 1.2, -0.9, 0.5, -0.4]])


def hierarchy(n=3, levels=1, adapt=0, lo=-4.0, hi=4.0, seed=5):
    h = kb.Hierarchy()
    orc = Oracle(ATOMS, n_pairs=2)
    a, b = kb.Mesh.box([lo] * 3, [hi] * 3, n), OMesh.box([lo] * 3, [hi] * 3, n)
    h.push(a)
    orc.push(b)
    for _ in range(levels):
        a, b = a.uniform_refine(), b.uniform_refine()
        h.push(a)
        orc.push(b)
    rng = np.random.default_rng(seed)
    for _ in range(adapt):
        marks = rng.integers(0, a.n_tets, 6)
        a, b = a.adapt_refine(marks), b.adapt_refine(marks)
        h.push(a)
        orc.push(b)
    return h, orc


def csr_of_oracle(op):
    ptr, idx, val = op.ii()
    A = sp.csc_matrix((val, idx, ptr), shape=(op.ni, op.ni)).tocsr()
    A.sort_indices()
    return A


@pytest.mark.parametrize("adapt", [0, 2])
def test_assembly_matches_oracle(ctx, adapt):
    h, orc = hierarchy(adapt=adapt)
    lev = h.n_levels - 1
    L = kb.Level(ctx, h, lev)
    w = np.sin(orc.meshes[lev].array("xyz") @ np.array([0.3, -0.2, 0.5]))
    dw = ctx.to_device(w)
    cases = [
        (dict(c_s=1.0), dict(c_s=1.0)),
        (dict(c_m=1.0), dict(c_m=1.0)),
        (dict(c_s=0.5, potential=(kb.POT_COULOMB, ATOMS)), dict(c_s=0.5, potential=(0, ATOMS))),
        (dict(potential=(kb.POT_GAUSSIAN, GAUSS)), dict(potential=(1, GAUSS))),
        (dict(w=dw), dict(w=w)),
    ]
    for gpu_kw, orc_kw in cases:
        L.assemble(kb.MAT_USER0, **gpu_kw)
        op = orc.operator(lev, **orc_kw)
        A = csr_of_oracle(op)
        assert np.array_equal(L.index("ii_ptr"), A.indptr), gpu_kw
        assert np.array_equal(L.index("ii_col"), A.indices), gpu_kw
        g = L.values(kb.MAT_USER0)
        scale = np.abs(A.data).max()
        assert np.abs(g - A.data).max() <= 1e-13 * scale, gpu_kw


def test_spmm_matches_oracle(ctx):
    h, orc = hierarchy(adapt=1)
    lev = h.n_levels - 1
    L = kb.Level(ctx, h, lev)
    L.assemble(kb.MAT_USER0, c_s=0.5, c_m=0.5, potential=(kb.POT_GAUSSIAN, GAUSS))
    op = orc.operator(lev, c_s=0.5, c_m=0.5, potential=(1, GAUSS))
    rng = np.random.default_rng(1)
    for N in [1, 2, 5, 16, 21, 64, 120]:
        ld = N if N == 1 else N + (N & 1)
        X = np.zeros((L.ni, ld))
        X[:, :N] = rng.standard_normal((L.ni, N))
        dX, dY = ctx.to_device(X), ctx.empty((L.ni, ld))
        L.spmm(kb.MAT_USER0, dX, dY, N, ld, ld)
        Y = dY.download()[:, :N]
        ref = np.stack([op.spmv(X[:, j]) for j in range(N)], 1)
        assert np.abs(Y - ref).max() <= 1e-12 * np.abs(ref).max(), N


@pytest.mark.parametrize("N", [1, 3, 4, 16, 24])
def test_cg_matches_oracle_jacobi(ctx, N):
    h, orc = hierarchy(adapt=1)
    lev = h.n_levels - 1
    L = kb.Level(ctx, h, lev)
    L.assemble(kb.MAT_USER0, c_s=0.5, c_m=2.0, potential=(kb.POT_COULOMB, ATOMS))
    op = orc.operator(lev, c_s=0.5, c_m=2.0, potential=(0, ATOMS), precond=1)
    rng = np.random.default_rng(2)
    B = rng.standard_normal((L.ni, N))
    if N > 1:
        B[:, 1] = 0.0  # zero right-hand side: converged with 0 iterations (proj/src/solver.cpp:62-66)
    X, st = L.cg_solve_host(kb.MAT_USER0, B, N, opts=L.cg_options(tol=1e-10))
    Xo, sto = op.pcg(B, tol=1e-10)
    for j in range(N):
        assert st[j].converged == sto[j]["converged"]
        assert abs(st[j].iterations - sto[j]["iterations"]) <= 1
    assert np.linalg.norm(X - Xo) <= 1e-9 * np.linalg.norm(Xo)
    if N > 1:
        assert st[1].iterations == 0 and st[1].converged and np.all(X[:, 1] == 0.0)


def test_t8_view_matches_csr(ctx):
    """The ELL-16 (T8) view of a Kuhn box mesh (<= 15 entries per row) holds every CSR row in order, padded
    with -1; refined levels with rows longer than 16 have none (and N = 16 solves take the CSR kernels)."""
    h, _ = hierarchy(n=12, levels=0)
    L = kb.Level(ctx, h, 0)
    ptr, col, t8 = L.index("ii_ptr"), L.index("ii_col"), L.index("t8_col").reshape(L.ni, 16)
    lens = np.diff(ptr)
    assert lens.max() <= 16
    for r in range(L.ni):
        assert np.array_equal(t8[r, :lens[r]], col[ptr[r]:ptr[r + 1]])
        assert np.all(t8[r, lens[r]:] == -1)
    ha, _ = hierarchy(adapt=2)
    La = kb.Level(ctx, ha, ha.n_levels - 1)
    if np.diff(La.index("ii_ptr")).max() > 16:
        with pytest.raises(RuntimeError):
            La.index("t8_col")


def test_locality_order(ctx):
    """Refined levels carry a locality order (interior rows by vertex z, y, x) that the multi-column CG runs on:
    a permutation whose pattern is the natural one renumbered and much narrower than the natural numbering; the
    reordered solve (N = 8: B, X permuted in and out) matches the oracle's Jacobi PCG."""
    h, orc = hierarchy(n=4, levels=2, adapt=1)
    lev = h.n_levels - 1
    L = kb.Level(ctx, h, lev)
    perm, lp, lc = L.index("lo_perm"), L.index("lo_ptr"), L.index("lo_col")
    ptr, col = L.index("ii_ptr"), L.index("ii_col")
    assert np.array_equal(np.sort(perm), np.arange(L.ni))
    iperm = np.empty_like(perm)
    iperm[perm] = np.arange(L.ni)
    bw_nat, bw_lo = 0, 0
    for i in range(L.ni):
        r = perm[i]
        assert np.array_equal(lc[lp[i]:lp[i + 1]], np.sort(iperm[col[ptr[r]:ptr[r + 1]]]))
        bw_lo += np.abs(lc[lp[i]:lp[i + 1]] - i).sum()
        bw_nat += np.abs(col[ptr[r]:ptr[r + 1]] - r).sum()
    assert bw_lo < 0.5 * bw_nat
    L.assemble(kb.MAT_USER0, c_s=0.5, c_m=0.5, potential=(kb.POT_GAUSSIAN, GAUSS))
    op = orc.operator(lev, c_s=0.5, c_m=0.5, potential=(1, GAUSS), precond=1)
    B = np.random.default_rng(11).standard_normal((L.ni, 8))
    # the order is used for blocks above 48 MB; KSB_CG_REORDER=2 forces it on this small one
    os.environ["KSB_CG_REORDER"] = "2"
    try:
        X, st = L.cg_solve_host(kb.MAT_USER0, B, 8, opts=L.cg_options(tol=1e-10))
    finally:
        del os.environ["KSB_CG_REORDER"]
    Xo, sto = op.pcg(B, tol=1e-10)
    for j in range(8):
        assert st[j].converged == sto[j]["converged"]
        assert abs(st[j].iterations - sto[j]["iterations"]) <= 1
    assert np.linalg.norm(X - Xo) <= 1e-9 * np.linalg.norm(Xo)


@pytest.mark.parametrize("N", [16, 32])
def test_cg_streamed_spmm_uniform(ctx, N):
    """Kuhn box meshes (rows of <= 15 entries, like cfg2) take the T8 SpMM (k_spmm_t8) at N = 16 and the
    streamed quad-layout SpMM (k_spmm_stream) at N = 32; same iterations and solution as the oracle's Jacobi
    PCG."""
    h, orc = hierarchy(n=14, levels=0)
    lev = 0
    L = kb.Level(ctx, h, lev)
    L.assemble(kb.MAT_USER0, c_s=0.5, c_m=0.5, potential=(kb.POT_GAUSSIAN, GAUSS))
    op = orc.operator(lev, c_s=0.5, c_m=0.5, potential=(1, GAUSS), precond=1)
    rng = np.random.default_rng(9)
    B = rng.standard_normal((L.ni, N))
    X, st = L.cg_solve_host(kb.MAT_USER0, B, N, opts=L.cg_options(tol=1e-10))
    Xo, sto = op.pcg(B, tol=1e-10)
    for j in range(N):
        assert st[j].converged == sto[j]["converged"]
        assert abs(st[j].iterations - sto[j]["iterations"]) <= 1
    assert np.linalg.norm(X - Xo) <= 1e-9 * np.linalg.norm(Xo)


def test_cg_breakdown_on_indefinite_operator(ctx):
    """a_op alone is indefinite (bound states): CG stops with breakdown like the reference."""
    h, orc = hierarchy(levels=1)
    L = kb.Level(ctx, h, 1)
    L.assemble(kb.MAT_USER0, c_s=0.5, potential=(kb.POT_COULOMB, 30 * ATOMS[:1]))
    op = orc.operator(1, c_s=0.5, potential=(0, 30 * ATOMS[:1]), precond=1)
    rng = np.random.default_rng(4)
    B = rng.standard_normal((L.ni, 2))
    X, st = L.cg_solve_host(kb.MAT_USER0, B, 2, opts=L.cg_options(tol=1e-10, max_iterations=3000))
    Xo, sto = op.pcg(B, tol=1e-10, maxit=3000)
    for j in range(2):
        assert st[j].breakdown == sto[j]["breakdown"]
        assert st[j].converged == sto[j]["converged"]
        if sto[j]["breakdown"]:
            assert st[j].iterations == sto[j]["iterations"]


def test_cg_fixed_iterations_and_shifts(ctx):
    """Per-column shifted operators A + sigma_j M (the level-shift ladder's dual-value SpMM)."""
    h, orc = hierarchy()
    L = kb.Level(ctx, h, 1)
    L.assemble(kb.MAT_AOP, c_s=0.5, potential=(kb.POT_COULOMB, ATOMS))
    L.assemble(kb.MAT_M, c_m=1.0)
    rng = np.random.default_rng(6)
    N = 3
    B = rng.standard_normal((L.ni, N))
    Bp = np.ascontiguousarray(np.pad(B, ((0, 0), (0, 1))))  # ld = 4 > N
    sig = np.array([3.0, 5.0, 8.0])  # lowest pencil eigenvalue is about -2.18: all shifted operators SPD
    X, st = L.cg_solve_host(kb.MAT_AOP, Bp, N, ld=4, opts=L.cg_options(tol=1e-11), shift_mat=kb.MAT_M, sigma=sig)
    for j in range(N):
        op = orc.operator(1, c_s=0.5, potential=(0, ATOMS), c_m=sig[j], precond=1)
        xo, so = op.pcg(B[:, j], tol=1e-11)
        assert st[j].converged and so[0]["converged"]
        assert abs(st[j].iterations - so[0]["iterations"]) <= 1
        assert np.linalg.norm(X[:, j] - xo[:, 0]) <= 1e-9 * np.linalg.norm(xo)
    # fixed-iteration benchmark mode runs exactly k iterations, no stopping test (indefinite shift included)
    sig = np.array([1.0, 2.5, 4.0])
    for k in (1, 2, 7):
        X, st = L.cg_solve_host(kb.MAT_AOP, Bp, N, ld=4, opts=L.cg_options(fixed_iterations=k), shift_mat=kb.MAT_M,
                                sigma=sig)
        assert all(s.iterations == k for s in st)
        for j in range(N):
            op = orc.operator(1, c_s=0.5, potential=(0, ATOMS), c_m=sig[j], precond=1)
            xo, so = op.pcg(B[:, j], fixed=k)
            # column 0 is indefinite (sigma below the spectrum): CG amplifies rounding there
            tol = 1e-10 if (k <= 2 or j > 0) else 1e-6
            assert np.linalg.norm(X[:, j] - xo[:, 0]) <= tol * np.linalg.norm(xo), (k, j)
