"""Union-tile ("UT") view and the wide-block SpMM built on it (k_spmm_ut, cg.cu; host/topology.hpp).

The multi-column CG on refined / adaptive levels (proj/src/solver.cpp:57-111 per column, all orbitals at once)
runs blocks of more than 16 columns through tiles of <= 4 spatially neighbouring rows whose distinct columns are
gathered once per tile (dense 4-vectors of values per column). Checked here:
* the view is a faithful re-tiling of the locality-ordered pattern (every row in exactly one tile, entries ascending
  and unique per tile, masks / value offsets / value map reproduce the CSR rows, limits respected);
* fixed-count and converged Jacobi-PCG solves through k_spmm_ut agree with the row kernel (KSB_SPMM_UT=0) and
  with the oracle, for full (N = 128, 64, 32), tail-masked (N = 120, 72, 40, 22) and odd (N = 67, 21) blocks --
  32, 16 and 8 lanes per tile --, with and without the
  per-column shift operator (the level-shift ladder's A + sigma_j M, proj/src/correction.cpp:50-61), on a uniformly
  refined and on an adaptively refined level.
"""
import os

import numpy as np
import pytest

import paper_2103_02824_b200 as kb
from oracle import OMesh, Oracle

pytestmark = pytest.mark.gpu

ATOMS = np.array([[2.0, 0.31, -0.17, 0.05], [1.0, -2.6, 1.4, 0.9]])


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def refined_pair(adaptive: bool):
    """8^3 Kuhn box refined twice uniformly, then (adaptive) four rounds of marks around the nuclei"""
    a, b = kb.Mesh.box([-6.0] * 3, [6.0] * 3, 8), OMesh.box([-6.0] * 3, [6.0] * 3, 8)
    h, orc = kb.Hierarchy(), Oracle(ATOMS, n_pairs=1)
    h.push(a)
    orc.push(b)
    for _ in range(2):
        a, b = a.uniform_refine(), b.uniform_refine()
        h.push(a)
        orc.push(b)
    if adaptive:
        for _ in range(4):
            xyz, tets = a.array("xyz"), a.array("tets")
            c = xyz[tets].mean(1)
            d = np.min(np.linalg.norm(c[:, None, :] - ATOMS[None, :, 1:], axis=2), axis=1)
            size = np.cbrt(np.abs(np.linalg.det(xyz[tets[:, 1:]] - xyz[tets[:, :1]])))
            marked = np.nonzero(size > 0.45 * (d + 0.25))[0].astype(np.int32)
            a, b = a.adapt_refine(marked), b.adapt_refine(marked)
            h.push(a)
            orc.push(b)
    return h, orc


@pytest.fixture(scope="module", params=["uniform", "adaptive"])
def level(request, ctx):
    h, orc = refined_pair(request.param == "adaptive")
    lev = h.n_levels - 1
    L = kb.Level(ctx, h, lev)
    L.assemble(kb.MAT_USER0, c_s=0.5, c_m=2.0, potential=(kb.POT_COULOMB, ATOMS))
    L.assemble(kb.MAT_M, c_m=1.0)
    op = orc.operator(lev, c_s=0.5, c_m=2.0, potential=(0, ATOMS), precond=1)
    yield L, op, request.param
    L.close()


def test_ut_view_is_a_retiling_of_the_ordered_pattern(level):
    L, _, kind = level
    nt, ne, R = (int(x) for x in L.index("ut_sizes"))
    assert nt > 0 and R == 4
    rows = L.index("ut_rows").reshape(nt, R)
    eptr = L.index("ut_eptr")
    ent = L.index("ut_ent")
    vmap = L.index("ut_map").reshape(ne, R)
    lo_ptr, lo_col, lo_map = L.index("lo_ptr"), L.index("lo_col"), L.index("lo_map")
    used = rows[rows >= 0]
    assert np.array_equal(np.sort(used), np.arange(L.ni))  # every ordered row in exactly one tile
    assert eptr[0] == 0 and eptr[-1] == ne
    assert np.all(np.diff(eptr) % 4 == 0) and np.diff(eptr).max() <= 64  # 16-byte aligned bulk copies, staging cap
    assert np.count_nonzero(vmap >= 0) == L.nnz_ii  # every nonzero exactly once
    assert np.array_equal(np.sort(vmap[vmap >= 0]), np.arange(L.nnz_ii))
    live_all = np.any(vmap >= 0, axis=1)
    assert np.all(ent >= 0) and np.all(ent < L.ni)  # padding entries gather a valid row
    rng = np.random.default_rng(3)
    for t in np.concatenate([[0, nt - 1], rng.integers(0, nt, 400)]):
        sl = slice(eptr[t], eptr[t + 1])
        live = live_all[sl]
        nl = int(np.count_nonzero(live))
        assert np.all(live[:nl]) and not np.any(live[nl:])  # padding last
        cols = ent[sl][:nl]
        assert np.all(np.diff(cols) > 0)  # ascending, unique
        tr = rows[t]
        assert np.all(np.diff(tr[tr >= 0]) > 0)
        for i in range(R):
            m = vmap[sl][:nl, i]
            if tr[i] < 0:
                assert np.all(m < 0)
                continue
            s = slice(lo_ptr[tr[i]], lo_ptr[tr[i] + 1])
            assert np.array_equal(cols[m >= 0], lo_col[s]) and np.array_equal(m[m >= 0], lo_map[s])
    if kind == "uniform":  # the point of the view: well under one gathered row per nonzero
        assert np.count_nonzero(live_all) / L.nnz_ii < 0.7


def solve(L, B, N, ut: bool, **kw):
    os.environ["KSB_CG_REORDER"] = "2"  # force the locality order (small blocks stay natural otherwise)
    os.environ["KSB_SPMM_UT"] = "2" if ut else "0"  # 2: also blocks of 17..64 columns (8 / 16 lanes per tile)
    try:
        return L.cg_solve_host(kb.MAT_USER0, B, N, **kw)
    finally:
        os.environ.pop("KSB_CG_REORDER", None)
        os.environ.pop("KSB_SPMM_UT", None)


@pytest.mark.parametrize("N", [128, 120, 72, 67, 64, 40, 32, 22, 21])
def test_ut_fixed_iterations_match_row_kernel_and_oracle(level, N):
    L, op, _ = level
    B = np.random.default_rng(N).standard_normal((L.ni, N))
    ld = N + (N & 1)
    Bp = np.zeros((L.ni, ld))
    Bp[:, :N] = B
    k = 6
    X1, st1 = solve(L, Bp, N, True, ld=ld, opts=L.cg_options(fixed_iterations=k))
    X0, st0 = solve(L, Bp, N, False, ld=ld, opts=L.cg_options(fixed_iterations=k))
    assert rel(X1[:, :N], X0[:, :N]) <= 1e-12
    cols = [0, N // 2, N - 1]
    Xo, sto = op.pcg(B[:, cols], fixed=k)
    assert rel(X1[:, cols], Xo) <= 1e-11
    for j, c in enumerate(cols):
        assert abs(st1[c].relative_residual - sto[j]["relative_residual"]) <= 1e-9 * sto[j]["relative_residual"]


@pytest.mark.parametrize("N", [96, 48, 21])
def test_ut_converged_solve_with_shift(level, N):
    """A + sigma_j M per column: the coefficient form (a + sigma_j b) x of k_spmm_ut against the row kernel's
    (sum a x) + sigma_j (sum b x)"""
    L, _, _ = level
    rng = np.random.default_rng(5)
    ld = N + (N & 1)
    B = np.zeros((L.ni, ld))
    B[:, :N] = rng.standard_normal((L.ni, N))
    sig = rng.uniform(1.0, 3.0, N)  # keeps every shifted operator definite on the adaptive level
    kw = dict(ld=ld, opts=L.cg_options(tol=1e-10), shift_mat=kb.MAT_M, sigma=sig)
    X1, st1 = solve(L, B, N, True, **kw)
    X0, st0 = solve(L, B, N, False, **kw)
    assert all(s.converged for s in st1)
    for a, b in zip(st1, st0):
        assert abs(a.iterations - b.iterations) <= 1
    assert rel(X1[:, :N], X0[:, :N]) <= 1e-8
    # residual of the shifted systems through the public SpMM (natural order, row kernel)
    dX = L.ctx.to_device(X1)
    dY, dZ = L.ctx.empty((L.ni, ld)), L.ctx.empty((L.ni, ld))
    L.spmm(kb.MAT_USER0, dX, dY, N, ld, ld)
    L.spmm(kb.MAT_M, dX, dZ, N, ld, ld)
    R = (B - dY.download() - dZ.download() * np.pad(sig, (0, ld - N))[None, :])[:, :N]
    assert np.max(np.linalg.norm(R, axis=0) / np.linalg.norm(B[:, :N], axis=0)) <= 5e-10
