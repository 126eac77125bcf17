"""Stencil (DIA) SpMM: the sliding-window kernel the CG takes on levels whose interior rows form a uniform stencil.

* a box mesh in its natural (lexicographic) order carries the Kuhn 15-point stencil (7 runs of offsets, centre
  {-1, 0, 1}); the cfg2 operator (BASELINE configs[1]) is such a level;
* a uniformly refined level sorted into the locality order carries the 27-point box stencil (9 runs of 3);
* adaptive levels have none (the CSR / T8 kernels stay).

Every lane-group variant (KSB_DIA_G = 4, 8, 16) is compared with the oracle's Jacobi PCG
(proj/src/solver.cpp:57-111 with Jacobi) and with the CSR kernels (KSB_SPMM_DIA=0) on the same device.
"""
import os

import numpy as np
import pytest

import paper_2103_02824_b200 as kb
from oracle import OMesh, Oracle

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def gauss():
    rng = np.random.default_rng(5)
    return np.column_stack([rng.uniform(1, 5, 4), rng.uniform(0.5, 1.5, 4), rng.uniform(-3, 3, (4, 3))])


class env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        for k, v in self.kv.items():
            os.environ[k] = str(v)

    def __exit__(self, *a):
        for k in self.kv:
            os.environ.pop(k, None)


@pytest.fixture(scope="module")
def box(ctx):
    n = 40  # 39^3 = 59,319 interior rows: ~7 tiles per warp of the resident grid at G = 16
    h = kb.Hierarchy()
    h.push(kb.Mesh.box([-10.0] * 3, [10.0] * 3, n))
    L = kb.Level(ctx, h, 0)
    L.assemble(kb.MAT_USER0, c_s=0.5, c_m=0.5, potential=(kb.POT_GAUSSIAN, gauss()))
    orc = Oracle([[1.0, 0.0, 0.0, 0.0]])
    orc.push(OMesh.box([-10.0] * 3, [10.0] * 3, n))
    op = orc.operator(0, c_s=0.5, c_m=0.5, potential=(1, gauss()), precond=1)
    yield L, op
    L.close()


def test_kuhn_stencil_detected(box):
    L, _ = box
    info = L.index("dia")
    m = 39
    assert list(info[:4]) == [7, 3, 2, 0]
    assert info[4] == -1
    assert sorted(info[5:11]) == sorted([-m * m - m - 1, -m * m - 1, -m - 1, m, m * m, m * m + m])


@pytest.mark.parametrize("G", [4, 8, 16])
def test_dia_cg_matches_oracle(ctx, box, G):
    L, op = box
    B = np.random.default_rng(G).standard_normal((L.ni, 16))
    B[:, 3] = 0.0
    with env(KSB_DIA_G=G):
        X, st = L.cg_solve_host(kb.MAT_USER0, B, 16, opts=L.cg_options(tol=1e-10, fixed_iterations=0))
        Xf, stf = L.cg_solve_host(kb.MAT_USER0, B, 16, opts=L.cg_options(fixed_iterations=7))
    with env(KSB_SPMM_DIA=0):
        Xc, stc = L.cg_solve_host(kb.MAT_USER0, B, 16, opts=L.cg_options(fixed_iterations=7))
    # indefinite (deep wells under a +0.5 M shift): columns may break down; both sides must agree
    Xo, sto = op.pcg(B, tol=1e-10)
    for j in range(16):
        assert bool(st[j].converged) == bool(sto[j]["converged"]), j
        assert bool(st[j].breakdown) == bool(sto[j]["breakdown"]), j
        assert abs(st[j].iterations - sto[j]["iterations"]) <= 1, (j, st[j].iterations, sto[j]["iterations"])
    assert st[3].iterations == 0 and np.all(X[:, 3] == 0.0)
    ok = [j for j in range(16) if sto[j]["converged"]]
    assert rel(X[:, ok], Xo[:, ok]) <= 1e-8
    # fixed-count iterations: stencil vs CSR kernels on the device (summation order differs only)
    assert rel(Xf, Xc) <= 1e-12
    Xof, _ = op.pcg(B, fixed=7)
    nz = [j for j in range(16) if j != 3]  # the oracle's fixed-count loop divides 0 / 0 on the zero column
    assert rel(Xf[:, nz], Xof[:, nz]) <= 1e-12


def test_box27_stencil_refined_level_locality_order(ctx):
    """8^3 Kuhn + 2 uniform refinements (29,791 rows, hierarchical numbering): the locality order is lexicographic
    on the refined grid, where the refined Kuhn cells carry the 27-point box stencil; N = 16 solves forced into the
    locality order (KSB_CG_REORDER=2) take the stencil kernel"""
    atoms = np.array([[2.0, 0.31, -0.17, 0.05]])
    h = kb.Hierarchy()
    orc = Oracle(atoms, n_pairs=1)
    a, b = kb.Mesh.box([-6.0] * 3, [6.0] * 3, 8), OMesh.box([-6.0] * 3, [6.0] * 3, 8)
    h.push(a)
    orc.push(b)
    for _ in range(2):
        a, b = a.uniform_refine(), b.uniform_refine()
        h.push(a)
        orc.push(b)
    L = kb.Level(ctx, h, 2)
    info = L.index("dia")
    assert list(info[:4]) == [9, 3, 3, 1]
    L.assemble(kb.MAT_USER0, c_s=0.5, c_m=2.0, potential=(kb.POT_COULOMB, atoms))
    op = orc.operator(2, c_s=0.5, c_m=2.0, potential=(0, atoms), precond=1)
    B = np.random.default_rng(4).standard_normal((L.ni, 16))
    for G in (8, 16):
        with env(KSB_CG_REORDER=2, KSB_DIA_G=G):
            X, st = L.cg_solve_host(kb.MAT_USER0, B, 16, opts=L.cg_options(tol=1e-10))
        Xo, sto = op.pcg(B, tol=1e-10)
        for j in range(16):
            assert st[j].converged and sto[j]["converged"]
            assert abs(st[j].iterations - sto[j]["iterations"]) <= 1
        assert rel(X, Xo) <= 1e-8
    L.close()


def test_adaptive_level_has_no_stencil(ctx):
    h = kb.Hierarchy()
    m = kb.Mesh.box([-4.0] * 3, [4.0] * 3, 4)
    h.push(m)
    marked = np.arange(0, m.n_tets, 7, dtype=np.int32)
    h.push(m.adapt_refine(marked))
    L = kb.Level(ctx, h, 1)
    assert L.index("dia")[0] == 0
    L.close()
