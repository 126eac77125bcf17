"""Host mesh pipeline vs the oracle's restatement: index data must be bit-exact.

Cases follow the reference's mesh tests (proj/tests/test_mesh.cpp:21-131): box counts,
uniform refinement, empty/full/single/random adaptive markings, hierarchy child maps.
"""
import numpy as np
import pytest

import paper_2103_02824_b200 as kb
from oracle import OMesh

ARRAYS = ["xyz", "tets", "tuple", "tag", "parent", "vparent", "on_boundary", "boundary_faces", "interior_faces",
          "interior_face_tets"]


def same(a, b):
    for k in ARRAYS:
        x, y = a.array(k), b.array(k)
        assert x.shape == y.shape, k
        assert np.array_equal(x, y), k
    assert a.sizes()[:6] == b.sizes()[:6]


def test_box_counts_and_bitexact():
    for lo, hi, n in [([0, 0, 0], [1, 1, 1], 1), ([-1, -1, -1], [1, 1, 1], 2), ([-10, -10, -10], [10, 10, 10], 8),
                      ([-3, -2, -1], [4, 5, 6], 3)]:
        a, b = kb.Mesh.box(lo, hi, n), OMesh.box(lo, hi, n)
        same(a, b)
        assert a.n_tets == 6 * n ** 3
        assert b.conforming()
    m2 = kb.Mesh.box([-1] * 3, [1] * 3, 2)
    assert len(m2.array("boundary_faces")) == 2 * 6 * 4  # proj/tests/test_mesh.cpp:42


def test_uniform_refine_bitexact():
    a, b = kb.Mesh.box([0] * 3, [1] * 3, 1), OMesh.box([0] * 3, [1] * 3, 1)
    for k in range(3):
        a, b = a.uniform_refine(), b.uniform_refine()
        same(a, b)
        assert b.conforming()
    assert a.n_tets == 6 * 8 ** 3
    assert abs(b.total_volume() - 1.0) < 1e-12


def test_adapt_refine_empty_full_single():
    a0, b0 = kb.Mesh.box([-1] * 3, [1] * 3, 2), OMesh.box([-1] * 3, [1] * 3, 2)
    same(a0.adapt_refine([]), b0.adapt_refine([]))
    assert np.array_equal(a0.adapt_refine([]).array("parent"), np.arange(a0.n_tets))
    allm = np.arange(a0.n_tets)
    a, b = a0.adapt_refine(allm), b0.adapt_refine(allm)
    same(a, b)
    assert b.conforming()
    assert np.all(np.bincount(a.array("parent"), minlength=a0.n_tets) >= 2)
    a, b = a0.adapt_refine([17]), b0.adapt_refine([17])
    same(a, b)
    assert b.conforming() and abs(b.total_volume() - 8.0) < 1e-12


def test_random_adaptive_sequence_bitexact():
    # proj/tests/test_mesh.cpp:104-120 style: 15 rounds of random markings (numpy generator, documented)
    rng = np.random.default_rng(7)
    a, b = kb.Mesh.box([0] * 3, [1] * 3, 1), OMesh.box([0] * 3, [1] * 3, 1)
    for r in range(15):
        marks = np.unique(rng.integers(0, a.n_tets, 1 + r % 4))
        a, b = a.adapt_refine(marks), b.adapt_refine(marks)
        same(a, b)
        assert b.conforming()
        assert abs(b.total_volume() - 1.0) < 1e-12
    assert a.level == 15


def test_marked_out_of_range_is_invalid_argument():
    a = kb.Mesh.box([0] * 3, [1] * 3, 1)
    with pytest.raises(kb.KsbError) as e:
        a.adapt_refine([6])
    assert e.value.code == "invalid-argument"


def test_hierarchy_prolongation_bitexact():
    from oracle import Oracle
    lo, hi = [-2.0] * 3, [2.0] * 3
    h = kb.Hierarchy()
    orc = Oracle([[1.0, 0, 0, 0]])
    a, b = kb.Mesh.box(lo, hi, 2), OMesh.box(lo, hi, 2)
    h.push(a)
    orc.push(b)
    a, b = a.uniform_refine(), b.uniform_refine()
    h.push(a)
    orc.push(b)
    rng = np.random.default_rng(3)
    for k in range(3):
        marks = rng.integers(0, a.n_tets, 4)
        a, b = a.adapt_refine(marks), b.adapt_refine(marks)
        h.push(a)
        orc.push(b)
    for lev in range(h.n_levels):
        c1, v1 = h.prolongation(lev)
        c2, v2 = orc.prolongation(lev)
        assert np.array_equal(c1, c2) and np.array_equal(v1, v2), lev
