"""Binary hierarchy / state dumps (include/ksb.h ksb_hier_save ...): lossless round trips, corruption detection.
Host-only (no device). The reference has no binary format; its text outputs are unaffected."""
import numpy as np
import pytest

import paper_2103_02824_b200 as kb

ARRAYS = ["xyz", "tets", "tuple", "tag", "parent", "vparent", "on_boundary", "boundary_faces", "interior_faces",
          "interior_face_tets", "interior_face_geom"]


def hierarchy():
    h = kb.Hierarchy()
    m = kb.Mesh.box([-2.0, -1.0, -3.0], [2.0, 1.5, 3.0], 3)
    h.push(m)
    m = m.uniform_refine()
    h.push(m)
    rng = np.random.default_rng(5)
    for _ in range(2):
        m = m.adapt_refine(np.sort(rng.choice(m.n_tets, 25, replace=False)).astype(np.int32))
        h.push(m)
    return h


def test_hierarchy_round_trip(tmp_path):
    h = hierarchy()
    p = tmp_path / "h.ksbh"
    h.save(p)
    g = kb.Hierarchy.load(p)
    assert g.n_levels == h.n_levels
    for a, b in zip(h.meshes, g.meshes):
        assert a.sizes() == b.sizes()
        for name in ARRAYS:
            assert np.array_equal(a.array(name), b.array(name)), name
    for k in range(h.n_levels):
        ca, va = h.prolongation(k)
        cb, vb = g.prolongation(k)
        assert np.array_equal(ca, cb) and np.array_equal(va, vb)
    # refinement continues identically from a loaded mesh
    marks = np.arange(0, h.meshes[-1].n_tets, 7, dtype=np.int32)
    ra, rb = h.meshes[-1].adapt_refine(marks), g.meshes[-1].adapt_refine(marks)
    assert np.array_equal(ra.array("tets"), rb.array("tets"))


def test_mesh_round_trip_and_corruption(tmp_path):
    m = kb.Mesh.box([-1.0] * 3, [1.0] * 3, 2).uniform_refine()
    p = tmp_path / "m.ksbh"
    m.save(p)
    n = kb.Mesh.load(p)
    for name in ARRAYS:
        assert np.array_equal(m.array(name), n.array(name)), name
    raw = bytearray(p.read_bytes())
    raw[len(raw) // 2] ^= 0x40
    bad = tmp_path / "bad.ksbh"
    bad.write_bytes(bytes(raw))
    with pytest.raises(kb.KsbError) as e:
        kb.Mesh.load(bad)
    assert e.value.code == "io"
    short = tmp_path / "short.ksbh"
    short.write_bytes(p.read_bytes()[:100])
    with pytest.raises(kb.KsbError, match="truncated"):
        kb.Mesh.load(short)
    with pytest.raises(kb.KsbError) as e:
        kb.Mesh.load(tmp_path / "missing.ksbh")
    assert e.value.code == "io"
    # a hierarchy file with several levels is not a single mesh
    hp = tmp_path / "h.ksbh"
    hierarchy().save(hp)
    with pytest.raises(kb.KsbError, match="holds 4 meshes"):
        kb.Mesh.load(hp)


def test_state_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    lam = rng.standard_normal(3)
    Phi = np.zeros((50, 4))
    Phi[:, :3] = rng.standard_normal((50, 3))
    w = rng.standard_normal(70)
    p = tmp_path / "s.ksbs"
    kb.save_state(p, 2, lam, Phi, w)
    s = kb.load_state(p)
    assert s["level"] == 2
    assert np.array_equal(s["lambdas"], lam)
    assert np.array_equal(s["Phi"], Phi[:, :3])
    assert np.array_equal(s["w"], w)
    with pytest.raises(kb.KsbError, match="not a KSBHIER"):
        kb.Mesh.load(p)
