"""BASELINE configs[2..4] (cfg3 H2O-like N = 5, cfg4 ring N = 21, cfg5 C60-like sphere N = 120) on their own
estimator-driven adaptive hierarchies (workloads.adaptive_hierarchy: device residual indicators, host Doerfler marks,
adapt_refine), cut at a size the oracle finishes in seconds.

* the oracle rebuilds every level from the device's marks: meshes bit-exact (proj/src/mesh.cpp adapt_refine);
* one correction step (proj/src/driver.cpp:106-150) from the same seeded state on both sides, with a fixed number of
  inner sweeps (the synthetic state is not self-consistent, so the inner loop is bounded the same way on both):
  shift-ladder attempts identical, eigenvalues 1e-8, density / Hartree potential / separated orbitals 1e-6.

bench.py runs the same comparison on the sample level of the full-size hierarchies (parity_sample).
"""
import numpy as np
import pytest

import paper_2103_02824_b200 as kb
from oracle import OMesh, Oracle
from paper_2103_02824_b200 import workloads

pytestmark = pytest.mark.gpu

SWEEPS = 3


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name,target", [("cfg3", 3.0e4), ("cfg4", 2.0e4), ("cfg5", 6.0e3)])
def test_adaptive_config_step_matches_oracle(ctx, name, target):
    gen, N, box, _ = workloads.ADAPTIVE_CONFIGS[name]
    atoms = getattr(workloads, gen)()
    cen = [a[1:] for a in atoms]
    h, meshes, L, recs, marks = workloads.adaptive_hierarchy(ctx, atoms, N, box, target)
    assert len(meshes) >= 3 and len(marks) == len(meshes) - 1
    assert 0.5 * target <= L.n <= 2.0 * target
    k = len(meshes) - 1
    orc = Oracle(atoms, n_pairs=N, occ=2.0, xc="lda")
    om = OMesh.box([-box] * 3, [box] * 3, 8)
    orc.push(om)
    for j in range(k):
        om = om.adapt_refine(marks[j])
        orc.push(om)
    assert np.array_equal(om.array("tets"), meshes[k].array("tets"))
    assert np.array_equal(om.array("xyz"), meshes[k].array("xyz"))
    it = L.index("interior")
    assert np.array_equal(it, orc.interior(k))

    lam0 = np.linspace(-1.5, -0.3, N)
    _, Phi, w, ld = workloads.synthetic_start_device(L, ctx, meshes[k], cen, N, zeta=1.0)
    orb = np.zeros((L.n, N))
    orb[it] = Phi.download()[:, :N]
    w0 = w.download()
    lam = lam0.copy()
    lg = L.correction_step(lam, Phi, w, ld=ld, fixed_sweeps=SWEEPS)
    lam_o, orb_o, w_o, lo = orc.correction_step(k, lam0.copy(), orb, w0, fixed_sweeps=SWEEPS)
    assert lg["attempts"] == lo["attempts"]
    assert lg["inner_iterations"] == lo["inner_iterations"] == SWEEPS
    assert np.abs(lam - lam_o).max() <= 1e-8 * np.abs(lam_o).max()
    P = Phi.download()[:, :N]
    O = orb_o[it]
    assert rel(2.0 * (P ** 2).sum(1), 2.0 * (O ** 2).sum(1)) <= 1e-6
    assert rel(w.download(), w_o) <= 1e-6
    for i in range(N):
        gap = min(abs(lam_o[i] - lam_o[j]) for j in range(N) if j != i)
        if gap > 1e-3:
            s = np.sign(P[:, i] @ O[:, i])
            assert rel(s * P[:, i], O[:, i]) <= 1e-6, (name, i)
    L.close()
