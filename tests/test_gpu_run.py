"""The accelerated adaptive run end to end on the device (driver::run, proj/src/driver.cpp:306-435) vs the same
loop composed from the oracle's pieces: coarse SCF, residual indicators, Doerfler marks (theta = 0.4), adaptive
refinement, nested warm start, corrected level solves. Identical meshes at every level (the marks agree),
eigenvalues and total energy 1e-8 relative, indicator totals 1e-9.
"""
import numpy as np
import pytest

import paper_2103_02824_b200 as kb
from oracle import OMesh, Oracle, dorfler_mark
from paper_2103_02824_b200.driver import run

pytestmark = pytest.mark.gpu


def oracle_run(atoms, n_pairs, occ, xc, box, n_coarse, max_levels, theta=0.4, tol=1e-6):
    orc = Oracle(atoms, n_pairs=n_pairs, occ=occ, xc=xc)
    m = OMesh.box([-box] * 3, [box] * 3, n_coarse)
    orc.push(m)
    recs = []
    lam, orb, w, _ = orc.coarse_scf(tol=tol, mixing=0.3, tol_eig=1e-9)
    rho = orc.last_scf_rho()
    for level in range(max_levels):
        if level > 0:
            m = m.adapt_refine(dorfler_mark(eta, tot, theta))
            orc.push(m)
            orb = orc.prolong(orb, level - 1, level)
            w = orc.prolong(w, level - 1, level)[:, 0]
            for outer in range(40):
                lam, orb, w, lg = orc.correction_step(level, lam, orb, w)
                if lg["delta"] < tol:
                    break
            rho = orc.density(orb)
        vxc = orc.xc_potential(rho)
        eta, tot = orc.indicators(level, lam, orb, w, vxc)
        recs.append(dict(n=orc.n(level), nt=m.sizes()[1], lam=np.array(lam), energy=orc.energy(level, orb, w),
                         eta_total=tot))
    return recs


def test_adaptive_run_matches_oracle(ctx):
    atoms = [[2.0, 0.3, -0.2, 0.1]]
    log = run(ctx, atoms, 1, 2.0, "lda", 6.0, 4, 4, refine="adaptive")
    assert not log.aborted, log.abort_reason
    ref = oracle_run(atoms, 1, 2.0, "lda", 6.0, 4, 4)
    assert len(log.records) == len(ref)
    for r, o in zip(log.records, ref):
        assert r.n_dofs == o["n"] and r.n_tets == o["nt"], r.level
        assert np.abs(np.asarray(r.lambdas) - o["lam"]).max() <= 1e-8 * np.abs(o["lam"]).max(), r.level
        assert abs(r.energy[4] - o["energy"][4]) <= 1e-8 * abs(o["energy"][4]), r.level
        assert abs(r.eta_sq_total - o["eta_total"]) <= 1e-9 * o["eta_total"], r.level
