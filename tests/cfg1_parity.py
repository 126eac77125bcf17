"""cfg1 (BASELINE.json configs[0]): He, one doubly occupied orbital, LDA, [-10,10]^3, 8^3 coarse
Kuhn mesh, 3 uniform refinements. Runs the corrected level loop on the device (levels 1..L)
from the oracle's coarse SCF and, optionally, the oracle's own loop for comparison.

Used by tests/test_gpu_cfg1.py; runnable directly for a timing report:
    python tests/cfg1_parity.py --levels 3 --oracle-levels 2
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

ATOMS = [[2.0, 0.0, 0.0, 0.0]]
BOX = 10.0
N_COARSE = 8


def run(levels=3, oracle_levels=0, tol_outer=1e-6, verbose=True, dump_dir=""):
    import paper_2103_02824_b200 as kb
    from paper_2103_02824_b200.driver import prolong, solve_level_corrected
    from oracle import OMesh, Oracle

    out = {"gpu": [], "oracle": []}
    orc = Oracle(ATOMS, n_pairs=1, occ=2.0, xc="lda")
    h = kb.Hierarchy()
    a, b = kb.Mesh.box([-BOX] * 3, [BOX] * 3, N_COARSE), OMesh.box([-BOX] * 3, [BOX] * 3, N_COARSE)
    h.push(a)
    orc.push(b)
    for _ in range(levels):
        a, b = a.uniform_refine(), b.uniform_refine()
        h.push(a)
        orc.push(b)
    t = time.time()
    lam0, orb0, w0, scf_it = orc.coarse_scf(tol=tol_outer, mixing=0.3, tol_eig=1e-9)
    out["coarse"] = {"lambda": lam0.tolist(), "iterations": scf_it, "s": time.time() - t}
    if verbose:
        print("coarse SCF", out["coarse"], flush=True)

    ctx = kb.Context(0)
    lam = lam0.copy()
    orb, w = orb0.copy(), w0.copy()
    for lev in range(1, levels + 1):
        orb = prolong(h.meshes[lev], orb)
        w = prolong(h.meshes[lev], w)
        L = kb.Level(ctx, h, lev)
        L.set_system(ATOMS, n_pairs=1, occupancy=2.0, xc="lda")
        L.level_ops()
        it = L.index("interior")
        Phi = ctx.to_device(np.ascontiguousarray(orb[it]))
        dw = ctx.to_device(w)
        if dump_dir:
            np.savez(Path(dump_dir) / f"cfg1_start_level{lev}.npz", lam=lam, orb=orb, w=w)
        t = time.time()
        try:
            r = solve_level_corrected(L, lam, Phi, dw, tol_outer=tol_outer, level=lev)
        except kb.KsbError as e:
            part = getattr(e, "partial", None)
            rec = {"level": lev, "failed_step": getattr(e, "step", None), "error": str(e),
                   "deltas": part.deltas if part else [], "inner": part.inner_iterations if part else [],
                   "lambdas": [lg["lambda"] for lg in part.logs] if part else []}
            print("gpu level", lev, "failed:", json.dumps(rec), flush=True)
            out["gpu_error"] = rec
            break
        wall = time.time() - t
        e = L.energy(Phi, dw)
        rec = {"level": lev, "n": L.n, "ni": L.ni, "nnz": L.nnz_ii, "outer": r.outer_iterations,
               "inner": r.inner_iterations, "lambda": lam.tolist(), "energy": e.tolist(), "wall_s": wall,
               "step_ms": [lg["ms_total"] for lg in r.logs], "bvp_ms": [lg["ms_bvp"] for lg in r.logs],
               "hartree_ms": [lg["ms_hartree"] for lg in r.logs], "project_ms": [lg["ms_project"] for lg in r.logs],
               "inner_ms": [lg["ms_inner"] for lg in r.logs], "cg_iterations": [lg["cg_iterations"] for lg in r.logs],
               "attempts": [lg["attempts"] for lg in r.logs], "deltas": r.deltas,
               "lambdas": [lg["lambda"] for lg in r.logs]}
        out["gpu"].append(rec)
        if verbose:
            print("gpu", json.dumps(rec), flush=True)
        full = np.zeros((L.n, 1))
        full[it] = Phi.download()
        orb, w = full, dw.download()
        out.setdefault("finals", {})[lev] = {"orb": orb.copy(), "w": w.copy()}
        L.close()

    lam = lam0.copy()
    orb, w = orb0.copy(), w0.copy()
    for lev in range(1, oracle_levels + 1):
        orb = orc.prolong(orb, lev - 1, lev)
        w = orc.prolong(w, lev - 1, lev)[:, 0]
        t = time.time()
        logs = []
        for outer in range(40):
            lam, orb, w, lg = orc.correction_step(lev, lam, orb, w)
            logs.append(lg)
            if lg["delta"] < tol_outer:
                break
        e = orc.energy(lev, orb, w)
        rec = {"level": lev, "outer": len(logs), "inner": [lg["inner_iterations"] for lg in logs],
               "lambda": lam.tolist(), "energy": e.tolist(), "wall_s": time.time() - t,
               "step_s": [lg["t_total"] for lg in logs], "attempts": [lg["attempts"] for lg in logs],
               "deltas": [lg["delta"] for lg in logs]}
        out["oracle"].append(rec)
        if verbose:
            print("oracle", json.dumps(rec), flush=True)
    ctx.close()
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--oracle-levels", type=int, default=0)
    ap.add_argument("--json", default="")
    ap.add_argument("--dump", default="")
    a = ap.parse_args()
    res = run(a.levels, a.oracle_levels, dump_dir=a.dump)
    if a.json:
        Path(a.json).write_text(json.dumps(res, indent=1))
