"""CPU-only: the oracle's own corrected level loop on cfg1 (BASELINE.json configs[0]), step by step.

Reference trajectory for the device loop in tests/cfg1_parity.py (same coarse SCF, same tolerances).
    python tests/cfg1_oracle.py --levels 3 --json out.json
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

from oracle import OMesh, Oracle, OracleError  # noqa: E402

ATOMS = [[2.0, 0.0, 0.0, 0.0]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--max-outer", type=int, default=40)
    ap.add_argument("--json", default="")
    ap.add_argument("--dump", default="")
    ap.add_argument("--final-npz", default="", help="save each converged level's final orbitals and w here")
    a = ap.parse_args()
    orc = Oracle(ATOMS, n_pairs=1, occ=2.0, xc="lda")
    m = OMesh.box([-10.0] * 3, [10.0] * 3, 8)
    orc.push(m)
    for _ in range(a.levels):
        m = m.uniform_refine()
        orc.push(m)
    lam, orb, w, it = orc.coarse_scf(tol=a.tol, mixing=0.3, tol_eig=1e-9)
    print("coarse", lam.tolist(), it, flush=True)
    out = []
    finals = {}
    for lev in range(1, a.levels + 1):
        orb = orc.prolong(orb, lev - 1, lev)
        w = orc.prolong(w, lev - 1, lev)[:, 0]
        if a.dump:
            np.savez(Path(a.dump) / f"oracle_start_level{lev}.npz", lam=lam, orb=orb, w=w)
        steps = []
        for outer in range(a.max_outer):
            t = time.time()
            try:
                lam, orb, w, lg = orc.correction_step(lev, lam, orb, w)
            except OracleError as e:
                print("level", lev, "step", outer, "failed:", e, flush=True)
                steps.append({"error": str(e)})
                break
            rec = {"lambda": lam.tolist(), "delta": lg["delta"], "inner": lg["inner_iterations"],
                   "attempts": lg["attempts"], "cg": lg["cg_iterations"], "s": time.time() - t}
            steps.append(rec)
            print("level", lev, "step", outer, json.dumps(rec), flush=True)
            if lg["delta"] < a.tol:
                break
        out.append({"level": lev, "steps": steps, "energy": orc.energy(lev, orb, w).tolist()})
        if a.final_npz and steps and "error" not in steps[-1]:
            finals[f"orb_level{lev}"] = orb
            finals[f"w_level{lev}"] = w
            np.savez_compressed(a.final_npz, **finals)
        if steps and "error" in steps[-1]:
            break
    if a.json:
        Path(a.json).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
