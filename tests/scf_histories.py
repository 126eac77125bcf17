"""Coarse-SCF density-change histories of BASELINE configs[2..4] in the CPU oracle (reference algorithm,
proj/src/scf.cpp:22-90), for the record in profiles/ (which coarse meshes the reference algorithm can start from).
Usage: python tests/scf_histories.py cfg3 8 [mixing] [max_it]"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import OMesh, Oracle  # noqa: E402
from paper_2103_02824_b200 import workloads  # noqa: E402

CFG = {"cfg3": (workloads.h2o_atoms, 5, 20.0), "cfg4": (workloads.ring_atoms, 21, 25.0),
       "cfg5": (workloads.sphere_atoms, 120, 30.0)}


def main():
    name, nc = sys.argv[1], int(sys.argv[2])
    mixing = float(sys.argv[3]) if len(sys.argv) > 3 else 0.3
    max_it = int(sys.argv[4]) if len(sys.argv) > 4 else 200
    gen, N, box = CFG[name]
    atoms = gen()
    orc = Oracle(atoms, n_pairs=N, occ=2.0, xc="lda")
    orc.push(OMesh.box([-box] * 3, [box] * 3, nc))
    t = time.time()
    err = None
    try:
        lam, _, _, it = orc.coarse_scf(tol=1e-6, max_it=max_it, mixing=mixing, tol_eig=1e-9)
    except Exception as e:  # noqa: BLE001
        err, lam = str(e)[:300], None
    hist = orc.last_scf_history()
    rec = {"config": name, "n_coarse": nc, "mixing": mixing, "max_it": max_it, "N": N, "box": box,
           "converged": err is None, "error": err, "iterations": len(hist), "wall_s": round(time.time() - t, 1),
           "lambdas": None if lam is None else [float(x) for x in lam], "history": [float(x) for x in hist]}
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
