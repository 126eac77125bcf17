"""Coarse-SCF density-change histories of BASELINE configs[2..4] on the device (ksb_coarse_scf, the reference's
scf::self_consistent_solve, proj/src/scf.cpp:22-90) for n_coarse = 8 (the configured mesh), 12 and 16 (the reference
default, proj/include/ksafem/runconfig.hpp:16): which coarse meshes the reference algorithm can start from.
The 8^3 oracle histories (tests/scf_histories.py, CPU) are in profiles/scf/.
Usage: python profiles/scf_device_histories.py [n_coarse ...]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2103_02824_b200 as kb  # noqa: E402
from paper_2103_02824_b200 import workloads  # noqa: E402

ncs = [int(x) for x in sys.argv[1:]] or [8, 12, 16]
ctx = kb.Context(0)
for name, (gen, N, box, _) in workloads.ADAPTIVE_CONFIGS.items():
    atoms = getattr(workloads, gen)()
    for nc in ncs:
        for mixing in (0.3, 0.1):
            h = kb.Hierarchy()
            h.push(kb.Mesh.box([-box] * 3, [box] * 3, nc))
            L = kb.Level(ctx, h, 0)
            t = time.time()
            rec = {"config": name, "n_coarse": nc, "n_coarse_interior": L.ni, "N": N, "mixing": mixing,
                   "max_it": 200}
            try:
                L.set_system(atoms, n_pairs=N, occupancy=2.0, xc="lda")
                L.level_ops()
                lam, Phi, rho, w, it, hist = L.coarse_scf(tol=1e-6, max_iterations=200, mixing=mixing)
                rec.update({"converged": True, "iterations": it, "lambdas": np.asarray(lam).tolist(),
                            "history": np.asarray(hist).tolist()})
            except kb.KsbError as e:
                rec.update({"converged": False, "error": str(e)[:200],
                            "history": np.asarray(getattr(L, "last_scf_history", [])).tolist()})
            rec["wall_s"] = round(time.time() - t, 1)
            L.close()
            print(json.dumps(rec), flush=True)
