"""K-PROJ timing on configs[4]'s adaptive hierarchy (N = 120) and on a uniform 12.6 M-tet level: correction steps with
the aggregated GEMM projection (default) and the per-tet kernel (KSB_PROJ_GEMM=0 in the environment).
Usage: python profiles/proj_probe.py [target_dofs]"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402,F401

import paper_2103_02824_b200 as kb  # noqa: E402
from paper_2103_02824_b200 import workloads  # noqa: E402

target = float(sys.argv[1]) if len(sys.argv) > 1 else 2e6
ctx = kb.Context(0)
gen, N, box, _ = workloads.ADAPTIVE_CONFIGS["cfg5"]
atoms = getattr(workloads, gen)()
cen = [a[1:] for a in atoms]


def run(L, mesh, tag):
    _, Phi, w, ld = workloads.synthetic_start_device(L, ctx, mesh, cen, N, zeta=1.0)
    phi0, w0 = Phi.download(), w.download()
    lam0 = np.linspace(-1.5, -0.3, N)
    for k in range(3):
        Phi.upload(phi0)
        w.upload(w0)
        lam = lam0.copy()
        t = time.time()
        lg = L.correction_step(lam, Phi, w, ld=ld, fixed_sweeps=3)
        print(json.dumps({"case": tag, "gemm": os.environ.get("KSB_PROJ_GEMM", "1"), "rep": k, "n": L.n, "tets": L.nt,
                          "ms_project": round(lg["ms_project"], 3), "ms_total": round(lg["ms_total"], 1),
                          "wall_s": round(time.time() - t, 2)}), flush=True)


h, meshes, L, recs, marks = workloads.adaptive_hierarchy(ctx, atoms, N, box, target)
run(L, meshes[-1], "cfg5-adaptive")
L.close()
h = kb.Hierarchy()
m = kb.Mesh.box([-box] * 3, [box] * 3, 8)
h.push(m)
for _ in range(4):
    m = m.uniform_refine()
    h.push(m)
L = kb.Level(ctx, h, 4)
L.set_system(atoms, n_pairs=N, occupancy=2.0, xc="lda")
L.level_ops()
run(L, m, "uniform-12.6M-tets")
