"""Diagnostics: per-kernel device time of correction steps (library event instrumentation)."""
import sys, time, json
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2103_02824_b200 as kb
from paper_2103_02824_b200.driver import prolong
from oracle import OMesh, Oracle

NAMES = ["spmm", "cg_update", "cg_trueres", "cg_setup", "assemble", "axpby", "elementwise", "rho_vxc", "moments",
         "bc", "sqload", "lift", "norm", "energy", "reduce", "project", "project_asm", "coarse", "inner_tridiag", "expand"] + ["inner:" + k for k in ["trsv_many", "border_scale", "schur", "coarse_wmass", "build_AH", "symmetrize", "orbital_border", "arrow_eig", "arrow_vec", "select", "coarse_sq", "coarse_vec_asm", "hartree_delta"]]
lev_target = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ATOMS = [[2.0, 0.0, 0.0, 0.0]]
orc = Oracle(ATOMS, n_pairs=1, occ=2.0, xc="lda")
h = kb.Hierarchy()
a, b = kb.Mesh.box([-10.0] * 3, [10.0] * 3, 8), OMesh.box([-10.0] * 3, [10.0] * 3, 8)
h.push(a); orc.push(b)
for _ in range(lev_target):
    a, b = a.uniform_refine(), b.uniform_refine(); h.push(a); orc.push(b)
lam, orb, w, _ = orc.coarse_scf(tol=1e-6, mixing=0.3)
for lev in range(1, lev_target + 1):
    orb = prolong(h.meshes[lev], orb); w = prolong(h.meshes[lev], w)
ctx = kb.Context(0)
L = kb.Level(ctx, h, lev_target)
L.set_system(ATOMS, n_pairs=1, occupancy=2.0, xc="lda"); L.level_ops()
it = L.index("interior")
Phi = ctx.to_device(np.ascontiguousarray(orb[it])); dw = ctx.to_device(w)
for k in range(3):
    ctx.reset_counters(); ctx.set_profiling(True)
    t = time.time(); lg = L.correction_step(lam, Phi, dw); wall = time.time() - t
    ctx.set_profiling(False)
    tab = {n: ctx.kernel_time(n) for n in NAMES}
    print(json.dumps({"step": k, "wall_ms": wall * 1e3, "log": {kk: (round(v, 3) if isinstance(v, float) else v) for kk, v in lg.items()},
                      "launches": ctx.launches(), "kernels_ms": {n: [round(v[0], 3), v[1]] for n, v in tab.items() if v[1]}}), flush=True)
