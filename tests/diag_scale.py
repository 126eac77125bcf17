"""GPU diagnostic: correction steps at cfg4/cfg5 orbital counts (N = 21, 120) on uniform Kuhn meshes, synthetic
start (one Gaussian-like orbital per center, columns beyond the centers get seeded polynomial factors),
fixed inner sweeps so the timing is defined whatever the inner dynamics do."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2103_02824_b200 as kb  # noqa: E402
from paper_2103_02824_b200.workloads import ring_atoms, sphere_atoms, synthetic_start  # noqa: E402


def run(name, atoms, N, box, refine, sweeps, steps=2, profile=True, ld=None):
    h = kb.Hierarchy()
    m = kb.Mesh.box([-box] * 3, [box] * 3, 8)
    h.push(m)
    for _ in range(refine):
        m = m.uniform_refine()
        h.push(m)
    ctx = kb.Context(0)
    L = kb.Level(ctx, h, refine)
    L.set_system(atoms, n_pairs=N, occupancy=2.0, xc="lda")
    t = time.time()
    L.level_ops()
    t_ops = time.time() - t
    cen = [a[1:] for a in atoms]
    lam, Phi, w, ld = synthetic_start(L, ctx, h.meshes[refine], cen, N, zeta=1.0, lam0=-0.5, ld=ld)
    lam = np.linspace(-1.5, -0.3, N)
    out = {"name": name, "N": N, "n_interior": L.ni, "ops_s": round(t_ops, 3), "steps": []}
    for s in range(steps):
        try:
            lg = L.correction_step(lam, Phi, w, ld=ld, fixed_sweeps=sweeps)
        except kb.KsbError as e:
            out["steps"].append({"error": str(e)[:200]})
            break
        out["steps"].append({k: round(lg[k], 3) for k in ("ms_bvp", "ms_hartree", "ms_project", "ms_inner", "ms_total")}
                            | {"cg": lg["cg_iterations"], "attempts": sorted(set(lg["attempts"]))})
    print(json.dumps(out), flush=True)
    if profile:
        ctx.reset_counters()
        ctx.set_profiling(True)
        try:
            L.correction_step(lam, Phi, w, ld=ld, fixed_sweeps=sweeps)
        except kb.KsbError:
            pass
        ctx.set_profiling(False)
        names = ["cg_coop", "spmm", "cg_update_r", "cg_update_px", "cg_trueres", "inner_tridiag", "inner:gemm",
                 "inner:gemv", "inner:border_pre", "inner:border_q", "inner:arrow_eig", "inner:arrow_vec",
                 "inner:select", "inner:hartree_delta", "inner:coarse_wmass", "inner:build_", "inner:coarse_sq",
                 "inner:coarse_vec_asm", "project", "project_asm", "assemble", "axpby", "sqload", "rho_vxc",
                 "elementwise", "norm", "expand", "moments"]
        rows = sorted(((ctx.kernel_time(n)[0], n, ctx.kernel_time(n)[1]) for n in names), reverse=True)
        for ms, n, cnt in rows[:14]:
            if cnt:
                print(f"  {n:24s} {ms:9.3f} ms {cnt:6d} launches", flush=True)
    L.close()
    ctx.close()


if __name__ == "__main__":
    cases = [("cfg4-like N=21, 250k dofs", ring_atoms(), 21, 25.0, 3, 10),
             ("cfg5-like N=120, 250k dofs", sphere_atoms(), 120, 30.0, 3, 10),
             ("cfg5-like N=120, 2.1M dofs", sphere_atoms(), 120, 30.0, 4, 10)]
    pick = [int(a) for a in sys.argv[1:]] or range(len(cases))
    for k in pick:
        run(*cases[k], steps=1 if len(sys.argv) > 1 else 2, profile=len(sys.argv) == 1)
