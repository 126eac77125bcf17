"""GPU diagnostic: correction steps on a cfg1 level from the synthetic start (paper_2103_02824_b200.workloads)."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2103_02824_b200 as kb  # noqa: E402
from paper_2103_02824_b200.workloads import cfg1_hierarchy, synthetic_start  # noqa: E402

lev = int(sys.argv[1]) if len(sys.argv) > 1 else 3
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
h = cfg1_hierarchy(lev)
ctx = kb.Context(0)
L = kb.Level(ctx, h, lev)
L.set_system([[2.0, 0, 0, 0]], n_pairs=1, occupancy=2.0, xc="lda")
L.level_ops()
t = time.time()
lam, Phi, w, ld = synthetic_start(L, ctx, h.meshes[lev], [[0, 0, 0]], 1)
print("start", time.time() - t, lam, flush=True)
for s in range(steps):
    try:
        lg = L.correction_step(lam, Phi, w)
    except kb.KsbError as e:
        print("step", s, "failed", e, flush=True)
        break
    print(json.dumps({"step": s, "lambda": lam.tolist(), "inner": lg["inner_iterations"], "delta": lg["delta"],
                      "ms": [round(lg[k], 3) for k in ("ms_bvp", "ms_hartree", "ms_project", "ms_inner", "ms_total")],
                      "cg": lg["cg_iterations"], "att": lg["attempts"]}), flush=True)
    if lg["delta"] < 1e-6:
        break

# per-kernel breakdown of one more step
NAMES = ["cg_coop", "spmm", "cg_update_r", "cg_update_px", "cg_trueres", "cg_setup", "inner_tridiag", "inner:gemm", "inner:gemv",
         "inner:orbital_border", "inner:border_pre", "inner:border_q", "inner:arrow_eig", "inner:arrow_vec", "inner:select", "inner:hartree_delta",
         "inner:coarse_wmass", "inner:build_", "inner:symmetrize", "inner:coarse_sq", "inner:coarse_vec_asm",
         "inner:border_scale", "inner:schur", "project", "project_asm", "assemble", "axpby", "sqload", "rho_vxc",
         "moments", "elementwise", "lift", "norm", "reduce", "expand"]
ctx.reset_counters()
ctx.set_profiling(True)
try:
    lg = L.correction_step(lam, Phi, w)
    print("profiled step: inner", lg["inner_iterations"], "ms_total", round(lg["ms_total"], 3))
except kb.KsbError as e:
    print("profiled step failed", e)
ctx.set_profiling(False)
rows = []
for n in NAMES:
    ms, cnt = ctx.kernel_time(n)
    if cnt:
        rows.append((ms, n, cnt))
for ms, n, cnt in sorted(rows, reverse=True):
    print(f"  {n:24s} {ms:9.3f} ms  {cnt:5d} launches  {1e3 * ms / cnt:8.1f} us/launch")
