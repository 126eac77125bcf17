"""Estimator-driven adaptive hierarchy for BASELINE configs[2..4] on the device (workloads.adaptive_hierarchy), then
one correction step on the finest level from the synthetic start: per-level and per-phase times.
Usage: python profiles/adaptive_probe.py cfg3 [target_dofs] [theta]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import torch  # noqa: E402,F401

import paper_2103_02824_b200 as kb  # noqa: E402
from paper_2103_02824_b200 import workloads  # noqa: E402

name = sys.argv[1]
gen, N, box, target = workloads.ADAPTIVE_CONFIGS[name]
if len(sys.argv) > 2:
    target = float(sys.argv[2])
theta = float(sys.argv[3]) if len(sys.argv) > 3 else 0.4
atoms = getattr(workloads, gen)()
ctx = kb.Context(0)
t0 = time.time()
h, meshes, L, recs, marks = workloads.adaptive_hierarchy(ctx, atoms, N, box, target, theta=theta,
                                                  log=lambda r: print(json.dumps(r), flush=True))
print("hierarchy_s", round(time.time() - t0, 1), "levels", len(meshes), flush=True)
t1 = time.time()
lam, Phi, w, ld = workloads.synthetic_start_device(L, ctx, meshes[-1], [a[1:] for a in atoms], N, zeta=1.0, lam0=-0.5)
lam = np.linspace(-1.5, -0.3, N)
print("start_s", round(time.time() - t1, 1), flush=True)
print("mem free/total GB", [round(x / 2**30, 1) for x in torch.cuda.mem_get_info()], flush=True)
for k in range(2):
    t2 = time.time()
    try:
        lg = L.correction_step(lam, Phi, w, ld=ld, fixed_sweeps=10)
    except kb.KsbError as e:
        print("step error", str(e)[:300])
        break
    ctx.sync()
    print(json.dumps({"step": k, "wall_s": round(time.time() - t2, 2)} | {kk: lg[kk] for kk in
          ("ms_bvp", "ms_hartree", "ms_project", "ms_inner", "ms_total", "cg_iterations", "inner_iterations")}
          | {"attempts": lg["attempts"][:8]}), flush=True)

# per-family CUDA-event times of one more step (the context's profiling counters; graphs are off while profiling)
import os  # noqa: E402

FAMS = ("assemble", "axpby", "rho_vxc", "moments", "bc", "sqload", "lift", "elementwise", "cg_setup", "spmm",
        "cg_update_r", "cg_update_px", "cg_trueres", "cg_coop", "mg", "project", "project_asm", "coarse",
        "inner_tridiag", "expand", "norm", "energy", "reduce")


def families(tag):
    ctx.sync()
    ctx.reset_counters()
    ctx.set_profiling(True)
    lg = L.correction_step(lam, Phi, w, ld=ld, fixed_sweeps=10)
    ctx.sync()
    ctx.set_profiling(False)
    fam = {}
    for nm in FAMS:
        ms, cnt = ctx.kernel_time(nm)
        if cnt:
            fam[nm] = {"ms": round(ms, 2), "launches": int(cnt), "avg_us": round(1e3 * ms / cnt, 1)}
    print(json.dumps({"tag": tag, "families": fam, "n_i": L.ni, "nnz": L.nnz_ii, "N": N, "ms_total": lg["ms_total"],
                      "ms_bvp": lg["ms_bvp"]}), flush=True)


if os.environ.get("KSB_PROBE_FAMILIES", "1") != "0":
    # KSB_PROBE_AB="NAME=v1,v2,...": one profiled step per value of an environment switch the library reads per launch
    ab = os.environ.get("KSB_PROBE_AB")
    if ab:
        name, vals = ab.split("=")
        for v in vals.split(","):
            os.environ[name] = v
            families(f"{name}={v}")
    else:
        families("default")
