"""Per-phase view of one correction step on a uniformly refined level (default: 8^3 refined 4x = 2,048,383 interior
DOFs, 12.6 M tets, N = 120): CUDA-event time per kernel family (the context's profiling counters), algorithmic bytes
per family and the fraction of the measured HBM peak. The same command under
`ncu --kernel-id ::regex:<names>:2 --set full` gives one capture per kernel (profiles/r02_phase_capture.sh).

Usage: python profiles/phase_probe.py [refinements] [N] [steps]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402,F401

import paper_2103_02824_b200 as kb  # noqa: E402
from paper_2103_02824_b200 import workloads  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 4
N = int(sys.argv[2]) if len(sys.argv) > 2 else 120
STEPS = int(sys.argv[3]) if len(sys.argv) > 3 else 2
SWEEPS = 3

ctx = kb.Context(0)
atoms = workloads.sphere_atoms() if N >= 60 else workloads.ring_atoms() if N >= 12 else [[1.0, 0.0, 0.0, 0.0]]
cen = [a[1:] for a in atoms]
box = 10.0
h = kb.Hierarchy()
m = kb.Mesh.box([-box] * 3, [box] * 3, 8)
h.push(m)
for _ in range(R):
    m = m.uniform_refine()
    h.push(m)
L = kb.Level(ctx, h, R)
L.set_system(atoms, n_pairs=N, occupancy=2.0, xc="lda")
L.level_ops()
_, Phi, w, ld = workloads.synthetic_start_device(L, ctx, m, cen, N, zeta=1.0)
phi0, w0 = Phi.download(), w.download()
lam0 = np.linspace(-1.5, -0.3, N)

NAMES = ["assemble", "axpby", "rho_vxc", "moments", "bc", "sqload", "lift", "elementwise", "cg_setup", "spmm",
         "cg_update_r", "cg_update_px", "cg_trueres", "cg_coop", "mg", "project", "project_asm", "coarse",
         "inner_tridiag", "expand", "norm", "energy", "reduce"]
for k in range(STEPS):
    Phi.upload(phi0)
    w.upload(w0)
    ctx.sync()
    ctx.reset_counters()
    ctx.set_profiling(k == STEPS - 1)
    lg = L.correction_step(lam0.copy(), Phi, w, ld=ld, fixed_sweeps=SWEEPS)
    ctx.sync()
ctx.set_profiling(False)

ni, nt, nnz = L.ni, L.nt, L.nnz_ii
n_all = L.n
peak = json.load(open(Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json")) if (
    Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else {}


def find_peak(d):
    for k, v in d.items():
        if isinstance(v, dict):
            r = find_peak(v)
            if r:
                return r
        elif "hbm" in k.lower() and isinstance(v, (int, float)) and v > 1000:
            return float(v)
    return None


hbm = find_peak(peak) or 6500.0
# algorithmic bytes per LAUNCH of each family's main kernel
BYTES = {
    # one operator: 16 element values out per tet (128 B) + tets/xyz in (16 + ~12 B) ; gather: 128 B in per tet, 8 B/nnz out
    "assemble": None,
    "rho_vxc": 8.0 * ni * N + 16.0 * n_all,
    "sqload": 8.0 * ni * N + 16.0 * nt + 8.0 * n_all,
    "spmm": 12.0 * nnz + 4.0 * (ni + 1) + 16.0 * ni * N,
    "cg_update_r": 24.0 * ni * N,
    "cg_update_px": 40.0 * ni * N,
    "expand": 16.0 * ni * N,
}
rows = {}
total = 0.0
for nm in NAMES:
    ms, cnt = ctx.kernel_time(nm)
    if cnt == 0:
        continue
    total += ms
    r = {"ms": round(ms, 3), "launches": int(cnt), "avg_us": round(1e3 * ms / cnt, 2)}
    b = BYTES.get(nm)
    if b:
        r["alg_GB_per_launch"] = round(b / 1e9, 3)
        r["GBps"] = round(b / (ms / cnt) / 1e6, 1)
        r["frac_hbm"] = round(b / (ms / cnt) / 1e6 / hbm, 3)
    rows[nm] = r
print(json.dumps({"case": f"uniform R={R}", "n_i": ni, "tets": nt, "nnz": nnz, "N": N, "sweeps": SWEEPS,
                  "hbm_peak_GBps": hbm, "step_ms": round(lg["ms_total"], 2),
                  "phases_ms": {k: round(lg[k], 2) for k in ("ms_bvp", "ms_hartree", "ms_project", "ms_inner")},
                  "kernel_ms_sum": round(total, 2), "families": rows}))
