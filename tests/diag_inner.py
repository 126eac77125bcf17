"""Diagnostics: GPU pieces of one cfg1 level-3 correction step + inner states after k sweeps."""
import sys, json
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2103_02824_b200 as kb

lev = 3
d = np.load(ROOT / "tests/_diag/cfg1_start_level3.npz")
ATOMS = [[2.0, 0.0, 0.0, 0.0]]
h = kb.Hierarchy()
a = kb.Mesh.box([-10.0] * 3, [10.0] * 3, 8)
h.push(a)
for _ in range(lev):
    a = a.uniform_refine(); h.push(a)
ctx = kb.Context(0)
L = kb.Level(ctx, h, lev)
L.set_system(ATOMS, n_pairs=1, occupancy=2.0, xc="lda"); L.level_ops()
it = L.index("interior")
bnd = np.setdiff1d(np.arange(L.n), it)
lam = d["lam"].copy()
Phi = ctx.to_device(np.ascontiguousarray(d["orb"][it])); w = ctx.to_device(d["w"])
rho, vxc = ctx.empty(L.n), ctx.empty(L.n)
L.density_xc(Phi, rho, vxc)
PhiT = ctx.empty((L.ni, 1))
att, its, md = L.outer_solve(w, vxc, lam, Phi, PhiT)
rt = ctx.empty(L.n)
L.density_xc(PhiT, rt)
m = L.moments(rt)
bcb = ctx.empty(L.nb); L.boundary_values(m, bcb)
wt = ctx.empty(L.n)
L.hartree_solve(PhiT, bcb, wt)
wt_h = wt.download(); ell = np.zeros(L.n); ell[bnd] = bcb.download()
L.prepare_blocks(PhiT, ctx.to_device(wt_h - ell), ctx.to_device(ell), vxc)
out = {"phiT": PhiT.download(), "wt": wt_h, "vxc": vxc.download(), "bc": ell, "lam": lam}
for k in [1, 2, 5, 10, 20, 40, 60, 100]:
    r = L.inner_scf(lam, fixed_sweeps=k)
    out[f"lam{k}"] = r["lambda_"]; out[f"phi{k}"] = r["phi_H"]; out[f"th2{k}"] = r["theta2"]
    out[f"wH{k}"] = r["w_H"]; out[f"th1{k}"] = np.array([r["theta1"]]); out[f"hist{k}"] = r["history"]
    print(k, r["lambda_"], r["theta2"], r["theta1"], r["history"][-1], flush=True)
for name in ["A_H1", "A_H3", "A_H4", "M_H", "C_H", "d_Hh", "lift_load", "A_h4", "b_H1", "b_H3", "b_H4", "rhs", "c_Hh",
             "d_phi", "beta1", "beta3", "beta4", "gamma", "zeta_phi", "scalars"]:
    out["B_" + name] = L.blocks(name)
np.savez(ROOT / "gpurun_out/diag_inner.npz", **out)
