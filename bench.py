#!/usr/bin/env python3
"""Benchmark of the correction-step hot path (BASELINE.json configs[1], "cfg2").

Workload (one step): the operator micro-benchmark of BASELINE.json configs[1] --
A = 1/2 K + M_V - sigma M (sigma = -0.5) on the Kuhn-split P1 mesh of a 128^3 vertex
grid over [-10,10]^3 (2,000,376 interior DOFs, 29.6 M interior nonzeros), V = -sum of
4 seeded Gaussians, and a block of N = 16 seeded N(0,1) right-hand sides driven through
exactly 200 iterations of the multi-RHS preconditioned CG (Jacobi). FP64.
value = interior DOFs * 16 orbitals * 200 iterations / step time  [DOF*orbital*iter/s].

Arms: default = the B200 path (libksb.so kernels); --impl reference = the CPU oracle's
restatement of the reference's own algorithm (SGS-PCG, proj/src/solver.cpp:57-111) on the
host cores (the reference itself cannot be built here: SURVEY.md section 8c).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fine-solve DOF*orbital*iter/s; correction-step time; SpMM % of HBM peak"
UNIT = "DOF*orbital*iter/s"
N_RHS = 16
ITERS = 200
GRID = 127  # cells per axis -> 128^3 vertices
BOX = 10.0
SEED = 20210304


def gaussians(seed=SEED):
    """4 seeded wells: centres U[-3,3]^3, widths U(0.5,1.5), depths U(1,5); V = -sum d exp(-|x-c|^2/(2 w^2))."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(-3.0, 3.0, (4, 3))
    w = rng.uniform(0.5, 1.5, 4)
    d = rng.uniform(1.0, 5.0, 4)
    return np.column_stack([d, w, c])


def rhs_block(ni, seed=SEED + 1):
    return np.random.default_rng(seed).standard_normal((ni, N_RHS))


def ncu_traffic(kernel):
    """DRAM bytes per launch from the committed ncu capture (profiles/ncu_traffic.json), or None."""
    try:
        return int(json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())[kernel]["dram_bytes_per_launch"])
    except Exception:
        return None


def measured_peak():
    try:
        j = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(j["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 7:
                try:
                    rows.append((float(p[0]), float(p[1]), p[3:7]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i in range(4) if r[i].lower().startswith("active")})
        return {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def dist_init(backend: str | None = None):
    """One process per GPU (torchrun env). NCCL on GPU boxes; gloo where CUDA is absent (the CPU tests of the
    replica plumbing, tests/test_replicas.py)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(units_per_rank: float, ms_local: float, world: int) -> tuple[float, float]:
    """Whole-job throughput of `world` replicas: all ranks' units over the slowest rank's time (max over ranks)."""
    ms = max_over_ranks(ms_local, world)
    return world * units_per_rank / (ms * 1e-3), ms


# ----------------------------------------------------------------------------------- CPU legs
_CFG2_ORACLE = {}


def cfg2_oracle_operator(precond):
    """The cfg2 operator in the CPU oracle (built once per process; precond 0 = SGS, the reference's
    proj/src/solver.cpp:50-55, 1 = Jacobi, the device's)"""
    from oracle import OMesh, Oracle
    if "orc" not in _CFG2_ORACLE:
        t0 = time.time()
        m = OMesh.box([-BOX] * 3, [BOX] * 3, GRID)
        orc = Oracle([[1.0, 0, 0, 0]])
        orc.push(m)
        _CFG2_ORACLE.update(orc=orc, mesh=m, setup_s=time.time() - t0)
    key = f"op{precond}"
    if key not in _CFG2_ORACLE:
        _CFG2_ORACLE[key] = _CFG2_ORACLE["orc"].operator(0, c_s=0.5, c_m=0.5, potential=(1, gaussians()),
                                                         precond=precond)
    return _CFG2_ORACLE[key]


def cpu_leg(iters_sample: int, precond: int = 0):
    """Oracle PCG on the same operator; a bounded sample: 16 columns x iters_sample iterations. precond 0 = SGS (the
    reference's algorithm), 1 = Jacobi (like for like with the device iteration)."""
    op = cfg2_oracle_operator(precond)
    B = rhs_block(op.ni)
    t1 = time.perf_counter()
    op.pcg(B, fixed=iters_sample)
    dt = time.perf_counter() - t1
    return op.ni, dt, _CFG2_ORACLE["setup_s"]


def parity_gate(X_dev, stats_dev, iters):
    """The timed cfg2 result against the oracle: the same fixed-count Jacobi PCG (iters iterations, 16 columns) on
    the host; relative L2 difference of the whole block and of the reported residuals."""
    op = cfg2_oracle_operator(1)
    B = rhs_block(op.ni)
    t = time.perf_counter()
    Xo, so = op.pcg(B, fixed=iters)
    dt = time.perf_counter() - t
    err = float(np.linalg.norm(X_dev - Xo) / np.linalg.norm(Xo))
    rr = max(abs(s.relative_residual - o["relative_residual"]) / max(o["relative_residual"], 1e-300)
             for s, o in zip(stats_dev, so))
    return {"checked": "timed cfg2 block X (200 Jacobi-PCG iterations, 16 columns) vs the oracle's Jacobi PCG",
            "x_rel_l2": err, "relres_max_rel_diff": float(rr), "tol": PARITY_TOL, "ok": bool(err <= PARITY_TOL),
            "oracle_s": round(dt, 1)}


PARITY_TOL = 1e-6


def run_reference(args, world, rank):
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    sample = args.cpu_iters
    op = cfg2_oracle_operator(0)
    B = rhs_block(op.ni)
    for _ in range(max(0, args.warmup)):
        op.pcg(B, fixed=1)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        op.pcg(B, fixed=sample)
        times.append(time.perf_counter() - t)
    dt = float(np.mean(times))
    value = op.ni * N_RHS * sample / dt
    used = min(cores, N_RHS)
    # like-for-like: the device's Jacobi iteration in the same oracle (one sample, reported beside the value)
    _, djac, _ = cpu_leg(sample, precond=1)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2 operator micro-benchmark: 128^3 Kuhn P1, A=1/2K+M_V+0.5M, N=16, 200 CG its",
                       "n_interior": op.ni, "n_rhs": N_RHS, "iterations": ITERS, "l2": "inputs larger than L2",
                       "step": f"one step = one measured sample of {sample} SGS-PCG iterations on all 16 columns "
                               f"(ms_per_step is that sample's time; value is per iteration, so it compares with "
                               f"the device's 200-iteration steps)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "port",
                             "sample": f"oracle SGS-PCG (reference algorithm), 16 columns x {sample} iterations per "
                                       f"step, OpenMP over columns"},
            "cpu_jacobi": {"value": op.ni * N_RHS * sample / djac, "unit": UNIT, "cores": used,
                           "sample": f"the same oracle with the device's Jacobi preconditioner, 16 x {sample} its"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------- correction step (cfg1)
CS_LEVEL = 3
CS_STEPS = 5
HE = [[2.0, 0.0, 0.0, 0.0]]


def correction_cpu(phi_full, w_full, lam0):
    """Oracle correction step (reference algorithm: SGS-PCG, dense bordered eigensolves) from the same state."""
    from oracle import OMesh, Oracle
    orc = Oracle(HE, n_pairs=1, occ=2.0, xc="lda")
    m = OMesh.box([-BOX] * 3, [BOX] * 3, 8)
    orc.push(m)
    for _ in range(CS_LEVEL):
        m = m.uniform_refine()
        orc.push(m)
    t = time.perf_counter()
    lam, _, _, lg = orc.correction_step(CS_LEVEL, lam0.copy(), phi_full, w_full)
    return (time.perf_counter() - t) * 1e3, lg["inner_iterations"], float(lam[0])


def correction_bench(args, ctx, stream, rank, world):
    """cfg1 (BASELINE.json configs[0]) finest level: CS_STEPS outer iterations from a synthetic start."""
    import torch

    import paper_2103_02824_b200 as kb
    from paper_2103_02824_b200.workloads import cfg1_hierarchy, synthetic_start
    h = cfg1_hierarchy(CS_LEVEL)
    L = kb.Level(ctx, h, CS_LEVEL)
    L.set_system(HE, n_pairs=1, occupancy=2.0, xc="lda")
    L.level_ops()
    lam0, Phi, w, ld = synthetic_start(L, ctx, h.meshes[CS_LEVEL], [[0, 0, 0]], 1)
    phi0, w0 = Phi.download(), w.download()

    def trajectory(timed):
        Phi.upload(phi0)
        w.upload(w0)
        lam = lam0.copy()
        logs, ms = [], []
        for _ in range(CS_STEPS):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            logs.append(L.correction_step(lam, Phi, w))
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return lam, logs, ms

    trajectory(False)  # warm-up (kernel caches, operator slots, workspaces)
    ctx.reset_counters()
    lam, logs, ms = trajectory(True)
    launches = ctx.launches()
    # end to end: host orbitals / potential in and out of every step (pinned host buffers)
    hphi = torch.empty(phi0.shape, dtype=torch.float64, pin_memory=True)
    hw = torch.empty(w0.shape, dtype=torch.float64, pin_memory=True)
    hphi.numpy()[:] = phi0
    hw.numpy()[:] = w0
    lam_h = lam0.copy()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(CS_STEPS):
        L.correction_step_host(lam_h, hphi.numpy(), hw.numpy())
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / CS_STEPS, world)
    out = {"workload": f"cfg1 level {CS_LEVEL}: He (Z=2) LDA, 1 doubly occupied orbital, [-10,10]^3, 8^3 Kuhn "
                       f"coarse + {CS_LEVEL} uniform refinements; synthetic hydrogenic start exp(-1.7 r), lambda -0.6",
           "n_interior": L.ni, "n_coarse_interior": L.nH, "steps": CS_STEPS,
           "ms_per_step": max_over_ranks(float(np.mean(ms)), world), "ms_steps": [round(x, 3) for x in ms],
           "inner_iterations": [lg["inner_iterations"] for lg in logs],
           "cg_iterations": [lg["cg_iterations"] for lg in logs],
           "breakdown_ms": {k: round(float(np.mean([lg["ms_" + k] for lg in logs])), 3)
                            for k in ("bvp", "hartree", "project", "inner")},
           "lambda_after": float(lam[0]), "gpu_launches": launches,
           "e2e": {"ms_per_step": e2e_ms, "h2d_bytes_per_step": phi0.nbytes + w0.nbytes,
                   "d2h_bytes_per_step": phi0.nbytes + w0.nbytes}}
    # the 49 MB operator is L2-resident, so the BVP phase is reported as algorithmic bytes per
    # time (CG iteration = 12 nnz + 4 (n_i + 1) + 16 n_i + 88 n_i N, N = 1) with the L2 hit rate of the committed ncu
    # capture of the single-column cooperative CG kernel, not as a fraction of the HBM peak
    it_bytes = 12 * L.nnz_ii + 4 * (L.ni + 1) + 16 * L.ni + 88 * L.ni
    cg_its = float(np.mean([lg["cg_iterations"] for lg in logs]))
    bvp_ms = float(np.mean([lg["ms_bvp"] for lg in logs]))
    l2 = None
    try:
        l2 = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())["k_cg_coop"]
    except Exception:
        pass
    out["bvp_algorithmic"] = {"bytes_per_cg_iteration": it_bytes, "cg_iterations_per_step": cg_its,
                              "ms_bvp": bvp_ms, "GBps": it_bytes * cg_its / (bvp_ms * 1e-3) / 1e9,
                              "l2_hit_pct": l2.get("l2_hit_pct") if l2 else None,
                              "l2_source": l2.get("source") if l2 else None,
                              "note": "whole BVP phase (operator build, lift, the cooperative CG solve) over the "
                                      "CG iterations' algorithmic bytes; L2-resident, so above-HBM rates are possible"}
    if rank == 0 and world == 1 and not args.no_cpu:
        it = L.index("interior")
        full = np.zeros((L.n, 1))
        full[it, 0] = phi0[:, 0]
        cms, cinner, clam = correction_cpu(full, w0, lam0)
        out["cpu_baseline"] = {"ms_per_step": cms, "kind": "port", "cores": os.cpu_count() or 1,
                               "sample": f"oracle correction step 0 from the same start ({cinner} inner sweeps, "
                                         f"lambda {clam:.10f}; device step 0: {logs[0]['inner_iterations']} sweeps)"}
    L.close()
    return out


# ----------------------------------------------------------------------------------- configs[2..4] at their sizes
ADAPTIVE_SWEEPS = 10  # inner sweeps per timed step: the work is defined whatever the inner dynamics do
# parity / CPU-sample level: the finest level of the same hierarchy with at most this many vertices
ADAPTIVE_SAMPLE_N = {"cfg3": 60000, "cfg4": 40000, "cfg5": 12000}
ADAPTIVE_SAMPLE_SWEEPS = 3  # inner sweeps of the sample step (the oracle's dense bordered eigensolves dominate it)
# k_proj_orbital_wide per (orbital, fine tet). N >= 64 (T_k form): sum_k phi_k T_k (80), M_phi phi closed form +
# mu^T y (~60), five E x / mu^T y / x.y (360). Below: M_phi element, P^T E P (256), six E x / mu^T y / x.y (432)
PROJ_FLOP_PER_TET_ORB = {True: 500, False: 720}


def fp64_peak():
    try:
        d = json.loads((ROOT / "profiles" / "r01_fp64_peak.json").read_text())
        return float(d["dfma_tflops"]), "measured DFMA (profiles/micro/fp64_peak.cu)"
    except (OSError, ValueError, KeyError):
        return 40.0, "vendor FP64"


def adaptive_case(name, args, ctx, stream, world, rank):
    """One correction step (proj/src/driver.cpp:106-150) on the finest level of an estimator-driven adaptive
    hierarchy of BASELINE configs[2..4] (workloads.adaptive_hierarchy), at the configured DOF count, from the seeded
    device synthetic start, ADAPTIVE_SWEEPS inner sweeps. Per-phase roofline; parity and the CPU oracle's step on
    the hierarchy's sample level; the oracle's full-size step extrapolated per phase from it."""
    import torch

    import paper_2103_02824_b200 as kb
    from oracle import OMesh, Oracle
    from paper_2103_02824_b200 import workloads
    gen, N, box, target = workloads.ADAPTIVE_CONFIGS[name]
    atoms = getattr(workloads, gen)()
    cen = [a[1:] for a in atoms]
    t0 = time.time()
    h, meshes, L, recs, marks = workloads.adaptive_hierarchy(ctx, atoms, N, box, target)
    hier_s = time.time() - t0
    rec = {"workload": f"{name} (BASELINE configs[{int(name[-1]) - 1}]): {len(atoms)} nuclei, N = {N}, LDA, "
                       f"[-{box:g},{box:g}]^3, 8^3 Kuhn coarse, residual-indicator Doerfler (theta 0.4) adaptive "
                       f"refinement to ~{target:.1e} DOFs (marks from the seeded synthetic state; the reference's "
                       f"coarse SCF diverges on this mesh, profiles/r02_scf_histories.json), synthetic start, "
                       f"{ADAPTIVE_SWEEPS} inner sweeps per step",
           "n_dofs": L.n, "n_interior": L.ni, "n_tets": L.nt, "nnz_interior": L.nnz_ii, "N": N,
           "levels": len(meshes), "hierarchy_s": round(hier_s, 1)}
    lam0 = np.linspace(-1.5, -0.3, N)
    _, Phi, w, ld = workloads.synthetic_start_device(L, ctx, meshes[-1], cen, N, zeta=1.0)
    phi0, w0 = Phi.download(), w.download()
    try:
        lam = lam0.copy()
        L.correction_step(lam, Phi, w, ld=ld, fixed_sweeps=ADAPTIVE_SWEEPS)  # warm-up (multigrid setup, caches)
        Phi.upload(phi0)
        w.upload(w0)
        lam = lam0.copy()
        ctx.reset_counters()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        lg = L.correction_step(lam, Phi, w, ld=ld, fixed_sweeps=ADAPTIVE_SWEEPS)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1), world)
        launches = ctx.launches()
    except kb.KsbError as e:
        rec["error"] = str(e)[:300]
        L.close()
        return rec
    its = np.asarray(lg["iterations"])
    block_its = int(its.max())
    # per-phase roofline. BVPs (HBM): per block iteration the matrix (12 nnz + 4 (n_i + 1) + 16 n_i) plus 88 n_i per
    # active column (SURVEY.md 8(d)'s CG-iteration bytes), summed over the columns' own iteration counts
    bvp_bytes = block_its * (12 * L.nnz_ii + 4 * (L.ni + 1) + 16 * L.ni) + 88 * L.ni * int(its.sum())
    peak, peak_kind = measured_peak()
    fpk, fp_kind = fp64_peak()
    proj_flop = PROJ_FLOP_PER_TET_ORB[N >= 64] * N * L.nt
    rec.update({
        "ms_per_step": ms, "gpu_launches": launches,
        "phases_ms": {k: round(lg["ms_" + k], 3) for k in ("bvp", "hartree", "project", "inner")},
        "cg_iterations": lg["cg_iterations"], "block_iterations": block_its,
        "shift_attempts": {str(a): int((np.asarray(lg["attempts"]) == a).sum()) for a in (-1, 0, 1, 2, 3)},
        "hartree_iterations": lg["hartree_iterations"], "inner_sweeps": lg["inner_iterations"],
        "roofline": {"bound": "hbm", "phase": "bvp (multi-column CG, CSR SpMM)",
                     "achieved": bvp_bytes / (lg["ms_bvp"] * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": bvp_bytes / (lg["ms_bvp"] * 1e-3) / 1e9 / peak, "traffic": None,
                     "bytes": bvp_bytes, "peak_kind": peak_kind},
        "roofline_project": {"bound": "fp64", "achieved": proj_flop / (lg["ms_project"] * 1e-3) / 1e12,
                             "peak": fpk, "unit": "TFLOP/s",
                             "frac": proj_flop / (lg["ms_project"] * 1e-3) / 1e12 / fpk, "peak_kind": fp_kind,
                             "flop": proj_flop},
        "lambda_after": [float(x) for x in lam[:4]],
    })
    # end to end: host orbitals / potential in and out of the step (pinned host buffers)
    del Phi
    torch.cuda.empty_cache()
    hphi = torch.empty(phi0.shape, dtype=torch.float64, pin_memory=True)
    hw = torch.empty(w0.shape, dtype=torch.float64, pin_memory=True)
    hphi.numpy()[:] = phi0
    hw.numpy()[:] = w0
    lam_h = lam0.copy()
    torch.cuda.synchronize()
    e0.record(stream)
    try:
        L.correction_step_host(lam_h, hphi.numpy(), hw.numpy(), fixed_sweeps=ADAPTIVE_SWEEPS)
        e1.record(stream)
        torch.cuda.synchronize()
        rec["e2e"] = {"ms_per_step": max_over_ranks(e0.elapsed_time(e1), world),
                      "h2d_bytes_per_step": phi0.nbytes + w0.nbytes, "d2h_bytes_per_step": phi0.nbytes + w0.nbytes}
    except kb.KsbError as e:
        rec["e2e"] = {"error": str(e)[:200]}
    del hphi, hw
    L.close()

    # parity and the CPU sample: the same hierarchy's level kp, device step vs oracle step from the same state
    kp = max(k for k, m in enumerate(meshes) if m.n_vertices <= ADAPTIVE_SAMPLE_N[name])
    Lk = kb.Level(ctx, h, kp)
    Lk.set_system(atoms, n_pairs=N, occupancy=2.0, xc="lda")
    Lk.level_ops()
    _, Pk, wk, ldk = workloads.synthetic_start_device(Lk, ctx, meshes[kp], cen, N, zeta=1.0)
    it = Lk.index("interior")
    orb = np.zeros((Lk.n, N))
    orb[it] = Pk.download()[:, :N]
    wk0 = wk.download()
    lam_d = lam0.copy()
    lgk = Lk.correction_step(lam_d, Pk, wk, ld=ldk, fixed_sweeps=ADAPTIVE_SAMPLE_SWEEPS)
    par = {"level": kp, "n_dofs": Lk.n, "N": N, "inner_sweeps": ADAPTIVE_SAMPLE_SWEEPS}
    if rank == 0 and not args.no_cpu:
        os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
        orc = Oracle(atoms, n_pairs=N, occ=2.0, xc="lda")
        om = OMesh.box([-box] * 3, [box] * 3, 8)
        orc.push(om)
        for j in range(kp):
            om = om.adapt_refine(marks[j])
            orc.push(om)
        t1 = time.time()
        lam_o, orb_o, w_o, lo = orc.correction_step(kp, lam0.copy(), orb, wk0, fixed_sweeps=ADAPTIVE_SAMPLE_SWEEPS)
        cpu_s = time.time() - t1
        P = Pk.download()[:, :N]
        O = orb_o[it]
        rho_g, rho_o = 2.0 * (P ** 2).sum(1), 2.0 * (O ** 2).sum(1)
        gaps = [min(abs(lam_o[i] - lam_o[j]) for j in range(N) if j != i) for i in range(N)]
        orb_err = max((np.linalg.norm(np.sign(P[:, i] @ O[:, i]) * P[:, i] - O[:, i]) / np.linalg.norm(O[:, i])
                       for i in range(N) if gaps[i] > 1e-3), default=0.0)
        par.update({
            "mesh_bitexact": bool(np.array_equal(om.array("tets"), meshes[kp].array("tets"))),
            "lambda_max_rel": float(np.abs(lam_d - lam_o).max() / np.abs(lam_o).max()),
            "rho_rel": float(np.linalg.norm(rho_g - rho_o) / np.linalg.norm(rho_o)),
            "w_rel": float(np.linalg.norm(wk.download() - w_o) / np.linalg.norm(w_o)),
            "orbital_max_rel": float(orb_err), "attempts_equal": lgk["attempts"] == lo["attempts"],
            "tol": {"lambda": 1e-8, "rho_w_orbitals": 1e-6}})
        par["ok"] = bool(par["mesh_bitexact"] and par["lambda_max_rel"] <= 1e-8 and par["rho_rel"] <= 1e-6
                         and par["w_rel"] <= 1e-6 and par["orbital_max_rel"] <= 1e-6)
        # oracle's full-size step, extrapolated per phase from the sample level: vector phases by the tet / DOF
        # ratio (the BVPs also by the device's block-CG iteration ratio), the coarse inner loop as measured
        r_n, r_t = rec["n_dofs"] / Lk.n, rec["n_tets"] / Lk.nt
        r_it = block_its / max(1, int(np.asarray(lgk["iterations"]).max()))
        ext = {"bvp": lo["t_bvp"] * r_n * r_it, "hartree": lo["t_hartree"] * r_n, "project": lo["t_blocks"] * r_t,
               "inner": lo["t_inner"] * ADAPTIVE_SWEEPS / ADAPTIVE_SAMPLE_SWEEPS}
        rec["cpu_baseline"] = {
            "ms_per_step": 1e3 * sum(ext.values()), "kind": "port", "cores": os.cpu_count() or 1,
            "extrapolated": True, "phases_ms": {k: round(1e3 * v, 1) for k, v in ext.items()},
            "sample": f"oracle correction step on level {kp} of the same hierarchy ({Lk.n} DOFs, {cpu_s:.1f} s, "
                      f"SGS-PCG, {ADAPTIVE_SAMPLE_SWEEPS} inner sweeps), phases scaled to {rec['n_dofs']} DOFs: BVPs "
                      f"x DOF ratio {r_n:.0f} x device block-CG iteration ratio {r_it:.2f}, Hartree x DOF ratio "
                      f"(iteration growth ignored: a lower bound), projection x tet ratio, inner loop x "
                      f"{ADAPTIVE_SWEEPS}/{ADAPTIVE_SAMPLE_SWEEPS} sweeps (its size does not depend on the level)"}
    rec["parity_sample"] = par
    Lk.close()
    return rec


def adaptive_bench(args, ctx, stream, world, rank):
    out = {}
    for name in ("cfg3", "cfg4", "cfg5"):
        try:
            out[name] = adaptive_case(name, args, ctx, stream, world, rank)
        except Exception as e:  # noqa: BLE001 -- a failed section is reported, the bench line still prints
            out[name] = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
        import torch
        torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------------- cfg1 run (levels 0-2)
RUN_LEVELS = 3  # coarse SCF + levels 1 and 2; on level 3 the reference algorithm itself stalls


def cfg1_run_cpu():
    """The same run composed from the oracle's pieces (reference algorithm) on the host cores."""
    from oracle import OMesh, Oracle
    t = time.perf_counter()
    orc = Oracle(HE, n_pairs=1, occ=2.0, xc="lda")
    m = OMesh.box([-BOX] * 3, [BOX] * 3, 8)
    orc.push(m)
    lam, orb, w, _ = orc.coarse_scf(tol=1e-6, mixing=0.3, tol_eig=1e-9)
    for level in range(1, RUN_LEVELS):
        m = m.uniform_refine()
        orc.push(m)
        orb = orc.prolong(orb, level - 1, level)
        w = orc.prolong(w, level - 1, level)[:, 0]
        for _ in range(40):
            lam, orb, w, lg = orc.correction_step(level, lam, orb, w)
            if lg["delta"] < 1e-6:
                break
    return time.perf_counter() - t, float(lam[0])


def cfg1_run_bench(args, ctx, rank, world):
    from paper_2103_02824_b200.driver import run
    run(ctx, HE, 1, 2.0, "lda", BOX, 8, 2, refine="uniform")  # warm-up: kernel caches, first-use allocations
    t = time.perf_counter()
    log = run(ctx, HE, 1, 2.0, "lda", BOX, 8, RUN_LEVELS, refine="uniform")
    wall = time.perf_counter() - t
    out = {"workload": "cfg1 (configs[0]) run from scratch on the device: coarse SCF on 8^3, uniform levels 1-2, "
                       "corrected level solves to tol_outer 1e-6, indicators per level",
           "wall_s": max_over_ranks(wall, world), "aborted": log.aborted,
           "levels": [{"level": r.level, "n_dofs": r.n_dofs, "lambda": r.lambdas[0], "energy": r.energy[4],
                       "outer": r.outer_iterations, "t_total_s": round(r.t_total, 4)} for r in log.records]}
    if rank == 0 and world == 1 and not args.no_cpu:
        cw, clam = cfg1_run_cpu()
        out["cpu_baseline"] = {"wall_s": cw, "kind": "port", "cores": os.cpu_count() or 1,
                               "sample": f"the same run from the oracle's pieces (SGS-PCG, dense eigensolves); "
                                         f"final lambda {clam:.12f}"}
    return out


# ----------------------------------------------------------------------------------- GPU leg
def run_b200(args, world, rank, local):
    import torch

    import paper_2103_02824_b200 as kb
    torch.cuda.set_device(local)
    ctx = kb.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))

    t0 = time.time()
    mesh = kb.Mesh.box([-BOX] * 3, [BOX] * 3, GRID)
    h = kb.Hierarchy()
    h.push(mesh)
    L = kb.Level(ctx, h, 0)
    L.assemble(kb.MAT_USER0, c_s=0.5, c_m=0.5, potential=(kb.POT_GAUSSIAN, gaussians()))
    setup_s = time.time() - t0
    ni = L.ni
    B = rhs_block(ni)
    dB = ctx.to_device(B)
    dX = ctx.empty((ni, N_RHS))
    opts = L.cg_options(fixed_iterations=ITERS)

    def step():
        return L.cg_solve(kb.MAT_USER0, dB, dX, N_RHS, opts=opts)

    for _ in range(max(3, args.warmup)):
        step()
    ctx.sync()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            stats = step()
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = ctx.launches() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    value, ms = replica_value(ni * N_RHS * ITERS, ms, world)
    # fixed-count mode reports, per column, the iterations that saw p.Ap <= 0 (A is indefinite: wells below -0.5)
    curvature_events = [int(s.breakdown) for s in stats]
    X_timed = dX.download() if (rank == 0 and not args.no_parity) else None

    # dominant kernel: the fused SpMM (Ap = A p + p.Ap partials), timed per launch with events on its stream
    ctx.reset_counters()
    ctx.set_profiling(True)
    step()
    ctx.set_profiling(False)
    spmm_ms, spmm_n = ctx.kernel_time("spmm")
    upd_ms, upd_n = ctx.kernel_time("cg_update_r")
    updp_ms, updp_n = ctx.kernel_time("cg_update_px")
    spmm_avg = spmm_ms / max(1, spmm_n)
    # algorithmic bytes per launch: SURVEY.md 8(d)'s CSR figure (12 nnz + 4 (n_i + 1) + 16 n_i N); the stencil kernel
    # that runs on this lexicographic Kuhn box streams its own format, 8 D n_i + 16 n_i N (D = 15 diagonals), fewer
    bytes_spmm = 12 * L.nnz_ii + 4 * (ni + 1) + 16 * ni * N_RHS
    dia = L.index("dia")
    stencil = dia[0] > 0 and os.environ.get("KSB_SPMM_DIA") != "0"
    grid_lvl = stencil and dia[15] > 0 and os.environ.get("KSB_DIA_ZT") != "0"
    spmm_kernel = ("k_spmm_dia_zw" if os.environ.get("KSB_DIA_ZW") != "0" else "k_spmm_dia_zt") if grid_lvl else \
        "k_spmm_dia_tv" if stencil else "k_spmm_t8"
    n_diag = 3 + (int(dia[0]) - 1) * int(dia[2]) if stencil else 0
    bytes_format = 8 * n_diag * ni + 16 * ni * N_RHS if stencil else bytes_spmm
    achieved = bytes_spmm / (spmm_avg * 1e-3) / 1e9
    peak, peak_kind = measured_peak()

    # end to end through the C-ABI with pinned host buffers (H2D of B, D2H of X inside the timed region)
    hB = torch.empty((ni, N_RHS), dtype=torch.float64, pin_memory=True)
    hX = torch.empty((ni, N_RHS), dtype=torch.float64, pin_memory=True)
    hB.numpy()[:] = B
    for _ in range(2):
        L.cg_solve_host(kb.MAT_USER0, hB.numpy(), N_RHS, opts=opts, out=hX.numpy())
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        L.cg_solve_host(kb.MAT_USER0, hB.numpy(), N_RHS, opts=opts, out=hX.numpy())
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    e2e = world * ni * N_RHS * ITERS / (e2e_ms * 1e-3)

    correction = correction_bench(args, ctx, stream, rank, world)
    cfg1_run = cfg1_run_bench(args, ctx, rank, world)
    adaptive = None if args.no_adaptive else adaptive_bench(args, ctx, stream, world, rank)

    parity = None
    if rank == 0 and not args.no_parity:
        os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
        parity = parity_gate(X_timed, stats, ITERS)
    cpu = cpu_jac = None
    if rank == 0 and world == 1 and not args.no_cpu:
        os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
        cni, cdt, _ = cpu_leg(args.cpu_iters)
        cpu = {"value": cni * N_RHS * args.cpu_iters / cdt, "unit": UNIT,
               "cores": min(os.cpu_count() or 1, N_RHS), "kind": "port",
               "sample": f"oracle SGS-PCG (reference algorithm) on the same operator: 16 columns x {args.cpu_iters} "
                         f"iterations ({cdt:.1f} s), OpenMP over columns"}
        _, jdt, _ = cpu_leg(args.cpu_iters, precond=1)
        cpu_jac = {"value": cni * N_RHS * args.cpu_iters / jdt, "unit": UNIT,
                   "cores": min(os.cpu_count() or 1, N_RHS), "kind": "port",
                   "sample": f"like for like: the oracle with the device's Jacobi preconditioner, 16 columns x "
                             f"{args.cpu_iters} iterations ({jdt:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Gaussians and N(0,1) RHS)",
            "config": {"workload": "cfg2 operator micro-benchmark: 128^3 Kuhn P1, A=1/2K+M_V+0.5M, N=16, 200 CG its",
                       "n_interior": ni, "nnz_interior": L.nnz_ii, "n_rhs": N_RHS, "iterations": ITERS,
                       "preconditioner": "jacobi", "parallelism": f"replicas{world}",
                       "l2": "inputs larger than L2 (256 MB blocks, 363 MB operator)",
                       "nonpositive_curvature_iterations": curvature_events, "setup_s": round(setup_s, 2)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": ncu_traffic(spmm_kernel), "kernel": spmm_kernel, "bytes_per_launch": bytes_spmm,
                         "avg_launch_ms": spmm_avg, "peak_kind": peak_kind,
                         "format_bytes_per_launch": bytes_format,
                         "format_frac": bytes_format / (spmm_avg * 1e-3) / 1e9 / peak,
                         "bytes_basis": "achieved uses SURVEY.md 8(d)'s CSR bytes for one A P; format_* the bytes the "
                                        "stencil (DIA) format itself moves (15 values per row, no column indices)"},
            "spmm_hbm_frac": achieved / peak,
            "cg_update_r_avg_ms": upd_ms / max(1, upd_n),
            "cg_update_px_avg_ms": updp_ms / max(1, updp_n),
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": B.nbytes, "d2h_bytes_per_step": B.nbytes,
                    "ms_per_step": e2e_ms},
            "gpu_launches": launches // max(1, args.steps) * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "cpu_baseline_jacobi": cpu_jac,
            "ratio_basis": "value / cpu_baseline compares a Jacobi-PCG iteration (device) with an SGS-PCG iteration "
                           "(the reference's algorithm); cpu_baseline_jacobi is the like-for-like iteration; the "
                           "time-to-solution comparison is correction_step (one outer iteration to tolerance, "
                           "device Jacobi/MG vs oracle SGS)",
            "parity": parity,
            "correction_step": correction,
            "cfg1_run": cfg1_run,
            "adaptive": adaptive,
        }
        print(json.dumps(line), flush=True)
    L.close()
    ctx.close()
    if parity is not None and not parity["ok"]:
        print(f"parity gate failed: {parity}", file=sys.stderr)
        sys.exit(3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-iters", type=int, default=96, help="CPU oracle sample: iterations per 16-column block")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-adaptive", "--no-scale", dest="no_adaptive", action="store_true",
                    help="skip the configs[2..4] section (adaptive hierarchies to 1e6 / 4e6 / 1.2e7 DOFs)")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the timed cfg2 result")
    args = ap.parse_args()
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_b200(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
