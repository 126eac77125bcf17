// One outer iteration of the corrected level solve on the device (see correction.cu).
#pragma once

#include "mg.cuh"
#include <array>
#include <vector>

#include "cg.cuh"
#include "inner.cuh"
#include "physics.cuh"
#include "project.cuh"

namespace ksb {

constexpr int MAT_H = 3;    // current outer operator a_op + M_{w_hat + v_xc}
constexpr int MAT_TMP = 4;  // scratch

struct System {
    std::vector<double> atoms;  // (Z, x, y, z) per nucleus
    int N = 1;
    double occ = 2.0;
    XcParams xc{2, 0.77298, 1.0 / 3.0};
    bool hartree_on = true, xc_on = true;
    bool set = false;
};

struct StepOptions {
    double tol_linear = 1e-9, tol_inner = 1e-8, score_floor = 1e-8;
    int max_inner = 400, nev_pad = 4, check_every = 8, fixed_sweeps = 0;
    bool norm_l1 = false;  // density change in L1 instead of H1 (RunConfig::outer_norm_l1)
    int precond = 0;       // 0: Jacobi BVPs + multigrid Hartree (production); 1: the reference's SGS everywhere
};

struct StepLog {
    int inner_iterations = 0, hartree_iterations = 0;
    double delta = 0;
    double ms_bvp = 0, ms_hartree = 0, ms_project = 0, ms_inner = 0, ms_total = 0;
    int64_t cg_iterations = 0;
    std::vector<int> attempts, iterations;  // per orbital: -1 unshifted, k = ladder rung
    std::vector<double> inner_history;
};

/// per-level correction machinery attached to a Level
struct Corrector {
    System sys;
    bool ops_ready = false;
    double min_diag = 0;
    DevBuf<double> eext;        // 16 per fine tet: M_ext element (Keast)
    CoarseOps coarse;
    ProjOut proj;
    InnerWork inner;
    PhysWork phys;
    // work vectors (full = n, int = ni, blocks = ni x ld)
    DevBuf<double> rho, vxc, pot, rho_t, bcb, wt_full, ell_full, what_full, diff, wtil_int, hrhs;
    DevBuf<double> R0, Bblk, Xblk, Bc, Xc, PhiT;
    DevBuf<double> colscale;    // per-column right-hand-side scales of the orbital solves
    DevBuf<double> potf, wscr;  // standard MLC: w + v_xc (full), scratch w of expand
    DevBuf<double> phiHT;       // coarse orbital coefficients, orbital index fastest (expand)
    DevBuf<int> idx;
    std::vector<double> scf_history;
    int precond = 0;  // preconditioner of the step in progress (StepOptions::precond)  // density changes of the last coarse_scf, kept when it fails (diagnostics)
    int ldT = 0;
    int mlc_ld = 0, mlc_sweeps = 0;  // standard MLC state: ld of PhiT, sweeps run
    EstimatorData est;
    Multigrid mg;  // V-cycle preconditioner of the stiffness solves (built on first use)
};

void level_ops(Level& L, Corrector& K);

/// scf::self_consistent_solve on level 0 (proj/src/scf.cpp:22-90): dense lowest eigenpairs of the current
/// Hamiltonian, linear density mixing, Poisson solve for the Hartree potential of the mixed density
struct ScfParams {
    double tol = 1e-6;
    int max_iterations = 200;
    double mixing = 0.3;
    bool hartree_on = true, xc_on = true;
    double tol_eig = 1e-9;
    bool norm_l1 = false;  // scf::Options::norm_l1 (proj/include/ksafem/scf.hpp:19)
};
struct ScfStats {
    int iterations = 0;
    std::vector<double> history;
};
ScfStats coarse_scf(Level& L, Corrector& K, CgWork& cg, const ScfParams& p, double* h_lambda, double* d_Phi, int ld,
                    double* d_rho_full, double* d_w_full);
void correction_step(Level& L, Corrector& K, CgWork& cg, const StepOptions& o, double* h_lambda, double* d_Phi, int ld,
                     double* d_w, StepLog* log);

/// standard multilevel correction (driver::solve_level_mlc, proj/src/driver.cpp:200-302), split at its loop:
/// begin = orbital BVPs with the warm potentials + Hartree boundary data; sweep = one correction-space
/// iteration (Hartree of the current density, pot = w + v_xc, bordered solves, expand, density change);
/// finish = Hartree potential of the final density.
void mlc_begin(Level& L, Corrector& K, CgWork& cg, const StepOptions& o, const double* h_lambda, const double* d_Phi,
               int ld, const double* d_w, StepLog* log);
double mlc_sweep(Level& L, Corrector& K, CgWork& cg, const StepOptions& o, double* h_lambda, double* d_Phi, int ld);
void mlc_finish(Level& L, Corrector& K, CgWork& cg, const StepOptions& o, double* d_w, double* d_rho);

// pieces (also exported through the C-ABI for parity tests)
double outer_operator(Level& L, Corrector& K, const double* d_what_full, const double* d_vxc_full, int aop = 2);
/// min over the interior diagonal of A_ii (EllipticSolver::min_diagonal, proj/src/solver.cpp:44)
double min_diagonal(Level& L, int mat, DevBuf<double>& scratch);
/// EllipticSolver::solve (proj/src/solver.cpp:113-131); d_bc_full NULL = solve_zero_bc
CgColumnStats elliptic_solve(Level& L, CgWork& cg, DevBuf<double>& scratch, int mat, const double* d_b_full,
                             const double* d_bc_full, const CgOptions& o, double* d_x_full);
void solve_orbitals(Level& L, Corrector& K, CgWork& cg, const StepOptions& o, const double* h_lambda,
                    const double* d_Phi, int ld, double* d_PhiT, int ldT, StepLog* log, int n_cols = 0);
int hartree_solve(Level& L, Corrector& K, CgWork& cg, const double* d_PhiT, int N, int ldT, const double* d_bcb,
                  double tol, double* d_w_full);
void expand(Level& L, Corrector& K, const double* d_PhiT, int ldT, const double* d_wt_full, const double* d_bcb,
            double* d_Phi, int ld, double* d_w_full);

}  // namespace ksb
