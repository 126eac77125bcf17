// Inner sweep (corr::inner_scf) on the device; see inner.cu.
#pragma once

#include <vector>

#include "project.cuh"

namespace ksb {

/// per-level coarse operators: M_H, C_H (interior blocks, dense row-major), their Cholesky factors and the
/// explicit inverse factors L_H^-1, L_H^-T (row-major) and C_H^-1 used by the sweep's products
struct CoarseOps {
    DevBuf<double> MH, CH, LH, LC, LHi, LHiT, CHi;
    bool ready = false;
};
void coarse_level_setup(Level& L, CoarseOps& co);

struct InnerParams {
    double tol = 1e-8;
    int max_iterations = 400;
    double score_floor = 1e-8;
    int nev_pad = 4;
    bool hartree = true;
    double occ = 2.0;
    int fixed_sweeps = 0;  // > 0: run exactly this many sweeps, no stopping test (diagnostics)
};

struct InnerStats {
    int iterations = 0;
    std::vector<double> history;
};

/// double-buffered augmented state + scratch; the result lives in buffers [cur]
struct InnerWork {
    int nh = 0, N = 0, nev = 0, cur = 0;
    DevBuf<double> AH, W, C, V, d, e, E16, E4, sq, l, u, s, c12, c22, lhat, lam, Y, Z, piv, score, ynorm, hu, scal, hpart;
    DevBuf<double> phi[2], th2[2], lamv[2], wH[2], th1[2];
    DevBuf<int> flag;
    void ensure(int nh, int N, int nev, int nct);
};

/// lowest nev eigenpairs of (A_ii(mat), M_H) on level 0 (dense path of eig::solve_smallest,
/// proj/src/eigensolve.cpp:321-367): ascending values to h_lambda, M-orthonormal sign-normalised vectors into
/// the interior block d_Phi (ld)
void dense_lowest_eigs(Level& L, const CoarseOps& co, InnerWork& w, int mat, int nev, double* h_lambda, double* d_Phi,
                       int ld);

/// runs sweeps from the pure augmentation state (phi_H = 0, theta2 = 1, w_H = 0, theta1 = hartree)
InnerStats inner_scf(Level& L, const CoarseOps& co, const ProjOut& P, const InnerParams& prm, const double* h_lambda,
                     InnerWork& w, bool start_pure = true);

}  // namespace ksb
