// Multi-RHS CG driver interface (see cg.cu).
#pragma once

#include "level.cuh"
#include "sgs.cuh"

namespace ksb {

struct CgOptions {
    double tol = 1e-9;
    int max_iterations = 20000;
    int fixed_iterations = 0;
    int check_every = 8;
    int precond = 0;  // 0: Jacobi (fused, production); 1: the reference's exact SGS (sgs.cu, parity runs)
};

struct CgColumnStats {
    int iterations = 0;
    double relative_residual = 0.0;
    int converged = 0;
    int breakdown = 0;
};

/// device pointers of the per-column scalar state (passed by value to kernels)
struct CgDev {
    double *bnorm, *rz, *rr, *alpha, *beta, *relres, *sigma;
    const double *diagA, *diagB;
    int *status, *check, *iters, *ctl;
    int* nonpos;  // fixed-iteration mode: iterations with !(p.Ap > 0) per column (recorded, column not retired)
    double *part0, *part1;
};

/// identity of a captured chunk of CG iterations: every kernel argument that can differ between solves
struct CgGraphKey {
    uint64_t level_uid;  // Level::uid: never reused, so a graph of a destroyed level can never match
    const void* ptrs[29];
    int ints[10];
    double tol;
};

struct CgGraph {
    CgGraphKey key;
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0;
};

struct CgWork {
    DevBuf<double> rbuf, pbuf, apbuf, scal, parts, diagA, diagB;
    DevBuf<double> lo_b, lo_x;  // B and X in the level's locality order (reordered solves)
    DevBuf<int> ints;
    double *R = nullptr, *P = nullptr, *AP = nullptr;
    int64_t cap_vec = 0;
    int cap_cols = 0, cap_blocks = 0;
    CgDev dev{};
    std::vector<CgGraph> graphs;  // chunks of iterations captured as CUDA graphs (small FIFO cache)
    SgsWork sgs;                  // blocks of the SGS parity path
    void ensure(int ni, int N, int ld, int max_blocks);
    /// drop the captured graphs of one level (ksb_level_destroy)
    void forget_level(uint64_t uid);
    ~CgWork();
};

void cg_solve(Ctx& c, Level& L, int mat, int shift_mat, const double* h_sigma, const double* d_B, double* d_X, int N,
              int ld, const CgOptions& o, CgColumnStats* stats, CgWork& w);
/// EllipticSolver::pcg with apply_sgs (proj/src/solver.cpp:50-111) for N columns, host-driven (sgs.cu)
void cg_solve_sgs(Ctx& c, Level& L, int mat, int shift_mat, const double* h_sigma, const double* d_B, double* d_X,
                  int N, int ld, const CgOptions& o, CgColumnStats* stats, CgWork& w);

} // namespace ksb
