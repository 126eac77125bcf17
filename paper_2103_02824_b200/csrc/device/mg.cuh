// Geometric multigrid on the nested hierarchy, used as the preconditioner of the single-column stiffness
// solves (Hartree potential). The reference solves these with SGS-PCG (proj/src/solver.cpp:50-111); the
// contract kept here is the same PCG recurrence, recursive-then-true residual acceptance, restart and
// breakdown test -- only the preconditioner differs.
//
//   levels      1 .. L-1 are uploaded from the hierarchy's meshes and assemble their own stiffness matrices;
//               level L is the caller's Level (its S); level 0 is solved exactly with C_H^-1 (dense, already
//               built for the inner iteration).
//   transfer    the one-step prolongation rows (fem::prolongation_matrix, proj/src/fespace.cpp:35-56)
//               restricted to interior rows and columns; restriction is its transpose, stored row-wise so the
//               sums run in a fixed order (no atomics).
//   smoother    nu sweeps of damped Jacobi before and after the coarse correction (symmetric V-cycle).
#pragma once

#include <memory>

#include "cg.cuh"
#include "level.cuh"

namespace ksb {

struct MgLevel {
    Level* L = nullptr;           // operator owner (S = mats[0])
    std::unique_ptr<Level> own;   // intermediate levels
    int ni = 0, nc = 0;           // interior dofs here and on the next coarser level
    DevBuf<int32_t> pcol;         // ni x 4: coarser interior index or -1
    DevBuf<double> pval;          // ni x 4
    DevBuf<int32_t> rptr, ridx;   // transpose: coarser row -> (row here, weight), ascending row
    DevBuf<double> rval;
    DevBuf<double> dinv, b, x, y, r;
};

struct Multigrid {
    bool ready = false;
    int top = 0;                  // fine level index L
    std::vector<std::unique_ptr<MgLevel>> lv;  // lv[1..top]
    const double* CHi = nullptr;  // level-0 interior stiffness inverse (n_H x n_H)
    int nH = 0;
    int nu = 2;
    double omega = 0.6;
    DevBuf<double> b0, x0, part, scal, p, q, z, r, t;
    // one PCG iteration past the convergence test (V-cycle, r.z, p update, A p, x/r update) as a CUDA graph,
    // one per parity of the r.z scalar slot; built on first use, pointers fixed for the Level's lifetime
    cudaGraphExec_t iter_exec[2] = {nullptr, nullptr};
    double* iter_x = nullptr;  // the x the graphs were captured with
    ~Multigrid();
};

/// builds levels 1..L-1, the transfers and the Jacobi diagonals (the top level's S must be assembled)
void mg_setup(Level& L, Multigrid& mg, const double* d_CHi);
/// PCG on the top level's S with one V-cycle as preconditioner; x = 0 start, b and x interior vectors
CgColumnStats mg_pcg(Level& L, Multigrid& mg, const double* d_b, double* d_x, double tol, int max_iterations);

} // namespace ksb
