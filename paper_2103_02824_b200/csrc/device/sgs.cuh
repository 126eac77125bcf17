// Exact SGS-preconditioned CG for parity runs (see sgs.cu).
#pragma once

#include "level.cuh"

namespace ksb {

struct CgOptions;
struct CgColumnStats;

struct SgsWork {
    DevBuf<double> R, Z, P, AP, T, part, scal;
    DevBuf<int> iact;
};

/// z = (D+U)^-1 D' (D+L)^-1 r for N columns (operator A + sigma_c B when B is given); tmp: ni x ld scratch
void sgs_apply(Level& L, SgsPlan& pl, const double* A, const double* Bv, const double* d_sigma, int N, int ld,
               const double* r, double* z, double* tmp);

}  // namespace ksb
