// K-PROJ interface (see project.cu).
#pragma once

#include "level.cuh"

namespace ksb {

constexpr int kSharedK = 58;  // A_H1, A_H3, A_H4 (3x16), d_Hh (4), zeta, lift_load (4), lift_load0
constexpr int kOrbK = 49;     // A_h4 (16), b_H1, b_H3, b_H4, c_Hh, d_phi (5x4), pad (4), rhs (4), 5 scalars
constexpr int kStride = 64;   // per (function, coarse tet) record in the partial buffer

/// coarse ledger on the device (row-major dense coarse blocks, interior coarse numbering)
struct ProjOut {
    int nh = 0, N = 0;
    DevBuf<double> part;
    DevBuf<double> pchunk;       // per-chunk partials on levels whose coarse tets are split into several chunks
    DevBuf<double> pgpart;       // per-item orbital partials of the aggregated (GEMM) projection
    DevBuf<double> shared_mats;  // A_H1, A_H3, A_H4
    DevBuf<double> A_h4;         // N x nh x nh
    DevBuf<double> shared_vecs;  // d_Hh, lift_load
    DevBuf<double> orb_vecs;     // per orbital: b_H1, b_H3, b_H4, c_Hh, d_phi, rhs
    DevBuf<double> shared_scal;  // zeta, lift_load0
    DevBuf<double> orb_scal;     // per orbital: beta1, beta3, beta4, gamma, zeta_phi
    DevBuf<int> offs;
    void ensure(int nh, int N, int nct);
};

/// wt_full = w_tilde0 (zero trace), ell_full = boundary lift, vxc_full: nodal, full length.
/// eext: per fine tet 16-entry M_ext element matrix (Keast rule), per level.
void project_blocks(Level& L, const double* Phi, int N, int ld, const double* wt_full, const double* ell_full,
                    const double* vxc_full, const double* eext, ProjOut& o);

}  // namespace ksb
