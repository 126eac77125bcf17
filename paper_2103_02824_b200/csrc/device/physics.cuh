// Fine-level physics kernels (see physics.cu for reference anchors).
#pragma once

#include <array>

#include "geom.cuh"
#include "level.cuh"

namespace ksb {

struct Moments {
    double q;
    double c[3];
    double dip[3];
    double Q[3][3];
};

struct PhysWork {
    DevBuf<double> part, out, e4;
    void ensure(const Level& L);
};

/// rho = occ sum_i phi_i^2 and v_xc(rho), nodal, full-length outputs (boundary entries zero)
void rho_vxc(Level& L, const double* Phi, int N, int ld, double occ, const XcParams& xc, double* rho_full,
             double* vxc_full);
Moments moments(Level& L, const double* rho_full, PhysWork& w, const double box_center[3]);
/// multipole Dirichlet data at boundary vertices (boundary numbering)
void boundary_values(Level& L, const Moments& m, double* bcb);
/// out_int = scale * (occ sum_i phi_i^2, psi_j) on interior rows
void sqload(Level& L, const double* Phi, int N, int ld, double occ, double scale, double* out_int, PhysWork& w);
/// hartree::squared_density_load, all n rows (proj/src/hartree.cpp:108-129)
void sqload_full(Level& L, const double* Phi, int N, int ld, double occ, double* out_full, PhysWork& w);
/// model::xc_potential_field (proj/src/ks_model.cpp:101-105)
void xc_field(Level& L, const XcParams& xc, const double* rho_full, double* vxc_full);
/// residual-indicator device data (face lists, per-tet face gather), uploaded on first use
struct EstimatorData {
    DevBuf<int32_t> ftets, tptr, tface;
    DevBuf<double> fgeom, contrib, part, scal, lam, atoms;
    bool ready = false;
    void ensure(Level& L);
};
/// est::compute_indicators (proj/src/estimator.cpp:11-85): eta_T^2 per tet into d_eta (nt); returns the total
double indicators(Level& L, EstimatorData& E, const std::vector<double>& atoms, const double* h_lambda, int N,
                  const double* d_Phi, int ld, const double* d_w, const double* d_vxc, double* d_eta);
/// y_int -= A_ib(mat) bcb (Dirichlet lift, reference proj/src/solver.cpp:123)
void lift(Level& L, int mat, const double* bcb, double* y_int);
/// squared L2 norm and squared H1 seminorm of a full-length nodal function
std::array<double, 2> norms_sq(Level& L, const double* f_full, PhysWork& w);
/// fem::l1_norm (proj/src/assembly.cpp:289-291): integral of |f| by the Keast rule
double l1_norm(Level& L, const double* f_full, PhysWork& w);
/// kinetic, external, hartree, xc, total
std::array<double, 5> energy(Level& L, const double* Phi, int N, int ld, const double* rho_full, const double* w_full,
                             const std::vector<double>& atoms, double occ, const XcParams& xc, PhysWork& w);

/// one-level prolongation of nodal columns (see ksb_prolong)
void prolong(Level& L, const double* in, bool in_interior, int ld_in, int ncols, double* out, bool out_interior,
             int ld_out);

} // namespace ksb
