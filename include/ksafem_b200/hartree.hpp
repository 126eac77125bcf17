// mirrors proj/include/ksafem/hartree.hpp for the functions on the path (K-MOM, K-SQLOAD, Poisson on S).
#pragma once

#include "ksafem_b200/solver.hpp"

namespace ksafem::hartree {

struct MultipoleMoments {
    double charge = 0;
    Vec3 center = Vec3::Zero();
    Vec3 dipole = Vec3::Zero();
    Mat3 quadrupole = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // row-major, traceless
};

MultipoleMoments compute_moments(const fem::FEFunction& rho);
/// Dirichlet data: full-length vector with multipole values at boundary nodes (interior entries zero)
VecX boundary_values(const MultipoleMoments& m, const fem::FESpace& space);
/// b_j = occupancy sum_i int phi_i^2 psi_j (exact degree-3 integrand), full length
VecX squared_density_load(const fem::FESpace& space, const std::vector<fem::FEFunction>& orbitals,
                          double occupancy);
/// (grad w, grad v) = 4 pi (occ sum phi_i^2, v) with Dirichlet data bc; `stiffness` must be the stiffness
/// solver of `space` (the level's S)
fem::FEFunction solve_hartree_exact(const fem::EllipticSolver& stiffness, const fem::FESpace& space,
                                    const std::vector<fem::FEFunction>& orbitals, double occupancy,
                                    const VecX& bc, double tol = 1e-9);

} // namespace ksafem::hartree
