// mirrors proj/include/ksafem/correction.hpp. The blocks of the augmented systems live on the device
// (K-PROJ ledger) and the inner iteration runs there (K-INNER); AugmentedBlocks is a handle with host
// accessors for the ledger, AugmentedState / InnerResult / Expanded carry host copies.
#pragma once

#include "ksafem_b200/hartree.hpp"
#include "ksafem_b200/ks_model.hpp"

namespace ksafem::corr {

class OuterOperator {
public:
    /// H = a_op + M_{w_hat + v_xc}; `mass` must be the unit mass of `space` (make_level_ops' M). One live
    /// OuterOperator per space: a newer one on the same space replaces the device H.
    OuterOperator(fem::SpacePtr space, const SpMat& a_op, const SpMat* mass, const fem::FEFunction& w_hat,
                  const fem::FEFunction& v_xc, double tol_linear, WorkerPool* pool = nullptr);

    const fem::FESpace& space() const { return *space_; }
    const SpMat& mass() const { return *mass_; }
    double min_diagonal() const { return min_diag_; }

    /// solve H u = lambda_prev M phi_prev (zero trace); on non-convergence the level-shift ladder
    fem::FEFunction solve_orbital(double lambda_prev, const fem::FEFunction& phi_prev) const;
    /// all orbitals as one multi-RHS block solve (the B200 form of the per-orbital parallel_for)
    std::vector<fem::FEFunction> solve_orbitals(const VecX& lambda_prev,
                                                const std::vector<fem::FEFunction>& phi_prev) const;

private:
    fem::SpacePtr space_;
    const SpMat* mass_;
    double tol_;
    double min_diag_ = 0;
    uint64_t generation_ = 0;
};

fem::FEFunction bvp_orbital(const OuterOperator& op, double lambda_prev, const fem::FEFunction& phi_prev);

fem::FEFunction bvp_hartree(const fem::EllipticSolver& stiffness, const SpMat& mass,
                            const std::vector<fem::FEFunction>& phi_tilde, double occupancy, const VecX& bc,
                            double tol);

struct AugmentedBlocks {
    fem::SpacePtr space_H;
    fem::SpacePtr space_h;
    int n_orbitals = 0;
    double occupancy = 2.0;
    bool hartree_on = true;
    std::vector<VecX> phi_tilde;  // augmentation vectors (fine, zero trace)
    VecX w_tilde0;
    VecX ell;
    uint64_t generation = 0;  // device ledger generation these blocks describe

    // ledger accessors (host copies of the device blocks; interior coarse indexing)
    MatX A_H1() const;
    MatX A_H3() const;
    MatX A_H4() const;
    MatX M_H() const;
    MatX C_H() const;
    VecX d_Hh() const;
    VecX lift_load() const;
    double zeta() const;
    double lift_load0() const;
    MatX A_h4(int i) const;
    VecX b_H1(int i) const;
    VecX b_H3(int i) const;
    VecX b_H4(int i) const;
    VecX rhs(int i) const;
    VecX c_Hh(int i) const;
    VecX d_phi(int i) const;
    VecX beta1() const;
    VecX beta3() const;
    VecX beta4() const;
    VecX gamma_mass() const;
    VecX zeta_phi() const;
};

/// P_full, S_f, M_f, a_f must be the level's own (driver::make_level_ops of space_h); the device reads them
/// from the level. hartree_bc: full-length Dirichlet data, or empty when the electrostatic term is off.
AugmentedBlocks prepare_blocks(fem::SpacePtr space_H, fem::SpacePtr space_h, const fem::Prolongation& P_full,
                               const SpMat& S_f, const SpMat& M_f, const SpMat& a_f,
                               const std::vector<fem::FEFunction>& phi_tilde, const fem::FEFunction& w_tilde,
                               const fem::FEFunction& v_xc, double occupancy, bool hartree_on,
                               const VecX& hartree_bc, WorkerPool* pool = nullptr);

struct AugmentedState {
    VecX lambda;
    std::vector<VecX> phi_H;
    VecX theta2;
    VecX w_H;
    double theta1 = 0;
};

AugmentedState pure_augmentation_state(const AugmentedBlocks& blocks, const VecX& lambda_init);

struct InnerOptions {
    double tol = 1e-8;
    int max_iterations = 400;
    int dense_threshold = 800;
    double score_floor = 1e-8;
    int nev_scan_pad = 4;
    WorkerPool* pool = nullptr;
};

struct InnerResult {
    AugmentedState state;
    int iterations = 0;
    std::vector<double> history;
};

/// from the pure augmentation state (the only start the reference uses)
InnerResult inner_scf(const AugmentedBlocks& blocks, const AugmentedState& init, const InnerOptions& opt);

struct Expanded {
    VecX lambda;
    std::vector<fem::FEFunction> orbitals;
    fem::FEFunction hartree;
};

/// phi_i = P phi_{i,H} + theta_{2,i} phi_tilde_i, w = ell + P w_H + theta_1 w_tilde0; `s` must be the state the
/// last inner_scf on these blocks returned (the device keeps it)
Expanded expand(const AugmentedState& s, const AugmentedBlocks& blocks);

} // namespace ksafem::corr
