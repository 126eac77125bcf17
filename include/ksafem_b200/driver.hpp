// The callers of the path (proj/src/driver.cpp:35-47 make_level_ops, :94-163 solve_level_corrected), with the
// fused device correction step as the B200 form of the outer iteration's body.
#pragma once

#include "ksafem_b200/correction.hpp"
#include "ksafem_b200/estimator.hpp"
#include "ksafem_b200/scf.hpp"

namespace ksafem::driver {

struct LevelOps {
    fem::SpacePtr space;
    SpMat S, M, a_op;  // a_op = 1/2 S + M_{v_ext}
    std::unique_ptr<fem::EllipticSolver> stiffness;
    fem::Prolongation P_full;
};

LevelOps make_level_ops(const fem::SpaceHierarchy& hier, int level, const model::MolecularSystem& sys,
                        WorkerPool* pool = nullptr);

struct StepOptions {
    double tol_linear = 1e-9;
    double tol_inner = 1e-8;
    double score_floor = 1e-8;
    int max_inner = 400;
    int nev_scan_pad = 4;
    bool hartree = true;
    bool xc = true;
    bool norm_l1 = false;  // density change in L1 instead of H1 (RunConfig::outer_norm_l1)
};

struct StepLog {
    int inner_iterations = 0;
    int hartree_iterations = 0;
    double delta = 0;  // H1 (L1 with norm_l1) norm of the density change
    double ms_bvp = 0, ms_hartree = 0, ms_project = 0, ms_inner = 0, ms_total = 0;
    std::vector<int> attempts, cg_iterations;
};

/// One outer iteration of solve_level_corrected (proj/src/driver.cpp:106-150) on device-resident state:
/// orbitals (interior block, row-major ni x N) and w stay in HBM between steps.
class CorrectionState {
public:
    CorrectionState(const LevelOps& ops, const model::MolecularSystem& sys, const StepOptions& opt,
                    const VecX& lambdas, const std::vector<fem::FEFunction>& orbitals, const fem::FEFunction& w);
    StepLog step();
    VecX lambdas() const { return lambda_; }
    std::vector<fem::FEFunction> orbitals() const;
    fem::FEFunction hartree() const;

private:
    fem::SpacePtr space_;
    int N_ = 0, ld_ = 0;
    StepOptions opt_;
    VecX lambda_;
    b200::DeviceBuffer phi_, w_;
};

struct LevelResult {
    VecX lambdas;
    std::vector<fem::FEFunction> orbitals;
    fem::FEFunction hartree;
    int outer_iterations = 0;
    std::vector<int> inner_iterations;
    std::vector<double> deltas;
};

/// outer loop until the density change drops below tol_outer; "nonconvergence" at max_outer
LevelResult solve_level_corrected(const LevelOps& ops, const model::MolecularSystem& sys, const StepOptions& opt,
                                  const VecX& lambdas, const std::vector<fem::FEFunction>& orbitals,
                                  const fem::FEFunction& w, double tol_outer = 1e-6, int max_outer = 40);

/// The standard multilevel correction on one level (driver::solve_level_mlc, proj/src/driver.cpp:200-302):
/// orbital BVPs with the warm potentials, then correction-space sweeps rebuilding the potential-weighted coarse
/// blocks from the current density until its H1 change drops below tol_outer ("nonconvergence" after max_scf).
LevelResult solve_level_mlc(const LevelOps& ops, const model::MolecularSystem& sys, const StepOptions& opt,
                            const VecX& lambdas, const std::vector<fem::FEFunction>& orbitals,
                            const fem::FEFunction& w, double tol_outer = 1e-6, int max_scf = 200);

/// RunConfig::Mode subset the device path runs (proj/include/ksafem/runconfig.hpp:9): the corrected method with
/// (accelerated) or without (linear) the nonlinear terms, and the standard MLC comparison method
enum class Mode { accelerated, linear, standard_mlc };

/// the adaptive run (proj/src/driver.cpp:306-435); refinement by Doerfler marks of the residual indicators, or
/// uniform (BASELINE's cfg1) when `uniform` is set
struct RunConfig {
    model::MolecularSystem system;
    int n_coarse = 16;
    int max_levels = 8;
    double theta = 0.4;
    double tol_outer = 1e-6;
    double tol_inner = 1e-8;
    double tol_linear = 1e-9;
    double tol_eig = 1e-9;
    double mixing = 0.3;
    int max_outer = 40;
    int max_inner = 400;
    int max_scf = 200;
    double score_floor = 1e-8;
    int nev_scan_pad = 4;
    bool uniform = false;
    bool outer_norm_l1 = false;  // density-change norm: H1 unless set (proj/include/ksafem/runconfig.hpp:32)
    Mode mode = Mode::accelerated;
};

struct LevelRecord {
    int level = 0;
    int n_tets = 0;
    int n_dofs = 0;
    VecX lambdas;
    model::EnergyBreakdown energy;
    double eta_sq_total = 0;
    int outer_iterations = 0;
    std::vector<int> inner_iterations;
    double t_solve = 0, t_estimate = 0, t_refine = 0, t_total = 0;
};

struct RunLog {
    std::vector<LevelRecord> records;
    bool aborted = false;
    std::string abort_reason;
    double wall_seconds = 0;
};

RunLog run(const RunConfig& cfg);

} // namespace ksafem::driver
