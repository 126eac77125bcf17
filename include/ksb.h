/*
 * ksb.h -- C-ABI of the B200-native correction-step hot path of the
 * multilevel-correction adaptive FEM for Kohn-Sham (arXiv 2103.02824).
 *
 * Drop-in boundary. The reference exposes the path as a C++ namespace API
 * (no FFI of its own); each entry point below names the reference interface it
 * replaces (file:line under /root/reference/proj). Conventions:
 *   - every function returns an int status; codes are 1:1 with the reference's
 *     ksafem::Error string codes (proj/include/ksafem/types.hpp:20-32);
 *     ksb_last_error() returns the message of the last failure on this thread;
 *   - no exceptions cross the ABI; plain pointers and sizes only;
 *   - "d_" pointers are device pointers, "h_" pointers host pointers;
 *   - one CUDA stream per context; a context is driven by one host thread;
 *   - reductions are fixed-order (no floating-point atomics): reruns are bitwise stable.
 * Vector layout: orbital blocks are row-major (rows = dofs, ld >= N columns), so a
 * gathered row is N contiguous doubles.
 */
#ifndef KSB_H
#define KSB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (reference proj/include/ksafem/types.hpp:20-32) */
#define KSB_OK 0
#define KSB_NONCONVERGENCE 1
#define KSB_MISMATCHED_SPACES 2
#define KSB_SINGULAR_QUADRATURE 3
#define KSB_AMBIGUOUS_SELECTION 4
#define KSB_INTERNAL 5
#define KSB_INVALID_ARGUMENT 6
#define KSB_INVALID_DOMAIN 7
#define KSB_HIERARCHY 8
#define KSB_IO 9
#define KSB_CUDA 10

typedef struct ksb_mesh ksb_mesh;
typedef struct ksb_hier ksb_hier;
typedef struct ksb_ctx ksb_ctx;
typedef struct ksb_level ksb_level;

const char* ksb_last_error(void);
const char* ksb_code_name(int code);
int ksb_version(void);

/* ---------------- host mesh pipeline (bit-exact index data) ----------------
 * replaces mesh::build_box_mesh / uniform_refine / adapt_refine
 * (proj/include/ksafem/mesh.hpp:93-105, proj/src/mesh.cpp:281-368) */
int ksb_mesh_box(const double lo[3], const double hi[3], int n_per_axis, ksb_mesh** out);
int ksb_mesh_uniform_refine(const ksb_mesh* m, ksb_mesh** out);
int ksb_mesh_adapt_refine(const ksb_mesh* m, const int32_t* marked, int64_t n_marked, ksb_mesh** out);
void ksb_mesh_free(ksb_mesh* m);
/* sizes[0..7] = n_vertices, n_tets, n_boundary_faces, n_interior_faces, level,
 * n_parent_vertices, 0, 0 */
int ksb_mesh_sizes(const ksb_mesh* m, int64_t sizes[8]);
/* what: 0 xyz(double n*3) 1 tets(int32 T*4) 2 tuple(int32 T*4) 3 tag(int8 T)
 *       4 parent(int32 T) 5 vparent(int32 n*2) 6 on_boundary(uint8 n)
 *       7 boundary faces(int32 nbf*3) 8 interior faces(int32 nif*3)
 *       9 interior face tets(int32 nif*2) 10 interior face geometry(double nif*5) */
int ksb_mesh_get(const ksb_mesh* m, int what, void* h_dst);

/* ---------------- hierarchy (fem::SpaceHierarchy, proj/include/ksafem/fespace.hpp:65-81) */
int ksb_hier_create(ksb_hier** out);
int ksb_hier_push(ksb_hier* h, const ksb_mesh* m); /* copies the mesh handle (shared) */
void ksb_hier_free(ksb_hier* h);
int ksb_hier_levels(const ksb_hier* h);
/* composite prolongation P(0, level): per vertex <=4 (level-0 vertex, value), -1 padded.
 * replaces SpaceHierarchy::prolongation (proj/src/fespace.cpp:64-74) */
int ksb_hier_prolongation(const ksb_hier* h, int level, int32_t* h_col, double* h_val);

/* level `level` of a hierarchy as a mesh handle (shared, free with ksb_mesh_free) */
int ksb_hier_mesh(const ksb_hier* h, int level, ksb_mesh** out);

/* ---------------- binary dumps (the reference has none: its CSV/VTK outputs, proj/src/driver.cpp:509-543,
 * proj/src/mesh.cpp:259-279, stay text). Versioned little-endian files with an FNV-1a 64 checksum; meshes keep
 * their defining arrays (coordinates, tets, bisection tuples and tags, parents), faces are recomputed on load.
 * Errors: KSB_IO (open/short/corrupt/checksum), KSB_HIERARCHY (stored levels not nested). */
int ksb_hier_save(const ksb_hier* h, const char* path);
int ksb_hier_load(const char* path, ksb_hier** out);
int ksb_mesh_save(const ksb_mesh* m, const char* path);
int ksb_mesh_load(const char* path, ksb_mesh** out);
/* solver state of one level: lambdas (N), orbitals (interior block ni x N, read with leading dim ld),
 * Hartree potential (n, full) */
int ksb_state_save(const char* path, int level, int N, int64_t ni, int64_t n, const double* h_lambda,
                   const double* h_Phi, int ld, const double* h_w);
int ksb_state_sizes(const char* path, int64_t sizes[4]); /* level, N, ni, n */
int ksb_state_load(const char* path, double* h_lambda, double* h_Phi, int ld, double* h_w);

/* ---------------- device context ---------------- */
int ksb_ctx_create(int device, ksb_ctx** out);
void ksb_ctx_destroy(ksb_ctx* c);
int ksb_ctx_stream(ksb_ctx* c, void** stream); /* cudaStream_t of the context */
int ksb_ctx_sync(ksb_ctx* c);
/* per-kernel CUDA-event instrumentation (off by default); names: "spmm", "cg_update",
 * "assemble", ... ms = summed device time, count = launches since reset */
int ksb_ctx_set_profiling(ksb_ctx* c, int on);
int ksb_ctx_kernel_time(ksb_ctx* c, const char* name, double* ms, int64_t* count);
int ksb_ctx_kernel_launches(ksb_ctx* c, int64_t* total); /* all kernels launched since reset */
int ksb_ctx_reset_counters(ksb_ctx* c);
int ksb_malloc(ksb_ctx* c, void** d_ptr, int64_t bytes);
int ksb_free(ksb_ctx* c, void* d_ptr);
int ksb_memcpy_h2d(ksb_ctx* c, void* d_dst, const void* h_src, int64_t bytes); /* async on ctx stream */
int ksb_memcpy_d2h(ksb_ctx* c, void* h_dst, const void* d_src, int64_t bytes); /* async on ctx stream */

/* ---------------- fine level on the device ----------------
 * Uploads the FE space split, interior CSR patterns, the deterministic assembly
 * gather lists, P_int and the coarse-ancestor grouping of level `level` of `h`.
 * replaces FESpace + EllipticSolver's pattern gather (proj/src/fespace.cpp:7-18,
 * proj/src/solver.cpp:11-48) */
int ksb_level_create(ksb_ctx* c, const ksb_hier* h, int level, ksb_level** out);
void ksb_level_destroy(ksb_level* l);
/* sizes[0..9] = n, n_interior, n_boundary, n_tets, nnz_ii, nnz_ib, n_coarse_interior,
 * n_coarse_tets, n_coarse_vertices, 0 */
int ksb_level_sizes(const ksb_level* l, int64_t sizes[10]);
/* host copies of index data for bit-exactness checks: what 0 ii.ptr 1 ii.col 2 ib.ptr
 * 3 ib.col 4 interior vertex ids 5 P_int cols (ni*4) 6 P_int vals (double ni*4)
 * 7 T8 view columns (ni*16, ELL with 16 slots per row, padding -1; KSB_INVALID_ARGUMENT when a row of
 * the interior pattern is longer than 16 and the level has no T8 view)
 * 8 locality order perm (ni: natural row of ordered row i) 9 its pattern ptr (ni+1) 10 its columns (nnz_ii);
 * KSB_INVALID_ARGUMENT on levels without a locality order (those with a T8 view)
 * 11 stencil (DIA) view, 16 int32: {runs, centre run length 3, other run length, 1 if on the locality order,
 * first offset of each run (centre run first), [15] = n when the rows are an n^3 grid (else 0)}; runs = 0 when
 * the level has none (the solver's sliding-window
 * SpMM then does not apply)
 * 12 union-tile view sizes, 3 int32 {tiles, entries, rows per tile R} (tiles = 0 without the view); 13 tile rows
 * (tiles*R ordered rows, -1 padded) 14 entry ptr (tiles+1) 15 entries (ordered column per entry, padding entries
 * hold a valid row) 16 natural CSR slot of each of the R dense values per entry (entries*R, -1 = zero) -- the
 * wide-block SpMM's tiling of the locality-ordered pattern; 17 natural CSR slot of each locality-ordered slot
 * (nnz_ii) */
int ksb_level_index(const ksb_level* l, int what, void* h_dst);

/* ---------------- operators (interior blocks stored on the shared pattern) ----------------
 * A matrix is an id in the level's operator table. The interior-interior values live
 * on the ii pattern and the interior-boundary values on the ib pattern. */
#define KSB_MAT_S 0        /* stiffness (grad, grad), assemble_stiffness proj/src/assembly.cpp:93-105 */
#define KSB_MAT_M 1        /* unit mass, assemble_mass proj/src/assembly.cpp:135-138 */
#define KSB_MAT_AOP 2      /* a_op = 1/2 S + M_ext, make_level_ops proj/src/driver.cpp:41-43 */
#define KSB_MAT_USER0 8    /* free ids 8..31 */

/* analytic potential descriptor, evaluated at quadrature points */
#define KSB_POT_COULOMB 0  /* params (Z, x, y, z) per center; -sum Z/r, r<1e-12 -> 1e-10 (proj/src/ks_model.cpp:33-41) */
#define KSB_POT_GAUSSIAN 1 /* params (depth, width, x, y, z) per center; -sum d exp(-|x-c|^2/(2 w^2)) */

/* values(mat) = c_s*S + c_m*M + c_p*M_{pot} + c_w*M_{w}, each term assembled by the
 * 11-point Keast rule (proj/src/assembly.cpp:109-131) and combined slot-wise.
 * pot may be NULL (c_p ignored); d_w (nodal weight, length n, device) may be NULL. */
int ksb_mat_assemble(ksb_level* l, int mat, double c_s, double c_m, int pot_kind, int n_centers,
                     const double* h_pot_params, double c_p, const double* d_w, double c_w);
/* values(dst) = a*values(x) + b*values(y) */
int ksb_mat_axpby(ksb_level* l, int dst, double a, int x, double b, int y);
/* host copies of values: part 0 = ii (nnz_ii), part 1 = ib (nnz_ib) */
int ksb_mat_values(ksb_level* l, int mat, int part, double* h_dst);

/* Y = A_ii X on interior blocks (ni x N, row-major, ld >= N). replaces A_ii_ * p
 * (proj/src/solver.cpp:72) -- the K-SpMM kernel */
int ksb_spmm(ksb_level* l, int mat, const double* d_X, int N, int ldx, double* d_Y, int ldy);

/* ---------------- multi-RHS conjugate gradients ----------------
 * N independent preconditioned CG recurrences sharing one SpMM per iteration.
 * Per column: x0 = 0, zero-rhs exit, breakdown on !(pAp > 0), convergence on the
 * recursive residual confirmed by the true residual (else restart), as
 * EllipticSolver::pcg (proj/src/solver.cpp:57-111). Operator of column j is
 * A + sigma_j * B (B = shift_mat, may be -1 when no shifts). */
typedef struct {
    double tol;            /* relative residual (SolverOptions::tol, default 1e-9) */
    int max_iterations;    /* SolverOptions::max_iterations (default 20000) */
    int fixed_iterations;  /* >0: run exactly this many iterations, no stopping test (benchmark) */
    int precond;           /* 0 = Jacobi (default, fused); 1 = the reference's exact SGS (solver.cpp:50-55), level-scheduled
                              triangular solves, host-driven iterations: parity runs, no fixed-iteration mode */
    int check_every;       /* host polls convergence flags every k iterations (default 8) */
} ksb_cg_opts;

typedef struct {
    int iterations;
    double relative_residual;
    int converged;
    int breakdown; /* 1 = stopped on !(pAp > 0); fixed-iteration mode (no stopping test): the number of
                      iterations that saw !(pAp > 0) -- the column keeps iterating, alpha = 0 when pAp is
                      0 or non-finite */
} ksb_cg_stats;

int ksb_cg_defaults(ksb_cg_opts* o);
/* d_B, d_X: interior blocks ni x N (ld; ld even when N > 1, 16-byte column pairs).
 * h_sigma: N shifts or NULL. stats: N entries (host). */
int ksb_cg_solve(ksb_level* l, int mat, int shift_mat, const double* h_sigma, const double* d_B,
                 double* d_X, int N, int ld, const ksb_cg_opts* o, ksb_cg_stats* h_stats);
/* same with host buffers (H2D of B and D2H of X inside the call): the e2e entry point.
 * Any ld >= N; only the first N columns of each host row of X are written. */
int ksb_cg_solve_host(ksb_level* l, int mat, int shift_mat, const double* h_sigma, const double* h_B,
                      double* h_X, int N, int ld, const ksb_cg_opts* o, ksb_cg_stats* h_stats);


/* fem::EllipticSolver::solve / solve_zero_bc (proj/src/solver.cpp:113-135): interior rhs b_I - A_ib bc_B,
 * PCG (Jacobi) on A_ii, full-length x whose boundary entries are bc (0 when d_bc_full is NULL).
 * b and bc are full-length (n); interior entries of bc are ignored. */
int ksb_solve(ksb_level* l, int mat, const double* d_b_full, const double* d_bc_full, const ksb_cg_opts* o,
              double* d_x_full, ksb_cg_stats* h_stats);
/* EllipticSolver::min_diagonal (proj/src/solver.cpp:44): min over the interior diagonal of A_ii */
int ksb_mat_min_diag(ksb_level* l, int mat, double* h_out);


/* ---------------- the correction step (one outer iteration, proj/src/driver.cpp:106-150) ----------------
 * Orbitals are interior blocks (ni x ld, row-major): the correction algorithm keeps them in the
 * zero-trace space, so boundary values are structurally zero. Potentials (w, v_xc, rho) are
 * full-length nodal vectors (n). */
typedef struct {
    double tol_linear;  /* RunConfig::tol_linear (1e-9) */
    double tol_inner;   /* RunConfig::tol_inner (1e-8) */
    double score_floor; /* RunConfig::score_floor (1e-8) */
    int max_inner;      /* RunConfig::max_inner (400) */
    int nev_pad;        /* RunConfig::nev_scan_pad (4) */
    int check_every;    /* CG convergence poll interval */
    int fixed_sweeps;   /* > 0: inner loop runs exactly this many sweeps (diagnostics), else 0 */
    int norm_l1;        /* density change in L1 instead of H1 (RunConfig::outer_norm_l1, runconfig.hpp:32) */
    int precond;        /* 0: Jacobi orbital BVPs + multigrid Hartree (default); 1: the reference's exact SGS
                           (solver.cpp:50-55) in every linear solve of the step -- parity runs */
} ksb_step_opts;

typedef struct {
    int inner_iterations;
    int hartree_iterations;
    double delta; /* H1 (or, with norm_l1, L1) norm of the density change (the outer stopping quantity) */
    double ms_bvp, ms_hartree, ms_project, ms_inner, ms_total;
    int64_t cg_iterations; /* summed over orbitals and shift attempts */
} ksb_step_log;

#define KSB_XC_NONE 0
#define KSB_XC_XALPHA 1
#define KSB_XC_LDA 2

int ksb_step_defaults(ksb_step_opts* o);
/* model::MolecularSystem + the mode switches (proj/include/ksafem/ks_model.hpp:26-34,
 * runconfig.hpp:39-46). atoms: (Z, x, y, z) per nucleus. */
int ksb_system_set(ksb_level* l, const double* h_atoms, int n_atoms, int n_pairs, double occupancy, int xc_kind,
                   double alpha, double exchange_exponent, int hartree_on, int xc_on);
/* make_level_ops (proj/src/driver.cpp:35-47): S, M, a_op, plus the coarse blocks M_H, C_H */
int ksb_level_ops(ksb_level* l);
/* one outer iteration: lambda (N, host) and Phi / w (device) are updated in place.
 * h_attempts[i] = -1 when the unshifted solve converged, else the ladder rung; h_iters = CG iterations. */
int ksb_correction_step(ksb_level* l, const ksb_step_opts* o, double* h_lambda, double* d_Phi, int ld, double* d_w,
                        ksb_step_log* log, int* h_attempts, int* h_iters);
/* same with host buffers (H2D/D2H inside the call): the e2e entry point */
int ksb_correction_step_host(ksb_level* l, const ksb_step_opts* o, double* h_lambda, double* h_Phi, int ld,
                             double* h_w, ksb_step_log* log, int* h_attempts, int* h_iters);

/* Standard multilevel correction, the reference's comparison method (driver::solve_level_mlc,
 * proj/src/driver.cpp:200-302), split at its sweep loop so the host keeps the loop, the stopping test and the
 * iteration-cap error:
 *   ksb_mlc_begin: orbital BVPs with the warm start's potentials (h_lambda, d_Phi, d_w unchanged), Hartree
 *     boundary data from the phi_tilde density; the correction-space state starts pure (phi_H = 0, theta = 1).
 *   ksb_mlc_sweep: Hartree potential of the current density, pot = w + v_xc, one bordered solve per orbital with
 *     A_H1 + P^T M_pot P (sign-aligned with the previous sweep), expansion into d_Phi, lambdas into h_lambda,
 *     h_delta = H1 norm of the density change.
 *   ksb_mlc_finish: Hartree potential of the final density (zero when Hartree is off) and, if d_rho is not NULL,
 *     the density itself (full length). */
int ksb_mlc_begin(ksb_level* l, const ksb_step_opts* o, const double* h_lambda, const double* d_Phi, int ld,
                  const double* d_w, ksb_step_log* log, int* h_attempts, int* h_iters);
int ksb_mlc_sweep(ksb_level* l, const ksb_step_opts* o, double* h_lambda, double* d_Phi, int ld, double* h_delta);
int ksb_mlc_finish(ksb_level* l, const ksb_step_opts* o, double* d_w_full, double* d_rho_full);

/* scf::self_consistent_solve on the coarsest space (proj/src/scf.cpp:22-90), level 0 of the hierarchy:
 * dense lowest eigenpairs of the current Hamiltonian, linear density mixing, Hartree potential of the mixed
 * density. Outputs: lambdas (N, host), orbitals (interior block, device), mixed density and Hartree potential
 * (full length, device); history = density change per iteration. */
typedef struct {
    double tol;          /* density-change stop (RunConfig::tol_outer, 1e-6) */
    int max_iterations;  /* RunConfig::max_scf (200) */
    double mixing;       /* RunConfig::mixing (0.3) */
    int hartree_on, xc_on;
    double tol_eig;      /* Hartree solve tolerance (RunConfig::tol_eig, 1e-9) */
    int norm_l1;         /* density change in L1 instead of H1 (scf::Options::norm_l1, scf.hpp:19) */
} ksb_scf_opts;
int ksb_scf_defaults(ksb_scf_opts* o);
int ksb_coarse_scf(ksb_level* l, const ksb_scf_opts* o, double* h_lambda, double* d_Phi, int ld, double* d_rho_full,
                   double* d_w_full, int* h_iterations, double* h_history, int hist_cap);

/* pieces of the step, for parity checks against the reference's functions */
/* model::density + xc_potential_field (proj/src/ks_model.cpp:43-52,101-105); d_vxc may be NULL */
int ksb_density_xc(ksb_level* l, const double* d_Phi, int N, int ld, double* d_rho, double* d_vxc);
/* model::density (proj/src/ks_model.cpp:43-52) with an explicit occupancy, full length (boundary entries 0) */
int ksb_density(ksb_level* l, const double* d_Phi, int N, int ld, double occupancy, double* d_rho_full);
/* hartree::compute_moments (proj/src/hartree.cpp:15-63): q, centre[3], dipole[3], quadrupole[9] */
int ksb_moments(ksb_level* l, const double* d_rho, double h_out[16]);
/* hartree::boundary_values at the boundary vertices, boundary numbering (proj/src/hartree.cpp:76-82) */
int ksb_boundary_values(ksb_level* l, const double h_moments[16], double* d_bcb);
/* hartree::squared_density_load restricted to interior rows (proj/src/hartree.cpp:108-129) */
int ksb_sqload(ksb_level* l, const double* d_Phi, int N, int ld, double* d_out_int);
/* hartree::squared_density_load, full length n incl. boundary rows (proj/src/hartree.cpp:108-129) */
int ksb_sqload_full(ksb_level* l, const double* d_Phi, int N, int ld, double occupancy, double* d_out_full);
/* model::xc_potential_field (proj/src/ks_model.cpp:101-105): v_xc(rho) nodewise, full length */
int ksb_xc_field(ksb_level* l, int xc_kind, double alpha, double exchange_exponent, const double* d_rho_full,
                 double* d_vxc_full);
/* corr::bvp_hartree (proj/src/correction.cpp:67-75): full-length w with boundary data d_bcb */
int ksb_hartree_solve(ksb_level* l, const double* d_Phi, int N, int ld, const double* d_bcb, double tol,
                      double* d_w_full, int* h_iters);
/* OuterOperator + bvp_orbital for every orbital (proj/src/correction.cpp:15-61) */
int ksb_outer_solve(ksb_level* l, const ksb_step_opts* o, const double* d_what_full, const double* d_vxc_full,
                    const double* h_lambda, const double* d_Phi, int ld, double* d_PhiT, int* h_attempts,
                    int* h_iters, double* h_min_diag);
/* OuterOperator constructor (proj/src/correction.cpp:15-24): H = values(aop_mat) + M_{what + vxc} into the level's
 * H slot (one live OuterOperator per level); h_min_diag = min interior diagonal of H */
int ksb_outer_build(ksb_level* l, int aop_mat, const double* d_what_full, const double* d_vxc_full,
                    double* h_min_diag);
/* OuterOperator::solve_orbital for N orbitals (columns of d_Phi, interior block) against the built H
 * (proj/src/correction.cpp:26-61): unshifted PCG, then the shift ladder on the columns that failed */
int ksb_outer_apply(ksb_level* l, const ksb_step_opts* o, const double* h_lambda, const double* d_Phi, int N, int ld,
                    double* d_PhiT, int* h_attempts, int* h_iters);
/* corr::prepare_blocks (proj/src/correction.cpp:113-212): w_tilde0 (zero trace) and the lift ell, full length */
int ksb_prepare_blocks(ksb_level* l, const double* d_PhiT, int ld, const double* d_wt_full, const double* d_ell_full,
                       const double* d_vxc_full);
/* ledger access, codes as the oracle: 0 A_H1 1 A_H3 2 A_H4 3 M_H 4 C_H (nh x nh, row-major) 5 d_Hh
 * 6 lift_load 7 [zeta, lift_load0] 10 A_h4 (N nh nh) 11 b_H1 12 b_H3 13 b_H4 14 rhs 15 c_Hh 16 d_phi (N nh)
 * 17 beta1 18 beta3 19 beta4 20 gamma 21 zeta_phi (N) */
int ksb_blocks_get(ksb_level* l, int what, double* h_dst);
/* corr::inner_scf from the pure augmentation state (proj/src/correction.cpp:279-368) */
int ksb_inner_scf(ksb_level* l, const ksb_step_opts* o, const double* h_lambda, double* h_lambda_out,
                  double* h_phi_H, double* h_theta2, double* h_w_H, double* h_theta1, int* h_iterations,
                  double* h_history, int hist_cap);
/* corr::expand of the last inner state (proj/src/correction.cpp:370-381) */
int ksb_expand(ksb_level* l, const double* d_PhiT, int ld, const double* d_wt_full, const double* d_bcb,
               double* d_Phi, double* d_w_full);
/* fem::SpaceHierarchy::prolong one level up (proj/src/fespace.cpp:76-84, rows of prolongation_matrix :35-56), the
 * nested warm start of driver::run (proj/src/driver.cpp:367-371): out = P_step in, per column, summed in ascending
 * previous-vertex order without fused multiply-add (bit-exact with the reference's sparse product).
 * in: previous level, full vertex layout (in_interior = 0, n_prev rows) or interior block (1, zero boundary);
 * out: this level, full (out_interior = 0, n rows) or interior block (1, ni rows). Row-major, leading dims given. */
int ksb_prolong(ksb_level* l, const double* d_in, int in_interior, int ld_in, int ncols, double* d_out,
                int out_interior, int ld_out);
/* est::compute_indicators (proj/src/estimator.cpp:11-85): element residual of (V_ext + w + v_xc - lambda_i) phi_i
 * plus half-flux jumps across interior faces; d_eta gets eta_T^2 for every tet (n_tets), h_total_sq their sum.
 * Orbitals: interior block (N = the system's n_pairs columns); w, v_xc full length. */
int ksb_indicators(ksb_level* l, const double* h_lambda, const double* d_Phi, int ld, const double* d_w_full,
                   const double* d_vxc_full, double* d_eta, double* h_total_sq);
/* est::dorfler_mark (proj/src/estimator.cpp:87-104), host: descending eta, lower index first on ties, minimal
 * prefix reaching theta * total. h_marked needs room for n_tets entries. No device needed. */
int ksb_dorfler_mark(const double* h_eta, int64_t n_tets, double total_sq, double theta, int32_t* h_marked,
                     int64_t* h_n_marked);
/* l2_norm^2, h1_seminorm^2, h1_norm of a full-length nodal function (proj/src/assembly.cpp:251-287) */
int ksb_norms(ksb_level* l, const double* d_f_full, double h_out[3]);
/* fem::l1_norm of a full-length nodal function: integral of |f| by the Keast rule (proj/src/assembly.cpp:234-249,
 * 289-291) */
int ksb_l1_norm(ksb_level* l, const double* d_f_full, double* h_out);
/* model::total_energy (proj/src/ks_model.cpp:107-143): kinetic, external, hartree, xc, total */
int ksb_energy(ksb_level* l, const double* d_Phi, int N, int ld, const double* d_w_full, double h_out[5]);

#ifdef __cplusplus
}
#endif

#endif /* KSB_H */
