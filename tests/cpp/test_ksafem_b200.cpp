// The reference's own tests for the path, restated against the ksafem-compatible B200 API
// (include/ksafem_b200/*.hpp -> libksafem_b200.so -> C-ABI -> sm_100a kernels). Needs a GPU.
// Each case cites the reference test it follows (proj/tests/<file>:<lines>). Run: test_ksafem_b200 [filter]
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "ksafem_b200/driver.hpp"

using namespace ksafem;

// ---------------------------------------------------------------- minimal harness
static std::vector<std::pair<std::string, std::function<void()>>>& registry() {
    static std::vector<std::pair<std::string, std::function<void()>>> r;
    return r;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().emplace_back(n, std::move(f)); }
};
static int g_fail = 0, g_checks = 0;
#define TEST_CASE(name, fn) \
    static void fn();       \
    static Reg reg_##fn(name, fn); \
    static void fn()
#define CHECK(cond)                                                                      \
    do {                                                                                 \
        ++g_checks;                                                                      \
        if (!(cond)) {                                                                   \
            ++g_fail;                                                                    \
            std::fprintf(stderr, "  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                                \
    } while (0)
#define CHECK_THROWS_CODE(expr, want)                                                          \
    do {                                                                                       \
        ++g_checks;                                                                            \
        std::string got = "none";                                                              \
        try {                                                                                  \
            expr;                                                                              \
        } catch (const ksafem::Error& e) {                                                     \
            got = e.code();                                                                    \
        }                                                                                      \
        if (got != (want)) {                                                                   \
            ++g_fail;                                                                          \
            std::fprintf(stderr, "  expected %s, got %s at %s:%d\n", want, got.c_str(), __FILE__, __LINE__); \
        }                                                                                      \
    } while (0)

static bool approx(double a, double b, double eps) {  // doctest::Approx(b).epsilon(eps) == a
    return std::fabs(a - b) < eps * (1.0 + std::max(std::fabs(a), std::fabs(b)));
}
static double nrm(const VecX& v) {
    double s = 0;
    for (double x : v) s += x * x;
    return std::sqrt(s);
}
static mesh::Box cube(double lo, double hi) {
    mesh::Box b;
    b.lo = Vec3(lo, lo, lo);
    b.hi = Vec3(hi, hi, hi);
    return b;
}

/// A x restricted to the interior rows, from the level's CSR values (host product: test checker only)
static VecX interior_product(const SpMat& A, const fem::FESpace& V, const VecX& x) {
    std::vector<int> pi, ci, pb, cb;
    A.pattern(0, pi, ci);
    A.pattern(1, pb, cb);
    const VecX vi = A.interior_values(), vb = A.boundary_values();
    const auto& I = V.interior_dofs();
    const auto& B = V.boundary_dofs();
    VecX y(I.size(), 0.0);
    for (size_t r = 0; r < I.size(); ++r) {
        for (int k = pi[r]; k < pi[r + 1]; ++k) y[r] += vi[size_t(k)] * x[size_t(I[size_t(ci[size_t(k)])])];
        for (int k = pb[r]; k < pb[r + 1]; ++k) y[r] += vb[size_t(k)] * x[size_t(B[size_t(cb[size_t(k)])])];
    }
    return y;
}

// ---------------------------------------------------------------- mesh (test_mesh.cpp)
TEST_CASE("box mesh and refinement counts", t_mesh) {
    auto m = mesh::build_box_mesh(cube(-1, 1), 8);
    CHECK(m->n_vertices() == 729 && m->n_tets() == 3072);
    auto f = mesh::uniform_refine(*m);
    CHECK(f->n_tets() == 8 * 3072 && f->n_vertices() == 17 * 17 * 17);
    auto a = mesh::adapt_refine(*m, {0, 100, 2000});
    CHECK(a->n_tets() > m->n_tets());
    CHECK_THROWS_CODE(mesh::build_box_mesh(cube(1, 1), 2), "invalid-domain");
}

// ---------------------------------------------------------------- assembly (test_assembly.cpp:64-274)
TEST_CASE("stiffness rows annihilate constants, l2 norm of 1 is the volume", t_assembly) {
    auto V = std::make_shared<fem::FESpace>(mesh::build_box_mesh(cube(-1, 1), 3));
    const SpMat S = fem::assemble_stiffness(*V);
    const VecX ones(size_t(V->n_dofs()), 1.0);
    double worst = 0;
    for (double y : interior_product(S, *V, ones)) worst = std::max(worst, std::fabs(y));
    CHECK(worst < 1e-12);
    fem::FEFunction one(V, ones);
    CHECK(std::fabs(fem::l2_norm(one) - std::sqrt(8.0)) < 1e-12);
    CHECK(fem::h1_seminorm(one) < 1e-12);
    // (grad x, grad x) = |Omega| for u = x
    fem::FEFunction u(V);
    const auto xyz = V->mesh().vertices();
    for (int i = 0; i < V->n_dofs(); ++i) u.coeffs[size_t(i)] = xyz[size_t(i)][0];
    CHECK(std::fabs(fem::h1_seminorm(u) * fem::h1_seminorm(u) - 8.0) < 1e-11);
    // weighted mass with a unit weight equals the mass matrix
    const SpMat M = fem::assemble_mass(*V), Mw = fem::assemble_mass(*V, one);
    const VecX a = M.interior_values(), b = Mw.interior_values();
    double d = 0;
    for (size_t k = 0; k < a.size(); ++k) d = std::max(d, std::fabs(a[k] - b[k]));
    CHECK(d < 1e-15);
    // linear combination on the device
    const SpMat H = 0.5 * S + M;
    const VecX h = H.interior_values(), s = S.interior_values();
    double e = 0;
    for (size_t k = 0; k < h.size(); ++k) e = std::max(e, std::fabs(h[k] - (0.5 * s[k] + a[k])));
    CHECK(e < 1e-15);
}

// ---------------------------------------------------------------- solver (test_assembly.cpp:184-230)
TEST_CASE("manufactured solves and the residual contract", t_solver) {
    auto V = std::make_shared<fem::FESpace>(mesh::build_box_mesh(cube(0, 1), 4));
    const SpMat S = fem::assemble_stiffness(*V);
    fem::EllipticSolver solver(S, V);
    // -lap u = 0 with u = x on the boundary reproduces u = x
    const auto xyz = V->mesh().vertices();
    VecX bc(size_t(V->n_dofs()), 0.0), zero(size_t(V->n_dofs()), 0.0);
    for (int d : V->boundary_dofs()) bc[size_t(d)] = xyz[size_t(d)][0];
    fem::SolverOptions opt;
    opt.tol = 1e-12;
    fem::SolveStats st;
    const VecX u = solver.solve(zero, bc, opt, &st);
    double worst = 0;
    for (int i = 0; i < V->n_dofs(); ++i) worst = std::max(worst, std::fabs(u[size_t(i)] - xyz[size_t(i)][0]));
    CHECK(st.converged && worst < 1e-9);
    // residual contract and the one-shot nonconvergence error
    const VecX b(size_t(V->n_dofs()), 1.0);
    opt.tol = 1e-10;
    solver.solve_zero_bc(b, opt, &st);
    CHECK(st.converged && st.relative_residual <= 1e-10);
    opt.max_iterations = 1;
    solver.solve_zero_bc(b, opt, &st);
    CHECK(!st.converged);
    CHECK_THROWS_CODE(fem::solve_spd(S, b, V, VecX(), 1e-30), "nonconvergence");
    CHECK(S.interior_values().size() > 0 && solver.min_diagonal() > 0);
}

// ---------------------------------------------------------------- hartree (test_hartree.cpp:57-143)
static fem::FEFunction gaussian(fem::SpacePtr V, double mass, double sigma, Vec3 c) {
    fem::FEFunction rho(V, fem::Role::density);
    const auto xyz = V->mesh().vertices();
    const double norm = mass / (std::pow(M_PI, 1.5) * sigma * sigma * sigma);
    for (int i = 0; i < V->n_dofs(); ++i) {
        double r2 = 0;
        for (int d = 0; d < 3; ++d) r2 += (xyz[size_t(i)][d] - c[d]) * (xyz[size_t(i)][d] - c[d]);
        rho.coeffs[size_t(i)] = norm * std::exp(-r2 / (sigma * sigma));
    }
    return rho;
}

TEST_CASE("moments, boundary data, exact-square Poisson solves", t_hartree) {
    auto V = std::make_shared<fem::FESpace>(mesh::build_box_mesh(cube(-4, 4), 6));
    const auto m0 = hartree::compute_moments(fem::FEFunction(V));
    CHECK(m0.charge == 0.0);
    CHECK(nrm(hartree::boundary_values(m0, *V)) == 0.0);
    const auto m = hartree::compute_moments(gaussian(V, 4.0, 1.0, Vec3()));
    CHECK(approx(m.charge, 4.0, 0.02));
    CHECK(std::sqrt(m.dipole[0] * m.dipole[0] + m.dipole[1] * m.dipole[1] + m.dipole[2] * m.dipole[2]) < 1e-8);
    CHECK(std::fabs(m.quadrupole[0] + m.quadrupole[4] + m.quadrupole[8]) < 1e-10);

    // zero-trace orbital: the load is positive and sums to occ * ||phi||^2
    fem::FEFunction phi(V, fem::Role::wavefunction);
    const auto xyz = V->mesh().vertices();
    for (int i : V->interior_dofs()) {
        const auto& x = xyz[size_t(i)];
        phi.coeffs[size_t(i)] = std::exp(-(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]));
    }
    const VecX load = hartree::squared_density_load(*V, {phi}, 2.0);
    double sum = 0;
    for (double x : load) sum += x;
    const double l2 = fem::l2_norm(phi);
    CHECK(std::fabs(sum - 2.0 * l2 * l2) < 1e-10 * sum);

    const SpMat S = fem::assemble_stiffness(*V);
    fem::EllipticSolver stiff(S, V);
    const auto w0 = hartree::solve_hartree_exact(stiff, *V, {fem::FEFunction(V, fem::Role::wavefunction)}, 2.0, VecX());
    CHECK(nrm(w0.coeffs) == 0.0);
    const auto rho = model::density({phi}, 2.0);
    const VecX bc = hartree::boundary_values(hartree::compute_moments(rho), *V);
    const auto w = hartree::solve_hartree_exact(stiff, *V, {phi}, 2.0, bc, 1e-11);
    bool trace = true;
    for (int d : V->boundary_dofs()) trace = trace && w.coeffs[size_t(d)] == bc[size_t(d)];
    CHECK(trace);
    // the potential of a centred density is centrally symmetric (test_hartree.cpp:123-143)
    int pairs = 0;
    std::map<std::array<long, 3>, int> key;
    for (int i = 0; i < V->n_dofs(); ++i)
        key[{std::lround(xyz[size_t(i)][0] * 1e6), std::lround(xyz[size_t(i)][1] * 1e6), std::lround(xyz[size_t(i)][2] * 1e6)}] = i;
    double asym = 0;
    for (int i = 0; i < V->n_dofs(); ++i) {
        auto it = key.find({-std::lround(xyz[size_t(i)][0] * 1e6), -std::lround(xyz[size_t(i)][1] * 1e6),
                            -std::lround(xyz[size_t(i)][2] * 1e6)});
        if (it != key.end()) {
            asym = std::max(asym, std::fabs(w.coeffs[size_t(i)] - w.coeffs[size_t(it->second)]));
            ++pairs;
        }
    }
    CHECK(pairs > 100 && asym < 1e-7);
}

// ---------------------------------------------------------------- model (test_model.cpp:36-176)
TEST_CASE("density, xc field, energy", t_model) {
    auto V = std::make_shared<fem::FESpace>(mesh::build_box_mesh(cube(-1, 1), 2));
    fem::FEFunction phi(V, fem::Role::wavefunction);
    for (int i : V->interior_dofs()) phi.coeffs[size_t(i)] = 0.5;
    const auto rho = model::density({phi}, 2.0);
    bool ok = true;
    for (int i : V->interior_dofs()) ok = ok && rho.coeffs[size_t(i)] == 0.5;
    CHECK(ok);
    model::XcFunctional xa;
    fem::FEFunction r(V, VecX(size_t(V->n_dofs()), M_PI / 3.0));
    const auto v = model::xc_potential_field(xa, r);
    CHECK(std::fabs(v.coeffs[0] - (-1.5 * 0.77298)) < 1e-14);
    const auto v0 = model::xc_potential_field(xa, fem::FEFunction(V));
    CHECK(nrm(v0.coeffs) == 0.0);
    model::MolecularSystem sys;
    sys.atoms.push_back({1.0, Vec3(0.3, 0, 0)});
    sys.domain = cube(-1, 1);
    const auto e0 = model::total_energy(sys, {fem::FEFunction(V, fem::Role::wavefunction)}, fem::FEFunction(V));
    CHECK(e0.total == 0.0 && e0.kinetic == 0.0);
    CHECK_THROWS_CODE(model::density({phi, fem::FEFunction(std::make_shared<fem::FESpace>(
                                                  mesh::build_box_mesh(cube(-1, 1), 2)))},
                                     2.0),
                      "mismatched-spaces");
}

// ---------------------------------------------------------------- correction (test_correction.cpp:86-478)
struct Fixture {  // test_correction.cpp:25-55
    fem::SpaceHierarchy hier;
    model::MolecularSystem sys;
    std::unique_ptr<driver::LevelOps> ops;
    int lev = 1;
    Fixture() {
        sys.atoms.push_back({2.0, Vec3(0.31, -0.17, 0.05)});
        sys.n_pairs = 2;
        sys.occupancy = 1.0;
        sys.domain = cube(-2, 2);
        sys.xc.kind = model::XcKind::x_alpha;
        auto m = mesh::build_box_mesh(sys.domain, 2);
        hier.push(m);
        hier.push(mesh::uniform_refine(*m));
        ops = std::make_unique<driver::LevelOps>(driver::make_level_ops(hier, lev, sys));
    }
    fem::FEFunction random_orbital(unsigned seed) {
        std::mt19937 g(seed);
        std::uniform_real_distribution<double> u(-1, 1);
        fem::FEFunction f(ops->space, fem::Role::wavefunction);
        for (int i : ops->space->interior_dofs()) f.coeffs[size_t(i)] = u(g);
        return f;
    }
};

TEST_CASE("orbital correction: trivial, deterministic, shift ladder", t_outer) {
    Fixture F;
    const auto& V = F.ops->space;
    const fem::FEFunction z(V);
    corr::OuterOperator op(V, F.ops->a_op, &F.ops->M, z, z, 1e-11);
    const auto zero = corr::bvp_orbital(op, 0.7, fem::FEFunction(V, fem::Role::wavefunction));
    CHECK(nrm(zero.coeffs) == 0.0);
    const auto phi = F.random_orbital(2);
    const auto a = corr::bvp_orbital(op, -0.4, phi), b = corr::bvp_orbital(op, -0.4, phi);
    CHECK(a.coeffs == b.coeffs);
    // the batched form equals the per-orbital calls
    const auto ab = op.solve_orbitals(VecX{-0.4, -0.4}, {phi, phi});
    double d = 0;
    for (size_t k = 0; k < ab[1].coeffs.size(); ++k) d = std::max(d, std::fabs(ab[1].coeffs[k] - a.coeffs[k]));
    CHECK(d < 1e-9 * nrm(a.coeffs));
    CHECK_THROWS_CODE(corr::OuterOperator(V, F.ops->a_op, &F.ops->S, z, z, 1e-9), "invalid-argument");
}

TEST_CASE("hartree correction contract", t_bvp_hartree) {  // test_correction.cpp:169-210
    Fixture F;
    const auto& V = F.ops->space;
    const auto p1 = F.random_orbital(5), p2 = F.random_orbital(6);
    const auto xyz = V->mesh().vertices();
    VecX bc(size_t(V->n_dofs()), 0.0);
    for (int d : V->boundary_dofs()) {
        const auto& x = xyz[size_t(d)];
        bc[size_t(d)] = 0.3 / (1.0 + std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]));
    }
    const auto w = corr::bvp_hartree(*F.ops->stiffness, F.ops->M, {p1, p2}, 1.0, bc, 1e-11);
    bool trace = true;
    for (int d : V->boundary_dofs()) trace = trace && w.coeffs[size_t(d)] == bc[size_t(d)];
    CHECK(trace);
    fem::FEFunction s1 = p1, s2 = p2;
    for (auto& x : s1.coeffs) x *= std::sqrt(3.0);
    for (auto& x : s2.coeffs) x *= std::sqrt(3.0);
    const auto ws = corr::bvp_hartree(*F.ops->stiffness, F.ops->M, {s1, s2}, 1.0, VecX(), 1e-11);
    const auto wu = corr::bvp_hartree(*F.ops->stiffness, F.ops->M, {p1, p2}, 1.0, VecX(), 1e-11);
    double d = 0, mx = 0;
    for (size_t k = 0; k < wu.coeffs.size(); ++k) {
        d = std::max(d, std::fabs(ws.coeffs[k] - 3.0 * wu.coeffs[k]));
        mx = std::max(mx, std::fabs(wu.coeffs[k]));
    }
    CHECK(d < 1e-8 * std::max(1.0, mx));
}

TEST_CASE("ledger symmetry, zero inputs, inner iteration and expansion", t_blocks) {
    Fixture F;
    const auto& V = F.ops->space;
    const fem::FEFunction z(V);
    // zero augmentation: the orbital-dependent blocks vanish (test_correction.cpp:322-340)
    auto B0 = corr::prepare_blocks(F.hier.space(0), V, F.ops->P_full, F.ops->S, F.ops->M, F.ops->a_op,
                                   {fem::FEFunction(V, fem::Role::wavefunction), fem::FEFunction(V, fem::Role::wavefunction)},
                                   z, z, 1.0, false, VecX());
    CHECK(nrm(B0.A_H3().a) == 0.0 && nrm(B0.b_H1(0)) == 0.0 && nrm(B0.rhs(1)) == 0.0);
    const MatX A1 = B0.A_H1(), MH = B0.M_H();
    double asym = 0, scale = 0;
    for (int i = 0; i < A1.rows; ++i)
        for (int j = 0; j < A1.cols; ++j) {
            asym = std::max(asym, std::fabs(A1(i, j) - A1(j, i)));
            scale = std::max(scale, std::fabs(A1(i, j)));
        }
    CHECK(asym <= 1e-13 * scale);
    // a realistic outer state: correct the eigen-ish start, then the inner loop converges and expands to
    // mass-normalised orbitals (test_correction.cpp:380-467)
    fem::FEFunction s1(V, fem::Role::wavefunction), s2(V, fem::Role::wavefunction);
    const auto xyz = V->mesh().vertices();
    for (int i : V->interior_dofs()) {
        const auto& x = xyz[size_t(i)];
        const double r = std::sqrt((x[0] - 0.31) * (x[0] - 0.31) + (x[1] + 0.17) * (x[1] + 0.17) + (x[2] - 0.05) * (x[2] - 0.05));
        s1.coeffs[size_t(i)] = std::exp(-2.0 * r);
        s2.coeffs[size_t(i)] = (x[0] - 0.31) * std::exp(-r);
    }
    const VecX lam{-1.5, -0.3};
    corr::OuterOperator op(V, F.ops->a_op, &F.ops->M, z, z, 1e-10);
    const auto pt = op.solve_orbitals(lam, {s1, s2});
    const auto rho = model::density(pt, 1.0);
    const VecX bc = hartree::boundary_values(hartree::compute_moments(rho), *V);
    const auto wt = corr::bvp_hartree(*F.ops->stiffness, F.ops->M, pt, 1.0, bc, 1e-10);
    const auto vxc = model::xc_potential_field(F.sys.xc, rho);
    auto B = corr::prepare_blocks(F.hier.space(0), V, F.ops->P_full, F.ops->S, F.ops->M, F.ops->a_op, pt, wt, vxc,
                                  1.0, true, bc);
    const auto init = corr::pure_augmentation_state(B, lam);
    corr::InnerOptions io;
    io.tol = 1e-9;
    const auto r = corr::inner_scf(B, init, io);
    CHECK(r.iterations >= 1 && r.iterations < 400);
    const auto e = corr::expand(r.state, B);
    for (const auto& f : e.orbitals) CHECK(std::fabs(fem::l2_norm(f) - 1.0) < 1e-6);
    CHECK_THROWS_CODE(corr::expand(init, B), "invalid-argument");
}

// ---------------------------------------------------------------- estimator (test_estimator.cpp:35-100)
TEST_CASE("indicators: zero state, linear function, marking", t_estimator) {
    fem::SpaceHierarchy hier;
    model::MolecularSystem sys;
    sys.n_pairs = 1;
    sys.occupancy = 1.0;
    sys.domain = cube(-1, 1);
    sys.xc.kind = model::XcKind::none;
    sys.atoms.push_back({1.0, Vec3(0.3, 0.1, -0.2)});
    auto m = mesh::build_box_mesh(sys.domain, 3);
    hier.push(m);
    const auto ops = driver::make_level_ops(hier, 0, sys);
    const auto& V = ops.space;
    const fem::FEFunction z(V);
    const auto ind0 = est::compute_indicators(*V, sys, VecX{0.0}, {fem::FEFunction(V, fem::Role::wavefunction)}, z, z);
    CHECK(ind0.total_sq == 0.0 && int(ind0.eta_sq.size()) == V->mesh().n_tets());
    CHECK(est::dorfler_mark(ind0, 0.4).empty());
    fem::FEFunction phi(V, fem::Role::wavefunction);
    const auto xyz = V->mesh().vertices();
    for (int i : V->interior_dofs()) {
        const auto& x = xyz[size_t(i)];
        phi.coeffs[size_t(i)] = std::exp(-2.0 * (x[0] * x[0] + x[1] * x[1] + x[2] * x[2]));
    }
    const auto ind = est::compute_indicators(*V, sys, VecX{-0.5}, {phi}, z, z);
    double sum = 0;
    for (double e : ind.eta_sq) sum += e;
    CHECK(ind.total_sq > 0 && std::fabs(sum - ind.total_sq) <= 1e-12 * ind.total_sq);
    const auto mk = est::dorfler_mark(ind, 0.4);
    double got = 0, mn = 1e300;
    for (int t : mk) {
        got += ind.eta_sq[size_t(t)];
        mn = std::min(mn, ind.eta_sq[size_t(t)]);
    }
    CHECK(got >= 0.4 * ind.total_sq && got - mn < 0.4 * ind.total_sq);
    CHECK_THROWS_CODE(est::dorfler_mark(ind, 1.5), "invalid-argument");
}

// ---------------------------------------------------------------- driver: a small level loop end to end
TEST_CASE("solve_level_corrected converges from a hydrogenic start", t_driver) {
    fem::SpaceHierarchy hier;
    model::MolecularSystem sys;
    sys.atoms.push_back({2.0, Vec3()});
    sys.n_pairs = 1;
    sys.occupancy = 2.0;
    sys.domain = cube(-6, 6);
    sys.xc.kind = model::XcKind::lda_pz81;
    auto m = mesh::build_box_mesh(sys.domain, 6);
    hier.push(m);
    hier.push(mesh::uniform_refine(*m));
    const auto ops = driver::make_level_ops(hier, 1, sys);
    const auto& V = ops.space;
    fem::FEFunction phi(V, fem::Role::wavefunction);
    const auto xyz = V->mesh().vertices();
    for (int i : V->interior_dofs()) {
        const auto& x = xyz[size_t(i)];
        phi.coeffs[size_t(i)] = std::exp(-1.7 * std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]));
    }
    const double n0 = fem::l2_norm(phi);
    for (auto& c : phi.coeffs) c /= n0;
    const auto rho = model::density({phi}, 2.0);
    const VecX bc = hartree::boundary_values(hartree::compute_moments(rho), *V);
    const auto w = hartree::solve_hartree_exact(*ops.stiffness, *V, {phi}, 2.0, bc, 1e-10);
    driver::StepOptions so;
    const auto res = driver::solve_level_corrected(ops, sys, so, VecX{-0.6}, {phi}, w, 1e-6, 40);
    CHECK(res.deltas.back() < 1e-6);
    CHECK(res.lambdas[0] < -0.3 && res.lambdas[0] > -1.2);
    const auto e = model::total_energy(sys, res.orbitals, res.hartree);
    CHECK(e.total < -2.0 && e.total > -3.5);
    std::printf("  level-1 He: lambda %.10f, E %.10f, %d outer steps\n", res.lambdas[0], e.total, res.outer_iterations);
}

TEST_CASE("solve_level_mlc and the standard_mlc run", t_mlc) {
    fem::SpaceHierarchy hier;
    model::MolecularSystem sys;
    sys.atoms.push_back({2.0, Vec3()});
    sys.n_pairs = 1;
    sys.occupancy = 2.0;
    sys.domain = cube(-6, 6);
    sys.xc.kind = model::XcKind::lda_pz81;
    auto m = mesh::build_box_mesh(sys.domain, 6);
    hier.push(m);
    hier.push(mesh::uniform_refine(*m));
    const auto ops = driver::make_level_ops(hier, 1, sys);
    const auto& V = ops.space;
    fem::FEFunction phi(V, fem::Role::wavefunction);
    const auto xyz = V->mesh().vertices();
    for (int i : V->interior_dofs()) {
        const auto& x = xyz[size_t(i)];
        phi.coeffs[size_t(i)] = std::exp(-1.7 * std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]));
    }
    const double n0 = fem::l2_norm(phi);
    for (auto& c : phi.coeffs) c /= n0;
    const auto rho = model::density({phi}, 2.0);
    const VecX bc = hartree::boundary_values(hartree::compute_moments(rho), *V);
    const auto w = hartree::solve_hartree_exact(*ops.stiffness, *V, {phi}, 2.0, bc, 1e-10);
    driver::StepOptions so;
    const auto res = driver::solve_level_mlc(ops, sys, so, VecX{-0.6}, {phi}, w, 1e-6, 200);
    CHECK(res.deltas.back() < 1e-6);
    CHECK(res.lambdas[0] < -0.2 && res.lambdas[0] > -1.2);
    std::printf("  level-1 He (standard MLC): lambda %.10f, %d sweeps\n", res.lambdas[0], res.outer_iterations);

    driver::RunConfig cfg;
    cfg.system = sys;
    cfg.n_coarse = 4;
    cfg.max_levels = 3;
    cfg.uniform = true;
    cfg.mode = driver::Mode::standard_mlc;
    const auto log = driver::run(cfg);
    CHECK(!log.aborted);
    CHECK(log.records.size() == 3);
}

// ---------------------------------------------------------------- scf + run (scf.cpp, driver.cpp:306-435)
TEST_CASE("coarse SCF of cfg1 and the adaptive run", t_run) {
    model::MolecularSystem sys;
    sys.atoms.push_back({2.0, Vec3()});
    sys.n_pairs = 1;
    sys.occupancy = 2.0;
    sys.domain = cube(-10, 10);
    sys.xc.kind = model::XcKind::lda_pz81;
    fem::SpaceHierarchy hier;
    hier.push(mesh::build_box_mesh(sys.domain, 8));
    const auto r = scf::initial_coarse_solve(sys, hier.space(0), 1e-6);
    // the oracle's coarse SCF of cfg1 (tests/golden/cfg1_oracle_trajectory.json via tests/cfg1_oracle.py)
    CHECK(r.iterations == 37);
    CHECK(std::fabs(r.lambdas[0] - (-0.00526096437936834)) < 1e-8 * 0.0053 + 1e-14);
    std::printf("  cfg1 coarse SCF: %d iterations, lambda %.14f\n", r.iterations, r.lambdas[0]);

    driver::RunConfig cfg;
    cfg.system = sys;
    cfg.system.domain = cube(-6, 6);
    cfg.system.atoms[0].position = Vec3(0.3, -0.2, 0.1);
    cfg.n_coarse = 4;
    cfg.max_levels = 4;
    const auto log = driver::run(cfg);
    CHECK(!log.aborted);
    CHECK(log.records.size() == 4);
    for (size_t k = 1; k < log.records.size(); ++k) CHECK(log.records[k].n_dofs >= log.records[k - 1].n_dofs);
    for (const auto& rec : log.records)
        std::printf("  level %d: %d dofs, lambda %.10f, E %.10f, eta^2 %.6e\n", rec.level, rec.n_dofs, rec.lambdas[0],
                    rec.energy.total, rec.eta_sq_total);
}

int main(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    if (filter && std::strcmp(filter, "--list") == 0) {
        for (auto& t : registry()) std::printf("%s\n", t.first.c_str());
        return 0;
    }
    int run = 0;
    for (auto& t : registry()) {
        if (filter && t.first.find(filter) == std::string::npos) continue;
        const int before = g_fail;
        try {
            t.second();
        } catch (const std::exception& e) {
            ++g_fail;
            std::fprintf(stderr, "  exception: %s\n", e.what());
        }
        ++run;
        std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", t.first.c_str());
    }
    std::printf("%d cases, %d checks, %d failed\n", run, g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
