// CPU ORACLE -- TEST INFRASTRUCTURE ONLY. C entry points for ctypes (tests/, smoke(), bench.py baseline legs).
// Arrays of orbitals are row-major (n rows = dofs, N columns), like the device layout.
#include <cmath>
#include <cstring>
#include <map>

#include "oracle_core.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const OrcError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return E_INTERNAL;
    }
}

struct Problem {
    System sys;
    Hier hier;
    std::map<int, std::unique_ptr<LevelOps>> ops;
    LevelOps& level(int k) {
        auto it = ops.find(k);
        if (it == ops.end()) it = ops.emplace(k, std::make_unique<LevelOps>(make_level_ops(hier, k, sys))).first;
        return *it->second;
    }
    const Space& space(int k) const { return *hier.spaces.at(k); }
};

std::vector<Vec> unpack(const double* rm, int n, int N) {
    std::vector<Vec> o(N, Vec(n));
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < N; ++j) o[j][i] = rm[size_t(i) * N + j];
    return o;
}
void pack(const std::vector<Vec>& o, double* rm) {
    const int N = int(o.size());
    if (!N) return;
    const int n = int(o[0].size());
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < N; ++j) rm[size_t(i) * N + j] = o[j][i];
}
void put_csc(const Csc& A, int* ptr, int* idx, double* val) {
    if (ptr) std::memcpy(ptr, A.ptr.data(), A.ptr.size() * sizeof(int));
    if (idx) std::memcpy(idx, A.idx.data(), A.idx.size() * sizeof(int));
    if (val) std::memcpy(val, A.val.data(), A.val.size() * sizeof(double));
}
}  // namespace

struct orc_mesh {
    MeshP m;
};
struct orc_problem {
    Problem p;
    Vec last_scf_rho;
    std::vector<double> last_scf_hist;
};
struct orc_operator {
    std::unique_ptr<Elliptic> E;
    Csc A;
};
struct orc_blocks {
    Blocks B;
    AState last;
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

// ---------------- mesh ----------------
int orc_mesh_box(const double* lo, const double* hi, int n, orc_mesh** out) {
    return guard([&] { *out = new orc_mesh{box_mesh(V3{{lo[0], lo[1], lo[2]}}, V3{{hi[0], hi[1], hi[2]}}, n)}; });
}
int orc_mesh_uniform(const orc_mesh* m, orc_mesh** out) {
    return guard([&] { *out = new orc_mesh{uniform_refine(*m->m)}; });
}
int orc_mesh_adapt(const orc_mesh* m, const int* marks, int64_t n, orc_mesh** out) {
    return guard([&] { *out = new orc_mesh{adapt_refine(*m->m, std::vector<int>(marks, marks + n))}; });
}
void orc_mesh_free(orc_mesh* m) { delete m; }
int orc_mesh_sizes(const orc_mesh* m, int64_t* s) {
    return guard([&] {
        s[0] = m->m->nv();
        s[1] = m->m->nt();
        s[2] = int64_t(m->m->bfaces.size());
        s[3] = int64_t(m->m->ifaces.size());
        s[4] = m->m->level;
        s[5] = m->m->n_parent_vertices;
    });
}
int orc_mesh_get(const orc_mesh* mh, int what, void* dst) {
    return guard([&] {
        const Mesh& m = *mh->m;
        switch (what) {
            case 0: std::memcpy(dst, m.verts.data(), m.verts.size() * sizeof(V3)); break;
            case 1: std::memcpy(dst, m.tets.data(), m.tets.size() * 16); break;
            case 2: std::memcpy(dst, m.tuple.data(), m.tuple.size() * 16); break;
            case 3: std::memcpy(dst, m.tag.data(), m.tag.size()); break;
            case 4: std::memcpy(dst, m.parent.data(), m.parent.size() * 4); break;
            case 5: std::memcpy(dst, m.vparent.data(), m.vparent.size() * 8); break;
            case 6: {
                auto* o = static_cast<uint8_t*>(dst);
                for (size_t i = 0; i < m.on_boundary.size(); ++i) o[i] = uint8_t(m.on_boundary[i]);
                break;
            }
            case 7: std::memcpy(dst, m.bfaces.data(), m.bfaces.size() * 12); break;
            case 8: std::memcpy(dst, m.ifaces.data(), m.ifaces.size() * 12); break;
            case 9: std::memcpy(dst, m.iface_tets.data(), m.iface_tets.size() * 8); break;
            default: fail(E_ARG, "unknown mesh array");
        }
    });
}
int orc_mesh_conforming(const orc_mesh* m) { return m->m->conforming(nullptr) ? 1 : 0; }
int orc_mesh_total_volume(const orc_mesh* m, double* v) {
    return guard([&] {
        double s = 0;
        for (int t = 0; t < m->m->nt(); ++t) s += m->m->tet_volume(t);
        *v = s;
    });
}

// ---------------- problem / hierarchy ----------------
int orc_problem_create(const double* atoms, int n_atoms, int n_pairs, double occ, int xc_kind, double alpha,
                       double p_exch, int hartree_on, int xc_on, orc_problem** out) {
    return guard([&] {
        auto* p = new orc_problem;
        p->p.sys.atoms.assign(atoms, atoms + 4 * n_atoms);
        p->p.sys.n_pairs = n_pairs;
        p->p.sys.occ = occ;
        p->p.sys.xc_kind = xc_kind;
        p->p.sys.alpha = alpha;
        p->p.sys.p_exch = p_exch;
        p->p.sys.hartree_on = hartree_on != 0;
        p->p.sys.xc_on = xc_on != 0 && xc_kind != 0;
        *out = p;
    });
}
void orc_problem_free(orc_problem* p) { delete p; }
int orc_problem_push(orc_problem* p, const orc_mesh* m) {
    return guard([&] { p->p.hier.push(m->m); });
}
int orc_level_sizes(orc_problem* p, int level, int64_t* s) {
    return guard([&] {
        auto& o = p->p.level(level);
        const Space& V = *o.V;
        s[0] = V.n();
        s[1] = V.ni();
        s[2] = int64_t(V.boundary.size());
        s[3] = V.mesh->nt();
        s[4] = o.stiff->Aii.nnz();
        s[5] = o.stiff->Aib.nnz();
        s[6] = p->p.space(0).ni();
    });
}
int orc_interior(orc_problem* p, int level, int* dst) {
    return guard([&] {
        const auto& v = p->p.space(level).interior;
        std::memcpy(dst, v.data(), v.size() * 4);
    });
}
/// composite P(0, level) rows, <=4 per row, -1 padded (col ascending)
int orc_prolongation(orc_problem* p, int level, int* col, double* val) {
    return guard([&] {
        const Csc P = p->p.hier.prolongation(0, level);
        const Csc Pt = P.transpose();  // columns = fine rows
        for (int r = 0; r < P.rows; ++r) {
            int w = 0;
            for (int k = Pt.ptr[r]; k < Pt.ptr[r + 1]; ++k) {
                if (w >= 4) fail(E_INTERNAL, "prolongation row wider than 4");
                col[4 * r + w] = Pt.idx[k];
                val[4 * r + w] = Pt.val[k];
                ++w;
            }
            for (; w < 4; ++w) {
                col[4 * r + w] = -1;
                val[4 * r + w] = 0.0;
            }
        }
    });
}

// ---------------- operators ----------------
/// A = c_s S + c_m M + c_p M_pot + c_w M_w, then Dirichlet-reduced with the chosen preconditioner
int orc_operator_build(orc_problem* p, int level, double c_s, double c_m, int pot_kind, int n_centers,
                       const double* params, double c_p, const double* w, double c_w, int precond, orc_operator** out) {
    return guard([&] {
        const auto& Vp = p->p.hier.spaces.at(level);
        const Space& V = *Vp;
        Csc A;
        bool have = false;
        auto acc = [&](const Csc& T, double c) {
            if (!have) {
                A = scale(T, c);
                have = true;
            } else {
                A = add(A, c, T);
            }
        };
        if (c_s != 0.0) acc(assemble_stiffness(V), c_s);
        if (c_m != 0.0) acc(assemble_mass(V), c_m);
        if (params && n_centers > 0 && c_p != 0.0) {
            Potential pot;
            pot.kind = pot_kind;
            pot.p.assign(params, params + (pot_kind == 0 ? 4 : 5) * n_centers);
            acc(assemble_mass_pot(V, pot), c_p);
        }
        if (w && c_w != 0.0) acc(assemble_mass_nodal(V, Vec(w, w + V.n())), c_w);
        if (!have) acc(assemble_mass(V), 0.0);
        auto* o = new orc_operator;
        o->A = std::move(A);
        o->E = std::make_unique<Elliptic>(o->A, Vp, precond);
        *out = o;
    });
}
void orc_operator_free(orc_operator* o) { delete o; }
int orc_operator_nnz(orc_operator* o, int64_t* s) {
    return guard([&] {
        s[0] = o->E->Aii.nnz();
        s[1] = o->E->Aib.nnz();
        s[2] = o->E->Aii.rows;
        s[3] = o->A.nnz();
        s[4] = o->A.rows;
    });
}
/// the full n x n matrix (CSC) before Dirichlet reduction
int orc_operator_full(orc_operator* o, int* ptr, int* idx, double* val) {
    return guard([&] { put_csc(o->A, ptr, idx, val); });
}
/// EllipticSolver::solve (proj/src/solver.cpp:113-131) with full-length b, bc (may be null), x;
/// stats: iterations, converged, breakdown
int orc_operator_solve(orc_operator* o, const double* b, const double* bc, double tol, int maxit, double* x,
                       int* stats, double* relres) {
    return guard([&] {
        const int n = o->A.rows;
        const Space& V = *o->E->V;
        const auto& bd = V.boundary;
        Vec xb(bd.size());
        for (size_t i = 0; i < bd.size(); ++i) xb[i] = bc ? bc[bd[i]] : 0.0;
        Vec rhs(V.ni());
        for (int i = 0; i < V.ni(); ++i) rhs[i] = b[V.interior[i]];
        if (!xb.empty()) {
            const Vec t = o->E->Aib.mul(xb);
            for (int i = 0; i < V.ni(); ++i) rhs[i] -= t[i];
        }
        SolveStats st;
        const Vec xi = o->E->pcg(rhs, tol, maxit, &st);
        for (int i = 0; i < n; ++i) x[i] = 0.0;
        for (int i = 0; i < V.ni(); ++i) x[V.interior[i]] = xi[i];
        for (size_t i = 0; i < bd.size(); ++i) x[bd[i]] = xb[i];
        stats[0] = st.iterations;
        stats[1] = st.converged;
        stats[2] = st.breakdown;
        *relres = st.relres;
    });
}
int orc_operator_ii(orc_operator* o, int* ptr, int* idx, double* val) {
    return guard([&] { put_csc(o->E->Aii, ptr, idx, val); });
}
int orc_operator_ib(orc_operator* o, int* ptr, int* idx, double* val) {
    return guard([&] { put_csc(o->E->Aib, ptr, idx, val); });
}
int orc_operator_min_diag(orc_operator* o, double* d) {
    return guard([&] { *d = o->E->min_diag; });
}
/// y = A_ii x (interior vectors)
int orc_operator_spmv(orc_operator* o, const double* x, double* y) {
    return guard([&] {
        const int ni = o->E->Aii.rows;
        const Vec r = o->E->Aii.mul(Vec(x, x + ni));
        std::memcpy(y, r.data(), sizeof(double) * ni);
    });
}
/// per-column PCG on interior blocks (row-major ni x N); stats: iterations, converged, breakdown (int[3N]), relres[N]
int orc_operator_pcg(orc_operator* o, const double* B, double* X, int N, double tol, int maxit, int fixed,
                     int* istats, double* relres) {
    return guard([&] {
        const int ni = o->E->Aii.rows;
        const auto cols = unpack(B, ni, N);
        std::vector<Vec> xs(N);
#pragma omp parallel for schedule(dynamic, 1)
        for (int j = 0; j < N; ++j) {
            SolveStats st;
            xs[j] = o->E->pcg(cols[j], tol, maxit, &st, fixed);
            if (istats) {
                istats[3 * j] = st.iterations;
                istats[3 * j + 1] = st.converged;
                istats[3 * j + 2] = st.breakdown;
            }
            if (relres) relres[j] = st.relres;
        }
        pack(xs, X);
    });
}

// ---------------- small pieces for the pinning tests ----------------
int orc_keast(double* bary, double* w) {
    return guard([&] {
        const auto& r = keast();
        for (size_t q = 0; q < r.size(); ++q) {
            w[q] = r[q].w;
            for (int k = 0; k < 4; ++k) bary[4 * q + k] = r[q].b[k];
        }
    });
}
int orc_prolongation_nnz(orc_problem* p, int from, int to, int64_t* nnz) {
    return guard([&] { *nnz = p->p.hier.prolongation(from, to).nnz(); });
}
int orc_prolongation_csc(orc_problem* p, int from, int to, int* ptr, int* idx, double* val) {
    return guard([&] { put_csc(p->p.hier.prolongation(from, to), ptr, idx, val); });
}
int orc_load_nodal(orc_problem* p, int level, const double* f, double* out) {
    return guard([&] {
        const Space& V = p->p.space(level);
        const Vec b = load_nodal(V, Vec(f, f + V.n()));
        std::memcpy(out, b.data(), sizeof(double) * V.n());
    });
}

// ---------------- level-ops matrices (S, M, a_op) ----------------
int orc_level_matrix(orc_problem* p, int level, int which, int part, int* ptr, int* idx, double* val) {
    return guard([&] {
        auto& o = p->p.level(level);
        const Csc* A = which == 0 ? &o.S : which == 1 ? &o.M : &o.a_op;
        Elliptic E(*A, o.V, 0);
        put_csc(part == 0 ? E.Aii : E.Aib, ptr, idx, val);
    });
}

// ---------------- physics ----------------
int orc_density(const double* orb, int n, int N, double occ, double* rho) {
    return guard([&] {
        const Vec r = density(unpack(orb, n, N), occ);
        std::memcpy(rho, r.data(), sizeof(double) * n);
    });
}
int orc_xc_potential(orc_problem* p, const double* rho, int n, double* out) {
    return guard([&] {
        for (int i = 0; i < n; ++i) out[i] = xc_potential(p->p.sys, rho[i]);
    });
}
int orc_xc_energy_density(orc_problem* p, const double* rho, int n, double* out) {
    return guard([&] {
        for (int i = 0; i < n; ++i) out[i] = xc_energy_density(p->p.sys, rho[i]);
    });
}
/// moments: q, c[3], dip[3], Q[9]
int orc_moments(orc_problem* p, int level, const double* rho, double* out) {
    return guard([&] {
        const Space& V = p->p.space(level);
        const Moments m = compute_moments(V, Vec(rho, rho + V.n()));
        out[0] = m.q;
        for (int d = 0; d < 3; ++d) {
            out[1 + d] = m.c[d];
            out[4 + d] = m.dip[d];
            for (int e = 0; e < 3; ++e) out[7 + 3 * d + e] = m.Q[d][e];
        }
    });
}
int orc_boundary_values(orc_problem* p, int level, const double* mom, double* bc) {
    return guard([&] {
        const Space& V = p->p.space(level);
        Moments m;
        m.q = mom[0];
        for (int d = 0; d < 3; ++d) {
            m.c[d] = mom[1 + d];
            m.dip[d] = mom[4 + d];
            for (int e = 0; e < 3; ++e) m.Q[d][e] = mom[7 + 3 * d + e];
        }
        const Vec b = boundary_values(m, V);
        std::memcpy(bc, b.data(), sizeof(double) * V.n());
    });
}
int orc_sqload(orc_problem* p, int level, const double* orb, int N, double* out) {
    return guard([&] {
        const Space& V = p->p.space(level);
        const Vec b = squared_density_load(V, unpack(orb, V.n(), N), p->p.sys.occ);
        std::memcpy(out, b.data(), sizeof(double) * V.n());
    });
}
int orc_hartree_exact(orc_problem* p, int level, const double* orb, int N, const double* bc, double tol, double* w,
                      int* iters) {
    return guard([&] {
        auto& o = p->p.level(level);
        const Space& V = *o.V;
        Vec load = squared_density_load(V, unpack(orb, V.n(), N), p->p.sys.occ);
        for (double& x : load) x *= 4.0 * 3.14159265358979323846;
        SolveStats st;
        const Vec r = o.stiff->solve(load, bc ? Vec(bc, bc + V.n()) : Vec(), tol, &st);
        if (!st.converged) fail(E_NONCONV, "hartree solve stalled");
        if (iters) *iters = st.iterations;
        std::memcpy(w, r.data(), sizeof(double) * V.n());
    });
}
int orc_energy(orc_problem* p, int level, const double* orb, int N, const double* w, double* out) {
    return guard([&] {
        const Space& V = p->p.space(level);
        const Energy e = total_energy(p->p.sys, V, unpack(orb, V.n(), N), Vec(w, w + V.n()));
        out[0] = e.kinetic;
        out[1] = e.external;
        out[2] = e.hartree;
        out[3] = e.xc;
        out[4] = e.total;
    });
}
int orc_indicators(orc_problem* p, int level, const double* lambdas, const double* orb, int N, const double* w,
                   const double* vxc, double* eta, double* total_sq) {
    return guard([&] {
        const Space& V = p->p.space(level);
        const Vec e = compute_indicators(p->p.sys, V, Vec(lambdas, lambdas + N), unpack(orb, V.n(), N),
                                         Vec(w, w + V.n()), Vec(vxc, vxc + V.n()), total_sq);
        std::copy(e.begin(), e.end(), eta);
    });
}
int orc_dorfler(const double* eta, int64_t nt, double total_sq, double theta, int32_t* marked, int64_t* n_marked) {
    return guard([&] {
        const auto mk = dorfler_mark(Vec(eta, eta + nt), total_sq, theta);
        for (size_t i = 0; i < mk.size(); ++i) marked[i] = mk[i];
        *n_marked = int64_t(mk.size());
    });
}
int orc_norms(orc_problem* p, int level, const double* f, double* out) {
    return guard([&] {
        const Space& V = p->p.space(level);
        const Vec x(f, f + V.n());
        out[0] = l2_norm(V, x);
        out[1] = h1_seminorm(V, x);
        out[2] = h1_norm(V, x);
    });
}
/// fem::l1_norm (proj/src/assembly.cpp:289-291)
int orc_l1_norm(orc_problem* p, int level, const double* f, double* out) {
    return guard([&] {
        const Space& V = p->p.space(level);
        *out = l1_norm(V, Vec(f, f + V.n()));
    });
}
int orc_prolong_vec(orc_problem* p, int from, int to, const double* in, int N, double* out) {
    return guard([&] {
        const auto cols = unpack(in, p->p.space(from).n(), N);
        std::vector<Vec> o;
        for (const auto& c : cols) o.push_back(p->p.hier.prolong(c, from, to));
        pack(o, out);
    });
}

// ---------------- coarse SCF and correction step ----------------
int orc_coarse_scf(orc_problem* p, double tol, int max_it, double mixing, double tol_eig, double* lambdas, double* orb,
                   double* hartree, int* iters) {
    return guard([&] {
        p->last_scf_hist.clear();
        const auto r = self_consistent_solve(p->p.sys, p->p.hier.spaces.at(0), tol, max_it, mixing, tol_eig,
                                             &p->last_scf_hist);
        std::memcpy(lambdas, r.lambdas.data(), sizeof(double) * r.lambdas.size());
        pack(r.orbitals, orb);
        std::memcpy(hartree, r.hartree.data(), sizeof(double) * r.hartree.size());
        if (iters) *iters = r.iterations;
        p->last_scf_rho = r.rho;
    });
}
/// H1 density changes of the last orc_coarse_scf, also after it failed (n_out: capacity in, count out)
int orc_last_scf_history(orc_problem* p, double* hist, int* n_out) {
    return guard([&] {
        const int n = std::min<int>(*n_out, int(p->last_scf_hist.size()));
        std::memcpy(hist, p->last_scf_hist.data(), sizeof(double) * n);
        *n_out = int(p->last_scf_hist.size());
    });
}
/// mixed density of the last orc_coarse_scf (ScfResult::rho, proj/src/scf.cpp:73)
int orc_last_scf_rho(orc_problem* p, double* rho) {
    return guard([&] { std::memcpy(rho, p->last_scf_rho.data(), sizeof(double) * p->last_scf_rho.size()); });
}

/// cfg_d: tol_linear, tol_inner, score_floor; cfg_i: max_inner, nev_pad, precond, fixed_sweeps
/// log_i: inner_iterations, hartree_iterations, attempts[N], cg_iters[N]; log_d: delta, t_bvp, t_hartree, t_blocks, t_inner, t_total
int orc_correction_step(orc_problem* p, int level, const double* cfg_d, const int* cfg_i, double* lambdas, double* orb,
                        double* w, int* log_i, double* log_d) {
    return guard([&] {
        auto& o = p->p.level(level);
        const int N = p->p.sys.n_pairs;
        const int n = o.V->n();
        StepConfig c;
        c.tol_linear = cfg_d[0];
        c.tol_inner = cfg_d[1];
        c.score_floor = cfg_d[2];
        c.max_inner = cfg_i[0];
        c.nev_pad = cfg_i[1];
        c.precond = cfg_i[2];
        c.fixed_sweeps = cfg_i[3];
        Vec lam(lambdas, lambdas + N);
        auto orbs = unpack(orb, n, N);
        Vec wv(w, w + n);
        StepLog lg;
        correction_step(p->p.sys, p->p.hier, o, c, lam, orbs, wv, &lg);
        std::memcpy(lambdas, lam.data(), sizeof(double) * N);
        pack(orbs, orb);
        std::memcpy(w, wv.data(), sizeof(double) * n);
        if (log_i) {
            log_i[0] = lg.inner_iterations;
            log_i[1] = lg.hartree_iterations;
            for (int i = 0; i < N; ++i) {
                log_i[2 + i] = lg.shifts.attempt[i];
                log_i[2 + N + i] = lg.shifts.iterations[i];
            }
        }
        if (log_d) {
            log_d[0] = lg.delta;
            log_d[1] = lg.t_bvp;
            log_d[2] = lg.t_hartree;
            log_d[3] = lg.t_blocks;
            log_d[4] = lg.t_inner;
            log_d[5] = lg.t_total;
        }
    });
}

int orc_solve_level_mlc(orc_problem* p, int level, const double* cfg_d, const int* cfg_i, double tol_outer,
                        int max_scf, double* lambdas, double* orb, double* w, double* rho, int* sweeps,
                        double* deltas, int deltas_cap) {
    return guard([&] {
        auto& o = p->p.level(level);
        const int N = p->p.sys.n_pairs;
        const int n = o.V->n();
        StepConfig c;
        c.tol_linear = cfg_d[0];
        c.tol_inner = cfg_d[1];
        c.score_floor = cfg_d[2];
        c.max_inner = cfg_i[0];
        c.nev_pad = cfg_i[1];
        c.precond = cfg_i[2];
        Vec lam(lambdas, lambdas + N);
        auto orbs = unpack(orb, n, N);
        Vec wv(w, w + n), r;
        std::vector<double> ds;
        solve_level_mlc(p->p.sys, p->p.hier, o, c, tol_outer, max_scf, lam, orbs, wv, r, sweeps, &ds);
        std::memcpy(lambdas, lam.data(), sizeof(double) * N);
        pack(orbs, orb);
        std::memcpy(w, wv.data(), sizeof(double) * n);
        std::memcpy(rho, r.data(), sizeof(double) * n);
        for (int k = 0; k < int(ds.size()) && k < deltas_cap; ++k) deltas[k] = ds[k];
    });
}

/// bvp_orbital for every orbital: phi_tilde (row-major n x N), attempts[N], iters[N]
int orc_outer_solve(orc_problem* p, int level, const double* w_hat, const double* vxc, const double* lambdas,
                    const double* orb, double tol, int precond, double* phi_tilde, int* attempts, int* iters,
                    double* sigmas) {
    return guard([&] {
        auto& o = p->p.level(level);
        const int N = p->p.sys.n_pairs;
        const int n = o.V->n();
        Outer op(o.V, o.a_op, &o.M, Vec(w_hat, w_hat + n), Vec(vxc, vxc + n), tol, precond);
        const auto orbs = unpack(orb, n, N);
        std::vector<Vec> out(N);
        for (int i = 0; i < N; ++i) out[i] = op.solve_orbital(lambdas[i], orbs[i], attempts + i, iters + i);
        pack(out, phi_tilde);
        if (sigmas) {
            const double base = std::abs(op.solver->min_diag);
            for (int k = 0; k < 4; ++k) sigmas[k] = k == 0 ? base : std::pow(4.0, k) * (base + 1.0);
        }
    });
}

int orc_prepare_blocks(orc_problem* p, int level, const double* phi_tilde, const double* w_tilde, const double* vxc,
                       const double* bc, int hartree_on, orc_blocks** out) {
    return guard([&] {
        auto& o = p->p.level(level);
        const int N = p->p.sys.n_pairs;
        const int n = o.V->n();
        auto* b = new orc_blocks;
        b->B = prepare_blocks(p->p.hier.spaces[0], o.V, o.P_full, o.S, o.M, o.a_op, unpack(phi_tilde, n, N),
                              Vec(w_tilde, w_tilde + n), Vec(vxc, vxc + n), p->p.sys.occ, hartree_on != 0,
                              bc ? Vec(bc, bc + n) : Vec());
        *out = b;
    });
}
void orc_blocks_free(orc_blocks* b) { delete b; }

/// what: 0 A_H1 1 A_H3 2 A_H4 3 M_H 4 C_H (nh*nh col-major) 5 d_Hh 6 lift_load (nh)
///       7 scalars [zeta, lift_load0, hartree_schur] 8 hartree_u (nh)
///       10 A_h4 (N*nh*nh) 11 b_H1 12 b_H3 13 b_H4 14 rhs 15 c_Hh 16 d_phi (N*nh)
///       17 beta1 18 beta3 19 beta4 20 gamma 21 zeta_phi (N)
int orc_blocks_get(orc_blocks* bh, int what, double* dst) {
    return guard([&] {
        const Blocks& B = bh->B;
        const int nh = B.M_H.n;
        auto putv = [&](const Vec& v) { std::memcpy(dst, v.data(), v.size() * sizeof(double)); };
        auto putvv = [&](const std::vector<Vec>& v) {
            for (size_t i = 0; i < v.size(); ++i) std::memcpy(dst + i * nh, v[i].data(), sizeof(double) * nh);
        };
        switch (what) {
            case 0: putv(B.A_H1.a); break;
            case 1: putv(B.A_H3.a); break;
            case 2: putv(B.A_H4.a); break;
            case 3: putv(B.M_H.a); break;
            case 4: putv(B.C_H.a); break;
            case 5: putv(B.d_Hh); break;
            case 6: putv(B.lift_load); break;
            case 7:
                dst[0] = B.zeta;
                dst[1] = B.lift_load0;
                dst[2] = B.hartree_schur;
                break;
            case 8: putv(B.hartree_u); break;
            case 10:
                for (int i = 0; i < B.n; ++i) std::memcpy(dst + size_t(i) * nh * nh, B.A_h4[i].a.data(), sizeof(double) * nh * nh);
                break;
            case 11: putvv(B.b_H1); break;
            case 12: putvv(B.b_H3); break;
            case 13: putvv(B.b_H4); break;
            case 14: putvv(B.rhs); break;
            case 15: putvv(B.c_Hh); break;
            case 16: putvv(B.d_phi); break;
            case 17: putv(B.beta1); break;
            case 18: putv(B.beta3); break;
            case 19: putv(B.beta4); break;
            case 20: putv(B.gamma); break;
            case 21: putv(B.zeta_phi); break;
            default: fail(E_ARG, "unknown block");
        }
    });
}

/// inner_scf from the pure augmentation state; outputs lambda[N], phi_H[N*nh], theta2[N], w_H[nh], theta1, iterations
int orc_inner_scf(orc_blocks* bh, const double* lambdas, double tol, int max_it, double floor, int pad, double* lam,
                  double* phi_H, double* theta2, double* w_H, double* theta1, int* iterations, double* history,
                  int hist_cap) {
    return guard([&] {
        const Blocks& B = bh->B;
        const int nh = B.M_H.n;
        // max_it < 0: run exactly -max_it sweeps and return the state (diagnostics)
        const bool fixed = max_it < 0;
        const auto r = inner_scf(B, pure_state(B, Vec(lambdas, lambdas + B.n)), tol, fixed ? -max_it : max_it, floor,
                                 pad, fixed);
        bh->last = r.state;
        std::memcpy(lam, r.state.lambda.data(), sizeof(double) * B.n);
        for (int i = 0; i < B.n; ++i) std::memcpy(phi_H + size_t(i) * nh, r.state.phi_H[i].data(), sizeof(double) * nh);
        std::memcpy(theta2, r.state.theta2.data(), sizeof(double) * B.n);
        std::memcpy(w_H, r.state.w_H.data(), sizeof(double) * nh);
        *theta1 = r.state.theta1;
        *iterations = r.iterations;
        for (int k = 0; k < std::min<int>(hist_cap, int(r.history.size())); ++k) history[k] = r.history[k];
    });
}
int orc_expand_last(orc_blocks* bh, double* orb, double* w) {
    return guard([&] {
        std::vector<Vec> o;
        Vec wv;
        expand(bh->last, bh->B, o, wv);
        pack(o, orb);
        std::memcpy(w, wv.data(), sizeof(double) * wv.size());
    });
}
int orc_blocks_f_g(orc_blocks* bh, const double* phi_H, const double* theta2, const double* w_H, double theta1,
                   double* f, double* g, double* A_H2) {
    return guard([&] {
        const Blocks& B = bh->B;
        const int nh = B.M_H.n;
        AState s;
        s.lambda.assign(B.n, 0.0);
        s.theta2.assign(theta2, theta2 + B.n);
        for (int i = 0; i < B.n; ++i) s.phi_H.push_back(Vec(phi_H + size_t(i) * nh, phi_H + size_t(i + 1) * nh));
        s.w_H.assign(w_H, w_H + nh);
        s.theta1 = theta1;
        const Vec fv = assemble_f_H(B, s);
        std::memcpy(f, fv.data(), sizeof(double) * nh);
        *g = assemble_g(B, s);
        if (A_H2) {
            const Dense D = assemble_A_H2(B, s.w_H);
            std::memcpy(A_H2, D.a.data(), sizeof(double) * nh * nh);
        }
    });
}

// ---------------- dense eigen pieces ----------------
int orc_gen_eig(int n, const double* A, const double* B, double* vals, double* vecs) {
    return guard([&] {
        Dense a(n, n), b(n, n);
        std::memcpy(a.a.data(), A, sizeof(double) * n * n);
        std::memcpy(b.a.data(), B, sizeof(double) * n * n);
        Vec v;
        Dense V;
        if (!gen_eig(a, b, v, V)) fail(E_AMBIG, "B not positive definite");
        std::memcpy(vals, v.data(), sizeof(double) * n);
        std::memcpy(vecs, V.a.data(), sizeof(double) * n * n);
    });
}
int orc_solve_bordered(int n, const double* A, const double* M, const double* b, double beta, const double* c,
                       double gamma, int nev, double floor, double* lambda, double* phi, double* theta, double* score) {
    return guard([&] {
        Dense a(n, n), m(n, n);
        std::memcpy(a.a.data(), A, sizeof(double) * n * n);
        std::memcpy(m.a.data(), M, sizeof(double) * n * n);
        Bordered s;
        s.A = &a;
        s.M = &m;
        s.b.assign(b, b + n);
        s.c.assign(c, c + n);
        s.beta = beta;
        s.gamma = gamma;
        const auto r = solve_bordered(s, nev, floor);
        *lambda = r.lambda;
        std::memcpy(phi, r.phi.data(), sizeof(double) * n);
        *theta = r.theta;
        *score = r.score;
    });
}

}  // extern "C"
