// ksafem-compatible C++ host API over the C-ABI (include/ksafem_b200/*.hpp). Every compute call goes to the
// device through include/ksb.h; this layer only moves FEFunction coefficients between host vectors and
// HBM, keeps the level's operator-slot table, and maps status codes to ksafem::Error.
//
// Reference interfaces mirrored (file:line under /root/reference/proj):
//   mesh::build_box_mesh / uniform_refine / adapt_refine   include/ksafem/mesh.hpp:93-105
//   fem::FESpace / FEFunction / SpaceHierarchy             include/ksafem/fespace.hpp:12-81, src/fespace.cpp:58-90
//   fem::assemble_stiffness / assemble_mass / norms        include/ksafem/assembly.hpp:16-38
//   fem::EllipticSolver / solve_spd                        include/ksafem/solver.hpp:25-51, src/solver.cpp:113-150
//   hartree::compute_moments / boundary_values / squared_density_load / solve_hartree_exact
//                                                          include/ksafem/hartree.hpp:18-48
//   model::density / xc_potential_field / total_energy     include/ksafem/ks_model.hpp:41-64
//   corr::OuterOperator / bvp_orbital / bvp_hartree / prepare_blocks / pure_augmentation_state / inner_scf /
//   expand                                                 include/ksafem/correction.hpp:21-172
//   driver make_level_ops / solve_level_corrected          src/driver.cpp:35-47, 94-163
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>

#include "ksafem_b200/driver.hpp"

namespace ksafem {

// ------------------------------------------------------------------ b200 plumbing
namespace b200 {

void check(int st) {
    if (st == KSB_OK) return;
    const char* code = ksb_code_name(st);
    throw Error(code ? code : "internal", ksb_last_error());
}

Device::Device(int ordinal) { check(ksb_ctx_create(ordinal, &ctx_)); }
Device::~Device() {
    if (ctx_) ksb_ctx_destroy(ctx_);
}
void Device::sync() const { check(ksb_ctx_sync(ctx_)); }
Device& Device::default_device() {
    static Device d(0);
    return d;
}

DeviceBuffer::DeviceBuffer(Device& d, int64_t n) : dev_(&d), n_(n) {
    void* p = nullptr;
    check(ksb_malloc(d.ctx(), &p, std::max<int64_t>(1, n) * int64_t(sizeof(double))));
    p_ = static_cast<double*>(p);
}
DeviceBuffer::DeviceBuffer(Device& d, const VecX& host) : DeviceBuffer(d, int64_t(host.size())) {
    upload(host.data(), int64_t(host.size()));
}
DeviceBuffer::~DeviceBuffer() {
    if (p_) ksb_free(dev_->ctx(), p_);
}
DeviceBuffer::DeviceBuffer(DeviceBuffer&& o) noexcept : dev_(o.dev_), p_(o.p_), n_(o.n_) {
    o.p_ = nullptr;
    o.n_ = 0;
}
DeviceBuffer& DeviceBuffer::operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
        if (p_) ksb_free(dev_->ctx(), p_);
        dev_ = o.dev_;
        p_ = o.p_;
        n_ = o.n_;
        o.p_ = nullptr;
        o.n_ = 0;
    }
    return *this;
}
void DeviceBuffer::upload(const double* h, int64_t n) {
    if (n > n_) fail("invalid-argument", "upload larger than the buffer");
    if (n == 0) return;
    check(ksb_memcpy_h2d(dev_->ctx(), p_, h, n * int64_t(sizeof(double))));
    dev_->sync();
}
void DeviceBuffer::download(double* h, int64_t n) const {
    if (n > n_) fail("invalid-argument", "download larger than the buffer");
    if (n == 0) return;
    check(ksb_memcpy_d2h(dev_->ctx(), h, p_, n * int64_t(sizeof(double))));
    dev_->sync();
}
VecX DeviceBuffer::to_host() const {
    VecX h(static_cast<size_t>(n_));
    download(h.data(), n_);
    return h;
}

} // namespace b200

// ------------------------------------------------------------------ mesh
namespace mesh {

bool Box::valid() const {
    for (int d = 0; d < 3; ++d)
        if (!(hi[d] > lo[d]) || !std::isfinite(lo[d]) || !std::isfinite(hi[d])) return false;
    return true;
}

TetMesh::TetMesh(ksb_mesh* h) : h_(h) {
    b200::check(ksb_mesh_sizes(h_, sizes_));
    level = int(sizes_[4]);
}
TetMesh::~TetMesh() {
    if (h_) ksb_mesh_free(h_);
}

namespace {
template <typename T>
std::vector<T> get_arr(ksb_mesh* h, int what, size_t count) {
    std::vector<T> out(count);
    if (count) b200::check(ksb_mesh_get(h, what, out.data()));
    return out;
}
} // namespace

std::vector<Vec3> TetMesh::vertices() const {
    const auto xyz = get_arr<double>(h_, 0, size_t(n_vertices()) * 3);
    std::vector<Vec3> v(static_cast<size_t>(n_vertices()));
    for (size_t i = 0; i < v.size(); ++i) v[i] = Vec3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    return v;
}
std::vector<std::array<int, 4>> TetMesh::tets() const {
    const auto t = get_arr<int32_t>(h_, 1, size_t(n_tets()) * 4);
    std::vector<std::array<int, 4>> out(static_cast<size_t>(n_tets()));
    for (size_t i = 0; i < out.size(); ++i) out[i] = {t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]};
    return out;
}
std::vector<std::array<int, 4>> TetMesh::bisect_tuple() const {
    const auto t = get_arr<int32_t>(h_, 2, size_t(n_tets()) * 4);
    std::vector<std::array<int, 4>> out(static_cast<size_t>(n_tets()));
    for (size_t i = 0; i < out.size(); ++i) out[i] = {t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]};
    return out;
}
std::vector<int8_t> TetMesh::tag() const { return get_arr<int8_t>(h_, 3, size_t(n_tets())); }
std::vector<int> TetMesh::parent_map() const {
    const auto p = get_arr<int32_t>(h_, 4, size_t(n_tets()));
    return std::vector<int>(p.begin(), p.end());
}
std::vector<std::array<int, 2>> TetMesh::vertex_parents() const {
    const auto p = get_arr<int32_t>(h_, 5, size_t(n_vertices()) * 2);
    std::vector<std::array<int, 2>> out(static_cast<size_t>(n_vertices()));
    for (size_t i = 0; i < out.size(); ++i) out[i] = {p[2 * i], p[2 * i + 1]};
    return out;
}
std::vector<char> TetMesh::vertex_on_boundary() const {
    const auto b = get_arr<uint8_t>(h_, 6, size_t(n_vertices()));
    return std::vector<char>(b.begin(), b.end());
}

MeshPtr build_box_mesh(const Box& box, int n_per_axis) {
    if (!box.valid()) fail("invalid-domain", "domain box is degenerate");
    ksb_mesh* h = nullptr;
    const double lo[3] = {box.lo[0], box.lo[1], box.lo[2]}, hi[3] = {box.hi[0], box.hi[1], box.hi[2]};
    b200::check(ksb_mesh_box(lo, hi, n_per_axis, &h));
    auto m = std::make_shared<TetMesh>(h);
    m->box = box;
    return m;
}
MeshPtr uniform_refine(const TetMesh& src) {
    ksb_mesh* h = nullptr;
    b200::check(ksb_mesh_uniform_refine(src.handle(), &h));
    auto m = std::make_shared<TetMesh>(h);
    m->box = src.box;
    return m;
}
MeshPtr adapt_refine(const TetMesh& src, const std::vector<int>& marked) {
    std::vector<int32_t> mk(marked.begin(), marked.end());
    ksb_mesh* h = nullptr;
    b200::check(ksb_mesh_adapt_refine(src.handle(), mk.data(), int64_t(mk.size()), &h));
    auto m = std::make_shared<TetMesh>(h);
    m->box = src.box;
    return m;
}

} // namespace mesh

// ------------------------------------------------------------------ spaces and operator slots
namespace fem {
namespace detail {

constexpr int kFirstUserSlot = KSB_MAT_USER0;
constexpr int kSlots = 32;

struct LevelState {
    b200::Device* dev = nullptr;
    std::shared_ptr<ksb_hier> hier;
    int level = 0;
    mesh::MeshPtr mesh;
    ksb_level* lev = nullptr;
    int n = 0, ni = 0, nb = 0, nH = 0;
    std::vector<int> interior, boundary, iidx;
    std::mutex mu;
    bool used[kSlots] = {};
    // correction-path bookkeeping
    std::string sys_key;        // last system pushed to the level
    uint64_t outer_gen = 0;     // generation of the device H (OuterOperator)
    uint64_t blocks_gen = 0;    // generation of the device ledger (prepare_blocks)
    uint64_t inner_of = 0;      // ledger generation the last inner_scf ran on
    VecX inner_lambda;          // last inner result (expand checks its state against it)
    double inner_theta1 = 0;

    ~LevelState() {
        if (lev) ksb_level_destroy(lev);
    }
    int alloc_slot() {
        std::lock_guard<std::mutex> lk(mu);
        for (int s = kFirstUserSlot; s < kSlots; ++s)
            if (!used[s]) {
                used[s] = true;
                return s;
            }
        fail("internal", "operator table of the level is full (24 user operators)");
    }
    void free_slot(int s) {
        std::lock_guard<std::mutex> lk(mu);
        if (s >= kFirstUserSlot && s < kSlots) used[s] = false;
    }
};

std::shared_ptr<LevelState> make_level(b200::Device& dev, std::shared_ptr<ksb_hier> hier, int level,
                                       mesh::MeshPtr m) {
    auto st = std::make_shared<LevelState>();
    st->dev = &dev;
    st->hier = std::move(hier);
    st->level = level;
    st->mesh = std::move(m);
    b200::check(ksb_level_create(dev.ctx(), st->hier.get(), level, &st->lev));
    int64_t s[10];
    b200::check(ksb_level_sizes(st->lev, s));
    st->n = int(s[0]);
    st->ni = int(s[1]);
    st->nb = int(s[2]);
    st->nH = int(s[6]);
    st->interior.resize(size_t(st->ni));
    std::vector<int32_t> itmp(static_cast<size_t>(st->ni));
    if (st->ni) b200::check(ksb_level_index(st->lev, 4, itmp.data()));
    st->interior.assign(itmp.begin(), itmp.end());
    st->iidx.assign(size_t(st->n), -1);
    for (int r = 0; r < st->ni; ++r) st->iidx[size_t(st->interior[r])] = r;
    for (int v = 0; v < st->n; ++v)
        if (st->iidx[size_t(v)] < 0) st->boundary.push_back(v);
    return st;
}

} // namespace detail

namespace {

using detail::LevelState;

const LevelState& S(const FESpace& V) { return *V.state(); }

void same_space(const FEFunction& f, const FESpace& V, const char* what) {
    if (!f.space || f.space->state() != V.state()) fail("mismatched-spaces", what);
    if (int(f.coeffs.size()) != V.n_dofs()) fail("invalid-argument", "coefficient vector has the wrong length");
}

/// interior block (ni x ld, row-major) of a set of zero-trace functions
b200::DeviceBuffer orbital_block(const FESpace& V, const std::vector<FEFunction>& fs, int& ld) {
    const auto& st = S(V);
    const int N = int(fs.size());
    ld = N == 1 ? 1 : N + (N & 1);
    VecX blk(size_t(st.ni) * size_t(ld), 0.0);
    for (int i = 0; i < N; ++i) {
        same_space(fs[size_t(i)], V, "orbitals live on different spaces");
        for (int r = 0; r < st.ni; ++r) blk[size_t(r) * ld + i] = fs[size_t(i)].coeffs[size_t(st.interior[size_t(r)])];
    }
    return b200::DeviceBuffer(*st.dev, blk);
}

std::vector<FEFunction> from_block(const SpacePtr& V, const VecX& blk, int N, int ld, Role role) {
    const auto& st = *V->state();
    std::vector<FEFunction> out;
    for (int i = 0; i < N; ++i) {
        FEFunction f(V, role);
        for (int r = 0; r < st.ni; ++r) f.coeffs[size_t(st.interior[size_t(r)])] = blk[size_t(r) * ld + i];
        out.push_back(std::move(f));
    }
    return out;
}

} // namespace

FESpace::FESpace(mesh::MeshPtr m, b200::Device& dev) {
    ksb_hier* h = nullptr;
    b200::check(ksb_hier_create(&h));
    std::shared_ptr<ksb_hier> hier(h, ksb_hier_free);
    b200::check(ksb_hier_push(h, m->handle()));
    st_ = detail::make_level(dev, hier, 0, std::move(m));
}

const mesh::TetMesh& FESpace::mesh() const { return *st_->mesh; }
mesh::MeshPtr FESpace::mesh_ptr() const { return st_->mesh; }
int FESpace::n_dofs() const { return st_->n; }
int FESpace::n_interior() const { return st_->ni; }
const std::vector<int>& FESpace::interior_dofs() const { return st_->interior; }
const std::vector<int>& FESpace::boundary_dofs() const { return st_->boundary; }
int FESpace::interior_index(int dof) const { return st_->iidx.at(size_t(dof)); }
ksb_level* FESpace::device_level() const { return st_->lev; }
b200::Device& FESpace::device() const { return *st_->dev; }

SpaceHierarchy::SpaceHierarchy(b200::Device& dev) : dev_(&dev) {
    ksb_hier* h = nullptr;
    b200::check(ksb_hier_create(&h));
    hier_ = std::shared_ptr<ksb_hier>(h, ksb_hier_free);
}
SpaceHierarchy::~SpaceHierarchy() = default;

void SpaceHierarchy::push(mesh::MeshPtr m) {
    b200::check(ksb_hier_push(hier_.get(), m->handle()));
    const int k = int(spaces_.size());
    meshes_.push_back(m);
    spaces_.push_back(std::make_shared<FESpace>(detail::make_level(*dev_, hier_, k, std::move(m))));
}

int SpaceHierarchy::level_of(const FESpace& s) const {
    for (int k = 0; k < n_levels(); ++k)
        if (spaces_[size_t(k)].get() == &s || spaces_[size_t(k)]->state() == s.state()) return k;
    return -1;
}

Prolongation SpaceHierarchy::prolongation(int from, int to) const {
    if (from > to || to >= n_levels()) fail("hierarchy", "levels are not nested");
    if (from != 0) fail("invalid-argument", "the device hierarchy keeps composite transfers to level 0 only");
    const int n = spaces_[size_t(to)]->n_dofs();
    std::vector<int32_t> col(size_t(n) * 4);
    VecX val(size_t(n) * 4);
    b200::check(ksb_hier_prolongation(hier_.get(), to, col.data(), val.data()));
    Prolongation P;
    P.from = from;
    P.to = to;
    P.rows = n;
    P.cols = spaces_[0]->n_dofs();
    P.ptr.assign(1, 0);
    for (int v = 0; v < n; ++v) {
        for (int k = 0; k < 4; ++k)
            if (col[size_t(v) * 4 + k] >= 0) {
                P.col.push_back(col[size_t(v) * 4 + k]);
                P.val.push_back(val[size_t(v) * 4 + k]);
            }
        P.ptr.push_back(int(P.col.size()));
    }
    return P;
}

FEFunction SpaceHierarchy::prolong(const FEFunction& coarse, int to) const {
    const int from = coarse.space ? level_of(*coarse.space) : -1;
    if (from < 0 || from > to || to >= n_levels()) fail("hierarchy", "levels are not nested");
    VecX c = coarse.coeffs;
    for (int k = from + 1; k <= to; ++k) {
        const auto& m = *meshes_[size_t(k)];
        const auto vp = m.vertex_parents();
        const int npv = m.n_parent_vertices(), n = m.n_vertices();
        VecX f(size_t(n), 0.0);
        std::vector<char> known(size_t(n), 0);
        for (int v = 0; v < npv; ++v) {
            f[size_t(v)] = c[size_t(v)];
            known[size_t(v)] = 1;
        }
        // new vertices average their parent edge; parents may be new themselves (bisection chains)
        bool progress = true;
        int left = n - npv;
        while (left > 0 && progress) {
            progress = false;
            for (int v = npv; v < n; ++v) {
                if (known[size_t(v)]) continue;
                const int a = vp[size_t(v)][0], b = vp[size_t(v)][1];
                if (known[size_t(a)] && known[size_t(b)]) {
                    f[size_t(v)] = 0.5 * f[size_t(a)] + 0.5 * f[size_t(b)];
                    known[size_t(v)] = 1;
                    --left;
                    progress = true;
                }
            }
        }
        if (left > 0) fail("internal", "prolongation parents form a cycle");
        c.swap(f);
    }
    return FEFunction(spaces_[size_t(to)], std::move(c), coarse.role);
}

// ------------------------------------------------------------------ operators
SpMat::SpMat(std::shared_ptr<LevelState> st, int id, bool owned) : st_(std::move(st)) {
    if (owned) {
        std::weak_ptr<LevelState> w = st_;
        id_ = std::shared_ptr<int>(new int(id), [w](int* p) {
            if (auto s = w.lock()) s->free_slot(*p);
            delete p;
        });
    } else {
        id_ = std::make_shared<int>(id);
    }
}
int SpMat::id() const {
    if (!st_) fail("invalid-argument", "empty operator");
    return *id_;
}
int SpMat::rows() const { return st_ ? st_->n : 0; }
int64_t SpMat::interior_nonzeros() const {
    int64_t s[10];
    b200::check(ksb_level_sizes(st_->lev, s));
    return s[4];
}
VecX SpMat::interior_values() const {
    int64_t s[10];
    b200::check(ksb_level_sizes(st_->lev, s));
    VecX v(static_cast<size_t>(s[4]));
    b200::check(ksb_mat_values(st_->lev, id(), 0, v.data()));
    return v;
}
VecX SpMat::boundary_values() const {
    int64_t s[10];
    b200::check(ksb_level_sizes(st_->lev, s));
    VecX v(static_cast<size_t>(s[5]));
    if (!v.empty()) b200::check(ksb_mat_values(st_->lev, id(), 1, v.data()));
    return v;
}

void SpMat::pattern(int part, std::vector<int>& ptr, std::vector<int>& col) const {
    if (part != 0 && part != 1) fail("invalid-argument", "part must be 0 (ii) or 1 (ib)");
    int64_t s[10];
    b200::check(ksb_level_sizes(st_->lev, s));
    std::vector<int32_t> p(size_t(s[1]) + 1), c(size_t(part == 0 ? s[4] : s[5]));
    b200::check(ksb_level_index(st_->lev, part == 0 ? 0 : 2, p.data()));
    if (!c.empty()) b200::check(ksb_level_index(st_->lev, part == 0 ? 1 : 3, c.data()));
    ptr.assign(p.begin(), p.end());
    col.assign(c.begin(), c.end());
}

namespace {
SpMat combine(double a, const SpMat& x, double b, const SpMat& y) {
    if (x.state() != y.state()) fail("mismatched-spaces", "operators live on different spaces");
    const int s = x.state()->alloc_slot();
    SpMat out(x.state(), s, true);
    b200::check(ksb_mat_axpby(x.state()->lev, s, a, x.id(), b, y.id()));
    return out;
}
} // namespace

SpMat SpMat::operator+(const SpMat& o) const { return combine(1.0, *this, 1.0, o); }
SpMat SpMat::operator-(const SpMat& o) const { return combine(1.0, *this, -1.0, o); }
SpMat operator*(double a, const SpMat& x) { return combine(a, x, 0.0, x); }

SpMat assemble_stiffness(const FESpace& V, WorkerPool*) {
    const int s = V.state()->alloc_slot();
    SpMat out(V.state(), s, true);
    b200::check(ksb_mat_assemble(V.device_level(), s, 1.0, 0.0, KSB_POT_COULOMB, 0, nullptr, 0.0, nullptr, 0.0));
    return out;
}
SpMat assemble_mass(const FESpace& V, WorkerPool*) {
    const int s = V.state()->alloc_slot();
    SpMat out(V.state(), s, true);
    b200::check(ksb_mat_assemble(V.device_level(), s, 0.0, 1.0, KSB_POT_COULOMB, 0, nullptr, 0.0, nullptr, 0.0));
    return out;
}
SpMat assemble_mass(const FESpace& V, const FEFunction& w, WorkerPool*) {
    if (!w.space || &w.space->mesh() != &V.mesh()) fail("mismatched-spaces", "weight lives on a different mesh");
    b200::DeviceBuffer dw(V.device(), w.coeffs);
    const int s = V.state()->alloc_slot();
    SpMat out(V.state(), s, true);
    b200::check(ksb_mat_assemble(V.device_level(), s, 0.0, 0.0, KSB_POT_COULOMB, 0, nullptr, 0.0, dw.data(), 1.0));
    return out;
}

namespace {
std::array<double, 3> norms(const FEFunction& f) {
    if (!f.space) fail("invalid-argument", "function without a space");
    b200::DeviceBuffer d(f.space->device(), f.coeffs);
    std::array<double, 3> o{};
    b200::check(ksb_norms(f.space->device_level(), d.data(), o.data()));
    return o;
}
} // namespace

double l2_norm(const FEFunction& f) { return std::sqrt(std::max(0.0, norms(f)[0])); }
double h1_seminorm(const FEFunction& f) { return std::sqrt(std::max(0.0, norms(f)[1])); }
double h1_norm(const FEFunction& f) {
    const auto o = norms(f);
    return std::sqrt(std::max(0.0, o[0]) + std::max(0.0, o[1]));
}

// ------------------------------------------------------------------ solver
EllipticSolver::EllipticSolver(const SpMat& A, SpacePtr space) : A_(A), space_(std::move(space)) {
    if (!space_ || A_.state() != space_->state()) fail("mismatched-spaces", "operator and space differ");
    b200::check(ksb_mat_min_diag(space_->device_level(), A_.id(), &min_diag_));
}

VecX EllipticSolver::solve(const VecX& b, const VecX& bc, const SolverOptions& opt, SolveStats* stats) const {
    const int n = space_->n_dofs();
    if (int(b.size()) != n) fail("invalid-argument", "load vector has the wrong length");
    if (!bc.empty() && int(bc.size()) != n) fail("invalid-argument", "boundary data has the wrong length");
    auto& dev = space_->device();
    b200::DeviceBuffer db(dev, b), dx(dev, int64_t(n));
    b200::DeviceBuffer dbc;
    if (!bc.empty()) dbc = b200::DeviceBuffer(dev, bc);
    ksb_cg_opts o;
    b200::check(ksb_cg_defaults(&o));
    o.tol = opt.tol;
    o.max_iterations = opt.max_iterations;
    ksb_cg_stats st{};
    b200::check(ksb_solve(space_->device_level(), A_.id(), db.data(), bc.empty() ? nullptr : dbc.data(), &o, dx.data(),
                          &st));
    if (stats) {
        stats->iterations = st.iterations;
        stats->relative_residual = st.relative_residual;
        stats->converged = st.converged != 0;
        stats->breakdown = st.breakdown != 0;
    }
    return dx.to_host();
}

VecX EllipticSolver::solve_zero_bc(const VecX& b, const SolverOptions& opt, SolveStats* stats) const {
    return solve(b, VecX(), opt, stats);
}

VecX solve_spd(const SpMat& A, const VecX& b, SpacePtr space, const VecX& bc, double tol, SolveStats* stats) {
    EllipticSolver solver(A, std::move(space));
    SolverOptions opt;
    opt.tol = tol;
    SolveStats st;
    VecX x = solver.solve(b, bc, opt, &st);
    if (stats) *stats = st;
    if (!st.converged)
        fail("nonconvergence", "linear solve stalled at relative residual " + std::to_string(st.relative_residual) +
                                   " after " + std::to_string(st.iterations) + " iterations");
    return x;
}

} // namespace fem

// ------------------------------------------------------------------ model
namespace model {

void MolecularSystem::validate() const {
    if (!domain.valid()) fail("invalid-domain", "domain box is degenerate");
    if (n_pairs < 1) fail("invalid-argument", "n_pairs must be >= 1");
    if (occupancy <= 0) fail("invalid-argument", "occupancy must be positive");
    for (const auto& a : atoms) {
        if (a.charge <= 0) fail("invalid-argument", "nuclear charge must be positive");
        bool inside = true;
        for (int d = 0; d < 3; ++d) inside = inside && a.position[d] > domain.lo[d] && a.position[d] < domain.hi[d];
        if (!inside) fail("invalid-argument", "nucleus outside the domain");
    }
}

namespace {
int xc_code(XcKind k) { return k == XcKind::none ? KSB_XC_NONE : k == XcKind::x_alpha ? KSB_XC_XALPHA : KSB_XC_LDA; }

/// push the system to the level (only when it changed: a new system rebuilds the level operators)
void set_system(const fem::FESpace& V, const MolecularSystem& sys, bool hartree_on, bool xc_on) {
    auto& st = *V.state();
    std::string key;
    auto add = [&](double x) { key.append(reinterpret_cast<const char*>(&x), sizeof x); };
    for (const auto& a : sys.atoms) {
        add(a.charge);
        for (int d = 0; d < 3; ++d) add(a.position[d]);
    }
    add(sys.n_pairs);
    add(sys.occupancy);
    add(xc_code(sys.xc.kind));
    add(sys.xc.alpha);
    add(sys.xc.exchange_exponent);
    add(hartree_on);
    add(xc_on);
    if (key == st.sys_key) return;
    std::vector<double> atoms;
    for (const auto& a : sys.atoms) atoms.insert(atoms.end(), {a.charge, a.position[0], a.position[1], a.position[2]});
    b200::check(ksb_system_set(st.lev, atoms.data(), int(sys.atoms.size()), sys.n_pairs, sys.occupancy,
                               xc_code(sys.xc.kind), sys.xc.alpha, sys.xc.exchange_exponent, hartree_on ? 1 : 0,
                               xc_on ? 1 : 0));
    st.sys_key = key;
}
} // namespace

fem::FEFunction density(const std::vector<fem::FEFunction>& orbitals, double occupancy) {
    if (orbitals.empty()) fail("invalid-argument", "empty orbital set");
    const auto V = orbitals.front().space;
    for (const auto& phi : orbitals)
        if (phi.space != V) fail("mismatched-spaces", "orbitals live on different spaces");
    const auto& st = *V->state();
    for (const auto& phi : orbitals)
        for (int b : st.boundary)
            if (phi.coeffs[size_t(b)] != 0.0)
                fail("invalid-argument", "orbitals must vanish on the boundary (zero-trace wavefunctions)");
    int ld = 0;
    auto blk = fem::orbital_block(*V, orbitals, ld);
    b200::DeviceBuffer rho(V->device(), int64_t(V->n_dofs()));
    b200::check(ksb_density(V->device_level(), blk.data(), int(orbitals.size()), ld, occupancy, rho.data()));
    return fem::FEFunction(V, rho.to_host(), fem::Role::density);
}

fem::FEFunction xc_potential_field(const XcFunctional& xc, const fem::FEFunction& rho) {
    if (!rho.space) fail("invalid-argument", "density without a space");
    b200::DeviceBuffer dr(rho.space->device(), rho.coeffs), dv(rho.space->device(), int64_t(rho.coeffs.size()));
    b200::check(ksb_xc_field(rho.space->device_level(), xc_code(xc.kind), xc.alpha, xc.exchange_exponent, dr.data(),
                             dv.data()));
    return fem::FEFunction(rho.space, dv.to_host(), fem::Role::generic);
}

EnergyBreakdown total_energy(const MolecularSystem& sys, const std::vector<fem::FEFunction>& orbitals,
                             const fem::FEFunction& hartree_fn) {
    EnergyBreakdown e;
    if (orbitals.empty()) return e;
    const auto V = orbitals.front().space;
    if (hartree_fn.space != V) fail("mismatched-spaces", "hartree potential on a different space");
    MolecularSystem s2 = sys;
    s2.n_pairs = int(orbitals.size());
    set_system(*V, s2, true, sys.xc.kind != XcKind::none);
    int ld = 0;
    auto blk = fem::orbital_block(*V, orbitals, ld);
    b200::DeviceBuffer dw(V->device(), hartree_fn.coeffs);
    double o[5];
    b200::check(ksb_energy(V->device_level(), blk.data(), int(orbitals.size()), ld, dw.data(), o));
    e.kinetic = o[0];
    e.external = o[1];
    e.hartree = o[2];
    e.xc = o[3];
    e.total = o[4];
    return e;
}

} // namespace model

// ------------------------------------------------------------------ hartree
namespace hartree {

MultipoleMoments compute_moments(const fem::FEFunction& rho) {
    if (!rho.space) fail("invalid-argument", "density without a space");
    b200::DeviceBuffer d(rho.space->device(), rho.coeffs);
    double o[16];
    b200::check(ksb_moments(rho.space->device_level(), d.data(), o));
    MultipoleMoments m;
    m.charge = o[0];
    m.center = Vec3(o[1], o[2], o[3]);
    m.dipole = Vec3(o[4], o[5], o[6]);
    for (int k = 0; k < 9; ++k) m.quadrupole[size_t(k)] = o[7 + k];
    return m;
}

VecX boundary_values(const MultipoleMoments& m, const fem::FESpace& space) {
    double mom[16] = {m.charge, m.center[0], m.center[1], m.center[2], m.dipole[0], m.dipole[1], m.dipole[2]};
    for (int k = 0; k < 9; ++k) mom[7 + k] = m.quadrupole[size_t(k)];
    const auto& st = *space.state();
    b200::DeviceBuffer db(space.device(), std::max<int64_t>(1, st.nb));
    b200::check(ksb_boundary_values(space.device_level(), mom, db.data()));
    const VecX bb = db.to_host();
    VecX out(size_t(st.n), 0.0);
    for (int k = 0; k < st.nb; ++k) out[size_t(st.boundary[size_t(k)])] = bb[size_t(k)];
    return out;
}

VecX squared_density_load(const fem::FESpace& space, const std::vector<fem::FEFunction>& orbitals,
                          double occupancy) {
    if (orbitals.empty()) return VecX(size_t(space.n_dofs()), 0.0);
    int ld = 0;
    auto blk = fem::orbital_block(space, orbitals, ld);
    b200::DeviceBuffer out(space.device(), int64_t(space.n_dofs()));
    b200::check(ksb_sqload_full(space.device_level(), blk.data(), int(orbitals.size()), ld, occupancy, out.data()));
    return out.to_host();
}

fem::FEFunction solve_hartree_exact(const fem::EllipticSolver& stiffness, const fem::FESpace& space,
                                    const std::vector<fem::FEFunction>& orbitals, double occupancy, const VecX& bc,
                                    double tol) {
    // (grad w, grad v) = 4 pi (occ sum phi_i^2, v): the exact squared load through the stiffness solver
    VecX b = squared_density_load(space, orbitals, occupancy);
    for (double& x : b) x *= 4.0 * M_PI;
    fem::SolverOptions opt;
    opt.tol = tol;
    fem::SolveStats st;
    VecX w = stiffness.solve(b, bc, opt, &st);
    if (!st.converged) fail("nonconvergence", "hartree solve stalled at residual " + std::to_string(st.relative_residual));
    return fem::FEFunction(orbitals.empty() ? nullptr : orbitals.front().space, std::move(w), fem::Role::hartree);
}

} // namespace hartree

// ------------------------------------------------------------------ correction
namespace corr {

namespace {
ksb_step_opts step_opts(double tol_linear, double tol_inner, int max_inner, double floor, int pad) {
    ksb_step_opts o;
    b200::check(ksb_step_defaults(&o));
    o.tol_linear = tol_linear;
    o.tol_inner = tol_inner;
    o.max_inner = max_inner;
    o.score_floor = floor;
    o.nev_pad = pad;
    return o;
}

void require_system(const fem::FESpace& V) {
    if (V.state()->sys_key.empty())
        fail("invalid-argument", "no molecular system on this space: build it with driver::make_level_ops");
}
} // namespace

OuterOperator::OuterOperator(fem::SpacePtr space, const SpMat& a_op, const SpMat* mass, const fem::FEFunction& w_hat,
                             const fem::FEFunction& v_xc, double tol_linear, WorkerPool*)
    : space_(std::move(space)), mass_(mass), tol_(tol_linear) {
    if (!space_ || a_op.state() != space_->state() || !mass || mass->state() != space_->state())
        fail("mismatched-spaces", "operators live on a different space");
    if (mass->id() != KSB_MAT_M) fail("invalid-argument", "mass must be the level's unit mass (make_level_ops)");
    require_system(*space_);
    fem::same_space(w_hat, *space_, "w_hat lives on a different space");
    fem::same_space(v_xc, *space_, "v_xc lives on a different space");
    auto& st = *space_->state();
    b200::DeviceBuffer dw(space_->device(), w_hat.coeffs), dv(space_->device(), v_xc.coeffs);
    b200::check(ksb_outer_build(st.lev, a_op.id(), dw.data(), dv.data(), &min_diag_));
    generation_ = ++st.outer_gen;
}

std::vector<fem::FEFunction> OuterOperator::solve_orbitals(const VecX& lambda_prev,
                                                           const std::vector<fem::FEFunction>& phi_prev) const {
    auto& st = *space_->state();
    if (generation_ != st.outer_gen) fail("invalid-argument", "a newer OuterOperator replaced this one on its space");
    const int N = int(phi_prev.size());
    if (N == 0) return {};
    if (int(lambda_prev.size()) != N) fail("invalid-argument", "one eigenvalue per orbital");
    int ld = 0;
    auto blk = fem::orbital_block(*space_, phi_prev, ld);
    b200::DeviceBuffer out(space_->device(), int64_t(st.ni) * ld);
    const auto o = step_opts(tol_, 1e-8, 400, 1e-8, 4);
    std::vector<int> att(static_cast<size_t>(N)), its(static_cast<size_t>(N));
    b200::check(ksb_outer_apply(st.lev, &o, lambda_prev.data(), blk.data(), N, ld, out.data(), att.data(), its.data()));
    return fem::from_block(space_, out.to_host(), N, ld, fem::Role::wavefunction);
}

fem::FEFunction OuterOperator::solve_orbital(double lambda_prev, const fem::FEFunction& phi_prev) const {
    return solve_orbitals(VecX{lambda_prev}, {phi_prev}).front();
}

fem::FEFunction bvp_orbital(const OuterOperator& op, double lambda_prev, const fem::FEFunction& phi_prev) {
    return op.solve_orbital(lambda_prev, phi_prev);
}

fem::FEFunction bvp_hartree(const fem::EllipticSolver& stiffness, const SpMat& mass,
                            const std::vector<fem::FEFunction>& phi_tilde, double occupancy, const VecX& bc,
                            double tol) {
    (void)mass;
    if (phi_tilde.empty()) fail("invalid-argument", "empty orbital set");
    return hartree::solve_hartree_exact(stiffness, *phi_tilde.front().space, phi_tilde, occupancy, bc, tol);
}

// ---- ledger
namespace {
const fem::detail::LevelState& ledger_level(const AugmentedBlocks& B) {
    const auto& st = *B.space_h->state();
    if (B.generation != st.blocks_gen) fail("invalid-argument", "blocks were replaced by a newer prepare_blocks");
    return st;
}
VecX get_block(const AugmentedBlocks& B, int what, size_t count) {
    const auto& st = ledger_level(B);
    VecX out(count);
    b200::check(ksb_blocks_get(st.lev, what, out.data()));
    return out;
}
MatX square(const AugmentedBlocks& B, int what) {
    const int nh = B.space_h->state()->nH;
    MatX m(nh, nh);
    m.a = get_block(B, what, size_t(nh) * nh);
    return m;
}
VecX orbital_vec(const AugmentedBlocks& B, int what, int i) {
    const int nh = B.space_h->state()->nH;
    if (i < 0 || i >= B.n_orbitals) fail("invalid-argument", "orbital index out of range");
    const VecX all = get_block(B, what, size_t(B.n_orbitals) * nh);
    return VecX(all.begin() + size_t(i) * nh, all.begin() + size_t(i + 1) * nh);
}
} // namespace

MatX AugmentedBlocks::A_H1() const { return square(*this, 0); }
MatX AugmentedBlocks::A_H3() const { return square(*this, 1); }
MatX AugmentedBlocks::A_H4() const { return square(*this, 2); }
MatX AugmentedBlocks::M_H() const { return square(*this, 3); }
MatX AugmentedBlocks::C_H() const { return square(*this, 4); }
VecX AugmentedBlocks::d_Hh() const { return get_block(*this, 5, size_t(space_h->state()->nH)); }
VecX AugmentedBlocks::lift_load() const { return get_block(*this, 6, size_t(space_h->state()->nH)); }
double AugmentedBlocks::zeta() const { return get_block(*this, 7, 2)[0]; }
double AugmentedBlocks::lift_load0() const { return get_block(*this, 7, 2)[1]; }
MatX AugmentedBlocks::A_h4(int i) const {
    const int nh = space_h->state()->nH;
    if (i < 0 || i >= n_orbitals) fail("invalid-argument", "orbital index out of range");
    const VecX all = get_block(*this, 10, size_t(n_orbitals) * nh * nh);
    MatX m(nh, nh);
    std::copy(all.begin() + size_t(i) * nh * nh, all.begin() + size_t(i + 1) * nh * nh, m.a.begin());
    return m;
}
VecX AugmentedBlocks::b_H1(int i) const { return orbital_vec(*this, 11, i); }
VecX AugmentedBlocks::b_H3(int i) const { return orbital_vec(*this, 12, i); }
VecX AugmentedBlocks::b_H4(int i) const { return orbital_vec(*this, 13, i); }
VecX AugmentedBlocks::rhs(int i) const { return orbital_vec(*this, 14, i); }
VecX AugmentedBlocks::c_Hh(int i) const { return orbital_vec(*this, 15, i); }
VecX AugmentedBlocks::d_phi(int i) const { return orbital_vec(*this, 16, i); }
VecX AugmentedBlocks::beta1() const { return get_block(*this, 17, size_t(n_orbitals)); }
VecX AugmentedBlocks::beta3() const { return get_block(*this, 18, size_t(n_orbitals)); }
VecX AugmentedBlocks::beta4() const { return get_block(*this, 19, size_t(n_orbitals)); }
VecX AugmentedBlocks::gamma_mass() const { return get_block(*this, 20, size_t(n_orbitals)); }
VecX AugmentedBlocks::zeta_phi() const { return get_block(*this, 21, size_t(n_orbitals)); }

AugmentedBlocks prepare_blocks(fem::SpacePtr space_H, fem::SpacePtr space_h, const fem::Prolongation& P_full,
                               const SpMat& S_f, const SpMat& M_f, const SpMat& a_f,
                               const std::vector<fem::FEFunction>& phi_tilde, const fem::FEFunction& w_tilde,
                               const fem::FEFunction& v_xc, double occupancy, bool hartree_on, const VecX& hartree_bc,
                               WorkerPool*) {
    if (!space_h || !space_H) fail("invalid-argument", "null space");
    auto& st = *space_h->state();
    if (S_f.state() != space_h->state() || M_f.state() != space_h->state() || a_f.state() != space_h->state())
        fail("mismatched-spaces", "operators live on a different space");
    if (S_f.id() != KSB_MAT_S || M_f.id() != KSB_MAT_M || a_f.id() != KSB_MAT_AOP)
        fail("invalid-argument", "prepare_blocks reads the level's own make_level_ops operators");
    if (P_full.from != 0 || P_full.rows != space_h->n_dofs() || P_full.cols != space_H->n_dofs())
        fail("mismatched-spaces", "P_full does not map the correction space to this level");
    require_system(*space_h);
    const int N = int(phi_tilde.size());
    if (N < 1) fail("invalid-argument", "empty orbital set");
    fem::same_space(w_tilde, *space_h, "w_tilde lives on a different space");
    fem::same_space(v_xc, *space_h, "v_xc lives on a different space");
    AugmentedBlocks B;
    B.space_H = space_H;
    B.space_h = space_h;
    B.n_orbitals = N;
    B.occupancy = occupancy;
    B.hartree_on = hartree_on;
    B.phi_tilde.reserve(size_t(N));
    for (const auto& f : phi_tilde) B.phi_tilde.push_back(f.coeffs);
    // lift split (proj/src/correction.cpp:129-132)
    const int n = space_h->n_dofs();
    B.ell.assign(size_t(n), 0.0);
    if (int(hartree_bc.size()) == n)
        for (int d : st.boundary) B.ell[size_t(d)] = hartree_bc[size_t(d)];
    B.w_tilde0 = w_tilde.coeffs;
    for (int i = 0; i < n; ++i) B.w_tilde0[size_t(i)] -= B.ell[size_t(i)];
    int ld = 0;
    auto blk = fem::orbital_block(*space_h, phi_tilde, ld);
    b200::DeviceBuffer dwt(space_h->device(), B.w_tilde0), dell(space_h->device(), B.ell),
        dvxc(space_h->device(), v_xc.coeffs);
    b200::check(ksb_prepare_blocks(st.lev, blk.data(), ld, dwt.data(), dell.data(), dvxc.data()));
    B.generation = ++st.blocks_gen;
    return B;
}

AugmentedState pure_augmentation_state(const AugmentedBlocks& blocks, const VecX& lambda_init) {
    AugmentedState s;
    const int nh = blocks.space_h->state()->nH;
    s.lambda = lambda_init;
    s.phi_H.assign(size_t(blocks.n_orbitals), VecX(size_t(nh), 0.0));
    s.theta2.assign(size_t(blocks.n_orbitals), 1.0);
    s.w_H.assign(size_t(nh), 0.0);
    s.theta1 = blocks.hartree_on ? 1.0 : 0.0;
    return s;
}

InnerResult inner_scf(const AugmentedBlocks& blocks, const AugmentedState& init, const InnerOptions& opt) {
    auto& st = *blocks.space_h->state();
    ledger_level(blocks);
    const int N = blocks.n_orbitals, nh = st.nH;
    // the device loop starts from the pure augmentation state, the only start the reference uses
    const auto pure = pure_augmentation_state(blocks, init.lambda);
    bool is_pure = init.theta2 == pure.theta2 && init.w_H == pure.w_H && init.theta1 == pure.theta1 &&
                   int(init.phi_H.size()) == N;
    for (const auto& p : init.phi_H) is_pure = is_pure && p == pure.phi_H.front();
    if (!is_pure) fail("invalid-argument", "the device inner iteration starts from pure_augmentation_state");
    const auto o = step_opts(1e-9, opt.tol, opt.max_iterations, opt.score_floor, opt.nev_scan_pad);
    InnerResult r;
    r.state.lambda.assign(size_t(N), 0.0);
    VecX phi(size_t(N) * nh);
    r.state.theta2.assign(size_t(N), 0.0);
    r.state.w_H.assign(size_t(nh), 0.0);
    int iters = 0;
    const int cap = std::max(1, opt.max_iterations);
    VecX hist(size_t(cap), 0.0);
    b200::check(ksb_inner_scf(st.lev, &o, init.lambda.data(), r.state.lambda.data(), phi.data(), r.state.theta2.data(),
                              r.state.w_H.data(), &r.state.theta1, &iters, hist.data(), cap));
    r.iterations = iters;
    r.history.assign(hist.begin(), hist.begin() + std::min(iters, cap));
    for (int i = 0; i < N; ++i) r.state.phi_H.emplace_back(phi.begin() + size_t(i) * nh, phi.begin() + size_t(i + 1) * nh);
    st.inner_of = blocks.generation;
    st.inner_lambda = r.state.lambda;
    st.inner_theta1 = r.state.theta1;
    return r;
}

Expanded expand(const AugmentedState& s, const AugmentedBlocks& blocks) {
    auto& st = *blocks.space_h->state();
    ledger_level(blocks);
    if (st.inner_of != blocks.generation || s.lambda != st.inner_lambda || s.theta1 != st.inner_theta1)
        fail("invalid-argument", "expand takes the state the last inner_scf on these blocks returned");
    const int N = blocks.n_orbitals, n = blocks.space_h->n_dofs();
    std::vector<fem::FEFunction> pt;
    for (const auto& c : blocks.phi_tilde) pt.emplace_back(blocks.space_h, c, fem::Role::wavefunction);
    int ld = 0;
    auto blk = fem::orbital_block(*blocks.space_h, pt, ld);
    VecX bcb(size_t(std::max(1, st.nb)), 0.0);
    for (int k = 0; k < st.nb; ++k) bcb[size_t(k)] = blocks.ell[size_t(st.boundary[size_t(k)])];
    auto& dev = blocks.space_h->device();
    b200::DeviceBuffer dwt(dev, blocks.w_tilde0), db(dev, bcb), dphi(dev, int64_t(st.ni) * ld), dw(dev, int64_t(n));
    b200::check(ksb_expand(st.lev, blk.data(), ld, dwt.data(), db.data(), dphi.data(), dw.data()));
    Expanded e;
    e.lambda = s.lambda;
    e.orbitals = fem::from_block(blocks.space_h, dphi.to_host(), N, ld, fem::Role::wavefunction);
    e.hartree = fem::FEFunction(blocks.space_h, dw.to_host(), fem::Role::hartree);
    return e;
}

} // namespace corr

// ------------------------------------------------------------------ scf
namespace scf {

ScfResult self_consistent_solve(const model::MolecularSystem& sys, fem::SpacePtr space, const ScfOptions& opt,
                                WorkerPool*) {
    sys.validate();
    if (!space || space->state()->level != 0 || space->n_interior() != space->state()->nH)
        fail("invalid-argument", "the device coarse solve runs on level 0 of a hierarchy");
    const auto& V = *space;
    model::set_system(V, sys, opt.hartree_on, opt.xc_on && sys.xc.kind != model::XcKind::none);
    ksb_scf_opts o;
    b200::check(ksb_scf_defaults(&o));
    o.tol = opt.tol;
    o.max_iterations = opt.max_iterations;
    o.mixing = opt.mixing;
    o.hartree_on = opt.hartree_on ? 1 : 0;
    o.xc_on = opt.xc_on ? 1 : 0;
    o.tol_eig = opt.tol_eig;
    o.norm_l1 = opt.norm_l1 ? 1 : 0;
    const int N = sys.n_pairs, ld = N == 1 ? 1 : N + (N & 1);
    auto& dev = V.device();
    b200::DeviceBuffer phi(dev, int64_t(V.n_interior()) * ld), rho(dev, int64_t(V.n_dofs())),
        w(dev, int64_t(V.n_dofs()));
    ScfResult r;
    r.lambdas.assign(size_t(N), 0.0);
    VecX hist(size_t(std::max(1, opt.max_iterations)), 0.0);
    int it = 0;
    b200::check(ksb_coarse_scf(V.device_level(), &o, r.lambdas.data(), phi.data(), ld, rho.data(), w.data(), &it,
                               hist.data(), int(hist.size())));
    r.iterations = it;
    r.history.assign(hist.begin(), hist.begin() + it);
    r.orbitals = fem::from_block(space, phi.to_host(), N, ld, fem::Role::wavefunction);
    r.rho = fem::FEFunction(space, rho.to_host(), fem::Role::density);
    r.hartree = fem::FEFunction(space, w.to_host(), fem::Role::hartree);
    return r;
}

ScfResult initial_coarse_solve(const model::MolecularSystem& sys, fem::SpacePtr space, double scf_tol, ScfOptions opt,
                               WorkerPool* pool) {
    opt.tol = scf_tol;
    return self_consistent_solve(sys, std::move(space), opt, pool);
}

} // namespace scf

// ------------------------------------------------------------------ estimator
namespace est {

Indicators compute_indicators(const fem::FESpace& V, const model::MolecularSystem& sys, const VecX& lambdas,
                              const std::vector<fem::FEFunction>& orbitals, const fem::FEFunction& hartree_fn,
                              const fem::FEFunction& vxc_fn, WorkerPool*) {
    if (orbitals.empty()) fail("invalid-argument", "empty orbital set");
    if (lambdas.size() != orbitals.size()) fail("invalid-argument", "one eigenvalue per orbital");
    fem::same_space(hartree_fn, V, "hartree potential on a different space");
    fem::same_space(vxc_fn, V, "v_xc on a different space");
    model::MolecularSystem s2 = sys;
    s2.n_pairs = int(orbitals.size());
    model::set_system(V, s2, true, sys.xc.kind != model::XcKind::none);
    int ld = 0;
    auto blk = fem::orbital_block(V, orbitals, ld);
    b200::DeviceBuffer dw(V.device(), hartree_fn.coeffs), dv(V.device(), vxc_fn.coeffs);
    b200::DeviceBuffer deta(V.device(), int64_t(V.mesh().n_tets()));
    Indicators ind;
    b200::check(ksb_indicators(V.device_level(), lambdas.data(), blk.data(), ld, dw.data(), dv.data(), deta.data(),
                               &ind.total_sq));
    ind.eta_sq = deta.to_host();
    return ind;
}

std::vector<int> dorfler_mark(const Indicators& ind, double theta) {
    std::vector<int32_t> mk(ind.eta_sq.size());
    int64_t n = 0;
    b200::check(ksb_dorfler_mark(ind.eta_sq.data(), int64_t(ind.eta_sq.size()), ind.total_sq, theta, mk.data(), &n));
    return std::vector<int>(mk.begin(), mk.begin() + n);
}

} // namespace est

// ------------------------------------------------------------------ driver
namespace driver {

LevelOps make_level_ops(const fem::SpaceHierarchy& hier, int level, const model::MolecularSystem& sys, WorkerPool*) {
    sys.validate();
    LevelOps ops;
    ops.space = hier.space(level);
    const auto& V = *ops.space;
    model::set_system(V, sys, true, sys.xc.kind != model::XcKind::none);
    b200::check(ksb_level_ops(V.device_level()));
    ops.S = SpMat(V.state(), KSB_MAT_S, false);
    ops.M = SpMat(V.state(), KSB_MAT_M, false);
    ops.a_op = SpMat(V.state(), KSB_MAT_AOP, false);
    ops.stiffness = std::make_unique<fem::EllipticSolver>(ops.S, ops.space);
    ops.P_full = hier.prolongation(0, level);
    return ops;
}

CorrectionState::CorrectionState(const LevelOps& ops, const model::MolecularSystem& sys, const StepOptions& opt,
                                 const VecX& lambdas, const std::vector<fem::FEFunction>& orbitals,
                                 const fem::FEFunction& w)
    : space_(ops.space), N_(int(orbitals.size())), opt_(opt), lambda_(lambdas) {
    if (N_ != sys.n_pairs || int(lambdas.size()) != N_) fail("invalid-argument", "one orbital and eigenvalue per pair");
    model::set_system(*space_, sys, opt.hartree, opt.xc && sys.xc.kind != model::XcKind::none);
    phi_ = fem::orbital_block(*space_, orbitals, ld_);
    fem::same_space(w, *space_, "w lives on a different space");
    w_ = b200::DeviceBuffer(space_->device(), w.coeffs);
}

StepLog CorrectionState::step() {
    auto o = corr::step_opts(opt_.tol_linear, opt_.tol_inner, opt_.max_inner, opt_.score_floor, opt_.nev_scan_pad);
    o.norm_l1 = opt_.norm_l1 ? 1 : 0;
    ksb_step_log lg{};
    StepLog out;
    out.attempts.assign(size_t(N_), 0);
    out.cg_iterations.assign(size_t(N_), 0);
    b200::check(ksb_correction_step(space_->device_level(), &o, lambda_.data(), phi_.data(), ld_, w_.data(), &lg,
                                    out.attempts.data(), out.cg_iterations.data()));
    out.inner_iterations = lg.inner_iterations;
    out.hartree_iterations = lg.hartree_iterations;
    out.delta = lg.delta;
    out.ms_bvp = lg.ms_bvp;
    out.ms_hartree = lg.ms_hartree;
    out.ms_project = lg.ms_project;
    out.ms_inner = lg.ms_inner;
    out.ms_total = lg.ms_total;
    return out;
}

std::vector<fem::FEFunction> CorrectionState::orbitals() const {
    return fem::from_block(space_, phi_.to_host(), N_, ld_, fem::Role::wavefunction);
}
fem::FEFunction CorrectionState::hartree() const { return fem::FEFunction(space_, w_.to_host(), fem::Role::hartree); }

RunLog run(const RunConfig& cfg) {
    using Clock = std::chrono::steady_clock;
    auto secs = [](Clock::time_point t) { return std::chrono::duration<double>(Clock::now() - t).count(); };
    const auto t_start = Clock::now();
    RunLog log;
    const auto& sys = cfg.system;
    fem::SpaceHierarchy hier;
    mesh::MeshPtr m = mesh::build_box_mesh(sys.domain, cfg.n_coarse);
    hier.push(m);
    VecX lam;
    std::vector<fem::FEFunction> orbs;
    fem::FEFunction w, rho;
    est::Indicators ind;
    StepOptions so;
    so.tol_linear = cfg.tol_linear;
    so.tol_inner = cfg.tol_inner;
    so.score_floor = cfg.score_floor;
    so.max_inner = cfg.max_inner;
    so.nev_scan_pad = cfg.nev_scan_pad;
    // RunConfig::hartree_enabled / xc_enabled (proj/include/ksafem/runconfig.hpp:39-45)
    so.hartree = cfg.mode != Mode::linear;
    so.xc = cfg.mode != Mode::linear;
    so.norm_l1 = cfg.outer_norm_l1;
    try {
        for (int level = 0; level < cfg.max_levels; ++level) {
            LevelRecord rec;
            rec.level = level;
            const auto t_level = Clock::now();
            auto t0 = Clock::now();
            if (level > 0) {
                m = cfg.uniform ? mesh::uniform_refine(*m) : mesh::adapt_refine(*m, est::dorfler_mark(ind, cfg.theta));
                hier.push(m);
            }
            const LevelOps ops = make_level_ops(hier, level, sys);
            rec.t_refine = secs(t0);
            t0 = Clock::now();
            if (level == 0) {
                scf::ScfOptions opt;
                opt.tol = cfg.tol_outer;
                opt.max_iterations = cfg.max_scf;
                opt.mixing = cfg.mixing;
                opt.tol_eig = cfg.tol_eig;
                opt.hartree_on = so.hartree;
                opt.xc_on = so.xc;
                opt.norm_l1 = cfg.outer_norm_l1;
                const auto r = scf::initial_coarse_solve(sys, hier.space(0), cfg.tol_outer, opt);
                rec.outer_iterations = r.iterations;
                lam = r.lambdas;
                orbs = r.orbitals;
                w = r.hartree;
                rho = r.rho;
            } else {
                std::vector<fem::FEFunction> warm;
                for (const auto& o : orbs) warm.push_back(hier.prolong(o, level));
                const auto res = cfg.mode == Mode::standard_mlc
                                     ? solve_level_mlc(ops, sys, so, lam, warm, hier.prolong(w, level), cfg.tol_outer,
                                                       cfg.max_scf)
                                     : solve_level_corrected(ops, sys, so, lam, warm, hier.prolong(w, level),
                                                             cfg.tol_outer, cfg.max_outer);
                lam = res.lambdas;
                orbs = res.orbitals;
                w = res.hartree;
                rho = model::density(orbs, sys.occupancy);
                rec.outer_iterations = res.outer_iterations;
                rec.inner_iterations = res.inner_iterations;
            }
            rec.t_solve = secs(t0);
            t0 = Clock::now();
            const auto vxc = sys.xc.kind == model::XcKind::none ? fem::FEFunction(ops.space)
                                                                : model::xc_potential_field(sys.xc, rho);
            ind = est::compute_indicators(*ops.space, sys, lam, orbs, w, vxc);
            rec.t_estimate = secs(t0);
            rec.n_tets = m->n_tets();
            rec.n_dofs = ops.space->n_dofs();
            rec.lambdas = lam;
            rec.energy = model::total_energy(sys, orbs, w);
            rec.eta_sq_total = ind.total_sq;
            rec.t_total = secs(t_level);
            log.records.push_back(rec);
        }
    } catch (const Error& e) {
        log.aborted = true;
        log.abort_reason = e.what();
    }
    log.wall_seconds = secs(t_start);
    return log;
}

LevelResult solve_level_corrected(const LevelOps& ops, const model::MolecularSystem& sys, const StepOptions& opt,
                                  const VecX& lambdas, const std::vector<fem::FEFunction>& orbitals,
                                  const fem::FEFunction& w, double tol_outer, int max_outer) {
    CorrectionState cs(ops, sys, opt, lambdas, orbitals, w);
    LevelResult r;
    for (int outer = 0; outer < max_outer; ++outer) {
        const StepLog lg = cs.step();
        r.inner_iterations.push_back(lg.inner_iterations);
        r.deltas.push_back(lg.delta);
        r.outer_iterations = outer + 1;
        if (lg.delta < tol_outer) {
            r.lambdas = cs.lambdas();
            r.orbitals = cs.orbitals();
            r.hartree = cs.hartree();
            return r;
        }
    }
    fail("nonconvergence", "outer iteration cap reached");
}

LevelResult solve_level_mlc(const LevelOps& ops, const model::MolecularSystem& sys, const StepOptions& opt,
                            const VecX& lambdas, const std::vector<fem::FEFunction>& orbitals,
                            const fem::FEFunction& w, double tol_outer, int max_scf) {
    const int N = int(orbitals.size());
    if (N != sys.n_pairs || int(lambdas.size()) != N) fail("invalid-argument", "one orbital and eigenvalue per pair");
    const auto& space = ops.space;
    model::set_system(*space, sys, opt.hartree, opt.xc && sys.xc.kind != model::XcKind::none);
    int ld = 0;
    b200::DeviceBuffer phi = fem::orbital_block(*space, orbitals, ld);
    fem::same_space(w, *space, "w lives on a different space");
    b200::DeviceBuffer wd(space->device(), w.coeffs);
    auto o = corr::step_opts(opt.tol_linear, opt.tol_inner, opt.max_inner, opt.score_floor, opt.nev_scan_pad);
    o.norm_l1 = opt.norm_l1 ? 1 : 0;
    VecX lam = lambdas;
    ksb_step_log lg{};
    std::vector<int> att(static_cast<size_t>(N)), its(static_cast<size_t>(N));
    b200::check(ksb_mlc_begin(space->device_level(), &o, lam.data(), phi.data(), ld, wd.data(), &lg, att.data(),
                              its.data()));
    LevelResult r;
    for (int s = 1; s <= max_scf; ++s) {
        double delta = 0.0;
        b200::check(ksb_mlc_sweep(space->device_level(), &o, lam.data(), phi.data(), ld, &delta));
        r.deltas.push_back(delta);
        r.outer_iterations = s;
        if (delta < tol_outer) break;
        if (s == max_scf) fail("nonconvergence", "correction-space iteration cap reached");
    }
    b200::check(ksb_mlc_finish(space->device_level(), &o, wd.data(), nullptr));
    r.lambdas = lam;
    r.orbitals = fem::from_block(space, phi.to_host(), N, ld, fem::Role::wavefunction);
    r.hartree = fem::FEFunction(space, wd.to_host(), fem::Role::hartree);
    return r;
}

} // namespace driver
} // namespace ksafem
