// C-ABI implementation (include/ksb.h). No exceptions cross this boundary.
#include "host/dump.hpp"
#include <algorithm>
#include <cstring>
#include <exception>
#include <new>

#include "device/cg.cuh"
#include "device/correction.cuh"
#include "device/level.cuh"
#include "ksb.h"

struct ksb_mesh {
    ksb::MeshPtr m;
};
struct ksb_hier {
    ksb::Hierarchy h;
};
struct ksb_level;
struct ksb_ctx {
    ksb::Ctx c;
    ksb::CgWork cg;
    std::vector<ksb_level*> levels;  // live levels created on this context (their owner pointers are cleared
                                     // when the context goes first)
    ksb::DevBuf<double> io_b, io_x;  // staging for the host-buffer entry points
};
struct ksb_level {
    ksb_ctx* owner = nullptr;
    ksb::Level L;
    std::unique_ptr<ksb::Corrector> K;
    ksb::DevBuf<double> scratch;  // EllipticSolver::solve staging (interior rhs / solution, boundary data)
    ksb::Corrector& corr() {
        if (!K) K = std::make_unique<ksb::Corrector>();
        return *K;
    }
};

namespace ksb {

void axpby_values(Level& L, int dst, double a, int x, double b, int y);

cudaEvent_t Ctx::take_event() {
    if (!event_pool.empty()) {
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    KSB_CUDA_CHECK(cudaEventCreate(&e));
    return e;
}

void Ctx::begin(const char*, cudaEvent_t* e0) {
    *e0 = take_event();
    KSB_CUDA_CHECK(cudaEventRecord(*e0, stream));
}

void Ctx::end(const char* name, cudaEvent_t e0) {
    cudaEvent_t e1 = take_event();
    KSB_CUDA_CHECK(cudaEventRecord(e1, stream));
    pending.push_back({name, {e0, e1}});
    if (pending.size() > 4096) harvest();
}

void Ctx::harvest() {
    if (pending.empty()) return;
    KSB_CUDA_CHECK(cudaStreamSynchronize(stream));
    for (auto& p : pending) {
        float ms = 0.f;
        KSB_CUDA_CHECK(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
        auto& t = timers[p.first];
        t.ms += ms;
        t.count += 1;
        event_pool.push_back(p.second.first);
        event_pool.push_back(p.second.second);
    }
    pending.clear();
}

} // namespace ksb

namespace {

thread_local std::string g_last_error;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return KSB_OK;
    } catch (const ksb::Failure& e) {
        g_last_error = std::string(ksb_code_name(e.code)) + ": " + e.what;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "internal: host allocation failed";
        return KSB_INTERNAL;
    } catch (const std::exception& e) {
        g_last_error = std::string("internal: ") + e.what();
        return KSB_INTERNAL;
    }
}

void need(bool ok, const char* what) {
    if (!ok) ksb::raise(KSB_INVALID_ARGUMENT, what);
}

} // namespace

extern "C" {

const char* ksb_last_error(void) { return g_last_error.c_str(); }

const char* ksb_code_name(int code) {
    switch (code) {
        case KSB_OK: return "ok";
        case KSB_NONCONVERGENCE: return "nonconvergence";
        case KSB_MISMATCHED_SPACES: return "mismatched-spaces";
        case KSB_SINGULAR_QUADRATURE: return "singular-quadrature";
        case KSB_AMBIGUOUS_SELECTION: return "ambiguous-selection";
        case KSB_INTERNAL: return "internal";
        case KSB_INVALID_ARGUMENT: return "invalid-argument";
        case KSB_INVALID_DOMAIN: return "invalid-domain";
        case KSB_HIERARCHY: return "hierarchy";
        case KSB_IO: return "io";
        case KSB_CUDA: return "cuda";
        default: return "unknown";
    }
}

int ksb_version(void) { return 1; }

// ---------------- mesh ----------------
int ksb_mesh_box(const double lo[3], const double hi[3], int n, ksb_mesh** out) {
    return guard([&] {
        need(out && lo && hi, "null argument");
        *out = new ksb_mesh{ksb::build_box_mesh(lo, hi, n)};
    });
}

int ksb_mesh_uniform_refine(const ksb_mesh* m, ksb_mesh** out) {
    return guard([&] {
        need(m && out, "null argument");
        *out = new ksb_mesh{ksb::uniform_refine(*m->m)};
    });
}

int ksb_mesh_adapt_refine(const ksb_mesh* m, const int32_t* marked, int64_t n, ksb_mesh** out) {
    return guard([&] {
        need(m && out && (n == 0 || marked), "null argument");
        *out = new ksb_mesh{ksb::adapt_refine(*m->m, marked, n)};
    });
}

void ksb_mesh_free(ksb_mesh* m) { delete m; }

int ksb_mesh_sizes(const ksb_mesh* m, int64_t s[8]) {
    return guard([&] {
        need(m && s, "null argument");
        const auto& M = *m->m;
        s[0] = M.n_vertices();
        s[1] = M.n_tets();
        s[2] = int64_t(M.bface.size() / 3);
        s[3] = int64_t(M.iface.size() / 3);
        s[4] = M.level;
        s[5] = M.n_parent_vertices;
        s[6] = s[7] = 0;
    });
}

int ksb_mesh_get(const ksb_mesh* m, int what, void* dst) {
    return guard([&] {
        need(m && dst, "null argument");
        const auto& M = *m->m;
        auto put = [&](const auto& v) { std::memcpy(dst, v.data(), v.size() * sizeof(v[0])); };
        switch (what) {
            case 0: put(M.xyz); break;
            case 1: put(M.tets); break;
            case 2: put(M.tuple); break;
            case 3: put(M.tag); break;
            case 4: put(M.parent); break;
            case 5: put(M.vparent); break;
            case 6: put(M.on_boundary); break;
            case 7: put(M.bface); break;
            case 8: put(M.iface); break;
            case 9: put(M.iface_tets); break;
            case 10: put(M.iface_geom); break;
            default: ksb::raise(KSB_INVALID_ARGUMENT, "unknown mesh array");
        }
    });
}

// ---------------- hierarchy ----------------
int ksb_hier_create(ksb_hier** out) {
    return guard([&] {
        need(out, "null argument");
        *out = new ksb_hier;
    });
}

int ksb_hier_push(ksb_hier* h, const ksb_mesh* m) {
    return guard([&] {
        need(h && m, "null argument");
        h->h.push(m->m);
    });
}

void ksb_hier_free(ksb_hier* h) { delete h; }

int ksb_hier_levels(const ksb_hier* h) { return h ? h->h.n_levels() : 0; }

int ksb_hier_mesh(const ksb_hier* h, int level, ksb_mesh** out) {
    return guard([&] {
        need(h && out, "null argument");
        if (level < 0 || level >= h->h.n_levels()) ksb::raise(KSB_HIERARCHY, "level out of range");
        *out = new ksb_mesh{h->h.mesh_ptr(level)};
    });
}

int ksb_hier_save(const ksb_hier* h, const char* path) {
    return guard([&] {
        need(h && path, "null argument");
        std::vector<ksb::MeshPtr> ms;
        for (int k = 0; k < h->h.n_levels(); ++k) ms.push_back(h->h.mesh_ptr(k));
        ksb::save_meshes(path, ms);
    });
}

int ksb_hier_load(const char* path, ksb_hier** out) {
    return guard([&] {
        need(path && out, "null argument");
        auto ms = ksb::load_meshes(path);
        auto* h = new ksb_hier;
        try {
            for (size_t k = 0; k < ms.size(); ++k) {
                if (k > 0 && ms[k]->n_parent_vertices != ms[k - 1]->n_vertices())
                    ksb::raise(KSB_HIERARCHY, "stored levels are not nested");
                h->h.push(ms[k]);
            }
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int ksb_mesh_save(const ksb_mesh* m, const char* path) {
    return guard([&] {
        need(m && path, "null argument");
        ksb::save_meshes(path, {m->m});
    });
}

int ksb_mesh_load(const char* path, ksb_mesh** out) {
    return guard([&] {
        need(path && out, "null argument");
        auto ms = ksb::load_meshes(path);
        if (ms.size() != 1) ksb::raise(KSB_IO, std::string(path) + ": holds " + std::to_string(ms.size()) + " meshes");
        *out = new ksb_mesh{ms[0]};
    });
}

int ksb_state_save(const char* path, int level, int N, int64_t ni, int64_t n, const double* h_lambda,
                   const double* h_Phi, int ld, const double* h_w) {
    return guard([&] {
        need(path && h_lambda && h_Phi && h_w, "null argument");
        if (N < 1 || ld < N || ni < 0 || n < ni) ksb::raise(KSB_INVALID_ARGUMENT, "bad state sizes");
        ksb::State s;
        s.level = level;
        s.N = N;
        s.ni = ni;
        s.n = n;
        s.lambdas.assign(h_lambda, h_lambda + N);
        s.phi.resize(size_t(ni) * N);
        for (int64_t r = 0; r < ni; ++r)
            for (int c = 0; c < N; ++c) s.phi[size_t(r) * N + c] = h_Phi[size_t(r) * ld + c];
        s.w.assign(h_w, h_w + n);
        ksb::save_state(path, s);
    });
}

int ksb_state_sizes(const char* path, int64_t sizes[4]) {
    return guard([&] {
        need(path && sizes, "null argument");
        const auto s = ksb::load_state(path);
        sizes[0] = s.level;
        sizes[1] = s.N;
        sizes[2] = s.ni;
        sizes[3] = s.n;
    });
}

int ksb_state_load(const char* path, double* h_lambda, double* h_Phi, int ld, double* h_w) {
    return guard([&] {
        need(path && h_lambda && h_Phi && h_w, "null argument");
        const auto s = ksb::load_state(path);
        if (ld < s.N) ksb::raise(KSB_INVALID_ARGUMENT, "ld < N");
        std::memcpy(h_lambda, s.lambdas.data(), sizeof(double) * size_t(s.N));
        for (int64_t r = 0; r < s.ni; ++r)
            for (int c = 0; c < s.N; ++c) h_Phi[size_t(r) * ld + c] = s.phi[size_t(r) * s.N + c];
        std::memcpy(h_w, s.w.data(), sizeof(double) * size_t(s.n));
    });
}

int ksb_hier_prolongation(const ksb_hier* h, int level, int32_t* col, double* val) {
    return guard([&] {
        need(h && col && val, "null argument");
        if (level < 0 || level >= h->h.n_levels()) ksb::raise(KSB_HIERARCHY, "level out of range");
        const auto& c = h->h.pcol(level);
        const auto& v = h->h.pval(level);
        std::memcpy(col, c.data(), c.size() * sizeof(int32_t));
        std::memcpy(val, v.data(), v.size() * sizeof(double));
    });
}

// ---------------- context ----------------
int ksb_ctx_create(int device, ksb_ctx** out) {
    return guard([&] {
        need(out, "null argument");
        int ndev = 0;
        KSB_CUDA_CHECK(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) ksb::raise(KSB_CUDA, "no such CUDA device");
        KSB_CUDA_CHECK(cudaSetDevice(device));
        auto* c = new ksb_ctx;
        c->c.device = device;
        cudaDeviceProp prop;
        KSB_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
        c->c.sm_count = prop.multiProcessorCount;
        KSB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
        KSB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->c.aux, cudaStreamNonBlocking));
        KSB_CUDA_CHECK(cudaEventCreateWithFlags(&c->c.fork, cudaEventDisableTiming));
        KSB_CUDA_CHECK(cudaEventCreateWithFlags(&c->c.join, cudaEventDisableTiming));
        *out = c;
    });
}

void ksb_ctx_destroy(ksb_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->c.device);
    cudaStreamSynchronize(c->c.stream);
    for (auto* l : c->levels) l->owner = nullptr;
    for (auto& p : c->c.pending) {
        cudaEventDestroy(p.second.first);
        cudaEventDestroy(p.second.second);
    }
    for (auto e : c->c.event_pool) cudaEventDestroy(e);
    cudaStreamSynchronize(c->c.aux);
    cudaEventDestroy(c->c.fork);
    cudaEventDestroy(c->c.join);
    cudaStreamDestroy(c->c.aux);
    cudaStreamDestroy(c->c.stream);
    delete c;
}

int ksb_ctx_stream(ksb_ctx* c, void** s) {
    return guard([&] {
        need(c && s, "null argument");
        *s = reinterpret_cast<void*>(c->c.stream);
    });
}

int ksb_ctx_sync(ksb_ctx* c) {
    return guard([&] {
        need(c, "null argument");
        KSB_CUDA_CHECK(cudaStreamSynchronize(c->c.stream));
    });
}

int ksb_ctx_set_profiling(ksb_ctx* c, int on) {
    return guard([&] {
        need(c, "null argument");
        c->c.harvest();
        c->c.profiling = on != 0;
    });
}

int ksb_ctx_kernel_time(ksb_ctx* c, const char* name, double* ms, int64_t* count) {
    return guard([&] {
        need(c && name && ms && count, "null argument");
        c->c.harvest();
        auto it = c->c.timers.find(name);
        *ms = it == c->c.timers.end() ? 0.0 : it->second.ms;
        *count = it == c->c.timers.end() ? 0 : it->second.count;
    });
}

int ksb_ctx_kernel_launches(ksb_ctx* c, int64_t* total) {
    return guard([&] {
        need(c && total, "null argument");
        *total = c->c.launches;
    });
}

int ksb_ctx_reset_counters(ksb_ctx* c) {
    return guard([&] {
        need(c, "null argument");
        c->c.harvest();
        c->c.timers.clear();
        c->c.launches = 0;
    });
}

int ksb_malloc(ksb_ctx* c, void** p, int64_t bytes) {
    return guard([&] {
        need(c && p && bytes >= 0, "bad argument");
        KSB_CUDA_CHECK(cudaSetDevice(c->c.device));
        KSB_CUDA_CHECK(cudaMalloc(p, size_t(bytes > 0 ? bytes : 1)));
    });
}

int ksb_free(ksb_ctx* c, void* p) {
    return guard([&] {
        need(c, "null argument");
        KSB_CUDA_CHECK(cudaFree(p));
    });
}

int ksb_memcpy_h2d(ksb_ctx* c, void* d, const void* h, int64_t bytes) {
    return guard([&] {
        need(c && d && h, "null argument");
        KSB_CUDA_CHECK(cudaMemcpyAsync(d, h, size_t(bytes), cudaMemcpyHostToDevice, c->c.stream));
    });
}

int ksb_memcpy_d2h(ksb_ctx* c, void* h, const void* d, int64_t bytes) {
    return guard([&] {
        need(c && d && h, "null argument");
        KSB_CUDA_CHECK(cudaMemcpyAsync(h, d, size_t(bytes), cudaMemcpyDeviceToHost, c->c.stream));
    });
}

// ---------------- level ----------------
int ksb_level_create(ksb_ctx* c, const ksb_hier* h, int level, ksb_level** out) {
    return guard([&] {
        need(c && h && out, "null argument");
        if (level < 0 || level >= h->h.n_levels()) ksb::raise(KSB_HIERARCHY, "level out of range");
        KSB_CUDA_CHECK(cudaSetDevice(c->c.device));
        auto* lv = new ksb_level;
        lv->owner = c;
        ksb::Level& L = lv->L;
        L.ctx = &c->c;
        try {
            ksb::upload_level(c->c, ksb::build_topology(h->h, level), L);
            for (int k = 0; k <= level; ++k) L.meshes.push_back(h->h.mesh_ptr(k));
            ksb::Ctx& cx = c->c;
            L.flag.alloc(4);
            KSB_CUDA_CHECK(cudaStreamSynchronize(cx.stream));
        } catch (...) {
            delete lv;
            throw;
        }
        c->levels.push_back(lv);
        *out = lv;
    });
}

void ksb_level_destroy(ksb_level* l) {
    if (!l) return;
    cudaDeviceSynchronize();
    if (ksb_ctx* c = l->owner) {  // null when the context was destroyed first
        c->cg.forget_level(l->L.uid);  // its captured CG graphs reference this level's arrays
        c->levels.erase(std::remove(c->levels.begin(), c->levels.end(), l), c->levels.end());
    }
    delete l;
}

int ksb_level_sizes(const ksb_level* l, int64_t s[10]) {
    return guard([&] {
        need(l && s, "null argument");
        const auto& L = l->L;
        s[0] = L.n;
        s[1] = L.ni;
        s[2] = L.nb;
        s[3] = L.nt;
        s[4] = L.nnz_ii;
        s[5] = L.nnz_ib;
        s[6] = L.nH;
        s[7] = L.nct;
        s[8] = L.ncv;
        s[9] = 0;
    });
}

int ksb_level_index(const ksb_level* l, int what, void* dst) {
    return guard([&] {
        need(l && dst, "null argument");
        const auto& T = *l->L.topo;
        auto put = [&](const auto& v) { std::memcpy(dst, v.data(), v.size() * sizeof(v[0])); };
        switch (what) {
            case 0: put(T.ii.ptr); break;
            case 1: put(T.ii.col); break;
            case 2: put(T.ib.ptr); break;
            case 3: put(T.ib.col); break;
            case 4: put(T.space->interior); break;
            case 5: put(T.pint_col); break;
            case 6: put(T.pint_val); break;
            case 7:
                if (T.t8_col.empty()) ksb::raise(KSB_INVALID_ARGUMENT, "level has no T8 view (a row is longer than 16)");
                put(T.t8_col);
                break;
            case 8:
            case 9:
            case 10:
                if (T.lo_perm.empty()) ksb::raise(KSB_INVALID_ARGUMENT, "level has no locality order");
                put(what == 8 ? T.lo_perm : what == 9 ? T.lo_ptr : T.lo_col);
                break;
            case 11: {  // stencil view: {ng, l0, lr, on_lo, first[0..ng)} (16 int32, ng = 0 without one)
                int32_t info[16] = {T.dia_ng, T.dia_l0, T.dia_lr, T.dia_lo};
                for (int q = 0; q < T.dia_ng && q < 9; ++q) info[4 + q] = T.dia_first[q];
                info[15] = T.dia_n;
                std::memcpy(dst, info, sizeof info);
                break;
            }
            case 12: {  // union-tile view sizes: {tiles, entries, rows per tile} (3 int32; tiles = 0 without the view)
                int32_t info[3] = {T.ut_nt, int32_t(T.ut_ent.size()), ksb::kUtR};
                std::memcpy(dst, info, sizeof info);
                break;
            }
            case 13: put(T.ut_rows); break;
            case 14: put(T.ut_eptr); break;
            case 15: put(T.ut_ent); break;
            case 16: put(T.ut_map); break;
            case 17: put(T.lo_map); break;
            default: ksb::raise(KSB_INVALID_ARGUMENT, "unknown index array");
        }
    });
}

// ---------------- operators ----------------
int ksb_mat_assemble(ksb_level* l, int mat, double c_s, double c_m, int pot_kind, int n_centers,
                     const double* pot_params, double c_p, const double* d_w, double c_w) {
    return guard([&] {
        need(l, "null argument");
        ksb::Potential pot;
        const ksb::Potential* pp = nullptr;
        if (pot_params && n_centers > 0) {
            if (pot_kind != KSB_POT_COULOMB && pot_kind != KSB_POT_GAUSSIAN)
                ksb::raise(KSB_INVALID_ARGUMENT, "unknown potential kind");
            pot.kind = pot_kind;
            pot.n = n_centers;
            const int stride = pot_kind == KSB_POT_COULOMB ? 4 : 5;
            pot.params.assign(pot_params, pot_params + size_t(stride) * n_centers);
            pp = &pot;
        }
        ksb::assemble_into(l->L, mat, c_s, c_m, pp, c_p, d_w, c_w);
    });
}

int ksb_mat_axpby(ksb_level* l, int dst, double a, int x, double b, int y) {
    return guard([&] {
        need(l, "null argument");
        ksb::axpby_values(l->L, dst, a, x, b, y);
    });
}

int ksb_mat_values(ksb_level* l, int mat, int part, double* dst) {
    return guard([&] {
        need(l && dst, "null argument");
        auto& L = l->L;
        if (mat < 0 || mat >= ksb::kMaxMats || !L.mats[mat].valid) ksb::raise(KSB_INVALID_ARGUMENT, "matrix not assembled");
        const auto& buf = part == 0 ? L.mats[mat].ii : L.mats[mat].ib;
        KSB_CUDA_CHECK(cudaMemcpyAsync(dst, buf.p, sizeof(double) * size_t(buf.n), cudaMemcpyDeviceToHost, L.ctx->stream));
        KSB_CUDA_CHECK(cudaStreamSynchronize(L.ctx->stream));
    });
}

int ksb_spmm(ksb_level* l, int mat, const double* X, int N, int ldx, double* Y, int ldy) {
    return guard([&] {
        need(l && X && Y, "null argument");
        auto& L = l->L;
        if (mat < 0 || mat >= ksb::kMaxMats || !L.mats[mat].valid) ksb::raise(KSB_INVALID_ARGUMENT, "matrix not assembled");
        ksb::spmm(*L.ctx, L, L.mats[mat].ii.p, nullptr, nullptr, X, N, ldx, Y, ldy);
    });
}

// ---------------- CG ----------------
int ksb_cg_defaults(ksb_cg_opts* o) {
    return guard([&] {
        need(o, "null argument");
        o->tol = 1e-9;
        o->max_iterations = 20000;
        o->fixed_iterations = 0;
        o->precond = 0;
        o->check_every = 8;
    });
}

static void run_cg(ksb_level* l, int mat, int shift_mat, const double* h_sigma, const double* d_B, double* d_X, int N,
                   int ld, const ksb_cg_opts* o, ksb_cg_stats* h_stats) {
    need(l && d_B && d_X && o, "null argument");
    if (o->precond != 0 && o->precond != 1)
        ksb::raise(KSB_INVALID_ARGUMENT, "precond must be 0 (Jacobi) or 1 (the reference's SGS)");
    if (mat < 0 || mat >= ksb::kMaxMats || (shift_mat >= ksb::kMaxMats)) ksb::raise(KSB_INVALID_ARGUMENT, "bad matrix id");
    ksb::CgOptions co;
    co.precond = o->precond;
    co.tol = o->tol;
    co.max_iterations = o->max_iterations;
    co.fixed_iterations = o->fixed_iterations;
    co.check_every = o->check_every;
    std::vector<ksb::CgColumnStats> st(N);
    ksb::cg_solve(*l->L.ctx, l->L, mat, shift_mat, h_sigma, d_B, d_X, N, ld, co, st.data(), l->owner->cg);
    if (h_stats)
        for (int j = 0; j < N; ++j) {
            h_stats[j].iterations = st[j].iterations;
            h_stats[j].relative_residual = st[j].relative_residual;
            h_stats[j].converged = st[j].converged;
            h_stats[j].breakdown = st[j].breakdown;
        }
}

int ksb_cg_solve(ksb_level* l, int mat, int shift_mat, const double* h_sigma, const double* d_B, double* d_X, int N,
                 int ld, const ksb_cg_opts* o, ksb_cg_stats* h_stats) {
    return guard([&] { run_cg(l, mat, shift_mat, h_sigma, d_B, d_X, N, ld, o, h_stats); });
}

int ksb_cg_solve_host(ksb_level* l, int mat, int shift_mat, const double* h_sigma, const double* h_B, double* h_X,
                      int N, int ld, const ksb_cg_opts* o, ksb_cg_stats* h_stats) {
    return guard([&] {
        need(l && h_B && h_X, "null argument");
        need(N >= 1 && ld >= N, "ld must be >= N");
        auto& c = *l->L.ctx;
        // device blocks keep an even leading dimension (16-byte column pairs); host rows may be odd
        const int dld = (N > 1 && (ld & 1)) ? ld + 1 : ld;
        auto& dB = l->owner->io_b;
        auto& dX = l->owner->io_x;
        const int64_t cnt = int64_t(l->L.ni) * dld;
        if (dB.n < cnt) dB.alloc(cnt);
        if (dX.n < cnt) dX.alloc(cnt);
        const size_t hp = sizeof(double) * size_t(ld), dp = sizeof(double) * size_t(dld);
        const size_t w = sizeof(double) * size_t(N);
        KSB_CUDA_CHECK(cudaMemcpy2DAsync(dB.p, dp, h_B, hp, w, size_t(l->L.ni), cudaMemcpyHostToDevice, c.stream));
        run_cg(l, mat, shift_mat, h_sigma, dB.p, dX.p, N, dld, o, h_stats);
        KSB_CUDA_CHECK(cudaMemcpy2DAsync(h_X, hp, dX.p, dp, w, size_t(l->L.ni), cudaMemcpyDeviceToHost, c.stream));
        KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    });
}


// ---------------- EllipticSolver ----------------
int ksb_solve(ksb_level* l, int mat, const double* d_b_full, const double* d_bc_full, const ksb_cg_opts* o,
              double* d_x_full, ksb_cg_stats* st) {
    return guard([&] {
        need(l && d_b_full && d_x_full, "null argument");
        if (mat < 0 || mat >= ksb::kMaxMats) ksb::raise(KSB_INVALID_ARGUMENT, "bad matrix id");
        ksb::CgOptions co;
        if (o) {
            if (o->precond != 0 && o->precond != 1)
                ksb::raise(KSB_INVALID_ARGUMENT, "precond must be 0 (Jacobi) or 1 (the reference's SGS)");
            co.precond = o->precond;
            co.tol = o->tol;
            co.max_iterations = o->max_iterations;
            co.fixed_iterations = o->fixed_iterations;
            co.check_every = o->check_every;
        }
        const auto r = ksb::elliptic_solve(l->L, l->owner->cg, l->scratch, mat, d_b_full, d_bc_full, co, d_x_full);
        if (st) {
            st->iterations = r.iterations;
            st->relative_residual = r.relative_residual;
            st->converged = r.converged;
            st->breakdown = r.breakdown;
        }
    });
}

int ksb_mat_min_diag(ksb_level* l, int mat, double* out) {
    return guard([&] {
        need(l && out, "null argument");
        if (mat < 0 || mat >= ksb::kMaxMats) ksb::raise(KSB_INVALID_ARGUMENT, "bad matrix id");
        *out = ksb::min_diagonal(l->L, mat, l->scratch);
    });
}

// ---------------- correction step ----------------
static ksb::StepOptions step_opts(const ksb_step_opts* o) {
    ksb::StepOptions so;
    if (o) {
        so.tol_linear = o->tol_linear;
        so.tol_inner = o->tol_inner;
        so.score_floor = o->score_floor;
        so.max_inner = o->max_inner;
        so.nev_pad = o->nev_pad;
        so.check_every = o->check_every;
        so.fixed_sweeps = o->fixed_sweeps;
        so.norm_l1 = o->norm_l1 != 0;
        if (o->precond < 0 || o->precond > 1) ksb::raise(KSB_INVALID_ARGUMENT, "precond must be 0 or 1");
        so.precond = o->precond;
    }
    return so;
}

static void fill_log(const ksb::StepLog& lg, ksb_step_log* log, int* att, int* its) {
    if (log) {
        log->inner_iterations = lg.inner_iterations;
        log->hartree_iterations = lg.hartree_iterations;
        log->delta = lg.delta;
        log->ms_bvp = lg.ms_bvp;
        log->ms_hartree = lg.ms_hartree;
        log->ms_project = lg.ms_project;
        log->ms_inner = lg.ms_inner;
        log->ms_total = lg.ms_total;
        log->cg_iterations = lg.cg_iterations;
    }
    for (size_t i = 0; i < lg.attempts.size(); ++i) {
        if (att) att[i] = lg.attempts[i];
        if (its) its[i] = lg.iterations[i];
    }
}

static ksb::Corrector& ready(ksb_level* l) {
    need(l != nullptr, "null level");
    auto& K = l->corr();
    if (!K.sys.set) ksb::raise(KSB_INVALID_ARGUMENT, "call ksb_system_set first");
    if (!K.ops_ready) ksb::level_ops(l->L, K);
    return K;
}

int ksb_step_defaults(ksb_step_opts* o) {
    return guard([&] {
        need(o, "null argument");
        o->tol_linear = 1e-9;
        o->tol_inner = 1e-8;
        o->score_floor = 1e-8;
        o->max_inner = 400;
        o->nev_pad = 4;
        o->check_every = 8;
        o->fixed_sweeps = 0;
        o->norm_l1 = 0;
        o->precond = 0;
    });
}

int ksb_system_set(ksb_level* l, const double* atoms, int n_atoms, int n_pairs, double occ, int xc_kind, double alpha,
                   double p_exch, int hartree_on, int xc_on) {
    return guard([&] {
        need(l && (n_atoms == 0 || atoms), "null argument");
        if (n_pairs < 1 || n_pairs > 128) ksb::raise(KSB_INVALID_ARGUMENT, "n_pairs must be in [1, 128]");
        if (!(occ > 0)) ksb::raise(KSB_INVALID_ARGUMENT, "occupancy must be positive");
        if (xc_kind < 0 || xc_kind > 2) ksb::raise(KSB_INVALID_ARGUMENT, "unknown xc kind");
        for (int a = 0; a < n_atoms; ++a)
            if (!(atoms[4 * a] > 0)) ksb::raise(KSB_INVALID_ARGUMENT, "nuclear charge must be positive");
        auto& K = l->corr();
        K.sys.atoms.assign(atoms, atoms + 4 * n_atoms);
        K.sys.N = n_pairs;
        K.sys.occ = occ;
        K.sys.xc = ksb::XcParams{xc_kind, alpha, p_exch};
        K.sys.hartree_on = hartree_on != 0;
        K.sys.xc_on = xc_on != 0 && xc_kind != 0;
        K.sys.set = true;
        K.ops_ready = false;
    });
}

int ksb_level_ops(ksb_level* l) {
    return guard([&] {
        need(l, "null argument");
        auto& K = l->corr();
        if (!K.sys.set) ksb::raise(KSB_INVALID_ARGUMENT, "call ksb_system_set first");
        ksb::level_ops(l->L, K);
    });
}

int ksb_scf_defaults(ksb_scf_opts* o) {
    return guard([&] {
        need(o, "null argument");
        o->tol = 1e-6;
        o->max_iterations = 200;
        o->mixing = 0.3;
        o->hartree_on = 1;
        o->xc_on = 1;
        o->tol_eig = 1e-9;
        o->norm_l1 = 0;
    });
}

int ksb_coarse_scf(ksb_level* l, const ksb_scf_opts* o, double* h_lambda, double* d_Phi, int ld, double* d_rho,
                   double* d_w, int* iters, double* hist, int cap) {
    return guard([&] {
        auto& K = ready(l);
        need(o && h_lambda && d_Phi && d_rho && d_w, "null argument");
        if (ld < K.sys.N || (K.sys.N > 1 && (ld & 1))) ksb::raise(KSB_INVALID_ARGUMENT, "bad block shape");
        ksb::ScfParams p;
        p.tol = o->tol;
        p.max_iterations = o->max_iterations;
        p.mixing = o->mixing;
        p.hartree_on = o->hartree_on != 0;
        p.xc_on = o->xc_on != 0;
        p.tol_eig = o->tol_eig;
        p.norm_l1 = o->norm_l1 != 0;
        ksb::ScfStats st;
        std::exception_ptr err;
        try {
            st = ksb::coarse_scf(l->L, K, l->owner->cg, p, h_lambda, d_Phi, ld, d_rho, d_w);
        } catch (...) {
            err = std::current_exception();
        }
        if (iters) *iters = err ? int(K.scf_history.size()) : st.iterations;
        if (hist)  // also when the cap was hit: the history says whether the iteration oscillates or creeps
            for (int k = 0; k < std::min<int>(cap, int(K.scf_history.size())); ++k) hist[k] = K.scf_history[k];
        if (err) std::rethrow_exception(err);
    });
}

int ksb_correction_step(ksb_level* l, const ksb_step_opts* o, double* h_lambda, double* d_Phi, int ld, double* d_w,
                        ksb_step_log* log, int* att, int* its) {
    return guard([&] {
        auto& K = ready(l);
        need(h_lambda && d_Phi && d_w, "null argument");
        if (ld < K.sys.N || (K.sys.N > 1 && (ld & 1))) ksb::raise(KSB_INVALID_ARGUMENT, "bad ld");
        ksb::StepLog lg;
        ksb::correction_step(l->L, K, l->owner->cg, step_opts(o), h_lambda, d_Phi, ld, d_w, &lg);
        fill_log(lg, log, att, its);
    });
}

int ksb_correction_step_host(ksb_level* l, const ksb_step_opts* o, double* h_lambda, double* h_Phi, int ld,
                             double* h_w, ksb_step_log* log, int* att, int* its) {
    return guard([&] {
        auto& K = ready(l);
        need(h_lambda && h_Phi && h_w, "null argument");
        auto& c = *l->L.ctx;
        const int64_t nb = int64_t(l->L.ni) * ld;
        auto& dP = l->owner->io_b;
        auto& dW = l->owner->io_x;
        if (dP.n < nb) dP.alloc(nb);
        if (dW.n < l->L.n) dW.alloc(l->L.n);
        KSB_CUDA_CHECK(cudaMemcpyAsync(dP.p, h_Phi, sizeof(double) * nb, cudaMemcpyHostToDevice, c.stream));
        KSB_CUDA_CHECK(cudaMemcpyAsync(dW.p, h_w, sizeof(double) * l->L.n, cudaMemcpyHostToDevice, c.stream));
        ksb::StepLog lg;
        ksb::correction_step(l->L, K, l->owner->cg, step_opts(o), h_lambda, dP.p, ld, dW.p, &lg);
        KSB_CUDA_CHECK(cudaMemcpyAsync(h_Phi, dP.p, sizeof(double) * nb, cudaMemcpyDeviceToHost, c.stream));
        KSB_CUDA_CHECK(cudaMemcpyAsync(h_w, dW.p, sizeof(double) * l->L.n, cudaMemcpyDeviceToHost, c.stream));
        KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
        fill_log(lg, log, att, its);
    });
}

int ksb_mlc_begin(ksb_level* l, const ksb_step_opts* o, const double* h_lambda, const double* d_Phi, int ld,
                  const double* d_w, ksb_step_log* log, int* att, int* its) {
    return guard([&] {
        auto& K = ready(l);
        need(h_lambda && d_Phi && d_w, "null argument");
        if (ld < K.sys.N || (K.sys.N > 1 && (ld & 1))) ksb::raise(KSB_INVALID_ARGUMENT, "bad ld");
        ksb::StepLog lg;
        ksb::mlc_begin(l->L, K, l->owner->cg, step_opts(o), h_lambda, d_Phi, ld, d_w, &lg);
        fill_log(lg, log, att, its);
    });
}

int ksb_mlc_sweep(ksb_level* l, const ksb_step_opts* o, double* h_lambda, double* d_Phi, int ld, double* h_delta) {
    return guard([&] {
        auto& K = ready(l);
        need(h_lambda && d_Phi, "null argument");
        const double d = ksb::mlc_sweep(l->L, K, l->owner->cg, step_opts(o), h_lambda, d_Phi, ld);
        if (h_delta) *h_delta = d;
    });
}

int ksb_mlc_finish(ksb_level* l, const ksb_step_opts* o, double* d_w, double* d_rho) {
    return guard([&] {
        auto& K = ready(l);
        need(d_w, "null argument");
        ksb::mlc_finish(l->L, K, l->owner->cg, step_opts(o), d_w, d_rho);
    });
}

int ksb_density_xc(ksb_level* l, const double* d_Phi, int N, int ld, double* d_rho, double* d_vxc) {
    return guard([&] {
        need(l && d_Phi && d_rho, "null argument");
        auto& K = l->corr();
        if (!K.sys.set) ksb::raise(KSB_INVALID_ARGUMENT, "call ksb_system_set first");
        ksb::rho_vxc(l->L, d_Phi, N, ld, K.sys.occ, K.sys.xc, d_rho, d_vxc);
    });
}

int ksb_density(ksb_level* l, const double* d_Phi, int N, int ld, double occ, double* d_rho) {
    return guard([&] {
        need(l && d_Phi && d_rho, "null argument");
        if (N < 1 || ld < N) ksb::raise(KSB_INVALID_ARGUMENT, "bad block shape");
        ksb::rho_vxc(l->L, d_Phi, N, ld, occ, ksb::XcParams{0, 0.0, 0.0}, d_rho, nullptr);
        KSB_CUDA_CHECK(cudaStreamSynchronize(l->L.ctx->stream));
    });
}

int ksb_moments(ksb_level* l, const double* d_rho, double out[16]) {
    return guard([&] {
        need(l && d_rho && out, "null argument");
        auto& L = l->L;
        const double ctr[3] = {0.5 * (L.box_lo[0] + L.box_hi[0]), 0.5 * (L.box_lo[1] + L.box_hi[1]),
                               0.5 * (L.box_lo[2] + L.box_hi[2])};
        const auto m = ksb::moments(L, d_rho, l->corr().phys, ctr);
        out[0] = m.q;
        for (int d = 0; d < 3; ++d) {
            out[1 + d] = m.c[d];
            out[4 + d] = m.dip[d];
            for (int e = 0; e < 3; ++e) out[7 + 3 * d + e] = m.Q[d][e];
        }
    });
}

int ksb_boundary_values(ksb_level* l, const double mom[16], double* d_bcb) {
    return guard([&] {
        need(l && mom && d_bcb, "null argument");
        ksb::Moments m{};
        m.q = mom[0];
        for (int d = 0; d < 3; ++d) {
            m.c[d] = mom[1 + d];
            m.dip[d] = mom[4 + d];
            for (int e = 0; e < 3; ++e) m.Q[d][e] = mom[7 + 3 * d + e];
        }
        ksb::boundary_values(l->L, m, d_bcb);
    });
}

int ksb_sqload(ksb_level* l, const double* d_Phi, int N, int ld, double* d_out) {
    return guard([&] {
        need(l && d_Phi && d_out, "null argument");
        auto& K = l->corr();
        if (!K.sys.set) ksb::raise(KSB_INVALID_ARGUMENT, "call ksb_system_set first");
        ksb::sqload(l->L, d_Phi, N, ld, K.sys.occ, 1.0, d_out, K.phys);
    });
}

int ksb_sqload_full(ksb_level* l, const double* d_Phi, int N, int ld, double occ, double* d_out_full) {
    return guard([&] {
        need(l && d_Phi && d_out_full, "null argument");
        if (N < 1 || ld < N) ksb::raise(KSB_INVALID_ARGUMENT, "bad block shape");
        ksb::sqload_full(l->L, d_Phi, N, ld, occ, d_out_full, l->corr().phys);
        KSB_CUDA_CHECK(cudaStreamSynchronize(l->L.ctx->stream));
    });
}

int ksb_xc_field(ksb_level* l, int xc_kind, double alpha, double p_exch, const double* d_rho, double* d_vxc) {
    return guard([&] {
        need(l && d_rho && d_vxc, "null argument");
        if (xc_kind < 0 || xc_kind > 2) ksb::raise(KSB_INVALID_ARGUMENT, "unknown xc kind");
        ksb::xc_field(l->L, ksb::XcParams{xc_kind, alpha, p_exch}, d_rho, d_vxc);
        KSB_CUDA_CHECK(cudaStreamSynchronize(l->L.ctx->stream));
    });
}

int ksb_hartree_solve(ksb_level* l, const double* d_Phi, int N, int ld, const double* d_bcb, double tol,
                      double* d_w_full, int* iters) {
    return guard([&] {
        auto& K = ready(l);
        need(d_Phi && d_bcb && d_w_full, "null argument");
        const int it = ksb::hartree_solve(l->L, K, l->owner->cg, d_Phi, N, ld, d_bcb, tol, d_w_full);
        if (iters) *iters = it;
    });
}

int ksb_outer_solve(ksb_level* l, const ksb_step_opts* o, const double* d_what, const double* d_vxc,
                    const double* h_lambda, const double* d_Phi, int ld, double* d_PhiT, int* att, int* its,
                    double* h_min_diag) {
    return guard([&] {
        auto& K = ready(l);
        need(d_what && d_vxc && h_lambda && d_Phi && d_PhiT, "null argument");
        const double md = ksb::outer_operator(l->L, K, d_what, d_vxc);
        if (h_min_diag) *h_min_diag = md;
        ksb::StepLog lg;
        ksb::solve_orbitals(l->L, K, l->owner->cg, step_opts(o), h_lambda, d_Phi, ld, d_PhiT, ld, &lg);
        fill_log(lg, nullptr, att, its);
    });
}

int ksb_outer_build(ksb_level* l, int aop_mat, const double* d_what, const double* d_vxc, double* h_min_diag) {
    return guard([&] {
        auto& K = ready(l);
        need(d_what && d_vxc, "null argument");
        if (aop_mat < 0 || aop_mat >= ksb::kMaxMats) ksb::raise(KSB_INVALID_ARGUMENT, "bad matrix id");
        const double md = ksb::outer_operator(l->L, K, d_what, d_vxc, aop_mat);
        if (h_min_diag) *h_min_diag = md;
    });
}

int ksb_outer_apply(ksb_level* l, const ksb_step_opts* o, const double* h_lambda, const double* d_Phi, int N, int ld,
                    double* d_PhiT, int* att, int* its) {
    return guard([&] {
        auto& K = ready(l);
        need(h_lambda && d_Phi && d_PhiT, "null argument");
        if (N < 1 || N > 128 || ld < N || (N > 1 && (ld & 1))) ksb::raise(KSB_INVALID_ARGUMENT, "bad block shape");
        if (!l->L.mats[ksb::MAT_H].valid) ksb::raise(KSB_INVALID_ARGUMENT, "call ksb_outer_build first");
        ksb::StepLog lg;
        ksb::solve_orbitals(l->L, K, l->owner->cg, step_opts(o), h_lambda, d_Phi, ld, d_PhiT, ld, &lg, N);
        for (int i = 0; i < N; ++i) {
            if (att) att[i] = lg.attempts[i];
            if (its) its[i] = lg.iterations[i];
        }
    });
}

int ksb_prepare_blocks(ksb_level* l, const double* d_PhiT, int ld, const double* d_wt, const double* d_ell,
                       const double* d_vxc) {
    return guard([&] {
        auto& K = ready(l);
        need(d_PhiT && d_wt && d_ell && d_vxc, "null argument");
        ksb::project_blocks(l->L, d_PhiT, K.sys.N, ld, d_wt, d_ell, d_vxc, K.eext.p, K.proj);
        KSB_CUDA_CHECK(cudaStreamSynchronize(l->L.ctx->stream));
    });
}

int ksb_blocks_get(ksb_level* l, int what, double* dst) {
    return guard([&] {
        auto& K = ready(l);
        need(dst, "null argument");
        auto& P = K.proj;
        auto& c = *l->L.ctx;
        const int64_t nh = l->L.nH, nh2 = nh * nh, N = K.sys.N;
        auto get = [&](const double* src, int64_t cnt) {
            KSB_CUDA_CHECK(cudaMemcpyAsync(dst, src, sizeof(double) * cnt, cudaMemcpyDeviceToHost, c.stream));
        };
        auto getv = [&](int o) {  // per orbital vector o of 6
            for (int64_t i = 0; i < N; ++i)
                KSB_CUDA_CHECK(cudaMemcpyAsync(dst + i * nh, P.orb_vecs.p + (i * 6 + o) * nh, sizeof(double) * nh,
                                               cudaMemcpyDeviceToHost, c.stream));
        };
        std::vector<double> sc;
        switch (what) {
            case 0: get(P.shared_mats.p, nh2); break;
            case 1: get(P.shared_mats.p + nh2, nh2); break;
            case 2: get(P.shared_mats.p + 2 * nh2, nh2); break;
            case 3: get(K.coarse.MH.p, nh2); break;
            case 4: get(K.coarse.CH.p, nh2); break;
            case 5: get(P.shared_vecs.p, nh); break;
            case 6: get(P.shared_vecs.p + nh, nh); break;
            case 7: get(P.shared_scal.p, 2); break;
            case 10: get(P.A_h4.p, N * nh2); break;
            case 11: getv(0); break;
            case 12: getv(1); break;
            case 13: getv(2); break;
            case 14: getv(5); break;
            case 15: getv(3); break;
            case 16: getv(4); break;
            case 17: case 18: case 19: case 20: case 21: {
                sc.resize(5 * N);
                KSB_CUDA_CHECK(cudaMemcpyAsync(sc.data(), P.orb_scal.p, sizeof(double) * 5 * N, cudaMemcpyDeviceToHost,
                                               c.stream));
                KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
                for (int64_t i = 0; i < N; ++i) dst[i] = sc[i * 5 + (what - 17)];
                break;
            }
            default: ksb::raise(KSB_INVALID_ARGUMENT, "unknown block");
        }
        KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    });
}

int ksb_inner_scf(ksb_level* l, const ksb_step_opts* o, const double* h_lambda, double* lam, double* phiH, double* th2,
                  double* wH, double* th1, int* iters, double* hist, int hist_cap) {
    return guard([&] {
        auto& K = ready(l);
        need(h_lambda, "null argument");
        const auto so = step_opts(o);
        ksb::InnerParams ip;
        ip.tol = so.tol_inner;
        ip.max_iterations = so.max_inner;
        ip.score_floor = so.score_floor;
        ip.nev_pad = so.nev_pad;
        ip.hartree = K.sys.hartree_on;
        ip.occ = K.sys.occ;
        ip.fixed_sweeps = so.fixed_sweeps;
        const auto st = ksb::inner_scf(l->L, K.coarse, K.proj, ip, h_lambda, K.inner, true);
        auto& w = K.inner;
        auto& c = *l->L.ctx;
        const int N = K.sys.N, nh = l->L.nH, cur = w.cur;
        if (lam) KSB_CUDA_CHECK(cudaMemcpyAsync(lam, w.lamv[cur].p, sizeof(double) * N, cudaMemcpyDeviceToHost, c.stream));
        if (phiH) KSB_CUDA_CHECK(cudaMemcpyAsync(phiH, w.phi[cur].p, sizeof(double) * N * nh, cudaMemcpyDeviceToHost, c.stream));
        if (th2) KSB_CUDA_CHECK(cudaMemcpyAsync(th2, w.th2[cur].p, sizeof(double) * N, cudaMemcpyDeviceToHost, c.stream));
        if (wH) KSB_CUDA_CHECK(cudaMemcpyAsync(wH, w.wH[cur].p, sizeof(double) * nh, cudaMemcpyDeviceToHost, c.stream));
        if (th1) KSB_CUDA_CHECK(cudaMemcpyAsync(th1, w.th1[cur].p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
        if (iters) *iters = st.iterations;
        if (hist)
            for (int k = 0; k < std::min<int>(hist_cap, int(st.history.size())); ++k) hist[k] = st.history[k];
    });
}

int ksb_expand(ksb_level* l, const double* d_PhiT, int ld, const double* d_wt, const double* d_bcb, double* d_Phi,
               double* d_w) {
    return guard([&] {
        auto& K = ready(l);
        need(d_PhiT && d_wt && d_bcb && d_Phi && d_w, "null argument");
        ksb::expand(l->L, K, d_PhiT, ld, d_wt, d_bcb, d_Phi, ld, d_w);
        KSB_CUDA_CHECK(cudaStreamSynchronize(l->L.ctx->stream));
    });
}

int ksb_prolong(ksb_level* l, const double* d_in, int in_interior, int ld_in, int ncols, double* d_out,
                int out_interior, int ld_out) {
    return guard([&] {
        need(l && d_in && d_out, "null argument");
        auto& L = l->L;
        if (L.n_prev == 0) ksb::raise(KSB_HIERARCHY, "level 0 has no previous level");
        if (ncols < 1 || ld_in < ncols || ld_out < ncols) ksb::raise(KSB_INVALID_ARGUMENT, "need 1 <= ncols <= ld");
        ksb::prolong(L, d_in, in_interior != 0, ld_in, ncols, d_out, out_interior != 0, ld_out);
        KSB_CUDA_CHECK(cudaStreamSynchronize(L.ctx->stream));
    });
}

int ksb_indicators(ksb_level* l, const double* h_lambda, const double* d_Phi, int ld, const double* d_w,
                   const double* d_vxc, double* d_eta, double* h_total_sq) {
    return guard([&] {
        auto& K = ready(l);
        need(h_lambda && d_Phi && d_w && d_vxc && d_eta, "null argument");
        const int N = K.sys.N;
        if (ld < N) ksb::raise(KSB_INVALID_ARGUMENT, "ld must be >= N");
        const double tot = ksb::indicators(l->L, K.est, K.sys.atoms, h_lambda, N, d_Phi, ld, d_w, d_vxc, d_eta);
        if (h_total_sq) *h_total_sq = tot;
    });
}

int ksb_dorfler_mark(const double* eta, int64_t nt, double total_sq, double theta, int32_t* marked, int64_t* n_marked) {
    return guard([&] {
        need(eta && marked && n_marked, "null argument");
        if (!(theta > 0.0) || theta >= 1.0) ksb::raise(KSB_INVALID_ARGUMENT, "theta must lie in (0,1)");
        *n_marked = 0;
        if (total_sq <= 0.0) return;
        *n_marked = ksb::dorfler_mark(eta, nt, total_sq, theta, marked);
    });
}

int ksb_norms(ksb_level* l, const double* d_f, double out[3]) {
    return guard([&] {
        need(l && d_f && out, "null argument");
        const auto a = ksb::norms_sq(l->L, d_f, l->corr().phys);
        out[0] = a[0];
        out[1] = a[1];
        const double l2 = std::sqrt(std::max(0.0, a[0])), semi = std::sqrt(std::max(0.0, a[1]));
        out[2] = std::sqrt(l2 * l2 + semi * semi);
    });
}

int ksb_l1_norm(ksb_level* l, const double* d_f, double* h_out) {
    return guard([&] {
        need(l && d_f && h_out, "null argument");
        *h_out = ksb::l1_norm(l->L, d_f, l->corr().phys);
    });
}

int ksb_energy(ksb_level* l, const double* d_Phi, int N, int ld, const double* d_w, double out[5]) {
    return guard([&] {
        need(l && d_Phi && d_w && out, "null argument");
        auto& K = l->corr();
        if (!K.sys.set) ksb::raise(KSB_INVALID_ARGUMENT, "call ksb_system_set first");
        ksb::DevBuf<double> rho;
        rho.alloc(l->L.n);
        ksb::rho_vxc(l->L, d_Phi, N, ld, K.sys.occ, K.sys.xc, rho.p, nullptr);
        const auto e = ksb::energy(l->L, d_Phi, N, ld, rho.p, d_w, K.sys.atoms, K.sys.occ, K.sys.xc, K.phys);
        for (int k = 0; k < 5; ++k) out[k] = e[k];
    });
}

} // extern "C"
