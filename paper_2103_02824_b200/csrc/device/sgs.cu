// Exact symmetric Gauss-Seidel preconditioned CG -- the reference's EllipticSolver::pcg with apply_sgs
// (proj/src/solver.cpp:50-111) on the device, for parity runs (CgOptions::precond = 1).
//
// z = (D+U)^-1 D' (D+L)^-1 r with the interior operator's own diagonal D in the triangular solves and D' = D with
// zeros replaced by 1 (solver.cpp:45). The triangular solves are level scheduled: row i of the forward solve depends
// on the rows j < i of its pattern, so rows are grouped by dependency depth (host, once per level) and each depth is
// one launch over its rows and the N columns. Every row accumulates in the order of the reference's column-oriented
// sparse solves (Eigen's / the oracle's): forward, subtractions in ascending column; backward, in descending column;
// products and differences rounded separately (the host reference has no fused multiply-add). The PCG control flow
// is solver.cpp:57-111 per column (zero right-hand side, breakdown on !(pAp > 0), recursive then true residual with
// restart), driven from the host with one synchronisation per iteration: this path is for parity, the production
// path is the fused Jacobi / multigrid CG of cg.cu.
#include <algorithm>
#include <cmath>

#include "cg.cuh"
#include "sgs.cuh"

namespace ksb {

namespace {

constexpr int kT = 256;

int grid_of(const Ctx& c, int64_t work) {
    const int64_t want = (work + kT - 1) / kT;
    return int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(c.sm_count) * 16)));
}

/// one dependency level of a triangular solve: y[i, c] = (rhs[i, c] - sum a_ij y[j, c]) / a_ii over the rows of the
/// level (lower: j < i ascending; upper: j > i descending); a = A + sigma_c B when B is given
__global__ void k_sgs_level(int nrows, const int32_t* __restrict__ rows, int N, int ld, const int32_t* __restrict__ ptr,
                            const int32_t* __restrict__ col, const double* __restrict__ A, const double* __restrict__ Bv,
                            const double* __restrict__ sigma, const double* __restrict__ rhs, double* __restrict__ y,
                            int lower) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(nrows) * N;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int i = rows[e / N], c = int(e % N);
        const int b = ptr[i], en = ptr[i + 1];
        double s = rhs[size_t(i) * ld + c], d = 0.0;
        auto val = [&](int q) { return Bv ? __dadd_rn(A[q], __dmul_rn(sigma[c], Bv[q])) : A[q]; };
        if (lower) {
            for (int q = b; q < en; ++q) {
                const int j = col[q];
                if (j < i)
                    s = __dsub_rn(s, __dmul_rn(y[size_t(j) * ld + c], val(q)));
                else if (j == i)
                    d = val(q);
            }
        } else {
            for (int q = en - 1; q >= b; --q) {
                const int j = col[q];
                if (j > i)
                    s = __dsub_rn(s, __dmul_rn(y[size_t(j) * ld + c], val(q)));
                else if (j == i)
                    d = val(q);
            }
        }
        y[size_t(i) * ld + c] = __ddiv_rn(s, d);
    }
}

/// y[i, c] *= D'_i (diagonal with zeros replaced by one)
__global__ void k_sgs_scale(int ni, int N, int ld, const int32_t* __restrict__ dslot, const double* __restrict__ A,
                            const double* __restrict__ Bv, const double* __restrict__ sigma, double* __restrict__ y) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(ni) * N;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e / N), c = int(e % N);
        const int q = dslot[i];
        const double d = Bv ? __dadd_rn(A[q], __dmul_rn(sigma[c], Bv[q])) : A[q];
        y[size_t(i) * ld + c] = __dmul_rn(y[size_t(i) * ld + c], d != 0.0 ? d : 1.0);
    }
}

/// per-column dot products of two blocks: block partials part[b * N + c], folded in fixed order by k_fold_cols
__global__ void k_coldot(int ni, int N, int ld, const double* __restrict__ X, const double* __restrict__ Y,
                         double* __restrict__ part) {
    extern __shared__ double red[];
    for (int c0 = 0; c0 < N; ++c0) {
        double s = 0.0;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ni; i += gridDim.x * blockDim.x)
            s += X[size_t(i) * ld + c0] * Y[size_t(i) * ld + c0];
        red[threadIdx.x] = s;
        __syncthreads();
        for (int o = blockDim.x / 2; o > 0; o >>= 1) {
            if (int(threadIdx.x) < o) red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) part[size_t(blockIdx.x) * N + c0] = red[0];
        __syncthreads();
    }
}

__global__ void k_fold_cols(int nb, int N, const double* __restrict__ part, double* __restrict__ out) {
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < nb; ++b) s += part[size_t(b) * N + c];
        out[c] = s;
    }
}

/// X[:, c] += a_c * P[:, c]; R[:, c] -= a_c * AP[:, c] for the columns with act_c
__global__ void k_sgs_xr(int ni, int N, int ld, const double* __restrict__ alpha, const int* __restrict__ act,
                         const double* __restrict__ P, const double* __restrict__ AP, double* __restrict__ X,
                         double* __restrict__ R) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(ni) * N;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(e % N);
        if (!act[c]) continue;
        const size_t k = size_t(e / N) * ld + c;
        X[k] = __dadd_rn(X[k], __dmul_rn(alpha[c], P[k]));
        R[k] = __dsub_rn(R[k], __dmul_rn(alpha[c], AP[k]));
    }
}

/// P[:, c] = Z[:, c] + beta_c P[:, c] (beta_c = 0: restart) for the columns with act_c; R = B - AX when mode 1
__global__ void k_sgs_p(int ni, int N, int ld, const double* __restrict__ beta, const int* __restrict__ act,
                        const double* __restrict__ Z, double* __restrict__ P) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(ni) * N;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(e % N);
        if (!act[c]) continue;
        const size_t k = size_t(e / N) * ld + c;
        P[k] = __dadd_rn(Z[k], __dmul_rn(beta[c], P[k]));
    }
}

__global__ void k_sgs_trueres(int ni, int N, int ld, const int* __restrict__ act, const double* __restrict__ B,
                              const double* __restrict__ AX, double* __restrict__ R) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(ni) * N;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(e % N);
        if (!act[c]) continue;
        const size_t k = size_t(e / N) * ld + c;
        R[k] = __dsub_rn(B[k], AX[k]);
    }
}

/// dependency levels of the forward (lower) and backward (upper) solves over the natural interior pattern
void build_plan(Level& L, SgsPlan& pl) {
    const auto& T = *L.topo;
    const int ni = L.ni;
    auto levels = [&](bool lower, std::vector<int32_t>& rows, std::vector<int>& bounds) {
        std::vector<int> lev(ni, 0);
        int maxl = 0;
        if (lower) {
            for (int i = 0; i < ni; ++i) {
                int l = 0;
                for (int q = T.ii.ptr[i]; q < T.ii.ptr[i + 1]; ++q)
                    if (T.ii.col[q] < i) l = std::max(l, lev[T.ii.col[q]] + 1);
                lev[i] = l;
                maxl = std::max(maxl, l);
            }
        } else {
            for (int i = ni - 1; i >= 0; --i) {
                int l = 0;
                for (int q = T.ii.ptr[i]; q < T.ii.ptr[i + 1]; ++q)
                    if (T.ii.col[q] > i) l = std::max(l, lev[T.ii.col[q]] + 1);
                lev[i] = l;
                maxl = std::max(maxl, l);
            }
        }
        bounds.assign(size_t(maxl) + 2, 0);
        for (int i = 0; i < ni; ++i) ++bounds[size_t(lev[i]) + 1];
        for (int l = 0; l <= maxl; ++l) bounds[size_t(l) + 1] += bounds[size_t(l)];
        rows.assign(size_t(ni), 0);
        std::vector<int> fill(bounds.begin(), bounds.end() - 1);
        for (int i = 0; i < ni; ++i) rows[size_t(fill[size_t(lev[i])]++)] = i;
    };
    std::vector<int32_t> fr, br;
    levels(true, fr, pl.f_bounds);
    levels(false, br, pl.b_bounds);
    pl.f_rows.upload(*L.ctx, fr);
    pl.b_rows.upload(*L.ctx, br);
    pl.ready = true;
}

}  // namespace

void sgs_apply(Level& L, SgsPlan& pl, const double* A, const double* Bv, const double* d_sigma, int N, int ld,
               const double* r, double* z, double* tmp) {
    Ctx& c = *L.ctx;
    if (!pl.ready) build_plan(L, pl);
    const int32_t* ptr = L.ii_ptr.p;
    const int32_t* col = L.ii_col.p;
    for (size_t l = 0; l + 1 < pl.f_bounds.size(); ++l) {
        const int b = pl.f_bounds[l], n = pl.f_bounds[l + 1] - b;
        launch(c, "sgs", k_sgs_level, grid_of(c, int64_t(n) * N), kT, 0, n, (const int32_t*)pl.f_rows.p + b, N, ld,
               ptr, col, A, Bv, d_sigma, r, tmp, 1);
    }
    launch(c, "sgs", k_sgs_scale, grid_of(c, int64_t(L.ni) * N), kT, 0, L.ni, N, ld, (const int32_t*)L.diag_slot.p, A,
           Bv, d_sigma, tmp);
    for (size_t l = 0; l + 1 < pl.b_bounds.size(); ++l) {
        const int b = pl.b_bounds[l], n = pl.b_bounds[l + 1] - b;
        launch(c, "sgs", k_sgs_level, grid_of(c, int64_t(n) * N), kT, 0, n, (const int32_t*)pl.b_rows.p + b, N, ld,
               ptr, col, A, Bv, d_sigma, (const double*)tmp, z, 0);
    }
}

void cg_solve_sgs(Ctx& c, Level& L, int mat, int shift_mat, const double* h_sigma, const double* d_B, double* d_X,
                  int N, int ld, const CgOptions& o, CgColumnStats* stats, CgWork& cw) {
    SgsWork& w = cw.sgs;
    SgsPlan& plan = L.sgs_plan;
    const bool shift = shift_mat >= 0;
    const double* A = L.mats[mat].ii.p;
    const double* Bv = shift ? L.mats[shift_mat].ii.p : nullptr;
    const int ni = L.ni;
    const int64_t vec = int64_t(ni) * ld;
    for (auto* b : {&w.R, &w.Z, &w.P, &w.AP, &w.T}) b->n < vec ? b->alloc(vec) : void();
    const int nb = std::max(1, std::min(c.sm_count * 2, ceil_div(ni, kT)));
    if (w.part.n < int64_t(nb) * N) w.part.alloc(int64_t(nb) * N);
    if (w.scal.n < 4 * int64_t(N)) w.scal.alloc(4 * int64_t(N));
    if (w.iact.n < N) w.iact.alloc(N);
    double* d_sigma = w.scal.p;
    double* d_coef = w.scal.p + N;
    double* d_dot = w.scal.p + 2 * N;
    std::vector<double> sig(N, 0.0);
    if (shift && h_sigma) std::copy(h_sigma, h_sigma + N, sig.begin());
    KSB_CUDA_CHECK(cudaMemcpyAsync(d_sigma, sig.data(), sizeof(double) * N, cudaMemcpyHostToDevice, c.stream));
    auto dots = [&](const double* X, const double* Y) {
        launch(c, "sgs", k_coldot, nb, kT, sizeof(double) * kT, ni, N, ld, X, Y, w.part.p);
        launch(c, "sgs", k_fold_cols, 1, 128, 0, nb, N, (const double*)w.part.p, d_dot);
        std::vector<double> h(N);
        KSB_CUDA_CHECK(cudaMemcpyAsync(h.data(), d_dot, sizeof(double) * N, cudaMemcpyDeviceToHost, c.stream));
        KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
        return h;
    };
    auto spmm_op = [&](const double* X, double* Y) { spmm(c, L, A, Bv, shift ? d_sigma : nullptr, X, N, ld, Y, ld); };
    auto set_act = [&](const std::vector<int>& act) {
        KSB_CUDA_CHECK(cudaMemcpyAsync(w.iact.p, act.data(), sizeof(int) * N, cudaMemcpyHostToDevice, c.stream));
    };
    auto set_coef = [&](const std::vector<double>& a) {
        KSB_CUDA_CHECK(cudaMemcpyAsync(d_coef, a.data(), sizeof(double) * N, cudaMemcpyHostToDevice, c.stream));
    };
    const int g = grid_of(c, vec);
    // x = 0, r = b, z = M^-1 r, p = z
    KSB_CUDA_CHECK(cudaMemsetAsync(d_X, 0, sizeof(double) * vec, c.stream));
    KSB_CUDA_CHECK(cudaMemcpyAsync(w.R.p, d_B, sizeof(double) * vec, cudaMemcpyDeviceToDevice, c.stream));
    const std::vector<double> bb = dots(d_B, d_B);
    std::vector<double> bnorm(N), rz(N), rel(N, 0.0);
    std::vector<int> act(N), it(N, 0), conv(N, 0), brk(N, 0);
    for (int j = 0; j < N; ++j) {
        bnorm[j] = std::sqrt(bb[j]);
        act[j] = bnorm[j] != 0.0;
        rel[j] = act[j] ? 1.0 : 0.0;  // r = b
        conv[j] = !act[j];  // zero right-hand side: converged with 0 iterations (solver.cpp:62-66)
    }
    sgs_apply(L, plan, A, Bv, d_sigma, N, ld, w.R.p, w.Z.p, w.T.p);
    KSB_CUDA_CHECK(cudaMemcpyAsync(w.P.p, w.Z.p, sizeof(double) * vec, cudaMemcpyDeviceToDevice, c.stream));
    rz = dots(w.R.p, w.Z.p);
    std::vector<double> coef(N);
    for (int k = 0; k < o.max_iterations; ++k) {
        if (std::none_of(act.begin(), act.end(), [](int a) { return a != 0; })) break;
        spmm_op(w.P.p, w.AP.p);
        const std::vector<double> pAp = dots(w.P.p, w.AP.p);
        for (int j = 0; j < N; ++j) {
            coef[j] = 0.0;
            if (!act[j]) continue;
            if (!(pAp[j] > 0.0)) {  // breakdown (solver.cpp:74-79): residual of the current r
                act[j] = 0;
                brk[j] = 1;
                it[j] = k;
                continue;
            }
            coef[j] = rz[j] / pAp[j];
        }
        const std::vector<int> upd = act;
        set_act(upd);
        set_coef(coef);
        launch(c, "sgs", k_sgs_xr, g, kT, 0, ni, N, ld, (const double*)d_coef, (const int*)w.iact.p,
               (const double*)w.P.p, (const double*)w.AP.p, d_X, w.R.p);
        const std::vector<double> rr = dots(w.R.p, w.R.p);
        std::vector<int> check(N, 0);
        bool any_check = false;
        for (int j = 0; j < N; ++j) {
            if (!upd[j]) continue;
            rel[j] = std::sqrt(rr[j]) / bnorm[j];
            it[j] = k + 1;
            if (rel[j] <= o.tol) {
                check[j] = 1;
                any_check = true;
            }
        }
        std::vector<int> restart(N, 0);
        if (any_check) {  // true residual b - A x (solver.cpp:84-101)
            set_act(check);
            spmm_op(d_X, w.AP.p);
            launch(c, "sgs", k_sgs_trueres, g, kT, 0, ni, N, ld, (const int*)w.iact.p, d_B, (const double*)w.AP.p,
                   w.R.p);
            const std::vector<double> tr = dots(w.R.p, w.R.p);
            for (int j = 0; j < N; ++j) {
                if (!check[j]) continue;
                rel[j] = std::sqrt(tr[j]) / bnorm[j];
                if (rel[j] <= o.tol) {
                    conv[j] = 1;
                    act[j] = 0;
                } else {
                    restart[j] = 1;
                }
            }
        }
        // z = M^-1 r for the live columns; p = z + beta p (restart: p = z)
        if (std::none_of(act.begin(), act.end(), [](int a) { return a != 0; })) break;
        sgs_apply(L, plan, A, Bv, d_sigma, N, ld, w.R.p, w.Z.p, w.T.p);
        const std::vector<double> rzn = dots(w.R.p, w.Z.p);
        for (int j = 0; j < N; ++j) {
            coef[j] = 0.0;
            if (!act[j]) continue;
            if (!restart[j]) coef[j] = rzn[j] / rz[j];
            rz[j] = rzn[j];
        }
        set_act(act);
        set_coef(coef);
        launch(c, "sgs", k_sgs_p, g, kT, 0, ni, N, ld, (const double*)d_coef, (const int*)w.iact.p,
               (const double*)w.Z.p, w.P.p);
    }
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    if (stats)
        for (int j = 0; j < N; ++j) {
            stats[j].iterations = it[j];
            stats[j].relative_residual = rel[j];
            stats[j].converged = conv[j];
            stats[j].breakdown = brk[j];
        }
}

}  // namespace ksb
