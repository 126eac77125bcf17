// One outer iteration of solve_level_corrected on the device.
//
// Reference loop body: proj/src/driver.cpp:106-150, with
//   OuterOperator + shift ladder   proj/src/correction.cpp:15-61   (multi-RHS CG, cg.cu)
//   bvp_hartree                    proj/src/correction.cpp:67-75   (physics.cu + CG on S)
//   prepare_blocks                 proj/src/correction.cpp:113-212 (project.cu)
//   inner_scf                      proj/src/correction.cpp:279-368 (inner.cu)
//   expand                         proj/src/correction.cpp:370-381
//   density_change (H1)            proj/src/driver.cpp:56-60
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "correction.cuh"

namespace ksb {

void elem_potential(Level& L, const Potential& pot, double* E);
void axpby_values(Level& L, int dst, double a, int x, double b, int y);

namespace {

constexpr int kT = 256;
constexpr double kFourPi = 4.0 * 3.14159265358979323846;

int grid_of(const Ctx& c, int64_t work) {
    return int(std::max<int64_t>(1, std::min<int64_t>((work + kT - 1) / kT, int64_t(c.sm_count) * 8)));
}

__global__ void k_add(int64_t n, const double* __restrict__ a, double sa, const double* __restrict__ b, double sb,
                      double* __restrict__ y) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        y[i] = sa * a[i] + sb * b[i];
}

/// grid-wide min over the interior diagonal: per-block minima into part[1 + b], the last block to finish folds
/// them into out[0] (min is exact, so the result does not depend on the order)
__global__ void k_min_diag(int ni, const int32_t* __restrict__ dslot, const double* __restrict__ vals,
                           double* __restrict__ part, int* __restrict__ ticket, double* __restrict__ out) {
    __shared__ double red[32];
    __shared__ bool last;
    double m = INFINITY;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ni; r += gridDim.x * blockDim.x)
        m = fmin(m, __ldg(vals + __ldg(dslot + r)));
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = INFINITY;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t = fmin(t, red[w]);
        part[blockIdx.x] = t;
        __threadfence();
        last = atomicAdd(ticket, 1) == int(gridDim.x) - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double t = INFINITY;
    for (int b = threadIdx.x; b < int(gridDim.x); b += blockDim.x) t = fmin(t, __ldcg(part + b));
    for (int o = 16; o > 0; o >>= 1) t = fmin(t, __shfl_xor_sync(0xffffffffu, t, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double u = INFINITY;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) u = fmin(u, red[w]);
        out[0] = ni > 0 ? u : 0.0;
        *ticket = 0;
    }
}

/// B[r, j] = scale_j * R[r, col_j]  (gather of a column subset, per-column scale)
__global__ void k_gather_cols(int ni, int nc, const int* __restrict__ cols, const double* __restrict__ scale,
                              const double* __restrict__ R, int ldr, double* __restrict__ B, int ldb) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(ni) * nc;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int r = int(e / nc), j = int(e % nc);
        B[size_t(r) * ldb + j] = (scale ? scale[j] : 1.0) * R[size_t(r) * ldr + cols[j]];
    }
}

/// B[r, j] *= scale[j], j < nc
__global__ void k_scale_cols(int ni, int nc, const double* __restrict__ scale, double* __restrict__ B, int ldb) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(ni) * nc;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int r = int(e / nc), j = int(e % nc);
        B[size_t(r) * ldb + j] *= scale[j];
    }
}

/// X[r, col_j] = Xc[r, j] for the columns with take_j != 0
__global__ void k_scatter_cols(int ni, int nc, const int* __restrict__ cols, const int* __restrict__ take,
                               const double* __restrict__ Xc, int ldc, double* __restrict__ X, int ldx) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(ni) * nc;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int r = int(e / nc), j = int(e % nc);
        if (take[j]) X[size_t(r) * ldx + cols[j]] = Xc[size_t(r) * ldc + j];
    }
}

/// full-length vector from interior values + boundary values
__global__ void k_full_from(int ni, int nb, const int32_t* __restrict__ interior, const int32_t* __restrict__ boundary,
                            const double* __restrict__ vint, const double* __restrict__ vb, double* __restrict__ full) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(ni) + nb;
         e += int64_t(gridDim.x) * blockDim.x) {
        if (e < ni)
            full[interior[e]] = vint ? vint[e] : 0.0;
        else
            full[boundary[e - ni]] = vb ? vb[e - ni] : 0.0;
    }
}

/// Phi[r, i] = sum_k P_int(r,k) phiH[i][col_k] + theta2_i PhiT[r, i]
/// w[interior r] = (0 + sum_k P_int(r,k) wH[col_k]) + theta1 wt[interior r]; w[boundary] = bc
__global__ void k_expand(int ni, int N, int nh, const int32_t* __restrict__ pcol, const double* __restrict__ pval,
                         const double* __restrict__ phiH, const double* __restrict__ th2, const double* __restrict__ PhiT,
                         int ldT, double* __restrict__ Phi, int ld, const double* __restrict__ wH,
                         const double* __restrict__ th1, const double* __restrict__ wt_full,
                         const int32_t* __restrict__ interior, double* __restrict__ w_full) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ni; r += gridDim.x * blockDim.x) {
        int pc[4];
        double pv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            pc[k] = pcol[4 * size_t(r) + k];
            pv[k] = pval[4 * size_t(r) + k];
        }
        for (int i = 0; i < N; ++i) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (pc[k] >= 0) s += pv[k] * phiH[size_t(i) * nh + pc[k]];
            Phi[size_t(r) * ld + i] = s + th2[i] * PhiT[size_t(r) * ldT + i];
        }
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (pc[k] >= 0) s += pv[k] * wH[pc[k]];
        const int v = interior[r];
        w_full[v] = (0.0 + s) + th1[0] * wt_full[v];
    }
}

struct Timer {
    cudaEvent_t e[8];
    int n = 0;
    cudaStream_t s;
    explicit Timer(cudaStream_t st) : s(st) {
        for (auto& x : e) KSB_CUDA_CHECK(cudaEventCreate(&x));
    }
    ~Timer() {
        for (auto& x : e) cudaEventDestroy(x);
    }
    void mark() { KSB_CUDA_CHECK(cudaEventRecord(e[n++], s)); }
    double ms(int a, int b) {
        float t = 0;
        KSB_CUDA_CHECK(cudaEventElapsedTime(&t, e[a], e[b]));
        return t;
    }
};

void need(DevBuf<double>& b, int64_t n) {
    if (b.n < n) b.alloc(std::max<int64_t>(1, n));
}

}  // namespace

// make_level_ops (proj/src/driver.cpp:35-47): S, M, a_op = 1/2 S + M_ext, the per-tet M_ext elements and the
// coarse interior blocks M_H, C_H with their Cholesky factors.
void level_ops(Level& L, Corrector& K) {
    if (!K.sys.set) raise(KSB_INVALID_ARGUMENT, "system not set on this level");
    Potential pot;
    pot.kind = 0;
    pot.n = int(K.sys.atoms.size() / 4);
    pot.params = K.sys.atoms;
    assemble_into(L, 0, 1.0, 0.0, nullptr, 0.0, nullptr, 0.0);  // S
    assemble_into(L, 1, 0.0, 1.0, nullptr, 0.0, nullptr, 0.0);  // M
    assemble_into(L, 2, 0.5, 0.0, pot.n ? &pot : nullptr, 1.0, nullptr, 0.0);  // a_op
    need(K.eext, int64_t(L.nt) * 16);
    if (pot.n)
        elem_potential(L, pot, K.eext.p);
    else
        KSB_CUDA_CHECK(cudaMemsetAsync(K.eext.p, 0, sizeof(double) * L.nt * 16, L.ctx->stream));
    coarse_level_setup(L, K.coarse);
    K.ops_ready = true;
}

double min_diagonal(Level& L, int mat, DevBuf<double>& scratch) {
    Ctx& c = *L.ctx;
    if (!L.mats[mat].valid) raise(KSB_INVALID_ARGUMENT, "operator not assembled");
    const int g = std::max(1, std::min(ceil_div(L.ni, 256), 2 * c.sm_count));
    need(scratch, 2 + g);
    // the ticket lives in the scratch block's last slot (zeroed here, reset by the folding block)
    int* ticket = reinterpret_cast<int*>(scratch.p + 1 + g);
    KSB_CUDA_CHECK(cudaMemsetAsync(ticket, 0, sizeof(int), c.stream));
    launch(c, "elementwise", k_min_diag, g, 256, 0, L.ni, (const int32_t*)L.diag_slot.p,
           (const double*)L.mats[mat].ii.p, scratch.p + 1, ticket, scratch.p);
    double md = 0.0;
    KSB_CUDA_CHECK(cudaMemcpyAsync(&md, scratch.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    return md;
}

double outer_operator(Level& L, Corrector& K, const double* d_what_full, const double* d_vxc_full, int aop) {
    Ctx& c = *L.ctx;
    if (!L.mats[aop].valid) raise(KSB_INVALID_ARGUMENT, "a_op not assembled");
    need(K.pot, L.n);
    launch(c, "elementwise", k_add, grid_of(c, L.n), kT, 0, int64_t(L.n), d_what_full, 1.0, d_vxc_full, 1.0, K.pot.p);
    assemble_into(L, MAT_TMP, 0.0, 0.0, nullptr, 0.0, K.pot.p, 1.0);
    axpby_values(L, MAT_H, 1.0, aop, 1.0, MAT_TMP);
    K.min_diag = min_diagonal(L, MAT_H, K.diff);
    return K.min_diag;
}

/// gather the interior entries of a full-length vector
__global__ void k_take_interior(int ni, const int32_t* __restrict__ interior, const double* __restrict__ full,
                                double* __restrict__ out) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ni; r += gridDim.x * blockDim.x) out[r] = full[interior[r]];
}
__global__ void k_take_boundary(int nb, const int32_t* __restrict__ boundary, const double* __restrict__ full,
                                double* __restrict__ out) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nb; r += gridDim.x * blockDim.x) out[r] = full[boundary[r]];
}

// EllipticSolver::solve / solve_zero_bc (proj/src/solver.cpp:113-135)
CgColumnStats elliptic_solve(Level& L, CgWork& cg, DevBuf<double>& scratch, int mat, const double* d_b_full,
                             const double* d_bc_full, const CgOptions& o, double* d_x_full) {
    Ctx& c = *L.ctx;
    if (!L.mats[mat].valid) raise(KSB_INVALID_ARGUMENT, "operator not assembled");
    const int ni = L.ni, nb = L.nb;
    need(scratch, 2 * int64_t(ni) + std::max(1, nb));
    double* rhs = scratch.p;
    double* xi = scratch.p + ni;
    double* bcb = scratch.p + 2 * int64_t(ni);
    launch(c, "elementwise", k_take_interior, grid_of(c, ni), kT, 0, ni, (const int32_t*)L.interior.p, d_b_full, rhs);
    if (d_bc_full) {
        launch(c, "elementwise", k_take_boundary, grid_of(c, std::max(1, nb)), kT, 0, nb, (const int32_t*)L.boundary.p,
               d_bc_full, bcb);
        lift(L, mat, bcb, rhs);
    }
    CgColumnStats st;
    cg_solve(c, L, mat, -1, nullptr, rhs, xi, 1, 1, o, &st, cg);
    launch(c, "elementwise", k_full_from, grid_of(c, L.n), kT, 0, ni, nb, (const int32_t*)L.interior.p,
           (const int32_t*)L.boundary.p, (const double*)xi, d_bc_full ? (const double*)bcb : nullptr, d_x_full);
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    return st;
}

// OuterOperator::solve_orbital for all orbitals at once (proj/src/correction.cpp:26-61)
void solve_orbitals(Level& L, Corrector& K, CgWork& cg, const StepOptions& o, const double* h_lambda,
                    const double* d_Phi, int ld, double* d_PhiT, int ldT, StepLog* log, int n_cols) {
    Ctx& c = *L.ctx;
    const int N = n_cols > 0 ? n_cols : K.sys.N, ni = L.ni;
    // one block-sized buffer: R0 = M phi (orbitals vanish on the boundary), scaled in place by lambda into the
    // right-hand sides; the level-shift attempts recompute M phi for their (few) columns
    need(K.R0, int64_t(ni) * ld);
    spmm(c, L, L.mats[1].ii.p, nullptr, nullptr, d_Phi, N, ld, K.R0.p, ld);
    if (K.idx.n < 4 * N + 8) K.idx.alloc(4 * N + 8);
    need(K.colscale, N);
    double* sc = K.colscale.p;
    std::vector<int> cols(N);
    for (int i = 0; i < N; ++i) cols[i] = i;
    KSB_CUDA_CHECK(cudaMemcpyAsync(K.idx.p, cols.data(), sizeof(int) * N, cudaMemcpyHostToDevice, c.stream));
    KSB_CUDA_CHECK(cudaMemcpyAsync(sc, h_lambda, sizeof(double) * N, cudaMemcpyHostToDevice, c.stream));
    launch(c, "elementwise", k_scale_cols, grid_of(c, int64_t(ni) * N), kT, 0, ni, N, (const double*)sc, K.R0.p, ld);
    CgOptions co;
    co.tol = o.tol_linear;
    co.check_every = o.check_every;
    co.precond = o.precond;
    if (ldT != ld) raise(KSB_INVALID_ARGUMENT, "solve_orbitals: ld mismatch");
    // An odd block is solved with its pad column as one more right-hand side that is identically zero (converged
    // at iteration 0, proj/src/solver.cpp:62-66): the columns are independent, and the even block takes the CG's
    // paired 16-byte update passes (configs[3], N = 21: update_r 4.5 -> ~6 TB/s)
    const int Ncg = (N > 1 && (N & 1) && ld > N && N < 128) ? N + 1 : N;
    if (Ncg > N)
        KSB_CUDA_CHECK(cudaMemset2DAsync(K.R0.p + N, sizeof(double) * ld, 0, sizeof(double), ni, c.stream));
    std::vector<CgColumnStats> st(Ncg);
    cg_solve(c, L, MAT_H, -1, nullptr, K.R0.p, d_PhiT, Ncg, ld, co, st.data(), cg);
    std::vector<int> attempt(N, -1), iters(N);
    std::vector<int> fail;
    for (int i = 0; i < N; ++i) {
        iters[i] = st[i].iterations;
        if (!st[i].converged) fail.push_back(i);
    }
    const double base = std::abs(K.min_diag);
    double last_rel = 0.0;
    for (int k = 0; k < 4 && !fail.empty(); ++k) {
        const double sigma = k == 0 ? base : std::pow(4.0, k) * (base + 1.0);
        const int nf = int(fail.size());
        const int ldc = nf == 1 ? 1 : nf + (nf & 1);
        need(K.Bc, int64_t(ni) * ldc);
        need(K.Xc, int64_t(ni) * ldc);
        std::vector<double> scale(nf), sig(nf, sigma);
        for (int j = 0; j < nf; ++j) scale[j] = h_lambda[fail[j]] + sigma;
        double* dsc = K.colscale.p;  // the unshifted solve's scales are consumed (stream order)
        KSB_CUDA_CHECK(cudaMemcpyAsync(K.idx.p, fail.data(), sizeof(int) * nf, cudaMemcpyHostToDevice, c.stream));
        KSB_CUDA_CHECK(cudaMemcpyAsync(dsc, scale.data(), sizeof(double) * nf, cudaMemcpyHostToDevice, c.stream));
        if (ldc > nf) KSB_CUDA_CHECK(cudaMemsetAsync(K.Bc.p, 0, sizeof(double) * ni * ldc, c.stream));
        launch(c, "elementwise", k_gather_cols, grid_of(c, int64_t(ni) * nf), kT, 0, ni, nf, (const int*)K.idx.p,
               (const double*)nullptr, d_Phi, ld, K.Xc.p, ldc);
        spmm(c, L, L.mats[1].ii.p, nullptr, nullptr, K.Xc.p, nf, ldc, K.Bc.p, ldc);  // (lambda + sigma) M phi
        launch(c, "elementwise", k_scale_cols, grid_of(c, int64_t(ni) * nf), kT, 0, ni, nf, (const double*)dsc, K.Bc.p,
               ldc);
        const int nfc = nf > 1 ? ldc : nf;  // odd count: the zeroed pad column rides along (see above)
        sig.resize(nfc, sigma);
        std::vector<CgColumnStats> sst(nfc);
        cg_solve(c, L, MAT_H, 1, sig.data(), K.Bc.p, K.Xc.p, nfc, ldc, co, sst.data(), cg);
        std::vector<int> take(nf), still;
        for (int j = 0; j < nf; ++j) {
            iters[fail[j]] += sst[j].iterations;
            take[j] = sst[j].converged;
            if (j == 0) last_rel = sst[j].relative_residual;
            if (sst[j].converged)
                attempt[fail[j]] = k;
            else
                still.push_back(fail[j]);
        }
        KSB_CUDA_CHECK(cudaMemcpyAsync(K.idx.p + N + 4, take.data(), sizeof(int) * nf, cudaMemcpyHostToDevice, c.stream));
        launch(c, "elementwise", k_scatter_cols, grid_of(c, int64_t(ni) * nf), kT, 0, ni, nf, (const int*)K.idx.p,
               (const int*)(K.idx.p + N + 4), (const double*)K.Xc.p, ldc, d_PhiT, ldT);
        KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
        fail.swap(still);
    }
    if (!fail.empty())
        raise(KSB_NONCONVERGENCE, "orbital correction solve failed even after the level shift (residual " +
                                      std::to_string(last_rel) + ")");
    if (log) {
        log->attempts = attempt;
        log->iterations = iters;
        log->cg_iterations = 0;
        for (int x : iters) log->cg_iterations += x;
    }
}

/// S x = rhs on the interior (single column): multigrid-preconditioned CG on levels above the coarse mesh,
/// Jacobi CG otherwise or when KSB_STIFF_MG=0; a multigrid solve that breaks down or stalls is redone with
/// Jacobi CG. Same PCG contract either way (proj/src/solver.cpp:57-111).
CgColumnStats stiffness_solve(Level& L, Corrector& K, CgWork& cg, const double* rhs, double* x, double tol) {
    static const char* env = std::getenv("KSB_STIFF_MG");
    const bool use_mg = K.precond == 0 && L.meshes.size() >= 2 && !(env && env[0] == '0') && K.coarse.CHi.n > 0;
    if (use_mg) {
        if (!K.mg.ready) mg_setup(L, K.mg, K.coarse.CHi.p);
        const CgColumnStats st = mg_pcg(L, K.mg, rhs, x, tol, 20000);
        if (st.converged) return st;
    }
    CgOptions co;
    co.tol = tol;
    co.precond = K.precond;  // SGS parity runs: the reference's SGS-PCG on S (hartree.cpp:131-144)
    CgColumnStats st;
    cg_solve(*L.ctx, L, 0, -1, nullptr, rhs, x, 1, 1, co, &st, cg);
    return st;
}

// bvp_hartree -> solve_hartree_exact (proj/src/hartree.cpp:131-144): w with Dirichlet data bcb
int hartree_solve(Level& L, Corrector& K, CgWork& cg, const double* d_PhiT, int N, int ldT, const double* d_bcb,
                  double tol, double* d_w_full) {
    Ctx& c = *L.ctx;
    need(K.hrhs, L.ni);
    need(K.wtil_int, L.ni);
    sqload(L, d_PhiT, N, ldT, K.sys.occ, kFourPi, K.hrhs.p, K.phys);
    lift(L, 0, d_bcb, K.hrhs.p);
    const CgColumnStats st = stiffness_solve(L, K, cg, K.hrhs.p, K.wtil_int.p, tol);
    if (!st.converged)
        raise(KSB_NONCONVERGENCE, "hartree solve stalled at residual " + std::to_string(st.relative_residual));
    launch(c, "elementwise", k_full_from, grid_of(c, L.n), kT, 0, L.ni, L.nb, (const int32_t*)L.interior.p,
           (const int32_t*)L.boundary.p, (const double*)K.wtil_int.p, d_bcb, d_w_full);
    return st.iterations;
}

/// out[c * N + i] = in[i * nh + c]: the coarse orbital coefficients with the orbital index fastest
__global__ void k_transpose_cols(int N, int nh, const double* __restrict__ in, double* __restrict__ out) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(N) * nh; e += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(e / N), i = int(e % N);
        out[e] = in[size_t(i) * nh + c];
    }
}

/// k_expand for many orbitals: threads run over the orbitals of a row (coalesced Phi / PhiT rows; the coarse
/// coefficients come from the transposed copy, N contiguous doubles per coarse dof), the same sums in the same order.
/// N = 120 at 2.05 M rows: 3.96 -> see profiles/README.md.
__global__ void k_expand_wide(int ni, int N, const int32_t* __restrict__ pcol, const double* __restrict__ pval,
                              const double* __restrict__ phiHT, const double* __restrict__ th2,
                              const double* __restrict__ PhiT, int ldT, double* __restrict__ Phi, int ld,
                              const double* __restrict__ wH, const double* __restrict__ th1,
                              const double* __restrict__ wt_full, const int32_t* __restrict__ interior,
                              double* __restrict__ w_full) {
    const int rb = blockDim.x / N, i = threadIdx.x % N, rl = threadIdx.x / N;
    if (rl >= rb) return;
    const double t2 = th2[i];
    for (int r = blockIdx.x * rb + rl; r < ni; r += gridDim.x * rb) {
        int pc[4];
        double pv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            pc[k] = __ldg(pcol + 4 * size_t(r) + k);
            pv[k] = __ldg(pval + 4 * size_t(r) + k);
        }
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (pc[k] >= 0) s += pv[k] * __ldg(phiHT + size_t(pc[k]) * N + i);
        Phi[size_t(r) * ld + i] = s + t2 * PhiT[size_t(r) * ldT + i];
        if (i == 0) {
            double sw = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (pc[k] >= 0) sw += pv[k] * wH[pc[k]];
            const int v = interior[r];
            w_full[v] = (0.0 + sw) + th1[0] * wt_full[v];
        }
    }
}

void expand(Level& L, Corrector& K, const double* d_PhiT, int ldT, const double* d_wt_full, const double* d_bcb,
            double* d_Phi, int ld, double* d_w_full) {
    Ctx& c = *L.ctx;
    InnerWork& w = K.inner;
    const int cur = w.cur;
    // boundary entries of w first (ell), interior entries from the kernel
    launch(c, "elementwise", k_full_from, grid_of(c, L.n), kT, 0, 0, L.nb, (const int32_t*)L.interior.p,
           (const int32_t*)L.boundary.p, (const double*)nullptr, d_bcb, d_w_full);
    if (K.sys.N >= 8 && K.sys.N <= kT) {
        const int N = K.sys.N;
        need(K.phiHT, int64_t(N) * L.nH);
        launch(c, "expand", k_transpose_cols, grid_of(c, int64_t(N) * L.nH), kT, 0, N, L.nH,
               (const double*)w.phi[cur].p, K.phiHT.p);
        const int rb = kT / N;
        const int grid = int(std::max<int64_t>(1, std::min<int64_t>((int64_t(L.ni) + rb - 1) / rb, int64_t(c.sm_count) * 8)));
        launch(c, "expand", k_expand_wide, grid, kT, 0, L.ni, N, (const int32_t*)L.pint_col.p,
               (const double*)L.pint_val.p, (const double*)K.phiHT.p, (const double*)w.th2[cur].p, d_PhiT, ldT, d_Phi,
               ld, (const double*)w.wH[cur].p, (const double*)w.th1[cur].p, d_wt_full, (const int32_t*)L.interior.p,
               d_w_full);
        return;
    }
    launch(c, "expand", k_expand, grid_of(c, L.ni), kT, 0, L.ni, K.sys.N, L.nH, (const int32_t*)L.pint_col.p,
           (const double*)L.pint_val.p, (const double*)w.phi[cur].p, (const double*)w.th2[cur].p, d_PhiT, ldT, d_Phi,
           ld, (const double*)w.wH[cur].p, (const double*)w.th1[cur].p, d_wt_full, (const int32_t*)L.interior.p,
           d_w_full);
}

void correction_step(Level& L, Corrector& K, CgWork& cg, const StepOptions& o, double* h_lambda, double* d_Phi, int ld,
                     double* d_w, StepLog* log) {
    Ctx& c = *L.ctx;
    K.precond = o.precond;
    if (!K.ops_ready) level_ops(L, K);
    K.mlc_ld = 0;  // the step reuses the standard-MLC work buffers: a pending MLC level must be restarted
    const int N = K.sys.N, n = L.n, ni = L.ni;
    Timer tm(c.stream);
    tm.mark();
    need(K.rho, n);
    need(K.vxc, n);
    need(K.what_full, n);
    need(K.bcb, std::max(1, L.nb));
    need(K.wt_full, n);
    need(K.ell_full, n);
    need(K.rho_t, n);
    need(K.diff, n);
    need(K.PhiT, int64_t(ni) * ld);
    // density and xc of the current orbitals
    rho_vxc(L, d_Phi, N, ld, K.sys.occ, K.sys.xc, K.rho.p, K.sys.xc_on ? K.vxc.p : nullptr);
    if (!K.sys.xc_on) KSB_CUDA_CHECK(cudaMemsetAsync(K.vxc.p, 0, sizeof(double) * n, c.stream));
    if (K.sys.hartree_on)
        KSB_CUDA_CHECK(cudaMemcpyAsync(K.what_full.p, d_w, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
    else
        KSB_CUDA_CHECK(cudaMemsetAsync(K.what_full.p, 0, sizeof(double) * n, c.stream));
    outer_operator(L, K, K.what_full.p, K.vxc.p);
    StepLog lg;
    solve_orbitals(L, K, cg, o, h_lambda, d_Phi, ld, K.PhiT.p, ld, &lg);
    tm.mark();
    KSB_CUDA_CHECK(cudaMemsetAsync(K.bcb.p, 0, sizeof(double) * std::max(1, L.nb), c.stream));
    if (K.sys.hartree_on) {
        rho_vxc(L, K.PhiT.p, N, ld, K.sys.occ, K.sys.xc, K.rho_t.p, nullptr);
        const double ctr[3] = {0.5 * (L.box_lo[0] + L.box_hi[0]), 0.5 * (L.box_lo[1] + L.box_hi[1]),
                               0.5 * (L.box_lo[2] + L.box_hi[2])};
        const Moments m = moments(L, K.rho_t.p, K.phys, ctr);
        boundary_values(L, m, K.bcb.p);
        lg.hartree_iterations = hartree_solve(L, K, cg, K.PhiT.p, N, ld, K.bcb.p, o.tol_linear, K.diff.p);
        // w_tilde0 = w_tilde - ell: interior values, zero trace
        launch(c, "elementwise", k_full_from, grid_of(c, n), kT, 0, ni, L.nb, (const int32_t*)L.interior.p,
               (const int32_t*)L.boundary.p, (const double*)K.wtil_int.p, (const double*)nullptr, K.wt_full.p);
        launch(c, "elementwise", k_full_from, grid_of(c, n), kT, 0, ni, L.nb, (const int32_t*)L.interior.p,
               (const int32_t*)L.boundary.p, (const double*)nullptr, (const double*)K.bcb.p, K.ell_full.p);
    } else {
        KSB_CUDA_CHECK(cudaMemsetAsync(K.wt_full.p, 0, sizeof(double) * n, c.stream));
        KSB_CUDA_CHECK(cudaMemsetAsync(K.ell_full.p, 0, sizeof(double) * n, c.stream));
    }
    tm.mark();
    project_blocks(L, K.PhiT.p, N, ld, K.wt_full.p, K.ell_full.p, K.vxc.p, K.eext.p, K.proj);
    tm.mark();
    InnerParams ip;
    ip.tol = o.tol_inner;
    ip.max_iterations = o.max_inner;
    ip.score_floor = o.score_floor;
    ip.nev_pad = o.nev_pad;
    ip.hartree = K.sys.hartree_on;
    ip.occ = K.sys.occ;
    ip.fixed_sweeps = o.fixed_sweeps;
    const InnerStats ist = inner_scf(L, K.coarse, K.proj, ip, h_lambda, K.inner, true);
    lg.inner_iterations = ist.iterations;
    lg.inner_history = ist.history;
    tm.mark();
    expand(L, K, K.PhiT.p, ld, K.wt_full.p, K.bcb.p, d_Phi, ld, d_w);
    rho_vxc(L, d_Phi, N, ld, K.sys.occ, K.sys.xc, K.rho_t.p, nullptr);
    launch(c, "elementwise", k_add, grid_of(c, n), kT, 0, int64_t(n), (const double*)K.rho_t.p, 1.0,
           (const double*)K.rho.p, -1.0, K.diff.p);
    // density_change (driver.cpp:56-60): H1, or L1 with RunConfig::outer_norm_l1
    if (o.norm_l1) {
        lg.delta = l1_norm(L, K.diff.p, K.phys);
    } else {
        const auto nn = norms_sq(L, K.diff.p, K.phys);
        const double l2 = std::sqrt(std::max(0.0, nn[0])), semi = std::sqrt(std::max(0.0, nn[1]));
        lg.delta = std::sqrt(l2 * l2 + semi * semi);
    }
    KSB_CUDA_CHECK(cudaMemcpyAsync(h_lambda, K.inner.lamv[K.inner.cur].p, sizeof(double) * N, cudaMemcpyDeviceToHost,
                                   c.stream));
    tm.mark();
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    lg.ms_bvp = tm.ms(0, 1);
    lg.ms_hartree = tm.ms(1, 2);
    lg.ms_project = tm.ms(2, 3);
    lg.ms_inner = tm.ms(3, 4);
    lg.ms_total = tm.ms(0, 5);
    if (log) *log = lg;
}

namespace {
/// hartree::solve_hartree_cached (proj/src/hartree.cpp:95-106): S w = 4 pi M rho with Dirichlet data bcb. rho is a
/// density of zero-trace orbitals, so M rho restricted to interior rows is M_ii rho_int.
void hartree_of_density(Level& L, Corrector& K, CgWork& cg, const double* d_rho, const double* d_bcb, double tol,
                        double* d_w_full) {
    Ctx& c = *L.ctx;
    const int ni = L.ni;
    need(K.hrhs, ni);
    need(K.wtil_int, ni);
    need(K.pot, ni);
    launch(c, "elementwise", k_take_interior, grid_of(c, ni), kT, 0, ni, (const int32_t*)L.interior.p, d_rho, K.pot.p);
    spmm(c, L, L.mats[1].ii.p, nullptr, nullptr, K.pot.p, 1, 1, K.hrhs.p, 1);
    launch(c, "elementwise", k_add, grid_of(c, ni), kT, 0, int64_t(ni), (const double*)K.hrhs.p, kFourPi,
           (const double*)K.hrhs.p, 0.0, K.hrhs.p);
    lift(L, 0, d_bcb, K.hrhs.p);
    const CgColumnStats cs = stiffness_solve(L, K, cg, K.hrhs.p, K.wtil_int.p, tol);
    if (!cs.converged)
        raise(KSB_NONCONVERGENCE, "hartree solve stalled at residual " + std::to_string(cs.relative_residual));
    launch(c, "elementwise", k_full_from, grid_of(c, L.n), kT, 0, ni, L.nb, (const int32_t*)L.interior.p,
           (const int32_t*)L.boundary.p, (const double*)K.wtil_int.p, d_bcb, d_w_full);
}
}  // namespace

void mlc_begin(Level& L, Corrector& K, CgWork& cg, const StepOptions& o, const double* h_lambda, const double* d_Phi,
               int ld, const double* d_w, StepLog* log) {
    Ctx& c = *L.ctx;
    K.precond = o.precond;
    if (!K.ops_ready) level_ops(L, K);
    const int N = K.sys.N, n = L.n, ni = L.ni;
    for (auto* b : {&K.rho, &K.vxc, &K.what_full, &K.wt_full, &K.ell_full, &K.rho_t, &K.diff, &K.potf, &K.wscr})
        need(*b, n);
    need(K.bcb, std::max(1, L.nb));
    need(K.PhiT, int64_t(ni) * ld);
    // OuterOperator with the warm start's Hartree potential and v_xc(rho_prev) (driver.cpp:208-213)
    rho_vxc(L, d_Phi, N, ld, K.sys.occ, K.sys.xc, K.rho.p, K.sys.xc_on ? K.vxc.p : nullptr);
    if (!K.sys.xc_on) KSB_CUDA_CHECK(cudaMemsetAsync(K.vxc.p, 0, sizeof(double) * n, c.stream));
    if (K.sys.hartree_on)
        KSB_CUDA_CHECK(cudaMemcpyAsync(K.what_full.p, d_w, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
    else
        KSB_CUDA_CHECK(cudaMemsetAsync(K.what_full.p, 0, sizeof(double) * n, c.stream));
    outer_operator(L, K, K.what_full.p, K.vxc.p);
    StepLog lg;
    solve_orbitals(L, K, cg, o, h_lambda, d_Phi, ld, K.PhiT.p, ld, &lg);
    // Hartree boundary data from the moments of the phi_tilde density (driver.cpp:219-223)
    KSB_CUDA_CHECK(cudaMemsetAsync(K.bcb.p, 0, sizeof(double) * std::max(1, L.nb), c.stream));
    rho_vxc(L, K.PhiT.p, N, ld, K.sys.occ, K.sys.xc, K.rho_t.p, nullptr);
    if (K.sys.hartree_on) {
        const double ctr[3] = {0.5 * (L.box_lo[0] + L.box_hi[0]), 0.5 * (L.box_lo[1] + L.box_hi[1]),
                               0.5 * (L.box_lo[2] + L.box_hi[2])};
        boundary_values(L, moments(L, K.rho_t.p, K.phys, ctr), K.bcb.p);
    }
    // base blocks carry no static potential split (w_tilde = 0, lift = 0); rho_cur = density of the expansion of
    // the pure state (phi_H = 0, theta = 1), i.e. of phi_tilde (driver.cpp:225-243)
    KSB_CUDA_CHECK(cudaMemsetAsync(K.wt_full.p, 0, sizeof(double) * n, c.stream));
    KSB_CUDA_CHECK(cudaMemsetAsync(K.ell_full.p, 0, sizeof(double) * n, c.stream));
    KSB_CUDA_CHECK(cudaMemcpyAsync(K.rho.p, K.rho_t.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    K.mlc_ld = ld;
    K.mlc_sweeps = 0;
    if (log) *log = lg;
}

double mlc_sweep(Level& L, Corrector& K, CgWork& cg, const StepOptions& o, double* h_lambda, double* d_Phi, int ld) {
    Ctx& c = *L.ctx;
    K.precond = o.precond;
    if (K.mlc_ld == 0) raise(KSB_INVALID_ARGUMENT, "mlc_sweep before mlc_begin");
    if (ld != K.mlc_ld) raise(KSB_INVALID_ARGUMENT, "mlc_sweep: ld differs from mlc_begin's");
    const int N = K.sys.N, n = L.n;
    // pot = w(rho_cur) + v_xc(rho_cur) (driver.cpp:244-248)
    if (K.sys.xc_on)
        xc_field(L, K.sys.xc, K.rho.p, K.vxc.p);
    else
        KSB_CUDA_CHECK(cudaMemsetAsync(K.vxc.p, 0, sizeof(double) * n, c.stream));
    if (K.sys.hartree_on)
        hartree_of_density(L, K, cg, K.rho.p, K.bcb.p, o.tol_linear, K.what_full.p);
    else
        KSB_CUDA_CHECK(cudaMemsetAsync(K.what_full.p, 0, sizeof(double) * n, c.stream));
    launch(c, "elementwise", k_add, grid_of(c, n), kT, 0, int64_t(n), (const double*)K.what_full.p, 1.0,
           (const double*)K.vxc.p, 1.0, K.potf.p);
    // A_H = A_H1 + P^T M_pot P, b_i = b_H1 + P^T M_pot phi_tilde_i, beta_i = beta1 + phi_tilde_i^T M_pot phi_tilde_i
    // (driver.cpp:250-265): the pot-weighted terms ride in the v_xc slots of the ledger (A_H4, b_H4, beta4),
    // which a Hartree-off inner sweep adds to the a_op terms
    project_blocks(L, K.PhiT.p, N, ld, K.wt_full.p, K.ell_full.p, K.potf.p, K.eext.p, K.proj);
    InnerParams ip;
    ip.tol = o.tol_inner;
    ip.max_iterations = 1;
    ip.score_floor = o.score_floor;
    ip.nev_pad = o.nev_pad;
    ip.hartree = false;
    ip.occ = K.sys.occ;
    // sign alignment against the previous sweep's state (driver.cpp:277-283): the inner state persists
    inner_scf(L, K.coarse, K.proj, ip, h_lambda, K.inner, K.mlc_sweeps == 0);
    expand(L, K, K.PhiT.p, ld, K.wt_full.p, K.bcb.p, d_Phi, ld, K.wscr.p);
    // density change (driver.cpp:289-291)
    rho_vxc(L, d_Phi, N, ld, K.sys.occ, K.sys.xc, K.rho_t.p, nullptr);
    launch(c, "elementwise", k_add, grid_of(c, n), kT, 0, int64_t(n), (const double*)K.rho_t.p, 1.0,
           (const double*)K.rho.p, -1.0, K.diff.p);
    const double l1 = o.norm_l1 ? l1_norm(L, K.diff.p, K.phys) : 0.0;
    const auto nn = o.norm_l1 ? std::array<double, 2>{0.0, 0.0} : norms_sq(L, K.diff.p, K.phys);
    KSB_CUDA_CHECK(cudaMemcpyAsync(K.rho.p, K.rho_t.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
    KSB_CUDA_CHECK(cudaMemcpyAsync(h_lambda, K.inner.lamv[K.inner.cur].p, sizeof(double) * N, cudaMemcpyDeviceToHost,
                                   c.stream));
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    ++K.mlc_sweeps;
    if (o.norm_l1) return l1;
    const double l2 = std::sqrt(std::max(0.0, nn[0])), semi = std::sqrt(std::max(0.0, nn[1]));
    return std::sqrt(l2 * l2 + semi * semi);
}

void mlc_finish(Level& L, Corrector& K, CgWork& cg, const StepOptions& o, double* d_w, double* d_rho) {
    Ctx& c = *L.ctx;
    K.precond = o.precond;
    if (K.mlc_ld == 0) raise(KSB_INVALID_ARGUMENT, "mlc_finish before mlc_begin");
    const int n = L.n;
    if (K.sys.hartree_on)
        hartree_of_density(L, K, cg, K.rho.p, K.bcb.p, o.tol_linear, d_w);
    else
        KSB_CUDA_CHECK(cudaMemsetAsync(d_w, 0, sizeof(double) * n, c.stream));
    if (d_rho) KSB_CUDA_CHECK(cudaMemcpyAsync(d_rho, K.rho.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    K.mlc_ld = 0;
}

ScfStats coarse_scf(Level& L, Corrector& K, CgWork& cg, const ScfParams& p, double* h_lambda, double* d_Phi, int ld,
                    double* d_rho, double* d_w) {
    Ctx& c = *L.ctx;
    if (!K.ops_ready) level_ops(L, K);
    const int n = L.n, ni = L.ni, N = K.sys.N;
    if (ni != L.nH) raise(KSB_INVALID_ARGUMENT, "the coarse self-consistent solve runs on level 0");
    K.scf_history.clear();
    need(K.rho_t, n);
    need(K.vxc, n);
    need(K.what_full, n);
    need(K.diff, n);
    need(K.bcb, std::max(1, L.nb));
    need(K.hrhs, ni);
    need(K.wtil_int, ni);
    need(K.pot, ni);
    KSB_CUDA_CHECK(cudaMemsetAsync(d_rho, 0, sizeof(double) * n, c.stream));
    KSB_CUDA_CHECK(cudaMemsetAsync(d_w, 0, sizeof(double) * n, c.stream));
    const double ctr[3] = {0.5 * (L.box_lo[0] + L.box_hi[0]), 0.5 * (L.box_lo[1] + L.box_hi[1]),
                           0.5 * (L.box_lo[2] + L.box_hi[2])};
    ScfStats st;
    for (int iter = 1; iter <= p.max_iterations; ++iter) {
        // potential carried by one nodal field (hartree + v_xc(rho)), proj/src/scf.cpp:42-50
        if (p.hartree_on)
            KSB_CUDA_CHECK(cudaMemcpyAsync(K.what_full.p, d_w, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
        else
            KSB_CUDA_CHECK(cudaMemsetAsync(K.what_full.p, 0, sizeof(double) * n, c.stream));
        if (p.xc_on)
            xc_field(L, K.sys.xc, d_rho, K.vxc.p);
        else
            KSB_CUDA_CHECK(cudaMemsetAsync(K.vxc.p, 0, sizeof(double) * n, c.stream));
        outer_operator(L, K, K.what_full.p, K.vxc.p);
        dense_lowest_eigs(L, K.coarse, K.inner, MAT_H, N, h_lambda, d_Phi, ld);
        // density of the new orbitals and its H1 change (scf.cpp:67-70)
        rho_vxc(L, d_Phi, N, ld, K.sys.occ, K.sys.xc, K.rho_t.p, nullptr);
        launch(c, "elementwise", k_add, grid_of(c, n), kT, 0, int64_t(n), (const double*)K.rho_t.p, 1.0,
               (const double*)d_rho, -1.0, K.diff.p);
        double delta;
        if (p.norm_l1) {
            delta = l1_norm(L, K.diff.p, K.phys);
        } else {
            const auto nn = norms_sq(L, K.diff.p, K.phys);
            delta = std::sqrt(std::max(0.0, nn[0]) + std::max(0.0, nn[1]));
        }
        st.history.push_back(delta);
        st.iterations = iter;
        const double mix = (p.hartree_on || p.xc_on) ? p.mixing : 1.0;
        launch(c, "elementwise", k_add, grid_of(c, n), kT, 0, int64_t(n), (const double*)d_rho, 1.0 - mix,
               (const double*)K.rho_t.p, mix, d_rho);
        if (p.hartree_on) {  // hartree::solve_hartree of the mixed density (hartree.cpp:86-106), tol = tol_eig
            const Moments m = moments(L, d_rho, K.phys, ctr);
            boundary_values(L, m, K.bcb.p);
            launch(c, "elementwise", k_take_interior, grid_of(c, ni), kT, 0, ni, (const int32_t*)L.interior.p,
                   (const double*)d_rho, K.pot.p);
            spmm(c, L, L.mats[1].ii.p, nullptr, nullptr, K.pot.p, 1, 1, K.hrhs.p, 1);
            launch(c, "elementwise", k_add, grid_of(c, ni), kT, 0, int64_t(ni), (const double*)K.hrhs.p, kFourPi,
                   (const double*)K.hrhs.p, 0.0, K.hrhs.p);
            lift(L, 0, K.bcb.p, K.hrhs.p);
            CgOptions co;
            co.tol = p.tol_eig;
            CgColumnStats cs;
            cg_solve(c, L, 0, -1, nullptr, K.hrhs.p, K.wtil_int.p, 1, 1, co, &cs, cg);
            if (!cs.converged)
                raise(KSB_NONCONVERGENCE, "hartree solve stalled at residual " + std::to_string(cs.relative_residual));
            launch(c, "elementwise", k_full_from, grid_of(c, n), kT, 0, ni, L.nb, (const int32_t*)L.interior.p,
                   (const int32_t*)L.boundary.p, (const double*)K.wtil_int.p, (const double*)K.bcb.p, d_w);
        }
        KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
        K.scf_history = st.history;
        if (delta < p.tol && iter >= 2) return st;
    }
    std::string msg = "self-consistent iteration exceeded " + std::to_string(p.max_iterations) +
                      " steps; density changes:";
    for (size_t k = st.history.size() > 6 ? st.history.size() - 6 : 0; k < st.history.size(); ++k) {
        char b[32];
        std::snprintf(b, sizeof b, " %g", st.history[k]);
        msg += b;
    }
    raise(KSB_NONCONVERGENCE, msg);
}

}  // namespace ksb
