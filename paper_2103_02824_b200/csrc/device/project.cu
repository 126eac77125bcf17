// K-PROJ: projection of the fine correction onto the coarse interior space, element by element.
//
// Replaces the fine assemblies + sparse Galerkin products of corr::prepare_blocks
// (reference proj/src/correction.cpp:113-212). Every fine operator X in the ledger is
// element-assembled, so P^T X P and P^T (X phi) decompose over fine tets T with coarse
// ancestor C:  (P^T X P)_ab = sum_T mu_T^T E^X_T mu_T, mu_T(i,a) = P_int(v_i, C_a).
// One streaming pass over the fine tets (grouped by ancestor) produces every block; a
// deterministic coarse assembly (per coarse dof, ascending coarse tet) finishes the job.
// No fine CSR matrix is formed for M_wt, M_xc, M_ell or the per-orbital M_phi.
#include <algorithm>

#include "geom.cuh"
#include "project.cuh"

namespace ksb {

namespace {

constexpr int kProjThreads = 128;
constexpr int kProjWideMin = 8;  // orbital count from which the staged (orbital-parallel) kernel is used

struct ProjIn {
    const int32_t *tets, *iidx, *anc_ptr, *anc_tets, *ctets, *ciidx, *pint_col;
    const double *xyz, *pint_val, *eext, *Phi, *wt, *ell, *vxc;
    int N, ld, nct;
    // work chunks: chunk k covers anc_tets[ch_b[k], ch_e[k]) of coarse tet ch_c[k] (a coarse tet with more fine
    // descendants than the chunk size is split, so adaptive levels keep every SM busy); partials per chunk
    const int32_t *ch_c, *ch_b, *ch_e;
    int nch;
};

__device__ __forceinline__ void load_mu(const ProjIn& in, int4 v, const int (&ci)[4], double (&mu)[4][4]) {
    const int vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = in.iidx[vv[i]];
        int pc[4] = {-1, -1, -1, -1};
        double pv[4] = {0, 0, 0, 0};
        if (r >= 0) {
            const int4 c4 = reinterpret_cast<const int4*>(in.pint_col)[r];
            pc[0] = c4.x;
            pc[1] = c4.y;
            pc[2] = c4.z;
            pc[3] = c4.w;
#pragma unroll
            for (int k = 0; k < 4; ++k) pv[k] = in.pint_val[4 * size_t(r) + k];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            double m = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (ci[a] >= 0 && pc[k] == ci[a]) m = pv[k];
            mu[i][a] = m;
        }
    }
}

/// out(a,b) += sum_ij mu(i,a) E(i,j) mu(j,b)
__device__ __forceinline__ void acc_proj(const double (&mu)[4][4], const double (&E)[4][4], double* out) {
    double t[4][4];  // t(i,b) = sum_j E(i,j) mu(j,b)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int b = 0; b < 4; ++b) t[i][b] = E[i][0] * mu[0][b] + E[i][1] * mu[1][b] + E[i][2] * mu[2][b] + E[i][3] * mu[3][b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) out[4 * a + b] += mu[0][a] * t[0][b] + mu[1][a] * t[1][b] + mu[2][a] * t[2][b] + mu[3][a] * t[3][b];
}

/// vector part: y = E x; outv(a) += mu(:,a).y ; returns x.y
__device__ __forceinline__ double acc_vec(const double (&mu)[4][4], const double (&E)[4][4], const double (&x)[4],
                                          double* outv) {
    double y[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) y[i] = E[i][0] * x[0] + E[i][1] * x[1] + E[i][2] * x[2] + E[i][3] * x[3];
#pragma unroll
    for (int a = 0; a < 4; ++a) outv[a] += mu[0][a] * y[0] + mu[1][a] * y[1] + mu[2][a] * y[2] + mu[3][a] * y[3];
    return x[0] * y[0] + x[1] * y[1] + x[2] * y[2] + x[3] * y[3];
}

template <int K>
__device__ void block_reduce_store(double (&acc)[K], double* __restrict__ dst) {
    __shared__ double red[kProjThreads / 32][K];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double s = warp_sum(acc[k]);
        if (lane == 0) red[warp][k] = s;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kProjThreads / 32; ++w) s += red[w][k];
        dst[k] = s;
    }
}

// shared part (function y == N): A_H1 (16) A_H3 (16) A_H4 (16) d_Hh (4) lift_load (4) zeta lift0
__global__ void __launch_bounds__(kProjThreads) k_proj_shared(ProjIn in, double* __restrict__ part) {
    const int ch = blockIdx.x;
    const int C = in.ch_c[ch];
    double acc[kSharedK];
#pragma unroll
    for (int k = 0; k < kSharedK; ++k) acc[k] = 0.0;
    const int4 cv = reinterpret_cast<const int4*>(in.ctets)[C];
    const int ci[4] = {in.ciidx[cv.x], in.ciidx[cv.y], in.ciidx[cv.z], in.ciidx[cv.w]};
    for (int p = in.ch_b[ch] + threadIdx.x; p < in.ch_e[ch]; p += blockDim.x) {
        const int t = in.anc_tets[p];
        const int4 v = reinterpret_cast<const int4*>(in.tets)[t];
        TetG G;
        tet_geometry(in.xyz, v, G);
        double mu[4][4];
        load_mu(in, v, ci, mu);
        const double wt[4] = {in.wt[v.x], in.wt[v.y], in.wt[v.z], in.wt[v.w]};
        const double el[4] = {in.ell[v.x], in.ell[v.y], in.ell[v.z], in.ell[v.w]};
        const double xc[4] = {in.vxc[v.x], in.vxc[v.y], in.vxc[v.z], in.vxc[v.w]};
        double S[4][4], E[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
                S[i][j] = G.vol * (G.g[i][0] * G.g[j][0] + G.g[i][1] * G.g[j][1] + G.g[i][2] * G.g[j][2]);
        // a_eff element: 1/2 S + M_ext + M_ell
        mass_elem(G.vol, el, E);
        const double* ex = in.eext + size_t(t) * 16;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) E[i][j] += 0.5 * S[i][j] + ex[4 * i + j];
        acc_proj(mu, E, acc + 0);
        mass_elem(G.vol, wt, E);
        acc_proj(mu, E, acc + 16);
        mass_elem(G.vol, xc, E);
        acc_proj(mu, E, acc + 32);
        acc[52] += acc_vec(mu, S, wt, acc + 48);  // d_Hh, zeta
        double y[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) y[i] = S[i][0] * el[0] + S[i][1] * el[1] + S[i][2] * el[2] + S[i][3] * el[3];
#pragma unroll
        for (int a = 0; a < 4; ++a) acc[53 + a] += mu[0][a] * y[0] + mu[1][a] * y[1] + mu[2][a] * y[2] + mu[3][a] * y[3];
        acc[57] += wt[0] * y[0] + wt[1] * y[1] + wt[2] * y[2] + wt[3] * y[3];
    }
    block_reduce_store<kSharedK>(acc, part + size_t(ch) * kStride);
}

// per orbital (function y = i): A_h4 (16) b_H1 b_H3 b_H4 c_Hh d_phi rhs (6 x 4) beta1 beta3 beta4 gamma zeta_phi (5)
__global__ void __launch_bounds__(kProjThreads) k_proj_orbital(ProjIn in, double* __restrict__ part) {
    const int ch = blockIdx.x;
    const int C = in.ch_c[ch];
    const int i = blockIdx.y;
    double acc[kOrbK];
#pragma unroll
    for (int k = 0; k < kOrbK; ++k) acc[k] = 0.0;
    const int4 cv = reinterpret_cast<const int4*>(in.ctets)[C];
    const int ci[4] = {in.ciidx[cv.x], in.ciidx[cv.y], in.ciidx[cv.z], in.ciidx[cv.w]};
    for (int p = in.ch_b[ch] + threadIdx.x; p < in.ch_e[ch]; p += blockDim.x) {
        const int t = in.anc_tets[p];
        const int4 v = reinterpret_cast<const int4*>(in.tets)[t];
        TetG G;
        tet_geometry(in.xyz, v, G);
        double mu[4][4];
        load_mu(in, v, ci, mu);
        const int vv[4] = {v.x, v.y, v.z, v.w};
        double ph[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int r = in.iidx[vv[k]];
            ph[k] = r >= 0 ? in.Phi[size_t(r) * in.ld + i] : 0.0;
        }
        const double wt[4] = {in.wt[v.x], in.wt[v.y], in.wt[v.z], in.wt[v.w]};
        const double el[4] = {in.ell[v.x], in.ell[v.y], in.ell[v.z], in.ell[v.w]};
        const double xc[4] = {in.vxc[v.x], in.vxc[v.y], in.vxc[v.z], in.vxc[v.w]};
        const double one[4] = {1.0, 1.0, 1.0, 1.0};
        double S[4][4], E[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
                S[a][b] = G.vol * (G.g[a][0] * G.g[b][0] + G.g[a][1] * G.g[b][1] + G.g[a][2] * G.g[b][2]);
        mass_elem(G.vol, ph, E);  // M_phi
        acc_proj(mu, E, acc + 0);
        acc_vec(mu, E, ph, acc + 40);  // rhs = P^T (M_phi phi)
        mass_elem(G.vol, el, E);
        const double* ex = in.eext + size_t(t) * 16;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) E[a][b] += 0.5 * S[a][b] + ex[4 * a + b];
        acc[44] += acc_vec(mu, E, ph, acc + 16);  // b_H1, beta1
        mass_elem(G.vol, wt, E);
        acc[45] += acc_vec(mu, E, ph, acc + 20);  // b_H3, beta3
        mass_elem(G.vol, xc, E);
        acc[46] += acc_vec(mu, E, ph, acc + 24);  // b_H4, beta4
        mass_elem(G.vol, one, E);
        acc[47] += acc_vec(mu, E, ph, acc + 28);  // c_Hh, gamma
        acc[48] += acc_vec(mu, S, ph, acc + 32);  // d_phi, zeta_phi
    }
    block_reduce_store<kOrbK>(acc, part + (size_t(1 + i) * in.nch + ch) * kStride);
}

// Wide variant for many orbitals: the orbital-independent per-tet data (mu, the element matrices of the
// a_eff, w~, v_xc, unit and stiffness operators) is staged in shared memory once per chunk of fine tets, and the
// block's threads then run (orbital, tet slot) pairs over it. Orbital values of a fine vertex are read by
// consecutive threads from one row of Phi (coalesced). Each thread owns the 49 accumulators of its orbital;
// tet slots are folded in fixed order at the end.
constexpr int kWideTets = 64;   // fine tets per staged chunk
constexpr int kWideRec = 104;   // doubles per staged tet: mu 16, E1 E3 E4 Eone S (5 x 16), vol, 4 rows (as int), pad

__global__ void __launch_bounds__(kProjThreads) k_proj_orbital_wide(ProjIn in, double* __restrict__ part) {
    extern __shared__ double st[];  // kWideTets * kWideRec, reused for the final fold
    const int ch = blockIdx.x;
    const int C = in.ch_c[ch];
    const int N = in.N;
    const int i0 = blockIdx.y * kProjThreads;
    const int NI = min(N - i0, kProjThreads);
    const int TS = kProjThreads / NI;  // tet slots per orbital
    const int oi = threadIdx.x % NI, slot = threadIdx.x / NI;
    const bool act = slot < TS;
    const int i = i0 + oi;
    double acc[kOrbK];
#pragma unroll
    for (int k = 0; k < kOrbK; ++k) acc[k] = 0.0;
    const int4 cv = reinterpret_cast<const int4*>(in.ctets)[C];
    const int ci[4] = {in.ciidx[cv.x], in.ciidx[cv.y], in.ciidx[cv.z], in.ciidx[cv.w]};
    const int pb = in.ch_b[ch], pe = in.ch_e[ch];
    for (int c0 = pb; c0 < pe; c0 += kWideTets) {
        const int nc = min(kWideTets, pe - c0);
        __syncthreads();
        if (threadIdx.x < nc) {
            double* R = st + threadIdx.x * kWideRec;
            const int t = in.anc_tets[c0 + threadIdx.x];
            const int4 v = reinterpret_cast<const int4*>(in.tets)[t];
            TetG G;
            tet_geometry(in.xyz, v, G);
            double mu[4][4];
            load_mu(in, v, ci, mu);
            const double wt[4] = {in.wt[v.x], in.wt[v.y], in.wt[v.z], in.wt[v.w]};
            const double el[4] = {in.ell[v.x], in.ell[v.y], in.ell[v.z], in.ell[v.w]};
            const double xc[4] = {in.vxc[v.x], in.vxc[v.y], in.vxc[v.z], in.vxc[v.w]};
            const double one[4] = {1.0, 1.0, 1.0, 1.0};
            double S[4][4], E[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    S[a][b] = G.vol * (G.g[a][0] * G.g[b][0] + G.g[a][1] * G.g[b][1] + G.g[a][2] * G.g[b][2]);
                    R[4 * a + b] = mu[a][b];
                    R[80 + 4 * a + b] = S[a][b];
                }
            mass_elem(G.vol, el, E);
            const double* ex = in.eext + size_t(t) * 16;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) R[16 + 4 * a + b] = E[a][b] + 0.5 * S[a][b] + ex[4 * a + b];
            mass_elem(G.vol, wt, E);
#pragma unroll
            for (int k = 0; k < 16; ++k) R[32 + k] = E[k / 4][k % 4];
            mass_elem(G.vol, xc, E);
#pragma unroll
            for (int k = 0; k < 16; ++k) R[48 + k] = E[k / 4][k % 4];
            mass_elem(G.vol, one, E);
#pragma unroll
            for (int k = 0; k < 16; ++k) R[64 + k] = E[k / 4][k % 4];
            R[96] = G.vol;
            int* ri = reinterpret_cast<int*>(R + 97);
            ri[0] = in.iidx[v.x];
            ri[1] = in.iidx[v.y];
            ri[2] = in.iidx[v.z];
            ri[3] = in.iidx[v.w];
        }
        __syncthreads();
        if (act)
            for (int q = slot; q < nc; q += TS) {
                const double* R = st + q * kWideRec;
                const int* ri = reinterpret_cast<const int*>(R + 97);
                double ph[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) ph[k] = ri[k] >= 0 ? in.Phi[size_t(ri[k]) * in.ld + i] : 0.0;
                double mu[4][4], E[4][4];
#pragma unroll
                for (int k = 0; k < 16; ++k) mu[k / 4][k % 4] = R[k];
                mass_elem(R[96], ph, E);  // M_phi
                acc_proj(mu, E, acc + 0);
                acc_vec(mu, E, ph, acc + 40);  // rhs = P^T (M_phi phi)
#pragma unroll
                for (int m = 0; m < 5; ++m) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) E[k / 4][k % 4] = R[16 + 16 * m + k];
                    // b_H1/beta1, b_H3/beta3, b_H4/beta4, c_Hh/gamma, d_phi/zeta_phi
                    acc[44 + m] += acc_vec(mu, E, ph, acc + 16 + 4 * m);
                }
            }
    }
    // fold the tet slots of each orbital in slot order
    __syncthreads();
    if (TS > 1) {
        if (act)
            for (int k = 0; k < kOrbK; ++k) st[(size_t(slot) * NI + oi) * kOrbK + k] = acc[k];
        __syncthreads();
        for (int e = threadIdx.x; e < NI * kOrbK; e += blockDim.x) {
            const int o = e / kOrbK, k = e % kOrbK;
            double s2 = 0.0;
            for (int sl = 0; sl < TS; ++sl) s2 += st[(size_t(sl) * NI + o) * kOrbK + k];
            part[(size_t(1 + i0 + o) * in.nch + ch) * kStride + k] = s2;
        }
    } else if (act) {
        double* dst = part + (size_t(1 + i) * in.nch + ch) * kStride;
        for (int k = 0; k < kOrbK; ++k) dst[k] = acc[k];
    }
}

/// dense coarse assembly: out[m][a][b] = sum over (C, la) of a, lb with ci[lb] >= 0 of part[m][C][off + 4 la + lb]
__global__ void k_coarse_mat(int nh, int nmats, const int32_t* __restrict__ cinc_ptr, const int32_t* __restrict__ cinc,
                             const int32_t* __restrict__ ctets, const int32_t* __restrict__ ciidx,
                             const double* __restrict__ part, int64_t mat_stride, int off, int nct,
                             double* __restrict__ out, int64_t out_stride) {
    const int a = blockIdx.x * blockDim.y + threadIdx.y;
    const int m = blockIdx.y;
    if (a >= nh || m >= nmats) return;
    double* row = out + m * out_stride + size_t(a) * nh;
    for (int b = threadIdx.x; b < nh; b += blockDim.x) row[b] = 0.0;
    __syncwarp();
    if (threadIdx.x != 0) return;
    const double* P = part + m * mat_stride;
    for (int k = cinc_ptr[a]; k < cinc_ptr[a + 1]; ++k) {
        const int C = cinc[k] >> 2, la = cinc[k] & 3;
        for (int lb = 0; lb < 4; ++lb) {
            const int b = ciidx[ctets[4 * C + lb]];
            if (b >= 0) row[b] += P[size_t(C) * kStride + off + 4 * la + lb];
        }
    }
    (void)nct;
}

/// coarse vectors: out[v][a] = sum over (C, la) of a of part[v][C][off + la]
__global__ void k_coarse_vec(int nh, int nvec, const int32_t* __restrict__ cinc_ptr, const int32_t* __restrict__ cinc,
                             const double* __restrict__ part, int64_t vec_stride, const int* __restrict__ offs,
                             int noffs, double* __restrict__ out) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y;  // v = m * noffs + o
    if (a >= nh || v >= nvec * noffs) return;
    const int m = v / noffs, o = offs[v % noffs];
    const double* P = part + m * vec_stride;
    double s = 0.0;
    for (int k = cinc_ptr[a]; k < cinc_ptr[a + 1]; ++k) {
        const int C = cinc[k] >> 2, la = cinc[k] & 3;
        s += P[size_t(C) * kStride + o + la];
    }
    out[size_t(v) * nh + a] = s;
}

/// scalars: out[v] = sum over C ascending of part[m][C][off]
__global__ void k_coarse_scalar(int nct, int nvals, const double* __restrict__ part, int64_t stride,
                                const int* __restrict__ offs, int noffs, double* __restrict__ out) {
    const int v = blockIdx.x;
    if (v >= nvals * noffs) return;
    const int m = v / noffs, o = offs[v % noffs];
    const double* P = part + m * stride;
    const int lane = threadIdx.x;
    double s = 0.0;
    for (int C = lane; C < nct; C += 32) s += P[size_t(C) * kStride + o];
    s = warp_sum(s);
    if (lane == 0) out[v] = s;
}

/// per-coarse-tet partials from the chunk partials, chunks in ascending order (deterministic)
__global__ void k_proj_fold(int nct, int nfun, int nch, const int32_t* __restrict__ cptr,
                            const double* __restrict__ pch, double* __restrict__ part) {
    const int64_t total = int64_t(nfun) * nct * kStride;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int k = int(e % kStride);
        const int64_t fc = e / kStride;
        const int C = int(fc % nct), f = int(fc / nct);
        double s = 0.0;
        for (int q = cptr[C]; q < cptr[C + 1]; ++q) s += pch[(size_t(f) * nch + q) * kStride + k];
        part[e] = s;
    }
}

}  // namespace

void project_blocks(Level& L, const double* Phi, int N, int ld, const double* wt_full, const double* ell_full,
                    const double* vxc_full, const double* eext, ProjOut& o) {
    Ctx& c = *L.ctx;
    const int nh = L.nH, nct = L.nct;
    o.ensure(nh, N, nct);
    const int nch = L.pj_n;
    const bool split = nch != nct;
    if (split && o.pchunk.n < int64_t(nch) * kStride * (N + 1)) o.pchunk.alloc(int64_t(nch) * kStride * (N + 1));
    double* dst = split ? o.pchunk.p : o.part.p;
    ProjIn in{(const int32_t*)L.tets.p, (const int32_t*)L.iidx.p, (const int32_t*)L.anc_ptr.p,
              (const int32_t*)L.anc_tets.p, (const int32_t*)L.ctets.p, (const int32_t*)L.ciidx.p,
              (const int32_t*)L.pint_col.p, (const double*)L.xyz.p, (const double*)L.pint_val.p, eext, Phi, wt_full,
              ell_full, vxc_full, N, ld, nct, (const int32_t*)L.pj_c.p, (const int32_t*)L.pj_b.p,
              (const int32_t*)L.pj_e.p, nch};
    launch(c, "project", k_proj_shared, nch, kProjThreads, 0, in, dst);
    if (N >= kProjWideMin) {
        const size_t smem = sizeof(double) * std::max(kWideTets * kWideRec, kProjThreads * kOrbK);
        static bool attr = false;
        if (!attr) {
            KSB_CUDA_CHECK(cudaFuncSetAttribute(k_proj_orbital_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            attr = true;
        }
        launch(c, "project", k_proj_orbital_wide, dim3(nch, ceil_div(N, kProjThreads)), kProjThreads, smem, in, dst);
    } else if (N > 0) {
        launch(c, "project", k_proj_orbital, dim3(nch, N), kProjThreads, 0, in, dst);
    }
    if (split)
        launch(c, "project", k_proj_fold, c.sm_count * 8, 256, 0, nct, N + 1, nch, (const int32_t*)L.pj_ptr.p,
               (const double*)o.pchunk.p, o.part.p);

    const int64_t fstride = int64_t(nct) * kStride;  // stride between functions in part
    const int64_t nh2 = int64_t(nh) * nh;
    if (nh > 0) {
        dim3 blk(32, 4);
        // shared matrices: A_H1 (off 0), A_H3 (16), A_H4 (32) of function 0
        for (int m = 0; m < 3; ++m)
            launch(c, "project_asm", k_coarse_mat, dim3(ceil_div(nh, 4), 1), blk, 0, nh, 1, (const int32_t*)L.cinc_ptr.p,
                   (const int32_t*)L.cinc.p, (const int32_t*)L.ctets.p, (const int32_t*)L.ciidx.p,
                   (const double*)o.part.p, fstride, 16 * m, nct, o.shared_mats.p + m * nh2, nh2);
        if (N > 0)
            launch(c, "project_asm", k_coarse_mat, dim3(ceil_div(nh, 4), N), blk, 0, nh, N, (const int32_t*)L.cinc_ptr.p,
                   (const int32_t*)L.cinc.p, (const int32_t*)L.ctets.p, (const int32_t*)L.ciidx.p,
                   (const double*)(o.part.p + fstride), fstride, 0, nct, o.A_h4.p, nh2);
        // shared vectors d_Hh (48), lift_load (53); orbital vectors b_H1 16, b_H3 20, b_H4 24, c_Hh 28, d_phi 32, rhs 40
        launch(c, "project_asm", k_coarse_vec, dim3(ceil_div(nh, 128), 2), 128, 0, nh, 1, (const int32_t*)L.cinc_ptr.p,
               (const int32_t*)L.cinc.p, (const double*)o.part.p, fstride, (const int*)o.offs.p, 2, o.shared_vecs.p);
        if (N > 0)
            launch(c, "project_asm", k_coarse_vec, dim3(ceil_div(nh, 128), N * 6), 128, 0, nh, N,
                   (const int32_t*)L.cinc_ptr.p, (const int32_t*)L.cinc.p, (const double*)(o.part.p + fstride), fstride,
                   (const int*)(o.offs.p + 2), 6, o.orb_vecs.p);
    }
    // scalars: shared zeta (52), lift0 (57); orbital beta1..zeta_phi (44..48)
    launch(c, "project_asm", k_coarse_scalar, 2, 32, 0, nct, 1, (const double*)o.part.p, fstride,
           (const int*)(o.offs.p + 8), 2, o.shared_scal.p);
    if (N > 0)
        launch(c, "project_asm", k_coarse_scalar, N * 5, 32, 0, nct, N, (const double*)(o.part.p + fstride), fstride,
               (const int*)(o.offs.p + 10), 5, o.orb_scal.p);
}

void ProjOut::ensure(int nh_, int N_, int nct_) {
    nh = nh_;
    N = N_;
    const int64_t nh2 = int64_t(nh) * nh;
    if (part.n < int64_t(nct_) * kStride * (N + 1)) part.alloc(int64_t(nct_) * kStride * (N + 1));
    if (shared_mats.n < 3 * nh2) shared_mats.alloc(std::max<int64_t>(1, 3 * nh2));
    if (A_h4.n < N * nh2) A_h4.alloc(std::max<int64_t>(1, N * nh2));
    if (shared_vecs.n < 2 * nh) shared_vecs.alloc(std::max<int64_t>(1, 2 * nh));
    if (orb_vecs.n < 6 * int64_t(N) * nh) orb_vecs.alloc(std::max<int64_t>(1, 6 * int64_t(N) * nh));
    if (shared_scal.n < 2) shared_scal.alloc(2);
    if (orb_scal.n < 5 * N) orb_scal.alloc(std::max(1, 5 * N));
    if (offs.n < 16) {
        offs.alloc(16);
        const std::vector<int> h = {48, 53, 16, 20, 24, 28, 32, 40, 52, 57, 44, 45, 46, 47, 48, 0};
        KSB_CUDA_CHECK(cudaMemcpy(offs.p, h.data(), sizeof(int) * 16, cudaMemcpyHostToDevice));
    }
}

}  // namespace ksb
