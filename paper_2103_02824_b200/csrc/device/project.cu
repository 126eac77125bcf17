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
#include <cstdlib>
#include <map>

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
constexpr int kWideRec0 = 104;  // record without the T_k block
constexpr int kWideRec = 144;   // doubles per staged tet: mu 16, E1 E3 E4 Eone S (5 x 16), vol, 4 rows (as int), pad,
                                // T_k = mu^T E^(k) mu for the four hat weights (4 x 10 unique entries) at 104

/// TK: the orbital mass element through the precomputed T_k (many orbitals: the 4 x (element + mu^T E mu) per tet of
/// the staging amortise over >= 64 orbitals; at N = 21 they cost more than they save, 32.6 -> 38.9 ms on configs[3])
template <bool TK>
__global__ void __launch_bounds__(kProjThreads) k_proj_orbital_wide(ProjIn in, double* __restrict__ part) {
    constexpr int REC = TK ? kWideRec : kWideRec0;
    extern __shared__ double st[];  // kWideTets * REC, reused for the final fold
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
            double* R = st + threadIdx.x * REC;
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
            // the orbital mass element is linear in the orbital's vertex values: M_phi = sum_k phi_k E^(k) with E^(k)
            // the element of the hat weight k, so mu^T M_phi mu = sum_k phi_k T_k with the orbital-independent
            // T_k = mu^T E^(k) mu (symmetric: 10 entries), 40 multiply-adds per (orbital, tet) instead of 128 + the element
#pragma unroll
            for (int k = 0; TK && k < 4; ++k) {
                double hat[4] = {0.0, 0.0, 0.0, 0.0};
                hat[k] = 1.0;
                mass_elem(G.vol, hat, E);
                double T[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) T[e] = 0.0;
                acc_proj(mu, E, T);
                int m = 0;
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = a; b < 4; ++b) R[104 + 10 * k + m++] = T[4 * a + b];
            }
        }
        __syncthreads();
        if (act)
            for (int q = slot; q < nc; q += TS) {
                const double* R = st + q * REC;
                const int* ri = reinterpret_cast<const int*>(R + 97);
                double ph[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) ph[k] = ri[k] >= 0 ? in.Phi[size_t(ri[k]) * in.ld + i] : 0.0;
                double mu[4][4], E[4][4];
#pragma unroll
                for (int k = 0; k < 16; ++k) mu[k / 4][k % 4] = R[k];
                if constexpr (!TK) {
                    mass_elem(R[96], ph, E);  // M_phi
                    acc_proj(mu, E, acc + 0);
                    acc_vec(mu, E, ph, acc + 40);  // rhs = P^T (M_phi phi)
                } else {  // A_h4 += mu^T M_phi mu = sum_k phi_k T_k (upper triangle; mirrored after the tet loop)
                    int m = 0;
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = a; b < 4; ++b, ++m)
                            acc[4 * a + b] += ph[0] * R[104 + m] + ph[1] * R[114 + m] + ph[2] * R[124 + m] + ph[3] * R[134 + m];
                    // rhs += mu^T (M_phi phi), (M_phi phi)_i = |T| / 120 (W^2 + q + 2 phi_i (W + phi_i)), W = sum phi, q = sum phi^2
                    const double W = ph[0] + ph[1] + ph[2] + ph[3];
                    const double q = ph[0] * ph[0] + ph[1] * ph[1] + ph[2] * ph[2] + ph[3] * ph[3];
                    const double sc = R[96] / 120.0, base = W * W + q;
                    double y[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) y[i] = sc * (base + 2.0 * ph[i] * (W + ph[i]));
#pragma unroll
                    for (int a = 0; a < 4; ++a) acc[40 + a] += mu[0][a] * y[0] + mu[1][a] * y[1] + mu[2][a] * y[2] + mu[3][a] * y[3];
                }
#pragma unroll
                for (int m = 0; m < 5; ++m) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) E[k / 4][k % 4] = R[16 + 16 * m + k];
                    // b_H1/beta1, b_H3/beta3, b_H4/beta4, c_Hh/gamma, d_phi/zeta_phi
                    acc[44 + m] += acc_vec(mu, E, ph, acc + 16 + 4 * m);
                }
            }
    }
    if constexpr (TK) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = a + 1; b < 4; ++b) acc[4 * b + a] = acc[4 * a + b];
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

// ---------------- aggregated projection (GEMM form) for many orbitals ----------------
// Every orbital-dependent ledger entry of a coarse tet is linear or quadratic in the orbital's nodal values, with
// coefficients that do not depend on the orbital: per fine tet T and corner l,
//   A_h4[ab] += phi_l (vol/120) (K_ab + mu_la (m_b + mu_lb) + mu_lb (m_a + mu_la)),  K_ab = m_a m_b + sum_j mu_ja mu_jb,
//   b_X[a]   += phi_l sum_j mu_ja E^X[j][l]                (X = a_eff, w~, v_xc, 1, S: b_H1, b_H3, b_H4, c_Hh, d_phi),
// and per vertex / edge of T
//   rhs[a] += phi_l^2 (vol/120)(2 m_a + 4 mu_la) + phi_k phi_l (vol/60)(m_a + mu_ka + mu_la),
//   beta_X += phi_l^2 E^X[l][l] + phi_k phi_l (E^X[k][l] + E^X[l][k])
// (m_a = sum_j mu_ja; mass_elem's weights (vol/120) c_jk (1 + delta_jl + delta_kl)). Summing the coefficients over the
// tets of a compact chunk first (per chunk vertex: R, 36 rows; per chunk vertex and edge: Q, 9 rows) turns the
// orbital loop into two small GEMMs per chunk, [36 x V] [V x N] and [9 x (V + E)] [(V + E) x N] (vertex squares and
// edge products as the second operand), run on the FP64 tensor cores (DMMA, mma.sync m8n8k4) -- about 20x fewer
// flops than the per-tet form. The coefficient sums are gathers over each vertex's / edge's incident tets in
// ascending order and the chunks of one work item accumulate in fixed order: deterministic.
constexpr int kPgThreads = 256;
constexpr int kPgSub = 16;     // tets per coefficient sub-block
constexpr int kPgStage = 117;  // per staged tet: mu 16, m 4, K 16, vol, E^X 5 x 16
constexpr int kPgCo = 234;     // coefficients per tet: G_A 64, G_X 80, vertex squares 36, edge products 54
constexpr int kPgSlice = 32;   // orbital columns per GEMM slice
constexpr int kPgRS = 84;      // R row stride (bank-conflict-free A fragments)
constexpr int kPgQS = 324;     // Q row stride
constexpr int kPgPS = 36;      // staged orbital-row stride
constexpr size_t kPgSmem =
    sizeof(double) * (size_t(kPgSub) * (kPgStage + kPgCo) + 36 * kPgRS + 9 * kPgQS + size_t(kPgV) * kPgPS) +
    sizeof(int32_t) * kPgE;

struct PgIn {
    const int32_t *item_c, *item_ch, *ch_t, *ch_v, *ch_e, *tets, *verts, *edges, *vinc_ptr, *vinc, *einc_ptr, *einc;
    int n_items;
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

/// index of the tet edge (c1 < c2) among the 6
__device__ __forceinline__ int pg_pair(int c1, int c2) { return c1 == 0 ? c2 - 1 : c1 == 1 ? c2 + 1 : 5; }

/// first incidence of a (t-sorted) list with tet >= tlo
__device__ __forceinline__ int pg_lower(const int32_t* __restrict__ inc, int b, int e, int tlo, int shift) {
    while (b < e) {
        const int m = (b + e) >> 1;
        if ((inc[m] >> shift) < tlo)
            b = m + 1;
        else
            e = m;
    }
    return b;
}

template <int NS>
__global__ void __launch_bounds__(kPgThreads, NS >= 3 ? 1 : 2) k_proj_gemm(ProjIn in, PgIn pg, double* __restrict__ part) {
    extern __shared__ __align__(16) double pgs[];
    double* ST = pgs;                    // kPgSub x kPgStage
    double* CO = ST + kPgSub * kPgStage;  // kPgSub x kPgCo
    double* R = CO + kPgSub * kPgCo;
    double* Q = R + 36 * kPgRS;
    double* PH = Q + 9 * kPgQS;
    int32_t* ED = reinterpret_cast<int32_t*>(PH + kPgV * kPgPS);
    const int N = in.N;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int item = blockIdx.x; item < pg.n_items; item += gridDim.x) {
        const int C = pg.item_c[item];
        const int4 cv = reinterpret_cast<const int4*>(in.ctets)[C];
        const int ci[4] = {in.ciidx[cv.x], in.ciidx[cv.y], in.ciidx[cv.z], in.ciidx[cv.w]};
        double acc[NS][7][2];
#pragma unroll
        for (int sl = 0; sl < NS; ++sl)
#pragma unroll
            for (int k = 0; k < 7; ++k) acc[sl][k][0] = acc[sl][k][1] = 0.0;
        for (int ch = pg.item_ch[item]; ch < pg.item_ch[item + 1]; ++ch) {
            const int t0 = pg.ch_t[ch], nt = pg.ch_t[ch + 1] - t0;
            const int v0 = pg.ch_v[ch], V = pg.ch_v[ch + 1] - v0;
            const int e0 = pg.ch_e[ch], E = pg.ch_e[ch + 1] - e0;
            const int nR = 36 * V, nQ = 9 * (V + E);
            __syncthreads();  // the previous chunk's shared data is consumed
            for (int k = threadIdx.x; k < E; k += blockDim.x) ED[k] = pg.edges[e0 + k];
            for (int sb = 0; sb * kPgSub < nt; ++sb) {
                const int tb = sb * kPgSub, ns = min(kPgSub, nt - tb);
                // stage: geometry, interpolation, the five element operators of each tet of the sub-block
                if (int(threadIdx.x) < ns) {
                    double* S = ST + threadIdx.x * kPgStage;
                    const int t = pg.tets[t0 + tb + threadIdx.x];
                    const int4 v = reinterpret_cast<const int4*>(in.tets)[t];
                    TetG G;
                    tet_geometry(in.xyz, v, G);
                    double mu[4][4];
                    load_mu(in, v, ci, mu);
                    double m[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        m[a] = mu[0][a] + mu[1][a] + mu[2][a] + mu[3][a];
                        S[16 + a] = m[a];
#pragma unroll
                        for (int i = 0; i < 4; ++i) S[4 * i + a] = mu[i][a];
                    }
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b)
                            S[20 + 4 * a + b] = m[a] * m[b] + (mu[0][a] * mu[0][b] + mu[1][a] * mu[1][b] +
                                                               mu[2][a] * mu[2][b] + mu[3][a] * mu[3][b]);
                    S[36] = G.vol;
                    const int vv[4] = {v.x, v.y, v.z, v.w};
                    double el[4], wt[4], xc[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        el[i] = in.ell[vv[i]];
                        wt[i] = in.wt[vv[i]];
                        xc[i] = in.vxc[vv[i]];
                    }
                    const double* ex = in.eext + size_t(t) * 16;
                    double E1[4][4], E3[4][4], E4[4][4];
                    mass_elem(G.vol, el, E1);
                    mass_elem(G.vol, wt, E3);
                    mass_elem(G.vol, xc, E4);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
#pragma unroll
                        for (int l = 0; l < 4; ++l) {
                            const double sjl = G.vol * (G.g[j][0] * G.g[l][0] + G.g[j][1] * G.g[l][1] + G.g[j][2] * G.g[l][2]);
                            S[37 + 4 * j + l] = E1[j][l] + 0.5 * sjl + ex[4 * j + l];
                            S[53 + 4 * j + l] = E3[j][l];
                            S[69 + 4 * j + l] = E4[j][l];
                            S[85 + 4 * j + l] = (G.vol / 120.0) * (j == l ? 2.0 : 1.0) * 6.0;
                            S[101 + 4 * j + l] = sjl;
                        }
                }
                __syncthreads();
                // coefficients: 16 threads per tet
                {
                    const int tl = threadIdx.x >> 4, part = threadIdx.x & 15;
                    if (tl < ns) {
                        const double* S = ST + tl * kPgStage;
                        double* co = CO + tl * kPgCo;
                        const double s120 = S[36] / 120.0;
                        for (int j = part; j < kPgCo; j += 16) {
                            double val;
                            if (j < 64) {  // A_h4 rows: (a b, corner l)
                                const int ab = j >> 2, l = j & 3, a = ab >> 2, b = ab & 3;
                                const double la = S[4 * l + a], lb = S[4 * l + b];
                                val = s120 * (S[20 + ab] + la * (S[16 + b] + lb) + lb * (S[16 + a] + la));
                            } else if (j < 144) {  // b_X rows: (X a, corner l)
                                const int xa = (j - 64) >> 2, l = j & 3, X = xa >> 2, a = xa & 3;
                                const double* EX = S + 37 + 16 * X;
                                val = S[a] * EX[l] + S[4 + a] * EX[4 + l] + S[8 + a] * EX[8 + l] + S[12 + a] * EX[12 + l];
                            } else if (j < 180) {  // vertex squares: (q, corner l)
                                const int q = (j - 144) >> 2, l = j & 3;
                                val = q < 4 ? s120 * (2.0 * S[16 + q] + 4.0 * S[4 * l + q]) : S[37 + 16 * (q - 4) + 5 * l];
                            } else {  // edge products: (q, pair)
                                const int q = (j - 180) / 6, pe = (j - 180) % 6;
                                const int c1 = pe < 3 ? 0 : pe < 5 ? 1 : 2, c2 = pe < 3 ? pe + 1 : pe < 5 ? pe - 1 : 3;
                                if (q < 4) {
                                    val = 2.0 * s120 * (S[16 + q] + S[4 * c1 + q] + S[4 * c2 + q]);
                                } else {
                                    const double* EX = S + 37 + 16 * (q - 4);
                                    val = EX[4 * c1 + c2] + EX[4 * c2 + c1];
                                }
                            }
                            co[j] = val;
                        }
                    }
                }
                __syncthreads();
                // gathers into R / Q: incidences of the sub-block's tets, ascending tet
                const int thi = tb + ns;
                for (int w = threadIdx.x; w < nR + nQ; w += blockDim.x) {
                    double sum = 0.0;
                    if (w < nR) {
                        const int r = w / V, vl = w % V;
                        const int pb = pg.vinc_ptr[v0 + vl], pe = pg.vinc_ptr[v0 + vl + 1];
                        for (int p = pg_lower(pg.vinc, pb, pe, tb, 2); p < pe; ++p) {
                            const int inc = pg.vinc[p], t = inc >> 2;
                            if (t >= thi) break;
                            sum += CO[(t - tb) * kPgCo + 4 * r + (inc & 3)];
                        }
                        R[r * kPgRS + vl] = (sb == 0 ? 0.0 : R[r * kPgRS + vl]) + sum;
                    } else {
                        const int w2 = w - nR, q = w2 / (V + E), k = w2 % (V + E);
                        if (k < V) {
                            const int pb = pg.vinc_ptr[v0 + k], pe = pg.vinc_ptr[v0 + k + 1];
                            for (int p = pg_lower(pg.vinc, pb, pe, tb, 2); p < pe; ++p) {
                                const int inc = pg.vinc[p], t = inc >> 2;
                                if (t >= thi) break;
                                sum += CO[(t - tb) * kPgCo + 144 + 4 * q + (inc & 3)];
                            }
                        } else {
                            const int pb = pg.einc_ptr[e0 + k - V], pe = pg.einc_ptr[e0 + k - V + 1];
                            for (int p = pg_lower(pg.einc, pb, pe, tb, 4); p < pe; ++p) {
                                const int inc = pg.einc[p], t = inc >> 4;
                                if (t >= thi) break;
                                sum += CO[(t - tb) * kPgCo + 180 + 6 * q + pg_pair((inc >> 2) & 3, inc & 3)];
                            }
                        }
                        Q[q * kPgQS + k] = (sb == 0 ? 0.0 : Q[q * kPgQS + k]) + sum;
                    }
                }
                __syncthreads();
            }
            // GEMMs, slice by slice of 32 orbitals: warp w owns n-tile w % 4 (8 orbitals) and every m-tile (5 x 8
            // linear rows, 2 x 8 quadratic rows) over the k-steps of parity w / 4, so each B fragment (an orbital
            // value, or a square / edge product of two) is formed once and feeds 5 or 2 DMMAs
#pragma unroll
            for (int sl = 0; sl < NS; ++sl) {
                for (int w = threadIdx.x; w < V * kPgSlice; w += blockDim.x) {
                    const int vl = w / kPgSlice, c = w % kPgSlice, col = sl * kPgSlice + c;
                    const int row = in.iidx[pg.verts[v0 + vl]];
                    PH[vl * kPgPS + c] = (row >= 0 && col < N) ? in.Phi[size_t(row) * in.ld + col] : 0.0;
                }
                __syncthreads();
                const int bcol = (warp & 3) * 8 + (lane >> 2);
                const int r8 = lane >> 2, kl = lane & 3;
                for (int k0 = 4 * (warp >> 2); k0 < V; k0 += 8) {
                    const int kk = k0 + kl;
                    const double b = kk < V ? PH[kk * kPgPS + bcol] : 0.0;
#pragma unroll
                    for (int mt = 0; mt < 5; ++mt) {
                        const int arow = mt * 8 + r8;
                        const double a = (arow < 36 && kk < V) ? R[arow * kPgRS + kk] : 0.0;
                        dmma(acc[sl][mt][0], acc[sl][mt][1], a, b);
                    }
                }
                for (int k0 = 4 * (warp >> 2); k0 < V + E; k0 += 8) {
                    const int kk = k0 + kl;
                    double b = 0.0;
                    if (kk < V) {
                        const double p = PH[kk * kPgPS + bcol];
                        b = p * p;
                    } else if (kk < V + E) {
                        const int ed = ED[kk - V];
                        b = PH[(ed & 0xffff) * kPgPS + bcol] * PH[(ed >> 16) * kPgPS + bcol];
                    }
                    const double a0 = kk < V + E ? Q[r8 * kPgQS + kk] : 0.0;
                    const double a1 = (r8 == 0 && kk < V + E) ? Q[8 * kPgQS + kk] : 0.0;
                    dmma(acc[sl][5][0], acc[sl][5][1], a0, b);
                    dmma(acc[sl][6][0], acc[sl][6][1], a1, b);
                }
                __syncthreads();  // before the next slice overwrites PH
            }
        }
        // the item's ledger partials: the two k-parities of each n-tile summed in fixed order (warps w and w + 4)
        double* RED = pgs;  // reused (all staging consumed): 4 warps x NS x 7 tiles x 32 lanes x 2 <= 7168 doubles
        __syncthreads();
        if (warp >= 4) {
#pragma unroll
            for (int sl = 0; sl < NS; ++sl)
#pragma unroll
                for (int mt = 0; mt < 7; ++mt)
#pragma unroll
                    for (int j = 0; j < 2; ++j)
                        RED[((((warp - 4) * NS + sl) * 7 + mt) * 32 + lane) * 2 + j] = acc[sl][mt][j];
        }
        __syncthreads();
        if (warp < 4) {
#pragma unroll
            for (int sl = 0; sl < NS; ++sl)
#pragma unroll
                for (int mt = 0; mt < 7; ++mt) {
                    int idx;
                    const int rr = mt * 8 + (lane >> 2);
                    if (mt < 5) {
                        idx = rr;  // 0-15 A_h4, 16-35 b_H1 b_H3 b_H4 c_Hh d_phi, 36-39 pad (zero rows)
                    } else {
                        const int q = (mt - 5) * 8 + (lane >> 2);
                        idx = q < 4 ? 40 + q : q < 9 ? 44 + (q - 4) : -1;  // rhs, beta1 beta3 beta4 gamma zeta_phi
                    }
                    if (idx < 0) continue;
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const double o = acc[sl][mt][j] + RED[(((warp * NS + sl) * 7 + mt) * 32 + lane) * 2 + j];
                        const int i = sl * kPgSlice + warp * 8 + 2 * (lane & 3) + j;
                        if (i < N) part[(size_t(i) * pg.n_items + item) * kStride + idx] = o;
                    }
                }
        }
    }
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
    bool split = nch != nct;
    // the aggregated GEMM (DMMA) form is opt-in (KSB_PROJ_GEMM=1): measured slower than the staged per-tet kernel
    // (12.6 M tets, N = 120: 261 vs 57 ms; profiles/README.md r02) -- its per-chunk coefficient sums serialise
    const char* ge = std::getenv("KSB_PROJ_GEMM");  // read per call (tests switch it)
    const bool gemm = N >= kProjWideMin && N <= kPgSlice * 4 && ge && ge[0] == '1';
    const int nfun_chunk = gemm ? 1 : N + 1;  // functions written per pj chunk (the GEMM form keeps its own items)
    if (split && o.pchunk.n < int64_t(nch) * kStride * nfun_chunk) o.pchunk.alloc(int64_t(nch) * kStride * nfun_chunk);
    double* dst = split ? o.pchunk.p : o.part.p;
    ProjIn in{(const int32_t*)L.tets.p, (const int32_t*)L.iidx.p, (const int32_t*)L.anc_ptr.p,
              (const int32_t*)L.anc_tets.p, (const int32_t*)L.ctets.p, (const int32_t*)L.ciidx.p,
              (const int32_t*)L.pint_col.p, (const double*)L.xyz.p, (const double*)L.pint_val.p, eext, Phi, wt_full,
              ell_full, vxc_full, N, ld, nct, (const int32_t*)L.pj_c.p, (const int32_t*)L.pj_b.p,
              (const int32_t*)L.pj_e.p, nch};
    launch(c, "project", k_proj_shared, nch, kProjThreads, 0, in, dst);
    if (gemm) {
        // orbital blocks by the aggregated GEMM form (DMMA); the shared block by k_proj_shared above
        if (!L.pg_ready) {
            const ProjChunks P = build_proj_chunks(*L.topo);
            L.pg_item_c.upload(c, P.item_c);
            L.pg_item_ch.upload(c, P.item_ch);
            L.pg_cptr.upload(c, P.cptr);
            L.pg_ch_t.upload(c, P.ch_t);
            L.pg_ch_v.upload(c, P.ch_v);
            L.pg_ch_e.upload(c, P.ch_e);
            L.pg_tets.upload(c, P.tets);
            L.pg_verts.upload(c, P.verts);
            L.pg_edges.upload(c, P.edges);
            L.pg_vinc_ptr.upload(c, P.vinc_ptr);
            L.pg_vinc.upload(c, P.vinc);
            L.pg_einc_ptr.upload(c, P.einc_ptr);
            L.pg_einc.upload(c, P.einc);
            L.pg_items = int(P.item_c.size());
            KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
            L.pg_ready = true;
        }
        if (split)
            launch(c, "project", k_proj_fold, c.sm_count * 8, 256, 0, nct, 1, nch, (const int32_t*)L.pj_ptr.p,
                   (const double*)o.pchunk.p, o.part.p);
        const int64_t need = int64_t(N) * L.pg_items * kStride;
        if (o.pgpart.n < need) o.pgpart.alloc(need);
        PgIn pg{(const int32_t*)L.pg_item_c.p, (const int32_t*)L.pg_item_ch.p, (const int32_t*)L.pg_ch_t.p,
                (const int32_t*)L.pg_ch_v.p, (const int32_t*)L.pg_ch_e.p, (const int32_t*)L.pg_tets.p,
                (const int32_t*)L.pg_verts.p, (const int32_t*)L.pg_edges.p, (const int32_t*)L.pg_vinc_ptr.p,
                (const int32_t*)L.pg_vinc.p, (const int32_t*)L.pg_einc_ptr.p, (const int32_t*)L.pg_einc.p, L.pg_items};
        auto go = [&](auto kern) {
            static std::map<const void*, bool> attr;
            if (!attr[reinterpret_cast<const void*>(kern)]) {
                KSB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPgSmem)));
                attr[reinterpret_cast<const void*>(kern)] = true;
            }
            const int grid = std::max(1, std::min(L.pg_items, 2 * c.sm_count));
            launch(c, "project", kern, grid, kPgThreads, kPgSmem, in, pg, o.pgpart.p);
        };
        const int ns = (N + kPgSlice - 1) / kPgSlice;
        if (ns == 1)
            go(k_proj_gemm<1>);
        else if (ns == 2)
            go(k_proj_gemm<2>);
        else if (ns == 3)
            go(k_proj_gemm<3>);
        else
            go(k_proj_gemm<4>);
        launch(c, "project", k_proj_fold, c.sm_count * 8, 256, 0, nct, N, L.pg_items, (const int32_t*)L.pg_cptr.p,
               (const double*)o.pgpart.p, o.part.p + size_t(nct) * kStride);
        split = false;  // every record is in place
    } else if (N >= kProjWideMin) {
        const size_t smem = sizeof(double) * std::max(kWideTets * (N >= 64 ? kWideRec : kWideRec0), kProjThreads * kOrbK);
        const size_t smem_max = sizeof(double) * std::max(kWideTets * kWideRec, kProjThreads * kOrbK);
        static bool attr = false;
        if (!attr) {
            KSB_CUDA_CHECK(cudaFuncSetAttribute(k_proj_orbital_wide<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_max)));
            KSB_CUDA_CHECK(cudaFuncSetAttribute(k_proj_orbital_wide<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_max)));
            attr = true;
        }
        if (N >= 64)
            launch(c, "project", k_proj_orbital_wide<true>, dim3(nch, ceil_div(N, kProjThreads)), kProjThreads, smem, in, dst);
        else
            launch(c, "project", k_proj_orbital_wide<false>, dim3(nch, ceil_div(N, kProjThreads)), kProjThreads, smem, in, dst);
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
