// Per-tet geometry, the 11-point Keast rule in constant memory, LDA/X-alpha functionals,
// and deterministic block/grid reductions shared by the physics kernels.
#pragma once

#include <cmath>

#include "common.cuh"

namespace ksb {

namespace {
// Keast degree-4 rule (reference proj/src/quadrature.cpp:9-36); one copy per translation unit.
__constant__ double g_qw[11];
__constant__ double g_qb[11][4];
bool g_rule_ready = false;

void ensure_rule(cudaStream_t s) {
    if (g_rule_ready) return;
    double w[11], b[11][4];
    const double a = 1.0 / 14.0;
    const double b1 = 0.25 * (1.0 + std::sqrt(5.0 / 14.0)), b2 = 0.25 * (1.0 - std::sqrt(5.0 / 14.0));
    int q = 0;
    w[q] = -444.0 / 5625.0;
    for (int k = 0; k < 4; ++k) b[q][k] = 0.25;
    ++q;
    for (int k = 0; k < 4; ++k, ++q) {
        w[q] = 6.0 * 343.0 / 45000.0;
        for (int j = 0; j < 4; ++j) b[q][j] = a;
        b[q][k] = 1.0 - 3.0 * a;
    }
    const int pr[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    for (int p = 0; p < 6; ++p, ++q) {
        w[q] = 6.0 * 56.0 / 2250.0;
        for (int j = 0; j < 4; ++j) b[q][j] = b2;
        b[q][pr[p][0]] = b1;
        b[q][pr[p][1]] = b1;
    }
    KSB_CUDA_CHECK(cudaMemcpyToSymbolAsync(g_qw, w, sizeof w, 0, cudaMemcpyHostToDevice, s));
    KSB_CUDA_CHECK(cudaMemcpyToSymbolAsync(g_qb, b, sizeof b, 0, cudaMemcpyHostToDevice, s));
    KSB_CUDA_CHECK(cudaStreamSynchronize(s));
    g_rule_ready = true;
}
}  // namespace

struct TetG {
    double x[4][3];
    double g[4][3];
    double vol;  // |det J| / 6
};

__device__ __forceinline__ void tet_geometry(const double* __restrict__ xyz, int4 v, TetG& G) {
    const int vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int d = 0; d < 3; ++d) G.x[i][d] = xyz[3 * vv[i] + d];
    double c[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) c[k][d] = G.x[k + 1][d] - G.x[0][d];
    double r[3][3];
    r[0][0] = c[1][1] * c[2][2] - c[1][2] * c[2][1];
    r[0][1] = c[1][2] * c[2][0] - c[1][0] * c[2][2];
    r[0][2] = c[1][0] * c[2][1] - c[1][1] * c[2][0];
    r[1][0] = c[2][1] * c[0][2] - c[2][2] * c[0][1];
    r[1][1] = c[2][2] * c[0][0] - c[2][0] * c[0][2];
    r[1][2] = c[2][0] * c[0][1] - c[2][1] * c[0][0];
    r[2][0] = c[0][1] * c[1][2] - c[0][2] * c[1][1];
    r[2][1] = c[0][2] * c[1][0] - c[0][0] * c[1][2];
    r[2][2] = c[0][0] * c[1][1] - c[0][1] * c[1][0];
    const double det = c[0][0] * r[0][0] + c[0][1] * r[0][1] + c[0][2] * r[0][2];
    G.vol = fabs(det) / 6.0;
    const double inv = 1.0 / det;
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) G.g[k + 1][d] = r[k][d] * inv;
#pragma unroll
    for (int d = 0; d < 3; ++d) G.g[0][d] = -(G.g[1][d] + G.g[2][d] + G.g[3][d]);
}

/// exact P1 x P1 x P1 weighted mass element: E(i,j) = |T| (1 + d_ij) (W + w_i + w_j) / 120
__device__ __forceinline__ void mass_elem(double vol, const double (&w)[4], double (&E)[4][4]) {
    const double W = w[0] + w[1] + w[2] + w[3];
    const double s = vol / 120.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) E[i][j] = s * (i == j ? 2.0 : 1.0) * (W + w[i] + w[j]);
}

struct XcParams {
    int kind;  // 0 none, 1 x-alpha, 2 LDA PZ81
    double alpha, p;
};

// reference proj/src/ks_model.cpp:57-97
__device__ __forceinline__ double pz_eps_c(double rs) {
    if (rs < 1.0) return 0.0311 * log(rs) + -0.048 + 0.0020 * rs * log(rs) + -0.0116 * rs;
    return -0.1423 / (1.0 + 1.0529 * sqrt(rs) + 0.3334 * rs);
}
__device__ __forceinline__ double pz_v_c(double rs) {
    if (rs < 1.0)
        return 0.0311 * log(rs) + (-0.048 - 0.0311 / 3.0) + (2.0 / 3.0) * 0.0020 * rs * log(rs) +
               (2.0 * -0.0116 - 0.0020) / 3.0 * rs;
    const double den = 1.0 + 1.0529 * sqrt(rs) + 0.3334 * rs;
    return pz_eps_c(rs) * (1.0 + (7.0 / 6.0) * 1.0529 * sqrt(rs) + (4.0 / 3.0) * 0.3334 * rs) / den;
}
constexpr double kPi = 3.14159265358979323846;
__device__ __forceinline__ double xc_potential(const XcParams& x, double rho) {
    if (rho < 0.0) rho = 0.0;
    if (rho == 0.0 || x.kind == 0) return 0.0;
    if (x.kind == 1) return -1.5 * x.alpha * cbrt(3.0 * rho / kPi);
    const double ex = -0.75 * cbrt(3.0 / kPi) * pow(rho, x.p);
    const double rs = cbrt(3.0 / (4.0 * kPi * rho));
    return (1.0 + x.p) * ex + pz_v_c(rs);
}
__device__ __forceinline__ double xc_energy_density(const XcParams& x, double rho) {
    if (rho < 0.0) rho = 0.0;
    if (rho == 0.0 || x.kind == 0) return 0.0;
    if (x.kind == 1) return -(9.0 / 8.0) * x.alpha * cbrt(3.0 / kPi) * pow(rho, 4.0 / 3.0);
    const double ex = -0.75 * cbrt(3.0 / kPi) * pow(rho, x.p);
    const double rs = cbrt(3.0 / (4.0 * kPi * rho));
    return (ex + pz_eps_c(rs)) * rho;
}

/// block-wide fixed-order sum of K per-thread values; result valid in threads < K of part[blockIdx*K + k]
template <int K>
__device__ __forceinline__ void block_sum_to(const double (&v)[K], double* __restrict__ part) {
    __shared__ double red[32][K];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double t[K];
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] = warp_sum(v[k]);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) red[warp][k] = t[k];
    __syncthreads();
    const int nw = blockDim.x >> 5;
    if (threadIdx.x < K) {
        double s = 0.0;
        for (int w = 0; w < nw; ++w) s += red[w][threadIdx.x];
        part[size_t(blockIdx.x) * K + threadIdx.x] = s;
    }
    __syncthreads();
}

namespace {
/// fixed-order fold of part[b*K + k] over b into out[k] (one warp per k, single block)
__global__ void k_fold(const double* __restrict__ part, int nblocks, int K, double* __restrict__ out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int k = warp; k < K; k += nw) {
        double s = 0.0;
        for (int b = lane; b < nblocks; b += 32) s += part[size_t(b) * K + k];
        s = warp_sum(s);
        if (lane == 0) out[k] = s;
    }
}
}  // namespace

} // namespace ksb
