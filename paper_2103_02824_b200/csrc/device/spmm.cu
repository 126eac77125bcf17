// Plain K-SpMM entry (Y = (A + sigma B) X). Used by ksb_spmm and the host-side operator products.
#include "level.cuh"
#include "spmm_core.cuh"

namespace ksb {

namespace {

template <int G, int CPL, bool SHIFT>
__global__ void __launch_bounds__(256) k_spmm(int ni, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                              const double* __restrict__ A, const double* __restrict__ B,
                                              const double* __restrict__ sigma, const double* __restrict__ X,
                                              int ldx, double* __restrict__ Y, int ldy, int N) {
    const int lane = threadIdx.x & 31;
    const int g = lane / G, l = lane % G;
    const int gbase = g * G;
    (void)gbase;
    const int rows_per_warp = 32 / G;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int c0t = 0; c0t < N; c0t += G * CPL) {
        const int c0 = c0t + l * CPL;
        for (int base = warp * rows_per_warp; base < ni; base += nwarps * rows_per_warp) {
            const int r = base + g;
            const bool valid = r < ni;
            double acc[CPL], accB[CPL];
            row_product<G, CPL, SHIFT>(valid ? r : 0, valid ? __ldg(ptr + r) : 0, valid ? __ldg(ptr + r + 1) : 0, col,
                                       A, B, X, ldx, c0, N, l, gbase, acc, accB);
            if (!valid) continue;
            if (SHIFT) {
#pragma unroll
                for (int q = 0; q < CPL; ++q)
                    if (c0 + q < N) acc[q] += __ldg(sigma + c0 + q) * accB[q];
            }
            if (c0 < N) store_cols<CPL>(Y + size_t(r) * ldy + c0, c0, N, acc);
        }
    }
}

/// single-vector SpMV: G lanes per row split the nonzeros, then a group shuffle reduction
template <int G, bool SHIFT>
__global__ void __launch_bounds__(256) k_spmv(int ni, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                              const double* __restrict__ A, const double* __restrict__ B,
                                              const double* __restrict__ sigma, const double* __restrict__ X,
                                              int ldx, double* __restrict__ Y, int ldy) {
    const int lane = threadIdx.x & 31;
    const int g = lane / G, l = lane % G;
    const int gbase = g * G;
    (void)gbase;
    const int rows_per_warp = 32 / G;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const double s = SHIFT ? sigma[0] : 0.0;
    for (int base = warp * rows_per_warp; base < ni; base += nwarps * rows_per_warp) {
        const int r = base + g;
        const bool valid = r < ni;
        const int rb = valid ? __ldg(ptr + r) : 0, re = valid ? __ldg(ptr + r + 1) : 0;
        double acc = 0.0, accB = 0.0;
        row_split<G, SHIFT>(rb, re, col, A, B, X, ldx, l, acc, accB);
        if (valid && l == 0) Y[size_t(r) * ldy] = SHIFT ? acc + s * accB : acc;
    }
}

template <int G, int CPL, bool SHIFT>
void run_spmm(Ctx& c, const Level& L, const double* A, const double* B, const double* sigma, const double* X,
              int N, int ldx, double* Y, int ldy) {
    const int rows_per_block = 256 / G;
    const int64_t want = (int64_t(L.ni) + rows_per_block - 1) / rows_per_block;
    const int grid = int(std::min<int64_t>(want, resident_grid(c, k_spmm<G, CPL, SHIFT>, 256, 0)));
    launch(c, "spmm", k_spmm<G, CPL, SHIFT>, std::max(grid, 1), 256, 0, L.ni, (const int32_t*)L.ii_ptr.p,
           (const int32_t*)L.ii_col.p, A, B, sigma, X, ldx, Y, ldy, N);
}

template <bool SHIFT>
void dispatch(Ctx& c, const Level& L, const double* A, const double* B, const double* sigma, const double* X,
              int N, int ldx, double* Y, int ldy) {
    if (N == 1) {
        const int64_t want = (int64_t(L.ni) + 31) / 32;
        const int grid = int(std::min<int64_t>(want, int64_t(c.sm_count) * 8));
        launch(c, "spmm", k_spmv<8, SHIFT>, std::max(grid, 1), 256, 0, L.ni, (const int32_t*)L.ii_ptr.p,
               (const int32_t*)L.ii_col.p, A, B, sigma, X, ldx, Y, ldy);
    } else if (N <= 4) {
        run_spmm<2, 2, SHIFT>(c, L, A, B, sigma, X, N, ldx, Y, ldy);
    } else if (N <= 8) {
        run_spmm<2, 4, SHIFT>(c, L, A, B, sigma, X, N, ldx, Y, ldy);
    } else if (N <= 16) {
        run_spmm<4, 4, SHIFT>(c, L, A, B, sigma, X, N, ldx, Y, ldy);
    } else if (N <= 32) {
        run_spmm<8, 4, SHIFT>(c, L, A, B, sigma, X, N, ldx, Y, ldy);
    } else if (N <= 64) {
        run_spmm<16, 4, SHIFT>(c, L, A, B, sigma, X, N, ldx, Y, ldy);
    } else {
        run_spmm<32, 4, SHIFT>(c, L, A, B, sigma, X, N, ldx, Y, ldy);
    }
}

} // namespace

void spmm(Ctx& c, const Level& L, const double* A, const double* B, const double* d_sigma, const double* X, int N,
          int ldx, double* Y, int ldy) {
    if (N < 1) raise(KSB_INVALID_ARGUMENT, "N must be >= 1");
    if (N > 1 && ((ldx & 1) || (ldy & 1))) raise(KSB_INVALID_ARGUMENT, "ld must be even for N > 1");
    if (ldx < N || ldy < N) raise(KSB_INVALID_ARGUMENT, "ld smaller than N");
    if (B)
        dispatch<true>(c, L, A, B, d_sigma, X, N, ldx, Y, ldy);
    else
        dispatch<false>(c, L, A, nullptr, nullptr, X, N, ldx, Y, ldy);
}

} // namespace ksb
