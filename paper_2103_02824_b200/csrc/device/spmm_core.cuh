// K-SpMM core: CSR (interior block) x row-major dense block, FP64.
//
// G lanes cooperate on one CSR row; lane l owns CPL consecutive columns of the
// N-column block, so the gathered X row (N contiguous doubles) is read with
// CPL-wide vector loads, coalesced across the G lanes. The G lanes first load G
// (col, val) pairs cooperatively (coalesced) and broadcast them with shuffles.
// Optional second value array B on the same pattern gives the per-column
// shifted operator (A + sigma_j B) used by the level-shift ladder
// (reference proj/src/correction.cpp:50-61). Epilogues fuse the CG dot products.
#pragma once

#include "common.cuh"

namespace ksb {

template <int CPL>
struct VecD {
    double v[CPL];
};

template <int CPL>
__device__ __forceinline__ void load_cols(const double* __restrict__ p, int c0, int N, double (&x)[CPL]) {
    if (c0 + CPL <= N) {
        if constexpr (CPL == 1) {
            x[0] = __ldg(p);
        } else if constexpr (CPL == 2) {
            const double2 a = __ldg(reinterpret_cast<const double2*>(p));
            x[0] = a.x;
            x[1] = a.y;
        } else {
            const double2 a = __ldg(reinterpret_cast<const double2*>(p));
            const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
            x[0] = a.x;
            x[1] = a.y;
            x[2] = b.x;
            x[3] = b.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k < CPL; ++k) x[k] = (c0 + k < N) ? __ldg(p + k) : 0.0;
    }
}

template <int CPL>
__device__ __forceinline__ void load_full(const double* __restrict__ p, double (&x)[CPL]) {
#pragma unroll
    for (int k = 0; k < CPL; k += 2) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(p + k));
        x[k] = a.x;
        x[k + 1] = a.y;
    }
}

template <int CPL>
__device__ __forceinline__ void store_cols(double* __restrict__ p, int c0, int N, const double (&y)[CPL]) {
    if (c0 + CPL <= N) {
        if constexpr (CPL == 1) {
            p[0] = y[0];
        } else if constexpr (CPL == 2) {
            *reinterpret_cast<double2*>(p) = make_double2(y[0], y[1]);
        } else {
            reinterpret_cast<double2*>(p)[0] = make_double2(y[0], y[1]);
            reinterpret_cast<double2*>(p)[1] = make_double2(y[2], y[3]);
        }
    } else {
#pragma unroll
        for (int k = 0; k < CPL; ++k)
            if (c0 + k < N) p[k] = y[k];
    }
}

/// Row product for one CSR row: acc = sum_k A_k X[col_k], accB = sum_k B_k X[col_k].
/// FULL: every lane's CPL columns are in range (N == G*CPL), no bounds logic in the gather loop.
/// Lanes past the row end gather the row's own X row with weight 0, so every chunk issues the
/// same unpredicated load sequence.
template <int G, int CPL, bool SHIFT, bool FULL = false>
__device__ __forceinline__ void row_product(int r, int rb, int re, const int32_t* __restrict__ col,
                                            const double* __restrict__ A, const double* __restrict__ B,
                                            const double* __restrict__ X, int ldx, int c0, int N, int l,
                                            unsigned gmask, int gbase, double (&acc)[CPL], double (&accB)[CPL]) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) acc[k] = accB[k] = 0.0;
    constexpr int UB = (G < 16 / CPL) ? G : 16 / CPL;
    for (int k0 = rb; k0 < re; k0 += G) {
        const int k = k0 + l;
        int mc = r;
        double ma = 0.0, mb = 0.0;
        if (k < re) {
            mc = __ldg(col + k);
            ma = __ldg(A + k);
            if (SHIFT) mb = __ldg(B + k);
        }
        const int cnt = min(G, re - k0);
#pragma unroll
        for (int s0 = 0; s0 < G; s0 += UB) {
            if (s0 >= cnt) break;
            double x[UB][CPL];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int j = __shfl_sync(gmask, mc, gbase + s0 + u);
                if (FULL)
                    load_full<CPL>(X + size_t(j) * ldx + c0, x[u]);
                else
                    load_cols<CPL>(X + size_t(j) * ldx + c0, c0, N, x[u]);
            }
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const double a = __shfl_sync(gmask, ma, gbase + s0 + u);
                double b = 0.0;
                if (SHIFT) b = __shfl_sync(gmask, mb, gbase + s0 + u);
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    acc[q] = fma(a, x[u][q], acc[q]);
                    if (SHIFT) accB[q] = fma(b, x[u][q], accB[q]);
                }
            }
        }
    }
}

} // namespace ksb
