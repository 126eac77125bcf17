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

/// Column of slot q of lane l in the FULL layout: pairs are interleaved across the G lanes, so each
/// 16-byte load instruction of a lane group reads 16*G contiguous bytes (whole sectors) of a row.
template <int G>
__device__ __forceinline__ int full_col(int l, int q) {
    return 2 * ((q >> 1) * G + l) + (q & 1);
}

/// FULL layout modes: 1 = every slot in range (N == G*CPL); 2 = tail mask (N < G*CPL): a column pair is
/// skipped when it starts at or beyond N. A pair straddling N (odd N) touches column N, which lies inside the
/// even leading dimension and is never consumed. 3 = quad layout, every slot in range: lane l owns the
/// 32-byte column quads l, l+G, ... and reads each with one 256-bit load (sm_100 LDG.256), so a group of
/// G = 4 lanes reads a 128-byte row in one instruction and a warp covers 8 rows per gather.
__device__ __forceinline__ bool pair_ok(int FULLMODE, int c, int N) { return FULLMODE != 2 || c < N; }

/// Column of slot q of lane l for FULL mode FM (see full_col / the quad layout above)
template <int G, int FM>
__device__ __forceinline__ int lay_col(int l, int q) {
    if constexpr (FM == 3)
        return 4 * ((q >> 2) * G + l) + (q & 3);
    else
        return full_col<G>(l, q);
}

/// 256-bit read-only load of 4 doubles (p 32-byte aligned)
__device__ __forceinline__ void ldg4(const double* p, double& a, double& b, double& c, double& d) {
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
                 : "l"(p));
}

/// 256-bit store of 4 doubles (p 32-byte aligned)
__device__ __forceinline__ void stg4(double* p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

/// L2 eviction-priority policies (wide SpMM: gathered rows evict-last, streamed matrix / output evict-first)
__device__ __forceinline__ uint64_t l2_policy_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ldg2_hint(const double* p, uint64_t pol) {
    double2 a;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(a.x), "=d"(a.y) : "l"(p), "l"(pol));
    return a;
}
template <typename T>
__device__ __forceinline__ T ldg_first(const T* p, uint64_t pol);
template <>
__device__ __forceinline__ double ldg_first<double>(const double* p, uint64_t pol) {
    double a;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(a) : "l"(p), "l"(pol));
    return a;
}
template <>
__device__ __forceinline__ int32_t ldg_first<int32_t>(const int32_t* p, uint64_t pol) {
    int32_t a;
    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(a) : "l"(p), "l"(pol));
    return a;
}

/// p points at the row start; loads lane l's CPL columns in the FULL layout
template <int G, int CPL, int FM = 1>
__device__ __forceinline__ void load_full(const double* __restrict__ p, int l, int N, double (&x)[CPL]) {
    if constexpr (FM == 3) {
        static_assert(CPL % 4 == 0, "quad layout needs CPL % 4 == 0");
#pragma unroll
        for (int k = 0; k < CPL; k += 4) ldg4(p + lay_col<G, 3>(l, k), x[k], x[k + 1], x[k + 2], x[k + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < CPL; k += 2) {
            double2 a = make_double2(0.0, 0.0);
            if (pair_ok(FM, full_col<G>(l, k), N)) {
                if constexpr (G >= 16)
                    a = ldg2_hint(p + full_col<G>(l, k), l2_policy_last());
                else
                    a = __ldg(reinterpret_cast<const double2*>(p + full_col<G>(l, k)));
            }
            x[k] = a.x;
            x[k + 1] = a.y;
        }
    }
}

template <int G, int CPL, int FM = 1>
__device__ __forceinline__ void store_full(double* __restrict__ p, int l, int N, const double (&y)[CPL]) {
    if constexpr (FM == 3) {
#pragma unroll
        for (int k = 0; k < CPL; k += 4) stg4(p + lay_col<G, 3>(l, k), y[k], y[k + 1], y[k + 2], y[k + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < CPL; k += 2)
            if (pair_ok(FM, full_col<G>(l, k), N)) {
                if constexpr (G >= 16)
                    __stcs(reinterpret_cast<double2*>(p + full_col<G>(l, k)), make_double2(y[k], y[k + 1]));
                else
                    *reinterpret_cast<double2*>(p + full_col<G>(l, k)) = make_double2(y[k], y[k + 1]);
            }
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

/// Row product for one CSR row per lane group: acc = sum_k A_k X[col_k], accB = sum_k B_k X[col_k].
/// Control flow is warp-uniform: every group of the warp runs max-over-the-warp chunks, exhausted
/// (or invalid) rows gather their own X row with weight 0. Shuffles therefore use the full mask and
/// compile to plain SHFL without divergence bookkeeping.
/// FULL (nonzero): interleaved pair layout; 1 = every lane's CPL columns in range (N == G*CPL), no bounds logic
/// in the gather loop; 2 = with the pair tail mask.
/// Slot blocks beyond the warp's longest row are skipped (warp-uniform), so wide groups (G = 32) on short rows
/// do not gather padding slots.
template <int G, int CPL, bool SHIFT, int FULL = 0>
__device__ __forceinline__ void row_product(int r, int rb, int re, const int32_t* __restrict__ col,
                                            const double* __restrict__ A, const double* __restrict__ B,
                                            const double* __restrict__ X, int ldx, int c0, int N, int l,
                                            int gbase, double (&acc)[CPL], double (&accB)[CPL],
                                            unsigned need = ~0u) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) acc[k] = accB[k] = 0.0;
    constexpr int NB = (G >= 16) ? 1 : 16 / G;
    constexpr int UB = (G < 16 / CPL) ? G : 16 / CPL;
    const int wmax = __reduce_max_sync(0xffffffffu, re - rb);
    for (int k0 = 0; k0 < wmax; k0 += G * NB) {
        int mc[NB];
        double ma[NB], mb[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int k = rb + k0 + b * G + l;
            mc[b] = r;
            ma[b] = 0.0;
            mb[b] = 0.0;
            if (k < re) {
                mc[b] = __ldg(col + k);
                ma[b] = __ldg(A + k);
                if (SHIFT) mb[b] = __ldg(B + k);
            }
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            if (k0 + b * G >= wmax) break;
#pragma unroll
            for (int s0 = 0; s0 < G; s0 += UB) {
                if (s0 > 0 && k0 + b * G + s0 >= wmax) break;
                double x[UB][CPL];
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                    const int j = __shfl_sync(0xffffffffu, mc[b], gbase + s0 + u);
                    if (FULL == 3) {
                        // need: bit k = quad k is wanted
#pragma unroll
                        for (int k = 0; k < CPL; k += 4) {
                            x[u][k] = x[u][k + 1] = x[u][k + 2] = x[u][k + 3] = 0.0;
                            if ((need >> (k >> 2)) & 1u)
                                ldg4(X + size_t(j) * ldx + lay_col<G, 3>(l, k), x[u][k], x[u][k + 1], x[u][k + 2],
                                     x[u][k + 3]);
                        }
                    } else if (FULL) {
                        // need: bit k of a FULL lane = its column pair k is wanted (skipped pairs read nothing)
#pragma unroll
                        for (int k = 0; k < CPL; k += 2) {
                            double2 a = make_double2(0.0, 0.0);
                            if (((need >> (k >> 1)) & 1u) && pair_ok(FULL, full_col<G>(l, k), N))
                                a = __ldg(reinterpret_cast<const double2*>(X + size_t(j) * ldx + full_col<G>(l, k)));
                            x[u][k] = a.x;
                            x[u][k + 1] = a.y;
                        }
                    } else if (need & 1u) {
                        load_cols<CPL>(X + size_t(j) * ldx + c0, c0, N, x[u]);
                    } else {
#pragma unroll
                        for (int k = 0; k < CPL; ++k) x[u][k] = 0.0;
                    }
                }
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                    const double a = __shfl_sync(0xffffffffu, ma[b], gbase + s0 + u);
                    double bb = 0.0;
                    if (SHIFT) bb = __shfl_sync(0xffffffffu, mb[b], gbase + s0 + u);
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        acc[q] = fma(a, x[u][q], acc[q]);
                        if (SHIFT) accB[q] = fma(bb, x[u][q], accB[q]);
                    }
                }
            }
        }
    }
}

/// First super-chunk of a row's (col, val) pairs, loaded one row tile ahead of its use.
template <int G, bool SHIFT>
struct RowChunk {
    static constexpr int NB = (G >= 16) ? 1 : 16 / G;
    int rb, re;
    int mc[NB];
    double ma[NB], mb[NB];
    __device__ __forceinline__ void load(int r, int rb_, int re_, int l, const int32_t* __restrict__ col,
                                         const double* __restrict__ A, const double* __restrict__ B) {
        rb = rb_;
        re = re_;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int k = rb + b * G + l;
            mc[b] = r;
            ma[b] = 0.0;
            mb[b] = 0.0;
            if (k < re) {
                if constexpr (G >= 16) {
                    const uint64_t pf = l2_policy_first();
                    mc[b] = ldg_first(col + k, pf);
                    ma[b] = ldg_first(A + k, pf);
                    if (SHIFT) mb[b] = ldg_first(B + k, pf);
                } else {
                    mc[b] = __ldg(col + k);
                    ma[b] = __ldg(A + k);
                    if (SHIFT) mb[b] = __ldg(B + k);
                }
            }
        }
    }
};

/// Row product with the first super-chunk already in registers (software-pipelined across row tiles);
/// further super-chunks (rows longer than NB*G entries, adaptive meshes) are loaded in place.
/// The super-chunk's NB*G slots are walked as one flat sequence in batches of UB gathers in flight per lane
/// (quad layout: 8 x 32 bytes; otherwise 16 doubles' worth).
template <int G, int CPL, bool SHIFT, int FULL>
__device__ __forceinline__ void row_product_pf(int r, RowChunk<G, SHIFT>& ch, const int32_t* __restrict__ col,
                                               const double* __restrict__ A, const double* __restrict__ B,
                                               const double* __restrict__ X, int ldx, int c0, int N, int l, int gbase,
                                               double (&acc)[CPL], double (&accB)[CPL]) {
    constexpr int NB = RowChunk<G, SHIFT>::NB;
    constexpr int SL = NB * G;
    constexpr int UB0 = (G < 16 / CPL) ? G : 16 / CPL;
    constexpr int UB = (FULL == 3) ? (SL < 8 ? SL : 8) : UB0;
#pragma unroll
    for (int k = 0; k < CPL; ++k) acc[k] = accB[k] = 0.0;
    const int wmax = __reduce_max_sync(0xffffffffu, ch.re - ch.rb);
    for (int k0 = 0; k0 < wmax; k0 += SL) {
        if (k0 > 0) ch.load(r, ch.rb + SL, ch.re, l, col, A, B);  // rows longer than one super-chunk
#pragma unroll
        for (int s0 = 0; s0 < SL; s0 += UB) {
            if (s0 > 0 && k0 + s0 >= wmax) break;
            double x[UB][CPL];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int j = __shfl_sync(0xffffffffu, ch.mc[(s0 + u) / G], gbase + (s0 + u) % G);
                if (FULL)
                    load_full<G, CPL, FULL>(X + size_t(j) * ldx, l, N, x[u]);
                else
                    load_cols<CPL>(X + size_t(j) * ldx + c0, c0, N, x[u]);
            }
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const double a = __shfl_sync(0xffffffffu, ch.ma[(s0 + u) / G], gbase + (s0 + u) % G);
                double bb = 0.0;
                if (SHIFT) bb = __shfl_sync(0xffffffffu, ch.mb[(s0 + u) / G], gbase + (s0 + u) % G);
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    acc[q] = fma(a, x[u][q], acc[q]);
                    if (SHIFT) accB[q] = fma(bb, x[u][q], accB[q]);
                }
            }
        }
    }
}

/// N == 1: G lanes split a row's nonzeros, warp-uniform trip count, full-mask reduction
template <int G, bool SHIFT>
__device__ __forceinline__ void row_split(int rb, int re, const int32_t* __restrict__ col,
                                          const double* __restrict__ A, const double* __restrict__ B,
                                          const double* __restrict__ X, int ldx, int l, double& acc, double& accB) {
    const int wmax = __reduce_max_sync(0xffffffffu, re - rb);
    double a = 0.0, b = 0.0;
    for (int k0 = 0; k0 < wmax; k0 += G) {
        const int k = rb + k0 + l;
        if (k < re) {
            const double x = __ldg(X + size_t(__ldg(col + k)) * ldx);
            a = fma(__ldg(A + k), x, a);
            if (SHIFT) b = fma(__ldg(B + k), x, b);
        }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        if (SHIFT) b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    acc = a;
    accB = b;
}

} // namespace ksb
