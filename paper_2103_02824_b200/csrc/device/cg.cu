// Multi-RHS preconditioned conjugate gradients (N independent recurrences, one SpMM per iteration).
//
// Per column this is EllipticSolver::pcg (reference proj/src/solver.cpp:57-111):
//   x0 = 0; zero rhs -> converged with 0 iterations;
//   breakdown when !(p.Ap > 0) (iterations = it, residual of the current r);
//   recursive residual <= tol -> true residual b - A x; accept, or restart with p = z;
// with the reference's SGS preconditioner replaced by Jacobi (fully parallel, fused into
// the vector updates). The operator of column j is A + sigma_j B (level-shift ladder,
// proj/src/correction.cpp:36-61).
//
// Kernel schedule per iteration (all reductions fixed-order; the last block of each
// producer kernel folds the per-block partials and runs the per-column scalar logic):
//   K1 spmm_dot : Ap = (A + sigma B) p, partial p.Ap            -> alpha / breakdown
//   K2 update_r : r -= alpha Ap, partial r.r, r.z               -> rel, check flags, beta
//   K3 trueres  : (only when some column flagged) t = b - A x - alpha Ap -> converge or restart
//   K4 update_px: x += alpha p (deferred from K2: K4 reads p anyway), p = D^-1 r + beta p
// Per iteration this streams 8 column blocks through HBM outside K1 (K2: r, Ap in, r out;
// K4: x, p, r in, x, p out) instead of 9 with the textbook x/r and p passes.
#include <algorithm>
#include <map>
#include <type_traits>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "cg.cuh"
#include "spmm_core.cuh"
#include "dia.cuh"

namespace ksb {

namespace {

constexpr int kThreads = 256;
#ifndef KSB_SPMM_MINB
#define KSB_SPMM_MINB 4
#endif

enum : int { kActive = 0, kConverged = 1, kBreakdown = 2 };
enum : int { kIt = 0, kAnyCheck = 1, kTicket1 = 2, kTicket2 = 3, kTicket3 = 4, kTicket0 = 5, kNActive = 6 };

struct Cols {
    int N, ld;
    double tol;
    int fixed;
};

/// Warp -> tile sequence of the SpMM kernels: tile = warp + k * nwarps, so at any moment the whole
/// grid streams through one band of rows (sequential HBM pages for the matrix, stencil neighbours of
/// the band shared in L2). Measured on B200: 0.31 ms per cfg2 SpMM against 0.41 ms for block-
/// contiguous ranges, which spread the live rows over 592 distant bands.
struct TileWalk {
    int t0, step, tend;
    __device__ explicit TileWalk(int ntiles) {
        const int wpb = blockDim.x >> 5, wib = threadIdx.x >> 5;
        t0 = blockIdx.x * wpb + wib;
        step = gridDim.x * wpb;
        tend = ntiles;
    }
};

__device__ __forceinline__ double dinv_of(const double* dA, const double* dB, const double* sigma, int r, int c) {
    double d = dA[r];
    if (dB) d += sigma[c] * dB[r];
    return d != 0.0 ? 1.0 / d : 1.0;
}

/// Grid-wide "last block" election; the returned block folds the partials.
__device__ bool last_block(int* ticket) {
    __shared__ bool am_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int t = atomicAdd(ticket, 1);
        am_last = (t == int(gridDim.x) - 1);
    }
    __syncthreads();
    if (am_last) {
        __threadfence();
        if (threadIdx.x == 0) *ticket = 0;
    }
    return am_last;
}

/// Deterministic fold of part[b*N + c] over b for every column into out[c]. Loads are batched (8
/// independent accumulators per lane) so the fold costs one or two L2 round trips, not nblocks/32; for
/// N < 8 the columns are split over several warps each. The order is fixed by (nblocks, N, blockDim).
__device__ void fold_partials(const double* part, int nblocks, int N, double* out_smem) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    __shared__ double fold_red[32];
    const int per = N >= nw ? 1 : nw / N;  // warps per column
    for (int c0 = 0; c0 < N; c0 += nw / per) {
        const int c = c0 + warp / per, sl = warp % per;
        double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        if (c < N && warp / per < nw / per) {
            const int stride = per * 32;
            int b = sl * 32 + lane;
            for (; b + 7 * stride < nblocks; b += 8 * stride) {
#pragma unroll
                for (int u = 0; u < 8; ++u) a[u] += __ldcg(part + size_t(b + u * stride) * N + c);
            }
            for (; b < nblocks; b += stride) a[0] += __ldcg(part + size_t(b) * N + c);
        }
        double s = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
        s = warp_sum(s);
        if (per == 1) {
            if (lane == 0 && c < N) out_smem[c] = s;
        } else {
            if (lane == 0) fold_red[warp] = s;
            __syncthreads();
            if (threadIdx.x < nw / per && c0 + int(threadIdx.x) < N) {
                double t = 0.0;
                for (int k = 0; k < per; ++k) t += fold_red[threadIdx.x * per + k];
                out_smem[c0 + threadIdx.x] = t;
            }
            __syncthreads();
        }
    }
    __syncthreads();
}

/// Column-lane layout for elementwise kernels: thread -> (row offset, column), rows strided.
struct ElemMap {
    int c, r0, rstep, valid;
    __device__ ElemMap(int N) {
        const int rb = max(1, int(blockDim.x) / N);
        c = threadIdx.x % N;
        const int rl = threadIdx.x / N;
        valid = rl < rb;
        r0 = blockIdx.x * rb + rl;
        rstep = gridDim.x * rb;
    }
};

template <int V>
__device__ __forceinline__ void ldv(const double* __restrict__ p, double (&v)[V]) {
    if constexpr (V == 2) {
        const double2 a = *reinterpret_cast<const double2*>(p);
        v[0] = a.x;
        v[1] = a.y;
    } else {
        v[0] = *p;
    }
}
template <int V>
__device__ __forceinline__ void stv(double* __restrict__ p, const double (&v)[V]) {
    if constexpr (V == 2)
        *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    else
        *p = v[0];
}

/// Elementwise layout with V adjacent columns per thread (V = 2 needs N and ld even).
template <int V>
struct EMap {
    int c, r0, rstep, valid;
    __device__ EMap(int N) {
        const int np = N / V;
        const int rb = max(1, int(blockDim.x) / np);
        c = (threadIdx.x % np) * V;
        const int rl = threadIdx.x / np;
        valid = rl < rb;
        r0 = blockIdx.x * rb + rl;
        rstep = gridDim.x * rb;
    }
};

/// block reduction of per-thread column partials (EMap<V> layout) -> part[blockIdx*N + c]. When the
/// number of column groups np divides 32 the lanes of one column are combined by shuffles first (a
/// fixed xor tree), so the final per-column sum runs over the 8 warps instead of 256 / np rows.
template <int V>
__device__ void block_cols_v(const double (&v)[V], int N, double* part, double* smem) {
    const int np = N / V;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (np <= 32 && (32 % np) == 0 && (int(blockDim.x) % np) == 0) {
        double x[V];
#pragma unroll
        for (int q = 0; q < V; ++q) {
            x[q] = v[q];
            for (int o = 16; o >= np; o >>= 1) x[q] += __shfl_xor_sync(0xffffffffu, x[q], o);
        }
        if (lane < np) {
#pragma unroll
            for (int q = 0; q < V; ++q) smem[warp * N + lane * V + q] = x[q];
        }
        __syncthreads();
        if (threadIdx.x < N) {
            double s = 0.0;
            for (int k = 0; k < nw; ++k) s += smem[k * N + threadIdx.x];
            part[size_t(blockIdx.x) * N + threadIdx.x] = s;
        }
        __syncthreads();
        return;
    }
    const int rb = max(1, int(blockDim.x) / np);
    if (threadIdx.x < rb * np) {
#pragma unroll
        for (int q = 0; q < V; ++q) smem[(threadIdx.x / np) * N + (threadIdx.x % np) * V + q] = v[q];
    }
    __syncthreads();
    if (threadIdx.x < N) {
        double s = 0.0;
        for (int k = 0; k < rb; ++k) s += smem[k * N + threadIdx.x];
        part[size_t(blockIdx.x) * N + threadIdx.x] = s;
    }
    __syncthreads();
}

// ---------------- K0: init ----------------
__global__ void __launch_bounds__(kThreads) k_init(int ni, Cols cc, const double* __restrict__ B, double* __restrict__ X,
                                                   double* __restrict__ R, double* __restrict__ P, CgDev s) {
    extern __shared__ double sm[];
    const int N = cc.N, ld = cc.ld;
    ElemMap em(N);
    double bb = 0.0, rz = 0.0;
    if (em.valid)
        for (int r = em.r0; r < ni; r += em.rstep) {
            const size_t i = size_t(r) * ld + em.c;
            const double b = B[i];
            const double z = dinv_of(s.diagA, s.diagB, s.sigma, r, em.c) * b;
            X[i] = 0.0;
            R[i] = b;
            P[i] = z;
            bb += b * b;
            rz += b * z;
        }
    {
        const double b1[1] = {bb}, z1[1] = {rz};
        block_cols_v<1>(b1, N, s.part0, sm);
        block_cols_v<1>(z1, N, s.part1, sm);
    }
    if (!last_block(s.ctl + kTicket0)) return;
    fold_partials(s.part0, gridDim.x, N, sm);
    fold_partials(s.part1, gridDim.x, N, sm + N);
    if (threadIdx.x < N) {
        const int c = threadIdx.x;
        const double bn = sqrt(sm[c]);
        s.bnorm[c] = bn;
        s.rz[c] = sm[N + c];
        s.rr[c] = sm[c];
        s.alpha[c] = 0.0;
        s.beta[c] = 0.0;
        s.iters[c] = 0;
        s.check[c] = 0;
        s.nonpos[c] = 0;
        s.relres[c] = 0.0;
        s.status[c] = (bn == 0.0) ? kConverged : kActive;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        s.ctl[kIt] = 0;
        s.ctl[kAnyCheck] = 0;
        int na = 0;
        for (int c = 0; c < N; ++c) na += s.status[c] == kActive;
        s.ctl[kNActive] = na;
    }
}

// ---------------- K1 epilogue ----------------
/// Last-block alpha / breakdown logic shared by the K1 variants (part0 already holds the block partials);
/// a breakdown retires its column, so the host loop can stop once none is active.
__device__ void k1_epilogue(double* sm, int N, const Cols& cc, CgDev& s) {
    if (!last_block(s.ctl + kTicket1)) return;
    if (threadIdx.x < 2) s.ctl[8 + threadIdx.x] = 0;  // die-split tickets of the wide SpMM
    fold_partials(s.part0, gridDim.x, N, sm);
    if (threadIdx.x < N) {
        const int c = threadIdx.x;
        const double pap = sm[c];
        double al = 0.0;
        if (s.status[c] == kActive) {
            if (!(pap > 0.0)) {
                if (!cc.fixed) {
                    s.status[c] = kBreakdown;
                    s.relres[c] = sqrt(s.rr[c]) / s.bnorm[c];
                } else {
                    // benchmark mode keeps iterating on an indefinite operator: record the event, and never
                    // let a zero / non-finite curvature poison the column with inf / NaN
                    s.nonpos[c] += 1;
                    if (pap != 0.0 && isfinite(pap)) al = s.rz[c] / pap;
                }
            } else {
                al = s.rz[c] / pap;
            }
        }
        s.alpha[c] = al;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int na = 0;
        for (int c = 0; c < N; ++c) na += s.status[c] == kActive;
        s.ctl[kNActive] = na;
    }
}

// ---------------- K1: Ap = A p, alpha ----------------
template <int G, int CPL, bool SHIFT, bool SPLIT, int FULL, int MINB = KSB_SPMM_MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_dot(int ni, Cols cc, const int32_t* __restrict__ ptr,
                                                       const int32_t* __restrict__ col, const double* __restrict__ A,
                                                       const double* __restrict__ Bv, const double* __restrict__ P,
                                                       double* __restrict__ AP, CgDev s, int sync_every) {
    // sync_every > 0 (cooperative launch only): a grid barrier every sync_every tile steps keeps the blocks in
    // one band of rows, so the band's stencil window of wide X rows stays in L2 instead of being re-read
    extern __shared__ double sm[];
    const int N = cc.N, ld = cc.ld;
    const int lane = threadIdx.x & 31;
    const int g = lane / G, l = lane % G;
    const int gbase = g * G;
    const int rows_per_warp = 32 / G;
    const int c0 = SPLIT ? 0 : l * CPL;
    double pd[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) pd[q] = 0.0;
    // row tiles are software-pipelined: the (col, val) chunk of the next tile and the row pointers of
    // the tile after it are in flight while the current tile's gathers run. The wide FULL path keeps
    // its registers for 16 gathers in flight instead (PF = false).
    constexpr bool PF = !SPLIT;
    TileWalk tw((ni + rows_per_warp - 1) / rows_per_warp);
    // sync_every bits 16+: die split (cooperative launch). Blocks on the two halves of the SM id range sweep the
    // two halves of the rows as separate bands (rank within the half from an atomic ticket), so each die's L2
    // holds one band's stencil window. 1: halves by smid < nsmid / 2, 2: by smid parity.
    const int die_split = sync_every >> 16;
    sync_every &= 0xffff;
    int ksteps = (tw.tend + tw.step - 1) / tw.step;  // the same count for every warp of the grid
    if (die_split > 0 && sync_every > 0) {
        __shared__ int s_half, s_rank;
        if (threadIdx.x == 0) {
            unsigned smid, nsm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            asm volatile("mov.u32 %0, %%nsmid;" : "=r"(nsm));
            const int h = die_split == 1 ? int(smid >= nsm / 2) : int(smid & 1);
            s_half = h;
            s_rank = atomicAdd(s.ctl + 8 + h, 1);
        }
        cooperative_groups::this_grid().sync();
        const int cnt0 = *(volatile int*)(s.ctl + 8), cnt1 = *(volatile int*)(s.ctl + 9);
        const int h = s_half, rank = s_rank;
        const int nt = tw.tend, wpb = blockDim.x >> 5;
        const int t_mid = cnt1 == 0 ? nt : cnt0 == 0 ? 0 : int((int64_t(nt) * cnt0) / (cnt0 + cnt1));
        const int k0 = cnt0 > 0 ? (t_mid + cnt0 * wpb - 1) / (cnt0 * wpb) : 0;
        const int k1 = cnt1 > 0 ? (nt - t_mid + cnt1 * wpb - 1) / (cnt1 * wpb) : 0;
        ksteps = max(k0, k1);
        tw.t0 = (h ? t_mid : 0) + rank * wpb + int(threadIdx.x >> 5);
        tw.step = (h ? cnt1 : cnt0) * wpb;
        tw.tend = h ? nt : t_mid;
    }
    int t = tw.t0;
    RowChunk<G, SHIFT> cur, nxt;
    int nb_rb = 0, nb_re = 0;
    if constexpr (PF) {
        const int r0 = t * rows_per_warp + g;
        const bool v0 = t < tw.tend && r0 < ni;
        cur.load(v0 ? r0 : 0, v0 ? __ldg(ptr + r0) : 0, v0 ? __ldg(ptr + r0 + 1) : 0, l, col, A, Bv);
        const int r1 = (t + tw.step) * rows_per_warp + g;
        const bool v1 = t + tw.step < tw.tend && r1 < ni;
        nb_rb = v1 ? __ldg(ptr + r1) : 0;
        nb_re = v1 ? __ldg(ptr + r1 + 1) : 0;
    }
    for (int ks = 0; ks < ksteps; ++ks, t += tw.step) {
        if (sync_every > 0 && ks > 0 && ks % sync_every == 0) cooperative_groups::this_grid().sync();
        const int r = t * rows_per_warp + g;
        const bool valid = r < ni && t < tw.tend;
        double acc[CPL], accB[CPL];
        if constexpr (SPLIT) {
            const int rb = valid ? __ldg(ptr + r) : 0, re = valid ? __ldg(ptr + r + 1) : 0;
            row_split<G, SHIFT>(rb, re, col, A, Bv, P, ld, l, acc[0], accB[0]);
        } else if constexpr (PF) {
            const int r1 = (t + tw.step) * rows_per_warp + g;
            const bool v1 = t + tw.step < tw.tend && r1 < ni;
            nxt.load(v1 ? r1 : 0, nb_rb, nb_re, l, col, A, Bv);
            const int r2 = (t + 2 * tw.step) * rows_per_warp + g;
            const bool v2 = t + 2 * tw.step < tw.tend && r2 < ni;
            nb_rb = v2 ? __ldg(ptr + r2) : 0;
            nb_re = v2 ? __ldg(ptr + r2 + 1) : 0;
            row_product_pf<G, CPL, SHIFT, FULL>(valid ? r : 0, cur, col, A, Bv, P, ld, c0, N, l, gbase, acc, accB);
            cur = nxt;
        } else {
            cur.load(valid ? r : 0, valid ? __ldg(ptr + r) : 0, valid ? __ldg(ptr + r + 1) : 0, l, col, A, Bv);
            row_product_pf<G, CPL, SHIFT, FULL>(valid ? r : 0, cur, col, A, Bv, P, ld, c0, N, l, gbase, acc, accB);
        }
        if (valid && (!SPLIT || l == 0)) {
            if constexpr (FULL) {
                if (SHIFT) {
#pragma unroll
                    for (int q = 0; q < CPL; ++q)
                        if (FULL != 2 || lay_col<G, FULL>(l, q) < N) acc[q] = fma(s.sigma[lay_col<G, FULL>(l, q)], accB[q], acc[q]);
                }
                double p[CPL];
                load_full<G, CPL, FULL>(P + size_t(r) * ld, l, N, p);
                store_full<G, CPL, FULL>(AP + size_t(r) * ld, l, N, acc);
#pragma unroll
                for (int q = 0; q < CPL; ++q) pd[q] = fma(p[q], acc[q], pd[q]);
            } else {
                if (SHIFT) {
#pragma unroll
                    for (int q = 0; q < CPL; ++q)
                        if (c0 + q < N) acc[q] = fma(s.sigma[c0 + q], accB[q], acc[q]);
                }
                if (c0 < N) {
                    double p[CPL];
                    load_cols<CPL>(P + size_t(r) * ld + c0, c0, N, p);
                    store_cols<CPL>(AP + size_t(r) * ld + c0, c0, N, acc);
#pragma unroll
                    for (int q = 0; q < CPL; ++q) pd[q] = fma(p[q], acc[q], pd[q]);
                }
            }
        }
    }
    // block reduce: groups with equal l hold the same columns -- xor tree over the groups of a warp,
    // then a fixed-order sum over the warps
    const int width = G * CPL;
    const int nwb = blockDim.x >> 5, wib = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
        for (int o = 16; o >= G; o >>= 1) pd[q] += __shfl_xor_sync(0xffffffffu, pd[q], o);
    if (lane < G) {
#pragma unroll
        for (int q = 0; q < CPL; ++q) sm[wib * width + (FULL ? lay_col<G, FULL>(l, q) : l * CPL + q)] = pd[q];
    }
    __syncthreads();
    if (threadIdx.x < N) {
        double t = 0.0;
        for (int k = 0; k < nwb; ++k) t += sm[k * width + threadIdx.x];
        s.part0[size_t(blockIdx.x) * N + threadIdx.x] = t;
    }
    k1_epilogue(sm, N, cc, s);
}

// ---------------- K1 (streamed quad variant): a continuous gather pipeline across row tiles ----------------
/// Quad layout, CPL = 4, no shift. The tile's SL = NB*G slots are consumed in order from a ring of D gather
/// buffers; every consumed slot immediately refills its buffer with the gather D slots ahead -- in the current
/// tile, and past its end in the NEXT tile (whose (col, val) chunk is already in registers). So every lane keeps
/// D gathers in flight through the tile boundaries and the row epilogue, instead of draining its batch before
/// each new one (k_spmm_dot). Used when no row of the pattern is longer than SL (the host checks
/// Level::max_row_ii); same accumulation order per row as k_spmm_dot.
template <int G, int D, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_stream(int ni, Cols cc, const int32_t* __restrict__ ptr,
                                                              const int32_t* __restrict__ col,
                                                              const double* __restrict__ A, const double* __restrict__ P,
                                                              double* __restrict__ AP, CgDev s) {
    constexpr int CPL = 4;
    using Ch = RowChunk<G, false>;
    constexpr int SL = Ch::NB * G;
    static_assert(SL % D == 0, "slots per tile must be a multiple of the pipeline depth");
    extern __shared__ double sm[];
    const int N = cc.N, ld = cc.ld;
    const int lane = threadIdx.x & 31;
    const int g = lane / G, l = lane % G;
    const int gbase = g * G;
    constexpr int RPW = 32 / G;
    const int xoff = lay_col<G, 3>(l, 0);
    double pd[CPL] = {0.0, 0.0, 0.0, 0.0};
    const TileWalk tw((ni + RPW - 1) / RPW);
    const int ksteps = (tw.tend + tw.step - 1) / tw.step;
    auto chunk_of = [&](int t, Ch& ch) {
        const int r = t * RPW + g;
        const bool v = t < tw.tend && r < ni;
        ch.load(v ? r : 0, v ? __ldg(ptr + r) : 0, v ? __ldg(ptr + r + 1) : 0, l, col, A, nullptr);
        return __reduce_max_sync(0xffffffffu, ch.re - ch.rb);
    };
    // gather of slot q of chunk ch into x (predicated off past the warp's longest row)
    auto gather = [&](const Ch& ch, int w, int q, double (&x)[CPL]) {
        const int j = __shfl_sync(0xffffffffu, ch.mc[q / G], gbase + q % G);
        if (q < w)
            ldg4(P + size_t(j) * ld + xoff, x[0], x[1], x[2], x[3]);
        else
            x[0] = x[1] = x[2] = x[3] = 0.0;
    };
    int t = tw.t0;
    Ch cur, nxt;
    int wc = chunk_of(t, cur);
    int wn = chunk_of(t + tw.step, nxt);
    double x[D][CPL];
#pragma unroll
    for (int q = 0; q < D; ++q) gather(cur, wc, q, x[q]);
    for (int ks = 0; ks < ksteps; ++ks, t += tw.step) {
        const int r = t * RPW + g;
        const bool valid = r < ni && t < tw.tend;
        double acc[CPL] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < SL; ++q) {
            const int b = q % D;
            const double a = __shfl_sync(0xffffffffu, cur.ma[q / G], gbase + q % G);
#pragma unroll
            for (int k = 0; k < CPL; ++k) acc[k] = fma(a, x[b][k], acc[k]);
            if (q + D < SL)
                gather(cur, wc, q + D, x[b]);
            else
                gather(nxt, wn, q + D - SL, x[b]);
        }
        if (valid) {
            double p[CPL];
            load_full<G, CPL, 3>(P + size_t(r) * ld, l, N, p);
            store_full<G, CPL, 3>(AP + size_t(r) * ld, l, N, acc);
#pragma unroll
            for (int q = 0; q < CPL; ++q) pd[q] = fma(p[q], acc[q], pd[q]);
        }
        cur = nxt;
        wc = wn;
        wn = chunk_of(t + 2 * tw.step, nxt);
    }
    const int width = G * CPL;
    const int nwb = blockDim.x >> 5, wib = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
        for (int o = 16; o >= G; o >>= 1) pd[q] += __shfl_xor_sync(0xffffffffu, pd[q], o);
    if (lane < G) {
#pragma unroll
        for (int q = 0; q < CPL; ++q) sm[wib * width + lay_col<G, 3>(l, q)] = pd[q];
    }
    __syncthreads();
    if (threadIdx.x < N) {
        double tt = 0.0;
        for (int k = 0; k < nwb; ++k) tt += sm[k * width + threadIdx.x];
        s.part0[size_t(blockIdx.x) * N + threadIdx.x] = tt;
    }
    k1_epilogue(sm, N, cc, s);
}

// ---------------- K1 (T8 variant, N = 16): ELL-16 rows, one load per tile, continuous gather pipeline ----------------
/// The T8 view is ELL with 16 slots per row (row-major), so a warp tile of 8 rows is one contiguous 512-byte
/// column run and one 1-KB value run: lane l of row group g loads slots 4l..4l+3 of its row with one 16-byte
/// and one 32-byte load (12 L1 wavefronts per tile instead of ~60 for the scattered CSR chunk loads of
/// k_spmm_stream), one tile ahead. Slot q's (col, val) is then broadcast from lane 4g + q/4, register q%4.
/// The slot stream runs across tile boundaries as in k_spmm_stream: consume slot s, issue the gather of slot
/// s + D. Lane l owns the column quad 4l..4l+3 of the N = 16 block. Padding slots (col = -1) gather nothing.
/// Same accumulation order per row as the CSR kernels.
struct EllChunk {
    int c[4];
    double v[4];
};

template <int D>
__global__ void __launch_bounds__(kThreads, 2) k_spmm_t8(int ni, Cols cc, const int32_t* __restrict__ tcol,
                                                       const double* __restrict__ tval, const double* __restrict__ P,
                                                       double* __restrict__ AP, CgDev s) {
    constexpr int G = 4, CPL = 4, RPW = 8, SL = 16;
    static_assert(SL % D == 0, "pipeline depth");
    extern __shared__ double sm[];
    const int N = cc.N, ld = cc.ld;
    const int lane = threadIdx.x & 31;
    const int g = lane / G, l = lane % G;
    const int gbase = g * G;
    const int xoff = CPL * l;
    double pd[CPL] = {0.0, 0.0, 0.0, 0.0};
    const TileWalk tw((ni + RPW - 1) / RPW);
    const int ksteps = (tw.tend + tw.step - 1) / tw.step;
    auto chunk_of = [&](int k, EllChunk& ch) {
        const int t = tw.t0 + k * tw.step;
        const int r = t * RPW + g;
        if (t < tw.tend && r < ni) {
            const int4 c4 = __ldg(reinterpret_cast<const int4*>(tcol + size_t(r) * SL) + l);
            ch.c[0] = c4.x, ch.c[1] = c4.y, ch.c[2] = c4.z, ch.c[3] = c4.w;
            ldg4(tval + size_t(r) * SL + 4 * l, ch.v[0], ch.v[1], ch.v[2], ch.v[3]);
        } else {
            ch.c[0] = ch.c[1] = ch.c[2] = ch.c[3] = -1;
            ch.v[0] = ch.v[1] = ch.v[2] = ch.v[3] = 0.0;
        }
    };
    auto gather = [&](const EllChunk& ch, int q, double (&x)[CPL]) {
        const int j = __shfl_sync(0xffffffffu, ch.c[q % 4], gbase + q / 4);
        if (j >= 0)
            ldg4(P + size_t(j) * ld + xoff, x[0], x[1], x[2], x[3]);
        else
            x[0] = x[1] = x[2] = x[3] = 0.0;
    };
    // two chunk buffers in ping-pong (tile loop unrolled by two), so no chunk is copied between tiles
    EllChunk ca, cb;
    chunk_of(0, ca);
    chunk_of(1, cb);
    double x[D][CPL];
#pragma unroll
    for (int q = 0; q < D; ++q) gather(ca, q, x[q]);
    auto tile = [&](int k, EllChunk& cur, const EllChunk& nxt) {
        double acc[CPL] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < SL; ++q) {
            const int b = q % D;
            const double a = __shfl_sync(0xffffffffu, cur.v[q % 4], gbase + q / 4);
#pragma unroll
            for (int e = 0; e < CPL; ++e) acc[e] = fma(a, x[b][e], acc[e]);
            if (q + D < SL)
                gather(cur, q + D, x[b]);
            else
                gather(nxt, q + D - SL, x[b]);
        }
        chunk_of(k + 2, cur);
        const int t = tw.t0 + k * tw.step;
        const int r = t * RPW + g;
        if (t < tw.tend && r < ni) {
            double p[CPL];
            load_full<G, CPL, 3>(P + size_t(r) * ld, l, N, p);
            store_full<G, CPL, 3>(AP + size_t(r) * ld, l, N, acc);
#pragma unroll
            for (int e = 0; e < CPL; ++e) pd[e] = fma(p[e], acc[e], pd[e]);
        }
    };
    for (int k = 0; k < ksteps; k += 2) {
        tile(k, ca, cb);
        if (k + 1 < ksteps) tile(k + 1, cb, ca);
    }
    const int width = G * CPL;
    const int nwb = blockDim.x >> 5, wib = threadIdx.x >> 5;
#pragma unroll
    for (int e = 0; e < CPL; ++e)
        for (int o = 16; o >= G; o >>= 1) pd[e] += __shfl_xor_sync(0xffffffffu, pd[e], o);
    if (lane < G) {
#pragma unroll
        for (int e = 0; e < CPL; ++e) sm[wib * width + xoff + e] = pd[e];
    }
    __syncthreads();
    if (threadIdx.x < N) {
        double tt = 0.0;
        for (int k = 0; k < nwb; ++k) tt += sm[k * width + threadIdx.x];
        s.part0[size_t(blockIdx.x) * N + threadIdx.x] = tt;
    }
    k1_epilogue(sm, N, cc, s);
}

// ---------------- K1 (stencil variant): sliding windows over a uniform-stencil level ----------------
/// Same contract as k_spmm_dot (AP = A P and the p.Ap partials, alpha in the last block) on a level with a stencil
/// (DIA) view (dia.cuh). G lanes own one row (lane l: the CPL contiguous columns l*CPL..), a warp carries WG = 32/G
/// rows per step, each lane group walks S consecutive rows. Run q of the stencil (offsets first[q] .. first[q] +
/// len - 1) keeps its len - 1 older block rows in registers; a step gathers the one new row per run (NG loads
/// instead of D), loads the row's D values with 16-byte broadcast loads (the WG groups of the warp read one
/// contiguous run), and accumulates run by run, offsets ascending inside a run. Row indices are clamped to
/// [0, ni): an offset that leaves the block has value 0. p.Ap takes P[r] from run 0's window (offset 0).
template <int NG, int LR, int G, int CPL, int MINB, int PFD>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_dia(int ni, Cols cc, DiaGeom dg, const double* __restrict__ dval,
                                                           const double* __restrict__ P, double* __restrict__ AP,
                                                           CgDev s) {
    constexpr int L0 = 3;
    constexpr int D = L0 + (NG - 1) * LR;
    constexpr int WG = 32 / G, S = kDiaS, T = WG * S;
    constexpr int SD = (D * WG + 1) & ~1;
    constexpr int PAIRS = D / 2;
    extern __shared__ double sm[];
    const int N = cc.N, ld = cc.ld;
    const int lane = threadIdx.x & 31;
    const int g = lane / G, l = lane % G;
    const int xoff = CPL * l;
    const bool act = xoff < N;  // lanes past the block's last column idle (N % CPL == 0)
    double pd[CPL];
#pragma unroll
    for (int e = 0; e < CPL; ++e) pd[e] = 0.0;
    auto ldx = [&](int row, double (&x)[CPL]) {
        row = min(max(row, 0), ni - 1);
        const double* p = P + size_t(row) * ld + xoff;
        if (!act) {
#pragma unroll
            for (int e = 0; e < CPL; ++e) x[e] = 0.0;
        } else if constexpr (CPL == 4) {
            ldg4(p, x[0], x[1], x[2], x[3]);
        } else if constexpr (CPL == 2) {
            const double2 a = __ldg(reinterpret_cast<const double2*>(p));
            x[0] = a.x;
            x[1] = a.y;
        } else {
            x[0] = __ldg(p);
        }
    };
    // L2 prefetch PFD steps ahead of the two DRAM streams: the values (one contiguous run per step) and the
    // stencil's leading block row (offset omax: the first touch of that row in the band sweep); the other runs'
    // rows were brought in by it and hit L2
    const int omax = dg.first[NG - 1] + LR - 1;
    auto prefetch_step = [&](const double* vb, int r0g, int sp) {
        if constexpr (PFD > 0) {
            if (lane * 16 < SD)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(vb + size_t(sp) * SD + lane * 16));
            else if (l == G - 1)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(P + size_t(min(r0g + sp + omax, ni - 1)) * ld));
        }
    };
    const TileWalk tw((ni + T - 1) / T);
    for (int t = tw.t0; t < tw.tend; t += tw.step) {
        const int r0 = t * T + g * S;
        const double* vb = dval + size_t(t) * S * SD;
        if constexpr (PFD > 0) {
#pragma unroll
            for (int sp = 0; sp < PFD; ++sp) prefetch_step(vb, r0, sp);
        }
        // carried window: run 0 keeps offsets -1, 0; run q >= 1 keeps first[q] .. first[q] + LR - 2
        double w0[L0 - 1][CPL];
        double wr[NG - 1][LR - 1][CPL];
#pragma unroll
        for (int j = 0; j < L0 - 1; ++j) ldx(r0 - 1 + j, w0[j]);
#pragma unroll
        for (int q = 1; q < NG; ++q)
#pragma unroll
            for (int j = 0; j < LR - 1; ++j) ldx(r0 + dg.first[q] + j, wr[q - 1][j]);
#pragma unroll 2
        for (int st = 0; st < S; ++st) {
            const int r = r0 + st;
            const double* vs = vb + size_t(st) * SD;
            if (PFD > 0 && st + PFD < S) prefetch_step(vb, r0, st + PFD);
            double v[D];
#pragma unroll
            for (int p = 0; p < PAIRS; ++p) {
                const double2 a = __ldg(reinterpret_cast<const double2*>(vs + 2 * (p * WG + g)));
                v[2 * p] = a.x;
                v[2 * p + 1] = a.y;
            }
            if constexpr (D & 1) v[D - 1] = __ldg(vs + 2 * PAIRS * WG + g);
            double n0[CPL], nr[NG - 1][CPL];
            ldx(r + 1, n0);
#pragma unroll
            for (int q = 1; q < NG; ++q) ldx(r + dg.first[q] + LR - 1, nr[q - 1]);
            double acc[CPL];
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                double a = v[0] * w0[0][e];
                a = fma(v[1], w0[1][e], a);
                a = fma(v[2], n0[e], a);
                acc[e] = a;
            }
#pragma unroll
            for (int q = 1; q < NG; ++q) {
                const int d0 = L0 + (q - 1) * LR;
#pragma unroll
                for (int j = 0; j < LR; ++j) {
#pragma unroll
                    for (int e = 0; e < CPL; ++e)
                        acc[e] = fma(v[d0 + j], j < LR - 1 ? wr[q - 1][j][e] : nr[q - 1][e], acc[e]);
                }
            }
            if (r < ni && act) {
#pragma unroll
                for (int e = 0; e < CPL; ++e) pd[e] = fma(w0[1][e], acc[e], pd[e]);
                double* y = AP + size_t(r) * ld + xoff;
                if constexpr (CPL == 4) {
                    stg4(y, acc[0], acc[1], acc[2], acc[3]);
                } else if constexpr (CPL == 2) {
                    *reinterpret_cast<double2*>(y) = make_double2(acc[0], acc[1]);
                } else {
                    y[0] = acc[0];
                }
            }
            // slide every window by one row
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                w0[0][e] = w0[1][e];
                w0[1][e] = n0[e];
            }
#pragma unroll
            for (int q = 1; q < NG; ++q) {
#pragma unroll
                for (int j = 0; j + 1 < LR - 1; ++j)
#pragma unroll
                    for (int e = 0; e < CPL; ++e) wr[q - 1][j][e] = wr[q - 1][j + 1][e];
#pragma unroll
                for (int e = 0; e < CPL; ++e) wr[q - 1][LR - 2][e] = nr[q - 1][e];
            }
        }
    }
    // p.Ap partials: fold the WG row groups of the warp, then the warps of the block (fixed order)
    const int nwb = blockDim.x >> 5, wib = threadIdx.x >> 5;
#pragma unroll
    for (int e = 0; e < CPL; ++e)
        for (int o = 16; o >= G; o >>= 1) pd[e] += __shfl_xor_sync(0xffffffffu, pd[e], o);
    if (lane < G && act) {
#pragma unroll
        for (int e = 0; e < CPL; ++e) sm[wib * N + xoff + e] = pd[e];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
        double tt = 0.0;
        for (int k = 0; k < nwb; ++k) tt += sm[k * N + c];
        s.part0[size_t(blockIdx.x) * N + c] = tt;
    }
    __syncthreads();
    k1_epilogue(sm, N, cc, s);
}

// bulk async copy helpers (cp.async.bulk + mbarrier completion)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

constexpr int kDiaCh = 8;    // steps per value chunk of the staged stencil SpMM
constexpr int kDiaRing = 3;  // chunks in flight per warp

/// dynamic shared memory of k_spmm_dia_tv: the per-warp value rings, their barriers, the epilogue scratch
inline size_t dia_tv_smem(int D, int wg, int N) {
    const size_t ring = size_t(kThreads / 32) * kDiaRing * kDiaCh * size_t(dia_step_stride(D, wg)) * sizeof(double);
    const size_t bars = size_t(kThreads / 32) * kDiaRing * sizeof(uint64_t);
    const size_t eps = sizeof(double) * std::max<size_t>(size_t(kThreads / 32) * N, 2 * size_t(N));
    return ring + bars + eps;
}

/// k_spmm_dia with the value stream staged in shared memory: lane 0 of each warp keeps kDiaRing chunks of
/// kDiaCh steps in flight as bulk async copies (the values never occupy registers or LSU slots while in flight, and
/// their DRAM latency hides behind kDiaRing - 1 chunks of work); a step reads its values with 16-byte broadcast LDS.
/// The block rows are gathered as in k_spmm_dia. Same accumulation order.
template <int NG, int LR, int G, int CPL, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_dia_tv(int ni, Cols cc, DiaGeom dg,
                                                              const double* __restrict__ dval,
                                                              const double* __restrict__ P, double* __restrict__ AP,
                                                              CgDev s) {
    constexpr int L0 = 3;
    constexpr int D = L0 + (NG - 1) * LR;
    constexpr int WG = 32 / G, S = kDiaS, T = WG * S;
    constexpr int SD = (D * WG + 1) & ~1;
    constexpr int PAIRS = D / 2;
    constexpr int CH = kDiaCh, RING = kDiaRing, NCH = S / CH, NWB = kThreads / 32;
    static_assert(S % CH == 0, "chunking");
    extern __shared__ __align__(128) double dsm[];
    double* ring_all = dsm;
    uint64_t* bars_all = reinterpret_cast<uint64_t*>(dsm + size_t(NWB) * RING * CH * SD);
    double* sm = reinterpret_cast<double*>(bars_all + NWB * RING);
    const int N = cc.N, ld = cc.ld;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int g = lane / G, l = lane % G;
    const int xoff = CPL * l;
    const bool act = xoff < N;
    double* ring = ring_all + size_t(wib) * RING * CH * SD;
    uint64_t* bars = bars_all + wib * RING;
    double pd[CPL];
#pragma unroll
    for (int e = 0; e < CPL; ++e) pd[e] = 0.0;
    auto ldx = [&](int row, double (&x)[CPL]) {
        row = min(max(row, 0), ni - 1);
        const double* p = P + size_t(row) * ld + xoff;
        if (!act) {
#pragma unroll
            for (int e = 0; e < CPL; ++e) x[e] = 0.0;
        } else if constexpr (CPL == 4) {
            ldg4(p, x[0], x[1], x[2], x[3]);
        } else if constexpr (CPL == 2) {
            const double2 a = __ldg(reinterpret_cast<const double2*>(p));
            x[0] = a.x;
            x[1] = a.y;
        } else {
            x[0] = __ldg(p);
        }
    };
    const TileWalk tw((ni + T - 1) / T);
    const int ktiles = tw.t0 < tw.tend ? (tw.tend - tw.t0 + tw.step - 1) / tw.step : 0;
    const int nchunks = ktiles * NCH;
    auto fetch = [&](int u) {  // lane 0: chunk u of this warp's stream into slot u % RING
        if (lane == 0 && u < nchunks) {
            const int k = u / NCH, c = u % NCH;
            const size_t t = size_t(tw.t0) + size_t(k) * tw.step;
            uint64_t* bar = bars + (u % RING);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar, CH * SD * sizeof(double));
            bulk_g2s(ring + size_t(u % RING) * CH * SD, dval + (t * S + size_t(c) * CH) * SD, CH * SD * sizeof(double),
                     bar);
        }
    };
    if (lane == 0) {
        for (int i = 0; i < RING; ++i) mbar_init(bars + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < RING; ++u) fetch(u);
    int u = 0;
    for (int k = 0; k < ktiles; ++k) {
        const int t = tw.t0 + k * tw.step;
        const int r0 = t * T + g * S;
        double w0[L0 - 1][CPL];
        double wr[NG - 1][LR - 1][CPL];
#pragma unroll
        for (int j = 0; j < L0 - 1; ++j) ldx(r0 - 1 + j, w0[j]);
#pragma unroll
        for (int q = 1; q < NG; ++q)
#pragma unroll
            for (int j = 0; j < LR - 1; ++j) ldx(r0 + dg.first[q] + j, wr[q - 1][j]);
        for (int c = 0; c < NCH; ++c, ++u) {
            mbar_wait(bars + (u % RING), (u / RING) & 1);
            const double* vchunk = ring + size_t(u % RING) * CH * SD;
#pragma unroll 2
            for (int sc = 0; sc < CH; ++sc) {
                const int r = r0 + c * CH + sc;
                const double* vs = vchunk + sc * SD;
                double n0[CPL], nr[NG - 1][CPL];
                ldx(r + 1, n0);
#pragma unroll
                for (int q = 1; q < NG; ++q) ldx(r + dg.first[q] + LR - 1, nr[q - 1]);
                double v[D];
#pragma unroll
                for (int p = 0; p < PAIRS; ++p) {
                    const double2 a = *reinterpret_cast<const double2*>(vs + 2 * (p * WG + g));
                    v[2 * p] = a.x;
                    v[2 * p + 1] = a.y;
                }
                if constexpr (D & 1) v[D - 1] = vs[2 * PAIRS * WG + g];
                double acc[CPL];
#pragma unroll
                for (int e = 0; e < CPL; ++e) {
                    double a = v[0] * w0[0][e];
                    a = fma(v[1], w0[1][e], a);
                    a = fma(v[2], n0[e], a);
                    acc[e] = a;
                }
#pragma unroll
                for (int q = 1; q < NG; ++q) {
                    const int d0 = L0 + (q - 1) * LR;
#pragma unroll
                    for (int j = 0; j < LR; ++j) {
#pragma unroll
                        for (int e = 0; e < CPL; ++e)
                            acc[e] = fma(v[d0 + j], j < LR - 1 ? wr[q - 1][j][e] : nr[q - 1][e], acc[e]);
                    }
                }
                if (r < ni && act) {
#pragma unroll
                    for (int e = 0; e < CPL; ++e) pd[e] = fma(w0[1][e], acc[e], pd[e]);
                    double* y = AP + size_t(r) * ld + xoff;
                    if constexpr (CPL == 4) {
                        stg4(y, acc[0], acc[1], acc[2], acc[3]);
                    } else if constexpr (CPL == 2) {
                        *reinterpret_cast<double2*>(y) = make_double2(acc[0], acc[1]);
                    } else {
                        y[0] = acc[0];
                    }
                }
#pragma unroll
                for (int e = 0; e < CPL; ++e) {
                    w0[0][e] = w0[1][e];
                    w0[1][e] = n0[e];
                }
#pragma unroll
                for (int q = 1; q < NG; ++q) {
#pragma unroll
                    for (int j = 0; j + 1 < LR - 1; ++j)
#pragma unroll
                        for (int e = 0; e < CPL; ++e) wr[q - 1][j][e] = wr[q - 1][j + 1][e];
#pragma unroll
                    for (int e = 0; e < CPL; ++e) wr[q - 1][LR - 2][e] = nr[q - 1][e];
                }
            }
            __syncwarp();
            fetch(u + RING);  // the slot just consumed
        }
    }
    const int nwb = blockDim.x >> 5;
#pragma unroll
    for (int e = 0; e < CPL; ++e)
        for (int o = 16; o >= G; o >>= 1) pd[e] += __shfl_xor_sync(0xffffffffu, pd[e], o);
    if (lane < G && act) {
#pragma unroll
        for (int e = 0; e < CPL; ++e) sm[wib * N + xoff + e] = pd[e];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
        double tt = 0.0;
        for (int k = 0; k < nwb; ++k) tt += sm[k * N + c];
        s.part0[size_t(blockIdx.x) * N + c] = tt;
    }
    __syncthreads();
    k1_epilogue(sm, N, cc, s);
}

__device__ __forceinline__ double2 ldg2_na(const double* p) {  // streamed once: no L1 allocation
    double2 a;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(a.x), "=d"(a.y) : "l"(p));
    return a;
}
__device__ __forceinline__ double ldg1_na(const double* p) {
    double a;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(a) : "l"(p));
    return a;
}

/// z-marching stencil SpMM (N = 16) on a cubic grid level (dia.cuh line-tiled layout). A block of NW warps owns an
/// (x, y) tile of 32 x NW rows and marches it through a range of z planes; warp w takes grid line y0 + w, its 4 lane
/// groups 8 consecutive rows each, sliding the per-run windows along x as in k_spmm_dia. Marching in z keeps the
/// three planes the tile touches (z - 1, z, z + 1 with a one-row / one-line halo: ~80 KB for NW = 4) in L1, so every
/// block row comes from L2 about once per tile instead of once per stencil run (7 times for Kuhn); the values stream
/// past L1 (no allocation). Same accumulation order as k_spmm_dia.
template <int NG, int LR, int NW, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) k_spmm_dia_z(int ni, Cols cc, DiaGeom dg, int nzc,
                                                            const double* __restrict__ dval,
                                                            const double* __restrict__ P, double* __restrict__ AP,
                                                            CgDev s) {
    constexpr int G = 8, CPL = 2, SX = 8, L0 = 3;
    constexpr int D = L0 + (NG - 1) * LR;
    constexpr int SD = (D * 4 + 1) & ~1;
    constexpr int PAIRS = D / 2;
    extern __shared__ double sm[];
    const int N = cc.N, ld = cc.ld;
    const int n = dg.n, nxt = (n + 31) / 32, nyt = (n + NW - 1) / NW;
    const int zlen = (n + nzc - 1) / nzc;
    const int nwork = nxt * nyt * nzc;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int g = lane / G, l = lane % G;
    const int xoff = CPL * l;
    double pd[CPL] = {0.0, 0.0};
    auto ldx = [&](int row, double (&x)[CPL]) {
        row = min(max(row, 0), ni - 1);
        const double2 a = __ldg(reinterpret_cast<const double2*>(P + size_t(row) * ld + xoff));
        x[0] = a.x;
        x[1] = a.y;
    };
    for (int wi = blockIdx.x; wi < nwork; wi += gridDim.x) {
        const int xt = wi % nxt, yt = (wi / nxt) % nyt, zc = wi / (nxt * nyt);
        const int y = yt * NW + wib;
        if (y >= n) continue;
        const int x0 = xt * 32 + g * SX;
        const int z0 = zc * zlen, z1 = min(n, z0 + zlen);
        for (int z = z0; z < z1; ++z) {
            const int r0 = x0 + n * (y + n * z);
            const double* vb = dval + ((size_t(z) * n + y) * nxt + xt) * 8 * SD;
            double w0[L0 - 1][CPL];
            double wr[NG - 1][LR - 1][CPL];
#pragma unroll
            for (int j = 0; j < L0 - 1; ++j) ldx(r0 - 1 + j, w0[j]);
#pragma unroll
            for (int q = 1; q < NG; ++q)
#pragma unroll
                for (int j = 0; j < LR - 1; ++j) ldx(r0 + dg.first[q] + j, wr[q - 1][j]);
#pragma unroll 2
            for (int st = 0; st < SX; ++st) {
                const int r = r0 + st;
                const double* vs = vb + st * SD;
                double v[D];
#pragma unroll
                for (int p = 0; p < PAIRS; ++p) {
                    const double2 a = ldg2_na(vs + 2 * (p * 4 + g));
                    v[2 * p] = a.x;
                    v[2 * p + 1] = a.y;
                }
                if constexpr (D & 1) v[D - 1] = ldg1_na(vs + 2 * PAIRS * 4 + g);
                double n0[CPL], nr[NG - 1][CPL];
                ldx(r + 1, n0);
#pragma unroll
                for (int q = 1; q < NG; ++q) ldx(r + dg.first[q] + LR - 1, nr[q - 1]);
                double acc[CPL];
#pragma unroll
                for (int e = 0; e < CPL; ++e) {
                    double a = v[0] * w0[0][e];
                    a = fma(v[1], w0[1][e], a);
                    a = fma(v[2], n0[e], a);
                    acc[e] = a;
                }
#pragma unroll
                for (int q = 1; q < NG; ++q) {
                    const int d0 = L0 + (q - 1) * LR;
#pragma unroll
                    for (int j = 0; j < LR; ++j) {
#pragma unroll
                        for (int e = 0; e < CPL; ++e)
                            acc[e] = fma(v[d0 + j], j < LR - 1 ? wr[q - 1][j][e] : nr[q - 1][e], acc[e]);
                    }
                }
                if (x0 + st < n) {
#pragma unroll
                    for (int e = 0; e < CPL; ++e) pd[e] = fma(w0[1][e], acc[e], pd[e]);
                    *reinterpret_cast<double2*>(AP + size_t(r) * ld + xoff) = make_double2(acc[0], acc[1]);
                }
#pragma unroll
                for (int e = 0; e < CPL; ++e) {
                    w0[0][e] = w0[1][e];
                    w0[1][e] = n0[e];
                }
#pragma unroll
                for (int q = 1; q < NG; ++q) {
#pragma unroll
                    for (int j = 0; j + 1 < LR - 1; ++j)
#pragma unroll
                        for (int e = 0; e < CPL; ++e) wr[q - 1][j][e] = wr[q - 1][j + 1][e];
#pragma unroll
                    for (int e = 0; e < CPL; ++e) wr[q - 1][LR - 2][e] = nr[q - 1][e];
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < CPL; ++e)
        for (int o = 16; o >= G; o >>= 1) pd[e] += __shfl_xor_sync(0xffffffffu, pd[e], o);
    if (lane < G) {
#pragma unroll
        for (int e = 0; e < CPL; ++e) sm[wib * N + xoff + e] = pd[e];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
        double tt = 0.0;
        for (int k = 0; k < NW; ++k) tt += sm[k * N + c];
        s.part0[size_t(blockIdx.x) * N + c] = tt;
    }
    __syncthreads();
    k1_epilogue(sm, N, cc, s);
}

// ---------------- K1 (stencil, TMA-staged z-marching, N = 16): the cfg2 kernel ----------------
constexpr int kZtSlots = 4;                  // plane slots: z - 1, z, z + 1 in use, z + 2 in flight
constexpr int kZtH = kZtT + 2;               // tile plus a one-row / one-line halo
constexpr int kZtRows = kZtH * kZtH;

inline size_t dia_zt_smem(int D) {
    return sizeof(double) * (size_t(kZtSlots) * kZtRows * 16 + 2 * size_t(kZtT) * kZtT * D) + 8 * sizeof(uint64_t) +
           sizeof(double) * 8 * 16;
}

/// Stencil SpMM for an N = 16 block (ld 16) on a cubic grid level, the block's planes staged by the TMA engine. A
/// block of 8 warps owns a 16 x 16 (x, y) tile and marches it through kZtLz planes: every plane of X it touches
/// (with a one-row / one-line halo, 18 x 18 rows x 128 B) arrives in shared memory by bulk async copies (18 line
/// segments) into a ring of 4 plane slots, the tile's values by one bulk copy per plane into a ring of 2, all
/// completing on mbarriers, so the loads of plane z + 2 are in flight while plane z is computed and no register or
/// LSU slot waits on HBM. Lane group g of warp w computes 8 consecutive rows of line 2w + g / 2 with the per-run
/// sliding windows of k_spmm_dia, reading the block rows from the staged planes. Each X row leaves HBM once and L2
/// about 1.3 times (halo), instead of once per stencil run. Same accumulation order as k_spmm_dia.
template <int NG, int LR>
__global__ void __launch_bounds__(kThreads, 1) k_spmm_dia_zt(int ni, Cols cc, DiaGeom dg, int nzc,
                                                           const double* __restrict__ dval,
                                                           const double* __restrict__ P, double* __restrict__ AP,
                                                           CgDev s) {
    constexpr int L0 = 3, G = 8, CPL = 2;
    constexpr int D = L0 + (NG - 1) * LR;
    constexpr int SD = 4 * D, PAIRS = D / 2, TB = kZtT * kZtT * D;
    extern __shared__ __align__(128) double dsm[];
    double* xs = dsm;
    double* vsm = xs + size_t(kZtSlots) * kZtRows * 16;
    uint64_t* bar = reinterpret_cast<uint64_t*>(vsm + 2 * TB);  // 0..3 planes, 4..5 values
    double* sm = reinterpret_cast<double*>(bar + 8);
    const int n = dg.n, nt = (n + kZtT - 1) / kZtT, ntile = nt * nt;
    const int lz = (n + nzc - 1) / nzc;
    const int nwork = ntile * nzc;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / G, l = lane % G;
    const int xoff = CPL * l;
    const int yl = 2 * warp + g / 2, sg = g % 2;
    double pd[CPL] = {0.0, 0.0};
    // stale slot rows (halo outside the grid, never copied) must be finite: their value is 0, 0 * x must be 0
    for (int i = threadIdx.x; i < kZtSlots * kZtRows * 16; i += blockDim.x) xs[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 6; ++i) mbar_init(bar + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    // One continuous stream per block over its work items (tile, z range): load j = plane z0 - 1 + k of the item it
    // belongs to, into slot j % 4 (fill j / 4 of that slot); compute step c uses the three loads of planes z - 1, z,
    // z + 1 and value block c % 2. Loads run ahead across item boundaries, so no item starts on a cold pipeline.
    auto item_of = [&](int m, int& xt_, int& yt_, int& z0_, int& z1_) -> bool {
        const int wi = blockIdx.x + m * gridDim.x;
        if (wi >= nwork) return false;
        const int tile = wi % ntile, zc = wi / ntile;
        xt_ = tile % nt;
        yt_ = tile / nt;
        z0_ = zc * lz;
        z1_ = min(n, z0_ + lz);
        return true;
    };
    // load cursor
    int lm = 0, lp = 0, lxt = 0, lyt = 0, lz0 = 0, lz1 = 0;
    bool lvalid = item_of(0, lxt, lyt, lz0, lz1);
    while (lvalid && lz0 >= lz1) lvalid = item_of(++lm, lxt, lyt, lz0, lz1);
    if (lvalid) lp = lz0 - 1;
    int jl = 0;  // next load index
    auto issue_next = [&]() {
        if (!lvalid) return;
        const int sl = jl & 3;
        if (warp == 0) {
            const int x0 = lxt * kZtT, y0 = lyt * kZtT;
            const bool pv = lp >= 0 && lp < n;
            int lo = 0, hi = 0;
            const int y = y0 - 1 + lane;
            const int64_t start = int64_t(x0 - 1) + int64_t(n) * (int64_t(y) + int64_t(n) * lp);
            if (pv && lane < kZtH && y >= 0 && y < n) {
                lo = int(start > 0 ? start : int64_t(0));
                hi = int(start + kZtH < int64_t(ni) ? start + kZtH : int64_t(ni));
            }
            int bytes = hi > lo ? (hi - lo) * 16 * int(sizeof(double)) : 0;
            for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(bar + sl, uint32_t(bytes));
            }
            __syncwarp();
            if (hi > lo)
                bulk_g2s(xs + (size_t(sl) * kZtRows + size_t(lane) * kZtH + size_t(lo - start)) * 16,
                         P + size_t(lo) * 16, uint32_t((hi - lo) * 16 * sizeof(double)), bar + sl);
        }
        ++jl;
        if (++lp > lz1) {
            do {
                lvalid = item_of(++lm, lxt, lyt, lz0, lz1);
            } while (lvalid && lz0 >= lz1);
            if (lvalid) lp = lz0 - 1;
        }
    };
    // value cursor (one block per compute step)
    int vm = 0, vz = 0, vxt = 0, vyt = 0, vz0 = 0, vz1 = 0;
    bool vvalid = item_of(0, vxt, vyt, vz0, vz1);
    while (vvalid && vz0 >= vz1) vvalid = item_of(++vm, vxt, vyt, vz0, vz1);
    if (vvalid) vz = vz0;
    int jv = 0;
    auto issue_vals = [&]() {
        if (!vvalid) return;
        const int vb = jv & 1;
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar + 4 + vb, uint32_t(TB * sizeof(double)));
            bulk_g2s(vsm + size_t(vb) * TB, dval + ((size_t(vz) * nt + vyt) * nt + vxt) * TB,
                     uint32_t(TB * sizeof(double)), bar + 4 + vb);
        }
        ++jv;
        if (++vz >= vz1) {
            do {
                vvalid = item_of(++vm, vxt, vyt, vz0, vz1);
            } while (vvalid && vz0 >= vz1);
            if (vvalid) vz = vz0;
        }
    };
    for (int k = 0; k < 4; ++k) issue_next();
    issue_vals();
    issue_vals();
    int jbase = 0;  // load index of the current item's plane z0 - 1
    int c = 0;      // compute step
    int xt = 0, yt = 0, z0 = 0, z1 = 0;
    for (int m = 0; item_of(m, xt, yt, z0, z1); ++m) {
        if (z0 >= z1) continue;
        const int x0 = xt * kZtT, y0 = yt * kZtT;
        const int y = y0 + yl;
        const int xs0 = x0 + 8 * sg;
        for (int z = z0; z < z1; ++z, ++c) {
            const int j0 = jbase + (z - z0);  // plane z - 1
            const int vb = c & 1;
            for (int t = 0; t < 3; ++t) mbar_wait(bar + ((j0 + t) & 3), ((j0 + t) >> 2) & 1);
            mbar_wait(bar + 4 + vb, (c >> 1) & 1);
            if (y < n) {
                const int slot_of[3] = {j0 & 3, (j0 + 1) & 3, (j0 + 2) & 3};
                auto xrow = [&](int dz, int dy, int col) -> const double* {
                    return xs + (size_t(slot_of[dz + 1]) * kZtRows + size_t(yl + 1 + dy) * kZtH + col) * 16 + xoff;
                };
                auto lds = [&](const double* p, double (&x)[CPL]) {
                    const double2 a = *reinterpret_cast<const double2*>(p);
                    x[0] = a.x;
                    x[1] = a.y;
                };
                const double* vbase = vsm + size_t(vb) * TB + size_t(warp) * 8 * SD;
                double w0[L0 - 1][CPL];
                double wr[NG - 1][LR - 1][CPL];
                const int c0 = 8 * sg + 1;  // slot column of x = xs0
#pragma unroll
                for (int j = 0; j < L0 - 1; ++j) lds(xrow(0, 0, c0 - 1 + j), w0[j]);
#pragma unroll
                for (int q = 1; q < NG; ++q)
#pragma unroll
                    for (int j = 0; j < LR - 1; ++j) lds(xrow(dg.rdz[q], dg.rdy[q], c0 + dg.rdx[q] + j), wr[q - 1][j]);
#pragma unroll 2
                for (int st = 0; st < 8; ++st) {
                    const double* vs = vbase + st * SD;
                    double v[D];
#pragma unroll
                    for (int p = 0; p < PAIRS; ++p) {
                        const double2 a = *reinterpret_cast<const double2*>(vs + 2 * (p * 4 + g));
                        v[2 * p] = a.x;
                        v[2 * p + 1] = a.y;
                    }
                    if constexpr (D & 1) v[D - 1] = vs[2 * PAIRS * 4 + g];
                    double n0[CPL], nr[NG - 1][CPL];
                    lds(xrow(0, 0, c0 + st + 1), n0);
#pragma unroll
                    for (int q = 1; q < NG; ++q) lds(xrow(dg.rdz[q], dg.rdy[q], c0 + st + dg.rdx[q] + LR - 1), nr[q - 1]);
                    double acc[CPL];
#pragma unroll
                    for (int e = 0; e < CPL; ++e) {
                        double a = v[0] * w0[0][e];
                        a = fma(v[1], w0[1][e], a);
                        a = fma(v[2], n0[e], a);
                        acc[e] = a;
                    }
#pragma unroll
                    for (int q = 1; q < NG; ++q) {
                        const int d0 = L0 + (q - 1) * LR;
#pragma unroll
                        for (int j = 0; j < LR; ++j) {
#pragma unroll
                            for (int e = 0; e < CPL; ++e)
                                acc[e] = fma(v[d0 + j], j < LR - 1 ? wr[q - 1][j][e] : nr[q - 1][e], acc[e]);
                        }
                    }
                    if (xs0 + st < n) {
#pragma unroll
                        for (int e = 0; e < CPL; ++e) pd[e] = fma(w0[1][e], acc[e], pd[e]);
                        const size_t r = size_t(xs0 + st) + size_t(n) * (size_t(y) + size_t(n) * z);
                        *reinterpret_cast<double2*>(AP + r * 16 + xoff) = make_double2(acc[0], acc[1]);
                    }
#pragma unroll
                    for (int e = 0; e < CPL; ++e) {
                        w0[0][e] = w0[1][e];
                        w0[1][e] = n0[e];
                    }
#pragma unroll
                    for (int q = 1; q < NG; ++q) {
#pragma unroll
                        for (int j = 0; j + 1 < LR - 1; ++j)
#pragma unroll
                            for (int e = 0; e < CPL; ++e) wr[q - 1][j][e] = wr[q - 1][j + 1][e];
#pragma unroll
                        for (int e = 0; e < CPL; ++e) wr[q - 1][LR - 2][e] = nr[q - 1][e];
                    }
                }
            }
            __syncthreads();  // the loads below z's planes and value block c are free
            // refill: keep loads up to the next step's first needed plane + 3 in flight
            const int jnext = (z + 1 < z1) ? j0 + 1 : j0 + 3;  // next item starts 3 loads later (its own z0 - 1)
            while (jl < jnext + 4 && lvalid) issue_next();
            issue_vals();
        }
        jbase += (z1 - z0) + 2;
    }
#pragma unroll
    for (int e = 0; e < CPL; ++e)
        for (int o = 16; o >= G; o >>= 1) pd[e] += __shfl_xor_sync(0xffffffffu, pd[e], o);
    const int N = cc.N;
    if (lane < G) {
#pragma unroll
        for (int e = 0; e < CPL; ++e) sm[warp * N + xoff + e] = pd[e];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
        double tt = 0.0;
        for (int k = 0; k < int(blockDim.x >> 5); ++k) tt += sm[k * N + c];
        s.part0[size_t(blockIdx.x) * N + c] = tt;
    }
    __syncthreads();
    k1_epilogue(sm, N, cc, s);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int kZwThreads = 288;  // 8 compute warps + 1 producer warp

/// k_spmm_dia_zt with a producer warp (warp specialisation): warp 8 issues the plane and value bulk copies as soon
/// as the compute warps release a slot (per-slot "empty" mbarriers, one arrival per compute warp), so the compute
/// warps never meet at a block barrier and a warp that finished plane z starts plane z + 1 as soon as its data has
/// landed. Same work decomposition, layouts and accumulation order as k_spmm_dia_zt.
template <int NG, int LR>
__global__ void __launch_bounds__(kZwThreads, 1) k_spmm_dia_zw(int ni, Cols cc, DiaGeom dg, int nzc,
                                                             const double* __restrict__ dval,
                                                             const double* __restrict__ P, double* __restrict__ AP,
                                                             CgDev s) {
    constexpr int L0 = 3, G = 8, CPL = 2, NCW = 8;
    constexpr int D = L0 + (NG - 1) * LR;
    constexpr int SD = 4 * D, PAIRS = D / 2, TB = kZtT * kZtT * D;
    extern __shared__ __align__(128) double dsm[];
    double* xs = dsm;
    double* vsm = xs + size_t(kZtSlots) * kZtRows * 16;
    uint64_t* full = reinterpret_cast<uint64_t*>(vsm + 2 * TB);  // 0..3 planes, 4..5 values
    uint64_t* empty = full + 6;                                  // 0..3 planes, 4..5 values
    double* sm = reinterpret_cast<double*>(empty + 6);
    const int n = dg.n, nt = (n + kZtT - 1) / kZtT, ntile = nt * nt;
    const int lz = (n + nzc - 1) / nzc;
    const int nwork = ntile * nzc;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kZtSlots * kZtRows * 16; i += blockDim.x) xs[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 6; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto item_of = [&](int m, int& xt_, int& yt_, int& z0_, int& z1_) -> bool {
        const int wi = blockIdx.x + m * gridDim.x;
        if (wi >= nwork) return false;
        const int tile = wi % ntile, zc = wi / ntile;
        xt_ = tile % nt;
        yt_ = tile / nt;
        z0_ = zc * lz;
        z1_ = min(n, z0_ + lz);
        return true;
    };
    double pd[CPL] = {0.0, 0.0};
    const int N = cc.N;
    if (warp == NCW) {
        // ---- producer: for every compute step, the plane loads it needs (up to z + 1) and its value block ----
        int jl = 0, jv = 0;
        auto load = [&](int xt, int yt, int p) {
            const int sl = jl & 3;
            if (jl >= 4) mbar_wait(empty + sl, ((jl >> 2) - 1) & 1);
            const int x0 = xt * kZtT, y0 = yt * kZtT;
            const bool pv = p >= 0 && p < n;
            int lo = 0, hi = 0;
            const int y = y0 - 1 + lane;
            const int64_t start = int64_t(x0 - 1) + int64_t(n) * (int64_t(y) + int64_t(n) * p);
            if (pv && lane < kZtH && y >= 0 && y < n) {
                lo = int(start > 0 ? start : int64_t(0));
                hi = int(start + kZtH < int64_t(ni) ? start + kZtH : int64_t(ni));
            }
            int bytes = hi > lo ? (hi - lo) * 16 * int(sizeof(double)) : 0;
            for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(full + sl, uint32_t(bytes));
            }
            __syncwarp();
            if (hi > lo)
                bulk_g2s(xs + (size_t(sl) * kZtRows + size_t(lane) * kZtH + size_t(lo - start)) * 16,
                         P + size_t(lo) * 16, uint32_t((hi - lo) * 16 * sizeof(double)), full + sl);
            ++jl;
        };
        auto vals = [&](int xt, int yt, int p) {
            const int vb = jv & 1;
            if (jv >= 2) mbar_wait(empty + 4 + vb, ((jv >> 1) - 1) & 1);
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(full + 4 + vb, uint32_t(TB * sizeof(double)));
                bulk_g2s(vsm + size_t(vb) * TB, dval + ((size_t(p) * nt + yt) * nt + xt) * TB,
                         uint32_t(TB * sizeof(double)), full + 4 + vb);
            }
            __syncwarp();
            ++jv;
        };
        int xt = 0, yt = 0, z0 = 0, z1 = 0;
        for (int m = 0; item_of(m, xt, yt, z0, z1); ++m) {
            if (z0 >= z1) continue;
            load(xt, yt, z0 - 1);
            load(xt, yt, z0);
            for (int z = z0; z < z1; ++z) {
                load(xt, yt, z + 1);
                vals(xt, yt, z);
            }
        }
    } else {
        // ---- compute warps ----
        const int g = lane / G, l = lane % G;
        const int xoff = CPL * l;
        const int yl = 2 * warp + g / 2, sg = g % 2;
        int jbase = 0, c = 0;
        int xt = 0, yt = 0, z0 = 0, z1 = 0;
        for (int m = 0; item_of(m, xt, yt, z0, z1); ++m) {
            if (z0 >= z1) continue;
            const int x0 = xt * kZtT, y0 = yt * kZtT;
            const int y = y0 + yl;
            const int xs0 = x0 + 8 * sg;
            for (int z = z0; z < z1; ++z, ++c) {
                const int j0 = jbase + (z - z0);  // load of plane z - 1
                const int vb = c & 1;
                for (int t = 0; t < 3; ++t) mbar_wait(full + ((j0 + t) & 3), ((j0 + t) >> 2) & 1);
                mbar_wait(full + 4 + vb, (c >> 1) & 1);
                if (y < n) {
                    const int slot_of[3] = {j0 & 3, (j0 + 1) & 3, (j0 + 2) & 3};
                    auto xrow = [&](int dz, int dy, int col) -> const double* {
                        return xs + (size_t(slot_of[dz + 1]) * kZtRows + size_t(yl + 1 + dy) * kZtH + col) * 16 + xoff;
                    };
                    auto lds = [&](const double* p, double (&x)[CPL]) {
                        const double2 a = *reinterpret_cast<const double2*>(p);
                        x[0] = a.x;
                        x[1] = a.y;
                    };
                    const double* vbase = vsm + size_t(vb) * TB + size_t(warp) * 8 * SD;
                    double w0[L0 - 1][CPL];
                    double wr[NG - 1][LR - 1][CPL];
                    const int c0 = 8 * sg + 1;  // slot column of x = xs0
#pragma unroll
                    for (int j = 0; j < L0 - 1; ++j) lds(xrow(0, 0, c0 - 1 + j), w0[j]);
#pragma unroll
                    for (int q = 1; q < NG; ++q)
#pragma unroll
                        for (int j = 0; j < LR - 1; ++j) lds(xrow(dg.rdz[q], dg.rdy[q], c0 + dg.rdx[q] + j), wr[q - 1][j]);
#pragma unroll 2
                    for (int st = 0; st < 8; ++st) {
                        const double* vs = vbase + st * SD;
                        double v[D];
#pragma unroll
                        for (int p = 0; p < PAIRS; ++p) {
                            const double2 a = *reinterpret_cast<const double2*>(vs + 2 * (p * 4 + g));
                            v[2 * p] = a.x;
                            v[2 * p + 1] = a.y;
                        }
                        if constexpr (D & 1) v[D - 1] = vs[2 * PAIRS * 4 + g];
                        double n0[CPL], nr[NG - 1][CPL];
                        lds(xrow(0, 0, c0 + st + 1), n0);
#pragma unroll
                        for (int q = 1; q < NG; ++q)
                            lds(xrow(dg.rdz[q], dg.rdy[q], c0 + st + dg.rdx[q] + LR - 1), nr[q - 1]);
                        double acc[CPL];
#pragma unroll
                        for (int e = 0; e < CPL; ++e) {
                            double a = v[0] * w0[0][e];
                            a = fma(v[1], w0[1][e], a);
                            a = fma(v[2], n0[e], a);
                            acc[e] = a;
                        }
#pragma unroll
                        for (int q = 1; q < NG; ++q) {
                            const int d0 = L0 + (q - 1) * LR;
#pragma unroll
                            for (int j = 0; j < LR; ++j) {
#pragma unroll
                                for (int e = 0; e < CPL; ++e)
                                    acc[e] = fma(v[d0 + j], j < LR - 1 ? wr[q - 1][j][e] : nr[q - 1][e], acc[e]);
                            }
                        }
                        if (xs0 + st < n) {
#pragma unroll
                            for (int e = 0; e < CPL; ++e) pd[e] = fma(w0[1][e], acc[e], pd[e]);
                            const size_t r = size_t(xs0 + st) + size_t(n) * (size_t(y) + size_t(n) * z);
                            *reinterpret_cast<double2*>(AP + r * 16 + xoff) = make_double2(acc[0], acc[1]);
                        }
#pragma unroll
                        for (int e = 0; e < CPL; ++e) {
                            w0[0][e] = w0[1][e];
                            w0[1][e] = n0[e];
                        }
#pragma unroll
                        for (int q = 1; q < NG; ++q) {
#pragma unroll
                            for (int j = 0; j + 1 < LR - 1; ++j)
#pragma unroll
                                for (int e = 0; e < CPL; ++e) wr[q - 1][j][e] = wr[q - 1][j + 1][e];
#pragma unroll
                            for (int e = 0; e < CPL; ++e) wr[q - 1][LR - 2][e] = nr[q - 1][e];
                        }
                    }
                }
                // release: plane z - 1 (and at the item's end z, z + 1) and value block c
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(empty + (j0 & 3));
                    if (z + 1 == z1) {
                        mbar_arrive(empty + ((j0 + 1) & 3));
                        mbar_arrive(empty + ((j0 + 2) & 3));
                    }
                    mbar_arrive(empty + 4 + vb);
                }
            }
            jbase += (z1 - z0) + 2;
        }
#pragma unroll
        for (int e = 0; e < CPL; ++e)
            for (int o = 16; o >= G; o >>= 1) pd[e] += __shfl_xor_sync(0xffffffffu, pd[e], o);
        if (lane < G) {
#pragma unroll
            for (int e = 0; e < CPL; ++e) sm[warp * N + xoff + e] = pd[e];
        }
    }
    __syncthreads();
    for (int cc2 = threadIdx.x; cc2 < N; cc2 += blockDim.x) {
        double tt = 0.0;
        for (int k = 0; k < NCW; ++k) tt += sm[k * N + cc2];
        s.part0[size_t(blockIdx.x) * N + cc2] = tt;
    }
    __syncthreads();
    k1_epilogue(sm, N, cc, s);
}

// ---------------- K1 (union-tile variant, N > 16 on a locality order): G lanes per tile of <= kUtR rows ----------------
/// Tiles of the level's union-tile view (host/topology.hpp). A group of G lanes (lane l owns the interleaved column
/// pairs of the FULL layout, two 16-byte loads per row) walks the union of its tile's columns once: it gathers each
/// X row once and feeds it from registers to all kUtR tile rows with the entry's dense value vector (zero where a row
/// does not hold the column) -- k_spmm_dot gathers a row once per nonzero and broadcasts (col, val) by shuffles.
/// No per-entry dispatch: the inner loop is loads and FMAs only. The tile's columns and values are staged in shared
/// memory by bulk async copies one warp step ahead (two buffers per warp on mbarriers, 32 / G tiles per step) and
/// read with broadcast loads. Per row the products are accumulated in ascending column order, as in k_spmm_dot (the
/// zero products of the other rows' columns change nothing). With a shift operator the per-column coefficient
/// a + sigma_j b is formed first, so one accumulator set serves (A + sigma_j B).
inline size_t ut_tile_bytes(bool shift) { return size_t(kUtE) * 4 + size_t(kUtE) * kUtR * 8 * (shift ? 2 : 1); }
inline size_t ut_smem(int G, int threads, bool shift, bool vsm) {
    const size_t nw = threads / 32, tpw = 32 / G;
    const size_t tile = vsm ? ut_tile_bytes(shift) : size_t(kUtE) * 4;
    return nw * 4 * G * sizeof(double) + nw * 2 * tpw * tile + nw * 2 * sizeof(uint64_t);
}

/// VSM: the tile's values are staged in shared memory with its columns (one warp per tile: G = 32). !VSM: only the
/// columns are staged (256 bytes per tile, so the staging no longer limits the resident warps) and each entry's four
/// values are read from global memory with the entry's gathers (one broadcast 32-byte load per lane group) -- the
/// narrow groups (G = 8, 16: four / two tiles per warp), whose value buffers would leave 6 warps per SM.
template <int G, bool SHIFT, int UB, int NT, int MINB, bool VSM, bool HINT = false>
__global__ void __launch_bounds__(NT, MINB) k_spmm_ut(int nt, Cols cc, const int32_t* __restrict__ trows,
                                                     const int32_t* __restrict__ eptr, const int32_t* __restrict__ ent,
                                                     const double* __restrict__ A, const double* __restrict__ Bv,
                                                     const double* __restrict__ P, double* __restrict__ AP, CgDev s,
                                                     int sync_every) {
    // sync_every > 0 (cooperative launch): a grid barrier every sync_every warp steps keeps all warps inside one
    // stretch of the Morton tile sequence, so the X rows that neighbouring tiles share are still in L2 when the
    // next tile asks for them (without it the warps drift apart over the ~1200 steps of a 1e7-row level)
    extern __shared__ double sm[];
    constexpr int CPL = 4, R = kUtR, TPW = 32 / G, W = 4 * G;
    constexpr int VS = SHIFT ? 2 : 1;
    constexpr int TB = kUtE * 4 + (VSM ? kUtE * R * 8 * VS : 0);  // staged bytes per tile
    static_assert(R == 4, "the value loads below read 4 doubles per entry");
    static_assert(VSM || UB == 4, "values from global memory: batches of 4 entries");
    const int N = cc.N, ld = cc.ld;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = NT / 32;
    const int g = lane / G, l = lane % G;
    char* stage = reinterpret_cast<char*>(sm) + size_t(nwb) * W * sizeof(double) + size_t(wib) * 2 * TPW * TB;
    uint64_t* bars =
        reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(sm) + size_t(nwb) * W * sizeof(double) + size_t(nwb) * 2 * TPW * TB) +
        wib * 2;
    // the lane's two column pairs (FULL layout); a pair that starts at or past N is clamped onto the block's last
    // pair, so every gather is unconditional (same 128-byte lines as the neighbouring lanes); its products land in
    // accumulators that are never stored or read
    const int c0 = full_col<G>(l, 0), c1 = full_col<G>(l, 2);
    const bool ok0 = c0 < N, ok1 = c1 < N;
    const int cmax = (N - 1) & ~1;
    const double* P0 = P + min(c0, cmax);
    const double* P1 = P + min(c1, cmax);
    const uint32_t uld = uint32_t(ld);
    const uint64_t pol = HINT ? l2_policy_last() : 0;
    double pd[CPL], sg[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
        pd[q] = 0.0;
        const int c = full_col<G>(l, q);
        sg[q] = (SHIFT && c < N) ? s.sigma[c] : 0.0;
    }
    const TileWalk tw((nt + TPW - 1) / TPW);
    const int ksteps = tw.t0 < tw.tend ? (tw.tend - tw.t0 + tw.step - 1) / tw.step : 0;
    auto fetch = [&](int k) {  // group leaders: the group's tile of warp step k into buffer k & 1
        if (l == 0 && k < ksteps) {
            const int t = (tw.t0 + k * tw.step) * TPW + g;
            uint64_t* bar = bars + (k & 1);
            if (t < nt) {
                const int e0 = __ldg(eptr + t), ne = __ldg(eptr + t + 1) - e0;
                char* b = stage + size_t((k & 1) * TPW + g) * TB;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(bar, uint32_t(ne * 4 + (VSM ? ne * R * 8 * VS : 0)));
                bulk_g2s(b, ent + e0, uint32_t(ne * 4), bar);
                if constexpr (VSM) {
                    bulk_g2s(b + kUtE * 4, A + size_t(e0) * R, uint32_t(ne * R * 8), bar);
                    if (SHIFT) bulk_g2s(b + kUtE * 4 + kUtE * R * 8, Bv + size_t(e0) * R, uint32_t(ne * R * 8), bar);
                }
            } else {
                mbar_arrive(bar);
            }
        }
    };
    if (lane == 0) {
        mbar_init(bars, TPW);
        mbar_init(bars + 1, TPW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    fetch(0);
    const int kall = (tw.tend + tw.step - 1) / tw.step;  // the same count for every warp of the grid
    for (int k = 0; k < kall; ++k) {
        if (sync_every > 0 && k > 0 && k % sync_every == 0) cooperative_groups::this_grid().sync();
        if (k >= ksteps) continue;
        const int t = (tw.t0 + k * tw.step) * TPW + g;
        const bool valid = t < nt;
        __syncwarp();  // every lane is done with the buffer step k + 1 lands in (step k - 1's)
        fetch(k + 1);
        const int e0 = valid ? __ldg(eptr + t) : 0;
        const int ne = valid ? __ldg(eptr + t + 1) - e0 : 0;
        const int myrow = (valid && l < R) ? __ldg(trows + size_t(t) * R + l) : -1;
        const char* b = stage + size_t((k & 1) * TPW + g) * TB;
        const int32_t* sc = reinterpret_cast<const int32_t*>(b);
        const double* sa = VSM ? reinterpret_cast<const double*>(b + kUtE * 4) : A + size_t(e0) * R;
        const double* sb = VSM ? reinterpret_cast<const double*>(b + kUtE * 4 + kUtE * R * 8) : Bv + size_t(e0) * R;
        double acc[R][CPL];
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
            for (int q = 0; q < CPL; ++q) acc[i][q] = 0.0;
        mbar_wait(bars + (k & 1), (k >> 1) & 1);
        // batches of 4 entries (the entry count is a multiple of 4): the gathers of one batch, then its products.
        // UB == 8: two batches' gathers at once. The groups of a warp run their own trip counts (no warp-level
        // operation inside).
        struct Vals {
            double2 a[4][2], b[SHIFT ? 4 : 1][2];
        };
        auto gather = [&](int e, double2 (&x0)[4], double2 (&x1)[4], Vals& v) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const size_t off = size_t(uint32_t(sc[e + u])) * uld;
                if constexpr (HINT) {  // gathered rows evict-last in L2 (the matrix and output streams pass by)
                    x0[u] = ldg2_hint(P0 + off, pol);
                    x1[u] = ldg2_hint(P1 + off, pol);
                } else {
                    x0[u] = __ldg(reinterpret_cast<const double2*>(P0 + off));
                    x1[u] = __ldg(reinterpret_cast<const double2*>(P1 + off));
                }
                if constexpr (!VSM) {
                    v.a[u][0] = __ldg(reinterpret_cast<const double2*>(sa + size_t(e + u) * R));
                    v.a[u][1] = __ldg(reinterpret_cast<const double2*>(sa + size_t(e + u) * R + 2));
                    if constexpr (SHIFT) {
                        v.b[u][0] = __ldg(reinterpret_cast<const double2*>(sb + size_t(e + u) * R));
                        v.b[u][1] = __ldg(reinterpret_cast<const double2*>(sb + size_t(e + u) * R + 2));
                    }
                }
            }
        };
        auto products = [&](int e, const double2 (&x0)[4], const double2 (&x1)[4], const Vals& v) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                double2 a01, a23, b01 = make_double2(0.0, 0.0), b23 = b01;
                if constexpr (VSM) {
                    a01 = *reinterpret_cast<const double2*>(sa + size_t(e + u) * R);
                    a23 = *reinterpret_cast<const double2*>(sa + size_t(e + u) * R + 2);
                    if constexpr (SHIFT) {
                        b01 = *reinterpret_cast<const double2*>(sb + size_t(e + u) * R);
                        b23 = *reinterpret_cast<const double2*>(sb + size_t(e + u) * R + 2);
                    }
                } else {
                    a01 = v.a[u][0];
                    a23 = v.a[u][1];
                    if constexpr (SHIFT) {
                        b01 = v.b[u][0];
                        b23 = v.b[u][1];
                    }
                }
                const double av[R] = {a01.x, a01.y, a23.x, a23.y};
                const double xv[CPL] = {x0[u].x, x0[u].y, x1[u].x, x1[u].y};
                if constexpr (SHIFT) {
                    const double bv[R] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
                    for (int i = 0; i < R; ++i)
#pragma unroll
                        for (int q = 0; q < CPL; ++q) acc[i][q] = fma(fma(sg[q], bv[i], av[i]), xv[q], acc[i][q]);
                } else {
#pragma unroll
                    for (int i = 0; i < R; ++i)
#pragma unroll
                        for (int q = 0; q < CPL; ++q) acc[i][q] = fma(av[i], xv[q], acc[i][q]);
                }
            }
        };
        double2 xa0[4], xa1[4];
        Vals va;
        if constexpr (UB == 8) {
            double2 xb0[4], xb1[4];
            int e = 0;
            for (; e + 8 <= ne; e += 8) {
                gather(e, xa0, xa1, va);
                gather(e + 4, xb0, xb1, va);
                products(e, xa0, xa1, va);
                products(e + 4, xb0, xb1, va);
            }
            if (e < ne) {
                gather(e, xa0, xa1, va);
                products(e, xa0, xa1, va);
            }
        } else {
            for (int e = 0; e < ne; e += 4) {
                gather(e, xa0, xa1, va);
                products(e, xa0, xa1, va);
            }
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int r = __shfl_sync(0xffffffffu, myrow, i, G);
            if (r >= 0) {
                const size_t off = size_t(uint32_t(r)) * uld;
                const double2 p0 = __ldg(reinterpret_cast<const double2*>(P0 + off));
                const double2 p1 = __ldg(reinterpret_cast<const double2*>(P1 + off));
                if (ok0) __stcs(reinterpret_cast<double2*>(AP + off + c0), make_double2(acc[i][0], acc[i][1]));
                if (ok1) __stcs(reinterpret_cast<double2*>(AP + off + c1), make_double2(acc[i][2], acc[i][3]));
                pd[0] = fma(p0.x, acc[i][0], pd[0]);
                pd[1] = fma(p0.y, acc[i][1], pd[1]);
                pd[2] = fma(p1.x, acc[i][2], pd[2]);
                pd[3] = fma(p1.y, acc[i][3], pd[3]);
            }
        }
    }
    // block reduce: groups with equal l hold the same columns -- xor tree over the groups of a warp, then a
    // fixed-order sum over the warps (k_spmm_dot's epilogue)
#pragma unroll
    for (int q = 0; q < CPL; ++q)
        for (int o = 16; o >= G; o >>= 1) pd[q] += __shfl_xor_sync(0xffffffffu, pd[q], o);
    if (lane < G) {
#pragma unroll
        for (int q = 0; q < CPL; ++q) sm[wib * W + full_col<G>(l, q)] = pd[q];
    }
    __syncthreads();
    if (threadIdx.x < N) {
        double t = 0.0;
        for (int k = 0; k < nwb; ++k) t += sm[k * W + threadIdx.x];
        s.part0[size_t(blockIdx.x) * N + threadIdx.x] = t;
    }
    k1_epilogue(sm, N, cc, s);
}

// ---------------- K1 (SELL-32 variant): one row per lane, all N <= 16 columns per lane ----------------
template <int NC>
__device__ __forceinline__ void load_row(const double* __restrict__ p, double (&x)[NC]) {
    if constexpr (NC == 1) {
        x[0] = __ldg(p);
    } else {
#pragma unroll
        for (int q = 0; q < NC; q += 2) {
            const double2 a = __ldg(reinterpret_cast<const double2*>(p + q));
            x[q] = a.x;
            x[q + 1] = a.y;
        }
    }
}

/// Same contract as k_spmm_dot for N == NC in {1, 2, 4, 8, 16}. A is read in SELL-32 order
/// (entry e of the 32 rows of a slice is contiguous: coalesced col/val loads, no shuffles); each
/// lane gathers whole X rows for its own row, U entries in flight.
template <int NC, bool SHIFT>
__global__ void __launch_bounds__(kThreads, 2) k_sell_dot(int ni, int nslices, Cols cc, const int32_t* __restrict__ sptr,
                                                         const int32_t* __restrict__ scol,
                                                         const double* __restrict__ sA,
                                                         const double* __restrict__ sB,
                                                         const double* __restrict__ P, double* __restrict__ AP,
                                                         CgDev s) {
    extern __shared__ double sm[];
    constexpr int U = NC >= 8 ? 2 : 4;
    const int N = cc.N, ld = cc.ld;
    const int lane = threadIdx.x & 31;
    const int nwb = blockDim.x >> 5, wib = threadIdx.x >> 5;
    const int warp = blockIdx.x * nwb + wib;
    const int nwarps = gridDim.x * nwb;
    double pd[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) pd[q] = 0.0;
    for (int sl = warp; sl < nslices; sl += nwarps) {
        const int r = sl * 32 + lane;
        const int b0 = __ldg(sptr + sl);
        const int w = (__ldg(sptr + sl + 1) - b0) >> 5;
        double acc[NC], accB[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) acc[q] = accB[q] = 0.0;
        for (int e = 0; e < w; e += U) {
            int j[U];
            double a[U], bb[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = b0 + (e + u) * 32 + lane;
                const bool in = e + u < w;
                j[u] = in ? __ldg(scol + k) : 0;
                a[u] = in ? __ldg(sA + k) : 0.0;
                bb[u] = (SHIFT && in) ? __ldg(sB + k) : 0.0;
            }
            double x[U][NC];
#pragma unroll
            for (int u = 0; u < U; ++u) load_row<NC>(P + size_t(j[u]) * ld, x[u]);
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < NC; ++q) {
                    acc[q] = fma(a[u], x[u][q], acc[q]);
                    if (SHIFT) accB[q] = fma(bb[u], x[u][q], accB[q]);
                }
        }
        if (r < ni) {
            if (SHIFT) {
#pragma unroll
                for (int q = 0; q < NC; ++q) acc[q] = fma(s.sigma[q], accB[q], acc[q]);
            }
            double p[NC];
            load_row<NC>(P + size_t(r) * ld, p);
            double* y = AP + size_t(r) * ld;
            if constexpr (NC == 1) {
                y[0] = acc[0];
            } else {
#pragma unroll
                for (int q = 0; q < NC; q += 2) *reinterpret_cast<double2*>(y + q) = make_double2(acc[q], acc[q + 1]);
            }
#pragma unroll
            for (int q = 0; q < NC; ++q) pd[q] = fma(p[q], acc[q], pd[q]);
        }
    }
    // block reduce per column: warp shuffle, then fixed-order sum over warps
    double* red = sm;  // nwb x NC
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        const double t = warp_sum(pd[q]);
        if (lane == 0) red[wib * NC + q] = t;
    }
    __syncthreads();
    if (threadIdx.x < N) {
        double t = 0.0;
        for (int k = 0; k < nwb; ++k) t += red[k * NC + threadIdx.x];
        s.part0[size_t(blockIdx.x) * N + threadIdx.x] = t;
    }
    k1_epilogue(red, N, cc, s);
}

// ---------------- persistent cooperative CG for N <= 2 ----------------
// Small solves (the orbital BVP at N = 1-2 and every Hartree solve) are latency bound as four kernels per
// iteration. This kernel runs a chunk of iterations in one cooperative launch: the same four phases
// (K1 SpMV + p.Ap, K2 r update + r.r/r.z, K3 true residual when flagged, K4 x/p update) separated by grid
// barriers. Every block folds the per-block partials in the same fixed order and advances an identical copy
// of the per-column scalar state in shared memory, so no block waits on another for alpha / beta; block 0
// writes the state back at the end of the chunk. Rows follow the SELL-32 slices (warp per slice, lane per
// row) in every phase, so each thread only touches its own rows between barriers.
struct CoopState {
    double alpha[2], beta[2], rz[2], rr[2], bnorm[2], relres[2];
    int status[2], check[2], iters[2], nonpos[2];
    int it, nactive, anycheck;
};

template <int NC>
__device__ void coop_load(CoopState& st, const CgDev& s) {
    if (threadIdx.x == 0) {
        for (int c = 0; c < NC; ++c) {
            st.alpha[c] = s.alpha[c];
            st.beta[c] = s.beta[c];
            st.rz[c] = s.rz[c];
            st.rr[c] = s.rr[c];
            st.bnorm[c] = s.bnorm[c];
            st.relres[c] = s.relres[c];
            st.status[c] = s.status[c];
            st.check[c] = s.check[c];
            st.iters[c] = s.iters[c];
            st.nonpos[c] = s.nonpos[c];
        }
        st.it = s.ctl[kIt];
        st.nactive = s.ctl[kNActive];
        st.anycheck = s.ctl[kAnyCheck];
    }
    __syncthreads();
}

template <int NC>
__device__ void coop_store(const CoopState& st, CgDev& s) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int c = 0; c < NC; ++c) {
            s.alpha[c] = st.alpha[c];
            s.beta[c] = st.beta[c];
            s.rz[c] = st.rz[c];
            s.rr[c] = st.rr[c];
            s.relres[c] = st.relres[c];
            s.status[c] = st.status[c];
            s.check[c] = st.check[c];
            s.iters[c] = st.iters[c];
            s.nonpos[c] = st.nonpos[c];
        }
        s.ctl[kIt] = st.it;
        s.ctl[kNActive] = st.nactive;
        s.ctl[kAnyCheck] = st.anycheck;
    }
}

/// per-block sum of K partial vectors (thread values v[k]) -> part[blockIdx * K + k], fixed order
template <int K>
__device__ void coop_block_sum(const double (&v)[K], double* part, double* red) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double t = warp_sum(v[k]);
        if (lane == 0) red[wib * K + k] = t;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t += red[w * K + threadIdx.x];
        part[size_t(blockIdx.x) * K + threadIdx.x] = t;
    }
    __syncthreads();
}

template <int NC, bool SHIFT>
__global__ void __launch_bounds__(kThreads) k_cg_coop(int ni, int nsl, Cols cc, const int32_t* __restrict__ sptr,
                                                      const int32_t* __restrict__ scol, const double* __restrict__ sA,
                                                      const double* __restrict__ sB, const double* __restrict__ Bb,
                                                      double* __restrict__ X, double* __restrict__ R,
                                                      double* __restrict__ P, double* __restrict__ AP, CgDev s,
                                                      int n_iters) {
    namespace cgx = cooperative_groups;
    cgx::grid_group grid = cgx::this_grid();
    __shared__ CoopState st;
    __shared__ double red[32 * 2 * NC];
    __shared__ double fold[4 * NC];
    const int ld = cc.ld;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    coop_load<NC>(st, s);
    double sig[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) sig[c] = SHIFT ? s.sigma[c] : 0.0;
    auto dinv = [&](int r, int c) {
        double d = s.diagA[r];
        if (s.diagB) d += s.sigma[c] * s.diagB[r];
        return d != 0.0 ? 1.0 / d : 1.0;
    };
    // SpMV of the own rows: y = (A + sigma B) v for every slice of this warp
    auto spmv_rows = [&](const double* __restrict__ V, auto&& per_row) {
        for (int sl = warp; sl < nsl; sl += nwarps) {
            const int r = sl * 32 + lane;
            const int b0 = __ldg(sptr + sl);
            const int w = (__ldg(sptr + sl + 1) - b0) >> 5;
            double acc[NC], accB[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[c] = accB[c] = 0.0;
            constexpr int U = 4;  // entries in flight per lane: index loads, then gathers, then FMAs
            for (int e0 = 0; e0 < w; e0 += U) {
                int j[U];
                double a[U], bb[U], x[U][NC];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = b0 + (e0 + u) * 32 + lane;
                    const bool in = e0 + u < w;
                    j[u] = in ? __ldg(scol + k) : 0;
                    a[u] = in ? __ldg(sA + k) : 0.0;
                    bb[u] = (SHIFT && in) ? __ldg(sB + k) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int c = 0; c < NC; ++c) x[u][c] = V[size_t(j[u]) * ld + c];
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        acc[c] = fma(a[u], x[u][c], acc[c]);
                        if (SHIFT) accB[c] = fma(bb[u], x[u][c], accB[c]);
                    }
            }
            if (r < ni) {
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    if (SHIFT) acc[c] = fma(sig[c], accB[c], acc[c]);
                per_row(r, acc);
            }
        }
    };
    for (int k = 0; k < n_iters; ++k) {
        if (!cc.fixed && st.nactive == 0) break;
        // ---- K1: Ap = A p, p.Ap
        {
            double pd[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) pd[c] = 0.0;
            spmv_rows(P, [&](int r, const double (&acc)[NC]) {
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    AP[size_t(r) * ld + c] = acc[c];
                    pd[c] = fma(P[size_t(r) * ld + c], acc[c], pd[c]);
                }
            });
            coop_block_sum<NC>(pd, s.part0, red);
        }
        grid.sync();
        fold_partials(s.part0, gridDim.x, NC, fold);
        if (threadIdx.x == 0) {
            for (int c = 0; c < NC; ++c) {
                const double pap = fold[c];
                double al = 0.0;
                if (st.status[c] == kActive) {
                    if (!(pap > 0.0)) {
                        if (!cc.fixed) {
                            st.status[c] = kBreakdown;
                            st.relres[c] = sqrt(st.rr[c]) / st.bnorm[c];
                        } else {
                            st.nonpos[c] += 1;
                            if (pap != 0.0 && isfinite(pap)) al = st.rz[c] / pap;
                        }
                    } else {
                        al = st.rz[c] / pap;
                    }
                }
                st.alpha[c] = al;
            }
            int na = 0;
            for (int c = 0; c < NC; ++c) na += st.status[c] == kActive;
            st.nactive = na;
        }
        __syncthreads();
        // ---- K2: r -= alpha Ap (active columns), r.r and r.z
        {
            double part[2 * NC];
#pragma unroll
            for (int c = 0; c < 2 * NC; ++c) part[c] = 0.0;
            for (int sl = warp; sl < nsl; sl += nwarps) {
                const int r = sl * 32 + lane;
                if (r >= ni) continue;
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    if (st.status[c] != kActive) continue;
                    const size_t i = size_t(r) * ld + c;
                    const double rv = fma(-st.alpha[c], AP[i], R[i]);
                    R[i] = rv;
                    part[c] = fma(rv, rv, part[c]);
                    part[NC + c] = fma(rv, dinv(r, c) * rv, part[NC + c]);
                }
            }
            coop_block_sum<2 * NC>(part, s.part1, red);
        }
        grid.sync();
        fold_partials(s.part1, gridDim.x, 2 * NC, fold);
        if (threadIdx.x == 0) {
            int any = 0;
            for (int c = 0; c < NC; ++c) {
                if (st.status[c] != kActive) continue;
                const double rr = fold[c], rz = fold[NC + c];
                const double rel = sqrt(rr) / st.bnorm[c];
                st.rr[c] = rr;
                st.iters[c] = st.it + 1;
                st.relres[c] = rel;
                if (!cc.fixed && rel <= cc.tol) {
                    st.check[c] = 1;
                    any = 1;
                } else {
                    st.beta[c] = rz / st.rz[c];
                    st.rz[c] = rz;
                }
            }
            st.it += 1;
            st.anycheck = any;
        }
        __syncthreads();
        // ---- K3: true residual t = b - A x - alpha Ap for flagged columns (x still x_k)
        if (!cc.fixed && st.anycheck) {
            double part[2 * NC];
#pragma unroll
            for (int c = 0; c < 2 * NC; ++c) part[c] = 0.0;
            spmv_rows(X, [&](int r, const double (&acc)[NC]) {
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    if (!st.check[c]) continue;
                    const size_t i = size_t(r) * ld + c;
                    const double t = Bb[i] - fma(st.alpha[c], AP[i], acc[c]);
                    R[i] = t;
                    part[c] = fma(t, t, part[c]);
                    part[NC + c] = fma(t, dinv(r, c) * t, part[NC + c]);
                }
            });
            coop_block_sum<2 * NC>(part, s.part0, red);
            grid.sync();
            fold_partials(s.part0, gridDim.x, 2 * NC, fold);
            if (threadIdx.x == 0) {
                for (int c = 0; c < NC; ++c) {
                    if (!st.check[c]) continue;
                    const double rel = sqrt(fold[c]) / st.bnorm[c];
                    st.relres[c] = rel;
                    st.rr[c] = fold[c];
                    if (rel <= cc.tol) {
                        st.status[c] = kConverged;
                    } else {
                        st.rz[c] = fold[NC + c];
                        st.beta[c] = 0.0;
                    }
                    st.check[c] = 0;
                }
                st.anycheck = 0;
                int na = 0;
                for (int c = 0; c < NC; ++c) na += st.status[c] == kActive;
                st.nactive = na;
            }
            __syncthreads();
        }
        // ---- K4: x += alpha p, p = z + beta p
        for (int sl = warp; sl < nsl; sl += nwarps) {
            const int r = sl * 32 + lane;
            if (r >= ni) continue;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const size_t i = size_t(r) * ld + c;
                const double pv = P[i];
                if (st.alpha[c] != 0.0) X[i] = fma(st.alpha[c], pv, X[i]);
                if (st.status[c] == kActive) P[i] = fma(st.beta[c], pv, dinv(r, c) * R[i]);
            }
        }
        grid.sync();
    }
    coop_store<NC>(st, s);
}

// ---------------- K2: r update (x is deferred to K4, which reads p anyway) ----------------
template <int V>
__global__ void __launch_bounds__(kThreads, 4) k_update_r(int ni, Cols cc, double* __restrict__ R,
                                                       const double* __restrict__ AP, CgDev s) {
    extern __shared__ double sm[];
    const int N = cc.N, ld = cc.ld;
    EMap<V> em(N);
    double rr[V], rz[V];
#pragma unroll
    for (int q = 0; q < V; ++q) rr[q] = rz[q] = 0.0;
    if (em.valid) {
        double al[V], sg[V];
        bool any = false;
#pragma unroll
        for (int q = 0; q < V; ++q) {
            al[q] = s.status[em.c + q] == kActive ? s.alpha[em.c + q] : 0.0;
            sg[q] = s.diagB ? s.sigma[em.c + q] : 0.0;
            any |= s.status[em.c + q] == kActive;
        }
        // U rows per trip, all loads issued before the first use (bytes in flight per thread)
        constexpr int U = 2;
        if (any)
            for (int r0 = em.r0; r0 < ni; r0 += U * em.rstep) {
                double rv[U][V], ap[U][V], da[U], db[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int r = r0 + u * em.rstep;
                    if (r < ni) {
                        const size_t i = size_t(r) * ld + em.c;
                        ldv<V>(R + i, rv[u]);
                        ldv<V>(AP + i, ap[u]);
                        da[u] = s.diagA[r];
                        db[u] = s.diagB ? s.diagB[r] : 0.0;
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int r = r0 + u * em.rstep;
                    if (r < ni) {
#pragma unroll
                        for (int q = 0; q < V; ++q) rv[u][q] = fma(-al[q], ap[u][q], rv[u][q]);
                        stv<V>(R + size_t(r) * ld + em.c, rv[u]);
#pragma unroll
                        for (int q = 0; q < V; ++q) {
                            const double d = fma(sg[q], db[u], da[u]);
                            const double dinv = d != 0.0 ? 1.0 / d : 1.0;
                            rr[q] = fma(rv[u][q], rv[u][q], rr[q]);
                            rz[q] = fma(rv[u][q], dinv * rv[u][q], rz[q]);
                        }
                    }
                }
            }
    }
    block_cols_v<V>(rr, N, s.part0, sm);
    block_cols_v<V>(rz, N, s.part1, sm);
    if (!last_block(s.ctl + kTicket2)) return;
    fold_partials(s.part0, gridDim.x, N, sm);
    fold_partials(s.part1, gridDim.x, N, sm + N);
    __shared__ int any;
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    const int it = s.ctl[kIt];
    if (threadIdx.x < N) {
        const int c = threadIdx.x;
        if (s.status[c] == kActive) {
            const double rel = sqrt(sm[c]) / s.bnorm[c];
            s.rr[c] = sm[c];
            s.iters[c] = it + 1;
            s.relres[c] = rel;
            if (!cc.fixed && rel <= cc.tol) {
                s.check[c] = 1;
                atomicOr(&any, 1);
            } else {
                s.beta[c] = sm[N + c] / s.rz[c];
                s.rz[c] = sm[N + c];
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        s.ctl[kIt] = it + 1;
        s.ctl[kAnyCheck] = any;
    }
}

// ---------------- K3: true residual for flagged columns ----------------
template <int G, int CPL, bool SHIFT, bool SPLIT, int FULL>
__global__ void __launch_bounds__(kThreads, 3) k_trueres(int ni, Cols cc, const int32_t* __restrict__ ptr,
                                                      const int32_t* __restrict__ col, const double* __restrict__ A,
                                                      const double* __restrict__ Bv, const double* __restrict__ Bb,
                                                      const double* __restrict__ X, const double* __restrict__ AP,
                                                      double* __restrict__ R, CgDev s) {
    extern __shared__ double sm[];
    if (s.ctl[kAnyCheck] == 0) return;  // uniform early exit: nothing flagged this iteration
    const int N = cc.N, ld = cc.ld;
    const int lane = threadIdx.x & 31;
    const int g = lane / G, l = lane % G;
    const int gbase = g * G;
    const int rows_per_warp = 32 / G;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int c0 = SPLIT ? 0 : l * CPL;
    double tt[CPL], tz[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) tt[q] = tz[q] = 0.0;
    // gather only the column pairs (FULL) / lane columns that have a flagged column: usually a few of N
    unsigned need = 0;
    if constexpr (FULL == 3) {
#pragma unroll
        for (int q = 0; q < CPL; ++q)
            if (s.check[lay_col<G, 3>(l, q)]) need |= 1u << (q >> 2);
    } else if constexpr (FULL != 0) {
#pragma unroll
        for (int q = 0; q < CPL; q += 2) {
            const int c = full_col<G>(l, q);
            if ((c < N && s.check[c]) || (c + 1 < N && s.check[c + 1])) need |= 1u << (q >> 1);
        }
    } else if constexpr (!SPLIT) {
#pragma unroll
        for (int q = 0; q < CPL; ++q)
            if (c0 + q < N && s.check[c0 + q]) need = 1u;
    }
    for (int base = warp * rows_per_warp; base < ni; base += nwarps * rows_per_warp) {
        const int r = base + g;
        const bool valid = r < ni;
        const int rb = valid ? __ldg(ptr + r) : 0, re = valid ? __ldg(ptr + r + 1) : 0;
        double acc[CPL], accB[CPL];
        if constexpr (SPLIT) {
            row_split<G, SHIFT>(rb, re, col, A, Bv, X, ld, l, acc[0], accB[0]);
        } else {
            row_product<G, CPL, SHIFT, FULL>(valid ? r : 0, rb, re, col, A, Bv, X, ld, c0, N, l, gbase, acc, accB,
                                             need);
        }
        if (valid && (!SPLIT || l == 0) && (FULL || c0 < N)) {
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int c = FULL ? lay_col<G, FULL>(l, q) : c0 + q;
                if (c < N && s.check[c]) {
                    // X still holds x_k (K4 applies x += alpha p): A x_{k+1} = A x_k + alpha Ap
                    const double ax = SHIFT ? fma(s.sigma[c], accB[q], acc[q]) : acc[q];
                    const size_t i = size_t(r) * ld + c;
                    const double t = Bb[i] - fma(s.alpha[c], AP[i], ax);
                    R[i] = t;
                    tt[q] = fma(t, t, tt[q]);
                    tz[q] = fma(t, dinv_of(s.diagA, s.diagB, s.sigma, r, c) * t, tz[q]);
                }
            }
        }
    }
    const int ngroups = blockDim.x / G;
    const int width = G * CPL;
    const int gid = threadIdx.x / G;
    for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
        for (int q = 0; q < CPL; ++q) sm[gid * width + (FULL ? lay_col<G, FULL>(l, q) : l * CPL + q)] = pass ? tz[q] : tt[q];
        __syncthreads();
        if (threadIdx.x < N) {
            double t = 0.0;
            for (int k = 0; k < ngroups; ++k) t += sm[k * width + threadIdx.x];
            (pass ? s.part1 : s.part0)[size_t(blockIdx.x) * N + threadIdx.x] = t;
        }
        __syncthreads();
    }
    if (!last_block(s.ctl + kTicket3)) return;
    fold_partials(s.part0, gridDim.x, N, sm);
    fold_partials(s.part1, gridDim.x, N, sm + N);
    if (threadIdx.x < N) {
        const int c = threadIdx.x;
        if (s.check[c]) {
            const double rel = sqrt(sm[c]) / s.bnorm[c];
            s.relres[c] = rel;
            s.rr[c] = sm[c];
            if (rel <= cc.tol) {
                s.status[c] = kConverged;
            } else {  // restart from the true residual: p = z
                s.rz[c] = sm[N + c];
                s.beta[c] = 0.0;
            }
            s.check[c] = 0;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        s.ctl[kAnyCheck] = 0;
        int na = 0;
        for (int c = 0; c < N; ++c) na += s.status[c] == kActive;
        s.ctl[kNActive] = na;
    }
}

// ---------------- K4: x += alpha p (deferred from K2), p = D^-1 r + beta p ----------------
template <int V>
__global__ void __launch_bounds__(kThreads, 4) k_update_px(int ni, Cols cc, double* __restrict__ X,
                                                        const double* __restrict__ R, double* __restrict__ P,
                                                        CgDev s) {
    const int N = cc.N, ld = cc.ld;
    EMap<V> em(N);
    if (!em.valid) return;
    double al[V], be[V], sg[V];
    bool act[V], anyx = false, anyp = false;
#pragma unroll
    for (int q = 0; q < V; ++q) {
        al[q] = s.alpha[em.c + q];  // 0 for columns not active at K1 of this iteration
        act[q] = s.status[em.c + q] == kActive;
        be[q] = s.beta[em.c + q];
        sg[q] = s.diagB ? s.sigma[em.c + q] : 0.0;
        anyx |= al[q] != 0.0;
        anyp |= act[q];
    }
    if (!anyx && !anyp) return;
    constexpr int U = 2;
    for (int r0 = em.r0; r0 < ni; r0 += U * em.rstep) {
        double pv[U][V], xv[U][V], rv[U][V], da[U], db[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = r0 + u * em.rstep;
            if (r < ni) {
                const size_t i = size_t(r) * ld + em.c;
                ldv<V>(P + i, pv[u]);
                if (anyx) ldv<V>(X + i, xv[u]);
                if (anyp) {
                    ldv<V>(R + i, rv[u]);
                    da[u] = s.diagA[r];
                    db[u] = s.diagB ? s.diagB[r] : 0.0;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = r0 + u * em.rstep;
            if (r < ni) {
                const size_t i = size_t(r) * ld + em.c;
                if (anyx) {
#pragma unroll
                    for (int q = 0; q < V; ++q) xv[u][q] = fma(al[q], pv[u][q], xv[u][q]);
                    stv<V>(X + i, xv[u]);
                }
                if (anyp) {
#pragma unroll
                    for (int q = 0; q < V; ++q) {
                        const double d = fma(sg[q], db[u], da[u]);
                        const double z = (d != 0.0 ? 1.0 / d : 1.0) * rv[u][q];
                        if (act[q]) pv[u][q] = fma(be[q], pv[u][q], z);
                    }
                    stv<V>(P + i, pv[u]);
                }
            }
        }
    }
}

__global__ void k_diag(int ni, const int32_t* __restrict__ dslot, const double* __restrict__ vals,
                       double* __restrict__ d) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ni; r += gridDim.x * blockDim.x) d[r] = vals[dslot[r]];
}

int elem_grid(const Ctx& c, int ni, int N) {
    const int rb = std::max(1, kThreads / N);
    const int64_t want = (int64_t(ni) + rb - 1) / rb;
    // narrow blocks (N <= 2) move few bytes per row: two blocks per SM are enough to saturate HBM and keep the
    // per-block partials (and their fences) few
    const int64_t cap = int64_t(c.sm_count) * (N <= 2 ? 2 : 8);
    return int(std::max<int64_t>(1, std::min<int64_t>(want, cap)));
}

struct Plan {
    int G, CPL;
    bool split;
};

Plan plan_for(int N) {
    // measured on B200 at N = 16 (cfg2): 8 lanes x 2 columns at <= 64 registers (32 warps/SM) beats
    // 4 lanes x 4 columns (0.306 vs 0.368 ms per SpMM): the kernel is gather-latency bound, so
    // warps in flight matter more than loads per warp. KSB_SPMM_PLAN=4 selects the wide variant.
    // Later measurement: 4 lanes x 4 columns in the quad layout (one 256-bit load per gathered row per lane, a
    // warp covers 8 rows per gather and the (col, val) shuffles feed 8 rows instead of 4) -- see iteration().
    // KSB_SPMM_PLAN=8 selects 8 lanes x 2 columns, =4 the pair-layout 4 x 4.
    static const char* env = std::getenv("KSB_SPMM_PLAN");
    if (N == 16 && env && env[0] == '8') return {8, 2, false};
    if (N == 1) return {8, 1, true};
    if (N <= 4) return {2, 2, false};
    if (N <= 8) return {2, 4, false};
    if (N <= 16) return {4, 4, false};
    if (N <= 32) return {8, 4, false};
    if (N <= 64) return {16, 4, false};
    return {32, 4, false};
}

struct SellOps {
    const double *A = nullptr, *B = nullptr;  // SELL-32 values (N <= 2)
    const double* T8 = nullptr;               // T8 values (N = 16, no shift, rows of <= 16 entries)
    const double *UT = nullptr, *UTB = nullptr;  // union-tile values (wide blocks on a locality order), shift operator
    const double* DIA = nullptr;              // tiled stencil values (dia.cuh) for dia_g lanes per row
    int dia_g = 0;
    int dia_z = 0;                            // > 0: z-marching kernel, lines per block
    bool dia_zt = false;                      // TMA-staged z-marching kernel
    // CSR pattern the row kernels walk: the level's natural interior pattern, or its locality-ordered copy
    const int32_t *ptr = nullptr, *col = nullptr;
    int max_row = 0;
};

/// dst row i = src row perm[i] (scatter = 0) or dst row perm[i] = src row i (scatter = 1), N columns, stride ld
__global__ void k_permute_rows(int ni, int N, int ld, const int32_t* __restrict__ perm, const double* __restrict__ src,
                               double* __restrict__ dst, int scatter) {
    const int64_t total = int64_t(ni) * N;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(k / N), c = int(k % N);
        const int j = perm[i];
        if (scatter)
            dst[size_t(j) * ld + c] = src[size_t(i) * ld + c];
        else
            dst[size_t(i) * ld + c] = src[size_t(j) * ld + c];
    }
}

template <int NC, bool SHIFT>
void launch_sell(Ctx& c, const Level& L, const CgWork& w, const Cols& cc, const SellOps& so) {
    const size_t sm = sizeof(double) * std::max<size_t>(size_t(kThreads / 32) * NC, 2 * size_t(cc.N));
    const int want = ceil_div(L.nslices, kThreads / 32);
    const int g = std::max(1, std::min(want, resident_grid(c, k_sell_dot<NC, SHIFT>, kThreads, sm)));
    launch(c, "spmm", k_sell_dot<NC, SHIFT>, g, kThreads, sm, L.ni, L.nslices, cc, (const int32_t*)L.sell_ptr.p,
           (const int32_t*)L.sell_col.p, so.A, so.B, (const double*)w.P, w.AP, w.dev);
}

template <bool SHIFT>
bool try_sell(Ctx& c, const Level& L, const CgWork& w, const Cols& cc, const SellOps& so) {
    if (!so.A) return false;
    switch (cc.N) {
        case 1: launch_sell<1, SHIFT>(c, L, w, cc, so); return true;
        case 2: launch_sell<2, SHIFT>(c, L, w, cc, so); return true;
        default: return false;
    }
}

/// lanes per row of the stencil SpMM for an N-column block (0: no stencil kernel for this N).
/// KSB_DIA_G selects 4 / 8 / 16 lanes at N = 16 (default 8: 2 columns per lane).
int dia_prefetch() {
    const char* env = std::getenv("KSB_DIA_PF");
    return env ? std::atoi(env) : 0;
}

int dia_lanes(int N) {
    const char* env = std::getenv("KSB_DIA_G");  // read per solve (tests switch it)
    if (N == 16) {
        const int g = env ? std::atoi(env) : 8;
        return (g == 4 || g == 16) ? g : 8;
    }
    return 0;
}

/// z-marching stencil kernel on cubic grid levels (N = 16), opt-in: KSB_DIA_Z=4 / 8 lines per block. Measured on
/// cfg2 (profiles/README.md, r02): L2->L1 traffic halves (1.84 -> 0.90 GB per SpMM, L1 hit 12 -> 55 %) but the
/// kernel stays latency bound at 16 warps per SM and runs 0.27-0.46 ms against 0.22 ms for k_spmm_dia_tv.
int dia_z(const Level& L, int N) {
    const char* env = std::getenv("KSB_DIA_Z");
    if (N != 16 || L.dia_n == 0 || !env || env[0] == '0') return 0;
    return std::atoi(env) == 8 ? 8 : 4;
}

/// TMA-staged z-marching kernel (default on cubic grid levels with an N = 16, ld = 16 block; KSB_DIA_ZT=0 keeps the
/// band kernel)
bool dia_zt(const Level& L, int N, int ld) {
    const char* env = std::getenv("KSB_DIA_ZT");
    const int D = L.dia_ng > 0 ? 3 + (L.dia_ng - 1) * L.dia_lr : 0;
    // the plane and value rings must fit one block's shared memory (Kuhn 15-point: 222 KB; the 27-point box does not)
    return N == 16 && ld == 16 && L.dia_n >= 3 && D > 0 && dia_zt_smem(D) <= 227 * 1024 && !(env && env[0] == '0');
}

bool try_dia(Ctx& c, const Level& L, const CgWork& w, const Cols& cc, const SellOps& so) {
    if (!so.DIA) return false;
    const DiaGeom dg = dia_geom(L);
    if (so.dia_zt) {
        auto go_zt = [&](auto kern) {
            const size_t smt = dia_zt_smem(dg.D);
            static std::map<const void*, bool> attr;
            if (!attr[reinterpret_cast<const void*>(kern)]) {
                KSB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smt)));
                attr[reinterpret_cast<const void*>(kern)] = true;
            }
            const int n = dg.n, nt = ceil_div(n, kZtT);
            const int res = std::max(1, std::min(resident_grid(c, kern, kThreads, smt), w.cap_blocks));
            // z ranges: the length that balances the items over the resident blocks best (each item also loads two
            // halo planes, from L2)
            int nzc = 1;
            double best = 1e30;
            for (int lz = 3; lz <= std::min(n, 24); ++lz) {
                const int zc = ceil_div(n, lz);
                const double cost = double(ceil_div(int64_t(nt) * nt * zc, res)) * (lz + 0.5);
                if (cost < best) {
                    best = cost;
                    nzc = zc;
                }
            }
            const int grid = std::max(1, std::min(res, nt * nt * nzc));
            launch(c, "spmm", kern, grid, kThreads, smt, L.ni, cc, dg, nzc, so.DIA, (const double*)w.P, w.AP, w.dev);
            return true;
        };
        const char* zw = std::getenv("KSB_DIA_ZW");
        if (!(zw && zw[0] == '0')) {  // warp-specialised producer (default)
            auto kern = k_spmm_dia_zw<7, 2>;
            const size_t smt = dia_zt_smem(dg.D) + 6 * sizeof(uint64_t);
            static bool attr = false;
            if (!attr) {
                KSB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smt)));
                attr = true;
            }
            const int n = dg.n, nt = ceil_div(n, kZtT);
            const int res = std::max(1, std::min(resident_grid(c, kern, kZwThreads, smt), w.cap_blocks));
            int nzc = 1;
            double best = 1e30;
            for (int lz = 3; lz <= std::min(n, 24); ++lz) {
                const int zc = ceil_div(n, lz);
                const double cost = double(ceil_div(int64_t(nt) * nt * zc, res)) * (lz + 0.5);
                if (cost < best) {
                    best = cost;
                    nzc = zc;
                }
            }
            const int grid = std::max(1, std::min(res, nt * nt * nzc));
            if (L.dia_ng == 7) {
                launch(c, "spmm", kern, grid, kZwThreads, smt, L.ni, cc, dg, nzc, so.DIA, (const double*)w.P, w.AP,
                       w.dev);
                return true;
            }
        }
        if (L.dia_ng == 7) return go_zt(k_spmm_dia_zt<7, 2>);
        if (L.dia_ng == 9) return go_zt(k_spmm_dia_zt<9, 3>);
    }
    if (so.dia_z) {
        const size_t sm = sizeof(double) * std::max<size_t>(8 * size_t(cc.N), 2 * size_t(cc.N));
        auto go_z = [&](auto kern, int nw) {
            static std::map<const void*, bool> attr;
            if (!attr[reinterpret_cast<const void*>(kern)]) {
                KSB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                                    int(cudaSharedmemCarveoutMaxL1)));
                attr[reinterpret_cast<const void*>(kern)] = true;
            }
            const int n = dg.n, tiles = ceil_div(n, 32) * ceil_div(n, nw);
            const int res = resident_grid(c, kern, nw * 32, sm);
            const char* zc_env = std::getenv("KSB_DIA_ZC");
            const int nzc = std::max(1, std::min(n, zc_env ? std::atoi(zc_env) : ceil_div(res, tiles)));
            const int grid = std::max(1, std::min({res, tiles * nzc, w.cap_blocks}));
            launch(c, "spmm", kern, grid, nw * 32, sm, L.ni, cc, dg, nzc, so.DIA, (const double*)w.P, w.AP, w.dev);
            return true;
        };
        if (L.dia_ng == 7) return so.dia_z == 8 ? go_z(k_spmm_dia_z<7, 2, 8, 2>, 8) : go_z(k_spmm_dia_z<7, 2, 4, 4>, 4);
        if (L.dia_ng == 9) return so.dia_z == 8 ? go_z(k_spmm_dia_z<9, 3, 8, 2>, 8) : go_z(k_spmm_dia_z<9, 3, 4, 4>, 4);
    }
    const size_t sm = sizeof(double) * std::max<size_t>(size_t(kThreads / 32) * cc.N, 2 * size_t(cc.N));
    auto go = [&](auto kern, int G) {
        const int T = (32 / G) * kDiaS;
        const int want = ceil_div(ceil_div(L.ni, T), kThreads / 32);
        const int grid = std::max(1, std::min(want, resident_grid(c, kern, kThreads, sm)));
        launch(c, "spmm", kern, grid, kThreads, sm, L.ni, cc, dg, so.DIA, (const double*)w.P, w.AP, w.dev);
        return true;
    };
    const int pf = dia_prefetch();
    const char* tv = std::getenv("KSB_DIA_TV");
    if (!(tv && tv[0] == '0')) {  // staged values (default)
        const DiaGeom g2 = dg;
        auto go_tv = [&](auto kern, int G) {
            const size_t smt = dia_tv_smem(g2.D, 32 / G, cc.N);
            static std::map<const void*, bool> attr;
            if (!attr[reinterpret_cast<const void*>(kern)]) {
                KSB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smt)));
                attr[reinterpret_cast<const void*>(kern)] = true;
            }
            const int T = (32 / G) * kDiaS;
            const int want = ceil_div(ceil_div(L.ni, T), kThreads / 32);
            const int grid = std::max(1, std::min(want, resident_grid(c, kern, kThreads, smt)));
            launch(c, "spmm", kern, grid, kThreads, smt, L.ni, cc, g2, so.DIA, (const double*)w.P, w.AP, w.dev);
            return true;
        };
        const char* mb = std::getenv("KSB_DIA_MINB");
        if (L.dia_ng == 7 && so.dia_g == 8 && mb && mb[0] == '3') return go_tv(k_spmm_dia_tv<7, 2, 8, 2, 3>, 8);
        if (L.dia_ng == 7 && so.dia_g == 8) return go_tv(k_spmm_dia_tv<7, 2, 8, 2, 2>, 8);
        if (L.dia_ng == 7 && so.dia_g == 4) return go_tv(k_spmm_dia_tv<7, 2, 4, 4, 1>, 4);
        if (L.dia_ng == 9 && so.dia_g == 8) return go_tv(k_spmm_dia_tv<9, 3, 8, 2, 2>, 8);
    }
    if (L.dia_ng == 7) {
        switch (so.dia_g) {
            case 4: return pf ? go(k_spmm_dia<7, 2, 4, 4, 1, 4>, 4) : go(k_spmm_dia<7, 2, 4, 4, 1, 0>, 4);
            case 8:
                return pf >= 8 ? go(k_spmm_dia<7, 2, 8, 2, 2, 8>, 8)
                               : pf ? go(k_spmm_dia<7, 2, 8, 2, 2, 4>, 8) : go(k_spmm_dia<7, 2, 8, 2, 2, 0>, 8);
            case 16: return pf ? go(k_spmm_dia<7, 2, 16, 1, 3, 4>, 16) : go(k_spmm_dia<7, 2, 16, 1, 3, 0>, 16);
        }
    } else if (L.dia_ng == 9) {
        switch (so.dia_g) {
            case 4: return go(k_spmm_dia<9, 3, 4, 4, 1, 4>, 4);
            case 8: return go(k_spmm_dia<9, 3, 8, 2, 2, 4>, 8);
            case 16: return go(k_spmm_dia<9, 3, 16, 1, 3, 4>, 16);
        }
    }
    return false;
}

/// union-tile SpMM (blocks of more than 16 columns on levels with the view; cg_solve sets so.UT)
template <int G, bool SHIFT>
bool try_ut(Ctx& c, const Level& L, const CgWork& w, const Cols& cc, const SellOps& so) {
    if constexpr (G < 8) {
        return false;
    } else {
        if (!so.UT || (SHIFT && !so.UTB)) return false;
        constexpr int NT = 256;
        constexpr bool VSM = G == 32;  // one warp per tile: values staged with the columns
        auto go = [&](auto kern) {
            const size_t smt = ut_smem(G, NT, SHIFT, VSM);
            static std::map<const void*, bool> attr;  // (the variants share one function-pointer type)
            if (!attr[reinterpret_cast<const void*>(kern)]) {
                KSB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smt)));
                attr[reinterpret_cast<const void*>(kern)] = true;
            }
            const int want = ceil_div(ceil_div(L.ut_nt, 32 / G), NT / 32);
            const int grid = std::max(1, std::min({want, resident_grid(c, kern, NT, smt), w.cap_blocks}));
            const char* senv = std::getenv("KSB_UT_SYNC");  // read per launch (the probes switch it)
            int se = senv ? std::atoi(senv) : 16;
            if (se > 0) {  // resident grid: cooperative launch with the periodic grid barrier
                int nt = L.ut_nt;
                Cols ccv = cc;
                const int32_t* rows = L.ut_rows.p;
                const int32_t* ep = L.ut_eptr.p;
                const int32_t* en = L.ut_ent.p;
                const double* A = so.UT;
                const double* Bv = so.UTB;
                const double* Pp = w.P;
                double* APp = w.AP;
                CgDev dv = w.dev;
                void* args[] = {&nt, &ccv, &rows, &ep, &en, &A, &Bv, &Pp, &APp, &dv, &se};
                cudaEvent_t e0 = nullptr;
                if (c.profiling) c.begin("spmm", &e0);
                KSB_CUDA_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(NT),
                                                           args, smt, c.stream));
                ++c.launches;
                if (c.profiling) c.end("spmm", e0);
            } else {
                launch(c, "spmm", kern, grid, NT, smt, L.ut_nt, cc, (const int32_t*)L.ut_rows.p,
                       (const int32_t*)L.ut_eptr.p, (const int32_t*)L.ut_ent.p, so.UT, so.UTB, (const double*)w.P,
                       w.AP, w.dev, 0);
            }
            return true;
        };
        if constexpr (VSM) {
            static const char* ube = std::getenv("KSB_UT_UB");  // gathers in flight per lane group (experiments)
            if (ube && std::atoi(ube) == 4) return go(k_spmm_ut<G, SHIFT, 4, NT, 2, true>);
            if (ube && std::atoi(ube) == 43) return go(k_spmm_ut<G, SHIFT, 4, NT, 3, true>);
            const char* henv = std::getenv("KSB_UT_HINT");  // read per launch (probes)
            if (henv && henv[0] == '1') return go(k_spmm_ut<G, SHIFT, 8, NT, 2, true, true>);
            return go(k_spmm_ut<G, SHIFT, 8, NT, 2, true>);
        } else {
            return go(k_spmm_ut<G, SHIFT, 4, NT, 2, false>);
        }
    }
}

template <int G, int CPL, bool SHIFT, bool SPLIT, int FULL>
void launch_iteration(Ctx& c, const Level& L, const CgWork& w, const Cols& cc, const double* A, const double* Bv,
                      const double* Bb, double* X, int grid_s, int grid_e, const SellOps& so) {
    const size_t sm_s = sizeof(double) * std::max<size_t>(size_t(kThreads / G) * G * CPL, 2 * size_t(cc.N));
    const size_t sm_e = sizeof(double) * std::max<size_t>(2 * kThreads, 2 * size_t(cc.N));
    const bool v2 = (cc.N % 2 == 0) && (cc.ld % 2 == 0);
    grid_e = std::min(grid_e, v2 ? resident_grid(c, k_update_r<2>, kThreads, sm_e)
                                 : resident_grid(c, k_update_r<1>, kThreads, sm_e));
    if (try_sell<SHIFT>(c, L, w, cc, so)) {
    } else if (!SPLIT && try_ut<G, SHIFT>(c, L, w, cc, so)) {
    } else if (!SHIFT && try_dia(c, L, w, cc, so)) {
    } else {
        // resident blocks per SM the row kernel is compiled for. Lane groups of up to 16 (N <= 64) keep two (col, val)
        // chunk sets of 16 / G x G slots in registers: at 64 registers (4 blocks) they spill 70-340 bytes, at 128
        // (2 blocks) nothing -- configs[3] (N = 21, shifted): BVPs 1.98 -> 1.54 s. One row per warp (G = 32) keeps 4.
        static const char* mb = std::getenv("KSB_SPMM_MINB");
        const int minb = mb ? std::atoi(mb) : (G <= 16 ? 2 : KSB_SPMM_MINB);
        static const char* senv = std::getenv("KSB_SPMM_SYNC");
        static const char* denv = std::getenv("KSB_SPMM_DIE");
        const int die = denv ? std::atoi(denv) : 0;
        const int sync_every = G >= 16 ? ((senv ? std::atoi(senv) : 16) | (die << 16)) : 0;
        auto go = [&](auto kern) {
            grid_s = std::min(grid_s, resident_grid(c, kern, kThreads, sm_s));
            if (sync_every > 0) {
                int ni = L.ni;
                Cols ccv = cc;
                const int32_t* ptr = so.ptr;
                const int32_t* col = so.col;
                const double* Pp = w.P;
                double* APp = w.AP;
                CgDev dv = w.dev;
                int se = sync_every;
                void* args[] = {&ni, &ccv, &ptr, &col, &A, &Bv, &Pp, &APp, &dv, &se};
                cudaEvent_t e0 = nullptr;
                if (c.profiling) c.begin("spmm", &e0);
                KSB_CUDA_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid_s),
                                                           dim3(kThreads), args, sm_s, c.stream));
                ++c.launches;
                if (c.profiling) c.end("spmm", e0);
            } else {
                launch(c, "spmm", kern, grid_s, kThreads, sm_s, L.ni, cc, so.ptr, so.col, A, Bv, (const double*)w.P,
                       w.AP, w.dev, 0);
            }
        };
        // streamed gather pipeline (quad layout, N = 4G); KSB_SPMM_STREAM=0 selects k_spmm_dot
        static const char* st = std::getenv("KSB_SPMM_STREAM");
        bool streamed = false;
        static const char* t8e = std::getenv("KSB_SPMM_T8");
        if constexpr (FULL == 3 && !SHIFT && CPL == 4 && G == 4) {
            if (so.T8 && cc.N == 16 && !(t8e && t8e[0] == '0')) {
                auto kern = k_spmm_t8<8>;
                grid_s = std::min(grid_s, resident_grid(c, kern, kThreads, sm_s));
                launch(c, "spmm", kern, grid_s, kThreads, sm_s, L.ni, cc, (const int32_t*)L.t8_col.p, so.T8,
                       (const double*)w.P, w.AP, w.dev);
                streamed = true;
            }
        }
        if constexpr (FULL == 3 && !SHIFT && CPL == 4 && G <= 8) {
            if (!streamed && !(st && st[0] == '0') && so.max_row <= RowChunk<G, false>::NB * G) {
                auto kern = (G == 4 && minb != 3) ? k_spmm_stream<G, 8, 2> : k_spmm_stream<G, 4, 3>;
                grid_s = std::min(grid_s, resident_grid(c, kern, kThreads, sm_s));
                launch(c, "spmm", kern, grid_s, kThreads, sm_s, L.ni, cc, so.ptr, so.col, A, (const double*)w.P,
                       w.AP, w.dev);
                streamed = true;
            }
        }
        if (streamed) {
        } else if (FULL && minb == 4)
            go(k_spmm_dot<G, CPL, SHIFT, SPLIT, FULL, 4>);
        else if (FULL && minb == 5)
            go(k_spmm_dot<G, CPL, SHIFT, SPLIT, FULL, 5>);
        else if (FULL == 3 && minb == 3)
            go(k_spmm_dot<G, CPL, SHIFT, SPLIT, FULL, 3>);
        else if (minb == 2)
            go(k_spmm_dot<G, CPL, SHIFT, SPLIT, FULL, 2>);
        else
            go(k_spmm_dot<G, CPL, SHIFT, SPLIT, FULL>);
    }
    if (v2)
        launch(c, "cg_update_r", k_update_r<2>, grid_e, kThreads, sm_e, L.ni, cc, w.R, (const double*)w.AP, w.dev);
    else
        launch(c, "cg_update_r", k_update_r<1>, grid_e, kThreads, sm_e, L.ni, cc, w.R, (const double*)w.AP, w.dev);
    if (!cc.fixed)
        // runs every iteration but only works when a column was flagged; with many columns that is most
        // iterations (N = 120: 40 of 41), so it gets the SpMM's full resident grid (the early exit stays ~2 us)
        launch(c, "cg_trueres", k_trueres<G, CPL, SHIFT, SPLIT, FULL>, grid_s, kThreads, sm_s, L.ni, cc, so.ptr,
               so.col, A, Bv, Bb, (const double*)X,
               (const double*)w.AP, w.R, w.dev);
    // the x / p pass streams 5 blocks per row with no reduction: two blocks per SM beat the residual pass's grid
    // (cfg2: 0.205 vs 0.214 ms; 3 per SM 0.207), whose dot products want more blocks in flight
    const int grid_px = std::min(grid_e, 2 * c.sm_count);
    if (v2)
        launch(c, "cg_update_px", k_update_px<2>, grid_px, kThreads, 0, L.ni, cc, X, (const double*)w.R, w.P, w.dev);
    else
        launch(c, "cg_update_px", k_update_px<1>, grid_px, kThreads, 0, L.ni, cc, X, (const double*)w.R, w.P, w.dev);
}

template <bool SHIFT>
void iteration(Ctx& c, const Level& L, const CgWork& w, const Cols& cc, const double* A, const double* Bv,
               const double* Bb, double* X, int grid_s, int grid_e, const SellOps& so) {
    const Plan p = plan_for(cc.N);
    const bool full = !p.split && cc.N == p.G * p.CPL;
    // partial blocks (N < G*CPL) keep the interleaved layout with a pair tail mask when the leading dimension
    // is even (the pair straddling an odd N then ends inside the row)
    const bool tail = !p.split && !full && p.CPL == 4 && p.G >= 4 && cc.ld % 2 == 0;
    // quad layout (256-bit gathers): every slot in range, rows 32-byte aligned (all internal blocks are; X is the
    // caller's block, read by the true-residual pass)
    static const char* env = std::getenv("KSB_SPMM_PLAN");
    const bool quad = full && p.CPL == 4 && cc.ld % 4 == 0 && (reinterpret_cast<uintptr_t>(X) & 31) == 0 &&
                      !(env && (env[0] == '4' || env[0] == '8'));
    if (p.split)
        launch_iteration<8, 1, SHIFT, true, 0>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 2 && p.CPL == 2)
        launch_iteration<2, 2, SHIFT, false, 0>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 2)
        launch_iteration<2, 4, SHIFT, false, 0>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 8 && p.CPL == 2 && full)
        launch_iteration<8, 2, SHIFT, false, 1>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 4 && quad)
        launch_iteration<4, 4, SHIFT, false, 3>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 8 && quad)
        launch_iteration<8, 4, SHIFT, false, 3>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 16 && quad)
        launch_iteration<16, 4, SHIFT, false, 3>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 32 && quad)
        launch_iteration<32, 4, SHIFT, false, 3>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 4 && full)
        launch_iteration<4, 4, SHIFT, false, 1>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 4 && tail)
        launch_iteration<4, 4, SHIFT, false, 2>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 4)
        launch_iteration<4, 4, SHIFT, false, 0>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 8 && full)
        launch_iteration<8, 4, SHIFT, false, 1>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 8 && tail)
        launch_iteration<8, 4, SHIFT, false, 2>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 8)
        launch_iteration<8, 4, SHIFT, false, 0>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 16 && full)
        launch_iteration<16, 4, SHIFT, false, 1>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 16 && tail)
        launch_iteration<16, 4, SHIFT, false, 2>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (p.G == 16)
        launch_iteration<16, 4, SHIFT, false, 0>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (full)
        launch_iteration<32, 4, SHIFT, false, 1>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else if (tail)
        launch_iteration<32, 4, SHIFT, false, 2>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
    else
        launch_iteration<32, 4, SHIFT, false, 0>(c, L, w, cc, A, Bv, Bb, X, grid_s, grid_e, so);
}

} // namespace

CgWork::~CgWork() {
    for (auto& g : graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
}

void CgWork::forget_level(uint64_t uid) {
    for (size_t k = 0; k < graphs.size();) {
        if (graphs[k].key.level_uid == uid) {
            if (graphs[k].exec) cudaGraphExecDestroy(graphs[k].exec);
            graphs.erase(graphs.begin() + k);
        } else {
            ++k;
        }
    }
}

void CgWork::ensure(int ni, int N, int ld, int max_blocks) {
    const int64_t vec = int64_t(ni) * ld;
    if (vec > cap_vec) {
        rbuf.alloc(vec);
        pbuf.alloc(vec);
        apbuf.alloc(vec);
        cap_vec = vec;
    }
    R = rbuf.p;
    P = pbuf.p;
    AP = apbuf.p;
    if (N > cap_cols || max_blocks > cap_blocks) {
        cap_cols = std::max(N, cap_cols);
        cap_blocks = std::max(max_blocks, cap_blocks);
        scal.alloc(int64_t(cap_cols) * 8);
        ints.alloc(int64_t(cap_cols) * 4 + 16);
        parts.alloc(int64_t(cap_blocks) * cap_cols * 2);
    }
}

void cg_solve(Ctx& c, Level& L, int mat, int shift_mat, const double* h_sigma, const double* d_B, double* d_X, int N,
              int ld, const CgOptions& o, CgColumnStats* stats, CgWork& w) {
    if (N < 1 || N > 128) raise(KSB_INVALID_ARGUMENT, "cg: N must be in [1, 128]");
    if (ld < N || (N > 1 && (ld & 1))) raise(KSB_INVALID_ARGUMENT, "cg: ld must be >= N and even for N > 1");
    if (!L.mats[mat].valid) raise(KSB_INVALID_ARGUMENT, "cg: operator not assembled");
    const bool shift = shift_mat >= 0;
    if (shift && !L.mats[shift_mat].valid) raise(KSB_INVALID_ARGUMENT, "cg: shift operator not assembled");
    if (o.precond == 1) {  // the reference's exact SGS preconditioner (parity runs, sgs.cu)
        if (o.fixed_iterations > 0) raise(KSB_INVALID_ARGUMENT, "cg: the SGS path has no fixed-iteration mode");
        cg_solve_sgs(c, L, mat, shift_mat, h_sigma, d_B, d_X, N, ld, o, stats, w);
        return;
    }
    if (o.precond != 0) raise(KSB_INVALID_ARGUMENT, "cg: precond must be 0 (Jacobi) or 1 (SGS)");

    const Plan p = plan_for(N);
    const int rows_per_block = kThreads / p.G;
    const int grid_s = int(std::max<int64_t>(
        1, std::min<int64_t>((int64_t(L.ni) + rows_per_block - 1) / rows_per_block, int64_t(c.sm_count) * 8)));
    const int grid_e = elem_grid(c, L.ni, N);
    w.ensure(L.ni, N, ld, std::max(grid_s, grid_e));

    CgDev& d = w.dev;
    double* sc = w.scal.p;
    const int cap = w.cap_cols;
    d.bnorm = sc + 0 * cap;
    d.rz = sc + 1 * cap;
    d.rr = sc + 2 * cap;
    d.alpha = sc + 3 * cap;
    d.beta = sc + 4 * cap;
    d.relres = sc + 5 * cap;
    d.sigma = sc + 6 * cap;
    d.status = w.ints.p;
    d.check = w.ints.p + cap;
    d.iters = w.ints.p + 2 * cap;
    d.nonpos = w.ints.p + 3 * cap;
    d.ctl = w.ints.p + 4 * cap;
    d.part0 = w.parts.p;
    d.part1 = w.parts.p + int64_t(w.cap_blocks) * cap;
    // Multi-column solves on levels with a locality order (refined / adaptive numbering) run on the reordered
    // pattern: B and X are permuted in and X out once per solve, so the SpMM's gathered rows come from a band of
    // the block instead of the whole block (N = 120 at 2 M DOFs: the block is ~2 GB and otherwise re-read ~6x
    // from DRAM per SpMM). KSB_CG_REORDER=0 disables it.
    // Blocks that fit in L2 anyway (< 48 MB: N = 21 at 250 k DOFs) keep the natural order and skip the permutes.
    const char* roenv = std::getenv("KSB_CG_REORDER");  // read per solve (tests switch it)
    const bool lo = N >= 4 && L.lo_perm.n == L.ni && L.ni > 0 && !(roenv && roenv[0] == '0') &&
                    ((roenv && roenv[0] == '2') || int64_t(L.ni) * ld * 8 > (int64_t(48) << 20));
    const int32_t* dslot = lo ? L.lo_dslot.p : L.diag_slot.p;
    const double* A = lo ? L.lo_values(mat) : L.mats[mat].ii.p;
    const double* Bv = shift ? (lo ? L.lo_values(shift_mat) : L.mats[shift_mat].ii.p) : nullptr;
    double* X_user = d_X;
    if (lo) {
        const int64_t vec = int64_t(L.ni) * ld;
        if (w.lo_b.n < vec) w.lo_b.alloc(vec);
        const int gp = elem_grid(c, L.ni, N);
        launch(c, "cg_setup", k_permute_rows, gp, kThreads, 0, L.ni, N, ld, (const int32_t*)L.lo_perm.p, d_B,
               w.lo_b.p, 0);
        // X is not permuted in: k_init starts every column from x0 = 0 (proj/src/solver.cpp:59). The caller's X
        // holds the ordered iterate during the solve and is put back in place at the end (through the free R block)
        d_B = w.lo_b.p;
    }
    if (w.diagA.n < L.ni) w.diagA.alloc(L.ni);
    if (w.diagB.n < L.ni) w.diagB.alloc(L.ni);
    launch(c, "cg_setup", k_diag, elem_grid(c, L.ni, 1), kThreads, 0, L.ni, dslot, A, w.diagA.p);
    d.diagA = w.diagA.p;
    d.diagB = nullptr;
    std::vector<double> sig(N, 0.0);
    if (shift) {
        launch(c, "cg_setup", k_diag, elem_grid(c, L.ni, 1), kThreads, 0, L.ni, dslot, Bv, w.diagB.p);
        d.diagB = w.diagB.p;
        if (h_sigma) std::copy(h_sigma, h_sigma + N, sig.begin());
    }
    KSB_CUDA_CHECK(cudaMemcpyAsync(d.sigma, sig.data(), sizeof(double) * N, cudaMemcpyHostToDevice, c.stream));
    KSB_CUDA_CHECK(cudaMemsetAsync(d.ctl, 0, sizeof(int) * 16, c.stream));

    Cols cc{N, ld, o.tol, o.fixed_iterations > 0 ? 1 : 0};
    const size_t sm_e = sizeof(double) * std::max<size_t>(kThreads, 2 * size_t(N));
    launch(c, "cg_setup", k_init, grid_e, kThreads, sm_e, L.ni, cc, d_B, d_X, w.R, w.P, d);

    SellOps so;
    so.ptr = lo ? L.lo_ptr.p : L.ii_ptr.p;
    so.col = lo ? L.lo_col.p : L.ii_col.p;
    so.max_row = lo ? L.lo_max_row : L.max_row_ii;
    if (N == 1 || N == 2) {  // thread-per-row SELL wins for narrow blocks; wider blocks use lane groups
        so.A = L.sell_values(mat);
        so.B = shift ? L.sell_values(shift_mat) : nullptr;
    }
    if (N == 16 && !shift) so.T8 = L.t8_values(mat);
    // blocks of more than 16 columns on a locality order: the union-tile SpMM (KSB_SPMM_UT=0 keeps the row kernel)
    const char* ut_env = std::getenv("KSB_SPMM_UT");
    // (measured on configs[3], N = 21: 8 lanes per tile run at 6 warps per SM and lose to the row kernel, 2.8 vs 2.3 ms
    // per SpMM, so narrower blocks take the view only with KSB_SPMM_UT=2)
    const int ut_min_g = (ut_env && ut_env[0] == '2') ? 8 : 32;
    if (lo && p.G >= ut_min_g && L.ut_nt > 0 && ld % 2 == 0 && !(ut_env && ut_env[0] == '0')) {
        so.UT = L.ut_values(mat);
        so.UTB = shift ? L.ut_values(shift_mat) : nullptr;
    }
    // stencil levels (cfg2's lexicographic box, uniformly refined levels in the locality order): the sliding-window
    // SpMM; KSB_SPMM_DIA=0 keeps the CSR / T8 kernels
    const char* dia_env = std::getenv("KSB_SPMM_DIA");
    if (!shift && L.dia_ng > 0 && L.dia_lo == int(lo) && dia_lanes(N) > 0 && !(dia_env && dia_env[0] == '0') &&
        ld % 2 == 0) {
        so.dia_g = dia_lanes(N);
        so.dia_zt = dia_zt(L, N, ld);
        so.dia_z = so.dia_zt ? 0 : dia_z(L, N);
        so.DIA = L.dia_values(mat, so.dia_zt ? kDiaZT : so.dia_z ? kDiaLine : 32 / so.dia_g);
    }
    const int total = cc.fixed ? o.fixed_iterations : o.max_iterations;
    const int every = std::max(1, o.check_every);
    auto run_chunk = [&](int chunk) {
        for (int k = 0; k < chunk; ++k) {
            if (shift)
                iteration<true>(c, L, w, cc, A, Bv, d_B, d_X, grid_s, grid_e, so);
            else
                iteration<false>(c, L, w, cc, A, nullptr, d_B, d_X, grid_s, grid_e, so);
        }
    };
    // After the first chunk (which also warms the occupancy caches), chunks replay as CUDA graphs: one launch
    // per check_every iterations instead of 3-4 per iteration. Off while profiling (per-kernel events) or with
    // KSB_CG_GRAPHS=0.
    static const char* genv = std::getenv("KSB_CG_GRAPHS");
    const bool graphs_on = !c.profiling && !(genv && genv[0] == '0');
    auto graph_for = [&](int chunk) -> CgGraph& {
        CgGraphKey key;
        std::memset(&key, 0, sizeof key);
        key.level_uid = L.uid;
        // every pointer a captured kernel dereferences
        const void* ptrs[29] = {A, Bv, d_B, d_X, so.A, so.B, w.R, w.P, w.AP, w.scal.p, w.parts.p, w.ints.p,
                                d.diagA, d.diagB, so.ptr, so.col, so.T8, L.t8_col.p, L.sell_ptr.p, L.sell_col.p,
                                L.ii_ptr.p, L.ii_col.p, L.lo_ptr.p, L.lo_col.p, so.DIA, so.UT, so.UTB, L.ut_ent.p,
                                L.ut_rows.p};
        std::memcpy(key.ptrs, ptrs, sizeof ptrs);
        const int ints[10] = {mat, shift_mat, N, ld, chunk, grid_s, grid_e, cc.fixed, L.ni, L.nslices * 64 + so.dia_g * 2 + (so.dia_z > 0) + (so.dia_zt ? 1 << 30 : 0)};
        std::memcpy(key.ints, ints, sizeof ints);
        key.tol = cc.tol;
        for (auto& g : w.graphs)
            if (std::memcmp(&g.key, &key, sizeof key) == 0) return g;
        if (w.graphs.size() >= 8) {
            cudaGraphExecDestroy(w.graphs.front().exec);
            w.graphs.erase(w.graphs.begin());
        }
        CgGraph g;
        g.key = key;
        const int64_t l0 = c.launches;
        KSB_CUDA_CHECK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeRelaxed));
        try {
            run_chunk(chunk);
        } catch (...) {
            cudaGraph_t bad = nullptr;
            cudaStreamEndCapture(c.stream, &bad);
            if (bad) cudaGraphDestroy(bad);
            throw;
        }
        cudaGraph_t graph = nullptr;
        KSB_CUDA_CHECK(cudaStreamEndCapture(c.stream, &graph));
        g.kernels = c.launches - l0;
        c.launches = l0;
        KSB_CUDA_CHECK(cudaGraphInstantiate(&g.exec, graph, 0));
        cudaGraphDestroy(graph);
        w.graphs.push_back(g);
        return w.graphs.back();
    };
    // N <= 2: the whole solve is one cooperative launch (the kernel stops itself once no column is active)
    static const char* cenv = std::getenv("KSB_CG_COOP");
    if (so.A && N <= 2 && !(cenv && cenv[0] == '0')) {
        auto coop = [&](auto kern) {
            const int block = kThreads;
            // resident blocks per SM for the cooperative grid: KSB_COOP_BLOCKS_PER_SM (default 2; fewer blocks make
            // the grid barriers cheaper but leave the SpMV phase latency bound)
            static const char* bpe = std::getenv("KSB_COOP_BLOCKS_PER_SM");
            const int bps = bpe ? std::max(1, std::atoi(bpe)) : 2;
            const int want = std::max(1, ceil_div(L.nslices, 2 * (block / 32)));
            const int grid =
                std::max(1, std::min({want, resident_grid(c, kern, block, 0), c.sm_count * bps}));
            int ni = L.ni, nsl = L.nslices, iters = total;
            const int32_t* sptr = L.sell_ptr.p;
            const int32_t* scol = L.sell_col.p;
            const double* sA = so.A;
            const double* sB = so.B;
            const double* Bb = d_B;
            double* Xp = d_X;
            double* Rp = w.R;
            double* Pp = w.P;
            double* APp = w.AP;
            CgDev dv = d;
            void* args[] = {&ni, &nsl, &cc, &sptr, &scol, &sA, &sB, &Bb, &Xp, &Rp, &Pp, &APp, &dv, &iters};
            cudaEvent_t e0 = nullptr;
            if (c.profiling) c.begin("cg_coop", &e0);
            KSB_CUDA_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(block),
                                                       args, 0, c.stream));
            ++c.launches;
            if (c.profiling) c.end("cg_coop", e0);
        };
        if (N == 1) {
            if (shift)
                coop(k_cg_coop<1, true>);
            else
                coop(k_cg_coop<1, false>);
        } else {
            if (shift)
                coop(k_cg_coop<2, true>);
            else
                coop(k_cg_coop<2, false>);
        }
    }
    int done = (so.A && N <= 2 && !(cenv && cenv[0] == '0')) ? total : 0;
    while (done < total) {
        const int chunk = std::min(every, total - done);
        if (graphs_on && done > 0) {
            CgGraph& g = graph_for(chunk);
            KSB_CUDA_CHECK(cudaGraphLaunch(g.exec, c.stream));
            c.launches += g.kernels;
        } else {
            run_chunk(chunk);
        }
        done += chunk;
        if (!cc.fixed) {
            int ctl[16];
            KSB_CUDA_CHECK(cudaMemcpyAsync(ctl, d.ctl, sizeof ctl, cudaMemcpyDeviceToHost, c.stream));
            KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
            if (ctl[kNActive] == 0) break;
        }
    }
    if (lo) {
        KSB_CUDA_CHECK(cudaMemcpyAsync(w.R, d_X, sizeof(double) * size_t(L.ni) * ld, cudaMemcpyDeviceToDevice, c.stream));
        launch(c, "cg_setup", k_permute_rows, elem_grid(c, L.ni, N), kThreads, 0, L.ni, N, ld,
               (const int32_t*)L.lo_perm.p, (const double*)w.R, X_user, 1);
    }
    if (stats) {
        std::vector<int> st(N), it(N), np(N);
        std::vector<double> rel(N);
        KSB_CUDA_CHECK(cudaMemcpyAsync(st.data(), d.status, sizeof(int) * N, cudaMemcpyDeviceToHost, c.stream));
        KSB_CUDA_CHECK(cudaMemcpyAsync(np.data(), d.nonpos, sizeof(int) * N, cudaMemcpyDeviceToHost, c.stream));
        KSB_CUDA_CHECK(cudaMemcpyAsync(it.data(), d.iters, sizeof(int) * N, cudaMemcpyDeviceToHost, c.stream));
        KSB_CUDA_CHECK(cudaMemcpyAsync(rel.data(), d.relres, sizeof(double) * N, cudaMemcpyDeviceToHost, c.stream));
        KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
        for (int j = 0; j < N; ++j) {
            stats[j].iterations = it[j];
            stats[j].relative_residual = rel[j];
            stats[j].converged = st[j] == kConverged;
            // fixed-iteration mode: the number of iterations that saw !(p.Ap > 0) (the column kept iterating)
            stats[j].breakdown = cc.fixed ? np[j] : int(st[j] == kBreakdown);
        }
    }
}

} // namespace ksb
