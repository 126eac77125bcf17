// K-BEIG + coarse sweep kernels: corr::inner_scf on the device.
//
// Reference: proj/src/correction.cpp:225-368 (inner_scf, A_H2, b_H2, beta2, f_H, g) and the
// dense bordered eigensolve + selection rule proj/src/eigensolve.cpp:371-396,425-443.
// The reference solves one (N_H+1)-dimensional generalized eigenproblem per orbital per
// sweep. Here the coarse mass Cholesky factor L_H is shared by all orbitals, so each
// bordered pencil reduces to  [C11 c12; c12^T c22]  with the SAME C11 = L_H^-1 A_H L_H^-T for
// every orbital. C11 is tridiagonalised once per sweep (Householder, one CTA); every
// orbital's problem is then an arrow-tridiagonal matrix [T c^; c^T c22] whose inertia at a
// shift is one O(N_H) LDL^T pass (Sylvester), so the lowest nev eigenvalues come from
// warp-parallel multisection and each eigenvector from one tridiagonal solve.
#include <algorithm>
#include <cfloat>

#include <cooperative_groups.h>

#include "geom.cuh"
#include "inner.cuh"

namespace ksb {

namespace {

// ------------------------------------------------------------------------------------------
// dense helpers (row-major n x n)

/// single-CTA Cholesky, lower factor in place (upper part zeroed). flag[0] = 1 if not SPD.
__global__ void k_potrf(int n, double* __restrict__ A, int* __restrict__ flag) {
    __shared__ double piv;
    for (int j = 0; j < n; ++j) {
        // A[j][j] -= sum_k<j A[j][k]^2 (lane-parallel over k, fixed order)
        if (threadIdx.x < 32) {
            double s = 0.0;
            for (int k = threadIdx.x; k < j; k += 32) s += A[size_t(j) * n + k] * A[size_t(j) * n + k];
            s = warp_sum(s);
            if (threadIdx.x == 0) {
                const double d = A[size_t(j) * n + j] - s;
                if (!(d > 0.0) || !isfinite(d)) flag[0] = 1;
                piv = sqrt(fmax(d, DBL_MIN));
                A[size_t(j) * n + j] = piv;
            }
        }
        __syncthreads();
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        for (int i = j + 1 + warp; i < n; i += nw) {
            double s = 0.0;
            for (int k = lane; k < j; k += 32) s += A[size_t(i) * n + k] * A[size_t(j) * n + k];
            s = warp_sum(s);
            if (lane == 0) A[size_t(i) * n + j] = (A[size_t(i) * n + j] - s) / piv;
        }
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x)
        if (idx % n > idx / n) A[idx] = 0.0;
}

/// warp-per-RHS triangular solve with the lower factor L (row-major):
///   trans = 0: L x = b ;  trans = 1: L^T x = b.
/// RHS j element k at B[j*bs + k*bc]; solution to X[j*xs + k*xc] (may alias B with equal strides).
__global__ void k_trsv_many(int n, int nrhs, const double* __restrict__ L, int trans, const double* B, int64_t bs,
                            int64_t bc, double* X, int64_t xs, int64_t xc, double scale) {
    extern __shared__ double ys[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x * (blockDim.x >> 5) + warp;
    if (j >= nrhs) return;
    double* y = ys + size_t(warp) * n;
    for (int k = lane; k < n; k += 32) y[k] = scale * B[j * bs + k * bc];
    __syncwarp();
    if (!trans) {
        for (int i = 0; i < n; ++i) {
            double s = 0.0;
            for (int k = lane; k < i; k += 32) s += L[size_t(i) * n + k] * y[k];
            s = warp_sum(s);
            if (lane == 0) y[i] = (y[i] - s) / L[size_t(i) * n + i];
            __syncwarp();
        }
    } else {
        for (int i = n - 1; i >= 0; --i) {
            double s = 0.0;
            for (int k = i + 1 + lane; k < n; k += 32) s += L[size_t(k) * n + i] * y[k];
            s = warp_sum(s);
            if (lane == 0) y[i] = (y[i] - s) / L[size_t(i) * n + i];
            __syncwarp();
        }
    }
    for (int k = lane; k < n; k += 32) X[j * xs + k * xc] = y[k];
}

/// lane-strided dot of a row with a vector, four independent accumulators: four row loads in flight per lane
/// (a single accumulator chain stalls the warp on every load -- these dense coarse kernels are latency-bound)
__device__ __forceinline__ double lane_dot(const double* __restrict__ a, const double* x, int n, int lane) {
    double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
    int c = lane;
    for (; c + 96 < n; c += 128) {
        t0 = fma(a[c], x[c], t0);
        t1 = fma(a[c + 32], x[c + 32], t1);
        t2 = fma(a[c + 64], x[c + 64], t2);
        t3 = fma(a[c + 96], x[c + 96], t3);
    }
    for (; c < n; c += 32) t0 = fma(a[c], x[c], t0);
    return (t0 + t1) + (t2 + t3);
}

/// Y[v*ldy + r] = alpha * sum_c A[r*lda + c] X[v*ldx + c] for r < n, v < nv (warp per (row, vector)).
/// The explicit inverse factors (L_H^-1, L_H^-T, C_H^-1, built once per level) turn every triangular
/// solve of the inner sweep into this fully parallel product.
__global__ void k_gemv_many(int n, int m, int nv, const double* __restrict__ A, int lda, const double* __restrict__ X,
                            int64_t ldx, double* __restrict__ Y, int64_t ldy, double alpha) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n * nv) return;
    const int r = warp % n, v = warp / n;
    const double* a = A + size_t(r) * lda;
    const double* x = X + size_t(v) * ldx;
    double t = lane_dot(a, x, m, lane);
    t = warp_sum(t);
    if (lane == 0) Y[size_t(v) * ldy + r] = alpha * t;
}

/// block-wide y = A x (A row-major n x n in global, x and y in shared memory), warp per row
__device__ void block_gemv(int n, const double* __restrict__ A, const double* x, double* y) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int r = warp; r < n; r += nw) {
        double t = lane_dot(A + size_t(r) * n, x, n, lane);
        t = warp_sum(t);
        if (lane == 0) y[r] = t;
    }
}

/// C = A B^T for n x n row-major A, B (32 x 32 output tiles, k in fixed ascending order)
__global__ void __launch_bounds__(256) k_gemm_nt(int n, const double* __restrict__ A, const double* __restrict__ B,
                                                 double* __restrict__ C) {
    __shared__ double As[32][33], Bs[32][33];
    const int bi = blockIdx.y * 32, bj = blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k0 = 0; k0 < n; k0 += 32) {
        for (int r = ty; r < 32; r += 8) {
            As[r][tx] = (bi + r < n && k0 + tx < n) ? A[size_t(bi + r) * n + k0 + tx] : 0.0;
            Bs[r][tx] = (bj + r < n && k0 + tx < n) ? B[size_t(bj + r) * n + k0 + tx] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
            const double b = Bs[tx][k];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(As[ty + 8 * q][k], b, acc[q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (bi + ty + 8 * q < n && bj + tx < n) C[size_t(bi + ty + 8 * q) * n + bj + tx] = acc[q];
}

__global__ void k_identity(int n, double* __restrict__ I) {
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x)
        I[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
}

/// single-CTA Householder tridiagonalisation of symmetric C (row-major, destroyed).
/// d[n], e[n-1]; V row k holds the unit Householder vector of step k in entries k+1..n-1.
__global__ void __launch_bounds__(1024) k_tridiag(int n, double* __restrict__ C, double* __restrict__ d,
                                                  double* __restrict__ e, double* __restrict__ V) {
    extern __shared__ double sh[];
    double* v = sh;          // n
    double* p = sh + n;      // n
    __shared__ double red[32];
    __shared__ double bc[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int k = 0; k + 2 < n; ++k) {
        const int m0 = k + 1, m = n - m0;
        // column k below the diagonal = row k right of the diagonal (symmetry)
        double s = 0.0;
        for (int i = tid; i < m; i += blockDim.x) {
            const double x = C[size_t(k) * n + m0 + i];
            v[m0 + i] = x;
            s += x * x;
        }
        s = warp_sum(s);
        if (lane == 0) red[warp] = s;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += red[w];
            const double nx = sqrt(t);
            const double x0 = v[m0];
            const double alpha = x0 >= 0.0 ? -nx : nx;
            const double nv2 = t - x0 * x0 + (x0 - alpha) * (x0 - alpha);
            bc[0] = alpha;
            bc[1] = (nx == 0.0 || nv2 <= 0.0) ? 0.0 : 1.0 / sqrt(nv2);
            v[m0] = x0 - alpha;
        }
        __syncthreads();
        const double alpha = bc[0], inv = bc[1];
        d[k] = C[size_t(k) * n + k];  // every thread writes the same value; harmless
        if (tid == 0) e[k] = inv == 0.0 ? v[m0] + alpha : alpha;
        if (inv == 0.0) {  // nothing to annihilate: identity reflector
            for (int i = tid; i < m; i += blockDim.x) V[size_t(k) * n + m0 + i] = 0.0;
            __syncthreads();
            continue;
        }
        for (int i = tid; i < m; i += blockDim.x) {
            v[m0 + i] *= inv;
            V[size_t(k) * n + m0 + i] = v[m0 + i];
        }
        __syncthreads();
        // p = C22 v (warp per row)
        for (int r = warp; r < m; r += nw) {
            const double* row = C + size_t(m0 + r) * n + m0;
            double t = 0.0;
            for (int c = lane; c < m; c += 32) t += row[c] * v[m0 + c];
            t = warp_sum(t);
            if (lane == 0) p[m0 + r] = t;
        }
        __syncthreads();
        // K = v.p ; q = p - K v (stored in p)
        s = 0.0;
        for (int i = tid; i < m; i += blockDim.x) s += v[m0 + i] * p[m0 + i];
        s = warp_sum(s);
        if (lane == 0) red[warp] = s;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += red[w];
            bc[0] = t;
        }
        __syncthreads();
        const double K = bc[0];
        for (int i = tid; i < m; i += blockDim.x) p[m0 + i] -= K * v[m0 + i];
        __syncthreads();
        // C22 -= 2 (v q^T + q v^T)
        for (int idx = tid; idx < m * m; idx += blockDim.x) {
            const int r = idx / m, c = idx % m;
            C[size_t(m0 + r) * n + m0 + c] -= 2.0 * (v[m0 + r] * p[m0 + c] + p[m0 + r] * v[m0 + c]);
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (n >= 2) {
            d[n - 2] = C[size_t(n - 2) * n + n - 2];
            e[n - 2] = C[size_t(n - 1) * n + n - 2];
        }
        if (n >= 1) d[n - 1] = C[size_t(n - 1) * n + n - 1];
    }
}

constexpr int kTriCluster = 8;

/// register slot r / 32 of a lane-distributed vector (element r lives on lane r % 32), unrolled select
template <int S>
__device__ __forceinline__ double reg_at(const double (&x)[S], int r) {
    double t = 0.0;
    const int j = r >> 5;
#pragma unroll
    for (int s = 0; s < S; ++s) t = (s == j) ? x[s] : t;
    return __shfl_sync(0xffffffffu, t, r & 31);
}

constexpr int kTriS = 12;  // register slots per lane: n <= 384

/// Cluster-of-8 Householder tridiagonalisation, one cluster barrier per step.
/// Rows are dealt cyclically: CTA q keeps rows q, q+8, q+16, ... of C in shared memory (343 x 343 doubles =
/// 941 KB over 8 SMs) and slot i of a CTA belongs to warp i % 8, so the active trailing rows stay balanced
/// over all 64 warps as the reduction proceeds. Every warp carries the pivot row, the Householder vector v
/// and w = p - (v.p) v in registers (element c on lane c % 32) and recomputes the scalars redundantly.
/// Per step the only exchange is p = C v: each warp pushes its rows' entries into every CTA's p buffer
/// (distributed shared memory stores), then one cluster barrier. The pivot rows travel in blocks of
/// kTriRep: every kTriRep steps their owners push the next block into a replica in every CTA, and each CTA
/// applies the per-step rank-2 updates to its replica locally, so the next pivot row is always local.
/// p and the replica are double-buffered, which makes the single barrier safe.
constexpr int kTriThreads = 256;
constexpr int kMaxDynSmem = 227 * 1024;  // sm_100 per-block opt-in shared memory
constexpr int kTriRep = kTriThreads / 32;  // one replica row per warp

__global__ void __cluster_dims__(kTriCluster, 1, 1) __launch_bounds__(kTriThreads, 1)
    k_tridiag_cluster(int n, int R, const double* __restrict__ Cin, double* __restrict__ d, double* __restrict__ e,
                      double* __restrict__ V) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ double sh[];
    constexpr int P = kTriCluster;
    const int q = int(cluster.block_rank());
    const int nslot = (n - q + P - 1) / P;     // rows q + P i < n
    double* A = sh;                            // R x n, slot i = row q + P i
    double* pbuf = sh + size_t(R) * n;         // 2 x n
    double* rep = pbuf + 2 * size_t(n);        // 2 x kTriRep x n
    double* vsh = rep + 2 * size_t(kTriRep) * n;  // n: this step's v (row scalars of the rank-2 update)
    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5, nw = blockDim.x >> 5;
    for (int idx = tid; idx < nslot * n; idx += blockDim.x) {
        const int i = idx / n, c = idx - i * n;
        A[idx] = Cin[size_t(q + P * i) * n + c];
    }
    double cur[kTriS];
#pragma unroll
    for (int s = 0; s < kTriS; ++s) {
        const int c = lane + 32 * s;
        cur[s] = c < n ? Cin[c] : 0.0;
    }
    cluster.sync();
    for (int k = 0; k + 2 < n; ++k) {
        const int m0 = k + 1;
        const int par = k & 1;
        const int blk = k / kTriRep;
        const int rb0 = 1 + blk * kTriRep;  // first pivot row of the replica block in use this step
        double* repb = rep + size_t(blk & 1) * kTriRep * n;
        const int s0 = m0 >> 5;  // register slots below s0 hold only finished columns
        // reflector from the pivot row (every warp, redundantly)
        double ss = 0.0;
#pragma unroll
        for (int s = 0; s < kTriS; ++s) {
            const int c = lane + 32 * s;
            if (s >= s0 && c >= m0 && c < n) ss = fma(cur[s], cur[s], ss);
        }
        ss = warp_sum(ss);
        const double x0 = reg_at(cur, m0);
        const double nx = sqrt(ss);
        const double alpha = x0 >= 0.0 ? -nx : nx;
        const double nv2 = ss - x0 * x0 + (x0 - alpha) * (x0 - alpha);
        const double inv = (nx == 0.0 || nv2 <= 0.0) ? 0.0 : 1.0 / sqrt(nv2);
        double v[kTriS];
#pragma unroll
        for (int s = 0; s < kTriS; ++s) {
            const int c = lane + 32 * s;
            v[s] = (c >= m0 && c < n) ? (c == m0 ? x0 - alpha : cur[s]) * inv : 0.0;
        }
        const double dk = reg_at(cur, k);
        if (wib == 0) {  // v for the row scalars; read after the cluster barrier below
#pragma unroll
            for (int s = 0; s < kTriS; ++s) {
                const int c = lane + 32 * s;
                if (s >= s0 && c < n) vsh[c] = v[s];
            }
        }
        if (q == 0 && wib == 0) {
            if (lane == 0) {
                d[k] = dk;
                e[k] = inv == 0.0 ? x0 : alpha;
            }
#pragma unroll
            for (int s = 0; s < kTriS; ++s) {
                const int c = lane + 32 * s;
                if (s >= s0 && c >= m0 && c < n) V[size_t(k) * n + c] = v[s];
            }
        }
        // every kTriRep steps: the owners push the next block of pivot rows (updated through step k-1)
        if (k % kTriRep == 0) {
            __syncthreads();  // the rows' own warps finished last step's update
            const int hi = min(rb0 + kTriRep, n - 1);
            for (int rr = rb0; rr < hi; ++rr) {
                if (rr % P != q) continue;
                const double* src = A + size_t(rr / P) * n;
                for (int idx = tid; idx < P * n; idx += blockDim.x) {
                    const int t = idx / n, c = idx - t * n;
                    cluster.map_shared_rank(repb, t)[size_t(rr - rb0) * n + c] = src[c];
                }
            }
        }
        // first own slot at or past row m0, then every nw-th slot belongs to this warp
        const int i0 = m0 > q ? (m0 - q + P - 1) / P : 0;
        const int ifirst = i0 + ((wib - i0 % nw) % nw + nw) % nw;
        // p = C v for the own rows, pushed to every CTA
        for (int i = ifirst; i < nslot; i += nw) {
            const double* row = A + size_t(i) * n;
            double t = 0.0;
#pragma unroll
            for (int s = 0; s < kTriS; ++s) {
                const int c = lane + 32 * s;
                if (s >= s0 && c < n) t = fma(row[c], v[s], t);
            }
            t = warp_sum(t);
            if (lane < P) cluster.map_shared_rank(pbuf, lane)[size_t(par) * n + q + P * i] = t;
        }
        cluster.sync();
        // w = p - (v.p) v
        const double* pf = pbuf + size_t(par) * n;
        double kk = 0.0;
        double w[kTriS];
#pragma unroll
        for (int s = 0; s < kTriS; ++s) {
            const int c = lane + 32 * s;
            w[s] = (s >= s0 && c >= m0 && c < n) ? pf[c] : 0.0;
            kk = fma(v[s], w[s], kk);
        }
        kk = warp_sum(kk);
#pragma unroll
        for (int s = 0; s < kTriS; ++s) w[s] = fma(-kk, v[s], w[s]);
        // replica rows still ahead take this step's update (warp j owns replica row j)
        {
            const int rr = rb0 + wib;
            if (rr >= m0 && rr < n - 1) {
                const double vr = 2.0 * vsh[rr], wr = 2.0 * fma(-kk, vsh[rr], pf[rr]);
                double* row = repb + size_t(wib) * n;
#pragma unroll
                for (int s = 0; s < kTriS; ++s) {
                    const int c = lane + 32 * s;
                    if (s >= s0 && c >= m0 && c < n) row[c] -= vr * w[s] + wr * v[s];
                }
            }
        }
        // rank-2 update of the own slab rows
        for (int i = ifirst; i < nslot; i += nw) {
            double* row = A + size_t(i) * n;
            const int r = q + P * i;
            const double vr = 2.0 * vsh[r], wr = 2.0 * fma(-kk, vsh[r], pf[r]);
#pragma unroll
            for (int s = 0; s < kTriS; ++s) {
                const int c = lane + 32 * s;
                if (s >= s0 && c >= m0 && c < n) row[c] -= vr * w[s] + wr * v[s];
            }
        }
        __syncthreads();  // replica row k+1 complete
        const double* nxt = repb + size_t(m0 - rb0) * n;
#pragma unroll
        for (int s = 0; s < kTriS; ++s) {
            const int c = lane + 32 * s;
            cur[s] = c < n ? nxt[c] : 0.0;
        }
    }
    // tail: rows n-2 and n-1 of the final matrix (row n-1 was updated by its own warp)
    __syncthreads();
    if (n >= 2 && q == 0 && wib == 0) {
        const double dn2 = reg_at(cur, n - 2), en2 = reg_at(cur, n - 1);
        if (lane == 0) {
            d[n - 2] = dn2;
            e[n - 2] = en2;
        }
    }
    if (n >= 1 && (n - 1) % P == q && tid == 0) d[n - 1] = A[size_t((n - 1) / P) * n + n - 1];
    if (n == 1 && q == 0 && tid == 0) d[0] = Cin[0];
    cluster.sync();  // keep remote shared memory alive until every push has landed
}

/// apply Q^T (forward = 1: H_0 first) or Q (forward = 0: H_{n-3} first) to one vector, one warp.
/// For n <= 32 kQR the vector lives in registers (element i on lane i % 32, slot i / 32) and the next
/// reflector's row is prefetched while the current one is applied, so the 341-step chain pays the
/// shuffle-reduction latency only, not an L2 round trip per step.
constexpr int kQR = 12;

__device__ void apply_q_warp(int n, const double* __restrict__ V, double* x, int forward) {
    const int lane = threadIdx.x & 31;
    const int steps = n - 2;
    if (steps <= 0) return;
    if (n <= 32 * kQR) {
        double xr[kQR], cur[kQR], nxt[kQR];
#pragma unroll
        for (int r = 0; r < kQR; ++r) {
            const int i = lane + 32 * r;
            xr[r] = i < n ? x[i] : 0.0;
        }
        auto load = [&](int k, double (&dst)[kQR]) {
            const double* vk = V + size_t(k) * n;
#pragma unroll
            for (int r = 0; r < kQR; ++r) {
                const int i = lane + 32 * r;
                dst[r] = (i > k && i < n) ? __ldg(vk + i) : 0.0;
            }
        };
        load(forward ? 0 : steps - 1, cur);
        for (int s = 0; s < steps; ++s) {
            if (s + 1 < steps) load(forward ? s + 1 : steps - 2 - s, nxt);
            double t = 0.0;
#pragma unroll
            for (int r = 0; r < kQR; ++r) t = fma(cur[r], xr[r], t);
            t = 2.0 * warp_sum(t);
#pragma unroll
            for (int r = 0; r < kQR; ++r) xr[r] = fma(-t, cur[r], xr[r]);
#pragma unroll
            for (int r = 0; r < kQR; ++r) cur[r] = nxt[r];
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < kQR; ++r) {
            const int i = lane + 32 * r;
            if (i < n) x[i] = xr[r];
        }
        __syncwarp();
        return;
    }
    for (int s = 0; s < steps; ++s) {
        const int k = forward ? s : steps - 1 - s;
        const double* vk = V + size_t(k) * n;
        double t = 0.0;
        for (int i = k + 1 + lane; i < n; i += 32) t += vk[i] * x[i];
        t = 2.0 * warp_sum(t);
        for (int i = k + 1 + lane; i < n; i += 32) x[i] -= t * vk[i];
        __syncwarp();
    }
}

// ------------------------------------------------------------------------------------------
// coarse-mesh element work (3072 coarse tets): A_H2(w_H) and the coarse square load

/// per coarse tet: 16-entry weighted mass (Keast) with nodal weight from interior coarse values wint
__global__ void k_coarse_wmass(int nct, const int32_t* __restrict__ ctets, const double* __restrict__ cxyz,
                               const int32_t* __restrict__ ciidx, const double* __restrict__ wint,
                               double* __restrict__ E) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nct; t += gridDim.x * blockDim.x) {
        const int4 v = reinterpret_cast<const int4*>(ctets)[t];
        TetG G;
        tet_geometry(cxyz, v, G);
        const int vv[4] = {v.x, v.y, v.z, v.w};
        double wn[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) wn[k] = ciidx[vv[k]] >= 0 ? wint[ciidx[vv[k]]] : 0.0;
        double K[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) K[i][j] = 0.0;
        for (int q = 0; q < 11; ++q) {
            const double wq = g_qb[q][0] * wn[0] + g_qb[q][1] * wn[1] + g_qb[q][2] * wn[2] + g_qb[q][3] * wn[3];
            const double s = g_qw[q] * G.vol * wq;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) K[i][j] += s * g_qb[q][i] * g_qb[q][j];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) E[size_t(t) * 16 + 4 * i + j] = K[i][j];
    }
}

/// per (coarse tet, orbital): coarse square load of the coarse function phi_H[i] (4 entries)
__global__ void k_coarse_sq(int nct, int nh, int N, const int32_t* __restrict__ ctets, const double* __restrict__ cxyz,
                            const int32_t* __restrict__ ciidx, const double* __restrict__ phiH, double* __restrict__ E4) {
    const int i = blockIdx.y;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nct; t += gridDim.x * blockDim.x) {
        const int4 v = reinterpret_cast<const int4*>(ctets)[t];
        const int vv[4] = {v.x, v.y, v.z, v.w};
        // |T| from the signed-volume formula, as the reference's coarse_square_load
        TetG G;
        tet_geometry(cxyz, v, G);
        double u4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) u4[k] = ciidx[vv[k]] >= 0 ? phiH[size_t(i) * nh + ciidx[vv[k]]] : 0.0;
        double out[4] = {0, 0, 0, 0};
        for (int q = 0; q < 11; ++q) {
            const double u = g_qb[q][0] * u4[0] + g_qb[q][1] * u4[1] + g_qb[q][2] * u4[2] + g_qb[q][3] * u4[3];
            const double s = g_qw[q] * G.vol * u * u;
#pragma unroll
            for (int k = 0; k < 4; ++k) out[k] += s * g_qb[q][k];
        }
        reinterpret_cast<double4*>(E4)[size_t(i) * nct + t] = make_double4(out[0], out[1], out[2], out[3]);
    }
    (void)N;
}

/// per coarse tet: 16-entry stiffness element |T| grad l_i . grad l_j
__global__ void k_coarse_stiff(int nct, const int32_t* __restrict__ ctets, const double* __restrict__ cxyz,
                               double* __restrict__ E) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nct; t += gridDim.x * blockDim.x) {
        const int4 v = reinterpret_cast<const int4*>(ctets)[t];
        TetG G;
        tet_geometry(cxyz, v, G);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
                E[size_t(t) * 16 + 4 * i + j] =
                    G.vol * (G.g[i][0] * G.g[j][0] + G.g[i][1] * G.g[j][1] + G.g[i][2] * G.g[j][2]);
    }
}

/// A_H = A_H1 + A_H4 [+ A_H2(E16 assembled) + theta1 A_H3], row per thread group (deterministic per row)
__global__ void k_build_AH(int nh, const int32_t* __restrict__ cinc_ptr, const int32_t* __restrict__ cinc,
                           const int32_t* __restrict__ ctets, const int32_t* __restrict__ ciidx,
                           const double* __restrict__ A1, const double* __restrict__ A3, const double* __restrict__ A4,
                           const double* __restrict__ E16, int with_h, const double* __restrict__ theta1,
                           double* __restrict__ AH) {
    const int a = blockIdx.x;
    double* row = AH + size_t(a) * nh;
    for (int b = threadIdx.x; b < nh; b += blockDim.x) row[b] = A1[size_t(a) * nh + b] + A4[size_t(a) * nh + b];
    __syncthreads();
    if (!with_h) return;
    // A_H2 row a: sum over coarse tets of a (ascending), exactly one writer per entry
    if (threadIdx.x == 0) {
        extern __shared__ double acc[];
        for (int b = 0; b < nh; ++b) acc[b] = 0.0;
        for (int k = cinc_ptr[a]; k < cinc_ptr[a + 1]; ++k) {
            const int C = cinc[k] >> 2, la = cinc[k] & 3;
            for (int lb = 0; lb < 4; ++lb) {
                const int b = ciidx[ctets[4 * C + lb]];
                if (b >= 0) acc[b] += E16[size_t(C) * 16 + 4 * la + lb];
            }
        }
    }
    __syncthreads();
    extern __shared__ double acc2[];
    const double th = theta1[0];
    for (int b = threadIdx.x; b < nh; b += blockDim.x) {
        double x = row[b] + acc2[b];
        if (th != 0.0) x += th * A3[size_t(a) * nh + b];
        row[b] = x;
    }
}

/// sum over (C, la) of a of E4[(i*nct + C)*4 + la] -> out[i*nh + a]
__global__ void k_coarse_vec_asm(int nh, int nct, const int32_t* __restrict__ cinc_ptr, const int32_t* __restrict__ cinc,
                                 const double* __restrict__ E4, double* __restrict__ out) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    if (a >= nh) return;
    double s = 0.0;
    for (int k = cinc_ptr[a]; k < cinc_ptr[a + 1]; ++k) s += E4[(size_t(i) * nct + (cinc[k] >> 2)) * 4 + (cinc[k] & 3)];
    out[size_t(i) * nh + a] = s;
}

__global__ void k_symmetrize(int n, double* __restrict__ A) {
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) {
        const int r = idx / n, c = idx % n;
        if (c > r) {
            const double m = 0.5 * (A[size_t(r) * n + c] + A[size_t(c) * n + r]);
            A[size_t(r) * n + c] = m;
            A[size_t(c) * n + r] = m;
        }
    }
}

// ------------------------------------------------------------------------------------------
// per-outer preparation: l_i = L_H^-1 c_i, s_i, u_i = L_H^-T l_i ; Hartree u and Schur scalar

__device__ double block_dot(const double* a, const double* b, int n) {
    __shared__ double red[32];
    __shared__ double out;
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += a[i] * b[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
        out = t;
    }
    __syncthreads();
    const double r = out;
    __syncthreads();
    return r;
}

/// s_i^2 = gamma_i - l_i.l_i ; flag on non-positive
__global__ void k_border_scale(int nh, int N, const double* __restrict__ l, const double* __restrict__ orb_scal,
                               double* __restrict__ s, int* __restrict__ flag) {
    const int i = blockIdx.x;
    const double ll = block_dot(l + size_t(i) * nh, l + size_t(i) * nh, nh);
    if (threadIdx.x == 0) {
        const double g = orb_scal[5 * i + 3];
        const double s2 = g - ll;
        if (!(g > 0.0) || !(s2 > 0.0)) flag[0] = 1;
        s[i] = sqrt(fmax(s2, DBL_MIN));
    }
    (void)N;
}

/// schur = zeta - d_Hh . u
__global__ void k_schur(int nh, const double* __restrict__ dHh, const double* __restrict__ u,
                        const double* __restrict__ shared_scal, double* __restrict__ out, int* __restrict__ flag) {
    const double du = block_dot(dHh, u, nh);
    if (threadIdx.x == 0) {
        out[0] = shared_scal[0] - du;
        if (!(out[0] > 0.0)) flag[0] = 1;
    }
}

// ------------------------------------------------------------------------------------------
// per sweep, per orbital: border, C12, C22, rotated vectors

struct SweepDev {
    const double *AH, *A3, *A_h4, *orb_vecs, *orb_scal, *LHi, *LHiT, *V, *l, *u, *s, *wH, *theta1;
    double *c12, *c22, *lhat, *work;
    int nh, N, hartree;
};

/// block per orbital, independent of the tridiagonalisation (runs on the side stream while it does):
/// b, beta, t = A_H u, c22, and x = L^-1 (b - t) / s into c12 (rotated by k_border_q)
__global__ void k_border_pre(SweepDev S) {
    extern __shared__ double sh[];
    const int i = blockIdx.x, nh = S.nh;
    double* b = sh;            // nh
    double* t = sh + nh;       // nh
    const double* ov = S.orb_vecs + size_t(i) * 6 * nh;  // b_H1, b_H3, b_H4, c_Hh, d_phi, rhs
    const double* sc = S.orb_scal + size_t(i) * 5;       // beta1, beta3, beta4, gamma, zeta_phi
    const double th1 = S.theta1[0];
    const double* Ah4 = S.A_h4 + size_t(i) * nh * nh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    // border b = b_H1 + b_H4 [+ (A_h4 w_H + theta1 b_H3)]
    for (int a = warp; a < nh; a += nw) {
        double x = 0.0;
        if (S.hartree) x = lane_dot(Ah4 + size_t(a) * nh, S.wH, nh, lane);
        x = warp_sum(x);
        if (lane == 0) {
            double bb = ov[a] + ov[2 * nh + a];
            if (S.hartree) bb += x + th1 * ov[nh + a];
            b[a] = bb;
        }
    }
    __syncthreads();
    double beta = sc[0] + sc[2];
    if (S.hartree) beta += block_dot(ov + 5 * nh, S.wH, nh) + th1 * sc[1];
    // t = A_H u
    const double* u = S.u + size_t(i) * nh;
    for (int a = warp; a < nh; a += nw) {
        double x = lane_dot(S.AH + size_t(a) * nh, u, nh, lane);
        x = warp_sum(x);
        if (lane == 0) t[a] = x;
    }
    __syncthreads();
    const double ub = block_dot(u, b, nh);
    const double ut = block_dot(u, t, nh);
    const double si = S.s[i];
    if (threadIdx.x == 0) S.c22[i] = (beta - 2.0 * ub + ut) / (si * si);
    for (int a = threadIdx.x; a < nh; a += blockDim.x) t[a] = (b[a] - t[a]) / si;
    __syncthreads();
    double* x = sh + 2 * nh;
    block_gemv(nh, S.LHi, t, x);
    __syncthreads();
    for (int a = threadIdx.x; a < nh; a += blockDim.x) S.c12[size_t(i) * nh + a] = x[a];
}

/// block per orbital (2 warps): c12 <- Q^T c12 (warp 0), l^ = Q^T l (warp 1)
__global__ void k_border_q(SweepDev S) {
    extern __shared__ double sh[];
    const int i = blockIdx.x, nh = S.nh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* vec = sh + size_t(warp) * nh;
    const double* src = warp == 0 ? S.c12 + size_t(i) * nh : S.l + size_t(i) * nh;
    double* dst = warp == 0 ? S.c12 + size_t(i) * nh : S.lhat + size_t(i) * nh;
    for (int a = lane; a < nh; a += 32) vec[a] = src[a];
    __syncwarp();
    apply_q_warp(nh, S.V, vec, 1);
    for (int a = lane; a < nh; a += 32) dst[a] = vec[a];
}

/// inertia of [T - x, c; c^T, c22 - x]: number of eigenvalues < x (Sylvester), one LDL^T pass with one
/// reciprocal per step on the dependency chain -- evaluated inline, two points per lane, in k_arrow_eig.
/// block per (orbital, k): k-th smallest eigenvalue by 513-way multisection -- 8 warps x 32 lanes x 2 points
/// per lane (two independent Sturm recurrences interleaved per lane), so an iteration gains 9 bits and the
/// eigenvalue needs ~7 iterations of the 343-step dependency chain instead of ~12 with one warp.
/// W warps per item: 8 when few items (latency: fewer multisection rounds), 1 when the items fill the GPU
/// (throughput: less total work per eigenvalue).
template <int W>
__global__ void __launch_bounds__(W * 32) k_arrow_eig(int nh, int N, int nev, const double* __restrict__ dg,
                                                              const double* __restrict__ eg,
                                                              const double* __restrict__ c12,
                                                              const double* __restrict__ c22,
                                                              double* __restrict__ lam) {
    extern __shared__ double she[];
    double* d = she;
    double* e = she + nh;
    double* c = she + 2 * nh;
    __shared__ int first_above[W];
    __shared__ double bounds[2];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int item = blockIdx.x;  // (orbital, k)
    const int i = item / nev, k = item % nev;
    for (int j = threadIdx.x; j < nh; j += blockDim.x) {
        d[j] = dg[j];
        e[j] = eg[j];
        c[j] = c12[size_t(i) * nh + j];
    }
    __syncthreads();
    const double cc = c22[i];
    if (threadIdx.x < 32) {  // Gershgorin bounds
        double lo = DBL_MAX, hi = -DBL_MAX, csum = 0.0;
        for (int j = lane; j < nh; j += 32) {
            const double r = (j > 0 ? fabs(e[j - 1]) : 0.0) + (j + 1 < nh ? fabs(e[j]) : 0.0) + fabs(c[j]);
            lo = fmin(lo, d[j] - r);
            hi = fmax(hi, d[j] + r);
            csum += fabs(c[j]);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        csum = warp_sum(csum);
        lo = fmin(lo, cc - csum);
        hi = fmax(hi, cc + csum);
        const double span = fmax(fabs(lo), fabs(hi));
        if (lane == 0) {
            bounds[0] = lo - (1e-12 * span + DBL_MIN);
            bounds[1] = hi + (1e-12 * span + DBL_MIN);
        }
    }
    __syncthreads();
    double lo = bounds[0], hi = bounds[1];
    const double span = fmax(fabs(lo), fabs(hi));
    const double pivmin = DBL_MIN / DBL_EPSILON * fmax(1.0, span * span);
    constexpr int P = W * 64;  // evaluation points; point index p = 2 * (32 wib + lane) + h
    for (int it = 0; it < 40; ++it) {
        const double w = hi - lo;
        if (w <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + DBL_MIN) break;
        const int p0 = 2 * (32 * wib + lane);
        const double x0 = lo + w * double(p0 + 1) / double(P + 1);
        const double x1 = lo + w * double(p0 + 2) / double(P + 1);
        // two interleaved Sturm recurrences (arrow_count at x0 and x1)
        int cnt0 = 0, cnt1 = 0;
        double rq0 = 0.0, rq1 = 0.0, z0 = 0.0, z1 = 0.0, acc0 = 0.0, acc1 = 0.0;
        for (int j = 0; j < nh; ++j) {
            const double dj = d[j], cj = c[j];
            double a0 = dj - x0, a1 = dj - x1, b0 = cj, b1 = cj;
            if (j > 0) {
                const double ej = e[j - 1];
                const double l0 = ej * rq0, l1 = ej * rq1;
                a0 -= l0 * ej;
                a1 -= l1 * ej;
                b0 -= l0 * z0;
                b1 -= l1 * z1;
            }
            if (fabs(a0) < pivmin) a0 = -pivmin;
            if (fabs(a1) < pivmin) a1 = -pivmin;
            cnt0 += a0 < 0.0;
            cnt1 += a1 < 0.0;
            rq0 = 1.0 / a0;
            rq1 = 1.0 / a1;
            acc0 += b0 * b0 * rq0;
            acc1 += b1 * b1 * rq1;
            z0 = b0;
            z1 = b1;
        }
        cnt0 += ((cc - x0) - acc0) < 0.0 ? 1 : 0;
        cnt1 += ((cc - x1) - acc1) < 0.0 ? 1 : 0;
        // first point whose count exceeds k: counts are monotone in x
        const unsigned a0m = __ballot_sync(0xffffffffu, cnt0 > k), a1m = __ballot_sync(0xffffffffu, cnt1 > k);
        int f = P;  // first point index above, this warp
        if (a0m || a1m) {
            const int l0 = a0m ? __ffs(a0m) - 1 : 32, l1 = a1m ? __ffs(a1m) - 1 : 32;
            f = min(l0 < 32 ? 2 * (32 * wib + l0) : P, l1 < 32 ? 2 * (32 * wib + l1) + 1 : P);
        }
        if (lane == 0) first_above[wib] = f;
        __syncthreads();
        int fa = P;
        for (int q = 0; q < W; ++q) fa = min(fa, first_above[q]);
        __syncthreads();
        const double nlo = fa == 0 ? lo : lo + w * double(fa) / double(P + 1);
        const double nhi = fa == P ? hi : lo + w * double(fa + 1) / double(P + 1);
        lo = nlo;
        hi = nhi;
    }
    if (threadIdx.x == 0) lam[item] = 0.5 * (lo + hi);
}

/// warp per (orbital, k): eigenvector of the arrow-tridiagonal [T c; c^T c22] at the computed eigenvalue by two
/// steps of inverse iteration with block elimination (robust when the eigenvalue is also an eigenvalue of T,
/// e.g. a degenerate coarse pair decoupled from the augmentation direction), and its selection score
/// |(L y)_last| / (|y| sqrt(gamma)), (L y)_last = l^T Q y_h + s y_l (proj/src/eigensolve.cpp:371-396).
__global__ void k_arrow_vec(int nh, int N, int nev, const double* __restrict__ d, const double* __restrict__ e,
                            const double* __restrict__ c12, const double* __restrict__ c22,
                            const double* __restrict__ lhat, const double* __restrict__ s,
                            const double* __restrict__ orb_scal, const double* __restrict__ lam, double* __restrict__ Y,
                            double* __restrict__ Z, double* __restrict__ piv, double* __restrict__ score,
                            double* __restrict__ ylast) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= N * nev) return;
    const int i = warp / nev;
    const double x = lam[warp];
    const double* c = c12 + size_t(i) * nh;
    // per-warp scratch in shared memory: the recurrences below read what they just wrote
    extern __shared__ double shv[];
    double* mul = shv + size_t(threadIdx.x >> 5) * 4 * nh;
    double* y = mul + nh;
    double* z = y + nh;
    double* pv = z + nh;
    (void)Z;
    (void)piv;
    if (lane == 0 && nh > 0) {
        double tn = 0.0;
        for (int j = 0; j < nh; ++j) tn = fmax(tn, fabs(d[j]) + (j > 0 ? fabs(e[j - 1]) : 0.0) + (j + 1 < nh ? fabs(e[j]) : 0.0));
        const double pivmin = DBL_EPSILON * fmax(tn, 1e-300);
        // LDL^T of T - x; pv <- 1 / pivot, z scratch <- multipliers e_j / pivot_j (the solves are then FMA chains)
        double q = 1.0;
        for (int j = 0; j < nh; ++j) {
            double dj = d[j] - x;
            if (j > 0) dj -= (e[j - 1] / q) * e[j - 1];
            if (fabs(dj) < pivmin) dj = dj < 0 ? -pivmin : pivmin;
            pv[j] = dj;
            q = dj;
        }
        double* lm = mul;
        for (int j = 0; j < nh; ++j) {
            const double r = 1.0 / pv[j];
            lm[j] = j + 1 < nh ? e[j] * r : 0.0;
            pv[j] = r;
        }
        auto solve = [&](double* vv, const double* mlt) {  // vv <- (T - x)^-1 vv
            for (int j = 1; j < nh; ++j) vv[j] -= mlt[j - 1] * vv[j - 1];
            vv[nh - 1] *= pv[nh - 1];
            for (int j = nh - 2; j >= 0; --j) vv[j] = vv[j] * pv[j] - mlt[j] * vv[j + 1];
        };
        for (int j = 0; j < nh; ++j) z[j] = c[j];
        solve(z, mul);
        double cz = 0.0;
        for (int j = 0; j < nh; ++j) cz += c[j] * z[j];
        double sch = (c22[i] - x) - cz;
        if (fabs(sch) < pivmin) sch = sch < 0 ? -pivmin : pivmin;
        // deterministic start vector, two inverse-iteration steps
        double yl = 1.0;
        for (int j = 0; j < nh; ++j) y[j] = 1.0 + 0.5 * double((j * 7919) % 97) / 97.0;
        for (int rep = 0; rep < 2; ++rep) {
            const double rl = yl;
            solve(y, mul);
            double cu = 0.0;
            for (int j = 0; j < nh; ++j) cu += c[j] * y[j];
            yl = (rl - cu) / sch;
            double nn = yl * yl;
            for (int j = 0; j < nh; ++j) {
                y[j] -= z[j] * yl;
                nn += y[j] * y[j];
            }
            const double inv = 1.0 / sqrt(nn);
            for (int j = 0; j < nh; ++j) y[j] *= inv;
            yl *= inv;
        }
        ylast[warp] = yl;
    }
    __syncwarp();
    double* yg = Y + size_t(warp) * nh;
    for (int j = lane; j < nh; j += 32) yg[j] = y[j];
    __syncwarp();
    const double* lh = lhat + size_t(i) * nh;
    double ov = 0.0;
    for (int j = lane; j < nh; j += 32) ov += lh[j] * y[j];
    ov = warp_sum(ov);
    if (lane == 0) {
        ov += s[i] * ylast[warp];
        score[warp] = fabs(ov) / sqrt(orb_scal[5 * i + 3]);
    }
}

/// block per orbital: select (strict >, first wins), back-transform, sign-align against the previous state
__global__ void k_select(SweepDev S, int nev, const double* __restrict__ lam, const double* __restrict__ Y,
                         const double* __restrict__ score, const double* __restrict__ ylast, double floor,
                         const double* __restrict__ MH, const double* __restrict__ phi_old,
                         const double* __restrict__ th2_old, double* __restrict__ lam_new, double* __restrict__ phi_new,
                         double* __restrict__ th2_new, int* __restrict__ flag) {
    extern __shared__ double sh[];
    const int i = blockIdx.x, nh = S.nh;
    __shared__ int best;
    __shared__ double th;
    if (threadIdx.x == 0) {
        int b = 0;
        double bs = -1.0;
        for (int k = 0; k < nev; ++k) {
            const double sc = score[i * nev + k];
            if (sc > bs) {
                bs = sc;
                b = k;
            }
        }
        if (bs < floor) flag[0] = 2;
        best = b;
        lam_new[i] = lam[i * nev + b];
    }
    __syncthreads();
    const int w = i * nev + best;
    const double nrm = 1.0;  // inverse iteration returns unit vectors
    double* x = sh;  // nh: Q y_h / nrm, then phi_H
    for (int a = threadIdx.x; a < nh; a += blockDim.x) x[a] = Y[size_t(w) * nh + a];
    __syncthreads();
    if (threadIdx.x < 32) apply_q_warp(nh, S.V, x, 0);
    __syncthreads();
    const double si = S.s[i];
    if (threadIdx.x == 0) th = ylast[w] / si;
    __syncthreads();
    const double theta = th;
    for (int a = threadIdx.x; a < nh; a += blockDim.x) x[a] = x[a] / nrm - S.l[size_t(i) * nh + a] * theta;
    __syncthreads();
    double* y = sh + nh;  // phi_H = L_H^-T x
    block_gemv(nh, S.LHiT, x, y);
    __syncthreads();
    for (int a = threadIdx.x; a < nh; a += blockDim.x) x[a] = y[a];
    __syncthreads();
    // ip = phi_new^T M_H phi_old + th_new c.phi_old + th_old c.phi_new + th_new th_old gamma
    const double* po = phi_old + size_t(i) * nh;
    const double* cH = S.orb_vecs + size_t(i) * 6 * nh + 3 * nh;
    double* tmp = sh + nh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int a = warp; a < nh; a += nw) {
        double t = lane_dot(MH + size_t(a) * nh, po, nh, lane);
        t = warp_sum(t);
        if (lane == 0) tmp[a] = t;
    }
    __syncthreads();
    const double t1 = block_dot(x, tmp, nh);
    const double t2 = block_dot(cH, po, nh);
    const double t3 = block_dot(cH, x, nh);
    const double to = th2_old[i];
    const double ip = t1 + theta * t2 + to * t3 + theta * to * S.orb_scal[5 * i + 3];
    const double sg = ip < 0 ? -1.0 : 1.0;
    for (int a = threadIdx.x; a < nh; a += blockDim.x) phi_new[size_t(i) * nh + a] = sg * x[a];
    if (threadIdx.x == 0) th2_new[i] = sg * theta;
}

/// f_H, g, Hartree bordered solve, theta1, w_H, and the H1 state change delta. Two kernels: one block per orbital
/// forms that orbital's load contribution, energy term and delta term (the nh x nh products dominate, so orbitals
/// run in parallel); one block sums them in orbital order and does the bordered solve.
struct HartreeDev {
    const double *sq, *A_h4, *A3, *orb_vecs, *orb_scal, *shared_vecs, *shared_scal, *CHi, *hu, *schur, *CH, *MH;
    const double *phi_new, *th2_new, *phi_old, *th2_old;
    double *wH_new, *theta1_new, *delta, *part;  // part: N*nh load contributions, then N energy, N delta terms
    int nh, N, hartree;
    double occ;
};

__global__ void __launch_bounds__(512) k_hartree_parts(HartreeDev H) {
    extern __shared__ double sh[];
    const int nh = H.nh, i = blockIdx.x;
    double* tmp = sh;       // nh
    double* dp = sh + nh;   // nh
    double* tmq = sh + 2 * nh;  // nh
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const double* ov = H.orb_vecs + size_t(i) * 6 * nh;
    const double* sc = H.orb_scal + size_t(i) * 5;
    if (H.hartree) {
        const double* ph = H.phi_new + size_t(i) * nh;
        const double t2 = H.th2_new[i];
        const double* Ah4 = H.A_h4 + size_t(i) * nh * nh;
        double* F = H.part + size_t(i) * nh;
        for (int a = warp; a < nh; a += nw) {
            double t = lane_dot(Ah4 + size_t(a) * nh, ph, nh, lane);
            double u = lane_dot(H.A3 + size_t(a) * nh, ph, nh, lane);
            t = warp_sum(t);
            u = warp_sum(u);
            if (lane == 0) {
                F[a] = H.sq[size_t(i) * nh + a] + 2.0 * t2 * t + t2 * t2 * ov[5 * nh + a];
                tmp[a] = u;
            }
        }
        __syncthreads();
        double g = block_dot(ph, tmp, nh);
        g += 2.0 * t2 * block_dot(ov + nh, ph, nh);
        g += t2 * t2 * sc[1];
        if (threadIdx.x == 0) H.part[size_t(H.N) * nh + i] = g;
        __syncthreads();
    }
    // delta_i^2 = dphi^T (C_H + M_H) dphi + 2 dth (d_phi + c_Hh).dphi + dth^2 (zeta_phi + gamma)
    for (int a = threadIdx.x; a < nh; a += blockDim.x)
        dp[a] = H.phi_new[size_t(i) * nh + a] - H.phi_old[size_t(i) * nh + a];
    __syncthreads();
    const double dth = H.th2_new[i] - H.th2_old[i];
    for (int a = warp; a < nh; a += nw) {
        double t = lane_dot(H.CH + size_t(a) * nh, dp, nh, lane);
        double u = lane_dot(H.MH + size_t(a) * nh, dp, nh, lane);
        t = warp_sum(t);
        u = warp_sum(u);
        if (lane == 0) {
            tmp[a] = t;
            tmq[a] = u;
        }
    }
    __syncthreads();
    const double semi = block_dot(dp, tmp, nh) + 2.0 * dth * block_dot(ov + 4 * nh, dp, nh) + dth * dth * sc[4];
    const double l2 = block_dot(dp, tmq, nh) + 2.0 * dth * block_dot(ov + 3 * nh, dp, nh) + dth * dth * sc[3];
    if (threadIdx.x == 0) H.part[size_t(H.N) * nh + H.N + i] = semi + l2;
}

__global__ void __launch_bounds__(512) k_hartree_final(HartreeDev H) {
    extern __shared__ double sh[];
    const int nh = H.nh, N = H.N;
    double* f = sh;           // nh
    double* dp = sh + nh;     // nh
    constexpr double four_pi = 4.0 * 3.14159265358979323846;
    const double* gpart = H.part + size_t(N) * nh;
    if (H.hartree) {
        for (int a = threadIdx.x; a < nh; a += blockDim.x) {
            double s = 0.0;
            for (int i = 0; i < N; ++i) s += H.part[size_t(i) * nh + a];
            f[a] = four_pi * (H.occ * s) - H.shared_vecs[nh + a];
        }
        double g = 0.0;
        for (int i = 0; i < N; ++i) g += gpart[i];
        g = four_pi * (H.occ * g) - H.shared_scal[1];
        __syncthreads();
        // t = C_H^-1 f
        block_gemv(nh, H.CHi, f, dp);
        __syncthreads();
        const double dt = block_dot(H.shared_vecs, dp, nh);
        const double th1 = (g - dt) / H.schur[0];
        for (int a = threadIdx.x; a < nh; a += blockDim.x) H.wH_new[a] = dp[a] - th1 * H.hu[a];
        if (threadIdx.x == 0) H.theta1_new[0] = th1;
    }
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int i = 0; i < N; ++i) tot += gpart[N + i];
        H.delta[0] = tot;
    }
}

// ------------------------------------------------------------------------------------------
// dense generalized eigensolve for the coarse SCF (eig::solve_smallest dense path,
// proj/src/eigensolve.cpp:306-367): C = L^-1 A L^-T, Householder tridiagonalisation, Sturm multisection
// for the lowest nev eigenvalues, inverse iteration + Gram-Schmidt, back-transform, normalize_sign.

__device__ __forceinline__ int tri_count(int n, const double* d, const double* e, double x, double pivmin) {
    int cnt = 0;
    double q = 1.0;
    for (int j = 0; j < n; ++j) {
        double dj = d[j] - x;
        if (j > 0) dj -= e[j - 1] * e[j - 1] / q;
        if (fabs(dj) < pivmin) dj = -pivmin;
        cnt += dj < 0.0;
        q = dj;
    }
    return cnt;
}

/// warp k: k-th smallest eigenvalue of the symmetric tridiagonal (d, e) by 33-way multisection
__global__ void k_tri_eig(int n, int nev, const double* __restrict__ dg, const double* __restrict__ eg,
                          double* __restrict__ lam) {
    extern __shared__ double she2[];
    double* d = she2;
    double* e = she2 + n;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        d[j] = dg[j];
        e[j] = j + 1 < n ? eg[j] : 0.0;
    }
    __syncthreads();
    const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (k >= nev) return;
    double lo = DBL_MAX, hi = -DBL_MAX;
    for (int j = lane; j < n; j += 32) {
        const double r = (j > 0 ? fabs(e[j - 1]) : 0.0) + (j + 1 < n ? fabs(e[j]) : 0.0);
        lo = fmin(lo, d[j] - r);
        hi = fmax(hi, d[j] + r);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const double span = fmax(fabs(lo), fabs(hi));
    lo -= 1e-12 * span + DBL_MIN;
    hi += 1e-12 * span + DBL_MIN;
    const double pivmin = DBL_MIN / DBL_EPSILON * fmax(1.0, span * span);
    for (int it = 0; it < 60; ++it) {
        const double w = hi - lo;
        if (w <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + DBL_MIN) break;
        const double x = lo + w * double(lane + 1) / 33.0;
        const int cnt = tri_count(n, d, e, x, pivmin);
        const unsigned above = __ballot_sync(0xffffffffu, cnt > k);
        const int f = above ? __ffs(above) - 1 : 32;
        const double nlo = f == 0 ? lo : lo + w * double(f) / 33.0;
        const double nhi = f == 32 ? hi : lo + w * double(f + 1) / 33.0;
        lo = nlo;
        hi = nhi;
    }
    if (lane == 0) lam[k] = 0.5 * (lo + hi);
}

/// warp k: eigenvector of T at lam[k] by three inverse-iteration steps (unit norm), into Y[k*n ..]
__global__ void k_tri_vec(int n, int nev, const double* __restrict__ d, const double* __restrict__ e,
                          const double* __restrict__ lam, double* __restrict__ Y) {
    extern __shared__ double shv2[];
    const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (k >= nev) return;
    double* mul = shv2 + size_t(threadIdx.x >> 5) * 3 * n;
    double* rp = mul + n;
    double* y = rp + n;
    if (lane == 0) {
        const double x = lam[k];
        double tn = 0.0;
        for (int j = 0; j < n; ++j) tn = fmax(tn, fabs(d[j]) + (j > 0 ? fabs(e[j - 1]) : 0.0) + (j + 1 < n ? fabs(e[j]) : 0.0));
        const double pivmin = DBL_EPSILON * fmax(tn, 1e-300);
        double q = 1.0;
        for (int j = 0; j < n; ++j) {
            double dj = d[j] - x;
            if (j > 0) dj -= (e[j - 1] / q) * e[j - 1];
            if (fabs(dj) < pivmin) dj = dj < 0 ? -pivmin : pivmin;
            rp[j] = dj;
            q = dj;
        }
        for (int j = 0; j < n; ++j) {
            const double r = 1.0 / rp[j];
            mul[j] = j + 1 < n ? e[j] * r : 0.0;
            rp[j] = r;
        }
        for (int j = 0; j < n; ++j) y[j] = 1.0 + 0.5 * double((j * 7919 + 31 * k) % 97) / 97.0;
        for (int rep = 0; rep < 3; ++rep) {
            for (int j = 1; j < n; ++j) y[j] -= mul[j - 1] * y[j - 1];
            y[n - 1] *= rp[n - 1];
            for (int j = n - 2; j >= 0; --j) y[j] = y[j] * rp[j] - mul[j] * y[j + 1];
            double nn = 0.0;
            for (int j = 0; j < n; ++j) nn += y[j] * y[j];
            const double inv = 1.0 / sqrt(nn);
            for (int j = 0; j < n; ++j) y[j] *= inv;
        }
    }
    __syncwarp();
    for (int j = lane; j < n; j += 32) Y[size_t(k) * n + j] = y[j];
}

/// one block: modified Gram-Schmidt over the nev vectors in ascending eigenvalue order (separates the
/// inverse-iteration vectors of a degenerate cluster; vectors of distinct eigenvalues are already orthogonal)
__global__ void k_mgs(int n, int nev, double* __restrict__ Y) {
    for (int k = 0; k < nev; ++k) {
        double* yk = Y + size_t(k) * n;
        for (int j = 0; j < k; ++j) {
            const double ip = block_dot(Y + size_t(j) * n, yk, n);
            for (int a = threadIdx.x; a < n; a += blockDim.x) yk[a] -= ip * Y[size_t(j) * n + a];
            __syncthreads();
        }
        const double nn = block_dot(yk, yk, n);
        const double inv = 1.0 / sqrt(nn);
        for (int a = threadIdx.x; a < n; a += blockDim.x) yk[a] *= inv;
        __syncthreads();
    }
}

/// block per vector k: x = Q y (Householder back-transform), v = L^-T x, then normalize_sign: the entry of
/// largest magnitude (lowest index on ties) made positive (proj/src/eigensolve.cpp:306-319); v into column k
/// of the interior block Phi (ld)
__global__ void k_back_sign(int n, const double* __restrict__ V, const double* __restrict__ LiT,
                            const double* __restrict__ Y, double* __restrict__ Phi, int ld) {
    extern __shared__ double shb[];
    double* x = shb;
    double* v = shb + n;
    const int k = blockIdx.x;
    for (int a = threadIdx.x; a < n; a += blockDim.x) x[a] = Y[size_t(k) * n + a];
    __syncthreads();
    if (threadIdx.x < 32) apply_q_warp(n, V, x, 0);
    __syncthreads();
    block_gemv(n, LiT, x, v);
    __syncthreads();
    __shared__ double bv[32];
    __shared__ int bi[32];
    double best = -1.0;
    int bidx = 0x7fffffff;
    for (int a = threadIdx.x; a < n; a += blockDim.x) {
        const double m = fabs(v[a]);
        if (m > best || (m == best && a < bidx)) {
            best = m;
            bidx = a;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (ob > best || (ob == best && oi < bidx)) {
            best = ob;
            bidx = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        bv[threadIdx.x >> 5] = best;
        bi[threadIdx.x >> 5] = bidx;
    }
    __syncthreads();
    __shared__ double sg;
    if (threadIdx.x == 0) {
        double b = -1.0;
        int i = 0x7fffffff;
        for (int w = 0; w < int(blockDim.x >> 5); ++w)
            if (bv[w] > b || (bv[w] == b && bi[w] < i)) {
                b = bv[w];
                i = bi[w];
            }
        sg = v[i] < 0.0 ? -1.0 : 1.0;
    }
    __syncthreads();
    for (int a = threadIdx.x; a < n; a += blockDim.x) Phi[size_t(a) * ld + k] = sg * v[a];
}

/// dense row-major copy of an interior CSR block
__global__ void k_csr_dense(int n, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                            const double* __restrict__ val, double* __restrict__ D) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        double* row = D + size_t(r) * n;
        for (int c = 0; c < n; ++c) row[c] = 0.0;
        for (int k = ptr[r]; k < ptr[r + 1]; ++k) row[col[k]] = val[k];
    }
}

}  // namespace

// ==========================================================================================
// host orchestration

void InnerWork::ensure(int nh_, int N_, int nev_, int nct) {
    nh = nh_;
    N = N_;
    nev = nev_;
    const int64_t nh2 = std::max<int64_t>(1, int64_t(nh) * nh);
    const int64_t v = std::max<int64_t>(1, int64_t(N) * nh);
    auto need = [](DevBuf<double>& b, int64_t n) {
        if (b.n < n) b.alloc(n);
    };
    need(AH, nh2);
    need(W, nh2);
    need(C, nh2);
    need(V, nh2);
    need(d, nh + 1);
    need(e, nh + 1);
    need(E16, int64_t(nct) * 16);
    need(E4, int64_t(nct) * 4 * std::max(1, N));
    need(sq, v);
    need(l, v);
    need(u, v);
    need(s, std::max(1, N));
    need(c12, v);
    need(c22, std::max(1, N));
    need(lhat, v);
    need(lam, int64_t(std::max(1, N)) * nev);
    need(Y, int64_t(std::max(1, N)) * nev * std::max(1, nh));
    need(piv, int64_t(std::max(1, N)) * nev * std::max(1, nh));
    need(score, int64_t(std::max(1, N)) * nev);
    need(ynorm, int64_t(std::max(1, N)) * nev);
    need(Z, int64_t(std::max(1, N)) * nev * std::max(1, nh));
    need(hu, std::max(1, nh));
    need(hpart, v + 2 * int64_t(std::max(1, N)));
    need(scal, 16);
    for (int k = 0; k < 2; ++k) {
        need(phi[k], v);
        need(th2[k], std::max(1, N));
        need(lamv[k], std::max(1, N));
        need(wH[k], std::max(1, nh));
        need(th1[k], 1);
    }
    if (flag.n < 4) flag.alloc(4);
}

namespace {

int check_flag(Ctx& c, DevBuf<int>& flag) {
    int h[4];
    KSB_CUDA_CHECK(cudaMemcpyAsync(h, flag.p, sizeof h, cudaMemcpyDeviceToHost, c.stream));
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    KSB_CUDA_CHECK(cudaMemsetAsync(flag.p, 0, sizeof h, c.stream));
    return h[0];
}

}  // namespace

void coarse_level_setup(Level& L, CoarseOps& co) {
    Ctx& c = *L.ctx;
    ensure_rule(c.stream);
    const int nh = L.nH, nct = L.nct;
    const int64_t nh2 = std::max<int64_t>(1, int64_t(nh) * nh);
    co.MH.alloc(nh2);
    co.CH.alloc(nh2);
    co.LH.alloc(nh2);
    co.LC.alloc(nh2);
    DevBuf<double> E;
    E.alloc(int64_t(nct) * 16);
    DevBuf<double> ones;
    ones.alloc(std::max(1, nh));
    std::vector<double> h1(std::max(1, nh), 1.0);
    KSB_CUDA_CHECK(cudaMemcpyAsync(ones.p, h1.data(), sizeof(double) * h1.size(), cudaMemcpyHostToDevice, c.stream));
    // M_H: the coarse unit mass restricted to interior dofs; the interior-only weight equals 1 on every
    // tet vertex that survives the interior restriction, but boundary vertices of the same tets carry
    // weight 1 in the reference's unit mass too -- use a dedicated all-ones weight per coarse vertex.
    DevBuf<double> wall;
    wall.alloc(std::max(1, L.ncv));
    std::vector<double> hw(std::max(1, L.ncv), 1.0);
    KSB_CUDA_CHECK(cudaMemcpyAsync(wall.p, hw.data(), sizeof(double) * hw.size(), cudaMemcpyHostToDevice, c.stream));
    DevBuf<int32_t> ident;
    ident.alloc(std::max(1, L.ncv));
    std::vector<int32_t> hid(std::max(1, L.ncv));
    for (int k = 0; k < L.ncv; ++k) hid[k] = k;
    KSB_CUDA_CHECK(cudaMemcpyAsync(ident.p, hid.data(), sizeof(int32_t) * hid.size(), cudaMemcpyHostToDevice, c.stream));
    launch(c, "coarse", k_coarse_wmass, ceil_div(nct, 128), 128, 0, nct, (const int32_t*)L.ctets.p,
           (const double*)L.cxyz.p, (const int32_t*)ident.p, (const double*)wall.p, E.p);
    DevBuf<double> zero, th0;
    zero.alloc(nh2);
    KSB_CUDA_CHECK(cudaMemsetAsync(zero.p, 0, sizeof(double) * nh2, c.stream));
    th0.alloc(1);
    KSB_CUDA_CHECK(cudaMemsetAsync(th0.p, 0, sizeof(double), c.stream));
    // M_H = 0 + 0 + assembled(E)
    if (nh > 0)
        launch(c, "coarse", k_build_AH, nh, 128, sizeof(double) * nh, nh, (const int32_t*)L.cinc_ptr.p,
               (const int32_t*)L.cinc.p, (const int32_t*)L.ctets.p, (const int32_t*)L.ciidx.p, (const double*)zero.p,
               (const double*)zero.p, (const double*)zero.p, (const double*)E.p, 1, (const double*)th0.p, co.MH.p);
    launch(c, "coarse", k_coarse_stiff, ceil_div(nct, 128), 128, 0, nct, (const int32_t*)L.ctets.p,
           (const double*)L.cxyz.p, E.p);
    if (nh > 0)
        launch(c, "coarse", k_build_AH, nh, 128, sizeof(double) * nh, nh, (const int32_t*)L.cinc_ptr.p,
               (const int32_t*)L.cinc.p, (const int32_t*)L.ctets.p, (const int32_t*)L.ciidx.p, (const double*)zero.p,
               (const double*)zero.p, (const double*)zero.p, (const double*)E.p, 1, (const double*)th0.p, co.CH.p);
    KSB_CUDA_CHECK(cudaMemcpyAsync(co.LH.p, co.MH.p, sizeof(double) * nh2, cudaMemcpyDeviceToDevice, c.stream));
    KSB_CUDA_CHECK(cudaMemcpyAsync(co.LC.p, co.CH.p, sizeof(double) * nh2, cudaMemcpyDeviceToDevice, c.stream));
    DevBuf<int> flag;
    flag.alloc(4);
    KSB_CUDA_CHECK(cudaMemsetAsync(flag.p, 0, sizeof(int) * 4, c.stream));
    if (nh > 0) {
        launch(c, "coarse", k_potrf, 1, 1024, 0, nh, co.LH.p, flag.p);
        launch(c, "coarse", k_potrf, 1, 1024, 0, nh, co.LC.p, flag.p);
    }
    if (check_flag(c, flag)) raise(KSB_INTERNAL, "coarse mass or stiffness factorization failed");
    // explicit inverse factors, once per level: columns of L^-1 e_j by triangular solves
    co.LHi.alloc(nh2);
    co.LHiT.alloc(nh2);
    co.CHi.alloc(nh2);
    if (nh > 0) {
        DevBuf<double> I, Y;
        I.alloc(nh2);
        Y.alloc(nh2);
        launch(c, "coarse", k_identity, ceil_div(int64_t(nh) * nh, 256), 256, 0, nh, I.p);
        const size_t sm = sizeof(double) * nh * 4;
        // L_H^-1 (row-major: x_j = L^-1 e_j is column j) and L_H^-T (row-major: x_j is row j)
        launch(c, "coarse", k_trsv_many, ceil_div(nh, 4), 128, sm, nh, nh, (const double*)co.LH.p, 0,
               (const double*)I.p, int64_t(nh), int64_t(1), co.LHi.p, int64_t(1), int64_t(nh), 1.0);
        launch(c, "coarse", k_trsv_many, ceil_div(nh, 4), 128, sm, nh, nh, (const double*)co.LH.p, 0,
               (const double*)I.p, int64_t(nh), int64_t(1), co.LHiT.p, int64_t(nh), int64_t(1), 1.0);
        // C_H^-1 = L_C^-T L_C^-1 (symmetric; column j = row j)
        launch(c, "coarse", k_trsv_many, ceil_div(nh, 4), 128, sm, nh, nh, (const double*)co.LC.p, 0,
               (const double*)I.p, int64_t(nh), int64_t(1), Y.p, int64_t(nh), int64_t(1), 1.0);
        launch(c, "coarse", k_trsv_many, ceil_div(nh, 4), 128, sm, nh, nh, (const double*)co.LC.p, 1,
               (const double*)Y.p, int64_t(nh), int64_t(1), co.CHi.p, int64_t(nh), int64_t(1), 1.0);
        launch(c, "coarse", k_symmetrize, ceil_div(int64_t(nh) * nh, 256), 256, 0, nh, co.CHi.p);
        KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    }
    co.ready = true;
}

void dense_lowest_eigs(Level& L, const CoarseOps& co, InnerWork& w, int mat, int nev, double* h_lambda, double* d_Phi,
                       int ld) {
    Ctx& c = *L.ctx;
    const int n = L.ni;
    if (n != L.nH) raise(KSB_INVALID_ARGUMENT, "the dense coarse eigensolve runs on level 0");
    if (nev < 1 || nev > n) raise(KSB_INVALID_ARGUMENT, "nev out of range");
    const int64_t n2 = std::max<int64_t>(1, int64_t(n) * n);
    auto need = [](DevBuf<double>& b, int64_t m) {
        if (b.n < m) b.alloc(m);
    };
    need(w.AH, n2);
    need(w.W, n2);
    need(w.C, n2);
    need(w.V, n2);
    need(w.d, n + 1);
    need(w.e, n + 1);
    need(w.lam, nev);
    need(w.Y, int64_t(nev) * n);
    launch(c, "scf:dense", k_csr_dense, ceil_div(n, 128), 128, 0, n, (const int32_t*)L.ii_ptr.p,
           (const int32_t*)L.ii_col.p, (const double*)L.mats[mat].ii.p, w.AH.p);
    const dim3 gt(ceil_div(n, 32), ceil_div(n, 32));
    launch(c, "scf:gemm", k_gemm_nt, gt, 256, 0, n, (const double*)co.LHi.p, (const double*)w.AH.p, w.W.p);
    launch(c, "scf:gemm", k_gemm_nt, gt, 256, 0, n, (const double*)w.W.p, (const double*)co.LHi.p, w.C.p);
    launch(c, "scf:symmetrize", k_symmetrize, ceil_div(int64_t(n) * n, 256), 256, 0, n, w.C.p);
    const int cl_R = (n + kTriCluster - 1) / kTriCluster;
    const size_t cl_smem = sizeof(double) * (size_t(cl_R) * n + (3 + 2 * kTriRep) * size_t(n));
    if (cl_smem <= size_t(kMaxDynSmem) && n <= 32 * kTriS) {
        KSB_CUDA_CHECK(cudaFuncSetAttribute(k_tridiag_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            int(kMaxDynSmem)));
        launch(c, "scf:tridiag", k_tridiag_cluster, kTriCluster, kTriThreads, cl_smem, n, cl_R, (const double*)w.C.p,
               w.d.p, w.e.p, w.V.p);
    } else {
        launch(c, "scf:tridiag", k_tridiag, 1, 1024, sizeof(double) * 2 * n, n, w.C.p, w.d.p, w.e.p, w.V.p);
    }
    launch(c, "scf:eig", k_tri_eig, ceil_div(nev, 4), 128, sizeof(double) * 2 * n, n, nev, (const double*)w.d.p,
           (const double*)w.e.p, w.lam.p);
    const size_t vsm = sizeof(double) * 4 * 3 * size_t(n);
    if (vsm > 48 * 1024)
        KSB_CUDA_CHECK(cudaFuncSetAttribute(k_tri_vec, cudaFuncAttributeMaxDynamicSharedMemorySize, int(vsm)));
    launch(c, "scf:vec", k_tri_vec, ceil_div(nev, 4), 128, vsm, n, nev, (const double*)w.d.p, (const double*)w.e.p,
           (const double*)w.lam.p, w.Y.p);
    launch(c, "scf:mgs", k_mgs, 1, 256, 0, n, nev, w.Y.p);
    launch(c, "scf:back", k_back_sign, nev, 256, sizeof(double) * 2 * n, n, (const double*)w.V.p,
           (const double*)co.LHiT.p, (const double*)w.Y.p, d_Phi, ld);
    KSB_CUDA_CHECK(cudaMemcpyAsync(h_lambda, w.lam.p, sizeof(double) * nev, cudaMemcpyDeviceToHost, c.stream));
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

InnerStats inner_scf(Level& L, const CoarseOps& co, const ProjOut& P, const InnerParams& prm, const double* h_lambda,
                     InnerWork& w, bool start_pure) {
    Ctx& c = *L.ctx;
    ensure_rule(c.stream);
    const int nh = L.nH, N = P.N, nct = L.nct;
    const int nev = std::min(nh + 1, N + prm.nev_pad);
    w.ensure(nh, N, nev, nct);
    KSB_CUDA_CHECK(cudaMemsetAsync(w.flag.p, 0, sizeof(int) * 4, c.stream));
    InnerStats st;
    if (nh == 0) raise(KSB_INVALID_ARGUMENT, "degenerate coarse space: use the host path");

    const double* A1 = P.shared_mats.p;
    const double* A3 = P.shared_mats.p + int64_t(nh) * nh;
    const double* A4 = P.shared_mats.p + 2 * int64_t(nh) * nh;
    // per outer: l_i = L_H^-1 c_i, s_i, u_i = L_H^-T l_i
    const size_t smem_trsv = sizeof(double) * nh * 4;
    (void)smem_trsv;
    auto gemv = [&](const double* A, const double* X, int64_t ldx, double* Y, int64_t ldy, int nv) {
        launch(c, "inner:gemv", k_gemv_many, ceil_div(nh * nv, 8), 256, 0, nh, nh, nv, A, nh, X, ldx, Y, ldy, 1.0);
    };
    gemv(co.LHi.p, P.orb_vecs.p + 3 * nh, int64_t(6) * nh, w.l.p, int64_t(nh), N);
    launch(c, "inner:border_scale", k_border_scale, N, 128, 0, nh, N, (const double*)w.l.p, (const double*)P.orb_scal.p, w.s.p,
           w.flag.p);
    gemv(co.LHiT.p, w.l.p, int64_t(nh), w.u.p, int64_t(nh), N);
    if (check_flag(c, w.flag)) raise(KSB_AMBIGUOUS_SELECTION, "bordered mass matrix is not positive definite");
    if (prm.hartree) {
        gemv(co.CHi.p, P.shared_vecs.p, int64_t(nh), w.hu.p, int64_t(nh), 1);
        launch(c, "inner:schur", k_schur, 1, 128, 0, nh, (const double*)P.shared_vecs.p, (const double*)w.hu.p,
               (const double*)P.shared_scal.p, w.scal.p, w.flag.p);
        if (check_flag(c, w.flag))
            raise(KSB_AMBIGUOUS_SELECTION, "electrostatic augmentation vector lies in the coarse space");
    }
    // initial state: pure augmentation (phi_H = 0, theta2 = 1, w_H = 0, theta1 = hartree ? 1 : 0)
    int cur = 0;
    if (start_pure) {
        KSB_CUDA_CHECK(cudaMemsetAsync(w.phi[0].p, 0, sizeof(double) * N * nh, c.stream));
        KSB_CUDA_CHECK(cudaMemsetAsync(w.wH[0].p, 0, sizeof(double) * nh, c.stream));
        std::vector<double> ones(N, 1.0);
        KSB_CUDA_CHECK(cudaMemcpyAsync(w.th2[0].p, ones.data(), sizeof(double) * N, cudaMemcpyHostToDevice, c.stream));
        const double t1 = prm.hartree ? 1.0 : 0.0;
        KSB_CUDA_CHECK(cudaMemcpyAsync(w.th1[0].p, &t1, sizeof(double), cudaMemcpyHostToDevice, c.stream));
        KSB_CUDA_CHECK(cudaMemcpyAsync(w.lamv[0].p, h_lambda, sizeof(double) * N, cudaMemcpyHostToDevice, c.stream));
    }
    const size_t tri_smem = sizeof(double) * 2 * nh;
    const int cl_R = (nh + kTriCluster - 1) / kTriCluster;
    const size_t cl_smem = sizeof(double) * (size_t(cl_R) * nh + (3 + 2 * kTriRep) * size_t(nh));
    const bool use_cluster = cl_smem <= size_t(kMaxDynSmem) && nh <= 32 * kTriS;

    if (use_cluster) {
        static bool attr = false;
        if (!attr) {
            KSB_CUDA_CHECK(cudaFuncSetAttribute(k_tridiag_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                int(kMaxDynSmem)));
            KSB_CUDA_CHECK(cudaFuncSetAttribute(k_arrow_vec, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                int(kMaxDynSmem)));
            attr = true;
        }
    }
    const int cap = prm.fixed_sweeps > 0 ? prm.fixed_sweeps : prm.max_iterations;
    for (int sweep = 1; sweep <= cap; ++sweep) {
        const int nx = cur ^ 1;
        // A_H
        if (prm.hartree)
            launch(c, "inner:coarse_wmass", k_coarse_wmass, ceil_div(nct, 128), 128, 0, nct, (const int32_t*)L.ctets.p,
                   (const double*)L.cxyz.p, (const int32_t*)L.ciidx.p, (const double*)w.wH[cur].p, w.E16.p);
        launch(c, "inner:build_", k_build_AH, nh, 128, sizeof(double) * nh, nh, (const int32_t*)L.cinc_ptr.p,
               (const int32_t*)L.cinc.p, (const int32_t*)L.ctets.p, (const int32_t*)L.ciidx.p, A1, A3, A4,
               (const double*)w.E16.p, prm.hartree ? 1 : 0, (const double*)w.th1[cur].p, w.AH.p);
        // the orbital borders depend on A_H but not on the tridiagonalisation: side stream, joined below
        SweepDev S{w.AH.p, A3, P.A_h4.p, P.orb_vecs.p, P.orb_scal.p, co.LHi.p, co.LHiT.p, w.V.p, w.l.p, w.u.p, w.s.p,
                   w.wH[cur].p, w.th1[cur].p, w.c12.p, w.c22.p, w.lhat.p, nullptr, nh, N, prm.hartree ? 1 : 0};
        stream_wait(c, c.stream, c.aux, c.fork);
        launch_on(c, c.aux, "inner:border_pre", k_border_pre, N, 256, sizeof(double) * 3 * nh, S);
        // C11 = L^-1 A_H L^-T as two products (A_H symmetric: L^-1 A_H = L^-1 A_H^T)
        const dim3 gt(ceil_div(nh, 32), ceil_div(nh, 32));
        launch(c, "inner:gemm", k_gemm_nt, gt, 256, 0, nh, (const double*)co.LHi.p, (const double*)w.AH.p, w.W.p);
        launch(c, "inner:gemm", k_gemm_nt, gt, 256, 0, nh, (const double*)w.W.p, (const double*)co.LHi.p, w.C.p);
        launch(c, "inner:symmetrize", k_symmetrize, ceil_div(int64_t(nh) * nh, 256), 256, 0, nh, w.C.p);
        if (use_cluster)
            launch(c, "inner_tridiag", k_tridiag_cluster, kTriCluster, kTriThreads, cl_smem, nh, cl_R, (const double*)w.C.p,
                   w.d.p, w.e.p, w.V.p);
        else
            launch(c, "inner_tridiag", k_tridiag, 1, 1024, tri_smem, nh, w.C.p, w.d.p, w.e.p, w.V.p);
        stream_wait(c, c.aux, c.stream, c.join);
        launch(c, "inner:border_q", k_border_q, N, 64, sizeof(double) * 2 * nh, S);
        const int warps = N * nev;
        if (warps >= 4 * c.sm_count)
            launch(c, "inner:arrow_eig", k_arrow_eig<1>, warps, 32, sizeof(double) * 3 * nh, nh, N, nev,
                   (const double*)w.d.p, (const double*)w.e.p, (const double*)w.c12.p, (const double*)w.c22.p,
                   w.lam.p);
        else
            launch(c, "inner:arrow_eig", k_arrow_eig<8>, warps, 8 * 32, sizeof(double) * 3 * nh, nh, N, nev,
               (const double*)w.d.p,
               (const double*)w.e.p, (const double*)w.c12.p, (const double*)w.c22.p, w.lam.p);
        launch(c, "inner:arrow_vec", k_arrow_vec, ceil_div(warps, 4), 128, sizeof(double) * 4 * 4 * nh, nh, N, nev,
               (const double*)w.d.p,
               (const double*)w.e.p, (const double*)w.c12.p, (const double*)w.c22.p, (const double*)w.lhat.p,
               (const double*)w.s.p, (const double*)P.orb_scal.p, (const double*)w.lam.p, w.Y.p, w.Z.p, w.piv.p,
               w.score.p, w.ynorm.p);
        launch(c, "inner:select", k_select, N, 256, sizeof(double) * 2 * nh, S, nev, (const double*)w.lam.p,
               (const double*)w.Y.p, (const double*)w.score.p, (const double*)w.ynorm.p, prm.score_floor,
               (const double*)co.MH.p, (const double*)w.phi[cur].p, (const double*)w.th2[cur].p, w.lamv[nx].p,
               w.phi[nx].p, w.th2[nx].p, w.flag.p);
        if (prm.hartree)
            launch(c, "inner:coarse_sq", k_coarse_sq, dim3(ceil_div(nct, 128), N), 128, 0, nct, nh, N, (const int32_t*)L.ctets.p,
                   (const double*)L.cxyz.p, (const int32_t*)L.ciidx.p, (const double*)w.phi[nx].p, w.E4.p);
        if (prm.hartree)
            launch(c, "inner:coarse_vec_asm", k_coarse_vec_asm, dim3(ceil_div(nh, 128), N), 128, 0, nh, nct,
                   (const int32_t*)L.cinc_ptr.p, (const int32_t*)L.cinc.p, (const double*)w.E4.p, w.sq.p);
        HartreeDev H{w.sq.p, P.A_h4.p, A3, P.orb_vecs.p, P.orb_scal.p, P.shared_vecs.p, P.shared_scal.p, co.CHi.p,
                     w.hu.p, w.scal.p, co.CH.p, co.MH.p, w.phi[nx].p, w.th2[nx].p, w.phi[cur].p, w.th2[cur].p,
                     w.wH[nx].p, w.th1[nx].p, w.scal.p + 1, w.hpart.p, nh, N, prm.hartree ? 1 : 0, prm.occ};
        if (!prm.hartree) {
            KSB_CUDA_CHECK(cudaMemcpyAsync(w.wH[nx].p, w.wH[cur].p, sizeof(double) * nh, cudaMemcpyDeviceToDevice, c.stream));
            KSB_CUDA_CHECK(cudaMemcpyAsync(w.th1[nx].p, w.th1[cur].p, sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
        }
        launch(c, "inner:hartree_delta", k_hartree_parts, N, 512, sizeof(double) * 3 * nh, H);
        launch(c, "inner:hartree_delta", k_hartree_final, 1, 512, sizeof(double) * 2 * nh, H);
        double dsq = 0.0;
        int fl[4];
        KSB_CUDA_CHECK(cudaMemcpyAsync(&dsq, w.scal.p + 1, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        KSB_CUDA_CHECK(cudaMemcpyAsync(fl, w.flag.p, sizeof fl, cudaMemcpyDeviceToHost, c.stream));
        KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
        if (fl[0] == 2) raise(KSB_AMBIGUOUS_SELECTION, "all scanned pairs have negligible augmentation component");
        const double delta = std::sqrt(dsq);
        st.history.push_back(delta);
        st.iterations = sweep;
        cur = nx;
        w.cur = cur;
        if (prm.fixed_sweeps <= 0 && (delta < prm.tol || !prm.hartree)) return st;
    }
    if (prm.fixed_sweeps > 0) return st;
    std::string msg = "inner iteration exceeded " + std::to_string(prm.max_iterations) + " sweeps; recent changes:";
    for (size_t k = st.history.size() > 6 ? st.history.size() - 6 : 0; k < st.history.size(); ++k)
        msg += " " + std::to_string(st.history[k]);
    raise(KSB_NONCONVERGENCE, msg);
}

}  // namespace ksb
