// Density / xc, Hartree pieces, norms and energy on the fine level.
//
//   K-RHOXC  model::density + xc_potential_field     reference proj/src/ks_model.cpp:43-52,89-105
//   K-MOM    hartree::compute_moments (two passes)   reference proj/src/hartree.cpp:15-63
//   K-BC     hartree::boundary_values                reference proj/src/hartree.cpp:65-82
//   K-SQLOAD hartree::squared_density_load           reference proj/src/hartree.cpp:108-129
//   K-NORM   fem::l2_norm / h1_seminorm               reference proj/src/assembly.cpp:251-287
//   K-ENERGY model::total_energy                      reference proj/src/ks_model.cpp:107-143
// Orbital blocks live in interior layout (ni x ld): orbitals have zero trace throughout the
// correction algorithm, so boundary values are structurally zero.
#include <algorithm>

#include "geom.cuh"
#include "physics.cuh"

namespace ksb {

namespace {

constexpr int kT = 256;

int grid_of(const Ctx& c, int64_t work, int per_block = kT) {
    const int64_t want = (work + per_block - 1) / per_block;
    return int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(c.sm_count) * 8)));
}

__device__ __forceinline__ double phi_at(const double* __restrict__ Phi, const int32_t* __restrict__ iidx, int v,
                                         int ld, int i) {
    const int r = iidx[v];
    return r >= 0 ? Phi[size_t(r) * ld + i] : 0.0;
}

__global__ void k_rho_vxc(int ni, int N, int ld, const double* __restrict__ Phi, double occ, XcParams xc, int want_vxc,
                          const int32_t* __restrict__ interior, double* __restrict__ rho, double* __restrict__ vxc) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ni; r += gridDim.x * blockDim.x) {
        const double* p = Phi + size_t(r) * ld;
        double s = 0.0;
        for (int i = 0; i < N; ++i) s += p[i] * p[i];
        s *= occ;
        const int v = interior[r];
        rho[v] = s;
        if (want_vxc) vxc[v] = xc_potential(xc, s);
    }
}

__global__ void k_moments1(int nt, const int32_t* __restrict__ tets, const double* __restrict__ xyz,
                           const double* __restrict__ rho, double* __restrict__ part) {
    double acc[4] = {0, 0, 0, 0};
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        const int4 v = reinterpret_cast<const int4*>(tets)[t];
        TetG G;
        tet_geometry(xyz, v, G);
        const double rv4[4] = {rho[v.x], rho[v.y], rho[v.z], rho[v.w]};
        for (int q = 0; q < 11; ++q) {
            double rv = 0, x[3] = {0, 0, 0};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                rv += g_qb[q][i] * rv4[i];
#pragma unroll
                for (int d = 0; d < 3; ++d) x[d] += g_qb[q][i] * G.x[i][d];
            }
            const double s = g_qw[q] * G.vol * rv;
            acc[0] += s;
#pragma unroll
            for (int d = 0; d < 3; ++d) acc[1 + d] += s * x[d];
        }
    }
    block_sum_to<4>(acc, part);
}

__global__ void k_moments2(int nt, const int32_t* __restrict__ tets, const double* __restrict__ xyz,
                           const double* __restrict__ rho, double cx, double cy, double cz, double* __restrict__ part) {
    double acc[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) acc[k] = 0.0;
    const double c[3] = {cx, cy, cz};
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        const int4 v = reinterpret_cast<const int4*>(tets)[t];
        TetG G;
        tet_geometry(xyz, v, G);
        const double rv4[4] = {rho[v.x], rho[v.y], rho[v.z], rho[v.w]};
        for (int q = 0; q < 11; ++q) {
            double rv = 0, d[3] = {0, 0, 0};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                rv += g_qb[q][i] * rv4[i];
#pragma unroll
                for (int e = 0; e < 3; ++e) d[e] += g_qb[q][i] * G.x[i][e];
            }
#pragma unroll
            for (int e = 0; e < 3; ++e) d[e] -= c[e];
            const double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
            const double s = g_qw[q] * G.vol * rv;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                acc[a] += s * d[a];
#pragma unroll
                for (int b = 0; b < 3; ++b) acc[3 + 3 * a + b] += s * (3.0 * d[a] * d[b] - (a == b ? r2 : 0.0));
            }
        }
    }
    block_sum_to<12>(acc, part);
}

__global__ void k_bc(int nb, const int32_t* __restrict__ boundary, const double* __restrict__ xyz, Moments m,
                     double* __restrict__ bcb) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nb; k += gridDim.x * blockDim.x) {
        const int v = boundary[k];
        const double d[3] = {xyz[3 * v] - m.c[0], xyz[3 * v + 1] - m.c[1], xyz[3 * v + 2] - m.c[2]};
        const double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        const double u[3] = {d[0] / r, d[1] / r, d[2] / r};
        double qu = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) qu += u[a] * m.Q[a][b] * u[b];
        bcb[k] = m.q / r + (m.dip[0] * u[0] + m.dip[1] * u[1] + m.dip[2] * u[2]) / (r * r) + 0.5 * qu / (r * r * r);
    }
}

/// per-tet contributions of occ * sum_i phi_i^2 tested against the four hat functions (Keast rule).
/// The density at a quadrature point is the quadratic form b_q^T Gm b_q of the vertex Gram matrix
/// Gm_kl = sum_i phi_i(v_k) phi_i(v_l) (10 unique entries), so the orbitals are read once per tet, not per point.
__device__ __forceinline__ int gram_idx(int k, int l) { return k <= l ? k * 4 - k * (k - 1) / 2 + (l - k) : l * 4 - l * (l - 1) / 2 + (k - l); }

__device__ __forceinline__ double4 sq_quad(double vol, double occ, const double (&gm)[10]) {
    double out[4] = {0, 0, 0, 0};
    for (int q = 0; q < 11; ++q) {
        double dens = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int l = 0; l < 4; ++l) dens += g_qb[q][k] * g_qb[q][l] * gm[gram_idx(k, l)];
        const double s = g_qw[q] * vol * occ * dens;
#pragma unroll
        for (int k = 0; k < 4; ++k) out[k] += s * g_qb[q][k];
    }
    return make_double4(out[0], out[1], out[2], out[3]);
}

__global__ void k_sqload_elem(int nt, const int32_t* __restrict__ tets, const double* __restrict__ xyz,
                              const int32_t* __restrict__ iidx, const double* __restrict__ Phi, int N, int ld,
                              double occ, double* __restrict__ E4) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        const int4 v = reinterpret_cast<const int4*>(tets)[t];
        TetG G;
        tet_geometry(xyz, v, G);
        const int rr[4] = {iidx[v.x], iidx[v.y], iidx[v.z], iidx[v.w]};
        double gm[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) gm[k] = 0.0;
        for (int i = 0; i < N; ++i) {
            double f[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) f[k] = rr[k] >= 0 ? Phi[size_t(rr[k]) * ld + i] : 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int l = k; l < 4; ++l) gm[gram_idx(k, l)] += f[k] * f[l];
        }
        reinterpret_cast<double4*>(E4)[t] = sq_quad(G.vol, occ, gm);
    }
}

/// many orbitals: one warp per tet, lanes stride the orbitals of the four vertex rows (coalesced row reads)
__global__ void k_sqload_elem_warp(int nt, const int32_t* __restrict__ tets, const double* __restrict__ xyz,
                                   const int32_t* __restrict__ iidx, const double* __restrict__ Phi, int N, int ld,
                                   double occ, double* __restrict__ E4) {
    const int lane = threadIdx.x & 31;
    const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int t = w0; t < nt; t += nw) {
        const int4 v = reinterpret_cast<const int4*>(tets)[t];
        const int rr[4] = {iidx[v.x], iidx[v.y], iidx[v.z], iidx[v.w]};
        double gm[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) gm[k] = 0.0;
        for (int i = lane; i < N; i += 32) {
            double f[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) f[k] = rr[k] >= 0 ? Phi[size_t(rr[k]) * ld + i] : 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int l = k; l < 4; ++l) gm[gram_idx(k, l)] += f[k] * f[l];
        }
#pragma unroll
        for (int k = 0; k < 10; ++k) gm[k] = warp_sum(gm[k]);
        if (lane == 0) {
            TetG G;
            tet_geometry(xyz, v, G);
            reinterpret_cast<double4*>(E4)[t] = sq_quad(G.vol, occ, gm);
        }
    }
}

/// many orbitals, even leading dimension: eight lanes per tet (four tets per warp), the lanes stride the orbital
/// pairs of the four vertex rows with 16-byte loads, the Gram entries are folded over 8 lanes (3 shuffle stages
/// instead of 5 over a whole warp), and the Keast quadrature of the quadratic form is a constant 4 x 10 matrix
/// built once per block: out_k = vol occ sum_m C[k][m] gm[m], C[k][(a,b)] = (2 - [a == b]) sum_q w_q b_qk b_qa b_qb
/// (k_sqload_elem_warp spent ~550 of its ~900 warp instructions per tet on that quadrature in one lane).
/// N = 120 at 12.6 M tets: 9.7 -> see profiles/README.md.
__global__ void __launch_bounds__(256) k_sqload_elem_g8(int nt, const int32_t* __restrict__ tets,
                                                        const double* __restrict__ xyz,
                                                        const int32_t* __restrict__ iidx,
                                                        const double* __restrict__ Phi, int N, int ld, double occ,
                                                        double* __restrict__ E4) {
    __shared__ double C[4][10];
    if (threadIdx.x < 40) {
        const int k = threadIdx.x / 10, m = threadIdx.x % 10;
        int a = 0, b = 0;
        for (int i = 0; i < 4; ++i)
            for (int j = i; j < 4; ++j)
                if (gram_idx(i, j) == m) {
                    a = i;
                    b = j;
                }
        double sum = 0.0;
        for (int q = 0; q < 11; ++q) sum += g_qw[q] * g_qb[q][k] * g_qb[q][a] * g_qb[q][b];
        C[k][m] = (a == b ? 1.0 : 2.0) * sum;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 3, l = lane & 7;
    const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const int nsteps = (nt + 3) / 4;
    for (int ws = w0; ws < nsteps; ws += nw) {
        const int t = ws * 4 + g;
        const bool valid = t < nt;
        const int4 v = valid ? reinterpret_cast<const int4*>(tets)[t] : make_int4(0, 0, 0, 0);
        int rr[4] = {-1, -1, -1, -1};
        if (valid) {
            rr[0] = iidx[v.x];
            rr[1] = iidx[v.y];
            rr[2] = iidx[v.z];
            rr[3] = iidx[v.w];
        }
        double gm[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) gm[k] = 0.0;
        for (int c = 2 * l; c < N; c += 16) {
            double2 f[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                f[k] = make_double2(0.0, 0.0);
                if (rr[k] >= 0) f[k] = __ldg(reinterpret_cast<const double2*>(Phi + size_t(rr[k]) * ld + c));
                if (c + 1 >= N) f[k].y = 0.0;  // odd N: the pad column is not an orbital
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int j = k; j < 4; ++j)
                    gm[gram_idx(k, j)] = fma(f[k].y, f[j].y, fma(f[k].x, f[j].x, gm[gram_idx(k, j)]));
        }
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            gm[k] += __shfl_xor_sync(0xffffffffu, gm[k], 4);
            gm[k] += __shfl_xor_sync(0xffffffffu, gm[k], 2);
            gm[k] += __shfl_xor_sync(0xffffffffu, gm[k], 1);
        }
        if (l == 0 && valid) {
            TetG G;
            tet_geometry(xyz, v, G);
            double out[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                double sum = 0.0;
#pragma unroll
                for (int m = 0; m < 10; ++m) sum = fma(C[k][m], gm[m], sum);
                out[k] = G.vol * occ * sum;
            }
            reinterpret_cast<double4*>(E4)[t] = make_double4(out[0], out[1], out[2], out[3]);
        }
    }
}

void launch_sqload_elem(Ctx& c, Level& L, const double* Phi, int N, int ld, double occ, double* e4) {
    if (N >= 32 && ld % 2 == 0 && (reinterpret_cast<uintptr_t>(Phi) & 15) == 0)
        launch(c, "sqload", k_sqload_elem_g8, grid_of(c, int64_t(L.nt) * 8, 256), 256, 0, L.nt,
               (const int32_t*)L.tets.p, (const double*)L.xyz.p, (const int32_t*)L.iidx.p, Phi, N, ld, occ, e4);
    else if (N >= 32)
        launch(c, "sqload", k_sqload_elem_warp, grid_of(c, int64_t(L.nt) * 32, 256), 256, 0, L.nt,
               (const int32_t*)L.tets.p, (const double*)L.xyz.p, (const int32_t*)L.iidx.p, Phi, N, ld, occ, e4);
    else
        launch(c, "sqload", k_sqload_elem, grid_of(c, L.nt, 128), 128, 0, L.nt, (const int32_t*)L.tets.p,
               (const double*)L.xyz.p, (const int32_t*)L.iidx.p, Phi, N, ld, occ, e4);
}

/// out[r] = scale * sum over incident (t, l) of E4[t*4 + l], ascending t
__global__ void k_gather_vinc(int ni, const int32_t* __restrict__ ptr, const int32_t* __restrict__ inc,
                              const double* __restrict__ E4, double scale, double* __restrict__ out) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ni; r += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = ptr[r]; k < ptr[r + 1]; ++k) s += E4[inc[k]];
        out[r] = scale * s;
    }
}

/// out[rows[r]] = scale * sum of the incident element contributions (full-length scatter)
__global__ void k_gather_vinc_rows(int nr, const int32_t* __restrict__ ptr, const int32_t* __restrict__ inc,
                                   const double* __restrict__ E4, double scale, const int32_t* __restrict__ rows,
                                   double* __restrict__ out) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = ptr[r]; k < ptr[r + 1]; ++k) s += E4[inc[k]];
        out[rows[r]] = scale * s;
    }
}

__global__ void k_xc_field(int n, XcParams xc, const double* __restrict__ rho, double* __restrict__ vxc) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) vxc[v] = xc_potential(xc, rho[v]);
}

/// y[r] -= sum_k A_ib[r,k] xb[k]
__global__ void k_lift(int ni, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                       const double* __restrict__ val, const double* __restrict__ xb, double* __restrict__ y) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ni; r += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = ptr[r]; k < ptr[r + 1]; ++k) s += val[k] * xb[col[k]];
        y[r] -= s;
    }
}

__global__ void k_norm_parts(int nt, const int32_t* __restrict__ tets, const double* __restrict__ xyz,
                             const double* __restrict__ f, double* __restrict__ part) {
    double acc[2] = {0, 0};
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        const int4 v = reinterpret_cast<const int4*>(tets)[t];
        TetG G;
        tet_geometry(xyz, v, G);
        const double fv[4] = {f[v.x], f[v.y], f[v.z], f[v.w]};
        double sum = 0, sq = 0, gr[3] = {0, 0, 0};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            sum += fv[i];
            sq += fv[i] * fv[i];
#pragma unroll
            for (int d = 0; d < 3; ++d) gr[d] += fv[i] * G.g[i][d];
        }
        acc[0] += G.vol * (sum * sum + sq) / 20.0;
        acc[1] += G.vol * (gr[0] * gr[0] + gr[1] * gr[1] + gr[2] * gr[2]);
    }
    block_sum_to<2>(acc, part);
}

// fem::l1_norm via integrate_of (reference proj/src/assembly.cpp:234-249,289-291): Keast rule, |f(x_q)|
__global__ void k_l1_parts(int nt, const int32_t* __restrict__ tets, const double* __restrict__ xyz,
                           const double* __restrict__ f, double* __restrict__ part) {
    double acc[1] = {0};
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        const int4 v = reinterpret_cast<const int4*>(tets)[t];
        TetG G;
        tet_geometry(xyz, v, G);
        const double fv[4] = {f[v.x], f[v.y], f[v.z], f[v.w]};
        for (int q = 0; q < 11; ++q) {
            const double val = g_qb[q][0] * fv[0] + g_qb[q][1] * fv[1] + g_qb[q][2] * fv[2] + g_qb[q][3] * fv[3];
            acc[0] += g_qw[q] * G.vol * fabs(val);
        }
    }
    block_sum_to<1>(acc, part);
}

__constant__ double c_atoms[4 * 256];

__global__ void k_energy_parts(int nt, const int32_t* __restrict__ tets, const double* __restrict__ xyz,
                               const int32_t* __restrict__ iidx, const double* __restrict__ Phi, int N, int ld,
                               const double* __restrict__ rho, const double* __restrict__ w, int natoms, XcParams xc,
                               double* __restrict__ part) {
    double acc[4] = {0, 0, 0, 0};  // sum |grad phi|^2, ext, hartree, xc
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        const int4 v = reinterpret_cast<const int4*>(tets)[t];
        TetG G;
        tet_geometry(xyz, v, G);
        const int vv[4] = {v.x, v.y, v.z, v.w};
        for (int i = 0; i < N; ++i) {
            double gr[3] = {0, 0, 0};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double p = phi_at(Phi, iidx, vv[k], ld, i);
#pragma unroll
                for (int d = 0; d < 3; ++d) gr[d] += p * G.g[k][d];
            }
            acc[0] += G.vol * (gr[0] * gr[0] + gr[1] * gr[1] + gr[2] * gr[2]);
        }
        const double rv4[4] = {rho[v.x], rho[v.y], rho[v.z], rho[v.w]};
        const double wv4[4] = {w[v.x], w[v.y], w[v.z], w[v.w]};
        for (int q = 0; q < 11; ++q) {
            double rv = 0, wv = 0, x[3] = {0, 0, 0};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                rv += g_qb[q][k] * rv4[k];
                wv += g_qb[q][k] * wv4[k];
#pragma unroll
                for (int d = 0; d < 3; ++d) x[d] += g_qb[q][k] * G.x[k][d];
            }
            double vext = 0.0;
            for (int a = 0; a < natoms; ++a) {
                const double dx = x[0] - c_atoms[4 * a + 1], dy = x[1] - c_atoms[4 * a + 2], dz = x[2] - c_atoms[4 * a + 3];
                double r = sqrt(dx * dx + dy * dy + dz * dz);
                if (r < 1e-12) r = 1e-10;
                vext -= c_atoms[4 * a] / r;
            }
            const double s = g_qw[q] * G.vol;
            acc[1] += s * (rv * vext);
            acc[2] += s * rv * wv;
            acc[3] += s * xc_energy_density(xc, rv);
        }
    }
    block_sum_to<4>(acc, part);
}

template <int K>
std::array<double, K> reduce_parts(Ctx& c, DevBuf<double>& part, DevBuf<double>& out, int grid) {
    launch(c, "reduce", k_fold, 1, 256, 0, (const double*)part.p, grid, K, out.p);
    std::array<double, K> h{};
    KSB_CUDA_CHECK(cudaMemcpyAsync(h.data(), out.p, sizeof(double) * K, cudaMemcpyDeviceToHost, c.stream));
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    return h;
}

} // namespace

void PhysWork::ensure(const Level& L) {
    const int64_t need = int64_t(L.ctx->sm_count) * 8 * 16;
    if (part.n < need) part.alloc(need);
    if (out.n < 16) out.alloc(16);
    if (e4.n < int64_t(L.nt) * 4) e4.alloc(int64_t(L.nt) * 4);
}

void rho_vxc(Level& L, const double* Phi, int N, int ld, double occ, const XcParams& xc, double* rho_full,
             double* vxc_full) {
    Ctx& c = *L.ctx;
    KSB_CUDA_CHECK(cudaMemsetAsync(rho_full, 0, sizeof(double) * L.n, c.stream));
    if (vxc_full) KSB_CUDA_CHECK(cudaMemsetAsync(vxc_full, 0, sizeof(double) * L.n, c.stream));
    launch(c, "rho_vxc", k_rho_vxc, grid_of(c, L.ni), kT, 0, L.ni, N, ld, Phi, occ, xc, vxc_full ? 1 : 0,
           (const int32_t*)L.interior.p, rho_full, vxc_full);
}

Moments moments(Level& L, const double* rho_full, PhysWork& w, const double box_center[3]) {
    Ctx& c = *L.ctx;
    ensure_rule(c.stream);
    w.ensure(L);
    const int g = grid_of(c, L.nt);
    launch(c, "moments", k_moments1, g, kT, 0, L.nt, (const int32_t*)L.tets.p, (const double*)L.xyz.p, rho_full, w.part.p);
    const auto a = reduce_parts<4>(c, w.part, w.out, g);
    Moments m{};
    m.q = a[0];
    for (int d = 0; d < 3; ++d) m.c[d] = std::abs(a[0]) > 1e-14 ? a[1 + d] / a[0] : box_center[d];
    launch(c, "moments", k_moments2, g, kT, 0, L.nt, (const int32_t*)L.tets.p, (const double*)L.xyz.p, rho_full,
           m.c[0], m.c[1], m.c[2], w.part.p);
    const auto b = reduce_parts<12>(c, w.part, w.out, g);
    for (int d = 0; d < 3; ++d) m.dip[d] = b[d];
    double Q[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Q[i][j] = b[3 + 3 * i + j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m.Q[i][j] = 0.5 * (Q[i][j] + Q[j][i]);
    const double tr = (m.Q[0][0] + m.Q[1][1] + m.Q[2][2]) / 3.0;
    for (int i = 0; i < 3; ++i) m.Q[i][i] -= tr;
    return m;
}

void boundary_values(Level& L, const Moments& m, double* bcb) {
    Ctx& c = *L.ctx;
    bool zero = m.q == 0.0;
    for (int i = 0; i < 3; ++i) {
        zero = zero && m.dip[i] == 0.0;
        for (int j = 0; j < 3; ++j) zero = zero && m.Q[i][j] == 0.0;
    }
    if (zero) {
        KSB_CUDA_CHECK(cudaMemsetAsync(bcb, 0, sizeof(double) * L.nb, c.stream));
        return;
    }
    launch(c, "bc", k_bc, grid_of(c, L.nb), kT, 0, L.nb, (const int32_t*)L.boundary.p, (const double*)L.xyz.p, m, bcb);
}

void sqload(Level& L, const double* Phi, int N, int ld, double occ, double scale, double* out_int, PhysWork& w) {
    Ctx& c = *L.ctx;
    ensure_rule(c.stream);
    w.ensure(L);
    launch_sqload_elem(c, L, Phi, N, ld, occ, w.e4.p);
    launch(c, "sqload", k_gather_vinc, grid_of(c, L.ni), kT, 0, L.ni, (const int32_t*)L.vinc_ptr.p,
           (const int32_t*)L.vinc.p, (const double*)w.e4.p, scale, out_int);
}

void sqload_full(Level& L, const double* Phi, int N, int ld, double occ, double* out_full, PhysWork& w) {
    Ctx& c = *L.ctx;
    ensure_rule(c.stream);
    w.ensure(L);
    launch_sqload_elem(c, L, Phi, N, ld, occ, w.e4.p);
    launch(c, "sqload", k_gather_vinc_rows, grid_of(c, L.ni), kT, 0, L.ni, (const int32_t*)L.vinc_ptr.p,
           (const int32_t*)L.vinc.p, (const double*)w.e4.p, 1.0, (const int32_t*)L.interior.p, out_full);
    if (L.nb > 0)
        launch(c, "sqload", k_gather_vinc_rows, grid_of(c, L.nb), kT, 0, L.nb, (const int32_t*)L.bvinc_ptr.p,
               (const int32_t*)L.bvinc.p, (const double*)w.e4.p, 1.0, (const int32_t*)L.boundary.p, out_full);
}

void xc_field(Level& L, const XcParams& xc, const double* rho_full, double* vxc_full) {
    Ctx& c = *L.ctx;
    launch(c, "rho_vxc", k_xc_field, grid_of(c, L.n), kT, 0, L.n, xc, rho_full, vxc_full);
}

void lift(Level& L, int mat, const double* bcb, double* y_int) {
    Ctx& c = *L.ctx;
    if (!L.nnz_ib) return;
    launch(c, "lift", k_lift, grid_of(c, L.ni), kT, 0, L.ni, (const int32_t*)L.ib_ptr.p, (const int32_t*)L.ib_col.p,
           (const double*)L.mats[mat].ib.p, bcb, y_int);
}

std::array<double, 2> norms_sq(Level& L, const double* f_full, PhysWork& w) {
    Ctx& c = *L.ctx;
    w.ensure(L);
    const int g = grid_of(c, L.nt);
    launch(c, "norm", k_norm_parts, g, kT, 0, L.nt, (const int32_t*)L.tets.p, (const double*)L.xyz.p, f_full, w.part.p);
    return reduce_parts<2>(c, w.part, w.out, g);
}

double l1_norm(Level& L, const double* f_full, PhysWork& w) {
    Ctx& c = *L.ctx;
    ensure_rule(c.stream);
    w.ensure(L);
    const int g = grid_of(c, L.nt);
    launch(c, "norm", k_l1_parts, g, kT, 0, L.nt, (const int32_t*)L.tets.p, (const double*)L.xyz.p, f_full, w.part.p);
    return reduce_parts<1>(c, w.part, w.out, g)[0];
}

std::array<double, 5> energy(Level& L, const double* Phi, int N, int ld, const double* rho_full, const double* w_full,
                             const std::vector<double>& atoms, double occ, const XcParams& xc, PhysWork& w) {
    Ctx& c = *L.ctx;
    ensure_rule(c.stream);
    w.ensure(L);
    const int na = int(atoms.size() / 4);
    if (na > 256) raise(KSB_INVALID_ARGUMENT, "too many nuclei");
    if (na) KSB_CUDA_CHECK(cudaMemcpyToSymbolAsync(c_atoms, atoms.data(), sizeof(double) * atoms.size(), 0,
                                                   cudaMemcpyHostToDevice, c.stream));
    const int g = grid_of(c, L.nt, 128);
    launch(c, "energy", k_energy_parts, g, 128, 0, L.nt, (const int32_t*)L.tets.p, (const double*)L.xyz.p,
           (const int32_t*)L.iidx.p, Phi, N, ld, rho_full, w_full, na, xc, w.part.p);
    const auto a = reduce_parts<4>(c, w.part, w.out, g);
    std::array<double, 5> e{};
    e[0] = 0.5 * occ * a[0];
    e[1] = a[1];
    e[2] = 0.5 * a[2];
    e[3] = a[3];
    e[4] = e[0] + e[1] + e[2] + e[3];
    return e;
}

namespace {
/// out row = sum over the step row's (u, w) of w * in(u), ascending u, mul and add rounded separately
/// (the reference's col-major sparse product compiled without contraction)
__global__ void k_prolong(int rows, int ncols, const int32_t* __restrict__ out_vertex, const int32_t* __restrict__ pcol,
                          const double* __restrict__ pval, const int32_t* __restrict__ prev_iidx,
                          const double* __restrict__ in, int ld_in, double* __restrict__ out, int ld_out) {
    const int64_t total = int64_t(rows) * ncols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int r = int(e / ncols), c = int(e % ncols);
        const int v = out_vertex ? out_vertex[r] : r;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int u = pcol[4 * size_t(v) + k];
            if (u < 0) break;
            double x;
            if (prev_iidx) {
                const int q = prev_iidx[u];
                x = q >= 0 ? in[size_t(q) * ld_in + c] : 0.0;
            } else {
                x = in[size_t(u) * ld_in + c];
            }
            acc = __dadd_rn(acc, __dmul_rn(pval[4 * size_t(v) + k], x));
        }
        out[size_t(r) * ld_out + c] = acc;
    }
}
}  // namespace

void prolong(Level& L, const double* in, bool in_interior, int ld_in, int ncols, double* out, bool out_interior,
             int ld_out) {
    Ctx& c = *L.ctx;
    const int rows = out_interior ? L.ni : L.n;
    launch(c, "prolong", k_prolong, grid_of(c, int64_t(rows) * ncols), kT, 0, rows, ncols,
           out_interior ? (const int32_t*)L.interior.p : nullptr, (const int32_t*)L.pstep_col.p,
           (const double*)L.pstep_val.p, in_interior ? (const int32_t*)L.prev_iidx.p : nullptr, in, ld_in, out, ld_out);
}

} // namespace ksb
