// K-ASM: element matrices (tet-parallel) + deterministic slot gather.
//
// Element integrals follow the reference assembly (proj/src/assembly.cpp:19-30 tet_geom,
// :93-105 stiffness, :109-131 weighted mass with the 11-point Keast rule,
// proj/src/quadrature.cpp:9-36). The slot gather sums each CSR slot's element entries
// in ascending tet order, which is the duplicate-summation order of Eigen's
// setFromTriplets over the reference's tet-ordered triplet list (:36-63): no atomics,
// bitwise reproducible.
#include <cmath>

#include "level.cuh"
#include "dia.cuh"

namespace ksb {

namespace {

__constant__ double c_qw[11];      // Keast weights (sum to 1)
__constant__ double c_qb[11][4];   // barycentric coordinates
__constant__ double c_pot[5 * 256];

bool g_rule_ready = false;

void upload_rule(cudaStream_t s) {
    if (g_rule_ready) return;
    double w[11], b[11][4];
    const double w0 = -444.0 / 5625.0, w1 = 6.0 * 343.0 / 45000.0, w2 = 6.0 * 56.0 / 2250.0;
    const double a = 1.0 / 14.0;
    const double b1 = 0.25 * (1.0 + std::sqrt(5.0 / 14.0)), b2 = 0.25 * (1.0 - std::sqrt(5.0 / 14.0));
    int q = 0;
    w[q] = w0;
    for (int k = 0; k < 4; ++k) b[q][k] = 0.25;
    ++q;
    for (int k = 0; k < 4; ++k, ++q) {
        w[q] = w1;
        for (int j = 0; j < 4; ++j) b[q][j] = a;
        b[q][k] = 1.0 - 3.0 * a;
    }
    const int pr[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    for (int p = 0; p < 6; ++p, ++q) {
        w[q] = w2;
        for (int j = 0; j < 4; ++j) b[q][j] = b2;
        b[q][pr[p][0]] = b1;
        b[q][pr[p][1]] = b1;
    }
    KSB_CUDA_CHECK(cudaMemcpyToSymbolAsync(c_qw, w, sizeof w, 0, cudaMemcpyHostToDevice, s));
    KSB_CUDA_CHECK(cudaMemcpyToSymbolAsync(c_qb, b, sizeof b, 0, cudaMemcpyHostToDevice, s));
    KSB_CUDA_CHECK(cudaStreamSynchronize(s));
    g_rule_ready = true;
}

struct Geo {
    double x[4][3];
    double g[4][3];
    double vol;
};

__device__ __forceinline__ void tet_geo(const double* __restrict__ xyz, const int32_t* __restrict__ tets,
                                        int t, Geo& G) {
    const int4 v = reinterpret_cast<const int4*>(tets)[t];
    const int vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int d = 0; d < 3; ++d) G.x[i][d] = xyz[3 * vv[i] + d];
    double c[3][3];  // Jacobian columns
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) c[k][d] = G.x[k + 1][d] - G.x[0][d];
    // rows of J^{-1}: (c1 x c2, c2 x c0, c0 x c1) / det
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

__global__ void k_elem_stiffness(const double* __restrict__ xyz, const int32_t* __restrict__ tets, int nt,
                                 double* __restrict__ E) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        Geo G;
        tet_geo(xyz, tets, t, G);
        double* e = E + size_t(t) * 16;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
                e[i * 4 + j] = G.vol * (G.g[i][0] * G.g[j][0] + G.g[i][1] * G.g[j][1] + G.g[i][2] * G.g[j][2]);
    }
}

// weight source: 0 unit, 1 nodal P1 field, 2 coulomb centers, 3 gaussian centers
template <int WK>
__global__ void k_elem_mass(const double* __restrict__ xyz, const int32_t* __restrict__ tets, int nt,
                            const double* __restrict__ w, int ncenters, double* __restrict__ E,
                            int* __restrict__ flag) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        Geo G;
        tet_geo(xyz, tets, t, G);
        double wn[4] = {0, 0, 0, 0};
        if (WK == 1) {
            const int4 v = reinterpret_cast<const int4*>(tets)[t];
            wn[0] = w[v.x];
            wn[1] = w[v.y];
            wn[2] = w[v.z];
            wn[3] = w[v.w];
        }
        double K[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) K[i][j] = 0.0;
        bool bad = false;
#pragma unroll 1
        for (int q = 0; q < 11; ++q) {
            const double b0 = c_qb[q][0], b1 = c_qb[q][1], b2 = c_qb[q][2], b3 = c_qb[q][3];
            double wq;
            if (WK == 0) {
                wq = 1.0;
            } else if (WK == 1) {
                wq = b0 * wn[0] + b1 * wn[1] + b2 * wn[2] + b3 * wn[3];
            } else {
                double xq[3];
#pragma unroll
                for (int d = 0; d < 3; ++d)
                    xq[d] = b0 * G.x[0][d] + b1 * G.x[1][d] + b2 * G.x[2][d] + b3 * G.x[3][d];
                wq = 0.0;
                for (int k = 0; k < ncenters; ++k) {
                    if (WK == 2) {
                        const double* p = c_pot + 4 * k;
                        const double dx = xq[0] - p[1], dy = xq[1] - p[2], dz = xq[2] - p[3];
                        double r = sqrt(dx * dx + dy * dy + dz * dz);
                        if (r < 1e-12) r = 1e-10;
                        wq -= p[0] / r;
                    } else {
                        const double* p = c_pot + 5 * k;
                        const double dx = xq[0] - p[2], dy = xq[1] - p[3], dz = xq[2] - p[4];
                        wq -= p[0] * exp(-(dx * dx + dy * dy + dz * dz) / (2.0 * p[1] * p[1]));
                    }
                }
            }
            if (!isfinite(wq)) bad = true;
            const double s = c_qw[q] * G.vol * wq;
            const double b[4] = {b0, b1, b2, b3};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) K[i][j] += s * b[i] * b[j];
        }
        if (bad) atomicExch(flag, 1);
        double* e = E + size_t(t) * 16;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) e[i * 4 + j] = K[i][j];
    }
}

/// out[s] = (acc ? out[s] : 0) + c * sum_{k} E[gent[k]], k over slot s's list in ascending tet order
__global__ void k_gather(const int32_t* __restrict__ gptr, const int32_t* __restrict__ gent,
                         const double* __restrict__ E, int64_t nslots, double c, int acc,
                         double* __restrict__ out) {
    for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < nslots;
         s += int64_t(gridDim.x) * blockDim.x) {
        const int b = gptr[s], e = gptr[s + 1];
        double v = 0.0;
        if (b < e) {
            v = E[gent[b]];
            for (int k = b + 1; k < e; ++k) v += E[gent[k]];
        }
        out[s] = acc ? out[s] + c * v : c * v;
    }
}

__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b,
                        const double* __restrict__ y, double* __restrict__ z) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        z[i] = a * x[i] + b * y[i];
}

int grid_for(const Ctx& c, int64_t work, int block) {
    const int64_t want = (work + block - 1) / block;
    const int64_t cap = int64_t(c.sm_count) * 16;
    return int(want < cap ? (want > 0 ? want : 1) : cap);
}

} // namespace

void elem_potential(Level& L, const Potential& pot, double* E) {
    Ctx& c = *L.ctx;
    upload_rule(c.stream);
    const int stride = pot.kind == 0 ? 4 : 5;
    if (pot.n > 256 || int(pot.params.size()) != stride * pot.n)
        raise(KSB_INVALID_ARGUMENT, "potential descriptor too large or malformed");
    KSB_CUDA_CHECK(cudaMemcpyToSymbolAsync(c_pot, pot.params.data(), sizeof(double) * pot.params.size(), 0,
                                           cudaMemcpyHostToDevice, c.stream));
    KSB_CUDA_CHECK(cudaMemsetAsync(L.flag.p, 0, sizeof(int), c.stream));
    const int g = grid_for(c, L.nt, 128);
    if (pot.kind == 0)
        launch(c, "assemble", k_elem_mass<2>, g, 128, 0, (const double*)L.xyz.p, (const int32_t*)L.tets.p, L.nt,
               (const double*)nullptr, pot.n, E, L.flag.p);
    else
        launch(c, "assemble", k_elem_mass<3>, g, 128, 0, (const double*)L.xyz.p, (const int32_t*)L.tets.p, L.nt,
               (const double*)nullptr, pot.n, E, L.flag.p);
    int h_flag = 0;
    KSB_CUDA_CHECK(cudaMemcpyAsync(&h_flag, L.flag.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    if (h_flag) raise(KSB_SINGULAR_QUADRATURE, "weight is not finite at a quadrature point");
}

__global__ void k_sell_pack(int64_t n, const int32_t* __restrict__ map, const double* __restrict__ csr,
                            double* __restrict__ out) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const int m = map[k];
        out[k] = m >= 0 ? csr[m] : 0.0;
    }
}

const double* Level::sell_values(int id) {
    Mat& M = mats[id];
    if (!M.valid) raise(KSB_INVALID_ARGUMENT, "matrix not assembled");
    if (M.sell_version != M.version) {
        if (M.sell.n < sell_map.n) M.sell.alloc(sell_map.n);
        launch(*ctx, "sell_pack", k_sell_pack, grid_for(*ctx, sell_map.n, 256), 256, 0, int64_t(sell_map.n),
               (const int32_t*)sell_map.p, (const double*)M.ii.p, M.sell.p);
        M.sell_version = M.version;
    }
    return M.sell.p;
}

const double* Level::t8_values(int id) {
    Mat& M = mats[id];
    if (!M.valid) raise(KSB_INVALID_ARGUMENT, "matrix not assembled");
    if (t8_map.n == 0) return nullptr;
    if (M.t8_version != M.version) {
        if (M.t8.n < t8_map.n) M.t8.alloc(t8_map.n);
        launch(*ctx, "t8_pack", k_sell_pack, grid_for(*ctx, t8_map.n, 256), 256, 0, int64_t(t8_map.n),
               (const int32_t*)t8_map.p, (const double*)M.ii.p, M.t8.p);
        M.t8_version = M.version;
    }
    return M.t8.p;
}

/// CSR rows -> tiled stencil layout (dia.cuh: dia_pos); every slot of a row whose column offset is diagonal d of
/// the stencil lands in (row, d); diagonals without an entry stay 0
__global__ void k_dia_pack(int ni, DiaGeom dg, int D, int wg, const int32_t* __restrict__ ptr,
                           const int32_t* __restrict__ col, const int32_t* __restrict__ map,
                           const double* __restrict__ csr, double* __restrict__ out) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ni; r += gridDim.x * blockDim.x) {
        for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
            const int o = col[k] - r;
            int d = -1;
            for (int e = 0; e < D; ++e)
                if (dg.off[e] == o) d = e;
            if (d >= 0)
                out[wg == kDiaZT     ? dia_zt_pos(r, d, D, dg.n)
                    : wg == kDiaLine ? dia_line_pos(r, d, D, dg.n)
                                     : dia_pos(r, d, D, wg)] = csr[map ? map[k] : k];
        }
    }
}

const double* Level::dia_values(int id, int wg) {
    Mat& M = mats[id];
    if (!M.valid) raise(KSB_INVALID_ARGUMENT, "matrix not assembled");
    if (dia_ng == 0) return nullptr;
    if (M.dia_version != M.version || M.dia_wg != wg) {
        const DiaGeom dg = dia_geom(*this);
        if ((wg == kDiaLine || wg == kDiaZT) && dg.n == 0)
            raise(KSB_INTERNAL, "grid-tiled stencil layout on a level without a grid");
        const int64_t need = wg == kDiaZT     ? dia_zt_size(dg.n, dg.D)
                             : wg == kDiaLine ? dia_line_size(dg.n, dg.D)
                                              : dia_size(ni, dg.D, wg);
        if (M.dia.n < need) M.dia.alloc(need);
        KSB_CUDA_CHECK(cudaMemsetAsync(M.dia.p, 0, sizeof(double) * need, ctx->stream));
        const int32_t* ptr = dia_lo ? lo_ptr.p : ii_ptr.p;
        const int32_t* col = dia_lo ? lo_col.p : ii_col.p;
        const int32_t* map = dia_lo ? lo_map.p : nullptr;
        launch(*ctx, "dia_pack", k_dia_pack, grid_for(*ctx, ni, 256), 256, 0, ni, dg, dg.D, wg, ptr, col, map,
               (const double*)M.ii.p, M.dia.p);
        M.dia_version = M.version;
        M.dia_wg = wg;
    }
    return M.dia.p;
}

const double* Level::lo_values(int id) {
    Mat& M = mats[id];
    if (!M.valid) raise(KSB_INVALID_ARGUMENT, "matrix not assembled");
    if (lo_map.n == 0) return nullptr;
    if (M.lo_version != M.version) {
        if (M.lo.n < lo_map.n) M.lo.alloc(lo_map.n);
        launch(*ctx, "lo_pack", k_sell_pack, grid_for(*ctx, lo_map.n, 256), 256, 0, int64_t(lo_map.n),
               (const int32_t*)lo_map.p, (const double*)M.ii.p, M.lo.p);
        M.lo_version = M.version;
    }
    return M.lo.p;
}

const double* Level::ut_values(int id) {
    Mat& M = mats[id];
    if (!M.valid) raise(KSB_INVALID_ARGUMENT, "matrix not assembled");
    if (ut_map.n == 0) return nullptr;
    if (M.ut_version != M.version) {
        if (M.ut.n < ut_map.n) M.ut.alloc(ut_map.n);
        launch(*ctx, "lo_pack", k_sell_pack, grid_for(*ctx, ut_map.n, 256), 256, 0, int64_t(ut_map.n),
               (const int32_t*)ut_map.p, (const double*)M.ii.p, M.ut.p);
        M.ut_version = M.version;
    }
    return M.ut.p;
}

Mat& Level::mat(int id) {
    if (id < 0 || id >= kMaxMats) raise(KSB_INVALID_ARGUMENT, "matrix id out of range");
    Mat& m = mats[id];
    if (!m.valid) {
        m.ii.alloc(nnz_ii);
        m.ib.alloc(nnz_ib);
        m.valid = true;
    }
    return m;
}

void axpby_values(Level& L, int dst, double a, int x, double b, int y) {
    Ctx& c = *L.ctx;
    if (!L.mats[x].valid || !L.mats[y].valid) raise(KSB_INVALID_ARGUMENT, "operand matrix not assembled");
    Mat& D = L.mat(dst);
    L.touch(dst);
    launch(c, "axpby", k_axpby, grid_for(c, L.nnz_ii, 256), 256, 0, L.nnz_ii, a,
           (const double*)L.mats[x].ii.p, b, (const double*)L.mats[y].ii.p, D.ii.p);
    if (L.nnz_ib)
        launch(c, "axpby", k_axpby, grid_for(c, L.nnz_ib, 256), 256, 0, L.nnz_ib, a,
               (const double*)L.mats[x].ib.p, b, (const double*)L.mats[y].ib.p, D.ib.p);
}

void assemble_into(Level& L, int mat, double c_s, double c_m, const Potential* pot, double c_p,
                   const double* d_w, double c_w) {
    Ctx& c = *L.ctx;
    upload_rule(c.stream);
    if (L.ebuf.n < int64_t(L.nt) * 16) L.ebuf.alloc(int64_t(L.nt) * 16);
    Mat& M = L.mat(mat);
    L.touch(mat);
    const int blk = 128;
    const int g = grid_for(c, L.nt, blk);
    bool first = true;
    auto gather = [&](double coef) {
        launch(c, "assemble", k_gather, grid_for(c, L.nnz_ii, 256), 256, 0, (const int32_t*)L.ii_gptr.p,
               (const int32_t*)L.ii_gent.p, (const double*)L.ebuf.p, L.nnz_ii, coef, first ? 0 : 1, M.ii.p);
        if (L.nnz_ib)
            launch(c, "assemble", k_gather, grid_for(c, L.nnz_ib, 256), 256, 0, (const int32_t*)L.ib_gptr.p,
                   (const int32_t*)L.ib_gent.p, (const double*)L.ebuf.p, L.nnz_ib, coef, first ? 0 : 1, M.ib.p);
        first = false;
    };
    KSB_CUDA_CHECK(cudaMemsetAsync(L.flag.p, 0, sizeof(int), c.stream));
    if (c_s != 0.0) {
        launch(c, "assemble", k_elem_stiffness, g, blk, 0, (const double*)L.xyz.p, (const int32_t*)L.tets.p,
               L.nt, L.ebuf.p);
        gather(c_s);
    }
    if (c_m != 0.0) {
        launch(c, "assemble", k_elem_mass<0>, g, blk, 0, (const double*)L.xyz.p, (const int32_t*)L.tets.p,
               L.nt, (const double*)nullptr, 0, L.ebuf.p, L.flag.p);
        gather(c_m);
    }
    if (pot && pot->kind >= 0 && c_p != 0.0) {
        const int stride = pot->kind == 0 ? 4 : 5;
        if (pot->n > 256 || int(pot->params.size()) != stride * pot->n)
            raise(KSB_INVALID_ARGUMENT, "potential descriptor too large or malformed");
        KSB_CUDA_CHECK(cudaMemcpyToSymbolAsync(c_pot, pot->params.data(), sizeof(double) * pot->params.size(), 0,
                                               cudaMemcpyHostToDevice, c.stream));
        if (pot->kind == 0)
            launch(c, "assemble", k_elem_mass<2>, g, blk, 0, (const double*)L.xyz.p, (const int32_t*)L.tets.p,
                   L.nt, (const double*)nullptr, pot->n, L.ebuf.p, L.flag.p);
        else
            launch(c, "assemble", k_elem_mass<3>, g, blk, 0, (const double*)L.xyz.p, (const int32_t*)L.tets.p,
                   L.nt, (const double*)nullptr, pot->n, L.ebuf.p, L.flag.p);
        gather(c_p);
    }
    if (d_w && c_w != 0.0) {
        launch(c, "assemble", k_elem_mass<1>, g, blk, 0, (const double*)L.xyz.p, (const int32_t*)L.tets.p,
               L.nt, d_w, 0, L.ebuf.p, L.flag.p);
        gather(c_w);
    }
    if (first) {  // all coefficients zero: the zero matrix on the pattern
        KSB_CUDA_CHECK(cudaMemsetAsync(M.ii.p, 0, sizeof(double) * L.nnz_ii, c.stream));
        if (L.nnz_ib) KSB_CUDA_CHECK(cudaMemsetAsync(M.ib.p, 0, sizeof(double) * L.nnz_ib, c.stream));
    }
    int h_flag = 0;
    KSB_CUDA_CHECK(cudaMemcpyAsync(&h_flag, L.flag.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    if (h_flag) raise(KSB_SINGULAR_QUADRATURE, "weight is not finite at a quadrature point");
}

} // namespace ksb
