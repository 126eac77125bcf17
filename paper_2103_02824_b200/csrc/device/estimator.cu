// K-EST: residual indicators (reference proj/src/estimator.cpp:11-85) on the device.
//
//   eta_T^2 = h_T^2 int_T sum_i ((V_ext + w + v_xc - lambda_i) phi_i)^2          (Keast rule, per tet)
//           + sum over interior faces e of T (ascending face index, as the reference's face loop adds them)
//             h_e |e| sum_i (1/2 [grad phi_i] . n_e)^2
//
// Three passes: element residual (tet-parallel), face jumps (face-parallel, one value per face), and a per-tet
// gather of its faces in ascending face order, so every eta_T is summed in the reference's order. The total is
// a fixed-order block reduction. Face geometry (unit normal oriented away from the lower tet, area, longest
// edge) is the mesh's own, computed on the host by the reference's formula (proj/src/mesh.cpp:196-211).
#include <algorithm>

#include "geom.cuh"
#include "physics.cuh"

namespace ksb {

namespace {

constexpr int kT = 256;

int grid_of(const Ctx& c, int64_t work, int block = kT) {
    return int(std::max<int64_t>(1, std::min<int64_t>((work + block - 1) / block, int64_t(c.sm_count) * 8)));
}

__global__ void k_est_elem(int nt, const int32_t* __restrict__ tets, const double* __restrict__ xyz,
                           const int32_t* __restrict__ iidx, const double* __restrict__ Phi, int N, int ld,
                           const double* __restrict__ w, const double* __restrict__ vxc, const double* __restrict__ atoms,
                           int natoms, const double* __restrict__ lam, double* __restrict__ eta) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        const int4 v = reinterpret_cast<const int4*>(tets)[t];
        TetG G;
        tet_geometry(xyz, v, G);
        const int vv[4] = {v.x, v.y, v.z, v.w};
        int ri[4];
        double wn[4], vn[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            ri[k] = iidx[vv[k]];
            wn[k] = w[vv[k]];
            vn[k] = vxc[vv[k]];
        }
        double acc = 0.0;
        for (int q = 0; q < 11; ++q) {
            double x[3] = {0.0, 0.0, 0.0}, wq = 0.0, vq = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
#pragma unroll
                for (int d = 0; d < 3; ++d) x[d] += g_qb[q][k] * G.x[k][d];
                wq += g_qb[q][k] * wn[k];
                vq += g_qb[q][k] * vn[k];
            }
            double ve = 0.0;  // model::v_ext (proj/src/ks_model.cpp:33-41)
            for (int a = 0; a < natoms; ++a) {
                const double* p = atoms + 4 * a;
                const double dx = x[0] - p[1], dy = x[1] - p[2], dz = x[2] - p[3];
                double r = sqrt(dx * dx + dy * dy + dz * dz);
                if (r < 1e-12) r = 1e-10;
                ve -= p[0] / r;
            }
            const double pot = ve + wq + vq;
            double sum_sq = 0.0;
            for (int i = 0; i < N; ++i) {
                double phi = 0.0;
#pragma unroll
                for (int k = 0; k < 4; ++k) phi += g_qb[q][k] * (ri[k] >= 0 ? Phi[size_t(ri[k]) * ld + i] : 0.0);
                const double r = (pot - lam[i]) * phi;
                sum_sq += r * r;
            }
            acc += g_qw[q] * G.vol * sum_sq;
        }
        double hT = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = i + 1; j < 4; ++j) {
                const double a = G.x[i][0] - G.x[j][0], b = G.x[i][1] - G.x[j][1], c = G.x[i][2] - G.x[j][2];
                hT = fmax(hT, sqrt(a * a + b * b + c * c));
            }
        eta[t] = hT * hT * acc;
    }
}

__global__ void k_est_face(int nif, const int32_t* __restrict__ ftets, const double* __restrict__ fgeom,
                           const int32_t* __restrict__ tets, const double* __restrict__ xyz,
                           const int32_t* __restrict__ iidx, const double* __restrict__ Phi, int N, int ld,
                           double* __restrict__ contrib) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nif; f += gridDim.x * blockDim.x) {
        const int tp = ftets[2 * f], tm = ftets[2 * f + 1];
        const double* gm = fgeom + 5 * size_t(f);
        TetG Gp, Gm;
        const int4 vp = reinterpret_cast<const int4*>(tets)[tp], vm = reinterpret_cast<const int4*>(tets)[tm];
        tet_geometry(xyz, vp, Gp);
        tet_geometry(xyz, vm, Gm);
        const int ap[4] = {vp.x, vp.y, vp.z, vp.w}, am[4] = {vm.x, vm.y, vm.z, vm.w};
        int rp[4], rm[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            rp[k] = iidx[ap[k]];
            rm[k] = iidx[am[k]];
        }
        double jump_sq = 0.0;
        for (int i = 0; i < N; ++i) {
            double g1[3] = {0.0, 0.0, 0.0}, g2[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double fp = rp[k] >= 0 ? Phi[size_t(rp[k]) * ld + i] : 0.0;
                const double fm = rm[k] >= 0 ? Phi[size_t(rm[k]) * ld + i] : 0.0;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    g1[d] += fp * Gp.g[k][d];
                    g2[d] += fm * Gm.g[k][d];
                }
            }
            double jn = 0.0;
#pragma unroll
            for (int d = 0; d < 3; ++d) jn += 0.5 * (g1[d] - g2[d]) * gm[d];
            jump_sq += jn * jn;
        }
        contrib[f] = gm[4] * jump_sq * gm[3];
    }
}

__global__ void k_est_gather(int nt, const int32_t* __restrict__ tptr, const int32_t* __restrict__ tf,
                             const double* __restrict__ contrib, double* __restrict__ eta, double* __restrict__ part) {
    __shared__ double red[32];
    double s = 0.0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        double e = eta[t];
        for (int k = tptr[t]; k < tptr[t + 1]; ++k) e += contrib[tf[k]];
        eta[t] = e;
        s += e;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}

__global__ void k_sum_parts(const double* __restrict__ part, int n, double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += part[i];
        out[0] = s;
    }
}

}  // namespace

void EstimatorData::ensure(Level& L) {
    if (ready) return;
    const Mesh& m = *L.topo->space->mesh;
    const int nif = int(m.iface_tets.size() / 2), nt = m.n_tets();
    Ctx& c = *L.ctx;
    ftets.upload(c, m.iface_tets);
    fgeom.upload(c, m.iface_geom);
    std::vector<int32_t> ptr(size_t(nt) + 1, 0), tf(size_t(2) * nif);
    for (int f = 0; f < nif; ++f) {
        ++ptr[size_t(m.iface_tets[2 * f]) + 1];
        ++ptr[size_t(m.iface_tets[2 * f + 1]) + 1];
    }
    for (int t = 0; t < nt; ++t) ptr[size_t(t) + 1] += ptr[size_t(t)];
    std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
    for (int f = 0; f < nif; ++f) {  // ascending f per tet: the reference's accumulation order
        tf[size_t(fill[size_t(m.iface_tets[2 * f])]++)] = f;
        tf[size_t(fill[size_t(m.iface_tets[2 * f + 1])]++)] = f;
    }
    tptr.upload(c, ptr);
    tface.upload(c, tf);
    contrib.alloc(std::max(1, nif));
    part.alloc(int64_t(c.sm_count) * 8);
    scal.alloc(4);
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));  // host staging vectors go out of scope
    ready = true;
}

double indicators(Level& L, EstimatorData& E, const std::vector<double>& atoms, const double* h_lambda, int N,
                  const double* d_Phi, int ld, const double* d_w, const double* d_vxc, double* d_eta) {
    Ctx& c = *L.ctx;
    ensure_rule(c.stream);
    E.ensure(L);
    if (int(E.lam.n) < N) E.lam.alloc(std::max(1, N));
    if (E.atoms.n < int64_t(std::max<size_t>(1, atoms.size()))) E.atoms.alloc(int64_t(std::max<size_t>(1, atoms.size())));
    KSB_CUDA_CHECK(cudaMemcpyAsync(E.lam.p, h_lambda, sizeof(double) * N, cudaMemcpyHostToDevice, c.stream));
    if (!atoms.empty())
        KSB_CUDA_CHECK(cudaMemcpyAsync(E.atoms.p, atoms.data(), sizeof(double) * atoms.size(), cudaMemcpyHostToDevice,
                                       c.stream));
    const int nif = int(L.topo->space->mesh->iface_tets.size() / 2);
    launch(c, "estimator", k_est_elem, grid_of(c, L.nt, 128), 128, 0, L.nt, (const int32_t*)L.tets.p,
           (const double*)L.xyz.p, (const int32_t*)L.iidx.p, d_Phi, N, ld, d_w, d_vxc, (const double*)E.atoms.p,
           int(atoms.size() / 4), (const double*)E.lam.p, d_eta);
    if (nif > 0)
        launch(c, "estimator", k_est_face, grid_of(c, nif, 128), 128, 0, nif, (const int32_t*)E.ftets.p,
               (const double*)E.fgeom.p, (const int32_t*)L.tets.p, (const double*)L.xyz.p, (const int32_t*)L.iidx.p,
               d_Phi, N, ld, E.contrib.p);
    const int g = grid_of(c, L.nt);
    launch(c, "estimator", k_est_gather, g, kT, 0, L.nt, (const int32_t*)E.tptr.p, (const int32_t*)E.tface.p,
           (const double*)E.contrib.p, d_eta, E.part.p);
    launch(c, "estimator", k_sum_parts, 1, 32, 0, (const double*)E.part.p, g, E.scal.p);
    double tot = 0.0;
    KSB_CUDA_CHECK(cudaMemcpyAsync(&tot, E.scal.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    KSB_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    return tot;
}

}  // namespace ksb
