// Device-resident fine level: index data uploaded once, operator values on the shared pattern.
#pragma once

#include "../host/topology.hpp"
#include "common.cuh"

namespace ksb {

constexpr int kMaxMats = 32;

template <typename T>
struct DevBuf {
    T* p = nullptr;
    int64_t n = 0;
    void alloc(int64_t count) {
        release();
        n = count;
        if (count > 0) {
            const cudaError_t e = cudaMalloc(&p, sizeof(T) * size_t(count));
            if (e != cudaSuccess) {
                size_t fr = 0, tot = 0;
                cudaGetLastError();
                cudaMemGetInfo(&fr, &tot);
                p = nullptr;
                n = 0;
                raise(KSB_CUDA, "cudaMalloc of " + std::to_string(sizeof(T) * size_t(count) >> 20) + " MiB failed (" +
                                    cudaGetErrorString(e) + "; " + std::to_string(fr >> 20) + " of " +
                                    std::to_string(tot >> 20) + " MiB free)");
            }
        }
    }
    void upload(Ctx& c, const std::vector<T>& h) {
        alloc(int64_t(h.size()));
        if (n) KSB_CUDA_CHECK(cudaMemcpyAsync(p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, c.stream));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

struct Mat {
    DevBuf<double> ii, ib;
    DevBuf<double> sell;         // ii values in the SELL-32 order (lazily converted)
    DevBuf<double> t8;           // ii values in the T8 order (lazily converted)
    DevBuf<double> lo;           // ii values on the locality-ordered pattern (lazily converted)
    DevBuf<double> ut;           // ii values in the union-tile order (lazily converted)
    DevBuf<double> dia;          // ii values in the tiled stencil (DIA) layout (lazily converted, see dia_values)
    uint64_t version = 0, sell_version = ~uint64_t(0), t8_version = ~uint64_t(0), lo_version = ~uint64_t(0);
    uint64_t dia_version = ~uint64_t(0), ut_version = ~uint64_t(0);
    int dia_wg = 0;              // rows per warp step the DIA values were packed for
    bool valid = false;
};

/// dependency levels of the forward / backward triangular solves of a level's interior pattern (sgs.cu)
struct SgsPlan {
    DevBuf<int32_t> f_rows, b_rows;
    std::vector<int> f_bounds, b_bounds;
    bool ready = false;
};

struct Level {
    Ctx* ctx = nullptr;
    uint64_t uid = 0;  // process-unique id (never reused): keys the CG graph cache (cg.cu)
    std::shared_ptr<FineTopology> topo;
    int n = 0, ni = 0, nb = 0, nt = 0;
    int64_t nnz_ii = 0, nnz_ib = 0;
    int nH = 0, nct = 0, ncv = 0;  // coarse interior dofs, coarse tets, coarse vertices

    DevBuf<double> xyz;
    DevBuf<int32_t> tets;
    DevBuf<int32_t> interior, iidx, boundary;
    DevBuf<int32_t> ii_ptr, ii_col, ib_ptr, ib_col, diag_slot;
    DevBuf<int32_t> ii_gptr, ii_gent, ib_gptr, ib_gent;
    DevBuf<int32_t> pint_col;
    DevBuf<double> pint_val;
    DevBuf<int32_t> ancestor, anc_ptr, anc_tets;
    // K-PROJ work chunks over anc_tets (project.cu): chunk k = [pj_b[k], pj_e[k]) of coarse tet pj_c[k]; pj_ptr[C] =
    // first chunk of coarse tet C; pj_n = number of chunks (== nct when no coarse tet is split)
    DevBuf<int32_t> pj_c, pj_b, pj_e, pj_ptr;
    int pj_n = 0;
    // aggregated K-PROJ (GEMM form): compact chunks of each coarse tet's fine tets (topology.hpp ProjChunks), built
    // on the first many-orbital projection
    DevBuf<int32_t> pg_item_c, pg_item_ch, pg_cptr, pg_ch_t, pg_ch_v, pg_ch_e, pg_tets, pg_verts, pg_edges,
        pg_vinc_ptr, pg_vinc, pg_einc_ptr, pg_einc;
    int pg_items = 0;
    bool pg_ready = false;
    DevBuf<int32_t> vinc_ptr, vinc;           // interior vertex -> incident (tet*4 + local)
    DevBuf<int32_t> bvinc_ptr, bvinc;         // boundary vertex -> incident (tet*4 + local)
    DevBuf<int32_t> cinc_ptr, cinc;           // coarse interior dof -> incident (coarse tet*4 + local)
    DevBuf<int32_t> ctets, ciidx;             // coarse mesh (level 0)
    DevBuf<double> cxyz;
    DevBuf<int32_t> sell_ptr, sell_col, sell_map;
    DevBuf<int32_t> t8_col, t8_map;  // T8 view (empty when a row is longer than 16)
    DevBuf<int32_t> lo_perm, lo_ptr, lo_col, lo_map, lo_dslot;  // locality-ordered pattern (topology.hpp)
    int lo_max_row = 0;
    DevBuf<int32_t> ut_rows, ut_eptr, ut_ent, ut_map;  // union-tile view of the ordered pattern (topology.hpp)
    int ut_nt = 0;
    // stencil (DIA) view (topology.hpp): dia_ng runs, run 0 = {-1, 0, 1}, the others of length dia_lr starting at
    // dia_first[q]; on the natural order (dia_lo = 0) or the locality order (dia_lo = 1); dia_ng = 0 without one
    int dia_ng = 0, dia_lr = 0, dia_lo = 0, dia_n = 0;
    int dia_first[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    int nslices = 0;
    int max_row_ii = 0;  // longest row of the interior pattern (selects the streamed SpMM when <= 16)
    DevBuf<int32_t> pstep_col, prev_iidx;   // one-step prolongation from level-1 (empty on level 0)
    DevBuf<double> pstep_val;
    int n_prev = 0;
    double box_lo[3] = {0, 0, 0}, box_hi[3] = {0, 0, 0};
    DevBuf<double> ebuf;      // element matrices, 16 per tet (scratch)
    DevBuf<double> scratch;   // term accumulation scratch (nnz_ii + nnz_ib)
    DevBuf<int> flag;         // device error flag (singular quadrature)
    Mat mats[kMaxMats];
    SgsPlan sgs_plan;  // level sets of the SGS triangular solves (sgs.cu, built on first use)
    std::vector<MeshPtr> meshes;  // the hierarchy's meshes 0..level (coarser levels for the multigrid)

    Mat& mat(int id);
    /// SELL-32 values of matrix id (converted on first use after its values changed)
    const double* sell_values(int id);
    /// T8 values of matrix id (converted on first use after its values changed); null without a T8 view
    const double* t8_values(int id);
    /// values of matrix id on the locality-ordered pattern (converted on first use after a change); null
    /// without a locality order
    const double* lo_values(int id);
    /// values of matrix id in the union-tile order (converted on first use after a change); null without the view
    const double* ut_values(int id);
    /// values of matrix id in the tiled stencil layout for wg rows per warp step (dia.cuh), converted on first use
    /// after a change; null without a stencil view
    const double* dia_values(int id, int wg);
    void touch(int id) { ++mats[id].version; }
};

/// host index data -> device arrays (level.cu); L.ctx and L.topo set, operator values not assembled
void upload_level(Ctx& cx, std::shared_ptr<FineTopology> topo, Level& L);

// assembly (assemble.cu)
struct Potential {
    int kind = -1;
    int n = 0;
    std::vector<double> params;
};
void assemble_into(Level& L, int mat, double c_s, double c_m, const Potential* pot, double c_p,
                   const double* d_w, double c_w);

// SpMM (spmm.cu): Y = (A + sigma_j B) X on interior blocks; B may be null (sigma ignored)
void spmm(Ctx& c, const Level& L, const double* A, const double* B, const double* d_sigma,
          const double* X, int N, int ldx, double* Y, int ldy);

} // namespace ksb
