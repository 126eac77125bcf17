// Host-side index data for one fine level: FE space split, composite
// prolongation to the coarse level, CSR patterns and the deterministic
// assembly gather lists the device kernels consume.
//
//   FESpace interior/boundary split   reference proj/src/fespace.cpp:7-18
//   prolongation_matrix + chaining    reference proj/src/fespace.cpp:35-56,64-74
//   interior_columns (P_int)          reference proj/src/correction.cpp:79-90
//   EllipticSolver gather (A_ii,A_ib) reference proj/src/solver.cpp:11-24,28-48
//   setFromTriplets duplicate order   reference proj/src/assembly.cpp:36-63
#pragma once

#include "mesh.hpp"

namespace ksb {

struct Space {
    MeshPtr mesh;
    std::vector<int32_t> interior;   // vertex ids, ascending
    std::vector<int32_t> boundary;   // vertex ids, ascending
    std::vector<int32_t> iidx;       // vertex -> interior position or -1
    std::vector<int32_t> bidx;       // vertex -> boundary position or -1
    explicit Space(MeshPtr m);
    int n() const { return mesh->n_vertices(); }
    int ni() const { return int(interior.size()); }
    int nb() const { return int(boundary.size()); }
};

/// Nested sequence of meshes with composite transfer data to level 0.
class Hierarchy {
public:
    void push(MeshPtr m);
    int n_levels() const { return int(meshes_.size()); }
    const Mesh& mesh(int k) const { return *meshes_.at(k); }
    MeshPtr mesh_ptr(int k) const { return meshes_.at(k); }
    /// composite prolongation row of vertex v of level k to level-0 vertices (<=4 entries, col ascending)
    const std::vector<int32_t>& pcol(int k) const { return pcol_.at(k); }   // n_k*4, -1 padded
    const std::vector<double>& pval(int k) const { return pval_.at(k); }    // n_k*4
    const std::vector<int32_t>& ancestor(int k) const { return anc_.at(k); } // level-0 tet per tet

private:
    std::vector<MeshPtr> meshes_;
    std::vector<std::vector<int32_t>> pcol_;
    std::vector<std::vector<double>> pval_;
    std::vector<std::vector<int32_t>> anc_;
};

/// CSR block over interior rows. Columns are in interior (ii) or boundary (ib) numbering.
struct Csr {
    int32_t rows = 0, cols = 0;
    std::vector<int32_t> ptr;
    std::vector<int32_t> col;
    int64_t nnz() const { return ptr.empty() ? 0 : ptr.back(); }
};

/// Everything the device needs to know about a fine level's index structure.
struct FineTopology {
    std::shared_ptr<Space> space;      // fine space
    std::shared_ptr<Space> coarse;     // level-0 space
    Csr ii, ib;                        // interior x interior, interior x boundary patterns
    std::vector<int32_t> diag_slot;    // ii slot of (r, r)
    // slot -> element-matrix entries (t*16 + li*4 + lj), ascending t (setFromTriplets order)
    std::vector<int32_t> ii_gptr, ib_gptr;
    std::vector<int32_t> ii_gent, ib_gent;
    // composite P_int restricted to fine interior rows: <=4 (coarse interior col, value) per row
    std::vector<int32_t> pint_col;     // ni*4, -1 padded
    std::vector<double> pint_val;      // ni*4
    std::vector<int32_t> ancestor;     // per fine tet, level-0 tet
    std::vector<int32_t> anc_ptr;      // coarse tet -> range in anc_tets
    std::vector<int32_t> anc_tets;     // fine tets grouped by coarse ancestor, ascending inside a group
    // interior fine vertex -> incident (tet*4 + local), ascending tet (load-vector gather order)
    std::vector<int32_t> vinc_ptr, vinc;
    // boundary fine vertex -> incident (tet*4 + local), ascending tet (full-length load vectors)
    std::vector<int32_t> bvinc_ptr, bvinc;
    // coarse level: interior coarse dof -> incident (coarse tet*4 + local), ascending tet
    std::vector<int32_t> cinc_ptr, cinc;
    // SELL-32 view of the ii pattern: slice s = rows [32s, 32s+32), entry e of lane i at
    // sell_ptr[s] + 32 e + i; padding entries point at the row itself with map = -1
    std::vector<int32_t> sell_ptr, sell_col, sell_map;
    // T8 view (only when no interior row is longer than 16): ELL with 16 slots per row, row-major:
    // t8_col[16 r + q] = column of slot q of row r, t8_map[16 r + q] = its CSR position; padding -1 / -1
    std::vector<int32_t> t8_col, t8_map;
    // Locality order for the multi-column CG (only when the T8 view is absent, i.e. refined / adaptive levels,
    // whose vertex numbering scatters a row's neighbours over the whole index range): interior rows sorted by
    // vertex (z, y, x). perm[i] = natural row of ordered row i; the ordered pattern (lo_ptr, lo_col, rows and
    // columns renumbered, columns ascending), lo_map = natural CSR slot of each ordered slot, lo_dslot = diagonal
    // slot. Empty when not built.
    std::vector<int32_t> lo_perm, lo_ptr, lo_col, lo_map, lo_dslot;
    int lo_max_row = 0;
    // Union-tile ("UT") view of the locality-ordered pattern for blocks of more than 16 columns: tiles of <= kUtR
    // ordered rows that are neighbours in space (consecutive in the Morton order of their vertices). A tile lists
    // the union of its rows' columns once (ascending) and stores a dense kUtR-vector of values per column (zero
    // where a row does not hold it), so the kernel gathers every distinct X row once per tile and feeds it to all
    // tile rows from registers, with no per-entry dispatch (~2x fewer gathered rows than row by row, ~2x the
    // multiply-adds). ut_rows[kUtR t + i] = ordered row of tile slot i (-1: none); entries
    // [ut_eptr[t], ut_eptr[t+1]) = ordered columns, padded to a multiple of 4 with a valid row whose values are
    // zero; values of entry e at [kUtR e, kUtR e + kUtR); ut_map = natural CSR slot of each value (-1: zero).
    // A tile holds <= kUtE entries. Empty when not built (no locality order, or a row longer than kUtE).
    std::vector<int32_t> ut_rows, ut_eptr, ut_ent, ut_map;
    int ut_nt = 0;
    // Stencil (DIA) view: the interior rows are a uniform stencil in the natural numbering (dia_lo = 0; box meshes,
    // lexicographic) or in the locality order (dia_lo = 1; uniformly refined levels): every column offset
    // (col - row) lies in a set that splits into runs of consecutive offsets -- a centre run {-1, 0, 1} and
    // dia_ng - 1 further runs of one common length dia_lr. dia_first[q] = first offset of run q (run 0 = centre,
    // the others ascending). Supported shapes: Kuhn 15-point (7 runs, 3 + 6 x 2) and box 27-point (9 x 3).
    // dia_ng = 0 when the level has no stencil view.
    int dia_ng = 0, dia_l0 = 0, dia_lr = 0, dia_lo = 0;
    int dia_n = 0;  // > 0: the rows are an n x n x n grid, row = x + n (y + n z), all couplings between neighbours
    std::vector<int32_t> dia_first;
    // one-step prolongation from level-1 (fem::prolongation_matrix, proj/src/fespace.cpp:35-56): per vertex <= 4
    // (previous-level vertex, weight), ascending vertex, -1 padded; empty on level 0. prev_iidx: the previous
    // level's vertex -> interior index (interior-block inputs).
    int n_prev = 0;
    std::vector<int32_t> pstep_col, prev_iidx;
    std::vector<double> pstep_val;
};

/// union-tile view limits: rows per tile and entries (distinct columns) per tile (cg.cu stages a tile's columns
/// and dense values in shared memory: kUtE * (4 + 8 kUtR) bytes per buffer)
constexpr int kUtR = 4, kUtE = 64;

/// lite: only what a multigrid level needs (interior / boundary patterns, assembly gathers, diagonal, SELL-32 view,
/// one-step prolongation); P_int, incidences, T8 / locality / stencil views and the ancestor grouping stay empty
std::shared_ptr<FineTopology> build_topology(const Hierarchy& h, int level, bool lite = false);

/// Aggregated projection (K-PROJ GEMM form, project.cu): the fine tets of every coarse tet in Morton order of their
/// centroids, cut greedily into compact chunks (<= kPgT tets, <= kPgV vertices, <= kPgE edges), each chunk with its
/// sorted vertex and edge lists and the incidence of every local vertex / edge (chunk-local tet, corners) in
/// ascending tet order; consecutive chunks of one coarse tet grouped into work items of <= kPgItem chunks.
constexpr int kPgT = 96, kPgV = 80, kPgE = 240, kPgItem = 32;
struct ProjChunks {
    std::vector<int32_t> item_c, item_ch;      // per item: coarse tet, first chunk (item_ch has n_items + 1 entries)
    std::vector<int32_t> cptr;                 // per coarse tet: first item (n_coarse_tets + 1)
    std::vector<int32_t> ch_t, ch_v, ch_e;     // per chunk: first tet / vertex / edge (n_chunks + 1 entries each)
    std::vector<int32_t> tets, verts, edges;   // fine tet ids; global vertex ids; local pairs lu | lv << 16 (lu < lv)
    std::vector<int32_t> vinc_ptr, vinc;       // per vertex slot: incidences t << 2 | corner
    std::vector<int32_t> einc_ptr, einc;       // per edge slot: incidences t << 4 | c1 << 2 | c2
};
ProjChunks build_proj_chunks(const FineTopology& T);

/// est::dorfler_mark (proj/src/estimator.cpp:87-104): tets by descending eta, ties by lower index, up to the first
/// cumulative sum >= theta * total; writes them to `marked` in that order and returns their count. The order is a
/// strict total order, so the parallel sort gives the reference's sequence exactly.
int64_t dorfler_mark(const double* eta, int64_t nt, double total_sq, double theta, int32_t* marked);

} // namespace ksb
