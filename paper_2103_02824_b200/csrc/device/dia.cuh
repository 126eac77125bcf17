// Stencil (DIA) view of a level's interior operator: layout shared by the pack kernel (assemble.cu) and the
// stencil SpMM (cg.cu, k_spmm_dia).
//
// On a level whose interior rows form a uniform stencil in the solver's row numbering (topology.hpp: box meshes in
// lexicographic order carry the Kuhn 15-point stencil, uniformly refined levels in the locality order the 27-point
// box), row r couples only to rows r + off[d] for D fixed offsets. The offsets split into runs of consecutive
// values (one per (dy, dz) line of the grid), so a warp that walks S consecutive rows slides one window per run:
// each step gathers ONE new block row per run (7 for Kuhn, 9 for the box) instead of one per nonzero (15), and the
// column indices disappear (the operator is D values per row, 0 where the pattern has no entry).
//
// Value layout ("tiled DIA"): rows are cut into tiles of T = wg * S rows; lane group g of a warp owns the S rows
// [tile * T + g * S, ... + S). For step s of a tile the values of the wg rows the warp processes together are
// contiguous: diagonal pair p of group g at 2 * (p * wg + g) (one 16-byte load per lane, the wg groups of a warp
// read one contiguous run), an odd last diagonal at 2 * (D / 2) * wg + g. Step stride = D * wg rounded up to even.
#pragma once

#include "level.cuh"

namespace ksb {

constexpr int kDiaS = 32;  // rows per lane group and tile

/// stencil geometry by value: D diagonals in kernel order (run 0 = {-1, 0, 1}, then the runs of length lr in
/// ascending order), the first offset of every run
struct DiaGeom {
    int D, ng, lr;
    int n;  // cubic grid dimension (rows = x + n (y + n z)), 0 when the level is not a grid
    int off[27];
    int first[9];
    int rdx[9], rdy[9], rdz[9];  // grid levels: (dx, dy, dz) of the first offset of every run
};

inline DiaGeom dia_geom(const Level& L) {
    DiaGeom g{};
    g.ng = L.dia_ng;
    g.lr = L.dia_lr;
    g.n = L.dia_n;
    g.D = 0;
    for (int q = 0; q < L.dia_ng; ++q) {
        g.first[q] = L.dia_first[q];
        const int len = q == 0 ? 3 : L.dia_lr;
        for (int j = 0; j < len; ++j) g.off[g.D++] = L.dia_first[q] + j;
        if (g.n > 0) {  // decode offset = dx + n (dy + n dz), |d| <= 1 (topology.cpp checked it)
            const int o = L.dia_first[q], n = g.n;
            const int dz = (o + n * n + (n * n) / 2) / (n * n) - 1;  // nearest multiple of n^2 (n >= 3)
            const int rem = o - dz * n * n;
            const int dy = (rem + n + n / 2) / n - 1;
            g.rdz[q] = dz;
            g.rdy[q] = dy;
            g.rdx[q] = rem - dy * n;
        }
    }
    return g;
}

__host__ __device__ inline int64_t dia_step_stride(int D, int wg) { return (int64_t(D) * wg + 1) & ~int64_t(1); }

__host__ __device__ inline int64_t dia_size(int ni, int D, int wg) {
    const int64_t T = int64_t(wg) * kDiaS;
    const int64_t tiles = (ni + T - 1) / T;
    return tiles * kDiaS * dia_step_stride(D, wg);
}

/// position of (row r, diagonal d) in the tiled layout
__host__ __device__ inline int64_t dia_pos(int r, int d, int D, int wg) {
    const int T = wg * kDiaS;
    const int t = r / T, rem = r % T, g = rem / kDiaS, s = rem % kDiaS;
    const int64_t base = (int64_t(t) * kDiaS + s) * dia_step_stride(D, wg);
    const int pairs = D / 2;
    return base + (d < 2 * pairs ? int64_t(2) * ((d / 2) * wg + g) + (d & 1) : int64_t(2) * pairs * wg + g);
}

// Line-tiled layout (z-marching kernel k_spmm_dia_z): every grid line (y, z) is cut into segments of kDiaSeg = 32
// rows (the last one padded); a segment is one warp's work for one plane: its 4 lane groups own 8 consecutive rows
// each (group g: x = 32 xt + 8 g + s, step s). Segment (xt, y, z) = ((z n + y) nxt + xt), nxt = ceil(n / 32); its 8
// steps follow each other, step s holding the 4 rows' diagonals as in the band layout (wg = 4).
constexpr int kDiaLine = 100;  // layout id of the line-tiled layout (band layouts use their wg = 1 .. 16)
constexpr int kDiaSeg = 32;

__host__ __device__ inline int64_t dia_line_size(int n, int D) {
    const int64_t nxt = (n + kDiaSeg - 1) / kDiaSeg;
    return int64_t(n) * n * nxt * 8 * dia_step_stride(D, 4);
}

__host__ __device__ inline int64_t dia_line_pos(int r, int d, int D, int n) {
    const int x = r % n, yz = r / n;
    const int nxt = (n + kDiaSeg - 1) / kDiaSeg;
    const int xt = x / kDiaSeg, xin = x % kDiaSeg, g = xin / 8, s = xin % 8;
    const int64_t SD = dia_step_stride(D, 4);
    const int64_t base = ((int64_t(yz) * nxt + xt) * 8 + s) * SD;
    const int pairs = D / 2;
    return base + (d < 2 * pairs ? int64_t(2) * ((d / 2) * 4 + g) + (d & 1) : int64_t(2) * pairs * 4 + g);
}

// Plane-tiled layout (TMA-staged z-marching kernel k_spmm_dia_zt): the grid is cut into (x, y) tiles of kZtT x kZtT
// rows; the values of one tile in one plane are one contiguous block of kZtT^2 D doubles, so a single bulk copy stages
// them. Inside a block: warp w (lines 2w, 2w + 1 of the tile), step s (x = 8 (g % 2) + s), diagonal pairs of the 4
// lane groups g (line 2w + g / 2) as in the band layout (wg = 4).
constexpr int kDiaZT = 200;  // layout id
constexpr int kZtT = 16;

__host__ __device__ inline int64_t dia_zt_size(int n, int D) {
    const int64_t nt = (n + kZtT - 1) / kZtT;
    return nt * nt * n * kZtT * kZtT * D;
}

__host__ __device__ inline int64_t dia_zt_pos(int r, int d, int D, int n) {
    const int x = r % n, y = (r / n) % n, z = r / (n * n);
    const int nt = (n + kZtT - 1) / kZtT;
    const int xt = x / kZtT, xl = x % kZtT, yt = y / kZtT, yl = y % kZtT;
    const int w = yl / 2, g = (yl % 2) * 2 + xl / 8, s = xl % 8;
    const int64_t base = ((int64_t(z) * nt + yt) * nt + xt) * (kZtT * kZtT * D) + int64_t(w) * 8 * 4 * D + s * 4 * D;
    const int pairs = D / 2;
    return base + (d < 2 * pairs ? int64_t(2) * ((d / 2) * 4 + g) + (d & 1) : int64_t(2) * pairs * 4 + g);
}

} // namespace ksb
