// Host index builders for a fine level. See topology.hpp for reference anchors.
#include "topology.hpp"

#include <algorithm>
#include <functional>
#include <iterator>
#include <parallel/algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>

namespace ksb {

Space::Space(MeshPtr m) : mesh(std::move(m)) {
    const int nv = mesh->n_vertices();
    iidx.assign(nv, -1);
    bidx.assign(nv, -1);
    for (int v = 0; v < nv; ++v) {
        if (mesh->on_boundary[v]) {
            bidx[v] = int32_t(boundary.size());
            boundary.push_back(v);
        } else {
            iidx[v] = int32_t(interior.size());
            interior.push_back(v);
        }
    }
}

void Hierarchy::push(MeshPtr m) {
    const int nv = m->n_vertices();
    std::vector<int32_t> col(size_t(nv) * 4, -1);
    std::vector<double> val(size_t(nv) * 4, 0.0);
    std::vector<int32_t> anc(m->n_tets());
    if (meshes_.empty()) {
        for (int v = 0; v < nv; ++v) {
            col[4 * v] = v;
            val[4 * v] = 1.0;
        }
        for (int t = 0; t < m->n_tets(); ++t) anc[t] = t;
    } else {
        if (m->n_parent_vertices != meshes_.back()->n_vertices())
            raise(KSB_HIERARCHY, "levels are not nested");
        const auto& pc = pcol_.back();
        const auto& pv = pval_.back();
        const int np = m->n_parent_vertices;
        std::copy(pc.begin(), pc.begin() + size_t(np) * 4, col.begin());
        std::copy(pv.begin(), pv.begin() + size_t(np) * 4, val.begin());
        // new vertices average their parent edge; parents precede children and
        // every row is a convex combination of <= 4 coarse vertices (dyadic, exact)
        for (int v = np; v < nv; ++v) {
            const int a = m->vparent[2 * v], b = m->vparent[2 * v + 1];
            // parents precede children (also guards loaded dumps against out-of-range or cyclic parents)
            if (a < 0 || b < 0 || a >= v || b >= v) raise(KSB_HIERARCHY, "vertex parent not created before its child");
            int32_t c[8];
            double w[8];
            int cnt = 0;
            auto add = [&](int src) {
                for (int k = 0; k < 4 && col[4 * src + k] >= 0; ++k) {
                    const int32_t cc = col[4 * src + k];
                    const double ww = 0.5 * val[4 * src + k];
                    int j = 0;
                    while (j < cnt && c[j] != cc) ++j;
                    if (j == cnt) {
                        c[cnt] = cc;
                        w[cnt] = ww;
                        ++cnt;
                    } else {
                        w[j] += ww;
                    }
                }
            };
            add(a);
            add(b);
            if (cnt > 4) raise(KSB_INTERNAL, "prolongation row wider than one coarse tet");
            // sort by coarse column
            for (int i = 1; i < cnt; ++i)
                for (int j = i; j > 0 && c[j - 1] > c[j]; --j) {
                    std::swap(c[j - 1], c[j]);
                    std::swap(w[j - 1], w[j]);
                }
            for (int k = 0; k < cnt; ++k) {
                col[4 * v + k] = c[k];
                val[4 * v + k] = w[k];
            }
        }
        const auto& pa = anc_.back();
        const int64_t npt = int64_t(pa.size());
        for (int t = 0; t < m->n_tets(); ++t) {
            const int32_t p = m->parent[t];
            if (p < 0 || p >= npt) raise(KSB_HIERARCHY, "tet parent out of range of the previous level");
            anc[t] = pa[p];
        }
    }
    meshes_.push_back(std::move(m));
    pcol_.push_back(std::move(col));
    pval_.push_back(std::move(val));
    anc_.push_back(std::move(anc));
}

namespace {

void check_i32(int64_t x, const char* what) {
    if (x > std::numeric_limits<int32_t>::max())
        raise(KSB_INVALID_ARGUMENT, std::string(what) + " exceeds the int32 index range");
}

/// 21 bits per axis interleaved (x lowest)
uint64_t morton3(uint32_t x, uint32_t y, uint32_t z) {
    auto spread = [](uint64_t v) {
        v &= 0x1fffffull;
        v = (v | v << 32) & 0x1f00000000ffffull;
        v = (v | v << 16) & 0x1f0000ff0000ffull;
        v = (v | v << 8) & 0x100f00f00f00f00full;
        v = (v | v << 4) & 0x10c30c30c30c30c3ull;
        v = (v | v << 2) & 0x1249249249249249ull;
        return v;
    };
    return spread(x) | spread(y) << 1 | spread(z) << 2;
}

/// rows sorted by the Morton code of their vertex: key[k] = (code, position in `rows`); rows[i] = natural interior row
std::vector<std::pair<uint64_t, int32_t>> morton_keys(const double* xyz, const int32_t* interior, int ni,
                                                      const std::vector<int32_t>& rows) {
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int i = 0; i < ni; ++i) {
        const double* p = xyz + 3 * size_t(interior[rows[i]]);
        for (int d = 0; d < 3; ++d) {
            lo[d] = std::min(lo[d], p[d]);
            hi[d] = std::max(hi[d], p[d]);
        }
    }
    double ext = 0.0;
    for (int d = 0; d < 3; ++d) ext = std::max(ext, hi[d] - lo[d]);
    if (!(ext > 0.0)) ext = 1.0;
    std::vector<std::pair<uint64_t, int32_t>> key(ni);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < ni; ++i) {
        const double* p = xyz + 3 * size_t(interior[rows[i]]);
        uint32_t q[3];
        for (int d = 0; d < 3; ++d) q[d] = uint32_t(std::min(2097151.0, (p[d] - lo[d]) / ext * 2097151.0));
        key[i] = {morton3(q[0], q[1], q[2]), i};
    }
    __gnu_parallel::sort(key.begin(), key.end());
    return key;
}

/// perm = the natural interior rows in Morton order of their vertices (ties by row)
void morton_order(const double* xyz, const int32_t* interior, int ni, std::vector<int32_t>& perm) {
    std::vector<int32_t> ident(ni);
    for (int i = 0; i < ni; ++i) ident[i] = i;
    const auto key = morton_keys(xyz, interior, ni, ident);
    perm.resize(ni);
    for (int i = 0; i < ni; ++i) perm[i] = key[i].second;
}

/// Union-tile view of the locality-ordered pattern (topology.hpp): ordered rows sorted by the Morton code of their
/// vertex, cut greedily into tiles of <= kUtR rows with <= kUtE distinct columns.
void build_union_tiles(FineTopology& T, const double* xyz, const int32_t* interior, int ni) {
    const auto& ptr = T.lo_ptr;
    const auto& col = T.lo_col;
    const auto key = morton_keys(xyz, interior, ni, T.lo_perm);

    // tile boundaries: independent greedy cuts inside fixed chunks of the Morton sequence
    const int chunk = 1 << 14, nchunks = (ni + chunk - 1) / chunk;
    std::vector<std::vector<int32_t>> starts(nchunks);
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < nchunks; ++c) {
        const int b = c * chunk, e = std::min(ni, b + chunk);
        std::vector<int32_t> uni, tmp;
        int rows = 0;
        for (int k = b; k < e; ++k) {
            const int r = key[k].second;
            tmp.clear();
            std::set_union(uni.begin(), uni.end(), col.begin() + ptr[r], col.begin() + ptr[r + 1], std::back_inserter(tmp));
            if (rows == 0 || rows == kUtR || int(tmp.size()) > kUtE) {
                starts[c].push_back(k);
                uni.assign(col.begin() + ptr[r], col.begin() + ptr[r + 1]);
                rows = 1;
            } else {
                uni.swap(tmp);
                ++rows;
            }
        }
    }
    std::vector<int32_t> tstart;
    for (auto& s : starts) tstart.insert(tstart.end(), s.begin(), s.end());
    const int nt = int(tstart.size());
    tstart.push_back(ni);

    // sizes, then the fill
    T.ut_nt = nt;
    T.ut_rows.assign(size_t(nt) * kUtR, -1);
    std::vector<int64_t> ecnt(size_t(nt) + 1, 0);
#pragma omp parallel for schedule(static)
    for (int t = 0; t < nt; ++t) {
        const int k0 = tstart[t], nr = tstart[t + 1] - k0;
        int32_t rows[16];  // (sized past kUtR: keeps the sort's insertion pass in bounds for the compiler)
        for (int i = 0; i < nr; ++i) rows[i] = key[k0 + i].second;
        std::sort(rows, rows + nr);
        std::vector<int32_t> uni, tmp;
        for (int i = 0; i < nr; ++i) {
            T.ut_rows[size_t(t) * kUtR + i] = rows[i];
            tmp.clear();
            std::set_union(uni.begin(), uni.end(), col.begin() + ptr[rows[i]], col.begin() + ptr[rows[i] + 1],
                           std::back_inserter(tmp));
            uni.swap(tmp);
        }
        ecnt[t + 1] = (int64_t(uni.size()) + 3) / 4 * 4;
    }
    for (int t = 0; t < nt; ++t) ecnt[t + 1] += ecnt[t];
    check_i32(ecnt[nt] * kUtR, "union-tile values");
    T.ut_eptr.resize(size_t(nt) + 1);
    for (int t = 0; t <= nt; ++t) T.ut_eptr[t] = int32_t(ecnt[t]);
    T.ut_ent.assign(size_t(ecnt[nt]), 0);
    T.ut_map.assign(size_t(ecnt[nt]) * kUtR, -1);
#pragma omp parallel for schedule(static)
    for (int t = 0; t < nt; ++t) {
        const int32_t* rows = T.ut_rows.data() + size_t(t) * kUtR;
        int head[kUtR], end[kUtR], nr = 0;
        while (nr < kUtR && rows[nr] >= 0) {
            head[nr] = ptr[rows[nr]];
            end[nr] = ptr[rows[nr] + 1];
            ++nr;
        }
        int64_t e = ecnt[t];
        for (;;) {
            int32_t cmin = std::numeric_limits<int32_t>::max();
            for (int i = 0; i < nr; ++i)
                if (head[i] < end[i]) cmin = std::min(cmin, col[head[i]]);
            if (cmin == std::numeric_limits<int32_t>::max()) break;
            for (int i = 0; i < nr; ++i)
                if (head[i] < end[i] && col[head[i]] == cmin) T.ut_map[size_t(e) * kUtR + i] = T.lo_map[head[i]++];
            T.ut_ent[e++] = cmin;
        }
        for (; e < ecnt[t + 1]; ++e) T.ut_ent[e] = rows[0];  // padding: a valid row to gather, all values zero
    }
}

} // namespace

std::shared_ptr<FineTopology> build_topology(const Hierarchy& h, int level, bool lite) {
    auto topo = std::make_shared<FineTopology>();
    const Mesh& m = h.mesh(level);
    topo->space = std::make_shared<Space>(h.mesh_ptr(level));
    topo->coarse = std::make_shared<Space>(h.mesh_ptr(0));
    const Space& S = *topo->space;
    const int nv = S.n(), ni = S.ni(), nt = m.n_tets();
    check_i32(int64_t(nt) * 16, "16 * n_tets");

    // vertex -> incident tets, ascending tet id (counting sort)
    std::vector<int32_t> vptr(size_t(nv) + 1, 0), vtet(size_t(nt) * 4);
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 4; ++k) ++vptr[m.tets[4 * t + k] + 1];
    for (int v = 0; v < nv; ++v) vptr[v + 1] += vptr[v];
    {
        std::vector<int32_t> fill(vptr.begin(), vptr.end() - 1);
        for (int t = 0; t < nt; ++t)
            for (int k = 0; k < 4; ++k) vtet[fill[m.tets[4 * t + k]]++] = t;
    }

    // interior-row patterns: all vertices sharing a tet with the row vertex
    std::vector<std::vector<int32_t>> rowv(ni);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int r = 0; r < ni; ++r) {
        const int v = S.interior[r];
        auto& nb = rowv[r];
        nb.reserve(32);
        for (int p = vptr[v]; p < vptr[v + 1]; ++p)
            for (int k = 0; k < 4; ++k) nb.push_back(m.tets[4 * vtet[p] + k]);
        std::sort(nb.begin(), nb.end());
        nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
    }
    auto& ii = topo->ii;
    auto& ib = topo->ib;
    ii.rows = ib.rows = ni;
    ii.cols = ni;
    ib.cols = S.nb();
    ii.ptr.assign(size_t(ni) + 1, 0);
    ib.ptr.assign(size_t(ni) + 1, 0);
    {
        int64_t ci = 0, cb = 0;
        for (int r = 0; r < ni; ++r) {
            for (int32_t c : rowv[r]) (S.iidx[c] >= 0 ? ci : cb)++;
            check_i32(ci, "interior nnz");
            ii.ptr[r + 1] = int32_t(ci);
            ib.ptr[r + 1] = int32_t(cb);
        }
    }
    ii.col.resize(ii.ptr.back());
    ib.col.resize(ib.ptr.back());
    topo->diag_slot.resize(ni);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < ni; ++r) {
        int32_t pi = ii.ptr[r], pb = ib.ptr[r];
        for (int32_t c : rowv[r]) {
            if (S.iidx[c] >= 0) {
                if (c == S.interior[r]) topo->diag_slot[r] = pi;
                ii.col[pi++] = S.iidx[c];
            } else {
                ib.col[pb++] = S.bidx[c];
            }
        }
    }

    // slot gather lists: element entry (t, li, lj) feeds slot (v[li], v[lj]) of an interior row.
    // Walking a row's incident tets in ascending order yields the setFromTriplets fold order.
    topo->ii_gptr.assign(size_t(ii.nnz()) + 1, 0);
    topo->ib_gptr.assign(size_t(ib.nnz()) + 1, 0);
    auto find_slot = [&](int r, int32_t vcol, bool& interior_col) -> int32_t {
        if (S.iidx[vcol] >= 0) {
            interior_col = true;
            const int32_t key = S.iidx[vcol];
            const int32_t* b = ii.col.data() + ii.ptr[r];
            const int32_t* e = ii.col.data() + ii.ptr[r + 1];
            return int32_t(std::lower_bound(b, e, key) - ii.col.data());
        }
        interior_col = false;
        const int32_t key = S.bidx[vcol];
        const int32_t* b = ib.col.data() + ib.ptr[r];
        const int32_t* e = ib.col.data() + ib.ptr[r + 1];
        return int32_t(std::lower_bound(b, e, key) - ib.col.data());
    };
#pragma omp parallel for schedule(dynamic, 1024)
    for (int r = 0; r < ni; ++r) {
        const int v = S.interior[r];
        for (int p = vptr[v]; p < vptr[v + 1]; ++p) {
            const int t = vtet[p];
            for (int lj = 0; lj < 4; ++lj) {
                bool in;
                const int32_t s = find_slot(r, m.tets[4 * t + lj], in);
                (in ? topo->ii_gptr : topo->ib_gptr)[s + 1]++;
            }
        }
    }
    for (size_t s = 0; s + 1 < topo->ii_gptr.size(); ++s) topo->ii_gptr[s + 1] += topo->ii_gptr[s];
    for (size_t s = 0; s + 1 < topo->ib_gptr.size(); ++s) topo->ib_gptr[s + 1] += topo->ib_gptr[s];
    topo->ii_gent.resize(topo->ii_gptr.back());
    topo->ib_gent.resize(topo->ib_gptr.back());
#pragma omp parallel for schedule(dynamic, 1024)
    for (int r = 0; r < ni; ++r) {
        const int v = S.interior[r];
        // per-row fill cursors (slots of one row are private to this iteration)
        std::vector<int32_t> fi(topo->ii_gptr.begin() + ii.ptr[r], topo->ii_gptr.begin() + ii.ptr[r + 1]);
        std::vector<int32_t> fb(topo->ib_gptr.begin() + ib.ptr[r], topo->ib_gptr.begin() + ib.ptr[r + 1]);
        for (int p = vptr[v]; p < vptr[v + 1]; ++p) {
            const int t = vtet[p];
            int li = 0;
            while (m.tets[4 * t + li] != v) ++li;
            for (int lj = 0; lj < 4; ++lj) {
                bool in;
                const int32_t s = find_slot(r, m.tets[4 * t + lj], in);
                const int32_t e = t * 16 + li * 4 + lj;
                if (in) topo->ii_gent[fi[s - ii.ptr[r]]++] = e;
                else topo->ib_gent[fb[s - ib.ptr[r]]++] = e;
            }
        }
    }

    if (!lite) {
    // composite prolongation restricted to interior coarse columns (P_int), interior fine rows
    const Space& C = *topo->coarse;
    const auto& pc = h.pcol(level);
    const auto& pv = h.pval(level);
    // fine boundary vertices interpolate coarse boundary vertices only, so their
    // P_int rows vanish (this is what lets every fine operator live on interior rows)
    for (int32_t v : S.boundary)
        for (int k = 0; k < 4 && pc[4 * size_t(v) + k] >= 0; ++k)
            if (C.iidx[pc[4 * size_t(v) + k]] >= 0)
                raise(KSB_INTERNAL, "fine boundary vertex couples to a coarse interior vertex");
    topo->pint_col.assign(size_t(ni) * 4, -1);
    topo->pint_val.assign(size_t(ni) * 4, 0.0);
    for (int r = 0; r < ni; ++r) {
        const int v = S.interior[r];
        int w = 0;
        for (int k = 0; k < 4; ++k) {
            const int32_t c = pc[4 * size_t(v) + k];
            if (c < 0) break;
            if (C.iidx[c] < 0) continue;
            topo->pint_col[4 * size_t(r) + w] = C.iidx[c];
            topo->pint_val[4 * size_t(r) + w] = pv[4 * size_t(v) + k];
            ++w;
        }
    }

    // interior vertex incidence (t*4 + local), ascending t
    topo->vinc_ptr.assign(size_t(ni) + 1, 0);
    for (int r = 0; r < ni; ++r) topo->vinc_ptr[r + 1] = topo->vinc_ptr[r] + (vptr[S.interior[r] + 1] - vptr[S.interior[r]]);
    topo->vinc.resize(topo->vinc_ptr.back());
#pragma omp parallel for schedule(static)
    for (int r = 0; r < ni; ++r) {
        const int v = S.interior[r];
        int32_t w = topo->vinc_ptr[r];
        for (int p = vptr[v]; p < vptr[v + 1]; ++p) {
            const int t = vtet[p];
            int li = 0;
            while (m.tets[4 * t + li] != v) ++li;
            topo->vinc[w++] = t * 4 + li;
        }
    }
    // boundary vertex incidence, same order rule
    {
        const int nb = S.nb();
        topo->bvinc_ptr.assign(size_t(nb) + 1, 0);
        for (int r = 0; r < nb; ++r)
            topo->bvinc_ptr[r + 1] = topo->bvinc_ptr[r] + (vptr[S.boundary[r] + 1] - vptr[S.boundary[r]]);
        topo->bvinc.resize(topo->bvinc_ptr.back());
#pragma omp parallel for schedule(static)
        for (int r = 0; r < nb; ++r) {
            const int v = S.boundary[r];
            int32_t w = topo->bvinc_ptr[r];
            for (int p = vptr[v]; p < vptr[v + 1]; ++p) {
                const int t = vtet[p];
                int li = 0;
                while (m.tets[4 * t + li] != v) ++li;
                topo->bvinc[w++] = t * 4 + li;
            }
        }
    }
    // coarse interior incidence
    {
        const Mesh& cm = *topo->coarse->mesh;
        const Space& Cs = *topo->coarse;
        topo->cinc_ptr.assign(size_t(Cs.ni()) + 1, 0);
        for (int t = 0; t < cm.n_tets(); ++t)
            for (int k = 0; k < 4; ++k) {
                const int a = Cs.iidx[cm.tets[4 * t + k]];
                if (a >= 0) ++topo->cinc_ptr[a + 1];
            }
        for (int a = 0; a < Cs.ni(); ++a) topo->cinc_ptr[a + 1] += topo->cinc_ptr[a];
        topo->cinc.resize(topo->cinc_ptr.back());
        std::vector<int32_t> fill(topo->cinc_ptr.begin(), topo->cinc_ptr.end() - 1);
        for (int t = 0; t < cm.n_tets(); ++t)
            for (int k = 0; k < 4; ++k) {
                const int a = Cs.iidx[cm.tets[4 * t + k]];
                if (a >= 0) topo->cinc[fill[a]++] = t * 4 + k;
            }
    }

    }  // !lite

    // SELL-32 view of the interior pattern (column-major inside each 32-row slice)
    {
        const int ns = (ni + 31) / 32;
        topo->sell_ptr.assign(size_t(ns) + 1, 0);
        int64_t off = 0;
        for (int sl = 0; sl < ns; ++sl) {
            int w = 0;
            for (int i = 0; i < 32 && 32 * sl + i < ni; ++i)
                w = std::max(w, ii.ptr[32 * sl + i + 1] - ii.ptr[32 * sl + i]);
            off += int64_t(w) * 32;
            check_i32(off, "SELL entries");
            topo->sell_ptr[sl + 1] = int32_t(off);
        }
        topo->sell_col.assign(size_t(off), 0);
        topo->sell_map.assign(size_t(off), -1);
#pragma omp parallel for schedule(static)
        for (int sl = 0; sl < ns; ++sl) {
            const int w = (topo->sell_ptr[sl + 1] - topo->sell_ptr[sl]) / 32;
            for (int i = 0; i < 32; ++i) {
                const int r = 32 * sl + i;
                const int rr = r < ni ? r : ni - 1;  // rows past the end replay the last row (never stored)
                for (int e = 0; e < w; ++e) {
                    const size_t k = size_t(topo->sell_ptr[sl]) + size_t(e) * 32 + i;
                    const int slot = ii.ptr[rr] + e;
                    if (r < ni && slot < ii.ptr[rr + 1]) {
                        topo->sell_col[k] = ii.col[slot];
                        topo->sell_map[k] = slot;
                    } else {
                        topo->sell_col[k] = rr;
                    }
                }
            }
        }
    }

    if (!lite) {
    // T8 view of the interior pattern (streamed N = 16 SpMM): built when every row fits 16 slots
    {
        int wmax = 0;
        for (int r = 0; r < ni; ++r) wmax = std::max(wmax, ii.ptr[r + 1] - ii.ptr[r]);
        if (wmax <= 16 && ni > 0) {
            check_i32(int64_t(ni) * 16, "T8 entries");
            topo->t8_col.assign(size_t(ni) * 16, -1);
            topo->t8_map.assign(size_t(ni) * 16, -1);
#pragma omp parallel for schedule(static)
            for (int r = 0; r < ni; ++r) {
                for (int q = 0; q < ii.ptr[r + 1] - ii.ptr[r]; ++q) {
                    topo->t8_col[size_t(r) * 16 + q] = ii.col[ii.ptr[r] + q];
                    topo->t8_map[size_t(r) * 16 + q] = ii.ptr[r] + q;
                }
            }
        }
    }

    // locality order for the multi-column CG (refined / adaptive levels, see topology.hpp): the ordered pattern of
    // a given row permutation
    auto build_lo = [&]() {
        const auto& perm = topo->lo_perm;
        std::vector<int32_t> iperm(ni);
        for (int i = 0; i < ni; ++i) iperm[perm[i]] = i;
        topo->lo_ptr.assign(size_t(ni) + 1, 0);
        for (int i = 0; i < ni; ++i) topo->lo_ptr[i + 1] = topo->lo_ptr[i] + (ii.ptr[perm[i] + 1] - ii.ptr[perm[i]]);
        topo->lo_col.resize(ii.col.size());
        topo->lo_map.resize(ii.col.size());
        topo->lo_dslot.assign(ni, -1);
        int wmax = 0;
#pragma omp parallel for schedule(static) reduction(max : wmax)
        for (int i = 0; i < ni; ++i) {
            const int r = perm[i], b = ii.ptr[r], len = ii.ptr[r + 1] - b;
            wmax = std::max(wmax, len);
            std::vector<std::pair<int32_t, int32_t>> e(len);
            for (int q = 0; q < len; ++q) e[q] = {iperm[ii.col[b + q]], b + q};
            std::sort(e.begin(), e.end());
            for (int q = 0; q < len; ++q) {
                topo->lo_col[topo->lo_ptr[i] + q] = e[q].first;
                topo->lo_map[topo->lo_ptr[i] + q] = e[q].second;
                if (e[q].first == i) topo->lo_dslot[i] = topo->lo_ptr[i] + q;
            }
        }
        topo->lo_max_row = wmax;
    };
    if (topo->t8_col.empty() && ni > 0) {
        auto& perm = topo->lo_perm;
        perm.resize(ni);
        for (int r = 0; r < ni; ++r) perm[r] = r;
        const double* X = m.xyz.data();
        std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) {
            const double* pa = X + 3 * size_t(S.interior[a]);
            const double* pb = X + 3 * size_t(S.interior[b]);
            if (pa[2] != pb[2]) return pa[2] < pb[2];
            if (pa[1] != pb[1]) return pa[1] < pb[1];
            return pa[0] < pb[0];
        });
        build_lo();
    }

    // stencil (DIA) view: natural order first, else the locality order
    {
        auto detect = [&](const std::vector<int32_t>& ptr, const std::vector<int32_t>& col, int on_lo) {
            if (ni < 2 || ptr.empty()) return false;
            constexpr int kMax = 27;
            std::vector<int32_t> offs;
            bool overflow = false;
#pragma omp parallel
            {
                std::vector<int32_t> mine;
                bool over = false;
#pragma omp for schedule(static) nowait
                for (int r = 0; r < ni; ++r) {
                    if (over) continue;
                    for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
                        const int32_t o = col[k] - r;
                        if (std::find(mine.begin(), mine.end(), o) == mine.end()) {
                            mine.push_back(o);
                            if (int(mine.size()) > kMax) {
                                over = true;
                                break;
                            }
                        }
                    }
                }
#pragma omp critical
                {
                    overflow = overflow || over;
                    for (int32_t o : mine)
                        if (std::find(offs.begin(), offs.end(), o) == offs.end()) offs.push_back(o);
                }
            }
            if (overflow || int(offs.size()) > kMax) return false;
            std::sort(offs.begin(), offs.end());
            std::vector<std::pair<int32_t, int>> runs;  // (first offset, length)
            for (int32_t o : offs) {
                if (!runs.empty() && runs.back().first + runs.back().second == o)
                    ++runs.back().second;
                else
                    runs.push_back({o, 1});
            }
            int centre = -1, lr = 0;
            for (int q = 0; q < int(runs.size()); ++q) {
                if (runs[q].first == -1 && runs[q].second == 3) {
                    centre = q;
                } else {
                    if (lr && runs[q].second != lr) return false;
                    lr = runs[q].second;
                }
            }
            const int ng = int(runs.size());
            const bool kuhn = ng == 7 && lr == 2, box = ng == 9 && lr == 3;
            if (centre < 0 || !(kuhn || box)) return false;
            topo->dia_first.assign(1, -1);
            for (int q = 0; q < ng; ++q)
                if (q != centre) topo->dia_first.push_back(runs[q].first);
            topo->dia_ng = ng;
            topo->dia_l0 = 3;
            topo->dia_lr = lr;
            topo->dia_lo = on_lo;
            // a cubic grid (rows = x + n (y + n z)) whose every entry couples geometric neighbours (no offset wraps
            // around a grid line or plane): the z-marching stencil SpMM may tile it by (x, y) blocks
            const int n = int(std::lround(std::cbrt(double(ni))));
            bool grid = n >= 3 && int64_t(n) * n * n == ni;
            for (int32_t o : offs) {
                if (!grid) break;
                const int dz = int(std::lround(double(o) / (double(n) * n)));
                const int rem = o - dz * n * n;
                const int dy = int(std::lround(double(rem) / n));
                const int dx = rem - dy * n;
                grid = std::abs(dx) <= 1 && std::abs(dy) <= 1 && std::abs(dz) <= 1;
            }
            if (grid) {
                int bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
                for (int r = 0; r < ni; ++r) {
                    const int x = r % n, y = (r / n) % n, z = r / (n * n);
                    for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
                        const int c = col[k];
                        const int dx = c % n - x, dy = (c / n) % n - y, dz = c / (n * n) - z;
                        bad += std::abs(dx) > 1 || std::abs(dy) > 1 || std::abs(dz) > 1;
                    }
                }
                grid = bad == 0;
            }
            topo->dia_n = grid ? n : 0;
            return true;
        };
        if (!detect(ii.ptr, ii.col, 0) && !topo->lo_perm.empty()) detect(topo->lo_ptr, topo->lo_col, 1);
    }

    // Opt-in (KSB_LO_MORTON=1): levels whose (z, y, x) order is no stencil (adaptive levels) take the Morton order
    // of the vertices instead (median |i - j| ~13 against ~180 rows, but a long tail across octant boundaries).
    // Measured at the configs' sizes: N = 120 union-tile SpMM at 11.56 M rows 15.9 -> 15.8 ms, N = 21 row kernel at
    // 4.4 M rows ~15 % slower (its far neighbours miss L2, which the (z, y, x) band keeps resident) -- so off.
    if (!topo->lo_perm.empty() && !(topo->dia_ng > 0 && topo->dia_lo == 1)) {
        const char* env = std::getenv("KSB_LO_MORTON");
        if (env && env[0] == '1') {
            morton_order(m.xyz.data(), S.interior.data(), ni, topo->lo_perm);
            build_lo();
        }
    }

    // union-tile view of the ordered pattern (wide blocks; topology.hpp)
    if (!topo->lo_perm.empty() && topo->lo_max_row <= kUtE) build_union_tiles(*topo, m.xyz.data(), S.interior.data(), ni);

    // fine tets grouped by coarse ancestor
    topo->ancestor = h.ancestor(level);
    const int nct = h.mesh(0).n_tets();
    topo->anc_ptr.assign(size_t(nct) + 1, 0);
    for (int t = 0; t < nt; ++t) ++topo->anc_ptr[topo->ancestor[t] + 1];
    for (int c = 0; c < nct; ++c) topo->anc_ptr[c + 1] += topo->anc_ptr[c];
    topo->anc_tets.resize(nt);
    {
        std::vector<int32_t> fill(topo->anc_ptr.begin(), topo->anc_ptr.end() - 1);
        for (int t = 0; t < nt; ++t) topo->anc_tets[fill[topo->ancestor[t]]++] = t;
    }
    }  // !lite
    if (level > 0) {
        // rows in creation order (parents precede children), accumulated like the reference's per-row map:
        // 0 + 0.5 w over the first parent's entries, then the second's; stored in ascending column order
        const Mesh& pm = h.mesh(level - 1);
        topo->n_prev = pm.n_vertices();
        topo->prev_iidx = Space(h.mesh_ptr(level - 1)).iidx;
        const int npv = m.n_parent_vertices;
        if (npv != topo->n_prev) raise(KSB_HIERARCHY, "levels are not nested");
        topo->pstep_col.assign(size_t(nv) * 4, -1);
        topo->pstep_val.assign(size_t(nv) * 4, 0.0);
        for (int v = 0; v < nv; ++v) {
            int32_t* pc = &topo->pstep_col[size_t(v) * 4];
            double* pv = &topo->pstep_val[size_t(v) * 4];
            if (v < npv) {
                pc[0] = v;
                pv[0] = 1.0;
                continue;
            }
            int32_t cc[8];
            double cv[8];
            int w = 0;
            for (int side = 0; side < 2; ++side) {
                const int32_t par = m.vparent[2 * size_t(v) + side];
                if (par >= v) raise(KSB_INTERNAL, "vertex parent created after its child");
                const int32_t* qc = &topo->pstep_col[size_t(par) * 4];
                const double* qv = &topo->pstep_val[size_t(par) * 4];
                for (int k = 0; k < 4 && qc[k] >= 0; ++k) {
                    int j = 0;
                    while (j < w && cc[j] != qc[k]) ++j;
                    if (j == w) {
                        cc[w] = qc[k];
                        cv[w++] = 0.0;
                    }
                    cv[j] += 0.5 * qv[k];
                }
            }
            if (w > 4) raise(KSB_INTERNAL, "prolongation row wider than 4");
            for (int i = 1; i < w; ++i)  // insertion sort by column
                for (int j = i; j > 0 && cc[j - 1] > cc[j]; --j) {
                    std::swap(cc[j - 1], cc[j]);
                    std::swap(cv[j - 1], cv[j]);
                }
            for (int k = 0; k < w; ++k) {
                pc[k] = cc[k];
                pv[k] = cv[k];
            }
        }
    }
    return topo;
}

int64_t dorfler_mark(const double* eta, int64_t nt, double total_sq, double theta, int32_t* marked) {
    std::vector<int32_t> order(static_cast<size_t>(nt));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nt; ++i) order[size_t(i)] = int32_t(i);
    __gnu_parallel::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
        if (eta[a] != eta[b]) return eta[a] > eta[b];
        return a < b;
    });
    double acc = 0.0;
    int64_t k = 0;
    for (int32_t t : order) {
        marked[k++] = t;
        acc += eta[t];
        if (acc >= theta * total_sq) break;
    }
    return k;
}

ProjChunks build_proj_chunks(const FineTopology& T) {
    const Mesh& m = *T.space->mesh;
    const int nct = int(T.anc_ptr.size()) - 1;
    struct Local {
        std::vector<int32_t> ch_t, ch_v, ch_e, tets, verts, edges, vcnt, vinc, ecnt, einc;
    };
    std::vector<Local> loc(size_t(std::max(nct, 0)));
#pragma omp parallel
    {
    std::vector<int32_t> stamp(size_t(m.n_vertices()), -1);
    int32_t stamp_id = 0;
#pragma omp for schedule(dynamic, 4)
    for (int C = 0; C < nct; ++C) {
        Local& L = loc[size_t(C)];
        const int b = T.anc_ptr[size_t(C)], e = T.anc_ptr[size_t(C) + 1];
        // Morton order of the centroids inside the coarse tet's bounding box
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        std::vector<std::pair<uint64_t, int32_t>> key(size_t(e - b));
        std::vector<double> cen(size_t(e - b) * 3);
        for (int p = b; p < e; ++p) {
            const int t = T.anc_tets[size_t(p)];
            for (int d = 0; d < 3; ++d) {
                double c = 0.0;
                for (int k = 0; k < 4; ++k) c += m.xyz[3 * size_t(m.tets[4 * size_t(t) + k]) + d];
                c *= 0.25;
                cen[3 * size_t(p - b) + d] = c;
                lo[d] = std::min(lo[d], c);
                hi[d] = std::max(hi[d], c);
            }
        }
        for (int p = b; p < e; ++p) {
            uint64_t code = 0;
            uint32_t q[3];
            for (int d = 0; d < 3; ++d) {
                const double span = hi[d] > lo[d] ? hi[d] - lo[d] : 1.0;
                q[d] = uint32_t(std::min(2097151.0, (cen[3 * size_t(p - b) + d] - lo[d]) / span * 2097151.0));
            }
            for (int bit = 20; bit >= 0; --bit)
                for (int d = 2; d >= 0; --d) code = (code << 1) | ((q[d] >> bit) & 1u);
            key[size_t(p - b)] = {code, T.anc_tets[size_t(p)]};
        }
        std::sort(key.begin(), key.end());
        // one chunk from key[lo, hi): sorted vertices, sorted local edges, incidences in ascending tet order; halved
        // while it has more than kPgE edges
        std::function<void(size_t, size_t)> emit = [&](size_t lo, size_t hi) {
            std::vector<int32_t> vs;
            vs.reserve((hi - lo) * 4);
            for (size_t k = lo; k < hi; ++k)
                for (int c = 0; c < 4; ++c) vs.push_back(m.tets[4 * size_t(key[k].second) + c]);
            std::sort(vs.begin(), vs.end());
            vs.erase(std::unique(vs.begin(), vs.end()), vs.end());
            auto lidx = [&](int32_t v) { return int32_t(std::lower_bound(vs.begin(), vs.end(), v) - vs.begin()); };
            std::vector<std::pair<int32_t, int32_t>> le;
            le.reserve((hi - lo) * 6);
            for (size_t k = lo; k < hi; ++k) {
                const int32_t* tv = &m.tets[4 * size_t(key[k].second)];
                for (int c = 0; c < 4; ++c)
                    for (int d = c + 1; d < 4; ++d) {
                        const int32_t a = lidx(tv[c]), bb = lidx(tv[d]);
                        le.push_back({std::min(a, bb), std::max(a, bb)});
                    }
            }
            std::sort(le.begin(), le.end());
            le.erase(std::unique(le.begin(), le.end()), le.end());
            if (int(le.size()) > kPgE && hi - lo > 1) {
                const size_t mid = lo + (hi - lo) / 2;
                emit(lo, mid);
                emit(mid, hi);
                return;
            }
            L.ch_t.push_back(int32_t(L.tets.size()));
            L.ch_v.push_back(int32_t(L.verts.size()));
            L.ch_e.push_back(int32_t(L.edges.size()));
            std::vector<std::vector<int32_t>> vi(vs.size()), ei(le.size());
            for (size_t k = lo; k < hi; ++k) {
                const int32_t tl = int32_t(k - lo);
                const int32_t* tv = &m.tets[4 * size_t(key[k].second)];
                for (int c = 0; c < 4; ++c) vi[size_t(lidx(tv[c]))].push_back(tl << 2 | c);
                for (int c = 0; c < 4; ++c)
                    for (int d = c + 1; d < 4; ++d) {
                        const int32_t a = lidx(tv[c]), bb = lidx(tv[d]);
                        const auto pr = std::make_pair(std::min(a, bb), std::max(a, bb));
                        ei[size_t(std::lower_bound(le.begin(), le.end(), pr) - le.begin())].push_back(tl << 4 | c << 2 | d);
                    }
                L.tets.push_back(key[k].second);
            }
            for (size_t k = 0; k < vs.size(); ++k) {
                L.verts.push_back(vs[k]);
                L.vcnt.push_back(int32_t(vi[k].size()));
                L.vinc.insert(L.vinc.end(), vi[k].begin(), vi[k].end());
            }
            for (size_t k = 0; k < le.size(); ++k) {
                L.edges.push_back(le[k].first | le[k].second << 16);
                L.ecnt.push_back(int32_t(ei[k].size()));
                L.einc.insert(L.einc.end(), ei[k].begin(), ei[k].end());
            }
        };
        // greedy compact chunks: <= kPgT tets and <= kPgV vertices (vertex membership by a per-thread stamp)
        size_t i = 0;
        while (i < key.size()) {
            ++stamp_id;
            const size_t start = i;
            int nvc = 0;
            for (; i < key.size() && i - start < size_t(kPgT); ++i) {
                const int32_t* tv = &m.tets[4 * size_t(key[i].second)];
                int add = 0;
                for (int c = 0; c < 4; ++c) {
                    bool dup = stamp[size_t(tv[c])] == stamp_id;
                    for (int d = 0; d < c && !dup; ++d) dup = tv[d] == tv[c];
                    add += !dup;
                }
                if (i > start && nvc + add > kPgV) break;
                for (int c = 0; c < 4; ++c) stamp[size_t(tv[c])] = stamp_id;
                nvc += add;
            }
            emit(start, i);
        }
    }
    }  // omp parallel
    // concatenate in coarse-tet order
    ProjChunks P;
    P.cptr.assign(size_t(std::max(nct, 0)) + 1, 0);
    P.vinc_ptr.push_back(0);
    P.einc_ptr.push_back(0);
    for (int C = 0; C < nct; ++C) {
        const Local& L = loc[size_t(C)];
        const int nch = int(L.ch_t.size());
        const int t0 = int(P.tets.size()), v0 = int(P.verts.size()), e0 = int(P.edges.size());
        const int chbase = int(P.ch_t.size());
        P.cptr[size_t(C)] = int32_t(P.item_c.size());
        for (int q = 0; q < nch; q += kPgItem) {
            P.item_c.push_back(C);
            P.item_ch.push_back(chbase + q);
        }
        for (int q = 0; q < nch; ++q) {
            P.ch_t.push_back(t0 + L.ch_t[size_t(q)]);
            P.ch_v.push_back(v0 + L.ch_v[size_t(q)]);
            P.ch_e.push_back(e0 + L.ch_e[size_t(q)]);
        }
        P.tets.insert(P.tets.end(), L.tets.begin(), L.tets.end());
        P.verts.insert(P.verts.end(), L.verts.begin(), L.verts.end());
        P.edges.insert(P.edges.end(), L.edges.begin(), L.edges.end());
        for (int32_t c : L.vcnt) P.vinc_ptr.push_back(P.vinc_ptr.back() + c);
        for (int32_t c : L.ecnt) P.einc_ptr.push_back(P.einc_ptr.back() + c);
        P.vinc.insert(P.vinc.end(), L.vinc.begin(), L.vinc.end());
        P.einc.insert(P.einc.end(), L.einc.begin(), L.einc.end());
        check_i32(int64_t(P.einc.size()), "projection chunk incidences");
    }
    if (nct >= 0) P.cptr[size_t(std::max(nct, 0))] = int32_t(P.item_c.size());
    P.item_ch.push_back(int32_t(P.ch_t.size()));
    P.ch_t.push_back(int32_t(P.tets.size()));
    P.ch_v.push_back(int32_t(P.verts.size()));
    P.ch_e.push_back(int32_t(P.edges.size()));
    return P;
}

} // namespace ksb
