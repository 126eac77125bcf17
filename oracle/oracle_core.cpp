// CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle_core.hpp header).
#include "oracle_core.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <map>
#include <numeric>
#include <unordered_map>

namespace orc {

void fail(int code, const std::string& what) { throw OrcError(code, what); }

namespace {
constexpr double kPi = 3.14159265358979323846;
inline V3 sub(const V3& a, const V3& b) { return V3{{a[0] - b[0], a[1] - b[1], a[2] - b[2]}}; }
inline V3 cross(const V3& a, const V3& b) {
    return V3{{a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]}};
}
inline double dot3(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline double nrm3(const V3& a) { return std::sqrt(dot3(a, a)); }
double signed_vol(const V3& a, const V3& b, const V3& c, const V3& d) {
    return dot3(cross(sub(b, a), sub(c, a)), sub(d, a)) / 6.0;
}
double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
}  // namespace

// =========================================================== mesh (proj/src/mesh.cpp)
double Mesh::tet_volume(int t) const {
    const auto& v = tets[t];
    return signed_vol(verts[v[0]], verts[v[1]], verts[v[2]], verts[v[3]]);
}

// proj/src/mesh.cpp:175-218 -- faces in sorted-key order, owners in tet order
void Mesh::finalize() {
    bfaces.clear();
    ifaces.clear();
    iface_tets.clear();
    on_boundary.assign(verts.size(), 0);
    struct FK {
        std::array<int, 3> k;
        int t;
    };
    std::vector<FK> all;
    all.reserve(size_t(nt()) * 4);
    const int loc[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
    for (int t = 0; t < nt(); ++t)
        for (const auto& f : loc) {
            std::array<int, 3> k{tets[t][f[0]], tets[t][f[1]], tets[t][f[2]]};
            std::sort(k.begin(), k.end());
            all.push_back({k, t});
        }
    std::stable_sort(all.begin(), all.end(), [](const FK& a, const FK& b) { return a.k < b.k; });
    for (size_t i = 0; i < all.size();) {
        size_t j = i + 1;
        while (j < all.size() && all[j].k == all[i].k) ++j;
        const auto& k = all[i].k;
        if (j - i == 1) {
            bfaces.push_back(k);
            for (int v : k) on_boundary[v] = 1;
        } else if (j - i == 2) {
            ifaces.push_back(k);
            iface_tets.push_back({std::min(all[i].t, all[i + 1].t), std::max(all[i].t, all[i + 1].t)});
        } else {
            fail(E_INTERNAL, "face shared by more than two tets");
        }
        i = j;
    }
}

bool Mesh::conforming(std::string* why) const {
    auto no = [&](const std::string& s) {
        if (why) *why = s;
        return false;
    };
    for (int t = 0; t < nt(); ++t)
        if (tet_volume(t) <= 0) return no("non-positive volume");
    std::map<std::array<int, 3>, int> cnt;
    const int loc[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
    for (int t = 0; t < nt(); ++t)
        for (const auto& f : loc) {
            std::array<int, 3> k{tets[t][f[0]], tets[t][f[1]], tets[t][f[2]]};
            std::sort(k.begin(), k.end());
            ++cnt[k];
        }
    double ext = 0;
    for (int d = 0; d < 3; ++d) ext = std::max(ext, hi[d] - lo[d]);
    const double eps = 1e-9 * ext;
    for (const auto& [k, c] : cnt) {
        if (c > 2) return no("face with more than two owners");
        if (c == 1) {
            bool on = false;
            for (int ax = 0; ax < 3 && !on; ++ax)
                for (double side : {lo[ax], hi[ax]}) {
                    bool all = true;
                    for (int v : k) all = all && std::abs(verts[v][ax] - side) <= eps;
                    if (all) on = true;
                }
            if (!on) return no("hanging face");
        }
    }
    return true;
}

namespace {
// proj/src/mesh.cpp:25-120 -- tagged (Maubach) bisection work list
struct Refiner {
    const Mesh& in;
    std::vector<V3> verts;
    std::vector<std::array<int, 2>> vpar;
    struct W {
        std::array<int, 4> t;
        int8_t tag;
        int root;
        bool alive;
    };
    std::vector<W> work;
    std::unordered_map<uint64_t, int> mid;
    static uint64_t key(int a, int b) {
        if (a > b) std::swap(a, b);
        return (uint64_t(a) << 32) | uint32_t(b);
    }
    explicit Refiner(const Mesh& m) : in(m), verts(m.verts), vpar(m.vparent) {
        for (int t = 0; t < m.nt(); ++t) work.push_back({m.tuple[t], m.tag[t], t, true});
    }
    int midpoint(int a, int b) {
        auto it = mid.find(key(a, b));
        if (it != mid.end()) return it->second;
        const int v = int(verts.size());
        V3 p;
        for (int d = 0; d < 3; ++d) p[d] = 0.5 * (verts[a][d] + verts[b][d]);
        verts.push_back(p);
        vpar.push_back({std::min(a, b), std::max(a, b)});
        mid.emplace(key(a, b), v);
        return v;
    }
    void bisect(int t) {
        const auto tup = work[t].t;
        const int d = work[t].tag;
        const int z = midpoint(tup[0], tup[d]);
        const int8_t ct = d > 1 ? int8_t(d - 1) : int8_t(3);
        std::array<int, 4> c1 = tup;
        c1[d] = z;
        std::array<int, 4> c2;
        int w = 0;
        for (int j = 1; j <= d; ++j) c2[w++] = tup[j];
        c2[w++] = z;
        for (int j = d + 1; j < 4; ++j) c2[w++] = tup[j];
        work[t].alive = false;
        work.push_back({c1, ct, work[t].root, true});
        work.push_back({c2, ct, work[t].root, true});
    }
    bool broken(const W& w) const {
        for (int i = 0; i < 4; ++i)
            for (int j = i + 1; j < 4; ++j)
                if (mid.count(key(w.t[i], w.t[j]))) return true;
        return false;
    }
    void close() {
        for (int pass = 0; pass < 200; ++pass) {
            bool changed = false;
            for (size_t t = 0; t < work.size(); ++t) {
                if (!work[t].alive) continue;
                if (broken(work[t])) {
                    bisect(int(t));
                    changed = true;
                }
            }
            if (!changed) return;
        }
        fail(E_INTERNAL, "conforming closure did not terminate");
    }
    MeshP build() const {
        auto out = std::make_shared<Mesh>();
        out->verts = verts;
        out->vparent = vpar;
        out->n_parent_vertices = in.nv();
        out->level = in.level + 1;
        out->lo = in.lo;
        out->hi = in.hi;
        for (const auto& w : work) {
            if (!w.alive) continue;
            auto t = w.t;
            if (signed_vol(verts[t[0]], verts[t[1]], verts[t[2]], verts[t[3]]) < 0) std::swap(t[2], t[3]);
            out->tets.push_back(t);
            out->tuple.push_back(w.t);
            out->tag.push_back(w.tag);
            out->parent.push_back(w.root);
        }
        out->finalize();
        return out;
    }
};
}  // namespace

// proj/src/mesh.cpp:281-331
MeshP box_mesh(const V3& lo, const V3& hi, int n) {
    for (int d = 0; d < 3; ++d)
        if (!(hi[d] > lo[d])) fail(E_DOMAIN, "box is degenerate");
    if (n < 1) fail(E_DOMAIN, "n_per_axis must be >= 1");
    auto m = std::make_shared<Mesh>();
    m->lo = lo;
    m->hi = hi;
    const int nv = n + 1;
    auto vid = [&](int i, int j, int k) { return (i * nv + j) * nv + k; };
    for (int i = 0; i < nv; ++i)
        for (int j = 0; j < nv; ++j)
            for (int k = 0; k < nv; ++k) {
                V3 p;
                p[0] = lo[0] + (hi[0] - lo[0]) * double(i) / n;
                p[1] = lo[1] + (hi[1] - lo[1]) * double(j) / n;
                p[2] = lo[2] + (hi[2] - lo[2]) * double(k) / n;
                m->verts.push_back(p);
            }
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < n; ++k)
                for (const auto& pm : perms) {
                    std::array<int, 3> c{i, j, k};
                    std::array<int, 4> t;
                    t[0] = vid(c[0], c[1], c[2]);
                    for (int s = 0; s < 3; ++s) {
                        ++c[pm[s]];
                        t[s + 1] = vid(c[0], c[1], c[2]);
                    }
                    m->tuple.push_back(t);
                    if (signed_vol(m->verts[t[0]], m->verts[t[1]], m->verts[t[2]], m->verts[t[3]]) < 0)
                        std::swap(t[2], t[3]);
                    m->tets.push_back(t);
                    m->tag.push_back(3);
                }
    m->parent.resize(m->tets.size());
    std::iota(m->parent.begin(), m->parent.end(), 0);
    for (int v = 0; v < m->nv(); ++v) m->vparent.push_back({v, v});
    m->n_parent_vertices = m->nv();
    m->finalize();
    return m;
}

// proj/src/mesh.cpp:333-343
MeshP uniform_refine(const Mesh& in) {
    Refiner r(in);
    for (int round = 0; round < 3; ++round) {
        const size_t cnt = r.work.size();
        for (size_t t = 0; t < cnt; ++t)
            if (r.work[t].alive) r.bisect(int(t));
    }
    return r.build();
}

// proj/src/mesh.cpp:345-368
MeshP adapt_refine(const Mesh& in, std::vector<int> marked) {
    for (int t : marked)
        if (t < 0 || t >= in.nt()) fail(E_ARG, "marked tet out of range");
    if (marked.empty()) {
        auto out = std::make_shared<Mesh>(in);
        out->level = in.level + 1;
        out->n_parent_vertices = in.nv();
        for (int v = 0; v < out->nv(); ++v) out->vparent[v] = {v, v};
        for (int t = 0; t < out->nt(); ++t) out->parent[t] = t;
        return out;
    }
    std::sort(marked.begin(), marked.end());
    marked.erase(std::unique(marked.begin(), marked.end()), marked.end());
    Refiner r(in);
    for (int t : marked) r.bisect(t);
    r.close();
    return r.build();
}

// =========================================================== sparse
Csc Csc::from_triplets(int rows, int cols, const std::vector<Trip>& t) {
    // Eigen setFromTriplets: duplicates summed in insertion order, rows sorted per column
    Csc A;
    A.rows = rows;
    A.cols = cols;
    std::vector<int> cnt(size_t(cols) + 1, 0);
    for (const auto& x : t) ++cnt[x.c + 1];
    for (int c = 0; c < cols; ++c) cnt[c + 1] += cnt[c];
    std::vector<int> order(t.size());
    {
        std::vector<int> fill(cnt.begin(), cnt.end() - 1);
        for (size_t i = 0; i < t.size(); ++i) order[fill[t[i].c]++] = int(i);
    }
    A.ptr.assign(size_t(cols) + 1, 0);
    std::vector<std::vector<std::pair<int, double>>> colv(cols);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int c = 0; c < cols; ++c) {
        // stable by row keeps insertion order among duplicates
        std::vector<int> ids(order.begin() + cnt[c], order.begin() + cnt[c + 1]);
        std::stable_sort(ids.begin(), ids.end(), [&](int a, int b) { return t[a].r < t[b].r; });
        auto& out = colv[c];
        for (size_t i = 0; i < ids.size();) {
            size_t j = i;
            double v = t[ids[i]].v;
            while (++j < ids.size() && t[ids[j]].r == t[ids[i]].r) v += t[ids[j]].v;
            out.push_back({t[ids[i]].r, v});
            i = j;
        }
    }
    for (int c = 0; c < cols; ++c) A.ptr[c + 1] = A.ptr[c] + int(colv[c].size());
    A.idx.resize(A.ptr.back());
    A.val.resize(A.ptr.back());
    for (int c = 0; c < cols; ++c)
        for (size_t k = 0; k < colv[c].size(); ++k) {
            A.idx[A.ptr[c] + k] = colv[c][k].first;
            A.val[A.ptr[c] + k] = colv[c][k].second;
        }
    return A;
}

double Csc::coeff(int r, int c) const {
    for (int k = ptr[c]; k < ptr[c + 1]; ++k)
        if (idx[k] == r) return val[k];
    return 0.0;
}

Vec Csc::mul(const Vec& x) const {
    Vec y(rows, 0.0);
    for (int c = 0; c < cols; ++c) {
        const double xc = x[c];
        for (int k = ptr[c]; k < ptr[c + 1]; ++k) y[idx[k]] += val[k] * xc;
    }
    return y;
}

Csc Csc::transpose() const {
    std::vector<Trip> t;
    t.reserve(val.size());
    for (int c = 0; c < cols; ++c)
        for (int k = ptr[c]; k < ptr[c + 1]; ++k) t.push_back({c, idx[k], val[k]});
    return from_triplets(cols, rows, t);
}

Csc add(const Csc& a, double s, const Csc& b) {
    std::vector<Trip> t;
    t.reserve(a.val.size() + b.val.size());
    for (int c = 0; c < a.cols; ++c) {
        // merge column c (sorted rows) so sums are a + s*b per entry
        int i = a.ptr[c], j = b.ptr[c];
        while (i < a.ptr[c + 1] || j < b.ptr[c + 1]) {
            if (j >= b.ptr[c + 1] || (i < a.ptr[c + 1] && a.idx[i] < b.idx[j])) {
                t.push_back({a.idx[i], c, a.val[i]});
                ++i;
            } else if (i >= a.ptr[c + 1] || b.idx[j] < a.idx[i]) {
                t.push_back({b.idx[j], c, s * b.val[j]});
                ++j;
            } else {
                t.push_back({a.idx[i], c, a.val[i] + s * b.val[j]});
                ++i;
                ++j;
            }
        }
    }
    return Csc::from_triplets(a.rows, a.cols, t);
}

Csc scale(const Csc& a, double s) {
    Csc r = a;
    for (double& v : r.val) v *= s;
    return r;
}

Csc matmul(const Csc& a, const Csc& b) {
    // Gustavson, column by column of b
    std::vector<Trip> t;
    Vec acc(a.rows, 0.0);
    std::vector<int> mark(a.rows, -1), rows;
    for (int c = 0; c < b.cols; ++c) {
        rows.clear();
        for (int k = b.ptr[c]; k < b.ptr[c + 1]; ++k) {
            const int j = b.idx[k];
            const double bv = b.val[k];
            for (int q = a.ptr[j]; q < a.ptr[j + 1]; ++q) {
                const int r = a.idx[q];
                if (mark[r] != c) {
                    mark[r] = c;
                    acc[r] = 0.0;
                    rows.push_back(r);
                }
                acc[r] += a.val[q] * bv;
            }
        }
        std::sort(rows.begin(), rows.end());
        for (int r : rows) t.push_back({r, c, acc[r]});
    }
    return Csc::from_triplets(a.rows, b.cols, t);
}

double dot(const Vec& a, const Vec& b) {
    double s = 0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}
double norm2(const Vec& a) { return std::sqrt(dot(a, a)); }

// =========================================================== spaces (proj/src/fespace.cpp)
Space::Space(MeshP m) : mesh(std::move(m)) {
    iidx.assign(mesh->nv(), -1);
    for (int v = 0; v < mesh->nv(); ++v) {
        if (mesh->on_boundary[v]) {
            boundary.push_back(v);
        } else {
            iidx[v] = int(interior.size());
            interior.push_back(v);
        }
    }
}

// proj/src/fespace.cpp:35-56
Csc prolongation_step(const Mesh& fine) {
    const int nc = fine.n_parent_vertices, nf = fine.nv();
    std::vector<std::map<int, double>> rows(nf);
    for (int v = 0; v < nf; ++v) {
        if (v < nc) {
            rows[v][v] = 1.0;
        } else {
            const auto [a, b] = fine.vparent[v];
            for (const auto& [c, w] : rows[a]) rows[v][c] += 0.5 * w;
            for (const auto& [c, w] : rows[b]) rows[v][c] += 0.5 * w;
        }
    }
    std::vector<Trip> t;
    for (int v = 0; v < nf; ++v)
        for (const auto& [c, w] : rows[v]) t.push_back({v, c, w});
    return Csc::from_triplets(nf, nc, t);
}

void Hier::push(MeshP m) {
    if (!spaces.empty()) steps.push_back(prolongation_step(*m));
    spaces.push_back(std::make_shared<Space>(std::move(m)));
}

// proj/src/fespace.cpp:64-74
Csc Hier::prolongation(int from, int to) const {
    if (from > to || to >= int(spaces.size())) fail(E_HIER, "levels are not nested");
    if (from == to) {
        std::vector<Trip> t;
        for (int i = 0; i < spaces[from]->n(); ++i) t.push_back({i, i, 1.0});
        return Csc::from_triplets(spaces[from]->n(), spaces[from]->n(), t);
    }
    Csc P = steps[from];
    for (int k = from + 1; k < to; ++k) P = matmul(steps[k], P);
    return P;
}

Vec Hier::prolong(const Vec& c, int from, int to) const {
    Vec x = c;
    for (int k = from; k < to; ++k) x = steps[k].mul(x);
    return x;
}

// =========================================================== quadrature (proj/src/quadrature.cpp:9-49)
const std::vector<QP>& keast() {
    static const std::vector<QP> rule = [] {
        std::vector<QP> r;
        const double w0 = -444.0 / 5625.0, w1 = 6.0 * 343.0 / 45000.0, w2 = 6.0 * 56.0 / 2250.0;
        const double a = 1.0 / 14.0;
        const double b1 = 0.25 * (1.0 + std::sqrt(5.0 / 14.0)), b2 = 0.25 * (1.0 - std::sqrt(5.0 / 14.0));
        r.push_back({{0.25, 0.25, 0.25, 0.25}, w0});
        for (int k = 0; k < 4; ++k) {
            QP q{{a, a, a, a}, w1};
            q.b[k] = 1.0 - 3.0 * a;
            r.push_back(q);
        }
        const int pr[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
        for (const auto& p : pr) {
            QP q{{b2, b2, b2, b2}, w2};
            q.b[p[0]] = b1;
            q.b[p[1]] = b1;
            r.push_back(q);
        }
        return r;
    }();
    return rule;
}

// =========================================================== assembly (proj/src/assembly.cpp)
Geo tet_geo(const Mesh& m, int t) {
    Geo g;
    for (int i = 0; i < 4; ++i) g.x[i] = m.verts[m.tets[t][i]];
    const V3 c0 = sub(g.x[1], g.x[0]), c1 = sub(g.x[2], g.x[0]), c2 = sub(g.x[3], g.x[0]);
    const V3 r0 = cross(c1, c2), r1 = cross(c2, c0), r2 = cross(c0, c1);
    const double det = dot3(c0, r0);
    g.vol = std::abs(det) / 6.0;
    const V3 rr[3] = {r0, r1, r2};
    for (int k = 0; k < 3; ++k)
        for (int d = 0; d < 3; ++d) g.g[k + 1][d] = rr[k][d] / det;
    for (int d = 0; d < 3; ++d) g.g[0][d] = -(g.g[1][d] + g.g[2][d] + g.g[3][d]);
    return g;
}

namespace {
constexpr int kChunks = 64;  // proj/src/assembly.cpp:11

template <class PerTet>
Csc assemble_matrix(const Space& V, PerTet&& per_tet) {
    const Mesh& m = *V.mesh;
    const int nt = m.nt();
    const int nc = std::clamp(nt, 1, kChunks);
    std::vector<std::vector<Trip>> ch(nc);
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < nc; ++c) {
        const int lo = int(int64_t(nt) * c / nc), hi = int(int64_t(nt) * (c + 1) / nc);
        ch[c].reserve(size_t(hi - lo) * 16);
        double K[4][4];
        for (int t = lo; t < hi; ++t) {
            per_tet(t, K);
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j) ch[c].push_back({m.tets[t][i], m.tets[t][j], K[i][j]});
        }
    }
    std::vector<Trip> all;
    size_t tot = 0;
    for (auto& c : ch) tot += c.size();
    all.reserve(tot);
    for (auto& c : ch) {
        all.insert(all.end(), c.begin(), c.end());
        std::vector<Trip>().swap(c);
    }
    m.quad_cells += nt;
    return Csc::from_triplets(V.n(), V.n(), all);
}

template <class WeightAt>
Csc weighted_mass(const Space& V, WeightAt&& wat) {
    const Mesh& m = *V.mesh;
    const auto& rule = keast();
    return assemble_matrix(V, [&](int t, double (&K)[4][4]) {
        const Geo g = tet_geo(m, t);
        for (auto& row : K)
            for (double& x : row) x = 0.0;
        for (const auto& q : rule) {
            const double w = wat(t, g, q.b);
            if (!std::isfinite(w)) fail(E_SINGULAR, "weight is not finite at a quadrature point");
            const double s = q.w * g.vol * w;
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j) K[i][j] += s * q.b[i] * q.b[j];
        }
    });
}
}  // namespace

Csc assemble_stiffness(const Space& V) {
    const Mesh& m = *V.mesh;
    return assemble_matrix(V, [&](int t, double (&K)[4][4]) {
        const Geo g = tet_geo(m, t);
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j)
                K[i][j] = g.vol * (g.g[i][0] * g.g[j][0] + g.g[i][1] * g.g[j][1] + g.g[i][2] * g.g[j][2]);
    });
}

Csc assemble_mass(const Space& V) {
    return weighted_mass(V, [](int, const Geo&, const double*) { return 1.0; });
}

Csc assemble_mass_nodal(const Space& V, const Vec& w) {
    const Mesh& m = *V.mesh;
    return weighted_mass(V, [&](int t, const Geo&, const double* b) {
        const auto& v = m.tets[t];
        return b[0] * w[v[0]] + b[1] * w[v[1]] + b[2] * w[v[2]] + b[3] * w[v[3]];
    });
}

double Potential::operator()(const V3& x) const {
    double v = 0;
    if (kind == 0) {
        for (size_t k = 0; k + 3 < p.size(); k += 4) {
            const double dx = x[0] - p[k + 1], dy = x[1] - p[k + 2], dz = x[2] - p[k + 3];
            double r = std::sqrt(dx * dx + dy * dy + dz * dz);
            if (r < 1e-12) r = 1e-10;
            v -= p[k] / r;
        }
    } else {
        for (size_t k = 0; k + 4 < p.size(); k += 5) {
            const double dx = x[0] - p[k + 2], dy = x[1] - p[k + 3], dz = x[2] - p[k + 4];
            v -= p[k] * std::exp(-(dx * dx + dy * dy + dz * dz) / (2.0 * p[k + 1] * p[k + 1]));
        }
    }
    return v;
}

Csc assemble_mass_pot(const Space& V, const Potential& pot) {
    return weighted_mass(V, [&](int, const Geo& g, const double* b) {
        V3 x;
        for (int d = 0; d < 3; ++d) x[d] = b[0] * g.x[0][d] + b[1] * g.x[1][d] + b[2] * g.x[2][d] + b[3] * g.x[3][d];
        return pot(x);
    });
}

// proj/src/assembly.cpp:181-220 (serial chunk order, per-chunk vectors summed in chunk order)
Vec load_nodal(const Space& V, const Vec& f) {
    const Mesh& m = *V.mesh;
    const auto& rule = keast();
    const int nt = m.nt();
    const int nc = std::clamp(nt, 1, kChunks);
    std::vector<Vec> ch(nc, Vec(V.n(), 0.0));
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < nc; ++c) {
        const int lo = int(int64_t(nt) * c / nc), hi = int(int64_t(nt) * (c + 1) / nc);
        for (int t = lo; t < hi; ++t) {
            const Geo g = tet_geo(m, t);
            const auto& v = m.tets[t];
            for (const auto& q : rule) {
                const double fq = q.b[0] * f[v[0]] + q.b[1] * f[v[1]] + q.b[2] * f[v[2]] + q.b[3] * f[v[3]];
                const double s = q.w * g.vol * fq;
                for (int i = 0; i < 4; ++i) ch[c][v[i]] += s * q.b[i];
            }
        }
    }
    Vec b(V.n(), 0.0);
    for (const auto& c : ch)
        for (int i = 0; i < V.n(); ++i) b[i] += c[i];
    return b;
}

// proj/src/assembly.cpp:251-287
double l2_norm(const Space& V, const Vec& f) {
    const Mesh& m = *V.mesh;
    double s = 0;
    for (int t = 0; t < m.nt(); ++t) {
        const auto& v = m.tets[t];
        const double vol = std::abs(m.tet_volume(t));
        double sum = 0, sq = 0;
        for (int i = 0; i < 4; ++i) {
            sum += f[v[i]];
            sq += f[v[i]] * f[v[i]];
        }
        s += vol * (sum * sum + sq) / 20.0;
    }
    return std::sqrt(std::max(0.0, s));
}

double h1_seminorm(const Space& V, const Vec& f) {
    const Mesh& m = *V.mesh;
    double s = 0;
    for (int t = 0; t < m.nt(); ++t) {
        const Geo g = tet_geo(m, t);
        const auto& v = m.tets[t];
        double gr[3] = {0, 0, 0};
        for (int i = 0; i < 4; ++i)
            for (int d = 0; d < 3; ++d) gr[d] += f[v[i]] * g.g[i][d];
        s += g.vol * (gr[0] * gr[0] + gr[1] * gr[1] + gr[2] * gr[2]);
    }
    return std::sqrt(std::max(0.0, s));
}

double h1_norm(const Space& V, const Vec& f) {
    const double a = l2_norm(V, f), b = h1_seminorm(V, f);
    return std::sqrt(a * a + b * b);
}

// proj/src/assembly.cpp:234-249 (integrate_of) with g = |v|, proj/src/assembly.cpp:289-291 (l1_norm)
double l1_norm(const Space& V, const Vec& f) {
    const Mesh& m = *V.mesh;
    const auto& rule = keast();
    double s = 0;
    for (int t = 0; t < m.nt(); ++t) {
        const Geo g = tet_geo(m, t);
        const auto& v = m.tets[t];
        for (const auto& q : rule) {
            const double val = q.b[0] * f[v[0]] + q.b[1] * f[v[1]] + q.b[2] * f[v[2]] + q.b[3] * f[v[3]];
            s += q.w * g.vol * std::abs(val);
        }
    }
    return s;
}

// proj/src/assembly.cpp:311-324
Csc interior_block(const Csc& A, const Space& V) {
    std::vector<Trip> t;
    for (int c = 0; c < A.cols; ++c)
        for (int k = A.ptr[c]; k < A.ptr[c + 1]; ++k) {
            const int r = V.iidx[A.idx[k]], cc = V.iidx[c];
            if (r >= 0 && cc >= 0) t.push_back({r, cc, A.val[k]});
        }
    return Csc::from_triplets(V.ni(), V.ni(), t);
}

// =========================================================== solver (proj/src/solver.cpp)
namespace {
Csc gather(const Csc& A, const std::vector<int>& row_of, int nr, const std::vector<int>& col_of, int nc) {
    std::vector<Trip> t;
    for (int c = 0; c < A.cols; ++c)
        for (int k = A.ptr[c]; k < A.ptr[c + 1]; ++k) {
            const int r = row_of[A.idx[k]], cc = col_of[c];
            if (r >= 0 && cc >= 0) t.push_back({r, cc, A.val[k]});
        }
    return Csc::from_triplets(nr, nc, t);
}
}  // namespace

// proj/src/solver.cpp:28-48
Elliptic::Elliptic(const Csc& A, SpaceP Vp, int pre) : V(std::move(Vp)), precond(pre) {
    const int n = V->n(), ni = V->ni();
    if (A.rows != n || A.cols != n) fail(E_MISMATCH, "matrix size does not match space");
    std::vector<int> io(n, -1), bo(n, -1);
    for (int i = 0; i < ni; ++i) io[V->interior[i]] = i;
    for (size_t i = 0; i < V->boundary.size(); ++i) bo[V->boundary[i]] = int(i);
    Aii = gather(A, io, ni, io, ni);
    Aib = gather(A, io, ni, bo, int(V->boundary.size()));
    diag.assign(ni, 1.0);
    min_diag = std::numeric_limits<double>::infinity();
    for (int i = 0; i < ni; ++i) {
        const double d = Aii.coeff(i, i);
        min_diag = std::min(min_diag, d);
        diag[i] = d != 0.0 ? d : 1.0;
    }
    if (ni == 0) min_diag = 0.0;
}

// proj/src/solver.cpp:50-55: z = (D+U)^-1 D (D+L)^-1 r, column-oriented sparse triangular solves
Vec Elliptic::apply_prec(const Vec& r) const {
    const int n = int(r.size());
    if (precond == 1) {
        Vec z(n);
        for (int i = 0; i < n; ++i) z[i] = r[i] / diag[i];
        return z;
    }
    Vec z = r;
    for (int i = 0; i < n; ++i) {  // lower
        double& tmp = z[i];
        if (tmp != 0.0) {
            int k = Aii.ptr[i];
            while (k < Aii.ptr[i + 1] && Aii.idx[k] < i) ++k;
            tmp /= Aii.val[k];
            ++k;
            for (; k < Aii.ptr[i + 1]; ++k) z[Aii.idx[k]] -= tmp * Aii.val[k];
        }
    }
    for (int i = 0; i < n; ++i) z[i] *= diag[i];
    for (int i = n - 1; i >= 0; --i) {  // upper
        if (z[i] != 0.0) {
            int k = Aii.ptr[i];
            while (Aii.idx[k] != i) ++k;
            z[i] /= Aii.val[k];
            const double tmp = z[i];
            for (int q = Aii.ptr[i]; q < Aii.ptr[i + 1] && Aii.idx[q] < i; ++q) z[Aii.idx[q]] -= tmp * Aii.val[q];
        }
    }
    return z;
}

// proj/src/solver.cpp:57-111 (fixed_iterations > 0: benchmark variant without the stopping test)
Vec Elliptic::pcg(const Vec& rhs, double tol, int maxit, SolveStats* st, int fixed) const {
    const int n = int(rhs.size());
    Vec x(n, 0.0);
    const double bnorm = norm2(rhs);
    SolveStats loc;
    if (bnorm == 0.0 && !fixed) {
        loc.converged = true;
        if (st) *st = loc;
        return x;
    }
    Vec r = rhs, z = apply_prec(r), p = z, Ap(n);
    double rz = dot(r, z);
    const int iters = fixed ? fixed : maxit;
    for (int it = 0; it < iters; ++it) {
        Ap = Aii.mul(p);
        const double pAp = dot(p, Ap);
        if (!fixed && !(pAp > 0.0)) {
            loc.breakdown = true;
            loc.iterations = it;
            loc.relres = norm2(r) / bnorm;
            break;
        }
        const double alpha = rz / pAp;
        for (int i = 0; i < n; ++i) {
            x[i] += alpha * p[i];
            r[i] -= alpha * Ap[i];
        }
        double rel = norm2(r) / bnorm;
        if (!fixed && rel <= tol) {
            const Vec Ax = Aii.mul(x);
            for (int i = 0; i < n; ++i) r[i] = rhs[i] - Ax[i];
            rel = norm2(r) / bnorm;
            if (rel <= tol) {
                loc.converged = true;
                loc.iterations = it + 1;
                loc.relres = rel;
                break;
            }
            z = apply_prec(r);
            p = z;
            rz = dot(r, z);
            loc.iterations = it + 1;
            loc.relres = rel;
            continue;
        }
        z = apply_prec(r);
        const double rzn = dot(r, z);
        const double beta = rzn / rz;
        for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        rz = rzn;
        loc.iterations = it + 1;
        loc.relres = rel;
    }
    if (st) *st = loc;
    return x;
}

// proj/src/solver.cpp:113-131
Vec Elliptic::solve(const Vec& b, const Vec& bc, double tol, SolveStats* st) const {
    const int n = V->n(), ni = V->ni();
    const auto& bd = V->boundary;
    Vec xb(bd.size());
    for (size_t i = 0; i < bd.size(); ++i) xb[i] = bc.empty() ? 0.0 : bc[bd[i]];
    Vec rhs(ni);
    for (int i = 0; i < ni; ++i) rhs[i] = b[V->interior[i]];
    if (!xb.empty()) {
        const Vec t = Aib.mul(xb);
        for (int i = 0; i < ni; ++i) rhs[i] -= t[i];
    }
    const Vec xi = pcg(rhs, tol, 20000, st);
    Vec x(n, 0.0);
    for (int i = 0; i < ni; ++i) x[V->interior[i]] = xi[i];
    for (size_t i = 0; i < bd.size(); ++i) x[bd[i]] = xb[i];
    return x;
}

// =========================================================== physics (proj/src/ks_model.cpp)
double v_ext(const System& s, const V3& x) {
    Potential p;
    p.kind = 0;
    p.p = s.atoms;
    return p(x);
}

Vec density(const std::vector<Vec>& orb, double occ) {
    if (orb.empty()) fail(E_ARG, "empty orbital set");
    Vec rho(orb[0].size(), 0.0);
    for (const auto& o : orb)
        for (size_t i = 0; i < rho.size(); ++i) rho[i] += o[i] * o[i];
    for (double& r : rho) r *= occ;
    return rho;
}

namespace {
constexpr double pa = 0.0311, pb = -0.048, pc = 0.0020, pd = -0.0116, pg = -0.1423, pb1 = 1.0529, pb2 = 0.3334;
double eps_c(double rs) {
    if (rs < 1.0) return pa * std::log(rs) + pb + pc * rs * std::log(rs) + pd * rs;
    return pg / (1.0 + pb1 * std::sqrt(rs) + pb2 * rs);
}
double v_c(double rs) {
    if (rs < 1.0)
        return pa * std::log(rs) + (pb - pa / 3.0) + (2.0 / 3.0) * pc * rs * std::log(rs) + (2.0 * pd - pc) / 3.0 * rs;
    const double den = 1.0 + pb1 * std::sqrt(rs) + pb2 * rs;
    return eps_c(rs) * (1.0 + (7.0 / 6.0) * pb1 * std::sqrt(rs) + (4.0 / 3.0) * pb2 * rs) / den;
}
}  // namespace

// proj/src/ks_model.cpp:76-97
double xc_energy_density(const System& s, double rho) {
    if (rho < 0.0) rho = 0.0;
    if (rho == 0.0 || s.xc_kind == 0) return 0.0;
    if (s.xc_kind == 1) return -(9.0 / 8.0) * s.alpha * std::cbrt(3.0 / kPi) * std::pow(rho, 4.0 / 3.0);
    const double ex = -0.75 * std::cbrt(3.0 / kPi) * std::pow(rho, s.p_exch);
    const double rs = std::cbrt(3.0 / (4.0 * kPi * rho));
    return (ex + eps_c(rs)) * rho;
}

double xc_potential(const System& s, double rho) {
    if (rho < 0.0) rho = 0.0;
    if (rho == 0.0 || s.xc_kind == 0) return 0.0;
    if (s.xc_kind == 1) return -1.5 * s.alpha * std::cbrt(3.0 * rho / kPi);
    const double ex = -0.75 * std::cbrt(3.0 / kPi) * std::pow(rho, s.p_exch);
    const double rs = std::cbrt(3.0 / (4.0 * kPi * rho));
    return (1.0 + s.p_exch) * ex + v_c(rs);
}

Vec xc_field(const System& s, const Vec& rho) {
    Vec v(rho.size());
    for (size_t i = 0; i < rho.size(); ++i) v[i] = xc_potential(s, rho[i]);
    return v;
}

// proj/src/ks_model.cpp:107-143
Energy total_energy(const System& s, const Space& V, const std::vector<Vec>& orb, const Vec& w) {
    Energy e;
    if (orb.empty()) return e;
    const Mesh& m = *V.mesh;
    for (const auto& o : orb) {
        const double semi = h1_seminorm(V, o);
        e.kinetic += 0.5 * s.occ * semi * semi;
    }
    const Vec rho = density(orb, s.occ);
    const auto& rule = keast();
    double ext = 0, har = 0, xc = 0;
    for (int t = 0; t < m.nt(); ++t) {
        const Geo g = tet_geo(m, t);
        const auto& v = m.tets[t];
        const double vol = std::abs(m.tet_volume(t));
        for (const auto& q : rule) {
            const double rv = q.b[0] * rho[v[0]] + q.b[1] * rho[v[1]] + q.b[2] * rho[v[2]] + q.b[3] * rho[v[3]];
            V3 x;
            for (int d = 0; d < 3; ++d) x[d] = q.b[0] * g.x[0][d] + q.b[1] * g.x[1][d] + q.b[2] * g.x[2][d] + q.b[3] * g.x[3][d];
            ext += q.w * g.vol * (rv * v_ext(s, x));
            double r2 = 0, w2 = 0;
            for (int i = 0; i < 4; ++i) {
                r2 += q.b[i] * rho[v[i]];
                w2 += q.b[i] * w[v[i]];
            }
            har += q.w * vol * r2 * w2;
            xc += q.w * g.vol * xc_energy_density(s, rv);
        }
    }
    e.external = ext;
    e.hartree = 0.5 * har;
    e.xc = xc;
    e.total = e.kinetic + e.external + e.hartree + e.xc;
    return e;
}

// =========================================================== estimator (proj/src/estimator.cpp)
// compute_indicators: estimator.cpp:11-85 (element residual per tet, then face jumps in face order)
Vec compute_indicators(const System& s, const Space& V, const Vec& lambdas, const std::vector<Vec>& orb,
                       const Vec& w, const Vec& vxc, double* total_sq) {
    const Mesh& m = *V.mesh;
    const int nt = m.nt(), N = int(orb.size());
    const auto& rule = keast();
    Vec eta(nt, 0.0);
#pragma omp parallel for schedule(static)
    for (int t = 0; t < nt; ++t) {
        const auto& v = m.tets[t];
        const double vol = std::abs(m.tet_volume(t));
        double acc = 0.0;
        for (const auto& q : rule) {
            V3 x{{0, 0, 0}};
            double wq = 0.0, vq = 0.0;
            for (int k = 0; k < 4; ++k) {
                for (int d = 0; d < 3; ++d) x[d] += q.b[k] * m.verts[v[k]][d];
                wq += q.b[k] * w[v[k]];
                vq += q.b[k] * vxc[v[k]];
            }
            const double pot = v_ext(s, x) + wq + vq;
            double sum_sq = 0.0;
            for (int i = 0; i < N; ++i) {
                double phi = 0.0;
                for (int k = 0; k < 4; ++k) phi += q.b[k] * orb[i][v[k]];
                const double r = (pot - lambdas[i]) * phi;
                sum_sq += r * r;
            }
            acc += q.w * vol * sum_sq;
        }
        double hT = 0.0;
        for (int i = 0; i < 4; ++i)
            for (int j = i + 1; j < 4; ++j) {
                double d2 = 0.0;
                for (int d = 0; d < 3; ++d) {
                    const double a = m.verts[v[i]][d] - m.verts[v[j]][d];
                    d2 += a * a;
                }
                hT = std::max(hT, std::sqrt(d2));
            }
        eta[t] += hT * hT * acc;
    }
    m.quad_cells += (unsigned long long)nt;
    // face geometry as TetMesh::finalize (mesh.cpp:196-211) and P1 gradients (mesh.cpp:164-173)
    auto grad = [&](int t, const Vec& f, double g[3]) {
        const Geo G = tet_geo(m, t);
        for (int d = 0; d < 3; ++d) g[d] = 0.0;
        for (int k = 0; k < 4; ++k)
            for (int d = 0; d < 3; ++d) g[d] += f[m.tets[t][k]] * G.g[k][d];
    };
    for (size_t fi = 0; fi < m.ifaces.size(); ++fi) {
        const auto& key = m.ifaces[fi];
        const int tp = m.iface_tets[fi][0], tm = m.iface_tets[fi][1];
        const V3 &a = m.verts[key[0]], &b = m.verts[key[1]], &c = m.verts[key[2]];
        const V3 ba = sub(b, a), ca = sub(c, a), cb = sub(c, b);
        V3 nrm = cross(ba, ca);
        const double len = std::sqrt(dot3(nrm, nrm));
        const double area = 0.5 * len;
        for (int d = 0; d < 3; ++d) nrm[d] /= len;
        const double diam = std::max({std::sqrt(dot3(ba, ba)), std::sqrt(dot3(ca, ca)), std::sqrt(dot3(cb, cb))});
        V3 cp{{0, 0, 0}};
        for (int i = 0; i < 4; ++i)
            for (int d = 0; d < 3; ++d) cp[d] += m.verts[m.tets[tp][i]][d];
        for (int d = 0; d < 3; ++d) cp[d] /= 4.0;
        double sgn = 0.0;
        for (int d = 0; d < 3; ++d) sgn += nrm[d] * ((a[d] + b[d] + c[d]) / 3.0 - cp[d]);
        if (sgn < 0)
            for (int d = 0; d < 3; ++d) nrm[d] = -nrm[d];
        double jump_sq = 0.0;
        for (int i = 0; i < N; ++i) {
            double gp[3], gm[3];
            grad(tp, orb[i], gp);
            grad(tm, orb[i], gm);
            double jn = 0.0;
            for (int d = 0; d < 3; ++d) jn += 0.5 * (gp[d] - gm[d]) * nrm[d];
            jump_sq += jn * jn;
        }
        const double contrib = diam * jump_sq * area;
        eta[tp] += contrib;
        eta[tm] += contrib;
    }
    double tot = 0.0;
    for (double x : eta) tot += x;
    if (total_sq) *total_sq = tot;
    return eta;
}

// dorfler_mark: estimator.cpp:87-104 (descending eta, lower index first on ties, stop at theta * total)
std::vector<int> dorfler_mark(const Vec& eta, double total_sq, double theta) {
    if (!(theta > 0.0) || theta >= 1.0) fail(E_ARG, "theta must lie in (0,1)");
    if (total_sq <= 0.0) return {};
    std::vector<int> order(eta.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = int(i);
    std::sort(order.begin(), order.end(), [&](int a, int b) {
        if (eta[a] != eta[b]) return eta[a] > eta[b];
        return a < b;
    });
    std::vector<int> marked;
    double acc = 0.0;
    for (int t : order) {
        marked.push_back(t);
        acc += eta[t];
        if (acc >= theta * total_sq) break;
    }
    return marked;
}

// =========================================================== hartree (proj/src/hartree.cpp)
Moments compute_moments(const Space& V, const Vec& rho) {
    const Mesh& m = *V.mesh;
    const auto& rule = keast();
    double q = 0;
    double first[3] = {0, 0, 0};
    for (int t = 0; t < m.nt(); ++t) {
        const auto& v = m.tets[t];
        const double vol = std::abs(m.tet_volume(t));
        for (const auto& p : rule) {
            double rv = 0, x[3] = {0, 0, 0};
            for (int i = 0; i < 4; ++i) {
                rv += p.b[i] * rho[v[i]];
                for (int d = 0; d < 3; ++d) x[d] += p.b[i] * m.verts[v[i]][d];
            }
            q += p.w * vol * rv;
            for (int d = 0; d < 3; ++d) first[d] += p.w * vol * rv * x[d];
        }
    }
    Moments out;
    out.q = q;
    for (int d = 0; d < 3; ++d) out.c[d] = std::abs(q) > 1e-14 ? first[d] / q : 0.5 * (m.lo[d] + m.hi[d]);
    double dip[3] = {0, 0, 0}, Q[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int t = 0; t < m.nt(); ++t) {
        const auto& v = m.tets[t];
        const double vol = std::abs(m.tet_volume(t));
        for (const auto& p : rule) {
            double rv = 0, x[3] = {0, 0, 0};
            for (int i = 0; i < 4; ++i) {
                rv += p.b[i] * rho[v[i]];
                for (int d = 0; d < 3; ++d) x[d] += p.b[i] * m.verts[v[i]][d];
            }
            double dd[3];
            for (int d = 0; d < 3; ++d) dd[d] = x[d] - out.c[d];
            const double r2 = dd[0] * dd[0] + dd[1] * dd[1] + dd[2] * dd[2];
            const double s = p.w * vol * rv;
            for (int a = 0; a < 3; ++a) {
                dip[a] += s * dd[a];
                for (int b = 0; b < 3; ++b) Q[a][b] += s * (3.0 * dd[a] * dd[b] - (a == b ? r2 : 0.0));
            }
        }
    }
    for (int a = 0; a < 3; ++a) out.dip[a] = dip[a];
    double tr = 0;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) out.Q[a][b] = 0.5 * (Q[a][b] + Q[b][a]);
    tr = (out.Q[0][0] + out.Q[1][1] + out.Q[2][2]) / 3.0;
    for (int a = 0; a < 3; ++a) out.Q[a][a] -= tr;
    return out;
}

double multipole(const Moments& m, const V3& x) {
    const double d[3] = {x[0] - m.c[0], x[1] - m.c[1], x[2] - m.c[2]};
    const double r = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (r == 0.0) fail(E_ARG, "multipole evaluated at its center");
    const double u[3] = {d[0] / r, d[1] / r, d[2] / r};
    double qu = 0;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) qu += u[a] * m.Q[a][b] * u[b];
    return m.q / r + (m.dip[0] * u[0] + m.dip[1] * u[1] + m.dip[2] * u[2]) / (r * r) + 0.5 * qu / (r * r * r);
}

Vec boundary_values(const Moments& m, const Space& V) {
    Vec bc(V.n(), 0.0);
    bool zero = m.q == 0.0;
    for (int a = 0; a < 3; ++a) {
        zero = zero && m.dip[a] == 0.0;
        for (int b = 0; b < 3; ++b) zero = zero && m.Q[a][b] == 0.0;
    }
    if (zero) return bc;
    for (int d : V.boundary) bc[d] = multipole(m, V.mesh->verts[d]);
    return bc;
}

// proj/src/hartree.cpp:108-129
Vec squared_density_load(const Space& V, const std::vector<Vec>& orb, double occ) {
    const Mesh& m = *V.mesh;
    const auto& rule = keast();
    Vec out(V.n(), 0.0);
    for (int t = 0; t < m.nt(); ++t) {
        const auto& v = m.tets[t];
        const double vol = std::abs(m.tet_volume(t));
        for (const auto& q : rule) {
            double dens = 0;
            for (const auto& o : orb) {
                double val = 0;
                for (int k = 0; k < 4; ++k) val += q.b[k] * o[v[k]];
                dens += val * val;
            }
            const double s = q.w * vol * occ * dens;
            for (int k = 0; k < 4; ++k) out[v[k]] += s * q.b[k];
        }
    }
    return out;
}

Vec solve_hartree_exact(const Elliptic& S, const Space& V, const std::vector<Vec>& orb, double occ, const Vec& bc,
                        double tol) {
    Vec load = squared_density_load(V, orb, occ);
    for (double& x : load) x *= 4.0 * kPi;
    SolveStats st;
    Vec w = S.solve(load, bc, tol, &st);
    if (!st.converged) fail(E_NONCONV, "hartree solve stalled");
    return w;
}

// =========================================================== dense linear algebra
Dense dense_of(const Csc& A) {
    Dense D(A.rows, A.cols);
    for (int c = 0; c < A.cols; ++c)
        for (int k = A.ptr[c]; k < A.ptr[c + 1]; ++k) D(A.idx[k], c) = A.val[k];
    return D;
}

bool cholesky(Dense& A) {
    const int n = A.n;
    for (int j = 0; j < n; ++j) {
        double d = A(j, j);
        for (int k = 0; k < j; ++k) d -= A(j, k) * A(j, k);
        if (!(d > 0.0) || !std::isfinite(d)) return false;
        const double l = std::sqrt(d);
        A(j, j) = l;
        for (int i = j + 1; i < n; ++i) {
            double s = A(i, j);
            for (int k = 0; k < j; ++k) s -= A(i, k) * A(j, k);
            A(i, j) = s / l;
        }
        for (int i = 0; i < j; ++i) A(i, j) = 0.0;
    }
    return true;
}

namespace {
// Householder tridiagonalisation with accumulation, then implicit QL (Wilkinson-type shift).
void sym_eig(Dense& A, Vec& d, Dense& Q) {
    const int n = A.n;
    Q = Dense(n, n);
    for (int i = 0; i < n; ++i) Q(i, i) = 1.0;
    Vec v(n), p(n);
    for (int k = 0; k + 2 < n; ++k) {
        double nx = 0;
        for (int i = k + 1; i < n; ++i) nx += A(i, k) * A(i, k);
        nx = std::sqrt(nx);
        if (nx == 0.0) continue;
        const double a = A(k + 1, k) >= 0 ? -nx : nx;
        for (int i = 0; i < n; ++i) v[i] = 0.0;
        for (int i = k + 1; i < n; ++i) v[i] = A(i, k);
        v[k + 1] -= a;
        double nv = 0;
        for (int i = k + 1; i < n; ++i) nv += v[i] * v[i];
        nv = std::sqrt(nv);
        if (nv == 0.0) continue;
        for (int i = k + 1; i < n; ++i) v[i] /= nv;
        // A <- H A H on the trailing block, H = I - 2 v v^T
        for (int i = k + 1; i < n; ++i) {
            double s = 0;
            for (int j = k + 1; j < n; ++j) s += A(i, j) * v[j];
            p[i] = s;
        }
        double K = 0;
        for (int i = k + 1; i < n; ++i) K += v[i] * p[i];
        for (int i = k + 1; i < n; ++i) p[i] -= K * v[i];
        for (int i = k + 1; i < n; ++i)
            for (int j = k + 1; j < n; ++j) A(i, j) -= 2.0 * (v[i] * p[j] + p[i] * v[j]);
        A(k + 1, k) = A(k, k + 1) = a;
        for (int i = k + 2; i < n; ++i) A(i, k) = A(k, i) = 0.0;
        for (int i = 0; i < n; ++i) {
            double s = 0;
            for (int j = k + 1; j < n; ++j) s += Q(i, j) * v[j];
            for (int j = k + 1; j < n; ++j) Q(i, j) -= 2.0 * s * v[j];
        }
    }
    d.assign(n, 0.0);
    Vec e(n, 0.0);
    for (int i = 0; i < n; ++i) d[i] = A(i, i);
    for (int i = 0; i + 1 < n; ++i) e[i] = A(i + 1, i);
    for (int l = 0; l < n; ++l) {
        for (int iter = 0;; ++iter) {
            int m = l;
            for (; m + 1 < n; ++m) {
                const double dd = std::abs(d[m]) + std::abs(d[m + 1]);
                if (std::abs(e[m]) <= 1e-16 * dd) break;
            }
            if (m == l) break;
            if (iter > 100) fail(E_NONCONV, "dense eigendecomposition failed");
            double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
            double r = std::hypot(g, 1.0);
            g = d[m] - d[l] + e[l] / (g + (g >= 0 ? r : -r));
            double s = 1, c = 1, pp = 0;
            int i = m - 1;
            bool early = false;
            for (; i >= l; --i) {
                double f = s * e[i], b = c * e[i];
                r = std::hypot(f, g);
                e[i + 1] = r;
                if (r == 0.0) {
                    d[i + 1] -= pp;
                    e[m] = 0.0;
                    early = true;
                    break;
                }
                s = f / r;
                c = g / r;
                g = d[i + 1] - pp;
                r = (d[i] - g) * s + 2.0 * c * b;
                pp = s * r;
                d[i + 1] = g + pp;
                g = c * r - b;
                for (int k = 0; k < n; ++k) {
                    f = Q(k, i + 1);
                    Q(k, i + 1) = s * Q(k, i) + c * f;
                    Q(k, i) = c * Q(k, i) - s * f;
                }
            }
            if (early) continue;
            d[l] -= pp;
            e[l] = g;
            e[m] = 0.0;
        }
    }
    // ascending order
    std::vector<int> ord(n);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return d[a] < d[b]; });
    Vec d2(n);
    Dense Q2(n, n);
    for (int j = 0; j < n; ++j) {
        d2[j] = d[ord[j]];
        for (int i = 0; i < n; ++i) Q2(i, j) = Q(i, ord[j]);
    }
    d = d2;
    Q = Q2;
}
}  // namespace

bool gen_eig(const Dense& A, const Dense& B, Vec& vals, Dense& vecs) {
    const int n = A.n;
    Dense L = B;
    if (!cholesky(L)) return false;
    // C = L^-1 A L^-T
    Dense W = A;  // W = L^-1 A
    for (int c = 0; c < n; ++c)
        for (int i = 0; i < n; ++i) {
            double s = W(i, c);
            for (int k = 0; k < i; ++k) s -= L(i, k) * W(k, c);
            W(i, c) = s / L(i, i);
        }
    Dense C(n, n);  // C^T = L^-1 W^T
    for (int c = 0; c < n; ++c)
        for (int i = 0; i < n; ++i) {
            double s = W(c, i);
            for (int k = 0; k < i; ++k) s -= L(i, k) * C(c, k);
            C(c, i) = s / L(i, i);
        }
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            const double m = 0.5 * (C(i, j) + C(j, i));
            C(i, j) = C(j, i) = m;
        }
    Dense Q;
    sym_eig(C, vals, Q);
    vecs = Dense(n, n);  // x = L^-T q
    for (int c = 0; c < n; ++c)
        for (int i = n - 1; i >= 0; --i) {
            double s = Q(i, c);
            for (int k = i + 1; k < n; ++k) s -= L(k, i) * vecs(k, c);
            vecs(i, c) = s / L(i, i);
        }
    return true;
}

// proj/src/eigensolve.cpp:306-319
void normalize_sign(Dense& V) {
    for (int j = 0; j < V.m; ++j) {
        int arg = 0;
        double best = -1.0;
        for (int i = 0; i < V.n; ++i) {
            const double a = std::abs(V(i, j));
            if (a > best + 1e-300 && a > best) {
                best = a;
                arg = i;
            }
        }
        if (V(arg, j) < 0)
            for (int i = 0; i < V.n; ++i) V(i, j) = -V(i, j);
    }
}

// proj/src/eigensolve.cpp:371-396,425-443
BorderedResult solve_bordered(const Bordered& s, int nev_scan, double floor) {
    const int n = int(s.b.size());
    const int dim = n + 1;
    const int nev = std::min(nev_scan, dim);
    Dense Ad(dim, dim), Md(dim, dim);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            Ad(i, j) = (*s.A)(i, j);
            Md(i, j) = (*s.M)(i, j);
        }
    for (int i = 0; i < n; ++i) {
        Ad(i, n) = Ad(n, i) = s.b[i];
        Md(i, n) = Md(n, i) = s.c[i];
    }
    Ad(n, n) = s.beta;
    Md(n, n) = s.gamma;
    {
        Dense L = Md;
        if (!cholesky(L)) fail(E_AMBIG, "bordered mass matrix is not positive definite");
    }
    Vec vals;
    Dense vecs;
    if (!gen_eig(Ad, Md, vals, vecs)) fail(E_NONCONV, "bordered eigendecomposition failed");
    if (!(s.gamma > 0)) fail(E_AMBIG, "augmentation vector has no mass");
    BorderedResult best;
    best.scanned = nev;
    double best_score = -1.0;
    for (int k = 0; k < nev; ++k) {
        double cdh = 0, hMh = 0;
        for (int i = 0; i < n; ++i) cdh += s.c[i] * vecs(i, k);
        for (int j = 0; j < n; ++j) {
            double t = 0;
            for (int i = 0; i < n; ++i) t += (*s.M)(i, j) * vecs(i, k);
            hMh += vecs(j, k) * t;
        }
        const double th = vecs(n, k);
        const double overlap = cdh + s.gamma * th;
        const double vn = std::sqrt(std::max(1e-300, hMh + 2.0 * th * cdh + s.gamma * th * th));
        const double score = std::abs(overlap) / (vn * std::sqrt(s.gamma));
        if (score > best_score) {
            best_score = score;
            best.lambda = vals[k];
            best.phi.assign(n, 0.0);
            for (int i = 0; i < n; ++i) best.phi[i] = vecs(i, k);
            best.theta = th;
            best.score = score;
        }
    }
    if (best_score < floor) fail(E_AMBIG, "all scanned pairs have negligible augmentation component");
    return best;
}

// =========================================================== correction (proj/src/correction.cpp)
namespace {
double inf_norm(const Vec& v) {
    double m = 0;
    for (double x : v) m = std::max(m, std::abs(x));
    return m;
}
}  // namespace

// proj/src/correction.cpp:15-24
Outer::Outer(SpaceP Vp, const Csc& a_op, const Csc* Mp, const Vec& w_hat, const Vec& v_xc, double t, int pre)
    : V(std::move(Vp)), M(Mp), tol(t), precond(pre) {
    Vec pot(w_hat.size());
    for (size_t i = 0; i < pot.size(); ++i) pot[i] = w_hat[i] + v_xc[i];
    H = a_op;
    if (inf_norm(pot) > 0) H = add(H, 1.0, assemble_mass_nodal(*V, pot));
    solver = std::make_unique<Elliptic>(H, V, precond);
}

// proj/src/correction.cpp:26-61
Vec Outer::solve_orbital(double lambda, const Vec& phi, int* attempt, int* iters) {
    const Vec Mphi = M->mul(phi);
    Vec rhs(Mphi.size());
    for (size_t i = 0; i < rhs.size(); ++i) rhs[i] = lambda * Mphi[i];
    SolveStats st;
    Vec u = solver->solve(rhs, Vec(), tol, &st);
    int total = st.iterations;
    if (st.converged) {
        if (attempt) *attempt = -1;
        if (iters) *iters = total;
        return u;
    }
    for (int k = 0; k < 4; ++k) {
        while (int(shifted.size()) <= k) {
            const int kk = int(shifted.size());
            const double base = std::abs(solver->min_diag);
            const double s = kk == 0 ? base : std::pow(4.0, kk) * (base + 1.0);
            shifted.push_back(std::make_unique<Elliptic>(add(H, s, *M), V, precond));
            sigmas.push_back(s);
        }
        const double sg = sigmas[k];
        for (size_t i = 0; i < rhs.size(); ++i) rhs[i] = (lambda + sg) * Mphi[i];
        u = shifted[k]->solve(rhs, Vec(), tol, &st);
        total += st.iterations;
        if (st.converged) {
            if (attempt) *attempt = k;
            if (iters) *iters = total;
            return u;
        }
    }
    fail(E_NONCONV, "orbital correction solve failed even after the level shift");
}

namespace {
Csc interior_columns(const Csc& P, const Space& C) {
    std::vector<Trip> t;
    for (int c = 0; c < P.cols; ++c)
        for (int k = P.ptr[c]; k < P.ptr[c + 1]; ++k)
            if (C.iidx[c] >= 0) t.push_back({P.idx[k], C.iidx[c], P.val[k]});
    return Csc::from_triplets(P.rows, C.ni(), t);
}

Vec coarse_square_load(const Space& V, const Vec& full) {
    const Mesh& m = *V.mesh;
    const auto& rule = keast();
    Vec out(V.n(), 0.0);
    for (int t = 0; t < m.nt(); ++t) {
        const auto& v = m.tets[t];
        const double vol = std::abs(m.tet_volume(t));
        for (const auto& q : rule) {
            double u = 0;
            for (int i = 0; i < 4; ++i) u += q.b[i] * full[v[i]];
            const double s = q.w * vol * u * u;
            for (int i = 0; i < 4; ++i) out[v[i]] += s * q.b[i];
        }
    }
    return out;
}

Vec interior_of(const Vec& full, const Space& V) {
    Vec o(V.ni());
    for (int i = 0; i < V.ni(); ++i) o[i] = full[V.interior[i]];
    return o;
}
Vec scatter_of(const Vec& in, const Space& V) {
    Vec o(V.n(), 0.0);
    for (int i = 0; i < V.ni(); ++i) o[V.interior[i]] = in[i];
    return o;
}
Vec dmul(const Dense& A, const Vec& x) {
    Vec y(A.n, 0.0);
    for (int j = 0; j < A.m; ++j)
        for (int i = 0; i < A.n; ++i) y[i] += A(i, j) * x[j];
    return y;
}
Vec chol_solve(const Dense& L, const Vec& b) {
    const int n = L.n;
    Vec y = b;
    for (int i = 0; i < n; ++i) {
        for (int k = 0; k < i; ++k) y[i] -= L(i, k) * y[k];
        y[i] /= L(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
        for (int k = i + 1; k < n; ++k) y[i] -= L(k, i) * y[k];
        y[i] /= L(i, i);
    }
    return y;
}
}  // namespace

// proj/src/correction.cpp:113-212
Blocks prepare_blocks(SpaceP VH, SpaceP Vh, const Csc& P_full, const Csc& S_f, const Csc& M_f, const Csc& a_f,
                      const std::vector<Vec>& phi_tilde, const Vec& w_tilde, const Vec& v_xc, double occ,
                      bool hartree_on, const Vec& bc) {
    Blocks B;
    B.VH = VH;
    B.Vh = Vh;
    B.n = int(phi_tilde.size());
    B.occ = occ;
    B.hartree_on = hartree_on;
    B.fine_mesh = Vh->mesh.get();
    B.P_int = interior_columns(P_full, *VH);
    const Csc Pt = B.P_int.transpose();
    const int nf = Vh->n();
    B.ell.assign(nf, 0.0);
    if (int(bc.size()) == nf)
        for (int d : Vh->boundary) B.ell[d] = bc[d];
    B.w_tilde0.resize(nf);
    for (int i = 0; i < nf; ++i) B.w_tilde0[i] = w_tilde[i] - B.ell[i];

    const Csc M_wt = assemble_mass_nodal(*Vh, B.w_tilde0);
    const bool has_xc = inf_norm(v_xc) > 0;
    Csc M_xc;
    if (has_xc) M_xc = assemble_mass_nodal(*Vh, v_xc);
    Csc a_eff = a_f;
    if (inf_norm(B.ell) > 0) a_eff = add(a_f, 1.0, assemble_mass_nodal(*Vh, B.ell));

    auto proj = [&](const Csc& X) { return dense_of(matmul(matmul(Pt, X), B.P_int)); };
    B.A_H1 = proj(a_eff);
    B.A_H3 = proj(M_wt);
    B.A_H4 = has_xc ? proj(M_xc) : Dense(VH->ni(), VH->ni());
    B.M_H = dense_of(interior_block(assemble_mass(*VH), *VH));
    B.C_H = dense_of(interior_block(assemble_stiffness(*VH), *VH));
    const Vec Sw = S_f.mul(B.w_tilde0), Sl = S_f.mul(B.ell);
    B.d_Hh = Pt.mul(Sw);
    B.zeta = dot(B.w_tilde0, Sw);
    B.lift_load = Pt.mul(Sl);
    B.lift_load0 = dot(B.w_tilde0, Sl);

    const int n = B.n;
    B.A_h4.resize(n);
    B.b_H1.resize(n);
    B.b_H3.resize(n);
    B.b_H4.resize(n);
    B.rhs.resize(n);
    B.c_Hh.resize(n);
    B.d_phi.resize(n);
    B.phi_tilde.resize(n);
    B.beta1.assign(n, 0);
    B.beta3.assign(n, 0);
    B.beta4.assign(n, 0);
    B.gamma.assign(n, 0);
    B.zeta_phi.assign(n, 0);
    for (int i = 0; i < n; ++i) {
        const Vec& ph = phi_tilde[i];
        B.phi_tilde[i] = ph;
        const Csc M_ph = assemble_mass_nodal(*Vh, ph);
        B.A_h4[i] = proj(M_ph);
        B.rhs[i] = Pt.mul(M_ph.mul(ph));
        Vec t = a_eff.mul(ph);
        B.b_H1[i] = Pt.mul(t);
        B.beta1[i] = dot(ph, t);
        t = M_wt.mul(ph);
        B.b_H3[i] = Pt.mul(t);
        B.beta3[i] = dot(ph, t);
        if (has_xc) {
            t = M_xc.mul(ph);
            B.b_H4[i] = Pt.mul(t);
            B.beta4[i] = dot(ph, t);
        } else {
            B.b_H4[i].assign(B.P_int.cols, 0.0);
        }
        t = M_f.mul(ph);
        B.c_Hh[i] = Pt.mul(t);
        B.gamma[i] = dot(ph, t);
        t = S_f.mul(ph);
        B.d_phi[i] = Pt.mul(t);
        B.zeta_phi[i] = dot(ph, t);
    }
    if (hartree_on) {
        B.CH_chol = B.C_H;
        if (!cholesky(B.CH_chol)) fail(E_INTERNAL, "coarse stiffness factorization failed");
        B.hartree_u = chol_solve(B.CH_chol, B.d_Hh);
        B.hartree_schur = B.zeta - dot(B.d_Hh, B.hartree_u);
        if (!(B.hartree_schur > 0)) fail(E_AMBIG, "electrostatic augmentation vector lies in the coarse space");
    }
    return B;
}

AState pure_state(const Blocks& B, const Vec& lambda) {
    AState s;
    const int nh = B.M_H.n;
    s.lambda = lambda;
    s.theta2.assign(B.n, 1.0);
    for (int i = 0; i < B.n; ++i) s.phi_H.push_back(Vec(nh, 0.0));
    s.w_H.assign(nh, 0.0);
    s.theta1 = B.hartree_on ? 1.0 : 0.0;
    return s;
}

Dense assemble_A_H2(const Blocks& B, const Vec& w_H) {
    return dense_of(interior_block(assemble_mass_nodal(*B.VH, scatter_of(w_H, *B.VH)), *B.VH));
}

Vec assemble_f_H(const Blocks& B, const AState& s) {
    Vec f(B.M_H.n, 0.0);
    for (int i = 0; i < B.n; ++i) {
        const Vec sq = interior_of(coarse_square_load(*B.VH, scatter_of(s.phi_H[i], *B.VH)), *B.VH);
        const Vec a = dmul(B.A_h4[i], s.phi_H[i]);
        for (size_t k = 0; k < f.size(); ++k) f[k] += sq[k];
        for (size_t k = 0; k < f.size(); ++k) f[k] += 2.0 * s.theta2[i] * a[k];
        for (size_t k = 0; k < f.size(); ++k) f[k] += s.theta2[i] * s.theta2[i] * B.rhs[i][k];
    }
    for (double& x : f) x *= B.occ;
    return f;
}

double assemble_g(const Blocks& B, const AState& s) {
    double g = 0;
    for (int i = 0; i < B.n; ++i) {
        g += dot(s.phi_H[i], dmul(B.A_H3, s.phi_H[i]));
        g += 2.0 * s.theta2[i] * dot(B.b_H3[i], s.phi_H[i]);
        g += s.theta2[i] * s.theta2[i] * B.beta3[i];
    }
    return B.occ * g;
}

namespace {
double state_change_sq(const Blocks& B, const AState& a, const AState& b) {
    double tot = 0;
    for (int i = 0; i < B.n; ++i) {
        Vec dp(a.phi_H[i].size());
        for (size_t k = 0; k < dp.size(); ++k) dp[k] = a.phi_H[i][k] - b.phi_H[i][k];
        const double dt = a.theta2[i] - b.theta2[i];
        const double semi = dot(dp, dmul(B.C_H, dp)) + 2.0 * dt * dot(B.d_phi[i], dp) + dt * dt * B.zeta_phi[i];
        const double l2 = dot(dp, dmul(B.M_H, dp)) + 2.0 * dt * dot(B.c_Hh[i], dp) + dt * dt * B.gamma[i];
        tot += semi + l2;
    }
    return tot;
}
}  // namespace

// proj/src/correction.cpp:279-368
InnerResult inner_scf(const Blocks& B, const AState& init, double tol, int max_it, double floor, int pad, bool fixed) {
    InnerResult out;
    out.state = init;
    const int n = B.n, nh = B.M_H.n;
    Dense A_base(nh, nh);
    for (size_t k = 0; k < A_base.a.size(); ++k) A_base.a[k] = B.A_H1.a[k] + B.A_H4.a[k];
    for (int sweep = 1; sweep <= max_it; ++sweep) {
        AState next = out.state;
        Dense A_H = A_base;
        if (B.hartree_on) {
            const Dense A2 = assemble_A_H2(B, out.state.w_H);
            for (size_t k = 0; k < A_H.a.size(); ++k) A_H.a[k] += A2.a[k];
            if (out.state.theta1 != 0.0)
                for (size_t k = 0; k < A_H.a.size(); ++k) A_H.a[k] += out.state.theta1 * B.A_H3.a[k];
        }
        for (int i = 0; i < n; ++i) {
            Vec border(nh);
            for (int k = 0; k < nh; ++k) border[k] = B.b_H1[i][k] + B.b_H4[i][k];
            double beta = B.beta1[i] + B.beta4[i];
            if (B.hartree_on) {
                const Vec b2 = dmul(B.A_h4[i], out.state.w_H);
                for (int k = 0; k < nh; ++k) border[k] += b2[k] + out.state.theta1 * B.b_H3[i][k];
                beta += dot(B.rhs[i], out.state.w_H) + out.state.theta1 * B.beta3[i];
            }
            Bordered sys;
            sys.A = &A_H;
            sys.M = &B.M_H;
            sys.b = border;
            sys.beta = beta;
            sys.c = B.c_Hh[i];
            sys.gamma = B.gamma[i];
            const auto r = solve_bordered(sys, std::min(nh + 1, n + pad), floor);
            next.lambda[i] = r.lambda;
            next.phi_H[i] = r.phi;
            next.theta2[i] = r.theta;
            const double ip = dot(next.phi_H[i], dmul(B.M_H, out.state.phi_H[i])) +
                              next.theta2[i] * dot(B.c_Hh[i], out.state.phi_H[i]) +
                              out.state.theta2[i] * dot(B.c_Hh[i], next.phi_H[i]) +
                              next.theta2[i] * out.state.theta2[i] * B.gamma[i];
            if (ip < 0) {
                for (double& x : next.phi_H[i]) x = -x;
                next.theta2[i] = -next.theta2[i];
            }
        }
        if (B.hartree_on) {
            const Vec fH = assemble_f_H(B, next);
            Vec f(nh);
            for (int k = 0; k < nh; ++k) f[k] = 4.0 * kPi * fH[k] - B.lift_load[k];
            const double g = 4.0 * kPi * assemble_g(B, next) - B.lift_load0;
            const Vec t = chol_solve(B.CH_chol, f);
            next.theta1 = (g - dot(B.d_Hh, t)) / B.hartree_schur;
            next.w_H.resize(nh);
            for (int k = 0; k < nh; ++k) next.w_H[k] = t[k] - next.theta1 * B.hartree_u[k];
        }
        const double delta = std::sqrt(state_change_sq(B, next, out.state));
        out.history.push_back(delta);
        out.state = std::move(next);
        out.iterations = sweep;
        if (!fixed && (delta < tol || !B.hartree_on)) return out;
    }
    if (fixed) return out;
    std::string msg = "inner iteration exceeded " + std::to_string(max_it) + " sweeps; recent changes:";
    for (size_t k = out.history.size() > 6 ? out.history.size() - 6 : 0; k < out.history.size(); ++k)
        msg += " " + std::to_string(out.history[k]);
    fail(E_NONCONV, msg);
}

// proj/src/correction.cpp:370-381
void expand(const AState& s, const Blocks& B, std::vector<Vec>& orb, Vec& w) {
    orb.assign(B.n, Vec());
    for (int i = 0; i < B.n; ++i) {
        Vec ph = B.P_int.mul(s.phi_H[i]);
        for (size_t k = 0; k < ph.size(); ++k) ph[k] += s.theta2[i] * B.phi_tilde[i][k];
        orb[i] = std::move(ph);
    }
    const Vec pw = B.P_int.mul(s.w_H);
    w.resize(pw.size());
    for (size_t k = 0; k < pw.size(); ++k) w[k] = B.ell[k] + pw[k] + s.theta1 * B.w_tilde0[k];
}

// =========================================================== driver (proj/src/driver.cpp, scf.cpp)
LevelOps make_level_ops(const Hier& h, int level, const System& s) {
    LevelOps o;
    o.V = h.spaces.at(level);
    o.S = assemble_stiffness(*o.V);
    o.M = assemble_mass(*o.V);
    Potential p;
    p.kind = 0;
    p.p = s.atoms;
    const Csc Mext = assemble_mass_pot(*o.V, p);
    o.a_op = add(scale(o.S, 0.5), 1.0, Mext);
    o.stiff = std::make_unique<Elliptic>(o.S, o.V, 0);
    o.P_full = h.prolongation(0, level);
    return o;
}

// proj/src/scf.cpp:22-90 with the dense branch of solve_smallest (proj/src/eigensolve.cpp:321-367)
ScfResult self_consistent_solve(const System& s, SpaceP V, double tol, int max_it, double mixing, double tol_eig,
                                std::vector<double>* hist_out) {
    const Csc S = assemble_stiffness(*V), M = assemble_mass(*V);
    Potential p;
    p.kind = 0;
    p.p = s.atoms;
    const Csc Mext = assemble_mass_pot(*V, p);
    const Csc M_ii = interior_block(M, *V);
    const Csc base = interior_block(add(scale(S, 0.5), 1.0, Mext), *V);
    const Dense Md = dense_of(M_ii);
    ScfResult res;
    res.rho.assign(V->n(), 0.0);
    res.hartree.assign(V->n(), 0.0);
    Elliptic stiff(S, V, 0);
    std::vector<double> hist;
    for (int it = 1; it <= max_it; ++it) {
        Vec w(V->n(), 0.0);
        if (s.hartree_on)
            for (int i = 0; i < V->n(); ++i) w[i] += res.hartree[i];
        if (s.xc_on)
            for (int i = 0; i < V->n(); ++i) w[i] += xc_potential(s, res.rho[i]);
        Csc A = base;
        if (s.hartree_on || s.xc_on) A = add(A, 1.0, interior_block(assemble_mass_nodal(*V, w), *V));
        Vec vals;
        Dense vecs;
        if (!gen_eig(dense_of(A), Md, vals, vecs)) fail(E_NONCONV, "dense eigendecomposition failed");
        const int nev = s.n_pairs;
        Dense X(V->ni(), nev);
        for (int j = 0; j < nev; ++j)
            for (int i = 0; i < V->ni(); ++i) X(i, j) = vecs(i, j);
        // M-orthonormalise through the Cholesky factor of X^T M X, then the sign convention
        Dense G(nev, nev);
        for (int a = 0; a < nev; ++a) {
            Vec xa(V->ni());
            for (int i = 0; i < V->ni(); ++i) xa[i] = X(i, a);
            const Vec Mx = M_ii.mul(xa);
            for (int b = 0; b < nev; ++b) {
                double t = 0;
                for (int i = 0; i < V->ni(); ++i) t += X(i, b) * Mx[i];
                G(b, a) = t;
            }
        }
        if (cholesky(G)) {
            for (int i = 0; i < V->ni(); ++i) {
                Vec row(nev);
                for (int j = 0; j < nev; ++j) row[j] = X(i, j);
                for (int j = 0; j < nev; ++j) {
                    double t = row[j];
                    for (int k = 0; k < j; ++k) t -= G(j, k) * row[k];
                    row[j] = t / G(j, j);
                }
                for (int j = 0; j < nev; ++j) X(i, j) = row[j];
            }
        }
        normalize_sign(X);
        res.lambdas.assign(vals.begin(), vals.begin() + nev);
        res.orbitals.clear();
        for (int j = 0; j < nev; ++j) {
            Vec c(V->ni());
            for (int i = 0; i < V->ni(); ++i) c[i] = X(i, j);
            res.orbitals.push_back(scatter_of(c, *V));
        }
        const Vec rn = density(res.orbitals, s.occ);
        Vec d(V->n());
        for (int i = 0; i < V->n(); ++i) d[i] = rn[i] - res.rho[i];
        const double delta = h1_norm(*V, d);
        res.iterations = it;
        if (hist_out) hist_out->push_back(delta);
        const double mix = (s.hartree_on || s.xc_on) ? mixing : 1.0;
        for (int i = 0; i < V->n(); ++i) res.rho[i] = (1.0 - mix) * res.rho[i] + mix * rn[i];
        if (s.hartree_on) {
            const Moments mo = compute_moments(*V, res.rho);
            const Vec bc = boundary_values(mo, *V);
            Vec load = M.mul(res.rho);
            for (double& x : load) x *= 4.0 * kPi;
            SolveStats st;
            res.hartree = stiff.solve(load, bc, tol_eig, &st);
            if (!st.converged) fail(E_NONCONV, "hartree solve stalled");
        }
        if (delta < tol && it >= 2) return res;
    }
    fail(E_NONCONV, "self-consistent iteration exceeded its cap");
}

// proj/src/driver.cpp:106-150
void correction_step(const System& s, const Hier& h, const LevelOps& ops, const StepConfig& cfg, Vec& lambdas,
                     std::vector<Vec>& orbitals, Vec& w, StepLog* log) {
    const double t0 = now();
    const int N = s.n_pairs;
    const Space& V = *ops.V;
    const Vec rho_cur = density(orbitals, s.occ);
    const Vec vxc = s.xc_on ? xc_field(s, rho_cur) : Vec(V.n(), 0.0);
    const Vec zero(V.n(), 0.0);
    Outer op(ops.V, ops.a_op, &ops.M, s.hartree_on ? w : zero, vxc, cfg.tol_linear, cfg.precond);
    std::vector<Vec> phi_t(N);
    if (log) {
        log->shifts.attempt.assign(N, -1);
        log->shifts.iterations.assign(N, 0);
        log->cg_iterations = 0;
    }
    for (int i = 0; i < N; ++i) {
        int att = -1, its = 0;
        phi_t[i] = op.solve_orbital(lambdas[i], orbitals[i], &att, &its);
        if (log) {
            log->shifts.attempt[i] = att;
            log->shifts.iterations[i] = its;
            log->cg_iterations += its;
        }
    }
    const double t1 = now();
    Vec w_tilde(V.n(), 0.0), bc;
    if (s.hartree_on) {
        const Moments mo = compute_moments(V, density(phi_t, s.occ));
        bc = boundary_values(mo, V);
        Vec load = squared_density_load(V, phi_t, s.occ);
        for (double& x : load) x *= 4.0 * kPi;
        SolveStats st;
        w_tilde = ops.stiff->solve(load, bc, cfg.tol_linear, &st);
        if (!st.converged) fail(E_NONCONV, "hartree solve stalled");
        if (log) log->hartree_iterations = st.iterations;
    }
    const double t2 = now();
    const Blocks B =
        prepare_blocks(h.spaces[0], ops.V, ops.P_full, ops.S, ops.M, ops.a_op, phi_t, w_tilde, vxc, s.occ, s.hartree_on, bc);
    const double t3 = now();
    const bool fixed = cfg.fixed_sweeps > 0;
    const InnerResult inner = inner_scf(B, pure_state(B, lambdas), cfg.tol_inner, fixed ? cfg.fixed_sweeps : cfg.max_inner,
                                        cfg.score_floor, cfg.nev_pad, fixed);
    const double t4 = now();
    std::vector<Vec> orb;
    Vec wn;
    expand(inner.state, B, orb, wn);
    const Vec rho_next = density(orb, s.occ);
    Vec d(V.n());
    for (int i = 0; i < V.n(); ++i) d[i] = rho_next[i] - rho_cur[i];
    const double delta = h1_norm(V, d);
    lambdas = inner.state.lambda;
    orbitals = std::move(orb);
    w = std::move(wn);
    if (log) {
        log->inner_iterations = inner.iterations;
        log->delta = delta;
        log->t_bvp = t1 - t0;
        log->t_hartree = t2 - t1;
        log->t_blocks = t3 - t2;
        log->t_inner = t4 - t3;
        log->t_total = now() - t0;
    }
}

// proj/src/driver.cpp:200-302. The reference builds A_H = A_H1 + P^T M_pot P, b = b_H1 + P^T M_pot phi_tilde and
// beta = beta1 + phi_tilde^T M_pot phi_tilde each sweep and solves the bordered problems directly; here the same
// terms come from prepare_blocks with pot in the v_xc slot (A_H4 = P^T M_pot P, b_H4, beta4 are exactly those
// products) and one Hartree-off inner sweep (A_H1 + A_H4, b_H1 + b_H4, beta1 + beta4), sign-aligned with the
// previous sweep's state as the reference does.
void solve_level_mlc(const System& s, const Hier& h, const LevelOps& ops, const StepConfig& cfg, double tol_outer,
                     int max_scf, Vec& lambdas, std::vector<Vec>& orbitals, Vec& w, Vec& rho, int* sweeps,
                     std::vector<double>* deltas) {
    const int N = s.n_pairs;
    const Space& V = *ops.V;
    const Vec zero(V.n(), 0.0);
    const Vec rho_prev = density(orbitals, s.occ);
    const Vec vxc_prev = s.xc_on ? xc_field(s, rho_prev) : zero;
    Outer op(ops.V, ops.a_op, &ops.M, s.hartree_on ? w : zero, vxc_prev, cfg.tol_linear, cfg.precond);
    std::vector<Vec> phi_t(N);
    for (int i = 0; i < N; ++i) phi_t[i] = op.solve_orbital(lambdas[i], orbitals[i], nullptr, nullptr);
    Vec bc(V.n(), 0.0);
    if (s.hartree_on) bc = boundary_values(compute_moments(V, density(phi_t, s.occ)), V);
    auto hartree_of = [&](const Vec& r) {  // hartree::solve_hartree_cached (proj/src/hartree.cpp:95-106)
        Vec load = ops.M.mul(r);
        for (double& x : load) x *= 4.0 * kPi;
        SolveStats st;
        Vec out = ops.stiff->solve(load, bc, cfg.tol_linear, &st);
        if (!st.converged) fail(E_NONCONV, "hartree solve stalled");
        return out;
    };
    const Blocks B0 = prepare_blocks(h.spaces[0], ops.V, ops.P_full, ops.S, ops.M, ops.a_op, phi_t, zero, zero, s.occ,
                                     false, Vec());
    AState state = pure_state(B0, lambdas);
    std::vector<Vec> orb;
    Vec wscr;
    expand(state, B0, orb, wscr);
    Vec rho_cur = density(orb, s.occ);
    Vec w_cur(V.n(), 0.0);
    int done = 0;
    for (int sw = 1; sw <= max_scf; ++sw) {
        const Vec vxc = s.xc_on ? xc_field(s, rho_cur) : zero;
        if (s.hartree_on) w_cur = hartree_of(rho_cur);
        Vec pot(V.n());
        for (int i = 0; i < V.n(); ++i) pot[i] = w_cur[i] + vxc[i];
        const Blocks B = prepare_blocks(h.spaces[0], ops.V, ops.P_full, ops.S, ops.M, ops.a_op, phi_t, zero, pot, s.occ,
                                        false, Vec());
        state = inner_scf(B, state, cfg.tol_inner, 1, cfg.score_floor, cfg.nev_pad).state;
        expand(state, B, orb, wscr);
        const Vec rho_next = density(orb, s.occ);
        Vec d(V.n());
        for (int i = 0; i < V.n(); ++i) d[i] = rho_next[i] - rho_cur[i];
        const double delta = h1_norm(V, d);
        if (deltas) deltas->push_back(delta);
        rho_cur = rho_next;
        done = sw;
        if (delta < tol_outer) break;
        if (sw == max_scf) fail(E_NONCONV, "correction-space iteration cap reached");
    }
    if (sweeps) *sweeps = done;
    lambdas = state.lambda;
    orbitals = orb;
    w = s.hartree_on ? hartree_of(rho_cur) : zero;
    rho = rho_cur;
}

}  // namespace orc
