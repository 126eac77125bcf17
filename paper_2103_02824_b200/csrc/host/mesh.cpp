// Host mesh pipeline. See mesh.hpp for the reference functions each part replaces.
#include "mesh.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace ksb {

void raise(int code, const std::string& what) { throw Failure{code, what}; }

namespace {

inline uint64_t edge_id(int32_t a, int32_t b) {
    if (a > b) std::swap(a, b);
    return (uint64_t(uint32_t(a)) << 32) | uint32_t(b);
}

/// Open-addressing edge -> midpoint-vertex table (edges split during one refinement call).
class EdgeTable {
public:
    EdgeTable() { rehash(1 << 12); }
    int32_t find(uint64_t key) const {
        size_t i = slot(key);
        while (keys_[i] != kEmpty) {
            if (keys_[i] == key) return vals_[i];
            i = (i + 1) & mask_;
        }
        return -1;
    }
    void insert(uint64_t key, int32_t v) {
        if ((count_ + 1) * 2 > keys_.size()) rehash(keys_.size() * 2);
        size_t i = slot(key);
        while (keys_[i] != kEmpty) i = (i + 1) & mask_;
        keys_[i] = key;
        vals_[i] = v;
        ++count_;
    }

private:
    static constexpr uint64_t kEmpty = ~uint64_t(0);
    size_t slot(uint64_t k) const {
        k ^= k >> 33;
        k *= 0xff51afd7ed558ccdULL;
        k ^= k >> 33;
        return size_t(k) & mask_;
    }
    void rehash(size_t cap) {
        std::vector<uint64_t> ok(std::move(keys_));
        std::vector<int32_t> ov(std::move(vals_));
        keys_.assign(cap, kEmpty);
        vals_.assign(cap, -1);
        mask_ = cap - 1;
        count_ = 0;
        for (size_t i = 0; i < ok.size(); ++i)
            if (ok[i] != kEmpty) insert(ok[i], ov[i]);
    }
    std::vector<uint64_t> keys_;
    std::vector<int32_t> vals_;
    size_t mask_ = 0, count_ = 0;
};

inline double orient6(const double* a, const double* b, const double* c, const double* d) {
    // (b-a) x (c-a) . (d-a), same operation order as the reference's signed volume
    const double u0 = b[0] - a[0], u1 = b[1] - a[1], u2 = b[2] - a[2];
    const double v0 = c[0] - a[0], v1 = c[1] - a[1], v2 = c[2] - a[2];
    const double w0 = d[0] - a[0], w1 = d[1] - a[1], w2 = d[2] - a[2];
    const double x0 = u1 * v2 - u2 * v1, x1 = u2 * v0 - u0 * v2, x2 = u0 * v1 - u1 * v0;
    return (x0 * w0 + x1 * w1 + x2 * w2) / 6.0;
}

/// Bisection work list for one refinement call. Live elements are bisected in
/// place (parent killed, two children appended), exactly the traversal order of
/// the reference Refiner so vertex and element numbering coincide.
struct Bisector {
    const Mesh& in;
    std::vector<double> xyz;
    std::vector<int32_t> vpar;
    struct Elem {
        std::array<int32_t, 4> t;
        int8_t tag;
        int32_t root;
        bool alive;
    };
    std::vector<Elem> work;
    EdgeTable split;
    std::vector<uint8_t> vsplit;  // vertex is an endpoint of a split edge: cheap pre-filter for the closure scan

    explicit Bisector(const Mesh& m) : in(m), xyz(m.xyz), vpar(m.vparent) {
        const int nt = m.n_tets();
        work.reserve(size_t(nt) * 2);
        for (int t = 0; t < nt; ++t) {
            Elem e;
            for (int k = 0; k < 4; ++k) e.t[k] = m.tuple[4 * t + k];
            e.tag = m.tag[t];
            e.root = t;
            e.alive = true;
            work.push_back(e);
        }
    }

    int32_t midpoint(int32_t a, int32_t b) {
        const uint64_t key = edge_id(a, b);
        const int32_t hit = split.find(key);
        if (hit >= 0) return hit;
        const int32_t v = int32_t(xyz.size() / 3);
        for (int d = 0; d < 3; ++d) xyz.push_back(0.5 * (xyz[3 * a + d] + xyz[3 * b + d]));
        vpar.push_back(std::min(a, b));
        vpar.push_back(std::max(a, b));
        split.insert(key, v);
        if (vsplit.size() < size_t(v) + 1) vsplit.resize(std::max(size_t(v) + 1, vsplit.size() * 2), 0);
        vsplit[size_t(a)] = vsplit[size_t(b)] = 1;
        return v;
    }

    void bisect(size_t idx) {
        const Elem e = work[idx];
        const int d = e.tag;
        const int32_t z = midpoint(e.t[0], e.t[d]);
        const int8_t ctag = d > 1 ? int8_t(d - 1) : int8_t(3);
        Elem c1{e.t, ctag, e.root, true};
        c1.t[d] = z;
        Elem c2{{}, ctag, e.root, true};
        int w = 0;
        for (int j = 1; j <= d; ++j) c2.t[w++] = e.t[j];
        c2.t[w++] = z;
        for (int j = d + 1; j < 4; ++j) c2.t[w++] = e.t[j];
        work[idx].alive = false;
        work.push_back(c1);
        work.push_back(c2);
    }

    bool touches_split_edge(const Elem& e) const {
        // an element can only contain a split edge if two of its vertices are split-edge endpoints
        int flagged = 0;
        for (int i = 0; i < 4; ++i) flagged += size_t(e.t[i]) < vsplit.size() && vsplit[size_t(e.t[i])];
        if (flagged < 2) return false;
        for (int i = 0; i < 4; ++i)
            for (int j = i + 1; j < 4; ++j)
                if (split.find(edge_id(e.t[i], e.t[j])) >= 0) return true;
        return false;
    }

    void close() {
        for (int pass = 0; pass < 200; ++pass) {
            bool changed = false;
            for (size_t i = 0; i < work.size(); ++i) {  // work grows inside the pass
                if (!work[i].alive) continue;
                if (touches_split_edge(work[i])) {
                    bisect(i);
                    changed = true;
                }
            }
            if (!changed) return;
        }
        raise(KSB_INTERNAL, "conforming closure did not terminate");
    }

    std::shared_ptr<Mesh> emit() const {
        auto out = std::make_shared<Mesh>();
        out->xyz = xyz;
        out->vparent = vpar;
        out->n_parent_vertices = in.n_vertices();
        out->level = in.level + 1;
        std::copy(in.lo, in.lo + 3, out->lo);
        std::copy(in.hi, in.hi + 3, out->hi);
        size_t live = 0;
        for (const auto& e : work) live += e.alive;
        out->tets.reserve(live * 4);
        out->tuple.reserve(live * 4);
        out->tag.reserve(live);
        out->parent.reserve(live);
        for (const auto& e : work) {
            if (!e.alive) continue;
            std::array<int32_t, 4> t = e.t;
            if (orient6(&xyz[3 * t[0]], &xyz[3 * t[1]], &xyz[3 * t[2]], &xyz[3 * t[3]]) < 0)
                std::swap(t[2], t[3]);
            out->tets.insert(out->tets.end(), t.begin(), t.end());
            out->tuple.insert(out->tuple.end(), e.t.begin(), e.t.end());
            out->tag.push_back(e.tag);
            out->parent.push_back(e.root);
        }
        out->finalize();
        return out;
    }
};

} // namespace

void Mesh::finalize() {
    const int nv = n_vertices();
    const int nt = n_tets();
    on_boundary.assign(nv, 0);

    // Face records bucketed by their smallest vertex (counting sort), then each
    // bucket sorted by (b, c, tet): identical to ordered-map key order with
    // owners in ascending tet order. Buckets are independent, so they are sorted
    // and classified in parallel; a count pass and a prefix sum place every
    // bucket's faces at their sequential (ascending key) position.
    struct Rec {
        int32_t b, c, t;
    };
    static const int local[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
    std::vector<std::array<int32_t, 3>> keys(size_t(nt) * 4);
#pragma omp parallel for schedule(static)
    for (int t = 0; t < nt; ++t)
        for (int f = 0; f < 4; ++f) {
            std::array<int32_t, 3> k{tets[4 * t + local[f][0]], tets[4 * t + local[f][1]], tets[4 * t + local[f][2]]};
            std::sort(k.begin(), k.end());
            keys[size_t(t) * 4 + f] = k;
        }
    std::vector<int64_t> start(size_t(nv) + 1, 0);
    for (size_t i = 0; i < keys.size(); ++i) ++start[keys[i][0] + 1];
    for (int v = 0; v < nv; ++v) start[v + 1] += start[v];
    std::vector<Rec> rec(size_t(nt) * 4);
    {
        std::vector<int64_t> fill(start.begin(), start.end() - 1);
        for (int t = 0; t < nt; ++t)
            for (int f = 0; f < 4; ++f) {
                const auto& k = keys[size_t(t) * 4 + f];
                rec[fill[k[0]]++] = Rec{k[1], k[2], t};
            }
    }
    keys.clear();
    keys.shrink_to_fit();
    // pass 1: sort each bucket, count its boundary and interior faces
    std::vector<int64_t> nb(size_t(nv) + 1, 0), ni(size_t(nv) + 1, 0);
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(| : bad)
    for (int a = 0; a < nv; ++a) {
        auto* lo_ = rec.data() + start[a];
        auto* hi_ = rec.data() + start[a + 1];
        std::sort(lo_, hi_, [](const Rec& x, const Rec& y) {
            if (x.b != y.b) return x.b < y.b;
            if (x.c != y.c) return x.c < y.c;
            return x.t < y.t;
        });
        int64_t cb = 0, ci = 0;
        for (auto* p = lo_; p < hi_;) {
            auto* q = p + 1;
            while (q < hi_ && q->b == p->b && q->c == p->c) ++q;
            const int64_t cnt = q - p;
            if (cnt == 1)
                ++cb;
            else if (cnt == 2)
                ++ci;
            else
                bad = 1;
            p = q;
        }
        nb[size_t(a) + 1] = cb;
        ni[size_t(a) + 1] = ci;
    }
    if (bad) raise(KSB_INTERNAL, "face shared by more than two tets");
    for (int a = 0; a < nv; ++a) {
        nb[size_t(a) + 1] += nb[size_t(a)];
        ni[size_t(a) + 1] += ni[size_t(a)];
    }
    bface.assign(size_t(nb[nv]) * 3, 0);
    iface.assign(size_t(ni[nv]) * 3, 0);
    iface_tets.assign(size_t(ni[nv]) * 2, 0);
    iface_geom.assign(size_t(ni[nv]) * 5, 0.0);
    // pass 2: write the faces at their offsets
#pragma omp parallel for schedule(dynamic, 4096)
    for (int a = 0; a < nv; ++a) {
        const auto* lo_ = rec.data() + start[a];
        const auto* hi_ = rec.data() + start[a + 1];
        int64_t jb = nb[a], ji = ni[a];
        for (auto* p = lo_; p < hi_;) {
            auto* q = p + 1;
            while (q < hi_ && q->b == p->b && q->c == p->c) ++q;
            const int32_t fa = a, fb = p->b, fc = p->c;
            if (q - p == 1) {
                int32_t* o = &bface[size_t(jb++) * 3];
                o[0] = fa;
                o[1] = fb;
                o[2] = fc;
            } else {
                const int32_t tp = std::min(p[0].t, p[1].t), tm = std::max(p[0].t, p[1].t);
                int32_t* o = &iface[size_t(ji) * 3];
                o[0] = fa;
                o[1] = fb;
                o[2] = fc;
                iface_tets[size_t(ji) * 2] = tp;
                iface_tets[size_t(ji) * 2 + 1] = tm;
                const double* A = &xyz[3 * fa];
                const double* B = &xyz[3 * fb];
                const double* C = &xyz[3 * fc];
                double u[3], w[3], nrm[3];
                for (int d = 0; d < 3; ++d) {
                    u[d] = B[d] - A[d];
                    w[d] = C[d] - A[d];
                }
                nrm[0] = u[1] * w[2] - u[2] * w[1];
                nrm[1] = u[2] * w[0] - u[0] * w[2];
                nrm[2] = u[0] * w[1] - u[1] * w[0];
                const double len = std::sqrt(nrm[0] * nrm[0] + nrm[1] * nrm[1] + nrm[2] * nrm[2]);
                const double area = 0.5 * len;
                if (len > 0)
                    for (double& x : nrm) x /= len;
                auto dist = [](const double* p0, const double* p1) {
                    const double d0 = p1[0] - p0[0], d1 = p1[1] - p0[1], d2 = p1[2] - p0[2];
                    return std::sqrt(d0 * d0 + d1 * d1 + d2 * d2);
                };
                const double diam = std::max({dist(A, B), dist(A, C), dist(B, C)});
                double cp[3] = {0, 0, 0};
                for (int i = 0; i < 4; ++i)
                    for (int d = 0; d < 3; ++d) cp[d] += xyz[3 * tets[4 * tp + i] + d];
                double s = 0;
                for (int d = 0; d < 3; ++d) s += nrm[d] * ((A[d] + B[d] + C[d]) / 3.0 - cp[d] / 4.0);
                if (s < 0)
                    for (double& x : nrm) x = -x;
                double* g = &iface_geom[size_t(ji) * 5];
                g[0] = nrm[0];
                g[1] = nrm[1];
                g[2] = nrm[2];
                g[3] = area;
                g[4] = diam;
                ++ji;
            }
            p = q;
        }
    }
    for (size_t i = 0; i < bface.size(); ++i) on_boundary[size_t(bface[i])] = 1;
}

MeshPtr build_box_mesh(const double lo[3], const double hi[3], int n) {
    for (int d = 0; d < 3; ++d)
        if (!(hi[d] > lo[d]) || !std::isfinite(lo[d]) || !std::isfinite(hi[d]))
            raise(KSB_INVALID_DOMAIN, "box is degenerate");
    if (n < 1) raise(KSB_INVALID_DOMAIN, "n_per_axis must be >= 1");
    auto m = std::make_shared<Mesh>();
    std::copy(lo, lo + 3, m->lo);
    std::copy(hi, hi + 3, m->hi);
    const int nv = n + 1;
    const double ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    m->xyz.resize(size_t(nv) * nv * nv * 3);
    size_t w = 0;
    for (int i = 0; i < nv; ++i)
        for (int j = 0; j < nv; ++j)
            for (int k = 0; k < nv; ++k) {
                m->xyz[w++] = lo[0] + ext[0] * double(i) / n;
                m->xyz[w++] = lo[1] + ext[1] * double(j) / n;
                m->xyz[w++] = lo[2] + ext[2] * double(k) / n;
            }
    auto vid = [nv](int i, int j, int k) { return int32_t((i * nv + j) * nv + k); };
    // Kuhn split: six monotone lattice paths from the low to the high corner.
    static const int paths[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const size_t nt = size_t(n) * n * n * 6;
    m->tets.reserve(nt * 4);
    m->tuple.reserve(nt * 4);
    m->tag.assign(nt, 3);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < n; ++k)
                for (const auto& p : paths) {
                    int c[3] = {i, j, k};
                    std::array<int32_t, 4> t;
                    t[0] = vid(c[0], c[1], c[2]);
                    for (int s = 0; s < 3; ++s) {
                        ++c[p[s]];
                        t[s + 1] = vid(c[0], c[1], c[2]);
                    }
                    m->tuple.insert(m->tuple.end(), t.begin(), t.end());
                    const double* X = m->xyz.data();
                    if (orient6(X + 3 * t[0], X + 3 * t[1], X + 3 * t[2], X + 3 * t[3]) < 0)
                        std::swap(t[2], t[3]);
                    m->tets.insert(m->tets.end(), t.begin(), t.end());
                }
    m->parent.resize(nt);
    std::iota(m->parent.begin(), m->parent.end(), 0);
    const int nvert = m->n_vertices();
    m->vparent.resize(size_t(nvert) * 2);
    for (int v = 0; v < nvert; ++v) m->vparent[2 * v] = m->vparent[2 * v + 1] = v;
    m->n_parent_vertices = nvert;
    m->finalize();
    return m;
}

MeshPtr uniform_refine(const Mesh& in) {
    Bisector r(in);
    // three bisection generations split every edge: 8 children per element
    for (int gen = 0; gen < 3; ++gen) {
        const size_t count = r.work.size();
        for (size_t i = 0; i < count; ++i)
            if (r.work[i].alive) r.bisect(i);
    }
    return r.emit();
}

MeshPtr adapt_refine(const Mesh& in, const int32_t* marked, int64_t n_marked) {
    const int nt = in.n_tets();
    for (int64_t i = 0; i < n_marked; ++i)
        if (marked[i] < 0 || marked[i] >= nt) raise(KSB_INVALID_ARGUMENT, "marked tet out of range");
    if (n_marked == 0) {
        auto out = std::make_shared<Mesh>(in);
        out->level = in.level + 1;
        out->n_parent_vertices = in.n_vertices();
        for (int v = 0; v < out->n_vertices(); ++v) out->vparent[2 * v] = out->vparent[2 * v + 1] = v;
        std::iota(out->parent.begin(), out->parent.end(), 0);
        return out;
    }
    std::vector<int32_t> marks(marked, marked + n_marked);
    std::sort(marks.begin(), marks.end());
    marks.erase(std::unique(marks.begin(), marks.end()), marks.end());
    Bisector r(in);
    for (int32_t t : marks) r.bisect(size_t(t));
    r.close();
    return r.emit();
}

} // namespace ksb
