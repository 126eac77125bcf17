#include "dump.hpp"

#include <cstdio>
#include <cstring>

namespace ksb {

namespace {

constexpr char kHierMagic[8] = {'K', 'S', 'B', 'H', 'I', 'E', 'R', 0};
constexpr char kStateMagic[8] = {'K', 'S', 'B', 'S', 'T', 'A', 'T', 0};
constexpr uint32_t kVersion = 1;

struct Writer {
    std::FILE* f = nullptr;
    uint64_t h = 1469598103934665603ULL;
    explicit Writer(const std::string& path) : f(std::fopen(path.c_str(), "wb")) {
        if (!f) raise(KSB_IO, "cannot open " + path + " for writing");
    }
    ~Writer() {
        if (f) std::fclose(f);
    }
    void raw(const void* p, size_t n, bool hash = true) {
        if (n && std::fwrite(p, 1, n, f) != n) raise(KSB_IO, "short write");
        if (hash) {
            const auto* b = static_cast<const unsigned char*>(p);
            for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ULL;
        }
    }
    template <class T>
    void put(const T& v) { raw(&v, sizeof(T)); }
    template <class T>
    void vec(const std::vector<T>& v) {
        put<int64_t>(int64_t(v.size()));
        raw(v.data(), v.size() * sizeof(T));
    }
    void close() {
        raw(&h, sizeof h, false);
        if (std::fclose(f) != 0) {
            f = nullptr;
            raise(KSB_IO, "close failed");
        }
        f = nullptr;
    }
};

struct Reader {
    std::FILE* f = nullptr;
    uint64_t h = 1469598103934665603ULL;
    std::string path;
    explicit Reader(const std::string& p) : f(std::fopen(p.c_str(), "rb")), path(p) {
        if (!f) raise(KSB_IO, "cannot open " + p);
    }
    ~Reader() {
        if (f) std::fclose(f);
    }
    void raw(void* p, size_t n, bool hash = true) {
        if (n && std::fread(p, 1, n, f) != n) raise(KSB_IO, path + ": truncated");
        if (hash) {
            const auto* b = static_cast<const unsigned char*>(p);
            for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ULL;
        }
    }
    template <class T>
    T get() {
        T v;
        raw(&v, sizeof(T));
        return v;
    }
    template <class T>
    std::vector<T> vec(int64_t expect) {
        const int64_t n = get<int64_t>();
        if (n != expect) raise(KSB_IO, path + ": array length mismatch");
        std::vector<T> v(static_cast<size_t>(n));
        raw(v.data(), v.size() * sizeof(T));
        return v;
    }
    void finish() {
        const uint64_t want = h;
        uint64_t got = 0;
        raw(&got, sizeof got, false);
        if (got != want) raise(KSB_IO, path + ": checksum mismatch");
        char extra;
        if (std::fread(&extra, 1, 1, f) != 0) raise(KSB_IO, path + ": trailing bytes");
    }
    void magic(const char (&m)[8]) {
        char b[8];
        raw(b, 8);
        if (std::memcmp(b, m, 8) != 0) raise(KSB_IO, path + ": not a " + std::string(m) + " file");
        const uint32_t v = get<uint32_t>();
        if (v != kVersion) raise(KSB_IO, path + ": unsupported version " + std::to_string(v));
    }
};

}  // namespace

void save_meshes(const std::string& path, const std::vector<MeshPtr>& meshes) {
    Writer w(path);
    w.raw(kHierMagic, 8);
    w.put<uint32_t>(kVersion);
    w.put<uint32_t>(uint32_t(meshes.size()));
    for (const auto& mp : meshes) {
        const Mesh& m = *mp;
        w.put<int32_t>(m.level);
        w.put<int32_t>(m.n_parent_vertices);
        w.raw(m.lo, sizeof m.lo);
        w.raw(m.hi, sizeof m.hi);
        w.put<int64_t>(m.n_vertices());
        w.put<int64_t>(m.n_tets());
        w.vec(m.xyz);
        w.vec(m.tets);
        w.vec(m.tuple);
        w.vec(m.tag);
        w.vec(m.parent);
        w.vec(m.vparent);
    }
    w.close();
}

std::vector<MeshPtr> load_meshes(const std::string& path) {
    Reader r(path);
    r.magic(kHierMagic);
    const uint32_t count = r.get<uint32_t>();
    std::vector<MeshPtr> out;
    for (uint32_t k = 0; k < count; ++k) {
        auto m = std::make_shared<Mesh>();
        m->level = r.get<int32_t>();
        m->n_parent_vertices = r.get<int32_t>();
        r.raw(m->lo, sizeof m->lo);
        r.raw(m->hi, sizeof m->hi);
        const int64_t nv = r.get<int64_t>(), nt = r.get<int64_t>();
        if (nv < 0 || nt < 0 || nv > INT32_MAX || nt > INT32_MAX / 16) raise(KSB_IO, path + ": bad sizes");
        m->xyz = r.vec<double>(3 * nv);
        m->tets = r.vec<int32_t>(4 * nt);
        m->tuple = r.vec<int32_t>(4 * nt);
        m->tag = r.vec<int8_t>(nt);
        m->parent = r.vec<int32_t>(nt);
        m->vparent = r.vec<int32_t>(2 * nv);
        for (int32_t v : m->tets)
            if (v < 0 || v >= nv) raise(KSB_IO, path + ": tet vertex out of range");
        for (int32_t v : m->tuple)
            if (v < 0 || v >= nv) raise(KSB_IO, path + ": bisection tuple vertex out of range");
        for (int32_t v : m->vparent)
            if (v < 0 || v >= nv) raise(KSB_IO, path + ": vertex parent out of range");
        for (int32_t v = m->n_parent_vertices; v < int32_t(nv); ++v)
            if (m->vparent[2 * size_t(v)] >= v || m->vparent[2 * size_t(v) + 1] >= v)
                raise(KSB_IO, path + ": vertex parent created after its child");
        if (k == 0) {
            for (int32_t p : m->parent)
                if (p < 0 || p >= nt) raise(KSB_IO, path + ": tet parent out of range");
        } else {
            const int64_t npt = out.back()->n_tets();
            for (int32_t p : m->parent)
                if (p < 0 || p >= npt) raise(KSB_IO, path + ": tet parent out of range of the previous level");
        }
        for (int8_t t : m->tag)
            if (t < 1 || t > 3) raise(KSB_IO, path + ": bisection tag out of range");
        m->finalize();
        out.push_back(std::move(m));
    }
    r.finish();
    return out;
}

void save_state(const std::string& path, const State& s) {
    if (int64_t(s.lambdas.size()) != s.N || int64_t(s.phi.size()) != s.ni * s.N || int64_t(s.w.size()) != s.n)
        raise(KSB_INVALID_ARGUMENT, "state arrays do not match their sizes");
    Writer w(path);
    w.raw(kStateMagic, 8);
    w.put<uint32_t>(kVersion);
    w.put(s.level);
    w.put(s.N);
    w.put(s.ni);
    w.put(s.n);
    w.vec(s.lambdas);
    w.vec(s.phi);
    w.vec(s.w);
    w.close();
}

State load_state(const std::string& path) {
    Reader r(path);
    r.magic(kStateMagic);
    State s;
    s.level = r.get<int32_t>();
    s.N = r.get<int32_t>();
    s.ni = r.get<int64_t>();
    s.n = r.get<int64_t>();
    if (s.N < 0 || s.ni < 0 || s.n < s.ni) raise(KSB_IO, path + ": bad sizes");
    s.lambdas = r.vec<double>(s.N);
    s.phi = r.vec<double>(s.ni * s.N);
    s.w = r.vec<double>(s.n);
    r.finish();
    return s;
}

} // namespace ksb
