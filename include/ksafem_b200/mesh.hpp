// mirrors proj/include/ksafem/mesh.hpp: Kuhn box meshes and tagged bisection, bit-exact with the
// reference (host C++ in libksb, reached through ksb_mesh_*). TetMesh exposes its arrays by copy.
#pragma once

#include "ksafem_b200/types.hpp"
#include "ksb.h"

#include <memory>

namespace ksafem::mesh {

struct Box {
    Vec3 lo{-1.0, -1.0, -1.0};
    Vec3 hi{1.0, 1.0, 1.0};
    bool valid() const;
    Vec3 center() const { return Vec3(0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])); }
};

class TetMesh {
public:
    explicit TetMesh(ksb_mesh* handle);  // takes ownership
    ~TetMesh();
    TetMesh(const TetMesh&) = delete;
    TetMesh& operator=(const TetMesh&) = delete;

    int n_vertices() const { return int(sizes_[0]); }
    int n_tets() const { return int(sizes_[1]); }
    int n_parent_vertices() const { return int(sizes_[5]); }
    std::vector<Vec3> vertices() const;
    std::vector<std::array<int, 4>> tets() const;          // positively oriented
    std::vector<std::array<int, 4>> bisect_tuple() const;  // Maubach ordering
    std::vector<int8_t> tag() const;
    std::vector<int> parent_map() const;
    std::vector<std::array<int, 2>> vertex_parents() const;
    std::vector<char> vertex_on_boundary() const;
    Box box;
    int level = 0;
    ksb_mesh* handle() const { return h_; }

private:
    ksb_mesh* h_ = nullptr;
    int64_t sizes_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

using MeshPtr = std::shared_ptr<const TetMesh>;

/// Kuhn triangulation of the box: n^3 cubes, 6 tets each (proj/src/mesh.cpp:281-343)
MeshPtr build_box_mesh(const Box& box, int n_per_axis);
/// every tet replaced by its 8 bisection grandchildren
MeshPtr uniform_refine(const TetMesh& m);
/// bisect the marked tets, then restore conformity (proj/src/mesh.cpp:345-368)
MeshPtr adapt_refine(const TetMesh& m, const std::vector<int>& marked);

} // namespace ksafem::mesh
