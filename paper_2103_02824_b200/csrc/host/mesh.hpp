// Host-side tetrahedral mesh pipeline (product code, not the oracle).
//
// Reproduces the index data of the reference mesh module bit-exactly:
//   build_box_mesh      reference proj/src/mesh.cpp:281-331
//   tagged bisection    reference proj/src/mesh.cpp:25-120 (Refiner)
//   uniform_refine      reference proj/src/mesh.cpp:333-343
//   adapt_refine        reference proj/src/mesh.cpp:345-368
//   finalize (faces)    reference proj/src/mesh.cpp:175-218
// The layout is flat SoA arrays (what the device upload consumes) and the
// face pass is a bucket sort instead of an ordered map, so it scales to 1e8 tets.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "ksb.h"

namespace ksb {

/// Error with a machine code identical to the reference's ksafem::Error codes
/// (reference proj/include/ksafem/types.hpp:20-32).
struct Failure {
    int code;
    std::string what;
};
[[noreturn]] void raise(int code, const std::string& what);

struct Mesh {
    // geometry / topology
    std::vector<double> xyz;            // n*3 vertex coordinates
    std::vector<int32_t> tets;          // T*4, positively oriented
    std::vector<int32_t> tuple;         // T*4 bisection tuple (Maubach ordering)
    std::vector<int8_t> tag;            // T, bisection tag in {1,2,3}
    std::vector<int32_t> parent;        // T, tet index in the previous level
    std::vector<int32_t> vparent;       // n*2, parent edge endpoints ({v,v} when inherited at creation)
    int32_t n_parent_vertices = 0;
    int32_t level = 0;
    double lo[3] = {-1, -1, -1};
    double hi[3] = {1, 1, 1};

    // derived by finalize()
    std::vector<int32_t> bface;         // nbf*3 sorted vertex triples, key order
    std::vector<int32_t> iface;         // nif*3 sorted vertex triples, key order
    std::vector<int32_t> iface_tets;    // nif*2 (plus = lower tet, minus)
    std::vector<double> iface_geom;     // nif*5: normal xyz, area, diameter
    std::vector<uint8_t> on_boundary;   // n

    int n_vertices() const { return static_cast<int>(xyz.size() / 3); }
    int n_tets() const { return static_cast<int>(tets.size() / 4); }
    void finalize();
};

using MeshPtr = std::shared_ptr<const Mesh>;

MeshPtr build_box_mesh(const double lo[3], const double hi[3], int n_per_axis);
MeshPtr uniform_refine(const Mesh& m);
MeshPtr adapt_refine(const Mesh& m, const int32_t* marked, int64_t n_marked);

} // namespace ksb
