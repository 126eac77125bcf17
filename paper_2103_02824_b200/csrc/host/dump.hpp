// Binary hierarchy / state dump (the reference has none; its CSV/VTK outputs,
// proj/src/driver.cpp:509-543 and proj/src/mesh.cpp:259-279, stay text). Little-endian, versioned, with an
// FNV-1a 64 checksum over the payload. Meshes store only their defining arrays (coordinates, tets, bisection
// tuples and tags, parents); the face data is recomputed by finalize(), which is deterministic.
#pragma once

#include <string>
#include <vector>

#include "mesh.hpp"

namespace ksb {

void save_meshes(const std::string& path, const std::vector<MeshPtr>& meshes);
std::vector<MeshPtr> load_meshes(const std::string& path);

struct State {
    int32_t level = 0, N = 0;
    int64_t ni = 0, n = 0;
    std::vector<double> lambdas;  // N
    std::vector<double> phi;      // ni x N, row-major (interior block)
    std::vector<double> w;        // n (full, with boundary values)
};
void save_state(const std::string& path, const State& s);
State load_state(const std::string& path);

} // namespace ksb
