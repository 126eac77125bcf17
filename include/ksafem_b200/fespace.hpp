// mirrors proj/include/ksafem/fespace.hpp. An FESpace is one fine level resident on the device (ksb_level:
// interior/boundary split, CSR patterns, gather lists, composite prolongation to level 0); FEFunction
// coefficients stay host vectors, as in the reference, and travel to the device per call.
#pragma once

#include "ksafem_b200/device.hpp"
#include "ksafem_b200/mesh.hpp"

#include <memory>
#include <vector>

namespace ksafem::fem {

namespace detail {
struct LevelState;  // device level + operator-slot table (host_api/ksafem_b200.cpp)
}

class FESpace {
public:
    /// standalone space on one mesh (a one-level hierarchy of its own)
    explicit FESpace(mesh::MeshPtr m, b200::Device& dev = b200::Device::default_device());

    const mesh::TetMesh& mesh() const;
    mesh::MeshPtr mesh_ptr() const;
    int n_dofs() const;
    int n_interior() const;
    const std::vector<int>& interior_dofs() const;
    const std::vector<int>& boundary_dofs() const;
    /// position in interior_dofs(), or -1 for boundary dofs
    int interior_index(int dof) const;

    // B200
    ksb_level* device_level() const;
    b200::Device& device() const;
    const std::shared_ptr<detail::LevelState>& state() const { return st_; }
    explicit FESpace(std::shared_ptr<detail::LevelState> st) : st_(std::move(st)) {}

private:
    std::shared_ptr<detail::LevelState> st_;
};

using SpacePtr = std::shared_ptr<const FESpace>;

enum class Role { generic, wavefunction, density, hartree };

struct FEFunction {
    SpacePtr space;
    VecX coeffs;
    Role role = Role::generic;

    FEFunction() = default;
    FEFunction(SpacePtr s, Role r = Role::generic) : space(std::move(s)), coeffs(space->n_dofs(), 0.0), role(r) {}
    FEFunction(SpacePtr s, VecX c, Role r = Role::generic) : space(std::move(s)), coeffs(std::move(c)), role(r) {}
};

/// composite transfer P(from, to) as host CSR (rows: fine vertices of `to`, cols: vertices of `from`)
struct Prolongation {
    int from = 0, to = 0;
    int rows = 0, cols = 0;
    std::vector<int> ptr, col;
    VecX val;
};

/// Nested spaces over a refinement hierarchy (mirrors fem::SpaceHierarchy, proj/src/fespace.cpp:58-84)
class SpaceHierarchy {
public:
    explicit SpaceHierarchy(b200::Device& dev = b200::Device::default_device());
    ~SpaceHierarchy();
    void push(mesh::MeshPtr m);
    int n_levels() const { return int(spaces_.size()); }
    SpacePtr space(int k) const { return spaces_.at(k); }
    /// composite transfer from level 0 to level `to` (from must be 0: the correction space)
    Prolongation prolongation(int from, int to) const;
    /// warm start: level to-1 values -> level `to` (inherited vertices keep theirs, new ones average
    /// their parent edge; proj/src/fespace.cpp:76-84)
    FEFunction prolong(const FEFunction& coarse, int to) const;
    int level_of(const FESpace& s) const;

private:
    b200::Device* dev_;
    std::shared_ptr<ksb_hier> hier_;
    std::vector<mesh::MeshPtr> meshes_;
    std::vector<SpacePtr> spaces_;
};

} // namespace ksafem::fem
