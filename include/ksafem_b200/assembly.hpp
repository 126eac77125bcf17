// mirrors proj/include/ksafem/assembly.hpp for the operators on the path. SpMat is a device operator:
// a slot of the level's operator table whose interior-interior / interior-boundary values live in HBM on
// the level's fixed CSR pattern (Keast-11 element quadrature scattered in setFromTriplets order).
#pragma once

#include "ksafem_b200/fespace.hpp"

namespace ksafem {
namespace fem {

class SpMat {
public:
    SpMat() = default;
    bool valid() const { return bool(st_); }
    /// operator id in the level's table (ksb_mat_* ids)
    int id() const;
    const std::shared_ptr<detail::LevelState>& state() const { return st_; }
    int rows() const;       // n_dofs of the space
    int64_t interior_nonzeros() const;
    /// host copies of the values: interior x interior (CSR on the level's pattern) and interior x boundary
    VecX interior_values() const;
    VecX boundary_values() const;
    /// CSR pattern of those values: part 0 interior x interior (interior numbering), part 1 interior x boundary
    /// (boundary numbering: position in FESpace::boundary_dofs())
    void pattern(int part, std::vector<int>& ptr, std::vector<int>& col) const;

    SpMat operator+(const SpMat& o) const;
    SpMat operator-(const SpMat& o) const;
    friend SpMat operator*(double a, const SpMat& x);

    /// internal: wrap an id (owned: released to the level's free list with the last copy)
    SpMat(std::shared_ptr<detail::LevelState> st, int id, bool owned);

private:
    std::shared_ptr<detail::LevelState> st_;
    std::shared_ptr<int> id_;
};

/// S_jk = (grad psi_k, grad psi_j)
SpMat assemble_stiffness(const FESpace& V, WorkerPool* pool = nullptr);
/// M_jk = int psi_k psi_j
SpMat assemble_mass(const FESpace& V, WorkerPool* pool = nullptr);
/// M_jk = int w psi_k psi_j, w P1-interpolated from its nodal values (exact with the degree-4 rule)
SpMat assemble_mass(const FESpace& V, const FEFunction& w, WorkerPool* pool = nullptr);

/// Sobolev norms through the assembled quadratic forms (proj/src/assembly.cpp:251-287)
double l2_norm(const FEFunction& f);
double h1_seminorm(const FEFunction& f);
double h1_norm(const FEFunction& f);

} // namespace fem
using fem::SpMat;
} // namespace ksafem
