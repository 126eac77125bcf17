// ksafem-compatible host types for the B200 path (mirrors proj/include/ksafem/types.hpp).
// Eigen is not available, so VecX / Vec3 / MatX are framework-native stand-ins with the same meaning;
// SpMat is a device operator handle (fem::SpMat, assembly.hpp). Error carries the reference's codes.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace ksafem {

using VecX = std::vector<double>;

struct Vec3 {
    double v[3] = {0.0, 0.0, 0.0};
    Vec3() = default;
    Vec3(double x, double y, double z) : v{x, y, z} {}
    static Vec3 Zero() { return Vec3(); }
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
};

/// 3x3 row-major (quadrupole moments)
using Mat3 = std::array<double, 9>;

/// dense row-major matrix (ledger blocks)
struct MatX {
    int rows = 0, cols = 0;
    std::vector<double> a;
    MatX() = default;
    MatX(int r, int c) : rows(r), cols(c), a(size_t(r) * size_t(c), 0.0) {}
    double& operator()(int i, int j) { return a[size_t(i) * cols + j]; }
    double operator()(int i, int j) const { return a[size_t(i) * cols + j]; }
};

/// Error with a short machine-readable code ("invalid-domain", "nonconvergence", ...); what() = "code: message"
class Error : public std::runtime_error {
public:
    Error(std::string code, const std::string& what)
        : std::runtime_error(code + ": " + what), code_(std::move(code)) {}
    const std::string& code() const noexcept { return code_; }

private:
    std::string code_;
};

[[noreturn]] inline void fail(const std::string& code, const std::string& what) { throw Error(code, what); }

/// The reference's worker pool parallelises host loops; the device path ignores it (kept for signatures).
class WorkerPool;

} // namespace ksafem
