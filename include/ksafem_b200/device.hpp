// B200 plumbing under the ksafem-compatible API: one CUDA context (ksb_ctx: device + stream) and RAII device
// buffers. Everything goes through the C-ABI in include/ksb.h.
#pragma once

#include "ksafem_b200/types.hpp"
#include "ksb.h"

#include <memory>

namespace ksafem::b200 {

/// status -> ksafem::Error(code, message) (codes 1:1 with the reference's)
void check(int status);

class Device {
public:
    explicit Device(int ordinal = 0);
    ~Device();
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    ksb_ctx* ctx() const { return ctx_; }
    void sync() const;
    /// process-wide context on device 0, created on first use
    static Device& default_device();

private:
    ksb_ctx* ctx_ = nullptr;
};

/// n doubles of device memory on a Device's context
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    DeviceBuffer(Device& d, int64_t n);
    DeviceBuffer(Device& d, const VecX& host);
    ~DeviceBuffer();
    DeviceBuffer(DeviceBuffer&& o) noexcept;
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept;
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    double* data() const { return p_; }
    int64_t size() const { return n_; }
    void upload(const double* h, int64_t n);
    void download(double* h, int64_t n) const;
    VecX to_host() const;

private:
    Device* dev_ = nullptr;
    double* p_ = nullptr;
    int64_t n_ = 0;
};

} // namespace ksafem::b200
