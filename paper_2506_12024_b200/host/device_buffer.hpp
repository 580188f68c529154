// Internal RAII device allocation for the host library (plain CUDA runtime, no torch).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "flexquant/error.hpp"

namespace flexquant {

class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t bytes) { reset(bytes); }
  ~DeviceBuffer() { release(); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }

  void reset(size_t bytes) {
    release();
    if (cudaMalloc(&p_, bytes ? bytes : 16) != cudaSuccess) throw DeviceError("cudaMalloc failed");
    n_ = bytes;
  }
  void upload(const void* host, size_t bytes) {
    if (cudaMemcpy(p_, host, bytes, cudaMemcpyHostToDevice) != cudaSuccess) throw DeviceError("H2D copy failed");
  }
  void download(void* host, size_t bytes) const {
    if (cudaMemcpy(host, p_, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) throw DeviceError("D2H copy failed");
  }
  void* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  void* p_ = nullptr;
  size_t n_ = 0;
};

}  // namespace flexquant
