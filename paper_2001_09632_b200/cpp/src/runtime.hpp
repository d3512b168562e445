// Internal plumbing of the abcs:: drop-in shim: one libabcs_b200 context per host
// thread, RAII device buffers, status -> exception mapping (the reference's
// exception types), and the double <-> u8/f32 conversions at the boundary.
#pragma once
#include <cuda_runtime_api.h>

#include <cmath>
#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "abcs/b200.hpp"
#include "abcs/image.hpp"
#include "abcs/recon.hpp"
#include "abcs/sensing.hpp"
#include "abcs_b200.h"

namespace abcs::detail {

abcs_ctx* ctx();
[[noreturn]] void raise_status(int status, int iteration = 0);
inline void check(int status) {
  if (status != ABCS_OK) raise_status(status);
}
void check_cuda(cudaError_t e, const char* what);

template <class T>
class DeviceBuffer {
 public:
  explicit DeviceBuffer(size_t count) : count_(count) {
    if (count_) check_cuda(cudaMalloc(&ptr_, count_ * sizeof(T)), "cudaMalloc");
  }
  DeviceBuffer(const T* host, size_t count) : DeviceBuffer(count) { upload(host, count); }
  ~DeviceBuffer() {
    if (ptr_) cudaFree(ptr_);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  T* get() const { return static_cast<T*>(ptr_); }
  void upload(const T* host, size_t count) {
    if (count) check_cuda(cudaMemcpy(ptr_, host, count * sizeof(T), cudaMemcpyHostToDevice), "H2D copy");
  }
  std::vector<T> download(size_t count) const {
    std::vector<T> out(count);
    if (count) check_cuda(cudaMemcpy(out.data(), ptr_, count * sizeof(T), cudaMemcpyDeviceToHost), "D2H copy");
    return out;
  }

 private:
  void* ptr_ = nullptr;
  size_t count_ = 0;
};

// Integer-valued pixels in [0, 255] -> u8 (the device path's input type).
std::vector<uint8_t> to_u8(const PixelImage& img, const char* who);
std::vector<float> to_f32(std::span<const double> v);
std::vector<double> to_f64(const std::vector<float>& v);

abcs_sensing_config to_c(const SensingConfig& cfg);

}  // namespace abcs::detail
