#include "runtime.hpp"

#include <stdexcept>

#include "abcs/sensing.hpp"

namespace abcs {
namespace detail {
namespace {

struct ThreadCtx {
  abcs_ctx* handle = nullptr;
  int device = -1;
  int wanted = -1;  // b200::set_device, -1 = current CUDA device
  ~ThreadCtx() {
    if (handle) abcs_ctx_destroy(handle);
  }
};
thread_local ThreadCtx t_ctx;

}  // namespace

abcs_ctx* ctx() {
  int dev = t_ctx.wanted;
  if (dev < 0) check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  if (!t_ctx.handle || t_ctx.device != dev) {
    if (t_ctx.handle) abcs_ctx_destroy(t_ctx.handle);
    t_ctx.handle = nullptr;
    check(abcs_ctx_create(dev, &t_ctx.handle));
    t_ctx.device = dev;
  }
  check_cuda(cudaSetDevice(dev), "cudaSetDevice");
  return t_ctx.handle;
}

void raise_status(int status, int iteration) {
  const std::string msg = abcs_last_error();
  switch (status) {
    case ABCS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case ABCS_ERR_FORMAT: throw FormatError(msg);
    case ABCS_ERR_DIVERGENCE: throw DivergenceError(msg, iteration);
    case ABCS_ERR_LOGIC: throw std::logic_error(msg);
    case ABCS_ERR_UNSUPPORTED: throw UnsupportedError(msg);
    default: throw std::runtime_error("abcs_b200: " + msg);
  }
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("abcs_b200: ") + what + ": " + cudaGetErrorString(e));
}

std::vector<uint8_t> to_u8(const PixelImage& img, const char* who) {
  if (img.height < 0 || img.width < 0 || img.data.size() != static_cast<size_t>(img.height) * img.width)
    throw std::invalid_argument(std::string(who) + ": image data does not match its dimensions");
  std::vector<uint8_t> out(img.data.size());
  for (size_t i = 0; i < out.size(); ++i) {
    const double v = img.data[i];
    if (!(v >= 0.0 && v <= 255.0) || v != std::floor(v))
      throw std::invalid_argument(std::string(who) +
                                  ": the device path takes integer pixel values in [0, 255]");
    out[i] = static_cast<uint8_t>(v);
  }
  return out;
}

std::vector<float> to_f32(std::span<const double> v) {
  std::vector<float> out(v.size());
  for (size_t i = 0; i < v.size(); ++i) out[i] = static_cast<float>(v[i]);
  return out;
}

std::vector<double> to_f64(const std::vector<float>& v) { return std::vector<double>(v.begin(), v.end()); }

abcs_sensing_config to_c(const SensingConfig& cfg) {
  abcs_sensing_config c{};
  c.block = cfg.block;
  c.cr_num = cfg.cr_num;
  c.cr_den = cfg.cr_den;
  c.algorithm = static_cast<int32_t>(cfg.algorithm);
  c.has_threshold = cfg.threshold.has_value() ? 1 : 0;
  c.threshold = cfg.threshold.value_or(0.0);
  return c;
}

}  // namespace detail

namespace b200 {
void set_device(int device) { detail::t_ctx.wanted = device; }
int device() {
  int d = detail::t_ctx.wanted;
  if (d < 0) detail::check_cuda(cudaGetDevice(&d), "cudaGetDevice");
  return d;
}
long long launch_count() { return detail::t_ctx.handle ? abcs_ctx_launch_count(detail::t_ctx.handle) : 0; }
}  // namespace b200

}  // namespace abcs
