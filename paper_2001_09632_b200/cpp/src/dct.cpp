// abcs::BlockDct over the C ABI (abcs_block_dct_f64): one block per call, as the reference's
// per-block API; batched callers use the ABI entry directly.
#include "abcs/dct.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

#include "runtime.hpp"

namespace abcs {

using detail::check;
using detail::ctx;
using detail::DeviceBuffer;

BlockDct::BlockDct(int size) : size_(size) {
  if (size < 1) throw std::invalid_argument("BlockDct: size must be >= 1");  // dct.cpp:10
}

static void run(int size, int inverse, std::span<const double> in, std::span<double> out, const char* who) {
  const size_t n2 = static_cast<size_t>(size) * size;
  if (in.size() != n2 || out.size() != n2) throw std::invalid_argument(std::string(who) + ": bad span size");
  DeviceBuffer<double> d_in(in.data(), n2);
  DeviceBuffer<double> d_out(n2);
  check(abcs_block_dct_f64(ctx(), size, inverse, d_in.get(), d_out.get(), 1, nullptr));
  const std::vector<double> h = d_out.download(n2);
  std::copy(h.begin(), h.end(), out.begin());
}

void BlockDct::forward(std::span<const double> pixels, std::span<double> coeffs) const {
  run(size_, 0, pixels, coeffs, "BlockDct::forward");
}

void BlockDct::inverse(std::span<const double> coeffs, std::span<double> pixels) const {
  run(size_, 1, coeffs, pixels, "BlockDct::inverse");
}

std::vector<double> dct2(const std::vector<double>& block, int size) {
  BlockDct plan(size);
  std::vector<double> out(block.size());
  plan.forward(block, out);
  return out;
}

std::vector<double> idct2(const std::vector<double>& coeffs, int size) {
  BlockDct plan(size);
  std::vector<double> out(coeffs.size());
  plan.inverse(coeffs, out);
  return out;
}

}  // namespace abcs
