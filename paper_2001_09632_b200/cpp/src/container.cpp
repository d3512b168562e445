// abcs::write_measurement_set / read_measurement_set over the C ABI (container.cpp:58-149).
#include "abcs/container.hpp"

#include <fstream>
#include <iterator>
#include <stdexcept>

#include "runtime.hpp"

namespace abcs {

using detail::check;
using detail::ctx;
using detail::DeviceBuffer;

namespace {

abcs_sense_plan plan_for(const MeasurementSet& ms) {
  const BlockGrid g = ms.grid();
  abcs_sense_plan p{};
  p.height = ms.height;
  p.width = ms.width;
  p.block = ms.block;
  p.rows = g.rows;
  p.cols = g.cols;
  p.n_blocks = g.count();
  p.algorithm = p.algorithm_used = static_cast<int32_t>(ms.algorithm);
  p.cr_num = ms.cr_num;
  p.cr_den = ms.cr_den;
  p.threshold = ms.threshold;
  p.coeffs_per_image = static_cast<int64_t>(ms.coeffs.size());
  p.side_per_image = static_cast<int64_t>(ms.side.size());
  return p;
}

}  // namespace

void write_measurement_set(const MeasurementSet& ms, const std::filesystem::path& path) {  // container.cpp:58-93
  if (ms.block < 2 || static_cast<long long>(ms.block) * ms.block > 65535)
    throw std::invalid_argument("container: block size must fit u16 counts");
  const BlockGrid grid = ms.grid();
  if (static_cast<int>(ms.counts.size()) != grid.count())
    throw std::invalid_argument("container: count table does not match grid");
  if (ms.total_coeffs() != static_cast<long long>(ms.coeffs.size()))
    throw std::invalid_argument("container: payload length does not match counts");
  const abcs_sense_plan plan = plan_for(ms);
  const int64_t size = abcs_container_size(&plan);
  const int64_t stride = (size + 3) / 4 * 4;
  const std::vector<float> coeffs = detail::to_f32(ms.coeffs), side = detail::to_f32(ms.side);
  DeviceBuffer<uint16_t> d_counts(ms.counts.data(), ms.counts.size());
  DeviceBuffer<float> d_payload(coeffs.data(), std::max<size_t>(coeffs.size(), 1));
  DeviceBuffer<float> d_side(side.data(), std::max<size_t>(side.size(), 1));
  DeviceBuffer<uint8_t> d_out(stride);
  check(abcs_container_pack_batch(ctx(), &plan, d_counts.get(), d_payload.get(), side.empty() ? nullptr : d_side.get(),
                                  1, d_out.get(), stride, nullptr));
  const std::vector<uint8_t> bytes = d_out.download(size);
  std::ofstream file(path, std::ios::binary);
  if (!file) throw FormatError("cannot create container: " + path.string());
  file.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
  if (!file) throw FormatError("write failed: " + path.string());
}

MeasurementSet read_measurement_set(const std::filesystem::path& path) {  // container.cpp:95-149
  std::ifstream file(path, std::ios::binary);
  if (!file) throw FormatError("cannot open container: " + path.string());
  const std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(file)), std::istreambuf_iterator<char>());
  abcs_sense_plan plan{};
  check(abcs_container_parse(bytes.empty() ? nullptr : bytes.data(), static_cast<int64_t>(bytes.size()), &plan));
  const int64_t stride = (static_cast<int64_t>(bytes.size()) + 3) / 4 * 4;
  std::vector<uint8_t> padded(stride, 0);
  std::copy(bytes.begin(), bytes.end(), padded.begin());
  DeviceBuffer<uint8_t> d_in(padded.data(), padded.size());
  DeviceBuffer<uint16_t> d_counts(plan.n_blocks);
  DeviceBuffer<float> d_payload(std::max<int64_t>(plan.coeffs_per_image, 1));
  DeviceBuffer<float> d_side(std::max<int64_t>(plan.side_per_image, 1));
  DeviceBuffer<abcs_container_info> d_info(1);
  check(abcs_container_unpack_batch(ctx(), &plan, d_in.get(), stride, 1, d_counts.get(), d_payload.get(),
                                    plan.side_per_image ? d_side.get() : nullptr, d_info.get(), nullptr));
  const abcs_container_info info = d_info.download(1)[0];
  if (info.status != ABCS_OK) throw FormatError("container: invalid contents: " + path.string());
  MeasurementSet ms;
  ms.height = plan.height;
  ms.width = plan.width;
  ms.block = plan.block;
  ms.algorithm = static_cast<Algorithm>(info.algorithm);
  ms.cr_num = info.cr_num;
  ms.cr_den = info.cr_den;
  ms.threshold = info.threshold;
  ms.counts = d_counts.download(plan.n_blocks);
  ms.coeffs = detail::to_f64(d_payload.download(plan.coeffs_per_image));
  ms.side = detail::to_f64(d_side.download(plan.side_per_image));
  return ms;
}

}  // namespace abcs
