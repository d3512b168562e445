// abcs:: sensing entry points over the C ABI (reference semantics: sensing.cpp,
// image.cpp:106-116,162-169, zigzag.cpp). Host-side derivations come from
// abcs_sense_plan_init; every per-pixel computation runs in libabcs_b200.
#include <numeric>
#include <stdexcept>

#include "abcs/sensing.hpp"
#include "abcs/operators.hpp"
#include "abcs/zigzag.hpp"
#include "runtime.hpp"

namespace abcs {

using detail::check;
using detail::ctx;
using detail::DeviceBuffer;

// ---- image / grid ----------------------------------------------------------------------
BlockGrid make_grid(int height, int width, int block) {  // image.cpp:106-116
  if (block < 2) throw std::invalid_argument("block size must be >= 2");
  if (block > height || block > width) throw std::invalid_argument("block size exceeds image dimensions");
  BlockGrid g;
  g.block = block;
  g.rows = height / block;
  g.cols = width / block;
  return g;
}

PixelImage crop_to_grid(const PixelImage& img, const BlockGrid& grid) {  // image.cpp:162-169
  PixelImage out(grid.cropped_height(), grid.cropped_width());
  for (int r = 0; r < out.height; ++r)
    for (int c = 0; c < out.width; ++c) out.at(r, c) = img.at(r, c);
  return out;
}

ZigzagOrder zigzag_order(int block) {
  ZigzagOrder z;
  z.block = block;
  z.index.resize(static_cast<size_t>(block) * block);
  check(abcs_zigzag_order(block, z.index.data()));
  z.rank.resize(z.index.size());
  for (size_t k = 0; k < z.index.size(); ++k) z.rank[z.index[k]] = static_cast<int>(k);
  return z;
}

// ---- config ------------------------------------------------------------------------------
const char* algorithm_name(Algorithm a) {
  switch (a) {
    case Algorithm::ZZ: return "zz";
    case Algorithm::BBV: return "bbv";
    case Algorithm::DD: return "dd";
  }
  return "?";
}

std::optional<Algorithm> algorithm_from_name(const std::string& name) {
  if (name == "zz") return Algorithm::ZZ;
  if (name == "bbv") return Algorithm::BBV;
  if (name == "dd") return Algorithm::DD;
  return std::nullopt;
}

void SensingConfig::validate() const {  // sensing.cpp:32-39
  if (block < 2 || block > 255) throw std::invalid_argument("block size must be in [2, 255]");
  if (cr_num == 0 || cr_den == 0) throw std::invalid_argument("C_R must be positive");
  if (cr_num > cr_den) throw std::invalid_argument("C_R must be in (0, 1]");
  if (threshold && *threshold < 0) throw std::invalid_argument("threshold must be >= 0");
}

long long SensingConfig::target_measurements(long long total_pixels) const {  // sensing.cpp:41-44
  return static_cast<long long>(static_cast<unsigned long long>(cr_num) * total_pixels / cr_den);
}

std::pair<uint32_t, uint32_t> SensingConfig::parse_ratio(const std::string& text) {
  uint32_t num = 0, den = 0;
  check(abcs_parse_ratio(text.c_str(), &num, &den));
  return {num, den};
}

SensingConfig& SensingConfig::set_cr(const std::string& text) {
  const auto [n, d] = parse_ratio(text);
  cr_num = n;
  cr_den = d;
  return *this;
}

SensingConfig& SensingConfig::set_cr(uint32_t num, uint32_t den) {  // sensing.cpp:89-95
  const uint32_t g = std::gcd(num, den);
  if (g == 0) throw std::invalid_argument("C_R must be positive");
  cr_num = num / g;
  cr_den = den / g;
  return *this;
}

long long AllocationPlan::actual() const {
  long long total = shared_overhead;
  for (int v : phase1) total += v;
  for (int v : phase2) total += v;
  return total;
}

long long MeasurementSet::total_coeffs() const {
  long long t = 0;
  for (uint16_t c : counts) t += c;
  return t;
}

double dd_threshold(int image_height, uint32_t cr_num, uint32_t cr_den) {
  return abcs_dd_threshold(image_height, cr_num, cr_den);
}

BudgetSummary measurement_budget(const MeasurementSet& ms) {  // sensing.cpp:472-487
  const BlockGrid g = ms.grid();
  BudgetSummary s;
  s.target = static_cast<long long>(static_cast<unsigned long long>(ms.cr_num) * g.pixel_count() / ms.cr_den);
  s.actual = ms.total_coeffs();
  if (ms.algorithm == Algorithm::BBV) {
    const long long L = static_cast<long long>(ms.cr_den / ms.cr_num);
    if (L >= 1 && L <= g.block) {
      const long long per_side = g.block / L;
      const long long extent = g.cropped_height() + g.cropped_width();
      s.actual += 2 * per_side * g.count() + (extent + L - 1) / L;
    }
  }
  return s;
}

// ---- device sensing ---------------------------------------------------------------------
namespace {

abcs_sense_plan make_plan(const SensingConfig& cfg, int height, int width) {
  const abcs_sensing_config c = detail::to_c(cfg);
  abcs_sense_plan plan{};
  check(abcs_sense_plan_init(&c, height, width, &plan));
  return plan;
}

// One image through abcs_sense_batch under `plan`.
MeasurementSet run_sense(const PixelImage& img, const SensingConfig& cfg, const abcs_sense_plan& plan) {
  const std::vector<uint8_t> u8 = detail::to_u8(img, "sense");
  DeviceBuffer<uint8_t> d_img(u8.data(), u8.size());
  DeviceBuffer<uint16_t> d_counts(plan.n_blocks);
  DeviceBuffer<float> d_payload(std::max<int64_t>(plan.coeffs_per_image, 1));
  DeviceBuffer<float> d_side(std::max<int64_t>(plan.side_per_image, 1));
  check(abcs_sense_batch(ctx(), &plan, d_img.get(), static_cast<int64_t>(img.height) * img.width, img.width, 1,
                         d_counts.get(), nullptr, d_payload.get(), plan.side_per_image ? d_side.get() : nullptr,
                         nullptr));
  MeasurementSet ms;
  ms.height = img.height;
  ms.width = img.width;
  ms.block = plan.block;
  ms.algorithm = static_cast<Algorithm>(plan.algorithm_used);
  ms.cr_num = cfg.cr_num;  // gather_prefixes stores the config's ratio (sensing.cpp:204-205)
  ms.cr_den = cfg.cr_den;
  ms.threshold = plan.threshold;
  ms.counts = d_counts.download(plan.n_blocks);
  ms.coeffs = detail::to_f64(d_payload.download(plan.coeffs_per_image));
  ms.side = detail::to_f64(d_side.download(plan.side_per_image));
  return ms;
}

SensingConfig with_algorithm(const SensingConfig& cfg, Algorithm a, bool keep_threshold) {
  SensingConfig c = cfg;
  c.algorithm = a;
  if (!keep_threshold) c.threshold.reset();
  return c;
}

}  // namespace

MeasurementSet sense(const PixelImage& img, const SensingConfig& cfg, std::string* warning) {  // sensing.cpp:418-470
  cfg.validate();
  const abcs_sense_plan plan = make_plan(cfg, img.height, img.width);
  auto warn = [&](const std::string& msg) {
    if (!warning) return;
    if (!warning->empty()) *warning += "\n";
    *warning += msg;
  };
  switch (plan.fallback) {
    case ABCS_FALLBACK_BBV_FULL_RATE: warn("full-rate sensing leaves nothing to adapt; reverting to non-adaptive zz"); break;
    case ABCS_FALLBACK_BBV_CF_EXCEEDS_BLOCK:
      warn("floor(C_F) = " + std::to_string(cfg.cf_floor()) + " exceeds block size " + std::to_string(cfg.block) +
           "; reverting to non-adaptive zz");
      break;
    case ABCS_FALLBACK_DD_PHASE1_ZERO:
      warn("phase-1 budget floor(B^2/(2 C_F)) is zero at this C_R; reverting to non-adaptive zz");
      break;
    default: break;
  }
  if (cfg.algorithm == Algorithm::ZZ && plan.zz_last_zero)
    warn("C_R is so low that some blocks receive zero coefficients");
  return run_sense(img, cfg, plan);
}

MeasurementSet sense_zz(const PixelImage& img, const SensingConfig& cfg) {
  cfg.validate();
  const SensingConfig c = with_algorithm(cfg, Algorithm::ZZ, false);
  return run_sense(img, c, make_plan(c, img.height, img.width));
}

MeasurementSet sense_dd(const PixelImage& img, const SensingConfig& cfg) {
  cfg.validate();
  const SensingConfig c = with_algorithm(cfg, Algorithm::DD, true);
  const abcs_sense_plan plan = make_plan(c, img.height, img.width);
  if (plan.dd_phase1 == 0)
    throw UnsupportedError("sense_dd with a zero phase-1 budget (sense() falls back to zz instead)");
  return run_sense(img, c, plan);
}

BbvParams bbv_measure(const PixelImage& img, const SensingConfig& cfg) {  // sensing.cpp:239-296
  cfg.validate();
  const BlockGrid g = make_grid(img.height, img.width, cfg.block);
  const long long L = cfg.cf_floor();
  BbvParams out;
  out.stride = L;
  out.offset = static_cast<int>(L / 2);
  out.per_side = (L > g.block) ? 0 : static_cast<int>(g.block / L);
  out.variation.assign(g.count(), 0.0);
  if (out.per_side == 0) return out;
  const long long extent = g.cropped_height() + g.cropped_width();
  out.phase1_total = 2LL * out.per_side * g.count() + (extent + L - 1) / L;
  int valid = 0;
  for (int j = 0; j < out.per_side; ++j) {
    const long long p = out.offset + j * L;
    if (!(p < 1 || p + 1 > g.block)) ++valid;
  }
  abcs_sense_plan plan{};
  plan.height = img.height;
  plan.width = img.width;
  plan.block = g.block;
  plan.rows = g.rows;
  plan.cols = g.cols;
  plan.n_blocks = g.count();
  plan.algorithm = plan.algorithm_used = ABCS_ALGO_BBV;
  plan.bbv_stride = L;
  plan.bbv_offset = out.offset;
  plan.bbv_per_side = out.per_side;
  plan.bbv_valid_probes = valid;
  plan.side_per_image = static_cast<int64_t>(valid) * (2LL * g.count() + g.cols + g.rows);
  const std::vector<uint8_t> u8 = detail::to_u8(img, "bbv_measure");
  DeviceBuffer<uint8_t> d_img(u8.data(), u8.size());
  DeviceBuffer<uint32_t> d_w(g.count());
  DeviceBuffer<float> d_side(std::max<int64_t>(plan.side_per_image, 1));
  check(abcs_sense_weights_batch(ctx(), &plan, d_img.get(), static_cast<int64_t>(img.height) * img.width, img.width,
                                 1, d_w.get(), d_side.get(), nullptr));
  const std::vector<uint32_t> w = d_w.download(g.count());
  for (int i = 0; i < g.count(); ++i) out.variation[i] = static_cast<double>(w[i]);
  out.side_values = detail::to_f64(d_side.download(plan.side_per_image));
  return out;
}

std::vector<int> largest_remainder_allocate(const std::vector<double>& weights, long long budget,
                                            const std::vector<int>& caps) {  // sensing.cpp:110-177
  const size_t n = weights.size();
  if (caps.size() != n) throw std::invalid_argument("allocate: weights/caps size mismatch");
  if (budget < 0) throw std::invalid_argument("allocate: negative budget");
  long long capacity = 0;
  bool integral = true;
  for (size_t i = 0; i < n; ++i) {
    if (weights[i] < 0 || !std::isfinite(weights[i]))
      throw std::invalid_argument("allocate: weights must be finite and >= 0");
    if (caps[i] < 0) throw std::invalid_argument("allocate: negative cap");
    capacity += caps[i];
    integral = integral && weights[i] == std::floor(weights[i]) && weights[i] < 4294967296.0 && caps[i] <= 65535;
  }
  if (budget > capacity) throw std::invalid_argument("allocate: budget exceeds capacity");
  if (!integral) throw UnsupportedError("device allocator takes integer weights < 2^32 and caps <= 65535");
  if (n == 0) return {};
  std::vector<uint32_t> w(n);
  for (size_t i = 0; i < n; ++i) w[i] = static_cast<uint32_t>(weights[i]);
  DeviceBuffer<uint32_t> d_w(w.data(), n);
  DeviceBuffer<int32_t> d_caps(caps.data(), n);
  DeviceBuffer<uint16_t> d_counts(n);
  DeviceBuffer<int32_t> d_status(1);
  const int32_t zero = 0;
  d_status.upload(&zero, 1);
  check(abcs_allocate_batch(ctx(), d_w.get(), static_cast<int32_t>(n), 1, budget, d_caps.get(), 0, 0, d_counts.get(),
                            nullptr, d_status.get(), nullptr));
  const int st = d_status.download(1)[0];
  if (st == ABCS_ERR_INVALID_ARGUMENT) throw std::invalid_argument("allocate: budget exceeds capacity");
  if (st == ABCS_ERR_LOGIC) throw std::logic_error("allocate: capacity exhausted before budget placed");
  if (st != ABCS_OK) detail::raise_status(st);
  const std::vector<uint16_t> c = d_counts.download(n);
  return std::vector<int>(c.begin(), c.end());
}

AllocationPlan allocate_bbv(const BbvParams& bbv, long long total_budget, int n_blocks, int block) {
  // sensing.cpp:298-321
  if (static_cast<int>(bbv.variation.size()) != n_blocks)
    throw std::invalid_argument("allocate_bbv: variation/block count mismatch");
  if (total_budget <= bbv.phase1_total)
    throw std::invalid_argument("allocate_bbv: measurement budget does not cover the phase-1 probes (M <= M_BBV)");
  const int per_block = 2 * bbv.per_side;
  const int cap = block * block - per_block;
  if (cap < 0) throw std::invalid_argument("allocate_bbv: probes exceed block capacity");
  AllocationPlan plan;
  plan.block_size = block;
  plan.phase1_is_dct = false;
  plan.phase1.assign(n_blocks, per_block);
  plan.target = total_budget;
  plan.shared_overhead = bbv.phase1_total - static_cast<long long>(per_block) * n_blocks;
  plan.phase2 = largest_remainder_allocate(bbv.variation, total_budget - bbv.phase1_total,
                                           std::vector<int>(n_blocks, cap));
  return plan;
}

MeasurementSet apply_plan(const PixelImage& img, const AllocationPlan& plan, const SensingConfig& cfg) {
  // sensing.cpp:386-403: DCT + zigzag-prefix gather under the plan's counts (SensingOperator::forward)
  cfg.validate();
  const BlockGrid g = make_grid(img.height, img.width, cfg.block);
  if (plan.block_size != cfg.block || static_cast<int>(plan.phase2.size()) != g.count() ||
      plan.phase1.size() != plan.phase2.size())
    throw std::invalid_argument("apply_plan: plan does not match image/config");
  std::vector<uint16_t> counts(g.count());
  for (int i = 0; i < g.count(); ++i) {
    const int c = plan.coeff_count(i);
    if (c < 0 || c > cfg.block * cfg.block) throw std::invalid_argument("apply_plan: per-block count out of range");
    counts[i] = static_cast<uint16_t>(c);
  }
  const PixelImage cropped = crop_to_grid(img, g);
  detail::to_u8(img, "apply_plan");  // same input contract as sense()
  const std::vector<uint16_t> kept = counts;
  SensingOperator op(g, std::move(counts));
  MeasurementSet ms;
  ms.height = img.height;
  ms.width = img.width;
  ms.block = g.block;
  ms.algorithm = cfg.algorithm;
  ms.cr_num = cfg.cr_num;
  ms.cr_den = cfg.cr_den;
  ms.threshold = cfg.threshold.value_or(0.0);
  ms.counts = kept;
  ms.coeffs = op.forward(cropped.data);
  return ms;
}

}  // namespace abcs
