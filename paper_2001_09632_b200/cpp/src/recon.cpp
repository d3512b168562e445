// abcs:: operator / reconstruction / denoise entry points over the C ABI (reference
// semantics: operators.cpp:8-76, recon.cpp:39-259, denoise.cpp:96-109).
#include <cmath>
#include <limits>
#include <stdexcept>

#include "abcs/operators.hpp"
#include "abcs/recon.hpp"
#include "runtime.hpp"

namespace abcs {

using detail::check;
using detail::ctx;
using detail::DeviceBuffer;

// ---- SensingOperator -----------------------------------------------------------------------
SensingOperator::SensingOperator(const BlockGrid& grid, std::vector<uint16_t> counts)
    : grid_(grid), counts_(std::move(counts)) {  // operators.cpp:8-21
  if (static_cast<int>(counts_.size()) != grid_.count()) throw std::invalid_argument("SensingOperator: counts/grid mismatch");
  const long long area = static_cast<long long>(grid_.block) * grid_.block;
  for (uint16_t c : counts_) {
    if (c > area) throw std::invalid_argument("SensingOperator: count exceeds B^2");
    measurements_ += c;
  }
}

std::vector<double> SensingOperator::forward(std::span<const double> field) const {  // operators.cpp:23-48
  if (static_cast<long long>(field.size()) != field_size()) throw std::invalid_argument("forward: field size mismatch");
  const std::vector<float> f = detail::to_f32(field);
  DeviceBuffer<float> d_f(f.data(), f.size());
  DeviceBuffer<uint16_t> d_c(counts_.data(), counts_.size());
  DeviceBuffer<float> d_y(std::max<long long>(measurements_, 1));
  check(abcs_forward_batch(ctx(), grid_.rows, grid_.cols, grid_.block, d_c.get(), nullptr, d_f.get(), field_size(),
                           field_width(), 1, d_y.get(), measurements_, nullptr));
  return detail::to_f64(d_y.download(measurements_));
}

std::vector<double> SensingOperator::adjoint(std::span<const double> y) const {  // operators.cpp:50-76
  if (static_cast<long long>(y.size()) != measurements_)
    throw std::invalid_argument("adjoint: measurement vector length mismatch");
  const std::vector<float> yf = detail::to_f32(y);
  DeviceBuffer<float> d_y(yf.data(), std::max<size_t>(yf.size(), 1));
  DeviceBuffer<uint16_t> d_c(counts_.data(), counts_.size());
  DeviceBuffer<float> d_x(field_size());
  check(abcs_decode_batch(ctx(), grid_.rows, grid_.cols, grid_.block, d_c.get(), nullptr, d_y.get(), measurements_, 1,
                          d_x.get(), field_size(), field_width(), nullptr, nullptr, nullptr));
  return detail::to_f64(d_x.download(field_size()));
}

// ---- recon -------------------------------------------------------------------------------
const char* recon_method_name(ReconMethod m) {
  switch (m) {
    case ReconMethod::Idct: return "idct";
    case ReconMethod::Ista: return "ista";
    case ReconMethod::Amp: return "amp";
    case ReconMethod::Damp: return "damp";
    case ReconMethod::DampD: return "dampd";
    case ReconMethod::Ida: return "ida";
  }
  return "?";
}

std::optional<ReconMethod> recon_method_from_name(const std::string& name) {
  if (name == "idct") return ReconMethod::Idct;
  if (name == "ista") return ReconMethod::Ista;
  if (name == "amp") return ReconMethod::Amp;
  if (name == "damp") return ReconMethod::Damp;
  if (name == "dampd") return ReconMethod::DampD;
  if (name == "ida") return ReconMethod::Ida;
  return std::nullopt;
}

void ReconConfig::validate() const {  // recon.cpp:39-43
  if (iterations < 1) throw std::invalid_argument("iterations must be >= 1");
  if (damping < 1.0) throw std::invalid_argument("damping factor D_F must be >= 1");
  if (lambda < 0.0) throw std::invalid_argument("lambda must be >= 0");
}

PixelImage decode_idct(const MeasurementSet& ms) {  // recon.cpp:109-117
  const SensingOperator op = SensingOperator::from(ms);
  if (static_cast<long long>(ms.coeffs.size()) != op.measurements())
    throw FormatError("decode: payload length does not match counts");
  PixelImage img(op.field_height(), op.field_width());
  img.data = op.adjoint(ms.coeffs);
  return img;
}

namespace {

abcs_recon_config recon_config(ReconMethod method, int iterations, double damping, double lambda, uint64_t seed,
                                const DenoiserSpec& d) {
  abcs_recon_config c{};
  c.method = static_cast<int32_t>(method);
  c.iterations = iterations;
  c.damping = damping;
  c.lambda = lambda;
  c.seed = seed;
  if (d.name == "dct_threshold") c.denoiser = ABCS_DENOISER_DCT_THRESHOLD;
  else if (d.name == "blur") c.denoiser = ABCS_DENOISER_BLUR;
  else if (d.name == "identity") c.denoiser = ABCS_DENOISER_IDENTITY;
  else throw std::invalid_argument("unknown denoiser: '" + d.name + "'");
  c.denoiser_block = static_cast<int32_t>(d.param("block", 8.0));
  c.k = d.param("k", 2.7);
  c.sigma_scale = d.param("sigma_scale", 25.0);
  return c;
}

// Device copies of an operator's counts and a measurement vector.
struct DeviceSet {
  DeviceBuffer<uint16_t> counts;
  DeviceBuffer<float> y;
  DeviceSet(const SensingOperator& op, std::span<const double> yv)
      : counts(op.counts().data(), op.counts().size()), y(std::max<size_t>(yv.size(), 1)) {
    const std::vector<float> f = detail::to_f32(yv);
    y.upload(f.data(), f.size());
  }
};

[[noreturn]] void diverged(int iteration, int kind) {
  const char* what = kind == 1 ? "non-finite estimate" : (kind == 2 ? "|x| > 1e6" : "non-finite residual");
  throw DivergenceError(std::string("solver diverged (") + what + ") at iteration " + std::to_string(iteration),
                        iteration);
}

}  // namespace

ReconState init_state(const SensingOperator& op, std::span<const double> y, bool warm) {  // recon.cpp:119-131
  if (static_cast<long long>(y.size()) != op.measurements())
    throw std::invalid_argument("init_state: measurement vector length mismatch");
  const BlockGrid& g = op.grid();
  DeviceSet set(op, y);
  DeviceBuffer<float> d_x(op.field_size());
  DeviceBuffer<float> d_z(std::max<size_t>(y.size(), 1));
  DeviceBuffer<double> d_sigma(1);
  check(abcs_ida_init_state(ctx(), g.rows, g.cols, g.block, set.counts.get(), nullptr, set.y.get(),
                            static_cast<int64_t>(y.size()), 1, warm ? 1 : 0, d_x.get(), d_z.get(), d_sigma.get(),
                            nullptr));
  ReconState st;
  st.x = detail::to_f64(d_x.download(op.field_size()));
  st.z = detail::to_f64(d_z.download(y.size()));
  st.sigma = d_sigma.download(1)[0];
  st.iteration = 0;
  return st;
}

namespace {

// One step of any method on the explicit state via abcs_recon_step_state (recon.cpp:133-197).
void device_step(ReconState& state, const SensingOperator& op, std::span<const double> y,
                 const abcs_recon_config& cfg) {
  if (static_cast<long long>(y.size()) != op.measurements() || state.z.size() != y.size() ||
      static_cast<long long>(state.x.size()) != op.field_size())
    throw std::invalid_argument("step: state / measurement size mismatch");
  const BlockGrid& g = op.grid();
  DeviceSet set(op, y);
  const std::vector<float> xf = detail::to_f32(state.x), zf = detail::to_f32(state.z);
  DeviceBuffer<float> d_x(xf.data(), xf.size());
  DeviceBuffer<float> d_z(zf.data(), std::max<size_t>(zf.size(), 1));
  DeviceBuffer<double> d_sigma(&state.sigma, 1);
  DeviceBuffer<int32_t> d_div(2);
  const int32_t zero2[2] = {0, 0};
  d_div.upload(zero2, 2);
  check(abcs_recon_step_state(ctx(), g.rows, g.cols, g.block, set.counts.get(), nullptr, set.y.get(),
                              static_cast<int64_t>(y.size()), 1, &cfg, d_x.get(), d_z.get(), d_sigma.get(),
                              state.iteration, d_div.get(), nullptr));
  state.x = detail::to_f64(d_x.download(xf.size()));
  state.z = detail::to_f64(d_z.download(zf.size()));
  state.sigma = d_sigma.download(1)[0];
  ++state.iteration;
  const std::vector<int32_t> div = d_div.download(2);
  if (div[0] > 0) diverged(div[0], div[1]);
}

}  // namespace

void ista_step(ReconState& state, const SensingOperator& op, std::span<const double> y, double lambda) {
  device_step(state, op, y, recon_config(ReconMethod::Ista, 1, 2.0, lambda, 42, DenoiserSpec{}));
}

void amp_step(ReconState& state, const SensingOperator& op, std::span<const double> y, double lambda) {
  device_step(state, op, y, recon_config(ReconMethod::Amp, 1, 2.0, lambda, 42, DenoiserSpec{}));
}

void damp_step(ReconState& state, const SensingOperator& op, std::span<const double> y, const DenoiserSpec& denoiser,
               ReconMethod variant, double damping, uint64_t seed) {  // recon.cpp:170-197
  if (variant != ReconMethod::Damp && variant != ReconMethod::DampD && variant != ReconMethod::Ida)
    throw std::invalid_argument("damp_step: variant must be damp, dampd or ida");
  if (damping < 1.0) throw std::invalid_argument("damping factor D_F must be >= 1");
  device_step(state, op, y, recon_config(variant, 1, damping, 1.0, seed, denoiser));
}

ReconResult reconstruct(const MeasurementSet& ms, const ReconConfig& cfg, const PixelImage* reference) {
  // recon.cpp:199-259
  cfg.validate();
  const BlockGrid g = ms.grid();
  std::vector<uint8_t> ref_u8;
  if (reference) {
    if (reference->height < g.cropped_height() || reference->width < g.cropped_width())
      throw std::invalid_argument("reconstruct: reference smaller than decoded image");
    ref_u8 = detail::to_u8(crop_to_grid(*reference, g), "reconstruct reference");
  }
  ReconResult result;
  if (cfg.method == ReconMethod::Idct) {
    result.image = decode_idct(ms);
    if (reference) {
      const std::vector<float> xf = detail::to_f32(result.image.data);
      DeviceBuffer<float> d_x(xf.data(), xf.size());
      DeviceBuffer<uint8_t> d_ref(ref_u8.data(), ref_u8.size());
      DeviceBuffer<double> d_psnr(1);
      check(abcs_psnr_batch(ctx(), d_ref.get(), static_cast<int64_t>(ref_u8.size()), g.cropped_width(), d_x.get(),
                            static_cast<int64_t>(xf.size()), g.cropped_width(), g.cropped_height(), g.cropped_width(),
                            1, d_psnr.get(), nullptr));
      result.trace.push_back({0, 0.0, 0.0, d_psnr.download(1)[0]});
    }
    return result;
  }
  const SensingOperator op = SensingOperator::from(ms);
  if (static_cast<long long>(ms.coeffs.size()) != op.measurements())
    throw std::invalid_argument("init_state: measurement vector length mismatch");
  const abcs_recon_config c = recon_config(cfg.method, cfg.iterations, cfg.damping, cfg.lambda, cfg.seed, cfg.denoiser);
  DeviceSet set(op, ms.coeffs);
  DeviceBuffer<float> d_out(op.field_size());
  DeviceBuffer<double> d_trace(static_cast<size_t>(cfg.iterations + 1) * 4);
  DeviceBuffer<int32_t> d_div(2);
  DeviceBuffer<uint8_t> d_ref(std::max<size_t>(ref_u8.size(), 1));
  d_ref.upload(ref_u8.data(), ref_u8.size());
  check(abcs_reconstruct_batch(ctx(), g.rows, g.cols, g.block, set.counts.get(), nullptr, set.y.get(),
                       static_cast<int64_t>(ms.coeffs.size()), 1, &c, reference ? d_ref.get() : nullptr,
                       static_cast<int64_t>(ref_u8.size()), g.cropped_width(), d_out.get(), op.field_size(),
                       g.cropped_width(), d_trace.get(), d_div.get(), nullptr));
  const std::vector<int32_t> div = d_div.download(2);
  if (div[0] > 0) diverged(div[0], div[1]);
  result.image = PixelImage(op.field_height(), op.field_width());
  result.image.data = detail::to_f64(d_out.download(op.field_size()));
  const std::vector<double> tr = d_trace.download(static_cast<size_t>(cfg.iterations + 1) * 4);
  for (int t = 0; t <= cfg.iterations; ++t)
    result.trace.push_back({static_cast<int>(tr[4 * t]), tr[4 * t + 1], tr[4 * t + 2], tr[4 * t + 3]});
  return result;
}

// ---- denoise -----------------------------------------------------------------------------
PixelImage denoise(const DenoiserSpec& spec, const PixelImage& field, double sigma) {  // denoise.cpp:96-109
  if (sigma < 0) throw std::invalid_argument("denoise: sigma must be >= 0");
  if (spec.name == "identity") return field;
  const abcs_recon_config c = recon_config(ReconMethod::Damp, 1, 2.0, 1.0, 42, spec);  // throws on unknown names
  const std::vector<float> f = detail::to_f32(field.data);
  DeviceBuffer<float> d_in(f.data(), f.size());
  DeviceBuffer<float> d_out(f.size());
  check(abcs_denoise_batch(ctx(), d_in.get(), field.height, field.width,
                           static_cast<int64_t>(field.height) * field.width, 1, &sigma, &c, d_out.get(), nullptr));
  PixelImage out(field.height, field.width);
  out.data = detail::to_f64(d_out.download(f.size()));
  return out;
}

}  // namespace abcs

namespace abcs {

double divergence(const DenoiserSpec& spec, const PixelImage& field, double sigma, double epsilon,
                  uint64_t seed) {  // denoise.cpp:111-128
  if (epsilon <= 0) throw std::invalid_argument("divergence: epsilon must be > 0");
  const abcs_recon_config c = recon_config(ReconMethod::Damp, 1, 2.0, 1.0, seed, spec);
  const std::vector<float> f = detail::to_f32(field.data);
  DeviceBuffer<float> d_in(f.data(), f.size());
  DeviceBuffer<double> d_div(1);
  check(abcs_divergence_batch(ctx(), d_in.get(), field.height, field.width, 1, &sigma, &epsilon, seed, &c,
                              d_div.get(), nullptr));
  return d_div.download(1)[0];
}

}  // namespace abcs
