// abcs:: metrics and THB/THI over the C ABI (metrics.cpp:63-225).
#include "abcs/metrics.hpp"

#include <stdexcept>

#include "runtime.hpp"

namespace abcs {

using detail::check;
using detail::ctx;
using detail::DeviceBuffer;

namespace {

QualityReport device_quality(const PixelImage& ref, const PixelImage& test, bool want_ssim) {
  if (ref.height != test.height || ref.width != test.width) throw std::invalid_argument("metric: image dimensions differ");
  if (want_ssim && (ref.height < 11 || ref.width < 11))
    throw std::invalid_argument("ssim: images smaller than the 11x11 window");
  const std::vector<uint8_t> r = detail::to_u8(ref, "metric reference");
  const std::vector<float> t = detail::to_f32(test.data);
  DeviceBuffer<uint8_t> d_r(r.data(), r.size());
  DeviceBuffer<float> d_t(t.data(), t.size());
  DeviceBuffer<double> d_out(3);
  double* o = d_out.get();
  check(abcs_quality_batch(ctx(), d_r.get(), static_cast<int64_t>(r.size()), ref.width, d_t.get(),
                           static_cast<int64_t>(t.size()), test.width, ref.height, ref.width, 1, o, o + 1,
                           want_ssim ? o + 2 : nullptr, nullptr));
  const std::vector<double> h = d_out.download(want_ssim ? 3 : 2);
  QualityReport q;
  q.mse = h[0];
  q.psnr_db = h[1];
  q.ssim = want_ssim ? h[2] : 0.0;
  return q;
}

ThresholdDecode device_threshold(const PixelImage& img, const SensingConfig& cfg, bool global) {
  cfg.validate();
  const BlockGrid g = make_grid(img.height, img.width, cfg.block);
  const std::vector<uint8_t> u8 = detail::to_u8(img, global ? "thi" : "thb");
  const abcs_sensing_config c = detail::to_c(cfg);
  DeviceBuffer<uint8_t> d_img(u8.data(), u8.size());
  DeviceBuffer<int32_t> d_counts(g.count());
  DeviceBuffer<double> d_out(g.pixel_count());
  check(abcs_threshold_decode_batch(ctx(), &c, d_img.get(), static_cast<int64_t>(u8.size()), img.width, img.height,
                                    img.width, 1, global ? 1 : 0, d_counts.get(), d_out.get(), g.pixel_count(),
                                    g.cropped_width(), nullptr));
  ThresholdDecode r;
  r.image = PixelImage(g.cropped_height(), g.cropped_width());
  r.image.data = d_out.download(g.pixel_count());
  const std::vector<int32_t> c32 = d_counts.download(g.count());
  r.counts.assign(c32.begin(), c32.end());
  return r;
}

}  // namespace

double mse(const PixelImage& ref, const PixelImage& test) { return device_quality(ref, test, false).mse; }
double psnr(const PixelImage& ref, const PixelImage& test) { return device_quality(ref, test, false).psnr_db; }
double ssim(const PixelImage& ref, const PixelImage& test) { return device_quality(ref, test, true).ssim; }
QualityReport quality(const PixelImage& ref, const PixelImage& test) { return device_quality(ref, test, true); }
ThresholdDecode thb(const PixelImage& img, const SensingConfig& cfg) { return device_threshold(img, cfg, false); }
ThresholdDecode thi(const PixelImage& img, const SensingConfig& cfg) { return device_threshold(img, cfg, true); }

}  // namespace abcs
