// abcs:: drop-in shim selftest: the reference call sequence of tools/abcs_main.cpp
// (sense -> reconstruct, SensingOperator, init_state/damp_step) on a seeded synthetic
// image, with self-consistency checks. Parity against the reference lives in
// tests/native/shim_vs_oracle.cpp. Exit 0 and "shim selftest ok" on success.
#include <abcs_b200.h>

#include <abcs/b200.hpp>
#include <abcs/container.hpp>
#include <abcs/metrics.hpp>
#include <abcs/recon.hpp>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace {

int failures = 0;
void expect(bool ok, const char* what) {
  if (!ok) {
    std::fprintf(stderr, "FAIL: %s\n", what);
    ++failures;
  }
}

double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {
  double m = a.size() == b.size() ? 0.0 : INFINITY;
  for (size_t i = 0; i < std::min(a.size(), b.size()); ++i) m = std::max(m, std::fabs(a[i] - b[i]));
  return m;
}

abcs::PixelImage synth(int h, int w, uint64_t seed) {
  abcs_synth_spec spec{};
  spec.height = h;
  spec.width = w;
  spec.n_ellipses = 20;
  spec.noise_sigma = 5.0;
  spec.seed = seed;
  std::vector<uint8_t> u8(static_cast<size_t>(h) * w);
  if (abcs_synth_generate_host(&spec, 0, 1, u8.data()) != ABCS_OK) std::abort();
  abcs::PixelImage img(h, w);
  for (size_t i = 0; i < u8.size(); ++i) img.data[i] = u8[i];
  return img;
}

}  // namespace

int main() {
  using namespace abcs;
  const PixelImage img = synth(128, 160, 7);

  // full-rate zz: the decode is the image (decode_idct is unclamped, recon.cpp:109-117)
  SensingConfig full;
  full.block = 16;
  full.set_cr("1");
  const MeasurementSet ms_full = sense(img, full);
  expect(max_abs_diff(decode_idct(ms_full).data, img.data) <= 1e-3, "C_R = 1 round trip");

  for (Algorithm a : {Algorithm::ZZ, Algorithm::BBV, Algorithm::DD}) {
    SensingConfig cfg;
    cfg.block = 16;
    cfg.algorithm = a;
    cfg.set_cr("3/10");
    std::string warning;
    const MeasurementSet ms = sense(img, cfg, &warning);
    expect(ms.total_coeffs() == static_cast<long long>(ms.coeffs.size()), "payload length == sum(counts)");
    const BudgetSummary b = measurement_budget(ms);
    expect(b.actual <= b.target, "budget within target");
    const SensingOperator op = SensingOperator::from(ms);
    const std::vector<double> again = op.forward(op.adjoint(ms.coeffs));
    expect(max_abs_diff(again, ms.coeffs) <= 1e-3, "A A* y == y");
    ReconConfig rc;
    rc.method = ReconMethod::Ida;
    rc.iterations = 4;
    const ReconResult r = reconstruct(ms, rc, &img);
    expect(r.trace.size() == 5, "trace rows = iterations + 1");
    expect(std::all_of(r.image.data.begin(), r.image.data.end(), [](double v) { return v >= 0 && v <= 255; }),
           "final clamp");
    ReconState st = init_state(op, ms.coeffs, true);
    for (int t = 0; t < rc.iterations; ++t) damp_step(st, op, ms.coeffs, rc.denoiser, ReconMethod::Ida, rc.damping, 42);
    std::vector<double> clamped = st.x;
    for (double& v : clamped) v = std::clamp(v, 0.0, 255.0);
    expect(max_abs_diff(clamped, r.image.data) <= 1e-3, "stepwise state == reconstruct");
    expect(std::fabs(st.sigma - r.trace.back().sigma) <= 1e-4 * r.trace.back().sigma, "sigma matches trace");
  }

  // .abcs container round trip (container.cpp:58-149)
  {
    SensingConfig cfg;
    cfg.block = 16;
    cfg.algorithm = Algorithm::BBV;
    cfg.set_cr("1/4");
    const MeasurementSet ms = sense(img, cfg);
    const std::filesystem::path path = std::filesystem::temp_directory_path() / "abcs_selftest.abcs";
    write_measurement_set(ms, path);
    const MeasurementSet back = read_measurement_set(path);
    expect(back.counts == ms.counts && back.coeffs == ms.coeffs && back.side == ms.side &&
               back.threshold == ms.threshold && back.algorithm == ms.algorithm,
           "container round trip");
    std::filesystem::remove(path);
  }

  {  // metrics and THB/THI (metrics.cpp:63-225)
    SensingConfig cfg;
    cfg.block = 16;
    cfg.set_cr("1/4");
    const ThresholdDecode tb = thb(img, cfg), ti = thi(img, cfg);
    long long kb = 0, ki = 0;
    for (int c : tb.counts) kb += c;
    for (int c : ti.counts) ki += c;
    const long long M = cfg.target_measurements(make_grid(img.height, img.width, 16).pixel_count());
    expect(kb == M && ki == M, "thb/thi keep M coefficients");
    const QualityReport qb = quality(crop_to_grid(img, make_grid(img.height, img.width, 16)), ti.image);
    expect(qb.psnr_db > 20 && qb.ssim > 0.5 && qb.ssim <= 1.0 && qb.mse > 0, "quality of the THI decode");
  }

  // reference error behaviour
  MeasurementSet bad = sense(img, full);
  bad.coeffs.pop_back();
  try {
    decode_idct(bad);
    expect(false, "FormatError on short payload");
  } catch (const FormatError&) {
  }
  PixelImage frac = img;
  frac.data[0] = 0.5;
  try {
    sense(frac, full);
    expect(false, "non-integer pixels rejected");
  } catch (const std::invalid_argument&) {
  }
  {  // the rest of the family: AMP, DAMP (divergence probe), blur-denoised IDA
    SensingConfig cfg;
    cfg.block = 16;
    cfg.algorithm = Algorithm::BBV;
    cfg.set_cr("1/4");
    const MeasurementSet ms = sense(img, cfg);
    for (ReconMethod m : {ReconMethod::Amp, ReconMethod::Damp, ReconMethod::DampD, ReconMethod::Ida}) {
      ReconConfig rc;
      rc.method = m;
      rc.iterations = 2;
      rc.lambda = 0.5;
      if (m == ReconMethod::Ida) rc.denoiser.name = "blur";
      const ReconResult r = reconstruct(ms, rc);
      expect(r.trace.size() == 3, "family trace rows");
    }
    DenoiserSpec blur;
    blur.name = "blur";
    const PixelImage b = denoise(blur, img, 50.0);
    expect(b.height == img.height && std::isfinite(divergence(blur, img, 50.0, 0.25, 7)), "blur + divergence");
  }
  try {
    ReconConfig bad;
    bad.method = ReconMethod::Ida;
    bad.denoiser.params["block"] = 16;
    reconstruct(sense(img, full), bad);
    expect(false, "dct_threshold block 16 is outside the device path");
  } catch (const UnsupportedError&) {
  }
  const std::vector<int> alloc = largest_remainder_allocate({3, 1, 0, 2}, 5, {4, 4, 4, 4});
  expect(alloc.size() == 4 && alloc[0] + alloc[1] + alloc[2] + alloc[3] == 5, "allocation sums to the budget");

  if (failures) {
    std::fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  std::printf("shim selftest ok (%lld kernel launches)\n", b200::launch_count());
  return 0;
}
