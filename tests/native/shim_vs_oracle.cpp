// TEST INFRASTRUCTURE: parity of the abcs:: C++ drop-in shim (libabcs_core_b200.so,
// GPU) against the C oracle (oracle/_build/libabcs_oracle.so, CPU restatement pinned
// to the reference). Built and run by tests/test_shim.py on a GPU box. Bars as in
// tests/test_gpu_parity.py: counts / side data / allocations bit-exact, payload
// <= 1e-2 absolute (fp32 vs fp64 DCT), pixels <= 1e-3, trace sigma rel 1e-4.
#include <abcs_b200.h>

#include <abcs/recon.hpp>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>

#include "../../oracle/abcs_oracle.h"

namespace {

int failures = 0;
void expect(bool ok, const std::string& what) {
  if (!ok) {
    std::fprintf(stderr, "FAIL: %s\n", what.c_str());
    ++failures;
  }
}

abcs::PixelImage synth(int h, int w, uint64_t seed, std::vector<uint8_t>& u8) {
  abcs_synth_spec spec{};
  spec.height = h;
  spec.width = w;
  spec.n_ellipses = 20;
  spec.noise_sigma = 5.0;
  spec.seed = seed;
  u8.assign(static_cast<size_t>(h) * w, 0);
  abcs_synth_generate_host(&spec, 0, 1, u8.data());
  abcs::PixelImage img(h, w);
  for (size_t i = 0; i < u8.size(); ++i) img.data[i] = u8[i];
  return img;
}

double max_diff(const std::vector<double>& a, const double* b, size_t n) {
  if (a.size() != n) return INFINITY;
  double m = 0;
  for (size_t i = 0; i < n; ++i) m = std::max(m, std::fabs(a[i] - b[i]));
  return m;
}

void check_case(int H, int W, int B, uint32_t num, uint32_t den, abcs::Algorithm algo, int iters, uint64_t seed) {
  using namespace abcs;
  const std::string tag = "H" + std::to_string(H) + " W" + std::to_string(W) + " B" + std::to_string(B) + " " +
                          std::to_string(num) + "/" + std::to_string(den) + " " + algorithm_name(algo) + ": ";
  std::vector<uint8_t> u8;
  const PixelImage img = synth(H, W, seed, u8);
  SensingConfig cfg;
  cfg.block = B;
  cfg.algorithm = algo;
  cfg.set_cr(num, den);
  const MeasurementSet ms = sense(img, cfg);

  const int nb = (H / B) * (W / B);
  std::vector<uint16_t> oc(nb);
  std::vector<double> ocoef(static_cast<size_t>(H) * W), oside(static_cast<size_t>(4) * H * W);
  long long info[O_INFO_SLOTS];
  double othr = 0;
  expect(o_sense(u8.data(), H, W, B, cfg.cr_num, cfg.cr_den, static_cast<int>(algo), 0, 0.0, oc.data(),
                 ocoef.data(), oside.data(), info, &othr) == 0, tag + "oracle sense");
  expect(ms.counts == oc, tag + "counts bit-exact");
  expect(static_cast<long long>(ms.algorithm) == info[O_INFO_ALGO], tag + "algorithm after fallbacks");
  expect(ms.threshold == othr, tag + "threshold");
  expect(max_diff(ms.coeffs, ocoef.data(), info[O_INFO_NCOEFFS]) <= 1e-2, tag + "payload");
  expect(max_diff(ms.side, oside.data(), info[O_INFO_NSIDE]) == 0.0, tag + "side data bit-exact");
  const BudgetSummary bs = measurement_budget(ms);
  expect(bs.target == info[O_INFO_TARGET] && bs.actual == info[O_INFO_ACTUAL], tag + "measurement_budget");

  const SensingOperator op = SensingOperator::from(ms);
  std::vector<double> odec(op.field_size());
  o_decode(op.grid().rows, op.grid().cols, B, oc.data(), ocoef.data(), info[O_INFO_NCOEFFS], odec.data());
  expect(max_diff(decode_idct(ms).data, odec.data(), odec.size()) <= 1e-3, tag + "decode_idct");

  if (iters > 0) {
    ReconConfig rc;
    rc.method = ReconMethod::Ida;
    rc.iterations = iters;
    const ReconResult r = reconstruct(ms, rc, &img);
    std::vector<double> ox(op.field_size()), otr(static_cast<size_t>(iters + 1) * 4);
    int div = 0;
    o_reconstruct_ida(op.grid().rows, op.grid().cols, B, oc.data(), ocoef.data(), info[O_INFO_NCOEFFS], iters, 2.0,
                      2.7, 8, u8.data(), H, W, ox.data(), otr.data(), &div);
    expect(max_diff(r.image.data, ox.data(), ox.size()) <= 1e-3, tag + "reconstruct(Ida) pixels");
    for (int t = 0; t <= iters; ++t) {
      expect(r.trace[t].iteration == static_cast<int>(otr[4 * t]), tag + "trace iteration");
      expect(std::fabs(r.trace[t].sigma - otr[4 * t + 2]) <= 1e-4 * otr[4 * t + 2], tag + "trace sigma");
      expect(std::fabs(r.trace[t].psnr_db - otr[4 * t + 3]) <= 0.01, tag + "trace psnr");
    }
  }
  if (algo == Algorithm::BBV && ms.algorithm == Algorithm::BBV) {
    const BbvParams bbv = bbv_measure(img, cfg);
    long long params[5];
    std::vector<double> var(nb), side(oside.size());
    o_bbv_measure(u8.data(), H, W, B, cfg.cr_num, cfg.cr_den, params, var.data(), side.data());
    expect(bbv.stride == params[0] && bbv.offset == params[1] && bbv.per_side == params[2] &&
               bbv.phase1_total == params[3], tag + "bbv params");
    expect(max_diff(bbv.variation, var.data(), nb) == 0.0, tag + "bbv variation bit-exact");
  }
}

}  // namespace

int main() {
  using abcs::Algorithm;
  check_case(128, 160, 16, 3, 10, Algorithm::DD, 5, 11);
  check_case(128, 160, 16, 1, 4, Algorithm::BBV, 5, 12);
  check_case(96, 128, 16, 1, 5, Algorithm::ZZ, 0, 13);
  check_case(96, 160, 8, 1, 5, Algorithm::BBV, 3, 14);
  check_case(100, 90, 16, 1, 1, Algorithm::BBV, 0, 15);   // ragged crop + full-rate fallback
  check_case(128, 128, 32, 1, 4, Algorithm::DD, 2, 16);

  std::mt19937_64 rng(5);  // largest_remainder_allocate: integer weights, ties, caps
  for (int trial = 0; trial < 200; ++trial) {
    const int n = 1 + static_cast<int>(rng() % 300);
    std::vector<double> w(n);
    std::vector<int> caps(n);
    long long cap_sum = 0;
    for (int i = 0; i < n; ++i) {
      w[i] = static_cast<double>(rng() % (trial % 3 == 0 ? 4 : 1000));
      caps[i] = static_cast<int>(rng() % 64);
      cap_sum += caps[i];
    }
    const long long budget = cap_sum ? static_cast<long long>(rng() % (cap_sum + 1)) : 0;
    std::vector<int> want(n);
    const int st = o_largest_remainder(w.data(), n, budget, caps.data(), want.data());
    if (st != 0) continue;
    expect(abcs::largest_remainder_allocate(w, budget, caps) == want, "largest_remainder_allocate bit-exact");
  }
  if (failures) {
    std::fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  std::printf("shim vs oracle ok\n");
  return 0;
}
