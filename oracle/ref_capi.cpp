// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/proj/core,
// compiled from its own sources by oracle/Makefile into oracle/_ref/). It lets
// the pytest parity suite, golden-fixture generator and bench.py's reference /
// cpu_baseline arm drive the reference's public C++ API (abcs::sense,
// abcs::decode_idct, abcs::reconstruct, abcs::largest_remainder_allocate, ...)
// through ctypes. Nothing here re-implements reference logic; each entry point
// forwards to the reference API named in its comment.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "abcs/container.hpp"
#include "abcs/dct.hpp"
#include "abcs/denoise.hpp"
#include "abcs/image.hpp"
#include "abcs/metrics.hpp"
#include "abcs/operators.hpp"
#include "abcs/recon.hpp"
#include "abcs/sensing.hpp"
#include "abcs/synth.hpp"
#include "abcs/zigzag.hpp"

namespace {

thread_local std::string g_err;

// Status codes shared with include/abcs_b200.h so the parity tests can compare
// error behaviour one-to-one.
enum { OK = 0, INVALID = 1, FORMAT = 2, DIVERGENCE = 3, LOGIC = 5, OTHER = 7 };

template <typename F>
int guarded(F&& f, int* div_iter = nullptr) {
  try {
    f();
    return OK;
  } catch (const abcs::DivergenceError& e) {
    g_err = e.what();
    if (div_iter) *div_iter = e.iteration();
    return DIVERGENCE;
  } catch (const abcs::FormatError& e) {
    g_err = e.what();
    return FORMAT;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return INVALID;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return LOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return OTHER;
  }
}

abcs::PixelImage to_image(const uint8_t* px, int h, int w) {
  abcs::PixelImage img(h, w);
  for (size_t i = 0; i < img.data.size(); ++i) img.data[i] = px[i];
  return img;
}

abcs::SensingConfig make_cfg(int block, uint32_t num, uint32_t den, int algo, int has_thr,
                             double thr) {
  abcs::SensingConfig cfg;
  cfg.block = block;
  cfg.set_cr(num, den);
  cfg.algorithm = static_cast<abcs::Algorithm>(algo);
  if (has_thr) cfg.threshold = thr;
  return cfg;
}

struct Handle {
  abcs::MeasurementSet ms;
  std::string warning;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// abcs::sense (sensing.hpp:98-99). Returns an opaque MeasurementSet handle.
int ref_sense(const uint8_t* px, int h, int w, int block, uint32_t num, uint32_t den, int algo,
              int has_thr, double thr, void** out) {
  return guarded([&] {
    auto* hd = new Handle;
    try {
      hd->ms = abcs::sense(to_image(px, h, w), make_cfg(block, num, den, algo, has_thr, thr),
                           &hd->warning);
    } catch (...) {
      delete hd;
      throw;
    }
    *out = hd;
  });
}

// Build a MeasurementSet from raw fields (for decode/IDA parity on given payloads).
void* ref_ms_make(int h, int w, int block, int algo, uint32_t num, uint32_t den, double thr,
                  const uint16_t* counts, int n_blocks, const double* coeffs, long long n_coeffs) {
  auto* hd = new Handle;
  hd->ms.height = h;
  hd->ms.width = w;
  hd->ms.block = block;
  hd->ms.algorithm = static_cast<abcs::Algorithm>(algo);
  hd->ms.cr_num = num;
  hd->ms.cr_den = den;
  hd->ms.threshold = thr;
  hd->ms.counts.assign(counts, counts + n_blocks);
  hd->ms.coeffs.assign(coeffs, coeffs + n_coeffs);
  return hd;
}

void ref_ms_free(void* p) { delete static_cast<Handle*>(p); }

void ref_ms_set_side(void* p, const double* side, long long n) {
  static_cast<Handle*>(p)->ms.side.assign(side, side + n);
}

// Denoiser spec from (name id, k, block, sigma_scale): 0 dct_threshold, 1 blur, 2 identity.
static abcs::DenoiserSpec make_spec(int kind, double k, double dblock, double sigma_scale) {
  abcs::DenoiserSpec spec;
  spec.name = kind == 1 ? "blur" : (kind == 2 ? "identity" : "dct_threshold");
  spec.params["k"] = k;
  spec.params["block"] = dblock;
  spec.params["sigma_scale"] = sigma_scale;
  return spec;
}

// abcs::reconstruct with every ReconConfig field (recon.cpp:199-259).
int ref_reconstruct2(void* p, int method, int iters, double damping, double lambda, unsigned long long seed,
                     int denoiser, double k, double dblock, double sigma_scale, const uint8_t* ref_px, int ref_h,
                     int ref_w, double* out, double* trace, int* trace_rows, int* div_iter) {
  return guarded(
      [&] {
        abcs::ReconConfig cfg;
        cfg.method = static_cast<abcs::ReconMethod>(method);
        cfg.iterations = iters;
        cfg.damping = damping;
        cfg.lambda = lambda;
        cfg.seed = seed;
        cfg.denoiser = make_spec(denoiser, k, dblock, sigma_scale);
        abcs::PixelImage refimg;
        if (ref_px) refimg = to_image(ref_px, ref_h, ref_w);
        const auto res = abcs::reconstruct(static_cast<Handle*>(p)->ms, cfg, ref_px ? &refimg : nullptr);
        std::memcpy(out, res.image.data.data(), res.image.data.size() * sizeof(double));
        if (trace) {
          for (size_t i = 0; i < res.trace.size(); ++i) {
            trace[4 * i + 0] = res.trace[i].iteration;
            trace[4 * i + 1] = res.trace[i].residual_norm;
            trace[4 * i + 2] = res.trace[i].sigma;
            trace[4 * i + 3] = res.trace[i].psnr_db;
          }
        }
        if (trace_rows) *trace_rows = static_cast<int>(res.trace.size());
      },
      div_iter);
}

// abcs::denoise with any spec; abcs::divergence (denoise.cpp:96-128).
int ref_denoise2(const double* field, int h, int w, double sigma, int denoiser, double k, double dblock,
                 double sigma_scale, double* out) {
  return guarded([&] {
    abcs::PixelImage img(h, w);
    std::memcpy(img.data.data(), field, img.data.size() * sizeof(double));
    const auto d = abcs::denoise(make_spec(denoiser, k, dblock, sigma_scale), img, sigma);
    std::memcpy(out, d.data.data(), d.data.size() * sizeof(double));
  });
}

int ref_divergence(const double* field, int h, int w, double sigma, double eps, unsigned long long seed, int denoiser,
                   double k, double dblock, double sigma_scale, double* out) {
  return guarded([&] {
    abcs::PixelImage img(h, w);
    std::memcpy(img.data.data(), field, img.data.size() * sizeof(double));
    *out = abcs::divergence(make_spec(denoiser, k, dblock, sigma_scale), img, sigma, eps, seed);
  });
}

// The first n outputs of std::mt19937_64(seed) (the generator behind the divergence probe).
void ref_mt19937_64(unsigned long long seed, long long n, unsigned long long* out) {
  std::mt19937_64 rng(seed);
  for (long long i = 0; i < n; ++i) out[i] = rng();
}

// abcs::thb / abcs::thi (metrics.cpp:219-225) -> decoded image (cropped) and per-block counts.
int ref_threshold_decode(const uint8_t* px, int h, int w, int block, uint32_t num, uint32_t den, int global,
                         double* out, int* counts) {
  return guarded([&] {
    const abcs::SensingConfig cfg = make_cfg(block, num, den, 0, 0, 0.0);
    const abcs::ThresholdDecode r = global ? abcs::thi(to_image(px, h, w), cfg) : abcs::thb(to_image(px, h, w), cfg);
    std::memcpy(out, r.image.data.data(), r.image.data.size() * sizeof(double));
    std::memcpy(counts, r.counts.data(), r.counts.size() * sizeof(int));
  });
}

// abcs::quality (metrics.cpp:118-125) of two images given as doubles.
int ref_quality(const double* a, const double* b, int h, int w, double* mse, double* psnr, double* ssim) {
  return guarded([&] {
    abcs::PixelImage x(h, w), y(h, w);
    x.data.assign(a, a + (size_t)h * w);
    y.data.assign(b, b + (size_t)h * w);
    const abcs::QualityReport q = abcs::quality(x, y);
    *mse = q.mse;
    *psnr = q.psnr_db;
    *ssim = q.ssim;
  });
}

// abcs::write_measurement_set / read_measurement_set (container.cpp:58-149)
int ref_container_write(void* p, const char* path) {
  return guarded([&] { abcs::write_measurement_set(static_cast<Handle*>(p)->ms, path); });
}

int ref_container_read(const char* path, void** out) {
  return guarded([&] {
    auto* hd = new Handle;
    try {
      hd->ms = abcs::read_measurement_set(path);
    } catch (...) {
      delete hd;
      throw;
    }
    *out = hd;
  });
}

// info: [height, width, block, algorithm, cr_num, cr_den, n_blocks, n_coeffs, n_side,
//        budget.target, budget.actual]; threshold separately.
void ref_ms_info(void* p, long long* info, double* threshold) {
  const auto& ms = static_cast<Handle*>(p)->ms;
  const auto b = abcs::measurement_budget(ms);
  info[0] = ms.height;
  info[1] = ms.width;
  info[2] = ms.block;
  info[3] = static_cast<long long>(ms.algorithm);
  info[4] = ms.cr_num;
  info[5] = ms.cr_den;
  info[6] = static_cast<long long>(ms.counts.size());
  info[7] = static_cast<long long>(ms.coeffs.size());
  info[8] = static_cast<long long>(ms.side.size());
  info[9] = b.target;
  info[10] = b.actual;
  *threshold = ms.threshold;
}

const char* ref_ms_warning(void* p) { return static_cast<Handle*>(p)->warning.c_str(); }

void ref_ms_counts(void* p, uint16_t* out) {
  const auto& v = static_cast<Handle*>(p)->ms.counts;
  std::memcpy(out, v.data(), v.size() * sizeof(uint16_t));
}
void ref_ms_coeffs(void* p, double* out) {
  const auto& v = static_cast<Handle*>(p)->ms.coeffs;
  std::memcpy(out, v.data(), v.size() * sizeof(double));
}
void ref_ms_side(void* p, double* out) {
  const auto& v = static_cast<Handle*>(p)->ms.side;
  std::memcpy(out, v.data(), v.size() * sizeof(double));
}

// abcs::decode_idct (recon.hpp:55). out has cropped_h*cropped_w entries.
int ref_decode(void* p, double* out) {
  return guarded([&] {
    const abcs::PixelImage img = abcs::decode_idct(static_cast<Handle*>(p)->ms);
    std::memcpy(out, img.data.data(), img.data.size() * sizeof(double));
  });
}

// abcs::reconstruct (recon.hpp:87-88). method: 0 idct, 5 ida (ReconMethod order).
// trace: (iters+1) rows of [iteration, residual_norm, sigma, psnr]; ref_px optional.
int ref_reconstruct(void* p, int method, int iters, double damping, double k, double dblock,
                    const uint8_t* ref_px, int ref_h, int ref_w, double* out, double* trace,
                    int* trace_rows, int* div_iter) {
  return guarded(
      [&] {
        abcs::ReconConfig cfg;
        cfg.method = static_cast<abcs::ReconMethod>(method);
        cfg.iterations = iters;
        cfg.damping = damping;
        cfg.denoiser.name = "dct_threshold";
        cfg.denoiser.params["k"] = k;
        cfg.denoiser.params["block"] = dblock;
        abcs::PixelImage refimg;
        if (ref_px) refimg = to_image(ref_px, ref_h, ref_w);
        const auto res =
            abcs::reconstruct(static_cast<Handle*>(p)->ms, cfg, ref_px ? &refimg : nullptr);
        std::memcpy(out, res.image.data.data(), res.image.data.size() * sizeof(double));
        if (trace) {
          for (size_t i = 0; i < res.trace.size(); ++i) {
            trace[4 * i + 0] = res.trace[i].iteration;
            trace[4 * i + 1] = res.trace[i].residual_norm;
            trace[4 * i + 2] = res.trace[i].sigma;
            trace[4 * i + 3] = res.trace[i].psnr_db;
          }
        }
        if (trace_rows) *trace_rows = static_cast<int>(res.trace.size());
      },
      div_iter);
}

// abcs::largest_remainder_allocate (sensing.hpp:119-121).
int ref_allocate(const double* w, int n, long long budget, const int* caps, int* out) {
  return guarded([&] {
    std::vector<double> wv(w, w + n);
    std::vector<int> cv(caps, caps + n);
    const auto a = abcs::largest_remainder_allocate(wv, budget, cv);
    std::memcpy(out, a.data(), a.size() * sizeof(int));
  });
}

// abcs::bbv_measure (sensing.hpp:104). params: [stride, offset, per_side, phase1_total, n_side]
int ref_bbv_measure(const uint8_t* px, int h, int w, int block, uint32_t num, uint32_t den,
                    long long* params, double* variation, double* side, long long side_cap) {
  return guarded([&] {
    const auto b = abcs::bbv_measure(to_image(px, h, w),
                                     make_cfg(block, num, den, 1, 0, 0.0));
    params[0] = b.stride;
    params[1] = b.offset;
    params[2] = b.per_side;
    params[3] = b.phase1_total;
    params[4] = static_cast<long long>(b.side_values.size());
    std::memcpy(variation, b.variation.data(), b.variation.size() * sizeof(double));
    if (side && static_cast<long long>(b.side_values.size()) <= side_cap) {
      std::memcpy(side, b.side_values.data(), b.side_values.size() * sizeof(double));
    }
  });
}

// abcs::allocate_bbv (sensing.hpp:105-106): phase2 out, [shared_overhead, target] in info.
int ref_allocate_bbv(const double* variation, int n_blocks, long long stride, int offset,
                     int per_side, long long phase1_total, long long total_budget, int block,
                     int* phase2, long long* info) {
  return guarded([&] {
    abcs::BbvParams b;
    b.stride = stride;
    b.offset = offset;
    b.per_side = per_side;
    b.phase1_total = phase1_total;
    b.variation.assign(variation, variation + n_blocks);
    const auto plan = abcs::allocate_bbv(b, total_budget, n_blocks, block);
    std::memcpy(phase2, plan.phase2.data(), plan.phase2.size() * sizeof(int));
    info[0] = plan.shared_overhead;
    info[1] = plan.target;
  });
}

double ref_dd_threshold(int h, uint32_t num, uint32_t den) {
  return abcs::dd_threshold(h, num, den);
}

int ref_parse_ratio(const char* text, uint32_t* num, uint32_t* den) {
  return guarded([&] {
    auto [n, d] = abcs::SensingConfig::parse_ratio(text);
    *num = n;
    *den = d;
  });
}

void ref_zigzag(int block, int* index) {
  const auto zz = abcs::zigzag_order(block);
  std::memcpy(index, zz.index.data(), zz.index.size() * sizeof(int));
}

// abcs::dct2 / idct2 (dct.hpp:30-31)
void ref_dct2(const double* in, int block, double* out) {
  const auto v = abcs::dct2(std::vector<double>(in, in + block * block), block);
  std::memcpy(out, v.data(), v.size() * sizeof(double));
}
void ref_idct2(const double* in, int block, double* out) {
  const auto v = abcs::idct2(std::vector<double>(in, in + block * block), block);
  std::memcpy(out, v.data(), v.size() * sizeof(double));
}

// abcs::denoise (denoise.hpp:31)
int ref_denoise(const double* field, int h, int w, double sigma, double k, double dblock,
                double* out) {
  return guarded([&] {
    abcs::PixelImage img(h, w);
    std::memcpy(img.data.data(), field, img.data.size() * sizeof(double));
    abcs::DenoiserSpec spec;
    spec.params["k"] = k;
    spec.params["block"] = dblock;
    const auto d = abcs::denoise(spec, img, sigma);
    std::memcpy(out, d.data.data(), d.data.size() * sizeof(double));
  });
}

// SensingOperator forward / adjoint (operators.hpp:35-39) for the operator of handle p.
int ref_op_forward(void* p, const double* field, double* y) {
  return guarded([&] {
    const auto op = abcs::SensingOperator::from(static_cast<Handle*>(p)->ms);
    const auto v = op.forward(std::span<const double>(field, op.field_size()));
    std::memcpy(y, v.data(), v.size() * sizeof(double));
  });
}
int ref_op_adjoint(void* p, const double* y, double* field) {
  return guarded([&] {
    const auto op = abcs::SensingOperator::from(static_cast<Handle*>(p)->ms);
    const auto v = op.adjoint(std::span<const double>(y, op.measurements()));
    std::memcpy(field, v.data(), v.size() * sizeof(double));
  });
}

// abcs::make_test_image (synth.hpp:15), as u8 (the scenes are integer valued).
int ref_make_test_image(const char* name, int size, uint8_t* out) {
  return guarded([&] {
    const auto img = abcs::make_test_image(name, size);
    for (size_t i = 0; i < img.data.size(); ++i) out[i] = static_cast<uint8_t>(img.data[i]);
  });
}

// CPU baseline harness: abcs::sense + abcs::reconstruct on each of n images
// (u8, contiguous h*w each) across `threads` std::threads on disjoint images —
// the reference is reentrant. method 0 = idct, 5 = ida.
// Writes the reconstructed (cropped) image of each as f32 into out (nullable).
int ref_sense_reconstruct_batch(const uint8_t* imgs, int n, int h, int w, int block,
                                uint32_t num, uint32_t den, int algo, int method, int iters,
                                int threads, float* out) {
  std::atomic<int> next{0};
  std::atomic<int> status{OK};
  std::string first_err;
  const long long hw = static_cast<long long>(h) * w;
  const long long out_px =
      static_cast<long long>(h / block) * block * static_cast<long long>(w / block) * block;
  auto worker = [&] {
    for (;;) {
      const int i = next.fetch_add(1);
      if (i >= n || status.load() != OK) return;
      const int st = guarded([&] {
        const auto cfg = make_cfg(block, num, den, algo, 0, 0.0);
        const auto ms = abcs::sense(to_image(imgs + i * hw, h, w), cfg);
        abcs::ReconConfig rc;
        rc.method = static_cast<abcs::ReconMethod>(method);
        rc.iterations = iters;
        const auto res = abcs::reconstruct(ms, rc);
        if (out) {
          for (long long j = 0; j < out_px; ++j) out[i * out_px + j] = static_cast<float>(res.image.data[j]);
        }
      });
      if (st != OK) status.store(st);
    }
  };
  if (threads <= 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
  }
  return status.load();
}

// The reference bench's per-cell work (tools/abcs_main.cpp:234-251) split into its two timed
// phases over a batch: abcs::sense of every image, then abcs::reconstruct of every measurement set
// (Idct, or Ida with `iters` iterations and the default dct_threshold denoiser, recon.cpp:199-259),
// each phase spread over `threads` host threads on disjoint images (the reference is reentrant).
// Wall seconds of each phase are returned; the payloads are not copied out.
int ref_bench_phases(const uint8_t* imgs, int n, int h, int w, int block, uint32_t num, uint32_t den, int algo,
                     int method, int iters, int threads, double* sense_sec, double* recon_sec) {
  std::vector<abcs::MeasurementSet> sets(static_cast<size_t>(n));
  std::atomic<int> status{OK};
  const long long hw = static_cast<long long>(h) * w;
  auto run = [&](auto&& body) {
    std::atomic<int> next{0};
    auto worker = [&] {
      for (;;) {
        const int i = next.fetch_add(1);
        if (i >= n || status.load() != OK) return;
        const int st = guarded([&] { body(i); });
        if (st != OK) status.store(st);
      }
    };
    const auto t0 = std::chrono::steady_clock::now();
    if (threads <= 1) {
      worker();
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
      for (auto& th : pool) th.join();
    }
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  const auto cfg = make_cfg(block, num, den, algo, 0, 0.0);
  const double ts = run([&](int i) { sets[i] = abcs::sense(to_image(imgs + i * hw, h, w), cfg); });
  if (status.load() != OK) return status.load();
  abcs::ReconConfig rc;
  rc.method = static_cast<abcs::ReconMethod>(method);
  rc.iterations = iters;
  const double tr = run([&](int i) { (void)abcs::reconstruct(sets[i], rc); });
  if (sense_sec) *sense_sec = ts;
  if (recon_sec) *recon_sec = tr;
  return status.load();
}

}  // extern "C"
