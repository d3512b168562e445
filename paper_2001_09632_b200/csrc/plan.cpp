// Host-side logic of the ABCS path: config validation and every derivation
// abcs::sense makes before touching a pixel, plus parse_ratio, dd_threshold,
// zigzag tables and the host synthetic generator. No GPU needed; the CPU test
// suite checks each function against the reference library (oracle/_ref).
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "internal.h"
#include "synth_gen.h"

namespace abcs_b200 {

static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
void clear_error() { g_last_error.clear(); }

}  // namespace abcs_b200

using abcs_b200::set_error;

extern "C" {

int abcs_abi_version(void) { return ABCS_B200_ABI_VERSION; }

const char* abcs_last_error(void) { return abcs_b200::g_last_error.c_str(); }

// SensingConfig::parse_ratio (sensing.cpp:46-80): "0.1" or "1/10" -> lowest terms.
int abcs_parse_ratio(const char* text_c, uint32_t* num_out, uint32_t* den_out) {
  if (!text_c || !num_out || !den_out) return set_error(ABCS_ERR_INVALID_ARGUMENT, "null argument");
  const std::string text(text_c);
  const std::string err = "cannot parse ratio: '" + text + "'";
  bool bad = false;
  auto digits = [&](const std::string& s) -> unsigned long long {
    if (s.empty() || s.size() > 9) { bad = true; return 0; }
    unsigned long long v = 0;
    for (char c : s) {
      if (c < '0' || c > '9') { bad = true; return 0; }
      v = v * 10 + static_cast<unsigned long long>(c - '0');
    }
    return v;
  };
  unsigned long long num = 0, den = 1;
  const size_t slash = text.find('/');
  if (slash != std::string::npos) {
    num = digits(text.substr(0, slash));
    if (bad) return set_error(ABCS_ERR_INVALID_ARGUMENT, err);
    den = digits(text.substr(slash + 1));
  } else {
    const size_t dot = text.find('.');
    const std::string whole = (dot == std::string::npos) ? text : text.substr(0, dot);
    const std::string frac = (dot == std::string::npos) ? "" : text.substr(dot + 1);
    if (whole.empty() && frac.empty()) return set_error(ABCS_ERR_INVALID_ARGUMENT, err);
    if (frac.size() > 9) return set_error(ABCS_ERR_INVALID_ARGUMENT, err);
    unsigned long long scale = 1;
    for (size_t i = 0; i < frac.size(); ++i) scale *= 10;
    const unsigned long long w = whole.empty() ? 0 : digits(whole);
    if (bad) return set_error(ABCS_ERR_INVALID_ARGUMENT, err);
    const unsigned long long f = frac.empty() ? 0 : digits(frac);
    num = w * scale + f;
    den = scale;
  }
  if (bad || num == 0 || den == 0) return set_error(ABCS_ERR_INVALID_ARGUMENT, err);
  const unsigned long long g = std::gcd(num, den);
  num /= g;
  den /= g;
  if (num > UINT32_MAX || den > UINT32_MAX) return set_error(ABCS_ERR_INVALID_ARGUMENT, err);
  *num_out = static_cast<uint32_t>(num);
  *den_out = static_cast<uint32_t>(den);
  return ABCS_OK;
}

// dd_threshold (sensing.cpp:405-416): exact rational compares of C_F = den/num.
double abcs_dd_threshold(int32_t image_height, uint32_t cr_num, uint32_t cr_den) {
  const unsigned long long num = cr_num, den = cr_den;
  if (image_height < 384) {
    if (den <= 2 * num) return 15.0;
    if (100 * den < 333 * num) return 30.0;
    return 60.0;
  }
  if (den <= 2 * num) return 15.0;
  if (den < 10 * num) return 30.0;
  return 60.0;
}

// zigzag_order (zigzag.cpp:8-26)
int abcs_zigzag_order(int32_t block, int32_t* index) {
  if (block < 1) return set_error(ABCS_ERR_INVALID_ARGUMENT, "zigzag_order: block must be >= 1");
  const int B = block;
  int k = 0;
  for (int s = 0; s <= 2 * (B - 1); ++s) {
    const int lo = std::max(0, s - B + 1), hi = std::min(s, B - 1);
    if (s % 2 == 0) {
      for (int r = hi; r >= lo; --r) index[k++] = r * B + (s - r);
    } else {
      for (int r = lo; r <= hi; ++r) index[k++] = r * B + (s - r);
    }
  }
  return ABCS_OK;
}

int abcs_sense_plan_init(const abcs_sensing_config* cfg, int32_t height, int32_t width,
                         abcs_sense_plan* p) {
  if (!cfg || !p) return set_error(ABCS_ERR_INVALID_ARGUMENT, "null argument");
  std::memset(p, 0, sizeof(*p));
  // SensingConfig::validate (sensing.cpp:32-39)
  if (cfg->block < 2 || cfg->block > 255)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "block size must be in [2, 255]");
  if (cfg->cr_num == 0 || cfg->cr_den == 0)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "C_R must be positive");
  if (cfg->cr_num > cfg->cr_den) return set_error(ABCS_ERR_INVALID_ARGUMENT, "C_R must be in (0, 1]");
  if (cfg->has_threshold && cfg->threshold < 0)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "threshold must be >= 0");
  if (cfg->algorithm < 0 || cfg->algorithm > 2)
    return set_error(ABCS_ERR_LOGIC, "sense: unknown algorithm");
  // make_grid (image.cpp:106-116)
  const int B = cfg->block;
  if (B > height || B > width)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "block size exceeds image dimensions");
  p->height = height;
  p->width = width;
  p->block = B;
  p->rows = height / B;
  p->cols = width / B;
  p->n_blocks = p->rows * p->cols;
  p->algorithm = cfg->algorithm;
  p->cr_num = cfg->cr_num;
  p->cr_den = cfg->cr_den;
  const unsigned long long num = cfg->cr_num, den = cfg->cr_den;
  const long long npx = static_cast<long long>(p->n_blocks) * B * B;
  // target_measurements (sensing.cpp:41-44)
  p->target = static_cast<long long>(num * static_cast<unsigned long long>(npx) / den);
  const long long L = static_cast<long long>(den / num);  // cf_floor
  const long long dd_phase1 = static_cast<long long>(B) * B * static_cast<long long>(num) / (2ULL * den);

  int used = cfg->algorithm;
  if (used == ABCS_ALGO_BBV) {  // sensing.cpp:445-451
    if (num == den) {
      used = ABCS_ALGO_ZZ;
      p->fallback = ABCS_FALLBACK_BBV_FULL_RATE;
    } else if (L > B) {
      used = ABCS_ALGO_ZZ;
      p->fallback = ABCS_FALLBACK_BBV_CF_EXCEEDS_BLOCK;
    }
  } else if (used == ABCS_ALGO_DD && dd_phase1 == 0) {  // sensing.cpp:461-465
    used = ABCS_ALGO_ZZ;
    p->fallback = ABCS_FALLBACK_DD_PHASE1_ZERO;
  }
  p->algorithm_used = used;
  const long long bb = static_cast<long long>(B) * B;

  if (used == ABCS_ALGO_ZZ) {  // sense_zz + balanced_counts (sensing.cpp:181-190,231-237)
    p->threshold = 0.0;
    p->zz_per_block = p->target / p->n_blocks;
    p->zz_extra = p->target % p->n_blocks;
    long long total = 0;
    // counts[i] = min(per + (i < extra), B^2); the last block holds `per` unless capped
    if (p->zz_per_block >= bb) {
      total = bb * p->n_blocks;
    } else {
      total = p->target;  // per < B^2 so per+1 <= B^2: nothing capped
    }
    p->coeffs_per_image = total;
    p->zz_last_zero = (std::min<long long>(p->zz_per_block + (p->n_blocks - 1 < p->zz_extra ? 1 : 0), bb) == 0);
    p->cap = 0;
  } else if (used == ABCS_ALGO_BBV) {
    // bbv_measure parameters (sensing.cpp:243-256)
    p->bbv_stride = L;
    p->bbv_offset = static_cast<int32_t>(L / 2);
    p->bbv_per_side = (L > B) ? 0 : static_cast<int32_t>(B / L);
    const long long extent = static_cast<long long>(p->rows) * B + static_cast<long long>(p->cols) * B;
    p->bbv_phase1_total = 2LL * p->bbv_per_side * p->n_blocks + (extent + L - 1) / L;
    int valid = 0;
    for (int j = 0; j < p->bbv_per_side; ++j) {  // sensing.cpp:260-264
      const long long pos = p->bbv_offset + static_cast<long long>(j) * L;
      if (!(pos < 1 || pos + 1 > B)) ++valid;
    }
    p->bbv_valid_probes = valid;
    p->side_per_image = static_cast<long long>(valid) * (2LL * p->n_blocks + p->cols + p->rows);
    // allocate_bbv (sensing.cpp:303-319)
    if (p->target <= p->bbv_phase1_total)
      return set_error(ABCS_ERR_INVALID_ARGUMENT,
                       "allocate_bbv: measurement budget does not cover the phase-1 probes (M <= M_BBV)");
    p->cap = static_cast<int32_t>(bb - 2LL * p->bbv_per_side);
    if (p->cap < 0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "allocate_bbv: probes exceed block capacity");
    p->alloc_budget = p->target - p->bbv_phase1_total;
    if (p->alloc_budget > static_cast<long long>(p->cap) * p->n_blocks)  // sensing.cpp:124
      return set_error(ABCS_ERR_INVALID_ARGUMENT, "allocate: budget exceeds capacity");
    p->count_base = 0;
    p->coeffs_per_image = p->alloc_budget;
    p->threshold = cfg->has_threshold ? cfg->threshold : 0.0;  // apply_plan: value_or(0.0)
  } else {  // DD (sensing.cpp:323-384)
    p->dd_phase1 = static_cast<int32_t>(dd_phase1);
    p->threshold = cfg->has_threshold ? cfg->threshold
                                      : abcs_dd_threshold(height, cfg->cr_num, cfg->cr_den);
    p->cap = static_cast<int32_t>(bb - dd_phase1);
    p->alloc_budget = static_cast<long long>(p->n_blocks) * dd_phase1;
    p->count_base = static_cast<int32_t>(dd_phase1);
    p->coeffs_per_image = 2LL * p->n_blocks * dd_phase1;
  }
  // measurement_budget (sensing.cpp:472-487)
  p->budget_actual = p->coeffs_per_image;
  if (used == ABCS_ALGO_BBV) {
    if (L >= 1 && L <= B) {
      const long long per_side = B / L;
      const long long extent = static_cast<long long>(p->rows) * B + static_cast<long long>(p->cols) * B;
      p->budget_actual += 2 * per_side * p->n_blocks + (extent + L - 1) / L;
    }
  }
  return ABCS_OK;
}

int abcs_synth_generate_host(const abcs_synth_spec* spec, int64_t first_index, int32_t n_images,
                             uint8_t* out) {
  if (!spec || !out || n_images < 0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad synth arguments");
  if (spec->height < 1 || spec->width < 1 || spec->n_ellipses < 0 || spec->n_ellipses > SG_MAX_ELLIPSES)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad synth spec");
  static_assert(sizeof(sg_spec) == sizeof(abcs_synth_spec), "spec layout");
  sg_spec sp;
  std::memcpy(&sp, spec, sizeof(sp));
  std::vector<sg_scene> scene(1);
  const uint64_t npx = static_cast<uint64_t>(spec->height) * spec->width;
  for (int32_t i = 0; i < n_images; ++i) {
    const uint32_t img = static_cast<uint32_t>(first_index + i);
    sg_make_scene(&sp, img, scene.data());
    uint8_t* o = out + static_cast<uint64_t>(i) * npx;
    for (uint64_t pr = 0; pr < (npx + 1) / 2; ++pr) {
      uint8_t a, b;
      sg_pixel_pair(&sp, scene.data(), img, pr, &a, &b);
      o[2 * pr] = a;
      if (2 * pr + 1 < npx) o[2 * pr + 1] = b;
    }
  }
  return ABCS_OK;
}

}  // extern "C"
