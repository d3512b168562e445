// Seeded synthetic scene generator for the BASELINE workloads.
//
// The reference ships no generator for these workloads (its synth.cpp scenes
// differ), so this is our own fixed definition, recorded in DESIGN.md:
//   * RNG: Philox4x32-10 keyed by the 64-bit seed; counter = (lo, hi, image, domain).
//   * uniforms: 53-bit mapping (((a<<32)|b) >> 11) * 2^-53 (idiom of synth.cpp:15-20).
//   * background: sum of 4 linear gradients a*c/W + b*r/H + c0, a,b ~ U(-64,64), c0 ~ U(0,64).
//   * E filled rotated ellipses painted in order: centre ~ U(W) x U(H), semi-axes
//     ~ U(H/64, H/4), angle ~ U(0, pi), intensity ~ U(0, 255).
//   * noise: Box-Muller N(0, sigma^2) per pixel; round half away from zero; clip [0,255].
//   * video: one base scene; frame f shifted by (dx,dy) ~ U{-8..8} with edge
//     replication; per-frame noise.
//
// The same source runs on the host (gcc/g++, -ffp-contract=off) and on the device
// (explicit __d*_rn intrinsics, so nvcc cannot contract into FMAs); only IEEE
// correctly-rounded +,-,*,/,sqrt and our own polynomial log/sincos are used, so
// host and device produce identical bytes (checked by a hash in the GPU tests).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define SG_HD __host__ __device__ __forceinline__
#else
#define SG_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define SG_ADD(a, b) __dadd_rn((a), (b))
#define SG_SUB(a, b) __dsub_rn((a), (b))
#define SG_MUL(a, b) __dmul_rn((a), (b))
#define SG_DIV(a, b) __ddiv_rn((a), (b))
#define SG_SQRT(a) __dsqrt_rn((a))
#define SG_FLOOR(a) floor((a))
#define SG_AS_U64(d) ((uint64_t)__double_as_longlong((d)))
#define SG_FROM_U64(u) __longlong_as_double((long long)(u))
#else
#include <math.h>
#include <string.h>
#define SG_ADD(a, b) ((a) + (b))
#define SG_SUB(a, b) ((a) - (b))
#define SG_MUL(a, b) ((a) * (b))
#define SG_DIV(a, b) ((a) / (b))
#define SG_SQRT(a) sqrt((a))
#define SG_FLOOR(a) floor((a))
SG_HD uint64_t sg_as_u64(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
SG_HD double sg_from_u64(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
#define SG_AS_U64(d) sg_as_u64((d))
#define SG_FROM_U64(u) sg_from_u64((u))
#endif

#define SG_MAX_ELLIPSES 256

typedef struct {
  int32_t height, width;   // frame size
  int32_t n_ellipses;
  int32_t video;           // 1: frames are shifted copies of one base scene
  int32_t max_shift;       // video translation bound (8)
  int32_t pad_;
  double noise_sigma;
  uint64_t seed;
} sg_spec;

typedef struct {
  double cx, cy, cs, sn, ia2, ib2, value;
  int32_t rmin, rmax, cmin, cmax;  // bounding box (inclusive), conservative
} sg_ellipse;

typedef struct {
  double ga[4], gb[4], gc[4];
  int32_t dx, dy;  // video shift
  int32_t n_ellipses;
  int32_t pad_;
  sg_ellipse e[SG_MAX_ELLIPSES];
} sg_scene;

// ---- Philox4x32-10 ----------------------------------------------------------
SG_HD void sg_philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int i = 0; i < 10; ++i) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c[1] ^ k0;
    const uint32_t n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

SG_HD double sg_u53(uint32_t a, uint32_t b) {
  const uint64_t v = (((uint64_t)a << 32) | b) >> 11;
  return SG_MUL((double)v, 1.1102230246251565e-16);  // 2^-53
}

// domain-separated uniform stream: draw j of (image, domain)
SG_HD double sg_uniform(uint64_t seed, uint32_t image, uint32_t domain, uint32_t j) {
  uint32_t c[4] = {j, 0u, image, domain};
  sg_philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  return sg_u53(c[0], c[1]);
}

SG_HD double sg_lerp(double lo, double hi, double u) { return SG_ADD(lo, SG_MUL(u, SG_SUB(hi, lo))); }

// natural log for x in (0, 1], polynomial only (identical on host and device)
SG_HD double sg_log(double x) {
  const uint64_t bits = SG_AS_U64(x);
  const int e = (int)((bits >> 52) & 0x7ff) - 1022;
  const double m = SG_FROM_U64((bits & 0x800FFFFFFFFFFFFFull) | (1022ull << 52));  // [0.5,1)
  const double s = SG_DIV(SG_SUB(m, 1.0), SG_ADD(m, 1.0));
  const double s2 = SG_MUL(s, s);
  double acc = 0.0;
  for (int k = 41; k >= 1; k -= 2) acc = SG_ADD(SG_DIV(1.0, (double)k), SG_MUL(acc, s2));
  const double lnm = SG_MUL(2.0, SG_MUL(s, acc));
  return SG_ADD(lnm, SG_MUL((double)e, 0.6931471805599453));
}

// sin and cos of t for t in [0, 2*pi), polynomial only
SG_HD void sg_sincos(double t, double* sn, double* cs) {
  const double half_pi = 1.5707963267948966;
  double q = SG_FLOOR(SG_ADD(SG_DIV(t, half_pi), 0.5));
  const double r = SG_SUB(t, SG_MUL(q, half_pi));  // |r| <= pi/4 (+ rounding)
  const double r2 = SG_MUL(r, r);
  double s = 0.0, c = 0.0;
  // Taylor to degree 21/20; |r| <= 0.79 so the tail is < 1e-20
  double term_s = r, term_c = 1.0;
  s = r;
  c = 1.0;
  for (int k = 1; k <= 10; ++k) {
    term_s = SG_DIV(SG_MUL(SG_MUL(term_s, r2), -1.0), (double)((2 * k) * (2 * k + 1)));
    term_c = SG_DIV(SG_MUL(SG_MUL(term_c, r2), -1.0), (double)((2 * k - 1) * (2 * k)));
    s = SG_ADD(s, term_s);
    c = SG_ADD(c, term_c);
  }
  const int qi = ((int)q) & 3;
  if (qi == 0) { *sn = s; *cs = c; }
  else if (qi == 1) { *sn = c; *cs = -s; }
  else if (qi == 2) { *sn = -s; *cs = -c; }
  else { *sn = -c; *cs = s; }
}

// Scene parameters for image `image` (host side; the device gets a copy).
SG_HD void sg_make_scene(const sg_spec* sp, uint32_t image, sg_scene* sc) {
  const double H = (double)sp->height, W = (double)sp->width;
  const uint32_t scene_id = sp->video ? 0u : image;
  uint32_t j = 0;
  for (int g = 0; g < 4; ++g) {
    sc->ga[g] = sg_lerp(-64.0, 64.0, sg_uniform(sp->seed, scene_id, 1u, j++));
    sc->gb[g] = sg_lerp(-64.0, 64.0, sg_uniform(sp->seed, scene_id, 1u, j++));
    sc->gc[g] = sg_lerp(0.0, 64.0, sg_uniform(sp->seed, scene_id, 1u, j++));
  }
  int n = sp->n_ellipses;
  if (n > SG_MAX_ELLIPSES) n = SG_MAX_ELLIPSES;
  if (n < 0) n = 0;
  sc->n_ellipses = n;
  for (int i = 0; i < n; ++i) {
    sg_ellipse* e = &sc->e[i];
    e->cx = sg_lerp(0.0, W, sg_uniform(sp->seed, scene_id, 1u, j++));
    e->cy = sg_lerp(0.0, H, sg_uniform(sp->seed, scene_id, 1u, j++));
    const double a = sg_lerp(SG_DIV(H, 64.0), SG_DIV(H, 4.0), sg_uniform(sp->seed, scene_id, 1u, j++));
    const double b = sg_lerp(SG_DIV(H, 64.0), SG_DIV(H, 4.0), sg_uniform(sp->seed, scene_id, 1u, j++));
    const double th = sg_lerp(0.0, 3.141592653589793, sg_uniform(sp->seed, scene_id, 1u, j++));
    e->value = sg_lerp(0.0, 255.0, sg_uniform(sp->seed, scene_id, 1u, j++));
    sg_sincos(th, &e->sn, &e->cs);
    e->ia2 = SG_DIV(1.0, SG_MUL(a, a));
    e->ib2 = SG_DIV(1.0, SG_MUL(b, b));
    const double ext = (a > b ? a : b) + 2.0;
    e->rmin = (int32_t)SG_FLOOR(SG_SUB(e->cy, ext));
    e->rmax = (int32_t)SG_FLOOR(SG_ADD(e->cy, ext)) + 1;
    e->cmin = (int32_t)SG_FLOOR(SG_SUB(e->cx, ext));
    e->cmax = (int32_t)SG_FLOOR(SG_ADD(e->cx, ext)) + 1;
  }
  if (sp->video) {
    const double span = (double)(2 * sp->max_shift + 1);
    sc->dx = (int32_t)SG_FLOOR(SG_MUL(sg_uniform(sp->seed, image, 2u, 0u), span)) - sp->max_shift;
    sc->dy = (int32_t)SG_FLOOR(SG_MUL(sg_uniform(sp->seed, image, 2u, 1u), span)) - sp->max_shift;
  } else {
    sc->dx = 0;
    sc->dy = 0;
  }
}

// Noise-free scene value at base-scene pixel (r, c).
SG_HD double sg_scene_value(const sg_spec* sp, const sg_scene* sc, int r, int c) {
  const double H = (double)sp->height, W = (double)sp->width;
  const double rd = (double)r, cd = (double)c;
  for (int i = sc->n_ellipses - 1; i >= 0; --i) {  // last painted wins
    const sg_ellipse* e = &sc->e[i];
    if (r < e->rmin || r > e->rmax || c < e->cmin || c > e->cmax) continue;
    const double dx = SG_SUB(cd, e->cx), dy = SG_SUB(rd, e->cy);
    const double u = SG_ADD(SG_MUL(dx, e->cs), SG_MUL(dy, e->sn));
    const double w = SG_SUB(SG_MUL(dy, e->cs), SG_MUL(dx, e->sn));
    const double q = SG_ADD(SG_MUL(SG_MUL(u, u), e->ia2), SG_MUL(SG_MUL(w, w), e->ib2));
    if (q <= 1.0) return e->value;
  }
  double v = 0.0;
  for (int g = 0; g < 4; ++g) {
    const double t = SG_ADD(SG_ADD(SG_DIV(SG_MUL(sc->ga[g], cd), W), SG_DIV(SG_MUL(sc->gb[g], rd), H)), sc->gc[g]);
    v = SG_ADD(v, t);
  }
  return v;
}

// Two N(0,1) draws for pixel pair `pair` of image `image` (Box-Muller).
SG_HD void sg_normal2(uint64_t seed, uint32_t image, uint64_t pair, double* n0, double* n1) {
  uint32_t c[4] = {(uint32_t)pair, (uint32_t)(pair >> 32), image, 0u};
  sg_philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const double u1 = SG_SUB(1.0, sg_u53(c[0], c[1]));  // (0, 1]
  const double u2 = sg_u53(c[2], c[3]);
  const double rad = SG_SQRT(SG_MUL(-2.0, sg_log(u1)));
  double sn, cs;
  sg_sincos(SG_MUL(6.283185307179586, u2), &sn, &cs);
  *n0 = SG_MUL(rad, cs);
  *n1 = SG_MUL(rad, sn);
}

SG_HD uint8_t sg_quantize(double v) {
  double a = v < 0.0 ? -v : v;
  a = SG_FLOOR(SG_ADD(a, 0.5));  // round half away from zero
  const double r = v < 0.0 ? -a : a;
  if (r <= 0.0) return 0;
  if (r >= 255.0) return 255;
  return (uint8_t)r;
}

// Pixels 2*pair and 2*pair+1 (row-major) of frame `image`.
SG_HD void sg_pixel_pair(const sg_spec* sp, const sg_scene* sc, uint32_t image, uint64_t pair,
                         uint8_t* p0, uint8_t* p1) {
  double n0, n1;
  sg_normal2(sp->seed, image, pair, &n0, &n1);
  const uint64_t W = (uint64_t)sp->width;
  for (int h = 0; h < 2; ++h) {
    const uint64_t idx = 2 * pair + (uint64_t)h;
    int r = (int)(idx / W), c = (int)(idx % W);
    r -= sc->dy;
    c -= sc->dx;
    if (r < 0) r = 0;
    if (r > sp->height - 1) r = sp->height - 1;
    if (c < 0) c = 0;
    if (c > sp->width - 1) c = sp->width - 1;
    const double v = SG_ADD(sg_scene_value(sp, sc, r, c), SG_MUL(sp->noise_sigma, h ? n1 : n0));
    if (h) *p1 = sg_quantize(v);
    else *p0 = sg_quantize(v);
  }
}
