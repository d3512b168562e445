/* TEST INFRASTRUCTURE ONLY — the CPU oracle (see abcs_oracle.h).
 *
 * A plain-C restatement of the reference's hot path. Arithmetic is kept in the
 * reference's exact operation order (double, no FMA contraction: built with
 * -ffp-contract=off, like the reference's no--march x86-64 build), and the
 * allocator keeps the reference's x87 `long double` ranking, so results are
 * bit-identical to the reference, which tests/test_oracle_vs_reference.py
 * checks against oracle/_ref/libabcs_ref.so.
 */
#include "abcs_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* o_last_error(void) { return g_err; }

/* dct.cpp:9-21 — basis[k*B+n] = a_k cos(pi (2n+1) k / (2B)), a_0 = sqrt(1/B), a_k = sqrt(2/B). */
void o_basis(int B, double* basis) {
  const double n0 = sqrt(1.0 / B);
  const double nk = sqrt(2.0 / B);
  for (int k = 0; k < B; ++k) {
    const double scale = (k == 0) ? n0 : nk;
    for (int n = 0; n < B; ++n) {
      basis[k * B + n] = scale * cos(3.14159265358979323846 * (2.0 * n + 1.0) * k / (2.0 * B));
    }
  }
}

/* zigzag.cpp:8-26 — anti-diagonals s = 0..2B-2; even s walks r from hi down, odd s walks up. */
void o_zigzag(int B, int* index) {
  int k = 0;
  for (int s = 0; s <= 2 * (B - 1); ++s) {
    const int lo = s - B + 1 > 0 ? s - B + 1 : 0;
    const int hi = s < B - 1 ? s : B - 1;
    if (s % 2 == 0) {
      for (int r = hi; r >= lo; --r) index[k++] = r * B + (s - r);
    } else {
      for (int r = lo; r <= hi; ++r) index[k++] = r * B + (s - r);
    }
  }
}

/* dct.cpp:23-50 — tmp = C X (accumulated over r ascending), Y = tmp C^T (acc over c ascending). */
void o_dct_forward(const double* basis, int B, const double* px, double* coef) {
  double* tmp = (double*)calloc((size_t)B * B, sizeof(double));
  for (int u = 0; u < B; ++u) {
    double* trow = tmp + (size_t)u * B;
    for (int r = 0; r < B; ++r) {
      const double a = basis[u * B + r];
      const double* xrow = px + (size_t)r * B;
      for (int c = 0; c < B; ++c) trow[c] += a * xrow[c];
    }
  }
  for (int u = 0; u < B; ++u) {
    const double* trow = tmp + (size_t)u * B;
    for (int v = 0; v < B; ++v) {
      const double* brow = basis + (size_t)v * B;
      double acc = 0.0;
      for (int c = 0; c < B; ++c) acc += trow[c] * brow[c];
      coef[u * B + v] = acc;
    }
  }
  free(tmp);
}

/* dct.cpp:52-79 — tmp = C^T Y (acc over u ascending), X = tmp C (acc over v ascending). */
void o_dct_inverse(const double* basis, int B, const double* coef, double* px) {
  double* tmp = (double*)calloc((size_t)B * B, sizeof(double));
  for (int u = 0; u < B; ++u) {
    const double* yrow = coef + (size_t)u * B;
    for (int r = 0; r < B; ++r) {
      const double a = basis[u * B + r];
      double* trow = tmp + (size_t)r * B;
      for (int v = 0; v < B; ++v) trow[v] += a * yrow[v];
    }
  }
  for (int r = 0; r < B; ++r) {
    const double* trow = tmp + (size_t)r * B;
    double* xrow = px + (size_t)r * B;
    for (int c = 0; c < B; ++c) xrow[c] = 0.0;
    for (int v = 0; v < B; ++v) {
      const double a = trow[v];
      const double* brow = basis + (size_t)v * B;
      for (int c = 0; c < B; ++c) xrow[c] += a * brow[c];
    }
  }
  free(tmp);
}

/* ---- largest_remainder_allocate, sensing.cpp:110-177 -------------------- */

typedef struct {
  long double frac;
  int pos;   /* position in active */
  int block; /* active[pos] */
} o_frac;

static int frac_cmp(const void* pa, const void* pb) {
  const o_frac* a = (const o_frac*)pa;
  const o_frac* b = (const o_frac*)pb;
  /* sensing.cpp:150-154: larger fraction first, ties to the lower block index */
  if (a->frac != b->frac) return a->frac > b->frac ? -1 : 1;
  return a->block < b->block ? -1 : (a->block > b->block ? 1 : 0);
}

int o_largest_remainder(const double* w, int n, long long budget, const int* caps, int* out) {
  if (budget < 0) return fail(1, "allocate: negative budget");
  long long capacity = 0;
  for (int i = 0; i < n; ++i) {
    if (w[i] < 0 || !isfinite(w[i])) return fail(1, "allocate: weights must be finite and >= 0");
    if (caps[i] < 0) return fail(1, "allocate: negative cap");
    capacity += caps[i];
  }
  if (budget > capacity) return fail(1, "allocate: budget exceeds capacity");

  int* active = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
  int* still = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
  long long* give = (long long*)malloc(sizeof(long long) * (n > 0 ? n : 1));
  o_frac* fr = (o_frac*)malloc(sizeof(o_frac) * (n > 0 ? n : 1));
  int n_active = 0;
  for (int i = 0; i < n; ++i) {
    out[i] = 0;
    if (caps[i] > 0) active[n_active++] = i;
  }
  long long remaining = budget;
  int status = 0;
  while (remaining > 0) {
    /* sensing.cpp:134-137 — total in long double; all-zero weights split uniformly */
    long double total = 0.0L;
    for (int k = 0; k < n_active; ++k) total += w[active[k]];
    const int uniform = (total <= 0.0L);
    if (uniform) total = (long double)n_active;
    long long handed = 0;
    /* sensing.cpp:142-149 — share = remaining * w / total; whole = trunc(share) */
    for (int k = 0; k < n_active; ++k) {
      const long double wk = uniform ? 1.0L : (long double)w[active[k]];
      const long double share = (long double)remaining * wk / total;
      const long long whole = (long long)share;
      give[k] = whole;
      handed += whole;
      fr[k].frac = share - (long double)whole;
      fr[k].pos = k;
      fr[k].block = active[k];
    }
    qsort(fr, (size_t)n_active, sizeof(o_frac), frac_cmp);
    long long leftover = remaining - handed;
    for (int j = 0; j < n_active && leftover > 0; ++j, --leftover) ++give[fr[j].pos];
    /* sensing.cpp:162-171 — clamp to caps, capped blocks leave the pool */
    int n_still = 0;
    for (int k = 0; k < n_active; ++k) {
      const int i = active[k];
      const long long room = (long long)caps[i] - out[i];
      const long long taken = give[k] < room ? give[k] : room;
      out[i] += (int)taken;
      remaining -= taken;
      if (out[i] < caps[i]) still[n_still++] = i;
    }
    memcpy(active, still, sizeof(int) * (size_t)n_still);
    n_active = n_still;
    if (remaining > 0 && n_active == 0) {
      status = fail(5, "allocate: capacity exhausted before budget placed");
      break;
    }
  }
  free(active);
  free(still);
  free(give);
  free(fr);
  return status;
}

/* sensing.cpp:405-416 */
double o_dd_threshold(int height, uint32_t num, uint32_t den) {
  const unsigned long long n = num, d = den;
  if (height < 384) {
    if (d <= 2 * n) return 15.0;
    if (100 * d < 333 * n) return 30.0;
    return 60.0;
  }
  if (d <= 2 * n) return 15.0;
  if (d < 10 * n) return 30.0;
  return 60.0;
}

/* ---- sensing ------------------------------------------------------------ */

static unsigned long long gcd_u64(unsigned long long a, unsigned long long b) {
  while (b) {
    const unsigned long long t = a % b;
    a = b;
    b = t;
  }
  return a;
}

/* sensing.cpp:32-39 + image.cpp:106-116 (make_grid) */
static int validate(int H, int W, int B, uint32_t num, uint32_t den, int has_thr, double thr) {
  if (B < 2 || B > 255) return fail(1, "block size must be in [2, 255]");
  if (num == 0 || den == 0) return fail(1, "C_R must be positive");
  if (num > den) return fail(1, "C_R must be in (0, 1]");
  if (has_thr && thr < 0) return fail(1, "threshold must be >= 0");
  if (B > H || B > W) return fail(1, "block size exceeds image dimensions");
  return 0;
}

/* sensing.cpp:192-227 — per block (row-major) DCT, append the zigzag prefix. */
static long long gather_prefixes(const uint8_t* img, int W, int rows, int cols, int B,
                                 const int* counts, double* coeffs) {
  double* basis = (double*)malloc(sizeof(double) * B * B);
  int* zz = (int*)malloc(sizeof(int) * B * B);
  double* blk = (double*)malloc(sizeof(double) * B * B);
  double* coef = (double*)malloc(sizeof(double) * B * B);
  o_basis(B, basis);
  o_zigzag(B, zz);
  long long pos = 0;
  for (int br = 0; br < rows; ++br) {
    for (int bc = 0; bc < cols; ++bc) {
      for (int r = 0; r < B; ++r)
        for (int c = 0; c < B; ++c) blk[r * B + c] = img[(size_t)(br * B + r) * W + bc * B + c];
      o_dct_forward(basis, B, blk, coef);
      const int m = counts[br * cols + bc];
      for (int k = 0; k < m; ++k) coeffs[pos++] = coef[zz[k]];
    }
  }
  free(basis);
  free(zz);
  free(blk);
  free(coef);
  return pos;
}

/* sensing.cpp:181-190 */
static void balanced_counts(long long m, int n_blocks, int B, int* counts) {
  const long long per = m / n_blocks, extra = m % n_blocks;
  for (int i = 0; i < n_blocks; ++i) {
    long long c = per + (i < extra ? 1 : 0);
    const long long cap = (long long)B * B;
    counts[i] = (int)(c < cap ? c : cap);
  }
}

/* sensing.cpp:239-296. params: [L, X0, n_S, M_BBV, n_side] */
int o_bbv_measure(const uint8_t* img, int H, int W, int B, uint32_t num, uint32_t den,
                  long long* params, double* variation, double* side) {
  unsigned long long g = gcd_u64(num, den);
  if (g == 0) return fail(1, "C_R must be positive");
  num /= (uint32_t)g;
  den /= (uint32_t)g;
  int st = validate(H, W, B, num, den, 0, 0.0);
  if (st) return st;
  const int rows = H / B, cols = W / B;
  const long long L = (long long)(den / num);
  params[0] = L;
  params[1] = L / 2;
  params[2] = (L > B) ? 0 : (int)(B / L);
  const int offset = (int)(L / 2), per_side = (int)params[2];
  for (int i = 0; i < rows * cols; ++i) variation[i] = 0.0;
  params[4] = 0;
  if (per_side == 0) {
    params[3] = 0;
    return 0;
  }
  const long long extent = (long long)rows * B + (long long)cols * B;
  params[3] = 2LL * per_side * rows * cols + (extent + L - 1) / L;
  long long ns = 0;
#define PX(r, c) ((double)img[(size_t)(r) * W + (c)])
  for (int br = 0; br < rows; ++br) {
    for (int bc = 0; bc < cols; ++bc) {
      const int r0 = br * B, c0 = bc * B;
      const int bottom = (br + 1 < rows) ? r0 + B : r0 + B - 1;
      const int right = (bc + 1 < cols) ? c0 + B : c0 + B - 1;
      double sum = 0.0;
      for (int j = 0; j < per_side; ++j) {
        const long long p = offset + (long long)j * L; /* 1-based, sensing.cpp:260-264 */
        if (p < 1 || p + 1 > B) continue;
        const int a = (int)(p - 1), b = (int)p;
        const double top = fabs(PX(r0, c0 + b) - PX(r0, c0 + a));
        const double left = fabs(PX(r0 + b, c0) - PX(r0 + a, c0));
        const double bot = fabs(PX(bottom, c0 + b) - PX(bottom, c0 + a));
        const double rgt = fabs(PX(r0 + b, right) - PX(r0 + a, right));
        sum += top + left + bot + rgt;
        if (side) side[ns] = top;
        ns++;
        if (side) side[ns] = left;
        ns++;
        if (br + 1 == rows) {
          if (side) side[ns] = bot;
          ns++;
        }
        if (bc + 1 == cols) {
          if (side) side[ns] = rgt;
          ns++;
        }
      }
      variation[br * cols + bc] = sum;
    }
  }
#undef PX
  params[4] = ns;
  return 0;
}

/* sensing.cpp:472-487 */
static long long budget_actual(int algo, uint32_t num, uint32_t den, int rows, int cols, int B,
                               long long total_coeffs) {
  long long actual = total_coeffs;
  if (algo == 1) {
    const long long L = (long long)(den / num);
    if (L >= 1 && L <= B) {
      const long long per_side = B / L;
      const long long extent = (long long)rows * B + (long long)cols * B;
      actual += 2 * per_side * rows * cols + (extent + L - 1) / L;
    }
  }
  return actual;
}

/* sensing.cpp:418-470 (sense), 231-237 (sense_zz), 298-321 (allocate_bbv),
 * 323-384 (sense_dd), 386-403 (apply_plan). counts: n_blocks entries;
 * coeffs: up to n_blocks*B*B; side: up to 4*B*n_blocks. */
int o_sense(const uint8_t* img, int H, int W, int B, uint32_t num, uint32_t den, int algo,
            int has_thr, double thr, uint16_t* counts, double* coeffs, double* side,
            long long* info, double* threshold_out) {
  {
    unsigned long long g = gcd_u64(num, den); /* set_cr, sensing.cpp:89-95 */
    if (g == 0) return fail(1, "C_R must be positive");
    num /= (uint32_t)g;
    den /= (uint32_t)g;
  }
  int st = validate(H, W, B, num, den, has_thr, thr);
  if (st) return st;
  const int rows = H / B, cols = W / B, nb = rows * cols;
  const long long npx = (long long)nb * B * B;
  const long long m_target = (long long)((unsigned long long)num * npx / den);
  int* cnt = (int*)calloc((size_t)nb, sizeof(int));
  int used = algo, fallback = 0;
  double T = 0.0;
  long long n_side = 0;

  if (algo == 1) {
    if (num == den || (long long)(den / num) > B) { used = 0; fallback = 1; }
  } else if (algo == 2) {
    const long long phase1 = (long long)B * B * num / (2ULL * den);
    if (phase1 == 0) { used = 0; fallback = 1; }
  } else if (algo != 0) {
    free(cnt);
    return fail(5, "sense: unknown algorithm");
  }

  if (used == 0) {
    balanced_counts(m_target, nb, B, cnt);
    T = 0.0; /* fallback resets the threshold override (sensing.cpp:428-430) */
    if (!fallback && has_thr) T = 0.0;
  } else if (used == 1) {
    long long params[5];
    double* var = (double*)malloc(sizeof(double) * nb);
    st = o_bbv_measure(img, H, W, B, num, den, params, var, side);
    if (st) { free(var); free(cnt); return st; }
    n_side = params[4];
    if (m_target <= params[3]) {
      free(var); free(cnt);
      return fail(1, "allocate_bbv: measurement budget does not cover the phase-1 probes (M <= M_BBV)");
    }
    const int cap = B * B - 2 * (int)params[2];
    if (cap < 0) { free(var); free(cnt); return fail(1, "allocate_bbv: probes exceed block capacity"); }
    int* caps = (int*)malloc(sizeof(int) * nb);
    for (int i = 0; i < nb; ++i) caps[i] = cap;
    st = o_largest_remainder(var, nb, m_target - params[3], caps, cnt);
    free(caps);
    free(var);
    if (st) { free(cnt); return st; }
    T = has_thr ? thr : 0.0; /* apply_plan: cfg.threshold.value_or(0.0) */
  } else {
    const long long phase1 = (long long)B * B * num / (2ULL * den);
    T = has_thr ? thr : o_dd_threshold(H, num, den);
    double* basis = (double*)malloc(sizeof(double) * B * B);
    int* zz = (int*)malloc(sizeof(int) * B * B);
    double* blk = (double*)malloc(sizeof(double) * B * B);
    double* coef = (double*)malloc(sizeof(double) * B * B);
    double* sig = (double*)malloc(sizeof(double) * nb);
    o_basis(B, basis);
    o_zigzag(B, zz);
    for (int br = 0; br < rows; ++br) {
      for (int bc = 0; bc < cols; ++bc) {
        for (int r = 0; r < B; ++r)
          for (int c = 0; c < B; ++c) blk[r * B + c] = img[(size_t)(br * B + r) * W + bc * B + c];
        o_dct_forward(basis, B, blk, coef);
        int n_i = 0;
        for (long long k = 0; k < phase1; ++k)
          if (fabs(coef[zz[k]]) > T) ++n_i; /* sensing.cpp:353-355, strict */
        sig[br * cols + bc] = n_i;
      }
    }
    const int cap = (int)((long long)B * B - phase1);
    int* caps = (int*)malloc(sizeof(int) * nb);
    for (int i = 0; i < nb; ++i) caps[i] = cap;
    st = o_largest_remainder(sig, nb, nb * phase1, caps, cnt);
    for (int i = 0; i < nb; ++i) cnt[i] = (int)(uint16_t)(phase1 + cnt[i]);
    free(caps); free(sig); free(basis); free(zz); free(blk); free(coef);
    if (st) { free(cnt); return st; }
  }
  for (int i = 0; i < nb; ++i) {
    if (cnt[i] < 0 || cnt[i] > B * B) { free(cnt); return fail(1, "apply_plan: per-block count out of range"); }
    counts[i] = (uint16_t)cnt[i];
  }
  const long long K = gather_prefixes(img, W, rows, cols, B, cnt, coeffs);
  free(cnt);
  info[O_INFO_ALGO] = used;
  info[O_INFO_NCOEFFS] = K;
  info[O_INFO_NSIDE] = n_side;
  info[O_INFO_FALLBACK] = fallback;
  info[O_INFO_ROWS] = rows;
  info[O_INFO_COLS] = cols;
  info[O_INFO_TARGET] = m_target;
  info[O_INFO_ACTUAL] = budget_actual(used, num, den, rows, cols, B, K);
  *threshold_out = T;
  return 0;
}

/* ---- operators.cpp ------------------------------------------------------ */

/* operators.cpp:50-76 — scatter prefix at zigzag positions, IDCT; count-0 blocks stay 0. */
int o_adjoint(int rows, int cols, int B, const uint16_t* counts, const double* y, double* field) {
  const int W = cols * B;
  double* basis = (double*)malloc(sizeof(double) * B * B);
  int* zz = (int*)malloc(sizeof(int) * B * B);
  double* coef = (double*)malloc(sizeof(double) * B * B);
  double* blk = (double*)malloc(sizeof(double) * B * B);
  o_basis(B, basis);
  o_zigzag(B, zz);
  memset(field, 0, sizeof(double) * (size_t)rows * B * W);
  long long off = 0;
  for (int br = 0; br < rows; ++br) {
    for (int bc = 0; bc < cols; ++bc) {
      const int m = counts[br * cols + bc];
      if (m == 0) continue;
      memset(coef, 0, sizeof(double) * B * B);
      for (int k = 0; k < m; ++k) coef[zz[k]] = y[off + k];
      off += m;
      o_dct_inverse(basis, B, coef, blk);
      for (int r = 0; r < B; ++r)
        for (int c = 0; c < B; ++c) field[(size_t)(br * B + r) * W + bc * B + c] = blk[r * B + c];
    }
  }
  free(basis); free(zz); free(coef); free(blk);
  return 0;
}

/* operators.cpp:23-48 — DCT each block, emit its zigzag prefix; count-0 blocks skipped. */
int o_forward(int rows, int cols, int B, const uint16_t* counts, const double* field, double* y) {
  const int W = cols * B;
  double* basis = (double*)malloc(sizeof(double) * B * B);
  int* zz = (int*)malloc(sizeof(int) * B * B);
  double* coef = (double*)malloc(sizeof(double) * B * B);
  double* blk = (double*)malloc(sizeof(double) * B * B);
  o_basis(B, basis);
  o_zigzag(B, zz);
  long long off = 0;
  for (int br = 0; br < rows; ++br) {
    for (int bc = 0; bc < cols; ++bc) {
      const int m = counts[br * cols + bc];
      if (m == 0) continue;
      for (int r = 0; r < B; ++r)
        for (int c = 0; c < B; ++c) blk[r * B + c] = field[(size_t)(br * B + r) * W + bc * B + c];
      o_dct_forward(basis, B, blk, coef);
      for (int k = 0; k < m; ++k) y[off + k] = coef[zz[k]];
      off += m;
    }
  }
  free(basis); free(zz); free(coef); free(blk);
  return 0;
}

static int check_counts(int rows, int cols, int B, const uint16_t* counts, long long* total) {
  long long t = 0;
  for (int i = 0; i < rows * cols; ++i) {
    if (counts[i] > B * B) return fail(1, "SensingOperator: count exceeds B^2");
    t += counts[i];
  }
  *total = t;
  return 0;
}

/* recon.cpp:109-117 */
int o_decode(int rows, int cols, int B, const uint16_t* counts, const double* y,
             long long n_coeffs, double* out) {
  long long total;
  int st = check_counts(rows, cols, B, counts, &total);
  if (st) return st;
  if (total != n_coeffs) return fail(2, "decode: payload length does not match counts");
  return o_adjoint(rows, cols, B, counts, y, out);
}

/* ---- denoise.cpp:52-92 (dct_soft_threshold) ----------------------------- */
int o_denoise_dct(const double* in, int H, int W, double threshold, int block, double* out) {
  int b = block;
  if (H < b) b = H;
  if (W < b) b = W;
  if (b < 1) b = 1;
  int stride = b / 2;
  if (stride < 1) stride = 1;
  int* ro = (int*)malloc(sizeof(int) * (H / stride + 2));
  int* co = (int*)malloc(sizeof(int) * (W / stride + 2));
  int nro = 0, nco = 0;
  for (int p = 0; p + b <= H; p += stride) ro[nro++] = p;
  if (nro == 0 || ro[nro - 1] != H - b) ro[nro++] = H - b;
  for (int p = 0; p + b <= W; p += stride) co[nco++] = p;
  if (nco == 0 || co[nco - 1] != W - b) co[nco++] = W - b;
  double* basis = (double*)malloc(sizeof(double) * b * b);
  double* pix = (double*)malloc(sizeof(double) * b * b);
  double* coef = (double*)malloc(sizeof(double) * b * b);
  double* weight = (double*)calloc((size_t)H * W, sizeof(double));
  o_basis(b, basis);
  memset(out, 0, sizeof(double) * (size_t)H * W);
  for (int i = 0; i < nro; ++i) {
    const int r0 = ro[i];
    for (int j = 0; j < nco; ++j) {
      const int c0 = co[j];
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c) pix[r * b + c] = in[(size_t)(r0 + r) * W + c0 + c];
      o_dct_forward(basis, b, pix, coef);
      for (int k = 1; k < b * b; ++k) { /* DC passes through */
        const double mag = fabs(coef[k]) - threshold;
        coef[k] = (mag > 0.0) ? copysign(mag, coef[k]) : 0.0;
      }
      o_dct_inverse(basis, b, coef, pix);
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c) {
          out[(size_t)(r0 + r) * W + c0 + c] += pix[r * b + c];
          weight[(size_t)(r0 + r) * W + c0 + c] += 1.0;
        }
    }
  }
  for (long long i = 0; i < (long long)H * W; ++i) out[i] /= weight[i];
  free(ro); free(co); free(basis); free(pix); free(coef); free(weight);
  return 0;
}

/* ---- recon.cpp ---------------------------------------------------------- */

static double norm2(const double* v, long long n) { /* recon.cpp:48-52 */
  double acc = 0.0;
  for (long long i = 0; i < n; ++i) acc += v[i] * v[i];
  return sqrt(acc);
}

/* metrics.cpp:63-77 */
double o_psnr(const double* ref, const double* test, long long n) {
  double acc = 0.0;
  for (long long i = 0; i < n; ++i) {
    const double d = ref[i] - test[i];
    acc += d * d;
  }
  const double err = acc / (double)n;
  if (err == 0.0) return INFINITY;
  return 10.0 * log10(255.0 * 255.0 / err);
}

/* metrics.cpp:27-48 (windowed_mean: horizontal then vertical Gaussian pass over the
 * valid window positions) and metrics.cpp:79-116 (ssim). Returns NAN below 11x11. */
static void o_windowed_mean(const double* img, int H, int W, const double* k, double* out) {
  const int Hv = H - 10, Wv = W - 10;
  double* horiz = (double*)malloc(sizeof(double) * (size_t)H * Wv);
  for (int r = 0; r < H; ++r)
    for (int c = 0; c < Wv; ++c) {
      double acc = 0.0;
      for (int i = 0; i < 11; ++i) acc += k[i] * img[(size_t)r * W + c + i];
      horiz[(size_t)r * Wv + c] = acc;
    }
  for (int r = 0; r < Hv; ++r)
    for (int c = 0; c < Wv; ++c) {
      double acc = 0.0;
      for (int j = 0; j < 11; ++j) acc += k[j] * horiz[(size_t)(r + j) * Wv + c];
      out[(size_t)r * Wv + c] = acc;
    }
  free(horiz);
}

double o_ssim(const double* ref, const double* test, int H, int W) {
  if (H < 11 || W < 11) return NAN;
  double k[11], sum = 0.0;
  for (int i = 0; i < 11; ++i) {
    const double d = i - 5.0;
    k[i] = exp(-0.5 * d * d / (1.5 * 1.5));
    sum += k[i];
  }
  for (int i = 0; i < 11; ++i) k[i] /= sum;
  const size_t n = (size_t)H * W, nv = (size_t)(H - 10) * (W - 10);
  double* buf = (double*)malloc(sizeof(double) * (3 * n + 5 * nv));
  double *xx = buf, *yy = buf + n, *xy = buf + 2 * n, *m = buf + 3 * n;
  for (size_t i = 0; i < n; ++i) {
    xx[i] = ref[i] * ref[i];
    yy[i] = test[i] * test[i];
    xy[i] = ref[i] * test[i];
  }
  o_windowed_mean(ref, H, W, k, m);
  o_windowed_mean(test, H, W, k, m + nv);
  o_windowed_mean(xx, H, W, k, m + 2 * nv);
  o_windowed_mean(yy, H, W, k, m + 3 * nv);
  o_windowed_mean(xy, H, W, k, m + 4 * nv);
  const double C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
  double acc = 0.0;
  for (size_t i = 0; i < nv; ++i) {
    const double mx = m[i], my = m[nv + i];
    const double vx = m[2 * nv + i] - mx * mx, vy = m[3 * nv + i] - my * my, cov = m[4 * nv + i] - mx * my;
    acc += ((2.0 * mx * my + C1) * (2.0 * cov + C2)) / ((mx * mx + my * my + C1) * (vx + vy + C2));
  }
  free(buf);
  return acc / (double)nv;
}

/* recon.cpp:53-73 */
static int check_finite(const double* x, long long nx, const double* z, long long nz, int it) {
  char msg[128];
  for (long long i = 0; i < nx; ++i) {
    if (!isfinite(x[i])) {
      snprintf(msg, sizeof msg, "solver diverged (non-finite estimate) at iteration %d", it);
      return fail(3, msg);
    }
    if (fabs(x[i]) > 1e6) {
      snprintf(msg, sizeof msg, "solver diverged (|x| > 1e6) at iteration %d", it);
      return fail(3, msg);
    }
  }
  for (long long i = 0; i < nz; ++i) {
    if (!isfinite(z[i])) {
      snprintf(msg, sizeof msg, "solver diverged (non-finite residual) at iteration %d", it);
      return fail(3, msg);
    }
  }
  return 0;
}

/* recon.cpp:199-259 with method Ida: warm init_state (:119-131), damp_step Ida (:170-197),
 * finish_step (:81-93), per-iteration record (:230-234), final clamp (:255-257).
 * trace: (iters+1) rows of [iteration, ||z||, sigma, psnr]. */
int o_reconstruct_ida(int rows, int cols, int B, const uint16_t* counts, const double* y,
                      long long n_coeffs, int iters, double damping, double k, int dblock,
                      const uint8_t* ref, int ref_h, int ref_w, double* out, double* trace,
                      int* div_iter) {
  if (iters < 1) return fail(1, "iterations must be >= 1");
  if (damping < 1.0) return fail(1, "damping factor D_F must be >= 1");
  const int Hc = rows * B, Wc = cols * B;
  const long long N = (long long)Hc * Wc;
  double* refc = NULL;
  if (ref) {
    if (ref_h < Hc || ref_w < Wc) return fail(1, "reconstruct: reference smaller than decoded image");
    refc = (double*)malloc(sizeof(double) * N);
    for (int r = 0; r < Hc; ++r)
      for (int c = 0; c < Wc; ++c) refc[(size_t)r * Wc + c] = ref[(size_t)r * ref_w + c];
  }
  long long M;
  int st = check_counts(rows, cols, B, counts, &M);
  if (st) { free(refc); return st; }
  if (M != n_coeffs) { free(refc); return fail(1, "init_state: measurement vector length mismatch"); }
  double* x = (double*)malloc(sizeof(double) * N);
  double* pseudo = (double*)malloc(sizeof(double) * N);
  double* az = (double*)malloc(sizeof(double) * N);
  double* z = (double*)malloc(sizeof(double) * (M > 0 ? M : 1));
  double* ax = (double*)malloc(sizeof(double) * (M > 0 ? M : 1));
  o_adjoint(rows, cols, B, counts, y, x);
  o_forward(rows, cols, B, counts, x, ax);
  for (long long i = 0; i < M; ++i) z[i] = y[i] - ax[i];
  double sigma = norm2(y, M) / sqrt((double)M);
  int row = 0;
#define RECORD(it)                                                   \
  do {                                                               \
    if (trace) {                                                     \
      trace[4 * row + 0] = (it);                                     \
      trace[4 * row + 1] = norm2(z, M);                              \
      trace[4 * row + 2] = sigma;                                    \
      trace[4 * row + 3] = refc ? o_psnr(refc, x, N) : NAN;          \
    }                                                                \
    ++row;                                                           \
  } while (0)
  RECORD(0);
  for (int t = 0; t < iters && st == 0; ++t) {
    o_adjoint(rows, cols, B, counts, z, az); /* pseudo_data, recon.cpp:75-79 */
    for (long long i = 0; i < N; ++i) pseudo[i] = az[i] + x[i];
    if (sigma < 0) { st = fail(1, "denoise: sigma must be >= 0"); break; }
    o_denoise_dct(pseudo, Hc, Wc, k * sigma, dblock, x); /* x <- D_sigma(pseudo) */
    const double onsager = 1.0 / damping;
    o_forward(rows, cols, B, counts, x, ax);
    for (long long i = 0; i < M; ++i) z[i] = y[i] - ax[i] + onsager * z[i];
    sigma = norm2(z, M) / sqrt((double)M);
    st = check_finite(x, N, z, M, t + 1);
    if (st) {
      if (div_iter) *div_iter = t + 1;
      break;
    }
    RECORD(t + 1);
  }
#undef RECORD
  if (st == 0) {
    for (long long i = 0; i < N; ++i) out[i] = x[i] < 0.0 ? 0.0 : (x[i] > 255.0 ? 255.0 : x[i]);
  }
  free(x); free(pseudo); free(az); free(z); free(ax); free(refc);
  return st;
}
