/* TEST INFRASTRUCTURE ONLY — the CPU oracle, never the product.
 *
 * Plain-C restatement of the reference's ABCS hot path
 * (/root/reference/proj/core/src/{dct,zigzag,sensing,operators,recon,denoise,metrics}.cpp),
 * one function per reference routine, each citing the file:line it follows.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it. It is pinned against the reference itself
 * (oracle/_ref/libabcs_ref.so, built from the reference sources by
 * oracle/Makefile) by tests/test_oracle_vs_reference.py and against the
 * committed golden fixtures in tests/golden/.
 *
 * Status codes match include/abcs_b200.h: 0 ok, 1 invalid argument,
 * 2 format error, 3 divergence, 5 logic error.
 */
#ifndef ABCS_ORACLE_H
#define ABCS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* info[] slots written by o_sense */
enum {
  O_INFO_ALGO = 0,      /* algorithm actually used (after fallbacks) */
  O_INFO_NCOEFFS = 1,   /* payload length */
  O_INFO_NSIDE = 2,     /* side-data length */
  O_INFO_FALLBACK = 3,  /* 1 when a fallback to zz fired */
  O_INFO_ROWS = 4,
  O_INFO_COLS = 5,
  O_INFO_TARGET = 6,    /* measurement_budget().target */
  O_INFO_ACTUAL = 7,    /* measurement_budget().actual */
  O_INFO_SLOTS = 8
};

const char* o_last_error(void);

void o_basis(int B, double* basis);
void o_zigzag(int B, int* index);
void o_dct_forward(const double* basis, int B, const double* px, double* coef);
void o_dct_inverse(const double* basis, int B, const double* coef, double* px);

int o_largest_remainder(const double* w, int n, long long budget, const int* caps, int* out);
double o_dd_threshold(int height, uint32_t num, uint32_t den);

int o_sense(const uint8_t* img, int H, int W, int B, uint32_t num, uint32_t den, int algo,
            int has_thr, double thr, uint16_t* counts, double* coeffs, double* side,
            long long* info, double* threshold_out);

int o_bbv_measure(const uint8_t* img, int H, int W, int B, uint32_t num, uint32_t den,
                  long long* params, double* variation, double* side);

int o_adjoint(int rows, int cols, int B, const uint16_t* counts, const double* y, double* field);
int o_forward(int rows, int cols, int B, const uint16_t* counts, const double* field, double* y);
int o_decode(int rows, int cols, int B, const uint16_t* counts, const double* y,
             long long n_coeffs, double* out);

int o_denoise_dct(const double* field, int H, int W, double threshold, int block, double* out);

int o_reconstruct_ida(int rows, int cols, int B, const uint16_t* counts, const double* y,
                      long long n_coeffs, int iters, double damping, double k, int dblock,
                      const uint8_t* ref, int ref_h, int ref_w, double* out, double* trace,
                      int* div_iter);

double o_psnr(const double* ref, const double* test, long long n);
double o_ssim(const double* ref, const double* test, int H, int W);

#ifdef __cplusplus
}
#endif
#endif
