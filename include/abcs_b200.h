/* abcs_b200.h — C ABI of the B200-native ABCS hot path (libabcs_b200.so).
 *
 * Drop-in boundary for the reference's C++ API in /root/reference/proj/core
 * (headers proj/core/include/abcs/<name>.hpp). The reference exposes no C ABI or
 * plugin registry; its public surface is the abcs:: C++ functions below. This
 * header is the thin, batched, device-pointer, stream-ordered C layer those
 * functions are re-implemented over (paper_2001_09632_b200/cpp/ is the C++
 * shim that restores the exact abcs:: signatures; INTEGRATION.md shows the
 * bindings). Plain pointers and sizes only: device buffers are caller-owned,
 * `stream` is a cudaStream_t passed as void*, no CUDA or torch types appear.
 *
 * Every call returns an abcs_status; on failure abcs_last_error() returns a
 * thread-local message. The status codes map to the reference's exceptions:
 *   ABCS_ERR_INVALID_ARGUMENT -> std::invalid_argument
 *   ABCS_ERR_FORMAT           -> abcs::FormatError        (image.hpp:12-15)
 *   ABCS_ERR_DIVERGENCE       -> abcs::DivergenceError    (recon.hpp:22-30)
 *   ABCS_ERR_LOGIC            -> std::logic_error
 * and ABCS_ERR_CUDA / ABCS_ERR_UNSUPPORTED have no reference counterpart
 * (device failure; a configuration the device path does not implement — it
 * never silently falls back to a CPU path).
 */
#ifndef ABCS_B200_H
#define ABCS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ABCS_B200_ABI_VERSION 1

typedef enum {
  ABCS_OK = 0,
  ABCS_ERR_INVALID_ARGUMENT = 1,
  ABCS_ERR_FORMAT = 2,
  ABCS_ERR_DIVERGENCE = 3,
  ABCS_ERR_CUDA = 4,
  ABCS_ERR_LOGIC = 5,
  ABCS_ERR_UNSUPPORTED = 6
} abcs_status;

/* abcs::Algorithm (sensing.hpp:12) */
typedef enum { ABCS_ALGO_ZZ = 0, ABCS_ALGO_BBV = 1, ABCS_ALGO_DD = 2 } abcs_algorithm;

/* fallback reasons of abcs::sense (sensing.cpp:445-465) */
typedef enum {
  ABCS_FALLBACK_NONE = 0,
  ABCS_FALLBACK_BBV_FULL_RATE = 1, /* C_R == 1 */
  ABCS_FALLBACK_BBV_CF_EXCEEDS_BLOCK = 2,
  ABCS_FALLBACK_DD_PHASE1_ZERO = 3
} abcs_fallback;

typedef struct abcs_ctx abcs_ctx;

/* abcs::SensingConfig (sensing.hpp:20-40). cr_num/cr_den need not be reduced. */
typedef struct {
  int32_t block;
  uint32_t cr_num;
  uint32_t cr_den;
  int32_t algorithm;     /* abcs_algorithm */
  int32_t has_threshold; /* SensingConfig::threshold engaged (DD override) */
  int32_t reserved;
  double threshold;
} abcs_sensing_config;

/* Everything abcs::sense derives from (config, image size) before touching a
 * pixel: grid (image.cpp:106-116), M (sensing.cpp:41-44), fallbacks
 * (sensing.cpp:445-465), BBV L/X0/n_S/M_BBV (sensing.cpp:243-256), allocate_bbv
 * cap/budget (sensing.cpp:303-319), DD phase1/T/cap (sensing.cpp:328-330,360),
 * measurement_budget (sensing.cpp:472-487). Computed on the host by
 * abcs_sense_plan_init; the same plan serves every image of that size. */
typedef struct {
  int32_t height, width, block;
  int32_t rows, cols, n_blocks;
  int32_t algorithm;       /* requested */
  int32_t algorithm_used;  /* MeasurementSet::algorithm after fallbacks */
  int32_t fallback;        /* abcs_fallback */
  int32_t zz_last_zero;    /* sense()'s "some blocks receive zero" warning */
  uint32_t cr_num, cr_den; /* as stored in the MeasurementSet */
  double threshold;        /* MeasurementSet::threshold */
  int64_t target;          /* M = floor(C_R * N) over the cropped grid */
  int64_t coeffs_per_image;/* K = sum(counts), identical for every image */
  int64_t side_per_image;  /* BBV side-data length */
  int64_t budget_actual;   /* measurement_budget().actual */
  int64_t bbv_stride;      /* L */
  int32_t bbv_offset;      /* X0 */
  int32_t bbv_per_side;    /* n_S */
  int64_t bbv_phase1_total;/* M_BBV */
  int32_t bbv_valid_probes;/* probes per side that stay inside the block */
  int32_t dd_phase1;       /* floor(B^2 C_R / 2) */
  int32_t cap;             /* per-block allocator cap */
  int32_t count_base;      /* added to each allocation (DD phase 1) */
  int64_t alloc_budget;    /* budget handed to largest_remainder_allocate */
  int64_t zz_per_block;    /* balanced_counts: floor(M / n_B) */
  int64_t zz_extra;        /* balanced_counts: M mod n_B */
} abcs_sense_plan;

/* abcs::ReconConfig for method Ida with the dct_threshold denoiser (recon.hpp:32-41,
 * denoise.hpp:19-27). */
typedef struct {
  int32_t iterations;      /* >= 1 */
  int32_t denoiser_block;  /* DenoiserSpec param "block" (8 supported on device) */
  double damping;          /* D_F >= 1 */
  double k;                /* DenoiserSpec param "k" (2.7) */
} abcs_ida_config;

/* abcs::ReconConfig (recon.hpp:32-41) + DenoiserSpec (denoise.hpp:19-27) for every method. */
typedef enum {
  ABCS_RECON_IDCT = 0,
  ABCS_RECON_ISTA = 1,
  ABCS_RECON_AMP = 2,
  ABCS_RECON_DAMP = 3,
  ABCS_RECON_DAMPD = 4,
  ABCS_RECON_IDA = 5
} abcs_recon_method;
typedef enum {
  ABCS_DENOISER_DCT_THRESHOLD = 0, /* params k (2.7), block (8) */
  ABCS_DENOISER_BLUR = 1,          /* param sigma_scale (25) */
  ABCS_DENOISER_IDENTITY = 2
} abcs_denoiser_kind;
typedef struct {
  int32_t method;          /* abcs_recon_method */
  int32_t iterations;      /* >= 1 */
  double damping;          /* D_F >= 1 */
  double lambda;           /* ISTA/AMP soft-threshold multiplier >= 0 */
  uint64_t seed;           /* DAMP divergence-probe seed */
  int32_t denoiser;        /* abcs_denoiser_kind */
  int32_t denoiser_block;  /* dct_threshold "block" */
  double k;                /* dct_threshold "k" */
  double sigma_scale;      /* blur "sigma_scale" */
} abcs_recon_config;

/* Seeded synthetic scene generator; mirrors csrc/synth_gen.h sg_spec. */
typedef struct {
  int32_t height, width;
  int32_t n_ellipses;
  int32_t video;
  int32_t max_shift;
  int32_t reserved;
  double noise_sigma;
  uint64_t seed;
} abcs_synth_spec;

/* ---- library / context --------------------------------------------------- */
int abcs_abi_version(void);
const char* abcs_last_error(void);
int abcs_ctx_create(int device, abcs_ctx** out);
int abcs_ctx_destroy(abcs_ctx* ctx);
/* number of kernels this ctx has launched (for bench's gpu_launches claim) */
int64_t abcs_ctx_launch_count(const abcs_ctx* ctx);

/* Opt-in per-kernel timing: with timing enabled the ctx records a CUDA event pair on
 * the launching stream around each hot kernel; abcs_ctx_kernel_times synchronizes the
 * device and returns per-kernel-name launch counts and summed/max durations (first-seen
 * order, at most `capacity` entries; *count = number of names). Enabling clears. */
typedef struct {
  char name[48];
  int64_t launches;
  double total_ms;
  double max_ms;
} abcs_kernel_time;
int abcs_ctx_kernel_timing(abcs_ctx* ctx, int32_t enable);
/* Batch calls split into up to `streams` chunks run on the ctx's pipeline streams so the
 * latency-bound phases of one chunk overlap the bandwidth-bound phases of another
 * (default 3; 1 = one stream, kernels serialised). */
int abcs_ctx_set_pipeline_streams(abcs_ctx* ctx, int32_t streams);
int abcs_ctx_kernel_times(abcs_ctx* ctx, abcs_kernel_time* out, int32_t capacity, int32_t* count);

/* ---- host-side logic (no GPU needed) -------------------------------------- */
/* SensingConfig::parse_ratio (sensing.cpp:46-80) */
int abcs_parse_ratio(const char* text, uint32_t* num, uint32_t* den);
/* dd_threshold (sensing.cpp:405-416) */
double abcs_dd_threshold(int32_t image_height, uint32_t cr_num, uint32_t cr_den);
/* zigzag_order (zigzag.cpp:8-26): index[k] = row*B + col */
int abcs_zigzag_order(int32_t block, int32_t* index);
/* config validation + every derivation of sense() for one image size */
int abcs_sense_plan_init(const abcs_sensing_config* cfg, int32_t height, int32_t width,
                         abcs_sense_plan* plan);
/* host generator (identical bytes to abcs_synth_generate) */
int abcs_synth_generate_host(const abcs_synth_spec* spec, int64_t first_index, int32_t n_images,
                             uint8_t* out);

/* ---- device hot path ------------------------------------------------------ */

/* abcs::sense (sensing.hpp:98-99) on n images of the plan's size. images: u8,
 * image i at d_images + i*image_stride, rows `pitch` bytes apart.
 * Outputs per image i: counts[i*n_blocks ..] (u16, row-major blocks),
 * offsets[i*n_blocks ..] (exclusive prefix sums of counts; nullable),
 * payload[i*K ..] (f32 zigzag prefixes, block-major), side[i*S ..] (f32 BBV
 * boundary differences; nullable when S == 0). */
int abcs_sense_batch(abcs_ctx* ctx, const abcs_sense_plan* plan, const uint8_t* d_images,
                     int64_t image_stride, int32_t pitch, int32_t n_images, uint16_t* d_counts,
                     int32_t* d_offsets, float* d_payload, float* d_side, void* stream);

/* abcs::sense followed by decode_idct of the result, fused: the decoded image
 * is computed from the same fp32 payload values the call writes (identical
 * to abcs_decode_batch on d_payload) without re-reading them from HBM.
 * d_out: image i at d_out + i*out_stride, rows out_pitch floats apart. */
int abcs_sense_decode_batch(abcs_ctx* ctx, const abcs_sense_plan* plan, const uint8_t* d_images,
                            int64_t image_stride, int32_t pitch, int32_t n_images, uint16_t* d_counts,
                            int32_t* d_offsets, float* d_payload, float* d_side, float* d_out,
                            int64_t out_stride, int32_t out_pitch, void* stream);

/* A subrate sweep: abcs_sense_decode_batch of the same images under n_plans
 * plans (the reference's bench runs sense() per --crs entry on each image,
 * tools/abcs_main.cpp:215-260). Every pointer argument indexed by plan is a
 * HOST array of n_plans device pointers (d_offsets / d_side may be NULL or hold
 * NULLs). When 2..4 plans are DD with B = 16 on the same geometry, DD phase 1
 * of all of them comes from one forward transform per block; each plan still
 * gets its own exact fixup, allocation, payload and decode, identical to
 * separate abcs_sense_decode_batch calls. Otherwise the plans run one by one. */
int abcs_sense_decode_sweep_batch(abcs_ctx* ctx, const abcs_sense_plan* plans, int32_t n_plans,
                                  const uint8_t* d_images, int64_t image_stride, int32_t pitch,
                                  int32_t n_images, uint16_t* const* d_counts, int32_t* const* d_offsets,
                                  float* const* d_payload, float* const* d_side, float* const* d_out,
                                  int64_t out_stride, int32_t out_pitch, void* stream);

/* Phase-1 weights only (bbv_measure variation / DD significance counts n_i),
 * u32 per block — exposes the pre-measurement of sensing.cpp:266-294 / :341-358. */
int abcs_sense_weights_batch(abcs_ctx* ctx, const abcs_sense_plan* plan, const uint8_t* d_images,
                             int64_t image_stride, int32_t pitch, int32_t n_images,
                             uint32_t* d_weights, float* d_side, void* stream);

/* apply_plan's gather (sensing.cpp:192-227, 386-403) from given counts and
 * offsets, fused with decode_idct (recon.cpp:109-117) when d_out is non-NULL:
 * the payload pass of a sense whose allocation was made elsewhere (a sharded
 * image: each shard gathers its block rows into its slice of the payload). */
int abcs_gather_decode_batch(abcs_ctx* ctx, int32_t rows, int32_t cols, int32_t block,
                             const uint8_t* d_images, int64_t image_stride, int32_t pitch,
                             int32_t n_images, const uint16_t* d_counts, const int32_t* d_offsets,
                             float* d_payload, int64_t payload_stride, float* d_out, int64_t out_stride,
                             int32_t out_pitch, void* stream);

/* bbv_measure (sensing.cpp:239-296) of one shard strip of an image: plan = the image's plan
 * with rows / height / n_blocks of the strip. has_below != 0: the strip is not the image's
 * bottom, and d_strip holds one more pixel row (the next strip's first) after its last block
 * row, which the bottom-side probes of that row read; side values then follow the image's
 * block-major order for these blocks (no bottom values). */
int abcs_bbv_weights_strip(abcs_ctx* ctx, const abcs_sense_plan* plan, const uint8_t* d_strip,
                           int64_t strip_stride, int32_t pitch, int32_t has_below, uint32_t* d_weights,
                           float* d_side, void* stream);

/* largest_remainder_allocate (sensing.cpp:110-177) of ONE weight vector split
 * into shards (contiguous block ranges in block order) held by different
 * devices/processes. The caller drives the rounds and the collectives between
 * the phases (paper_2001_09632_b200/sharded.py):
 *   phase 0: load d_weights (n_blocks, u32) into d_scratch; d_out[0] = 1 if a
 *            weight exceeds wmax.
 *   phase 1: d_out[0..wmax] = active-weight histogram, d_out[wmax+1] = sum of
 *            active weights, d_out[wmax+2] = active blocks   -> sum over shards.
 *   phase 2: d_in = that sum, remaining = units left: the round's class table
 *            and threshold (identical on every shard); d_out[0] = the shard's
 *            exact-tie blocks                                 -> prefix over shards.
 *   phase 3: prefix = tie blocks of the lower shards: apply and clamp;
 *            d_out[0] = units taken, d_out[1] = blocks still open -> sum.
 *   phase 4: prefix = the shard's offset in the image's payload:
 *            d_counts = base + allocation, d_offsets (nullable); d_out[0] = total.
 * d_scratch: abcs_allocate_shard_scratch_bytes(n_blocks, wmax) bytes, kept
 * across the phases; d_out: wmax + 3 int64. */
size_t abcs_allocate_shard_scratch_bytes(int32_t n_blocks, int32_t wmax);
int abcs_allocate_shard_step(abcs_ctx* ctx, int32_t phase, const uint32_t* d_weights, int32_t n_blocks,
                             int32_t wmax, int32_t cap, int32_t base, void* d_scratch, int64_t* d_out,
                             const int64_t* d_in, int64_t remaining, int64_t prefix, uint16_t* d_counts,
                             int32_t* d_offsets, void* stream);

/* largest_remainder_allocate (sensing.cpp:110-177) for n independent weight
 * vectors of n_blocks integer weights; caps per block (nullable -> uniform
 * `cap`). counts = base + allocation (u16), offsets = exclusive scan (nullable).
 * d_status[i] (nullable) receives an abcs_status per vector. */
int abcs_allocate_batch(abcs_ctx* ctx, const uint32_t* d_weights, int32_t n_blocks,
                        int32_t n_vectors, int64_t budget, const int32_t* d_caps, int32_t cap,
                        int32_t base, uint16_t* d_counts, int32_t* d_offsets, int32_t* d_status,
                        void* stream);

/* largest_remainder_allocate (sensing.cpp:110-177) for n independent vectors of small integer
 * weights (0 <= w <= wmax <= 127, n_blocks <= 4096, uniform cap): the DD phase-2 allocation,
 * one warp per vector (csrc/warp_alloc.cuh), bit-exact. counts = base + allocation (u16),
 * offsets = exclusive scan (required). d_status[i] (nullable) receives ABCS_OK, or
 * ABCS_ERR_LOGIC for a weight above wmax, a negative budget or budget > cap * n_blocks. */
int abcs_allocate_small_batch(abcs_ctx* ctx, const uint32_t* d_weights, int32_t n_blocks,
                              int32_t n_vectors, int64_t budget, int32_t cap, int32_t base,
                              int32_t wmax, uint16_t* d_counts, int32_t* d_offsets,
                              int32_t* d_status, void* stream);

/* decode_idct (recon.cpp:109-117) = SensingOperator::adjoint (operators.cpp:50-76):
 * out image i (cropped rows*B x cols*B, f32, `out_pitch` floats per row) from
 * counts/payload. offsets nullable (computed). d_format_error (nullable, per
 * image) receives ABCS_ERR_FORMAT when sum(counts) != d_payload_len[i]
 * (nullable) or ABCS_ERR_INVALID_ARGUMENT when a count exceeds B^2. */
int abcs_decode_batch(abcs_ctx* ctx, int32_t rows, int32_t cols, int32_t block,
                      const uint16_t* d_counts, const int32_t* d_offsets, const float* d_payload,
                      int64_t payload_stride, int32_t n_images, float* d_out, int64_t out_stride,
                      int32_t out_pitch, const int64_t* d_payload_len, int32_t* d_error,
                      void* stream);

/* BlockDct::forward / inverse (dct.cpp:9-79; replaces abcs::BlockDct, abcs::dct2, abcs::idct2 of
 * dct.hpp:14-31) on n_blocks row-major size x size fp64 blocks in device memory, any size >= 1.
 * Bit-identical to the reference: its basis expression (glibc cos) and summation order, no FMA.
 * inverse = 0: pixels -> coefficients; 1: coefficients -> pixels. Synchronizes `stream`. */
int abcs_block_dct_f64(abcs_ctx* ctx, int32_t size, int32_t inverse, const double* d_in, double* d_out,
                       int64_t n_blocks, void* stream);

/* SensingOperator::forward (operators.cpp:23-48) on f32 fields. */
int abcs_forward_batch(abcs_ctx* ctx, int32_t rows, int32_t cols, int32_t block,
                       const uint16_t* d_counts, const int32_t* d_offsets, const float* d_field,
                       int64_t field_stride, int32_t field_pitch, int32_t n_images, float* d_y,
                       int64_t y_stride, void* stream);

/* denoise(dct_threshold) (denoise.cpp:52-92,96-109) on f32 fields; sigma per image (host array). */
int abcs_denoise_dct_batch(abcs_ctx* ctx, const float* d_field, int32_t height, int32_t width,
                           int64_t field_stride, int32_t n_images, const double* sigma, double k,
                           int32_t block, float* d_out, void* stream);

/* reconstruct() with method Ida (recon.cpp:199-259): warm start, `iterations`
 * damp_step(Ida) steps with the dct_threshold denoiser, final clamp to [0,255].
 * d_ref (nullable): u8 reference images for the per-iteration PSNR trace.
 * d_trace (nullable): n*(iterations+1) rows of {iteration, ||z||, sigma, psnr}.
 * d_diverged (nullable): per image {first diverged iteration or 0, kind}
 * (kind 1 non-finite estimate, 2 |x| > 1e6, 3 non-finite residual). Async;
 * abcs_ida_check() turns the device record into a status after the stream syncs. */
int abcs_ida_batch(abcs_ctx* ctx, int32_t rows, int32_t cols, int32_t block,
                   const uint16_t* d_counts, const int32_t* d_offsets, const float* d_y,
                   int64_t y_stride, int32_t n_images, const abcs_ida_config* cfg,
                   const uint8_t* d_ref, int64_t ref_stride, int32_t ref_pitch, float* d_out,
                   int64_t out_stride, int32_t out_pitch, double* d_trace, int32_t* d_diverged,
                   void* stream);
int abcs_ida_check(const int32_t* h_diverged, int32_t n_images, int32_t* first_image);

/* init_state (recon.cpp:119-131) on caller-owned device state, n images at once:
 * warm != 0: x0 = A* y, z0 = y - A x0; warm == 0: x0 = 0, z0 = y. Either way
 * sigma0 = ||y|| / sqrt(M) (M = sum of counts). d_x: n*(rows*B)*(cols*B) f32,
 * d_z: n*y_stride f32, d_sigma: n f64. Replaces abcs::init_state (recon.hpp:61). */
int abcs_ida_init_state(abcs_ctx* ctx, int32_t rows, int32_t cols, int32_t block,
                        const uint16_t* d_counts, const int32_t* d_offsets, const float* d_y,
                        int64_t y_stride, int32_t n_images, int32_t warm, float* d_x, float* d_z,
                        double* d_sigma, void* stream);

/* damp_step with variant Ida (recon.cpp:170-197 + finish_step :81-93) on that state,
 * in place: pseudo = A* z + x; x <- dct_threshold(pseudo, k*sigma); z <- (y - A x) + z/D_F;
 * sigma <- ||z|| / sqrt(M). `iteration` is the state's iteration count after the step
 * (recorded in d_diverged like abcs_ida_batch). Uses cfg->damping, cfg->k,
 * cfg->denoiser_block. Replaces abcs::damp_step(.., ReconMethod::Ida, ..) (recon.hpp:67-69). */
int abcs_ida_step_state(abcs_ctx* ctx, int32_t rows, int32_t cols, int32_t block,
                        const uint16_t* d_counts, const int32_t* d_offsets, const float* d_y,
                        int64_t y_stride, int32_t n_images, const abcs_ida_config* cfg, float* d_x,
                        float* d_z, double* d_sigma, int32_t iteration, int32_t* d_diverged,
                        void* stream);

/* psnr (metrics.cpp:63-77) of f32 images against u8 references, per image (f64,
 * +inf when mse == 0): reconstruct()'s Idct trace row (recon.cpp:217-221). */
int abcs_psnr_batch(abcs_ctx* ctx, const uint8_t* d_ref, int64_t ref_stride, int32_t ref_pitch,
                    const float* d_img, int64_t img_stride, int32_t img_pitch, int32_t height,
                    int32_t width, int32_t n_images, double* d_psnr, void* stream);

/* ssim (metrics.cpp:79-116) of f32 images against u8 references, per image (f64): 11x11
 * Gaussian window (sigma 1.5), valid window positions only, fp64 statistics in the
 * reference's operation order. Images must be at least 11x11. */
int abcs_ssim_batch(abcs_ctx* ctx, const uint8_t* d_ref, int64_t ref_stride, int32_t ref_pitch,
                    const float* d_img, int64_t img_stride, int32_t img_pitch, int32_t height,
                    int32_t width, int32_t n_images, double* d_ssim, void* stream);

/* quality (metrics.cpp:63-130): mse, psnr and ssim per image (each output nullable; f64). */
int abcs_quality_batch(abcs_ctx* ctx, const uint8_t* d_ref, int64_t ref_stride, int32_t ref_pitch,
                       const float* d_img, int64_t img_stride, int32_t img_pitch, int32_t height,
                       int32_t width, int32_t n_images, double* d_mse, double* d_psnr, double* d_ssim,
                       void* stream);

/* thb / thi (metrics.cpp:126-225): full-sensing oracle decodes of u8 images. Keep the
 * M = floor(C_R N) largest-|coefficient| entries per block with balanced counts (global = 0,
 * THB) or across the image (global = 1, THI), ties to the lower zigzag index then block,
 * and invert. fp64 transforms in the reference's operation order: counts and images are
 * bit-identical to the reference. d_counts: n*n_blocks i32; d_out: f64 (cropped grid). */
int abcs_threshold_decode_batch(abcs_ctx* ctx, const abcs_sensing_config* cfg,
                                const uint8_t* d_images, int64_t image_stride, int32_t pitch,
                                int32_t height, int32_t width, int32_t n_images, int32_t global,
                                int32_t* d_counts, double* d_out, int64_t out_stride, int32_t out_pitch,
                                void* stream);

/* ---- .abcs v1 measurement container (container.cpp:58-149) ------------------
 * Layout (little-endian, packed): "ABCS" | version u16 = 1 | H u32 | W u32 | B u16 |
 * algorithm u8 | C_R num u32 | C_R den u32 | threshold f64 | n_B u32 | counts u16[n_B] |
 * coeffs f32[K] | side count u32 | side f32[S]. A batch of containers shares one plan. */
typedef struct {
  int32_t algorithm;  /* header algorithm id */
  uint32_t cr_num, cr_den;
  int32_t status;     /* ABCS_OK or ABCS_ERR_FORMAT (the reference reader's checks) */
  double threshold;
} abcs_container_info;

/* bytes of one container of this plan: 41 + 2 n_B + 4 K + 4 S */
int64_t abcs_container_size(const abcs_sense_plan* plan);
/* write_measurement_set's byte image for n sensed images, straight from the device
 * buffers of abcs_sense_batch (header from the plan; container i at d_out + i*out_stride,
 * out_stride % 4 == 0). Byte-identical to the reference writer on the same set. */
int abcs_container_pack_batch(abcs_ctx* ctx, const abcs_sense_plan* plan, const uint16_t* d_counts,
                              const float* d_payload, const float* d_side, int32_t n_images,
                              uint8_t* d_out, int64_t out_stride, void* stream);
/* read_measurement_set on the device for n containers of the plan's layout: counts,
 * payload and side into the batched buffers, plus per-container header fields and a
 * status (ABCS_ERR_FORMAT where the reference reader would throw FormatError). */
int abcs_container_unpack_batch(abcs_ctx* ctx, const abcs_sense_plan* plan, const uint8_t* d_in,
                                int64_t in_stride, int32_t n_images, uint16_t* d_counts,
                                float* d_payload, float* d_side, abcs_container_info* d_info,
                                void* stream);
/* Host: the layout of one container (header checks, counts summed for K, side count,
 * exact size) as a plan for abcs_container_unpack_batch. */
int abcs_container_parse(const uint8_t* h_bytes, int64_t size, abcs_sense_plan* plan);

/* reconstruct() (recon.cpp:199-259) for every iterative method (Ista, Amp, Damp, DampD,
 * Ida with any denoiser) and Idct; arguments as abcs_ida_batch. Ida with the 8x8
 * dct_threshold takes the fused kernel path of abcs_ida_batch. */
int abcs_reconstruct_batch(abcs_ctx* ctx, int32_t rows, int32_t cols, int32_t block,
                           const uint16_t* d_counts, const int32_t* d_offsets, const float* d_y,
                           int64_t y_stride, int32_t n_images, const abcs_recon_config* cfg,
                           const uint8_t* d_ref, int64_t ref_stride, int32_t ref_pitch, float* d_out,
                           int64_t out_stride, int32_t out_pitch, double* d_trace, int32_t* d_diverged,
                           void* stream);

/* ista_step / amp_step / damp_step (recon.cpp:133-197) on caller-owned state (layout as
 * abcs_ida_init_state), in place; `iteration` is the state's iteration count BEFORE the step
 * (the AMP first-step convention and the DAMP probe seed depend on it). */
int abcs_recon_step_state(abcs_ctx* ctx, int32_t rows, int32_t cols, int32_t block,
                          const uint16_t* d_counts, const int32_t* d_offsets, const float* d_y,
                          int64_t y_stride, int32_t n_images, const abcs_recon_config* cfg, float* d_x,
                          float* d_z, double* d_sigma, int32_t iteration, int32_t* d_diverged,
                          void* stream);

/* denoise (denoise.cpp:96-109) with any denoiser of cfg; sigma per image (host array). */
int abcs_denoise_batch(abcs_ctx* ctx, const float* d_field, int32_t height, int32_t width,
                       int64_t field_stride, int32_t n_images, const double* sigma,
                       const abcs_recon_config* cfg, float* d_out, void* stream);

/* divergence (denoise.cpp:111-128): Monte-Carlo divergence of cfg's denoiser at each field
 * with a std::mt19937_64(seed) Rademacher probe; sigma and epsilon per image (host arrays),
 * result per image into d_div (f64). */
int abcs_divergence_batch(abcs_ctx* ctx, const float* d_field, int32_t height, int32_t width,
                          int32_t n_images, const double* sigma, const double* epsilon, uint64_t seed,
                          const abcs_recon_config* cfg, double* d_div, void* stream);

/* The first n outputs' parity bits of std::mt19937_64(seed) as +1/-1 floats (the probe). */
int abcs_rademacher_probe(abcs_ctx* ctx, uint64_t seed, int64_t n, float* d_probe, void* stream);

/* Synthetic inputs on the device (same bytes as abcs_synth_generate_host). */
int abcs_synth_generate(abcs_ctx* ctx, const abcs_synth_spec* spec, int64_t first_index,
                        int32_t n_images, uint8_t* d_out, int64_t image_stride, void* stream);

/* End-to-end host-buffer pipeline: u8 host images in -> sense -> decode_idct ->
 * f32 host pixels out (cropped), with H2D / kernels / D2H overlapped in chunks
 * on the ctx's streams. h_images/h_out should be pinned for full PCIe rate.
 * Optional host outputs: counts (n*n_blocks) and payload (n*K). Blocks until done. */
/* The subrate sweep end to end from host buffers: each chunk of images is uploaded once and
 * sensed + decoded under every plan (abcs_sense_decode_sweep_batch), and each plan's decoded
 * pixels go to h_out[j] (HOST array of n_plans pinned host pointers), chunks pipelined over
 * the ctx's streams as abcs_sense_decode_host. Plans share the image size. */
int abcs_sense_decode_sweep_host(abcs_ctx* ctx, const abcs_sense_plan* plans, int32_t n_plans,
                                 const uint8_t* h_images, int32_t n_images, float* const* h_out,
                                 int32_t chunk_images);

/* The reference bench step (tools/abcs_main.cpp:226-258, `abcs bench`) from host buffers:
 * sense + decode_idct every image under every plan, then mse, psnr and ssim of each decoded
 * image against the input cropped to the block grid (metrics.cpp:63-125). Only the cells come
 * back: h_mse/h_psnr/h_ssim (each nullable, not all null) hold n_plans*n_images f64, plan-major
 * (cell [j*n_images + i]). Chunks pipelined as abcs_sense_decode_sweep_host. */
int abcs_bench_cells_host(abcs_ctx* ctx, const abcs_sense_plan* plans, int32_t n_plans,
                          const uint8_t* h_images, int32_t n_images, double* h_mse, double* h_psnr,
                          double* h_ssim, int32_t chunk_images);

int abcs_sense_decode_host(abcs_ctx* ctx, const abcs_sense_plan* plan, const uint8_t* h_images,
                           int32_t n_images, float* h_out, uint16_t* h_counts, float* h_payload,
                           int32_t chunk_images);

#ifdef __cplusplus
}
#endif
#endif /* ABCS_B200_H */
