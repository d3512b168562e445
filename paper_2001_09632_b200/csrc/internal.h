// Internal declarations shared by the host entry points (capi.cu, plan.cpp)
// and the kernel translation units.
#pragma once
#include <nvtx3/nvToolsExt.h>
#include <vector>
#include <cstdint>
#include <string>

#include "../../include/abcs_b200.h"

#if defined(__CUDACC__) || defined(ABCS_WITH_CUDA_RUNTIME)
#include <cuda_runtime.h>
#endif

namespace abcs_b200 {

// NVTX range over a host entry point / phase (header-only nvtx3: no link, inert without a tool)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define ABCS_NVTX(name) ::abcs_b200::NvtxRange abcs_nvtx_range_(name)


int set_error(int code, const std::string& msg);
void clear_error();

#if defined(__CUDACC__) || defined(ABCS_WITH_CUDA_RUNTIME)

struct Ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t pipe[3] = {nullptr, nullptr, nullptr};  // e2e pipeline streams
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  int64_t launches = 0;
  void* pipe_buf = nullptr;  // abcs_sense_decode_host slot buffers
  cudaEvent_t ev_fork = nullptr, ev_join[3] = {nullptr, nullptr, nullptr};
  // sweep: per pipe lane, a side stream for the allocations of the later plans
  cudaStream_t side[3] = {nullptr, nullptr, nullptr};
  cudaStream_t ida_side[3] = {};                     // abcs_ida_batch: the chains after the first of a split batch
  cudaEvent_t ida_ev[4] = {};                         // fork, and one join per side chain
  cudaEvent_t ev_side[3][5] = {};
  size_t pipe_bytes = 0;
  // opt-in per-kernel CUDA-event timing (abcs_ctx_kernel_timing): events recorded on the
  // launching stream around each hot kernel, drained by abcs_ctx_kernel_times
  struct KRec {
    const char* name;
    cudaEvent_t start, stop;
  };
  int pipe_streams = 3;  // abcs_ctx_set_pipeline_streams: chunked batch pipelining width (1 = serial)
  bool timing = false;
  std::vector<KRec> krecs;
  std::vector<cudaEvent_t> kpool;
  size_t kpool_used = 0;
  // abcs_ida_batch as a CUDA graph per distinct argument set (the init + per-iteration launches
  // replayed with one cudaGraphLaunch; small batches are launch-bound): captured on a private
  // stream, launched on the caller's
  struct GraphEntry {
    std::vector<uint64_t> key;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;
  };
  std::vector<GraphEntry> graphs;
  cudaStream_t capture = nullptr;
  bool use_graphs = true;
};

// Kernel timing brackets (no-ops unless timing is enabled on the ctx).
int ktimer_begin(Ctx* ctx, cudaStream_t s, const char* name);
void ktimer_end(Ctx* ctx, cudaStream_t s, int slot);

// Stream-ordered scratch owned by the ctx (grows; never shrinks).
void* ctx_scratch(Ctx* ctx, size_t bytes, cudaStream_t stream, int* status);

int cuda_status(cudaError_t e, const char* what);

// Kernel launchers (return abcs_status).
int launch_sense_weights(Ctx* ctx, const abcs_sense_plan& p, const uint8_t* imgs, int64_t img_stride,
                         int32_t pitch, int32_t n, uint32_t* weights, float* side, cudaStream_t s,
                         uint32_t* fix_scratch = nullptr, bool bbv_below = false);
// u32 words of fixup scratch launch_sense_weights needs (count + one entry per block)
inline size_t sense_fix_words(int64_t n_blocks_total) { return (size_t)n_blocks_total * 5 + 8; }
int launch_allocate(Ctx* ctx, const uint32_t* weights, int32_t n_blocks, int32_t n_vectors,
                    int64_t budget, const int32_t* caps, int32_t cap, int32_t base, uint16_t* counts,
                    int32_t* offsets, int32_t* status, void* scratch, cudaStream_t s, int32_t wmax = -1);
size_t allocate_scratch_bytes(int32_t n_blocks, int32_t n_vectors);
size_t shard_scratch_bytes(int32_t n_blocks, int32_t wmax);
int launch_alloc_shard(Ctx* ctx, int phase, const uint32_t* weights, int32_t n_blocks, int32_t wmax, int32_t cap,
                       int32_t base, void* scratch, long long* out, const long long* in, long long remaining,
                       long long prefix, uint16_t* counts, int32_t* offsets, cudaStream_t s);
int launch_zz_counts(Ctx* ctx, const abcs_sense_plan& p, int32_t n, uint16_t* counts, int32_t* offsets,
                     cudaStream_t s);
int launch_gather(Ctx* ctx, int32_t rows, int32_t cols, int32_t block, const uint8_t* imgs,
                  const float* fimgs, int64_t img_stride, int32_t pitch, int32_t n,
                  const uint16_t* counts, const int32_t* offsets, float* payload, int64_t payload_stride,
                  cudaStream_t s);
int launch_offsets(Ctx* ctx, int32_t n_blocks, int32_t n, int32_t block, const uint16_t* counts,
                   int32_t* offsets, const int64_t* payload_len, int32_t* error, cudaStream_t s);
int launch_decode(Ctx* ctx, int32_t rows, int32_t cols, int32_t block, const uint16_t* counts,
                  const int32_t* offsets, const float* payload, int64_t payload_stride, int32_t n,
                  float* out, int64_t out_stride, int32_t out_pitch, cudaStream_t s);
int launch_denoise(Ctx* ctx, const float* field, int32_t h, int32_t w, int64_t stride, int32_t n,
                   const double* thresholds_dev, float* out, cudaStream_t s);
int launch_ida(Ctx* ctx, int32_t rows, int32_t cols, int32_t block, const uint16_t* counts,
               const int32_t* offsets, const float* y, int64_t y_stride, int32_t n,
               const abcs_ida_config& cfg, const uint8_t* ref, int64_t ref_stride, int32_t ref_pitch,
               float* out, int64_t out_stride, int32_t out_pitch, double* trace, int32_t* diverged,
               void* scratch, cudaStream_t s);
struct IdaParams;
int ida_mma_region();
void launch_ida_mma_kernel(int block, const IdaParams& P, dim3 grid, cudaStream_t s);
int launch_psnr(Ctx* ctx, const uint8_t* ref, int64_t ref_stride, int ref_pitch, const float* img, int64_t img_stride,
                int img_pitch, int h, int w, int n, double* psnr, cudaStream_t s, double* mse = nullptr,
                void* scratch = nullptr);
int launch_ssim(Ctx* ctx, const uint8_t* ref, int64_t ref_stride, int ref_pitch, const float* img, int64_t img_stride,
                int img_pitch, int h, int w, int n, double* ssim, cudaStream_t s, void* scratch = nullptr);
size_t psnr_scratch_bytes(int h, int n);
size_t ssim_scratch_bytes(int h, int w, int n);
int launch_threshold_decode(Ctx* ctx, int block, const uint8_t* imgs, int64_t img_stride, int pitch, int rows, int cols,
                            int n, int64_t m_target, bool global, int* counts, double* out, int64_t out_stride,
                            int out_pitch, cudaStream_t s);
// reconstruction family (recon.cu)
int launch_soft_threshold(Ctx* ctx, const float* pseudo, float* x, int64_t N, int n, const double* sigma,
                          double lambda, unsigned long long* active, cudaStream_t s);
int launch_measurements(Ctx* ctx, const uint16_t* counts, const int32_t* offsets, int nb, int n, double* M,
                        cudaStream_t s);
int launch_amp_onsager(Ctx* ctx, const unsigned long long* active, int n, const double* M, double N, bool first,
                       double* onsager, cudaStream_t s);
int launch_blur(Ctx* ctx, const float* in, float* tmp, float* out, int H, int W, int n, const double* sigma_dev,
                double scale, int rmax, double* wscratch, int* rscratch, cudaStream_t s);
int launch_probe(Ctx* ctx, uint64_t seed, int64_t N, float* probe, cudaStream_t s);
// the probes of iterations it0 .. it0 + count - 1 (seeds as probe_seed_for) at probes + k * N
int launch_probes(Ctx* ctx, uint64_t seed, int it0, int count, int64_t N, float* probes, cudaStream_t s);
int launch_divergence_prep(Ctx* ctx, const float* pseudo, const float* probe, int64_t N, int n, unsigned* maxbits,
                           float* perturbed, double* eps, cudaStream_t s);
int launch_damp_onsager(Ctx* ctx, const float* probe, const float* moved, const float* base, int64_t N, int n,
                        const double* eps, const double* M, double divisor, double* partials, double* onsager,
                        cudaStream_t s);
size_t divergence_partials(Ctx* ctx, int64_t N, int n);
int launch_scale(Ctx* ctx, const double* sigma, double k, int n, double* thr, cudaStream_t s);
int launch_divergence_given(Ctx* ctx, const float* field, const float* probe, const float* base, int64_t N, int n,
                            const double* eps, float* perturbed, const float* moved, double* partials,
                            double* div, bool perturb_only, cudaStream_t s);
int run_denoiser(Ctx* ctx, const abcs_recon_config& cfg, const float* in, float* out, float* tmp, int H, int W, int n,
                 const double* sigma, double* thr, cudaStream_t s);
int launch_recon(Ctx* ctx, bool one_step, int32_t rows, int32_t cols, int32_t block, const uint16_t* counts,
                 const int32_t* offsets, const float* y, int64_t y_stride, int32_t n, const abcs_recon_config& cfg,
                 const uint8_t* ref, int64_t ref_stride, int32_t ref_pitch, float* x, float* z, double* sigma,
                 int32_t iteration0, float* out, int64_t out_stride, int32_t out_pitch, double* trace,
                 int32_t* diverged, cudaStream_t s);
size_t ida_state_scratch_bytes(int32_t rows, int32_t cols, int32_t block, int64_t y_stride, int32_t n);
int launch_ida_state(Ctx* ctx, bool init, int32_t rows, int32_t cols, int32_t block, const uint16_t* counts,
                     const int32_t* offsets, const float* y, int64_t y_stride, int32_t n, int warm, double damping,
                     double k, float* x, float* z, double* sigma, int32_t iteration, int32_t* diverged, void* scratch,
                     cudaStream_t s);
size_t ida_scratch_bytes(int32_t rows, int32_t cols, int32_t block, int64_t y_stride, int32_t n,
                         const abcs_ida_config& cfg);
bool mma16_supported(int rows, int cols, int n);
// allocation fused into the B=16 DD weights pass (small images: n_blocks <= 4096, phase1 <= 127)
struct FusedAlloc {
  uint32_t* runs_done;  // n u32 scratch
  int32_t* status;      // n u32 scratch
  uint16_t* counts;
  int32_t* offsets;
  long long budget;
  int cap, base, wmax;
};
bool fused_alloc_supported(Ctx* ctx, int rows, int cols, int n, int wmax);
// every plan's allocation of a DD sweep in one launch (plan = blockIdx.y)
int launch_alloc_cta_plans(Ctx* ctx, int np, int rows, int cols, int n, uint32_t* const* weights,
                           const FusedAlloc* fa, cudaStream_t s);
// mode 1: DD weights; 2: payload; 3: payload + fused decode
bool umma16_enabled();
int launch_sense16_umma(Ctx* ctx, int mode, int rows, int cols, int n, const uint8_t* imgs, int64_t img_stride,
                        int pitch, const uint16_t* counts, const int32_t* offsets, float* payload,
                        int64_t payload_stride, float* out, int64_t out_stride, int out_pitch, cudaStream_t s);
int launch_sense16_multi(Ctx* ctx, int np, int rows, int cols, int n, const uint8_t* imgs, int64_t img_stride,
                         int pitch, const uint16_t* const* counts, const int32_t* const* offsets,
                         float* const* payload, const int64_t* payload_stride, float* const* out, int64_t out_stride,
                         int out_pitch, cudaStream_t s);
int launch_sense16_sweep(Ctx* ctx, int n_sw, int rows, int cols, int n, const uint8_t* imgs, int64_t img_stride,
                         int pitch, const int* phase1, const double* T, uint32_t* const* weights,
                         uint32_t* const* fix_scratch, cudaStream_t s);
// one warp per vector of n_blocks (<= 4096) weights in [0, fa.wmax <= 127] (warp_alloc.cuh)
int launch_alloc_small(Ctx* ctx, int n_blocks, int n, const uint32_t* weights, const FusedAlloc& fa, cudaStream_t s);
int launch_alloc_cta(Ctx* ctx, int rows, int cols, int n, const uint32_t* weights, const FusedAlloc& fa,
                     cudaStream_t s);
int launch_sense16(Ctx* ctx, int mode, int rows, int cols, int n, const uint8_t* imgs, int64_t img_stride, int pitch,
                   int phase1, double T, uint32_t* weights, const uint16_t* counts, const int32_t* offsets,
                   float* payload, int64_t payload_stride, float* out, int64_t out_stride, int out_pitch,
                   cudaStream_t s, uint32_t* fix_scratch = nullptr, const FusedAlloc* fa = nullptr);
int launch_sense8(Ctx* ctx, bool from_image, bool decode, int rows, int cols, int n, const uint8_t* imgs,
                  int64_t img_stride, int pitch, const uint16_t* counts, const int32_t* offsets, float* payload,
                  int64_t payload_stride, float* out, int64_t out_stride, int out_pitch, cudaStream_t s);
int launch_decode16(Ctx* ctx, int rows, int cols, int n, const uint16_t* counts, const int32_t* offsets,
                    const float* payload, int64_t payload_stride, float* out, int64_t out_stride, int out_pitch,
                    cudaStream_t s);
int launch_synth(Ctx* ctx, const abcs_synth_spec& spec, int64_t first, int32_t n, uint8_t* out,
                 int64_t stride, void* scratch, cudaStream_t s);

#endif

}  // namespace abcs_b200
