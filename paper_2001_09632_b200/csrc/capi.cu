// extern "C" entry points of libabcs_b200.so (declared in include/abcs_b200.h).
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "synth_gen.h"

namespace abcs_b200 {

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ABCS_OK;
  return set_error(ABCS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void* ctx_scratch(Ctx* ctx, size_t bytes, cudaStream_t stream, int* status) {
  *status = ABCS_OK;
  if (bytes <= ctx->scratch_bytes) return ctx->scratch;
  if (ctx->scratch) {
    // growth is rare (first call of a bigger batch): drain users of the old buffer
    cudaError_t e = cudaStreamSynchronize(stream);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      *status = cuda_status(e, "scratch sync");
      return nullptr;
    }
    cudaFree(ctx->scratch);
    ctx->scratch = nullptr;
    ctx->scratch_bytes = 0;
    for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.exec);  // they point into the old scratch
    ctx->graphs.clear();
  }
  const size_t want = bytes + bytes / 4 + (1u << 20);
  cudaError_t e = cudaMalloc(&ctx->scratch, want);
  if (e != cudaSuccess) {
    ctx->scratch = nullptr;
    *status = cuda_status(e, "scratch alloc");
    return nullptr;
  }
  ctx->scratch_bytes = want;
  return ctx->scratch;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

static bool block_supported(int B) { return B == 8 || B == 16 || B == 32; }

}  // namespace abcs_b200

using namespace abcs_b200;

#define CHECK_CTX(ctx) \
  if (!(ctx)) return set_error(ABCS_ERR_INVALID_ARGUMENT, "null context")

extern "C" {

int abcs_ctx_create(int device, abcs_ctx** out) {
  if (!out) return set_error(ABCS_ERR_INVALID_ARGUMENT, "null output");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return set_error(ABCS_ERR_CUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e));
  if (device < 0 || device >= n) return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad device index");
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDeviceProperties");
  if (prop.major != 10) return set_error(ABCS_ERR_UNSUPPORTED, "libabcs_b200 is built for sm_100a (B200) only");
  auto* ctx = new Ctx;
  ctx->device = device;
  ctx->sm_count = prop.multiProcessorCount;
  if (const char* g = getenv("ABCS_NO_GRAPHS")) ctx->use_graphs = !(g[0] == '1');
  for (auto& st : ctx->pipe) {
    e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete ctx;
      return cuda_status(e, "stream create");
    }
  }
  *out = reinterpret_cast<abcs_ctx*>(ctx);
  return ABCS_OK;
}

int abcs_ctx_destroy(abcs_ctx* c) {
  if (!c) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  if (ctx->scratch) cudaFree(ctx->scratch);
  if (ctx->pipe_buf) cudaFree(ctx->pipe_buf);
  for (int k = 0; k < 3; ++k) {
    if (ctx->side[k]) cudaStreamDestroy(ctx->side[k]);
    for (auto& e : ctx->ev_side[k])
      if (e) cudaEventDestroy(e);
  }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  for (auto& e : ctx->ev_join)
    if (e) cudaEventDestroy(e);
  for (auto& st : ctx->pipe)
    if (st) cudaStreamDestroy(st);
  for (auto& e : ctx->kpool) cudaEventDestroy(e);
  for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.exec);
  if (ctx->capture) cudaStreamDestroy(ctx->capture);
  for (auto& q : ctx->ida_side)
    if (q) cudaStreamDestroy(q);
  for (auto& e : ctx->ida_ev)
    if (e) cudaEventDestroy(e);
  delete ctx;
  return ABCS_OK;
}

int64_t abcs_ctx_launch_count(const abcs_ctx* c) {
  return c ? reinterpret_cast<const Ctx*>(c)->launches : 0;
}

int abcs_ctx_set_pipeline_streams(abcs_ctx* c, int32_t streams) {
  CHECK_CTX(c);
  if (streams < 1 || streams > 3) return set_error(ABCS_ERR_INVALID_ARGUMENT, "pipeline streams must be in [1, 3]");
  reinterpret_cast<Ctx*>(c)->pipe_streams = streams;
  return ABCS_OK;
}

int abcs_ctx_kernel_timing(abcs_ctx* c, int32_t enable) {
  CHECK_CTX(c);
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaDeviceSynchronize();
  ctx->krecs.clear();
  ctx->kpool_used = 0;
  ctx->timing = enable != 0;
  return cuda_status(e, "kernel timing");
}

int abcs_ctx_kernel_times(abcs_ctx* c, abcs_kernel_time* out, int32_t capacity, int32_t* count) {
  CHECK_CTX(c);
  if (!count || capacity < 0 || (capacity > 0 && !out)) return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_status(e, "kernel times");
  std::vector<abcs_kernel_time> agg;
  for (const auto& r : ctx->krecs) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.start, r.stop) != cudaSuccess) continue;
    abcs_kernel_time* k = nullptr;
    for (auto& a : agg)
      if (std::strncmp(a.name, r.name, sizeof(a.name)) == 0) k = &a;
    if (!k) {
      agg.push_back(abcs_kernel_time{});
      k = &agg.back();
      std::strncpy(k->name, r.name, sizeof(k->name) - 1);
    }
    k->launches += 1;
    k->total_ms += ms;
    k->max_ms = std::max(k->max_ms, (double)ms);
  }
  *count = (int32_t)agg.size();
  for (int i = 0; i < (int)agg.size() && i < capacity; ++i) out[i] = agg[i];
  return ABCS_OK;
}

int abcs_sense_weights_batch(abcs_ctx* c, const abcs_sense_plan* p, const uint8_t* d_images, int64_t image_stride,
                             int32_t pitch, int32_t n, uint32_t* d_weights, float* d_side, void* stream) {
  ABCS_NVTX("abcs_sense_weights_batch");
  CHECK_CTX(c);
  if (!p || (!d_images && n > 0) || !d_weights || n < 0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int st;
  uint32_t* fix = static_cast<uint32_t*>(ctx_scratch(ctx, sense_fix_words((int64_t)n * p->n_blocks) * 4, s, &st));
  if (st) return st;
  return launch_sense_weights(ctx, *p, d_images, image_stride, pitch, n, d_weights, d_side, s, fix);
}

int abcs_bbv_weights_strip(abcs_ctx* c, const abcs_sense_plan* p, const uint8_t* d_strip, int64_t strip_stride,
                           int32_t pitch, int32_t has_below, uint32_t* d_weights, float* d_side, void* stream) {
  CHECK_CTX(c);
  if (!p || !d_strip || !d_weights || p->algorithm_used != ABCS_ALGO_BBV)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bbv strip weights: bad arguments");
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  return launch_sense_weights(ctx, *p, d_strip, strip_stride, pitch, 1, d_weights, d_side,
                              reinterpret_cast<cudaStream_t>(stream), nullptr, has_below != 0);
}

}  // extern "C"

namespace abcs_b200 {

static size_t sense_scratch_bytes(const abcs_sense_plan* p, int32_t n, bool have_offsets) {
  const int64_t nbt = (int64_t)n * p->n_blocks;
  const size_t off_bytes = have_offsets ? 0 : align_up(nbt * 4, 256);
  const size_t w_bytes = align_up(nbt * 4, 256);
  const size_t a_bytes = align_up(allocate_scratch_bytes(p->n_blocks, n), 256);
  const size_t f_bytes = align_up(sense_fix_words(nbt) * 4, 256);
  return off_bytes + w_bytes + a_bytes + f_bytes;
}

static int sense_validate(const abcs_sense_plan* p, const uint8_t* d_images, int64_t image_stride, int32_t pitch,
                          int32_t n, uint16_t* d_counts, float* d_payload, float* d_side) {
  if (!p || n < 0 || (n > 0 && (!d_images || !d_counts || !d_payload)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!block_supported(p->block)) return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  if (pitch < p->width || image_stride < (int64_t)pitch * (p->height - 1) + p->width)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "image pitch/stride smaller than the image");
  if (p->algorithm_used == ABCS_ALGO_BBV && p->side_per_image > 0 && !d_side && n > 0)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bbv sensing needs a side-data buffer");
  return ABCS_OK;
}

// sense() on n images with caller-provided scratch (sense_scratch_bytes);
// with d_out, also the decode of the result (fused into the payload pass when
// the tensor-core path applies).
static int sense_impl(Ctx* ctx, const abcs_sense_plan* p, const uint8_t* d_images, int64_t image_stride, int32_t pitch,
                      int32_t n, uint16_t* d_counts, int32_t* d_offsets, float* d_payload, float* d_side, char* scr,
                      cudaStream_t s, float* d_out = nullptr, int64_t out_stride = 0, int32_t out_pitch = 0) {
  if (n == 0) return ABCS_OK;
  const int64_t nbt = (int64_t)n * p->n_blocks;
  const size_t off_bytes = d_offsets ? 0 : align_up(nbt * 4, 256);
  const size_t w_bytes = align_up(nbt * 4, 256);
  int32_t* offsets = d_offsets ? d_offsets : reinterpret_cast<int32_t*>(scr);
  uint32_t* weights = reinterpret_cast<uint32_t*>(scr + off_bytes);
  void* ascr = scr + off_bytes + w_bytes;
  uint32_t* fix = reinterpret_cast<uint32_t*>(scr + off_bytes + w_bytes + align_up(allocate_scratch_bytes(p->n_blocks, n), 256));
  int st;
  // largest possible phase-1 weight: DD counts <= phase1; BBV sums <= 4 * valid probes * 255
  const int32_t wmax = p->algorithm_used == ABCS_ALGO_DD ? p->dd_phase1 : 4 * p->bbv_valid_probes * 255;
  if (p->algorithm_used == ABCS_ALGO_ZZ) {
    st = launch_zz_counts(ctx, *p, n, d_counts, offsets, s);
    if (st) return st;
  } else if (p->algorithm_used == ABCS_ALGO_DD && p->block == 16 &&
             fused_alloc_supported(ctx, p->rows, p->cols, n, wmax)) {
    // DD phase 1 + allocation in one launch: the last warp to finish an image allocates it
    FusedAlloc fa;
    fa.runs_done = nullptr;
    fa.status = nullptr;
    fa.counts = d_counts;
    fa.offsets = offsets;
    fa.budget = p->alloc_budget;
    fa.cap = p->cap;
    fa.base = p->count_base;
    fa.wmax = wmax;
    st = launch_sense16(ctx, 1, p->rows, p->cols, n, d_images, image_stride, pitch, p->dd_phase1, p->threshold,
                        weights, nullptr, nullptr, nullptr, 0, nullptr, 0, 0, s, fix, &fa);
    if (st) return st;
  } else {
    st = launch_sense_weights(ctx, *p, d_images, image_stride, pitch, n, weights, d_side, s, fix);
    if (st) return st;
    st = launch_allocate(ctx, weights, p->n_blocks, n, p->alloc_budget, nullptr, p->cap, p->count_base, d_counts,
                         offsets, nullptr, ascr, s, wmax);
    if (st) return st;
  }
  if (d_out && p->block == 16 && mma16_supported(p->rows, p->cols, n) && out_pitch % 2 == 0 && out_stride % 2 == 0 &&
      ((uintptr_t)d_out % 8) == 0) {
    return launch_sense16(ctx, 3, p->rows, p->cols, n, d_images, image_stride, pitch, 0, 0.0, nullptr, d_counts,
                          offsets, d_payload, p->coeffs_per_image, d_out, out_stride, out_pitch, s);
  }
  if (d_out && p->block == 8 && mma16_supported(p->rows, p->cols, n) && out_pitch % 2 == 0 && out_stride % 2 == 0 &&
      ((uintptr_t)d_out % 8) == 0) {
    return launch_sense8(ctx, true, true, p->rows, p->cols, n, d_images, image_stride, pitch, d_counts, offsets,
                         d_payload, p->coeffs_per_image, d_out, out_stride, out_pitch, s);
  }
  st = launch_gather(ctx, p->rows, p->cols, p->block, d_images, nullptr, image_stride, pitch, n, d_counts, offsets,
                     d_payload, p->coeffs_per_image, s);
  if (st || !d_out) return st;
  return launch_decode(ctx, p->rows, p->cols, p->block, d_counts, offsets, d_payload, p->coeffs_per_image, n, d_out,
                       out_stride, out_pitch, s);
}

// Batch pipelining across the ctx's streams: the batch is cut into chunks that run
// on the three pipe streams (each with its own scratch), so one chunk's
// latency-bound steps (fp64 fixup, per-image allocation, kernel tails) overlap
// the other chunks' transform kernels. Joined back to the caller's stream.
static int sense_chunked(Ctx* ctx, const abcs_sense_plan* p, const uint8_t* d_images, int64_t image_stride,
                         int32_t pitch, int32_t n, uint16_t* d_counts, int32_t* d_offsets, float* d_payload,
                         float* d_side, cudaStream_t s, float* d_out, int64_t out_stride, int32_t out_pitch) {
  const int min_chunk = 64;
  int nchunks = std::min<int>(ctx->pipe_streams, n / min_chunk);
  if (nchunks < 2) {
    int st;
    char* scr = static_cast<char*>(ctx_scratch(ctx, sense_scratch_bytes(p, n, d_offsets != nullptr), s, &st));
    if (st) return st;
    return sense_impl(ctx, p, d_images, image_stride, pitch, n, d_counts, d_offsets, d_payload, d_side, scr, s, d_out,
                      out_stride, out_pitch);
  }
  const int chunk = (n + nchunks - 1) / nchunks;
  const size_t per = align_up(sense_scratch_bytes(p, chunk, d_offsets != nullptr), 256);
  int st;
  char* scr = static_cast<char*>(ctx_scratch(ctx, per * nchunks, s, &st));
  if (st) return st;
  if (!ctx->ev_fork) {
    cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
    for (auto& e : ctx->ev_join) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  cudaError_t e = cudaEventRecord(ctx->ev_fork, s);
  if (e != cudaSuccess) return cuda_status(e, "fork");
  const int64_t NB = p->n_blocks, K = p->coeffs_per_image, S = p->side_per_image;
  for (int k = 0; k < nchunks; ++k) {
    const int first = k * chunk, cnt = std::min(chunk, n - first);
    cudaStream_t cs = ctx->pipe[k];
    cudaStreamWaitEvent(cs, ctx->ev_fork, 0);
    st = sense_impl(ctx, p, d_images + first * image_stride, image_stride, pitch, cnt, d_counts + first * NB,
                    d_offsets ? d_offsets + first * NB : nullptr, d_payload + first * K,
                    d_side ? d_side + first * S : nullptr, scr + per * k, cs,
                    d_out ? d_out + first * out_stride : nullptr, out_stride, out_pitch);
    if (st) return st;
    e = cudaEventRecord(ctx->ev_join[k], cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ctx->ev_join[k], 0);
    if (e != cudaSuccess) return cuda_status(e, "join");
  }
  return ABCS_OK;
}

// ---- subrate sweep (abcs_main.cpp:215-260: sense() of one image per --crs entry) ---------
// DD plans of B = 16 on the same geometry share DD phase 1's forward transform: one
// launch_sense16_sweep computes every plan's significance counts, then each plan gets its
// own fp64 fixup, allocation, payload and decode -- the same outputs as separate calls.
static bool sweep_shared(Ctx* ctx, const abcs_sense_plan* plans, int32_t np, int32_t n) {
  if (np < 2 || np > 4) return false;
  for (int j = 0; j < np; ++j) {
    const abcs_sense_plan& q = plans[j];
    if (q.algorithm_used != ABCS_ALGO_DD || q.block != 16 || q.rows != plans[0].rows || q.cols != plans[0].cols ||
        q.height != plans[0].height || q.width != plans[0].width)
      return false;
    if (!fused_alloc_supported(ctx, q.rows, q.cols, n, q.dd_phase1) || !mma16_supported(q.rows, q.cols, n)) return false;
  }
  return true;
}

static size_t sweep_scratch_bytes(const abcs_sense_plan* plans, int32_t np, int32_t n, int32_t* const* d_offsets) {
  size_t b = 0;
  for (int j = 0; j < np; ++j) {
    const int64_t nbt = (int64_t)n * plans[j].n_blocks;
    b += (d_offsets && d_offsets[j] ? 0 : align_up(nbt * 4, 256)) + align_up(nbt * 4, 256) +
         align_up(sense_fix_words(nbt) * 4, 256);
  }
  return b;
}

static int sweep_impl(Ctx* ctx, const abcs_sense_plan* plans, int32_t np, const uint8_t* d_images,
                      int64_t image_stride, int32_t pitch, int32_t n, int64_t first, uint16_t* const* d_counts,
                      int32_t* const* d_offsets, float* const* d_payload, float* const* d_out, int64_t out_stride,
                      int32_t out_pitch, char* scr, cudaStream_t s, int lane) {
  if (n == 0) return ABCS_OK;
  const abcs_sense_plan& p0 = plans[0];
  int32_t* offs[4];
  uint32_t* weights[4];
  uint32_t* fix[4];
  int phase1[4];
  double T[4];
  for (int j = 0; j < np; ++j) {
    const int64_t nbt = (int64_t)n * plans[j].n_blocks;
    if (d_offsets && d_offsets[j]) {
      offs[j] = d_offsets[j] + first * plans[j].n_blocks;
    } else {
      offs[j] = reinterpret_cast<int32_t*>(scr);
      scr += align_up(nbt * 4, 256);
    }
    weights[j] = reinterpret_cast<uint32_t*>(scr);
    scr += align_up(nbt * 4, 256);
    fix[j] = reinterpret_cast<uint32_t*>(scr);
    scr += align_up(sense_fix_words(nbt) * 4, 256);
    phase1[j] = plans[j].dd_phase1;
    T[j] = plans[j].threshold;
  }
  const uint8_t* imgs = d_images + first * image_stride;
  int st = launch_sense16_sweep(ctx, np, p0.rows, p0.cols, n, imgs, image_stride, pitch, phase1, T, weights, fix, s);
  if (st) return st;
  auto fa_of = [&](int j) {
    const abcs_sense_plan& q = plans[j];
    FusedAlloc fa;
    fa.runs_done = nullptr;
    fa.status = nullptr;
    fa.counts = d_counts[j] + first * q.n_blocks;
    fa.offsets = offs[j];
    fa.budget = q.alloc_budget;
    fa.cap = q.cap;
    fa.base = q.count_base;
    fa.wmax = q.dd_phase1;
    return fa;
  };
  const char* multi_env = getenv("ABCS_SWEEP_MULTI");
  if (!(multi_env && multi_env[0] == '0') && p0.block == 16 && out_stride % 2 == 0 && out_pitch % 2 == 0) {
    // every plan's allocation in one launch, then one payload pass that transforms each block
    // once for all plans
    FusedAlloc fas[4];
    for (int j = 0; j < np; ++j) fas[j] = fa_of(j);
    st = launch_alloc_cta_plans(ctx, np, p0.rows, p0.cols, n, weights, fas, s);
    if (st) return st;
    const uint16_t* cnts[4];
    const int32_t* offc[4];
    float* pays[4];
    int64_t pstr[4];
    float* outs[4];
    for (int j = 0; j < np; ++j) {
      cnts[j] = d_counts[j] + first * plans[j].n_blocks;
      offc[j] = offs[j];
      pays[j] = d_payload[j] + first * plans[j].coeffs_per_image;
      pstr[j] = plans[j].coeffs_per_image;
      outs[j] = d_out[j] + first * out_stride;
    }
    return launch_sense16_multi(ctx, np, p0.rows, p0.cols, n, imgs, image_stride, pitch, cnts, offc, pays, pstr,
                                outs, out_stride, out_pitch, s);
  }
  // the later plans' allocations (latency-bound, one CTA per image) run on a side stream,
  // under the earlier plans' payload passes (not when the ctx is set to serialise: 1 pipe stream)
  if (ctx->pipe_streams <= 1) {
    for (int j = 0; j < np; ++j) {
      const abcs_sense_plan& q = plans[j];
      st = launch_alloc_cta(ctx, q.rows, q.cols, n, weights[j], fa_of(j), s);
      if (st) return st;
      st = launch_sense16(ctx, 3, q.rows, q.cols, n, imgs, image_stride, pitch, 0, 0.0, nullptr,
                          d_counts[j] + first * q.n_blocks, offs[j], d_payload[j] + first * q.coeffs_per_image,
                          q.coeffs_per_image, d_out[j] + first * out_stride, out_stride, out_pitch, s);
      if (st) return st;
    }
    return ABCS_OK;
  }
  cudaStream_t side = ctx->side[lane];
  if (!side) {
    cudaStreamCreateWithFlags(&ctx->side[lane], cudaStreamNonBlocking);
    for (auto& e : ctx->ev_side[lane]) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    side = ctx->side[lane];
  }
  cudaError_t e = cudaEventRecord(ctx->ev_side[lane][0], s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ctx->ev_side[lane][0], 0);
  if (e != cudaSuccess) return cuda_status(e, "sweep fork");
  for (int j = 1; j < np; ++j) {
    const abcs_sense_plan& q = plans[j];
    st = launch_alloc_cta(ctx, q.rows, q.cols, n, weights[j], fa_of(j), side);
    if (st) return st;
    e = cudaEventRecord(ctx->ev_side[lane][j], side);
    if (e != cudaSuccess) return cuda_status(e, "sweep event");
  }
  for (int j = 0; j < np; ++j) {
    const abcs_sense_plan& q = plans[j];
    uint16_t* counts = d_counts[j] + first * q.n_blocks;
    if (j == 0) st = launch_alloc_cta(ctx, q.rows, q.cols, n, weights[j], fa_of(j), s);
    else st = cuda_status(cudaStreamWaitEvent(s, ctx->ev_side[lane][j], 0), "sweep join");
    if (st) return st;
    st = launch_sense16(ctx, 3, q.rows, q.cols, n, imgs, image_stride, pitch, 0, 0.0, nullptr, counts, offs[j],
                        d_payload[j] + first * q.coeffs_per_image, q.coeffs_per_image, d_out[j] + first * out_stride,
                        out_stride, out_pitch, s);
    if (st) return st;
  }
  return ABCS_OK;
}

// ---- per-kernel timing -----------------------------------------------------------------
static cudaEvent_t take_event(Ctx* ctx) {
  if (ctx->kpool_used == ctx->kpool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    ctx->kpool.push_back(e);
  }
  return ctx->kpool[ctx->kpool_used++];
}

int ktimer_begin(Ctx* ctx, cudaStream_t s, const char* name) {
  if (!ctx->timing) return -1;
  cudaEvent_t a = take_event(ctx), b = take_event(ctx);
  if (!a || !b) return -1;
  cudaEventRecord(a, s);
  ctx->krecs.push_back({name, a, b});
  return (int)ctx->krecs.size() - 1;
}

void ktimer_end(Ctx* ctx, cudaStream_t s, int slot) {
  if (slot >= 0) cudaEventRecord(ctx->krecs[slot].stop, s);
}

}  // namespace abcs_b200

extern "C" {

int abcs_sense_batch(abcs_ctx* c, const abcs_sense_plan* p, const uint8_t* d_images, int64_t image_stride,
                     int32_t pitch, int32_t n, uint16_t* d_counts, int32_t* d_offsets, float* d_payload,
                     float* d_side, void* stream) {
  ABCS_NVTX("abcs_sense_batch");
  CHECK_CTX(c);
  int st = sense_validate(p, d_images, image_stride, pitch, n, d_counts, d_payload, d_side);
  if (st || n == 0) return st;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return sense_chunked(ctx, p, d_images, image_stride, pitch, n, d_counts, d_offsets, d_payload, d_side, s, nullptr,
                       0, 0);
}

int abcs_sense_decode_batch(abcs_ctx* c, const abcs_sense_plan* p, const uint8_t* d_images, int64_t image_stride,
                            int32_t pitch, int32_t n, uint16_t* d_counts, int32_t* d_offsets, float* d_payload,
                            float* d_side, float* d_out, int64_t out_stride, int32_t out_pitch, void* stream) {
  ABCS_NVTX("abcs_sense_decode_batch");
  CHECK_CTX(c);
  int st = sense_validate(p, d_images, image_stride, pitch, n, d_counts, d_payload, d_side);
  if (st || n == 0) return st;
  const int Wc = p->cols * p->block, Hc = p->rows * p->block;
  if (!d_out || out_pitch < Wc || out_stride < (int64_t)out_pitch * (Hc - 1) + Wc)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "output pitch/stride smaller than the image");
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return sense_chunked(ctx, p, d_images, image_stride, pitch, n, d_counts, d_offsets, d_payload, d_side, s, d_out,
                       out_stride, out_pitch);
}

int abcs_sense_decode_sweep_batch(abcs_ctx* c, const abcs_sense_plan* plans, int32_t n_plans,
                                  const uint8_t* d_images, int64_t image_stride, int32_t pitch, int32_t n,
                                  uint16_t* const* d_counts, int32_t* const* d_offsets, float* const* d_payload,
                                  float* const* d_side, float* const* d_out, int64_t out_stride, int32_t out_pitch,
                                  void* stream) {
  ABCS_NVTX("abcs_sense_decode_sweep_batch");
  CHECK_CTX(c);
  if (!plans || n_plans < 1 || !d_counts || !d_payload || !d_out)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  for (int j = 0; j < n_plans; ++j) {
    int st = sense_validate(&plans[j], d_images, image_stride, pitch, n, d_counts[j], d_payload[j],
                            d_side ? d_side[j] : nullptr);
    if (st) return st;
    const int Wc = plans[j].cols * plans[j].block, Hc = plans[j].rows * plans[j].block;
    if (!d_out[j] || out_pitch < Wc || out_stride < (int64_t)out_pitch * (Hc - 1) + Wc)
      return set_error(ABCS_ERR_INVALID_ARGUMENT, "output pitch/stride smaller than the image");
  }
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool aligned_out = out_pitch % 2 == 0 && out_stride % 2 == 0;
  bool out_ok = aligned_out;
  for (int j = 0; j < n_plans; ++j) out_ok = out_ok && ((uintptr_t)d_out[j] % 8) == 0;
  if (!out_ok || !sweep_shared(ctx, plans, n_plans, n)) {  // no shared transform: one plan at a time
    for (int j = 0; j < n_plans; ++j) {
      const int st = sense_chunked(ctx, &plans[j], d_images, image_stride, pitch, n, d_counts[j],
                                   d_offsets ? d_offsets[j] : nullptr, d_payload[j], d_side ? d_side[j] : nullptr,
                                   s, d_out[j], out_stride, out_pitch);
      if (st) return st;
    }
    return ABCS_OK;
  }
  // chunks of the batch round-robin on the pipe streams, as sense_chunked
  static const int chunks_env = [] {
    const char* e = getenv("ABCS_SWEEP_CHUNKS");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  const int want_chunks = chunks_env ? chunks_env : ctx->pipe_streams;
  const int nchunks = ctx->pipe_streams <= 1 ? 1 : std::max(1, std::min<int>(want_chunks, n / 64));
  const int chunk = (n + nchunks - 1) / nchunks;
  const size_t per = align_up(sweep_scratch_bytes(plans, n_plans, chunk, d_offsets), 256);
  int st;
  char* scr = static_cast<char*>(ctx_scratch(ctx, per * nchunks, s, &st));
  if (st) return st;
  if (nchunks == 1)
    return sweep_impl(ctx, plans, n_plans, d_images, image_stride, pitch, n, 0, d_counts, d_offsets, d_payload,
                      d_out, out_stride, out_pitch, scr, s, 0);
  if (!ctx->ev_fork) {
    cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
    for (auto& e : ctx->ev_join) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  cudaError_t e = cudaEventRecord(ctx->ev_fork, s);
  if (e != cudaSuccess) return cuda_status(e, "fork");
  for (int k = 0; k < nchunks; ++k) {
    const int first = k * chunk, cnt = std::min(chunk, n - first);
    if (cnt <= 0) break;
    const int lane = k % ctx->pipe_streams;
    cudaStream_t cs = ctx->pipe[lane];
    cudaStreamWaitEvent(cs, ctx->ev_fork, 0);
    st = sweep_impl(ctx, plans, n_plans, d_images, image_stride, pitch, cnt, first, d_counts, d_offsets, d_payload,
                    d_out, out_stride, out_pitch, scr + per * k, cs, lane);
    if (st) return st;
    e = cudaEventRecord(ctx->ev_join[lane], cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ctx->ev_join[lane], 0);
    if (e != cudaSuccess) return cuda_status(e, "join");
  }
  return ABCS_OK;
}

int abcs_allocate_small_batch(abcs_ctx* c, const uint32_t* d_weights, int32_t n_blocks, int32_t n_vectors,
                              int64_t budget, int32_t cap, int32_t base, int32_t wmax, uint16_t* d_counts,
                              int32_t* d_offsets, int32_t* d_status, void* stream) {
  ABCS_NVTX("abcs_allocate_small_batch");
  CHECK_CTX(c);
  if (n_blocks < 0 || n_vectors < 0 || n_blocks > 4096 || wmax < 0 || wmax > 127 || cap < 0 || cap > 65535 ||
      (n_blocks * (int64_t)n_vectors > 0 && (!d_weights || !d_counts || !d_offsets)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments (n_blocks <= 4096, 0 <= wmax <= 127)");
  if (n_blocks == 0 || n_vectors == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  FusedAlloc fa{};
  fa.status = d_status;
  fa.counts = d_counts;
  fa.offsets = d_offsets;
  fa.budget = budget;
  fa.cap = cap;
  fa.base = base;
  fa.wmax = wmax;
  return launch_alloc_small(ctx, n_blocks, n_vectors, d_weights, fa, reinterpret_cast<cudaStream_t>(stream));
}

int abcs_allocate_batch(abcs_ctx* c, const uint32_t* d_weights, int32_t n_blocks, int32_t n_vectors, int64_t budget,
                        const int32_t* d_caps, int32_t cap, int32_t base, uint16_t* d_counts, int32_t* d_offsets,
                        int32_t* d_status, void* stream) {
  ABCS_NVTX("abcs_allocate_batch");
  CHECK_CTX(c);
  if (n_blocks < 0 || n_vectors < 0 || (n_blocks * (int64_t)n_vectors > 0 && (!d_weights || !d_counts)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int st;
  void* scr = ctx_scratch(ctx, allocate_scratch_bytes(n_blocks, n_vectors), s, &st);
  if (st) return st;
  return launch_allocate(ctx, d_weights, n_blocks, n_vectors, budget, d_caps, cap, base, d_counts, d_offsets, d_status,
                         scr, s);
}

size_t abcs_allocate_shard_scratch_bytes(int32_t n_blocks, int32_t wmax) {
  if (n_blocks < 0 || wmax < 0 || wmax > 65535) return 0;
  return shard_scratch_bytes(n_blocks, wmax);
}

int abcs_allocate_shard_step(abcs_ctx* c, int32_t phase, const uint32_t* d_weights, int32_t n_blocks, int32_t wmax,
                             int32_t cap, int32_t base, void* d_scratch, int64_t* d_out, const int64_t* d_in,
                             int64_t remaining, int64_t prefix, uint16_t* d_counts, int32_t* d_offsets,
                             void* stream) {
  CHECK_CTX(c);
  if (phase < 0 || phase > 4 || n_blocks < 0 || wmax < 0 || wmax > 65535 || cap < 0 || cap > 65535 || !d_scratch ||
      !d_out || (phase == 0 && n_blocks > 0 && !d_weights) || (phase == 2 && !d_in) || (phase == 4 && !d_counts))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  return launch_alloc_shard(ctx, phase, d_weights, n_blocks, wmax, cap, base, d_scratch,
                            reinterpret_cast<long long*>(d_out), reinterpret_cast<const long long*>(d_in), remaining,
                            prefix, d_counts, d_offsets, reinterpret_cast<cudaStream_t>(stream));
}

int abcs_gather_decode_batch(abcs_ctx* c, int32_t rows, int32_t cols, int32_t block, const uint8_t* d_images,
                             int64_t image_stride, int32_t pitch, int32_t n, const uint16_t* d_counts,
                             const int32_t* d_offsets, float* d_payload, int64_t payload_stride, float* d_out,
                             int64_t out_stride, int32_t out_pitch, void* stream) {
  ABCS_NVTX("abcs_gather_decode_batch");
  CHECK_CTX(c);
  if (rows < 1 || cols < 1 || n < 0 || (n > 0 && (!d_images || !d_counts || !d_offsets || !d_payload)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!block_supported(block)) return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  if (pitch < cols * block || image_stride < (int64_t)pitch * (rows * block - 1) + cols * block)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "image pitch/stride smaller than the image");
  if (d_out && (out_pitch < cols * block || out_stride < (int64_t)out_pitch * (rows * block - 1) + cols * block))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "output pitch/stride smaller than the image");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool vec_out = d_out && out_pitch % 2 == 0 && out_stride % 2 == 0 && ((uintptr_t)d_out % 8) == 0;
  if (vec_out && block == 16 && mma16_supported(rows, cols, n))
    return launch_sense16(ctx, 3, rows, cols, n, d_images, image_stride, pitch, 0, 0.0, nullptr, d_counts, d_offsets,
                          d_payload, payload_stride, d_out, out_stride, out_pitch, s);
  if (vec_out && block == 8 && mma16_supported(rows, cols, n))
    return launch_sense8(ctx, true, true, rows, cols, n, d_images, image_stride, pitch, d_counts, d_offsets,
                         d_payload, payload_stride, d_out, out_stride, out_pitch, s);
  int st = launch_gather(ctx, rows, cols, block, d_images, nullptr, image_stride, pitch, n, d_counts, d_offsets,
                         d_payload, payload_stride, s);
  if (st || !d_out) return st;
  return launch_decode(ctx, rows, cols, block, d_counts, d_offsets, d_payload, payload_stride, n, d_out, out_stride,
                       out_pitch, s);
}

int abcs_decode_batch(abcs_ctx* c, int32_t rows, int32_t cols, int32_t block, const uint16_t* d_counts,
                      const int32_t* d_offsets, const float* d_payload, int64_t payload_stride, int32_t n,
                      float* d_out, int64_t out_stride, int32_t out_pitch, const int64_t* d_payload_len,
                      int32_t* d_error, void* stream) {
  ABCS_NVTX("abcs_decode_batch");
  CHECK_CTX(c);
  if (rows < 1 || cols < 1 || n < 0 || (n > 0 && (!d_counts || !d_out)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!block_supported(block)) return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  if (out_pitch < cols * block || out_stride < (int64_t)out_pitch * (rows * block - 1) + cols * block)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "output pitch/stride smaller than the image");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int st;
  const int32_t* offsets = d_offsets;
  if (!offsets || d_error) {
    int32_t* tmp = nullptr;
    if (!d_offsets) {
      tmp = static_cast<int32_t*>(ctx_scratch(ctx, (size_t)n * rows * cols * 4, s, &st));
      if (st) return st;
      offsets = tmp;
    }
    st = launch_offsets(ctx, rows * cols, n, block, d_counts, tmp, d_payload_len, d_error, s);
    if (st) return st;
  }
  return launch_decode(ctx, rows, cols, block, d_counts, offsets, d_payload, payload_stride, n, d_out, out_stride,
                       out_pitch, s);
}

int abcs_forward_batch(abcs_ctx* c, int32_t rows, int32_t cols, int32_t block, const uint16_t* d_counts,
                       const int32_t* d_offsets, const float* d_field, int64_t field_stride, int32_t field_pitch,
                       int32_t n, float* d_y, int64_t y_stride, void* stream) {
  ABCS_NVTX("abcs_forward_batch");
  CHECK_CTX(c);
  if (rows < 1 || cols < 1 || n < 0 || (n > 0 && (!d_counts || !d_field || !d_y)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!block_supported(block)) return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int st;
  const int32_t* offsets = d_offsets;
  if (!offsets) {
    int32_t* tmp = static_cast<int32_t*>(ctx_scratch(ctx, (size_t)n * rows * cols * 4, s, &st));
    if (st) return st;
    st = launch_offsets(ctx, rows * cols, n, block, d_counts, tmp, nullptr, nullptr, s);
    if (st) return st;
    offsets = tmp;
  }
  return launch_gather(ctx, rows, cols, block, nullptr, d_field, field_stride, field_pitch, n, d_counts, offsets, d_y,
                       y_stride, s);
}

int abcs_denoise_dct_batch(abcs_ctx* c, const float* d_field, int32_t height, int32_t width, int64_t field_stride,
                           int32_t n, const double* sigma, double k, int32_t block, float* d_out, void* stream) {
  ABCS_NVTX("abcs_denoise_dct_batch");
  CHECK_CTX(c);
  if (height < 1 || width < 1 || n < 0 || (n > 0 && (!d_field || !d_out || !sigma)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  for (int i = 0; i < n; ++i)
    if (sigma[i] < 0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "denoise: sigma must be >= 0");
  const int b = std::max(1, std::min(block, std::min(height, width)));
  if (b != 8 || height % 4 != 0 || width % 4 != 0)
    return set_error(ABCS_ERR_UNSUPPORTED, "device dct_threshold supports 8x8 tiles on dims divisible by 4");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int st;
  double* thr = static_cast<double*>(ctx_scratch(ctx, (size_t)n * 8, s, &st));
  if (st) return st;
  std::vector<double> h(n);
  for (int i = 0; i < n; ++i) h[i] = k * sigma[i];
  cudaError_t e = cudaMemcpyAsync(thr, h.data(), n * 8, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_status(e, "threshold upload");
  e = cudaStreamSynchronize(s);  // h goes out of scope
  if (e != cudaSuccess) return cuda_status(e, "threshold upload");
  return launch_denoise(ctx, d_field, height, width, field_stride, n, thr, d_out, s);
}

int abcs_ida_batch(abcs_ctx* c, int32_t rows, int32_t cols, int32_t block, const uint16_t* d_counts,
                   const int32_t* d_offsets, const float* d_y, int64_t y_stride, int32_t n, const abcs_ida_config* cfg,
                   const uint8_t* d_ref, int64_t ref_stride, int32_t ref_pitch, float* d_out, int64_t out_stride,
                   int32_t out_pitch, double* d_trace, int32_t* d_diverged, void* stream) {
  ABCS_NVTX("abcs_ida_batch");
  CHECK_CTX(c);
  if (!cfg) return set_error(ABCS_ERR_INVALID_ARGUMENT, "null config");
  // ReconConfig::validate (recon.cpp:39-43)
  if (cfg->iterations < 1) return set_error(ABCS_ERR_INVALID_ARGUMENT, "iterations must be >= 1");
  if (cfg->damping < 1.0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "damping factor D_F must be >= 1");
  if (rows < 1 || cols < 1 || n < 0 || (n > 0 && (!d_counts || !d_y || !d_out)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!block_supported(block)) return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  const int Hc = rows * block, Wc = cols * block;
  const int b = std::max(1, std::min(cfg->denoiser_block, std::min(Hc, Wc)));
  if (b != 8) return set_error(ABCS_ERR_UNSUPPORTED, "device IDA supports the 8x8 dct_threshold denoiser");
  if (out_pitch < Wc) return set_error(ABCS_ERR_INVALID_ARGUMENT, "output pitch smaller than the image");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int st;
  const size_t off_bytes = d_offsets ? 0 : align_up((size_t)n * rows * cols * 4, 256);
  // Images are independent through every iteration (sigma and the halos are per image), so a batch
  // runs as `chains` sub-batch chains on their own streams: each step's last, partial wave of CTAs
  // overlaps another chain's step instead of idling SMs (ABCS_IDA_SPLIT=1 keeps one chain; one chain
  // while the ctx times kernels, so per-launch durations stay those of one step).
  static const int split_env = [] {  // chains per batch (1..4)
    const char* e = getenv("ABCS_IDA_SPLIT");
    return e ? std::max(1, std::min(4, atoi(e))) : 2;
  }();
  const int chains = (!ctx->timing && n >= 8 * split_env && (block == 8 || block == 16)) ? split_env : 1;
  int first[5];
  size_t soff[5];
  soff[0] = 0;
  for (int k = 0; k <= chains; ++k) first[k] = (int)((int64_t)n * k / chains);
  for (int k = 0; k < chains; ++k)
    soff[k + 1] = soff[k] + align_up(ida_scratch_bytes(rows, cols, block, y_stride, first[k + 1] - first[k], *cfg), 256);
  const size_t need = off_bytes + soff[chains];
  char* scr = static_cast<char*>(ctx_scratch(ctx, need, s, &st));
  if (st) return st;
  for (int k = 1; k < chains; ++k)
    if (!ctx->ida_side[k - 1] && cudaStreamCreateWithFlags(&ctx->ida_side[k - 1], cudaStreamNonBlocking) != cudaSuccess)
      return set_error(ABCS_ERR_CUDA, "ida stream");
  if (chains > 1)
    for (auto& e : ctx->ida_ev)
      if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
        return set_error(ABCS_ERR_CUDA, "ida event");
  auto body = [&](cudaStream_t q) -> int {
    const int32_t* offsets = d_offsets;
    if (!offsets) {
      const int r = launch_offsets(ctx, rows * cols, n, block, d_counts, reinterpret_cast<int32_t*>(scr), nullptr,
                                   nullptr, q);
      if (r) return r;
      offsets = reinterpret_cast<int32_t*>(scr);
    }
    if (chains > 1) {
      cudaError_t e = cudaEventRecord(ctx->ida_ev[0], q);
      for (int k = 1; k < chains && e == cudaSuccess; ++k) e = cudaStreamWaitEvent(ctx->ida_side[k - 1], ctx->ida_ev[0], 0);
      if (e != cudaSuccess) return cuda_status(e, "ida fork");
    }
    const int64_t nbk = (int64_t)rows * cols;
    for (int k = 0; k < chains; ++k) {
      const int f0 = first[k], cnt = first[k + 1] - first[k];
      cudaStream_t qk = k ? ctx->ida_side[k - 1] : q;
      const int r = launch_ida(ctx, rows, cols, block, d_counts + f0 * nbk, offsets + f0 * nbk, d_y + f0 * y_stride,
                               y_stride, cnt, *cfg, d_ref ? d_ref + f0 * ref_stride : nullptr, ref_stride, ref_pitch,
                               d_out + f0 * out_stride, out_stride, out_pitch,
                               d_trace ? d_trace + (int64_t)f0 * (cfg->iterations + 1) * 4 : nullptr,
                               d_diverged ? d_diverged + 2 * (int64_t)f0 : nullptr, scr + off_bytes + soff[k], qk);
      if (r) return r;
    }
    for (int k = 1; k < chains; ++k) {
      cudaError_t e = cudaEventRecord(ctx->ida_ev[k], ctx->ida_side[k - 1]);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(q, ctx->ida_ev[k], 0);
      if (e != cudaSuccess) return cuda_status(e, "ida join");
    }
    return ABCS_OK;
  };
  if (!ctx->use_graphs || ctx->timing) return body(s);
  // one CUDA graph per distinct argument set (every pointer, size and setting of this call)
  auto u = [](const void* p) { return (uint64_t)reinterpret_cast<uintptr_t>(p); };
  uint64_t dbits, kbits;
  memcpy(&dbits, &cfg->damping, 8);
  memcpy(&kbits, &cfg->k, 8);
  const std::vector<uint64_t> key = {(uint64_t)rows, (uint64_t)cols, (uint64_t)block, u(d_counts), u(d_offsets),
                                     u(d_y), (uint64_t)y_stride, (uint64_t)n, (uint64_t)cfg->iterations,
                                     (uint64_t)cfg->denoiser_block, dbits, kbits, u(d_ref), (uint64_t)ref_stride,
                                     (uint64_t)ref_pitch, u(d_out), (uint64_t)out_stride, (uint64_t)out_pitch,
                                     u(d_trace), u(d_diverged), u(scr)};
  Ctx::GraphEntry* hit = nullptr;
  for (auto& g : ctx->graphs)
    if (g.key == key) hit = &g;
  if (!hit) {
    if (!ctx->capture && cudaStreamCreateWithFlags(&ctx->capture, cudaStreamNonBlocking) != cudaSuccess)
      return body(s);
    const int64_t l0 = ctx->launches;
    if (cudaStreamBeginCapture(ctx->capture, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return body(s);
    const int r = body(ctx->capture);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(ctx->capture, &graph);
    if (r) {
      if (graph) cudaGraphDestroy(graph);
      ctx->launches = l0;
      return r;
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = ce == cudaSuccess ? cudaGraphInstantiate(&exec, graph, 0) : ce;
    if (graph) cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      cudaGetLastError();
      ctx->launches = l0;
      return body(s);  // capture unsupported here: plain launches
    }
    if (ctx->graphs.size() >= 16) {  // bounded cache: drop the oldest
      cudaGraphExecDestroy(ctx->graphs.front().exec);
      ctx->graphs.erase(ctx->graphs.begin());
    }
    ctx->graphs.push_back({key, exec, ctx->launches - l0});
    ctx->launches = l0;
    hit = &ctx->graphs.back();
  }
  ctx->launches += hit->launches;
  return cuda_status(cudaGraphLaunch(hit->exec, s), "ida graph launch");
}

// Shared argument checks and offsets for the explicit-state entry points.
static int ida_state_common(abcs_ctx* c, int32_t rows, int32_t cols, int32_t block, const uint16_t* d_counts,
                            const int32_t* d_offsets, const float* d_y, int32_t n, const float* d_x, const float* d_z,
                            const double* d_sigma, int64_t y_stride, void* stream, char** scr_out,
                            const int32_t** offsets_out) {
  if (rows < 1 || cols < 1 || n < 0 || (n > 0 && (!d_counts || !d_y || !d_x || !d_z || !d_sigma)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!block_supported(block)) return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int st;
  const size_t off_bytes = d_offsets ? 0 : align_up((size_t)n * rows * cols * 4, 256);
  const size_t need = off_bytes + ida_state_scratch_bytes(rows, cols, block, y_stride, n);
  char* scr = static_cast<char*>(ctx_scratch(ctx, need, s, &st));
  if (st) return st;
  const int32_t* offsets = d_offsets;
  if (!offsets) {
    st = launch_offsets(ctx, rows * cols, n, block, d_counts, reinterpret_cast<int32_t*>(scr), nullptr, nullptr, s);
    if (st) return st;
    offsets = reinterpret_cast<int32_t*>(scr);
  }
  *scr_out = scr + off_bytes;
  *offsets_out = offsets;
  return ABCS_OK;
}

int abcs_ida_init_state(abcs_ctx* c, int32_t rows, int32_t cols, int32_t block, const uint16_t* d_counts,
                        const int32_t* d_offsets, const float* d_y, int64_t y_stride, int32_t n, int32_t warm,
                        float* d_x, float* d_z, double* d_sigma, void* stream) {
  ABCS_NVTX("abcs_ida_init_state");
  CHECK_CTX(c);
  if (n == 0) return ABCS_OK;
  char* scr;
  const int32_t* offsets;
  int st = ida_state_common(c, rows, cols, block, d_counts, d_offsets, d_y, n, d_x, d_z, d_sigma, y_stride, stream,
                            &scr, &offsets);
  if (st) return st;
  return launch_ida_state(reinterpret_cast<Ctx*>(c), true, rows, cols, block, d_counts, offsets, d_y, y_stride, n,
                          warm ? 1 : 0, 1.0, 0.0, d_x, d_z, d_sigma, 0, nullptr, scr,
                          reinterpret_cast<cudaStream_t>(stream));
}

int abcs_ida_step_state(abcs_ctx* c, int32_t rows, int32_t cols, int32_t block, const uint16_t* d_counts,
                        const int32_t* d_offsets, const float* d_y, int64_t y_stride, int32_t n,
                        const abcs_ida_config* cfg, float* d_x, float* d_z, double* d_sigma, int32_t iteration,
                        int32_t* d_diverged, void* stream) {
  ABCS_NVTX("abcs_ida_step_state");
  CHECK_CTX(c);
  if (!cfg) return set_error(ABCS_ERR_INVALID_ARGUMENT, "null config");
  if (cfg->damping < 1.0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "damping factor D_F must be >= 1");
  const int Hc = rows * block, Wc = cols * block;
  const int b = std::max(1, std::min(cfg->denoiser_block, std::min(Hc, Wc)));
  if (b != 8) return set_error(ABCS_ERR_UNSUPPORTED, "device IDA supports the 8x8 dct_threshold denoiser");
  if (iteration < 1) return set_error(ABCS_ERR_INVALID_ARGUMENT, "iteration numbers start at 1");
  if (n == 0) return ABCS_OK;
  char* scr;
  const int32_t* offsets;
  int st = ida_state_common(c, rows, cols, block, d_counts, d_offsets, d_y, n, d_x, d_z, d_sigma, y_stride, stream,
                            &scr, &offsets);
  if (st) return st;
  return launch_ida_state(reinterpret_cast<Ctx*>(c), false, rows, cols, block, d_counts, offsets, d_y, y_stride, n, 1,
                          cfg->damping, cfg->k, d_x, d_z, d_sigma, iteration, d_diverged, scr,
                          reinterpret_cast<cudaStream_t>(stream));
}

int abcs_psnr_batch(abcs_ctx* c, const uint8_t* d_ref, int64_t ref_stride, int32_t ref_pitch, const float* d_img,
                    int64_t img_stride, int32_t img_pitch, int32_t height, int32_t width, int32_t n, double* d_psnr,
                    void* stream) {
  CHECK_CTX(c);
  if (height < 1 || width < 1 || n < 0 || ref_pitch < width || img_pitch < width ||
      (n > 0 && (!d_ref || !d_img || !d_psnr)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  return launch_psnr(ctx, d_ref, ref_stride, ref_pitch, d_img, img_stride, img_pitch, height, width, n, d_psnr,
                     reinterpret_cast<cudaStream_t>(stream));
}

int abcs_ssim_batch(abcs_ctx* c, const uint8_t* d_ref, int64_t ref_stride, int32_t ref_pitch, const float* d_img,
                    int64_t img_stride, int32_t img_pitch, int32_t height, int32_t width, int32_t n, double* d_ssim,
                    void* stream) {
  CHECK_CTX(c);
  if (height < 1 || width < 1 || n < 0 || ref_pitch < width || img_pitch < width ||
      (n > 0 && (!d_ref || !d_img || !d_ssim)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (height < 11 || width < 11)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "ssim: images smaller than the 11x11 window");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  return launch_ssim(ctx, d_ref, ref_stride, ref_pitch, d_img, img_stride, img_pitch, height, width, n, d_ssim,
                     reinterpret_cast<cudaStream_t>(stream));
}

int abcs_quality_batch(abcs_ctx* c, const uint8_t* d_ref, int64_t ref_stride, int32_t ref_pitch, const float* d_img,
                       int64_t img_stride, int32_t img_pitch, int32_t height, int32_t width, int32_t n,
                       double* d_mse, double* d_psnr, double* d_ssim, void* stream) {
  ABCS_NVTX("abcs_quality_batch");
  CHECK_CTX(c);
  if (height < 1 || width < 1 || n < 0 || ref_pitch < width || img_pitch < width ||
      (n > 0 && (!d_ref || !d_img || (!d_mse && !d_psnr && !d_ssim))))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (d_ssim && (height < 11 || width < 11))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "ssim: images smaller than the 11x11 window");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (d_mse || d_psnr) {
    const int st = launch_psnr(ctx, d_ref, ref_stride, ref_pitch, d_img, img_stride, img_pitch, height, width, n,
                               d_psnr, s, d_mse);
    if (st) return st;
  }
  if (d_ssim) return launch_ssim(ctx, d_ref, ref_stride, ref_pitch, d_img, img_stride, img_pitch, height, width, n,
                                 d_ssim, s);
  return ABCS_OK;
}

// ReconConfig::validate (recon.cpp:39-43) + the device path's denoiser restrictions
static int recon_config_check(const abcs_recon_config* cfg, int32_t Hc, int32_t Wc) {
  if (!cfg) return set_error(ABCS_ERR_INVALID_ARGUMENT, "null config");
  if (cfg->iterations < 1) return set_error(ABCS_ERR_INVALID_ARGUMENT, "iterations must be >= 1");
  if (cfg->damping < 1.0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "damping factor D_F must be >= 1");
  if (cfg->lambda < 0.0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "lambda must be >= 0");
  if (cfg->method < ABCS_RECON_IDCT || cfg->method > ABCS_RECON_IDA)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "unknown reconstruction method");
  const bool uses_denoiser = cfg->method >= ABCS_RECON_DAMP;
  if (uses_denoiser) {
    if (cfg->denoiser == ABCS_DENOISER_DCT_THRESHOLD) {
      const int b = std::max(1, std::min(cfg->denoiser_block, std::min(Hc, Wc)));
      if (b != 8 || Hc % 4 || Wc % 4)
        return set_error(ABCS_ERR_UNSUPPORTED, "device dct_threshold supports 8x8 tiles on dims divisible by 4");
    } else if (cfg->denoiser == ABCS_DENOISER_BLUR) {
      if (!(cfg->sigma_scale > 0.0)) return set_error(ABCS_ERR_UNSUPPORTED, "blur denoiser needs sigma_scale > 0");
    } else if (cfg->denoiser != ABCS_DENOISER_IDENTITY) {
      return set_error(ABCS_ERR_INVALID_ARGUMENT, "unknown denoiser");
    }
  }
  return ABCS_OK;
}

int abcs_reconstruct_batch(abcs_ctx* c, int32_t rows, int32_t cols, int32_t block, const uint16_t* d_counts,
                           const int32_t* d_offsets, const float* d_y, int64_t y_stride, int32_t n,
                           const abcs_recon_config* cfg, const uint8_t* d_ref, int64_t ref_stride, int32_t ref_pitch,
                           float* d_out, int64_t out_stride, int32_t out_pitch, double* d_trace, int32_t* d_diverged,
                           void* stream) {
  ABCS_NVTX("abcs_reconstruct_batch");
  CHECK_CTX(c);
  if (rows < 1 || cols < 1 || n < 0 || (n > 0 && (!d_counts || !d_y || !d_out)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!block_supported(block)) return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  int st = recon_config_check(cfg, rows * block, cols * block);
  if (st) return st;
  if (out_pitch < cols * block) return set_error(ABCS_ERR_INVALID_ARGUMENT, "output pitch smaller than the image");
  if (n == 0) return ABCS_OK;
  if (cfg->method == ABCS_RECON_IDCT)
    return abcs_decode_batch(c, rows, cols, block, d_counts, d_offsets, d_y, y_stride, n, d_out, out_stride,
                             out_pitch, nullptr, nullptr, stream);
  if (cfg->method == ABCS_RECON_IDA && cfg->denoiser == ABCS_DENOISER_DCT_THRESHOLD) {
    abcs_ida_config ic{};
    ic.iterations = cfg->iterations;
    ic.denoiser_block = cfg->denoiser_block;
    ic.damping = cfg->damping;
    ic.k = cfg->k;
    return abcs_ida_batch(c, rows, cols, block, d_counts, d_offsets, d_y, y_stride, n, &ic, d_ref, ref_stride,
                          ref_pitch, d_out, out_stride, out_pitch, d_trace, d_diverged, stream);
  }
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  return launch_recon(ctx, false, rows, cols, block, d_counts, d_offsets, d_y, y_stride, n, *cfg, d_ref, ref_stride,
                      ref_pitch, nullptr, nullptr, nullptr, 0, d_out, out_stride, out_pitch, d_trace, d_diverged,
                      reinterpret_cast<cudaStream_t>(stream));
}

int abcs_recon_step_state(abcs_ctx* c, int32_t rows, int32_t cols, int32_t block, const uint16_t* d_counts,
                          const int32_t* d_offsets, const float* d_y, int64_t y_stride, int32_t n,
                          const abcs_recon_config* cfg, float* d_x, float* d_z, double* d_sigma, int32_t iteration,
                          int32_t* d_diverged, void* stream) {
  ABCS_NVTX("abcs_recon_step_state");
  CHECK_CTX(c);
  if (rows < 1 || cols < 1 || n < 0 || (n > 0 && (!d_counts || !d_y || !d_x || !d_z || !d_sigma)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!block_supported(block)) return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  int st = recon_config_check(cfg, rows * block, cols * block);
  if (st) return st;
  if (cfg->method == ABCS_RECON_IDCT) return set_error(ABCS_ERR_INVALID_ARGUMENT, "Idct has no iteration step");
  if (iteration < 0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "iteration must be >= 0");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  return launch_recon(ctx, true, rows, cols, block, d_counts, d_offsets, d_y, y_stride, n, *cfg, nullptr, 0, 0, d_x,
                      d_z, d_sigma, iteration, nullptr, 0, 0, nullptr, d_diverged,
                      reinterpret_cast<cudaStream_t>(stream));
}

int abcs_denoise_batch(abcs_ctx* c, const float* d_field, int32_t height, int32_t width, int64_t field_stride,
                       int32_t n, const double* sigma, const abcs_recon_config* cfg, float* d_out, void* stream) {
  ABCS_NVTX("abcs_denoise_batch");
  CHECK_CTX(c);
  if (!cfg || height < 1 || width < 1 || n < 0 || (n > 0 && (!d_field || !d_out || !sigma)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  for (int i = 0; i < n; ++i)
    if (sigma[i] < 0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "denoise: sigma must be >= 0");
  if (cfg->denoiser == ABCS_DENOISER_DCT_THRESHOLD)
    return abcs_denoise_dct_batch(c, d_field, height, width, field_stride, n, sigma, cfg->k, cfg->denoiser_block,
                                  d_out, stream);
  if (field_stride != (int64_t)height * width)
    return set_error(ABCS_ERR_UNSUPPORTED, "blur / identity denoisers take dense fields");
  if (cfg->denoiser == ABCS_DENOISER_BLUR && !(cfg->sigma_scale > 0.0))
    return set_error(ABCS_ERR_UNSUPPORTED, "blur denoiser needs sigma_scale > 0");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t N = (int64_t)height * width;
  int st;
  char* scr = static_cast<char*>(ctx_scratch(ctx, align_up((size_t)n * N * 4, 256) + align_up((size_t)n * 8, 256),
                                             s, &st));
  if (st) return st;
  double* sig = reinterpret_cast<double*>(scr + align_up((size_t)n * N * 4, 256));
  cudaError_t e = cudaMemcpyAsync(sig, sigma, (size_t)n * 8, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e, "sigma upload");
  return run_denoiser(ctx, *cfg, d_field, d_out, reinterpret_cast<float*>(scr), height, width, n, sig, nullptr, s);
}

int abcs_rademacher_probe(abcs_ctx* c, uint64_t seed, int64_t n, float* d_probe, void* stream) {
  CHECK_CTX(c);
  if (n < 0 || (n > 0 && !d_probe)) return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  return launch_probe(ctx, seed, n, d_probe, reinterpret_cast<cudaStream_t>(stream));
}

int abcs_divergence_batch(abcs_ctx* c, const float* d_field, int32_t height, int32_t width, int32_t n,
                          const double* sigma, const double* epsilon, uint64_t seed, const abcs_recon_config* cfg,
                          double* d_div, void* stream) {
  ABCS_NVTX("abcs_divergence_batch");
  CHECK_CTX(c);
  if (!cfg || height < 1 || width < 1 || n < 0 || (n > 0 && (!d_field || !d_div || !sigma || !epsilon)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  for (int i = 0; i < n; ++i)
    if (!(epsilon[i] > 0)) return set_error(ABCS_ERR_INVALID_ARGUMENT, "divergence: epsilon must be > 0");
  if (cfg->denoiser == ABCS_DENOISER_DCT_THRESHOLD && (height % 4 || width % 4 ||
                                                       std::max(1, std::min(cfg->denoiser_block,
                                                                            std::min(height, width))) != 8))
    return set_error(ABCS_ERR_UNSUPPORTED, "device dct_threshold supports 8x8 tiles on dims divisible by 4");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t N = (int64_t)height * width;
  const size_t fld = align_up((size_t)n * N * 4, 256);
  const size_t parts = divergence_partials(ctx, N, n);
  int st;
  char* p = static_cast<char*>(ctx_scratch(ctx, 4 * fld + align_up((size_t)N * 4, 256) + 3 * align_up((size_t)n * 8, 256) +
                                                   align_up(parts * 8, 256), s, &st));
  if (st) return st;
  float* base = reinterpret_cast<float*>(p);
  float* pert = reinterpret_cast<float*>(p + fld);
  float* moved = reinterpret_cast<float*>(p + 2 * fld);
  float* tmp = reinterpret_cast<float*>(p + 3 * fld);
  float* probe = reinterpret_cast<float*>(p + 4 * fld);
  double* sig = reinterpret_cast<double*>(p + 4 * fld + align_up((size_t)N * 4, 256));
  double* eps = sig + align_up((size_t)n * 8, 256) / 8;
  double* thr = eps + align_up((size_t)n * 8, 256) / 8;
  double* partials = thr + align_up((size_t)n * 8, 256) / 8;
  cudaError_t e = cudaMemcpyAsync(sig, sigma, (size_t)n * 8, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(eps, epsilon, (size_t)n * 8, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e, "divergence upload");
  st = launch_probe(ctx, seed, N, probe, s);
  if (!st) st = launch_divergence_given(ctx, d_field, probe, nullptr, N, n, eps, pert, nullptr, nullptr, nullptr, true, s);
  if (!st) st = run_denoiser(ctx, *cfg, d_field, base, tmp, height, width, n, sig, thr, s);
  if (!st) st = run_denoiser(ctx, *cfg, pert, moved, tmp, height, width, n, sig, thr, s);
  if (!st) st = launch_divergence_given(ctx, nullptr, probe, base, N, n, eps, nullptr, moved, partials, d_div, false, s);
  return st;
}

int abcs_ida_check(const int32_t* h_diverged, int32_t n, int32_t* first_image) {
  if (first_image) *first_image = -1;
  if (!h_diverged) return ABCS_OK;
  for (int i = 0; i < n; ++i) {
    const int it = h_diverged[2 * i], kind = h_diverged[2 * i + 1];
    if (it > 0) {
      if (first_image) *first_image = i;
      const char* what = kind == 1 ? "non-finite estimate" : (kind == 2 ? "|x| > 1e6" : "non-finite residual");
      return set_error(ABCS_ERR_DIVERGENCE,
                       std::string("solver diverged (") + what + ") at iteration " + std::to_string(it));
    }
  }
  return ABCS_OK;
}

int abcs_synth_generate(abcs_ctx* c, const abcs_synth_spec* spec, int64_t first_index, int32_t n, uint8_t* d_out,
                        int64_t image_stride, void* stream) {
  CHECK_CTX(c);
  if (!spec || n < 0 || (n > 0 && !d_out)) return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (spec->height < 1 || spec->width < 1 || spec->n_ellipses < 0 || spec->n_ellipses > SG_MAX_ELLIPSES)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad synth spec");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int st;
  void* scr = ctx_scratch(ctx, (size_t)n * sizeof(sg_scene), s, &st);
  if (st) return st;
  return launch_synth(ctx, *spec, first_index, n, d_out, image_stride, scr, s);
}

// Chunked H2D -> sense -> decode -> D2H over the ctx's three streams: each
// stream owns one slot of device buffers, so chunk i's copies overlap the other
// streams' kernels. Inputs/outputs are host buffers (pinned for full PCIe
// rate); the slot buffers are cached in the ctx across calls.
// The host-buffer sweep. h_out (per plan decoded pixels) and/or h_cells (mse, psnr, ssim per
// plan and image: the bench cells of abcs_main.cpp:226-258) come back to the host.
static int sweep_host_impl(Ctx* ctx, const abcs_sense_plan* plans, int32_t n_plans, const uint8_t* h_images,
                           int32_t n, float* const* h_out, double* const* h_cells, int32_t chunk) {
  if (n == 0) return ABCS_OK;
  cudaSetDevice(ctx->device);
  if (chunk <= 0) chunk = 16;
  if (chunk > n) chunk = n;
  constexpr int kSlots = 3;
  const abcs_sense_plan& p0 = plans[0];
  const bool want_px = h_out != nullptr, want_cells = h_cells != nullptr;
  const int64_t px_in = (int64_t)p0.height * p0.width;
  // per slot: the images once; per plan counts, offsets, payload, side, pixels; the sweep scratch
  size_t b_plan[4], per_slot = align_up(chunk * px_in, 256);
  int64_t px_out[4];
  for (int j = 0; j < n_plans; ++j) {
    const abcs_sense_plan& q = plans[j];
    px_out[j] = (int64_t)q.rows * q.block * q.cols * q.block;
    b_plan[j] = align_up(chunk * q.n_blocks * 2, 256) + align_up(chunk * q.n_blocks * 4, 256) +
                align_up(chunk * q.coeffs_per_image * 4 + 4, 256) + align_up(chunk * q.side_per_image * 4 + 4, 256) +
                align_up(chunk * px_out[j] * 4, 256);
    per_slot += b_plan[j];
  }
  // cells plus the metric kernels' partial sums: each slot owns its own (the slots run concurrently)
  size_t b_mpart = 0;
  for (int j = 0; j < n_plans && want_cells; ++j) {
    const int h = plans[j].rows * plans[j].block, w = plans[j].cols * plans[j].block;
    b_mpart = std::max(b_mpart, align_up(std::max(psnr_scratch_bytes(h, chunk),
                                                  h_cells[2] ? ssim_scratch_bytes(h, w, chunk) : 0), 256));
  }
  const size_t b_cells = want_cells ? align_up(3 * n_plans * chunk * sizeof(double), 256) + b_mpart : 0;
  per_slot += b_cells;
  const bool shared = sweep_shared(ctx, plans, n_plans, chunk);
  size_t b_scr = 0;
  if (shared) {
    b_scr = align_up(sweep_scratch_bytes(plans, n_plans, chunk, nullptr), 256);
  } else {
    for (int j = 0; j < n_plans; ++j) b_scr = std::max(b_scr, align_up(sense_scratch_bytes(&plans[j], chunk, true), 256));
  }
  per_slot += b_scr;
  if (per_slot * kSlots > ctx->pipe_bytes) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess && ctx->pipe_buf) e = cudaFree(ctx->pipe_buf);
    if (e != cudaSuccess) return cuda_status(e, "pipeline realloc");
    ctx->pipe_buf = nullptr;
    ctx->pipe_bytes = 0;
    e = cudaMalloc(&ctx->pipe_buf, per_slot * kSlots);
    if (e != cudaSuccess) return cuda_status(e, "pipeline alloc");
    ctx->pipe_bytes = per_slot * kSlots;
  }
  const int saved_streams = ctx->pipe_streams;
  ctx->pipe_streams = 1;  // each slot's sweep runs serialised on its own stream; the slots overlap
  int st = ABCS_OK;
  const int nchunks = (n + chunk - 1) / chunk;
  for (int ci = 0; ci < nchunks && st == ABCS_OK; ++ci) {
    const int k = ci % kSlots;
    char* base = static_cast<char*>(ctx->pipe_buf) + per_slot * k;
    uint8_t* img = reinterpret_cast<uint8_t*>(base);
    char* q = base + align_up(chunk * px_in, 256);
    uint16_t* counts[4];
    int32_t* offsets[4];
    float *payload[4], *side[4], *out[4];
    for (int j = 0; j < n_plans; ++j) {
      const abcs_sense_plan& pl = plans[j];
      counts[j] = reinterpret_cast<uint16_t*>(q);
      q += align_up(chunk * pl.n_blocks * 2, 256);
      offsets[j] = reinterpret_cast<int32_t*>(q);
      q += align_up(chunk * pl.n_blocks * 4, 256);
      payload[j] = reinterpret_cast<float*>(q);
      q += align_up(chunk * pl.coeffs_per_image * 4 + 4, 256);
      side[j] = reinterpret_cast<float*>(q);
      q += align_up(chunk * pl.side_per_image * 4 + 4, 256);
      out[j] = reinterpret_cast<float*>(q);
      q += align_up(chunk * px_out[j] * 4, 256);
    }
    double* cells = reinterpret_cast<double*>(q);  // [plan][mse, psnr, ssim][chunk]
    q += b_cells;
    char* scr = q;
    const int first = ci * chunk;
    const int cnt = std::min(chunk, n - first);
    cudaStream_t s = ctx->pipe[k];
    cudaError_t e = cudaMemcpyAsync(img, h_images + first * px_in, cnt * px_in, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) {
      st = cuda_status(e, "h2d");
      break;
    }
    if (shared) {
      st = sweep_impl(ctx, plans, n_plans, img, px_in, p0.width, cnt, 0, counts, offsets, payload, out,
                      px_out[0], plans[0].cols * plans[0].block, scr, s, k);
    } else {
      for (int j = 0; j < n_plans && st == ABCS_OK; ++j)
        st = sense_impl(ctx, &plans[j], img, px_in, p0.width, cnt, counts[j], offsets[j], payload[j], side[j], scr, s,
                        out[j], px_out[j], plans[j].cols * plans[j].block);
    }
    if (st) break;
    void* mpart = reinterpret_cast<char*>(cells) + align_up(3 * n_plans * chunk * sizeof(double), 256);
    for (int j = 0; j < n_plans && want_cells && st == ABCS_OK; ++j) {
      // psnr/ssim against the image cropped to the block grid (abcs_main.cpp:230, 254-255)
      const abcs_sense_plan& pl = plans[j];
      const int h = pl.rows * pl.block, w = pl.cols * pl.block;
      double* cj = cells + 3 * j * chunk;
      st = launch_psnr(ctx, img, px_in, p0.width, out[j], px_out[j], w, h, w, cnt, cj + chunk, s, cj, mpart);
      if (st == ABCS_OK && h_cells[2])
        st = launch_ssim(ctx, img, px_in, p0.width, out[j], px_out[j], w, h, w, cnt, cj + 2 * chunk, s, mpart);
    }
    if (st) break;
    for (int j = 0; j < n_plans && want_px && e == cudaSuccess; ++j)
      e = cudaMemcpyAsync(h_out[j] + first * px_out[j], out[j], cnt * px_out[j] * 4, cudaMemcpyDeviceToHost, s);
    for (int j = 0; j < n_plans && want_cells && e == cudaSuccess; ++j)
      for (int m = 0; m < 3 && e == cudaSuccess; ++m)
        if (h_cells[m])
          e = cudaMemcpyAsync(h_cells[m] + (int64_t)j * n + first, cells + (3 * j + m) * chunk, cnt * sizeof(double),
                              cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) st = cuda_status(e, "d2h");
  }
  for (auto& s : ctx->pipe) {
    const cudaError_t e = cudaStreamSynchronize(s);
    if (st == ABCS_OK && e != cudaSuccess) st = cuda_status(e, "pipeline sync");
  }
  ctx->pipe_streams = saved_streams;
  return st;
}

static int sweep_host_check(const abcs_sense_plan* plans, int32_t n_plans, const uint8_t* h_images, int32_t n,
                            bool have_out) {
  if (!plans || n_plans < 1 || n_plans > 4 || n < 0 || (n > 0 && (!h_images || !have_out)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  for (int j = 0; j < n_plans; ++j) {
    if (!block_supported(plans[j].block)) return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
    if (plans[j].height != plans[0].height || plans[j].width != plans[0].width)
      return set_error(ABCS_ERR_INVALID_ARGUMENT, "sweep plans must share the image size");
  }
  return ABCS_OK;
}

int abcs_sense_decode_sweep_host(abcs_ctx* c, const abcs_sense_plan* plans, int32_t n_plans, const uint8_t* h_images,
                                 int32_t n, float* const* h_out, int32_t chunk) {
  ABCS_NVTX("abcs_sense_decode_sweep_host");
  CHECK_CTX(c);
  if (int st = sweep_host_check(plans, n_plans, h_images, n, h_out != nullptr)) return st;
  for (int j = 0; j < n_plans && n > 0; ++j)
    if (!h_out[j]) return set_error(ABCS_ERR_INVALID_ARGUMENT, "null output for a plan");
  return sweep_host_impl(reinterpret_cast<Ctx*>(c), plans, n_plans, h_images, n, h_out, nullptr, chunk);
}

int abcs_bench_cells_host(abcs_ctx* c, const abcs_sense_plan* plans, int32_t n_plans, const uint8_t* h_images,
                          int32_t n, double* h_mse, double* h_psnr, double* h_ssim, int32_t chunk) {
  ABCS_NVTX("abcs_bench_cells_host");
  CHECK_CTX(c);
  if (int st = sweep_host_check(plans, n_plans, h_images, n, h_mse || h_psnr || h_ssim)) return st;
  for (int j = 0; j < n_plans && h_ssim; ++j)
    if (plans[j].rows * plans[j].block < 11 || plans[j].cols * plans[j].block < 11)
      return set_error(ABCS_ERR_INVALID_ARGUMENT, "ssim: images smaller than the 11x11 window");
  double* const cells[3] = {h_mse, h_psnr, h_ssim};
  return sweep_host_impl(reinterpret_cast<Ctx*>(c), plans, n_plans, h_images, n, nullptr, cells, chunk);
}

int abcs_sense_decode_host(abcs_ctx* c, const abcs_sense_plan* p, const uint8_t* h_images, int32_t n, float* h_out,
                           uint16_t* h_counts, float* h_payload, int32_t chunk) {
  ABCS_NVTX("abcs_sense_decode_host");
  CHECK_CTX(c);
  if (!p || n < 0 || (n > 0 && (!h_images || !h_out))) return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!block_supported(p->block)) return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  if (n == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  if (chunk <= 0) chunk = 16;
  if (chunk > n) chunk = n;
  constexpr int kSlots = 3;
  const int64_t px_in = (int64_t)p->height * p->width;
  const int64_t px_out = (int64_t)p->rows * p->block * p->cols * p->block;
  const int64_t K = p->coeffs_per_image, S = p->side_per_image, NB = p->n_blocks;
  const size_t b_img = align_up(chunk * px_in, 256), b_cnt = align_up(chunk * NB * 2, 256),
               b_off = align_up(chunk * NB * 4, 256), b_pay = align_up(chunk * K * 4 + 4, 256),
               b_side = align_up(chunk * S * 4 + 4, 256), b_out = align_up(chunk * px_out * 4, 256),
               b_scr = align_up(sense_scratch_bytes(p, chunk, true), 256);
  const size_t per_slot = b_img + b_cnt + b_off + b_pay + b_side + b_out + b_scr;
  if (per_slot * kSlots > ctx->pipe_bytes) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess && ctx->pipe_buf) e = cudaFree(ctx->pipe_buf);
    if (e != cudaSuccess) return cuda_status(e, "pipeline realloc");
    ctx->pipe_buf = nullptr;
    ctx->pipe_bytes = 0;
    e = cudaMalloc(&ctx->pipe_buf, per_slot * kSlots);
    if (e != cudaSuccess) return cuda_status(e, "pipeline alloc");
    ctx->pipe_bytes = per_slot * kSlots;
  }
  int st = ABCS_OK;
  const int nchunks = (n + chunk - 1) / chunk;
  for (int ci = 0; ci < nchunks && st == ABCS_OK; ++ci) {
    const int k = ci % kSlots;
    char* base = static_cast<char*>(ctx->pipe_buf) + per_slot * k;
    uint8_t* img = reinterpret_cast<uint8_t*>(base);
    uint16_t* counts = reinterpret_cast<uint16_t*>(base + b_img);
    int32_t* offsets = reinterpret_cast<int32_t*>(base + b_img + b_cnt);
    float* payload = reinterpret_cast<float*>(base + b_img + b_cnt + b_off);
    float* side = reinterpret_cast<float*>(base + b_img + b_cnt + b_off + b_pay);
    float* out = reinterpret_cast<float*>(base + b_img + b_cnt + b_off + b_pay + b_side);
    char* scr = base + b_img + b_cnt + b_off + b_pay + b_side + b_out;
    const int first = ci * chunk;
    const int cnt = std::min(chunk, n - first);
    cudaStream_t s = ctx->pipe[k];
    cudaError_t e = cudaMemcpyAsync(img, h_images + first * px_in, cnt * px_in, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { st = cuda_status(e, "h2d"); break; }
    st = sense_impl(ctx, p, img, px_in, p->width, cnt, counts, offsets, payload, side, scr, s, out, px_out,
                    p->cols * p->block);
    if (st) break;
    e = cudaMemcpyAsync(h_out + first * px_out, out, cnt * px_out * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && h_counts)
      e = cudaMemcpyAsync(h_counts + first * NB, counts, cnt * NB * 2, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && h_payload)
      e = cudaMemcpyAsync(h_payload + first * K, payload, cnt * K * 4, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) { st = cuda_status(e, "d2h"); break; }
  }
  for (auto& s : ctx->pipe) {
    const cudaError_t e = cudaStreamSynchronize(s);
    if (st == ABCS_OK && e != cudaSuccess) st = cuda_status(e, "pipeline sync");
  }
  return st;
}

}  // extern "C"
