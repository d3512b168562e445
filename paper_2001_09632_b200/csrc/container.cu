// The .abcs v1 measurement container (container.cpp:58-149, container.hpp:8-14) packed
// and unpacked on the device, straight from / into the batched sense buffers:
//
//   "ABCS" | version u16 = 1 | H u32 | W u32 | B u16 | algorithm u8 | C_R num u32 |
//   C_R den u32 | threshold f64 | n_B u32 | counts u16[n_B] | coeffs f32[K] |
//   side count u32 | side f32[S]                     (little-endian, packed)
//
// The 37-byte header puts counts and coefficients at byte (not word) alignment, so
// each pack thread builds one aligned output word from two aligned source words with
// a funnel shift (byte-wise only where a word straddles two segments), and each unpack
// thread assembles one count / coefficient / side value the same way. A batch shares
// one plan, hence one header layout; unpack validates every container against it
// with the reference reader's checks (magic, version, header fields, counts <= B^2,
// sum(counts) == K, side count) and reports a status per container.
#include <cstring>

#include "internal.h"

namespace abcs_b200 {

constexpr int kHdr = 37;

struct ContainerLayout {
  int64_t nB, K, S;
  int64_t c_end, p_end, sc_end, total;
};

static ContainerLayout layout_of(const abcs_sense_plan& p) {
  ContainerLayout L;
  L.nB = p.n_blocks;
  L.K = p.coeffs_per_image;
  L.S = p.side_per_image;
  L.c_end = kHdr + 2 * L.nB;
  L.p_end = L.c_end + 4 * L.K;
  L.sc_end = L.p_end + 4;
  L.total = L.sc_end + 4 * L.S;
  return L;
}

template <typename T>
static void put_le(uint8_t*& p, T v) {  // host is little-endian (x86-64 / aarch64 LE)
  std::memcpy(p, &v, sizeof(T));
  p += sizeof(T);
}

static void header_bytes(const abcs_sense_plan& p, uint8_t* out) {
  uint8_t* q = out;
  const char magic[4] = {'A', 'B', 'C', 'S'};
  std::memcpy(q, magic, 4);
  q += 4;
  put_le<uint16_t>(q, 1);
  put_le<uint32_t>(q, (uint32_t)p.height);
  put_le<uint32_t>(q, (uint32_t)p.width);
  put_le<uint16_t>(q, (uint16_t)p.block);
  put_le<uint8_t>(q, (uint8_t)p.algorithm_used);
  put_le<uint32_t>(q, p.cr_num);
  put_le<uint32_t>(q, p.cr_den);
  put_le<double>(q, p.threshold);
  put_le<uint32_t>(q, (uint32_t)p.n_blocks);
}

struct ContainerArgs {
  uint8_t hdr[40];
  ContainerLayout L;
  const uint16_t* counts;
  const float* payload;
  const float* side;
  uint8_t* out;
  const uint8_t* in;
  int64_t stride;  // bytes between containers
  uint16_t* counts_out;
  float* payload_out;
  float* side_out;
  abcs_container_info* info;
  int block;
  int n;
};

__device__ __forceinline__ uint32_t pack_byte(const ContainerArgs& a, int64_t img, int64_t pos) {
  const ContainerLayout& L = a.L;
  if (pos < kHdr) return a.hdr[pos];
  if (pos < L.c_end) {
    const int64_t o = pos - kHdr;
    const uint32_t c = a.counts[img * L.nB + (o >> 1)];
    return (o & 1) ? (c >> 8) : (c & 0xffu);
  }
  if (pos < L.p_end) {
    const int64_t o = pos - L.c_end;
    return (__float_as_uint(a.payload[img * L.K + (o >> 2)]) >> (8 * (o & 3))) & 0xffu;
  }
  if (pos < L.sc_end) return ((uint32_t)L.S >> (8 * (pos - L.p_end))) & 0xffu;
  const int64_t o = pos - L.sc_end;
  return (__float_as_uint(a.side[img * L.S + (o >> 2)]) >> (8 * (o & 3))) & 0xffu;
}

// 4 bytes at byte offset `o` of a float array row (whole words in range)
__device__ __forceinline__ uint32_t f32_bytes(const float* row, int64_t o) {
  const int sh = (int)(o & 3) * 8;
  const uint32_t lo = __float_as_uint(__ldg(row + (o >> 2)));
  if (!sh) return lo;
  return __funnelshift_r(lo, __float_as_uint(__ldg(row + (o >> 2) + 1)), sh);
}

// grid: x strides over the words of one container, y = container (image) index
__global__ void container_pack_kernel(ContainerArgs a, int64_t words_per, int img0) {
  const ContainerLayout& L = a.L;
  const int64_t img = img0 + blockIdx.y;
  uint8_t* base = a.out + img * a.stride;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words_per; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = 4 * w;
    if (pos + 4 > L.total) {  // trailing partial word
      for (int64_t q = pos; q < L.total; ++q) base[q] = (uint8_t)pack_byte(a, img, q);
      continue;
    }
    uint32_t v;
    if (pos >= L.c_end && pos + 4 <= L.p_end) {
      v = f32_bytes(a.payload + img * L.K, pos - L.c_end);
    } else if (pos >= L.sc_end) {
      v = f32_bytes(a.side + img * L.S, pos - L.sc_end);
    } else {  // header / counts / segment boundaries
      v = pack_byte(a, img, pos) | (pack_byte(a, img, pos + 1) << 8) | (pack_byte(a, img, pos + 2) << 16) |
          (pack_byte(a, img, pos + 3) << 24);
    }
    *reinterpret_cast<uint32_t*>(base + pos) = v;
  }
}

// little-endian u32 at byte offset pos of a container (aligned loads inside the container)
__device__ __forceinline__ uint32_t in_u32(const uint8_t* base, int64_t pos, int64_t total) {
  const int64_t w = pos >> 2;
  const int sh = (int)(pos & 3) * 8;
  const int64_t full_words = total >> 2;
  auto word = [&](int64_t k) -> uint32_t {
    if (k < full_words) return __ldg(reinterpret_cast<const uint32_t*>(base) + k);
    uint32_t r = 0;
    for (int b = 0; b < 4 && 4 * k + b < total; ++b) r |= (uint32_t)base[4 * k + b] << (8 * b);
    return r;
  };
  const uint32_t lo = word(w);
  return sh ? __funnelshift_r(lo, word(w + 1), sh) : lo;
}

__global__ void container_unpack_kernel(ContainerArgs a, int img0) {
  const ContainerLayout& L = a.L;
  const int64_t per = L.nB + L.K + L.S;
  const int64_t img = img0 + blockIdx.y;
  const uint8_t* base = a.in + img * a.stride;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < per; j += (int64_t)gridDim.x * blockDim.x) {
    if (j < L.nB) {
      a.counts_out[img * L.nB + j] = (uint16_t)(in_u32(base, kHdr + 2 * j, L.total) & 0xffffu);
    } else if (j < L.nB + L.K) {
      const int64_t k = j - L.nB;
      a.payload_out[img * L.K + k] = __uint_as_float(in_u32(base, L.c_end + 4 * k, L.total));
    } else {
      const int64_t k = j - L.nB - L.K;
      a.side_out[img * L.S + k] = __uint_as_float(in_u32(base, L.sc_end + 4 * k, L.total));
    }
  }
}

// One CTA per container: the reference reader's checks (container.cpp:104-147).
__global__ void container_validate_kernel(ContainerArgs a) {
  const int img = blockIdx.x;
  const uint8_t* base = a.in + (int64_t)img * a.stride;
  const ContainerLayout& L = a.L;
  __shared__ long long s_sum;
  __shared__ int s_bad;
  if (threadIdx.x == 0) {
    s_sum = 0;
    s_bad = 0;
  }
  __syncthreads();
  long long sum = 0;
  bool bad = false;
  const uint32_t area = (uint32_t)a.block * (uint32_t)a.block;
  for (int64_t i = threadIdx.x; i < L.nB; i += blockDim.x) {
    const uint32_t c = in_u32(base, kHdr + 2 * i, L.total) & 0xffffu;
    bad |= c > area;  // "per-block count exceeds B^2"
    sum += c;
  }
  atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum), (unsigned long long)sum);
  if (bad) atomicOr(&s_bad, 1);
  __syncthreads();
  if (threadIdx.x != 0) return;
  int st = ABCS_OK;
  for (int b = 0; b < 4; ++b)
    if (base[b] != a.hdr[b]) st = ABCS_ERR_FORMAT;  // magic
  const uint32_t ver = in_u32(base, 4, L.total) & 0xffffu;
  if (ver != 1) st = ABCS_ERR_FORMAT;
  // H, W, B, and n_B must describe this batch's layout
  for (int b = 6; b < 16; ++b)
    if (base[b] != a.hdr[b]) st = ABCS_ERR_FORMAT;
  const uint32_t algo = base[16];
  const uint32_t num = in_u32(base, 17, L.total), den = in_u32(base, 21, L.total);
  if (algo > 2 || num == 0 || den == 0 || num > den) st = ABCS_ERR_FORMAT;
  for (int b = 33; b < 37; ++b)
    if (base[b] != a.hdr[b]) st = ABCS_ERR_FORMAT;
  if (s_bad || s_sum != L.K) st = ABCS_ERR_FORMAT;
  if (in_u32(base, L.p_end, L.total) != (uint32_t)L.S) st = ABCS_ERR_FORMAT;
  abcs_container_info inf;
  inf.algorithm = (int32_t)algo;
  inf.cr_num = num;
  inf.cr_den = den;
  inf.status = st;
  const uint64_t tb = (uint64_t)in_u32(base, 25, L.total) | ((uint64_t)in_u32(base, 29, L.total) << 32);
  inf.threshold = __longlong_as_double((long long)tb);
  a.info[img] = inf;
}

}  // namespace abcs_b200

using namespace abcs_b200;

extern "C" {

int64_t abcs_container_size(const abcs_sense_plan* plan) { return plan ? layout_of(*plan).total : -1; }

int abcs_container_pack_batch(abcs_ctx* c, const abcs_sense_plan* plan, const uint16_t* d_counts,
                              const float* d_payload, const float* d_side, int32_t n, uint8_t* d_out,
                              int64_t out_stride, void* stream) {
  if (!c) return set_error(ABCS_ERR_INVALID_ARGUMENT, "null context");
  if (!plan || n < 0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (plan->block < 2 || (int64_t)plan->block * plan->block > 65535)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "container: block size must fit u16 counts");
  const ContainerLayout L = layout_of(*plan);
  if (n == 0) return ABCS_OK;
  if (!d_counts || !d_out || (L.K && !d_payload) || (L.S && !d_side) || out_stride < L.total || out_stride % 4 ||
      (uintptr_t)d_out % 4)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "container: bad buffers (output rows must be 4-byte aligned)");
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  ContainerArgs a{};
  header_bytes(*plan, a.hdr);
  a.L = L;
  a.counts = d_counts;
  a.payload = d_payload;
  a.side = d_side;
  a.out = d_out;
  a.stride = out_stride;
  a.n = n;
  const int64_t words = (L.total + 3) / 4;
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((words + 255) / 256,
                                                                         ((int64_t)ctx->sm_count * 16 + n - 1) / n));
  const int kt = ktimer_begin(ctx, s, "container_pack");
  for (int done = 0; done < n; done += 65535) {
    container_pack_kernel<<<dim3(gx, (unsigned)std::min(n - done, 65535)), 256, 0, s>>>(a, words, done);
    ctx->launches++;
  }
  ktimer_end(ctx, s, kt);
  return cuda_status(cudaGetLastError(), "container pack launch");
}

int abcs_container_unpack_batch(abcs_ctx* c, const abcs_sense_plan* plan, const uint8_t* d_in, int64_t in_stride,
                                int32_t n, uint16_t* d_counts, float* d_payload, float* d_side,
                                abcs_container_info* d_info, void* stream) {
  if (!c) return set_error(ABCS_ERR_INVALID_ARGUMENT, "null context");
  if (!plan || n < 0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  const ContainerLayout L = layout_of(*plan);
  if (n == 0) return ABCS_OK;
  if (!d_in || !d_counts || !d_info || (L.K && !d_payload) || (L.S && !d_side) || in_stride < L.total ||
      in_stride % 4 || (uintptr_t)d_in % 4)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "container: bad buffers (input rows must be 4-byte aligned)");
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  ContainerArgs a{};
  header_bytes(*plan, a.hdr);
  a.L = L;
  a.in = d_in;
  a.stride = in_stride;
  a.counts_out = d_counts;
  a.payload_out = d_payload;
  a.side_out = d_side;
  a.info = d_info;
  a.block = plan->block;
  a.n = n;
  int kt = ktimer_begin(ctx, s, "container_validate");
  container_validate_kernel<<<(unsigned)n, 256, 0, s>>>(a);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  const int64_t per = L.nB + L.K + L.S;
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((per + 255) / 256,
                                                                         ((int64_t)ctx->sm_count * 16 + n - 1) / n));
  kt = ktimer_begin(ctx, s, "container_unpack");
  for (int done = 0; done < n; done += 65535) {
    container_unpack_kernel<<<dim3(gx, (unsigned)std::min(n - done, 65535)), 256, 0, s>>>(a, done);
    ctx->launches++;
  }
  ktimer_end(ctx, s, kt);
  return cuda_status(cudaGetLastError(), "container unpack launch");
}

int abcs_container_parse(const uint8_t* h_bytes, int64_t size, abcs_sense_plan* plan) {
  // Host-side layout of one container (the reader's header checks, container.cpp:104-141):
  // fills the plan fields a batch unpack needs. Counts are summed to size the payload.
  if (!h_bytes || !plan || size < 0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  auto need = [&](int64_t n) { return size >= n; };
  if (!need(kHdr)) return set_error(ABCS_ERR_FORMAT, "container truncated");
  if (std::memcmp(h_bytes, "ABCS", 4) != 0) return set_error(ABCS_ERR_FORMAT, "not an ABCS container");
  auto rd = [&](int64_t off, void* dst, size_t n) { std::memcpy(dst, h_bytes + off, n); };
  uint16_t ver, block;
  uint32_t H, W, num, den, nb;
  uint8_t algo;
  double thr;
  rd(4, &ver, 2);
  if (ver != 1) return set_error(ABCS_ERR_FORMAT, "unsupported container version " + std::to_string(ver));
  rd(6, &H, 4);
  rd(10, &W, 4);
  rd(14, &block, 2);
  rd(16, &algo, 1);
  rd(17, &num, 4);
  rd(21, &den, 4);
  rd(25, &thr, 8);
  if (algo > 2) return set_error(ABCS_ERR_FORMAT, "container: unknown algorithm id");
  if ((int32_t)H <= 0 || (int32_t)W <= 0 || H > (1u << 20) || W > (1u << 20) || block < 2 || block > H ||
      block > W || num == 0 || den == 0 || num > den)
    return set_error(ABCS_ERR_FORMAT, "container: invalid header");
  rd(33, &nb, 4);
  const int32_t rows = (int32_t)(H / block), cols = (int32_t)(W / block);
  if ((int64_t)nb != (int64_t)rows * cols) return set_error(ABCS_ERR_FORMAT, "container: block count does not match dimensions");
  if (!need(kHdr + 2 * (int64_t)nb)) return set_error(ABCS_ERR_FORMAT, "container truncated");
  int64_t K = 0;
  for (uint32_t i = 0; i < nb; ++i) {
    uint16_t cnt;
    rd(kHdr + 2 * (int64_t)i, &cnt, 2);
    if (cnt > (uint32_t)block * block) return set_error(ABCS_ERR_FORMAT, "container: per-block count exceeds B^2");
    K += cnt;
  }
  const int64_t sc = kHdr + 2 * (int64_t)nb + 4 * K;
  if (!need(sc + 4)) return set_error(ABCS_ERR_FORMAT, "container truncated");
  uint32_t S;
  rd(sc, &S, 4);
  if ((int64_t)S * 4 > size) return set_error(ABCS_ERR_FORMAT, "container: side data count exceeds file size");
  if (!need(sc + 4 + 4 * (int64_t)S)) return set_error(ABCS_ERR_FORMAT, "container truncated");
  if (size != sc + 4 + 4 * (int64_t)S) return set_error(ABCS_ERR_FORMAT, "container: trailing bytes");
  std::memset(plan, 0, sizeof(*plan));
  plan->height = (int32_t)H;
  plan->width = (int32_t)W;
  plan->block = block;
  plan->rows = rows;
  plan->cols = cols;
  plan->n_blocks = (int32_t)nb;
  plan->algorithm = plan->algorithm_used = algo;
  plan->cr_num = num;
  plan->cr_den = den;
  plan->threshold = thr;
  plan->coeffs_per_image = K;
  plan->side_per_image = S;
  return ABCS_OK;
}

}  // extern "C"
