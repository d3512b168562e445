// Device side of the seeded synthetic generator (synth_gen.h): scene
// parameters are built on the host (same code) and uploaded; each thread
// produces one pixel pair (one Philox draw -> two Box-Muller normals).
#include <vector>

#include "internal.h"
#include "synth_gen.h"

namespace abcs_b200 {

__global__ void __launch_bounds__(256)
synth_kernel(sg_spec sp, const sg_scene* __restrict__ scenes, int64_t first, int n, uint8_t* __restrict__ out,
             int64_t stride) {
  const uint64_t npx = (uint64_t)sp.height * sp.width;
  const uint64_t pairs = (npx + 1) / 2;
  const int img = blockIdx.y;
  const sg_scene* sc = scenes + img;
  uint8_t* o = out + (int64_t)img * stride;
  for (uint64_t pr = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; pr < pairs;
       pr += (uint64_t)gridDim.x * blockDim.x) {
    uint8_t a, b;
    sg_pixel_pair(&sp, sc, (uint32_t)(first + img), pr, &a, &b);
    o[2 * pr] = a;
    if (2 * pr + 1 < npx) o[2 * pr + 1] = b;
  }
}

int launch_synth(Ctx* ctx, const abcs_synth_spec& spec, int64_t first, int32_t n, uint8_t* out, int64_t stride,
                 void* scratch, cudaStream_t s) {
  sg_spec sp;
  static_assert(sizeof(sg_spec) == sizeof(abcs_synth_spec), "spec layout");
  memcpy(&sp, &spec, sizeof(sp));
  std::vector<sg_scene> scenes(n);
  for (int i = 0; i < n; ++i) sg_make_scene(&sp, (uint32_t)(first + i), &scenes[i]);
  sg_scene* d = static_cast<sg_scene*>(scratch);
  cudaError_t e = cudaMemcpyAsync(d, scenes.data(), sizeof(sg_scene) * n, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_status(e, "synth upload");
  const uint64_t pairs = ((uint64_t)spec.height * spec.width + 1) / 2;
  unsigned gx = (unsigned)std::min<uint64_t>((pairs + 255) / 256, 4096);
  int64_t done = 0;
  while (done < n) {  // gridDim.y <= 65535
    const int cnt = (int)std::min<int64_t>(n - done, 65535);
    synth_kernel<<<dim3(gx, cnt), 256, 0, s>>>(sp, d + done, first + done, cnt, out + done * stride, stride);
    ctx->launches++;
    done += cnt;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "synth launch");
  // the host vector is released on return: make the upload complete first
  return cuda_status(cudaStreamSynchronize(s), "synth sync");
}

}  // namespace abcs_b200
