/* TEST INFRASTRUCTURE ONLY — the BASELINE input generator for the CPU arms.
 *
 * The seeded scene generator is a fixed input
 * definition shared by every arm, not part of the reference (whose synth.cpp
 * scenes differ). Its single source is the header-only csrc/synth_gen.h; this
 * file compiles that header's host path into the oracle library so bench.py's
 * reference arm and the CPU baselines generate their inputs without loading the
 * product library (libabcs_b200.so). Bytes are pinned by tests/golden/synth_hashes.txt.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

#include "../paper_2001_09632_b200/csrc/synth_gen.h"

typedef struct {
  const sg_spec* sp;
  int64_t first;
  int32_t lo, hi;
  uint8_t* out;
} synth_job;

static void* synth_worker(void* arg) {
  synth_job* j = (synth_job*)arg;
  const uint64_t npx = (uint64_t)j->sp->height * (uint64_t)j->sp->width;
  sg_scene* sc = (sg_scene*)malloc(sizeof(sg_scene));
  if (!sc) return (void*)1;
  for (int32_t i = j->lo; i < j->hi; ++i) {
    const uint32_t img = (uint32_t)(j->first + i);
    sg_make_scene(j->sp, img, sc);
    uint8_t* o = j->out + (uint64_t)i * npx;
    for (uint64_t pr = 0; pr < (npx + 1) / 2; ++pr) {
      uint8_t a, b;
      sg_pixel_pair(j->sp, sc, img, pr, &a, &b);
      o[2 * pr] = a;
      if (2 * pr + 1 < npx) o[2 * pr + 1] = b;
    }
  }
  free(sc);
  return NULL;
}

/* n images [first, first + n) of the spec into out (n x H x W u8), on `threads` host threads. */
int o_synth_images(int32_t height, int32_t width, int32_t n_ellipses, double sigma, uint64_t seed, int32_t video,
                   int64_t first, int32_t n, uint8_t* out, int32_t threads) {
  if (height < 1 || width < 1 || n_ellipses < 0 || n_ellipses > SG_MAX_ELLIPSES || n < 0 || !out) return 1;
  sg_spec sp = {height, width, n_ellipses, video ? 1 : 0, 8, 0, sigma, seed};
  if (threads < 1) threads = 1;
  if (threads > n) threads = n > 0 ? n : 1;
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  synth_job* jobs = (synth_job*)calloc((size_t)threads, sizeof(synth_job));
  if (!tid || !jobs) return 5;
  int rc = 0;
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (synth_job){&sp, first, (int32_t)((int64_t)n * t / threads), (int32_t)((int64_t)n * (t + 1) / threads),
                          out};
    if (pthread_create(&tid[t], NULL, synth_worker, &jobs[t]) != 0) rc = 5;
  }
  for (int t = 0; t < threads; ++t) {
    void* r = NULL;
    pthread_join(tid[t], &r);
    if (r) rc = 5;
  }
  free(tid);
  free(jobs);
  return rc;
}
