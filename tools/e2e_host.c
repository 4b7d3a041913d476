/* End-to-end decode through the C ABI from host buffers, timed from C (no
 * Python in the loop): the serving-loop shape of bench.py's e2e key. Each
 * step copies that step's tokens (host memory) into a pinned staging buffer,
 * calls oea_moe_decode_host (zero-copy fused decode; returns when the output
 * is in the pinned output buffer), and touches the output.
 *
 *   e2e_host D H N B k0 steps warmup [layers]
 * prints one JSON object: mean / median / p90 us per call and the breakdown
 * of a step (host copy in, library call).
 */
#define _POSIX_C_SOURCE 200809L
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "oea_cuda.h"

static double now_us(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
}
static int cmp(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : x > y;
}
#define CK(x)                                                              \
  do {                                                                     \
    int rc_ = (x);                                                         \
    if (rc_) {                                                             \
      fprintf(stderr, "%s failed: %d %s\n", #x, rc_, oea_last_error(ctx)); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 8) {
    fprintf(stderr, "usage: e2e_host D H N B k0 steps warmup [layers]\n");
    return 2;
  }
  const int D = atoi(argv[1]), H = atoi(argv[2]), N = atoi(argv[3]), B = atoi(argv[4]);
  const int k0 = atoi(argv[5]), steps = atoi(argv[6]), warm = atoi(argv[7]);
  const int R = argc > 8 ? atoi(argv[8]) : 4;
  /* mode 0: oea_moe_decode_host (zero copy) after a host copy of the step's
   * tokens from pageable memory into one pinned staging buffer; 1: H2D
   * memcpy + device decode + D2H memcpy + sync; 2: H2D memcpy + device decode
   * writing the mapped out + sync (experiments); 3: every step's tokens
   * already in pinned host memory (one slice per step), oea_moe_decode_host
   * reads that step's slice zero-copy (no host copy) */
  const int mode = argc > 9 ? atoi(argv[9]) : 0;
  oea_ctx_t ctx = NULL;
  if (oea_ctx_create(0, &ctx)) {
    fprintf(stderr, "ctx: %s\n", oea_last_error(NULL));
    return 1;
  }
  oea_layer_t L[16];
  for (int r = 0; r < R && r < 16; ++r) {
    CK(oea_layer_create(ctx, D, H, N, OEA_DTYPE_BF16, &L[r]));
    CK(oea_layer_init_random(L[r], 1 + r));
  }
  oea_routing_cfg cfg = {OEA_MODE_SIMPLIFIED, 8, k0, 1.0, 8, 0, OEA_CAP_EXACT};
  const int total = steps + warm;
  const size_t xb = (size_t)B * D * 2, ob = (size_t)B * D * 4;
  uint16_t* src = (uint16_t*)malloc(xb * total); /* the steps' tokens, pageable host memory */
  uint32_t s = 777u;
  for (size_t i = 0; i < (size_t)B * D * total; ++i) {
    s = s * 1664525u + 1013904223u;
    const float f = ((float)(s >> 8) / 16777216.0f - 0.5f) * 3.0f;
    uint32_t u;
    memcpy(&u, &f, 4);
    src[i] = (uint16_t)(u >> 16);
  }
  void *xs = NULL, *out = NULL, *xall = NULL;
  if (cudaHostAlloc(&xs, xb, cudaHostAllocMapped) || cudaHostAlloc(&out, ob, cudaHostAllocMapped)) {
    fprintf(stderr, "cudaHostAlloc failed\n");
    return 1;
  }
  if (mode == 3) {
    if (cudaHostAlloc(&xall, xb * total, cudaHostAllocMapped)) {
      fprintf(stderr, "cudaHostAlloc failed\n");
      return 1;
    }
    memcpy(xall, src, xb * total);
  }
  void *xdev = NULL, *odev = NULL, *st = NULL;
  cudaMalloc(&xdev, xb);
  cudaMalloc(&odev, ob);
  CK(oea_ctx_stream(ctx, &st));
  double* t_call = (double*)malloc(sizeof(double) * steps);
  double* t_step = (double*)malloc(sizeof(double) * steps);
  double t_copy = 0.0, sink = 0.0;
  for (int i = 0; i < total; ++i) {
    const double t0 = now_us();
    if (mode != 3) memcpy(xs, src + (size_t)i * B * D, xb);
    const double t1 = now_us();
    if (mode == 0) {
      CK(oea_moe_decode_host(ctx, L[i % R], xs, NULL, B, &cfg, out));
    } else if (mode == 3) {
      CK(oea_moe_decode_host(ctx, L[i % R], (const char*)xall + (size_t)i * xb, NULL, B, &cfg, out));
    } else {
      cudaMemcpyAsync(xdev, xs, xb, cudaMemcpyHostToDevice, (cudaStream_t)st);
      CK(oea_moe_decode(ctx, L[i % R], xdev, NULL, B, &cfg, mode == 1 ? odev : out, st));
      if (mode == 1) cudaMemcpyAsync(out, odev, ob, cudaMemcpyDeviceToHost, (cudaStream_t)st);
      cudaStreamSynchronize((cudaStream_t)st);
    }
    const double t2 = now_us();
    sink += ((const float*)out)[i % (B * D)];
    if (i >= warm) {
      t_call[i - warm] = t2 - t1;
      t_step[i - warm] = t2 - t0;
      t_copy += t1 - t0;
    }
  }
  double mean = 0.0, mean_call = 0.0;
  for (int i = 0; i < steps; ++i) {
    mean += t_step[i];
    mean_call += t_call[i];
  }
  mean /= steps;
  mean_call /= steps;
  qsort(t_step, steps, sizeof(double), cmp);
  qsort(t_call, steps, sizeof(double), cmp);
  printf("{\"us_per_step_mean\": %.3f, \"us_per_step_median\": %.3f, \"us_per_step_p90\": %.3f, "
         "\"us_call_mean\": %.3f, \"us_call_median\": %.3f, \"us_host_copy_in_mean\": %.3f, "
         "\"steps\": %d, \"warmup\": %d, \"h2d_bytes_per_step\": %zu, \"d2h_bytes_per_step\": %zu, "
         "\"checksum\": %.6g}\n",
         mean, t_step[steps / 2], t_step[(steps * 9) / 10], mean_call, t_call[steps / 2],
         t_copy / steps, steps, warm, xb, ob, sink);
  if (getenv("OEA_FFN_TRACE")) {  /* per-launch spans of the last 16 launches */
    const int LEG = 8192, PER = 16384, NL = 16;
    uint64_t* tr = (uint64_t*)malloc(sizeof(uint64_t) * (LEG + NL * PER));
    CK(oea_debug_ffn_trace(ctx, tr, LEG + NL * PER));
    for (int l = 0; l < NL; ++l) {
      const uint64_t* t = tr + LEG + (size_t)l * PER;
      uint64_t t0 = ~0ull, staged = 0, done = 0, pub = 0;
      for (int c = 0; c < 148; ++c) {
        if (t[c * 16] && t[c * 16] < t0) t0 = t[c * 16];
        if (t[c * 16 + 8] > staged) staged = t[c * 16 + 8];
        if (t[c * 16 + 5] > pub) pub = t[c * 16 + 5];
        if (t[c * 16 + 15] > done) done = t[c * 16 + 15];
      }
      if (t0 != ~0ull && done)
        fprintf(stderr, "launch %2d: x staged %.2f logits %.2f combine done %.2f us (T=%d)\n", l,
                (staged - t0) / 1e3, (pub - t0) / 1e3, (done - t0) / 1e3, (int)t[2400]);
    }
    free(tr);
  }
  for (int r = 0; r < R && r < 16; ++r) oea_layer_destroy(L[r]);
  cudaFreeHost(xs);
  cudaFreeHost(out);
  if (xall) cudaFreeHost(xall);
  oea_ctx_destroy(ctx);
  return 0;
}
