// Latency of a dependent chain of warp reductions on B200: redux.sync.max
// (__reduce_max_sync) vs a 5-step shfl_xor max, and the cost of
// shared-memory / DSMEM-free building blocks used by the router's selection.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned* out, long long* cyc, int iters) {
  unsigned v = threadIdx.x * 2654435761u;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __reduce_max_sync(0xffffffffu, v ^ i) + threadIdx.x;
  long long t1 = clock64();
  unsigned w = threadIdx.x * 2654435761u;
  for (int i = 0; i < iters; ++i) {
    unsigned x = w ^ i;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
    w = x + threadIdx.x;
  }
  long long t2 = clock64();
  unsigned b = 0;
  for (int i = 0; i < iters; ++i) b += __popc(__ballot_sync(0xffffffffu, ((v + i) & 1) != 0));
  long long t3 = clock64();
  out[threadIdx.x] = v + w + b;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  unsigned* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 32>>>(o, c, 1000);
    long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("per op cycles: redux.sync.max %.1f   shfl-tree max (5 steps) %.1f   ballot+popc %.1f\n",
           h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0);
  }
  return 0;
}
