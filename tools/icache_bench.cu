// Cost of executing cold straight-line code on B200: one warp runs N unrolled
// independent FFMAs (16 B each); clock64 around the block. First launch vs
// repeated launches vs a launch after evicting L2 with a 512 MB memset.
#include <cstdio>
#include <cuda_runtime.h>
template <int N>
__global__ void straight(float* out, long long* cyc) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N / 8; ++i) {
    asm volatile("fma.rn.f32 %0, %0, 1.0001, 0.5;" : "+f"(a0)); asm volatile("fma.rn.f32 %0, %0, 1.0001, 0.5;" : "+f"(a1));
    asm volatile("fma.rn.f32 %0, %0, 1.0001, 0.5;" : "+f"(a2)); asm volatile("fma.rn.f32 %0, %0, 1.0001, 0.5;" : "+f"(a3));
    asm volatile("fma.rn.f32 %0, %0, 1.0001, 0.5;" : "+f"(a4)); asm volatile("fma.rn.f32 %0, %0, 1.0001, 0.5;" : "+f"(a5));
    asm volatile("fma.rn.f32 %0, %0, 1.0001, 0.5;" : "+f"(a6)); asm volatile("fma.rn.f32 %0, %0, 1.0001, 0.5;" : "+f"(a7));
  }
  long long t1 = clock64();
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int N>
void run(float* out, long long* dcyc, char* big) {
  long long c;
  straight<N><<<1, 32>>>(out, dcyc); cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost);
  long long first = c;
  straight<N><<<1, 32>>>(out, dcyc); cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost);
  long long second = c;
  cudaMemset(big, 1, size_t(512) << 20);
  straight<N><<<1, 32>>>(out, dcyc); cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost);
  long long evicted = c;
  straight<N><<<148, 32>>>(out, dcyc); cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost);
  long long grid = c;
  printf("N=%6d instr (%4d KB): first %8lld cyc (%.2f/instr)  second %8lld (%.2f)  after-L2-evict %8lld (%.2f) grid148 %8lld\n",
         N, N * 16 / 1024, first, (double)first / N, second, (double)second / N, evicted, (double)evicted / N, grid);
}
int main() {
  float* out; long long* cyc; char* big;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8); cudaMalloc(&big, size_t(512) << 20);
  run<512>(out, cyc, big); run<2048>(out, cyc, big); run<4096>(out, cyc, big); run<8192>(out, cyc, big); run<16384>(out, cyc, big);
  return 0;
}
