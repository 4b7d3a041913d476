// Resolution of %globaltimer vs clock64 on this GPU (what the in-kernel
// timeline stamps of tools/trace_ffn.py can resolve).
#include <cstdio>
__global__ void k(unsigned long long* out) {
  unsigned long long prev, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  int n = 0;
  long long c0 = clock64();
  while (n < 16) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { out[n++] = t - prev; prev = t; out[16 + n - 1] = clock64() - c0; }
  }
}
int main() {
  unsigned long long* d; unsigned long long h[32];
  cudaMalloc(&d, sizeof(h));
  k<<<1, 1>>>(d);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("globaltimer increments (ns):");
  for (int i = 0; i < 16; ++i) printf(" %llu", h[i]);
  printf("\nclock64 at each change:");
  for (int i = 0; i < 16; ++i) printf(" %llu", h[16 + i]);
  printf("\n");
}
