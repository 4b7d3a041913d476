// Streaming microbenchmark on B200: how fast can a persistent grid pull a
// large read-only buffer through shared memory with TMA bulk copies
// (cp.async.bulk + mbarrier ring) vs plain 128-bit loads? Used to size the
// FFN weight-stream pipeline. Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench tools/stream_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_nohint(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Each CTA streams its contiguous share; a stage = `copies` bulk copies of
// `chunk` bytes; `stages` deep ring; consumers = 8 warps that just release.
__global__ void k_tma(const uint8_t* src, size_t total, int chunk, int copies, int stages, int hint,
                      int stride_mode, int hold) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int stage_bytes = chunk * copies;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t per = (total / gridDim.x) & ~static_cast<size_t>((1 << 20) - 1);
  const uint8_t* base = src + per * blockIdx.x;
  const size_t nstage = per / stage_bytes;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (warp == 8) {
    if (lane == 0) {
      int st = 0; uint32_t ph = 0;
      for (size_t i = 0; i < nstage; ++i) {
        mbar_wait(&empty[st], ph ^ 1u);
        mbar_expect(&full[st], stage_bytes);
        for (int c = 0; c < copies; ++c) {
          // stride_mode 0: stage is contiguous; 1: copies come from `copies`
          // streams 64 KiB apart (the FFN's 8-units-per-round pattern)
          const uint8_t* p = stride_mode == 0 ? base + i * stage_bytes + c * chunk
                                              : base + (i / 16) * (16 * stage_bytes) + c * (16 * chunk) + (i % 16) * chunk;
          if (hint) bulk(smem + st * stage_bytes + c * chunk, p, chunk, &full[st], pol);
          else bulk_nohint(smem + st * stage_bytes + c * chunk, p, chunk, &full[st]);
        }
        if (++st == stages) { st = 0; ph ^= 1u; }
      }
    }
    return;
  }
  int st = 0; uint32_t ph = 0;
  for (size_t i = 0; i < nstage; ++i) {
    mbar_wait(&full[st], ph);
    if (hold) {  // emulate the consumer's per-stage math: hold the slot `hold` cycles
      const long long t0 = clock64();
      while (clock64() - t0 < hold) {}
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (++st == stages) { st = 0; ph ^= 1u; }
  }
}

__global__ void k_ldg(const uint4* src, size_t n16, unsigned long long* sink) {
  const size_t per = (n16 / gridDim.x) & ~static_cast<size_t>(4095);
  const uint4* p = src + per * blockIdx.x;
  uint32_t acc = 0;
  for (size_t i = threadIdx.x; i + 7 * blockDim.x < per; i += 8 * blockDim.x) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcs(p + i + j * blockDim.x);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  const size_t total = size_t(1) << 30;  // 1 GiB per pass
  uint8_t* buf[4];
  for (int i = 0; i < 4; ++i) { cudaMalloc(&buf[i], total); cudaMemset(buf[i], i, total); }
  unsigned long long* sink; cudaMalloc(&sink, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run_tma = [&](int chunk, int copies, int stages, int ctas_per_sm, int hint, int stride_mode, int hold = 0) {
    const int smem = chunk * copies * stages + 2 * stages * 8;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = sms * ctas_per_sm;
    for (int w = 0; w < 2; ++w) k_tma<<<grid, 288, smem>>>(buf[w], total, chunk, copies, stages, hint, stride_mode, hold);
    cudaEventRecord(e0);
    const int reps = 8;
    for (int r = 0; r < reps; ++r) k_tma<<<grid, 288, smem>>>(buf[r % 4], total, chunk, copies, stages, hint, stride_mode, hold);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("tma chunk=%6d copies=%d stages=%d (ring %3d KiB) ctas/sm=%d hint=%d mode=%d hold=%5d : %7.1f GB/s %s\n", chunk, copies,
           stages, smem >> 10, ctas_per_sm, hint, stride_mode, hold, reps * (double)((total / grid) & ~((size_t(1) << 20) - 1)) * grid / (ms * 1e6), err ? cudaGetErrorString(err) : "");
  };
  // the FFN's pattern: one 32 KiB copy per stage; ring depth x consumer hold
  for (int stages : {3, 4, 5, 6})
    for (int hold : {0, 500, 1000, 2000})
      run_tma(32768, 1, stages, 1, 1, 0, hold);
  run_tma(65536, 1, 3, 1, 1, 0, 0);
  run_tma(65536, 1, 3, 1, 1, 0, 1000);
  run_tma(16384, 1, 8, 1, 1, 0, 0);
  run_tma(16384, 1, 8, 1, 1, 0, 1000);
  if (getenv("LDG_TOO") == nullptr) return 0;
  for (int threads : {256, 512, 1024}) {
    for (int cps : {1, 2, 4}) {
      k_ldg<<<sms * cps, threads>>>(reinterpret_cast<uint4*>(buf[0]), total / 16, sink);
      cudaEventRecord(e0);
      for (int r = 0; r < 8; ++r) k_ldg<<<sms * cps, threads>>>(reinterpret_cast<uint4*>(buf[r % 4]), total / 16, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("ldg threads=%4d ctas/sm=%d : %7.1f GB/s\n", threads, cps, 8.0 * (double)(((total / 16) / (sms * cps)) & ~size_t(4095)) * 16 * sms * cps / (ms * 1e6));
    }
  }
  return 0;
}
