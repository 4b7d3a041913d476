// oea_device.cuh — device helpers: order-preserving keys, the warp bitonic
// sort that ranks experts, mbarrier / bulk-copy / mma PTX wrappers.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace oea_dev {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// Ranking keys. The reference orders experts by (score desc, index asc) with
// double `!=` / `>` comparisons (routing.cpp:196-199), so -0.0 == +0.0. We map
// a score to an unsigned key whose integer order equals the double order
// (after canonicalising -0.0), so one 64-bit compare + an index tie-break
// reproduces the comparator exactly. NaN is outside the contract
// (ScoreMatrix::validate rejects it, routing.cpp:67).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t order_key_f64(double v) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v == 0.0 ? 0.0 : v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ uint64_t order_key_f32(float v) {
  const uint32_t b = __float_as_uint(v == 0.0f ? 0.0f : v);
  const uint32_t k = (b >> 31) ? ~b : (b | 0x80000000u);
  return static_cast<uint64_t>(k) << 32;
}

// a ranks before b
__device__ __forceinline__ bool ranks_before(uint64_t ka, uint32_t ia, uint64_t kb,
                                             uint32_t ib) {
  return ka > kb || (ka == kb && ia < ib);
}

// Warp-wide bitonic sort of 32*E (key, index) pairs into rank order.
// Element position p = j*32 + lane; after the call position p holds rank p.
// Padding elements must carry key 0 (below every real key) and distinct
// indices >= N.
template <int E>
__device__ __forceinline__ void warp_rank_sort(uint64_t (&k)[E], uint32_t (&id)[E]) {
  const int lane = threadIdx.x & 31;
  constexpr int NP = 32 * E;
#pragma unroll
  for (int size = 2; size <= NP; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int js = stride >> 5;
#pragma unroll
        for (int j = 0; j < E; ++j) {
          if ((j & js) == 0) {
            const int jj = j | js;
            const bool asc = ((j * 32 + lane) & size) == 0;
            const bool sw = asc ? ranks_before(k[jj], id[jj], k[j], id[j])
                                : ranks_before(k[j], id[j], k[jj], id[jj]);
            if (sw) {
              const uint64_t tk = k[j];
              k[j] = k[jj];
              k[jj] = tk;
              const uint32_t ti = id[j];
              id[j] = id[jj];
              id[jj] = ti;
            }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const uint64_t ok = __shfl_xor_sync(kFull, k[j], stride);
          const uint32_t oi = __shfl_xor_sync(kFull, id[j], stride);
          const bool lower = (lane & stride) == 0;
          const bool asc = ((j * 32 + lane) & size) == 0;
          const bool other_first = ranks_before(ok, oi, k[j], id[j]);
          if ((lower == asc) ? other_first : !other_first) {
            k[j] = ok;
            id[j] = oi;
          }
        }
      }
    }
  }
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------------------
// mbarrier + TMA bulk copy (cp.async.bulk, 1-D) wrappers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// Global -> shared bulk copy completing on `bar` (bytes % 16 == 0, 16B aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Bulk copy without a cache hint (data other CTAs re-read: default policy).
__device__ __forceinline__ void bulk_g2s_nohint(void* dst, const void* src, uint32_t bytes,
                                                uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Orders this thread's prior generic-proxy view of global memory (e.g. data
// acquired from other CTAs) before its subsequent async-proxy (TMA) reads.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// 16-byte cp.async global -> shared (src_bytes 0 zero-fills the destination).
// L2 prefetch of a contiguous block (no shared-memory destination).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

// Programmatic dependent launch (griddepcontrol).
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Release increment of a cross-CTA counter (cumulative release at gpu scope:
// orders every write this thread has observed, e.g. the warp's stores after a
// __syncwarp, before the increment; no full fence / L1 invalidation).
__device__ __forceinline__ void red_release_gpu_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_gpu_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Epoch-tagged 64-bit exchange words {tag:32 | payload:32}: a reader polls
// the word itself until its tag is the current launch's, so no separate
// arrival counter / grid barrier round trip is needed.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long tagged(uint32_t tag, uint32_t payload) {
  return (static_cast<unsigned long long>(tag) << 32) | payload;
}

// Acquire / relaxed loads for cross-CTA flags and data written in-kernel.
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---------------------------------------------------------------------------
// Tensor-core tile: D(16x8 f32) += A(16x16 bf16, row) * B(16x8 bf16, col).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint4& a, uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// Fragment position of A(r, c) inside a 512-byte tile: lane and element 0..7
// (mma.m16n8k16 A-operand register layout: a0/a1 rows g / g+8, cols 2q..;
// a2/a3 the same rows, cols 2q+8..).
__host__ __device__ __forceinline__ int frag_offset(int r, int c) {
  const int g = r & 7, hi_r = r >> 3;   // row group, upper half
  const int hi_c = c >> 3, cc = c & 7;  // upper k half
  const int q = cc >> 1, lo = cc & 1;
  const int lane = g * 4 + q;
  const int elem = (hi_c * 2 + hi_r) * 2 + lo;
  return lane * 8 + elem;  // in bf16 elements
}

__device__ __forceinline__ float silu_f(float z) { return z / (1.0f + __expf(-z)); }

}  // namespace oea_dev
