// umma_ffn.cu — the grouped SwiGLU expert FFN of large decode batches
// (64 < B <= 256) on the 5th-generation tensor cores: tcgen05.mma with the
// accumulators in tensor memory (TMEM), operands staged in shared memory by
// TMA bulk copies, one elected thread issuing the MMAs.
//
// Same computation as k_ffn_bf16<0> (moe_layer.hpp:92-158: per active expert
// e and its token group, h = silu(x Wg) * (x Wu), y = h Wd; then out[t] =
// sum_j w_j y_j in set order), fed by the same plan tables (k_compact: token
// groups of <= 64 rows per expert, row -> (token, slot)).
//
// Operand layout ("CM", the canonical K-major no-swizzle UMMA layout): a
// matrix [M rows][K] is cut into 128-wide K slices; inside a slice, 8-row
// groups of 2 KiB = [16 k-groups][8 rows][8 k] (one 8x8 core matrix = 128 B
// contiguous). UMMA descriptor: LBO (K-adjacent core matrices) = 128 B, SBO
// (M/N-adjacent 8-row groups) = 2 KiB; the K=16 step kk starts at +256 kk.
//   w1u (expert): [Hp/64 m-blocks][Dp/128 slices][16 row groups] 2 KiB blocks;
//                 m-block mb = W1 rows 128 mb .. (8 row blocks of 8 gate + 8
//                 up rows of h = 8 rb + i, as the fragment layout)
//   w2u (expert): [Dp/128 m-blocks][Hp/128 slices][16 row groups]
//   xg  (batch):  [Dp/128 slices][row groups] token rows in plan-row order
//   hg  (batch):  [Hp/128 slices][row groups] h in plan-row order
// so a pipeline stage (one 128-wide K slice of one unit) is ONE 32 KiB bulk
// copy of weights + ONE contiguous copy of the group's token rows (N x 256 B).
//
// Units: W1 (group, m-block of 64 h) with K = Dp, then W2 (group, m-block of
// 128 output columns) with K = Hp; claimed dynamically (all W1 before any
// W2). Per unit: M = 128, N = the group's rows rounded up to 16 (<= 64),
// accumulator D[128 lanes][N columns] fp32 in TMEM (double-buffered).
// Warp roles (6 warps): 0 producer (bulk copies), 1 MMA issuer (+ TMEM
// alloc), 2-5 epilogue (TMEM -> registers; W1: silu(g) * u -> bf16 hg, then a
// release of the group's K-slot count; W2: y[t][slot][d] fp32).
// W2 stage s reads h slice s only: it waits for that slice's two W1 m-blocks
// (8-bit slot fields of one 64-bit counter per group, as the dense path).
#include <algorithm>

#include "layout.cuh"

namespace oea_dev {

constexpr int kUmStages = 4;
constexpr int kUmABytes = 32 * 1024;          // 128 rows x 128 k bf16
constexpr int kUmBBytes = kTokGroup * 256;    // <= 64 token rows x 128 k bf16
constexpr int kUmStageBytes = kUmABytes + kUmBBytes;
constexpr int kUmUnitRing = 8;
constexpr int kUmWarps = 6;
constexpr int kUmThreads = kUmWarps * 32;
constexpr int kUmAccCols = 64;                // one accumulator: N <= 64 fp32 columns
constexpr int kUmTmemCols = 2 * kUmAccCols;   // double-buffered

struct UmmaParams {
  const uint8_t* w1u;  // CM, per expert w1u_stride bytes
  const uint8_t* w2u;
  size_t w1u_stride, w2u_stride;
  const uint8_t* xg;   // CM token rows [Dp/128][RG] x 2 KiB
  uint8_t* hg;         // CM h rows [Hp/128][RG] x 2 KiB
  int RG;              // row-group capacity of xg / hg
  int Dp, Hp, B, stride;
  const int32_t* row_tok;
  const int32_t* row_slot;
  const int32_t* group_a;
  const int32_t* group_row0;
  const int32_t* group_rows;
  const FfnHeader* hdr;
  unsigned long long* w1_slots;  // [max_groups] 8-bit slot fields (W1 m-blocks done)
  unsigned long long w1_full;    // the word of a group whose W1 is complete
  int slot_q;                    // h slices per slot field
  int* claims;                   // [0] W1 units, [1] W2 units, [2] exit count
  float* ybuf;                   // [B][stride][Dp]
};

struct UmUnit {
  int kind;   // 1 = W1, 2 = W2, 0 = end of work
  int g, mb;  // token group, m-block
  int n;      // MMA N (rows rounded up to 16)
  int nst;    // K stages
};

__device__ __forceinline__ uint64_t umma_smem_desc(uint32_t saddr) {
  // K-major, SWIZZLE_NONE: LBO 128 B (K), SBO 2048 B (M/N), version 1 (sm_100)
  return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(128 >> 4) << 16) |
         (static_cast<uint64_t>(2048 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint32_t umma_idesc(int n) {
  // D fp32 (bit 4), A bf16 (7), B bf16 (10), K-major A and B, N >> 3 at 17, M >> 4 at 24
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(128 >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` once every tcgen05 op this thread issued so far has completed
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// 16 consecutive fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__global__ void __launch_bounds__(kUmThreads, 1) k_ffn_umma(const UmmaParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kUmStages * kUmStageBytes);
  uint64_t* empty = full + kUmStages;
  uint64_t* tfull = empty + kUmStages;     // [2] accumulator ready (MMA commit)
  uint64_t* tempty = tfull + 2;            // [2] accumulator drained (4 epilogue warps)
  uint64_t* dfull = tempty + 2;            // [ring] unit descriptor written
  uint64_t* dempty = dfull + kUmUnitRing;  // [ring] read by the MMA thread + 4 epilogue warps
  UmUnit* units = reinterpret_cast<UmUnit*>(dempty + kUmUnitRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(units + kUmUnitRing);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kUmStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    for (int u = 0; u < kUmUnitRing; ++u) {
      mbar_init(&dfull[u], 1);
      mbar_init(&dempty[u], 5);
    }
    fence_mbar_init();
  }
  if (warp == 1) {  // TMEM: 2 accumulators of 64 fp32 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kUmTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // plan tables and x come from the preceding launches
  pdl_launch_dependents();  // (the combine waits for this grid's completion)

  const int G = P.hdr->n_groups;
  const int M1 = P.Hp >> 6, M2 = P.Dp >> 7;  // m-blocks per group (W1: 64 h; W2: 128 d)
  const int S1 = P.Dp >> 7, S2 = P.Hp >> 7;  // K stages
  const int U1 = G * M1, U2 = G * M2;

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      bool w1_left = true;
      for (int seq = 0;; ++seq) {
        UmUnit u{0, 0, 0, 0, 0};
        if (w1_left) {
          const int r = atomicAdd(&P.claims[0], 1);
          if (r < U1) u = UmUnit{1, r / M1, r % M1, 0, S1};
          else w1_left = false;
        }
        if (!w1_left) {
          const int r = atomicAdd(&P.claims[1], 1);
          if (r < U2) u = UmUnit{2, r / M2, r % M2, 0, S2};
        }
        int row0 = 0;
        const uint8_t* wbase = nullptr;
        if (u.kind) {
          row0 = P.group_row0[u.g];
          u.n = (P.group_rows[u.g] + 15) & ~15;
          const int e = P.group_a[u.g];
          wbase = u.kind == 1 ? P.w1u + e * P.w1u_stride + static_cast<size_t>(u.mb) * S1 * kUmABytes
                              : P.w2u + e * P.w2u_stride + static_cast<size_t>(u.mb) * S2 * kUmABytes;
        }
        const int ds = seq & (kUmUnitRing - 1);
        mbar_wait(&dempty[ds], ((seq / kUmUnitRing) & 1u) ^ 1u);
        units[ds] = u;
        mbar_arrive(&dfull[ds]);
        if (!u.kind) break;
        const uint32_t bbytes = static_cast<uint32_t>(u.n) * 256u;
        const uint8_t* bsrc = u.kind == 1 ? P.xg : P.hg;
        unsigned long long miss = ~0ull;  // W2: h slot fields not yet complete
        for (int s = 0; s < u.nst; ++s) {
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* st = ring + stage * kUmStageBytes;
          mbar_arrive_expect_tx(&full[stage], kUmABytes + bbytes);
          bulk_g2s(st, wbase + static_cast<size_t>(s) * kUmABytes, kUmABytes, &full[stage], pol);
          if (u.kind == 2) {
            // h slice s (its two W1 m-blocks of this group) must be complete
            const int c = s / P.slot_q;
            bool acq = s == 0;
            if (s == 0) miss = ld_acquire_u64(P.w1_slots + u.g) ^ P.w1_full;
            while ((miss >> (8 * c)) & 0xffu) {
              __nanosleep(64);
              miss = ld_acquire_u64(P.w1_slots + u.g) ^ P.w1_full;
              acq = true;
            }
            if (acq) fence_proxy_async_global();
          }
          bulk_g2s_nohint(st + kUmABytes,
                          bsrc + (static_cast<size_t>(s) * P.RG + (row0 >> 3)) * 2048, bbytes,
                          &full[stage]);
          if (++stage == kUmStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread) ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int seq = 0;; ++seq) {
        const int ds = seq & (kUmUnitRing - 1);
        mbar_wait(&dfull[ds], (seq / kUmUnitRing) & 1u);
        const UmUnit u = units[ds];
        mbar_arrive(&dempty[ds]);
        if (!u.kind) break;
        const int buf = seq & 1;
        mbar_wait(&tempty[buf], ((seq >> 1) & 1u) ^ 1u);  // the epilogue drained it
        tc_fence_after();
        const uint32_t idesc = umma_idesc(u.n);
        const uint32_t dt = tmem + buf * kUmAccCols;
        for (int s = 0; s < u.nst; ++s) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(ring + stage * kUmStageBytes);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_f16(dt, umma_smem_desc(sa + kk * 256), umma_smem_desc(sa + kUmABytes + kk * 256),
                     idesc, (s | kk) != 0);
          umma_commit(&empty[stage]);  // the stage's smem is free once these MMAs are done
          if (++stage == kUmStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        umma_commit(&tfull[buf]);  // accumulator complete
      }
    }
  } else {
    // ---------------- epilogue (warps 2-5 <-> TMEM lanes 32 (warp % 4) ..) ----------------
    const int q = warp & 3;
    const int m = 32 * q + lane;  // accumulator row (TMEM lane)
    for (int seq = 0;; ++seq) {
      const int ds = seq & (kUmUnitRing - 1);
      mbar_wait(&dfull[ds], (seq / kUmUnitRing) & 1u);
      const UmUnit u = units[ds];
      __syncwarp();
      if (lane == 0) mbar_arrive(&dempty[ds]);
      if (!u.kind) break;
      const int buf = seq & 1;
      mbar_wait(&tfull[buf], (seq >> 1) & 1u);
      tc_fence_after();
      const int row0 = P.group_row0[u.g], rows = P.group_rows[u.g];
      const uint32_t ta = tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * kUmAccCols;
      if (u.kind == 1) {
        // rows m: slot j = m / 16 holds gate (m % 16 < 8) and up (>= 8) of
        // h = 64 mb + 8 j + m % 8; the gate lane takes up from lane + 8
        const bool gate = (m & 15) < 8;
        const int hh = 64 * u.mb + 8 * (m >> 4) + (m & 7);
        const size_t hcol = (static_cast<size_t>(hh >> 7) * P.RG) * 2048 + ((hh & 127) >> 3) * 128 +
                            (hh & 7) * 2;
        for (int c = 0; c < u.n; c += 16) {
          float v[16];
          tmem_ld16(ta + c, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float up = __shfl_down_sync(0xffffffffu, v[j], 8);
            const int r = row0 + c + j;
            if (gate && c + j < rows) {
              const float hv = silu_f(v[j]) * up;
              *reinterpret_cast<__nv_bfloat16*>(P.hg + hcol + static_cast<size_t>(r >> 3) * 2048 +
                                                (r & 7) * 16) = __float2bfloat16_rn(hv);
            }
          }
        }
      } else {
        const int d = 128 * u.mb + m;
        for (int c = 0; c < u.n; c += 16) {
          float v[16];
          tmem_ld16(ta + c, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (c + j < rows) {
              const int r = row0 + c + j;
              const int t = P.row_tok[r];
              if (t >= 0)
                P.ybuf[(static_cast<size_t>(t) * P.stride + P.row_slot[r]) * P.Dp + d] = v[j];
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      if (u.kind == 1) {
        // publish this m-block of the group's h: the epilogue barrier orders
        // all 128 threads' stores before thread 0's cumulative release
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 2 && lane == 0)
          red_release_gpu_add_u64(P.w1_slots + u.g, 1ull << (8 * ((u.mb >> 1) / P.slot_q)));
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kUmTmemCols)
                 : "memory");
  }
  if (threadIdx.x == 0) {
    // the last CTA out resets the claims and the groups' slot counts
    __threadfence();
    if (atomicAdd(&P.claims[2], 1) == static_cast<int>(gridDim.x) - 1) {
      for (int g = 0; g < G; ++g) P.w1_slots[g] = 0ull;
      P.claims[0] = 0;
      P.claims[1] = 0;
      P.claims[2] = 0;
      __threadfence();
    }
  }
}

// Token rows of the plan (row -> token, -1 = padding) gathered into the CM
// layout of xg: one thread per 16-byte chunk (8 k of one row), threads in
// destination order (8 rows of a core matrix, then its 16 k-groups), so a
// warp's stores are one contiguous 512-byte run.
__global__ void k_gather_xg(const __nv_bfloat16* __restrict__ x, int Dp, const int32_t* __restrict__ row_tok,
                            const FfnHeader* __restrict__ hdr, int RG, uint8_t* __restrict__ xg) {
  const int nrows = hdr->n_rows;
  const int rgs = min((nrows + 16 + 7) >> 3, RG);  // row groups to fill (+ the N round-up slack)
  const int S = Dp >> 7;
  const int total = S * rgs * 128;                 // 16-byte chunks
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int r8 = i & 7, kg = (i >> 3) & 15, blk = i >> 7;
    const int rg = blk % rgs, s = blk / rgs;
    const int r = rg * 8 + r8;
    const int t = r < nrows ? row_tok[r] : -1;
    const uint4 v = t >= 0 ? __ldg(reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * Dp +
                                                                   s * 128 + kg * 8))
                           : make_uint4(0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(xg + (static_cast<size_t>(s) * RG + rg) * 2048 + kg * 128 + r8 * 16) = v;
  }
}

// out[t][d] = sum_j w[t][j] y[t][j][d] in set order (moe_layer.hpp:148-155):
// a thread per 4 outputs, all slots' y loads in flight before the ordered FMAs
__global__ void __launch_bounds__(256) k_umma_combine(int D, int Dp, int stride,
                                                      const int32_t* __restrict__ set_len,
                                                      const float* __restrict__ w32,
                                                      const float* __restrict__ y,
                                                      float* __restrict__ out) {
  pdl_wait();
  const int t = blockIdx.y;
  const int d = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (d >= D) return;
  const int len = set_len[t];
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j0 = 0; j0 < len; j0 += 8) {
    float4 v[8];
    float w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const bool ok = j0 + j < len;
      w[j] = ok ? w32[t * stride + j0 + j] : 0.0f;
      v[j] = ok ? __ldcg(reinterpret_cast<const float4*>(
                      y + (static_cast<size_t>(t) * stride + j0 + j) * Dp + d))
                : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j0 + j < len) {
        s.x = fmaf(w[j], v[j].x, s.x);
        s.y = fmaf(w[j], v[j].y, s.y);
        s.z = fmaf(w[j], v[j].z, s.z);
        s.w = fmaf(w[j], v[j].w, s.w);
      }
  }
  *reinterpret_cast<float4*>(out + static_cast<size_t>(t) * D + d) = s;
}

// Fragment-ordered bf16 expert weights -> CM layout (one 16-byte output
// chunk = 8 k of one row per thread; src_idx maps (row, k) to the fragment
// layout of layer.cu).
template <int KIND>  // 1: W1 (rows 2 Hp, k = d), 2: W2 (rows Dp, k = h)
__global__ void k_repack_cm(const __nv_bfloat16* __restrict__ src, int n_exp, int Dp, int Hp,
                            __nv_bfloat16* __restrict__ dst) {
  const int rows = KIND == 1 ? 2 * Hp : Dp, K = KIND == 1 ? Dp : Hp;
  const size_t per = static_cast<size_t>(rows) * K;
  const size_t nch = per / 8 * n_exp;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < nch;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int e = static_cast<int>(i / (per / 8));
    const size_t rem = i - static_cast<size_t>(e) * (per / 8);
    const int m = static_cast<int>(rem / (K / 8)), ch = static_cast<int>(rem % (K / 8));
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = ch * 8 + j;
      size_t o;
      if (KIND == 1) {
        const int h = 8 * (m >> 4) + (m & 7);
        o = w1_frag_index(k, h, (m & 15) >= 8, Dp);
      } else {
        o = w2_frag_index(k, m, Hp);
      }
      v[j] = src[static_cast<size_t>(e) * per + o];
    }
    const int mb = m >> 7, s = ch >> 4, kg = ch & 15, rg = (m & 127) >> 3;
    const int S = K >> 7;
    const size_t off = static_cast<size_t>(e) * per +
                       ((((static_cast<size_t>(mb) * S + s) * 16 + rg) * 16 + kg) * 64) + (m & 7) * 8;
    *reinterpret_cast<uint4*>(dst + off) = *reinterpret_cast<const uint4*>(v);
  }
}

}  // namespace oea_dev

namespace oea_host {

using namespace oea_dev;

// Makes the UMMA-layout copy (first use) or refreshes it IN PLACE (the
// weights changed): graphs captured with its pointers stay valid.
int layer_prepare_umma(oea_ctx* ctx, oea_layer* L, cudaStream_t s) {
  if (L->w1u == nullptr) {
    const size_t b1 = static_cast<size_t>(2 * L->Hp) * L->Dp * 2 * L->n_local;
    const size_t b2 = static_cast<size_t>(L->Dp) * L->Hp * 2 * L->n_local;
    OEA_CUDA_TRY(ctx, cudaMalloc(&L->w1u, b1));
    OEA_CUDA_TRY(ctx, cudaMalloc(&L->w2u, b2));
  }
  k_repack_cm<1><<<4 * 148, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(L->w1), L->n_local,
                                          L->Dp, L->Hp, static_cast<__nv_bfloat16*>(L->w1u));
  OEA_LAUNCHED(ctx);
  k_repack_cm<2><<<4 * 148, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(L->w2), L->n_local,
                                          L->Dp, L->Hp, static_cast<__nv_bfloat16*>(L->w2u));
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

void layer_drop_umma(oea_layer* L) {
  if (L->w1u) cudaFree(L->w1u);
  if (L->w2u) cudaFree(L->w2u);
  L->w1u = L->w2u = nullptr;
}

size_t umma_smem_bytes() {
  return kUmStages * kUmStageBytes + (2 * kUmStages + 4 + 2 * kUmUnitRing) * sizeof(uint64_t) +
         kUmUnitRing * sizeof(UmUnit) + 16;
}

int ffn_umma_launch(oea_ctx* ctx, const oea_layer* L, int B, int stride, const FfnBuffers& fb,
                    void* xg, int RG, cudaStream_t s, bool gathered) {
  // one 16-byte chunk per thread (all loads in one wave; rows past the plan's
  // are cut off in-kernel)
  // (gathered: the route-only launch already wrote xg with the compaction)
  if (!gathered) {
    const int gx = static_cast<int>(std::min<size_t>(65535, (static_cast<size_t>(L->Dp >> 7) * RG * 128 + 255) / 256));
    k_gather_xg<<<gx, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(fb.x), L->Dp, fb.row_tok,
                                   fb.hdr, RG, static_cast<uint8_t*>(xg));
    OEA_LAUNCHED(ctx);
  }
  UmmaParams P;
  P.w1u = static_cast<const uint8_t*>(L->w1u);
  P.w2u = static_cast<const uint8_t*>(L->w2u);
  P.w1u_stride = static_cast<size_t>(2 * L->Hp) * L->Dp * 2;
  P.w2u_stride = static_cast<size_t>(L->Dp) * L->Hp * 2;
  P.xg = static_cast<const uint8_t*>(xg);
  P.hg = static_cast<uint8_t*>(fb.hbuf);
  P.RG = RG;
  P.Dp = L->Dp;
  P.Hp = L->Hp;
  P.B = B;
  P.stride = stride;
  P.row_tok = fb.row_tok;
  P.row_slot = fb.row_slot;
  P.group_a = fb.group_a;
  P.group_row0 = fb.group_row0;
  P.group_rows = fb.group_rows;
  P.hdr = fb.hdr;
  P.w1_slots = reinterpret_cast<unsigned long long*>(fb.slice_done);
  {
    // slot field c: the h slices [c q, (c + 1) q), two W1 m-blocks each
    const int ns = L->Hp >> 7, q = (ns + 7) / 8;
    P.slot_q = q;
    P.w1_full = 0ull;
    for (int c = 0; c * q < ns; ++c)
      P.w1_full |= static_cast<unsigned long long>(2 * (std::min(ns, (c + 1) * q) - c * q)) << (8 * c);
  }
  P.claims = fb.counters + fb.max_groups;
  P.ybuf = static_cast<float*>(fb.ybuf);
  const size_t smem = umma_smem_bytes();
  static bool attr = false;
  if (!attr) {
    OEA_CUDA_TRY(ctx, cudaFuncSetAttribute(k_ffn_umma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
    attr = true;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(ctx->num_sms);
  lc.blockDim = dim3(kUmThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  OEA_CUDA_TRY(ctx, cudaLaunchKernelEx(&lc, k_ffn_umma, P));
  OEA_LAUNCHED(ctx);
  {
    // (programmatic dependent: launched while the FFN drains, waits for it)
    cudaLaunchConfig_t cc = {};
    cc.gridDim = dim3((L->D / 4 + 255) / 256, B);
    cc.blockDim = dim3(256);
    cc.stream = s;
    cc.attrs = at;
    cc.numAttrs = 1;
    OEA_CUDA_TRY(ctx, cudaLaunchKernelEx(&cc, k_umma_combine, L->D, L->Dp, stride, fb.set_len,
                                         static_cast<const float*>(fb.weights_f32),
                                         static_cast<const float*>(fb.ybuf), static_cast<float*>(fb.out)));
    OEA_LAUNCHED(ctx);
  }
  return OEA_OK;
}

}  // namespace oea_host
