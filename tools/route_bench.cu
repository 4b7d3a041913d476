// Cycle cost of the per-token ranking primitives (route_dev.cuh) on B200:
// one CTA, 9 warps, 16 tokens x 128 fp32 logits in shared memory; each warp
// ranks its tokens' top-k0 and we time (clock64) warp 0's selections.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_02237_b200/csrc \
//        -I include -o tools/route_bench tools/route_bench.cu
#include <cstdio>
#include <cstdlib>

#include "route_dev.cuh"

using namespace oea_dev;

// variant 0: tok_select as used by the fused prologue (+ the lane-0 bookkeeping)
// variant 1: tok_select only
// variant 2: lane-local sorted heads (each lane keeps its 4 keys sorted; a
//            selection = 1 redux on the head key + ballot/min-index on ties)
__device__ __forceinline__ void sort4_desc(uint32_t (&k)[4], int (&id)[4]) {
  auto cas = [&](int a, int b) {
    const bool sw = k[b] > k[a] || (k[b] == k[a] && id[b] < id[a]);
    if (sw) {
      uint32_t tk = k[a]; k[a] = k[b]; k[b] = tk;
      int ti = id[a]; id[a] = id[b]; id[b] = ti;
    }
  };
  cas(0, 1); cas(2, 3); cas(0, 2); cas(1, 3); cas(1, 2);
}

// Bitonic sort (descending) of 32*E packed keys per token, T tokens at once
// (independent networks interleaved for ILP). Position p = j*32 + lane.
template <int E, int T>
__device__ __forceinline__ void sort_desc(unsigned long long (&v)[T][E]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32 * E; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int js = stride >> 5;
#pragma unroll
        for (int t = 0; t < T; ++t)
#pragma unroll
          for (int j = 0; j < E; ++j)
            if ((j & js) == 0) {
              const int jj = j | js;
              const bool desc = ((j * 32 + lane) & size) == 0;
              const bool sw = desc ? v[t][jj] > v[t][j] : v[t][j] > v[t][jj];
              if (sw) { const auto x = v[t][j]; v[t][j] = v[t][jj]; v[t][jj] = x; }
            }
      } else {
#pragma unroll
        for (int t = 0; t < T; ++t)
#pragma unroll
          for (int j = 0; j < E; ++j) {
            const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[t][j], stride);
            const bool lower = (lane & stride) == 0;
            const bool desc = ((j * 32 + lane) & size) == 0;
            // lower lane keeps the larger when descending
            const bool take = (lower == desc) ? o > v[t][j] : o < v[t][j];
            if (take) v[t][j] = o;
          }
      }
    }
  }
}

// Thread-per-token scan: lane t keeps its token's top-K (key, index) sorted in
// registers while scanning the token's logits from a transposed [e][16] tile.
template <int K>
__device__ __forceinline__ void scan_topk(const float* lgT, int t, int N, uint32_t (&lk)[K], int (&li)[K]) {
#pragma unroll
  for (int i = 0; i < K; ++i) { lk[i] = 0u; li[i] = -1; }
#pragma unroll 8
  for (int e = 0; e < N; ++e) {
    const uint32_t kx = order_key32(lgT[e * 16 + t]);
    if (kx > lk[K - 1]) {
#pragma unroll
      for (int i = K - 1; i > 0; --i) {
        const bool up = kx > lk[i - 1];
        const bool here = !up && kx > lk[i];
        lk[i] = up ? lk[i - 1] : (here ? kx : lk[i]);
        li[i] = up ? li[i - 1] : (here ? e : li[i]);
      }
      if (kx > lk[0]) { lk[0] = kx; li[0] = e; }
    }
  }
}

// Two independent selections in one basic block (interleaved redux chains).
template <int E>
__device__ __forceinline__ void tok_select2(const TokRank<E>& A, const TokRank<E>& B2, uint32_t& ka,
                                            uint32_t& kb, int& ida, int& idb) {
  const int lane = threadIdx.x & 31;
  uint32_t ha = 0, la = 0, hb = 0, lb = 0;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const uint32_t l2 = 0xFFFFu - static_cast<uint32_t>(j * 32 + lane);
    const bool oka = A.key[j] != 0u && !((A.taken >> j) & 1u);
    const bool okb = B2.key[j] != 0u && !((B2.taken >> j) & 1u);
    if (oka && (A.key[j] > ha || (A.key[j] == ha && l2 > la))) { ha = A.key[j]; la = l2; }
    if (okb && (B2.key[j] > hb || (B2.key[j] == hb && l2 > lb))) { hb = B2.key[j]; lb = l2; }
  }
  const uint32_t wha = __reduce_max_sync(kFull, ha);
  const uint32_t whb = __reduce_max_sync(kFull, hb);
  const uint32_t wla = __reduce_max_sync(kFull, ha == wha ? la : 0u);
  const uint32_t wlb = __reduce_max_sync(kFull, hb == whb ? lb : 0u);
  ka = wha; kb = whb;
  ida = wha ? static_cast<int>(0xFFFFu - wla) : -1;
  idb = whb ? static_cast<int>(0xFFFFu - wlb) : -1;
}

__global__ void k_bench(const float* logits_g, int k0, int variant, long long* out, int* sel_out) {
  __shared__ float lg[16 * 128];
  __shared__ int srow[16 * 16];
  __shared__ float se[16 * 16];
  __shared__ uint32_t uni[4];
  for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) lg[i] = logits_g[i];
  if (threadIdx.x < 4) uni[threadIdx.x] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long t0 = clock64();
  __shared__ float lgT[128 * 16];
  if (variant == 6) {
    for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) lgT[(i % 128) * 16 + i / 128] = lg[i];
    __syncthreads();
    t0 = clock64();
  }
  for (int rep = 0; rep < 4; ++rep) {
    if (variant == 7) {
      // two tokens per warp, selections interleaved (independent redux chains)
      const int nw = blockDim.x >> 5;
      for (int ta = warp; ta < 16; ta += 2 * nw) {
        const int tb = ta + nw;
        const bool hb = tb < 16;
        TokRank<4> Ra, Rb;
        tok_load<4>(128, lg + ta * 128, Ra);
        tok_load<4>(128, lg + (hb ? tb : ta) * 128, Rb);
#pragma unroll 1
        for (int n = 0; n < k0; ++n) {
          uint32_t ka = 0, kb = 0;
          int ida, idb;
          tok_select2<4>(Ra, Rb, ka, kb, ida, idb);
          if (lane == 0) {
            srow[ta * 16 + n] = ida;
            if (hb) srow[tb * 16 + n] = idb;
          }
          tok_take<4>(Ra, ida);
          tok_take<4>(Rb, idb);
        }
      }
      __syncwarp();
      continue;
    }
    if (variant == 6) {
      if (warp == 0 && lane < 16) {
        if (k0 == 4) {
          uint32_t lk[4]; int li[4];
          scan_topk<4>(lgT, lane, 128, lk, li);
#pragma unroll
          for (int i = 0; i < 4; ++i) srow[lane * 16 + i] = li[i];
        } else {
          uint32_t lk[8]; int li[8];
          scan_topk<8>(lgT, lane, 128, lk, li);
#pragma unroll
          for (int i = 0; i < 8; ++i) srow[lane * 16 + i] = li[i];
        }
      }
      __syncwarp();
      continue;
    }
    if (variant == 5) {
      const int nw = blockDim.x >> 5;
      const int ta = warp, tb = warp + nw;
      unsigned long long v[2][4];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int t = u ? tb : ta;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          v[u][j] = t < 16 ? (static_cast<unsigned long long>(order_key32(lg[t * 128 + j * 32 + lane])) << 32) |
                                 (0xFFFFu - static_cast<unsigned>(j * 32 + lane))
                           : 0ull;
      }
      sort_desc<4, 2>(v);
      if (lane < k0) {
        srow[ta * 16 + lane] = 0xFFFF - static_cast<int>(v[0][0] & 0xFFFFu);
        if (tb < 16) srow[tb * 16 + lane] = 0xFFFF - static_cast<int>(v[1][0] & 0xFFFFu);
      }
      if (nw == 1) {  // 1 warp: the remaining 14 tokens pairwise
        for (int t2 = 2; t2 < 16; t2 += 2) {
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              v[u][j] = (static_cast<unsigned long long>(order_key32(lg[(t2 + u) * 128 + j * 32 + lane])) << 32) |
                        (0xFFFFu - static_cast<unsigned>(j * 32 + lane));
          sort_desc<4, 2>(v);
          if (lane < k0) {
            srow[t2 * 16 + lane] = 0xFFFF - static_cast<int>(v[0][0] & 0xFFFFu);
            srow[(t2 + 1) * 16 + lane] = 0xFFFF - static_cast<int>(v[1][0] & 0xFFFFu);
          }
        }
      }
      __syncwarp();
      continue;
    }
    for (int t = warp; t < 16; t += blockDim.x >> 5) {
      const float* row = lg + t * 128;
      if (variant <= 1) {
        TokRank<4> R;
        tok_load<4>(128, row, R);
        float rowmax = 0.0f;
#pragma unroll 1
        for (int n = 0; n < k0; ++n) {
          uint32_t key = 0;
          const int id = tok_select<4>(R, false, nullptr, key);
          if (id < 0) break;
          if (n == 0) rowmax = key32_to_logit(key);
          if (variant == 0 && lane == 0) {
            srow[t * 16 + n] = id;
            se[t * 16 + n] = expf(key32_to_logit(key) - rowmax);
            atomicOr(&uni[id >> 5], 1u << (id & 31));
          } else if (lane == 0) {
            srow[t * 16 + n] = id;
          }
          tok_take<4>(R, id);
        }
      } else if (variant == 4) {
        unsigned long long v[1][4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          v[0][j] = (static_cast<unsigned long long>(order_key32(row[j * 32 + lane])) << 32) |
                    (0xFFFFu - static_cast<unsigned>(j * 32 + lane));
        sort_desc<4, 1>(v);
        // ranks 0..k0-1 live in slot 0, lanes 0..k0-1
        if (lane < k0) srow[t * 16 + lane] = 0xFFFF - static_cast<int>(v[0][0] & 0xFFFFu);
      } else if (variant == 3) {
        uint32_t k[4];
        int id[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          k[j] = order_key32(row[j * 32 + lane]);
          id[j] = j * 32 + lane;
        }
        sort4_desc(k, id);
        int head = 0;
#pragma unroll 1
        for (int n = 0; n < k0; ++n) {
          unsigned long long v = head < 4 ? (static_cast<unsigned long long>(k[head & 3]) << 32) |
                                                (0xFFFFu - static_cast<unsigned>(id[head & 3]))
                                          : 0ull;
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long o2 = __shfl_xor_sync(kFull, v, off);
            v = o2 > v ? o2 : v;
          }
          const int win = 0xFFFF - static_cast<int>(v & 0xFFFFu);
          if (head < 4 && id[head & 3] == win) ++head;
          if (lane == 0) srow[t * 16 + n] = win;
        }
      } else {
        uint32_t k[4];
        int id[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          k[j] = order_key32(row[j * 32 + lane]);
          id[j] = j * 32 + lane;
        }
        sort4_desc(k, id);
        int head = 0;
#pragma unroll 1
        for (int n = 0; n < k0; ++n) {
          const uint32_t mine = head < 4 ? k[head & 3] : 0u;
          const int myid = head < 4 ? id[head & 3] : 0xFFFF;
          const uint32_t best = __reduce_max_sync(kFull, mine);
          const unsigned tie = __ballot_sync(kFull, mine == best);
          int win;
          if (__popc(tie) == 1) {
            win = __shfl_sync(kFull, myid, __ffs(tie) - 1);
          } else {
            win = static_cast<int>(__reduce_min_sync(kFull, mine == best ? static_cast<unsigned>(myid) : 0xFFFFu));
          }
          if (myid == win) ++head;
          if (lane == 0) srow[t * 16 + n] = win;
        }
      }
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *out = (t1 - t0) / 4;
  if (threadIdx.x < 16 * 16 && sel_out) sel_out[threadIdx.x] = srow[threadIdx.x];
}

int main() {
  float h[16 * 128];
  srand(7);
  for (int i = 0; i < 16 * 128; ++i) h[i] = (rand() / (float)RAND_MAX) * 4.0f - 2.0f;
  float* d;
  long long* o;
  int* sel;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&o, 8);
  cudaMalloc(&sel, 256 * 4);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  int ref[2][256], got[256];
  for (int variant = 0; variant < 8; ++variant) {
    for (int ki = 0; ki < 2; ++ki) {
      const int k0 = ki ? 8 : 4;
      long long c;
      for (int w = 0; w < 3; ++w) k_bench<<<1, 288>>>(d, k0, variant, o, sel);
      long long c1;
      k_bench<<<1, 32>>>(d, k0, variant, o, nullptr);
      cudaMemcpy(&c1, o, 8, cudaMemcpyDeviceToHost);
      printf("   1 warp x 16 tokens: %.0f cycles/select\n", c1 / (16.0 * k0));
      k_bench<<<1, 288>>>(d, k0, variant, o, sel);
      cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(variant == 0 ? ref[ki] : got, sel, sizeof(got), cudaMemcpyDeviceToHost);
      bool same = true;
      if (variant > 0)
        for (int t = 0; t < 16; ++t)
          for (int n = 0; n < k0; ++n) same &= ref[ki][t * 16 + n] == got[t * 16 + n];
      printf("variant %d k0=%d: %lld cycles per pass (2 tokens/warp) -> %.0f cycles/select %s\n",
             variant, k0, c, c / (2.0 * k0), same ? "" : "MISMATCH");
    }
  }
  return 0;
}
