// router_fused.cu — K2 + K3: the fused OEA router and active-expert
// compaction for bf16 layers, plus the generic compaction used by the fp32/fp64
// path and the fp64 router_scores kernel (moe_layer.hpp:71-90).
//
// k_router_fused: one thread-block cluster of 8 CTAs x 16 warps.
//   1. gate GEMV  logits = x . R  — split-K across the cluster: CTA c owns
//      K-slice c; warps issue fragment-ordered 16 B/lane router tile loads
//      (mma.sync m16n8k16, experts as M, tokens as N), partials land in each
//      CTA's shared memory and are reduced over DSMEM in a fixed CTA order
//      (deterministic) into fp32 logits.
//   2. CTA 0 routes (the batch union is a barrier across all tokens):
//      per-token warp bitonic rank sort on fp32 logits (score desc, index
//      asc: softmax is monotone so ranking logits equals ranking the
//      reference's softmax scores wherever exp does not underflow to ties,
//      i.e. logit spreads < ~700), Phase-1 baseline + shared-memory union
//      bitmap, Phase-2 ballot scan with both cap semantics, fp64
//      renormalisation w = e_j / sum_set e (the softmax denominator cancels
//      in routing.cpp:33-49), per-expert loads.
//   3. CTA 0 compacts: active_union, expert slots, per-expert token lists in
//      token order with the token's slot (inverse permutation), 64-token
//      groups padded to 8-row n-blocks, FFN header, counter reset, and the
//      zero-padded bf16 copy of x the FFN streams B fragments from.
#include <cooperative_groups.h>

#include <climits>

#include "oea_device.cuh"
#include "oea_internal.cuh"

namespace cg = cooperative_groups;

namespace oea_dev {

// ---------------------------------------------------------------------------
// Block-wide helpers.
// ---------------------------------------------------------------------------
// In-place exclusive scan of v[0..n) (shared memory); returns the total.
__device__ int block_exclusive_scan(int* v, int n, int* s_tmp /* >= 33 ints */) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  int carry = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int x = i < n ? v[i] : 0;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_tmp[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int w = 0; w < nwarps; ++w) {
        const int c = s_tmp[w];
        s_tmp[w] = run;
        run += c;
      }
      s_tmp[32] = run;
    }
    __syncthreads();
    if (i < n) v[i] = carry + s_tmp[warp] + incl - x;
    carry += s_tmp[32];
    __syncthreads();
  }
  return carry;
}

// Shared compaction (one CTA). Inputs: sets/set_len in global memory.
// Scratch: loads/eslot/row_base/group_base: shared [N]; tokbits: [N][Bw]
// zero-initialised (shared or global).
struct CompactOut {
  int32_t* active_union;
  int32_t* active_count;
  int64_t* total_load;
  int32_t* loads_out;  // may be null
  int32_t* row_tok;
  int32_t* row_slot;
  int32_t* group_a;
  int32_t* group_row0;
  int32_t* group_rows;
  FfnHeader* hdr;
  int32_t* counters;
  int n_counters;
};

__device__ void compact_plan(int B, int N, int stride, const int32_t* sets, const int32_t* set_len,
                             int* s_loads, int* s_eslot, int* s_rowb, int* s_grpb, uint32_t* tokbits,
                             int* s_tmp, const CompactOut& o) {
  const int Bw = (B + 31) >> 5;
  for (int e = threadIdx.x; e < N; e += blockDim.x) s_loads[e] = 0;
  __syncthreads();
  for (int idx = threadIdx.x; idx < B * stride; idx += blockDim.x) {
    const int t = idx / stride, sl = idx % stride;
    if (sl < set_len[t]) {
      const int e = sets[idx];
      atomicAdd(&s_loads[e], 1);
      atomicOr(&tokbits[e * Bw + (t >> 5)], 1u << (t & 31));
    }
  }
  __syncthreads();
  // active_union = ascending experts with load > 0 (fill_aggregates, routing.cpp:27-30)
  for (int e = threadIdx.x; e < N; e += blockDim.x) s_eslot[e] = s_loads[e] > 0 ? 1 : 0;
  __syncthreads();
  const int T = block_exclusive_scan(s_eslot, N, s_tmp);
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    const bool act = s_loads[e] > 0;
    const int slot = s_eslot[e];
    if (act) o.active_union[slot] = e;
    if (o.loads_out) o.loads_out[e] = s_loads[e];
    s_rowb[e] = 0;
    s_grpb[e] = 0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    if (s_loads[e] > 0) {
      const int a = s_eslot[e];
      const int m = s_loads[e];
      s_grpb[a] = (m + kTokGroup - 1) / kTokGroup;
      // all groups but the last hold exactly 64 rows; the last pads to 8
      s_rowb[a] = (m / kTokGroup) * kTokGroup + ((m % kTokGroup) + 7) / 8 * 8;
    } else {
      s_eslot[e] = -1;
    }
    if (e >= T) o.active_union[e] = -1;
  }
  __syncthreads();
  const int n_groups = block_exclusive_scan(s_grpb, T, s_tmp);
  const int n_rows = block_exclusive_scan(s_rowb, T, s_tmp);
  for (int r = threadIdx.x; r < n_rows; r += blockDim.x) {
    o.row_tok[r] = -1;
    o.row_slot[r] = 0;
  }
  for (int a = threadIdx.x; a < T; a += blockDim.x) {
    const int e = o.active_union[a];
    const int m = s_loads[e];
    const int ng = (m + kTokGroup - 1) / kTokGroup;
    for (int gi = 0; gi < ng; ++gi) {
      o.group_a[s_grpb[a] + gi] = e;
      o.group_row0[s_grpb[a] + gi] = s_rowb[a] + gi * kTokGroup;
      o.group_rows[s_grpb[a] + gi] = min(kTokGroup, m - gi * kTokGroup);
    }
  }
  __syncthreads();
  // Inverse permutation: (token t, slot s) -> row = row_base[a] + rank of t
  // among the expert's tokens (token order).
  int my_total = 0;
  for (int idx = threadIdx.x; idx < B * stride; idx += blockDim.x) {
    const int t = idx / stride, sl = idx % stride;
    if (sl < set_len[t]) {
      ++my_total;
      const int e = sets[idx];
      const uint32_t* bits = tokbits + e * Bw;
      int rank = __popc(bits[t >> 5] & ((1u << (t & 31)) - 1u));
      for (int w = 0; w < (t >> 5); ++w) rank += __popc(bits[w]);
      const int row = s_rowb[s_eslot[e]] + rank;
      o.row_tok[row] = t;
      o.row_slot[row] = sl;
    }
  }
  for (int c = threadIdx.x; c < o.n_counters; c += blockDim.x) o.counters[c] = 0;
  // total load
  for (int off = 16; off > 0; off >>= 1) my_total += __shfl_xor_sync(kFull, my_total, off);
  __syncthreads();
  if (threadIdx.x == 0) s_tmp[0] = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicAdd(&s_tmp[0], my_total);
  __syncthreads();
  if (threadIdx.x == 0) {
    o.hdr->n_groups = n_groups;
    o.hdr->T = T;
    o.hdr->total_load = s_tmp[0];
    o.hdr->n_rows = n_rows;
    *o.active_count = T;
    if (o.total_load) *o.total_load = s_tmp[0];
  }
  __syncthreads();
}

// Generic compaction kernel (fp32/fp64 path, drop-in moe_forward on a plan).
__global__ void __launch_bounds__(512)
    k_compact(int B, int N, int stride, const int32_t* __restrict__ sets,
              const int32_t* __restrict__ set_len, uint32_t* __restrict__ tokbits,
              int32_t* __restrict__ active_union, int32_t* __restrict__ active_count,
              int32_t* __restrict__ row_tok, int32_t* __restrict__ row_slot,
              int32_t* __restrict__ group_a, int32_t* __restrict__ group_row0,
              int32_t* __restrict__ group_rows, FfnHeader* __restrict__ hdr,
              int32_t* __restrict__ counters, int n_counters) {
  extern __shared__ int s_dyn[];
  int* s_loads = s_dyn;
  int* s_eslot = s_loads + N;
  int* s_rowb = s_eslot + N;
  int* s_grpb = s_rowb + N;
  __shared__ int s_tmp[40];
  CompactOut o{active_union, active_count, nullptr, nullptr, row_tok, row_slot, group_a,
               group_row0, group_rows, hdr, counters, n_counters};
  compact_plan(B, N, stride, sets, set_len, s_loads, s_eslot, s_rowb, s_grpb, tokbits, s_tmp, o);
}

// ---------------------------------------------------------------------------
// router_scores in fp64 (f32/f64 layers): thread per (t, n) logit with a
// sequential sum over d, then a row softmax with a sequential sum.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_router_logits_f64(const double* __restrict__ x, const T* __restrict__ R, int B,
                                    int D, int N, double* __restrict__ logits) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  if (n >= N) return;
  double acc = 0.0;
  for (int d = 0; d < D; ++d)
    acc = __dadd_rn(acc, __dmul_rn(x[static_cast<size_t>(t) * D + d],
                                   static_cast<double>(R[static_cast<size_t>(d) * N + n])));
  logits[static_cast<size_t>(t) * N + n] = acc;
}

__global__ void k_softmax_f64(const double* __restrict__ logits, int B, int N,
                              double* __restrict__ scores) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B) return;
  const double* l = logits + static_cast<size_t>(t) * N;
  double* s = scores + static_cast<size_t>(t) * N;
  double m = l[0];
  for (int j = 1; j < N; ++j) m = l[j] > m ? l[j] : m;
  double sum = 0.0;
  for (int j = 0; j < N; ++j) {
    const double e = exp(l[j] - m);
    s[j] = e;
    sum = __dadd_rn(sum, e);
  }
  for (int j = 0; j < N; ++j) s[j] = __ddiv_rn(s[j], sum);
}

// ---------------------------------------------------------------------------
// The fused router.
// ---------------------------------------------------------------------------
struct RouterParams {
  const uint4* rfrag;  // [Np/16][Dp/16][32] uint4
  const __nv_bfloat16* x;
  const uint8_t* mask;
  __nv_bfloat16* xpad;
  int B, D, Dp, N, Np;
  Cfg cfg;
  float* logits;  // [B][Np]
  int32_t* order;  // [B][Np]
  int32_t* sets;
  int32_t* set_len;
  float* wts32;
  double* wts64;
  int32_t* loads;
  int32_t* active_union;
  int32_t* active_count;
  int64_t* total_load;
  int32_t* row_tok;
  int32_t* row_slot;
  int32_t* group_a;
  int32_t* group_row0;
  int32_t* group_rows;
  FfnHeader* hdr;
  int32_t* counters;
  int n_counters;
  float* out;
  int32_t* phase1_n;
  int32_t* base_union;
  int32_t* base_union_count;
};

constexpr int kRW = kRouterThreads / 32;  // 16 warps

__device__ __forceinline__ uint32_t load_x_pair(const __nv_bfloat16* xrow, int k, int D) {
  // elements k, k+1 of a bf16 row (zero beyond D)
  if ((D & 1) == 0 && k + 1 < D) return __ldg(reinterpret_cast<const uint32_t*>(xrow + k));
  const unsigned short lo = k < D ? __bfloat16_as_ushort(xrow[k]) : 0;
  const unsigned short hi = k + 1 < D ? __bfloat16_as_ushort(xrow[k + 1]) : 0;
  return static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
}

template <int E>
__device__ void route_token_sort(const RouterParams& P, int t, float* s_rowmax) {
  const int lane = threadIdx.x & 31;
  const float* l = P.logits + static_cast<size_t>(t) * P.Np;
  uint64_t k[E];
  uint32_t id[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int p = j * 32 + lane;
    k[j] = p < P.N ? order_key_f32(__ldcg(l + p)) : 0ull;
    id[j] = static_cast<uint32_t>(p);
  }
  warp_rank_sort<E>(k, id);
  int32_t* ord = P.order + static_cast<size_t>(t) * P.Np;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int p = j * 32 + lane;
    if (p < P.N) ord[p] = static_cast<int32_t>(id[j]);
  }
  if (lane == 0) s_rowmax[t] = __ldcg(l + id[0]);
}

__global__ void __cluster_dims__(kRouterCluster, 1, 1) __launch_bounds__(kRouterThreads, 1)
    k_router_fused(const RouterParams P) {
  extern __shared__ __align__(16) uint8_t smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned crank = cluster.block_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, q = lane & 3;

  // Let the FFN grid get resident early; it waits (griddepcontrol.wait) for
  // this grid's completion before touching any of its outputs.
  pdl_launch_dependents();

  const int Np = P.Np, B = P.B;
  float* part = reinterpret_cast<float*>(smem);  // [kRouterTokChunk][Np]

  // ---- x -> zero-padded bf16 copy for the FFN (all CTAs share the work) ----
  {
    const size_t total = static_cast<size_t>(B) * P.Dp;
    for (size_t f = crank * kRouterThreads + threadIdx.x; f < total;
         f += kRouterCluster * kRouterThreads) {
      const int t = static_cast<int>(f / P.Dp), d = static_cast<int>(f % P.Dp);
      P.xpad[f] = d < P.D ? P.x[static_cast<size_t>(t) * P.D + d] : __float2bfloat16_rn(0.0f);
    }
  }

  // ---- 1. split-K gate GEMV over the cluster ----
  const int KT = P.Dp >> 4, nrb = Np >> 4;
  const int kt0 = static_cast<int>(crank) * KT / kRouterCluster;
  const int kt1 = (static_cast<int>(crank) + 1) * KT / kRouterCluster;
  const int ks_split = nrb <= kRW / 2 ? 2 : 1;
  for (int tc = 0; tc < B; tc += kRouterTokChunk) {
    const int ntok = min(kRouterTokChunk, B - tc);
    const int nbc = (ntok + 7) >> 3;
    for (int i = threadIdx.x; i < kRouterTokChunk * Np; i += kRouterThreads) part[i] = 0.0f;
    __syncthreads();
    for (int job = warp; job < nrb * ks_split; job += kRW) {
      const int rb = job % nrb, ks = job / nrb;
      const int ka = kt0 + (kt1 - kt0) * ks / ks_split;
      const int kb = kt0 + (kt1 - kt0) * (ks + 1) / ks_split;
      float acc[8][4];
#pragma unroll
      for (int nb = 0; nb < 8; ++nb) acc[nb][0] = acc[nb][1] = acc[nb][2] = acc[nb][3] = 0.0f;
      const __nv_bfloat16* xr[8];
#pragma unroll
      for (int nb = 0; nb < 8; ++nb) {
        const int tt = tc + nb * 8 + gq;
        xr[nb] = (nb < nbc && tt < B) ? P.x + static_cast<size_t>(tt) * P.D : nullptr;
      }
      for (int kt = ka; kt < kb; ++kt) {
        const uint4 a = __ldg(P.rfrag + (static_cast<size_t>(rb) * KT + kt) * 32 + lane);
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
          if (nb < nbc) {
            uint32_t b0 = 0, b1 = 0;
            if (xr[nb]) {
              b0 = load_x_pair(xr[nb], kt * 16 + 2 * q, P.D);
              b1 = load_x_pair(xr[nb], kt * 16 + 8 + 2 * q, P.D);
            }
            mma_bf16_16816(acc[nb], a, b0, b1);
          }
        }
      }
      // C: rows = experts 16rb + gq (+8), cols = tokens 2q, 2q+1 of the n-block.
      // Two K halves meet with 0 + a + b, which is order-independent.
#pragma unroll
      for (int nb = 0; nb < 8; ++nb) {
        if (nb < nbc) {
          const int n0 = rb * 16 + gq;
          const int t0 = nb * 8 + 2 * q;
          atomicAdd(&part[t0 * Np + n0], acc[nb][0]);
          atomicAdd(&part[(t0 + 1) * Np + n0], acc[nb][1]);
          atomicAdd(&part[t0 * Np + n0 + 8], acc[nb][2]);
          atomicAdd(&part[(t0 + 1) * Np + n0 + 8], acc[nb][3]);
        }
      }
    }
    cluster.sync();
    // Distributed fixed-order reduction over DSMEM: CTA c sums slice c of
    // every CTA's partial (ranks 0..7 in order) into the global logits.
    {
      const int elems = ntok * Np;
      const int e0 = static_cast<int>(crank) * elems / kRouterCluster;
      const int e1 = (static_cast<int>(crank) + 1) * elems / kRouterCluster;
      for (int i = e0 + threadIdx.x; i < e1; i += kRouterThreads) {
        float s = 0.0f;
#pragma unroll
        for (int r = 0; r < kRouterCluster; ++r) s += cluster.map_shared_rank(part, r)[i];
        const int tt = i / Np, n = i % Np;
        P.logits[static_cast<size_t>(tc + tt) * Np + n] = s;
      }
    }
    cluster.sync();
  }
  if (crank != 0) return;

  // ---- 2. routing (CTA 0) ----
  int* s_n = reinterpret_cast<int*>(smem);                   // [B]
  float* s_rowmax = reinterpret_cast<float*>(s_n + B);        // [B]
  int* s_len = reinterpret_cast<int*>(s_rowmax + B);          // [B]
  uint32_t* s_union = reinterpret_cast<uint32_t*>(s_len + B); // [Np/32]
  const int uw = (Np + 31) >> 5;
  int* s_loads = reinterpret_cast<int*>(s_union + uw);        // [Np]
  int* s_eslot = s_loads + Np;
  int* s_rowb = s_eslot + Np;
  int* s_grpb = s_rowb + Np;
  int* s_tmp = s_grpb + Np;                                   // [40]
  uint32_t* s_tokbits = reinterpret_cast<uint32_t*>(s_tmp + 40);  // [Np][Bw]
  const int Bw = (B + 31) >> 5;
  for (int i = threadIdx.x; i < uw; i += kRouterThreads) s_union[i] = 0u;
  for (int i = threadIdx.x; i < Np * Bw; i += kRouterThreads) s_tokbits[i] = 0u;
  __syncthreads();

  const Cfg& cfg = P.cfg;
  for (int t = warp; t < B; t += kRW) {
    const int E = (Np <= 32) ? 1 : (Np <= 64) ? 2 : (Np <= 128) ? 4 : 8;
    if (E == 1)
      route_token_sort<1>(P, t, s_rowmax);
    else if (E == 2)
      route_token_sort<2>(P, t, s_rowmax);
    else if (E == 4)
      route_token_sort<4>(P, t, s_rowmax);
    else
      route_token_sort<8>(P, t, s_rowmax);
    __syncwarp();
    const bool real = P.mask == nullptr || P.mask[t] != 0;
    int n_i = 0;
    if (real && cfg.mode != OEA_MODE_VANILLA) {
      const int32_t* ord = P.order + static_cast<size_t>(t) * Np;
      int t_i = P.N;
      if (cfg.p != 1.0) {
        // Best-effort parity (documented): fp64 softmax of the fp32 logits,
        // then the reference's sequential cumulative mass in rank order.
        const float* l = P.logits + static_cast<size_t>(t) * Np;
        const double m = static_cast<double>(s_rowmax[t]);
        double z = 0.0;
        for (int j = lane; j < P.N; j += 32) z += exp(static_cast<double>(__ldcg(l + j)) - m);
        for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(kFull, z, off);
        if (lane == 0) {
          double cum = 0.0;
          for (int j = 0; j < P.N; ++j) {
            cum = __dadd_rn(cum, exp(static_cast<double>(__ldcg(l + ord[j])) - m) / z);
            if (cum >= cfg.p) {
              t_i = j + 1;
              break;
            }
          }
        }
        t_i = __shfl_sync(kFull, t_i, 0);
      }
      n_i = min(cfg.k0, t_i);
      for (int j = lane; j < n_i; j += 32) {
        const int e = ord[j];
        atomicOr(&s_union[e >> 5], 1u << (e & 31));
      }
    }
    if (lane == 0) s_n[t] = n_i;
  }
  __syncthreads();

  for (int i = threadIdx.x; i < Np; i += kRouterThreads) s_loads[i] = 0;
  __syncthreads();
  for (int t = warp; t < B; t += kRW) {
    const bool real = P.mask == nullptr || P.mask[t] != 0;
    const int32_t* ord = P.order + static_cast<size_t>(t) * Np;
    int32_t* srow = P.sets + static_cast<size_t>(t) * cfg.stride;
    int len = 0;
    if (real) {
      if (cfg.mode == OEA_MODE_VANILLA) {
        len = cfg.k;
        for (int j = lane; j < len; j += 32) srow[j] = ord[j];
      } else {
        const int n_i = s_n[t];
        for (int j = lane; j < n_i; j += 32) srow[j] = ord[j];
        len = n_i;
        if (cfg.mode != OEA_MODE_PRUNED) {
          for (int base = n_i; base < cfg.max_p && len < cfg.limit; base += 32) {
            const int j = base + lane;
            const int e = j < cfg.max_p ? ord[j] : -1;
            const bool member = e >= 0 && ((s_union[e >> 5] >> (e & 31)) & 1u);
            const unsigned mm = __ballot_sync(kFull, member);
            const int pos = __popc(mm & lanemask_lt());
            const int take = cfg.limit - len;
            if (member && pos < take) srow[len + pos] = e;
            len += min(__popc(mm), take);
          }
        }
      }
    }
    for (int j = len + lane; j < cfg.stride; j += 32) {
      srow[j] = -1;
      P.wts32[static_cast<size_t>(t) * cfg.stride + j] = 0.0f;
      if (P.wts64) P.wts64[static_cast<size_t>(t) * cfg.stride + j] = 0.0;
    }
    __syncwarp();
    // Weights: w_j = e_j / sum_set e with e = exp(l - max) in fp64.
    const float* l = P.logits + static_cast<size_t>(t) * Np;
    const double m = static_cast<double>(s_rowmax[t]);
    double mass = 0.0;
    if (lane == 0)
      for (int j = 0; j < len; ++j)
        mass = __dadd_rn(mass, exp(static_cast<double>(__ldcg(l + srow[j])) - m));
    mass = __shfl_sync(kFull, mass, 0);
    for (int j = lane; j < len; j += 32) {
      const double w = exp(static_cast<double>(__ldcg(l + srow[j])) - m) / mass;
      P.wts32[static_cast<size_t>(t) * cfg.stride + j] = static_cast<float>(w);
      if (P.wts64) P.wts64[static_cast<size_t>(t) * cfg.stride + j] = w;
    }
    if (lane == 0) {
      P.set_len[t] = len;
      s_len[t] = len;
      if (P.phase1_n) P.phase1_n[t] = s_n[t];
    }
  }
  __syncthreads();
  if (P.base_union || P.base_union_count) {
    if (threadIdx.x == 0) {
      int c = 0;
      for (int e = 0; e < P.N; ++e)
        if ((s_union[e >> 5] >> (e & 31)) & 1u) {
          if (P.base_union) P.base_union[c] = e;
          ++c;
        }
      if (P.base_union_count) *P.base_union_count = c;
    }
  }

  // ---- 3. compaction for the FFN ----
  CompactOut o{P.active_union, P.active_count, P.total_load, P.loads, P.row_tok, P.row_slot,
               P.group_a, P.group_row0, P.group_rows, P.hdr, P.counters, P.n_counters};
  compact_plan(B, P.N, cfg.stride, P.sets, P.set_len, s_loads, s_eslot, s_rowb, s_grpb, s_tokbits,
               s_tmp, o);
  if (P.hdr->n_groups == 0) {
    for (size_t f = threadIdx.x; f < static_cast<size_t>(B) * P.D; f += kRouterThreads)
      P.out[f] = 0.0f;
  }
}

}  // namespace oea_dev

namespace oea_host {

using namespace oea_dev;

size_t router_fused_smem_bytes(int B, int Np) {
  const size_t gemv = static_cast<size_t>(kRouterTokChunk) * Np * sizeof(float);
  const size_t route = (3 * static_cast<size_t>(B) + ((Np + 31) >> 5) + 4 * Np + 40) * 4 +
                       static_cast<size_t>(Np) * ((B + 31) / 32) * 4;
  return gemv > route ? gemv : route;
}

int router_fused_launch(oea_ctx* ctx, const oea_layer* L, const Cfg& cfg, int B,
                        const FusedRouterBuffers& rb, cudaStream_t s) {
  RouterParams P;
  P.rfrag = static_cast<const uint4*>(L->router);
  P.x = rb.x;
  P.mask = rb.mask;
  P.xpad = rb.xpad;
  P.B = B;
  P.D = L->D;
  P.Dp = L->Dp;
  P.N = L->N;
  P.Np = L->Np;
  P.cfg = cfg;
  P.logits = rb.logits;
  P.order = rb.order;
  P.sets = rb.sets;
  P.set_len = rb.set_len;
  P.wts32 = rb.weights_f32;
  P.wts64 = rb.weights_f64;
  P.loads = rb.loads;
  P.active_union = rb.active_union;
  P.active_count = rb.active_count;
  P.total_load = rb.total_load;
  P.row_tok = rb.row_tok;
  P.row_slot = rb.row_slot;
  P.group_a = rb.group_a;
  P.group_row0 = rb.group_row0;
  P.group_rows = rb.group_rows;
  P.hdr = rb.hdr;
  P.counters = rb.counters;
  P.n_counters = rb.n_counters;
  P.out = rb.out;
  P.phase1_n = rb.phase1_n;
  P.base_union = rb.base_union;
  P.base_union_count = rb.base_union_count;
  const size_t smem = router_fused_smem_bytes(B, L->Np);
  OEA_CUDA_TRY(ctx, cudaFuncSetAttribute(k_router_fused,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
  k_router_fused<<<kRouterCluster, kRouterThreads, smem, s>>>(P);
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

int compact_launch(oea_ctx* ctx, int B, int N, int stride, const CompactBuffers& cb,
                   uint32_t* tokbits, int32_t* active_union, int32_t* active_count,
                   cudaStream_t s) {
  const size_t bits = static_cast<size_t>(N) * ((B + 31) / 32) * 4;
  OEA_CUDA_TRY(ctx, cudaMemsetAsync(tokbits, 0, bits, s));
  const size_t smem = static_cast<size_t>(4) * N * sizeof(int);
  if (smem > 48 * 1024)
    OEA_CUDA_TRY(ctx, cudaFuncSetAttribute(k_compact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
  k_compact<<<1, 512, smem, s>>>(B, N, stride, cb.sets, cb.set_len, tokbits, active_union,
                                 active_count, cb.row_tok, cb.row_slot, cb.group_a, cb.group_row0,
                                 cb.group_rows, cb.hdr, cb.counters, cb.n_counters);
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

int router_scores_launch(oea_ctx* ctx, const oea_layer* L, const double* x, int B,
                         double* logits_ws, double* scores, cudaStream_t s) {
  dim3 g((L->N + 127) / 128, B);
  if (L->dtype == OEA_DTYPE_F64)
    k_router_logits_f64<double><<<g, 128, 0, s>>>(x, static_cast<const double*>(L->router), B,
                                                  L->D, L->N, logits_ws);
  else
    k_router_logits_f64<float><<<g, 128, 0, s>>>(x, static_cast<const float*>(L->router), B, L->D,
                                                 L->N, logits_ws);
  OEA_LAUNCHED(ctx);
  k_softmax_f64<<<(B + 127) / 128, 128, 0, s>>>(logits_ws, B, L->N, scores);
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

}  // namespace oea_host
