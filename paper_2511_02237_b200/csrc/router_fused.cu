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

#include <algorithm>
#include <cstdlib>
#include <climits>

#include "oea_device.cuh"
#include "oea_internal.cuh"
#include "route_dev.cuh"

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
    // (e < 0: a duplicate (token, expert) slot of a caller plan, served by the
    // y of its first occurrence, oea_moe_forward_plan_host)
    if (sl < set_len[t] && sets[idx] >= 0) {
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
    if (sl < set_len[t] && sets[idx] >= 0) {
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
              int32_t* __restrict__ counters, int n_counters, int32_t* __restrict__ loads_out,
              int64_t* __restrict__ total_load) {
  extern __shared__ int s_dyn[];
  int* s_loads = s_dyn;
  int* s_eslot = s_loads + N;
  int* s_rowb = s_eslot + N;
  int* s_grpb = s_rowb + N;
  // token bitmaps in shared memory when they fit (else the zeroed global copy)
  const int nbits = N * ((B + 31) >> 5);
  uint32_t* s_bits = reinterpret_cast<uint32_t*>(s_grpb + N);
  if (tokbits == nullptr) {
    for (int i = threadIdx.x; i < nbits; i += blockDim.x) s_bits[i] = 0u;
    tokbits = s_bits;
    __syncthreads();
  }
  __shared__ int s_tmp[40];
  CompactOut o{active_union, active_count, total_load, loads_out, row_tok, row_slot, group_a,
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
  __nv_bfloat16* xpad;  // null when D == Dp (the FFN then reads x directly)
  int B, D, Dp, N, Np;
  Cfg cfg;
  float* logits;  // [B][Np]
  int32_t* order;  // [B][Np] (export only)
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
  unsigned long long* trace;  // debug: rows 1000+rank of the FFN trace buffer
  int late_trigger;           // debug: launch the FFN only at the end (OEA_LATE_TRIGGER)
};

__device__ __forceinline__ void rstamp(const RouterParams& P, int rank, int slot) {
  if (P.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.trace[(1000 + rank) * 8 + slot] = t;
  }
}

constexpr int kRW = kRouterThreads / 32;  // 16 warps
constexpr int kXsPad = 8;                  // bf16 elements of row padding (bank spread)
constexpr int kAStageMax = 64 * 1024;      // router A-tile staging per pass

// Phase 1 (routing.cpp:226-268): the baseline = the first n_i = min(k0, t_i)
// ranks; p == 1 short-circuits t_i = N. For p < 1 the cumulative mass uses an
// fp64 softmax of the fp32 logits (documented best-effort parity). The
// baseline experts are OR-ed into the cluster's union bitmap (DSMEM atomics on
// CTA 0's copy).
template <int E, bool kMass>
__device__ __forceinline__ int tok_phase1(const RouterParams& P, TokRank<E>& R, uint32_t* g_union,
                                          int* srow, float* se, float& rowmax) {
  const int lane = threadIdx.x & 31;
  uint32_t key = 0;
  int id = tok_select<E>(R, false, nullptr, key);  // rank 0 anchors the weights
  rowmax = key32_to_logit(key);
  if (P.cfg.mode == OEA_MODE_VANILLA) return 0;
  constexpr bool mass_rule = kMass;  // p < 1: compiled into its own kernel variant
  double z = 0.0;
  if (mass_rule) {
#pragma unroll
    for (int j = 0; j < E; ++j)
      if (R.key[j] != 0u) z += exp(static_cast<double>(key32_to_logit(R.key[j])) - rowmax);
    #pragma unroll 1
    for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(kFull, z, off);
  }
  int n = 0;
  double cum = 0.0;
#pragma unroll 1
  while (n < P.cfg.k0 && id >= 0) {
    if (lane == 0) {
      srow[n] = id;
      se[n] = expf(key32_to_logit(key) - rowmax);
      atomicOr(&g_union[id >> 5], 1u << (id & 31));
    }
    tok_take<E>(R, id);
    ++n;
    if (mass_rule) {
      cum = __dadd_rn(cum, exp(static_cast<double>(key32_to_logit(key)) - rowmax) / z);
      if (cum >= P.cfg.p) break;
    }
    if (n >= P.cfg.k0) break;
    id = tok_select<E>(R, false, nullptr, key);
  }
  return n;
}

// Phase 2 (routing.cpp:270-303): piggyback the best union members of ranks
// n_i..max_p-1 until the cap; vanilla takes the top k. Then weights
// (renormalisation over the set, routing.cpp:33-49); the set, its length and
// the per-expert load / token-bitmap updates go to CTA 0 (DSMEM) for the
// compaction.
struct Gather {
  int* sets;           // CTA 0: [B][stride]
  int* len;            // CTA 0: [B]
  int* loads;          // CTA 0: [Np]
  uint32_t* tokbits;   // CTA 0: [Np][Bw]
  int Bw;
};

template <int E>
__device__ __forceinline__ void tok_phase2(const RouterParams& P, int t, TokRank<E>& R, int n_i,
                                           float rowmax, const uint32_t* l_union, int* srow,
                                           float* se, const Gather& G0) {
  const int lane = threadIdx.x & 31;
  const int stride = P.cfg.stride;
  int len = n_i;
  uint32_t key = 0;
  const bool vanilla = P.cfg.mode == OEA_MODE_VANILLA;
  if (vanilla) len = 0;
  if (P.cfg.mode != OEA_MODE_PRUNED) {
    const int cap = vanilla ? P.cfg.k : P.cfg.limit;
    const bool full_scan = vanilla || P.cfg.max_p >= P.N;
#pragma unroll 1
    while (len < cap) {
      const int id = tok_select<E>(R, !vanilla, l_union, key);
      if (id < 0) break;
      if (!full_scan && tok_rank_of<E>(R, key, id) >= P.cfg.max_p) break;
      if (lane == 0) {
        srow[len] = id;
        se[len] = expf(key32_to_logit(key) - rowmax);
      }
      tok_take<E>(R, id);
      ++len;
    }
  }
  __syncwarp();
  // sequential fp32 mass in set order, then w = e / mass
  float mass = 0.0f;
  #pragma unroll 1
  for (int j = 0; j < len; ++j) mass += se[j];
  #pragma unroll 1
  for (int j = lane; j < stride; j += 32) {
    const size_t o = static_cast<size_t>(t) * stride + j;
    if (j < len) {
      const int e = srow[j];
      const float w = se[j] / mass;
      P.sets[o] = e;
      P.wts32[o] = w;
      if (P.wts64) P.wts64[o] = static_cast<double>(w);
      G0.sets[t * stride + j] = e;
      atomicAdd(&G0.loads[e], 1);
      atomicOr(&G0.tokbits[e * G0.Bw + (t >> 5)], 1u << (t & 31));
    } else {
      P.sets[o] = -1;
      P.wts32[o] = 0.0f;
      if (P.wts64) P.wts64[o] = 0.0;
    }
  }
  if (lane == 0) {
    P.set_len[t] = len;
    G0.len[t] = len;
    if (P.phase1_n) P.phase1_n[t] = n_i;
  }
}

__device__ __forceinline__ void tok_phase2_masked(const RouterParams& P, int t, const Gather& G0) {
  const int lane = threadIdx.x & 31;
  #pragma unroll 1
  for (int j = lane; j < P.cfg.stride; j += 32) {
    const size_t o = static_cast<size_t>(t) * P.cfg.stride + j;
    P.sets[o] = -1;
    P.wts32[o] = 0.0f;
    if (P.wts64) P.wts64[o] = 0.0;
  }
  if (lane == 0) {
    P.set_len[t] = 0;
    G0.len[t] = 0;
    if (P.phase1_n) P.phase1_n[t] = 0;
  }
}

// Token ownership: within each 64-token chunk, CTA c owns tokens 8c..8c+7;
// local token li = chunk * 8 + i (<= 32 per CTA, <= 2 per warp).
__device__ __forceinline__ int owned_token(int crank, int li) {
  return (li >> 3) * kRouterTokChunk + crank * 8 + (li & 7);
}

template <int E, bool kMass>
__device__ __forceinline__ void route_cluster(const RouterParams& P, cg::cluster_group& cluster,
                                              unsigned crank, const float* s_lg, uint32_t* s_union,
                                              uint32_t* s_lunion, int* srow_all, float* se_all,
                                              int* s_nloc, float* s_mloc, const Gather& G0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stride = P.cfg.stride;
  const int nloc = ((P.B + kRouterTokChunk - 1) / kRouterTokChunk) * 8;
  uint32_t* g_union = cluster.map_shared_rank(s_union, 0);
  // Phase 1 for this CTA's tokens; per-token state goes to shared memory so
  // the token loop stays rolled (small code: this runs cold once per launch).
#pragma unroll 1
  for (int li = warp; li < nloc; li += kRW) {
    const int t = owned_token(crank, li);
    int n_i = 0;
    float rmax = 0.0f;
    if (t < P.B && (P.mask == nullptr || P.mask[t] != 0)) {
      TokRank<E> R;
      tok_load<E>(P.N, s_lg + li * P.Np, R);
      n_i = tok_phase1<E, kMass>(P, R, g_union, srow_all + li * stride, se_all + li * stride, rmax);
    }
    if (lane == 0) {
      s_nloc[li] = n_i;
      s_mloc[li] = rmax;
    }
  }
  if (crank == 0 && warp == 0) rstamp(P, 8, 1);
  cluster.sync();  // union complete (CTA 0's bitmap)
  if (crank == 0 && warp == 0) rstamp(P, 8, 2);
  #pragma unroll 1
  for (int i = threadIdx.x; i < ((P.Np + 31) >> 5); i += kRouterThreads) s_lunion[i] = g_union[i];
  __syncthreads();
#pragma unroll 1
  for (int li = warp; li < nloc; li += kRW) {
    const int t = owned_token(crank, li);
    if (t >= P.B) continue;
    if (P.mask != nullptr && P.mask[t] == 0) {
      tok_phase2_masked(P, t, G0);
      continue;
    }
    TokRank<E> R;
    tok_load<E>(P.N, s_lg + li * P.Np, R);
    const int n_i = s_nloc[li];
    const int* srow = srow_all + li * stride;
#pragma unroll 1
    for (int j = 0; j < n_i; ++j) tok_take<E>(R, srow[j]);
    tok_phase2<E>(P, t, R, n_i, s_mloc[li], s_lunion, srow_all + li * stride, se_all + li * stride,
                  G0);
  }
  if (crank == 0 && warp == 0) rstamp(P, 8, 3);
  cluster.sync();  // CTA 0 holds every token's set, length, loads, token bits
}

// Fused-path compaction (K3) from CTA 0's gathered shared memory: warp 0
// scans the experts (ballot prefix sums) and writes active_union / groups /
// padding rows; then all warps place each (token, slot) at
// row_base[slot(e)] + rank of t among the expert's tokens (token order, from
// the token bitmaps).
__device__ void compact_fused(const RouterParams& P, const int* s_sets, const int* s_len,
                              const int* s_loads, int* s_eslot, int* s_rowb,
                              const uint32_t* s_tokbits, int* s_tmp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int B = P.B, N = P.N, stride = P.cfg.stride;
  const int Bw = (B + 31) >> 5;
  if (warp == 0) {
    int T = 0, G = 0, R = 0, load = 0;
    #pragma unroll 1
    for (int base = 0; base < N; base += 32) {
      const int e = base + lane;
      const int m = e < N ? s_loads[e] : 0;
      const bool act = m > 0;
      const unsigned am = __ballot_sync(kFull, act);
      const int slot = T + __popc(am & lanemask_lt());
      const int ng = act ? (m + kTokGroup - 1) / kTokGroup : 0;
      const int nr = act ? (m / kTokGroup) * kTokGroup + ((m % kTokGroup) + 7) / 8 * 8 : 0;
      int gi = ng, ri = nr, li = m;  // inclusive scans
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int g2 = __shfl_up_sync(kFull, gi, o), r2 = __shfl_up_sync(kFull, ri, o),
                  l2 = __shfl_up_sync(kFull, li, o);
        if (lane >= o) {
          gi += g2;
          ri += r2;
          li += l2;
        }
      }
      const int g0 = G + gi - ng, r0 = R + ri - nr;
      if (e < N) {
        P.loads[e] = m;
        s_eslot[e] = act ? slot : -1;
      }
      if (act) {
        P.active_union[slot] = e;
        s_rowb[e] = r0;
        #pragma unroll 1
        for (int k = 0; k < ng; ++k) {
          P.group_a[g0 + k] = e;
          P.group_row0[g0 + k] = r0 + k * kTokGroup;
          P.group_rows[g0 + k] = min(kTokGroup, m - k * kTokGroup);
        }
        #pragma unroll 1
        for (int r = r0 + m; r < r0 + nr; ++r) P.row_tok[r] = -1;  // n-block padding
      }
      T += __popc(am);
      G += __shfl_sync(kFull, gi, 31);
      R += __shfl_sync(kFull, ri, 31);
      load += __shfl_sync(kFull, li, 31);
    }
    #pragma unroll 1
    for (int e = T + lane; e < N; e += 32) P.active_union[e] = -1;
    if (lane == 0) {
      P.hdr->n_groups = G;
      P.hdr->T = T;
      P.hdr->total_load = load;
      P.hdr->n_rows = R;
      *P.active_count = T;
      *P.total_load = load;
      s_tmp[0] = G;
    }
  } else {
    #pragma unroll 1
    for (int c = threadIdx.x - 32; c < P.n_counters; c += kRouterThreads - 32) P.counters[c] = 0;
  }
  __syncthreads();
  #pragma unroll 1
  for (int idx = threadIdx.x; idx < B * stride; idx += kRouterThreads) {
    const int t = idx / stride, sl = idx % stride;
    if (sl < s_len[t]) {
      const int e = s_sets[idx];
      const uint32_t* bits = s_tokbits + e * Bw;
      int rank = __popc(bits[t >> 5] & ((1u << (t & 31)) - 1u));
      #pragma unroll 1
      for (int w = 0; w < (t >> 5); ++w) rank += __popc(bits[w]);
      const int row = s_rowb[e] + rank;
      P.row_tok[row] = t;
      P.row_slot[row] = sl;
    }
  }
  if (s_tmp[0] == 0) {
    #pragma unroll 1
    for (size_t f = threadIdx.x; f < static_cast<size_t>(B) * P.D; f += kRouterThreads)
      P.out[f] = 0.0f;
  }
}

// Shared-memory carve-up of the router kernel (identical in every CTA).
struct RouterSmem {
  size_t part, xs, abuf, bar, lg, uni, luni, len, sets, srow, se, loads, eslot, rowb, tmp, tokbits,
      nloc, mloc, total;
  int ks_split, nkt, kslice, xs_stride, rb_per;
};

__host__ __device__ inline RouterSmem router_smem_layout(int B, int Np, int Dp, int stride) {
  RouterSmem L;
  const int KT = Dp >> 4, nrb = Np >> 4;
  L.ks_split = nrb <= kRW / 2 ? 2 : 1;
  L.nkt = (KT + kRouterCluster - 1) / kRouterCluster;
  L.kslice = L.nkt * 16;
  L.xs_stride = L.kslice + kXsPad;
  const int per_rb = L.nkt * kTileBytes;
  L.rb_per = nrb < kAStageMax / per_rb ? nrb : (kAStageMax / per_rb > 0 ? kAStageMax / per_rb : 1);
  const int uw = (Np + 31) >> 5, Bw = (B + 31) >> 5;
  const int nloc = ((B + kRouterTokChunk - 1) / kRouterTokChunk) * 8;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = (o + bytes + 127) & ~static_cast<size_t>(127);
    return at;
  };
  L.part = take(static_cast<size_t>(L.ks_split) * kRouterTokChunk * Np * 4);
  L.xs = take(static_cast<size_t>(kRouterTokChunk) * L.xs_stride * 2);
  L.abuf = take(static_cast<size_t>(L.rb_per) * per_rb);
  L.bar = take(8);
  L.lg = take(static_cast<size_t>(nloc) * Np * 4);
  L.uni = take(uw * 4);
  L.luni = take(uw * 4);
  L.len = take(B * 4);
  L.sets = take(static_cast<size_t>(B) * stride * 4);
  L.srow = take(static_cast<size_t>(nloc) * stride * 4);
  L.se = take(static_cast<size_t>(nloc) * stride * 4);
  L.loads = take(Np * 4);
  L.eslot = take(Np * 4);
  L.rowb = take(Np * 4);
  L.tmp = take(8 * 4);
  L.tokbits = take(static_cast<size_t>(Np) * Bw * 4);
  L.nloc = take(static_cast<size_t>(nloc) * 4);
  L.mloc = take(static_cast<size_t>(nloc) * 4);
  L.total = o;
  return L;
}

template <bool kMass>
__global__ void __cluster_dims__(kRouterCluster, 1, 1) __launch_bounds__(kRouterThreads, 1)
    k_router_fused(const RouterParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned crank = cluster.block_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, q = lane & 3;

  // Let the FFN grid get resident early; it waits (griddepcontrol.wait) for
  // this grid's completion before touching any of its outputs.
  if (!P.late_trigger) pdl_launch_dependents();
  rstamp(P, crank, 0);

  const int Np = P.Np, B = P.B;
  const int KT = P.Dp >> 4, nrb = Np >> 4;
  const RouterSmem SL = router_smem_layout(B, Np, P.Dp, P.cfg.stride);
  const int kt0 = static_cast<int>(crank) * KT / kRouterCluster;
  const int kt1 = (static_cast<int>(crank) + 1) * KT / kRouterCluster;
  const int nkt = kt1 - kt0;
  const int kslice = nkt * 16;
  const int xs_stride = SL.xs_stride;
  float* part = reinterpret_cast<float*>(smem + SL.part);  // [ks][kRouterTokChunk][Np]
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(smem + SL.xs);
  uint8_t* abuf = smem + SL.abuf;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SL.bar);
  float* s_lg = reinterpret_cast<float*>(smem + SL.lg);
  uint32_t* s_union = reinterpret_cast<uint32_t*>(smem + SL.uni);
  uint32_t* s_lunion = reinterpret_cast<uint32_t*>(smem + SL.luni);
  int* s_len = reinterpret_cast<int*>(smem + SL.len);
  int* s_sets = reinterpret_cast<int*>(smem + SL.sets);
  int* s_srow = reinterpret_cast<int*>(smem + SL.srow);
  float* s_se = reinterpret_cast<float*>(smem + SL.se);
  int* s_loads = reinterpret_cast<int*>(smem + SL.loads);
  int* s_eslot = reinterpret_cast<int*>(smem + SL.eslot);
  int* s_rowb = reinterpret_cast<int*>(smem + SL.rowb);
  int* s_tmp = reinterpret_cast<int*>(smem + SL.tmp);
  uint32_t* s_tokbits = reinterpret_cast<uint32_t*>(smem + SL.tokbits);
  const int Bw = (B + 31) >> 5;
  const int rb_per = SL.rb_per;
  // x rows can be bulk-copied when every K-slice start/end is 16 B aligned in
  // the caller's row (D % 8 == 0) and the slice lies inside D.
  const bool x_bulk = (P.D & 7) == 0 && kt1 * 16 <= P.D;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  // gather targets live in CTA 0; zero them before the first cluster barrier
#pragma unroll 1
  for (int i = threadIdx.x; i < ((Np + 31) >> 5); i += kRouterThreads) s_union[i] = 0u;
#pragma unroll 1
  for (int i = threadIdx.x; i < Np; i += kRouterThreads) s_loads[i] = 0;
#pragma unroll 1
  for (int i = threadIdx.x; i < Np * Bw; i += kRouterThreads) s_tokbits[i] = 0u;

  // ---- x -> zero-padded bf16 copy for the FFN when D is not a tile multiple ----
  if (P.xpad) {
    for (int t = crank; t < B; t += kRouterCluster)
      for (int d = threadIdx.x; d < P.Dp; d += kRouterThreads)
        P.xpad[static_cast<size_t>(t) * P.Dp + d] =
            d < P.D ? P.x[static_cast<size_t>(t) * P.D + d] : __float2bfloat16_rn(0.0f);
  }
  __syncthreads();

  // ---- 1. split-K gate GEMV over the cluster ----
  const int ks_split = SL.ks_split;
  uint32_t bar_phase = 0;
  for (int tc = 0, chunk = 0; tc < B; tc += kRouterTokChunk, ++chunk) {
    const int ntok = min(kRouterTokChunk, B - tc);
    const int nbc = (ntok + 7) >> 3;
    for (int rb0 = 0; rb0 < nrb; rb0 += rb_per) {
      const int nrbp = min(rb_per, nrb - rb0);
      // one elected thread issues every bulk copy of this pass on one mbarrier
      if (threadIdx.x == 0) {
        const uint64_t pol = l2_policy_evict_first();
        uint32_t bytes = static_cast<uint32_t>(nrbp) * nkt * kTileBytes;
        if (rb0 == 0 && x_bulk) bytes += static_cast<uint32_t>(ntok) * kslice * 2;
        mbar_arrive_expect_tx(bar, bytes);
        for (int r = 0; r < nrbp; ++r)
          bulk_g2s(abuf + static_cast<size_t>(r) * nkt * kTileBytes,
                   P.rfrag + (static_cast<size_t>(rb0 + r) * KT + kt0) * 32, nkt * kTileBytes, bar,
                   pol);
        if (rb0 == 0 && x_bulk)
          for (int tt = 0; tt < ntok; ++tt)
            bulk_g2s(xs + tt * xs_stride, P.x + static_cast<size_t>(tc + tt) * P.D + kt0 * 16,
                     kslice * 2, bar, pol);
      }
      if (rb0 == 0) {
        // zero rows beyond the chunk; generic (unaligned / ragged-D) x staging
        for (int i = threadIdx.x; i < nbc * 8 * (kslice >> 1); i += kRouterThreads) {
          const int tt = i / (kslice >> 1), kk = (i % (kslice >> 1)) * 2;
          if (x_bulk && tt < ntok) continue;
          const int k = kt0 * 16 + kk;
          uint32_t v = 0;
          if (tt < ntok) {
            const __nv_bfloat16* xr = P.x + static_cast<size_t>(tc + tt) * P.D;
            const unsigned short lo = k < P.D ? __bfloat16_as_ushort(xr[k]) : 0;
            const unsigned short hi = k + 1 < P.D ? __bfloat16_as_ushort(xr[k + 1]) : 0;
            v = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
          }
          *reinterpret_cast<uint32_t*>(xs + tt * xs_stride + kk) = v;
        }
      }
      __syncthreads();
      mbar_wait(bar, bar_phase);
      bar_phase ^= 1u;
      if (rb0 == 0) rstamp(P, crank, 1);
      for (int job = warp; job < nrbp * ks_split; job += kRW) {
        const int rl = job % nrbp, ks = job / nrbp;
        const int rb = rb0 + rl;
        const int ka = nkt * ks / ks_split, kb = nkt * (ks + 1) / ks_split;
        float acc[8][4];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) acc[nb][0] = acc[nb][1] = acc[nb][2] = acc[nb][3] = 0.0f;
        const uint4* at = reinterpret_cast<const uint4*>(abuf + static_cast<size_t>(rl) * nkt * kTileBytes);
        for (int kk = ka; kk < kb; ++kk) {
          const uint4 a = at[kk * 32 + lane];
          const int xo = kk * 16 + 2 * q;
#pragma unroll
          for (int nb = 0; nb < 8; ++nb) {
            if (nb < nbc) {
              const __nv_bfloat16* xr = xs + (nb * 8 + gq) * xs_stride + xo;
              mma_bf16_16816(acc[nb], a, *reinterpret_cast<const uint32_t*>(xr),
                             *reinterpret_cast<const uint32_t*>(xr + 8));
            }
          }
        }
        // C: rows = experts 16rb + gq (+8), cols = tokens 2q, 2q+1; each K half
        // owns its own partial buffer (no atomics, fixed reduction order).
        float* pk = part + static_cast<size_t>(ks) * kRouterTokChunk * Np;
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
          if (nb < nbc) {
            const int n0 = rb * 16 + gq;
            const int t0 = nb * 8 + 2 * q;
            pk[t0 * Np + n0] = acc[nb][0];
            pk[(t0 + 1) * Np + n0] = acc[nb][1];
            pk[t0 * Np + n0 + 8] = acc[nb][2];
            pk[(t0 + 1) * Np + n0 + 8] = acc[nb][3];
          }
        }
      }
      __syncthreads();  // abuf reuse by the next pass
    }
    rstamp(P, crank, 2);
    cluster.sync();
    rstamp(P, crank, 3);
    // Token-sliced fixed-order reduction over DSMEM: CTA c sums, for its 8
    // tokens of this chunk, every CTA's partials (ranks 0..7, K halves in
    // order) into its local logits rows (and the exported global logits).
    for (int i = threadIdx.x; i < 8 * Np; i += kRouterThreads) {
      const int tl = i / Np, n = i % Np;
      const int row = static_cast<int>(crank) * 8 + tl;  // row within the chunk
      if (row >= ntok) continue;
      float v[kRouterCluster * 2];
#pragma unroll
      for (int r = 0; r < kRouterCluster; ++r) {
        const float* pr = cluster.map_shared_rank(part, r);
        v[2 * r] = pr[row * Np + n];
        v[2 * r + 1] = ks_split == 2 ? pr[kRouterTokChunk * Np + row * Np + n] : 0.0f;
      }
      float s = 0.0f;
#pragma unroll
      for (int r = 0; r < 2 * kRouterCluster; ++r) s += v[r];
      s_lg[(chunk * 8 + tl) * Np + n] = s;
      P.logits[static_cast<size_t>(tc + row) * Np + n] = s;
    }
    cluster.sync();  // partials may be overwritten by the next chunk
  }
  rstamp(P, crank, 4);
  __syncthreads();

  // ---- 2. routing, distributed: each CTA ranks its own tokens ----
  Gather G0;
  G0.sets = cluster.map_shared_rank(s_sets, 0);
  G0.len = cluster.map_shared_rank(s_len, 0);
  G0.loads = cluster.map_shared_rank(s_loads, 0);
  G0.tokbits = cluster.map_shared_rank(s_tokbits, 0);
  G0.Bw = Bw;
  int* s_nloc = reinterpret_cast<int*>(smem + SL.nloc);      // per local token: n_i
  float* s_mloc = reinterpret_cast<float*>(smem + SL.mloc);  // per local token: max logit
  if (Np <= 128)
    route_cluster<4, kMass>(P, cluster, crank, s_lg, s_union, s_lunion, s_srow, s_se, s_nloc, s_mloc, G0);
  else
    route_cluster<8, kMass>(P, cluster, crank, s_lg, s_union, s_lunion, s_srow, s_se, s_nloc, s_mloc, G0);
  rstamp(P, crank, 5);
  if (crank != 0) return;

  if ((P.base_union || P.base_union_count) && warp == 1) {
    int c = 0;
    for (int base = 0; base < P.N; base += 32) {
      const int e = base + lane;
      const bool f = e < P.N && ((s_union[e >> 5] >> (e & 31)) & 1u);
      const unsigned m = __ballot_sync(kFull, f);
      if (f && P.base_union) P.base_union[c + __popc(m & lanemask_lt())] = e;
      c += __popc(m);
    }
    if (lane == 0 && P.base_union_count) *P.base_union_count = c;
  }

  // ---- 3. compaction for the FFN (CTA 0, from the gathered shared memory) ----
  compact_fused(P, s_sets, s_len, s_loads, s_eslot, s_rowb, s_tokbits, s_tmp);
  rstamp(P, 0, 6);
}

}  // namespace oea_dev

namespace oea_host {

using namespace oea_dev;

size_t router_fused_smem_bytes(int B, int Np, int Dp, int stride) {
  return router_smem_layout(B, Np, Dp, stride).total;
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
  P.trace = rb.trace;
  P.late_trigger = getenv("OEA_LATE_TRIGGER") != nullptr;
  const size_t smem = router_fused_smem_bytes(B, L->Np, L->Dp, cfg.stride);
  if (cfg.p != 1.0 && cfg.mode != OEA_MODE_VANILLA) {
    OEA_CUDA_TRY(ctx, cudaFuncSetAttribute(k_router_fused<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
    k_router_fused<true><<<kRouterCluster, kRouterThreads, smem, s>>>(P);
  } else {
    OEA_CUDA_TRY(ctx, cudaFuncSetAttribute(k_router_fused<false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
    k_router_fused<false><<<kRouterCluster, kRouterThreads, smem, s>>>(P);
  }
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

int compact_launch(oea_ctx* ctx, int B, int N, int stride, const CompactBuffers& cb,
                   uint32_t* tokbits, int32_t* active_union, int32_t* active_count,
                   cudaStream_t s) {
  const size_t bits = static_cast<size_t>(N) * ((B + 31) / 32) * 4;
  // token bitmaps in shared memory (zeroed in-kernel) when they fit
  const bool sbits = static_cast<size_t>(4) * N * sizeof(int) + bits <= 96 * 1024;
  if (!sbits) OEA_CUDA_TRY(ctx, cudaMemsetAsync(tokbits, 0, bits, s));
  const size_t smem = static_cast<size_t>(4) * N * sizeof(int) + (sbits ? bits : 0);
  if (smem > 48 * 1024)
    OEA_CUDA_TRY(ctx, cudaFuncSetAttribute(k_compact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
  k_compact<<<1, 512, smem, s>>>(B, N, stride, cb.sets, cb.set_len, sbits ? nullptr : tokbits,
                                 active_union,
                                 active_count, cb.row_tok, cb.row_slot, cb.group_a, cb.group_row0,
                                 cb.group_rows, cb.hdr, cb.counters, cb.n_counters, cb.loads_out,
                                 cb.total_load);
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
