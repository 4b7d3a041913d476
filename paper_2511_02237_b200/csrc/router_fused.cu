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
};

__device__ __forceinline__ void rstamp(const RouterParams& P, int rank, int slot) {
  if (P.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.trace[(1000 + rank) * 8 + slot] = t;
  }
}

constexpr int kRW = kRouterThreads / 32;  // 16 warps
constexpr int kMaxKtPerWarp = 16;          // k-tiles loaded per HBM round trip
constexpr int kXsPad = 8;                  // bf16 elements of row padding (bank spread)

__device__ __forceinline__ float key_to_logit(uint64_t k) {
  const uint32_t u = static_cast<uint32_t>(k >> 32);
  return __uint_as_float((u >> 31) ? (u & 0x7fffffffu) : ~u);
}

// Per-token routing state kept in registers between the two union phases.
template <int E>
struct TokState {
  uint64_t k[E];
  uint32_t id[E];
  int n_i;
};

template <int E>
__device__ __forceinline__ void tok_load_sort(const RouterParams& P, int t, TokState<E>& S) {
  const int lane = threadIdx.x & 31;
  const float* l = P.logits + static_cast<size_t>(t) * P.Np;
  float v[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int p = j * 32 + lane;
    v[j] = p < P.N ? __ldcg(l + p) : 0.0f;
  }
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int p = j * 32 + lane;
    S.k[j] = p < P.N ? order_key_f32(v[j]) : 0ull;
    S.id[j] = static_cast<uint32_t>(p);
  }
  warp_rank_sort<E>(S.k, S.id);
}

// Phase 1 (routing.cpp:226-268): baseline size n_i and the union bitmap.
template <int E>
__device__ __forceinline__ void tok_phase1(const RouterParams& P, int t, TokState<E>& S,
                                           uint32_t* s_union) {
  const int lane = threadIdx.x & 31;
  const Cfg& cfg = P.cfg;
  const bool real = P.mask == nullptr || P.mask[t] != 0;
  S.n_i = 0;
  if (!real || cfg.mode == OEA_MODE_VANILLA) return;
  int t_i = P.N;
  if (cfg.p != 1.0) {
    // Best-effort parity (documented): fp64 softmax of the fp32 logits, then
    // the reference's sequential cumulative mass in rank order.
    const double m = static_cast<double>(key_to_logit(__shfl_sync(kFull, S.k[0], 0)));
    double e[E], z = 0.0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
      e[j] = (j * 32 + lane) < P.N ? exp(static_cast<double>(key_to_logit(S.k[j])) - m) : 0.0;
      z += e[j];
    }
    for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(kFull, z, off);
    double cum = 0.0;
    bool done = false;
    for (int j = 0; j < E && !done; ++j)
      for (int src = 0; src < 32; ++src) {
        const int p = j * 32 + src;
        if (p >= P.N) {
          done = true;
          break;
        }
        cum = __dadd_rn(cum, __shfl_sync(kFull, e[j], src) / z);
        if (cum >= cfg.p) {
          t_i = p + 1;
          done = true;
          break;
        }
      }
  }
  S.n_i = min(cfg.k0, t_i);
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int p = j * 32 + lane;
    if (p < S.n_i) atomicOr(&s_union[S.id[j] >> 5], 1u << (S.id[j] & 31));
  }
}

// Phase 2 (routing.cpp:270-303) + weights (routing.cpp:33-49) + outputs.
// The selected set is always in ascending rank order (baseline ranks, then
// piggybacked ranks in scan order), so each lane knows which of its sorted
// positions are selected and the fp64 renormalisation runs over registers.
template <int E>
__device__ __forceinline__ void tok_phase2(const RouterParams& P, int t, const TokState<E>& S,
                                           const uint32_t* s_union, int* s_sets, int* s_len) {
  const int lane = threadIdx.x & 31;
  const Cfg& cfg = P.cfg;
  const bool real = P.mask == nullptr || P.mask[t] != 0;
  bool sel[E];
  int len = 0;
#pragma unroll
  for (int j = 0; j < E; ++j) sel[j] = false;
  if (real) {
    if (cfg.mode == OEA_MODE_VANILLA) {
#pragma unroll
      for (int j = 0; j < E; ++j) sel[j] = (j * 32 + lane) < cfg.k;
      len = cfg.k;
    } else {
#pragma unroll
      for (int j = 0; j < E; ++j) sel[j] = (j * 32 + lane) < S.n_i;
      len = S.n_i;
      if (cfg.mode != OEA_MODE_PRUNED) {
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const int p = j * 32 + lane;
          const bool cand = p >= S.n_i && p < cfg.max_p && p < P.N &&
                            ((s_union[S.id[j] >> 5] >> (S.id[j] & 31)) & 1u);
          const unsigned m = __ballot_sync(kFull, cand);
          const int take = max(cfg.limit - len, 0);
          if (cand && __popc(m & lanemask_lt()) < take) sel[j] = true;
          len += min(__popc(m), take);
        }
      }
    }
  }
  // fp64 weights: w = e / sum_set e, e = exp(l - max) (the softmax
  // denominator cancels); sequential sum in set order by lane 0.
  const double m = static_cast<double>(key_to_logit(__shfl_sync(kFull, S.k[0], 0)));
  double e[E];
#pragma unroll
  for (int j = 0; j < E; ++j)
    e[j] = sel[j] ? exp(static_cast<double>(key_to_logit(S.k[j])) - m) : 0.0;
  double mass = 0.0;
  int pos = 0;
  int32_t* gset = P.sets + static_cast<size_t>(t) * cfg.stride;
  int* sset = s_sets + t * cfg.stride;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    unsigned m2 = __ballot_sync(kFull, sel[j]);
    // set slots of the selected positions of this j-row, in lane order
    const int my = pos + __popc(m2 & lanemask_lt());
    if (sel[j]) {
      gset[my] = static_cast<int32_t>(S.id[j]);
      sset[my] = static_cast<int>(S.id[j]);
    }
    while (m2) {
      const int src = __ffs(m2) - 1;
      m2 &= m2 - 1;
      mass = __dadd_rn(mass, __shfl_sync(kFull, e[j], src));
    }
    pos += __popc(__ballot_sync(kFull, sel[j]));
  }
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const unsigned m2 = __ballot_sync(kFull, sel[j]);
    int before = 0;
#pragma unroll
    for (int jj = 0; jj < j; ++jj) before += __popc(__ballot_sync(kFull, sel[jj]));
    if (sel[j]) {
      const int slot = before + __popc(m2 & lanemask_lt());
      const double w = e[j] / mass;
      P.wts32[static_cast<size_t>(t) * cfg.stride + slot] = static_cast<float>(w);
      if (P.wts64) P.wts64[static_cast<size_t>(t) * cfg.stride + slot] = w;
    }
  }
  for (int j = len + lane; j < cfg.stride; j += 32) {
    gset[j] = -1;
    P.wts32[static_cast<size_t>(t) * cfg.stride + j] = 0.0f;
    if (P.wts64) P.wts64[static_cast<size_t>(t) * cfg.stride + j] = 0.0;
  }
  // export of the full order (sort_experts) for the parity harness
  int32_t* ord = P.order + static_cast<size_t>(t) * P.Np;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int p = j * 32 + lane;
    if (p < P.N) ord[p] = static_cast<int32_t>(S.id[j]);
  }
  if (lane == 0) {
    P.set_len[t] = len;
    s_len[t] = len;
    if (P.phase1_n) P.phase1_n[t] = S.n_i;
  }
}

template <int E>
__device__ void route_all(const RouterParams& P, uint32_t* s_union, int* s_sets, int* s_len,
                          int* s_n) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (P.B <= kRW) {
    // one token per warp: the sorted row stays in registers across the
    // union barrier
    TokState<E> S;
    const int t = warp;
    if (t < P.B) {
      tok_load_sort<E>(P, t, S);
      tok_phase1<E>(P, t, S, s_union);
    }
    __syncthreads();
    if (t < P.B) tok_phase2<E>(P, t, S, s_union, s_sets, s_len);
  } else {
    for (int t = warp; t < P.B; t += kRW) {
      TokState<E> S;
      tok_load_sort<E>(P, t, S);
      tok_phase1<E>(P, t, S, s_union);
      if (lane == 0) s_n[t] = S.n_i;
    }
    __syncthreads();
    for (int t = warp; t < P.B; t += kRW) {
      TokState<E> S;
      tok_load_sort<E>(P, t, S);  // re-rank (cheaper than keeping B rows)
      S.n_i = s_n[t];
      tok_phase2<E>(P, t, S, s_union, s_sets, s_len);
    }
  }
  __syncthreads();
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
  rstamp(P, crank, 0);

  const int Np = P.Np, B = P.B;
  const int KT = P.Dp >> 4, nrb = Np >> 4;
  const int kt0 = static_cast<int>(crank) * KT / kRouterCluster;
  const int kt1 = (static_cast<int>(crank) + 1) * KT / kRouterCluster;
  const int kslice = (kt1 - kt0) * 16;
  const int xs_stride = kslice + kXsPad;  // bf16 elements
  float* part = reinterpret_cast<float*>(smem);  // [kRouterTokChunk][Np]
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(part + kRouterTokChunk * Np);

  // ---- x -> zero-padded bf16 copy for the FFN when D is not a tile multiple ----
  if (P.xpad) {
    for (int t = crank; t < B; t += kRouterCluster)
      for (int d = threadIdx.x; d < P.Dp; d += kRouterThreads)
        P.xpad[static_cast<size_t>(t) * P.Dp + d] =
            d < P.D ? P.x[static_cast<size_t>(t) * P.D + d] : __float2bfloat16_rn(0.0f);
  }

  // ---- 1. split-K gate GEMV over the cluster ----
  const int ks_split = nrb <= kRW / 2 ? 2 : 1;
  for (int tc = 0; tc < B; tc += kRouterTokChunk) {
    const int ntok = min(kRouterTokChunk, B - tc);
    const int nbc = (ntok + 7) >> 3;
    // stage this CTA's K-slice of x (zero beyond D / the chunk)
    for (int i = threadIdx.x; i < kRouterTokChunk * Np; i += kRouterThreads) part[i] = 0.0f;
    for (int i = threadIdx.x; i < nbc * 8 * (kslice >> 1); i += kRouterThreads) {
      const int tt = i / (kslice >> 1), kk = (i % (kslice >> 1)) * 2;
      const int k = kt0 * 16 + kk;
      uint32_t v = 0;
      if (tt < ntok) {
        const __nv_bfloat16* xr = P.x + static_cast<size_t>(tc + tt) * P.D;
        if ((P.D & 1) == 0 && k + 1 < P.D) {
          v = __ldg(reinterpret_cast<const uint32_t*>(xr + k));
        } else {
          const unsigned short lo = k < P.D ? __bfloat16_as_ushort(xr[k]) : 0;
          const unsigned short hi = k + 1 < P.D ? __bfloat16_as_ushort(xr[k + 1]) : 0;
          v = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
        }
      }
      *reinterpret_cast<uint32_t*>(xs + tt * xs_stride + kk) = v;
    }
    __syncthreads();
    rstamp(P, crank, 1);
    for (int job = warp; job < nrb * ks_split; job += kRW) {
      const int rb = job % nrb, ks = job / nrb;
      const int ka = kt0 + (kt1 - kt0) * ks / ks_split;
      const int kb = kt0 + (kt1 - kt0) * (ks + 1) / ks_split;
      float acc[8][4];
#pragma unroll
      for (int nb = 0; nb < 8; ++nb) acc[nb][0] = acc[nb][1] = acc[nb][2] = acc[nb][3] = 0.0f;
      // A-tile loads of up to 16 k-tiles in flight at once (one HBM round
      // trip per 16 k-tiles; a single trip at D <= 4096, N <= 128).
      for (int kc = ka; kc < kb; kc += kMaxKtPerWarp) {
        uint4 a[kMaxKtPerWarp];
#pragma unroll
        for (int i = 0; i < kMaxKtPerWarp; ++i)
          if (kc + i < kb)
            a[i] = __ldg(P.rfrag + (static_cast<size_t>(rb) * KT + kc + i) * 32 + lane);
#pragma unroll
        for (int i = 0; i < kMaxKtPerWarp; ++i) {
          if (kc + i < kb) {
            const int kk = (kc + i - kt0) * 16 + 2 * q;
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
              if (nb < nbc) {
                const __nv_bfloat16* xr = xs + (nb * 8 + gq) * xs_stride + kk;
                const uint32_t b0 = *reinterpret_cast<const uint32_t*>(xr);
                const uint32_t b1 = *reinterpret_cast<const uint32_t*>(xr + 8);
                mma_bf16_16816(acc[nb], a[i], b0, b1);
              }
            }
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
    __syncthreads();
    rstamp(P, crank, 2);
    cluster.sync();
    rstamp(P, crank, 3);
    // Distributed fixed-order reduction over DSMEM: CTA c sums slice c of
    // every CTA's partial (ranks 0..7 in order) into the global logits.
    {
      const int elems = ntok * Np;
      const int e0 = static_cast<int>(crank) * elems / kRouterCluster;
      const int e1 = (static_cast<int>(crank) + 1) * elems / kRouterCluster;
      for (int i = e0 + threadIdx.x; i < e1; i += kRouterThreads) {
        float v[kRouterCluster];
#pragma unroll
        for (int r = 0; r < kRouterCluster; ++r) v[r] = cluster.map_shared_rank(part, r)[i];
        float s = 0.0f;
#pragma unroll
        for (int r = 0; r < kRouterCluster; ++r) s += v[r];
        P.logits[static_cast<size_t>(tc) * Np + i] = s;
      }
    }
    cluster.sync();
  }
  rstamp(P, crank, 4);
  if (crank != 0) return;

  // ---- 2. routing (CTA 0), register-resident per token ----
  uint32_t* s_union = reinterpret_cast<uint32_t*>(smem);      // [ceil(Np/32)]
  const int uw = (Np + 31) >> 5;
  int* s_len = reinterpret_cast<int*>(s_union + uw);           // [B]
  int* s_sets = s_len + B;                                     // [B][stride]
  int* s_loads = s_sets + B * P.cfg.stride;                    // [Np]
  int* s_eslot = s_loads + Np;
  int* s_rowb = s_eslot + Np;
  int* s_grpb = s_rowb + Np;
  int* s_tmp = s_grpb + Np;                                    // [40]
  int* s_n = s_tmp + 40;                                       // [B]
  uint32_t* s_tokbits = reinterpret_cast<uint32_t*>(s_n + B);  // [Np][Bw]
  const int Bw = (B + 31) >> 5;
  for (int i = threadIdx.x; i < uw; i += kRouterThreads) s_union[i] = 0u;
  for (int i = threadIdx.x; i < Np * Bw; i += kRouterThreads) s_tokbits[i] = 0u;
  __syncthreads();

  if (Np <= 32)
    route_all<1>(P, s_union, s_sets, s_len, s_n);
  else if (Np <= 64)
    route_all<2>(P, s_union, s_sets, s_len, s_n);
  else if (Np <= 128)
    route_all<4>(P, s_union, s_sets, s_len, s_n);
  else
    route_all<8>(P, s_union, s_sets, s_len, s_n);

  rstamp(P, 0, 5);
  if ((P.base_union || P.base_union_count) && warp == 0) {
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

  // ---- 3. compaction for the FFN (from shared memory) ----
  CompactOut o{P.active_union, P.active_count, P.total_load, P.loads, P.row_tok, P.row_slot,
               P.group_a, P.group_row0, P.group_rows, P.hdr, P.counters, P.n_counters};
  compact_plan(B, P.N, P.cfg.stride, s_sets, s_len, s_loads, s_eslot, s_rowb, s_grpb, s_tokbits,
               s_tmp, o);
  rstamp(P, 0, 6);
  if (o.hdr->n_groups == 0) {
    for (size_t f = threadIdx.x; f < static_cast<size_t>(B) * P.D; f += kRouterThreads)
      P.out[f] = 0.0f;
  }
}

}  // namespace oea_dev

namespace oea_host {

using namespace oea_dev;

size_t router_fused_smem_bytes(int B, int Np, int Dp, int stride) {
  const int KT = Dp >> 4;
  const int kslice_max = ((KT + kRouterCluster - 1) / kRouterCluster) * 16;
  const size_t gemv = static_cast<size_t>(kRouterTokChunk) * Np * sizeof(float) +
                      static_cast<size_t>(kRouterTokChunk) * (kslice_max + kXsPad) * 2;
  const size_t route = (static_cast<size_t>((Np + 31) >> 5) + 2 * B + static_cast<size_t>(B) * stride +
                        4 * Np + 40) * 4 + static_cast<size_t>(Np) * ((B + 31) / 32) * 4;
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
  P.trace = rb.trace;
  const size_t smem = router_fused_smem_bytes(B, L->Np, L->Dp, cfg.stride);
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
