// routing.cu — K1 `route_f64`: batch-aware OEA routing on fp64 router
// probabilities, bit-exact with the reference's route() (routing.cpp:305-326).
//
// Three launches on one stream (the batch union is a global barrier):
//   A  k_rank_phase1   warp per token: bitonic rank sort of the row
//                      (sort_experts, routing.cpp:184-203), Phase-1 baseline
//                      size t/n (phase1_baseline :226-268) and the base union
//                      as an atomicOr bitmap.
//   B  k_build_sets    warp per token: top-k / baseline / Phase-2 piggyback
//                      scan with both cap semantics (phase2_piggyback
//                      :270-303) as a ballot scan, sequential fp64
//                      renormalisation (renormalize_weights :33-49), per-expert
//                      loads by integer atomics (fill_aggregates :17-31).
//   C  k_aggregate     one CTA: active_union (ascending, load > 0), T, and the
//                      exported base union.
// Bit-exactness: ranking uses an order-preserving integer image of each double
// (-0.0 canonicalised), so comparisons equal the reference's `!=`/`>`; the
// cumulative mass and the renormalisation are sequential __dadd_rn/__ddiv_rn in
// the reference's order (no FMA contraction is possible: adds and divides only).
#include <climits>

#include "oea_device.cuh"
#include "oea_internal.cuh"

namespace oea_dev {

constexpr int kRouteWarps = 8;

template <int E>
__global__ void __launch_bounds__(kRouteWarps * 32)
    k_rank_phase1(const Cfg cfg, const int B, const int N, const double* __restrict__ scores,
                  const uint8_t* __restrict__ mask, int32_t* __restrict__ order,
                  int32_t* __restrict__ t_out, int32_t* __restrict__ n_out,
                  uint32_t* __restrict__ union_bits, const int order_given,
                  const int run_phase1, const int32_t* __restrict__ seg) {
  __shared__ int32_t s_ord[kRouteWarps][32 * E];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kRouteWarps + warp;
  if (i >= B) return;
  const double* row = scores + static_cast<size_t>(i) * N;
  int32_t* ord_row = order + static_cast<size_t>(i) * N;
  int32_t* so = s_ord[warp];

  if (!order_given) {
    uint64_t k[E];
    uint32_t id[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int p = j * 32 + lane;
      k[j] = p < N ? order_key_f64(__ldcg(row + p)) : 0ull;
      id[j] = static_cast<uint32_t>(p);
    }
    warp_rank_sort<E>(k, id);
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int p = j * 32 + lane;
      so[p] = static_cast<int32_t>(id[j]);
      if (p < N) ord_row[p] = static_cast<int32_t>(id[j]);
    }
  } else {
    for (int p = lane; p < N; p += 32) so[p] = ord_row[p];
  }
  __syncwarp();
  if (!run_phase1) return;

  const bool real = mask == nullptr || mask[i] != 0;
  int t_i = 0, n_i = 0;
  if (real) {
    if (cfg.p == 1.0) {
      t_i = N;  // exact-compare short-circuit, routing.cpp:243-245
    } else {
      if (lane == 0) {
        t_i = N;
        double cum = 0.0;
        for (int j = 0; j < N; ++j) {  // routing.cpp:247-255, sequential
          cum = __dadd_rn(cum, row[so[j]]);
          if (cum >= cfg.p) {
            t_i = j + 1;
            break;
          }
        }
      }
      t_i = __shfl_sync(kFull, t_i, 0);
    }
    n_i = min(cfg.k0, t_i);
    // batched records: each record's own base union ([R][ceil(N/32)] words)
    uint32_t* ub = seg ? union_bits + static_cast<size_t>(seg[i]) * ((N + 31) >> 5) : union_bits;
    for (int j = lane; j < n_i; j += 32) {
      const int e = so[j];
      atomicOr(&ub[e >> 5], 1u << (e & 31));
    }
  }
  if (lane == 0) {
    if (t_out) t_out[i] = t_i;
    n_out[i] = n_i;
  }
}

// set_mode: 0 = first k ranks (route_topk), 1 = baseline only (pruned),
//           2 = baseline + piggyback scan (oea / simplified / phase2).
__global__ void __launch_bounds__(kRouteWarps * 32)
    k_build_sets(const Cfg cfg, const int B, const int N, const int set_mode,
                 const int do_weights, const double* __restrict__ scores,
                 const uint8_t* __restrict__ mask, const int32_t* __restrict__ order,
                 const int32_t* __restrict__ n_in, const uint32_t* __restrict__ union_bits,
                 int32_t* __restrict__ sets, int32_t* __restrict__ set_len,
                 double* __restrict__ weights, float* __restrict__ weights_f32,
                 int32_t* __restrict__ loads, unsigned long long* __restrict__ total_load,
                 int32_t* __restrict__ err_token, const int32_t* __restrict__ seg) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kRouteWarps + warp;
  if (i >= B) return;
  if (seg) {  // batched records: the record's union and aggregates
    const int sg = seg[i];
    union_bits += static_cast<size_t>(sg) * ((N + 31) >> 5);
    loads += static_cast<size_t>(sg) * N;
    total_load += sg;
  }
  const int stride = cfg.stride;
  const int32_t* ord = order + static_cast<size_t>(i) * N;
  int32_t* srow = sets + static_cast<size_t>(i) * stride;
  const bool real = mask == nullptr || mask[i] != 0;

  int len = 0;
  if (real) {
    if (set_mode == 0) {
      len = cfg.k;
      for (int j = lane; j < len; j += 32) srow[j] = ord[j];
    } else {
      const int n_i = n_in[i];
      for (int j = lane; j < n_i; j += 32) srow[j] = ord[j];
      len = n_i;
      if (set_mode == 2) {
        // Phase 2 (routing.cpp:291-299): candidates are ranks n_i..max_p-1 in
        // order; the cap is checked before each candidate, so members are
        // appended until |S| reaches `limit` (k_max, or k_max+1 for the
        // pseudocode cap); non-members are skipped without stopping.
        for (int base = n_i; base < cfg.max_p && len < cfg.limit; base += 32) {
          const int j = base + lane;
          const int e = j < cfg.max_p ? ord[j] : -1;
          const bool member = e >= 0 && ((union_bits[e >> 5] >> (e & 31)) & 1u);
          const unsigned m = __ballot_sync(kFull, member);
          const int pos = __popc(m & lanemask_lt());
          const int take = cfg.limit - len;
          if (member && pos < take) srow[len + pos] = e;
          len += min(__popc(m), take);
        }
      }
    }
  }
  for (int j = len + lane; j < stride; j += 32) {
    srow[j] = -1;
    if (weights) weights[static_cast<size_t>(i) * stride + j] = 0.0;
    if (weights_f32) weights_f32[static_cast<size_t>(i) * stride + j] = 0.0f;
  }
  __syncwarp();
  for (int j = lane; j < len; j += 32) atomicAdd(&loads[srow[j]], 1);
  if (lane == 0) {
    set_len[i] = len;
    atomicAdd(total_load, static_cast<unsigned long long>(len));
  }
  if (!do_weights || len == 0) return;

  // renormalize_weights (routing.cpp:33-49): sequential mass in set order.
  const double* row = scores + static_cast<size_t>(i) * N;
  double mass = 0.0;
  if (lane == 0) {
    for (int j = 0; j < len; ++j) mass = __dadd_rn(mass, row[srow[j]]);
    if (!(mass > 1e-12)) atomicMin(err_token, i);
  }
  mass = __shfl_sync(kFull, mass, 0);
  for (int j = lane; j < len; j += 32) {
    const double w = __ddiv_rn(row[srow[j]], mass);
    if (weights) weights[static_cast<size_t>(i) * stride + j] = w;
    if (weights_f32) weights_f32[static_cast<size_t>(i) * stride + j] = static_cast<float>(w);
  }
}

// Ascending compaction of {e : pred(e)} with a block-wide ballot scan.
template <typename Pred>
__device__ void block_compact(int N, Pred pred, int32_t* out, int32_t* count) {
  __shared__ int s_warp[32];
  __shared__ int s_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int base = 0; base < N; base += blockDim.x) {
    const int e = base + threadIdx.x;
    const bool f = e < N && pred(e);
    const unsigned m = __ballot_sync(kFull, f);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    int off = s_base;
    for (int w = 0; w < warp; ++w) off += s_warp[w];
    if (f && out) out[off + __popc(m & lanemask_lt())] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < nwarps; ++w) tot += s_warp[w];
      s_base += tot;
    }
    __syncthreads();
  }
  const int total = s_base;
  if (out)
    for (int e = total + threadIdx.x; e < N; e += blockDim.x) out[e] = -1;
  if (threadIdx.x == 0 && count) *count = total;
}

__global__ void __launch_bounds__(1024)
    k_aggregate(const int N, const int32_t* __restrict__ loads, int32_t* __restrict__ active_union,
                int32_t* __restrict__ active_count, const uint32_t* __restrict__ union_bits,
                int32_t* __restrict__ base_union, int32_t* __restrict__ base_count,
                int64_t* __restrict__ total_load) {
  pdl_wait();  // (programmatic dependent of the fast set kernels; else a no-op)
  // batched routing (route_f64_batched): CTA b aggregates record b, whose
  // per-record buffers sit at stride N (bitmaps: ceil(N / 32) words)
  if (blockIdx.x > 0) {
    const int b = blockIdx.x;
    loads += static_cast<size_t>(b) * N;
    active_union += static_cast<size_t>(b) * N;
    active_count += b;
    union_bits += static_cast<size_t>(b) * ((N + 31) >> 5);
    if (base_union) base_union += static_cast<size_t>(b) * N;
    if (base_count) base_count += b;
    if (total_load) total_load += b;
  }
  if (total_load) {  // fast path: total_load = sum of the loads (fill_aggregates)
    __shared__ long long s_part[32];
    long long mine = 0;
    for (int e = threadIdx.x; e < N; e += blockDim.x) mine += loads[e];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(kFull, mine, off);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t = 0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += s_part[w];
      *total_load = t;
    }
  }
  block_compact(N, [&](int e) { return loads[e] > 0; }, active_union, active_count);
  if (base_union || base_count)
    block_compact(N, [&](int e) { return (union_bits[e >> 5] >> (e & 31)) & 1u; },
                  base_union, base_count);
}

__global__ void k_union_from_list(const int32_t* __restrict__ list, const int count, const int N,
                                  uint32_t* __restrict__ bits) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < count; j += gridDim.x * blockDim.x) {
    const int e = list[j];
    if (e >= 0 && e < N) atomicOr(&bits[e >> 5], 1u << (e & 31));
  }
}

// ---------------------------------------------------------------------------
// Fast path (p == 1, max_p >= N, N <= 128, no full order requested): the
// reference's selections are all top-m picks in the composite order (score
// desc, index asc) with m <= k_max + 1, so no full sort is needed. Each lane
// keeps its <= 4 experts sorted in registers; a pick is a 5-step shuffle
// butterfly argmax over the lane heads (no redux: a redux.sync step costs
// several hundred cycles on this part, tools/route_bench.cu).
//   F1 k_fast_p1  warp per token: the first n_i = min(k0, N) ranks (p == 1:
//                 t_i = N, routing.cpp:243-245) or, vanilla, the first k
//                 (route_topk :205-224); the base union bitmap; for vanilla /
//                 pruned also the weights and loads (no second pass).
//   F2 k_fast_p2  warp per token (Oea / Simplified): the next union members
//                 in rank order until the cap (phase2_piggyback :270-303),
//                 then the weights and loads.
// ---------------------------------------------------------------------------
template <int E>
__device__ __forceinline__ void lane_sort_desc(uint64_t (&k)[E], int (&id)[E]) {
  if constexpr (E == 8) {
    // optimal 8-input network (19 compare-exchanges, depth 6) instead of the
    // 28 of the bubble network below
    constexpr int net[19][2] = {{0, 2}, {1, 3}, {4, 6}, {5, 7}, {0, 4}, {1, 5}, {2, 6},
                                {3, 7}, {0, 1}, {2, 3}, {4, 5}, {6, 7}, {2, 4}, {3, 5},
                                {1, 4}, {3, 6}, {1, 2}, {3, 4}, {5, 6}};
#pragma unroll
    for (int c = 0; c < 19; ++c) {
      const int a = net[c][0], b = net[c][1];
      const bool sw = ranks_before(k[b], id[b], k[a], id[a]);
      const uint64_t ka = k[a], kb = k[b];
      const int ia = id[a], ib = id[b];
      k[a] = sw ? kb : ka;
      k[b] = sw ? ka : kb;
      id[a] = sw ? ib : ia;
      id[b] = sw ? ia : ib;
    }
  } else {
#pragma unroll
    for (int a = 0; a < E; ++a)
#pragma unroll
      for (int b = E - 1; b > a; --b)
        if (ranks_before(k[b], id[b], k[b - 1], id[b - 1])) {
          const uint64_t tk = k[b];
          k[b] = k[b - 1];
          k[b - 1] = tk;
          const int ti = id[b];
          id[b] = id[b - 1];
          id[b - 1] = ti;
        }
  }
}

// Best (key desc, id asc) over the warp, in every lane.
__device__ __forceinline__ void warp_best(uint64_t& k, int& id) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const uint64_t ok = __shfl_xor_sync(kFull, k, off);
    const int oi = __shfl_xor_sync(kFull, id, off);
    if (ranks_before(ok, oi, k, id)) {
      k = ok;
      id = oi;
    }
  }
}

// Picks up to m more elements in rank order from the lanes' sorted lists
// (key 0 = no element) into srow[at..]; returns how many were picked.
template <int E>
__device__ __forceinline__ int pick_top(const uint64_t (&k)[E], const int (&id)[E], int m,
                                        int32_t* srow, int at) {
  const int lane = threadIdx.x & 31;
  int head = 0, got = 0;
#pragma unroll 1
  for (; got < m; ++got) {
    uint64_t bk = 0;
    int bid = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < E; ++j)
      if (j == head) {
        bk = k[j];
        bid = id[j];
      }
    warp_best(bk, bid);
    if (bk == 0) break;
    if ((bid & 31) == lane) ++head;  // the owning lane advances its list
    if (lane == 0) srow[at + got] = bid;
  }
  return got;
}

// Weights (renormalize_weights, routing.cpp:33-49: sequential fp64 mass in
// set order; the set's scores are loaded in parallel, one per lane, and the
// sum runs over shuffles) and the per-CTA load histogram.
__device__ __forceinline__ void fast_finish(const Cfg& cfg, int i, int len, const double* row,
                                            int32_t* srow, double* weights, float* weights_f32,
                                            int32_t* set_len, int* s_loads, int32_t* err_token,
                                            int do_weights) {
  const int lane = threadIdx.x & 31;
  const int stride = cfg.stride;
  __syncwarp();  // lane 0's set stores before the lanes read them
  const int e = lane < len ? srow[lane] : 0;
  const double sc = lane < len ? __ldcg(row + e) : 0.0;
  if (lane < len) atomicAdd(&s_loads[e], 1);
  for (int j = len + lane; j < stride; j += 32) {
    srow[j] = -1;
    if (weights) weights[static_cast<size_t>(i) * stride + j] = 0.0;
    if (weights_f32) weights_f32[static_cast<size_t>(i) * stride + j] = 0.0f;
  }
  if (lane == 0) set_len[i] = len;
  if (!do_weights || len == 0) return;
  double mass = 0.0;
#pragma unroll 1
  for (int j = 0; j < len; ++j) mass = __dadd_rn(mass, __shfl_sync(kFull, sc, j));
  if (lane == 0 && !(mass > 1e-12)) atomicMin(err_token, i);
  if (lane < len) {
    const double w = __ddiv_rn(sc, mass);
    if (weights) weights[static_cast<size_t>(i) * stride + lane] = w;
    if (weights_f32) weights_f32[static_cast<size_t>(i) * stride + lane] = static_cast<float>(w);
  }
}

__device__ __forceinline__ void flush_loads(int N, int* s_loads, int32_t* loads) {
  __syncthreads();
  for (int e = threadIdx.x; e < N; e += blockDim.x)
    if (s_loads[e]) atomicAdd(&loads[e], s_loads[e]);
}

// set_mode: 0 vanilla, 1 pruned (both complete here), 2 piggyback (F2 follows).
template <int E>
__global__ void __launch_bounds__(kRouteWarps * 32)
    k_fast_p1(const Cfg cfg, const int B, const int N, const int set_mode, const int do_weights,
              const double* __restrict__ scores, const uint8_t* __restrict__ mask,
              int32_t* __restrict__ sets, int32_t* __restrict__ set_len,
              int32_t* __restrict__ t_out, int32_t* __restrict__ n_out,
              uint32_t* __restrict__ union_bits, double* __restrict__ weights,
              float* __restrict__ weights_f32, int32_t* __restrict__ loads,
              int32_t* __restrict__ err_token, const int32_t* __restrict__ seg) {
  __shared__ int s_loads[128];
  pdl_launch_dependents();  // F2 / the aggregate may launch; they wait for this grid
  for (int e = threadIdx.x; e < 128; e += blockDim.x) s_loads[e] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kRouteWarps + warp;
  if (i < B) {
    const double* row = scores + static_cast<size_t>(i) * N;
    int32_t* srow = sets + static_cast<size_t>(i) * cfg.stride;
    const bool real = mask == nullptr || mask[i] != 0;
    // batched records: the token's record owns its union bitmap and loads
    const int sg = seg ? seg[i] : 0;
    uint32_t* ub = union_bits + static_cast<size_t>(sg) * ((N + 31) >> 5);
    int* cnt = seg ? loads + static_cast<size_t>(sg) * N : s_loads;
    uint64_t k[E];
    int id[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int p = j * 32 + lane;
      k[j] = p < N && real ? order_key_f64(__ldcg(row + p)) : 0ull;
      id[j] = p;
    }
    lane_sort_desc<E>(k, id);
    const int want = set_mode == 0 ? cfg.k : cfg.k0;
    const int n = real ? pick_top<E>(k, id, min(want, N), srow, 0) : 0;
    __syncwarp();
    if (set_mode != 0 && lane < n) {
      const int e = srow[lane];
      atomicOr(&ub[e >> 5], 1u << (e & 31));
    }
    if (lane == 0) {
      if (t_out) t_out[i] = set_mode == 0 ? 0 : (real ? N : 0);
      if (n_out) n_out[i] = set_mode == 0 ? 0 : n;
    }
    if (set_mode != 2)
      fast_finish(cfg, i, n, row, srow, weights, weights_f32, set_len, cnt, err_token,
                  do_weights);
  }
  if (set_mode != 2 && seg == nullptr) flush_loads(N, s_loads, loads);
}

template <int E>
__global__ void __launch_bounds__(kRouteWarps * 32)
    k_fast_p2(const Cfg cfg, const int B, const int N, const int do_weights,
              const double* __restrict__ scores, const uint8_t* __restrict__ mask,
              const int32_t* __restrict__ n_in, const uint32_t* __restrict__ union_bits,
              int32_t* __restrict__ sets, int32_t* __restrict__ set_len,
              double* __restrict__ weights, float* __restrict__ weights_f32,
              int32_t* __restrict__ loads, int32_t* __restrict__ err_token,
              const int32_t* __restrict__ seg) {
  __shared__ int s_loads[128];
  pdl_launch_dependents();  // the aggregate may launch; it waits for this grid
  for (int e = threadIdx.x; e < 128; e += blockDim.x) s_loads[e] = 0;
  __syncthreads();
  pdl_wait();  // F1's base sets, n and union bitmap (programmatic dependent)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kRouteWarps + warp;
  if (i < B) {
    const double* row = scores + static_cast<size_t>(i) * N;
    int32_t* srow = sets + static_cast<size_t>(i) * cfg.stride;
    const bool real = mask == nullptr || mask[i] != 0;
    const int sg = seg ? seg[i] : 0;
    const uint32_t* ub = union_bits + static_cast<size_t>(sg) * ((N + 31) >> 5);
    int* cnt = seg ? loads + static_cast<size_t>(sg) * N : s_loads;
    const int n = real ? n_in[i] : 0;
    int len = n;
    if (real && n < cfg.limit) {
      // candidates: union members not in the base set (the base set is the
      // top n overall, so every remaining member ranks after it). Base
      // bitmap: lane j < n contributes its expert, OR-reduced by shuffles.
      uint32_t bw[4] = {0u, 0u, 0u, 0u};
      if (lane < n) {
        const int e = srow[lane];
#pragma unroll
        for (int w = 0; w < 4; ++w) bw[w] = (e >> 5) == w ? 1u << (e & 31) : 0u;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int w = 0; w < 4; ++w) bw[w] |= __shfl_xor_sync(kFull, bw[w], off);
      uint64_t k[E];
      int id[E];
#pragma unroll
      for (int j = 0; j < E; ++j) {
        const int p = j * 32 + lane;
        const bool cand = p < N && ((ub[j] >> lane) & 1u) && !((bw[j] >> lane) & 1u);
        k[j] = cand ? order_key_f64(__ldcg(row + p)) : 0ull;
        id[j] = p;
      }
      lane_sort_desc<E>(k, id);
      len += pick_top<E>(k, id, cfg.limit - n, srow, n);
    }
    fast_finish(cfg, i, real ? len : 0, row, srow, weights, weights_f32, set_len, cnt,
                err_token, do_weights);
  }
  if (seg == nullptr) flush_loads(N, s_loads, loads);
}


// ---------------------------------------------------------------------------
// Single-launch fast path (same conditions as k_fast_p1/p2, one batch):
// TPT threads per token, thread q holds experts e = TPT j + q (EPT = 128 /
// TPT of them). A pick is the best (score desc, index asc) expert ranked
// after the previous pick: each thread scans its EPT keys (ascending index,
// so the strict compare keeps the lowest index among equal scores), then
// log2(TPT) shuffle levels inside the group. Picks come out in rank order,
// like pick_top, but a pick costs EPT register compares + 4 shuffle levels
// instead of 5 levels of 64-bit butterflies over the whole warp.
//   phase 1: the first n_i = min(k0, N) (p == 1: t_i = N, routing.cpp:243-245)
//            or, vanilla, k picks (route_topk :205-224); base union bitmap.
//   phase 2 (Oea / Simplified, after a grid barrier): union members ranked
//            after the base set, in rank order, until the cap
//            (phase2_piggyback :270-303); weights (renormalize_weights :33-49)
//            and loads.
// ---------------------------------------------------------------------------

template <int TPT>
__device__ __forceinline__ unsigned group_mask() {
  const int lane = threadIdx.x & 31;
  return (TPT == 32 ? 0xffffffffu : ((1u << TPT) - 1u)) << (lane & ~(TPT - 1));
}

// Single-launch route (one batch, grid co-resident: cooperative launch): G1
// and G2 above as two phases of one kernel, with everything a token needs
// after the picks kept in registers (its keys and raw scores; each pick's
// expert and score round robin over the group: pick r in thread r % TPT,
// slot r / TPT), so the only global round trip is the score load; one grid
// exchange for the batch union: CTA c stores its 4 pick-bitmap words as
// epoch-tagged words {tag:32 | bits:32} in its own slot, every CTA polls all
// slots until the tags are this launch's (no counter, no fence round trip,
// no reset: the next launch has another tag). The aggregates
// (fill_aggregates, routing.cpp:17-31) need no second grid-wide step: the
// experts with a load are the union of the phase-1 picks (every base-set
// member stays in its token's set, phase 2 only adds union members;
// vanilla: the picks are the sets), so CTA 0 writes the union exports right
// after the exchange, and the per-expert loads / total load / first
// degenerate token are atomics into the outputs, which CTA 0 clears before
// it publishes its words (release). CTA 0 advances the epoch once every
// CTA's words are in (every CTA read it before). No memsets precede the
// launch, no CTA waits at the end.
struct RouteScratch {
  int32_t epoch;  // launches so far (tag = (epoch & 0x7fffffff) + 1, never 0)
  int32_t pad[7];
  unsigned long long words[1];  // [grid][4] tagged union words
};
constexpr int kRouteMaxCtas = static_cast<int>((kRouteScratchBytes - 32) / 32);

// m picks (ranked after (pk, pe), eligible by elig_mask) in rank order; pick
// r lands in thread r % TPT's slot r / TPT (expert, raw score). Returns the
// number of picks (uniform over the group); (pk, pe) = the last pick.
// inverse of order_key_f64 (exact but for the sign of a zero score)
__device__ __forceinline__ double key_to_f64(uint64_t k) {
  return __longlong_as_double(static_cast<long long>((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

template <int TPT, int EPT, int U>
__device__ __forceinline__ int group_pick_regs(const uint64_t (&k)[EPT], uint32_t elig_mask, int q,
                                               int m, int at, int (&ex)[U], uint64_t (&sk)[U],
                                               uint64_t& pk, int& pe) {
  // (m is uniform over the warp and nothing diverges around the shuffles:
  // the whole warp takes part, so the full mask, no sub-warp syncs)
  const unsigned gm = 0xffffffffu;
  int got = 0;
#pragma unroll 1
  for (int r = 0; r < m; ++r) {
    uint64_t bk = 0ull;
    int be = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int e = TPT * j + q;
      const bool after = k[j] < pk || (k[j] == pk && e > pe);
      if (((elig_mask >> j) & 1u) && after && k[j] > bk) {
        bk = k[j];
        be = e;
      }
    }
#pragma unroll
    for (int off = 1; off < TPT; off <<= 1) {
      const uint64_t ok = __shfl_xor_sync(gm, bk, off);
      const int oe = __shfl_xor_sync(gm, be, off);
      if (ranks_before(ok, static_cast<uint32_t>(oe), bk, static_cast<uint32_t>(be))) {
        bk = ok;
        be = oe;
      }
    }
    if (bk != 0ull) {
      const int slot = at + got;
      // (selects, not an indexed store: ex / sk stay in registers)
      const bool mine = q == slot % TPT;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool hit = mine && u == slot / TPT;
        ex[u] = hit ? be : ex[u];
        sk[u] = hit ? bk : sk[u];
      }
      ++got;
      pk = bk;
      pe = be;
    } else {
      pk = 0ull;
      pe = 0x7fffffff;
    }
  }
  return got;
}

// The same picks from per-thread lists sorted once (lane_sort_desc): a
// pick's candidate is the thread's head, the owner of the group's best
// shifts its list, so a pick costs the group reduction only.
// KEYPICK: the group reduces the keys alone (2 shuffles a level instead of
// 3, a max instead of the (key, index) compare); the best key's head owner
// is found by a ballot, and only when several heads share that key (an
// exact tie, rare) does the warp reduce the indices too.
template <int TPT, int EPT, int U, bool KEYPICK = false>
__device__ __forceinline__ int group_pick_sorted(uint64_t (&k)[EPT], int (&id)[EPT], int q, int m,
                                                 int at, int (&ex)[U], uint64_t (&sk)[U],
                                                 uint64_t& pk, int& pe, bool track = true) {
  const unsigned gm = 0xffffffffu;  // (m uniform over the warp: converged)
  int got = 0;
#pragma unroll 1
  for (int r = 0; r < m; ++r) {
    uint64_t bk = k[0];
    int be;
    if constexpr (KEYPICK) {
#pragma unroll
      for (int off = 1; off < TPT; off <<= 1) {
        const uint64_t ok = __shfl_xor_sync(gm, bk, off);
        bk = ok > bk ? ok : bk;
      }
      const unsigned grp = group_mask<TPT>();
      const unsigned heads = __ballot_sync(gm, bk != 0ull && k[0] == bk) & grp;
      be = __shfl_sync(gm, id[0], heads ? __ffs(heads) - 1 : 0);
      if (__any_sync(gm, (heads & (heads - 1u)) != 0u)) {
        // equal best keys at several heads: the lowest index among them
        int ce = (heads >> (threadIdx.x & 31)) & 1u ? id[0] : 0x7fffffff;
#pragma unroll
        for (int off = 1; off < TPT; off <<= 1) ce = min(ce, __shfl_xor_sync(gm, ce, off));
        if (heads & (heads - 1u)) be = ce;
      }
    } else {
      be = k[0] != 0ull ? id[0] : 0x7fffffff;
#pragma unroll
      for (int off = 1; off < TPT; off <<= 1) {
        const uint64_t ok = __shfl_xor_sync(gm, bk, off);
        const int oe = __shfl_xor_sync(gm, be, off);
        if (ranks_before(ok, static_cast<uint32_t>(oe), bk, static_cast<uint32_t>(be))) {
          bk = ok;
          be = oe;
        }
      }
    }
    if (bk == 0ull) continue;  // nothing left (uniform over the group)
    const bool own = k[0] == bk && id[0] == be;
#pragma unroll
    for (int j = 0; j + 1 < EPT; ++j) {
      k[j] = own ? k[j + 1] : k[j];
      id[j] = own ? id[j + 1] : id[j];
    }
    if (own) k[EPT - 1] = 0ull;
    if (track) {
      pk = bk;
      pe = be;
    }
    const int slot = at + got;
    // (selects, not an indexed store: ex / sk stay in registers)
    const bool mine = q == slot % TPT;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool hit = mine && u == slot / TPT;
      ex[u] = hit ? be : ex[u];
      sk[u] = hit ? bk : sk[u];
    }
    ++got;
  }
  return got;
}

template <int TPT, int kGroupThreads, bool KEYPICK>
__global__ void __launch_bounds__(kGroupThreads)
    k_group_route(const Cfg cfg, const int B, const int N, const int set_mode, const int do_weights,
                  const double* __restrict__ scores, const uint8_t* __restrict__ mask,
                  int32_t* __restrict__ sets, int32_t* __restrict__ set_len,
                  int32_t* __restrict__ t_out, int32_t* __restrict__ n_out,
                  double* __restrict__ weights, float* __restrict__ weights_f32,
                  RouteScratch* __restrict__ scr, int32_t* __restrict__ loads_out,
                  int32_t* __restrict__ active_union, int32_t* __restrict__ active_count,
                  int64_t* __restrict__ total_load, int32_t* __restrict__ base_union,
                  int32_t* __restrict__ base_count, uint32_t* __restrict__ union_out,
                  int32_t* __restrict__ err_token, unsigned long long* __restrict__ trace) {
  constexpr int EPT = 128 / TPT;
  constexpr int U = 32 / TPT;  // sets of <= 32 (route_fast_ok)
  auto stamp = [&](int sl) {  // (debug timeline, OEA_FFN_TRACE=1)
    if (trace != nullptr && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[blockIdx.x * 8 + sl] = t;
    }
  };
  // programmatic dependent: the next launch in the stream may get resident
  // now; this grid's global reads (scores, the scratch epoch the previous
  // route advanced) wait for its predecessor
  pdl_launch_dependents();
  __shared__ int s_loads[128];
  __shared__ uint32_t s_union[4];
  __shared__ uint32_t s_batch[4];
  __shared__ int s_err;
  __shared__ int s_total;
  for (int e = threadIdx.x; e < 128; e += blockDim.x) s_loads[e] = 0;
  if (threadIdx.x < 4) {
    s_union[threadIdx.x] = 0u;
    s_batch[threadIdx.x] = 0u;
  }
  if (threadIdx.x == 0) {
    s_err = INT_MAX;
    s_total = 0;
  }
  pdl_wait();
  stamp(0);
  const int q = threadIdx.x & (TPT - 1);
  const int i = blockIdx.x * (kGroupThreads / TPT) + static_cast<int>(threadIdx.x) / TPT;
  const bool valid = i < B;
  const bool real = valid && (mask == nullptr || mask[i] != 0);
  const double* row = scores + static_cast<size_t>(valid ? i : 0) * N;
  // every score load of the thread issued before the first use (read-only
  // path, unconditional addresses): one memory round trip, not EPT
  double raw[EPT];
#pragma unroll
  for (int j = 0; j < EPT; ++j) raw[j] = __ldg(row + min(TPT * j + q, N - 1));
  const int epoch = __ldcg(&scr->epoch);
  const uint32_t tag = (static_cast<uint32_t>(epoch) & 0x7fffffffu) + 1u;
  __syncthreads();
  uint64_t k[EPT];
#pragma unroll
  for (int j = 0; j < EPT; ++j) k[j] = real && TPT * j + q < N ? order_key_f64(raw[j]) : 0ull;
  if (trace != nullptr) {  // (debug timeline: the keys are in registers)
    uint64_t any = 0ull;
#pragma unroll
    for (int j = 0; j < EPT; ++j) any |= k[j];
    if (any == 1ull) trace[0] = 0ull;
    stamp(6);
  }
  int ex[U];
  uint64_t sk[U];  // the picks' keys (the score is recovered from the key)
#pragma unroll
  for (int u = 0; u < U; ++u) {
    ex[u] = -1;
    sk[u] = 0ull;
  }
  // phase 1: base set (vanilla: the top k)
  const int want = min(set_mode == 0 ? cfg.k : cfg.k0, N);
  int id[EPT];
#pragma unroll
  for (int j = 0; j < EPT; ++j) id[j] = TPT * j + q;
  lane_sort_desc<EPT>(k, id);
  if (trace != nullptr && k[0] == 1ull) trace[1] = 0ull;
  stamp(7);
  uint64_t pk = 0ull;  // the last base pick (phase 2 picks rank after it)
  int pe = -1;
  const int n = group_pick_sorted<TPT, EPT, U, KEYPICK>(k, id, q, want, 0, ex, sk, pk, pe);
  stamp(1);
  if (valid) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q + TPT * u < n) atomicOr(&s_union[ex[u] >> 5], 1u << (ex[u] & 31));
  }
  if (valid && q == 0) {
    if (t_out) t_out[i] = set_mode == 0 ? 0 : (real ? N : 0);
    if (n_out) n_out[i] = set_mode == 0 ? 0 : n;
  }
  // the batch union: CTA 0 clears the accumulated outputs, then every CTA
  // publishes its pick bits as tagged words (CTA 0 with release: its clears
  // before any CTA's adds)
  __syncthreads();
  if (blockIdx.x == 0) {
    if (loads_out)
      for (int e = threadIdx.x; e < N; e += blockDim.x) loads_out[e] = 0;
    if (threadIdx.x == 0) {
      if (total_load) *total_load = 0;
      *err_token = INT_MAX;
    }
    __syncthreads();
  }
  if (threadIdx.x < 4) {
    unsigned long long* wp = &scr->words[blockIdx.x * 4 + threadIdx.x];
    const unsigned long long v = tagged(tag, s_union[threadIdx.x]);
    if (blockIdx.x == 0)
      st_release_u64(wp, v);
    else
      st_relaxed_u64(wp, v);
    stamp(2);
  }
  // phase 2, speculatively while the other CTAs' words arrive: the next
  // picks over the whole list (the lists' remaining entries all rank after
  // the base). They are phase2_piggyback's picks (routing.cpp:270-303)
  // whenever every one is a union member, checked after the exchange; else
  // the warp picks again among the members (rare at large B, where the
  // union is full).
  const int m = set_mode == 2 ? max(0, cfg.limit - min(cfg.k0, N)) : 0;
  int len = n;
  if (set_mode == 2) {
    const int got = group_pick_sorted<TPT, EPT, U, KEYPICK>(k, id, q, m, n, ex, sk, pk, pe, false);
    len = real ? n + min(got, max(0, cfg.limit - n)) : 0;
  }
  const int stride = cfg.stride;
  int32_t* srow = sets + static_cast<size_t>(valid ? i : 0) * stride;
  // the set, its length, loads and weights (renormalize_weights,
  // routing.cpp:33-49: sequential fp64 mass in set order, through group
  // shuffles); returns whether the mass is degenerate. sign = -1 takes the
  // set's slots from `from` on back out (a speculative set replaced).
  auto count = [&](int from, int sign) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = q + TPT * u;
      if (r >= from && r < len) atomicAdd(&s_loads[ex[u]], sign);
    }
    if (q == 0 && len > from) atomicAdd(&s_total, sign * (len - from));
  };
  auto emit = [&](int from) -> bool {
    bool bad = false;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = q + TPT * u;
      if (r >= from && r < len) srow[r] = ex[u];
    }
    for (int j = max(len, from) + q; j < stride; j += TPT) {
      srow[j] = -1;
      if (weights) weights[static_cast<size_t>(i) * stride + j] = 0.0;
      if (weights_f32) weights_f32[static_cast<size_t>(i) * stride + j] = 0.0f;
    }
    if (q == 0) set_len[i] = len;
    if (do_weights && len > 0) {
      // scores from the keys; a zero key may be a -0.0 score: read it back
      double sc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        sc[u] = key_to_f64(sk[u]);
        if (q + TPT * u < len && sk[u] == 0x8000000000000000ull) sc[u] = __ldg(row + ex[u]);
      }
      const unsigned gm = group_mask<TPT>();
      double mass = 0.0;
#pragma unroll 1
      for (int r = 0; r < len; ++r) {  // (len uniform over the group)
        double v = sc[0];
#pragma unroll
        for (int u = 1; u < U; ++u) v = r / TPT == u ? sc[u] : v;
        mass = __dadd_rn(mass, __shfl_sync(gm, v, r % TPT, TPT));
      }
      bad = !(mass > 1e-12);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = q + TPT * u;
        if (r < len) {
          const double w = __ddiv_rn(sc[u], mass);
          if (weights) weights[static_cast<size_t>(i) * stride + r] = w;
          if (weights_f32) weights_f32[static_cast<size_t>(i) * stride + r] = static_cast<float>(w);
        }
      }
    }
    return bad;
  };
  bool bad = false;
  if (valid) {
    bad = emit(0);
    count(0, 1);
  }
  stamp(4);
  // the batch union: poll every CTA's words (thread t: CTAs t, t + blockDim, ..)
  {
    uint32_t acc[4] = {0u, 0u, 0u, 0u};
    for (int c = threadIdx.x; c < static_cast<int>(gridDim.x); c += blockDim.x) {
      const unsigned long long* wp = &scr->words[c * 4];
      unsigned long long v[4];
      for (;;) {
#pragma unroll
        for (int w = 0; w < 4; ++w) v[w] = ld_relaxed_u64(wp + w);
        if ((v[0] >> 32) == tag && (v[1] >> 32) == tag && (v[2] >> 32) == tag && (v[3] >> 32) == tag) break;
      }
      if (c == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");  // (acquire: CTA 0's clears)
#pragma unroll
      for (int w = 0; w < 4; ++w) acc[w] |= static_cast<uint32_t>(v[w]);
    }
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t o = __reduce_or_sync(0xffffffffu, acc[w]);
      if ((threadIdx.x & 31) == 0 && o) atomicOr(&s_batch[w], o);
    }
  }
  __syncthreads();
  stamp(3);
  uint32_t uw[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) uw[w] = s_batch[w];
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    // the union exports (fill_aggregates): active experts = the union of
    // the picks; the base union (pruned / piggyback modes) is the same set
    const int lane = threadIdx.x;
    const unsigned below = lanemask_lt();
    const bool base = set_mode != 0;
    if (lane < 4 && union_out) union_out[lane] = base ? uw[lane] : 0u;
    int na = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int e = 32 * w + lane;
      const bool f = e < N && ((uw[w] >> lane) & 1u);
      const unsigned mb = __ballot_sync(0xffffffffu, f);
      if (f && active_union) active_union[na + __popc(mb & below)] = e;
      if (f && base && base_union) base_union[na + __popc(mb & below)] = e;
      na += __popc(mb);
    }
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int e = 32 * w + lane;
      if (e >= na && e < N && active_union) active_union[e] = -1;
      if ((e >= na || !base) && e < N && base_union) base_union[e] = -1;
    }
    if (lane == 0) {
      if (active_count) *active_count = na;
      if (base_count) *base_count = base ? na : 0;
      scr->epoch = epoch + 1;  // (every CTA has read it: its words are in)
    }
  }
  auto member = [&](int e) -> bool {
    const uint32_t word = e < 32 ? uw[0] : e < 64 ? uw[1] : e < 96 ? uw[2] : uw[3];
    return (word >> (e & 31)) & 1u;
  };
  bool miss = false;
  if (set_mode == 2) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = q + TPT * u;
      if (r >= n && r < len && !member(ex[u])) miss = true;
    }
  }
  if (__syncthreads_or(miss)) {
    // (taken by whole warps: the picks' full-warp shuffles; a group whose
    // picks were all members gets the same picks again)
    if (__any_sync(0xffffffffu, miss)) {
      if (valid) count(n, -1);
      // the union members ranked after the base set, from the raw scores
      uint32_t elig = 0u;
      uint64_t kk[EPT];
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const int e = TPT * j + q;
        kk[j] = real && e < N ? order_key_f64(raw[j]) : 0ull;
        if (e < N && member(e)) elig |= 1u << j;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q + TPT * u >= n) {
          ex[u] = -1;
          sk[u] = 0ull;
        }
      uint64_t ak = pk;
      int ae = pe;
      const int got = group_pick_regs<TPT, EPT, U>(kk, elig, q, m, n, ex, sk, ak, ae);
      len = real ? n + min(got, max(0, cfg.limit - n)) : 0;
      if (valid) {
        bad = emit(n);
        count(n, 1);
      }
    }
    __syncthreads();
  }
  if (valid && q == 0 && bad) atomicMin(&s_err, i);
  // this CTA's loads, total load and first degenerate token into the outputs
  // (cleared by CTA 0 before it published its words)
  __syncthreads();
  if (loads_out)
    for (int e = threadIdx.x; e < N; e += blockDim.x)
      if (s_loads[e]) atomicAdd(&loads_out[e], s_loads[e]);
  if (threadIdx.x == 0) {
    if (total_load && s_total)
      atomicAdd(reinterpret_cast<unsigned long long*>(total_load), static_cast<unsigned long long>(s_total));
    if (s_err != INT_MAX) atomicMin(err_token, s_err);
  }
  stamp(5);
}

}  // namespace oea_dev

namespace oea_host {

using namespace oea_dev;

template <int E>
static void launch_rank(const Cfg& cfg, int B, int N, const RouteBuffers& rb, int order_given,
                        int run_phase1, const int32_t* seg, cudaStream_t s) {
  const int grid = (B + kRouteWarps - 1) / kRouteWarps;
  k_rank_phase1<E><<<grid, kRouteWarps * 32, 0, s>>>(cfg, B, N, rb.scores, rb.mask, rb.order,
                                                     rb.t, rb.n, rb.union_bits, order_given,
                                                     run_phase1, seg);
}

// R > 1: batched independent records (see route_f64_fast_launch).
int route_f64_launch(oea_ctx* ctx, const Cfg& cfg, int B, int N, const RouteBuffers& rb,
                     bool order_given, bool run_phase1, int set_mode, bool n_given,
                     cudaStream_t s, int R, const int32_t* seg) {
  const int words = (N + 31) / 32;
  const int32_t* sg = R > 1 ? seg : nullptr;
  if (!n_given) OEA_CUDA_TRY(ctx, cudaMemsetAsync(rb.union_bits, 0, sizeof(uint32_t) * words * R, s));
  OEA_CUDA_TRY(ctx, cudaMemsetAsync(rb.loads, 0, sizeof(int32_t) * N * R, s));
  OEA_CUDA_TRY(ctx, cudaMemsetAsync(rb.total_load, 0, sizeof(int64_t) * R, s));
  OEA_CUDA_TRY(ctx, cudaMemsetAsync(rb.err_token, 0x7f, sizeof(int32_t), s));

  if (!n_given) {
    const int Np = round_up(N, 32);
    const int need_phase1 = run_phase1 ? 1 : 0;
    if (Np <= 32)
      launch_rank<1>(cfg, B, N, rb, order_given, need_phase1, sg, s);
    else if (Np <= 64)
      launch_rank<2>(cfg, B, N, rb, order_given, need_phase1, sg, s);
    else if (Np <= 128)
      launch_rank<4>(cfg, B, N, rb, order_given, need_phase1, sg, s);
    else if (Np <= 256)
      launch_rank<8>(cfg, B, N, rb, order_given, need_phase1, sg, s);
    else if (Np <= 512)
      launch_rank<16>(cfg, B, N, rb, order_given, need_phase1, sg, s);
    else
      launch_rank<32>(cfg, B, N, rb, order_given, need_phase1, sg, s);
    OEA_LAUNCHED(ctx);
  }
  // Set construction: 0 vanilla (route_topk), 1 pruned (baseline), 2 piggyback.
  const int do_weights = (rb.weights != nullptr || rb.weights_f32 != nullptr) ? 1 : 0;
  const int grid = (B + kRouteWarps - 1) / kRouteWarps;
  k_build_sets<<<grid, kRouteWarps * 32, 0, s>>>(
      cfg, B, N, set_mode, do_weights, rb.scores, rb.mask, rb.order, rb.n, rb.union_bits,
      rb.sets, rb.set_len, rb.weights, rb.weights_f32, rb.loads,
      reinterpret_cast<unsigned long long*>(rb.total_load), rb.err_token, sg);
  OEA_LAUNCHED(ctx);
  k_aggregate<<<R, 1024, 0, s>>>(N, rb.loads, rb.active_union, rb.active_count, rb.union_bits,
                                 rb.base_union, rb.base_union_count, nullptr);
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

// Launch as a programmatic dependent of the previous kernel in the stream
// (PDL): its launch and prologue overlap the predecessor's tail; the kernel
// calls griddepcontrol.wait before it reads the predecessor's results.
template <typename... Params, typename... Args>
static cudaError_t launch_pdl(void (*kern)(Params...), int grid, int block, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(grid);
  c.blockDim = dim3(block);
  c.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = a;
  c.numAttrs = 1;
  return cudaLaunchKernelEx(&c, kern, static_cast<Params>(args)...);
}

template <int E>
static cudaError_t launch_fast(const Cfg& cfg, int B, int N, const RouteBuffers& rb, int set_mode,
                               int do_weights, const int32_t* seg, cudaStream_t s) {
  const int grid = (B + kRouteWarps - 1) / kRouteWarps;
  k_fast_p1<E><<<grid, kRouteWarps * 32, 0, s>>>(cfg, B, N, set_mode, do_weights, rb.scores,
                                                 rb.mask, rb.sets, rb.set_len, rb.t, rb.n,
                                                 rb.union_bits, rb.weights, rb.weights_f32,
                                                 rb.loads, rb.err_token, seg);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && set_mode == 2)
    e = launch_pdl(k_fast_p2<E>, grid, kRouteWarps * 32, s, cfg, B, N, do_weights, rb.scores,
                   rb.mask, rb.n, rb.union_bits, rb.sets, rb.set_len, rb.weights, rb.weights_f32,
                   rb.loads, rb.err_token, seg);
  return e;
}

bool route_fast_ok(const Cfg& cfg, int N, bool need_order) {
  // (sets of <= 32 so the set's scores fit one lane each)
  return !need_order && cfg.p == 1.0 && cfg.max_p >= N && N <= 128 && cfg.k <= 32 &&
         cfg.limit <= 32;
}

// The single-launch route if its grid fits co-resident (cooperative launch):
// OEA_OK / an error, or -1 when it does not fit (the caller falls back).
template <int TPT, int BT, bool KEYPICK = false>
static int launch_group_route(oea_ctx* ctx, const Cfg& cfg, int B, int N, const RouteBuffers& rb,
                              int set_mode, cudaStream_t s) {
  const int grid = (B + BT / TPT - 1) / (BT / TPT);
  static int max_blocks = -1;
  if (max_blocks < 0) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_group_route<TPT, BT, KEYPICK>, BT, 0);
    max_blocks = per_sm * ctx->num_sms;
  }
  if (grid > max_blocks || grid > kRouteMaxCtas) return -1;
  // (OEA_ROUTE_PDL=1: launched as a programmatic dependent; measured slower
  // back to back, 15.8 -> 21.2 us: the next grid's CTAs sit on the SMs)
  static const bool route_pdl = getenv("OEA_ROUTE_PDL") != nullptr && atoi(getenv("OEA_ROUTE_PDL")) != 0;
  const int do_weights = (rb.weights != nullptr || rb.weights_f32 != nullptr) ? 1 : 0;
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(grid);
  c.blockDim = dim3(BT);
  c.stream = s;
  cudaLaunchAttribute a[2];
  a[0].id = cudaLaunchAttributeCooperative;
  a[0].val.cooperative = 1;
  a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[1].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = a;
  c.numAttrs = route_pdl ? 2 : 1;
  OEA_CUDA_TRY(ctx, cudaLaunchKernelEx(&c, k_group_route<TPT, BT, KEYPICK>, cfg, B, N, set_mode, do_weights,
                                       rb.scores, rb.mask, rb.sets, rb.set_len, rb.t, rb.n,
                                       rb.weights, rb.weights_f32,
                                       static_cast<RouteScratch*>(ctx->route_scratch), rb.loads,
                                       rb.active_union, rb.active_count, rb.total_load,
                                       rb.base_union, rb.base_union_count, rb.union_bits,
                                       rb.err_token, ctx->ffn_trace));
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

// R > 1: batched independent records (route_f64_batched); seg[i] = record of
// row i, and union_bits / loads / active_union / active_count / total_load /
// base_union / base_union_count are per record ([R][4] words, [R][N], [R]).
int route_f64_fast_launch(oea_ctx* ctx, const Cfg& cfg, int B, int N, const RouteBuffers& rb,
                          int set_mode, cudaStream_t s, int R, const int32_t* seg) {
  const int words = ((N + 31) / 32) * R;
  const int32_t* sg = R > 1 ? seg : nullptr;
  cudaError_t e;
  static const int fused = getenv("OEA_ROUTE_FUSED") ? atoi(getenv("OEA_ROUTE_FUSED")) : 1;
  if (fused && R == 1 && N <= 128 && ctx->route_scratch != nullptr) {
    // one cooperative launch (phase 1, union exchange, phase 2, exports):
    // 16 threads per token, 28 tokens per CTA (B = 4096: 147 CTAs, one per
    // SM; 16 per CTA put 2 CTAs on most SMs and 3 on some: stragglers),
    // key-only pick reductions (C5 10.0 us vs 10.3 us with (key, index))
    const int rc = launch_group_route<16, 448, true>(ctx, cfg, B, N, rb, set_mode, s);
    if (rc >= 0) return rc;
  }
  OEA_CUDA_TRY(ctx, cudaMemsetAsync(rb.union_bits, 0, words * 4, s));
  OEA_CUDA_TRY(ctx, cudaMemsetAsync(rb.loads, 0, sizeof(int32_t) * N * R, s));
  OEA_CUDA_TRY(ctx, cudaMemsetAsync(rb.err_token, 0x7f, sizeof(int32_t), s));
  const int do_weights = (rb.weights != nullptr || rb.weights_f32 != nullptr) ? 1 : 0;
  if (N <= 32)
    e = launch_fast<1>(cfg, B, N, rb, set_mode, do_weights, sg, s);
  else if (N <= 64)
    e = launch_fast<2>(cfg, B, N, rb, set_mode, do_weights, sg, s);
  else
    e = launch_fast<4>(cfg, B, N, rb, set_mode, do_weights, sg, s);
  OEA_CUDA_TRY(ctx, e);
  OEA_LAUNCHED(ctx);
  if (set_mode == 2) OEA_LAUNCHED(ctx);
  OEA_CUDA_TRY(ctx, launch_pdl(k_aggregate, R, N <= 128 ? 128 : 1024, s, N, rb.loads,
                               rb.active_union, rb.active_count, rb.union_bits, rb.base_union,
                               rb.base_union_count, rb.total_load));
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

int union_from_list_launch(oea_ctx* ctx, const int32_t* list, int count, int N, uint32_t* bits,
                           cudaStream_t s) {
  OEA_CUDA_TRY(ctx, cudaMemsetAsync(bits, 0, ((N + 31) / 32) * 4, s));
  if (count > 0) {
    k_union_from_list<<<1, 256, 0, s>>>(list, count, N, bits);
    OEA_LAUNCHED(ctx);
  }
  return OEA_OK;
}

}  // namespace oea_host
