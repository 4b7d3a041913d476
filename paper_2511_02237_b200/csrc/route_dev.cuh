// route_dev.cuh — warp-level ranking primitives shared by the fused router
// (router_fused.cu) and the in-kernel routing of the FFN (expert_ffn.cu).
//
// The reference orders experts by (score desc, index asc) (routing.cpp:
// 196-199). On the fused bf16 path the router output is fp32 logits, and
// softmax is monotone, so the order is (logit desc, index asc). Lane l owns
// experts j*32 + l (j < E) with their order keys in registers; a selection of
// the best remaining element costs two redux.sync.max (high word = order key
// of the logit, low word = 0xFFFF - index).
#pragma once

#include <stdint.h>

#include "oea_device.cuh"

namespace oea_dev {

__device__ __forceinline__ uint32_t order_key32(float v) {
  const uint32_t b = __float_as_uint(v == 0.0f ? 0.0f : v);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key32_to_logit(uint32_t u) {
  return __uint_as_float((u >> 31) ? (u & 0x7fffffffu) : ~u);
}

// Per-token ranking, register resident: lane l owns experts j*32 + l
// (j < E) and their order keys (0 = padding / taken). The composite order of
// routing.cpp:196-199 is (logit desc, index asc); a selection returns the best
// remaining element with two redux.sync.max (high word = order key of the
// logit, low word = 0xFFFF - index). Everything is force-inlined so the kernel
// parameters stay in the constant bank and nothing spills to local memory
// (the CTA's large shared-memory carve-out leaves little L1 for a stack).
template <int E>
struct TokRank {
  uint32_t key[E];  // order keys (0 = no element)
  uint32_t taken;   // bit j: expert j*32 + lane selected
};

// Keys of one token from its logits row (shared memory), N experts.
template <int E>
__device__ __forceinline__ void tok_load(int N, const float* lrow, TokRank<E>& R) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int p = j * 32 + lane;
    R.key[j] = p < N ? order_key32(lrow[p]) : 0u;
  }
  R.taken = 0u;
}

// Best remaining element (optionally restricted to the union bitmap `u`).
template <int E>
__device__ __forceinline__ int tok_select(const TokRank<E>& R, bool union_only, const uint32_t* u,
                                          uint32_t& key_out) {
  const int lane = threadIdx.x & 31;
  uint32_t hi = 0, lo = 0;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int e = j * 32 + lane;
    const bool ok = R.key[j] != 0u && !((R.taken >> j) & 1u) &&
                    (!union_only || ((u[e >> 5] >> (e & 31)) & 1u));
    const uint32_t l2 = 0xFFFFu - static_cast<uint32_t>(e);
    if (ok && (R.key[j] > hi || (R.key[j] == hi && l2 > lo))) {
      hi = R.key[j];
      lo = l2;
    }
  }
  const uint32_t whi = __reduce_max_sync(kFull, hi);
  if (whi == 0u) return -1;
  const uint32_t wlo = __reduce_max_sync(kFull, hi == whi ? lo : 0u);
  key_out = whi;
  return static_cast<int>(0xFFFFu - wlo);
}

template <int E>
__device__ __forceinline__ void tok_take(TokRank<E>& R, int id) {
  if ((id & 31) == (threadIdx.x & 31)) R.taken |= 1u << (id >> 5);
}

// Rank of element (key, id) in the full order (# elements before it).
template <int E>
__device__ __forceinline__ int tok_rank_of(const TokRank<E>& R, uint32_t key, int id) {
  const int lane = threadIdx.x & 31;
  int c = 0;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int e = j * 32 + lane;
    c += __popc(__ballot_sync(kFull, R.key[j] != 0u && (R.key[j] > key || (R.key[j] == key && e < id))));
  }
  return c;
}


}  // namespace oea_dev
