// layout.cuh — index maps of the fragment-ordered bf16 weight layout
// (DESIGN.md §2), shared by the upload / init kernels (layer.cu) and the
// CM repack of the tensor-core path (umma_ffn.cu).
#pragma once
#include "oea_device.cuh"
#include "oea_internal.cuh"

namespace oea_dev {

// Fragment-layout index (bf16 elements) of logical elements.
__device__ __forceinline__ size_t router_frag_idx(int d, int n, int Dp) {
  const int rb = n >> 4, r = n & 15, kt = d >> 4, c = d & 15;
  return (static_cast<size_t>(rb) * (Dp >> 4) + kt) * 256 + frag_offset(r, c);
}
// Expert tiles are stored round-interleaved: a round = 8 consecutive row
// blocks (one per FFN consumer warp); inside a round the k-tiles are ordered
// [stage][warp][k-tile within the stage's slot], so every pipeline stage of a
// round is one contiguous kStageBytes block (a single TMA bulk copy).
__device__ __forceinline__ size_t round_tile(int rb, int kt, int KT) {
  const int rr = rb / kFfnWarps, w = rb % kFfnWarps;
  const int s = kt / kKtPerSlot, j = kt % kKtPerSlot;
  const int S = KT / kKtPerSlot;
  return ((static_cast<size_t>(rr) * S + s) * kFfnWarps + w) * kKtPerSlot + j;
}
// Expert K permutation: inside every 128-wide K slice (one FFN pipeline
// stage) k-tile j's fragment columns {2q, 2q+1, 2q+8, 2q+9} (the ones mma
// lane quad q holds) carry k = 32q + 4j + {0, 1, 2, 3}. The contraction is
// unchanged (A and B see the same order) and a lane's B operand for a whole
// stage becomes one contiguous 64-byte run of the token row.
__device__ __forceinline__ void kperm(int k, int& kt, int& c) {
  const int s = k >> 7, w = k & 127;
  const int q = w >> 5, j = (w >> 2) & 7, e = w & 3;
  kt = s * 8 + j;
  c = 2 * q + (e & 1) + ((e >> 1) << 3);
}
__device__ __forceinline__ size_t w1_frag_idx(int d, int h, int up, int Dp) {
  const int rb = h >> 3, r = (h & 7) + (up ? 8 : 0);
  int kt, c;
  kperm(d, kt, c);
  return round_tile(rb, kt, Dp >> 4) * 256 + frag_offset(r, c);
}
__device__ __forceinline__ size_t w2_frag_idx(int h, int d, int Hp) {
  const int rb = d >> 4, r = d & 15;
  int kt, c;
  kperm(h, kt, c);
  return round_tile(rb, kt, Hp >> 4) * 256 + frag_offset(r, c);
}

// (names used by umma_ffn.cu)
__device__ __forceinline__ size_t w1_frag_index(int d, int h, int up, int Dp) {
  return w1_frag_idx(d, h, up, Dp);
}
__device__ __forceinline__ size_t w2_frag_index(int h, int d, int Hp) { return w2_frag_idx(h, d, Hp); }

}  // namespace oea_dev
