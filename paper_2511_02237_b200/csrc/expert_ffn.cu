// expert_ffn.cu — K4/K5: the grouped SwiGLU expert FFN over the batch's
// active experts, fused with the weighted combine.
//
// Reference semantics: expert_forward (moe_layer.hpp:92-107)
//   h = silu(x Wg) * (x Wu);  y = h Wd
// and the Eq.-1 mixture of moe_forward (moe_layer.hpp:148-155)
//   out[t] = sum_j w[t][j] * y_{S_t[j]}(x_t)   (set order)
// The reference re-reads an expert's weights for every (token, expert) pair;
// here every active expert's weights are streamed from HBM exactly once per
// token group (<= 64 tokens), which is the point of OEA.
//
// k_ffn_bf16 (persistent, one CTA per SM, 8 consumer warps + 1 producer warp)
//   work unit  = one 16-row A block of one expert and one token group:
//                W1 unit: 8 gate + 8 up rows (h = 8rb..8rb+7) x K=Dp
//                W2 unit: 16 down rows (d = 16rb..16rb+15) x K=Hp
//   global order: all W1 units (expert-major) then all W2 units; each CTA
//   owns a contiguous, byte-balanced range and processes it in rounds of up to
//   8 units, one per consumer warp, so no cross-warp reduction is needed.
//   producer  : one lane issues cp.async.bulk (TMA bulk copies, L2
//               evict_first) of 4 KiB slots into a 6-stage x 32 KiB smem ring
//               with mbarrier complete_tx; it runs ahead across unit and
//               W1/W2 boundaries (W2 weights do not depend on h).
//   consumers : per k-tile one LDS.128 A fragment + per 8-token n-block two
//               32-bit B fragment loads + one mma.sync.m16n8k16 (bf16 in,
//               fp32 accumulate). Tokens are the mma N dimension (swap-AB),
//               so a 1-3 token expert pads to 8, not 16.
//   W1 epilogue: h = silu(g) * u -> bf16 hbuf, then a release counter per
//               token group. W2 units acquire-wait on that counter (units of
//               the same group were issued earlier in global order, so the
//               wait cannot deadlock), write y per (token, slot) to ybuf, and
//               the last W2 unit of each 16-column block (arrival counter)
//               performs the deterministic slot-ordered combine for it.
// k_ffn_simt<T> (f32 / f64 layers, drop-in moe_forward<float/double>)
//   plain FMA kernels over the same compaction (rows/groups) metadata.
#include <climits>

#include "oea_device.cuh"
#include "oea_internal.cuh"
#include "route_dev.cuh"

#ifndef P_NA_MAXNB
#define P_NA_MAXNB 2
#endif

namespace oea_dev {

// 8 consumer warps, 1 producer warp (lane 0 streams weights), 1 router warp
// (fused dense path: this CTA's token's phase 2 while the weights stream).
constexpr int kProducerWarp = kFfnWarps;
constexpr int kRouterWarp = kFfnWarps + 1;
constexpr int kFfnThreads = (kFfnWarps + 2) * 32;

struct FfnParams {
  const uint4* w1;
  const uint4* w2;
  const __nv_bfloat16* xpad;  // [B][Dp]
  int D, Dp, Hp, B, stride;
  const int32_t* row_tok;
  const int32_t* row_slot;
  const int32_t* group_a;
  const int32_t* group_row0;
  const int32_t* group_rows;
  const FfnHeader* hdr;
  int* w1_done;  // [max_groups]
  // dense path: W1 release counts per group as 8 byte-wide K-slot fields of
  // one 64-bit word [max_groups] (a slot = the h columns of ceil(Hp/128 / 8)
  // W2 K slices): one release RMW per W1 unit, one acquire per W2 round
  unsigned long long* w1_slots;
  unsigned long long w1_full;  // the count word of a group whose W1 is complete
  int* claims;   // grid counters after w1_done (fixed offset, see the kernel)
  __nv_bfloat16* hbuf;  // [rows][Hp]
  float* ybuf;          // [B][stride][Dp]
  const int32_t* set_len;
  const float* wts;     // [B][stride]
  float* out;           // [B][D]
  unsigned long long* trace;  // debug: [gridDim][8] globaltimer stamps, or null
  int mode;                   // debug: 1 = stream weights only (no math)
  // Fused single-launch decode (k_ffn_bf16<1|2>, see fused_gemv /
  // rank_phase1/2). Dense path (<2>, B <= 16): W1 computes h for ALL
  // tokens of the batch, so it needs only the union (phase 1); the token lists
  // (phase 2) are needed only from the first W2 round on.
  int xs_row;                   // bytes per token row of the shared-memory x tile
  int split_ok;                 // split rounds allowed (OEA_SPLIT=1; off by default)
  int e_begin, e_count;         // experts this (possibly EP-shard) layer holds
  // Epoch-tagged exchange words (fused path): logits [B][Np], per-token base
  // bitmaps [B][4], plan rows [B][1 + 2 stride] (length, then expert and weight
  // per slot); tag = launch epoch + 1.
  unsigned long long* xlog;
  unsigned long long* xuni;
  unsigned long long* xplan;
  const uint4* router_t;        // [Np][Dp/8] expert-major bf16 router
  const uint4* router_frag;     // [Np/16][Dp/16] fragment-ordered router tiles
  const __nv_bfloat16* x_in;    // [B][D] caller tokens
  __nv_bfloat16* xpad_out;      // [B][Dp], written in-kernel when D != Dp, else null
  int x_stage;                  // x_in is mapped host memory: staged into xpad_out first
  int prefetch_bytes;           // speculative L2 prefetch of every held expert's first W1 bytes
  int pf_early;                 // issue that prefetch before griddepcontrol.wait (PDL launch)
  int w2_ks;                    // dense path: W2 rounds split into w2_ks K parts (1 = whole)
  float* logits;        // [B][Np]
  const uint8_t* mask;
  int N, Np;
  Cfg cfg;
  int32_t* x_sets;
  int32_t* x_set_len;
  float* x_w32;
  double* x_w64;
  int32_t* x_loads;
  int32_t* x_active;
  int32_t* x_active_count;
  int64_t* x_total_load;
  int32_t* x_phase1_n;
  int32_t* x_base_union;
  int32_t* x_base_union_count;
  FfnHeader* x_hdr;
  // Host-buffer decode (oea_moe_decode_host): mapped host flag the last CTA
  // to finish its slice of out sets to 1 (the caller spins on it instead of
  // a stream synchronisation), or null.
  int* done_flag;
  // Expert-parallel combine over peer memory (oea_moe_decode_ep_partial): the
  // partial mixture of token t goes straight to its owner's receive buffer,
  // slot [rank][t - owner * tpr], then every CTA bumps every owner's counter.
  // (Last member: the offsets of the hot fields stay as they were.)
  const EpPeers* ep;  // null: local combine into out
  // MODE 6 (dense decode on tcgen05): the UMMA-layout expert weights
  const uint8_t* w1u;
  const uint8_t* w2u;
  size_t w1u_stride, w2u_stride;
  int r0;             // dense W1: rounds claimed round-major first
  // route-only launch: L2 prefetch of the tcgen05 FFN's first W1 bytes (the
  // active experts' UMMA-layout W1 in group order), while this launch routes
  const uint8_t* pf_w1u;
  size_t pf_w1u_stride;
  size_t pf_total;
  int pf_guess_hi, pf_guess_lo;  // W1-head prefetch of guessed-active / -inactive own experts
  float pf_tau;                  // guess: max logit > pf_tau x rms of the batch's logits
  int host_pf_guess;             // x in host memory: the guided prefetch after the GEMV too
  // Route-only launch (B > 64): the compaction in the same launch (CTA e
  // builds expert e's token groups; route_compact_dist) and, for the tcgen05
  // FFN, the token rows gathered into the CM layout (xg, xg_rg row groups)
  int compact_in_kernel;
  uint8_t* xg;
  int xg_rg;
};

// The compacted plan's tables (global from the router kernel, or this CTA's
// shared-memory copy when the FFN routes in its prologue). Kept in shared
// memory and read where needed so they do not occupy registers in the
// consumer loop (the kernel runs at its 168-register cap).
struct alignas(16) PlanRef {  // (16-byte multiple: the shared-memory tables follow it)
  const int32_t* row_tok;
  const int32_t* row_slot;
  const int32_t* group_a;
  const int32_t* group_row0;
  const int32_t* group_rows;
  const int32_t* set_len;
  const float* wts;
  uint8_t* btile;  // token-list units with >= 2 n-blocks: shared B-operand stage tiles
  int G;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// debug timeline: this launch's region of the trace buffer (16 launches deep,
// indexed by the launch epoch), set by thread 0 at kernel start
__shared__ unsigned long long* s_trace;
__device__ __forceinline__ void stamp(const FfnParams& P, int slot) {
  if (P.trace && s_trace) s_trace[blockIdx.x * 16 + slot] = gtimer();
}

struct Unit {
  int g;       // token group
  int rb;      // row block
  int row0;    // first padded row of the group
  int rows;    // real rows (tokens) in the group
  int ready;   // W2: the group's h is known complete (acquired by the producer)
  int nw;      // warps with a unit in this round (they share the B tile)
  int sb;      // first K slice (stage) of this round's part (W2 K split; else 0)
  int kp;      // K part: y plane this unit writes (W2 K split; else 0)
};

// Dense path: W2 stage s (h columns 128 s .. 128 s + 127) needs only the W1
// row blocks 16 s .. 16 s + 15 of its group, so W1 releases and W2 waits go
// per K slot instead of per group: a W2 round starts on a group's first h
// columns while later W1 rounds of the group are still streaming.
constexpr int kW1Slots = 8;
__device__ __forceinline__ int w1_slot_q(int Hp) {
  return ((Hp >> 7) + kW1Slots - 1) / kW1Slots;
}

// Shared B-operand tiles (token-list units with >= 2 n-blocks): the 8 units
// of a round are 8 row blocks of ONE expert, so they multiply the same token
// rows. Instead of every warp loading those rows from L2 per stage (8x the
// L2 traffic: ~13 TB/s of L2 reads at B=256, the bound of that path), the
// round's warps cp.async each stage's [rows][128-wide K slice] tile once into
// shared memory, 2 stages ahead (3 buffers, one named barrier per stage).
// Layout: row r at r * 256 B; 16-byte chunk c stored at c ^ (c[3] << 1) ^ r[0]
// so the 8 lanes of an LDS.128 phase (2 rows x 4 quads) hit 8 bank groups.
constexpr int kBTileRows = 64;                   // 8 n-blocks
constexpr int kBTileBuf = kBTileRows * 256;      // one stage slice
constexpr int kBTileBytes = 3 * kBTileBuf;
__device__ __forceinline__ int btile_chunk(int c, int r) {
  return c ^ (((c >> 3) & 1) << 1) ^ (r & 1);
}

// Shared-memory x tile of the dense path: 16 token rows of Dp bf16, row
// stride Dp*2 + 32 bytes; inside every 256-byte K slice (one stage) the 16
// chunks of 16 bytes are placed at xs_chunk(cc) so that the 8 lanes of one
// LDS.128 phase (two token rows x four lane quads) hit 8 distinct bank groups.
__device__ __forceinline__ int xs_chunk(int cc) { return (cc & 8) | ((cc + (cc >> 3)) & 7); }

constexpr int kSplitRedBytes = kFfnWarps * 32 * 16 * 4;  // split-round reduction buffer

// Dense path (B <= 16) h layout: per group [Hp/128 K slices][16 token rows]
// [128] bf16, the 16-byte chunk c of row r stored at chunk hs_chunk(c, r).
// One K slice of a W2 round is then ONE contiguous 4 KiB block, which the
// producer bulk-copies into the stage next to the weights (no per-warp L2
// loads of the B operand, no exposed L2 latency at round starts), and the
// LDS.128 B-fragment loads of a quarter warp (2 token rows x 4 quads, chunks
// {i, 4+i, 8+i, 12+i}) hit 8 distinct bank groups.
constexpr int kHSlice = 16 * 128 * 2;  // one K slice of a group's h (4 KiB)
static_assert(kStages * kHSlice <= kSplitRedBytes, "h slices live in the split-reduction area");
__host__ __device__ __forceinline__ int hs_chunk(int c, int r) {
  return (c & 8) | ((c + 2 * (c >> 3) + (r & 1)) & 7);
}
__host__ __device__ __forceinline__ size_t hs_index(int g, int r, int hh, int Hp) {
  return static_cast<size_t>(g) * 16 * Hp + (hh >> 7) * 2048 + r * 128 +
         hs_chunk((hh & 127) >> 3, r) * 8 + (hh & 7);
}

// Split rounds (few active experts): ONE unit per round, its K slices spread
// over the 8 consumer warps (warp w takes slices w, w+8, ...), partial sums
// reduced through shared memory into warp 0, which runs the epilogue. This
// keeps all SMs streaming when T x units-per-expert is small (B <= 8).
struct SplitRed {
  float* buf;       // [8 warps][32 lanes][16] partial accumulators
  uint64_t* free;   // warp 0 has read buf (count 1)
  int* idx;         // split rounds this CTA has run (per warp copy in registers)
};

template <int NB, bool W1, bool DENSE, bool SPLIT>
__device__ __forceinline__ void consume_unit(const FfnParams& P, const PlanRef* PR,
                                             const uint8_t* ring, uint64_t* full, uint64_t* empty,
                                             int& stage, uint32_t& phase, int nst, const Unit& U,
                                             const uint8_t* xs, const SplitRed& SR, int& sidx) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int RB1 = P.Hp >> 3;
  // dense W1: B operand = all B tokens from the swizzled shared-memory x tile;
  // dense W2: token lists as usual, h rows at [group][token] (written by W1)
  constexpr bool XSM = DENSE && W1;
  constexpr bool HSM = DENSE && !W1 && !SPLIT;       // W2: h slices staged in the ring
  constexpr bool SHB = !DENSE && !SPLIT && NB >= 2;  // shared B tile

  // B-operand rows (uint4 view) for this lane's token in each n-block. The
  // weights are packed with the k-permutation of layer.cu (kperm): in every
  // 128-wide K slice (one pipeline stage) lane quad q of k-tile j covers
  // k = 32q + 4j .. 32q + 4j + 3, so the lane's B operand for a whole stage is
  // ONE contiguous 64-byte run of its token row: 4 x 16-byte loads.
  // Token rows are read through L2 only (ld.global.cg): the caller's x
  // buffers are rewritten between launches and a non-coherent (L1/texture)
  // line of a previous launch could otherwise be returned.
  const uint4* bp[NB];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    const int r = nb * 8 + g;
    bp[nb] = nullptr;
    if (SHB) {
      // (rows come from the shared tile)
    } else if (HSM) {
      // (rows come from the staged h slice: hrow_off below)
    } else if (XSM) {
      // token r; the per-quarter chunk offsets are added at the load
      bp[nb] = reinterpret_cast<const uint4*>(xs + r * P.xs_row);
    } else if (r < U.rows) {
      if (W1) {
        const int t = PR->row_tok[U.row0 + r];
        bp[nb] = reinterpret_cast<const uint4*>(P.xpad + static_cast<size_t>(t) * P.Dp) + 4 * q;
      } else {
        const int hrow = DENSE ? U.g * 16 + PR->row_tok[U.row0 + r] : U.row0 + r;
        bp[nb] = reinterpret_cast<const uint4*>(P.hbuf + static_cast<size_t>(hrow) * P.Hp) + 4 * q;
      }
    }
  }
  // HSM: byte offsets of this lane's token row (n-block nb) in an h slice;
  // rows past the group's list read row 0 (their output columns are dropped)
  int hoff[HSM ? NB : 1][4];
  if constexpr (HSM) {
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const int r = nb * 8 + g;
      const int tr = r < U.rows ? PR->row_tok[U.row0 + r] : 0;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) hoff[nb][jj] = tr * 256 + hs_chunk(4 * q + jj, tr) * 16;
    }
  }
  if (!W1 && !HSM && !U.ready) {
    // h of this token group must be complete (all RB1 W1 units released):
    // lane 0 acquires, the warp barrier orders the other lanes after it.
    // (U.ready: the producer already acquired it when it issued the round.)
    if (lane == 0)
      while (ld_acquire_gpu(&P.w1_done[U.g]) < RB1) __nanosleep(64);
    __syncwarp();
  }

  // two accumulator sets (even / odd k-tiles) halve the dependent HMMA chain
  // (one n-block: two sets halve the dependent HMMA chain; more n-blocks
  // already interleave independent chains, so they use one set)
  constexpr int NA = NB <= P_NA_MAXNB ? 2 : 1;
  float acc2[NA][NB][4];
#pragma unroll
  for (int h2 = 0; h2 < NA; ++h2)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
      acc2[h2][nb][0] = acc2[h2][nb][1] = acc2[h2][nb][2] = acc2[h2][nb][3] = 0.0f;

  auto ldb = [&](const uint4* p) -> uint4 {
    if (p == nullptr) return make_uint4(0u, 0u, 0u, 0u);
    return __ldcg(p);  // x / h rows may change between launches: L2 (coherent) only
  };
  // dense W1: byte offsets of this lane's quarter-stage chunks inside a slice
  int xoff[4];
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) xoff[jj] = xs_chunk(4 * q + jj) * 16;
  // shared B tile: this warp's slice of the round's tile loads (chunk k of
  // stage slice s: row k / 16, 16-byte chunk k % 16), one commit group each
  const bool math = P.mode != 1;
  const int nthr = U.nw * 32, ctid = warp * 32 + lane;
  auto issue_tile = [&](int s, int buf) {
    uint8_t* dst0 = PR->btile + buf * kBTileBuf;
    for (int k = ctid; k < U.rows * 16; k += nthr) {
      const int r = k >> 4, c = k & 15;
      const __nv_bfloat16* row =
          W1 ? P.xpad + static_cast<size_t>(PR->row_tok[U.row0 + r]) * P.Dp
             : P.hbuf + static_cast<size_t>(U.row0 + r) * P.Hp;
      cp_async16(smem_u32(dst0 + r * 256 + btile_chunk(c, r) * 16),
                 reinterpret_cast<const uint8_t*>(row) + s * 256 + c * 16, 16);
    }
    cp_async_commit();
  };
  int boff[4];  // this lane's chunk offsets (row g of an n-block; n-block nb adds nb * 2 KiB)
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) boff[jj] = g * 256 + btile_chunk(4 * q + jj, g) * 16;
  if (SHB && math) {
    issue_tile(0, 0);
    if (nst > 1) issue_tile(1, 1);
  }
  // One n-block (global B): the next stage's 4 loads are issued right after
  // the current stage is consumed, so their latency hides behind the stage
  // barrier wait (two n-blocks measured slower: spills at the register cap).
  // More n-blocks: per quarter stage (2 k-tiles) one 16-byte load per n-block.
  constexpr bool kPref = !XSM && !HSM && NB <= 1 && !SPLIT;
  constexpr int PB = 1;  // prefetched n-blocks
  // slices of this unit (K / 128); SPLIT: this warp's slice of split-stage s
  const int nslices = (W1 ? P.Dp : P.Hp) >> 7;
  uint4 bpre[PB][4];
  if (kPref && math)
#pragma unroll
    for (int nb = 0; nb < PB; ++nb)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        bpre[nb][i] = ldb(bp[nb] == nullptr ? nullptr : bp[nb] + U.sb * 16 + i);

  for (int s0 = 0; s0 < nst; ++s0) {
    if (SHB && math) {
      // tile s0 landed for every warp of the round (and every warp is past
      // stage s0 - 1, so buffer (s0 + 2) % 3 is free for the prefetch)
      if (s0 + 1 < nst)
        cp_async_wait_group<1>();
      else
        cp_async_wait_group<0>();
      asm volatile("bar.sync 5, %0;" ::"r"(nthr) : "memory");
      if (s0 + 2 < nst) issue_tile(s0 + 2, (s0 + 2) % 3);
    }
    mbar_wait(&full[stage], phase);
    const int s = SPLIT ? s0 * kFfnWarps + warp : U.sb + s0;  // K slice of this stage for this warp
    const uint4* tiles =
        reinterpret_cast<const uint4*>(ring + stage * kStageBytes + warp * kSlotBytes);
    if (math && (!SPLIT || s < nslices)) {
      if (kPref) {
#pragma unroll
        for (int j = 0; j < kKtPerSlot; ++j) {
          const uint4 a = tiles[j * 32 + lane];
#pragma unroll
          for (int nb = 0; nb < PB; ++nb) {
            const uint4& v = bpre[nb][j >> 1];
            mma_bf16_16816(acc2[(j & 1) % NA][nb], a, (j & 1) ? v.z : v.x, (j & 1) ? v.w : v.y);
          }
        }
        if (s0 + 1 < nst)
#pragma unroll
          for (int nb = 0; nb < PB; ++nb)
#pragma unroll
            for (int i = 0; i < 4; ++i)
              bpre[nb][i] = ldb(bp[nb] == nullptr ? nullptr : bp[nb] + (s + 1) * 16 + i);
      } else {
#pragma unroll
        for (int jj = 0; jj < kKtPerSlot / 2; ++jj) {
          uint4 v[NB];
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            if (P.mode == 2)  // (debug: no B-operand loads)
              v[nb] = make_uint4(0u, 0u, 0u, 0u);
            else if (SHB)
              v[nb] = lds128(PR->btile + (s0 % 3) * kBTileBuf + nb * 2048 + boff[jj]);
            else if (XSM)
              v[nb] = lds128(reinterpret_cast<const uint8_t*>(bp[nb]) + s * 256 + xoff[jj]);
            else if (HSM)
              v[nb] = lds128(reinterpret_cast<const uint8_t*>(SR.buf) + stage * kHSlice +
                             hoff[HSM ? nb : 0][jj]);
            else
              v[nb] = ldb(bp[nb] == nullptr ? nullptr : bp[nb] + s * 16 + jj);
          }
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const uint4 a = tiles[(2 * jj + h2) * 32 + lane];
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
              mma_bf16_16816(acc2[h2 % NA][nb], a, h2 ? v[nb].z : v[nb].x, h2 ? v[nb].w : v[nb].y);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1u;
    }
  }

  float acc[NB][4];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[nb][i] = NA == 2 ? acc2[0][nb][i] + acc2[1][nb][i] : acc2[0][nb][i];

  if constexpr (SPLIT) {
    // deterministic cross-warp reduction (warp order 0..7) into warp 0
    static_assert(NB * 4 <= 16, "split rounds keep <= 2 n-blocks");
    if (sidx > 0) mbar_wait(SR.free, (sidx - 1) & 1);  // warp 0 read the previous buffer
    ++sidx;
    float* mine = SR.buf + (warp * 32 + lane) * 16;
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int i = 0; i < 4; ++i) mine[nb * 4 + i] = acc[nb][i];
    asm volatile("bar.sync 1, %0;" ::"r"(kFfnWarps * 32) : "memory");
    if (warp != 0) return;
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float v = 0.0f;
#pragma unroll
        for (int w = 0; w < kFfnWarps; ++w) v += SR.buf[(w * 32 + lane) * 16 + nb * 4 + i];
        acc[nb][i] = v;
      }
    __syncwarp();
    if (lane == 0) mbar_arrive(SR.free);
  }

  if (W1) {
    // Thread (g, q) holds gate[h][tok 2q, 2q+1] (c0, c1) and up[h][...] (c2, c3)
    // for h = 8 rb + g.
    const int h = U.rb * 8 + g;
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r = nb * 8 + 2 * q + i;
        if (r < U.rows) {
          const float hv = silu_f(acc[nb][i]) * acc[nb][2 + i];
          const size_t hi = DENSE ? hs_index(U.g, r, h, P.Hp)
                                  : static_cast<size_t>(U.row0 + r) * P.Hp + h;
          P.hbuf[hi] = __float2bfloat16_rn(hv);
        }
      }
    }
    // release: the warp barrier orders the lanes' h stores before lane 0's
    // gpu-scope release increment (cumulative; no full fence, no L1 flush)
    __syncwarp();
    if (lane == 0) {
      if (DENSE)
        red_release_gpu_add_u64(&P.w1_slots[U.g], 1ull << (8 * ((U.rb >> 4) / w1_slot_q(P.Hp))));
      else
        red_release_gpu_add(&P.w1_done[U.g], 1);
    }
  } else {
    const int d0 = U.rb * 16;
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r = nb * 8 + 2 * q + i;
        if (r < U.rows) {
          const int row = U.row0 + r;
          const int t = PR->row_tok[row], sl = PR->row_slot[row];
          float* y = P.ybuf +
                     (static_cast<size_t>(U.kp * P.B + t) * P.stride + sl) * P.Dp + d0;
          y[g] = acc[nb][i];
          y[g + 8] = acc[nb][2 + i];
        }
      }
    }
    // y is combined by the grid-wide pass at the end of the kernel.
  }
}

// Idle warp in a short round: keeps the stage barrier protocol in step.
__device__ __forceinline__ void skip_unit(uint64_t* full, uint64_t* empty, int& stage,
                                          uint32_t& phase, int nst) {
  const int lane = threadIdx.x & 31;
  for (int s = 0; s < nst; ++s) {
    mbar_wait(&full[stage], phase);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1u;
    }
  }
}

#define OEA_CU(NB_, W1_, DN_, SP_) \
  consume_unit<NB_, W1_, DN_, SP_>(P, PR, ring, full, empty, stage, phase, nst, U, xs, SR, sidx)
template <bool W1, bool DENSE>
__device__ __forceinline__ void dispatch_unit(int nbk, const FfnParams& P, const PlanRef* PR,
                                              const uint8_t* ring, uint64_t* full, uint64_t* empty,
                                              int& stage, uint32_t& phase, int nst, const Unit& U,
                                              const uint8_t* xs, const SplitRed& SR, int& sidx) {
  if (DENSE) {  // B <= 16: at most two n-blocks
    if (nbk == 1)
      OEA_CU(1, W1, true, false);
    else
      OEA_CU(2, W1, true, false);
    return;
  }
  switch (nbk) {
    case 1: OEA_CU(1, W1, false, false); break;
    case 2: OEA_CU(2, W1, false, false); break;
    case 3: OEA_CU(3, W1, false, false); break;
    case 4: OEA_CU(4, W1, false, false); break;
    case 5:
    case 6: OEA_CU(6, W1, false, false); break;
    default: OEA_CU(8, W1, false, false); break;
  }
}

// Split round of one unit (<= 2 n-blocks; more rows never take split rounds).
template <bool W1, bool DENSE>
__device__ __forceinline__ void dispatch_split(int nbk, const FfnParams& P, const PlanRef* PR,
                                               const uint8_t* ring, uint64_t* full, uint64_t* empty,
                                               int& stage, uint32_t& phase, int nst, const Unit& U,
                                               const uint8_t* xs, const SplitRed& SR, int& sidx) {
  if (nbk == 1)
    OEA_CU(1, W1, DENSE, true);
  else
    OEA_CU(2, W1, DENSE, true);
}

// Dense path W2: token lists of the group (router warp), h rows at
// [group][token]; consume_unit<NB, false, true> (W2 ignores the x tile).
__device__ __forceinline__ void dispatch_w2_dense(int nbk, const FfnParams& P, const PlanRef* PR,
                                                  const uint8_t* ring, uint64_t* full,
                                                  uint64_t* empty, int& stage, uint32_t& phase,
                                                  int nst, const Unit& U, const uint8_t* xs,
                                                  const SplitRed& SR, int& sidx) {
  if (nbk == 1)
    OEA_CU(1, false, true, false);
  else
    OEA_CU(2, false, true, false);
}

// ---------------------------------------------------------------------------
// Fused single-launch decode (B <= 64): the FFN grid computes the router
// logits itself, exchanges them through one grid barrier, and every CTA then
// ranks the whole batch redundantly from shared memory (deterministic code on
// identical inputs -> identical plans, no plan round trip through HBM).
//
//   G  gate GEMV (router_scores, moe_layer.hpp:71-90, on bf16 weights):
//      CTA c computes the logits of experts c, c + grid, ... for every token
//      from the expert-major router copy (4 KiB per expert at D=2048) and the
//      bf16 tokens; fixed-order warp transpose-reduction + fixed warp order,
//      so logits are deterministic. Then one grid barrier.
//   R1 Phase 1 (routing.cpp:226-268) for every token (all 9 warps): the
//      baseline top-k0 (vanilla: top-k, route_topk routing.cpp:205-224) and
//      the batch union bitmap. active_union == base_union for the OEA modes
//      (conservation, acceptance.cpp:158-184), so the union IS the list of
//      expert groups: the producer warp starts streaming weights here.
//   R2 Phase 2 (routing.cpp:270-303) + fp32 renormalisation (routing.cpp:
//      33-49) + compaction (token lists in token order, inverse permutation)
//      on the 8 consumer warps, overlapped with the producer's first stages.
// ---------------------------------------------------------------------------
struct RouteSmem {
  size_t keys, ukeys, uni, sets, e, len, n, mx, loads, tokbits, active, eslot, rowb, rows, rtok,
      rslot, red, misc, lgp, thr, pe, total;
};

__host__ __device__ inline RouteSmem route_smem_layout(int B, int Np, int stride) {
  RouteSmem L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = (o + bytes + 15) & ~static_cast<size_t>(15);
    return at;
  };
  const int Bw = (B + 31) >> 5, uw = (Np + 31) >> 5;
  const int rmax = B * stride + 8 * Np;
  L.keys = take(static_cast<size_t>(Np) * 4);
  L.ukeys = take(static_cast<size_t>(Np) * 4);
  L.uni = take(uw * 4);
  L.sets = take(static_cast<size_t>(B) * stride * 4);
  L.e = take(static_cast<size_t>(B) * stride * 4);
  L.len = take(B * 4);
  L.n = take(B * 4);
  L.mx = take(B * 4);
  L.loads = take(Np * 4);
  // (also the union's [B][4] scratch)
  L.tokbits = take(static_cast<size_t>(Np * Bw * 4 > B * 16 ? Np * Bw * 4 : B * 16));
  L.active = take(Np * 4);
  L.eslot = take(Np * 4);
  L.rowb = take(Np * 4);
  L.rows = take(Np * 4);
  L.rtok = take(rmax * 4);
  L.rslot = take(rmax * 4);
  L.red = take((kFfnThreads / 32) * 16 * 4);
  L.lgp = take(64 * 4);  // this CTA's expert's logits (first 64 tokens): the prefetch guess
  L.misc = take(8 * 4);
  L.thr = take(static_cast<size_t>(B) * 8);  // max_p < N: (key, expert) at rank max_p - 1
  // p < 1: the base candidates' exp(l - max) by rank, 4 warp partials of the
  // softmax denominator, the resulting n, the phase-2 placed count
  L.pe = take(static_cast<size_t>(Np) * 8 + 4 * 8 + 16);
  L.total = o;
  return L;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

// G: logits[t][e] for this CTA's experts; also the zero-padded x copy the
// FFN's B fragments read when D is not a tile multiple. Ends with the grid
// barrier after which every CTA may read all logits (and xpad).
__device__ __forceinline__ void fused_gemv(const FfnParams& P, float* red, int* sync_cnt,
                                           uint32_t tag, float* lgp = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NT = kFfnThreads;
  const int nch = P.Dp >> 3;
  // token rows the GEMV reads: the caller's x, or (x in mapped host memory,
  // oea_moe_decode_host) the device copy staged below
  const __nv_bfloat16* xsrc = P.x_stage ? P.xpad_out : P.x_in;
  const int xrow = P.x_stage ? P.Dp : P.D;
  if (P.x_stage) {
    // zero-copy input: CTA c copies a 1/grid slice of x (16-byte chunks, one
    // host round trip, zero-padded to Dp), then a grid barrier. Reading x
    // from every CTA instead would cross the host link grid-size times.
    const int n = P.B * nch;
    const int c0 = static_cast<int>(static_cast<int64_t>(n) * blockIdx.x / gridDim.x);
    const int c1 = static_cast<int>(static_cast<int64_t>(n) * (blockIdx.x + 1) / gridDim.x);
    for (int i = c0 + tid; i < c1; i += NT) {
      const int t = i / nch, c = i % nch;
      const uint4 v = c * 8 < P.D
                          ? *reinterpret_cast<const uint4*>(P.x_in + static_cast<size_t>(t) * P.D + c * 8)
                          : make_uint4(0u, 0u, 0u, 0u);
      *reinterpret_cast<uint4*>(P.xpad_out + static_cast<size_t>(t) * P.Dp + c * 8) = v;
    }
    __syncthreads();
    if (tid == 0) {
      red_release_gpu_add(sync_cnt, 1);
      while (ld_acquire_gpu(sync_cnt) < static_cast<int>(gridDim.x)) {
      }
    }
    __syncthreads();
  } else if (P.xpad_out != nullptr) {
#pragma unroll 1
    for (int t = blockIdx.x; t < P.B; t += gridDim.x)
#pragma unroll 1
      for (int d = tid; d < P.Dp; d += NT)
        P.xpad_out[static_cast<size_t>(t) * P.Dp + d] =
            d < P.D ? P.x_in[static_cast<size_t>(t) * P.D + d] : __float2bfloat16_rn(0.0f);
  }
  if (tid == 0) stamp(P, 8);
#pragma unroll 1
  for (int e = blockIdx.x; e < P.N; e += gridDim.x) {
    const uint4* rrow = P.router_t + static_cast<size_t>(e) * nch;
#pragma unroll 1
    for (int tc = 0; tc < P.B; tc += 16) {
      float a[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) a[t] = 0.0f;
      // all 16 token chunks + the router chunk in flight before any FMA
#pragma unroll 1
      for (int c = tid; c < nch; c += NT) {
        const uint4 rv = __ldcg(rrow + c);
        uint4 xv[16];
#pragma unroll
        for (int t = 0; t < 16; ++t)
          xv[t] = (tc + t < P.B && c * 8 < P.D)
                      ? __ldcg(reinterpret_cast<const uint4*>(
                            xsrc + static_cast<size_t>(tc + t) * xrow + c * 8))
                      : make_uint4(0u, 0u, 0u, 0u);
        float rf[8];
        bf16x8_to_f32(rv, rf);
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          float xf[8];
          bf16x8_to_f32(xv[t], xf);
#pragma unroll
          for (int i = 0; i < 8; ++i) a[t] = fmaf(rf[i], xf[i], a[t]);
        }
      }
      // warp transpose-reduction: 16 values -> lane pair (2i, 2i+1) holds the
      // warp sum of value idx(lane), fixed order
#pragma unroll
      for (int off = 16, n = 16; off >= 2; off >>= 1, n >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int j = 0; j < n / 2; ++j) {
          const float send = up ? a[j] : a[j + n / 2];
          const float keep = up ? a[j + n / 2] : a[j];
          a[j] = keep + __shfl_xor_sync(kFull, send, off);
        }
      }
      a[0] += __shfl_xor_sync(kFull, a[0], 1);
      const int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                      ((lane >> 1) & 1);
      if ((lane & 1) == 0) red[warp * 16 + idx] = a[0];
      __syncthreads();
      if (tid < 16 && tc + tid < P.B) {
        float s = 0.0f;
#pragma unroll
        for (int w = 0; w < kFfnThreads / 32; ++w) s += red[w * 16 + tid];
        // the token's router CTA polls this word (no grid barrier needed)
        if (e == static_cast<int>(blockIdx.x) && lgp != nullptr && tc + tid < 64) lgp[tc + tid] = s;
        st_relaxed_u64(P.xlog + static_cast<size_t>(tc + tid) * P.Np + e,
                       tagged(tag, __float_as_uint(s)));
      }
      __syncthreads();
    }
  }
  // grid barrier only for the zero-padded x copy (D != Dp): its readers are
  // every CTA (x tile, W1); the logits travel as tagged words
  if (P.xpad_out == nullptr || P.x_stage) return;
  __syncthreads();
  if (tid == 0) {
    stamp(P, 9);
    __threadfence();
    atomicAdd(sync_cnt, 1);
    stamp(P, 10);
    while (ld_acquire_gpu(sync_cnt) < static_cast<int>(gridDim.x)) __nanosleep(32);
  }
  __syncthreads();
}

// HBM idles until the union is known: warm L2 with the first W1 stages of
// every held expert (each is active with probability ~T/N; the stream reads
// them as L2 hits, and its evict_first lines leave before these). Producer
// warp, one 32 KiB prefetch per lane.
__device__ __forceinline__ void prefetch_w1_heads(const FfnParams& P, int lane,
                                                  const float* lgp = nullptr) {
  const size_t per = static_cast<size_t>(P.Hp >> 3) * (P.Dp >> 4) * 512;  // W1 bytes per expert
  size_t want = static_cast<size_t>(P.prefetch_bytes);
  const int nt = min(P.B, 64);
  if (lgp != nullptr && P.pf_guess_hi > 0 && nt >= 4) {
    // Guess from this CTA's own expert's logits (known right after its GEMV,
    // no exchange): a base-set member ranks in some token's top k0 of N, so
    // its largest logit over the batch sits far above this expert's mean
    // (C1: ~2 standard deviations for a top-4 of 128). Likely-active experts
    // get a deep prefetch (1.5 MiB: their first W1 rounds), the others none:
    // HBM idles during the routing prologue, and a right guess turns it into
    // stream time (C1 82.6 -> 78.7 us; a wrong one only costs traffic).
    float mx = -INFINITY, sm = 0.0f, ss = 0.0f;
    for (int t = 0; t < nt; ++t) {
      mx = fmaxf(mx, lgp[t]);
      sm += lgp[t];
      ss += lgp[t] * lgp[t];
    }
    const float mean = sm / nt, sd = sqrtf(fmaxf(ss / nt - mean * mean, 0.0f));
    want = mx - mean > P.pf_tau * sd ? static_cast<size_t>(P.pf_guess_hi)
                                     : static_cast<size_t>(P.pf_guess_lo);
  }
  for (int e = blockIdx.x; e < P.e_count; e += gridDim.x) {
    const uint32_t nb = static_cast<uint32_t>(
        min(per, e == static_cast<int>(blockIdx.x) ? want : static_cast<size_t>(P.prefetch_bytes)));
    for (uint32_t o = 32u * 1024u * lane; o < nb; o += 32u * 32u * 1024u)
      bulk_prefetch_l2(reinterpret_cast<const uint8_t*>(P.w1) + e * per + o,
                       min(32u * 1024u, nb - o));
  }
}

// ---------------------------------------------------------------------------
// Token-parallel rank routing (fused path). CTA t < B routes token t with one
// thread per expert: every selection of routing.cpp is a RANK in the total
// order (logit desc, index asc; softmax is monotone, routing.cpp:196-199), so
// each thread counts the experts ordered before its own and no serial
// select chain remains.
//   R1 (routing.cpp:226-268, p == 1): the base set = ranks < n_i = k0
//      (vanilla: route_topk, ranks < k) -> union bits in global memory.
//   union barrier (the batch union is global, routing.cpp:262-266).
//   R2 (routing.cpp:270-303, max_p = N): piggyback = the union members in rank
//      order until |S| = cap; with base = the top n_i experts, S is exactly the
//      union members of union-rank < max(n_i, cap) (conservation:
//      acceptance.cpp:158-184). Weights w_j = e_j / sum_set e in set order
//      (routing.cpp:33-49, e_j = exp(l_j - l_max): the softmax denominator
//      cancels), exported as the token's plan row.
//   plan barrier; every CTA gathers the batch plan and compacts the token
//   lists of the expert groups (inverse permutation) in shared memory.
// ---------------------------------------------------------------------------
// Gate GEMV for large batches (route-only launch, B > 64): tensor-core tiles
// of 16 experts x 16 tokens (mma.m16n8k16 on the fragment-ordered router
// tiles, x rows as B), K split over the 8 consumer warps, partials reduced
// in fixed warp order; logits go out as tagged words like fused_gemv's.
__device__ __forceinline__ void tile_gemv(const FfnParams& P, float* red, uint32_t tag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, q = lane & 3;
  const int KT = P.Dp >> 4, nEb = P.Np >> 4, nTb = (P.B + 15) >> 4;
#pragma unroll 1
  for (int item = blockIdx.x; item < nEb * nTb; item += gridDim.x) {
    const int eb = item % nEb, tb = item / nEb;
    if (warp < kFfnWarps) {
      float acc[2][4];
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) acc[nb][0] = acc[nb][1] = acc[nb][2] = acc[nb][3] = 0.0f;
      const int kt0 = warp * KT / kFfnWarps, kt1 = (warp + 1) * KT / kFfnWarps;
      // (route-only launches have D == Dp; tokens past B read row B-1 and
      // their logits are dropped below: no branches around the loads, so a
      // warp's loads for up to 16 k-tiles are all in flight at once)
      const uint32_t* xr[2];
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
        xr[nb] = reinterpret_cast<const uint32_t*>(
            P.x_in + static_cast<size_t>(min(tb * 16 + nb * 8 + gq, P.B - 1)) * P.D);
      const uint4* arow = P.router_frag + static_cast<size_t>(eb) * KT * 32 + lane;
#pragma unroll 1
      for (int k0 = kt0; k0 < kt1; k0 += 16) {
        uint4 a[16];
        uint32_t b[16][2][2];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int kt = min(k0 + i, kt1 - 1);
          a[i] = __ldg(arow + static_cast<size_t>(kt) * 32);
          const int kw = (kt * 16 + 2 * q) >> 1;
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) {
            b[i][nb][0] = __ldg(xr[nb] + kw);
            b[i][nb][1] = __ldg(xr[nb] + kw + 4);
          }
        }
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (k0 + i < kt1)
#pragma unroll
            for (int nb = 0; nb < 2; ++nb) mma_bf16_16816(acc[nb], a[i], b[i][nb][0], b[i][nb][1]);
      }
      if (threadIdx.x == 0) stamp(P, 9);
      float* mine = red + (warp * 32 + lane) * 8;
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int i = 0; i < 4; ++i) mine[nb * 4 + i] = acc[nb][i];
    }
    __syncthreads();
    if (threadIdx.x == 0) stamp(P, 10);
    if (warp == 0) {
      // lane (gq, q): experts 16eb + gq (+8), tokens 16tb + 8nb + 2q (+1)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float v = 0.0f;
#pragma unroll
          for (int w = 0; w < kFfnWarps; ++w) v += red[(w * 32 + lane) * 8 + nb * 4 + i];
          const int e = eb * 16 + gq + (i >= 2 ? 8 : 0);
          const int t = tb * 16 + nb * 8 + 2 * q + (i & 1);
          if (e < P.N && t < P.B)
            st_relaxed_u64(P.xlog + static_cast<size_t>(t) * P.Np + e, tagged(tag, __float_as_uint(v)));
        }
    }
    __syncthreads();
  }
}

// R1 for token t on warps 0..3 (thread e <-> expert e, Np <= 128).
__device__ __forceinline__ void rank_phase1(const FfnParams& P, int t, uint8_t* rs,
                                            const RouteSmem& L, uint32_t tag) {
  const int e = threadIdx.x;  // < 128
  const int N = P.N, stride = P.cfg.stride;
  uint32_t* keys = reinterpret_cast<uint32_t*>(rs + L.keys);
  float* mx = reinterpret_cast<float*>(rs + L.mx);
  int* sets = reinterpret_cast<int*>(rs + L.sets) + t * stride;
  float* se = reinterpret_cast<float*>(rs + L.e) + t * stride;
  const bool masked = P.mask != nullptr && P.mask[t] == 0;
  float l = 0.0f;
  if (e < N) {  // expert e's CTA publishes logit (t, e) as a tagged word
    const unsigned long long* w = P.xlog + static_cast<size_t>(t) * P.Np + e;
    unsigned long long v = ld_relaxed_u64(w);
    while (static_cast<uint32_t>(v >> 32) != tag) {
      __nanosleep(20);
      v = ld_relaxed_u64(w);
    }
    l = __uint_as_float(static_cast<uint32_t>(v));
    P.logits[static_cast<size_t>(t) * P.Np + e] = l;  // exported plan: logits
  }
  const uint32_t key = e < N && !masked ? order_key32(l) : 0u;
  if (e < P.Np) keys[e] = key;  // (keys[] holds Np entries)
  if (s_trace && e == 0 && t < 16) s_trace[2368 + 2 * t] = gtimer();  // (debug: own word polled)
  asm volatile("bar.sync 3, 128;" ::: "memory");
  if (s_trace && e == 0 && t < 16) s_trace[2368 + 2 * t + 1] = gtimer();  // (debug: all polled)
  // experts ranked before e: four keys per 16-byte shared load, two
  // accumulators (the padding keys past N are 0 and never count for a real
  // key; a zero key's rank is not used)
  int r0 = 0, r1 = 0;
  const uint4* k4 = reinterpret_cast<const uint4*>(keys);
#pragma unroll 4
  for (int f4 = 0; f4 < (P.Np >> 2); ++f4) {
    const uint4 kv = k4[f4];
    const int f = 4 * f4;
    r0 += (kv.x > key) | ((kv.x == key) & (f < e));
    r1 += (kv.y > key) | ((kv.y == key) & (f + 1 < e));
    r0 += (kv.z > key) | ((kv.z == key) & (f + 2 < e));
    r1 += (kv.w > key) | ((kv.w == key) & (f + 3 < e));
  }
  const int rank = r0 + r1;
  int n = masked ? 0 : min(P.cfg.mode == OEA_MODE_VANILLA ? P.cfg.k : P.cfg.k0, N);
  if (P.cfg.mode != OEA_MODE_VANILLA && P.cfg.max_p < N && key != 0u && rank == P.cfg.max_p - 1) {
    uint32_t* thr = reinterpret_cast<uint32_t*>(rs + L.thr) + 2 * t;
    thr[0] = key;
    thr[1] = static_cast<uint32_t>(e);
  }
  if (P.cfg.mode != OEA_MODE_VANILLA && P.cfg.p < 1.0 && n > 0) {
    // mass rule (routing.cpp:243-257): t_i = the first rank whose cumulative
    // softmax mass reaches p, n = min(k0, t_i); fp64 softmax of the fp32
    // logits as the router cluster computes it (tok_phase1)
    double* pe = reinterpret_cast<double*>(rs + L.pe);
    double* zp = pe + P.Np;
    int* nn = reinterpret_cast<int*>(zp + 4);
    if (key != 0u && rank == 0) mx[t] = l;
    asm volatile("bar.sync 3, 128;" ::: "memory");
    const double ed = key != 0u ? exp(static_cast<double>(l) - static_cast<double>(mx[t])) : 0.0;
    double z = ed;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(kFull, z, off);
    if ((e & 31) == 0) zp[e >> 5] = z;
    if (key != 0u && rank < n) pe[rank] = ed;
    asm volatile("bar.sync 3, 128;" ::: "memory");
    if (e == 0) {
      const double zz = (zp[0] + zp[1]) + (zp[2] + zp[3]);
      double cum = 0.0;
      int m = n;
      for (int j = 0; j < n; ++j) {
        cum = __dadd_rn(cum, pe[j] / zz);
        if (cum >= P.cfg.p) {
          m = j + 1;
          break;
        }
      }
      *nn = m;
    }
    asm volatile("bar.sync 3, 128;" ::: "memory");
    n = *nn;
  }
  const bool base = key != 0u && rank < n;
  if (base) sets[rank] = e;
  const unsigned bw = __ballot_sync(kFull, base);  // warp w holds experts 32w..32w+31
  if ((e & 31) == 0) st_relaxed_u64(P.xuni + 4 * t + (e >> 5), tagged(tag, bw));
  if (key != 0u && rank == 0) mx[t] = l;
  asm volatile("bar.sync 3, 128;" ::: "memory");
  if (base) se[rank] = expf(l - mx[t]);
  if (e == 0) reinterpret_cast<int*>(rs + L.n)[t] = n;
}

// R2 for token t on NT threads (thread gt of the group; experts e = gt + NT*i),
// `sync` a barrier of the group. Exports the token's plan row.
template <int NT, typename Sync>
__device__ __forceinline__ void rank_phase2(const FfnParams& P, int t, uint8_t* rs,
                                            const RouteSmem& L, int T, int gt, Sync sync) {
  const int N = P.N, stride = P.cfg.stride;
  const uint32_t* uni = reinterpret_cast<const uint32_t*>(rs + L.uni);
  const float rowmax = reinterpret_cast<const float*>(rs + L.mx)[t];
  int* sets = reinterpret_cast<int*>(rs + L.sets) + t * stride;
  float* se = reinterpret_cast<float*>(rs + L.e) + t * stride;
  const bool masked = P.mask != nullptr && P.mask[t] == 0;
  const int n = reinterpret_cast<const int*>(rs + L.n)[t];
  const bool piggy = !masked && (P.cfg.mode == OEA_MODE_OEA || P.cfg.mode == OEA_MODE_SIMPLIFIED);
  const int cap = max(n, P.cfg.limit);
  // max_p < N: members ranked at or after max_p (overall) are not candidates;
  // they are a suffix of the members' rank order, so `placed` counts the rest
  const bool lim = piggy && P.cfg.max_p < N;
  const uint32_t* thr = reinterpret_cast<const uint32_t*>(rs + L.thr) + 2 * t;
  int* placed = reinterpret_cast<int*>(reinterpret_cast<double*>(rs + L.pe) + P.Np + 4) + 1;
  int len = masked ? 0 : piggy ? min(T, cap) : n;
  if (piggy) {
    // the union members' keys, compacted in ascending expert order (member i
    // is the i-th set bit): union ranks then cost T compares, not N
    uint32_t* ukeys = reinterpret_cast<uint32_t*>(rs + L.ukeys);
    if (gt == 0 && lim) *placed = 0;
    if (gt < 32) {
      const uint32_t below = lanemask_lt();
      // (published by the GEMV; keys[] is per CTA, not per token): the lane's
      // four words are loaded before any is used, one round trip instead of
      // four (the relaxed loads are ordered asm: a use between them, a shared
      // store, would serialise them)
      unsigned long long v[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int e = 32 * w + gt;
        v[w] = e < N && ((uni[w] >> gt) & 1u) ? ld_relaxed_u64(P.xlog + static_cast<size_t>(t) * P.Np + e)
                                               : 0ull;
      }
      int ub = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t uw = uni[w];
        const int e = 32 * w + gt;
        if (e < N && ((uw >> gt) & 1u))
          ukeys[ub + __popc(uw & below)] = order_key32(__uint_as_float(static_cast<uint32_t>(v[w])));
        ub += __popc(uw);
      }
    }
    sync();
    // members before member i: larger key, or equal key and lower index
    auto rank_part = [&](int i, uint32_t key, int j0, int j1) {
      int c = 0;
#pragma unroll 4
      for (int j = j0; j < j1; ++j) {
        const uint32_t kj = ukeys[j];
        c += (kj > key) | ((kj == key) & (j < i));
      }
      return c;
    };
    auto member_expert = [&](int i) {  // expert index of member i: the i-th set bit of the union
      int e = 0, r = i;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int c = __popc(uni[w]);
        if (r < c) {
          uint32_t m = uni[w];
          for (int k = 0; k < r; ++k) m &= m - 1;  // drop the r lowest set bits
          e = 32 * w + __ffs(m) - 1;
          break;
        }
        r -= c;
      }
      return e;
    };
    auto place = [&](int i, uint32_t key, int urank) {
      bool ok = urank >= n && urank < len;
      if (lim && ok)  // overall rank < max_p: ranks before (or is) the rank max_p - 1 expert
        ok = key != thr[0] ? key > thr[0] : member_expert(i) <= static_cast<int>(thr[1]);
      if (ok) {
        const int e = member_expert(i);
        if (lim) atomicAdd(placed, 1);
        sets[urank] = e;
        se[urank] = expf(key32_to_logit(key) - rowmax);
      }
    };
    if constexpr (NT >= 256) {
      // T <= 128: thread (part, i) counts half of member i's compares; the
      // halves meet in shared memory (R1's per-CTA keys[] is dead by now)
      int* pc = reinterpret_cast<int*>(rs + L.keys);
      const int part = gt >> 7, i = gt & 127, half = (T + 1) >> 1;
      const uint32_t key = i < T ? ukeys[i] : 0u;
      int urank = i < T ? rank_part(i, key, part * half, min(T, (part + 1) * half)) : 0;
      if (part == 1 && i < T) pc[i] = urank;
      sync();
      if (part == 0 && i < T) place(i, key, urank + pc[i]);
    } else {
#pragma unroll 1
      for (int i = gt; i < T; i += NT) {
        const uint32_t key = ukeys[i];
        place(i, key, rank_part(i, key, 0, T));
      }
    }
  }
  sync();
  if (lim && !masked) len = n + *placed;
  if (gt == 0) {
    float mass = 0.0f;  // sequential fp32 mass in set order
    for (int j = 0; j < len; ++j) mass += se[j];
    for (int j = 0; j < len; ++j) se[j] = se[j] / mass;
  }
  sync();
#pragma unroll 1
  for (int j = gt; j < stride; j += NT) {
    const size_t o = static_cast<size_t>(t) * stride + j;
    const float w = j < len ? se[j] : 0.0f;
    P.x_sets[o] = j < len ? sets[j] : -1;
    P.x_w32[o] = w;
    if (P.x_w64) P.x_w64[o] = static_cast<double>(w);
  }
  if (gt == 0) {
    reinterpret_cast<int*>(rs + L.len)[t] = len;
    P.x_set_len[t] = len;
    if (P.x_phase1_n) P.x_phase1_n[t] = P.cfg.mode == OEA_MODE_VANILLA ? 0 : n;
  }
}

// After R1 (all CTAs): wait for every token's base set, then the union
// (ascending active experts, expert -> group slot) in shared memory.
// Expert-parallel shard: the groups are the active experts this layer holds
// (slot -1 for the others). Returns the number of groups; CTA 0 exports the
// full base / active union.
__device__ __forceinline__ int union_barrier(const FfnParams& P, uint8_t* rs, const RouteSmem& L,
                                             uint32_t tag, const int* arrived = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* uni = reinterpret_cast<uint32_t*>(rs + L.uni);
  int* active = reinterpret_cast<int*>(rs + L.active);
  int* eslot = reinterpret_cast<int*>(rs + L.eslot);
  int* misc = reinterpret_cast<int*>(rs + L.misc);
  const bool exporter = blockIdx.x == 0;
  {
    // many tokens (route-only launch): one poller per CTA on the count of
    // routed tokens instead of B pollers per CTA on the words themselves
    if (arrived != nullptr) {
      if (threadIdx.x == 0)
        while (ld_acquire_gpu(arrived) < P.B) __nanosleep(64);
      __syncthreads();
    }
    // union = OR of the tokens' base bitmaps: thread t < B polls token t's
    // four tagged words (all in flight at once) until they carry this
    // launch's tag; rows OR-ed by lanes 0..3 of warp 0 below
    uint32_t* rows = reinterpret_cast<uint32_t*>(rs + L.tokbits);  // [B][4] scratch
#pragma unroll 1
    for (int t = threadIdx.x; t < P.B; t += blockDim.x) {
      uint4 v4;
      bool ready;
      do {
        unsigned long long v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = ld_relaxed_u64(P.xuni + 4 * t + i);
        ready = true;
#pragma unroll
        for (int i = 0; i < 4; ++i) ready &= static_cast<uint32_t>(v[i] >> 32) == tag;
        v4 = make_uint4(static_cast<uint32_t>(v[0]), static_cast<uint32_t>(v[1]),
                        static_cast<uint32_t>(v[2]), static_cast<uint32_t>(v[3]));
        // every CTA polls the same words: back off (more with many pollers)
        if (!ready) __nanosleep(P.B > 64 ? 200 : 40);
      } while (!ready);
      reinterpret_cast<uint4*>(rows)[t] = v4;
    }
    __syncthreads();
    if (P.B <= 32) {
      if (threadIdx.x < 4) {
        uint32_t o = 0u;
#pragma unroll 4
        for (int t = 0; t < P.B; ++t) o |= rows[4 * t + threadIdx.x];
        uni[threadIdx.x] = o;
      }
    } else if (warp < 4) {
      // many tokens: warp w ORs word w of every row, 32 rows per step, then
      // a shuffle butterfly (a serial loop over B rows would cost ~B x 30 cycles)
      uint32_t o = 0u;
      for (int t = lane; t < P.B; t += 32) o |= rows[4 * t + warp];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) o |= __shfl_xor_sync(kFull, o, off);
      if (lane == 0) uni[warp] = o;
    }
    __syncthreads();
  }
  if (warp == 0) {
    // parameters the scan below needs, read before the poll (their
    // constant-cache misses overlap the wait instead of following it)
    const int N = P.N, e_lo = P.e_begin, e_hi = P.e_begin + P.e_count, nB = P.B;
    int32_t* const x_active = P.x_active;
    int32_t* const x_base_union = P.x_base_union;
    const bool vanilla = P.cfg.mode == OEA_MODE_VANILLA;
    asm volatile("" ::"r"(N), "r"(e_lo), "r"(e_hi), "r"(nB), "l"(x_active), "l"(x_base_union));
    const uint32_t uw[4] = {uni[0], uni[1], uni[2], uni[3]};
    if (lane == 0) stamp(P, 12);
    // Slots by population counts of the union words held in every lane (no
    // warp collectives): slot(e) = #union members below e; the held groups
    // (an EP shard's experts [e_lo, e_hi)) the same over the masked words.
    uint32_t om[4];
    int T = 0, G = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int lo = max(e_lo - 32 * w, 0), hi = min(e_hi - 32 * w, 32);
      const uint32_t range = hi <= lo ? 0u
                                      : ((hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u)) &
                                         ~((1u << lo) - 1u));
      om[w] = uw[w] & range;
      T += __popc(uw[w]);
      G += __popc(om[w]);
    }
    const uint32_t below = lanemask_lt();
    int ub = 0, ob = 0;  // members below this lane's word
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int e = 32 * w + lane;
      if (e < N) {
        const bool f = (uw[w] >> lane) & 1u, own = (om[w] >> lane) & 1u;
        const int slot = ub + __popc(uw[w] & below), gslot = ob + __popc(om[w] & below);
        eslot[e] = own ? gslot : -1;
        if (own) active[gslot] = e;
        if (exporter) {
          // active_union == base_union for the OEA modes; vanilla: the top-k union
          if (f && x_base_union && !vanilla) x_base_union[slot] = e;
          x_active[e] = -1;
        }
      }
      ub += __popc(uw[w]);
      ob += __popc(om[w]);
    }
    if (exporter) {
      __syncwarp();
      int c = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int e = 32 * w + lane;
        if (e < N && ((uw[w] >> lane) & 1u)) x_active[c + __popc(uw[w] & below)] = e;
        c += __popc(uw[w]);
      }
    }
    if (lane == 0) {
      stamp(P, 13);
      misc[0] = G;
      misc[1] = T;  // the full union (R2's |U|)
      if (exporter) {
        *P.x_active_count = T;
        if (P.x_base_union_count)
          *P.x_base_union_count = P.cfg.mode == OEA_MODE_VANILLA ? 0 : T;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) stamp(P, 14);
  return misc[0];
}

// Compaction from the CTA's plan in shared memory (sets / len / loads / token
// bitmaps): row base per active expert (slot order), token lists in token
// order, inverse permutation; CTA 0 exports the aggregates.
template <int NW>
__device__ __forceinline__ void compact_smem(const FfnParams& P, uint8_t* rs, const RouteSmem& L,
                                             int T, bool exporter) {
  const int warp = NW == 1 ? 0 : threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ltid = warp * 32 + lane;
  constexpr int NC = NW * 32;
  auto sync = [&]() {
    if (NW == 1)
      __syncwarp();
    else
      asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
  };
  const int B = P.B, N = P.N, stride = P.cfg.stride;
  const int Bw = (B + 31) >> 5;
  const int* len = reinterpret_cast<const int*>(rs + L.len);
  const int* loads = reinterpret_cast<const int*>(rs + L.loads);
  const int* active = reinterpret_cast<const int*>(rs + L.active);
  const int* eslot = reinterpret_cast<const int*>(rs + L.eslot);
  int* rowb = reinterpret_cast<int*>(rs + L.rowb);
  int* rows = reinterpret_cast<int*>(rs + L.rows);
  int* rtok = reinterpret_cast<int*>(rs + L.rtok);
  int* rslot = reinterpret_cast<int*>(rs + L.rslot);
  const uint32_t* tokbits = reinterpret_cast<const uint32_t*>(rs + L.tokbits);
  if (warp == 0) {
    int R = 0, load = 0;
#pragma unroll 1
    for (int base = 0; base < T; base += 32) {
      const int a = base + lane;
      const int m = a < T ? loads[active[a]] : 0;
      const int nr = (m + 7) / 8 * 8;
      int ri = nr, li = m;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int r2 = __shfl_up_sync(kFull, ri, o), l2 = __shfl_up_sync(kFull, li, o);
        if (lane >= o) {
          ri += r2;
          li += l2;
        }
      }
      const int r0 = R + ri - nr;
      if (a < T) {
        rowb[a] = r0;
        rows[a] = m;
#pragma unroll 1
        for (int r = r0 + m; r < r0 + nr; ++r) rtok[r] = -1;
      }
      R += __shfl_sync(kFull, ri, 31);
      load += __shfl_sync(kFull, li, 31);
    }
    if (exporter) {
#pragma unroll 1
      for (int e = lane; e < N; e += 32) P.x_loads[e] = loads[e];
      if (lane == 0) {
        int tl = 0;  // total load over all experts (load above: the held groups)
        for (int e = 0; e < N; ++e) tl += loads[e];
        *P.x_total_load = tl;
        P.x_hdr->n_groups = T;
        P.x_hdr->T = T;
        P.x_hdr->total_load = tl;
        P.x_hdr->n_rows = R;
      }
    }
  }
  sync();
  const int* sets = reinterpret_cast<const int*>(rs + L.sets);
#pragma unroll 1
  for (int idx = ltid; idx < B * stride; idx += NC) {
    const int t = idx / stride, sl = idx % stride;
    if (sl < len[t] && eslot[sets[idx]] >= 0) {  // (shard: held experts only)
      const int e = sets[idx];
      const uint32_t* bits = tokbits + e * Bw;
      int rank = __popc(bits[t >> 5] & ((1u << (t & 31)) - 1u));
#pragma unroll 1
      for (int w = 0; w < (t >> 5); ++w) rank += __popc(bits[w]);
      const int row = rowb[eslot[e]] + rank;
      rtok[row] = t;
      rslot[row] = sl;
    }
  }
  sync();
}

// R2 + plan exchange + compaction on NW warps (8 consumer warps on the token
// list path, the router warp on the dense path).
template <int NW>
__device__ __forceinline__ void route_phase2_plan(const FfnParams& P, uint8_t* rs,
                                                  const RouteSmem& L, int T, uint32_t tag,
                                                  bool gather = true) {
  const int warp = NW == 1 ? 0 : threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gt = warp * 32 + lane;
  constexpr int NC = NW * 32;
  auto sync = [&]() {
    if (NW == 1)
      __syncwarp();
    else
      asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
  };
  const int B = P.B, stride = P.cfg.stride, Np = P.Np;
  const int Bw = (B + 31) >> 5;
  // plan row of token t as self-validating tagged words {tag | payload}:
  // [0] = set length, [1 + 2j] = expert of slot j (-1 past the length),
  // [2 + 2j] = its fp32 weight; readers take all rows in one pass
  const int W = 1 + 2 * stride;
#pragma unroll 1
  for (int t = blockIdx.x; t < B; t += gridDim.x) {
    rank_phase2<NC>(P, t, rs, L, reinterpret_cast<const int*>(rs + L.misc)[1], gt, sync);
    sync();  // (the row's sets / weights in shared memory are final)
    const int* srow = reinterpret_cast<const int*>(rs + L.sets) + t * stride;
    const float* erow = reinterpret_cast<const float*>(rs + L.e) + t * stride;
    const int ln = reinterpret_cast<const int*>(rs + L.len)[t];
    for (int k = gt; k < W; k += NC) {
      const int j = (k - 1) >> 1;
      const uint32_t v = k == 0 ? static_cast<uint32_t>(ln)
                         : ((k - 1) & 1) == 0 ? static_cast<uint32_t>(j < ln ? srow[j] : -1)
                                              : __float_as_uint(j < ln ? erow[j] : 0.0f);
      st_relaxed_u64(P.xplan + static_cast<size_t>(t) * W + k, tagged(tag, v));
    }
  }
  if (!gather) return;
  int* len = reinterpret_cast<int*>(rs + L.len);
  int* sets = reinterpret_cast<int*>(rs + L.sets);
  float* wts = reinterpret_cast<float*>(rs + L.e);
  int* loads = reinterpret_cast<int*>(rs + L.loads);
  uint32_t* tokbits = reinterpret_cast<uint32_t*>(rs + L.tokbits);
  sync();  // (this CTA's own rows were read above; the arrays are rebuilt below)
  // every token's plan row in one pass: each word carries its own tag
#pragma unroll 2
  for (int idx = gt; idx < B * W; idx += NC) {
    const unsigned long long* w = P.xplan + idx;
    unsigned long long v = ld_relaxed_u64(w);
    while (static_cast<uint32_t>(v >> 32) != tag) v = ld_relaxed_u64(w);
    const int t = idx / W, k = idx % W;
    const uint32_t pv = static_cast<uint32_t>(v);
    if (k == 0)
      len[t] = static_cast<int>(pv);
    else if (((k - 1) & 1) == 0)
      sets[t * stride + ((k - 1) >> 1)] = static_cast<int>(pv);
    else
      wts[t * stride + ((k - 1) >> 1)] = __uint_as_float(pv);
  }
#pragma unroll 1
  for (int i = gt; i < Np; i += NC) loads[i] = 0;
#pragma unroll 1
  for (int i = gt; i < Np * Bw; i += NC) tokbits[i] = 0u;
  sync();
#pragma unroll 4
  for (int idx = gt; idx < B * stride; idx += NC) {
    const int t = idx / stride, sl = idx % stride;
    if (sl < len[t]) {
      const int e = sets[idx];
      atomicAdd(&loads[e], 1);
      atomicOr(&tokbits[e * Bw + (t >> 5)], 1u << (t & 31));
    }
  }
  sync();
  compact_smem<NW>(P, rs, L, T, blockIdx.x == 0);
}

// Route-only launch (64 < B <= 256): the compaction of k_compact
// (router_fused.cu compact_plan) distributed over the grid in the same
// launch. Once every token's plan row is out (claims[0] = B), CTA e takes
// expert e: its tokens in token order (a ballot scan of the batch's sets) and
// its load (x_loads); the same scan counts every expert's load in shared
// memory, so each CTA places its expert's token groups (<= 64 rows, the last padded to 8) and
// rows after the groups / rows of the experts before it (ascending experts =
// the active-union order), writes row -> (token, slot) and, for the tcgen05
// FFN, the token rows in the CM layout (xg). CTA 0 writes the header and the
// total load.
__device__ __forceinline__ void route_compact_dist(const FfnParams& P, uint8_t* rs,
                                                   const RouteSmem& L, int* claims) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NT = kFfnThreads, NWARP = kFfnThreads / 32;
  const int B = P.B, N = P.N, stride = P.cfg.stride;
  int* tl_tok = reinterpret_cast<int*>(rs + L.rtok);   // [<= B] this expert's tokens
  int* tl_slot = reinterpret_cast<int*>(rs + L.rslot);
  int* wcnt = reinterpret_cast<int*>(rs + L.red);      // [NWARP]
  int* misc = reinterpret_cast<int*>(rs + L.misc);
  int* cnt = reinterpret_cast<int*>(rs + L.loads);     // [N] every expert's load
  for (int i = tid; i < N; i += NT) cnt[i] = 0;
  if (tid == 0)
    while (ld_acquire_gpu(claims) < B) __nanosleep(32);
  __syncthreads();
  const int e = blockIdx.x;
  int load = 0;
  if (e < N) {
#pragma unroll 1
    for (int t0 = 0; t0 < B; t0 += NT) {
      const int t = t0 + tid;
      // (the exported rows are -1 past the set length: the whole row's loads
      // go out at once, no length round trip, no early exit); every CTA
      // counts every expert's load from the same scan, so the group / row
      // bases need no second grid-wide exchange
      int slot = -1;
      if (t < B) {
        const int32_t* row = P.x_sets + static_cast<size_t>(t) * stride;
#pragma unroll 8
        for (int j = 0; j < stride; ++j) {
          const int v = __ldcg(row + j);
          if (v >= 0) atomicAdd(&cnt[v], 1);
          if (v == e && slot < 0) slot = j;
        }
      }
      const unsigned m = __ballot_sync(kFull, slot >= 0);
      if (lane == 0) wcnt[warp] = __popc(m);
      __syncthreads();
      int before = load, tot = 0;
#pragma unroll
      for (int w = 0; w < NWARP; ++w) {
        before += w < warp ? wcnt[w] : 0;
        tot += wcnt[w];
      }
      if (slot >= 0) {
        const int pos = before + __popc(m & lanemask_lt());
        tl_tok[pos] = t;
        tl_slot[pos] = slot;
      }
      __syncthreads();
      load += tot;
    }
    if (tid == 0) P.x_loads[e] = load;
  }
  __syncthreads();
  // groups / rows of the experts before e (k_compact's formulas)
  if (warp == 0) {
    int gb = 0, rb = 0, ng_all = 0, nr_all = 0, act = 0, tl = 0;
    for (int i = lane; i < N; i += 32) {
      const int m = cnt[i];
      const int ng = (m + kTokGroup - 1) / kTokGroup;
      const int nr = m > 0 ? (m / kTokGroup) * kTokGroup + ((m % kTokGroup) + 7) / 8 * 8 : 0;
      if (i < e) {
        gb += ng;
        rb += nr;
      }
      ng_all += ng;
      nr_all += nr;
      act += m > 0;
      tl += m;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      gb += __shfl_xor_sync(kFull, gb, off);
      rb += __shfl_xor_sync(kFull, rb, off);
      ng_all += __shfl_xor_sync(kFull, ng_all, off);
      nr_all += __shfl_xor_sync(kFull, nr_all, off);
      act += __shfl_xor_sync(kFull, act, off);
      tl += __shfl_xor_sync(kFull, tl, off);
    }
    if (lane == 0) {
      misc[2] = gb;
      misc[3] = rb;
      if (blockIdx.x == 0) {
        P.x_hdr->n_groups = ng_all;
        P.x_hdr->T = act;
        P.x_hdr->total_load = tl;
        P.x_hdr->n_rows = nr_all;
        *P.x_total_load = tl;
      }
    }
  }
  __syncthreads();
  if (e < N && load > 0) {
    const int gb = misc[2], rb = misc[3];
    const int ng = (load + kTokGroup - 1) / kTokGroup;
    const int nr = (load / kTokGroup) * kTokGroup + ((load % kTokGroup) + 7) / 8 * 8;
    int32_t* ga = const_cast<int32_t*>(P.group_a);
    int32_t* g0 = const_cast<int32_t*>(P.group_row0);
    int32_t* gr = const_cast<int32_t*>(P.group_rows);
    int32_t* rt = const_cast<int32_t*>(P.row_tok);
    int32_t* rsl = const_cast<int32_t*>(P.row_slot);
    for (int k = tid; k < ng; k += NT) {
      ga[gb + k] = e;
      g0[gb + k] = rb + k * kTokGroup;
      gr[gb + k] = min(kTokGroup, load - k * kTokGroup);
    }
    for (int i = tid; i < nr; i += NT) {
      rt[rb + i] = i < load ? tl_tok[i] : -1;
      rsl[rb + i] = i < load ? tl_slot[i] : 0;
    }
    if (P.xg != nullptr) {
      // token rows -> xg (CM: [Dp/128 slices][row groups] x 2 KiB, 16-byte
      // chunk (kg, row % 8) at kg * 128 + (row % 8) * 16), rows past the
      // expert's tokens zero
      const int nch = P.Dp >> 3, total = nr * nch;
      constexpr int kU = 8;  // a thread's chunks: all loads in flight, then the stores
#pragma unroll 1
      for (int i0 = tid; i0 < total; i0 += NT * kU) {
        uint4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int idx = i0 + u * NT;
          const int i = idx / nch, ch = idx - i * nch;
          const int t = idx < total && i < load ? tl_tok[i] : -1;
          v[u] = t >= 0 ? __ldg(reinterpret_cast<const uint4*>(P.x_in + static_cast<size_t>(t) * P.Dp +
                                                              ch * 8))
                        : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int idx = i0 + u * NT;
          if (idx < total) {
            const int i = idx / nch, ch = idx - i * nch, r = rb + i;
            *reinterpret_cast<uint4*>(P.xg + (static_cast<size_t>(ch >> 4) * P.xg_rg + (r >> 3)) * 2048 +
                                      (ch & 15) * 128 + (r & 7) * 16) = v[u];
          }
        }
      }
    }
  }
}

// The last CTA to leave resets the grid's counters (round claims, combine /
// logits barriers, per-group W1 release counters), so the next launch (fused
// or two-kernel, graph-captured or not) starts from zero. Called by thread 0
// once its CTA no longer touches any counter.
__device__ __forceinline__ void grid_exit(const FfnParams& P, int* claims, int G) {
  __threadfence();
  if (atomicAdd(&claims[4], 1) == static_cast<int>(gridDim.x) - 1) {
    for (int g = 0; g < G; ++g) P.w1_done[g] = 0;
    for (int c = 0; c < 16; ++c)
      if (c != 4 && c != 7) claims[c] = 0;
    claims[7] += 1;  // launch epoch: the tag of the next launch's exchange words
    __threadfence();
    claims[4] = 0;
  }
}

// ---- tcgen05 helpers of the dense tensor-core consumer (MODE 6) ----------
// canonical K-major no-swizzle UMMA operand: LBO 128 B (K), SBO 2 KiB (M/N)
__device__ __forceinline__ uint64_t d_umma_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(128 >> 4) << 16) |
         (static_cast<uint64_t>(2048 >> 4) << 32) | (1ull << 46);
}
// D fp32, A / B bf16 K-major, N = 16, M = 128
constexpr uint32_t kDenseIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (2u << 17) | (8u << 24);
__device__ __forceinline__ void d_umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(acc), "r"(kDenseIdesc)
      : "memory");
}
__device__ __forceinline__ void d_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void d_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void d_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void d_tmem_ld16(uint32_t taddr, float (&v)[16]) {
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
// dense h / x tiles in the UMMA layout: [128-wide K slice][2 row groups of 8
// tokens][16 k-groups][8 tokens][8 k] bf16 (4 KiB per slice)
__host__ __device__ __forceinline__ size_t cm16_index(int r, int k) {
  return static_cast<size_t>(k >> 7) * 2048 + (r >> 3) * 1024 + ((k & 127) >> 3) * 64 + (r & 7) * 8 +
         (k & 7);
}

// Round descriptor published by the producer through the stage barrier.
struct RoundDesc {
  int u0;    // first unit
  int n;     // units (one per consumer warp); 0 = end of work
  int kind;  // 1 = W1, 2 = W2
  int ready; // W2: the group's h was acquired complete by the producer
  int sb;    // stages [sb, se) of the units' K (W2 K split: one part; else all)
  int se;
  int kp;    // K part (y plane)
};
constexpr int kRoundRing = 8;  // > kStages: a round spans >= 1 stage

// MODE 0: two-kernel path (plan from the router kernel); 1: fused, token
// lists (B <= 64); 2: fused, dense-over-batch W1 (B <= 16). Separate
// instantiations keep each variant's register allocation and code small.
template <int MODE>
__global__ void __launch_bounds__(kFfnThreads, 1) k_ffn_bf16(const FfnParams P) {
  constexpr bool kFused = MODE != 0;
  constexpr bool kUmma = MODE == 6;  // dense decode, tcgen05 consumer
  constexpr bool kDense = MODE == 2 || MODE == 5 || kUmma;
  constexpr bool kRouteOnly = MODE == 3;  // plan only (B > 64); the FFN runs as MODE 0
  constexpr bool kEp = MODE == 4 || MODE == 5;  // MODE 1 / 2 with the peer-memory EP combine
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  RoundDesc* rdesc = reinterpret_cast<RoundDesc*>(empty + kStages);
  uint64_t* plan_bar = reinterpret_cast<uint64_t*>(
      reinterpret_cast<PlanRef*>(rdesc + kRoundRing) + 1);  // dense: router warp -> W2
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // Programmatic dependent launch: the next kernel of the stream (the next
  // layer's decode, a norm, ...) may be launched now; its CTAs take SMs as
  // ours exit and do their own pre-wait setup while our tail runs. Nothing
  // below depends on it (it cannot pass its griddepcontrol.wait until this
  // grid has completed), so the trigger is safe at the very start.
  if (kFused) pdl_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kUmma ? 1 : kFfnWarps);  // (MODE 6: the MMA commit frees it)
    }
    mbar_init(plan_bar, 1);
    mbar_init(plan_bar + 1, 1);  // split rounds: warp 0 has read the reduction buffer
    fence_mbar_init();
  }
  // Before the wait (PDL launch: overlapping the previous kernel's tail),
  // only what reads no predecessor output: the L2 prefetch of the weights.
  const bool pf_early = kFused && !kRouteOnly && P.pf_early && P.prefetch_bytes > 0;
  if (pf_early && warp == kProducerWarp) prefetch_w1_heads(P, lane);
  __syncthreads();
  // Everything below reads the router kernel's outputs (two-kernel path) or
  // the previous launch's workspace (epoch, counters: fused path).
  pdl_wait();

  PlanRef* PR = reinterpret_cast<PlanRef*>(rdesc + kRoundRing);
  uint8_t* rs = reinterpret_cast<uint8_t*>(PR + 1) + 16;
  const RouteSmem RL = route_smem_layout(P.B, P.Np, P.stride);
  uint8_t* xs = rs + (kFused ? RL.total : 0);  // dense path: x tile (16 B aligned)
  SplitRed SR;
  SR.buf = reinterpret_cast<float*>(xs + (kDense ? 16 * P.xs_row : 0));
  uint8_t* btile = reinterpret_cast<uint8_t*>(SR.buf) + kSplitRedBytes;  // (token-list modes)
  SR.free = plan_bar + 1;
  SR.idx = nullptr;
  int sidx = 0;  // split rounds consumed by this warp
  // [0..1] round claims, [2]/[5] combine arrivals (epoch parity), [3] padded-x barrier,
  // [4] exit (route-only launch), [7] launch epoch
  int* claims = P.claims;  // independent of the layer's shape (one workspace, many layers)
  // this launch's exchange tag (the epoch only changes when a launch retires)
  const uint32_t tag = static_cast<uint32_t>(__ldcg(claims + 7)) + 1u;
  if (P.trace) {  // (debug builds of the context only; uniform branch)
    if (threadIdx.x == 0) {
      s_trace = P.trace + kTraceLegacy + (tag & (kTraceLaunches - 1)) * kTracePerLaunch;
      stamp(P, 0);
    }
    __syncthreads();
  } else if (threadIdx.x == 0) {
    s_trace = nullptr;
  }
  if (kFused) {
    if (warp == kRouterWarp && lane == 0) {
      // Touch every line of the parameter block once, early and all at once
      // (the router warp has no GEMV chunk): the prologue would otherwise
      // take a constant-cache miss, serially, per newly used line.
      asm volatile("" ::"l"(P.w1), "l"(P.hbuf), "l"(P.out), "r"(P.xs_row), "r"(P.e_begin),
                   "l"(P.xuni), "l"(P.xplan), "l"(P.router_t), "l"(P.logits), "l"(P.mask),
                   "r"(P.N), "r"(P.cfg.mode), "r"(P.cfg.limit));
      asm volatile("" ::"l"(P.x_sets), "l"(P.x_w64), "l"(P.x_active), "l"(P.x_active_count),
                   "l"(P.x_phase1_n), "l"(P.x_base_union), "l"(P.x_base_union_count),
                   "l"(P.x_hdr), "l"(P.x_loads), "l"(P.x_total_load), "l"(P.trace));
    }
    if (threadIdx.x == 0) {
      PR->row_tok = reinterpret_cast<const int32_t*>(rs + RL.rtok);
      PR->row_slot = reinterpret_cast<const int32_t*>(rs + RL.rslot);
      PR->group_a = reinterpret_cast<const int32_t*>(rs + RL.active);
      PR->group_row0 = reinterpret_cast<const int32_t*>(rs + RL.rowb);
      PR->group_rows = reinterpret_cast<const int32_t*>(rs + RL.rows);
      PR->set_len = reinterpret_cast<const int32_t*>(rs + RL.len);
      PR->wts = reinterpret_cast<const float*>(rs + RL.e);
      PR->btile = btile;
    }
    // (x in host memory: before the GEMV, inside the host round trip of
    // the x staging, when HBM idles longest)
    if (!kRouteOnly && !pf_early && P.x_stage && warp == kProducerWarp && P.prefetch_bytes > 0)
      prefetch_w1_heads(P, lane);
    if (kRouteOnly) {
      if (threadIdx.x == 0) stamp(P, 8);
      tile_gemv(P, SR.buf, tag);
    } else
      fused_gemv(P, reinterpret_cast<float*>(rs + RL.red), claims + 3, tag,
                 reinterpret_cast<float*>(rs + RL.lgp));
    if (threadIdx.x == 0) stamp(P, 5);
    // (x in device memory: after the GEMV, whose loads it would delay)
    // (x in host memory: the blind heads went out before the staging; the
    // guided ones follow here when the guess is on: OEA_HOST_PF_GUESS)
    if (!kRouteOnly && !pf_early && (!P.x_stage || P.host_pf_guess) && warp == kProducerWarp &&
        (P.prefetch_bytes > 0 || P.pf_guess_hi > 0))
      prefetch_w1_heads(P, lane, P.e_begin == 0 && P.e_count == P.N ? reinterpret_cast<const float*>(rs + RL.lgp) : nullptr);
    // R1: CTA t routes token t (thread per expert), then the union barrier
    if (threadIdx.x < 128) {
#pragma unroll 1
      for (int t = blockIdx.x; t < P.B; t += gridDim.x) {
        rank_phase1(P, t, rs, RL, tag);
        asm volatile("bar.sync 3, 128;" ::: "memory");  // keys[] reused by the next token
      }
      // route-only: count this CTA's routed tokens (the barrier above orders
      // the 4 warps' base-bitmap words before the cumulative release)
      if (kRouteOnly && threadIdx.x == 0 && static_cast<int>(blockIdx.x) < P.B)
        red_release_gpu_add(claims + 3, (P.B - 1 - static_cast<int>(blockIdx.x)) /
                                                static_cast<int>(gridDim.x) + 1);
      if (threadIdx.x == 0) stamp(P, 11);
    }
    // (ends with __syncthreads)
    const int T = union_barrier(P, rs, RL, tag, kRouteOnly ? claims + 3 : nullptr);
    if (threadIdx.x == 0) {
      PR->G = T;
      stamp(P, 6);
      if (s_trace && blockIdx.x == 0) s_trace[kTraceInfo] = static_cast<unsigned long long>(T);
    }
    if (kRouteOnly && P.pf_w1u != nullptr && warp == kProducerWarp) {
      // HBM idles until the FFN launch: the first pf_total bytes of the
      // active experts' W1 streams (the FFN claims W1 group-major, experts
      // ascending) into L2, 32 KiB per lane, spread over the grid
      const int* act = reinterpret_cast<const int*>(rs + RL.active);
      const size_t total = min(P.pf_total, static_cast<size_t>(T) * P.pf_w1u_stride);
      for (size_t c = static_cast<size_t>(blockIdx.x) * 32 + lane; c * 32768 < total;
           c += static_cast<size_t>(gridDim.x) * 32) {
        const size_t byte = c * 32768, i = byte / P.pf_w1u_stride, off = byte - i * P.pf_w1u_stride;
        bulk_prefetch_l2(P.pf_w1u + static_cast<size_t>(act[i] - P.e_begin) * P.pf_w1u_stride + off,
                         static_cast<uint32_t>(min(static_cast<size_t>(32768), P.pf_w1u_stride - off)));
      }
    }
    if (kRouteOnly) {
      // plan rows (CTA t: token t, t + grid, ...); the FFN tables and the
      // aggregates (loads, header) follow: in this launch (route_compact_dist)
      // or from k_compact.
      if (warp < kFfnWarps) route_phase2_plan<kFfnWarps>(P, rs, RL, T, tag, false);
      if (P.compact_in_kernel) {
        __syncthreads();  // (this CTA's rows are out: cumulative release below)
        if (threadIdx.x == 0) stamp(P, 1);
        if (threadIdx.x == 0 && static_cast<int>(blockIdx.x) < P.B)
          red_release_gpu_add(claims, (P.B - 1 - static_cast<int>(blockIdx.x)) /
                                          static_cast<int>(gridDim.x) + 1);
        route_compact_dist(P, rs, RL, claims);
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        stamp(P, 7);
        grid_exit(P, claims, 0);
        stamp(P, 15);
      }
      return;
    }
  } else if (threadIdx.x == 0) {
    PR->row_tok = P.row_tok;
    PR->row_slot = P.row_slot;
    PR->group_a = P.group_a;
    PR->group_row0 = P.group_row0;
    PR->group_rows = P.group_rows;
    PR->set_len = P.set_len;
    PR->wts = P.wts;
    PR->btile = btile;
    PR->G = P.hdr->n_groups;
  }
  __syncthreads();
  // G == 0 (every token masked) needs no special case: the producer's first
  // claim ends the work, and the combine writes zeros (empty sets).
  const int G = PR->G;
  const int KT1 = P.Dp >> 4, KT2 = P.Hp >> 4;
  const int RB1 = P.Hp >> 3, RB2 = P.Dp >> 4;
  const int U1 = G * RB1, U2 = G * RB2;
  // Split rounds (one unit per round, K over the 8 warps) when there are too
  // few 8-unit rounds to keep every SM streaming (B <= 16: <= 2 n-blocks).
  const bool split = kFused && !kDense && P.B <= 16 && P.split_ok &&
                     (U1 + kFfnWarps - 1) / kFfnWarps + (U2 + kFfnWarps - 1) / kFfnWarps <
                         2 * static_cast<int>(gridDim.x);
  // W2 K parts per round (dense path; the combine sums the y planes)
  const int w2ks = kDense && !split ? max(1, min(P.w2_ks, KT2 / kKtPerSlot)) : 1;
  // Dynamic scheduling: rounds of up to 8 consecutive units are claimed from
  // two global counters, all W1 (gate/up) rounds before any W2 (down) round.
  // A CTA therefore finishes its own W1 rounds before it starts W2 rounds,
  // and W2 units only wait for W1 units claimed earlier (by any CTA), so the
  // acquire-waits cannot deadlock; faster SMs simply claim more rounds.

  int stage = 0;
  uint32_t phase = 0;

  if (warp == kRouterWarp) {
    // ---------------- router warp ----------------
    // Dense path: phase 2, weights and the token lists of the W2 units for
    // the whole batch (redundantly per CTA, like phase 1) while the W1
    // weights stream; consumers wait for it only before their first W2 round.
    if (kDense) {
      // few (token, member) pairs: every CTA ranks the whole batch itself (no
      // exchange latency before W2, which matters when W1 is short); many:
      // CTA t ranks token t and the plan rows are exchanged (the O(B T^2)
      // redundant work would otherwise steal issue slots from the consumers)
      route_phase2_plan<1>(P, rs, RL, G, tag);
      if (lane == 0) {
        stamp(P, 7);
        mbar_arrive(plan_bar);  // W2 rounds may start
      }
    }
  } else if (warp == kProducerWarp) {
    // ---------------- producer: claims rounds, TMA bulk weight stream ----------
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      bool w1_left = true;
      const int nst2 = KT2 / kKtPerSlot, ks2 = w2ks;
      auto claim = [&]() {
        RoundDesc d{0, 0, 0, 0, 0, 0, 0};
        if (split) {  // one unit per round: kind 3 (W1) / 4 (W2)
          if (w1_left) {
            const int r = atomicAdd(&claims[0], 1);
            if (r < U1) return RoundDesc{r, 1, 3, 0, 0, 0, 0};
            w1_left = false;
          }
          const int r = atomicAdd(&claims[1], 1);
          if (r < U2) d = RoundDesc{U1 + r, 1, 4, 0, 0, 0, 0};
          return d;
        }
        if (w1_left) {
          const int r = atomicAdd(&claims[0], 1);
          if (r * kFfnWarps < U1) {
            // the first r0 rounds of every group first (round-major: the
            // heads the prologue prefetched into L2), then group-major
            const int RR = RB1 / kFfnWarps, r0 = min(P.r0, RR);
            int g, rr;
            if (r < r0 * G) {
              rr = r / G;
              g = r - rr * G;
            } else {
              const int q = r - r0 * G;
              g = q / (RR - r0);
              rr = r0 + (q - g * (RR - r0));
            }
            d.u0 = g * RB1 + rr * kFfnWarps;
            d.n = min(kFfnWarps, U1 - d.u0);
            d.kind = 1;
            d.se = KT1 / kKtPerSlot;
            return d;
          }
          w1_left = false;
        }
        // W2 (dense path): each round's K in w2_ks parts claimed one by one
        // (consecutive claims: the parts of one round run on different SMs),
        // so the last rounds are short and the SMs finish together; part kp
        // writes y plane kp, summed in part order by the combine
        const int rk = atomicAdd(&claims[1], 1);
        const int r = rk / ks2, kp = rk - r * ks2;
        if (r * kFfnWarps < U2) {
          d.u0 = U1 + r * kFfnWarps;
          d.n = min(kFfnWarps, U2 - r * kFfnWarps);
          d.kind = 2;
          d.sb = kp * nst2 / ks2;
          d.se = (kp + 1) * nst2 / ks2;
          d.kp = kp;
        }
        return d;
      };
      RoundDesc next = claim();
      // debug round log: per CTA kTraceRounds x {start, kind/group/unit, W2 h ready}
      unsigned long long* rlog =
          s_trace ? s_trace + kTraceRoundLog + blockIdx.x * kTraceRounds * 3 : nullptr;
      for (int seq = 0;; ++seq) {
        const RoundDesc d = next;
        mbar_wait(&empty[stage], phase ^ 1u);
        if (rlog != nullptr && seq < kTraceRounds) {
          rlog[3 * seq] = gtimer();
          rlog[3 * seq + 1] = (static_cast<unsigned long long>(d.kind) << 56) |
                              (static_cast<unsigned long long>(d.n) << 48) |
                              static_cast<unsigned long long>(static_cast<uint32_t>(d.u0));
        }
        rdesc[seq & (kRoundRing - 1)] = d;
        if (d.n == 0) {
          mbar_arrive(&full[stage]);  // end-of-work message, no payload
          break;
        }
        if (d.kind >= 3) {
          // split round: unit u's K slices, 8 per stage (one 4 KiB copy per
          // warp slot), from its place in the round-interleaved layout
          const bool s1 = d.kind == 3;
          const int KT = s1 ? KT1 : KT2, RB = s1 ? RB1 : RB2;
          const int v = s1 ? d.u0 : d.u0 - U1;
          const int g = v / RB, rb = v % RB, rr = rb / kFfnWarps, wl = rb % kFfnWarps;
          const int S = KT / kKtPerSlot, nss = (S + kFfnWarps - 1) / kFfnWarps;
          const uint4* rbase = (s1 ? P.w1 : P.w2) +
                               (static_cast<size_t>(PR->group_a[g] - P.e_begin) * RB +
                                rr * kFfnWarps) * KT * 32;
          for (int s2 = 0; s2 < nss; ++s2) {
            if (s2 > 0) mbar_wait(&empty[stage], phase ^ 1u);
            const int np = min(kFfnWarps, S - s2 * kFfnWarps);
            mbar_expect_tx(&full[stage], np * kSlotBytes);
            for (int w = 0; w < np; ++w)
              bulk_g2s(ring + stage * kStageBytes + w * kSlotBytes,
                       rbase + static_cast<size_t>(((s2 * kFfnWarps + w) * kFfnWarps + wl) *
                                                   kKtPerSlot) * 32,
                       kSlotBytes, &full[stage], pol);
            if (s2 == 0 && !s1)
              rdesc[seq & (kRoundRing - 1)].ready = ld_acquire_gpu(&P.w1_done[g]) >= RB1;
            mbar_arrive(&full[stage]);
            if (s2 == 0) next = claim();
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1u;
            }
          }
          continue;
        }
        const bool is1 = d.kind == 1;
        const int KT = is1 ? KT1 : KT2;
        // The round's 8 units are 8 consecutive row blocks of one expert (RB1
        // and RB2 are multiples of 8, rounds start at multiples of 8), stored
        // round-interleaved: stage s is one contiguous block.
        const int v = is1 ? d.u0 : d.u0 - U1;
        const int RB = is1 ? RB1 : RB2;
        const int g = v / RB, rr = (v % RB) / kFfnWarps;
        // (MODE 6: the UMMA-layout copy, m-block rr = these 8 row blocks;
        // a stage is the same 32 KiB block size in both layouts)
        const uint4* base =
            kUmma ? reinterpret_cast<const uint4*>(
                        (is1 ? P.w1u : P.w2u) +
                        static_cast<size_t>(PR->group_a[g] - P.e_begin) * (is1 ? P.w1u_stride : P.w2u_stride) +
                        static_cast<size_t>(rr) * (KT / kKtPerSlot) * kStageBytes)
                  : (is1 ? P.w1 : P.w2) +
                        (static_cast<size_t>(PR->group_a[g] - P.e_begin) * RB + rr * kFfnWarps) * KT * 32;
        // dense W2: the group's h slice of each stage rides in the stage
        const bool hst = kDense && !is1;
        const uint32_t sbytes = d.n * kSlotBytes + (hst ? kHSlice : 0);
        const __nv_bfloat16* hsrc = P.hbuf + static_cast<size_t>(g) * 16 * P.Hp;
        const int sq = hst ? w1_slot_q(P.Hp) : 1;
        unsigned long long* const wsl = hst ? P.w1_slots + g : nullptr;
        // slot field c is complete when it equals its row-block count, so
        // (count word ^ full) has a zero byte c exactly for the complete slots
        unsigned long long miss = ~0ull;
        for (int s = d.sb; s < d.se; ++s) {
          if (s > d.sb) mbar_wait(&empty[stage], phase ^ 1u);
          if (hst) {
            // the stage's weights first, then wait for its h slot and copy it
            // (h rides in the stage: consumers never wait on W1 themselves)
            if (s == d.sb) rdesc[seq & (kRoundRing - 1)].ready = 1;
            mbar_arrive_expect_tx(&full[stage], sbytes);
            bulk_g2s(ring + stage * kStageBytes,
                     base + static_cast<size_t>(s) * kFfnWarps * kKtPerSlot * 32, d.n * kSlotBytes,
                     &full[stage], pol);
            const int c = s / sq;
            if (s == d.sb) miss = ld_acquire_u64(wsl) ^ P.w1_full;  // every slot, one acquire
            bool acq = s == d.sb;
            while ((miss >> (8 * c)) & 0xffu) {
              __nanosleep(32);
              miss = ld_acquire_u64(wsl) ^ P.w1_full;
              acq = true;
            }
            if (acq) {  // h acquired since the last fence: order it before the async-proxy copy
              if (rlog != nullptr && seq < kTraceRounds && s == d.sb) rlog[3 * seq + 2] = gtimer();
              fence_proxy_async_global();
            }
            bulk_g2s_nohint(reinterpret_cast<uint8_t*>(SR.buf) + stage * kHSlice,
                            hsrc + static_cast<size_t>(s) * 2048, kHSlice, &full[stage]);
          } else if (s == d.sb && !is1) {
            // W2: while the first stage's weights are in flight, check that
            // the group's h is complete (dense path: wait for it, then order
            // the acquired h before the bulk copies of its slices); the
            // descriptor is published by the arrive below, and consumers
            // skip their own acquire-wait
            mbar_expect_tx(&full[stage], sbytes);
            bulk_g2s(ring + stage * kStageBytes,
                     base + static_cast<size_t>(s) * kFfnWarps * kKtPerSlot * 32, d.n * kSlotBytes,
                     &full[stage], pol);
            rdesc[seq & (kRoundRing - 1)].ready = ld_acquire_gpu(&P.w1_done[g]) >= RB1;
            mbar_arrive(&full[stage]);
          } else {
            mbar_arrive_expect_tx(&full[stage], sbytes);
            bulk_g2s(ring + stage * kStageBytes,
                     base + static_cast<size_t>(s) * kFfnWarps * kKtPerSlot * 32, d.n * kSlotBytes,
                     &full[stage], pol);
          }
          if (s == d.sb) next = claim();  // overlap the next claim with this round
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
      stamp(P, 4);
    }
    return;
  } else {
  // ---------------- consumers ----------------
  if (kDense) {
    // x (final since the logits barrier) -> swizzled shared tile, 16 rows
    // (rows >= B zero-filled), while the producer's first stages land
    // (MODE 6: the UMMA layout, cm16_index)
    const int nch = P.Dp >> 3;
#pragma unroll 4
    for (int i = threadIdx.x; i < 16 * nch; i += kFfnWarps * 32) {
      const int t = i / nch, c = i % nch;
      const uint32_t dst =
          kUmma ? smem_u32(xs + cm16_index(t, c * 8) * 2)
                : smem_u32(xs + t * P.xs_row + (c >> 4) * 256 + xs_chunk(c & 15) * 16);
      const __nv_bfloat16* src = P.xpad + static_cast<size_t>(t < P.B ? t : 0) * P.Dp + c * 8;
      cp_async16(dst, src, t < P.B ? 16 : 0);
    }
    cp_async_commit();
    cp_async_wait_all();
    if (kUmma) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // (tcgen05 reads it)
    asm volatile("bar.sync 1, %0;" ::"r"(kFfnWarps * 32) : "memory");
  } else if (kFused) {
    route_phase2_plan<kFfnWarps>(P, rs, RL, G, tag);  // overlaps the first stages
    if (threadIdx.x == 0) stamp(P, 7);
  }
  if constexpr (kUmma) {
    // ---- tcgen05 consumer (dense decode): warp 0 allocates TMEM and its lane
    // 0 issues the MMAs (M = 128 rows of the round, N = the 16 token rows,
    // K = 16 per instruction, 8 per stage; A = the stage, B = the x tile slice
    // (W1) or the stage's h slice (W2)); warps 4-7 drain the accumulator
    // (TMEM lanes 32 (warp % 4) ..): W1 -> silu(g) * u -> h, W2 -> y[group][token]
    uint8_t* ext = xs + static_cast<size_t>(16) * P.Dp * 2;  // (the tile's row padding)
    uint64_t* tfull = reinterpret_cast<uint64_t*>(ext);      // [2] accumulator ready
    uint64_t* tempty = tfull + 2;                             // [2] drained (4 warps)
    uint64_t* dready = tempty + 2;                            // [2] round descriptor out
    RoundDesc* udesc = reinterpret_cast<RoundDesc*>(dready + 2);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(udesc + 2);
    if (threadIdx.x == 0) {
      for (int b = 0; b < 2; ++b) {
        mbar_init(&tfull[b], 1);
        mbar_init(&tempty[b], 4);
        mbar_init(&dready[b], 1);
      }
      fence_mbar_init();
    }
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tslot)),
                   "r"(32)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    d_fence_before();
    asm volatile("bar.sync 1, %0;" ::"r"(kFfnWarps * 32) : "memory");
    d_fence_after();
    const uint32_t tmem = *tslot;
    if (warp == 0) {
      if (lane == 0) {
        for (int seq = 0;; ++seq) {
          mbar_wait(&full[stage], phase);  // the round's first stage carries its descriptor
          const RoundDesc d = rdesc[seq & (kRoundRing - 1)];
          const int buf = seq & 1;
          if (d.n == 0) {
            udesc[buf] = d;
            mbar_arrive(&dready[buf]);
            break;
          }
          mbar_wait(&tempty[buf], ((seq >> 1) & 1) ^ 1u);
          d_fence_after();
          const bool is1 = d.kind == 1;
          const uint32_t dt = tmem + buf * 16;
          const int nst = d.se - d.sb;
          for (int s0 = 0; s0 < nst; ++s0) {
            if (s0 > 0) mbar_wait(&full[stage], phase);
            d_fence_after();
            const int s = d.sb + s0;
            const uint32_t a0 = smem_u32(ring + stage * kStageBytes);
            const uint32_t b0 = is1 ? smem_u32(xs + s * 4096)
                                    : smem_u32(reinterpret_cast<uint8_t*>(SR.buf) + stage * kHSlice);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              d_umma(dt, d_umma_desc(a0 + kk * 256), d_umma_desc(b0 + kk * 256), (s0 | kk) != 0);
            d_commit(&empty[stage]);  // the stage is free once these MMAs are done
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1u;
            }
          }
          udesc[buf] = d;
          mbar_arrive(&dready[buf]);
          d_commit(&tfull[buf]);
        }
      }
      __syncwarp();
    } else if (warp >= 4) {
      const int q = warp & 3, m = 32 * q + lane;
      for (int seq = 0;; ++seq) {
        const int buf = seq & 1;
        mbar_wait(&dready[buf], (seq >> 1) & 1);
        const RoundDesc d = udesc[buf];
        if (d.n == 0) break;
        mbar_wait(&tfull[buf], (seq >> 1) & 1);
        d_fence_after();
        float v[16];
        d_tmem_ld16(tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * 16, v);
        d_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        const bool is1 = d.kind == 1;
        const int vu = is1 ? d.u0 : d.u0 - U1;
        const int RB = is1 ? RB1 : RB2;
        const int g = vu / RB, rr = (vu % RB) / kFfnWarps;
        if (is1) {
          // rows m: row block j = m / 16 holds gate (m % 16 < 8) and up of
          // h = 64 rr + 8 j + m % 8; the gate lane takes up from lane + 8
          const bool gate = (m & 15) < 8;
          const int hh = 64 * rr + 8 * (m >> 4) + (m & 7);
          __nv_bfloat16* hgp = P.hbuf + static_cast<size_t>(g) * 16 * P.Hp;
#pragma unroll
          for (int n = 0; n < 16; ++n) {
            const float up = __shfl_down_sync(kFull, v[n], 8);
            if (gate) hgp[cm16_index(n, hh)] = __float2bfloat16_rn(silu_f(v[n]) * up);
          }
          // the round's h (8 row blocks) out: the epilogue barrier orders the
          // 128 threads' stores before one cumulative release
          asm volatile("bar.sync 6, 128;" ::: "memory");
          if (warp == 4 && lane == 0)
            red_release_gpu_add_u64(&P.w1_slots[g], 8ull << (8 * ((rr >> 1) / w1_slot_q(P.Hp))));
        } else {
          float* yg = P.ybuf + static_cast<size_t>(g) * 16 * P.Dp + 128 * rr + m;
#pragma unroll
          for (int n = 0; n < 16; ++n) yg[static_cast<size_t>(n) * P.Dp] = v[n];
        }
      }
    }
  } else {
  bool in_w2 = false;
  for (int seq = 0;; ++seq) {
    mbar_wait(&full[stage], phase);  // the round's first stage carries its descriptor
    const RoundDesc d = rdesc[seq & (kRoundRing - 1)];
    if (d.n == 0) break;
    const bool sp = d.kind >= 3;  // split round (one unit, K over the warps)
    const bool is1 = d.kind == 1 || d.kind == 3;
    if (!is1 && !in_w2) {
      in_w2 = true;
      if (kDense) mbar_wait(plan_bar, 0);  // token lists of the W2 units
      if (threadIdx.x == 0) stamp(P, 1);
    }
    const int nsl = (is1 ? KT1 : KT2) / kKtPerSlot;
    const int nst = sp ? (nsl + kFfnWarps - 1) / kFfnWarps : d.se - d.sb;
    if (sp || warp < d.n) {
      const int uu = sp ? d.u0 : d.u0 + warp;
      Unit U;
      if (is1) {
        U.g = uu / RB1;
        U.rb = uu % RB1;
      } else {
        const int v = uu - U1;
        U.g = v / RB2;
        U.rb = v % RB2;
      }
      if (kDense && is1) {
        U.row0 = U.g * 16;
        U.rows = P.B;
      } else {
        U.row0 = PR->group_row0[U.g];
        U.rows = PR->group_rows[U.g];
      }
      U.ready = d.ready;
      U.nw = d.n;
      U.sb = sp ? 0 : d.sb;
      U.kp = d.kp;
      const int nbk = (U.rows + 7) >> 3;
      if (sp) {
        if (is1)
          dispatch_split<true, kDense>(nbk, P, PR, ring, full, empty, stage, phase, nst, U, xs,
                                       SR, sidx);
        else
          dispatch_split<false, kDense>(nbk, P, PR, ring, full, empty, stage, phase, nst, U, xs,
                                        SR, sidx);
      } else if (is1) {
        dispatch_unit<true, kDense>(nbk, P, PR, ring, full, empty, stage, phase, nst, U, xs, SR,
                                    sidx);
      } else if (kDense) {
        dispatch_w2_dense(nbk, P, PR, ring, full, empty, stage, phase, nst, U, xs, SR, sidx);
      } else {
        dispatch_unit<false, false>(nbk, P, PR, ring, full, empty, stage, phase, nst, U, xs, SR,
                                    sidx);
      }
    } else {
      skip_unit(full, empty, stage, phase, nst);
    }
  }
  }  // (mma.sync consumers)
  if (threadIdx.x == 0) stamp(P, 3);
  }

  // ---- grid-wide deterministic combine (moe_layer.hpp:148-155) ----
  // out[t][d] = sum_s w[t][s] * y_s[t][d] in set order. Every CTA publishes
  // its y writes (and, dense path, its token's plan) with one gpu-scope
  // release after a barrier of the consumer + router warps, waits until all
  // CTAs have, then combines a contiguous slice of the B x D outputs with all
  // slot loads of an output issued together.
  // The router warp (idle by now) arrives for the CTA and polls; meanwhile
  // the consumer warps fetch the plan side (set length, weights) of their
  // first output, so only the y loads remain after the barrier.
  constexpr int kComb = kFfnWarps * 32;  // combining threads (consumer warps)
  asm volatile("bar.sync 2, %0;" ::"r"(kComb + 32) : "memory");  // + router warp: all y stored
  const bool kShard = kFused && P.e_count < P.N;
  const int* eslot = reinterpret_cast<const int*>(rs + RL.eslot);
  const int* ssets = reinterpret_cast<const int*>(rs + RL.sets);
  const int64_t BD = static_cast<int64_t>(P.B) * P.D;
  const int64_t f0 = BD * blockIdx.x / gridDim.x, f1 = BD * (blockIdx.x + 1) / gridDim.x;
  constexpr int kSlotBatch = 16;
  // plan side of output f: y offsets (in floats, -1 = no contribution) and weights
  auto prep = [&](int64_t f, int& len, int (&yo)[kSlotBatch], float (&w)[kSlotBatch], int s0) {
    const int t = static_cast<int>(f / P.D), d = static_cast<int>(f % P.D);
    len = PR->set_len[t];
#pragma unroll
    for (int j = 0; j < kSlotBatch; ++j) {
      const int o = t * P.stride + s0 + j;
      // expert-parallel shard: this layer's partial sum over its experts
      const bool ok = s0 + j < len && (!kShard || eslot[ssets[o]] >= 0);
      // (MODE 6: y per (expert group, token): [G][16][Dp])
      yo[j] = ok ? (kUmma ? (eslot[ssets[o]] * 16 + t) * P.Dp + d : o * P.Dp + d) : -1;
      w[j] = ok ? PR->wts[o] : 0.0f;
    }
  };
  int len = 0, yo[kSlotBatch];
  float w[kSlotBatch];
  if (warp == kRouterWarp) {
    if (lane == 0) {
      stamp(P, 9);
      // Arrival counter of this launch: claims[2] / claims[5] by epoch parity.
      // The LAST CTA to arrive knows every CTA is past all other counter uses
      // (round claims, W1 release counts, prologue barrier) and resets them
      // here, with the other parity's arrival counter (its launch has
      // retired) and the new epoch: no exit round trip at the end of the
      // kernel. The arrival is acq_rel: it releases this CTA's y (cumulative
      // over the CTA barrier) and, for the last CTA, acquires everyone else's.
      int* done = claims + ((tag & 1u) ? 5 : 2);
      if (atom_add_acq_rel_gpu(done, 1) == static_cast<int>(gridDim.x) - 1) {
        for (int g = 0; g < G; ++g) P.w1_done[g] = 0;
        if (kDense)
          for (int g = 0; g < G; ++g) P.w1_slots[g] = 0ull;
        claims[0] = 0;
        claims[1] = 0;
        claims[3] = 0;
        claims[(tag & 1u) ? 2 : 5] = 0;
        claims[7] = static_cast<int>(tag);  // launch epoch + 1
      } else {
        while (ld_acquire_gpu(done) < static_cast<int>(gridDim.x)) {
        }
      }
      stamp(P, 10);
    }
  } else if (f0 + threadIdx.x < f1) {
    prep(f0 + threadIdx.x, len, yo, w, 0);
  }
  asm volatile("bar.sync 2, %0;" ::"r"(kComb + 32) : "memory");
  if (warp == kRouterWarp) return;
  if (kUmma && warp == 0) {  // (every tcgen05 op of the CTA is done: the barrier above)
    d_fence_after();
    const uint32_t* tslot = reinterpret_cast<const uint32_t*>(
        reinterpret_cast<const RoundDesc*>(
            reinterpret_cast<const uint64_t*>(xs + static_cast<size_t>(16) * P.Dp * 2) + 6) + 2);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tslot), "r"(32)
                 : "memory");
  }
  if (threadIdx.x == 0) stamp(P, 2);
  // (the local and the EP store are separate instantiations of the loop)
  auto combine = [&](auto store) {
    for (int64_t f = f0 + threadIdx.x; f < f1; f += kComb) {
      if (f != f0 + threadIdx.x) prep(f, len, yo, w, 0);
      float sum = 0.0f;
      for (int s0 = 0;;) {
        float y[kSlotBatch];
#pragma unroll
        for (int j = 0; j < kSlotBatch; ++j) y[j] = yo[j] >= 0 ? __ldcg(P.ybuf + yo[j]) : 0.0f;
        for (int kp = 1; kp < w2ks; ++kp) {  // W2 K parts, in part order
          const float* yk = P.ybuf + static_cast<size_t>(kp) * P.B * P.stride * P.Dp;
#pragma unroll
          for (int j = 0; j < kSlotBatch; ++j)
            if (yo[j] >= 0) y[j] += __ldcg(yk + yo[j]);
        }
#pragma unroll
        for (int j = 0; j < kSlotBatch; ++j)
          if (s0 + j < len) sum = fmaf(w[j], y[j], sum);
        s0 += kSlotBatch;
        if (s0 >= len) break;
        prep(f, len, yo, w, s0);
      }
      store(f, sum);
    }
  };
  if constexpr (!kEp) {
    combine([&](int64_t f, float v) { P.out[f] = v; });
    if (P.done_flag != nullptr) {
      // out lives in mapped host memory: once every CTA's slice is visible
      // system-wide, the last CTA raises the caller's flag (claims[6]: the
      // completion count, reset by that last CTA)
      asm volatile("bar.sync 2, %0;" ::"r"(kComb) : "memory");
      if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(&claims[6], 1) == static_cast<int>(gridDim.x) - 1) {
          claims[6] = 0;
          __threadfence_system();
          *reinterpret_cast<volatile int*>(P.done_flag) = 1;
        }
      }
    }
  } else {
    // Expert-parallel combine: token t's partial goes to its owner's receive
    // buffer (peer memory), slot [rank][t - owner * tpr], 4 outputs per store
    // (16-byte NVLink writes; D % 4 == 0 on this path) over the CTA's slice
    // of whole float4 quads; then the CTA adds the number of quads it wrote
    // for each owner whose tokens its slice touched (an owner expects
    // world x tpr x D / 4 per launch, whatever the grid)
    const EpPeers* ep = P.ep;
    const int tpr = ep->tpr, rank = ep->rank;
    const int64_t Q = BD >> 2;  // float4 quads
    const int64_t q0 = Q * blockIdx.x / gridDim.x, q1 = Q * (blockIdx.x + 1) / gridDim.x;
    for (int64_t qd = q0 + threadIdx.x; qd < q1; qd += kComb) {
      const int64_t f = qd << 2;
      const int t = static_cast<int>(f / P.D), d = static_cast<int>(f % P.D);
      const int len = PR->set_len[t];
      float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int j = 0; j < len; ++j) {
        const int o = t * P.stride + j;
        if (eslot[ssets[o]] < 0) continue;  // (an expert this shard does not hold)
        const float w = PR->wts[o];
        float4 y = __ldcg(reinterpret_cast<const float4*>(P.ybuf + static_cast<size_t>(o) * P.Dp + d));
        for (int kp = 1; kp < w2ks; ++kp) {
          const float4 yk = __ldcg(reinterpret_cast<const float4*>(
              P.ybuf + (static_cast<size_t>(kp) * P.B * P.stride + o) * P.Dp + d));
          y.x += yk.x;
          y.y += yk.y;
          y.z += yk.z;
          y.w += yk.w;
        }
        sum.x = fmaf(w, y.x, sum.x);
        sum.y = fmaf(w, y.y, sum.y);
        sum.z = fmaf(w, y.z, sum.z);
        sum.w = fmaf(w, y.w, sum.w);
      }
      const int owner = t / tpr;
      *reinterpret_cast<float4*>(
          ep->recv[owner] + (static_cast<size_t>(rank) * tpr + (t - owner * tpr)) * P.D + d) = sum;
    }
    // this CTA's remote stores are issued (all combining threads), made
    // visible system-wide, then counted at the owners its slice covers
    asm volatile("bar.sync 2, %0;" ::"r"(kComb) : "memory");
    if (threadIdx.x == 0 && q1 > q0) {
      __threadfence_system();
      const int64_t qpo = static_cast<int64_t>(tpr) * P.D / 4;  // quads per owner
      for (int o = static_cast<int>(q0 / qpo); o <= static_cast<int>((q1 - 1) / qpo); ++o) {
        const int64_t n = min(q1, (o + 1) * qpo) - max(q0, o * qpo);
        atomicAdd_system(ep->cnt[o], static_cast<int>(n));
      }
    }
  }
  if (threadIdx.x == 0) stamp(P, 15);
}

// Owner side of the peer-memory EP combine (one CTA): cnt[0] counts the
// arriving CTAs of all ranks, cnt[1] the arrivals already consumed; wait
// until this launch's `per_launch` arrivals are in, then out[i] = sum over
// source ranks in rank order (deterministic). The target lives on the device,
// so the pair (partial decode, combine) can be captured in a CUDA graph.
__global__ void __launch_bounds__(1024)
    k_ep_sum(const float* __restrict__ recv, int* __restrict__ cnt, int per_launch, int world,
             int n, float* __restrict__ out) {
  if (threadIdx.x == 0) {
    const uint32_t target = static_cast<uint32_t>(cnt[1]) + static_cast<uint32_t>(per_launch);
    uint32_t v;
    do {  // (wrap-around safe: both counters only grow)
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
    } while (static_cast<int32_t>(v - target) < 0);
    cnt[1] = static_cast<int>(target);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    float s = 0.0f;
    for (int r = 0; r < world; ++r) s += __ldcg(recv + static_cast<size_t>(r) * n + i);
    out[i] = s;
  }
}

// ---------------------------------------------------------------------------
// SIMT FFN for f32 / f64 layers (reference layout weights).
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T silu_t(T z) {
  return z / (T(1) + exp(-z));
}

// h[row][h] = silu(x Wg) * (x Wu) for the group's rows; thread per h column,
// 8 rows per pass, sequential sum over d (the reference's dot order).
template <typename T>
__global__ void __launch_bounds__(128)
    k_simt_gateup(const T* __restrict__ x, int D, int H, const T* __restrict__ wg,
                  const T* __restrict__ wu, const int32_t* __restrict__ row_tok,
                  const int32_t* __restrict__ group_a, const int32_t* __restrict__ group_row0,
                  const int32_t* __restrict__ group_rows, const FfnHeader* __restrict__ hdr,
                  T* __restrict__ hbuf) {
  const int g = blockIdx.y;
  if (g >= hdr->n_groups) return;
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= H) return;
  const int e = group_a[g], row0 = group_row0[g], rows = group_rows[g];
  const T* Wg = wg + static_cast<size_t>(e) * D * H;
  const T* Wu = wu + static_cast<size_t>(e) * D * H;
  for (int r0 = 0; r0 < rows; r0 += 8) {
    T ag[8], au[8];
    const T* xr[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      ag[r] = au[r] = T(0);
      xr[r] = r0 + r < rows ? x + static_cast<size_t>(row_tok[row0 + r0 + r]) * D : nullptr;
    }
    for (int d = 0; d < D; ++d) {
      const T vg = Wg[static_cast<size_t>(d) * H + h];
      const T vu = Wu[static_cast<size_t>(d) * H + h];
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (xr[r]) {
          const T xv = xr[r][d];
          ag[r] += xv * vg;
          au[r] += xv * vu;
        }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (xr[r]) hbuf[static_cast<size_t>(row0 + r0 + r) * H + h] = silu_t(ag[r]) * au[r];
  }
}

template <typename T>
__global__ void __launch_bounds__(128)
    k_simt_down(int D, int H, const T* __restrict__ wd, const int32_t* __restrict__ row_tok,
                const int32_t* __restrict__ row_slot, const int32_t* __restrict__ group_a,
                const int32_t* __restrict__ group_row0, const int32_t* __restrict__ group_rows,
                const FfnHeader* __restrict__ hdr, const T* __restrict__ hbuf, int stride,
                T* __restrict__ ybuf) {
  const int g = blockIdx.y;
  if (g >= hdr->n_groups) return;
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= D) return;
  const int e = group_a[g], row0 = group_row0[g], rows = group_rows[g];
  const T* Wd = wd + static_cast<size_t>(e) * H * D;
  for (int r0 = 0; r0 < rows; r0 += 8) {
    T acc[8];
    const T* hr[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      acc[r] = T(0);
      hr[r] = r0 + r < rows ? hbuf + static_cast<size_t>(row0 + r0 + r) * H : nullptr;
    }
    for (int h = 0; h < H; ++h) {
      const T w = Wd[static_cast<size_t>(h) * D + d];
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (hr[r]) acc[r] += hr[r][h] * w;
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (hr[r]) {
        const int row = row0 + r0 + r;
        ybuf[(static_cast<size_t>(row_tok[row]) * stride + row_slot[row]) * D + d] = acc[r];
      }
  }
}

// out[t][d] = sum_j w[t][j] * double(y[t][j][d]) in set order, fp64
// (moe_layer.hpp:153: out.row(i) += w[j] * expert_forward(...)). y rows are
// ldy apart; alias (optional, [B][stride]): slot j reads the y of slot
// alias[t][j] (a duplicated expert in a caller plan is computed once and
// accumulated once per occurrence, as the reference does).
template <typename T>
__global__ void k_simt_combine(int B, int D, int ldy, int stride,
                               const int32_t* __restrict__ set_len, const double* __restrict__ w,
                               const int32_t* __restrict__ alias, const T* __restrict__ ybuf,
                               double* __restrict__ out) {
  const size_t total = static_cast<size_t>(B) * D;
  for (size_t f = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(f / D), d = static_cast<int>(f % D);
    double acc = 0.0;
    for (int j = 0; j < set_len[t]; ++j) {
      const size_t o = static_cast<size_t>(t) * stride + j;
      const int js = alias ? alias[o] : j;
      acc = __dadd_rn(acc, __dmul_rn(w[o], static_cast<double>(
                                               ybuf[(static_cast<size_t>(t) * stride + js) * ldy + d])));
    }
    out[f] = acc;
  }
}

template <typename S, typename T>
__global__ void k_cast(const S* __restrict__ src, size_t n, T* __restrict__ dst) {
  for (size_t f = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[f] = static_cast<T>(src[f]);
}

}  // namespace oea_dev

namespace oea_host {

using namespace oea_dev;

size_t ffn_bf16_smem_bytes() {
  return kStages * kStageBytes + 2 * kStages * sizeof(uint64_t) + kRoundRing * sizeof(RoundDesc) +
         sizeof(PlanRef) + 16 + kSplitRedBytes;
}
size_t ffn_btile_bytes() { return kBTileBytes; }

size_t ffn_route_smem_bytes(int B, int Np, int stride) {
  return route_smem_layout(B, Np, stride).total;
}

size_t ffn_dense_xs_bytes(int Dp) { return static_cast<size_t>(16) * (Dp * 2 + 32); }

int ffn_bf16_launch(oea_ctx* ctx, const oea_layer* L, int B, int stride, const FfnBuffers& fb,
                    bool pdl, cudaStream_t s) {
  FfnParams P;
  P.w1 = static_cast<const uint4*>(L->w1);
  P.w2 = static_cast<const uint4*>(L->w2);
  P.xpad = static_cast<const __nv_bfloat16*>(fb.x);
  P.D = L->D;
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
  P.w1_done = fb.counters;
  P.w1_slots = reinterpret_cast<unsigned long long*>(fb.slice_done);
  {
    const int ns = L->Hp >> 7, q = (ns + kW1Slots - 1) / kW1Slots;
    P.w1_full = 0ull;
    for (int c = 0; c * q < ns; ++c)
      P.w1_full |= static_cast<unsigned long long>(16 * (std::min(ns, (c + 1) * q) - c * q)) << (8 * c);
  }
  P.claims = fb.counters + fb.max_groups;
  P.hbuf = static_cast<__nv_bfloat16*>(fb.hbuf);
  P.ybuf = static_cast<float*>(fb.ybuf);
  P.set_len = fb.set_len;
  P.wts = fb.weights_f32;
  P.out = static_cast<float*>(fb.out);
  P.trace = fb.trace;
  P.mode = fb.mode;
  P.xs_row = L->Dp * 2 + 32;
  // split rounds measured slower than 8-unit rounds at small T (per-round
  // reduction overhead, tools/trace_ffn.py): opt-in for experiments
  P.split_ok = getenv("OEA_SPLIT") != nullptr;
  P.x_stage = fb.x_stage;
  P.done_flag = fb.done_flag;
  P.ep = fb.ep;
  {
    // ~32 MiB in total, about what HBM delivers while the prologue routes
    // (measured C1, N=128: 128 KiB per expert saves ~1.3 us, 224-288 KiB
    // ~2.2 us, 320 KiB less again; issuing it before the gate GEMV is slower)
    // Round 2: full layers use the logit-guided prefetch instead (below,
    // prefetch_w1_heads); the blind heads stay for EP shards (no guess: a
    // shard's CTAs compute other experts' logits than the ones it holds)
    static const int pf = getenv("OEA_PREFETCH_KB") ? atoi(getenv("OEA_PREFETCH_KB")) : -1;
    P.prefetch_bytes = pf >= 0 ? pf * 1024
                       : L->n_local < L->N ? ((32 << 20) / max(L->n_local, 1)) & ~(32 * 1024 - 1)
                                           : 0;
  }
  {
    // (issuing it before the wait was measured slower: the CTAs only become
    // resident as the previous grid's exit, so it just delays the GEMV's loads)
    static const bool early = getenv("OEA_PF_EARLY") != nullptr;
    P.pf_early = early && !fb.x_stage;
  }
  {
    static const int ks = getenv("OEA_W2_KSPLIT") ? atoi(getenv("OEA_W2_KSPLIT")) : kW2KSplit;
    P.w2_ks = std::max(1, std::min(ks, kW2KSplitMax));
  }
  {
    static const int hi = getenv("OEA_PF_HI_KB") ? atoi(getenv("OEA_PF_HI_KB")) : 1536;
    static const int lo = getenv("OEA_PF_LO_KB") ? atoi(getenv("OEA_PF_LO_KB")) : 0;
    static const int tau = getenv("OEA_PF_TAU") ? atoi(getenv("OEA_PF_TAU")) : 215;
    P.pf_guess_hi = hi * 1024;
    P.pf_guess_lo = lo * 1024;
    P.pf_tau = tau / 100.0f;
    static const int hg = getenv("OEA_HOST_PF_GUESS") ? atoi(getenv("OEA_HOST_PF_GUESS")) : 1;
    P.host_pf_guess = hg;
  }
  P.pf_w1u = static_cast<const uint8_t*>(fb.pf_w1u);
  P.w1u = static_cast<const uint8_t*>(L->w1u);
  P.w2u = static_cast<const uint8_t*>(L->w2u);
  P.w1u_stride = static_cast<size_t>(2 * L->Hp) * L->Dp * 2;
  P.w2u_stride = static_cast<size_t>(L->Dp) * L->Hp * 2;
  P.pf_w1u_stride = static_cast<size_t>(2 * L->Hp) * L->Dp * 2;
  {
    static const int mb = getenv("OEA_BIG_PF_MB") ? atoi(getenv("OEA_BIG_PF_MB")) : 32;
    P.pf_total = static_cast<size_t>(mb) << 20;
  }
  {
    static const int r0 = getenv("OEA_R0") ? atoi(getenv("OEA_R0")) : 2;
    P.r0 = fb.dense ? r0 : 0;
  }
  P.compact_in_kernel = fb.compact_in_kernel;
  P.xg = static_cast<uint8_t*>(fb.xg);
  P.xg_rg = fb.xg_rg;
  P.e_begin = L->e_begin;
  P.e_count = L->n_local;
  P.router_t = static_cast<const uint4*>(L->router_t);
  P.router_frag = static_cast<const uint4*>(L->router);
  P.x_in = fb.x_in;
  P.xpad_out = fb.xpad_out;
  P.logits = fb.logits;
  P.xlog = fb.xlog;
  P.xuni = fb.xuni;
  P.xplan = fb.xplan;
  P.mask = fb.mask;
  P.N = L->N;
  P.Np = L->Np;
  P.cfg = fb.cfg;
  P.x_sets = fb.x_sets;
  P.x_set_len = fb.x_set_len;
  P.x_w32 = fb.x_w32;
  P.x_w64 = fb.x_w64;
  P.x_loads = fb.x_loads;
  P.x_active = fb.x_active;
  P.x_active_count = fb.x_active_count;
  P.x_total_load = fb.x_total_load;
  P.x_phase1_n = fb.x_phase1_n;
  P.x_base_union = fb.x_base_union;
  P.x_base_union_count = fb.x_base_union_count;
  P.x_hdr = fb.x_hdr;

  const size_t smem = ffn_bf16_smem_bytes() +
                      (fb.fused ? ffn_route_smem_bytes(B, L->Np, stride) : 0) +
                      (fb.dense ? ffn_dense_xs_bytes(L->Dp) : 0) +
                      (fb.dense || fb.route_only ? 0 : ffn_btile_bytes());
  if (fb.ep != nullptr && (!fb.fused || fb.route_only))
    return oea_set_error(ctx, OEA_ERR_INVALID_ARGUMENT, "moe_decode_ep: needs the fused path");
  const int mode = fb.route_only ? 3
                   : fb.dense   ? (fb.ep ? 5 : fb.umma_dense ? 6 : 2)
                   : fb.fused   ? (fb.ep ? 4 : 1)
                                : 0;
  auto kern = mode == 6   ? k_ffn_bf16<6>
              : mode == 5 ? k_ffn_bf16<5>
              : mode == 4 ? k_ffn_bf16<4>
              : mode == 3 ? k_ffn_bf16<3>
              : mode == 2 ? k_ffn_bf16<2>
              : mode == 1 ? k_ffn_bf16<1>
                          : k_ffn_bf16<0>;
  if (static_cast<int>(smem) > ctx->ffn_smem_set[mode]) {  // once per size, not per launch
    OEA_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
    ctx->ffn_smem_set[mode] = static_cast<int>(smem);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctx->num_sms);
  cfg.blockDim = dim3(kFfnThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  // The kernel is persistent and spins on grid-wide counters (union
  // exchange, W1 release, combine arrival): every CTA must be resident at
  // once. The cooperative attribute makes the driver guarantee that (or fail
  // the launch loudly, e.g. under an MPS SM limit), instead of a CTA waiting
  // for an SM held by a concurrent kernel that may itself wait on this one.
  // PDL only as the router kernel's dependent (two-kernel path); the fused
  // launch carries no programmatic-serialization attribute at all.
  static const bool coop = getenv("OEA_NO_COOP") == nullptr;
  // Fused launches are programmatic dependents of the previous kernel in the
  // stream (see the kernel head): launch latency and setup overlap its tail.
  static const bool fused_pdl = getenv("OEA_NO_PDL") == nullptr;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (coop) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  if (pdl || (fb.fused && fused_pdl)) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  OEA_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, kern, P));
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

int ep_sum_launch(oea_ctx* ctx, const float* recv, int* cnt, int per_launch, int world, int n,
                  float* out, cudaStream_t s) {
  k_ep_sum<<<1, 1024, 0, s>>>(recv, cnt, per_launch, world, n, out);
  OEA_LAUNCHED(ctx);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? OEA_OK : oea_check_cuda(ctx, e, "k_ep_sum");
}

// Host-path graph replays (capi.cu decode_host_graph) patch a captured fused
// launch's parameter block: the caller's x (mapped host rows) and out.
size_t ffn_params_bytes() { return sizeof(FfnParams); }
void ffn_params_set_io(void* params, const void* x_in, void* out) {
  auto* P = static_cast<FfnParams*>(params);
  P->x_in = static_cast<const __nv_bfloat16*>(x_in);
  P->out = static_cast<float*>(out);
}

template <typename T>
static int simt_impl(oea_ctx* ctx, const oea_layer* L, int B, int stride, const FfnBuffers& fb,
                     int max_groups, cudaStream_t s) {
  const int D = L->D, H = L->H;
  dim3 g1((H + 127) / 128, max_groups), g2((D + 127) / 128, max_groups);
  k_simt_gateup<T><<<g1, 128, 0, s>>>(static_cast<const T*>(fb.x), D, H,
                                      static_cast<const T*>(L->w1), static_cast<const T*>(L->w_up),
                                      fb.row_tok, fb.group_a, fb.group_row0, fb.group_rows, fb.hdr,
                                      static_cast<T*>(fb.hbuf));
  OEA_LAUNCHED(ctx);
  k_simt_down<T><<<g2, 128, 0, s>>>(D, H, static_cast<const T*>(L->w2), fb.row_tok, fb.row_slot,
                                    fb.group_a, fb.group_row0, fb.group_rows, fb.hdr,
                                    static_cast<const T*>(fb.hbuf), stride,
                                    static_cast<T*>(fb.ybuf));
  OEA_LAUNCHED(ctx);
  const size_t total = static_cast<size_t>(B) * D;
  const int blocks = static_cast<int>((total + 255) / 256 > 4096 ? 4096 : (total + 255) / 256);
  k_simt_combine<T><<<blocks, 256, 0, s>>>(B, D, D, stride, fb.set_len, fb.weights_f64,
                                           fb.alias, static_cast<const T*>(fb.ybuf),
                                           static_cast<double*>(fb.out));
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

// bf16 layers, caller plan with duplicated experts: the fp64 set-order
// combine over the FFN's fp32 y ([B][stride][Dp]) with the slot aliases.
int combine_alias_f32_launch(oea_ctx* ctx, int B, int D, int Dp, int stride, const FfnBuffers& fb,
                             cudaStream_t s) {
  const size_t total = static_cast<size_t>(B) * D;
  const int blocks = static_cast<int>((total + 255) / 256 > 4096 ? 4096 : (total + 255) / 256);
  k_simt_combine<float><<<blocks, 256, 0, s>>>(B, D, Dp, stride, fb.set_len, fb.weights_f64,
                                               fb.alias, static_cast<const float*>(fb.ybuf),
                                               static_cast<double*>(fb.out));
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

int ffn_simt_launch(oea_ctx* ctx, const oea_layer* L, int B, int stride, const FfnBuffers& fb,
                    int max_groups, cudaStream_t s) {
  if (L->dtype == OEA_DTYPE_F64) return simt_impl<double>(ctx, L, B, stride, fb, max_groups, s);
  return simt_impl<float>(ctx, L, B, stride, fb, max_groups, s);
}

int cast_f64_launch(oea_ctx* ctx, const double* src, size_t n, int dst_dtype, void* dst,
                    cudaStream_t s) {
  const int blocks = static_cast<int>((n + 255) / 256 > 4096 ? 4096 : (n + 255) / 256 + 0);
  if (dst_dtype == OEA_DTYPE_F64)
    k_cast<double, double><<<blocks > 0 ? blocks : 1, 256, 0, s>>>(src, n, static_cast<double*>(dst));
  else
    k_cast<double, float><<<blocks > 0 ? blocks : 1, 256, 0, s>>>(src, n, static_cast<float*>(dst));
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

}  // namespace oea_host
