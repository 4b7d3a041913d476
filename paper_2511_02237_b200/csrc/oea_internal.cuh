// oea_internal.cuh — shared definitions for the sm_100a OEA kernels and the
// host runtime behind include/oea_cuda.h.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "oea_cuda.h"

namespace oea_dev {

// ---------------------------------------------------------------------------
// Tiling constants of the tensor-core decode path.
// ---------------------------------------------------------------------------
constexpr int kTile = 16;              // mma.m16n8k16: 16 rows x 16 k per A tile
constexpr int kTileBytes = 512;        // one bf16 A tile, fragment-ordered
constexpr int kNb = 8;                 // tokens per n-block (mma n = 8)
constexpr int kTokGroup = 64;          // tokens per FFN unit (<= 8 n-blocks)
constexpr int kFfnWarps = 8;           // consumer warps per FFN CTA
constexpr int kKtPerSlot = 8;          // k-tiles per warp per pipeline stage
constexpr int kSlotBytes = kKtPerSlot * kTileBytes;   // 4 KiB
constexpr int kStageBytes = kFfnWarps * kSlotBytes;   // 32 KiB
#ifndef OEA_FFN_STAGES
#define OEA_FFN_STAGES 4
#endif
constexpr int kStages = OEA_FFN_STAGES;               // 4 x 32 KiB ring (tools/stream_bench.cu)
constexpr int kPadD = 128;             // D padded so D/16 % 8 == 0
constexpr int kPadH = 128;             // H padded so H/16 % 8 == 0
constexpr int kRouterCluster = 8;      // CTAs in the fused-router cluster
constexpr int kRouterThreads = 512;
constexpr int kRouterTokChunk = 64;    // tokens per GEMV pass in the router
constexpr int kMaxFusedB = 256;        // fused decode batch limit
constexpr int kMaxFusedN = 256;        // fused router expert limit (Np <= 256)
// Dense decode (B <= 16): W2 rounds split into this many K parts (the tail
// of the weight stream is one part long instead of one round); y then holds
// one [B][stride][Dp] plane per part.
constexpr int kW2KSplit = 1;  // (2-6 measured slower at C1: per-round B-operand restarts, y traffic)
constexpr int kW2KSplitMax = 4;
constexpr int kMaxEpWorld = 8;  // expert-parallel group size of the peer-memory combine
// Peer table of the EP combine (device memory, read by the combine stage).
struct EpPeers {
  float* recv[kMaxEpWorld];
  int* cnt[kMaxEpWorld];
  int world, rank, tpr;
};
constexpr int kMaxRouteN = 1024;       // route_f64 expert limit
// Debug timeline buffer (OEA_FFN_TRACE=1): the router kernels' legacy area,
// then one [grid][16] stamp region per FFN launch, 16 launches deep (indexed
// by the launch epoch); word kTraceInfo of a region = the launch's T.
constexpr int kTraceLegacy = 8192;
constexpr int kTraceLaunches = 16;
constexpr int kTracePerLaunch = 16384;
constexpr int kTraceRoundLog = 4096;  // per-CTA producer round log inside a launch region
constexpr int kTraceRounds = 24;
constexpr int kTraceInfo = 2400;
constexpr size_t kTraceWords = kTraceLegacy + static_cast<size_t>(kTraceLaunches) * kTracePerLaunch;

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

// Device-side routing configuration (resolved).
struct Cfg {
  int mode, k, k0;
  double p;
  int k_max, max_p, cap;
  int limit;   // final set-size cap of phase 2 (k_max or k_max + 1)
  int stride;  // set stride used in workspace
};

// FFN plan header written by the router/compaction kernel, read by the FFN.
struct FfnHeader {
  int n_groups;   // token groups (expert, <=64 tokens)
  int T;          // active experts
  int total_load;
  int n_rows;     // padded rows
  int err_token;  // domain error token (INT_MAX = none)
  int pad[3];
};

// Single-launch route scratch (routing.cu, RouteScratch): a 32-byte header
// (the launch epoch) + 4 tagged union words per CTA.
constexpr size_t kRouteScratchBytes = 64 * 1024;

}  // namespace oea_dev

// ---------------------------------------------------------------------------
// Host-side objects.
// ---------------------------------------------------------------------------
struct oea_ctx {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  std::string last_error;
  int64_t launches = 0;
  // Workspace arena (grown on demand outside the timed path).
  void* ws = nullptr;
  size_t ws_bytes = 0;
  // Pinned staging for *_host entry points.
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // Last decode, for oea_last_plan_host.
  int last_B = 0, last_N = 0, last_stride = 0, last_kind = 0;  // kind 1 = fused bf16, 2 = f64 route
  // Debug instrumentation of the FFN (env OEA_FFN_TRACE=1 / OEA_FFN_MODE=n).
  unsigned long long* ffn_trace = nullptr;
  void* route_scratch = nullptr;  // single-launch route: epoch + per-CTA tagged union words
  int ffn_mode = 0;
  // dynamic shared memory already allowed per k_ffn_bf16<MODE> on this device
  int ffn_smem_set[7] = {0, 0, 0, 0, 0, 0, 0};
  // EP peer tables uploaded so far (device copies; matched by content)
  void* ep_tables = nullptr;
  std::vector<oea_dev::EpPeers> ep_host_tables;
};

struct oea_layer {
  oea_ctx* ctx = nullptr;
  int D = 0, H = 0, N = 0, dtype = OEA_DTYPE_BF16;
  // Expert-parallel shard: this layer holds experts [e_begin, e_begin + n_local)
  // of the N routed by its (full) router; a full layer has e_begin 0, n_local N.
  int e_begin = 0, n_local = 0;
  int Dp = 0, Hp = 0, Np = 0;  // padded (bf16 fragment layout)
  // bf16: fragment-ordered weights. f32/f64: reference layout.
  void* router = nullptr;      // bf16: [Np/16][Dp/16][32][8]; else [D][N]
  void* router_t = nullptr;    // bf16 only: [Np][Dp] expert-major copy (fused gate GEMV)
  void* w1 = nullptr;          // bf16: [N][Hp/8][Dp/16][32][8] (gate|up); else gate [N][D][H]
  void* w_up = nullptr;        // f32/f64 only: [N][D][H]
  void* w2 = nullptr;          // bf16: [N][Dp/16][Hp/16][32][8]; else down [N][H][D]
  size_t router_bytes = 0, w1_bytes = 0, w2_bytes = 0, up_bytes = 0;
  // bf16, large batches (B > 64): the expert weights again in the canonical
  // K-major UMMA layout for the tcgen05 FFN (umma_ffn.cu), made on first use;
  // umma_stale: the weights changed since (re-packed in place on next use)
  void* w1u = nullptr;
  void* w2u = nullptr;
  int umma_stale = 0;
};

struct oea_graph {
  oea_ctx* ctx = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int kernels = 0;  // kernels launched per graph launch (launch accounting)
};

// Status helpers (defined in capi.cu).
int oea_set_error(oea_ctx* ctx, int code, const std::string& msg);
int oea_check_cuda(oea_ctx* ctx, cudaError_t e, const char* what);

#define OEA_CUDA_TRY(ctx, expr)                                   \
  do {                                                            \
    cudaError_t oea_e_ = (expr);                                  \
    if (oea_e_ != cudaSuccess) return oea_check_cuda(ctx, oea_e_, #expr); \
  } while (0)

// Launch accounting + error check after every kernel launch.
#define OEA_LAUNCHED(ctx)                                           \
  do {                                                              \
    (ctx)->launches++;                                              \
    cudaError_t oea_e_ = cudaGetLastError();                        \
    if (oea_e_ != cudaSuccess) return oea_check_cuda(ctx, oea_e_, "kernel launch"); \
  } while (0)

// ---------------------------------------------------------------------------
// Kernel-family entry points (host wrappers), implemented per .cu file.
// ---------------------------------------------------------------------------
namespace oea_host {

// routing.cu — K1 family on fp64 scores. All device pointers.
struct RouteBuffers {
  const double* scores;
  const uint8_t* mask;        // may be null
  int32_t* order;             // [B*N] workspace (or caller), written unless order_given
  int32_t* t;                 // [B] may be null
  int32_t* n;                 // [B] workspace
  uint32_t* union_bits;       // [ceil(N/32)] workspace
  int32_t* sets;              // [B*stride]
  int32_t* set_len;           // [B]
  double* weights;            // [B*stride] may be null
  float* weights_f32;         // may be null
  int32_t* loads;             // [N] workspace
  int32_t* active_union;      // [N]
  int32_t* active_count;      // [1]
  int64_t* total_load;        // [1]
  int32_t* base_union;        // [N] may be null
  int32_t* base_union_count;  // [1] may be null
  int32_t* err_token;         // [1]
};
int route_f64_launch(oea_ctx* ctx, const oea_dev::Cfg& cfg, int B, int N,
                     const RouteBuffers& rb, bool order_given, bool run_phase1,
                     int set_mode, bool n_given, cudaStream_t s, int R = 1,
                     const int32_t* seg = nullptr);
// Fast path of route_f64 (p == 1, max_p >= N, N <= 128, no full order
// requested): top-m picks instead of a full sort; same results bit for bit.
bool route_fast_ok(const oea_dev::Cfg& cfg, int N, bool need_order);
int route_f64_fast_launch(oea_ctx* ctx, const oea_dev::Cfg& cfg, int B, int N,
                          const RouteBuffers& rb, int set_mode, cudaStream_t s, int R = 1,
                          const int32_t* seg = nullptr);
int union_from_list_launch(oea_ctx* ctx, const int32_t* list, int count, int N, uint32_t* bits,
                           cudaStream_t s);

// router_scores in fp64 (f32/f64 layers): scores [B][N].
int router_scores_launch(oea_ctx* ctx, const oea_layer* L, const double* x, int B,
                         double* logits_ws, double* scores, cudaStream_t s);

// compaction of a device plan into FFN rows/groups (SIMT path and drop-in).
struct CompactBuffers {
  const int32_t* sets;
  const int32_t* set_len;
  int32_t* row_tok;
  int32_t* row_slot;
  int32_t* group_a;      // [G] expert id per group
  int32_t* group_row0;   // [G]
  int32_t* group_rows;   // [G] real rows
  oea_dev::FfnHeader* hdr;
  int32_t* counters;     // zeroed: [G + Dp/16 + 1]
  int n_counters;
  int32_t* loads_out = nullptr;  // [N] per-expert loads (exported plan), or null
  int64_t* total_load = nullptr;
};
int compact_launch(oea_ctx* ctx, int B, int N, int stride, const CompactBuffers& cb,
                   uint32_t* tokbits, int32_t* active_union, int32_t* active_count,
                   cudaStream_t s);
int cast_f64_launch(oea_ctx* ctx, const double* src, size_t n, int dst_dtype, void* dst,
                    cudaStream_t s);

// expert_ffn.cu
struct FfnBuffers {
  const void* x;           // bf16 [B][Dp] padded (bf16 path) / T [B][D] (simt)
  const int32_t* row_tok;
  const int32_t* row_slot;
  const int32_t* group_a;
  const int32_t* group_row0;
  const int32_t* group_rows;
  const oea_dev::FfnHeader* hdr;
  int32_t* counters;       // [max_groups] w1_done then [Dp/16] combine counters
  int32_t* slice_done = nullptr;  // dense path: [max_groups] u64, 8-bit W1 K-slot counts
  int max_groups;
  void* hbuf;              // [rows][Hp] (bf16) / [rows][H] (T)
  void* ybuf;              // [B][stride][Dp] f32 / [B][stride][D] T
  const int32_t* set_len;
  const float* weights_f32;
  const double* weights_f64;
  void* out;               // [B][D] f32 (bf16 path) / f64 (simt)
  const int32_t* alias = nullptr;       // [B][stride] y slot per plan slot (duplicates), or null
  unsigned long long* trace = nullptr;  // debug timeline (OEA_FFN_TRACE)
  int mode = 0;                         // debug mode (OEA_FFN_MODE)
  // Fused single-launch decode (B <= 64): the FFN grid computes the logits
  // (gate GEMV), routes the batch in every CTA and exports the plan (CTA 0).
  int fused = 0;
  int dense = 0;                        // dense-over-batch FFN (fused, B <= 16)
  int route_only = 0;                   // plan only (B > 64): k_compact + FFN follow
  const __nv_bfloat16* x_in = nullptr;  // [B][D] caller tokens
  __nv_bfloat16* xpad_out = nullptr;    // [B][Dp] when D != Dp (or x_stage)
  int x_stage = 0;                      // x_in is mapped host memory (staged in-kernel)
  int* done_flag = nullptr;             // mapped host flag set to 1 when out is on the host
  const oea_dev::EpPeers* ep = nullptr;  // peer-memory EP combine (device table), or null
  int compact_in_kernel = 0;            // route-only: the compaction in the same launch
  const void* pf_w1u = nullptr;         // route-only: the tcgen05 FFN's W1 copy to prefetch (or null)
  int umma_dense = 0;                   // dense decode on tcgen05 (MODE 6; the layer's UMMA copy)
  void* xg = nullptr;                   // ... and the tcgen05 FFN's gathered rows (or null)
  int xg_rg = 0;
  float* logits = nullptr;              // [B][Np]
  unsigned long long* xlog = nullptr;   // tagged exchange words (fused path)
  unsigned long long* xuni = nullptr;
  unsigned long long* xplan = nullptr;
  const uint8_t* mask = nullptr;
  oea_dev::Cfg cfg{};
  int32_t* x_sets = nullptr;
  int32_t* x_set_len = nullptr;
  float* x_w32 = nullptr;
  double* x_w64 = nullptr;
  int32_t* x_loads = nullptr;
  int32_t* x_active = nullptr;
  int32_t* x_active_count = nullptr;
  int64_t* x_total_load = nullptr;
  int32_t* x_phase1_n = nullptr;
  int32_t* x_base_union = nullptr;
  int32_t* x_base_union_count = nullptr;
  oea_dev::FfnHeader* x_hdr = nullptr;
};
size_t ffn_route_smem_bytes(int B, int Np, int stride);
size_t ffn_bf16_smem_bytes();
int gen_scores_launch(oea_ctx* ctx, const oea_score_gen_cfg& c, int step0, int nsteps,
                      double* out, cudaStream_t s);
int ep_sum_launch(oea_ctx* ctx, const float* recv, int* cnt, int per_launch, int world, int n,
                  float* out, cudaStream_t s);
size_t ffn_params_bytes();
void ffn_params_set_io(void* params, const void* x_in, void* out);
size_t ffn_btile_bytes();
size_t ffn_dense_xs_bytes(int Dp);
// tcgen05 grouped FFN (umma_ffn.cu)
int layer_prepare_umma(oea_ctx* ctx, oea_layer* L, cudaStream_t s);
void layer_drop_umma(oea_layer* L);
int ffn_umma_launch(oea_ctx* ctx, const oea_layer* L, int B, int stride, const FfnBuffers& fb,
                    void* xg, int RG, cudaStream_t s, bool gathered = false);
int ffn_bf16_launch(oea_ctx* ctx, const oea_layer* L, int B, int stride,
                    const FfnBuffers& fb, bool pdl, cudaStream_t s);
int ffn_simt_launch(oea_ctx* ctx, const oea_layer* L, int B, int stride,
                    const FfnBuffers& fb, int max_rows, cudaStream_t s);
int combine_alias_f32_launch(oea_ctx* ctx, int B, int D, int Dp, int stride, const FfnBuffers& fb,
                             cudaStream_t s);

// router_fused.cu — K2+K3 for bf16 layers.
struct FusedRouterBuffers {
  const __nv_bfloat16* x;   // [B][D] caller
  const uint8_t* mask;      // may be null
  __nv_bfloat16* xpad;      // [B][Dp]
  float* logits;            // [B][Np]
  int32_t* order;           // [B][Np]
  int32_t* sets;            // [B][stride]
  int32_t* set_len;
  float* weights_f32;
  double* weights_f64;
  int32_t* loads;
  int32_t* active_union;
  int32_t* active_count;
  int64_t* total_load;
  int32_t* row_tok;
  int32_t* row_slot;
  int32_t* group_a;
  int32_t* group_row0;
  int32_t* group_rows;
  oea_dev::FfnHeader* hdr;
  int32_t* counters;
  int n_counters;
  float* out;               // zeroed here when no expert is active
  int32_t* phase1_n;        // [B] may be null
  int32_t* base_union;      // [N] may be null
  int32_t* base_union_count;
  unsigned long long* trace = nullptr;
};
size_t router_fused_smem_bytes(int B, int Np, int Dp, int stride);
int router_fused_launch(oea_ctx* ctx, const oea_layer* L, const oea_dev::Cfg& cfg, int B,
                        const FusedRouterBuffers& rb, cudaStream_t s);

// layer.cu
int layer_upload_router(oea_layer* L, const void* src, int src_dtype, int on_device);
int layer_upload_expert(oea_layer* L, int e, const void* wg, const void* wu, const void* wd,
                        int src_dtype, int on_device);
int layer_init_random(oea_layer* L, uint64_t seed);
int layer_router_refresh(oea_layer* L);  // router_t from the fragment-ordered router
int layer_download_router(oea_layer* L, void* dst, int dst_dtype);
int layer_download_expert(oea_layer* L, int e, void* wg, void* wu, void* wd, int dst_dtype);

}  // namespace oea_host
