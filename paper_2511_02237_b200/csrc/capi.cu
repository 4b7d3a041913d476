// capi.cu — the extern "C" boundary (include/oea_cuda.h): contexts, the
// workspace arena, argument validation with the reference's error texts, and
// the orchestration of the kernel families. No arithmetic of the hot path
// happens on the host: every compute entry point launches CUDA work (and the
// context refuses to exist without an sm_100 device).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <cstdio>
#include <string>
#include <vector>

#include "oea_device.cuh"
#include "oea_internal.cuh"

using namespace oea_dev;

namespace {

thread_local std::string t_last_error;

struct Workspace {
  void* base = nullptr;
  size_t bytes = 0;
  // capacities
  int B = 0, N = 0, Np = 0, D = 0, Dp = 0, H = 0, Hp = 0, S = 0, R = 0, G = 0;
  // carved pointers
  double* scores = nullptr;
  double* logits64 = nullptr;
  double* x64 = nullptr;
  void* xT = nullptr;
  float* logits = nullptr;
  int32_t* order = nullptr;
  int32_t* t = nullptr;
  int32_t* n = nullptr;
  uint32_t* union_bits = nullptr;
  int32_t* sets = nullptr;
  int32_t* set_len = nullptr;
  double* w64 = nullptr;
  float* w32 = nullptr;
  int32_t* loads = nullptr;
  int32_t* active_union = nullptr;
  int32_t* active_count = nullptr;
  int64_t* total_load = nullptr;
  int32_t* base_union = nullptr;
  int32_t* base_union_count = nullptr;
  int32_t* err_token = nullptr;
  uint32_t* tokbits = nullptr;
  int32_t* row_tok = nullptr;
  int32_t* row_slot = nullptr;
  int32_t* group_a = nullptr;
  int32_t* group_row0 = nullptr;
  int32_t* group_rows = nullptr;
  FfnHeader* hdr = nullptr;
  int32_t* counters = nullptr;
  int32_t* slice_done = nullptr;  // dense path: per-group 64-bit W1 K-slot counts
  void* xg = nullptr;             // tcgen05 FFN: token rows in plan order, UMMA layout
  unsigned long long* xlog = nullptr;   // fused decode: tagged logits [B][Np]
  unsigned long long* xuni = nullptr;   // tagged per-token base bitmaps [B][4]
  unsigned long long* xplan = nullptr;  // tagged plan rows [B][1 + 2 S]
  __nv_bfloat16* xpad = nullptr;
  void* hbuf = nullptr;
  void* ybuf = nullptr;
  uint8_t* mask = nullptr;
  void* xin = nullptr;   // device copy of caller input (host entry points)
  void* out = nullptr;   // device output (host entry points)
  float* out32 = nullptr;
  int32_t* alias = nullptr;  // caller plans with duplicated experts: y slot per plan slot
};

struct Need {
  int B, N, D, H, S;
};

size_t carve(Workspace& w, bool assign) {
  size_t off = 0;
  auto take = [&](auto*& ptr, size_t bytes) {
    off = (off + 255) & ~static_cast<size_t>(255);
    if (assign) ptr = reinterpret_cast<std::remove_reference_t<decltype(ptr)>>(
                    static_cast<char*>(w.base) + off);
    off += bytes;
  };
  const size_t B = w.B, N = w.N, Np = w.Np, D = w.D, Dp = w.Dp, H = w.H, Hp = w.Hp, S = w.S,
               R = w.R, G = w.G;
  const size_t Nmax = std::max(N, Np);
  take(w.scores, B * N * 8);
  take(w.logits64, B * N * 8);
  take(w.x64, B * D * 8);
  take(w.xT, B * D * 8);
  take(w.logits, B * Np * 4);
  take(w.order, B * Nmax * 4);
  take(w.t, B * 4);
  take(w.n, B * 4);
  take(w.union_bits, ((Nmax + 31) / 32 + 1) * 4);
  take(w.sets, B * S * 4);
  take(w.set_len, B * 4);
  take(w.w64, B * S * 8);
  take(w.w32, B * S * 4);
  take(w.loads, Nmax * 4);
  take(w.active_union, Nmax * 4);
  take(w.active_count, 4);
  take(w.total_load, 8);
  take(w.base_union, Nmax * 4);
  take(w.base_union_count, 4);
  take(w.err_token, 4);
  take(w.tokbits, Nmax * ((B + 31) / 32) * 4);
  take(w.row_tok, R * 4);
  take(w.row_slot, R * 4);
  take(w.group_a, G * 4);
  take(w.group_row0, G * 4);
  take(w.group_rows, G * 4);
  take(w.hdr, sizeof(FfnHeader));
  // [G] per-group W1 release counters | [16] grid counters | per-token base bitmaps
  take(w.counters, (G + 16 + 4 * std::max<size_t>(B, 64) + 8) * 4);
  take(w.xlog, B * Nmax * 8);
  take(w.xuni, B * 8 * 8);
  take(w.xplan, B * (1 + 2 * S) * 8);  // tagged plan rows: len, then (expert, weight) per slot
  take(w.xpad, B * Dp * 2);
  // (dense decode: h [G][16][Hp] bf16, y [G][16][Dp] f32 with G <= N)
  take(w.hbuf, std::max(R * std::max(Hp, H) * 8, Nmax * 16 * Hp * 2));
  // (y: kW2KSplitMax K-part planes of [B][S][Dp] f32 on the dense path)
  take(w.ybuf, std::max({B * S * std::max(Dp, D) * 8, Nmax * 16 * Dp * 4,
                         std::min<size_t>(B, 16) * S * Dp * 4 * kW2KSplitMax}));
  take(w.mask, B);
  take(w.xin, B * D * 8);
  take(w.out, B * D * 8);
  take(w.out32, B * D * 4);
  take(w.alias, B * S * 4);
  take(w.slice_done, G * 8);
  take(w.xg, (R + 16) * Dp * 2);  // (zeroed at allocation; the kernel self-resets)
  return off + 256;
}

void set_caps(Workspace& w, const Need& nd) {
  w.B = nd.B;
  w.N = nd.N;
  w.Np = round_up(nd.N, 16);
  w.D = nd.D;
  w.Dp = round_up(nd.D, kPadD);
  w.H = nd.H;
  w.Hp = round_up(nd.H, kPadH);
  w.S = std::max(nd.S, 1);
  w.G = nd.N + (nd.B * w.S) / kTokGroup + 2;
  w.R = nd.B * w.S + 8 * w.G;
}

bool covers(const Workspace& w, const Need& nd) {
  return w.base && nd.B <= w.B && nd.N <= w.N && nd.D <= w.D && nd.H <= w.H && nd.S <= w.S;
}

int ensure(oea_ctx* ctx, Workspace& w, Need nd) {
  if (covers(w, nd)) return OEA_OK;
  if (w.base) {
    // grow monotonically in every dimension
    nd.B = std::max(nd.B, w.B);
    nd.N = std::max(nd.N, w.N);
    nd.D = std::max(nd.D, w.D);
    nd.H = std::max(nd.H, w.H);
    nd.S = std::max(nd.S, w.S);
    OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    cudaFree(w.base);
    w.base = nullptr;
  }
  set_caps(w, nd);
  const size_t bytes = carve(w, false);
  OEA_CUDA_TRY(ctx, cudaMalloc(&w.base, bytes));
  // the fused decode's grid counters must start at zero (they self-reset)
  OEA_CUDA_TRY(ctx, cudaMemsetAsync(w.base, 0, bytes, ctx->stream));
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  w.bytes = bytes;
  carve(w, true);
  return OEA_OK;
}

// OEA_HOST_PROFILE=1: per-phase host times of oea_moe_decode_host's zero-copy
// path (mean us, printed at exit): checks, pointer lookups, node patch,
// graph launch, the spin until the completion flag.
struct HostProfile {
  bool on = getenv("OEA_HOST_PROFILE") != nullptr;
  double sum[5] = {0, 0, 0, 0, 0};
  long n = 0, calls = 0;
  static double now() {
    timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
  }
  ~HostProfile() {
    if (on && n)
      fprintf(stderr, "host profile (%ld calls, mean us): checks %.2f lookups %.2f patch %.2f launch %.2f spin %.2f\n",
              n, sum[0] / n, sum[1] / n, sum[2] / n, sum[3] / n, sum[4] / n);
  }
};
HostProfile g_hprof;

// oea_moe_decode_host's zero-copy launches, captured once per (layer, B,
// config, workspace) as a one-kernel graph; each call patches the kernel
// node's x / out pointers and replays it (a graph launch costs ~2 us of host
// time, a direct launch of the fused kernel ~5 us).
struct HostGraph {
  const oea_layer* L = nullptr;
  int B = 0;
  oea_routing_cfg rc{};
  const void* ws_base = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t node = nullptr;  // the kernel node
  cudaKernelNodeParams kp{};
  std::vector<unsigned char> params;  // the node's FfnParams, patched per call
  void* args[1] = {nullptr};
  const void* x_set = nullptr;  // x / out the exec node currently points at
  void* out_set = nullptr;
  uint64_t used = 0;
};

struct CtxExtra {
  Workspace ws;
  // batched routing (oea_route_f64_batched_host): per-record aggregates
  void* seg_buf = nullptr;
  size_t seg_bytes = 0;
  std::vector<HostGraph> host_graphs;
  uint64_t host_graph_clock = 0;
  // completion flag of host-buffer decodes (mapped pinned int), lazily
  int* done_flag = nullptr;
  int* done_flag_dev = nullptr;
};

void host_graph_release(HostGraph& h) {
  if (h.exec) cudaGraphExecDestroy(h.exec);
  if (h.graph) cudaGraphDestroy(h.graph);
  h = HostGraph{};
}

CtxExtra* extra(oea_ctx* ctx) { return reinterpret_cast<CtxExtra*>(ctx->ws); }

int fail(oea_ctx* ctx, int code, const std::string& msg) { return oea_set_error(ctx, code, msg); }

#define CHECK_CTX(ctx)                                                              \
  do {                                                                             \
    if ((ctx) == nullptr) return fail(nullptr, OEA_ERR_INVALID_ARGUMENT, "null context"); \
  } while (0)

// RoutingConfig::resolved (routing.cpp:153-182), same messages.
int resolve(oea_ctx* ctx, const oea_routing_cfg* in, int n, oea_routing_cfg* out) {
  if (in == nullptr) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "null routing config");
  if (n < 1) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "RoutingConfig: expert count must be >= 1");
  oea_routing_cfg c = *in;
  if (c.mode < OEA_MODE_VANILLA || c.mode > OEA_MODE_SIMPLIFIED)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "unknown routing mode");
  if (c.cap != OEA_CAP_EXACT && c.cap != OEA_CAP_PSEUDOCODE)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "unknown cap semantics");
  if (c.mode == OEA_MODE_SIMPLIFIED) {
    c.p = 1.0;
    c.k_max = c.k;
    c.max_p = n;
  }
  if (c.max_p == 0) c.max_p = n;
  if (c.k < 1 || c.k > n) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "RoutingConfig: k must be in [1, N]");
  if (c.mode != OEA_MODE_VANILLA) {
    if (c.k0 < 1 || c.k0 > n)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "RoutingConfig: k0 must be in [1, N]");
    if (!(c.p > 0.0) || c.p > 1.0)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "RoutingConfig: p must be in (0, 1]");
    if (c.k_max < c.k0 || c.k_max > n)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "RoutingConfig: need k0 <= k_max <= N");
    if (c.max_p < 1 || c.max_p > n)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "RoutingConfig: max_p must be in [1, N]");
  }
  *out = c;
  return OEA_OK;
}

int32_t stride_of(const oea_routing_cfg& c) {
  switch (c.mode) {
    case OEA_MODE_VANILLA: return c.k;
    case OEA_MODE_PRUNED: return c.k0;
    default: return c.k_max + (c.cap == OEA_CAP_PSEUDOCODE ? 1 : 0);
  }
}

Cfg dev_cfg(const oea_routing_cfg& c, int stride) {
  Cfg d;
  d.mode = c.mode;
  d.k = c.k;
  d.k0 = c.k0;
  d.p = c.p;
  d.k_max = c.k_max;
  d.max_p = c.max_p;
  d.cap = c.cap;
  d.limit = c.k_max + (c.cap == OEA_CAP_PSEUDOCODE ? 1 : 0);
  d.stride = stride;
  return d;
}

oea_host::RouteBuffers route_buffers(Workspace& w, const double* scores, const uint8_t* mask) {
  oea_host::RouteBuffers rb;
  rb.scores = scores;
  rb.mask = mask;
  rb.order = w.order;
  rb.t = w.t;
  rb.n = w.n;
  rb.union_bits = w.union_bits;
  rb.sets = w.sets;
  rb.set_len = w.set_len;
  rb.weights = w.w64;
  rb.weights_f32 = w.w32;
  rb.loads = w.loads;
  rb.active_union = w.active_union;
  rb.active_count = w.active_count;
  rb.total_load = w.total_load;
  rb.base_union = w.base_union;
  rb.base_union_count = w.base_union_count;
  rb.err_token = w.err_token;
  return rb;
}

template <typename T>
int d2h(oea_ctx* ctx, T* host, const T* dev, size_t n) {
  if (host == nullptr || n == 0) return OEA_OK;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  return OEA_OK;
}

// Copy a [B][dev_stride] int/double matrix into a host [B][host_stride] one.
template <typename T>
int d2h_rows(oea_ctx* ctx, T* host, int host_stride, const T* dev, int dev_stride, int B, int cols) {
  if (host == nullptr) return OEA_OK;
  OEA_CUDA_TRY(ctx, cudaMemcpy2DAsync(host, host_stride * sizeof(T), dev, dev_stride * sizeof(T),
                                      cols * sizeof(T), B, cudaMemcpyDeviceToHost, ctx->stream));
  return OEA_OK;
}

int check_domain(oea_ctx* ctx, Workspace& w, int B) {
  int32_t tok = INT_MAX;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(&tok, w.err_token, 4, cudaMemcpyDeviceToHost, ctx->stream));
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (tok >= 0 && tok < B)
    return fail(ctx, OEA_ERR_DOMAIN, "route: degenerate selected-set mass for token " +
                                         std::to_string(tok) + " (sum <= 1e-12)");
  return OEA_OK;
}

// Export a device plan held in the workspace to caller host buffers.
int export_plan(oea_ctx* ctx, Workspace& w, const oea_plan_view* plan, int B, int N, int stride,
                int order_stride) {
  if (plan == nullptr) return OEA_OK;
  const int ps = plan->set_stride;
  const int cols = std::min(ps, stride);
  int rc = OEA_OK;
  if (plan->sets) {
    if (ps > stride) std::fill(plan->sets, plan->sets + static_cast<size_t>(B) * ps, -1);
    rc = d2h_rows(ctx, plan->sets, ps, w.sets, stride, B, cols);
  }
  if (!rc && plan->weights) {
    if (ps > stride) std::fill(plan->weights, plan->weights + static_cast<size_t>(B) * ps, 0.0);
    rc = d2h_rows(ctx, plan->weights, ps, w.w64, stride, B, cols);
  }
  if (!rc && plan->weights_f32) {
    if (ps > stride) std::fill(plan->weights_f32, plan->weights_f32 + static_cast<size_t>(B) * ps, 0.0f);
    rc = d2h_rows(ctx, plan->weights_f32, ps, w.w32, stride, B, cols);
  }
  if (!rc) rc = d2h(ctx, plan->set_len, w.set_len, B);
  if (!rc) rc = d2h(ctx, plan->loads, w.loads, N);
  if (!rc) rc = d2h(ctx, plan->active_union, w.active_union, N);
  if (!rc) rc = d2h(ctx, plan->active_count, w.active_count, 1);
  if (!rc) rc = d2h(ctx, plan->total_load, w.total_load, 1);
  if (!rc && plan->order) rc = d2h_rows(ctx, plan->order, N, w.order, order_stride, B, N);
  if (!rc) rc = d2h(ctx, plan->phase1_t, w.t, B);
  if (!rc) rc = d2h(ctx, plan->phase1_n, w.n, B);
  if (!rc) rc = d2h(ctx, plan->base_union, w.base_union, N);
  if (!rc) rc = d2h(ctx, plan->base_union_count, w.base_union_count, 1);
  if (rc) return rc;
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return OEA_OK;
}

__global__ void k_pad_x_bf16_from_f64(const double* __restrict__ x, int B, int D, int Dp,
                                      __nv_bfloat16* __restrict__ xpad) {
  const size_t total = static_cast<size_t>(B) * Dp;
  for (size_t f = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(f / Dp), d = static_cast<int>(f % Dp);
    xpad[f] = d < D ? __double2bfloat16(x[static_cast<size_t>(t) * D + d]) : __float2bfloat16_rn(0.f);
  }
}

__global__ void k_f32_to_f64(const float* __restrict__ a, size_t n, double* __restrict__ b) {
  for (size_t f = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<size_t>(gridDim.x) * blockDim.x)
    b[f] = static_cast<double>(a[f]);
}

// Kernel nodes of a captured decode graph (launch accounting per replay).
int count_kernel_nodes(cudaGraph_t graph) {
  size_t n = 0;
  if (cudaGraphGetNodes(graph, nullptr, &n) != cudaSuccess || n == 0) return 0;
  std::vector<cudaGraphNode_t> nodes(n);
  if (cudaGraphGetNodes(graph, nodes.data(), &n) != cudaSuccess) return 0;
  int k = 0;
  for (size_t i = 0; i < n; ++i) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nodes[i], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

int blocks_for(size_t n) {
  return static_cast<int>(std::max<size_t>(1, std::min<size_t>(4096, (n + 255) / 256)));
}

// ---------------------------------------------------------------------------
// Decode orchestration (shared by the direct call and graph capture).
// ---------------------------------------------------------------------------
// The fused single-launch decode covers B <= 64, N <= 128, D % 8 == 0 and
// p == 1 with a full piggyback window (max_p = N); expert-parallel shards run
// only on it.
static bool rank_routing_ok(const oea_layer* L, const oea_routing_cfg& rc) {
  static const bool mass = getenv("OEA_FUSED_MASS") == nullptr || atoi(getenv("OEA_FUSED_MASS")) != 0;
  return mass || rc.mode == OEA_MODE_VANILLA || (rc.p == 1.0 && rc.max_p >= L->N);
}

bool fused_ok(const oea_layer* L, int B, const oea_routing_cfg& rc) {
  // (every routing config: p < 1 and max_p < N are part of the rank routing;
  // OEA_FUSED_MASS=0 sends them to the router cluster + FFN pair instead)
  return B <= kRouterTokChunk && L->router_t != nullptr && L->Np <= 128 && (L->D & 7) == 0 &&
         rank_routing_ok(L, rc) &&
         oea_host::ffn_bf16_smem_bytes() + oea_host::ffn_btile_bytes() +
                 oea_host::ffn_route_smem_bytes(B, L->Np, stride_of(rc)) <= 227 * 1024;
}

// Large batches take the tcgen05 FFN unless OEA_UMMA=0. Its weight copy is
// allocated on first use, which a stream capture cannot do: captured before
// that first use, the mma.sync FFN is captured instead.
bool umma_ok(oea_ctx* ctx, const oea_layer* L, cudaStream_t s) {
  static const bool off = getenv("OEA_UMMA") != nullptr && atoi(getenv("OEA_UMMA")) == 0;
  if (off || L->dtype != OEA_DTYPE_BF16 || L->n_local < L->N) return false;
  if (L->w1u != nullptr && !L->umma_stale) return true;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s == nullptr ? ctx->stream : s, &cs) != cudaSuccess) return false;
  return cs == cudaStreamCaptureStatusNone;
}

// part: 0 = router + FFN (PDL-chained), 1 = router only, 2 = FFN only.
constexpr int kNotFused = -1000;  // decode_bf16(x_mapped): not on the fused path, nothing launched
// x_mapped: x and out are device views of mapped (pinned) host memory; only
// the fused single launch takes them (the caller checks fused_path()).
int decode_bf16(oea_ctx* ctx, Workspace& w, oea_layer* L, const void* x, const uint8_t* mask,
                int B, const oea_routing_cfg& rc, void* out, cudaStream_t s, int part = 0,
                bool x_mapped = false, const oea_dev::EpPeers* ep = nullptr) {
  const int stride = stride_of(rc);
  const Cfg cfg = dev_cfg(rc, stride);
  oea_host::FusedRouterBuffers rb;
  rb.x = static_cast<const __nv_bfloat16*>(x);
  rb.mask = mask;
  const bool padded = L->D != L->Dp;
  rb.xpad = padded ? w.xpad : nullptr;
  rb.logits = w.logits;
  rb.order = w.order;
  rb.sets = w.sets;
  rb.set_len = w.set_len;
  rb.weights_f32 = w.w32;
  rb.weights_f64 = w.w64;
  rb.loads = w.loads;
  rb.active_union = w.active_union;
  rb.active_count = w.active_count;
  rb.total_load = w.total_load;
  rb.row_tok = w.row_tok;
  rb.row_slot = w.row_slot;
  rb.group_a = w.group_a;
  rb.group_row0 = w.group_row0;
  rb.group_rows = w.group_rows;
  rb.hdr = w.hdr;
  rb.counters = w.counters;
  rb.n_counters = w.G + 7;  // w1_done + grid counters 0..6 (not the launch epoch, [7])
  rb.out = static_cast<float*>(out);
  rb.phase1_n = w.n;
  rb.base_union = w.base_union;
  rb.base_union_count = w.base_union_count;
  rb.trace = ctx->ffn_trace;
  // Fused single launch (B <= 64): the FFN grid computes the logits, routes
  // the batch in every CTA and streams the union's weights as soon as it is
  // known (expert_ffn.cu fused_*). OEA_TWO_KERNEL=1 forces the router-cluster
  // + FFN pair (always used for B > 64 and for the router-only stage graph).
  // (The fused prologue is kept small — it runs cold once per launch — so it
  // covers N <= 128, p == 1 and D % 8 == 0; other shapes/configs use the pair.)
  const bool shard = L->n_local < L->N;
  // Large batches (B > 64, and from OEA_BIG_MIN = 32 when the tcgen05 FFN is
  // available for the layer: measured faster than the fused token-list
  // launch from ~B = 32, e.g. B = 64 194 -> 172 us) with the rank-routing
  // conditions: a route-only launch of the fused prologue (tensor-core gate
  // GEMV, rank routing, union, plan rows, compaction), then the FFN.
  static const int big_min = getenv("OEA_BIG_MIN") ? atoi(getenv("OEA_BIG_MIN")) : 32;
  const bool fused_cand = part == 0 && fused_ok(L, B, rc) &&
                          (shard || getenv("OEA_TWO_KERNEL") == nullptr);
  const bool big_shape = part == 0 && !shard && B > 16 && B <= kMaxFusedB &&
                         L->router_t != nullptr && L->Np <= 128 && L->D == L->Dp &&
                         rank_routing_ok(L, rc) &&
                         getenv("OEA_TWO_KERNEL") == nullptr &&
                         oea_host::ffn_bf16_smem_bytes() +
                                 oea_host::ffn_route_smem_bytes(B, L->Np, stride) <= 227 * 1024;
  const bool big = big_shape && (B > kRouterTokChunk
                                     ? !fused_cand
                                     : B >= big_min && !x_mapped && umma_ok(ctx, L, s));
  const bool fused = fused_cand && !big;
  if (x_mapped && !fused) return kNotFused;  // the caller stages x itself
  int r = OEA_OK;
  // large batches: the tcgen05 FFN (its weight copy made / refreshed here,
  // outside any capture), and the compaction (+ its token-row gather) inside
  // the route-only launch (OEA_BIG_COMPACT=0: the separate k_compact)
  const bool use_umma = big && umma_ok(ctx, L, s);
  if (use_umma && (L->w1u == nullptr || L->umma_stale)) {
    r = oea_host::layer_prepare_umma(ctx, L, s);
    if (r) return r;
    L->umma_stale = 0;
  }
  static const bool big_compact = getenv("OEA_BIG_COMPACT") == nullptr || atoi(getenv("OEA_BIG_COMPACT")) != 0;
  const int xg_rg = static_cast<int>((w.R + 16) / 8);
  if (rb.trace && !fused) OEA_CUDA_TRY(ctx, cudaMemsetAsync(rb.trace, 0, 8 * 8 * 1024, s));
  if (big) {
    oea_host::FfnBuffers rf;
    rf.route_only = 1;
    rf.fused = 1;
    rf.x = x;
    rf.counters = w.counters;
    rf.max_groups = w.G;
    rf.hdr = w.hdr;
    rf.x_in = static_cast<const __nv_bfloat16*>(x);
    rf.logits = w.logits;
    rf.xlog = w.xlog;
    rf.xuni = w.xuni;
    rf.xplan = w.xplan;
    rf.mask = mask;
    rf.cfg = cfg;
    rf.x_sets = w.sets;
    rf.x_set_len = w.set_len;
    rf.x_w32 = w.w32;
    rf.x_w64 = w.w64;
    rf.x_loads = w.loads;
    rf.x_active = w.active_union;
    rf.x_active_count = w.active_count;
    rf.x_total_load = w.total_load;
    rf.x_phase1_n = w.n;
    rf.x_base_union = w.base_union;
    rf.x_base_union_count = w.base_union_count;
    rf.x_hdr = w.hdr;
    rf.trace = ctx->ffn_trace;
    rf.row_tok = w.row_tok;
    rf.row_slot = w.row_slot;
    rf.group_a = w.group_a;
    rf.group_row0 = w.group_row0;
    rf.group_rows = w.group_rows;
    rf.compact_in_kernel = big_compact ? 1 : 0;
    rf.xg = big_compact && use_umma ? w.xg : nullptr;
    rf.pf_w1u = use_umma ? L->w1u : nullptr;
    rf.xg_rg = xg_rg;
    r = oea_host::ffn_bf16_launch(ctx, L, B, stride, rf, false, s);
    if (r) return r;
    if (!big_compact) {
      oea_host::CompactBuffers cb{w.sets, w.set_len, w.row_tok, w.row_slot, w.group_a,
                                  w.group_row0, w.group_rows, w.hdr, w.counters, w.G + 7,
                                  w.loads, w.total_load};
      r = oea_host::compact_launch(ctx, B, L->N, stride, cb, w.tokbits, w.active_union,
                                   w.active_count, s);
      if (r) return r;
    }
  } else if (part != 2 && !fused) {
    r = oea_host::router_fused_launch(ctx, L, cfg, B, rb, s);
    if (r || part == 1) return r;
  }
  oea_host::FfnBuffers fb;
  fb.ep = ep;
  fb.x = padded || x_mapped ? static_cast<const void*>(w.xpad) : x;
  fb.row_tok = w.row_tok;
  fb.row_slot = w.row_slot;
  fb.group_a = w.group_a;
  fb.group_row0 = w.group_row0;
  fb.group_rows = w.group_rows;
  fb.hdr = w.hdr;
  fb.counters = w.counters;
  fb.slice_done = w.slice_done;
  fb.max_groups = w.G;
  fb.hbuf = w.hbuf;
  fb.ybuf = w.ybuf;
  fb.set_len = w.set_len;
  fb.weights_f32 = w.w32;
  fb.weights_f64 = w.w64;
  fb.out = out;
  fb.trace = ctx->ffn_trace;
  fb.mode = ctx->ffn_mode;
  if (fused) {
    fb.fused = 1;
    // dense-over-batch FFN when the batch is one or two n-blocks and the
    // swizzled x tile fits next to the ring (OEA_SPARSE=1 forces token lists)
    // (Hp <= 8192: the per-group W1 K-slot counts are 8-bit fields)
    fb.dense = B <= 16 && L->Hp <= 8192 && getenv("OEA_SPARSE") == nullptr &&
               oea_host::ffn_bf16_smem_bytes() + oea_host::ffn_route_smem_bytes(B, L->Np, stride) +
                       oea_host::ffn_dense_xs_bytes(L->Dp) <= 227 * 1024;
    // OEA_UMMA_DENSE=1 (experimental, off by default: measured slower, DESIGN.md
    // §3b): dense decode on tcgen05 (MODE 6) when the layer's UMMA-layout copy
    // exists or can be made now (not during a capture, enough free memory)
    static const bool udense = getenv("OEA_UMMA_DENSE") != nullptr && atoi(getenv("OEA_UMMA_DENSE")) != 0;
    if (fb.dense && udense && !ep && !shard && !x_mapped && umma_ok(ctx, L, s)) {
      bool have = L->w1u != nullptr;
      if (!have) {
        size_t fr = 0, tot = 0;
        const size_t need = static_cast<size_t>(3 * L->Hp) * L->Dp * 2 * L->n_local;
        if (cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr > need + (size_t(4) << 30)) {
          r = oea_host::layer_prepare_umma(ctx, L, s);
          if (r) return r;
          L->umma_stale = 0;
          have = true;
        }
      } else if (L->umma_stale) {
        r = oea_host::layer_prepare_umma(ctx, L, s);
        if (r) return r;
        L->umma_stale = 0;
      }
      fb.umma_dense = have ? 1 : 0;
    }
    fb.x_in = static_cast<const __nv_bfloat16*>(x);
    fb.xpad_out = padded || x_mapped ? w.xpad : nullptr;
    fb.x_stage = x_mapped ? 1 : 0;
    fb.done_flag = x_mapped ? extra(ctx)->done_flag_dev : nullptr;
    fb.logits = w.logits;
    fb.xlog = w.xlog;
    fb.xuni = w.xuni;
    fb.xplan = w.xplan;
    fb.mask = mask;
    fb.cfg = cfg;
    fb.x_sets = w.sets;
    fb.x_set_len = w.set_len;
    fb.x_w32 = w.w32;
    fb.x_w64 = w.w64;
    fb.x_loads = w.loads;
    fb.x_active = w.active_union;
    fb.x_active_count = w.active_count;
    fb.x_total_load = w.total_load;
    fb.x_phase1_n = w.n;
    fb.x_base_union = w.base_union;
    fb.x_base_union_count = w.base_union_count;
    fb.x_hdr = w.hdr;
  }
  if (use_umma)  // tcgen05 (UMMA + TMEM) grouped FFN
    return oea_host::ffn_umma_launch(ctx, L, B, stride, fb, w.xg, xg_rg, s, big_compact);
  return oea_host::ffn_bf16_launch(ctx, L, B, stride, fb, part == 0 && !fused && !big, s);
}

// f32/f64 layers: router_scores (fp64) -> route_f64 -> compaction -> SIMT FFN.
int decode_simt(oea_ctx* ctx, Workspace& w, oea_layer* L, const double* x, const uint8_t* mask,
                int B, const oea_routing_cfg& rc, double* out, cudaStream_t s) {
  const int stride = stride_of(rc);
  const Cfg cfg = dev_cfg(rc, stride);
  int r = oea_host::router_scores_launch(ctx, L, x, B, w.logits64, w.scores, s);
  if (r) return r;
  const int set_mode = rc.mode == OEA_MODE_VANILLA ? 0 : rc.mode == OEA_MODE_PRUNED ? 1 : 2;
  r = oea_host::route_f64_launch(ctx, cfg, B, L->N, route_buffers(w, w.scores, mask), false,
                                 rc.mode != OEA_MODE_VANILLA, set_mode, false, s);
  if (r) return r;
  oea_host::CompactBuffers cb{w.sets, w.set_len, w.row_tok, w.row_slot, w.group_a,
                              w.group_row0, w.group_rows, w.hdr, w.counters, w.G + 1};
  r = oea_host::compact_launch(ctx, B, L->N, stride, cb, w.tokbits, w.active_union,
                               w.active_count, s);
  if (r) return r;
  r = oea_host::cast_f64_launch(ctx, x, static_cast<size_t>(B) * L->D, L->dtype, w.xT, s);
  if (r) return r;
  oea_host::FfnBuffers fb{};
  fb.x = w.xT;
  fb.row_tok = w.row_tok;
  fb.row_slot = w.row_slot;
  fb.group_a = w.group_a;
  fb.group_row0 = w.group_row0;
  fb.group_rows = w.group_rows;
  fb.hdr = w.hdr;
  fb.hbuf = w.hbuf;
  fb.ybuf = w.ybuf;
  fb.set_len = w.set_len;
  fb.weights_f64 = w.w64;
  fb.out = out;
  return oea_host::ffn_simt_launch(ctx, L, B, stride, fb, w.G, s);
}

int validate_decode(oea_ctx* ctx, oea_layer* L, int B, const oea_routing_cfg* cfg,
                    oea_routing_cfg* rc) {
  if (L == nullptr) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "null layer");
  if (B < 1) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "moe_decode: batch must be >= 1");
  int r = resolve(ctx, cfg, L->N, rc);
  if (r) return r;
  if (L->dtype == OEA_DTYPE_BF16) {
    if (B > kMaxFusedB)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT,
                  "moe_decode: bf16 fused decode supports B <= " + std::to_string(kMaxFusedB));
    if (L->N > kMaxFusedN)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT,
                  "moe_decode: bf16 fused router supports N <= " + std::to_string(kMaxFusedN));
    if (oea_host::router_fused_smem_bytes(B, L->Np, L->Dp, stride_of(*rc)) > 227 * 1024)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT,
                  "moe_decode: B x N too large for the single-CTA fused router");
    if (L->n_local < L->N && !fused_ok(L, B, *rc))
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT,
                  "moe_decode: expert-parallel shards need the fused path (B <= 64, N <= 128, "
                  "D % 8 == 0, p == 1, max_p = N, and the batch's routing tables within the "
                  "227 KiB of shared memory)");
  }
  return OEA_OK;
}

Need need_for(const oea_layer* L, int B, int S) { return Need{B, L->N, L->D, L->H, S}; }

}  // namespace

// ===========================================================================
// Status helpers.
// ===========================================================================
int oea_set_error(oea_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->last_error = msg;
  t_last_error = msg;
  return code;
}

int oea_check_cuda(oea_ctx* ctx, cudaError_t e, const char* what) {
  return oea_set_error(ctx, OEA_ERR_CUDA,
                       std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

extern "C" {

int oea_abi_version(void) { return OEA_ABI_VERSION; }

int oea_ctx_create(int32_t device, oea_ctx_t* out) {
  if (out == nullptr) return fail(nullptr, OEA_ERR_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(nullptr, OEA_ERR_CUDA,
                std::string("no CUDA device available (oea has no CPU path): ") +
                    (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
  if (device < 0 || device >= count) return fail(nullptr, OEA_ERR_INVALID_ARGUMENT, "bad device index");
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return oea_check_cuda(nullptr, e, "cudaGetDeviceProperties");
  if (prop.major != 10)
    return fail(nullptr, OEA_ERR_CUDA,
                "oea kernels are built for sm_100a; device is sm_" + std::to_string(prop.major) +
                    std::to_string(prop.minor));
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return oea_check_cuda(nullptr, e, "cudaSetDevice");
  auto* ctx = new oea_ctx;
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  // (zeroed once; the single-launch route resets it at every launch's end)
  if (cudaMalloc(&ctx->route_scratch, oea_dev::kRouteScratchBytes) == cudaSuccess)
    cudaMemset(ctx->route_scratch, 0, oea_dev::kRouteScratchBytes);
  else
    ctx->route_scratch = nullptr;
  e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return oea_check_cuda(nullptr, e, "cudaStreamCreate");
  }
  ctx->ws = new CtxExtra;
  if (const char* tr = getenv("OEA_FFN_TRACE")) {
    if (tr[0] == '1') {
      if (cudaMalloc(&ctx->ffn_trace, 8 * oea_dev::kTraceWords) != cudaSuccess)
        ctx->ffn_trace = nullptr;
      else
        cudaMemset(ctx->ffn_trace, 0, 8 * oea_dev::kTraceWords);
    }
  }
  if (const char* md = getenv("OEA_FFN_MODE")) ctx->ffn_mode = atoi(md);
  *out = ctx;
  return OEA_OK;
}

int oea_debug_ffn_trace(oea_ctx_t ctx, uint64_t* host, int32_t n) {
  CHECK_CTX(ctx);
  if (ctx->ffn_trace == nullptr) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "OEA_FFN_TRACE not enabled");
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  OEA_CUDA_TRY(ctx, cudaMemcpy(host, ctx->ffn_trace, sizeof(uint64_t) * std::min<size_t>(n, oea_dev::kTraceWords),
                               cudaMemcpyDeviceToHost));
  return OEA_OK;
}

int oea_ctx_destroy(oea_ctx_t ctx) {
  if (ctx == nullptr) return OEA_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  CtxExtra* x = extra(ctx);
  if (x) {
    for (auto& h : x->host_graphs) host_graph_release(h);
    if (x->ws.base) cudaFree(x->ws.base);
    if (x->seg_buf) cudaFree(x->seg_buf);
    if (x->done_flag) cudaFreeHost(x->done_flag);
    delete x;
  }
  if (ctx->ffn_trace) cudaFree(ctx->ffn_trace);
  if (ctx->route_scratch) cudaFree(ctx->route_scratch);
  if (ctx->ep_tables) cudaFree(ctx->ep_tables);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return OEA_OK;
}

const char* oea_last_error(oea_ctx_t ctx) {
  return ctx ? ctx->last_error.c_str() : t_last_error.c_str();
}

int oea_ctx_stream(oea_ctx_t ctx, void** stream_out) {
  CHECK_CTX(ctx);
  *stream_out = ctx->stream;
  return OEA_OK;
}

int oea_ctx_synchronize(oea_ctx_t ctx) {
  CHECK_CTX(ctx);
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return OEA_OK;
}

int64_t oea_ctx_kernel_launches(oea_ctx_t ctx) { return ctx ? ctx->launches : 0; }

int oea_config_resolve(const oea_routing_cfg* in, int32_t n_experts, oea_routing_cfg* out) {
  if (out == nullptr) return fail(nullptr, OEA_ERR_INVALID_ARGUMENT, "null output pointer");
  return resolve(nullptr, in, n_experts, out);
}

int32_t oea_plan_set_stride(const oea_routing_cfg* resolved) {
  return resolved ? stride_of(*resolved) : 0;
}

// ---------------------------------------------------------------------------
// K1 routing entry points.
// ---------------------------------------------------------------------------
int oea_route_f64(oea_ctx_t ctx, const double* scores_dev, const uint8_t* mask_dev, int32_t B,
                  int32_t N, const oea_routing_cfg* cfg, const oea_plan_view* plan, void* stream) {
  CHECK_CTX(ctx);
  oea_routing_cfg rc;
  int r = resolve(ctx, cfg, N, &rc);
  if (r) return r;
  if (B < 1 || N < 1) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "sort_experts: dimensions must be >= 1");
  if (N > kMaxRouteN)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "route: N > " + std::to_string(kMaxRouteN));
  if (plan == nullptr || plan->sets == nullptr || plan->set_len == nullptr)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "route: plan sets/set_len are required");
  const int stride = stride_of(rc);
  if (plan->set_stride < stride)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "route: plan set_stride too small");
  Workspace& w = extra(ctx)->ws;
  r = ensure(ctx, w, Need{B, N, 1, 1, plan->set_stride});
  if (r) return r;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  oea_host::RouteBuffers rb = route_buffers(w, scores_dev, mask_dev);
  rb.sets = plan->sets;
  rb.set_len = plan->set_len;
  rb.weights = plan->weights;
  rb.weights_f32 = plan->weights_f32;
  if (plan->loads) rb.loads = plan->loads;
  if (plan->active_union) rb.active_union = plan->active_union;
  if (plan->active_count) rb.active_count = plan->active_count;
  if (plan->total_load) rb.total_load = plan->total_load;
  if (plan->order) rb.order = plan->order;
  if (plan->phase1_t) rb.t = plan->phase1_t;
  if (plan->phase1_n) rb.n = plan->phase1_n;
  rb.base_union = plan->base_union;
  rb.base_union_count = plan->base_union_count;
  if (rb.weights == nullptr && rb.weights_f32 == nullptr) rb.weights = w.w64;  // domain check
  const Cfg dc = dev_cfg(rc, plan->set_stride);
  const int set_mode = rc.mode == OEA_MODE_VANILLA ? 0 : rc.mode == OEA_MODE_PRUNED ? 1 : 2;
  if (oea_host::route_fast_ok(dc, N, plan->order != nullptr) && getenv("OEA_ROUTE_SORT") == nullptr)
    return oea_host::route_f64_fast_launch(ctx, dc, B, N, rb, set_mode, s);
  return oea_host::route_f64_launch(ctx, dc, B, N, rb, false, rc.mode != OEA_MODE_VANILLA,
                                    set_mode, false, s);
}

int oea_route_f64_host(oea_ctx_t ctx, const double* scores, const uint8_t* mask, int32_t B,
                       int32_t N, const oea_routing_cfg* cfg, const oea_plan_view* plan) {
  CHECK_CTX(ctx);
  oea_routing_cfg rc;
  int r = resolve(ctx, cfg, N, &rc);
  if (r) return r;
  if (B < 1 || N < 1) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "sort_experts: dimensions must be >= 1");
  if (N > kMaxRouteN)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "route: N > " + std::to_string(kMaxRouteN));
  if (plan == nullptr || plan->sets == nullptr || plan->set_len == nullptr)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "route: plan sets/set_len are required");
  const int stride = stride_of(rc);
  if (plan->set_stride < stride)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "route: plan set_stride too small");
  Workspace& w = extra(ctx)->ws;
  r = ensure(ctx, w, Need{B, N, 1, 1, stride});
  if (r) return r;
  cudaStream_t s = ctx->stream;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.scores, scores, sizeof(double) * B * N,
                                    cudaMemcpyHostToDevice, s));
  if (mask) OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.mask, mask, B, cudaMemcpyHostToDevice, s));
  const Cfg dc = dev_cfg(rc, stride);
  const int set_mode = rc.mode == OEA_MODE_VANILLA ? 0 : rc.mode == OEA_MODE_PRUNED ? 1 : 2;
  if (oea_host::route_fast_ok(dc, N, plan->order != nullptr) && getenv("OEA_ROUTE_SORT") == nullptr)
    r = oea_host::route_f64_fast_launch(ctx, dc, B, N,
                                        route_buffers(w, w.scores, mask ? w.mask : nullptr),
                                        set_mode, s);
  else
    r = oea_host::route_f64_launch(ctx, dc, B, N,
                                   route_buffers(w, w.scores, mask ? w.mask : nullptr), false,
                                   rc.mode != OEA_MODE_VANILLA, set_mode, false, s);
  if (r) return r;
  r = check_domain(ctx, w, B);
  if (r) return r;
  ctx->last_B = B;
  ctx->last_N = N;
  ctx->last_stride = stride;
  ctx->last_kind = 2;
  return export_plan(ctx, w, plan, B, N, stride, N);
}

// Many independent records (a score trace's (step, layer) batches) in one
// launch sequence: the route kernels (fast path, or the general sort path
// for p < 1 / max_p < N / N > 128) with a row -> record map, so each record
// has its own union and aggregates (io.cpp:85-172 + route() per record in the
// reference's `route` command, oea_cli.cpp:153-175).
int oea_route_f64_batched_host(oea_ctx_t ctx, const double* scores, const uint8_t* mask,
                               const int32_t* rows, int32_t R, int32_t N,
                               const oea_routing_cfg* cfg, const oea_plan_view* plan) {
  CHECK_CTX(ctx);
  if (R < 1 || rows == nullptr)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "route_batched: need R >= 1 records");
  int64_t total = 0;
  for (int r = 0; r < R; ++r) {
    if (rows[r] < 1) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "sort_experts: dimensions must be >= 1");
    total += rows[r];
  }
  if (total > INT_MAX / 2) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "route_batched: too many rows");
  const int B = static_cast<int>(total);
  oea_routing_cfg rc;
  int r = resolve(ctx, cfg, N, &rc);
  if (r) return r;
  if (plan == nullptr) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "route: null plan");
  if (plan->order != nullptr)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "route_batched: order is not exported");
  const int stride = stride_of(rc);
  if ((plan->sets || plan->weights || plan->weights_f32) && plan->set_stride < stride)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "route: plan set_stride too small");
  if (N > kMaxRouteN)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "route: N > " + std::to_string(kMaxRouteN));
  const Cfg dc = dev_cfg(rc, stride);
  Workspace& w = extra(ctx)->ws;
  r = ensure(ctx, w, Need{B, N, 1, 1, stride});
  if (r) return r;
  // per-record buffers: seg [B] | union [R][4] | loads, active, base [R][N] | counts [R] x2 | total [R]
  CtxExtra* ex = extra(ctx);
  const size_t words = (static_cast<size_t>(N) + 31) / 32;
  const size_t need = static_cast<size_t>(B) * 4 + static_cast<size_t>(R) * (4 * words + 12 * N + 8 + 8) + 256;
  cudaStream_t s = ctx->stream;
  if (need > ex->seg_bytes) {
    OEA_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    if (ex->seg_buf) cudaFree(ex->seg_buf);
    ex->seg_buf = nullptr;
    ex->seg_bytes = 0;
    OEA_CUDA_TRY(ctx, cudaMalloc(&ex->seg_buf, need));
    ex->seg_bytes = need;
  }
  char* p = static_cast<char*>(ex->seg_buf);
  auto take = [&](size_t bytes) {
    char* q = p;
    p += (bytes + 15) & ~size_t(15);
    return q;
  };
  int64_t* d_total = reinterpret_cast<int64_t*>(take(8 * static_cast<size_t>(R)));
  int32_t* d_seg = reinterpret_cast<int32_t*>(take(4 * static_cast<size_t>(B)));
  uint32_t* d_union = reinterpret_cast<uint32_t*>(take(4 * words * static_cast<size_t>(R)));
  int32_t* d_loads = reinterpret_cast<int32_t*>(take(4 * static_cast<size_t>(R) * N));
  int32_t* d_active = reinterpret_cast<int32_t*>(take(4 * static_cast<size_t>(R) * N));
  int32_t* d_base = reinterpret_cast<int32_t*>(take(4 * static_cast<size_t>(R) * N));
  int32_t* d_cnt = reinterpret_cast<int32_t*>(take(4 * static_cast<size_t>(R)));
  int32_t* d_bcnt = reinterpret_cast<int32_t*>(take(4 * static_cast<size_t>(R)));
  std::vector<int32_t> seg(B);
  for (int q = 0, i = 0; q < R; ++q)
    for (int j = 0; j < rows[q]; ++j) seg[i++] = q;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(d_seg, seg.data(), 4 * static_cast<size_t>(B), cudaMemcpyHostToDevice, s));
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.scores, scores, sizeof(double) * B * N, cudaMemcpyHostToDevice, s));
  if (mask) OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.mask, mask, B, cudaMemcpyHostToDevice, s));
  oea_host::RouteBuffers rb = route_buffers(w, w.scores, mask ? w.mask : nullptr);
  rb.union_bits = d_union;
  rb.loads = d_loads;
  rb.active_union = d_active;
  rb.active_count = d_cnt;
  rb.total_load = d_total;
  rb.base_union = d_base;
  rb.base_union_count = d_bcnt;
  const int set_mode = rc.mode == OEA_MODE_VANILLA ? 0 : rc.mode == OEA_MODE_PRUNED ? 1 : 2;
  if (oea_host::route_fast_ok(dc, N, false) && getenv("OEA_ROUTE_SORT") == nullptr)
    r = oea_host::route_f64_fast_launch(ctx, dc, B, N, rb, set_mode, s, R, d_seg);
  else
    r = oea_host::route_f64_launch(ctx, dc, B, N, rb, false, rc.mode != OEA_MODE_VANILLA,
                                   set_mode, false, s, R, d_seg);
  if (r) return r;
  int32_t tok = INT_MAX;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(&tok, w.err_token, 4, cudaMemcpyDeviceToHost, s));
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  if (tok >= 0 && tok < B) {
    int q = seg[tok], row0 = 0;
    for (int j = 0; j < q; ++j) row0 += rows[j];
    return fail(ctx, OEA_ERR_DOMAIN, "record " + std::to_string(q) +
                                         ": route: degenerate selected-set mass for token " +
                                         std::to_string(tok - row0) + " (sum <= 1e-12)");
  }
  const int ps = plan->set_stride, cols = std::min(ps, stride);
  if (plan->sets) r = d2h_rows(ctx, plan->sets, ps, w.sets, stride, B, cols);
  if (!r && plan->weights) r = d2h_rows(ctx, plan->weights, ps, w.w64, stride, B, cols);
  if (!r && plan->weights_f32) r = d2h_rows(ctx, plan->weights_f32, ps, w.w32, stride, B, cols);
  if (!r) r = d2h(ctx, plan->set_len, w.set_len, B);
  if (!r) r = d2h(ctx, plan->loads, d_loads, static_cast<size_t>(R) * N);
  if (!r) r = d2h(ctx, plan->active_union, d_active, static_cast<size_t>(R) * N);
  if (!r) r = d2h(ctx, plan->active_count, d_cnt, R);
  if (!r) r = d2h(ctx, plan->total_load, d_total, R);
  if (!r) r = d2h(ctx, plan->phase1_t, w.t, B);
  if (!r) r = d2h(ctx, plan->phase1_n, w.n, B);
  if (!r) r = d2h(ctx, plan->base_union, d_base, static_cast<size_t>(R) * N);
  if (!r) r = d2h(ctx, plan->base_union_count, d_bcnt, R);
  if (r) return r;
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  if (ps > stride) {  // pad the caller's wider rows
    for (int i = 0; i < B; ++i)
      for (int j = stride; j < ps; ++j) {
        if (plan->sets) plan->sets[static_cast<size_t>(i) * ps + j] = -1;
        if (plan->weights) plan->weights[static_cast<size_t>(i) * ps + j] = 0.0;
        if (plan->weights_f32) plan->weights_f32[static_cast<size_t>(i) * ps + j] = 0.0f;
      }
  }
  return OEA_OK;
}

// ScoreGenConfig::validate (score_gen.cpp:46-76) + the ScoreSource range check.
static int check_gen(oea_ctx* ctx, const oea_score_gen_cfg* c, int step0, int nsteps) {
  if (c == nullptr) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "null generator config");
  if (c->steps < 1 || c->layers < 1)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "score gen: steps and layers must be >= 1");
  if (c->kind != OEA_GEN_DIRICHLET && c->kind != OEA_GEN_CLUSTERED)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "score gen: replay is read on the host (read_score_trace)");
  if (c->n_experts < 1 || c->batch < 1)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "score gen: n_experts and batch must be >= 1");
  if (c->kind == OEA_GEN_DIRICHLET && !(c->alpha > 0.0))
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "score gen: alpha must be > 0");
  if (c->kind == OEA_GEN_CLUSTERED) {
    if (c->groups < 1 || c->groups > c->n_experts)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "score gen: groups must be in [1, n_experts]");
    if (!(c->within_group_concentration > 0.0))
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "score gen: within_group_concentration must be > 0");
    if (c->between_group_spread < 0.0)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "score gen: between_group_spread must be >= 0");
  }
  if (nsteps < 1 || step0 < 0 || static_cast<int64_t>(step0) + nsteps > c->steps)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "score source: step/layer out of range");
  return OEA_OK;
}

int oea_gen_scores(oea_ctx_t ctx, const oea_score_gen_cfg* cfg, int32_t step0, int32_t nsteps,
                   double* out_dev, void* stream) {
  CHECK_CTX(ctx);
  int r = check_gen(ctx, cfg, step0, nsteps);
  if (r) return r;
  if (out_dev == nullptr) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "gen_scores: null output");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  return oea_host::gen_scores_launch(ctx, *cfg, step0, nsteps, out_dev, s);
}

int oea_gen_scores_host(oea_ctx_t ctx, const oea_score_gen_cfg* cfg, int32_t step0,
                        int32_t nsteps, double* out_host) {
  CHECK_CTX(ctx);
  int r = check_gen(ctx, cfg, step0, nsteps);
  if (r) return r;
  if (out_host == nullptr) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "gen_scores: null output");
  const size_t n = static_cast<size_t>(nsteps) * cfg->layers * cfg->batch * cfg->n_experts;
  cudaStream_t s = ctx->stream;
  double* d = nullptr;
  OEA_CUDA_TRY(ctx, cudaMallocAsync(reinterpret_cast<void**>(&d), n * sizeof(double), s));
  r = oea_host::gen_scores_launch(ctx, *cfg, step0, nsteps, d, s);
  if (r == OEA_OK) r = d2h(ctx, out_host, d, n);
  cudaFreeAsync(d, s);
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return r;
}

int oea_sort_experts_f64_host(oea_ctx_t ctx, const double* scores, int32_t B, int32_t N,
                              int32_t* order) {
  CHECK_CTX(ctx);
  if (B < 1 || N < 1) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "sort_experts: dimensions must be >= 1");
  if (N > kMaxRouteN)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "sort_experts: N > " + std::to_string(kMaxRouteN));
  Workspace& w = extra(ctx)->ws;
  int r = ensure(ctx, w, Need{B, N, 1, 1, 1});
  if (r) return r;
  cudaStream_t s = ctx->stream;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.scores, scores, sizeof(double) * B * N,
                                    cudaMemcpyHostToDevice, s));
  oea_routing_cfg rc{OEA_MODE_VANILLA, 1, 1, 1.0, 1, N, OEA_CAP_EXACT};
  Cfg dc = dev_cfg(rc, 1);
  oea_host::RouteBuffers rb = route_buffers(w, w.scores, nullptr);
  rb.weights = nullptr;
  rb.weights_f32 = nullptr;
  r = oea_host::route_f64_launch(ctx, dc, B, N, rb, false, false, 0, false, s);
  if (r) return r;
  r = d2h(ctx, order, w.order, static_cast<size_t>(B) * N);
  if (r) return r;
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return OEA_OK;
}

int oea_phase1_f64_host(oea_ctx_t ctx, const double* scores, const uint8_t* mask, int32_t B,
                        int32_t N, const int32_t* order, const oea_routing_cfg* cfg, int32_t* t,
                        int32_t* n, int32_t* base_sets, int32_t base_stride, int32_t* base_union,
                        int32_t* base_union_count) {
  CHECK_CTX(ctx);
  oea_routing_cfg rc;
  int r = resolve(ctx, cfg, N, &rc);
  if (r) return r;
  if (B < 1 || N < 1) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "sort_experts: dimensions must be >= 1");
  if (order == nullptr) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "phase1: order is required");
  const int k0 = std::max(rc.k0, 1);
  if (base_sets && base_stride < k0)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "phase1: base_stride must be >= k0");
  Workspace& w = extra(ctx)->ws;
  r = ensure(ctx, w, Need{B, N, 1, 1, k0});
  if (r) return r;
  cudaStream_t s = ctx->stream;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.scores, scores, sizeof(double) * B * N,
                                    cudaMemcpyHostToDevice, s));
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.order, order, sizeof(int32_t) * B * N,
                                    cudaMemcpyHostToDevice, s));
  if (mask) OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.mask, mask, B, cudaMemcpyHostToDevice, s));
  Cfg dc = dev_cfg(rc, k0);
  oea_host::RouteBuffers rb = route_buffers(w, w.scores, mask ? w.mask : nullptr);
  rb.weights = nullptr;
  rb.weights_f32 = nullptr;
  r = oea_host::route_f64_launch(ctx, dc, B, N, rb, true, true, 1, false, s);
  if (r) return r;
  r = d2h(ctx, t, w.t, B);
  if (!r) r = d2h(ctx, n, w.n, B);
  if (!r && base_sets) r = d2h_rows(ctx, base_sets, base_stride, w.sets, k0, B, k0);
  if (!r) r = d2h(ctx, base_union, w.base_union, N);
  if (!r) r = d2h(ctx, base_union_count, w.base_union_count, 1);
  if (r) return r;
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  if (base_sets && base_stride > k0)
    for (int i = 0; i < B; ++i)
      for (int j = k0; j < base_stride; ++j) base_sets[static_cast<size_t>(i) * base_stride + j] = -1;
  return OEA_OK;
}

int oea_phase2_f64_host(oea_ctx_t ctx, const uint8_t* mask, int32_t B, int32_t N,
                        const int32_t* order, const int32_t* n, const int32_t* base_union,
                        int32_t base_union_count, const oea_routing_cfg* cfg,
                        const oea_plan_view* plan) {
  CHECK_CTX(ctx);
  oea_routing_cfg rc;
  int r = resolve(ctx, cfg, N, &rc);
  if (r) return r;
  if (B < 1 || N < 1) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "sort_experts: dimensions must be >= 1");
  if (order == nullptr || n == nullptr || plan == nullptr || plan->sets == nullptr ||
      plan->set_len == nullptr)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "phase2: order, n and plan sets are required");
  int max_n = 0;
  for (int i = 0; i < B; ++i) {
    if (n[i] < 0 || n[i] > N) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "phase2: n out of range");
    max_n = std::max(max_n, n[i]);
  }
  const int limit = rc.k_max + (rc.cap == OEA_CAP_PSEUDOCODE ? 1 : 0);
  const int stride = std::max(std::max(limit, max_n), 1);
  if (plan->set_stride < stride)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "phase2: plan set_stride too small");
  Workspace& w = extra(ctx)->ws;
  r = ensure(ctx, w, Need{B, N, 1, 1, stride});
  if (r) return r;
  cudaStream_t s = ctx->stream;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.order, order, sizeof(int32_t) * B * N, cudaMemcpyHostToDevice, s));
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.n, n, sizeof(int32_t) * B, cudaMemcpyHostToDevice, s));
  if (base_union_count > 0)
    OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.base_union, base_union, sizeof(int32_t) * base_union_count,
                                      cudaMemcpyHostToDevice, s));
  if (mask) OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.mask, mask, B, cudaMemcpyHostToDevice, s));
  r = oea_host::union_from_list_launch(ctx, w.base_union, base_union_count, N, w.union_bits, s);
  if (r) return r;
  Cfg dc = dev_cfg(rc, stride);
  oea_host::RouteBuffers rb = route_buffers(w, w.scores, mask ? w.mask : nullptr);
  rb.weights = nullptr;
  rb.weights_f32 = nullptr;
  rb.base_union = nullptr;
  rb.base_union_count = nullptr;
  r = oea_host::route_f64_launch(ctx, dc, B, N, rb, true, false, 2, true, s);
  if (r) return r;
  oea_plan_view pv = *plan;
  pv.weights = nullptr;
  pv.weights_f32 = nullptr;
  pv.order = nullptr;
  pv.phase1_t = nullptr;
  pv.phase1_n = nullptr;
  pv.base_union = nullptr;
  pv.base_union_count = nullptr;
  return export_plan(ctx, w, &pv, B, N, stride, N);
}

// ---------------------------------------------------------------------------
// Layers.
// ---------------------------------------------------------------------------
int oea_layer_create_shard(oea_ctx_t ctx, int32_t D, int32_t H, int32_t N, int32_t dtype,
                           int32_t e_begin, int32_t e_end, oea_layer_t* out) {
  CHECK_CTX(ctx);
  if (out == nullptr) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  if (D < 1 || H < 1 || N < 1)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "make_random_layer: dims must be positive");
  if (dtype != OEA_DTYPE_BF16 && dtype != OEA_DTYPE_F32 && dtype != OEA_DTYPE_F64)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "layer: unknown dtype");
  if (e_begin < 0 || e_end > N || e_begin >= e_end)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "layer shard: need 0 <= e_begin < e_end <= N");
  if ((e_begin > 0 || e_end < N) && dtype != OEA_DTYPE_BF16)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "layer shard: expert-parallel shards are bf16");
  auto* L = new oea_layer;
  L->e_begin = e_begin;
  L->n_local = e_end - e_begin;
  const int NL = L->n_local;
  L->ctx = ctx;
  L->D = D;
  L->H = H;
  L->N = N;
  L->dtype = dtype;
  L->Dp = round_up(D, kPadD);
  L->Hp = round_up(H, kPadH);
  L->Np = round_up(N, 16);
  cudaError_t e = cudaSuccess;
  if (dtype == OEA_DTYPE_BF16) {
    L->router_bytes = static_cast<size_t>(L->Np) * L->Dp * 2;
    L->w1_bytes = static_cast<size_t>(NL) * 2 * L->Dp * L->Hp * 2;
    L->w2_bytes = static_cast<size_t>(NL) * L->Dp * L->Hp * 2;
  } else {
    const size_t es = dtype == OEA_DTYPE_F64 ? 8 : 4;
    L->router_bytes = static_cast<size_t>(D) * N * es;
    L->w1_bytes = static_cast<size_t>(NL) * D * H * es;
    L->up_bytes = L->w1_bytes;
    L->w2_bytes = static_cast<size_t>(NL) * H * D * es;
  }
  e = cudaMalloc(&L->router, L->router_bytes);
  if (e == cudaSuccess && dtype == OEA_DTYPE_BF16) {
    e = cudaMalloc(&L->router_t, L->router_bytes);
    if (e == cudaSuccess) e = cudaMemsetAsync(L->router_t, 0, L->router_bytes, ctx->stream);
  }
  if (e == cudaSuccess) e = cudaMalloc(&L->w1, L->w1_bytes);
  if (e == cudaSuccess && L->up_bytes) e = cudaMalloc(&L->w_up, L->up_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&L->w2, L->w2_bytes);
  if (e == cudaSuccess) e = cudaMemsetAsync(L->router, 0, L->router_bytes, ctx->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(L->w1, 0, L->w1_bytes, ctx->stream);
  if (e == cudaSuccess && L->up_bytes) e = cudaMemsetAsync(L->w_up, 0, L->up_bytes, ctx->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(L->w2, 0, L->w2_bytes, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    oea_layer_destroy(L);
    return oea_check_cuda(ctx, e, "layer allocation");
  }
  *out = L;
  return OEA_OK;
}

int oea_layer_create(oea_ctx_t ctx, int32_t D, int32_t H, int32_t N, int32_t dtype,
                     oea_layer_t* out) {
  return oea_layer_create_shard(ctx, D, H, N, dtype, 0, N > 0 ? N : 1, out);
}

int oea_layer_destroy(oea_layer_t L) {
  if (L == nullptr) return OEA_OK;
  if (L->ctx) {
    cudaStreamSynchronize(L->ctx->stream);
    if (CtxExtra* x = extra(L->ctx)) {
      auto& v = x->host_graphs;
      for (auto& h : v)
        if (h.L == L) host_graph_release(h);
      v.erase(std::remove_if(v.begin(), v.end(), [](const HostGraph& h) { return h.L == nullptr; }),
              v.end());
    }
  }
  cudaFree(L->router);
  cudaFree(L->router_t);
  cudaFree(L->w1);
  cudaFree(L->w_up);
  cudaFree(L->w2);
  oea_host::layer_drop_umma(L);
  delete L;
  return OEA_OK;
}

static int check_dtype(oea_ctx* ctx, int dt) {
  if (dt != OEA_DTYPE_F64 && dt != OEA_DTYPE_F32 && dt != OEA_DTYPE_BF16)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "unknown dtype");
  return OEA_OK;
}

int oea_layer_upload_router(oea_layer_t L, const void* router, int32_t src_dtype,
                            int32_t src_on_device) {
  if (L == nullptr || router == nullptr) return fail(nullptr, OEA_ERR_INVALID_ARGUMENT, "null argument");
  int r = check_dtype(L->ctx, src_dtype);
  if (r) return r;
  return oea_host::layer_upload_router(L, router, src_dtype, src_on_device);
}

int oea_layer_upload_expert(oea_layer_t L, int32_t e, const void* w_gate, const void* w_up,
                            const void* w_down, int32_t src_dtype, int32_t src_on_device) {
  if (L == nullptr || !w_gate || !w_up || !w_down)
    return fail(nullptr, OEA_ERR_INVALID_ARGUMENT, "null argument");
  if (e < L->e_begin || e >= L->e_begin + L->n_local)
    return fail(L->ctx, OEA_ERR_INVALID_ARGUMENT, "expert index out of range");
  int r = check_dtype(L->ctx, src_dtype);
  if (r) return r;
  L->umma_stale = 1;
  return oea_host::layer_upload_expert(L, e, w_gate, w_up, w_down, src_dtype, src_on_device);
}

int oea_layer_init_random(oea_layer_t L, uint64_t seed) {
  if (L == nullptr) return fail(nullptr, OEA_ERR_INVALID_ARGUMENT, "null layer");
  L->umma_stale = 1;
  return oea_host::layer_init_random(L, seed);
}

int oea_layer_download_router(oea_layer_t L, void* router, int32_t dst_dtype) {
  if (L == nullptr || router == nullptr) return fail(nullptr, OEA_ERR_INVALID_ARGUMENT, "null argument");
  int r = check_dtype(L->ctx, dst_dtype);
  if (r) return r;
  return oea_host::layer_download_router(L, router, dst_dtype);
}

int oea_layer_download_expert(oea_layer_t L, int32_t e, void* w_gate, void* w_up, void* w_down,
                              int32_t dst_dtype) {
  if (L == nullptr || !w_gate || !w_up || !w_down)
    return fail(nullptr, OEA_ERR_INVALID_ARGUMENT, "null argument");
  if (e < L->e_begin || e >= L->e_begin + L->n_local)
    return fail(L->ctx, OEA_ERR_INVALID_ARGUMENT, "expert index out of range");
  int r = check_dtype(L->ctx, dst_dtype);
  if (r) return r;
  return oea_host::layer_download_expert(L, e, w_gate, w_up, w_down, dst_dtype);
}

int oea_layer_info(oea_layer_t L, int32_t* D, int32_t* H, int32_t* N, int32_t* dtype,
                   int64_t* bytes_per_expert, int64_t* device_bytes) {
  if (L == nullptr) return fail(nullptr, OEA_ERR_INVALID_ARGUMENT, "null layer");
  if (D) *D = L->D;
  if (H) *H = L->H;
  if (N) *N = L->N;
  if (dtype) *dtype = L->dtype;
  if (bytes_per_expert)
    *bytes_per_expert = static_cast<int64_t>((L->w1_bytes + L->up_bytes + L->w2_bytes) / L->n_local);
  if (device_bytes)
    *device_bytes = static_cast<int64_t>(L->router_bytes + L->w1_bytes + L->up_bytes + L->w2_bytes);
  return OEA_OK;
}

// ---------------------------------------------------------------------------
// Decode.
// ---------------------------------------------------------------------------
int oea_moe_decode(oea_ctx_t ctx, oea_layer_t L, const void* x_dev, const uint8_t* mask_dev,
                   int32_t B, const oea_routing_cfg* cfg, void* out_dev, void* stream) {
  CHECK_CTX(ctx);
  oea_routing_cfg rc;
  int r = validate_decode(ctx, L, B, cfg, &rc);
  if (r) return r;
  if (x_dev == nullptr || out_dev == nullptr)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "moe_decode: null x/out");
  Workspace& w = extra(ctx)->ws;
  r = ensure(ctx, w, need_for(L, B, stride_of(rc)));
  if (r) return r;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  ctx->last_B = B;
  ctx->last_N = L->N;
  ctx->last_stride = stride_of(rc);
  if (L->dtype == OEA_DTYPE_BF16) {
    ctx->last_kind = 1;
    return decode_bf16(ctx, w, L, x_dev, mask_dev, B, rc, out_dev, s);
  }
  ctx->last_kind = 2;
  return decode_simt(ctx, w, L, static_cast<const double*>(x_dev), mask_dev, B, rc,
                     static_cast<double*>(out_dev), s);
}

int oea_moe_decode_ep_partial(oea_ctx_t ctx, oea_layer_t L, const void* x_all_dev, int32_t B,
                              const oea_routing_cfg* cfg, int32_t world, int32_t rank,
                              float* const* recv, int32_t* const* cnt, void* stream) {
  CHECK_CTX(ctx);
  oea_routing_cfg rc;
  int r = validate_decode(ctx, L, B, cfg, &rc);
  if (r) return r;
  if (L->dtype != OEA_DTYPE_BF16)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "moe_decode_ep: bf16 layers only");
  if (world < 1 || world > oea_dev::kMaxEpWorld || rank < 0 || rank >= world || B % world != 0)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT,
                "moe_decode_ep: need 1 <= world <= 8, 0 <= rank < world and B % world == 0");
  if (x_all_dev == nullptr || recv == nullptr || cnt == nullptr)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "moe_decode_ep: null buffers");
  for (int o = 0; o < world; ++o)
    if (recv[o] == nullptr || cnt[o] == nullptr)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "moe_decode_ep: null peer buffer");
  Workspace& w = extra(ctx)->ws;
  r = ensure(ctx, w, need_for(L, B, stride_of(rc)));
  if (r) return r;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  ctx->last_B = B;
  ctx->last_N = L->N;
  ctx->last_stride = stride_of(rc);
  ctx->last_kind = 1;
  // (world == 1 keeps the combine local: out = the receive buffer itself)
  if (world == 1) return decode_bf16(ctx, w, L, x_all_dev, nullptr, B, rc, recv[0], s);
  // the peer table lives in device memory (uploaded once per distinct table,
  // outside any stream capture; later calls, captured or not, reuse it)
  oea_dev::EpPeers t{};
  for (int o = 0; o < world; ++o) {
    t.recv[o] = recv[o];
    t.cnt[o] = cnt[o];
  }
  t.world = world;
  t.rank = rank;
  t.tpr = B / world;
  constexpr int kMaxTables = 16;
  if (ctx->ep_tables == nullptr)
    OEA_CUDA_TRY(ctx, cudaMalloc(&ctx->ep_tables, kMaxTables * sizeof(oea_dev::EpPeers)));
  int slot = -1;
  for (int i = 0; i < static_cast<int>(ctx->ep_host_tables.size()); ++i)
    if (std::memcmp(&ctx->ep_host_tables[i], &t, sizeof t) == 0) slot = i;
  if (slot < 0) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs != cudaStreamCaptureStatusNone)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT,
                  "moe_decode_ep: run a new EP group once outside graph capture first");
    if (static_cast<int>(ctx->ep_host_tables.size()) >= kMaxTables)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "moe_decode_ep: too many EP groups on one context");
    slot = static_cast<int>(ctx->ep_host_tables.size());
    OEA_CUDA_TRY(ctx, cudaMemcpy(static_cast<oea_dev::EpPeers*>(ctx->ep_tables) + slot, &t,
                                 sizeof t, cudaMemcpyHostToDevice));
    ctx->ep_host_tables.push_back(t);
  }
  return decode_bf16(ctx, w, L, x_all_dev, nullptr, B, rc, nullptr, s, 0, false,
                     static_cast<const oea_dev::EpPeers*>(ctx->ep_tables) + slot);
}

int oea_ep_combine(oea_ctx_t ctx, const float* recv_local, int32_t* cnt_local, int32_t world,
                   int32_t tokens_per_rank, int32_t D, float* out_local, void* stream) {
  CHECK_CTX(ctx);
  if (recv_local == nullptr || cnt_local == nullptr || out_local == nullptr || world < 1 ||
      world > oea_dev::kMaxEpWorld || tokens_per_rank < 1 || D < 1)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "ep_combine: bad arguments");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  if (world == 1) {
    // oea_moe_decode_ep_partial with world == 1 decodes straight into
    // recv[0] (no peer stores, no arrivals to wait for): the combine is a copy
    if (recv_local != out_local)
      OEA_CUDA_TRY(ctx, cudaMemcpyAsync(out_local, recv_local,
                                        sizeof(float) * static_cast<size_t>(tokens_per_rank) * D,
                                        cudaMemcpyDeviceToDevice, s));
    return OEA_OK;
  }
  if (D % 4 != 0) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "ep_combine: D must be a multiple of 4");
  // every rank's shard decode adds the float4 quads it wrote for this owner
  return oea_host::ep_sum_launch(ctx, recv_local, cnt_local, world * tokens_per_rank * (D / 4),
                                 world, tokens_per_rank * D, out_local, s);
}

// Zero-filled device allocation of its own (IPC handles of a cudaMalloc base
// map exactly, unlike sub-allocations of a caching allocator).
int oea_device_alloc(oea_ctx_t ctx, uint64_t bytes, void** dev_ptr) {
  CHECK_CTX(ctx);
  if (dev_ptr == nullptr || bytes == 0) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "device_alloc: bad arguments");
  OEA_CUDA_TRY(ctx, cudaMalloc(dev_ptr, bytes));
  OEA_CUDA_TRY(ctx, cudaMemset(*dev_ptr, 0, bytes));
  return OEA_OK;
}

int oea_device_free(oea_ctx_t ctx, void* dev_ptr) {
  CHECK_CTX(ctx);
  if (dev_ptr) OEA_CUDA_TRY(ctx, cudaFree(dev_ptr));
  return OEA_OK;
}

int oea_ipc_close_handle(oea_ctx_t ctx, void* dev_ptr) {
  CHECK_CTX(ctx);
  if (dev_ptr) OEA_CUDA_TRY(ctx, cudaIpcCloseMemHandle(dev_ptr));
  return OEA_OK;
}

int oea_ipc_get_handle(oea_ctx_t ctx, const void* dev_ptr, void* handle) {
  CHECK_CTX(ctx);
  cudaIpcMemHandle_t h;
  OEA_CUDA_TRY(ctx, cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  std::memcpy(handle, &h, sizeof h);
  return OEA_OK;
}

int oea_ipc_open_handle(oea_ctx_t ctx, const void* handle, void** dev_ptr) {
  CHECK_CTX(ctx);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  OEA_CUDA_TRY(ctx, cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return OEA_OK;
}

// The zero-copy fused decode through the context's graph cache (see
// HostGraph). kNotFused when the shape/config is not on the fused path.
int decode_host_graph(oea_ctx* ctx, Workspace& w, oea_layer* L, const void* xd, int B,
                      const oea_routing_cfg& rc, void* od) {
  CtxExtra* ex = extra(ctx);
  cudaStream_t s = ctx->stream;
  if (ctx->ffn_trace) return decode_bf16(ctx, w, L, xd, nullptr, B, rc, od, s, 0, true);
  HostGraph* h = nullptr;
  for (auto& c : ex->host_graphs)
    if (c.L == L && c.B == B && c.ws_base == w.base &&
        std::memcmp(&c.rc, &rc, sizeof rc) == 0) {
      h = &c;
      break;
    }
  if (h == nullptr) {
    constexpr size_t kMaxHostGraphs = 16;
    if (ex->host_graphs.size() >= kMaxHostGraphs) {  // evict the least recently used
      auto lru = std::min_element(ex->host_graphs.begin(), ex->host_graphs.end(),
                                  [](const HostGraph& a, const HostGraph& b) { return a.used < b.used; });
      host_graph_release(*lru);
      ex->host_graphs.erase(lru);
    }
    HostGraph n;
    n.L = L;
    n.B = B;
    n.rc = rc;
    n.ws_base = w.base;
    const int64_t launches = ctx->launches;
    OEA_CUDA_TRY(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    const int r = decode_bf16(ctx, w, L, xd, nullptr, B, rc, od, s, 0, true);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(s, &graph);
    ctx->launches = launches;  // a capture launches nothing
    if (r != OEA_OK || e != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      return r != OEA_OK ? r : oea_check_cuda(ctx, e, "cudaStreamEndCapture");
    }
    n.graph = graph;
    size_t nn = 0;
    cudaGraphGetNodes(graph, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) cudaGraphGetNodes(graph, nodes.data(), &nn);
    cudaGraphNodeType t;
    if (nn != 1 || cudaGraphNodeGetType(nodes[0], &t) != cudaSuccess ||
        t != cudaGraphNodeTypeKernel ||
        cudaGraphKernelNodeGetParams(nodes[0], &n.kp) != cudaSuccess) {
      host_graph_release(n);
      return fail(ctx, OEA_ERR_CUDA, "moe_decode_host: unexpected decode graph");
    }
    n.node = nodes[0];
    n.params.assign(static_cast<unsigned char*>(n.kp.kernelParams[0]),
                    static_cast<unsigned char*>(n.kp.kernelParams[0]) + oea_host::ffn_params_bytes());
    const cudaError_t ie = cudaGraphInstantiate(&n.exec, graph, 0);
    if (ie != cudaSuccess) {
      host_graph_release(n);
      return oea_check_cuda(ctx, ie, "cudaGraphInstantiate");
    }
    ex->host_graphs.push_back(std::move(n));
    h = &ex->host_graphs.back();
  }
  h->used = ++ex->host_graph_clock;
  const double tp0 = g_hprof.on ? HostProfile::now() : 0.0;
  if (xd != h->x_set || od != h->out_set) {  // serving loops reuse their pinned buffers
    oea_host::ffn_params_set_io(h->params.data(), xd, od);
    h->args[0] = h->params.data();
    h->kp.kernelParams = h->args;
    h->kp.extra = nullptr;
    OEA_CUDA_TRY(ctx, cudaGraphExecKernelNodeSetParams(h->exec, h->node, &h->kp));
    h->x_set = xd;
    h->out_set = od;
  }
  const double tp1 = g_hprof.on ? HostProfile::now() : 0.0;
  OEA_CUDA_TRY(ctx, cudaGraphLaunch(h->exec, s));
  OEA_LAUNCHED(ctx);
  if (g_hprof.on) {
    g_hprof.sum[2] += tp1 - tp0;
    g_hprof.sum[3] += HostProfile::now() - tp1;
  }
  return OEA_OK;
}

// Device view of a host buffer when all of [p, p + bytes) lies in pinned,
// mapped host memory (cudaHostAlloc / cudaHostRegister, e.g. torch's
// pin_memory); nullptr for pageable memory.
const void* mapped_view(const void* p, size_t bytes) {
  cudaPointerAttributes a{}, b{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess || a.type != cudaMemoryTypeHost ||
      a.devicePointer == nullptr) {
    cudaGetLastError();
    return nullptr;
  }
  const char* last = static_cast<const char*>(p) + bytes - 1;
  if (cudaPointerGetAttributes(&b, last) != cudaSuccess || b.type != cudaMemoryTypeHost ||
      static_cast<const char*>(b.devicePointer) !=
          static_cast<const char*>(a.devicePointer) + (bytes - 1)) {
    cudaGetLastError();
    return nullptr;
  }
  return a.devicePointer;
}

int oea_moe_decode_host(oea_ctx_t ctx, oea_layer_t L, const void* x_host,
                        const uint8_t* mask_host, int32_t B, const oea_routing_cfg* cfg,
                        void* out_host) {
  CHECK_CTX(ctx);
  const double th0 = g_hprof.on ? HostProfile::now() : 0.0;
  oea_routing_cfg rc;
  int r = validate_decode(ctx, L, B, cfg, &rc);
  if (r) return r;
  if (x_host == nullptr || out_host == nullptr)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "moe_decode: null x/out");
  Workspace& w = extra(ctx)->ws;
  r = ensure(ctx, w, need_for(L, B, stride_of(rc)));
  if (r) return r;
  cudaStream_t s = ctx->stream;
  const bool bf = L->dtype == OEA_DTYPE_BF16;
  const size_t xbytes = static_cast<size_t>(B) * L->D * (bf ? 2 : 8);
  const size_t obytes = static_cast<size_t>(B) * L->D * (bf ? 4 : 8);
  ctx->last_B = B;
  ctx->last_N = L->N;
  ctx->last_stride = stride_of(rc);
  if (bf && mask_host == nullptr) {
    // Zero copy: x and out in pinned (mapped) host memory go straight to the
    // fused kernel, which stages x into HBM itself and writes out over the
    // host link; no DMA copies, one launch. Other buffers take the copies.
    const double th1 = g_hprof.on ? HostProfile::now() : 0.0;
    const void* xd = mapped_view(x_host, xbytes);
    void* od = const_cast<void*>(mapped_view(out_host, obytes));
    const double th2 = g_hprof.on ? HostProfile::now() : 0.0;
    CtxExtra* ex = extra(ctx);
    if (ex->done_flag == nullptr) {
      void* f = nullptr;
      OEA_CUDA_TRY(ctx, cudaHostAlloc(&f, 64, cudaHostAllocMapped));
      ex->done_flag = static_cast<int*>(f);
      OEA_CUDA_TRY(ctx, cudaHostGetDevicePointer(reinterpret_cast<void**>(&ex->done_flag_dev), f, 0));
    }
    if (xd != nullptr && od != nullptr) {
      ctx->last_kind = 1;
      volatile int* flag = ex->done_flag;
      *flag = 0;
      r = decode_host_graph(ctx, w, L, xd, B, rc, od);
      const double th3 = g_hprof.on ? HostProfile::now() : 0.0;
      if (r == OEA_OK && g_hprof.on && ++g_hprof.calls > 8) {  // (steady state: past the captures)
        while (*flag == 0) {
        }
        g_hprof.sum[0] += th1 - th0;
        g_hprof.sum[1] += th2 - th1;
        g_hprof.sum[4] += HostProfile::now() - th3;
        ++g_hprof.n;
      }
      if (r == OEA_OK) {
        // out is on the host once the kernel raises the flag: spin on it
        // (cheaper than a stream synchronisation's wake-up); a fault ends
        // the wait through the stream status
        for (uint32_t spin = 1;; ++spin) {
          if (*flag != 0) return OEA_OK;
          if ((spin & 1023u) == 0) {
            const cudaError_t q = cudaStreamQuery(s);
            if (q == cudaSuccess) {
              if (*flag != 0) return OEA_OK;
              return fail(ctx, OEA_ERR_CUDA, "moe_decode_host: kernel finished without completion flag");
            }
            if (q != cudaErrorNotReady) return oea_check_cuda(ctx, q, "moe_decode_host");
          }
        }
      }
      if (r != kNotFused) return r;
    }
  }
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.xin, x_host, xbytes, cudaMemcpyHostToDevice, s));
  if (mask_host) OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.mask, mask_host, B, cudaMemcpyHostToDevice, s));
  ctx->last_B = B;
  ctx->last_N = L->N;
  ctx->last_stride = stride_of(rc);
  if (bf) {
    ctx->last_kind = 1;
    r = decode_bf16(ctx, w, L, w.xin, mask_host ? w.mask : nullptr, B, rc, w.out, s);
  } else {
    ctx->last_kind = 2;
    r = decode_simt(ctx, w, L, static_cast<const double*>(w.xin), mask_host ? w.mask : nullptr, B,
                    rc, static_cast<double*>(w.out), s);
  }
  if (r) return r;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(out_host, w.out, obytes, cudaMemcpyDeviceToHost, s));
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  if (!bf) return check_domain(ctx, w, B);
  return OEA_OK;
}

int oea_last_plan_host(oea_ctx_t ctx, const oea_plan_view* plan, float* logits, double* scores) {
  CHECK_CTX(ctx);
  if (ctx->last_kind == 0) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "no decode/route has run");
  Workspace& w = extra(ctx)->ws;
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  const int B = ctx->last_B, N = ctx->last_N;
  const int order_stride = ctx->last_kind == 1 ? round_up(N, 16) : N;
  int r = export_plan(ctx, w, plan, B, N, ctx->last_stride, order_stride);
  if (r) return r;
  if (logits && ctx->last_kind == 1) {
    r = d2h_rows(ctx, logits, N, w.logits, round_up(N, 16), B, N);
    if (r) return r;
  }
  if (scores && ctx->last_kind == 2) {
    r = d2h(ctx, scores, w.scores, static_cast<size_t>(B) * N);
    if (r) return r;
  }
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return OEA_OK;
}

int oea_decode_graph_create(oea_ctx_t ctx, oea_layer_t L, const void* x_dev,
                            const uint8_t* mask_dev, int32_t B, const oea_routing_cfg* cfg,
                            void* out_dev, oea_graph_t* out) {
  CHECK_CTX(ctx);
  if (out == nullptr) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  oea_routing_cfg rc;
  int r = validate_decode(ctx, L, B, cfg, &rc);
  if (r) return r;
  Workspace& w = extra(ctx)->ws;
  r = ensure(ctx, w, need_for(L, B, stride_of(rc)));
  if (r) return r;
  // The graph binds the context workspace as sized now; later calls that need
  // a larger workspace re-allocate it, so create graphs after sizing (or
  // destroy/re-create them).
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  auto* g = new oea_graph;
  g->ctx = ctx;
  cudaStream_t s = ctx->stream;
  cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    delete g;
    return oea_check_cuda(ctx, e, "cudaStreamBeginCapture");
  }
  if (L->dtype == OEA_DTYPE_BF16)
    r = decode_bf16(ctx, w, L, x_dev, mask_dev, B, rc, out_dev, s);
  else
    r = decode_simt(ctx, w, L, static_cast<const double*>(x_dev), mask_dev, B, rc,
                    static_cast<double*>(out_dev), s);
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(s, &graph);
  if (r || e != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    delete g;
    return r ? r : oea_check_cuda(ctx, e, "cudaStreamEndCapture");
  }
  g->graph = graph;
  g->kernels = count_kernel_nodes(graph);
  e = cudaGraphInstantiate(&g->exec, graph, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(graph);
    delete g;
    return oea_check_cuda(ctx, e, "cudaGraphInstantiate");
  }
  // upload now, so the first launch does not pay it
  e = cudaGraphUpload(g->exec, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaGraphExecDestroy(g->exec);
    cudaGraphDestroy(graph);
    delete g;
    return oea_check_cuda(ctx, e, "cudaGraphUpload");
  }
  ctx->last_B = B;
  ctx->last_N = L->N;
  ctx->last_stride = stride_of(rc);
  ctx->last_kind = L->dtype == OEA_DTYPE_BF16 ? 1 : 2;
  *out = g;
  return OEA_OK;
}

int oea_decode_chain_graph_create(oea_ctx_t ctx, int32_t n, const oea_layer_t* layers,
                                  const void* const* xs_dev, const uint8_t* mask_dev, int32_t B,
                                  const oea_routing_cfg* cfg, void* const* outs_dev,
                                  oea_graph_t* out) {
  CHECK_CTX(ctx);
  if (out == nullptr || layers == nullptr || xs_dev == nullptr || outs_dev == nullptr)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  if (n < 1) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "chain graph: need n >= 1 decode calls");
  oea_routing_cfg rc;
  Workspace& w = extra(ctx)->ws;
  for (int i = 0; i < n; ++i) {
    int r = validate_decode(ctx, layers[i], B, cfg, &rc);
    if (r) return r;
    r = ensure(ctx, w, need_for(layers[i], B, stride_of(rc)));
    if (r) return r;
  }
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  auto* g = new oea_graph;
  g->ctx = ctx;
  cudaStream_t s = ctx->stream;
  cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    delete g;
    return oea_check_cuda(ctx, e, "cudaStreamBeginCapture");
  }
  // n decode calls back to back on one stream, as a decode step's layers run:
  // the fused launches carry the programmatic-serialization attribute, so the
  // captured kernel -> kernel edges are programmatic (PDL) edges.
  int r = OEA_OK;
  for (int i = 0; i < n && r == OEA_OK; ++i) {
    oea_layer* L = layers[i];
    if (L->dtype == OEA_DTYPE_BF16)
      r = decode_bf16(ctx, w, L, xs_dev[i], mask_dev, B, rc, outs_dev[i], s);
    else
      r = decode_simt(ctx, w, L, static_cast<const double*>(xs_dev[i]), mask_dev, B, rc,
                      static_cast<double*>(outs_dev[i]), s);
  }
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(s, &graph);
  if (r || e != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    delete g;
    return r ? r : oea_check_cuda(ctx, e, "cudaStreamEndCapture");
  }
  g->graph = graph;
  g->kernels = count_kernel_nodes(graph);
  e = cudaGraphInstantiate(&g->exec, graph, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(graph);
    delete g;
    return oea_check_cuda(ctx, e, "cudaGraphInstantiate");
  }
  // upload now, so the first launch does not pay it
  e = cudaGraphUpload(g->exec, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaGraphExecDestroy(g->exec);
    cudaGraphDestroy(graph);
    delete g;
    return oea_check_cuda(ctx, e, "cudaGraphUpload");
  }
  oea_layer* last = layers[n - 1];
  ctx->last_B = B;
  ctx->last_N = last->N;
  ctx->last_stride = stride_of(rc);
  ctx->last_kind = last->dtype == OEA_DTYPE_BF16 ? 1 : 2;
  *out = g;
  return OEA_OK;
}

int oea_decode_stage_graphs_create(oea_ctx_t ctx, oea_layer_t L, const void* x_dev,
                                   const uint8_t* mask_dev, int32_t B, const oea_routing_cfg* cfg,
                                   void* out_dev, oea_graph_t* router_out, oea_graph_t* ffn_out) {
  CHECK_CTX(ctx);
  if (router_out == nullptr || ffn_out == nullptr)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "null output pointer");
  *router_out = *ffn_out = nullptr;
  oea_routing_cfg rc;
  int r = validate_decode(ctx, L, B, cfg, &rc);
  if (r) return r;
  if (L->dtype != OEA_DTYPE_BF16)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "stage graphs: bf16 layers only");
  Workspace& w = extra(ctx)->ws;
  r = ensure(ctx, w, need_for(L, B, stride_of(rc)));
  if (r) return r;
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  oea_graph_t gs[2] = {nullptr, nullptr};
  for (int part = 1; part <= 2; ++part) {
    auto* g = new oea_graph;
    g->ctx = ctx;
    cudaStream_t s = ctx->stream;
    cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
      delete g;
      return oea_check_cuda(ctx, e, "cudaStreamBeginCapture");
    }
    r = decode_bf16(ctx, w, L, x_dev, mask_dev, B, rc, out_dev, s, part);
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(s, &graph);
    if (r || e != cudaSuccess || cudaGraphInstantiate(&g->exec, graph, 0) != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      delete g;
      if (gs[0]) oea_graph_destroy(gs[0]);
      return r ? r : oea_check_cuda(ctx, e == cudaSuccess ? cudaErrorUnknown : e, "stage graph");
    }
    g->graph = graph;
    g->kernels = 1;
    gs[part - 1] = g;
  }
  ctx->last_B = B;
  ctx->last_N = L->N;
  ctx->last_stride = stride_of(rc);
  ctx->last_kind = 1;
  *router_out = gs[0];
  *ffn_out = gs[1];
  return OEA_OK;
}

int oea_graph_launch(oea_graph_t g, void* stream) {
  if (g == nullptr) return fail(nullptr, OEA_ERR_INVALID_ARGUMENT, "null graph");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->ctx->stream;
  OEA_CUDA_TRY(g->ctx, cudaGraphLaunch(g->exec, s));
  g->ctx->launches += g->kernels;
  return OEA_OK;
}

int oea_graph_destroy(oea_graph_t g) {
  if (g == nullptr) return OEA_OK;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  return OEA_OK;
}

// ---------------------------------------------------------------------------
// Drop-in layer math on a given plan.
// ---------------------------------------------------------------------------
int oea_moe_forward_plan_host(oea_ctx_t ctx, oea_layer_t L, const double* x, int32_t B,
                              const int32_t* sets, const int32_t* set_len, const double* weights,
                              int32_t set_stride, const uint8_t* mask, double* out) {
  CHECK_CTX(ctx);
  if (L == nullptr || x == nullptr || out == nullptr || sets == nullptr || set_len == nullptr ||
      weights == nullptr)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "moe_forward: null argument");
  if (B < 1) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "moe_forward: plan batch size mismatch");
  if (set_stride < 1) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "moe_forward: bad set stride");
  // Plan validation (moe_layer.hpp:134-152), host-side argument checks.
  for (int i = 0; i < B; ++i) {
    if (set_len[i] < 0 || set_len[i] > set_stride)
      return fail(ctx, OEA_ERR_INVALID_ARGUMENT,
                  "moe_forward: weights/set size mismatch for token " + std::to_string(i));
    const bool real = mask == nullptr || mask[i] != 0;
    if (set_len[i] == 0) {
      if (real && mask != nullptr)
        return fail(ctx, OEA_ERR_INVALID_ARGUMENT,
                    "moe_forward: empty selected set for unmasked token " + std::to_string(i));
      continue;
    }
    for (int j = 0; j < set_len[i]; ++j) {
      const int e = sets[static_cast<size_t>(i) * set_stride + j];
      if (e < 0 || e >= L->N)
        return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "moe_forward: expert index out of range");
    }
  }
  // A caller plan may name an expert twice in one set: the reference then
  // adds w_j * y_e once per occurrence, in set order (moe_layer.hpp:146-155).
  // Each (token, expert) is computed once (the first occurrence's FFN row);
  // later occurrences are dropped from the compaction (expert -1) and the
  // fp64 set-order combine reads the first occurrence's y for them (alias).
  std::vector<int32_t> usets, alias;
  bool dups = false;
  for (int i = 0; i < B && !dups; ++i)
    for (int j = 1; j < set_len[i] && !dups; ++j)
      for (int jj = 0; jj < j; ++jj)
        if (sets[static_cast<size_t>(i) * set_stride + jj] == sets[static_cast<size_t>(i) * set_stride + j])
          dups = true;
  if (dups) {
    usets.assign(sets, sets + static_cast<size_t>(B) * set_stride);
    alias.resize(usets.size());
    for (int i = 0; i < B; ++i)
      for (int j = 0; j < set_stride; ++j) {
        const size_t o = static_cast<size_t>(i) * set_stride + j;
        alias[o] = j;
        if (j >= set_len[i]) continue;
        for (int jj = 0; jj < j; ++jj)
          if (sets[static_cast<size_t>(i) * set_stride + jj] == sets[o]) {
            alias[o] = jj;
            usets[o] = -1;
            break;
          }
      }
  }
  Workspace& w = extra(ctx)->ws;
  int r = ensure(ctx, w, need_for(L, B, set_stride));
  if (r) return r;
  cudaStream_t s = ctx->stream;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.x64, x, sizeof(double) * B * L->D, cudaMemcpyHostToDevice, s));
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.sets, dups ? usets.data() : sets,
                                    sizeof(int32_t) * B * set_stride, cudaMemcpyHostToDevice, s));
  if (dups)
    OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.alias, alias.data(), sizeof(int32_t) * B * set_stride,
                                      cudaMemcpyHostToDevice, s));
  // zero lengths of masked rows are already 0 in the caller's plan
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.set_len, set_len, sizeof(int32_t) * B, cudaMemcpyHostToDevice, s));
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.w64, weights, sizeof(double) * B * set_stride,
                                    cudaMemcpyHostToDevice, s));
  oea_host::CompactBuffers cb{w.sets, w.set_len, w.row_tok, w.row_slot, w.group_a,
                              w.group_row0, w.group_rows, w.hdr, w.counters, w.G + 7};
  r = oea_host::compact_launch(ctx, B, L->N, set_stride, cb, w.tokbits, w.active_union,
                               w.active_count, s);
  if (r) return r;
  if (L->dtype == OEA_DTYPE_BF16) {
    // weights to fp32 for the tensor-core combine; x to padded bf16
    r = oea_host::cast_f64_launch(ctx, w.w64, static_cast<size_t>(B) * set_stride, OEA_DTYPE_F32,
                                  w.w32, s);
    if (r) return r;
    k_pad_x_bf16_from_f64<<<blocks_for(static_cast<size_t>(B) * L->Dp), 256, 0, s>>>(
        w.x64, B, L->D, L->Dp, w.xpad);
    OEA_LAUNCHED(ctx);
    OEA_CUDA_TRY(ctx, cudaMemsetAsync(w.out32, 0, sizeof(float) * B * L->D, s));
    oea_host::FfnBuffers fb{};
    fb.x = w.xpad;
    fb.row_tok = w.row_tok;
    fb.row_slot = w.row_slot;
    fb.group_a = w.group_a;
    fb.group_row0 = w.group_row0;
    fb.group_rows = w.group_rows;
    fb.hdr = w.hdr;
    fb.counters = w.counters;
    fb.max_groups = w.G;
    fb.hbuf = w.hbuf;
    fb.ybuf = w.ybuf;
    fb.set_len = w.set_len;
    fb.weights_f32 = w.w32;
    fb.out = w.out32;
    r = oea_host::ffn_bf16_launch(ctx, L, B, set_stride, fb, false, s);
    if (r) return r;
    if (dups) {
      fb.alias = w.alias;
      fb.weights_f64 = w.w64;
      fb.out = w.out;
      r = oea_host::combine_alias_f32_launch(ctx, B, L->D, L->Dp, set_stride, fb, s);
      if (r) return r;
    } else {
      k_f32_to_f64<<<blocks_for(static_cast<size_t>(B) * L->D), 256, 0, s>>>(
          w.out32, static_cast<size_t>(B) * L->D, static_cast<double*>(w.out));
      OEA_LAUNCHED(ctx);
    }
  } else {
    r = oea_host::cast_f64_launch(ctx, w.x64, static_cast<size_t>(B) * L->D, L->dtype, w.xT, s);
    if (r) return r;
    oea_host::FfnBuffers fb{};
    fb.x = w.xT;
    fb.row_tok = w.row_tok;
    fb.row_slot = w.row_slot;
    fb.group_a = w.group_a;
    fb.group_row0 = w.group_row0;
    fb.group_rows = w.group_rows;
    fb.hdr = w.hdr;
    fb.hbuf = w.hbuf;
    fb.ybuf = w.ybuf;
    fb.set_len = w.set_len;
    fb.weights_f64 = w.w64;
    fb.out = w.out;
    fb.alias = dups ? w.alias : nullptr;
    r = oea_host::ffn_simt_launch(ctx, L, B, set_stride, fb, w.G, s);
    if (r) return r;
  }
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(out, w.out, sizeof(double) * B * L->D, cudaMemcpyDeviceToHost, s));
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return OEA_OK;
}

int oea_router_scores_host(oea_ctx_t ctx, oea_layer_t L, const double* x, int32_t B,
                           double* scores) {
  CHECK_CTX(ctx);
  if (L == nullptr || x == nullptr || scores == nullptr)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "router_scores: null argument");
  if (L->dtype == OEA_DTYPE_BF16)
    return fail(ctx, OEA_ERR_INVALID_ARGUMENT,
                "router_scores: bf16 layers route on fused fp32 logits; use oea_last_plan_host");
  if (B < 1) return fail(ctx, OEA_ERR_INVALID_ARGUMENT, "router_scores: batch must be >= 1");
  Workspace& w = extra(ctx)->ws;
  int r = ensure(ctx, w, need_for(L, B, 1));
  if (r) return r;
  cudaStream_t s = ctx->stream;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(w.x64, x, sizeof(double) * B * L->D, cudaMemcpyHostToDevice, s));
  r = oea_host::router_scores_launch(ctx, L, w.x64, B, w.logits64, w.scores, s);
  if (r) return r;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(scores, w.scores, sizeof(double) * B * L->N,
                                    cudaMemcpyDeviceToHost, s));
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return OEA_OK;
}

int oea_ep_owner(int32_t N, int32_t world, int32_t expert) {
  if (N < 1 || world < 1 || expert < 0 || expert >= N) return -1;
  // rank r owns experts [floor(N r / P), floor(N (r+1) / P))
  for (int r = 0; r < world; ++r) {
    const int64_t hi = static_cast<int64_t>(N) * (r + 1) / world;
    if (expert < hi) return r;
  }
  return world - 1;
}

}  // extern "C"
