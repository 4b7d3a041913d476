// oea/device_layer.hpp — C++ RAII interface to the resident bf16 decode hot
// path (the fused single-launch OEA MoE layer) of the B200-native library.
//
// The reference has no device-resident layer: its decode cell is
// router_scores -> route -> moe_forward on host matrices
// (proj/src/simulate.cpp:181-189 over proj/include/oea/moe_layer.hpp:71-158).
// oea/moe_layer.hpp keeps that drop-in API (host matrices in, host matrices
// out); this header is what a C++ serving loop uses instead: the layer's
// weights stay in HBM, tokens and outputs are device (or pinned host)
// buffers, and a decode is one kernel launch (or one CUDA-graph replay).
//
// Header-only over include/oea_cuda.h (link liboea_cuda.so). Errors throw the
// reference's exception types with the C ABI's message: std::invalid_argument
// (OEA_ERR_INVALID_ARGUMENT), std::domain_error (OEA_ERR_DOMAIN), else
// std::runtime_error. No Eigen dependency: RoutingConfig here is the C ABI's
// field-for-field struct; oea::RoutingConfig (routing.hpp) converts with
// to_c().
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "oea_cuda.h"

namespace oea {
namespace device {

[[noreturn]] inline void throw_status(int rc, const char* msg) {
  const std::string m = msg ? msg : "oea: unknown error";
  if (rc == OEA_ERR_INVALID_ARGUMENT) throw std::invalid_argument(m);
  if (rc == OEA_ERR_DOMAIN) throw std::domain_error(m);
  throw std::runtime_error("oea: " + m);
}

// Routing configuration of the C ABI (oea_routing_cfg, routing.hpp:56-76).
struct Routing {
  oea_routing_cfg c{};
  static Routing vanilla(int k) { return make(OEA_MODE_VANILLA, k, k, k); }
  static Routing simplified(int k0, int k) { return make(OEA_MODE_SIMPLIFIED, k, k0, k); }
  static Routing oea(int k0, int k_max, double p = 1.0, int k = 8, int max_p = 0) {
    Routing r = make(OEA_MODE_OEA, k, k0, k_max);
    r.c.p = p;
    r.c.max_p = max_p;
    return r;
  }

 private:
  static Routing make(int mode, int k, int k0, int k_max) {
    Routing r;
    r.c.mode = mode;
    r.c.k = k;
    r.c.k0 = k0;
    r.c.p = 1.0;
    r.c.k_max = k_max;
    r.c.max_p = 0;
    r.c.cap = OEA_CAP_EXACT;
    return r;
  }
};

// One CUDA stream + workspace on one device (oea_ctx_t).
class Context {
 public:
  explicit Context(int device = 0) {
    const int rc = oea_ctx_create(device, &h_);
    if (rc != OEA_OK) throw_status(rc, oea_last_error(nullptr));
  }
  ~Context() {
    if (h_) oea_ctx_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  Context(Context&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}

  oea_ctx_t handle() const { return h_; }
  void check(int rc) const {
    if (rc != OEA_OK) throw_status(rc, oea_last_error(h_));
  }
  void* stream() const {
    void* s = nullptr;
    check(oea_ctx_stream(h_, &s));
    return s;
  }
  void synchronize() const { check(oea_ctx_synchronize(h_)); }
  int64_t kernel_launches() const { return oea_ctx_kernel_launches(h_); }

 private:
  oea_ctx_t h_ = nullptr;
};

// A captured decode (one call, or n calls back to back with PDL edges).
class Graph {
 public:
  Graph(const Context& ctx, oea_graph_t g) : ctx_(&ctx), g_(g) {}
  ~Graph() {
    if (g_) oea_graph_destroy(g_);
  }
  Graph(const Graph&) = delete;
  Graph& operator=(const Graph&) = delete;
  Graph(Graph&& o) noexcept : ctx_(o.ctx_), g_(std::exchange(o.g_, nullptr)) {}
  // stream nullptr: the context's stream
  void launch(void* stream = nullptr) const { ctx_->check(oea_graph_launch(g_, stream)); }

 private:
  const Context* ctx_;
  oea_graph_t g_ = nullptr;
};

// A device-resident MoE layer (oea_layer_t): router [D x N] and N SwiGLU
// experts (w_gate, w_up: D x H, w_down: H x D), stored as `dtype` in HBM.
// experts [e_begin, e_end) < [0, N): an expert-parallel shard (its decode
// writes the partial mixture over the experts it holds).
class Layer {
 public:
  Layer(const Context& ctx, int D, int H, int N, oea_dtype dtype = OEA_DTYPE_BF16,
        int e_begin = 0, int e_end = -1)
      : ctx_(&ctx), D_(D), N_(N) {
    ctx.check(oea_layer_create_shard(ctx.handle(), D, H, N, dtype, e_begin,
                                     e_end < 0 ? N : e_end, &h_));
  }
  ~Layer() {
    if (h_) oea_layer_destroy(h_);
  }
  Layer(const Layer&) = delete;
  Layer& operator=(const Layer&) = delete;
  Layer(Layer&& o) noexcept : ctx_(o.ctx_), D_(o.D_), N_(o.N_), h_(std::exchange(o.h_, nullptr)) {}

  oea_layer_t handle() const { return h_; }
  int embed() const { return D_; }
  int experts() const { return N_; }

  // make_random_layer's distributions (moe_layer.cpp), generated on the device.
  void init_random(uint64_t seed) { ctx_->check(oea_layer_init_random(h_, seed)); }
  // Host weights of src_dtype (row-major, reference layouts).
  void upload_router(const void* router_DxN, oea_dtype src_dtype) {
    ctx_->check(oea_layer_upload_router(h_, router_DxN, src_dtype, 0));
  }
  void upload_expert(int e, const void* w_gate, const void* w_up, const void* w_down,
                     oea_dtype src_dtype) {
    ctx_->check(oea_layer_upload_expert(h_, e, w_gate, w_up, w_down, src_dtype, 0));
  }

  // THE hot path: x_dev [B x D] bf16 -> out_dev [B x D] fp32 (bf16 layers),
  // asynchronous on `stream` (nullptr: the context's stream). mask_dev: B
  // bytes (0 = padding row) or nullptr.
  void decode(const void* x_dev, int B, const Routing& cfg, void* out_dev,
              void* stream = nullptr, const uint8_t* mask_dev = nullptr) const {
    ctx_->check(oea_moe_decode(ctx_->handle(), h_, x_dev, mask_dev, B, &cfg.c, out_dev, stream));
  }
  // End to end from host (pinned or pageable) buffers; returns when out is on
  // the host. bf16 layers: x as bf16 bits (uint16), out fp32.
  void decode_host(const uint16_t* x_host, int B, const Routing& cfg, float* out_host,
                   const uint8_t* mask_host = nullptr) const {
    ctx_->check(oea_moe_decode_host(ctx_->handle(), h_, x_host, mask_host, B, &cfg.c, out_host));
  }
  // One decode captured as a CUDA graph (fixed pointers, B and cfg).
  Graph graph(const void* x_dev, int B, const Routing& cfg, void* out_dev,
              const uint8_t* mask_dev = nullptr) const {
    oea_graph_t g = nullptr;
    ctx_->check(oea_decode_graph_create(ctx_->handle(), h_, x_dev, mask_dev, B, &cfg.c, out_dev,
                                        &g));
    return Graph(*ctx_, g);
  }

  // The most recent decode's routing (synchronises): sets [B x stride],
  // set lengths, fp64 weights, the union of active experts (ascending).
  struct Plan {
    int stride = 0;
    std::vector<int32_t> sets, set_len, active;
    std::vector<double> weights;
    std::vector<float> logits;  // [B x N] router logits (fp32, bf16 layers)
    int64_t total_load = 0;
  };
  Plan last_plan(int B, const Routing& cfg) const {
    oea_routing_cfg rc{};
    ctx_->check(oea_config_resolve(&cfg.c, N_, &rc));
    Plan p;
    p.stride = oea_plan_set_stride(&rc);
    if (p.stride < 1) p.stride = 1;
    p.sets.assign(static_cast<size_t>(B) * p.stride, -1);
    p.set_len.assign(static_cast<size_t>(B), 0);
    p.weights.assign(static_cast<size_t>(B) * p.stride, 0.0);
    p.active.assign(static_cast<size_t>(N_), -1);
    p.logits.assign(static_cast<size_t>(B) * N_, 0.0f);
    int32_t count = 0;
    oea_plan_view v{};
    v.set_stride = p.stride;
    v.sets = p.sets.data();
    v.set_len = p.set_len.data();
    v.weights = p.weights.data();
    v.active_union = p.active.data();
    v.active_count = &count;
    v.total_load = &p.total_load;
    ctx_->check(oea_last_plan_host(ctx_->handle(), &v, p.logits.data(), nullptr));
    p.active.resize(static_cast<size_t>(count));
    return p;
  }

 private:
  const Context* ctx_;
  int D_, N_;
  oea_layer_t h_ = nullptr;
};

// n decode calls (layers[i]: xs[i] -> outs[i]) back to back in ONE graph, the
// fused launches chained with programmatic dependent launch.
inline Graph chain_graph(const Context& ctx, const std::vector<const Layer*>& layers,
                         const std::vector<const void*>& xs, int B, const Routing& cfg,
                         const std::vector<void*>& outs, const uint8_t* mask_dev = nullptr) {
  if (layers.empty() || layers.size() != xs.size() || layers.size() != outs.size())
    throw std::invalid_argument("chain_graph: need matching non-empty layers / xs / outs");
  std::vector<oea_layer_t> hs;
  for (const Layer* l : layers) hs.push_back(l->handle());
  oea_graph_t g = nullptr;
  ctx.check(oea_decode_chain_graph_create(ctx.handle(), static_cast<int32_t>(hs.size()), hs.data(),
                                          xs.data(), mask_dev, B, &cfg.c, outs.data(), &g));
  return Graph(ctx, g);
}

}  // namespace device
}  // namespace oea
