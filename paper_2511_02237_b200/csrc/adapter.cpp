// adapter.cpp — liboea.so: the drop-in C++ API (include/oea/routing.hpp,
// moe_layer.hpp) implemented over the C ABI (include/oea_cuda.h).
//
// Every routing / layer computation goes to the GPU kernels through the C ABI;
// the adapter only marshals Eigen containers to flat buffers and rethrows the
// ABI's status as the reference's exception types with its messages. Host-side
// pieces are exactly those the reference keeps on the host as well: input
// validation (ScoreMatrix::validate), config factories, recounting a
// host-resident plan (batch_stats), the seeded input generators
// (make_random_layer / make_random_batch, bit-identical to the reference),
// the divergence metric and JSON save/load.
//
// One context per host thread (the reference's functions are reentrant and
// are called from a thread pool, simulate.cpp:142-150).
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>

#include "oea/moe_layer.hpp"
#include "oea/routing.hpp"
#include "oea_cuda.h"

namespace oea {

namespace {

struct ThreadCtx {
  oea_ctx_t h = nullptr;
  ~ThreadCtx() {
    if (h) oea_ctx_destroy(h);
  }
};
thread_local ThreadCtx t_ctx;

[[noreturn]] void rethrow(int rc, const std::string& msg) {
  if (rc == OEA_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == OEA_ERR_DOMAIN) throw std::domain_error(msg);
  throw std::runtime_error("oea: " + msg);
}

oea_ctx_t ctx() {
  if (t_ctx.h == nullptr) {
    const char* dev = std::getenv("OEA_DEVICE");
    const int rc = oea_ctx_create(dev ? std::atoi(dev) : 0, &t_ctx.h);
    if (rc != OEA_OK) {
      t_ctx.h = nullptr;
      rethrow(rc, oea_last_error(nullptr));
    }
  }
  return t_ctx.h;
}

void check(int rc, oea_ctx_t c) {
  if (rc != OEA_OK) rethrow(rc, oea_last_error(c));
}

oea_routing_cfg to_c(const RoutingConfig& c) {
  oea_routing_cfg o;
  o.mode = static_cast<int32_t>(c.mode);
  o.k = c.k;
  o.k0 = c.k0;
  o.p = c.p;
  o.k_max = c.k_max;
  o.max_p = c.max_p;
  o.cap = static_cast<int32_t>(c.cap);
  return o;
}

RoutingConfig from_c(const oea_routing_cfg& o) {
  RoutingConfig c;
  c.mode = static_cast<RoutingMode>(o.mode);
  c.k = o.k;
  c.k0 = o.k0;
  c.p = o.p;
  c.k_max = o.k_max;
  c.max_p = o.max_p;
  c.cap = static_cast<CapSemantics>(o.cap);
  return c;
}

std::vector<uint8_t> mask_bytes(const ScoreMatrix& s) {
  std::vector<uint8_t> m;
  if (s.mask.size() != 0) {
    m.resize(static_cast<std::size_t>(s.batch()));
    for (Eigen::Index i = 0; i < s.batch(); ++i)
      m[static_cast<std::size_t>(i)] = (i < s.mask.size() && s.mask[i]) ? 1 : 0;
  }
  return m;
}

// Flat plan buffers -> RoutingPlan.
struct FlatPlan {
  int B = 0, N = 0, stride = 1;
  std::vector<int32_t> sets, set_len, loads, active;
  std::vector<double> weights;
  int32_t active_count = 0;
  int64_t total_load = 0;
  oea_plan_view view() {
    oea_plan_view v{};
    v.set_stride = stride;
    v.sets = sets.data();
    v.set_len = set_len.data();
    v.weights = weights.empty() ? nullptr : weights.data();
    v.loads = loads.data();
    v.active_union = active.data();
    v.active_count = &active_count;
    v.total_load = &total_load;
    return v;
  }
  FlatPlan(int b, int n, int s, bool with_weights) : B(b), N(n), stride(s < 1 ? 1 : s) {
    sets.assign(static_cast<std::size_t>(B) * stride, -1);
    set_len.assign(static_cast<std::size_t>(B), 0);
    loads.assign(static_cast<std::size_t>(N), 0);
    active.assign(static_cast<std::size_t>(N), -1);
    if (with_weights) weights.assign(static_cast<std::size_t>(B) * stride, 0.0);
  }
  RoutingPlan to_plan(bool with_weights) const {
    RoutingPlan p;
    p.n_experts = N;
    p.sets.resize(static_cast<std::size_t>(B));
    if (with_weights) p.weights.resize(static_cast<std::size_t>(B));
    for (int i = 0; i < B; ++i) {
      const int len = set_len[static_cast<std::size_t>(i)];
      for (int j = 0; j < len; ++j) {
        p.sets[static_cast<std::size_t>(i)].push_back(sets[static_cast<std::size_t>(i) * stride + j]);
        if (with_weights)
          p.weights[static_cast<std::size_t>(i)].push_back(weights[static_cast<std::size_t>(i) * stride + j]);
      }
    }
    p.loads = Eigen::VectorXi::Zero(N);
    for (int e = 0; e < N; ++e) p.loads[e] = loads[static_cast<std::size_t>(e)];
    for (int a = 0; a < active_count; ++a) p.active_union.push_back(active[static_cast<std::size_t>(a)]);
    p.active_count = active_count;
    p.total_load = static_cast<long>(total_load);
    return p;
  }
};

}  // namespace

// ---- host validation and configuration -------------------------------------
void ScoreMatrix::validate() const {
  if (scores.rows() < 1 || scores.cols() < 1)
    throw std::invalid_argument("ScoreMatrix: dimensions must be >= 1");
  if (mask.size() != 0 && mask.size() != scores.rows())
    throw std::invalid_argument("ScoreMatrix: mask length " + std::to_string(mask.size()) +
                                " does not match batch size " + std::to_string(scores.rows()));
  for (Eigen::Index i = 0; i < scores.rows(); ++i) {
    double sum = 0.0;
    for (Eigen::Index j = 0; j < scores.cols(); ++j) {
      const double v = scores(i, j);
      if (!std::isfinite(v) || v < 0.0)
        throw std::invalid_argument("ScoreMatrix: row " + std::to_string(i) +
                                    " has a negative or non-finite score");
      sum += v;
    }
    if (is_real(i) && std::abs(sum - 1.0) > 1e-6)
      throw std::invalid_argument("ScoreMatrix: row " + std::to_string(i) +
                                  " is off the simplex (sum = " + std::to_string(sum) + ")");
  }
}

const char* to_string(RoutingMode mode) {
  switch (mode) {
    case RoutingMode::Vanilla: return "vanilla";
    case RoutingMode::Pruned: return "pruned";
    case RoutingMode::Oea: return "oea";
    case RoutingMode::SimplifiedOea: return "simplified";
  }
  return "?";
}

const char* to_string(CapSemantics cap) {
  return cap == CapSemantics::ExactCap ? "exact" : "pseudocode";
}

RoutingMode routing_mode_from_string(const std::string& s) {
  for (const RoutingMode m : {RoutingMode::Vanilla, RoutingMode::Pruned, RoutingMode::Oea,
                              RoutingMode::SimplifiedOea})
    if (s == to_string(m)) return m;
  throw std::invalid_argument("unknown routing mode: " + s);
}

CapSemantics cap_semantics_from_string(const std::string& s) {
  for (const CapSemantics c : {CapSemantics::ExactCap, CapSemantics::PseudocodeStrict})
    if (s == to_string(c)) return c;
  throw std::invalid_argument("unknown cap semantics: " + s);
}

RoutingConfig RoutingConfig::vanilla(int k) {
  RoutingConfig c;
  c.mode = RoutingMode::Vanilla;
  c.k = c.k0 = c.k_max = k;
  return c;
}

RoutingConfig RoutingConfig::pruned(int k0, double p, int k) {
  RoutingConfig c;
  c.mode = RoutingMode::Pruned;
  c.k = k;
  c.k0 = k0;
  c.p = p;
  c.k_max = k0 > k ? k0 : k;
  return c;
}

RoutingConfig RoutingConfig::oea(int k0, double p, int k_max, int max_p, int k, CapSemantics cap) {
  RoutingConfig c;
  c.mode = RoutingMode::Oea;
  c.k = k;
  c.k0 = k0;
  c.p = p;
  c.k_max = k_max;
  c.max_p = max_p;
  c.cap = cap;
  return c;
}

RoutingConfig RoutingConfig::simplified(int k0, int k, CapSemantics cap) {
  RoutingConfig c;
  c.mode = RoutingMode::SimplifiedOea;
  c.k = k;
  c.k0 = k0;
  c.p = 1.0;
  c.k_max = k;
  c.max_p = 0;
  c.cap = cap;
  return c;
}

RoutingConfig RoutingConfig::resolved(int n_experts) const {
  const oea_routing_cfg in = to_c(*this);
  oea_routing_cfg out;
  const int rc = oea_config_resolve(&in, n_experts, &out);
  if (rc != OEA_OK) rethrow(rc, oea_last_error(nullptr));
  return from_c(out);
}

// ---- routing on the GPU (kernel family K1) ---------------------------------
SortedExperts sort_experts(const ScoreMatrix& scores) {
  const int B = static_cast<int>(scores.batch()), N = static_cast<int>(scores.experts());
  if (B < 1 || N < 1) throw std::invalid_argument("sort_experts: dimensions must be >= 1");
  SortedExperts out;
  out.order.resize(B, N);
  oea_ctx_t c = ctx();
  check(oea_sort_experts_f64_host(c, scores.scores.data(), B, N, out.order.data()), c);
  return out;
}

RoutingPlan route_topk(const ScoreMatrix& scores, int k) {
  const int n = static_cast<int>(scores.experts());
  if (k < 1 || k > n) throw std::invalid_argument("route_topk: k must be in [1, N]");
  return route(scores, RoutingConfig::vanilla(k));
}

RoutingPlan route(const ScoreMatrix& scores, const RoutingConfig& cfg) {
  const int B = static_cast<int>(scores.batch()), N = static_cast<int>(scores.experts());
  const RoutingConfig rc = cfg.resolved(N);
  const oea_routing_cfg crc = to_c(rc);
  FlatPlan fp(B, N, oea_plan_set_stride(&crc), true);
  const std::vector<uint8_t> m = mask_bytes(scores);
  oea_plan_view v = fp.view();
  oea_ctx_t c = ctx();
  const oea_routing_cfg raw = to_c(cfg);
  check(oea_route_f64_host(c, scores.scores.data(), m.empty() ? nullptr : m.data(), B, N, &raw, &v),
        c);
  return fp.to_plan(true);
}

Phase1Result phase1_baseline(const ScoreMatrix& scores, const SortedExperts& sorted,
                             const RoutingConfig& cfg) {
  const int B = static_cast<int>(scores.batch()), N = static_cast<int>(scores.experts());
  const RoutingConfig rc = cfg.resolved(N);
  Phase1Result res;
  res.t = Eigen::VectorXi::Zero(B);
  res.n = Eigen::VectorXi::Zero(B);
  res.base_sets.assign(static_cast<std::size_t>(B), {});
  if (B == 0) return res;
  const int k0 = rc.k0 < 1 ? 1 : rc.k0;
  std::vector<int32_t> base(static_cast<std::size_t>(B) * k0, -1), bu(static_cast<std::size_t>(N));
  int32_t bucount = 0;
  const std::vector<uint8_t> m = mask_bytes(scores);
  const oea_routing_cfg raw = to_c(cfg);
  oea_ctx_t c = ctx();
  check(oea_phase1_f64_host(c, scores.scores.data(), m.empty() ? nullptr : m.data(), B, N,
                            sorted.order.data(), &raw, res.t.data(), res.n.data(), base.data(), k0,
                            bu.data(), &bucount),
        c);
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < res.n[i]; ++j)
      res.base_sets[static_cast<std::size_t>(i)].push_back(base[static_cast<std::size_t>(i) * k0 + j]);
  res.base_union.assign(bu.begin(), bu.begin() + bucount);
  return res;
}

RoutingPlan phase2_piggyback(const ScoreMatrix& scores, const SortedExperts& sorted,
                             const Phase1Result& phase1, const RoutingConfig& cfg) {
  const int B = static_cast<int>(scores.batch()), N = static_cast<int>(scores.experts());
  const RoutingConfig rc = cfg.resolved(N);
  RoutingPlan empty;
  empty.n_experts = N;
  if (B == 0) {
    empty.loads = Eigen::VectorXi::Zero(N);
    return empty;
  }
  int max_n = 0;
  for (int i = 0; i < B; ++i) max_n = std::max(max_n, static_cast<int>(phase1.n[i]));
  const int stride = std::max(std::max(rc.k_max + (rc.cap == CapSemantics::PseudocodeStrict ? 1 : 0), max_n), 1);
  FlatPlan fp(B, N, stride, false);
  oea_plan_view v = fp.view();
  const std::vector<uint8_t> m = mask_bytes(scores);
  const oea_routing_cfg raw = to_c(cfg);
  std::vector<int32_t> n(phase1.n.data(), phase1.n.data() + B);
  oea_ctx_t c = ctx();
  check(oea_phase2_f64_host(c, m.empty() ? nullptr : m.data(), B, N, sorted.order.data(), n.data(),
                            phase1.base_union.data(), static_cast<int32_t>(phase1.base_union.size()),
                            &raw, &v),
        c);
  RoutingPlan p = fp.to_plan(false);
  p.weights.clear();  // phase 2 leaves weights empty, as in the reference
  return p;
}

BatchStats batch_stats(const RoutingPlan& plan) {
  BatchStats st;
  st.loads = Eigen::VectorXi::Zero(plan.n_experts);
  for (const auto& set : plan.sets) {
    for (const int e : set) ++st.loads[e];
    st.total_load += static_cast<long>(set.size());
  }
  st.active_count = static_cast<int>((st.loads.array() > 0).count());
  return st;
}

// ---- layer math on the GPU (SIMT kernels in the Scalar precision) ----------
namespace detail {

namespace {

struct DeviceLayer {
  oea_layer_t h = nullptr;
  ~DeviceLayer() {
    if (h) oea_layer_destroy(h);
  }
};

// experts: which experts' weights to upload (null: none). moe_forward reads
// only the experts its plan names, so only those cross the host link (the
// others stay unwritten device memory that no kernel reads).
void upload(const LayerView& v, DeviceLayer& dl, bool router, const std::vector<char>* experts) {
  oea_ctx_t c = ctx();
  check(oea_layer_create(c, v.D, v.H < 1 ? 1 : v.H, v.N, v.dtype, &dl.h), c);
  if (router && v.router) check(oea_layer_upload_router(dl.h, v.router, v.dtype, 0), c);
  if (experts)
    for (int e = 0; e < static_cast<int>(v.gate.size()); ++e)
      if ((*experts)[static_cast<std::size_t>(e)])
        check(oea_layer_upload_expert(dl.h, e, v.gate[static_cast<std::size_t>(e)],
                                      v.up[static_cast<std::size_t>(e)],
                                      v.down[static_cast<std::size_t>(e)], v.dtype, 0),
              c);
}

}  // namespace

void router_scores_device(const LayerView& layer, const double* x, int B, double* scores) {
  if (B == 0) return;
  DeviceLayer dl;
  upload(layer, dl, true, nullptr);
  oea_ctx_t c = ctx();
  check(oea_router_scores_host(c, dl.h, x, B, scores), c);
}

void moe_forward_device(const LayerView& layer, const double* x, int B,
                        const std::vector<int>& sets, const std::vector<int>& set_len,
                        const std::vector<double>& weights, int stride, const bool* mask,
                        double* out) {
  if (B == 0) return;
  std::vector<char> used(layer.gate.size(), 0);
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < set_len[static_cast<std::size_t>(i)] && j < stride; ++j) {
      const int e = sets[static_cast<std::size_t>(i) * stride + j];
      if (e >= 0 && e < static_cast<int>(used.size())) used[static_cast<std::size_t>(e)] = 1;
    }
  DeviceLayer dl;
  upload(layer, dl, false, &used);
  std::vector<int32_t> s(sets.begin(), sets.end()), l(set_len.begin(), set_len.end());
  oea_ctx_t c = ctx();
  check(oea_moe_forward_plan_host(c, dl.h, x, B, s.data(), l.data(), weights.data(), stride,
                                  reinterpret_cast<const uint8_t*>(mask), out),
        c);
}

}  // namespace detail

// ---- metric, generators, JSON (host, as in the reference) ------------------
Divergence output_divergence(const RowMatrixXd& ref, const RowMatrixXd& test) {
  if (ref.rows() != test.rows() || ref.cols() != test.cols())
    throw std::invalid_argument("output_divergence: shape mismatch");
  if (ref.rows() == 0) throw std::invalid_argument("output_divergence: empty input");
  Divergence d;
  double total = 0.0;
  for (Eigen::Index i = 0; i < ref.rows(); ++i) {
    double nr = 0.0, nd = 0.0;
    for (Eigen::Index j = 0; j < ref.cols(); ++j) {
      const double a = ref(i, j), b = test(i, j);
      nr += a * a;
      nd += (a - b) * (a - b);
    }
    const double rel = std::sqrt(nd) / std::max(std::sqrt(nr), 1e-12);
    total += rel;
    d.max_relative_error = std::max(d.max_relative_error, rel);
  }
  d.mean_relative_error = total / static_cast<double>(ref.rows());
  return d;
}

MoeLayerParams<double> make_random_layer(const LayerDims& dims, std::uint64_t seed) {
  if (dims.embed < 1 || dims.hidden < 1 || dims.experts < 1)
    throw std::invalid_argument("make_random_layer: dims must be positive");
  const double ds = 1.0 / std::sqrt(static_cast<double>(dims.embed));
  const double hs = 1.0 / std::sqrt(static_cast<double>(dims.hidden));
  CounterRng rng(stream_key({seed, 101}));
  auto fill = [&rng](DenseMatrix<double>& m, int rows, int cols, double scale) {
    m.resize(rows, cols);
    for (Eigen::Index i = 0; i < m.size(); ++i) m.data()[i] = scale * rng.next_normal();
  };
  MoeLayerParams<double> L;
  fill(L.router, dims.embed, dims.experts, ds);
  L.experts.resize(static_cast<std::size_t>(dims.experts));
  for (auto& ex : L.experts) {
    fill(ex.w_gate, dims.embed, dims.hidden, ds);
    fill(ex.w_up, dims.embed, dims.hidden, ds);
    fill(ex.w_down, dims.hidden, dims.embed, hs);
  }
  return L;
}

TokenBatch make_random_batch(int batch, int embed_dim, std::uint64_t seed, int step, int layer) {
  if (batch < 1 || embed_dim < 1) throw std::invalid_argument("make_random_batch: dims must be positive");
  TokenBatch out;
  out.embeddings.resize(batch, embed_dim);
  for (int i = 0; i < batch; ++i) {
    CounterRng rng(seed, static_cast<std::uint64_t>(step), static_cast<std::uint64_t>(layer),
                   static_cast<std::uint64_t>(i), 102);
    for (int c = 0; c < embed_dim; ++c) out.embeddings(i, c) = rng.next_normal();
  }
  return out;
}

namespace {

nlohmann::json to_json(const DenseMatrix<double>& m) {
  nlohmann::json rows = nlohmann::json::array();
  for (Eigen::Index r = 0; r < m.rows(); ++r) {
    nlohmann::json row = nlohmann::json::array();
    for (Eigen::Index c = 0; c < m.cols(); ++c) row.push_back(m(r, c));
    rows.push_back(std::move(row));
  }
  return rows;
}

DenseMatrix<double> from_json(const nlohmann::json& j, int rows, int cols, const std::string& what) {
  if (!j.is_array() || static_cast<int>(j.size()) != rows)
    throw std::invalid_argument("load_layer_json: bad row count for " + what);
  DenseMatrix<double> m(rows, cols);
  for (int r = 0; r < rows; ++r) {
    const auto& row = j[static_cast<std::size_t>(r)];
    if (!row.is_array() || static_cast<int>(row.size()) != cols)
      throw std::invalid_argument("load_layer_json: bad column count for " + what + " row " +
                                  std::to_string(r));
    for (int c = 0; c < cols; ++c) m(r, c) = row[static_cast<std::size_t>(c)].get<double>();
  }
  return m;
}

}  // namespace

void save_layer_json(const std::string& path, const MoeLayerParams<double>& layer) {
  nlohmann::json j;
  j["schema_version"] = 1;
  j["type"] = "moe_layer";
  j["embed_dim"] = layer.embed_dim();
  j["hidden_dim"] = layer.hidden_dim();
  j["n_experts"] = layer.expert_count();
  j["router"] = to_json(layer.router);
  nlohmann::json ex = nlohmann::json::array();
  for (const auto& e : layer.experts)
    ex.push_back({{"w_gate", to_json(e.w_gate)}, {"w_up", to_json(e.w_up)}, {"w_down", to_json(e.w_down)}});
  j["experts"] = std::move(ex);
  std::ofstream f(path);
  if (!f) throw std::invalid_argument("save_layer_json: cannot open " + path);
  f << j.dump() << "\n";
}

MoeLayerParams<double> load_layer_json(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw std::invalid_argument("load_layer_json: cannot open " + path);
  nlohmann::json j;
  try {
    f >> j;
  } catch (const nlohmann::json::parse_error& e) {
    throw std::invalid_argument("load_layer_json: parse error in " + path + ": " + e.what());
  }
  if (j.value("schema_version", 0) != 1 || j.value("type", "") != std::string("moe_layer"))
    throw std::invalid_argument("load_layer_json: unsupported schema in " + path);
  const int d = j.at("embed_dim").get<int>(), h = j.at("hidden_dim").get<int>(),
            n = j.at("n_experts").get<int>();
  if (d < 1 || h < 1 || n < 1) throw std::invalid_argument("load_layer_json: non-positive dims in " + path);
  MoeLayerParams<double> L;
  L.router = from_json(j.at("router"), d, n, "router");
  const auto& ex = j.at("experts");
  if (!ex.is_array() || static_cast<int>(ex.size()) != n)
    throw std::invalid_argument("load_layer_json: expert count mismatch");
  L.experts.resize(static_cast<std::size_t>(n));
  for (int e = 0; e < n; ++e) {
    const std::string tag = "expert " + std::to_string(e);
    const auto& je = ex[static_cast<std::size_t>(e)];
    L.experts[static_cast<std::size_t>(e)].w_gate = from_json(je.at("w_gate"), d, h, tag + " w_gate");
    L.experts[static_cast<std::size_t>(e)].w_up = from_json(je.at("w_up"), d, h, tag + " w_up");
    L.experts[static_cast<std::size_t>(e)].w_down = from_json(je.at("w_down"), h, d, tag + " w_down");
  }
  return L;
}

}  // namespace oea
