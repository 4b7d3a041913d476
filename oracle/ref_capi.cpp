// ref_capi.cpp — extern "C" entry points into the reference implementation
// compiled from /root/reference/proj sources (oracle/Makefile -> oracle/_ref).
//
// TEST INFRASTRUCTURE ONLY: used by tests/golden/make_golden.py to produce the
// committed golden vectors, by tests/test_oracle.py to pin the C restatement
// against the real reference when oracle/_ref exists, and by bench.py
// --impl reference (the reference's own CPU path on the GPU box's host).
//
// Every function converts flat arrays to the reference's Eigen-typed structs,
// calls the reference function unchanged, and flattens the result. Exceptions
// become status codes: 1 std::invalid_argument, 2 std::domain_error, 3 other.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "oea/latency.hpp"
#include "oea/moe_layer.hpp"
#include "oea/routing.hpp"
#include "oea/score_gen.hpp"
#include "oea/simulate.hpp"
#include "oea/sweep.hpp"
#include "oracle.hpp"

#include <thread>

extern "C" double oo_stream_normal(uint64_t key, uint64_t f);
extern "C" uint64_t oo_stream_key(const uint64_t* parts, int32_t n);

using namespace oea;

namespace {

thread_local std::string g_err;

int record(int code, const char* what) {
  g_err = what;
  return code;
}

#define REF_GUARD(body)                                          \
  try {                                                          \
    body;                                                        \
    return 0;                                                    \
  } catch (const std::domain_error& e) {                         \
    return record(2, e.what());                                  \
  } catch (const std::invalid_argument& e) {                     \
    return record(1, e.what());                                  \
  } catch (const std::exception& e) {                            \
    return record(3, e.what());                                  \
  }

RoutingConfig make_cfg(int mode, int k, int k0, double p, int k_max, int max_p, int cap) {
  RoutingConfig c;
  c.mode = static_cast<RoutingMode>(mode);
  c.k = k;
  c.k0 = k0;
  c.p = p;
  c.k_max = k_max;
  c.max_p = max_p;
  c.cap = static_cast<CapSemantics>(cap);
  return c;
}

ScoreMatrix make_scores(const double* s, const uint8_t* mask, int B, int N) {
  ScoreMatrix m;
  m.scores.resize(B, N);
  std::memcpy(m.scores.data(), s, sizeof(double) * B * N);
  if (mask) {
    m.mask.resize(B);
    for (int i = 0; i < B; ++i) m.mask[i] = mask[i] != 0;
  }
  return m;
}

void flatten_plan(const RoutingPlan& plan, int B, int N, int stride, int32_t* sets,
                  int32_t* set_len, double* weights, int32_t* loads,
                  int32_t* active_union, int32_t* active_count, int64_t* total_load) {
  for (int i = 0; i < B; ++i) {
    const auto& s = plan.sets[i];
    set_len[i] = static_cast<int32_t>(s.size());
    for (int j = 0; j < stride; ++j) {
      sets[i * stride + j] = j < static_cast<int>(s.size()) ? s[j] : -1;
      if (weights) {
        const auto& w = plan.weights[i];
        weights[i * stride + j] = j < static_cast<int>(w.size()) ? w[j] : 0.0;
      }
    }
  }
  if (loads)
    for (int e = 0; e < N; ++e) loads[e] = plan.loads[e];
  if (active_union) {
    for (int e = 0; e < N; ++e)
      active_union[e] = e < static_cast<int>(plan.active_union.size()) ? plan.active_union[e] : -1;
  }
  if (active_count) *active_count = plan.active_count;
  if (total_load) *total_load = plan.total_load;
}

template <typename Scalar>
struct RefLayer {
  MoeLayerParams<Scalar> p;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_resolve(int mode, int k, int k0, double p, int k_max, int max_p, int cap, int n,
                int32_t* out7, double* out_p) {
  REF_GUARD({
    const auto r = make_cfg(mode, k, k0, p, k_max, max_p, cap).resolved(n);
    out7[0] = static_cast<int>(r.mode);
    out7[1] = r.k;
    out7[2] = r.k0;
    out7[3] = r.k_max;
    out7[4] = r.max_p;
    out7[5] = static_cast<int>(r.cap);
    out7[6] = 0;
    *out_p = r.p;
  })
}

int ref_sort_experts(const double* scores, int B, int N, int32_t* order) {
  REF_GUARD({
    ScoreMatrix m = make_scores(scores, nullptr, B, N);
    const auto s = sort_experts(m);
    for (int i = 0; i < B; ++i)
      for (int j = 0; j < N; ++j) order[i * N + j] = s.order(i, j);
  })
}

// route(): the reference production path (routing.cpp:305-326).
int ref_route(const double* scores, const uint8_t* mask, int B, int N, int mode, int k,
              int k0, double p, int k_max, int max_p, int cap, int stride, int32_t* sets,
              int32_t* set_len, double* weights, int32_t* loads, int32_t* active_union,
              int32_t* active_count, int64_t* total_load) {
  REF_GUARD({
    ScoreMatrix m = make_scores(scores, mask, B, N);
    const auto plan = route(m, make_cfg(mode, k, k0, p, k_max, max_p, cap));
    flatten_plan(plan, B, N, stride, sets, set_len, weights, loads, active_union,
                 active_count, total_load);
  })
}

// The reference's own naive oracle (tests/oracle/oracle.cpp:212-215).
int ref_reference_route(const double* scores, const uint8_t* mask, int B, int N, int mode,
                        int k, int k0, double p, int k_max, int max_p, int cap, int stride,
                        int32_t* sets, int32_t* set_len, double* weights, int32_t* loads,
                        int32_t* active_union, int32_t* active_count,
                        int64_t* total_load) {
  REF_GUARD({
    ScoreMatrix m = make_scores(scores, mask, B, N);
    const auto plan = oracle::reference_route(m, make_cfg(mode, k, k0, p, k_max, max_p, cap));
    flatten_plan(plan, B, N, stride, sets, set_len, weights, loads, active_union,
                 active_count, total_load);
  })
}

int ref_phase1(const double* scores, const uint8_t* mask, int B, int N, int mode, int k,
               int k0, double p, int k_max, int max_p, int cap, int32_t* t, int32_t* n,
               int32_t* base_union, int32_t* base_union_count) {
  REF_GUARD({
    ScoreMatrix m = make_scores(scores, mask, B, N);
    const auto cfg = make_cfg(mode, k, k0, p, k_max, max_p, cap);
    const auto ph = phase1_baseline(m, sort_experts(m), cfg);
    for (int i = 0; i < B; ++i) {
      t[i] = ph.t[i];
      n[i] = ph.n[i];
    }
    for (int e = 0; e < N; ++e)
      base_union[e] = e < static_cast<int>(ph.base_union.size()) ? ph.base_union[e] : -1;
    *base_union_count = static_cast<int32_t>(ph.base_union.size());
  })
}

int ref_check_invariants(const double* scores, const uint8_t* mask, int B, int N, int mode,
                         int k, int k0, double p, int k_max, int max_p, int cap, int stride,
                         const int32_t* sets, const int32_t* set_len, const double* weights,
                         const int32_t* loads, const int32_t* active_union, int active_count,
                         int64_t total_load, char* msg, int msglen) {
  REF_GUARD({
    ScoreMatrix m = make_scores(scores, mask, B, N);
    RoutingPlan plan;
    plan.n_experts = N;
    plan.sets.resize(B);
    plan.weights.resize(B);
    for (int i = 0; i < B; ++i)
      for (int j = 0; j < set_len[i]; ++j) {
        plan.sets[i].push_back(sets[i * stride + j]);
        plan.weights[i].push_back(weights[i * stride + j]);
      }
    plan.loads = Eigen::VectorXi::Zero(N);
    for (int e = 0; e < N; ++e) plan.loads[e] = loads[e];
    for (int e = 0; e < active_count; ++e) plan.active_union.push_back(active_union[e]);
    plan.active_count = active_count;
    plan.total_load = total_load;
    const std::string r =
        oracle::check_plan_invariants(m, make_cfg(mode, k, k0, p, k_max, max_p, cap), plan);
    std::strncpy(msg, r.c_str(), msglen - 1);
    msg[msglen - 1] = '\0';
  })
}

int ref_exhaustive_small_check(int max_n, int max_b, int denom, int64_t* checks,
                               int64_t* mismatches, int64_t* violations) {
  REF_GUARD({
    const auto rep = oracle::exhaustive_small_check(max_n, max_b, denom);
    *checks = rep.checks;
    *mismatches = rep.mismatches;
    *violations = rep.violations;
  })
}

double ref_expected_active_experts(int N, int k, int B) {
  return expected_active_experts(N, k, B);
}

// fit_linear (latency.cpp:39-85) on n (T, us) observations; out = b, intercept,
// r2, residual_std, slope_stderr, intercept_stderr.
int ref_fit_linear(const int32_t* T, const double* us, int n, double* out) {
  REF_GUARD({
    std::vector<LatencyObservation> obs(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      obs[i].active_experts = T[i];
      obs[i].latency_us = us[i];
    }
    const FitResult f = fit_linear(obs);
    out[0] = f.params.b_us;
    out[1] = f.intercept_us;
    out[2] = f.r_squared;
    out[3] = f.residual_std;
    out[4] = f.slope_stderr;
    out[5] = f.intercept_stderr;
  })
}

// make_random_layer / make_random_batch (moe_layer.cpp:76-116) into flat arrays.
int ref_make_random_layer(int D, int H, int N, uint64_t seed, double* router, double* wg,
                          double* wu, double* wd) {
  REF_GUARD({
    const auto layer = make_random_layer({D, H, N}, seed);
    std::memcpy(router, layer.router.data(), sizeof(double) * D * N);
    for (int e = 0; e < N; ++e) {
      std::memcpy(wg + static_cast<size_t>(e) * D * H, layer.experts[e].w_gate.data(),
                  sizeof(double) * D * H);
      std::memcpy(wu + static_cast<size_t>(e) * D * H, layer.experts[e].w_up.data(),
                  sizeof(double) * D * H);
      std::memcpy(wd + static_cast<size_t>(e) * H * D, layer.experts[e].w_down.data(),
                  sizeof(double) * H * D);
    }
  })
}

int ref_make_random_batch(int B, int D, uint64_t seed, int step, int layer, double* x) {
  REF_GUARD({
    const auto b = make_random_batch(B, D, seed, step, layer);
    std::memcpy(x, b.embeddings.data(), sizeof(double) * B * D);
  })
}

// A reference MoE layer held across calls (bench reference arm). Values are
// copied from flat arrays in reference layout.
void* ref_layer_create(int scalar_is_float, int D, int H, int N, const double* router,
                       const double* wg, const double* wu, const double* wd) {
  try {
    if (scalar_is_float) {
      auto* L = new RefLayer<float>;
      L->p.router.resize(D, N);
      for (int i = 0; i < D * N; ++i) L->p.router.data()[i] = static_cast<float>(router[i]);
      L->p.experts.resize(N);
      for (int e = 0; e < N; ++e) {
        auto& ex = L->p.experts[e];
        ex.w_gate.resize(D, H);
        ex.w_up.resize(D, H);
        ex.w_down.resize(H, D);
        for (size_t i = 0; i < static_cast<size_t>(D) * H; ++i) {
          ex.w_gate.data()[i] = static_cast<float>(wg[static_cast<size_t>(e) * D * H + i]);
          ex.w_up.data()[i] = static_cast<float>(wu[static_cast<size_t>(e) * D * H + i]);
          ex.w_down.data()[i] = static_cast<float>(wd[static_cast<size_t>(e) * H * D + i]);
        }
      }
      return L;
    }
    auto* L = new RefLayer<double>;
    L->p.router.resize(D, N);
    std::memcpy(L->p.router.data(), router, sizeof(double) * D * N);
    L->p.experts.resize(N);
    for (int e = 0; e < N; ++e) {
      auto& ex = L->p.experts[e];
      ex.w_gate.resize(D, H);
      ex.w_up.resize(D, H);
      ex.w_down.resize(H, D);
      std::memcpy(ex.w_gate.data(), wg + static_cast<size_t>(e) * D * H, sizeof(double) * D * H);
      std::memcpy(ex.w_up.data(), wu + static_cast<size_t>(e) * D * H, sizeof(double) * D * H);
      std::memcpy(ex.w_down.data(), wd + static_cast<size_t>(e) * H * D, sizeof(double) * H * D);
    }
    return L;
  } catch (const std::exception& e) {
    record(3, e.what());
    return nullptr;
  }
}

// A reference MoeLayerParams<Scalar> holding exactly make_random_layer(dims,
// seed)'s values (moe_layer.cpp:76-98), filled by `threads` threads from the
// counter stream instead of one sequential pass (bench CPU baseline setup).
void* ref_layer_random(int scalar_is_float, int D, int H, int N, uint64_t seed, int threads) {
  try {
    const uint64_t parts[2] = {seed, 101};
    const uint64_t key = oo_stream_key(parts, 2);
    const double ds = 1.0 / std::sqrt(static_cast<double>(D));
    const double hs = 1.0 / std::sqrt(static_cast<double>(H));
    auto fill = [&](auto& L) {
      L.router.resize(D, N);
      L.experts.resize(N);
      for (auto& ex : L.experts) {
        ex.w_gate.resize(D, H);
        ex.w_up.resize(D, H);
        ex.w_down.resize(H, D);
      }
      const int64_t nr = static_cast<int64_t>(D) * N, per = static_cast<int64_t>(D) * H;
      const int64_t total = nr + static_cast<int64_t>(N) * 3 * per;
      std::vector<std::thread> th;
      if (threads < 1) threads = 1;
      for (int t = 0; t < threads; ++t)
        th.emplace_back([&, t] {
          for (int64_t f = total * t / threads; f < total * (t + 1) / threads; ++f) {
            const double z = oo_stream_normal(key, static_cast<uint64_t>(f));
            if (f < nr) {
              L.router.data()[f] = static_cast<typename std::decay_t<decltype(L.router)>::Scalar>(ds * z);
              continue;
            }
            const int64_t g = f - nr, e = g / (3 * per), r = g % (3 * per);
            auto& ex = L.experts[e];
            if (r < per)
              ex.w_gate.data()[r] = ds * z;
            else if (r < 2 * per)
              ex.w_up.data()[r - per] = ds * z;
            else
              ex.w_down.data()[r - 2 * per] = hs * z;
          }
        });
      for (auto& x : th) x.join();
    };
    if (scalar_is_float) {
      auto* L = new RefLayer<float>;
      fill(L->p);
      return L;
    }
    auto* L = new RefLayer<double>;
    fill(L->p);
    return L;
  } catch (const std::exception& e) {
    record(3, e.what());
    return nullptr;
  }
}

void ref_layer_destroy(void* layer, int scalar_is_float) {
  if (scalar_is_float)
    delete static_cast<RefLayer<float>*>(layer);
  else
    delete static_cast<RefLayer<double>*>(layer);
}

int ref_router_scores(void* layer, int scalar_is_float, const double* x, int B, int D,
                      double* scores) {
  REF_GUARD({
    TokenBatch batch;
    batch.embeddings.resize(B, D);
    std::memcpy(batch.embeddings.data(), x, sizeof(double) * B * D);
    const ScoreMatrix s = scalar_is_float
                              ? router_scores(static_cast<RefLayer<float>*>(layer)->p, batch)
                              : router_scores(static_cast<RefLayer<double>*>(layer)->p, batch);
    std::memcpy(scores, s.scores.data(), sizeof(double) * s.scores.size());
  })
}

// moe_forward (moe_layer.hpp:114-158) on a flat plan.
int ref_moe_forward(void* layer, int scalar_is_float, const double* x, int B, int D,
                    const int32_t* sets, const int32_t* set_len, const double* weights,
                    int stride, int n_experts, const uint8_t* mask, double* out) {
  REF_GUARD({
    TokenBatch batch;
    batch.embeddings.resize(B, D);
    std::memcpy(batch.embeddings.data(), x, sizeof(double) * B * D);
    RoutingPlan plan;
    plan.n_experts = n_experts;
    plan.sets.resize(B);
    plan.weights.resize(B);
    for (int i = 0; i < B; ++i)
      for (int j = 0; j < set_len[i]; ++j) {
        plan.sets[i].push_back(sets[i * stride + j]);
        plan.weights[i].push_back(weights[i * stride + j]);
      }
    MaskArray m;
    if (mask) {
      m.resize(B);
      for (int i = 0; i < B; ++i) m[i] = mask[i] != 0;
    }
    const RowMatrixXd r =
        scalar_is_float
            ? moe_forward(static_cast<RefLayer<float>*>(layer)->p, batch, plan, mask ? &m : nullptr)
            : moe_forward(static_cast<RefLayer<double>*>(layer)->p, batch, plan, mask ? &m : nullptr);
    std::memcpy(out, r.data(), sizeof(double) * B * D);
  })
}

// The reference's full CPU decode cell for one batch: router_scores -> route
// -> moe_forward (the toy-layer cell of simulate.cpp:181-189, minus the
// shadow vanilla run). Returns T via *active_count.
int ref_decode(void* layer, int scalar_is_float, const double* x, int B, int D, int mode,
               int k, int k0, double p, int k_max, int max_p, int cap, double* out,
               int32_t* active_count, int64_t* total_load) {
  REF_GUARD({
    TokenBatch batch;
    batch.embeddings.resize(B, D);
    std::memcpy(batch.embeddings.data(), x, sizeof(double) * B * D);
    const auto cfg = make_cfg(mode, k, k0, p, k_max, max_p, cap);
    RowMatrixXd r;
    RoutingPlan plan;
    if (scalar_is_float) {
      const auto& L = static_cast<RefLayer<float>*>(layer)->p;
      plan = route(router_scores(L, batch), cfg);
      r = moe_forward(L, batch, plan);
    } else {
      const auto& L = static_cast<RefLayer<double>*>(layer)->p;
      plan = route(router_scores(L, batch), cfg);
      r = moe_forward(L, batch, plan);
    }
    std::memcpy(out, r.data(), sizeof(double) * B * D);
    *active_count = plan.active_count;
    *total_load = plan.total_load;
  })
}

// gen_scores (score_gen.cpp:100-160) for one (step, layer): kind 0 =
// Dirichlet(alpha), 1 = clustered. out [batch][n_experts].
int ref_gen_scores(int kind, int n_experts, int batch, int steps, int layers, uint64_t seed,
                   double alpha, int groups, double conc, double spread, int step, int layer,
                   double* out) {
  REF_GUARD({
    ScoreGenConfig cfg;
    cfg.kind = kind == 0 ? GenKind::Dirichlet : GenKind::Clustered;
    cfg.n_experts = n_experts;
    cfg.batch = batch;
    cfg.steps = steps;
    cfg.layers = layers;
    cfg.seed = seed;
    cfg.alpha = alpha;
    cfg.groups = groups;
    cfg.within_group_concentration = conc;
    cfg.between_group_spread = spread;
    const ScoreMatrix m = gen_scores(cfg, step, layer);
    std::memcpy(out, m.scores.data(), sizeof(double) * batch * n_experts);
  })
}

static ScoreGenConfig gen_cfg(const int32_t* gi, uint64_t seed, const double* gd) {
  // gi: kind, n_experts, batch, steps, layers, groups; gd: alpha, conc, spread
  ScoreGenConfig cfg;
  cfg.kind = gi[0] == 0 ? GenKind::Dirichlet : GenKind::Clustered;
  cfg.n_experts = gi[1];
  cfg.batch = gi[2];
  cfg.steps = gi[3];
  cfg.layers = gi[4];
  cfg.groups = gi[5];
  cfg.seed = seed;
  cfg.alpha = gd[0];
  cfg.within_group_concentration = gd[1];
  cfg.between_group_spread = gd[2];
  return cfg;
}

static void put_records(const std::vector<StepRecord>& v, int32_t* T, int64_t* load, double* lat) {
  for (size_t i = 0; i < v.size(); ++i) {
    T[i] = v[i].active_experts;
    load[i] = v[i].total_load;
    lat[i] = v[i].modeled_latency_us;
  }
}

// simulate_decode (simulate.cpp:128-151): per (step, layer) records of the
// routed and the vanilla shadow run, plus the 8 aggregates
// (compute_aggregates :69-103, in TraceAggregates field order).
int ref_simulate_decode(const int32_t* gi, uint64_t seed, const double* gd, int mode, int k,
                        int k0, double p, int k_max, int max_p, int cap, double a_us,
                        double b_us, int32_t* T, int64_t* load, double* lat, int32_t* vT,
                        int64_t* vload, double* vlat, double* agg) {
  REF_GUARD({
    const auto tr = simulate_decode(gen_cfg(gi, seed, gd), make_cfg(mode, k, k0, p, k_max, max_p, cap),
                                    LatencyParams{a_us, b_us}, 1);
    put_records(tr.records, T, load, lat);
    put_records(tr.vanilla_records, vT, vload, vlat);
    const auto& a = tr.aggregates;
    agg[0] = a.mean_active_experts;
    agg[1] = a.mean_total_load;
    agg[2] = a.mean_latency_us;
    agg[3] = a.vanilla_mean_active_experts;
    agg[4] = a.vanilla_mean_total_load;
    agg[5] = a.vanilla_mean_latency_us;
    agg[6] = a.normalized_active_experts;
    agg[7] = a.normalized_latency;
  })
}

// padding_experiment (simulate.cpp:185-257): records of the three variants
// (no / naive / masked padding) and masked_matches_no_padding.
int ref_padding_experiment(const int32_t* gi, uint64_t seed, const double* gd, int mode, int k,
                           int k0, double p, int k_max, int max_p, int cap, int pad_to,
                           double a_us, double b_us, int32_t* T3, int64_t* load3, double* lat3,
                           int32_t* matches) {
  REF_GUARD({
    const auto rep = padding_experiment(gen_cfg(gi, seed, gd),
                                        make_cfg(mode, k, k0, p, k_max, max_p, cap), pad_to,
                                        LatencyParams{a_us, b_us}, 1);
    const size_t n = rep.no_padding.records.size();
    put_records(rep.no_padding.records, T3, load3, lat3);
    put_records(rep.naive_padding.records, T3 + n, load3 + n, lat3 + n);
    put_records(rep.masked_padding.records, T3 + 2 * n, load3 + 2 * n, lat3 + 2 * n);
    *matches = rep.masked_matches_no_padding ? 1 : 0;
  })
}

// sweep (sweep.cpp:77-106) over default_sweep_grid(N, k) (:48-75): the mean
// T of every grid point, in grid order (n_out = grid size; buffer >= 4096).
int ref_sweep_default(const int32_t* gi, uint64_t seed, const double* gd, int k, double a_us,
                      double b_us, int rounding, double* mean_t, int32_t* n_out) {
  REF_GUARD({
    const ScoreGenConfig gen = gen_cfg(gi, seed, gd);
    const auto grid = default_sweep_grid(gen.n_experts, k);
    RoundingRule rr;
    rr.enabled = rounding != 0;
    const auto pts = sweep(gen, grid, LatencyParams{a_us, b_us}, nullptr, rr, 1);
    for (size_t i = 0; i < pts.size(); ++i) mean_t[i] = pts[i].mean_active_experts;
    *n_out = static_cast<int32_t>(pts.size());
  })
}

// pareto_indices (sweep.cpp:108-122) of points (T, quality or NaN = none).
int ref_pareto_indices(const double* t, const double* q, int n, int32_t* out, int32_t* count) {
  REF_GUARD({
    std::vector<SweepPoint> pts(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      pts[i].mean_active_experts = t[i];
      if (!std::isnan(q[i])) pts[i].quality_delta = q[i];
    }
    const auto idx = pareto_indices(pts);
    for (size_t i = 0; i < idx.size(); ++i) out[i] = static_cast<int32_t>(idx[i]);
    *count = static_cast<int32_t>(idx.size());
  })
}

// simulate_decode(layer, gen, ...) (simulate.cpp:153-183) on
// make_random_layer({D, H, N}, layer_seed): T / load / latency and the
// divergence per record, plus the vanilla records' T.
int ref_simulate_decode_layer(int D, int H, int N, uint64_t layer_seed, const int32_t* gi,
                              uint64_t seed, const double* gd, int mode, int k, int k0, double p,
                              int k_max, int max_p, int cap, double a_us, double b_us,
                              int32_t* T, int64_t* load, double* lat, double* div, int32_t* vT,
                              double* mean_div) {
  REF_GUARD({
    LayerDims dims;
    dims.embed = D;
    dims.hidden = H;
    dims.experts = N;
    const auto layer = make_random_layer(dims, layer_seed);
    const auto tr = simulate_decode(layer, gen_cfg(gi, seed, gd),
                                    make_cfg(mode, k, k0, p, k_max, max_p, cap),
                                    LatencyParams{a_us, b_us}, 1);
    for (size_t i = 0; i < tr.records.size(); ++i) {
      T[i] = tr.records[i].active_experts;
      load[i] = tr.records[i].total_load;
      lat[i] = tr.records[i].modeled_latency_us;
      div[i] = tr.records[i].divergence.value_or(-1.0);
      vT[i] = tr.vanilla_records[i].active_experts;
    }
    *mean_div = tr.aggregates.mean_divergence.value_or(-1.0);
  })
}

}  // extern "C"
