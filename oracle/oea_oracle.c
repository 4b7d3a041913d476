/*
 * oea_oracle.c — plain-C restatement of the reference's routing and MoE-layer
 * arithmetic. TEST INFRASTRUCTURE ONLY (see oea_oracle.h).
 *
 * Compiled with -ffp-contract=off so every fp64 add/mul/div rounds exactly as
 * written, like the reference's scalar loops on x86-64 SSE2.
 */
#include "oea_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define OO_PI 3.14159265358979323846

static int fail(char* err, int32_t errlen, int code, const char* msg) {
  if (err && errlen > 0) {
    strncpy(err, msg, (size_t)errlen - 1);
    err[errlen - 1] = '\0';
  }
  return code;
}

/* routing.cpp:153-182 */
int oo_resolve(const oo_cfg* in, int32_t n, oo_cfg* out, char* err, int32_t errlen) {
  if (n < 1) return fail(err, errlen, 1, "RoutingConfig: expert count must be >= 1");
  oo_cfg c = *in;
  if (c.mode == 3) { /* SimplifiedOea pins p, k_max, max_p (:158-162) */
    c.p = 1.0;
    c.k_max = c.k;
    c.max_p = n;
  }
  if (c.max_p == 0) c.max_p = n; /* :163 */
  if (c.k < 1 || c.k > n) return fail(err, errlen, 1, "RoutingConfig: k must be in [1, N]");
  if (c.mode != 0) {
    if (c.k0 < 1 || c.k0 > n)
      return fail(err, errlen, 1, "RoutingConfig: k0 must be in [1, N]");
    if (!(c.p > 0.0) || c.p > 1.0)
      return fail(err, errlen, 1, "RoutingConfig: p must be in (0, 1]");
    if (c.k_max < c.k0 || c.k_max > n)
      return fail(err, errlen, 1, "RoutingConfig: need k0 <= k_max <= N");
    if (c.max_p < 1 || c.max_p > n)
      return fail(err, errlen, 1, "RoutingConfig: max_p must be in [1, N]");
  }
  *out = c;
  return 0;
}

/* Comparator of routing.cpp:196-199: a ranks before b iff its score is
 * greater, ties (double ==, so -0.0 == +0.0) by smaller index. */
static int ranks_before(const double* row, int32_t a, int32_t b) {
  if (row[a] != row[b]) return row[a] > row[b];
  return a < b;
}

/* Bottom-up merge sort of expert indices (the order is total, so any correct
 * sort reproduces std::sort's output). */
static void sort_row(const double* row, int32_t n, int32_t* idx, int32_t* tmp) {
  for (int32_t i = 0; i < n; ++i) idx[i] = i;
  for (int32_t w = 1; w < n; w *= 2) {
    for (int32_t lo = 0; lo < n; lo += 2 * w) {
      int32_t mid = lo + w < n ? lo + w : n;
      int32_t hi = lo + 2 * w < n ? lo + 2 * w : n;
      int32_t a = lo, b = mid, o = lo;
      while (a < mid && b < hi) tmp[o++] = ranks_before(row, idx[b], idx[a]) ? idx[b++] : idx[a++];
      while (a < mid) tmp[o++] = idx[a++];
      while (b < hi) tmp[o++] = idx[b++];
    }
    memcpy(idx, tmp, sizeof(int32_t) * (size_t)n);
  }
}

/* routing.cpp:184-203 */
int oo_sort_experts(const double* scores, int32_t B, int32_t N, int32_t* order,
                    char* err, int32_t errlen) {
  if (B < 1 || N < 1) return fail(err, errlen, 1, "sort_experts: dimensions must be >= 1");
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
  for (int32_t i = 0; i < B; ++i) sort_row(scores + (size_t)i * N, N, order + (size_t)i * N, tmp);
  free(tmp);
  return 0;
}

int oo_route(const double* scores, const uint8_t* mask, int32_t B, int32_t N,
             const oo_cfg* raw, int32_t stride, int32_t* sets, int32_t* set_len,
             double* weights, int32_t* loads, int32_t* active_union,
             int32_t* active_count, int64_t* total_load, int32_t* order_out,
             int32_t* t_out, int32_t* n_out, int32_t* base_union,
             int32_t* base_union_count, char* err, int32_t errlen) {
  oo_cfg cfg;
  int st = oo_resolve(raw, N, &cfg, err, errlen); /* route :306-307 */
  if (st) return st;
  if (B < 1) return fail(err, errlen, 1, "sort_experts: dimensions must be >= 1");
  if (cfg.mode == 0 && (cfg.k < 1 || cfg.k > N))
    return fail(err, errlen, 1, "route_topk: k must be in [1, N]");

  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)B * N);
  st = oo_sort_experts(scores, B, N, order, err, errlen);
  if (st) {
    free(order);
    return st;
  }
  unsigned char* in_union = (unsigned char*)calloc((size_t)N, 1);
  int32_t* nb = (int32_t*)calloc((size_t)B, sizeof(int32_t));

  for (int32_t i = 0; i < B; ++i) {
    set_len[i] = 0;
    for (int32_t j = 0; j < stride; ++j) {
      sets[(size_t)i * stride + j] = -1;
      if (weights) weights[(size_t)i * stride + j] = 0.0;
    }
    if (t_out) t_out[i] = 0;
    if (n_out) n_out[i] = 0;
  }

  if (cfg.mode == 0) {
    /* route_topk, routing.cpp:205-224: first k ranks of real rows */
    for (int32_t i = 0; i < B; ++i) {
      if (mask && !mask[i]) continue;
      for (int32_t j = 0; j < cfg.k; ++j) sets[(size_t)i * stride + j] = order[(size_t)i * N + j];
      set_len[i] = cfg.k;
    }
  } else {
    /* phase1_baseline, routing.cpp:226-268 */
    for (int32_t i = 0; i < B; ++i) {
      if (mask && !mask[i]) continue;
      const double* row = scores + (size_t)i * N;
      const int32_t* ord = order + (size_t)i * N;
      int32_t t_i = N;
      if (cfg.p != 1.0) { /* p == 1 short-circuit :243-245 */
        double cum = 0.0;
        for (int32_t j = 0; j < N; ++j) { /* :247-255 */
          cum += row[ord[j]];
          if (cum >= cfg.p) {
            t_i = j + 1;
            break;
          }
        }
      }
      int32_t n_i = cfg.k0 < t_i ? cfg.k0 : t_i; /* :257 */
      if (t_out) t_out[i] = t_i;
      if (n_out) n_out[i] = n_i;
      nb[i] = n_i;
      for (int32_t j = 0; j < n_i; ++j) {
        sets[(size_t)i * stride + j] = ord[j];
        in_union[ord[j]] = 1; /* :262-266 */
      }
      set_len[i] = n_i;
    }
    if (cfg.mode == 2 || cfg.mode == 3) {
      /* phase2_piggyback, routing.cpp:270-303 */
      for (int32_t i = 0; i < B; ++i) {
        if (mask && !mask[i]) continue;
        const int32_t* ord = order + (size_t)i * N;
        int32_t len = set_len[i];
        for (int32_t j = nb[i]; j < cfg.max_p; ++j) {
          if (cfg.cap == 0) {
            if (len >= cfg.k_max) break; /* ExactCap :292-293 */
          } else {
            if (len > cfg.k_max) break; /* PseudocodeStrict :294-295 */
          }
          int32_t e = ord[j];
          if (in_union[e]) sets[(size_t)i * stride + len++] = e; /* :298 */
        }
        set_len[i] = len;
      }
    }
  }
  if (base_union) {
    int32_t c = 0;
    for (int32_t e = 0; e < N; ++e)
      if (in_union[e]) base_union[c++] = e;
    if (base_union_count) *base_union_count = c;
  } else if (base_union_count) {
    int32_t c = 0;
    for (int32_t e = 0; e < N; ++e) c += in_union[e];
    *base_union_count = c;
  }

  /* fill_aggregates, routing.cpp:17-31 */
  int32_t* ld = (int32_t*)calloc((size_t)N, sizeof(int32_t));
  int64_t total = 0;
  for (int32_t i = 0; i < B; ++i) {
    for (int32_t j = 0; j < set_len[i]; ++j) ld[sets[(size_t)i * stride + j]]++;
    total += set_len[i];
  }
  int32_t tcount = 0;
  for (int32_t e = 0; e < N; ++e) {
    if (loads) loads[e] = ld[e];
    if (ld[e] > 0) {
      if (active_union) active_union[tcount] = e;
      ++tcount;
    }
  }
  if (active_union)
    for (int32_t e = tcount; e < N; ++e) active_union[e] = -1;
  if (active_count) *active_count = tcount;
  if (total_load) *total_load = total;

  /* renormalize_weights, routing.cpp:33-49: sequential mass in set order */
  st = 0;
  for (int32_t i = 0; i < B && st == 0; ++i) {
    if (set_len[i] == 0) continue;
    const double* row = scores + (size_t)i * N;
    double mass = 0.0;
    for (int32_t j = 0; j < set_len[i]; ++j) mass += row[sets[(size_t)i * stride + j]];
    if (!(mass > 1e-12)) {
      char msg[160];
      snprintf(msg, sizeof msg,
               "route: degenerate selected-set mass for token %d (sum <= 1e-12)", i);
      st = fail(err, errlen, 2, msg);
      break;
    }
    if (weights)
      for (int32_t j = 0; j < set_len[i]; ++j)
        weights[(size_t)i * stride + j] = row[sets[(size_t)i * stride + j]] / mass;
  }
  if (order_out) memcpy(order_out, order, sizeof(int32_t) * (size_t)B * N);
  free(ld);
  free(nb);
  free(in_union);
  free(order);
  return st;
}

/* moe_layer.hpp:84-88: e = exp(l - max), s = e / sum(e) (sum left to right) */
void oo_softmax_rows(const double* logits, int32_t B, int32_t N, double* scores) {
  double* e = (double*)malloc(sizeof(double) * (size_t)N);
  for (int32_t i = 0; i < B; ++i) {
    const double* l = logits + (size_t)i * N;
    double m = l[0];
    for (int32_t j = 1; j < N; ++j) m = l[j] > m ? l[j] : m;
    double sum = 0.0;
    for (int32_t j = 0; j < N; ++j) {
      e[j] = exp(l[j] - m);
      sum += e[j];
    }
    for (int32_t j = 0; j < N; ++j) scores[(size_t)i * N + j] = e[j] / sum;
  }
  free(e);
}

/* moe_layer.hpp:71-90 */
void oo_router_scores(const double* x, const double* router, int32_t B, int32_t D,
                      int32_t N, double* scores) {
  double* logits = (double*)calloc((size_t)B * N, sizeof(double));
  for (int32_t i = 0; i < B; ++i)
    for (int32_t d = 0; d < D; ++d) {
      const double xv = x[(size_t)i * D + d];
      for (int32_t n = 0; n < N; ++n) logits[(size_t)i * N + n] += xv * router[(size_t)d * N + n];
    }
  oo_softmax_rows(logits, B, N, scores);
  free(logits);
}

/* moe_forward validation, moe_layer.hpp:119-152 */
static int check_plan(int32_t B, int32_t N, const int32_t* sets, const int32_t* set_len,
                      int32_t stride, const uint8_t* mask, char* err, int32_t errlen) {
  for (int32_t i = 0; i < B; ++i) {
    const int real = mask == NULL || mask[i];
    if (set_len[i] == 0) {
      if (real && mask != NULL) {
        char msg[128];
        snprintf(msg, sizeof msg, "moe_forward: empty selected set for unmasked token %d", i);
        return fail(err, errlen, 1, msg);
      }
      continue;
    }
    for (int32_t j = 0; j < set_len[i]; ++j) {
      int32_t e = sets[(size_t)i * stride + j];
      if (e < 0 || e >= N) return fail(err, errlen, 1, "moe_forward: expert index out of range");
    }
  }
  return 0;
}

static double silu_d(double z) { return z / (1.0 + exp(-z)); }
static float silu_f(float z) { return z / (1.0f + expf(-z)); }

int oo_moe_forward_f64(const double* wg, const double* wu, const double* wd,
                       int32_t D, int32_t H, int32_t N, const double* x, int32_t B,
                       const int32_t* sets, const int32_t* set_len,
                       const double* weights, int32_t stride, const uint8_t* mask,
                       double* out, char* err, int32_t errlen) {
  int st = check_plan(B, N, sets, set_len, stride, mask, err, errlen);
  if (st) return st;
  double* g = (double*)malloc(sizeof(double) * (size_t)H);
  double* u = (double*)malloc(sizeof(double) * (size_t)H);
  double* y = (double*)malloc(sizeof(double) * (size_t)D);
  memset(out, 0, sizeof(double) * (size_t)B * D);
  for (int32_t i = 0; i < B; ++i) {
    const double* xi = x + (size_t)i * D;
    for (int32_t j = 0; j < set_len[i]; ++j) {
      const int32_t e = sets[(size_t)i * stride + j];
      const double* Wg = wg + (size_t)e * D * H;
      const double* Wu = wu + (size_t)e * D * H;
      const double* Wd = wd + (size_t)e * H * D;
      /* expert_forward, moe_layer.hpp:100-106 */
      for (int32_t h = 0; h < H; ++h) g[h] = u[h] = 0.0;
      for (int32_t d = 0; d < D; ++d)
        for (int32_t h = 0; h < H; ++h) {
          g[h] += xi[d] * Wg[(size_t)d * H + h];
          u[h] += xi[d] * Wu[(size_t)d * H + h];
        }
      for (int32_t h = 0; h < H; ++h) g[h] = silu_d(g[h]) * u[h];
      for (int32_t d = 0; d < D; ++d) y[d] = 0.0;
      for (int32_t h = 0; h < H; ++h)
        for (int32_t d = 0; d < D; ++d) y[d] += g[h] * Wd[(size_t)h * D + d];
      /* out.row(i) += w[j] * y, in set order (:148-155) */
      const double w = weights[(size_t)i * stride + j];
      for (int32_t d = 0; d < D; ++d) out[(size_t)i * D + d] += w * y[d];
    }
  }
  free(g);
  free(u);
  free(y);
  return 0;
}

int oo_moe_forward_f32(const float* wg, const float* wu, const float* wd, int32_t D,
                       int32_t H, int32_t N, const double* x, int32_t B,
                       const int32_t* sets, const int32_t* set_len,
                       const double* weights, int32_t stride, const uint8_t* mask,
                       double* out, char* err, int32_t errlen) {
  int st = check_plan(B, N, sets, set_len, stride, mask, err, errlen);
  if (st) return st;
  float* xs = (float*)malloc(sizeof(float) * (size_t)D);
  float* g = (float*)malloc(sizeof(float) * (size_t)H);
  float* u = (float*)malloc(sizeof(float) * (size_t)H);
  float* y = (float*)malloc(sizeof(float) * (size_t)D);
  memset(out, 0, sizeof(double) * (size_t)B * D);
  for (int32_t i = 0; i < B; ++i) {
    for (int32_t d = 0; d < D; ++d) xs[d] = (float)x[(size_t)i * D + d];
    for (int32_t j = 0; j < set_len[i]; ++j) {
      const int32_t e = sets[(size_t)i * stride + j];
      const float* Wg = wg + (size_t)e * D * H;
      const float* Wu = wu + (size_t)e * D * H;
      const float* Wd = wd + (size_t)e * H * D;
      for (int32_t h = 0; h < H; ++h) g[h] = u[h] = 0.0f;
      for (int32_t d = 0; d < D; ++d)
        for (int32_t h = 0; h < H; ++h) {
          g[h] += xs[d] * Wg[(size_t)d * H + h];
          u[h] += xs[d] * Wu[(size_t)d * H + h];
        }
      for (int32_t h = 0; h < H; ++h) g[h] = silu_f(g[h]) * u[h];
      for (int32_t d = 0; d < D; ++d) y[d] = 0.0f;
      for (int32_t h = 0; h < H; ++h)
        for (int32_t d = 0; d < D; ++d) y[d] += g[h] * Wd[(size_t)h * D + d];
      const double w = weights[(size_t)i * stride + j];
      for (int32_t d = 0; d < D; ++d) out[(size_t)i * D + d] += w * (double)y[d];
    }
  }
  free(xs);
  free(g);
  free(u);
  free(y);
  return 0;
}

/* ---- counter RNG, rng.hpp:24-117 ---------------------------------------- */
#define OO_GOLDEN 0x9E3779B97F4A7C15ULL

uint64_t oo_splitmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

uint64_t oo_stream_key(const uint64_t* parts, int32_t n) {
  uint64_t h = 0x853C49E6748FEA9BULL;
  for (int32_t i = 0; i < n; ++i) h = oo_splitmix64(h + OO_GOLDEN + parts[i]);
  return h;
}

/* draw c (1-based) -> unit in (0, 1] (rng.hpp:54-62) */
static double unit_at(uint64_t key, uint64_t c) {
  uint64_t u = oo_splitmix64(key + c * OO_GOLDEN);
  return (double)((u >> 11) + 1) * 0x1.0p-53;
}

/* Normal #f uses draws 2*(f/2)+1 and +2; even f is the cosine branch, odd f
 * the cached sine (rng.hpp:65-77). */
double oo_stream_normal(uint64_t key, uint64_t f) {
  const uint64_t pair = f / 2;
  const double u1 = unit_at(key, 2 * pair + 1);
  const double u2 = unit_at(key, 2 * pair + 2);
  const double r = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * OO_PI * u2;
  return (f & 1) ? r * sin(theta) : r * cos(theta);
}

typedef struct {
  uint64_t key;
  int64_t begin, end; /* normal indices */
  int32_t D, H, N;
  double dscale, hscale;
  double *router, *wg, *wu, *wd;
} fill_job;

/* Stream order: router (D x N), then per expert gate (D x H), up (D x H),
 * down (H x D) (moe_layer.cpp:85-96). */
static void* fill_range(void* arg) {
  fill_job* j = (fill_job*)arg;
  const int64_t nr = (int64_t)j->D * j->N;
  const int64_t per = (int64_t)j->D * j->H;
  const int64_t pe = 3 * per;
  for (int64_t f = j->begin; f < j->end; ++f) {
    const double z = oo_stream_normal(j->key, (uint64_t)f);
    if (f < nr) {
      j->router[f] = j->dscale * z;
      continue;
    }
    const int64_t g = f - nr;
    const int64_t e = g / pe, r = g % pe;
    if (r < per)
      j->wg[e * per + r] = j->dscale * z;
    else if (r < 2 * per)
      j->wu[e * per + (r - per)] = j->dscale * z;
    else
      j->wd[e * per + (r - 2 * per)] = j->hscale * z;
  }
  return NULL;
}

void oo_make_random_layer(int32_t D, int32_t H, int32_t N, uint64_t seed,
                          double* router, double* wg, double* wu, double* wd,
                          int32_t n_threads) {
  const uint64_t parts[2] = {seed, 101};
  fill_job base;
  base.key = oo_stream_key(parts, 2);
  base.D = D;
  base.H = H;
  base.N = N;
  base.dscale = 1.0 / sqrt((double)D);
  base.hscale = 1.0 / sqrt((double)H);
  base.router = router;
  base.wg = wg;
  base.wu = wu;
  base.wd = wd;
  const int64_t total = (int64_t)D * N + (int64_t)N * 3 * D * H;
  if (n_threads < 1) n_threads = 1;
  if (n_threads > 64) n_threads = 64;
  pthread_t th[64];
  fill_job jobs[64];
  for (int32_t t = 0; t < n_threads; ++t) {
    jobs[t] = base;
    jobs[t].begin = total * t / n_threads;
    jobs[t].end = total * (t + 1) / n_threads;
    if (n_threads == 1)
      fill_range(&jobs[t]);
    else
      pthread_create(&th[t], NULL, fill_range, &jobs[t]);
  }
  if (n_threads > 1)
    for (int32_t t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
}

void oo_make_random_batch(int32_t B, int32_t D, uint64_t seed, int32_t step,
                          int32_t layer, double* x) {
  for (int32_t i = 0; i < B; ++i) {
    const uint64_t parts[5] = {seed, (uint64_t)step, (uint64_t)layer, (uint64_t)i, 102};
    const uint64_t key = oo_stream_key(parts, 5);
    for (int32_t c = 0; c < D; ++c) x[(size_t)i * D + c] = oo_stream_normal(key, (uint64_t)c);
  }
}

/* moe_layer.cpp:57-74 */
int oo_output_divergence(const double* ref, const double* test, int32_t B,
                         int32_t D, double* mean_rel, double* max_rel) {
  if (B == 0) return 1;
  double sum = 0.0, mx = 0.0;
  for (int32_t i = 0; i < B; ++i) {
    double nr = 0.0, nd = 0.0;
    for (int32_t d = 0; d < D; ++d) {
      const double a = ref[(size_t)i * D + d], b = test[(size_t)i * D + d];
      nr += a * a;
      nd += (a - b) * (a - b);
    }
    double denom = sqrt(nr);
    if (denom < 1e-12) denom = 1e-12;
    const double rel = sqrt(nd) / denom;
    sum += rel;
    if (rel > mx) mx = rel;
  }
  *mean_rel = sum / (double)B;
  *max_rel = mx;
  return 0;
}

/* latency.cpp:30-37 */
double oo_expected_active_experts(int32_t N, int32_t k, int32_t B) {
  const double miss = 1.0 - (double)k / N;
  return N * (1.0 - pow(miss, B));
}

/* ---- score generators, score_gen.cpp:100-160 + rng.hpp:46-102 ----------- */
/* Sequential CounterRng (rng.hpp:46-117): counter, cached Box-Muller spare. */
typedef struct {
  uint64_t key, counter;
  double spare;
  int has_spare;
} oo_rng;

static double rng_unit(oo_rng* r) { /* rng.hpp:54-62 */
  r->counter += 1;
  const uint64_t u = oo_splitmix64(r->key + r->counter * OO_GOLDEN);
  return (double)((u >> 11) + 1) * 0x1.0p-53;
}

static double rng_normal(oo_rng* r) { /* rng.hpp:65-77 */
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  const double u1 = rng_unit(r);
  const double u2 = rng_unit(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * OO_PI * u2;
  r->spare = rad * sin(theta);
  r->has_spare = 1;
  return rad * cos(theta);
}

static double rng_gamma(oo_rng* r, double alpha) { /* rng.hpp:82-98, Marsaglia-Tsang */
  if (alpha < 1.0) {
    const double u = rng_unit(r);
    return rng_gamma(r, alpha + 1.0) * pow(u, 1.0 / alpha);
  }
  const double d = alpha - 1.0 / 3.0;
  const double c = 1.0 / sqrt(9.0 * d);
  for (;;) {
    const double x = rng_normal(r);
    double v = 1.0 + c * x;
    if (v <= 0.0) continue;
    v = v * v * v;
    const double u = rng_unit(r);
    const double x2 = x * x;
    if (u < 1.0 - 0.0331 * x2 * x2) return d * v;
    if (log(u) < 0.5 * x2 + d * (1.0 - v + log(v))) return d * v;
  }
}

static oo_rng rng_for(uint64_t seed, int32_t step, int32_t layer, int32_t token, uint64_t tag) {
  const uint64_t parts[5] = {seed, (uint64_t)step, (uint64_t)layer, (uint64_t)token, tag};
  oo_rng r = {oo_stream_key(parts, 5), 0, 0.0, 0};
  return r;
}

/* Dirichlet(alpha) rows for (step, layer): per token i its own stream
 * (seed, step, layer, i, 201), N gammas, divided by their sequential sum
 * (score_gen.cpp:119-133). out [B][N]. */
void oo_gen_dirichlet(int32_t N, int32_t B, uint64_t seed, double alpha, int32_t step,
                      int32_t layer, double* out) {
  for (int32_t i = 0; i < B; ++i) {
    oo_rng r = rng_for(seed, step, layer, i, 201);
    double sum = 0.0;
    double* row = out + (size_t)i * N;
    for (int32_t e = 0; e < N; ++e) {
      row[e] = rng_gamma(&r, alpha);
      sum += row[e];
    }
    for (int32_t e = 0; e < N; ++e) row[e] /= sum;
  }
}

/* Clustered rows (score_gen.cpp:136-160): group templates from streams
 * (seed, step, layer, g, 202), token i in group i % groups, logits
 * spread * (template + noise / concentration) with noise from
 * (seed, step, layer, i, 203), then softmax (max-subtracted, sequential sum). */
void oo_gen_clustered(int32_t N, int32_t B, uint64_t seed, int32_t groups, double conc,
                      double spread, int32_t step, int32_t layer, double* out) {
  double* tpl = (double*)malloc(sizeof(double) * (size_t)groups * N);
  for (int32_t g = 0; g < groups; ++g) {
    oo_rng r = rng_for(seed, step, layer, g, 202);
    for (int32_t e = 0; e < N; ++e) tpl[(size_t)g * N + e] = rng_normal(&r);
  }
  for (int32_t i = 0; i < B; ++i) {
    oo_rng r = rng_for(seed, step, layer, i, 203);
    const int32_t g = i % groups;
    double* row = out + (size_t)i * N;
    for (int32_t e = 0; e < N; ++e) row[e] = spread * (tpl[(size_t)g * N + e] + rng_normal(&r) / conc);
    double m = row[0];
    for (int32_t e = 1; e < N; ++e) m = row[e] > m ? row[e] : m;
    double sum = 0.0;
    for (int32_t e = 0; e < N; ++e) {
      row[e] = exp(row[e] - m);
      sum += row[e];
    }
    for (int32_t e = 0; e < N; ++e) row[e] /= sum;
  }
  free(tpl);
}
