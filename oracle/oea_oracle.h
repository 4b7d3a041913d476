/*
 * oea_oracle.h — CPU restatement of the reference's hot path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_2511_02237_b200/,
 * include/) links or calls this; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg use it, and only as the checker / CPU baseline.
 *
 * Every function restates one reference function (file:line under
 * /root/reference/proj). Pinned by tests/test_oracle.py against (a) the
 * reference's known-answer tests (test_routing.cpp, test_moe_layer.cpp),
 * (b) golden vectors produced by the reference itself compiled here
 * (oracle/_ref, tests/golden/make_golden.py) and (c) live comparison with
 * oracle/_ref when it is present.
 */
#ifndef OEA_ORACLE_H_
#define OEA_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t mode; /* 0 vanilla, 1 pruned, 2 oea, 3 simplified */
  int32_t k;
  int32_t k0;
  double p;
  int32_t k_max;
  int32_t max_p;
  int32_t cap; /* 0 exact, 1 pseudocode */
} oo_cfg;

/* status codes: 0 ok, 1 invalid_argument, 2 domain_error */

/* RoutingConfig::resolved, routing.cpp:153-182 */
int oo_resolve(const oo_cfg* in, int32_t n, oo_cfg* out, char* err, int32_t errlen);

/* sort_experts, routing.cpp:184-203 (all rows, including masked ones) */
int oo_sort_experts(const double* scores, int32_t B, int32_t N, int32_t* order,
                    char* err, int32_t errlen);

/* route, routing.cpp:305-326, with its phases. Optional outputs may be NULL.
 * sets/weights: [B * stride], -1 / 0 padded. */
int oo_route(const double* scores, const uint8_t* mask, int32_t B, int32_t N,
             const oo_cfg* cfg, int32_t stride, int32_t* sets, int32_t* set_len,
             double* weights, int32_t* loads, int32_t* active_union,
             int32_t* active_count, int64_t* total_load, int32_t* order_out,
             int32_t* t_out, int32_t* n_out, int32_t* base_union,
             int32_t* base_union_count, char* err, int32_t errlen);

/* router_scores, moe_layer.hpp:71-90 (logits = x . R in fp64, row softmax) */
void oo_router_scores(const double* x, const double* router, int32_t B, int32_t D,
                      int32_t N, double* scores);
/* the softmax half only: scores from given logits (moe_layer.hpp:84-88) */
void oo_softmax_rows(const double* logits, int32_t B, int32_t N, double* scores);

/* moe_forward<double>, moe_layer.hpp:114-158 with expert_forward :92-107.
 * Weights flat: wg/wu [N][D][H], wd [N][H][D]. mask may be NULL (then empty
 * sets are zero rows). Returns 1 on the reference's invalid_argument cases. */
int oo_moe_forward_f64(const double* wg, const double* wu, const double* wd,
                       int32_t D, int32_t H, int32_t N, const double* x, int32_t B,
                       const int32_t* sets, const int32_t* set_len,
                       const double* weights, int32_t stride, const uint8_t* mask,
                       double* out, char* err, int32_t errlen);
/* moe_forward<float>: expert math in float, mixture in double. */
int oo_moe_forward_f32(const float* wg, const float* wu, const float* wd, int32_t D,
                       int32_t H, int32_t N, const double* x, int32_t B,
                       const int32_t* sets, const int32_t* set_len,
                       const double* weights, int32_t stride, const uint8_t* mask,
                       double* out, char* err, int32_t errlen);

/* Counter RNG, rng.hpp:24-117 */
uint64_t oo_splitmix64(uint64_t z);
uint64_t oo_stream_key(const uint64_t* parts, int32_t n);
/* normal #f (0-based) of the stream `key` (Box-Muller pairs, rng.hpp:65-77) */
double oo_stream_normal(uint64_t key, uint64_t f);

/* Score generators (score_gen.cpp:100-160): one (step, layer) batch, [B][N]. */
void oo_gen_dirichlet(int32_t N, int32_t B, uint64_t seed, double alpha, int32_t step,
                      int32_t layer, double* out);
void oo_gen_clustered(int32_t N, int32_t B, uint64_t seed, int32_t groups, double conc,
                      double spread, int32_t step, int32_t layer, double* out);

/* make_random_layer, moe_layer.cpp:76-98 (exact); fills the flat arrays.
 * n_threads > 1 splits the counter stream across pthreads (identical bits). */
void oo_make_random_layer(int32_t D, int32_t H, int32_t N, uint64_t seed,
                          double* router, double* wg, double* wu, double* wd,
                          int32_t n_threads);
/* make_random_batch, moe_layer.cpp:100-116 */
void oo_make_random_batch(int32_t B, int32_t D, uint64_t seed, int32_t step,
                          int32_t layer, double* x);

/* output_divergence, moe_layer.cpp:57-74 */
int oo_output_divergence(const double* ref, const double* test, int32_t B,
                         int32_t D, double* mean_rel, double* max_rel);

/* expected_active_experts, latency.cpp:30-37 */
double oo_expected_active_experts(int32_t N, int32_t k, int32_t B);

#ifdef __cplusplus
}
#endif

#endif
