/*
 * oea_cuda.h — the C ABI of the B200-native Opportunistic Expert Activation
 * (OEA) MoE decode layer.
 *
 * This is the drop-in boundary. The reference (arxiv 2511.02237, proj/) has no
 * plugin registry or FFI: its "operator API" is the C++ free functions in
 *   proj/include/oea/routing.hpp:111-141   (sort_experts, route_topk,
 *                                           phase1_baseline, phase2_piggyback,
 *                                           route, batch_stats)
 *   proj/include/oea/moe_layer.hpp:70-178  (router_scores, expert_forward,
 *                                           moe_forward, make_random_layer, ...)
 * This repo keeps that C++ API verbatim in include/oea/ (routing.hpp,
 * moe_layer.hpp, rng.hpp); its adapter
 * (paper_2511_02237_b200/csrc/adapter.cpp) and the Python mirror
 * (paper_2511_02237_b200/__init__.py) both call the entry points below, which
 * run hand-written sm_100a kernels. There is no CPU fallback: every compute
 * entry point either launches CUDA work or returns an error.
 *
 * Conventions
 *   - Plain C types only. Matrices are dense row-major. Sizes are int32 unless
 *     a count can exceed 2^31.
 *   - Every function returns an oea_status. On failure the message is
 *     available from oea_last_error(); messages for OEA_ERR_INVALID_ARGUMENT
 *     and OEA_ERR_DOMAIN are the reference's exception texts (what() of the
 *     std::invalid_argument / std::domain_error it would throw), so adapters
 *     can rethrow the same type with the same text.
 *   - "_host" entry points take host buffers, do the H2D/D2H copies and
 *     synchronise. The others take device pointers and a cudaStream_t passed
 *     as void* (NULL = the context's stream) and are asynchronous.
 *   - A context owns one CUDA stream and a pre-sized workspace; use one
 *     context per host thread (the reference's functions are pure and
 *     reentrant, simulate.cpp:142-150, so the adapter keeps a thread_local
 *     context).
 */
#ifndef OEA_CUDA_H_
#define OEA_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OEA_ABI_VERSION 1

typedef enum {
  OEA_OK = 0,
  OEA_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  OEA_ERR_DOMAIN = 2,           /* reference: std::domain_error (routing.cpp:41-44) */
  OEA_ERR_CUDA = 3,             /* CUDA runtime / launch failure, or no GPU */
  OEA_ERR_NCCL = 4,             /* expert-parallel communicator failure */
  OEA_ERR_INTERNAL = 5
} oea_status;

/* RoutingMode, routing.hpp:45 */
typedef enum {
  OEA_MODE_VANILLA = 0,
  OEA_MODE_PRUNED = 1,
  OEA_MODE_OEA = 2,
  OEA_MODE_SIMPLIFIED = 3
} oea_mode;

/* CapSemantics, routing.hpp:49 */
typedef enum { OEA_CAP_EXACT = 0, OEA_CAP_PSEUDOCODE = 1 } oea_cap;

typedef enum { OEA_DTYPE_F64 = 0, OEA_DTYPE_F32 = 1, OEA_DTYPE_BF16 = 2 } oea_dtype;

/* RoutingConfig, routing.hpp:56-76 (field for field). */
typedef struct {
  int32_t mode;  /* oea_mode */
  int32_t k;
  int32_t k0;
  double p;
  int32_t k_max;
  int32_t max_p; /* 0 = "all N" */
  int32_t cap;   /* oea_cap */
} oea_routing_cfg;

/*
 * Caller-owned buffers for a RoutingPlan (routing.hpp:95-103) plus the
 * optional intermediate products of route(). Pointers are host pointers for
 * *_host calls and device pointers otherwise. Optional members may be NULL.
 *   sets/weights are [B x set_stride]; row i holds set_len[i] entries in
 *   descending-score (rank) order, the rest is -1 / 0.
 */
typedef struct {
  int32_t set_stride;        /* >= oea_plan_set_stride(resolved cfg) */
  int32_t* sets;             /* [B * set_stride]            required */
  int32_t* set_len;          /* [B]                          required */
  double* weights;           /* [B * set_stride] f64         optional */
  float* weights_f32;        /* [B * set_stride] f32         optional */
  int32_t* loads;            /* [N]                          optional */
  int32_t* active_union;     /* [N], ascending               optional */
  int32_t* active_count;     /* [1]  (T)                     optional */
  int64_t* total_load;       /* [1]                          optional */
  int32_t* order;            /* [B * N] sort_experts output  optional */
  int32_t* phase1_t;         /* [B]                          optional */
  int32_t* phase1_n;         /* [B]                          optional */
  int32_t* base_union;       /* [N], ascending               optional */
  int32_t* base_union_count; /* [1]                          optional */
} oea_plan_view;

typedef struct oea_ctx* oea_ctx_t;
typedef struct oea_layer* oea_layer_t;
typedef struct oea_graph* oea_graph_t;

/* ---- context ------------------------------------------------------------ */
int oea_abi_version(void);
/* Creates a context on `device` (its own non-blocking stream + workspace).
 * Fails with OEA_ERR_CUDA when no sm_100 GPU is present: there is no CPU path. */
int oea_ctx_create(int32_t device, oea_ctx_t* out);
int oea_ctx_destroy(oea_ctx_t ctx);
/* Last error message of `ctx` (or of the calling thread when ctx is NULL). */
const char* oea_last_error(oea_ctx_t ctx);
int oea_ctx_stream(oea_ctx_t ctx, void** stream_out);
int oea_ctx_synchronize(oea_ctx_t ctx);
/* Number of kernels this context has launched (for launch accounting). */
int64_t oea_ctx_kernel_launches(oea_ctx_t ctx);

/* ---- config (host logic, routing.cpp:153-182) --------------------------- */
/* RoutingConfig::resolved(n_experts): pins Simplified, resolves max_p=0 and
 * validates with the reference's messages. No device work. */
int oea_config_resolve(const oea_routing_cfg* in, int32_t n_experts,
                       oea_routing_cfg* out);
/* Minimum set_stride for a resolved config: k (vanilla), k0 (pruned),
 * k_max or k_max+1 (oea/simplified, exact/pseudocode cap). */
int32_t oea_plan_set_stride(const oea_routing_cfg* resolved);

/* ---- K1: routing on fp64 scores (route(), routing.cpp:305-326) ----------
 * Bit-exact with the reference: composite order (score desc, index asc)
 * compared as doubles, p==1 short-circuit, sequential fp64 cumsum and
 * renormalisation. mask: B bytes (0 = padding row) or NULL. */
int oea_route_f64_host(oea_ctx_t ctx, const double* scores, const uint8_t* mask,
                       int32_t B, int32_t N, const oea_routing_cfg* cfg,
                       const oea_plan_view* plan);
/* Device-buffer route() on `stream` (asynchronous). The single-launch path
 * (p == 1, max_p >= N, N <= 128) exchanges the batch union through the
 * context's epoch-tagged scratch: like decodes, routes of one context must
 * not run concurrently on different streams. */
int oea_route_f64(oea_ctx_t ctx, const double* scores_dev, const uint8_t* mask_dev,
                  int32_t B, int32_t N, const oea_routing_cfg* cfg,
                  const oea_plan_view* plan_dev, void* stream);
/* Batched route(): R independent records (e.g. the (step, layer) batches of a
 * score trace, io.cpp:85-172) of rows[r] x N scores each, concatenated row-wise
 * (mask: sum(rows) bytes or NULL). Each record is routed exactly as
 * oea_route_f64_host would route it alone (its own union and aggregates);
 * replaces the per-record loop of the reference's `route` command
 * (oea_cli.cpp:153-175). Plan layout: sets/weights/set_len/phase1_* per row
 * as in oea_plan_view over sum(rows) rows; loads/active_union/base_union are
 * [R][N], active_count/total_load/base_union_count are [R]; every member is
 * optional here (e.g. only active_count for a sweep) and order must be NULL. One launch sequence for every configuration (the fast path when
 * p == 1, max_p >= N, N <= 128; the general rank-sort path otherwise). */
int oea_route_f64_batched_host(oea_ctx_t ctx, const double* scores, const uint8_t* mask,
                               const int32_t* rows, int32_t R, int32_t N,
                               const oea_routing_cfg* cfg, const oea_plan_view* plan);
/* sort_experts (routing.cpp:184-203): order[B*N]; sorts masked rows too. */
int oea_sort_experts_f64_host(oea_ctx_t ctx, const double* scores, int32_t B,
                              int32_t N, int32_t* order);
/* phase1_baseline (routing.cpp:226-268) from a caller-supplied order.
 * base_sets: [B * base_stride] (base_stride >= k0), -1 padded. */
int oea_phase1_f64_host(oea_ctx_t ctx, const double* scores, const uint8_t* mask,
                        int32_t B, int32_t N, const int32_t* order,
                        const oea_routing_cfg* cfg, int32_t* t, int32_t* n,
                        int32_t* base_sets, int32_t base_stride,
                        int32_t* base_union, int32_t* base_union_count);
/* phase2_piggyback (routing.cpp:270-303) from caller-supplied order, baseline
 * sizes n and base union. Fills sets/set_len/loads/active_union/active_count/
 * total_load (weights are left untouched, as in the reference). */
int oea_phase2_f64_host(oea_ctx_t ctx, const uint8_t* mask, int32_t B, int32_t N,
                        const int32_t* order, const int32_t* n,
                        const int32_t* base_union, int32_t base_union_count,
                        const oea_routing_cfg* cfg, const oea_plan_view* plan);

/* Expert parallelism with the combine fused into the decode over peer memory
 * (NVLink / NVSwitch; no NCCL on the data path). Rank r of `world` (<= 8)
 * decodes the whole batch x_all (B x D, B % world == 0) on its shard; the
 * kernel's combine stores token t's partial mixture straight into its owner
 * o = t / (B / world): recv[o][r][t - o B / world][D] (fp32), then every CTA
 * adds 1 to every owner's arrival counter cnt[o] (system-scope release).
 * recv[] / cnt[] are this rank's views of every rank's buffers
 * (oea_ipc_open_handle); recv[o] holds [world][B / world][D] floats, cnt[o]
 * two ints (arrivals, consumed; zero-filled at allocation).
 * oea_ep_combine (owner side, after its own partial launch) waits for this
 * launch's world x grid arrivals (the target is kept on the device, so both
 * calls can be captured in a CUDA graph) and sums the world slots in rank
 * order into out_local [B / world][D]. */
int oea_moe_decode_ep_partial(oea_ctx_t ctx, oea_layer_t layer, const void* x_all_dev, int32_t B,
                              const oea_routing_cfg* cfg, int32_t world, int32_t rank,
                              float* const* recv, int32_t* const* cnt, void* stream);
int oea_ep_combine(oea_ctx_t ctx, const float* recv_local, int32_t* cnt_local, int32_t world,
                   int32_t tokens_per_rank, int32_t D, float* out_local, void* stream);
/* CUDA IPC of a device buffer between the ranks' processes (64-byte handle;
 * use buffers from oea_device_alloc, whose base the handle maps exactly). */
int oea_device_alloc(oea_ctx_t ctx, uint64_t bytes, void** dev_ptr); /* zero-filled */
int oea_device_free(oea_ctx_t ctx, void* dev_ptr);
int oea_ipc_get_handle(oea_ctx_t ctx, const void* dev_ptr, void* handle);
int oea_ipc_open_handle(oea_ctx_t ctx, const void* handle, void** dev_ptr);
int oea_ipc_close_handle(oea_ctx_t ctx, void* dev_ptr);

/* Decoder glue between stacked MoE layers (the C4 stack, attention omitted):
 * h += add (when add != NULL), then x = bf16(h * rsqrt(mean(h^2) + eps)) per
 * row; h, add: [rows][D] fp32 device, x: [rows][D] bf16 device. One launch. */
int oea_residual_rmsnorm(oea_ctx_t ctx, float* h, const float* add, void* x_bf16, int32_t rows,
                         int32_t D, double eps, void* stream);

/* ---- router-score generators (score_gen.cpp:100-160) ----------------------
 * ScoreSource batches on the device: Dirichlet(alpha) rows (Marsaglia-Tsang
 * gammas over the counter RNG) or clustered rows (softmax of group template +
 * token noise). Steps [step0, step0 + nsteps) x all layers in one launch,
 * out [nsteps][layers][batch][n_experts] f64, cell (step, layer) = the
 * reference's gen_scores(cfg, step, layer) within ~1e-15 relative (device
 * libm). Errors: the reference's ScoreGenConfig::validate texts. */
enum { OEA_GEN_DIRICHLET = 0, OEA_GEN_CLUSTERED = 1 };
typedef struct {
  int32_t kind;
  int32_t n_experts, batch, steps, layers;
  uint64_t seed;
  double alpha;                      /* Dirichlet */
  int32_t groups;                    /* clustered */
  double within_group_concentration; /* clustered */
  double between_group_spread;       /* clustered */
} oea_score_gen_cfg;
int oea_gen_scores(oea_ctx_t ctx, const oea_score_gen_cfg* cfg, int32_t step0, int32_t nsteps,
                   double* out_dev, void* stream);
int oea_gen_scores_host(oea_ctx_t ctx, const oea_score_gen_cfg* cfg, int32_t step0,
                        int32_t nsteps, double* out_host);

/* ---- device-resident MoE layer ------------------------------------------
 * dtype BF16: the decode hot path (fragment-ordered bf16 weights streamed by
 * TMA bulk copies, mma.sync tensor tiles). F32 / F64: SIMT FFN kept for the
 * drop-in moe_forward<float/double> tolerances (1e-5 / fp64). */
int oea_layer_create(oea_ctx_t ctx, int32_t D, int32_t H, int32_t N, int32_t dtype,
                     oea_layer_t* out);
/* Expert-parallel shard (bf16): holds experts [e_begin, e_end) of the N its
 * full router routes over (ownership: oea_ep_owner). Routing is global, so the
 * expert sets equal the unsharded layer's bit for bit; oea_moe_decode returns
 * this shard's partial sum out[t] = sum over held j in S_t of w_j y_j (set
 * order), to be summed across the EP group (bench/EP: NCCL reduce-scatter).
 * Expert indices of upload/download stay global. */
int oea_layer_create_shard(oea_ctx_t ctx, int32_t D, int32_t H, int32_t N, int32_t dtype,
                           int32_t e_begin, int32_t e_end, oea_layer_t* out);
int oea_layer_destroy(oea_layer_t layer);
/* router: D x N row-major (moe_layer.hpp:46). src_dtype: oea_dtype of src.
 * src_on_device: 0 host, 1 device. Values are rounded to the layer dtype
 * (round-to-nearest-even). */
int oea_layer_upload_router(oea_layer_t layer, const void* router, int32_t src_dtype,
                            int32_t src_on_device);
/* expert e: w_gate D x H, w_up D x H, w_down H x D row-major (moe_layer.hpp:29-34). */
int oea_layer_upload_expert(oea_layer_t layer, int32_t e, const void* w_gate,
                            const void* w_up, const void* w_down, int32_t src_dtype,
                            int32_t src_on_device);
/* make_random_layer(dims, seed) distributions (moe_layer.cpp:76-98): one
 * counter stream keyed (seed, 101), router then per-expert gate/up/down,
 * N(0,1/D) / N(0,1/H). Generated on the device in fp64, then rounded. */
int oea_layer_init_random(oea_layer_t layer, uint64_t seed);
/* Read back the stored (rounded) values in reference layout, as dst_dtype
 * (F64 or F32 or BF16) into host buffers. */
int oea_layer_download_router(oea_layer_t layer, void* router, int32_t dst_dtype);
int oea_layer_download_expert(oea_layer_t layer, int32_t e, void* w_gate, void* w_up,
                              void* w_down, int32_t dst_dtype);
int oea_layer_info(oea_layer_t layer, int32_t* D, int32_t* H, int32_t* N,
                   int32_t* dtype, int64_t* bytes_per_expert, int64_t* device_bytes);

/* ---- the decode layer: router -> route -> compaction -> grouped FFN ------
 * x: B x D in the layer dtype (bf16 layers: bf16), mask: B bytes or NULL,
 * out: B x D fp32 (bf16 layers) or fp64 (f32/f64 layers).
 * BF16 layers run the fused router (K2, fp32 logits, ranking on logits) and
 * the tensor-core FFN (K4/K5); F32/F64 layers run router_scores in fp64 +
 * route_f64 + the SIMT FFN.
 * stream: NULL = the context's own (non-blocking) stream; pass
 * cudaStreamLegacy ((void*)0x1) to order with the legacy default stream.
 * Launches of one context are serialised on its workspace: do not run two
 * decodes of the same context concurrently on different streams. */
int oea_moe_decode(oea_ctx_t ctx, oea_layer_t layer, const void* x_dev,
                   const uint8_t* mask_dev, int32_t B, const oea_routing_cfg* cfg,
                   void* out_dev, void* stream);
/* Same, end to end from host buffers; synchronises before returning.
 * When x and out both lie in pinned host memory (cudaHostAlloc /
 * cudaHostRegister / torch pin_memory), mask is NULL and the call takes the
 * fused single launch (bf16, B <= 64), the kernel reads x and writes out over
 * the host link itself (zero copy), replayed from a per-context graph cache
 * keyed by (layer, B, cfg). Otherwise x/mask are copied in and out copied
 * back around the device decode. */
int oea_moe_decode_host(oea_ctx_t ctx, oea_layer_t layer, const void* x_host,
                        const uint8_t* mask_host, int32_t B,
                        const oea_routing_cfg* cfg, void* out_host);
/* Export of the most recent decode's routing (synchronises): the plan
 * (weights as f64 and/or f32), and logits [B x N] fp32 (bf16 layers) — the
 * router output the parity harness feeds to the CPU reference. */
int oea_last_plan_host(oea_ctx_t ctx, const oea_plan_view* plan, float* logits,
                       double* scores);

/* CUDA-graph capture of one decode call (fixed pointers/B/cfg). */
int oea_decode_graph_create(oea_ctx_t ctx, oea_layer_t layer, const void* x_dev,
                            const uint8_t* mask_dev, int32_t B,
                            const oea_routing_cfg* cfg, void* out_dev,
                            oea_graph_t* out);
/* n decode calls (layers[i]: xs_dev[i] -> outs_dev[i], same B / cfg / mask)
 * captured back to back in ONE graph, as a decode step's layers run. The fused
 * launches are programmatic dependents of the previous kernel (PDL), so each
 * call's launch and setup overlap the previous call's tail. */
int oea_decode_chain_graph_create(oea_ctx_t ctx, int32_t n, const oea_layer_t* layers,
                                  const void* const* xs_dev, const uint8_t* mask_dev, int32_t B,
                                  const oea_routing_cfg* cfg, void* const* outs_dev,
                                  oea_graph_t* out);
/* The same decode captured as two graphs (router+compaction | FFN), without
 * the programmatic overlap, so each stage can be timed on its own (bench). */
int oea_decode_stage_graphs_create(oea_ctx_t ctx, oea_layer_t layer, const void* x_dev,
                                   const uint8_t* mask_dev, int32_t B,
                                   const oea_routing_cfg* cfg, void* out_dev,
                                   oea_graph_t* router_graph, oea_graph_t* ffn_graph);
int oea_graph_launch(oea_graph_t graph, void* stream);
int oea_graph_destroy(oea_graph_t graph);

/* ---- drop-in layer math on a given plan ---------------------------------
 * moe_forward (moe_layer.hpp:114-158) with a caller plan: x B x D fp64 (cast
 * to the layer dtype), sets/set_len/weights as in oea_plan_view, mask B bytes
 * or NULL (reference semantics: an empty set on a real token is an error only
 * when a mask is given). out: B x D fp64, host buffers. */
int oea_moe_forward_plan_host(oea_ctx_t ctx, oea_layer_t layer, const double* x,
                              int32_t B, const int32_t* sets, const int32_t* set_len,
                              const double* weights, int32_t set_stride,
                              const uint8_t* mask, double* out);
/* router_scores (moe_layer.hpp:71-90): softmax(x . router) in fp64. */
int oea_router_scores_host(oea_ctx_t ctx, oea_layer_t layer, const double* x,
                           int32_t B, double* scores);

/* Debug: per-CTA globaltimer stamps of the last FFN launch when the process
 * ran with OEA_FFN_TRACE=1 ([grid][8]: start, end of W1 phase, first W2 unit
 * ready, end, producer done). */
int oea_debug_ffn_trace(oea_ctx_t ctx, uint64_t* host, int32_t n);

/* ---- expert parallelism (Qwen3-235B stack, NCCL all-to-all) ------------ */
/* Expert-block ownership: rank r owns experts [N*r/P, N*(r+1)/P). */
int oea_ep_owner(int32_t N, int32_t world, int32_t expert);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* OEA_CUDA_H_ */
