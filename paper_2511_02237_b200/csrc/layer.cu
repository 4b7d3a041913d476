// layer.cu — device-resident MoE layer: upload + repack into the
// fragment-ordered bf16 layout the decode kernels stream, the on-device
// make_random_layer generator (K8), and read-back in reference layout.
//
// bf16 layout: every matrix is cut into 16x16 A-operand tiles
// of mma.m16n8k16 and each 512-byte tile is stored in register-fragment
// order (lane-major, 16 B per lane), so a warp loads one tile with one
// coalesced 16 B/lane access and no ldmatrix/shuffle:
//   router  [Np/16][Dp/16] tiles, A(r,c) = R[d=16kt+c][n=16rb+r]
//   W1 (e)  row blocks rb < Hp/8, rows 0-7 gate, 8-15 up of h = 8rb + (r&7):
//           A(r,c) = (r<8 ? Wg : Wu)[d=16kt+c][h]
//   W2 (e)  row blocks rb < Dp/16, A(r,c) = Wd[h=16kt+c][d=16rb+r]
// Expert tiles are round-interleaved (round_tile): 8 row blocks (= 8 FFN
// units, one per consumer warp) form a round, and each pipeline stage of a
// round (8 warps x 8 k-tiles = 32 KiB) is contiguous, so the FFN producer
// streams a stage with one TMA bulk copy.
#include <cmath>
#include <vector>

#include "oea_device.cuh"
#include "oea_internal.cuh"
#include "layout.cuh"

namespace oea_dev {

template <typename T>
__device__ __forceinline__ double to_f64(T v);
template <>
__device__ __forceinline__ double to_f64<double>(double v) {
  return v;
}
template <>
__device__ __forceinline__ double to_f64<float>(float v) {
  return static_cast<double>(v);
}
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 v) {
  return static_cast<double>(__bfloat162float(v));
}

template <typename T>
__device__ __forceinline__ T from_f64(double v);
template <>
__device__ __forceinline__ double from_f64<double>(double v) {
  return v;
}
template <>
__device__ __forceinline__ float from_f64<float>(double v) {
  return static_cast<float>(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_f64<__nv_bfloat16>(double v) {
  return __double2bfloat16(v);  // single rounding, nearest-even
}

// kind: 0 router (rows=D, cols=N), 1 gate (D,H), 2 up (D,H), 3 down (H,D).
template <typename S>
__global__ void k_pack_bf16(const S* __restrict__ src, int rows, int cols, int kind, int Dp,
                            int Hp, __nv_bfloat16* __restrict__ dst) {
  const size_t total = static_cast<size_t>(rows) * cols;
  for (size_t f = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(f / cols), c = static_cast<int>(f % cols);
    const __nv_bfloat16 v = from_f64<__nv_bfloat16>(to_f64<S>(src[f]));
    size_t o;
    if (kind == 0)
      o = router_frag_idx(r, c, Dp);
    else if (kind == 3)
      o = w2_frag_idx(r, c, Hp);
    else
      o = w1_frag_idx(r, c, kind == 2, Dp);
    dst[o] = v;
  }
}

template <typename S, typename Dt>
__global__ void k_convert(const S* __restrict__ src, size_t n, Dt* __restrict__ dst) {
  for (size_t f = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[f] = from_f64<Dt>(to_f64<S>(src[f]));
}

template <typename Dt>
__global__ void k_unpack_bf16(const __nv_bfloat16* __restrict__ src, int rows, int cols,
                              int kind, int Dp, int Hp, Dt* __restrict__ dst) {
  const size_t total = static_cast<size_t>(rows) * cols;
  for (size_t f = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(f / cols), c = static_cast<int>(f % cols);
    size_t o;
    if (kind == 0)
      o = router_frag_idx(r, c, Dp);
    else if (kind == 3)
      o = w2_frag_idx(r, c, Hp);
    else
      o = w1_frag_idx(r, c, kind == 2, Dp);
    dst[f] = from_f64<Dt>(to_f64<__nv_bfloat16>(src[o]));
  }
}

// ---- counter RNG (rng.hpp:24-117) -----------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
__device__ __forceinline__ double unit_at(uint64_t key, uint64_t c) {
  const uint64_t u = splitmix64(key + c * 0x9E3779B97F4A7C15ull);
  return static_cast<double>((u >> 11) + 1) * 0x1.0p-53;
}
// Normal #f of the stream: Box-Muller on draws 2(f/2)+1, 2(f/2)+2; even f the
// cosine, odd f the cached sine (rng.hpp:65-77).
__device__ __forceinline__ double stream_normal(uint64_t key, uint64_t f) {
  const uint64_t pair = f >> 1;
  const double u1 = unit_at(key, 2 * pair + 1);
  const double u2 = unit_at(key, 2 * pair + 2);
  const double r = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.14159265358979323846 * u2;
  return (f & 1) ? r * sin(theta) : r * cos(theta);
}

// One logical matrix of make_random_layer: element (r, c) is normal number
// `base + r*cols + c` of the layer stream (moe_layer.cpp:85-96).
template <typename Dt>
__global__ void k_init_matrix(uint64_t key, uint64_t base, int rows, int cols, double scale,
                              int kind, int Dp, int Hp, int frag, Dt* __restrict__ dst) {
  const size_t total = static_cast<size_t>(rows) * cols;
  for (size_t f = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const double v = scale * stream_normal(key, base + f);
    size_t o = f;
    if (frag) {
      const int r = static_cast<int>(f / cols), c = static_cast<int>(f % cols);
      if (kind == 0)
        o = router_frag_idx(r, c, Dp);
      else if (kind == 3)
        o = w2_frag_idx(r, c, Hp);
      else
        o = w1_frag_idx(r, c, kind == 2, Dp);
    }
    dst[o] = from_f64<Dt>(v);
  }
}

// Expert-major router copy for the fused gate GEMV: router_t[n][d] = R[d][n]
// (zero padding included), unpacked from the fragment-ordered tiles.
__global__ void k_router_unpack(const __nv_bfloat16* __restrict__ frag, int Np, int Dp,
                                __nv_bfloat16* __restrict__ out) {
  const size_t total = static_cast<size_t>(Np) * Dp;
  for (size_t f = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(f / Dp), d = static_cast<int>(f % Dp);
    out[f] = frag[router_frag_idx(d, n, Dp)];
  }
}

}  // namespace oea_dev

namespace oea_host {

using namespace oea_dev;

static size_t dtype_size(int dt) {
  return dt == OEA_DTYPE_F64 ? 8 : dt == OEA_DTYPE_F32 ? 4 : 2;
}

static int grid_for(size_t n) {
  size_t g = (n + 255) / 256;
  return static_cast<int>(g > 8192 ? 8192 : (g < 1 ? 1 : g));
}

// Device copy of a (host or device) source array.
struct Staged {
  void* p = nullptr;
  bool owned = false;
  ~Staged() {
    if (owned && p) cudaFree(p);
  }
};
static int stage(oea_ctx* ctx, const void* src, size_t bytes, int on_device, Staged& out) {
  if (on_device) {
    out.p = const_cast<void*>(src);
    return OEA_OK;
  }
  OEA_CUDA_TRY(ctx, cudaMalloc(&out.p, bytes));
  out.owned = true;
  OEA_CUDA_TRY(ctx, cudaMemcpyAsync(out.p, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return OEA_OK;
}

template <typename S>
static void launch_pack(const void* src, int rows, int cols, int kind, const oea_layer* L,
                        void* dst, cudaStream_t s) {
  const size_t n = static_cast<size_t>(rows) * cols;
  k_pack_bf16<S><<<grid_for(n), 256, 0, s>>>(static_cast<const S*>(src), rows, cols, kind,
                                              L->Dp, L->Hp, static_cast<__nv_bfloat16*>(dst));
}

static int pack_or_convert(oea_layer* L, const void* src, int rows, int cols, int kind,
                           int src_dtype, void* dst) {
  oea_ctx* ctx = L->ctx;
  cudaStream_t s = ctx->stream;
  const size_t n = static_cast<size_t>(rows) * cols;
  if (L->dtype == OEA_DTYPE_BF16) {
    if (src_dtype == OEA_DTYPE_F64)
      launch_pack<double>(src, rows, cols, kind, L, dst, s);
    else if (src_dtype == OEA_DTYPE_F32)
      launch_pack<float>(src, rows, cols, kind, L, dst, s);
    else
      launch_pack<__nv_bfloat16>(src, rows, cols, kind, L, dst, s);
  } else {
    // f32 / f64 layers keep the reference layout.
#define OEA_CONVERT(S, Dt)                                                            \
  k_convert<S, Dt><<<grid_for(n), 256, 0, s>>>(static_cast<const S*>(src), n,         \
                                               static_cast<Dt*>(dst))
    if (L->dtype == OEA_DTYPE_F64) {
      if (src_dtype == OEA_DTYPE_F64) OEA_CONVERT(double, double);
      else if (src_dtype == OEA_DTYPE_F32) OEA_CONVERT(float, double);
      else OEA_CONVERT(__nv_bfloat16, double);
    } else {
      if (src_dtype == OEA_DTYPE_F64) OEA_CONVERT(double, float);
      else if (src_dtype == OEA_DTYPE_F32) OEA_CONVERT(float, float);
      else OEA_CONVERT(__nv_bfloat16, float);
    }
#undef OEA_CONVERT
  }
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

int layer_router_refresh(oea_layer* L) {
  if (L->router_t == nullptr) return OEA_OK;
  oea_ctx* ctx = L->ctx;
  const size_t n = static_cast<size_t>(L->Np) * L->Dp;
  k_router_unpack<<<grid_for(n), 256, 0, ctx->stream>>>(
      static_cast<const __nv_bfloat16*>(L->router), L->Np, L->Dp,
      static_cast<__nv_bfloat16*>(L->router_t));
  OEA_LAUNCHED(ctx);
  return OEA_OK;
}

int layer_upload_router(oea_layer* L, const void* src, int src_dtype, int on_device) {
  oea_ctx* ctx = L->ctx;
  Staged st;
  int rc = stage(ctx, src, static_cast<size_t>(L->D) * L->N * dtype_size(src_dtype), on_device, st);
  if (rc) return rc;
  rc = pack_or_convert(L, st.p, L->D, L->N, 0, src_dtype, L->router);
  if (!rc) rc = layer_router_refresh(L);
  if (rc) return rc;
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return OEA_OK;
}

static size_t expert_offset(const oea_layer* L, int which, int e) {
  // which: 1 gate/w1, 2 up, 3 down/w2 ; returns element offset of (global)
  // expert e in this layer's (possibly expert-parallel shard) storage
  e -= L->e_begin;
  if (L->dtype == OEA_DTYPE_BF16) {
    if (which == 3) return static_cast<size_t>(e) * L->Dp * L->Hp;
    return static_cast<size_t>(e) * 2 * L->Dp * L->Hp;
  }
  return static_cast<size_t>(e) * L->D * L->H;
}

int layer_upload_expert(oea_layer* L, int e, const void* wg, const void* wu, const void* wd,
                        int src_dtype, int on_device) {
  oea_ctx* ctx = L->ctx;
  const size_t dh = static_cast<size_t>(L->D) * L->H, es = dtype_size(src_dtype);
  const size_t ls = dtype_size(L->dtype);
  Staged sg, su, sd;
  int rc = stage(ctx, wg, dh * es, on_device, sg);
  if (!rc) rc = stage(ctx, wu, dh * es, on_device, su);
  if (!rc) rc = stage(ctx, wd, dh * es, on_device, sd);
  if (rc) return rc;
  char* w1 = static_cast<char*>(L->w1) + expert_offset(L, 1, e) * ls;
  char* w2 = static_cast<char*>(L->w2) + expert_offset(L, 3, e) * ls;
  if (L->dtype == OEA_DTYPE_BF16) {
    rc = pack_or_convert(L, sg.p, L->D, L->H, 1, src_dtype, w1);
    if (!rc) rc = pack_or_convert(L, su.p, L->D, L->H, 2, src_dtype, w1);
  } else {
    char* up = static_cast<char*>(L->w_up) + expert_offset(L, 2, e) * ls;
    rc = pack_or_convert(L, sg.p, L->D, L->H, 1, src_dtype, w1);
    if (!rc) rc = pack_or_convert(L, su.p, L->D, L->H, 2, src_dtype, up);
  }
  if (!rc) rc = pack_or_convert(L, sd.p, L->H, L->D, 3, src_dtype, w2);
  if (rc) return rc;
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return OEA_OK;
}

template <typename Dt>
static int init_all(oea_layer* L, uint64_t key) {
  oea_ctx* ctx = L->ctx;
  cudaStream_t s = ctx->stream;
  const int D = L->D, H = L->H, N = L->N;
  const int frag = L->dtype == OEA_DTYPE_BF16 ? 1 : 0;
  const double ds = 1.0 / std::sqrt(static_cast<double>(D));
  const double hs = 1.0 / std::sqrt(static_cast<double>(H));
  const size_t dh = static_cast<size_t>(D) * H;
  k_init_matrix<Dt><<<grid_for(static_cast<size_t>(D) * N), 256, 0, s>>>(
      key, 0, D, N, ds, 0, L->Dp, L->Hp, frag, static_cast<Dt*>(L->router));
  OEA_LAUNCHED(ctx);
  for (int e = L->e_begin; e < L->e_begin + L->n_local; ++e) {
    const uint64_t base = static_cast<uint64_t>(D) * N + static_cast<uint64_t>(e) * 3 * dh;
    Dt* w1 = static_cast<Dt*>(L->w1) + expert_offset(L, 1, e);
    Dt* up = frag ? w1 : static_cast<Dt*>(L->w_up) + expert_offset(L, 2, e);
    Dt* w2 = static_cast<Dt*>(L->w2) + expert_offset(L, 3, e);
    k_init_matrix<Dt><<<grid_for(dh), 256, 0, s>>>(key, base, D, H, ds, 1, L->Dp, L->Hp, frag, w1);
    OEA_LAUNCHED(ctx);
    k_init_matrix<Dt><<<grid_for(dh), 256, 0, s>>>(key, base + dh, D, H, ds, 2, L->Dp, L->Hp,
                                                   frag, up);
    OEA_LAUNCHED(ctx);
    k_init_matrix<Dt><<<grid_for(dh), 256, 0, s>>>(key, base + 2 * dh, H, D, hs, 3, L->Dp,
                                                   L->Hp, frag, w2);
    OEA_LAUNCHED(ctx);
  }
  OEA_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return OEA_OK;
}

static uint64_t host_splitmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

int layer_init_random(oea_layer* L, uint64_t seed) {
  // stream_key({seed, 101}) (rng.hpp:38-44, moe_layer.cpp:85)
  uint64_t h = 0x853C49E6748FEA9Bull;
  h = host_splitmix64(h + 0x9E3779B97F4A7C15ull + seed);
  h = host_splitmix64(h + 0x9E3779B97F4A7C15ull + 101);
  if (L->dtype == OEA_DTYPE_BF16) {
    int rc = init_all<__nv_bfloat16>(L, h);
    if (!rc) rc = layer_router_refresh(L);
    if (!rc) OEA_CUDA_TRY(L->ctx, cudaStreamSynchronize(L->ctx->stream));
    return rc;
  }
  if (L->dtype == OEA_DTYPE_F32) return init_all<float>(L, h);
  return init_all<double>(L, h);
}

template <typename Dt>
static int download_matrix(oea_layer* L, const void* src, int rows, int cols, int kind,
                           void* host_dst) {
  oea_ctx* ctx = L->ctx;
  cudaStream_t s = ctx->stream;
  const size_t n = static_cast<size_t>(rows) * cols;
  Dt* tmp = nullptr;
  OEA_CUDA_TRY(ctx, cudaMalloc(&tmp, n * sizeof(Dt)));
  if (L->dtype == OEA_DTYPE_BF16) {
    k_unpack_bf16<Dt><<<grid_for(n), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(src), rows,
                                                  cols, kind, L->Dp, L->Hp, tmp);
  } else if (L->dtype == OEA_DTYPE_F32) {
    k_convert<float, Dt><<<grid_for(n), 256, 0, s>>>(static_cast<const float*>(src), n, tmp);
  } else {
    k_convert<double, Dt><<<grid_for(n), 256, 0, s>>>(static_cast<const double*>(src), n, tmp);
  }
  ctx->launches++;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(host_dst, tmp, n * sizeof(Dt), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(tmp);
  if (e != cudaSuccess) return oea_check_cuda(ctx, e, "layer download");
  return OEA_OK;
}

static int download_dispatch(oea_layer* L, const void* src, int rows, int cols, int kind,
                             void* dst, int dst_dtype) {
  if (dst_dtype == OEA_DTYPE_F64) return download_matrix<double>(L, src, rows, cols, kind, dst);
  if (dst_dtype == OEA_DTYPE_F32) return download_matrix<float>(L, src, rows, cols, kind, dst);
  return download_matrix<__nv_bfloat16>(L, src, rows, cols, kind, dst);
}

int layer_download_router(oea_layer* L, void* dst, int dst_dtype) {
  return download_dispatch(L, L->router, L->D, L->N, 0, dst, dst_dtype);
}

int layer_download_expert(oea_layer* L, int e, void* wg, void* wu, void* wd, int dst_dtype) {
  const size_t ls = dtype_size(L->dtype);
  const char* w1 = static_cast<const char*>(L->w1) + expert_offset(L, 1, e) * ls;
  const char* up = L->dtype == OEA_DTYPE_BF16
                       ? w1
                       : static_cast<const char*>(L->w_up) + expert_offset(L, 2, e) * ls;
  const char* w2 = static_cast<const char*>(L->w2) + expert_offset(L, 3, e) * ls;
  int rc = download_dispatch(L, w1, L->D, L->H, 1, wg, dst_dtype);
  if (!rc) rc = download_dispatch(L, up, L->D, L->H, 2, wu, dst_dtype);
  if (!rc) rc = download_dispatch(L, w2, L->H, L->D, 3, wd, dst_dtype);
  return rc;
}

}  // namespace oea_host

// ---------------------------------------------------------------------------
// Residual + RMSNorm between stacked MoE layers (the decoder glue of the C4
// stack: h += moe(x); x' = bf16(h * rsqrt(mean(h^2) + eps))), one CTA per
// token row, fixed-order block reduction (deterministic). add == null: only
// the normalisation (the stack's first layer).
// ---------------------------------------------------------------------------
namespace oea_dev {
__global__ void __launch_bounds__(256)
    k_residual_rmsnorm(float* __restrict__ h, const float* __restrict__ add,
                       __nv_bfloat16* __restrict__ x, int D, float eps) {
  __shared__ float part[8];
  const size_t row = static_cast<size_t>(blockIdx.x) * D;
  float ss = 0.0f;
  for (int d = threadIdx.x; d < D; d += 256) {
    float v = h[row + d];
    if (add) {
      v += add[row + d];
      h[row + d] = v;
    }
    ss = fmaf(v, v, ss);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.0f;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += part[w];
  const float scale = rsqrtf(tot / static_cast<float>(D) + eps);
  for (int d = threadIdx.x; d < D; d += 256) x[row + d] = __float2bfloat16_rn(h[row + d] * scale);
}
}  // namespace oea_dev

int oea_residual_rmsnorm(oea_ctx_t ctx, float* h, const float* add, void* x_bf16, int32_t rows,
                         int32_t D, double eps, void* stream) {
  if (ctx == nullptr) return oea_set_error(nullptr, OEA_ERR_INVALID_ARGUMENT, "null context");
  if (h == nullptr || x_bf16 == nullptr || rows < 1 || D < 1)
    return oea_set_error(ctx, OEA_ERR_INVALID_ARGUMENT, "residual_rmsnorm: bad arguments");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  oea_dev::k_residual_rmsnorm<<<rows, 256, 0, s>>>(h, add, static_cast<__nv_bfloat16*>(x_bf16), D,
                                                   static_cast<float>(eps));
  OEA_LAUNCHED(ctx);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? OEA_OK : oea_check_cuda(ctx, e, "k_residual_rmsnorm");
}
