// Router-score generators on the device: the
// reference's ScoreSource for Dirichlet and clustered batches
// (score_gen.cpp:100-160) over its counter RNG (rng.hpp:24-117), one thread
// per generated row, every (step, layer) cell of a run in one launch.
//
// Each row owns an independent counter stream (seed, step, layer, token,
// tag), so rows are embarrassingly parallel and the sequential per-row
// semantics (draw order, the cached Box-Muller spare, Marsaglia-Tsang
// rejection, sequential normalisation sums) are kept exactly. The
// transcendentals are CUDA's double-precision log/sin/cos/pow/exp (<= 2 ulp),
// not glibc's, so rows match the reference to ~1e-15 relative, not bit for
// bit (tests/test_score_gen_gpu.py bounds it at 1e-12).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "oea_internal.cuh"

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kDirichletTag = 201, kTemplateTag = 202, kNoiseTag = 203;  // score_gen.cpp:15-17
constexpr double kPi = 3.14159265358979323846;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // rng.hpp:24-31
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

struct Rng {  // CounterRng (rng.hpp:46-117)
  uint64_t key, counter;
  double spare;
  bool has_spare;
  __device__ Rng(uint64_t seed, uint64_t step, uint64_t layer, uint64_t token, uint64_t tag)
      : counter(0), spare(0.0), has_spare(false) {
    uint64_t h = 0x853C49E6748FEA9Bull;  // stream_key (rng.hpp:38-44)
    const uint64_t parts[5] = {seed, step, layer, token, tag};
#pragma unroll
    for (int i = 0; i < 5; ++i) h = mix64(h + kGolden + parts[i]);
    key = h;
  }
  __device__ double unit() {  // (0, 1], rng.hpp:54-62
    ++counter;
    return static_cast<double>((mix64(key + counter * kGolden) >> 11) + 1) * 0x1.0p-53;
  }
  __device__ double normal() {  // Box-Muller pairs, rng.hpp:65-77
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    const double u1 = unit();
    const double u2 = unit();
    const double r = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * kPi * u2;
    spare = r * sin(theta);
    has_spare = true;
    return r * cos(theta);
  }
  // Marsaglia-Tsang (rng.hpp:82-98); alpha < 1 boosts: Gamma(a + 1) * u^(1/a)
  // with u drawn first (the recursion, unrolled: at most one boost level).
  __device__ double gamma(double alpha) {
    double boost = 1.0;
    if (alpha < 1.0) {
      const double u = unit();
      boost = pow(u, 1.0 / alpha);
      alpha += 1.0;
    }
    const double d = alpha - 1.0 / 3.0;
    const double c = 1.0 / sqrt(9.0 * d);
    for (;;) {
      const double x = normal();
      double v = 1.0 + c * x;
      if (v <= 0.0) continue;
      v = v * v * v;
      const double u = unit();
      const double x2 = x * x;
      if (u < 1.0 - 0.0331 * x2 * x2) return d * v * boost;
      if (log(u) < 0.5 * x2 + d * (1.0 - v + log(v))) return d * v * boost;
    }
  }
};

// row r of the run: cell (step0 + r / (L B), (r / B) % L), token r % B
__global__ void k_gen_dirichlet(uint64_t seed, int step0, int L, int B, int N, double alpha,
                                long long rows, double* __restrict__ out) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const long long cell = r / B;
  Rng rng(seed, static_cast<uint64_t>(step0 + cell / L), static_cast<uint64_t>(cell % L),
          static_cast<uint64_t>(r % B), kDirichletTag);
  double* row = out + r * N;
  double sum = 0.0;  // sequential, as the reference's row sum
  for (int e = 0; e < N; ++e) {
    const double g = rng.gamma(alpha);
    row[e] = g;
    sum += g;
  }
  for (int e = 0; e < N; ++e) row[e] /= sum;
}

// group templates: row (cell, g) of N standard normals
__global__ void k_gen_templates(uint64_t seed, int step0, int L, int G, int N, long long rows,
                                double* __restrict__ tpl) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const long long cell = r / G;
  Rng rng(seed, static_cast<uint64_t>(step0 + cell / L), static_cast<uint64_t>(cell % L),
          static_cast<uint64_t>(r % G), kTemplateTag);
  for (int e = 0; e < N; ++e) tpl[r * N + e] = rng.normal();
}

// token rows: logits = spread * (template_{i % G} + noise / concentration),
// then the max-subtracted softmax with a sequential sum (score_gen.cpp:19-23)
__global__ void k_gen_clustered(uint64_t seed, int step0, int L, int B, int G, int N,
                                double conc, double spread, long long rows,
                                const double* __restrict__ tpl, double* __restrict__ out) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const long long cell = r / B;
  const int i = static_cast<int>(r % B);
  Rng rng(seed, static_cast<uint64_t>(step0 + cell / L), static_cast<uint64_t>(cell % L),
          static_cast<uint64_t>(i), kNoiseTag);
  const double* t = tpl + (cell * G + i % G) * N;
  double* row = out + r * N;
  double m = 0.0;
  for (int e = 0; e < N; ++e) {
    const double l = spread * (t[e] + rng.normal() / conc);
    row[e] = l;
    m = e == 0 || l > m ? l : m;
  }
  double sum = 0.0;
  for (int e = 0; e < N; ++e) {
    const double v = exp(row[e] - m);
    row[e] = v;
    sum += v;
  }
  for (int e = 0; e < N; ++e) row[e] /= sum;
}

}  // namespace

namespace oea_host {

int gen_scores_launch(oea_ctx* ctx, const oea_score_gen_cfg& c, int step0, int nsteps,
                      double* out, cudaStream_t s) {
  const long long cells = static_cast<long long>(nsteps) * c.layers;
  const long long rows = cells * c.batch;
  constexpr int kThreads = 128;
  if (c.kind == OEA_GEN_DIRICHLET) {
    k_gen_dirichlet<<<static_cast<unsigned>((rows + kThreads - 1) / kThreads), kThreads, 0, s>>>(
        c.seed, step0, c.layers, c.batch, c.n_experts, c.alpha, rows, out);
    OEA_LAUNCHED(ctx);
    return OEA_OK;
  }
  double* tpl = nullptr;
  const long long trows = cells * c.groups;
  OEA_CUDA_TRY(ctx, cudaMallocAsync(reinterpret_cast<void**>(&tpl),
                                    sizeof(double) * trows * c.n_experts, s));
  k_gen_templates<<<static_cast<unsigned>((trows + kThreads - 1) / kThreads), kThreads, 0, s>>>(
      c.seed, step0, c.layers, c.groups, c.n_experts, trows, tpl);
  OEA_LAUNCHED(ctx);
  k_gen_clustered<<<static_cast<unsigned>((rows + kThreads - 1) / kThreads), kThreads, 0, s>>>(
      c.seed, step0, c.layers, c.batch, c.groups, c.n_experts, c.within_group_concentration,
      c.between_group_spread, rows, tpl, out);
  OEA_LAUNCHED(ctx);
  OEA_CUDA_TRY(ctx, cudaFreeAsync(tpl, s));
  return OEA_OK;
}

}  // namespace oea_host
