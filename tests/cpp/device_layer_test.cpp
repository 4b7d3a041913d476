// C++ caller of the resident decode hot path through include/oea/device_layer.hpp
// (run by tests/test_dropin_gpu.py on a B200): eager device decode, host-buffer
// decode, one-call graph and a PDL chain graph must give bit-identical outputs,
// the exported plan must be well formed, and argument errors must throw the
// reference's exception types.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "oea/device_layer.hpp"

using namespace oea::device;

static int fails = 0;
#define EXPECT(c)                                              \
  do {                                                         \
    if (!(c)) {                                                \
      std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                 \
    }                                                          \
  } while (0)

static uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return static_cast<uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

int main() {
  const int D = 512, H = 256, N = 64, B = 16;
  Context ctx(0);
  Layer a(ctx, D, H, N), b(ctx, D, H, N);
  a.init_random(3);
  b.init_random(4);
  const Routing cfg = Routing::simplified(4, 8);

  std::vector<uint16_t> x(static_cast<size_t>(B) * D);
  uint32_t s = 12345u;
  for (auto& v : x) {
    s = s * 1664525u + 1013904223u;
    v = to_bf16((static_cast<float>(s >> 8) / 16777216.0f - 0.5f) * 4.0f);
  }
  void *xd = nullptr, *o1 = nullptr, *o2 = nullptr, *o3 = nullptr;
  cudaMalloc(&xd, x.size() * 2);
  cudaMalloc(&o1, static_cast<size_t>(B) * D * 4);
  cudaMalloc(&o2, static_cast<size_t>(B) * D * 4);
  cudaMalloc(&o3, static_cast<size_t>(B) * D * 4);
  cudaMemcpy(xd, x.data(), x.size() * 2, cudaMemcpyHostToDevice);

  std::vector<float> eager(static_cast<size_t>(B) * D), host(eager.size()), gr(eager.size()),
      ch(eager.size());
  a.decode(xd, B, cfg, o1);
  ctx.synchronize();
  cudaMemcpy(eager.data(), o1, eager.size() * 4, cudaMemcpyDeviceToHost);
  const Layer::Plan plan = a.last_plan(B, cfg);
  EXPECT(!plan.active.empty());
  for (int t = 0; t < B; ++t) {
    EXPECT(plan.set_len[t] >= 4 && plan.set_len[t] <= 8);
    double w = 0.0;
    for (int j = 0; j < plan.set_len[t]; ++j) {
      const int e = plan.sets[t * plan.stride + j];
      EXPECT(e >= 0 && e < N);
      w += plan.weights[t * plan.stride + j];
    }
    EXPECT(w > 0.999 && w < 1.001);
  }

  a.decode_host(x.data(), B, cfg, host.data());
  EXPECT(std::memcmp(host.data(), eager.data(), eager.size() * 4) == 0);

  {
    Graph g = a.graph(xd, B, cfg, o2);
    g.launch();
    ctx.synchronize();
    cudaMemcpy(gr.data(), o2, gr.size() * 4, cudaMemcpyDeviceToHost);
    EXPECT(std::memcmp(gr.data(), eager.data(), eager.size() * 4) == 0);
  }
  {
    // a, b, a: the last output (o3) is layer a's again
    Graph g = chain_graph(ctx, {&a, &b, &a}, {xd, xd, xd}, B, cfg, {o2, o1, o3});
    g.launch();
    g.launch();
    ctx.synchronize();
    cudaMemcpy(ch.data(), o3, ch.size() * 4, cudaMemcpyDeviceToHost);
    EXPECT(std::memcmp(ch.data(), eager.data(), eager.size() * 4) == 0);
    std::vector<float> ob(eager.size());
    cudaMemcpy(ob.data(), o1, ob.size() * 4, cudaMemcpyDeviceToHost);
    EXPECT(std::memcmp(ob.data(), eager.data(), eager.size() * 4) != 0);  // layer b differs
  }

  bool threw = false;
  try {
    a.decode(xd, B, Routing::simplified(9, 8), o1);  // k0 > k_max
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    Layer bad(ctx, 0, H, N);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);

  cudaFree(xd);
  cudaFree(o1);
  cudaFree(o2);
  cudaFree(o3);
  if (fails) return 1;
  std::printf("device_layer_test ok (T=%zu, launches=%lld)\n", plan.active.size(),
              static_cast<long long>(ctx.kernel_launches()));
  return 0;
}
