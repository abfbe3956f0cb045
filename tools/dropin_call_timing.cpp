// Per-call host timing of the C++ drop-in at acceptance criterion 6's shape (acceptance.cpp:267-289:
// windowed(w=256), N=4096, d=64, one head, Matrix<float>): blocked_forward / blocked_backward.
//   g++ -std=c++20 -O2 -Iinclude tools/dropin_call_timing.cpp -Lpaper_2409_15097_b200 -lbbm -Wl,-rpath,$PWD/paper_2409_15097_b200 -o build/dropin_call_timing
#include <chrono>
#include <cstdio>
#include <random>

#include "blockmask/engine.hpp"
#include "blockmask/generators.hpp"

using namespace blockmask;

int main() {
  const std::size_t n = 4096, d = 64;
  const Mask mask = gen_longformer_windowed(n, 256);
  std::mt19937_64 gen(1);
  auto rnd = [&] {
    Matrix<float> m(n, d);
    for (std::size_t i = 0; i < m.size(); ++i) m.data()[i] = static_cast<float>((gen() >> 40) * 0x1.0p-24 * 2 - 1);
    return m;
  };
  const Matrix<float> q = rnd(), k = rnd(), v = rnd(), g = rnd();
  auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  for (Variant var : {Variant::dense, Variant::binblk}) {
    const double p0 = now();
    const MaskPrep prep = preprocess_mask(mask, BlockSpec{64, 64});
    const double p1 = now();
    std::printf("%s: preprocess %.3f ms\n", to_string(var), p1 - p0);
    for (int it = 0; it < 5; ++it) {
      const double t0 = now();
      const auto f = blocked_forward(q, k, v, 0.125, mask, prep, var);
      const double t1 = now();
      const auto b = blocked_backward(q, k, v, 0.125, mask, prep, var, f, g);
      const double t2 = now();
      std::printf("  iter %d: fwd %.3f ms, bwd %.3f ms\n", it, t1 - t0, t2 - t1);
    }
  }
  return 0;
}
