// Adapter event-cache exactness (GPU test driver, tests/test_adapter_gpu.py):
// an EventSet is destroyed and a different one -- one event moved at an index
// the old sampled check never looked at -- is rebuilt at the very same heap
// addresses. hawkes::logLikelihood must return the new set's value, equal to
// the value of an identical set at other addresses (which forces a reload).
// Prints one JSON line.
#include <cstdio>
#include <cstdint>
#include <memory>
#include <utility>

#include "sthawkes/likelihood.hpp"
#include "sthawkes/rng.hpp"
#include "sthawkes/simulate.hpp"

using namespace hawkes;

int main() {
  const Index n = 20000;
  Rng rng(static_cast<std::uint64_t>(n));
  const EventSet base = generateBenchmarkCloud(n, SimWindow{0, 15, 0, 15, 4750}, rng);
  Params p;
  p.mu0 = 0.66;
  p.tauX = 1.6;
  p.tauT = 14.0;
  p.theta = 0.344;
  p.omega = 1440.0;
  p.h = 0.0695;
  // an index the sampled check (first, last, (k * golden) % n for k <= 509) skips
  Index moved = n / 2;
  for (;; ++moved) {
    bool sampled = moved == 0 || moved == n - 1;
    for (std::uint64_t k = 1; k <= 509 && !sampled; ++k) {
      sampled = static_cast<Index>((k * 0x9E3779B97F4A7C15ULL) % static_cast<std::uint64_t>(n)) == moved;
    }
    if (!sampled) break;
  }
  auto build = [&](double dx) {
    Eigen::ArrayXd x(n), y(n), t(n);
    for (Index i = 0; i < n; ++i) {
      x[i] = base.xs()[i];
      y[i] = base.ys()[i];
      t[i] = base.ts()[i];
    }
    x[moved] += dx;
    return std::make_unique<EventSet>(std::move(x), std::move(y), std::move(t), base.windowEnd());
  };
  auto a = build(0.0);
  const double* ax = a->xs().data();
  const double la = logLikelihood(*a, p, Backend{}, false).logLik;
  a.reset();  // freed ...
  auto b = build(0.5);  // ... and a different set, likely at the same addresses
  const bool reused = b->xs().data() == ax;
  const double lb = logLikelihood(*b, p, Backend{}, false).logLik;
  auto keep = build(0.0);  // (holds the old block so the copy below lands elsewhere)
  auto c = build(0.5);     // B's data at other addresses: forces a reload
  const double lc = logLikelihood(*c, p, Backend{}, false).logLik;
  const double lb2 = logLikelihood(*b, p, Backend{}, false).logLik;
  std::printf(
      "{\"n\": %ld, \"moved_index\": %ld, \"addresses_reused\": %s, \"ll_a\": %.17g, "
      "\"ll_b\": %.17g, \"ll_b_elsewhere\": %.17g, \"ll_b_again\": %.17g}\n",
      static_cast<long>(n), static_cast<long>(moved), reused ? "true" : "false", la, lb, lc, lb2);
  return (lb == lc && lb2 == lc && la != lb) ? 0 : 1;
}
