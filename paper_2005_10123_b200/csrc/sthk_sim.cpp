// Seeded synthetic-event generators (benchmark inputs), restating the
// reference's generators so that a seed reproduces the reference's data
// bit for bit (checked against the reference build in tests/):
//   Rng                    proj/include/sthawkes/rng.hpp:27-96
//   generateBenchmarkCloud proj/src/simulate.cpp:83-95
//   simulateClusterProcess proj/src/simulate.cpp:10-81
// Compiled with the reference's CMake-equivalent floating-point flags
// (gnu++20 => -ffp-contract=fast, FMA-capable -march) so expression
// contraction matches. Not on the likelihood hot path.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

#include "../../include/sthk_sim.h"

namespace {

// mt19937_64 stream with explicit variate converters (rng.hpp:27-96).
class SimRng {
 public:
  explicit SimRng(uint64_t seed) : gen_(seed) {}

  // 53-bit uniform on [0, 1)
  double u01() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  double uab(double lo, double hi) { return lo + (hi - lo) * u01(); }

  // Box-Muller, two words per variate
  double gauss() {
    const double a = 1.0 - u01();
    const double b = u01();
    return std::sqrt(-2.0 * std::log(a)) * std::cos(2.0 * M_PI * b);
  }

  double expo(double rate) {
    while (true) {
      const double e = -std::log1p(-u01());
      if (e > 0.0) return e / rate;
    }
  }

  // inversion below mean 30, PTRS (Hormann 1993) above
  long poisson(double mean) {
    if (mean <= 0.0) return 0;
    if (mean < 30.0) {
      const double stop = std::exp(-mean);
      long k = 0;
      double prod = u01();
      while (prod > stop) {
        ++k;
        prod *= u01();
      }
      return k;
    }
    const double b = 0.931 + 2.53 * std::sqrt(mean);
    const double a = -0.059 + 0.02483 * b;
    const double inv_alpha = 1.1239 + 1.1328 / (b - 3.4);
    const double vr = 0.9277 - 3.6224 / (b - 2.0);
    while (true) {
      double u = u01() - 0.5;
      double v = u01();
      if (v == 0.0) continue;
      double us = 0.5 - std::fabs(u);
      double k = std::floor((2.0 * a / us + b) * u + mean + 0.43);
      if (us >= 0.07 && v <= vr) return static_cast<long>(k);
      if (k < 0.0 || (us < 0.013 && v > us)) continue;
      if (std::log(v * inv_alpha / (a / (us * us) + b)) <=
          k * std::log(mean) - mean - std::lgamma(k + 1.0)) {
        return static_cast<long>(k);
      }
    }
  }

 private:
  std::mt19937_64 gen_;
};

bool window_ok(const double* w) { return w[1] > w[0] && w[3] > w[2] && w[4] > 0.0; }

std::vector<int64_t> time_order(const std::vector<double>& t) {
  std::vector<int64_t> idx(t.size());
  std::iota(idx.begin(), idx.end(), int64_t{0});
  std::stable_sort(idx.begin(), idx.end(), [&t](int64_t a, int64_t b) { return t[a] < t[b]; });
  return idx;
}

}  // namespace

extern "C" int sthk_sim_cloud(int64_t n, const double* window, uint64_t seed, double* x,
                              double* y, double* t, double* window_end) {
  if (n < 1 || !window || !window_ok(window) || !x || !y || !t) return 1;
  SimRng rng(seed);
  std::vector<double> vx(n), vy(n), vt(n);
  for (int64_t i = 0; i < n; ++i) {
    vx[i] = rng.uab(window[0], window[1]);
    vy[i] = rng.uab(window[2], window[3]);
    vt[i] = rng.uab(0.0, window[4]);
  }
  const auto ord = time_order(vt);
  for (int64_t i = 0; i < n; ++i) {
    x[i] = vx[ord[i]];
    y[i] = vy[ord[i]];
    t[i] = vt[ord[i]];
  }
  if (window_end) *window_end = window[4];
  return 0;
}

extern "C" int sthk_sim_cluster(const double* p, const double* window, double rate,
                                uint64_t seed, int64_t capacity, double* x, double* y,
                                double* t, int* parent, int64_t* count) {
  if (!p || !window || !window_ok(window) || !(rate > 0.0) || !count) return 1;
  for (int k = 0; k < 6; ++k) {
    if (!std::isfinite(p[k])) return 1;
  }
  if (!(p[0] > 0 && p[1] > 0 && p[2] > 0 && p[4] > 0 && p[5] > 0 && p[3] >= 0)) return 1;
  if (!(p[3] < 1.0)) return 1;  // subcritical only
  const double theta = p[3], omega = p[4], h = p[5];
  SimRng rng(seed);
  std::vector<double> vx, vy, vt;
  std::vector<int64_t> par;  // -1 immigrant, else creation index
  const double area = (window[1] - window[0]) * (window[3] - window[2]);
  const long imm = rng.poisson(rate * area * window[4]);
  for (long i = 0; i < imm; ++i) {
    vx.push_back(rng.uab(window[0], window[1]));
    vy.push_back(rng.uab(window[2], window[3]));
    vt.push_back(rng.uab(0.0, window[4]));
    par.push_back(-1);
  }
  for (size_t i = 0; i < vt.size(); ++i) {  // breadth-first cascade
    const long kids = rng.poisson(theta);
    for (long c = 0; c < kids; ++c) {
      const double dt = rng.expo(omega);
      const double dx = h * rng.gauss();
      const double dy = h * rng.gauss();
      const double ct = vt[i] + dt;
      if (ct >= window[4]) continue;
      vx.push_back(vx[i] + dx);
      vy.push_back(vy[i] + dy);
      vt.push_back(ct);
      par.push_back(static_cast<int64_t>(i));
    }
  }
  const int64_t n = static_cast<int64_t>(vt.size());
  *count = n;
  if (n == 0) return 2;
  const auto ord = time_order(vt);
  std::vector<int64_t> pos(n);
  for (int64_t i = 0; i < n; ++i) pos[ord[i]] = i;
  const int64_t m = std::min(n, capacity);
  for (int64_t i = 0; i < m; ++i) {
    const int64_t src = ord[i];
    if (x) x[i] = vx[src];
    if (y) y[i] = vy[src];
    if (t) t[i] = vt[src];
    if (parent) parent[i] = par[src] < 0 ? 0 : static_cast<int>(pos[par[src]]) + 1;
  }
  return 0;
}
