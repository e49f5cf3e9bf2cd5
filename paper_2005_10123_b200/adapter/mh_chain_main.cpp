// MH-chain driver for BASELINE config 5: runs the reference's adaptive
// Metropolis-Hastings sampler (hawkes::runChain, proj/src/sampler.cpp:134-175,
// compiled verbatim) on synthetic data, with hawkes::logLikelihood provided
// either by the reference CPU engine (likelihood.cpp) or by the B200 adapter
// -- the same source, linked two ways (adapter/Makefile).
//
// usage: mh_chain_* [--n N] [--data c2|cloud] [--iters K] [--burnin B]
//                   [--seed S] [--threads T] [--lanes L] [--draws-out FILE]
// Prints one JSON line.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>

#include "sthawkes/likelihood.hpp"
#include "sthawkes/rng.hpp"
#include "sthawkes/sampler.hpp"
#include "sthawkes/simulate.hpp"

using namespace hawkes;

namespace {

EventSet makeData(const std::string& kind, Index n) {
  if (kind == "cloud") {
    Rng rng(static_cast<std::uint64_t>(n));
    return generateBenchmarkCloud(n, SimWindow{0, 15, 0, 15, 4750}, rng);
  }
  // C2: DC-shaped cluster process, first n events in time
  Params truth;
  truth.mu0 = 1.0;
  truth.tauX = 1.6;
  truth.tauT = 14.0;
  truth.theta = 0.344;
  truth.omega = 1440.0;
  truth.h = 0.0695;
  Rng rng(2005);
  const SimTruth sim = simulateClusterProcess(truth, SimWindow{0, 15, 0, 15, 4750}, 0.053217, rng);
  const Index m = std::min<Index>(n, sim.events.size());
  Eigen::ArrayXd x(m), y(m), t(m);
  for (Index i = 0; i < m; ++i) {
    x[i] = sim.events.xs()[i];
    y[i] = sim.events.ys()[i];
    t[i] = sim.events.ts()[i];
  }
  return EventSet(std::move(x), std::move(y), std::move(t));
}

std::uint64_t fnv1a(const void* p, size_t bytes, std::uint64_t h = 1469598103934665603ull) {
  const unsigned char* c = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < bytes; ++i) {
    h ^= c[i];
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace

int main(int argc, char** argv) {
  Index n = 85000;
  std::string data = "c2", drawsOut, impl = STHK_DRIVER_IMPL;
  long iters = 100, burn = 10;
  std::uint64_t seed = 1;
  int threads = 1, lanes = 1;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string a = argv[i], v = argv[i + 1];
    if (a == "--n") n = std::stol(v);
    else if (a == "--data") data = v;
    else if (a == "--iters") iters = std::stol(v);
    else if (a == "--burnin") burn = std::stol(v);
    else if (a == "--seed") seed = std::stoull(v);
    else if (a == "--threads") threads = std::stoi(v);
    else if (a == "--lanes") lanes = std::stoi(v);
    else if (a == "--draws-out") drawsOut = v;
  }
  if (threads == 0) threads = static_cast<int>(std::thread::hardware_concurrency());
  const EventSet events = makeData(data, n);
  SamplerConfig cfg;
  cfg.iterations = iters;
  cfg.burnIn = burn < iters ? burn : iters - 1;
  cfg.seed = seed;
  if (threads > 1 && lanes > 1) cfg.backend = Backend::threadedVectorized(threads, lanes);
  else if (threads > 1) cfg.backend = Backend::threaded(threads);
  else if (lanes > 1) cfg.backend = Backend::vectorized(lanes);
  const PriorSpec priors;

  {
    // One-time process setup outside the timed region (for the B200 engine:
    // CUDA context, module loading): a 2-event evaluation, so the chain's
    // own event upload and every per-iteration cost stay timed.
    Eigen::ArrayXd tt(2);
    tt[0] = 0.5;
    tt[1] = 1.0;
    const EventSet tiny(Eigen::ArrayXd::Zero(2), Eigen::ArrayXd::Zero(2), tt, 1.0);
    (void)logLikelihood(tiny, Params{}, cfg.backend);
  }
  const auto t0 = std::chrono::steady_clock::now();
  const Chain chain = runChain(events, priors, cfg);
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

  long acc[4] = {0, 0, 0, 0}, prop[4] = {0, 0, 0, 0};
  for (long i = 0; i < iters; ++i) {
    prop[chain.scannedCoord[i]] += 1;
    acc[chain.scannedCoord[i]] += chain.accepted[i];
  }
  std::vector<double> draws(static_cast<size_t>(iters) * 4);
  for (long i = 0; i < iters; ++i) {
    for (int d = 0; d < 4; ++d) draws[static_cast<size_t>(i) * 4 + d] = chain.draws(i, d);
  }
  const std::uint64_t hd = fnv1a(draws.data(), draws.size() * sizeof(double));
  const std::uint64_t hl = fnv1a(chain.logPost.data(), sizeof(double) * iters);
  if (!drawsOut.empty()) {
    FILE* f = std::fopen(drawsOut.c_str(), "wb");
    if (f) {
      std::fwrite(draws.data(), sizeof(double), draws.size(), f);
      std::fwrite(chain.logPost.data(), sizeof(double), static_cast<size_t>(iters), f);
      std::fclose(f);
    }
  }
  std::printf(
      "{\"impl\": \"%s\", \"n\": %ld, \"data\": \"%s\", \"iterations\": %ld, \"burn_in\": %ld, "
      "\"seed\": %llu, \"backend\": \"%s\", \"seconds\": %.6f, \"s_per_iter\": %.9f, "
      "\"accepted\": [%ld, %ld, %ld, %ld], \"proposed\": [%ld, %ld, %ld, %ld], "
      "\"final_state\": [%.17g, %.17g, %.17g, %.17g], \"final_logpost\": %.17g, "
      "\"draws_fnv1a\": \"%016llx\", \"logpost_fnv1a\": \"%016llx\"}\n",
      impl.c_str(), static_cast<long>(events.size()), data.c_str(), iters, cfg.burnIn,
      static_cast<unsigned long long>(seed), cfg.backend.label().c_str(), sec, sec / iters,
      acc[0], acc[1], acc[2], acc[3], prop[0], prop[1], prop[2], prop[3], chain.draws(iters - 1, 0),
      chain.draws(iters - 1, 1), chain.draws(iters - 1, 2), chain.draws(iters - 1, 3),
      chain.logPost[iters - 1], static_cast<unsigned long long>(hd),
      static_cast<unsigned long long>(hl));
  return 0;
}
