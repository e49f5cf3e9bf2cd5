// The reference's own timing harness (hawkes::timeLikelihood /
// formatTimingTable, proj/src/bench.cpp:15-88, compiled verbatim) driving
// hawkes::logLikelihood -- over the B200 adapter (timing_b200) or over the
// reference CPU likelihood.cpp (timing_ref_{v4,v3}). Same C2 data as
// bench.py. For the B200 build, set STHK_SWEEP_CACHE=0 to time full
// evaluations (with the caches on, repeated identical calls are finalize-only).
//
//   timing_<impl> [--n 85000] [--repeats 10] [--warmups 2] [--threads 0] [--lanes 8]
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "sthawkes/bench.hpp"
#include "sthawkes/likelihood.hpp"
#include "sthawkes/rng.hpp"
#include "sthawkes/simulate.hpp"

#ifndef STHK_DRIVER_IMPL
#define STHK_DRIVER_IMPL "b200"
#endif

using namespace hawkes;

int main(int argc, char** argv) {
  Index n = 85000;
  int repeats = 10, warmups = 2, threads = 0, lanes = 8;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string a = argv[i], v = argv[i + 1];
    if (a == "--n") n = std::stol(v);
    else if (a == "--repeats") repeats = std::stoi(v);
    else if (a == "--warmups") warmups = std::stoi(v);
    else if (a == "--threads") threads = std::stoi(v);
    else if (a == "--lanes") lanes = std::stoi(v);
  }
  if (threads == 0) threads = static_cast<int>(std::thread::hardware_concurrency());
  // C2: simulateClusterProcess(truth, {0,15,0,15,4750}, 0.053217, Rng(2005)),
  // first n events in time order
  Params truth;
  truth.mu0 = 1.0;
  truth.tauX = 1.6;
  truth.tauT = 14.0;
  truth.theta = 0.344;
  truth.omega = 1440.0;
  truth.h = 0.0695;
  Rng rng(2005);
  const SimTruth sim = simulateClusterProcess(truth, SimWindow{0, 15, 0, 15, 4750}, 0.053217, rng);
  const Index m = sim.events.size() < n ? sim.events.size() : n;
  Eigen::ArrayXd x(m), y(m), t(m);
  for (Index i = 0; i < m; ++i) {
    x[i] = sim.events.xs()[i];
    y[i] = sim.events.ys()[i];
    t[i] = sim.events.ts()[i];
  }
  const EventSet events(std::move(x), std::move(y), std::move(t));
  Params post;
  post.mu0 = 0.66;
  post.tauX = 1.6;
  post.tauT = 14.0;
  post.theta = 0.344;
  post.omega = 1440.0;
  post.h = 0.0695;
  const Backend backend = std::string(STHK_DRIVER_IMPL) == "b200"
                              ? Backend::serial()  // (ignored by the B200 adapter)
                              : Backend::threadedVectorized(threads, lanes);
  std::vector<TimingRecord> recs;
  recs.push_back(timeLikelihood(events, post, backend, repeats, warmups));
  recs.back().backend = std::string(STHK_DRIVER_IMPL) + ":" + recs.back().backend;
  std::printf("%s", formatTimingTable(recs).c_str());
  const LikelihoodResult r = logLikelihood(events, post, backend);
  std::printf("{\"impl\": \"%s\", \"n\": %lld, \"median_s\": %.9f, \"min_s\": %.9f, "
              "\"repeats\": %d, \"loglik\": %.17g, \"hardware\": \"%s\"}\n",
              STHK_DRIVER_IMPL, static_cast<long long>(m), recs[0].medianSeconds,
              recs[0].minSeconds, repeats, r.logLik, recs[0].hardware.c_str());
  return 0;
}
