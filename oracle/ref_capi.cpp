// C entry points over the VERBATIM reference engine, compiled from
// /root/reference/proj sources into oracle/_ref/ (see oracle/Makefile).
// TEST / BASELINE INFRASTRUCTURE ONLY: imported by tests/, smoke() and the
// cpu_baseline / --impl reference legs of bench.py, never by the product.
//
// Wraps:
//   hawkes::logLikelihood        proj/src/likelihood.cpp:10-55
//   hawkes::timeLikelihood       proj/src/bench.cpp:15-55
//   hawkes::hardwareDescriptor   proj/src/bench.cpp:57-73
//   hawkes::generateBenchmarkCloud / simulateClusterProcess
//                                proj/src/simulate.cpp:10-95
//   hawkes::runChain             proj/src/sampler.cpp:134-175
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "sthawkes/bench.hpp"
#include "sthawkes/likelihood.hpp"
#include "sthawkes/rng.hpp"
#include "sthawkes/sampler.hpp"
#include "sthawkes/simulate.hpp"

using namespace hawkes;

namespace {

thread_local std::string g_err;

EventSet makeEvents(const double* x, const double* y, const double* t,
                    int64_t n, double windowEnd) {
  Eigen::ArrayXd ax(n), ay(n), at(n);
  for (int64_t i = 0; i < n; ++i) {
    ax[i] = x[i];
    ay[i] = y[i];
    at[i] = t[i];
  }
  return EventSet(std::move(ax), std::move(ay), std::move(at), windowEnd);
}

Params makeParams(const double* p) {
  Params q;
  q.mu0 = p[0];
  q.tauX = p[1];
  q.tauT = p[2];
  q.theta = p[3];
  q.omega = p[4];
  q.h = p[5];
  return q;
}

Backend makeBackend(int threads, int lanes) {
  if (threads <= 1 && lanes <= 1) return Backend::serial();
  if (threads <= 1) return Backend::vectorized(lanes);
  if (lanes <= 1) return Backend::threaded(threads);
  return Backend::threadedVectorized(threads, lanes);
}

int fail(const std::exception& e) {
  g_err = e.what();
  return dynamic_cast<const std::invalid_argument*>(&e) ? 1 : 5;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Status: 0 ok, 1 invalid argument, 5 other exception.
int ref_loglik(const double* x, const double* y, const double* t, int64_t n,
               double window_end, const double* params, int threads,
               int lanes, double* loglik, int* valid, double* per_event) {
  try {
    const EventSet ev = makeEvents(x, y, t, n, window_end);
    const LikelihoodResult r = logLikelihood(ev, makeParams(params),
                                             makeBackend(threads, lanes),
                                             per_event != nullptr);
    *loglik = r.logLik;
    *valid = r.valid ? 1 : 0;
    if (per_event) std::memcpy(per_event, r.perEvent.data(), sizeof(double) * n);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_time_loglik(const double* x, const double* y, const double* t,
                    int64_t n, double window_end, const double* params,
                    int threads, int lanes, int repeats, int warmups,
                    double* median_s, double* min_s) {
  try {
    const EventSet ev = makeEvents(x, y, t, n, window_end);
    const TimingRecord rec = timeLikelihood(
        ev, makeParams(params), makeBackend(threads, lanes), repeats, warmups);
    *median_s = rec.medianSeconds;
    *min_s = rec.minSeconds;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_hardware_descriptor(char* buf, int len) {
  const std::string s = hardwareDescriptor();
  std::snprintf(buf, static_cast<size_t>(len), "%s", s.c_str());
  return 0;
}

// window = {xmin, xmax, ymin, ymax, tEnd}. Writes n events, time-sorted.
int ref_sim_cloud(int64_t n, const double* window, uint64_t seed, double* x,
                  double* y, double* t, double* window_end) {
  try {
    Rng rng(seed);
    const SimWindow w{window[0], window[1], window[2], window[3], window[4]};
    const EventSet ev = generateBenchmarkCloud(n, w, rng);
    std::memcpy(x, ev.xs().data(), sizeof(double) * n);
    std::memcpy(y, ev.ys().data(), sizeof(double) * n);
    std::memcpy(t, ev.ts().data(), sizeof(double) * n);
    *window_end = ev.windowEnd();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Cluster simulation; writes min(count, capacity) events and parents
// (0 = immigrant, else 1-based parent index); *count = total simulated.
int ref_sim_cluster(const double* params, const double* window, double rate,
                    uint64_t seed, int64_t capacity, double* x, double* y,
                    double* t, int* parent, int64_t* count) {
  try {
    Rng rng(seed);
    const SimWindow w{window[0], window[1], window[2], window[3], window[4]};
    const SimTruth s = simulateClusterProcess(makeParams(params), w, rate, rng);
    const int64_t n = s.events.size();
    *count = n;
    const int64_t m = n < capacity ? n : capacity;
    std::memcpy(x, s.events.xs().data(), sizeof(double) * m);
    std::memcpy(y, s.events.ys().data(), sizeof(double) * m);
    std::memcpy(t, s.events.ts().data(), sizeof(double) * m);
    for (int64_t i = 0; i < m; ++i) parent[i] = s.parentIndex[i];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
