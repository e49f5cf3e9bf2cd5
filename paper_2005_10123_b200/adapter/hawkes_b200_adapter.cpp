// hawkes::logLikelihood / logLikelihoodBatch over the sthk C ABI.
//
// Behaviour kept from the reference (proj/src/likelihood.cpp:10-75):
//   * params.validate() and backend.validate() run first and throw
//     std::invalid_argument exactly as before (test_likelihood.cpp:148-154);
//     the Backend is otherwise ignored -- the B200 engine replaces the CPU
//     backends.
//   * valid=false / logLik=-inf on a degenerate rate, perEvent sized N only
//     when requested, 0 on degenerate rows.
//   * logLikelihoodBatch rethrows "logLikelihoodBatch: entry i: ...".
// Engine errors other than invalid arguments become std::runtime_error.
//
// State: one process-wide engine on the devices in $STHK_DEVICES (default
// "0"), created on first use. The device copy of the events is cached; a call
// reuses it only if the EventSet's data are byte-identical to the cached
// copy (pointer, size and windowEnd first, then a memcmp), so a new set at a
// recycled address can never be confused with the old one.
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "sthawkes_b200.hpp"
#include "sthk.h"

namespace hawkes {

namespace {

struct AdapterEngine {
  std::mutex mu;
  sthk_engine* h = nullptr;
  const double* px = nullptr;
  const double* py = nullptr;
  const double* pt = nullptr;
  Index n = -1;
  double windowEnd = 0;
  std::vector<double> cx, cy, ct;  // host copy of the cached set

  AdapterEngine() {
    std::vector<int> devs;
    const char* env = std::getenv("STHK_DEVICES");
    std::stringstream ss(env && *env ? env : "0");
    std::string tok;
    while (std::getline(ss, tok, ',')) devs.push_back(std::stoi(tok));
    if (sthk_create(devs.data(), static_cast<int>(devs.size()), &h) != STHK_OK) {
      throw std::runtime_error(std::string("sthk_create: ") + sthk_last_error(nullptr));
    }
  }
  ~AdapterEngine() {
    if (h) sthk_destroy(h);
  }

  void check(int rc) {
    if (rc == STHK_OK) return;
    const std::string msg = sthk_last_error(h);
    if (rc == STHK_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("B200 engine: " + msg);
  }

  void ensureLoaded(const EventSet& ev) {
    const Index m = ev.size();
    const double* x = ev.xs().data();
    const double* y = ev.ys().data();
    const double* t = ev.ts().data();
    const size_t bytes = sizeof(double) * static_cast<size_t>(m);
    if (m == n && x == px && y == py && t == pt && ev.windowEnd() == windowEnd &&
        std::memcmp(x, cx.data(), bytes) == 0 && std::memcmp(y, cy.data(), bytes) == 0 &&
        std::memcmp(t, ct.data(), bytes) == 0) {
      return;
    }
    check(sthk_load_events(h, x, y, t, m, ev.windowEnd()));
    px = x;
    py = y;
    pt = t;
    n = m;
    windowEnd = ev.windowEnd();
    cx.assign(x, x + m);
    cy.assign(y, y + m);
    ct.assign(t, t + m);
  }

  void setParams(const Params& p) {
    const double v[6] = {p.mu0, p.tauX, p.tauT, p.theta, p.omega, p.h};
    check(sthk_set_params(h, v));
  }
};

AdapterEngine& engine() {
  static AdapterEngine e;
  return e;
}

}  // namespace

LikelihoodResult logLikelihood(const EventSet& events, const Params& params,
                               const Backend& backend, bool keepPerEvent) {
  params.validate();
  backend.validate();
  AdapterEngine& e = engine();
  std::lock_guard<std::mutex> lock(e.mu);
  e.ensureLoaded(events);
  e.setParams(params);
  LikelihoodResult r;
  if (keepPerEvent) r.perEvent.setZero(events.size());
  double ll = 0;
  int ok = 0;
  e.check(sthk_loglik(e.h, &ll, &ok, keepPerEvent ? r.perEvent.data() : nullptr));
  r.valid = ok != 0;
  r.logLik = r.valid ? ll : -std::numeric_limits<double>::infinity();
  return r;
}

LikelihoodGradient logLikelihoodGradient(const EventSet& events, const Params& params,
                                         const Backend& backend, bool keepPerEvent) {
  params.validate();
  backend.validate();
  AdapterEngine& e = engine();
  std::lock_guard<std::mutex> lock(e.mu);
  e.ensureLoaded(events);
  e.setParams(params);
  LikelihoodGradient out;
  if (keepPerEvent) out.result.perEvent.setZero(events.size());
  double ll = 0;
  int ok = 0;
  e.check(sthk_loglik_grad(e.h, &ll, &ok, out.grad.data(),
                           keepPerEvent ? out.result.perEvent.data() : nullptr));
  out.result.valid = ok != 0;
  out.result.logLik = out.result.valid ? ll : -std::numeric_limits<double>::infinity();
  return out;
}

std::vector<LikelihoodResult> logLikelihoodBatch(const EventSet& events,
                                                 const std::vector<Params>& paramsList,
                                                 const Backend& backend, bool keepPerEvent) {
  if (paramsList.empty()) {
    throw std::invalid_argument("logLikelihoodBatch: empty parameter list");
  }
  std::vector<LikelihoodResult> results;
  results.reserve(paramsList.size());
  for (size_t i = 0; i < paramsList.size(); ++i) {
    try {
      results.push_back(logLikelihood(events, paramsList[i], backend, keepPerEvent));
    } catch (const std::exception& ex) {
      throw std::invalid_argument("logLikelihoodBatch: entry " + std::to_string(i) + ": " +
                                  ex.what());
    }
  }
  return results;
}

}  // namespace hawkes
