// hawkes::logLikelihood / logLikelihoodBatch / excitationProbabilities /
// posteriorExcitation over the sthk C ABI.
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
// Linked in place of likelihood.cpp; excitationProbabilities and
// posteriorExcitation here take precedence over the reference's (whose
// excitation.o is linked with those two symbols weakened, for thinIndices).
// Excitation semantics: proj/src/excitation.cpp:13-130.
//
// State: one process-wide engine on the devices in $STHK_DEVICES (default
// "0"), created on first use. The device copy of the events is reused only
// for a set whose size, windowEnd and full contents equal the cached host
// copy -- the reference API is stateless, so an EventSet
// destroyed and rebuilt at the same heap addresses with different data must
// never see the old set's results. The full comparison (3 x N doubles,
// parallel over the host cores) of a set at the cached addresses runs while
// the device evaluates on the cached copy; on a mismatch the result is
// discarded, the set reloaded and the evaluation repeated. A set at other
// addresses is compared before anything is enqueued.
// STHK_ADAPTER_FAST_CHECK=1 (opt-in) trusts the cached addresses after a
// sampled check (first, last and 509 spread indices): faster MH iterations,
// but it can miss a rebuilt set that differs only at unsampled indices.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <fstream>

#include "sthawkes/excitation.hpp"
#include "sthawkes_b200.hpp"
#include "sthk.h"

namespace hawkes {

namespace {

// Exact content comparison of an EventSet against the adapter's host copy,
// split over a small persistent team of host threads (the 3 x N doubles are
// compared in 64 KB blocks). Workers spin briefly between calls -- MH
// iterations arrive every few tens of microseconds -- then sleep.
class CompareTeam {
 public:
  CompareTeam() {
    const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    const int workers = static_cast<int>(std::min(7u, hc > 2 ? hc / 2 - 1 : 0u));
    for (int w = 0; w < workers; ++w) th_.emplace_back([this, w] { loop(w + 1); });
  }
  ~CompareTeam() {
    {
      std::lock_guard<std::mutex> l(m_);
      stop_ = true;
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  bool equal(const double* const* a, const double* const* b, int64_t n) {
    a_ = a;
    b_ = b;
    n_ = n;
    nb_ = (n + kBlock - 1) / kBlock;
    diff_.store(0);
    const int team = static_cast<int>(th_.size()) + 1;
    if (3 * nb_ < 2 * team || th_.empty()) {
      work(0, 1);
      return diff_.load() == 0;
    }
    pending_.store(static_cast<int>(th_.size()));
    {
      std::lock_guard<std::mutex> l(m_);
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    work(0, team);
    while (pending_.load(std::memory_order_acquire) != 0) std::this_thread::yield();
    return diff_.load() == 0;
  }

 private:
  static constexpr int64_t kBlock = 8192;
  void work(int w, int team) {
    int d = 0;
    for (int64_t k = w; k < 3 * nb_; k += team) {
      const int64_t arr = k / nb_, b0 = (k % nb_) * kBlock;
      const int64_t len = std::min(kBlock, n_ - b0);
      d |= std::memcmp(a_[arr] + b0, b_[arr] + b0, sizeof(double) * static_cast<size_t>(len)) != 0;
    }
    if (d) diff_.store(1);
  }
  void loop(int w) {
    uint64_t seen = 0;
    for (;;) {
      int spins = 0;
      while (gen_.load(std::memory_order_acquire) == seen && spins < 200000) ++spins;
      if (gen_.load(std::memory_order_acquire) == seen) {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return gen_.load() != seen; });
      }
      seen = gen_.load();
      if (stop_) return;
      work(w, static_cast<int>(th_.size()) + 1);
      pending_.fetch_sub(1, std::memory_order_release);
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_;
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> pending_{0}, diff_{0};
  bool stop_ = false;
  const double* const* a_ = nullptr;
  const double* const* b_ = nullptr;
  int64_t n_ = 0, nb_ = 0;
};

struct AdapterEngine {
  std::mutex mu;
  sthk_engine* h = nullptr;
  const double* px = nullptr;
  const double* py = nullptr;
  const double* pt = nullptr;
  Index n = -1;
  double windowEnd = 0;
  std::vector<double> cx, cy, ct;  // host copy of the cached set
  bool fast_check = false;
  std::unique_ptr<CompareTeam> team = std::make_unique<CompareTeam>();

  AdapterEngine() {
    std::vector<int> devs;
    const char* env = std::getenv("STHK_DEVICES");
    std::stringstream ss(env && *env ? env : "0");
    std::string tok;
    while (std::getline(ss, tok, ',')) devs.push_back(std::stoi(tok));
    const char* fc = std::getenv("STHK_ADAPTER_FAST_CHECK");
    fast_check = fc && *fc == '1';
    if (sthk_create(devs.data(), static_cast<int>(devs.size()), &h) != STHK_OK) {
      throw std::runtime_error(std::string("sthk_create: ") + sthk_last_error(nullptr));
    }
    // STHK_SWEEP_CACHE=0: every call a full evaluation (timing harnesses)
    const char* sc = std::getenv("STHK_SWEEP_CACHE");
    if (sc && *sc == '0') sthk_set_background_cache(h, 0);
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

  // Makes the device hold `ev`. Returns true when the cached copy is reused
  // on the strength of the set's addresses alone: the caller must confirm
  // with contentEqual() before trusting the result.
  bool ensureLoaded(const EventSet& ev) {
    const Index m = ev.size();
    const double* x = ev.xs().data();
    const double* y = ev.ys().data();
    const double* t = ev.ts().data();
    if (m == n && ev.windowEnd() == windowEnd) {
      const bool same_ptrs = x == px && y == py && t == pt;
      if (same_ptrs && fast_check && sampled_equal(x, y, t, m)) return false;
      if (same_ptrs) return true;
      if (contentEqual(ev)) {
        px = x;  // same data at new addresses: keep the device copy
        py = y;
        pt = t;
        return false;
      }
    }
    reload(ev);
    return false;
  }

  // Exact: every coordinate of every event, over the host cores.
  bool contentEqual(const EventSet& ev) const {
    const Index m = ev.size();
    if (m != n) return false;
    const double* src[3] = {ev.xs().data(), ev.ys().data(), ev.ts().data()};
    const double* mine[3] = {cx.data(), cy.data(), ct.data()};
    return team->equal(src, mine, static_cast<int64_t>(m));
  }

  void reload(const EventSet& ev) {
    const Index m = ev.size();
    const double* x = ev.xs().data();
    const double* y = ev.ys().data();
    const double* t = ev.ts().data();
    n = -1;  // a failed load leaves the engine without events
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

  bool sampled_equal(const double* x, const double* y, const double* t, Index m) const {
    auto same = [&](Index i) { return x[i] == cx[i] && y[i] == cy[i] && t[i] == ct[i]; };
    if (!same(0) || !same(m - 1)) return false;
    const uint64_t mm = static_cast<uint64_t>(m);
    for (uint64_t k = 1; k <= 509; ++k) {
      if (!same(static_cast<Index>((k * 0x9E3779B97F4A7C15ULL) % mm))) return false;
    }
    return true;
  }

  void setParams(const Params& p) {
    const double v[6] = {p.mu0, p.tauX, p.tauT, p.theta, p.omega, p.h};
    check(sthk_set_params(h, v));
  }

  // One evaluation of `ev` at the current params: enqueued on the cached
  // copy while the host confirms the contents; redone after a reload on a
  // mismatch. per_event (nullable, length n) as sthk_result.
  void evaluate(const EventSet& ev, bool grad, double* ll, int* ok, double* g, double* pe) {
    const bool verify = ensureLoaded(ev);
    check(sthk_enqueue(h, grad ? 1 : 0, pe != nullptr ? 1 : 0));
    if (verify && !contentEqual(ev)) {
      check(sthk_result(h, nullptr, nullptr, nullptr, nullptr));  // (discarded)
      reload(ev);
      check(sthk_enqueue(h, grad ? 1 : 0, pe != nullptr ? 1 : 0));
    }
    check(sthk_result(h, ll, ok, g, pe));
  }

  // Contents confirmed before anything is enqueued (batch / excitation paths).
  void ensureLoadedExact(const EventSet& ev) {
    if (ensureLoaded(ev) && !contentEqual(ev)) reload(ev);
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
  e.setParams(params);
  LikelihoodResult r;
  if (keepPerEvent) r.perEvent.setZero(events.size());
  double ll = 0;
  int ok = 0;
  e.evaluate(events, false, &ll, &ok, nullptr, keepPerEvent ? r.perEvent.data() : nullptr);
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
  e.setParams(params);
  LikelihoodGradient out;
  if (keepPerEvent) out.result.perEvent.setZero(events.size());
  double ll = 0;
  int ok = 0;
  e.evaluate(events, true, &ll, &ok, out.grad.data(),
             keepPerEvent ? out.result.perEvent.data() : nullptr);
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
  if (!keepPerEvent) {
    // one engine call: entries validated in order (the reference's message
    // for the first invalid one), evaluated grouped by (tauX, tauT, omega, h)
    // so the exact sweep caches are shared across entries
    for (size_t i = 0; i < paramsList.size(); ++i) {
      try {
        paramsList[i].validate();
      } catch (const std::exception& ex) {
        throw std::invalid_argument("logLikelihoodBatch: entry " + std::to_string(i) + ": " +
                                    ex.what());
      }
    }
    backend.validate();
    AdapterEngine& e = engine();
    std::lock_guard<std::mutex> lock(e.mu);
    e.ensureLoadedExact(events);
    const size_t P = paramsList.size();
    std::vector<double> pv(6 * P), ll(P);
    std::vector<int> ok(P);
    for (size_t i = 0; i < P; ++i) {
      const Params& p = paramsList[i];
      const double v[6] = {p.mu0, p.tauX, p.tauT, p.theta, p.omega, p.h};
      std::copy(v, v + 6, pv.begin() + static_cast<std::ptrdiff_t>(6 * i));
    }
    e.check(sthk_loglik_batch(e.h, pv.data(), static_cast<int64_t>(P), ll.data(), ok.data(),
                              nullptr));
    for (size_t i = 0; i < P; ++i) {
      LikelihoodResult r;
      r.valid = ok[i] != 0;
      r.logLik = r.valid ? ll[i] : -std::numeric_limits<double>::infinity();
      results.push_back(std::move(r));
    }
    return results;
  }
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

ExcitationVector excitationProbabilities(const EventSet& events, const Params& params,
                                         const Backend& backend) {
  params.validate();
  backend.validate();
  AdapterEngine& e = engine();
  std::lock_guard<std::mutex> lock(e.mu);
  e.ensureLoadedExact(events);
  e.setParams(params);
  const Index n = events.size();
  ExcitationVector out;
  out.pi.resize(n);
  out.mu.resize(n);
  out.xi.resize(n);
  const int rc = sthk_excitation(e.h, out.mu.data(), out.xi.data(), out.pi.data());
  if (rc == STHK_ERANGE) throw std::runtime_error(sthk_last_error(e.h));
  e.check(rc);
  return out;
}

// posteriorExcitation (excitation.hpp:43-47) on the batched device path. The
// thinning is the reference's own thinIndices (excitation.cpp, linked from
// the verbatim build with this file's two functions taking precedence); the
// kept draws go to the engine in batches (sthk_excitation_batch: one
// background sweep for draws sharing tauX, tauT, pi summed on the device in
// draw order). Errors surface at the same draw, after the same dump lines,
// with the same messages as the reference's draw-by-draw loop
// (excitation.cpp:72-130).
PosteriorExcitation posteriorExcitation(const EventSet& events, const std::vector<Params>& draws,
                                        const Backend& backend,
                                        const PosteriorExcitationOptions& options) {
  if (draws.empty()) throw std::invalid_argument("posteriorExcitation: no draws");
  if (options.thinTo < 1) {
    throw std::invalid_argument("posteriorExcitation: thinTo must be >= 1");
  }
  const Index n = events.size();
  PosteriorExcitation out;
  out.drawIndices = thinIndices(static_cast<Index>(draws.size()), options.thinTo);
  const Index kept = static_cast<Index>(out.drawIndices.size());
  const bool retain = kept * n <= options.memoryCapEntries;
  if (retain) out.perDraw.setZero(kept, n);
  out.meanPi.setZero(n);

  std::ofstream dump;
  if (options.dumpPath) {
    dump.open(*options.dumpPath);
    if (!dump) {
      throw std::runtime_error("posteriorExcitation: cannot open dump file " + *options.dumpPath);
    }
    dump << "# sthawkes pi draws v1, events=" << n << "\n";
  }
  // the loop ends at the first kept draw the reference's
  // excitationProbabilities would reject (params, backend)
  Index stop = kept;
  std::string stop_msg;
  for (Index j = 0; j < kept && stop == kept; ++j) {
    const Index d = out.drawIndices[static_cast<size_t>(j)];
    try {
      draws[static_cast<size_t>(d)].validate();
      backend.validate();
    } catch (const std::exception& err) {
      stop = j;
      stop_msg = "posteriorExcitation: draw " + std::to_string(d) + ": " + err.what();
    }
  }
  const bool rows_needed = retain || dump.is_open();
  const Index step =
      rows_needed ? std::max<Index>(1, std::min<Index>(std::max<Index>(stop, 1), 10000000 / n))
                  : std::max<Index>(stop, 1);
  std::vector<double> rows(rows_needed ? static_cast<size_t>(step * n) : 0);
  std::vector<double> pv;
  std::string line;
  char num[40];
  AdapterEngine& e = engine();
  for (Index j0 = 0; j0 < stop; j0 += step) {
    const Index j1 = std::min(stop, j0 + step);
    pv.assign(static_cast<size_t>(6 * (j1 - j0)), 0.0);
    for (Index j = j0; j < j1; ++j) {
      const Params& p = draws[static_cast<size_t>(out.drawIndices[static_cast<size_t>(j)])];
      const double v[6] = {p.mu0, p.tauX, p.tauT, p.theta, p.omega, p.h};
      std::copy(v, v + 6, pv.begin() + 6 * (j - j0));
    }
    int64_t bad = -1;
    {
      std::lock_guard<std::mutex> lock(e.mu);
      e.ensureLoadedExact(events);
      const int rc = sthk_excitation_batch(e.h, pv.data(), j1 - j0, out.meanPi.data(),
                                           rows_needed ? rows.data() : nullptr, &bad);
      if (rc != STHK_ERANGE) e.check(rc);
    }
    const Index done = bad < 0 ? j1 : j0 + static_cast<Index>(bad);
    for (Index j = j0; j < done; ++j) {
      const double* pi = rows.data() + (j - j0) * n;
      if (retain) {
        for (Index i = 0; i < n; ++i) out.perDraw(j, i) = pi[i];
      }
      if (dump.is_open()) {
        line = std::to_string(out.drawIndices[static_cast<size_t>(j)]);
        for (Index i = 0; i < n; ++i) {
          std::snprintf(num, sizeof num, "\t%.17g", pi[i]);
          line += num;
        }
        line += '\n';
        dump << line;
      }
    }
    if (bad >= 0) {
      throw std::runtime_error(
          "posteriorExcitation: draw " +
          std::to_string(out.drawIndices[static_cast<size_t>(j0 + bad)]) +
          ": excitationProbabilities: per-event rate underflowed to zero");
    }
  }
  if (!stop_msg.empty()) throw std::runtime_error(stop_msg);
  out.meanPi /= static_cast<double>(kept);
  if (dump.is_open() && !dump) {
    throw std::runtime_error("posteriorExcitation: failed writing dump file");
  }
  return out;
}

}  // namespace hawkes
