// Drop-in B200 backend for the reference's likelihood interface.
//
// Link hawkes_b200_adapter.o (+ libsthk.so) IN PLACE OF the reference's
// src/likelihood.cpp: it defines, with identical signatures,
//   hawkes::logLikelihood       (proj/include/sthawkes/likelihood.hpp:24-26)
//   hawkes::logLikelihoodBatch  (proj/include/sthawkes/likelihood.hpp:28-31)
// so the reference's sampler.cpp (MH driver), bench.cpp and tests link
// against the GPU engine unmodified. It adds the gradient the reference lacks.
#ifndef STHAWKES_B200_HPP
#define STHAWKES_B200_HPP

#include <array>

#include "sthawkes/likelihood.hpp"

namespace hawkes {

struct LikelihoodGradient {
  LikelihoodResult result;
  // d logLik / d params in Params order (mu0, tauX, tauT, theta, omega, h);
  // NaN when result.valid is false.
  std::array<double, 6> grad{};
};

LikelihoodGradient logLikelihoodGradient(const EventSet& events, const Params& params,
                                         const Backend& backend, bool keepPerEvent = false);

}  // namespace hawkes

#endif  // STHAWKES_B200_HPP
