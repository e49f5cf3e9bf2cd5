// Device-side building blocks of the B200 Hawkes engine: the FP64 exp used on
// every pair, the constants it needs, and the TMA (cp.async.bulk) / mbarrier
// helpers that stage source tiles into shared memory.
//
// Why a hand-written exp: the pair kernels are bound by the FP64 pipe
// (SURVEY.md §8 d2-d3), and the exps are the largest share of the FP64
// instructions. CUDA's double exp costs 14 DFMA + 1 DADD on sm_100a; this one
// costs 7 FP64 instructions (3 DADD for an exact reduction, 3 polynomial,
// 1 reconstruction): the caller folds 2048/ln2 into its exponent constants,
// 2^(j/2048) comes from a 2048-entry (16 KB) shared-memory table and the 2^m
// scaling is a single integer IMAD on the table entry's hi word.
//
// Semantics vs the reference (pack.hpp:86-154, laneExp at pack.hpp:157):
//   * accuracy: table entries correctly rounded, the reduction is exact,
//     polynomial max abs error 5.9e-18 on |u| <= 1/2 (tools/gen_exp_table.py
//     --check) -> about 1 ulp worst, the same class as the reference's Pack
//     exp (<= 2 ulp, test_pack.cpp:21-46); folding 2048/ln2 into the
//     exponent adds one rounding of the argument (pinned by
//     tests/test_parity_gpu.py::test_exp_l_accuracy);
//   * underflow: returns exactly +0 when k = rint(2048 x / ln2) < -2093056,
//     i.e. for every x < -708.40 (and -inf). The reference's Pack exp flushes
//     x < -708 to 0 (pack.hpp:124); libm returns subnormals down to -745.13.
//     The difference is below 3.3e-308 per pair (SURVEY.md §7 "lane-exp flush").
//   * domain: callers pass x <= 0. Positive x (masked-out trigger lanes) give
//     garbage that the caller discards with a select, never a multiply.
#pragma once

#include <cstdint>

#include "sthk_exp_table.cuh"

namespace sthk {

// kExpL = 2048/ln2 (callers pass exponents pre-multiplied by it: "L units"),
// the polynomial kE1..kE3 and the 2^(j/2048) table come from
// tools/gen_exp_table.py (200-bit arithmetic).
constexpr double kRoundMagic = 0x1.8p52;
// Smallest k = rint(x) whose 2^(k/2048) is a normal double is -1022*2048.
constexpr int kMinK = -1022 * kExpTableSize;
// bits(1.5*2^52) + kMinK: rounded-t bit patterns below this flush to +0.
constexpr long long kFlushBits = 0x4338000000000000LL + kMinK;
// Exponents (L units) above this never flush: kernels use the unchecked exp
// for stages whose exponent lower bound clears it (-706.7 in natural units).
constexpr double kSafeExpL = -2088000.0;
constexpr int kExpMask = kExpTableSize - 1;

// exp(x / kExpL) for an exponent x given in L units (x <= 0), with the 2048
// table entries above in shared memory. 7 FP64 instructions: 3 DADD for the
// exact reduction x = k + u (|u| <= 1/2), 3 for the polynomial, 1 to
// reconstruct. CHECK selects the flush of k < kMinK (and -inf) to +0; callers
// pass CHECK=false only when the exponent is provably >= kSafeExpL.
template <bool CHECK>
__device__ __forceinline__ double exp_l(double x, const uint2* __restrict__ tab) {
  const double t = x + kRoundMagic;  // low word = k = rint(x)
  const double kd = t - kRoundMagic;
  const double u = x - kd;           // exact
  double q = fma(kE3, u, kE2);
  q = fma(q, u, kE1);
  const double p = q * u;            // expm1(u ln2/2048)
  const long long tb = __double_as_longlong(t);
  const int k = static_cast<int>(tb);
  const uint2 tj = tab[k & kExpMask];
  const double ts =
      __hiloint2double(static_cast<int>(tj.y) + (k << kExpShift), static_cast<int>(tj.x));
  const double res = fma(ts, p, ts);
  if constexpr (CHECK) return tb < kFlushBits ? 0.0 : res;
  return res;
}

// N independent exp_l evaluations written in lockstep (stage by stage), so
// the dependent 8-instruction chains are interleaved in program order and the
// FP64 pipe's latency is covered by N-way ILP even at low occupancy.
#ifndef STHK_EXP_CVT
#define STHK_EXP_CVT 0
#endif
template <bool CHECK, int N>
__device__ __forceinline__ void exp_l_batch(const double (&x)[N], double (&out)[N],
                                            const uint2* __restrict__ tab) {
#if STHK_EXP_CVT
  // k = rint(x) by F2I.F64 (round to nearest even, exactly as the magic-number
  // rounding below) and kd = k by I2F.F64: both on the conversion pipe, so
  // the exp costs 5 FP64-pipe instructions instead of 7; bitwise identical.
  int k[N];
  double u[N], q[N];
#pragma unroll
  for (int i = 0; i < N; ++i) k[i] = __double2int_rn(x[i]);
#pragma unroll
  for (int i = 0; i < N; ++i) u[i] = x[i] - static_cast<double>(k[i]);
#pragma unroll
  for (int i = 0; i < N; ++i) q[i] = fma(kE3, u[i], kE2);
#pragma unroll
  for (int i = 0; i < N; ++i) q[i] = fma(q[i], u[i], kE1);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double p = q[i] * u[i];
    const uint2 tj = tab[k[i] & kExpMask];
    const double ts = __hiloint2double(static_cast<int>(tj.y) + (k[i] << kExpShift),
                                       static_cast<int>(tj.x));
    const double res = fma(ts, p, ts);
    out[i] = CHECK ? (k[i] < kMinK ? 0.0 : res) : res;
  }
#else
  double t[N], u[N], q[N];
#pragma unroll
  for (int i = 0; i < N; ++i) t[i] = x[i] + kRoundMagic;
#pragma unroll
  for (int i = 0; i < N; ++i) u[i] = x[i] - (t[i] - kRoundMagic);
#pragma unroll
  for (int i = 0; i < N; ++i) q[i] = fma(kE3, u[i], kE2);
#pragma unroll
  for (int i = 0; i < N; ++i) q[i] = fma(q[i], u[i], kE1);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double p = q[i] * u[i];
    const long long tb = __double_as_longlong(t[i]);
    const int k = static_cast<int>(tb);
    const uint2 tj = tab[k & kExpMask];
    const double ts = __hiloint2double(static_cast<int>(tj.y) + (k << kExpShift),
                                       static_cast<int>(tj.x));
    const double res = fma(ts, p, ts);
    out[i] = CHECK ? (tb < kFlushBits ? 0.0 : res) : res;
  }
#endif
}

// ---------------------------------------------------------------------------
// Deterministic fixed-point accumulation.
//
// Partial sums (always >= 0: every summand is e, e*r^2, e*dt^2, e*dt with
// dt > 0) are converted to a two-word fixed-point number -- hi in units of
// 2^-40, lo holding the exact remainder in units of 2^-80 -- and added with
// 64-bit integer atomics. Integer addition is associative, so the totals are
// bitwise independent of the order in which CTAs, devices or ranks add their
// contributions; the representation error is <= 2^-81 per conversion (far
// below the rounding of the double partial itself). Callers normalise each
// sum to O(1) per pair first (|total| < 2^23).
// ---------------------------------------------------------------------------
constexpr double kFxHi = 0x1p40;
constexpr double kFxHiInv = 0x1p-40;
constexpr double kFxLo = 0x1p80;
constexpr double kFxLoInv = 0x1p-80;

__device__ __forceinline__ void fx_add(unsigned long long* hi, unsigned long long* lo, double v) {
  const long long h = __double2ll_rn(v * kFxHi);
  // exact: either v*2^40 >= 2^53 (already an integer, remainder 0) or
  // h*2^-40 is exact and within a factor 2 of v (Sterbenz)
  const double rem = fma(static_cast<double>(h), -kFxHiInv, v);
  const long long l = __double2ll_rn(rem * kFxLo);
  if (h != 0) atomicAdd(hi, static_cast<unsigned long long>(h));
  if (l != 0) atomicAdd(lo, static_cast<unsigned long long>(l));
}

__device__ __forceinline__ double fx_value(unsigned long long hi, unsigned long long lo) {
  long long H = static_cast<long long>(hi);
  long long L = static_cast<long long>(lo);
  const long long carry = L >> 40;  // floor(L / 2^40)
  H += carry;
  L -= carry * (1LL << 40);  // now 0 <= L < 2^40
  return fma(static_cast<double>(H), kFxHiInv, static_cast<double>(L) * kFxLoInv);
}

// ---------------------------------------------------------------------------
// TMA bulk copy (cp.async.bulk, SASS UBLKCP) + mbarrier helpers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Global -> shared bulk copy of `bytes` (multiple of 16, 16-byte aligned),
// completion signalled on `bar` as transaction bytes.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

}  // namespace sthk
