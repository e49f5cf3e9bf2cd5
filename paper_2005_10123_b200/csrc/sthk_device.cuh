// Device-side building blocks of the B200 Hawkes engine: the FP64 exp used on
// every pair, the constants it needs, and the TMA (cp.async.bulk) / mbarrier
// helpers that stage source tiles into shared memory.
//
// Why a hand-written exp: the pair kernels are bound by the FP64 pipe
// (SURVEY.md §8 d2-d3), and the two exps per pair are ~70% of the FP64
// instructions. CUDA's double exp costs 14 DFMA + 1 DADD on sm_100a; this one
// costs 10 FP64 instructions (2 rounding, 2 Cody-Waite, 5 polynomial, 1
// reconstruction) by moving 2^(j/64) into a 64-entry shared-memory table and
// the 2^m scaling onto the integer pipe.
//
// Semantics vs the reference (pack.hpp:86-154, laneExp at pack.hpp:157):
//   * accuracy: table entries correctly rounded, |reduction error| < 2^-60,
//     polynomial max abs error 1.4e-18 on |r| <= ln2/128 -> about 1 ulp worst,
//     the same class as the reference's Pack exp (<= 2 ulp, test_pack.cpp:21-46);
//   * underflow: returns exactly +0 when k = rint(64 x / ln2) < -65408, i.e.
//     for every x < -708.40 (and -inf). The reference's Pack exp flushes
//     x < -708 to 0 (pack.hpp:124); libm returns subnormals down to -745.13.
//     The difference is below 3.3e-308 per pair (SURVEY.md §7 "lane-exp flush").
//   * domain: callers pass x <= 0. Positive x (masked-out trigger lanes) give
//     garbage that the caller discards with a select, never a multiply.
#pragma once

#include <cstdint>

namespace sthk {

// 64/ln2, the 1.5*2^52 rounding constant, and ln2/64 split hi/lo.
constexpr double kExpL = 0x1.71547652b82fep+6;
constexpr double kRoundMagic = 0x1.8p52;
constexpr double kLn2By64Hi = 0x1.62e42fefa39efp-7;
constexpr double kLn2By64Lo = 0x1.abc9e3b39803fp-62;
// expm1(r) ~= r + c2 r^2 + c3 r^3 + c4 r^4 + c5 r^5 on |r| <= ln2/128
// (least-squares near-minimax fit in 150-bit arithmetic; max abs err 1.4e-18).
constexpr double kC2 = 0x1.fffffffffdb37p-2;
constexpr double kC3 = 0x1.55555555548b9p-3;
constexpr double kC4 = 0x1.555573f3a97b8p-5;
constexpr double kC5 = 0x1.111123d00afbbp-7;
// bits(1.5*2^52) + kMinK: t-bit patterns below this flush to +0.
constexpr long long kFlushBits = 0x4338000000000000LL - 65408LL;

// 2^(j/64), j = 0..63, correctly rounded (generated with mpmath, 200 bits).
__device__ __constant__ double kExpTable[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0,
    0x1.0874518759bc8p+0, 0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0,
    0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0, 0x1.172b83c7d517bp+0,
    0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0,
    0x1.2d285a6e4030bp+0, 0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0,
    0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0, 0x1.3dea64c123422p+0,
    0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0,
    0x1.56f4736b527dap+0, 0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0,
    0x1.6247eb03a5585p+0, 0x1.6623882552225p+0, 0x1.6a09e667f3bcdp+0,
    0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0,
    0x1.868d99b4492edp+0, 0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0,
    0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0, 0x1.9c49182a3f090p+0,
    0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0,
    0x1.bcc1e904bc1d2p+0, 0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0,
    0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0, 0x1.d5818dcfba487p+0,
    0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0,
    0x1.fa7c1819e90d8p+0};

// exp(x) for x <= 0 with the table `tab` (the 64 entries above) in shared
// memory. See the header comment for accuracy and underflow semantics.
__device__ __forceinline__ double fexp(double x, const double* __restrict__ tab) {
  const double t = fma(x, kExpL, kRoundMagic);  // low word = k = rint(64x/ln2)
  const double kd = t - kRoundMagic;
  double r = fma(kd, -kLn2By64Hi, x);
  r = fma(kd, -kLn2By64Lo, r);
  double p = fma(kC5, r, kC4);
  p = fma(p, r, kC3);
  p = fma(p, r, kC2);
  p = fma(p, r, 1.0);
  p = p * r;  // expm1(r)
  const long long tb = __double_as_longlong(t);
  const int k = static_cast<int>(tb);
  const double tj = tab[k & 63];
  // 2^(k/64) = 2^(k>>6) * 2^((k&63)/64): add (k>>6) to tj's exponent field.
  const int hi = __double2hiint(tj) + ((k >> 6) << 20);
  const double ts = __hiloint2double(hi, __double2loint(tj));
  const double res = fma(ts, p, ts);
  return tb < kFlushBits ? 0.0 : res;
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
