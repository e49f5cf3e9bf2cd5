// Device-side building blocks of the B200 Hawkes engine: the FP64 exp used on
// every pair, the constants it needs, and the TMA (cp.async.bulk) / mbarrier
// helpers that stage source tiles into shared memory.
//
// Why a hand-written exp: the pair kernels are bound by the FP64 pipe
// (SURVEY.md §8 d2-d3), and the two exps per pair are ~70% of the FP64
// instructions. CUDA's double exp costs 14 DFMA + 1 DADD on sm_100a; this one
// costs 8 FP64 instructions (3 DADD for an exact reduction, 4 polynomial,
// 1 reconstruction): the caller folds 256/ln2 into its exponent constants,
// 2^(j/256) comes from a 256-entry shared-memory table and the 2^m scaling is
// a single integer IMAD on the table entry's hi word.
//
// Semantics vs the reference (pack.hpp:86-154, laneExp at pack.hpp:157):
//   * accuracy: table entries correctly rounded, the reduction is exact,
//     polynomial max abs error 2.4e-18 on |u| <= 1/2 -> about 1 ulp worst,
//     the same class as the reference's Pack exp (<= 2 ulp, test_pack.cpp:21-46);
//     folding 256/ln2 into the exponent adds one rounding of the argument;
//   * underflow: returns exactly +0 when k = rint(256 x / ln2) < -261632, i.e.
//     for every x < -708.40 (and -inf). The reference's Pack exp flushes
//     x < -708 to 0 (pack.hpp:124); libm returns subnormals down to -745.13.
//     The difference is below 3.3e-308 per pair (SURVEY.md §7 "lane-exp flush").
//   * domain: callers pass x <= 0. Positive x (masked-out trigger lanes) give
//     garbage that the caller discards with a select, never a multiply.
#pragma once

#include <cstdint>

namespace sthk {

// 256/ln2 (callers pass exponents pre-multiplied by it: "L units") and the
// 1.5*2^52 rounding constant.
constexpr double kExpL = 0x1.71547652b82fep+8;
constexpr double kRoundMagic = 0x1.8p52;
// expm1(u ln2/256) ~= u (e1 + u (e2 + u (e3 + u e4))) on |u| <= 1/2
// (least-squares near-minimax fit in 200-bit arithmetic; max abs err 2.4e-18).
constexpr double kE1 = 0x1.62e42fefa39b9p-9;
constexpr double kE2 = 0x1.ebfbdff82c56bp-19;
constexpr double kE3 = 0x1.c6b090da1e21bp-29;
constexpr double kE4 = 0x1.3b2ab8bfe4dbcp-39;
// Smallest k = rint(x) whose 2^(k/256) is a normal double is -1022*256.
constexpr int kMinK = -261632;
// bits(1.5*2^52) + kMinK: rounded-t bit patterns below this flush to +0.
constexpr long long kFlushBits = 0x4338000000000000LL + kMinK;
// Exponents (L units) above this never flush: kernels use the unchecked exp
// for stages whose exponent lower bound clears it.
constexpr double kSafeExpL = -261000.0;

// 2^(j/256), j = 0..255, correctly rounded (mpmath, 200 bits), stored as
// {lo word, hi word - (j << 12)}: adding (k << 12) to the stored hi word of
// entry j = k & 255 yields the hi word of 2^(k>>8) * 2^(j/256) in one IMAD.
__device__ __constant__ uint2 kExpTable[256] = {
    {0x00000000u, 0x3ff00000u}, {0xfa5abcbfu, 0x3feffb1au}, {0xa9fb3335u, 0x3feff63du}, {0x143b0281u, 0x3feff168u},
    {0x3e778061u, 0x3fefec9au}, {0x2e11bbccu, 0x3fefe7d4u}, {0xe86e7f85u, 0x3fefe315u}, {0x72f654b1u, 0x3fefde5fu},
    {0xd3158574u, 0x3fefd9b0u}, {0x0e3c1f89u, 0x3fefd50au}, {0x29ddf6deu, 0x3fefd06bu}, {0x2b72a836u, 0x3fefcbd4u},
    {0x18759bc8u, 0x3fefc745u}, {0xf66607e0u, 0x3fefc2bdu}, {0xcac6f383u, 0x3fefbe3eu}, {0x9b1f3919u, 0x3fefb9c7u},
    {0x6cf9890fu, 0x3fefb558u}, {0x45e46c85u, 0x3fefb0f1u}, {0x2b7247f7u, 0x3fefac92u}, {0x23395decu, 0x3fefa83bu},
    {0x32d3d1a2u, 0x3fefa3ecu}, {0x5fdfa9c5u, 0x3fef9fa5u}, {0xaffed31bu, 0x3fef9b66u}, {0x28d7233eu, 0x3fef9730u},
    {0xd0125b51u, 0x3fef9301u}, {0xab5e2ab6u, 0x3fef8edbu}, {0xc06c31ccu, 0x3fef8abdu}, {0x14f204abu, 0x3fef86a8u},
    {0xaea92de0u, 0x3fef829au}, {0x934f312eu, 0x3fef7e95u}, {0xc8a58e51u, 0x3fef7a98u}, {0x5471c3c2u, 0x3fef76a4u},
    {0x3c7d517bu, 0x3fef72b8u}, {0x8695bbc0u, 0x3fef6ed4u}, {0x388c8deau, 0x3fef6af9u}, {0x58375d2fu, 0x3fef6726u},
    {0xeb6fcb75u, 0x3fef635bu}, {0xf8138a1cu, 0x3fef5f99u}, {0x84045cd4u, 0x3fef5be0u}, {0x95281c6bu, 0x3fef582fu},
    {0x3168b9aau, 0x3fef5487u}, {0x5eb44027u, 0x3fef50e7u}, {0x22fcd91du, 0x3fef4d50u}, {0x8438ce4du, 0x3fef49c1u},
    {0x88628cd6u, 0x3fef463bu}, {0x3578a819u, 0x3fef42beu}, {0x917ddc96u, 0x3fef3f49u}, {0xa27912d1u, 0x3fef3bddu},
    {0x6e756238u, 0x3fef387au}, {0xfb82140au, 0x3fef351fu}, {0x4fb2a63fu, 0x3fef31ceu}, {0x711ece75u, 0x3fef2e85u},
    {0x65e27cddu, 0x3fef2b45u}, {0x341ddf29u, 0x3fef280eu}, {0xe1f56381u, 0x3fef24dfu}, {0x7591bb70u, 0x3fef21bau},
    {0xf51fdee1u, 0x3fef1e9du}, {0x66d10f13u, 0x3fef1b8au}, {0xd0dad990u, 0x3fef187fu}, {0x39771b2fu, 0x3fef157eu},
    {0xa6e4030bu, 0x3fef1285u}, {0x1f641589u, 0x3fef0f96u}, {0xa93e2f56u, 0x3fef0cafu}, {0x4abd886bu, 0x3fef09d2u},
    {0x0a31b715u, 0x3fef06feu}, {0xedeeb2fdu, 0x3fef0432u}, {0xfc4cd831u, 0x3fef0170u}, {0x3ba8ea32u, 0x3feefeb8u},
    {0xb26416ffu, 0x3feefc08u}, {0x66e3fa2du, 0x3feef962u}, {0x5f929ff1u, 0x3feef6c5u}, {0xa2de883bu, 0x3feef431u},
    {0x373aa9cbu, 0x3feef1a7u}, {0x231e754au, 0x3feeef26u}, {0x6d05d866u, 0x3feeecaeu}, {0x1b7140efu, 0x3feeea40u},
    {0x34e59ff7u, 0x3feee7dbu}, {0xbfec6cf4u, 0x3feee57fu}, {0xc313a8e5u, 0x3feee32du}, {0x44ede173u, 0x3feee0e5u},
    {0x4c123422u, 0x3feedea6u}, {0xdf1c5175u, 0x3feedc70u}, {0x04ac801cu, 0x3feeda45u}, {0xc367a024u, 0x3feed822u},
    {0x21f72e2au, 0x3feed60au}, {0x2709468au, 0x3feed3fbu}, {0xd950a897u, 0x3feed1f5u}, {0x3f84b9d4u, 0x3feecffau},
    {0x6061892du, 0x3feece08u}, {0x42a7d232u, 0x3feecc20u}, {0xed1d0057u, 0x3feeca41u}, {0x668b3237u, 0x3feec86du},
    {0xb5c13cd0u, 0x3feec6a2u}, {0xe192aed2u, 0x3feec4e1u}, {0xf0d7d3deu, 0x3feec32au}, {0xea6db7d7u, 0x3feec17du},
    {0xd5362a27u, 0x3feebfdau}, {0xb817c114u, 0x3feebe41u}, {0x99fddd0du, 0x3feebcb2u}, {0x81d8abffu, 0x3feebb2du},
    {0x769d2ca7u, 0x3feeb9b2u}, {0x7f4531eeu, 0x3feeb841u}, {0xa2cf6642u, 0x3feeb6dau}, {0xe83f4eefu, 0x3feeb57du},
    {0x569d4f82u, 0x3feeb42bu}, {0xf4f6ad27u, 0x3feeb2e2u}, {0xca5d920fu, 0x3feeb1a4u}, {0xdde910d2u, 0x3feeb070u},
    {0x36b527dau, 0x3feeaf47u}, {0xdbe2c4cfu, 0x3feeae27u}, {0xd497c7fdu, 0x3feead12u}, {0x27ff07ccu, 0x3feeac08u},
    {0xdd485429u, 0x3feeab07u}, {0xfba87a03u, 0x3feeaa11u}, {0x8a5946b7u, 0x3feea926u}, {0x90998b93u, 0x3feea845u},
    {0x15ad2148u, 0x3feea76fu}, {0x20dceb71u, 0x3feea6a3u}, {0xb976dc09u, 0x3feea5e1u}, {0xe6cdf6f4u, 0x3feea52au},
    {0xb03a5585u, 0x3feea47eu}, {0x1d1929fdu, 0x3feea3ddu}, {0x34ccc320u, 0x3feea346u}, {0xfebc8fb7u, 0x3feea2b9u},
    {0x82552225u, 0x3feea238u}, {0xc70833f6u, 0x3feea1c1u}, {0xd44ca973u, 0x3feea155u}, {0xb19e9538u, 0x3feea0f4u},
    {0x667f3bcdu, 0x3feea09eu}, {0xfa75173eu, 0x3feea052u}, {0x750bdabfu, 0x3feea012u}, {0xddd47645u, 0x3fee9fdcu},
    {0x3c651a2fu, 0x3fee9fb2u}, {0x98593ae5u, 0x3fee9f92u}, {0xf9519484u, 0x3fee9f7du}, {0x66f42e87u, 0x3fee9f74u},
    {0xe8ec5f74u, 0x3fee9f75u}, {0x86ead08au, 0x3fee9f82u}, {0x48a58174u, 0x3fee9f9au}, {0x35d7cbfdu, 0x3fee9fbdu},
    {0x564267c9u, 0x3fee9febu}, {0xb1ab6e09u, 0x3feea024u}, {0x4fde5d3fu, 0x3feea069u}, {0x38ac1cf6u, 0x3feea0b9u},
    {0x73eb0187u, 0x3feea114u}, {0x0976cfdbu, 0x3feea17bu}, {0x0130c132u, 0x3feea1edu}, {0x62ff86f0u, 0x3feea26au},
    {0x36cf4e62u, 0x3feea2f3u}, {0x8491c491u, 0x3feea387u}, {0x543e1a12u, 0x3feea427u}, {0xadd106d9u, 0x3feea4d2u},
    {0x994cce13u, 0x3feea589u}, {0x1eb941f7u, 0x3feea64cu}, {0x4623c7adu, 0x3feea71au}, {0x179f5b21u, 0x3feea7f4u},
    {0x9b4492edu, 0x3feea8d9u}, {0xd931a436u, 0x3feea9cau}, {0xd98a6699u, 0x3feeaac7u}, {0xa478580fu, 0x3feeabd0u},
    {0x422aa0dbu, 0x3feeace5u}, {0xbad61778u, 0x3feeae05u}, {0x16b5448cu, 0x3feeaf32u}, {0x5e0866d9u, 0x3feeb06au},
    {0x99157736u, 0x3feeb1aeu}, {0xd0282c8au, 0x3feeb2feu}, {0x0b91ffc6u, 0x3feeb45bu}, {0x53aa2fe2u, 0x3feeb5c3u},
    {0xb0cdc5e5u, 0x3feeb737u}, {0x2b5f98e5u, 0x3feeb8b8u}, {0xcbc8520fu, 0x3feeba44u}, {0x9a7670b3u, 0x3feebbddu},
    {0x9fde4e50u, 0x3feebd82u}, {0xe47a22a2u, 0x3feebf33u}, {0x70ca07bau, 0x3feec0f1u}, {0x4d53fe0du, 0x3feec2bbu},
    {0x82a3f090u, 0x3feec491u}, {0x194bb8d5u, 0x3feec674u}, {0x19e32323u, 0x3feec863u}, {0x8d07f29eu, 0x3feeca5eu},
    {0x7b5de565u, 0x3feecc66u}, {0xed8eb8bbu, 0x3feece7au}, {0xec4a2d33u, 0x3feed09bu}, {0x80460ad8u, 0x3feed2c9u},
    {0xb23e255du, 0x3feed503u}, {0x8af46052u, 0x3feed74au}, {0x1330b358u, 0x3feed99eu}, {0x53c12e59u, 0x3feedbfeu},
    {0x5579fdbfu, 0x3feede6bu}, {0x21356ebau, 0x3feee0e5u}, {0xbfd3f37au, 0x3feee36bu}, {0x3a3c2774u, 0x3feee5ffu},
    {0x995ad3adu, 0x3feee89fu}, {0xe622f2ffu, 0x3feeeb4cu}, {0x298db666u, 0x3feeee07u}, {0x6c9a8952u, 0x3feef0ceu},
    {0xb84f15fbu, 0x3feef3a2u}, {0x15b749b1u, 0x3feef684u}, {0x8de5593au, 0x3feef972u}, {0x29f1c52au, 0x3feefc6eu},
    {0xf2fb5e47u, 0x3feeff76u}, {0xf22749e4u, 0x3fef028cu}, {0x30a1064au, 0x3fef05b0u}, {0xb79a6f1fu, 0x3fef08e0u},
    {0x904bc1d2u, 0x3fef0c1eu}, {0xc3f3a207u, 0x3fef0f69u}, {0x5bd71e09u, 0x3fef12c2u}, {0x6141b33du, 0x3fef1628u},
    {0xdd85529cu, 0x3fef199bu}, {0xd9fa652cu, 0x3fef1d1cu}, {0x5fffd07au, 0x3fef20abu}, {0x78fafb22u, 0x3fef2447u},
    {0x2e57d14bu, 0x3fef27f1u}, {0x8988c933u, 0x3fef2ba8u}, {0x9406e7b5u, 0x3fef2f6du}, {0x5751c4dbu, 0x3fef3340u},
    {0xdcef9069u, 0x3fef3720u}, {0x2e6d1675u, 0x3fef3b0fu}, {0x555dc3fau, 0x3fef3f0bu}, {0x5b5bab74u, 0x3fef4315u},
    {0x4a07897cu, 0x3fef472du}, {0x2b08c968u, 0x3fef4b53u}, {0x080d89f2u, 0x3fef4f87u}, {0xeacaa1d6u, 0x3fef53c8u},
    {0xdcfba487u, 0x3fef5818u}, {0xe862e6d3u, 0x3fef5c76u}, {0x16c98398u, 0x3fef60e3u}, {0x71ff6075u, 0x3fef655du},
    {0x03db3285u, 0x3fef69e6u}, {0xd63a8315u, 0x3fef6e7cu}, {0xf301b460u, 0x3fef7321u}, {0x641c0658u, 0x3fef77d5u},
    {0x337b9b5fu, 0x3fef7c97u}, {0x6b197d17u, 0x3fef8167u}, {0x14f5a129u, 0x3fef8646u}, {0x3b16ee12u, 0x3fef8b33u},
    {0xe78b3ff6u, 0x3fef902eu}, {0x24676d76u, 0x3fef9539u}, {0xfbc74c83u, 0x3fef9a51u}, {0x77cdb740u, 0x3fef9f79u},
    {0xa2a490dau, 0x3fefa4afu}, {0x867cca6eu, 0x3fefa9f4u}, {0x2d8e67f1u, 0x3fefaf48u}, {0xa2188510u, 0x3fefb4aau},
    {0xee615a27u, 0x3fefba1bu}, {0x1cb6412au, 0x3fefbf9cu}, {0x376bba97u, 0x3fefc52bu}, {0x48dd7274u, 0x3fefcac9u},
    {0x5b6e4540u, 0x3fefd076u}, {0x798844f8u, 0x3fefd632u}, {0xad9cbe14u, 0x3fefdbfdu}, {0x02243c89u, 0x3fefe1d8u},
    {0x819e90d8u, 0x3fefe7c1u}, {0x3692d514u, 0x3fefedbau}, {0x2b8f71f1u, 0x3feff3c2u}, {0x6b2a23d9u, 0x3feff9d9u},
};

// exp(x / kExpL) for an exponent x given in L units (x <= 0), with the 256
// table entries above in shared memory. 8 FP64 instructions: 3 DADD for the
// exact reduction x = k + u (|u| <= 1/2), 4 for the polynomial, 1 to
// reconstruct. CHECK selects the flush of k < kMinK (and -inf) to +0; callers
// pass CHECK=false only when the exponent is provably >= kSafeExpL.
template <bool CHECK>
__device__ __forceinline__ double exp_l(double x, const uint2* __restrict__ tab) {
  const double t = x + kRoundMagic;  // low word = k = rint(x)
  const double kd = t - kRoundMagic;
  const double u = x - kd;           // exact
  double q = fma(kE4, u, kE3);
  q = fma(q, u, kE2);
  q = fma(q, u, kE1);
  const double p = q * u;            // expm1(u ln2/256)
  const long long tb = __double_as_longlong(t);
  const int k = static_cast<int>(tb);
  const uint2 tj = tab[k & 255];
  const double ts = __hiloint2double(static_cast<int>(tj.y) + (k << 12), static_cast<int>(tj.x));
  const double res = fma(ts, p, ts);
  if constexpr (CHECK) return tb < kFlushBits ? 0.0 : res;
  return res;
}

// N independent exp_l evaluations written in lockstep (stage by stage), so
// the dependent 8-instruction chains are interleaved in program order and the
// FP64 pipe's latency is covered by N-way ILP even at low occupancy.
template <bool CHECK, int N>
__device__ __forceinline__ void exp_l_batch(const double (&x)[N], double (&out)[N],
                                            const uint2* __restrict__ tab) {
  double t[N], u[N], q[N];
#pragma unroll
  for (int i = 0; i < N; ++i) t[i] = x[i] + kRoundMagic;
#pragma unroll
  for (int i = 0; i < N; ++i) u[i] = x[i] - (t[i] - kRoundMagic);
#pragma unroll
  for (int i = 0; i < N; ++i) q[i] = fma(kE4, u[i], kE3);
#pragma unroll
  for (int i = 0; i < N; ++i) q[i] = fma(q[i], u[i], kE2);
#pragma unroll
  for (int i = 0; i < N; ++i) q[i] = fma(q[i], u[i], kE1);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double p = q[i] * u[i];
    const long long tb = __double_as_longlong(t[i]);
    const int k = static_cast<int>(tb);
    const uint2 tj = tab[k & 255];
    const double ts =
        __hiloint2double(static_cast<int>(tj.y) + (k << 12), static_cast<int>(tj.x));
    const double res = fma(ts, p, ts);
    out[i] = CHECK ? (tb < kFlushBits ? 0.0 : res) : res;
  }
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
