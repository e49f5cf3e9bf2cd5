// sm_100a kernels of the B200 spatiotemporal-Hawkes likelihood engine.
//
// One evaluation = (plan || prep) -> pair kernels -> finalize [-> NCCL
// all-reduce -> final sum]; the host side is sthk_engine.cpp, the reference
// algorithm pairReduceBlock (backend.hpp:95-137) with HawkesPairTerm
// (kernels.hpp:76-106) and logLikelihood (likelihood.cpp:10-55).
//
//  tile_box_kernel        (once per load) per 128-event tile bounding box and
//                         time range, pad zeroing, the EventSet checks.
//  plan_kernel            per 128-row target tile the live source ranges from
//                         sorted-time searches (exact underflow culling), split
//                         into the general near list, the trigger-free near
//                         list and the FP32 far list, each ordered largest
//                         item first.
//  prep_kernel            scaled FP64 / FP32 coordinates, zeroed fixed-point
//                         accumulators, compensator terms (kernels.hpp:54-65).
//  sym_kernel<GRAD, BGONLY>  the FP64 near sweep: symmetric background (row
//                         and column sums, fixed-point integer atomics),
//                         trigger rows (the strict t_src < t_tgt rule,
//                         kernels.hpp:99-100), gradient sums fused (SURVEY.md
//                         §8 a16); BGONLY: the trigger-free variant.
//  far_kernel<GRAD>       the FP32 far tier (every exponent < -40), concurrent
//                         with the near sweep on a second stream.
//  pair_kernel<GRAD>      the row-only (non-symmetric) sweep, kernel mode 0.
//  finalize_kernel<GRAD>  per row: chunk partials in chunk order, lambda, log,
//                         gradient terms, degenerate flag (likelihood.cpp:
//                         34-43); block partials, and for one shard the fused
//                         fixed-order final sum into host-mapped memory.
//  final_sum_kernel       fixed-order sum of the block partials (several
//                         shards, after the NCCL all-reduce).
//
// Determinism: every floating-point sum has a fixed order that depends only
// on (events, params) -- not on scheduling, culling decisions or the number
// of GPUs -- so results are bitwise reproducible.
#include <cmath>

#include "sthk_device.cuh"
#include "sthk_kernels.cuh"

#ifndef STHK_PAIR_MINB
#define STHK_PAIR_MINB 5  // resident pair CTAs per SM the register budget targets
#endif

namespace sthk {

namespace {

constexpr double kInvSqrt2 = 0.7071067811865475244;     // kernels.hpp:14


// Work-item hand-out of the persistent pair kernels. STHK_STATIC_FIRST: a
// CTA's first item is its block index (consecutive blocks are dispatched to
// different SMs, so with fewer items than CTAs -- small N -- the items spread
// over the SMs instead of piling onto the first CTAs to arrive), later items
// come from the atomic counter. Scheduling only: every item's partials have
// fixed destinations, so results do not depend on it.
#ifndef STHK_STATIC_FIRST
#define STHK_STATIC_FIRST 1
#endif
__device__ __forceinline__ int next_item(int* counter, int iter) {
#if STHK_STATIC_FIRST
  return iter == 0 ? static_cast<int>(blockIdx.x) : static_cast<int>(gridDim.x) + atomicAdd(counter, 1);
#else
  return atomicAdd(counter, 1);
#endif
}
constexpr double kInvSqrt2Pi = 0.3989422804014326779;   // kernels.hpp:13

// Sorted-time searches in two levels: kPivots evenly spaced pivots
// piv[k] = t[k * stride] (computed at load, +inf padded) in shared memory
// narrow the range to one stride, then a binary search over global memory
// finishes it (log2(stride) loads, 4 at C2). The plan is one CTA, so its
// global loads are bounded by one SM's outstanding-miss capacity: fewer loads
// per search, not fewer dependent steps, is what shortens it.
constexpr int kPivots = kPlanPivots;
__device__ __forceinline__ int64_t pivot_stride(int64_t n) { return (n + kPivots - 1) / kPivots; }

// Tile pivots (N <= kPivots * 128): piv[k] = the last time of 128-event tile
// k, and a search answers at tile granularity -- the start of the tile that
// holds the exact answer, in shared memory only. Every consumer rounds its
// range starts down to whole 128-source stages, so this changes no stage set
// (the row kernel's upper bound is rounded up instead: the extra sources lie
// beyond the exact-underflow window, exact zeros). Larger N: strided pivots
// piv[k] = t[k * stride] and log2(stride) global rounds to the exact index.
struct Pivots {
  const double* piv;  // shared memory, np entries
  int np;
  int64_t stride;
  bool tiles;
};

// K independent searches in lockstep. Result: the first index in [0, n) whose
// time is not "before" v (t < v when strict, t <= v otherwise).
template <int K>
__device__ __forceinline__ void bounds_lockstep(const double* t, int64_t n, const Pivots& p,
                                                const double (&v)[K], const bool (&strict)[K],
                                                int64_t (&out)[K]) {
  auto before = [&](int k, double tv) { return strict[k] ? tv < v[k] : tv <= v[k]; };
  // pivot level: branch-free power-of-two steps over the +inf-padded pivots,
  // the K shared-memory chains interleaved; kp = number of pivots before v
  int kp[K];
#pragma unroll
  for (int k = 0; k < K; ++k) kp[k] = 0;
#pragma unroll
  for (int step = kPivots / 2; step > 0; step >>= 1) {
#pragma unroll
    for (int k = 0; k < K; ++k) kp[k] = before(k, p.piv[kp[k] + step - 1]) ? kp[k] + step : kp[k];
  }
#pragma unroll
  for (int k = 0; k < K; ++k) kp[k] = before(k, p.piv[kPivots - 1]) ? kPivots : kp[k];
  if (p.tiles) {  // the first tile with an event not before v starts at kp * 128
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = min(static_cast<int64_t>(kp[k]) * kTS, n);
    return;
  }
  int lo[K], hi[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {  // (kp == 0: t[0] is not before v)
    lo[k] = kp[k] == 0 ? 0 : (kp[k] - 1) * static_cast<int>(p.stride) + 1;
    hi[k] = kp[k] == 0 ? 0 : static_cast<int>(min(static_cast<int64_t>(kp[k]) * p.stride, n));
  }
  // global level: a uniform number of binary rounds (segments are at most
  // stride - 1 long), one load per search per round (clamped in range; an
  // empty segment ignores it)
  const int nmax = static_cast<int>(n) - 1;
  int rounds = 0;
  for (int64_t len = p.stride - 1; len > 0; len >>= 1) ++rounds;
  for (int it = 0; it < rounds; ++it) {
    int m[K];
    double tv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      m[k] = (lo[k] + hi[k]) >> 1;
      tv[k] = t[min(m[k], nmax)];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool live = lo[k] < hi[k];
      const bool b = before(k, tv[k]);
      lo[k] = live && b ? m[k] + 1 : lo[k];
      hi[k] = live && !b ? m[k] : hi[k];
    }
  }
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = lo[k];
}

// ---------------------------------------------------------------------------
// Plan
// ---------------------------------------------------------------------------
// Live source range [lo, hi) and chunk range [c0, c1] of one row tile.
__device__ __forceinline__ void tile_plan(const PlanArgs& a, const Pivots& pv, int tile, int2& rg,
                                          int2& cr, int2& rgf, int2& crf, int2& rgb, int2& crb) {
  const int64_t first = static_cast<int64_t>(tile) * kTM;
  const int64_t last = min(first + kTM, a.n) - 1;
  const double2 tr = a.tile_trange[tile];  // (t[first], t[last]), one load
  const double tmin = tr.x, tmax = tr.y;
  // searches: live-range start, live-range end (full row-kernel sweeps) or,
  // in symmetric mode, the far tier's exact-cull start; the far split
  double v[3] = {a.trig_only ? tmin - a.dT : tmin - fmax(a.dB, a.dT),
                 a.sym ? tmin - a.dFar : tmax + a.dB, tmin - a.tfar};
  const bool strict[3] = {true, false, true};
  int64_t b[3];
  bounds_lockstep<3>(a.t, a.n, pv, v, strict, b);
  int lo, hi;
  if (a.dense) {
    lo = 0;
    hi = static_cast<int>(a.n);
  } else if (a.trig_only) {
    lo = min(static_cast<int>(b[0]), static_cast<int>(first));
    hi = static_cast<int>(last + 1);
  } else {
    // the tile's own rows are always live (background self term); (tile
    // pivots: the row kernel's end rounded up to the end of its tile)
    lo = min(static_cast<int>(b[0]), static_cast<int>(first));
    const int64_t b1 = pv.tiles ? min(b[1] + kTS, a.n) : b[1];
    hi = a.sym ? static_cast<int>(last + 1)
               : max(static_cast<int>(b1), static_cast<int>(last + 1));
  }
  // symmetric mode: later tiles reach this one through their column sums
  if (a.sym || a.trig_only) hi = static_cast<int>(last + 1);
  // far split: whole 128-stages of sources earlier than t[first] - tfar
  // (every term below e^-A) go to the far list; the rest stay near
  int fb = lo, flo = lo;
  if (a.tfar > 0.0 && last + 1 - first == kTM) {  // (full row tiles only)
    const int bb = static_cast<int>(b[2]);
    fb = max(lo, bb - bb % kTS);
    // far sources before t[first] - dFar are culled (invisible in the FP64 sums)
    if (!a.dense) flo = min(max(lo, static_cast<int>(b[1])), fb);
  }
  // background-only split of the near range: the near stages before the
  // last bg_adj stages ahead of the tile go to the trigger-free kernel. The
  // host picks bg_adj so that those sources are beyond every tile's trigger
  // window; the split is structural (it does not move with omega), so the
  // background sums' grouping -- hence their cached values -- stays the same.
  int fbt = fb;
  if (a.ranges_bg && !a.trig_only) {
    fbt = min(max(fb, static_cast<int>(first) - a.bg_adj * kTS), static_cast<int>(first));
  }
  rg = make_int2(fbt, hi);
  cr = make_int2(fbt / a.sc, (hi - 1) / a.sc);
  rgf = make_int2(flo, fb);
  crf = fb > flo ? make_int2(flo / a.sc_far, (fb - 1) / a.sc_far) : make_int2(0, -1);
  // (the trigger-free kernel takes the background of every near stage before
  // the diagonal one; the general kernel keeps the trigger terms of the
  // bg_adj stages ahead of the tile and the diagonal stage)
  const int fbe = !a.ranges_bg ? fbt : a.bg_all ? hi : static_cast<int>(first);
  rgb = make_int2(fb, fbe);
  crb = fbe > fb ? make_int2(fb / a.sc_bg, (fbe - 1) / a.sc_bg) : make_int2(0, -1);
  if (a.bg_all && a.ranges_bg) {  // (the general list is empty)
    rg = make_int2(hi, hi);
    cr = make_int2(0, -1);
  }
}

// Number of 128-source stages of work item (tile, chunk) -- the same bounds
// the pair kernels compute.
__device__ __forceinline__ int item_stages(int sc, int2 rg, int chunk) {
  int s_begin = max(rg.x, chunk * sc);
  s_begin -= s_begin % kTS;
  const int s_end = min(rg.y, (chunk + 1) * sc);
  return max((s_end - s_begin + kTS - 1) / kTS, 0);
}

constexpr int kPlanBins = 1024;  // item-size classes (stages, clamped)


// Single CTA: per-tile ranges, then the (tile, chunk) work list ordered by
// decreasing item size (a counting sort on the stage count), so the
// persistent pair kernel hands out the long items first and ends on short
// ones (less idle time in the tail); resets the pair kernel's work counter.
// The order only affects scheduling: every partial has a fixed destination
// and integer (fixed-point) accumulation, so results do not depend on it.
// The work lists (near, far, trigger-free) ordered by decreasing item size,
// all in one pass: per list a histogram of the items' stage counts, one
// exclusive scan over the bins in decreasing size for every list at once,
// then placement (1024 threads, one CTA; five barriers whatever the number
// of lists).
struct PlanList {
  int sc;
  const int2* ranges;
  const int2* crange;
  int2* items;
  int* n_items;
  int* work_counter;
};
constexpr int kPlanLists = 3;

// (my_rg / my_cr: this thread's first tile per list, kept in registers since
// the range phase)
// (per tile and list the first and the last chunk may be partial; every chunk
// between them is a full chunk of sc / 128 stages, counted and placed with one
// shared atomic per warp)
__device__ __forceinline__ void plan_lists(const PlanArgs& a, const PlanList (&pl)[kPlanLists],
                                           const bool (&on)[kPlanLists],
                                           const int2 (&my_rg)[kPlanLists],
                                           const int2 (&my_cr)[kPlanLists],
                                           int (*s_hist)[kPlanBins], int (*s_warp)[32]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntiles = a.tile1 - a.tile0;
  _Pragma("unroll") for (int l = 0; l < kPlanLists; ++l) {
    if (!on[l]) continue;
    for (int b = tid; b < kPlanBins; b += 1024) s_hist[l][b] = 0;
  }
  __syncthreads();
  auto tile_lists = [&](int l, int i, int2& rg, int2& cr) {
    rg = make_int2(0, 0);
    cr = make_int2(0, -1);
    if (i < ntiles) {
      rg = i == tid ? my_rg[l] : pl[l].ranges[a.tile0 + i];
      cr = i == tid ? my_cr[l] : pl[l].crange[a.tile0 + i];
    }
  };
  auto bin_of = [&](int l, int2 rg, int c) { return min(item_stages(pl[l].sc, rg, c), kPlanBins - 1); };
  for (int i0 = 0; i0 < ntiles; i0 += 1024) {  // (warp-uniform trip count)
    _Pragma("unroll") for (int l = 0; l < kPlanLists; ++l) {
      if (!on[l]) continue;
      int2 rg, cr;
      tile_lists(l, i0 + tid, rg, cr);
      int nfull = 0;
      if (cr.y >= cr.x) {
        atomicAdd(&s_hist[l][bin_of(l, rg, cr.x)], 1);
        if (cr.y > cr.x) atomicAdd(&s_hist[l][bin_of(l, rg, cr.y)], 1);
        nfull = max(cr.y - cr.x - 1, 0);
      }
      const int wsum = __reduce_add_sync(0xffffffffu, nfull);
      if (lane == 0 && wsum) atomicAdd(&s_hist[l][min(pl[l].sc / kTS, kPlanBins - 1)], wsum);
    }
  }
  __syncthreads();
  const int bin = kPlanBins - 1 - tid;  // thread t owns bin kPlanBins - 1 - t of every list
  int cnt[kPlanLists], v[kPlanLists];
  _Pragma("unroll") for (int l = 0; l < kPlanLists; ++l) {
    if (!on[l]) continue;
    cnt[l] = s_hist[l][bin];
    v[l] = cnt[l];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v[l], off);
      if (lane >= off) v[l] += u;
    }
    if (lane == 31) s_warp[l][warp] = v[l];
  }
  __syncthreads();
  if (warp < kPlanLists && on[warp]) {  // warp l scans list l's 32 warp totals
    int w = s_warp[warp][lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += u;
    }
    s_warp[warp][lane] = w;
  }
  __syncthreads();
  _Pragma("unroll") for (int l = 0; l < kPlanLists; ++l) {
    if (!on[l]) continue;
    const int incl = v[l] + (warp > 0 ? s_warp[l][warp - 1] : 0);
    if (tid == 1023) {
      *pl[l].n_items = incl;
      *pl[l].work_counter = 0;
    }
    s_hist[l][bin] = incl - cnt[l];  // start offset of the bin
  }
  __syncthreads();
  for (int i0 = 0; i0 < ntiles; i0 += 1024) {
    const int tile = a.tile0 + i0 + tid;
    _Pragma("unroll") for (int l = 0; l < kPlanLists; ++l) {
      if (!on[l]) continue;
      int2 rg, cr;
      tile_lists(l, i0 + tid, rg, cr);
      int nfull = 0;
      if (cr.y >= cr.x) {
        pl[l].items[atomicAdd(&s_hist[l][bin_of(l, rg, cr.x)], 1)] = make_int2(tile, cr.x);
        if (cr.y > cr.x) pl[l].items[atomicAdd(&s_hist[l][bin_of(l, rg, cr.y)], 1)] = make_int2(tile, cr.y);
        nfull = max(cr.y - cr.x - 1, 0);
      }
      // the full chunks: one reservation per warp, lanes at their prefix offsets
      int incl = nfull;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += u;
      }
      int base = 0;
      if (lane == 31 && incl) base = atomicAdd(&s_hist[l][min(pl[l].sc / kTS, kPlanBins - 1)], incl);
      base = __shfl_sync(0xffffffffu, base, 31);
      int pos = base + incl - nfull;
      for (int c = cr.x + 1; c < cr.y; ++c) pl[l].items[pos++] = make_int2(tile, c);
    }
  }
}

// Small sets with no trigger term in the near lists (row-window trigger sums:
// every item one background stage, equal work) and at most 1024 tiles: the
// lists in tile order -- the size order buys nothing -- by one block-wide
// scan of the per-tile item counts (two barriers instead of the histogram's
// five). (With trigger stages, whose items cost more, the sorted placement
// stays: measured 36.5 -> 39.4 us at 10k events, Θ_init, in tile order.)
__device__ __forceinline__ void plan_lists_tile_order(const PlanArgs& a, const PlanList (&pl)[kPlanLists],
                                                      const bool (&on)[kPlanLists],
                                                      const int2 (&my_cr)[kPlanLists],
                                                      int (*s_warp)[32]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntiles = a.tile1 - a.tile0;
  int cnt[kPlanLists], incl[kPlanLists];
  _Pragma("unroll") for (int l = 0; l < kPlanLists; ++l) {
    cnt[l] = 0;
    if (on[l] && tid < ntiles && my_cr[l].y >= my_cr[l].x) cnt[l] = my_cr[l].y - my_cr[l].x + 1;
    incl[l] = cnt[l];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl[l], off);
      if (lane >= off) incl[l] += u;
    }
    if (lane == 31) s_warp[l][warp] = incl[l];
  }
  __syncthreads();
  if (warp < kPlanLists && on[warp]) {  // warp l scans list l's 32 warp totals
    int w = s_warp[warp][lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += u;
    }
    s_warp[warp][lane] = w;
  }
  __syncthreads();
  _Pragma("unroll") for (int l = 0; l < kPlanLists; ++l) {
    if (!on[l]) continue;
    const int end = incl[l] + (warp > 0 ? s_warp[l][warp - 1] : 0);
    if (tid == 1023) {
      *pl[l].n_items = end;
      *pl[l].work_counter = 0;
    }
    int pos = end - cnt[l];
    for (int c = my_cr[l].x; c <= my_cr[l].y && cnt[l] > 0; ++c) {
      pl[l].items[pos++] = make_int2(a.tile0 + tid, c);
    }
  }
}

// Single CTA: per-tile near / far ranges, then each work list ordered by
// decreasing item size, so the persistent pair kernels hand out the long
// items first and end on short ones (less idle time in the tail); resets the
// kernels' work counters. The order only affects scheduling: every partial
// has a fixed destination and integer (fixed-point) accumulation, so results
// do not depend on it.
__device__ __forceinline__ void plan_body(const PlanArgs& a) {
  __shared__ int s_hist[kPlanLists][kPlanBins];
  __shared__ int s_warp[kPlanLists][32];
  __shared__ __align__(8) uint64_t s_bar;
  extern __shared__ __align__(128) double s_piv[];  // kPivots (dynamic: 64 KB)
  const int tid = threadIdx.x;
  // (graph mode: the trigger-free kernel is launched by a programmatic edge
  // from here; its CTAs set up while the plan runs and wait for its lists)
  asm volatile("griddepcontrol.launch_dependents;");
  const unsigned long long trace_t0 = (a.trace && tid == 0) ? global_ns() : 0ULL;
  if (tid == 0) stamp_min(a.tstamp, 0);
  const int ntiles = a.tile1 - a.tile0;
  Pivots pv;
  pv.tiles = a.tile_pivots != 0;
  pv.stride = pv.tiles ? kTS : pivot_stride(a.n);
  pv.np = static_cast<int>((a.n + pv.stride - 1) / pv.stride);
  pv.piv = s_piv;
  if (tid == 0) {  // the pivots (precomputed at load): one bulk copy
    mbar_init(&s_bar, 1);
    mbar_fence_init();
    mbar_arrive_expect_tx(&s_bar, kPivots * sizeof(double));
    tma_load_1d(s_piv, a.piv, kPivots * sizeof(double), &s_bar);
  }
  __syncthreads();
  mbar_wait(&s_bar, 0);
  if (a.trace && tid == 0) trace_cta(a.trace, a.trace_cap, 7, trace_t0);  // (phase: pivots staged)
  int2 my[6] = {make_int2(0, 0), make_int2(0, -1), make_int2(0, 0), make_int2(0, -1),
                make_int2(0, 0), make_int2(0, -1)};  // first tile: near, far, bg (range, chunks)
  for (int i = tid; i < ntiles; i += 1024) {
    int2 rg, cr, rgf, crf, rgb, crb;
    tile_plan(a, pv, a.tile0 + i, rg, cr, rgf, crf, rgb, crb);
    a.ranges[a.tile0 + i] = rg;
    a.crange[a.tile0 + i] = cr;
    if (a.ranges_far) {
      a.ranges_far[a.tile0 + i] = rgf;
      a.crange_far[a.tile0 + i] = crf;
    }
    if (a.ranges_bg) {
      a.ranges_bg[a.tile0 + i] = rgb;
      a.crange_bg[a.tile0 + i] = crb;
    }
    if (i == tid) {
      my[0] = rg;
      my[1] = cr;
      my[2] = rgf;
      my[3] = crf;
      my[4] = rgb;
      my[5] = crb;
    }
  }
  __syncthreads();
  if (a.trace && tid == 0) trace_cta(a.trace, a.trace_cap, 8, trace_t0);  // (phase: tile ranges)
  // fixed slots: 0 near, 1 far, 2 trigger-free (inactive lists are skipped)
  const PlanList pl[kPlanLists] = {
      PlanList{a.sc, a.ranges, a.crange, a.items, a.n_items, a.work_counter},
      PlanList{a.sc_far, a.ranges_far, a.crange_far, a.items_far, a.n_items_far, a.work_counter_far},
      PlanList{a.sc_bg, a.ranges_bg, a.crange_bg, a.items_bg, a.n_items_bg, a.work_counter_bg}};
  const bool on[kPlanLists] = {true, a.ranges_far != nullptr, a.ranges_bg != nullptr};
  const int2 mrg[kPlanLists] = {my[0], my[2], my[4]};
  const int2 mcr[kPlanLists] = {my[1], my[3], my[5]};
  const int nt = a.tile1 - a.tile0;
  if (a.tile_order && nt <= 1024 && a.sc == kTS && (!on[1] || a.sc_far == kTS) &&
      (!on[2] || a.sc_bg == kTS)) {
    plan_lists_tile_order(a, pl, on, mcr, s_warp);
  } else {
    plan_lists(a, pl, on, mrg, mcr, s_hist, s_warp);
  }
  if (a.trace && tid == 0) trace_cta(a.trace, a.trace_cap, 4, trace_t0);
}

__global__ void __launch_bounds__(1024) plan_kernel(const PlanArgs a) { plan_body(a); }

// ---------------------------------------------------------------------------
// Pair kernel
// ---------------------------------------------------------------------------
// TR: 0 = no trigger term, 1 = trigger without mask (every source strictly
// earlier than every target of the tile), 2 = trigger with the strict
// t_src < t_tgt mask (kernels.hpp:99-100), applied as a select so masked-out
// lanes (whose exponent may be positive) contribute exactly +0.
// CHECK = false when the stage's exponent lower bound proves no pair can
// underflow, so exp_l may skip its flush test.
template <bool GRAD, bool BG, int TR, bool CHECK>
__device__ __forceinline__ void stage_loop(const double* __restrict__ sx,
                                           const double* __restrict__ sy,
                                           const double* __restrict__ st, int cnt,
                                           double xi, double yi, double ti,
                                           const PairConsts& k,
                                           const uint2* __restrict__ tab,
                                           double* acc) {
#pragma unroll 4
  for (int j = 0; j < cnt; ++j) {
    const double sj = st[j];
    const double dx = xi - sx[j];
    const double dy = yi - sy[j];
    const double dt = ti - sj;
    const double r2 = fma(dx, dx, dy * dy);
    if constexpr (BG) {
      const double dt2 = dt * dt;
      const double e = exp_l<CHECK>(fma(k.cxL, r2, k.ctL * dt2), tab);
      acc[0] += e;
      if constexpr (GRAD) {
        acc[1] = fma(e, r2, acc[1]);
        acc[2] = fma(e, dt2, acc[2]);
      }
    }
    if constexpr (TR != 0) {
      double e = exp_l<CHECK>(fma(k.nomL, dt, k.chL * r2), tab);
      if constexpr (TR == 2) e = (sj < ti) ? e : 0.0;
      if constexpr (GRAD) {
        acc[3] += e;
        acc[4] = fma(e, dt, acc[4]);
        acc[5] = fma(e, r2, acc[5]);
      } else {
        acc[1] += e;
      }
    }
  }
}

template <bool GRAD, bool CHECK>
__device__ __forceinline__ void stage_dispatch(bool bg, int tr, const double* sx,
                                               const double* sy, const double* st, int cnt,
                                               double xi, double yi, double ti,
                                               const PairConsts& k, const uint2* tab,
                                               double* acc) {
  if (bg) {
    if (tr == 0) stage_loop<GRAD, true, 0, CHECK>(sx, sy, st, cnt, xi, yi, ti, k, tab, acc);
    else if (tr == 1) stage_loop<GRAD, true, 1, CHECK>(sx, sy, st, cnt, xi, yi, ti, k, tab, acc);
    else stage_loop<GRAD, true, 2, CHECK>(sx, sy, st, cnt, xi, yi, ti, k, tab, acc);
  } else {
    if (tr == 1) stage_loop<GRAD, false, 1, CHECK>(sx, sy, st, cnt, xi, yi, ti, k, tab, acc);
    else if (tr == 2) stage_loop<GRAD, false, 2, CHECK>(sx, sy, st, cnt, xi, yi, ti, k, tab, acc);
  }
}

// Item-end row output. Background sums (which also receive column
// contributions in kSym mode; S_B >= 1 always, the self term) go to the
// fixed-point accumulators; trigger sums, which are row-only and may be
// arbitrarily small, keep full relative precision as double partials per
// (chunk, row), summed in chunk order by finalize.
template <bool GRAD>
__device__ __forceinline__ void store_row_sums(const PairArgs& a, int chunk, int64_t row,
                                               const double* acc) {
  constexpr int NB = GRAD ? 3 : 1;  // background sums
  constexpr int NT = GRAD ? 3 : 1;  // trigger sums
  if (row >= a.n) return;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    if (a.bg_off) break;
    fx_add(a.fx + static_cast<size_t>(2 * q) * a.npad + row,
           a.fx + static_cast<size_t>(2 * q + 1) * a.npad + row, acc[q] * a.fxq[q]);
  }
  if (a.tr_off) return;
  double* out = a.tpart + static_cast<size_t>(chunk) * NT * a.npad + row;
#pragma unroll
  for (int q = 0; q < NT; ++q) out[static_cast<size_t>(q) * a.npad] = acc[NB + q];
}

constexpr uint32_t kBoxBytes = sizeof(double4);
constexpr uint32_t kTabBytes = sizeof(uint2) * kExpTableSize;

template <bool GRAD>
__global__ void __launch_bounds__(kTM, STHK_PAIR_MINB) pair_kernel(const PairArgs a) {
  constexpr int NS = GRAD ? kNSumGrad : kNSumVal;
  __shared__ __align__(128) double s_src[2][3][kTS];
  extern __shared__ __align__(128) uint2 s_tab[];  // kExpTableSize entries (dynamic)
  __shared__ __align__(32) double4 s_box[2];  // bounding box of the staged source tile
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ int s_item[2];

  const int tid = threadIdx.x;
  __shared__ unsigned long long s_cta_t0;  // (development trace)
  if (a.trace && tid == 0) s_cta_t0 = global_ns();
  if (tid == 0) {
    stamp_min(a.tstamp, 0);
    stamp_min(a.tstamp, 2);
  }
  __shared__ __align__(8) uint64_t s_tbar;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_init(&s_tbar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {  // the exp table: one 16 KB bulk copy (L2-resident source)
    mbar_arrive_expect_tx(&s_tbar, kTabBytes);
    tma_load_1d(s_tab, kExpTable, kTabBytes, &s_tbar);
  }
  mbar_wait(&s_tbar, 0);

  const int n_items = *a.n_items;
  const int64_t n = a.n;
  uint32_t phase = 0;
  unsigned long long cBg = 0, cTr = 0, cAny = 0;

  for (int iter = 0;; ++iter) {
    if (tid == 0) s_item[iter & 1] = next_item(a.work_counter, iter);
    __syncthreads();
    const int item = s_item[iter & 1];
    if (item >= n_items) break;

    const int2 it = a.items[item];
    const int tile = it.x, chunk = it.y;
    const int2 rg = a.ranges[tile];
    const int64_t first = static_cast<int64_t>(tile) * kTM;
    const int64_t row = first + tid;
    const double xi = a.x[row], yi = a.y[row], ti = a.t[row];
    const int64_t last = min(first + kTM, n) - 1;
    const double tmin = a.t[first], tmax = a.t[last];
    const double4 bt = a.tile_box[tile];
    const int rows_real = static_cast<int>(last - first + 1);

    int s_begin = max(rg.x, chunk * a.sc);
    s_begin -= s_begin % kTS;
    const int s_end = min(rg.y, (chunk + 1) * a.sc);
    const int nst = (s_end - s_begin + kTS - 1) / kTS;

    double acc[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) acc[q] = 0.0;

    constexpr uint32_t kStageBytes = kTS * sizeof(double);
    if (tid == 0 && nst > 0) {
      mbar_arrive_expect_tx(&s_bar[0], 3 * kStageBytes + kBoxBytes);
      tma_load_1d(&s_box[0], a.tile_box + s_begin / kTS, kBoxBytes, &s_bar[0]);
      tma_load_1d(s_src[0][0], a.x + s_begin, kStageBytes, &s_bar[0]);
      tma_load_1d(s_src[0][1], a.y + s_begin, kStageBytes, &s_bar[0]);
      tma_load_1d(s_src[0][2], a.t + s_begin, kStageBytes, &s_bar[0]);
    }
    for (int s = 0; s < nst; ++s) {
      const int buf = s & 1;
      // every thread is done with the other buffer (stage s-1) -> refill it
      __syncthreads();
      if (tid == 0 && s + 1 < nst) {
        const int nb = buf ^ 1;
        const int64_t s0n = s_begin + static_cast<int64_t>(s + 1) * kTS;
        mbar_arrive_expect_tx(&s_bar[nb], 3 * kStageBytes + kBoxBytes);
        tma_load_1d(&s_box[nb], a.tile_box + s0n / kTS, kBoxBytes, &s_bar[nb]);
        tma_load_1d(s_src[nb][0], a.x + s0n, kStageBytes, &s_bar[nb]);
        tma_load_1d(s_src[nb][1], a.y + s0n, kStageBytes, &s_bar[nb]);
        tma_load_1d(s_src[nb][2], a.t + s0n, kStageBytes, &s_bar[nb]);
      }
      const int64_t s0 = s_begin + static_cast<int64_t>(s) * kTS;
      const int cnt = static_cast<int>(min(static_cast<int64_t>(kTS), n - s0));
      mbar_wait(&s_bar[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
      // stage metadata from the staged copy (no global-memory round trip)
      const double4 bs = s_box[buf];
      const double smin = s_src[buf][2][0], smax = s_src[buf][2][cnt - 1];

      const bool bg = !a.bg_off && !(smin > tmax + a.k.dB || smax < tmin - a.k.dB);
      int tr;
      if (smin >= tmax || smax < tmin - a.k.dT) tr = 0;
      else if (smax < tmin) tr = 1;
      else tr = 2;
      // exponent lower bounds over the (tile, stage) box pair
      const double dxm = fmax(bt.y - bs.x, bs.y - bt.x);
      const double dym = fmax(bt.w - bs.z, bs.w - bt.z);
      const double r2m = dxm * dxm + dym * dym;
      const double dtm = fmax(tmax - smin, smax - tmin);
      const bool safe = (!bg || a.k.cxL * r2m + a.k.ctL * (dtm * dtm) > kSafeExpL) &&
                        (!tr || a.k.nomL * dtm + a.k.chL * r2m > kSafeExpL);


      const double* sx = s_src[buf][0];
      const double* sy = s_src[buf][1];
      const double* st = s_src[buf][2];
      if (safe) stage_dispatch<GRAD, false>(bg, tr, sx, sy, st, cnt, xi, yi, ti, a.k, s_tab, acc);
      else stage_dispatch<GRAD, true>(bg, tr, sx, sy, st, cnt, xi, yi, ti, a.k, s_tab, acc);
      if (tid == 0) {
        const unsigned long long pr = static_cast<unsigned long long>(cnt) * rows_real;
        if (bg) cBg += pr;
        if (tr) cTr += pr;
        if (bg || tr) cAny += pr;
      }
    }

    store_row_sums<GRAD>(a, chunk, row, acc);
  }

  if (tid == 0) {  // the last CTA out re-arms the work counter for the next launch
    __threadfence();
    if (atomicAdd(a.done_counter, 1u) == gridDim.x - 1) {
      *a.work_counter = 0;
      *a.done_counter = 0u;
    }
    if (a.trace) trace_cta(a.trace, a.trace_cap, a.trace_kernel, s_cta_t0);
    stamp_max(a.tstamp, 3);
  }
  if (tid == 0 && a.pair_counts) {
    atomicAdd(&a.pair_counts[0], cBg);
    atomicAdd(&a.pair_counts[1], cTr);
    atomicAdd(&a.pair_counts[2], cAny);
    atomicAdd(&a.pair_counts[3], cBg);   // background exps executed
    atomicAdd(&a.pair_counts[4], cAny);  // pair geometries executed
  }
}

// ---------------------------------------------------------------------------
// Symmetric-background pair kernel (kSym)
// ---------------------------------------------------------------------------
// A CTA owns a 128-row target tile I; lane l of every warp holds rows
// l + 32q (q < 4) in registers, and warp w sweeps columns 32w..32w+31 of each
// 128-source stage, so each thread evaluates a 4-row x 32-column block per
// stage with the column's coordinates broadcast from shared memory.
//   * J < I ("sym" stages): every background exp is added to its row sums
//     and to its column's sums (b_ij = b_ji); the 4-row column partials are
//     reduce-scattered across the warp with shuffles once per 4 columns and
//     flushed to the fixed-point column accumulators once per stage. The
//     trigger term (t_j < t_i) only feeds rows.
//   * J == I ("diag" stage): all ordered pairs of the tile, rows only.
// Row partials of the 4 warps are combined in a fixed order at item end.
constexpr int kSymR = 4;  // rows per thread
#ifndef STHK_SYM_G
#define STHK_SYM_G 4      // columns per shuffle reduce-scatter group (the far tier assumes 4)
#endif
#ifndef STHK_SPLIT_TRIG
#define STHK_SPLIT_TRIG 0  // 1: background and trigger terms of a stage in separate passes (measured slower)
#endif
#ifndef STHK_SYM_MINB
#if STHK_SPLIT_TRIG
#define STHK_SYM_MINB 4   // resident sym CTAs per SM the register budget targets
#else
#define STHK_SYM_MINB 3
#endif
#endif
constexpr int kSymG = STHK_SYM_G;
#ifndef STHK_G_UNROLL
#define STHK_G_UNROLL 1  // column groups per unrolled step of the stage loop (register-bound)
#endif
constexpr int kGUnroll = STHK_G_UNROLL;

template <bool GRAD, bool SYM, bool BG, int TR, bool CHECK, bool VALID, bool TS>
__device__ __forceinline__ void sym_pairs(int g, int perm, const double* __restrict__ sx,
                                          const double* __restrict__ sy,
                                          const double* __restrict__ st, int col0, int cnt,
                                          const double (&xi)[kSymR], const double (&yi)[kSymR],
                                          const double (&ti)[kSymR], const bool (&rv)[kSymR],
                                          const PairConsts& k, const uint2* __restrict__ tab,
                                          double (&racc)[kSymR][GRAD ? kNSumGrad : kNSumVal],
                                          double (&cp)[kSymG][GRAD ? 3 : 1]) {
  constexpr int T0 = GRAD ? 3 : 1;
#pragma unroll
  for (int q = 0; q < kSymG; ++q) {
    // lane-permuted column order: slot q of this lane is column q ^ perm, so
    // the reduce-scatter below needs no lane-dependent selects
    const int j = col0 + kSymG * g + (q ^ perm);
    const double xj = sx[j], yj = sy[j], tj = st[j];
    bool cv = true;
    if constexpr (VALID) cv = j < cnt;
    // geometry for the 4 rows (coordinates pre-scaled so that r2 is
    // -cxL * r^2), then the exps in lockstep
    double dt[kSymR], r2[kSymR], dt2[kSymR], arg[kSymR], e[kSymR];
#pragma unroll
    for (int r = 0; r < kSymR; ++r) {
      const double dx = xi[r] - xj;
      const double dy = yi[r] - yj;
      dt[r] = ti[r] - tj;
      r2[r] = fma(dx, dx, dy * dy);
    }
    if constexpr (BG) {
      // TS (trigger-free kernel, scaled times): the exponent is -(r2 + dts^2)
      // in one DFMA and the third sum weights each term by the exponent itself
      // (S_Bt = -sum - S_Br at the flush); else dt^2 is formed and weighted
#pragma unroll
      for (int r = 0; r < kSymR; ++r) {
        if constexpr (TS) {
          arg[r] = fma(-dt[r], dt[r], -r2[r]);
          dt2[r] = arg[r];
        } else {
          dt2[r] = dt[r] * dt[r];
          arg[r] = fma(k.ctL, dt2[r], -r2[r]);
        }
      }
      exp_l_batch<CHECK>(arg, e, tab);
#pragma unroll
      for (int r = 0; r < kSymR; ++r) {
        if constexpr (VALID) e[r] = (cv && rv[r]) ? e[r] : 0.0;
        racc[r][0] += e[r];
        if constexpr (GRAD) {
          racc[r][1] = fma(e[r], r2[r], racc[r][1]);
          racc[r][2] = fma(e[r], dt2[r], racc[r][2]);
        }
      }
      if constexpr (SYM) {
        cp[q][0] = (e[0] + e[1]) + (e[2] + e[3]);
        if constexpr (GRAD) {
          cp[q][1] = fma(e[3], r2[3], fma(e[2], r2[2], fma(e[1], r2[1], e[0] * r2[0])));
          cp[q][2] = fma(e[3], dt2[3], fma(e[2], dt2[2], fma(e[1], dt2[1], e[0] * dt2[0])));
        }
      }
    }
    if constexpr (TR != 0) {
#pragma unroll
      for (int r = 0; r < kSymR; ++r) arg[r] = fma(k.nomL, dt[r], k.chS * r2[r]);
      exp_l_batch<CHECK>(arg, e, tab);
#pragma unroll
      for (int r = 0; r < kSymR; ++r) {
        if constexpr (TR == 2) e[r] = (tj < ti[r]) ? e[r] : 0.0;
        if constexpr (VALID) e[r] = (cv && rv[r]) ? e[r] : 0.0;
        racc[r][T0] += e[r];
        if constexpr (GRAD) {
          racc[r][4] = fma(e[r], dt[r], racc[r][4]);
          racc[r][5] = fma(e[r], r2[r], racc[r][5]);
        }
      }
    }
  }
}

// Reduce-scatter of the kSymG x NSC column partials over the 32 lanes. Slot
// q of a lane holds column q ^ perm, where perm takes its bits from lane bits
// 4 (and 3): the first xor steps then always keep the low slots and send the
// high ones, and the remaining steps finish the butterfly. Every lane ends
// with the total of column `perm` (all copies bitwise identical: each add is
// commutative); one lane per column writes it.
template <bool GRAD, bool SYM, bool BG>
__device__ __forceinline__ void sym_reduce(int g, int perm, int col0,
                                           double (&cp)[kSymG][GRAD ? 3 : 1],
                                           double* __restrict__ s_col) {
  constexpr int NSC = GRAD ? 3 : 1;
  const int lane = threadIdx.x & 31;
  if constexpr (SYM && BG) {
    double v1[NSC];
    if constexpr (kSymG == 4) {
      double v2[2][NSC];
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
#pragma unroll
        for (int c = 0; c < NSC; ++c) {
          v2[qq][c] = cp[qq][c] + __shfl_xor_sync(0xffffffffu, cp[2 + qq][c], 16);
        }
      }
#pragma unroll
      for (int c = 0; c < NSC; ++c) v1[c] = v2[0][c] + __shfl_xor_sync(0xffffffffu, v2[1][c], 8);
#pragma unroll
      for (int off = 4; off > 0; off >>= 1) {
#pragma unroll
        for (int c = 0; c < NSC; ++c) v1[c] += __shfl_xor_sync(0xffffffffu, v1[c], off);
      }
      if ((lane & 7) == 0) {
#pragma unroll
        for (int c = 0; c < NSC; ++c) s_col[(col0 + kSymG * g + perm) * NSC + c] = v1[c];
      }
    } else {
#pragma unroll
      for (int c = 0; c < NSC; ++c) v1[c] = cp[0][c] + __shfl_xor_sync(0xffffffffu, cp[1][c], 16);
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) {
#pragma unroll
        for (int c = 0; c < NSC; ++c) v1[c] += __shfl_xor_sync(0xffffffffu, v1[c], off);
      }
      if ((lane & 15) == 0) {
#pragma unroll
        for (int c = 0; c < NSC; ++c) s_col[(col0 + kSymG * g + perm) * NSC + c] = v1[c];
      }
    }
  }
}

// One stage for one warp: 32 columns x this thread's 4 rows, in groups of
// kSymG columns, each group's column partials reduce-scattered right away.
// (Interleaving group g's reduction with group g+1's pair math doubles the
// live registers and spills; measured slower.)
template <bool GRAD, bool SYM, bool BG, int TR, bool CHECK, bool VALID, bool TS>
__device__ __forceinline__ void sym_block(const double* __restrict__ sx,
                                          const double* __restrict__ sy,
                                          const double* __restrict__ st, int col0, int cnt,
                                          const double (&xi)[kSymR], const double (&yi)[kSymR],
                                          const double (&ti)[kSymR], const bool (&rv)[kSymR],
                                          const PairConsts& k, const uint2* __restrict__ tab,
                                          double (&racc)[kSymR][GRAD ? kNSumGrad : kNSumVal],
                                          double* __restrict__ s_col) {
  const int lane = threadIdx.x & 31;
  const int perm = kSymG == 4 ? (((lane >> 4) & 1) << 1) | ((lane >> 3) & 1) : (lane >> 4) & 1;
#pragma unroll kGUnroll
  for (int g = 0; g < 32 / kSymG; ++g) {
    double cp[kSymG][GRAD ? 3 : 1];
    sym_pairs<GRAD, SYM, BG, TR, CHECK, VALID, TS>(g, perm, sx, sy, st, col0, cnt, xi, yi, ti, rv,
                                                   k, tab, racc, cp);
    sym_reduce<GRAD, SYM, BG>(g, perm, col0, cp, s_col);
  }
}

// ---------------------------------------------------------------------------
// Far tier (FP32): stages whose every pair has a background (and, if live,
// trigger) exponent below -A (A = 40, e < 4.3e-18) on the tile/stage bounding
// boxes. Their terms are below 2^-57 of the self term that every S_B holds,
// so they are evaluated in FP32 (ex2.approx on the MUFU pipe, FP32 FMA pipe)
// instead of FP64; the FP64 pipe keeps every term that can reach the sums'
// precision. Relative error of a far term <= ~4% (FP32 coordinates, guarded
// on the host), i.e. <= 2e-19 absolute per pair: far below the 1e-10 / 1e-8
// tolerances. Coordinates: xf = (x - x0) sxf, tf = (t - t0) stf
// with sxf = 1/(tauX sqrt(2 ln2)), stf = 1/(tauT sqrt(2 ln2)), so the
// background exponent in log2 units is -(dxf^2 + dyf^2 + dtf^2).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float ex2f(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Packed FP32x2 arithmetic (sm_100 FADD2 / FMUL2 / FFMA2): rows (0,1) and
// (2,3) share each instruction, halving the far tier's issue slots.
struct f2 {
  uint64_t v;
};

__device__ __forceinline__ f2 pk2(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo2(f2 a) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a.v));
  return lo;
}
__device__ __forceinline__ float hi2(f2 a) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a.v));
  return hi;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return d;
}
__device__ __forceinline__ f2 ex2x2(f2 a) { return pk2(ex2f(lo2(a)), ex2f(hi2(a))); }

// rows are held as two packed pairs: P = 0 -> rows (0, 1), P = 1 -> rows (2, 3)
template <bool GRAD, bool BG, bool TR>
__device__ __forceinline__ void far_pairs(int g, int perm, const float* __restrict__ sx,
                                          const float* __restrict__ sy,
                                          const float* __restrict__ st, int col0,
                                          const f2 (&xi)[2], const f2 (&yi)[2],
                                          const f2 (&ti)[2], f2 c1, f2 c2,
                                          f2 (&rf)[2][GRAD ? kNSumGrad : kNSumVal],
                                          float (&cp)[kSymG][GRAD ? 3 : 1]) {
  constexpr int T0 = GRAD ? 3 : 1;
#pragma unroll
  for (int q = 0; q < kSymG; ++q) {
    const int j = col0 + kSymG * g + (q ^ perm);
    const float xs = sx[j], ys = sy[j], ts = st[j];
    const f2 xj = pk2(xs, xs), yj = pk2(ys, ys), tj = pk2(ts, ts);
    f2 dt[2], r2[2], dt2[2], e[2];
#pragma unroll
    for (int P = 0; P < 2; ++P) {
      const f2 dx = sub2(xi[P], xj);
      const f2 dy = sub2(yi[P], yj);
      dt[P] = sub2(ti[P], tj);
      r2[P] = fma2(dx, dx, mul2(dy, dy));
    }
    if constexpr (BG) {
#pragma unroll
      for (int P = 0; P < 2; ++P) {
        dt2[P] = mul2(dt[P], dt[P]);
        const f2 sum = add2(r2[P], dt2[P]);
        e[P] = pk2(ex2f(-lo2(sum)), ex2f(-hi2(sum)));  // (negation folds into MUFU)
        rf[P][0] = add2(rf[P][0], e[P]);
        if constexpr (GRAD) {
          rf[P][1] = fma2(e[P], r2[P], rf[P][1]);
          rf[P][2] = fma2(e[P], dt2[P], rf[P][2]);
        }
      }
      const f2 es = add2(e[0], e[1]);  // (e0 + e2, e1 + e3)
      cp[q][0] = lo2(es) + hi2(es);
      if constexpr (GRAD) {
        const f2 wr = fma2(e[1], r2[1], mul2(e[0], r2[0]));
        const f2 wt = fma2(e[1], dt2[1], mul2(e[0], dt2[0]));
        cp[q][1] = lo2(wr) + hi2(wr);
        cp[q][2] = lo2(wt) + hi2(wt);
      }
    }
    if constexpr (TR) {  // unmasked: every source strictly earlier than every row
#pragma unroll
      for (int P = 0; P < 2; ++P) {
        const f2 et = ex2x2(fma2(c1, dt[P], mul2(c2, r2[P])));
        rf[P][T0] = add2(rf[P][T0], et);
        if constexpr (GRAD) {
          rf[P][4] = fma2(et, dt[P], rf[P][4]);
          rf[P][5] = fma2(et, r2[P], rf[P][5]);
        }
      }
    }
  }
}

// One far stage for one warp: 32 columns x this lane's 4 rows in FP32x2.
// Row sums stay in FP32 registers for the whole item (every far term is
// below 2^-57 of a row's self term, so FP32 accumulation error is
// irrelevant); column partials are reduce-scattered with FP32 shuffles
// (lane-permuted order, see sym_reduce) and stored to s_col in the FP64
// path's units for the fixed-point flush.
template <bool GRAD, bool BG, bool TR>
__device__ __forceinline__ void far_stage(const float* __restrict__ sx, const float* __restrict__ sy,
                                          const float* __restrict__ st, int col0,
                                          const f2 (&px)[2], const f2 (&py)[2],
                                          const f2 (&pt)[2], f2 c1, f2 c2,
                                          const double (&cscale)[3],
                                          f2 (&rf)[2][GRAD ? kNSumGrad : kNSumVal],
                                          double* __restrict__ s_col) {
  constexpr int NSC = GRAD ? 3 : 1;
  const int lane = threadIdx.x & 31;
  const int perm = (((lane >> 4) & 1) << 1) | ((lane >> 3) & 1);
  static_assert(kSymG == 4, "far tier assumes 4-column groups");
#pragma unroll 1
  for (int g = 0; g < 32 / kSymG; ++g) {
    float cp[kSymG][NSC];
    far_pairs<GRAD, BG, TR>(g, perm, sx, sy, st, col0, px, py, pt, c1, c2, rf, cp);
    if constexpr (BG) {
      float v2[2][NSC], v1[NSC];
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
#pragma unroll
        for (int c = 0; c < NSC; ++c) {
          v2[qq][c] = cp[qq][c] + __shfl_xor_sync(0xffffffffu, cp[2 + qq][c], 16);
        }
      }
#pragma unroll
      for (int c = 0; c < NSC; ++c) v1[c] = v2[0][c] + __shfl_xor_sync(0xffffffffu, v2[1][c], 8);
#pragma unroll
      for (int off = 4; off > 0; off >>= 1) {
#pragma unroll
        for (int c = 0; c < NSC; ++c) v1[c] += __shfl_xor_sync(0xffffffffu, v1[c], off);
      }
      if ((lane & 7) == 0) {
#pragma unroll
        for (int c = 0; c < NSC; ++c) {
          s_col[(col0 + kSymG * g + perm) * NSC + c] = static_cast<double>(v1[c]) * cscale[c];
        }
      }
    }
  }
}

template <bool GRAD, bool SYM, bool CHECK, bool VALID, bool BGONLY = false>
__device__ __forceinline__ void sym_dispatch(bool bg, int tr, const double* sx, const double* sy,
                                             const double* st, int col0, int cnt,
                                             const double (&xi)[kSymR], const double (&yi)[kSymR],
                                             const double (&ti)[kSymR], const bool (&rv)[kSymR],
                                             const PairConsts& k, const uint2* tab,
                                             double (&racc)[kSymR][GRAD ? kNSumGrad : kNSumVal],
                                             double* s_col) {
#define STHK_SYM_CALL(B, T) \
  sym_block<GRAD, SYM, B, T, CHECK, VALID, BGONLY>(sx, sy, st, col0, cnt, xi, yi, ti, rv, k, tab, racc, s_col)
  if constexpr (BGONLY) {  // (the plan guarantees no live trigger term)
    if (bg) STHK_SYM_CALL(true, 0);
    return;
  }
  if (bg) {
    if (tr == 0) STHK_SYM_CALL(true, 0);
    else if (tr == 1) STHK_SYM_CALL(true, 1);
    else STHK_SYM_CALL(true, 2);
  } else {
    if (tr == 1) STHK_SYM_CALL(false, 1);
    else if (tr == 2) STHK_SYM_CALL(false, 2);
  }
#undef STHK_SYM_CALL
}

#ifndef STHK_SYMBG_MINB
#define STHK_SYMBG_MINB 4  // trigger-free variant: fewer registers, 4 CTAs per SM
#endif

// BGONLY: the trigger-free variant for the background-only list (stages of
// sources earlier than t_tile_first - dT, never the diagonal stage): no
// trigger code paths, so it fits 128 registers and 4 CTAs per SM; it stores
// only background (fixed-point) row sums.
template <bool GRAD, bool BGONLY = false>
__global__ void __launch_bounds__(kTM, BGONLY ? STHK_SYMBG_MINB : STHK_SYM_MINB)
    sym_kernel(const PairArgs a) {
  constexpr int NS = GRAD ? kNSumGrad : kNSumVal;
  constexpr int NSC = GRAD ? 3 : 1;
  __shared__ __align__(128) double s_src[2][3][kTS];
  extern __shared__ __align__(128) uint2 s_tab[];  // kExpTableSize entries (dynamic)
  __shared__ double s_col[kTS * NSC];
  __shared__ double s_red[4][NS][kTM];
  __shared__ __align__(32) double4 s_box[2];  // bounding box of the staged source tile
  __shared__ __align__(16) double2 s_tr[2];   // its first / last time (BGONLY: the staged times are scaled)
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ int s_item[2];
  // BGONLY stages carry tile-relative scaled times (PairArgs::tsl)
  const double* __restrict__ src_t = BGONLY ? a.tsl : a.t;
  constexpr uint32_t kTrBytesS = BGONLY ? sizeof(double2) : 0;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  __shared__ unsigned long long s_cta_t0;  // (development trace)
  if (a.trace && tid == 0) s_cta_t0 = global_ns();
  if (tid == 0) {
    stamp_min(a.tstamp, 0);
    stamp_min(a.tstamp, 2);
  }
  __shared__ __align__(8) uint64_t s_tbar;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_init(&s_tbar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {  // the exp table: one 16 KB bulk copy (L2-resident source)
    mbar_arrive_expect_tx(&s_tbar, kTabBytes);
    tma_load_1d(s_tab, kExpTable, kTabBytes, &s_tbar);
  }
  mbar_wait(&s_tbar, 0);

  // (launched by a programmatic edge from the plan: wait for its work lists
  // and counters -- a no-op otherwise)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n_pre = (!BGONLY && a.pre_items) ? *a.pre_n_items : 0;
  const int n_items = *a.n_items + n_pre;
  const int64_t n = a.n;
  uint32_t phase = 0;
  // ordered pairs covered (bg, trigger, any) and work executed (background
  // exps, pair geometries, symmetric pairs with a column accumulation)
  unsigned long long cBg = 0, cTr = 0, cAny = 0, xBg = 0, xGeo = 0, xSym = 0;

  for (int iter = 0;; ++iter) {
    if (tid == 0) s_item[iter & 1] = next_item(a.work_counter, iter);
    __syncthreads();
    const int item = s_item[iter & 1];
    if (item >= n_items) break;
    __shared__ unsigned long long s_trace_t0;  // (development trace: kept out of registers)
    if (a.trace && tid == 0) s_trace_t0 = global_ns();

    // (merged lists: the trigger-free items first, the general items after)
    const bool pre = BGONLY || item < n_pre;
    const int2 it = item < n_pre ? a.pre_items[item] : a.items[item - n_pre];
    const int tile = it.x, chunk = it.y;
    const int2 rg = item < n_pre ? a.pre_ranges[tile] : a.ranges[tile];
    const int sc = item < n_pre ? a.pre_sc : a.sc;
    const int64_t first = static_cast<int64_t>(tile) * kTM;
    const int64_t last = min(first + kTM, n) - 1;
    const int rows_real = static_cast<int>(last - first + 1);
    const double tmin = a.t[first], tmax = a.t[last];
    const double4 bt = a.tile_box[tile];
    double xi[kSymR], yi[kSymR], ti[kSymR];
    bool rv[kSymR];
#pragma unroll
    for (int r = 0; r < kSymR; ++r) {
      const int64_t row = first + lane + 32 * r;
      xi[r] = a.xs[row];
      yi[r] = a.ys[row];
      ti[r] = BGONLY ? a.tsl[row] : a.t[row];
      rv[r] = row < n;
    }
    // Background row sums live in registers for the whole item; the trigger
    // row sums (rarely active) are parked in this thread's s_red slots
    // between trigger stages so the background-only loops keep their
    // registers for ILP.
    constexpr int NB = GRAD ? 3 : 1;
    double racc[kSymR][NS];
#pragma unroll
    for (int r = 0; r < kSymR; ++r) {
#pragma unroll
      for (int q = 0; q < NS; ++q) racc[r][q] = 0.0;
#pragma unroll
      for (int q = NB; q < NS; ++q) s_red[warp][q][lane + 32 * r] = 0.0;
    }

    int s_begin = max(rg.x, chunk * sc);
    s_begin -= s_begin % kTS;
    const int s_end = min(rg.y, (chunk + 1) * sc);
    const int nst = (s_end - s_begin + kTS - 1) / kTS;

    constexpr uint32_t kStageBytes = kTS * sizeof(double);
    if (tid == 0 && nst > 0) {
      mbar_arrive_expect_tx(&s_bar[0], 3 * kStageBytes + kBoxBytes + kTrBytesS);
      tma_load_1d(&s_box[0], a.tile_box + s_begin / kTS, kBoxBytes, &s_bar[0]);
      if constexpr (BGONLY) tma_load_1d(&s_tr[0], a.tile_trange + s_begin / kTS, kTrBytesS, &s_bar[0]);
      tma_load_1d(s_src[0][0], a.xs + s_begin, kStageBytes, &s_bar[0]);
      tma_load_1d(s_src[0][1], a.ys + s_begin, kStageBytes, &s_bar[0]);
      tma_load_1d(s_src[0][2], src_t + s_begin, kStageBytes, &s_bar[0]);
    }
    for (int s = 0; s < nst; ++s) {
      const int buf = s & 1;
      // every thread is done with stage s-1 (its buffer and s_col)
      __syncthreads();
      if (tid == 0 && s + 1 < nst) {
        const int nb = buf ^ 1;
        const int64_t s0n = s_begin + static_cast<int64_t>(s + 1) * kTS;
        mbar_arrive_expect_tx(&s_bar[nb], 3 * kStageBytes + kBoxBytes + kTrBytesS);
        tma_load_1d(&s_box[nb], a.tile_box + s0n / kTS, kBoxBytes, &s_bar[nb]);
        if constexpr (BGONLY) tma_load_1d(&s_tr[nb], a.tile_trange + s0n / kTS, kTrBytesS, &s_bar[nb]);
        tma_load_1d(s_src[nb][0], a.xs + s0n, kStageBytes, &s_bar[nb]);
        tma_load_1d(s_src[nb][1], a.ys + s0n, kStageBytes, &s_bar[nb]);
        tma_load_1d(s_src[nb][2], src_t + s0n, kStageBytes, &s_bar[nb]);
      }
      const int64_t s0 = s_begin + static_cast<int64_t>(s) * kTS;
      const int cnt = static_cast<int>(min(static_cast<int64_t>(kTS), n - s0));
      const bool diag = s0 == first;
      mbar_wait(&s_bar[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
      // stage metadata from the staged copy (no global-memory round trip)
      const double4 bs = s_box[buf];
      const double smin = BGONLY ? s_tr[buf].x : s_src[buf][2][0];
      const double smax = BGONLY ? s_tr[buf].y : s_src[buf][2][cnt - 1];

      const bool bg = !a.bg_off && (!a.bg_diag_only || diag || pre) &&
                      !(smin > tmax + a.k.dB || smax < tmin - a.k.dB);
      int tr;
      if (pre || a.tr_off || smin >= tmax || smax < tmin - a.k.dT) tr = 0;
      else if (smax < tmin) tr = 1;
      else tr = 2;
      const double dxm = fmax(bt.y - bs.x, bs.y - bt.x);
      const double dym = fmax(bt.w - bs.z, bs.w - bt.z);
      const double r2m = dxm * dxm + dym * dym;
      const double dtm = fmax(tmax - smin, smax - tmin);
      const bool safe = (!bg || a.k.cxL * r2m + a.k.ctL * (dtm * dtm) > kSafeExpL) &&
                        (!tr || a.k.nomL * dtm + a.k.chL * r2m > kSafeExpL);

      const double* sx = s_src[buf][0];
      const double* sy = s_src[buf][1];
      const double* st = s_src[buf][2];
      const int col0 = warp * 32;
      // BGONLY: row times relative to this stage's tile origin (scaled), so
      // dts = tv - tsl_j; otherwise the raw times
      double tsh[kSymR];
      if constexpr (BGONLY) {
        const double D = (tmin - smin) * a.stl;
#pragma unroll
        for (int r = 0; r < kSymR; ++r) tsh[r] = ti[r] + D;
      }
      const double(&tv)[kSymR] = BGONLY ? tsh : ti;
      auto pass = [&](bool pbg, int ptr) {
        if (diag) {
          sym_dispatch<GRAD, false, true, true, BGONLY>(pbg, ptr, sx, sy, st, col0, cnt, xi, yi, tv,
                                                        rv, a.k, s_tab, racc, s_col);
        } else if (rows_real < kTM) {
          sym_dispatch<GRAD, true, true, true, BGONLY>(pbg, ptr, sx, sy, st, col0, cnt, xi, yi, tv,
                                                       rv, a.k, s_tab, racc, s_col);
        } else if (safe) {
          sym_dispatch<GRAD, true, false, false, BGONLY>(pbg, ptr, sx, sy, st, col0, cnt, xi, yi,
                                                         tv, rv, a.k, s_tab, racc, s_col);
        } else {
          sym_dispatch<GRAD, true, true, false, BGONLY>(pbg, ptr, sx, sy, st, col0, cnt, xi, yi, tv,
                                                        rv, a.k, s_tab, racc, s_col);
        }
      };
      auto load_tr = [&] {
#pragma unroll
        for (int r = 0; r < kSymR; ++r) {
#pragma unroll
          for (int q = NB; q < NS; ++q) racc[r][q] = s_red[warp][q][lane + 32 * r];
        }
      };
      auto store_tr = [&] {
#pragma unroll
        for (int r = 0; r < kSymR; ++r) {
#pragma unroll
          for (int q = NB; q < NS; ++q) s_red[warp][q][lane + 32 * r] = racc[r][q];
        }
      };
#if STHK_SPLIT_TRIG
      // Background and trigger in two passes over the stage: the trigger sums
      // are live only in the second (fewer registers, more resident warps);
      // every sum sees the same terms in the same order, so the result is
      // bitwise that of one fused pass.
      if (bg) pass(true, 0);
      if (tr) {
        load_tr();
        pass(false, tr);
        store_tr();
      }
#else
      if (tr) load_tr();
      pass(bg, tr);
      if (tr) store_tr();
#endif
      if (!diag && bg) {  // (never in a trigger-only sweep)
        // column sums of source tile J: one fixed-point flush per column.
        // Warp w owns columns 32w..32w+31 (it wrote their s_col entries), so
        // it flushes them itself after a warp-level sync: no CTA barrier.
        __syncwarp();
        const int jc = col0 + lane;
        const int64_t col = s0 + jc;
#pragma unroll
        for (int c = 0; c < NSC; ++c) {
          double cv = s_col[jc * NSC + c], cq = a.fxq[c];
          if constexpr (BGONLY && GRAD) {  // third sum: -(sum e * exponent) - S_Br = sum e dts^2
            if (c == 2) {
              cv = -cv - s_col[jc * NSC + 1];
              cq = a.fxq[1];
            }
          }
          fx_add(a.fx + static_cast<size_t>(2 * c) * a.npad + col,
                 a.fx + static_cast<size_t>(2 * c + 1) * a.npad + col, cv * cq);
        }
      }
      if (tid == 0) {
        const unsigned long long pr = static_cast<unsigned long long>(cnt) * rows_real;
        if (diag) {
          if (bg) cBg += pr;
          if (tr) cTr += pr;
          if (bg || tr) cAny += pr;
          if (bg) xBg += pr;
          if (bg || tr) xGeo += pr;
        } else {
          if (bg) cBg += 2 * pr;
          if (tr) cTr += pr;
          cAny += bg ? 2 * pr : (tr ? pr : 0);
          if (bg) xBg += pr;
          if (bg) xSym += pr;
          if (bg || tr) xGeo += pr;
        }
      }
    }

    // combine the 4 warps' row partials in a fixed order, then flush
#pragma unroll
    for (int r = 0; r < kSymR; ++r) {
#pragma unroll
      for (int q = 0; q < NB; ++q) s_red[warp][q][lane + 32 * r] = racc[r][q];
    }
    __syncthreads();
    double v[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      v[q] = ((s_red[0][q][tid] + s_red[1][q][tid]) + s_red[2][q][tid]) + s_red[3][q][tid];
    }
    if (pre) {  // background rows only (no trigger partials)
      if (first + tid < n && !a.bg_off) {
#pragma unroll
        for (int q = 0; q < NB; ++q) {
          double rv_ = v[q], rq = a.fxq[q];
          if constexpr (BGONLY && GRAD) {  // (as the column flush)
            if (q == 2) {
              rv_ = -v[2] - v[1];
              rq = a.fxq[1];
            }
          }
          fx_add(a.fx + static_cast<size_t>(2 * q) * a.npad + first + tid,
                 a.fx + static_cast<size_t>(2 * q + 1) * a.npad + first + tid, rv_ * rq);
        }
      }
    } else {
      store_row_sums<GRAD>(a, chunk, first + tid, v);
    }
    if (a.trace && tid == 0) trace_item(a, item, nst, s_begin <= first && first < s_end, s_trace_t0);
  }

  // (no more items for this CTA: a programmatically dependent kernel may
  // start launching -- it still waits for this grid's completion)
  asm volatile("griddepcontrol.launch_dependents;");
  if (tid == 0) {  // the last CTA out re-arms the work counter for the next launch
    __threadfence();
    if (atomicAdd(a.done_counter, 1u) == gridDim.x - 1) {
      *a.work_counter = 0;
      *a.done_counter = 0u;
    }
    if (a.trace) trace_cta(a.trace, a.trace_cap, a.trace_kernel, s_cta_t0);
    stamp_max(a.tstamp, 3);
  }
  if (tid == 0 && a.pair_counts) {
    atomicAdd(&a.pair_counts[0], cBg);
    atomicAdd(&a.pair_counts[1], cTr);
    atomicAdd(&a.pair_counts[2], cAny);
    atomicAdd(&a.pair_counts[3], xBg);
    atomicAdd(&a.pair_counts[4], xGeo);
    atomicAdd(&a.pair_counts[5], xSym);
  }
}

// ---------------------------------------------------------------------------
// Far kernel (kSym far tier): the far work list -- source stages whose every
// pair with the row tile is at least tfar earlier, so every background and
// trigger exponent is below -A (A = 40) -- in FP32 on the FP32 / MUFU pipes,
// with far fewer registers than the FP64 kernel (more resident warps).
// Same structure as sym_kernel: persistent CTAs of 128 rows, bulk-copied
// 128-source stages, symmetric background (rows and columns), unmasked
// trigger (every far source is strictly earlier). Background sums go to the
// same fixed-point accumulators; trigger partials to their own per-(chunk,
// row) buffer (tpart_far), summed by finalize after the near ones.
// ---------------------------------------------------------------------------
#ifndef STHK_FAR_MINB
#define STHK_FAR_MINB 5  // 96 registers, no spill (6: 80 registers with a 40 B spill; same speed)
#endif

template <bool GRAD>
__global__ void __launch_bounds__(kTM, STHK_FAR_MINB) far_kernel(const PairArgs a) {
  constexpr int NS = GRAD ? kNSumGrad : kNSumVal;
  constexpr int NSC = GRAD ? 3 : 1;
  constexpr int NB = GRAD ? 3 : 1;
  constexpr int NT = GRAD ? 3 : 1;
  __shared__ __align__(128) float s_srcf[2][3][kTS];
  __shared__ __align__(16) double2 s_tr[2];
  __shared__ double s_col[kTS * NSC];
  __shared__ float s_red[4][NS][kTM];
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ int s_item[2];

  const int tid = threadIdx.x;
  __shared__ unsigned long long s_cta_t0;  // (development trace)
  if (a.trace && tid == 0) s_cta_t0 = global_ns();
  const int lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    stamp_min(a.tstamp, 0);
    stamp_min(a.tstamp, 2);
  }
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();

  const int n_items = *a.n_items;
  uint32_t phase = 0;
  unsigned long long cBg = 0, cTr = 0, cAny = 0, xBg = 0, xGeo = 0, xSym = 0, xFar = 0;
  const double cscale[3] = {1.0, a.k.fkr, a.k.fkt2};
  const double tscale[3] = {1.0, a.k.fkt1, a.k.fkr};  // S_T, S_Tt, S_Tr
  const f2 c1 = pk2(a.k.fc1, a.k.fc1), c2 = pk2(a.k.fc2, a.k.fc2);
  constexpr uint32_t kStageBytesF = kTS * sizeof(float);
  constexpr uint32_t kTrBytes = sizeof(double2);

  for (int iter = 0;; ++iter) {
    if (tid == 0) s_item[iter & 1] = next_item(a.work_counter, iter);
    __syncthreads();
    const int item = s_item[iter & 1];
    if (item >= n_items) break;
    __shared__ unsigned long long s_trace_t0;  // (development trace: kept out of registers)
    if (a.trace && tid == 0) s_trace_t0 = global_ns();

    const int2 it = a.items[item];
    const int tile = it.x, chunk = it.y;
    const int2 rg = a.ranges[tile];
    const int64_t first = static_cast<int64_t>(tile) * kTM;  // (full tiles only)
    const double tmin = a.t[first], tmax = a.t[first + kTM - 1];
    float xr[kSymR], yr[kSymR], tr_[kSymR];
#pragma unroll
    for (int r = 0; r < kSymR; ++r) {
      const int64_t row = first + lane + 32 * r;
      xr[r] = a.xf[row];
      yr[r] = a.yf[row];
      tr_[r] = a.tf[row];
    }
    const f2 px[2] = {pk2(xr[0], xr[1]), pk2(xr[2], xr[3])};
    const f2 py[2] = {pk2(yr[0], yr[1]), pk2(yr[2], yr[3])};
    const f2 ptr[2] = {pk2(tr_[0], tr_[1]), pk2(tr_[2], tr_[3])};
    f2 rf[2][NS];
#pragma unroll
    for (int P = 0; P < 2; ++P) {
#pragma unroll
      for (int q = 0; q < NS; ++q) rf[P][q] = pk2(0.0f, 0.0f);
    }

    int s_begin = max(rg.x, chunk * a.sc);
    s_begin -= s_begin % kTS;
    const int s_end = min(rg.y, (chunk + 1) * a.sc);
    const int nst = (s_end - s_begin + kTS - 1) / kTS;
    if (tid == 0 && nst > 0) {
      mbar_arrive_expect_tx(&s_bar[0], 3 * kStageBytesF + kTrBytes);
      tma_load_1d(&s_tr[0], a.tile_trange + s_begin / kTS, kTrBytes, &s_bar[0]);
      tma_load_1d(s_srcf[0][0], a.xf + s_begin, kStageBytesF, &s_bar[0]);
      tma_load_1d(s_srcf[0][1], a.yf + s_begin, kStageBytesF, &s_bar[0]);
      tma_load_1d(s_srcf[0][2], a.tf + s_begin, kStageBytesF, &s_bar[0]);
    }
    for (int s = 0; s < nst; ++s) {
      const int buf = s & 1;
      __syncthreads();  // every warp is done with stage s-1's buffer
      if (tid == 0 && s + 1 < nst) {
        const int nb = buf ^ 1;
        const int64_t s0n = s_begin + static_cast<int64_t>(s + 1) * kTS;
        mbar_arrive_expect_tx(&s_bar[nb], 3 * kStageBytesF + kTrBytes);
        tma_load_1d(&s_tr[nb], a.tile_trange + s0n / kTS, kTrBytes, &s_bar[nb]);
        tma_load_1d(s_srcf[nb][0], a.xf + s0n, kStageBytesF, &s_bar[nb]);
        tma_load_1d(s_srcf[nb][1], a.yf + s0n, kStageBytesF, &s_bar[nb]);
        tma_load_1d(s_srcf[nb][2], a.tf + s0n, kStageBytesF, &s_bar[nb]);
      }
      const int64_t s0 = s_begin + static_cast<int64_t>(s) * kTS;
      mbar_wait(&s_bar[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
      const double smin = s_tr[buf].x, smax = s_tr[buf].y;
      // live in FP32 (the far tier's exact cull; all sources strictly earlier)
      const bool bg = !a.bg_off && !(smin > tmax + a.k.dBf || smax < tmin - a.k.dBf);
      const bool trg = !(smin >= tmax || smax < tmin - a.k.dTf);
      // row times re-based onto the source tile's origin (tf is tile-relative)
      const float dtile = static_cast<float>((tmin - smin) * a.k.fstf);
      const f2 dd = pk2(dtile, dtile);
      const f2 pt[2] = {add2(ptr[0], dd), add2(ptr[1], dd)};
      const float* sx = s_srcf[buf][0];
      const float* sy = s_srcf[buf][1];
      const float* st = s_srcf[buf][2];
      const int col0 = warp * 32;
      if (bg && trg) far_stage<GRAD, true, true>(sx, sy, st, col0, px, py, pt, c1, c2, cscale, rf, s_col);
      else if (bg) far_stage<GRAD, true, false>(sx, sy, st, col0, px, py, pt, c1, c2, cscale, rf, s_col);
      else if (trg) far_stage<GRAD, false, true>(sx, sy, st, col0, px, py, pt, c1, c2, cscale, rf, s_col);
      if (bg) {  // this warp's 32 columns: fixed-point flush (no CTA barrier)
        __syncwarp();
        const int jc = col0 + lane;
        const int64_t col = s0 + jc;
#pragma unroll
        for (int c = 0; c < NSC; ++c) {
          fx_add(a.fx + static_cast<size_t>(2 * c) * a.npad + col,
                 a.fx + static_cast<size_t>(2 * c + 1) * a.npad + col,
                 s_col[jc * NSC + c] * a.fxq[c]);
        }
      }
      if (tid == 0) {
        const unsigned long long pr = static_cast<unsigned long long>(kTS) * kTM;
        if (bg) cBg += 2 * pr;
        if (trg) cTr += pr;
        cAny += bg ? 2 * pr : (trg ? pr : 0);
        if (bg) xBg += pr;
        if (bg) xSym += pr;
        if (bg || trg) {
          xGeo += pr;
          xFar += pr;
        }
      }
    }

    // rows: combine the 4 warps' FP32 partials in a fixed order, then store
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      s_red[warp][q][lane] = lo2(rf[0][q]);
      s_red[warp][q][lane + 32] = hi2(rf[0][q]);
      s_red[warp][q][lane + 64] = lo2(rf[1][q]);
      s_red[warp][q][lane + 96] = hi2(rf[1][q]);
    }
    __syncthreads();
    // (lane l's packed pairs hold rows l, l+32 | l+64, l+96 of the tile)
    const int64_t row = first + tid;
    float v[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      v[q] = ((s_red[0][q][tid] + s_red[1][q][tid]) + s_red[2][q][tid]) + s_red[3][q][tid];
    }
    if (!a.bg_off) {
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        fx_add(a.fx + static_cast<size_t>(2 * q) * a.npad + row,
               a.fx + static_cast<size_t>(2 * q + 1) * a.npad + row,
               static_cast<double>(v[q]) * cscale[q] * a.fxq[q]);
      }
    }
    if (a.tpart) {  // (nullptr: the host proved every far trigger term culled)
      double* out = a.tpart + static_cast<size_t>(chunk) * NT * a.npad + row;
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        out[static_cast<size_t>(q) * a.npad] = static_cast<double>(v[NB + q]) * tscale[q];
      }
    }
    if (a.trace && tid == 0) trace_item(a, item, -1, 0, s_trace_t0);
  }

  if (tid == 0) {  // the last CTA out re-arms the work counter for the next launch
    __threadfence();
    if (atomicAdd(a.done_counter, 1u) == gridDim.x - 1) {
      *a.work_counter = 0;
      *a.done_counter = 0u;
    }
    if (a.trace) trace_cta(a.trace, a.trace_cap, a.trace_kernel, s_cta_t0);
    stamp_max(a.tstamp, 3);
  }
  if (tid == 0 && a.pair_counts) {
    atomicAdd(&a.pair_counts[0], cBg);
    atomicAdd(&a.pair_counts[1], cTr);
    atomicAdd(&a.pair_counts[2], cAny);
    atomicAdd(&a.pair_counts[3], xBg);
    atomicAdd(&a.pair_counts[4], xGeo);
    atomicAdd(&a.pair_counts[5], xSym);
    atomicAdd(&a.pair_counts[6], xFar);
  }
}

// Per 128-event tile bounding box of the (x, y) coordinates (params
// independent; computed once per load). Feeds the no-underflow proofs.
// Event load, pass 1 (one warp per 128-event tile): reads the tile from its
// source -- the caller's pinned host arrays over PCIe (zero-copy: this pass
// is the host-to-device copy) or the device arrays themselves after a
// cudaMemcpy -- writes the device copy, and computes the tile's bounding box
// and (first, last) time and the EventSet checks (types.hpp:85-109: finite,
// t >= 0, nondecreasing; the predecessor of each element from a shuffle, one
// source read per tile for the element before it). Also zeroes the pad tail
// and writes the tile pivots (PlanArgs::piv).
__global__ void tile_load_kernel(const double* __restrict__ sx, const double* __restrict__ sy,
                                 const double* __restrict__ st, double* __restrict__ x,
                                 double* __restrict__ y, double* __restrict__ t, int64_t n,
                                 int64_t npad, double4* box, double2* trange,
                                 double* __restrict__ piv, unsigned long long* bad, bool tiles) {
  // (tile_stats_kernel is launched programmatically behind this one)
  asm volatile("griddepcontrol.launch_dependents;");
  const bool copy = sx != x;
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid < npad - n) {  // pad tail [n, npad): never read as sources
    x[n + gid] = 0.0;
    y[n + gid] = 0.0;
    t[n + gid] = 0.0;
  }
  const int lane = threadIdx.x & 31;
  const int64_t tile = gid >> 5;
  const int64_t first = tile * kTS;
  if (first >= n) return;
  const int64_t last = min(first + kTS, n);
  double x0 = __longlong_as_double(0x7ff0000000000000LL), x1 = -x0, y0 = x0, y1 = -x0;
  double carry = (lane == 0 && first > 0) ? st[first - 1] : 0.0;  // element before the tile
  double tfirst = 0.0, tlast = 0.0;
  int64_t first_bad = INT64_MAX;
#pragma unroll
  for (int it = 0; it < kTS / 32; ++it) {
    const int64_t i = first + lane + 32 * it;
    const bool live = i < last;
    double xv = 0.0, yv = 0.0, tv = 0.0;
    if (live) {
      xv = sx[i];
      yv = sy[i];
      tv = st[i];
      if (copy) {
        x[i] = xv;
        y[i] = yv;
        t[i] = tv;
      }
      x0 = fmin(x0, xv);
      x1 = fmax(x1, xv);
      y0 = fmin(y0, yv);
      y1 = fmax(y1, yv);
    }
    const double up = __shfl_up_sync(0xffffffffu, tv, 1);
    const double prev = lane == 0 ? carry : up;
    carry = __shfl_sync(0xffffffffu, tv, 31);  // (lane 0 of the next round)
    const bool ok = isfinite(xv) && isfinite(yv) && isfinite(tv) && tv >= prev;
    if (live && !ok && i < first_bad) first_bad = i;
    if (it == 0) tfirst = __shfl_sync(0xffffffffu, tv, 0);
    const int64_t lk = last - 1 - first - 32 * it;  // lane holding t[last - 1] in this round
    const double tl = __shfl_sync(0xffffffffu, tv, static_cast<int>(lk < 0 ? 0 : (lk > 31 ? 31 : lk)));
    if (lk >= 0 && lk < 32) tlast = tl;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    first_bad = min(first_bad, static_cast<int64_t>(__shfl_xor_sync(
                                   0xffffffffu, static_cast<long long>(first_bad), off)));
    x0 = fmin(x0, __shfl_xor_sync(0xffffffffu, x0, off));
    x1 = fmax(x1, __shfl_xor_sync(0xffffffffu, x1, off));
    y0 = fmin(y0, __shfl_xor_sync(0xffffffffu, y0, off));
    y1 = fmax(y1, __shfl_xor_sync(0xffffffffu, y1, off));
  }
  if (lane == 0) {
    if (first_bad != INT64_MAX) atomicMin(bad, static_cast<unsigned long long>(first_bad));
    box[tile] = make_double4(x0, x1, y0, y1);
    trange[tile] = make_double2(tfirst, tlast);
    if (tiles) piv[tile] = tlast;  // (see Pivots)
  }
}

// Event load, pass 2 (one warp per tile, after pass 1): the remaining plan
// pivots, and the load statistics (kLoadStats) -- per tile one value per
// lane, reduced over the block in shared memory, then one device atomic per
// statistic and block (every value is >= 0, so its bit pattern orders like
// the double). The last block out hands the first bad index and the
// statistics to the host (mapped) and re-arms the device copies.
__global__ void tile_stats_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                  const double* __restrict__ t, int64_t n, const double4* box,
                                  const double2* trange, double* __restrict__ piv, bool tiles,
                                  unsigned long long* bad, unsigned int* done,
                                  unsigned long long* h_bad, double* h_stats,
                                  unsigned long long* __restrict__ dstats) {
  // (launched programmatically: wait for tile_load_kernel's device copy,
  // boxes and time ranges -- its launch latency is hidden)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ unsigned long long s_st[kLoadStats];
  for (int q = threadIdx.x; q < kLoadStats; q += blockDim.x) {
    s_st[q] = q < 3 ? 0ULL : 0x7ff0000000000000ULL;
  }
  __syncthreads();
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nt = (n + kTS - 1) / kTS;
  {  // pivots: +inf beyond the tiles (tile pivots), or strided t[k * stride]
    const int64_t stride = tiles ? kTS : pivot_stride(n), np = (n + stride - 1) / stride;
    for (int64_t k = gid; k < kPivots; k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      if (k >= np) piv[k] = __longlong_as_double(0x7ff0000000000000LL);
      else if (!tiles) piv[k] = t[k * stride];
    }
  }
  const int lane = threadIdx.x & 31;
  const int64_t tile = gid >> 5;
  if (tile < nt) {
    const double2 tr = trange[tile];
    if (lane == 0) {  // extents relative to event 0, the tile's time span
      const double4 b = box[tile];
      const double x00 = x[0], y00 = y[0];
      const double e[3] = {fmax(fabs(b.x - x00), fabs(b.y - x00)), fmax(fabs(b.z - y00), fabs(b.w - y00)),
                           tr.y - tr.x};
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        atomicMax(&s_st[q], static_cast<unsigned long long>(__double_as_longlong(fmax(e[q], 0.0))));
      }
    }
    // lanes 0..15: the gap a = lane + 1 stages ahead of the tile's first event
    // (t[first] - t[first - 128 a - 1]); lanes 16..31: the span of 2^L whole
    // tiles from this one, L = lane - 16 (whole: a partial last tile holds
    // fewer than 128 events, so its short span bounds nothing)
    double v = __longlong_as_double(0x7ff0000000000000LL);
    if (lane < kLoadAdj) {
      const int64_t a = lane + 1;
      if (tile >= a + 1) v = tr.x - trange[tile - a - 1].y;
    } else {
      const int64_t L = lane - kLoadAdj;
      if (L < kLoadSpan && (tile + (int64_t{1} << L)) * kTS <= n) {
        v = trange[tile + (int64_t{1} << L) - 1].y - tr.x;
      }
    }
    if (lane < kLoadAdj + kLoadSpan) {
      atomicMin(&s_st[3 + lane], static_cast<unsigned long long>(__double_as_longlong(fmax(v, 0.0))));
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < kLoadStats; q += blockDim.x) {
    if (q < 3) atomicMax(&dstats[q], s_st[q]);
    else atomicMin(&dstats[q], s_st[q]);
  }
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int q = threadIdx.x; q < kLoadStats; q += blockDim.x) {
    h_stats[q] = __longlong_as_double(static_cast<long long>(atomicAdd(&dstats[q], 0ULL)));
    dstats[q] = q < 3 ? 0ULL : 0x7ff0000000000000ULL;
  }
  if (threadIdx.x == 0) {
    *h_bad = atomicExch(bad, ~0ULL);
    *done = 0u;
  }
}

// Per-evaluation preparation, one pass over the (padded) events, each part
// optional:
//  * kSym coordinates: xs, ys = (x, y) * sx, so the symmetric kernels' squared
//    distance is already the background exponent's spatial part; the far
//    tier's FP32 copies xf, yf (relative to event 0) and tf (relative to the
//    first event of the event's own 128-tile), in log2-exponent units;
//  * zero the fixed-point background accumulators (6 words per event);
//  * the compensator terms (kernels.hpp:54-65 and their derivatives), which
//    depend only on (t, T, tauT, omega): comp[0] = Phi((T-t)/tauT) -
//    Phi(-t/tauT), comp[1] = (phi(z1) D + phi(z0) t) / tauT^2 (d Lambda / d tauT
//    = -mu0 comp[1]), comp[2] = expm1(-omega D), comp[3] = D exp(-omega D),
//    D = T - t; finalize combines them with mu0 and theta.
// One event's compensator terms (compensatorTerm, kernels.hpp:54-65, and its
// tauT / omega derivatives): shared by prep_kernel and the fused
// trigger-only finalize, so both produce the same bits.
__device__ __forceinline__ void comp_terms(double ti, double window_end, double tauT, double omega,
                                           double (&c)[4]) {
  const double D = window_end - ti;
  // normalCdf = 0.5 erfc(-z/sqrt2), kernels.hpp:21
  const double Phi1 = 0.5 * erfc(-(D / tauT) * kInvSqrt2);
  const double Phi0 = 0.5 * erfc(-(-ti / tauT) * kInvSqrt2);
  const double z1 = D / tauT, z0 = ti / tauT;
  const double phi1 = kInvSqrt2Pi * exp(-0.5 * z1 * z1);
  const double phi0 = kInvSqrt2Pi * exp(-0.5 * z0 * z0);
  c[0] = Phi1 - Phi0;
  c[1] = (phi1 * D + phi0 * ti) / (tauT * tauT);
  c[2] = expm1(-omega * D);
  // exp(-omega D) directly: 1 + expm1 cancels when omega D is large
  c[3] = D * exp(-omega * D);
}

__device__ __forceinline__ void prep_body(const PrepArgs& a, int64_t i) {
  if (i >= a.npad) return;
  const unsigned long long trace_t0 = (a.trace && threadIdx.x == 0) ? global_ns() : 0ULL;
  if (threadIdx.x == 0) stamp_min(a.tstamp, 0);
  if (a.xs) {
    const double xv = a.x[i], yv = a.y[i];  // (the pad tail of x, y, t is zero)
    a.xs[i] = xv * a.sx;
    a.ys[i] = yv * a.sx;
    if (a.tsl) a.tsl[i] = (a.t[i] - a.t[i - i % kTS]) * a.stl;
    if (a.xf) {
      a.xf[i] = static_cast<float>((xv - a.x[0]) * a.sxf);
      a.yf[i] = static_cast<float>((yv - a.y[0]) * a.sxf);
      a.tf[i] = static_cast<float>((a.t[i] - a.t[i - i % kTS]) * a.stf);
    }
  }
  if (a.fx) {
#pragma unroll
    for (int k = 0; k < 6; ++k) a.fx[static_cast<size_t>(k) * a.npad + i] = 0ULL;
  }
  if (a.comp && i < a.n) {
    double c[4];
    comp_terms(a.t[i], a.window_end, a.tauT, a.omega, c);
#pragma unroll
    for (int k = 0; k < 4; ++k) a.comp[static_cast<size_t>(k) * a.npad + i] = c[k];
  }
  if (a.trace && threadIdx.x == 0) trace_cta(a.trace, a.trace_cap, 5, trace_t0);
}

__global__ void prep_kernel(const PrepArgs a) {
  prep_body(a, static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x);
}

// Small sets, graph mode: the plan and the prep pass as one grid (block 0
// plans, the others prepare 1024 events each), so the pair kernel has a
// single predecessor and its programmatic edge holds: its CTAs launch while
// this grid runs and wait for it (griddepcontrol.wait).
__global__ void __launch_bounds__(1024) plan_prep_kernel(const PlanPrepArgs a) {
  asm volatile("griddepcontrol.launch_dependents;");
  if (blockIdx.x == 0) {
    plan_body(a.plan);
    return;
  }
  prep_body(a.prep, static_cast<int64_t>(blockIdx.x - 1) * 1024 + threadIdx.x);
}

// exp_l on a vector of natural-unit exponents (accuracy tests; the argument
// is scaled to L units by one multiply, as the pair kernels' constants are).
__global__ void exp_probe_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  extern __shared__ uint2 s_tab[];
  for (int i = threadIdx.x; i < kExpTableSize; i += blockDim.x) s_tab[i] = kExpTable[i];
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = exp_l<true>(x[i] * kExpL, s_tab);
}

// ---------------------------------------------------------------------------
// Finalize: per-row lambda / compensator / log / gradient, block partials.
// ---------------------------------------------------------------------------
// Fixed-order sum of the block partials by one 256-thread block: thread t
// sums blocks t, t+256, ... in order, then a fixed tree over the threads.
// Fixed-order sum of kNOut values over a 256-thread block: a butterfly
// within each warp (every lane ends with the same bits: each add is
// commutative), then the 8 warp totals in warp order. Two barriers instead
// of a shared-memory tree's eight.
__device__ __forceinline__ void block_sum8(double (&v)[kNOut], double (*s_w)[kNOut]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int q = 0; q < kNOut; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < kNOut; ++q) s_w[warp][q] = v[q];
  }
  __syncthreads();
  if (threadIdx.x < kNOut) {
    const int q = threadIdx.x;
    double r = s_w[0][q];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) r += s_w[w][q];
    v[0] = r;  // (thread q holds the block total of output q)
  }
  __syncthreads();
}

__device__ __forceinline__ void final_sum_block(const double* __restrict__ bp, int nblocks,
                                                double* out, double (*s_w)[kNOut]) {
  const int tid = threadIdx.x;
  double acc[kNOut];
#pragma unroll
  for (int q = 0; q < kNOut; ++q) acc[q] = 0.0;
  for (int b = tid; b < nblocks; b += 256) {
#pragma unroll
    for (int q = 0; q < kNOut; ++q) acc[q] += bp[static_cast<size_t>(b) * kNOut + q];
  }
  block_sum8(acc, s_w);
  if (tid < kNOut) out[tid] = acc[0];
}

// ---------------------------------------------------------------------------
// Trigger sums over each row's own time window (short windows: every tile
// spans more than dT = 709 / omega, beyond which every trigger term is +0).
// The tiled sweep gives a row all 128-256 sources of the stages its window
// touches; here a thread walks back from j = i - 1 while t_i - t_j <= dT, so
// the work is the pairs in the window only -- at Θ_post (ω = 1440, half a
// day) about ten per row instead of ~200 -- and every term that is not +0 is
// summed, as in the reference. Same term as the general kernel (exponent
// nomL dt + chS r2 on scaled coordinates, strict t_j < t_i), sums added in
// descending j. Every evaluation whose window qualifies -- full sweep or
// trigger-only, cached or not, any shard count, dense or culled -- takes this
// path, so those stay bitwise identical.
// ---------------------------------------------------------------------------
constexpr int kTrigRowsThreads = 256;
#ifndef STHK_TRIG_ROWS_W
#define STHK_TRIG_ROWS_W 4  // sources per step of the row-window walk
#endif
// sources a row's window can reach before its block's first row: a window
// holds at most 254 events (every tile spans more than it), plus the one
// just outside that ends the walk
constexpr int kTrigRowsBack = 256;

// Where trig_row_sums reads the events: global memory through L1 (the fused
// finalize), or a shared-memory copy of [base, ...) with the exp table
// (trig_rows_kernel: it runs beside the near kernel, whose shared-memory
// carveout leaves little L1). Same values either way, so the same bits.
struct RowSrcGlobal {
  const double* t;
  const double* x;
  const double* y;
  __device__ __forceinline__ double tt(int64_t j) const { return __ldg(t + j); }
  __device__ __forceinline__ double xx(int64_t j) const { return __ldg(x + j); }
  __device__ __forceinline__ double yy(int64_t j) const { return __ldg(y + j); }
  __device__ __forceinline__ const uint2* tab() const { return kExpTable; }
};
struct RowSrcShared {
  const double* t;
  const double* x;
  const double* y;
  int64_t base;
  const uint2* table;
  __device__ __forceinline__ double tt(int64_t j) const { return t[j - base]; }
  __device__ __forceinline__ double xx(int64_t j) const { return x[j - base]; }
  __device__ __forceinline__ double yy(int64_t j) const { return y[j - base]; }
  __device__ __forceinline__ const uint2* tab() const { return table; }
};

// Row i's trigger sums (S_T, and for GRAD S_Tt, S_Tr') over its window,
// written to trow; returns the pairs evaluated. Shared by trig_rows_kernel
// and the fused trigger-only finalize, so both produce the same bits.
template <bool GRAD, class Src>
__device__ __forceinline__ unsigned long long trig_row_sums(const TrigRowsArgs& a, const Src& src,
                                                            int64_t i, double (&st)[GRAD ? 3 : 1]) {
  unsigned long long pairs = 0;
  const double ti = src.tt(i), xi = src.xx(i), yi = src.yy(i);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  // kW sources per step (j, j - 1, ...), their exps in lockstep; a source
  // outside the window, tied with t_i or before index 0 adds an exact 0
  // (s + 0 == s: every sum >= 0), so the sums are those of the one-at-a-time
  // loop, bit for bit
  constexpr int kW = STHK_TRIG_ROWS_W;
  for (int64_t j = i - 1; j >= 0; j -= kW) {
    double dt[kW], r2[kW], x[kW], e[kW];
    bool v[kW];
#pragma unroll
    for (int w = 0; w < kW; ++w) {
      const int64_t jw = j - w >= 0 ? j - w : j;  // (no source: dt 0, masked)
      const double tj = j - w >= 0 ? src.tt(jw) : ti;
      dt[w] = ti - tj;
      v[w] = dt[w] > 0.0 && dt[w] <= a.dT;  // ties: strict t_j < t_i
      const double dx = xi - src.xx(jw), dy = yi - src.yy(jw);
      r2[w] = fma(dx, dx, dy * dy);
      x[w] = fma(a.nomL, dt[w], a.chS * r2[w]);
    }
    if (dt[0] > a.dT) break;
    exp_l_batch<true, kW>(x, e, src.tab());
#pragma unroll
    for (int w = 0; w < kW; ++w) {
      const double ew = v[w] ? e[w] : 0.0;
      s0 += ew;
      if constexpr (GRAD) {
        s1 = fma(ew, dt[w], s1);
        s2 = fma(ew, r2[w], s2);
      }
      pairs += static_cast<unsigned long long>(v[w]);
    }
    if (!(dt[kW - 1] <= a.dT)) break;  // (time-sorted: every earlier source is outside too)
  }
  st[0] = s0;
  a.trow[i] = s0;
  if constexpr (GRAD) {
    st[1] = s1;
    st[2] = s2;
    a.trow[a.npad + i] = s1;
    a.trow[2 * a.npad + i] = s2;
  }
  return pairs;
}

template <bool GRAD>
__global__ void __launch_bounds__(kTrigRowsThreads) trig_rows_kernel(const TrigRowsArgs a) {
  const int tid = threadIdx.x;
  const unsigned long long trace_t0 = (a.trace && tid == 0) ? global_ns() : 0ULL;
  if (tid == 0) {
    stamp_min(a.tstamp, 0);
    stamp_min(a.tstamp, 2);
  }
  // stage the exp table and the events [first - kTrigRowsBack, last] of this
  // block's rows (coalesced), then walk the windows in shared memory
  extern __shared__ __align__(128) uint2 s_rtab[];  // kExpTableSize (dynamic)
  __shared__ double s_rt[kTrigRowsBack + kTrigRowsThreads];
  __shared__ double s_rx[kTrigRowsBack + kTrigRowsThreads];
  __shared__ double s_ry[kTrigRowsBack + kTrigRowsThreads];
  const int64_t first = static_cast<int64_t>(a.row0) + static_cast<int64_t>(blockIdx.x) * kTrigRowsThreads;
  const int64_t last = min(first + kTrigRowsThreads, static_cast<int64_t>(a.row1)) - 1;
  const int64_t base = max(first - kTrigRowsBack, int64_t{0});
  const int cnt = static_cast<int>(last + 1 - base);
  for (int k = tid; k < kExpTableSize; k += kTrigRowsThreads) s_rtab[k] = kExpTable[k];
  for (int k = tid; k < cnt; k += kTrigRowsThreads) {
    s_rt[k] = a.t[base + k];
    s_rx[k] = a.xs[base + k];
    s_ry[k] = a.ys[base + k];
  }
  __syncthreads();
  const int64_t i = first + tid;
  unsigned long long pairs = 0;
  if (i <= last) {
    double st[GRAD ? 3 : 1];
    const RowSrcShared src{s_rt, s_rx, s_ry, base, s_rtab};
    pairs = trig_row_sums<GRAD>(a, src, i, st);
  }
  if (a.pair_counts) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) pairs += __shfl_xor_sync(0xffffffffu, pairs, off);
    if ((tid & 31) == 0 && pairs) {
      atomicAdd(&a.pair_counts[1], pairs);
      atomicAdd(&a.pair_counts[4], pairs);
    }
  }
  if (a.trace && tid == 0) trace_cta(a.trace, a.trace_cap, 11, trace_t0);
  if (tid == 0) stamp_max(a.tstamp, 3);
}

// ROWS: trigger-only evaluation by row windows over cached background sums
// (h, omega, theta moves): the row's trigger sums (trig_row_sums) and, if
// a.comp_inline, its compensator terms (comp_terms) are computed here and
// stored for the caches -- one kernel for the whole evaluation.
template <bool GRAD, bool ROWS>
__global__ void __launch_bounds__(kFinThreads) finalize_kernel(const FinArgs a) {
  constexpr int NS = GRAD ? kNSumGrad : kNSumVal;
  constexpr int NB = GRAD ? 3 : 1;
  constexpr int NT = NS - NB;
  __shared__ double s_w[kFinThreads / 32][kNOut];
  const int tid = threadIdx.x;
  __shared__ unsigned long long s_cta_t0;  // (development trace)
  // (graph mode: launched by a programmatic edge while the last pair kernel
  // drains; wait for its completion and memory -- a no-op otherwise)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (a.trace && tid == 0) s_cta_t0 = global_ns();
  if (tid == 0) stamp_min(a.tstamp, 0);
  const int64_t base = static_cast<int64_t>(a.row0) + static_cast<int64_t>(blockIdx.x) * kFB;
  double acc[kNOut];
#pragma unroll
  for (int q = 0; q < kNOut; ++q) acc[q] = 0.0;
  unsigned long long rows_pairs = 0;  // (ROWS: trigger pairs evaluated, timing counters)

  do {  // one row per thread; `continue` / `break` skip to the reduction
    const int64_t r = base + tid;
    if (r >= a.row1) break;
    // every independent load first (the row is latency-bound at small N)
    const int2 cr = (ROWS || a.trow) ? make_int2(0, -1) : a.crange[r / kTM];
    const int2 cf = a.tpart_far ? a.crange_far[r / kTM] : make_int2(0, -1);
    unsigned long long fw[2 * NB];
#pragma unroll
    for (int k = 0; k < 2 * NB; ++k) fw[k] = a.fx[static_cast<size_t>(k) * a.npad + r];
    double cc[4];
    if (ROWS && a.comp_inline) {
      comp_terms(a.t[r], a.window_end, a.tauT, a.omega, cc);
#pragma unroll
      for (int k = 0; k < 4; ++k) a.comp[static_cast<size_t>(k) * a.npad + r] = cc[k];
    } else {
      cc[0] = a.comp[r];
      cc[2] = a.comp[2 * a.npad + r];
      if constexpr (GRAD) {
        cc[1] = a.comp[a.npad + r];
        cc[3] = a.comp[3 * a.npad + r];
      }
    }
    const double dPhi = cc[0];
    const double em1 = cc[2];
    double dL2c = 0.0, dec = 0.0;
    if constexpr (GRAD) {
      dL2c = cc[1];
      dec = cc[3];
    }
    // trigger partials: chunks in order (then the far kernel's), four
    // chunks' loads in flight at a time; the additions keep chunk order
    double st[NT];
#pragma unroll
    for (int k = 0; k < NT; ++k) st[k] = 0.0;
    auto sum_chunks = [&](const double* tp, int2 c) {
      for (int c0 = c.x; c0 <= c.y; c0 += 4) {
        double v[4][NT];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double* q = tp + static_cast<size_t>(c0 + u) * NT * a.npad + r;
#pragma unroll
          for (int k = 0; k < NT; ++k) v[u][k] = c0 + u <= c.y ? q[static_cast<size_t>(k) * a.npad] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (c0 + u <= c.y) {
#pragma unroll
            for (int k = 0; k < NT; ++k) st[k] += v[u][k];
          }
        }
      }
    };
    if constexpr (ROWS) {
      rows_pairs = trig_row_sums<GRAD>(a.rows, RowSrcGlobal{a.rows.t, a.rows.xs, a.rows.ys}, r, st);
    } else if (a.trow) {  // (trig_rows_kernel: one sum per row)
#pragma unroll
      for (int k = 0; k < NT; ++k) st[k] = a.trow[static_cast<size_t>(k) * a.npad + r];
    } else {
      sum_chunks(a.tpart, cr);
    }
    if (a.tpart_far) sum_chunks(a.tpart_far, cf);  // (after the near ones: fixed order)
    double xb[NB];  // background sums, fixed-point word values (S_B; S_Br, S_Bt scaled)
#pragma unroll
    for (int k = 0; k < NB; ++k) xb[k] = fx_value(fw[2 * k], fw[2 * k + 1]);
    const double sB = xb[0];  // (fxq[0] = 1)
    const double sT = st[0];
    const double B = a.bgNorm * sB;
    const double Tr = a.trNorm * sT;
    const double lam = a.mu0 * B + Tr;  // likelihood.cpp:35

    // compensatorTerm, kernels.hpp:54-65, from the prepared terms (prep_kernel)
    const double Lam = a.mu0 * dPhi + (-a.theta * em1);

    if (a.ex_out) {  // excitation split, excitation.cpp:31-51
      a.ex_out[r] = a.mu0 * B;
      a.ex_out[a.npad + r] = Tr;
      a.ex_out[2 * a.npad + r] = (!(lam > 0.0) || !isfinite(lam)) ? 0.0 : Tr / lam;
    }
    if (!(lam > 0.0) || !isfinite(lam)) {  // likelihood.cpp:36-39
      acc[7] += 1.0;
      if (a.per_event) a.per_event[r] = 0.0;
      continue;
    }
    const double term = log(lam) - Lam;
    acc[0] += term;
    if (a.per_event) a.per_event[r] = term;
    if constexpr (GRAD) {
      const double inv = 1.0 / lam;
      // d lambda / d p with host-folded constants
      const double dl1 = fma(a.gB[0], sB, a.gB[1] * xb[1]);
      const double dl2 = fma(a.gB[2], sB, a.gB[3] * xb[2]);
      const double dl3 = a.cT * sT;
      const double dl4 = fma(a.gT[0], sT, a.gT[1] * st[1]);
      const double dl5 = fma(a.gT[2], sT, a.gT[3] * st[2]);
      // d Lambda / d p (prepared: dPhi, em1, (phi1 D + phi0 t) / tauT^2, D e^(-omega D))
      acc[1] = fma(B, inv, acc[1]) - dPhi;
      acc[2] = fma(dl1, inv, acc[2]);
      acc[3] = fma(dl2, inv, acc[3]) + a.mu0 * dL2c;
      acc[4] = fma(dl3, inv, acc[4]) + em1;
      acc[5] = fma(dl4, inv, acc[5]) - a.theta * dec;
      acc[6] = fma(dl5, inv, acc[6]);
    }
  } while (false);

  if (ROWS && a.rows.pair_counts) {  // (one atomic per warp)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) rows_pairs += __shfl_xor_sync(0xffffffffu, rows_pairs, off);
    if ((tid & 31) == 0 && rows_pairs) {
      atomicAdd(&a.rows.pair_counts[1], rows_pairs);
      atomicAdd(&a.rows.pair_counts[4], rows_pairs);
    }
  }
  block_sum8(acc, s_w);
  if (tid < kNOut) a.block_partial[(base / kFB) * kNOut + tid] = acc[0];
  if (a.fused_out) {  // single shard: the last block to finish does the final sum
    __shared__ bool s_last;
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      s_last = atomicAdd(a.done_counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      final_sum_block(a.block_partial, a.nblocks_total, a.fused_out, s_w);
      if (a.counts && tid < kNCounts) {
        a.counts_out[tid] = a.counts[tid];
        a.counts[tid] = 0ULL;
      }
      if (a.tstamp && tid < 4) {  // timing stamps out (mapped), re-armed for the next evaluation
        const unsigned long long v = tid == 1 ? max(a.tstamp[1], global_ns()) : a.tstamp[tid];
        a.tstamp_out[tid] = v;
        a.tstamp[tid] = (tid & 1) ? 0ULL : ~0ULL;
      }
      if (tid == 0) *a.done_counter = 0u;
    }
  }
  if (a.trace && tid == 0) trace_cta(a.trace, a.trace_cap, 6, s_cta_t0);
}

__global__ void __launch_bounds__(256) final_sum_kernel(const double* __restrict__ bp,
                                                        int nblocks, double* out,
                                                        unsigned long long* counts,
                                                        unsigned long long* counts_out) {
  __shared__ double s_w[8][kNOut];
  if (out) final_sum_block(bp, nblocks, out, s_w);
  if (counts && threadIdx.x < kNCounts) {
    counts_out[threadIdx.x] = counts[threadIdx.x];
    counts[threadIdx.x] = 0ULL;
  }
}

// Adds received fx segments (blockIdx.y = segment) into this rank's
// accumulators; several senders may cover the same rows, hence the atomics.
__global__ void __launch_bounds__(256) fx_accumulate_kernel(const FxAccArgs a) {
  const FxSeg sg = a.seg[blockIdx.y];
  const int64_t words = 6 * sg.len;
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < words;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = w / sg.len, i = w - k * sg.len;
    const unsigned long long v = a.stage[sg.off + w];
    if (v != 0ULL) atomicAdd(&a.fx[k * a.npad + sg.row + i], v);
  }
}

__global__ void __launch_bounds__(256) pi_accumulate_kernel(const double* __restrict__ ex,
                                                            int64_t npad, int row0, int row1,
                                                            double* __restrict__ sum_pi, int* bad) {
  const int64_t i = row0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= row1) return;
  const double lam = ex[i] + ex[npad + i];
  if (!(lam > 0.0) || !isfinite(lam)) *bad = 1;
  sum_pi[i] += ex[2 * npad + i];
}

}  // namespace

namespace {
thread_local LaunchSink* t_sink = nullptr;

// One single-struct-argument kernel launch, to the sink when one is set.
template <typename A>
cudaError_t launch_one(void (*kernel)(A), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       const A& args) {
  if (t_sink) {
    t_sink->launch(reinterpret_cast<const void*>(kernel), grid, block, smem, stream, &args,
                   sizeof(A));
    return cudaSuccess;
  }
  kernel<<<grid, block, smem, stream>>>(args);
  return cudaGetLastError();
}
}  // namespace

void set_launch_sink(LaunchSink* sink) { t_sink = sink; }

cudaError_t launch_pi_accumulate(const double* ex, int64_t npad, int row0, int row1,
                                 double* sum_pi, int* bad, cudaStream_t stream) {
  if (row1 <= row0) return cudaSuccess;
  pi_accumulate_kernel<<<(row1 - row0 + 255) / 256, 256, 0, stream>>>(ex, npad, row0, row1,
                                                                      sum_pi, bad);
  return cudaGetLastError();
}

cudaError_t launch_fx_accumulate(const FxAccArgs& a, cudaStream_t stream) {
  if (a.nseg <= 0) return cudaSuccess;
  int64_t maxlen = 0;
  for (int s = 0; s < a.nseg; ++s) maxlen = a.seg[s].len > maxlen ? a.seg[s].len : maxlen;
  const int64_t bx = (6 * maxlen + 255) / 256;
  const dim3 grid(static_cast<unsigned>(bx < 592 ? (bx > 0 ? bx : 1) : 592), a.nseg);
  fx_accumulate_kernel<<<grid, 256, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_tile_boxes(const double* sx, const double* sy, const double* st, double* x,
                              double* y, double* t, int64_t n, int64_t npad, double4* box,
                              double2* trange, double* piv, unsigned long long* bad,
                              unsigned int* done, unsigned long long* h_bad, double* h_stats,
                              unsigned long long* dstats, bool tile_pivots, cudaStream_t stream) {
  const int64_t ntiles = (n + kTS - 1) / kTS;
  const unsigned blocks = static_cast<unsigned>((ntiles + 7) / 8);
  tile_load_kernel<<<blocks, 256, 0, stream>>>(sx, sy, st, x, y, t, n, npad, box, trange, piv, bad,
                                               tile_pivots);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  const double* cx = x;
  const double* cy = y;
  const double* ct = t;
  const double4* cbox = box;
  const double2* ctr = trange;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, tile_stats_kernel, cx, cy, ct, n, cbox, ctr, piv,
                                           tile_pivots, bad, done, h_bad, h_stats, dstats);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_prep(const PrepArgs& a, cudaStream_t stream) {
  return launch_one(prep_kernel, dim3(static_cast<unsigned>((a.npad + 255) / 256)), dim3(256), 0,
                    stream, a);
}

cudaError_t launch_exp_probe(const double* x, int64_t n, double* out, cudaStream_t stream) {
  exp_probe_kernel<<<static_cast<unsigned>((n + 255) / 256), 256,
                     sizeof(uint2) * kExpTableSize, stream>>>(x, n, out);
  return cudaGetLastError();
}

cudaError_t launch_plan(const PlanArgs& a, cudaStream_t stream) {
  const int ntiles = a.tile1 - a.tile0;
  if (ntiles <= 0) return cudaSuccess;
  return launch_one(plan_kernel, dim3(1), dim3(1024), kPivots * sizeof(double), stream, a);
}

cudaError_t launch_plan_prep(const PlanArgs& plan, const PrepArgs& prep, cudaStream_t stream) {
  const PlanPrepArgs a{plan, prep};
  const unsigned nb = 1u + static_cast<unsigned>((prep.npad + 1023) / 1024);
  return launch_one(plan_prep_kernel, dim3(nb), dim3(1024), kPivots * sizeof(double), stream, a);
}

// The exp table (pair kernels) and the search pivots (plan) live in dynamic
// shared memory (static + dynamic > 48 KB needs the opt-in attribute); set
// once per device before the first launch.
cudaError_t prepare_pair_kernels() {
  cudaError_t err = cudaSuccess;
  auto set = [&](const void* f) {
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(kTabBytes));
    if (e != cudaSuccess) err = e;
  };
  set(reinterpret_cast<const void*>(&sym_kernel<true>));
  set(reinterpret_cast<const void*>(&sym_kernel<false>));
  set(reinterpret_cast<const void*>(&sym_kernel<true, true>));
  set(reinterpret_cast<const void*>(&sym_kernel<false, true>));
  set(reinterpret_cast<const void*>(&pair_kernel<true>));
  set(reinterpret_cast<const void*>(&pair_kernel<false>));
  const cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(&plan_kernel),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kPivots * sizeof(double)));
  if (e != cudaSuccess) err = e;
  const cudaError_t e2 = cudaFuncSetAttribute(reinterpret_cast<const void*>(&plan_prep_kernel),
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(kPivots * sizeof(double)));
  if (e2 != cudaSuccess) err = e2;
  // Kernels that run beside the pair kernels (or just before them) ask for
  // the pair kernels' shared-memory carveout: an SM changes its L1 / shared
  // split only when idle, so a small kernel configured for the largest L1
  // holds whole SMs away from the pair kernels' CTAs until it drains
  // (measured: trig_rows_kernel beside the trigger-free kernel delayed its
  // first CTA from 7.5 to 14.5 us into the evaluation).
  auto carve = [&](const void* f) {
    const cudaError_t c = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                               cudaSharedmemCarveoutMaxShared);
    if (c != cudaSuccess) err = c;
  };
  carve(reinterpret_cast<const void*>(&trig_rows_kernel<true>));
  carve(reinterpret_cast<const void*>(&trig_rows_kernel<false>));
  carve(reinterpret_cast<const void*>(&prep_kernel));
  carve(reinterpret_cast<const void*>(&far_kernel<true>));
  carve(reinterpret_cast<const void*>(&far_kernel<false>));
  carve(reinterpret_cast<const void*>(&finalize_kernel<true, false>));
  carve(reinterpret_cast<const void*>(&finalize_kernel<false, false>));
  for (const void* f : {reinterpret_cast<const void*>(&sym_kernel<true>),
                        reinterpret_cast<const void*>(&sym_kernel<false>),
                        reinterpret_cast<const void*>(&sym_kernel<true, true>),
                        reinterpret_cast<const void*>(&sym_kernel<false, true>)}) {
    carve(f);
  }
  return err;
}

cudaError_t launch_pairs(const PairArgs& a, bool grad, int mode, int grid, cudaStream_t stream) {
  if (mode == kSym) {
    return grad ? launch_one(sym_kernel<true>, dim3(grid), dim3(kTM), kTabBytes, stream, a)
                : launch_one(sym_kernel<false>, dim3(grid), dim3(kTM), kTabBytes, stream, a);
  } else {
    return grad ? launch_one(pair_kernel<true>, dim3(grid), dim3(kTM), kTabBytes, stream, a)
                : launch_one(pair_kernel<false>, dim3(grid), dim3(kTM), kTabBytes, stream, a);
  }
}

cudaError_t launch_finalize(const FinArgs& a, bool grad, cudaStream_t stream) {
  const int nblocks = (a.row1 - a.row0 + kFB - 1) / kFB;
  if (nblocks <= 0) return cudaSuccess;
  static_assert(kFinThreads == 256, "fused final sum uses the 256-thread final_sum_block");
  if (a.rows.trow) {
    return grad ? launch_one(finalize_kernel<true, true>, dim3(nblocks), dim3(kFinThreads), 0, stream, a)
                : launch_one(finalize_kernel<false, true>, dim3(nblocks), dim3(kFinThreads), 0, stream, a);
  }
  return grad ? launch_one(finalize_kernel<true, false>, dim3(nblocks), dim3(kFinThreads), 0, stream, a)
              : launch_one(finalize_kernel<false, false>, dim3(nblocks), dim3(kFinThreads), 0, stream, a);
}

cudaError_t launch_trig_rows(const TrigRowsArgs& a, bool grad, cudaStream_t stream) {
  const int nblocks = (a.row1 - a.row0 + kTrigRowsThreads - 1) / kTrigRowsThreads;
  if (nblocks <= 0) return cudaSuccess;
  return grad ? launch_one(trig_rows_kernel<true>, dim3(nblocks), dim3(kTrigRowsThreads), kTabBytes, stream, a)
              : launch_one(trig_rows_kernel<false>, dim3(nblocks), dim3(kTrigRowsThreads), kTabBytes, stream, a);
}

cudaError_t launch_final_sum(const double* block_partial, int nblocks, double* out,
                             unsigned long long* counts, unsigned long long* counts_out,
                             cudaStream_t stream) {
  final_sum_kernel<<<1, 256, 0, stream>>>(block_partial, nblocks, out, counts, counts_out);
  return cudaGetLastError();
}

cudaError_t launch_bgonly(const PairArgs& a, bool grad, int grid, cudaStream_t stream) {
  return grad ? launch_one(sym_kernel<true, true>, dim3(grid), dim3(kTM), kTabBytes, stream, a)
              : launch_one(sym_kernel<false, true>, dim3(grid), dim3(kTM), kTabBytes, stream, a);
}

int bgonly_kernel_occupancy(bool grad) {
  int occ = 0;
  if (prepare_pair_kernels() != cudaSuccess) return 1;
  if (grad) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sym_kernel<true, true>, kTM, kTabBytes);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sym_kernel<false, true>, kTM, kTabBytes);
  return occ > 0 ? occ : 1;
}

cudaError_t launch_far(const PairArgs& a, bool grad, int grid, cudaStream_t stream) {
  return grad ? launch_one(far_kernel<true>, dim3(grid), dim3(kTM), 0, stream, a)
              : launch_one(far_kernel<false>, dim3(grid), dim3(kTM), 0, stream, a);
}

int far_kernel_occupancy(bool grad) {
  int occ = 0;
  if (grad) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, far_kernel<true>, kTM, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, far_kernel<false>, kTM, 0);
  return occ > 0 ? occ : 1;
}

int pair_kernel_occupancy(bool grad, int mode) {
  int occ = 0;
  if (prepare_pair_kernels() != cudaSuccess) return 1;
  if (mode == kSym) {
    if (grad) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sym_kernel<true>, kTM, kTabBytes);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sym_kernel<false>, kTM, kTabBytes);
  } else {
    if (grad) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pair_kernel<true>, kTM, kTabBytes);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pair_kernel<false>, kTM, kTabBytes);
  }
  return occ > 0 ? occ : 1;
}

}  // namespace sthk
