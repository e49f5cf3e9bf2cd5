// Kernel-side interface of the B200 Hawkes engine (shared by sthk_kernels.cu
// and the host engine). Plain structs passed by value as kernel parameters.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace sthk {

constexpr int kTM = 128;    // target rows per tile (= threads per pair CTA)
constexpr int kTS = 128;    // sources per shared-memory stage (= tile size)
constexpr int kRB = 1024;   // rows per reduction block (multi-GPU partition unit)
constexpr int kFinThreads = 256;
constexpr int kFB = kFinThreads;  // rows per finalize block / block partial
constexpr int kNSumGrad = 6;  // S_B, S_Br, S_Bt, S_T, S_Tt, S_Tr
constexpr int kNSumVal = 2;   // S_B, S_T
constexpr int kNOut = 8;      // loglik, 6 gradient terms, degenerate-row count
// pair counters: ordered pairs covered (bg, trigger, any), then work executed
// (background exps, pair geometries, symmetric column accumulations)
constexpr int kNCounts = 7;  // [6]: pairs evaluated in the FP32 far tier

// Exponent cut (natural units) used for exact culling: every pair whose
// time-only exponent bound is below -kCullExponent has exp_l(...) == +0
// exactly (exp_l flushes below -708.40), so skipping it leaves every sum
// bitwise unchanged.
constexpr double kCullExponent = 709.0;

// Pair-kernel variants.
//  kRows: each CTA owns 128 target rows and sweeps every live source
//         (ordered pairs; row sums only).
//  kSym:  the background term is symmetric (b_ij = b_ji), so each CTA
//         sweeps only the source tiles J <= I; for J < I every background exp
//         is added to the row sums of I and the column sums of J. The
//         trigger term stays one-directional (t_j < t_i implies j < i).
enum PairMode : int { kRows = 0, kSym = 1 };

// Exponent constants are pre-multiplied by kExpL = 2048/ln2 ("L units", see
// exp_l in sthk_device.cuh).
struct PairConsts {
  double cxL;   // -L/(2 tauX^2)
  double ctL;   // -L/(2 tauT^2)
  double chL;   // -L/(2 h^2)
  double chS;   // chL / sx^2: trigger spatial constant on pre-scaled coordinates (kSym)
  double nomL;  // -L omega
  double dB;    // background live iff |dt| <= dB   (inf when dense)
  double dT;    // trigger live iff 0 < dt <= dT    (inf when dense)
  // far tier (kSym, FP32 far_kernel): coordinates xf, yf, tf in log2 units
  float fc1;    // trigger exponent, log2 units: fc1 * dtf + fc2 * r2f
  float fc2;
  double fkr;   // r2f -> r2 (kSym units, -cxL r^2)
  double fkt1;  // dtf -> dt (days)
  double fkt2;  // dtf^2 -> dt^2
  double fstf;  // time scale of tf (tf = (t - t_tile0) * fstf)
  double dBf;   // far tier: background evaluated iff |dt| <= dBf (beyond: < 2^-54 S_B in total)
  double dTf;   // far tier: trigger evaluated iff dt <= dTf (same bound)
};

constexpr int kPlanPivots = 8192;  // sorted-time search pivots (a power of two; 64 KB)

struct PlanArgs {
  const double* t;
  const double* piv;            // [kPlanPivots] t[k * ceil(n / kPlanPivots)], +inf padded (load)
  const double2* tile_trange;   // per 128-event tile: t first, t last (load)
  int64_t n;
  int tile0, tile1;     // this shard's row tiles [tile0, tile1)
  double dB, dT;
  int dense;
  int sym;              // kSym: the live range ends at the tile's own end
  int trig_only;        // trigger-only sweep: [t_min - dT, tile end)
  int sc;               // sources per chunk (multiple of kTS)
  int nchunks;          // ceil(n / sc)
  int2* ranges;         // [ntiles] live source range [lo, hi) per row tile
  int2* crange;         // [ntiles] chunk range [c0, c1] per row tile
  int2* items;          // (row tile, chunk) work list
  int* n_items;         // device scalar
  int* work_counter;    // device scalar, reset here
  // far tier (kSym): sources earlier than t_tile_first - tfar (whole
  // 128-stages) go to a second list for the FP32 far kernel; tfar <= 0: off
  double tfar;
  // far-tier cull: far sources earlier than t_tile_first - dFar are not
  // evaluated (their terms sum to under half an ulp of every row's S_B, see
  // make_plan in sthk_engine.cpp and DESIGN.md §3)
  double dFar;
  int2* ranges_far;     // [ntiles] far source range [lo, fb)
  int2* crange_far;     // [ntiles] far chunk range (empty: y < x)
  int2* items_far;
  int* n_items_far;
  int* work_counter_far;
  // background-only split of the near range (kSym full sweeps): near stages
  // before first - bg_adj * 128 (no live trigger, host-checked) go to a third
  // list for the trigger-free FP64 kernel; nullptr: off
  int tile_pivots;      // piv holds tile last times (see use_tile_pivots), else strided times
  int bg_adj;           // near stages kept with the tile for the general kernel (>= 1)
  int tile_order;       // equal one-stage items (no near trigger term): lists in tile order
  int bg_all;           // no near trigger term (trig_rows_kernel): every near stage,
                        // the diagonal one included, to the trigger-free list
  int sc_bg;            // sources per chunk of the background-only list (multiple of kTS)
  int sc_far;           // sources per chunk of the far list (multiple of kTS)
  int2* ranges_bg;
  int2* crange_bg;
  int2* items_bg;
  int* n_items_bg;
  int* work_counter_bg;
  unsigned long long* trace;  // development trace (PairArgs::trace), nullptr: off
  int trace_cap;
  unsigned long long* tstamp;  // timing stamps (PairArgs::tstamp), nullptr: off
};

// Background sums (k = 0..2: S_B, S_Br, S_Bt) are fixed point,
// fx[(k * 2 + h) * npad + row], h = 0 hi / 1 lo, scaled by fxq[k] before
// conversion so they are O(1) per pair; trigger sums are double partials
// tpart[(chunk * NT + k) * npad + row].
struct PairArgs {
  const double* x;
  const double* y;
  const double* t;
  const double* xs;         // kSym: x, y pre-scaled by sx = sqrt(-cxL) (r2 = -cxL r^2)
  const double* ys;
  const float* xf;          // kSym far tier: FP32 (x - x0) sxf, (y - y0) sxf, (t - t_tile0) stf
  const float* yf;
  const float* tf;
  const double4* tile_box;  // per 128-event tile: xmin, xmax, ymin, ymax
  const double2* tile_trange;  // per 128-event tile: t first, t last
  int64_t n;
  int64_t npad;
  PairConsts k;
  int sc;
  const int2* ranges;
  const int2* items;
  const int* n_items;
  int* work_counter;
  unsigned int* done_counter;  // CTAs finished (the last one re-arms work_counter)
  unsigned long long* fx;
  double fxq[kNSumGrad];
  double* tpart;        // trigger partials [nchunks][3 or 1][npad]
  int bg_off;           // trigger-only sweep (background sums come from a cache)
  int tr_off;           // no trigger terms: trig_rows_kernel computes them (sparse window)
  int bg_diag_only;     // general kernel beside the trigger-free one: background on the
                        // diagonal stage only (the trigger-free kernel has every earlier stage)
  unsigned long long* pair_counts;  // [kNCounts] (tile granularity)
  // merged trigger-free list (general sym_kernel only; nullptr: none): work
  // items [0, *pre_n_items) are the background-only list's -- its ranges,
  // items and chunk size, no trigger, fixed-point row sums only -- and the
  // rest the general list's, all from the general list's work counter
  const int2* pre_ranges;
  const int2* pre_items;
  const int* pre_n_items;
  int pre_sc;
  // trigger-free kernel: tile-relative times scaled by stl = sqrt(-ctL), so
  // the background exponent is -(r2 + dts^2) (one DFMA) and S_Bt is
  // recovered per flush as -(sum e * exponent) - S_Br
  const double* tsl;
  double stl;
  // development trace (nullptr: off): trace[0] counts entries, entry e at
  // trace[4 + 4e ..]: (kernel << 48 | smid << 32 | item), (stages << 8 | diag),
  // globaltimer at item start, at item end
  unsigned long long* trace;
  int trace_kernel;
  int trace_cap;
  // timing without events between kernels (graph mode): %globaltimer stamps,
  // [0] first CTA start of the evaluation (min), [1] end (finalize, max),
  // [2] first pair CTA start (min), [3] last pair CTA end (max); nullptr: off
  unsigned long long* tstamp;
};

#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned int sm_id() {
  unsigned int r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
// one entry per CTA (item field all ones): kernel id, SM, block, start, end
__device__ __forceinline__ void trace_cta(unsigned long long* trace, int cap, int kernel,
                                          unsigned long long t0) {
  const unsigned long long t1 = global_ns();
  const unsigned long long e = atomicAdd(trace, 1ULL);
  if (e < static_cast<unsigned long long>(cap)) {
    unsigned long long* p = trace + 4 + 4 * e;
    p[0] = (static_cast<unsigned long long>(kernel) << 48) |
           (static_cast<unsigned long long>(sm_id()) << 32) | 0xFFFFFFFFULL;
    p[1] = static_cast<unsigned long long>(blockIdx.x) << 8;
    p[2] = t0;
    p[3] = t1;
  }
}
// (timing stamps: CTA start -> min into slot, CTA end -> max into slot)
__device__ __forceinline__ void stamp_min(unsigned long long* ts, int slot) {
  if (ts) atomicMin(ts + slot, global_ns());
}
__device__ __forceinline__ void stamp_max(unsigned long long* ts, int slot) {
  if (ts) atomicMax(ts + slot, global_ns());
}
__device__ __forceinline__ void trace_item(const PairArgs& a, int item, int nst, int diag,
                                           unsigned long long t0) {
  const unsigned long long t1 = global_ns();
  const unsigned long long e = atomicAdd(a.trace, 1ULL);
  if (e < static_cast<unsigned long long>(a.trace_cap)) {
    unsigned long long* p = a.trace + 4 + 4 * e;
    p[0] = (static_cast<unsigned long long>(a.trace_kernel) << 48) |
           (static_cast<unsigned long long>(sm_id()) << 32) | static_cast<unsigned int>(item);
    p[1] = (static_cast<unsigned long long>(nst) << 8) | static_cast<unsigned>(diag);
    p[2] = t0;
    p[3] = t1;
  }
}
#endif

// Trigger sums over each row's own window (trig_rows_kernel): every source
// j < i with 0 < t_i - t_j <= dT (the exact underflow window 709/omega), for
// windows shorter than every 128-event tile's time span (at most 254 sources
// per row, usually a handful).
struct TrigRowsArgs {
  const double* xs;     // scaled coordinates (prep_kernel): r2 = sx^2 r^2
  const double* ys;
  const double* t;
  int64_t npad;
  int row0, row1;
  double nomL, chS, dT;  // PairConsts::nomL, chS; the window (709 / omega)
  double* trow;         // [NT][npad]: S_T (, S_Tt, S_Tr') per row
  unsigned long long* pair_counts;  // nullable (timing): [1] trigger pairs, [4] geometries
  unsigned long long* tstamp;
  unsigned long long* trace;  // development trace (PairArgs::trace), nullptr: off
  int trace_cap;
};

struct FinArgs {
  const double* t;
  int64_t n;
  int64_t npad;
  int row0, row1;       // shard rows (row0 multiple of kRB)
  double window_end;
  // parameters and folded constants
  double mu0, tauX, tauT, theta, omega, h;
  double bgNorm;        // (2pi)^-1.5 / (tauX^2 tauT)       kernels.hpp:79
  double trNorm;        // theta omega / (2 pi h^2)          kernels.hpp:82
  double cT;            // omega / (2 pi h^2)  (d lambda / d theta)
  // gradient constants folded on the host (no divisions per row), applied to
  // the raw fixed-point / trigger sums: with mb = mu0 bgNorm,
  //   d lambda / d tauX  = gB[0] S_B + gB[1] X_Br   (X_Br = fixed-point S_Br word value)
  //   d lambda / d tauT  = gB[2] S_B + gB[3] X_Bt
  //   d lambda / d omega = gT[0] S_T + gT[1] S_Tt
  //   d lambda / d h     = gT[2] S_T + gT[3] S_Tr'
  double gB[4], gT[4];
  const unsigned long long* fx;
  double fxq[kNSumGrad];
  const double* tpart;
  double tr_r2_scale;   // 1 (kRows) or 1/sx^2 (kSym: trigger r^2 sums on scaled coordinates)
  const int2* crange;
  double* comp;         // prepared compensator terms [4][npad] (prep_kernel)
  const double* tpart_far;  // far kernel's trigger partials (same layout), chunks crange_far
  const int2* crange_far;
  const double* trow;   // non-null: trigger sums per row (trig_rows_kernel) instead of tpart
  // rows.trow non-null: trigger-only evaluation by row windows, the trigger
  // sums computed (and stored to rows.trow) by finalize itself; comp_inline:
  // the compensator terms too (stored to comp)
  TrigRowsArgs rows;
  int comp_inline;
  double* per_event;    // nullable
  double* ex_out;       // nullable: excitation mu, xi, pi as [3][npad]
  double* block_partial;  // [ceil(n / kFB)][kNOut]
  // single shard: fuse the final sum (the last block sums all nblocks_total
  // block partials into fused_out -- host-mapped pinned memory, so no D2H
  // copy follows); nullptr when a collective sits between
  double* fused_out;
  int nblocks_total;
  unsigned int* done_counter;
  // with fused_out: the pair counters are copied to counts_out (host-mapped)
  // and re-zeroed for the next evaluation; nullptr: untouched
  unsigned long long* counts;
  unsigned long long* counts_out;
  unsigned long long* tstamp_out;  // with tstamp: the last block copies the stamps here (mapped) and re-arms them
  unsigned long long* trace;  // development trace (PairArgs::trace), nullptr: off
  int trace_cap;
  unsigned long long* tstamp;  // timing stamps (PairArgs::tstamp), nullptr: off
};

// Launch sink: while set (per host thread), the evaluation-path launch
// wrappers (plan, prep, pair, trigger-free, far, finalize) hand their launch
// to the sink instead of issuing it -- the engine records an evaluation's
// kernels and replays them as a CUDA graph (sthk_engine.cpp).
struct LaunchSink {
  virtual void launch(const void* func, dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                      const void* args, size_t arg_bytes) = 0;
  virtual ~LaunchSink() = default;
};
void set_launch_sink(LaunchSink* sink);

// Launch wrappers (sthk_kernels.cu). All enqueue on `stream`.
// Load-time statistics of an event set (tile_box_kernel, host-mapped):
// [0] max |x - x[0]|, [1] max |y - y[0]|, [2] max time span of a 128-event
// tile, [3 + k - 1] (k = 1..kLoadAdj) min over tiles of t[first] -
// t[first - 128 k - 1] (the gap k stages ahead of a tile's first event),
// [3 + kLoadAdj + L] (L = 0..kLoadSpan-1) min over runs of 2^L consecutive
// whole tiles of their time span (+inf: no such run): a time window shorter
// than level L's span holds fewer than (2^L + 1) * 128 events.
constexpr int kLoadAdj = 16;
constexpr int kLoadSpan = 16;
constexpr int kLoadStats = 3 + kLoadAdj + kLoadSpan;

// Event load into x, y, t from sources sx, sy, st -- the caller's pinned
// host arrays (device-mapped: the load kernel itself is the H2D copy) or x,
// y, t themselves after a cudaMemcpy -- with the per-tile bounding boxes and
// time ranges, the plan's search pivots (PlanArgs::piv), the pad tail zeroed
// and the EventSet checks (finite, t >= 0, sorted). The second kernel's last
// block writes the first failing index (all ones: none) to *h_bad and the
// load statistics to h_stats (both host-mapped), and re-arms *bad (device,
// all ones between loads), *done (0) and dstats (kLoadStats device words,
// maxima 0 / minima +inf bits).
cudaError_t launch_tile_boxes(const double* sx, const double* sy, const double* st, double* x,
                              double* y, double* t, int64_t n, int64_t npad, double4* box,
                              double2* trange, double* piv, unsigned long long* bad,
                              unsigned int* done, unsigned long long* h_bad, double* h_stats,
                              unsigned long long* dstats, bool tile_pivots, cudaStream_t stream);
// Tile pivots (tile last times, tile-granular plan searches) are used up to
// kPlanPivots tiles; above, strided pivots t[k ceil(n / kPlanPivots)].
inline bool use_tile_pivots(int64_t n) { return (n + kTS - 1) / kTS <= kPlanPivots; }
// Per-evaluation preparation (prep_kernel); every output optional (nullptr):
// kSym coordinates xs, ys = (x, y) * sx and the far tier's FP32 copies
// xf, yf = (x - x[0], y - y[0]) * sxf, tf = (t - t[tile start]) * stf; zeroed
// fixed-point accumulators fx[6][npad]; compensator terms comp[4][npad].
struct PrepArgs {
  const double* x;
  const double* y;
  const double* t;
  int64_t n, npad;
  double sx;
  double* xs;
  double* ys;
  double sxf, stf;
  float* xf;
  float* yf;
  float* tf;
  unsigned long long* fx;
  double* comp;
  double window_end, tauT, omega;
  // trigger-free kernel: tile-relative scaled times tsl = (t - t_tile0) * stl
  double stl;
  double* tsl;
  unsigned long long* trace;  // development trace (PairArgs::trace), nullptr: off
  int trace_cap;
  unsigned long long* tstamp;  // timing stamps (PairArgs::tstamp), nullptr: off
};
cudaError_t launch_prep(const PrepArgs& a, cudaStream_t stream);
cudaError_t launch_plan(const PlanArgs& a, cudaStream_t stream);
// plan + prep as one grid (block 0 plans, the rest prepare; small sets)
struct PlanPrepArgs {
  PlanArgs plan;
  PrepArgs prep;
};
cudaError_t launch_plan_prep(const PlanArgs& plan, const PrepArgs& prep, cudaStream_t stream);
cudaError_t launch_exp_probe(const double* x, int64_t n, double* out, cudaStream_t stream);
cudaError_t launch_pairs(const PairArgs& a, bool grad, int mode, int grid, cudaStream_t stream);
// Trigger-free symmetric FP64 kernel over the background-only list (PairArgs'
// ranges / items / counters point at that list's buffers).
cudaError_t launch_bgonly(const PairArgs& a, bool grad, int grid, cudaStream_t stream);
int bgonly_kernel_occupancy(bool grad);
// FP32 far kernel over the far work list (PairArgs' ranges / items / counters
// / tpart point at the far list's buffers).
cudaError_t launch_far(const PairArgs& a, bool grad, int grid, cudaStream_t stream);
int far_kernel_occupancy(bool grad);
cudaError_t launch_finalize(const FinArgs& a, bool grad, cudaStream_t stream);
cudaError_t launch_trig_rows(const TrigRowsArgs& a, bool grad, cudaStream_t stream);
// (out and counts_out may be host-mapped; counts, if non-null, are copied to
// counts_out and re-zeroed; out == nullptr: counters only)
cudaError_t launch_final_sum(const double* block_partial, int nblocks, double* out,
                             unsigned long long* counts, unsigned long long* counts_out,
                             cudaStream_t stream);

// Owner-directed exchange of the fixed-point background sums (multi-rank
// symmetric sweeps): a rank's column sums land on earlier rows,
// some owned by other ranks; each sender ships rows [row, row + len) of its
// six fx words to their owner, which adds them into its own accumulators.
// Segment s of `stage` is laid out [6][len] at word offset off. Integer
// addition: exact and order-free.
struct FxSeg {
  int64_t row, len, off;
};
constexpr int kMaxFxSegs = 32;  // segments per launch (the host loops beyond)
struct FxAccArgs {
  unsigned long long* fx;
  int64_t npad;
  const unsigned long long* stage;
  int nseg;
  FxSeg seg[kMaxFxSegs];
};
cudaError_t launch_fx_accumulate(const FxAccArgs& a, cudaStream_t stream);

// Posterior-excitation batch (sthk_excitation_batch): after a draw's
// finalize wrote mu, xi, pi ([3][npad], ex), rows [row0, row1) add pi into
// sum_pi (draws in order: the reference's meanPi += pi, excitation.cpp:112)
// and flag the draw (*bad = 1) if some rate mu + xi is not positive and
// finite (excitation.cpp:40-46).
cudaError_t launch_pi_accumulate(const double* ex, int64_t npad, int row0, int row1,
                                 double* sum_pi, int* bad, cudaStream_t stream);
// Resident CTAs per SM of a pair kernel (for the persistent grid size).
int pair_kernel_occupancy(bool grad, int mode);

}  // namespace sthk
