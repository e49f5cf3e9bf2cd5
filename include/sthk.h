/* sthk.h -- C ABI of the B200 spatiotemporal-Hawkes likelihood engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj):
 *
 *   hawkes::logLikelihood(const EventSet&, const Params&, const Backend&,
 *                         bool keepPerEvent) -> LikelihoodResult
 *       include/sthawkes/likelihood.hpp:24-26, src/likelihood.cpp:10-55
 *   hawkes::logLikelihoodBatch(...)      likelihood.hpp:28-31, likelihood.cpp:57-75
 *
 * The reference's own plugin slot (pairReduce + PairReduceSpec,
 * backend.hpp:65-88,170-192) carries host-side callables that
 * capture host pointers, so a device engine plugs in one level up, at
 * logLikelihood. The reference API is stateless; this engine is stateful
 * (events stay resident in HBM across evaluations), and the C++ adapter
 * (paper_2005_10123_b200/adapter/hawkes_b200_adapter.cpp)
 * restores the stateless reference signature on top of it.
 *
 * Conventions
 *   Status codes: every entry point is noexcept and returns STHK_OK or one of
 *     the errors below; the message is available from sthk_last_error().
 *     A numerically degenerate evaluation (some lambda_i <= 0 or non-finite,
 *     likelihood.cpp:36-39,47-54) is NOT an error: status STHK_OK with
 *     *valid = 0, *loglik = -inf and grad[] = NaN.
 *   Params order is hawkes::Params order (types.hpp:51-57):
 *     p[0]=mu0 p[1]=tauX p[2]=tauT p[3]=theta p[4]=omega p[5]=h.
 *   Ownership: the engine owns all device memory; the caller owns every host
 *     buffer passed in; no host pointer is retained after a call returns.
 *   Threading: one handle must not be used from two threads at once.
 *   Determinism: results are bitwise identical for identical (events,
 *     params), and independent of the number of devices / ranks.
 */
#ifndef STHK_H
#define STHK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STHK_OK 0
#define STHK_EINVAL 1     /* invalid argument (maps to std::invalid_argument) */
#define STHK_ENOTLOADED 2 /* evaluation before sthk_load_events / set_params */
#define STHK_ECUDA 3      /* CUDA runtime error (maps to std::runtime_error) */
#define STHK_ENCCL 4      /* NCCL error */
#define STHK_ERANGE 5     /* excitation: a per-event rate underflowed to zero
                             (excitation.cpp:52-55; maps to std::runtime_error) */

#define STHK_NCCL_ID_BYTES 128

typedef struct sthk_engine sthk_engine;

/* Engine over n_devices GPUs driven from this process (n_devices >= 1).
 * Target rows are partitioned across the devices (one shard per entry of
 * device_ids, cost-balanced 1024-row blocks). Distinct device ids combine
 * the shards with NCCL (ncclCommInitAll): each shard ships the column sums it
 * added to other shards' rows to their owner (ncclSend / ncclRecv), and one
 * all-reduce combines the per-block partials. A device id may repeat: the
 * shards that share a device are separate rank engines (own accumulators,
 * plans and partials) combined by device copies along exactly the same
 * owner-directed routes -- the multi-GPU data flow emulated on one GPU. */
int sthk_create(const int* device_ids, int n_devices, sthk_engine** out);

/* One-process-per-GPU engine: this process owns `device` and is `rank` of
 * `world`; `nccl_id` is the STHK_NCCL_ID_BYTES blob from
 * sthk_nccl_unique_id() on rank 0, broadcast by the caller. */
int sthk_nccl_unique_id(void* nccl_id);
int sthk_create_rank(int device, int rank, int world, const void* nccl_id,
                     sthk_engine** out);

/* Rank engine whose two collectives run through caller-supplied host
 * callbacks instead of NCCL (e.g. torch.distributed gloo in tests, several
 * ranks sharing one GPU). Buffers passed to the callbacks are host memory
 * owned by the engine, valid for the duration of the call; a callback
 * returns 0 on success (anything else fails the evaluation, STHK_ENCCL). */
#define STHK_DTYPE_U64 0
#define STHK_DTYPE_F64 1
typedef struct sthk_host_comm {
  void* ctx;
  /* in-place element-wise sum over all ranks of `count` elements */
  int (*allreduce_sum)(void* ctx, void* buf, int64_t count, int dtype);
  /* post every send and receive (byte buffers, peers are ranks), return
   * once all have completed */
  int (*exchange)(void* ctx, int n_send, const int* send_peer, const void* const* send_buf,
                  const int64_t* send_bytes, int n_recv, const int* recv_peer,
                  void* const* recv_buf, const int64_t* recv_bytes);
} sthk_host_comm;
int sthk_create_rank_hosted(int device, int rank, int world, const sthk_host_comm* comm,
                            sthk_engine** out);

int sthk_destroy(sthk_engine* e);

/* Copies n events (time-sorted SoA, km / days) to every device.
 * Validation and messages follow the EventSet constructor (types.hpp:85-109):
 * n >= 1, finite entries, t >= 0, t nondecreasing, window_end finite and
 * >= t[n-1]. At most 2^23 events (the fixed-point background sums hold
 * totals below 2^23 per row). Replaces any previously loaded set. */
int sthk_load_events(sthk_engine* e, const double* x, const double* y,
                     const double* t, int64_t n, double window_end);

/* Validates like Params::validate (types.hpp:59-72). */
int sthk_set_params(sthk_engine* e, const double* params6);

/* Synchronous evaluations with the current params.
 * per_event (nullable, length n): log(lambda_i) - Lambda_i, 0 for degenerate
 * rows (likelihood.cpp:25,41); a rank engine fills its own rows only.
 * grad6 receives d loglik / d params in Params order. */
int sthk_loglik(sthk_engine* e, double* loglik, int* valid, double* per_event);
int sthk_loglik_grad(sthk_engine* e, double* loglik, int* valid, double* grad6,
                     double* per_event);

/* Batch over P parameter vectors (params: P x 6, row-major), elementwise
 * identical to P single calls (logLikelihoodBatch, likelihood.cpp:57-75).
 * grad (nullable): P x 6. */
int sthk_loglik_batch(sthk_engine* e, const double* params, int64_t P,
                      double* loglik, int* valid, double* grad);

/* Per-event split of the rate into background mu_i = mu0 * B_i and
 * self-excitation xi_i = T_i with pi_i = xi_i / (mu_i + xi_i), for the
 * current params (hawkes::excitationProbabilities, excitation.cpp:13-58).
 * Each output (nullable, length n) is filled; if any rate underflowed, pi is
 * 0 on those rows and STHK_ERANGE is returned. */
int sthk_excitation(sthk_engine* e, double* mu, double* xi, double* pi);

/* Posterior excitation over S parameter draws (the device half of
 * hawkes::posteriorExcitation, excitation.cpp:72-130, without thinning and
 * dump): every draw's pi_i is added, draws in order, to sum_pi[i] (in/out,
 * length n; start from zeros and divide by S afterwards: bitwise the
 * reference's meanPi loop, also across consecutive calls); per_draw (nullable, S x n row-major)
 * receives every draw's pi. Draws sharing tauX, tauT (every draw of the
 * reference MH sampler) share one background sweep. If a draw's rate
 * underflowed, returns STHK_ERANGE with *bad_draw = the first such draw
 * (else *bad_draw = -1). A rank engine fills its own rows only. */
int sthk_excitation_batch(sthk_engine* e, const double* params, int64_t S, double* sum_pi,
                          double* per_draw, int64_t* bad_draw);

/* Asynchronous pair: enqueue one evaluation of the current params on the
 * engine's stream(s); sthk_result() waits for and returns the latest one. */
int sthk_enqueue(sthk_engine* e, int want_grad, int want_per_event);
int sthk_result(sthk_engine* e, double* loglik, int* valid, double* grad6,
                double* per_event);

/* Introspection for benchmarks / tests. */
typedef struct sthk_stats {
  int64_t n;                 /* events loaded */
  int64_t pairs_bg;          /* ordered background pairs covered (tile granularity) */
  int64_t pairs_tr;          /* trigger pairs evaluated (tile granularity) */
  int64_t pairs_any;         /* pairs with either term evaluated */
  int64_t pairs_dense;       /* n * n */
  double pair_kernel_ms;     /* device time of the last pair kernel(s), max over
                                local devices; 0 unless timing is enabled */
  double eval_ms;            /* device time of the last whole evaluation */
  int32_t source_chunk;      /* sources per work item (SC) of the last eval */
  int32_t work_items;        /* live (row tile, chunk) items of the last eval */
  int32_t n_devices;         /* devices driven by this handle */
  int32_t rank, world;       /* rank-mode coordinates (0, 1 otherwise) */
  /* work executed by the last pair kernel(s): in symmetric mode one
   * background exp serves 2 ordered pairs (pairs_bg counts ordered pairs) */
  int64_t exec_bg;           /* background exps evaluated */
  int64_t exec_geom;         /* pair geometries (dx, dy, dt, r^2) evaluated */
  int64_t exec_sym;          /* background pairs also accumulated into columns */
  int32_t kernel_mode;       /* STHK_KERNEL_ROWS or STHK_KERNEL_SYM */
  int32_t cache_hit;         /* 1 if the last evaluation reused cached
                                background sums (trigger-only sweep) */
  int32_t trigger_cache_hit; /* 1 if it also reused the trigger sums (only mu0 /
                                theta changed: no pair sweep at all) */
  int64_t exec_far;          /* pairs evaluated in the FP32 far tier (every exponent
                                provably < -A, A in [30, 40]) */
  int64_t kernel_launches;   /* kernels the last evaluation launched (all devices) */
  double far_threshold;      /* far tier's threshold A of the last evaluation */
  double far_split_days;     /* its split tfar (sources further back run in FP32) */
  int64_t graph_launches;    /* evaluations launched as a cached CUDA graph (updated in place) */
  int64_t graph_builds;      /* evaluation graphs built and instantiated */
  int32_t load_zero_copy;    /* 1 if the last load read pinned caller arrays in place
                                (0: copied first -- pageable arrays, several devices,
                                or another engine's evaluation running on the device) */
  int32_t trigger_rows;      /* 1 if the last evaluation summed its trigger terms by row
                                windows (trigger window shorter than every 128-event
                                tile: trig_rows_kernel), 0 if by the tiled sweep */
} sthk_stats;

/* Timing and pair counters (sthk_get_stats): 0 off, 1 whole evaluation and
 * pair phase (device events), 2 whole evaluation only (no events between the
 * kernels: the one-shard evaluation graph keeps its kernel-to-kernel
 * dependencies, as with timing off). */
int sthk_set_timing(sthk_engine* e, int enable);
/* One-shard evaluations as CUDA graphs (default on): the evaluation's stream
 * operations are recorded and replayed as one graph launch; a graph of the
 * same topology is kept and its kernel arguments updated in place. Results
 * are bitwise identical either way (same kernels, same order of sums). */
int sthk_set_graphs(sthk_engine* e, int enable);
int sthk_get_stats(sthk_engine* e, sthk_stats* out);
/* cudaStream_t of local device slot `slot` (for event-based timing). */
int sthk_get_stream(sthk_engine* e, int slot, void** stream);
/* Development: the pair-kernel work-item trace of the last evaluation on a
 * slot (only with STHK_ITEM_TRACE=<entries> in the environment at create
 * time; else *count = 0). Four words per item: (kernel << 48 | smid << 32 |
 * item), (stages << 8 | contains the diagonal stage), start ns, end ns
 * (%globaltimer); kernel 1 general near, 2 trigger-free near, 3 far. */
int sthk_debug_item_trace(sthk_engine* e, int slot, unsigned long long* out, int64_t cap,
                          int64_t* count);
/* Debug/testing knob: 0 = exact tile culling on (default), 1 = evaluate the
 * dense pair set (results are bitwise identical either way). */
int sthk_set_dense(sthk_engine* e, int dense);
/* Pair-kernel variant. STHK_KERNEL_SYM (default) evaluates each background
 * pair once and adds it to both events' sums (b_ij = b_ji); STHK_KERNEL_ROWS
 * sweeps ordered pairs per target row. Both are deterministic; they agree to
 * rounding (different summation grouping), not bitwise. */
/* Sweep caches (default on). The background sums depend only on the
 * events, tauX and tauT, which the reference MH sampler keeps fixed for a
 * whole chain (sampler.cpp:48-49); while they are unchanged an evaluation
 * sweeps only the trigger band. The trigger sums depend only on the events,
 * omega and h; while those are unchanged too (an MH move of mu0 or theta) an
 * evaluation runs no pair sweep at all, only the per-event finalize. The
 * work plan (live ranges, work list) is reused while the culling windows are
 * unchanged. Results are bitwise identical with the caches on or off (fixed
 * chunk grid, same kernels). Benchmarks of full evaluations turn them off. */
int sthk_set_background_cache(sthk_engine* e, int enable);

/* Far tier of the symmetric kernel. 1 (default): source stages whose every
 * term is provably below e^-A of the row's self term (A in [30, 40]) run in
 * FP32 on the FMA/MUFU pipes, and far terms whose total is provably below
 * half an ulp of lambda are not evaluated. 2: the same far
 * list and windows evaluated by the FP64 kernel (what the FP32 tier saves).
 * 0: no far tier -- every pair within the exact-underflow windows in FP64. */
int sthk_set_far_tier(sthk_engine* e, int enable);
/* Trigger-free near kernel (default on): in full symmetric sweeps whose
 * trigger window dT is narrower than the near band, near stages of sources
 * earlier than t_tile_first - dT run in a variant without trigger code paths
 * (fewer registers, more resident warps). 0 = one near kernel for all. */
int sthk_set_bgonly_kernel(sthk_engine* e, int enable);
/* Far-tier schedule (tuning): concurrent = run the FP32 far kernel on a second
 * stream beside the FP64 near kernel, which then uses near_ctas CTAs per SM;
 * far_ctas far CTAs per SM are launched (extra ones start as near CTAs
 * retire). Sequential (concurrent = 0) uses full occupancy for both. */
int sthk_set_far_schedule(sthk_engine* e, int concurrent, int near_ctas, int far_ctas);

#define STHK_KERNEL_ROWS 0
#define STHK_KERNEL_SYM 1
int sthk_set_kernel(sthk_engine* e, int mode);

/* Bytes of fixed-point background sums this handle's shards sent to other
 * shards' owners in the last evaluation (owner-directed exchange; 0 with one
 * shard, for a cached background or in row mode). */
int sthk_get_exchange_bytes(sthk_engine* e, int64_t* bytes);

/* Host-only planning (no device): the cost-balanced row partition the engine
 * uses for `shards` devices/ranks -- cuts[0..shards], multiples of 1024 rows,
 * cuts[shards] = n -- and the source-chunk size. Identical on every rank for
 * identical (times, params). */
int sthk_plan_partition(const double* t, int64_t n, const double* params6,
                        int shards, int dense, int* cuts, int* source_chunk);

/* DFMA throughput probe on `device` (roofline denominator for the FP64
 * pair kernels): best and mean TFLOP/s over `reps` timed launches. */
int sthk_measure_fp64_peak(int device, int reps, double* tflops_best,
                           double* tflops_mean);

/* Diagnostic: the pair kernels' device exp (exp_l) on n natural-unit
 * exponents x <= 0 (accuracy tests against libm). */
int sthk_debug_exp(int device, const double* x, int64_t n, double* out);

const char* sthk_last_error(const sthk_engine* e);
const char* sthk_version(void);

#ifdef __cplusplus
}
#endif

#endif /* STHK_H */
