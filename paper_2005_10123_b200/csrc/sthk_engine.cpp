// Host engine behind the sthk.h C ABI: device-resident event sets, per-eval
// planning (exact culling windows, chunk size, cost-balanced row partition),
// kernel sequencing on one CUDA stream per device, and the two multi-rank
// collectives: the owner-directed exchange of the symmetric sweep's column
// sums and the all-reduce of the per-block partials, over NCCL, device copies
// (ranks sharing a GPU) or caller-supplied host callbacks.
//
// Reference behaviour mirrored here (file:line under /root/reference/proj):
//   Params::validate         include/sthawkes/types.hpp:59-72 (same message)
//   EventSet validation      include/sthawkes/types.hpp:85-109 (same messages)
//   logLikelihood            src/likelihood.cpp:10-55 (valid/-inf semantics,
//                            per-event terms 0 on degenerate rows)
//   logLikelihoodBatch       src/likelihood.cpp:57-75 (elementwise identical)
//   pairReduceRun            include/sthawkes/backend.hpp:142-166 (contiguous
//                            target blocks -> here contiguous 1024-row blocks
//                            per device, partials combined in block order)
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/sthk.h"
#include "sthk_kernels.cuh"

namespace {

using sthk::kNOut;
using sthk::kRB;
using sthk::kTM;
using sthk::kTS;

struct InvalidArg : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NotLoaded : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CommErr : std::runtime_error {  // host-callback collective failed
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaErr(std::string(what) + ": " + cudaGetErrorString(e));
  }
}
void ckn(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    throw NcclErr(std::string(what) + ": " + ncclGetErrorString(r));
  }
}

template <typename T>
void dev_grow(T*& p, size_t& cap, size_t need) {
  if (need <= cap && p) return;
  if (p) ck(cudaFree(p), "cudaFree");
  p = nullptr;
  const size_t bytes = std::max<size_t>(need, 1) * sizeof(T);
  ck(cudaMalloc(reinterpret_cast<void**>(&p), bytes), "cudaMalloc");
  cap = need;
}

struct Slot {
  int dev = 0;
  int sms = 148;
  int occ[2][2] = {{1, 1}, {1, 1}};  // [mode][grad]
  int occ_far[2] = {1, 1};           // far kernel [grad]
  int occ_bg[2] = {1, 1};            // trigger-free near kernel [grad]
  int2 *ranges_bg = nullptr, *crange_bg = nullptr, *items_bg = nullptr;
  size_t ranges_bg_cap = 0, crange_bg_cap = 0, items_bg_cap = 0;
  int2 *ranges_far = nullptr, *crange_far = nullptr, *items_far = nullptr;
  size_t ranges_far_cap = 0, crange_far_cap = 0, items_far_cap = 0;
  double* tpart_far = nullptr;       // far kernel trigger partials [nchunks_far][3][npad]
  size_t tpart_far_cap = 0;
  double2* tile_trange = nullptr;    // per tile: t first, t last
  double* comp = nullptr;            // compensator terms [4][npad] (prep_kernel)
  double* piv = nullptr;             // plan search pivots [kPlanPivots] (written at load)
  size_t comp_cap = 0;
  cudaEvent_t prepped = nullptr;     // prep done (stream 2) -> pair kernels (stream 1)
  size_t trange_cap = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;    // far kernel, concurrent with the near sweep
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaEvent_t pairs_done = nullptr, fin_done = nullptr;  // cross-slot ordering (local transport)
  ncclComm_t comm = nullptr;
  int shard = 0;                     // this slot's shard (= rank)
  unsigned long long* fx_stage = nullptr;  // received fx segments ([6][len] each)
  size_t fx_stage_cap = 0;
  double *x = nullptr, *y = nullptr, *t = nullptr;
  size_t x_cap = 0, y_cap = 0, t_cap = 0;
  double *xs = nullptr, *ys = nullptr;  // kSym: x, y scaled by sqrt(-cxL) (per evaluation)
  size_t xs_cap = 0, ys_cap = 0;
  double* tsl = nullptr;  // kSym trigger-free kernel: (t - t_tile0) * sqrt(-ctL) (per evaluation)
  size_t tsl_cap = 0;
  float *xf = nullptr, *yf = nullptr, *tf = nullptr;  // kSym far tier: FP32 coordinates
  size_t xf_cap = 0, yf_cap = 0, tf_cap = 0;
  double* h_stats = nullptr;  // pinned, device-mapped: load statistics (sthk::kLoadStats)
  double4* tile_box = nullptr;
  size_t box_cap = 0;
  int2* ranges = nullptr;
  size_t ranges_cap = 0;
  int* counts = nullptr;
  size_t counts_cap = 0;
  int2* items = nullptr;
  size_t items_cap = 0;
  int* scalars = nullptr;  // [0] n_items, [1] work counter, [2] pair CTAs done, [3] finalize
                           // blocks done, [4..5] first invalid event index (uint64),
                           // [6] far n_items, [7] far work counter, [8] far CTAs done,
                           // [9] bg-only n_items, [10] its work counter, [11] its CTAs done,
                           // [12] load-check blocks done
  unsigned long long* h_bad = nullptr;  // pinned
  unsigned long long* fx = nullptr;  // fixed-point background sums [6][npad]
  size_t fx_cap = 0;
  double* tpart = nullptr;           // trigger partials [nchunks][3][npad]
  size_t tpart_cap = 0;
  double* trow = nullptr;            // trigger sums per row [3][npad] (trig_rows_kernel)
  size_t trow_cap = 0;
  cudaEvent_t trow_ev = nullptr;     // trig_rows_kernel done (second stream)
  int2* crange = nullptr;
  size_t crange_cap = 0;
  double* block_partial = nullptr;
  size_t bp_cap = 0;
  double* per_event = nullptr;
  size_t pe_cap = 0;
  double* ex = nullptr;  // excitation mu, xi, pi [3][npad]
  size_t ex_cap = 0;
  double* pi_sum = nullptr;  // excitation batch: sum of pi over the draws [npad]
  size_t pi_sum_cap = 0;
  int* pi_bad = nullptr;     // excitation batch: per-draw degenerate flags
  size_t pi_bad_cap = 0;
  double* pi_rows = nullptr;  // excitation batch: per-draw pi rows staged [kPiChunk][npad]
  size_t pi_rows_cap = 0;
  double* h_pi_rows = nullptr;  // pinned copy of pi_rows
  size_t h_pi_rows_cap = 0;
  double* h_ex = nullptr;  // pinned
  size_t h_ex_cap = 0;
  unsigned long long* pair_counts = nullptr;
  double* h_out = nullptr;                 // pinned, device-mapped kNOut (kernels write it)
  double* d_hout = nullptr;                // device alias of h_out
  unsigned long long* d_hcounts = nullptr;  // device alias of h_counts
  unsigned long long* h_counts = nullptr;  // pinned kNCounts
  double* h_per_event = nullptr;           // pinned
  size_t h_pe_cap = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int row0 = 0, row1 = 0;  // rows of the last enqueued eval (first..last run)
  // plan cache (with the sweep caches on): the last plan's inputs; the plan
  // is a function of (times, culling windows, mode, rows, chunking) only
  bool plan_valid = false;
  double plan_dB = 0, plan_dT = 0;
  int plan_key[7] = {0, 0, 0, 0, 0, 0, 0};  // tile0, tile1, sc, dense, sym, trig_only, bg split
  double plan_tfar = 0, plan_dfar = 0;
  std::vector<std::pair<int, int>> runs;  // row ranges run on this slot
  unsigned long long* trace = nullptr;     // development item trace (STHK_ITEM_TRACE)
  unsigned long long* load_dstats = nullptr;  // load statistics accumulators (tile_box_kernel)
  unsigned long long* tstamp = nullptr;    // kernel timing stamps [4] (graph-mode timing)
  unsigned long long* h_tstamp = nullptr;  // pinned, device-mapped copy written by finalize
  unsigned long long* d_htstamp = nullptr;
  bool last_stamps = false;                // the last evaluation was timed by stamps
};

// (development knob: STHK_ITEM_TRACE=<entries> records every pair-kernel work
// item's SM and start / end time, sthk_debug_item_trace)
int item_trace_cap() {
  static const int v = [] {
    const char* s = std::getenv("STHK_ITEM_TRACE");
    const int k = s ? std::atoi(s) : 0;
    return k > 0 ? std::min(k, 1 << 22) : 0;
  }();
  return v;
}

struct EvalPlan;  // (defined with the planner below)
}  // namespace

// How the shards of one evaluation are combined.
enum class Xport {
  kSingle,  // one shard
  kNccl,    // NCCL: ncclSend / ncclRecv + ncclAllReduce (devices or torchrun ranks)
  kLocal,   // shards of one process, possibly sharing a GPU: device copies
  kHosted,  // rank engine with caller-supplied host callbacks (sthk_host_comm)
};

// One stream operation of an evaluation (graph mode records these and
// replays them as a CUDA graph).
struct GraphOp {
  enum Kind : int { kKernel, kRecord, kRecordTimed, kWait, kMemset, kMemcpy } kind = kKernel;
  cudaStream_t st = nullptr;
  cudaEvent_t ev = nullptr;
  const void* func = nullptr;
  dim3 grid, block;
  size_t smem = 0;
  std::vector<unsigned char> args;
  void* dst = nullptr;
  const void* src = nullptr;
  size_t bytes = 0;
  int value = 0;
  cudaMemcpyKind ckind = cudaMemcpyDefault;
  // kernels: 1 = programmatic dependency on the previous kernel of the same
  // stream (the kernel waits with griddepcontrol.wait; it may launch while
  // that one drains)
  int dep_kind = 0;
};

struct OpSink final : sthk::LaunchSink {
  std::vector<GraphOp>* ops;
  explicit OpSink(std::vector<GraphOp>* o) : ops(o) {}
  void launch(const void* func, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
              const void* args, size_t arg_bytes) override {
    GraphOp op;
    op.kind = GraphOp::kKernel;
    op.st = st;
    op.func = func;
    op.grid = grid;
    op.block = block;
    op.smem = smem;
    op.args.assign(static_cast<const unsigned char*>(args),
                   static_cast<const unsigned char*>(args) + arg_bytes);
    ops->push_back(std::move(op));
  }
};

// An instantiated evaluation graph: its topology signature, the template
// graph (owner of the kernel nodes) and the kernel nodes in issue order with
// the arguments they were last set to.
struct GraphEntry {
  uint64_t sig = 0;
  std::vector<uint64_t> key;  // full topology (ops_topology)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaGraphNode_t> knodes;
  std::vector<std::vector<unsigned char>> kargs;
};

struct sthk_engine {
  std::vector<Slot> slots;
  bool rank_mode = false;
  int rank = 0, world = 1;
  Xport xport = Xport::kSingle;
  // One-shard evaluations are captured into a CUDA graph and launched as one
  // (the instantiated graph is updated in place while its topology holds):
  // one host submission instead of ~20 launch / event calls, and device-side
  // dependencies between the kernels (development knob STHK_GRAPH=0: off).
  bool use_graph = [] {
    const char* v = std::getenv("STHK_GRAPH");
    return !(v && *v == '0');
  }();
  bool recording = false;
  std::vector<GraphOp> ops;    // the evaluation's stream operations, in issue order
  OpSink sink{&ops};
  // instantiated graphs by topology signature (an MH chain alternates a few
  // evaluation shapes: finalize only, trigger sweep, full sweep), most
  // recently used first
  std::vector<GraphEntry> graphs;
  int64_t graph_updates = 0, graph_instantiations = 0;
  sthk_host_comm hcomm{};
  int64_t exch_bytes = 0;  // fx bytes sent to other owners by the last evaluation
  int64_t launches = 0;    // kernels launched by the last evaluation (all slots)
  std::vector<double> ht;  // host copy of times (multi-shard planning only; lazy)
  bool ht_valid = false;
  int64_t n = 0, npad = 0;
  double window_end = 0;
  double p[6] = {0, 0, 0, 0, 0, 0};
  bool loaded = false, has_params = false;
  bool timing = false, dense = false;
  bool timing_pairs = true;  // timing: also the pair-phase events (sthk_set_timing 1; 2: whole evaluation only)
  int mode = sthk::kSym;   // pair-kernel variant (sthk_set_kernel)
  bool far_tier = true;    // far tier of the symmetric kernel (sthk_set_far_tier)
  bool far_fp64 = false;   // ... its list evaluated by the FP64 kernel (same windows)
  bool bg_split = true;    // trigger-free near kernel for stages beyond the trigger window
  // ... its list merged into the general kernel's launch (development knob
  // STHK_MERGE_BG=0/1 at creation)
  bool merge_bg = [] {
    const char* v = std::getenv("STHK_MERGE_BG");
    return v ? *v == '1' : false;
  }();
  // The far kernel runs concurrently with the near (FP64) sweep on a second
  // stream: the near kernel is limited to near_ctas CTAs per SM so that
  // far_ctas_resident far CTAs fit beside it (FP64 and FP32/MUFU pipes busy
  // at once); extra far CTAs queue until near CTAs retire.
  bool far_concurrent = true;
  // trigger sums by row windows when the window is shorter than every tile
  // (development knob STHK_TRIG_ROWS=0 at creation: always the tiled sweep)
  bool trig_rows = [] {
    const char* v = std::getenv("STHK_TRIG_ROWS");
    return v ? *v != '0' : true;
  }();
  bool last_trig_rows = false;
  bool tr_cache_rows = false;
  int far_order = 1;  // 1: far launched first, 2: near first
  int near_ctas = 3, far_ctas = 6;
  double ext_x = 0, ext_y = 0;  // max |x - x[0]|, |y - y[0]| of the loaded set
  double tile_tspan = 0;        // max time span of a 128-event tile
  // adj_gap[k-1]: min over tiles of t[first] - t[first - 128k - 1], the time
  // from a tile's first event back to the last source before its k preceding
  // stages (the trigger-free split keeps those k stages with the tile)
  bool tile_pivots = true;  // plan searches on tile pivots (set at load)
  std::vector<double> adj_gap;
  // span_min[L]: min time span of 2^L consecutive whole tiles (load
  // statistics): bounds the number of events in any time window (far tier)
  std::vector<double> span_min;
  // Background-sum cache: S_B (and S_Br, S_Bt) depend only on the events,
  // tauX, tauT -- fixed for a whole MH chain (sampler.cpp:48-49) -- so while
  // they are unchanged an evaluation sweeps only the trigger band. The
  // fixed chunk grid makes the cached path bitwise identical to a fresh one.
  bool bg_cache = true;
  bool cache_valid = false, cache_grad = false, last_cache_hit = false;
  // Trigger-sum cache (same switch): with the background cached, the trigger
  // partials of the last sweep stay valid while omega and h are unchanged,
  // so an evaluation that moves only mu0 / theta is a finalize pass.
  bool tr_cache_valid = false, tr_cache_grad = false, last_tr_cache_hit = false;
  // compensator terms depend only on (events, tauT, omega)
  bool comp_valid = false;
  uint64_t comp_gen = 0;
  double comp_tt = 0, comp_om = 0;
  double tr_cache_omega = 0, tr_cache_h = 0, tr_cache_dT = 0, tr_cache_dTf = 0;
  bool tr_cache_far_tr = false;  // the cached sweep stored far-tier trigger partials
  uint64_t load_gen = 0, cache_gen = 0;
  bool load_zero_copy = false;  // the last load read pinned caller arrays in place
  // last evaluation plan and its inputs (make_plan is a pure function of
  // them; repeated evaluations at the same parameters skip ~1.5 us of host work)
  std::unique_ptr<EvalPlan> plan_memo;
  double plan_memo_p[6] = {};
  uint64_t plan_memo_gen = 0;
  int plan_memo_shards = 0;
  int plan_memo_flags = -1;
  double cache_tx = 0, cache_tt = 0;
  int cache_mode = -1;
  bool cache_dense = false;
  bool cache_far_full = false;
  bool cache_far_fp64 = false;
  double cache_tfar = 0.0;
  int cache_bg_adj = 0;
  std::vector<int> cache_cuts;  // shard cuts the cached sums were combined under
  std::string err;
  bool pending = false, last_grad = false, last_pe = false, last_ex = false;
  int last_sc = 0, last_items_est = 0;
  double last_far_a = 0.0, last_tfar = 0.0;
};

namespace {

constexpr int kChunksTarget = 64;  // source chunks across N (work-item granularity; measured 32/48/64/96)
// Far tier: a stage runs in FP32 when every exponent on its bounding boxes is
// below -kFarExponent (terms < 4.3e-18), and only if the FP32 coordinates
// (space relative to event 0, time relative to each 128-event tile's first
// event, in kernel units) stay within kFarCoordMax: a coordinate rounding of
// <= 2.4e-4 units perturbs an exponent near the threshold by < 0.01 (log2),
// i.e. < 1% of a term below 4.3e-18.
constexpr double kFarExponent = 40.0;     // far threshold A: at most (error-bound driven below)
constexpr double kFarExponentMin = 30.0;  // ... and at least
constexpr double kFarRowBound = 1e-13;    // bound on the far tier's error, relative to each S_B
constexpr double kFarCoordMax = 4096.0;
constexpr int kMaxAdj = sthk::kLoadAdj;  // trigger-free split: at most 16 stages kept with the tile
constexpr int64_t kBgSplitMinEvents = 36 * 1024;  // trigger-free split only from 36k events
// plan + prep as one grid up to this many events (graph mode): whole
// evaluation Θ_post / Θ_init, two kernels -> one grid: 1.5k 22.6 -> 20.8 /
// 30.3 -> 27.3 us, 10k 26.4 -> 26.2 / 36.6 -> 32.3 us; at 20k-24k Θ_post
// turns slower (the prep blocks take longer than the plan)
constexpr int64_t kPlanPrepMaxEvents = 16 * 1024;

void set_dev(const Slot& s) { ck(cudaSetDevice(s.dev), "cudaSetDevice"); }

// Main streams of every live engine slot, by device. A load whose device is
// running another engine's evaluation copies the caller's arrays with the
// copy engines instead of the zero-copy gather: the gather kernel would wait
// for SM slots until that evaluation ends, the copies overlap it.
std::mutex g_streams_mu;
std::vector<std::pair<int, cudaStream_t>> g_streams;

void register_stream(int dev, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_streams_mu);
  g_streams.emplace_back(dev, st);
}

void unregister_stream(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_streams_mu);
  g_streams.erase(std::remove_if(g_streams.begin(), g_streams.end(),
                                 [&](const std::pair<int, cudaStream_t>& v) {
                                   return v.second == st;
                                 }),
                  g_streams.end());
}

bool device_busy_elsewhere(int dev, cudaStream_t own) {
  std::lock_guard<std::mutex> lk(g_streams_mu);
  bool busy = false;
  for (const auto& v : g_streams) {
    if (v.first == dev && v.second != own && cudaStreamQuery(v.second) == cudaErrorNotReady) {
      busy = true;
      break;
    }
  }
  (void)cudaGetLastError();
  return busy;
}

void init_slot(Slot& s, int dev) {
  s.dev = dev;
  set_dev(s);
  ck(cudaDeviceGetAttribute(&s.sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
  ck(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "stream");
  ck(cudaStreamCreateWithFlags(&s.stream2, cudaStreamNonBlocking), "stream");
  register_stream(dev, s.stream);
  ck(cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&s.prepped, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&s.pairs_done, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&s.trow_ev, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&s.fin_done, cudaEventDisableTiming), "event");
  for (auto& e : s.ev) ck(cudaEventCreate(&e), "event");
  ck(cudaMalloc(&s.scalars, 16 * sizeof(int)), "cudaMalloc");
  ck(cudaMemset(s.scalars, 0, 16 * sizeof(int)), "memset");
  ck(cudaHostAlloc(&s.h_bad, sizeof(unsigned long long),
                   cudaHostAllocMapped | cudaHostAllocPortable),
     "cudaHostAlloc");
  ck(cudaHostAlloc(&s.h_stats, sizeof(double) * sthk::kLoadStats,
                   cudaHostAllocMapped | cudaHostAllocPortable),
     "cudaHostAlloc");
  // the load checks' device minimum starts (and is re-armed) at all ones
  ck(cudaMemset(s.scalars + 4, 0xff, sizeof(unsigned long long)), "memset");
  ck(cudaMalloc(&s.pair_counts, sthk::kNCounts * sizeof(unsigned long long)), "cudaMalloc");
  ck(cudaMemset(s.pair_counts, 0, sthk::kNCounts * sizeof(unsigned long long)), "memset");
  {
    std::vector<unsigned long long> ls(sthk::kLoadStats, 0x7ff0000000000000ULL);
    std::fill(ls.begin(), ls.begin() + 3, 0ULL);
    ck(cudaMalloc(&s.load_dstats, sizeof(unsigned long long) * ls.size()), "cudaMalloc");
    ck(cudaMemcpy(s.load_dstats, ls.data(), sizeof(unsigned long long) * ls.size(),
                  cudaMemcpyHostToDevice), "H2D");
  }
  {
    const unsigned long long init[4] = {~0ULL, 0ULL, ~0ULL, 0ULL};
    ck(cudaMalloc(&s.tstamp, sizeof(init)), "cudaMalloc");
    ck(cudaMemcpy(s.tstamp, init, sizeof(init), cudaMemcpyHostToDevice), "H2D");
    ck(cudaHostAlloc(&s.h_tstamp, sizeof(init), cudaHostAllocMapped | cudaHostAllocPortable),
       "cudaHostAlloc");
    ck(cudaHostGetDevicePointer(&s.d_htstamp, s.h_tstamp, 0), "cudaHostGetDevicePointer");
    std::fill(s.h_tstamp, s.h_tstamp + 4, 0ULL);
  }
  if (item_trace_cap() > 0) {
    ck(cudaMalloc(&s.trace, (4 + 4 * static_cast<size_t>(item_trace_cap())) * sizeof(unsigned long long)),
       "cudaMalloc");
  }
  // results and counters are written by the last kernel straight into
  // device-mapped pinned memory: no D2H copy on the evaluation's stream
  constexpr unsigned kMapped = cudaHostAllocMapped | cudaHostAllocPortable;
  ck(cudaHostAlloc(&s.h_out, kNOut * sizeof(double), kMapped), "cudaHostAlloc");
  ck(cudaHostAlloc(&s.h_counts, sthk::kNCounts * sizeof(unsigned long long), kMapped),
     "cudaHostAlloc");
  ck(cudaHostGetDevicePointer(&s.d_hout, s.h_out, 0), "cudaHostGetDevicePointer");
  ck(cudaHostGetDevicePointer(&s.d_hcounts, s.h_counts, 0), "cudaHostGetDevicePointer");
  std::fill(s.h_out, s.h_out + kNOut, 0.0);
  std::fill(s.h_counts, s.h_counts + sthk::kNCounts, 0ULL);
  for (int m = 0; m < 2; ++m) {
    s.occ[m][1] = sthk::pair_kernel_occupancy(true, m);
    s.occ[m][0] = sthk::pair_kernel_occupancy(false, m);
    s.occ_far[1] = sthk::far_kernel_occupancy(true);
    s.occ_far[0] = sthk::far_kernel_occupancy(false);
    s.occ_bg[1] = sthk::bgonly_kernel_occupancy(true);
    s.occ_bg[0] = sthk::bgonly_kernel_occupancy(false);
  }
  ck(cudaGetLastError(), "occupancy");
}

void free_slot(Slot& s) {
  cudaSetDevice(s.dev);
  if (s.stream) {
    cudaStreamSynchronize(s.stream);
    unregister_stream(s.stream);
  }
  if (s.comm) ncclCommDestroy(s.comm);
  for (void* p : {static_cast<void*>(s.x), static_cast<void*>(s.y), static_cast<void*>(s.t),
                  static_cast<void*>(s.xs), static_cast<void*>(s.ys), static_cast<void*>(s.tsl),
                  static_cast<void*>(s.xf), static_cast<void*>(s.yf), static_cast<void*>(s.tf),
                  static_cast<void*>(s.ranges_far), static_cast<void*>(s.crange_far),
                  static_cast<void*>(s.items_far), static_cast<void*>(s.tpart_far),
                  static_cast<void*>(s.tile_trange), static_cast<void*>(s.comp),
                  static_cast<void*>(s.piv),
                  static_cast<void*>(s.ranges_bg), static_cast<void*>(s.crange_bg),
                  static_cast<void*>(s.items_bg),
                  static_cast<void*>(s.ranges), static_cast<void*>(s.counts),
                  static_cast<void*>(s.items), static_cast<void*>(s.scalars),
                  static_cast<void*>(s.fx), static_cast<void*>(s.block_partial),
                  static_cast<void*>(s.tpart), static_cast<void*>(s.crange),
                  static_cast<void*>(s.trow),
                  static_cast<void*>(s.ex),
                  static_cast<void*>(s.per_event),
                  static_cast<void*>(s.pair_counts), static_cast<void*>(s.tile_box),
                  static_cast<void*>(s.fx_stage), static_cast<void*>(s.pi_sum),
                  static_cast<void*>(s.pi_bad), static_cast<void*>(s.pi_rows),
                  static_cast<void*>(s.trace), static_cast<void*>(s.tstamp),
                  static_cast<void*>(s.load_dstats)}) {
    if (p) cudaFree(p);
  }
  for (void* p : {static_cast<void*>(s.h_out), static_cast<void*>(s.h_counts),
                  static_cast<void*>(s.h_bad), static_cast<void*>(s.h_stats),
                  static_cast<void*>(s.h_per_event), static_cast<void*>(s.h_ex),
                  static_cast<void*>(s.h_pi_rows), static_cast<void*>(s.h_tstamp)}) {
    if (p) cudaFreeHost(p);
  }
  for (auto& e : s.ev) {
    if (e) cudaEventDestroy(e);
  }
  if (s.stream2) cudaStreamSynchronize(s.stream2);
  if (s.fork) cudaEventDestroy(s.fork);
  if (s.join) cudaEventDestroy(s.join);
  if (s.prepped) cudaEventDestroy(s.prepped);
  if (s.pairs_done) cudaEventDestroy(s.pairs_done);
  if (s.trow_ev) cudaEventDestroy(s.trow_ev);
  if (s.fin_done) cudaEventDestroy(s.fin_done);
  if (s.stream2) cudaStreamDestroy(s.stream2);
  if (s.stream) cudaStreamDestroy(s.stream);
}

// Params::validate, types.hpp:59-72.
void validate_params(const double* p) {
  auto pos = [](double v) { return std::isfinite(v) && v > 0.0; };
  if (!(pos(p[0]) && pos(p[1]) && pos(p[2]) && pos(p[4]) && pos(p[5]) &&
        std::isfinite(p[3]) && p[3] >= 0.0)) {
    throw InvalidArg(
        "Params: mu0, tauX, tauT, omega, h must be positive and finite; "
        "theta must be nonnegative and finite");
  }
}

// EventSet constructor checks, types.hpp:85-109. The O(1) argument checks
// run on the host; the per-event checks (finite, t >= 0, nondecreasing) run
// on the device inside the tile-box pass over the uploaded copy, which
// reports the first failing index; the message for it is rebuilt here in the
// reference's order (non-finite, negative, unsorted), then windowEnd.
void validate_event_args(const double* x, const double* y, const double* t, int64_t n) {
  if (n < 1) throw InvalidArg("EventSet: need at least one event");
  if (!x || !y || !t) throw InvalidArg("EventSet: coordinate/time length mismatch");
  // The fixed-point background sums (sthk_device.cuh fx_add) hold per-row
  // totals below 2^23; a row's S_B can reach N (every term <= 1).
  if (n > (int64_t{1} << 23)) throw InvalidArg("sthk: at most 2^23 events supported");
}

[[noreturn]] void throw_event_error(const double* x, const double* y, const double* t, int64_t i) {
  if (!std::isfinite(x[i]) || !std::isfinite(y[i]) || !std::isfinite(t[i])) {
    throw InvalidArg("EventSet: non-finite entry at index " + std::to_string(i));
  }
  if (t[i] < 0.0) throw InvalidArg("EventSet: negative time at index " + std::to_string(i));
  throw InvalidArg("EventSet: times not sorted at index " + std::to_string(i));
}

void validate_window_end(const double* t, int64_t n, double window_end) {
  if (!std::isfinite(window_end) || window_end < t[n - 1]) {
    throw InvalidArg("EventSet: windowEnd precedes last event");
  }
}

struct EvalPlan {
  sthk::PairConsts k;
  double sx = 1.0;  // kSym coordinate scale sqrt(-cxL)
  double stl = 1.0;  // kSym trigger-free kernel time scale sqrt(-ctL)
  double sxf = 1.0, stf = 1.0;  // far-tier FP32 coordinate scales
  double tfar = 0.0;            // far split time gap (days)
  double boost = 0.0;           // ln(trNorm / (mu0 bgNorm)) when > 0
  double far_a = 0.0;           // far threshold A actually used
  int sc = 0;
  int nchunks = 0;
  int sc_bg = 0;       // chunk size of the background-only list (finer: a function of N only)
  int nchunks_bg = 0;
  int sc_far = 0;      // chunk size of the far list (finer: a function of N only)
  int nchunks_far = 0;
  std::vector<int> cuts;  // shard row boundaries (size shards+1)
};

constexpr double kFarPairCost = 0.4;     // FP32 far pair vs FP64 near pair (208 vs 485 instr / 16 pairs)
constexpr double kNearExponentNominal = 35.0;  // partition cost only: typical far threshold A

// ln(trNorm / (mu0 bgNorm)) when positive, else 0 -- the trigger's weight in
// lambda against the background self term's (kernels.hpp:78-84) -- rounded
// up to an integer. Every window built on it is conservative in the boost,
// and the rounding makes the windows (and the sweep caches keyed on them)
// move only in whole steps as theta and mu0 move.
double trigger_boost(const double* p) {
  const double kPi_ = 3.14159265358979323846;
  const double cB = p[0] * std::pow(2.0 * kPi_, -1.5) / (p[1] * p[1] * p[2]);
  const double cT = p[3] * p[4] / (2.0 * kPi_ * p[5] * p[5]);
  return cT > cB ? std::ceil(std::log(cT / cB)) : 0.0;
}

double far_cull_exponent(int64_t n);
int64_t lb(const std::vector<double>& t, int64_t n, double v);
int64_t ub(const std::vector<double>& t, int64_t n, double v);

// Cost-balanced partition of the rows into `shards` contiguous ranges cut at
// 1024-row block boundaries (the reference's contiguous target blocks,
// backend.hpp:139-166). The cost model uses only the background windows --
// functions of (events, tauT, N), which the reference MH sampler keeps fixed
// (sampler.cpp:48-49) -- so the cuts do not move with mu0, theta, omega, h
// and the cached background sums of a shard's rows stay valid across a chain.
// A row block costs its live source width times its rows; in symmetric
// sweeps the width ends at the block (sources J <= I), and far-tier pairs
// (FP32) are charged kFarPairCost of an FP64 near pair.
std::vector<int> plan_cuts(const std::vector<double>& ht, int64_t n, const double* p, bool dense,
                           bool sym, bool far, int shards) {
  std::vector<int> cuts(shards + 1, 0);
  cuts[shards] = static_cast<int>(n);
  if (shards <= 1) return cuts;
  const int64_t nb = (n + kRB - 1) / kRB;
  const double dB = p[2] * std::sqrt(2.0 * sthk::kCullExponent);
  const double dnear = p[2] * std::sqrt(2.0 * kNearExponentNominal);
  const double dfar = p[2] * std::sqrt(2.0 * far_cull_exponent(n));
  std::vector<double> cost(nb);
  double tot = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t first = b * kRB, last = std::min(first + kRB, n) - 1;
    double w;
    if (dense) {
      w = static_cast<double>(sym ? last + 1 : n);
    } else if (sym && far) {
      const int64_t near_lo = lb(ht, n, ht[first] - dnear), far_lo = lb(ht, n, ht[first] - dfar);
      w = static_cast<double>(last + 1 - near_lo) + kFarPairCost * static_cast<double>(near_lo - far_lo);
    } else {
      const int64_t lo = lb(ht, n, ht[first] - dB);
      const int64_t hi = sym ? last + 1 : ub(ht, n, ht[last] + dB);
      w = static_cast<double>(hi - lo);
    }
    cost[b] = std::max(w, 1.0) * static_cast<double>(last - first + 1);
    tot += cost[b];
  }
  double run = 0;
  int64_t b = 0;
  for (int s = 1; s < shards; ++s) {
    const double target = tot * s / shards;
    while (b < nb && run + 0.5 * cost[b] < target) run += cost[b++];
    cuts[s] = static_cast<int>(std::min<int64_t>(b * kRB, n));
  }
  return cuts;
}

// Culling windows: the background term is exactly 0 when |dt| > dB (fexp
// flushes below -708.40; we cut at -709). The trigger term is cut at
// dt > dT, the nearer of its exact underflow (omega dt > 709) and the
// half-ulp window omega dt > C + boost (C = ln N + 54 ln 2): lambda >=
// mu0 bgNorm S_B >= mu0 bgNorm, so the skipped trigger terms sum, over at
// most N sources, to < 2^-54 lambda -- invisible in FP64. The
// boost is a whole number (trigger_boost), so the window (and with it the
// trigger sums, cached per window) moves only in whole steps.
int64_t max_events_in_window(const std::vector<double>* span_min, int64_t n, double w);

// Half-ulp cull exponents, tighter than C = ln N + 54 ln 2
// wherever the load statistics bound the events per time window. Culled
// terms lie beyond a time cut d; split that region into shells of width w:
// each holds at most M(w) events per side (max_events_in_window), and the
// exponent grows by at least a = d w / tauT^2 (background, Gaussian in dt)
// or omega w (trigger, exponential) per shell, so the culled terms of one
// event total at most K e^-z with K = sides * M(w) / (1 - e^-a). With
// z = ln K + 54 ln 2 that is below half an ulp of S_B (and of lambda for the
// trigger, after its boost). zb: background (two-sided), zt: trigger (earlier
// sources only, before adding the boost); both <= C.
void cull_exponents(const std::vector<double>* span, int64_t n, const double* p, double& zb,
                    double& zt) {
  const double ln2 = 0.693147180559945309417232121458176568;
  const double zN = far_cull_exponent(n);
  const double tt2 = p[2] * p[2];
  auto kb = [&](double d) {  // background K at cut d, minimised over shell widths
    double best = static_cast<double>(n);
    for (int k = -3; k <= 6; ++k) {
      const double w = std::ldexp(tt2 / d, k);
      const double a = d * w / tt2;
      const double m = static_cast<double>(max_events_in_window(span, n, w));
      best = std::min(best, 2.0 * m / -std::expm1(-a));
    }
    return std::max(best, 1.0);
  };
  // candidate from the cut of C, then made valid at its own (shorter) cut:
  // K only shrinks as the cut moves out, so max(z_c, ln K(d_c) + 54 ln 2) holds
  const double zc = std::min(zN, std::log(kb(p[2] * std::sqrt(2.0 * zN))) + 54.0 * ln2);
  zb = std::min(zN, std::max(zc, std::log(kb(p[2] * std::sqrt(2.0 * zc))) + 54.0 * ln2));
  double kt = static_cast<double>(n);
  for (int k = -3; k <= 6; ++k) {
    const double w = std::ldexp(1.0 / p[4], k);
    const double m = static_cast<double>(max_events_in_window(span, n, w));
    kt = std::min(kt, m / -std::expm1(-p[4] * w));
  }
  zt = std::min(zN, std::log(std::max(kt, 1.0)) + 54.0 * ln2);
}

void culling_windows(const double* p, int64_t n, const std::vector<double>* span, double& dB,
                     double& dT) {
  dB = p[2] * std::sqrt(2.0 * sthk::kCullExponent) * (1.0 + 1e-9);
  double zb, zt;
  cull_exponents(span, n, p, zb, zt);
  dT = std::min(sthk::kCullExponent, zt + trigger_boost(p)) / p[4] * (1.0 + 1e-9);
}

int64_t lb(const std::vector<double>& t, int64_t n, double v) {
  return std::lower_bound(t.begin(), t.begin() + n, v) - t.begin();
}
int64_t ub(const std::vector<double>& t, int64_t n, double v) {
  return std::upper_bound(t.begin(), t.begin() + n, v) - t.begin();
}

struct PlanInput {
  const std::vector<double>& ht;
  int64_t n, npad;
  const double* p;
  bool dense;
  bool sym;
  bool far;  // far tier enabled (partition cost)
  // load statistics (far-tier error bound): max |x - x0|, |y - y0|, tile time span
  double ext_x = 0, ext_y = 0, tile_tspan = 0;
  const std::vector<double>* span_min = nullptr;  // (see sthk_engine::span_min)
};

// Upper bound on the number of events in any time window of length w, from
// the load statistics: a window holding (2^L + 1) * 128 events contains 2^L
// consecutive whole tiles, whose span is then <= w; so if every such run
// spans more than w, the window holds fewer.
int64_t max_events_in_window(const std::vector<double>* span_min, int64_t n, double w) {
  if (span_min) {
    for (size_t L = 0; L < span_min->size(); ++L) {
      if ((*span_min)[L] > w) {
        return std::min<int64_t>(n, ((int64_t{1} << L) + 1) * sthk::kTS - 1);
      }
    }
  }
  return n;
}

// (development knob: STHK_MIN_CHUNK_STAGES overrides the minimum item length)
int min_chunk_stages() {
  static const int v = [] {
    const char* s = std::getenv("STHK_MIN_CHUNK_STAGES");
    const int k = s ? std::atoi(s) : 0;
    return k >= 1 && k <= 64 ? k : 4;
  }();
  return v;
}

// Row-window evaluations run every near stage in the trigger-free kernel from
// this many events; below it the general kernel (trigger terms off) keeps them
// (measured, whole evaluation at Θ_post: 1.5k-5k events 29.6 vs 23.8 us,
// 10k 34.8 vs 29.7, 20k 49.8 vs 46.4, 36k 88.5 vs 90.0; development knob
// STHK_BG_ALL_MIN overrides it)
constexpr int64_t kBgAllMinEvents = 32 * 1024;
int64_t bg_all_min_events() {
  static const int64_t v = [] {
    const char* s = std::getenv("STHK_BG_ALL_MIN");
    return s ? static_cast<int64_t>(std::atoll(s)) : kBgAllMinEvents;
  }();
  return v;
}

// (development knob: STHK_CHUNKS_TARGET overrides the chunk count target)
int chunks_target() {
  static const int v = [] {
    const char* s = std::getenv("STHK_CHUNKS_TARGET");
    const int k = s ? std::atoi(s) : 0;
    return k >= 1 && k <= 65536 ? k : kChunksTarget;
  }();
  return v;
}

// Small event sets (N <= kOneStageChunkMaxN): one-stage chunks. With few row
// tiles the pair kernels hold fewer items than CTA slots, so an evaluation
// lasts as long as its longest item: measured N = 10k 80.8 -> 56 us, 20k
// 97 -> 75 us per loglik+grad evaluation; neutral at 30-40k, slower from 50k.
constexpr int64_t kOneStageChunkMaxN = 24 * 1024;

int chunk_size(int64_t n, int64_t npad) {
  static const bool target_set = std::getenv("STHK_CHUNKS_TARGET") != nullptr;
  if (n <= kOneStageChunkMaxN && !target_set) {
    return static_cast<int>(std::min<int64_t>(sthk::kTS, npad));
  }
  const int64_t ct = chunks_target();
  int64_t sc = (n + ct - 1) / ct;
  sc = (sc + kTS - 1) / kTS * kTS;
  sc = std::max<int64_t>(sc, static_cast<int64_t>(min_chunk_stages()) * kTS);
  sc = std::min<int64_t>(sc, npad);
  return static_cast<int>(sc);
}

// Far list chunk: a quarter of the trigger partials' chunk grid (a function
// of N only), so the far kernel's tail is finer and each FP32 row partial sums
// fewer terms (the far tier's error bound counts them: A 30.27 -> 30.00 at
// C2). Measured whole evaluation (Θ_post) with sc, sc/2, sc/4: 50k 130.6 /
// 129.5 / 127.0 us, C2 308.1 / 306.5 / 307.2 us, 250k 2.377 / 2.371 / 2.364
// ms, 1M 36.98 / 36.81 / 36.66 ms. Development knob STHK_FAR_DIV.
int far_chunk_size(int64_t n, int64_t npad) {
  static const int div = [] {
    const char* s = std::getenv("STHK_FAR_DIV");
    const int k = s ? std::atoi(s) : 0;
    return k >= 1 && k <= 16 ? k : 4;
  }();
  const int sc = chunk_size(n, npad);
  return std::max(static_cast<int>(kTS), sc / div / kTS * kTS);
}

// Far-tier cull exponent C = ln N + 54 ln 2, capped by the FP32 flush point
// 126 ln 2 + 1: far terms below e^-C sum to < 2^-54 of every row's S_B
// (DESIGN.md §3).
double far_cull_exponent(int64_t n) {
  const double ln2 = 0.693147180559945309417232121458176568;
  return std::min(126.0 * ln2 + 1.0,
                  std::log(static_cast<double>(std::max<int64_t>(n, 2))) + 54.0 * ln2);
}

EvalPlan make_plan(const PlanInput& e, int shards) {
  EvalPlan pl;
  const double* p = e.p;
  double dB, dT;
  culling_windows(p, e.n, e.span_min, dB, dT);
  double zb = 0.0, zt = 0.0;
  cull_exponents(e.span_min, e.n, p, zb, zt);
  // exponent constants in L units (x 2048/ln2), see exp_l (sthk_device.cuh)
  const long double L = 2048.0L / 0.693147180559945309417232121458176568L;
  pl.k.cxL = static_cast<double>(-0.5L * L / (static_cast<long double>(p[1]) * p[1]));
  pl.k.ctL = static_cast<double>(-0.5L * L / (static_cast<long double>(p[2]) * p[2]));
  pl.k.chL = static_cast<double>(-0.5L * L / (static_cast<long double>(p[5]) * p[5]));
  // symmetric kernel: coordinates scaled by sx so that r2 = sx^2 r^2 ~ -cxL r^2
  pl.sx = std::sqrt(-pl.k.cxL);
  pl.stl = static_cast<double>(std::sqrt(0.5L * L) / static_cast<long double>(p[2]));
  pl.k.chS = pl.k.chL / (pl.sx * pl.sx);
  // far tier (FP32, log2 units): xf = (x - x0) sxf, tf = (t - t0) stf
  const double kLn2 = 0.693147180559945309417232121458176568;
  pl.sxf = 1.0 / (p[1] * std::sqrt(2.0 * kLn2));
  pl.stf = 1.0 / (p[2] * std::sqrt(2.0 * kLn2));
  pl.k.fc1 = static_cast<float>(-p[4] / (pl.stf * kLn2));
  pl.k.fc2 = static_cast<float>(-(p[1] * p[1]) / (p[5] * p[5]));
  pl.k.fkr = pl.sx * pl.sx * 2.0 * p[1] * p[1] * kLn2;
  pl.k.fkt1 = 1.0 / pl.stf;
  pl.k.fkt2 = 1.0 / (pl.stf * pl.stf);
  pl.k.fstf = pl.stf;
  // far split: sources earlier than t_tile_first - tfar have every
  // background exponent below -A (dt^2 / 2 tauT^2 >= A) and every trigger
  // term below e^-A relative to the row's background self term: the trigger
  // enters lambda with weight trNorm against mu0 bgNorm for the background,
  // so its cut is omega dt >= A + ln(trNorm / (mu0 bgNorm)) when that ratio
  // exceeds 1 (far-tier error bound).
  {
    const double boost = trigger_boost(p);
    pl.boost = boost;
    // Far threshold A: the FP32 far terms (< e^-A of S_B each, at most N of
    // them per row) carry a relative error eps, bounded from the actual FP32
    // coordinate magnitudes (load statistics), ex2.approx (<= 2 ulp) and the
    // FP32 accumulation of at most one chunk of terms; A is the smallest value
    // in [kFarExponentMin, kFarExponent] keeping N e^-A eps <= kFarRowBound of
    // every row's S_B (1e-13: the loglik moves by < 3e-13 relative at C2).
    const double zc = std::max(zb, zt);
    const double u = std::ldexp(1.0, -24);
    const double dmax = std::sqrt(zc / kLn2);  // max |coordinate difference| of a far pair
    const double sxf = 1.0 / (p[1] * std::sqrt(2.0 * kLn2));
    const double stf = 1.0 / (p[2] * std::sqrt(2.0 * kLn2));
    const double dfar = std::max(p[2] * std::sqrt(2.0 * zc), (zc + boost) / p[4]);
    const double cc = std::max({e.ext_x * sxf, e.ext_y * sxf, (e.tile_tspan + dfar) * stf});
    const double dd = (2.0 * cc + dmax) * u + dmax * u;
    const double dE = 3.0 * (2.0 * dmax * dd + dmax * dmax * u) + 3.0 * dmax * dmax * u;
    const double eps = kLn2 * dE + 4.0 * u + static_cast<double>(far_chunk_size(e.n, e.npad)) * u;
    // far terms in one event's S_B: its far sources (rows) plus the later
    // rows it is a far source of (columns), each within dfar + one tile's
    // span of it, so at most twice the events of such a window (<= N)
    const int64_t far_terms = std::min<int64_t>(
        e.n, 2 * max_events_in_window(e.span_min, e.n, dfar + e.tile_tspan));
    const double a_need =
        std::log(static_cast<double>(std::max<int64_t>(far_terms, 2)) * eps / kFarRowBound);
    pl.far_a = std::min(kFarExponent, std::max(kFarExponentMin, a_need));
    pl.tfar = std::max(p[2] * std::sqrt(2.0 * pl.far_a), (pl.far_a + boost) / p[4]) *
              (1.0 + 1e-9);
  }

  pl.k.nomL = static_cast<double>(-L * p[4]);
  const double inf = std::numeric_limits<double>::infinity();
  pl.k.dB = e.dense ? inf : dB;
  pl.k.dT = dT;  // (dense too: the half-ulp trigger window applies in both modes, so dense == culled)
  // far-tier cull. Every background term has a self term e^0 = 1 in its row's
  // S_B, and lambda >= mu0 bgNorm S_B, so far terms below e^-C relative to
  // that (background exponent < -C; trigger: omega dt > C + ln(trNorm /
  // (mu0 bgNorm))) sum, over at most N sources, to less than N e^-C of S_B.
  // With C = ln N + 54 ln 2 that is below 2^-54 S_B: under half an ulp of
  // S_B, invisible in the FP64 sums, so those pairs are not evaluated. (The
  // FP32 exponent itself underflows to +0 below 126 ln 2 + 1, which caps C.)
  // The same windows apply with culling off (dense), so dense == culled.
  {
    const double zf = 126.0 * kLn2 + 1.0;
    pl.k.dBf = p[2] * std::sqrt(2.0 * zb) * (1.0 + 1e-9);
    pl.k.dTf = std::min(zf, zt + pl.boost) / p[4] * (1.0 + 1e-9);
    // (never beyond the FP64 culling windows)
    pl.k.dBf = std::min(pl.k.dBf, pl.k.dB);
    pl.k.dTf = std::min(pl.k.dTf, pl.k.dT);
    // A trigger term that matters can sit below the FP32 flush point once
    // C + boost > 126 ln 2 + 1 (the far kernel's exponent omits the boost):
    // then every live trigger source stays in the FP64 near list, and the far
    // tier carries background terms only (its trigger window dTf <= tfar).
    if (zt + pl.boost > zf) pl.tfar = std::max(pl.tfar, dT * (1.0 + 1e-9));
  }

  // Chunk size: a function of N only (never of the parameters, the device
  // count or the culling mode). Partial sums are grouped per (tile, chunk), so
  // a fixed chunk grid makes every evaluation path -- fused, trigger-only
  // over a cached background, culled or dense, 1..k devices -- produce the
  // same partials and hence bitwise-identical results.
  const int64_t n = e.n;
  pl.sc = chunk_size(n, e.npad);
  pl.nchunks = static_cast<int>((n + pl.sc - 1) / pl.sc);
  // The trigger-free kernel stores only fixed-point sums, so its items may
  // be finer than the trigger partials' chunk grid: more, shorter items
  // balance its persistent CTAs better (its per-item sums are still grouped
  // by a function of N only, so the background cache stays exact).
  // (measured: half-size items below 64k events, e.g. 14% faster at a 50k
  // cloud; at C2 (85k) and above the full chunk is as fast or faster)
  const int bg_div = n < 64 * 1024 ? 2 : 1;
  pl.sc_bg = std::max(kTS, (pl.sc / bg_div + kTS - 1) / kTS * kTS);
  pl.sc_far = far_chunk_size(n, e.npad);
  pl.nchunks_far = static_cast<int>((n + pl.sc_far - 1) / pl.sc_far);
  pl.nchunks_bg = static_cast<int>((n + pl.sc_bg - 1) / pl.sc_bg);
  pl.cuts = plan_cuts(e.ht, n, p, e.dense, e.sym, e.far, shards);

  return pl;
}

// fxq: per-sum normalisation applied before fixed-point conversion so every
// accumulated sum is O(1) per pair (S_B, S_Br/2tauX^2, S_Bt/2tauT^2, S_T,
// omega S_Tt, S_Tr/2h^2).
void fixed_point_scales(const double* p, double* q) {
  q[0] = 1.0;
  q[1] = 0.5 / (p[1] * p[1]);
  q[2] = 0.5 / (p[2] * p[2]);
  q[3] = 1.0;
  q[4] = p[4];
  q[5] = 0.5 / (p[5] * p[5]);
}

constexpr int kFxRows = 2 * 3;  // fixed-point words per event (3 background sums)

// One owner-directed transfer of fixed-point background sums: rows
// [row, row + len) of shard `from`'s accumulators go to their owner `to`.
struct FxXfer {
  int from, to;
  int64_t row, len;
};

// First source row a shard's symmetric sweep can touch (its column sums land
// on rows >= this): the live-range start of plan_kernel's tile_plan for the
// shard's first tile -- the far tier's culled start when the far list is on
// -- and, for the globally last (partial) tile, its own exact-window start;
// every start is monotone in the tile. One stage of slack below the
// stage-aligned start keeps the host computation conservative (extra rows
// carry zeros).
int64_t sweep_floor(const sthk_engine& e, const EvalPlan& pl, bool far_on, int row0, int row1) {
  if (e.dense) return 0;
  auto start = [&](int64_t first) {
    const int64_t last = std::min<int64_t>(first + kTM, e.n) - 1;
    const double tmin = e.ht[first];
    int64_t lo = std::min(lb(e.ht, e.n, tmin - std::max(pl.k.dB, pl.k.dT)), first);
    if (far_on && last + 1 - first == kTM) {
      const int64_t bb = lb(e.ht, e.n, tmin - pl.tfar);
      const int64_t fb = std::max(lo, bb - bb % kTS);
      const int64_t b1 = lb(e.ht, e.n, tmin - std::max(pl.k.dBf, pl.k.dTf));
      lo = std::min(std::max(lo, b1), fb);
    }
    return lo;
  };
  int64_t lo = start(row0);
  const int64_t last_tile = (static_cast<int64_t>(row1) - 1) / kTM * kTM;
  if (e.n % kTM != 0 && row1 == e.n) lo = std::min(lo, start(last_tile));
  return std::max<int64_t>(0, lo / kTS * kTS - kTS);
}

std::vector<FxXfer> fx_transfers(const sthk_engine& e, const EvalPlan& pl, bool far_on,
                                 int shards) {
  std::vector<FxXfer> v;
  for (int r = 1; r < shards; ++r) {
    if (pl.cuts[r] >= pl.cuts[r + 1]) continue;
    const int64_t lo = sweep_floor(e, pl, far_on, pl.cuts[r], pl.cuts[r + 1]);
    for (int o = 0; o < r; ++o) {
      const int64_t a = std::max<int64_t>(lo, pl.cuts[o]);
      const int64_t b = std::min<int64_t>(pl.cuts[o + 1], pl.cuts[r]);
      if (b > a) v.push_back({r, o, a, b - a});
    }
  }
  return v;
}

// Owner-directed exchange of the fixed-point background sums after the pair
// kernels (symmetric full sweeps with several shards). Every transport moves
// the same segments along the same routes and ends with fx_accumulate on
// the owner, so a shard's own rows end up holding exactly the single-shard
// sums (integer addition).
void exchange_fx(sthk_engine& e, const std::vector<FxXfer>& xf) {
  e.exch_bytes = 0;
  const int nslots = static_cast<int>(e.slots.size());
  auto slot_of = [&](int shard) -> int {  // local slot running `shard`, or -1
    for (int i = 0; i < nslots; ++i) {
      if (e.slots[i].shard == shard) return i;
    }
    return -1;
  };
  // receive-side staging layout: per owner, its incoming segments in order
  std::vector<std::vector<sthk::FxSeg>> segs(nslots);
  std::vector<int64_t> need(nslots, 0);
  std::vector<std::vector<int>> seg_xfer(nslots);
  for (size_t i = 0; i < xf.size(); ++i) {
    const int sf = slot_of(xf[i].from);
    if (sf >= 0) e.exch_bytes += 6 * 8 * xf[i].len;
    const int st = slot_of(xf[i].to);
    if (st < 0) continue;
    segs[st].push_back({xf[i].row, xf[i].len, need[st]});
    seg_xfer[st].push_back(static_cast<int>(i));
    need[st] += 6 * xf[i].len;
  }
  for (int i = 0; i < nslots; ++i) {
    if (need[i] == 0) continue;
    Slot& s = e.slots[i];
    set_dev(s);
    dev_grow(s.fx_stage, s.fx_stage_cap, static_cast<size_t>(need[i]));
  }
  const size_t seg_bytes_per_row = sizeof(unsigned long long);
  if (e.xport == Xport::kLocal) {
    for (int i = 0; i < nslots; ++i) {
      Slot& d = e.slots[i];
      if (segs[i].empty()) continue;
      set_dev(d);
      for (size_t k = 0; k < segs[i].size(); ++k) {
        const FxXfer& x = xf[seg_xfer[i][k]];
        const Slot& src = e.slots[slot_of(x.from)];
        ck(cudaStreamWaitEvent(d.stream, src.pairs_done, 0), "wait");
        for (int w = 0; w < kFxRows; ++w) {
          unsigned long long* dst = d.fx_stage + segs[i][k].off + w * x.len;
          const unsigned long long* from = src.fx + static_cast<size_t>(w) * e.npad + x.row;
          const size_t bytes = seg_bytes_per_row * static_cast<size_t>(x.len);
          if (src.dev == d.dev) {
            ck(cudaMemcpyAsync(dst, from, bytes, cudaMemcpyDeviceToDevice, d.stream), "fx copy");
          } else {
            ck(cudaMemcpyPeerAsync(dst, d.dev, from, src.dev, bytes, d.stream), "fx peer copy");
          }
        }
      }
    }
  } else if (e.xport == Xport::kNccl) {
    ckn(ncclGroupStart(), "ncclGroupStart");
    for (int i = 0; i < nslots; ++i) {
      Slot& s = e.slots[i];
      for (const FxXfer& x : xf) {
        if (x.from != s.shard) continue;
        for (int w = 0; w < kFxRows; ++w) {
          ckn(ncclSend(s.fx + static_cast<size_t>(w) * e.npad + x.row, static_cast<size_t>(x.len),
                       ncclUint64, x.to, s.comm, s.stream),
              "ncclSend(fx)");
        }
      }
      for (size_t k = 0; k < segs[i].size(); ++k) {
        const FxXfer& x = xf[seg_xfer[i][k]];
        for (int w = 0; w < kFxRows; ++w) {
          ckn(ncclRecv(s.fx_stage + segs[i][k].off + w * x.len, static_cast<size_t>(x.len),
                       ncclUint64, x.from, s.comm, s.stream),
              "ncclRecv(fx)");
        }
      }
    }
    ckn(ncclGroupEnd(), "ncclGroupEnd");
  } else if (e.xport == Xport::kHosted) {
    Slot& s = e.slots[0];
    set_dev(s);
    std::vector<std::vector<unsigned long long>> sbuf;
    std::vector<int> speer, rpeer;
    std::vector<const void*> sptr;
    std::vector<void*> rptr;
    std::vector<int64_t> sbytes, rbytes;
    for (const FxXfer& x : xf) {
      if (x.from != s.shard) continue;
      sbuf.emplace_back(static_cast<size_t>(6 * x.len));
      for (int w = 0; w < kFxRows; ++w) {
        ck(cudaMemcpyAsync(sbuf.back().data() + w * x.len,
                           s.fx + static_cast<size_t>(w) * e.npad + x.row,
                           seg_bytes_per_row * static_cast<size_t>(x.len), cudaMemcpyDeviceToHost,
                           s.stream),
           "D2H fx");
      }
      speer.push_back(x.to);
      sbytes.push_back(6 * 8 * x.len);
    }
    std::vector<unsigned long long> rbuf(static_cast<size_t>(need[0]));
    for (size_t k = 0; k < segs[0].size(); ++k) {
      const FxXfer& x = xf[seg_xfer[0][k]];
      rpeer.push_back(x.from);
      rptr.push_back(rbuf.data() + segs[0][k].off);
      rbytes.push_back(6 * 8 * x.len);
    }
    for (auto& b : sbuf) sptr.push_back(b.data());
    ck(cudaStreamSynchronize(s.stream), "D2H fx");
    if (e.hcomm.exchange(e.hcomm.ctx, static_cast<int>(speer.size()), speer.data(), sptr.data(),
                         sbytes.data(), static_cast<int>(rpeer.size()), rpeer.data(), rptr.data(),
                         rbytes.data()) != 0) {
      throw CommErr("sthk: host exchange callback failed");
    }
    if (need[0] > 0) {
      ck(cudaMemcpyAsync(s.fx_stage, rbuf.data(), sizeof(unsigned long long) * rbuf.size(),
                         cudaMemcpyHostToDevice, s.stream),
         "H2D fx");
    }
    ck(cudaStreamSynchronize(s.stream), "H2D fx");  // (rbuf is pageable and local)
  }
  for (int i = 0; i < nslots; ++i) {
    Slot& s = e.slots[i];
    set_dev(s);
    for (size_t k0 = 0; k0 < segs[i].size(); k0 += sthk::kMaxFxSegs) {
      sthk::FxAccArgs aa{};
      aa.fx = s.fx;
      aa.npad = e.npad;
      aa.stage = s.fx_stage;
      aa.nseg = static_cast<int>(std::min<size_t>(sthk::kMaxFxSegs, segs[i].size() - k0));
      for (int k = 0; k < aa.nseg; ++k) aa.seg[k] = segs[i][k0 + k];
      ck(sthk::launch_fx_accumulate(aa, s.stream), "fx accumulate");
      e.launches += 1;
    }
  }
}

// Combination of the per-block partials (each block has exactly one
// non-zero contributor, so every transport is exact), then the fixed-order
// final sum into the host-mapped result.
void combine_blocks(sthk_engine& e, int nb_total) {
  const size_t words = static_cast<size_t>(nb_total) * kNOut;
  if (e.xport == Xport::kNccl) {
    ckn(ncclGroupStart(), "ncclGroupStart");
    for (Slot& s : e.slots) {
      ckn(ncclAllReduce(s.block_partial, s.block_partial, words, ncclDouble, ncclSum, s.comm,
                        s.stream),
          "ncclAllReduce(blocks)");
    }
    ckn(ncclGroupEnd(), "ncclGroupEnd");
  } else if (e.xport == Xport::kHosted) {
    Slot& s = e.slots[0];
    set_dev(s);
    std::vector<double> hb(words);
    ck(cudaMemcpyAsync(hb.data(), s.block_partial, sizeof(double) * words, cudaMemcpyDeviceToHost,
                       s.stream),
       "D2H blocks");
    ck(cudaStreamSynchronize(s.stream), "D2H blocks");
    if (e.hcomm.allreduce_sum(e.hcomm.ctx, hb.data(), static_cast<int64_t>(words),
                              STHK_DTYPE_F64) != 0) {
      throw CommErr("sthk: host all-reduce callback failed");
    }
    ck(cudaMemcpyAsync(s.block_partial, hb.data(), sizeof(double) * words, cudaMemcpyHostToDevice,
                       s.stream),
       "H2D blocks");
    ck(cudaStreamSynchronize(s.stream), "H2D blocks");
  } else if (e.xport == Xport::kLocal) {
    // gather every shard's own blocks into slot 0 (the one that is read)
    Slot& s0 = e.slots[0];
    set_dev(s0);
    for (size_t i = 1; i < e.slots.size(); ++i) {
      const Slot& s = e.slots[i];
      if (s.row1 <= s.row0) continue;
      ck(cudaStreamWaitEvent(s0.stream, s.fin_done, 0), "wait");
      const size_t b0 = static_cast<size_t>(s.row0 / sthk::kFB);
      const size_t b1 = static_cast<size_t>((s.row1 + sthk::kFB - 1) / sthk::kFB);
      const size_t bytes = sizeof(double) * kNOut * (b1 - b0);
      if (s.dev == s0.dev) {
        ck(cudaMemcpyAsync(s0.block_partial + b0 * kNOut, s.block_partial + b0 * kNOut, bytes,
                           cudaMemcpyDeviceToDevice, s0.stream),
           "block copy");
      } else {
        ck(cudaMemcpyPeerAsync(s0.block_partial + b0 * kNOut, s0.dev, s.block_partial + b0 * kNOut,
                               s.dev, bytes, s0.stream),
           "block peer copy");
      }
    }
  }
  for (size_t i = 0; i < e.slots.size(); ++i) {
    Slot& s = e.slots[i];
    set_dev(s);
    const bool reads_out = e.xport != Xport::kLocal || i == 0;
    ck(sthk::launch_final_sum(s.block_partial, nb_total, reads_out ? s.d_hout : nullptr,
                              e.timing ? s.pair_counts : nullptr, s.d_hcounts, s.stream),
       "final sum");
    e.launches += 1;
  }
}

// Stream operations of an evaluation: issued directly, or recorded while
// the engine builds / replays its evaluation graph.
cudaError_t op_record(sthk_engine& e, cudaEvent_t ev, cudaStream_t st) {
  if (!e.recording) return cudaEventRecord(ev, st);
  GraphOp op;
  op.kind = GraphOp::kRecord;
  op.st = st;
  op.ev = ev;
  e.ops.push_back(std::move(op));
  return cudaSuccess;
}
// (timing events: event-record nodes in a graph)
cudaError_t record_timing(sthk_engine& e, cudaEvent_t ev, cudaStream_t st) {
  if (!e.recording) return cudaEventRecord(ev, st);
  GraphOp op;
  op.kind = GraphOp::kRecordTimed;
  op.st = st;
  op.ev = ev;
  e.ops.push_back(std::move(op));
  return cudaSuccess;
}
cudaError_t op_wait(sthk_engine& e, cudaStream_t st, cudaEvent_t ev) {
  if (!e.recording) return cudaStreamWaitEvent(st, ev, 0);
  GraphOp op;
  op.kind = GraphOp::kWait;
  op.st = st;
  op.ev = ev;
  e.ops.push_back(std::move(op));
  return cudaSuccess;
}
cudaError_t op_memset(sthk_engine& e, void* dst, int value, size_t bytes, cudaStream_t st) {
  if (!e.recording) return cudaMemsetAsync(dst, value, bytes, st);
  GraphOp op;
  op.kind = GraphOp::kMemset;
  op.st = st;
  op.dst = dst;
  op.value = value;
  op.bytes = bytes;
  e.ops.push_back(std::move(op));
  return cudaSuccess;
}
cudaError_t op_memcpy(sthk_engine& e, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                      cudaStream_t st) {
  if (!e.recording) return cudaMemcpyAsync(dst, src, bytes, kind, st);
  GraphOp op;
  op.kind = GraphOp::kMemcpy;
  op.st = st;
  op.dst = dst;
  op.src = src;
  op.bytes = bytes;
  op.ckind = kind;
  e.ops.push_back(std::move(op));
  return cudaSuccess;
}

// (graph mode: annotate the kernel just recorded with a dependency kind, see
// GraphOp::dep_kind; no effect with direct launches)
void mark_last_kernel(sthk_engine& e, int kind) {
  if (!e.recording || e.ops.empty() || e.ops.back().kind != GraphOp::kKernel) return;
  e.ops.back().dep_kind = kind;
}

// Topology of a recorded evaluation: every operation's kind, stream, event,
// and for kernels the function, launch shape and dependency kind, for copies
// and memsets their operands. Kernel arguments are not part of it: they are
// updated in place on a graph of the same topology (looked up by its FNV-1a
// hash, confirmed by comparing the full key).
std::vector<uint64_t> ops_topology(const std::vector<GraphOp>& ops) {
  std::vector<uint64_t> key;
  key.reserve(8 * ops.size() + 1);
  key.push_back(ops.size());
  for (const GraphOp& op : ops) {
    key.push_back(static_cast<uint64_t>(op.kind));
    key.push_back(reinterpret_cast<uint64_t>(op.st));
    key.push_back(reinterpret_cast<uint64_t>(op.ev));
    if (op.kind == GraphOp::kKernel) {
      key.push_back(reinterpret_cast<uint64_t>(op.func));
      key.push_back((static_cast<uint64_t>(op.grid.x) << 32) | op.block.x);
      key.push_back(op.smem);
      key.push_back(op.args.size());
      key.push_back(static_cast<uint64_t>(op.dep_kind));
    } else if (op.kind == GraphOp::kMemset || op.kind == GraphOp::kMemcpy) {
      key.push_back(reinterpret_cast<uint64_t>(op.dst));
      key.push_back(reinterpret_cast<uint64_t>(op.src));
      key.push_back(op.bytes);
      key.push_back(static_cast<uint64_t>(op.value));
      key.push_back(static_cast<uint64_t>(op.ckind));
    }
  }
  return key;
}

uint64_t fnv1a(const std::vector<uint64_t>& key) {
  uint64_t h = 1469598103934665603ULL;
  for (const uint64_t v : key) {
    for (int b = 0; b < 8; ++b) {
      h ^= (v >> (8 * b)) & 0xff;
      h *= 1099511628211ULL;
    }
  }
  return h;
}

// The graph of a recorded operation list: a node per kernel, memset, copy and
// timing-event record; dependencies follow stream order and event waits.
GraphEntry build_graph(const std::vector<GraphOp>& ops) {
  GraphEntry g;
  ck(cudaGraphCreate(&g.graph, 0), "graph create");
  try {
    std::vector<std::pair<cudaStream_t, std::vector<cudaGraphNode_t>>> tail;
    std::vector<std::pair<cudaEvent_t, std::vector<cudaGraphNode_t>>> evn;
    auto tail_of = [&](cudaStream_t st) -> std::vector<cudaGraphNode_t>& {
      for (auto& kv : tail) {
        if (kv.first == st) return kv.second;
      }
      tail.push_back({st, {}});
      return tail.back().second;
    };
    auto ev_of = [&](cudaEvent_t ev) -> std::vector<cudaGraphNode_t>& {
      for (auto& kv : evn) {
        if (kv.first == ev) return kv.second;
      }
      evn.push_back({ev, {}});
      return evn.back().second;
    };
    std::vector<std::pair<cudaStream_t, cudaGraphNode_t>> last_kernel;
    auto last_kernel_of = [&](cudaStream_t st) -> cudaGraphNode_t {
      for (auto& kv : last_kernel) {
        if (kv.first == st) return kv.second;
      }
      return nullptr;
    };
    for (const GraphOp& op : ops) {
      std::vector<cudaGraphNode_t>& deps = tail_of(op.st);
      cudaGraphNode_t nd = nullptr;
      switch (op.kind) {
        case GraphOp::kKernel: {
          cudaKernelNodeParams kp{};
          kp.func = const_cast<void*>(op.func);
          kp.gridDim = op.grid;
          kp.blockDim = op.block;
          kp.sharedMemBytes = static_cast<unsigned>(op.smem);
          void* argp = const_cast<unsigned char*>(op.args.data());
          kp.kernelParams = &argp;
          // programmatic edge from the previous kernel of this stream (taken
          // out of the full-completion dependencies)
          cudaGraphNode_t prog_from = nullptr;
          std::vector<cudaGraphNode_t> full = deps;
          if (op.dep_kind == 1) {
            cudaGraphNode_t prev = last_kernel_of(op.st);
            auto it = std::find(full.begin(), full.end(), prev);
            if (prev && it != full.end()) {
              full.erase(it);
              prog_from = prev;
            }
          }
          ck(cudaGraphAddKernelNode(&nd, g.graph, full.data(), full.size(), &kp), "graph kernel");
          if (prog_from) {
            cudaGraphEdgeData ed{};
            ed.type = cudaGraphDependencyTypeProgrammatic;
            ed.from_port = cudaGraphKernelNodePortProgrammatic;
            ck(cudaGraphAddDependencies_v2(g.graph, &prog_from, &nd, &ed, 1), "graph edge");
          }
          bool found = false;
          for (auto& kv : last_kernel) {
            if (kv.first == op.st) {
              kv.second = nd;
              found = true;
            }
          }
          if (!found) last_kernel.push_back({op.st, nd});
          g.knodes.push_back(nd);
          g.kargs.push_back(op.args);
          break;
        }
        case GraphOp::kMemset: {
          cudaMemsetParams mp{};
          mp.dst = op.dst;
          mp.value = static_cast<unsigned>(op.value);
          mp.elementSize = 1;
          mp.width = op.bytes;
          mp.height = 1;
          ck(cudaGraphAddMemsetNode(&nd, g.graph, deps.data(), deps.size(), &mp), "graph memset");
          break;
        }
        case GraphOp::kMemcpy:
          ck(cudaGraphAddMemcpyNode1D(&nd, g.graph, deps.data(), deps.size(), op.dst, op.src,
                                      op.bytes, op.ckind),
             "graph memcpy");
          break;
        case GraphOp::kRecordTimed:
          ck(cudaGraphAddEventRecordNode(&nd, g.graph, deps.data(), deps.size(), op.ev),
             "graph event");
          break;
        case GraphOp::kRecord:
          ev_of(op.ev) = deps;
          break;
        case GraphOp::kWait: {
          const std::vector<cudaGraphNode_t>& w = ev_of(op.ev);
          for (cudaGraphNode_t x : w) {
            if (std::find(deps.begin(), deps.end(), x) == deps.end()) deps.push_back(x);
          }
          break;
        }
      }
      if (nd) {
        deps.assign(1, nd);
        if (op.kind == GraphOp::kRecordTimed) ev_of(op.ev) = deps;
      }
    }
    ck(cudaGraphInstantiate(&g.exec, g.graph, 0), "graph instantiate");
  } catch (...) {
    cudaGraphDestroy(g.graph);
    throw;
  }
  return g;
}

// End the recording of a one-shard evaluation and launch it: a graph of the
// same topology gets the new kernel arguments in place (only those that
// changed), else one is built, instantiated and kept (LRU, at most 16).
void launch_recorded(sthk_engine& e, cudaStream_t st) {
  constexpr size_t kMaxGraphs = 16;
  e.recording = false;
  sthk::set_launch_sink(nullptr);
  std::vector<uint64_t> key = ops_topology(e.ops);
  const uint64_t sig = fnv1a(key);
  auto it = std::find_if(e.graphs.begin(), e.graphs.end(),
                         [&](const GraphEntry& g) { return g.sig == sig && g.key == key; });
  if (it != e.graphs.end()) {
    std::rotate(e.graphs.begin(), it, it + 1);  // most recently used first
    GraphEntry& g = e.graphs.front();
    size_t k = 0;
    for (const GraphOp& op : e.ops) {
      if (op.kind != GraphOp::kKernel) continue;
      if (op.args != g.kargs[k]) {
        cudaKernelNodeParams kp{};
        kp.func = const_cast<void*>(op.func);
        kp.gridDim = op.grid;
        kp.blockDim = op.block;
        kp.sharedMemBytes = static_cast<unsigned>(op.smem);
        void* argp = const_cast<unsigned char*>(op.args.data());
        kp.kernelParams = &argp;
        ck(cudaGraphExecKernelNodeSetParams(g.exec, g.knodes[k], &kp), "graph kernel update");
        g.kargs[k] = op.args;
      }
      ++k;
    }
    ++e.graph_updates;
  } else {
    GraphEntry g = build_graph(e.ops);
    g.sig = sig;
    g.key = std::move(key);
    ++e.graph_instantiations;
    if (e.graphs.size() >= kMaxGraphs) {
      cudaGraphExecDestroy(e.graphs.back().exec);
      cudaGraphDestroy(e.graphs.back().graph);
      e.graphs.pop_back();
    }
    e.graphs.insert(e.graphs.begin(), std::move(g));
  }
  ck(cudaGraphLaunch(e.graphs.front().exec, st), "graph launch");
}

void enqueue_eval_body(sthk_engine& e, bool grad, bool want_pe, bool want_ex, bool ex_to_host);

void enqueue_eval(sthk_engine& e, bool grad, bool want_pe, bool want_ex = false,
                  bool ex_to_host = true) {
  try {
    enqueue_eval_body(e, grad, want_pe, want_ex, ex_to_host);
  } catch (...) {
    if (e.recording) {  // nothing of the recorded evaluation was issued
      e.recording = false;
      e.ops.clear();
      sthk::set_launch_sink(nullptr);
    }
    throw;
  }
}

void enqueue_eval_body(sthk_engine& e, bool grad, bool want_pe, bool want_ex, bool ex_to_host) {
  if (!e.loaded) throw NotLoaded("sthk: no events loaded");
  if (!e.has_params) throw NotLoaded("sthk: no parameters set");
  const int shards = e.rank_mode ? e.world : static_cast<int>(e.slots.size());
  const bool sym = e.mode == sthk::kSym;
  if (shards > 1 && !e.ht_valid) {  // the cost-balanced partition needs the times on the host
    Slot& s0 = e.slots[0];
    set_dev(s0);
    e.ht.resize(static_cast<size_t>(e.n));
    ck(cudaMemcpyAsync(e.ht.data(), s0.t, sizeof(double) * e.n, cudaMemcpyDeviceToHost,
                       s0.stream), "D2H");
    ck(cudaStreamSynchronize(s0.stream), "D2H");
    e.ht_valid = true;
  }
  const int plan_flags = (e.dense ? 1 : 0) | (sym ? 2 : 0) | (sym && e.far_tier ? 4 : 0) |
                         (e.ht_valid ? 8 : 0);
  if (!e.plan_memo || e.plan_memo_gen != e.load_gen || e.plan_memo_shards != shards ||
      e.plan_memo_flags != plan_flags || std::memcmp(e.plan_memo_p, e.p, sizeof e.plan_memo_p)) {
    e.plan_memo.reset();  // (stays empty if make_plan throws)
    e.plan_memo = std::make_unique<EvalPlan>(
        make_plan(PlanInput{e.ht, e.n, e.npad, e.p, e.dense, sym, sym && e.far_tier, e.ext_x,
                            e.ext_y, e.tile_tspan, &e.span_min},
                  shards));
    std::memcpy(e.plan_memo_p, e.p, sizeof e.plan_memo_p);
    e.plan_memo_gen = e.load_gen;
    e.plan_memo_shards = shards;
    e.plan_memo_flags = plan_flags;
  }
  const EvalPlan& pl = *e.plan_memo;
  e.last_sc = pl.sc;
  e.last_far_a = pl.far_a;
  e.last_tfar = pl.tfar;
  e.exch_bytes = 0;
  e.launches = 0;
  // Split structure of a full sweep (it fixes how the background sums are
  // grouped, so a cached background is reused only under the same structure):
  //  * far tier on/off and its split tfar;
  //  * the trigger-free near split bg_adj, chosen from the physical trigger
  //    window 709/omega -- not the dense mode's infinite one -- so dense and
  //    culled sweeps split alike; it moves only when omega crosses a
  //    threshold (then the background is recomputed);
  //  * the shard cuts (a shard's accumulators hold its own rows only).
  const bool far_guard = sym && e.far_tier && e.ext_x * pl.sxf <= kFarCoordMax &&
                         e.ext_y * pl.sxf <= kFarCoordMax && e.tile_tspan * pl.stf <= kFarCoordMax;
  const bool far_full = far_guard && !(std::max(pl.k.dB, pl.k.dT) <= pl.tfar);
  // Trigger sums by row windows (trig_rows_kernel) when the trigger's exact
  // underflow window 709/omega -- beyond it every trigger term is +0, in the
  // reference's exp as in ours -- is shorter than every 128-event tile's time
  // span (load statistics) and no trigger term goes to the far tier. Each row
  // then sums every trigger term that is not +0, exactly the reference's set,
  // at a few pairs per row. A function of omega and the load only -- never
  // of the cache state, the shard count or the culling mode -- so every
  // evaluation path sums the same terms alike.
  const double dT_rows = sthk::kCullExponent / e.p[4] * (1.0 + 1e-9);
  const bool tr_rows = sym && e.trig_rows && !e.span_min.empty() && dT_rows < e.span_min[0] &&
                       !(far_full && pl.k.dTf > pl.tfar);
  e.last_trig_rows = tr_rows;
  // With the trigger sums by row windows no near stage has a trigger term:
  // every near stage, the diagonal one included, goes to the trigger-free
  // kernel and the general kernel is not launched (bg_adj -1 in the cache
  // and plan keys: the split fixes each background term's rounding).
  const bool bg_all_struct = tr_rows && e.bg_split && !e.merge_bg && e.n >= bg_all_min_events();
  // (a third kernel only pays off with enough row tiles to amortise its
  // launch and per-CTA setup: measured break-even between N = 30k and 40k)
  int bg_adj = 0;
  if (bg_all_struct) {
    bg_adj = -1;
  } else if (sym && e.bg_split && !e.adj_gap.empty() && e.n >= kBgSplitMinEvents) {
    // (choosing it from the half-ulp window pl.k.dT instead was measured: 6%
    // slower at Theta_init, where the general kernel's fused background +
    // trigger stages beat a trigger-only pass beside the trigger-free kernel)
    const double dT_phys = sthk::kCullExponent / e.p[4] * (1.0 + 1e-9);
    for (int k = 1; k <= kMaxAdj; ++k) {
      if (e.adj_gap[k - 1] > dT_phys) {
        bg_adj = k;
        break;
      }
    }
  }
  const bool cached = e.bg_cache && e.cache_valid && e.cache_gen == e.load_gen &&
                      e.cache_tx == e.p[1] && e.cache_tt == e.p[2] && e.cache_mode == e.mode &&
                      e.cache_far_full == far_full && e.cache_tfar == (far_full ? pl.tfar : 0.0) &&
                      e.cache_far_fp64 == e.far_fp64 &&
                      e.cache_bg_adj == bg_adj && e.cache_dense == e.dense &&
                      e.cache_cuts == pl.cuts && (e.cache_grad || !grad);
  e.last_cache_hit = cached;
  const bool bg_all = !cached && bg_all_struct;
  const bool bg_split = !cached && (bg_adj > 0 || bg_all);
  // (a far list that is provably empty -- every live source within tfar of
  // its tile, e.g. a trigger-only sweep at large omega -- is not planned or
  // launched; results are the same either way)
  const bool far_on = far_full && !(cached && pl.k.dT <= pl.tfar);
  // every far source lies more than tfar before its tile's rows: with the far
  // tier's trigger cull window dTf <= tfar no far trigger term is live, and
  // its (all-zero) trigger partials are neither stored nor summed
  const bool far_tr = far_on && !(pl.k.dTf <= pl.tfar);
  // Trigger sums cached from the last sweep: same omega, h and trigger
  // windows, and the same far-tier trigger split (which fixes whether far
  // trigger partials exist and which chunks finalize sums).
  const bool tr_cached = cached && e.tr_cache_valid && e.tr_cache_omega == e.p[4] &&
                         e.tr_cache_h == e.p[5] && e.tr_cache_dT == pl.k.dT &&
                         e.tr_cache_dTf == pl.k.dTf && e.tr_cache_far_tr == far_tr &&
                         e.tr_cache_rows == tr_rows &&
                         e.tr_cache_grad == grad;  // (tpart layout)
  e.last_tr_cache_hit = tr_cached;
  e.cache_valid = false;  // re-armed below once the sweep is enqueued
  e.tr_cache_valid = false;
  const int64_t ntiles_total = (e.n + kTM - 1) / kTM;
  const int nb_total = static_cast<int>((e.n + sthk::kFB - 1) / sthk::kFB);
  const double* p = e.p;
  const double kPi = 3.14159265358979323846;
  double fxq[sthk::kNSumGrad];
  fixed_point_scales(p, fxq);

  for (size_t si = 0; si < e.slots.size(); ++si) {
    Slot& s = e.slots[si];
    s.row0 = pl.cuts[s.shard];
    s.row1 = pl.cuts[s.shard + 1];
  }

  // compensator terms: cached (exact) while tauT and omega are unchanged
  const bool need_comp = !(e.bg_cache && e.comp_valid && e.comp_gen == e.load_gen &&
                           e.comp_tt == p[2] && e.comp_om == p[4]);
  // trigger-only sweep by row windows over the cached background (h, omega
  // moves): finalize computes each row's trigger sums -- and, when tauT or
  // omega moved, its compensator terms -- itself: one kernel per evaluation
  const bool fin_rows = tr_rows && cached && !tr_cached;
  if (need_comp) e.comp_valid = false;  // re-armed once the prep pass is enqueued
  // Timing in graph mode: kernel-side %globaltimer stamps instead of event
  // nodes, which would sit between the kernels and add their latency.
  const bool graph_mode = e.use_graph && e.xport == Xport::kSingle && e.slots.size() == 1;
  const bool stamps = graph_mode && e.timing;
  // phase 1: zero the accumulators, plan and run the pair kernels per shard
  for (Slot& s : e.slots) {
    s.last_stamps = stamps;
    bool prep_pending = false, prep_unlaunched = false;
    sthk::PrepArgs pr{};
    set_dev(s);
    const int tile0 = s.row0 / kTM;
    const int tile1 = static_cast<int>((s.row1 + kTM - 1) / kTM);
    const int ntiles = std::max(tile1 - tile0, 0);
    dev_grow(s.ranges, s.ranges_cap, static_cast<size_t>(ntiles_total));
    dev_grow(s.items, s.items_cap, static_cast<size_t>(std::max(ntiles, 1)) * pl.nchunks);
    dev_grow(s.fx, s.fx_cap, static_cast<size_t>(kFxRows) * e.npad);
    // (row-window trigger sums: no chunk partials, ~1.5 KB/event less at 1M)
    if (tr_rows) dev_grow(s.trow, s.trow_cap, static_cast<size_t>(3) * e.npad);
    else dev_grow(s.tpart, s.tpart_cap, static_cast<size_t>(pl.nchunks) * 3 * e.npad);
    dev_grow(s.crange, s.crange_cap, static_cast<size_t>(ntiles_total));
    if (bg_split) {
      dev_grow(s.ranges_bg, s.ranges_bg_cap, static_cast<size_t>(ntiles_total));
      dev_grow(s.crange_bg, s.crange_bg_cap, static_cast<size_t>(ntiles_total));
      dev_grow(s.items_bg, s.items_bg_cap,
               static_cast<size_t>(std::max(ntiles, 1)) * pl.nchunks_bg);
    }
    if (far_on) {
      dev_grow(s.ranges_far, s.ranges_far_cap, static_cast<size_t>(ntiles_total));
      dev_grow(s.crange_far, s.crange_far_cap, static_cast<size_t>(ntiles_total));
      dev_grow(s.items_far, s.items_far_cap,
               static_cast<size_t>(std::max(ntiles, 1)) * pl.nchunks_far);
      if (far_tr || e.far_fp64) {
        dev_grow(s.tpart_far, s.tpart_far_cap, static_cast<size_t>(pl.nchunks_far) * 3 * e.npad);
      }
    }
    dev_grow(s.block_partial, s.bp_cap, static_cast<size_t>(nb_total) * kNOut);
    dev_grow(s.comp, s.comp_cap, static_cast<size_t>(4) * e.npad);
    if (want_pe) dev_grow(s.per_event, s.pe_cap, static_cast<size_t>(e.npad));
    if (want_ex) dev_grow(s.ex, s.ex_cap, static_cast<size_t>(3) * e.npad);
    if (sym && bg_split) dev_grow(s.tsl, s.tsl_cap, static_cast<size_t>(e.npad));
    if (want_pe && s.h_pe_cap < static_cast<size_t>(e.npad)) {
      if (s.h_per_event) ck(cudaFreeHost(s.h_per_event), "cudaFreeHost");
      s.h_per_event = nullptr;
      ck(cudaMallocHost(&s.h_per_event, sizeof(double) * e.npad), "cudaMallocHost");
      s.h_pe_cap = static_cast<size_t>(e.npad);
    }
    if (want_ex && ex_to_host && s.h_ex_cap < static_cast<size_t>(3 * e.npad)) {
      if (s.h_ex) ck(cudaFreeHost(s.h_ex), "cudaFreeHost");
      s.h_ex = nullptr;
      ck(cudaMallocHost(&s.h_ex, sizeof(double) * 3 * e.npad), "cudaMallocHost");
      s.h_ex_cap = static_cast<size_t>(3 * e.npad);
    }

    cudaStream_t st = s.stream;
    // (one shard: every stream operation from here on is recorded and
    // replayed as the evaluation graph)
    if (graph_mode && !e.recording) {
      e.ops.clear();
      e.recording = true;
      sthk::set_launch_sink(&e.sink);
    }
    if (e.timing && !stamps) ck(record_timing(e, s.ev[0], st), "event");
    if (s.trace) ck(op_memset(e, s.trace, 0, sizeof(unsigned long long), st), "memset");
    // (pair counters, timing only, are zero here: the final kernel of the
    // previous timed evaluation re-zeroed them after copying them out)
    // one prep pass on stream 2, beside the plan (stream 1): scaled / FP32
    // coordinates (a cached sweep has the same tauX, tauT: copies still
    // valid), zeroed background accumulators, compensator terms
    pr.x = s.x;
    pr.y = s.y;
    pr.t = s.t;
    pr.n = e.n;
    pr.npad = e.npad;
    if (sym && !cached) {
      pr.sx = pl.sx;
      pr.xs = s.xs;
      pr.ys = s.ys;
      if (bg_split) {
        pr.tsl = s.tsl;
        pr.stl = pl.stl;
      }
      if (far_on) {
        pr.sxf = pl.sxf;
        pr.stf = pl.stf;
        pr.xf = s.xf;
        pr.yf = s.yf;
        pr.tf = s.tf;
      }
    }
    if (!cached) pr.fx = s.fx;
    if (need_comp && !fin_rows) {
      pr.comp = s.comp;
      pr.window_end = e.window_end;
      pr.tauT = p[2];
      pr.omega = p[4];
    }
    pr.trace = s.trace;
    pr.trace_cap = item_trace_cap();
    pr.tstamp = stamps ? s.tstamp : nullptr;
    if (pr.xs || pr.fx || pr.comp) {  // (launched right after the plan, see below)
      ck(op_record(e, s.fork, st), "event");
      prep_unlaunched = true;
    }
    if (shards > 1) {
      ck(op_memset(e, s.block_partial, 0, sizeof(double) * nb_total * kNOut, st), "memset");
    }
    // The plan kernel goes first: its few CTAs take whole SMs (1024 threads,
    // the full register file) before the prep pass spreads over the rest, so
    // the plan's latency-bound searches do not queue behind prep traffic.
    auto launch_prep_now = [&] {
      if (!prep_unlaunched) return;
      ck(op_wait(e, s.stream2, s.fork), "wait");
      ck(sthk::launch_prep(pr, s.stream2), "prep");
      e.launches += 1;
      ck(op_record(e, s.prepped, s.stream2), "event");
      prep_unlaunched = false;
      prep_pending = true;
    };
    auto join_prep = [&] {
      if (!prep_pending) return;
      ck(op_wait(e, st, s.prepped), "wait");
      prep_pending = false;
    };
    auto launch_trig_rows = [&](cudaStream_t ts) {
      sthk::TrigRowsArgs ra{};
      ra.xs = s.xs;
      ra.ys = s.ys;
      ra.t = s.t;
      ra.npad = e.npad;
      ra.row0 = s.row0;
      ra.row1 = s.row1;
      ra.nomL = pl.k.nomL;
      ra.chS = pl.k.chS;
      ra.dT = dT_rows;
      ra.trow = s.trow;
      ra.pair_counts = e.timing ? s.pair_counts : nullptr;
      ra.tstamp = stamps ? s.tstamp : nullptr;
      ck(sthk::launch_trig_rows(ra, grad, ts), "trigger rows");
      e.launches += 1;
    };
    if (ntiles == 0 || tr_cached || fin_rows) {
      launch_prep_now();
      join_prep();
      ck(e.timing && e.timing_pairs && !stamps ? record_timing(e, s.ev[1], st)
                                                : op_record(e, s.ev[1], st),
         "event");
      if (e.timing && e.timing_pairs && !stamps) ck(record_timing(e, s.ev[2], st), "event");
      ck(op_record(e, s.pairs_done, st), "event");
      continue;  // (tr_cached: every pair sum is cached, finalize only)
    }
    sthk::PlanArgs pa{};
    pa.t = s.t;
    pa.piv = s.piv;
    pa.tile_trange = s.tile_trange;
    pa.n = e.n;
    pa.tile0 = tile0;
    pa.tile1 = tile1;
    pa.dB = pl.k.dB;
    pa.dT = pl.k.dT;
    pa.dense = e.dense ? 1 : 0;
    pa.sym = sym ? 1 : 0;
    pa.trig_only = cached ? 1 : 0;
    pa.sc = pl.sc;
    pa.tile_order = tr_rows ? 1 : 0;
    pa.sc_far = pl.sc_far;
    pa.nchunks = pl.nchunks;
    pa.ranges = s.ranges;
    pa.crange = s.crange;
    pa.items = s.items;
    pa.n_items = s.scalars;
    pa.work_counter = s.scalars + 1;
    pa.tfar = far_on ? pl.tfar : 0.0;
    pa.tile_pivots = e.tile_pivots ? 1 : 0;
    pa.trace = s.trace;
    pa.trace_cap = item_trace_cap();
    pa.tstamp = stamps ? s.tstamp : nullptr;
    // far list start: the far tier's cull window (trigger-only sweeps: trigger only)
    // (only with a far list: its window then keys the plan cache)
    pa.dFar = !far_on ? 0.0 : cached ? pl.k.dTf : std::max(pl.k.dBf, pl.k.dTf);
    if (bg_split) {
      pa.bg_adj = std::max(bg_adj, 0);
      pa.bg_all = bg_all ? 1 : 0;
      pa.sc_bg = pl.sc_bg;
      pa.ranges_bg = s.ranges_bg;
      pa.crange_bg = s.crange_bg;
      pa.items_bg = s.items_bg;
      pa.n_items_bg = s.scalars + 9;
      pa.work_counter_bg = s.scalars + 10;
    }
    if (far_on) {
      pa.ranges_far = s.ranges_far;
      pa.crange_far = s.crange_far;
      pa.items_far = s.items_far;
      pa.n_items_far = s.scalars + 6;
      pa.work_counter_far = s.scalars + 7;
    }
    const int key[7] = {tile0, tile1, pl.sc, pa.dense, pa.sym, pa.trig_only + 2 * pa.tile_order,
                        bg_split ? bg_adj : 0};  // (-1: bg_all)
    const bool plan_hit = e.bg_cache && s.plan_valid && s.plan_dB == pa.dB &&
                          s.plan_dT == pa.dT && s.plan_tfar == pa.tfar && s.plan_dfar == pa.dFar &&
                          std::equal(key, key + 7, s.plan_key);
    // Small sets in graph mode: plan and prep as one grid, so the pair kernel's
    // programmatic edge from it holds (a second predecessor on another stream
    // makes it a full edge) -- development knob STHK_PLAN_PREP=0 disables
    static const bool plan_prep_knob = [] {
      const char* v = std::getenv("STHK_PLAN_PREP");
      return !v || *v != '0';
    }();
    // (the symmetric kernel waits for its programmatic predecessor; the row
    // kernel does not, so it keeps the two-kernel structure)
    const bool plan_prep = plan_prep_knob && graph_mode && sym && !plan_hit && prep_unlaunched &&
                           !bg_split && e.n <= kPlanPrepMaxEvents;
    if (plan_prep) {
      ck(sthk::launch_plan_prep(pa, pr, st), "plan + prep");
      e.launches += 1;
      ck(op_record(e, s.prepped, st), "event");
      prep_unlaunched = false;
    }
    if (!plan_hit) {  // (the work counters are re-armed by the last pair CTAs)
      if (!plan_prep) {
        ck(sthk::launch_plan(pa, st), "plan");
        e.launches += 1;
      }
      s.plan_valid = e.bg_cache;
      s.plan_dB = pa.dB;
      s.plan_dT = pa.dT;
      s.plan_tfar = pa.tfar;
      s.plan_dfar = pa.dFar;
      std::copy(key, key + 7, s.plan_key);
    }
    launch_prep_now();
    const bool rows_forked = tr_rows && !cached;
    if (rows_forked) {  // beside the pair kernels, after prep (scaled coordinates)
      if (plan_prep) {
        ck(op_wait(e, s.stream2, s.prepped), "wait");
      } else if (!prep_pending) {
        ck(op_record(e, s.fork, st), "event");
        ck(op_wait(e, s.stream2, s.fork), "wait");
      }
      launch_trig_rows(s.stream2);
      ck(op_record(e, s.trow_ev, s.stream2), "event");
    }
    join_prep();  // pair kernels need the prepared coordinates / zeroed sums

    sthk::PairArgs qa{};
    qa.x = s.x;
    qa.y = s.y;
    qa.t = s.t;
    qa.xs = s.xs;
    qa.ys = s.ys;
    qa.tsl = s.tsl;
    qa.stl = pl.stl;
    qa.xf = s.xf;
    qa.yf = s.yf;
    qa.tf = s.tf;
    qa.tile_box = s.tile_box;
    qa.tile_trange = s.tile_trange;
    qa.n = e.n;
    qa.npad = e.npad;
    qa.k = pl.k;
    qa.sc = pl.sc;
    qa.ranges = s.ranges;
    qa.items = s.items;
    qa.n_items = s.scalars;
    qa.work_counter = s.scalars + 1;
    qa.done_counter = reinterpret_cast<unsigned int*>(s.scalars + 2);
    qa.fx = s.fx;
    qa.tpart = s.tpart;
    qa.bg_off = cached ? 1 : 0;
    qa.tr_off = tr_rows ? 1 : 0;
    qa.bg_diag_only = bg_split ? 1 : 0;
    for (int k = 0; k < sthk::kNSumGrad; ++k) qa.fxq[k] = fxq[k];
    if (sym) qa.fxq[1] = fxq[1] / (pl.sx * pl.sx);  // S_Br accumulates sx^2 r^2
    qa.pair_counts = e.timing ? s.pair_counts : nullptr;
    qa.tstamp = stamps ? s.tstamp : nullptr;
    if (s.trace) {
      qa.trace = s.trace;
      qa.trace_cap = item_trace_cap();
      qa.trace_kernel = 1;
    }
    // a trigger-only sweep runs the same kernel with the background switched
    // off, so its trigger partials are summed exactly as in a full sweep
    // merged: the general kernel takes the background-only list's items first
    // (one launch; the general items fill the tail), else a separate launch
    // of the trigger-free kernel
    if (bg_split && e.merge_bg) {
      qa.pre_ranges = s.ranges_bg;
      qa.pre_items = s.items_bg;
      qa.pre_n_items = s.scalars + 9;
      qa.pre_sc = pl.sc_bg;
    }
    auto launch_bg = [&] {  // the trigger-free kernel over the background-only list
      if (!bg_split || e.merge_bg) return;
      sthk::PairArgs ba = qa;
      ba.ranges = s.ranges_bg;
      ba.sc = pl.sc_bg;
      ba.items = s.items_bg;
      ba.n_items = s.scalars + 9;
      ba.work_counter = s.scalars + 10;
      ba.done_counter = reinterpret_cast<unsigned int*>(s.scalars + 11);
      ba.bg_diag_only = 0;
      ba.trace_kernel = 2;
      ck(sthk::launch_bgonly(ba, grad, s.sms * s.occ_bg[grad ? 1 : 0], st), "bg-only kernel");
      e.launches += 1;
      // (graph mode, every near stage here: a programmatic edge from the plan,
      // so its CTAs are resident when the lists are ready)
      if (bg_all) mark_last_kernel(e, 1);
    };
    const int occ = s.occ[e.mode][grad ? 1 : 0];
    const bool conc = far_on && e.far_concurrent;
    const int grid = s.sms * (conc ? std::min(e.near_ctas, occ) : occ);
    auto launch_general = [&] {  // (bg_all: its list is empty, not launched)
      if (bg_all) return;
      ck(sthk::launch_pairs(qa, grad, e.mode, grid, st), "pair kernel");
      e.launches += 1;
      if (plan_prep) mark_last_kernel(e, 1);  // (programmatic edge from plan + prep)
    };
    // ev[1] (pair-phase start) is recorded whether or not timing is on: a
    // timing event here, between the prep join and the far fork, measurably
    // lets the near kernel's CTAs reach the SMs ahead of the far kernel's
    // (C2, Θ_post: 0.472 -> 0.444 ms with timing off; no effect at Θ_init)
    // (an event-record node in graph mode too, where it has the same effect
    // with a trigger-free list; without one -- small N -- the node only adds
    // latency: measured 5 us at N = 10k)
    // (graph mode: without this node the far kernel's CTAs reach the SMs
    // first and the near kernel starts 20 us later -- measured 4.5% slower at
    // C2; graph node priorities do not change that order, and a
    // launch-completion edge from the trigger-free kernel to the far kernel
    // defers the far kernel behind the general one: 1.5% slower)
    // (with every near stage in the trigger-free kernel the node only adds
    // latency: measured C2 0.313 -> 0.308 ms, 50k 0.138 -> 0.134 ms without it)
    ck((e.timing && e.timing_pairs && !stamps) || (bg_split && !bg_all)
           ? record_timing(e, s.ev[1], st)
           : op_record(e, s.ev[1], st),
       "event");
    if (far_on) {  // the far work list in FP32
      sthk::PairArgs fa_ = qa;
      fa_.pre_items = nullptr;
      fa_.sc = pl.sc_far;
      fa_.ranges = s.ranges_far;
      fa_.items = s.items_far;
      fa_.n_items = s.scalars + 6;
      fa_.work_counter = s.scalars + 7;
      fa_.done_counter = reinterpret_cast<unsigned int*>(s.scalars + 8);
      fa_.tpart = far_tr ? s.tpart_far : nullptr;
      fa_.bg_diag_only = 0;
      fa_.trace_kernel = 3;
      // far list in FP64 (sthk_set_far_tier(2)): the general near kernel over
      // the same list with the far tier's windows -- the precision policy's
      // cost measured with identical culling
      auto launch_far_list = [&](int grid_far, cudaStream_t fs) {
        if (e.far_fp64) {
          sthk::PairArgs f64 = fa_;
          f64.k.dB = pl.k.dBf;
          f64.k.dT = pl.k.dTf;
          f64.tpart = s.tpart_far;  // (read by finalize only when far_tr)
          return sthk::launch_pairs(f64, grad, e.mode, s.sms * s.occ[e.mode][grad ? 1 : 0], fs);
        }
        return sthk::launch_far(fa_, grad, grid_far, fs);
      };
      if (conc) {  // forked onto the second stream, joined before finalize
        ck(op_record(e, s.fork, st), "event");
        ck(op_wait(e, s.stream2, s.fork), "wait");
        if (e.far_order == 2) {  // near first: its CTAs are resident before far CTAs fill in
          launch_bg();
          launch_general();
          ck(launch_far_list(s.sms * e.far_ctas, s.stream2), "far kernel");
          e.launches += 1;
        } else {
          launch_bg();
          ck(launch_far_list(s.sms * e.far_ctas, s.stream2), "far kernel");
          e.launches += 1;
          launch_general();
        }
        ck(op_record(e, s.join, s.stream2), "event");
        ck(op_wait(e, st, s.join), "wait");
      } else {
        launch_bg();
        launch_general();
        ck(launch_far_list(s.sms * s.occ_far[grad ? 1 : 0], st), "far kernel");
        e.launches += 1;
      }
    } else {
      launch_bg();
      launch_general();
    }
    if (rows_forked) ck(op_wait(e, st, s.trow_ev), "wait");
    if (e.timing && e.timing_pairs && !stamps) ck(record_timing(e, s.ev[2], st), "event");
    ck(op_record(e, s.pairs_done, st), "event");
  }

  // phase 2: symmetric sweeps add column sums to earlier rows, some owned by
  // other shards: each shard ships those rows to their owner
  if (sym && !cached && shards > 1) exchange_fx(e, fx_transfers(e, pl, far_on, shards));

  // phase 3: per-row finalize into 256-row block partials
  for (Slot& s : e.slots) {
    set_dev(s);
    if (s.row1 > s.row0) {
      sthk::FinArgs fa{};
      fa.t = s.t;
      fa.n = e.n;
      fa.npad = e.npad;
      fa.row0 = s.row0;
      fa.row1 = s.row1;
      fa.window_end = e.window_end;
      fa.mu0 = p[0];
      fa.tauX = p[1];
      fa.tauT = p[2];
      fa.theta = p[3];
      fa.omega = p[4];
      fa.h = p[5];
      // HawkesPairTerm constants, kernels.hpp:78-84
      fa.bgNorm = std::pow(2.0 * kPi, -1.5) / (p[1] * p[1] * p[2]);
      fa.trNorm = p[3] * p[4] / (2.0 * kPi * p[5] * p[5]);
      fa.cT = p[4] / (2.0 * kPi * p[5] * p[5]);
      {  // gradient constants (FinArgs::gB, gT), folded in long double
        const long double mb = static_cast<long double>(p[0]) * fa.bgNorm;
        const long double tx = p[1], tt = p[2], om = p[4], h = p[5], tn = fa.trNorm;
        fa.gB[0] = static_cast<double>(-2.0L * mb / tx);
        fa.gB[1] = static_cast<double>(mb / (tx * tx * tx) / fxq[1]);
        fa.gB[2] = static_cast<double>(-mb / tt);
        fa.gB[3] = static_cast<double>(mb / (tt * tt * tt) / fxq[2]);
        fa.gT[0] = static_cast<double>(tn / om);
        fa.gT[1] = static_cast<double>(-tn);
        fa.gT[2] = static_cast<double>(-2.0L * tn / h);
        fa.gT[3] = static_cast<double>(tn / (h * h * h) * (sym ? 1.0L / (static_cast<long double>(pl.sx) * pl.sx) : 1.0L));
      }
      fa.fx = s.fx;
      fa.tpart = s.tpart;
      fa.tr_r2_scale = sym ? 1.0 / (pl.sx * pl.sx) : 1.0;
      fa.crange = s.crange;
      fa.comp = s.comp;
      fa.tpart_far = far_tr ? s.tpart_far : nullptr;
      fa.trow = tr_rows ? s.trow : nullptr;
      if (fin_rows) {
        fa.rows.xs = s.xs;
        fa.rows.ys = s.ys;
        fa.rows.t = s.t;
        fa.rows.npad = e.npad;
        fa.rows.row0 = s.row0;
        fa.rows.row1 = s.row1;
        fa.rows.nomL = pl.k.nomL;
        fa.rows.chS = pl.k.chS;
        fa.rows.dT = dT_rows;
        fa.rows.trow = s.trow;
        fa.rows.pair_counts = e.timing ? s.pair_counts : nullptr;
        fa.comp_inline = need_comp ? 1 : 0;
      }
      fa.crange_far = s.crange_far;
      for (int k = 0; k < sthk::kNSumGrad; ++k) fa.fxq[k] = fxq[k];
      fa.per_event = want_pe ? s.per_event : nullptr;
      fa.ex_out = want_ex ? s.ex : nullptr;
      fa.block_partial = s.block_partial;
      // one shard and no collective: the final sum rides along
      fa.fused_out = (shards == 1) ? s.d_hout : nullptr;
      fa.counts = (shards == 1 && e.timing) ? s.pair_counts : nullptr;
      fa.counts_out = s.d_hcounts;
      fa.nblocks_total = nb_total;
      fa.done_counter = reinterpret_cast<unsigned int*>(s.scalars + 3);
      fa.trace = s.trace;
      fa.trace_cap = item_trace_cap();
      fa.tstamp = stamps ? s.tstamp : nullptr;
      fa.tstamp_out = s.d_htstamp;
      ck(sthk::launch_finalize(fa, grad, s.stream), "finalize");
      mark_last_kernel(e, 1);  // (graph mode: launched while the last pair kernel drains)
      e.launches += 1;
    }
    ck(op_record(e, s.fin_done, s.stream), "event");
  }

  // phase 4: exact combination of the block partials, fixed-order final sum
  if (shards > 1) combine_blocks(e, nb_total);

  for (Slot& s : e.slots) {
    set_dev(s);
    cudaStream_t st = s.stream;
    if (!e.timing) std::fill(s.h_counts, s.h_counts + sthk::kNCounts, 0ULL);
    if (want_pe && s.row1 > s.row0) {
      ck(op_memcpy(e, s.h_per_event + s.row0, s.per_event + s.row0,
                         sizeof(double) * (s.row1 - s.row0), cudaMemcpyDeviceToHost, st),
         "D2H");
    }
    if (want_ex && ex_to_host && s.row1 > s.row0) {
      for (int k = 0; k < 3; ++k) {
        ck(op_memcpy(e, s.h_ex + k * e.npad + s.row0, s.ex + k * e.npad + s.row0,
                           sizeof(double) * (s.row1 - s.row0), cudaMemcpyDeviceToHost, st),
           "D2H");
      }
    }
    if (e.timing && !stamps) ck(record_timing(e, s.ev[3], st), "event");
    if (e.recording) launch_recorded(e, st);
  }
  e.pending = true;
  e.last_grad = grad;
  e.last_pe = want_pe;
  e.last_ex = want_ex;
  if (!cached) {
    e.cache_grad = grad;
    e.cache_gen = e.load_gen;
    e.cache_tx = e.p[1];
    e.cache_tt = e.p[2];
    e.cache_mode = e.mode;
    e.cache_dense = e.dense;
    e.cache_far_full = far_full;
    e.cache_far_fp64 = e.far_fp64;
    e.cache_tfar = far_full ? pl.tfar : 0.0;
    e.cache_bg_adj = bg_adj;
    e.cache_cuts = pl.cuts;
  }
  e.cache_valid = true;
  if (!tr_cached) {
    e.tr_cache_grad = grad;
    e.tr_cache_omega = e.p[4];
    e.tr_cache_h = e.p[5];
    e.tr_cache_dT = pl.k.dT;
    e.tr_cache_dTf = pl.k.dTf;
    e.tr_cache_far_tr = far_tr;
    e.tr_cache_rows = tr_rows;
  }
  e.tr_cache_valid = e.bg_cache;
  e.comp_valid = e.bg_cache;
  e.comp_gen = e.load_gen;
  e.comp_tt = p[2];
  e.comp_om = p[4];
}

void collect(sthk_engine& e, double* loglik, int* valid, double* grad6, double* per_event) {
  if (!e.pending) throw NotLoaded("sthk: no evaluation enqueued");
  for (Slot& s : e.slots) {
    set_dev(s);
    ck(cudaStreamSynchronize(s.stream), "evaluation");
  }
  e.pending = false;
  const double* o = e.slots[0].h_out;
  const bool ok = o[7] == 0.0 && std::isfinite(o[0]);
  if (valid) *valid = ok ? 1 : 0;
  if (loglik) *loglik = ok ? o[0] : -std::numeric_limits<double>::infinity();
  if (grad6) {
    for (int k = 0; k < 6; ++k) {
      grad6[k] = (ok && e.last_grad) ? o[1 + k] : std::numeric_limits<double>::quiet_NaN();
    }
  }
  if (per_event && e.last_pe) {
    for (Slot& s : e.slots) {
      if (s.row1 > s.row0) {
        std::memcpy(per_event + s.row0, s.h_per_event + s.row0,
                    sizeof(double) * (s.row1 - s.row0));
      }
    }
  }
}

int fail(sthk_engine* e, int code, const char* msg) {
  if (e) e->err = msg;
  return code;
}

template <typename F>
int guarded(sthk_engine* e, F&& f) {
  if (!e) return STHK_EINVAL;
  try {
    f();
    e->err.clear();
    return STHK_OK;
  } catch (const InvalidArg& x) {
    return fail(e, STHK_EINVAL, x.what());
  } catch (const NotLoaded& x) {
    return fail(e, STHK_ENOTLOADED, x.what());
  } catch (const NcclErr& x) {
    return fail(e, STHK_ENCCL, x.what());
  } catch (const CommErr& x) {
    return fail(e, STHK_ENCCL, x.what());
  } catch (const CudaErr& x) {
    return fail(e, STHK_ECUDA, x.what());
  } catch (const std::exception& x) {
    return fail(e, STHK_ECUDA, x.what());
  }
}

thread_local std::string g_create_err;

}  // namespace

extern "C" {

int sthk_debug_exp(int device, const double* x, int64_t n, double* out) {
  if (!x || !out || n < 0) return STHK_EINVAL;
  if (n == 0) return STHK_OK;
  if (cudaSetDevice(device) != cudaSuccess) return STHK_ECUDA;
  double *dx = nullptr, *dy = nullptr;
  const size_t bytes = sizeof(double) * static_cast<size_t>(n);
  int rc = STHK_OK;
  if (cudaMalloc(&dx, bytes) != cudaSuccess || cudaMalloc(&dy, bytes) != cudaSuccess ||
      cudaMemcpy(dx, x, bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
      sthk::launch_exp_probe(dx, n, dy, nullptr) != cudaSuccess ||
      cudaMemcpy(out, dy, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) {
    rc = STHK_ECUDA;
  }
  if (dx) cudaFree(dx);
  if (dy) cudaFree(dy);
  return rc;
}

const char* sthk_version(void) { return "sthk 0.2 (sm_100a, fp64)"; }

const char* sthk_last_error(const sthk_engine* e) {
  return e ? e->err.c_str() : g_create_err.c_str();
}

int sthk_create(const int* device_ids, int n_devices, sthk_engine** out) {
  if (!out || n_devices < 1 || !device_ids) {
    g_create_err = "sthk_create: need n_devices >= 1";
    return STHK_EINVAL;
  }
  *out = nullptr;
  auto e = std::make_unique<sthk_engine>();
  try {
    int count = 0;
    ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    for (int i = 0; i < n_devices; ++i) {
      if (device_ids[i] < 0 || device_ids[i] >= count) {
        g_create_err = "sthk_create: device id out of range";
        return STHK_EINVAL;
      }
    }
    e->slots.resize(n_devices);
    for (int i = 0; i < n_devices; ++i) {
      init_slot(e->slots[i], device_ids[i]);
      e->slots[i].shard = i;
    }
    // a repeated device id: shards sharing a GPU, combined by device copies
    // (NCCL needs one rank per device)
    std::vector<int> ids(device_ids, device_ids + n_devices);
    std::sort(ids.begin(), ids.end());
    const bool dup = std::adjacent_find(ids.begin(), ids.end()) != ids.end();
    e->xport = n_devices == 1 ? Xport::kSingle : dup ? Xport::kLocal : Xport::kNccl;
    if (e->xport == Xport::kNccl) {
      std::vector<ncclComm_t> comms(n_devices);
      ckn(ncclCommInitAll(comms.data(), n_devices, device_ids), "ncclCommInitAll");
      for (int i = 0; i < n_devices; ++i) e->slots[i].comm = comms[i];
    }
  } catch (const NcclErr& x) {
    g_create_err = x.what();
    for (auto& s : e->slots) free_slot(s);
    return STHK_ENCCL;
  } catch (const std::exception& x) {
    g_create_err = x.what();
    for (auto& s : e->slots) free_slot(s);
    return STHK_ECUDA;
  }
  *out = e.release();
  return STHK_OK;
}

int sthk_nccl_unique_id(void* nccl_id) {
  if (!nccl_id) return STHK_EINVAL;
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    g_create_err = ncclGetErrorString(r);
    return STHK_ENCCL;
  }
  static_assert(sizeof(ncclUniqueId) == STHK_NCCL_ID_BYTES, "nccl id size");
  std::memcpy(nccl_id, &id, sizeof(id));
  return STHK_OK;
}

int sthk_create_rank(int device, int rank, int world, const void* nccl_id,
                     sthk_engine** out) {
  if (!out || world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_id)) {
    g_create_err = "sthk_create_rank: invalid rank/world";
    return STHK_EINVAL;
  }
  *out = nullptr;
  auto e = std::make_unique<sthk_engine>();
  e->rank_mode = true;
  e->rank = rank;
  e->world = world;
  e->xport = world > 1 ? Xport::kNccl : Xport::kSingle;
  try {
    e->slots.resize(1);
    init_slot(e->slots[0], device);
    e->slots[0].shard = rank;
    if (world > 1) {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      ckn(ncclCommInitRank(&e->slots[0].comm, world, id, rank), "ncclCommInitRank");
    }
  } catch (const NcclErr& x) {
    g_create_err = x.what();
    for (auto& s : e->slots) free_slot(s);
    return STHK_ENCCL;
  } catch (const std::exception& x) {
    g_create_err = x.what();
    for (auto& s : e->slots) free_slot(s);
    return STHK_ECUDA;
  }
  *out = e.release();
  return STHK_OK;
}

int sthk_create_rank_hosted(int device, int rank, int world, const sthk_host_comm* comm,
                            sthk_engine** out) {
  if (!out || world < 1 || rank < 0 || rank >= world || !comm || !comm->allreduce_sum ||
      !comm->exchange) {
    g_create_err = "sthk_create_rank_hosted: invalid rank/world/callbacks";
    return STHK_EINVAL;
  }
  *out = nullptr;
  auto e = std::make_unique<sthk_engine>();
  e->rank_mode = true;
  e->rank = rank;
  e->world = world;
  e->xport = world > 1 ? Xport::kHosted : Xport::kSingle;
  e->hcomm = *comm;
  try {
    e->slots.resize(1);
    init_slot(e->slots[0], device);
    e->slots[0].shard = rank;
  } catch (const std::exception& x) {
    g_create_err = x.what();
    for (auto& s : e->slots) free_slot(s);
    return STHK_ECUDA;
  }
  *out = e.release();
  return STHK_OK;
}

int sthk_destroy(sthk_engine* e) {
  if (!e) return STHK_EINVAL;
  if (!e->graphs.empty()) {
    cudaSetDevice(e->slots[0].dev);
    cudaStreamSynchronize(e->slots[0].stream);
    for (auto& g : e->graphs) {
      cudaGraphExecDestroy(g.exec);
      cudaGraphDestroy(g.graph);
    }
  }
  for (auto& s : e->slots) free_slot(s);
  delete e;
  return STHK_OK;
}

int sthk_load_events(sthk_engine* e, const double* x, const double* y, const double* t,
                     int64_t n, double window_end) {
  return guarded(e, [&] {
    validate_event_args(x, y, t, n);
    if (e->pending) collect(*e, nullptr, nullptr, nullptr, nullptr);
    e->loaded = false;  // until the device-side checks pass
    const int64_t npad = (n + kTM - 1) / kTM * kTM;
    // (development knob STHK_PLAN_STRIDED=1: strided pivots at any N, to
    // check that tile-granular plan searches change no result)
    static const bool force_strided = [] {
      const char* v = std::getenv("STHK_PLAN_STRIDED");
      return v && *v == '1';
    }();
    e->tile_pivots = sthk::use_tile_pivots(n) && !force_strided;
    const bool multi = e->slots.size() > 1 || e->rank_mode;
    if (multi) e->ht.assign(t, t + n);
    e->ht_valid = multi;
    // Straight from the caller's buffers (pinned or pageable) to every
    // device; the pad tail is zero and is never read as a source (stage
    // loops are bounded by n) nor reported as a target.
    const size_t bytes = sizeof(double) * static_cast<size_t>(n);
    for (Slot& s : e->slots) {
      set_dev(s);
      dev_grow(s.x, s.x_cap, static_cast<size_t>(npad));
      dev_grow(s.y, s.y_cap, static_cast<size_t>(npad));
      dev_grow(s.t, s.t_cap, static_cast<size_t>(npad));
      dev_grow(s.xs, s.xs_cap, static_cast<size_t>(npad));
      dev_grow(s.ys, s.ys_cap, static_cast<size_t>(npad));
      dev_grow(s.xf, s.xf_cap, static_cast<size_t>(npad));
      dev_grow(s.yf, s.yf_cap, static_cast<size_t>(npad));
      dev_grow(s.tf, s.tf_cap, static_cast<size_t>(npad));
      // Pinned (device-mapped) caller arrays on one device: the load kernel
      // reads them over PCIe itself -- one pass instead of three copies and a
      // kernel (measured 69 -> 57 us at C2). Otherwise, or while another
      // engine's evaluation occupies the device, copy first.
      const double* srcx = s.x;
      const double* srcy = s.y;
      const double* srct = s.t;
      const double* mapped[3] = {nullptr, nullptr, nullptr};
      if (e->slots.size() == 1 && !device_busy_elsewhere(s.dev, s.stream)) {
        const double* hp[3] = {x, y, t};
        for (int k = 0; k < 3; ++k) {
          cudaPointerAttributes at{};
          if (cudaPointerGetAttributes(&at, hp[k]) == cudaSuccess && at.type == cudaMemoryTypeHost &&
              at.devicePointer) {
            mapped[k] = static_cast<const double*>(at.devicePointer);
          }
        }
        (void)cudaGetLastError();
      }
      e->load_zero_copy = mapped[0] && mapped[1] && mapped[2];
      if (e->load_zero_copy) {
        srcx = mapped[0];
        srcy = mapped[1];
        srct = mapped[2];
      } else {
        ck(cudaMemcpyAsync(s.x, x, bytes, cudaMemcpyHostToDevice, s.stream), "H2D");
        ck(cudaMemcpyAsync(s.y, y, bytes, cudaMemcpyHostToDevice, s.stream), "H2D");
        ck(cudaMemcpyAsync(s.t, t, bytes, cudaMemcpyHostToDevice, s.stream), "H2D");
      }
      dev_grow(s.tile_box, s.box_cap, static_cast<size_t>(npad / kTS));
      dev_grow(s.tile_trange, s.trange_cap, static_cast<size_t>(npad / kTS));
      auto* bad = reinterpret_cast<unsigned long long*>(s.scalars + 4);
      auto* done = reinterpret_cast<unsigned int*>(s.scalars + 12);
      unsigned long long* d_hbad = nullptr;
      ck(cudaHostGetDevicePointer(&d_hbad, s.h_bad, 0), "cudaHostGetDevicePointer");
      double* d_hstats = nullptr;
      ck(cudaHostGetDevicePointer(&d_hstats, s.h_stats, 0), "cudaHostGetDevicePointer");
      if (!s.piv) ck(cudaMalloc(&s.piv, sizeof(double) * sthk::kPlanPivots), "cudaMalloc");
      ck(sthk::launch_tile_boxes(srcx, srcy, srct, s.x, s.y, s.t, n, npad, s.tile_box, s.tile_trange, s.piv, bad,
                                 done, d_hbad, d_hstats, s.load_dstats, e->tile_pivots, s.stream),
         "tile boxes + checks");
    }
    for (Slot& s : e->slots) {
      set_dev(s);
      ck(cudaStreamSynchronize(s.stream), "H2D");
    }
    const unsigned long long first_bad = *e->slots[0].h_bad;
    if (first_bad != ~0ULL) throw_event_error(x, y, t, static_cast<int64_t>(first_bad));
    validate_window_end(t, n, window_end);
    {  // load statistics from the check kernel (coordinate extents for the far-tier
       // guard, tile time span, stage gaps for the trigger-free split)
      const double* st = e->slots[0].h_stats;
      e->ext_x = st[0];
      e->ext_y = st[1];
      e->tile_tspan = st[2];
      e->adj_gap.assign(st + 3, st + 3 + kMaxAdj);
      e->span_min.assign(st + 3 + kMaxAdj, st + 3 + kMaxAdj + sthk::kLoadSpan);
    }
    e->n = n;
    e->npad = npad;
    e->window_end = window_end;
    e->loaded = true;
    e->load_gen += 1;
    e->cache_valid = false;
    e->tr_cache_valid = false;
    e->comp_valid = false;
    for (Slot& s : e->slots) s.plan_valid = false;
  });
}

int sthk_set_params(sthk_engine* e, const double* params6) {
  return guarded(e, [&] {
    if (!params6) throw InvalidArg("sthk_set_params: null params");
    validate_params(params6);
    std::memcpy(e->p, params6, sizeof(e->p));
    e->has_params = true;
  });
}

int sthk_enqueue(sthk_engine* e, int want_grad, int want_per_event) {
  return guarded(e, [&] {
    if (e->pending) throw InvalidArg("sthk_enqueue: previous result not collected");
    enqueue_eval(*e, want_grad != 0, want_per_event != 0);
  });
}

int sthk_result(sthk_engine* e, double* loglik, int* valid, double* grad6, double* per_event) {
  return guarded(e, [&] { collect(*e, loglik, valid, grad6, per_event); });
}

int sthk_loglik(sthk_engine* e, double* loglik, int* valid, double* per_event) {
  return guarded(e, [&] {
    if (e->pending) collect(*e, nullptr, nullptr, nullptr, nullptr);
    enqueue_eval(*e, false, per_event != nullptr);
    collect(*e, loglik, valid, nullptr, per_event);
  });
}

int sthk_loglik_grad(sthk_engine* e, double* loglik, int* valid, double* grad6,
                     double* per_event) {
  return guarded(e, [&] {
    if (e->pending) collect(*e, nullptr, nullptr, nullptr, nullptr);
    enqueue_eval(*e, true, per_event != nullptr);
    collect(*e, loglik, valid, grad6, per_event);
  });
}

int sthk_excitation(sthk_engine* e, double* mu, double* xi, double* pi) {
  int degenerate = 0;
  const int rc = guarded(e, [&] {
    if (e->pending) collect(*e, nullptr, nullptr, nullptr, nullptr);
    enqueue_eval(*e, false, false, true);
    collect(*e, nullptr, nullptr, nullptr, nullptr);
    double* outs[3] = {mu, xi, pi};
    for (Slot& s : e->slots) {
      if (s.row1 <= s.row0) continue;
      for (int k = 0; k < 3; ++k) {
        if (outs[k]) {
          std::memcpy(outs[k] + s.row0, s.h_ex + k * e->npad + s.row0,
                      sizeof(double) * (s.row1 - s.row0));
        }
      }
    }
    degenerate = e->slots[0].h_out[7] > 0.0;
  });
  if (rc == STHK_OK && degenerate) {
    return fail(e, STHK_ERANGE, "excitationProbabilities: per-event rate underflowed to zero");
  }
  return rc;
}

int sthk_excitation_batch(sthk_engine* e, const double* params, int64_t S, double* sum_pi,
                          double* per_draw, int64_t* bad_draw) {
  int64_t bad = -1;
  const int rc = guarded(e, [&] {
    if (S < 1 || !params || !sum_pi) throw InvalidArg("sthk_excitation_batch: no draws");
    for (int64_t j = 0; j < S; ++j) {
      try {
        validate_params(params + 6 * j);
      } catch (const InvalidArg& x) {
        throw InvalidArg("sthk_excitation_batch: draw " + std::to_string(j) + ": " + x.what());
      }
    }
    if (!e->loaded) throw NotLoaded("sthk: no events loaded");
    if (e->pending) collect(*e, nullptr, nullptr, nullptr, nullptr);
    double saved[6];
    std::memcpy(saved, e->p, sizeof(saved));
    const bool had = e->has_params;
    constexpr int64_t kPiChunk = 32;  // per-draw rows staged per host copy
    const int64_t n = e->n, npad = e->npad;
    for (Slot& s : e->slots) {
      set_dev(s);
      dev_grow(s.pi_sum, s.pi_sum_cap, static_cast<size_t>(npad));
      dev_grow(s.pi_bad, s.pi_bad_cap, static_cast<size_t>(S));
      // (in/out: the draws' pi are added to the caller's sums)
      ck(cudaMemcpyAsync(s.pi_sum, sum_pi, sizeof(double) * n, cudaMemcpyHostToDevice, s.stream),
         "H2D pi sums");
      ck(cudaMemsetAsync(s.pi_bad, 0, sizeof(int) * S, s.stream), "memset");
      if (per_draw) {
        dev_grow(s.pi_rows, s.pi_rows_cap, static_cast<size_t>(kPiChunk * npad));
        if (s.h_pi_rows_cap < static_cast<size_t>(kPiChunk * npad)) {
          if (s.h_pi_rows) ck(cudaFreeHost(s.h_pi_rows), "cudaFreeHost");
          ck(cudaMallocHost(&s.h_pi_rows, sizeof(double) * kPiChunk * npad), "cudaMallocHost");
          s.h_pi_rows_cap = static_cast<size_t>(kPiChunk * npad);
        }
      }
    }
    // Draws in order, each an excitation evaluation on the device (with the
    // sweep caches on, draws that share tauX, tauT -- every draw of the
    // reference MH sampler -- reuse one background sweep, and consecutive
    // draws with equal omega, h one trigger sweep); pi is accumulated on the
    // device in draw order, so the sum equals the reference's meanPi +=
    // ex.pi loop bitwise (excitation.cpp:110-112).
    auto flush_rows = [&](int64_t j0, int64_t j1) {  // draws [j0, j1) staged in pi_rows
      for (Slot& s : e->slots) {
        set_dev(s);
        ck(cudaStreamSynchronize(s.stream), "excitation batch");
        if (s.row1 <= s.row0) continue;
        for (int64_t j = j0; j < j1; ++j) {
          std::memcpy(per_draw + j * n + s.row0, s.h_pi_rows + (j - j0) * npad + s.row0,
                      sizeof(double) * (s.row1 - s.row0));
        }
      }
    };
    int64_t chunk0 = 0;
    for (int64_t j = 0; j < S; ++j) {
      std::memcpy(e->p, params + 6 * j, sizeof(e->p));
      e->has_params = true;
      enqueue_eval(*e, false, false, true, false);
      for (Slot& s : e->slots) {
        set_dev(s);
        ck(sthk::launch_pi_accumulate(s.ex, npad, s.row0, s.row1, s.pi_sum, s.pi_bad + j,
                                      s.stream),
           "pi accumulate");
        e->launches += 1;
        if (per_draw && s.row1 > s.row0) {
          const size_t off = static_cast<size_t>(j - chunk0) * npad + s.row0;
          const size_t bytes = sizeof(double) * (s.row1 - s.row0);
          ck(cudaMemcpyAsync(s.h_pi_rows + off, s.ex + 2 * npad + s.row0, bytes,
                             cudaMemcpyDeviceToHost, s.stream),
             "D2H pi");
        }
      }
      if (per_draw && (j + 1 - chunk0 == kPiChunk || j + 1 == S)) {
        flush_rows(chunk0, j + 1);
        chunk0 = j + 1;
      }
    }
    std::vector<int> flags(static_cast<size_t>(S), 0);
    for (Slot& s : e->slots) {
      set_dev(s);
      ck(cudaStreamSynchronize(s.stream), "excitation batch");
      std::vector<int> f(static_cast<size_t>(S));
      ck(cudaMemcpy(f.data(), s.pi_bad, sizeof(int) * S, cudaMemcpyDeviceToHost), "D2H");
      for (int64_t j = 0; j < S; ++j) flags[j] |= f[j];
      if (s.row1 > s.row0) {
        ck(cudaMemcpy(sum_pi + s.row0, s.pi_sum + s.row0, sizeof(double) * (s.row1 - s.row0),
                      cudaMemcpyDeviceToHost),
           "D2H");
      }
    }
    e->pending = false;
    for (int64_t j = 0; j < S && bad < 0; ++j) {
      if (flags[j]) bad = j;
    }
    std::memcpy(e->p, saved, sizeof(saved));
    e->has_params = had;
  });
  if (bad_draw) *bad_draw = bad;
  if (rc == STHK_OK && bad >= 0) {
    return fail(e, STHK_ERANGE, "excitationProbabilities: per-event rate underflowed to zero");
  }
  return rc;
}

int sthk_loglik_batch(sthk_engine* e, const double* params, int64_t P, double* loglik,
                      int* valid, double* grad) {
  return guarded(e, [&] {
    if (P < 1 || !params) throw InvalidArg("logLikelihoodBatch: empty parameter list");
    for (int64_t i = 0; i < P; ++i) {
      try {
        validate_params(params + 6 * i);
      } catch (const InvalidArg& x) {
        throw InvalidArg("logLikelihoodBatch: entry " + std::to_string(i) + ": " + x.what());
      }
    }
    if (e->pending) collect(*e, nullptr, nullptr, nullptr, nullptr);
    double saved[6];
    std::memcpy(saved, e->p, sizeof(saved));
    const bool had = e->has_params;
    // Evaluation order grouped by (tauX, tauT, omega, h): consecutive entries
    // then reuse the cached background sums (same tauX, tauT) and trigger
    // sums (same omega, h too), so a batch that varies mu0 / theta costs one
    // sweep plus a finalize per entry. The caches are exact, so every result
    // is bitwise the single-call result whatever the order.
    std::vector<int64_t> order(static_cast<size_t>(P));
    for (int64_t i = 0; i < P; ++i) order[static_cast<size_t>(i)] = i;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
      const double* pa = params + 6 * a;
      const double* pb = params + 6 * b;
      for (int k : {1, 2, 4, 5}) {
        if (pa[k] != pb[k]) return pa[k] < pb[k];
      }
      return false;
    });
    for (const int64_t i : order) {
      std::memcpy(e->p, params + 6 * i, sizeof(e->p));
      e->has_params = true;
      enqueue_eval(*e, grad != nullptr, false);
      collect(*e, loglik + i, valid + i, grad ? grad + 6 * i : nullptr, nullptr);
    }
    std::memcpy(e->p, saved, sizeof(saved));
    e->has_params = had;
  });
}

int sthk_set_timing(sthk_engine* e, int enable) {
  return guarded(e, [&] {
    if (enable < 0 || enable > 2) throw InvalidArg("sthk_set_timing: enable must be 0, 1 or 2");
    e->timing = enable != 0;
    e->timing_pairs = enable == 1;
  });
}

int sthk_set_graphs(sthk_engine* e, int enable) {
  return guarded(e, [&] { e->use_graph = enable != 0; });
}

int sthk_set_dense(sthk_engine* e, int dense) {
  return guarded(e, [&] { e->dense = dense != 0; });
}

int sthk_plan_partition(const double* t, int64_t n, const double* params6, int shards,
                        int dense, int* cuts, int* source_chunk) {
  if (!t || n < 1 || !params6 || shards < 1 || !cuts) return STHK_EINVAL;
  try {
    validate_params(params6);
    const std::vector<double> ht(t, t + n);
    const int64_t npad = (n + kTM - 1) / kTM * kTM;
    const EvalPlan pl = make_plan(PlanInput{ht, n, npad, params6, dense != 0, true, true}, shards);
    for (int k = 0; k <= shards; ++k) cuts[k] = pl.cuts[k];
    if (source_chunk) *source_chunk = pl.sc;
    return STHK_OK;
  } catch (const std::exception& x) {
    g_create_err = x.what();
    return STHK_EINVAL;
  }
}

int sthk_set_background_cache(sthk_engine* e, int enable) {
  return guarded(e, [&] {
    e->bg_cache = enable != 0;
    if (!e->bg_cache) {
      e->cache_valid = false;
      e->tr_cache_valid = false;
      for (Slot& s : e->slots) s.plan_valid = false;
    }
  });
}

int sthk_set_far_schedule(sthk_engine* e, int concurrent, int near_ctas, int far_ctas) {
  return guarded(e, [&] {
    if (near_ctas < 1 || far_ctas < 1) throw InvalidArg("sthk_set_far_schedule: CTA counts must be >= 1");
    e->far_concurrent = concurrent != 0;
    e->far_order = concurrent == 2 ? 2 : 1;
    e->near_ctas = near_ctas;
    e->far_ctas = far_ctas;
  });
}

int sthk_set_bgonly_kernel(sthk_engine* e, int enable) {
  return guarded(e, [&] {
    e->bg_split = enable != 0;
    for (Slot& s : e->slots) s.plan_valid = false;
  });
}

int sthk_set_far_tier(sthk_engine* e, int enable) {
  return guarded(e, [&] {
    if (enable < 0 || enable > 2) throw InvalidArg("sthk_set_far_tier: mode must be 0, 1 or 2");
    e->far_tier = enable != 0;
    e->far_fp64 = enable == 2;
  });
}

int sthk_set_kernel(sthk_engine* e, int mode) {
  return guarded(e, [&] {
    if (mode != sthk::kRows && mode != sthk::kSym) {
      throw InvalidArg("sthk_set_kernel: mode must be 0 (rows) or 1 (symmetric)");
    }
    e->mode = mode;
  });
}

int sthk_get_exchange_bytes(sthk_engine* e, int64_t* bytes) {
  return guarded(e, [&] {
    if (!bytes) throw InvalidArg("sthk_get_exchange_bytes: null");
    *bytes = e->exch_bytes;
  });
}

int sthk_debug_item_trace(sthk_engine* e, int slot, unsigned long long* out, int64_t cap,
                          int64_t* count) {
  return guarded(e, [&] {
    if (slot < 0 || slot >= static_cast<int>(e->slots.size()) || !count) {
      throw InvalidArg("sthk_debug_item_trace: bad slot or count pointer");
    }
    Slot& s = e->slots[slot];
    *count = 0;
    if (!s.trace) return;
    set_dev(s);
    ck(cudaStreamSynchronize(s.stream), "sync");
    ck(cudaStreamSynchronize(s.stream2), "sync");
    unsigned long long n = 0;
    ck(cudaMemcpy(&n, s.trace, sizeof(n), cudaMemcpyDeviceToHost), "D2H");
    n = std::min<unsigned long long>(n, static_cast<unsigned long long>(item_trace_cap()));
    *count = static_cast<int64_t>(n);
    const size_t k = std::min<size_t>(static_cast<size_t>(n), static_cast<size_t>(std::max<int64_t>(cap, 0)));
    if (out && k) {
      ck(cudaMemcpy(out, s.trace + 4, 4 * k * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "D2H");
    }
  });
}

int sthk_get_stream(sthk_engine* e, int slot, void** stream) {
  return guarded(e, [&] {
    if (slot < 0 || slot >= static_cast<int>(e->slots.size()) || !stream) {
      throw InvalidArg("sthk_get_stream: bad slot");
    }
    *stream = e->slots[slot].stream;
  });
}

int sthk_get_stats(sthk_engine* e, sthk_stats* out) {
  return guarded(e, [&] {
    if (!out) throw InvalidArg("sthk_get_stats: null");
    std::memset(out, 0, sizeof(*out));
    out->n = e->n;
    out->pairs_dense = e->n * e->n;
    out->n_devices = static_cast<int>(e->slots.size());
    out->rank = e->rank;
    out->world = e->world;
    out->source_chunk = e->last_sc;
    out->far_threshold = e->last_far_a;
    out->graph_launches = e->graph_updates;
    out->graph_builds = e->graph_instantiations;
    out->load_zero_copy = e->load_zero_copy ? 1 : 0;
    out->trigger_rows = e->last_trig_rows ? 1 : 0;
    out->far_split_days = e->last_tfar;
    out->kernel_mode = e->mode;
    out->cache_hit = e->last_cache_hit ? 1 : 0;
    out->trigger_cache_hit = e->last_tr_cache_hit ? 1 : 0;
    out->kernel_launches = e->launches;
    for (Slot& s : e->slots) {
      out->pairs_bg += static_cast<int64_t>(s.h_counts[0]);
      out->pairs_tr += static_cast<int64_t>(s.h_counts[1]);
      out->pairs_any += static_cast<int64_t>(s.h_counts[2]);
      out->exec_bg += static_cast<int64_t>(s.h_counts[3]);
      out->exec_geom += static_cast<int64_t>(s.h_counts[4]);
      out->exec_sym += static_cast<int64_t>(s.h_counts[5]);
      out->exec_far += static_cast<int64_t>(s.h_counts[6]);
      if (e->timing && s.row1 > s.row0 && s.last_stamps) {
        const unsigned long long* h = s.h_tstamp;
        if (h[1] > h[0]) out->eval_ms = std::max(out->eval_ms, (h[1] - h[0]) * 1e-6);
        if (e->timing_pairs && h[3] > h[2]) {
          out->pair_kernel_ms = std::max(out->pair_kernel_ms, (h[3] - h[2]) * 1e-6);
        }
      } else if (e->timing && s.row1 > s.row0) {
        float a = 0, b = 0;
        set_dev(s);
        if (e->timing_pairs && cudaEventElapsedTime(&a, s.ev[1], s.ev[2]) == cudaSuccess) {
          out->pair_kernel_ms = std::max(out->pair_kernel_ms, static_cast<double>(a));
        }
        if (cudaEventElapsedTime(&b, s.ev[0], s.ev[3]) == cudaSuccess) {
          out->eval_ms = std::max(out->eval_ms, static_cast<double>(b));
        }
      }
    }
    cudaGetLastError();
  });
}

}  // extern "C"
