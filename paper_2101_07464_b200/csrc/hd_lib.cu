// Host side of the B200 Householder Dice library: operator state, the
// per-probe launch sequences, device dynamics, CUDA-graph
// replay, instrumentation and the C-ABI declared in include/hd.h.
//
// Reference semantics restated here (file:line into /root/reference/proj):
//   GinibreOperator::probe   include/lazymat/ginibre.hpp:58-106
//   HaarOperator::probe      include/lazymat/haar.hpp:40-67
//   GOEOperator::probe       include/lazymat/ensembles.hpp:117-127
//   run_dynamics             include/lazymat/dynamics.hpp:42-76
//   check_probe_input        include/lazymat/operators.hpp:44-48
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "hd_complex.cuh"
#include "hd_complex_fused.cuh"
#include "hd_complex_gin.cuh"
#include "hd_refrng.hpp"
#include "hd_shard.cuh"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "../../include/hd.h"
#include "hd_kernels.cuh"
#include "hd_fused.cuh"
#include "hd_gin2p.cuh"

using namespace hd;

namespace {

thread_local std::string g_err;

struct HdError : std::runtime_error {
  int code;
  HdError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void require(bool cond, const std::string& msg) {
  if (!cond) throw HdError(HD_ERR_INVALID_ARGUMENT, msg);
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw HdError(HD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// HD_POISON=1 (debug): fill every fresh allocation with 0xFF bytes (NaN for
// doubles, -1 for ints) so a read-before-write shows up in the parity tests.
bool poison_allocs() {
  const char* e = std::getenv("HD_POISON");
  return e && e[0] == '1';
}

template <typename P>
P* dmalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  ck(cudaMalloc(&p, count * sizeof(P)), "cudaMalloc");
  if (poison_allocs()) {
    ck(cudaMemset(p, 0xFF, count * sizeof(P)), "poison");
    ck(cudaDeviceSynchronize(), "poison sync");
  }
  return static_cast<P*>(p);
}

// ----------------------------------------------------------------- chains
struct Panel {
  void* P = nullptr;  // tile-major, dtype bytes esz
  int64_t K = 0;      // column capacity
  int64_t count = 0;  // columns in use
};

struct Chain {
  Panel pan;
  int pend = -1;  // column whose Gram/T column is not yet known
  ChainDev dev;   // K-sized small state
};

struct FlushBufs {
  double* partials = nullptr;
  double* scratch = nullptr;
  int* counters = nullptr;
};

struct KStat {
  int64_t launches = 0;
  double ms = 0.0;
  double bytes = 0.0;
};

struct PendingEv {
  cudaEvent_t a, b;
  std::string kind;
  double bytes;
  std::string note;
};
constexpr int kDrawBlock = 16;  // probes per block of the small-operator draw cache
thread_local std::string g_prof_note;  // HD_PROF_LOG: shape of the next launch (launch_nt)

// host-side counters, snapshotted per step so a failed probe / aborted run
// can restore the exact reference state (operators.hpp:44-48: a failed probe
// leaves the operator untouched)
struct Counters {
  int64_t r = 0, l = 0, t = 0;  // Ginibre right/left; Haar probes
  int64_t rc_count = 0, lc_count = 0, u_count = 0, v_count = 0;
  int rc_pend = -1, lc_pend = -1;
  uint32_t probe_index = 0;
  int64_t inj_pos = 0;
  // speculative mix-Gram dots left by the previous Haar k_apply(OTHER):
  // chain (0 = R, 1 = L) dotted with the draw of probe `spec_probe`
  int spec_chain = -1;
  uint32_t spec_probe = 0;
  int64_t spec_inj = -1;
  int spec_count = 0, spec_nblk = 0, spec_slot0 = 0;
  int spec_col = 0;  // ... and wrote the next mix column, its norm^2 and pivot
};

}  // namespace

// Row layout of one dimension (n: right-probe input; m: its output). An
// unsharded operator owns all rows; a shard owns [lo, hi) plus, on shards
// > 0, a replica of the head rows [0, H) in its first local tiles.
struct ShardDim {
  int64_t N = 0;
  int64_t lo = 0, hi = 0;
  int64_t own_tiles = 0;
  hd::RowMap rm;
  int64_t rows_pad = 0;  // local panel rows
  int64_t vlen() const { return hi - lo; }
};

struct hd_exchange {
  std::unique_ptr<hd::Exchange> ex;
};

namespace {
struct CxState;  // complex-field operator state (hd_complex_host.inc)
}

// One recorded launch of a single operator (batched runs, hd_batch_run): the
// kernel, its launch shape and its one by-value parameter.
struct BatchRec {
  const void* fn = nullptr;
  dim3 grid, block;
  size_t smem = 0;
  std::vector<unsigned char> arg;
};
struct BatchPlan;

// Shape and schedule knobs of the two-pass kernels (hd_gin2p_host.inc), read
// from the environment when an operator is created (A/B measurements, tests):
// HD_NT_STAGE_KB, HD_NT_MAX_RS, HD_NT_MIN_STAGES, HD_NT_SCHED, HD_NT_L2PROMO,
// HD_NT_EVICT, HD_NT_DEAL.
struct NtKnobs {
  int stage_kb = 56;   // target stage size; 48 -> 56 KB: config 4 2.689 -> 2.661 s
  int max_rs = 256;    // tallest sub-tile (16..256 rows)
  int min_stages = 4;  // below this stage count a shorter sub-tile is taken
  int sched = -1;      // slot schedule: -1 auto (two-slot at 4 stages), 0 / 1 forced
  int l2promo = -1;    // L2 promotion bytes of the boxes: -1 auto (the column segment)
  int evict = 0;       // panel boxes evict_first (0) or evict_normal (1)
  int deal = 0;        // sub-tiles round robin (0) or by tile (1)
};

struct hd_op {
  hd_config cfg{};
  int ens = 0;
  bool f32 = false;
  size_t esz = 8;
  int64_t m = 0, n = 0;  // inner Ginibre m x n (Haar/GOE: n x n)
  int64_t rows_pad_m = 0, rows_pad_n = 0;  // local panel rows (= dm/dn.rows_pad)
  ShardDim dm, dn;
  CxState* cx = nullptr;  // set for HD_C128 operators
  // row sharding: shard_count > 1 => exchange after every
  // streaming kernel; head_rows H = rows the single-CTA stages read
  int shard_count = 1, shard_rank = 0;
  hd::Exchange* ex = nullptr;
  int64_t head_rows = 0, shard_cap = 0;
  double* xch[3] = {nullptr, nullptr, nullptr};  // exchange buffers: dots / fold / other
  int64_t xch_cap = 0;
  int64_t budget = 0;    // inner probes
  Chain R, L;            // right chain (dim n), left chain (dim m)
  Panel U, V;            // Ginibre basis stores: U (m) right probes, V (n) left probes
  Counters c;
  // scratch
  double* partials = nullptr;
  double* partials2 = nullptr;  // per-tile partials of update kernels
  double* partsF = nullptr;     // k_apply(FOLD) partials [slot][block]
  double* partsO = nullptr;     // k_apply(OTHER) partials (live until next probe)
  size_t partsF_cap = 0, partsO_cap = 0;
  double* specbuf = nullptr;    // [K] reduced speculative dots
  FlushBufs fbD, fbF, fbO;      // group partials / per-CTA scratch / tickets
  FlushBufs fbA[2], fbB;        // two-pass Ginibre: fold passes (ping-pong) and output passes
  double* drawbuf[2] = {nullptr, nullptr};  // two-pass Ginibre: device draws of a probe (io_len each)
  // small square operators: two blocks of kDrawBlock future draws each, one k_draw_fill
  // launch per block instead of one per probe (ensure_draw)
  double* drawcache = nullptr;
  NtKnobs nt;                   // two-pass kernel shapes (HD_NT_* environment)
  int gin2p = 1;                // two-pass Ginibre / GOE runs: 1 auto, 2 forced (HD_GIN2P=1), 0 off (HD_GIN2P=0)
  size_t flush_slots = 0;       // slot capacity of the buffers above
  double* red = nullptr;
  size_t red_cap = 0;
  double* scal = nullptr;
  int* status = nullptr;
  double *beta1 = nullptr, *beta3 = nullptr, *tmp = nullptr, *tmp2 = nullptr, *coefS = nullptr;
  double *head = nullptr, *zbuf = nullptr, *csp = nullptr;
  int64_t small_cap = 0;  // length of the K-sized scratch above
  void* xbuf = nullptr;   // dtype, rows_pad(max)
  void* ybuf[3] = {nullptr, nullptr, nullptr};
  void* gtmp = nullptr;   // GOE right-probe partial output
  int64_t io_len = 0;
  // queued draws (HD_DRAWS_INJECTED / HD_DRAWS_REFERENCE): inj[i] is draw
  // number inj_base + i of the operator's flat Gaussian stream; c.inj_pos is
  // the next one a probe consumes
  double* inj = nullptr;
  int64_t inj_cap = 0, inj_size = 0, inj_base = 0;
  std::unique_ptr<hd::refrng::Source> ref;  // HD_DRAWS_REFERENCE generator
  std::vector<double> ref_host;             // staging for generated draws
  cudaStream_t stream = nullptr;  // every kernel of the handle runs here
  cudaEvent_t ev_fork = nullptr;  // orders `stream` after the caller's stream
  int nsm = 148;
  std::map<long, int> dots_bps;  // smem bytes -> co-resident clusters
  std::map<long, int> apply_bps;
  int last_other_grid = 0, last_other_slot_ss = 0;  // normalize partials of k_apply(OTHER)
  bool pdl = true;  // programmatic dependent launch (HD_NO_PDL=1 disables)
  std::vector<BatchRec>* rec = nullptr;  // recording instead of launching (hd_batch_run)
  int batch_hint = 1;                    // operators sharing each launch (grid sizing)
  std::shared_ptr<BatchPlan> batch;      // cached batched run (this op leads it)
  int spare_sms = 0;  // SMs the persistent streaming grids leave free (HD_SPARE_SMS)
  int max_warps = 8;  // streaming warps per CTA cap (HD_WARPS fixes it)
  bool warps_fixed = false;
  int late_launch = 0;   // three-pass single-CTA stages trigger the next launch on exit (HD_LATE_LAUNCH=1)
  bool dots_split = true;  // k_dots shares tiles among warps at small n (HD_DOTS_SPLIT=0 disables)
  bool apply_split = true; // k_apply: one CTA per tile at small n (HD_APPLY_SPLIT=0 disables)
  bool gin_merge = true;   // square Ginibre: draw dots as k_dots' third job (HD_GIN_MERGE=0 disables)
  int fused = 1;         // two-pass Haar runs (hd_fused.cuh; HD_FUSED=0 disables)
  bool fused_retry = false;  // the current run fell back to the three-pass sequence
  // two-pass tuning / A/B knobs, read at hd_create (hd_fused_host.inc)
  double fused_guard = -1.0, fused_check = -1.0;  // HD_FUSED_GUARD / HD_FUSED_CHECK (< 0: defaults)
  int fused_late = -1;                             // HD_2P_LATE (< 0: default)
  bool fused_reverse = false;                      // HD_2P_REVERSE=1
  bool fused_cluster = true;                       // stage on a 2-CTA cluster (HD_2P_CLUSTER=0: one CTA)
  std::string fused_stage_order;                   // HD_2P_STAGE_ORDER
  int fold_reverse = 1;  // fold streams its panel last-to-first (HD_FOLD_FORWARD=1 disables)
  int64_t l2_keep = 96ll << 20;  // k_dots keeps its last bytes in L2 for that fold (HD_L2_KEEP_MB)
  int64_t l2_fold_keep = 0;  // ... and the fold its last bytes for the next k_dots (HD_L2_FOLD_KEEP_MB)
  unsigned long long* seed_dev = nullptr;  // Philox key (device word, hd_reseed)
  // hd_run_async bookkeeping, completed by hd_wait
  bool run_pending = false;
  hd_run_args pend_args{};
  std::vector<Counters> pend_snaps;
  int64_t pend_fdim = 0, pend_dim1 = 0;
  void* pend_traj_dev = nullptr;
  bool pend_final_deferred = false;  // device x_{T+1} copied out by hd_wait (two-pass runs)
  // normalize runs on the two-pass Ginibre sequence: the previous step's 1 / ||y|| is left to
  // the next probe's k_small_dots (flush_norm launches k_small_norm if that stage is not taken)
  bool norm_defer = false;
  const double* norm_parts = nullptr;
  int norm_nblk = 0, norm_step = 0;
  cudaStream_t pend_stream = nullptr;
  unsigned long long* trace = nullptr;  // HD_TRACE=1: phase stamps of k_small_dots
  std::vector<double> trace_acc;        // accumulated phase durations (ns)
  int64_t trace_n = 0;
  unsigned long long* trace2 = nullptr;  // HD_TRACE=2: [probe][16] stage stamps of two-pass runs
  unsigned long long* trace3 = nullptr;  // HD_TRACE=3: k_nt cycle breakdown [fold, gin][8][SMs]
  int64_t trace2_cap = 0, trace2_used = 0;
  // graph cache (hd_run from a fresh state)
  cudaGraphExec_t graph = nullptr;
  std::string graph_key;
  std::vector<Counters> graph_snaps;  // per-step host state recorded at capture
  int64_t graph_launches = 0;         // kernels inside the captured graph
  int64_t layout_gen = 0;  // bumped by every reallocation a captured graph could point into
  // device-resident application runs (hd_run_amp / hd_run_spiked, hd_apps.inc)
  void* appv[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t appv_bytes[6] = {0, 0, 0, 0, 0, 0};
  double* app_out = nullptr;
  int64_t app_out_cap = 0;
  double* app_red = nullptr;  // row-sharded runs: the map's sums, exchanged
  cudaGraphExec_t app_graph = nullptr;
  std::string app_graph_key;
  Counters app_graph_end;
  int64_t app_graph_launches = 0;
  // instrumentation
  bool prof = false;
  std::map<std::string, KStat> stats;
  std::vector<PendingEv> evq;
  std::vector<cudaEvent_t> evpool;
  int64_t launches = 0;
};

// A batched run (hd_batch_run): the launch sequence of one run recorded for
// every operator of the batch, each launch replayed ONCE with gridDim.y =
// operators and the per-operator parameters in a device table (arena), and
// the whole sequence captured in one CUDA graph. Operators run in lockstep
// (same shape, iterations and side schedule), so their sequences match.
struct BatchPlan {
  std::string key;
  std::vector<hd_op*> ops;
  cudaGraphExec_t graph = nullptr;
  unsigned char* arena = nullptr;
  std::vector<Counters> end_state;   // host counters of each operator after the run
  std::vector<const void*> fin;      // where each operator's x_{T+1} ends up
  int64_t dim1 = 0, fdim = 0;
  int64_t launches = 0;              // batched kernels in the graph
  int64_t op_launches = 0;           // kernels one operator would have launched
  ~BatchPlan() {
    if (graph) cudaGraphExecDestroy(graph);
    if (arena) cudaFree(arena);
  }
};

namespace {

// ============================================================ allocation
void alloc_chain(hd_op* op, Chain& ch, int64_t rows_pad, int64_t K) {
  ch.pan.K = K;
  ch.pan.count = 0;
  ch.pend = -1;
  ch.pan.P = dmalloc<unsigned char>((size_t)rows_pad * K * op->esz);
  ck(cudaMemsetAsync(ch.pan.P, 0, (size_t)rows_pad * K * op->esz, op->stream), "memset panel");
  ch.dev.K = K;
  ch.dev.Dlen = K;
  ch.dev.sig = dmalloc<double>(K);
  ch.dev.c = dmalloc<double>(K);
  ch.dev.s = dmalloc<double>(K);
  ch.dev.G = dmalloc<double>((size_t)K * K);
  ch.dev.Tm = dmalloc<double>((size_t)K * K);
  ch.dev.Drow = dmalloc<double>(K);
  ch.dev.Dtail = dmalloc<double>(1);
  ck(cudaMemsetAsync(ch.dev.G, 0, sizeof(double) * K * K, op->stream), "memset");
  ck(cudaMemsetAsync(ch.dev.Tm, 0, sizeof(double) * K * K, op->stream), "memset");
}

void free_chain(Chain& ch) {
  cudaFree(ch.pan.P);
  cudaFree(ch.dev.sig);
  cudaFree(ch.dev.c);
  cudaFree(ch.dev.s);
  cudaFree(ch.dev.G);
  cudaFree(ch.dev.Tm);
  cudaFree(ch.dev.Drow);
  cudaFree(ch.dev.Dtail);
  ch = Chain{};
}

void alloc_store(hd_op* op, Panel& p, int64_t rows_pad, int64_t K) {
  p.K = K;
  p.count = 0;
  p.P = dmalloc<unsigned char>((size_t)rows_pad * K * op->esz);
  ck(cudaMemsetAsync(p.P, 0, (size_t)rows_pad * K * op->esz, op->stream), "memset store");
}

__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }

__global__ void k_fill(double* p, int64_t n, const double* v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = *v;
}

// Grow a panel's column capacity (tile-major re-layout via pitched copy).
void grow_panel(hd_op* op, Panel& p, int64_t rows_pad, int64_t Knew) {
  void* np = dmalloc<unsigned char>((size_t)rows_pad * Knew * op->esz);
  ck(cudaMemsetAsync(np, 0, (size_t)rows_pad * Knew * op->esz, op->stream), "memset");
  const int64_t ntiles = rows_pad / kTile;
  if (p.count > 0)
    ck(cudaMemcpy2DAsync(np, (size_t)Knew * kTile * op->esz, p.P, (size_t)p.K * kTile * op->esz,
                         (size_t)p.count * kTile * op->esz, (size_t)ntiles, cudaMemcpyDeviceToDevice, op->stream),
       "grow copy");
  ck(cudaStreamSynchronize(op->stream), "sync");
  cudaFree(p.P);
  p.P = np;
  p.K = Knew;
  op->layout_gen++;
}

void grow_chain(hd_op* op, Chain& ch, int64_t rows_pad, int64_t Knew) {
  const int64_t Kold = ch.pan.K;
  op->c.spec_col = 0;  // a mix column pre-written beyond `count` is not carried over
  grow_panel(op, ch.pan, rows_pad, Knew);
  auto grow_vec = [&](double*& v) {
    double* nv = dmalloc<double>(Knew);
    ck(cudaMemcpyAsync(nv, v, sizeof(double) * Kold, cudaMemcpyDeviceToDevice, op->stream), "grow");
    ck(cudaStreamSynchronize(op->stream), "sync");
    cudaFree(v);
    v = nv;
  };
  auto grow_mat = [&](double*& M) {
    double* nm = dmalloc<double>((size_t)Knew * Knew);
    ck(cudaMemsetAsync(nm, 0, sizeof(double) * Knew * Knew, op->stream), "memset");
    ck(cudaMemcpy2DAsync(nm, sizeof(double) * Knew, M, sizeof(double) * Kold, sizeof(double) * Kold, Kold,
                         cudaMemcpyDeviceToDevice, op->stream),
       "grow mat");
    ck(cudaStreamSynchronize(op->stream), "sync");
    cudaFree(M);
    M = nm;
  };
  grow_vec(ch.dev.sig);
  grow_vec(ch.dev.c);
  grow_vec(ch.dev.s);
  grow_vec(ch.dev.Drow);
  grow_mat(ch.dev.G);
  grow_mat(ch.dev.Tm);
  // rows [Kold, Knew) lie beyond every existing offset: D = Dtail there
  k_fill<<<(unsigned)ceil_div(Knew - Kold, 256), 256, 0, op->stream>>>(ch.dev.Drow + Kold, Knew - Kold, ch.dev.Dtail);
  ck(cudaGetLastError(), "k_fill");
  ch.dev.K = Knew;
  ch.dev.Dlen = Knew;
}

void ensure_small(hd_op* op, int64_t K) {
  if (K <= op->small_cap) return;
  for (double** p : {&op->beta1, &op->beta3, &op->tmp, &op->tmp2, &op->coefS, &op->head, &op->zbuf, &op->csp,
                     &op->specbuf}) {
    cudaFree(*p);
    *p = dmalloc<double>(K + 8);
  }
  op->small_cap = K;
  op->layout_gen++;
}

void ensure_red(hd_op* op, size_t nslots) {
  if (nslots > op->red_cap) {
    cudaFree(op->red);
    op->red_cap = nslots * 2;
    op->red = dmalloc<double>(op->red_cap);
    op->layout_gen++;
  }
}

// Capacity for `nr` more right and `nl` more left inner probes (Haar: both
// chains gain one column per probe; Ginibre: R/U per right, L/V per left).
void ensure_capacity(hd_op* op, int64_t nr, int64_t nl) {
  auto target = [&](int64_t K, int64_t need) {
    int64_t k = std::max<int64_t>(K, 1);
    while (k < need) k *= 2;
    return std::min(std::max(k, need), std::max<int64_t>(op->budget, 1));
  };
  int64_t total;
  if (op->ens == HD_HAAR) {
    total = std::min(op->c.t + nr + nl, op->budget);
    if (op->R.pan.K < total) grow_chain(op, op->R, op->rows_pad_n, target(op->R.pan.K, total));
    if (op->L.pan.K < total) grow_chain(op, op->L, op->rows_pad_n, target(op->L.pan.K, total));
  } else {
    total = std::min(op->c.r + op->c.l + nr + nl, op->budget);
    const int64_t needR = std::min(op->c.r + nr, op->budget), needL = std::min(op->c.l + nl, op->budget);
    if (op->R.pan.K < needR) grow_chain(op, op->R, op->rows_pad_n, target(op->R.pan.K, needR));
    if (op->U.K < needR) grow_panel(op, op->U, op->rows_pad_m, target(op->U.K, needR));
    if (op->L.pan.K < needL) grow_chain(op, op->L, op->rows_pad_m, target(op->L.pan.K, needL));
    if (op->V.K < needL) grow_panel(op, op->V, op->rows_pad_n, target(op->V.K, needL));
  }
  const int64_t K = std::max({op->R.pan.K, op->L.pan.K, op->U.K, op->V.K});
  ensure_small(op, std::max<int64_t>(K, total) + 1);
  // partial buffers sized for the widest launch (<= 8 CTAs of 256 per SM), so
  // nothing is allocated inside a captured CUDA graph. fbO.partials may hold
  // the previous probe's speculative dots: preserved across growth.
  const size_t blocks = (size_t)op->nsm;
  const size_t groups = ceil_div((int64_t)blocks, kGroup);
  const size_t slots = (size_t)(4 * K + 16);
  if (slots > op->flush_slots) {
    for (FlushBufs* fb : {&op->fbD, &op->fbF, &op->fbO, &op->fbA[0], &op->fbA[1], &op->fbB}) {
      double* np = dmalloc<double>(slots * groups);
      if (fb->partials && fb == &op->fbO)
        ck(cudaMemcpy(np, fb->partials, sizeof(double) * op->flush_slots * groups, cudaMemcpyDeviceToDevice), "keep");
      cudaFree(fb->partials);
      fb->partials = np;
      cudaFree(fb->scratch);
      fb->scratch = dmalloc<double>(slots * blocks);
      if (!fb->counters) {
        fb->counters = dmalloc<int>(groups);
        ck(cudaMemset(fb->counters, 0, sizeof(int) * groups), "memset");
      }
    }
    op->flush_slots = slots;
    op->layout_gen++;
  }
  if (op->ens != HD_HAAR && !op->drawbuf[0])  // two-pass Ginibre draw buffers (before any graph capture)
    for (double*& b : op->drawbuf) b = dmalloc<double>(std::max<int64_t>(op->io_len, 2));
  if (op->ens != HD_HAAR && !op->drawcache && op->m == op->n && op->ex == nullptr && op->cfg.draw_mode == HD_DRAWS_PHILOX &&
      op->io_len * 8 * 2 * kDrawBlock <= (int64_t(16) << 20))
    op->drawcache = dmalloc<double>(2 * kDrawBlock * op->io_len);
  op->partials = op->fbD.partials;
  op->partsF = op->fbF.partials;
  op->partsO = op->fbO.partials;
  ensure_red(op, slots);
}

// The handle's stream is non-blocking, so nothing orders it after the
// caller's stream implicitly (not even the legacy NULL stream). Every entry
// point that reads caller data first makes op->stream wait for the work
// already enqueued on the caller's stream. No join is needed: every entry
// point returns after a host sync of op->stream (hd_wait for async runs).
void fork_from(hd_op* op, cudaStream_t caller) {
  if (caller == op->stream) return;
  ck(cudaEventRecord(op->ev_fork, caller), "fork record");
  ck(cudaStreamWaitEvent(op->stream, op->ev_fork, 0), "fork wait");
}

// ========================================================= instrumentation
cudaEvent_t get_event(hd_op* op) {
  if (!op->evpool.empty()) {
    cudaEvent_t e = op->evpool.back();
    op->evpool.pop_back();
    return e;
  }
  cudaEvent_t e;
  ck(cudaEventCreate(&e), "event");
  return e;
}

struct LaunchScope {
  hd_op* op;
  cudaStream_t s;
  const char* kind;
  double bytes;
  cudaEvent_t a = nullptr;
  LaunchScope(hd_op* o, cudaStream_t st, const char* k, double b) : op(o), s(st), kind(k), bytes(b) {
    op->launches++;
    if (op->prof) {
      a = get_event(op);
      cudaEventRecord(a, s);
    }
  }
  ~LaunchScope() {
    if (op->prof) {
      cudaEvent_t b = get_event(op);
      cudaEventRecord(b, s);
      op->evq.push_back({a, b, kind, bytes, g_prof_note});
      g_prof_note.clear();
      KStat& st = op->stats[kind];
      st.launches++;
      st.bytes += bytes;
    }
  }
};

void drain_events(hd_op* op) {
  if (op->evq.empty()) return;
  cudaStreamSynchronize(op->stream);
  // HD_PROF_LOG=path: one line per launch (kind, algorithmic bytes, ms) — a
  // diagnostic of profiling runs (hd_set_profiling), never on by default
  static const char* log_path = std::getenv("HD_PROF_LOG");
  FILE* lf = log_path ? std::fopen(log_path, "a") : nullptr;
  for (auto& e : op->evq) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    op->stats[e.kind].ms += ms;
    if (lf) std::fprintf(lf, "%s %.0f %.6f %s\n", e.kind.c_str(), e.bytes, (double)ms, e.note.c_str());
    op->evpool.push_back(e.a);
    op->evpool.push_back(e.b);
  }
  if (lf) std::fclose(lf);
  op->evq.clear();
}

void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw HdError(HD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Raise (never lower) a kernel's dynamic shared-memory limit. A captured
// graph keeps each node's launch size, and a node must stay within the
// function's limit when the graph is replayed (ncu re-checks it per node), so
// a later, smaller launch must not shrink the limit an earlier node needs.
void raise_smem_limit(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  cudaFuncAttributes fa{};
  ck(cudaFuncGetAttributes(&fa, fn), "func attr");
  if ((size_t)fa.maxDynamicSharedSizeBytes < bytes)
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes), "smem attr");
}

// =========================================================== launchers
// Persistent launch of a streaming kernel: grid = SMs x co-resident CTAs
// (at most one warp-tile per warp); partial sums leave through Flush in
// groups of kGroup CTAs. Returns the number of partial rows (groups).
// Every kernel of the probe sequence is launched with programmatic stream
// serialization (PDL); the kernels order themselves with
// griddepcontrol.wait / launch_dependents.
template <typename... KArgs, typename... Args>
void launch_k(hd_op* op, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
              Args&&... args) {
  if (op->rec) {  // batched-run recording: keep the launch, do not issue it
    if constexpr (sizeof...(KArgs) == 1) {
      using A = std::decay_t<std::tuple_element_t<0, std::tuple<KArgs...>>>;
      const A v(std::forward<Args>(args)...);
      BatchRec r;
      r.fn = reinterpret_cast<const void*>(kernel);
      r.grid = grid;
      r.block = block;
      r.smem = smem;
      r.arg.resize(sizeof(A));
      std::memcpy(r.arg.data(), &v, sizeof(A));
      op->rec->push_back(std::move(r));
      return;
    } else {
      throw HdError(HD_ERR_RUNTIME, "hd: this launch cannot be batched");
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = op->pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  ck(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

// Persistent launch of a per-warp TMA streaming kernel: up to kMaxWarps
// warps per CTA (up to as many as the per-warp ring + slot rows fit in the
// opt-in shared memory), one CTA per SM; partial sums leave through Flush in
// groups of kGroup CTAs. Returns the number of partial rows.
//
// Each warp streams a contiguous run of tiles, so a launch ends with the warps
// that hold ceil(ntiles / W) tiles (W = CTAs x warps) streaming alone, and too
// few warps with 3-stage rings cannot keep HBM saturated in that last round.
// Among the three largest feasible warp counts, the one whose W divides the
// tiles most evenly is used (ties: more warps). Measured on config 2
// (n = 1e6, 3907 tiles): 8 warps (balance 0.83) 24.3 ms, 7 warps (0.94)
// 23.3 ms; at n = 1e7 8 warps (0.9998) stays best. HD_WARPS fixes the count.
template <typename Args>
int launch_tma(hd_op* op, cudaStream_t s, void (*kernel)(Args), Args& args, size_t shared_fixed, size_t per_warp,
               int64_t ntiles, const FlushBufs& fb, int64_t fixed_grid = 0) {
  int optin = 0;
  ck(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, op->cfg.device), "attr");
  const size_t budget = (size_t)optin - 1024;
  if (shared_fixed + per_warp > budget) throw HdError(HD_ERR_RESOURCE_CAP, "hd: chain too long for one CTA");
  const int nw_cap = (int)std::min<size_t>(std::min(kMaxWarps, op->max_warps), (budget - shared_fixed) / per_warp);
  // a batched launch shares the SMs among its operators
  const int sms = std::max(1, (op->nsm - op->spare_sms) / std::max(1, op->batch_hint));
  int nw = nw_cap;
  if (!op->warps_fixed) {
    double best = -1.0;
    for (int cand = nw_cap; cand >= std::max(1, nw_cap - 2); --cand) {
      const int64_t g = std::max<int64_t>(1, std::min<int64_t>(ceil_div(ntiles, cand), sms));
      const int64_t W = g * cand;
      const double balance = (double)ntiles / (double)(W * ceil_div(ntiles, W));
      if (balance > best + 1e-9) {
        best = balance;
        nw = cand;
      }
    }
  }
  const size_t smem = shared_fixed + (size_t)nw * per_warp;
  raise_smem_limit(reinterpret_cast<const void*>(kernel), smem);
  const int grid = fixed_grid > 0 ? (int)fixed_grid : (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(ntiles, nw), sms));
  args.out.partials = fb.partials;
  args.out.scratch = fb.scratch;
  args.out.counters = fb.counters;
  launch_k(op, kernel, dim3(grid), dim3(nw * 32), smem, s, args);
  return (int)ceil_div(grid, kGroup);
}

template <typename T>
int launch_dots(hd_op* op, cudaStream_t s, DotArgs<T>& a, double bytes) {
  // slot layout: per job [dot: ncols][pend: pend+1][sumsq: 1]
  int slot = 0;
  for (int jb = 0; jb < a.njobs; ++jb) {
    DotJob<T>& J = a.job[jb];
    J.slot_dot = slot;
    slot += J.ncols;
    if (J.pend >= 0) {
      J.slot_pend = slot;
      slot += J.pend + 1;
    }
    J.slot_sumsq = slot++;
  }
  a.nslots = slot;
  a.status = op->status;
  const size_t per_warp = ring_bytes<T>() + sizeof(double) * ((a.nslots + 1) & ~1) + 8 * kRing;
  // few tiles (small n): split each tile's chunks over several warps, up to
  // about half the warp slots of the SMs this launch may use
  {
    int64_t chunks = 0;
    for (int j = 0; j < a.njobs; ++j) chunks += (a.job[j].ncols + chunk_cols<T>() - 1) / chunk_cols<T>();
    // launch_tma picks one of the three largest feasible warp counts and caps
    // the grid at the SMs: every (tile, group) work item needs a warp
    int optin = 0;
    ck(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, op->cfg.device), "attr");
    const int nw_cap = (int)std::min<size_t>(std::min(kMaxWarps, op->max_warps), ((size_t)optin - 1024) / per_warp);
    const int nw_min = op->warps_fixed ? nw_cap : std::max(1, nw_cap - 2);
    const int64_t sms = std::max(1, (op->nsm - op->spare_sms) / std::max(1, op->batch_hint));
    const int64_t slots = std::min<int64_t>(sms * kMaxWarps / 2, sms * nw_min);
    // the single-CTA stage stages nslots x (CTAs / kGroup) partial rows:
    // keep that under 64 KB (at >= 6 warps per CTA)
    const int64_t max_groups = std::max<int64_t>(1, 65536 / (8 * std::max(1, a.nslots)));
    const int64_t max_warps = max_groups * kGroup * 6;
    a.split = 1;
    if (op->dots_split && a.ntiles > 0 && a.ntiles * 2 <= slots && chunks >= 2)
      a.split = (int)std::max<int64_t>(1, std::min<int64_t>({chunks, slots / a.ntiles, max_warps / a.ntiles, 64}));
  }
  int grid;
  {
    LaunchScope ls(op, s, "dots", bytes);
    grid = launch_tma(op, s, k_dots<T>, a, 0, per_warp, a.ntiles * a.split, op->fbD);
  }
  check_launch("k_dots");
  return grid;
}

template <typename T, int MODE>
int launch_apply(hd_op* op, cudaStream_t s, ApplyArgs<T>& a, bool fold_buffer, double bytes, const char* kind) {
  int slot = 0;
  if (a.spec.kind != kSrcNone) {
    a.slot_spec = slot;
    slot += a.ncols + (MODE == kApplyFold ? 1 : 0);
    if (a.gcol) a.slot_gss = slot++;  // = slot_spec + ncols (k_small_dots reads it as spec row kB)
  }
  a.slot_ss = slot++;
  a.nslots = slot;
  a.status = op->status;
  // few tiles (small n): one CTA per tile, its warps splitting the chunks
  const int sms = std::max(1, (op->nsm - op->spare_sms) / std::max(1, op->batch_hint));
  a.cta_split = (op->apply_split && a.ntiles * 2 <= sms && a.ncols >= 2 * chunk_cols<T>()) ? 1 : 0;
  const size_t per_warp = ring_bytes<T>() + sizeof(double) * ((a.nslots + 1) & ~1) + 8 * kRing +
                          (a.cta_split ? sizeof(double2) * 128 : 0);
  int grid;
  {
    LaunchScope ls(op, s, kind, bytes);
    grid = launch_tma(op, s, k_apply<T, MODE>, a, sizeof(double) * ((a.ncols + 1) & ~1) + 16, per_warp, a.ntiles,
                      fold_buffer ? op->fbF : op->fbO, a.cta_split ? a.ntiles : 0);
  }
  check_launch("k_apply");
  return grid;
}

// Shared memory of a single-CTA stage (k_small_dots = 0, k_small_fold = 1,
// k_small_gin = 2); decides what is staged within the budget: the partial
// rows, heads and sparse-input corner first, then the T corners (k x (k|1)).
size_t small_smem_bytes(SmallArgs& a, int which, size_t esz) {
  const size_t kv = (size_t)small_kv(a.kA, a.kB);
  const size_t budget = 210 * 1024;
  size_t bytes = sizeof(double) * (12 * kv + 16);
  a.stageA = a.stageB = a.stageC = 0;
  bool needA = false, needB = false;
  size_t nr = 0;
  if (which == 0) {
    bytes += sizeof(double) * (size_t)a.nslots_in * a.nblk;
    if (a.is_haar && a.mix_from_spec) bytes += sizeof(double) * (size_t)(a.kB + a.spec_ss) * a.spec_nblk;
    needA = true;
    needB = a.is_haar != 0;
  } else if (which == 1) {
    nr = (size_t)a.off + 1;
    bytes += sizeof(double) * 2 * nr;
    needB = a.is_haar != 0;
  } else {
    nr = (size_t)a.csplen;
    bytes += sizeof(double) * ((size_t)a.nslots_in * a.nblk + 2 * nr);
    needB = true;
  }
  if (nr > 0 && (which == 2 || a.is_haar)) {
    const size_t c = esz * (size_t)a.kB * nr + 16;
    if (bytes + c <= budget) {
      a.stageC = 1;
      bytes += c;
    }
  }
  const size_t tA = sizeof(double) * (size_t)a.kA * (size_t)(a.kA | 1);
  const size_t tB = sizeof(double) * (size_t)a.kB * (size_t)(a.kB | 1);
  if (needA && a.kA > 0 && bytes + tA <= budget) {
    a.stageA = 1;
    bytes += tA;
  }
  if (needB && a.kB > 0 && bytes + tB <= budget) {
    a.stageB = 1;
    bytes += tB;
  }
  if (bytes > 227 * 1024) throw HdError(HD_ERR_RESOURCE_CAP, "hd: single-CTA stage exceeds shared memory");
  return bytes;
}

template <typename K>
void allow_smem(K kernel, size_t bytes) {
  raise_smem_limit(reinterpret_cast<const void*>(kernel), bytes);
}

template <typename T>
Src<T> vec_src(const void* x, const double* xscale) {
  Src<T> s;
  s.kind = kSrcVec;
  s.x = static_cast<const T*>(x);
  s.xscale = xscale;
  return s;
}

int64_t inj_avail(const hd_op* op) { return op->inj_base + op->inj_size - op->c.inj_pos; }
const double* inj_at(const hd_op* op, int64_t pos) { return op->inj + (pos - op->inj_base); }

// Append `len` draws (host or device pointer) to the queue.
void inj_append(hd_op* op, const double* g, int64_t len, bool on_device) {
  // slack of one padded row range: the two-pass kernels bulk-copy whole
  // sub-tiles of a probe's draws (rows past the dimension are masked)
  const int64_t slack = op->io_len;
  if (op->inj_size + len + slack > op->inj_cap) {
    const int64_t ncap = std::max<int64_t>(op->inj_cap * 2, op->inj_size + len + slack);
    double* np = dmalloc<double>(ncap);
    if (op->inj_size > 0)
      ck(cudaMemcpyAsync(np, op->inj, sizeof(double) * op->inj_size, cudaMemcpyDeviceToDevice, op->stream), "grow");
    ck(cudaStreamSynchronize(op->stream), "sync");
    cudaFree(op->inj);
    op->inj = np;
    op->inj_cap = ncap;
    op->layout_gen++;
  }
  ck(cudaMemcpyAsync(op->inj + op->inj_size, g, sizeof(double) * len,
                     on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, op->stream),
     "push");
  ck(cudaStreamSynchronize(op->stream), "sync");
  op->inj_size += len;
}

// HD_DRAWS_REFERENCE: make at least `count` unconsumed draws of the
// reference stream RandomSource(seed, stream) available. Consumed draws are
// dropped first (no probe can rewind below c.inj_pos: every snapshot is
// taken after this call), so the queue holds at most one run's draws.
void ref_ensure(hd_op* op, int64_t count) {
  if (op->cfg.draw_mode != HD_DRAWS_REFERENCE) return;
  const int64_t avail = inj_avail(op);
  if (avail >= count) return;
  const int64_t drop = op->c.inj_pos - op->inj_base;
  if (drop > 0) {
    if (avail > 0) {
      double* np = dmalloc<double>(std::max<int64_t>(op->inj_cap, 1));
      ck(cudaMemcpyAsync(np, op->inj + drop, sizeof(double) * avail, cudaMemcpyDeviceToDevice, op->stream), "compact");
      ck(cudaStreamSynchronize(op->stream), "sync");
      cudaFree(op->inj);
      op->inj = np;
    }
    op->inj_size = avail;
    op->inj_base = op->c.inj_pos;
  }
  const int64_t need = count - avail;
  op->ref_host.resize((size_t)need);
  op->ref->normal_fill(op->ref_host.data(), need);
  inj_append(op, op->ref_host.data(), need, false);
}

// The fresh draw of the current inner probe (ginibre.hpp:67/86, haar.hpp:48).
template <typename T>
Src<T> draw_src(hd_op* op, int64_t len) {
  Src<T> s;
  if (op->cfg.draw_mode != HD_DRAWS_PHILOX) {
    if (inj_avail(op) < len)
      throw HdError(HD_ERR_INVALID_ARGUMENT, "hd: injected draws exhausted (push one vector per probe)");
    s.kind = kSrcInjected;
    s.inj = inj_at(op, op->c.inj_pos);
    op->c.inj_pos += len;
  } else {
    s.kind = kSrcPhilox;
    s.seedp = op->seed_dev;
    s.stream = (uint32_t)op->cfg.stream;
    s.probe = op->c.probe_index;
  }
  op->c.probe_index++;
  return s;
}

double bytes_of(hd_op* op, double elems) { return elems * (double)op->esz; }

#include "hd_probe.inc"

#include "hd_run.inc"

#include "hd_apps.inc"

}  // namespace

#include "hd_cabi.inc"
