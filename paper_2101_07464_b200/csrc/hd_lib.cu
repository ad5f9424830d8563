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
#include <cuda_runtime.h>

#include "hd_complex.cuh"
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
#include <vector>

#include "../../include/hd.h"
#include "hd_kernels.cuh"

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
};

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
  int spare_sms = 0;  // SMs the persistent streaming grids leave free (HD_SPARE_SMS)
  int max_warps = 8;  // streaming warps per CTA cap (HD_WARPS fixes it)
  bool warps_fixed = false;
  unsigned long long* seed_dev = nullptr;  // Philox key (device word, hd_reseed)
  // hd_run_async bookkeeping, completed by hd_wait
  bool run_pending = false;
  hd_run_args pend_args{};
  std::vector<Counters> pend_snaps;
  int64_t pend_fdim = 0, pend_dim1 = 0;
  void* pend_traj_dev = nullptr;
  cudaStream_t pend_stream = nullptr;
  unsigned long long* trace = nullptr;  // HD_TRACE=1: phase stamps of k_small_dots
  std::vector<double> trace_acc;        // accumulated phase durations (ns)
  int64_t trace_n = 0;
  // graph cache (hd_run from a fresh state)
  cudaGraphExec_t graph = nullptr;
  std::string graph_key;
  std::vector<Counters> graph_snaps;  // per-step host state recorded at capture
  int64_t graph_launches = 0;         // kernels inside the captured graph
  // instrumentation
  bool prof = false;
  std::map<std::string, KStat> stats;
  std::vector<PendingEv> evq;
  std::vector<cudaEvent_t> evpool;
  int64_t launches = 0;
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
}

void ensure_red(hd_op* op, size_t nslots) {
  if (nslots > op->red_cap) {
    cudaFree(op->red);
    op->red_cap = nslots * 2;
    op->red = dmalloc<double>(op->red_cap);
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
    for (FlushBufs* fb : {&op->fbD, &op->fbF, &op->fbO}) {
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
  }
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
      op->evq.push_back({a, b, kind});
      KStat& st = op->stats[kind];
      st.launches++;
      st.bytes += bytes;
    }
  }
};

void drain_events(hd_op* op) {
  if (op->evq.empty()) return;
  cudaStreamSynchronize(op->stream);
  for (auto& e : op->evq) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    op->stats[e.kind].ms += ms;
    op->evpool.push_back(e.a);
    op->evpool.push_back(e.b);
  }
  op->evq.clear();
}

void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw HdError(HD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
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
               int64_t ntiles, const FlushBufs& fb) {
  int optin = 0;
  ck(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, op->cfg.device), "attr");
  const size_t budget = (size_t)optin - 1024;
  if (shared_fixed + per_warp > budget) throw HdError(HD_ERR_RESOURCE_CAP, "hd: chain too long for one CTA");
  const int nw_cap = (int)std::min<size_t>(std::min(kMaxWarps, op->max_warps), (budget - shared_fixed) / per_warp);
  const int sms = std::max(1, op->nsm - op->spare_sms);
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
  ck(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(ntiles, nw), sms));
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
  int grid;
  {
    LaunchScope ls(op, s, "dots", bytes);
    grid = launch_tma(op, s, k_dots<T>, a, 0, per_warp, a.ntiles, op->fbD);
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
  const size_t per_warp = ring_bytes<T>() + sizeof(double) * ((a.nslots + 1) & ~1) + 8 * kRing;
  int grid;
  {
    LaunchScope ls(op, s, kind, bytes);
    grid = launch_tma(op, s, k_apply<T, MODE>, a, sizeof(double) * ((a.ncols + 1) & ~1), per_warp, a.ntiles,
                      fold_buffer ? op->fbF : op->fbO);
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
  if (bytes > 48 * 1024) ck(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes), "smem");
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
  if (op->inj_size + len > op->inj_cap) {
    const int64_t ncap = std::max<int64_t>(op->inj_cap * 2, op->inj_size + len);
    double* np = dmalloc<double>(ncap);
    if (op->inj_size > 0)
      ck(cudaMemcpyAsync(np, op->inj, sizeof(double) * op->inj_size, cudaMemcpyDeviceToDevice, op->stream), "grow");
    ck(cudaStreamSynchronize(op->stream), "sync");
    cudaFree(op->inj);
    op->inj = np;
    op->inj_cap = ncap;
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

// ------------------------------------------------------------ row shards
void plan_dim(ShardDim& d, int64_t N, int count, int rank, int64_t head_rows) {
  d.N = N;
  if (count <= 1) {
    d.lo = 0;
    d.hi = N;
    d.own_tiles = ceil_div(N, kTile);
    d.rm = hd::RowMap{};
    d.rows_pad = d.own_tiles * kTile;
    return;
  }
  hd::shard_plan(N, count, rank, head_rows, &d.lo, &d.hi);
  d.own_tiles = ceil_div(d.hi - d.lo, kTile);
  const int64_t htiles = (rank == 0) ? 0 : ceil_div(head_rows, kTile);
  d.rm.tile0 = htiles;
  d.rm.gdelta = d.lo - htiles * kTile;
  d.rm.vbase = d.lo;
  d.rows_pad = (htiles + d.own_tiles) * kTile;
}

// An operator with an exchange runs the sharded protocol, even a 1-shard
// group (which exercises the NCCL path on a single GPU).
bool sharded(const hd_op* op) { return op->ex != nullptr; }

// One exchange after a streaming kernel (hd_shard.cuh): pack the group
// partials (fixed order) + shard 0's head payload + status flags into
// xch[which], allreduce over the shards, unpack the payload on shards > 0.
// Returns the reduced partials, laid out as [slot][1].
template <typename T>
const double* shard_exchange(hd_op* op, cudaStream_t s, int which, const double* partials, int nslots, int ngroups,
                             std::initializer_list<hd::XItem> items) {
  hd::XArgs a;
  a.partials = partials;
  a.nslots = nslots;
  a.ngroups = ngroups;
  int64_t len = nslots + kStWords;
  for (const hd::XItem& it : items) {
    if (a.nitems == hd::kXMaxItems) throw HdError(HD_ERR_RUNTIME, "hd: exchange payload overflow");
    a.item[a.nitems++] = it;
    len += hd::xitem_len(it, op->head_rows);
  }
  if (len > op->xch_cap) {  // grow; xch[2] may hold the speculative dots of the previous probe
    ck(cudaStreamSynchronize(s), "sync");
    for (double*& b : op->xch) {
      double* nb = dmalloc<double>(len * 2);
      if (b) ck(cudaMemcpy(nb, b, sizeof(double) * op->xch_cap, cudaMemcpyDeviceToDevice), "keep");
      cudaFree(b);
      b = nb;
    }
    op->xch_cap = len * 2;
  }
  a.X = op->xch[which];
  a.status = op->status;
  a.lead = (op->shard_rank == 0) ? 1 : 0;
  {
    LaunchScope ls(op, s, "xpack", 0.0);
    launch_k(op, hd::k_xpack<T>, dim3(1), dim3(256), 0, s, a, op->head_rows);
  }
  check_launch("k_xpack");
  {
    LaunchScope ls(op, s, "allreduce", 8.0 * len);
    op->ex->allreduce_sum(a.X, len, s, op->shard_rank);
  }
  {
    LaunchScope ls(op, s, "xunpack", 0.0);
    launch_k(op, hd::k_xunpack<T>, dim3(1), dim3(256), 0, s, a, op->head_rows);
  }
  check_launch("k_xunpack");
  return a.X;
}

hd::XItem xcol(const Panel& p, int64_t col) {
  hd::XItem it;
  it.pan = p.P;
  it.K = p.K;
  it.col = col;
  return it;
}

hd::XItem xvec(double* v, int64_t len) {
  hd::XItem it;
  it.vec = v;
  it.len = len;
  return it;
}

// --------------------------------------------------------------- Haar
// haar.hpp:40-67. fold = chain of the probed side, other = the opposite.
// Passes over HBM per probe: GEMV-T over fold (k_dots), GEMV-N over fold
// (k_apply FOLD), GEMV-N over other (k_apply OTHER). The other chain's Gram
// dots with this probe's draw come from the previous probe's OTHER pass
// when both probes hit the same side (speculative, Philox regenerated);
// otherwise k_dots streams the other chain too.
template <typename T>
void enqueue_haar(hd_op* op, int side, const Src<T>& xsrc, const Epi<T>& epi, cudaStream_t s) {
  const int64_t n = op->n;
  const int64_t ntiles = op->dn.own_tiles;
  const bool first = (op->c.t == 0);
  Src<T> xs = xsrc;
  xs.vbase = op->dn.rm.vbase;
  op->c.t += 1;
  const int64_t off = op->c.t - 1;
  Chain& F = (side == HD_RIGHT) ? op->R : op->L;
  Chain& O = (side == HD_RIGHT) ? op->L : op->R;
  const int ochain = (side == HD_RIGHT) ? 1 : 0;
  const bool append_fold = !(op->cfg.skip_reflector && first);
  const int64_t inj_before = op->c.inj_pos;
  Src<T> g = draw_src<T>(op, n);
  g.mask_begin = off;
  const bool key_ok = (g.kind == kSrcInjected) ? (op->c.spec_inj == inj_before) : (op->c.spec_probe == g.probe);
  const bool use_spec = op->c.spec_chain == ochain && key_ok && op->c.spec_count == (int)O.pan.count && O.pend < 0;
  const int spec_nblk = op->c.spec_nblk, spec_slot0 = op->c.spec_slot0, spec_count = op->c.spec_count;
  op->c.spec_chain = -1;

  // K1: a = P_F^T x (+ pending Gram), g[off:] -> new column of O, ||g_tail||^2,
  // and (no speculation) P_O^T g[off:] (+ pending Gram of O)
  // with the speculation the previous k_apply(OTHER) also wrote this probe's
  // mix column, its tail norm^2 and pivot: k_dots streams the fold chain only
  const bool mix_written = use_spec && op->c.spec_col;
  DotArgs<T> da;
  da.njobs = mix_written ? 1 : 2;
  da.n = n;
  da.ntiles = ntiles;
  da.rm = op->dn.rm;
  da.job[0].P = static_cast<const T*>(F.pan.P);
  da.job[0].K = F.pan.K;
  da.job[0].ncols = (int)F.pan.count;
  da.job[0].pend = F.pend;
  da.job[0].rhs = xs;
  da.job[0].check_finite = 1;
  da.job[1].P = static_cast<const T*>(O.pan.P);
  da.job[1].K = O.pan.K;
  da.job[1].ncols = use_spec ? 0 : (int)O.pan.count;
  da.job[1].pend = use_spec ? -1 : O.pend;
  da.job[1].rhs = g;
  da.job[1].wcol = static_cast<T*>(O.pan.P);
  da.job[1].wK = O.pan.K;
  da.job[1].wj = O.pan.count;
  da.job[1].pivot_out = op->scal + kScPivotG;
  da.job[1].pivot_row = off;
  da.trace = op->trace;
  // predecessor = previous probe's k_apply(OTHER) (writes y / x_{t+1} only)
  da.prefetch = 1;
  const double b1 = mix_written ? bytes_of(op, (double)n * (F.pan.count + (F.pend >= 0) + 1))
                                 : bytes_of(op, (double)n * (F.pan.count + da.job[1].ncols + (F.pend >= 0) +
                                                             (da.job[1].pend >= 0) + 2)) +
                                       (g.kind == kSrcInjected ? 8.0 * n : 0.0);
  const int grid = launch_dots<T>(op, s, da, b1);

  SmallArgs sa;
  sa.partials = op->partials;
  sa.nblk = grid;
  if (sharded(op)) {  // the new mix column's head rows and its pivot draw come from shard 0
    sa.partials = shard_exchange<T>(op, s, 0, op->partials, da.nslots, grid,
                                    {xcol(O.pan, O.pan.count), xvec(op->scal + kScPivotG, 1)});
    sa.nblk = 1;
  }
  sa.scal = op->scal;
  sa.status = op->status;
  sa.chA = F.dev;
  sa.chB = O.dev;
  sa.PA = F.pan.P;
  sa.PB = O.pan.P;
  sa.kA = (int)F.pan.count;
  sa.kB = (int)O.pan.count;
  sa.pendA = F.pend;
  sa.pendB = use_spec ? -1 : O.pend;
  sa.slotA_dot = da.job[0].slot_dot;
  sa.slotA_pend = da.job[0].slot_pend;
  sa.slotA_ss = da.job[0].slot_sumsq;
  sa.slotB_dot = mix_written ? 0 : da.job[1].slot_dot;
  sa.slotB_pend = mix_written ? 0 : da.job[1].slot_pend;
  sa.slotB_ss = mix_written ? -1 : da.job[1].slot_sumsq;
  sa.spec_ss = mix_written ? 1 : 0;
  sa.off = off;
  sa.rule = op->cfg.sign_rule;
  sa.beta1 = op->beta1;
  sa.beta3 = op->beta3;
  sa.head = op->head;
  sa.zbuf = op->zbuf;
  sa.csp = op->csp;
  sa.coefS = op->coefS;
  sa.is_haar = 1;
  sa.trace = op->trace;
  sa.mix_from_spec = use_spec ? 1 : 0;
  if (use_spec) {
    sa.spec_parts = sharded(op) ? op->xch[2] : op->partsO;
    sa.spec_nblk = spec_nblk;
    sa.spec_slot0 = spec_slot0;
    sa.spec_count = spec_count;
  }
  {
    LaunchScope ls(op, s, "small_dots", 0.0);
    sa.nslots_in = da.nslots;
    const size_t sm = small_smem_bytes(sa, 0, op->esz);
    allow_smem(k_small_dots<T, true>, sm);
    launch_k(op, k_small_dots<T, true>, dim3(1), dim3(kSmallThreads), sm, s, sa);
  }
  check_launch("k_small_dots");
  F.pend = -1;
  O.pend = -1;
  O.pan.count += 1;  // mix reflector appended (haar.hpp:63), Gram known

  // K2: p = D_F (x - P_F beta), new fold column, ||p[off:]||^2
  ApplyArgs<T> fa;
  fa.P = static_cast<const T*>(F.pan.P);
  fa.K = F.pan.K;
  fa.ncols = (int)F.pan.count;
  fa.beta = op->beta1;
  fa.n = n;
  fa.ntiles = ntiles;
  fa.rm = op->dn.rm;
  fa.D = F.dev.Drow;
  fa.Dtail = F.dev.Dtail;
  fa.Dlen = F.dev.Dlen;
  fa.x = xs;
  fa.Pw = static_cast<T*>(F.pan.P);
  fa.newj = F.pan.count;
  fa.off = off;
  fa.escale = op->scal + kScEscale;
  fa.head = op->head;
  fa.prefetch = 1;  // predecessor k_small_dots writes chain O's pivot, not P_F
  const int gridF = launch_apply<T, kApplyFold>(op, s, fa, true, bytes_of(op, (double)n * (F.pan.count + 2)), "fold");

  sa.partials = op->partsF;
  sa.nblk = gridF;
  if (sharded(op)) {  // the new fold column's head rows and p[0..off] come from shard 0
    sa.partials = shard_exchange<T>(op, s, 1, op->partsF, fa.nslots, gridF,
                                    {xcol(F.pan, F.pan.count), xvec(op->head, off + 1)});
    sa.nblk = 1;
  }
  sa.fold_slot_ss = fa.slot_ss;
  sa.kA = (int)F.pan.count;
  sa.kB = (int)O.pan.count;
  sa.append = append_fold ? 1 : 0;
  sa.spec_parts = nullptr;
  {
    LaunchScope ls(op, s, "small_fold", 0.0);
    const size_t sm = small_smem_bytes(sa, 1, op->esz);
    allow_smem(k_small_fold<T, true>, sm);
    launch_k(op, k_small_fold<T, true>, dim3(1), dim3(kSmallThreads), sm, s, sa);
  }
  check_launch("k_small_fold");
  if (append_fold) {
    F.pend = (int)F.pan.count;
    F.pan.count += 1;
  }

  // K3: y = D_O z - P_O beta (+ dynamics), and the speculative Gram dots of
  // P_O with the next probe's draw (rows >= off + 1)
  ApplyArgs<T> oa;
  oa.P = static_cast<const T*>(O.pan.P);
  oa.K = O.pan.K;
  oa.ncols = (int)O.pan.count;
  oa.beta = op->beta1;
  oa.n = n;
  oa.ntiles = ntiles;
  oa.rm = op->dn.rm;
  oa.D = O.dev.Drow;
  oa.Dtail = O.dev.Dtail;
  oa.Dlen = O.dev.Dlen;
  oa.z = op->zbuf;
  oa.zlen = off + 1;
  oa.epi = epi;
  oa.prefetch = 1;  // predecessor k_small_fold writes chain F's pivot, not P_O
  const bool next_ok = (op->c.t < op->n) &&
                       (op->cfg.draw_mode == HD_DRAWS_PHILOX || inj_avail(op) >= n);
  if (next_ok) {
    if (op->cfg.draw_mode != HD_DRAWS_PHILOX) {
      oa.spec.kind = kSrcInjected;
      oa.spec.inj = inj_at(op, op->c.inj_pos);
    } else {
      oa.spec.kind = kSrcPhilox;
      oa.spec.seedp = op->seed_dev;
      oa.spec.stream = (uint32_t)op->cfg.stream;
      oa.spec.probe = op->c.probe_index;
    }
    oa.spec.mask_begin = off + 1;
    // the next same-side probe's mix column goes to O[:, O.count] (when the
    // panel has room); if the next probe hits the other side, that column is
    // simply overwritten by its fold
    if (O.pan.count < O.pan.K) {
      oa.gcol = static_cast<T*>(O.pan.P);
      oa.gK = O.pan.K;
      oa.gj = O.pan.count;
      oa.gpivot = op->scal + kScPivotG;
      oa.gpivot_row = off + 1;
    }
  }
  double eb = (double)n * (O.pan.count + 1 + (next_ok ? 1 : 0));
  if (epi.kind == kEpiTanhMix) eb += (double)n * ((epi.xprev ? 1 : 0) + (epi.y ? 1 : 0));
  int gridO = launch_apply<T, kApplyOther>(op, s, oa, false, bytes_of(op, eb), "other");
  if (sharded(op)) {  // speculative dots and ||y||^2 summed over the shards (kept in xch[2])
    shard_exchange<T>(op, s, 2, op->partsO, oa.nslots, gridO, {});
    gridO = 1;
  }
  op->last_other_grid = gridO;
  op->last_other_slot_ss = oa.slot_ss;
  if (next_ok) {
    op->c.spec_chain = ochain;
    op->c.spec_probe = op->c.probe_index;
    op->c.spec_inj = (op->cfg.draw_mode != HD_DRAWS_PHILOX) ? op->c.inj_pos : -1;
    op->c.spec_count = (int)O.pan.count;
    op->c.spec_col = oa.gcol ? 1 : 0;
    op->c.spec_nblk = gridO;
    op->c.spec_slot0 = oa.slot_spec;
  }
}

// ------------------------------------------------------------- Ginibre
// ginibre.hpp:58-106. Right probe: fold chain R (dim n), store S = U (dim m),
// opposite chain L (dim m), opposite store V (dim n). Left probe mirrored.
template <typename T>
void enqueue_ginibre(hd_op* op, int side, const Src<T>& xsrc, const Epi<T>& epi, cudaStream_t s) {
  const bool right = (side == HD_RIGHT);
  const bool first = (op->c.r + op->c.l == 0);
  Chain& F = right ? op->R : op->L;       // fold chain (input dimension)
  Chain& O = right ? op->L : op->R;       // opposite chain (output dimension)
  Panel& S = right ? op->U : op->V;       // same-side store (output dim)
  Panel& Sopp = right ? op->V : op->U;    // opposite-side store (input dim)
  const int64_t nin = right ? op->n : op->m;
  const int64_t nout = right ? op->m : op->n;
  const ShardDim& din = right ? op->dn : op->dm;
  const ShardDim& dout = right ? op->dm : op->dn;
  const int64_t tin = din.own_tiles;
  const int64_t tout = dout.own_tiles;
  Src<T> xs = xsrc;
  xs.vbase = din.rm.vbase;
  int64_t& cnt = right ? op->c.r : op->c.l;
  const int64_t opp_cnt = right ? op->c.l : op->c.r;
  cnt += 1;
  const int64_t off = cnt - 1;
  const bool append_fold = !(op->cfg.skip_reflector && first);
  Src<T> g = draw_src<T>(op, nout);
  g.mask_begin = opp_cnt;  // ginibre.hpp:73 / :92
  g.D = O.dev.Drow;
  g.Dtail = O.dev.Dtail;
  g.Dlen = O.dev.Dlen;

  // K1 (input side): a = P_F^T x (+ pending), c = Sopp^T x
  DotArgs<T> da;
  da.njobs = 2;
  da.n = nin;
  da.ntiles = tin;
  da.rm = din.rm;
  da.job[0].P = static_cast<const T*>(F.pan.P);
  da.job[0].K = F.pan.K;
  da.job[0].ncols = (int)F.pan.count;
  da.job[0].pend = F.pend;
  da.job[0].rhs = xs;
  da.job[0].check_finite = 1;
  da.job[1].P = static_cast<const T*>(Sopp.P);
  da.job[1].K = Sopp.K;
  da.job[1].ncols = (int)Sopp.count;
  da.job[1].rhs = xs;
  const double b1 = bytes_of(op, (double)nin * (F.pan.count + Sopp.count + (F.pend >= 0) + 1));
  int grid = launch_dots<T>(op, s, da, b1);

  SmallArgs sa;
  sa.partials = op->partials;
  sa.nblk = grid;
  if (sharded(op)) {
    sa.partials = shard_exchange<T>(op, s, 0, op->partials, da.nslots, grid, {});
    sa.nblk = 1;
  }
  sa.scal = op->scal;
  sa.status = op->status;
  sa.chA = F.dev;
  sa.chB = O.dev;
  sa.PA = F.pan.P;
  sa.PB = O.pan.P;
  sa.kA = (int)F.pan.count;
  sa.kB = (int)Sopp.count;
  sa.pendA = F.pend;
  sa.pendB = -1;
  sa.slotA_dot = da.job[0].slot_dot;
  sa.slotA_pend = da.job[0].slot_pend;
  sa.slotA_ss = da.job[0].slot_sumsq;
  sa.slotB_dot = da.job[1].slot_dot;
  sa.slotB_ss = -1;
  sa.off = off;
  sa.rule = op->cfg.sign_rule;
  sa.beta1 = op->beta1;
  sa.beta3 = op->beta3;
  sa.head = op->head;
  sa.zbuf = op->zbuf;
  sa.csp = op->csp;
  sa.coefS = op->coefS;
  sa.is_haar = 0;
  {
    LaunchScope ls(op, s, "small_dots", 0.0);
    sa.nslots_in = da.nslots;
    const size_t sm = small_smem_bytes(sa, 0, op->esz);
    allow_smem(k_small_dots<T, false>, sm);
    launch_k(op, k_small_dots<T, false>, dim3(1), dim3(kSmallThreads), sm, s, sa);
  }
  check_launch("k_small_dots");
  F.pend = -1;

  // K2: p = D_F (x - P_F beta), new fold column, head p[0..off]
  ApplyArgs<T> fa;
  fa.P = static_cast<const T*>(F.pan.P);
  fa.K = F.pan.K;
  fa.ncols = (int)F.pan.count;
  fa.beta = op->beta1;
  fa.n = nin;
  fa.ntiles = tin;
  fa.rm = din.rm;
  fa.D = F.dev.Drow;
  fa.Dtail = F.dev.Dtail;
  fa.Dlen = F.dev.Dlen;
  fa.x = xs;
  fa.Pw = static_cast<T*>(F.pan.P);
  fa.newj = F.pan.count;
  fa.off = off;
  fa.escale = op->scal + kScEscale;
  fa.head = op->head;
  const int gridF = launch_apply<T, kApplyFold>(op, s, fa, true, bytes_of(op, (double)nin * (F.pan.count + 2)), "fold");
  sa.partials = op->partsF;
  sa.nblk = gridF;
  if (sharded(op)) {
    sa.partials = shard_exchange<T>(op, s, 1, op->partsF, fa.nslots, gridF,
                                    {xcol(F.pan, F.pan.count), xvec(op->head, off + 1)});
    sa.nblk = 1;
  }
  sa.fold_slot_ss = fa.slot_ss;
  sa.append = append_fold ? 1 : 0;
  {
    LaunchScope ls(op, s, "small_fold", 0.0);
    const size_t sm = small_smem_bytes(sa, 1, op->esz);
    allow_smem(k_small_fold<T, false>, sm);
    launch_k(op, k_small_fold<T, false>, dim3(1), dim3(kSmallThreads), sm, s, sa);
  }
  check_launch("k_small_fold");
  if (append_fold) {
    F.pend = (int)F.pan.count;
    F.pan.count += 1;
  }

  // K3 (output side): a_g = P_O^T (D_O g_m) (+ pending of O)
  DotArgs<T> db;
  db.njobs = 1;
  db.n = nout;
  db.ntiles = tout;
  db.rm = dout.rm;
  db.job[0].P = static_cast<const T*>(O.pan.P);
  db.job[0].K = O.pan.K;
  db.job[0].ncols = (int)O.pan.count;
  db.job[0].pend = O.pend;
  db.job[0].rhs = g;
  const double b3 = bytes_of(op, (double)nout * (O.pan.count + (O.pend >= 0))) +
                    (g.kind == kSrcInjected ? 8.0 * nout : 0.0);
  grid = launch_dots<T>(op, s, db, b3);

  SmallArgs sg = sa;
  sg.partials = op->partials;
  sg.nblk = grid;
  if (sharded(op)) {
    sg.partials = shard_exchange<T>(op, s, 0, op->partials, db.nslots, grid, {});
    sg.nblk = 1;
  }
  sg.chB = O.dev;
  sg.PB = O.pan.P;
  sg.kB = (int)O.pan.count;
  sg.pendB = O.pend;
  sg.slotB_dot = db.job[0].slot_dot;
  sg.slotB_pend = db.job[0].slot_pend;
  sg.csplen = Sopp.count;  // rows < opp count carry <v_i, x>
  sg.nS = (int)S.count;
  {
    LaunchScope ls(op, s, "small_gin", 0.0);
    sg.nslots_in = db.nslots;
    const size_t sm = small_smem_bytes(sg, 2, op->esz);
    allow_smem(k_small_gin<T>, sm);
    launch_k(op, k_small_gin<T>, dim3(1), dim3(kSmallThreads), sm, s, sg);
  }
  check_launch("k_small_gin");
  O.pend = -1;

  // K4: u = D_O g_m - P_O beta1 -> S[:, cnt-1];  y = sigma(S coef + c u + D_O c - P_O beta3)
  GinArgs<T> ga;
  ga.P = static_cast<const T*>(O.pan.P);
  ga.K = O.pan.K;
  ga.ncols = (int)O.pan.count;
  ga.beta1 = op->beta1;
  ga.beta3 = op->beta3;
  ga.S = static_cast<const T*>(S.P);
  ga.KS = S.K;
  ga.nS = (int)S.count;
  ga.coefS = op->coefS;
  ga.Sw = static_cast<T*>(S.P);
  ga.newj = S.count;
  ga.g = g;
  ga.csp = op->csp;
  ga.csplen = Sopp.count;
  ga.D = O.dev.Drow;
  ga.Dtail = O.dev.Dtail;
  ga.Dlen = O.dev.Dlen;
  ga.coef_cur = op->scal + kScCoefCur;
  ga.sigma = op->cfg.sigma;
  ga.n = nout;
  ga.rm = dout.rm;
  ga.status = op->status;
  ga.epi = epi;
  double eb = (double)nout * (O.pan.count + S.count + 2 + (g.kind == kSrcInjected ? 1 : 0));
  if (epi.yadd) eb += nout;
  {
    LaunchScope ls(op, s, "ginout", bytes_of(op, eb));
    const size_t smem = sizeof(double) * (2 * O.pan.K + std::max<int64_t>(S.K, 1));
    launch_k(op, k_ginout<T>, dim3((unsigned)tout), dim3(kUpdThreads), smem, s, ga);
  }
  check_launch("k_ginout");
  S.count += 1;
}

template <typename T>
void enqueue_probe(hd_op* op, int side, const Src<T>& xsrc, const Epi<T>& epi, cudaStream_t s) {
  if (op->ens == HD_HAAR) {
    enqueue_haar<T>(op, side, xsrc, epi, s);
  } else if (op->ens == HD_GINIBRE) {
    enqueue_ginibre<T>(op, side, xsrc, epi, s);
  } else {
    // GOE: y = (inner.right(x) + inner.left(x)) / sqrt(2)  (ensembles.hpp:117-127)
    Epi<T> e1;
    e1.kind = kEpiPlain;
    e1.y = static_cast<T*>(op->gtmp);
    e1.step = epi.step;
    enqueue_ginibre<T>(op, HD_RIGHT, xsrc, e1, s);
    Epi<T> e2 = epi;
    e2.yadd = static_cast<const T*>(op->gtmp);
    e2.add_scale = 0.7071067811865475244;
    enqueue_ginibre<T>(op, HD_LEFT, xsrc, e2, s);
  }
}

int64_t remaining(const hd_op* op) {
  if (op->ens == HD_HAAR) return op->n - op->c.t;
  if (op->ens == HD_GINIBRE) return std::min(op->m, op->n) - (op->c.r + op->c.l);
  return (std::min(op->m, op->n) - (op->c.r + op->c.l)) / 2;
}

const char* budget_msg(const hd_op* op) {
  if (op->ens == HD_HAAR) return "HaarOperator: probe budget n spent";
  if (op->ens == HD_GINIBRE) return "GinibreOperator: probe budget min(m, n) spent";
  return "GOEOperator: budget floor(n/2) spent";
}

int64_t inner_per_outer(const hd_op* op) { return op->ens == HD_GOE ? 2 : 1; }

void snapshot_chains(const hd_op* op, Counters& c) {
  c.rc_count = op->R.pan.count;
  c.lc_count = op->L.pan.count;
  c.u_count = op->U.count;
  c.v_count = op->V.count;
  c.rc_pend = op->R.pend;
  c.lc_pend = op->L.pend;
}

void restore(hd_op* op, const Counters& c) {
  op->c = c;
  op->R.pan.count = c.rc_count;
  op->L.pan.count = c.lc_count;
  op->U.count = c.u_count;
  op->V.count = c.v_count;
  op->R.pend = c.rc_pend;
  op->L.pend = c.lc_pend;
}

Counters take_snapshot(const hd_op* op) {
  Counters c = op->c;
  snapshot_chains(op, c);
  return c;
}

void reset_device_state(hd_op* op, cudaStream_t s) {
  {
    LaunchScope ls(op, s, "reset", 0.0);
    launch_k(op, k_reset_status, dim3(1), dim3(32), 0, s, op->status);
  }
  for (Chain* ch : {&op->R, &op->L}) {
    if (!ch->pan.P) continue;
    LaunchScope ls(op, s, "reset", 0.0);
    launch_k(op, k_reset_chain, dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(ch->dev.Dlen, 256), 1024))),
             dim3(256), 0, s, ch->dev);
  }
  check_launch("reset");
}

void hard_reset(hd_op* op) {
  op->c = Counters{};
  op->R.pan.count = op->L.pan.count = op->U.count = op->V.count = 0;
  op->R.pend = op->L.pend = -1;
  op->inj_size = 0;
  op->inj_base = 0;
  if (op->cfg.draw_mode == HD_DRAWS_REFERENCE)
    op->ref = std::make_unique<hd::refrng::Source>(op->cfg.seed, op->cfg.stream);
  reset_device_state(op, op->stream);
  ck(cudaStreamSynchronize(op->stream), "sync");
}

// Read status after a synchronous section; returns bad step (or 0).
void read_status(hd_op* op, int st[kStWords]) {
  ck(cudaMemcpy(st, op->status, sizeof(int) * kStWords, cudaMemcpyDeviceToHost), "status");
}

void clear_status(hd_op* op, cudaStream_t s) {
  launch_k(op, k_reset_status, dim3(1), dim3(32), 0, s, op->status);
  check_launch("reset status");
}

bool host_all_finite(const void* x, int64_t n, bool f32);

#include "hd_complex_host.inc"

bool host_all_finite(const void* x, int64_t n, bool f32) {
  if (f32) {
    const float* p = static_cast<const float*>(x);
    for (int64_t i = 0; i < n; ++i)
      if (!std::isfinite(p[i])) return false;
  } else {
    const double* p = static_cast<const double*>(x);
    for (int64_t i = 0; i < n; ++i)
      if (!std::isfinite(p[i])) return false;
  }
  return true;
}

// ================================================================= probe
template <typename T>
void do_probe(hd_op* op, const void* x, int64_t x_len, void* y, int64_t y_len, int side, int on_device,
              cudaStream_t s) {
  require(side == HD_RIGHT || side == HD_LEFT, "side must be 'right' or 'left'");
  const int eff_side = (op->ens == HD_GOE) ? HD_RIGHT : side;  // ensembles.hpp:118-119
  const int64_t rows = op->m, cols = op->n;
  // this shard's rows of x and y (all rows when unsharded)
  const int64_t want = (eff_side == HD_RIGHT) ? op->dn.vlen() : op->dm.vlen();
  const int64_t out_len = (eff_side == HD_RIGHT) ? op->dm.vlen() : op->dn.vlen();
  require(x_len == want, "probe: input dimension mismatch");
  require(y_len == out_len, "probe: output dimension mismatch");
  const bool budget_left = remaining(op) > 0;
  if (!on_device) require(host_all_finite(x, x_len, op->f32), "probe: non-finite input");
  if (!budget_left) {
    if (on_device) {
      std::vector<unsigned char> h((size_t)x_len * op->esz);
      ck(cudaMemcpy(h.data(), x, h.size(), cudaMemcpyDeviceToHost), "copy");
      require(host_all_finite(h.data(), x_len, op->f32), "probe: non-finite input");
    }
    throw HdError(HD_ERR_BUDGET_EXHAUSTED, budget_msg(op));
  }
  if (sharded(op)) {  // every pivot row must lie in the replicated head rows
    const int64_t next = (op->ens == HD_HAAR) ? op->c.t + 1
                         : (op->ens == HD_GOE) ? std::max(op->c.r, op->c.l) + 1
                                               : (eff_side == HD_RIGHT ? op->c.r : op->c.l) + 1;
    if (next > op->shard_cap)
      throw HdError(HD_ERR_RESOURCE_CAP, "hd: sharded operator capacity of " + std::to_string(op->shard_cap) +
                                             " probes per chain spent (hd_config.capacity)");
  }
  if (op->ens == HD_GOE) ensure_capacity(op, 1, 1);
  else ensure_capacity(op, eff_side == HD_RIGHT ? 1 : 0, eff_side == HD_LEFT ? 1 : 0);
  if (op->cfg.draw_mode == HD_DRAWS_REFERENCE) {
    // this probe's draws (GOE: inner right then inner left); Haar also queues
    // the next probe's draw so its Gram dots can be computed speculatively
    int64_t need = (op->ens == HD_GOE) ? 2 * op->n : (op->ens == HD_HAAR) ? op->n : (eff_side == HD_RIGHT ? rows : cols);
    if (op->ens == HD_HAAR && remaining(op) >= 2) need += op->n;
    ref_ensure(op, need);
  }
  const Counters snap = take_snapshot(op);
  // stage input (16 B aligned for vector loads)
  const void* xin = x;
  if (!on_device || (reinterpret_cast<uintptr_t>(x) % 16) != 0) {
    ck(cudaMemcpyAsync(op->xbuf, x, (size_t)x_len * op->esz, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       s),
       "copy x");
    xin = op->xbuf;
  }
  void* yout = (on_device && (reinterpret_cast<uintptr_t>(y) % 16) == 0) ? y : op->ybuf[0];
  clear_status(op, s);
  Epi<T> epi;
  epi.kind = kEpiPlain;
  epi.y = static_cast<T*>(yout);
  epi.step = 1;
  try {
    enqueue_probe<T>(op, eff_side, vec_src<T>(xin, nullptr), epi, s);
    // k_ginout's status flags (Haar's last kernel already exchanged them)
    if (sharded(op) && op->ens != HD_HAAR) shard_exchange<T>(op, s, 1, nullptr, 0, 0, {});
  } catch (...) {
    restore(op, snap);
    throw;
  }
  if (yout != y)
    ck(cudaMemcpyAsync(y, yout, (size_t)out_len * op->esz, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       s),
       "copy y");
  ck(cudaStreamSynchronize(s), "probe sync");
  if (op->trace) {
    unsigned long long h[16];
    ck(cudaMemcpy(h, op->trace, sizeof h, cudaMemcpyDeviceToHost), "trace");
    // [0] dots exit -> small start, [1] start -> after wait, [2] wait -> phase 1,
    // [3] phase 1 -> beta, [4] beta -> end
    const double cyc = 1.965;  // SM cycles per ns at max clock (stamps 5..11 are clock64)
    const double d[8] = {(double)h[0] - (double)h[8], (double)h[1] - (double)h[0], (double)h[2] - (double)h[1],
                         ((double)h[6] - (double)h[5]) / cyc, ((double)h[7] - (double)h[6]) / cyc,
                         ((double)h[9] - (double)h[7]) / cyc, ((double)h[10] - (double)h[9]) / cyc,
                         ((double)h[11] - (double)h[10]) / cyc};
    for (int i = 0; i < 8; ++i) op->trace_acc[i] += d[i];
    op->trace_n++;
    ck(cudaMemset(op->trace, 0, sizeof h), "trace reset");
  }
  int st[kStWords];
  read_status(op, st);
  if (st[kStBadInput]) {
    restore(op, snap);
    throw HdError(HD_ERR_INVALID_ARGUMENT, "probe: non-finite input");
  }
  if (st[kStAbort]) {
    restore(op, snap);
    throw HdError(HD_ERR_RUNTIME, "hd: probe aborted on device");
  }
}

// =============================================================== dynamics
int side_for(int rule, int64_t t) {
  if (rule == HD_SIDES_RIGHT) return HD_RIGHT;
  if (rule == HD_SIDES_LEFT) return HD_LEFT;
  return (t % 2 == 1) ? HD_RIGHT : HD_LEFT;
}

template <typename T>
__global__ void k_copy_scaled(const T* y, const double* scale, T* x, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = scale ? (T)(*scale * (double)y[i]) : y[i];
}

template <typename T>
struct RunPlan {
  // iterate x_t lives in buffer xb[t] (optionally times *xs[t])
  const void* xb = nullptr;
  const double* xs = nullptr;
};

template <typename T>
void enqueue_run(hd_op* op, const hd_run_args& a, int64_t dim_of_x1, cudaStream_t s, std::vector<Counters>* snaps,
                 void* traj_dev, bool reset_first) {
  if (reset_first) reset_device_state(op, s);
  const int64_t T_ = a.iterations;
  // buffers: xbuf holds x1 (and x0 in ybuf[2] for tanh mix); ybuf ping-pong
  const void* x_cur = op->xbuf;
  const double* x_scale = nullptr;
  const void* x_prev = (a.update == HD_UPDATE_TANH_MIX) ? op->ybuf[2] : nullptr;
  // tanh mix rotates three buffers: xbuf, ybuf[0], ybuf[1], ybuf[2]
  void* tri[4] = {op->xbuf, op->ybuf[0], op->ybuf[1], op->ybuf[2]};
  int idx_cur = 0, idx_prev = 3;
  for (int64_t t = 1; t <= T_; ++t) {
    const int side = side_for(a.side_rule, t);
    const int eff_side = (op->ens == HD_GOE) ? HD_RIGHT : side;
    const int64_t out_dim = (eff_side == HD_RIGHT) ? op->m : op->n;
    Epi<T> epi;
    epi.step = (int)std::min<int64_t>(t, INT_MAX - 1);
    void* out_buf = nullptr;
    if (a.update == HD_UPDATE_TANH_MIX) {
      int idx_next = 0;
      while (idx_next == idx_cur || idx_next == idx_prev) ++idx_next;
      epi.kind = kEpiTanhMix;
      epi.xprev = static_cast<const T*>(tri[idx_prev]);
      epi.xnext = static_cast<T*>(tri[idx_next]);
      enqueue_probe<T>(op, eff_side, vec_src<T>(tri[idx_cur], nullptr), epi, s);
      idx_prev = idx_cur;
      idx_cur = idx_next;
      x_cur = tri[idx_cur];
      x_scale = nullptr;
      out_buf = tri[idx_cur];
    } else {
      out_buf = op->ybuf[t % 2];
      epi.y = static_cast<T*>(out_buf);
      epi.kind = (a.update == HD_UPDATE_NORMALIZE) ? kEpiNormalize : kEpiPlain;
      epi.partials = op->partials2;
      enqueue_probe<T>(op, eff_side, vec_src<T>(x_cur, x_scale), epi, s);
      if (a.update == HD_UPDATE_NORMALIZE) {
        // ||y||^2 partials: k_apply(OTHER) slot (Haar) or per-tile (Ginibre/GOE)
        const double* parts = op->partials2;
        int64_t nblk = ((eff_side == HD_RIGHT) ? op->rows_pad_m : op->rows_pad_n) / kTile;
        if (op->ens == HD_HAAR) {
          parts = op->partsO + (size_t)op->last_other_slot_ss * op->last_other_grid;
          nblk = op->last_other_grid;
        }
        {
          LaunchScope ls(op, s, "small_norm", 0.0);
          launch_k(op, k_small_norm, dim3(1), dim3(kSmallThreads), 0, s, parts, (int)nblk, op->scal, op->status,
                   epi.step);
        }
        check_launch("k_small_norm");
        // the next probe reads y * inv lazily; keep a private copy of inv
        // per step so later steps cannot overwrite it before use
        x_scale = op->scal + kScInv;
      } else {
        x_scale = nullptr;
      }
      x_cur = out_buf;
    }
    if (traj_dev) {
      LaunchScope ls(op, s, "scale_copy", bytes_of(op, 2.0 * out_dim));
      k_copy_scaled<T><<<(unsigned)ceil_div(out_dim, 256), 256, 0, s>>>(
          static_cast<const T*>(x_cur), x_scale, static_cast<T*>(traj_dev) + (size_t)t * dim_of_x1, out_dim);
      check_launch("traj copy");
    }
    if (snaps) snaps->push_back(take_snapshot(op));
  }
  // materialise x_{T+1} into ybuf[2]... caller copies from (x_cur, x_scale)
  (void)x_prev;
  // final iterate into op->ybuf slot "final": reuse gtmp-free buffer xbuf? use k_copy to ybuf[... ]
  {
    const int64_t fdim = dim_of_x1;
    void* fin = (a.update == HD_UPDATE_TANH_MIX) ? nullptr : op->gtmp;
    if (fin && T_ > 0) {
      LaunchScope ls(op, s, "scale_copy", bytes_of(op, 2.0 * fdim));
      k_copy_scaled<T><<<(unsigned)ceil_div(fdim, 256), 256, 0, s>>>(static_cast<const T*>(x_cur), x_scale,
                                                                      static_cast<T*>(fin), fdim);
      check_launch("final copy");
    }
  }
}

// Where x_{T+1} lives after enqueue_run (device pointer).
template <typename T>
const void* final_location(hd_op* op, const hd_run_args& a) {
  if (a.iterations == 0) return op->xbuf;
  if (a.update == HD_UPDATE_TANH_MIX) {
    // replay the buffer rotation
    int idx_cur = 0, idx_prev = 3;
    for (int64_t t = 1; t <= a.iterations; ++t) {
      int idx_next = 0;
      while (idx_next == idx_cur || idx_next == idx_prev) ++idx_next;
      idx_prev = idx_cur;
      idx_cur = idx_next;
    }
    void* tri[4] = {op->xbuf, op->ybuf[0], op->ybuf[1], op->ybuf[2]};
    return tri[idx_cur];
  }
  return op->gtmp;
}

template <typename T>
void do_run_enqueue(hd_op* op, const hd_run_args& a) {
  cudaStream_t s = op->stream;
  require(!sharded(op), "hd_run: row-sharded operators are driven through hd_probe");
  require(!op->run_pending, "hd_run: the previous hd_run_async was not waited for");
  require(a.iterations >= 0, "run_dynamics: negative iteration count");
  require(a.update >= 0 && a.update <= 2, "run_dynamics: unknown update map");
  require(a.side_rule >= 0 && a.side_rule <= 2, "run_dynamics: unknown side schedule");
  require(a.x1 != nullptr, "run_dynamics: initial history must hold d + 1 vectors");
  require(a.iterations <= remaining(op), "run_dynamics: iteration count exceeds the operator's probe budget");
  // dimensions: x_1 is the input of probe 1
  const int side1 = side_for(a.side_rule, 1);
  const int eff1 = (op->ens == HD_GOE) ? HD_RIGHT : side1;
  const int64_t dim1 = (eff1 == HD_RIGHT) ? op->n : op->m;
  if (a.update == HD_UPDATE_TANH_MIX || a.traj)
    require(op->m == op->n, "run_dynamics: this update map needs a square operator");
  // x_1 finiteness (check_probe_input, operators.hpp:44-48) is checked by the
  // first k_dots pass on the device (kStBadInput -> "probe: non-finite input"),
  // so host inputs are not scanned here
  {
    int64_t nr = 0, nl = 0;
    for (int64_t t = 1; t <= a.iterations; ++t) {
      if (op->ens == HD_GOE) { ++nr; ++nl; }
      else if (side_for(a.side_rule, t) == HD_RIGHT) ++nr;
      else ++nl;
    }
    ensure_capacity(op, nr, nl);
    if (op->cfg.draw_mode == HD_DRAWS_REFERENCE)  // draws of every inner probe of the run
      ref_ensure(op, (op->ens == HD_HAAR) ? (nr + nl) * op->n : nr * op->m + nl * op->n);
  }
  fork_from(op, static_cast<cudaStream_t>(a.stream));
  const Counters snap0 = take_snapshot(op);
  const bool fresh = (op->c.r == 0 && op->c.l == 0 && op->c.t == 0 && op->R.pan.count == 0 && op->L.pan.count == 0);
  const size_t xbytes = (size_t)dim1 * op->esz;
  const cudaMemcpyKind k = a.on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  ck(cudaMemcpyAsync(op->xbuf, a.x1, xbytes, k, s), "copy x1");
  if (a.update == HD_UPDATE_TANH_MIX) {
    if (a.x0)
      ck(cudaMemcpyAsync(op->ybuf[2], a.x0, xbytes, k, s), "copy x0");
    else
      ck(cudaMemsetAsync(op->ybuf[2], 0, xbytes, s), "zero x0");
  }
  void* traj_dev = nullptr;
  if (a.traj) {
    if (a.on_device) {
      traj_dev = a.traj;
    } else {
      traj_dev = dmalloc<unsigned char>(xbytes * (size_t)(a.iterations + 1));
    }
    ck(cudaMemcpyAsync(traj_dev, a.x1, xbytes, k, s), "traj x1");
  }
  std::vector<Counters> snaps;
  snaps.push_back(snap0);
  const bool graphable = a.use_graph && fresh && op->cfg.draw_mode == HD_DRAWS_PHILOX && !op->prof && !a.traj;
  try {
    if (graphable) {
      char keybuf[160];
      std::snprintf(keybuf, sizeof keybuf, "%d/%d/%lld/%p", a.update, a.side_rule, (long long)a.iterations, (void*)s);
      const std::string key(keybuf);
      if (!op->graph || op->graph_key != key) {
        if (op->graph) {
          cudaGraphExecDestroy(op->graph);
          op->graph = nullptr;
        }
        cudaGraph_t gr;
        const int64_t before = op->launches;
        ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture begin");
        enqueue_run<T>(op, a, dim1, s, &snaps, nullptr, true);
        ck(cudaStreamEndCapture(s, &gr), "capture end");
        ck(cudaGraphInstantiate(&op->graph, gr, 0), "graph instantiate");
        cudaGraphDestroy(gr);
        op->graph_key = key;
        op->graph_launches = op->launches - before;
        op->graph_snaps = snaps;
        op->launches = before;
      } else {
        // the run starts from the fresh state, so it ends where the capture did
        snaps = op->graph_snaps;
        restore(op, snaps.back());
      }
      ck(cudaGraphLaunch(op->graph, s), "graph launch");
      op->launches += op->graph_launches;
    } else {
      if (fresh) reset_device_state(op, s);
      else clear_status(op, s);
      enqueue_run<T>(op, a, dim1, s, &snaps, traj_dev, false);
    }
  } catch (...) {
    restore(op, snap0);
    if (traj_dev && !a.on_device) cudaFree(traj_dev);
    throw;
  }
  const void* fin = final_location<T>(op, a);
  int64_t fdim = dim1;  // dimension of x_{T+1}
  if (a.iterations > 0) {
    const int sideT = side_for(a.side_rule, a.iterations);
    const int effT = (op->ens == HD_GOE) ? HD_RIGHT : sideT;
    fdim = (effT == HD_RIGHT) ? op->m : op->n;
  }
  if (a.final_out && a.on_device)
    ck(cudaMemcpyAsync(a.final_out, fin, (size_t)fdim * op->esz, cudaMemcpyDeviceToDevice, s), "copy final");
  op->run_pending = true;
  op->pend_args = a;
  op->pend_snaps = std::move(snaps);
  op->pend_fdim = fdim;
  op->pend_dim1 = dim1;
  op->pend_traj_dev = traj_dev;
  op->pend_stream = s;
}

// Completion of a run: status words, error restore (dynamics.hpp:64-67),
// host copies of x_{T+1} / the trajectory.
template <typename T>
void do_run_complete(hd_op* op) {
  require(op->run_pending, "hd_wait: no run in flight");
  op->run_pending = false;
  const hd_run_args a = op->pend_args;
  cudaStream_t s = op->pend_stream;
  void* traj_dev = op->pend_traj_dev;
  auto free_traj = [&] {
    if (traj_dev && !a.on_device) cudaFree(traj_dev);
  };
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    free_traj();
    ck(e, "run sync");
  }
  int st[kStWords];
  read_status(op, st);
  if (st[kStBadInput]) {
    restore(op, op->pend_snaps.front());
    free_traj();
    throw HdError(HD_ERR_INVALID_ARGUMENT, "probe: non-finite input");
  }
  if (st[kStBadStep] != INT_MAX) {
    const int64_t bad = st[kStBadStep];
    restore(op, op->pend_snaps[(size_t)std::min<int64_t>(bad, (int64_t)op->pend_snaps.size() - 1)]);
    free_traj();
    throw HdError(HD_ERR_RUNTIME, "run_dynamics: non-finite iterate at step " + std::to_string(bad));
  }
  if (a.final_out && !a.on_device)
    ck(cudaMemcpy(a.final_out, final_location<T>(op, a), (size_t)op->pend_fdim * op->esz, cudaMemcpyDeviceToHost),
       "copy final");
  if (a.traj && !a.on_device)
    ck(cudaMemcpy(a.traj, traj_dev, (size_t)op->pend_dim1 * op->esz * (size_t)(a.iterations + 1),
                  cudaMemcpyDeviceToHost),
       "copy traj");
  free_traj();
}

template <typename T>
void do_run(hd_op* op, const hd_run_args& a) {
  do_run_enqueue<T>(op, a);
  do_run_complete<T>(op);
}

// ------------------------------------------------- user callback dynamics
template <typename T>
void do_run_callback(hd_op* op, int64_t T_, int32_t depth, const void* const* initial, hd_side_fn side_of,
                     hd_update_fn update, void* user, void* final_out) {
  require(!sharded(op), "hd_run_callback: row-sharded operators are driven through hd_probe");
  require(T_ >= 0, "run_dynamics: negative iteration count");
  require(depth >= 0, "run_dynamics: negative history depth");
  require(initial != nullptr, "run_dynamics: initial history must hold d + 1 vectors");
  require(side_of != nullptr, "run_dynamics: no side schedule");
  require(update != nullptr, "run_dynamics: no update map");
  require(T_ <= remaining(op), "run_dynamics: iteration count exceeds the operator's probe budget");
  require(op->m == op->n || depth == 0, "run_dynamics: this update map needs a square operator");
  cudaStream_t s = op->stream;
  const int64_t dim = std::max(op->m, op->n);
  const size_t bytes = (size_t)dim * op->esz;
  std::vector<void*> hist(depth + 1);
  for (auto& h : hist) h = dmalloc<unsigned char>(std::max<size_t>(bytes, 16));
  void* ybuf = nullptr;
  void* nbuf = nullptr;
  ybuf = dmalloc<unsigned char>(std::max<size_t>(bytes, 16));
  nbuf = dmalloc<unsigned char>(std::max<size_t>(bytes, 16));
  auto cleanup = [&] {
    for (auto h : hist) cudaFree(h);
    cudaFree(ybuf);
    cudaFree(nbuf);
  };
  try {
    int64_t cur_dim = op->n;
    {
      const int s1 = side_of(user, 1);
      cur_dim = (op->ens == HD_GOE || s1 == HD_RIGHT) ? op->n : op->m;
    }
    for (int i = 0; i <= depth; ++i)
      ck(cudaMemcpyAsync(hist[i], initial[i], (size_t)cur_dim * op->esz, cudaMemcpyDeviceToDevice, s), "copy init");
    ensure_capacity(op, T_ * inner_per_outer(op), T_ * inner_per_outer(op));
    for (int64_t t = 1; t <= T_; ++t) {
      const int side = side_of(user, t);
      require(side == HD_RIGHT || side == HD_LEFT, "side must be 'right' or 'left'");
      const int eff = (op->ens == HD_GOE) ? HD_RIGHT : side;
      const int64_t in_dim = (eff == HD_RIGHT) ? op->n : op->m;
      const int64_t out_dim = (eff == HD_RIGHT) ? op->m : op->n;
      (void)in_dim;
      do_probe<T>(op, hist[0], in_dim, ybuf, out_dim, side, 1, s);
      const int rc = update(user, t, ybuf, hist.data(), depth, nbuf, out_dim, (void*)s);
      if (rc != 0) throw HdError(HD_ERR_RUNTIME, "run_dynamics: update callback failed at step " + std::to_string(t));
      ck(cudaStreamSynchronize(s), "sync");
      std::vector<unsigned char> h((size_t)out_dim * op->esz);
      ck(cudaMemcpy(h.data(), nbuf, h.size(), cudaMemcpyDeviceToHost), "check");
      if (!host_all_finite(h.data(), out_dim, op->f32))
        throw HdError(HD_ERR_RUNTIME, "run_dynamics: non-finite iterate at step " + std::to_string(t));
      void* oldest = hist.back();
      for (int i = depth; i > 0; --i) hist[i] = hist[i - 1];
      hist[0] = nbuf;
      nbuf = oldest;
      cur_dim = out_dim;
    }
    if (final_out) ck(cudaMemcpy(final_out, hist[0], (size_t)cur_dim * op->esz, cudaMemcpyDeviceToDevice), "final");
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

}  // namespace

// ================================================================= C-ABI
#define HD_TRY try {
#define HD_CATCH                          \
  }                                       \
  catch (const HdError& e) {              \
    g_err = e.what();                     \
    return e.code;                        \
  }                                       \
  catch (const std::invalid_argument& e) { \
    g_err = e.what();                     \
    return HD_ERR_INVALID_ARGUMENT;       \
  }                                       \
  catch (const std::exception& e) {       \
    g_err = e.what();                     \
    return HD_ERR_RUNTIME;                \
  }                                       \
  catch (...) {                           \
    g_err = "hd: unknown error";          \
    return HD_ERR_RUNTIME;                \
  }

extern "C" {

const char* hd_last_error(void) { return g_err.c_str(); }
const char* hd_version(void) { return "hd-b200 0.1.0 (sm_100a)"; }

int hd_create(const hd_config* cfg, hd_op** out) {
  HD_TRY
  require(cfg != nullptr && out != nullptr, "hd_create: null argument");
  const hd_config& c = *cfg;
  require(c.dtype == HD_F64 || c.dtype == HD_F32 || c.dtype == HD_C128,
          "hd_create: dtype must be HD_F64, HD_F32 or HD_C128");
  require(c.dtype != HD_C128 || c.exchange == nullptr, "hd_create: complex operators are not row-sharded");
  require(c.draw_mode == HD_DRAWS_PHILOX || c.draw_mode == HD_DRAWS_INJECTED || c.draw_mode == HD_DRAWS_REFERENCE,
          "hd_create: unknown draw mode");
  require(c.sign_rule >= 0 && c.sign_rule <= 2, "hd_create: unknown sign rule");
  int64_t m = c.m, n = c.n;
  if (c.ensemble == HD_GINIBRE) {
    require(m >= 1 && n >= 1, "GinibreOperator: dims must be positive");  // ginibre.hpp:40
    require(c.sigma > 0.0, "GinibreOperator: sigma must be positive");     // ginibre.hpp:41
  } else if (c.ensemble == HD_HAAR) {
    require(n >= 1, "HaarOperator: n must be positive");  // haar.hpp:30
    m = n;
  } else if (c.ensemble == HD_GOE) {
    require(n >= 1, "GinibreOperator: dims must be positive");
    require(c.sigma > 0.0, "GinibreOperator: sigma must be positive");
    m = n;
  } else {
    throw HdError(HD_ERR_INVALID_ARGUMENT, "hd_create: unknown ensemble");
  }
  ck(cudaSetDevice(c.device), "cudaSetDevice");
  auto op = std::make_unique<hd_op>();
  op->cfg = c;
  op->ens = c.ensemble;
  op->f32 = (c.dtype == HD_F32);
  op->esz = op->f32 ? 4 : 8;
  op->m = m;
  op->n = n;
  op->budget = (c.ensemble == HD_HAAR) ? n : std::min(m, n);
  if (c.shard_count > 1)
    require(c.exchange != nullptr, "hd_create: a sharded operator needs an exchange (hd_exchange_create_*)");
  if (c.exchange != nullptr) {
    require(c.shard_count >= 1, "hd_create: shard_count must be >= 1 with an exchange");
    require(c.shard_rank >= 0 && c.shard_rank < c.shard_count, "hd_create: shard_rank out of range");
    require(c.exchange->ex->size() == c.shard_count, "hd_create: exchange size differs from shard_count");
    require(c.capacity >= 1, "hd_create: a sharded operator needs capacity (max probes)");
    op->shard_count = c.shard_count;
    op->shard_rank = c.shard_rank;
    op->ex = c.exchange->ex.get();
  }
  if (const char* e = std::getenv("HD_NO_PDL")) op->pdl = !(e[0] == '1');
  if (const char* e = std::getenv("HD_SPARE_SMS"); e && e[0] != '\0') op->spare_sms = std::max(0, std::min(std::atoi(e), 64));
  if (const char* e = std::getenv("HD_WARPS"); e && e[0] != '\0') {
    op->max_warps = std::max(1, std::min(std::atoi(e), (int)kMaxWarps));
    op->warps_fixed = true;
  }
  if (const char* e = std::getenv("HD_TRACE")) {
    if (e[0] == '1') {
      op->trace = dmalloc<unsigned long long>(16);
      op->trace_acc.assign(16, 0.0);
    }
  }
  ck(cudaStreamCreateWithFlags(&op->stream, cudaStreamNonBlocking), "stream");
  ck(cudaEventCreateWithFlags(&op->ev_fork, cudaEventDisableTiming), "event");
  ck(cudaDeviceGetAttribute(&op->nsm, cudaDevAttrMultiProcessorCount, c.device), "attr");
  const int64_t per_outer = (c.ensemble == HD_GOE) ? 2 : 1;
  int64_t K;
  if (c.capacity > 0) {
    K = std::min((int64_t)(c.capacity * per_outer), op->budget);
  } else {
    K = std::min(op->budget, (int64_t)64);
  }
  K = std::max<int64_t>(K, 1);
  const int64_t Kside = (c.ensemble == HD_GOE) ? std::max<int64_t>(1, (K + 1) / 2) : K;
  if (sharded(op.get())) {
    op->shard_cap = Kside;
    op->head_rows = ceil_div(Kside + 1, kTile) * kTile;
  }
  plan_dim(op->dn, n, op->shard_count, op->shard_rank, op->head_rows);
  plan_dim(op->dm, m, op->shard_count, op->shard_rank, op->head_rows);
  op->rows_pad_n = op->dn.rows_pad;
  op->rows_pad_m = op->dm.rows_pad;
  if (c.dtype == HD_C128) {  // complex field: its own state (hd_complex_host.inc)
    op->scal = dmalloc<double>(kScWords);
    op->status = dmalloc<int>(kStWords);
    op->seed_dev = dmalloc<unsigned long long>(1);
    k_set_u64<<<1, 1, 0, op->stream>>>(op->seed_dev, (unsigned long long)c.seed);
    ck(cudaGetLastError(), "seed");
    cx_create(op.get(), K);
    hard_reset(op.get());
    *out = op.release();
    return HD_OK;
  }
  alloc_chain(op.get(), op->R, op->rows_pad_n, Kside);
  alloc_chain(op.get(), op->L, op->rows_pad_m, Kside);
  if (c.ensemble != HD_HAAR) {
    alloc_store(op.get(), op->U, op->rows_pad_m, Kside);
    alloc_store(op.get(), op->V, op->rows_pad_n, Kside);
  }
  ensure_small(op.get(), K + 1);
  op->scal = dmalloc<double>(kScWords);
  ck(cudaMemsetAsync(op->scal, 0, sizeof(double) * kScWords, op->stream), "memset");
  op->status = dmalloc<int>(kStWords);
  op->seed_dev = dmalloc<unsigned long long>(1);
  k_set_u64<<<1, 1, 0, op->stream>>>(op->seed_dev, (unsigned long long)c.seed);
  ck(cudaGetLastError(), "seed");
  const int64_t rp = std::max(op->rows_pad_m, op->rows_pad_n);
  op->io_len = rp;
  op->xbuf = dmalloc<unsigned char>((size_t)rp * op->esz);
  for (auto& b : op->ybuf) b = dmalloc<unsigned char>((size_t)rp * op->esz);
  op->gtmp = dmalloc<unsigned char>((size_t)rp * op->esz);
  op->partials2 = dmalloc<double>(rp / kTile + 8);
  ensure_capacity(op.get(), 0, 0);
  hard_reset(op.get());
  *out = op.release();
  return HD_OK;
  HD_CATCH
}

int hd_destroy(hd_op* op) {
  HD_TRY
  if (!op) return HD_OK;
  if (op->trace && op->trace_n > 0) {
    std::fprintf(stderr, "HD_TRACE k_small_dots over %lld probes (us):", (long long)op->trace_n);
    const char* nm[8] = {"dots_end->start", "start->wait", "wait->phase1end(gt)", "stageT_issue(clk)",
                         "rest_issue(clk)", "cp_async_wait(clk)", "sync(clk)", "reduce(clk)"};
    for (int i = 0; i < 8; ++i) std::fprintf(stderr, " %s %.2f", nm[i], op->trace_acc[i] / op->trace_n / 1e3);
    std::fprintf(stderr, "\n");
  }
  cudaSetDevice(op->cfg.device);
  cudaStreamSynchronize(op->stream);
  if (op->graph) cudaGraphExecDestroy(op->graph);
  free_chain(op->R);
  free_chain(op->L);
  cudaFree(op->U.P);
  cudaFree(op->V.P);
  for (FlushBufs* fb : {&op->fbD, &op->fbF, &op->fbO}) {
    cudaFree(fb->partials);
    cudaFree(fb->scratch);
    cudaFree(fb->counters);
  }
  for (double* p : {op->partials2, op->specbuf, op->red, op->scal, op->beta1, op->beta3, op->tmp, op->tmp2,
                    op->coefS, op->head, op->zbuf, op->csp, op->inj})
    cudaFree(p);
  cudaFree(op->status);
  cudaFree(op->seed_dev);
  cx_free(op->cx);
  for (double* b : op->xch) cudaFree(b);
  cudaFree(op->xbuf);
  for (auto b : op->ybuf) cudaFree(b);
  cudaFree(op->gtmp);
  for (auto& e : op->evq) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : op->evpool) cudaEventDestroy(e);
  if (op->ev_fork) cudaEventDestroy(op->ev_fork);
  cudaStreamDestroy(op->stream);
  delete op;
  return HD_OK;
  HD_CATCH
}

int hd_shape(const hd_op* op, int64_t* rows, int64_t* cols) {
  HD_TRY
  require(op && rows && cols, "hd_shape: null argument");
  *rows = op->m;
  *cols = op->n;
  return HD_OK;
  HD_CATCH
}

int hd_remaining(const hd_op* op, int64_t* r) {
  HD_TRY
  require(op && r, "hd_remaining: null argument");
  *r = remaining(op);
  return HD_OK;
  HD_CATCH
}

int hd_counts(const hd_op* op, int64_t* right, int64_t* left) {
  HD_TRY
  require(op && right && left, "hd_counts: null argument");
  if (op->ens == HD_HAAR) {
    *right = op->c.t;
    *left = 0;
  } else {
    *right = op->c.r;
    *left = op->c.l;
  }
  return HD_OK;
  HD_CATCH
}

int hd_chain_sizes(const hd_op* op, int64_t* rc, int64_t* lc) {
  HD_TRY
  require(op && rc && lc, "hd_chain_sizes: null argument");
  *rc = op->cx ? op->cx->R.count : op->R.pan.count;
  *lc = op->cx ? op->cx->L.count : op->L.pan.count;
  return HD_OK;
  HD_CATCH
}

int hd_probe(hd_op* op, const void* x, int64_t x_len, void* y, int64_t y_len, int32_t side, int32_t on_device,
             void* stream) {
  HD_TRY
  require(op && x && y, "hd_probe: null argument");
  cudaSetDevice(op->cfg.device);
  fork_from(op, static_cast<cudaStream_t>(stream));
  if (op->cx)
    cx_do_probe(op, x, x_len, y, y_len, side, on_device);
  else if (op->f32)
    do_probe<float>(op, x, x_len, y, y_len, side, on_device, op->stream);
  else
    do_probe<double>(op, x, x_len, y, y_len, side, on_device, op->stream);
  return HD_OK;
  HD_CATCH
}

int hd_push_draws(hd_op* op, const double* g, int64_t len, int32_t on_device) {
  HD_TRY
  require(op && g, "hd_push_draws: null argument");
  require(op->cfg.draw_mode == HD_DRAWS_INJECTED, "hd_push_draws: operator was not created with HD_DRAWS_INJECTED");
  require(len >= 1, "normal_vector: len must be >= 1");
  cudaSetDevice(op->cfg.device);
  // compact consumed prefix, then grow
  inj_append(op, g, len, on_device != 0);
  return HD_OK;
  HD_CATCH
}

int hd_reset(hd_op* op) {
  HD_TRY
  require(op, "hd_reset: null argument");
  cudaSetDevice(op->cfg.device);
  hard_reset(op);
  if (op->cx) cx_reset(op);
  return HD_OK;
  HD_CATCH
}

int hd_run(hd_op* op, const hd_run_args* args) {
  HD_TRY
  require(op && args, "hd_run: null argument");
  require(!op->cx, "hd_run: complex operators are driven through hd_probe");
  cudaSetDevice(op->cfg.device);
  if (op->f32)
    do_run<float>(op, *args);
  else
    do_run<double>(op, *args);
  return HD_OK;
  HD_CATCH
}

int hd_run_async(hd_op* op, const hd_run_args* args) {
  HD_TRY
  require(op && args, "hd_run_async: null argument");
  require(!op->cx, "hd_run_async: complex operators are driven through hd_probe");
  cudaSetDevice(op->cfg.device);
  if (op->f32)
    do_run_enqueue<float>(op, *args);
  else
    do_run_enqueue<double>(op, *args);
  return HD_OK;
  HD_CATCH
}

int hd_wait(hd_op* op) {
  HD_TRY
  require(op, "hd_wait: null argument");
  cudaSetDevice(op->cfg.device);
  if (op->f32)
    do_run_complete<float>(op);
  else
    do_run_complete<double>(op);
  return HD_OK;
  HD_CATCH
}

int hd_exchange_create_local(int32_t nshards, hd_exchange** out) {
  HD_TRY
  require(out != nullptr && nshards >= 1, "hd_exchange_create_local: need nshards >= 1");
  *out = new hd_exchange{std::make_unique<hd::LocalExchange>(nshards)};
  return HD_OK;
  HD_CATCH
}

int hd_exchange_nccl_id(void* id_out) {
  HD_TRY
  require(id_out != nullptr, "hd_exchange_nccl_id: null argument");
  try {
    hd::NcclExchange::unique_id(id_out);
  } catch (const std::runtime_error& e) {
    throw HdError(HD_ERR_NCCL, e.what());
  }
  return HD_OK;
  HD_CATCH
}

int hd_exchange_create_nccl(const void* id, int32_t nranks, int32_t rank, int32_t device, hd_exchange** out) {
  HD_TRY
  require(id && out && nranks >= 1 && rank >= 0 && rank < nranks, "hd_exchange_create_nccl: bad arguments");
  try {
    *out = new hd_exchange{std::make_unique<hd::NcclExchange>(id, nranks, rank, device)};
  } catch (const std::runtime_error& e) {
    throw HdError(HD_ERR_NCCL, e.what());
  }
  return HD_OK;
  HD_CATCH
}

int hd_exchange_destroy(hd_exchange* ex) {
  delete ex;
  return HD_OK;
}

int hd_shard_plan(int64_t N, int32_t count, int32_t rank, int64_t head_rows, int64_t* begin, int64_t* end) {
  HD_TRY
  require(begin && end, "hd_shard_plan: null argument");
  try {
    hd::shard_plan(N, count, rank, head_rows, begin, end);
  } catch (const std::invalid_argument& e) {
    throw HdError(HD_ERR_INVALID_ARGUMENT, e.what());
  }
  return HD_OK;
  HD_CATCH
}

int hd_shard_range(const hd_op* op, int32_t dim, int64_t* begin, int64_t* end) {
  HD_TRY
  require(op && begin && end, "hd_shard_range: null argument");
  require(dim == 0 || dim == 1, "hd_shard_range: dim must be 0 (cols, n) or 1 (rows, m)");
  const ShardDim& d = dim == 0 ? op->dn : op->dm;
  *begin = d.lo;
  *end = d.hi;
  return HD_OK;
  HD_CATCH
}

struct hd_rs {
  hd::refrng::Source src;
};

int hd_rs_create(uint64_t seed, uint64_t stream, hd_rs** out) {
  HD_TRY
  require(out != nullptr, "hd_rs_create: null argument");
  *out = new hd_rs{hd::refrng::Source(seed, stream)};
  return HD_OK;
  HD_CATCH
}

void hd_rs_destroy(hd_rs* rs) { delete rs; }
uint64_t hd_rs_next_u64(hd_rs* rs) { return rs->src.next(); }
double hd_rs_uniform(hd_rs* rs) { return rs->src.uniform(); }
double hd_rs_normal(hd_rs* rs) { return rs->src.normal(); }

int hd_rs_normal_vector(hd_rs* rs, int64_t len, double* out) {
  HD_TRY
  require(rs && out, "hd_rs_normal_vector: null argument");
  require(len >= 1, "normal_vector: len must be >= 1");
  rs->src.normal_fill(out, len);
  return HD_OK;
  HD_CATCH
}

int hd_rs_bernoulli_gaussian(hd_rs* rs, int64_t n, double rho, double sigma_s, double* out) {
  HD_TRY
  require(rs && out, "hd_rs_bernoulli_gaussian: null argument");
  require(n >= 1, "sample_bernoulli_gaussian: n must be positive");  // experiments.cpp:21-23
  require(rho >= 0.0 && rho <= 1.0, "sample_bernoulli_gaussian: rho in [0,1]");
  require(sigma_s > 0.0, "sample_bernoulli_gaussian: sigma_s must be positive");
  rs->src.bernoulli_gaussian(out, n, rho, sigma_s);
  return HD_OK;
  HD_CATCH
}

uint64_t hd_derive_seed(uint64_t base, uint64_t index) { return hd::refrng::derive_seed(base, index); }

int hd_reseed(hd_op* op, uint64_t seed) {
  HD_TRY
  require(op, "hd_reseed: null argument");
  require(!op->cx, "hd_reseed: complex operators are driven through hd_probe");
  require(!op->run_pending, "hd_reseed: a run is in flight (hd_wait first)");
  require(op->cfg.draw_mode != HD_DRAWS_INJECTED, "hd_reseed: injected-draw operators take their draws from the caller");
  cudaSetDevice(op->cfg.device);
  if (op->cfg.draw_mode == HD_DRAWS_REFERENCE) {  // host generator: a synchronous fresh start
    op->cfg.seed = seed;
    hard_reset(op);
    return HD_OK;
  }
  // fresh state without a host sync: counters on the host, device words and
  // D tables by kernels on the handle's stream (graph replays reset too)
  op->cfg.seed = seed;
  op->c = Counters{};
  op->R.pan.count = op->L.pan.count = op->U.count = op->V.count = 0;
  op->R.pend = op->L.pend = -1;
  k_set_u64<<<1, 1, 0, op->stream>>>(op->seed_dev, (unsigned long long)seed);
  ck(cudaGetLastError(), "seed");
  reset_device_state(op, op->stream);
  return HD_OK;
  HD_CATCH
}

int hd_run_callback(hd_op* op, int64_t iterations, int32_t depth, const void* const* initial_dev, hd_side_fn side_of,
                    hd_update_fn update, void* user, void* final_out_dev) {
  HD_TRY
  require(op, "hd_run_callback: null argument");
  require(!op->cx, "hd_run_callback: complex operators are driven through hd_probe");
  cudaSetDevice(op->cfg.device);
  if (op->f32)
    do_run_callback<float>(op, iterations, depth, initial_dev, side_of, update, user, final_out_dev);
  else
    do_run_callback<double>(op, iterations, depth, initial_dev, side_of, update, user, final_out_dev);
  return HD_OK;
  HD_CATCH
}

int hd_reflector_apply(const double* p, int64_t n, int64_t offset, double zero_tol, int32_t sign_rule,
                       const double* x, double* y, int64_t count, int32_t on_device, double* info) {
  HD_TRY
  // validation order of make_reflector (reflect.hpp:124-127)
  require(p != nullptr && n >= 1, "make_reflector: empty vector");
  require(offset >= 0 && offset < n, "make_reflector: offset out of range");
  require(sign_rule >= 0 && sign_rule <= 2, "make_reflector: unknown sign rule");
  require(count >= 0 && (count == 0 || (x && y)), "Reflector::apply: dimension mismatch");
  const size_t pb = sizeof(double) * (size_t)n, xb = pb * (size_t)count;
  std::vector<double> hp;
  if (!on_device) {
    require(host_all_finite(p, n, false), "make_reflector: non-finite entries");
  } else {
    hp.resize((size_t)n);
    ck(cudaMemcpy(hp.data(), p, pb, cudaMemcpyDeviceToHost), "copy p");
    require(host_all_finite(hp.data(), n, false), "make_reflector: non-finite entries");
  }
  double *dp = nullptr, *dx = nullptr, *dy = nullptr, *di = nullptr;
  ck(cudaMalloc(&dp, pb), "alloc");
  ck(cudaMalloc(&di, 4 * sizeof(double)), "alloc");
  if (count > 0) {
    ck(cudaMalloc(&dx, xb), "alloc");
    ck(cudaMalloc(&dy, xb), "alloc");
  }
  const cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  ck(cudaMemcpy(dp, p, pb, k), "copy p");
  if (count > 0) ck(cudaMemcpy(dx, x, xb, k), "copy x");
  k_reflector<<<1, kReflThreads>>>(dp, n, offset, zero_tol, sign_rule, dx, dy, count, di);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess && count > 0) ck(cudaMemcpy(y, dy, xb, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost), "copy y");
  if (e == cudaSuccess && info) ck(cudaMemcpy(info, di, 3 * sizeof(double), cudaMemcpyDeviceToHost), "copy info");
  cudaFree(dp);
  cudaFree(di);
  cudaFree(dx);
  cudaFree(dy);
  ck(e, "k_reflector");
  return HD_OK;
  HD_CATCH
}

int hd_set_profiling(hd_op* op, int32_t enabled) {
  HD_TRY
  require(op, "hd_set_profiling: null argument");
  drain_events(op);
  op->prof = enabled != 0;
  return HD_OK;
  HD_CATCH
}

int hd_get_stats(hd_op* op, hd_kernel_stats* out, int32_t max, int32_t* count) {
  HD_TRY
  require(op && count, "hd_get_stats: null argument");
  drain_events(op);
  int32_t i = 0;
  for (auto& kv : op->stats) {
    if (out && i < max) {
      std::memset(out[i].name, 0, sizeof(out[i].name));
      std::strncpy(out[i].name, kv.first.c_str(), sizeof(out[i].name) - 1);
      out[i].launches = kv.second.launches;
      out[i].ms = kv.second.ms;
      out[i].alg_bytes = kv.second.bytes;
    }
    ++i;
  }
  *count = i;
  return HD_OK;
  HD_CATCH
}

int hd_reset_stats(hd_op* op) {
  HD_TRY
  require(op, "hd_reset_stats: null argument");
  drain_events(op);
  op->stats.clear();
  return HD_OK;
  HD_CATCH
}

int hd_launch_count(const hd_op* op, int64_t* count) {
  HD_TRY
  require(op && count, "hd_launch_count: null argument");
  *count = op->launches;
  return HD_OK;
  HD_CATCH
}

}  // extern "C"
