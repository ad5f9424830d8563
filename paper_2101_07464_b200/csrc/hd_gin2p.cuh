// Two-pass Ginibre / GOE probes: every panel is streamed
// ONCE per probe, and each pass does a GEMV-N and a GEMV-T over the same
// bytes.
//
// Per probe (ginibre.hpp:58-106; F = the probed side's chain, O = the other
// chain, S = the same-side basis store):
//   pass A (k_nt<FOLD>) over F:  N: p = D_F (x - W_F beta1) -> new column
//       p[off:] 2^-e, head p[0..off], ||p[off:]||^2;
//     T: W_F^T w_new (the new reflector's Gram column, rows > off; the pivot
//       row is added by the stage) and W_F^T g' for the NEXT probe's draw g'
//       (it lands on this chain when the next probe is on the other side:
//       the dots k_dots would otherwise stream F again for).
//   pass B (k_nt<GIN>) over O and S:  N: u = D_O g - W_O beta1 -> S's new
//       column, y = sigma (S coef + c u + D_O c - W_O beta3) -> update map;
//     T: O^T x_{t+1} and S^T x_{t+1} — the next probe's K1 dots (its F is
//       this O, its opposite store this S) — with x_{t+1} the update map's
//       output row (or, for the GOE inner right probe, the step's input x).
// The GEMV-T needs the GEMV-N's result row by row, so the panel cannot be a
// 256-row tile per warp streamed in column chunks as in k_dots/k_apply: a
// CTA stages a row SUB-TILE of all columns of the pass's panels in shared
// memory (3-D TMA box {Rs rows, columns, 1 tile} of the tile-major panel,
// SASS UTMALDG), runs the GEMV-N (thread = row, column groups), the epilogue
// (thread = row), then the GEMV-T (thread = column, rows rotated by lane:
// conflict-free) from the same shared bytes. A producer warp keeps the stage
// ring full (mbarrier full/empty pairs); consumer warps never wait on HBM
// while a stage is ready. Partial column sums stay in registers across the
// CTA's contiguous sub-tile range and leave through the deterministic group
// flush (flush_row), in the slot layouts the single-CTA stages read.
#pragma once

#include <cuda.h>

#include "hd_kernels.cuh"

#ifndef HD_NT_TRACE
#define HD_NT_TRACE 0  // 1: HD_TRACE=3 per-slot cycle counters in k_nt (A/B builds only)
#endif

namespace hd {

#ifndef HD_NT_CONSUMERS
#define HD_NT_CONSUMERS 352  // consumer threads of a k_nt CTA (A/B builds: 480)
#endif
constexpr int kNtConsumers = HD_NT_CONSUMERS;       // consumer warps: 1-2 epilogue, the rest workers
constexpr int kNtThreads = kNtConsumers + 32;       // + 1 producer warp
constexpr int kNtMaxMaps = 4;
constexpr int kNtMaxVecs = 5;
constexpr int kNtMaxStages = 16;
constexpr int kNtMaxCols = 512;                     // columns of an output pass
constexpr int kNtMaxFoldCols = 288;                 // columns of a fold pass
constexpr int kNtBarId = 1;                         // named barrier of the consumer warps

enum NtMode : int { kNtFold = 0, kNtGin = 1 };
// Compile-time output-pass epilogue (the map and where the T phase's
// right-hand side comes from): one kernel instance per kind, no runtime
// branching on the map in the row-serial epilogue.
enum NtEpi : int {
  kEkPlain = 0,  // plain / normalize map, T rhs = y
  kEkSrc = 1,    // plain map, T rhs = a given vector (GOE inner right: the step's x)
  kEkTanh = 2,
  kEkAmpInit = 3,
  kEkAmpX = 4,
  kEkAmpZ = 5,
  kEkSpike = 6,
};
enum NtRhs : int { kRhsEpi = 0, kRhsSrc = 1 };

// One 3-D TMA box family: panel `panel`, stage columns [scol, scol + cols),
// panel columns [pcol, pcol + cols).
struct NtMapInfo {
  int scol = 0, pcol = 0, cols = 0;
};

template <typename T>
struct NtArgs {
  CUtensorMap maps[kNtMaxMaps];  // __grid_constant__ parameter space (64-B aligned)
  NtMapInfo mi[kNtMaxMaps];
  int nmaps = 0;
  int rs = 32;        // rows per sub-tile (16..256, divides 256)
  int nst = 2;        // stages
  int C = 0;          // columns of the pass (stage layout [C][rs])
  int kP0 = 0;        // columns of panel 0 (F or O); panel 1 (S) = C - kP0
  int64_t n = 0;      // rows of the dimension (global)
  int64_t nsub = 0;   // sub-tiles of this shard's rows
  RowMap rm;
  // vectors bulk-copied per sub-tile (rs elements each; 8 B slots): x / g_inj /
  // yadd / state / aux / xprev, by role index below
  const void* vec[kNtMaxVecs] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  int vesz[kNtMaxVecs] = {0, 0, 0, 0, 0};
  int nvec = 0;
  int64_t stage_bytes = 0;  // per stage
  int64_t tx_bytes = 0;     // TMA bytes per stage (boxes + vectors)
  // N-phase coefficients: fold beta1 (F); gin beta1, beta3 (O), coefS (S)
  const double* beta1 = nullptr;
  const double* beta3 = nullptr;
  const double* coefS = nullptr;
  // D of the panel's chain (fold: F; gin: O)
  const double* D = nullptr;
  const double* Dtail = nullptr;
  int64_t Dlen = 0;
  // ---- fold
  int vx = -1;                      // vector role: x (dtype T)
  const double* xscale = nullptr;   // x * scale (lazily normalised iterate)
  T* Pw = nullptr;                  // panel F (new column newj)
  int64_t K = 0, newj = 0, off = 0;
  const double* escale = nullptr;
  double* head = nullptr;
  Src<T> spec;                      // next probe's draw (kSrcPhilox / kSrcInjected via vinj2) or none
  int vspec = -1;                   // vector role of injected spec draws
  // ---- gin
  Src<T> g;                         // this probe's draw (mask, D of O)
  int vg = -1;                      // vector role of injected draws
  T* Sw = nullptr;                  // store S (new column newjS)
  int64_t KS = 0, newjS = 0;
  const double* csp = nullptr;
  int64_t csplen = 0;
  const double* coef_cur = nullptr;
  double sigma = 1.0;
  Epi<T> epi;
  int vyadd = -1, vstate = -1, vaux = -1, vxprev = -1;
  int rhs_mode = kRhsEpi;           // T-phase right-hand side: epilogue output or the Src below
  int vrhs = -1;                    // vector role of that Src (dtype T, times rhs_scale)
  const double* rhs_scale = nullptr;
  int do_t = 1;                     // run the T phase at all
  // ---- output slots
  int slot_t0 = 0;    // T-phase column sums of RHS 0: columns [0, kP0) at slot_t0 + c, columns >= kP0 at slot_t1 + c - kP0
  int slot_t1 = 0;
  int slot_t2 = -1;   // fold: RHS 1 (spec draw) column sums at slot_t2 + c
  int slot_r0 = -1, slot_r1 = -1, slot_r2 = -1, slot_r3 = -1, slot_r4 = -1;  // scalar reductions
  int nslots = 0;
  Flush out;
  int* status = nullptr;
  int prefetch = 0;
  int evict = 0;      // L2 policy of the panel boxes (nt_l2_policy)
  int sched = 1;      // slot schedule (k_nt_impl): 0 T of j - 1 in slot j, 1 T of j in slot j
  int deal = 0;       // sub-tile order (k_nt_impl: 0 round robin, 1 by tile)
  unsigned long long* trace = nullptr;  // HD_TRACE=3: [8][grid] cycle counters
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// L2 policy of the panel boxes: evict_first (panel bytes are read once per
// pass) or evict_normal (NtArgs::evict, HD_NT_EVICT A/B knob)
__device__ __forceinline__ uint64_t nt_l2_policy(int evict) {
  uint64_t pol;
  if (evict == 0)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// mbarrier wait that backs off between probes: the producer warp waits for
// stages to drain most of the time and must not steal issue slots from the
// consumer warps of its SM partition.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  while (!done) {
    __nanosleep(64);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// mbarrier wait that suspends the thread (suspend-time hint) instead of
// spinning: the producer warp waits for a stage to drain most of the time.
__device__ __forceinline__ void mbar_wait_suspend(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITS_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

template <typename T>
__device__ __forceinline__ double ld_vec(const unsigned char* slot, int esz, int r) {
  if (esz == 8) return reinterpret_cast<const double*>(slot)[r];
  return (double)reinterpret_cast<const float*>(slot)[r];
}

// Warp roles of a k_nt CTA (kNtThreads = 9 warps):
//   warps [0, E)      epilogue warps: one sub-tile row per thread (rs <= 32 E)
//   warps [E, 11)     workers: GEMV-N of sub-tile j + 1 and GEMV-T of j - 1
//   warp 11           producer: the TMA ring
// In "slot" j the epilogue warps finish sub-tile j while the workers run the
// N phase of j + 1 and the T phase of j - 1 — one barrier per slot, so the
// row-serial epilogue is off the critical path.
__host__ __device__ constexpr int nt_ewarps(int rs) { return rs <= 32 ? 1 : 2; }
__host__ __device__ constexpr int nt_workers(int rs) { return kNtConsumers - 32 * nt_ewarps(rs); }
// Column capacity of a pass with sub-tiles of rs rows (the stage-size rule
// keeps C * rs * 8 B near 56 KB): the per-thread register arrays below are
// sized from it, and nt_shape takes a shorter sub-tile for a wider pass.
__host__ __device__ constexpr int nt_max_cols(int mode, int rs) {
  return (mode == kNtFold && 8192 / rs > kNtMaxFoldCols) ? kNtMaxFoldCols : 8192 / rs;
}
// N-phase column groups (workers per row pair) and the columns one worker
// thread owns at most; T-phase columns per round (8 lanes each) and rounds
__host__ __device__ constexpr int nt_ngroups(int rs) { return nt_workers(rs) / ((rs > 64 ? 64 : rs) / 2); }
__host__ __device__ constexpr int nt_ncols(int mode, int rs) {
  return (nt_max_cols(mode, rs) + nt_ngroups(rs) - 1) / nt_ngroups(rs);
}
__host__ __device__ constexpr int nt_trounds(int mode, int rs) {
  return (nt_max_cols(mode, rs) + nt_workers(rs) / 8 - 1) / (nt_workers(rs) / 8);
}


// Shared-memory carve-up (sized per launch): [stages][stage_bytes] | N-phase
// partials [2][1 or 2][NP][rs] | rhs [2][2][rs] | barriers. The T-phase
// partials, the scalar partials and the slot row reuse the stages at the end.
struct NtSmem {
  unsigned char* stages;
  double* red;
  double* rhs;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* rdy;  // [2] rhs of sub-tile j ready (sched 1)
};

__host__ __device__ inline size_t nt_fixed_doubles(int mode, int C, int kP0, int rs) {
  (void)kP0;
  (void)C;
  const size_t np_rs = (size_t)(nt_workers(rs) / 32) * rs;  // NP partials x rs rows per array
  return 2 * (mode == kNtGin ? 2 : 1) * np_rs + 4 * (size_t)rs;
}

__host__ __device__ inline size_t nt_fixed_bytes(int mode, int C, int kP0, int rs, int nst) {
  return sizeof(double) * nt_fixed_doubles(mode, C, kP0, rs) + (2 * (size_t)nst + 2) * sizeof(uint64_t) + 128;
}

// Bytes of the stage ring the final flush reuses: T partials [WT][6], scalar
// partials [4][kNtConsumers], the slot row.
__host__ __device__ inline size_t nt_flush_bytes(int nslots) {
  return sizeof(double) * (4 * (size_t)kNtConsumers + (size_t)nslots + 8);
}

__device__ __forceinline__ NtSmem nt_smem(unsigned char* base, int mode, int C, int kP0, int rs, int nst,
                                          int64_t stage_bytes) {
  NtSmem m;
  m.stages = base;
  double* p = reinterpret_cast<double*>(base + (size_t)nst * stage_bytes);
  (void)kP0;
  (void)C;
  const int np_rs = (nt_workers(rs) / 32) * rs;
  m.red = p; p += 2 * (mode == kNtGin ? 2 : 1) * np_rs;
  m.rhs = p; p += 4 * rs;
  m.full = reinterpret_cast<uint64_t*>(p);
  m.empty = m.full + nst;
  m.rdy = m.empty + nst;
  return m;
}

template <typename T, int MODE, int RS, int EK>
__device__ __forceinline__ void k_nt_impl(const NtArgs<T>& a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const NtSmem m = nt_smem(smem, MODE, a.C, a.kP0, a.rs, a.nst, a.stage_bytes);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const bool producer = (w == kNtConsumers / 32);
  constexpr int rs = RS;
  const int C = a.C, nst = a.nst;
  // sub-tiles taller than 64 rows (narrow passes: the per-slot costs spread
  // over more bytes) run as NB blocks of RB = 64 rows through the same thread
  // mappings; the blocks of a slot are independent (instruction-level overlap)
  constexpr int RB = (RS > 64) ? 64 : RS, NB = RS / RB;
  constexpr int E = (RB <= 32) ? 1 : 2, WT = kNtConsumers - 32 * E;
  const bool epi_thr = !producer && tid < 32 * E;
  const bool worker = !producer && !epi_thr;
  const int wt = tid - 32 * E;  // worker index
  // sub-tiles dealt round robin: at any moment the CTAs stream neighbouring
  // sub-tiles, so each column's contiguous 2 KB tile segment is read by
  // neighbouring CTAs close together in time (DRAM row-buffer locality)
  // deal 0: sub-tile s = blockIdx.x + k gridDim.x; deal 1: whole tiles dealt
  // round robin, a CTA streams the 256 / RS sub-tiles of its tile in order
  constexpr int SPT = kTile / RS;
  const int64_t ntl = a.nsub / SPT;
  const int64_t nk = (a.deal == 0)
                         ? ((a.nsub > (int64_t)blockIdx.x) ? (a.nsub - blockIdx.x + gridDim.x - 1) / gridDim.x : 0)
                         : ((ntl > (int64_t)blockIdx.x) ? (ntl - blockIdx.x + gridDim.x - 1) / gridDim.x : 0) * SPT;
  if (tid == 0) {
    for (int q = 0; q < nst; ++q) {
      mbar_init(m.full + q, 1);
      mbar_init(m.empty + q, 1);
    }
    mbar_init(m.rdy, E);
    mbar_init(m.rdy + 1, E);
    mbar_fence_init();
  }
  __syncthreads();
  const size_t vec_off = (size_t)C * rs * sizeof(T);  // vector slots after the panel columns (8 B each)
  auto row_of = [&](int64_t k) {
    const int64_t sidx = (a.deal == 0) ? (int64_t)blockIdx.x + k * gridDim.x
                                       : ((int64_t)blockIdx.x + (k / SPT) * gridDim.x) * SPT + (k % SPT);
    return a.rm.tile0 * kTile + sidx * rs;
  };
  const uint64_t l2pol = nt_l2_policy(a.evict);
  auto issue = [&](int64_t k, int q) {  // producer lane 0: sub-tile k into stage q
    unsigned char* st = m.stages + (size_t)q * a.stage_bytes;
    const int64_t li = row_of(k);  // local panel row
    const int tile = (int)(li >> kTileShift), rin = (int)(li & (kTile - 1));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(m.full + q, (uint32_t)a.tx_bytes);
    for (int b = 0; b < a.nmaps; ++b)
      tma_load_3d(st + (size_t)a.mi[b].scol * rs * sizeof(T), &a.maps[b], rin, a.mi[b].pcol, tile, m.full + q, l2pol);
    const int64_t vi = li + a.rm.gdelta - a.rm.vbase;  // vector index of the sub-tile's first row
    for (int v = 0; v < a.nvec; ++v)
      bulk_g2s(st + vec_off + (size_t)v * rs * 8, static_cast<const unsigned char*>(a.vec[v]) + vi * a.vesz[v],
               (uint32_t)(rs * a.vesz[v]), m.full + q);
  };
  int64_t prefetched = 0;
  if (producer && lane == 0) {
    for (int b = 0; b < a.nmaps; ++b) prefetch_map(&a.maps[b]);
    if (a.prefetch)
      for (; prefetched < nk && prefetched < nst; ++prefetched) issue(prefetched, (int)prefetched);
  }
  pdl_wait();
  pdl_launch();
  __shared__ int s_abort;
  if (tid == 0) s_abort = aborted(a.status) ? 1 : 0;
  __syncthreads();
  const bool abort_all = s_abort != 0;
  if (producer && lane == 0) {
    int64_t k = prefetched;
    int q = (int)(k % nst);
    uint32_t ph = (uint32_t)((k / nst) & 1);  // phase of the empty barrier to wait for: use (k / nst) - 1
    if (!abort_all) {
      for (; k < nk; ++k) {
        if (k >= nst) mbar_wait_suspend(m.empty + q, ph ^ 1u);
        issue(k, q);
        if (++q == nst) {
          q = 0;
          ph ^= 1u;
        }
      }
    } else {
      for (int64_t j = 0; j < prefetched; ++j) mbar_wait(m.full + j, 0);  // drain what was prefetched
    }
  }
  // ------------------------------------------------------------ consumers
  const int kP0 = a.kP0;
  // worker T-phase mapping: 8 consecutive lanes share a column (lane g of the
  // 8 takes row pairs g, g + 8, ... of the sub-tile: 128 contiguous bytes per
  // quarter warp, conflict-free, and each right-hand-side pair is loaded once
  // for all of the thread's columns); the thread's columns are
  // cb + r NCOL, r < R (NCOL = WT / 8 columns per round)
  constexpr int NCOL = WT / 8;
  const int cb = wt >> 3, tg8 = wt & 7;
  const int Rt = (C > cb) ? (C - cb + NCOL - 1) / NCOL : 0;  // this thread's column rounds
  const bool t_active = worker && C > 0 && a.do_t;
  constexpr int RMAX = nt_trounds(MODE, RS);
  double tA[RMAX], tB[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    tA[r] = 0.0;
    tB[r] = 0.0;
  }
  // worker N-phase mapping: row pair nrp, column group ncg (CG groups) of
  // contiguous columns [cga, cgb)
  constexpr int RP = RB / 2;
  constexpr int CG = WT / RP;
  const int nrp = wt % RP, ncg = wt / RP;
  constexpr int NP = (RP >= 32) ? CG : WT / 32;         // N-phase partials per row
  const int npart = (RP >= 32) ? ncg : (wt >> 5);         // this thread's partial index
  const int cga = (int)((int64_t)C * ncg / CG), cgb = (int)((int64_t)C * (ncg + 1) / CG);
  const int kc = cgb - cga;  // <= KN
  constexpr int KN = nt_ncols(MODE, RS);
  // the thread's N-phase coefficients, in registers for the whole launch:
  // n1 = W beta1 (O or F columns), nm = S coefS - W_O beta3 (output pass: one
  // sum over both panels: O columns (beta1, -beta3), S columns (0, coefS))
  double cfa[KN], cfb[KN];
#pragma unroll
  for (int r = 0; r < KN; ++r) {
    const int c = cga + r;
    cfa[r] = 0.0;
    cfb[r] = 0.0;
    if (worker && r < kc) {
      if (MODE == kNtGin) {
        if (c < kP0) {
          cfa[r] = a.beta1[c];
          cfb[r] = -a.beta3[c];
        } else {
          cfb[r] = a.coefS[c - kP0];
        }
      } else {
        cfa[r] = a.beta1[c];
      }
    }
  }
  constexpr int nred = (MODE == kNtGin) ? 2 : 1;
  const int red_stride = NP * RS;  // one partial array: NP x rs doubles
  // epilogue scalar accumulators
  double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
  bool bad = false;
  const double dtail = (a.Dtail != nullptr) ? *a.Dtail : 1.0;
  double escale = 1.0, xsc = 1.0, rsc = 1.0, cc = 0.0, esc = 0.0;
  if (MODE == kNtFold) {
    escale = *a.escale;
    if (a.xscale) xsc = *a.xscale;
  } else {
    cc = *a.coef_cur;
    if (a.rhs_scale) rsc = *a.rhs_scale;
    if (a.epi.sc) esc = *a.epi.sc;
  }
  auto stage_ptr = [&](int q) { return m.stages + (size_t)q * a.stage_bytes; };
  // ---- N phase of sub-tile k (stage q): workers -> red[k & 1]
  auto nphase = [&](int64_t k, int q, uint32_t ph) {
    mbar_wait(m.full + q, ph);
    const T* sp = reinterpret_cast<const T*>(stage_ptr(q)) + 2 * nrp;
    double2 n1[NB], nm[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      n1[b] = make_double2(0.0, 0.0);
      nm[b] = make_double2(0.0, 0.0);
    }
    const T* sc0 = sp + cga * RS;
#pragma unroll
    for (int r = 0; r < KN; ++r) {  // one 2-row load per column and block, coefficients in registers
      if (r < kc) {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const double2 v = lds_pair(sc0 + r * RS + b * RB);
          n1[b].x = fma(v.x, cfa[r], n1[b].x);
          n1[b].y = fma(v.y, cfa[r], n1[b].y);
          if (MODE == kNtGin) {
            nm[b].x = fma(v.x, cfb[r], nm[b].x);
            nm[b].y = fma(v.y, cfb[r], nm[b].y);
          }
        }
      }
    }
    // the column groups of one warp (lanes with the same row pair) add up in
    // a fixed shuffle tree, so the epilogue sums only NP = WT / 32 partials
    // per row (RB <= 32; RB = 64: one column group per warp, NP = CG)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
#pragma unroll
      for (int sh = RP; sh < 32; sh <<= 1) {
        n1[b].x += __shfl_xor_sync(0xffffffffu, n1[b].x, sh);
        n1[b].y += __shfl_xor_sync(0xffffffffu, n1[b].y, sh);
        if (MODE == kNtGin) {
          nm[b].x += __shfl_xor_sync(0xffffffffu, nm[b].x, sh);
          nm[b].y += __shfl_xor_sync(0xffffffffu, nm[b].y, sh);
        }
      }
      if (RP >= 32 || lane < RP) {
        double* red = m.red + (k & 1) * nred * red_stride + npart * RS + b * RB + 2 * nrp;  // [partial][rs]
        *reinterpret_cast<double2*>(red) = n1[b];
        if (MODE == kNtGin) *reinterpret_cast<double2*>(red + red_stride) = nm[b];
      }
    }
  };
  // ---- epilogue of sub-tile k (stage q): epilogue threads, one row each -> rhs[k & 1]
  unsigned long long epi_tr[2] = {0, 0};  // HD_TRACE=3: epilogue reduction / whole
  auto epilogue = [&](int64_t k, int q, uint32_t ph) {
    // LPR lanes per row add the NP column-group partials in fixed order (four
    // chains each), then combine with a shuffle; lane et < RB runs row et of
    // each of the NB blocks
    constexpr int LPR = (RB >= 32) ? 1 : 32 / RB;
    const int et0 = tid % RB, half = tid / RB;
    if (tid >= RB * LPR) return;
    const bool etr = HD_NT_TRACE && a.trace && tid == 0;
    const long long ec0 = etr ? clock64() : 0;
    const double* red = m.red + (k & 1) * nred * red_stride;
#pragma unroll
    for (int blk = 0; blk < NB; ++blk) {
    const int et = et0 + blk * RB;
    double r1 = 0.0, rm = 0.0;
    {
      constexpr int per = (NP + LPR - 1) / LPR;
      const int g0 = half * per;
      double a1[4] = {0.0, 0.0, 0.0, 0.0}, am[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int jg = 0; jg < per; ++jg) {  // compile-time chain index jg & 3
        const int g = g0 + jg;
        if (g < NP) {
          a1[jg & 3] += red[g * RS + et];
          if (MODE == kNtGin) am[jg & 3] += red[red_stride + g * RS + et];
        }
      }
      r1 = (a1[0] + a1[1]) + (a1[2] + a1[3]);
      rm = (am[0] + am[1]) + (am[2] + am[3]);
      if (LPR > 1) {
        for (int sh = RB; sh < 32; sh <<= 1) {
          r1 += __shfl_xor_sync(0xffffffffu, r1, sh);
          if (MODE == kNtGin) rm += __shfl_xor_sync(0xffffffffu, rm, sh);
        }
      }
    }
    if (LPR > 1 && half != 0) continue;  // (NB == 1 when LPR > 1)
    if (etr) epi_tr[0] += clock64() - ec0;
    const unsigned char* vs = stage_ptr(q) + vec_off;
    double* rb = m.rhs + (k & 1) * 2 * rs;
    if (blk == 0) mbar_wait(m.full + q, ph);  // complete (the workers waited for it a slot ago): orders the vector reads
    const int64_t li = row_of(k) + et;
    const int64_t i = li + a.rm.gdelta;
    const double d = (i < a.Dlen) ? a.D[i] : dtail;
    if (MODE == kNtFold) {
      const double xv = ld_vec<T>(vs + (size_t)a.vx * rs * 8, sizeof(T), et) * xsc;
      const double p = (i < a.n) ? d * (xv - r1) : 0.0;
      const double cv = (i >= a.off) ? p : 0.0;
      const double wv = cv * escale;
      a.Pw[paddr(li, a.newj, a.K)] = (T)wv;
      if (i <= a.off) a.head[i] = p;
      e0 += cv * cv;  // ||p[off:]||^2
      const double g_rhs0 = (i > a.off) ? (double)(T)wv : 0.0;  // Gram RHS (the stored values)
      double g_rhs1 = 0.0;
      if (a.spec.kind != kSrcNone && i < a.n && i >= a.spec.mask_begin) {
        // device draws: pre-generated vector (k_draw_fill); injected: parity mode only
        g_rhs1 = (a.spec.kind == kSrcPhilox) ? ld_vec<T>(vs + (size_t)a.vspec * RS * 8, 8, et) : a.spec.inj[i];
        if constexpr (sizeof(T) == 4) g_rhs1 = (double)(float)g_rhs1;
      }
      e1 += g_rhs0 * g_rhs1;  // new column . next draw
      rb[et] = g_rhs0;
      rb[rs + et] = g_rhs1;
    } else {
      double gv = 0.0;
      if (i < a.n && i >= a.g.mask_begin) {
        gv = (a.g.kind == kSrcPhilox) ? ld_vec<T>(vs + (size_t)a.vg * RS * 8, 8, et) : a.g.inj[i];
        if constexpr (sizeof(T) == 4) gv = (double)(float)gv;
        gv *= d;
      }
      const double u = (i < a.n) ? gv - r1 : 0.0;
      a.Sw[paddr(li, a.newjS, a.KS)] = (T)u;
      const double uu = (double)(T)u;
      const double cs = (i < a.csplen) ? d * a.csp[i] : 0.0;
      double y = a.sigma * (rm + cc * u + cs);  // rm = S coefS - W_O beta3
      const Epi<T>& e = a.epi;
      const int64_t vi = i - a.rm.vbase;
      double out = 0.0;
      constexpr int kind = (EK == kEkAmpInit) ? kEpiAmpInit : (EK == kEkAmpX) ? kEpiAmpX
                           : (EK == kEkAmpZ) ? kEpiAmpZ : (EK == kEkSpike) ? kEpiSpike : kEpiPlain;
      if (i < a.n) {
        if (e.yadd) y = (ld_vec<T>(vs + (size_t)a.vyadd * RS * 8, sizeof(T), et) + y) * e.add_scale;
        if constexpr (EK >= kEkAmpInit) {
          const double stv = (EK != kEkAmpInit) ? ld_vec<T>(vs + (size_t)a.vstate * RS * 8, sizeof(T), et) : 0.0;
          const double axv = ld_vec<T>(vs + (size_t)a.vaux * RS * 8, sizeof(T), et);
          double q0, q1;
          const double o = epi_row(kind, y, stv, axv, esc, q0, q1);
          if (EK != kEkSpike) e.state[vi] = (T)o;
          if (EK == kEkAmpInit || EK == kEkSpike) y = o;
          out = (double)(T)o;
          e2 += q0;
          e3 += q1;
          bad |= !isfinite(o);
        } else if constexpr (EK == kEkTanh) {
          double xp = e.xprev ? ld_vec<T>(vs + (size_t)a.vxprev * RS * 8, sizeof(T), et) : 0.0;
          if (e.xprev_scale) xp *= *e.xprev_scale;
          const double o = tanh(2.0 * y) + 0.1 * xp;
          e.xnext[vi] = (T)o;
          out = (double)(T)o;
          bad |= !isfinite(o);
        } else {
          out = (double)(T)y;
          bad |= !isfinite(y);
          e2 += y * y;  // normalize: ||y||^2 (also the plain map's)
        }
        if (e.y) e.y[vi] = (T)y;
      }
      double rhs = out;
      if constexpr (EK == kEkSrc) rhs = (i < a.n) ? ld_vec<T>(vs + (size_t)a.vrhs * RS * 8, sizeof(T), et) * rsc : 0.0;
      e0 += rhs * rhs;  // ||x_{t+1}||^2 (the next probe's K1 sum of squares)
      e1 += uu * rhs;   // new S column . x_{t+1}
      rb[et] = rhs;
    }
    }  // blocks
    if (etr) epi_tr[1] += clock64() - ec0;
  };
  // ---- T phase of sub-tile k (stage q): workers (mapping above)
  auto tphase = [&](int64_t k, int q) {
    if (!t_active) return;
    constexpr int PPL = RP / 8;  // row pairs per lane per column and block
#pragma unroll 1
    for (int blk = 0; blk < NB; ++blk) {
    const double* r0 = m.rhs + (k & 1) * 2 * RS + blk * RB + 2 * tg8;
    double2 x[PPL], z[PPL];
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
      x[u] = *reinterpret_cast<const double2*>(r0 + 16 * u);
      z[u] = make_double2(0.0, 0.0);
      if (MODE == kNtFold) z[u] = *reinterpret_cast<const double2*>(r0 + RS + 16 * u);
    }
    const T* pr = reinterpret_cast<const T*>(stage_ptr(q)) + cb * RS + blk * RB + 2 * tg8;
    // the thread's column rounds, unrolled to the smallest of 4 / 8 / RMAX
    // that covers them (the accumulators need compile-time indices)
#define HD_NT_TROUNDS(RM)                                                         \
  _Pragma("unroll") for (int r = 0; r < (RM); ++r) {                              \
    if (r < Rt) {                                                                 \
      _Pragma("unroll") for (int u = 0; u < PPL; ++u) {                           \
        const double2 v = lds_pair(pr + 16 * u);                                  \
        tA[r] = fma(v.y, x[u].y, fma(v.x, x[u].x, tA[r]));                        \
        if (MODE == kNtFold) tB[r] = fma(v.y, z[u].y, fma(v.x, z[u].x, tB[r]));   \
      }                                                                           \
    }                                                                             \
    pr += NCOL * RS;                                                              \
  }
    if (Rt <= 4) {
      HD_NT_TROUNDS(4)
    } else if (Rt <= 8) {
      HD_NT_TROUNDS(8)
    } else {
      HD_NT_TROUNDS(RMAX)
    }
    }  // blocks
#undef HD_NT_TROUNDS
  };
  // ---- the slot loop (see the warp roles above): one named barrier per slot;
  // each role runs its own loop (32-bit counters, stage indices advanced
  // without divisions)
  if (!producer && !abort_all && nk > 0) {
    const int nki = (int)nk;
    // HD_TRACE=3: per-CTA cycle breakdown (epilogue thread 0, worker 0)
    unsigned long long tr[6] = {0, 0, 0, 0, 0, 0};
    const bool trace = HD_NT_TRACE && a.trace && (tid == 0 || wt == 0);
    if (a.sched == 1 && worker) {
      // slot j: N of j + 1, then (once the epilogue warps publish it) the T
      // phase of j from its rhs: a stage is held for two slots, not three
      nphase(0, 0, 0);
      int qN = (nst > 1) ? 1 : 0, qT = 0;  // stages of N (j + 1) and T (j)
      uint32_t phN = (nst > 1) ? 0u : 1u;
      named_sync(kNtBarId, kNtConsumers);
      for (int j = 0; j < nki; ++j) {
        const long long c0t = trace ? clock64() : 0;
        long long c2t = c0t;
        if (j + 1 < nki) {
          if (trace) {
            mbar_wait(m.full + qN, phN);
            c2t = clock64();
          }
          nphase(j + 1, qN, phN);
        }
        const long long c3t = trace ? clock64() : 0;
        mbar_wait(m.rdy + (j & 1), (uint32_t)(j >> 1) & 1u);
        tphase(j, qT);
        if (++qT == nst) qT = 0;
        const long long c4t = trace ? clock64() : 0;
        named_sync(kNtBarId, kNtConsumers);  // red of j + 1 ready; stage of j free
        if (trace) {
          tr[3] += c2t - c0t;
          tr[4] += c3t - c2t;
          tr[5] += c4t - c3t;
          tr[1] += clock64() - c4t;
        }
        if (++qN == nst) {
          qN = 0;
          phN ^= 1u;
        }
      }
    } else if (a.sched == 1) {  // epilogue warps; thread 0 frees the stages
      named_sync(kNtBarId, kNtConsumers);
      int qE = 0;
      uint32_t phE = 0;
      for (int j = 0; j < nki; ++j) {
        const long long c0t = trace ? clock64() : 0;
        epilogue(j, qE, phE);
        __syncwarp();
        if (lane == 0) mbar_arrive(m.rdy + (j & 1));
        const long long c4t = trace ? clock64() : 0;
        named_sync(kNtBarId, kNtConsumers);
        if (trace) {
          tr[0] += c4t - c0t;
          tr[1] += clock64() - c4t;
        }
        if (tid == 0) mbar_arrive(m.empty + qE);
        if (++qE == nst) {
          qE = 0;
          phE ^= 1u;
        }
      }
    } else if (worker) {
      nphase(0, 0, 0);
      int qN = (nst > 1) ? 1 : 0, qT = 0;  // stages of N (j + 1) and T (j - 1)
      uint32_t phN = (nst > 1) ? 0u : 1u;
      named_sync(kNtBarId, kNtConsumers);
      for (int j = 0; j <= nki; ++j) {
        const long long c0t = trace ? clock64() : 0;
        long long c2t = c0t;
        if (j + 1 < nki) {
          if (trace) {
            mbar_wait(m.full + qN, phN);
            c2t = clock64();
          }
          nphase(j + 1, qN, phN);
        }
        const long long c3t = trace ? clock64() : 0;
        if (j >= 1) {
          tphase(j - 1, qT);
          if (++qT == nst) qT = 0;
        }
        const long long c4t = trace ? clock64() : 0;
        named_sync(kNtBarId, kNtConsumers);  // red of j + 1, rhs of j ready; stage of j - 1 free
        if (trace) {
          tr[3] += c2t - c0t;          // waiting for the stage
          tr[4] += c3t - c2t;          // N phase
          tr[5] += c4t - c3t;          // T phase
          tr[1] += clock64() - c4t;    // workers at the barrier
        }
        if (++qN == nst) {
          qN = 0;
          phN ^= 1u;
        }
      }
    } else {  // epilogue warps; thread 0 frees the stages
      named_sync(kNtBarId, kNtConsumers);
      int qE = 0, qT = 0;  // stages of the epilogue (j) and of T (j - 1)
      uint32_t phE = 0;
      for (int j = 0; j <= nki; ++j) {
        const long long c0t = trace ? clock64() : 0;
        if (j < nki) epilogue(j, qE, phE);
        const long long c4t = trace ? clock64() : 0;
        named_sync(kNtBarId, kNtConsumers);
        if (trace) {
          tr[0] += c4t - c0t;          // epilogue
          tr[1] += clock64() - c4t;    // epilogue warp at the barrier
        }
        if (j >= 1) {
          if (tid == 0) mbar_arrive(m.empty + qT);
          if (++qT == nst) qT = 0;
        }
        if (++qE == nst) {
          qE = 0;
          phE ^= 1u;
        }
      }
    }
    if (trace) {
      if (tid == 0) {
        a.trace[0 * gridDim.x + blockIdx.x] += tr[0];
        a.trace[1 * gridDim.x + blockIdx.x] += tr[1];
        a.trace[8 * gridDim.x + blockIdx.x] += epi_tr[0];
        a.trace[9 * gridDim.x + blockIdx.x] += epi_tr[1];
        a.trace[7 * gridDim.x + blockIdx.x] += (unsigned long long)nk;
      } else {
        a.trace[6 * gridDim.x + blockIdx.x] += tr[1];
        a.trace[3 * gridDim.x + blockIdx.x] += tr[3];
        a.trace[4 * gridDim.x + blockIdx.x] += tr[4];
        a.trace[5 * gridDim.x + blockIdx.x] += tr[5];
      }
    }
  }
  // ---- partial sums -> slot row (fixed order) -> group flush; the stages
  // are free now: [T partials: 6 x 256][scalar partials: 4 x 256][slot row]
  __syncthreads();
  double* sc = reinterpret_cast<double*>(m.stages);
  double* acc = sc + 4 * kNtConsumers;
  if (!producer) {
    sc[tid] = e0;
    sc[kNtConsumers + tid] = e1;
    sc[2 * kNtConsumers + tid] = e2;
    sc[3 * kNtConsumers + tid] = e3;
  }
  for (int sl = tid; sl < a.nslots; sl += kNtThreads) acc[sl] = 0.0;
  __syncthreads();
  if (worker && C > 0 && a.do_t) {  // each column's 8 lanes add up (fixed shuffle tree), lane g = 0 stores
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      double va = tA[r], vb = tB[r];
      va += __shfl_xor_sync(0xffffffffu, va, 1);
      va += __shfl_xor_sync(0xffffffffu, va, 2);
      va += __shfl_xor_sync(0xffffffffu, va, 4);
      if (MODE == kNtFold) {
        vb += __shfl_xor_sync(0xffffffffu, vb, 1);
        vb += __shfl_xor_sync(0xffffffffu, vb, 2);
        vb += __shfl_xor_sync(0xffffffffu, vb, 4);
      }
      const int c = cb + r * NCOL;
      if (tg8 == 0 && r < Rt && c < C) {
        acc[(c < kP0) ? a.slot_t0 + c : a.slot_t1 + (c - kP0)] = va;
        if (MODE == kNtFold && a.slot_t2 >= 0) acc[a.slot_t2 + c] = vb;
      }
    }
  }
  if (tid < 4) {  // scalar reductions of the epilogue threads, fixed order
    const int slot = tid == 0 ? a.slot_r0 : tid == 1 ? a.slot_r1 : tid == 2 ? a.slot_r2 : a.slot_r3;
    if (slot >= 0) {
      double v = 0.0;
      for (int t = 0; t < RB; ++t) v += sc[tid * kNtConsumers + t];
      acc[slot] = v;
    }
  }
  if (bad && MODE == kNtGin) {
    atomicMin(a.status + kStBadStep, a.epi.step);
    atomicOr(a.status + kStAbort, 1);
  }
  flush_row(acc, a.nslots, a.out);
}

// The device draw of one probe (Philox4x32-10 + Box-Muller, the stream every
// streaming kernel regenerates: philox_normal_pair) written once for rows
// [0, rows) of a (local) dimension, global row = local row + gdelta; the two
// passes that need it read it as a bulk-copied vector instead of each
// regenerating the fp64 transcendentals inside their streams.
struct DrawArgs {
  const unsigned long long* seedp = nullptr;
  uint32_t stream = 0, probe = 0;
  int64_t rows = 0, gdelta = 0;
  double* out = nullptr;
  // nprobe > 1: the draws of probes probe .. probe + nprobe - 1 in one launch (small
  // operators keep a block of future draws: hd_gin2p_host.inc), `rows` apart in out
  int nprobe = 1;
};

__device__ __forceinline__ void k_draw_fill_impl(const DrawArgs& a) {
  pdl_wait();
  pdl_launch();
  const uint64_t seed = *a.seedp;
  const int64_t half = a.rows / 2;  // rows is a multiple of the tile height
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < half * a.nprobe; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pi = (a.nprobe > 1) ? w / half : 0;
    const int64_t q = w - pi * half;
    const int64_t i = 2 * q + a.gdelta;  // gdelta is even (tile-aligned)
    const double2 v = philox_normal_pair(seed, a.stream, a.probe + (uint32_t)pi, (uint64_t)(i >> 1));
    *reinterpret_cast<double2*>(a.out + pi * a.rows + 2 * q) = v;
  }
}
__global__ void __launch_bounds__(256) k_draw_fill(const __grid_constant__ DrawArgs a) { k_draw_fill_impl(a); }
// batched twin: one launch serves gridDim.y operators (hd_batch_run)
__global__ void __launch_bounds__(256) k_draw_fill_b(const DrawArgs* __restrict__ argv) {
  k_draw_fill_impl(argv[blockIdx.y]);
}

template <typename T, int MODE, int RS, int EK>
__global__ void __launch_bounds__(kNtThreads, 1) k_nt(const __grid_constant__ NtArgs<T> a) {
  k_nt_impl<T, MODE, RS, EK>(a);
}
// batched twin: operator blockIdx.y's arguments — tensor maps included (the
// TMA unit reads a 64-B aligned descriptor from global memory) — from the
// device table of hd_batch_run
template <typename T, int MODE, int RS, int EK>
__global__ void __launch_bounds__(kNtThreads, 1) k_nt_b(const NtArgs<T>* __restrict__ argv) {
  k_nt_impl<T, MODE, RS, EK>(argv[blockIdx.y]);
}

}  // namespace hd
