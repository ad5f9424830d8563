// Streaming (HBM-bound) and small (k x k) kernels of the HD hot path.
//
// One probe of the reference (ginibre.hpp:58-106, haar.hpp:40-67) becomes a
// short fixed sequence of launches:
//   k_dots   GEMV-T  a = P^T v over a chain panel (+ a second panel), with
//            the chain's pending Gram column and side reductions fused in
//   k_small_* one CTA: deterministic reduction of the per-block partials and
//            all O(k^2) compact-WY algebra (T update, T / T^T solves,
//            reflector finalisation, sparse corner products)
//   k_fold   GEMV-N  p = D (x - P beta) writing the new reflector column
//   k_other / k_ginout  GEMV-N producing the probe output with the
//            dynamics update fused into the epilogue.
#pragma once

#include <climits>
#include <cstdint>

#include "hd_device.cuh"

namespace hd {


// Cross-CTA reduction of a CTA's slot row acc[nslots] (shared memory):
// groups of kGroup consecutive CTAs — each CTA parks its row in `scratch`,
// and the last CTA of the group to arrive (fence + atomic ticket) adds the
// group's rows in fixed CTA order, so one partial per group reaches the
// single-CTA kernels and results stay bitwise deterministic:
//   partials[s * ngroups + group].
// Kernels using this never return early (every CTA must take a ticket).
constexpr int kGroup = 8;

struct Flush {
  double* partials = nullptr;  // [nslots][ngroups]
  double* scratch = nullptr;   // [gridDim.x][nslots]
  int* counters = nullptr;     // [ngroups], zero between launches
};

__device__ __forceinline__ void flush_row(const double* acc, int nslots, const Flush& f) {
  __shared__ int s_last;
  __syncthreads();
  double* row = f.scratch + (size_t)blockIdx.x * nslots;
  for (int s = threadIdx.x; s < nslots; s += blockDim.x) row[s] = acc[s];
  __threadfence();
  __syncthreads();
  const int grp = blockIdx.x / kGroup;
  const int b0 = grp * kGroup;
  const int gsz = min(kGroup, (int)gridDim.x - b0);
  if (threadIdx.x == 0) s_last = (atomicAdd(f.counters + grp, 1) == gsz - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int ng = ((int)gridDim.x + kGroup - 1) / kGroup;
  for (int s = threadIdx.x; s < nslots; s += blockDim.x) {
    double v = 0.0;
    for (int b = 0; b < gsz; ++b) v += __ldcg(f.scratch + (size_t)(b0 + b) * nslots + s);
    f.partials[(size_t)s * ng + grp] = v;
  }
  if (threadIdx.x == 0) f.counters[grp] = 0;
}

// ------------------------------------------- TMA-pipelined streaming warps
// Each warp streams its own contiguous run of 256-row tiles through a
// private ring of kRing shared-memory stages: lane 0 keeps kRing chunks
// (kCW columns of one tile = kCW x 2 KB contiguous in the tile-major panel)
// in flight with cp.async.bulk, the whole warp consumes a chunk and lane 0
// refills the slot. No inter-warp synchronisation in the streaming loop;
// per-warp slot rows keep the GEMV-T sums deterministic.
constexpr int kCW = 4;
#ifndef HD_KRING
#define HD_KRING 3
#endif
constexpr int kRing = HD_KRING;
constexpr int kMaxWarps = 8;

template <typename T>
__device__ __forceinline__ double2 lds_pair(const T* p) {
  if constexpr (sizeof(T) == 8) {
    return *reinterpret_cast<const double2*>(p);
  } else {
    const float2 f = *reinterpret_cast<const float2*>(p);
    return make_double2(f.x, f.y);
  }
}

// Position of a chunk in a warp's stream (tile-major, then job, then chunk).
struct StreamPos {
  int64_t tile;
  int job, chunk;
};


// ------------------------------------------------------------------ status
// status[0]: abort (non-zero: every later kernel of this op returns at once)
// status[1]: first non-finite dynamics step (INT_MAX = none)
// status[2]: non-finite probe input seen
enum { kStAbort = 0, kStBadStep = 1, kStBadInput = 2, kStWords = 4 };

__device__ __forceinline__ bool aborted(const int* st) { return *(volatile const int*)st != 0; }

// --------------------------------------------------------- chain (device)
struct ChainDev {
  double* sig = nullptr;   // [K] column scale: w_j = sig_j * P[:, j]
  double* c = nullptr;     // [K] reflector coefficient (reflect.hpp:173)
  double* s = nullptr;     // [K] leading factor s_j = -sign (reflect.hpp:174)
  double* G = nullptr;     // [K*K] Gram of normalised w (col-major, upper)
  double* Tm = nullptr;    // [K*K] compact-WY T, P_1..P_k = I - W T W^T
  double* Drow = nullptr;  // [Dlen] cumulative-sign diagonal, head rows
  double* Dtail = nullptr; // [1] D for rows >= Dlen
  int64_t K = 0;           // column capacity
  int64_t Dlen = 0;
};

// ---------------------------------------------------------- row shards
// A streaming kernel processes local panel tiles [tile0, tile0 + ntiles);
// local panel row li is global row li + gdelta, and the row's entry of a
// dense vector (input x, output y, ...) sits at index (global row - vbase).
// Unsharded (and shard 0): all zero. A shard s > 0 keeps a replica of the
// head rows [0, H) in local tiles [0, H/256) for the single-CTA stages and
// streams only its own rows [lo, hi): tile0 = H/256, gdelta = lo - H,
// vbase = lo.
struct RowMap {
  int64_t tile0 = 0;
  int64_t gdelta = 0;
  int64_t vbase = 0;
};

// ============================================================== k_dots
template <typename T>
struct DotJob {
  const T* P = nullptr;
  int64_t K = 0;
  int ncols = 0;
  int pend = -1;        // pending column (Gram not yet known) or -1
  Src<T> rhs;
  int slot_dot = 0;     // [ncols] slots of P[:, j] . rhs
  int slot_pend = -1;   // [pend + 1] slots of P[:, j] . P[:, pend]
  int slot_sumsq = -1;  // rhs . rhs
  T* wcol = nullptr;    // optional: write rhs into this panel's column wj
  int64_t wK = 0, wj = 0;
  double* pivot_out = nullptr;  // optional: rhs value at pivot_row
  int64_t pivot_row = -1;
  int check_finite = 0;
};

template <typename T>
struct DotArgs {
  DotJob<T> job[3];  // up to three panels (Ginibre: fold chain + opposite store with x, other chain with g)
  int njobs = 1;
  int64_t n = 0, ntiles = 0;
  RowMap rm;
  Flush out;
  int nslots = 0;
  int* status = nullptr;
  int prefetch = 0;  // host-asserted: the previous launch writes no panel read here
  unsigned long long* trace = nullptr;  // debug: latest CTA exit time -> trace[8]
  // bytes of the END of the stream to keep in L2 (evict-last): the fold
  // that follows streams the same panel last-to-first (ApplyArgs::reverse)
  int64_t l2_keep = 0;
  int same_rhs = 0;  // host-asserted: job[1].rhs == job[0].rhs (reuse job 0's rows)
  // > 1: few tiles (small n): `split` warps share each tile, warp g of a tile
  // streaming the g-th of `split` contiguous chunk ranges of each job (the
  // per-column sums add up in the flush); the row side effects (sums of
  // squares, pivot, column write) belong to warp 0 of the tile
  int split = 1;
};

// Shared-memory carve-up of the streaming kernels (per warp: ring + slots).
// Columns per chunk: 4 for fp64, 8 for fp32, so a chunk is 8 KB either way
// and the per-chunk costs (barrier wait, butterfly, slot update) are spread
// over the same bytes (fp32: 3.0 -> see DESIGN.md §4.2a).
#ifndef HD_CW64
#define HD_CW64 4  // fp64 columns per chunk (A/B builds: 2)
#endif
template <typename T>
__host__ __device__ constexpr int chunk_cols() {
  return sizeof(T) == 8 ? HD_CW64 : 8;
}

template <typename T>
__host__ __device__ constexpr size_t ring_bytes() {
  return (size_t)kRing * chunk_cols<T>() * kTile * sizeof(T);
}

// Add the warp sums of a chunk's CW per-lane column partials to dst[col0 + u]
// for col0 + u < lim (fixed butterfly order: deterministic).
template <int CW>
__device__ __forceinline__ void add_chunk_sums(const double* d, int lane, int col0, int lim, double* dst) {
  if constexpr (CW == 2) {
    const double f = warp_sum2(d[0], d[1], lane);
    const int u = lane >> 4;
    if ((lane & 15) == 0 && col0 + u < lim) dst[col0 + u] += f;
  } else if constexpr (CW == 4) {
    const double f = warp_sum4(d[0], d[1], d[2], d[3], lane);
    const int u = lane >> 3;
    if ((lane & 7) == 0 && col0 + u < lim) dst[col0 + u] += f;
  } else {
    static_assert(CW == 8, "chunk of 4 or 8 columns");
    const double f = warp_sum8(d, lane);
    const int u = lane >> 2;
    if ((lane & 3) == 0 && col0 + u < lim) dst[col0 + u] += f;
  }
}

// GEMV-T a = P^T v (k_dots). Lane l holds rows 2(l + 32q) + {0, 1} of the
// current tile's right-hand side(s); each 4-column chunk costs 16 LDS.128,
// 32 (or 64 with a pending column) DFMA and one 4-way butterfly.
template <typename T>
__device__ __forceinline__ void k_dots_impl(const DotArgs<T>& a) {
  constexpr int kCW = chunk_cols<T>();
  extern __shared__ __align__(128) unsigned char smem[];
  const int nw = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nsl = (a.nslots + 1) & ~1;
  unsigned char* ring = smem + (size_t)w * ring_bytes<T>();
  double* accs = reinterpret_cast<double*>(smem + (size_t)nw * ring_bytes<T>());
  double* acc = accs + (size_t)w * nsl;
  uint64_t* full = reinterpret_cast<uint64_t*>(accs + (size_t)nw * nsl) + w * kRing;
  for (int s = lane; s < nsl; s += 32) acc[s] = 0.0;
  if (lane == 0) {
    for (int s = 0; s < kRing; ++s) mbar_init(full + s, 1);
    mbar_fence_init();
  }
  __syncwarp();
  const int64_t W = (int64_t)gridDim.x * nw;
  const int64_t gw = (int64_t)blockIdx.x * nw + w;
  int64_t t0, t1;
  int grp = 0;
  if (a.split > 1) {
    const int64_t tile = gw / a.split;
    grp = (int)(gw % a.split);
    t0 = tile < a.ntiles ? tile : a.ntiles;
    t1 = tile < a.ntiles ? tile + 1 : a.ntiles;
  } else {
    t0 = gw * a.ntiles / W;
    t1 = (gw + 1) * a.ntiles / W;
  }
  const bool owner = (grp == 0);
  // this warp's chunks of each job: [lo[j], lo[j] + nchw[j])
  int lo[3], nchw[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int nc = (j < a.njobs) ? (a.job[j].ncols + kCW - 1) / kCW : 0;
    lo[j] = grp * nc / a.split;
    nchw[j] = (grp + 1) * nc / a.split - lo[j];
  }
  const uint32_t nst = (uint32_t)((t1 - t0) * (nchw[0] + nchw[1] + nchw[2]));
  const int64_t keep = a.l2_keep / (W * (int64_t)(kCW * kTile * sizeof(T)));
  const uint32_t keep_from = keep >= (int64_t)nst ? 0u : nst - (uint32_t)keep;
  // cursor of the next chunk to issue (issue() is called with it = 0, 1, 2, ...):
  // stream order is tile, then job 0's chunks, then job 1's
  int64_t cur_k = 0;
  auto first_job = [&]() {
    int j = 0;
    while (j < 2 && nchw[j] == 0) ++j;
    return j;
  };
  int cur_j = first_job(), cur_c = 0;
  auto issue = [&](uint32_t it) {
    StreamPos p;
    p.tile = t0 + cur_k;
    p.job = cur_j;
    p.chunk = cur_c;
    if (++cur_c == nchw[cur_j]) {
      cur_c = 0;
      int nj = cur_j + 1;
      while (nj < 3 && nchw[nj] == 0) ++nj;
      if (nj < 3) {
        cur_j = nj;
      } else {
        cur_j = first_job();
        ++cur_k;
      }
    }
    const DotJob<T>& J = a.job[p.job];
    p.chunk += lo[p.job];
    const int nc = min(kCW, J.ncols - p.chunk * kCW);
    const uint32_t bytes = (uint32_t)(nc * kTile * sizeof(T));
    const int s = it % kRing;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot precede the refill
    mbar_arrive_expect_tx(full + s, bytes);
    bulk_g2s(ring + (size_t)s * kCW * kTile * sizeof(T),
             J.P + (size_t)(p.tile + a.rm.tile0) * (size_t)(J.K << kTileShift) + (size_t)p.chunk * kCW * kTile, bytes,
             full + s, it >= keep_from);
  };
  // panel chunks written two or more launches back: prefetch, then wait
  if (a.prefetch && lane == 0)
    for (uint32_t it = 0; it < (uint32_t)kRing && it < nst; ++it) issue(it);
  pdl_wait();
  pdl_launch();
  if (!a.prefetch && lane == 0)
    for (uint32_t it = 0; it < (uint32_t)kRing && it < nst; ++it) issue(it);
  if (aborted(a.status)) {  // drain the prefetched stages, then do nothing
    for (uint32_t it = 0; it < (uint32_t)kRing && it < nst; ++it) mbar_wait(full + it % kRing, 0);
    t1 = t0;
  }

  double ss0 = 0.0, ss1 = 0.0, ss2 = 0.0;
  bool bad = false;
  double2 x[4], x0[4], pv[4];
  float2 xf[4], pf[4];  // fp32 panels: the right-hand sides in fp32 for FFMA
  // software pipeline: job 0's vector rows and pending column of the NEXT
  // tile are loaded while the current tile is processed; the rows are then
  // finished (scale / mask, or the Philox + Box-Muller draw itself) one row
  // pair per chunk during the current tile's last job-0 chunks, so draw
  // generation overlaps the TMA stream instead of stalling it
  double2 nx[4], np[4], nxf[4];
  const DotJob<T>& J0 = a.job[0];
  const int nch0r = (J0.ncols + kCW - 1) / kCW;
  auto fetch0 = [&](int64_t tile) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t li = (tile + a.rm.tile0) * kTile + 2 * (lane + 32 * q);
      nx[q] = src_raw(J0.rhs, li + a.rm.gdelta, a.n);
      np[q] = (J0.pend >= 0) ? ld_pair(J0.P + paddr(li, J0.pend, J0.K)) : make_double2(0.0, 0.0);
    }
  };
  auto finish0 = [&](int64_t tile, int q) {
    const int64_t i = (tile + a.rm.tile0) * kTile + a.rm.gdelta + 2 * (lane + 32 * q);
    double2 raw = nx[0];
#pragma unroll
    for (int u = 1; u < 4; ++u)
      if (u == q) raw = nx[u];
    const double2 v = src_finish(J0.rhs, i, a.n, raw);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (u == q) nxf[u] = v;
  };
  if (t0 < t1) {
    fetch0(t0);
    for (int q = 0; q < 4; ++q) finish0(t0, q);
  }
  uint32_t it = 0;
  for (int64_t tile = t0; tile < t1; ++tile) {
    double2 cp[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      x0[q] = nxf[q];
      cp[q] = np[q];
    }
    const bool has_next = tile + 1 < t1;
    if (has_next) fetch0(tile + 1);
    for (int jb = 0; jb < a.njobs; ++jb) {
      const DotJob<T>& J = a.job[jb];
      // no chunks and no row side effects for this warp (job 0 also finishes the next tile's rows)
      if (jb > 0 && !owner && nchw[jb] == 0) continue;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t li = (tile + a.rm.tile0) * kTile + 2 * (lane + 32 * q);  // local panel row
        const int64_t i = li + a.rm.gdelta;                                    // global row
        x[q] = (jb == 0 || (jb == 1 && a.same_rhs)) ? x0[q] : src_pair(J.rhs, i, a.n);
        if (owner) {
          const double sq = x[q].x * x[q].x + x[q].y * x[q].y;
          if (jb == 0) ss0 += sq;
          else if (jb == 1) ss1 += sq;
          else ss2 += sq;
          if (J.check_finite) bad |= !(isfinite(x[q].x) && isfinite(x[q].y));
          if (J.pivot_out && (i == J.pivot_row || i + 1 == J.pivot_row)) *J.pivot_out = (i == J.pivot_row) ? x[q].x : x[q].y;
          if (J.wcol) st_pair(J.wcol + paddr(li, J.wj, J.wK), x[q].x, x[q].y);
        }
        pv[q] = (jb == 0) ? cp[q] : (J.pend >= 0) ? ld_pair(J.P + paddr(li, J.pend, J.K)) : make_double2(0.0, 0.0);
        if constexpr (sizeof(T) == 4) {
          xf[q] = make_float2((float)x[q].x, (float)x[q].y);
          pf[q] = make_float2((float)pv[q].x, (float)pv[q].y);
        }
      }
      const int nch = nchw[jb];
      const int clo = lo[jb];
      for (int c = 0; c < nch; ++c, ++it) {
        const int s = it % kRing;
        mbar_wait(full + s, (it / kRing) & 1);
        const T* sp = reinterpret_cast<const T*>(ring + (size_t)s * kCW * kTile * sizeof(T)) + 2 * lane;
        double d[kCW], e[kCW];
        if constexpr (sizeof(T) == 4) {
          // fp32 panels: the lane's 8 products per column are summed in fp32
          // (FFMA) and only the partial sums converted, 8 instead of 32
          // F2F.F64.F32 per chunk; the chunk loop is otherwise conversion-
          // latency bound at half the fp64 bandwidth
#pragma unroll
          for (int u = 0; u < kCW; ++u) {
            float df = 0.f, ef = 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 wv = *reinterpret_cast<const float2*>(sp + u * kTile + 64 * q);
              df = fmaf(wv.x, xf[q].x, fmaf(wv.y, xf[q].y, df));
              ef = fmaf(wv.x, pf[q].x, fmaf(wv.y, pf[q].y, ef));
            }
            d[u] = (double)df;
            e[u] = (double)ef;
          }
        } else {
#pragma unroll
          for (int u = 0; u < kCW; ++u) {
            d[u] = 0.0;
            e[u] = 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const double2 wv = lds_pair(sp + u * kTile + 64 * q);
              d[u] += wv.x * x[q].x + wv.y * x[q].y;
              e[u] += wv.x * pv[q].x + wv.y * pv[q].y;
            }
          }
        }
        __syncwarp();
        if (lane == 0 && it + kRing < nst) issue(it + kRing);
        const int col0 = (c + clo) * kCW;
        add_chunk_sums<kCW>(d, lane, col0, J.ncols, acc + J.slot_dot);
        if (J.pend >= 0 && col0 <= J.pend) add_chunk_sums<kCW>(e, lane, col0, J.pend + 1, acc + J.slot_pend);
        if (jb == 0 && has_next && c >= nch0r - 4) finish0(tile + 1, c - (nch0r - 4));
      }
      if (jb == 0 && has_next)
        for (int q = 0; q < 4 - nch0r; ++q) finish0(tile + 1, q);
    }
  }
  ss0 = warp_sum(ss0);
  ss1 = warp_sum(ss1);
  ss2 = warp_sum(ss2);
  if (lane == 0) {
    if (a.job[0].slot_sumsq >= 0) acc[a.job[0].slot_sumsq] += ss0;
    if (a.njobs > 1 && a.job[1].slot_sumsq >= 0) acc[a.job[1].slot_sumsq] += ss1;
    if (a.njobs > 2 && a.job[2].slot_sumsq >= 0) acc[a.job[2].slot_sumsq] += ss2;
  }
  if (bad) atomicOr(a.status + kStBadInput, 1);
  __syncthreads();
  for (int s = threadIdx.x; s < a.nslots; s += blockDim.x) {
    double v = 0.0;
    for (int u = 0; u < nw; ++u) v += accs[(size_t)u * nsl + s];
    accs[s] = v;  // row 0 (each slot owned by one thread here)
  }
  flush_row(accs, a.nslots, a.out);
  if (a.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    atomicMax(a.trace + 8, t);
  }
}
template <typename T>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) k_dots(const __grid_constant__ DotArgs<T> a) {
  k_dots_impl<T>(a);
}
// batched twin: one launch serves gridDim.y operators, trial blockIdx.y's
// arguments read from a device table (BatchPlan, hd_batch_run)
template <typename T>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) k_dots_b(const DotArgs<T>* __restrict__ argv) {
  k_dots_impl<T>(argv[blockIdx.y]);
}

// ============================================================ GEMV-N core
// Thread layout for the update kernels: one 256-row tile per block of 128
// threads, each thread owns rows (2 t, 2 t + 1) of the tile and streams all
// k columns of that tile (16 B per column, coalesced 2 KB per column).
constexpr int kUpdThreads = 128;

template <typename T, int NACC>
__device__ __forceinline__ void panel_accumulate(const T* P, int64_t K, int ncols, int64_t tile, int tid,
                                                 const double* const* beta_s, double2* acc) {
  const T* base = P + (size_t)tile * (size_t)(K << kTileShift) + 2 * tid;
#pragma unroll
  for (int u = 0; u < NACC; ++u) acc[u] = make_double2(0.0, 0.0);
  int j = 0;
  for (; j + 8 <= ncols; j += 8) {
    double2 w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) w[q] = ld_pair(base + (size_t)(j + q) * kTile);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
#pragma unroll
      for (int u = 0; u < NACC; ++u) {
        const double b = beta_s[u][j + q];
        acc[u].x += w[q].x * b;
        acc[u].y += w[q].y * b;
      }
    }
  }
  for (; j < ncols; ++j) {
    const double2 w = ld_pair(base + (size_t)j * kTile);
#pragma unroll
    for (int u = 0; u < NACC; ++u) {
      const double b = beta_s[u][j];
      acc[u].x += w.x * b;
      acc[u].y += w.y * b;
    }
  }
}

__device__ __forceinline__ double dval(const double* D, const double* Dtail, int64_t Dlen, int64_t i) {
  return i < Dlen ? D[i] : *Dtail;
}

// ------------------------------------------------------------ epilogue
// Built-in update maps fused into the output pass. The AMP and spiked-power
// maps (BASELINE configs 4 and 5; restated from the test oracle's or_amp /
// or_spiked_power) read their scalars (threshold, Onsager coefficient, spike
// overlap) from device words written by the reduction stage of the previous
// probe, so a whole run is one CUDA graph.
//   kEpiAmpInit : yw = y + w (aux = w), z = yw (state)         -> ||z||^2
//   kEpiAmpX    : x = soft(x + y, *sc) (state = x, aux = beta) -> nnz(x), ||x - beta||^2
//   kEpiAmpZ    : z = yw - y + (*sc) z (state = z, aux = yw)   -> ||z||^2
//   kEpiSpike   : g = y + (*sc) u (aux = u; y <- g)            -> ||g||^2, <u, g>
enum EpiKind : int {
  kEpiPlain = 0, kEpiNormalize = 1, kEpiTanhMix = 2, kEpiAmpInit = 3, kEpiAmpX = 4, kEpiAmpZ = 5, kEpiSpike = 6
};

__host__ __device__ constexpr int epi_nred(int kind) {
  return kind == kEpiNormalize || kind == kEpiAmpInit || kind == kEpiAmpZ ? 1
         : (kind == kEpiAmpX || kind == kEpiSpike)                       ? 2
                                                                         : 0;
}

// The per-row arithmetic of the maps above, shared by every output kernel
// (same operation order as the oracle: experiments.cpp:31-39 soft threshold,
// or_amp's z update, or_spiked_power's spike term). Returns the value stored
// in the state / output vector; r0, r1 receive the row's reduction terms.
__device__ __forceinline__ double epi_row(int kind, double v, double st, double aux, double sc, double& r0,
                                          double& r1) {
  r0 = 0.0;
  r1 = 0.0;
  switch (kind) {
    case kEpiAmpInit: {
      const double z = v + aux;
      r0 = z * z;
      return z;
    }
    case kEpiAmpX: {
      const double r = st + v;
      const double mag = fabs(r) - sc;
      const double x = (mag > 0.0) ? (r > 0.0 ? mag : -mag) : 0.0;
      r0 = (mag > 0.0) ? 1.0 : 0.0;
      const double d = x - aux;
      r1 = d * d;
      return x;
    }
    case kEpiAmpZ: {
      const double z = aux - v + sc * st;
      r0 = z * z;
      return z;
    }
    case kEpiSpike: {
      const double g = v + sc * aux;
      r0 = g * g;
      r1 = aux * g;
      return g;
    }
    default:
      r0 = v * v;
      return v;
  }
}

// Store rows (i, i+1) of a user-visible length-n vector (odd n safe).
template <typename T>
__device__ __forceinline__ void st_pair_guard(T* p, int64_t i, int64_t n, double a, double b) {
  if (i + 1 < n) st_pair(p + i, a, b);
  else if (i < n) p[i] = (T)a;
}

template <typename T>
struct Epi {
  int kind = kEpiPlain;
  T* y = nullptr;                 // probe output (optional for tanh mix)
  const T* yadd = nullptr;        // GOE: v = (yadd + v) * add_scale
  double add_scale = 1.0;
  const T* xprev = nullptr;       // tanh mix: x_{t-1}
  const double* xprev_scale = nullptr;
  T* xnext = nullptr;             // tanh mix: x_{t+1}
  double* partials = nullptr;     // normalize / app maps: per-block sums [block][epi_nred]
  T* state = nullptr;             // app maps: the state vector updated in place (x or z)
  const T* aux = nullptr;         // app maps: w, beta, yw or u
  const double* sc = nullptr;     // app maps: device scalar (threshold, Onsager, theta <u, x>)
  int step = 0;
};

// Epilogue of global rows (i, i + 1); the row's vector entries sit at i - vbase.
template <typename T>
__device__ __forceinline__ void epilogue(const Epi<T>& e, int* status, int64_t i, int64_t n, double2 v,
                                         double* red_s, int64_t vbase) {
  double ss = 0.0, ss2 = 0.0;
  bool bad = false;
  const int64_t vi = i - vbase;
  if (i < n) {
    if (e.yadd) {
      double2 ya;
      if (i + 1 < n) {
        if constexpr (sizeof(T) == 8) ya = *reinterpret_cast<const double2*>(e.yadd + vi);
        else { const float2 f = *reinterpret_cast<const float2*>(e.yadd + vi); ya = make_double2(f.x, f.y); }
      } else {
        ya = make_double2((double)e.yadd[vi], 0.0);
      }
      v.x = (ya.x + v.x) * e.add_scale;
      v.y = (ya.y + v.y) * e.add_scale;
    }
    if (i + 1 >= n) v.y = 0.0;
    if (e.kind >= kEpiAmpInit) {
      const double sc = e.sc ? *e.sc : 0.0;
      double2 st = make_double2(0.0, 0.0), ax = make_double2(0.0, 0.0);
      if (e.state && e.kind != kEpiAmpInit) st = make_double2((double)e.state[vi], (i + 1 < n) ? (double)e.state[vi + 1] : 0.0);
      if (e.aux) ax = make_double2((double)e.aux[vi], (i + 1 < n) ? (double)e.aux[vi + 1] : 0.0);
      double a0, a1, b0, b1;
      const double o0 = epi_row(e.kind, v.x, st.x, ax.x, sc, a0, a1);
      double o1 = epi_row(e.kind, v.y, st.y, ax.y, sc, b0, b1);
      if (i + 1 >= n) {
        o1 = 0.0;
        b0 = b1 = 0.0;
      }
      if (e.state) st_pair_guard(e.state - vbase, i, n, o0, o1);
      if (e.kind == kEpiAmpInit || e.kind == kEpiSpike) v = make_double2(o0, o1);  // y <- yw / g
      bad = !(isfinite(o0) && isfinite(o1));
      ss = a0 + b0;
      ss2 = a1 + b1;
    } else if (e.kind == kEpiTanhMix) {
      double2 xp = make_double2(0.0, 0.0);
      if (e.xprev) {
        if constexpr (sizeof(T) == 8) xp = *reinterpret_cast<const double2*>(e.xprev + vi);
        else { const float2 f = *reinterpret_cast<const float2*>(e.xprev + vi); xp = make_double2(f.x, f.y); }
        if (e.xprev_scale) { xp.x *= *e.xprev_scale; xp.y *= *e.xprev_scale; }
      }
      const double a = tanh(2.0 * v.x) + 0.1 * xp.x;
      const double b = (i + 1 < n) ? tanh(2.0 * v.y) + 0.1 * xp.y : 0.0;
      st_pair_guard(e.xnext - vbase, i, n, a, b);
      bad = !(isfinite(a) && isfinite(b));
    } else {
      bad = !(isfinite(v.x) && isfinite(v.y));
      ss = v.x * v.x + v.y * v.y;
    }
    if (e.y) st_pair_guard(e.y - vbase, i, n, v.x, v.y);
  }
  if (bad) {
    atomicMin(status + kStBadStep, e.step);
    atomicOr(status + kStAbort, 1);
  }
  const int nred = epi_nred(e.kind);
  if (nred >= 1) {
    const double t = block_sum<kUpdThreads>(ss, red_s);
    if (threadIdx.x == 0) e.partials[(size_t)blockIdx.x * nred] = t;
  }
  if (nred >= 2) {
    const double t = block_sum<kUpdThreads>(ss2, red_s);
    if (threadIdx.x == 0) e.partials[(size_t)blockIdx.x * nred + 1] = t;
  }
}

// ============================================================= k_apply
// GEMV-N on the TMA ring: warp w accumulates P[:, 8c + w] beta_{8c+w} into
// its 8 rows-per-lane registers over all chunks of the tile; the 8 warps'
// row partials are combined through shared memory (fixed order) and the
// tile epilogue runs on 128 threads x 2 rows. The same column loads can also
// feed a GEMV-T against the NEXT probe's fresh draw (regenerated on-chip
// from Philox, or read from the injected queue): the Gram dots the next Haar
// mix reflector needs (haar.hpp:57,63), so no extra pass over the other
// chain is required.
//   FOLD : p = D (x - acc)  -> new column p[off:] * 2^-e, head p[0..off],
//          ||p[off:]||^2
//   OTHER: y = D z - acc    -> epilogue (output / dynamics), ||y||^2
enum ApplyMode : int { kApplyFold = 0, kApplyOther = 1 };

template <typename T>
struct ApplyArgs {
  const T* P = nullptr;
  int64_t K = 0;
  int ncols = 0;
  const double* beta = nullptr;
  int64_t n = 0, ntiles = 0;
  RowMap rm;
  const double* D = nullptr;
  const double* Dtail = nullptr;
  int64_t Dlen = 0;
  // fold
  Src<T> x;
  T* Pw = nullptr;
  int64_t newj = 0, off = 0;
  const double* escale = nullptr;
  double* head = nullptr;
  // other
  const double* z = nullptr;
  int64_t zlen = 0;
  Epi<T> epi;
  // speculative dots with the next draw (kind kSrcNone = off; OTHER only)
  Src<T> spec;
  int slot_spec = 0;  // [ncols]
  // ... and, when the next probe hits the same side, the next mix column
  // itself: the draw written to gcol[:, gj], its tail norm^2 (slot_gss =
  // slot_spec + ncols) and its pivot value (gpivot at global row gpivot_row),
  // so the next k_dots need not regenerate it
  T* gcol = nullptr;
  int64_t gK = 0, gj = 0;
  double* gpivot = nullptr;
  int64_t gpivot_row = -1;
  int slot_gss = -1;
  int slot_ss = 0;    // fold: ||p[off:]||^2; other: ||y||^2
  Flush out;
  int nslots = 0;
  int* status = nullptr;
  int prefetch = 0;  // host-asserted: the previous launch writes no panel read here
  // Stream each warp's tiles (and each tile's chunks) last to first. A fold
  // right after the k_dots pass over the same panel then starts on the
  // chunks k_dots read last, which are still in L2.
  int reverse = 0;
  // bytes of the END of the stream to keep in L2 (evict-last); for a
  // reversed fold that is the panel's head of every warp range, which the
  // next probe's k_dots reads first
  int64_t l2_keep = 0;
  // 1: few tiles (small n): one CTA per tile, warp w streaming the w-th
  // contiguous range of its chunks; the row partial sums meet in shared
  // memory (fixed order) and warp 0 runs the epilogue
  int cta_split = 0;
};

template <typename T, int MODE>
__device__ __forceinline__ void k_apply_impl(const ApplyArgs<T>& a) {
  constexpr int kCW = chunk_cols<T>();
  extern __shared__ __align__(128) unsigned char smem[];
  const int nw = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nsl = (a.nslots + 1) & ~1;
  const int nb = (a.ncols + 1) & ~1;
  unsigned char* ring = smem + (size_t)w * ring_bytes<T>();
  double* beta_s = reinterpret_cast<double*>(smem + (size_t)nw * ring_bytes<T>());
  double* accs = beta_s + nb;
  double* acc = accs + (size_t)w * nsl;
  uint64_t* full = reinterpret_cast<uint64_t*>(accs + (size_t)nw * nsl) + w * kRing;
  // cta_split: [nw][128] row pairs after the barriers (16-byte aligned)
  double2* red = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(full + (nw - w) * kRing) + 15) & ~(uintptr_t)15);
  for (int j = threadIdx.x; j < a.ncols; j += blockDim.x) beta_s[j] = a.beta[j];
  for (int s = lane; s < nsl; s += 32) acc[s] = 0.0;
  if (lane == 0) {
    for (int s = 0; s < kRing; ++s) mbar_init(full + s, 1);
    mbar_fence_init();
  }
  const bool spec = (a.spec.kind != kSrcNone);
  const int64_t W = (int64_t)gridDim.x * nw;
  const int64_t gw = (int64_t)blockIdx.x * nw + w;
  const bool cs = a.cta_split != 0;
  int64_t t0 = cs ? (int64_t)blockIdx.x : gw * a.ntiles / W;
  int64_t t1 = cs ? t0 + 1 : (gw + 1) * a.ntiles / W;
  const int ncht = (a.ncols + kCW - 1) / kCW;
  const int clo = cs ? w * ncht / nw : 0;  // this warp's chunks [clo, clo + nch)
  const int nch = cs ? (w + 1) * ncht / nw - clo : ncht;
  const bool epi_warp = !cs || w == 0;     // runs the row epilogue and side effects
  const uint32_t nst = (uint32_t)((t1 - t0) * nch);
  const int64_t tlast = t1 - 1;
  const bool rev = a.reverse != 0;
  const int64_t keep = a.l2_keep / (W * (int64_t)(kCW * kTile * sizeof(T)));
  const uint32_t keep_from = keep >= (int64_t)nst ? 0u : nst - (uint32_t)keep;
  int64_t cur_k = 0;  // cursor of the next chunk to issue (it = 0, 1, 2, ...)
  int cur_c = 0;
  auto issue = [&](uint32_t it) {
    const int64_t tile = rev ? tlast - cur_k : t0 + cur_k;
    const int c = clo + (rev ? nch - 1 - cur_c : cur_c);
    if (++cur_c == nch) {
      cur_c = 0;
      ++cur_k;
    }
    const int nc = min(kCW, a.ncols - c * kCW);
    const uint32_t bytes = (uint32_t)(nc * kTile * sizeof(T));
    const int s = it % kRing;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(full + s, bytes);
    bulk_g2s(ring + (size_t)s * kCW * kTile * sizeof(T),
             a.P + (size_t)(tile + a.rm.tile0) * (size_t)(a.K << kTileShift) + (size_t)c * kCW * kTile, bytes,
             full + s, it >= keep_from);
  };
  __syncwarp();
  if (a.prefetch && lane == 0)
    for (uint32_t it = 0; it < (uint32_t)kRing && it < nst; ++it) issue(it);
  pdl_wait();
  pdl_launch();
  if (!a.prefetch && lane == 0)
    for (uint32_t it = 0; it < (uint32_t)kRing && it < nst; ++it) issue(it);
  for (int j = threadIdx.x; j < a.ncols; j += blockDim.x) beta_s[j] = a.beta[j];
  __shared__ int s_abort;  // one decision per CTA (cta_split warps meet at barriers)
  if (threadIdx.x == 0) s_abort = aborted(a.status) ? 1 : 0;
  __syncthreads();
  if (s_abort) {
    for (uint32_t it = 0; it < (uint32_t)kRing && it < nst; ++it) mbar_wait(full + it % kRing, 0);
    t1 = t0;
  }

  double ss = 0.0, gss = 0.0;
  bool bad = false;
  // software pipeline: the next tile's x (fold) or x_{t-1} (tanh mix) rows
  double2 nv[4];
  auto fetchv = [&](int64_t tile) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = (tile + a.rm.tile0) * kTile + a.rm.gdelta + 2 * (lane + 32 * q);
      if constexpr (MODE == kApplyFold) {
        nv[q] = src_raw(a.x, i, a.n);
      } else {
        nv[q] = make_double2(0.0, 0.0);
        if (a.epi.kind == kEpiTanhMix && a.epi.xprev && i < a.n) {
          const int64_t vi = i - a.rm.vbase;
          nv[q].x = (double)a.epi.xprev[vi];
          if (i + 1 < a.n) nv[q].y = (double)a.epi.xprev[vi + 1];
        }
      }
    }
  };
  if (t0 < t1) fetchv(rev ? tlast : t0);
  // The next draw (Philox + Box-Muller: fp64 transcendentals) of the NEXT
  // tile is generated one row pair per chunk inside the current tile's
  // streaming loop, so it overlaps the TMA stream instead of stalling it
  // at the tile boundary; the first tile's rows are generated up front.
  double2 gn[4];
  auto gen = [&](int64_t tile, int q) {
    const int64_t i = (tile + a.rm.tile0) * kTile + a.rm.gdelta + 2 * (lane + 32 * q);
    const double2 v = src_pair(a.spec, i, a.n);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (u == q) gn[u] = v;
  };
#pragma unroll
  for (int q = 0; q < 4; ++q) gn[q] = make_double2(0.0, 0.0);
  if (spec && t0 < t1)
    for (int q = 0; q < 4; ++q) gen(rev ? tlast : t0, q);
  // Epilogue of the lane's rows q of `tile`, given the tile's GEMV-N sums
  // rq and prefetched rows cvq. (Deferring OTHER's epilogue into the next
  // tile's streaming loop, like the draw, measured neutral: not done.)
  auto epi = [&](int64_t tile, int q, double2 rq, double2 cvq) {
    const int64_t li = (tile + a.rm.tile0) * kTile + 2 * (lane + 32 * q);  // local panel row
    const int64_t i = li + a.rm.gdelta;                                    // global row
    const double d0 = (i < a.Dlen) ? a.D[i] : *a.Dtail;
    const double d1 = (i + 1 < a.Dlen) ? a.D[i + 1] : *a.Dtail;
    if constexpr (MODE == kApplyFold) {
      const double2 xv = src_finish(a.x, i, a.n, cvq);
      const double p0 = (i < a.n) ? d0 * (xv.x - rq.x) : 0.0;
      const double p1 = (i + 1 < a.n) ? d1 * (xv.y - rq.y) : 0.0;
      const double c0 = (i >= a.off) ? p0 : 0.0, c1 = (i + 1 >= a.off) ? p1 : 0.0;
      const double es = *a.escale;
      st_pair(a.Pw + paddr(li, a.newj, a.K), c0 * es, c1 * es);
      if (i <= a.off) a.head[i] = p0;
      if (i + 1 <= a.off) a.head[i + 1] = p1;
      ss += c0 * c0 + c1 * c1;
    } else {
      double z0 = 0.0, z1 = 0.0;
      if (i < a.zlen) z0 = d0 * a.z[i];
      if (i + 1 < a.zlen) z1 = d1 * a.z[i + 1];
      double2 y = make_double2(z0 - rq.x, z1 - rq.y);
      const Epi<T>& e = a.epi;
      if (i < a.n) {
        if (i + 1 >= a.n) y.y = 0.0;
        const int64_t vi = i - a.rm.vbase;
        if (e.kind == kEpiTanhMix) {
          double2 xp = make_double2(0.0, 0.0);
          if (e.xprev) {
            xp = cvq;  // prefetched x_{t-1} rows
            if (e.xprev_scale) {
              xp.x *= *e.xprev_scale;
              xp.y *= *e.xprev_scale;
            }
          }
          const double o0 = tanh(2.0 * y.x) + 0.1 * xp.x;
          const double o1 = (i + 1 < a.n) ? tanh(2.0 * y.y) + 0.1 * xp.y : 0.0;
          st_pair_guard(e.xnext - a.rm.vbase, i, a.n, o0, o1);
          bad |= !(isfinite(o0) && isfinite(o1));
        } else {
          bad |= !(isfinite(y.x) && isfinite(y.y));
          ss += y.x * y.x + y.y * y.y;
        }
        if (e.y) st_pair_guard(e.y - a.rm.vbase, i, a.n, y.x, y.y);
      }
    }
  };
  uint32_t it = 0;
  for (int64_t k = 0; k < t1 - t0; ++k) {
    const int64_t tile = rev ? tlast - k : t0 + k;
    const int64_t next = rev ? tile - 1 : tile + 1;
    const bool has_next = k + 1 < t1 - t0;
    double2 g[4], r[4], cv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      cv[q] = nv[q];
      g[q] = gn[q];
    }
    if (has_next) fetchv(next);
    const bool gen_next = spec && has_next;
    float2 gf[4];  // fp32 panels: the next draw in fp32 (exact: fp32 draws are fp32-rounded)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t li = (tile + a.rm.tile0) * kTile + 2 * (lane + 32 * q);
      const int64_t i = li + a.rm.gdelta;
      r[q] = make_double2(0.0, 0.0);
      gf[q] = make_float2((float)g[q].x, (float)g[q].y);
      if (a.gcol && epi_warp) {  // the next probe's mix column (masked draw), its norm and pivot
        st_pair(a.gcol + paddr(li, a.gj, a.gK), g[q].x, g[q].y);
        gss += g[q].x * g[q].x + g[q].y * g[q].y;
        if (i == a.gpivot_row || i + 1 == a.gpivot_row) *a.gpivot = (i == a.gpivot_row) ? g[q].x : g[q].y;
      }
    }
    for (int c = 0; c < nch; ++c, ++it) {
      const int s = it % kRing;
      mbar_wait(full + s, (it / kRing) & 1);
      const T* sp = reinterpret_cast<const T*>(ring + (size_t)s * kCW * kTile * sizeof(T)) + 2 * lane;
      const int col0 = (clo + (rev ? nch - 1 - c : c)) * kCW;
      double d[kCW];
      if constexpr (sizeof(T) == 4) {
        // fp32 panels: chunk-local sums in fp32 (FFMA), converted once per
        // row pair / column instead of per element (see k_dots)
        float2 rf[4];
        float df[kCW];
#pragma unroll
        for (int q = 0; q < 4; ++q) rf[q] = make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < kCW; ++u) {
          const float b = (col0 + u < a.ncols) ? (float)beta_s[col0 + u] : 0.f;
          df[u] = 0.f;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float2 wv = *reinterpret_cast<const float2*>(sp + u * kTile + 64 * q);
            if (col0 + u >= a.ncols) wv = make_float2(0.f, 0.f);
            rf[q].x = fmaf(wv.x, b, rf[q].x);
            rf[q].y = fmaf(wv.y, b, rf[q].y);
            df[u] = fmaf(wv.x, gf[q].x, fmaf(wv.y, gf[q].y, df[u]));
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          r[q].x += (double)rf[q].x;
          r[q].y += (double)rf[q].y;
        }
#pragma unroll
        for (int u = 0; u < kCW; ++u) d[u] = (double)df[u];
      } else {
#pragma unroll
        for (int u = 0; u < kCW; ++u) {
          const double b = (col0 + u < a.ncols) ? beta_s[col0 + u] : 0.0;
          d[u] = 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            double2 wv = lds_pair(sp + u * kTile + 64 * q);
            if (col0 + u >= a.ncols) wv = make_double2(0.0, 0.0);
            r[q].x += wv.x * b;
            r[q].y += wv.y * b;
            d[u] += wv.x * g[q].x + wv.y * g[q].y;
          }
        }
      }
      __syncwarp();
      if (lane == 0 && it + kRing < nst) issue(it + kRing);
      if (spec) add_chunk_sums<kCW>(d, lane, col0, a.ncols, acc + a.slot_spec);
      if (gen_next && c < 4) gen(next, c);
    }
    if (gen_next)
      for (int q = nch; q < 4; ++q) gen(next, q);
    if (cs) {  // row partial sums of the CTA's warps, fixed order, to warp 0
#pragma unroll
      for (int q = 0; q < 4; ++q) red[w * 128 + lane + 32 * q] = r[q];
      __syncthreads();
      if (w == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double2 v = red[lane + 32 * q];
          for (int u = 1; u < nw; ++u) {
            const double2 o = red[u * 128 + lane + 32 * q];
            v.x += o.x;
            v.y += o.y;
          }
          r[q] = v;
        }
      }
    }
    // epilogue on the lane's 8 rows
    if (epi_warp)
#pragma unroll
      for (int q = 0; q < 4; ++q) epi(tile, q, r[q], cv[q]);
  }
  ss = warp_sum(ss);
  if (lane == 0) acc[a.slot_ss] += ss;
  if (a.slot_gss >= 0) {
    gss = warp_sum(gss);
    if (lane == 0) acc[a.slot_gss] += gss;
  }
  if constexpr (MODE == kApplyOther) {
    if (bad) {
      atomicMin(a.status + kStBadStep, a.epi.step);
      atomicOr(a.status + kStAbort, 1);
    }
  }
  __syncthreads();
  for (int s = threadIdx.x; s < a.nslots; s += blockDim.x) {
    double v = 0.0;
    for (int u = 0; u < nw; ++u) v += accs[(size_t)u * nsl + s];
    accs[s] = v;
  }
  flush_row(accs, a.nslots, a.out);
}
template <typename T, int MODE>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) k_apply(const __grid_constant__ ApplyArgs<T> a) {
  k_apply_impl<T, MODE>(a);
}
// batched twin: one launch serves gridDim.y operators, trial blockIdx.y's
// arguments read from a device table (BatchPlan, hd_batch_run)
template <typename T, int MODE>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) k_apply_b(const ApplyArgs<T>* __restrict__ argv) {
  k_apply_impl<T, MODE>(argv[blockIdx.y]);
}

// ============================================================ k_ginout
// Ginibre output side (ginibre.hpp:73-83 / 92-102 restated):
//   u = D g_m - P beta1                      (new basis vector, stored)
//   y = sigma (S coef + coef_cur u + D c - P beta3)
// with g_m the masked fresh draw, S the same-side basis store and c the
// sparse coefficient vector of the opposite-side probes.
template <typename T>
struct GinArgs {
  const T* P = nullptr;
  int64_t K = 0;
  int ncols = 0;
  const double* beta1 = nullptr;
  const double* beta3 = nullptr;
  const T* S = nullptr;
  int64_t KS = 0;
  int nS = 0;
  const double* coefS = nullptr;
  T* Sw = nullptr;
  int64_t newj = 0;
  Src<T> g;  // masked draw with D applied
  const double* csp = nullptr;
  int64_t csplen = 0;
  const double* D = nullptr;
  const double* Dtail = nullptr;
  int64_t Dlen = 0;
  const double* coef_cur = nullptr;
  double sigma = 1.0;
  int64_t n = 0;
  RowMap rm;
  int* status = nullptr;
  Epi<T> epi;
};

template <typename T>
__device__ __forceinline__ void k_ginout_impl(const GinArgs<T>& a) {
  extern __shared__ double beta_s[];  // [3][K]
  __shared__ double red_s[32];
  pdl_wait();
  pdl_launch();
  if (aborted(a.status)) return;
  double* b1 = beta_s;
  double* b3 = beta_s + a.K;
  double* cs = beta_s + 2 * a.K;
  for (int j = threadIdx.x; j < a.ncols; j += kUpdThreads) {
    b1[j] = a.beta1[j];
    b3[j] = a.beta3[j];
  }
  for (int j = threadIdx.x; j < a.nS; j += kUpdThreads) cs[j] = a.coefS[j];
  __syncthreads();
  const int64_t tile = blockIdx.x + a.rm.tile0;              // local panel tile
  const int64_t li = tile * kTile + 2 * threadIdx.x;
  const int64_t i = li + a.rm.gdelta;                         // global row
  const double* bp[2] = {b1, b3};
  double2 acc[2];
  panel_accumulate<T, 2>(a.P, a.K, a.ncols, tile, threadIdx.x, bp, acc);
  double2 accS = make_double2(0.0, 0.0);
  if (a.nS > 0) {
    const double* sp[1] = {cs};
    panel_accumulate<T, 1>(a.S, a.KS, a.nS, tile, threadIdx.x, sp, &accS);
  }
  const double2 g = src_pair(a.g, i, a.n);
  double u0 = g.x - acc[0].x, u1 = g.y - acc[0].y;
  if (i >= a.n) u0 = 0.0;
  if (i + 1 >= a.n) u1 = 0.0;
  st_pair(a.Sw + paddr(li, a.newj, a.KS), u0, u1);
  double c0 = 0.0, c1 = 0.0;
  if (i < a.csplen) c0 = dval(a.D, a.Dtail, a.Dlen, i) * a.csp[i];
  if (i + 1 < a.csplen) c1 = dval(a.D, a.Dtail, a.Dlen, i + 1) * a.csp[i + 1];
  const double cc = *a.coef_cur;
  const double y0 = a.sigma * (accS.x + cc * u0 + (c0 - acc[1].x));
  const double y1 = a.sigma * (accS.y + cc * u1 + (c1 - acc[1].y));
  epilogue(a.epi, a.status, i, a.n, make_double2(y0, y1), red_s, a.rm.vbase);
}
template <typename T>
__global__ void __launch_bounds__(kUpdThreads) k_ginout(const __grid_constant__ GinArgs<T> a) {
  k_ginout_impl<T>(a);
}
// batched twin: one launch serves gridDim.y operators, trial blockIdx.y's
// arguments read from a device table (BatchPlan, hd_batch_run)
template <typename T>
__global__ void __launch_bounds__(kUpdThreads) k_ginout_b(const GinArgs<T>* __restrict__ argv) {
  k_ginout_impl<T>(argv[blockIdx.y]);
}

// Scratch words shared between the small kernels of one probe.
enum ScalarSlot {
  kScEscale = 0,   // 2^-e (fold column scale)
  kScIscale = 1,   // 2^e
  kScNrm = 2,      // ||p[off:]||
  kScCoefCur = 3,  // <v_cur, x> (Ginibre) / z[off] (Haar)
  kScPivotG = 4,   // fresh draw at the pivot row (Haar mix)
  kScInv = 5,      // 1/||y|| for the normalize dynamics
  kScSign = 6,
  kScAppA = 10,    // app maps: AMP threshold / spike coefficient theta <u, x>
  kScAppB = 11,    // app maps: AMP Onsager coefficient
  kScWords = 16,
};

// ======================================================= small kernels
// One CTA of 1024 threads per stage. All small state a stage needs is
// staged in shared memory in one global round (thread-per-slot reduction of
// the group partials, sig/c, pivot rows, heads); the two chains touched by a
// stage are then handled by two independent halves of the CTA (named
// barriers 1 and 2), so the critical path is ~3 dependent L2 round trips
// (DESIGN.md §4.3). T stays in global memory (k x k, up to 512^2).
constexpr int kSmallThreads = 1024;
constexpr int kHalf = kSmallThreads / 2;

struct SmallArgs {
  int head_late = 0;  // k_small_gin: read head after griddepcontrol.wait (paired launch)
  // k_small_dots: the normalize map's scalar of the previous step, inv = 1 / ||y||, is taken
  // from this stage's own ||rhs||^2 slot (rhs = y) and published in scal[kScInv] instead
  // of a k_small_norm launch (same rule and abort as k_small_norm_impl)
  int norm_from_ss = 0;
  int norm_step = 0;
  const double* partials = nullptr;  // [slot][nblk] group partials
  int nblk = 0;
  double* scal = nullptr;
  int* status = nullptr;
  ChainDev chA, chB;   // fold chain / other chain
  void* PA = nullptr;  // panels (dtype by template)
  void* PB = nullptr;
  int kA = 0, kB = 0;  // member counts seen by this stage
  int pendA = -1, pendB = -1;
  int slotA_dot = 0, slotA_pend = 0, slotA_ss = 0;
  int slotB_dot = 0, slotB_pend = 0, slotB_ss = 0;
  int64_t off = 0;
  int rule = 0;
  int append = 1;      // fold / mix appended (skip_reflector fault)
  double* beta1 = nullptr;
  double* beta3 = nullptr;
  double* head = nullptr;  // p[0..off]
  double* zbuf = nullptr;
  double* csp = nullptr;
  int64_t csplen = 0;
  double* coefS = nullptr;
  int nS = 0;
  int is_haar = 0;
  int mix_from_spec = 0;   // Haar mix Gram dots from the speculative pass
  const double* spec_parts = nullptr;  // [slot][spec_nblk] of the previous k_apply(OTHER)
  int spec_nblk = 0, spec_slot0 = 0, spec_count = 0;
  int spec_ss = 0;         // ... and the mix draw's tail norm^2 (spec row kB)
  int fold_slot_ss = 0;
  int stageA = 0, stageB = 0;  // stage T_A / T_B in shared memory (host: fits the budget)
  int nslots_in = 0;           // slot rows of `partials` staged by the stage
  int stageC = 0;              // stage the sparse-input corner of P_B in shared memory
  unsigned long long* trace = nullptr;  // debug: %globaltimer stamps per phase (HD_TRACE)
  // 1: do not trigger the next launch early (griddepcontrol.launch_dependents
  // right after the wait); it then starts when this stage exits, and its
  // early TMA prefetch no longer competes with the stage (HD_LATE_LAUNCH)
  int late_launch = 0;
  // two-pass Ginibre (hd_gin2p.cuh): the K1 dots came from the previous output
  // pass with right-hand side y while the probe input is x = y * (*xscale)
  // (lazily normalised): dots scale by it, the sum of squares by its square
  const double* xscale = nullptr;
  // ... and k_small_gin's draw dots from the previous fold pass without the
  // cumulative-sign diagonal (every unmasked row sees D = Dtail of chain B)
  int ag_dtail = 0;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define HD_STAMP(a, k)                                   \
  do {                                                   \
    if ((a).trace && threadIdx.x == 0) (a).trace[k] = gtimer(); \
  } while (0)
// intra-kernel stamps in SM cycles (globaltimer is too coarse for sub-us)
#define HD_CLK(a, k)                                               \
  do {                                                             \
    if ((a).trace && threadIdx.x == 0) (a).trace[k] = clock64();   \
  } while (0)

// The single-CTA helpers are all inlined: after the stages were restructured
// the calls (each a jump into not-yet-fetched code at the start of a launch)
// cost more than the extra code size — measured 23.33 -> 23.14 ms per config-2
// run and 66 -> 64 us per probe at tiny n.

// One slot's sum over the group partials (fixed order; four independent
// accumulators so the loads are in flight together).
// The stages below pick each output's slot from the concatenation of their
// reduction segments, so all segments reduce in one parallel pass (instead
// of one reduction call after another, with the single-slot sums serialised
// on thread 0): bitwise identical results.
__device__ __forceinline__ double st_sum_slot(const double* parts, int nblk, int slot) {
  const double* ps = parts + (size_t)slot * nblk;
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
  int b = 0;
#pragma unroll 1
  for (; b + 4 <= nblk; b += 4) {
    v0 += ps[b];
    v1 += ps[b + 1];
    v2 += ps[b + 2];
    v3 += ps[b + 3];
  }
#pragma unroll 1
  for (; b < nblk; ++b) v0 += ps[b];
  return (v0 + v1) + (v2 + v3);
}

// Async-stage `count` contiguous doubles (global -> shared).
__device__ __forceinline__ void st_stage(const double* src, int64_t count, double* dst, int t, int nthr) {
#pragma unroll 1
  for (int64_t e = t; e < count; e += nthr) cp_async8(dst + e, src + e);
}

// Read view of a compact-WY T (column-major, leading dimension ld): either
// the chain's HBM copy or a shared-memory stage of its k x k corner.
struct TView {
  const double* p;
  int64_t ld;
  __device__ __forceinline__ double operator()(int i, int j) const { return p[i + (int64_t)j * ld]; }
};

// Stage T[:k, :k] into shared memory (ld = k | 1, conflict-free rows) with
// one fully parallel coalesced sweep; threads [t0, t0 + nthr).
__device__ __forceinline__ TView st_stage_T(const ChainDev& ch, int k, double* dst, int t, int nthr) {
  const int64_t ld = k | 1;
  const int w = t >> 5, lane = t & 31, nw = nthr >> 5;  // warp per column, no integer division
#pragma unroll 1
  for (int j = w; j < k; j += nw)
#pragma unroll 1
    for (int i = lane; i < k; i += 32) cp_async8(dst + i + (int64_t)j * ld, ch.Tm + i + (int64_t)j * ch.K);
  return TView{dst, ld};  // valid after cp_async_wait_all() + barrier
}

// T_new[:k, k] = -c T[:k, :k] g (g in shared memory), T_new[k, k] = c; the
// new column is written to global memory and to tcol (shared). Warps
// [w0, w0 + nw) of the CTA, warp per row.
__device__ __forceinline__ void st_T_column(const ChainDev& ch, const TView& tv, int k, double c, const double* g,
                                            double* tcol, int w0, int nw) {
  const int w = (threadIdx.x >> 5) - w0, lane = threadIdx.x & 31;
#pragma unroll 1
  for (int i = w; i < k; i += nw) {
    double v = 0.0;
#pragma unroll 1
    for (int l = i + lane; l < k; l += 32) v += tv(i, l) * g[l];
    v = warp_sum(v);
    if (lane == 0) {
      tcol[i] = -c * v;
      ch.Tm[i + (int64_t)k * ch.K] = -c * v;
    }
  }
  if (threadIdx.x == w0 * 32) {
    tcol[k] = c;
    ch.Tm[k + (int64_t)k * ch.K] = c;
  }
}

// out[j] = sum_{i <= j} T[i, j] u[i] for j < k (column p, if >= 0, comes
// from tcol in shared memory). Warp per column.
__device__ __forceinline__ void st_Tt(const TView& tv, int k, const double* u, double* out, int p,
                                      const double* tcol, int w0, int nw) {
  const int w = (threadIdx.x >> 5) - w0, lane = threadIdx.x & 31;
#pragma unroll 1
  for (int j = w; j < k; j += nw) {
    double v = 0.0;
    const double* col = (j == p) ? tcol : tv.p + (int64_t)j * tv.ld;
#pragma unroll 1
    for (int i = lane; i <= j; i += 32) v += col[i] * u[i];
    v = warp_sum(v);
    if (lane == 0) out[j] = v;
  }
}

// out[i] = sum_{j >= i} T[i, j] u[j] for i < k (column p from tcol).
__device__ __forceinline__ void st_T(const TView& tv, int k, const double* u, double* out, int p,
                                     const double* tcol, int w0, int nw) {
  const int w = (threadIdx.x >> 5) - w0, lane = threadIdx.x & 31;
#pragma unroll 1
  for (int i = w; i < k; i += nw) {
    double v = 0.0;
#pragma unroll 1
    for (int j = i + lane; j < k; j += 32) v += ((j == p) ? tcol[i] : tv(i, j)) * u[j];
    v = warp_sum(v);
    if (lane == 0) out[i] = v;
  }
}

// make_reflector (reflect.hpp:120-176) scalars for a column streamed into
// the panel: pivot fix-up, scale, coefficient, leading factor; returns the
// sign (0 under the zeroing negative control). Single thread.
template <typename T>
__device__ __forceinline__ double st_reflector(const ChainDev& ch, T* P, int j, int64_t off, double nrm, double pivot,
                                               int rule, double colscale, double unscale, bool append) {
  double sign;
  if (rule == 0) sign = (pivot >= 0.0) ? 1.0 : -1.0;
  else if (rule == 1) sign = (pivot > 0.0) ? 1.0 : -1.0;
  else sign = (pivot >= 0.0) ? 1.0 : 0.0;
  if (nrm == 0.0) sign = 1.0;
  if (append) {
    if (nrm == 0.0) {  // identity reflector: zero column, c = 0, s = 1
      ch.sig[j] = 0.0;
      ch.c[j] = 0.0;
      ch.s[j] = 1.0;
    } else {
      P[paddr(off, j, ch.K)] = (T)((pivot + sign * nrm) * colscale);
      const double r = pivot / nrm;
      ch.sig[j] = unscale / nrm;
      ch.c[j] = 2.0 / (1.0 + 2.0 * sign * r + sign * sign);
      ch.s[j] = -sign;
    }
  }
  return sign;
}

// D update for a member with offset off and leading factor s: D[i] *= s for
// i >= off (threads [t0, t0 + nthr)).
__device__ __forceinline__ void st_D_update(const ChainDev& ch, int64_t off, double s, int t, int nthr) {
  for (int64_t i = off + t; i < ch.Dlen; i += nthr) ch.Drow[i] *= s;
  if (t == 0) *ch.Dtail *= s;
}

// Vector length of the single-CTA stages' shared-memory layout (>= 32 so a
// vector can also hold the <= 19 group partials of one slot).
__host__ __device__ inline int small_kv(int kA, int kB) {
  const int k = (kA > kB ? kA : kB) + 2;
  return k < 32 ? 32 : k;
}

// Shared-memory layout of the small kernels: 12 vectors of length kv.
struct SmallSmem {
  double *v0, *v1, *v2, *v3, *v4, *v5, *v6, *v7, *v8, *v9, *v10, *v11;
  double* sc;  // scalars [16]
};

__device__ __forceinline__ SmallSmem small_smem(double* base, int kv) {
  SmallSmem m;
  double* p = base;
  double** v[12] = {&m.v0, &m.v1, &m.v2, &m.v3, &m.v4, &m.v5, &m.v6, &m.v7, &m.v8, &m.v9, &m.v10, &m.v11};
  for (int i = 0; i < 12; ++i) {
    *v[i] = p;
    p += kv;
  }
  m.sc = p;
  return m;
}

// After k_dots of a probe: finalise chain A's pending column and its forward
// coefficients beta1 = sig (T_A^T (sig a)) (half 1), the Haar mix reflector
// H(g, off) appended to chain B or (Ginibre) the opposite-side sparse
// coefficients (half 2), and the power-of-two fold-column scale.
template <typename T, bool HAAR>
__device__ __forceinline__ void k_small_dots_impl(const SmallArgs& a) {
  extern __shared__ double ssm[];
  HD_STAMP(a, 0);
  const int kv = small_kv(a.kA, a.kB);
  const SmallSmem m = small_smem(ssm, kv);
  double* aA = m.v0;     // red A dot
  double* pA = m.v1;     // red A pend
  double* sgA = m.v2;    // sig A
  double* gA = m.v3;     // G col A / scratch
  double* tA = m.v4;     // new T col A
  double* uA = m.v5;     // sig * a
  double* aB = m.v6;     // mix dots (spec or red) / csp
  double* pB = m.v7;     // red B pend
  double* sgB = m.v8;    // sig B
  double* rowB = m.v9;   // P_B[off, :]
  double* gB = m.v10;    // G col B
  double* tB = m.v11;    // new T col B
  double* tsA = m.sc + 16;
  double* tsB = tsA + (a.stageA ? (size_t)a.kA * (a.kA | 1) : 0);
  double* ps = tsB + (a.stageB ? (size_t)a.kB * (a.kB | 1) : 0);  // [nslots_in][nblk]
  double* ss = ps + (size_t)a.nslots_in * a.nblk;                  // spec rows [kB][spec_nblk]
  T* rowT = reinterpret_cast<T*>(gB);                               // raw pivot row (converted below)
  int* st = reinterpret_cast<int*>(m.sc + 12);                      // staged status words
  const int tid = threadIdx.x;
  const bool spec = HAAR && a.mix_from_spec && a.kB > 0;
  // ---- phase 1: every global load issued asynchronously (no register round
  // trips: the panel row and scalars miss L2 right after a streaming pass).
  // What earlier stages / the previous probe's passes wrote (T, sig, the pivot
  // row of the existing members, the speculative dots, c of the pending
  // members) is issued before griddepcontrol.wait: those kernels completed
  // before this launch; only k_dots' outputs wait.
  HD_CLK(a, 5);
  const TView tvA = a.stageA ? st_stage_T(a.chA, a.kA, tsA, tid, kSmallThreads) : TView{a.chA.Tm, a.chA.K};
  const TView tvB = (HAAR && a.stageB) ? st_stage_T(a.chB, a.kB, tsB, tid, kSmallThreads) : TView{a.chB.Tm, a.chB.K};
  HD_CLK(a, 6);
  if (spec)
    st_stage(a.spec_parts + (size_t)a.spec_slot0 * a.spec_nblk, (int64_t)(a.kB + a.spec_ss) * a.spec_nblk, ss, tid,
             kSmallThreads);
  #pragma unroll 1
  for (int j = tid; j < a.kA; j += kSmallThreads) cp_async8(sgA + j, a.chA.sig + j);
  if (HAAR) {
    const T* PB = (const T*)a.PB;
    #pragma unroll 1
    for (int j = tid; j < a.kB; j += kSmallThreads) {
      cp_async8(sgB + j, a.chB.sig + j);
      cp_async_elem(rowT + j, PB + paddr(a.off, j, a.chB.K));
    }
  }
  if (tid == 0) {
    if (a.pendA >= 0) cp_async8(m.sc + 2, a.chA.c + a.pendA);
    if (a.pendB >= 0) cp_async8(m.sc + 3, a.chB.c + a.pendB);
  }
  pdl_wait();
  HD_STAMP(a, 1);
  if (!a.late_launch) pdl_launch();
  st_stage(a.partials, (int64_t)a.nslots_in * a.nblk, ps, tid, kSmallThreads);
  if (tid == 0) {
    cp_async8(m.sc + 4, a.scal + kScPivotG);
    cp_async4(st + 0, a.status + kStAbort);
    cp_async4(st + 1, a.status + kStBadInput);
  }
  HD_CLK(a, 7);
  cp_async_wait_all();
  HD_CLK(a, 9);
  __syncthreads();
  HD_CLK(a, 10);
  if (st[0] != 0) return;
  if (st[1] != 0) {  // non-finite probe input seen by k_dots: abort the probe
    if (tid == 0) *(volatile int*)(a.status + kStAbort) = 1;
    return;
  }
  if (a.pendA < 0 && tid == 0) m.sc[2] = 0.0;
  if (a.pendB < 0 && tid == 0) m.sc[3] = 0.0;
  if (HAAR)
    #pragma unroll 1
    for (int j = tid; j < a.kB; j += kSmallThreads) rowB[j] = (double)rowT[j];
  {  // all reductions of this stage in one pass (see st_sum_slot)
    const int nA = a.kA, nPA = a.pendA >= 0 ? a.pendA + 1 : 0, nB = a.kB, nPB = a.pendB >= 0 ? a.pendB + 1 : 0;
    const bool ssB = a.slotB_ss >= 0 || (spec && a.spec_ss);
    const int e0 = nA, e1 = e0 + nPA, e2 = e1 + nB, e3 = e2 + nPB, e4 = e3 + 1, e5 = e4 + (ssB ? 1 : 0);
    #pragma unroll 1
    for (int t = tid; t < e5; t += kSmallThreads) {
      if (t < e0) aA[t] = st_sum_slot(ps, a.nblk, a.slotA_dot + t);
      else if (t < e1) pA[t - e0] = st_sum_slot(ps, a.nblk, a.slotA_pend + t - e0);
      else if (t < e2) aB[t - e1] = spec ? st_sum_slot(ss, a.spec_nblk, t - e1) : st_sum_slot(ps, a.nblk, a.slotB_dot + t - e1);
      else if (t < e3) pB[t - e2] = st_sum_slot(ps, a.nblk, a.slotB_pend + t - e2);
      else if (t < e4) m.sc[0] = st_sum_slot(ps, a.nblk, a.slotA_ss);
      else m.sc[1] = (a.slotB_ss >= 0) ? st_sum_slot(ps, a.nblk, a.slotB_ss) : st_sum_slot(ss, a.spec_nblk, a.kB);
    }
  }
  __syncthreads();
  if (!HAAR && (a.xscale || a.norm_from_ss)) {  // two-pass Ginibre: x = y * xscale
    double xs;
    if (a.norm_from_ss) {
      const double nrm = sqrt(m.sc[0]);
      xs = nrm > 0.0 ? 1.0 / nrm : 1.0;
      if (tid == 0) {
        a.scal[kScInv] = xs;
        if (!isfinite(xs)) {
          atomicMin(a.status + kStBadStep, a.norm_step);
          atomicOr(a.status + kStAbort, 1);
        }
      }
      if (!isfinite(xs)) return;  // uniform: every thread reads the same sum
    } else {
      xs = *a.xscale;
    }
    __syncthreads();  // every thread has read m.sc[0] before it is rescaled
    #pragma unroll 1
    for (int t = tid; t < a.kA + a.kB + 1; t += kSmallThreads) {
      if (t < a.kA) aA[t] *= xs;
      else if (t < a.kA + a.kB) aB[t - a.kA] *= xs;
      else m.sc[0] *= xs * xs;
    }
    __syncthreads();
  }
  HD_CLK(a, 11);
  HD_STAMP(a, 2);
  if (tid < kHalf) {
    // ---- half 1: chain A
    const int p = a.pendA;
    if (p >= 0) {
      #pragma unroll 1
      for (int j = tid; j <= p; j += kHalf) {
        gA[j] = sgA[j] * sgA[p] * pA[j];
        a.chA.G[j + (int64_t)p * a.chA.K] = gA[j];
      }
      named_sync(1, kHalf);
      st_T_column(a.chA, tvA, p, m.sc[2], gA, tA, 0, kHalf / 32);
    }
    #pragma unroll 1
    for (int j = tid; j < a.kA; j += kHalf) uA[j] = sgA[j] * aA[j];
    named_sync(1, kHalf);
    st_Tt(tvA, a.kA, uA, gA, p, tA, 0, kHalf / 32);
    named_sync(1, kHalf);
    #pragma unroll 1
    for (int j = tid; j < a.kA; j += kHalf) a.beta1[j] = sgA[j] * gA[j];
    HD_STAMP(a, 3);
    if (tid == 0) {
      const double xn = sqrt(m.sc[0]);
      int e = 0;
      if (xn > 0.0 && isfinite(xn)) frexp(xn, &e);
      a.scal[kScEscale] = ldexp(1.0, -e);
      a.scal[kScIscale] = ldexp(1.0, e);
    }
  } else {
    // ---- half 2: chain B
    const int t2 = tid - kHalf;
    if (HAAR) {
      int kB = a.kB;
      const int p = a.pendB;
      if (p >= 0) {  // fallback path only (same-side speculation unavailable)
        #pragma unroll 1
        for (int j = t2; j <= p; j += kHalf) {
          gB[j] = a.chB.sig[j] * a.chB.sig[p] * pB[j];
          a.chB.G[j + (int64_t)p * a.chB.K] = gB[j];
        }
        named_sync(2, kHalf);
        st_T_column(a.chB, tvB, p, m.sc[3], gB, tB, kHalf / 32, kHalf / 32);
        named_sync(2, kHalf);
        if (a.stageB)  // the staged copy must see the finished column p
          #pragma unroll 1
          for (int i = t2; i <= p; i += kHalf) tsB[i + (int64_t)p * tvB.ld] = tB[i];
        named_sync(2, kHalf);
      }
      // mix reflector H(g, off) -> column kB of chain B
      const double nrm = sqrt(m.sc[1]);
      const double piv = m.sc[4];
      if (t2 == 0) {
        const double sign = st_reflector<T>(a.chB, (T*)a.PB, kB, a.off, nrm, piv, a.rule, 1.0, 1.0, true);
        m.sc[5] = sign;
        m.sc[6] = (nrm == 0.0) ? 0.0 : a.chB.c[kB];
      }
      named_sync(2, kHalf);
      const double sign = m.sc[5], cB = m.sc[6];
      #pragma unroll 1
      for (int j = t2; j < kB; j += kHalf) {
        gB[j] = (nrm == 0.0) ? 0.0 : sgB[j] * (aB[j] / nrm + sign * rowB[j]);
        a.chB.G[j + (int64_t)kB * a.chB.K] = gB[j];
      }
      if (t2 == 0) a.chB.G[kB + (int64_t)kB * a.chB.K] = (nrm == 0.0) ? 0.0 : 2.0 / cB;
      if (nrm != 0.0) st_D_update(a.chB, a.off, -sign, t2, kHalf);
      named_sync(2, kHalf);
      st_T_column(a.chB, tvB, kB, cB, gB, tB, kHalf / 32, kHalf / 32);
    } else {
      // Ginibre: opposite-side coefficients <v_i, x> (or <u_i, x>), rows < kB
      #pragma unroll 1
      for (int q = t2; q < a.kB; q += kHalf) a.csp[q] = aB[q];
    }
  }
  if (a.trace) {
    __syncthreads();
    HD_STAMP(a, 4);
  }
}
template <typename T, bool HAAR>
__global__ void __launch_bounds__(kSmallThreads) k_small_dots(const __grid_constant__ SmallArgs a) {
  k_small_dots_impl<T, HAAR>(a);
}
// batched twin: one launch serves gridDim.y operators, trial blockIdx.y's
// arguments read from a device table (BatchPlan, hd_batch_run)
template <typename T, bool HAAR>
__global__ void __launch_bounds__(kSmallThreads) k_small_dots_b(const SmallArgs* __restrict__ argv) {
  k_small_dots_impl<T, HAAR>(argv[blockIdx.y]);
}

// After k_apply(FOLD): finalise the fold reflector H(p, off) (appended
// unless the skip fault fires), then (Haar) beta = sig (T_B (W_B^T D_B z))
// for the sparse folded iterate z = H p, or (Ginibre) the current coefficient.
template <typename T, bool HAAR>
__device__ __forceinline__ void k_small_fold_impl(const SmallArgs& a) {
  extern __shared__ double ssm[];
  const int kv = small_kv(a.kA, a.kB);
  const SmallSmem m = small_smem(ssm, kv);
  double* az = m.v0;    // corner partial sum_{i<off} P_B[i,j] D_B(i) p_i
  double* rowB = m.v1;  // P_B[off, :]
  double* tmp = m.v2;
  double* sgB = m.v3;
  double* psf = m.v4;   // ||p[off:]||^2 group partials (nblk <= kv)
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const T* PB = (const T*)a.PB;
  const int64_t nr = a.off + 1;
  double* tsB = m.sc + 16;
  double* hs = tsB + (a.stageB ? (size_t)a.kB * (a.kB | 1) : 0);  // head p[0..off]
  double* ds = hs + nr;                                               // D_B[0..off]
  T* cs = reinterpret_cast<T*>(ds + nr);                              // corner [kB][nr]
  // ---- phase 1: every global load issued asynchronously, one wait; what
  // the earlier stages wrote (T_B, the scales, D_B, sig, the corner) before
  // griddepcontrol.wait, the fold pass's outputs after it
  const TView tvB = (HAAR && a.stageB) ? st_stage_T(a.chB, a.kB, tsB, tid, kSmallThreads)
                                            : TView{a.chB.Tm, a.chB.K};
  int* st = reinterpret_cast<int*>(m.sc + 12);
  if (tid == 0) {
    cp_async8(m.sc + 8, a.scal + kScEscale);
    cp_async8(m.sc + 9, a.scal + kScIscale);
  }
  if (HAAR) {
    #pragma unroll 1
    for (int64_t i = tid; i < nr; i += kSmallThreads) cp_async8(ds + i, i < a.chB.Dlen ? a.chB.Drow + i : a.chB.Dtail);
    #pragma unroll 1
    for (int j = tid; j < a.kB; j += kSmallThreads) cp_async8(sgB + j, a.chB.sig + j);
    if (a.stageC)
      #pragma unroll 1
      for (int j = w; j < a.kB; j += kSmallThreads / 32)
        #pragma unroll 1
        for (int64_t i = lane; i < nr; i += 32) cp_async_elem(cs + j * nr + i, PB + paddr(i, j, a.chB.K));
  }
  pdl_wait();
  if (!a.late_launch) pdl_launch();
  st_stage(a.partials + (size_t)a.fold_slot_ss * a.nblk, a.nblk, psf, tid, kSmallThreads);
  st_stage(a.head, nr, hs, tid, kSmallThreads);
  if (tid == 0) cp_async4(st, a.status + kStAbort);
  cp_async_wait_all();
  __syncthreads();
  if (st[0] != 0) return;
  if (HAAR) {
    #pragma unroll 1
    for (int j = w; j < a.kB; j += kSmallThreads / 32) {
      double v = 0.0;
      if (a.stageC) {
        #pragma unroll 1
        for (int64_t i = lane; i < a.off; i += 32) v += (double)cs[j * nr + i] * ds[i] * hs[i];
      } else {
        #pragma unroll 1
        for (int64_t i = lane; i < a.off; i += 32) v += (double)PB[paddr(i, j, a.chB.K)] * ds[i] * hs[i];
      }
      v = warp_sum(v);
      if (lane == 0) {
        az[j] = v;
        rowB[j] = a.stageC ? (double)cs[j * nr + a.off] : (double)PB[paddr(a.off, j, a.chB.K)];
      }
    }
    #pragma unroll 1
    for (int64_t i = tid; i < a.off; i += kSmallThreads) a.zbuf[i] = hs[i];
  }
  if (w == 0) {
    double v = 0.0;
    #pragma unroll 1
    for (int b = lane; b < a.nblk; b += 32) v += psf[b];
    v = warp_sum(v);
    if (lane == 0) {
      m.sc[0] = sqrt(v);
      m.sc[1] = hs[a.off];
      m.sc[2] = HAAR ? ds[a.off] : 0.0;
    }
  }
  __syncthreads();
  const double nrm = m.sc[0], piv = m.sc[1];
  if (tid == 0) {
    const double sign = st_reflector<T>(a.chA, (T*)a.PA, a.kA, a.off, nrm, piv, a.rule, m.sc[8], m.sc[9],
                                        a.append != 0);
    // (H p)[off]: +||p[off:]|| (0 under the zeroing negative control)
    const double zoff = (nrm == 0.0) ? piv : (sign == 0.0 ? 0.0 : nrm);
    m.sc[3] = sign;
    m.sc[4] = zoff;
    a.scal[kScNrm] = nrm;
    a.scal[kScCoefCur] = a.append ? zoff : piv;
    a.scal[kScSign] = sign;
    if (HAAR) a.zbuf[a.off] = zoff;
  }
  __syncthreads();
  if (a.append && nrm != 0.0) st_D_update(a.chA, a.off, -m.sc[3], tid, kSmallThreads);
  if (HAAR) {
    const double zoff = m.sc[4], doff = m.sc[2];
    #pragma unroll 1
    for (int j = tid; j < a.kB; j += kSmallThreads) tmp[j] = sgB[j] * (az[j] + rowB[j] * doff * zoff);
    __syncthreads();
    st_T(tvB, a.kB, tmp, az, -1, nullptr, 0, kSmallThreads / 32);
    __syncthreads();
    #pragma unroll 1
    for (int j = tid; j < a.kB; j += kSmallThreads) a.beta1[j] = sgB[j] * az[j];
  }
}
template <typename T, bool HAAR>
__global__ void __launch_bounds__(kSmallThreads) k_small_fold(const __grid_constant__ SmallArgs a) {
  k_small_fold_impl<T, HAAR>(a);
}
// batched twin: one launch serves gridDim.y operators, trial blockIdx.y's
// arguments read from a device table (BatchPlan, hd_batch_run)
template <typename T, bool HAAR>
__global__ void __launch_bounds__(kSmallThreads) k_small_fold_b(const SmallArgs* __restrict__ argv) {
  k_small_fold_impl<T, HAAR>(argv[blockIdx.y]);
}

// Ginibre, after k_dots over the opposite chain with v = D g_m: pending
// column, beta1 = sig (T (sig a_g)) for the new basis vector (half 1), beta3
// for the sparse part L-rev-adj(c) (half 2), same-side store coefficients.
template <typename T>
__device__ __forceinline__ void k_small_gin_impl(const SmallArgs& a) {
  extern __shared__ double ssm[];
  const int kv = small_kv(0, a.kB);
  const SmallSmem m = small_smem(ssm, kv);
  double* ag = m.v0;
  double* pB = m.v1;
  double* sg = m.v2;
  double* gB = m.v3;
  double* tB = m.v4;
  double* u1 = m.v5;
  double* o1 = m.v6;
  double* ac = m.v7;
  double* o3 = m.v8;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const T* PB = (const T*)a.PB;
  const int64_t nr = a.csplen;
  double* tsB = m.sc + 16;
  double* ps = tsB + (a.stageB ? (size_t)a.kB * (a.kB | 1) : 0);  // [nslots_in][nblk]
  double* cps = ps + (size_t)a.nslots_in * a.nblk;                  // D_B(i) c_i, i < nr
  double* dsg = cps + nr;                                           // D_B rows (staging)
  T* cs = reinterpret_cast<T*>(dsg + nr);                           // corner [kB][nr]
  // ---- phase 1: every global load issued asynchronously, one wait; what
  // the earlier stages / passes wrote before griddepcontrol.wait, the dots
  // pass's partials after it
  const TView tvB = a.stageB ? st_stage_T(a.chB, a.kB, tsB, tid, kSmallThreads) : TView{a.chB.Tm, a.chB.K};
  st_stage(a.csp, nr, cps, tid, kSmallThreads);
  #pragma unroll 1
  for (int64_t i = tid; i < nr; i += kSmallThreads) cp_async8(dsg + i, i < a.chB.Dlen ? a.chB.Drow + i : a.chB.Dtail);
  #pragma unroll 1
  for (int j = tid; j < a.kB; j += kSmallThreads) cp_async8(sg + j, a.chB.sig + j);
  if (a.stageC)
    #pragma unroll 1
    for (int j = w; j < a.kB; j += kSmallThreads / 32)
      #pragma unroll 1
      for (int64_t i = lane; i < nr; i += 32) cp_async_elem(cs + j * nr + i, PB + paddr(i, j, a.chB.K));
  // head = p[0..off] of the fold pass: two launches old when the fold stage ran in between,
  // the immediate predecessor's output when the two stages share a launch (head_late)
  if (!a.head_late)
    #pragma unroll 1
    for (int q = tid; q < a.nS; q += kSmallThreads) a.coefS[q] = a.head[q];
  if (tid == 0) m.sc[0] = (a.pendB >= 0) ? a.chB.c[a.pendB] : 0.0;
  pdl_wait();
  if (!a.late_launch) pdl_launch();
  if (aborted(a.status)) {
    cp_async_wait_all();
    return;
  }
  if (a.head_late)
    #pragma unroll 1
    for (int q = tid; q < a.nS; q += kSmallThreads) a.coefS[q] = a.head[q];
  st_stage(a.partials, (int64_t)a.nslots_in * a.nblk, ps, tid, kSmallThreads);
  cp_async_wait_all();
  __syncthreads();
  {  // both reductions in one pass (see st_sum_slot)
    const int e0 = a.kB, e1 = e0 + (a.pendB >= 0 ? a.pendB + 1 : 0);
    const double dt = a.ag_dtail ? *a.chB.Dtail : 1.0;
    #pragma unroll 1
    for (int t = tid; t < e1; t += kSmallThreads) {
      if (t < e0) ag[t] = dt * st_sum_slot(ps, a.nblk, a.slotB_dot + t);
      else pB[t - e0] = st_sum_slot(ps, a.nblk, a.slotB_pend + t - e0);
    }
  }
  #pragma unroll 1
  for (int64_t i = tid; i < nr; i += kSmallThreads) cps[i] *= dsg[i];
  __syncthreads();
  // corner W_B^T (D_B c) over rows < csplen (does not involve the pending T)
  #pragma unroll 1
  for (int j = w; j < a.kB; j += kSmallThreads / 32) {
    double v = 0.0;
    if (a.stageC) {
      #pragma unroll 1
      for (int64_t i = lane; i < nr; i += 32) v += (double)cs[j * nr + i] * cps[i];
    } else {
      #pragma unroll 1
      for (int64_t i = lane; i < nr; i += 32) v += (double)PB[paddr(i, j, a.chB.K)] * cps[i];
    }
    v = warp_sum(v);
    if (lane == 0) ac[j] = v;
  }
  __syncthreads();
  const int p = a.pendB;
  if (p >= 0) {
    #pragma unroll 1
    for (int j = tid; j <= p; j += kSmallThreads) {
      gB[j] = sg[j] * sg[p] * pB[j];
      a.chB.G[j + (int64_t)p * a.chB.K] = gB[j];
    }
    __syncthreads();
    st_T_column(a.chB, tvB, p, m.sc[0], gB, tB, 0, kSmallThreads / 32);
  }
  #pragma unroll 1
  for (int j = tid; j < a.kB; j += kSmallThreads) {
    u1[j] = sg[j] * ag[j];
    ac[j] = sg[j] * ac[j];
  }
  __syncthreads();
  if (tid < kHalf) st_T(tvB, a.kB, u1, o1, p, tB, 0, kHalf / 32);
  else st_T(tvB, a.kB, ac, o3, p, tB, kHalf / 32, kHalf / 32);
  __syncthreads();
  #pragma unroll 1
  for (int j = tid; j < a.kB; j += kSmallThreads) {
    a.beta1[j] = sg[j] * o1[j];
    a.beta3[j] = sg[j] * o3[j];
  }
}
template <typename T>
__global__ void __launch_bounds__(kSmallThreads) k_small_gin(const __grid_constant__ SmallArgs a) {
  k_small_gin_impl<T>(a);
}
// batched twin: one launch serves gridDim.y operators, trial blockIdx.y's
// arguments read from a device table (BatchPlan, hd_batch_run)
template <typename T>
__global__ void __launch_bounds__(kSmallThreads) k_small_gin_b(const SmallArgs* __restrict__ argv) {
  k_small_gin_impl<T>(argv[blockIdx.y]);
}

// Two-pass Ginibre (hd_gin2p.cuh), after k_nt<FOLD>: finalise the fold
// reflector H(p, off) (k_small_fold) AND its compact-WY T column at once: the
// Gram column W_F^T w_new came out of the same pass for rows > off; the
// pivot row's term W_F[off, j] * w_new[off] (w_new[off] is fixed here, after
// the norm) is added from the panel row. No pending column is left behind.
template <typename T>
__device__ __forceinline__ void k_small_fold2_impl(const SmallArgs& a) {
  extern __shared__ double ssm[];
  const int kv = small_kv(a.kA, 0);
  const SmallSmem m = small_smem(ssm, kv);
  double* gram = m.v0;  // reduced Gram dots (rows > off)
  double* sgA = m.v1;
  double* rowA = m.v2;  // W_F[off, j]
  double* gcol = m.v3;  // new G column
  double* tcol = m.v4;
  T* rowT = reinterpret_cast<T*>(m.v5);
  const int tid = threadIdx.x;
  double* tsA = m.sc + 16;
  double* ps = tsA + (a.stageA ? (size_t)a.kA * (a.kA | 1) : 0);  // [nslots_in][nblk]
  int* st = reinterpret_cast<int*>(m.sc + 12);
  const T* PA = (const T*)a.PA;
  // ---- phase 1: what earlier launches wrote before griddepcontrol.wait
  const TView tvA = a.stageA ? st_stage_T(a.chA, a.kA, tsA, tid, kSmallThreads) : TView{a.chA.Tm, a.chA.K};
  #pragma unroll 1
  for (int j = tid; j < a.kA; j += kSmallThreads) {
    cp_async8(sgA + j, a.chA.sig + j);
    cp_async_elem(rowT + j, PA + paddr(a.off, j, a.chA.K));
  }
  if (tid == 0) {
    cp_async8(m.sc + 8, a.scal + kScEscale);
    cp_async8(m.sc + 9, a.scal + kScIscale);
  }
  pdl_wait();
  if (!a.late_launch) pdl_launch();
  st_stage(a.partials, (int64_t)a.nslots_in * a.nblk, ps, tid, kSmallThreads);
  if (tid == 0) {
    cp_async8(m.sc + 1, a.head + a.off);
    cp_async4(st, a.status + kStAbort);
  }
  cp_async_wait_all();
  __syncthreads();
  if (st[0] != 0) return;
  #pragma unroll 1
  for (int t = tid; t <= a.kA; t += kSmallThreads) {
    if (t < a.kA) {
      gram[t] = st_sum_slot(ps, a.nblk, a.slotA_pend + t);
      rowA[t] = (double)rowT[t];
    } else {
      m.sc[0] = sqrt(st_sum_slot(ps, a.nblk, a.fold_slot_ss));
    }
  }
  __syncthreads();
  const double nrm = m.sc[0], piv = m.sc[1];
  if (tid == 0) {
    const double sign = st_reflector<T>(a.chA, (T*)a.PA, a.kA, a.off, nrm, piv, a.rule, m.sc[8], m.sc[9],
                                        a.append != 0);
    const double zoff = (nrm == 0.0) ? piv : (sign == 0.0 ? 0.0 : nrm);
    a.scal[kScNrm] = nrm;
    a.scal[kScCoefCur] = a.append ? zoff : piv;
    a.scal[kScSign] = sign;
    m.sc[3] = sign;
    m.sc[4] = (nrm == 0.0) ? 0.0 : (double)(T)((piv + sign * nrm) * m.sc[8]);  // the stored pivot entry
    m.sc[5] = (nrm == 0.0) ? 0.0 : m.sc[9] / nrm;                              // sig of the new column
    m.sc[6] = (nrm == 0.0) ? 0.0 : a.chA.c[a.kA];
  }
  __syncthreads();
  if (a.append && nrm != 0.0) st_D_update(a.chA, a.off, -m.sc[3], tid, kSmallThreads);
  const double wfix = m.sc[4], signew = m.sc[5], cnew = m.sc[6];
  const int k = a.kA;
  #pragma unroll 1
  for (int j = tid; j < k; j += kSmallThreads) {
    gcol[j] = sgA[j] * signew * (gram[j] + rowA[j] * wfix);
    a.chA.G[j + (int64_t)k * a.chA.K] = gcol[j];
  }
  if (tid == 0) a.chA.G[k + (int64_t)k * a.chA.K] = (nrm == 0.0) ? 0.0 : 2.0 / cnew;
  __syncthreads();
  st_T_column(a.chA, tvA, k, cnew, gcol, tcol, 0, kSmallThreads / 32);
}
template <typename T>
__global__ void __launch_bounds__(kSmallThreads) k_small_fold2(const __grid_constant__ SmallArgs a) {
  k_small_fold2_impl<T>(a);
}
template <typename T>
__global__ void __launch_bounds__(kSmallThreads) k_small_fold2_b(const SmallArgs* __restrict__ argv) {
  k_small_fold2_impl<T>(argv[blockIdx.y]);
}

// The two single-CTA stages between the passes of a two-pass Ginibre probe in ONE
// launch of two CTAs: CTA 0 the fold stage (chain F, the reflector scalars), CTA 1 the
// output-side stage (chain O, the coefficients; its draw dots were taken a probe earlier).
// They share no data: the fold stage touches chain F / scal / the fold pass's partials,
// the output-side stage chain O / csp / head / beta1, beta3, coefS.
struct SmallPair {
  SmallArgs f, g;
};
template <typename T>
__global__ void __launch_bounds__(kSmallThreads) k_small_fold2_gin(const __grid_constant__ SmallPair a) {
  if (blockIdx.x == 0)
    k_small_fold2_impl<T>(a.f);
  else
    k_small_gin_impl<T>(a.g);
}
template <typename T>
__global__ void __launch_bounds__(kSmallThreads) k_small_fold2_gin_b(const SmallPair* __restrict__ argv) {
  if (blockIdx.x == 0)
    k_small_fold2_impl<T>(argv[blockIdx.y].f);
  else
    k_small_gin_impl<T>(argv[blockIdx.y].g);
}

// Normalize dynamics: inv = ||y|| > 0 ? 1/||y|| : 1 (bench.cpp:25-28).
struct NormArgs {
  const double* partials = nullptr;
  int nblk = 0;
  double* scal = nullptr;
  int* status = nullptr;
  int step = 0;
};

__device__ __forceinline__ void k_small_norm_impl(const NormArgs& na) {
  const double* partials = na.partials;
  const int nblk = na.nblk;
  double* scal = na.scal;
  int* status = na.status;
  const int step = na.step;
  pdl_wait();
  pdl_launch();
  if (aborted(status)) return;
  __shared__ double ws[kSmallThreads / 32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v = 0.0;
  for (int b = threadIdx.x; b < nblk; b += kSmallThreads) v += partials[b];
  v = warp_sum(v);
  if (lane == 0) ws[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int u = 0; u < kSmallThreads / 32; ++u) t += ws[u];
    const double nrm = sqrt(t);
    const double inv = nrm > 0.0 ? 1.0 / nrm : 1.0;
    scal[kScInv] = inv;
    if (!isfinite(inv)) {
      atomicMin(status + kStBadStep, step);
      atomicOr(status + kStAbort, 1);
    }
  }
}
__global__ void __launch_bounds__(kSmallThreads) k_small_norm(const __grid_constant__ NormArgs a) { k_small_norm_impl(a); }
__global__ void __launch_bounds__(kSmallThreads) k_small_norm_b(const NormArgs* __restrict__ argv) {
  k_small_norm_impl(argv[blockIdx.y]);
}

// Reduction stage of the app maps (kEpiAmp*, kEpiSpike): the per-block
// partial sums of the output pass, summed in fixed order (deterministic),
// turned into the scalar the next probe's epilogue reads.
enum AppStage : int { kAppTh = 0, kAppOns = 1, kAppSpike = 2, kAppSpikeInit = 3, kAppSum = 4 };
struct AppArgs {
  const double* partials = nullptr;  // [nblk][nred]
  int nblk = 0, nred = 1, stage = 0;
  double alpha = 0.0;   // AMP alpha / spike theta
  double dimA = 1.0;    // AMP: m (threshold) or n (Onsager, MSE); spike: unused
  double delta = 1.0;   // AMP: m / n
  double* out = nullptr;  // mse[t] / overlap[t] (optional)
  double* scal = nullptr;
  int* status = nullptr;
  int step = 0;
  // partials layout: [block][nred] (k_ginout epilogue) or, when strided,
  // group partials [slot0 + r][nblk] (two-pass Ginibre output pass)
  int strided = 0, slot0 = 0;
};

__device__ __forceinline__ void k_app_scalars_impl(const AppArgs& a) {
  pdl_wait();
  pdl_launch();
  if (aborted(a.status)) return;
  __shared__ double ws[2][kSmallThreads / 32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v0 = 0.0, v1 = 0.0;
  for (int b = threadIdx.x; b < a.nblk; b += kSmallThreads) {
    if (a.strided) {
      v0 += a.partials[(size_t)a.slot0 * a.nblk + b];
      if (a.nred > 1) v1 += a.partials[(size_t)(a.slot0 + 1) * a.nblk + b];
    } else {
      v0 += a.partials[(size_t)b * a.nred];
      if (a.nred > 1) v1 += a.partials[(size_t)b * a.nred + 1];
    }
  }
  v0 = warp_sum(v0);
  v1 = warp_sum(v1);
  if (lane == 0) {
    ws[0][w] = v0;
    ws[1][w] = v1;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double s0 = 0.0, s1 = 0.0;
  for (int u = 0; u < kSmallThreads / 32; ++u) {
    s0 += ws[0][u];
    s1 += ws[1][u];
  }
  bool bad = false;
  if (a.stage == kAppTh) {  // tau_t: alpha ||z|| / sqrt(m)
    const double th = a.alpha * sqrt(s0) / sqrt(a.dimA);
    a.scal[kScAppA] = th;
    bad = !isfinite(th);
  } else if (a.stage == kAppOns) {  // Onsager b = (nnz / n) / delta; mse = ||x - beta||^2 / n
    a.scal[kScAppB] = (s0 / a.dimA) / a.delta;
    if (a.out) a.out[0] = s1 / a.dimA;
  } else if (a.stage == kAppSpike) {  // x_{t+1} = g / ||g||; next coefficient theta <u, x_{t+1}>
    const double nr = sqrt(s0);
    const double inv = nr > 0.0 ? 1.0 / nr : 1.0;
    const double ux = s1 * inv;
    a.scal[kScInv] = inv;
    a.scal[kScAppA] = a.alpha * ux;
    if (a.out) a.out[0] = ux;
    bad = !isfinite(inv) || !isfinite(ux);
  } else if (a.stage == kAppSpikeInit) {  // theta <u, x_1>
    a.scal[kScAppA] = a.alpha * s0;
    a.scal[kScInv] = 1.0;
  } else {  // kAppSum: this shard's sums, for the exchange (row-sharded runs)
    a.out[0] = s0;
    a.out[1] = s1;
  }
  if (bad) {
    atomicMin(a.status + kStBadStep, a.step);
    atomicOr(a.status + kStAbort, 1);
  }
}
__global__ void __launch_bounds__(kSmallThreads) k_app_scalars(const __grid_constant__ AppArgs a) { k_app_scalars_impl(a); }

// Per-block partial sums of <u, x> (n rows; grid-stride; one partial per block).
template <typename T>
__global__ void __launch_bounds__(256) k_dot_blocks(const T* u, const T* x, int64_t n, double* partials) {
  pdl_wait();
  pdl_launch();
  __shared__ double red[32];
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v += (double)u[i] * (double)x[i];
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = v;
}

// x = scale * y (materialise a lazily normalised iterate).
template <typename T>
__global__ void k_scale_copy(const T* y, const double* scale, T* x, int64_t n) {
  pdl_wait();
  pdl_launch();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = (T)(*scale * (double)y[i]);
}

// ---------------------------------------------------- standalone reflector
// make_reflector(p, offset, zero_tol, rule) + Reflector::apply on `count`
// vectors (reflect.hpp:70-83,120-176; bindings module.cpp:48-66). One CTA;
// norms are scaled by the largest magnitude (the stableNorm branch of
// reflect.hpp:132-136), so inputs at 1e-300 .. 1e290 stay finite.
constexpr int kReflThreads = 1024;

__device__ double block_max(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int u = 0; u < kReflThreads / 32; ++u) t = fmax(t, sh[u]);
  __syncthreads();
  return t;
}

__device__ double scaled_norm(const double* x, int64_t n, double* sh) {
  double mx = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kReflThreads) mx = fmax(mx, fabs(x[i]));
  const double scale = block_max(mx, sh);
  if (scale == 0.0 || !isfinite(scale)) return scale;
  double ss = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kReflThreads) {
    const double v = x[i] / scale;
    ss += v * v;
  }
  return scale * sqrt(block_sum<kReflThreads>(ss, sh));
}

__global__ void __launch_bounds__(kReflThreads) k_reflector(const double* p, int64_t n, int64_t off, double zero_tol,
                                                            int rule, const double* x, double* y, int64_t count,
                                                            double* info) {
  __shared__ double sh[32];
  const int64_t len = n - off;
  const double* tail = p + off;
  const double nrm = scaled_norm(tail, len, sh);
  bool ident = (nrm == 0.0);
  if (!ident && zero_tol > 0.0) ident = nrm <= zero_tol * scaled_norm(p, n, sh);
  const double v1 = tail[0];
  double sign = 1.0;
  if (rule == 0) sign = (v1 >= 0.0) ? 1.0 : -1.0;
  else if (rule == 1) sign = (v1 > 0.0) ? 1.0 : -1.0;
  else sign = (v1 >= 0.0) ? 1.0 : 0.0;
  double c = 0.0, s = 1.0;
  if (!ident) {
    double a2 = 0.0;
    for (int64_t i = threadIdx.x; i < len; i += kReflThreads) {
      const double ai = tail[i] / nrm + (i == 0 ? sign : 0.0);
      a2 += ai * ai;
    }
    a2 = block_sum<kReflThreads>(a2, sh);
    c = 2.0 / a2;
    s = -sign;
  }
  if (threadIdx.x == 0 && info) {
    info[0] = c;
    info[1] = s;
    info[2] = ident ? 1.0 : 0.0;
  }
  for (int64_t v = 0; v < count; ++v) {
    const double* xv = x + v * n;
    double* yv = y + v * n;
    for (int64_t i = threadIdx.x; i < off; i += kReflThreads) yv[i] = xv[i];
    if (ident) {
      for (int64_t i = threadIdx.x; i < len; i += kReflThreads) yv[off + i] = xv[off + i];
      continue;
    }
    double proj = 0.0;
    for (int64_t i = threadIdx.x; i < len; i += kReflThreads)
      proj += (tail[i] / nrm + (i == 0 ? sign : 0.0)) * xv[off + i];
    proj = block_sum<kReflThreads>(proj, sh);
    const double cp = c * proj;
    for (int64_t i = threadIdx.x; i < len; i += kReflThreads) {
      const double ai = tail[i] / nrm + (i == 0 ? sign : 0.0);
      yv[off + i] = (xv[off + i] - cp * ai) * s;
    }
  }
}

__device__ __forceinline__ void k_reset_chain_impl(const ChainDev& ch) {
  pdl_wait();
  pdl_launch();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ch.Dlen; i += (int64_t)gridDim.x * blockDim.x)
    ch.Drow[i] = 1.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) *ch.Dtail = 1.0;
}
__global__ void k_reset_chain(ChainDev ch) { k_reset_chain_impl(ch); }
__global__ void k_reset_chain_b(const ChainDev* __restrict__ argv) { k_reset_chain_impl(argv[blockIdx.y]); }

// The PHILOX draw stream itself: out[i] = draw i of probe `probe`
// (hd_philox_normals; the same function the streaming kernels evaluate).
__global__ void k_philox_normals(uint64_t seed, uint32_t stream, uint32_t probe, int64_t n, double* out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; 2 * q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = philox_normal_pair(seed, stream, probe, (uint64_t)q);
    out[2 * q] = v.x;
    if (2 * q + 1 < n) out[2 * q + 1] = v.y;
  }
}

__device__ __forceinline__ void k_reset_status_impl(int* status) {
  pdl_wait();
  pdl_launch();
  if (threadIdx.x == 0) {
    status[kStAbort] = 0;
    status[kStBadStep] = INT_MAX;
    status[kStBadInput] = 0;
    status[3] = 0;  // kStFused (hd_fused.cuh)
  }
}
__global__ void k_reset_status(int* status) { k_reset_status_impl(status); }
__global__ void k_reset_status_b(int* const* __restrict__ argv) { k_reset_status_impl(argv[blockIdx.y]); }

}  // namespace hd
