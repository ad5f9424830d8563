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
constexpr int kRing = 3;
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

// Stage `it` of a warp's stream -> (tile, job, chunk) given per-job chunk
// counts; the stream is tile-major, then job, then chunk.
struct StreamPos {
  int64_t tile;
  int job, chunk;
};

__device__ __forceinline__ StreamPos stream_pos(int64_t t0, uint32_t it, int nch0, int nch1) {
  const int per = nch0 + nch1;
  StreamPos p;
  p.tile = t0 + it / per;
  const int r = (int)(it % per);
  p.job = (r < nch0) ? 0 : 1;
  p.chunk = (r < nch0) ? r : r - nch0;
  return p;
}

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
  DotJob<T> job[2];
  int njobs = 1;
  int64_t n = 0, ntiles = 0;
  Flush out;
  int nslots = 0;
  int* status = nullptr;
};

// Shared-memory carve-up of the streaming kernels (per warp: ring + slots).
template <typename T>
__host__ __device__ constexpr size_t ring_bytes() {
  return (size_t)kRing * kCW * kTile * sizeof(T);
}

// GEMV-T a = P^T v (k_dots). Lane l holds rows 2(l + 32q) + {0, 1} of the
// current tile's right-hand side(s); each 4-column chunk costs 16 LDS.128,
// 32 (or 64 with a pending column) DFMA and one 4-way butterfly.
template <typename T>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) k_dots(const __grid_constant__ DotArgs<T> a) {
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
  const bool skip = aborted(a.status);
  const int64_t W = (int64_t)gridDim.x * nw;
  const int64_t gw = (int64_t)blockIdx.x * nw + w;
  const int64_t t0 = gw * a.ntiles / W, t1 = skip ? t0 : (gw + 1) * a.ntiles / W;
  const int nch0 = (a.job[0].ncols + kCW - 1) / kCW;
  const int nch1 = (a.njobs > 1) ? (a.job[1].ncols + kCW - 1) / kCW : 0;
  const uint32_t nst = (uint32_t)((t1 - t0) * (nch0 + nch1));
  auto issue = [&](uint32_t it) {
    const StreamPos p = stream_pos(t0, it, nch0, nch1);
    const DotJob<T>& J = a.job[p.job];
    const int nc = min(kCW, J.ncols - p.chunk * kCW);
    const uint32_t bytes = (uint32_t)(nc * kTile * sizeof(T));
    const int s = it % kRing;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot precede the refill
    mbar_arrive_expect_tx(full + s, bytes);
    bulk_g2s(ring + (size_t)s * kCW * kTile * sizeof(T),
             J.P + (size_t)p.tile * (size_t)(J.K << kTileShift) + (size_t)p.chunk * kCW * kTile, bytes, full + s);
  };
  if (lane == 0)
    for (uint32_t it = 0; it < (uint32_t)kRing && it < nst; ++it) issue(it);

  double ss0 = 0.0, ss1 = 0.0;
  bool bad = false;
  double2 x[4], pv[4];
  uint32_t it = 0;
  for (int64_t tile = t0; tile < t1; ++tile) {
    for (int jb = 0; jb < a.njobs; ++jb) {
      const DotJob<T>& J = a.job[jb];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t i = tile * kTile + 2 * (lane + 32 * q);
        x[q] = src_pair(J.rhs, i, a.n);
        const double sq = x[q].x * x[q].x + x[q].y * x[q].y;
        if (jb == 0) ss0 += sq;
        else ss1 += sq;
        if (J.check_finite) bad |= !(isfinite(x[q].x) && isfinite(x[q].y));
        if (J.pivot_out && (i == J.pivot_row || i + 1 == J.pivot_row)) *J.pivot_out = (i == J.pivot_row) ? x[q].x : x[q].y;
        if (J.wcol) st_pair(J.wcol + paddr(i, J.wj, J.wK), x[q].x, x[q].y);
        pv[q] = (J.pend >= 0) ? ld_pair(J.P + paddr(i, J.pend, J.K)) : make_double2(0.0, 0.0);
      }
      const int nch = (J.ncols + kCW - 1) / kCW;
      for (int c = 0; c < nch; ++c, ++it) {
        const int s = it % kRing;
        mbar_wait(full + s, (it / kRing) & 1);
        const T* sp = reinterpret_cast<const T*>(ring + (size_t)s * kCW * kTile * sizeof(T)) + 2 * lane;
        double d[kCW], e[kCW];
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
        __syncwarp();
        if (lane == 0 && it + kRing < nst) issue(it + kRing);
        const int col0 = c * kCW;
        const double f = warp_sum4(d[0], d[1], d[2], d[3], lane);
        const int u = lane >> 3;
        if ((lane & 7) == 0 && col0 + u < J.ncols) acc[J.slot_dot + col0 + u] += f;
        if (J.pend >= 0 && col0 <= J.pend) {
          const double g = warp_sum4(e[0], e[1], e[2], e[3], lane);
          if ((lane & 7) == 0 && col0 + u <= J.pend) acc[J.slot_pend + col0 + u] += g;
        }
      }
    }
  }
  ss0 = warp_sum(ss0);
  ss1 = warp_sum(ss1);
  if (lane == 0) {
    if (a.job[0].slot_sumsq >= 0) acc[a.job[0].slot_sumsq] += ss0;
    if (a.njobs > 1 && a.job[1].slot_sumsq >= 0) acc[a.job[1].slot_sumsq] += ss1;
  }
  if (bad) atomicOr(a.status + kStBadInput, 1);
  __syncthreads();
  for (int s = threadIdx.x; s < a.nslots; s += blockDim.x) {
    double v = 0.0;
    for (int u = 0; u < nw; ++u) v += accs[(size_t)u * nsl + s];
    accs[s] = v;  // row 0 (each slot owned by one thread here)
  }
  flush_row(accs, a.nslots, a.out);
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
enum EpiKind : int { kEpiPlain = 0, kEpiNormalize = 1, kEpiTanhMix = 2 };

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
  double* partials = nullptr;     // normalize: per-block sum of squares
  int step = 0;
};

template <typename T>
__device__ __forceinline__ void epilogue(const Epi<T>& e, int* status, int64_t i, int64_t n, double2 v,
                                         double* red_s) {
  double ss = 0.0;
  bool bad = false;
  if (i < n) {
    if (e.yadd) {
      double2 ya;
      if (i + 1 < n) {
        if constexpr (sizeof(T) == 8) ya = *reinterpret_cast<const double2*>(e.yadd + i);
        else { const float2 f = *reinterpret_cast<const float2*>(e.yadd + i); ya = make_double2(f.x, f.y); }
      } else {
        ya = make_double2((double)e.yadd[i], 0.0);
      }
      v.x = (ya.x + v.x) * e.add_scale;
      v.y = (ya.y + v.y) * e.add_scale;
    }
    if (i + 1 >= n) v.y = 0.0;
    if (e.kind == kEpiTanhMix) {
      double2 xp = make_double2(0.0, 0.0);
      if (e.xprev) {
        if constexpr (sizeof(T) == 8) xp = *reinterpret_cast<const double2*>(e.xprev + i);
        else { const float2 f = *reinterpret_cast<const float2*>(e.xprev + i); xp = make_double2(f.x, f.y); }
        if (e.xprev_scale) { xp.x *= *e.xprev_scale; xp.y *= *e.xprev_scale; }
      }
      const double a = tanh(2.0 * v.x) + 0.1 * xp.x;
      const double b = (i + 1 < n) ? tanh(2.0 * v.y) + 0.1 * xp.y : 0.0;
      st_pair_guard(e.xnext, i, n, a, b);
      bad = !(isfinite(a) && isfinite(b));
    } else {
      bad = !(isfinite(v.x) && isfinite(v.y));
      ss = v.x * v.x + v.y * v.y;
    }
    if (e.y) st_pair_guard(e.y, i, n, v.x, v.y);
  }
  if (bad) {
    atomicMin(status + kStBadStep, e.step);
    atomicOr(status + kStAbort, 1);
  }
  if (e.kind == kEpiNormalize) {
    const double t = block_sum<kUpdThreads>(ss, red_s);
    if (threadIdx.x == 0) e.partials[blockIdx.x] = t;
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
  int slot_ss = 0;    // fold: ||p[off:]||^2; other: ||y||^2
  Flush out;
  int nslots = 0;
  int* status = nullptr;
};

template <typename T, int MODE>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) k_apply(const __grid_constant__ ApplyArgs<T> a) {
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
  for (int j = threadIdx.x; j < a.ncols; j += blockDim.x) beta_s[j] = a.beta[j];
  for (int s = lane; s < nsl; s += 32) acc[s] = 0.0;
  if (lane == 0) {
    for (int s = 0; s < kRing; ++s) mbar_init(full + s, 1);
    mbar_fence_init();
  }
  __syncthreads();
  const bool skip = aborted(a.status);
  const bool spec = (a.spec.kind != kSrcNone);
  const int64_t W = (int64_t)gridDim.x * nw;
  const int64_t gw = (int64_t)blockIdx.x * nw + w;
  const int64_t t0 = gw * a.ntiles / W, t1 = skip ? t0 : (gw + 1) * a.ntiles / W;
  const int nch = (a.ncols + kCW - 1) / kCW;
  const uint32_t nst = (uint32_t)((t1 - t0) * nch);
  auto issue = [&](uint32_t it) {
    const int64_t tile = t0 + it / nch;
    const int c = (int)(it % nch);
    const int nc = min(kCW, a.ncols - c * kCW);
    const uint32_t bytes = (uint32_t)(nc * kTile * sizeof(T));
    const int s = it % kRing;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(full + s, bytes);
    bulk_g2s(ring + (size_t)s * kCW * kTile * sizeof(T),
             a.P + (size_t)tile * (size_t)(a.K << kTileShift) + (size_t)c * kCW * kTile, bytes, full + s);
  };
  if (lane == 0)
    for (uint32_t it = 0; it < (uint32_t)kRing && it < nst; ++it) issue(it);

  double ss = 0.0;
  bool bad = false;
  uint32_t it = 0;
  for (int64_t tile = t0; tile < t1; ++tile) {
    double2 g[4], r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      g[q] = spec ? src_pair(a.spec, tile * kTile + 2 * (lane + 32 * q), a.n) : make_double2(0.0, 0.0);
      r[q] = make_double2(0.0, 0.0);
    }
    for (int c = 0; c < nch; ++c, ++it) {
      const int s = it % kRing;
      mbar_wait(full + s, (it / kRing) & 1);
      const T* sp = reinterpret_cast<const T*>(ring + (size_t)s * kCW * kTile * sizeof(T)) + 2 * lane;
      const int col0 = c * kCW;
      double d[kCW];
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
      __syncwarp();
      if (lane == 0 && it + kRing < nst) issue(it + kRing);
      if (spec) {
        const double f = warp_sum4(d[0], d[1], d[2], d[3], lane);
        const int u = lane >> 3;
        if ((lane & 7) == 0 && col0 + u < a.ncols) acc[a.slot_spec + col0 + u] += f;
      }
    }
    // epilogue on the lane's 8 rows
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = tile * kTile + 2 * (lane + 32 * q);
      const double d0 = (i < a.Dlen) ? a.D[i] : *a.Dtail;
      const double d1 = (i + 1 < a.Dlen) ? a.D[i + 1] : *a.Dtail;
      if constexpr (MODE == kApplyFold) {
        const double2 xv = src_pair(a.x, i, a.n);
        const double p0 = (i < a.n) ? d0 * (xv.x - r[q].x) : 0.0;
        const double p1 = (i + 1 < a.n) ? d1 * (xv.y - r[q].y) : 0.0;
        const double c0 = (i >= a.off) ? p0 : 0.0, c1 = (i + 1 >= a.off) ? p1 : 0.0;
        const double es = *a.escale;
        st_pair(a.Pw + paddr(i, a.newj, a.K), c0 * es, c1 * es);
        if (i <= a.off) a.head[i] = p0;
        if (i + 1 <= a.off) a.head[i + 1] = p1;
        ss += c0 * c0 + c1 * c1;
      } else {
        double z0 = 0.0, z1 = 0.0;
        if (i < a.zlen) z0 = d0 * a.z[i];
        if (i + 1 < a.zlen) z1 = d1 * a.z[i + 1];
        double2 y = make_double2(z0 - r[q].x, z1 - r[q].y);
        const Epi<T>& e = a.epi;
        if (i < a.n) {
          if (i + 1 >= a.n) y.y = 0.0;
          if (e.kind == kEpiTanhMix) {
            double2 xp = make_double2(0.0, 0.0);
            if (e.xprev) {
              xp.x = (double)e.xprev[i];
              if (i + 1 < a.n) xp.y = (double)e.xprev[i + 1];
              if (e.xprev_scale) {
                xp.x *= *e.xprev_scale;
                xp.y *= *e.xprev_scale;
              }
            }
            const double o0 = tanh(2.0 * y.x) + 0.1 * xp.x;
            const double o1 = (i + 1 < a.n) ? tanh(2.0 * y.y) + 0.1 * xp.y : 0.0;
            st_pair_guard(e.xnext, i, a.n, o0, o1);
            bad |= !(isfinite(o0) && isfinite(o1));
          } else {
            bad |= !(isfinite(y.x) && isfinite(y.y));
            ss += y.x * y.x + y.y * y.y;
          }
          if (e.y) st_pair_guard(e.y, i, a.n, y.x, y.y);
        }
      }
    }
  }
  ss = warp_sum(ss);
  if (lane == 0) acc[a.slot_ss] += ss;
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
  int* status = nullptr;
  Epi<T> epi;
};

template <typename T>
__global__ void __launch_bounds__(kUpdThreads) k_ginout(const __grid_constant__ GinArgs<T> a) {
  extern __shared__ double beta_s[];  // [3][K]
  __shared__ double red_s[32];
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
  const int64_t tile = blockIdx.x;
  const int64_t i = tile * kTile + 2 * threadIdx.x;
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
  st_pair(a.Sw + paddr(i, a.newj, a.KS), u0, u1);
  double c0 = 0.0, c1 = 0.0;
  if (i < a.csplen) c0 = dval(a.D, a.Dtail, a.Dlen, i) * a.csp[i];
  if (i + 1 < a.csplen) c1 = dval(a.D, a.Dtail, a.Dlen, i + 1) * a.csp[i + 1];
  const double cc = *a.coef_cur;
  const double y0 = a.sigma * (accS.x + cc * u0 + (c0 - acc[1].x));
  const double y1 = a.sigma * (accS.y + cc * u1 + (c1 - acc[1].y));
  epilogue(a.epi, a.status, i, a.n, make_double2(y0, y1), red_s);
}

// ======================================================= small kernels
constexpr int kSmallThreads = 512;

// Deterministic sum over blocks: red[s] = sum_b partials[b][s].
__device__ void sm_reduce(const double* partials, int nblk, int nslots, double* red) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int s = w; s < nslots; s += kSmallThreads / 32) {
    double v = 0.0;
    const double* ps = partials + (size_t)s * nblk;
    for (int b = lane; b < nblk; b += 32) v += ps[b];
    v = warp_sum(v);
    if (lane == 0) red[s] = v;
  }
  __syncthreads();
}

// T_new[:k, k] = -c_k T[:k, :k] g  (g = G[:k, k]); warp per row, lanes
// split the reduction so every load is independent (no serial chains).
__device__ void sm_T_column(const ChainDev& ch, int k, double ck) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* g = ch.G + (int64_t)k * ch.K;
  for (int i = w; i < k; i += kSmallThreads / 32) {
    double v = 0.0;
    for (int l = i + lane; l < k; l += 32) v += ch.Tm[i + (int64_t)l * ch.K] * g[l];
    v = warp_sum(v);
    if (lane == 0) ch.Tm[i + (int64_t)k * ch.K] = -ck * v;
  }
  if (threadIdx.x == 0) ch.Tm[k + (int64_t)k * ch.K] = ck;
  __syncthreads();
}

// Gram column + T column of a pending reflector (Schreiber-Van Loan):
// T_new[:k, k] = -c_k T[:k, :k] G[:k, k], T_new[k, k] = c_k.
__device__ void sm_finalize_pending(const ChainDev& ch, int pend, const double* rdots) {
  const int64_t K = ch.K;
  const double sp = ch.sig[pend];
  for (int j = threadIdx.x; j <= pend; j += kSmallThreads) ch.G[j + pend * K] = ch.sig[j] * sp * rdots[j];
  __syncthreads();
  sm_T_column(ch, pend, ch.c[pend]);
}

// out = T^T a (k x k upper T): warp per output column.
__device__ void sm_Tt(const ChainDev& ch, int k, const double* a, double* out) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = w; j < k; j += kSmallThreads / 32) {
    double v = 0.0;
    for (int i = lane; i <= j; i += 32) v += ch.Tm[i + (int64_t)j * ch.K] * a[i];
    v = warp_sum(v);
    if (lane == 0) out[j] = v;
  }
  __syncthreads();
}

// out = T a: warp per output row, lanes split the row.
__device__ void sm_T(const ChainDev& ch, int k, const double* a, double* out) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = w; i < k; i += kSmallThreads / 32) {
    double v = 0.0;
    for (int j = i + lane; j < k; j += 32) v += ch.Tm[i + (int64_t)j * ch.K] * a[j];
    v = warp_sum(v);
    if (lane == 0) out[i] = v;
  }
  __syncthreads();
}

// out_j = sig_j * sum_{i < len} P[i, j] D(i) v[i]  (sparse-input corner).
template <typename T>
__device__ void sm_corner(const ChainDev& ch, const T* P, int k, const double* v, int64_t len, double* out) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = w; j < k; j += kSmallThreads / 32) {
    double acc = 0.0;
    for (int64_t i = lane; i < len; i += 32) acc += (double)P[paddr(i, j, ch.K)] * dval(ch.Drow, ch.Dtail, ch.Dlen, i) * v[i];
    acc = warp_sum(acc);
    if (lane == 0) out[j] = ch.sig[j] * acc;
  }
  __syncthreads();
}

// make_reflector (reflect.hpp:120-176) on the device, for a column whose
// tail has already been streamed into the panel: pivot fix-up, scale,
// coefficient, leading factor and the D update (for i >= off: D *= s).
// Returns the sign used (0 for the negative-control rule's zeroing case).
template <typename T>
__device__ double sm_make_reflector(const ChainDev& ch, T* P, int j, int64_t off, double nrm, double pivot,
                                    int rule, double colscale, double unscale, bool append, double* sign_out) {
  __shared__ double s_sign;
  if (threadIdx.x == 0) {
    double sign;
    if (rule == 0) sign = (pivot >= 0.0) ? 1.0 : -1.0;
    else if (rule == 1) sign = (pivot > 0.0) ? 1.0 : -1.0;
    else sign = (pivot >= 0.0) ? 1.0 : 0.0;
    if (nrm == 0.0) sign = 1.0;
    s_sign = sign;
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
  }
  __syncthreads();
  const double sign = s_sign;
  if (append && nrm != 0.0) {
    const double s = -sign;
    for (int64_t i = off + threadIdx.x; i < ch.Dlen; i += kSmallThreads) ch.Drow[i] *= s;
    if (threadIdx.x == 0) *ch.Dtail *= s;
  }
  if (sign_out) *sign_out = sign;
  __syncthreads();
  return sign;
}

// Append a column whose Gram column is known now (Haar mix reflector):
// G[:k, k] from the streamed dots, then the T column.
__device__ void sm_append_known_gram(const ChainDev& ch, int k, const double* G_col /*[k+1]*/) {
  for (int j = threadIdx.x; j <= k; j += kSmallThreads) ch.G[j + (int64_t)k * ch.K] = G_col[j];
  __syncthreads();
  sm_T_column(ch, k, ch.c[k]);
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
  kScWords = 16,
};

struct SmallArgs {
  const double* partials = nullptr;
  int nblk = 0;
  int nslots = 0;
  double* red = nullptr;
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
  double* tmp = nullptr;   // [K] scratch
  double* tmp2 = nullptr;  // [K] scratch
  double* head = nullptr;  // p[0..off]
  double* zbuf = nullptr;
  double* csp = nullptr;
  int64_t csplen = 0;
  double* coefS = nullptr;
  int nS = 0;
  int is_haar = 0;
  // Haar mix Gram dots P_B^T g[off:]: from k_dots (red + slotB_dot) or from
  // the speculative pass of the previous probe (spec buffer)
  const double* mix_dots = nullptr;
  // reduce a previous k_apply(OTHER)'s speculative slots into spec_dst
  const double* spec_parts = nullptr;
  int spec_nblk = 0, spec_slot0 = 0, spec_count = 0;
  double* spec_dst = nullptr;
  // k_small_fold: ||p[off:]||^2 slot and speculative slots of k_apply(FOLD)
  int fold_slot_ss = 0;
  int fold_slot_spec = -1;
  double* fold_spec_dst = nullptr;
};

// dst[s] = sum_b parts[(slot0 + s) * nblk + b] for s < count (fixed order).
__device__ void sm_reduce_slots(const double* parts, int nblk, int slot0, int count, double* dst) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int s = w; s < count; s += kSmallThreads / 32) {
    const double* ps = parts + (size_t)(slot0 + s) * nblk;
    double v = 0.0;
    for (int b = lane; b < nblk; b += 32) v += ps[b];
    v = warp_sum(v);
    if (lane == 0) dst[s] = v;
  }
  __syncthreads();
}

// After k_dots of a probe (Haar and Ginibre "fold" side): finalise pending
// columns, the Haar mix reflector (chain B), the forward coefficients
// beta1 = sig (T^T (sig a)) for k_fold, the power-of-two column scale, and
// (Ginibre) the opposite-side sparse coefficients c.
template <typename T>
__global__ void __launch_bounds__(kSmallThreads) k_small_dots(const __grid_constant__ SmallArgs a) {
  if (aborted(a.status)) return;
  if (a.spec_parts) sm_reduce_slots(a.spec_parts, a.spec_nblk, a.spec_slot0, a.spec_count, a.spec_dst);
  sm_reduce(a.partials, a.nblk, a.nslots, a.red);
  if (threadIdx.x == 0 && *(volatile int*)(a.status + kStBadInput)) *(volatile int*)(a.status + kStAbort) = 1;
  __syncthreads();
  if (aborted(a.status)) return;
  if (a.pendA >= 0) sm_finalize_pending(a.chA, a.pendA, a.red + a.slotA_pend);
  if (a.pendB >= 0) sm_finalize_pending(a.chB, a.pendB, a.red + a.slotB_pend);
  // forward coefficients for the fold chain
  for (int j = threadIdx.x; j < a.kA; j += kSmallThreads) a.tmp[j] = a.chA.sig[j] * a.red[a.slotA_dot + j];
  __syncthreads();
  sm_Tt(a.chA, a.kA, a.tmp, a.tmp2);
  for (int j = threadIdx.x; j < a.kA; j += kSmallThreads) a.beta1[j] = a.chA.sig[j] * a.tmp2[j];
  if (threadIdx.x == 0) {
    const double xn = sqrt(a.red[a.slotA_ss]);
    int e = 0;
    if (xn > 0.0 && isfinite(xn)) frexp(xn, &e);
    a.scal[kScEscale] = ldexp(1.0, -e);
    a.scal[kScIscale] = ldexp(1.0, e);
  }
  if (a.is_haar) {
    // mix reflector H(g, off) appended to chain B at column kB
    const double nrm = sqrt(a.red[a.slotB_ss]);
    const double piv = a.scal[kScPivotG];
    double sign;
    sm_make_reflector<T>(a.chB, (T*)a.PB, a.kB, a.off, nrm, piv, a.rule, 1.0, 1.0, true, &sign);
    // Gram column: G[j, kB] = sig_j (P[:,j].g_tail / nrm + sign P[off, j])
    const T* PB = (const T*)a.PB;
    for (int j = threadIdx.x; j < a.kB; j += kSmallThreads) {
      a.tmp[j] = (nrm == 0.0) ? 0.0
                              : a.chB.sig[j] * (a.mix_dots[j] / nrm + sign * (double)PB[paddr(a.off, j, a.chB.K)]);
    }
    if (threadIdx.x == 0) a.tmp[a.kB] = (nrm == 0.0) ? 0.0 : 2.0 / a.chB.c[a.kB];
    __syncthreads();
    sm_append_known_gram(a.chB, a.kB, a.tmp);
  } else {
    // Ginibre: opposite-side coefficients <v_i, x> (or <u_i, x>), rows < nB
    for (int q = threadIdx.x; q < a.kB; q += kSmallThreads) a.csp[q] = a.red[a.slotB_dot + q];
  }
}

// After k_fold: finalise the fold reflector H(p, off) (appended unless the
// skip fault fires), then either (Haar) the sparse reverse application of
// chain B to z = H p, or (Ginibre) the coefficient of the current probe.
template <typename T>
__global__ void __launch_bounds__(kSmallThreads) k_small_fold(const __grid_constant__ SmallArgs a) {
  if (aborted(a.status)) return;
  __shared__ double s_nrm;
  // deterministic sum of the per-block ||p[off:]||^2 partials
  {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ double ws[kSmallThreads / 32];
    const double* ps = a.partials + (size_t)a.fold_slot_ss * a.nblk;
    double v = 0.0;
    for (int b = threadIdx.x; b < a.nblk; b += kSmallThreads) v += ps[b];
    v = warp_sum(v);
    if (lane == 0) ws[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int u = 0; u < kSmallThreads / 32; ++u) t += ws[u];
      s_nrm = sqrt(t);
    }
    __syncthreads();
  }
  if (a.fold_slot_spec >= 0) sm_reduce_slots(a.partials, a.nblk, a.fold_slot_spec, a.kA + 1, a.fold_spec_dst);
  const double nrm = s_nrm;
  const double piv = a.head[a.off];
  double sign;
  sm_make_reflector<T>(a.chA, (T*)a.PA, a.kA, a.off, nrm, piv, a.rule, a.scal[kScEscale], a.scal[kScIscale],
                       a.append != 0, &sign);
  // (H p)[off]: +||p[off:]|| (0 under the zeroing negative control)
  const double zoff = (nrm == 0.0) ? piv : (sign == 0.0 ? 0.0 : nrm);
  if (threadIdx.x == 0) {
    a.scal[kScNrm] = nrm;
    a.scal[kScCoefCur] = a.append ? zoff : piv;
    a.scal[kScSign] = sign;
  }
  if (a.is_haar) {
    for (int64_t i = threadIdx.x; i <= a.off; i += kSmallThreads) a.zbuf[i] = (i < a.off) ? a.head[i] : zoff;
    __syncthreads();
    // beta = sig (T_B (W_B^T (D_B z)))
    sm_corner<T>(a.chB, (const T*)a.PB, a.kB, a.zbuf, a.off + 1, a.tmp);
    sm_T(a.chB, a.kB, a.tmp, a.tmp2);
    for (int j = threadIdx.x; j < a.kB; j += kSmallThreads) a.beta1[j] = a.chB.sig[j] * a.tmp2[j];
  }
}

// Ginibre, after k_dots over the opposite chain with v = D g_m: pending
// column, beta1 = sig (T (sig a_g)) for the new basis vector, beta3 for the
// sparse part L-rev-adj(c), and the coefficients of the same-side store.
template <typename T>
__global__ void __launch_bounds__(kSmallThreads) k_small_gin(const __grid_constant__ SmallArgs a) {
  if (aborted(a.status)) return;
  sm_reduce(a.partials, a.nblk, a.nslots, a.red);
  if (a.pendB >= 0) sm_finalize_pending(a.chB, a.pendB, a.red + a.slotB_pend);
  for (int j = threadIdx.x; j < a.kB; j += kSmallThreads) a.tmp[j] = a.chB.sig[j] * a.red[a.slotB_dot + j];
  __syncthreads();
  sm_T(a.chB, a.kB, a.tmp, a.tmp2);
  for (int j = threadIdx.x; j < a.kB; j += kSmallThreads) a.beta1[j] = a.chB.sig[j] * a.tmp2[j];
  __syncthreads();
  sm_corner<T>(a.chB, (const T*)a.PB, a.kB, a.csp, a.csplen, a.tmp);
  sm_T(a.chB, a.kB, a.tmp, a.tmp2);
  for (int j = threadIdx.x; j < a.kB; j += kSmallThreads) a.beta3[j] = a.chB.sig[j] * a.tmp2[j];
  // same-side store coefficients: column q <-> head p[q]
  for (int q = threadIdx.x; q < a.nS; q += kSmallThreads) a.coefS[q] = a.head[q];
}

// Normalize dynamics: inv = ||y|| > 0 ? 1/||y|| : 1 (bench.cpp:25-28).
__global__ void __launch_bounds__(kSmallThreads) k_small_norm(const double* partials, int nblk, double* scal,
                                                              int* status, int step) {
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

// x = scale * y (materialise a lazily normalised iterate).
template <typename T>
__global__ void k_scale_copy(const T* y, const double* scale, T* x, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = (T)(*scale * (double)y[i]);
}

__global__ void k_reset_chain(ChainDev ch) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ch.Dlen; i += (int64_t)gridDim.x * blockDim.x)
    ch.Drow[i] = 1.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) *ch.Dtail = 1.0;
}

__global__ void k_reset_status(int* status) {
  if (threadIdx.x == 0) {
    status[kStAbort] = 0;
    status[kStBadStep] = INT_MAX;
    status[kStBadInput] = 0;
  }
}

}  // namespace hd
