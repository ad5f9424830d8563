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
  double* partials = nullptr;  // [gridDim.x][nslots]
  int nslots = 0;
  int* status = nullptr;
};

// Each warp owns a contiguous run of 256-row tiles and streams every panel
// column of its tile once (4 x 16 B loads per lane per column, coalesced
// 2 KB per warp); per-column lane partials are warp-reduced and accumulated
// into the warp's own shared-memory slots, so no atomics are involved and
// the result is bitwise deterministic for a fixed grid.
template <typename T, int NW>
__global__ void __launch_bounds__(NW * 32) k_dots(const __grid_constant__ DotArgs<T> a) {
  extern __shared__ double acc_s[];
  if (aborted(a.status)) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* acc = acc_s + (size_t)w * a.nslots;
  for (int s = lane; s < a.nslots; s += 32) acc[s] = 0.0;
  __syncwarp();

  const int64_t W = (int64_t)gridDim.x * NW;
  const int64_t gw = (int64_t)blockIdx.x * NW + w;
  const int64_t t0 = gw * a.ntiles / W, t1 = (gw + 1) * a.ntiles / W;
  double ss[2] = {0.0, 0.0};
  bool bad = false;

  for (int64_t tile = t0; tile < t1; ++tile) {
    for (int jb = 0; jb < a.njobs; ++jb) {
      const DotJob<T>& J = a.job[jb];
      double2 x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t i = tile * kTile + 2 * (lane + 32 * q);
        x[q] = src_pair(J.rhs, i, a.n);
        ss[jb] += x[q].x * x[q].x + x[q].y * x[q].y;
        if (J.check_finite) bad |= !(isfinite(x[q].x) && isfinite(x[q].y));
        if (J.pivot_out && (i == J.pivot_row || i + 1 == J.pivot_row)) *J.pivot_out = (i == J.pivot_row) ? x[q].x : x[q].y;
        if (J.wcol) st_pair(J.wcol + paddr(i, J.wj, J.wK), x[q].x, x[q].y);
      }
      const T* base = J.P + (size_t)tile * (size_t)(J.K << kTileShift) + 2 * lane;
      if (J.pend >= 0) {
        double2 pv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) pv[q] = ld_pair(base + (size_t)J.pend * kTile + 64 * q);
        int j = 0;
        for (; j + 2 <= J.ncols; j += 2) {
          double2 w0[4], w1[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            w0[q] = ld_pair(base + (size_t)j * kTile + 64 * q);
            w1[q] = ld_pair(base + (size_t)(j + 1) * kTile + 64 * q);
          }
          double d0 = 0, d1 = 0, e0 = 0, e1 = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            d0 += w0[q].x * x[q].x + w0[q].y * x[q].y;
            d1 += w1[q].x * x[q].x + w1[q].y * x[q].y;
            e0 += w0[q].x * pv[q].x + w0[q].y * pv[q].y;
            e1 += w1[q].x * pv[q].x + w1[q].y * pv[q].y;
          }
          d0 = warp_sum(d0);
          d1 = warp_sum(d1);
          e0 = warp_sum(e0);
          e1 = warp_sum(e1);
          if (lane == 0) {
            acc[J.slot_dot + j] += d0;
            acc[J.slot_dot + j + 1] += d1;
            if (j <= J.pend) acc[J.slot_pend + j] += e0;
            if (j + 1 <= J.pend) acc[J.slot_pend + j + 1] += e1;
          }
        }
        for (; j < J.ncols; ++j) {
          double d0 = 0, e0 = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double2 w0 = ld_pair(base + (size_t)j * kTile + 64 * q);
            d0 += w0.x * x[q].x + w0.y * x[q].y;
            e0 += w0.x * pv[q].x + w0.y * pv[q].y;
          }
          d0 = warp_sum(d0);
          e0 = warp_sum(e0);
          if (lane == 0) {
            acc[J.slot_dot + j] += d0;
            if (j <= J.pend) acc[J.slot_pend + j] += e0;
          }
        }
      } else {
        int j = 0;
        for (; j + 4 <= J.ncols; j += 4) {
          double2 w[4][4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q) w[u][q] = ld_pair(base + (size_t)(j + u) * kTile + 64 * q);
          double d[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            d[u] = 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) d[u] += w[u][q].x * x[q].x + w[u][q].y * x[q].y;
            d[u] = warp_sum(d[u]);
          }
          if (lane == 0) {
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[J.slot_dot + j + u] += d[u];
          }
        }
        for (; j < J.ncols; ++j) {
          double d0 = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double2 w0 = ld_pair(base + (size_t)j * kTile + 64 * q);
            d0 += w0.x * x[q].x + w0.y * x[q].y;
          }
          d0 = warp_sum(d0);
          if (lane == 0) acc[J.slot_dot + j] += d0;
        }
      }
    }
  }
  for (int jb = 0; jb < a.njobs; ++jb) {
    const double v = warp_sum(ss[jb]);
    if (lane == 0 && a.job[jb].slot_sumsq >= 0) acc[a.job[jb].slot_sumsq] += v;
  }
  if (bad) atomicOr(a.status + kStBadInput, 1);
  __syncthreads();
  for (int s = threadIdx.x; s < a.nslots; s += NW * 32) {
    double v = 0.0;
#pragma unroll
    for (int u = 0; u < NW; ++u) v += acc_s[(size_t)u * a.nslots + s];
    a.partials[(size_t)blockIdx.x * a.nslots + s] = v;
  }
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

// ============================================================== k_fold
// p = D (x - P beta): the forward chain application of ginibre.hpp:68 /
// haar.hpp:55 in compact-WY form. Also writes the new reflector column
// (p[off:] times an exact power of two; the pivot is fixed once ||p[off:]||
// is known), keeps p[0..off] and the per-block sums of p[off:]^2.
template <typename T>
struct FoldArgs {
  const T* P = nullptr;
  int64_t K = 0;
  int ncols = 0;
  const double* beta = nullptr;
  Src<T> x;
  const double* D = nullptr;
  const double* Dtail = nullptr;
  int64_t Dlen = 0;
  T* Pw = nullptr;       // panel receiving the new column (== P for the fold chain)
  int64_t newj = 0;
  int64_t off = 0;
  const double* escale = nullptr;  // 2^-e
  double* head = nullptr;          // p[0..off]
  double* partials = nullptr;      // [gridDim.x]
  int64_t n = 0;
  int* status = nullptr;
};

template <typename T>
__global__ void __launch_bounds__(kUpdThreads) k_fold(const __grid_constant__ FoldArgs<T> a) {
  extern __shared__ double beta_s[];
  __shared__ double red_s[32];
  if (aborted(a.status)) return;
  for (int j = threadIdx.x; j < a.ncols; j += kUpdThreads) beta_s[j] = a.beta[j];
  __syncthreads();
  const int64_t tile = blockIdx.x;
  const int64_t i = tile * kTile + 2 * threadIdx.x;
  const double* bp[1] = {beta_s};
  double2 acc[1];
  panel_accumulate<T, 1>(a.P, a.K, a.ncols, tile, threadIdx.x, bp, acc);
  const double2 xv = src_pair(a.x, i, a.n);
  double p0 = 0.0, p1 = 0.0;
  if (i < a.n) p0 = dval(a.D, a.Dtail, a.Dlen, i) * (xv.x - acc[0].x);
  if (i + 1 < a.n) p1 = dval(a.D, a.Dtail, a.Dlen, i + 1) * (xv.y - acc[0].y);
  const double es = *a.escale;
  const double c0 = (i >= a.off) ? p0 : 0.0, c1 = (i + 1 >= a.off) ? p1 : 0.0;
  st_pair(a.Pw + paddr(i, a.newj, a.K), c0 * es, c1 * es);
  if (i <= a.off) a.head[i] = p0;
  if (i + 1 <= a.off) a.head[i + 1] = p1;
  const double t = block_sum<kUpdThreads>(c0 * c0 + c1 * c1, red_s);
  if (threadIdx.x == 0) a.partials[blockIdx.x] = t;
}

// ============================================================= k_other
// y = D z - P beta with z supported on rows < zlen: the reverse-adjoint
// application of the other chain to the folded iterate (haar.hpp:65).
template <typename T>
struct OtherArgs {
  const T* P = nullptr;
  int64_t K = 0;
  int ncols = 0;
  const double* beta = nullptr;
  const double* z = nullptr;
  int64_t zlen = 0;
  const double* D = nullptr;
  const double* Dtail = nullptr;
  int64_t Dlen = 0;
  int64_t n = 0;
  int* status = nullptr;
  Epi<T> epi;
};

template <typename T>
__global__ void __launch_bounds__(kUpdThreads) k_other(const __grid_constant__ OtherArgs<T> a) {
  extern __shared__ double beta_s[];
  __shared__ double red_s[32];
  if (aborted(a.status)) return;
  for (int j = threadIdx.x; j < a.ncols; j += kUpdThreads) beta_s[j] = a.beta[j];
  __syncthreads();
  const int64_t tile = blockIdx.x;
  const int64_t i = tile * kTile + 2 * threadIdx.x;
  const double* bp[1] = {beta_s};
  double2 acc[1];
  panel_accumulate<T, 1>(a.P, a.K, a.ncols, tile, threadIdx.x, bp, acc);
  double z0 = 0.0, z1 = 0.0;
  if (i < a.zlen) z0 = dval(a.D, a.Dtail, a.Dlen, i) * a.z[i];
  if (i + 1 < a.zlen) z1 = dval(a.D, a.Dtail, a.Dlen, i + 1) * a.z[i + 1];
  epilogue(a.epi, a.status, i, a.n, make_double2(z0 - acc[0].x, z1 - acc[0].y), red_s);
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
    for (int b = lane; b < nblk; b += 32) v += partials[(size_t)b * nslots + s];
    v = warp_sum(v);
    if (lane == 0) red[s] = v;
  }
  __syncthreads();
}

// Gram column + T column of a pending reflector (Schreiber-Van Loan):
// T_new[:k, k] = -c_k T[:k, :k] G[:k, k], T_new[k, k] = c_k.
__device__ void sm_finalize_pending(const ChainDev& ch, int pend, const double* rdots) {
  const int64_t K = ch.K;
  const double sp = ch.sig[pend];
  for (int j = threadIdx.x; j <= pend; j += kSmallThreads) ch.G[j + pend * K] = ch.sig[j] * sp * rdots[j];
  __syncthreads();
  const double cp = ch.c[pend];
  for (int i = threadIdx.x; i < pend; i += kSmallThreads) {
    double v = 0.0;
    for (int l = i; l < pend; ++l) v += ch.Tm[i + l * K] * ch.G[l + pend * K];
    ch.Tm[i + pend * K] = -cp * v;
  }
  if (threadIdx.x == 0) ch.Tm[pend + pend * K] = cp;
  __syncthreads();
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

// out = T a: thread per output row.
__device__ void sm_T(const ChainDev& ch, int k, const double* a, double* out) {
  for (int i = threadIdx.x; i < k; i += kSmallThreads) {
    double v = 0.0;
    for (int j = i; j < k; ++j) v += ch.Tm[i + (int64_t)j * ch.K] * a[j];
    out[i] = v;
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
  const double ck = ch.c[k];
  for (int i = threadIdx.x; i < k; i += kSmallThreads) {
    double v = 0.0;
    for (int l = i; l < k; ++l) v += ch.Tm[i + l * ch.K] * ch.G[l + (int64_t)k * ch.K];
    ch.Tm[i + (int64_t)k * ch.K] = -ck * v;
  }
  if (threadIdx.x == 0) ch.Tm[k + (int64_t)k * ch.K] = ck;
  __syncthreads();
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
};

// After k_dots of a probe (Haar and Ginibre "fold" side): finalise pending
// columns, the Haar mix reflector (chain B), the forward coefficients
// beta1 = sig (T^T (sig a)) for k_fold, the power-of-two column scale, and
// (Ginibre) the opposite-side sparse coefficients c.
template <typename T>
__global__ void __launch_bounds__(kSmallThreads) k_small_dots(const __grid_constant__ SmallArgs a) {
  if (aborted(a.status)) return;
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
                              : a.chB.sig[j] * (a.red[a.slotB_dot + j] / nrm + sign * (double)PB[paddr(a.off, j, a.chB.K)]);
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
    double v = 0.0;
    for (int b = threadIdx.x; b < a.nblk; b += kSmallThreads) v += a.partials[b];
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
