// Fused complex-field Haar probe (haar.hpp:40-67 with
// Scalar = complex<double>): three to four panel passes in seven launches
// instead of the generic sequence's five passes in 22 (hd_complex.cuh).
//
//   kc_gemv_t2   one grid, two GEMV-T jobs: a_F = W_F^H x over all rows and the
//                fresh draw's dots W_O^H g[off:] (they do not depend on x) with
//                ||g[off:]||^2; each thread keeps its rows' right-hand side in
//                registers and walks the columns (independent 16-B loads),
//                warp-shuffle + block reduction per column
//   kc_reduce2   both jobs' block partials and the norm, one warp per column
//   kc_small_a   single CTA: beta_F = T_F^H a_F and the draw's reflector scalars
//   kc_nfold     GEMV-N p = D_F o (x - W_F beta_F), ||p[off:]||^2 partials; writes
//                the draw's normalised column into W_O on the way. CTA 0 does no
//                rows: it appends the draw's member to chain O meanwhile (Gram
//                column = dots / nrm + phase conj(W_O[off, :]), T_O / G_O columns,
//                D_O) - nothing in this pass reads them
//   kc_small_b   single CTA: fold reflector scalars, the reverse application's
//                corner dots W_O^H (conj(D_O) z) (z lives on rows <= off) and
//                beta_O = T_O a_O
//   kc_nother    GEMV-N y = conj(D_O) o z - W_O beta_O with z read from p on the
//                fly; writes the fold member's normalised column into W_F. CTA 0
//                appends the fold member to chain F meanwhile, its Gram column
//                WITHOUT a panel pass: on rows >= off the diagonal D_F is the
//                scalar d = D_tail, so
//                  W^H p[off:] = d (a - G beta - W_head^H (p_head / D_head)),
//                with G = W_F^H W_F kept per chain (k x k) and the head a t x k
//                corner; T_F / G_F columns, D_F update (needed by the next probe)
//   kc_nother_spec  kc_nother that also takes the NEXT probe's draw dots with chain
//                O' from the columns it streams (a Haar draw never depends on x): the
//                next probe's second kc_gemv_t2 job disappears when its side repeats
// Device inputs are validated inside the first GEMV-T job that streams them: a
// non-finite entry raises a flag the state-changing kernels test (`bad`) and its
// host-mapped mirror, so a probe is one enqueue and one synchronisation.
#pragma once

#include "hd_complex.cuh"

namespace hd {
namespace cx {

constexpr int kTRows = 4;        // most rows per thread of the GEMV-T kernels (template R = 2 or 4; a CTA holds R * kCxThreads rows)
constexpr int kTColGroup = 128;  // columns per shared-memory round
constexpr int kCxWarps = kCxThreads / 32;

struct TJob {
  const c2* W = nullptr;
  int64_t ld = 0;
  int k = 0;
  const c2* v = nullptr;     // right-hand side (rows [r0, r1))
  int64_t r0 = 0, r1 = 0;
  int nb = 0;                // row blocks of this job
  c2* part = nullptr;        // nb x k
  double* npart = nullptr;   // nb: ||v||^2 over the block's rows (or null)
  int* flag = nullptr;       // non-null: v is a device input to validate (raise_bad on a non-finite entry)
  int* hflag = nullptr;
};

__device__ __forceinline__ c2 warp_csum(c2 a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
    a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
  }
  return a;
}

// part_row[j] = sum over this CTA's rows of conj(W[row, j]) v[row], j < k: every thread
// holds kTRows rows of the right-hand side; two columns per step (eight independent
// loads), warp-shuffle then cross-warp reduction through shared memory
template <int R>
__device__ __forceinline__ void gemv_t_cols(const c2* W, int64_t ld, int k, const int64_t* row, const c2* v,
                                            c2* part_row, c2 (*wp)[kTColGroup]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int g0 = 0; g0 < k; g0 += kTColGroup) {
    const int gk = min(kTColGroup, k - g0);
    int j = 0;
    for (; j + 1 < gk; j += 2) {
      const c2* ca = W + (size_t)(g0 + j) * ld;
      const c2* cb = ca + ld;
      c2 la[R], lb[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        la[r] = ca[row[r]];
        lb[r] = cb[row[r]];
      }
      c2 sa = cmk(0.0, 0.0), sb = cmk(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        sa = cadd(sa, cconjmul(la[r], v[r]));
        sb = cadd(sb, cconjmul(lb[r], v[r]));
      }
      sa = warp_csum(sa);
      sb = warp_csum(sb);
      if (lane == 0) {
        wp[wid][j] = sa;
        wp[wid][j + 1] = sb;
      }
    }
    if (j < gk) {
      const c2* ca = W + (size_t)(g0 + j) * ld;
      c2 sa = cmk(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < R; ++r) sa = cadd(sa, cconjmul(ca[row[r]], v[r]));
      sa = warp_csum(sa);
      if (lane == 0) wp[wid][j] = sa;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < gk; c += kCxThreads) {
      c2 s = wp[0][c];
#pragma unroll
      for (int w = 1; w < kCxWarps; ++w) s = cadd(s, wp[w][c]);
      part_row[g0 + c] = s;
    }
    __syncthreads();
  }
}

template <int R>
__global__ void __launch_bounds__(kCxThreads) kc_gemv_t2(TJob j0, TJob j1) {
  pdl_wait();
  pdl_launch();
  __shared__ c2 wp[kCxWarps][kTColGroup];
  __shared__ double red[32];
  const bool second = (int)blockIdx.x >= j0.nb;
  TJob J;  // field-wise select (no dynamic indexing of the parameter space)
  J.W = second ? j1.W : j0.W;
  J.ld = second ? j1.ld : j0.ld;
  J.k = second ? j1.k : j0.k;
  J.v = second ? j1.v : j0.v;
  J.r0 = second ? j1.r0 : j0.r0;
  J.r1 = second ? j1.r1 : j0.r1;
  J.part = second ? j1.part : j0.part;
  J.npart = second ? j1.npart : j0.npart;
  J.flag = second ? j1.flag : j0.flag;
  J.hflag = second ? j1.hflag : j0.hflag;
  const int bb = second ? (int)blockIdx.x - j0.nb : (int)blockIdx.x;
  const int64_t b0 = J.r0 + (int64_t)bb * (R * kCxThreads);
  c2 v[R];
  int64_t row[R];
  double n2 = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = b0 + r * kCxThreads + threadIdx.x;
    const bool ok = i < J.r1;
    row[r] = ok ? i : J.r1 - 1;  // clamped: loads stay unconditional, the product is zero
    v[r] = ok ? J.v[i] : cmk(0.0, 0.0);
    if (J.flag && !(isfinite(v[r].x) && isfinite(v[r].y))) raise_bad(J.flag, J.hflag);
    n2 += cnorm2(v[r]);
  }
  if (J.npart) {
    n2 = block_sum<kCxThreads>(n2, red);
    if (threadIdx.x == 0) J.npart[bb] = n2;
  }
  gemv_t_cols<R>(J.W, J.ld, J.k, row, v, J.part + (size_t)bb * J.k, wp);
}

// out0[j] = sum_b part0[b, j], out1[j] = sum_b part1[b, j], nrm2 = sum_b npart[b]:
// one warp per column (fixed order: deterministic), the last warp takes the norm
__global__ void kc_reduce2(const c2* part0, int nb0, int k0, c2* out0, const c2* part1, int nb1, int k1, c2* out1,
                           const double* npart, int nbn, double* nrm2) {
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31;
  int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j == k0 + k1) {
    double s = 0.0;
    for (int b = lane; b < nbn; b += 32) s += npart[b];
    s = warp_sum(s);
    if (lane == 0) *nrm2 = s;
    return;
  }
  if (j > k0 + k1) return;
  const c2* part = part0;
  int nb = nb0, k = k0;
  c2* out = out0;
  if (j >= k0) {
    j -= k0;
    part = part1;
    nb = nb1;
    k = k1;
    out = out1;
  }
  c2 s = cmk(0.0, 0.0);
  for (int b = lane; b < nb; b += 32) s = cadd(s, part[(size_t)b * k + j]);
  s = warp_csum(s);
  if (lane == 0) out[j] = s;
}

// reflector scalars (reflect.hpp:142-153) from ||tail||^2 and the tail's first
// entry: scal = {nrm, c, s.re, s.im, phase.re, phase.im, ||w||^2}
__device__ __forceinline__ void reflector_scalars(double nrm2, c2 v1, double* scal) {
  const double nrm = sqrt(nrm2);
  scal[0] = nrm;
  if (nrm == 0.0) {
    scal[1] = 0.0;
    scal[2] = 1.0;
    scal[3] = 0.0;
    scal[4] = 1.0;
    scal[5] = 0.0;
    scal[6] = 0.0;
    return;
  }
  const double av = hypot(v1.x, v1.y);
  const double r = av / nrm;
  const c2 ph = (av == 0.0) ? cmk(1.0, 0.0) : cmk(v1.x / av, v1.y / av);
  scal[1] = 1.0 / (1.0 + r);
  scal[2] = -ph.x;  // s = -conj(phase)
  scal[3] = ph.y;
  scal[4] = ph.x;
  scal[5] = ph.y;
  scal[6] = 2.0 * (1.0 + r);  // ||tail / nrm + phase e_off||^2
}

// A chain's small state as the single-CTA stages see it
struct ChainRef {
  const c2* W = nullptr;
  int64_t ld = 0;
  c2* T = nullptr;
  c2* G = nullptr;
  int64_t K = 0;
  double* c = nullptr;
  c2* s = nullptr;
  c2* Dhead = nullptr;
  int64_t Dlen = 0;
  c2* Dtail = nullptr;
  __device__ __forceinline__ c2 d_at(int64_t i) const { return (i < Dlen) ? Dhead[i] : *Dtail; }
};

// member k joins the chain: T and G columns from its Gram column gs[0..k),
// c / s, D from row off on. All threads of the CTA (after a barrier on gs).
__device__ __forceinline__ void append_member(const ChainRef& ch, int k, const c2* gs, const double* scal, int64_t off) {
  const double c = scal[1];
  const c2 s = cmk(scal[2], scal[3]);
  for (int i = threadIdx.x; i < k; i += blockDim.x) {  // T[i, k] = -c sum_{j >= i} T[i, j] gs[j]
    c2 a0 = cmk(0.0, 0.0), a1 = cmk(0.0, 0.0);
    int j = i;
#pragma unroll 4
    for (; j + 1 < k; j += 2) {
      a0 = cadd(a0, cmul(ch.T[(size_t)j * ch.K + i], gs[j]));
      a1 = cadd(a1, cmul(ch.T[(size_t)(j + 1) * ch.K + i], gs[j + 1]));
    }
    if (j < k) a0 = cadd(a0, cmul(ch.T[(size_t)j * ch.K + i], gs[j]));
    ch.T[(size_t)k * ch.K + i] = cscale(cadd(a0, a1), -c);
    ch.G[(size_t)k * ch.K + i] = gs[i];
    ch.G[(size_t)i * ch.K + k] = cconj(gs[i]);
  }
  if (threadIdx.x == 0) {
    ch.T[(size_t)k * ch.K + k] = cmk(c, 0.0);
    ch.G[(size_t)k * ch.K + k] = cmk(scal[6], 0.0);
    ch.c[k] = c;
    ch.s[k] = s;
    *ch.Dtail = cmul(*ch.Dtail, s);
  }
  for (int64_t i = off + threadIdx.x; i < ch.Dlen; i += blockDim.x) ch.Dhead[i] = cmul(ch.Dhead[i], s);
}

// beta[i] = sum_{j <= i} conj(T[j, i]) a[j] (T^H a): a warp per output (column i of T
// is contiguous), two outputs in flight. All threads of the CTA.
__device__ __forceinline__ void tmul_herm(const c2* T, int64_t K, int k, const c2* a, c2* beta) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = wid; i < k; i += 2 * nw) {
    const int i2 = i + nw;
    const bool two = i2 < k;
    const c2* c1 = T + (size_t)i * K;
    const c2* c2p = T + (size_t)(two ? i2 : i) * K;
    c2 s1 = cmk(0.0, 0.0), s2 = cmk(0.0, 0.0);
    const int jmax = two ? i2 : i;
    for (int j = lane; j <= jmax; j += 32) {
      const c2 av = a[j];
      if (j <= i) s1 = cadd(s1, cconjmul(c1[j], av));
      if (two) s2 = cadd(s2, cconjmul(c2p[j], av));
    }
    s1 = warp_csum(s1);
    s2 = warp_csum(s2);
    if (lane == 0) {
      beta[i] = s1;
      if (two) beta[i2] = s2;
    }
  }
}

// beta[i] = sum_{j >= i} T[i, j] a[j] (T a): a warp per output, lanes over the columns
__device__ __forceinline__ void tmul_plain(const c2* T, int64_t K, int k, const c2* a, c2* beta) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = wid; i < k; i += 2 * nw) {
    const int i2 = i + nw;
    const bool two = i2 < k;
    c2 s1 = cmk(0.0, 0.0), sb = cmk(0.0, 0.0);
    for (int j = i + lane; j < k; j += 32) {
      const c2 av = a[j];
      s1 = cadd(s1, cmul(T[(size_t)j * K + i], av));
      if (two && j >= i2) sb = cadd(sb, cmul(T[(size_t)j * K + i2], av));
    }
    s1 = warp_csum(s1);
    sb = warp_csum(sb);
    if (lane == 0) {
      beta[i] = s1;
      if (two) beta[i2] = sb;
    }
  }
}

// The fold member (built from p at offset off, scalars in scal) joins chain F without a
// panel pass for its Gram column: on rows >= off the diagonal D_F is the scalar d = D_tail, so
//   W^H p[off:] = d (a - G beta - W_head^H (p_head / D_head)),  a = W^H x, beta = T^H a,
// and the column is p[off:] / nrm + phase e_off. aF is overwritten with the Gram column.
// All threads of the CTA.
__device__ __forceinline__ void append_fold_member(const ChainRef& F, int k, int64_t off, const c2* p, c2* aF,
                                                   const c2* betaF, const double* scal) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double nrm = scal[0];
  const c2 ph = cmk(scal[4], scal[5]);
  const c2 dt = *F.Dtail;  // D_F on rows >= off (before this member's s)
  for (int j = threadIdx.x; j < k; j += blockDim.x) {  // a_j - (G beta)_j
    c2 a0 = cmk(0.0, 0.0), a1 = cmk(0.0, 0.0);
    int l = 0;
#pragma unroll 4
    for (; l + 1 < k; l += 2) {
      a0 = cadd(a0, cmul(F.G[(size_t)l * F.K + j], betaF[l]));
      a1 = cadd(a1, cmul(F.G[(size_t)(l + 1) * F.K + j], betaF[l + 1]));
    }
    if (l < k) a0 = cadd(a0, cmul(F.G[(size_t)l * F.K + j], betaF[l]));
    aF[j] = csub(aF[j], cadd(a0, a1));
  }
  __syncthreads();
  // minus the head corner W_head^H (p_head / D_head), a warp per column
  for (int j = wid; j < k; j += nw) {
    const c2* col = F.W + (size_t)j * F.ld;
    c2 acc = cmk(0.0, 0.0);
    for (int64_t i = lane; i < off; i += 32) {
      const c2 d = F.d_at(i);
      const c2 xv = cscale(cconjmul(d, p[i]), 1.0 / cnorm2(d));  // p / D
      acc = cadd(acc, cconjmul(col[i], xv));
    }
    acc = warp_csum(acc);
    if (lane == 0) {
      c2 v = cmk(0.0, 0.0);
      if (nrm > 0.0) {
        const c2 S = cmul(dt, csub(aF[j], acc));  // W[:, j]^H p[off:]
        v = cadd(cscale(S, 1.0 / nrm), cmul(ph, cconj(col[off])));
      }
      aF[j] = v;
    }
  }
  __syncthreads();
  append_member(F, k, aF, scal, off);
}

constexpr int kSmallThreads = 512;

struct SmallA {
  const c2* aF = nullptr;
  const c2* TF = nullptr;
  int64_t KF = 0;
  int kF = 0;
  c2* betaF = nullptr;
  const double* nrm2g = nullptr;  // ||g[off:]||^2
  const c2* g = nullptr;
  int64_t off = 0;
  double* scal2 = nullptr;
};

__global__ void __launch_bounds__(kSmallThreads) kc_small_a(SmallA A) {
  pdl_wait();
  pdl_launch();
  if (threadIdx.x == 0) reflector_scalars(*A.nrm2g, A.g[A.off], A.scal2);
  tmul_herm(A.TF, A.KF, A.kF, A.aF, A.betaF);
}

struct NFold {
  const c2* W = nullptr;
  int64_t ld = 0;
  int k = 0;
  const c2* beta = nullptr;
  const c2* x = nullptr;
  DView d;
  int64_t n = 0, off = 0;
  c2* p = nullptr;
  double* npart = nullptr;
  const int* bad = nullptr;
  // the draw's member
  const c2* g = nullptr;
  const double* scal2 = nullptr;
  c2* colO = nullptr;
  ChainRef O;
  int kO = 0;
  c2* dotsO = nullptr;  // W_O[:, :kO]^H g[off:], turned into the Gram column in place
};

// acc[r] = sum_j W[row[r], j] beta[j], R consecutive rows per thread
template <int R>
__device__ __forceinline__ void gemv_n_rows(const c2* W, int64_t ld, int k, const c2* beta, const int64_t* row, c2* acc) {
  c2 a0[R], a1[R];
#pragma unroll
  for (int r = 0; r < R; ++r) a0[r] = a1[r] = cmk(0.0, 0.0);
  int j = 0;
#pragma unroll 2
  for (; j + 1 < k; j += 2) {  // two columns per step
    const c2* w0 = W + (size_t)j * ld;
    const c2* w1 = w0 + ld;
    c2 l0[R], l1[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      l0[r] = w0[row[r]];
      l1[r] = w1[row[r]];
    }
    const c2 b0 = __ldg(beta + j), b1 = __ldg(beta + j + 1);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      a0[r] = cadd(a0[r], cmul(l0[r], b0));
      a1[r] = cadd(a1[r], cmul(l1[r], b1));
    }
  }
  if (j < k) {
    const c2* w0 = W + (size_t)j * ld;
    const c2 b0 = __ldg(beta + j);
#pragma unroll
    for (int r = 0; r < R; ++r) a0[r] = cadd(a0[r], cmul(w0[row[r]], b0));
  }
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = cadd(a0[r], a1[r]);
}

// normalised reflector column entry from its source vector (zero above off
// and for the identity reflector)
__device__ __forceinline__ c2 column_entry(c2 src, int64_t i, int64_t off, const double* scal) {
  const double nrm = scal[0];
  if (i < off || !(nrm > 0.0)) return cmk(0.0, 0.0);
  c2 w = cscale(src, 1.0 / nrm);
  if (i == off) w = cadd(w, cmk(scal[4], scal[5]));
  return w;
}

// grid = 1 + ceil(n / (R * kCxThreads)); CTA 0 appends the draw's member
template <int R>
__global__ void __launch_bounds__(kCxThreads) kc_nfold(NFold A) {
  pdl_wait();
  pdl_launch();
  if (A.bad && *A.bad) return;
  __shared__ double red[32];
  if (blockIdx.x == 0) {
    const double nrm = A.scal2[0];
    const c2 ph = cmk(A.scal2[4], A.scal2[5]);
    for (int j = threadIdx.x; j < A.kO; j += blockDim.x) {
      c2 v = cmk(0.0, 0.0);
      if (nrm > 0.0) v = cadd(cscale(A.dotsO[j], 1.0 / nrm), cmul(ph, cconj(A.O.W[(size_t)j * A.O.ld + A.off])));
      A.dotsO[j] = v;
    }
    __syncthreads();
    append_member(A.O, A.kO, A.dotsO, A.scal2, A.off);
    return;
  }
  const int64_t i0 = ((int64_t)(blockIdx.x - 1) * kCxThreads + threadIdx.x) * R;
  int64_t row[R];
#pragma unroll
  for (int r = 0; r < R; ++r) row[r] = (i0 + r < A.n) ? i0 + r : A.n - 1;
  c2 acc[R];
  gemv_n_rows<R>(A.W, A.ld, A.k, A.beta, row, acc);
  double n2 = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = i0 + r;
    if (i < A.n) {
      const c2 pv = cmul(A.d.at(i), csub(A.x[i], acc[r]));
      A.p[i] = pv;
      if (i >= A.off) n2 += cnorm2(pv);
      A.colO[i] = column_entry(A.g[i], i, A.off, A.scal2);
    }
  }
  n2 = block_sum<kCxThreads>(n2, red);
  if (threadIdx.x == 0) A.npart[blockIdx.x - 1] = n2;
}

struct SmallB {
  int64_t off = 0;
  const double* npart = nullptr;
  int nbn = 0;
  const c2* p = nullptr;
  double* scal = nullptr;
  // other chain (kO1 members, the draw's included): corner of the reverse application
  ChainRef O;
  int kO1 = 0;
  c2* aO = nullptr;
  c2* betaO = nullptr;
};

__global__ void __launch_bounds__(kSmallThreads) kc_small_b(SmallB A) {
  pdl_wait();
  pdl_launch();
  __shared__ double red[32];
  __shared__ double sc[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double s2 = 0.0;
  for (int b = threadIdx.x; b < A.nbn; b += blockDim.x) s2 += A.npart[b];
  s2 = block_sum<kSmallThreads>(s2, red);
  if (threadIdx.x == 0) {
    reflector_scalars(s2, A.p[A.off], sc);
    for (int q = 0; q < 7; ++q) A.scal[q] = sc[q];
  }
  __syncthreads();
  const double nrm = sc[0];
  // a_O[j] = sum_{i <= off} conj(W_O[i, j]) conj(D_O[i]) z[i], z = [p[0:off], nrm]:
  // a warp per column, two columns in flight
  for (int j = wid; j < A.kO1; j += 2 * nw) {
    const int j2 = j + nw;
    const bool two = j2 < A.kO1;
    const c2* c1 = A.O.W + (size_t)j * A.O.ld;
    const c2* c2p = A.O.W + (size_t)(two ? j2 : j) * A.O.ld;
    c2 s1 = cmk(0.0, 0.0), sb = cmk(0.0, 0.0);
    for (int64_t i = lane; i <= A.off; i += 32) {
      const c2 z = (i < A.off) ? A.p[i] : cmk(nrm, 0.0);
      const c2 dz = cconjmul(A.O.d_at(i), z);
      s1 = cadd(s1, cconjmul(c1[i], dz));
      sb = cadd(sb, cconjmul(c2p[i], dz));
    }
    s1 = warp_csum(s1);
    sb = warp_csum(sb);
    if (lane == 0) {
      A.aO[j] = s1;
      if (two) A.aO[j2] = sb;
    }
  }
  __syncthreads();
  tmul_plain(A.O.T, A.O.K, A.kO1, A.aO, A.betaO);
}

struct NOther {
  const c2* W = nullptr;
  int64_t ld = 0;
  int k = 0;
  const c2* beta = nullptr;
  DView d;  // conjugated (adjoint mode)
  int64_t n = 0, off = 0;
  const c2* p = nullptr;
  const double* scal = nullptr;
  c2* y = nullptr;
  const int* bad = nullptr;
  // the fold member
  int appendF = 0;
  c2* colF = nullptr;
  ChainRef F;
  int kF = 0;
  c2* aF = nullptr;  // W_F^H x, turned into the Gram column in place
  const c2* betaF = nullptr;
};

// grid = 1 + ceil(n / (R * kCxThreads)); CTA 0 appends the fold member
template <int R>
__global__ void __launch_bounds__(kCxThreads) kc_nother(NOther A) {
  pdl_wait();
  pdl_launch();
  if (A.bad && *A.bad) return;
  if (blockIdx.x == 0) {
    if (!A.appendF) return;
    append_fold_member(A.F, A.kF, A.off, A.p, A.aF, A.betaF, A.scal);
    return;
  }
  const int64_t i0 = ((int64_t)(blockIdx.x - 1) * kCxThreads + threadIdx.x) * R;
  if (i0 >= A.n) return;
  int64_t row[R];
#pragma unroll
  for (int r = 0; r < R; ++r) row[r] = (i0 + r < A.n) ? i0 + r : A.n - 1;
  c2 acc[R];
  gemv_n_rows<R>(A.W, A.ld, A.k, A.beta, row, acc);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = i0 + r;
    if (i < A.n) {
      const c2 pv = A.p[i];
      const c2 z = (i < A.off) ? pv : (i == A.off ? cmk(A.scal[0], 0.0) : cmk(0.0, 0.0));
      A.y[i] = csub(cmul(A.d.at(i), z), acc[r]);
      if (A.colF) A.colF[i] = column_entry(pv, i, A.off, A.scal);
    }
  }
}


// ---- the other chain's GEMV-N with the NEXT probe's draw dots from the same bytes.
// A Haar probe's draw never depends on x, so when the next probe keeps its side the
// dots W_O'^H g'[off + 1:] and ||g'[off + 1:]||^2 it needs (kc_gemv_t2's second job) are
// taken here, from the columns this pass streams anyway: three panel passes per probe.
// Rows per thread / CTA as in the GEMV-T kernel (the shuffle reduction per column is
// amortised over kTRows rows).
constexpr int kSpecCols = 8;  // columns per shared-memory reduction round (kc_nother_spec)

struct SpecOut {
  const c2* g = nullptr;     // the next probe's draw
  int64_t off = 0;           // its offset: rows below are masked
  c2* part = nullptr;        // (grid - 1) x k block partials
  double* npart = nullptr;   // (grid - 1) partial ||g[off:]||^2
};

// grid = 1 + ceil(n / (R kCxThreads)); CTA 0 appends the fold member. R rows per thread:
// fewer rows = more CTAs (finer waves), more rows = fewer shared-memory partials per byte
template <int R>
__global__ void __launch_bounds__(kCxThreads, 4) kc_nother_spec(NOther A, SpecOut S) {
  pdl_wait();
  pdl_launch();
  if (A.bad && *A.bad) return;
  if (blockIdx.x == 0) {
    if (A.appendF) append_fold_member(A.F, A.kF, A.off, A.p, A.aF, A.betaF, A.scal);
    return;
  }
  // per-thread column partials go to shared memory; one warp per column reduces them
  // every kSpecCols columns (no shuffle chain inside the streaming loop)
  __shared__ c2 tp[kSpecCols][kCxThreads];
  __shared__ double red[32];
  const int bb = (int)blockIdx.x - 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t b0 = (int64_t)bb * (R * kCxThreads);
  int row[R];  // offsets from the CTA's first row (clamped: loads stay unconditional)
  c2 gv[R], acc[R];
  double n2 = 0.0;
  const int nrem = (int)min((int64_t)(R * kCxThreads), A.n - b0);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int o = r * kCxThreads + threadIdx.x;
    const bool ok = o < nrem;
    row[r] = ok ? o : nrem - 1;
    gv[r] = (ok && b0 + o >= S.off) ? S.g[b0 + o] : cmk(0.0, 0.0);
    n2 += cnorm2(gv[r]);
    acc[r] = cmk(0.0, 0.0);
  }
  n2 = block_sum<kCxThreads>(n2, red);
  if (threadIdx.x == 0) S.npart[bb] = n2;
  c2* part_row = S.part + (size_t)bb * A.k;
  const c2* Wb = A.W + b0;
  for (int g0 = 0; g0 < A.k; g0 += kSpecCols) {
    const int gk = min(kSpecCols, A.k - g0);
#pragma unroll 2
    for (int j = 0; j < gk; ++j) {
      const c2* ca = Wb + (size_t)(g0 + j) * A.ld;
      c2 la[R];
#pragma unroll
      for (int r = 0; r < R; ++r) la[r] = ca[row[r]];
      const c2 ba = __ldg(A.beta + g0 + j);
      c2 sa = cmk(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        acc[r] = cadd(acc[r], cmul(la[r], ba));
        sa = cadd(sa, cconjmul(la[r], gv[r]));
      }
      tp[j][threadIdx.x] = sa;
    }
    __syncthreads();
    for (int c = wid; c < gk; c += kCxWarps) {
      c2 t = cmk(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < kCxThreads / 32; ++q) t = cadd(t, tp[c][q * 32 + lane]);
      t = warp_csum(t);
      if (lane == 0) part_row[g0 + c] = t;
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = b0 + r * kCxThreads + threadIdx.x;
    if (i < A.n) {
      const c2 pv = A.p[i];
      const c2 z = (i < A.off) ? pv : (i == A.off ? cmk(A.scal[0], 0.0) : cmk(0.0, 0.0));
      A.y[i] = csub(cmul(A.d.at(i), z), acc[r]);
      if (A.colF) A.colF[i] = column_entry(pv, i, A.off, A.scal);
    }
  }
}

}  // namespace cx
}  // namespace hd
