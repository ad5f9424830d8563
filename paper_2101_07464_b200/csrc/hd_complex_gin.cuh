// Fused complex-field Ginibre probe (ginibre.hpp:58-106 with
// Scalar = complex<double>; GOE = two inner probes, ensembles.hpp:117-127):
// seven launches per probe instead of ~40, the three independent GEMV-T jobs
// in one grid and the GEMV-N jobs in two dual-job grids. With F the fold chain
// (on the input dimension), O the other chain, S_in / S_out the basis stores:
//
//   kc_draw       g (output dimension; rows below the other side's count zero)
//   kc_gemv_t3    a_F = W_F^H x, a_O = W_O^H (conj(D_O) g), a_S = S_in^H x
//   kc_reduce3    the three jobs' block partials, one warp per column
//   kc_small_ag   two CTAs: beta_F = T_F^H a_F | beta_O = T_O a_O
//   kc_gemv_n2    p = D_F o (x - W_F beta_F) with ||p[off:]||^2 partials |
//                 S_out[:, cnt] = conj(D_O) o g - W_O beta_O
//   kc_small_bg   single CTA: fold reflector scalars, the fold member joins chain F
//                 (Gram column from G = W_F^H W_F and the head corner, no panel
//                 pass: hd_complex_fused.cuh), the corner of F'-rev-adj(e_off):
//                 a_e = conj(D'_off W'[off, :]), beta_e = T' a_e, and the new basis
//                 coefficient <v_new, x> = (F'-fwd(x))[off] = ||p[off:]||
//   kc_gemv_n2    S_in[:, cnt] = conj(D'_F) o e_off - W'_F beta_e (the new fold column is
//                 generated from p on the fly and written to W_F) |
//                 y = sigma S_out a_S (GOE: (y_right + .) / sqrt 2 in the epilogue)
#pragma once

#include "hd_complex_fused.cuh"

namespace hd {
namespace cx {

struct TJobD {
  const c2* W = nullptr;
  int64_t ld = 0;
  int k = 0;
  const c2* v = nullptr;  // right-hand side, rows [r0, r1)
  DView d;                // ... times d(i) when use_d
  int use_d = 0;
  int64_t r0 = 0, r1 = 0;
  int nb = 0;
  c2* part = nullptr;  // nb x k
  int* flag = nullptr;  // non-null: v is a device input to validate
  int* hflag = nullptr;
};

struct TJobs3 {
  TJobD j[3];
};

template <int R>
__global__ void __launch_bounds__(kCxThreads) kc_gemv_t3(TJobs3 A) {
  pdl_wait();
  pdl_launch();
  __shared__ c2 wp[kCxWarps][kTColGroup];
  int bb = (int)blockIdx.x;
  int jid = 0;
  if (bb >= A.j[0].nb) {
    bb -= A.j[0].nb;
    jid = 1;
    if (bb >= A.j[1].nb) {
      bb -= A.j[1].nb;
      jid = 2;
    }
  }
  const TJobD J = jid == 0 ? A.j[0] : (jid == 1 ? A.j[1] : A.j[2]);
  const int64_t b0 = J.r0 + (int64_t)bb * (R * kCxThreads);
  c2 v[R];
  int64_t row[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = b0 + r * kCxThreads + threadIdx.x;
    const bool ok = i < J.r1;
    row[r] = ok ? i : J.r1 - 1;
    c2 t = ok ? J.v[i] : cmk(0.0, 0.0);
    if (J.flag && !(isfinite(t.x) && isfinite(t.y))) raise_bad(J.flag, J.hflag);
    if (ok && J.use_d) t = cmul(J.d.at(i), t);
    v[r] = t;
  }
  gemv_t_cols<R>(J.W, J.ld, J.k, row, v, J.part + (size_t)bb * J.k, wp);
}

struct RJob {
  const c2* part = nullptr;
  int nb = 0, k = 0;
  c2* out = nullptr;
};

// out_q[j] = sum_b part_q[b, j] for three jobs: one warp per column (fixed order)
__global__ void kc_reduce3(RJob r0, RJob r1, RJob r2) {
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31;
  int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  RJob R = r0;
  if (j >= r0.k) {
    j -= r0.k;
    R = r1;
    if (j >= r1.k) {
      j -= r1.k;
      R = r2;
      if (j >= r2.k) return;
    }
  }
  c2 s = cmk(0.0, 0.0);
  for (int b = lane; b < R.nb; b += 32) s = cadd(s, R.part[(size_t)b * R.k + j]);
  s = warp_csum(s);
  if (lane == 0) R.out[j] = s;
}

// CTA 0: beta_F = T_F^H a_F; CTA 1: beta_O = T_O a_O
__global__ void __launch_bounds__(kSmallThreads) kc_small_ag(const c2* TF, int64_t KF, int kF, const c2* aF, c2* betaF,
                                                             const c2* TO, int64_t KO, int kO, const c2* aO,
                                                             c2* betaO) {
  pdl_wait();
  pdl_launch();
  if (blockIdx.x == 0)
    tmul_herm(TF, KF, kF, aF, betaF);
  else
    tmul_plain(TO, KO, kO, aO, betaO);
}

enum : int { kNFwd = 0, kNRevG = 1, kNRevE = 2, kNPlain = 3 };

struct NJob {
  int kind = kNFwd;
  const c2* W = nullptr;
  int64_t ld = 0;
  int k = 0;
  const c2* beta = nullptr;
  int64_t n = 0;
  int nb = 0;  // row blocks (kCxThreads rows each)
  DView d;
  int64_t off = 0;
  const c2* x = nullptr;          // Fwd: x; RevG: g; RevE: p; Plain: the vector to add (or null)
  c2* out = nullptr;              // Fwd: p; RevG / RevE: the new basis column; Plain: y
  double* npart = nullptr;        // Fwd: ||p[off:]||^2 block partials
  const double* scal = nullptr;   // RevE: the fold member's scalars
  c2* colF = nullptr;             // RevE: the fold member's column (null: no member joined)
  double sigma = 1.0, add_s = 1.0;  // Plain: y = (sigma W beta + add) add_s
};

__global__ void __launch_bounds__(kCxThreads) kc_gemv_n2(NJob a, NJob b, const int* bad) {
  pdl_wait();
  pdl_launch();
  if (bad && *bad) return;
  __shared__ double red[32];
  const bool second = (int)blockIdx.x >= a.nb;
  const NJob J = second ? b : a;
  const int bb = second ? (int)blockIdx.x - a.nb : (int)blockIdx.x;
  const int64_t i = (int64_t)bb * kCxThreads + threadIdx.x;
  const bool ok = i < J.n;
  int64_t row[1] = {ok ? i : J.n - 1};
  c2 acc[1];
  gemv_n_rows<1>(J.W, J.ld, J.k, J.beta, row, acc);
  if (J.kind == kNFwd) {
    double n2 = 0.0;
    if (ok) {
      const c2 pv = cmul(J.d.at(i), csub(J.x[i], acc[0]));
      J.out[i] = pv;
      if (i >= J.off) n2 = cnorm2(pv);
    }
    n2 = block_sum<kCxThreads>(n2, red);
    if (threadIdx.x == 0) J.npart[bb] = n2;
    return;
  }
  if (!ok) return;
  if (J.kind == kNRevG) {
    J.out[i] = csub(cmul(J.d.at(i), J.x[i]), acc[0]);
  } else if (J.kind == kNRevE) {
    c2 s = acc[0];
    if (J.colF) {
      const c2 wn = column_entry(J.x[i], i, J.off, J.scal);
      J.colF[i] = wn;
      s = cadd(s, cmul(wn, __ldg(J.beta + J.k)));
    }
    const c2 e = (i == J.off) ? J.d.at(i) : cmk(0.0, 0.0);
    J.out[i] = csub(e, s);
  } else {
    c2 yv = cscale(acc[0], J.sigma);
    if (J.x) yv = cadd(yv, J.x[i]);
    J.out[i] = cscale(yv, J.add_s);
  }
}

struct SmallBG {
  ChainRef F;
  int appendF = 0;
  int kF = 0;
  int64_t off = 0;
  const double* npart = nullptr;
  int nbn = 0;
  const c2* p = nullptr;
  c2* aF = nullptr;
  const c2* betaF = nullptr;
  double* scal = nullptr;
  c2* ae = nullptr;      // corner of F'-rev-adj(e_off)
  c2* betaE = nullptr;   // T' a_e
  c2* aS_new = nullptr;  // <v_new, x>
  const int* bad = nullptr;
};

__global__ void __launch_bounds__(kSmallThreads) kc_small_bg(SmallBG A) {
  pdl_wait();
  pdl_launch();
  if (A.bad && *A.bad) return;
  __shared__ double red[32];
  __shared__ double sc[8];
  double s2 = 0.0;
  for (int b = threadIdx.x; b < A.nbn; b += blockDim.x) s2 += A.npart[b];
  s2 = block_sum<kSmallThreads>(s2, red);
  if (threadIdx.x == 0) {
    reflector_scalars(s2, A.p[A.off], sc);
    for (int q = 0; q < 7; ++q) A.scal[q] = sc[q];
    *A.aS_new = A.appendF ? cmk(sc[0], 0.0) : A.p[A.off];
  }
  __syncthreads();
  if (A.appendF) {
    append_fold_member(A.F, A.kF, A.off, A.p, A.aF, A.betaF, sc);
    __syncthreads();  // D'_off, T' column
  }
  const int k1 = A.kF + A.appendF;
  const c2 dc = cconj(A.F.d_at(A.off));
  for (int j = threadIdx.x; j < k1; j += blockDim.x) {
    c2 w;
    if (j < A.kF) {
      w = A.F.W[(size_t)j * A.F.ld + A.off];
    } else {
      w = column_entry(A.p[A.off], A.off, A.off, sc);  // the member's own pivot entry
    }
    A.ae[j] = cmul(cconj(w), dc);
  }
  __syncthreads();
  tmul_plain(A.F.T, A.F.K, k1, A.ae, A.betaE);
}

}  // namespace cx
}  // namespace hd
