// Complex-field HD operators: the reference's
// GinibreOperator / HaarOperator with Scalar = std::complex<double>
// (ginibre.hpp:58-106, haar.hpp:40-67, unitary reflectors reflect.hpp:142-153).
//
// Same compact-WY algebra as the real path over C: members
// P_j = I - c_j w_j w_j^H (c real), leading phases s_j (complex, unit) factored
// into the cumulative diagonal D[i] = prod_{off_j <= i} s_j (conj for adjoint):
//   forward(x) = D o (x - W T^H W^H x),   reverse(x) = D o x - W T W^H (D o x),
//   T_new[:k, k] = -c_k T (W^H w_k), T[k, k] = c_k.
// Built from generic kernels — a coalesced two-stage GEMV-T over row blocks
// (right-hand side staged in shared memory, one warp per column), a
// thread-per-row GEMV-N with the D epilogue, single-block k x k algebra —
// rather than the fused TMA/PDL pipeline of the real path (no BASELINE
// workload is complex). Vectors are interleaved (re, im) fp64 = double2;
// panels are column-major (ld = dim), zero above each member's offset.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "hd_device.cuh"

namespace hd {
namespace cx {

using c2 = double2;

__host__ __device__ __forceinline__ c2 cmk(double re, double im) { return make_double2(re, im); }
__device__ __forceinline__ c2 cadd(c2 a, c2 b) { return cmk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ c2 csub(c2 a, c2 b) { return cmk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ c2 cmul(c2 a, c2 b) { return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ c2 cconjmul(c2 a, c2 b) {  // conj(a) * b
  return cmk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ c2 cconj(c2 a) { return cmk(a.x, -a.y); }
__device__ __forceinline__ c2 cscale(c2 a, double s) { return cmk(a.x * s, a.y * s); }
__device__ __forceinline__ double cnorm2(c2 a) { return a.x * a.x + a.y * a.y; }

// D(i) of a chain (conjugated in adjoint mode)
struct DView {
  const c2* head = nullptr;
  const c2* tail = nullptr;
  int64_t len = 0;
  int conj = 0;
  __device__ __forceinline__ c2 at(int64_t i) const {
    const c2 d = (i < len) ? head[i] : *tail;
    return conj ? cconj(d) : d;
  }
};

// v(i) = (D(i) if d) * x[i], rows outside [r0, r1) or < mask read as zero
struct CSrc {
  const c2* x = nullptr;
  DView d;
  int use_d = 0;
  int64_t mask = 0;
};

__device__ __forceinline__ c2 csrc(const CSrc& s, int64_t i) {
  if (i < s.mask) return cmk(0.0, 0.0);
  c2 v = s.x[i];
  return s.use_d ? cmul(s.d.at(i), v) : v;
}

constexpr int kCxRows = 1024;   // rows per block of the GEMV-T
constexpr int kCxThreads = 256;

// part[b * k + j] = sum_{i in block b} conj(W[i, j]) v(i), i in [r0, r1)
__global__ void __launch_bounds__(kCxThreads) kc_gemv_t(const c2* W, int64_t ld, int k, CSrc v, int64_t r0, int64_t r1,
                                                        c2* part) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  __shared__ c2 vs[kCxRows];
  const int64_t b0 = r0 + (int64_t)blockIdx.x * kCxRows;
  const int64_t rem = r1 - b0;
  const int nr = (int)(rem < kCxRows ? rem : (int64_t)kCxRows);
  for (int i = threadIdx.x; i < nr; i += blockDim.x) vs[i] = csrc(v, b0 + i);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = wid; j < k; j += nw) {
    const c2* col = W + (size_t)j * ld + b0;
    c2 acc = cmk(0.0, 0.0), acc2 = cmk(0.0, 0.0);
    int i = lane;
#pragma unroll 4
    for (; i + 32 < nr; i += 64) {  // two independent loads in flight per step
      acc = cadd(acc, cconjmul(col[i], vs[i]));
      acc2 = cadd(acc2, cconjmul(col[i + 32], vs[i + 32]));
    }
    if (i < nr) acc = cadd(acc, cconjmul(col[i], vs[i]));
    acc = cadd(acc, acc2);
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) part[(size_t)blockIdx.x * k + j] = acc;
  }
}

// out[j] = sum_b part[b * k + j]: one warp per column, lane-strided over the
// blocks then a shuffle tree (fixed order: deterministic)
__global__ void kc_reduce(const c2* part, int nb, int k, c2* out) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= k) return;
  c2 s = cmk(0.0, 0.0);
  for (int b = lane; b < nb; b += 32) s = cadd(s, part[(size_t)b * k + j]);
  for (int o = 16; o > 0; o >>= 1) {
    s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
    s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
  }
  if (lane == 0) out[j] = s;
}

// beta = T a (herm = 0) or T^H a (herm = 1), T upper triangular k x k (ld K)
__global__ void kc_tmul(const c2* T, int64_t K, int k, const c2* a, int herm, c2* beta) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
    c2 s = cmk(0.0, 0.0);
    if (!herm) {
      for (int j = i; j < k; ++j) s = cadd(s, cmul(T[(size_t)j * K + i], a[j]));  // T[i, j], j >= i
    } else {
      for (int j = 0; j <= i; ++j) s = cadd(s, cconjmul(T[(size_t)i * K + j], a[j]));  // conj(T[j, i]), j <= i
    }
    beta[i] = s;
  }
}

// GEMV-N with the chain epilogues (beta read through L1: a broadcast):
//   mode 0 (forward): y = D o (x - W beta)
//   mode 1 (reverse): y = D o x - W beta
//   mode 2 (plain)  : y = W beta
// x rows >= xlen read as zero (sparse inputs)
__global__ void kc_gemv_n(const c2* W, int64_t ld, int k, const c2* beta, const c2* x, int64_t xlen, DView d, int mode,
                          int64_t n, c2* y) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  c2 acc = cmk(0.0, 0.0), acc2 = cmk(0.0, 0.0);
  int j = 0;
#pragma unroll 4
  for (; j + 1 < k; j += 2) {  // two independent column loads in flight per step
    acc = cadd(acc, cmul(W[(size_t)j * ld + i], __ldg(beta + j)));
    acc2 = cadd(acc2, cmul(W[(size_t)(j + 1) * ld + i], __ldg(beta + j + 1)));
  }
  if (j < k) acc = cadd(acc, cmul(W[(size_t)j * ld + i], __ldg(beta + j)));
  acc = cadd(acc, acc2);
  if (mode == 2) {
    y[i] = acc;
    return;
  }
  const c2 xv = (i < xlen) ? x[i] : cmk(0.0, 0.0);
  const c2 di = d.at(i);
  y[i] = (mode == 0) ? cmul(di, csub(xv, acc)) : csub(cmul(di, xv), acc);
}

// ||p[off:]||^2 partial sums per block
__global__ void kc_tail_norm2(const c2* p, int64_t off, int64_t n, double* part) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = off + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += cnorm2(p[i]);
  s = block_sum<kCxThreads>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Reflector scalars from the tail norm (reflect.hpp:142-153): scal = {nrm,
// c, s.re, s.im, phase.re, phase.im}; identity (nrm == 0) -> c = 0, s = 1.
__global__ void kc_reflector_scalars(const double* part, int nb, const c2* p, int64_t off, double* scal) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  __shared__ double red[32];
  double s2 = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s2 += part[b];
  s2 = block_sum<kCxThreads>(s2, red);  // launched with kCxThreads threads
  if (threadIdx.x != 0) return;
  const double nrm = sqrt(s2);
  scal[0] = nrm;
  if (nrm == 0.0) {
    scal[1] = 0.0;
    scal[2] = 1.0;
    scal[3] = 0.0;
    scal[4] = 1.0;
    scal[5] = 0.0;
    return;
  }
  const c2 v1 = p[off];
  const double av = hypot(v1.x, v1.y);
  const double r = av / nrm;
  const c2 ph = (av == 0.0) ? cmk(1.0, 0.0) : cmk(v1.x / av, v1.y / av);
  scal[1] = 1.0 / (1.0 + r);
  scal[2] = -ph.x;  // s = -conj(phase)
  scal[3] = ph.y;
  scal[4] = ph.x;
  scal[5] = ph.y;
}

// column k of W: w = p[off:] / nrm (+ phase at off), zero above off and for
// the identity reflector
__global__ void kc_write_column(const c2* p, int64_t off, int64_t n, const double* scal, c2* col) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double nrm = scal[0];
  c2 w = cmk(0.0, 0.0);
  if (i >= off && nrm > 0.0) {
    w = cscale(p[i], 1.0 / nrm);
    if (i == off) w = cadd(w, cmk(scal[4], scal[5]));
  }
  col[i] = w;
}

// T column k from the Gram column G = W[:, :k]^H w_k; c/s stored; D updated
// with s from row off on (single block)
__global__ void kc_append_small(c2* T, int64_t K, int k, const c2* G, const double* scal, double* cs, c2* ss, c2* Dhead,
                                int64_t Dlen, c2* Dtail, int64_t off) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  const double c = scal[1];
  const c2 s = cmk(scal[2], scal[3]);
  for (int i = threadIdx.x; i < k; i += blockDim.x) {  // T[i, k] = -c sum_{j >= i} T[i, j] G[j]
    c2 acc = cmk(0.0, 0.0);
    for (int j = i; j < k; ++j) acc = cadd(acc, cmul(T[(size_t)j * K + i], G[j]));
    T[(size_t)k * K + i] = cscale(acc, -c);
  }
  if (threadIdx.x == 0) {
    T[(size_t)k * K + k] = cmk(c, 0.0);
    cs[k] = c;
    ss[k] = s;
  }
  for (int64_t i = off + threadIdx.x; i < Dlen; i += blockDim.x) Dhead[i] = cmul(Dhead[i], s);
  if (threadIdx.x == 0) *Dtail = cmul(*Dtail, s);
}

// z = H_fold p = [p[0:off], ||p[off:]||, 0, ...] (reflect.hpp: the reflector
// maps the tail onto +||tail|| e_off)
__global__ void kc_fold_z(const c2* p, int64_t off, int64_t n, const double* scal, c2* z) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  z[i] = (i < off) ? p[i] : (i == off ? cmk(scal[0], 0.0) : cmk(0.0, 0.0));
}

// complex draws of one probe: Philox (z = (n1 + i n2)/sqrt 2 per row) or the
// queued interleaved draws; rows < mask zero
__global__ void kc_draw(int philox, const unsigned long long* seedp, uint32_t stream, uint32_t probe, const c2* inj,
                        int64_t n, int64_t mask, c2* g) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  c2 v;
  if (philox) {
    const double2 z = philox_normal_pair(*seedp, stream, probe, (uint64_t)i);
    v = cmk(z.x * 0.7071067811865475244, z.y * 0.7071067811865475244);
  } else {
    v = inj[i];
  }
  g[i] = (i < mask) ? cmk(0.0, 0.0) : v;
}

__global__ void kc_unit(c2* v, int64_t n, int64_t at) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (i == at) ? cmk(1.0, 0.0) : cmk(0.0, 0.0);
}

// y = (add + y) * add_s * s, or y *= s without add
__global__ void kc_scale(c2* y, int64_t n, double s, const c2* add, double add_s) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  c2 v = y[i];
  if (add) v = cscale(cadd(add[i], v), add_s);
  y[i] = cscale(v, s);
}

// A non-finite entry raises the device flag (tested by the state-changing fused kernels)
// and its host-mapped mirror (read by the host after the probe's synchronisation)
__device__ __forceinline__ void raise_bad(int* flag, int* hflag) {
  atomicOr(flag, 1);
  if (hflag) {
    *reinterpret_cast<volatile int*>(hflag) = 1;
    __threadfence_system();
  }
}

// 1 if any entry is non-finite
__global__ void kc_check_finite(const c2* x, int64_t n, int* flag, int* hflag) {
  pdl_wait();  // programmatic dependent launch (as the real path)
  pdl_launch();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i].x) || !isfinite(x[i].y)) raise_bad(flag, hflag);
}

}  // namespace cx
}  // namespace hd
