// Device-side building blocks of the Householder Dice hot path on sm_100a.
//
// Data layout: every reflector chain, and the Ginibre basis
// stores, live in HBM as tall-skinny panels in TILE-MAJOR order
//   element (row i, column j) -> P[(i / 256) * (K * 256) + j * 256 + (i % 256)]
// so the j used columns of a 256-row tile are one contiguous j*2 KB block
// (fp64) and appending a column writes 2 KB contiguous per tile. K is the
// column capacity fixed at operator creation (hd_config.capacity).
//
// Column j of a chain panel holds the Householder vector up to an exact
// power-of-two / per-column scale: w_j = sig[j] * P[:, j], where w_j is the
// reference's normalised reflection vector (reflect.hpp:168-174).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hd {

constexpr int kTile = 256;       // panel tile height (rows)
constexpr int kTileShift = 8;

__host__ __device__ __forceinline__ size_t paddr(int64_t i, int64_t j, int64_t K) {
  return (size_t)(i >> kTileShift) * (size_t)(K << kTileShift) + (size_t)(j << kTileShift) + (size_t)(i & (kTile - 1));
}

// ------------------------------------------------------------ Philox4x32-10
// Counter-based generator (Salmon et al., SC'11). Keyed by the operator seed;
// counter = (row-pair index lo/hi, probe index, stream) so any row of any
// probe's draw can be regenerated independently, in any kernel, any number
// of times (generated twice per Ginibre probe instead of stored).
struct Philox {
  uint32_t k0, k1;
};

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += W0;
    k1 += W1;
  }
  return c;
}

// Straight-line fp64 kernels for the Box-Muller transform (the streaming
// kernels regenerate draws on the fly, so their instruction count is on the
// critical path; libdevice's log/sincospi carry special-case branches and
// range reduction the bounded arguments here never need).
//
// ln(x) for x in [2^-53, 1]: x = m 2^e with m in [sqrt(1/2), sqrt(2)),
// f = m - 1, s = f / (2 + f), ln(1 + f) = f - f^2/2 + s (f^2/2 + R(s^2)) with
// the degree-14 minimax R of fdlibm's e_log.c (Sun Microsystems, 1993);
// max error 1 ulp (checked against libm over 2e6 arguments incl. both ends).
__device__ __forceinline__ double log_unit(double x) {
  constexpr double Lg1 = 6.666666666666735130e-01, Lg2 = 3.999999999940941908e-01,
                   Lg3 = 2.857142874366239149e-01, Lg4 = 2.222219843214978396e-01,
                   Lg5 = 1.818357216161805012e-01, Lg6 = 1.531383769920937332e-01,
                   Lg7 = 1.479819860511658591e-01;
  constexpr double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  int e = (hi >> 20) - 1023;
  hi = (hi & 0x000fffff) | 0x3ff00000;  // m in [1, 2)
  if (hi > 0x3ff6a09e) {                // m > sqrt(2): halve it
    hi -= 0x00100000;
    e += 1;
  }
  const double f = __hiloint2double(hi, lo) - 1.0;  // exact
  const double d = 2.0 + f;
  double r;  // d in [1.7, 2.5]: hardware approximation, two Newton steps
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = fma(r, fma(-d, r, 1.0), r);
  r = fma(r, fma(-d, r, 1.0), r);
  double s = f * r;
  s = fma(fma(-s, d, f), r, s);
  const double z = s * s, w = z * z;
  const double t1 = w * fma(w, fma(w, Lg6, Lg4), Lg2);
  const double t2 = z * fma(w, fma(w, fma(w, Lg7, Lg5), Lg3), Lg1);
  const double R = t1 + t2, hfsq = 0.5 * f * f, k = (double)e;
  return k * ln2_hi - ((hfsq - fma(s, hfsq + R, k * ln2_lo)) - f);
}

// sqrt(t) for finite t >= 0 without the special-value paths of sqrt():
// hardware rsqrt approximation, two Newton steps, one residual correction.
__device__ __forceinline__ double sqrt_nonneg(double t) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
  const double h = 0.5 * t;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  double r = t * y;
  r = fma(fma(-r, r, t), 0.5 * y, r);
  return t > 0.0 ? r : 0.0;
}

// (sin 2 pi u, cos 2 pi u) for u in [0, 1): u = k/4 + t with |t| <= 1/8 is
// exact, then fdlibm's __kernel_sin / __kernel_cos minimax polynomials on
// [-pi/4, pi/4] and a quadrant rotation; max abs error 7e-16.
__device__ __forceinline__ void sincos_2pi_unit(double u, double* sp, double* cp) {
  constexpr double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
                   S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
                   S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
  constexpr double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
                   C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
                   C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
  const double kq = rint(u * 4.0);
  const double x = (u - kq * 0.25) * 6.283185307179586232;
  const double z = x * x;
  const double ps = fma(z, fma(z, fma(z, fma(z, fma(z, S6, S5), S4), S3), S2), S1);
  const double pc = fma(z, fma(z, fma(z, fma(z, fma(z, C6, C5), C4), C3), C2), C1);
  const double sn = fma(x * z, ps, x);
  const double cs = fma(z * z, pc, fma(-0.5, z, 1.0));
  const int q = (int)kq & 3;
  const double a = (q & 1) ? cs : sn, b = (q & 1) ? sn : cs;
  *sp = (q & 2) ? -a : a;
  *cp = ((q + 1) & 2) ? -b : b;
}

// Two N(0,1) draws for rows (2q, 2q+1) of probe `probe` (Box-Muller on two
// 53-bit uniforms, computed in fp64 for every dtype).
__device__ __forceinline__ double2 philox_normal_pair(uint64_t seed, uint32_t stream, uint32_t probe, uint64_t q) {
  const uint4 w = philox4x32_10(make_uint4((uint32_t)q, (uint32_t)(q >> 32), probe, stream), (uint32_t)seed,
                                (uint32_t)(seed >> 32));
  const uint64_t a = ((uint64_t)w.x << 32) | w.y;
  const uint64_t b = ((uint64_t)w.z << 32) | w.w;
  const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
  const double u2 = (double)(b >> 11) * 0x1.0p-53;          // [0, 1)
  const double r = sqrt_nonneg(-2.0 * log_unit(u1));
  double s, c;
  sincos_2pi_unit(u2, &s, &c);
  return make_double2(r * c, r * s);
}

// ------------------------------------------------------------ vector source
// Where a streamed right-hand side comes from: a dense device vector (the
// iterate, optionally times a device scalar), fresh Philox normals, or draws
// injected by the caller (parity mode). Rows < mask_begin read as zero
// (ginibre.hpp:73 `g.head(l).setZero()`, and the Haar tail restriction); the
// optional D factor is the chain's cumulative-sign diagonal.
enum SrcKind : int { kSrcNone = 0, kSrcVec = 1, kSrcPhilox = 2, kSrcInjected = 3 };

template <typename T>
struct Src {
  int kind = kSrcNone;
  const T* x = nullptr;
  const double* xscale = nullptr;  // device scalar or null
  const unsigned long long* seedp = nullptr;  // device word: one graph serves every reseed
  uint32_t stream = 0;
  uint32_t probe = 0;
  const double* inj = nullptr;  // this probe's injected draws (length n)
  int64_t mask_begin = 0;
  const double* D = nullptr;    // D(i) = i < Dlen ? D[i] : *Dtail
  const double* Dtail = nullptr;
  int64_t Dlen = 0;
  int64_t vbase = 0;  // kSrcVec: x holds global rows [vbase, ...) (row shard)
};

template <typename T>
__device__ __forceinline__ double dvalue(const Src<T>& s, int64_t i) {
  if (s.D == nullptr) return 1.0;
  return i < s.Dlen ? s.D[i] : *s.Dtail;
}

// The global-load half of src_pair: raw vector values of global rows
// (i, i+1) (kSrcVec; other kinds return zeros). Issued a tile ahead by the
// streaming kernels so the load latency overlaps the current tile.
template <typename T>
__device__ __forceinline__ double2 src_raw(const Src<T>& s, int64_t i, int64_t n) {
  double2 v = make_double2(0.0, 0.0);
  if (s.kind == kSrcVec) {
    const T* xp = s.x + (i - s.vbase);
    if (i + 1 < n) {
      if constexpr (sizeof(T) == 8) {
        v = *reinterpret_cast<const double2*>(xp);
      } else {
        const float2 f = *reinterpret_cast<const float2*>(xp);
        v = make_double2(f.x, f.y);
      }
    } else if (i < n) {
      v.x = (double)xp[0];
    }
  }
  return v;
}

// Values of global rows (i, i+1), i even, given src_raw's result: vector
// scale, fresh Philox or injected draws, the mask and D; rows >= n are zero.
template <typename T>
__device__ __forceinline__ double2 src_finish(const Src<T>& s, int64_t i, int64_t n, double2 v) {
  if (s.kind == kSrcVec) {
    if (s.xscale) {
      const double sc = *s.xscale;
      v.x *= sc;
      v.y *= sc;
    }
  } else if (s.kind == kSrcPhilox) {
    // generated unconditionally (branch-free in i, so the unrolled row pairs
    // of a lane interleave their Box-Muller chains), zeroed beyond n
    v = philox_normal_pair(*s.seedp, s.stream, s.probe, (uint64_t)(i >> 1));
    if constexpr (sizeof(T) == 4) {  // fp32 path consumes fp32-rounded draws
      v.x = (double)(float)v.x;
      v.y = (double)(float)v.y;
    }
    if (i >= n) v.x = 0.0;
    if (i + 1 >= n) v.y = 0.0;
  } else if (s.kind == kSrcInjected) {
    if (i < n) v.x = s.inj[i];
    if (i + 1 < n) v.y = s.inj[i + 1];
    if constexpr (sizeof(T) == 4) {
      v.x = (double)(float)v.x;
      v.y = (double)(float)v.y;
    }
  }
  if (i < s.mask_begin) v.x = 0.0;
  if (i + 1 < s.mask_begin) v.y = 0.0;
  if (s.D) {
    v.x *= dvalue(s, i);
    v.y *= dvalue(s, i + 1);
  }
  return v;
}

// Values of global rows (i, i+1), i even; rows >= n read as zero.
template <typename T>
__device__ __forceinline__ double2 src_pair(const Src<T>& s, int64_t i, int64_t n) {
  return src_finish(s, i, n, src_raw(s, i, n));
}

// Load two consecutive panel entries as doubles.
template <typename T>
__device__ __forceinline__ double2 ld_pair(const T* p) {
  if constexpr (sizeof(T) == 8) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
  } else {
    float2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
    return make_double2(r.x, r.y);
  }
}

template <typename T>
__device__ __forceinline__ void st_pair(T* p, double a, double b) {
  if constexpr (sizeof(T) == 8) {
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
  } else {
    *reinterpret_cast<float2*>(p) = make_float2((float)a, (float)b);
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Eight warp sums at once (9 shuffles): the full sum of v[(lane >> 2) & 7]
// in every lane.
__device__ __forceinline__ double warp_sum8(const double* v, int lane) {
  const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
  double e[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const double keep = b16 ? v[u + 4] : v[u], send = b16 ? v[u] : v[u + 4];
    e[u] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  double f[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const double keep = b8 ? e[u + 2] : e[u], send = b8 ? e[u] : e[u + 2];
    f[u] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double g = (b4 ? f[1] : f[0]) + __shfl_xor_sync(0xffffffffu, b4 ? f[0] : f[1], 4);
  g += __shfl_xor_sync(0xffffffffu, g, 2);
  g += __shfl_xor_sync(0xffffffffu, g, 1);
  return g;
}

// Two warp sums at once (fixed butterfly, 5 shuffles instead of 10).
// Returns the full sum of d[(lane >> 4) & 1] in every lane.
__device__ __forceinline__ double warp_sum2(double d0, double d1, int lane) {
  const bool hi = lane & 16;
  double f = (hi ? d1 : d0) + __shfl_xor_sync(0xffffffffu, hi ? d0 : d1, 16);
  f += __shfl_xor_sync(0xffffffffu, f, 8);
  f += __shfl_xor_sync(0xffffffffu, f, 4);
  f += __shfl_xor_sync(0xffffffffu, f, 2);
  f += __shfl_xor_sync(0xffffffffu, f, 1);
  return f;
}

// Four warp sums at once (fixed butterfly, 6 shuffles instead of 20).
// Returns the full sum of d[(lane >> 3) & 3] in every lane.
__device__ __forceinline__ double warp_sum4(double d0, double d1, double d2, double d3, int lane) {
  const bool hi = lane & 16;
  const double k0 = hi ? d2 : d0, k1 = hi ? d3 : d1;
  const double s0 = hi ? d0 : d2, s1 = hi ? d1 : d3;
  const double e0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 16);
  const double e1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 16);
  const bool hb = lane & 8;
  double f = (hb ? e1 : e0) + __shfl_xor_sync(0xffffffffu, hb ? e0 : e1, 8);
  f += __shfl_xor_sync(0xffffffffu, f, 4);
  f += __shfl_xor_sync(0xffffffffu, f, 2);
  f += __shfl_xor_sync(0xffffffffu, f, 1);
  return f;
}

// Deterministic block sum (fixed tree); result valid in all threads.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = (l < NT / 32) ? sh[l] : 0.0;
    t = warp_sum(t);
    if (l == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

// ------------------------------------------- TMA bulk copies + mbarriers
// The streaming kernels stage panel chunks global -> shared with
// cp.async.bulk (SASS UBLKCP) completing on an mbarrier transaction count;
// a single producer thread keeps a ring of stages in flight while the
// consumer warps compute.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy (bytes % 16 == 0, 16 B aligned), evict-first
// in L2: every panel byte is streamed exactly once per pass.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         bool keep = false) {
  // streamed panels are read once: evict-first, except chunks the next
  // kernel re-reads at once (keep: evict-last, see k_dots / ApplyArgs::reverse)
  if (keep) {
    asm volatile(
        "{\n"
        ".reg .b64 pol;\n"
        "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n"
        "}\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
  } else {
    asm volatile(
        "{\n"
        ".reg .b64 pol;\n"
        "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n"
        "}\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
  }
}

// Ampere-style asynchronous 8-byte global -> shared copies (LDGSTS): the
// single-CTA stages issue every load of their staging phase back to back
// and wait once, instead of paying one L2 round trip per dependent load.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* smem, const T* gmem) {
  if constexpr (sizeof(T) == 8) cp_async8(smem, gmem);
  else cp_async4(smem, gmem);
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Programmatic dependent launch: every kernel of the probe
// sequence waits for its predecessor's completion before reading anything
// the predecessor writes, and only then lets its own successor launch; so
// the code before pdl_wait() may read data written two or more launches
// back (the streaming kernels prefetch their panel chunks there).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace hd
