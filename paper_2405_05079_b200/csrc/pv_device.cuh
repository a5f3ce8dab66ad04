// Device helpers for the PoVar hot path (sm_100a, fp64, CUDA cores only).
//
// Everything here is per-observation / per-landmark / per-camera arithmetic that
// the kernels in pv_kernels.cuh fuse together.  The algebra follows the
// reference (pkg/src/stratba/objective.py:68-146, normal_eq.py:145-198,
// riemannian.py:37-56) but is re-derived into forms that never materialise the
// per-observation Jacobians or W blocks:
//
//   stage 1:  W_ij = [x a^T; x b^T; x c^T] with
//             a = p0 - s m0 p2,  b = p1 - s m1 p2,  c = -s (m0 e0 + m1 e1),
//             e_r = p_r - m_r p2,  s = 1 - eta,  p_r = P[r, 0:3]
//   stage 2:  W_ij = [x g0^T; x g1^T; x g2^T] (unprojected 12x4) with
//             u = P x, iz = 1/u2, pi = u01 * iz, J_r = iz (P_r - pi_r P_2),
//             g0 = iz J0, g1 = iz J1, g2 = -iz (pi0 J0 + pi1 J1)
//
// so W^T v = sum_c (x . v_c) G_c and W t = [x (G_0.t); x (G_1.t); x (G_2.t)].
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define PV_FULL 0xffffffffu

// PV_CHECKED builds (tools/checked_build.sh): device-side bounds / invariant checks on the
// indirect accesses of the hot kernels -- the stand-in for compute-sanitizer, which this
// pool does not allow.  A failed check prints and traps (the launch then reports an error).
#ifdef PV_CHECKED
#include <cstdio>
#define PV_CHECK(cond)                                                                     \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("PV_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);                  \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define PV_CHECK(cond) ((void)0)
#endif

namespace pv {

// ---------------------------------------------------------------------------
// 256-bit vector memory access (Blackwell LDG.E.ENL2.256 / STG.E.ENL2.256)

__device__ __forceinline__ double4 ldg4(const double* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
      : "l"(p));
  return v;
}

// coherent (no .nc) variant for data written earlier in the same kernel
__device__ __forceinline__ double4 ld4(const double* p) {
  double4 v;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ void st4(double* p, double4 v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y),
               "d"(v.z), "d"(v.w)
               : "memory");
}

// L2 eviction-priority hints (createpolicy + .L2::cache_hint): streaming data
// is marked evict_first so that the reused landmark vectors stay resident.
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_normal() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 0 normal, 1 evict_first, 2 evict_last (one createpolicy per call: `which` is uniform)
__device__ __forceinline__ uint64_t pol_sel(int which) {
  uint64_t p;
  if (which == 2)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else if (which == 1)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double4 ldg4p(const double* p, uint64_t pol) {
  double4 v;
  asm("ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
      : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ldg2p(const double* p, uint64_t pol) {
  double2 v;
  asm("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ldgip(const int* p, uint64_t pol) {
  int v;
  asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st4p(double* p, double4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "d"(v.x),
               "d"(v.y), "d"(v.z), "d"(v.w), "l"(pol)
               : "memory");
}

// 128-bit halves (k_series: ptxas 12.9 dropped three of the four components of a 256-bit
// st.global.v4.f64 -- and the loads feeding them -- inside a non-inlined device function,
// profiles/r2_series.md; two v2.f64 accesses are compiled correctly)
__device__ __forceinline__ double4 ldg4_h(const double* p) {
  double4 v;
  asm("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  asm("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.z), "=d"(v.w) : "l"(p + 2));
  return v;
}
__device__ __forceinline__ double4 ld4cg_h(const double* p, uint64_t pol) {
  double4 v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol)
               : "memory");
  asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(v.z), "=d"(v.w)
               : "l"(p + 2), "l"(pol)
               : "memory");
  return v;
}
// coherent (L2) 256-bit load of data other CTAs wrote earlier in the same launch
__device__ __forceinline__ double4 ld4cg(const double* p, uint64_t pol) {
  double4 v;
  asm volatile("ld.global.cg.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p), "l"(pol)
               : "memory");
  return v;
}
__device__ __forceinline__ void st4p_h(double* p, double4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
               "l"(pol)
               : "memory");
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p + 2), "d"(v.z),
               "d"(v.w), "l"(pol)
               : "memory");
}

__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

__device__ __forceinline__ double dot4(const double4& a, const double4& b) {
  return fma(a.x, b.x, fma(a.y, b.y, fma(a.z, b.z, a.w * b.w)));
}
__device__ __forceinline__ double dot3(const double4& a, const double4& b) {
  return fma(a.x, b.x, fma(a.y, b.y, a.z * b.z));
}
__device__ __forceinline__ double4 axpy4(double a, const double4& x, const double4& y) {
  return make_double4(fma(a, x.x, y.x), fma(a, x.y, y.y), fma(a, x.z, y.z), fma(a, x.w, y.w));
}
__device__ __forceinline__ double4 scale4(double a, const double4& x) {
  return make_double4(a * x.x, a * x.y, a * x.z, a * x.w);
}
__device__ __forceinline__ double4 zero4() { return make_double4(0.0, 0.0, 0.0, 0.0); }

// ---------------------------------------------------------------------------
// warp reductions (deterministic trees)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(PV_FULL, v, d);
  return v;
}

// Segmented suffix reduce: after the call, lane l holds the sum over
// [l, min(l+32, seg_end)).  Segment heads therefore hold their segment total.
template <int N>
__device__ __forceinline__ void seg_reduce(double (&v)[N], int lane, int seg_end) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double o = __shfl_down_sync(PV_FULL, v[k], d);
      if (lane + d < seg_end) v[k] += o;
    }
  }
}

// Same, with only as many steps as the longest segment needs (max_len <= 32).
template <int N>
__device__ __forceinline__ void seg_reduce_n(double (&v)[N], int lane, int seg_end, int max_len) {
  for (int d = 1; d < max_len; d <<= 1) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double o = __shfl_down_sync(PV_FULL, v[k], d);
      if (lane + d < seg_end) v[k] += o;
    }
  }
}

template <int N>
__device__ __forceinline__ void warp_reduce_all(double (&v)[N]) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] += __shfl_xor_sync(PV_FULL, v[k], d);
  }
}

// Fixed-order strided sum of per-item partials written earlier in the launch by other CTAs:
// thread t adds part[(t + k * blockDim.x) * NV + v] for k = 0, 1, ... in order.  UB loads of
// each chain are in flight at once (one L2 round trip per UB items instead of one per item: a
// last-CTA reduction over 13,682 cameras went from ~54 to 4 dependent round trips); the
// additions keep the one-at-a-time order, so the bits do too.
template <int NV, int UB = 16>
__device__ __forceinline__ void strided_sum_ordered(const double* part, int n, double (&a)[NV]) {
  const int T = blockDim.x;
  int i = threadIdx.x;
  for (; i + (UB - 1) * T < n; i += UB * T) {
    double v[UB][NV];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      if (NV == 2) {
        const double2 w = __ldcg(reinterpret_cast<const double2*>(part) + (i + u * T));
        v[u][0] = w.x;
        v[u][NV - 1] = w.y;
      } else {
#pragma unroll
        for (int q = 0; q < NV; ++q) v[u][q] = __ldcg(part + (size_t)(i + u * T) * NV + q);
      }
    }
#pragma unroll
    for (int u = 0; u < UB; ++u)
#pragma unroll
      for (int q = 0; q < NV; ++q) a[q] += v[u][q];
  }
  for (; i < n; i += T)
#pragma unroll
    for (int q = 0; q < NV; ++q) a[q] += __ldcg(part + (size_t)i * NV + q);
}

// Sum of 12 per-lane values over the warp, returned in lane i for component i (i < 12).
// A transposed butterfly: at each level a lane keeps half of its (padded to 16) values and
// adds its partner's copy of them, so every component sees exactly the additions of
// warp_reduce_all (own + partner at xor distance 16, 8, 4, 2, 1) -- identical bits -- for
// ~80 instead of ~180 instructions.  After the levels lanes 2I and 2I+1 hold component I.
__device__ __forceinline__ double warp_reduce12_lane(const double (&acc)[12], int lane) {
  double b[8];
  const bool h16 = lane & 16;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double lo = acc[j], hi = j + 8 < 12 ? acc[j + 8] : 0.0;
    const double r = __shfl_xor_sync(PV_FULL, h16 ? lo : hi, 16);
    b[j] = (h16 ? hi : lo) + r;
  }
  double c[4];
  const bool h8 = lane & 8;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double r = __shfl_xor_sync(PV_FULL, h8 ? b[j] : b[j + 4], 8);
    c[j] = (h8 ? b[j + 4] : b[j]) + r;
  }
  double e[2];
  const bool h4 = lane & 4;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double r = __shfl_xor_sync(PV_FULL, h4 ? c[j] : c[j + 2], 4);
    e[j] = (h4 ? c[j + 2] : c[j]) + r;
  }
  const bool h2 = lane & 2;
  const double f = (h2 ? e[1] : e[0]) + __shfl_xor_sync(PV_FULL, h2 ? e[0] : e[1], 2);
  const double g = f + __shfl_xor_sync(PV_FULL, f, 1);
  return __shfl_sync(PV_FULL, g, (2 * lane) & 31);
}

// Same for 32 values: lane i returns the warp sum of component i (bit-identical to
// warp_reduce_all, ~100 instead of ~480 instructions).
__device__ __forceinline__ double warp_reduce32_lane(const double (&acc)[32], int lane) {
  double b[16];
  const bool h16 = lane & 16;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double r = __shfl_xor_sync(PV_FULL, h16 ? acc[j] : acc[j + 16], 16);
    b[j] = (h16 ? acc[j + 16] : acc[j]) + r;
  }
  double c[8];
  const bool h8 = lane & 8;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double r = __shfl_xor_sync(PV_FULL, h8 ? b[j] : b[j + 8], 8);
    c[j] = (h8 ? b[j + 8] : b[j]) + r;
  }
  double e[4];
  const bool h4 = lane & 4;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double r = __shfl_xor_sync(PV_FULL, h4 ? c[j] : c[j + 4], 4);
    e[j] = (h4 ? c[j + 4] : c[j]) + r;
  }
  double f[2];
  const bool h2 = lane & 2;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double r = __shfl_xor_sync(PV_FULL, h2 ? e[j] : e[j + 2], 2);
    f[j] = (h2 ? e[j + 2] : e[j]) + r;
  }
  const bool h1 = lane & 1;
  return (h1 ? f[1] : f[0]) + __shfl_xor_sync(PV_FULL, h1 ? f[0] : f[1], 1);
}

// ---------------------------------------------------------------------------
// observation generators

struct Gen {
  double4 g0, g1, g2;
};

// stage 1 (pOSE): W^T generators a, b, c (3-vectors; .w = 0)
__device__ __forceinline__ Gen gen_s1(const double4& P0, const double4& P1, const double4& P2,
                                      double m0, double m1, double s) {
  double4 e0 = make_double4(P0.x - m0 * P2.x, P0.y - m0 * P2.y, P0.z - m0 * P2.z, 0.0);
  double4 e1 = make_double4(P1.x - m1 * P2.x, P1.y - m1 * P2.y, P1.z - m1 * P2.z, 0.0);
  double q = 1.0 - s;
  Gen G;
  G.g0 = make_double4(fma(s, e0.x, q * P0.x), fma(s, e0.y, q * P0.y), fma(s, e0.z, q * P0.z), 0.0);
  G.g1 = make_double4(fma(s, e1.x, q * P1.x), fma(s, e1.y, q * P1.y), fma(s, e1.z, q * P1.z), 0.0);
  G.g2 = make_double4(-s * fma(m0, e0.x, m1 * e1.x), -s * fma(m0, e0.y, m1 * e1.y),
                      -s * fma(m0, e0.z, m1 * e1.z), 0.0);
  return G;
}

// stage 2 (projective): unprojected W^T generators g0, g1, g2 (4-vectors)
__device__ __forceinline__ Gen gen_s2(const double4& P0, const double4& P1, const double4& P2,
                                      const double4& x) {
  double u0 = dot4(P0, x), u1 = dot4(P1, x), u2 = dot4(P2, x);
  double iz = 1.0 / u2;
  double p0 = u0 * iz, p1 = u1 * iz;
  double4 J0 = make_double4(iz * (P0.x - p0 * P2.x), iz * (P0.y - p0 * P2.y),
                            iz * (P0.z - p0 * P2.z), iz * (P0.w - p0 * P2.w));
  double4 J1 = make_double4(iz * (P1.x - p1 * P2.x), iz * (P1.y - p1 * P2.y),
                            iz * (P1.z - p1 * P2.z), iz * (P1.w - p1 * P2.w));
  Gen G;
  G.g0 = scale4(iz, J0);
  G.g1 = scale4(iz, J1);
  G.g2 = make_double4(-iz * fma(p0, J0.x, p1 * J1.x), -iz * fma(p0, J0.y, p1 * J1.y),
                      -iz * fma(p0, J0.z, p1 * J1.z), -iz * fma(p0, J0.w, p1 * J1.w));
  return G;
}

// ---------------------------------------------------------------------------
// "dot-product form" of the two W applications (never forms G):
//   W t   : y[4c + a] += sigma_c x_a,  sigma_c = G_c . t from q_r = P_r . t
//   W^T v : s = sum_r f_r P_r (stage 1: rows restricted to xyz) from d_c = x . v_c
// stage 1: sigma = (q0 - s m0 q2, q1 - s m1 q2, -s m0 q0 - s m1 q1 + s |m|^2 q2)
//          f     = (d0 - s m0 d2, d1 - s m1 d2, -s m0 d0 - s m1 d1 + s |m|^2 d2)
// stage 2: w = iz^2, e_r = q_r - pi_r q2 (resp. d_r - pi_r d2):
//          sigma = w (e0, e1, -(pi0 e0 + pi1 e1)),  f = w (e0, e1, -(pi0 e0 + pi1 e1))

struct Proj {  // per-observation projection scalars
  double a0, a1;  // stage 1: s m0, s m1      stage 2: pi0, pi1
  double c2;      // stage 1: s |m|^2         stage 2: unused
  double w;       // stage 1: 1               stage 2: iz^2
};

__device__ __forceinline__ Proj proj_s1(double m0, double m1, double s) {
  Proj p;
  p.a0 = s * m0;
  p.a1 = s * m1;
  p.c2 = s * fma(m0, m0, m1 * m1);
  p.w = 1.0;
  return p;
}

__device__ __forceinline__ Proj proj_s2(const double4& P0, const double4& P1, const double4& P2,
                                        const double4& x) {
  const double u0 = dot4(P0, x), u1 = dot4(P1, x), u2 = dot4(P2, x);
  const double iz = 1.0 / u2;
  Proj p;
  p.a0 = u0 * iz;
  p.a1 = u1 * iz;
  p.c2 = 0.0;
  p.w = iz * iz;
  return p;
}

// maps (q0, q1, q2) -> (sigma0, sigma1, sigma2); same map for d -> f
template <int STAGE>
__device__ __forceinline__ void proj_map(const Proj& p, double q0, double q1, double q2,
                                         double& o0, double& o1, double& o2) {
  if (STAGE == 1) {
    o0 = fma(-p.a0, q2, q0);
    o1 = fma(-p.a1, q2, q1);
    o2 = fma(p.c2, q2, -fma(p.a0, q0, p.a1 * q1));
  } else {
    const double e0 = fma(-p.a0, q2, q0), e1 = fma(-p.a1, q2, q1);
    o0 = p.w * e0;
    o1 = p.w * e1;
    o2 = -p.w * fma(p.a0, e0, p.a1 * e1);
  }
}

// ---------------------------------------------------------------------------
// Householder tangent bases (riemannian.py:37-56), applied implicitly.
// B = (I - 2 h h^T)[:, 1:], h = (v + sign(v0) e0) / ||v + sign(v0) e0||.

template <int N>
__device__ __forceinline__ void householder_h(const double* v, double* h) {
  double sg = v[0] >= 0.0 ? 1.0 : -1.0;
  double nn = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    h[i] = v[i] + (i == 0 ? sg : 0.0);
    nn = fma(h[i], h[i], nn);
  }
  double inv = 1.0 / sqrt(nn);
#pragma unroll
  for (int i = 0; i < N; ++i) h[i] *= inv;
}

// out (N) = B t  with t (N-1)
template <int N>
__device__ __forceinline__ void basis_apply(const double* h, const double* t, double* out) {
  double d = 0.0;
#pragma unroll
  for (int i = 1; i < N; ++i) d = fma(h[i], t[i - 1], d);
#pragma unroll
  for (int i = 0; i < N; ++i) out[i] = fma(-2.0 * h[i], d, i == 0 ? 0.0 : t[i - 1]);
}

// out (N-1) = B^T s  with s (N)
template <int N>
__device__ __forceinline__ void basis_apply_t(const double* h, const double* s, double* out) {
  double d = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) d = fma(h[i], s[i], d);
#pragma unroll
  for (int i = 1; i < N; ++i) out[i - 1] = fma(-2.0 * h[i], d, s[i]);
}

// ---------------------------------------------------------------------------
// 3x3 symmetric eigen-decomposition by cyclic Jacobi; pseudo-inverse with the
// reference's cutoff w <= rel_tol * max(trace, 0) (normal_eq.py:145-153).
// Symmetric 3x3 packed as (xx, xy, xz, yy, yz, zz).

__device__ inline bool pinv_sym3(const double* a6, double rel_tol, double* out6) {
  double A[3][3] = {{a6[0], a6[1], a6[2]}, {a6[1], a6[3], a6[4]}, {a6[2], a6[4], a6[5]}};
  double Q[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  double tr = a6[0] + a6[3] + a6[5];
  constexpr double EPS = 2.220446049250313e-16;
  for (int sweep = 0; sweep < 12; ++sweep) {
    bool rotated = false;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0;
      const int q = pq == 0 ? 1 : 2;
      double apq = A[p][q];
      // classic cyclic-Jacobi skip rule: off-diagonal below eps of the diagonals
      if (fabs(apq) <= EPS * sqrt(fabs(A[p][p] * A[q][q])) || apq == 0.0) continue;
      rotated = true;
      double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
      double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(fma(theta, theta, 1.0)));
      double c = 1.0 / sqrt(fma(t, t, 1.0));
      double s = t * c;
#pragma unroll
      for (int k = 0; k < 3; ++k) {  // A <- A J
        double akp = A[k][p], akq = A[k][q];
        A[k][p] = c * akp - s * akq;
        A[k][q] = s * akp + c * akq;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {  // A <- J^T A
        double apk = A[p][k], aqk = A[q][k];
        A[p][k] = c * apk - s * aqk;
        A[q][k] = s * apk + c * aqk;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double qkp = Q[k][p], qkq = Q[k][q];
        Q[k][p] = c * qkp - s * qkq;
        Q[k][q] = s * qkp + c * qkq;
      }
    }
    if (!rotated) break;
  }
  double tol = rel_tol * fmax(tr, 0.0);
  double wi[3];
  bool degenerate = false;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    bool keep = A[i][i] > tol;
    degenerate |= !keep;
    wi[i] = keep ? 1.0 / A[i][i] : 0.0;
  }
  int k = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j) {
      out6[k++] = Q[i][0] * wi[0] * Q[j][0] + Q[i][1] * wi[1] * Q[j][1] + Q[i][2] * wi[2] * Q[j][2];
    }
  return degenerate;
}

__device__ __forceinline__ void sym3_apply(const double* a6, const double* v, double* o) {
  // explicit fma chains: the same bits in every kernel that inlines this (implicit contraction
  // is chosen per inlining context and differed between k_lm_reduce and k_series)
  o[0] = fma(a6[2], v[2], fma(a6[1], v[1], a6[0] * v[0]));
  o[1] = fma(a6[4], v[2], fma(a6[3], v[1], a6[1] * v[0]));
  o[2] = fma(a6[5], v[2], fma(a6[4], v[1], a6[2] * v[0]));
}

__device__ __forceinline__ double damp_diag(double d, double lam) {
  double s = fmin(fmax(sqrt(d), 1e-6), 1e6);  // normal_eq.py:182-185
  return d + lam * (s * s);
}

// ---------------------------------------------------------------------------
// Givens-row update of a 4x4 upper-triangular R (packed row-major, 10 values:
// r00 r01 r02 r03 r11 r12 r13 r22 r23 r33) with a new row w (4).

__device__ __forceinline__ void givens_row(double* R, double w0, double w1, double w2, double w3) {
  double w[4] = {w0, w1, w2, w3};
  const int base[4] = {0, 4, 7, 9};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double wk = w[k];
    if (wk != 0.0) {
      double rkk = R[base[k]];
      double rho = hypot(rkk, wk);
      double c = rkk / rho, s = wk / rho;
      R[base[k]] = rho;
#pragma unroll
      for (int j = k + 1; j < 4; ++j) {
        double rkj = R[base[k] + (j - k)];
        R[base[k] + (j - k)] = fma(c, rkj, s * w[j]);
        w[j] = fma(-s, rkj, c * w[j]);
      }
    }
  }
}

// merge R <- qr([R; O]) for two packed 4x4 upper triangles
__device__ __forceinline__ void givens_merge(double* R, const double* O) {
  givens_row(R, O[0], O[1], O[2], O[3]);
  givens_row(R, 0.0, O[4], O[5], O[6]);
  givens_row(R, 0.0, 0.0, O[7], O[8]);
  givens_row(R, 0.0, 0.0, 0.0, O[9]);
}

// Min-norm least squares from R = qr([A | c]): returns -A^+ c in v and whether
// A is full rank at the reference tolerance s > 1e-10 s_max (objective.py:284-292),
// computed by a one-sided Jacobi SVD of the 3x3 triangle.
__device__ inline bool lsq_from_r(const double* R, double rel_tol, double* v) {
  // columns of R_A (3x3 upper triangle) and z = first 3 entries of column 4
  double M[3][3] = {{R[0], R[1], R[2]}, {0.0, R[4], R[5]}, {0.0, 0.0, R[7]}};  // M[row][col]
  double z[3] = {R[3], R[6], R[8]};
  double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 15; ++sweep) {
    bool rotated = false;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0;
      const int q = pq == 0 ? 1 : 2;
      double al = 0, be = 0, ga = 0;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        al = fma(M[i][p], M[i][p], al);
        be = fma(M[i][q], M[i][q], be);
        ga = fma(M[i][p], M[i][q], ga);
      }
      if (ga == 0.0 || fabs(ga) <= 2.220446049250313e-16 * sqrt(al * be)) continue;
      rotated = true;
      double zeta = (be - al) / (2.0 * ga);
      double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
      double c = 1.0 / sqrt(fma(t, t, 1.0));
      double s = c * t;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double mp = M[i][p], mq = M[i][q];
        M[i][p] = c * mp - s * mq;
        M[i][q] = s * mp + c * mq;
        double vp = V[i][p], vq = V[i][q];
        V[i][p] = c * vp - s * vq;
        V[i][q] = s * vp + c * vq;
      }
    }
    if (!rotated) break;
  }
  double s2[3], smax = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    s2[k] = M[0][k] * M[0][k] + M[1][k] * M[1][k] + M[2][k] * M[2][k];
    smax = fmax(smax, sqrt(s2[k]));
  }
  bool full = smax > 0.0;
  v[0] = v[1] = v[2] = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double sk = sqrt(s2[k]);
    bool keep = sk > rel_tol * smax;
    full &= keep;
    if (keep) {
      double coef = (M[0][k] * z[0] + M[1][k] * z[1] + M[2][k] * z[2]) / s2[k];
#pragma unroll
      for (int i = 0; i < 3; ++i) v[i] = fma(-coef, V[i][k], v[i]);
    }
  }
  return full;
}

}  // namespace pv
