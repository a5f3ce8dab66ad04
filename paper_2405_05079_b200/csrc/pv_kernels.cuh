// sm_100a kernels of the PoVar / RiPoBA hot path.  See DESIGN.md for the data
// layout and the roofline of each kernel.  Two traversal orders are used:
//
//  * landmark-major "tasks": one warp owns a run of whole landmarks whose
//    observations fit in 32 lanes (or one long landmark, looped in 32-obs
//    slabs).  Used by K1/K2 (k_lin_lm), K5 gather (k_phase1), K7 (back-sub),
//    K9 (k_cost) and K10 (k_resolve).  Segment sums use a deterministic
//    shuffle tree.
//  * camera-major "chunks": one warp owns <= PV_CHUNK consecutive
//    observations of a single camera (camera-sorted permutation).  Used by
//    K3 (k_lin_cam) and the K5 scatter half (k_phase2): per-camera sums are
//    register accumulations + a fixed-order chunk reduction, so no atomics and
//    bit-reproducible results.
#pragma once
#include "pv_device.cuh"

namespace pv {

constexpr int PV_CHUNK = 256;
constexpr int CREC = 24;  // camera record: P (12) | v (12)
constexpr int LREC = 8;   // landmark record: x (4) | t (4)
constexpr int LSYS = 8;   // V+ (6) | degenerate (1) | pad
constexpr int LINP = 90;  // camera linearization partial: U upper (78) | b_p (12)

enum { F_INVALID_Z = 0, F_ZERO_NORM = 1, F_SINGULAR_U = 2, F_N_DEGEN = 3, F_N_RANKDEF = 4,
       F_COUNT = 8 };

struct Graph {
  int n_p, n_l, n_o;
  int n_tasks, n_chunks;
  const int* ls_cam;     // [n_o] camera of each landmark-sorted observation
  const double* ls_m;    // [n_o*2]
  const int* lm_off;     // [n_l+1]
  const int* task_lm;    // [n_tasks+1]
  const int* cs_lm;      // [n_o] local landmark of each camera-sorted observation
  const double* cs_m;    // [n_o*2]
  const int* chunk_off;  // [n_chunks+1]
  const int* chunk_cam;  // [n_chunks]
  const int* cam_chunk;  // [n_p+1]
};

struct PowerCtl {
  int stopped;
  int order;
  int term;
  int pad;
  double trunc;
  double xnorm;
  double tnorm;
};

struct Coef {
  double s1, s2;  // sqrt(1-eta), sqrt(eta)
  double s;       // 1 - eta
};

// ---------------------------------------------------------------------------
// landmark task decoding

struct Task {
  int l0, l1, o0, n;
  bool long_task;
  unsigned heads;
};

__device__ __forceinline__ Task load_task(const Graph& g, int w, int lane) {
  Task t;
  t.l0 = g.task_lm[w];
  t.l1 = g.task_lm[w + 1];
  t.o0 = g.lm_off[t.l0];
  t.n = g.lm_off[t.l1] - t.o0;
  t.long_task = (t.l1 - t.l0 == 1) && t.n > 32;
  unsigned bit = 0;
  if (!t.long_task && lane < t.l1 - t.l0) bit = 1u << (g.lm_off[t.l0 + lane] - t.o0);
  t.heads = t.long_task ? 1u : __reduce_or_sync(PV_FULL, bit);
  return t;
}

__device__ __forceinline__ unsigned lanemask_le(int lane) { return 0xffffffffu >> (31 - lane); }

// local landmark and segment end of this lane in a short task
__device__ __forceinline__ void lane_segment(const Task& t, int lane, int& l, int& seg_end) {
  unsigned le = t.heads & lanemask_le(lane);
  l = t.l0 + __popc(le) - 1;
  unsigned gt = t.heads & ~lanemask_le(lane);
  seg_end = gt ? (__ffs(gt) - 1) : t.n;
  if (lane >= t.n) {
    l = t.l0;
    seg_end = t.n;
  }
}

__device__ __forceinline__ int seg_start_lane(const Task& t, int lane) {
  return 31 - __clz(t.heads & lanemask_le(lane));
}

// ---------------------------------------------------------------------------
// K5 gather half / K7: landmark-major  W^T v  (+ V+ and the landmark epilogue)

enum { P1_TERM = 0, P1_BACKSUB = 1 };

template <int STAGE>
__device__ __forceinline__ void wtv_obs(const double* __restrict__ crec, int cam, double m0,
                                        double m1, const double4& x, const Coef& k,
                                        double (&acc)[4]) {
  const double* c = crec + (size_t)cam * CREC;
  double4 P0 = ldg4(c), P1 = ldg4(c + 4), P2 = ldg4(c + 8);
  double4 v0 = ldg4(c + 12), v1 = ldg4(c + 16), v2 = ldg4(c + 20);
  Gen G = STAGE == 1 ? gen_s1(P0, P1, P2, m0, m1, k.s) : gen_s2(P0, P1, P2, x);
  double d0 = dot4(x, v0), d1 = dot4(x, v1), d2 = dot4(x, v2);
  acc[0] = fma(d0, G.g0.x, fma(d1, G.g1.x, fma(d2, G.g2.x, acc[0])));
  acc[1] = fma(d0, G.g0.y, fma(d1, G.g1.y, fma(d2, G.g2.y, acc[1])));
  acc[2] = fma(d0, G.g0.z, fma(d1, G.g1.z, fma(d2, G.g2.z, acc[2])));
  if (STAGE == 2) acc[3] = fma(d0, G.g0.w, fma(d1, G.g1.w, fma(d2, G.g2.w, acc[3])));
}

template <int STAGE, int MODE>
__device__ __forceinline__ void phase1_finish(int l, const double (&acc)[4], const double4& x,
                                              double* __restrict__ lrec,
                                              const double* __restrict__ lsys,
                                              const double* __restrict__ lbl,
                                              double* __restrict__ ldl, double* __restrict__ tlm,
                                              int* __restrict__ flags) {
  double s3[3], h[4];
  double xv[4] = {x.x, x.y, x.z, x.w};
  if (STAGE == 1) {
    s3[0] = acc[0];
    s3[1] = acc[1];
    s3[2] = acc[2];
  } else {
    householder_h<4>(xv, h);
    basis_apply_t<4>(h, acc, s3);
  }
  const double* vs = lsys + (size_t)l * LSYS;
  double vp[6] = {vs[0], vs[1], vs[2], vs[3], vs[4], vs[5]};
  if (MODE == P1_TERM) {
    double t[3];
    sym3_apply(vp, s3, t);
    if (STAGE == 1) {
      st4(lrec + (size_t)l * LREC + 4, make_double4(t[0], t[1], t[2], 0.0));
    } else {
      double t4[4];
      basis_apply<4>(h, t, t4);
      st4(lrec + (size_t)l * LREC + 4, make_double4(t4[0], t4[1], t4[2], t4[3]));
    }
  } else {
    const double* bl = lbl + (size_t)l * 4;
    double q[3] = {s3[0] + bl[0], s3[1] + bl[1], s3[2] + bl[2]};
    double dl[3];
    sym3_apply(vp, q, dl);
    bool degen = vs[6] != 0.0;
    for (int i = 0; i < 3; ++i) dl[i] = degen ? 0.0 : -dl[i];
    st4(ldl + (size_t)l * 4, make_double4(dl[0], dl[1], dl[2], 0.0));
    if (STAGE == 1) {
      st4(tlm + (size_t)l * 4, make_double4(x.x + dl[0], x.y + dl[1], x.z + dl[2], x.w));
    } else {
      double b[4];
      basis_apply<4>(h, dl, b);
      double y0 = x.x + b[0], y1 = x.y + b[1], y2 = x.z + b[2], y3 = x.w + b[3];
      double nn = sqrt(y0 * y0 + y1 * y1 + y2 * y2 + y3 * y3);
      if (nn == 0.0) {
        atomicOr(flags + F_ZERO_NORM, 1);
        nn = 1.0;
      }
      st4(tlm + (size_t)l * 4, make_double4(y0 / nn, y1 / nn, y2 / nn, y3 / nn));
    }
  }
}

template <int STAGE, int MODE>
__global__ void __launch_bounds__(256) k_phase1(Graph g, const double* __restrict__ crec,
                                                double* __restrict__ lrec,
                                                const double* __restrict__ lsys,
                                                const double* __restrict__ lbl,
                                                double* __restrict__ ldl, double* __restrict__ tlm,
                                                const PowerCtl* __restrict__ ctl, int* flags,
                                                Coef k) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= g.n_tasks) return;
  if (MODE == P1_TERM && ctl->stopped) return;
  Task t = load_task(g, w, lane);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (t.long_task) {
    double4 x = ldg4(lrec + (size_t)t.l0 * LREC);
    for (int o = t.o0 + lane; o < t.o0 + t.n; o += 32) {
      double2 m = ldg2(g.ls_m + 2 * (size_t)o);
      wtv_obs<STAGE>(crec, __ldg(g.ls_cam + o), m.x, m.y, x, k, acc);
    }
    warp_reduce_all(acc);
    if (lane == 0) phase1_finish<STAGE, MODE>(t.l0, acc, x, lrec, lsys, lbl, ldl, tlm, flags);
  } else {
    int l, seg_end;
    lane_segment(t, lane, l, seg_end);
    double4 x = ldg4(lrec + (size_t)l * LREC);
    if (lane < t.n) {
      int o = t.o0 + lane;
      double2 m = ldg2(g.ls_m + 2 * (size_t)o);
      wtv_obs<STAGE>(crec, __ldg(g.ls_cam + o), m.x, m.y, x, k, acc);
    }
    seg_reduce(acc, lane, seg_end);
    if (lane < t.n && ((t.heads >> lane) & 1u))
      phase1_finish<STAGE, MODE>(l, acc, x, lrec, lsys, lbl, ldl, tlm, flags);
  }
}

// ---------------------------------------------------------------------------
// K5 scatter half: camera-major  y_chunk = sum_j W_ij t_j

template <int STAGE>
__global__ void __launch_bounds__(256) k_phase2(Graph g, const double* __restrict__ crec,
                                                const double* __restrict__ lrec,
                                                double* __restrict__ cyc,
                                                const PowerCtl* __restrict__ ctl, int check_stop,
                                                Coef k) {
  const int lane = threadIdx.x & 31;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= g.n_chunks) return;
  if (check_stop && ctl->stopped) return;
  const int cam = __ldg(g.chunk_cam + c);
  const int o0 = __ldg(g.chunk_off + c), o1 = __ldg(g.chunk_off + c + 1);
  const double* cp = crec + (size_t)cam * CREC;
  const double4 P0 = ldg4(cp), P1 = ldg4(cp + 4), P2 = ldg4(cp + 8);
  double acc[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) acc[i] = 0.0;
#pragma unroll 2
  for (int o = o0 + lane; o < o1; o += 32) {
    const int j = __ldg(g.cs_lm + o);
    const double2 m = ldg2(g.cs_m + 2 * (size_t)o);
    const double* lr = lrec + (size_t)j * LREC;
    const double4 X = ldg4(lr), T = ldg4(lr + 4);
    Gen G = STAGE == 1 ? gen_s1(P0, P1, P2, m.x, m.y, k.s) : gen_s2(P0, P1, P2, X);
    const double sg[3] = {dot4(G.g0, T), dot4(G.g1, T), dot4(G.g2, T)};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      acc[4 * q + 0] = fma(sg[q], X.x, acc[4 * q + 0]);
      acc[4 * q + 1] = fma(sg[q], X.y, acc[4 * q + 1]);
      acc[4 * q + 2] = fma(sg[q], X.z, acc[4 * q + 2]);
      acc[4 * q + 3] = fma(sg[q], X.w, acc[4 * q + 3]);
    }
  }
  warp_reduce_all(acc);
  double mine = 0.0;
#pragma unroll
  for (int i = 0; i < 12; ++i)
    if (lane == i) mine = acc[i];
  if (lane < 12) cyc[(size_t)c * 12 + lane] = mine;
}

// ---------------------------------------------------------------------------
// K4/K6 epilogue: per camera (half-warp), reduce chunk partials, U^-1, series
// accumulation, stop test (last block), next term's camera vector.

enum { EPI_RHS = 0, EPI_TERM = 1, EPI_RAW = 2 };
enum { EPI_FULL = 0, EPI_REDUCE_ONLY = 1, EPI_APPLY_ONLY = 2 };

__device__ __forceinline__ double hw_sum(double v) {
#pragma unroll
  for (int d = 8; d > 0; d >>= 1) v += __shfl_xor_sync(PV_FULL, v, d, 16);
  return v;
}

template <int STAGE, int MODE>
__global__ void __launch_bounds__(256) k_epilogue(
    Graph g, double* __restrict__ crec, const double* __restrict__ cyc, double* __restrict__ cyr,
    const double* __restrict__ cbp, const double* __restrict__ cUi, double* __restrict__ cx,
    double* __restrict__ crhs, const double* __restrict__ ch, double* __restrict__ nrm,
    PowerCtl* __restrict__ ctl, volatile PowerCtl* host_ctl, unsigned* __restrict__ ticket,
    int part, int term, double thr) {
  __shared__ double red[2][256];
  __shared__ bool last;
  const int lane = threadIdx.x & 31;
  const int r = lane & 15;
  const int cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  if (MODE == EPI_TERM && ctl->stopped) return;  // uniform over the grid
  const bool valid = cam < g.n_p;
  constexpr int D = STAGE == 1 ? 12 : 11;
  double u = 0.0;
  if (valid && r < 12) {
    if (part == EPI_APPLY_ONLY) {
      u = cyr[(size_t)cam * 12 + r];
    } else {
      const int c0 = g.cam_chunk[cam], c1 = g.cam_chunk[cam + 1];
      for (int c = c0; c < c1; ++c) u += cyc[(size_t)c * 12 + r];
    }
  }
  if (part == EPI_REDUCE_ONLY) {
    if (valid && r < 12) cyr[(size_t)cam * 12 + r] = u;
    return;
  }
  double h = 0.0;
  if (STAGE == 2) {  // project y (12) -> tangent (11)
    h = (valid && r < 12) ? ch[(size_t)cam * 12 + r] : 0.0;
    double hu = hw_sum(h * u);
    double proj = u - 2.0 * h * hu;  // component r of H y
    u = __shfl_sync(PV_FULL, proj, (r + 1) & 15, 16);
    if (r >= 11) u = 0.0;
  }
  if (MODE == EPI_RAW) {
    if (valid && r < 12) cyr[(size_t)cam * 12 + r] = u;
    return;
  }
  double vin = u;
  if (MODE == EPI_RHS) {
    double b = (valid && r < D) ? cbp[(size_t)cam * 12 + r] : 0.0;
    vin = (r < D) ? -(b - u) : 0.0;
    if (valid && r < 12) crhs[(size_t)cam * 12 + r] = vin;
  }
  double t = 0.0;
  const double* Ui = cUi + (size_t)cam * 144 + r * 12;
#pragma unroll
  for (int kk = 0; kk < 12; ++kk) {
    double vk = __shfl_sync(PV_FULL, vin, kk, 16);
    if (valid && r < D && kk < D) t = fma(Ui[kk], vk, t);
  }
  double xr = 0.0;
  if (valid && r < D) {
    xr = MODE == EPI_RHS ? t : cx[(size_t)cam * 12 + r] + t;
    cx[(size_t)cam * 12 + r] = xr;
  }
  double v = t;
  if (STAGE == 2) {  // camera vector for the next gather: B t (11 -> 12)
    double tprev = __shfl_sync(PV_FULL, t, (r + 15) & 15, 16);  // t_{r-1}
    double e = (r >= 1 && r < 12) ? tprev : 0.0;
    double hd = hw_sum(h * e);
    v = e - 2.0 * h * hd;
  }
  if (valid && r < 12) crec[(size_t)cam * CREC + 12 + r] = v;
  double tn = hw_sum(r < D ? t * t : 0.0);
  double xn = hw_sum(r < D ? xr * xr : 0.0);
  if (valid && r == 0) {
    nrm[2 * (size_t)cam] = tn;
    nrm[2 * (size_t)cam + 1] = xn;
  }
  // ---- grid-wide fixed-order norm reduction in the last block
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned tk = atomicAdd(ticket, 1u);
    last = tk == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < g.n_p; i += blockDim.x) {
    a += __ldcg(nrm + 2 * (size_t)i);
    b += __ldcg(nrm + 2 * (size_t)i + 1);
  }
  red[0][threadIdx.x] = a;
  red[1][threadIdx.x] = b;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      red[0][threadIdx.x] += red[0][threadIdx.x + s];
      red[1][threadIdx.x] += red[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double TN = sqrt(red[0][0]), XN = sqrt(red[1][0]);
    PowerCtl c = *ctl;
    if (MODE == EPI_RHS) {  // solvers.py:134-139
      c.stopped = 0;
      c.order = 0;
      c.term = 0;
      c.trunc = XN > 0.0 ? 1.0 : 0.0;
    } else {  // solvers.py:140-149
      double ratio = XN > 0.0 ? TN / XN : 0.0;
      c.trunc = ratio;
      c.term = term;
      if (ratio <= thr) {
        c.order = term - 1;
        c.stopped = 1;
      } else {
        c.order = term;
      }
    }
    c.xnorm = XN;
    c.tnorm = TN;
    *ctl = c;
    host_ctl->stopped = c.stopped;
    host_ctl->order = c.order;
    host_ctl->term = c.term;
    host_ctl->trunc = c.trunc;
    host_ctl->xnorm = c.xnorm;
    host_ctl->tnorm = c.tnorm;
    __threadfence_system();
    *ticket = 0u;
  }
}

// ---------------------------------------------------------------------------
// K1 + K2 (landmark side of the linearization): V = sum Jl^T Jl, b_l = sum Jl^T r

template <int STAGE>
__device__ __forceinline__ void lin_lm_obs(const double* __restrict__ crec, int cam, double m0,
                                           double m1, const double4& x, const Coef& k,
                                           double (&acc)[14], int* flags) {
  const double* c = crec + (size_t)cam * CREC;
  double4 P0 = ldg4(c), P1 = ldg4(c + 4), P2 = ldg4(c + 8);
  double u0 = dot4(P0, x), u1 = dot4(P1, x), u2 = dot4(P2, x);
  if (STAGE == 1) {
    // objective.py:75-81,105-109
    double j[4][3] = {{k.s1 * (P0.x - m0 * P2.x), k.s1 * (P0.y - m0 * P2.y), k.s1 * (P0.z - m0 * P2.z)},
                      {k.s1 * (P1.x - m1 * P2.x), k.s1 * (P1.y - m1 * P2.y), k.s1 * (P1.z - m1 * P2.z)},
                      {k.s2 * P0.x, k.s2 * P0.y, k.s2 * P0.z},
                      {k.s2 * P1.x, k.s2 * P1.y, k.s2 * P1.z}};
    double rr[4] = {k.s1 * (u0 - u2 * m0), k.s1 * (u1 - u2 * m1), k.s2 * (u0 - m0),
                    k.s2 * (u1 - m1)};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      acc[0] = fma(j[q][0], j[q][0], acc[0]);
      acc[1] = fma(j[q][0], j[q][1], acc[1]);
      acc[2] = fma(j[q][0], j[q][2], acc[2]);
      acc[3] = fma(j[q][1], j[q][1], acc[3]);
      acc[4] = fma(j[q][1], j[q][2], acc[4]);
      acc[5] = fma(j[q][2], j[q][2], acc[5]);
      acc[6] = fma(j[q][0], rr[q], acc[6]);
      acc[7] = fma(j[q][1], rr[q], acc[7]);
      acc[8] = fma(j[q][2], rr[q], acc[8]);
    }
  } else {
    // objective.py:117-146
    if (!(fabs(u2) > 1e-12)) {
      atomicOr(flags + F_INVALID_Z, 1);
      return;
    }
    double iz = 1.0 / u2;
    double p0 = u0 * iz, p1 = u1 * iz;
    double J[2][4] = {{iz * (P0.x - p0 * P2.x), iz * (P0.y - p0 * P2.y), iz * (P0.z - p0 * P2.z), iz * (P0.w - p0 * P2.w)},
                      {iz * (P1.x - p1 * P2.x), iz * (P1.y - p1 * P2.y), iz * (P1.z - p1 * P2.z), iz * (P1.w - p1 * P2.w)}};
    double rr[2] = {u0 / u2 - m0, u1 / u2 - m1};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      int e = 0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = a; b < 4; ++b) {
          acc[e] = fma(J[q][a], J[q][b], acc[e]);
          ++e;
        }
#pragma unroll
      for (int a = 0; a < 4; ++a) acc[10 + a] = fma(J[q][a], rr[q], acc[10 + a]);
    }
  }
}

template <int STAGE>
__device__ __forceinline__ void lin_lm_finish(int l, const double (&acc)[14], const double4& x,
                                              double* __restrict__ lvr, double* __restrict__ lbl) {
  double V6[6], b3[3];
  if (STAGE == 1) {
    for (int i = 0; i < 6; ++i) V6[i] = acc[i];
    for (int i = 0; i < 3; ++i) b3[i] = acc[6 + i];
  } else {  // riemannian.py:67-85: B^T V B, B^T b with the Householder basis of x
    double xv[4] = {x.x, x.y, x.z, x.w}, h[4];
    householder_h<4>(xv, h);
    double V[4][4];
    int e = 0;
    for (int a = 0; a < 4; ++a)
      for (int b = a; b < 4; ++b) {
        V[a][b] = acc[e];
        V[b][a] = acc[e];
        ++e;
      }
    double w[4], al = 0.0;
    for (int a = 0; a < 4; ++a) {
      w[a] = V[a][0] * h[0] + V[a][1] * h[1] + V[a][2] * h[2] + V[a][3] * h[3];
      al = fma(h[a], w[a], al);
    }
    e = 0;
    for (int a = 1; a < 4; ++a)
      for (int b = a; b < 4; ++b) {
        V6[e++] = V[a][b] - 2.0 * h[a] * w[b] - 2.0 * w[a] * h[b] + 4.0 * al * h[a] * h[b];
      }
    double bb[4] = {acc[10], acc[11], acc[12], acc[13]};
    basis_apply_t<4>(h, bb, b3);
  }
  double* o = lvr + (size_t)l * 8;
  for (int i = 0; i < 6; ++i) o[i] = V6[i];
  st4(lbl + (size_t)l * 4, make_double4(b3[0], b3[1], b3[2], 0.0));
}

template <int STAGE>
__global__ void __launch_bounds__(256) k_lin_lm(Graph g, const double* __restrict__ crec,
                                                const double* __restrict__ lrec,
                                                double* __restrict__ lvr, double* __restrict__ lbl,
                                                int* flags, Coef k) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= g.n_tasks) return;
  Task t = load_task(g, w, lane);
  double acc[14];
#pragma unroll
  for (int i = 0; i < 14; ++i) acc[i] = 0.0;
  if (t.long_task) {
    double4 x = ldg4(lrec + (size_t)t.l0 * LREC);
    for (int o = t.o0 + lane; o < t.o0 + t.n; o += 32) {
      double2 m = ldg2(g.ls_m + 2 * (size_t)o);
      lin_lm_obs<STAGE>(crec, __ldg(g.ls_cam + o), m.x, m.y, x, k, acc, flags);
    }
    warp_reduce_all(acc);
    if (lane == 0) lin_lm_finish<STAGE>(t.l0, acc, x, lvr, lbl);
  } else {
    int l, seg_end;
    lane_segment(t, lane, l, seg_end);
    double4 x = ldg4(lrec + (size_t)l * LREC);
    if (lane < t.n) {
      int o = t.o0 + lane;
      double2 m = ldg2(g.ls_m + 2 * (size_t)o);
      lin_lm_obs<STAGE>(crec, __ldg(g.ls_cam + o), m.x, m.y, x, k, acc, flags);
    }
    seg_reduce(acc, lane, seg_end);
    if (lane < t.n && ((t.heads >> lane) & 1u)) lin_lm_finish<STAGE>(l, acc, x, lvr, lbl);
  }
}

// ---------------------------------------------------------------------------
// K3 (camera side of the linearization): U = sum (A (x) x x^T), b_p = sum h (x) x
// U[4c+a][4d+b] = sum A_cd x_a x_b,  b_p[4c+a] = sum h_c x_a.

__constant__ unsigned char c_lin_idx[LINP][3];  // record offsets of the three factors

template <int STAGE>
__global__ void __launch_bounds__(256) k_lin_cam(Graph g, const double* __restrict__ crec,
                                                 const double* __restrict__ lrec,
                                                 double* __restrict__ part, Coef k) {
  constexpr int RS = 15;  // record: x(4) A(6: 00 01 02 11 12 22) h(3) one(1) pad
  __shared__ double rec[8][32 * RS];
  const int lane = threadIdx.x & 31;
  const int wb = threadIdx.x >> 5;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= g.n_chunks) return;
  const int cam = __ldg(g.chunk_cam + c);
  const int o0 = __ldg(g.chunk_off + c), o1 = __ldg(g.chunk_off + c + 1);
  const double* cp = crec + (size_t)cam * CREC;
  const double4 P0 = ldg4(cp), P1 = ldg4(cp + 4), P2 = ldg4(cp + 8);
  int idx[3][3];
  bool has[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    int e = lane + 32 * q;
    has[q] = e < LINP;
    int ee = has[q] ? e : 0;
    idx[q][0] = c_lin_idx[ee][0];
    idx[q][1] = c_lin_idx[ee][1];
    idx[q][2] = c_lin_idx[ee][2];
  }
  double acc[3] = {0.0, 0.0, 0.0};
  double* my = &rec[wb][0];
  for (int base = o0; base < o1; base += 32) {
    const int o = base + lane;
    double r_[RS];
#pragma unroll
    for (int i = 0; i < RS; ++i) r_[i] = 0.0;
    if (o < o1) {
      const int j = __ldg(g.cs_lm + o);
      const double2 m = ldg2(g.cs_m + 2 * (size_t)o);
      const double4 X = ldg4(lrec + (size_t)j * LREC);
      r_[0] = X.x;
      r_[1] = X.y;
      r_[2] = X.z;
      r_[3] = X.w;
      double u0 = dot4(P0, X), u1 = dot4(P1, X), u2 = dot4(P2, X);
      if (STAGE == 1) {
        double s1 = k.s1, s2 = k.s2, a = s1 * s1;
        double rr0 = s1 * (u0 - u2 * m.x), rr1 = s1 * (u1 - u2 * m.y);
        double rr2 = s2 * (u0 - m.x), rr3 = s2 * (u1 - m.y);
        r_[4] = a + s2 * s2;
        r_[5] = 0.0;
        r_[6] = -a * m.x;
        r_[7] = a + s2 * s2;
        r_[8] = -a * m.y;
        r_[9] = a * (m.x * m.x + m.y * m.y);
        r_[10] = fma(s1, rr0, s2 * rr2);
        r_[11] = fma(s1, rr1, s2 * rr3);
        r_[12] = -s1 * fma(m.x, rr0, m.y * rr1);
        r_[13] = 1.0;
      } else {
        double iz = 1.0 / u2, i2 = iz * iz;
        double p0 = u0 * iz, p1 = u1 * iz;
        double rr0 = u0 / u2 - m.x, rr1 = u1 / u2 - m.y;
        r_[4] = i2;
        r_[5] = 0.0;
        r_[6] = -p0 * i2;
        r_[7] = i2;
        r_[8] = -p1 * i2;
        r_[9] = (p0 * p0 + p1 * p1) * i2;
        r_[10] = iz * rr0;
        r_[11] = iz * rr1;
        r_[12] = -iz * fma(p0, rr0, p1 * rr1);
        r_[13] = 1.0;
      }
    }
#pragma unroll
    for (int i = 0; i < RS; ++i) my[lane * RS + i] = r_[i];
    __syncwarp();
    const int nb = min(32, o1 - base);
    for (int qo = 0; qo < nb; ++qo) {
      const double* rq = my + qo * RS;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        if (has[q]) acc[q] = fma(rq[idx[q][0]] * rq[idx[q][1]], rq[idx[q][2]], acc[q]);
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int q = 0; q < 3; ++q)
    if (has[q]) part[(size_t)c * LINP + lane + 32 * q] = acc[q];
}

// per camera: sum chunk partials (fixed order) -> cUraw (90 per camera)
__global__ void k_lin_cam_reduce(Graph g, const double* __restrict__ part,
                                 double* __restrict__ cUraw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n_p * LINP) return;
  const int cam = i / LINP, e = i - cam * LINP;
  double s = 0.0;
  for (int c = g.cam_chunk[cam]; c < g.cam_chunk[cam + 1]; ++c) s += part[(size_t)c * LINP + e];
  cUraw[i] = s;
}

// per camera: unpack, project (stage 2), store U_lin (row stride 12) and b_p
template <int STAGE>
__global__ void k_lin_cam_project(int n_p, const double* __restrict__ cUraw,
                                  const double* __restrict__ crec, double* __restrict__ cU,
                                  double* __restrict__ cbp, double* __restrict__ ch) {
  const int cam = blockIdx.x * blockDim.x + threadIdx.x;
  if (cam >= n_p) return;
  const double* src = cUraw + (size_t)cam * LINP;
  double U[12][12];
  int e = 0;
  for (int i = 0; i < 12; ++i)
    for (int j = i; j < 12; ++j) {
      U[i][j] = src[e];
      U[j][i] = src[e];
      ++e;
    }
  double b[12];
  for (int i = 0; i < 12; ++i) b[i] = src[78 + i];
  double* uo = cU + (size_t)cam * 144;
  double* bo = cbp + (size_t)cam * 12;
  if (STAGE == 1) {
    for (int i = 0; i < 12; ++i) {
      for (int j = 0; j < 12; ++j) uo[i * 12 + j] = U[i][j];
      bo[i] = b[i];
    }
    return;
  }
  double p[12], h[12];
  for (int i = 0; i < 12; ++i) p[i] = crec[(size_t)cam * CREC + i];
  householder_h<12>(p, h);
  for (int i = 0; i < 12; ++i) ch[(size_t)cam * 12 + i] = h[i];
  double w[12], al = 0.0;
  for (int i = 0; i < 12; ++i) {
    double s = 0.0;
    for (int j = 0; j < 12; ++j) s = fma(U[i][j], h[j], s);
    w[i] = s;
    al = fma(h[i], s, al);
  }
  for (int i = 0; i < 12; ++i)
    for (int j = 0; j < 12; ++j)
      uo[i * 12 + j] = (i < 11 && j < 11)
                           ? U[i + 1][j + 1] - 2.0 * h[i + 1] * w[j + 1] -
                                 2.0 * w[i + 1] * h[j + 1] + 4.0 * al * h[i + 1] * h[j + 1]
                           : 0.0;
  double bt[11];
  basis_apply_t<12>(h, b, bt);
  for (int i = 0; i < 12; ++i) bo[i] = i < 11 ? bt[i] : 0.0;
}

// ---------------------------------------------------------------------------
// K3 damping + U^-1 (Cholesky; reference uses LU, difference <= 1e-13)

__global__ void k_damp_cam(int n_p, int D, const double* __restrict__ cU, double lam,
                           double* __restrict__ cUd, double* __restrict__ cUi, int* flags) {
  const int cam = blockIdx.x * blockDim.x + threadIdx.x;
  if (cam >= n_p) return;
  const double* a = cU + (size_t)cam * 144;
  double L[78];  // packed lower, row i starts at i(i+1)/2
  for (int i = 0; i < D; ++i)
    for (int j = 0; j <= i; ++j) {
      double v = a[i * 12 + j];
      if (i == j) v = damp_diag(v, lam);
      L[i * (i + 1) / 2 + j] = v;
    }
  double* ud = cUd + (size_t)cam * 144;
  for (int i = 0; i < 12; ++i)
    for (int j = 0; j < 12; ++j) {
      const int hi = max(i, j), lo = min(i, j);
      ud[i * 12 + j] = (i < D && j < D) ? L[hi * (hi + 1) / 2 + lo] : 0.0;
    }
  bool ok = true;
  for (int j = 0; j < D; ++j) {
    double d = L[j * (j + 1) / 2 + j];
    for (int kk = 0; kk < j; ++kk) d -= L[j * (j + 1) / 2 + kk] * L[j * (j + 1) / 2 + kk];
    if (!(d > 0.0)) {
      ok = false;
      d = 1.0;
    }
    d = sqrt(d);
    L[j * (j + 1) / 2 + j] = d;
    for (int i = j + 1; i < D; ++i) {
      double s = L[i * (i + 1) / 2 + j];
      for (int kk = 0; kk < j; ++kk) s -= L[i * (i + 1) / 2 + kk] * L[j * (j + 1) / 2 + kk];
      L[i * (i + 1) / 2 + j] = s / d;
    }
  }
  if (!ok) atomicOr(flags + F_SINGULAR_U, 1);
  // Linv (lower) in place
  double M[78];
  for (int i = 0; i < D; ++i) {
    M[i * (i + 1) / 2 + i] = 1.0 / L[i * (i + 1) / 2 + i];
    for (int j = 0; j < i; ++j) {
      double s = 0.0;
      for (int kk = j; kk < i; ++kk) s += L[i * (i + 1) / 2 + kk] * M[kk * (kk + 1) / 2 + j];
      M[i * (i + 1) / 2 + j] = -s / L[i * (i + 1) / 2 + i];
    }
  }
  double* ui = cUi + (size_t)cam * 144;
  for (int i = 0; i < 12; ++i)
    for (int j = 0; j < 12; ++j) {
      double s = 0.0;
      if (i < D && j < D) {
        for (int kk = max(i, j); kk < D; ++kk)
          s += M[kk * (kk + 1) / 2 + i] * M[kk * (kk + 1) / 2 + j];
      }
      ui[i * 12 + j] = s;
    }
}

// K2 damping + V+ (per landmark); also the RHS landmark vector t = V+ b_l
template <int STAGE>
__global__ void k_damp_lm(int n_l, const double* __restrict__ lvr, const double* __restrict__ lbl,
                          double* __restrict__ lrec, double* __restrict__ lsys, double lam,
                          int both, int* flags) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  bool degen = false;
  if (l < n_l) {
    const double* v = lvr + (size_t)l * 8;
    double V6[6] = {v[0], v[1], v[2], v[3], v[4], v[5]};
    if (both) {
      V6[0] = damp_diag(V6[0], lam);
      V6[3] = damp_diag(V6[3], lam);
      V6[5] = damp_diag(V6[5], lam);
    }
    double P6[6];
    degen = pinv_sym3(V6, 1e-10, P6);
    double* o = lsys + (size_t)l * LSYS;
    st4(o, make_double4(P6[0], P6[1], P6[2], P6[3]));
    st4(o + 4, make_double4(P6[4], P6[5], degen ? 1.0 : 0.0, 0.0));
  }
  unsigned bal = __ballot_sync(PV_FULL, degen);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(flags + F_N_DEGEN, __popc(bal));
}

// RHS landmark vector t = V+ b_l (normal_eq.py:221-226), lifted by B_lm in stage 2
template <int STAGE>
__global__ void k_lm_rhs_t(int n_l, const double* __restrict__ lbl,
                           const double* __restrict__ lsys, double* __restrict__ lrec) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= n_l) return;
  const double* vs = lsys + (size_t)l * LSYS;
  double P6[6] = {vs[0], vs[1], vs[2], vs[3], vs[4], vs[5]};
  const double* bl = lbl + (size_t)l * 4;
  double b3[3] = {bl[0], bl[1], bl[2]}, t[3];
  sym3_apply(P6, b3, t);
  if (STAGE == 1) {
    st4(lrec + (size_t)l * LREC + 4, make_double4(t[0], t[1], t[2], 0.0));
  } else {
    const double* xp = lrec + (size_t)l * LREC;
    double xv[4] = {xp[0], xp[1], xp[2], xp[3]}, h[4], t4[4];
    householder_h<4>(xv, h);
    basis_apply<4>(h, t, t4);
    st4(lrec + (size_t)l * LREC + 4, make_double4(t4[0], t4[1], t4[2], t4[3]));
  }
}

// camera vector for a gather pass: v = src (stage 1) or B src (stage 2)
template <int STAGE>
__global__ void k_setv(int n_p, const double* __restrict__ src, const double* __restrict__ ch,
                       double* __restrict__ crec) {
  const int cam = blockIdx.x * blockDim.x + threadIdx.x;
  if (cam >= n_p) return;
  double v[12];
  if (STAGE == 1) {
    for (int i = 0; i < 12; ++i) v[i] = src[(size_t)cam * 12 + i];
  } else {
    double h[12], t[11];
    for (int i = 0; i < 12; ++i) h[i] = ch[(size_t)cam * 12 + i];
    for (int i = 0; i < 11; ++i) t[i] = src[(size_t)cam * 12 + i];
    basis_apply<12>(h, t, v);
  }
  for (int i = 0; i < 12; ++i) crec[(size_t)cam * CREC + 12 + i] = v[i];
}

// K8 camera half of the trial state (solvers.py:311-315, riemannian.py:110-122)
template <int STAGE>
__global__ void k_trial_cam(int n_p, const double* __restrict__ crec, const double* __restrict__ cx,
                            const double* __restrict__ ch, double* __restrict__ tcam, int* flags) {
  const int cam = blockIdx.x * blockDim.x + threadIdx.x;
  if (cam >= n_p) return;
  double p[12];
  if (STAGE == 1) {
    for (int i = 0; i < 12; ++i) p[i] = crec[(size_t)cam * CREC + i] + cx[(size_t)cam * 12 + i];
  } else {
    double h[12], t[11], b[12];
    for (int i = 0; i < 12; ++i) h[i] = ch[(size_t)cam * 12 + i];
    for (int i = 0; i < 11; ++i) t[i] = cx[(size_t)cam * 12 + i];
    basis_apply<12>(h, t, b);
    double nn = 0.0;
    for (int i = 0; i < 12; ++i) {
      p[i] = crec[(size_t)cam * CREC + i] + b[i];
      nn = fma(p[i], p[i], nn);
    }
    nn = sqrt(nn);
    if (nn == 0.0) {
      atomicOr(flags + F_ZERO_NORM, 1);
      nn = 1.0;
    }
    for (int i = 0; i < 12; ++i) p[i] /= nn;
  }
  for (int i = 0; i < 12; ++i) tcam[(size_t)cam * 12 + i] = p[i];
}

// ---------------------------------------------------------------------------
// K9 cost (objective.py:194-211) and K10 closed-form landmark re-solve
// (objective.py:251-298), landmark-major, deterministic block partials.

template <int STAGE>
__device__ __forceinline__ double obs_cost(const double* __restrict__ cams, int cstride, int cam,
                                           double m0, double m1, const double4& x, const Coef& k,
                                           int* flags) {
  const double* c = cams + (size_t)cam * cstride;
  double4 P0 = ldg4(c), P1 = ldg4(c + 4), P2 = ldg4(c + 8);
  double u0 = dot4(P0, x), u1 = dot4(P1, x), u2 = dot4(P2, x);
  if (STAGE == 1) {
    double r0 = k.s1 * (u0 - u2 * m0), r1 = k.s1 * (u1 - u2 * m1);
    double r2 = k.s2 * (u0 - m0), r3 = k.s2 * (u1 - m1);
    return r0 * r0 + r1 * r1 + r2 * r2 + r3 * r3;
  }
  if (!(fabs(u2) > 1e-12)) {
    atomicOr(flags + F_INVALID_Z, 1);
    return 0.0;
  }
  double r0 = u0 / u2 - m0, r1 = u1 / u2 - m1;
  return r0 * r0 + r1 * r1;
}

__device__ __forceinline__ void block_partial(double v, double* __restrict__ out) {
  __shared__ double red[8];
  v = warp_sum(v);
  const int wb = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[wb] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    out[blockIdx.x] = s;
  }
}

template <int STAGE>
__global__ void __launch_bounds__(256) k_cost(Graph g, const double* __restrict__ cams, int cstride,
                                              const double* __restrict__ lms, int lstride,
                                              double* __restrict__ part, int* flags, Coef k) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double acc = 0.0;
  if (w < g.n_tasks) {
    Task t = load_task(g, w, lane);
    if (t.long_task) {
      double4 x = ldg4(lms + (size_t)t.l0 * lstride);
      for (int o = t.o0 + lane; o < t.o0 + t.n; o += 32) {
        double2 m = ldg2(g.ls_m + 2 * (size_t)o);
        acc += obs_cost<STAGE>(cams, cstride, __ldg(g.ls_cam + o), m.x, m.y, x, k, flags);
      }
    } else {
      int l, seg_end;
      lane_segment(t, lane, l, seg_end);
      if (lane < t.n) {
        double4 x = ldg4(lms + (size_t)l * lstride);
        int o = t.o0 + lane;
        double2 m = ldg2(g.ls_m + 2 * (size_t)o);
        acc = obs_cost<STAGE>(cams, cstride, __ldg(g.ls_cam + o), m.x, m.y, x, k, flags);
      }
    }
  }
  block_partial(acc, part);
}

__device__ __forceinline__ void resolve_rows(const double* __restrict__ cams, int cam, double m0,
                                             double m1, const Coef& k, double* R) {
  const double* c = cams + (size_t)cam * 12;
  double4 P0 = ldg4(c), P1 = ldg4(c + 4), P2 = ldg4(c + 8);
  // rows [A | c] of the affine model r = A v + c at x = (0, 0, 0, 1)
  givens_row(R, k.s1 * (P0.x - m0 * P2.x), k.s1 * (P0.y - m0 * P2.y), k.s1 * (P0.z - m0 * P2.z),
             k.s1 * (P0.w - P2.w * m0));
  givens_row(R, k.s1 * (P1.x - m1 * P2.x), k.s1 * (P1.y - m1 * P2.y), k.s1 * (P1.z - m1 * P2.z),
             k.s1 * (P1.w - P2.w * m1));
  givens_row(R, k.s2 * P0.x, k.s2 * P0.y, k.s2 * P0.z, k.s2 * (P0.w - m0));
  givens_row(R, k.s2 * P1.x, k.s2 * P1.y, k.s2 * P1.z, k.s2 * (P1.w - m1));
}

__global__ void __launch_bounds__(256) k_resolve(Graph g, const double* __restrict__ tcam,
                                                 double* __restrict__ tlm,
                                                 double* __restrict__ part, int* flags, Coef k) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double acc = 0.0;
  int rankdef = 0;
  if (w < g.n_tasks) {
    Task t = load_task(g, w, lane);
    double R[10];
#pragma unroll
    for (int i = 0; i < 10; ++i) R[i] = 0.0;
    if (t.long_task) {
      for (int o = t.o0 + lane; o < t.o0 + t.n; o += 32) {
        double2 m = ldg2(g.ls_m + 2 * (size_t)o);
        resolve_rows(tcam, __ldg(g.ls_cam + o), m.x, m.y, k, R);
      }
      for (int d = 16; d > 0; d >>= 1) {
        double O[10];
#pragma unroll
        for (int i = 0; i < 10; ++i) O[i] = __shfl_down_sync(PV_FULL, R[i], d);
        if (lane < d) givens_merge(R, O);
      }
      double xn[4] = {0.0, 0.0, 0.0, 0.0};
      if (lane == 0) {
        double v[3];
        bool full = lsq_from_r(R, 1e-10, v);
        double4 old = ld4(tlm + (size_t)t.l0 * 4);
        xn[0] = full ? v[0] : old.x;
        xn[1] = full ? v[1] : old.y;
        xn[2] = full ? v[2] : old.z;
        xn[3] = full ? 1.0 : old.w;
        rankdef = !full;
        st4(tlm + (size_t)t.l0 * 4, make_double4(xn[0], xn[1], xn[2], xn[3]));
      }
      double4 x;
      x.x = __shfl_sync(PV_FULL, xn[0], 0);
      x.y = __shfl_sync(PV_FULL, xn[1], 0);
      x.z = __shfl_sync(PV_FULL, xn[2], 0);
      x.w = __shfl_sync(PV_FULL, xn[3], 0);
      for (int o = t.o0 + lane; o < t.o0 + t.n; o += 32) {
        double2 m = ldg2(g.ls_m + 2 * (size_t)o);
        acc += obs_cost<1>(tcam, 12, __ldg(g.ls_cam + o), m.x, m.y, x, k, flags);
      }
    } else {
      int l, seg_end;
      lane_segment(t, lane, l, seg_end);
      int cam = 0;
      double2 m = make_double2(0.0, 0.0);
      if (lane < t.n) {
        int o = t.o0 + lane;
        m = ldg2(g.ls_m + 2 * (size_t)o);
        cam = __ldg(g.ls_cam + o);
        resolve_rows(tcam, cam, m.x, m.y, k, R);
      }
      for (int d = 1; d < 32; d <<= 1) {
        double O[10];
#pragma unroll
        for (int i = 0; i < 10; ++i) O[i] = __shfl_down_sync(PV_FULL, R[i], d);
        if (lane + d < seg_end) givens_merge(R, O);
      }
      double xn[4] = {0.0, 0.0, 0.0, 0.0};
      if (lane < t.n && ((t.heads >> lane) & 1u)) {
        double v[3];
        bool full = lsq_from_r(R, 1e-10, v);
        double4 old = ld4(tlm + (size_t)l * 4);
        xn[0] = full ? v[0] : old.x;
        xn[1] = full ? v[1] : old.y;
        xn[2] = full ? v[2] : old.z;
        xn[3] = full ? 1.0 : old.w;
        rankdef = !full;
        st4(tlm + (size_t)l * 4, make_double4(xn[0], xn[1], xn[2], xn[3]));
      }
      const int src = seg_start_lane(t, lane < t.n ? lane : 0);
      double4 x;
      x.x = __shfl_sync(PV_FULL, xn[0], src);
      x.y = __shfl_sync(PV_FULL, xn[1], src);
      x.z = __shfl_sync(PV_FULL, xn[2], src);
      x.w = __shfl_sync(PV_FULL, xn[3], src);
      if (lane < t.n) acc = obs_cost<1>(tcam, 12, cam, m.x, m.y, x, k, flags);
    }
  }
  unsigned bal = __ballot_sync(PV_FULL, rankdef);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(flags + F_N_RANKDEF, __popc(bal));
  block_partial(acc, part);
}

// fixed-order single-block sum of block partials
__global__ void k_sum(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

// trial -> current
__global__ void k_accept(int n_p, int n_l, const double* __restrict__ tcam,
                         const double* __restrict__ tlm, double* __restrict__ crec,
                         double* __restrict__ lrec) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_p)
    for (int q = 0; q < 12; ++q) crec[(size_t)i * CREC + q] = tcam[(size_t)i * 12 + q];
  if (i < n_l) st4(lrec + (size_t)i * LREC, ld4(tlm + (size_t)i * 4));
}

// state upload helpers
__global__ void k_put_state(int n_p, int n_l, const double* __restrict__ cams,
                            const double* __restrict__ lms, double* __restrict__ crec,
                            double* __restrict__ lrec) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_p)
    for (int q = 0; q < 12; ++q) crec[(size_t)i * CREC + q] = cams[(size_t)i * 12 + q];
  if (i < n_l)
    for (int q = 0; q < 4; ++q) lrec[(size_t)i * LREC + q] = lms[(size_t)i * 4 + q];
}

__global__ void k_get_state(int n_p, int n_l, const double* __restrict__ crec,
                            const double* __restrict__ lrec, double* __restrict__ cams,
                            double* __restrict__ lms) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_p)
    for (int q = 0; q < 12; ++q) cams[(size_t)i * 12 + q] = crec[(size_t)i * CREC + q];
  if (i < n_l)
    for (int q = 0; q < 4; ++q) lms[(size_t)i * 4 + q] = lrec[(size_t)i * LREC + q];
}

// debug: W blocks per landmark-sorted observation (tangent-projected in stage 2)
template <int STAGE>
__global__ void k_debug_w(Graph g, const double* __restrict__ crec, const double* __restrict__ lrec,
                          const double* __restrict__ ch, double* __restrict__ out, Coef k) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= g.n_l) return;
  const double* xp = lrec + (size_t)l * LREC;
  double4 x = make_double4(xp[0], xp[1], xp[2], xp[3]);
  double xv[4] = {x.x, x.y, x.z, x.w}, hl[4];
  if (STAGE == 2) householder_h<4>(xv, hl);
  for (int o = g.lm_off[l]; o < g.lm_off[l + 1]; ++o) {
    const int cam = g.ls_cam[o];
    const double* c = crec + (size_t)cam * CREC;
    double4 P0 = make_double4(c[0], c[1], c[2], c[3]), P1 = make_double4(c[4], c[5], c[6], c[7]),
            P2 = make_double4(c[8], c[9], c[10], c[11]);
    double m0 = g.ls_m[2 * (size_t)o], m1 = g.ls_m[2 * (size_t)o + 1];
    Gen G = STAGE == 1 ? gen_s1(P0, P1, P2, m0, m1, k.s) : gen_s2(P0, P1, P2, x);
    double gg[3][4] = {{G.g0.x, G.g0.y, G.g0.z, G.g0.w}, {G.g1.x, G.g1.y, G.g1.z, G.g1.w},
                       {G.g2.x, G.g2.y, G.g2.z, G.g2.w}};
    double W[12][4];
    for (int cc = 0; cc < 3; ++cc)
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) W[4 * cc + a][b] = xv[a] * gg[cc][b];
    double* wo = out + (size_t)o * 36;
    if (STAGE == 1) {
      for (int i = 0; i < 12; ++i)
        for (int b = 0; b < 3; ++b) wo[i * 3 + b] = W[i][b];
    } else {
      double hc[12];
      for (int i = 0; i < 12; ++i) hc[i] = ch[(size_t)cam * 12 + i];
      // Wt = Bc^T W Bl : (11 x 3)
      double WB[12][3];
      for (int i = 0; i < 12; ++i) basis_apply_t<4>(hl, W[i], WB[i]);
      for (int b = 0; b < 3; ++b) {
        double col[12], pc[11];
        for (int i = 0; i < 12; ++i) col[i] = WB[i][b];
        basis_apply_t<12>(hc, col, pc);
        for (int i = 0; i < 11; ++i) wo[i * 3 + b] = pc[i];
      }
      for (int b = 0; b < 3; ++b) wo[33 + b] = 0.0;
    }
  }
}

}  // namespace pv
