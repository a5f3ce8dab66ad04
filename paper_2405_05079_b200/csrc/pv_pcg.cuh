// Block-Jacobi preconditioned conjugate gradients on the reduced camera system
// (the reference's "iterative" / "ripcg" inner solver, solvers.py:153-187), on
// the device.  The S'.p product is the L2-blocked term of pv_kernels.cuh; this
// header adds
//
//   k_schur_diag    exact block diagonal  U_i - sum_j W_ij V+_j W_ij^T
//                   (normal_eq.py:253-260) without materialising W:
//                   W_ij V+ W_ij^T = G_ij (x) x_j x_j^T with
//                   G_ij[c][c'] = g~_c V+_j g~_c'  (3x3, the landmark-projected
//                   generator rows), so a camera accumulates 6 x 10 moments
//   k_diag_finish   12x12 assembly, stage-2 tangent projection, U - sum
//   k_inv_lu / k_pinv_jacobi   the np.linalg.inv / _pinv_psd(diag, 1e-12)
//                   fallbacks of solvers.py:163-166
//   k_pcg_init / k_pcg_curv / k_pcg_update / k_pcg_dir   the vector recurrences,
//                   one warp per camera, with fixed-order grid reductions in the
//                   last CTA (deterministic) and the stop decision written to the
//                   shared PowerCtl so the term kernels of later (look-ahead)
//                   iterations return immediately.
#pragma once

#include "pv_kernels.cuh"

namespace pv {

// thread (c, c') of the 6 unique entries of a symmetric 3x3, and (a, b) of 10 of a 4x4
__device__ __forceinline__ int sym3_idx(int i, int j) {
  const int lo = min(i, j), hi = max(i, j);
  return lo == 0 ? hi : (lo == 1 ? 2 + hi : 5);
}
__device__ __forceinline__ int sym4_idx(int i, int j) {
  const int lo = min(i, j), hi = max(i, j);
  // rows: (0,0..3) 0-3, (1,1..3) 4-6, (2,2..3) 7-8, (3,3) 9
  return lo == 0 ? hi : (lo == 1 ? 3 + hi : (lo == 2 ? 5 + hi : 9));
}

// fixed-order sum of NV per-camera partials in the last CTA to finish (thread 0 gets
// the totals).  Deterministic for a fixed blockDim.
template <int NV>
__device__ __forceinline__ bool last_cta_sum(const double* part, int n, unsigned* ticket,
                                             double (&tot)[NV]) {
  __shared__ bool last;
  __shared__ double rr[NV][32];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double a[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) a[v] = 0.0;
  strided_sum_ordered<NV>(part, n, a);
  warp_reduce_all(a);
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int v = 0; v < NV; ++v) rr[v][threadIdx.x >> 5] = a[v];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double s = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += rr[v][q];
      tot[v] = s;
    }
    *ticket = 0u;
  }
  return true;
}

// ---------------------------------------------------------------------------
// exact block diagonal of the reduced system

// one warp per camera: the 60 moments sum_j G_ij[q] * (x_j x_j^T)[r] -> mom[cam*60 + q*10 + r]
template <int STAGE>
__global__ void __launch_bounds__(256) k_schur_diag(Graph g, const double* __restrict__ crec,
                                                    const double* __restrict__ cs_x,
                                                    const double* __restrict__ lsys,
                                                    double* __restrict__ mom, Coef k) {
  const int lane = threadIdx.x & 31;
  const int cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (cam >= g.n_p) return;
  const double* cp = crec + (size_t)cam * CREC;
  const double4 P0 = ldg4(cp), P1 = ldg4(cp + 4), P2 = ldg4(cp + 8);
  double acc[60];
#pragma unroll
  for (int i = 0; i < 60; ++i) acc[i] = 0.0;
  for (int b = 0; b < g.n_blk; ++b) {
    const int o_lo = __ldg(g.seg + (size_t)b * g.n_p + cam);
    const int o_hi = __ldg(g.seg + (size_t)b * g.n_p + cam + 1);
    for (int o = o_lo + lane; o < o_hi; o += 32) {
      const double4 X = ldg4(cs_x + 4 * (size_t)o);
      const double2 m = ldg2(g.cs_m + 2 * (size_t)o);
      const int l = __ldg(g.cs_kpos + o);  // slot position of V+
      const Gen G = STAGE == 1 ? gen_s1(P0, P1, P2, m.x, m.y, k.s) : gen_s2(P0, P1, P2, X);
      const double4 gr[3] = {G.g0, G.g1, G.g2};
      double gt[3][3];
      if (STAGE == 1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          gt[c][0] = gr[c].x;
          gt[c][1] = gr[c].y;
          gt[c][2] = gr[c].z;
        }
      } else {
        double xv[4] = {X.x, X.y, X.z, X.w}, h[4];
        householder_h<4>(xv, h);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double gv[4] = {gr[c].x, gr[c].y, gr[c].z, gr[c].w};
          basis_apply_t<4>(h, gv, gt[c]);
        }
      }
      const double4 va = ldg4(lsys + (size_t)l * LSYS), vb = ldg4(lsys + (size_t)l * LSYS + 4);
      const double vp[6] = {va.x, va.y, va.z, va.w, vb.x, vb.y};
      double Gq[6];
      {
        double u[3][3];
#pragma unroll
        for (int c = 0; c < 3; ++c) sym3_apply(vp, gt[c], u[c]);
        Gq[0] = gt[0][0] * u[0][0] + gt[0][1] * u[0][1] + gt[0][2] * u[0][2];
        Gq[1] = gt[0][0] * u[1][0] + gt[0][1] * u[1][1] + gt[0][2] * u[1][2];
        Gq[2] = gt[0][0] * u[2][0] + gt[0][1] * u[2][1] + gt[0][2] * u[2][2];
        Gq[3] = gt[1][0] * u[1][0] + gt[1][1] * u[1][1] + gt[1][2] * u[1][2];
        Gq[4] = gt[1][0] * u[2][0] + gt[1][1] * u[2][1] + gt[1][2] * u[2][2];
        Gq[5] = gt[2][0] * u[2][0] + gt[2][1] * u[2][1] + gt[2][2] * u[2][2];
      }
      const double xa[4] = {X.x, X.y, X.z, X.w};
      double XX[10];
      {
        int r = 0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int bb = a; bb < 4; ++bb) XX[r++] = xa[a] * xa[bb];
      }
#pragma unroll
      for (int q = 0; q < 6; ++q)
#pragma unroll
        for (int r = 0; r < 10; ++r) acc[q * 10 + r] = fma(Gq[q], XX[r], acc[q * 10 + r]);
    }
  }
  warp_reduce_all(acc);
  double mine0 = 0.0, mine1 = 0.0;
#pragma unroll
  for (int i = 0; i < 60; ++i) {
    if (lane == (i & 31)) {
      if (i < 32) mine0 = acc[i];
      else mine1 = acc[i];
    }
  }
  mom[(size_t)cam * 60 + lane] = mine0;
  if (lane < 28) mom[(size_t)cam * 60 + 32 + lane] = mine1;
}

// one warp per camera, lane i < 12 owns row i: A = sum G (x) xx^T, stage-2 tangent
// projection B^T A B = (H A H)[1:, 1:], S = U_damped - A  -> sd (12x12 layout, D used)
template <int STAGE>
__global__ void k_diag_finish(int n_p, const double* __restrict__ mom,
                              const double* __restrict__ ch, const double* __restrict__ cUd,
                              double* __restrict__ sd) {
  constexpr int D = STAGE == 1 ? 12 : 11;
  __shared__ double sm[8][60];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (cam >= n_p) return;
  sm[w][lane] = mom[(size_t)cam * 60 + lane];
  if (lane < 28) sm[w][32 + lane] = mom[(size_t)cam * 60 + 32 + lane];
  __syncwarp();
  const int i = lane < 12 ? lane : 0;
  double row[12];
#pragma unroll
  for (int j = 0; j < 12; ++j)
    row[j] = sm[w][sym3_idx(i >> 2, j >> 2) * 10 + sym4_idx(i & 3, j & 3)];
  double out[12];
  if (STAGE == 1) {
#pragma unroll
    for (int j = 0; j < 12; ++j) out[j] = row[j];
  } else {
    double h[12];
#pragma unroll
    for (int j = 0; j < 12; ++j) h[j] = ch[(size_t)cam * 12 + j];
    double u = 0.0;  // (A h)_i
#pragma unroll
    for (int j = 0; j < 12; ++j) u = fma(row[j], h[j], u);
    const double hi = h[i];
    const double s = warp_sum(lane < 12 ? hi * u : 0.0);  // h^T A h
    double uj[12];
#pragma unroll
    for (int j = 0; j < 12; ++j) uj[j] = __shfl_sync(PV_FULL, u, j);
    // (H A H)[i][j] = A - 2 h_i u_j - 2 u_i h_j + 4 s h_i h_j ; keep [1:, 1:]
    double full[12];
#pragma unroll
    for (int j = 0; j < 12; ++j)
      full[j] = row[j] - 2.0 * hi * uj[j] - 2.0 * u * h[j] + 4.0 * s * hi * h[j];
    // shift: tangent row i-1 <- full row i (lane i+1 -> lane i), columns 1..11 -> 0..10
#pragma unroll
    for (int j = 0; j < 12; ++j) {
      const double v = __shfl_sync(PV_FULL, full[j], (lane + 1) & 31);
      if (j >= 1) out[j - 1] = v;
    }
    out[11] = 0.0;
  }
  if (lane < 12) {
    const double* ud = cUd + (size_t)cam * 144 + lane * 12;
    double* o = sd + (size_t)cam * 144 + lane * 12;
#pragma unroll
    for (int j = 0; j < 12; ++j) o[j] = (lane < D && j < D) ? ud[j] - out[j] : 0.0;
  }
}

// np.linalg.inv semantics for the whole batch (LU with partial pivoting, here as
// Gauss-Jordan); sets flags[F_SINGULAR_M2] on an exactly singular block
__global__ void k_inv_lu(int n_p, int D, const double* __restrict__ sd, double* __restrict__ mi,
                         int* flags) {
  const int cam = blockIdx.x * blockDim.x + threadIdx.x;
  if (cam >= n_p) return;
  double a[12][24];
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) {
      a[i][j] = sd[(size_t)cam * 144 + i * 12 + j];
      a[i][D + j] = i == j ? 1.0 : 0.0;
    }
  bool sing = false;
  for (int c = 0; c < D; ++c) {
    int piv = c;
    for (int r = c + 1; r < D; ++r)
      if (fabs(a[r][c]) > fabs(a[piv][c])) piv = r;
    if (a[piv][c] == 0.0) {
      sing = true;
      break;
    }
    if (piv != c)
      for (int j = 0; j < 2 * D; ++j) {
        const double t = a[c][j];
        a[c][j] = a[piv][j];
        a[piv][j] = t;
      }
    const double inv = 1.0 / a[c][c];
    for (int j = 0; j < 2 * D; ++j) a[c][j] *= inv;
    for (int r = 0; r < D; ++r) {
      if (r == c) continue;
      const double f = a[r][c];
      if (f != 0.0)
        for (int j = 0; j < 2 * D; ++j) a[r][j] -= f * a[c][j];
    }
  }
  if (sing) atomicOr(flags + F_SINGULAR_M2, 1);
  for (int i = 0; i < 12; ++i)
    for (int j = 0; j < 12; ++j)
      mi[(size_t)cam * 144 + i * 12 + j] = (!sing && i < D && j < D) ? a[i][D + j] : 0.0;
}

// _pinv_psd(diag, 1e-12) (normal_eq.py:145-153): cyclic Jacobi eigen-decomposition,
// eigenvalues w <= 1e-12 * max(trace, 0) dropped
__global__ void k_pinv_jacobi(int n_p, int D, const double* __restrict__ sd,
                              double* __restrict__ mi) {
  const int cam = blockIdx.x * blockDim.x + threadIdx.x;
  if (cam >= n_p) return;
  double a[12][12], q[12][12];
  double tr = 0.0;
  for (int i = 0; i < D; ++i) {
    for (int j = 0; j < D; ++j) {
      a[i][j] = sd[(size_t)cam * 144 + i * 12 + j];
      q[i][j] = i == j ? 1.0 : 0.0;
    }
    tr += a[i][i];
  }
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int i = 0; i < D; ++i) {
      dia += a[i][i] * a[i][i];
      for (int j = i + 1; j < D; ++j) off += a[i][j] * a[i][j];
    }
    if (!(off > 1e-32 * dia)) break;
    for (int p = 0; p < D; ++p)
      for (int r = p + 1; r < D; ++r) {
        const double apr = a[p][r];
        if (apr == 0.0) continue;
        const double theta = (a[r][r] - a[p][p]) / (2.0 * apr);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < D; ++k) {  // A <- A J
          const double akp = a[k][p], akr = a[k][r];
          a[k][p] = c * akp - s * akr;
          a[k][r] = s * akp + c * akr;
        }
        for (int k = 0; k < D; ++k) {  // A <- J^T A
          const double apk = a[p][k], ark = a[r][k];
          a[p][k] = c * apk - s * ark;
          a[r][k] = s * apk + c * ark;
        }
        for (int k = 0; k < D; ++k) {
          const double qkp = q[k][p], qkr = q[k][r];
          q[k][p] = c * qkp - s * qkr;
          q[k][r] = s * qkp + c * qkr;
        }
      }
  }
  const double tol = 1e-12 * fmax(tr, 0.0);
  double wi[12];
  for (int i = 0; i < D; ++i) wi[i] = a[i][i] > tol ? 1.0 / a[i][i] : 0.0;
  for (int i = 0; i < 12; ++i)
    for (int j = 0; j < 12; ++j) {
      double s = 0.0;
      if (i < D && j < D)
        for (int k = 0; k < D; ++k) s += q[i][k] * wi[k] * q[j][k];
      mi[(size_t)cam * 144 + i * 12 + j] = s;
    }
}

// ---------------------------------------------------------------------------
// CG recurrences (solvers.py:167-187); one warp per camera, lane r < D owns row r

__device__ __forceinline__ double block_apply_row(const double* __restrict__ M, int cam, int lane,
                                                  int D, double v) {
  double t = 0.0;
  const double* Mr = M + (size_t)cam * 144 + (lane < D ? lane : 0) * 12;
#pragma unroll
  for (int kk = 0; kk < 12; ++kk) {
    const double vk = __shfl_sync(PV_FULL, v, kk);
    if (lane < D && kk < D) t = fma(Mr[kk], vk, t);
  }
  return t;
}

// v = B p (stage 2, 11 -> 12) / p (stage 1) into the camera record slot read by the term
template <int STAGE>
__device__ __forceinline__ void store_camera_vector(double* __restrict__ crec,
                                                    const double* __restrict__ ch, int cam,
                                                    int lane, double p) {
  double v = p;
  if (STAGE == 2) {
    const double h = lane < 12 ? ch[(size_t)cam * 12 + lane] : 0.0;
    const double pprev = __shfl_sync(PV_FULL, p, (lane + 31) & 31);
    const double e = (lane >= 1 && lane < 12) ? pprev : 0.0;
    const double hd = warp_sum(h * e);
    v = fma(-2.0 * h, hd, e);
  }
  if (lane < 12) crec[(size_t)cam * CREC + 12 + lane] = v;
}

__device__ __forceinline__ void publish(PowerCtl* ctl, volatile PowerCtl* host_ctl,
                                        const PowerCtl& c) {
  *ctl = c;
  // `order` (the iteration that stopped) before `stopped`: see op_pcg's look-ahead loop
  host_ctl->order = c.order;
  host_ctl->pad = c.pad;
  host_ctl->trunc = c.trunc;
  __threadfence_system();
  host_ctl->stopped = c.stopped;
  __threadfence_system();
}

struct PcgVec {
  double *x, *r, *z, *p, *sp;  // n_p x 12 each
};

// r = rhs, x = 0, z = M^-1 r, p = z; rhs norm and r.z
template <int STAGE>
__global__ void k_pcg_init(int n_p, const double* __restrict__ crhs, const double* __restrict__ mi,
                           const double* __restrict__ ch, double* __restrict__ crec, PcgVec v,
                           double* __restrict__ part, PowerCtl* ctl, volatile PowerCtl* host_ctl,
                           unsigned* ticket) {
  constexpr int D = STAGE == 1 ? 12 : 11;
  const int lane = threadIdx.x & 31;
  const int cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (cam < n_p) {
    const bool row = lane < D;
    const double r = row ? crhs[(size_t)cam * 12 + lane] : 0.0;
    const double z = block_apply_row(mi, cam, lane, D, r);
    if (lane < 12) {
      v.x[(size_t)cam * 12 + lane] = 0.0;
      v.r[(size_t)cam * 12 + lane] = r;
      v.z[(size_t)cam * 12 + lane] = z;
      v.p[(size_t)cam * 12 + lane] = z;
    }
    store_camera_vector<STAGE>(crec, ch, cam, lane, z);
    const double rr = warp_sum(r * r), rz = warp_sum(r * z);
    if (lane == 0) {
      part[2 * (size_t)cam] = rr;
      part[2 * (size_t)cam + 1] = rz;
    }
  }
  double tot[2];
  if (!last_cta_sum<2>(part, n_p, ticket, tot) || threadIdx.x != 0) return;
  PowerCtl c{};
  c.rhs_norm = sqrt(tot[0]);
  c.rz = tot[1];
  c.order = 0;                                   // iterations
  c.trunc = c.rhs_norm == 0.0 ? 0.0 : 1.0;       // rel
  c.stopped = c.rhs_norm == 0.0 ? 1 : 0;         // zero RHS: x = 0, no iteration
  c.pad = 0;
  publish(ctl, host_ctl, c);
}

// sp = U p - S'p (y from the term kernels), curvature p.sp, alpha; breakdown stop
template <int STAGE>
__global__ void k_pcg_curv(int n_p, int it, const double* __restrict__ cy,
                           const double* __restrict__ ch, const double* __restrict__ cUd, PcgVec v,
                           double* __restrict__ part, PowerCtl* ctl, volatile PowerCtl* host_ctl,
                           unsigned* ticket) {
  constexpr int D = STAGE == 1 ? 12 : 11;
  if (ctl->stopped) return;  // grid-uniform
  const int lane = threadIdx.x & 31;
  const int cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (cam < n_p) {
    double u = lane < 12 ? cy[(size_t)cam * 12 + lane] : 0.0;
    if (STAGE == 2) {  // raw 12 -> tangent 11
      const double h = lane < 12 ? ch[(size_t)cam * 12 + lane] : 0.0;
      const double hu = warp_sum(h * u);
      const double pr = fma(-2.0 * h, hu, u);
      u = __shfl_sync(PV_FULL, pr, (lane + 1) & 31);
    }
    const double p = lane < D ? v.p[(size_t)cam * 12 + lane] : 0.0;
    const double up = block_apply_row(cUd, cam, lane, D, p);
    const double sp = lane < D ? up - u : 0.0;
    if (lane < 12) v.sp[(size_t)cam * 12 + lane] = sp;
    const double ps = warp_sum(p * sp);
    if (lane == 0) part[cam] = ps;
  }
  double tot[1];
  if (!last_cta_sum<1>(part, n_p, ticket, tot) || threadIdx.x != 0) return;
  PowerCtl c = *ctl;
  c.order = it >= 0 ? it : c.order + 1;  // iterations = it (solvers.py:174); -1: count here
                                          // (the iteration replayed as a captured graph)
  if (tot[0] <= 0.0) {  // solvers.py:177-179
    c.stopped = 1;
    c.pad = 1;  // "breakdown"
  } else {
    c.alpha = c.rz / tot[0];
  }
  publish(ctl, host_ctl, c);
}

// x += alpha p, r -= alpha sp, rel = |r| / |rhs| (stop), z = M^-1 r, beta
template <int STAGE>
__global__ void k_pcg_update(int n_p, double tol, const double* __restrict__ mi, PcgVec v,
                             double* __restrict__ part, PowerCtl* ctl, volatile PowerCtl* host_ctl,
                             unsigned* ticket) {
  constexpr int D = STAGE == 1 ? 12 : 11;
  if (ctl->stopped) return;
  const double alpha = ctl->alpha;
  const int lane = threadIdx.x & 31;
  const int cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (cam < n_p) {
    const size_t o = (size_t)cam * 12 + (lane < 12 ? lane : 0);
    double r = 0.0;
    if (lane < D) {
      v.x[o] = fma(alpha, v.p[o], v.x[o]);
      r = fma(-alpha, v.sp[o], v.r[o]);
      v.r[o] = r;
    }
    const double z = block_apply_row(mi, cam, lane, D, r);
    if (lane < D) v.z[o] = z;
    const double rr = warp_sum(r * r), rz = warp_sum(r * z);
    if (lane == 0) {
      part[2 * (size_t)cam] = rr;
      part[2 * (size_t)cam + 1] = rz;
    }
  }
  double tot[2];
  if (!last_cta_sum<2>(part, n_p, ticket, tot) || threadIdx.x != 0) return;
  PowerCtl c = *ctl;
  c.trunc = sqrt(tot[0]) / c.rhs_norm;  // rel (solvers.py:183)
  if (c.trunc <= tol) {
    c.stopped = 1;
  } else {
    c.beta = tot[1] / c.rz;
    c.rz = tot[1];
  }
  publish(ctl, host_ctl, c);
}

// p = z + beta p, and the camera vector of the next S'.p
template <int STAGE>
__global__ void k_pcg_dir(int n_p, const double* __restrict__ ch, double* __restrict__ crec,
                          PcgVec v, const PowerCtl* ctl) {
  constexpr int D = STAGE == 1 ? 12 : 11;
  if (ctl->stopped) return;
  const double beta = ctl->beta;
  const int lane = threadIdx.x & 31;
  const int cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (cam >= n_p) return;
  const size_t o = (size_t)cam * 12 + (lane < 12 ? lane : 0);
  double p = 0.0;
  if (lane < D) {
    p = fma(beta, v.p[o], v.z[o]);
    v.p[o] = p;
  }
  store_camera_vector<STAGE>(crec, ch, cam, lane, p);
}

}  // namespace pv
