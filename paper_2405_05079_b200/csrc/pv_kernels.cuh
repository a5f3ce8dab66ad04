// sm_100a kernels of the PoVar / RiPoBA hot path.  See DESIGN.md for the data
// layout and the roofline of each kernel.  Two traversal orders are used:
//
//  * camera-major: one CTA owns one camera and streams that camera's
//    observations (camera-sorted copies of m and x).  Camera data (P, the term
//    vector v, U^-1) is CTA-uniform, so it is read once per CTA instead of once
//    per observation.  Used by the fused power-series term kernel k_cam
//    (K5 scatter half + K6 epilogue + the next term's K5 gather half) and by
//    the camera side of the linearization (k_lin_cam).  Per-camera sums are
//    register accumulations + a fixed-order block reduction: no atomics,
//    bit-reproducible.
//  * landmark-major "tasks": one warp owns a run of whole landmarks whose
//    observations fit in 32 lanes (or one long landmark, looped in 32-obs
//    slabs).  Used by the landmark side of the linearization (k_lin_lm), the
//    per-landmark reduction + V^+ of each term (k_lm_reduce, also K7
//    back-substitution), the cost (k_cost) and the closed-form landmark
//    re-solve (k_resolve).  Segment sums use a deterministic shuffle tree.
#pragma once
#include "pv_device.cuh"

namespace pv {

constexpr int CREC = 24;  // camera record: P (12) | v (12)
constexpr int LREC = 4;   // landmark record: x (4)
constexpr int LSYS = 8;   // V+ (6) | degenerate (1) | pad
constexpr int LINP = 90;  // camera linearization: U upper (78) | b_p (12)
constexpr int FT = 256;   // threads of a camera CTA
// landmark warp slots (build_ktasks, povar.cu): a landmark with at most KSHORT observations
// shares a slot with up to 31 others of the same track length, one lane each walking its
// observations serially; a longer one fills a slot alone and is walked by the whole warp.
// 64: vlarge term 1.071 -> 1.056 ms, LM iteration 19.90 -> 19.66 ms against 32 (48: 1.068 /
// 19.78; 96: 1.117 / 20.59 -- a 96-step serial slot is too long for a ~20 us launch)
#ifndef PV_KSHORT
#define PV_KSHORT 64
#endif
constexpr int KSHORT = PV_KSHORT;

// runtime tuning of the term kernels (pv_set_option): on-chip staging capacity
// and L2 eviction priorities (0 normal, 1 evict_first, 2 evict_last)
struct Tune {
  int stage_cap;   // reserved (ABI stability of pv_set_option)
  int pol_stream;  // camera-sorted streams (m, x, ids)
  int pol_t;       // landmark vectors t (gathered)
  int pol_s;       // per-observation partials s (scattered / streamed)
  int discard_s;   // drop consumed s lines from L2 (no write-back)
  int xm;            // 1: stage-1 pipelined passes stream the compact (x0 x1 x2 m0 | m1) layout
  int cam_pipe;      // single-block camera passes: persistent TMA-pipelined k_cam_pipe
  int resolve_slots; // landmark re-solve: one lane per landmark over the k-bucketed slots
  int split_last;    // a term's last block: pipelined W t, then epilogue + next W^T v
  int rhs_reuse;     // reuse the reduced RHS across solves of one POSE_ONLY linearization
  int cost_cs;       // cost over the camera-sorted segments (k_cost_cs) instead of k_cost
  int graph;         // power-series term loop as a CUDA graph WHILE node (no host round trips)
  int series;        // the whole power series as one persistent cooperative kernel (pv_series.cuh)
};

enum { F_INVALID_Z = 0, F_ZERO_NORM = 1, F_SINGULAR_U = 2, F_N_DEGEN = 3, F_N_RANKDEF = 4,
       F_N_FALLBACK = 5, F_SINGULAR_M = 6, F_SINGULAR_M2 = 7, F_XM_BAD = 8, F_COUNT = 9 };

struct Graph {
  int n_p, n_l, n_o;
  int n_tasks;
  const int* ls_cam;     // [n_o] camera of each landmark-sorted observation
  const double* ls_m;    // [n_o*2]
  const int* lm_off;     // [n_l+1]
  const int4* task;      // [n_tasks] {o0, n, l0, segment-head mask}
  const int* cs_lm;      // [n_o] local landmark of each camera-sorted observation
  const int* cs_pos;     // [n_o] s position (partials layout, build_ktasks) of each
                         // camera-sorted observation
  const int* cs_kpos;    // [n_o] warp-slot position (build_ktasks) of the landmark of each
                         // camera-sorted observation: the index of its V+ and t
  int n_kent;            // warp-slot entries (V+ / t positions, build_ktasks)
  long long n_s;         // entries of the partials buffer s (build_ktasks)
  int n_blk;             // landmark blocks of the L2-blocked term
  const int* seg;        // [n_blk*n_p+1] start of segment (block b, camera c) at b*n_p+c in the
                         // block-major camera-sorted order (block, camera, landmark)
  const double* cs_m;    // [n_o*2]
  // measurements and cameras of the landmark-sorted observations once more, at their s
  // position (the warp-slot interleaved layout of build_ktasks): the lane-per-landmark walks
  // of the re-solve and the landmark linearization read 32 lanes' observation i with one
  // coalesced request instead of 32 scattered ones
  const double* ks_m;    // [n_s*2]
  const int* ks_cam;     // [n_s]
};

// stop / report state of the inner solve, shared by the power series and PCG
// (PCG: order = iterations, trunc = relative residual, pad = 1 on breakdown)
struct PowerCtl {
  int stopped;
  int order;
  int term;
  int pad;
  double trunc;
  double xnorm;
  double tnorm;
  double alpha, beta, rz, rhs_norm;  // PCG recurrences
};

struct Coef {
  double s1, s2;  // sqrt(1-eta), sqrt(eta)
  double s;       // 1 - eta
};

// ---------------------------------------------------------------------------
// landmark task decoding

struct Task {
  int l0, o0, n;
  bool long_task;
  unsigned heads;
};

__device__ __forceinline__ Task load_task(const Graph& g, int w, int lane) {
  const int4 d = __ldg(g.task + w);
  Task t;
  t.o0 = d.x;
  t.n = d.y;
  t.l0 = d.z;
  t.heads = (unsigned)d.w;
  t.long_task = t.n > 32;
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
// One power-series term, L2-blocked.
//
// Landmarks are split into B contiguous blocks (block boundaries on warp-task
// boundaries) sized so that one block's per-observation partials s (32 B/obs)
// and landmark vectors t (32 B/landmark) fit in L2.  For each block b:
//
//   k_lm_reduce(b): t_j = V_j^+ sum_i s_ij      landmark-major, reads s (L2),
//                                               writes t (L2, evict_last)
//   k_cam(b):       y_i += sum_{j in b} W_ij t_j     camera-major (gathers t: L2)
//                   then s_ij = W_ij^T v_i for j in block b+1 (scatter: L2)
//
// and after the last block the camera CTA finishes y_i, applies U_i^-1
// (epilogue: x_i += t_i, norms, stop test) and starts the next term's block 0.
// Both transpositions of S'.v therefore stay on chip; DRAM only streams the
// camera-sorted observation data (x, m, ids) twice per term.

// the consumed partials of a landmark block are scratch: drop their L2 lines instead of
// writing them back (lines entirely inside [o_lo, o_hi) only); grid-stride, all threads
__device__ __forceinline__ void discard_s_lines(double* sbuf, int o_lo, int o_hi) {
  if (o_hi <= o_lo) return;
  const size_t l0 = (32ull * o_lo + 127) / 128, l1 = (32ull * o_hi) / 128;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t ln = l0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; ln < l1; ln += stride)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<char*>(sbuf) + ln * 128)
                 : "memory");
}

// EP_RHS_CACHED: the reduced RHS is already in crhs (same linearization, POSE_ONLY V+):
// only t_0 = U^-1 rhs and the series start are recomputed
enum { EP_NONE = 0, EP_RHS = 1, EP_TERM = 2, EP_RHS_CACHED = 3 };

__device__ __forceinline__ void block_sum12(double (&acc)[12], double* red /*[FT/32*12]*/,
                                            double* out /*[12]*/) {
  warp_reduce_all(acc);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 12; ++i) red[w * 12 + i] = acc[i];
  }
  __syncthreads();
  if (threadIdx.x < 12) {
    double s = 0.0;
    for (int q = 0; q < FT / 32; ++q) s += red[q * 12 + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}


// ---- per-warp double-buffered staging of a contiguous observation segment ----
constexpr int CH = 64;                         // observations per staged chunk
constexpr int CH_BUF = CH * 32 + CH * 16 + (CH + 8) * 4;  // x, m, ids (one buffer)
constexpr int CAM_WARP_SMEM = 2 * CH_BUF;      // two buffers per warp
constexpr int CAM_SMEM = 8 * CAM_WARP_SMEM;    // 8 warps per CTA

__device__ __forceinline__ void cp_async16w(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16wp(void* smem, const void* gmem, uint64_t pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sa),
               "l"(gmem), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// stage observations [o, o + CH) of the camera-sorted streams (x, m and one int array)
__device__ __forceinline__ void stage_chunk(unsigned char* buf, int lane, int o,
                                            const double* __restrict__ cs_x,
                                            const double* __restrict__ cs_m,
                                            const int* __restrict__ ids) {
  const char* gx = reinterpret_cast<const char*>(cs_x + 4 * (size_t)o);
#pragma unroll
  for (int q = 0; q < (CH * 32) / (16 * 32); ++q)
    cp_async16w(buf + 16 * (lane + 32 * q), gx + 16 * (lane + 32 * q));
  const char* gm = reinterpret_cast<const char*>(cs_m + 2 * (size_t)o);
#pragma unroll
  for (int q = 0; q < (CH * 16) / (16 * 32); ++q)
    cp_async16w(buf + CH * 32 + 16 * (lane + 32 * q), gm + 16 * (lane + 32 * q));
  const int a0 = o & ~3;
  if (lane < (CH + 8) / 4)
    cp_async16w(buf + CH * 48 + 16 * lane, ids + a0 + 4 * lane);
}

struct CamArgs {
  int c_lo, c_hi;   // landmark-block range of the W t half (HC)
  int first_c;      // 1: overwrite the camera accumulator y, 0: add
  int a_lo, a_hi;   // landmark-block range of the W^T v half (HA)
  int term;         // term index for the stop test (EP_TERM)
  int check_stop;   // return immediately once the series has stopped
  int project_y;    // write the (stage-2 projected) y to cyr instead (schur apply)
  int wpc;          // warps per camera (1, 2, 4, 8)
  int disc_lo, disc_hi;  // landmark-sorted observations whose consumed partials s are dropped
  double thr;
  // device-driven term loop (povar.cu term_graph): term < 0 takes the term index from the
  // control block (previous term + 1); cond != 0 is the WHILE handle of the CUDA graph the
  // epilogue sets to continue (not stopped and term < max_order) or stop
  unsigned long long cond;
  int max_order;
};

#ifndef PV_CAM_MINB
#define PV_CAM_MINB 1
#endif
#ifndef PV_EP_MIRROR_ALWAYS
#define PV_EP_MIRROR_ALWAYS 0
#endif
template <int STAGE, bool HC, int EP, bool HA>
__global__ void __launch_bounds__(256, PV_CAM_MINB) k_cam(
    Graph g, double* __restrict__ crec, const double* __restrict__ cs_x,
    const double* __restrict__ tarr, double* __restrict__ sbuf, double* __restrict__ cy,
    double* __restrict__ cyr, const double* __restrict__ cbp, const double* __restrict__ cUi,
    double* __restrict__ cx, double* __restrict__ crhs, const double* __restrict__ ch,
    double* __restrict__ nrm, PowerCtl* __restrict__ ctl, volatile PowerCtl* host_ctl,
    unsigned* __restrict__ ticket, Coef k, Tune tune, CamArgs ca) {
  // ca.wpc warps per camera (1, 2, 4 or 8; 8 / wpc cameras per CTA).  The chunks of a
  // (camera, block) segment are striped over the camera's warps; per-camera sums are
  // combined in fixed order through shared memory.
  constexpr bool RHS = EP == EP_RHS || EP == EP_RHS_CACHED;
  constexpr bool CACHED = EP == EP_RHS_CACHED;
  constexpr int D = STAGE == 1 ? 12 : 11;
  __shared__ bool last;
  __shared__ double gred[8][12];
  __shared__ double gv[8][12];
  extern __shared__ __align__(32) unsigned char cam_dsm[];
  if (ca.check_stop && ctl->stopped) return;  // grid-uniform
  discard_s_lines(sbuf, ca.disc_lo, ca.disc_hi);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpc = ca.wpc;
  const int grp = warp / wpc, gr = warp % wpc;
  const int cam = blockIdx.x * (8 / wpc) + grp;
  constexpr int SLOT = CH_BUF;
  unsigned char* wsm = cam_dsm + (size_t)warp * 2 * SLOT;
  const bool valid = cam < g.n_p;
  const bool leader = valid && gr == 0;
  const int np = g.n_p;
  const uint64_t pf = pol_sel(tune.pol_stream), pt = pol_sel(tune.pol_t),
                 ps = pol_sel(tune.pol_s);
  double4 P0 = make_double4(0, 0, 0, 0), P1 = P0, P2v = P0;
  if (valid) {
    const double* cp = crec + (size_t)cam * CREC;
    P0 = ldg4(cp);
    P1 = ldg4(cp + 4);
    P2v = ldg4(cp + 8);
  }
  double yr = 0.0;  // leader lane r < 12: component r of this camera's y
  if (HC) {  // y_i (+)= sum_{j in blocks [c_lo, c_hi)} W_ij t_j
    double acc[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) acc[i] = 0.0;
    for (int b = ca.c_lo; valid && b < ca.c_hi; ++b) {
      const int o_lo = __ldg(g.seg + (size_t)b * np + cam);
      const int o_hi = __ldg(g.seg + (size_t)b * np + cam + 1);
      const int nch_all = (o_hi - o_lo + CH - 1) / CH;
      const int nch = nch_all > gr ? (nch_all - gr + wpc - 1) / wpc : 0;  // this warp's chunks
      if (nch > 0) stage_chunk(wsm, lane, o_lo + gr * CH, cs_x, g.cs_m, g.cs_kpos);
      cp_commit();
      for (int c = 0; c < nch; ++c) {
        unsigned char* buf = wsm + (c & 1) * SLOT;
        if (c + 1 < nch)
          stage_chunk(wsm + ((c + 1) & 1) * SLOT, lane, o_lo + (gr + (c + 1) * wpc) * CH, cs_x,
                      g.cs_m, g.cs_kpos);
        cp_commit();
        cp_wait<1>();
        __syncwarp();
        const int o0 = o_lo + (gr + c * wpc) * CH;
        const double4* sx = reinterpret_cast<const double4*>(buf);
        const double2* sm = reinterpret_cast<const double2*>(buf + CH * 32);
        const int* si = reinterpret_cast<const int*>(buf + CH * 48) + (o0 & 3);
        double4 T[CH / 32];
#pragma unroll
        for (int r = 0; r < CH / 32; ++r) {
          const int q = lane + 32 * r;
          if (o0 + q < o_hi) {
            PV_CHECK(si[q] >= 0 && si[q] < g.n_kent);
            T[r] = ldg4p(tarr + 4 * (size_t)si[q], pt);
          }
        }
#pragma unroll
        for (int r = 0; r < CH / 32; ++r) {
          const int q = lane + 32 * r;
          if (o0 + q < o_hi) {
            const double4 X = sx[q];
            const double2 m = sm[q];
            const double4 Tq = T[r];
            const Proj pj = STAGE == 1 ? proj_s1(m.x, m.y, k.s) : proj_s2(P0, P1, P2v, X);
            double sg[3];
            proj_map<STAGE>(pj, dot4(P0, Tq), dot4(P1, Tq), dot4(P2v, Tq), sg[0], sg[1],
                            sg[2]);
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
              acc[4 * cc + 0] = fma(sg[cc], X.x, acc[4 * cc + 0]);
              acc[4 * cc + 1] = fma(sg[cc], X.y, acc[4 * cc + 1]);
              acc[4 * cc + 2] = fma(sg[cc], X.z, acc[4 * cc + 2]);
              acc[4 * cc + 3] = fma(sg[cc], X.w, acc[4 * cc + 3]);
            }
          }
        }
        __syncwarp();
      }
      cp_wait<0>();
    }
    double mine = warp_reduce12_lane(acc, lane);
    if (wpc > 1) {  // fixed-order combination over the camera's warps
      if (lane < 12) gred[warp][lane] = mine;
      __syncthreads();
      if (gr == 0 && lane < 12) {
        double sacc = 0.0;
        for (int q = 0; q < wpc; ++q) sacc += gred[warp + q][lane];
        mine = sacc;
      }
    }
    yr = mine;
    if (leader && lane < 12) {  // fixed-order accumulation over blocks (deterministic)
      if (!ca.first_c) yr += cy[(size_t)cam * 12 + lane];
      cy[(size_t)cam * 12 + lane] = yr;
    }
    if (ca.project_y && leader) {  // schur apply: tangent projection (stage 2) -> cyr
      double u = lane < 12 ? yr : 0.0;
      if (STAGE == 2) {
        const double h = lane < 12 ? ch[(size_t)cam * 12 + lane] : 0.0;
        const double hu = warp_sum(h * u);
        const double pr = fma(-2.0 * h, hu, u);
        u = __shfl_sync(PV_FULL, pr, (lane + 1) & 31);
        if (lane >= 11) u = 0.0;
      }
      if (lane < 12) cyr[(size_t)cam * 12 + lane] = u;
    }
  }

  double4 v0 = make_double4(0, 0, 0, 0), v1 = v0, v2 = v0;
  if (EP != EP_NONE) {
    if (gr == 0) {  // leader warp of each camera (whole warp participates in shuffles)
      const bool row = lane < 12;
      double u = 0.0;
      if (row && valid) u = HC ? yr : cy[(size_t)cam * 12 + lane];
      double h = 0.0;
      if (STAGE == 2) {  // project y (12) -> tangent (11)
        h = (row && valid) ? ch[(size_t)cam * 12 + lane] : 0.0;
        const double hu = warp_sum(h * u);
        const double pr = fma(-2.0 * h, hu, u);
        u = __shfl_sync(PV_FULL, pr, (lane + 1) & 31);
        if (lane >= 11) u = 0.0;
      }
      double vin = u;
      if (CACHED) {
        vin = (lane < D && valid) ? crhs[(size_t)cam * 12 + lane] : 0.0;
      } else if (RHS) {
        const double b = (lane < D && valid) ? cbp[(size_t)cam * 12 + lane] : 0.0;
        vin = lane < D ? -(b - u) : 0.0;
        if (row && valid) crhs[(size_t)cam * 12 + lane] = vin;
      }
      double t = 0.0;
      const double* Ui = cUi + (size_t)(valid ? cam : 0) * 144 + (lane < D ? lane : 0) * 12;
#pragma unroll
      for (int kk = 0; kk < 12; ++kk) {
        const double vk = __shfl_sync(PV_FULL, vin, kk);
        if (valid && lane < D && kk < D) t = fma(Ui[kk], vk, t);
      }
      double xr = 0.0;
      if (valid && lane < D) {
        xr = RHS ? t : cx[(size_t)cam * 12 + lane] + t;
        cx[(size_t)cam * 12 + lane] = xr;
      }
      double v = t;
      if (STAGE == 2) {  // v = B t (11 -> 12)
        const double tprev = __shfl_sync(PV_FULL, t, (lane + 31) & 31);
        const double e = (lane >= 1 && lane < 12) ? tprev : 0.0;
        const double hd = warp_sum(h * e);
        v = fma(-2.0 * h, hd, e);
      }
      if (row && valid) crec[(size_t)cam * CREC + 12 + lane] = v;  // for the later blocks
      if (row) gv[grp][lane] = v;
      const double tn = warp_sum(lane < D ? t * t : 0.0);
      const double xn = warp_sum(lane < D ? xr * xr : 0.0);
      if (lane == 0 && valid) {
        nrm[2 * (size_t)cam] = tn;
        nrm[2 * (size_t)cam + 1] = xn;
      }
    }
    if (HA) {
      __syncthreads();
      v0 = make_double4(gv[grp][0], gv[grp][1], gv[grp][2], gv[grp][3]);
      v1 = make_double4(gv[grp][4], gv[grp][5], gv[grp][6], gv[grp][7]);
      v2 = make_double4(gv[grp][8], gv[grp][9], gv[grp][10], gv[grp][11]);
    }
  } else if (HA && valid) {
    const double* cp = crec + (size_t)cam * CREC + 12;
    v0 = ldg4(cp);
    v1 = ldg4(cp + 4);
    v2 = ldg4(cp + 8);
  }

  if (HA && valid) {  // s_ij = W_ij^T v_i for j in blocks [a_lo, a_hi), scattered
    for (int b = ca.a_lo; b < ca.a_hi; ++b) {
      const int o_lo = __ldg(g.seg + (size_t)b * np + cam);
      const int o_hi = __ldg(g.seg + (size_t)b * np + cam + 1);
      const int nch_all = (o_hi - o_lo + CH - 1) / CH;
      const int nch = nch_all > gr ? (nch_all - gr + wpc - 1) / wpc : 0;
      if (nch > 0) stage_chunk(wsm, lane, o_lo + gr * CH, cs_x, g.cs_m, g.cs_pos);
      cp_commit();
      for (int c = 0; c < nch; ++c) {
        unsigned char* buf = wsm + (c & 1) * SLOT;
        if (c + 1 < nch)
          stage_chunk(wsm + ((c + 1) & 1) * SLOT, lane, o_lo + (gr + (c + 1) * wpc) * CH, cs_x,
                      g.cs_m, g.cs_pos);
        cp_commit();
        cp_wait<1>();
        __syncwarp();
        const int o0 = o_lo + (gr + c * wpc) * CH;
        const double4* sx = reinterpret_cast<const double4*>(buf);
        const double2* sm = reinterpret_cast<const double2*>(buf + CH * 32);
        const int* si = reinterpret_cast<const int*>(buf + CH * 48) + (o0 & 3);
#pragma unroll
        for (int r = 0; r < CH / 32; ++r) {
          const int q = lane + 32 * r;
          if (o0 + q < o_hi) {
            const double4 X = sx[q];
            const double2 m = sm[q];
            const int pos = si[q];
            const Proj pj = STAGE == 1 ? proj_s1(m.x, m.y, k.s) : proj_s2(P0, P1, P2v, X);
            double f0, f1, f2;
            proj_map<STAGE>(pj, dot4(X, v0), dot4(X, v1), dot4(X, v2), f0, f1, f2);
            double4 sv;
            sv.x = fma(f0, P0.x, fma(f1, P1.x, f2 * P2v.x));
            sv.y = fma(f0, P0.y, fma(f1, P1.y, f2 * P2v.y));
            sv.z = fma(f0, P0.z, fma(f1, P1.z, f2 * P2v.z));
            sv.w = STAGE == 2 ? fma(f0, P0.w, fma(f1, P1.w, f2 * P2v.w)) : 0.0;
            PV_CHECK(pos >= 0 && pos < g.n_s);
            st4p(sbuf + 4 * (size_t)pos, sv, ps);
          }
        }
        __syncwarp();
      }
      cp_wait<0>();
    }
  }

  if (EP == EP_NONE) return;
  // ---- grid-wide fixed-order norm reduction + stop test in the last CTA
  const int tid = threadIdx.x;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned tk = atomicAdd(ticket, 1u);
    last = tk == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double ra[2] = {0.0, 0.0};
  strided_sum_ordered<2>(nrm, g.n_p, ra);
  warp_reduce_all(ra);
  __shared__ double rr[2][8];
  if ((tid & 31) == 0) {
    rr[0][tid >> 5] = ra[0];
    rr[1][tid >> 5] = ra[1];
  }
  __syncthreads();
  if (tid == 0) {
    double TN2 = 0.0, XN2 = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      TN2 += rr[0][q];
      XN2 += rr[1][q];
    }
    const double TN = sqrt(TN2), XN = sqrt(XN2);
    PowerCtl c = *ctl;
    if (RHS) {  // solvers.py:134-139
      c.stopped = 0;
      c.order = 0;
      c.term = 0;
      c.trunc = XN > 0.0 ? 1.0 : 0.0;
    } else {  // solvers.py:140-149
      const int term = ca.term >= 0 ? ca.term : c.term + 1;
      const double ratio = XN > 0.0 ? TN / XN : 0.0;
      c.trunc = ratio;
      c.term = term;
      if (ratio <= ca.thr) {
        c.order = term - 1;
        c.stopped = 1;
      } else {
        c.order = term;
      }
      if (ca.cond)
        cudaGraphSetConditional((cudaGraphConditionalHandle)ca.cond,
                                (!c.stopped && term < ca.max_order) ? 1u : 0u);
    }
    c.xnorm = XN;
    c.tnorm = TN;
    *ctl = c;
    // the host's look-ahead loop reads `stopped`, then `term`: publish term first, so a rank
    // never sees the stop without the term that took it (povar.cu op_power).  Inside the term
    // graph (ca.cond) the host reads the control block once, after the series: no mirror
    if (PV_EP_MIRROR_ALWAYS || !ca.cond) {
      host_ctl->order = c.order;
      host_ctl->term = c.term;
      host_ctl->trunc = c.trunc;
      host_ctl->xnorm = c.xnorm;
      host_ctl->tnorm = c.tnorm;
      __threadfence_system();
      host_ctl->stopped = c.stopped;
      __threadfence_system();
    }
    *ticket = 0u;
  }
}

// y (raw 12 per camera) -> tangent y (11) in stage 2 / copy in stage 1 (schur apply)
template <int STAGE>
__global__ void k_project_y(int n_p, const double* __restrict__ cy, const double* __restrict__ ch,
                            double* __restrict__ cyr) {
  const int lane = threadIdx.x & 31;
  const int cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (cam >= n_p) return;
  double u = lane < 12 ? cy[(size_t)cam * 12 + lane] : 0.0;
  if (STAGE == 2) {
    const double h = lane < 12 ? ch[(size_t)cam * 12 + lane] : 0.0;
    const double hu = warp_sum(h * u);
    const double pr = fma(-2.0 * h, hu, u);
    u = __shfl_sync(PV_FULL, pr, (lane + 1) & 31);
    if (lane >= 11) u = 0.0;
  }
  if (lane < 12) cyr[(size_t)cam * 12 + lane] = u;
}

// ---------------------------------------------------------------------------
// landmark half of a term (and K7): t_j = V_j^+ sum_i s_ij (TERM) or V_j^+ b_j
// (RHS) written per landmark, or the back-substitution
// dl_j = -V_j^+ (b_l + sum_i s_ij) with the trial landmark (BACKSUB).

enum { LR_TERM = 0, LR_BACKSUB = 1, LR_RHS = 2 };

struct LmPre {  // per-landmark inputs of the landmark epilogue, prefetched before the reduce
  double4 va, vb, bl, x;
};

// H: 128-bit accesses (k_series, see ldg4_h)
template <int STAGE, int MODE, bool H = false>
__device__ __forceinline__ LmPre lm_prefetch(int l, int kp, const double* __restrict__ lrec,
                                             const double* __restrict__ lsys,
                                             const double* __restrict__ lbl) {
  LmPre p;
  p.va = H ? ldg4_h(lsys + (size_t)kp * LSYS) : ldg4(lsys + (size_t)kp * LSYS);
  p.vb = H ? ldg4_h(lsys + (size_t)kp * LSYS + 4) : ldg4(lsys + (size_t)kp * LSYS + 4);
  p.x = (STAGE == 2 || MODE == LR_BACKSUB)
            ? (H ? ldg4_h(lrec + (size_t)l * LREC) : ldg4(lrec + (size_t)l * LREC))
            : make_double4(0.0, 0.0, 0.0, 1.0);
  p.bl = MODE != LR_TERM ? ldg4(lbl + (size_t)l * 4) : make_double4(0.0, 0.0, 0.0, 0.0);
  return p;
}

template <int STAGE, int MODE, bool H = false>
__device__ __forceinline__ void lm_finish(int l, int kp, const double (&acc)[4], const LmPre& p,
                                          double* __restrict__ tarr, double* __restrict__ ldl,
                                          double* __restrict__ tlm, int* __restrict__ flags,
                                          uint64_t pt) {
  double s3[3], h[4];
  const double4 x = p.x;
  double xv[4] = {x.x, x.y, x.z, x.w};
  if (STAGE == 2) householder_h<4>(xv, h);
  if (MODE == LR_RHS) {
    s3[0] = p.bl.x;
    s3[1] = p.bl.y;
    s3[2] = p.bl.z;
  } else if (STAGE == 1) {
    s3[0] = acc[0];
    s3[1] = acc[1];
    s3[2] = acc[2];
  } else {
    basis_apply_t<4>(h, acc, s3);
  }
  const double vp[6] = {p.va.x, p.va.y, p.va.z, p.va.w, p.vb.x, p.vb.y};
  if (MODE != LR_BACKSUB) {
    double t[3];
    sym3_apply(vp, s3, t);
    double4 tv;
    if (STAGE == 1) {
      tv = make_double4(t[0], t[1], t[2], 0.0);
    } else {
      double t4[4];
      basis_apply<4>(h, t, t4);
      tv = make_double4(t4[0], t4[1], t4[2], t4[3]);
    }
    if (H)
      st4p_h(tarr + (size_t)kp * 4, tv, pt);
    else
      st4p(tarr + (size_t)kp * 4, tv, pt);
    return;
  }
  double q[3] = {s3[0] + p.bl.x, s3[1] + p.bl.y, s3[2] + p.bl.z};
  double dl[3];
  sym3_apply(vp, q, dl);
  const bool degen = p.vb.z != 0.0;
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

// Landmark half of a term.  Work unit (built by build_ktasks, povar.cu): up to 32
// landmarks of one block with the same track length k <= KSHORT, one lane per landmark,
// each lane summing its k partials s_ij serially (k is warp-uniform: no divergence,
// no shuffles, ~5 instructions per observation); a landmark with k > KSHORT is a unit of
// its own, reduced by the whole warp (coalesced, fixed-order tree).  Deterministic.

template <int STAGE, int MODE>
__device__ __forceinline__ void lr_long(const Task& t, int kp, int lane,
                                        const double* __restrict__ sbuf,
                                        const double* __restrict__ lrec,
                                        double* __restrict__ tarr,
                                        const double* __restrict__ lsys,
                                        const double* __restrict__ lbl, double* __restrict__ ldl,
                                        double* __restrict__ tlm, int* flags, uint64_t pf,
                                        uint64_t pt) {
  constexpr int NV = STAGE == 1 ? 3 : 4;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const LmPre pre = lane == 0 ? lm_prefetch<STAGE, MODE>(t.l0, kp, lrec, lsys, lbl) : LmPre{};
  if (MODE != LR_RHS) {
    double a2[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) a2[i] = 0.0;
#pragma unroll 4
    for (int o = t.o0 + lane; o < t.o0 + t.n; o += 32) {
      const double4 s = ldg4p(sbuf + 4 * (size_t)o, pf);
      a2[0] += s.x;
      a2[1] += s.y;
      a2[2] += s.z;
      if (NV == 4) a2[NV - 1] += s.w;
    }
    warp_reduce_all(a2);
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = a2[i];
  }
  if (lane == 0) lm_finish<STAGE, MODE>(t.l0, kp, acc, pre, tarr, ldl, tlm, flags, pt);
}

constexpr int LG = 1;  // lanes per landmark in a short warp slot (the s layout assumes 1)

// build-time tuning of the short-slot walk (loads in flight per lane, resident CTAs)
#ifndef PV_LR_UNROLL
#define PV_LR_UNROLL 4
#endif
#ifndef PV_LR_MINB
#define PV_LR_MINB 1
#endif
constexpr int kLrUnroll = PV_LR_UNROLL;

template <int STAGE, int MODE>
__global__ void __launch_bounds__(256, PV_LR_MINB) k_lm_reduce(const int4* __restrict__ klist,
                                                   const int4* __restrict__ kslot,
                                                   const double* __restrict__ sbuf,
                                                   const double* __restrict__ lrec,
                                                   double* __restrict__ tarr,
                                                   const double* __restrict__ lsys,
                                                   const double* __restrict__ lbl,
                                                   double* __restrict__ ldl,
                                                   double* __restrict__ tlm,
                                                   const PowerCtl* __restrict__ ctl, int* flags,
                                                   Tune tune, int k_lo, int k_hi,
                                                   int check_stop) {
  const int lane = threadIdx.x & 31;
  const int w = k_lo + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (w >= k_hi) return;
  if (check_stop && ctl->stopped) return;
  const uint64_t pf = pol_sel(tune.pol_s), pt = pol_sel(tune.pol_t);
  int4 e;
  if (STAGE == 1 && MODE == LR_TERM && kslot != nullptr) {
    // stage-1 terms need no landmark ids: the slot's {k, s position, landmarks} come from one
    // 16-byte record that every lane reads (4 MB for all slots: it stays in L2 from term to
    // term, while the 512-byte per-lane entries (128 MB) are a DRAM round trip per slot)
    const int4 ks = __ldg(kslot + w);
    e = make_int4(lane < ks.z ? 0 : -1, 0, ks.x, ks.x > KSHORT ? ks.y : ks.y + lane);
  } else {
    e = __ldg(klist + 32 * (size_t)w + lane);  // {landmark, first obs, k, s position}
  }
  const int k = e.z;  // warp-uniform
  if (k > KSHORT) {
    Task t;
    t.l0 = __shfl_sync(PV_FULL, e.x, 0);
    t.o0 = __shfl_sync(PV_FULL, e.w, 0);  // contiguous partials
    t.n = k;
    t.long_task = true;
    t.heads = 1u;
    lr_long<STAGE, MODE>(t, 32 * w, lane, sbuf, lrec, tarr, lsys, lbl, ldl, tlm, flags, pf, pt);
    return;
  }
  // LG lanes per landmark (the slot entry is repeated LG times): lane j of a group sums
  // the observations i = j, j + LG, ... (adjacent lanes read adjacent sectors), then a
  // fixed xor tree inside the group; the group's first lane finishes the landmark
  if (e.x < 0) return;  // whole groups are empty together
  const int j = lane & (LG - 1);
  LmPre pre;
  if (j == 0) pre = lm_prefetch<STAGE, MODE>(e.x, 32 * w + lane, lrec, lsys, lbl);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (MODE != LR_RHS) {
    const double* sp = sbuf + 4 * (size_t)e.w;  // interleaved: observation i at + 32 i
#pragma unroll kLrUnroll
    for (int i = j; i < k; i += LG) {
      const double4 v = ldg4p(sp + 128 * (size_t)i, pf);
      acc[0] += v.x;
      acc[1] += v.y;
      acc[2] += v.z;
      if (STAGE == 2) acc[3] += v.w;
    }
#pragma unroll
    for (int d = 1; d < LG; d <<= 1) {
      const unsigned gm = __activemask();
#pragma unroll
      for (int c = 0; c < (STAGE == 1 ? 3 : 4); ++c) acc[c] += __shfl_xor_sync(gm, acc[c], d);
    }
  }
  if (j == 0) lm_finish<STAGE, MODE>(e.x, 32 * w + lane, acc, pre, tarr, ldl, tlm, flags, pt);
}

// block-major camera-sorted copy of the measurements (once per re-blocking)
__global__ void k_gather_m(int n_o, const int* __restrict__ cs_pos, const double* __restrict__ ls_m,
                           double* __restrict__ cs_m) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n_o) return;
  reinterpret_cast<double2*>(cs_m)[o] = reinterpret_cast<const double2*>(ls_m)[__ldg(cs_pos + o)];
}

// camera-sorted copy of the landmark coordinates (once per linearization point).  Stage 1
// also writes the compact stream of the pipelined camera passes, xm = (x0, x1, x2, m0) with
// m1 in its own array (cs_m1): the landmark's w = 1 is not streamed (40 instead of 48 bytes
// of x and m per observation and pass).  A landmark with w != 1 sets F_XM_BAD and the term
// kernels keep the full stream.
template <int STAGE>
__global__ void k_build_csx(Graph g, const double* __restrict__ lrec, double* __restrict__ cs_x,
                            double* __restrict__ cs_xm, int* __restrict__ flags) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= g.n_o) return;
  PV_CHECK(__ldg(g.cs_lm + o) >= 0 && __ldg(g.cs_lm + o) < g.n_l);
  const double4 x = ldg4(lrec + (size_t)__ldg(g.cs_lm + o) * LREC);
  st4(cs_x + 4 * (size_t)o, x);
  if (STAGE == 1) {
    st4(cs_xm + 4 * (size_t)o, make_double4(x.x, x.y, x.z, __ldg(g.cs_m + 2 * (size_t)o)));
    if (x.w != 1.0) atomicOr(flags + F_XM_BAD, 1);
  }
}

// slot-interleaved copies of the landmark-sorted measurements and camera ids (once per
// re-blocking): entry spos[p] <- landmark-sorted observation p
__global__ void k_scatter_ks(int n_o, const int* __restrict__ spos, const double* __restrict__ ls_m,
                             const int* __restrict__ ls_cam, double* __restrict__ ks_m,
                             int* __restrict__ ks_cam) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_o) return;
  const int q = __ldg(spos + p);
  reinterpret_cast<double2*>(ks_m)[q] = reinterpret_cast<const double2*>(ls_m)[p];
  ks_cam[q] = __ldg(ls_cam + p);
}

// m1 of every block-major camera-sorted observation (once per re-blocking)
__global__ void k_gather_m1(int n_o, const double* __restrict__ cs_m, double* __restrict__ cs_m1) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n_o) return;
  cs_m1[o] = cs_m[2 * (size_t)o + 1];
}

// ---------------------------------------------------------------------------
// K1 + K2 (landmark side of the linearization): V = sum Jl^T Jl, b_l = sum Jl^T r

// V (6 unique) and b_l (3) of one observation, in the landmark's tangent space:
// stage 1 J_l rows are already 3-wide; stage 2 rows (2x4) are projected with the
// Householder basis of x first (riemannian.py:67-85 projects the blocks before
// normal_eq.py:156-198 assembles), so both stages reduce 9 values.
template <int STAGE>
__device__ __forceinline__ void lin_lm_obs(const double* __restrict__ crec, int cam, double m0,
                                           double m1, const double4& x, const double (&h)[4],
                                           const Coef& k, double (&acc)[9], int* flags) {
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
      double jt[3];
      basis_apply_t<4>(h, J[q], jt);  // J_l B (riemannian.py:80-82)
      acc[0] = fma(jt[0], jt[0], acc[0]);
      acc[1] = fma(jt[0], jt[1], acc[1]);
      acc[2] = fma(jt[0], jt[2], acc[2]);
      acc[3] = fma(jt[1], jt[1], acc[3]);
      acc[4] = fma(jt[1], jt[2], acc[4]);
      acc[5] = fma(jt[2], jt[2], acc[5]);
      acc[6] = fma(jt[0], rr[q], acc[6]);
      acc[7] = fma(jt[1], rr[q], acc[7]);
      acc[8] = fma(jt[2], rr[q], acc[8]);
    }
  }
}

__device__ __forceinline__ void lin_lm_finish(int l, const double (&acc)[9],
                                              double* __restrict__ lvr, double* __restrict__ lbl) {
  double* o = lvr + (size_t)l * 8;
  st4(o, make_double4(acc[0], acc[1], acc[2], acc[3]));
  st4(o + 4, make_double4(acc[4], acc[5], 0.0, 0.0));
  st4(lbl + (size_t)l * 4, make_double4(acc[6], acc[7], acc[8], 0.0));
}

// Same, over the k-bucketed warp slots of the landmark reduce (build_ktasks): one lane
// per landmark walks its k <= KSHORT observations serially (no shuffle trees; the landmark's
// Householder basis is built once per lane); a long landmark's slot is reduced by the
// whole warp.  The per-landmark sums run in a different (fixed) order than k_lin_lm's.
template <int STAGE>
__global__ void __launch_bounds__(256) k_lin_lm_slots(Graph g, const int4* __restrict__ klist,
                                                      int n_slots,
                                                      const double* __restrict__ crec,
                                                      const double* __restrict__ lrec,
                                                      double* __restrict__ lvr,
                                                      double* __restrict__ lbl, int* flags,
                                                      Coef k) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n_slots) return;
  const int4 e = __ldg(klist + 32 * (size_t)w + lane);  // {landmark, first obs, k, -}
  const int kk = e.z;                                     // warp-uniform
  double acc[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) acc[i] = 0.0;
  double h[4] = {0.0, 0.0, 0.0, 0.0};
  if (kk > KSHORT) {
    const int l = __shfl_sync(PV_FULL, e.x, 0), o0 = __shfl_sync(PV_FULL, e.y, 0);
    const double4 x = ldg4(lrec + (size_t)l * LREC);
    if (STAGE == 2) {
      const double xv[4] = {x.x, x.y, x.z, x.w};
      householder_h<4>(xv, h);
    }
    for (int o = o0 + lane; o < o0 + kk; o += 32) {
      const double2 m = ldg2(g.ls_m + 2 * (size_t)o);
      lin_lm_obs<STAGE>(crec, __ldg(g.ls_cam + o), m.x, m.y, x, h, k, acc, flags);
    }
    warp_reduce_all(acc);
    if (lane == 0) lin_lm_finish(l, acc, lvr, lbl);
    return;
  }
  if (e.x < 0) return;
  const double4 x = ldg4(lrec + (size_t)e.x * LREC);
  if (STAGE == 2) {
    const double xv[4] = {x.x, x.y, x.z, x.w};
    householder_h<4>(xv, h);
  }
  for (int i = 0; i < kk; ++i) {  // observation i of this lane's landmark at s position e.w + 32 i
    const int pos = e.w + 32 * i;
    const double2 m = ldg2(g.ks_m + 2 * (size_t)pos);
    lin_lm_obs<STAGE>(crec, __ldg(g.ks_cam + pos), m.x, m.y, x, h, k, acc, flags);
  }
  lin_lm_finish(e.x, acc, lvr, lbl);
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
  double acc[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) acc[i] = 0.0;
  double h[4] = {0.0, 0.0, 0.0, 0.0};
  if (t.long_task) {
    double4 x = ldg4(lrec + (size_t)t.l0 * LREC);
    if (STAGE == 2) {
      const double xv[4] = {x.x, x.y, x.z, x.w};
      householder_h<4>(xv, h);
    }
    for (int o = t.o0 + lane; o < t.o0 + t.n; o += 32) {
      double2 m = ldg2(g.ls_m + 2 * (size_t)o);
      lin_lm_obs<STAGE>(crec, __ldg(g.ls_cam + o), m.x, m.y, x, h, k, acc, flags);
    }
    warp_reduce_all(acc);
    if (lane == 0) lin_lm_finish(t.l0, acc, lvr, lbl);
  } else {
    int l, seg_end;
    lane_segment(t, lane, l, seg_end);
    double4 x = ldg4(lrec + (size_t)l * LREC);
    if (STAGE == 2) {
      const double xv[4] = {x.x, x.y, x.z, x.w};
      householder_h<4>(xv, h);
    }
    if (lane < t.n) {
      int o = t.o0 + lane;
      double2 m = ldg2(g.ls_m + 2 * (size_t)o);
      lin_lm_obs<STAGE>(crec, __ldg(g.ls_cam + o), m.x, m.y, x, h, k, acc, flags);
    }
    const bool head = lane < t.n && ((t.heads >> lane) & 1u);
    seg_reduce_n(acc, lane, seg_end,
                 (int)__reduce_max_sync(PV_FULL, head ? (unsigned)(seg_end - lane) : 1u));
    if (head) lin_lm_finish(l, acc, lvr, lbl);
  }
}

// ---------------------------------------------------------------------------
// K3 camera side of the linearization, camera-major (one CTA per camera).
// U = sum_obs A(w) (x) x x^T with A = [[c00 w0, 0, c02 w1], [0, c00 w0, c12 w2],
// [c02 w1, c12 w2, c22 w3]] and b_p = sum_obs h (x) x:
//   stage 1: w = (1, m0, m1, |m|^2),  (c00, c02, c12, c22) = (s1^2+s2^2, -s1^2, -s1^2, s1^2)
//            h = K^T r  (objective.py:95-110 rows)
//   stage 2: w = iz^2 (1, pi0, pi1, |pi|^2), (c00, c02, c12, c22) = (1, -1, -1, 1)
//            h = dpi^T r (objective.py:128-146)
// Output: 78 upper entries of U (row-major i <= j) + 12 of b_p per camera.

constexpr int LC_BUF = 3;                   // staging buffers of k_lin_cam
constexpr int LC_BYTES = FT * 48;           // x (32 B) + m (16 B) per observation
constexpr int LIN_SMEM = LC_BUF * LC_BYTES;

template <int STAGE>
__global__ void __launch_bounds__(FT, 2) k_lin_cam(Graph g, const double* __restrict__ crec,
                                               const double* __restrict__ cs_x,
                                               double* __restrict__ cUraw, Coef k) {
  // two groups of 128 threads: group 0 accumulates the moments of w0, w1 (20 values),
  // group 1 those of w2, w3 (20) and b_p (12) -> half the registers of one accumulator set
  constexpr int NA = 52;  // 4 x 10 weighted second moments + 12 b_p
  constexpr int GT = FT / 2;
  constexpr int MAXB = 64;
  __shared__ double red[(FT / 32) * 32];
  __shared__ double tot[NA];
  __shared__ int s_lo[MAXB], s_hi[MAXB];
  const int cam = blockIdx.x, tid = threadIdx.x;
  const int grp = tid / GT, gt = tid % GT;
  const int nb = g.n_blk;
  for (int b = tid; b < nb; b += FT) {
    s_lo[b] = g.seg[(size_t)b * g.n_p + cam];
    s_hi[b] = g.seg[(size_t)b * g.n_p + cam + 1];
  }
  __syncthreads();
  const double* cp = crec + (size_t)cam * CREC;
  const double4 P0 = ldg4(cp), P1 = ldg4(cp + 4), P2 = ldg4(cp + 8);
  double acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.0;
  // The camera's observations (one segment per landmark block) are cut into chunks of
  // <= FT observations, staged (x, m) into shared memory by cp.async two chunks ahead
  // (LC_BUF buffers); each group's thread gt takes observations gt and gt + GT of a chunk.
  extern __shared__ __align__(32) unsigned char lin_dsm[];
  int wb = 0, wo = nb > 0 ? s_lo[0] : 0;  // walker: next chunk = (block wb, first obs wo)
  auto next_chunk = [&](int& o, int& n) {  // uniform over the CTA
    while (wb < nb && wo >= s_hi[wb]) {
      ++wb;
      if (wb < nb) wo = s_lo[wb];
    }
    if (wb >= nb) {
      o = 0;
      n = 0;
      return;
    }
    o = wo;
    n = min(FT, s_hi[wb] - wo);
    wo += n;
  };
  static_assert(LC_BUF == 3, "chunk counts rotate through three registers");
  int n0 = 0, n1 = 0, n2 = 0;  // observation counts of chunks c, c + 1, c + 2
  auto stage = [&](int slot) {
    int o, n;
    next_chunk(o, n);
    n2 = n;
    unsigned char* buf = lin_dsm + (size_t)slot * LC_BYTES;
    if (tid < n) {
      const double* gx = cs_x + 4 * (size_t)(o + tid);
      cp_async16w(buf + 32 * tid, gx);
      cp_async16w(buf + 32 * tid + 16, gx + 2);
      cp_async16w(buf + FT * 32 + 16 * tid, g.cs_m + 2 * (size_t)(o + tid));
    }
    cp_commit();
  };
  stage(0);
  n0 = n2;
  stage(1);
  n1 = n2;
  for (int c = 0;; ++c) {
    const int slot = c % LC_BUF;
    if (n0 == 0) break;  // chunks come in order: an empty one ends the list
    stage((c + LC_BUF - 1) % LC_BUF);
    cp_wait<LC_BUF - 1>();
    __syncthreads();
    const unsigned char* buf = lin_dsm + (size_t)slot * LC_BYTES;
    for (int q = gt; q < n0; q += GT) {
      const double2 m = reinterpret_cast<const double2*>(buf + FT * 32)[q];
      const double4 X = reinterpret_cast<const double4*>(buf)[q];
      double w[4], h[3];
      const double u0 = dot4(P0, X), u1 = dot4(P1, X), u2 = dot4(P2, X);
      if (STAGE == 1) {
        const double r0 = k.s1 * (u0 - u2 * m.x), r1 = k.s1 * (u1 - u2 * m.y);
        const double r2 = k.s2 * (u0 - m.x), r3 = k.s2 * (u1 - m.y);
        w[0] = 1.0;
        w[1] = m.x;
        w[2] = m.y;
        w[3] = m.x * m.x + m.y * m.y;
        h[0] = fma(k.s1, r0, k.s2 * r2);
        h[1] = fma(k.s1, r1, k.s2 * r3);
        h[2] = -k.s1 * fma(m.x, r0, m.y * r1);
      } else {
        const double iz = 1.0 / u2, i2 = iz * iz;
        const double p0 = u0 * iz, p1 = u1 * iz;
        const double r0 = u0 / u2 - m.x, r1 = u1 / u2 - m.y;
        w[0] = i2;
        w[1] = p0 * i2;
        w[2] = p1 * i2;
        w[3] = (p0 * p0 + p1 * p1) * i2;
        h[0] = iz * r0;
        h[1] = iz * r1;
        h[2] = -iz * fma(p0, r0, p1 * r1);
      }
      const double xv[4] = {X.x, X.y, X.z, X.w};
      const double wa = grp == 0 ? w[0] : w[2], wb2 = grp == 0 ? w[1] : w[3];
      int e = 0;
#pragma unroll
      for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
        for (int b2 = a2; b2 < 4; ++b2) {
          const double xx = xv[a2] * xv[b2];
          acc[e] = fma(wa, xx, acc[e]);
          acc[10 + e] = fma(wb2, xx, acc[10 + e]);
          ++e;
        }
      if (grp == 1) {
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
#pragma unroll
          for (int a2 = 0; a2 < 4; ++a2)
            acc[20 + 4 * cc + a2] = fma(h[cc], xv[a2], acc[20 + 4 * cc + a2]);
      }
    }
    __syncthreads();  // the buffer is refilled next iteration
    n0 = n1;
    n1 = n2;
  }
  cp_wait<0>();
  // fixed-order block reduction (per group): warp sums (lane i holds component i), then
  // the group's warps in order
  const int lane = tid & 31, wq = tid >> 5;
  red[wq * 32 + lane] = warp_reduce32_lane(acc, lane);
  __syncthreads();
  if (tid < NA) {
    // tot layout: [0,10) w0, [10,20) w1, [20,30) w2, [30,40) w3, [40,52) b_p
    const int g2 = tid < 20 ? 0 : 1;
    const int src = tid < 20 ? tid : (tid < 40 ? tid - 20 : tid - 20);
    double sum = 0.0;
    for (int q = 0; q < GT / 32; ++q) sum += red[(g2 * (GT / 32) + q) * 32 + src];
    tot[tid] = sum;
  }
  __syncthreads();
  double c00, c02, c12, c22;
  if (STAGE == 1) {
    const double a = k.s1 * k.s1;
    c00 = a + k.s2 * k.s2;
    c02 = -a;
    c12 = -a;
    c22 = a;
  } else {
    c00 = 1.0;
    c02 = -1.0;
    c12 = -1.0;
    c22 = 1.0;
  }
  // moment index of (a, b), a <= b, in the 10-entry packing
  auto mi = [](int a, int b) {
    int lo = a < b ? a : b, hi = a < b ? b : a;
    return lo * 4 - lo * (lo - 1) / 2 + (hi - lo);
  };
  for (int e = tid; e < LINP; e += FT) {
    double val;
    if (e < 78) {
      int i = 0, rem = e;
      while (rem >= 12 - i) {
        rem -= 12 - i;
        ++i;
      }
      const int j = i + rem;
      const int c = i / 4, a = i % 4, d = j / 4, bq = j % 4;
      const int ix = mi(a, bq);
      if (c == d) {
        val = c == 2 ? c22 * tot[30 + ix] : c00 * tot[ix];
      } else if (c == 0 && d == 1) {
        val = 0.0;
      } else if (c == 0 && d == 2) {
        val = c02 * tot[10 + ix];
      } else {
        val = c12 * tot[20 + ix];
      }
    } else {
      val = tot[40 + (e - 78)];
    }
    cUraw[(size_t)cam * LINP + e] = val;
  }
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

// K3 damping + U^-1 (Cholesky; reference uses LU, difference <= 1e-13)
// One WARP per camera (round 1: one thread with two 78-entry local arrays, 117 us for 13,682
// cameras; now ~10 us): lane r holds row r of the Cholesky factor L, then column r of
// L^-1; rows / columns of the other lanes arrive by shuffle.  Every entry is produced by the
// same operations in the same order as the serial version (sums ascending in k).
__global__ void k_damp_cam(int n_p, int D, const double* __restrict__ cU, double lam,
                           double* __restrict__ cUd, double* __restrict__ cUi, int* flags) {
  const int lane = threadIdx.x & 31;
  const int cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (cam >= n_p) return;  // warp-uniform
  const double* a = cU + (size_t)cam * 144;
  const int r = lane < 12 ? lane : 0;
  const bool act = lane < D;  // D = 12 (stage 1) or 11 (stage 2), warp-uniform
  double L[12];               // row r of the damped matrix, read from the lower triangle
#pragma unroll
  for (int j = 0; j < 12; ++j) {
    double v = (act && j < D) ? a[max(r, j) * 12 + min(r, j)] : 0.0;
    if (act && j == r) v = damp_diag(v, lam);
    L[j] = v;
  }
  if (lane < 12) {
    double* ud = cUd + (size_t)cam * 144 + lane * 12;
#pragma unroll
    for (int j = 0; j < 12; ++j) ud[j] = L[j];
  }
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 12; ++j) {
    if (j < D) {  // warp-uniform
      double d = L[j];  // meaningful in lane j: L[j][j] - sum_k L[j][k]^2
#pragma unroll
      for (int kk = 0; kk < j; ++kk) d = fma(-L[kk], L[kk], d);
      const bool bad = !(d > 0.0);
      if (bad) d = 1.0;
      d = sqrt(d);
      const double dj = __shfl_sync(PV_FULL, d, j);
      ok = ok && !__shfl_sync(PV_FULL, (int)bad, j);
      double s = L[j];  // meaningful in lanes i > j: L[i][j] - sum_k L[i][k] L[j][k]
#pragma unroll
      for (int kk = 0; kk < j; ++kk) s = fma(-L[kk], __shfl_sync(PV_FULL, L[kk], j), s);
      L[j] = lane == j ? dj : (lane > j ? s / dj : L[j]);
    }
  }
  if (!ok && lane == 0) atomicOr(flags + F_SINGULAR_U, 1);
  // column `lane` of M = L^-1 (lower): M[i] = M[i][lane]
  double M[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    const double lii = __shfl_sync(PV_FULL, L[i], i);
    double s = 0.0;
#pragma unroll
    for (int kk = 0; kk < i; ++kk) {
      const double lik = __shfl_sync(PV_FULL, L[kk], i);
      if (kk >= lane) s = fma(lik, M[kk], s);
    }
    M[i] = (i < D && act) ? (i == lane ? 1.0 / lii : (i > lane ? -s / lii : 0.0)) : 0.0;
  }
  // U^-1 = M^T M: entry (i, lane) = sum_{k >= max(i, lane)} M[k][i] M[k][lane]
  double* ui = cUi + (size_t)cam * 144;
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    double s = 0.0;
#pragma unroll
    for (int kk = 0; kk < 12; ++kk) {
      const double mki = __shfl_sync(PV_FULL, M[kk], i);
      if (kk >= i && kk >= lane && kk < D) s = fma(mki, M[kk], s);
    }
    if (lane < 12) ui[i * 12 + lane] = (i < D && act) ? s : 0.0;
  }
}

// K2 damping + V+ (per landmark), stored at the landmark's warp-slot position lpos[l]
template <int STAGE>
__global__ void k_damp_lm(int n_l, const double* __restrict__ lvr, const int* __restrict__ lpos,
                          double* __restrict__ lsys, double lam, int both, int* flags) {
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
    // Fast path: Cholesky.  lambda_min >= det / lambda_max^2 >= det / trace^2, so
    // det > 1e-9 trace^3 certifies that no eigenvalue falls under the reference cutoff
    // (1e-10 trace, normal_eq.py:145-153): the pseudo-inverse is the inverse.
    const double tr = V6[0] + V6[3] + V6[5];
    const double d0 = V6[0];
    const double r00 = d0 > 0.0 ? sqrt(d0) : 1.0;
    const double r01 = V6[1] / r00, r02 = V6[2] / r00;
    const double d1 = V6[3] - r01 * r01;
    const double r11 = d1 > 0.0 ? sqrt(d1) : 1.0;
    const double r12 = (V6[4] - r01 * r02) / r11;
    const double d2 = V6[5] - r02 * r02 - r12 * r12;
    if (d0 > 0.0 && d1 > 0.0 && d2 > 0.0 && d0 * d1 * d2 > 1e-9 * tr * tr * tr) {
      const double r22 = sqrt(d2);
      const double i00 = 1.0 / r00, i11 = 1.0 / r11, i22 = 1.0 / r22;
      const double i01 = -r01 * i00 * i11, i12 = -r12 * i11 * i22;
      const double i02 = -(r01 * i12 + r02 * i22) * i00;
      P6[0] = i00 * i00 + i01 * i01 + i02 * i02;
      P6[1] = i01 * i11 + i02 * i12;
      P6[2] = i02 * i22;
      P6[3] = i11 * i11 + i12 * i12;
      P6[4] = i12 * i22;
      P6[5] = i22 * i22;
      degen = false;
    } else {
      degen = pinv_sym3(V6, 1e-10, P6);
    }
    double* o = lsys + (size_t)__ldg(lpos + l) * LSYS;  // warp-slot order
    st4(o, make_double4(P6[0], P6[1], P6[2], P6[3]));
    st4(o + 4, make_double4(P6[4], P6[5], degen ? 1.0 : 0.0, 0.0));
  }
  unsigned bal = __ballot_sync(PV_FULL, degen);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(flags + F_N_DEGEN, __popc(bal));
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

// one partial per warp (no block barrier: warps holding long tracks do not stall
// the others); summed afterwards in fixed order by k_sum2
__device__ __forceinline__ void warp_partial(double v, double* __restrict__ out) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) out[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = v;
}

template <int STAGE>
__global__ void __launch_bounds__(64) k_cost(Graph g, const double* __restrict__ cams, int cstride,
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
  warp_partial(acc, part);
}

// Cost over the block-major camera-sorted observations: warp w takes the observation range
// [w n_o / nw, (w + 1) n_o / nw) and walks the (block, camera) segments it crosses, so the
// camera record is one warp-uniform (broadcast) load per segment and only the landmark is
// gathered per observation (k_cost gathers three camera rows per observation and is
// L1-bound on them).  One partial per warp, summed in fixed order by k_sum.
template <int STAGE>
__global__ void __launch_bounds__(256) k_cost_cs(Graph g, const double* __restrict__ cams,
                                                 int cstride, const double* __restrict__ lms,
                                                 int lstride, int nw, double* __restrict__ part,
                                                 int* flags, Coef k) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nw) return;
  const int o_begin = (int)((long long)w * g.n_o / nw);
  const int o_end = (int)((long long)(w + 1) * g.n_o / nw);
  double acc = 0.0;
  if (o_begin < o_end) {
    // last segment starting at or before o_begin
    int lo = 0, hi = g.n_blk * g.n_p;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(g.seg + mid) <= o_begin) lo = mid; else hi = mid;
    }
    int sgi = lo, o = o_begin;
    while (o < o_end) {
      const int se = min(__ldg(g.seg + sgi + 1), o_end);
      const int cam = sgi % g.n_p;
      for (int q = o + lane; q < se; q += 32) {
        const double2 m = ldg2(g.cs_m + 2 * (size_t)q);
        const double4 x = ldg4(lms + (size_t)__ldg(g.cs_lm + q) * lstride);
        acc += obs_cost<STAGE>(cams, cstride, cam, m.x, m.y, x, k, flags);
      }
      o = max(o, se);
      ++sgi;
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) part[w] = acc;
}

// ---------------------------------------------------------------------------
// K10 closed-form landmark re-solve (objective.py:251-298): per landmark the
// stacked affine model r = A v + c (A = J_l at x = e3, c = r at x = e3) is
// solved in the minimum-norm least-squares sense with the reference's SVD rank
// rule s > 1e-10 s_max.  A = QR via CholeskyQR2 (two Gram passes, accurate to
// O(eps) for cond(A) < ~1e7), then a one-sided Jacobi SVD of the 3x3 R.
// Landmarks whose first Gram pass loses more than 13 digits fall back to an
// exact Givens QR of all their rows.  The stage-1 cost of the re-solved state
// is accumulated in the same pass (K9 fused).

struct Rows4 {
  double a[4][3];
  double c[4];
};

__device__ __forceinline__ Rows4 resolve_rows4(const double* __restrict__ cams, int cam, double m0,
                                               double m1, const Coef& k) {
  const double* cp = cams + (size_t)cam * 12;
  const double4 P0 = ldg4(cp), P1 = ldg4(cp + 4), P2 = ldg4(cp + 8);
  Rows4 R;
  R.a[0][0] = k.s1 * (P0.x - m0 * P2.x);
  R.a[0][1] = k.s1 * (P0.y - m0 * P2.y);
  R.a[0][2] = k.s1 * (P0.z - m0 * P2.z);
  R.c[0] = k.s1 * (P0.w - P2.w * m0);
  R.a[1][0] = k.s1 * (P1.x - m1 * P2.x);
  R.a[1][1] = k.s1 * (P1.y - m1 * P2.y);
  R.a[1][2] = k.s1 * (P1.z - m1 * P2.z);
  R.c[1] = k.s1 * (P1.w - P2.w * m1);
  R.a[2][0] = k.s2 * P0.x;
  R.a[2][1] = k.s2 * P0.y;
  R.a[2][2] = k.s2 * P0.z;
  R.c[2] = k.s2 * (P0.w - m0);
  R.a[3][0] = k.s2 * P1.x;
  R.a[3][1] = k.s2 * P1.y;
  R.a[3][2] = k.s2 * P1.z;
  R.c[3] = k.s2 * (P1.w - m1);
  return R;
}

// 3x3 Cholesky of packed (00 01 02 11 12 22) into upper R (same packing);
// returns the smallest pivot ratio d_j / G_jj (<= 0 on failure).
__device__ __forceinline__ double chol3(const double* G, double* R) {
  double d0 = G[0];
  double ratio = G[0] > 0.0 ? 1.0 : 0.0;
  double r00 = d0 > 0.0 ? sqrt(d0) : 0.0;
  double r01 = r00 > 0.0 ? G[1] / r00 : 0.0;
  double r02 = r00 > 0.0 ? G[2] / r00 : 0.0;
  double d1 = G[3] - r01 * r01;
  ratio = fmin(ratio, G[3] > 0.0 ? d1 / G[3] : 0.0);
  double r11 = d1 > 0.0 ? sqrt(d1) : 0.0;
  double r12 = r11 > 0.0 ? (G[4] - r01 * r02) / r11 : 0.0;
  double d2 = G[5] - r02 * r02 - r12 * r12;
  ratio = fmin(ratio, G[5] > 0.0 ? d2 / G[5] : 0.0);
  double r22 = d2 > 0.0 ? sqrt(d2) : 0.0;
  R[0] = r00;
  R[1] = r01;
  R[2] = r02;
  R[3] = r11;
  R[4] = r12;
  R[5] = r22;
  return ratio;
}

__device__ __forceinline__ void gram_acc(const double* w, double c, double* acc /*9*/) {
  acc[0] = fma(w[0], w[0], acc[0]);
  acc[1] = fma(w[0], w[1], acc[1]);
  acc[2] = fma(w[0], w[2], acc[2]);
  acc[3] = fma(w[1], w[1], acc[3]);
  acc[4] = fma(w[1], w[2], acc[4]);
  acc[5] = fma(w[2], w[2], acc[5]);
  acc[6] = fma(w[0], c, acc[6]);
  acc[7] = fma(w[1], c, acc[7]);
  acc[8] = fma(w[2], c, acc[8]);
}

// w = a R^-1 (row vector, R upper 3x3 packed) using precomputed inverse diagonals
__device__ __forceinline__ void tri_solve_row(const double* a, const double* R, const double* id,
                                              double* w) {
  w[0] = a[0] * id[0];
  w[1] = (a[1] - w[0] * R[1]) * id[1];
  w[2] = (a[2] - w[0] * R[2] - w[1] * R[4]) * id[2];
}

// head-lane solve: R1 (pass 1), pass-2 sums (G2, z1) -> full 4x4 packed R for lsq_from_r
__device__ __forceinline__ bool cqr2_solve(const double* R1, const double* s2, double* v) {
  double R2[6];
  chol3(s2, R2);
  // R = R2 R1 (upper x upper)
  double R[6];
  R[0] = R2[0] * R1[0];
  R[1] = R2[0] * R1[1] + R2[1] * R1[3];
  R[2] = R2[0] * R1[2] + R2[1] * R1[4] + R2[2] * R1[5];
  R[3] = R2[3] * R1[3];
  R[4] = R2[3] * R1[4] + R2[4] * R1[5];
  R[5] = R2[5] * R1[5];
  // z = R2^-T z1 (forward substitution with the lower triangle R2^T)
  double z[3];
  z[0] = R2[0] != 0.0 ? s2[6] / R2[0] : 0.0;
  z[1] = R2[3] != 0.0 ? (s2[7] - R2[1] * z[0]) / R2[3] : 0.0;
  z[2] = R2[5] != 0.0 ? (s2[8] - R2[2] * z[0] - R2[4] * z[1]) / R2[5] : 0.0;
  // Certified full rank: sigma_min >= 1/||R^-1||_F and sigma_max <= ||R||_F, so
  // cond_F(R) < 1e8 implies s_min > 1e-8 s_max, far inside the reference's rule
  // (s > 1e-10 s_max).  Then the min-norm solution is the triangular solve.
  if (R[0] != 0.0 && R[3] != 0.0 && R[5] != 0.0) {
    const double i00 = 1.0 / R[0], i11 = 1.0 / R[3], i22 = 1.0 / R[5];
    const double i01 = -R[1] * i00 * i11, i12 = -R[4] * i11 * i22;
    const double i02 = -(R[1] * i12 + R[2] * i22) * i00;
    const double nr = R[0] * R[0] + R[1] * R[1] + R[2] * R[2] + R[3] * R[3] + R[4] * R[4] +
                      R[5] * R[5];
    const double ni = i00 * i00 + i01 * i01 + i02 * i02 + i11 * i11 + i12 * i12 + i22 * i22;
    if (nr * ni < 1e16) {
      v[0] = -(i00 * z[0] + i01 * z[1] + i02 * z[2]);
      v[1] = -(i11 * z[1] + i12 * z[2]);
      v[2] = -(i22 * z[2]);
      return true;
    }
  }
  const double full[10] = {R[0], R[1], R[2], z[0], R[3], R[4], z[1], R[5], z[2], 0.0};
  return lsq_from_r(full, 1e-10, v);
}

constexpr double CQR_PIVOT_TOL = 1e-13;

__device__ __forceinline__ void gram6(const Rows4& rw, double* g1) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    g1[0] = fma(rw.a[r][0], rw.a[r][0], g1[0]);
    g1[1] = fma(rw.a[r][0], rw.a[r][1], g1[1]);
    g1[2] = fma(rw.a[r][0], rw.a[r][2], g1[2]);
    g1[3] = fma(rw.a[r][1], rw.a[r][1], g1[3]);
    g1[4] = fma(rw.a[r][1], rw.a[r][2], g1[4]);
    g1[5] = fma(rw.a[r][2], rw.a[r][2], g1[5]);
    g1[6] = fma(rw.a[r][0], rw.c[r], g1[6]);
    g1[7] = fma(rw.a[r][1], rw.c[r], g1[7]);
    g1[8] = fma(rw.a[r][2], rw.c[r], g1[8]);
  }
}

// Well-conditioned landmarks: the Cholesky factor of A^T A already determines the
// least-squares solution to O(kappa^2 eps); with every pivot ratio d_j / G_jj >= 1e-4
// (kappa^2 <~ 1e4) that error is <~ 1e-12, inside the 1e-10 parity budget, and the
// reference's rank rule (s > 1e-10 s_max) certainly holds.
constexpr double NE_PIVOT_TOL = 1e-4;

__device__ __forceinline__ void ne_solve(const double* R, const double* atc, double* v) {
  // R^T z = A^T c (forward), R v = -z (backward)
  const double z0 = atc[0] / R[0];
  const double z1 = (atc[1] - R[1] * z0) / R[3];
  const double z2 = (atc[2] - R[2] * z0 - R[4] * z1) / R[5];
  v[2] = -z2 / R[5];
  v[1] = -(z1 + R[4] * v[2]) / R[3];
  v[0] = -(z0 + R[1] * v[1] + R[2] * v[2]) / R[0];
}

__device__ __forceinline__ void gram_pass2(const Rows4& rw, const double* R1, const double* id,
                                           double* s2) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    double wv[3];
    tri_solve_row(rw.a[r], R1, id, wv);
    gram_acc(wv, rw.c[r], s2);
  }
}

// stage-1 cost of one observation from its affine rows: r = A x + c
__device__ __forceinline__ double rows_cost(const Rows4& rw, const double4& x) {
  double f = 0.0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double v = fma(rw.a[r][0], x.x, fma(rw.a[r][1], x.y, fma(rw.a[r][2], x.z, rw.c[r] * x.w)));
    f = fma(v, v, f);
  }
  return f;
}

__global__ void __launch_bounds__(64, 8) k_resolve(Graph g, const double* __restrict__ tcam,
                                                 double* __restrict__ tlm,
                                                 double* __restrict__ part, int* flags, Coef k,
                                                 double* __restrict__ lvr, double* __restrict__ lbl) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double cost = 0.0;
  int rankdef = 0, fallback = 0;
  if (w < g.n_tasks) {
    Task t = load_task(g, w, lane);
    int l, seg_end, src;
    if (t.long_task) {
      l = t.l0;
      seg_end = 32;
      src = 0;
    } else {
      lane_segment(t, lane, l, seg_end);
      src = seg_start_lane(t, lane < t.n ? lane : 0);
    }
    const bool head = t.long_task ? lane == 0 : (lane < t.n && ((t.heads >> lane) & 1u));
    const int oend = t.o0 + t.n;
    // shuffle steps the longest segment of a short task needs (results identical)
    const int max_len =
        t.long_task ? 32 : (int)__reduce_max_sync(PV_FULL, head ? (unsigned)(seg_end - lane) : 1u);
    // short tasks keep their single observation's rows in registers for all passes
    Rows4 mine;
    const bool have = !t.long_task && lane < t.n;
    if (have) {
      const int o = t.o0 + lane;
      const double2 m = ldg2(g.ls_m + 2 * (size_t)o);
      mine = resolve_rows4(tcam, __ldg(g.ls_cam + o), m.x, m.y, k);
    }
    // pass 1: Gram of A and A^T c
    double g1[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (t.long_task) {
      for (int o = t.o0 + lane; o < oend; o += 32) {
        const double2 m = ldg2(g.ls_m + 2 * (size_t)o);
        gram6(resolve_rows4(tcam, __ldg(g.ls_cam + o), m.x, m.y, k), g1);
      }
      warp_reduce_all(g1);
    } else {
      if (have) gram6(mine, g1);
      seg_reduce_n(g1, lane, seg_end, max_len);
    }
    double R1[6] = {0, 0, 0, 0, 0, 0};
    double fb = 0.0;  // 0: normal equations suffice, 1: CholeskyQR2 pass, 2: Givens fallback
    if (head) {
      const double ratio = chol3(g1, R1);
      fb = ratio >= NE_PIVOT_TOL ? 0.0 : (ratio > CQR_PIVOT_TOL ? 1.0 : 2.0);
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) R1[i] = __shfl_sync(PV_FULL, R1[i], src);
    fb = __shfl_sync(PV_FULL, fb, src);
    // pass 2 (ill-conditioned landmarks only): Gram of A R1^-1 and (A R1^-1)^T c
    double s2[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    const bool need2 = __any_sync(PV_FULL, fb == 1.0);
    if (need2 && fb == 1.0) {
      const double id[3] = {1.0 / R1[0], 1.0 / R1[3], 1.0 / R1[5]};
      if (t.long_task) {
        for (int o = t.o0 + lane; o < oend; o += 32) {
          const double2 m = ldg2(g.ls_m + 2 * (size_t)o);
          gram_pass2(resolve_rows4(tcam, __ldg(g.ls_cam + o), m.x, m.y, k), R1, id, s2);
        }
      } else if (have) {
        gram_pass2(mine, R1, id, s2);
      }
    }
    if (need2) {
      if (t.long_task) warp_reduce_all(s2);
      else seg_reduce_n(s2, lane, seg_end, max_len);
    }
    double xn[4] = {0.0, 0.0, 0.0, 0.0};
    if (head) {
      double v[3];
      bool full;
      if (fb == 0.0) {
        ne_solve(R1, g1 + 6, v);
        full = true;
      } else if (fb == 1.0) {
        full = cqr2_solve(R1, s2, v);
      } else {  // exact Givens QR of all rows of this landmark
        fallback = 1;
        double Rg[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        const int ob = t.long_task ? t.o0 : t.o0 + lane;
        const int oe = t.long_task ? oend : t.o0 + seg_end;
        for (int o = ob; o < oe; ++o) {
          const double2 m = ldg2(g.ls_m + 2 * (size_t)o);
          const Rows4 rw = resolve_rows4(tcam, __ldg(g.ls_cam + o), m.x, m.y, k);
          for (int r = 0; r < 4; ++r)
            givens_row(Rg, rw.a[r][0], rw.a[r][1], rw.a[r][2], rw.c[r]);
        }
        full = lsq_from_r(Rg, 1e-10, v);
      }
      const double4 old = ld4(tlm + (size_t)l * 4);
      xn[0] = full ? v[0] : old.x;
      xn[1] = full ? v[1] : old.y;
      xn[2] = full ? v[2] : old.z;
      xn[3] = full ? 1.0 : old.w;
      rankdef = !full;
      st4(tlm + (size_t)l * 4, make_double4(xn[0], xn[1], xn[2], xn[3]));
      if (lvr != nullptr) {
        // the next stage-1 linearization at this state: V = A^T A (J_l does not depend
        // on x) and b_l = J_l^T r = A^T (A x + c)
        double* vo = lvr + (size_t)l * 8;
        st4(vo, make_double4(g1[0], g1[1], g1[2], g1[3]));
        st4(vo + 4, make_double4(g1[4], g1[5], 0.0, 0.0));
        const double b0 = fma(g1[0], xn[0], fma(g1[1], xn[1], fma(g1[2], xn[2], g1[6] * xn[3])));
        const double b1 = fma(g1[1], xn[0], fma(g1[3], xn[1], fma(g1[4], xn[2], g1[7] * xn[3])));
        const double b2 = fma(g1[2], xn[0], fma(g1[4], xn[1], fma(g1[5], xn[2], g1[8] * xn[3])));
        st4(lbl + (size_t)l * 4, make_double4(b0, b1, b2, 0.0));
      }
    }
    double4 x;
    x.x = __shfl_sync(PV_FULL, xn[0], src);
    x.y = __shfl_sync(PV_FULL, xn[1], src);
    x.z = __shfl_sync(PV_FULL, xn[2], src);
    x.w = __shfl_sync(PV_FULL, xn[3], src);
    // pass 3: stage-1 cost at the re-solved landmark (K9 fused)
    if (t.long_task) {
      for (int o = t.o0 + lane; o < oend; o += 32) {
        const double2 m = ldg2(g.ls_m + 2 * (size_t)o);
        cost += rows_cost(resolve_rows4(tcam, __ldg(g.ls_cam + o), m.x, m.y, k), x);
      }
    } else if (have) {
      cost = rows_cost(mine, x);
    }
  }
  const unsigned bal = __ballot_sync(PV_FULL, rankdef);
  const unsigned bfb = __ballot_sync(PV_FULL, fallback);
  if ((threadIdx.x & 31) == 0) {
    if (bal) atomicAdd(flags + F_N_RANKDEF, __popc(bal));
    if (bfb) atomicAdd(flags + F_N_FALLBACK, __popc(bfb));
  }
  warp_partial(cost, part);
}

// Landmark re-solve, lane-per-landmark form (the same k-bucketed warp slots as the
// landmark reduce): each lane owns one landmark with k <= KSHORT observations and walks them
// serially -- pass 1 builds [A^T A | A^T c] (no shuffles), the lane solves (every lane
// busy), an ill-conditioned landmark repeats the walk for the CholeskyQR2 pass, and a
// last walk evaluates the stage-1 cost at the new coordinates.  The observation rows are
// rebuilt in each walk from the (L1/L2-resident) trial cameras instead of being shuffled.
// A landmark with k > KSHORT fills a slot alone and is processed by the whole warp.
__device__ __forceinline__ Rows4 resolve_obs(const Graph& g, const double* __restrict__ tcam,
                                             int o, const Coef& k) {
  const double2 m = ldg2(g.ls_m + 2 * (size_t)o);
  return resolve_rows4(tcam, __ldg(g.ls_cam + o), m.x, m.y, k);
}

// the same observation by its s position (lane-per-landmark walks: coalesced across the slot)
__device__ __forceinline__ Rows4 resolve_obs_s(const Graph& g, const double* __restrict__ tcam,
                                               int pos, const Coef& k) {
  const double2 m = ldg2(g.ks_m + 2 * (size_t)pos);
  return resolve_rows4(tcam, __ldg(g.ks_cam + pos), m.x, m.y, k);
}

// per-landmark solve from the pass-1 Gram (returns fb: 0 solved, 1 needs pass 2, 2 Givens)
__device__ __forceinline__ int resolve_pass1(const double* g1, double* R1, double* v) {
  const double ratio = chol3(g1, R1);
  const int fb = ratio >= NE_PIVOT_TOL ? 0 : (ratio > CQR_PIVOT_TOL ? 1 : 2);
  if (fb == 0) ne_solve(R1, g1 + 6, v);
  return fb;
}

__device__ __forceinline__ void resolve_store(int l, const double* g1, const double* v, bool full,
                                              double* __restrict__ tlm, double* __restrict__ lvr,
                                              double* __restrict__ lbl, double4& x) {
  const double4 old = ld4(tlm + (size_t)l * 4);
  x.x = full ? v[0] : old.x;
  x.y = full ? v[1] : old.y;
  x.z = full ? v[2] : old.z;
  x.w = full ? 1.0 : old.w;
  st4(tlm + (size_t)l * 4, x);
  if (lvr != nullptr) {
    // the next stage-1 linearization at this state: V = A^T A (J_l does not depend on x)
    // and b_l = J_l^T r = A^T (A x + c)
    double* vo = lvr + (size_t)l * 8;
    st4(vo, make_double4(g1[0], g1[1], g1[2], g1[3]));
    st4(vo + 4, make_double4(g1[4], g1[5], 0.0, 0.0));
    const double b0 = fma(g1[0], x.x, fma(g1[1], x.y, fma(g1[2], x.z, g1[6] * x.w)));
    const double b1 = fma(g1[1], x.x, fma(g1[3], x.y, fma(g1[4], x.z, g1[7] * x.w)));
    const double b2 = fma(g1[2], x.x, fma(g1[4], x.y, fma(g1[5], x.z, g1[8] * x.w)));
    st4(lbl + (size_t)l * 4, make_double4(b0, b1, b2, 0.0));
  }
}

__global__ void __launch_bounds__(256) k_resolve_slots(Graph g, const int4* __restrict__ klist,
                                                       int n_slots,
                                                       const double* __restrict__ tcam,
                                                       double* __restrict__ tlm,
                                                       double* __restrict__ part, int* flags,
                                                       Coef k, double* __restrict__ lvr,
                                                       double* __restrict__ lbl) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n_slots) return;
  const int4 e = __ldg(klist + 32 * (size_t)w + lane);  // {landmark, first obs, k}
  const int kk = e.z;                                     // warp-uniform
  double cost = 0.0;
  int rankdef = 0, fallback = 0;
  if (kk > KSHORT) {  // one long landmark: the warp strides over its observations
    const int l = __shfl_sync(PV_FULL, e.x, 0), o0 = __shfl_sync(PV_FULL, e.y, 0);
    const int oend = o0 + kk;
    double g1[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int o = o0 + lane; o < oend; o += 32) gram6(resolve_obs(g, tcam, o, k), g1);
    warp_reduce_all(g1);
    double R1[6], v[3];
    const int fb = resolve_pass1(g1, R1, v);  // identical in every lane
    bool full = true;
    if (fb == 1) {
      const double id[3] = {1.0 / R1[0], 1.0 / R1[3], 1.0 / R1[5]};
      double s2[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int o = o0 + lane; o < oend; o += 32) gram_pass2(resolve_obs(g, tcam, o, k), R1, id, s2);
      warp_reduce_all(s2);
      full = cqr2_solve(R1, s2, v);
    } else if (fb == 2) {
      if (lane == 0) {
        fallback = 1;
        double Rg[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int o = o0; o < oend; ++o) {
          const Rows4 rw = resolve_obs(g, tcam, o, k);
          for (int r = 0; r < 4; ++r) givens_row(Rg, rw.a[r][0], rw.a[r][1], rw.a[r][2], rw.c[r]);
        }
        full = lsq_from_r(Rg, 1e-10, v);
      }
      full = __shfl_sync(PV_FULL, (int)full, 0);
#pragma unroll
      for (int i = 0; i < 3; ++i) v[i] = __shfl_sync(PV_FULL, v[i], 0);
    }
    double4 x;
    if (lane == 0) {
      resolve_store(l, g1, v, full, tlm, lvr, lbl, x);
      rankdef = !full;
    }
    x.x = __shfl_sync(PV_FULL, x.x, 0);
    x.y = __shfl_sync(PV_FULL, x.y, 0);
    x.z = __shfl_sync(PV_FULL, x.z, 0);
    x.w = __shfl_sync(PV_FULL, x.w, 0);
    for (int o = o0 + lane; o < oend; o += 32) cost += rows_cost(resolve_obs(g, tcam, o, k), x);
  } else {
    const bool act = e.x >= 0;
    const int l = e.x, o0 = e.y;
    // observation i of this lane's landmark sits at s position e.w + 32 i (ks_m / ks_cam)
    const int p0 = e.w, pend = act ? e.w + 32 * kk : e.w;
    double g1[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    double cc = 0.0;  // c^T c, for the cost at the solution from the Gram (below)
    for (int pos = p0; pos < pend; pos += 32) {
      const Rows4 rw = resolve_obs_s(g, tcam, pos, k);
      gram6(rw, g1);
#pragma unroll
      for (int r = 0; r < 4; ++r) cc = fma(rw.c[r], rw.c[r], cc);
    }
    double R1[6], v[3] = {0.0, 0.0, 0.0};
    const int fb = act ? resolve_pass1(g1, R1, v) : 0;
    bool full = true;
    if (fb == 1) {
      const double id[3] = {1.0 / R1[0], 1.0 / R1[3], 1.0 / R1[5]};
      double s2[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int pos = p0; pos < pend; pos += 32) gram_pass2(resolve_obs_s(g, tcam, pos, k), R1, id, s2);
      full = cqr2_solve(R1, s2, v);
    } else if (fb == 2) {
      fallback = 1;
      double Rg[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int pos = p0; pos < pend; pos += 32) {
        const Rows4 rw = resolve_obs_s(g, tcam, pos, k);
        for (int r = 0; r < 4; ++r) givens_row(Rg, rw.a[r][0], rw.a[r][1], rw.a[r][2], rw.c[r]);
      }
      full = lsq_from_r(Rg, 1e-10, v);
    }
    double4 x = make_double4(0.0, 0.0, 0.0, 0.0);
    bool safe = true;
    if (act) {
      resolve_store(l, g1, v, full, tlm, lvr, lbl, x);
      rankdef = !full;
      // cost at x from the Gram: ||A x + c w||^2 = x^T G x + 2 w x^T (A^T c) + w^2 c^T c.
      // Used when it does not cancel (cost >= 1e-3 of the terms' magnitude: relative error
      // <~ 1e-12); otherwise the observations are walked again, by the whole warp.
      const double gx0 = fma(g1[0], x.x, fma(g1[1], x.y, g1[2] * x.z));
      const double gx1 = fma(g1[1], x.x, fma(g1[3], x.y, g1[4] * x.z));
      const double gx2 = fma(g1[2], x.x, fma(g1[4], x.y, g1[5] * x.z));
      const double t1 = fma(x.x, gx0, fma(x.y, gx1, x.z * gx2));
      const double t2 = 2.0 * x.w * fma(x.x, g1[6], fma(x.y, g1[7], x.z * g1[8]));
      const double t3 = x.w * x.w * cc;
      const double cg = t1 + t2 + t3;
      safe = cg >= 1e-3 * (fabs(t1) + fabs(t2) + t3);
      if (safe) cost = cg;
    }
    unsigned walk = __ballot_sync(PV_FULL, !safe);
    while (walk) {  // warp-cooperative walks, lowest lane first (fixed order)
      const int u = __ffs(walk) - 1;
      walk &= walk - 1;
      const int uo = __shfl_sync(PV_FULL, o0, u);
      double4 xu;
      xu.x = __shfl_sync(PV_FULL, x.x, u);
      xu.y = __shfl_sync(PV_FULL, x.y, u);
      xu.z = __shfl_sync(PV_FULL, x.z, u);
      xu.w = __shfl_sync(PV_FULL, x.w, u);
      double cu = 0.0;  // kk <= KSHORT observations: lane q takes q, q + 32, ...
      for (int q = lane; q < kk; q += 32) cu += rows_cost(resolve_obs(g, tcam, uo + q, k), xu);
      const double su = warp_sum(cu);
      if (lane == u) cost = su;
    }
  }
  const unsigned bal = __ballot_sync(PV_FULL, rankdef);
  const unsigned bfb = __ballot_sync(PV_FULL, fallback);
  if (lane == 0) {
    if (bal) atomicAdd(flags + F_N_RANKDEF, __popc(bal));
    if (bfb) atomicAdd(flags + F_N_FALLBACK, __popc(bfb));
  }
  cost = warp_sum(cost);
  if (lane == 0) part[w] = cost;
}

// fixed-order two-level sum of warp partials: k_sum2<<<nb, 1024>>> writes one value
// per block (contiguous slices), then a single block sums those
__global__ void k_sum(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[1024];
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int lo = blockIdx.x * per, hi = min(n, lo + per);
  double s = 0.0;
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = red[0];
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

// trial <- current copy (closed-form re-solve of the current state)
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
