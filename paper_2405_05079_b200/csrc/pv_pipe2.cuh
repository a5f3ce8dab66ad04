// Warp-specialized, dynamically scheduled form of the persistent camera kernel (k_cam_pipe,
// pv_pipe.cuh): y_i (+)= sum_{j in block bc} W_ij t_j, then s_ij = W_ij^T v_i for j in
// block ba.
//
// Why (profiles/r2_pipe.md):
//   * ncu of k_cam_pipe: ~270 of the ~340 warp instructions per 64-observation item are
//     bookkeeping -- descriptor window shuffles, the lane-0 TMA issue and its branches, slot
//     and parity arithmetic -- executed by the warps that do the fp64 math;
//   * per-warp timers of one launch (tools/pipe_tail.py): with static, cost-balanced camera
//     ranges per warp the consumers finish between 49 and 65 us (median 58): a ~12% tail.
//
// Here each CTA has NC consumer warps and ONE producer warp:
//
//   * the unit of work is a (camera, landmark block) segment of the block-major camera-sorted
//     order: first the W t segments of block bc (every camera: y is written even for an
//     empty segment), then the W^T v segments of block ba.  Producer lane w (< NC) takes the
//     next segment for consumer w from a grid-wide counter (one atomicAdd per segment, one
//     segment ahead), cuts it into items of <= PCH observations and refills consumer w's
//     D-slot ring with TMA bulk copies (x, m, ids, the 192-byte camera record) as soon as the
//     consumer releases a slot; when the counter runs out it posts an END item.  Lanes poll
//     their consumer's "empty" mbarrier without blocking (test_wait), in lock step;
//   * a consumer waits on the slot's "full" mbarrier, issues the L2 gathers of t for the NEXT
//     item (cp.async, one item ahead), computes the current item and releases the slot with an
//     mbarrier arrive -- the standard TMA producer / consumer handshake (the refill is ordered
//     after the consumer's reads by the empty barrier; no proxy fence).
//
// Deterministic: a segment is always processed whole by one warp with the observation-to-lane
// assignment, per-lane accumulation order and warp reduction of k_cam_pipe (and of k_cam with
// one warp per camera), so every path gives the same bits whichever warp takes a segment.
// The counter resets itself: the last CTA to finish zeroes it for the next launch.
#pragma once
#include "pv_pipe.cuh"

namespace pv {

#ifndef PV_PIPE2_NC
#define PV_PIPE2_NC 3
#endif
#ifndef PV_PIPE2_D
#define PV_PIPE2_D 3
#endif
#ifndef PV_PIPE2_MINB
#define PV_PIPE2_MINB 5
#endif

constexpr int P2C = PV_PIPE2_NC;  // consumer warps per CTA
constexpr int P2D = PV_PIPE2_D;   // ring depth per consumer
constexpr int P2T = (P2C + 1) * 32;
constexpr int P2WARP = P2D * PSLOT + 2 * PT_BYTES;  // one consumer's ring + t double buffer
constexpr int P2BAR = ((2 * P2C * P2D * 8 + 127) / 128) * 128;
constexpr int PIPE2_SMEM = P2BAR + P2C * P2WARP;
constexpr int PF_END = 4;  // no more work for this consumer

__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

#ifdef PV_PIPE2_TIMING
// diagnostic build: per consumer warp, globaltimer at its start and end of the last launch
__device__ unsigned long long g_pipe2_t[2 * 8192];
__device__ int g_pipe2_items[8192];
__device__ unsigned long long g_pipe2_entry[4096];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

// ctr[0]: next segment (0 .. n_hc + n_ha - 1), ctr[1]: CTAs done (self-reset)
template <int STAGE, bool HC, bool HA>
__global__ void __launch_bounds__(P2T, PV_PIPE2_MINB) k_cam_pipe2(
    Graph g, const double* __restrict__ crec, const double* __restrict__ cs_x,
    const double* __restrict__ tarr, double* __restrict__ sbuf, double* __restrict__ cy,
    const PowerCtl* __restrict__ ctl, Coef k, Tune tune, int bc, int first_c, int ba,
    int check_stop, int disc_lo, int disc_hi, int* __restrict__ ctr) {
  extern __shared__ __align__(128) unsigned char pipe_dsm[];
#ifdef PV_PIPE2_TIMING
  if (HC && HA && threadIdx.x == 0) g_pipe2_entry[blockIdx.x] = gtimer();
#endif
  if (check_stop && ctl->stopped) return;  // grid-uniform
  discard_s_lines(sbuf, disc_lo, disc_hi);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint64_t* full = reinterpret_cast<uint64_t*>(pipe_dsm);  // [P2C][P2D]
  uint64_t* empty = full + P2C * P2D;                       // [P2C][P2D]
  if (threadIdx.x < P2C * P2D) {
    mbar_init(full + threadIdx.x, 1);
    mbar_init(empty + threadIdx.x, 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int np = g.n_p;
  const int n_hc = HC ? np : 0, n_tasks = n_hc + (HA ? np : 0);

  if (warp == P2C) {  // ---------------------------------------------------------- producer
    const uint64_t pf = pol_sel(tune.pol_stream), pt = pol_sel(tune.pol_t);
    const bool mine = lane < P2C;
    unsigned char* ring = pipe_dsm + P2BAR + (size_t)(mine ? lane : 0) * P2WARP;
    uint64_t* myfull = full + (mine ? lane : 0) * P2D;
    uint64_t* myempty = empty + (mine ? lane : 0) * P2D;
    // a segment: task index -> (camera, first observation, count, pass flag)
    auto seg_of = [&](int t, int& cam, int& lo, int& cnt, int& fl) {
      if (t >= n_tasks) {
        cam = lo = cnt = 0;
        fl = PF_END;
        return;
      }
      const bool ha = t >= n_hc;
      cam = ha ? t - n_hc : t;
      const int* sb = g.seg + (size_t)(ha ? ba : bc) * np + cam;
      lo = __ldg(sb);
      cnt = __ldg(sb + 1) - lo;
      fl = ha ? PF_HA : 0;
    };
    int nxt = mine ? atomicAdd(ctr, 1) : n_tasks;  // one segment ahead
    int cam = 0, lo = 0, cnt = 0, fl = PF_END, q = 0, nq = 0;
    bool active = mine;
    int n = 0;  // ring position
    while (__any_sync(PV_FULL, active)) {
      const int s = n % P2D;
      bool ready =
          active && (n < P2D || mbar_test(myempty + s, (unsigned)(((n / P2D) - 1) & 1)));
      if (ready) {
        while (q >= nq) {  // next non-empty segment (a W t segment always has one item)
          seg_of(nxt, cam, lo, cnt, fl);
          if (fl & PF_END) break;
          nxt = atomicAdd(ctr, 1);
          q = 0;
          nq = (cnt + PCH - 1) / PCH;
          if (!(fl & PF_HA)) nq = max(1, nq);
        }
        unsigned char* slot = ring + s * PSLOT;
        uint64_t* f = myfull + s;
        if (fl & PF_END) {
          *reinterpret_cast<int4*>(slot + PH_OFF) = make_int4(0, 0, 0, PF_END);
          mbar_arrive(f);
          active = false;
        } else {
          const int o = lo + q * PCH, c = max(0, min(PCH, cnt - q * PCH));
          const int flags = fl | (q == nq - 1 ? PF_LAST : 0);
          *reinterpret_cast<int4*>(slot + PH_OFF) = make_int4(cam, o, c, flags);
          if (c > 0) {
            const int* ids = (fl & PF_HA) ? g.cs_pos : g.cs_kpos;
            const int i0 = o & ~3, i1 = (o + c + 3) & ~3;
            const unsigned bx = (unsigned)c * 32u, bm = (unsigned)c * 16u,
                           bi = (unsigned)(i1 - i0) * 4u;
            mbar_arrive_tx(f, bx + bm + bi + 192u);
            bulk_g2s(slot + PX_OFF, cs_x + 4 * (size_t)o, bx, f, pf);
            bulk_g2s(slot + PM_OFF, g.cs_m + 2 * (size_t)o, bm, f, pf);
            bulk_g2s(slot + PI_OFF, ids + i0, bi, f, pf);
            bulk_g2s(slot + PC_OFF, crec + (size_t)cam * CREC, 192u, f, pt);
          } else {
            mbar_arrive(f);  // header only (a camera without observations in block bc)
          }
          ++q;
        }
        ++n;
      }
      if (!__any_sync(PV_FULL, ready)) __nanosleep(64);
    }
  } else {  // -------------------------------------------------------------------- consumer
    const int cw = warp;
#ifdef PV_PIPE2_TIMING
    const unsigned long long t_start = gtimer();
    int n_items = 0;
#endif
    const uint64_t pt = pol_sel(tune.pol_t), ps = pol_sel(tune.pol_s);
    unsigned char* wsm = pipe_dsm + P2BAR + (size_t)cw * P2WARP;
    unsigned char* tbuf = wsm + P2D * PSLOT;
    uint64_t* myfull = full + cw * P2D;
    uint64_t* myempty = empty + cw * P2D;

    // t_j of every observation of a W t item (its ids have landed)
    auto gather = [&](int item, const int4& h) {
      if (h.w & (PF_HA | PF_END)) return;
      const unsigned char* slot = wsm + (item % P2D) * PSLOT;
      const int* si = reinterpret_cast<const int*>(slot + PI_OFF) + (h.y & 3);
      unsigned char* tb = tbuf + (item & 1) * PT_BYTES;
#pragma unroll
      for (int r = 0; r < (PCH + 31) / 32; ++r) {
        const int qq = lane + 32 * r;
        if (qq >= h.z) continue;
        const double* src = tarr + 4 * (size_t)si[qq];
        cp_async16wp(tb + 32 * qq, src, pt);
        cp_async16wp(tb + 32 * qq + 16, src + 2, pt);
      }
    };

    mbar_wait(myfull, 0);
    __syncwarp();
    int4 hn = *reinterpret_cast<const int4*>(wsm + PH_OFF);
    gather(0, hn);
    cp_commit();

    double acc[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) acc[i] = 0.0;

    for (int c = 0; !(hn.w & PF_END); ++c) {
      const int4 h = hn;
      // t gathers of the next item, in flight while this one computes
      mbar_wait(myfull + (c + 1) % P2D, (unsigned)(((c + 1) / P2D) & 1));
      __syncwarp();
      hn = *reinterpret_cast<const int4*>(wsm + ((c + 1) % P2D) * PSLOT + PH_OFF);
      gather(c + 1, hn);
      cp_commit();
      cp_wait<1>();
      __syncwarp();

      const unsigned char* slot = wsm + (c % P2D) * PSLOT;
      const int cam = h.x, o0 = h.y, n = h.z, fl = h.w;
      const double4* cr = reinterpret_cast<const double4*>(slot + PC_OFF);
      const double4* sx = reinterpret_cast<const double4*>(slot + PX_OFF);
      const double2* sm = reinterpret_cast<const double2*>(slot + PM_OFF);
      if (!(fl & PF_HA)) {
        if (HC) {
          if (n > 0) {
            const double4 P0 = cr[0], P1 = cr[1], P2v = cr[2];
            const double4* tq = reinterpret_cast<const double4*>(tbuf + (c & 1) * PT_BYTES);
#pragma unroll
            for (int r = 0; r < (PCH + 31) / 32; ++r) {
              const int qq = lane + 32 * r;
              if (qq >= n) continue;
              const double4 X = sx[qq];
              const double2 m = sm[qq];
              const double4 T = tq[qq];
              const Proj pj = STAGE == 1 ? proj_s1(m.x, m.y, k.s) : proj_s2(P0, P1, P2v, X);
              double sg[3];
              proj_map<STAGE>(pj, dot4(P0, T), dot4(P1, T), dot4(P2v, T), sg[0], sg[1], sg[2]);
#pragma unroll
              for (int cc = 0; cc < 3; ++cc) {
                acc[4 * cc + 0] = fma(sg[cc], X.x, acc[4 * cc + 0]);
                acc[4 * cc + 1] = fma(sg[cc], X.y, acc[4 * cc + 1]);
                acc[4 * cc + 2] = fma(sg[cc], X.z, acc[4 * cc + 2]);
                acc[4 * cc + 3] = fma(sg[cc], X.w, acc[4 * cc + 3]);
              }
            }
          }
          if (fl & PF_LAST) {  // camera done: fixed-order warp reduction, write y
            const double mine = warp_reduce12_lane(acc, lane);
            if (lane < 12) {
              double* yp = cy + (size_t)cam * 12 + lane;
              *yp = first_c ? mine : *yp + mine;
            }
#pragma unroll
            for (int i = 0; i < 12; ++i) acc[i] = 0.0;
          }
        }
      } else if (HA) {
        const double4 P0 = cr[0], P1 = cr[1], P2v = cr[2];
        const double4 v0 = cr[3], v1 = cr[4], v2 = cr[5];
        const int* si = reinterpret_cast<const int*>(slot + PI_OFF) + (o0 & 3);
#pragma unroll
        for (int r = 0; r < (PCH + 31) / 32; ++r) {
          const int qq = lane + 32 * r;
          if (qq >= n) continue;
          const double4 X = sx[qq];
          const double2 m = sm[qq];
          const int pos = si[qq];
          const Proj pj = STAGE == 1 ? proj_s1(m.x, m.y, k.s) : proj_s2(P0, P1, P2v, X);
          double f0, f1, f2;
          proj_map<STAGE>(pj, dot4(X, v0), dot4(X, v1), dot4(X, v2), f0, f1, f2);
          double4 sv;
          sv.x = fma(f0, P0.x, fma(f1, P1.x, f2 * P2v.x));
          sv.y = fma(f0, P0.y, fma(f1, P1.y, f2 * P2v.y));
          sv.z = fma(f0, P0.z, fma(f1, P1.z, f2 * P2v.z));
          sv.w = STAGE == 2 ? fma(f0, P0.w, fma(f1, P1.w, f2 * P2v.w)) : 0.0;
          st4p(sbuf + 4 * (size_t)pos, sv, ps);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(myempty + c % P2D);  // slot c may be refilled
#ifdef PV_PIPE2_TIMING
      ++n_items;
#endif
    }
    cp_wait<0>();
#ifdef PV_PIPE2_TIMING
    if (HC && HA && lane == 0) {  // the fused launches only
      const int gw = blockIdx.x * P2C + cw;
      g_pipe2_t[2 * gw] = t_start;
      g_pipe2_t[2 * gw + 1] = gtimer();
      g_pipe2_items[gw] = n_items;
    }
#endif
  }
  // the last CTA out resets the segment counter for the next launch (stream order)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
  }
}

}  // namespace pv
