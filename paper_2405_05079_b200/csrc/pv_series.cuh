// The whole power series x = sum_i (U^-1 S')^i t_0 (solvers.py:140-149) as ONE persistent
// cooperative kernel: every term's landmark reduces, camera passes, U^-1 epilogue and stop
// test run inside it, separated by grid barriers instead of kernel boundaries.
//
// Why (profiles/r2_series.md; measured outcome: no gain, opt-in): with one launch per landmark block and pass a term is 26
// dependent launches of 20-70 us at vlarge; the HC-only + HA-only launches of a block take
// ~8.5 us longer than the fused one, i.e. every launch boundary costs ~8 us of drain, launch
// latency and pipeline refill -- ~0.2 ms of a 1.06 ms term.
//
// Schedule of one term over B landmark blocks (s, t, y as in pv_pipe.cuh; every step ends
// with a grid barrier, B + 2 per term):
//
//   step -2:  W^T v (0)
//   step -1:  R(0), W^T v (1)
//   step  k:  R(k+1), W t (k), W^T v (k+2)           k = 0 .. B-1 (out-of-range parts dropped)
//
// In step B-1 the warp that completes a camera's y runs the epilogue for it at once (v = U^-1 y,
// x += v, norms, y still in registers), and the LAST CTA to arrive at that step's barrier sums
// the norms in the order of k_cam's last CTA and takes the stop decision before it releases
// the others.
//
// R(b) is the landmark reduce t_j = V+_j sum_i s_ij of block b (k_lm_reduce's slots, here
// from a per-warp slot list); inside a step each warp first reduces its slots -- so the
// consumed partials s(k+1) are dropped from L2 (per slot, 128-byte aligned regions) before
// s(k+2) grows -- then walks its W t and W^T v items through the TMA ring of k_cam_pipe.
// The three parts of a step are independent (R(k+1) needs s(k+1) from step k-1, W t (k)
// needs t(k) from step k-1), and y accumulates over the blocks in order, so every number is
// produced by the same operations in the same order as in the launch-per-block path: the
// results are bit-identical to it (tests/test_gpu_variants.py).
//
// Work lists (povar.cu build_pipe_items): W t items family 0, W^T v items family 1 (alone)
// and family 3 (compensating the R and W t load of the same step), R slots per block.
#pragma once
#include "pv_pipe.cuh"

namespace pv {

#ifdef PV_SER_INLINE
#define PV_SER_FN __forceinline__
#else
#define PV_SER_FN __noinline__
#endif

struct SeriesArgs {
  const int4* item;
  const int* off;     // [(L * B + b) * (W + 1) + w]
  const int* rslot;   // slot ids of the per-warp R lists
  const int* roff;    // [b * (W + 1) + w]
  int B, W;
  const int4* klist;
  double* crec;
  const double* cs_x;
  const double* cs_m1;
  double* tarr;
  double* sbuf;
  double* cy;
  const double* lsys;
  const double* lrec;
  const double* cUi;
  double* cx;
  const double* ch;
  double* nrm;
  PowerCtl* ctl;
  unsigned* bar;  // [0] arrivals (monotonic within a launch), [1] released generation
  int max_order;
  double thr;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_all() {
  asm volatile("fence.proxy.async;" ::: "memory");
}

// Grid barrier over the co-resident CTAs of a cooperative launch.  `last` runs in the CTA
// that arrives last, after every other CTA's writes are visible and before anyone is released.
template <class F>
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& phase, int* s_last, F&& last) {
  fence_proxy_async_all();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(bar, 1u);
    *s_last = t == (phase + 1) * gridDim.x - 1;
  }
  __syncthreads();
  if (*s_last) {
    __threadfence();
    last();
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      st_release_u32(bar + 1, phase + 1);
    }
  } else if (threadIdx.x == 0) {
    while (ld_acquire_u32(bar + 1) < phase + 1) {
    }
  }
  __syncthreads();
  fence_proxy_async_all();
  ++phase;
}

// The landmark reduce of one warp's slot list [r0, r1) (k_lm_reduce in TERM mode: the same
// loads, additions and V+ product per landmark) with coherent loads of s, then each slot's
// consumed partials dropped from L2.  Software-pipelined over the slots -- the slot ids are
// read 32 at a time, the next slot's entry and V+ are loaded while the current slot is
// summed -- so a slot costs one dependent load latency instead of three (profiles/r2_series.md).
template <int STAGE>
__device__ PV_SER_FN void series_reduce_list(const SeriesArgs& a, int r0, int r1, int lane,
                                             uint64_t pf, uint64_t pt) {
  constexpr int NV = STAGE == 1 ? 3 : 4;
  for (int rbase = r0; rbase < r1; rbase += 32) {
    const int n = min(32, r1 - rbase);
    const int my_id = lane < n ? __ldg(a.rslot + rbase + lane) : 0;
    int w_n = __shfl_sync(PV_FULL, my_id, 0);
    int4 e_n = __ldg(a.klist + 32 * (size_t)w_n + lane);  // {landmark, first obs, k, s position}
    double4 va_n = ldg4(a.lsys + (size_t)(32 * w_n + lane) * LSYS);
    double4 vb_n = ldg4(a.lsys + (size_t)(32 * w_n + lane) * LSYS + 4);
    for (int j = 0; j < n; ++j) {
      const int w = w_n;
      const int4 e = e_n;
      LmPre pre;
      pre.va = va_n;
      pre.vb = vb_n;
      pre.bl = make_double4(0.0, 0.0, 0.0, 0.0);
      pre.x = make_double4(0.0, 0.0, 0.0, 1.0);
      if (j + 1 < n) {  // warp-uniform
        w_n = __shfl_sync(PV_FULL, my_id, j + 1);
        e_n = __ldg(a.klist + 32 * (size_t)w_n + lane);
        va_n = ldg4(a.lsys + (size_t)(32 * w_n + lane) * LSYS);
        vb_n = ldg4(a.lsys + (size_t)(32 * w_n + lane) * LSYS + 4);
      }
      const int k = e.z;  // warp-uniform
      const int kp = 32 * w + lane;
      const int s0 = __shfl_sync(PV_FULL, e.w, 0);  // lane 0's entry = the slot's base
      char* base = reinterpret_cast<char*>(a.sbuf) + 32 * (size_t)s0;
      if (k > KSHORT) {  // one long landmark: the whole warp, coalesced, fixed-order tree (lr_long)
        const int l0 = __shfl_sync(PV_FULL, e.x, 0);
        if (STAGE == 2 && lane == 0) pre.x = ldg4_h(a.lrec + (size_t)l0 * LREC);
        double a2[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) a2[i] = 0.0;
#pragma unroll 4
        for (int o = s0 + lane; o < s0 + k; o += 32) {
          const double4 sv = ld4cg(a.sbuf + 4 * (size_t)o, pf);
          a2[0] += sv.x;
          a2[1] += sv.y;
          a2[2] += sv.z;
          if (NV == 4) a2[NV - 1] += sv.w;
        }
        warp_reduce_all(a2);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < NV; ++i) acc[i] = a2[i];
        if (lane == 0)
          lm_finish<STAGE, LR_TERM, true>(l0, 32 * w, acc, pre, a.tarr, nullptr, nullptr, nullptr, pt);
        // entries [s0, s0 + k) padded to whole 128-byte lines (build_ktasks)
#ifndef PV_SER_NO_DISCARD
        for (int ln = lane; ln < (k + 3) / 4; ln += 32)
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + 128 * (size_t)ln) : "memory");
#endif
        continue;
      }
      if (e.x >= 0) {
        if (STAGE == 2) pre.x = ldg4_h(a.lrec + (size_t)e.x * LREC);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const double* sp = a.sbuf + 4 * (size_t)e.w;  // interleaved: observation i at + 32 i
#pragma unroll kLrUnroll
        for (int i = 0; i < k; ++i) {
          const double4 v = ld4cg(sp + 128 * (size_t)i, pf);
          acc[0] += v.x;
          acc[1] += v.y;
          acc[2] += v.z;
          if (STAGE == 2) acc[3] += v.w;
        }
        lm_finish<STAGE, LR_TERM, true>(e.x, kp, acc, pre, a.tarr, nullptr, nullptr, nullptr, pt);
      }
      __syncwarp();
#ifndef PV_SER_NO_DISCARD
      for (int ln = lane; ln < 8 * k; ln += 32)  // 32 k entries = 8 k lines
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + 128 * (size_t)ln) : "memory");
#endif
    }
  }
}

// epilogue of a term for one camera (k_cam EP_TERM, one warp): v = U^-1 y, x += v, norms.
// Called by the warp that finishes the camera's y in the term's last W t pass, with y in
// lanes 0-11 (u): no separate pass over the cameras, and no re-read of y.
template <int STAGE>
__device__ PV_SER_FN void series_epilogue(const SeriesArgs& a, int cam, int lane, double u) {
  constexpr int D = STAGE == 1 ? 12 : 11;
  const bool row = lane < 12;
  if (!row) u = 0.0;
  double h = 0.0;
  if (STAGE == 2) {  // project y (12) -> tangent (11)
    h = row ? a.ch[(size_t)cam * 12 + lane] : 0.0;
    const double hu = warp_sum(h * u);
    const double pr = fma(-2.0 * h, hu, u);
    u = __shfl_sync(PV_FULL, pr, (lane + 1) & 31);
    if (lane >= 11) u = 0.0;
  }
  const double vin = u;
  double t = 0.0;
  const double* Ui = a.cUi + (size_t)cam * 144 + (lane < D ? lane : 0) * 12;
  const double xold = lane < D ? a.cx[(size_t)cam * 12 + lane] : 0.0;  // in flight with U^-1
  double ui[12];  // the row of U^-1, all loads in flight before the shuffle chain
#pragma unroll
  for (int kk = 0; kk < 12; ++kk) ui[kk] = (lane < D && kk < D) ? __ldg(Ui + kk) : 0.0;
#pragma unroll
  for (int kk = 0; kk < 12; ++kk) {
    const double vk = __shfl_sync(PV_FULL, vin, kk);
    if (lane < D && kk < D) t = fma(ui[kk], vk, t);
  }
  double xr = 0.0;
  if (lane < D) {
    xr = xold + t;
    a.cx[(size_t)cam * 12 + lane] = xr;
  }
  double v = t;
  if (STAGE == 2) {  // v = B t (11 -> 12)
    const double tprev = __shfl_sync(PV_FULL, t, (lane + 31) & 31);
    const double e = (lane >= 1 && lane < 12) ? tprev : 0.0;
    const double hd = warp_sum(h * e);
    v = fma(-2.0 * h, hd, e);
  }
  // the camera records of this step's other W t items are read concurrently (TMA), but only
  // their P half is used there; the next W^T v pass reads v after the grid barrier
  if (row) a.crec[(size_t)cam * CREC + 12 + lane] = v;
  const double tn = warp_sum(lane < D ? t * t : 0.0);
  const double xn = warp_sum(lane < D ? xr * xr : 0.0);
  if (lane == 0) {
    a.nrm[2 * (size_t)cam] = tn;
    a.nrm[2 * (size_t)cam + 1] = xn;
  }
}

#ifdef PV_SER_TIMING
// diagnostic build (tools/series_times.py): globaltimer of CTA 0 after every grid barrier of
// term g_ser_term, and per warp {step start, after R, after the ring} of step g_ser_step
__device__ unsigned long long g_ser_bar[64];
__device__ unsigned long long g_ser_warp[3 * 8192];
__device__ int g_ser_term = 2, g_ser_step = 5;
#define SER_T(dst)                                                   \
  do {                                                               \
    unsigned long long t_;                                           \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));          \
    dst = t_;                                                        \
  } while (0)
#endif
template <int STAGE, bool XM>
#ifdef PV_PIPE_MAXNREG
__global__ void __maxnreg__(PV_PIPE_MAXNREG) k_series(Graph g, SeriesArgs a, Coef k, Tune tune) {
#else
__global__ void __launch_bounds__(PW * 32, PV_PIPE_MINB) k_series(Graph g, SeriesArgs a, Coef k,
                                                                  Tune tune) {
#endif
  extern __shared__ __align__(128) unsigned char pipe_dsm[];
  __shared__ int s_last;
  __shared__ double s_rr[2][8];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * PW + warp;
  const int W = a.W, B = a.B;
  uint64_t* bars = reinterpret_cast<uint64_t*>(pipe_dsm) + warp * PD;
  unsigned char* wsm = pipe_dsm + PBAR + (size_t)warp * PWARP;
  unsigned char* tbuf = wsm + PD * PSLOT;
  const uint64_t pf = pol_sel(tune.pol_stream), pt = pol_sel(tune.pol_t),
                 ps = pol_sel(tune.pol_s);
  if (lane == 0) {
    for (int s = 0; s < PD; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned phase = 0;  // grid barriers passed
  int gbase = 0;       // ring items this warp has consumed in earlier steps (slot / parity)
  auto nothing = [] {};

  for (int term = 1; term <= a.max_order; ++term) {
    for (int step = -2; step < B; ++step) {
      const int rb = step + 1, hb = step, ab = step + 2;
#ifdef PV_SER_TIMING
      const bool tme = term == g_ser_term && step == g_ser_step && lane == 0 && gw < 8192;
      if (tme) SER_T(g_ser_warp[3 * gw]);
      if (term == g_ser_term && step == -2 && threadIdx.x == 0 && blockIdx.x == 0) SER_T(g_ser_bar[0]);
#endif
      // ---- R(rb): this warp's slots of the landmark reduce
      if (rb >= 0 && rb < B) {
        const int* ro = a.roff + (size_t)rb * (W + 1) + gw;
        series_reduce_list<STAGE>(a, __ldg(ro), __ldg(ro + 1), lane, ps, pt);
      }
#ifdef PV_SER_TIMING
      if (tme) SER_T(g_ser_warp[3 * gw + 1]);
#endif
      // ---- W t (hb) then W^T v (ab) through the ring
      int h0 = 0, nh = 0, a0 = 0, na = 0;
      if (hb >= 0) {
        const int* o = a.off + (size_t)hb * (W + 1) + gw;
        h0 = __ldg(o);
        nh = __ldg(o + 1) - h0;
      }
      if (ab < B) {
        const int fam = ab >= 1 ? 3 : 1;
        const int* o = a.off + (size_t)(fam * B + ab) * (W + 1) + gw;
        a0 = __ldg(o);
        na = __ldg(o + 1) - a0;
      }
      const int first_c = hb == 0;
      const int total = nh + na;
      auto fetch = [&](int i) {
        return i < total ? __ldg(a.item + (i < nh ? h0 + i : a0 + (i - nh))) : make_int4(0, 0, 0, 0);
      };
      int base = 0;
      int4 wcur = fetch(lane), wnxt = fetch(32 + lane);
      __syncwarp();
      int n_prod = 0;
      auto produce = [&]() {
        if (n_prod >= total) return;
        if (n_prod >= base + 32) {  // warp-uniform window shift
          base += 32;
          wcur = wnxt;
          wnxt = fetch(base + 32 + lane);
        }
        const int src = n_prod - base;
        const int cam = __shfl_sync(PV_FULL, wcur.x, src), o = __shfl_sync(PV_FULL, wcur.y, src),
                  n = __shfl_sync(PV_FULL, wcur.z, src), fl = __shfl_sync(PV_FULL, wcur.w, src);
        const int s = (gbase + n_prod) % PD;
        unsigned char* slot = wsm + s * PSLOT;
        PV_CHECK(cam >= 0 && cam < g.n_p && n >= 0 && n <= PCH && o >= 0 && o + n <= g.n_o);
        if (hb == B - 1 && (fl & (PF_HA | PF_LAST)) == PF_LAST && lane < 10) {
          // this item completes a camera's y in the term's last block: its epilogue follows
          // two items later; pull U^-1 (9 lines) and x (1 line) into L2 now
          const char* pa = lane < 9 ? reinterpret_cast<const char*>(a.cUi + (size_t)cam * 144) + 128 * lane
                                    : reinterpret_cast<const char*>(a.cx + (size_t)cam * 12);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pa));
        }
        if (lane == 0) {
#if PV_PIPE_FENCE
          fence_proxy_async();
#endif
          *reinterpret_cast<int4*>(slot + PH_OFF) = make_int4(cam, o, n, fl);
          if (n > 0) {
            const int* ids = (fl & PF_HA) ? g.cs_pos : g.cs_kpos;
            const int i0 = o & ~3;
            const int i1 = (o + n + 3) & ~3;
            const unsigned bx = (unsigned)n * 32u,
                           bm = XM ? (unsigned)(((o + n + 1) & ~1) - (o & ~1)) * 8u : (unsigned)n * 16u,
                           bi = (unsigned)(i1 - i0) * 4u;
            mbar_arrive_tx(bars + s, bx + bm + bi + 192u);
            bulk_g2s(slot + PX_OFF, a.cs_x + 4 * (size_t)o, bx, bars + s, pf);
            if (XM)
              bulk_g2s(slot + PM_OFF, a.cs_m1 + (o & ~1), bm, bars + s, pf);
            else
              bulk_g2s(slot + PM_OFF, g.cs_m + 2 * (size_t)o, bm, bars + s, pf);
            bulk_g2s(slot + PI_OFF, ids + i0, bi, bars + s, pf);
            bulk_g2s(slot + PC_OFF, a.crec + (size_t)cam * CREC, 192u, bars + s, pt);
          } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bars + s))
                         : "memory");
          }
        }
        ++n_prod;
      };
      double4 Tn[(PCH + 31) / 32];  // PV_PIPE_TREG: t_j of the next W t item
      auto gather = [&](int item) {  // item: index within this step
        const unsigned char* slot = wsm + ((gbase + item) % PD) * PSLOT;
        const int4 h = *reinterpret_cast<const int4*>(slot + PH_OFF);
        if (h.w & PF_HA) return;
        const int* si = reinterpret_cast<const int*>(slot + PI_OFF) + (h.y & 3);
#if PV_PIPE_TREG
#pragma unroll
        for (int r = 0; r < (PCH + 31) / 32; ++r) {
          const int q = lane + 32 * r;
          if (q < h.z) {
            PV_CHECK(si[q] >= 0 && si[q] < g.n_kent);
            Tn[r] = ld4cg(a.tarr + 4 * (size_t)si[q], pt);
          }
        }
        return;
#endif
        unsigned char* tb = tbuf + (item & 1) * PT_BYTES;
#pragma unroll
        for (int r = 0; r < (PCH + 31) / 32; ++r) {
          const int q = lane + 32 * r;
          if (q >= h.z) continue;
          PV_CHECK(si[q] >= 0 && si[q] < g.n_kent);
          const double* src = a.tarr + 4 * (size_t)si[q];
          cp_async16wp(tb + 32 * q, src, pt);
          cp_async16wp(tb + 32 * q + 16, src + 2, pt);
        }
      };

      for (int i = 0; i < PD - 1; ++i) produce();
      __syncwarp();
      if (total > 0) {
        mbar_wait(bars + gbase % PD, (unsigned)((gbase / PD) & 1));
        gather(0);
      }
      cp_commit();

      double acc[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) acc[i] = 0.0;

      for (int c = 0; c < total; ++c) {
        produce();
#if PV_PIPE_TREG
        double4 Tc[(PCH + 31) / 32];  // this item's t_j, loaded during the previous item
#pragma unroll
        for (int r = 0; r < (PCH + 31) / 32; ++r) Tc[r] = Tn[r];
#endif
        if (c + 1 < total) {
          const int gi = gbase + c + 1;
          mbar_wait(bars + gi % PD, (unsigned)((gi / PD) & 1));
          __syncwarp();
          gather(c + 1);
        }
        cp_commit();
        cp_wait<1>();
        __syncwarp();

        const unsigned char* slot = wsm + ((gbase + c) % PD) * PSLOT;
        const int4 h = *reinterpret_cast<const int4*>(slot + PH_OFF);
        const int cam = h.x, o0 = h.y, n = h.z, fl = h.w;
        const double4* cr = reinterpret_cast<const double4*>(slot + PC_OFF);
        const double4* sx = reinterpret_cast<const double4*>(slot + PX_OFF);
        const double2* sm = reinterpret_cast<const double2*>(slot + PM_OFF);
        const double* sm1 = reinterpret_cast<const double*>(slot + PM_OFF) + (o0 & 1);
        auto xm_at = [&](int q, double4& X, double2& m) {
          X = sx[q];
          if (XM) {
            m = make_double2(X.w, sm1[q]);
            X.w = 1.0;
          } else {
            m = sm[q];
          }
        };
        if (!(fl & PF_HA)) {
          if (n > 0) {
            const double4 P0 = cr[0], P1 = cr[1], P2v = cr[2];
            const double4* tq = reinterpret_cast<const double4*>(tbuf + (c & 1) * PT_BYTES);
#pragma unroll
            for (int r = 0; r < (PCH + 31) / 32; ++r) {
              const int q = lane + 32 * r;
              if (q >= n) continue;
              double4 X;
              double2 m;
              xm_at(q, X, m);
              #if PV_PIPE_TREG
            const double4 T = Tc[r];
#else
            const double4 T = tq[q];
#endif
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
            double yv = 0.0;
            if (lane < 12) {
              double* yp = a.cy + (size_t)cam * 12 + lane;
              yv = first_c ? mine : __ldcg(yp) + mine;
              *yp = yv;
            }
            if (hb == B - 1) series_epilogue<STAGE>(a, cam, lane, yv);  // y is complete
#pragma unroll
            for (int i = 0; i < 12; ++i) acc[i] = 0.0;
          }
        } else {
          const double4 P0 = cr[0], P1 = cr[1], P2v = cr[2];
          const double4 v0 = cr[3], v1 = cr[4], v2 = cr[5];
          const int* si = reinterpret_cast<const int*>(slot + PI_OFF) + (o0 & 3);
#pragma unroll
          for (int r = 0; r < (PCH + 31) / 32; ++r) {
            const int q = lane + 32 * r;
            if (q >= n) continue;
            double4 X;
            double2 m;
            xm_at(q, X, m);
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
            st4p(a.sbuf + 4 * (size_t)pos, sv, ps);
          }
        }
        __syncwarp();
      }
      cp_wait<0>();
      gbase += total;
#ifdef PV_SER_TIMING
      if (tme) SER_T(g_ser_warp[3 * gw + 2]);
#endif
      // the last step's barrier also carries the stop decision: the LAST CTA to arrive sums the
      // norms (k_cam's order: 256 strided partial sums, a butterfly per 32, then 8 in order)
      // and decides (solvers.py:140-149) before it releases the others
      if (step < B - 1) {
        grid_sync(a.bar, phase, &s_last, nothing);
      } else {
        grid_sync(a.bar, phase, &s_last, [&] {
          // 256 strided chains (virtual thread vt sums cameras vt, vt + 256, ... in order); a warp
          // walks its up to three virtual warps together, eight loads of each in flight
          {
            constexpr int NVW = (8 + PW - 1) / PW;
            double ra[NVW][2];
#pragma unroll
            for (int q = 0; q < NVW; ++q) ra[q][0] = ra[q][1] = 0.0;
            const double2* nr = reinterpret_cast<const double2*>(a.nrm);
            for (int i0 = 0; i0 < g.n_p; i0 += 8 * 256) {
              double2 v[NVW][8];
#pragma unroll
              for (int q = 0; q < NVW; ++q) {
                const int vw = warp + q * PW;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  const int i = i0 + u * 256 + vw * 32 + lane;
                  v[q][u] = (vw < 8 && i < g.n_p) ? __ldcg(nr + i) : make_double2(0.0, 0.0);
                }
              }
#pragma unroll
              for (int q = 0; q < NVW; ++q) {
                const int vw = warp + q * PW;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  const int i = i0 + u * 256 + vw * 32 + lane;
                  if (vw < 8 && i < g.n_p) {  // added in camera order; skipped terms add nothing
                    ra[q][0] += v[q][u].x;
                    ra[q][1] += v[q][u].y;
                  }
                }
              }
            }
#pragma unroll
            for (int q = 0; q < NVW; ++q) {
              const int vw = warp + q * PW;
              if (vw < 8) {  // warp-uniform
                double r2[2] = {ra[q][0], ra[q][1]};
                warp_reduce_all(r2);
                if (lane == 0) {
                  s_rr[0][vw] = r2[0];
                  s_rr[1][vw] = r2[1];
                }
              }
            }
          }
          __syncthreads();
          if (threadIdx.x == 0) {
            double TN2 = 0.0, XN2 = 0.0;
            for (int q = 0; q < 8; ++q) {
              TN2 += s_rr[0][q];
              XN2 += s_rr[1][q];
            }
            const double TN = sqrt(TN2), XN = sqrt(XN2);
            PowerCtl c = *a.ctl;
            const double ratio = XN > 0.0 ? TN / XN : 0.0;
            c.trunc = ratio;
            c.term = term;
            if (ratio <= a.thr) {
              c.order = term - 1;
              c.stopped = 1;
            } else {
              c.order = term;
            }
            c.xnorm = XN;
            c.tnorm = TN;
            *a.ctl = c;  // the host reads it after the launch (no mapped mirror: nobody polls)
          }
        });
      }
#ifdef PV_SER_TIMING
      if (term == g_ser_term && threadIdx.x == 0 && blockIdx.x == 0) SER_T(g_ser_bar[step + 3]);
#endif
    }
#ifdef PV_SER_TIMING
    if (term == g_ser_term && threadIdx.x == 0 && blockIdx.x == 0) SER_T(g_ser_bar[B + 3]);
#endif
    if (__ldcg(&a.ctl->stopped)) break;
  }
}

}  // namespace pv
