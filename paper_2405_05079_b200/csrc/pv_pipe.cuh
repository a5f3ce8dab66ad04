// Persistent, software-pipelined camera kernel of the L2-blocked power-series term
// (the EP_NONE form of k_cam: y_i (+)= sum_{j in block bc} W_ij t_j, then
// s_ij = W_ij^T v_i for j in block ba).
//
// Why: in k_cam every warp owns one (camera, block) segment of ~176 observations,
// i.e. 2-3 staged chunks per phase, so its cp.async double buffer never reaches a
// steady state: ncu (profiles/r1_history.md, "Round 1, second session") attributes
// ~60% of the stall samples to the dependent t gathers, the stream waits at the start
// of each segment and the segment-offset loads.  Here each warp walks a long work list
// (the W t chunks of its cameras in block bc, then the W^T v chunks of its cameras
// in block ba) through a D-deep ring of shared-memory slots:
//
//   * streams (x, m, ids of a chunk + the 192-byte camera record) are fetched by
//     TMA bulk copies (cp.async.bulk, one elected lane, mbarrier completion)
//     D-1 chunks ahead, across camera and phase boundaries;
//   * the t_j of chunk c+1 (L2) are loaded before chunk c is computed, by one 256-bit load
//     per observation straight into registers (PV_PIPE_TREG; round 1: two 16-byte cp.async
//     per observation into a shared-memory double buffer);
//   * the work list itself (item descriptors, built on the host) is read 32 items
//     at a time, one window ahead.
//
// Deterministic (fixed per-lane accumulation order + fixed warp reduction); with one
// warp per camera in k_cam (wpc = 1, the large configs) the two kernels agree bit for bit.
#pragma once
#include "pv_kernels.cuh"

namespace pv {

#ifndef PV_PIPE_CH
#define PV_PIPE_CH 64
#endif
#ifndef PV_PIPE_D
#define PV_PIPE_D 3
#endif
// Shape.  Round 1 (t gathered through shared memory): 3 warps x 5 CTAs per SM (15 resident
// warps, 120 registers) 18.24 ms per LM iteration; 2 x 8 18.29; ring depth 2 19.06; depth 4
// (12 warps) 18.57.  Round 2, with t in registers (PV_PIPE_TREG) the ring is 10.4 KB per warp
// and the registers (120-124) are the only limit: term 1.051 ms (shared-memory t, 3 x 5) ->
// 1.022 (3 x 5) -> 1.010 (4 x 4) / 1.012 (2 x 8) -> 0.980 ms with ONE warp per CTA (17 resident
// CTAs per SM); register caps of 112 / 104 / 96 (18-21 warps) spill into the item loop and
// lose (1.13 / 1.36 / 1.48 ms); depth 4 no gain (profiles/r2_series.md section 6).
#ifndef PV_PIPE_W
#define PV_PIPE_W 1
#endif
#ifndef PV_PIPE_MINB
#define PV_PIPE_MINB 16
#endif
// The slot refilled at iteration c was consumed at iteration c-1, whose shared-memory
// reads all fed instructions that have retired (and a __syncwarp) before the TMA is
// issued, so no proxy fence is needed in practice; PV_PIPE_FENCE=1 adds it anyway.
#ifndef PV_PIPE_FENCE
#define PV_PIPE_FENCE 0
#endif

constexpr int PCH = PV_PIPE_CH;  // observations per chunk
constexpr int PD = PV_PIPE_D;    // ring depth (slots per warp)
constexpr int PW = PV_PIPE_W;    // warps per CTA
constexpr int PX_OFF = 0;
constexpr int PM_OFF = PCH * 32;
constexpr int PI_OFF = PCH * 48;
constexpr int PI_BYTES = (PCH + 4) * 4;
constexpr int PC_OFF = PI_OFF + PI_BYTES;  // camera record: P (12) | v (12)
constexpr int PH_OFF = PC_OFF + 192;       // header {cam, o, n, flags}
constexpr int PSLOT = ((PH_OFF + 16 + 31) / 32) * 32;
// PV_PIPE_TREG = 1: the t_j of the next W t item are loaded straight into registers by 256-bit
// loads (one L1TEX request per observation) instead of two 16-byte cp.async per observation
// into a shared-memory double buffer; the 4 KB per warp this frees can hold a deeper ring.
#ifndef PV_PIPE_TREG
#define PV_PIPE_TREG 1
#endif
constexpr int PT_BYTES = PV_PIPE_TREG ? 0 : PCH * 32;  // gathered t of one chunk
constexpr int PWARP = PD * PSLOT + 2 * PT_BYTES;
constexpr int PBAR = ((PW * PD * 8 + 127) / 128) * 128;
constexpr int PIPE_SMEM = PBAR + PW * PWARP;

enum { PF_HA = 1, PF_LAST = 2 };

#ifdef PV_PIPE_TIMING
// diagnostic build (tools/pipe_times.py): per warp of the fused launch of block g_pipe_dbg_block,
// {globaltimer at entry, after the last W^T v / W t item, SM id}
__device__ unsigned long long g_pipe_t[3 * 8192];
__device__ int g_pipe_dbg_block = 5;
__device__ __forceinline__ unsigned long long pipe_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Work lists (built on the host by build_blocks, pv_build_pipe_items): per landmark
// block b and list L (0: W t items over block b with landmark ids, 1: W^T v items
// with landmark-sorted positions), each warp of the persistent grid owns a
// contiguous camera range balanced by observation count; an item is {camera,
// first observation, count <= PCH, flags}.  Every camera has >= 1 item in list 0
// (so y is always written); PF_LAST marks its last one.
struct PipeItems {
  const int4* item;
  const int* off;  // [(L * B + b) * (W + 1) + w]: first item of warp w; L = 0 W t, 1 W^T v on
                   // its own, 2 W^T v of block b launched with the W t items of block b - 1
  int B, W;
};

// XM (stage 1, every landmark w = 1): cs_x is the compact stream xm = (x0, x1, x2, m0) and
// cs_m1 holds m1 -- 40 instead of 48 bytes of x and m per observation (k_build_csx); x.w = 1
// and m are rebuilt in registers, so both layouts give the same bits.
template <int STAGE, bool HC, bool HA, bool XM>
#ifdef PV_PIPE_MAXNREG
__global__ void __maxnreg__(PV_PIPE_MAXNREG) k_cam_pipe(Graph g, PipeItems it,
#else
__global__ void __launch_bounds__(PW * 32, PV_PIPE_MINB) k_cam_pipe(Graph g, PipeItems it,
#endif
                                                      const double* __restrict__ crec,
                                                      const double* __restrict__ cs_x,
                                                      const double* __restrict__ cs_m1,
                                                      const double* __restrict__ tarr,
                                                      double* __restrict__ sbuf,
                                                      double* __restrict__ cy,
                                                      const PowerCtl* __restrict__ ctl, Coef k,
                                                      Tune tune, int bc, int first_c, int ba,
                                                      int check_stop, int disc_lo, int disc_hi) {
  extern __shared__ __align__(128) unsigned char pipe_dsm[];
  if (check_stop && ctl->stopped) return;  // grid-uniform
#ifdef PV_PIPE_TIMING
  const unsigned long long t_entry = pipe_gtimer();
#endif
  discard_s_lines(sbuf, disc_lo, disc_hi);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * PW + warp;
  uint64_t* bars = reinterpret_cast<uint64_t*>(pipe_dsm) + warp * PD;
  unsigned char* wsm = pipe_dsm + PBAR + (size_t)warp * PWARP;
  unsigned char* tbuf = wsm + PD * PSLOT;
  const uint64_t pf = pol_sel(tune.pol_stream), pt = pol_sel(tune.pol_t),
                 ps = pol_sel(tune.pol_s);
  if (lane == 0) {
    for (int s = 0; s < PD; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  int h0 = 0, nh = 0, a0 = 0, na = 0;
  if (HC) {
    const int* o = it.off + (size_t)bc * (it.W + 1) + gw;
    h0 = __ldg(o);
    nh = __ldg(o + 1) - h0;
  }
  if (HA) {  // family 2 when this launch also runs the W t items of block ba - 1
    const int* o = it.off + (size_t)((HC ? 2 : 1) * it.B + ba) * (it.W + 1) + gw;
    a0 = __ldg(o);
    na = __ldg(o + 1) - a0;
  }
  const int total = nh + na;
  // descriptor windows: lane l holds item base + l (current) and base + 32 + l (next)
  auto fetch = [&](int i) {
    return i < total ? __ldg(it.item + (i < nh ? h0 + i : a0 + (i - nh))) : make_int4(0, 0, 0, 0);
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
    const int s = n_prod % PD;
    unsigned char* slot = wsm + s * PSLOT;
    PV_CHECK(cam >= 0 && cam < g.n_p && n >= 0 && n <= PCH && o >= 0 && o + n <= g.n_o);
    PV_CHECK(((o + n + 3) & ~3) - (o & ~3) <= PCH + 4);
    if (lane == 0) {
#if PV_PIPE_FENCE
      fence_proxy_async();  // the warp's generic reads of this slot precede the refill
#endif
      *reinterpret_cast<int4*>(slot + PH_OFF) = make_int4(cam, o, n, fl);
      if (n > 0) {
        const int* ids = (fl & PF_HA) ? g.cs_pos : g.cs_kpos;
        const int i0 = o & ~3;
        const int i1 = (o + n + 3) & ~3;
        // XM: m1 copied from the 16-byte aligned o & ~1 (one extra leading double)
        const unsigned bx = (unsigned)n * 32u,
                       bm = XM ? (unsigned)(((o + n + 1) & ~1) - (o & ~1)) * 8u : (unsigned)n * 16u,
                       bi = (unsigned)(i1 - i0) * 4u;
        mbar_arrive_tx(bars + s, bx + bm + bi + 192u);
        bulk_g2s(slot + PX_OFF, cs_x + 4 * (size_t)o, bx, bars + s, pf);
        if (XM)
          bulk_g2s(slot + PM_OFF, cs_m1 + (o & ~1), bm, bars + s, pf);
        else
          bulk_g2s(slot + PM_OFF, g.cs_m + 2 * (size_t)o, bm, bars + s, pf);
        bulk_g2s(slot + PI_OFF, ids + i0, bi, bars + s, pf);
        bulk_g2s(slot + PC_OFF, crec + (size_t)cam * CREC, 192u, bars + s, pt);
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bars + s))
                     : "memory");
      }
    }
    ++n_prod;
  };
  // t_j of every observation of a W t item (its ids have landed)
  double4 Tn[(PCH + 31) / 32];  // PV_PIPE_TREG: t_j of the next W t item
  auto gather = [&](int item) {
    const unsigned char* slot = wsm + (item % PD) * PSLOT;
    const int4 h = *reinterpret_cast<const int4*>(slot + PH_OFF);
    if (h.w & PF_HA) return;
    const int* si = reinterpret_cast<const int*>(slot + PI_OFF) + (h.y & 3);
#if PV_PIPE_TREG
#pragma unroll
    for (int r = 0; r < (PCH + 31) / 32; ++r) {
      const int q = lane + 32 * r;
      if (q < h.z) {
        PV_CHECK(si[q] >= 0 && si[q] < g.n_kent);
        Tn[r] = ld4cg(tarr + 4 * (size_t)si[q], pt);
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
      const double* src = tarr + 4 * (size_t)si[q];
      cp_async16wp(tb + 32 * q, src, pt);
      cp_async16wp(tb + 32 * q + 16, src + 2, pt);
    }
  };

  for (int i = 0; i < PD - 1; ++i) produce();
  __syncwarp();
  if (total > 0) {
    mbar_wait(bars + 0, 0);
    gather(0);
  }
  cp_commit();

  double acc[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) acc[i] = 0.0;

  for (int c = 0; c < total; ++c) {
    produce();  // refills the slot consumed in the previous iteration
#if PV_PIPE_TREG
    double4 Tc[(PCH + 31) / 32];  // this item's t_j, loaded during the previous item
#pragma unroll
    for (int r = 0; r < (PCH + 31) / 32; ++r) Tc[r] = Tn[r];
#endif
    if (c + 1 < total) {  // t gathers of the next item, in flight while this one computes
      mbar_wait(bars + (c + 1) % PD, (unsigned)(((c + 1) / PD) & 1));
      __syncwarp();
      gather(c + 1);
    }
    cp_commit();
    cp_wait<1>();
    __syncwarp();

    const unsigned char* slot = wsm + (c % PD) * PSLOT;
    const int4 h = *reinterpret_cast<const int4*>(slot + PH_OFF);
    const int cam = h.x, o0 = h.y, n = h.z, fl = h.w;
    const double4* cr = reinterpret_cast<const double4*>(slot + PC_OFF);
    const double4* sx = reinterpret_cast<const double4*>(slot + PX_OFF);
    const double2* sm = reinterpret_cast<const double2*>(slot + PM_OFF);
    const double* sm1 = reinterpret_cast<const double*>(slot + PM_OFF) + (o0 & 1);
    // observation q's x (w = 1 rebuilt under XM) and m
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
      if (HC) {
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
        st4p(sbuf + 4 * (size_t)pos, sv, ps);
      }
    }
    __syncwarp();
  }
  cp_wait<0>();
#ifdef PV_PIPE_TIMING
  if (HC && HA && bc == g_pipe_dbg_block && lane == 0 && gw < 8192) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_pipe_t[3 * gw] = t_entry;
    g_pipe_t[3 * gw + 1] = pipe_gtimer();
    g_pipe_t[3 * gw + 2] = smid;
  }
#endif
}

}  // namespace pv
