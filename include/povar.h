/* C-ABI of the B200-native PoVar / RiPoBA hot path (libpovar.so).
 *
 * The reference (/root/reference/pkg/src/stratba) is a pure-Python package with
 * no FFI; its plug points on this path are Python functions.  Each entry point
 * below names the reference interface whose work it takes over (file:line,
 * relative to pkg/src/stratba).  Python binds them with ctypes
 * (paper_2405_05079_b200/_lib.py); INTEGRATION.md shows the stub a stratba
 * maintainer would add.
 *
 * Conventions
 *  - All arithmetic is fp64.  Cameras are (n_p, 3, 4) row-major (12 per camera,
 *    objective.py:16); landmarks are (n_l, 4) homogeneous.
 *  - Host arrays are borrowed for the duration of a call and copied; device
 *    memory, the CUDA stream and the NCCL communicator belong to the context.
 *  - Calls on one context must be serialized by the caller; distinct contexts
 *    are independent (the reference allows concurrent lm_minimize calls on
 *    distinct problems).
 *  - A context owns the landmark shard [lm_begin, lm_end) of one rank; with
 *    world > 1 every entry point is collective over the world (NCCL), camera
 *    quantities are replicated and every rank returns identical scalars.
 *  - Return value: PV_OK or one of the status codes; pv_last_error() gives text.
 */
#ifndef POVAR_H_
#define POVAR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pv_ctx pv_ctx;

enum {
  PV_OK = 0,
  PV_EINVAL = 1,       /* -> ValueError            (solvers.py:82-93, normal_eq.py:163-166) */
  PV_ECUDA = 2,        /* -> RuntimeError                                                   */
  PV_ENCCL = 3,        /* -> RuntimeError                                                   */
  PV_ENONFINITE = 4,   /* -> NumericFailureError   (solvers.py:336-338)                     */
  PV_EDEGENERATE = 5,  /* -> FloatingPointError    (normal_eq.py:86-87)                     */
  PV_ESINGULAR = 6     /* -> numpy.linalg.LinAlgError (np.linalg.inv of a singular pose
                          block, solvers.py:108-109)                                       */
};

enum { PV_CURRENT = 0, PV_TRIAL = 1 };

/* debug buffers for pv_debug_get (per-kernel parity); sizes in doubles */
enum {
  PV_DBG_U = 0,        /* damped U blocks, n_p x 144 (12x12; 11x11 top-left in stage 2)  */
  PV_DBG_UINV = 1,     /* U^-1, n_p x 144                                               */
  PV_DBG_BP = 2,       /* b_p, n_p x 12                                                  */
  PV_DBG_V = 3,        /* undamped (projected) V, n_ls x 6 (xx xy xz yy yz zz)           */
  PV_DBG_VPINV = 4,    /* V+ of the damped V, n_ls x 6                                   */
  PV_DBG_BL = 5,       /* b_l, n_ls x 3                                                  */
  PV_DBG_DEGEN = 6,    /* degenerate flag, n_ls                                          */
  PV_DBG_W = 7,        /* W per landmark-sorted observation, n_obs_local x 36 (12x3/11x3) */
  PV_DBG_RHS = 8,      /* reduced RHS, n_p x 12                                          */
  PV_DBG_X = 9,        /* power-series pose update, n_p x 12                             */
  PV_DBG_DL = 10,      /* landmark update, n_ls x 3                                      */
  PV_DBG_ULIN = 11,    /* undamped (projected) U, n_p x 144                              */
  PV_DBG_SDIAG = 12,   /* exact Schur block diagonal of the last pv_pcg_solve, n_p x 144 */
  PV_DBG_MINV = 13     /* its inverse (the block-Jacobi preconditioner), n_p x 144       */
};

/* info fields for pv_info */
enum {
  PV_INFO_NP = 0, PV_INFO_NL_LOCAL = 1, PV_INFO_NO_LOCAL = 2, PV_INFO_TASKS = 3,
  PV_INFO_CHUNKS = 4, PV_INFO_LAUNCHES = 5, PV_INFO_RANK = 6, PV_INFO_WORLD = 7,
  PV_INFO_DEVICE_BYTES = 8, PV_INFO_NL_GLOBAL = 9, PV_INFO_RESOLVE_FALLBACKS = 10,
  PV_INFO_BLOCKS = 11, PV_INFO_PERSIST_L2 = 12, PV_INFO_WARPS_PER_CAM = 13,
  /* last pv_power_solve, device microseconds (CUDA events): reduced RHS + t_0, the term
   * loop, the back-substitution; terms launched (incl. the look-ahead one) */
  PV_INFO_SOLVE_RHS_US = 14, PV_INFO_SOLVE_TERMS_US = 15, PV_INFO_SOLVE_BACKSUB_US = 16,
  PV_INFO_SOLVE_TERMS_LAUNCHED = 17,
  /* bytes of x and m streamed per observation by a stage-1 camera pass (48, or 40 with the
   * compact stream of PV_OPT_XM) */
  PV_INFO_XM_BYTES = 18,
  /* warps of the persistent camera kernel (resident CTAs per SM x SMs x warps per CTA) */
  PV_INFO_PIPE_WARPS = 19,
  PV_INFO_COUNT = 24
};

/* tuning knobs of the term kernels (pv_set_option); results do not depend on them */
enum {
  PV_OPT_STAGE_CAP = 0,   /* observations per camera staged in shared memory (0..2048)     */
  PV_OPT_POL_STREAM = 1,  /* L2 priority of camera-sorted streams: 0 normal 1 first 2 last */
  PV_OPT_POL_T = 2,       /* L2 priority of the gathered landmark vectors t              */
  PV_OPT_POL_S = 3,       /* L2 priority of the per-observation partials s               */
  PV_OPT_DISCARD_S = 4,   /* 1: drop consumed partials from L2 without write-back          */
  PV_OPT_BLOCK_BYTES = 5, /* L2 budget of one landmark block's partials (re-blocks)        */
  PV_OPT_FORCE_COLLECTIVE = 6, /* world == 1: run the sharded code path (split kernels +
                                  ncclAllReduce) over a 1-rank communicator (testing)       */
  /* 7: reserved (a removed camera-kernel variant; rejected as an unknown option)          */
  PV_OPT_CAM_PIPE = 8,         /* 1: single-block camera passes run the persistent kernel
                                  with a TMA-fed shared-memory ring (pv_pipe.cuh)          */
  PV_OPT_RESOLVE_SLOTS = 9,    /* 1: landmark re-solve and landmark-side linearization with
                                  one lane per landmark (k-bucketed warp slots); 0: warp per
                                  landmark task                                            */
  PV_OPT_SPLIT_LAST = 10,      /* 1: a term's last block runs its W t pass on the pipelined
                                  kernel and the epilogue + next W^T v pass separately     */
  PV_OPT_RHS_REUSE = 11,       /* 1: a solve after a rejected stage-1 step (same linearization,
                                  POSE_ONLY) reuses the reduced RHS -(b_p - W V+ b_l)      */
  PV_OPT_COST_CS = 12,         /* 1: pv_cost walks the camera-sorted segments (one camera load
                                  per warp segment); 0: landmark-task order                */
  PV_OPT_BENCH_SPLIT = 13,     /* diagnostic: pv_bench_terms times the W^T v passes (ms[0]) and
                                  the W t passes (ms[1]) of all blocks on their own         */
  PV_OPT_XM = 14,              /* 1 (default): stage-1 pipelined camera passes stream x and m as
                                  (x0 x1 x2 m0 | m1), 40 instead of 48 bytes per observation,
                                  when every landmark has w = 1                             */
  PV_OPT_GRAPH = 15,           /* 1 (default): the power-series term loop runs as one CUDA graph
                                  (WHILE conditional node, stop test on the device); 0: host
                                  loop with a one-term look-ahead                            */
  PV_OPT_BALANCE = 16,         /* work lists of the persistent camera kernel: 1 (default) whole
                                  cameras packed longest-first (W t) and item-granular cuts
                                  (W^T v); 0 contiguous equal-cost camera ranges              */
  PV_OPT_BAL_ITEM = 17,        /* cost model of that balance, in observation-equivalents: fixed */
  PV_OPT_BAL_ROUND = 18,       /* cost of an item, of each 32-observation round, and of a        */
  PV_OPT_BAL_LAST = 19,        /* camera's last W t item (its warp reduction)                    */
  PV_OPT_BAL_RFIX = 20,        /* ... and of a landmark-reduce slot of the series kernel: fixed  */
  PV_OPT_BAL_ROBS8 = 21,       /* + (partials * value) / 8                                       */
  PV_OPT_SERIES = 22,          /* 1: the whole power series (every term's landmark reduces, camera
                                  passes, U^-1 epilogue and stop test) runs as ONE persistent
                                  cooperative kernel with grid barriers (pv_series.cuh), bit-
                                  identical to 0 (default): one launch per landmark block and
                                  pass inside the term graph.  Measured 4% slower per LM
                                  iteration at vlarge (profiles/r2_series.md), so opt-in        */
  PV_OPT_KSLOT = 23            /* 1 (default): the stage-1 landmark reduce of a term reads one
                                  16-byte record per warp slot (L2-resident) instead of the
                                  512-byte per-lane entries (results unchanged)                 */
};

/* NCCL unique id (128 bytes) for a multi-rank world; rank 0 creates it and the
 * host broadcasts it (torch.distributed store) before pv_create. */
int pv_nccl_unique_id(unsigned char out[128]);

/* In-process loopback "communicator" for testing the sharded path on ONE device: returns an
 * id to pass as nccl_id to pv_create for each of `world` contexts (ranks) of this process on
 * the same device, each driven by its own host thread.  Allreduces become rank-ordered
 * device sums between host barriers (bit-identical replicas, as with NCCL). */
int pv_loopback_id(int world, unsigned char out[128]);

/* Upload the observation graph once: landmark-CSR order, camera-sorted
 * permutation, warp work units; replaces the per-iteration landmark_order +
 * _group_blocks bucketing (objective.py:237-248, normal_eq.py:92-106).
 * cam_idx/lm_idx/meas describe the WHOLE problem (BaProblem, bal_io.py:53-92);
 * the context keeps the observations of landmarks in [lm_begin, lm_end).
 * nccl_id may be NULL when world == 1. */
int pv_create(pv_ctx** out, int device, int rank, int world, const unsigned char* nccl_id,
              int64_t n_cameras, int64_t n_landmarks, int64_t n_obs, const int64_t* cam_idx,
              const int64_t* lm_idx, const double* meas, int64_t lm_begin, int64_t lm_end,
              double eta);
void pv_destroy(pv_ctx* ctx);
const char* pv_last_error(pv_ctx* ctx); /* ctx may be NULL (thread-local create error) */
int pv_info(pv_ctx* ctx, int64_t* out /* PV_INFO_COUNT */);
int pv_set_option(pv_ctx* ctx, int key, int64_t value);
/* cudaStream_t of the context, for event timing by the caller */
void* pv_stream(pv_ctx* ctx);

/* ProjectiveState in/out (bal_io.py:95-112).  lms is the full (n_l, 4) array;
 * pv_get_state writes only this shard's observed landmarks. */
int pv_set_state(pv_ctx* ctx, const double* cams, const double* lms);
int pv_get_state(pv_ctx* ctx, double* cams, double* lms);
int pv_get_trial(pv_ctx* ctx, double* cams, double* lms);

/* total_cost (objective.py:194-211); +inf for a degenerate stage-2 state */
int pv_cost(pv_ctx* ctx, int stage, int which, double* f);

/* build_stage{1,2}_blocks + project_blocks + the undamped half of assemble
 * (normal_eq.py:62-89,156-180; riemannian.py:67-85).  Stage 2 returns
 * PV_EDEGENERATE on |z| <= 1e-12. */
int pv_linearize(pv_ctx* ctx, int stage);

/* damping + U^-1 + V^+ (normal_eq.py:182-198, solvers.py:108-109);
 * both = 1 for BOTH mode (joint stage 1, stage 2). */
int pv_damp(pv_ctx* ctx, double lam, int both, int64_t* n_degenerate);

/* power_schur_solve (solvers.py:126-150) incl. schur_rhs and back_substitute
 * (normal_eq.py:221-250); leaves the pose update, landmark update and trial
 * landmarks on the device. */
int pv_power_solve(pv_ctx* ctx, int max_order, double threshold, int* order_used,
                   double* truncation);

/* pcg_schur_solve (solvers.py:153-187): block-Jacobi preconditioned CG on the
 * reduced system, preconditioner = inverse of the exact block diagonal
 * (schur_diag_blocks, normal_eq.py:253-260; np.linalg.inv with the
 * _pinv_psd(., 1e-12) fallback).  Stops at relative residual <= tolerance or
 * after max_iterations; *flag = 1 on non-positive curvature ("breakdown").
 * Leaves the same device results as pv_power_solve (pv_get_step, pv_trial). */
int pv_pcg_solve(pv_ctx* ctx, int max_iterations, double tolerance, int* iterations,
                 double* relative_residual, int* flag);

/* trial state (solvers.py:311-315 / riemannian.py:110-122); *ok = 0 when a
 * stage-2 norm collapses (apply_tangent_step returns None). */
int pv_trial(pv_ctx* ctx, int stage, int* ok);

/* accept the trial; resolve = 1 runs solve_landmarks on it (objective.py:251-298)
 * and returns the stage-1 cost of the re-solved state in *f_new. */
int pv_accept(pv_ctx* ctx, int stage, int resolve, double* f_new, int64_t* n_rank_deficient);

/* closed-form landmarks for the CURRENT cameras with current landmarks as the
 * fallback (solve_landmarks on the current state); result kept as current. */
int pv_resolve_current(pv_ctx* ctx, int64_t* n_rank_deficient);

/* back_substitute (normal_eq.py:239-250) of a given pose update dx (n_p*d, d = 12 stage 1,
 * 11 stage 2) on the current damped system: dl = -V+ (b_l + W^T dx), zero for degenerate
 * landmark blocks.  Replaces the device step (pv_get_step, pv_trial use it afterwards). */
int pv_back_substitute(pv_ctx* ctx, const double* dx);

/* StepReport arrays of the last pv_power_solve / pv_pcg_solve: dx (n_p*d), dl (n_l*dl) for the
 * whole problem (unobserved / foreign-shard landmarks left untouched). */
int pv_get_step(pv_ctx* ctx, double* dx, double* dl);

/* S'.v = W V^+ W^T v (_coupling_round_trip, solvers.py:117-123) on host vectors
 * of length n_p*d (d = 12 stage 1, 11 stage 2) for the current linearization. */
int pv_schur_apply(pv_ctx* ctx, int stage, const double* v, double* out);

/* Timed power-series terms (no stop test), for the bench: runs n_terms terms on the
 * context stream twice each -- once with CUDA events around every launch group, once
 * back to back -- and returns per term: ms[0] the landmark reduces (all blocks), ms[1]
 * the camera passes (all blocks, incl. the epilogue), ms[2] the block count, ms[3] the
 * whole term (event to event, no events inside). */
int pv_bench_terms(pv_ctx* ctx, int stage, int n_terms, float* ms);

int pv_debug_get(pv_ctx* ctx, int which, double* out);

#ifdef __cplusplus
}
#endif
#endif /* POVAR_H_ */
