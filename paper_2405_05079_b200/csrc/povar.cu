// libpovar.so: device-resident context + C-ABI (include/povar.h).
//
// Host side of the B200 PoVar hot path: builds the landmark-CSR / camera-chunk
// work decomposition once per problem, owns the device buffers, the CUDA
// stream and (world > 1) the NCCL communicator, and sequences the kernels of
// pv_kernels.cuh.  The LM state machine itself stays in Python
// (paper_2405_05079_b200/solver.py, mirroring solvers.py:318-393).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <numeric>
#include <queue>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/povar.h"
#include "pv_kernels.cuh"
#include "pv_pcg.cuh"
#include "pv_pipe.cuh"
#include "pv_series.cuh"

using namespace pv;

namespace {

thread_local std::string g_create_error;

struct PvError : std::runtime_error {
  int code;
  PvError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw PvError(PV_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));            \
  } while (0)

#define NK(x)                                                                              \
  do {                                                                                     \
    ncclResult_t r_ = (x);                                                                 \
    if (r_ != ncclSuccess)                                                                 \
      throw PvError(PV_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_));            \
  } while (0)

inline int blocks_for(long long n, int per) { return (int)std::max(1LL, (n + per - 1) / per); }
const double* const g_null_d = nullptr;

// In-process loopback communicator: W contexts of one process on one device, one host
// thread per rank, standing in for NCCL so the sharded code path (split camera kernels,
// replicated epilogue, collective flags) runs and is tested on a single GPU.  An allreduce
// is two host barriers around device work: every rank records "my buffer is ready", then
// sums ALL ranks' buffers in rank order into a scratch buffer (same-device reads ordered by
// cudaStreamWaitEvent), records "read done", and after the second barrier copies the sum
// back once every rank has read its buffer.  Every rank adds the same values in the same
// order, so the replicas are bit-identical, as with NCCL.
struct LoopGroup {
  static constexpr uint64_t MAGIC = 0x4b4250504f4f4c50ull;  // "PLOOPPBK"
  int world = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const void*> bufs;
  std::vector<cudaEvent_t> ready, done;
  int members = 0;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

__global__ void k_loop_sum(int world, const double* const* bufs, size_t n, double* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    double s = bufs[0][i];
    for (int q = 1; q < world; ++q) s += bufs[q][i];
    out[i] = s;
  }
}
__global__ void k_loop_max(int world, const int* const* bufs, int n, int* out) {
  const int i = threadIdx.x;
  if (i >= n) return;
  int s = bufs[0][i];
  for (int q = 1; q < world; ++q) s = max(s, bufs[q][i]);
  out[i] = s;
}

}  // namespace

// a captured term loop (term_graph) and the configuration it was captured for
struct TermGraph {
  int stage = 0, max_order = 0, n_blk = 0, wpc = 0, xm = 0, layout_gen = -1;
  double thr = 0.0;
  Tune tune{};
  bool coll = false;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  long long body_launches = 0;
};

struct pv_ctx {
  int device = 0, rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> bev;  // per-launch timing events of pv_bench_terms
  std::string err;
  long long launches = 0;
  size_t device_bytes = 0;
  std::vector<void*> allocs;

  int64_t n_p = 0, n_l_global = 0, n_o_global = 0;
  int n_ls = 0, n_os = 0, n_tasks = 0;
  size_t cpart_cap = 0;  // warp partials held by cpart (level-2 sums live after them)
  std::vector<int64_t> lm_gid;  // local -> global landmark id
  Coef coef{};

  // graph (device)
  Graph g{};
  int *d_ls_cam = nullptr, *d_lm_off = nullptr, *d_task_lm = nullptr, *d_cs_lm = nullptr,
      *d_cs_pos = nullptr, *d_seg = nullptr;
  // host copies kept for re-blocking (pv_set_option PV_OPT_BLOCK_BYTES)
  std::vector<int> h_ls_cam, h_ls_lid, h_task_desc;
  std::vector<int> blk_task;  // [n_blk+1] task boundaries of the landmark blocks
  std::vector<int> blk_s;     // [n_blk+1] boundaries of the blocks' partials s (s positions)
  size_t sbuf_doubles = 0;
  std::vector<int> h_lm_off;  // [n_ls+1]
  // landmark-reduce work (k_lm_reduce): per block, landmarks bucketed by track length
  std::vector<int> blk_ktask;  // [n_blk+1] warp slots
  int4* d_klist = nullptr;
  size_t klist_bytes = 0;
  int use_kslot = 1;        // PV_OPT_KSLOT
  int4* d_kslot = nullptr;  // per slot {k, s position, landmarks, first landmark} (stage-1 terms)
  size_t kslot_bytes = 0;
  // V+ (lsys) and t (tarr) live in warp-slot order: landmark l at slot position h_lpos[l]
  // (klist entry index), camera-sorted observation o's landmark at d_cs_kpos[o]
  std::vector<int> h_lpos;
  int* d_lpos = nullptr;
  int* d_cs_kpos = nullptr;
  size_t n_kent = 0;  // klist entries = slot positions (padding lanes included)
  int n_blk = 1;
  int64_t block_bytes = 80ll << 20;
  size_t seg_bytes = 0;
  int64_t persist_l2 = 0;
  bool lm_lin_fresh = false;
  int num_sms = 148;
  int wpc = 1;  // warps per camera in the camera kernels (from the mean segment size)
  // work lists of the persistent camera kernel (k_cam_pipe)
  int pipe_W = 0;
  int bench_split = 0;  // pv_bench_terms diagnostic (PV_OPT_BENCH_SPLIT)
  int64_t solve_us[3] = {0, 0, 0};  // last power solve: RHS, terms, back-substitution
  int64_t solve_terms_launched = 0;
  TermGraph tgraph;
  TermGraph bsgraph;  // the blocked back-substitution as one captured graph (same validity key)
  TermGraph pcggraph; // one PCG iteration (blocked S'.p + the three vector kernels), thr = tolerance
  int4* d_items = nullptr;
  int* d_item_off = nullptr;
  size_t items_bytes = 0, item_off_bytes = 0;
  std::vector<int> h_seg;  // [(n_blk * n_p) + 1] (block, camera) segment starts (re-balancing)
  // cost model of the work-list balance, in observation-equivalents (PV_OPT_BALANCE ...)
  int bal_mode = 1, bal_item = 24, bal_round = 0, bal_last = 0;
  int bal_rfix = 30, bal_robs8 = 3;  // landmark-reduce slot: fixed + (partials * robs8) / 8
  // per-warp landmark-reduce slot lists of the series kernel (k_series)
  int* d_rslot = nullptr;
  int* d_roff = nullptr;
  size_t rslot_bytes = 0, roff_bytes = 0;
  std::vector<int> h_slot_n;  // partials (padding lanes included) of every warp slot
  unsigned* sbar = nullptr;   // grid barrier of k_series
  bool skip_next_gather = false;
  // pinned staging of large pageable host transfers (pv_set_state / pv_get_state)
  char* stage_pin[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};  // the RHS launches leave block 0's W^T v pass to k_series
  int layout_gen = 0;  // bumped whenever device work lists are rebuilt (term-graph cache key)
  int lr_ctas_per_sm = 3;  // lvr/lbl hold the stage-1 landmark linearization of the current state
  double *d_ls_m = nullptr, *d_cs_m = nullptr;
  double* d_ks_m = nullptr;  // slot-interleaved copies of ls_m / ls_cam (s positions)
  int* d_ks_cam = nullptr;
  size_t ks_entries = 0;

  // state and solve buffers (device)
  double *crec, *lrec, *lvr, *lbl, *ldl, *tlm, *tcam, *cs_x, *cs_xm;
  double* d_cs_m1 = nullptr;  // m1 per camera-sorted observation (compact stage-1 stream)
  bool xm_ok = false;         // cs_xm holds the current linearization point (stage 1, w == 1)
  double *lsys = nullptr, *tarr = nullptr, *sbuf = nullptr;
  double *cU, *cUd, *cUi, *cbp, *cx, *crhs, *ch, *cy, *cyr, *cUraw, *nrm, *ctmp, *scal;
  double* cpart = nullptr;
  int* flags;
  unsigned* ticket;
  PowerCtl* ctl;
  PowerCtl* host_ctl = nullptr;  // mapped pinned mirror
  // PCG (allocated on first use): moments, Schur diagonal, scratch, preconditioner,
  // vectors x r z p sp, per-camera partials
  double *cmom = nullptr, *csd = nullptr, *csdd = nullptr, *cmi = nullptr, *pvec = nullptr,
         *ppart = nullptr;
  PowerCtl* host_ctl_dev = nullptr;

  Tune tune{0, 1, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1, 0};
  int64_t last_fallbacks = 0;  // landmarks that took the exact Givens path in the last re-solve
  int lin_stage = 0;
  bool vp_cached = false;  // V+ valid for POSE_ONLY damping of the current linearization
  // reduced RHS reuse: -(b_p - W V+ b_l) depends on the linearization only when V+ is
  // undamped (POSE_ONLY), so a rejected step's next solve skips its camera pass
  int64_t lin_id = 0, rhs_lin_id = -1, damp_lin_id = -1;
  bool last_damp_both = true;
  int step_stage = 0;

  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
    CK(cudaMalloc(&p, bytes));
    CK(cudaMemsetAsync(p, 0, bytes, stream));
    allocs.push_back(p);
    device_bytes += bytes;
    return static_cast<T*>(p);
  }

  void launched(int n = 1) { launches += n; }
  void check_launch() { CK(cudaGetLastError()); }

  // the collective (sharded) code path: world > 1, or forced on one GPU with a
  // 1-rank NCCL communicator to exercise the split kernels + NCCL calls
  bool collective() const { return comm != nullptr || loop != nullptr; }
  void allreduce(double* p, size_t n) {
    if (comm) NK(ncclAllReduce(p, p, n, ncclDouble, ncclSum, comm, stream));
    if (loop) loop_allreduce(p, n, false);
  }
  void allreduce_flags() {
    if (comm) NK(ncclAllReduce(flags, flags, F_COUNT, ncclInt32, ncclMax, comm, stream));
    if (loop) loop_allreduce(flags, F_COUNT, true);
  }
  // loopback communicator (LoopGroup): one host thread per rank
  LoopGroup* loop = nullptr;
  void* loop_tmp = nullptr;     // rank-order sum (n_p * 144 doubles)
  void** loop_ptrs = nullptr;   // device array of the ranks' buffer pointers
  void loop_allreduce(void* p, size_t n, bool is_flags) {
    LoopGroup& G = *loop;
    G.bufs[rank] = p;
    CK(cudaEventRecord(G.ready[rank], stream));
    G.barrier();  // every rank's buffer pointer and ready event are posted
    for (int q = 0; q < world; ++q)
      if (q != rank) CK(cudaStreamWaitEvent(stream, G.ready[q], 0));
    CK(cudaMemcpyAsync(loop_ptrs, G.bufs.data(), sizeof(void*) * world, cudaMemcpyHostToDevice,
                       stream));
    if (is_flags)
      k_loop_max<<<1, 32, 0, stream>>>(world, (const int* const*)loop_ptrs, (int)n,
                                       (int*)loop_tmp);
    else
      k_loop_sum<<<(int)std::min<size_t>(1024, (n + 255) / 256), 256, 0, stream>>>(
          world, (const double* const*)loop_ptrs, n, (double*)loop_tmp);
    launched();
    CK(cudaEventRecord(G.done[rank], stream));
    CK(cudaStreamSynchronize(stream));  // the host-side pointer array copy is consumed
    G.barrier();  // every rank has enqueued (and finished) its reads
    for (int q = 0; q < world; ++q)
      if (q != rank) CK(cudaStreamWaitEvent(stream, G.done[q], 0));
    CK(cudaMemcpyAsync(p, loop_tmp, n * (is_flags ? sizeof(int) : sizeof(double)),
                       cudaMemcpyDeviceToDevice, stream));
    // (no third barrier: a rank re-records its events only after the next collective's first
    // barrier, i.e. after every rank has enqueued its waits on this collective's events)
  }
  void sync() { CK(cudaStreamSynchronize(stream)); }

  int nblk_tasks() const { return blocks_for((long long)n_tasks * 32, 256); }
  // deterministic sum of n_tasks warp partials into scal[0] (two levels)
  // deterministic sum of n (default n_tasks <= the buffer's capacity) warp partials
  void sum_partials(int n = -1) {
    if (n < 0) n = n_tasks;
    if ((size_t)n > cpart_cap) throw PvError(PV_ECUDA, "partials exceed the cpart capacity");
    const int nb2 = std::max(1, std::min(256, (n + 4095) / 4096));
    double* lvl2 = cpart + cpart_cap + 8;
    k_sum<<<nb2, 1024, 0, stream>>>(cpart, std::max(n, 1), lvl2);
    k_sum<<<1, 1024, 0, stream>>>(lvl2, nb2, scal);
    launched(2);
  }
  // cudaFuncSetAttribute is per device context: remember it per kernel and context
  std::vector<const void*> attr_set;
  void max_dyn_smem(const void* fn, int bytes) {
    if (std::find(attr_set.begin(), attr_set.end(), fn) != attr_set.end()) return;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    attr_set.push_back(fn);
  }
};

// ---------------------------------------------------------------------------
// graph construction (host, O(n) counting sorts)

static void build_graph(pv_ctx* c, const int64_t* cam_idx, const int64_t* lm_idx,
                        const double* meas, int64_t lm_begin, int64_t lm_end) {
  const int64_t n_o = c->n_o_global, n_p = c->n_p;
  const int64_t span = lm_end - lm_begin;
  std::vector<int64_t> cnt(span, 0);
  for (int64_t o = 0; o < n_o; ++o) {
    int64_t l = lm_idx[o];
    if (l >= lm_begin && l < lm_end) cnt[l - lm_begin]++;
  }
  std::vector<int> lid(span, -1);
  c->lm_gid.clear();
  for (int64_t j = 0; j < span; ++j)
    if (cnt[j] > 0) {
      lid[j] = (int)c->lm_gid.size();
      c->lm_gid.push_back(lm_begin + j);
    }
  const int n_ls = (int)c->lm_gid.size();
  int64_t n_os = 0;
  for (int64_t j = 0; j < span; ++j) n_os += cnt[j];
  if (n_os >= (int64_t)INT32_MAX) throw PvError(PV_EINVAL, "shard has too many observations");
  c->n_ls = n_ls;
  c->n_os = (int)n_os;

  // landmark-major order with the cameras of a landmark ascending (ties in input order): one
  // counting sort by local landmark, then a stable insertion sort of each landmark's few
  // observations by camera -- the same order as a stable sort by camera followed by a stable
  // sort by landmark, with one random pass over the observations instead of two
  std::vector<int> lm_off(n_ls + 1, 0);
  for (int j = 0; j < n_ls; ++j) lm_off[j + 1] = lm_off[j] + (int)cnt[c->lm_gid[j] - lm_begin];
  std::vector<int> ls_cam(n_os), ls_lid(n_os);
  std::vector<double> ls_m(2 * n_os);
  {
    std::vector<int64_t> src(n_os);  // input index of every landmark-sorted slot
    std::vector<int> pos(lm_off.begin(), lm_off.end() - 1);
    for (int64_t o = 0; o < n_o; ++o) {
      const int64_t l = lm_idx[o];
      if (l >= lm_begin && l < lm_end) src[pos[lid[l - lm_begin]]++] = o;
    }
    for (int j = 0; j < n_ls; ++j) {
      int64_t* a = src.data() + lm_off[j];
      const int k = lm_off[j + 1] - lm_off[j];
      for (int i = 1; i < k; ++i) {  // stable: equal cameras keep their input order
        const int64_t v = a[i];
        const int64_t cv = cam_idx[v];
        int q = i - 1;
        while (q >= 0 && cam_idx[a[q]] > cv) {
          a[q + 1] = a[q];
          --q;
        }
        a[q + 1] = v;
      }
      for (int i = 0; i < k; ++i) {
        const int64_t o = a[i];
        const int p = lm_off[j] + i;
        ls_cam[p] = (int)cam_idx[o];
        ls_lid[p] = j;
        ls_m[2 * p] = meas[2 * o];
        ls_m[2 * p + 1] = meas[2 * o + 1];
      }
    }
  }
  // landmark tasks: whole landmarks packed into <= 32 lanes, or one long landmark;
  // descriptor {first obs, obs count, first landmark, segment-head lane mask}
  std::vector<int> task_desc;
  {
    int j = 0;
    while (j < n_ls) {
      const int l0 = j;
      const int o0 = lm_off[j];
      int k = lm_off[j + 1] - lm_off[j];
      unsigned heads = 1u;
      if (k > 32) {
        ++j;
      } else {
        int total = k, nl = 1;
        ++j;
        while (j < n_ls && nl < 32) {
          int kk = lm_off[j + 1] - lm_off[j];
          if (kk > 32 || total + kk > 32) break;
          heads |= 1u << total;
          total += kk;
          ++nl;
          ++j;
        }
        k = total;
      }
      task_desc.push_back(o0);
      task_desc.push_back(k);
      task_desc.push_back(l0);
      task_desc.push_back((int)heads);
    }
  }
  c->n_tasks = (int)task_desc.size() / 4;

  auto up_i = [&](const std::vector<int>& v) {
    int* d = c->alloc<int>(v.size());
    CK(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    return d;
  };
  auto up_d = [&](const std::vector<double>& v) {
    double* d = c->alloc<double>(v.size());
    CK(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice,
                       c->stream));
    return d;
  };
  c->d_ls_cam = up_i(ls_cam);
  c->d_ls_m = up_d(ls_m);
  c->d_lm_off = up_i(lm_off);
  c->d_task_lm = up_i(task_desc);
  // camera-sorted arrays are (re)built by build_blocks in block-major order
  // padded by one staging chunk (k_cam copies whole chunks)
  c->d_cs_lm = c->alloc<int>((size_t)n_os + 128);
  c->d_cs_pos = c->alloc<int>((size_t)n_os + 128);
  c->d_cs_kpos = c->alloc<int>((size_t)n_os + 128);
  c->d_lpos = c->alloc<int>((size_t)n_ls + 1);
  c->d_cs_m = c->alloc<double>(2 * ((size_t)n_os + 128));
  c->d_cs_m1 = c->alloc<double>((size_t)n_os + 128);
  c->sync();  // host vectors go out of scope
  c->h_ls_cam = std::move(ls_cam);
  c->h_ls_lid = std::move(ls_lid);
  c->h_task_desc = task_desc;
  c->h_lm_off = lm_off;

  Graph& g = c->g;
  g.n_p = (int)n_p;
  g.n_l = n_ls;
  g.n_o = (int)n_os;
  g.n_tasks = c->n_tasks;
  g.ls_cam = c->d_ls_cam;
  g.ls_m = c->d_ls_m;
  g.lm_off = c->d_lm_off;
  g.task = reinterpret_cast<const int4*>(c->d_task_lm);
  g.cs_lm = c->d_cs_lm;
  g.cs_m = c->d_cs_m;
  g.cs_pos = c->d_cs_pos;
  g.cs_kpos = c->d_cs_kpos;
}

// Landmark blocks of the L2-blocked term: contiguous task ranges with ~equal
// observation counts, sized so one block's partials s (32 B/obs) fit in the
// budget; per camera, the camera-sorted sub-range of each block.
template <class T>
static void free_tracked(pv_ctx* c, T*& p, size_t bytes) {
  if (!p) return;
  CK(cudaFree(p));
  auto it = std::find(c->allocs.begin(), c->allocs.end(), (void*)p);
  if (it != c->allocs.end()) c->allocs.erase(it);
  c->device_bytes -= bytes;
  p = nullptr;
}

// warp partials of the deterministic two-level sums: one per landmark task (k_cost,
// k_resolve), per cost segment (k_cost_cs, <= n_tasks) or per landmark warp slot
// (k_resolve_slots: blk_ktask[n_blk], which depends on the blocking), then the level-2 sums
static void ensure_cpart(pv_ctx* c) {
  const size_t ns = c->blk_ktask.empty() ? 0 : (size_t)c->blk_ktask[c->n_blk];
  const size_t need = std::max<size_t>({(size_t)c->n_tasks, ns, 1});
  if (c->cpart && need <= c->cpart_cap) return;
  free_tracked(c, c->cpart, (c->cpart_cap + 8 + 256) * sizeof(double));
  c->cpart = c->alloc<double>(need + 8 + 256);
  c->cpart_cap = need;
}

// Work lists of k_cam_pipe (pv_pipe.cuh) and k_series (pv_series.cuh).  Every (camera, block)
// segment is cut into items of <= PCH observations; per landmark block there are four
// families of per-warp lists, plus the per-warp landmark-reduce slot lists of k_series:
//   0: W t items (>= 1 per camera so that y is always written).  A camera's items stay with
//      one warp (it owns the camera's sum);
//   1: W^T v items for a pass launched on its own;
//   2: W^T v items of block b for the launch that also runs the W t items of block b - 1;
//   3: W^T v items of block b for the k_series step that also runs the reduce slots of block
//      b - 1 and the W t items of block b - 2.
// Balance (bal_mode 1): the cost of an item is n + bal_item + bal_round * ceil(n / 32)
// (+ bal_last on a camera's last W t item), in observation-equivalents.  Family 0 packs
// whole cameras longest-first onto the least loaded warp; W^T v items are independent, so
// families 1 and 2 cut the stream at item granularity, family 2 giving each warp what its
// W t list of block b - 1 leaves below the launch's mean.  With contiguous equal-cost camera
// ranges (bal_mode 0, round 1) the heaviest warp carried 17-18% more than the mean at vlarge
// (a camera's segment is ~1/6 of a warp's share) and the launch waited for it.
static void build_pipe_items(pv_ctx* c, const std::vector<int>& seg) {
  if (!c->pipe_W) {
    int occ = 1 << 30;
    auto occ_of = [&](const void* fn) {
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, PIPE_SMEM));
      int o = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, PW * 32, PIPE_SMEM));
      occ = std::min(occ, o);
    };
    occ_of((const void*)k_cam_pipe<1, true, true, false>);
    occ_of((const void*)k_cam_pipe<2, true, true, false>);
    occ_of((const void*)k_cam_pipe<1, false, true, false>);
    occ_of((const void*)k_cam_pipe<2, false, true, false>);
    occ_of((const void*)k_cam_pipe<1, true, false, false>);
    occ_of((const void*)k_cam_pipe<2, true, false, false>);
    occ_of((const void*)k_cam_pipe<1, true, true, true>);
    occ_of((const void*)k_cam_pipe<1, false, true, true>);
    occ_of((const void*)k_cam_pipe<1, true, false, true>);
    occ_of((const void*)k_series<1, false>);
    occ_of((const void*)k_series<1, true>);
    occ_of((const void*)k_series<2, false>);
    c->pipe_W = std::max(1, occ) * c->num_sms * PW;
  }
  const int B = c->n_blk, W = c->pipe_W;
  const int64_t np = c->n_p;
  const int IC = c->bal_item, RC = c->bal_round, LC = c->bal_last;
  auto item_cost = [&](int n, bool last_hc) {
    return (int64_t)n + IC + (int64_t)RC * ((n + 31) / 32) + (last_hc ? LC : 0);
  };
  std::vector<int4> items;
  std::vector<int> off((size_t)4 * B * (W + 1), 0);
  items.reserve((size_t)4 * ((size_t)c->n_os / PCH + (size_t)B * np + 16));
  auto push_cam = [&](int64_t cam, const int* sb, int L) {  // all items of one camera
    const int o_lo = sb[cam], n = sb[cam + 1] - o_lo;
    const int k0 = (n + PCH - 1) / PCH, k = L == 0 ? std::max(1, k0) : k0;
    for (int q = 0; q < k; ++q) {
      const int o = o_lo + q * PCH;
      const int cnt = std::max(0, std::min(PCH, o_lo + n - o));
      items.push_back(make_int4((int)cam, o, cnt, (L ? PF_HA : 0) | (q == k - 1 ? PF_LAST : 0)));
    }
  };
  auto cam_cost = [&](int64_t cam, const int* sb, int L) {
    const int n = sb[cam + 1] - sb[cam];
    const int k0 = (n + PCH - 1) / PCH, k = L == 0 ? std::max(1, k0) : k0;
    int64_t t = 0;
    for (int q = 0; q < k; ++q)
      t += item_cost(std::max(0, std::min(PCH, n - q * PCH)), L == 0 && q == k - 1);
    return t;
  };
  std::vector<std::vector<int64_t>> hc_load(B, std::vector<int64_t>(W, 0));
  std::vector<std::vector<int64_t>> r_load(B, std::vector<int64_t>(W, 0));
  double worst[5] = {1.0, 1.0, 1.0, 1.0, 1.0};
  using Slot = std::pair<int64_t, int>;  // (load, warp): smallest load first, then warp
  // longest-first packing of (cost, id) units onto the warps, starting from `init` loads;
  // mine[w] = the ids of warp w in increasing order, load[w] = its packed cost (init excluded)
  auto pack = [&](std::vector<std::pair<int64_t, int>>& units, const std::vector<int64_t>* init,
                  std::vector<std::vector<int>>& mine, std::vector<int64_t>& load) {
    std::stable_sort(units.begin(), units.end(),
                     [](const std::pair<int64_t, int>& a, const std::pair<int64_t, int>& x) {
                       return a.first > x.first;
                     });
    std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> heap;
    for (int w = 0; w < W; ++w) heap.push({init ? (*init)[w] : 0, w});
    mine.assign(W, {});
    load.assign(W, 0);
    for (const auto& u : units) {
      Slot sl = heap.top();
      heap.pop();
      mine[sl.second].push_back(u.second);
      sl.first += u.first;
      load[sl.second] += u.first;
      heap.push(sl);
    }
    for (int w = 0; w < W; ++w) std::sort(mine[w].begin(), mine[w].end());
  };
  auto imbalance = [&](const std::vector<int64_t>& a, const std::vector<int64_t>* b2,
                       const std::vector<int64_t>* b3) {
    int64_t tot = 0, mx = 0;
    for (int w = 0; w < W; ++w) {
      const int64_t v = a[w] + (b2 ? (*b2)[w] : 0) + (b3 ? (*b3)[w] : 0);
      tot += v;
      mx = std::max(mx, v);
    }
    return tot > 0 ? (double)mx * W / (double)tot : 1.0;
  };
  // family 0: W t items, whole cameras per warp
  for (int b = 0; b < B; ++b) {
    const int* sb = seg.data() + (size_t)b * np;
    int* ob = off.data() + (size_t)(0 * B + b) * (W + 1);
    ob[0] = (int)items.size();
    if (c->bal_mode == 0) {  // contiguous camera ranges of equal cost
      int64_t tot = 0, cum = 0;
      for (int64_t cam = 0; cam < np; ++cam) tot += cam_cost(cam, sb, 0);
      int w = 0;
      for (int64_t cam = 0; cam < np; ++cam) {
        while (w < W - 1 && cum * W >= (int64_t)(w + 1) * tot) ob[++w] = (int)items.size();
        push_cam(cam, sb, 0);
        cum += cam_cost(cam, sb, 0);
        hc_load[b][w] += cam_cost(cam, sb, 0);
      }
      while (w < W) ob[++w] = (int)items.size();
    } else {
      std::vector<std::pair<int64_t, int>> cams((size_t)np);
      for (int64_t cam = 0; cam < np; ++cam) cams[cam] = {cam_cost(cam, sb, 0), (int)cam};
      std::vector<std::vector<int>> mine;
      pack(cams, nullptr, mine, hc_load[b]);
      for (int w = 0; w < W; ++w) {
        for (int cam : mine[w]) push_cam(cam, sb, 0);
        ob[w + 1] = (int)items.size();
      }
    }
    worst[0] = std::max(worst[0], imbalance(hc_load[b], nullptr, nullptr));
  }
  // landmark-reduce slots of block b for k_series, packed on top of the W t load of block
  // b - 1 (the same step of the series schedule)
  std::vector<int> rslot;
  std::vector<int> roff((size_t)B * (W + 1), 0);
  rslot.reserve(c->h_slot_n.size());
  for (int b = 0; b < B; ++b) {
    const int k0 = c->blk_ktask[b], k1 = c->blk_ktask[b + 1];
    std::vector<std::pair<int64_t, int>> units;
    units.reserve(k1 - k0);
    for (int w = k0; w < k1; ++w)
      units.push_back({(int64_t)c->bal_rfix + ((int64_t)c->h_slot_n[w] * c->bal_robs8) / 8, w});
    std::vector<std::vector<int>> mine;
    pack(units, b > 0 ? &hc_load[b - 1] : nullptr, mine, r_load[b]);
    int* ro = roff.data() + (size_t)b * (W + 1);
    ro[0] = (int)rslot.size();
    for (int w = 0; w < W; ++w) {
      for (int sl : mine[w]) rslot.push_back(sl);
      ro[w + 1] = (int)rslot.size();
    }
    worst[4] = std::max(worst[4], imbalance(r_load[b], b > 0 ? &hc_load[b - 1] : nullptr, nullptr));
  }
  // families 1-3: W^T v items of block b, cut at item granularity so that warp w gets what
  // the other work of its launch / step leaves below the mean: nothing else (1), the W t
  // items of block b - 1 (2), the reduce slots of block b - 1 and the W t items of block
  // b - 2 (3, k_series)
  for (int L = 1; L <= 3; ++L) {
    for (int b = 0; b < B; ++b) {
      const int* sb = seg.data() + (size_t)b * np;
      int* ob = off.data() + (size_t)(L * B + b) * (W + 1);
      ob[0] = (int)items.size();
      std::vector<int64_t> other(W, 0);
      if (c->bal_mode != 0) {
        if (L == 2 && b >= 1) other = hc_load[b - 1];
        if (L == 3 && b >= 1) {
          other = r_load[b - 1];
          if (b >= 2)
            for (int w = 0; w < W; ++w) other[w] += hc_load[b - 2][w];
        }
      }
      if (c->bal_mode == 0) {
        int64_t tot = 0, cum = 0;
        for (int64_t cam = 0; cam < np; ++cam) tot += cam_cost(cam, sb, 1);
        int w = 0;
        for (int64_t cam = 0; cam < np; ++cam) {
          while (w < W - 1 && cum * W >= (int64_t)(w + 1) * tot) ob[++w] = (int)items.size();
          push_cam(cam, sb, 1);
          cum += cam_cost(cam, sb, 1);
        }
        while (w < W) ob[++w] = (int)items.size();
        continue;
      }
      const size_t first = items.size();
      int64_t tot_a = 0, tot_o = 0;
      for (int64_t cam = 0; cam < np; ++cam) {
        push_cam(cam, sb, 1);
        tot_a += cam_cost(cam, sb, 1);
      }
      for (int w = 0; w < W; ++w) tot_o += other[w];
      const double mean = (double)(tot_o + tot_a) / W;
      std::vector<double> want(W);
      double wsum = 0.0;
      for (int w = 0; w < W; ++w) wsum += (want[w] = std::max(0.0, mean - (double)other[w]));
      if (wsum <= 0.0) {
        std::fill(want.begin(), want.end(), 1.0);
        wsum = W;
      }
      size_t i = first;
      double cum = 0.0, bound = 0.0, mx = 0.0;
      for (int w = 0; w < W; ++w) {
        bound += want[w] / wsum * (double)tot_a;
        const double start = cum;
        while (i < items.size()) {  // an item goes to the warp that holds its midpoint
          const double ci = (double)item_cost(items[i].z, false);
          if (w < W - 1 && cum + 0.5 * ci > bound) break;
          cum += ci;
          ++i;
        }
        ob[w + 1] = (int)i;
        mx = std::max(mx, cum - start + (double)other[w]);
      }
      if (mean > 0) worst[L] = std::max(worst[L], mx / mean);
    }
  }
  if (std::getenv("PV_DEBUG_BALANCE"))
    std::fprintf(stderr,
                 "pipe items: B=%d W=%d mode=%d cost(item=%d round=%d last=%d rfix=%d robs8=%d) worst "
                 "max/mean: Wt %.4f  WTv %.4f  Wt+WTv %.4f  R+Wt+WTv %.4f  R+Wt %.4f\n",
                 B, W, c->bal_mode, IC, RC, LC, c->bal_rfix, c->bal_robs8, worst[0], worst[1],
                 worst[2], worst[3], worst[4]);
  free_tracked(c, c->d_rslot, c->rslot_bytes);
  free_tracked(c, c->d_roff, c->roff_bytes);
  c->d_rslot = c->alloc<int>(std::max<size_t>(rslot.size(), 1));
  c->d_roff = c->alloc<int>(roff.size());
  c->rslot_bytes = std::max<size_t>(rslot.size(), 1) * sizeof(int);
  c->roff_bytes = roff.size() * sizeof(int);
  CK(cudaMemcpyAsync(c->d_rslot, rslot.data(), rslot.size() * sizeof(int), cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemcpyAsync(c->d_roff, roff.data(), roff.size() * sizeof(int), cudaMemcpyHostToDevice,
                     c->stream));
  free_tracked(c, c->d_items, c->items_bytes);
  free_tracked(c, c->d_item_off, c->item_off_bytes);
  c->d_items = c->alloc<int4>(items.size());
  c->d_item_off = c->alloc<int>(off.size());
  c->items_bytes = std::max<size_t>(items.size(), 1) * sizeof(int4);
  c->item_off_bytes = std::max<size_t>(off.size(), 1) * sizeof(int);
  CK(cudaMemcpyAsync(c->d_items, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemcpyAsync(c->d_item_off, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice,
                     c->stream));
  c->sync();
  ++c->layout_gen;
}

// Work of the landmark reduce (k_lm_reduce, pv_kernels.cuh) and of the lane-per-landmark
// re-solve, and the layout of the per-observation partials s.  Per landmark block, the
// landmarks are bucketed by track length k and laid out as 32-entry warp slots of
// {landmark, first landmark-sorted observation, k, s position}: a short slot holds up to
// 32 landmarks of equal k <= KSHORT (one lane each; unused lanes have landmark -1); a long
// landmark (k > KSHORT) fills a slot alone.  Longest first, so a grid's tail is made of short
// slots.  The partials s of a short slot are interleaved -- observation i of lane q at
// base + 32 i + q -- so the reduce's k-step walk reads 1 KB contiguous per warp load; a
// long landmark's partials are contiguous.  cs_ls holds the landmark-sorted position of
// every camera-sorted observation; the camera kernels scatter s to g.cs_pos = its
// s position.
static void build_ktasks(pv_ctx* c, const std::vector<int>& cs_ls, const std::vector<int>& cs_lm) {
  const int B = c->n_blk;
  const std::vector<int>& off = c->h_lm_off;
  std::vector<int4> kl;
  kl.reserve((size_t)c->n_ls + 64 * (size_t)B);
  std::vector<int> spos((size_t)c->n_os + 1, 0);  // s position of each landmark-sorted obs
  std::vector<int> lpos((size_t)c->n_ls + 1, 0);  // slot position of each landmark
  int64_t sn = 0;                                 // s entries so far
  c->blk_ktask.assign(B + 1, 0);
  c->blk_s.assign(B + 1, 0);
  c->h_slot_n.clear();
  std::vector<int4> kslot;
  std::vector<std::vector<int>> bucket(KSHORT + 1);
  for (int b = 0; b < B; ++b) {
    const int t0 = c->blk_task[b], t1 = c->blk_task[b + 1];
    const int l0 = t0 < c->n_tasks ? c->h_task_desc[4 * t0 + 2] : c->n_ls;
    const int l1 = t1 < c->n_tasks ? c->h_task_desc[4 * t1 + 2] : c->n_ls;
    std::vector<std::pair<int, int>> longs;  // (k, landmark)
    for (auto& v : bucket) v.clear();
    for (int l = l0; l < l1; ++l) {
      const int k = off[l + 1] - off[l];
      if (k > KSHORT)
        longs.emplace_back(k, l);
      else
        bucket[k].push_back(l);
    }
    std::stable_sort(longs.begin(), longs.end(),
                     [](const std::pair<int, int>& a, const std::pair<int, int>& x) {
                       return a.first > x.first;
                     });
    for (auto& kvl : longs) {  // entry 0, rest empty; contiguous partials
      const int k = kvl.first, l = kvl.second;
      lpos[l] = (int)kl.size();
      kl.push_back(make_int4(l, off[l], k, (int)sn));
      for (int q = 1; q < 32; ++q) kl.push_back(make_int4(-1, 0, k, 0));
      for (int i = 0; i < k; ++i) spos[off[l] + i] = (int)(sn + i);
      kslot.push_back(make_int4(k, (int)sn, 1, l));
      sn += (k + 3) & ~3;  // whole 128-byte lines per slot (dropped from L2 slot by slot)
      c->h_slot_n.push_back(k);
    }
    for (int k = KSHORT; k >= 0; --k) {
      const std::vector<int>& v = bucket[k];
      for (size_t i = 0; i < v.size(); i += 32) {
        const int n = (int)std::min<size_t>(32, v.size() - i);
        for (int q = 0; q < 32; ++q) {
          if (q < n) {
            const int l = v[i + q];
            lpos[l] = (int)kl.size();
            kl.push_back(make_int4(l, off[l], k, (int)(sn + q)));
            for (int j = 0; j < k; ++j) spos[off[l] + j] = (int)(sn + q + 32 * j);
          } else {
            kl.push_back(make_int4(-1, 0, k, 0));
          }
        }
        kslot.push_back(make_int4(k, (int)sn, n, v[i]));
        sn += 32 * (int64_t)k;
        c->h_slot_n.push_back(32 * k);
      }
    }
    if (sn >= (int64_t)INT32_MAX) throw PvError(PV_EINVAL, "too many partial slots for int32");
    c->blk_ktask[b + 1] = (int)(kl.size() / 32);
    c->blk_s[b + 1] = (int)sn;
  }
  free_tracked(c, c->d_klist, c->klist_bytes);
  c->d_klist = c->alloc<int4>(kl.size());
  c->klist_bytes = std::max<size_t>(kl.size(), 1) * sizeof(int4);
  CK(cudaMemcpyAsync(c->d_klist, kl.data(), kl.size() * sizeof(int4), cudaMemcpyHostToDevice,
                     c->stream));
  free_tracked(c, c->d_kslot, c->kslot_bytes);
  c->d_kslot = c->alloc<int4>(std::max<size_t>(kslot.size(), 1));
  c->kslot_bytes = std::max<size_t>(kslot.size(), 1) * sizeof(int4);
  CK(cudaMemcpyAsync(c->d_kslot, kslot.data(), kslot.size() * sizeof(int4), cudaMemcpyHostToDevice,
                     c->stream));
  // the partials buffer holds every slot's entries (padding lanes included)
  const size_t need = std::max<size_t>((size_t)sn, 1) * 4;
  if (need > c->sbuf_doubles) {
    free_tracked(c, c->sbuf, c->sbuf_doubles * sizeof(double));
    c->sbuf = c->alloc<double>(need);
    c->sbuf_doubles = need;
  }
  {  // slot-interleaved copies of the landmark-sorted measurements and camera ids
    const size_t ne = std::max<size_t>((size_t)sn, 1);
    free_tracked(c, c->d_ks_m, c->ks_entries * 2 * sizeof(double));
    free_tracked(c, c->d_ks_cam, c->ks_entries * sizeof(int));
    c->d_ks_m = c->alloc<double>(ne * 2);
    c->d_ks_cam = c->alloc<int>(ne);
    c->ks_entries = ne;
    int* d_spos = nullptr;
    CK(cudaMalloc(&d_spos, std::max<size_t>((size_t)c->n_os, 1) * sizeof(int)));
    CK(cudaMemcpyAsync(d_spos, spos.data(), (size_t)c->n_os * sizeof(int), cudaMemcpyHostToDevice,
                       c->stream));
    k_scatter_ks<<<blocks_for(c->n_os, 256), 256, 0, c->stream>>>(c->n_os, d_spos, c->d_ls_m,
                                                                 c->d_ls_cam, c->d_ks_m,
                                                                 c->d_ks_cam);
    c->launched();
    c->sync();
    CK(cudaFree(d_spos));
    c->g.ks_m = c->d_ks_m;
    c->g.ks_cam = c->d_ks_cam;
  }
  // s position of every camera-sorted observation (the scatter target of W^T v) and the
  // slot position of its landmark (the gather index of t and V+)
  std::vector<int> cs_s(cs_ls.size(), 0), cs_k(cs_lm.size(), 0);
  for (int p = 0; p < c->n_os; ++p) {
    cs_s[p] = spos[cs_ls[p]];
    cs_k[p] = lpos[cs_lm[p]];
  }
  CK(cudaMemcpyAsync(c->d_cs_pos, cs_s.data(), cs_s.size() * sizeof(int), cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemcpyAsync(c->d_cs_kpos, cs_k.data(), cs_k.size() * sizeof(int),
                     cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->d_lpos, lpos.data(), lpos.size() * sizeof(int), cudaMemcpyHostToDevice,
                     c->stream));
  // V+ and t in slot order; a re-blocking moves a damped V+ to the new positions
  const size_t nk = std::max<size_t>(kl.size(), 1);
  std::vector<double> vold;
  if (c->lsys && !c->h_lpos.empty()) {
    vold.resize(c->n_kent * LSYS);
    CK(cudaMemcpyAsync(vold.data(), c->lsys, vold.size() * sizeof(double),
                       cudaMemcpyDeviceToHost, c->stream));
    c->sync();
  }
  free_tracked(c, c->lsys, c->n_kent * LSYS * sizeof(double));
  free_tracked(c, c->tarr, c->n_kent * 4 * sizeof(double));
  c->lsys = c->alloc<double>(nk * LSYS);
  c->tarr = c->alloc<double>(nk * 4);
  if (!vold.empty()) {
    std::vector<double> vnew(nk * LSYS, 0.0);
    for (int l = 0; l < c->n_ls; ++l)
      for (int q = 0; q < LSYS; ++q)
        vnew[(size_t)lpos[l] * LSYS + q] = vold[(size_t)c->h_lpos[l] * LSYS + q];
    CK(cudaMemcpyAsync(c->lsys, vnew.data(), vnew.size() * sizeof(double),
                       cudaMemcpyHostToDevice, c->stream));
  }
  c->n_kent = nk;
  c->g.n_kent = (int)nk;
  c->g.n_s = (long long)c->sbuf_doubles / 4;
  c->sync();
  c->h_lpos = std::move(lpos);
}

static void build_blocks(pv_ctx* c) {
  const auto tbb = std::chrono::steady_clock::now();
  const int n_os = c->n_os, n_tasks = c->n_tasks;
  const int64_t n_p = c->n_p;
  const int64_t want = std::max<int64_t>(1, ((int64_t)n_os * 32 + c->block_bytes - 1) /
                                                std::max<int64_t>(c->block_bytes, 1));
  const int nb = (int)std::min<int64_t>(want, std::max(1, n_tasks));
  std::vector<int> bt(1, 0);
  int64_t cum = 0;
  for (int t = 0; t < n_tasks; ++t) {
    cum += c->h_task_desc[4 * t + 1];
    if ((int)bt.size() < nb && cum * nb >= (int64_t)bt.size() * n_os && t + 1 < n_tasks)
      bt.push_back(t + 1);
  }
  bt.push_back(n_tasks);
  const int B = (int)bt.size() - 1;
  // block of every landmark-sorted observation (blocks are contiguous in ls order)
  std::vector<int> obs_blk_end(B);
  for (int b = 0; b < B; ++b) {
    const int t1 = bt[b + 1];
    obs_blk_end[b] = t1 < n_tasks ? c->h_task_desc[4 * t1] : n_os;
  }
  // block-major camera-sorted order: stable counting sort of ls rows by (block, camera)
  std::vector<int> seg((size_t)B * n_p + 1, 0);
  {
    int b = 0;
    for (int k = 0; k < n_os; ++k) {
      while (k >= obs_blk_end[b]) ++b;
      seg[(size_t)b * n_p + c->h_ls_cam[k] + 1]++;
    }
    for (size_t i = 0; i + 1 < seg.size(); ++i) seg[i + 1] += seg[i];
  }
  std::vector<int> cs_lm((size_t)n_os + 128, 0), cs_pos((size_t)n_os + 128, 0);
  {
    std::vector<int> pos(seg.begin(), seg.end() - 1);
    int b = 0;
    for (int k = 0; k < n_os; ++k) {
      while (k >= obs_blk_end[b]) ++b;
      const int p = pos[(size_t)b * n_p + c->h_ls_cam[k]]++;
      cs_lm[p] = c->h_ls_lid[k];
      cs_pos[p] = k;
    }
  }
  free_tracked(c, c->d_seg, c->seg_bytes);
  c->d_seg = c->alloc<int>(seg.size());
  c->seg_bytes = seg.size() * sizeof(int);
  CK(cudaMemcpyAsync(c->d_seg, seg.data(), seg.size() * sizeof(int), cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemcpyAsync(c->d_cs_lm, cs_lm.data(), cs_lm.size() * sizeof(int),
                     cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->d_cs_pos, cs_pos.data(), cs_pos.size() * sizeof(int),
                     cudaMemcpyHostToDevice, c->stream));
  k_gather_m<<<blocks_for(n_os, 256), 256, 0, c->stream>>>(n_os, c->d_cs_pos, c->d_ls_m,
                                                           c->d_cs_m);
  k_gather_m1<<<blocks_for(n_os, 256), 256, 0, c->stream>>>(n_os, c->d_cs_m, c->d_cs_m1);
  c->launched(2);
  c->sync();
  c->blk_task = bt;
  c->n_blk = B;
  {  // ~4 staged chunks per warp: warps per camera from the mean (camera, block) segment
    const double mean_seg = (double)n_os / std::max<int64_t>(1, (int64_t)B * n_p);
    int w = 1;
    while (w < 8 && mean_seg > 4.0 * CH * w) w *= 2;
    c->wpc = w;
  }
  c->g.n_blk = B;
  c->g.seg = c->d_seg;
  c->lin_stage = 0;  // camera-sorted copies of x must be rebuilt
  const auto tb0 = std::chrono::steady_clock::now();
  build_ktasks(c, cs_pos, cs_lm);  // replaces d_cs_pos (landmark-sorted positions) by s positions
  const auto tb1 = std::chrono::steady_clock::now();
  build_pipe_items(c, seg);
  if (std::getenv("PV_DEBUG_SETUP"))
    std::fprintf(stderr, "build_blocks: sort+upload %.0f ms, ktasks %.0f ms, pipe items %.0f ms\n",
                 std::chrono::duration<double, std::milli>(tb0 - tbb).count(),
                 std::chrono::duration<double, std::milli>(tb1 - tb0).count(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tb1).count());
  c->h_seg = seg;
  if (c->cpart) ensure_cpart(c);   // re-blocking changes the number of warp slots
}

static void alloc_buffers(pv_ctx* c) {
  const size_t np = c->n_p, nl = c->n_ls;
  c->crec = c->alloc<double>(np * CREC);
  c->lrec = c->alloc<double>(nl * LREC);
  c->lvr = c->alloc<double>(nl * 8);
  // c->lsys, c->tarr: allocated by build_ktasks (warp-slot order)
  c->cs_x = c->alloc<double>(((size_t)c->n_os + 128) * 4);
  c->cs_xm = c->alloc<double>(((size_t)c->n_os + 128) * 4);
  // c->sbuf: sized by build_ktasks (slot layout, padding lanes included)
  c->lbl = c->alloc<double>(nl * 4);
  c->ldl = c->alloc<double>(nl * 4);
  c->tlm = c->alloc<double>(nl * 4);
  c->tcam = c->alloc<double>(np * 12);
  c->cU = c->alloc<double>(np * 144);
  c->cUd = c->alloc<double>(np * 144);
  c->cUi = c->alloc<double>(np * 144);
  c->cbp = c->alloc<double>(np * 12);
  c->cx = c->alloc<double>(np * 12);
  c->crhs = c->alloc<double>(np * 12);
  c->ch = c->alloc<double>(np * 12);
  c->cy = c->alloc<double>(np * 12);
  c->cyr = c->alloc<double>(np * 12);
  c->cUraw = c->alloc<double>(np * LINP);
  c->nrm = c->alloc<double>(np * 2);
  ensure_cpart(c);  // warp partials + level 2
  c->ctmp = c->alloc<double>(np * 12);
  c->scal = c->alloc<double>(8);
  c->flags = c->alloc<int>(F_COUNT);
  c->ticket = c->alloc<unsigned>(4);
  c->sbar = c->alloc<unsigned>(4);
  c->ctl = c->alloc<PowerCtl>(1);
  CK(cudaHostAlloc((void**)&c->host_ctl, sizeof(PowerCtl), cudaHostAllocMapped));
  std::memset(c->host_ctl, 0, sizeof(PowerCtl));
  CK(cudaHostGetDevicePointer((void**)&c->host_ctl_dev, c->host_ctl, 0));
}

// ---------------------------------------------------------------------------
// operations

#ifndef PV_COST_OBS
#define PV_COST_OBS 512
#endif
template <int S>
static void op_cost(pv_ctx* c, int which, double* f) {
  const double* cams = which == PV_TRIAL ? c->tcam : c->crec;
  const int cs = which == PV_TRIAL ? 12 : CREC;
  const double* lms = which == PV_TRIAL ? c->tlm : c->lrec;
  const int ls = which == PV_TRIAL ? 4 : LREC;
  CK(cudaMemsetAsync(c->flags + F_INVALID_Z, 0, sizeof(int), c->stream));
  int nparts = c->n_tasks;
  if (c->tune.cost_cs) {  // camera-sorted walk, ~PV_COST_OBS observations per warp
    nparts = (int)std::max<long long>(
        1, std::min<long long>(c->n_tasks, ((long long)c->n_os + PV_COST_OBS - 1) / PV_COST_OBS));
    k_cost_cs<S><<<blocks_for((long long)nparts * 32, 256), 256, 0, c->stream>>>(
        c->g, cams, cs, lms, ls, nparts, c->cpart, c->flags, c->coef);
  } else {
    k_cost<S><<<blocks_for((long long)c->n_tasks * 32, 64), 64, 0, c->stream>>>(
        c->g, cams, cs, lms, ls, c->cpart, c->flags, c->coef);
  }
  c->launched();
  c->sum_partials(nparts);
  c->check_launch();
  c->allreduce(c->scal, 1);
  c->allreduce_flags();
  double v = 0.0;
  int fl[F_COUNT];
  CK(cudaMemcpyAsync(&v, c->scal, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(fl, c->flags, sizeof(fl), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  *f = (S == 2 && fl[F_INVALID_Z]) ? INFINITY : v;
}

template <int S>
static int op_linearize(pv_ctx* c) {
  ++c->lin_id;
  CK(cudaMemsetAsync(c->flags, 0, F_COUNT * sizeof(int), c->stream));
  k_build_csx<S><<<blocks_for(c->n_os, 256), 256, 0, c->stream>>>(c->g, c->lrec, c->cs_x,
                                                                   c->cs_xm, c->flags);
  if (!(S == 1 && c->lm_lin_fresh)) {
    if (c->tune.resolve_slots) {  // the lane-per-landmark slot kernels (same knob)
      const int ns = c->blk_ktask[c->n_blk];
      k_lin_lm_slots<S><<<blocks_for((long long)ns * 32, 256), 256, 0, c->stream>>>(
          c->g, c->d_klist, ns, c->crec, c->lrec, c->lvr, c->lbl, c->flags, c->coef);
    } else {
      k_lin_lm<S><<<c->nblk_tasks(), 256, 0, c->stream>>>(c->g, c->crec, c->lrec, c->lvr,
                                                          c->lbl, c->flags, c->coef);
    }
    c->launched();
  }
  c->lm_lin_fresh = false;
  c->max_dyn_smem((const void*)k_lin_cam<S>, LIN_SMEM);
  k_lin_cam<S><<<(int)c->n_p, FT, LIN_SMEM, c->stream>>>(c->g, c->crec, c->cs_x, c->cUraw,
                                                         c->coef);
  c->launched(2);
  c->check_launch();
  c->allreduce(c->cUraw, (size_t)c->n_p * LINP);
  k_lin_cam_project<S><<<blocks_for(c->n_p, 128), 128, 0, c->stream>>>(
      (int)c->n_p, c->cUraw, c->crec, c->cU, c->cbp, c->ch);
  c->launched();
  c->check_launch();
  c->allreduce_flags();
  int fl[F_COUNT];
  CK(cudaMemcpyAsync(fl, c->flags, sizeof(fl), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  c->lin_stage = S;
  c->vp_cached = false;
  c->xm_ok = S == 1 && !fl[F_XM_BAD];
  if (S == 2 && fl[F_INVALID_Z]) {
    c->lin_stage = 0;
    return PV_EDEGENERATE;
  }
  return PV_OK;
}

template <int S>
static void op_damp(pv_ctx* c, double lam, int both, int64_t* n_deg) {
  const int D = S == 1 ? 12 : 11;
  c->last_damp_both = both != 0;
  c->damp_lin_id = -1;
  CK(cudaMemsetAsync(c->flags + F_SINGULAR_U, 0, 2 * sizeof(int), c->stream));
  CK(cudaMemsetAsync(c->flags + F_SINGULAR_M2, 0, sizeof(int), c->stream));
  k_damp_cam<<<blocks_for(c->n_p * 32, 128), 128, 0, c->stream>>>((int)c->n_p, D, c->cU, lam, c->cUd,
                                                           c->cUi, c->flags);
  c->launched();
  if (both || !c->vp_cached) {
    k_damp_lm<S><<<blocks_for(c->n_ls, 256), 256, 0, c->stream>>>(
        c->n_ls, c->lvr, c->d_lpos, c->lsys, lam, both, c->flags);
    c->launched();
    c->vp_cached = !both;
  }
  c->check_launch();
  c->allreduce_flags();
  int fl[F_COUNT];
  CK(cudaMemcpyAsync(fl, c->flags, sizeof(fl), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (fl[F_SINGULAR_U]) {
    // a damped pose block that is not positive definite (lam = 0 and an unconstrained
    // camera): np.linalg.inv (solvers.py:108-109) inverts it exactly by LU with partial
    // pivoting, or raises LinAlgError on an exactly singular block
    k_inv_lu<<<blocks_for(c->n_p, 32), 32, 0, c->stream>>>((int)c->n_p, D, c->cUd, c->cUi,
                                                           c->flags);
    c->launched();
    c->check_launch();
    c->allreduce_flags();
    CK(cudaMemcpyAsync(fl, c->flags, sizeof(fl), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (fl[F_SINGULAR_M2]) throw PvError(PV_ESINGULAR, "Singular matrix");
  }
  c->damp_lin_id = c->lin_id;
  if (n_deg) *n_deg = fl[F_N_DEGEN];
}

template <int S, bool HC, int EP, bool HA>
static void launch_cam_v(pv_ctx* c, const CamArgs& ca) {
  constexpr int smem = CAM_SMEM;
  c->max_dyn_smem((const void*)k_cam<S, HC, EP, HA>, smem);
  CamArgs a = ca;
  a.wpc = c->wpc;
  const int cams_per_cta = 8 / c->wpc;
  k_cam<S, HC, EP, HA><<<blocks_for(c->n_p, cams_per_cta), 256, smem, c->stream>>>(
      c->g, c->crec, c->cs_x, c->tarr, c->sbuf, c->cy, c->cyr, c->cbp, c->cUi, c->cx, c->crhs,
      c->ch, c->nrm, c->ctl, c->host_ctl_dev, c->ticket, c->coef, c->tune, a);
  c->launched();
}

template <int S, bool HC, bool HA>
static void launch_cam_pipe(pv_ctx* c, const CamArgs& ca) {
  PipeItems it{c->d_items, c->d_item_off, c->n_blk, c->pipe_W};
  if (S == 1 && c->xm_ok && c->tune.xm) {  // compact stage-1 stream (x0 x1 x2 m0 | m1)
    k_cam_pipe<S, HC, HA, true><<<c->pipe_W / PW, PW * 32, PIPE_SMEM, c->stream>>>(
        c->g, it, c->crec, c->cs_xm, c->d_cs_m1, c->tarr, c->sbuf, c->cy, c->ctl, c->coef,
        c->tune, ca.c_lo, ca.first_c, ca.a_lo, ca.check_stop, ca.disc_lo, ca.disc_hi);
  } else {
    k_cam_pipe<S, HC, HA, false><<<c->pipe_W / PW, PW * 32, PIPE_SMEM, c->stream>>>(
        c->g, it, c->crec, c->cs_x, g_null_d, c->tarr, c->sbuf, c->cy, c->ctl, c->coef, c->tune,
        ca.c_lo, ca.first_c, ca.a_lo, ca.check_stop, ca.disc_lo, ca.disc_hi);
  }
  c->launched();
}

// ca.disc_lo = landmark block whose partials s were consumed by the preceding landmark
// reduce (dropped from L2 at the start of this kernel), -1 for none
template <int S, bool HC, int EP, bool HA>
static void launch_cam(pv_ctx* c, const CamArgs& ca0) {
  CamArgs ca = ca0;
  const int db = ca.disc_lo;
  ca.disc_lo = ca.disc_hi = 0;
  // never drop lines this kernel itself writes (its W^T v pass scatters into blocks [a_lo, a_hi))
  const bool writes_db = HA && db >= ca.a_lo && db < ca.a_hi;
  if (db >= 0 && db < c->n_blk && c->tune.discard_s && !writes_db) {
    ca.disc_lo = c->blk_s[db];
    ca.disc_hi = c->blk_s[db + 1];
  }
  // the persistent kernel runs one warp per camera: with wpc == 1 it reproduces k_cam's
  // summation order bit for bit, so every path (fused, sharded, blocked) stays consistent
  if (EP == EP_NONE && c->tune.cam_pipe && c->wpc == 1 && !ca.project_y &&
      (!HC || ca.c_hi == ca.c_lo + 1) && (!HA || ca.a_hi == ca.a_lo + 1) &&
      (!(HC && HA) || ca.a_lo == ca.c_lo + 1)) {  // the paired W^T v lists assume block b + 1
    launch_cam_pipe<S, HC, HA>(c, ca);
    return;
  }
  launch_cam_v<S, HC, EP, HA>(c, ca);
}

// landmark half of a term over the landmark blocks [b_lo, b_hi)
template <int S, int MODE>
static void launch_lm_reduce(pv_ctx* c, int b_lo, int b_hi, int check_stop) {
  const int k_lo = c->blk_ktask[b_lo], k_hi = c->blk_ktask[b_hi];
  const int nb = blocks_for((long long)(k_hi - k_lo) * 32, 256);  // one task per warp
  k_lm_reduce<S, MODE><<<nb, 256, 0, c->stream>>>(c->d_klist, c->use_kslot ? c->d_kslot : nullptr, c->sbuf, c->lrec,
                                                  c->tarr, c->lsys, c->lbl, c->ldl, c->tlm,
                                                  c->ctl, c->flags, c->tune, k_lo, k_hi,
                                                  check_stop);
  c->launched();
}

static CamArgs cam_args(int c_lo, int c_hi, int first_c, int a_lo, int a_hi, int term,
                        double thr, int check_stop) {
  CamArgs a{};
  a.c_lo = c_lo;
  a.c_hi = c_hi;
  a.first_c = first_c;
  a.a_lo = a_lo;
  a.a_hi = a_hi;
  a.term = term;
  a.check_stop = check_stop;
  a.project_y = 0;
  a.wpc = 1;
  a.thr = thr;
  // a W t pass over one block follows that block's landmark reduce: its s is consumed
  a.disc_lo = c_hi == c_lo + 1 ? c_lo : -1;
  a.disc_hi = 0;
  return a;
}

// finish y over blocks [c_lo, c_hi) (if any), the epilogue, and the gather of block 0
template <int S, int EP>
static void launch_cam_last(pv_ctx* c, int c_lo, int c_hi, int first_c, int term, double thr,
                            int check_stop, unsigned long long cond = 0, int max_order = 0) {
  auto ep_args = [&](CamArgs a) {  // the epilogue launch carries the term-graph condition
    a.cond = cond;
    a.max_order = max_order;
    return a;
  };
  if (!c->collective() && c->tune.split_last && c->wpc == 1) {
    // one warp per camera: the W t pass on the pipelined kernel (a single block) or on k_cam
    // together with the epilogue (all blocks, the RHS), the epilogue alone (U^-1, x, v,
    // norms, stop test), then the next W^T v pass of block 0 on the pipelined kernel
    if (c_hi == c_lo + 1) {
      launch_cam<S, true, EP_NONE, false>(
          c, cam_args(c_lo, c_hi, first_c, 0, 0, term, thr, check_stop));
      launch_cam<S, false, EP, false>(c, ep_args(cam_args(0, 0, 0, 0, 0, term, thr, check_stop)));
    } else {
      launch_cam<S, true, EP, false>(c, ep_args(cam_args(c_lo, c_hi, first_c, 0, 0, term, thr, check_stop)));
    }
    if (!c->skip_next_gather)
      launch_cam<S, false, EP_NONE, true>(c, cam_args(0, 0, 0, 0, 1, term, thr, 1));
  } else if (!c->collective()) {
    launch_cam<S, true, EP, true>(c, ep_args(cam_args(c_lo, c_hi, first_c, 0, 1, term, thr, check_stop)));
  } else {
    launch_cam<S, true, EP_NONE, false>(c,
                                        cam_args(c_lo, c_hi, first_c, 0, 0, term, thr, check_stop));
    c->allreduce(c->cy, (size_t)c->n_p * 12);
    launch_cam<S, false, EP, true>(c, ep_args(cam_args(0, 0, 0, 0, 1, term, thr, check_stop)));
  }
}

// one power-series term i >= 1 (s of block 0 already scattered by the previous kernel)
template <int S>
static void launch_term(pv_ctx* c, int i, double thr, unsigned long long cond = 0,
                        int max_order = 0) {
  const int B = c->n_blk;
  // Launched ahead by the host loop, a term's kernels return at once when an earlier term
  // took the stop (one load of the control block at the head of every kernel).  Inside the
  // term graph the body only runs while the series continues, so that load -- an L2 round
  // trip in front of each of the 2 B + 2 kernels -- is dropped; only the next term's first
  // W^T v pass, which follows the stop decision inside the same body, keeps it.
  const int cs = cond ? 0 : 1;
  for (int b = 0; b < B; ++b) {
    launch_lm_reduce<S, LR_TERM>(c, b, b + 1, cs);
    if (b + 1 < B)
      launch_cam<S, true, EP_NONE, true>(c, cam_args(b, b + 1, b == 0, b + 1, b + 2, i, thr, cs));
    else
      launch_cam_last<S, EP_TERM>(c, b, b + 1, b == 0, i, thr, cs, cond, max_order);
  }
}

// The term loop as ONE CUDA graph: a WHILE conditional node whose body is one term (its
// kernels captured once, the term index read from the control block); the epilogue kernel
// of each term sets the condition (continue while not stopped and term < max_order), so the
// whole series runs with no host round trip per term (solvers.py:140-149).  Cached per
// configuration; single-process contexts only (the loopback group synchronizes on the
// host between ranks, which a graph cannot).
template <int S>
static TermGraph& term_graph(pv_ctx* c, int max_order, double thr) {
  TermGraph& G = c->tgraph;
  const int xm = c->xm_ok ? 1 : 0;
  if (G.exec && G.stage == S && G.max_order == max_order && G.thr == thr && G.n_blk == c->n_blk &&
      G.wpc == c->wpc && G.xm == xm && G.coll == c->collective() &&
      G.layout_gen == c->layout_gen &&
      std::memcmp(&G.tune, &c->tune, sizeof(Tune)) == 0)
    return G;
  if (G.exec) cudaGraphExecDestroy(G.exec);
  if (G.graph) cudaGraphDestroy(G.graph);
  G = TermGraph{};
  CK(cudaGraphCreate(&G.graph, 0));
  cudaGraphConditionalHandle handle;
  CK(cudaGraphConditionalHandleCreate(&handle, G.graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np{};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = handle;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, G.graph, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  const long long l0 = c->launches;
  CK(cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeRelaxed));
  launch_term<S>(c, -1, thr, (unsigned long long)handle, max_order);
  cudaGraph_t captured = nullptr;
  CK(cudaStreamEndCapture(c->stream, &captured));
  G.body_launches = c->launches - l0;
  c->launches = l0;  // counted per executed term instead (op_power)
  CK(cudaGraphInstantiate(&G.exec, G.graph, 0));
  G.stage = S;
  G.max_order = max_order;
  G.thr = thr;
  G.n_blk = c->n_blk;
  G.wpc = c->wpc;
  G.xm = xm;
  G.layout_gen = c->layout_gen;
  G.tune = c->tune;
  G.coll = c->collective();
  return G;
}

// The whole term loop as one persistent cooperative kernel (pv_series.cuh): single-process
// contexts with one warp per camera (the configuration the pipelined camera kernel covers).
static bool series_ok(const pv_ctx* c) {
  return c->tune.series && c->tune.cam_pipe && c->wpc == 1 && !c->collective();
}
template <int S>
static void launch_series(pv_ctx* c, int max_order, double thr) {
  const bool xm = S == 1 && c->xm_ok && c->tune.xm;
  SeriesArgs a{};
  a.item = c->d_items;
  a.off = c->d_item_off;
  a.rslot = c->d_rslot;
  a.roff = c->d_roff;
  a.B = c->n_blk;
  a.W = c->pipe_W;
  a.klist = c->d_klist;
  a.crec = c->crec;
  a.cs_x = xm ? c->cs_xm : c->cs_x;
  a.cs_m1 = xm ? c->d_cs_m1 : g_null_d;
  a.tarr = c->tarr;
  a.sbuf = c->sbuf;
  a.cy = c->cy;
  a.lsys = c->lsys;
  a.lrec = c->lrec;
  a.cUi = c->cUi;
  a.cx = c->cx;
  a.ch = c->ch;
  a.nrm = c->nrm;
  a.ctl = c->ctl;
  a.bar = c->sbar;
  a.max_order = max_order;
  a.thr = thr;
  CK(cudaMemsetAsync(c->sbar, 0, 4 * sizeof(unsigned), c->stream));
  void* args[] = {(void*)&c->g, (void*)&a, (void*)&c->coef, (void*)&c->tune};
  const void* fn = (const void*)k_series<S, false>;
  if constexpr (S == 1) {
    if (xm) fn = (const void*)k_series<1, true>;
  }
  CK(cudaLaunchCooperativeKernel(fn, dim3(c->pipe_W / PW), dim3(PW * 32), args, PIPE_SMEM,
                                 c->stream));
  c->launched();
}

template <int S>
static bool rhs_reusable(const pv_ctx* c) {
  return S == 1 && !c->last_damp_both && c->rhs_lin_id == c->lin_id && c->tune.rhs_reuse;
}
template <int S>
static void mark_rhs(pv_ctx* c) {
  c->rhs_lin_id = (S == 1 && !c->last_damp_both) ? c->lin_id : -1;
}

// K7: dl = -V+ (b_l + W^T x) (zero for degenerate blocks) and the trial landmarks, with
// v = x (the pose update in cx), block by block so that each block's s stays in L2
// (back_substitute, normal_eq.py:239-250)
template <int S>
static void back_substitute_launches(pv_ctx* c);

// The 2 B + 1 launches of the back-substitution replayed as one CUDA graph (single-rank
// contexts, PV_OPT_GRAPH): no control flow, only the launch gaps of a stream are saved.
template <int S>
static void back_substitute_dev(pv_ctx* c) {
  if (!(c->tune.graph && !c->loop && c->world == 1)) {
    back_substitute_launches<S>(c);
    return;
  }
  TermGraph& G = c->bsgraph;
  const int xm = c->xm_ok ? 1 : 0;
  if (!(G.exec && G.stage == S && G.n_blk == c->n_blk && G.wpc == c->wpc && G.xm == xm &&
        G.coll == c->collective() && G.layout_gen == c->layout_gen &&
        std::memcmp(&G.tune, &c->tune, sizeof(Tune)) == 0)) {
    if (G.exec) cudaGraphExecDestroy(G.exec);
    if (G.graph) cudaGraphDestroy(G.graph);
    G = TermGraph{};
    const long long l0 = c->launches;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
    back_substitute_launches<S>(c);
    CK(cudaStreamEndCapture(c->stream, &G.graph));
    G.body_launches = c->launches - l0;
    c->launches = l0;
    CK(cudaGraphInstantiate(&G.exec, G.graph, 0));
    G.stage = S;
    G.n_blk = c->n_blk;
    G.wpc = c->wpc;
    G.xm = xm;
    G.layout_gen = c->layout_gen;
    G.tune = c->tune;
    G.coll = c->collective();
  }
  CK(cudaGraphLaunch(G.exec, c->stream));
  c->launches += G.body_launches;
}

template <int S>
static void back_substitute_launches(pv_ctx* c) {
  k_setv<S><<<blocks_for(c->n_p, 128), 128, 0, c->stream>>>((int)c->n_p, c->cx, c->ch, c->crec);
  c->launched();
  for (int b = 0; b < c->n_blk; ++b) {
    CamArgs a = cam_args(0, 0, 0, b, b + 1, 0, 0.0, 0);
    a.disc_lo = b - 1;  // consumed by the previous block's back-substitution
    launch_cam<S, false, EP_NONE, true>(c, a);
    launch_lm_reduce<S, LR_BACKSUB>(c, b, b + 1, 0);
  }
  c->check_launch();
}

template <int S>
static void op_power(pv_ctx* c, int max_order, double thr, int* order, double* trunc) {
  CK(cudaMemsetAsync(c->ctl, 0, sizeof(PowerCtl), c->stream));
  CK(cudaMemsetAsync(c->flags + F_ZERO_NORM, 0, sizeof(int), c->stream));
  c->sync();
  std::memset(c->host_ctl, 0, sizeof(PowerCtl));
  CK(cudaEventRecord(c->tev[0], c->stream));
  // K4: t = V+ b_l for all landmarks, then y = W t over all blocks, the reduced RHS,
  // t_0 = U^-1 rhs and the gather of block 0 (a single pass; blocking does not pay here)
  const int B = c->n_blk;
  const bool series = series_ok(c) && max_order > 0;
  c->skip_next_gather = series;
  if (rhs_reusable<S>(c)) {  // t_0 = U^-1 rhs from the stored RHS, then block 0's gather
    if (!c->collective() && c->tune.split_last && c->wpc == 1) {
      launch_cam<S, false, EP_RHS_CACHED, false>(c, cam_args(0, 0, 0, 0, 0, 0, thr, 0));
      if (!c->skip_next_gather)
        launch_cam<S, false, EP_NONE, true>(c, cam_args(0, 0, 0, 0, 1, 0, thr, 0));
    } else {
      launch_cam<S, false, EP_RHS_CACHED, true>(c, cam_args(0, 0, 0, 0, 1, 0, thr, 0));
    }
  } else {
    launch_lm_reduce<S, LR_RHS>(c, 0, c->n_blk, 0);
    launch_cam_last<S, EP_RHS>(c, 0, B, 1, 0, thr, 0);
    mark_rhs<S>(c);
  }
  c->skip_next_gather = false;
  c->check_launch();
  CK(cudaEventRecord(c->tev[1], c->stream));
  int launched_terms = 0;
  // the device-driven term loop: single-rank contexts (with world > 1 the host look-ahead
  // loop below drives the terms, an NCCL call between kernels: a multi-rank collective inside
  // a conditional graph body has never been executed on this 1-GPU pool)
  if (series || (c->tune.graph && !c->loop && c->world == 1 && max_order > 0)) {
    long long body_launches = 0;
    if (series) {
      launch_series<S>(c, max_order, thr);
    } else {
      TermGraph& G = term_graph<S>(c, max_order, thr);
      CK(cudaGraphLaunch(G.exec, c->stream));
      body_launches = G.body_launches;
    }
    CK(cudaEventRecord(c->tev[2], c->stream));
    back_substitute_dev<S>(c);
    CK(cudaEventRecord(c->tev[3], c->stream));
    PowerCtl h;
    CK(cudaMemcpyAsync(&h, c->ctl, sizeof(PowerCtl), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    c->launches += body_launches * h.term;  // kernels of the executed terms
    *order = h.order;
    *trunc = h.trunc;
    c->step_stage = S;
    for (int q = 0; q < 3; ++q) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->tev[q], c->tev[q + 1]));
      c->solve_us[q] = (int64_t)(1000.0 * ms);
    }
    c->solve_terms_launched = h.term;
    return;
  }
  // K5 + K6 terms with a one-term lookahead on the device stop flag.  The decision to stop
  // launching must be the same on every rank (each launch of a term holds collectives):
  // after term i-1 is known complete, stop only on a stop taken AT a term <= i-1 -- a faster
  // rank may already see the stop of the in-flight term i, and must not act on it earlier
  // than the others (the loopback test caught exactly that divergence).
  for (int i = 1; i <= max_order; ++i) {
    launch_term<S>(c, i, thr);
    ++launched_terms;
    CK(cudaEventRecord(c->ev[i & 1], c->stream));
    if (i >= 2) {
      CK(cudaEventSynchronize(c->ev[(i - 1) & 1]));
      const volatile PowerCtl* h = c->host_ctl;
      if (h->stopped && h->term <= i - 1) break;
    }
  }
  c->check_launch();
  CK(cudaEventRecord(c->tev[2], c->stream));
  back_substitute_dev<S>(c);
  CK(cudaEventRecord(c->tev[3], c->stream));
  PowerCtl h;
  CK(cudaMemcpyAsync(&h, c->ctl, sizeof(PowerCtl), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  *order = h.order;
  *trunc = h.trunc;
  c->step_stage = S;
  for (int q = 0; q < 3; ++q) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->tev[q], c->tev[q + 1]));
    c->solve_us[q] = (int64_t)(1000.0 * ms);
  }
  c->solve_terms_launched = launched_terms;
}

// K5 as apply_schur inside block-Jacobi PCG (solvers.py:153-187)
template <int S>
static void op_pcg(pv_ctx* c, int max_it, double tol, int* its, double* rel, int* flag) {
  const int D = S == 1 ? 12 : 11;
  const size_t np = c->n_p;
  if (!c->cmom) {
    c->cmom = c->alloc<double>(np * 60);
    c->csd = c->alloc<double>(np * 144);
    c->csdd = c->alloc<double>(np * 144);
    c->cmi = c->alloc<double>(np * 144);
    c->pvec = c->alloc<double>(np * 12 * 4);
    c->ppart = c->alloc<double>(np * 2);
  }
  PcgVec v{c->cx, c->pvec, c->pvec + np * 12, c->pvec + np * 24, c->pvec + np * 36};
  const int B = c->n_blk;
  const int wg = blocks_for((long long)np * 32, 256);  // one warp per camera
  CK(cudaMemsetAsync(c->flags + F_SINGULAR_M, 0, 2 * sizeof(int), c->stream));
  // a collapsed norm of an earlier trial must not leak into this solve (op_power does the same)
  CK(cudaMemsetAsync(c->flags + F_ZERO_NORM, 0, sizeof(int), c->stream));
  // K4: the reduced RHS (its U^-1 epilogue output is unused here)
  if (!rhs_reusable<S>(c)) {
    launch_lm_reduce<S, LR_RHS>(c, 0, c->n_blk, 0);
    launch_cam_last<S, EP_RHS>(c, 0, B, 1, 0, 0.0, 0);
    mark_rhs<S>(c);
  }
  // preconditioner: exact block diagonal and its inverse (solvers.py:161-166)
  k_schur_diag<S><<<wg, 256, 0, c->stream>>>(c->g, c->crec, c->cs_x, c->lsys, c->cmom, c->coef);
  c->launched();
  c->check_launch();
  c->allreduce(c->cmom, np * 60);
  k_diag_finish<S><<<wg, 256, 0, c->stream>>>((int)np, c->cmom, c->ch, c->cUd, c->csd);
  k_damp_cam<<<blocks_for(np * 32, 128), 128, 0, c->stream>>>((int)np, D, c->csd, 0.0, c->csdd, c->cmi,
                                                       c->flags + (F_SINGULAR_M - F_SINGULAR_U));
  c->launched(2);
  c->check_launch();
  int fl[F_COUNT];
  CK(cudaMemcpyAsync(fl, c->flags, sizeof(fl), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (fl[F_SINGULAR_M]) {  // not positive definite: general inverse, then pinv
    k_inv_lu<<<blocks_for(np, 32), 32, 0, c->stream>>>((int)np, D, c->csd, c->cmi, c->flags);
    c->launched();
    CK(cudaMemcpyAsync(fl, c->flags, sizeof(fl), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (fl[F_SINGULAR_M2]) {
      k_pinv_jacobi<<<blocks_for(np, 32), 32, 0, c->stream>>>((int)np, D, c->csd, c->cmi);
      c->launched();
    }
    c->check_launch();
  }
  k_pcg_init<S><<<wg, 256, 0, c->stream>>>((int)np, c->crhs, c->cmi, c->ch, c->crec, v, c->ppart,
                                           c->ctl, c->host_ctl_dev, c->ticket);
  c->launched();
  c->check_launch();
  c->sync();
  // iterations with a one-iteration look-ahead on the device stop flag; as in op_power the
  // host acts only on a stop taken at an iteration known complete (rank-consistent)
  const bool stopped0 = ((volatile PowerCtl*)c->host_ctl)->stopped != 0;  // after the sync
  // one iteration: the blocked S'.p (the term kernels, launched ahead of the stop flag) and the
  // three vector kernels; `it` < 0: the iteration count is kept on the device
  auto launch_iteration = [&](int it) {
    launch_cam<S, false, EP_NONE, true>(c, cam_args(0, 0, 0, 0, 1, 0, 0.0, 1));
    for (int b = 0; b < B; ++b) {
      launch_lm_reduce<S, LR_TERM>(c, b, b + 1, 1);
      if (b + 1 < B)
        launch_cam<S, true, EP_NONE, true>(c, cam_args(b, b + 1, b == 0, b + 1, b + 2, 0, 0.0, 1));
      else
        launch_cam<S, true, EP_NONE, false>(c, cam_args(b, b + 1, b == 0, 0, 0, 0, 0.0, 1));
    }
    c->allreduce(c->cy, np * 12);
    k_pcg_curv<S><<<wg, 256, 0, c->stream>>>((int)np, it, c->cy, c->ch, c->cUd, v, c->ppart,
                                             c->ctl, c->host_ctl_dev, c->ticket);
    k_pcg_update<S><<<wg, 256, 0, c->stream>>>((int)np, tol, c->cmi, v, c->ppart, c->ctl,
                                               c->host_ctl_dev, c->ticket);
    k_pcg_dir<S><<<wg, 256, 0, c->stream>>>((int)np, c->ch, c->crec, v, c->ctl);
    c->launched(3);
  };
  // single-rank contexts replay the iteration as a captured graph (PV_OPT_GRAPH): the same
  // kernels without a stream's launch gaps; the host look-ahead loop stays
  TermGraph* PG = nullptr;
  if (c->tune.graph && !c->loop && c->world == 1 && !stopped0 && max_it > 0) {
    TermGraph& G = c->pcggraph;
    const int xm = c->xm_ok ? 1 : 0;
    if (!(G.exec && G.stage == S && G.thr == tol && G.n_blk == c->n_blk && G.wpc == c->wpc &&
          G.xm == xm && G.coll == c->collective() && G.layout_gen == c->layout_gen &&
          std::memcmp(&G.tune, &c->tune, sizeof(Tune)) == 0)) {
      if (G.exec) cudaGraphExecDestroy(G.exec);
      if (G.graph) cudaGraphDestroy(G.graph);
      G = TermGraph{};
      const long long l0 = c->launches;
      CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
      launch_iteration(-1);
      CK(cudaStreamEndCapture(c->stream, &G.graph));
      G.body_launches = c->launches - l0;
      c->launches = l0;
      CK(cudaGraphInstantiate(&G.exec, G.graph, 0));
      G.stage = S;
      G.thr = tol;
      G.n_blk = c->n_blk;
      G.wpc = c->wpc;
      G.xm = xm;
      G.layout_gen = c->layout_gen;
      G.tune = c->tune;
      G.coll = c->collective();
    }
    PG = &G;
  }
  for (int it = 1; it <= max_it && !stopped0; ++it) {
    if (PG) {
      CK(cudaGraphLaunch(PG->exec, c->stream));
      c->launches += PG->body_launches;
    } else {
      launch_iteration(it);
    }
    CK(cudaEventRecord(c->ev[it & 1], c->stream));
    if (it >= 2) {
      CK(cudaEventSynchronize(c->ev[(it - 1) & 1]));
      const volatile PowerCtl* h = c->host_ctl;
      if (h->stopped && h->order <= it - 1) break;
    }
  }
  c->check_launch();
  back_substitute_dev<S>(c);
  PowerCtl h;
  CK(cudaMemcpyAsync(&h, c->ctl, sizeof(PowerCtl), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  *its = h.order;
  *rel = h.trunc;
  *flag = h.pad;
  c->step_stage = S;
}

template <int S>
static void op_trial(pv_ctx* c, int* ok) {
  k_trial_cam<S><<<blocks_for(c->n_p, 128), 128, 0, c->stream>>>((int)c->n_p, c->crec, c->cx,
                                                                  c->ch, c->tcam, c->flags);
  c->launched();
  c->check_launch();
  c->allreduce_flags();
  int fl[F_COUNT];
  CK(cudaMemcpyAsync(fl, c->flags, sizeof(fl), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  *ok = fl[F_ZERO_NORM] ? 0 : 1;
}

static void op_resolve_trial(pv_ctx* c, double* f_new, int64_t* n_rd) {
  CK(cudaMemsetAsync(c->flags + F_N_RANKDEF, 0, 2 * sizeof(int), c->stream));
  if (c->tune.resolve_slots) {
    const int ns = c->blk_ktask[c->n_blk];  // every landmark block's slots, in order
    k_resolve_slots<<<blocks_for((long long)ns * 32, 256), 256, 0, c->stream>>>(
        c->g, c->d_klist, ns, c->tcam, c->tlm, c->cpart, c->flags, c->coef, c->lvr, c->lbl);
    c->launched();
    c->sum_partials(ns);
  } else {
    k_resolve<<<blocks_for((long long)c->n_tasks * 32, 64), 64, 0, c->stream>>>(
        c->g, c->tcam, c->tlm, c->cpart, c->flags, c->coef, c->lvr, c->lbl);
    c->launched();
    c->sum_partials();
  }
  c->check_launch();
  c->allreduce(c->scal, 1);
  c->allreduce_flags();
  double v;
  int fl[F_COUNT];
  CK(cudaMemcpyAsync(&v, c->scal, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(fl, c->flags, sizeof(fl), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (f_new) *f_new = v;
  if (n_rd) *n_rd = fl[F_N_RANKDEF];
  c->last_fallbacks = fl[F_N_FALLBACK];
}

static void op_accept(pv_ctx* c, bool lm_lin_fresh = false) {
  const int n = (int)std::max<int64_t>(c->n_p, c->n_ls);
  k_accept<<<blocks_for(n, 256), 256, 0, c->stream>>>((int)c->n_p, c->n_ls, c->tcam, c->tlm,
                                                      c->crec, c->lrec);
  c->launched();
  c->check_launch();
  c->lin_stage = 0;
  c->vp_cached = false;
  c->lm_lin_fresh = lm_lin_fresh;  // the re-solve already produced V, b_l at this state
}

// ---------------------------------------------------------------------------
// C-ABI

#define API_BEGIN(ctx) \
  if (!(ctx)) return PV_EINVAL; \
  try {
#define API_END(ctx)                              \
  }                                               \
  catch (const PvError& e) {                      \
    (ctx)->err = e.what();                        \
    return e.code;                                \
  }                                               \
  catch (const std::exception& e) {               \
    (ctx)->err = e.what();                        \
    return PV_ECUDA;                              \
  }                                               \
  return PV_OK;

#define STAGE_DISPATCH(stage, fn, ...)                                          \
  ((stage) == 1 ? fn<1>(__VA_ARGS__)                                            \
                : ((stage) == 2 ? fn<2>(__VA_ARGS__)                            \
                                : throw PvError(PV_EINVAL, "stage must be 1 or 2")))

extern "C" {

int pv_loopback_id(int world, unsigned char out[128]) {
  if (world < 1 || !out) return PV_EINVAL;
  LoopGroup* G = new LoopGroup();  // lives for the process (a test / single-node utility)
  G->world = world;
  G->bufs.assign(world, nullptr);
  G->ready.assign(world, nullptr);
  G->done.assign(world, nullptr);
  std::memset(out, 0, 128);
  const uint64_t magic = LoopGroup::MAGIC;
  std::memcpy(out, &magic, sizeof(magic));
  std::memcpy(out + 8, &G, sizeof(G));
  return PV_OK;
}

int pv_nccl_unique_id(unsigned char out[128]) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return PV_ENCCL;
  static_assert(sizeof(id) == 128, "nccl id size");
  std::memcpy(out, &id, 128);
  return PV_OK;
}

int pv_create(pv_ctx** out, int device, int rank, int world, const unsigned char* nccl_id,
              int64_t n_cameras, int64_t n_landmarks, int64_t n_obs, const int64_t* cam_idx,
              const int64_t* lm_idx, const double* meas, int64_t lm_begin, int64_t lm_end,
              double eta) {
  g_create_error.clear();
  if (!out) return PV_EINVAL;
  *out = nullptr;
  pv_ctx* c = new pv_ctx();
  try {
    if (n_cameras < 0 || n_landmarks < 0 || n_obs < 0 || world < 1 || rank < 0 ||
        rank >= world || lm_begin < 0 || lm_end > n_landmarks || lm_begin > lm_end)
      throw PvError(PV_EINVAL, "invalid sizes or shard range");
    if (n_cameras >= INT32_MAX || n_landmarks >= INT32_MAX)
      throw PvError(PV_EINVAL, "problem too large for int32 indexing");
    if (!(eta >= 0.0 && eta <= 1.0)) throw PvError(PV_EINVAL, "eta must lie in [0, 1]");
    if (n_obs > 0 && (!cam_idx || !lm_idx || !meas)) throw PvError(PV_EINVAL, "null arrays");
    for (int64_t o = 0; o < n_obs; ++o) {
      if (cam_idx[o] < 0 || cam_idx[o] >= n_cameras)
        throw PvError(PV_EINVAL, "camera index out of range");
      if (lm_idx[o] < 0 || lm_idx[o] >= n_landmarks)
        throw PvError(PV_EINVAL, "landmark index out of range");
    }
    c->device = device;
    c->rank = rank;
    c->world = world;
    c->n_p = n_cameras;
    c->n_l_global = n_landmarks;
    c->n_o_global = n_obs;
    c->coef.s1 = std::sqrt(1.0 - eta);
    c->coef.s2 = std::sqrt(eta);
    c->coef.s = 1.0 - eta;
    CK(cudaSetDevice(device));
    {
      // evict_last (L2::cache_hint) lines live in the persisting L2 carve-out, which
      // defaults to 0 bytes: reserve the maximum so a landmark block's partials stay on chip
      int max_persist = 0;
      CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device));
      size_t cur = 0;
      CK(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
      if (cur < (size_t)max_persist)
        CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist));
      c->persist_l2 = max_persist;
    }
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    for (auto& e : c->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : c->tev) CK(cudaEventCreate(&e));
    if (world > 1) {
      if (!nccl_id) throw PvError(PV_EINVAL, "nccl id required for world > 1");
      uint64_t magic = 0;
      std::memcpy(&magic, nccl_id, sizeof(magic));
      if (magic == LoopGroup::MAGIC) {  // in-process loopback (pv_loopback_id)
        LoopGroup* G = nullptr;
        std::memcpy(&G, nccl_id + 8, sizeof(G));
        if (!G || G->world != world) throw PvError(PV_EINVAL, "loopback group size mismatch");
        c->loop = G;
        {
          std::lock_guard<std::mutex> lk(G->m);
          if (!G->ready[rank]) {
            CK(cudaEventCreateWithFlags(&G->ready[rank], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&G->done[rank], cudaEventDisableTiming));
          }
          ++G->members;
        }
        c->loop_tmp = c->alloc<double>((size_t)std::max<int64_t>(n_cameras, 1) * 144);
        c->loop_ptrs = c->alloc<void*>(world);
      } else {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        NK(ncclCommInitRank(&c->comm, world, id, rank));
      }
    }
    const bool dbg = std::getenv("PV_DEBUG_SETUP") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    const auto t0 = now();
    build_graph(c, cam_idx, lm_idx, meas, lm_begin, lm_end);
    const auto t1 = now();
    build_blocks(c);
    const auto t2 = now();
    alloc_buffers(c);
    c->sync();
    if (dbg)
      std::fprintf(stderr, "pv_create: build_graph %.0f ms, build_blocks %.0f ms, alloc %.0f ms\n",
                   ms(t0, t1), ms(t1, t2), ms(t2, now()));
  } catch (const std::exception& e) {
    g_create_error = e.what();
    int code = PV_ECUDA;
    if (auto pe = dynamic_cast<const PvError*>(&e)) code = pe->code;
    pv_destroy(c);
    return code;
  }
  *out = c;
  return PV_OK;
}

void pv_destroy(pv_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : c->allocs) cudaFree(p);
  if (c->host_ctl) cudaFreeHost(c->host_ctl);
  for (int i = 0; i < 2; ++i) {
    if (c->stage_pin[i]) cudaFreeHost(c->stage_pin[i]);
    if (c->stage_ev[i]) cudaEventDestroy(c->stage_ev[i]);
  }
  for (auto e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto e : c->tev)
    if (e) cudaEventDestroy(e);
  for (auto e : c->bev)
    if (e) cudaEventDestroy(e);
  if (c->tgraph.exec) cudaGraphExecDestroy(c->tgraph.exec);
  if (c->tgraph.graph) cudaGraphDestroy(c->tgraph.graph);
  if (c->bsgraph.exec) cudaGraphExecDestroy(c->bsgraph.exec);
  if (c->bsgraph.graph) cudaGraphDestroy(c->bsgraph.graph);
  if (c->pcggraph.exec) cudaGraphExecDestroy(c->pcggraph.exec);
  if (c->pcggraph.graph) cudaGraphDestroy(c->pcggraph.graph);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* pv_last_error(pv_ctx* c) { return c ? c->err.c_str() : g_create_error.c_str(); }

void* pv_stream(pv_ctx* c) { return c ? (void*)c->stream : nullptr; }

int pv_info(pv_ctx* c, int64_t* out) {
  API_BEGIN(c)
  std::fill(out, out + PV_INFO_COUNT, 0);
  out[PV_INFO_NP] = c->n_p;
  out[PV_INFO_NL_LOCAL] = c->n_ls;
  out[PV_INFO_NO_LOCAL] = c->n_os;
  out[PV_INFO_TASKS] = c->n_tasks;
  out[PV_INFO_CHUNKS] = c->n_p;
  out[PV_INFO_LAUNCHES] = c->launches;
  out[PV_INFO_RANK] = c->rank;
  out[PV_INFO_WORLD] = c->world;
  out[PV_INFO_DEVICE_BYTES] = (int64_t)c->device_bytes;
  out[PV_INFO_NL_GLOBAL] = c->n_l_global;
  out[PV_INFO_RESOLVE_FALLBACKS] = c->last_fallbacks;
  out[PV_INFO_BLOCKS] = c->n_blk;
  out[PV_INFO_PERSIST_L2] = c->persist_l2;
  out[PV_INFO_WARPS_PER_CAM] = c->wpc;
  out[PV_INFO_SOLVE_RHS_US] = c->solve_us[0];
  out[PV_INFO_SOLVE_TERMS_US] = c->solve_us[1];
  out[PV_INFO_SOLVE_BACKSUB_US] = c->solve_us[2];
  out[PV_INFO_SOLVE_TERMS_LAUNCHED] = c->solve_terms_launched;
  out[PV_INFO_PIPE_WARPS] = c->pipe_W;
  out[PV_INFO_XM_BYTES] = (c->xm_ok && c->tune.xm && c->tune.cam_pipe && c->wpc == 1) ? 40 : 48;
  API_END(c)
}

int pv_set_option(pv_ctx* c, int key, int64_t value) {
  API_BEGIN(c)
  switch (key) {
    case PV_OPT_STAGE_CAP:
      c->tune.stage_cap = (int)value;  // unused by the blocked term (kept for ABI stability)
      break;
    case PV_OPT_POL_STREAM:
      c->tune.pol_stream = (int)value;
      break;
    case PV_OPT_POL_T:
      c->tune.pol_t = (int)value;
      break;
    case PV_OPT_POL_S:
      c->tune.pol_s = (int)value;
      break;
    case PV_OPT_DISCARD_S:
      c->tune.discard_s = (int)value;
      break;
    case PV_OPT_FORCE_COLLECTIVE:
      if (value && !c->comm) {  // 1-rank communicator: same kernels/collectives as world > 1
        if (c->world != 1) throw PvError(PV_EINVAL, "already collective");
        ncclUniqueId id;
        NK(ncclGetUniqueId(&id));
        CK(cudaSetDevice(c->device));
        NK(ncclCommInitRank(&c->comm, 1, id, 0));
      } else if (!value && c->comm && c->world == 1) {
        ncclCommDestroy(c->comm);
        c->comm = nullptr;
      }
      break;
    case PV_OPT_RESOLVE_SLOTS:
      c->tune.resolve_slots = value ? 1 : 0;
      break;
    case PV_OPT_RHS_REUSE:
      c->tune.rhs_reuse = value ? 1 : 0;
      break;
    case PV_OPT_GRAPH:
      c->tune.graph = value ? 1 : 0;
      break;
    case PV_OPT_XM:
      c->tune.xm = value ? 1 : 0;
      break;
    case PV_OPT_BENCH_SPLIT:
      c->bench_split = value ? 1 : 0;
      break;
    case PV_OPT_COST_CS:
      c->tune.cost_cs = value ? 1 : 0;
      break;
    case PV_OPT_SPLIT_LAST:
      c->tune.split_last = value ? 1 : 0;
      break;
    case PV_OPT_CAM_PIPE:
      c->tune.cam_pipe = value ? 1 : 0;
      break;
    case PV_OPT_BALANCE:
    case PV_OPT_BAL_ITEM:
    case PV_OPT_BAL_ROUND:
    case PV_OPT_BAL_LAST:
    case PV_OPT_BAL_RFIX:
    case PV_OPT_BAL_ROBS8:
      if (value < 0 || value > 4096) throw PvError(PV_EINVAL, "balance option out of range");
      (key == PV_OPT_BALANCE ? c->bal_mode : key == PV_OPT_BAL_ITEM ? c->bal_item
       : key == PV_OPT_BAL_ROUND ? c->bal_round : key == PV_OPT_BAL_LAST ? c->bal_last
       : key == PV_OPT_BAL_RFIX ? c->bal_rfix : c->bal_robs8) = (int)value;
      build_pipe_items(c, c->h_seg);
      break;
    case PV_OPT_SERIES:
      c->tune.series = value ? 1 : 0;
      break;
    case PV_OPT_KSLOT:
      c->use_kslot = value ? 1 : 0;
      ++c->layout_gen;  // the term graph captured the kernel argument
      break;
    case PV_OPT_BLOCK_BYTES:
      if (value < 4096) throw PvError(PV_EINVAL, "block budget too small");
      c->block_bytes = value;
      build_blocks(c);
      break;
    default:
      throw PvError(PV_EINVAL, "unknown option");
  }
  API_END(c)
}

// true when this shard's observed landmarks are exactly the contiguous global
// rows lm_gid[0] .. lm_gid[0] + n_ls - 1 (direct host <-> device copies)
static bool lm_contiguous(const pv_ctx* c) {
  return c->n_ls == 0 || c->lm_gid.back() - c->lm_gid.front() + 1 == (int64_t)c->n_ls;
}

// Large transfers between PAGEABLE host memory and the device (the state arrays of
// pv_set_state / pv_get_state: 143 MB at vlarge) go through two pinned staging buffers:
// the DMA of chunk i overlaps the multi-threaded host copy of chunk i -+ 1 (first-touch
// page faults of a fresh destination array included).  cudaMemcpy on pageable memory ran
// at 4.6 GB/s device-to-host and 10.6 GB/s host-to-device here; pinned user memory is
// copied directly.
constexpr size_t STAGE_CHUNK = 8u << 20;
static void par_memcpy(char* dst, const char* src, size_t n) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int T = (int)std::min<size_t>(std::min(8u, std::max(1u, hw / 2)), std::max<size_t>(1, n >> 20));
  if (T <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  std::vector<std::thread> th;
  const size_t part = ((n / T) + 4095) & ~(size_t)4095;
  for (int t = 1; t < T; ++t) {
    const size_t o = std::min(n, part * t), e = std::min(n, part * (t + 1));
    if (e > o) th.emplace_back([=] { std::memcpy(dst + o, src + o, e - o); });
  }
  std::memcpy(dst, src, std::min(n, part));
  for (auto& x : th) x.join();
}
static bool host_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}
static void stage_init(pv_ctx* c) {
  if (c->stage_pin[0]) return;
  for (int i = 0; i < 2; ++i) {
    CK(cudaHostAlloc((void**)&c->stage_pin[i], STAGE_CHUNK, cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&c->stage_ev[i], cudaEventDisableTiming));
  }
}
// synchronous on return
static void copy_d2h(pv_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes < 2 * STAGE_CHUNK || host_pinned(dst)) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    return;
  }
  stage_init(c);
  const size_t nch = (bytes + STAGE_CHUNK - 1) / STAGE_CHUNK;
  for (size_t i = 0; i <= nch; ++i) {
    if (i < nch) {
      const size_t o = i * STAGE_CHUNK, n = std::min(STAGE_CHUNK, bytes - o);
      CK(cudaMemcpyAsync(c->stage_pin[i & 1], (const char*)src + o, n, cudaMemcpyDeviceToHost,
                         c->stream));
      CK(cudaEventRecord(c->stage_ev[i & 1], c->stream));
    }
    if (i > 0) {
      const size_t o = (i - 1) * STAGE_CHUNK, n = std::min(STAGE_CHUNK, bytes - o);
      CK(cudaEventSynchronize(c->stage_ev[(i - 1) & 1]));
      par_memcpy((char*)dst + o, c->stage_pin[(i - 1) & 1], n);
    }
  }
}
static void copy_h2d(pv_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes < 2 * STAGE_CHUNK || host_pinned(src)) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
    c->sync();
    return;
  }
  stage_init(c);
  const size_t nch = (bytes + STAGE_CHUNK - 1) / STAGE_CHUNK;
  for (size_t i = 0; i < nch; ++i) {
    const size_t o = i * STAGE_CHUNK, n = std::min(STAGE_CHUNK, bytes - o);
    if (i >= 2) CK(cudaEventSynchronize(c->stage_ev[i & 1]));  // chunk i - 2 left the buffer
    par_memcpy(c->stage_pin[i & 1], (const char*)src + o, n);
    CK(cudaMemcpyAsync((char*)dst + o, c->stage_pin[i & 1], n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaEventRecord(c->stage_ev[i & 1], c->stream));
  }
  c->sync();
}

int pv_set_state(pv_ctx* c, const double* cams, const double* lms) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpy2DAsync(c->crec, CREC * sizeof(double), cams, 12 * sizeof(double),
                       12 * sizeof(double), c->n_p, cudaMemcpyHostToDevice, c->stream));
  std::vector<double> lm_local;
  if (c->n_ls > 0) {
    const double* src = lms + c->lm_gid.front() * 4;
    if (!lm_contiguous(c)) {
      lm_local.resize((size_t)c->n_ls * 4);
      for (int j = 0; j < c->n_ls; ++j)
        for (int q = 0; q < 4; ++q) lm_local[(size_t)j * 4 + q] = lms[c->lm_gid[j] * 4 + q];
      src = lm_local.data();
    }
    copy_h2d(c, c->lrec, src, sizeof(double) * 4 * c->n_ls);
  }
  c->sync();
  c->lin_stage = 0;
  c->vp_cached = false;
  c->lm_lin_fresh = false;
  API_END(c)
}

static void get_state_impl(pv_ctx* c, const double* dcam, int cstride, const double* dlm,
                           double* cams, double* lms) {
  CK(cudaMemcpy2DAsync(cams, 12 * sizeof(double), dcam, cstride * sizeof(double),
                       12 * sizeof(double), c->n_p, cudaMemcpyDeviceToHost, c->stream));
  if (c->n_ls > 0) {
    if (lm_contiguous(c)) {
      copy_d2h(c, lms + c->lm_gid.front() * 4, dlm, sizeof(double) * 4 * c->n_ls);
    } else {
      std::vector<double> lm_local((size_t)c->n_ls * 4);
      CK(cudaMemcpyAsync(lm_local.data(), dlm, sizeof(double) * lm_local.size(),
                         cudaMemcpyDeviceToHost, c->stream));
      c->sync();
      for (int j = 0; j < c->n_ls; ++j)
        for (int q = 0; q < 4; ++q) lms[c->lm_gid[j] * 4 + q] = lm_local[(size_t)j * 4 + q];
    }
  }
  c->sync();
}

int pv_get_state(pv_ctx* c, double* cams, double* lms) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  get_state_impl(c, c->crec, CREC, c->lrec, cams, lms);
  API_END(c)
}

int pv_get_trial(pv_ctx* c, double* cams, double* lms) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  get_state_impl(c, c->tcam, 12, c->tlm, cams, lms);
  API_END(c)
}

int pv_cost(pv_ctx* c, int stage, int which, double* f) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  if (which != PV_CURRENT && which != PV_TRIAL) throw PvError(PV_EINVAL, "which");
  STAGE_DISPATCH(stage, op_cost, c, which, f);
  API_END(c)
}

int pv_linearize(pv_ctx* c, int stage) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  int rc = STAGE_DISPATCH(stage, op_linearize, c);
  if (rc == PV_EDEGENERATE) c->err = "degenerate projection while linearizing stage 2";
  return rc;
  API_END(c)
}

int pv_damp(pv_ctx* c, double lam, int both, int64_t* n_deg) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  if (!(lam >= 0.0)) throw PvError(PV_EINVAL, "damping must be non-negative");
  if (c->lin_stage == 0) throw PvError(PV_EINVAL, "pv_damp before pv_linearize");
  STAGE_DISPATCH(c->lin_stage, op_damp, c, lam, both, n_deg);
  API_END(c)
}

int pv_power_solve(pv_ctx* c, int max_order, double thr, int* order, double* trunc) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  if (max_order < 0 || !(thr >= 0.0)) throw PvError(PV_EINVAL, "power series settings");
  if (c->lin_stage == 0 || c->damp_lin_id != c->lin_id)
    throw PvError(PV_EINVAL, "pv_power_solve needs pv_linearize + pv_damp first");
  int o = 0;
  double t = 0.0;
  STAGE_DISPATCH(c->lin_stage, op_power, c, max_order, thr, &o, &t);
  if (order) *order = o;
  if (trunc) *trunc = t;
  API_END(c)
}

int pv_pcg_solve(pv_ctx* c, int max_iterations, double tolerance, int* iterations,
                 double* relative_residual, int* flag) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  if (c->lin_stage == 0 || c->damp_lin_id != c->lin_id)
    throw PvError(PV_EINVAL, "pv_pcg_solve needs pv_linearize + pv_damp first");
  if (max_iterations < 0) throw PvError(PV_EINVAL, "max_iterations must be >= 0");
  int its = 0, fl = 0;
  double r = 0.0;
  STAGE_DISPATCH(c->lin_stage, op_pcg, c, max_iterations, tolerance, &its, &r, &fl);
  if (iterations) *iterations = its;
  if (relative_residual) *relative_residual = r;
  if (flag) *flag = fl;
  API_END(c)
}

int pv_trial(pv_ctx* c, int stage, int* ok) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  int k = 0;
  STAGE_DISPATCH(stage, op_trial, c, &k);
  if (ok) *ok = k;
  API_END(c)
}

int pv_accept(pv_ctx* c, int stage, int resolve, double* f_new, int64_t* n_rd) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  if (stage != 1 && stage != 2) throw PvError(PV_EINVAL, "stage");
  if (resolve) {
    if (stage != 1) throw PvError(PV_EINVAL, "landmark re-solve is a stage-1 operation");
    op_resolve_trial(c, f_new, n_rd);
  }
  op_accept(c, resolve != 0);
  c->sync();
  API_END(c)
}

int pv_resolve_current(pv_ctx* c, int64_t* n_rd) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  const int n = (int)std::max<int64_t>(c->n_p, c->n_ls);
  k_get_state<<<blocks_for(n, 256), 256, 0, c->stream>>>((int)c->n_p, c->n_ls, c->crec, c->lrec,
                                                         c->tcam, c->tlm);
  c->launched();
  op_resolve_trial(c, nullptr, n_rd);
  op_accept(c, true);
  c->sync();
  API_END(c)
}

int pv_back_substitute(pv_ctx* c, const double* dx) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  if (c->lin_stage == 0 || c->damp_lin_id != c->lin_id)
    throw PvError(PV_EINVAL, "pv_back_substitute needs pv_linearize + pv_damp first");
  if (!dx) throw PvError(PV_EINVAL, "null pose update");
  const int S = c->lin_stage, D = S == 1 ? 12 : 11;
  std::vector<double> h((size_t)c->n_p * 12, 0.0);
  for (int64_t i = 0; i < c->n_p; ++i)
    for (int q = 0; q < D; ++q) h[i * 12 + q] = dx[i * D + q];
  CK(cudaMemcpyAsync(c->cx, h.data(), h.size() * 8, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(c->flags + F_ZERO_NORM, 0, sizeof(int), c->stream));
  if (S == 1)
    back_substitute_dev<1>(c);
  else
    back_substitute_dev<2>(c);
  c->sync();
  c->step_stage = S;
  API_END(c)
}

int pv_get_step(pv_ctx* c, double* dx, double* dl) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  if (c->step_stage == 0) throw PvError(PV_EINVAL, "no step computed");
  const int D = c->step_stage == 1 ? 12 : 11;
  std::vector<double> x((size_t)c->n_p * 12), l((size_t)c->n_ls * 4);
  CK(cudaMemcpyAsync(x.data(), c->cx, x.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(l.data(), c->ldl, l.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (dx)
    for (int64_t i = 0; i < c->n_p; ++i)
      for (int q = 0; q < D; ++q) dx[i * D + q] = x[i * 12 + q];
  if (dl)
    for (int j = 0; j < c->n_ls; ++j)
      for (int q = 0; q < 3; ++q) dl[c->lm_gid[j] * 3 + q] = l[(size_t)j * 4 + q];
  API_END(c)
}

}  // extern "C"

template <int S>
static void op_schur_apply(pv_ctx* c, const double* v, double* out) {
  const int D = S == 1 ? 12 : 11;
  std::vector<double> h((size_t)c->n_p * 12, 0.0);
  for (int64_t i = 0; i < c->n_p; ++i)
    for (int q = 0; q < D; ++q) h[i * 12 + q] = v[i * D + q];
  CK(cudaMemcpyAsync(c->ctmp, h.data(), h.size() * 8, cudaMemcpyHostToDevice, c->stream));
  k_setv<S><<<blocks_for(c->n_p, 128), 128, 0, c->stream>>>((int)c->n_p, c->ctmp, c->ch, c->crec);
  c->launched();
  launch_cam<S, false, EP_NONE, true>(c, cam_args(0, 0, 0, 0, c->n_blk, 0, 0.0, 0));
  launch_lm_reduce<S, LR_TERM>(c, 0, c->n_blk, 0);
  launch_cam<S, true, EP_NONE, false>(c, cam_args(0, c->n_blk, 1, 0, 0, 0, 0.0, 0));
  c->allreduce(c->cy, (size_t)c->n_p * 12);
  k_project_y<S><<<blocks_for(c->n_p * 32, 256), 256, 0, c->stream>>>((int)c->n_p, c->cy, c->ch,
                                                                     c->cyr);
  c->launched();
  c->check_launch();
  CK(cudaMemcpyAsync(h.data(), c->cyr, h.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  for (int64_t i = 0; i < c->n_p; ++i)
    for (int q = 0; q < D; ++q) out[i * D + q] = h[i * 12 + q];
}


extern "C" {

int pv_schur_apply(pv_ctx* c, int stage, const double* v, double* out) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  if (c->lin_stage != stage) throw PvError(PV_EINVAL, "no linearization of that stage");
  if (c->damp_lin_id != c->lin_id) throw PvError(PV_EINVAL, "pv_damp first");
  STAGE_DISPATCH(stage, op_schur_apply, c, v, out);
  API_END(c)
}

}  // extern "C"

template <int S>
static void op_bench_terms(pv_ctx* c, int n, float* ms) {
  CK(cudaMemsetAsync(c->ctl, 0, sizeof(PowerCtl), c->stream));
  if (series_ok(c) && !c->bench_split && n > 0) {  // n terms inside one series launch
    CK(cudaEventRecord(c->tev[0], c->stream));
    launch_series<S>(c, n, -1.0);
    CK(cudaEventRecord(c->tev[3], c->stream));
    CK(cudaEventSynchronize(c->tev[3]));
    float d;
    CK(cudaEventElapsedTime(&d, c->tev[0], c->tev[3]));
    ms[0] = ms[1] = 0.f;
    ms[2] = (float)c->n_blk;
    ms[3] = d / n;
    return;
  }
  // seed s of block 0 from the current camera vector
  launch_cam<S, false, EP_NONE, true>(c, cam_args(0, 0, 0, 0, 1, 0, 0.0, 0));
  const int B = c->n_blk;
  // events around EVERY launch group of a term: per block the landmark reduce and the
  // camera pass (the last block's camera group = its W t pass, the epilogue and block 0's
  // next W^T v pass)
  if (c->bev.size() < (size_t)(2 * B + 1)) {
    for (auto e : c->bev) cudaEventDestroy(e);
    c->bev.assign(2 * B + 1, nullptr);
    for (auto& e : c->bev) CK(cudaEventCreate(&e));
  }
  double acc[4] = {0, 0, 0, 0};
  auto term = [&](bool per_kernel) {
    for (int b = 0; b < B; ++b) {
      if (per_kernel) CK(cudaEventRecord(c->bev[2 * b], c->stream));
      launch_lm_reduce<S, LR_TERM>(c, b, b + 1, 0);
      if (per_kernel) CK(cudaEventRecord(c->bev[2 * b + 1], c->stream));
      if (b + 1 < B)
        launch_cam<S, true, EP_NONE, true>(c, cam_args(b, b + 1, b == 0, b + 1, b + 2, 1 << 20,
                                                       -1.0, 0));
      else
        launch_cam_last<S, EP_TERM>(c, b, b + 1, b == 0, 1 << 20, -1.0, 0);
    }
    if (per_kernel) CK(cudaEventRecord(c->bev[2 * B], c->stream));
  };
  if (c->bench_split) {
    // diagnostic: the two camera passes on their own -- every block's W^T v pass (HA
    // only), then every block's W t pass (HC only) -- ms[0] / ms[1] per term
    for (int i = 0; i < n; ++i) {
      CK(cudaEventRecord(c->tev[0], c->stream));
      for (int b = 0; b < B; ++b)
        launch_cam<S, false, EP_NONE, true>(c, cam_args(0, 0, 0, b, b + 1, 0, 0.0, 0));
      CK(cudaEventRecord(c->tev[1], c->stream));
      for (int b = 0; b < B; ++b)
        launch_cam<S, true, EP_NONE, false>(c, cam_args(b, b + 1, b == 0, 0, 0, 0, 0.0, 0));
      CK(cudaEventRecord(c->tev[2], c->stream));
      CK(cudaEventSynchronize(c->tev[2]));
      float a, d;
      CK(cudaEventElapsedTime(&a, c->tev[0], c->tev[1]));
      CK(cudaEventElapsedTime(&d, c->tev[1], c->tev[2]));
      acc[0] += a;
      acc[1] += d;
      acc[2] += B;
    }
    for (int q = 0; q < 4; ++q) ms[q] = (float)(acc[q] / std::max(n, 1));
    return;
  }
  for (int i = 0; i < n; ++i) {
    // pass 1: the per-kernel split (the events add small gaps between launches)
    term(true);
    CK(cudaEventSynchronize(c->bev[2 * B]));
    for (int b = 0; b < B; ++b) {
      float a, d;
      CK(cudaEventElapsedTime(&a, c->bev[2 * b], c->bev[2 * b + 1]));
      CK(cudaEventElapsedTime(&d, c->bev[2 * b + 1], c->bev[2 * b + 2]));
      acc[0] += a;
      acc[1] += d;
    }
    acc[2] += B;
    // pass 2: the whole term, back to back with no events inside
    CK(cudaEventRecord(c->tev[0], c->stream));
    term(false);
    CK(cudaEventRecord(c->tev[3], c->stream));
    CK(cudaEventSynchronize(c->tev[3]));
    float d;
    CK(cudaEventElapsedTime(&d, c->tev[0], c->tev[3]));
    acc[3] += d;
  }
  for (int q = 0; q < 4; ++q) ms[q] = (float)(acc[q] / std::max(n, 1));
}


extern "C" {

int pv_bench_terms(pv_ctx* c, int stage, int n, float* ms) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  if (c->lin_stage != stage) throw PvError(PV_EINVAL, "no linearization of that stage");
  STAGE_DISPATCH(stage, op_bench_terms, c, n, ms);
  API_END(c)
}


#ifdef PV_PIPE_TIMING
// diagnostic build only (not part of include/povar.h): per-warp timers of the fused camera
// launch of block `block` in whatever ran last, and the work lists they belong to
int pv_debug_pipe_times(pv_ctx* c, int block, unsigned long long* t /*3*W*/, int* n_items,
                        int4* items /*cap*/, int cap, int* off /*3*B*(W+1)*/) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  c->sync();
  if (t) CK(cudaMemcpyFromSymbol(t, g_pipe_t, sizeof(unsigned long long) * 3 * std::min(c->pipe_W, 8192)));
  CK(cudaMemcpyToSymbol(g_pipe_dbg_block, &block, sizeof(int)));
  const int n = (int)(c->items_bytes / sizeof(int4));
  if (n_items) *n_items = n;
  if (items) CK(cudaMemcpy(items, c->d_items, sizeof(int4) * std::min(n, cap), cudaMemcpyDeviceToHost));
  if (off) CK(cudaMemcpy(off, c->d_item_off, c->item_off_bytes, cudaMemcpyDeviceToHost));
  API_END(c)
}
#endif

#ifdef PV_SER_TIMING
// diagnostic build only: barrier and per-warp timers of k_series (tools/series_times.py)
int pv_debug_series_times(pv_ctx* c, int term, int step, unsigned long long* bar /*64*/,
                          unsigned long long* warp /*3*W*/, int* rslot, int* roff) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  c->sync();
  if (bar) CK(cudaMemcpyFromSymbol(bar, g_ser_bar, sizeof(unsigned long long) * 64));
  if (warp) CK(cudaMemcpyFromSymbol(warp, g_ser_warp, sizeof(unsigned long long) * 3 * std::min(c->pipe_W, 8192)));
  CK(cudaMemcpyToSymbol(g_ser_term, &term, sizeof(int)));
  CK(cudaMemcpyToSymbol(g_ser_step, &step, sizeof(int)));
  if (rslot) CK(cudaMemcpy(rslot, c->d_rslot, c->rslot_bytes, cudaMemcpyDeviceToHost));
  if (roff) CK(cudaMemcpy(roff, c->d_roff, c->roff_bytes, cudaMemcpyDeviceToHost));
  API_END(c)
}
#endif

int pv_debug_get(pv_ctx* c, int which, double* out) {
  API_BEGIN(c)
  CK(cudaSetDevice(c->device));
  auto down = [&](const double* src, size_t n) {
    std::vector<double> h(n);
    CK(cudaMemcpyAsync(h.data(), src, n * 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    return h;
  };
  const size_t np = c->n_p, nl = c->n_ls;
  switch (which) {
    case PV_DBG_U: {
      auto h = down(c->cUd, np * 144);
      std::copy(h.begin(), h.end(), out);
      break;
    }
    case PV_DBG_ULIN: {
      auto h = down(c->cU, np * 144);
      std::copy(h.begin(), h.end(), out);
      break;
    }
    case PV_DBG_UINV: {
      auto h = down(c->cUi, np * 144);
      std::copy(h.begin(), h.end(), out);
      break;
    }
    case PV_DBG_BP: {
      auto h = down(c->cbp, np * 12);
      std::copy(h.begin(), h.end(), out);
      break;
    }
    case PV_DBG_RHS: {
      auto h = down(c->crhs, np * 12);
      std::copy(h.begin(), h.end(), out);
      break;
    }
    case PV_DBG_X: {
      auto h = down(c->cx, np * 12);
      std::copy(h.begin(), h.end(), out);
      break;
    }
    case PV_DBG_V: {
      auto h = down(c->lvr, nl * 8);
      for (size_t j = 0; j < nl; ++j)
        for (int q = 0; q < 6; ++q) out[j * 6 + q] = h[j * 8 + q];
      break;
    }
    case PV_DBG_VPINV:
    case PV_DBG_DEGEN: {
      auto h = down(c->lsys, c->n_kent * LSYS);  // warp-slot order
      for (size_t j = 0; j < nl; ++j) {
        const size_t k = (size_t)c->h_lpos[j] * LSYS;
        if (which == PV_DBG_VPINV)
          for (int q = 0; q < 6; ++q) out[j * 6 + q] = h[k + q];
        else
          out[j] = h[k + 6];
      }
      break;
    }
    case PV_DBG_BL:
    case PV_DBG_DL: {
      auto h = down(which == PV_DBG_BL ? c->lbl : c->ldl, nl * 4);
      for (size_t j = 0; j < nl; ++j)
        for (int q = 0; q < 3; ++q) out[j * 3 + q] = h[j * 4 + q];
      break;
    }
    case PV_DBG_W: {
      if (c->lin_stage == 0) throw PvError(PV_EINVAL, "no linearization");
      double* w = c->alloc<double>((size_t)c->n_os * 36);
      if (c->lin_stage == 1)
        k_debug_w<1><<<blocks_for(nl, 128), 128, 0, c->stream>>>(c->g, c->crec, c->lrec, c->ch, w,
                                                                  c->coef);
      else
        k_debug_w<2><<<blocks_for(nl, 128), 128, 0, c->stream>>>(c->g, c->crec, c->lrec, c->ch, w,
                                                                  c->coef);
      c->launched();
      c->check_launch();
      auto h = down(w, (size_t)c->n_os * 36);
      std::copy(h.begin(), h.end(), out);
      cudaFree(w);
      c->allocs.pop_back();
      c->device_bytes -= std::max<size_t>((size_t)c->n_os * 36, 1) * 8;
      break;
    }
    case PV_DBG_SDIAG:
    case PV_DBG_MINV: {
      if (!c->csd) throw PvError(PV_EINVAL, "no pv_pcg_solve yet");
      auto h = down(which == PV_DBG_SDIAG ? c->csd : c->cmi, np * 144);
      std::copy(h.begin(), h.end(), out);
      break;
    }
    default:
      throw PvError(PV_EINVAL, "unknown debug buffer");
  }
  API_END(c)
}

}  // extern "C"
