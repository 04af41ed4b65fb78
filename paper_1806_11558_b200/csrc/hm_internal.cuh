// hm_internal.cuh — libhm internals shared by the .cu translation units.
// B200 (sm_100a) only.  Built with --fmad=false: no implicit contraction anywhere; FMAs
// appear only where the arithmetic reading writes them (A15) via fma().
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/hm.h"

namespace hm {

constexpr double kInv4Pi = 0.07957747154594767;  // 1/(4 pi), correctly rounded

// One panel in internal (Morton) order; 128 B, one L2 line.
struct __align__(16) Panel {
  double v[9];      // vertices v0, v1, v2 (xyz each)
  double c[3];      // centroid ((v0+v1)+v2)/3
  double area;      // |T|
  double h;         // max edge length
  int32_t vid[3];   // vertex ids (singular-class detection)
  int32_t app;      // application index
};
static_assert(sizeof(Panel) == 128, "Panel must be one 128-B line");

struct Quad { int32_t rlo, rhi, clo, chi; };   // leaf tau x sigma, internal half-open ranges

// Error plumbing -------------------------------------------------------------------------
struct Error {
  hm_status st;
  std::string msg;
};

#define HM_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::hm::Error{e_ == cudaErrorMemoryAllocation ? HM_ERR_OOM : HM_ERR_CUDA,       \
                        std::string(#call) + ": " + cudaGetErrorString(e_)};              \
  } while (0)

#define HM_NCCL(call)                                                                     \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess)                                                                \
      throw ::hm::Error{HM_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)}; \
  } while (0)

// every kernel launch of libhm is followed by HM_CHECK_LAUNCH(), which also counts it
extern unsigned long long g_launches;
#define HM_CHECK_LAUNCH()            \
  do {                               \
    ++::hm::g_launches;              \
    HM_CUDA(cudaGetLastError());     \
  } while (0)

inline void fail(hm_status st, const std::string& m) { throw Error{st, m}; }

// Device buffer (RAII) -------------------------------------------------------------------
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {  // discards contents
    if (count <= n && p) return;
    release();
    size_t bytes = (count ? count : 1) * sizeof(T) + 16;   // +16: bulk-copy tail slack
    HM_CUDA(cudaMalloc(&p, bytes));
    n = count;
  }
  void alloc_exact(size_t count) {
    release();
    alloc(count);
  }
  T* get() const { return p; }
};

// Grow-only pinned host buffer: page-faulted and registered once, reused by every hm_setup,
// and a true DMA source for the plan upload.
template <class T>
struct PinnedVec {
  T* p = nullptr;
  size_t n = 0, cap = 0;
  PinnedVec() = default;
  PinnedVec(const PinnedVec&) = delete;
  PinnedVec& operator=(const PinnedVec&) = delete;
  ~PinnedVec() { if (p) cudaFreeHost(p); }
  void resize(size_t m) {
    if (m > cap) {
      const size_t c = std::max(m, cap + cap / 2);
      T* q = nullptr;
      HM_CUDA(cudaHostAlloc(&q, c * sizeof(T) + 16, cudaHostAllocDefault));
      if (p) { std::memcpy(q, p, n * sizeof(T)); cudaFreeHost(p); }
      p = q;
      cap = c;
    }
    n = m;
  }
  T* data() { return p; }
  const T* data() const { return p; }
  size_t size() const { return n; }
  void clear() { n = 0; }
  T& operator[](size_t i) { return p[i]; }
  const T& operator[](size_t i) const { return p[i]; }
};

// Growable device pool backed by CUDA virtual memory management: one reserved VA range,
// physical 2 MiB granules mapped on demand (no copy on growth).  Holds the ACA factors.
struct VmmPool {
  CUdeviceptr base = 0;
  size_t reserved = 0, mapped = 0, used = 0, gran = 0;
  int device = 0;
  std::vector<CUmemGenericAllocationHandle> handles;
  std::vector<size_t> sizes;
  void init(int dev, size_t max_bytes);
  void ensure(size_t bytes);   // make [0, bytes) mapped
  void release();
  ~VmmPool() { release(); }
};

// matvec plan records (matvec.cu).  A batch is one pipeline stage of k_mv_batched:
//   [header + task records | x_sigma segments | leaf storage], each part 16-B aligned,
// filled by bulk copies (MvSeg) from four bases: 0 dense store, 1 factor pool, 2 the task
// stream (C.mv_tasks), 3 the x vector.
struct MvTask {
  int32_t rlo;              // first internal row of the leaf (y += ...)
  int32_t xoff;             // stage offset (doubles) of x[clo]
  int32_t loff;             // stage offset of the leaf's storage, in doubles (dense leaves) or in
                            // factor elements (low-rank leaves: doubles, or floats with lr_f32)
  uint32_t mnk;             // m | n << 11 | k << 22 (k == 0: dense m x n row-major)
};                          // header record of a batch: {count, 0, 0, 0}
struct MvSeg {              // one bulk copy: [src, src + bytes) of base -> stage offset dst
  int64_t src;              // byte offset (16-B aligned) from the base pointer
  uint16_t bytes;           // multiple of 16
  uint16_t dst;             // byte offset in the stage (16-B aligned)
  uint16_t base;            // 0 dense store, 1 factor pool, 2 task stream, 3 x
  uint16_t pad;
};
struct MvBatch {
  int32_t first_seg, nseg;  // bulk copies filling one stage
  int32_t bytes, count;     // total bytes of the stage (expect_tx), tasks
};
struct MvLarge {
  int32_t rlo, clo, m, n, k, pad;
  int64_t off;              // elements (C.lr_esz bytes) from the factor pool base; dense: doubles of the store
  int64_t toff;             // offset into the t buffer
};
struct MvTileV { int32_t blk, l, j0, j1; };
struct MvTileU { int32_t blk, t0, t1, pad; };

// Persistent scratch of hm_build_tree (grow-only: reused across calls, no allocation churn)
struct TreeWs {
  DBuf<double> cen, area, hh, part, gbox;
  DBuf<double> tcen, tarea, th;   // quads: geometry of the 2N split triangles
  DBuf<uint64_t> code_sorted, ksorted, admk, denk, fk[2];
  DBuf<int32_t> idx, flag, scan;
  DBuf<int2> fr[2];
  DBuf<Quad> admq, denq;
  DBuf<unsigned long long> ctr;
  DBuf<unsigned int> bad;
  DBuf<int64_t> cost, pref, bounds;
  DBuf<unsigned long long> bout;
  DBuf<char> tmp;
};
struct EntryBatchWork;   // entry_batch.cuh
struct PlanWs;           // matvec.cu
struct AcaWork;          // aca.cu

// Timers ----------------------------------------------------------------------------------
struct PhaseTimes {
  double tree_ms = 0, near_ms = 0, aca_ms = 0, plan_ms = 0, setup_ms = 0;
  double tree_phase_ms[6] = {0, 0, 0, 0, 0, 0};   // geometry, morton+sort, cluster, block, leafsort, partition
  double plan_phase_ms[3] = {0, 0, 0};              // items, batches, upload (host)
  double aca_phase_ms[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};   // chunk prep, step loop, of which in sync, store, pre, post,
                                                        // pre up to the budget, budget, pre up to the VA reserve (host)
  double last_matvec_ms = 0, solve_ms = 0;
  int solve_iters = 0;
  double solve_relres = 0;
};

// Per-kernel-family device timing (option "kernel_timing"): CUDA events recorded on the
// launching stream around every launch of a family, resolved at the next synchronous point.
// When the near field runs beside ACA (option setup_overlap) the two evaluation families
// overlap in time; eval_union_ms is the length of the union of their intervals, measured
// against a reference event recorded before the streams fork (mark()).
enum KFam { KF_EVAL_NEAR = 0, KF_EVAL_ACA = 1, KF_ACA_OTHER = 2, KF_MATVEC = 3, KF_KRYLOV = 4, KF_COMM = 5, KF_NUM = 6 };
struct KTimer {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  struct P { int fam; cudaEvent_t a, b; };
  std::vector<P> pend;
  cudaEvent_t ref = nullptr;   // set by mark(): intervals of this batch measured from it
  double ms[KF_NUM] = {0, 0, 0, 0, 0, 0};
  int64_t n[KF_NUM] = {0, 0, 0, 0, 0, 0};
  double eval_union_ms = 0;
  cudaEvent_t get();
  void mark(cudaStream_t st);
  void adopt(KTimer& o);   // move o's pending intervals into this timer (o's thread has joined)
  void resolve();   // caller has synchronised the streams
  void reset();
  ~KTimer();
};

// P2P exchange buffers of the sharded solve (p2p.cu; hm_p2p_export / hm_p2p_import)
constexpr int kMaxPeers = 8;
struct P2PState {
  char* own = nullptr;               // this rank's exchange buffer (cudaMalloc, IPC-exported)
  char* peer[kMaxPeers] = {};        // every rank's buffer mapped into this process (own at rank)
  bool opened[kMaxPeers] = {};
  int64_t F = 0, n_max = 0;          // doubles per vector region; largest N it serves
  unsigned long long ep_ag = 0, ep_rs = 0, ep_ar = 0;   // epochs per collective kind
  bool ready = false;
};

// Context ---------------------------------------------------------------------------------
struct Context {
  int device = 0, rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;
  std::string err;

  // options
  int k_max = 64, solver = 0, restart = 100, max_iter = 10000;
  int record_pivots = -1;      // -1 auto (N <= 25000), 0 off, 1 on
  double aca_chunk_mb = 32768, aca_kws = 16;

  // tree state
  bool have_tree = false, have_setup = false;
  int64_t N = 0, nv = 0;
  int leaf_size = 32;
  double eta = 1.0;
  bool quad = false;           // quadrilateral panels (A25): 2 triangle panels per node
  int64_t npanel = 0;          // triangle panels: N, or 2N for quads (panel 2s+a of node s)
  DBuf<Panel> qnode;           // quads: node panels (v = q0,q1,q2; c, h, area, app of the node)
  DBuf<int4> qv;               // quads: the four vertex ids per node, internal order
  DBuf<Panel> panel;           // internal order
  DBuf<int32_t> perm, iperm;   // perm[s] = app index; iperm[app] = s
  DBuf<uint64_t> codes_app;    // Morton codes, application order
  DBuf<double> vert;           // vertex coordinates (device copy of the mesh)
  DBuf<int32_t> tri;
  // cluster tree (level order)
  int64_t ncl = 0;
  DBuf<int32_t> cl_lo, cl_hi, cl_child, cl_depth;
  DBuf<double> cl_box, cl_diam2;
  // leaves (canonical DFS order)
  int64_t nadm = 0, ndense = 0;
  DBuf<Quad> adm, dense;
  PinnedVec<Quad> h_adm, h_dense;   // host copies of the leaf lists (pinned: fast D2H each setup)
  int64_t adm_begin = 0, adm_end = 0, dense_begin = 0, dense_end = 0;

  // setup state
  double eps_aca = 0;
  DBuf<double> dstore;         // packed dense blocks (owned dense leaves), row-major each
  DBuf<int64_t> doff;          // per owned dense leaf: offset in doubles (+1 sentinel)
  VmmPool fpool;               // packed low-rank factors: per block [U m x k | V n x k], col-major
  DBuf<int64_t> foff;          // per owned adm leaf: offset in doubles
  DBuf<int32_t> frank;         // per owned adm leaf: rank k
  DBuf<int32_t> fpiv;          // per owned adm leaf: 2*k_max pivots (row, col)
  std::vector<int32_t> h_rank;
  std::vector<std::vector<int32_t>> h_piv;   // per owned adm leaf (recorded when N <= 4e5)
  std::vector<int64_t> h_foff;
  int64_t dense_doubles = 0, factor_doubles = 0;
  double evals_near = 0, evals_aca = 0, entries_aca = 0;
  int aca_steps = 0, aca_chunks = 0, aca_overflow = 0, aca_releases = 0;
  bool aca_prev_valid = false;   // a previous hm_setup of the same owned block list: its pool size
  int64_t aca_prev_sig[2] = {0, 0};
  double aca_prev_bytes = 0, aca_prev_eps = -1;
  int aca_prev_kmax = 0, aca_prev_esz = 0;
  int part_ranks = 1, part_rank = 0;   // diagnostic options: emulate rank part_rank of a part_ranks-way partition (world 1)
  int cost_model = 0;          // option "cost_model": leaf cost of the partition (A18): 0 (default) size proxy, 1 evaluation model, 2 kind weights + per-block ACA cost
  int aca_upd_occ = 1;         // option "aca_upd_occ": CTAs per SM of k_aca_update (0: 16, 1: 24 default, 2: 32)
  int lr_f32 = 0;              // option "lr_f32": store the ACA factors U, V in binary32 (dense blocks stay FP64)
  int lr_esz = 8;              // bytes per stored factor entry of the current setup (8, or 4 with lr_f32)

  // matvec plan (matvec.cu)
  DBuf<MvBatch> mv_batches;
  DBuf<MvSeg> mv_segs;
  DBuf<MvTask> mv_tasks;
  DBuf<int32_t> mv_cta;
  DBuf<MvLarge> mv_large, mv_dense_big;
  DBuf<MvTileV> mv_tiles_v;
  DBuf<MvTileU> mv_tiles_u;
  DBuf<double> mv_tbuf;
  int mv_grid = 0;
  DBuf<unsigned long long> mv_prof;   // option "mv_profile": [producer empty-wait, consumer full-wait, consumer work] cycles
  int mv_small_max = 16384;    // option "mv_small_max": low-rank leaves up to this many bytes go through the pipeline
  int mv_scramble = 0;         // diagnostic option "mv_scramble" (wrong results): see k_mv_batched
  int mv_concurrent = 1;       // option "mv_concurrent": large low-rank kernels on a side stream
  cudaStream_t mv_side = nullptr;
  cudaEvent_t mv_ev[2] = {nullptr, nullptr};
  int mv_kind = 0;             // option "mv_kernel": 0 two CTA rings per SM, 2 x 48 KiB each (default); 1 one ring of 4
  int64_t mv_nbatches = 0, mv_tlen = 0, mv_nsegs = 0;
  int64_t n_lr_small = 0, n_lr_large = 0;

  // work vectors (internal order)
  DBuf<double> xin, yin, xapp, yapp, work, pot_x, pot_out;
  DBuf<double> sh_x, sh_y, sh_sol;   // sharded Krylov (p > 1): gathered x, partial y, local solution
  P2PState p2p;
  int aca_perf = 0;            // option "aca_perf": ACA order-3/4 entries in perf mode (deviates from A15; measured)
  int near_perf = 1;           // option "near_perf": near-field entries in perf mode (A15; <= 1e-13 relative)
  int solve_comm = 0;          // option "solve_comm": 0 NCCL, 1 libhm P2P kernels (after hm_p2p_import)
  DBuf<double> krylov;         // GMRES basis / CG vectors
  DBuf<double> red;            // reduction scratch
  double* h_red = nullptr;     // pinned host scratch for scalar read-back

  // persistent scratch (grow-only)
  TreeWs tws;
  DBuf<int64_t> near_sz;
  DBuf<int32_t> near_tab;
  DBuf<char> near_tmp;
  std::shared_ptr<EntryBatchWork> near_ws;
  std::vector<int64_t> near_hoff;   // host copy of doff (near_prepare)
  // near field beside ACA (option setup_overlap): ACA on s_hi (greatest priority), the
  // near-field evaluation on s_lo (least priority) from its own host thread and timer
  int setup_overlap = 1;
  cudaStream_t s_hi = nullptr, s_lo = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
  KTimer kt_near;
  double near_eval_ms = 0;          // host time of the near-field evaluation (its own thread)
  std::shared_ptr<AcaWork> aca_ws;
  std::shared_ptr<PlanWs> plan_ws;
  int64_t mv_n_large = 0, mv_n_dense_big = 0, mv_n_tiles_v = 0, mv_n_tiles_u = 0;

  PhaseTimes times;
  KTimer kt;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

// scope = one timed launch (or a group of launches) of family f on the library stream
struct KScope {
  KTimer& kt;
  cudaStream_t st;
  int f;
  cudaEvent_t a = nullptr;
  KScope(KTimer& t, cudaStream_t s, int fam) : kt(t), st(s), f(fam) {
    if (kt.on) { a = kt.get(); cudaEventRecord(a, st); }
  }
  KScope(Context& c, int fam) : KScope(c.kt, c.stream, fam) {}
  ~KScope() {
    if (!a) return;
    cudaEvent_t b = kt.get();
    cudaEventRecord(b, st);
    kt.pend.push_back(KTimer::P{f, a, b});
  }
};

// tree.cu
void build_tree(Context& C, const hm_mesh& mesh, int leaf_size, double eta);
// nearfield.cu
void near_prepare(Context& C);                                 // sizes, offsets, storage (synchronous)
void near_eval(Context& C, cudaStream_t st, KTimer& kt);       // evaluation, no allocation; syncs st
void near_check(Context& C);                                   // non-finite check (C.stream)
// aca.cu
void setup_aca(Context& C);
// matvec.cu
void plan_dense_abort(Context& C);   // join a still-running dense planner (error path / tree rebuild)
void plan_dense_begin(Context& C);   // dense half of the plan on host threads (overlaps ACA)
void plan_matvec(Context& C);
void matvec_internal(Context& C, const double* x_int, double* y_int, bool reduce = true);   // y = H x (local
                                                                                          // leaves; + global sum)
void gather_perm(Context& C, const double* x_app, double* x_int);
void scatter_perm(Context& C, const double* y_int, double* y_app);
// solver.cu
void solve(Context& C, const double* rhs_int, double* sol_int, double tol, int* iters,
           double* relres);
// comm
void allreduce_sum(Context& C, double* buf, int64_t n);
// p2p.cu
bool p2p_on(const Context& C);
double* p2p_xfull(Context& C);
double* p2p_ypart(Context& C);
void p2p_export(Context& C, int64_t n_max, void* handle_out);
void p2p_import(Context& C, const void* handles);
void p2p_release(Context& C);
void p2p_check_capacity(Context& C, int64_t S);
void p2p_allgather(Context& C, const double* x, int64_t n, int64_t S, bool into_ypart = false);
void p2p_reduce_scatter(Context& C, double* y, int64_t n, int64_t S);
void p2p_scale_publish(Context& C, const double* a, const double* sden, double* out, int64_t n, int64_t S);
void p2p_allreduce(Context& C, double* buf, int64_t n);
// entries (entry.cu)
void eval_entries(Context& C, int64_t n, const int64_t* d_pairs, double* d_out);
void assemble_rhs(Context& C, int kind, double* f_app);
// potential.cu
void potential(Context& C, const double* alpha_app, int64_t M, const double* X_dev, double* out_dev);
void upload_quadrature_tables();
void quadrature_table_host(int n, double* nodes, double* weights);

// Utilities
// Segment lookup for flattened work: largest c with pre[c] <= e (pre ascending, nseg entries).
// One binary search per warp (for the warp's smallest e), then a short forward walk per lane:
// consecutive lanes hold consecutive e, so each lane walks over at most a few short segments.
template <class I>
__device__ __forceinline__ int64_t warp_find_segment(const I* __restrict__ pre, int64_t nseg, int64_t e, bool valid) {
  const unsigned mask = __activemask();
  int64_t emin = valid ? e : INT64_MAX;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t other = __shfl_xor_sync(mask, emin, o);
    emin = other < emin ? other : emin;
  }
  int64_t lo = 0;
  if (emin != INT64_MAX) {
    int64_t hi = nseg;
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if ((int64_t)__ldg(pre + mid) <= emin) lo = mid; else hi = mid;
    }
  }
  if (valid)
    while (lo + 1 < nseg && (int64_t)__ldg(pre + lo + 1) <= e) ++lo;
  return lo;
}

// Segment-start table of a flattened batch of nseg non-empty segments (prefix pre, entries
// counted from e0): tab[w] = segment holding entry 32 w.  One thread per segment; with it an
// entry finds its segment by one load and a short forward walk instead of a binary search.
__global__ void k_seg_table(const int64_t* __restrict__ pre, int64_t nseg, int64_t e0, int32_t* __restrict__ tab);

inline unsigned grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 2147483647LL) g = 2147483647LL;
  return (unsigned)g;
}

}  // namespace hm
