// nearfield.cu — batched dense assembly of the rank's non-admissible leaves:
// every entry of every owned dense leaf, stored contiguously without padding, row-major per
// block, offsets = exclusive scan of |tau||sigma|.  Entries are evaluated by the
// class-bucketed batch machinery (entry_batch.cuh) in chunks of at most 2^26 entries.

#include <algorithm>

#include "entry_batch.cuh"
#include "primitives.cuh"

namespace hm {

namespace {

__global__ void k_dense_sizes(const Quad* __restrict__ q, int64_t n, int64_t* __restrict__ sz) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= n) return;
  sz[b] = (int64_t)(q[b].rhi - q[b].rlo) * (q[b].chi - q[b].clo);
}

// leaves [b0, b0 + nseg) of the owned dense list; flattened entry e counts from off[b0].
// QUAD: quadrilateral mesh (P = node panels, PT = split triangles, QV = vertex ids; A25)
template <bool QUAD>
struct NearMap {
  static constexpr bool kQuad = QUAD;
  const Panel* P;
  const Panel* PT;
  const int4* QV;
  const Quad* q;
  const int64_t* off;    // owned-list offsets (nb + 1)
  int64_t b0, nseg;      // first leaf of the chunk, leaves in the chunk
  int64_t e0;            // off[b0]
  double* store;
  const int32_t* tab;    // segment-start table of the chunk (k_seg_table)
  __device__ bool locate(int64_t e, bool valid, EntryRef& r) const {
    if (!valid) return false;
    int64_t b = b0 + tab[e >> 5];
    while (off[b + 1] - e0 <= e) ++b;
    r.seg = (int32_t)b;
    r.idx = (int32_t)(e + e0 - off[b]);
    return true;
  }
  __device__ void pair(EntryRef r, int& s, int& t) const {
    const Quad Q = q[r.seg];
    const int ncol = Q.chi - Q.clo;
    s = Q.rlo + r.idx / ncol;
    t = Q.clo + r.idx % ncol;
  }
  __device__ void put(EntryRef r, double a) const { store[off[r.seg] + r.idx] = a; }

};

// bad[0] = number of non-finite entries, bad[1] = smallest offset of one (if any)
__global__ void k_check_finite(const double* __restrict__ a, int64_t n, unsigned long long* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(a[i])) { atomicAdd(bad, 1ull); atomicMin(bad + 1, (unsigned long long)i); }
}

}  // namespace

// Chunks of at most 2^26 entries (at least one leaf each) over the owned dense leaves.
static constexpr int64_t kNearChunk = 1LL << 26;
static int64_t near_chunk_end(const std::vector<int64_t>& hoff, int64_t nb, int64_t b0) {
  int64_t b1 = std::upper_bound(hoff.begin() + b0 + 1, hoff.begin() + nb + 1, hoff[b0] + kNearChunk) - hoff.begin() - 1;
  return std::max(b1, b0 + 1);
}

void near_prepare(Context& C) {
  cudaStream_t st = C.stream;
  const int64_t nb = C.dense_end - C.dense_begin;
  const Quad* q = C.dense.get() + C.dense_begin;
  C.doff.alloc(nb + 1);
  DBuf<int64_t>& sz = C.near_sz;
  sz.alloc(nb + 1);
  HM_CUDA(cudaMemsetAsync(sz.get(), 0, (nb + 1) * sizeof(int64_t), st));
  if (nb) {
    k_dense_sizes<<<grid_for(nb, 256), 256, 0, st>>>(q, nb, sz.get());
    HM_CHECK_LAUNCH();
  }
  DBuf<char>& tmp = C.near_tmp;
  prim::exclusive_scan<int64_t>(sz.get(), C.doff.get(), nb + 1, tmp, st);
  std::vector<int64_t>& hoff = C.near_hoff;
  hoff.assign(nb + 1, 0);
  HM_CUDA(cudaMemcpyAsync(hoff.data(), C.doff.get(), (nb + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HM_CUDA(cudaStreamSynchronize(st));
  const int64_t total = hoff[nb];
  C.dense_doubles = total;
  C.dstore.alloc(total);
  C.evals_near = 0;
  if (total == 0) return;
  // pre-size the evaluation workspace for the largest chunk, so that the evaluation (which
  // may run on its own thread beside ACA) never allocates
  int64_t maxc = 0;
  for (int64_t b0 = 0; b0 < nb;) {
    const int64_t b1 = near_chunk_end(hoff, nb, b0);
    maxc = std::max(maxc, hoff[b1] - hoff[b0]);
    b0 = b1;
  }
  if (!C.near_ws) C.near_ws = std::make_shared<EntryBatchWork>();
  EntryBatchWork& W = *C.near_ws;
  W.cnt.alloc(kNumClass);
  W.cursor.alloc(kNumClass);
  W.qev.alloc(1);
  W.list.alloc(maxc);
  W.ecls.alloc(maxc);
  C.near_tab.alloc(maxc / 32 + 2);
}

void near_eval(Context& C, cudaStream_t st, KTimer& kt) {
  const int64_t nb = C.dense_end - C.dense_begin;
  const std::vector<int64_t>& hoff = C.near_hoff;
  if (nb == 0 || hoff[nb] == 0) return;
  const Quad* q = C.dense.get() + C.dense_begin;
  EntryBatchWork& W = *C.near_ws;
  HM_CUDA(cudaMemsetAsync(W.qev.get(), 0, sizeof(unsigned long long), st));
  double evals = 0;
  for (int64_t b0 = 0; b0 < nb;) {
    const int64_t b1 = near_chunk_end(hoff, nb, b0);
    k_seg_table<<<grid_for(b1 - b0, 256), 256, 0, st>>>(C.doff.get() + b0, b1 - b0, hoff[b0], C.near_tab.get());
    HM_CHECK_LAUNCH();
    if (C.quad) {
      NearMap<true> m{C.qnode.get(), C.panel.get(), C.qv.get(), q, C.doff.get(), b0, b1 - b0, hoff[b0],
                      C.dstore.get(), C.near_tab.get()};
      evals += C.near_perf ? eval_batched<true>(m, hoff[b1] - hoff[b0], W, st, kt)
                           : eval_batched<false>(m, hoff[b1] - hoff[b0], W, st, kt);
    } else {
      NearMap<false> m{C.panel.get(), nullptr, nullptr, q, C.doff.get(), b0, b1 - b0, hoff[b0], C.dstore.get(),
                       C.near_tab.get()};
      evals += C.near_perf ? eval_batched<true>(m, hoff[b1] - hoff[b0], W, st, kt)
                           : eval_batched<false>(m, hoff[b1] - hoff[b0], W, st, kt);
    }
    b0 = b1;
  }
  unsigned long long qev = 0;
  HM_CUDA(cudaMemcpyAsync(&qev, W.qev.get(), sizeof(qev), cudaMemcpyDeviceToHost, st));
  HM_CUDA(cudaStreamSynchronize(st));
  C.evals_near = evals + (double)qev;
}

void near_check(Context& C) {
  cudaStream_t st = C.stream;
  const int64_t total = C.dense_doubles;
  if (total == 0) return;
  DBuf<unsigned long long> bad;
  bad.alloc(2);
  unsigned long long hb[2] = {0ull, ~0ull};
  HM_CUDA(cudaMemcpyAsync(bad.get(), hb, sizeof(hb), cudaMemcpyHostToDevice, st));
  k_check_finite<<<148 * 4, 256, 0, st>>>(C.dstore.get(), total, bad.get());
  HM_CHECK_LAUNCH();
  HM_CUDA(cudaMemcpyAsync(hb, bad.get(), sizeof(hb), cudaMemcpyDeviceToHost, st));
  HM_CUDA(cudaStreamSynchronize(st));
  if (hb[0]) {
    // name the first offending entry: owned dense leaf (offsets near_hoff), local row and column
    const std::vector<int64_t>& hoff = C.near_hoff;
    const int64_t e = (int64_t)hb[1];
    const int64_t b = std::upper_bound(hoff.begin(), hoff.end(), e) - hoff.begin() - 1;
    const Quad& q = C.h_dense[C.dense_begin + b];
    const int64_t n = q.chi - q.clo, r = (e - hoff[b]) / n, c = (e - hoff[b]) % n;
    fail(HM_ERR_NUMERIC, "hm_setup: " + std::to_string(hb[0]) + " non-finite near-field entries; first in dense leaf " +
                             std::to_string(C.dense_begin + b) + " at internal (row, col) = (" +
                             std::to_string(q.rlo + r) + ", " + std::to_string(q.clo + c) + ")");
  }
}

}  // namespace hm
