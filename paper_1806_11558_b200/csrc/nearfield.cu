// nearfield.cu — batched dense assembly of the rank's non-admissible leaves:
// every entry of every owned dense leaf, stored contiguously without padding, row-major per
// block, offsets = exclusive scan of |tau||sigma|.
//
// Two passes keep warps uniform: pass 1 (one thread per entry, consecutive entries of a
// block row share the row panel) evaluates all regular entries and queues the ~1% touching
// entries; pass 2 evaluates the queued singular entries (Sauter-Schwab / closed form).
#include <cub/cub.cuh>

#include "entry.cuh"

namespace hm {

namespace {

__global__ void k_dense_sizes(const Quad* __restrict__ q, int64_t n, int64_t* __restrict__ sz) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= n) return;
  sz[b] = (int64_t)(q[b].rhi - q[b].rlo) * (q[b].chi - q[b].clo);
}

__device__ __forceinline__ int64_t find_block(const int64_t* __restrict__ off, int64_t nb, int64_t e) {
  int64_t lo = 0, hi = nb;   // largest b with off[b] <= e
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= e) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void k_near_regular(const Panel* __restrict__ P, const Quad* __restrict__ q, const int64_t* __restrict__ off,
                               int64_t nb, int64_t total, double* __restrict__ store,
                               int64_t* __restrict__ sing, int64_t sing_cap,
                               unsigned long long* __restrict__ ctr /*[nsing, evals, bad]*/) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long ev = 0;
  if (e < total) {
    int64_t b = find_block(off, nb, e);
    const Quad Q = q[b];
    int64_t loc = e - off[b];
    int ncol = Q.chi - Q.clo;
    int s = Q.rlo + (int)(loc / ncol), t = Q.clo + (int)(loc % ncol);
    const bool swap = __ldg(&P[t].app) < __ldg(&P[s].app);
    const int xs = swap ? t : s, ys = swap ? s : t;
    const int cls = entry_class(P[xs], P[ys]);
    if (cls >= 3) {
      double X[9], Y[9], I;
      load_panel_vertices(P, xs, X);
      load_panel_vertices(P, ys, Y);
      switch (cls) {
        case 3: I = regular_sum<3>(X, Y); break;
        case 4: I = regular_sum<4>(X, Y); break;
        case 5: I = regular_sum<5>(X, Y); break;
        default: I = regular_sum<6>(X, Y); break;
      }
      const double v = dmul(dmul(I, dmul(dmul(2.0, P[xs].area), dmul(2.0, P[ys].area))), kInv4Pi);
      store[e] = v;
      if (!isfinite(v)) atomicAdd(&ctr[2], 1ull);
      ev = (unsigned long long)(cls * cls * cls * cls);
    } else {
      unsigned long long slot = atomicAdd(&ctr[0], 1ull);
      if ((int64_t)slot < sing_cap) sing[slot] = e;
      ev = (unsigned long long)rule_evals(cls);
    }
  }
  // block-aggregated evaluation count
  typedef cub::BlockReduce<unsigned long long, 128> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long tot = BR(tmp).Sum(ev);
  if (threadIdx.x == 0 && tot) atomicAdd(&ctr[1], tot);
}

__global__ void k_near_singular(const Panel* __restrict__ P, const Quad* __restrict__ q, const int64_t* __restrict__ off,
                                int64_t nb, const int64_t* __restrict__ sing, const unsigned long long* __restrict__ nsing,
                                double* __restrict__ store, unsigned long long* __restrict__ ctr) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= (int64_t)*nsing) return;
  int64_t e = sing[k];
  int64_t b = find_block(off, nb, e);
  const Quad Q = q[b];
  int64_t loc = e - off[b];
  int ncol = Q.chi - Q.clo;
  int s = Q.rlo + (int)(loc / ncol), t = Q.clo + (int)(loc % ncol);
  const double v = entry_st(P, s, t);
  store[e] = v;
  if (!isfinite(v)) atomicAdd(&ctr[2], 1ull);
}

}  // namespace

void setup_nearfield(Context& C) {
  cudaStream_t st = C.stream;
  const int64_t nb = C.dense_end - C.dense_begin;
  const Quad* q = C.dense.get() + C.dense_begin;
  C.doff.alloc_exact(nb + 1);
  DBuf<int64_t> sz;
  sz.alloc(nb + 1);
  HM_CUDA(cudaMemsetAsync(sz.get(), 0, (nb + 1) * sizeof(int64_t), st));
  if (nb) {
    k_dense_sizes<<<grid_for(nb, 256), 256, 0, st>>>(q, nb, sz.get());
    HM_CHECK_LAUNCH();
  }
  DBuf<char> tmp;
  size_t bytes = 0;
  HM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, sz.get(), C.doff.get(), nb + 1, st));
  tmp.alloc(bytes);
  HM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, sz.get(), C.doff.get(), nb + 1, st));
  int64_t total = 0;
  HM_CUDA(cudaMemcpyAsync(&total, C.doff.get() + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HM_CUDA(cudaStreamSynchronize(st));
  C.dense_doubles = total;
  C.dstore.alloc_exact(total);
  if (total == 0) { C.evals_near = 0; return; }
  DBuf<unsigned long long> ctr;
  ctr.alloc(3);
  HM_CUDA(cudaMemsetAsync(ctr.get(), 0, 3 * sizeof(unsigned long long), st));
  // touching pairs are ~13 per row panel on the paper-type meshes; the queue is re-sized and
  // the pass repeated if a mesh has more
  int64_t sing_cap = std::min<int64_t>(total, 16 * (C.N + 1) + 1024);
  DBuf<int64_t> sing;
  unsigned long long hc[3];
  for (;;) {
    sing.alloc(sing_cap);
    HM_CUDA(cudaMemsetAsync(ctr.get(), 0, 3 * sizeof(unsigned long long), st));
    k_near_regular<<<grid_for(total, 128), 128, 0, st>>>(C.panel.get(), q, C.doff.get(), nb, total, C.dstore.get(),
                                                          sing.get(), sing_cap, ctr.get());
    HM_CHECK_LAUNCH();
    HM_CUDA(cudaMemcpyAsync(hc, ctr.get(), sizeof(hc), cudaMemcpyDeviceToHost, st));
    HM_CUDA(cudaStreamSynchronize(st));
    if ((int64_t)hc[0] <= sing_cap) break;
    sing_cap = (int64_t)hc[0];
  }
  if (hc[0]) {
    k_near_singular<<<grid_for((int64_t)hc[0], 64), 64, 0, st>>>(C.panel.get(), q, C.doff.get(), nb, sing.get(),
                                                                  ctr.get(), C.dstore.get(), ctr.get());
    HM_CHECK_LAUNCH();
  }
  HM_CUDA(cudaMemcpyAsync(hc, ctr.get(), sizeof(hc), cudaMemcpyDeviceToHost, st));
  HM_CUDA(cudaStreamSynchronize(st));
  C.evals_near = (double)hc[1];
  if (hc[2]) fail(HM_ERR_NUMERIC, "hm_setup: non-finite near-field entry (" + std::to_string(hc[2]) + " entries)");
}

}  // namespace hm
