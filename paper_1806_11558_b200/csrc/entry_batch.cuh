// entry_batch.cuh — batched evaluation of many Galerkin entries, bucketed by quadrature class
// so that every warp runs one rule (the paper's "batching of many small similar tasks",
// P:413-438, applied at the level of single entries).
//
//   pass 1  k_class_count    classify every entry of the batch, count per class
//   pass 2  k_class_scatter  write (segment, index) references into per-class lists
//   pass 3  one kernel per class: regular orders 3/4/5/6 (thread per entry), common edge,
//           common vertex (Sauter-Schwab), identical panel (closed form)
//
// A batch is described by a mapping M (device-side functor, passed by value):
//   bool locate(int64_t e, bool valid, EntryRef& r)  flattened entry -> reference (warp-collective)
//   void pair(EntryRef r, int& s, int& t)            internal row / column indices of the entry
//   void put(EntryRef r, double a)                   consume the value (store / residual update)
//   kQuad, P (node panels), PT, QV                   quadrilateral meshes (A25): class 0 = touching
//                                                    quads (four triangle pairs over PT), classes
//                                                    3..6 = separated quads, tensor rule on P
#pragma once

#include "entry.cuh"
#include "primitives.cuh"

namespace hm {

constexpr int kNumClass = 7;   // 0 identical, 1 edge, 2 vertex, 3..6 regular order n

struct EntryRef {
  int32_t seg, idx;
};


__device__ __forceinline__ int canonical_class(const Panel* __restrict__ P, int s, int t, int& xs, int& ys) {
  const bool swap = __ldg(&P[t].app) < __ldg(&P[s].app);
  xs = swap ? t : s;
  ys = swap ? s : t;
  return entry_class(P[xs], P[ys]);
}

// mapping-level class and regular entry (triangles: A14/A15 on the panels; quads: A25)
template <class M>
__device__ __forceinline__ int map_class(const M& m, int s, int t, int& xs, int& ys) {
  if constexpr (M::kQuad) return quad_class(m.P, m.QV, s, t, xs, ys);
  else return canonical_class(m.P, s, t, xs, ys);
}
template <int n, class M, bool PERF = false>
__device__ __forceinline__ double map_regular(const M& m, int xs, int ys) {
  if constexpr (M::kQuad) {
    return quad_regular_entry<n, PERF>(m.P, xs, ys);
  } else {
    double X[9], Y[9];
    load_panel_vertices(m.P, xs, X);
    load_panel_vertices(m.P, ys, Y);
    const double I = regular_sum<n, false, PERF>(X, Y);
    return dmul(dmul(I, dmul(dmul(2.0, __ldg(&m.P[xs].area)), dmul(2.0, __ldg(&m.P[ys].area)))), kInv4Pi);
  }
}
// any class (rare-rest paths); evals += the rule's kernel evaluations
template <class M>
__device__ __forceinline__ double map_entry(const M& m, int s, int t, unsigned long long& evals) {
  if constexpr (M::kQuad) {
    return quad_entry(m.P, m.PT, m.QV, s, t, evals);
  } else {
    int cls;
    const double v = entry_st(m.P, s, t, &cls);
    evals += (unsigned long long)rule_evals(cls);
    return v;
  }
}

// pass 1 also records every entry's class (one byte) for pass 2
template <class M>
__global__ void k_class_count(M m, int64_t total, unsigned long long* __restrict__ cnt,
                              unsigned char* __restrict__ ecls) {
  __shared__ unsigned int sc[kNumClass];
  if (threadIdx.x < kNumClass) sc[threadIdx.x] = 0;
  __syncthreads();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  EntryRef r;
  if (m.locate(e, e < total, r)) {
    int s, t, xs, ys;
    m.pair(r, s, t);
    const int cls = map_class(m, s, t, xs, ys);
    ecls[e] = (unsigned char)cls;
    atomicAdd(&sc[cls], 1u);
  }
  __syncthreads();
  if (threadIdx.x < kNumClass && sc[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], (unsigned long long)sc[threadIdx.x]);
}

template <class M>
__global__ void k_class_scatter(M m, int64_t total, const unsigned char* __restrict__ ecls,
                                unsigned long long* __restrict__ cursor, EntryRef* __restrict__ lists) {
  __shared__ unsigned int sc[kNumClass];
  __shared__ unsigned long long base[kNumClass];
  if (threadIdx.x < kNumClass) sc[threadIdx.x] = 0;
  __syncthreads();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  EntryRef r;
  int cls = -1;
  unsigned int pos = 0;
  if (m.locate(e, e < total, r)) {
    cls = ecls[e];
    pos = atomicAdd(&sc[cls], 1u);
  }
  __syncthreads();
  if (threadIdx.x < kNumClass) base[threadIdx.x] = sc[threadIdx.x] ? atomicAdd(&cursor[threadIdx.x], (unsigned long long)sc[threadIdx.x]) : 0;
  __syncthreads();
  if (cls >= 0) lists[base[cls] + pos] = r;
}

template <int n, class M, bool PERF>
__global__ void __launch_bounds__(128) k_eval_regular(M m, const EntryRef* __restrict__ list, int64_t cnt) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= cnt) return;
  const EntryRef r = list[k];
  int s, t, xs, ys;
  m.pair(r, s, t);
  map_class(m, s, t, xs, ys);
  m.put(r, map_regular<n, M, PERF>(m, xs, ys));
}

// triangles: KIND 0 identical, 1 edge, 2 vertex; quads: KIND 0 = touching quads (the four
// triangle pairs; their evaluations are counted into qev)
template <int KIND, class M, bool PERF>
__global__ void __launch_bounds__(64) k_eval_touching(M m, const EntryRef* __restrict__ list, int64_t cnt,
                                                      unsigned long long* __restrict__ qev) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if constexpr (M::kQuad) {
    unsigned long long ev = 0;
    if (k < cnt) {
      const EntryRef r = list[k];
      int s, t, xs, ys;
      m.pair(r, s, t);
      map_class(m, s, t, xs, ys);
      m.put(r, quad_split_entry<PERF>(m.PT, xs, ys, ev));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
    if ((threadIdx.x & 31) == 0 && ev) atomicAdd(qev, ev);
    return;
  }
  if (k >= cnt) return;
  const EntryRef r = list[k];
  int s, t, xs, ys;
  m.pair(r, s, t);
  canonical_class(m.P, s, t, xs, ys);
  const Panel& A = m.P[xs];
  const Panel& B = m.P[ys];
  double X[9], Y[9], v;
  if (KIND == 0) {
    load_panel_vertices(m.P, xs, X);
    v = dmul(selfterm_closed(X, A.area), kInv4Pi);
  } else {
    orient_touching(KIND, A, B, X, Y);
    const double I = ss_sum_t<KIND, PERF>(X, Y);
    v = dmul(dmul(I, dmul(dmul(2.0, A.area), dmul(2.0, B.area))), kInv4Pi);
  }
  m.put(r, v);
}

// Three-kernel, host-sync-free variant for ACA rows / columns (nearly all entries are order 3,
// most of the rest order 4).  The batch size is read on the device (*dtot: the step's row or
// column total, written by the step's scans), so the host never waits for it:
//   k_eval_class3   persistent pass over the batch (warps take groups of entries from a
//                   counter): evaluates the order-3 entries in place and appends order-4
//                   references to the front of `lists`, all other classes to the back
//                   (warp-aggregated atomics);
//   k_eval_list<4>  persistent grid-stride over the order-4 list (count read on the device);
//   k_eval_rest     persistent, the remaining few (orders 5, 6, touching pairs).
// one 32-entry group of a warp (lanes e = e0 + lane): classify, append non-order-3 entries,
// evaluate order 3 in place
template <class M>
__device__ __forceinline__ void class3_group(const M& m, int64_t e, int64_t total, int lane, EntryRef* __restrict__ lists,
                                             unsigned long long* __restrict__ cnt, unsigned long long& ev) {
  EntryRef r;
  int cls = -1, xs = 0, ys = 0;
  if (m.locate(e, e < total, r)) {
    int s, t;
    m.pair(r, s, t);
    cls = map_class(m, s, t, xs, ys);
  }
  const unsigned below = (1u << lane) - 1u;
  const unsigned b4 = __ballot_sync(0xffffffffu, cls == 4), br = __ballot_sync(0xffffffffu, cls >= 0 && cls != 3 && cls != 4);
  unsigned long long base4 = 0, baser = 0;
  if (lane == 0) {
    if (b4) base4 = atomicAdd(&cnt[0], (unsigned long long)__popc(b4));
    if (br) baser = atomicAdd(&cnt[1], (unsigned long long)__popc(br));
  }
  base4 = __shfl_sync(0xffffffffu, base4, 0);
  baser = __shfl_sync(0xffffffffu, baser, 0);
  if (cls == 4) lists[base4 + __popc(b4 & below)] = r;
  else if (cls >= 0 && cls != 3) lists[total - 1 - (baser + __popc(br & below))] = r;
  if (cls == 3) {
    m.put(r, map_regular<3, M, M::kPerf>(m, xs, ys));
    ev += M::kQuad ? 81 : tri_rule_points(3) * tri_rule_points(3);
  }
}

// Persistent, dynamically balanced: every warp takes groups of kDynGroups x 32 consecutive
// entries from the counter cnt[2] until the batch is exhausted (a fixed grid-stride split or
// one thread per entry leave SMs idle at the tail: C4 ACA evaluation 1.85 s resp. 1.75 s vs
// 1.61 s, profiles/r02_setup_ab1.jsonl).  Groups per fetch: 1 / 2 / 4 / 8 / 16 / 32 give
// 1735 / 1607 / 1579 / 1560 / 1561 / 1581 ms (profiles/r02_setup_ab22/23_dyngroups.jsonl).
constexpr int kDynGroups = 8;
template <class M>
__global__ void __launch_bounds__(128, 4) k_eval_class3(M m, const int64_t* __restrict__ dtot,
                                                     EntryRef* __restrict__ lists,
                                                     unsigned long long* __restrict__ cnt /* [n4, nrest, next] */,
                                                     unsigned long long* __restrict__ evals) {
  const int64_t total = *dtot;
  const int lane = threadIdx.x & 31;
  unsigned long long ev = 0;
  for (;;) {
    unsigned long long b0 = 0;
    if (lane == 0) b0 = atomicAdd(&cnt[2], (unsigned long long)(32 * kDynGroups));
    b0 = __shfl_sync(0xffffffffu, b0, 0);
    if ((int64_t)b0 >= total) break;
#pragma unroll 1
    for (int g = 0; g < kDynGroups; ++g) class3_group(m, (int64_t)b0 + 32 * g + lane, total, lane, lists, cnt, ev);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
  if (lane == 0 && ev) atomicAdd(evals, ev);
}

template <int n, class M>
__global__ void __launch_bounds__(128) k_eval_list(M m, const EntryRef* __restrict__ list,
                                                   const unsigned long long* __restrict__ cnt,
                                                   unsigned long long* __restrict__ evals) {
  const int64_t c = (int64_t)*cnt;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < c; k += (int64_t)gridDim.x * blockDim.x) {
    const EntryRef r = list[k];
    int s, t, xs, ys;
    m.pair(r, s, t);
    map_class(m, s, t, xs, ys);
    m.put(r, map_regular<n, M, M::kPerf>(m, xs, ys));
  }
  constexpr int np = M::kQuad ? n * n : tri_rule_points(n);
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(evals, (unsigned long long)(np * np) * (unsigned long long)c);
}

// the rare rest (orders 5, 6 and touching pairs), read from the back of `lists`
template <class M>
__global__ void __launch_bounds__(128) k_eval_rest(M m, const EntryRef* __restrict__ lists,
                                                   const int64_t* __restrict__ dtot,
                                                   const unsigned long long* __restrict__ cnt,
                                                   unsigned long long* __restrict__ evals) {
  const int64_t total = *dtot;
  const int64_t c = (int64_t)cnt[1];
  unsigned long long ev = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < c; k += (int64_t)gridDim.x * blockDim.x) {
    const EntryRef r = lists[total - 1 - k];
    int s, t;
    m.pair(r, s, t);
    m.put(r, map_entry(m, s, t, ev));
  }
  if (ev) atomicAdd(evals, ev);
}

// Touching quads (A25) sorted by the classes of their four triangle pairs (3 bits each), so
// that the warps of k_eval_touching<0> run one rule sequence.
template <class M>
__global__ void k_quad_sig(M m, const EntryRef* __restrict__ list, int64_t cnt, uint16_t* __restrict__ key,
                           unsigned long long* __restrict__ ref) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= cnt) return;
  const EntryRef r = list[k];
  int s, t, xs, ys;
  m.pair(r, s, t);
  map_class(m, s, t, xs, ys);
  unsigned sig = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) sig |= (unsigned)entry_class(m.PT[2 * xs + (q >> 1)], m.PT[2 * ys + (q & 1)]) << (3 * q);
  key[k] = (uint16_t)sig;
  ref[k] = reinterpret_cast<const unsigned long long&>(r);
}

struct EntryBatchWork {
  DBuf<unsigned long long> cnt, cursor, qev;   // qev: evaluations of touching quads (device)
  DBuf<unsigned char> ecls;                    // class of every entry of the batch (pass 1)
  DBuf<uint16_t> qkey[2];                      // touching quads: signature sort
  DBuf<unsigned long long> qref[2];
  DBuf<char> qtmp;
  DBuf<EntryRef> list;
  unsigned long long hcnt[kNumClass];
};

// Evaluate all `total` entries of mapping m on stream st; returns the number of kernel
// evaluations.  Allocates only when W is smaller than this batch (near_prepare pre-sizes it).
// PERF: perf-mode kernel evaluations (option near_perf; near-field entries only, A15)
template <bool PERF, class M>
double eval_batched(const M& m, int64_t total, EntryBatchWork& W, cudaStream_t st, KTimer& kt) {
  if (total <= 0) return 0.0;
  W.cnt.alloc(kNumClass);
  W.cursor.alloc(kNumClass);
  W.qev.alloc(1);
  W.ecls.alloc(total);
  HM_CUDA(cudaMemsetAsync(W.cnt.get(), 0, kNumClass * sizeof(unsigned long long), st));
  k_class_count<M><<<grid_for(total, 256), 256, 0, st>>>(m, total, W.cnt.get(), W.ecls.get());
  HM_CHECK_LAUNCH();
  HM_CUDA(cudaMemcpyAsync(W.hcnt, W.cnt.get(), sizeof(W.hcnt), cudaMemcpyDeviceToHost, st));
  HM_CUDA(cudaStreamSynchronize(st));
  unsigned long long base[kNumClass], acc = 0;
  for (int c = 0; c < kNumClass; ++c) { base[c] = acc; acc += W.hcnt[c]; }
  W.list.alloc(acc);
  HM_CUDA(cudaMemcpyAsync(W.cursor.get(), base, sizeof(base), cudaMemcpyHostToDevice, st));
  k_class_scatter<M><<<grid_for(total, 256), 256, 0, st>>>(m, total, W.ecls.get(), W.cursor.get(), W.list.get());
  HM_CHECK_LAUNCH();
  const EntryRef* L = W.list.get();
  double evals = 0;
  // heavy classes first so that the light ones fill the tail
  KScope ks(kt, st, KF_EVAL_NEAR);
  if constexpr (M::kQuad) {        // touching quads first, sorted by their sub-pair classes
    const int64_t c0 = (int64_t)W.hcnt[0];
    if (c0) {
      for (int b = 0; b < 2; ++b) { W.qkey[b].alloc(c0); W.qref[b].alloc(c0); }
      k_quad_sig<M><<<grid_for(c0, 256), 256, 0, st>>>(m, L + base[0], c0, W.qkey[0].get(), W.qref[0].get());
      HM_CHECK_LAUNCH();
      prim::radix_sort_pairs<uint16_t, unsigned long long>(W.qkey[0].get(), W.qkey[1].get(), W.qref[0].get(),
                                                           W.qref[1].get(), c0, 0, 12, W.qtmp, st);
      const EntryRef* Ls = reinterpret_cast<const EntryRef*>(W.qref[1].get());
      k_eval_touching<0, M, PERF><<<grid_for(c0, 64), 64, 0, st>>>(m, Ls, c0, W.qev.get());
      HM_CHECK_LAUNCH();
    }
  }
  if (W.hcnt[1]) { k_eval_touching<1, M, PERF><<<grid_for(W.hcnt[1], 64), 64, 0, st>>>(m, L + base[1], W.hcnt[1], W.qev.get()); HM_CHECK_LAUNCH(); }
  if (W.hcnt[2]) { k_eval_touching<2, M, PERF><<<grid_for(W.hcnt[2], 64), 64, 0, st>>>(m, L + base[2], W.hcnt[2], W.qev.get()); HM_CHECK_LAUNCH(); }
  if (W.hcnt[6]) { k_eval_regular<6, M, PERF><<<grid_for(W.hcnt[6], 128), 128, 0, st>>>(m, L + base[6], W.hcnt[6]); HM_CHECK_LAUNCH(); }
  if (W.hcnt[5]) { k_eval_regular<5, M, PERF><<<grid_for(W.hcnt[5], 128), 128, 0, st>>>(m, L + base[5], W.hcnt[5]); HM_CHECK_LAUNCH(); }
  if (W.hcnt[4]) { k_eval_regular<4, M, PERF><<<grid_for(W.hcnt[4], 128), 128, 0, st>>>(m, L + base[4], W.hcnt[4]); HM_CHECK_LAUNCH(); }
  if (W.hcnt[3]) { k_eval_regular<3, M, PERF><<<grid_for(W.hcnt[3], 128), 128, 0, st>>>(m, L + base[3], W.hcnt[3]); HM_CHECK_LAUNCH(); }
  if (W.hcnt[0] && !M::kQuad) { k_eval_touching<0, M, PERF><<<grid_for(W.hcnt[0], 64), 64, 0, st>>>(m, L + base[0], W.hcnt[0], W.qev.get()); HM_CHECK_LAUNCH(); }
  // (quads: class 0 = touching quads, counted on the device into W.qev, read by the caller)
  const double per[kNumClass] = {0, 6480, 2592, M::kQuad ? 81.0 : 49.0, 256, 625, 1296};
  for (int c = 0; c < kNumClass; ++c) evals += per[c] * (double)W.hcnt[c];
  return evals;
}

}  // namespace hm
