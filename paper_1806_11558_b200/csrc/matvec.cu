// matvec.cu — batched H-matrix-vector product: non-admissible leaves apply their
// stored dense block, admissible leaves apply U (V^T x) ("two matrix-vector
// products of skinny matrices"); application <-> internal permutation at the ends.
//
// Memory-bound (0.25 flop/B): the stored H is streamed from HBM exactly once per product.
//
//   small leaves   (dense blocks and low-rank blocks with (m+n)k*8 <= 16 KiB, ~all leaves):
//                  k_mv_batched — one persistent CTA per SM walks a contiguous, byte-balanced
//                  range of "batches" (consecutive leaves filling <= 44 KiB).  One elected
//                  thread streams each batch into shared memory with one cp.async.bulk (TMA
//                  bulk copy, mbarrier completion) per contiguous run of leaves, 4 stages deep
//                  (~176 KiB per SM in flight); warp 0 produces, 15 consumer warps compute
//                  the staged batches out of shared memory (dense rows with s lanes per row,
//                  low-rank t = V^T x then y += U t), releasing each stage through an "empty"
//                  mbarrier.  One FP64 atomic per row into the L2-resident y.
//   large low-rank (blocks above 16 KiB): two barrier-free warp-task kernels with direct
//                  coalesced loads, k_mv_large_v (t += V^T x over 8-column x 2048-row tiles,
//                  atomics into t) then k_mv_large_u (y += U t, k independent loads per row).
//   dense blocks too big for a stage (only with large leaf_size): k_mv_dense_direct.
#include <cub/cub.cuh>

#include <algorithm>

#include "entry.cuh"

namespace hm {

constexpr int kMvStages = 4;
constexpr int kMvStageBytes = 48 * 1024;
constexpr int kMvThreads = 512;
constexpr int kMvSmallMax = 16 * 1024;

namespace {

__global__ void k_gather(const double* __restrict__ x_app, const int32_t* __restrict__ perm, int64_t N,
                         double* __restrict__ x_int) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < N) x_int[s] = x_app[perm[s]];
}

__global__ void k_scatter(const double* __restrict__ y_int, const int32_t* __restrict__ perm, int64_t N,
                          double* __restrict__ y_app) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < N) y_app[perm[s]] = y_int[s];
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Dense m x n row-major block out of shared memory, x_sigma staged beside it: S lanes per
// row (consecutive columns -> conflict-free shared loads for the leaf widths of CBC), 32/S
// rows per pass, P passes held in registers so the P shuffle reductions are independent.
template <int S, int P>
__device__ __forceinline__ void dense_block(const double* __restrict__ B, int m, int n, const double* __restrict__ xs,
                                            double* __restrict__ y, int lane) {
  constexpr int RPP = 32 / S;
  const int sub = lane % S, rr = lane / S;
  for (int r0 = 0; r0 < m; r0 += RPP * P) {
    double acc[P];
#pragma unroll
    for (int p = 0; p < P; ++p) acc[p] = 0.0;
    for (int c = sub; c < n; c += S) {
      const double xc = xs[c];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int r = r0 + rr + p * RPP;
        if (r < m) acc[p] = __fma_rn(B[r * n + c], xc, acc[p]);
      }
    }
#pragma unroll
    for (int o = S / 2; o > 0; o >>= 1)
#pragma unroll
      for (int p = 0; p < P; ++p) acc[p] += __shfl_xor_sync(0xffffffffu, acc[p], o);
    if (sub == 0)
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int r = r0 + rr + p * RPP;
        if (r < m) atomicAdd(y + r, acc[p]);
      }
  }
}

__device__ __forceinline__ void dense_any(const double* B, int m, int n, const double* xs, double* y, int lane) {
  if (n <= 16) dense_block<2, 4>(B, m, n, xs, y, lane);
  else if (n <= 64) dense_block<4, 4>(B, m, n, xs, y, lane);
  else dense_block<8, 4>(B, m, n, xs, y, lane);
}

// Low-rank block U (m x k) | V (n x k), column-major, columns [l0, l0 + kc) (kc <= KB), out of
// shared memory: t = V^T x with all kc column sums in registers, one butterfly over the kc
// sums at once, then y += U t (one FP64 atomic per row).
template <int KB>
__device__ __forceinline__ void lowrank_block(const double* __restrict__ U0, int m, int n, int k, int l0, int kc,
                                              const double* __restrict__ xs, double* __restrict__ y, int lane) {
  const double* V = U0 + m * k + l0 * n;
  const double* U = U0 + l0 * m;
  double acc[KB];
#pragma unroll
  for (int l = 0; l < KB; ++l) acc[l] = 0.0;
  for (int j = lane; j < n; j += 32) {
    const double xj = xs[j];
#pragma unroll
    for (int l = 0; l < KB; ++l)
      if (l < kc) acc[l] = __fma_rn(V[j + l * n], xj, acc[l]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int l = 0; l < KB; ++l) acc[l] += __shfl_xor_sync(0xffffffffu, acc[l], o);
  for (int t = lane; t < m; t += 32) {
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < KB; ++l)
      if (l < kc) s = __fma_rn(U[t + l * m], acc[l], s);
    atomicAdd(y + t, s);
  }
}

__device__ __forceinline__ void lowrank_any(const double* U, int m, int n, int k, const double* xs, double* y,
                                            int lane) {
  if (k <= 8) lowrank_block<8>(U, m, n, k, 0, k, xs, y, lane);
  else if (k <= 16) lowrank_block<16>(U, m, n, k, 0, k, xs, y, lane);
  else
    for (int l0 = 0; l0 < k; l0 += 16) lowrank_block<16>(U, m, n, k, l0, min(16, k - l0), xs, y, lane);
}

// Warp-specialised pipeline.  Warp 0 is the producer: per batch, lane 0 posts the stage's
// byte count on its "full" mbarrier, then the 32 lanes issue the batch's bulk copies
// (task records, x_sigma segments, leaf storage) after the stage's "empty" barrier has
// flipped.  Warps 1..NW-1 consume every stage entirely out of shared memory (tasks
// round-robin) — no global load on the consumer side, only fire-and-forget atomics into
// the L2-resident y — then arrive on the stage's "empty" barrier.
__global__ void __launch_bounds__(kMvThreads, 1)
    k_mv_batched(const MvBatch* __restrict__ batches, const MvSeg* __restrict__ segs, const int32_t* __restrict__ cta_first,
                 const char* __restrict__ base0, const char* __restrict__ base1, const char* __restrict__ base2,
                 const double* __restrict__ x, double* __restrict__ y) {
  constexpr int NW = kMvThreads / 32, NC = NW - 1;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMvStages;
  unsigned char* buf = smem + 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b0 = cta_first[blockIdx.x], nb = cta_first[blockIdx.x + 1] - b0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMvStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    for (int it = 0; it < nb; ++it) {
      const int stage = it % kMvStages;
      if (it >= kMvStages) mbar_wait(&empty[stage], (unsigned)(((it / kMvStages) - 1) & 1));
      const MvBatch B = batches[b0 + it];
      if (lane == 0) mbar_expect_tx(&full[stage], (unsigned)B.bytes);
      __syncwarp();
      unsigned char* sb = buf + stage * kMvStageBytes;
      for (int s = lane; s < B.nseg; s += 32) {
        const MvSeg S = segs[B.first_seg + s];
        const char* base = S.base == 0 ? base0 : S.base == 1 ? base1 : S.base == 2 ? base2
                                                                     : reinterpret_cast<const char*>(x);
        bulk_g2s(sb + S.dst, base + S.src, (unsigned)S.bytes, &full[stage]);
      }
    }
    return;
  }
  for (int it = 0; it < nb; ++it) {
    const int stage = it % kMvStages;
    mbar_wait(&full[stage], (unsigned)((it / kMvStages) & 1));
    const unsigned char* sb = buf + stage * kMvStageBytes;
    const double* sd = reinterpret_cast<const double*>(sb);
    const int4* rec = reinterpret_cast<const int4*>(sb);
    const int count = rec[0].x;
    for (int t = warp - 1; t < count; t += NC) {
      const int4 T = rec[1 + t];
      const uint32_t mnk = (uint32_t)T.w;
      const int m = mnk & 2047, n = (mnk >> 11) & 2047, k = mnk >> 22;
      if (k == 0) dense_any(sd + T.z, m, n, sd + T.y, y + T.x, lane);
      else lowrank_any(sd + T.z, m, n, k, sd + T.y, y + T.x, lane);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[stage])) : "memory");
  }
}

// Large low-rank blocks (storage > 16 KiB), barrier-free warp tasks with direct coalesced loads.
// Phase 1, tile = (block, 8 columns l0.., 2048 rows j0..): t[l] += sum_j V[j, l] x[clo + j];
// each lane keeps 8 column sums (x_j loaded once per row, 8 independent loads in flight).
__global__ void __launch_bounds__(256) k_mv_large_v(const MvTileV* __restrict__ tiles, int64_t ntiles,
                                                    const MvLarge* __restrict__ L, const double* __restrict__ pool,
                                                    const double* __restrict__ x, double* __restrict__ tbuf) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < ntiles; i += nw) {
    const MvTileV T = tiles[i];
    const MvLarge B = L[T.blk];
    const int kc = min(8, B.k - T.l);
    const double* V = pool + B.off + (int64_t)B.m * B.k + (int64_t)T.l * B.n;
    const double* xs = x + B.clo;
    double acc[8];
#pragma unroll
    for (int l = 0; l < 8; ++l) acc[l] = 0.0;
    for (int j = T.j0 + lane; j < T.j1; j += 64) {
      const bool two = j + 32 < T.j1;
      const double xa = __ldg(xs + j), xb = two ? __ldg(xs + j + 32) : 0.0;
      double va[8], vb[8];
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        va[l] = l < kc ? __ldg(V + j + (int64_t)l * B.n) : 0.0;
        vb[l] = (l < kc && two) ? __ldg(V + j + 32 + (int64_t)l * B.n) : 0.0;
      }
#pragma unroll
      for (int l = 0; l < 8; ++l) acc[l] = __fma_rn(vb[l], xb, __fma_rn(va[l], xa, acc[l]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int l = 0; l < 8; ++l) acc[l] += __shfl_xor_sync(0xffffffffu, acc[l], o);
    if (lane < kc) {
      double v = acc[0];
#pragma unroll
      for (int l = 1; l < 8; ++l) v = lane == l ? acc[l] : v;
      atomicAdd(tbuf + B.toff + T.l + lane, v);
    }
  }
}

// Phase 2, tile = (block, 256 rows t0..): y[rlo + t] += sum_l U[t, l] t_l (k independent loads per row)
__global__ void __launch_bounds__(256) k_mv_large_u(const MvTileU* __restrict__ tiles, int64_t ntiles,
                                                    const MvLarge* __restrict__ L, const double* __restrict__ pool,
                                                    const double* __restrict__ tbuf, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < ntiles; i += nw) {
    const MvTileU T = tiles[i];
    const MvLarge B = L[T.blk];
    const double* U = pool + B.off;
    const double* tl = tbuf + B.toff;
    for (int t = T.t0 + lane; t < T.t1; t += 64) {
      const bool two = t + 32 < T.t1;
      double s0 = 0.0, s1 = 0.0, r0 = 0.0, r1 = 0.0;
      int l = 0;
      for (; l + 1 < B.k; l += 2) {
        const double ta = __ldg(tl + l), tb = __ldg(tl + l + 1);
        const double u0 = __ldg(U + t + (int64_t)l * B.m), u1 = __ldg(U + t + (int64_t)(l + 1) * B.m);
        const double w0 = two ? __ldg(U + t + 32 + (int64_t)l * B.m) : 0.0;
        const double w1 = two ? __ldg(U + t + 32 + (int64_t)(l + 1) * B.m) : 0.0;
        s0 = __fma_rn(u0, ta, s0); s1 = __fma_rn(u1, tb, s1); r0 = __fma_rn(w0, ta, r0); r1 = __fma_rn(w1, tb, r1);
      }
      if (l < B.k) {
        const double ta = __ldg(tl + l);
        s0 = __fma_rn(__ldg(U + t + (int64_t)l * B.m), ta, s0);
        if (two) r0 = __fma_rn(__ldg(U + t + 32 + (int64_t)l * B.m), ta, r0);
      }
      atomicAdd(y + B.rlo + t, s0 + s1);
      if (two) atomicAdd(y + B.rlo + t + 32, r0 + r1);
    }
  }
}

// dense blocks that do not fit a stage (large leaf_size only): warp per block, direct loads
__global__ void k_mv_dense_direct(const MvLarge* __restrict__ L, int64_t nl, const double* __restrict__ store,
                                  const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = w0; b < nl; b += nw) {
    const MvLarge B = L[b];
    dense_any(store + B.off, B.m, B.n, x + B.clo, y + B.rlo, lane);
  }
}

}  // namespace

void plan_matvec(Context& C) {
  cudaStream_t st = C.stream;
  const int64_t nd = C.dense_end - C.dense_begin, na = C.adm_end - C.adm_begin;
  std::vector<int64_t> hoff(nd + 1);
  HM_CUDA(cudaMemcpyAsync(hoff.data(), C.doff.get(), (nd + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  if (C.h_dense.size() != (size_t)C.ndense) {
    C.h_dense.resize(C.ndense);
    HM_CUDA(cudaMemcpyAsync(C.h_dense.data(), C.dense.get(), C.ndense * sizeof(Quad), cudaMemcpyDeviceToHost, st));
  }
  HM_CUDA(cudaStreamSynchronize(st));
  struct Item { int64_t byte0, bytes; int base; int32_t rlo, clo, n; uint32_t mnk; };
  std::vector<Item> items;
  items.reserve(nd + na);
  std::vector<MvLarge> dense_big, large;
  for (int64_t b = 0; b < nd; ++b) {
    const Quad& q = C.h_dense[C.dense_begin + b];
    const int m = q.rhi - q.rlo, n = q.chi - q.clo;
    const int64_t bytes = 8 * (int64_t)m * n;
    if (bytes + 8 * n + 64 > kMvStageBytes || m > 2047 || n > 2047) {
      dense_big.push_back(MvLarge{q.rlo, q.clo, m, n, 0, 0, hoff[b], 0});
      continue;
    }
    items.push_back(Item{8 * hoff[b], bytes, 0, q.rlo, q.clo, n, (uint32_t)m | ((uint32_t)n << 11)});
  }
  std::vector<int64_t> lr_order;
  for (int64_t b = 0; b < na; ++b)
    if (C.h_rank[b] > 0) lr_order.push_back(b);
  if (!std::is_sorted(lr_order.begin(), lr_order.end(), [&](int64_t a, int64_t b) { return C.h_foff[a] < C.h_foff[b]; }))
    std::sort(lr_order.begin(), lr_order.end(), [&](int64_t a, int64_t b) { return C.h_foff[a] < C.h_foff[b]; });
  int64_t tl = 0;
  for (int64_t b : lr_order) {
    const Quad& q = C.h_adm[C.adm_begin + b];
    const int m = q.rhi - q.rlo, n = q.chi - q.clo, k = C.h_rank[b];
    const int64_t bytes = 8 * (int64_t)k * (m + n);
    if (bytes <= kMvSmallMax && m <= 2047 && n <= 2047 && k <= 1023) {
      items.push_back(Item{8 * C.h_foff[b], bytes, 1, q.rlo, q.clo, n,
                           (uint32_t)m | ((uint32_t)n << 11) | ((uint32_t)k << 22)});
    } else {
      large.push_back(MvLarge{q.rlo, q.clo, m, n, k, 0, C.h_foff[b], tl});
      tl += k;
    }
  }
  // Batches: consecutive items filling one stage = [header + task records | x_sigma ranges |
  // storage runs].  x ranges are 16-B aligned supersets [clo & ~1, (clo + n + 1) & ~1) in
  // doubles, shared by the leaves of a batch with the same sigma; storage runs are maximal
  // runs of contiguous items (16-B aligned supersets), one bulk copy each.
  std::vector<MvBatch> batches;
  std::vector<MvSeg> segs;
  std::vector<MvTask> stream;     // per batch: header {count,0,0,0} + count task records
  stream.reserve(items.size() + items.size() / 4 + 16);
  struct XR { int64_t a0, a1; };
  struct Run { int base; int64_t a0, a1, end; };
  std::vector<XR> xr;
  std::vector<Run> runs;
  std::vector<int> item_x, item_run;
  for (size_t i = 0; i < items.size();) {
    xr.clear(); runs.clear(); item_x.clear(); item_run.clear();
    int64_t xb = 0, db = 0;
    size_t j = i;
    for (; j < items.size(); ++j) {
      const Item& it = items[j];
      const int64_t xa0 = it.clo & ~int64_t(1), xa1 = (it.clo + it.n + 1) & ~int64_t(1);
      int xi = -1;
      for (int r = (int)xr.size() - 1; r >= 0 && r >= (int)xr.size() - 8; --r)
        if (xr[r].a0 <= xa0 && xa1 <= xr[r].a1) { xi = r; break; }
      const int64_t xcost = xi >= 0 ? 0 : 8 * (xa1 - xa0);
      const bool ext = !runs.empty() && runs.back().base == it.base && runs.back().end == it.byte0;
      const int64_t ra0 = ext ? runs.back().a0 : (it.byte0 & ~int64_t(15));
      const int64_t ra1 = (it.byte0 + it.bytes + 15) & ~int64_t(15);
      const int64_t dcost = ext ? ra1 - runs.back().a1 : ra1 - ra0;
      const int64_t hb = 16 * (int64_t)(item_x.size() + 2);
      if (hb + xb + xcost + db + dcost > kMvStageBytes) break;
      if (xi < 0) { xr.push_back(XR{xa0, xa1}); xi = (int)xr.size() - 1; }
      xb += xcost;
      if (ext) { runs.back().a1 = ra1; runs.back().end = it.byte0 + it.bytes; }
      else runs.push_back(Run{it.base, ra0, ra1, it.byte0 + it.bytes});
      db += dcost;
      item_x.push_back(xi);
      item_run.push_back((int)runs.size() - 1);
    }
    if (j == i) fail(HM_ERR_CUDA, "matvec plan: leaf larger than a pipeline stage");
    const int count = (int)(j - i);
    MvBatch B{};
    B.first_seg = (int32_t)segs.size();
    B.count = count;
    // layout
    const int64_t hbytes = 16 * (int64_t)(count + 1);
    std::vector<int64_t> xoff(xr.size()), roff(runs.size());
    int64_t off = hbytes;
    for (size_t r = 0; r < xr.size(); ++r) { xoff[r] = off; off += 8 * (xr[r].a1 - xr[r].a0); }
    for (size_t r = 0; r < runs.size(); ++r) { roff[r] = off; off += runs[r].a1 - runs[r].a0; }
    B.bytes = (int32_t)off;
    segs.push_back(MvSeg{16 * (int64_t)stream.size(), (uint16_t)hbytes, 0, 2, 0});
    for (size_t r = 0; r < xr.size(); ++r)
      segs.push_back(MvSeg{8 * xr[r].a0, (uint16_t)(8 * (xr[r].a1 - xr[r].a0)), (uint16_t)xoff[r], 3, 0});
    for (size_t r = 0; r < runs.size(); ++r)
      segs.push_back(MvSeg{runs[r].a0, (uint16_t)(runs[r].a1 - runs[r].a0), (uint16_t)roff[r], (uint16_t)runs[r].base, 0});
    B.nseg = (int32_t)segs.size() - B.first_seg;
    stream.push_back(MvTask{count, 0, 0, 0});
    for (int c = 0; c < count; ++c) {
      const Item& it = items[i + c];
      const XR& X = xr[item_x[c]];
      const Run& R = runs[item_run[c]];
      MvTask t;
      t.rlo = it.rlo;
      t.xoff = (int32_t)((xoff[item_x[c]] + 8 * (it.clo - X.a0)) / 8);
      t.loff = (int32_t)((roff[item_run[c]] + (it.byte0 - R.a0)) / 8);
      t.mnk = it.mnk;
      stream.push_back(t);
    }
    batches.push_back(B);
    i = j;
  }
  // byte-balanced contiguous batch ranges, one persistent CTA per SM
  int sms = 148;
  HM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, C.device));
  const int G = std::max(1, std::min<int>(sms, (int)batches.size()));
  std::vector<int32_t> cta_first(G + 1, (int32_t)batches.size());
  {
    double total = 0;
    for (auto& B : batches) total += B.bytes;
    double acc = 0;
    int g = 0;
    cta_first[0] = 0;
    for (size_t b = 0; b < batches.size() && g + 1 < G; ++b) {
      while (g + 1 < G && acc >= total * (g + 1) / G) cta_first[++g] = (int32_t)b;
      acc += batches[b].bytes;
    }
    while (g + 1 < G) cta_first[++g] = (int32_t)batches.size();
  }
  // tiles of the large low-rank blocks
  std::vector<MvTileV> tv;
  std::vector<MvTileU> tu;
  for (size_t i = 0; i < large.size(); ++i) {
    const MvLarge& B = large[i];
    for (int l0 = 0; l0 < B.k; l0 += 8)
      for (int j0 = 0; j0 < B.n; j0 += 2048) tv.push_back(MvTileV{(int32_t)i, l0, j0, std::min(B.n, j0 + 2048)});
    const int rows = 256;
    for (int t0 = 0; t0 < B.m; t0 += rows) tu.push_back(MvTileU{(int32_t)i, t0, std::min(B.m, t0 + rows), 0});
  }
  auto up = [&](auto& dbuf, const auto& v) {
    dbuf.alloc(v.size());
    if (!v.empty())
      HM_CUDA(cudaMemcpyAsync(dbuf.get(), v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice, st));
  };
  up(C.mv_batches, batches);
  up(C.mv_segs, segs);
  up(C.mv_tasks, stream);
  up(C.mv_cta, cta_first);
  up(C.mv_large, large);
  up(C.mv_dense_big, dense_big);
  up(C.mv_tiles_v, tv);
  up(C.mv_tiles_u, tu);
  C.mv_grid = G;
  C.mv_nbatches = (int64_t)batches.size();
  C.mv_tbuf.alloc(tl + 1);
  C.mv_n_large = (int64_t)large.size();
  C.mv_n_dense_big = (int64_t)dense_big.size();
  C.mv_n_tiles_v = (int64_t)tv.size();
  C.mv_n_tiles_u = (int64_t)tu.size();
  C.mv_tlen = tl;
  C.n_lr_small = (int64_t)(lr_order.size() - large.size());
  C.n_lr_large = (int64_t)large.size();
  HM_CUDA(cudaStreamSynchronize(st));
  static bool attr = false;
  if (!attr) {
    const int smem = 128 + kMvStages * kMvStageBytes;
    HM_CUDA(cudaFuncSetAttribute(k_mv_batched, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
}

void gather_perm(Context& C, const double* x_app, double* x_int) {
  k_gather<<<grid_for(C.N, 256), 256, 0, C.stream>>>(x_app, C.perm.get(), C.N, x_int);
  HM_CHECK_LAUNCH();
}

void scatter_perm(Context& C, const double* y_int, double* y_app) {
  k_scatter<<<grid_for(C.N, 256), 256, 0, C.stream>>>(y_int, C.perm.get(), C.N, y_app);
  HM_CHECK_LAUNCH();
}

// y_int = (local leaves of H) x_int, then summed over ranks
void matvec_internal(Context& C, const double* x_int, double* y_int) {
  cudaStream_t st = C.stream;
  // the staged x_sigma copies need a 16-B aligned x with one readable double past N (every
  // internal caller passes such a vector; anything else goes through an aligned copy)
  if (reinterpret_cast<uintptr_t>(x_int) & 15) {
    C.work.alloc(C.N + 2);
    HM_CUDA(cudaMemcpyAsync(C.work.get(), x_int, C.N * sizeof(double), cudaMemcpyDeviceToDevice, st));
    x_int = C.work.get();
  }
  std::unique_ptr<KScope> ks(new KScope(C, KF_MATVEC));
  HM_CUDA(cudaMemsetAsync(y_int, 0, C.N * sizeof(double), st));
  if (C.mv_tlen) HM_CUDA(cudaMemsetAsync(C.mv_tbuf.get(), 0, C.mv_tlen * sizeof(double), st));
  const double* pool = (const double*)C.fpool.base;
  if (C.mv_nbatches) {
    const int smem = 128 + kMvStages * kMvStageBytes;
    k_mv_batched<<<C.mv_grid, kMvThreads, smem, st>>>(C.mv_batches.get(), C.mv_segs.get(), C.mv_cta.get(),
                                                       (const char*)C.dstore.get(), (const char*)pool,
                                                       (const char*)C.mv_tasks.get(), x_int, y_int);
    HM_CHECK_LAUNCH();
  }
  if (C.mv_n_dense_big) {
    k_mv_dense_direct<<<148 * 8, 256, 0, st>>>(C.mv_dense_big.get(), C.mv_n_dense_big, C.dstore.get(),
                                               x_int, y_int);
    HM_CHECK_LAUNCH();
  }
  if (C.mv_n_tiles_v) {
    k_mv_large_v<<<148 * 8, 256, 0, st>>>(C.mv_tiles_v.get(), C.mv_n_tiles_v, C.mv_large.get(), pool, x_int,
                                          C.mv_tbuf.get());
    HM_CHECK_LAUNCH();
    k_mv_large_u<<<148 * 8, 256, 0, st>>>(C.mv_tiles_u.get(), C.mv_n_tiles_u, C.mv_large.get(), pool,
                                          C.mv_tbuf.get(), y_int);
    HM_CHECK_LAUNCH();
  }
  ks.reset();
  if (C.world > 1) allreduce_sum(C, y_int, C.N);
}

}  // namespace hm
