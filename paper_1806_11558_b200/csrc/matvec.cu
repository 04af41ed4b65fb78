// matvec.cu — batched H-matrix-vector product: non-admissible leaves apply their
// stored dense block, admissible leaves apply U (V^T x) ("two matrix-vector
// products of skinny matrices"); application <-> internal permutation at the ends.
//
// Memory-bound (0.25 flop/B): the stored H is streamed from HBM exactly once per product.
//
//   small leaves   (dense blocks and low-rank blocks with (m+n)k*8 <= 16 KiB, ~90% of leaves):
//                  k_mv_batched — persistent CTAs (two per SM by default), each over a
//                  contiguous, byte-balanced range of "batches" (48 KiB shared-memory stages:
//                  task records | x_sigma ranges | leaf storage).  Warp 0 streams the batch /
//                  segment descriptors through register windows and issues each batch's bulk
//                  copies (cp.async.bulk, mbarrier completion) from its 32 lanes; the consumer
//                  warps compute the staged batches entirely out of shared memory and release
//                  each stage through an "empty" mbarrier.  One FP64 atomic per row into the
//                  L2-resident y.
//   large low-rank (blocks above 16 KiB): two barrier-free warp-task kernels with direct
//                  coalesced loads, k_mv_large_v (t += V^T x over 16-column x 1024-row tiles,
//                  one atomic per column into t) then k_mv_large_u (y += U t, 256-row tiles,
//                  8 rows per lane in registers).
//   dense blocks too big for a stage (only with large leaf_size): k_mv_dense_direct.

#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <thread>

#include "entry.cuh"

namespace hm {

constexpr int kMvStageBytes = 48 * 1024;   // one k_mv_batched pipeline stage (= one batch)
// stage bytes of option mv_kernel: 0 two CTAs x 2 x 48 KiB (default), 1 one CTA x 4 x 48 KiB,
// 2 two CTAs x 3 x 36 KiB, 3 two CTAs x 2 x 56 KiB
// 4 two CTAs x 4 x 24 KiB, 5 two CTAs x 3 x 32 KiB
inline int64_t mv_stage_bytes(const Context& C) {
  switch (C.mv_kind) {
    case 2: return 36 * 1024;
    case 3: return 56 * 1024;
    case 4: return 24 * 1024;
    case 5: return 32 * 1024;
    default: return kMvStageBytes;
  }
}
constexpr int kMaxX = 12;         // x_sigma ranges (bulk copies) per batch
constexpr int64_t kXGap = 64;     // doubles: merge x ranges closer than this

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
#pragma unroll 2
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

// Warp sum of KB per-lane values (KB = 8 or 16) by recursive halving (KB - 1 shuffles + the
// last levels), then every lane gets all KB totals back (KB shuffles): 2 KB + 1 shuffles
// instead of 5 KB for KB independent butterflies.
template <int KB>
__device__ __forceinline__ void warp_allreduce_vec(double (&a)[KB], int lane) {
  constexpr int LV = KB == 16 ? 4 : 3;           // halving levels: offsets 16, 8, (4, (2))
  double v[KB];
#pragma unroll
  for (int i = 0; i < KB; ++i) v[i] = a[i];
#pragma unroll
  for (int lvl = 0; lvl < LV; ++lvl) {
    const int o = 16 >> lvl, half = (KB >> 1) >> lvl;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < KB / 2; ++i)
      if (i < half) {
        const double send = up ? v[i] : v[i + half];
        const double keep = up ? v[i + half] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
  }
#pragma unroll
  for (int o = 16 >> LV; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  // lane L now holds the total of index sum_j bit(L, 4 - j) << (LV - 1 - j)
#pragma unroll
  for (int l = 0; l < KB; ++l) {
    int src = 0;
#pragma unroll
    for (int j = 0; j < LV; ++j) src |= ((l >> (LV - 1 - j)) & 1) << (4 - j);
    a[l] = __shfl_sync(0xffffffffu, v[0], src);
  }
}

// Low-rank block U (m x k) | V (n x k), column-major, columns [l0, l0 + kc) (kc <= KB), out of
// shared memory: t = V^T x with all kc column sums in registers, one vector all-reduce over
// the warp, then y += U t (one FP64 atomic per row).
// T = float: binary32 factors (option lr_f32), widened exactly to FP64 before every FMA.
template <int KB, class T>
__device__ __forceinline__ void lowrank_block(const T* __restrict__ U0, int m, int n, int k, int l0, int kc,
                                              const double* __restrict__ xs, double* __restrict__ y, int lane) {
  const T* V = U0 + m * k + l0 * n;
  const T* U = U0 + l0 * m;
  double acc[KB];
#pragma unroll
  for (int l = 0; l < KB; ++l) acc[l] = 0.0;
#pragma unroll 2
  for (int j = lane; j < n; j += 32) {
    const double xj = xs[j];
#pragma unroll
    for (int l = 0; l < KB; ++l)
      if (l < kc) acc[l] = __fma_rn((double)V[j + l * n], xj, acc[l]);
  }
  warp_allreduce_vec<KB>(acc, lane);
  for (int t = lane; t < m; t += 32) {
    double s0 = 0.0, s1 = 0.0;                  // two chains: half the dependent-FMA latency
#pragma unroll
    for (int l = 0; l < KB; l += 2) {
      if (l < kc) s0 = __fma_rn((double)U[t + l * m], acc[l], s0);
      if (l + 1 < kc) s1 = __fma_rn((double)U[t + (l + 1) * m], acc[l + 1], s1);
    }
    atomicAdd(y + t, s0 + s1);
  }
}

template <class T>
__device__ __forceinline__ void lowrank_any(const T* U, int m, int n, int k, const double* xs, double* y, int lane) {
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
// A sequence of 16-byte records read through two 32-record register windows (one record per
// lane): record i is available for w0 <= i < w0 + 64; advancing past a window issues the load
// of the window after next, 32 records ahead of use.  Warp-collective.
struct RecWindow {
  const int4* src;
  int64_t w0, end;
  int4 cur, nxt;
  __device__ __forceinline__ int4 load(int64_t i) const { return i < end ? __ldg(src + i) : make_int4(0, 0, 0, 0); }
  __device__ __forceinline__ void init(const int4* p, int64_t begin, int64_t e, int lane) {
    src = p; w0 = begin; end = e;
    cur = load(w0 + lane);
    nxt = load(w0 + 32 + lane);
  }
  __device__ __forceinline__ void advance_to(int64_t i, int lane) {
    while (i >= w0 + 32) { cur = nxt; w0 += 32; nxt = load(w0 + 32 + lane); }
  }
  __device__ __forceinline__ int4 get(int64_t i, int lane) const {
    const int64_t d = i - w0;
    const int sl = (int)(d & 31);
    int4 a, b;
    a.x = __shfl_sync(0xffffffffu, cur.x, sl); a.y = __shfl_sync(0xffffffffu, cur.y, sl);
    a.z = __shfl_sync(0xffffffffu, cur.z, sl); a.w = __shfl_sync(0xffffffffu, cur.w, sl);
    b.x = __shfl_sync(0xffffffffu, nxt.x, sl); b.y = __shfl_sync(0xffffffffu, nxt.y, sl);
    b.z = __shfl_sync(0xffffffffu, nxt.z, sl); b.w = __shfl_sync(0xffffffffu, nxt.w, sl);
    return d < 32 ? a : b;
  }
};

template <int STAGES, int SBYTES, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
    k_mv_batched(const MvBatch* __restrict__ batches, const MvSeg* __restrict__ segs, int64_t nsegs_total,
                 const int32_t* __restrict__ cta_first,
                 const char* __restrict__ base0, const char* __restrict__ base1, const char* __restrict__ base2,
                 const double* __restrict__ x, double* __restrict__ y, int64_t scramble_n,
                 unsigned long long* __restrict__ prof, int lr32) {
  constexpr int NW = THREADS / 32, NC = NW - 1;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + STAGES;
  // per-stage task counters (dynamic task assignment: a warp takes the next task of the stage
  // when it is free, so the stage is released one task after the average, not after the
  // round-robin share of the slowest warp); reset by the producer before it refills the stage
  int* tctr = reinterpret_cast<int*>(empty + STAGES);
  unsigned char* buf = smem + 256;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b0 = cta_first[blockIdx.x], nb = cta_first[blockIdx.x + 1] - b0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long pw_empty = 0;
  if (warp == 0) {
    // batch and segment descriptors stream through register windows 32-64 records ahead, so
    // no descriptor read sits on the producer's critical path
    RecWindow wb, ws;
    wb.init(reinterpret_cast<const int4*>(batches), b0, b0 + nb, lane);
    bool ws_ready = false;
    for (int it = 0; it < nb; ++it) {
      const int stage = it % STAGES;
      wb.advance_to(b0 + it, lane);
      const int4 Bv = wb.get(b0 + it, lane);
      const int first_seg = Bv.x, nseg = Bv.y, bytes = Bv.z;
      if (!ws_ready) { ws.init(reinterpret_cast<const int4*>(segs), first_seg, nsegs_total, lane); ws_ready = true; }
      const long long tw0 = prof ? clock64() : 0;
      if (it >= STAGES) mbar_wait(&empty[stage], (unsigned)(((it / STAGES) - 1) & 1));
      if (prof && lane == 0) pw_empty += clock64() - tw0;
      if (lane == 0) {
        tctr[stage] = 0;                       // ordered before the consumers' full-wait by the arrive
        mbar_expect_tx(&full[stage], (unsigned)bytes);
      }
      __syncwarp();
      unsigned char* sb = buf + stage * SBYTES;
      for (int s0 = 0; s0 < nseg; s0 += 32) {
        ws.advance_to(first_seg + s0, lane);
        const int4 Sv = ws.get(first_seg + s0 + lane, lane);
        if (s0 + lane < nseg) {
          const int64_t src = (int64_t)(((uint64_t)(uint32_t)Sv.y << 32) | (uint32_t)Sv.x);
          const unsigned sbytes = (uint32_t)Sv.z & 0xffffu, dst = (uint32_t)Sv.z >> 16, sbase = (uint32_t)Sv.w & 0xffffu;
          const char* base = sbase == 0 ? base0 : sbase == 1 ? base1 : sbase == 2 ? base2
                                                                 : reinterpret_cast<const char*>(x);
          bulk_g2s(sb + dst, base + src, sbytes, &full[stage]);
        }
      }
    }
    if (prof && lane == 0) atomicAdd(&prof[0], (unsigned long long)pw_empty);
    return;
  }
  long long cw_full = 0, cw_work = 0;
  for (int it = 0; it < nb; ++it) {
    const int stage = it % STAGES;
    const long long t0 = prof ? clock64() : 0;
    mbar_wait(&full[stage], (unsigned)((it / STAGES) & 1));
    const long long t1 = prof ? clock64() : 0;
    cw_full += t1 - t0;
    const unsigned char* sb = buf + stage * SBYTES;
    const double* sd = reinterpret_cast<const double*>(sb);
    const int4* rec = reinterpret_cast<const int4*>(sb);
    const int count = rec[0].x;
    for (;;) {
      int t = 0;
      if (lane == 0) t = atomicAdd(&tctr[stage], 1);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= count) break;
      const int4 T = rec[1 + t];
      const uint32_t mnk = (uint32_t)T.w;
      const int m = mnk & 2047, n = (mnk >> 11) & 2047, k = mnk >> 22;
      // scramble_n > 0: diagnostic only (wrong result) — task row bases spread over y, to
      // measure same-address atomic contention
      const int64_t r0 = scramble_n > 0 ? ((int64_t)T.x * 2654435761ll) % scramble_n : T.x;
      if (k == 0) dense_any(sd + T.z, m, n, sd + T.y, y + r0, lane);
      else if (lr32) lowrank_any(reinterpret_cast<const float*>(sb) + T.z, m, n, k, sd + T.y, y + r0, lane);
      else lowrank_any(sd + T.z, m, n, k, sd + T.y, y + r0, lane);
    }
    __syncwarp();
    if (prof) cw_work += clock64() - t1;
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[stage])) : "memory");
  }
  if (prof && lane == 0) {
    atomicAdd(&prof[1], (unsigned long long)cw_full);
    atomicAdd(&prof[2], (unsigned long long)cw_work);
  }
}

// Large low-rank blocks (storage > 16 KiB), barrier-free warp tasks with direct coalesced loads.
// Phase 1, tile = (block, 16 columns l0.., 1024 rows j0..): t[l] += sum_j V[j, l] x[clo + j];
// all 16 column sums in registers, two rows per lane per pass (32 independent loads), one
// halving butterfly for the 16 sums, one atomic per column.
template <int KB>
__device__ __forceinline__ void warp_reduce_halving(double (&v)[KB], int lane) {
  constexpr int LV = KB == 16 ? 4 : 3;
#pragma unroll
  for (int lvl = 0; lvl < LV; ++lvl) {
    const int o = 16 >> lvl, half = (KB >> 1) >> lvl;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < KB / 2; ++i)
      if (i < half) {
        const double send = up ? v[i] : v[i + half];
        const double keep = up ? v[i + half] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
  }
#pragma unroll
  for (int o = 16 >> LV; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
}

// binary32 factors: every widening must wait for the LAST raw load, else ptxas issues each
// F2F right behind its load and the in-order warp stalls once per load (measured 1.8 TB/s).
// zmask is 0 at run time but opaque to the compiler: OR-ing (all raw bits & zmask) into each
// value makes every widening depend on every load, so all loads issue first.
template <int K>
__device__ __forceinline__ void order_after_all_loads(float (&a)[K], float (&b)[K], unsigned zmask) {
  unsigned z = 0;
#pragma unroll
  for (int l = 0; l < K; ++l) z |= __float_as_uint(a[l]) | __float_as_uint(b[l]);
  z &= zmask;
#pragma unroll
  for (int l = 0; l < K; ++l) {
    a[l] = __uint_as_float(__float_as_uint(a[l]) | z);
    b[l] = __uint_as_float(__float_as_uint(b[l]) | z);
  }
}
template <int K>
__device__ __forceinline__ void order_after_all_loads(double (&)[K], double (&)[K], unsigned) {}

template <class E>
__global__ void __launch_bounds__(256) k_mv_large_v(const MvTileV* __restrict__ tiles, int64_t ntiles,
                                                      const MvLarge* __restrict__ L, const E* __restrict__ pool,
                                                      const double* __restrict__ x, double* __restrict__ tbuf,
                                                      unsigned zmask) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < ntiles; i += nw) {
    const MvTileV T = tiles[i];
    const MvLarge B = L[T.blk];
    const int kc = min(16, B.k - T.l);
    const E* V = pool + B.off + (int64_t)B.m * B.k + (int64_t)T.l * B.n;
    const double* xs = x + B.clo;
    double acc[16];
#pragma unroll
    for (int l = 0; l < 16; ++l) acc[l] = 0.0;
    for (int j = T.j0 + lane; j < T.j1; j += 64) {
      const bool two = j + 32 < T.j1;
      const double xa = __ldg(xs + j), xb = two ? __ldg(xs + j + 32) : 0.0;
      // the raw factor loads all issue before the first use (binary32: widening each load
      // right after it would stall the warp on every load)
      E va[16], vb[16];
#pragma unroll
      for (int l = 0; l < 16; ++l) {
        va[l] = l < kc ? __ldg(V + j + (int64_t)l * B.n) : E(0);
        vb[l] = (l < kc && two) ? __ldg(V + j + 32 + (int64_t)l * B.n) : E(0);
      }
      order_after_all_loads<16>(va, vb, zmask);
#pragma unroll
      for (int l = 0; l < 16; ++l) acc[l] = __fma_rn((double)vb[l], xb, __fma_rn((double)va[l], xa, acc[l]));
    }
    warp_reduce_halving<16>(acc, lane);
    // lane L holds column 8*b4 + 4*b3 + 2*b2 + b1 (two lanes per column)
    const int col = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
    if ((lane & 1) == 0 && col < kc) atomicAdd(tbuf + B.toff + T.l + col, acc[0]);
  }
}

// Phase 2, tile = (block, 256 rows t0..): y[rlo + t] += sum_l U[t, l] t_l; each lane keeps its
// 8 rows of the tile in registers: per column l one broadcast t_l and 8 independent loads of U.
template <class E>
__global__ void __launch_bounds__(256) k_mv_large_u(const MvTileU* __restrict__ tiles, int64_t ntiles,
                                                     const MvLarge* __restrict__ L, const E* __restrict__ pool,
                                                     const double* __restrict__ tbuf, double* __restrict__ y,
                                                     unsigned zmask) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < ntiles; i += nw) {
    const MvTileU T = tiles[i];
    const MvLarge B = L[T.blk];
    const E* U = pool + B.off + T.t0 + lane;
    const double* tl = tbuf + B.toff;
    const int rows = T.t1 - T.t0;
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    int l = 0;
    for (; l + 1 < B.k; l += 2) {
      const double ta = __ldg(tl + l), tb = __ldg(tl + l + 1);
      const E* Ua = U + (int64_t)l * B.m;
      const E* Ub = Ua + B.m;
      E ua[8], ub[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const bool ok = lane + 32 * q < rows;
        ua[q] = ok ? __ldg(Ua + 32 * q) : E(0);
        ub[q] = ok ? __ldg(Ub + 32 * q) : E(0);
      }
      order_after_all_loads<8>(ua, ub, zmask);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = __fma_rn((double)ub[q], tb, __fma_rn((double)ua[q], ta, acc[q]));
    }
    if (l < B.k) {
      const double ta = __ldg(tl + l);
      const E* Ua = U + (int64_t)l * B.m;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (lane + 32 * q < rows) acc[q] = __fma_rn((double)__ldg(Ua + 32 * q), ta, acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (lane + 32 * q < rows) atomicAdd(y + B.rlo + T.t0 + lane + 32 * q, acc[q]);
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

// ---- plan (host) ----------------------------------------------------------------------------
namespace {
struct Item { int64_t byte0, bytes; int base; int32_t rlo, clo, n; uint32_t mnk; };
// one planner thread's output over a contiguous slice of the item sequence
struct PlanPart {
  int lr_esz = 8;                      // bytes per factor entry (task offsets of low-rank items)
  std::vector<MvBatch> batches;
  std::vector<MvSeg> segs;
  std::vector<MvTask> stream;
  std::vector<MvLarge> dense_big, large;
  std::vector<Item> items;
  struct XR { int64_t a0, a1; };
  struct Run { int base; int64_t a0, a1, end; };
  std::vector<XR> xr;
  std::vector<Run> runs;
  std::vector<int> item_x, item_run;
  std::vector<int64_t> xoff, roff;
  void clear() {
    batches.clear(); segs.clear(); stream.clear(); dense_big.clear(); large.clear(); items.clear();
  }
  // Batches over items[0, n): consecutive items filling one stage = [header + task records |
  // x_sigma ranges | storage runs].  x ranges are 16-B aligned supersets [clo & ~1,
  // (clo + n + 1) & ~1) in doubles, shared by the leaves of a batch with the same sigma;
  // storage runs are maximal runs of contiguous items (16-B aligned supersets), one bulk copy
  // each.  Stream offsets (base 2) are local to the part and shifted when parts are joined.
  void batch(int64_t cap) {
    for (size_t i = 0; i < items.size();) {
      xr.clear(); runs.clear(); item_x.clear(); item_run.clear();
      int64_t xb = 0, db = 0;
      size_t j = i;
      for (; j < items.size(); ++j) {
        const Item& it = items[j];
        const int64_t xa0 = it.clo & ~int64_t(1), xa1 = (it.clo + it.n + 1) & ~int64_t(1);
        // x_sigma: reuse / widen a staged range within kXGap doubles, else a new range (a
        // batch holds at most kMaxX ranges: more small bulk copies per stage cost bandwidth,
        // tools/tma_stream_bench.cu)
        int xi = -1;
        int64_t xcost = 8 * (xa1 - xa0);
        for (int r = (int)xr.size() - 1; r >= 0; --r)
          if (xa0 <= xr[r].a1 + kXGap && xr[r].a0 <= xa1 + kXGap) {
            const int64_t c = 8 * ((std::max(xr[r].a1, xa1) - std::min(xr[r].a0, xa0)) - (xr[r].a1 - xr[r].a0));
            if (xi < 0 || c < xcost) { xi = r; xcost = c; }
          }
        if (xi < 0 && (int)xr.size() >= kMaxX) break;
        const bool ext = !runs.empty() && runs.back().base == it.base && runs.back().end == it.byte0;
        const int64_t ra0 = ext ? runs.back().a0 : (it.byte0 & ~int64_t(15));
        const int64_t ra1 = (it.byte0 + it.bytes + 15) & ~int64_t(15);
        const int64_t dcost = ext ? ra1 - runs.back().a1 : ra1 - ra0;
        const int64_t hb = 16 * (int64_t)(item_x.size() + 2);
        if (hb + xb + xcost + db + dcost > cap) break;
        if (xi < 0) { xr.push_back(XR{xa0, xa1}); xi = (int)xr.size() - 1; }
        else { xr[xi].a0 = std::min(xr[xi].a0, xa0); xr[xi].a1 = std::max(xr[xi].a1, xa1); }
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
      const int64_t hbytes = 16 * (int64_t)(count + 1);
      xoff.resize(xr.size());
      roff.resize(runs.size());
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
        t.loff = (int32_t)((roff[item_run[c]] + (it.byte0 - R.a0)) / (it.base == 1 ? lr_esz : 8));
        t.mnk = it.mnk;
        stream.push_back(t);
      }
      batches.push_back(B);
      i = j;
    }
  }
};
}  // namespace

struct PlanWs {
  std::vector<int64_t> hoff, lr_order;
  std::vector<PlanPart> parts;       // dense parts [0, nd_parts), then low-rank parts
  int nd_parts = 0;
  std::thread dense_thread;          // plans the dense leaves while ACA runs on the GPU
  std::exception_ptr dense_err;
  bool dense_started = false;
  ~PlanWs() { if (dense_thread.joinable()) dense_thread.join(); }
  PinnedVec<MvBatch> batches;
  PinnedVec<MvSeg> segs;
  PinnedVec<MvTask> stream;
  PinnedVec<MvLarge> large, dense_big;
  PinnedVec<MvTileV> tv;
  PinnedVec<MvTileU> tu;
  PinnedVec<int32_t> cta;
};

// The matvec plan, built on the host by T threads over contiguous slices of the item sequence
// (owned dense leaves in list order, then owned low-rank leaves in factor-pool order); batches
// never straddle two slices.
namespace {
// Items of the leaf sequence slice [i0, i1) -> one part's batches.  Dense leaves: sequence
// position = owned dense index; low-rank leaves: position in lr_order.
void plan_dense_part(Context& C, PlanWs& W, PlanPart& P, int64_t i0, int64_t i1) {
  P.clear();
  P.items.reserve(i1 - i0);
  const int64_t cap = mv_stage_bytes(C);
  const int64_t* hoff = W.hoff.data();
  for (int64_t b = i0; b < i1; ++b) {
    const Quad& q = C.h_dense[C.dense_begin + b];
    const int m = q.rhi - q.rlo, n = q.chi - q.clo;
    const int64_t bytes = 8 * (int64_t)m * n;
    if (bytes + 8 * n + 64 > cap || m > 2047 || n > 2047)
      P.dense_big.push_back(MvLarge{q.rlo, q.clo, m, n, 0, 0, hoff[b], 0});
    else
      P.items.push_back(Item{8 * hoff[b], bytes, 0, q.rlo, q.clo, n, (uint32_t)m | ((uint32_t)n << 11)});
  }
  P.batch(cap);
}
void plan_lowrank_part(Context& C, PlanWs& W, PlanPart& P, int64_t i0, int64_t i1) {
  P.clear();
  P.items.reserve(i1 - i0);
  P.lr_esz = C.lr_esz;
  const int64_t cap = mv_stage_bytes(C), esz = C.lr_esz;
  for (int64_t i = i0; i < i1; ++i) {
    const int64_t b = W.lr_order[i];
    const Quad& q = C.h_adm[C.adm_begin + b];
    const int m = q.rhi - q.rlo, n = q.chi - q.clo, k = C.h_rank[b];
    const int64_t bytes = esz * (int64_t)k * (m + n);
    if (bytes <= std::min<int64_t>(C.mv_small_max, cap - 8 * n - 64) && m <= 2047 && n <= 2047 && k <= 1023)
      P.items.push_back(Item{esz * C.h_foff[b], bytes, 1, q.rlo, q.clo, n,
                             (uint32_t)m | ((uint32_t)n << 11) | ((uint32_t)k << 22)});
    else
      P.large.push_back(MvLarge{q.rlo, q.clo, m, n, k, 0, C.h_foff[b], 0});
  }
  P.batch(cap);
}
// run f(t) for t in [0, T) on T host threads (the caller's thread included)
template <class F>
void run_threads(int T, F&& f) {
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(T);
  for (int t = 1; t < T; ++t)
    th.emplace_back([&, t]() { try { f(t); } catch (...) { err[t] = std::current_exception(); } });
  try { f(0); } catch (...) { err[0] = std::current_exception(); }
  for (auto& x : th) x.join();
  for (auto& e : err) if (e) std::rethrow_exception(e);
}
int planner_threads(Context& C, int64_t work) {
  // the host's cores shared by the ranks of this node (one process per GPU)
  const int64_t hw = std::max<int64_t>(1, (int64_t)std::thread::hardware_concurrency() / std::max(1, C.world));
  return (int)std::max<int64_t>(1, std::min<int64_t>({hw, 16, work / 20000 + 1}));
}
}  // namespace

// Dense half of the matvec plan: depends only on the tree and the near-field offsets, so it
// is planned on host threads while ACA runs on the GPU (joined by plan_matvec).
void plan_dense_begin(Context& C) {
  if (!C.plan_ws) C.plan_ws = std::make_shared<PlanWs>();
  PlanWs& W = *C.plan_ws;
  if (W.dense_thread.joinable()) W.dense_thread.join();
  const int64_t nd = C.dense_end - C.dense_begin;
  W.hoff.resize(nd + 1);
  HM_CUDA(cudaMemcpyAsync(W.hoff.data(), C.doff.get(), (nd + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, C.stream));
  if (C.h_dense.size() != (size_t)C.ndense) {
    C.h_dense.resize(C.ndense);
    HM_CUDA(cudaMemcpyAsync(C.h_dense.data(), C.dense.get(), C.ndense * sizeof(Quad), cudaMemcpyDeviceToHost, C.stream));
  }
  HM_CUDA(cudaStreamSynchronize(C.stream));
  // leave cores for the setup thread that keeps launching ACA kernels meanwhile
  const int64_t hw = std::max<int64_t>(1, (int64_t)std::thread::hardware_concurrency() / std::max(1, C.world));
  const int Td = std::max(1, std::min<int>(planner_threads(C, nd), (int)hw - 2));
  W.nd_parts = Td;
  if (W.parts.size() < (size_t)Td) W.parts.resize(Td);
  W.dense_err = nullptr;
  W.dense_started = true;
  Context* pc = &C;
  W.dense_thread = std::thread([pc, &W, Td, nd]() {
    try {
      run_threads(Td, [&](int t) { plan_dense_part(*pc, W, W.parts[t], nd * t / Td, nd * (t + 1) / Td); });
    } catch (...) {
      W.dense_err = std::current_exception();
    }
  });
}

// Join a dense planner thread that is still running (hm_setup failed between
// plan_dense_begin and plan_matvec, or the tree is being rebuilt): it reads h_dense,
// dense_begin and the offsets, which hm_build_tree is about to rewrite.
void plan_dense_abort(Context& C) {
  if (!C.plan_ws) return;
  PlanWs& W = *C.plan_ws;
  if (W.dense_thread.joinable()) W.dense_thread.join();
  W.dense_started = false;
  W.dense_err = nullptr;
}

// The matvec plan, built on the host by threads over contiguous slices of the item sequence
// (owned dense leaves in list order — planned during ACA by plan_dense_begin — then owned
// low-rank leaves in block order); batches never straddle two slices.
void plan_matvec(Context& C) {
  cudaStream_t st = C.stream;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  if (!C.plan_ws) C.plan_ws = std::make_shared<PlanWs>();
  PlanWs& W = *C.plan_ws;
  if (!W.dense_started) plan_dense_begin(C);        // re-plan (options) or no overlap
  W.dense_thread.join();
  W.dense_started = false;
  if (W.dense_err) std::rethrow_exception(W.dense_err);
  const int64_t na = C.adm_end - C.adm_begin;
  std::vector<int64_t>& lr_order = W.lr_order;
  lr_order.clear();
  for (int64_t b = 0; b < na; ++b)
    if (C.h_rank[b] > 0) lr_order.push_back(b);
  // block order = factor-pool order except for the few blocks re-run after a workspace
  // overflow (stored at the end): they just become separate bulk-copy runs, no sort needed
  const int64_t nlr = (int64_t)lr_order.size();
  const int Td = W.nd_parts, Tl = planner_threads(C, nlr), T = Td + Tl;
  W.parts.resize(T);
  run_threads(Tl, [&](int t) { plan_lowrank_part(C, W, W.parts[Td + t], nlr * t / Tl, nlr * (t + 1) / Tl); });
  const auto t1 = clk::now();
  // join the parts: shift segment indices and task-stream offsets
  size_t nbat = 0, nseg = 0, nstr = 0, nlarge = 0, nbig = 0;
  for (auto& P : W.parts) {
    nbat += P.batches.size(); nseg += P.segs.size(); nstr += P.stream.size();
    nlarge += P.large.size(); nbig += P.dense_big.size();
  }
  W.batches.resize(nbat); W.segs.resize(nseg); W.stream.resize(nstr); W.large.resize(nlarge); W.dense_big.resize(nbig);
  {
    // per-part output offsets (exclusive prefix), then the parts are copied in parallel
    const size_t np = W.parts.size();
    std::vector<size_t> ob(np + 1, 0), os(np + 1, 0), ot(np + 1, 0), ol(np + 1, 0), od(np + 1, 0);
    std::vector<int64_t> tl(np + 1, 0);
    for (size_t p = 0; p < np; ++p) {
      const PlanPart& P = W.parts[p];
      ob[p + 1] = ob[p] + P.batches.size(); os[p + 1] = os[p] + P.segs.size();
      ot[p + 1] = ot[p] + P.stream.size(); ol[p + 1] = ol[p] + P.large.size();
      od[p + 1] = od[p] + P.dense_big.size();
      int64_t ks = 0;
      for (const MvLarge& L : P.large) ks += L.k;
      tl[p + 1] = tl[p] + ks;
    }
    run_threads((int)np, [&](int p) {
      const PlanPart& P = W.parts[p];
      size_t b = ob[p], g = os[p], l = ol[p], d = od[p];
      int64_t t = tl[p];
      for (const MvBatch& B : P.batches) { MvBatch x = B; x.first_seg += (int32_t)os[p]; W.batches[b++] = x; }
      for (const MvSeg& S : P.segs) { MvSeg x = S; if (x.base == 2) x.src += 16 * (int64_t)ot[p]; W.segs[g++] = x; }
      std::memcpy(W.stream.data() + ot[p], P.stream.data(), P.stream.size() * sizeof(MvTask));
      for (MvLarge L : P.large) { L.toff = t; t += L.k; W.large[l++] = L; }
      for (const MvLarge& L : P.dense_big) W.dense_big[d++] = L;
    });
    C.mv_tlen = tl[np];
  }
  const auto t2 = clk::now();
  // byte-balanced contiguous batch ranges, one per persistent CTA (two or one per SM)
  int sms = 148;
  HM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, C.device));
  const int G = std::max(1, std::min<int>(C.mv_kind == 1 ? sms : 2 * sms, (int)nbat));
  W.cta.resize(G + 1);
  {
    double tot = 0;
    for (size_t b = 0; b < nbat; ++b) tot += W.batches[b].bytes;
    for (int g = 0; g <= G; ++g) W.cta[g] = (int32_t)nbat;
    double acc = 0;
    int g = 0;
    W.cta[0] = 0;
    for (size_t b = 0; b < nbat && g + 1 < G; ++b) {
      while (g + 1 < G && acc >= tot * (g + 1) / G) W.cta[++g] = (int32_t)b;
      acc += W.batches[b].bytes;
    }
    while (g + 1 < G) W.cta[++g] = (int32_t)nbat;
  }
  // tiles of the large low-rank blocks
  const int vcols = 16, vrows = 1024;
  size_t ntv = 0, ntu = 0;
  for (size_t i = 0; i < nlarge; ++i) {
    const MvLarge& B = W.large[i];
    ntv += (size_t)((B.k + vcols - 1) / vcols) * ((B.n + vrows - 1) / vrows);
    ntu += (size_t)((B.m + 255) / 256);
  }
  W.tv.resize(ntv);
  W.tu.resize(ntu);
  {
    size_t a = 0, c = 0;
    for (size_t i = 0; i < nlarge; ++i) {
      const MvLarge& B = W.large[i];
      for (int l0 = 0; l0 < B.k; l0 += vcols)
        for (int j0 = 0; j0 < B.n; j0 += vrows) W.tv[a++] = MvTileV{(int32_t)i, l0, j0, std::min(B.n, j0 + vrows)};
      for (int t0 = 0; t0 < B.m; t0 += 256) W.tu[c++] = MvTileU{(int32_t)i, t0, std::min(B.m, t0 + 256), 0};
    }
  }
  auto up = [&](auto& dbuf, auto& v) {
    dbuf.alloc(v.size());
    if (v.size())
      HM_CUDA(cudaMemcpyAsync(dbuf.get(), v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice, st));
  };
  up(C.mv_batches, W.batches);
  up(C.mv_segs, W.segs);
  up(C.mv_tasks, W.stream);
  up(C.mv_cta, W.cta);
  up(C.mv_large, W.large);
  up(C.mv_dense_big, W.dense_big);
  up(C.mv_tiles_v, W.tv);
  up(C.mv_tiles_u, W.tu);
  C.mv_grid = G;
  C.mv_nbatches = (int64_t)nbat;
  C.mv_nsegs = (int64_t)nseg;
  C.mv_tbuf.alloc(C.mv_tlen + 1);
  C.mv_n_large = (int64_t)nlarge;
  C.mv_n_dense_big = (int64_t)nbig;
  C.mv_n_tiles_v = (int64_t)ntv;
  C.mv_n_tiles_u = (int64_t)ntu;
  C.n_lr_small = nlr - (int64_t)nlarge;
  C.n_lr_large = (int64_t)nlarge;
  HM_CUDA(cudaStreamSynchronize(st));
  const auto t3 = clk::now();
  C.times.plan_phase_ms[0] = std::chrono::duration<double, std::milli>(t1 - t0).count();
  C.times.plan_phase_ms[1] = std::chrono::duration<double, std::milli>(t2 - t1).count();
  C.times.plan_phase_ms[2] = std::chrono::duration<double, std::milli>(t3 - t2).count();
  static bool attr_done[64] = {false};            // function attributes are per device
  bool& attr = attr_done[C.device & 63];
  if (!attr) {
    HM_CUDA(cudaFuncSetAttribute(k_mv_batched<2, kMvStageBytes, 256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 256 + 2 * kMvStageBytes));
    HM_CUDA(cudaFuncSetAttribute(k_mv_batched<4, kMvStageBytes, 512, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 256 + 4 * kMvStageBytes));
    HM_CUDA(cudaFuncSetAttribute(k_mv_batched<3, 36 * 1024, 256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 256 + 3 * 36 * 1024));
    HM_CUDA(cudaFuncSetAttribute(k_mv_batched<2, 56 * 1024, 256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 256 + 2 * 56 * 1024));
    HM_CUDA(cudaFuncSetAttribute(k_mv_batched<4, 24 * 1024, 256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 256 + 4 * 24 * 1024));
    HM_CUDA(cudaFuncSetAttribute(k_mv_batched<3, 32 * 1024, 256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 256 + 3 * 32 * 1024));
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
void matvec_internal(Context& C, const double* x_int, double* y_int, bool reduce) {
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
  const float* pool32 = (const float*)C.fpool.base;     // option lr_f32
  const bool f32 = C.lr_esz == 4;
  auto large_v = [&](cudaStream_t s) {
    if (f32) k_mv_large_v<float><<<148 * 8, 256, 0, s>>>(C.mv_tiles_v.get(), C.mv_n_tiles_v, C.mv_large.get(), pool32,
                                                          x_int, C.mv_tbuf.get(), 0u);
    else k_mv_large_v<double><<<148 * 8, 256, 0, s>>>(C.mv_tiles_v.get(), C.mv_n_tiles_v, C.mv_large.get(), pool,
                                                       x_int, C.mv_tbuf.get(), 0u);
    HM_CHECK_LAUNCH();
  };
  auto large_u = [&](cudaStream_t s) {
    if (f32) k_mv_large_u<float><<<148 * 8, 256, 0, s>>>(C.mv_tiles_u.get(), C.mv_n_tiles_u, C.mv_large.get(), pool32,
                                                          C.mv_tbuf.get(), y_int, 0u);
    else k_mv_large_u<double><<<148 * 8, 256, 0, s>>>(C.mv_tiles_u.get(), C.mv_n_tiles_u, C.mv_large.get(), pool,
                                                       C.mv_tbuf.get(), y_int, 0u);
    HM_CHECK_LAUNCH();
  };
  // option mv_concurrent (default on): the large low-rank blocks (V^T x, then U z) stream on
  // a side stream while the CTA rings stream the small blocks, so one kernel family's tail
  // overlaps the other's streaming (C4: 27.9 -> 27.6 ms)
  const bool conc = C.mv_concurrent && C.mv_n_tiles_v && C.mv_nbatches;
  if (conc) {
    if (!C.mv_side) {
      HM_CUDA(cudaStreamCreateWithFlags(&C.mv_side, cudaStreamNonBlocking));
      HM_CUDA(cudaEventCreateWithFlags(&C.mv_ev[0], cudaEventDisableTiming));
      HM_CUDA(cudaEventCreateWithFlags(&C.mv_ev[1], cudaEventDisableTiming));
    }
    HM_CUDA(cudaEventRecord(C.mv_ev[0], st));
    HM_CUDA(cudaStreamWaitEvent(C.mv_side, C.mv_ev[0], 0));
    large_v(C.mv_side);
    large_u(C.mv_side);
    HM_CUDA(cudaEventRecord(C.mv_ev[1], C.mv_side));
  }
  if (C.mv_nbatches) {
    unsigned long long* prof = C.mv_prof.n ? C.mv_prof.get() : nullptr;
    const int64_t scramble = C.mv_scramble ? C.N - 4096 : 0;
    if (C.mv_kind == 0)      // two CTA rings per SM, 2 x 48 KiB stages, 7 consumer warps each
      k_mv_batched<2, kMvStageBytes, 256, 2><<<C.mv_grid, 256, 256 + 2 * kMvStageBytes, st>>>(
          C.mv_batches.get(), C.mv_segs.get(), C.mv_nsegs, C.mv_cta.get(), (const char*)C.dstore.get(), (const char*)pool,
          (const char*)C.mv_tasks.get(), x_int, y_int, scramble, prof, f32 ? 1 : 0);
    else if (C.mv_kind == 2)
      k_mv_batched<3, 36 * 1024, 256, 2><<<C.mv_grid, 256, 256 + 3 * 36 * 1024, st>>>(
          C.mv_batches.get(), C.mv_segs.get(), C.mv_nsegs, C.mv_cta.get(), (const char*)C.dstore.get(), (const char*)pool,
          (const char*)C.mv_tasks.get(), x_int, y_int, scramble, prof, f32 ? 1 : 0);
    else if (C.mv_kind == 3)
      k_mv_batched<2, 56 * 1024, 256, 2><<<C.mv_grid, 256, 256 + 2 * 56 * 1024, st>>>(
          C.mv_batches.get(), C.mv_segs.get(), C.mv_nsegs, C.mv_cta.get(), (const char*)C.dstore.get(), (const char*)pool,
          (const char*)C.mv_tasks.get(), x_int, y_int, scramble, prof, f32 ? 1 : 0);
    else if (C.mv_kind == 4)
      k_mv_batched<4, 24 * 1024, 256, 2><<<C.mv_grid, 256, 256 + 4 * 24 * 1024, st>>>(
          C.mv_batches.get(), C.mv_segs.get(), C.mv_nsegs, C.mv_cta.get(), (const char*)C.dstore.get(), (const char*)pool,
          (const char*)C.mv_tasks.get(), x_int, y_int, scramble, prof, f32 ? 1 : 0);
    else if (C.mv_kind == 5)
      k_mv_batched<3, 32 * 1024, 256, 2><<<C.mv_grid, 256, 256 + 3 * 32 * 1024, st>>>(
          C.mv_batches.get(), C.mv_segs.get(), C.mv_nsegs, C.mv_cta.get(), (const char*)C.dstore.get(), (const char*)pool,
          (const char*)C.mv_tasks.get(), x_int, y_int, scramble, prof, f32 ? 1 : 0);
    else                     // one CTA ring per SM, 4 x 48 KiB stages, 15 consumer warps
      k_mv_batched<4, kMvStageBytes, 512, 1><<<C.mv_grid, 512, 256 + 4 * kMvStageBytes, st>>>(
          C.mv_batches.get(), C.mv_segs.get(), C.mv_nsegs, C.mv_cta.get(), (const char*)C.dstore.get(), (const char*)pool,
          (const char*)C.mv_tasks.get(), x_int, y_int, scramble, prof, f32 ? 1 : 0);
    HM_CHECK_LAUNCH();
  }
  if (C.mv_n_dense_big) {
    k_mv_dense_direct<<<148 * 8, 256, 0, st>>>(C.mv_dense_big.get(), C.mv_n_dense_big, C.dstore.get(),
                                               x_int, y_int);
    HM_CHECK_LAUNCH();
  }
  if (conc) {
    HM_CUDA(cudaStreamWaitEvent(st, C.mv_ev[1], 0));
  } else if (C.mv_n_tiles_v) {
    large_v(st);
    large_u(st);
  }
  ks.reset();
  if (C.world > 1 && reduce) allreduce_sum(C, y_int, C.N);
}

}  // namespace hm
