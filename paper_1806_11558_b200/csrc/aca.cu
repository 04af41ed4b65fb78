// aca.cu — batched adaptive cross approximation of the rank's admissible leaves
// (batching P:413-430), partial pivoting with the Frobenius stop (A11-A12).
//
// Design: all blocks of a chunk advance in lock-step, one ACA step per
// round of five kernels —
//   row   : one thread per residual-row entry  r_j = a(i,j) - sum_l U[i,l] V[j,l]
//   pivot : one warp per block, argmax |r_j| (lowest j on ties), v = r / r_j*
//   col   : one thread per residual-column entry u_t = a(t,j*) - sum_l U[t,l] V[j*,l]
//   update: one warp per block, ||S_k||_F^2 update, stop test, next row = argmax unused |u_t|
// Residual updates are sequential in l with separately rounded products and differences,
// so r, u and therefore every pivot are bit-identical to the reading; only the norms
// (which feed the stop test alone) are tree-reduced.  Workspace per block holds KWS
// columns; blocks that reach KWS without stopping are re-run with k_max columns.
// Finished blocks are packed into the factor pool as [U (m x k) | V (n x k)], col-major.

#include <algorithm>
#include <chrono>
#include <thread>
#include <type_traits>

#include "entry_batch.cuh"
#include "primitives.cuh"

namespace hm {

struct AcaBlk {
  Quad q;
  int32_t m, n, kmax, pad;
  int64_t uoff, voff, boff;
};

struct AcaState {
  int32_t i, k, js, status;   // status: 0 active, 1 done, 2 workspace overflow
  int32_t skip, pad0;
  double S2, vv;
};

struct AcaWork {
  DBuf<AcaBlk> blk;
  DBuf<AcaState> state;
  DBuf<int32_t> owned, piv, act, flag, pos, big, rtab, ctab;
  DBuf<int64_t> rsz, csz, rpre, cpre;
  DBuf<double> ws;      // chunk workspace: [U: m*kws per block | V: n*kws per block]
  DBuf<uint32_t> bmap;
  DBuf<char> tmp;
  DBuf<unsigned long long> ev, cnt;
  DBuf<int64_t> tot;
  DBuf<int32_t> ovf;
  DBuf<unsigned long long> novf;
  DBuf<int32_t> bad;    // smallest owned block index with a non-finite factor entry (INT_MAX: none)
  PinnedVec<int64_t> h_tot;
  PinnedVec<AcaBlk> h_blk;
  PinnedVec<int32_t> h_idsp;
  std::vector<AcaState> h_state;
  std::vector<int32_t> h_ids, h_big;
  DBuf<EntryRef> lists;
  PinnedVec<int64_t> h_ring;          // per-step totals read back kLag steps late
  cudaEvent_t ring_ev[3] = {nullptr, nullptr, nullptr};
  ~AcaWork() { for (auto& e : ring_ev) if (e) cudaEventDestroy(e); }
};

namespace {

// Active-block compaction for one ACA step: flag[c] = block c still running; after the scan
// pos, act[pos[c]] = c and the row / column lengths of the active blocks are packed in front
// (the rest of rsz / csz stays 0), so the entry batches, pivot and update kernels only see
// the active blocks.
__global__ void k_step_flags(const AcaState* __restrict__ S, int64_t nb, int32_t* __restrict__ flag) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > nb) return;
  flag[c] = c < nb && S[c].status == 0;
}

__global__ void k_step_compact(const AcaBlk* __restrict__ B, const int32_t* __restrict__ flag,
                               const int32_t* __restrict__ pos, int64_t nb, int32_t* __restrict__ act,
                               int64_t* __restrict__ rsz, int64_t* __restrict__ csz) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > nb) return;
  if (c >= pos[nb]) { rsz[c] = 0; csz[c] = 0; }   // slots past the active count (disjoint from the writes below)
  if (c == nb || !flag[c]) return;
  const int32_t a = pos[c];
  act[a] = (int32_t)c;
  rsz[a] = B[c].n;
  csz[a] = B[c].m;
}

__global__ void k_store_totals(const int64_t* __restrict__ add, const unsigned long long* __restrict__ novf,
                               int64_t* __restrict__ tot) {
  tot[0] = *add;
  tot[1] = (int64_t)*novf;
}

__global__ void k_step_totals(const int64_t* __restrict__ rpre, const int64_t* __restrict__ cpre,
                              const int32_t* __restrict__ pos, int64_t nb, int64_t* __restrict__ tot) {
  tot[0] = rpre[nb];
  tot[1] = cpre[nb];
  tot[2] = pos[nb];
}

// Residual row (ROW) or column entries of the active blocks of a chunk, as a batch mapping
// for entry_batch.cuh.  put() applies the rank-one corrections of the previous k steps in
// ascending l, each product and difference separately rounded (A15), and stores the residual
// into column k of the block's V (row step) or U (column step) workspace.
template <bool ROW, bool QUAD = false, bool PERF = false>
struct AcaMap {
  static constexpr bool kQuad = QUAD;
  static constexpr bool kPerf = PERF;   // option aca_perf: order-3/4 entries in perf mode (A15 deviation, measured)
  const Panel* P;       // triangle panels, or node panels of a quadrilateral mesh (A25)
  const Panel* PT;      // quads: the split triangles
  const int4* QV;       // quads: vertex ids
  const AcaBlk* B;
  const AcaState* S;
  const int64_t* pre;   // nb + 1 prefix of this step's row (or column) lengths, active blocks first
  const int32_t* act;   // compact index -> block
  const int32_t* tab;   // tab[e / 32] = compact segment of entry 32 * (e / 32)
  int64_t nb;
  double* Uw;
  double* Vw;
  __device__ bool locate(int64_t e, bool valid, EntryRef& r) const {
    if (!valid) return false;
    int64_t a = tab[e >> 5];
    while (pre[a + 1] <= e) ++a;
    const int32_t c = act[a];
    if (!ROW && (S[c].skip || S[c].status != 0)) return false;
    r.seg = c;
    r.idx = (int32_t)(e - pre[a]);
    return true;
  }
  __device__ void pair(EntryRef r, int& s, int& t) const {
    const AcaBlk& b = B[r.seg];
    const AcaState& st = S[r.seg];
    s = ROW ? b.q.rlo + st.i : b.q.rlo + r.idx;
    t = ROW ? b.q.clo + r.idx : b.q.clo + st.js;
  }
  __device__ void put(EntryRef r, double a) const {
    const AcaBlk& b = B[r.seg];
    const AcaState st = S[r.seg];
    const double* U = Uw + b.uoff;
    const double* V = Vw + b.voff;
    if (ROW) {
      for (int l = 0; l < st.k; ++l) a = dsub(a, dmul(U[st.i + (int64_t)l * b.m], V[r.idx + (int64_t)l * b.n]));
      Vw[b.voff + (int64_t)st.k * b.n + r.idx] = a;
    } else {
      for (int l = 0; l < st.k; ++l) a = dsub(a, dmul(U[r.idx + (int64_t)l * b.m], V[st.js + (int64_t)l * b.n]));
      Uw[b.uoff + (int64_t)st.k * b.m + r.idx] = a;
    }
  }
};

__device__ __forceinline__ void warp_argmax(double& v, int& idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ bool is_used(const uint32_t* bm, int t) { return (bm[t >> 5] >> (t & 31)) & 1u; }

// smallest unused row, or -1
__device__ int first_unused(const uint32_t* bm, int m, int lane) {
  int words = (m + 31) >> 5;
  int best = INT_MAX;
  for (int w = lane; w < words; w += 32) {
    uint32_t free_bits = ~bm[w];
    if (w == words - 1 && (m & 31)) free_bits &= (1u << (m & 31)) - 1u;
    if (free_bits) { best = min(best, w * 32 + __ffs(free_bits) - 1); }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  return best == INT_MAX ? -1 : best;
}

// blocks with m + n >= kBigMN get a CTA (not a warp) in the pivot and update kernels
constexpr int kBigMN = 2048;

__device__ __forceinline__ void aca_pivot_block(const AcaBlk* __restrict__ B, AcaState* __restrict__ S, int64_t c,
                                                double* __restrict__ Vw, uint32_t* __restrict__ bmap, int lane) {
  AcaState st = S[c];
  if (st.status != 0) return;
  const AcaBlk b = B[c];
  if (b.m + b.n >= kBigMN) return;                      // k_aca_pivot_big
  double* r = Vw + b.voff + (int64_t)st.k * b.n;
  uint32_t* bm = bmap + b.boff;
  double best = -1.0;
  int bj = INT_MAX;
  for (int j = lane; j < b.n; j += 32) {
    double a = fabs(r[j]);
    if (a > best) { best = a; bj = j; }
  }
  warp_argmax(best, bj);
  __syncwarp();
  if (lane == 0) bm[st.i >> 5] |= 1u << (st.i & 31);   // row i is used (A12)
  __syncwarp();
  const double piv = r[bj];
  if (piv == 0.0) {                                     // zero residual row: next unused row
    int nx = first_unused(bm, b.m, lane);
    if (lane == 0) {
      if (nx < 0) st.status = 1;
      else { st.i = nx; st.skip = 1; }
      S[c] = st;
    }
    return;
  }
  double vv = 0.0;
  for (int j = lane; j < b.n; j += 32) {
    double v = ddiv(r[j], piv);
    r[j] = v;
    vv += v * v;
  }
  vv = warp_sum(vv);
  if (lane == 0) {
    st.js = bj;
    st.vv = vv;
    st.skip = 0;
    S[c] = st;
  }
}


// one warp per active block; the step's active count *dnact is read on the device, the grid
// covers an upper bound of it known to the host (the count read back kLag steps earlier: the
// active set only shrinks)
__global__ void k_aca_pivot(const AcaBlk* __restrict__ B, AcaState* __restrict__ S, const int32_t* __restrict__ act,
                            const int64_t* __restrict__ dnact, double* __restrict__ Vw, uint32_t* __restrict__ bmap) {
  const int64_t a = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (a >= *dnact) return;
  aca_pivot_block(B, S, act[a], Vw, bmap, threadIdx.x & 31);
}

// k_aca_pivot for the big blocks of the chunk (m + n >= kBigMN): one CTA per block
__global__ void __launch_bounds__(256) k_aca_pivot_big(const AcaBlk* __restrict__ B, AcaState* __restrict__ S,
                                                       const int32_t* __restrict__ big, double* __restrict__ Vw,
                                                       uint32_t* __restrict__ bmap) {
  __shared__ double sbest[8];
  __shared__ int sidx[8];
  const int64_t c = big[blockIdx.x];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  AcaState st = S[c];
  if (st.status != 0) return;
  const AcaBlk b = B[c];
  double* r = Vw + b.voff + (int64_t)st.k * b.n;
  uint32_t* bm = bmap + b.boff;
  double best = -1.0;
  int bj = INT_MAX;
  for (int j = threadIdx.x; j < b.n; j += 256) {
    const double a = fabs(r[j]);
    if (a > best) { best = a; bj = j; }
  }
  warp_argmax(best, bj);
  if (lane == 0) { sbest[w] = best; sidx[w] = bj; }
  __syncthreads();
  best = sbest[0]; bj = sidx[0];
  for (int g = 1; g < 8; ++g)
    if (sbest[g] > best || (sbest[g] == best && sidx[g] < bj)) { best = sbest[g]; bj = sidx[g]; }
  if (threadIdx.x == 0) bm[st.i >> 5] |= 1u << (st.i & 31);   // row i is used (A12)
  __syncthreads();
  const double piv = r[bj];
  if (piv == 0.0) {                                            // zero residual row: next unused row
    if (w == 0) {
      const int nx = first_unused(bm, b.m, lane);
      if (lane == 0) {
        if (nx < 0) st.status = 1;
        else { st.i = nx; st.skip = 1; }
        S[c] = st;
      }
    }
    return;
  }
  double vv = 0.0;
  for (int j = threadIdx.x; j < b.n; j += 256) {
    const double v = ddiv(r[j], piv);
    r[j] = v;
    vv += v * v;
  }
  vv = warp_sum(vv);
  __syncthreads();
  if (lane == 0) sbest[w] = vv;
  __syncthreads();
  if (threadIdx.x == 0) {
    vv = 0.0;
    for (int g = 0; g < 8; ++g) vv += sbest[g];
    st.js = bj;
    st.vv = vv;
    st.skip = 0;
    S[c] = st;
  }
}

// Sum 16 per-lane values over the warp by recursive halving (16 shuffles instead of 16 x 5):
// on return a[0] of lane L holds the warp total of value index
// 8*bit4(L) + 4*bit3(L) + 2*bit2(L) + bit1(L)  (two lanes per index).
__device__ __forceinline__ void warp_reduce16(double (&a)[16], int lane) {
#pragma unroll
  for (int lvl = 0; lvl < 4; ++lvl) {
    const int o = 16 >> lvl, half = 8 >> lvl;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < half) {
        const double send = up ? a[i] : a[i + half];
        const double keep = up ? a[i + half] : a[i];
        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
  }
  a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
}
__device__ __forceinline__ int reduce16_index(int lane) {
  return ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
}

// Frobenius update of step k (A11): S2 += 2 sum_l (u^T U_l)(V_l^T v) + |u|^2 |v|^2, the stop
// test, and the next row pivot.  A group of G warps works on one block (G = 1 for most
// blocks, G = 8 for blocks with m + n >= kBigMN); the cross products are formed 8 columns per
// pass with the 8 (u^T U_l) and 8 (V_l^T v) partial sums in registers (u_t / v_j loaded once
// per pass, 8 independent loads in flight) and reduced together by one recursive-halving
// butterfly.  Norms feed the stop test only (A15: tree-reduced on the GPU).

template <int G>
__device__ __forceinline__ void aca_update_block(const AcaBlk& b, AcaState& st, const double* __restrict__ Uw,
                                                 const double* __restrict__ Vw, const uint32_t* __restrict__ bmap,
                                                 int32_t* __restrict__ piv, int64_t c, int kws, double eps, int gw,
                                                 int lane, double* red /* smem [G][17] (G > 1) */) {
  const double* U = Uw + b.uoff;
  const double* V = Vw + b.voff;
  const double* u = U + (int64_t)st.k * b.m;
  const double* v = V + (int64_t)st.k * b.n;
  const int t0 = gw * 32 + lane, stride = G * 32;
  double uu = 0.0;   // ||u_k||^2, accumulated in the first pass over u (one pass also when k = 0)
  double cross = 0.0;
  for (int l0 = 0; l0 < max(st.k, 1); l0 += 8) {
    const int kc = min(8, st.k - l0);
    double acc[16];
#pragma unroll
    for (int l = 0; l < 16; ++l) acc[l] = 0.0;
    for (int t = t0; t < b.m; t += stride) {
      const double ut = u[t];
      if (l0 == 0) uu = fma(ut, ut, uu);
#pragma unroll
      for (int l = 0; l < 8; ++l)
        if (l < kc) acc[l] = fma(ut, U[t + (int64_t)(l0 + l) * b.m], acc[l]);
    }
    if (kc <= 0) break;
    for (int j = t0; j < b.n; j += stride) {
      const double vj = v[j];
#pragma unroll
      for (int l = 0; l < 8; ++l)
        if (l < kc) acc[8 + l] = fma(V[j + (int64_t)(l0 + l) * b.n], vj, acc[8 + l]);
    }
    warp_reduce16(acc, lane);   // lane L: total of index reduce16_index(L); du_l at bit4 = 0, dv_l at L ^ 16
    if (G > 1) {
      if ((lane & 1) == 0) red[gw * 17 + reduce16_index(lane)] = acc[0];
      __syncthreads();
      double tsum = 0.0;
      if (lane < 16)
        for (int g = 0; g < G; ++g) tsum += red[g * 17 + lane];
      const double other = __shfl_down_sync(0xffffffffu, tsum, 8);
      const double part = (lane < 8 && lane < kc) ? tsum * other : 0.0;
      cross += warp_sum(part);
      __syncthreads();
    } else {
      const double other = __shfl_xor_sync(0xffffffffu, acc[0], 16);
      const int idx = reduce16_index(lane);
      const double part = ((lane & 17) == 0 && idx < kc) ? acc[0] * other : 0.0;
      cross += warp_sum(part);
    }
  }
  uu = warp_sum(uu);
  if (G > 1) {
    if (lane == 0) red[gw * 17 + 16] = uu;
    __syncthreads();
    uu = 0.0;
    for (int g = 0; g < G; ++g) uu += red[g * 17 + 16];
    __syncthreads();
  }
  st.S2 = (st.S2 + 2.0 * cross) + uu * st.vv;
  if (gw == 0 && lane == 0) {
    piv[c * 2 * kws + 2 * st.k] = st.i;
    piv[c * 2 * kws + 2 * st.k + 1] = st.js;
  }
  st.k += 1;
  if (sqrt(uu) * sqrt(st.vv) <= eps * sqrt(st.S2)) st.status = 1;    // stop test (A11)
  else if (st.k >= b.kmax) st.status = 1;                              // rank budget
  else if (st.k >= kws) st.status = 2;                                 // workspace full: re-run
  if (st.status == 0) {                                                // next row pivot (A12)
    const uint32_t* bm = bmap + b.boff;
    double best = -1.0;
    int bt = INT_MAX;
    for (int t = t0; t < b.m; t += stride) {
      if (is_used(bm, t)) continue;
      const double a = fabs(u[t]);
      if (a > best) { best = a; bt = t; }
    }
    warp_argmax(best, bt);
    if (G > 1) {
      int* ri = reinterpret_cast<int*>(red + G * 17);
      if (lane == 0) { red[gw * 17] = best; ri[gw] = bt; }
      __syncthreads();
      best = red[0]; bt = ri[0];
      for (int g = 1; g < G; ++g) {
        const double ob = red[g * 17];
        const int oi = ri[g];
        if (ob > best || (ob == best && oi < bt)) { best = ob; bt = oi; }
      }
    }
    if (bt == INT_MAX) st.status = 1;
    else st.i = bt;
  }
}

// G = 1: one warp per active block (small blocks; big ones are skipped), act[] = compact list;
// the active count *dnact is read on the device (grid: a host-side upper bound, see k_aca_pivot)
template <int MINB>
__global__ void __launch_bounds__(64, MINB) k_aca_update(const AcaBlk* __restrict__ B, AcaState* __restrict__ S,
                                                    const int32_t* __restrict__ act, const int64_t* __restrict__ dnact,
                                                    const double* __restrict__ Uw, const double* __restrict__ Vw,
                                                    const uint32_t* __restrict__ bmap, int32_t* __restrict__ piv,
                                                    int kws, double eps) {
  const int64_t a = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (a >= *dnact) return;
  const int64_t c = act[a];
  AcaState st = S[c];
  const AcaBlk b = B[c];
  if (st.status != 0 || st.skip) return;
  if (b.m + b.n >= kBigMN) return;
  aca_update_block<1>(b, st, Uw, Vw, bmap, piv, c, kws, eps, 0, lane, nullptr);
  if (lane == 0) S[c] = st;
}

// G = 8: one CTA per big block of the chunk (list fixed per chunk; finished blocks return)
__global__ void __launch_bounds__(256, 4) k_aca_update_big(const AcaBlk* __restrict__ B, AcaState* __restrict__ S,
                                                        const int32_t* __restrict__ big, const double* __restrict__ Uw,
                                                        const double* __restrict__ Vw, const uint32_t* __restrict__ bmap,
                                                        int32_t* __restrict__ piv, int kws, double eps) {
  __shared__ double red[8 * 17 + 8];
  const int64_t c = big[blockIdx.x];
  AcaState st = S[c];
  if (st.status != 0 || st.skip) return;
  const AcaBlk b = B[c];
  aca_update_block<8>(b, st, Uw, Vw, bmap, piv, c, kws, eps, threadIdx.x >> 5, threadIdx.x & 31, red);
  if (threadIdx.x == 0) S[c] = st;
}

__global__ void k_init_state(AcaState* __restrict__ S, int64_t nb) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nb) return;
  AcaState s;
  s.i = 0; s.k = 0; s.js = 0; s.status = 0; s.skip = 0; s.pad0 = 0; s.S2 = 0.0; s.vv = 0.0;
  S[c] = s;
}

// factor-pool size of every finished block; blocks that filled the workspace (status 2) are
// appended to the overflow list (re-run with k_max columns)
__global__ void k_final_sizes(const AcaBlk* __restrict__ B, const AcaState* __restrict__ S, int64_t nb,
                              int64_t* __restrict__ fsz, const int32_t* __restrict__ owned,
                              int32_t* __restrict__ ovf, unsigned long long* __restrict__ novf) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > nb) return;
  if (c == nb) { fsz[c] = 0; return; }
  const AcaState st = S[c];
  fsz[c] = st.status == 1 ? (int64_t)st.k * (B[c].m + B[c].n) : 0;
  if (st.status == 2) ovf[atomicAdd(novf, 1ull)] = owned[c];
}
// pack finished blocks: [U (m x k) | V (n x k)] column-major, straight copies of the
// first k workspace columns (T = float: option lr_f32, each entry rounded to binary32 once).
// The copy also checks every factor entry for finiteness (hm.h: HM_ERR_NUMERIC names the first
// offending block): bad = min owned index.  G threads per block: a warp per small block
// (k_aca_store<.., 32>, 8 blocks per CTA), a CTA per big block (m + n >= kBigMN, list `big`).
template <class T, int G>
__device__ __forceinline__ void aca_store_block(const AcaBlk& b, const AcaState& st, int64_t c,
                                                const int32_t* __restrict__ owned, const int64_t* __restrict__ fpre,
                                                int64_t base, const double* __restrict__ Uw,
                                                const double* __restrict__ Vw, T* __restrict__ pool,
                                                int64_t* __restrict__ foff, int32_t* __restrict__ frank,
                                                int32_t* __restrict__ bad, int tid) {
  const int64_t o = base + fpre[c];
  const int64_t mu = (int64_t)st.k * b.m, nv = (int64_t)st.k * b.n;
  bool fin = true;
  for (int64_t x = tid; x < mu; x += G) { const T a = (T)Uw[b.uoff + x]; fin &= isfinite(a); pool[o + x] = a; }
  for (int64_t x = tid; x < nv; x += G) { const T a = (T)Vw[b.voff + x]; fin &= isfinite(a); pool[o + mu + x] = a; }
  if (!fin) atomicMin(bad, owned[c]);
  if (tid == 0) {
    foff[owned[c]] = o;
    frank[owned[c]] = st.k;
  }
}

template <class T>
__global__ void __launch_bounds__(256) k_aca_store(const AcaBlk* __restrict__ B, const AcaState* __restrict__ S,
                                                   int64_t nb, const int32_t* __restrict__ owned,
                                                   const int64_t* __restrict__ fpre, int64_t base,
                                                   const double* __restrict__ Uw, const double* __restrict__ Vw,
                                                   T* __restrict__ pool, int64_t* __restrict__ foff,
                                                   int32_t* __restrict__ frank, int32_t* __restrict__ bad) {
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (c >= nb) return;
  const AcaState st = S[c];
  const AcaBlk b = B[c];
  if (st.status != 1 || b.m + b.n >= kBigMN) return;
  aca_store_block<T, 32>(b, st, c, owned, fpre, base, Uw, Vw, pool, foff, frank, bad, threadIdx.x & 31);
}

template <class T>
__global__ void __launch_bounds__(256) k_aca_store_big(const AcaBlk* __restrict__ B, const AcaState* __restrict__ S,
                                                       const int32_t* __restrict__ big, const int32_t* __restrict__ owned,
                                                       const int64_t* __restrict__ fpre, int64_t base,
                                                       const double* __restrict__ Uw, const double* __restrict__ Vw,
                                                       T* __restrict__ pool, int64_t* __restrict__ foff,
                                                       int32_t* __restrict__ frank, int32_t* __restrict__ bad) {
  const int64_t c = big[blockIdx.x];
  const AcaState st = S[c];
  if (st.status != 1) return;
  aca_store_block<T, 256>(B[c], st, c, owned, fpre, base, Uw, Vw, pool, foff, frank, bad, threadIdx.x);
}

// one batch of residual entries (row or column step): order-3 in place, then the order-4
// list, then the rest; the batch size *dtot lives on the device, `upper` bounds it (grid size)
template <class M>
void aca_eval(Context& C, const M& m, const int64_t* dtot, int64_t upper, AcaWork& W) {
  if (upper <= 0) return;
  cudaStream_t st = C.stream;
  HM_CUDA(cudaMemsetAsync(W.cnt.get(), 0, 3 * sizeof(unsigned long long), st));
  KScope ks(C, KF_EVAL_ACA);
  const unsigned g = (unsigned)std::min<int64_t>(grid_for(upper, 128), 148 * 4);   // one wave, persistent
  k_eval_class3<M><<<g, 128, 0, st>>>(m, dtot, W.lists.get(), W.cnt.get(), W.ev.get());
  HM_CHECK_LAUNCH();
  const unsigned g4 = (unsigned)std::min<int64_t>(grid_for(upper, 128), 148 * 16);
  k_eval_list<4, M><<<g4, 128, 0, st>>>(m, W.lists.get(), W.cnt.get(), W.ev.get());
  HM_CHECK_LAUNCH();
  k_eval_rest<M><<<std::min<unsigned>(g4, 148 * 4), 128, 0, st>>>(m, W.lists.get(), dtot, W.cnt.get(), W.ev.get());
  HM_CHECK_LAUNCH();
}

// Run ACA on the owned admissible leaves listed in `ids` (indices into the owned list) with
// `kws` workspace columns; appends blocks that overflowed to `overflow`.
void run_chunk(Context& C, AcaWork& W, const std::vector<int32_t>& ids, int kws, std::vector<int32_t>& overflow,
               std::vector<std::vector<int32_t>>* pivots_out) {
  cudaStream_t st = C.stream;
  using clk = std::chrono::steady_clock;
  auto ms_since = [](clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); };
  const auto t0 = clk::now();
  const int64_t nb = (int64_t)ids.size();
  PinnedVec<AcaBlk>& hb = W.h_blk;
  hb.resize(nb);
  std::vector<int32_t>& hbig = W.h_big;
  hbig.clear();
  int64_t uo = 0, vo = 0, bo = 0, rmax = 0, cmax = 0;   // rmax / cmax: entries of the first row / column step
  {
    // block records and workspace offsets on host threads over contiguous slices (two passes:
    // per-slice sizes, then the slices' offsets), the big-block list in slice order
    const int64_t hw = std::max<int64_t>(1, (int64_t)std::thread::hardware_concurrency() / std::max(1, C.world));
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>({hw, 8, nb / 50000 + 1}));
    struct Part { int64_t u = 0, v = 0, b = 0, r = 0, c = 0; std::vector<int32_t> big; };
    std::vector<Part> part(T);
    auto slice = [&](int t, bool fill, const Part& off) {
      const int64_t c0 = nb * t / T, c1 = nb * (t + 1) / T;
      Part acc = off;
      for (int64_t c = c0; c < c1; ++c) {
        const Quad& q = C.h_adm[C.adm_begin + ids[c]];
        const int32_t m = q.rhi - q.rlo, n = q.chi - q.clo;
        if (fill) {
          AcaBlk& b = hb[c];
          b.q = q;
          b.m = m;
          b.n = n;
          b.kmax = std::min(std::min(m, n), C.k_max);
          b.pad = 0;
          b.uoff = acc.u; b.voff = acc.v; b.boff = acc.b;
        } else if (m + n >= kBigMN) {
          part[t].big.push_back((int32_t)c);
        }
        acc.u += (int64_t)m * kws;
        acc.v += (int64_t)n * kws;
        acc.b += (m + 31) / 32;
        acc.r += n;
        acc.c += m;
      }
      if (!fill) { part[t].u = acc.u; part[t].v = acc.v; part[t].b = acc.b; part[t].r = acc.r; part[t].c = acc.c; }
    };
    auto run = [&](auto&& f) {
      std::vector<std::thread> th;
      for (int t = 1; t < T; ++t) th.emplace_back([&, t]() { f(t); });
      f(0);
      for (auto& x : th) x.join();
    };
    run([&](int t) { part[t].big.clear(); slice(t, false, Part{}); });
    std::vector<Part> off(T);
    for (int t = 0; t < T; ++t) {
      off[t].u = uo; off[t].v = vo; off[t].b = bo;
      uo += part[t].u; vo += part[t].v; bo += part[t].b; rmax += part[t].r; cmax += part[t].c;
      hbig.insert(hbig.end(), part[t].big.begin(), part[t].big.end());
    }
    run([&](int t) { slice(t, true, off[t]); });
  }
  const int64_t nbig = (int64_t)hbig.size();
  W.blk.alloc(nb); W.state.alloc(nb); W.owned.alloc(nb); W.piv.alloc(nb * 2 * kws);
  W.act.alloc(nb + 1); W.flag.alloc(nb + 1); W.pos.alloc(nb + 1); W.tot.alloc(3); W.big.alloc(nbig);
  W.ovf.alloc(nb); W.novf.alloc(1); W.h_tot.resize(4);
  if (nbig) HM_CUDA(cudaMemcpyAsync(W.big.get(), hbig.data(), nbig * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  W.rsz.alloc(nb + 1); W.csz.alloc(nb + 1); W.rpre.alloc(nb + 1); W.cpre.alloc(nb + 1);
  W.ws.alloc(uo + vo); W.bmap.alloc(bo);
  double* const Uw = W.ws.get();          // one workspace buffer: U columns, then V columns
  double* const Vw = Uw + uo;
  HM_CUDA(cudaMemcpyAsync(W.blk.get(), hb.data(), nb * sizeof(AcaBlk), cudaMemcpyHostToDevice, st));
  W.h_idsp.resize(nb);
  std::memcpy(W.h_idsp.data(), ids.data(), nb * sizeof(int32_t));
  HM_CUDA(cudaMemcpyAsync(W.owned.get(), W.h_idsp.data(), nb * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  HM_CUDA(cudaMemsetAsync(W.bmap.get(), 0, bo * sizeof(uint32_t), st));
  k_init_state<<<grid_for(nb, 256), 256, 0, st>>>(W.state.get(), nb);
  HM_CHECK_LAUNCH();
  const Panel* P = C.panel.get();
  const Panel* Pn = C.qnode.get();
  const int4* QV = C.qv.get();
  C.times.aca_phase_ms[0] += ms_since(t0);
  const auto t1 = clk::now();
  // Host-sync-free step loop: every kernel of a step reads the step's sizes (active blocks,
  // row / column entry totals) from device memory, so the host enqueues step after step and
  // only reads each step's totals back kLag steps later (pinned ring + events) to learn when
  // the chunk is done; the at most kLag steps enqueued past the last active one find no active
  // block and return at once.
  constexpr int kLag = 2;
  W.lists.alloc(std::max(rmax, cmax));
  W.rtab.alloc(rmax / 32 + 2);
  W.ctab.alloc(cmax / 32 + 2);
  W.cnt.alloc(3);                 // [n4, nrest, next entry group]
  W.h_ring.resize(3 * (kLag + 1));
  for (auto& e : W.ring_ev)
    if (!e) HM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const int64_t* drow = W.tot.get();          // tot[0]: row entries, tot[1]: column entries, tot[2]: active blocks
  const int64_t* dcol = W.tot.get() + 1;
  const int64_t* dnact = W.tot.get() + 2;
  int64_t nact_ub = nb;              // upper bound of the active count of every step still to be enqueued
  for (int step = 0;; ++step) {
    std::unique_ptr<KScope> ks(new KScope(C, KF_ACA_OTHER));
    k_step_flags<<<grid_for(nb + 1, 256), 256, 0, st>>>(W.state.get(), nb, W.flag.get());
    HM_CHECK_LAUNCH();
    prim::exclusive_scan<int32_t>(W.flag.get(), W.pos.get(), nb + 1, W.tmp, st);
    k_step_compact<<<grid_for(nb + 1, 256), 256, 0, st>>>(W.blk.get(), W.flag.get(), W.pos.get(), nb, W.act.get(),
                                                          W.rsz.get(), W.csz.get());
    HM_CHECK_LAUNCH();
    prim::exclusive_scan<int64_t>(W.rsz.get(), W.rpre.get(), nb + 1, W.tmp, st);
    prim::exclusive_scan<int64_t>(W.csz.get(), W.cpre.get(), nb + 1, W.tmp, st);
    k_step_totals<<<1, 1, 0, st>>>(W.rpre.get(), W.cpre.get(), W.pos.get(), nb, W.tot.get());
    HM_CHECK_LAUNCH();
    const int slot = step % (kLag + 1);
    HM_CUDA(cudaMemcpyAsync(W.h_ring.data() + 3 * slot, W.tot.get(), 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HM_CUDA(cudaEventRecord(W.ring_ev[slot], st));
    // segment tables over all nb slots: slots past the active count have empty ranges
    k_seg_table<<<grid_for(nb, 256), 256, 0, st>>>(W.rpre.get(), nb, 0, W.rtab.get());
    HM_CHECK_LAUNCH();
    k_seg_table<<<grid_for(nb, 256), 256, 0, st>>>(W.cpre.get(), nb, 0, W.ctab.get());
    HM_CHECK_LAUNCH();
    ks.reset();
    if (C.quad)
      aca_eval(C, AcaMap<true, true>{Pn, P, QV, W.blk.get(), W.state.get(), W.rpre.get(), W.act.get(), W.rtab.get(),
                                     nb, Uw, Vw}, drow, rmax, W);
    else if (C.aca_perf)
      aca_eval(C, AcaMap<true, false, true>{P, nullptr, nullptr, W.blk.get(), W.state.get(), W.rpre.get(), W.act.get(),
                                            W.rtab.get(), nb, Uw, Vw}, drow, rmax, W);
    else
      aca_eval(C, AcaMap<true>{P, nullptr, nullptr, W.blk.get(), W.state.get(), W.rpre.get(), W.act.get(),
                               W.rtab.get(), nb, Uw, Vw}, drow, rmax, W);
    ks.reset(new KScope(C, KF_ACA_OTHER));
    k_aca_pivot<<<grid_for(nact_ub * 32, 256), 256, 0, st>>>(W.blk.get(), W.state.get(), W.act.get(), dnact, Vw,
                                                             W.bmap.get());
    HM_CHECK_LAUNCH();
    if (nbig) {
      k_aca_pivot_big<<<(unsigned)nbig, 256, 0, st>>>(W.blk.get(), W.state.get(), W.big.get(), Vw, W.bmap.get());
      HM_CHECK_LAUNCH();
    }
    ks.reset();
    if (C.quad)
      aca_eval(C, AcaMap<false, true>{Pn, P, QV, W.blk.get(), W.state.get(), W.cpre.get(), W.act.get(), W.ctab.get(),
                                      nb, Uw, Vw}, dcol, cmax, W);
    else if (C.aca_perf)
      aca_eval(C, AcaMap<false, false, true>{P, nullptr, nullptr, W.blk.get(), W.state.get(), W.cpre.get(),
                                             W.act.get(), W.ctab.get(), nb, Uw, Vw}, dcol, cmax, W);
    else
      aca_eval(C, AcaMap<false>{P, nullptr, nullptr, W.blk.get(), W.state.get(), W.cpre.get(), W.act.get(),
                                W.ctab.get(), nb, Uw, Vw}, dcol, cmax, W);
    ks.reset(new KScope(C, KF_ACA_OTHER));
    auto upd = C.aca_upd_occ == 2 ? k_aca_update<32> : C.aca_upd_occ == 1 ? k_aca_update<24> : k_aca_update<16>;
    upd<<<grid_for(nact_ub * 32, 64), 64, 0, st>>>(W.blk.get(), W.state.get(), W.act.get(), dnact, Uw, Vw,
                                                            W.bmap.get(), W.piv.get(), kws, C.eps_aca);
    HM_CHECK_LAUNCH();
    if (nbig) {
      k_aca_update_big<<<(unsigned)nbig, 256, 0, st>>>(W.blk.get(), W.state.get(), W.big.get(), Uw, Vw,
                                                       W.bmap.get(), W.piv.get(), kws, C.eps_aca);
      HM_CHECK_LAUNCH();
    }
    ks.reset();
    // read back the totals of step - kLag (all earlier ones were read already)
    if (step >= kLag) {
      const int rs = (step - kLag) % (kLag + 1);
      const auto ts = clk::now();
      HM_CUDA(cudaEventSynchronize(W.ring_ev[rs]));
      C.times.aca_phase_ms[2] += ms_since(ts);
      const int64_t* t = W.h_ring.data() + 3 * rs;
      if (t[0] == 0) break;        // no active block since step - kLag: the later steps were no-ops
      nact_ub = t[2];
      C.aca_steps++;
      C.entries_aca += (double)(t[0] + t[1]);
    }
  }
  C.times.aca_phase_ms[1] += ms_since(t1);
  const auto t2 = clk::now();
  // pack finished blocks into the factor pool
  HM_CUDA(cudaMemsetAsync(W.novf.get(), 0, sizeof(unsigned long long), st));
  k_final_sizes<<<grid_for(nb + 1, 256), 256, 0, st>>>(W.blk.get(), W.state.get(), nb, W.rsz.get(), W.owned.get(),
                                                       W.ovf.get(), W.novf.get());
  HM_CHECK_LAUNCH();
  prim::exclusive_scan<int64_t>(W.rsz.get(), W.rpre.get(), nb + 1, W.tmp, st);
  k_store_totals<<<1, 1, 0, st>>>(W.rpre.get() + nb, W.novf.get(), W.tot.get());
  HM_CHECK_LAUNCH();
  int64_t* ht = W.h_tot.data();
  HM_CUDA(cudaMemcpyAsync(ht, W.tot.get(), 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HM_CUDA(cudaStreamSynchronize(st));
  const int64_t add = ht[0], nov = ht[1];
  // factor pool in elements of C.lr_esz bytes (8, or 4 with option lr_f32)
  const int64_t esz = C.lr_esz;
  const int64_t base = (int64_t)(C.fpool.used / esz);
  C.fpool.ensure((base + add) * esz + 64);
  C.fpool.used = (base + add) * esz;
  auto store = [&](auto* pool) {
    using T = std::remove_pointer_t<decltype(pool)>;
    k_aca_store<T><<<grid_for(nb * 32, 256), 256, 0, st>>>(W.blk.get(), W.state.get(), nb, W.owned.get(), W.rpre.get(),
                                                           base, Uw, Vw, pool, C.foff.get(), C.frank.get(), W.bad.get());
    HM_CHECK_LAUNCH();
    if (nbig)
      k_aca_store_big<T><<<(unsigned)nbig, 256, 0, st>>>(W.blk.get(), W.state.get(), W.big.get(), W.owned.get(),
                                                         W.rpre.get(), base, Uw, Vw, pool, C.foff.get(), C.frank.get(),
                                                         W.bad.get());
  };
  if (esz == 4) store((float*)C.fpool.base);
  else store((double*)C.fpool.base);
  HM_CHECK_LAUNCH();
  if (nov) {
    const size_t o0 = overflow.size();
    overflow.resize(o0 + nov);
    HM_CUDA(cudaMemcpyAsync(overflow.data() + o0, W.ovf.get(), nov * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  }
  if (pivots_out) {
    std::vector<AcaState>& hs = W.h_state;
    hs.resize(nb);
    HM_CUDA(cudaMemcpyAsync(hs.data(), W.state.get(), nb * sizeof(AcaState), cudaMemcpyDeviceToHost, st));
    std::vector<int32_t> hp(nb * 2 * kws);
    HM_CUDA(cudaMemcpyAsync(hp.data(), W.piv.get(), hp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HM_CUDA(cudaStreamSynchronize(st));
    for (int64_t c = 0; c < nb; ++c)
      if (hs[c].status == 1)
        (*pivots_out)[ids[c]].assign(hp.begin() + c * 2 * kws, hp.begin() + c * 2 * kws + 2 * hs[c].k);
  }
  HM_CUDA(cudaStreamSynchronize(st));
  if (nov) std::sort(overflow.end() - nov, overflow.end());
  C.times.aca_phase_ms[3] += ms_since(t2);
}

}  // namespace



void setup_aca(Context& C) {
  cudaStream_t st = C.stream;
  using clk = std::chrono::steady_clock;
  auto ms_since = [](clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); };
  const auto t0 = clk::now();
  const int64_t nb = C.adm_end - C.adm_begin;
  C.lr_esz = C.lr_f32 ? 4 : 8;          // factor storage precision of this setup (option lr_f32)
  C.foff.alloc(nb + 1);
  C.frank.alloc(nb + 1);
  HM_CUDA(cudaMemsetAsync(C.frank.get(), 0, (nb + 1) * sizeof(int32_t), st));
  C.fpool.used = 0;
  C.aca_steps = 0; C.aca_chunks = 0; C.aca_overflow = 0; C.aca_releases = 0;
  for (double& t : C.times.aca_phase_ms) t = 0;
  C.entries_aca = 0;
  if (nb == 0) { C.factor_doubles = 0; C.evals_aca = 0; return; }
  if (C.h_adm.size() != (size_t)C.nadm) {
    C.h_adm.resize(C.nadm);
    HM_CUDA(cudaMemcpyAsync(C.h_adm.data(), C.adm.get(), C.nadm * sizeof(Quad), cudaMemcpyDeviceToHost, st));
    HM_CUDA(cudaStreamSynchronize(st));
  }
  C.times.aca_phase_ms[8] = ms_since(t0);
  // reserve VA for the worst case (k_max terms per block), map on demand
  size_t worst = 0;
  int64_t sum_mn = 0;
  for (int64_t b = C.adm_begin; b < C.adm_end; ++b) {
    const Quad& q = C.h_adm[b];
    int64_t m = q.rhi - q.rlo, n = q.chi - q.clo;
    worst += (size_t)std::min<int64_t>(std::min(m, n), C.k_max) * (m + n);
    sum_mn += m + n;
  }
  const size_t need_va = worst * sizeof(double) + (64u << 20);
  if (!C.fpool.base || C.fpool.reserved < need_va) C.fpool.init(C.device, need_va);   // else reuse the mapped pool
  C.fpool.used = 0;
  if (!C.aca_ws) C.aca_ws = std::make_shared<AcaWork>();
  AcaWork& W = *C.aca_ws;
  W.ev.alloc(1);
  HM_CUDA(cudaMemsetAsync(W.ev.get(), 0, sizeof(unsigned long long), st));
  W.bad.alloc(1);
  {
    const int32_t none = INT_MAX;
    HM_CUDA(cudaMemcpyAsync(W.bad.get(), &none, sizeof(none), cudaMemcpyHostToDevice, st));
  }
  const bool rec = C.record_pivots == 1 || (C.record_pivots < 0 && C.N <= 25000);
  auto& pivots = C.h_piv;
  pivots.clear();
  if (rec) pivots.resize(nb);
  // eps_aca = 0: the paper's fixed-rank mode — no Frobenius stop, every block runs to
  // k = min(m, n, k_max) (or an exactly zero residual), so the workspace holds k_max columns
  const int kws = C.eps_aca == 0.0 ? C.k_max : std::max(1, std::min(C.k_max, (int)C.aca_kws));
  // workspace per chunk: the option, capped by the device memory left at the start of the chunk
  // (the factor pool grows by ~k_mean/KWS of the workspace per chunk, so 0.45 of what is free
  // plus the current workspace leaves room for it)
  // 4 GiB stay free for what follows setup (GMRES basis: (restart+2) N doubles, matvec plan)
  constexpr double kAcaReserve = 4.0 * 1073741824.0;
  // Free device memory is queried once (cudaMemGetInfo costs ~20 ms with a large VMM pool
  // mapped) and then tracked: minus the factor pool's newly mapped bytes and the workspace's
  // growth, plus what a workspace release returns.
  size_t free0 = 0, total0 = 0;
  HM_CUDA(cudaMemGetInfo(&free0, &total0));
  const double mapped0 = (double)C.fpool.mapped;
  const double ws0 = 8.0 * (double)W.ws.n;
  // Chunk budget b (workspace bytes of one chunk): the workspace must fit in `room` (free
  // memory + the current workspace), and a chunk's factor output (<= b) must fit in the pool's
  // mapped-but-unused slack plus the memory beside the workspace.  In repeated setups the
  // pool stays mapped (slack ~ all factors), so chunks can use most of the free memory.
  // The allocated workspace is kept (no multi-GB free/malloc, tens to hundreds of ms) while
  // it is at most twice the budget and the factor growth still fits in the free memory.
  // the same owned block list (signature) with the same ACA options as the previous setup
  const bool steady = C.aca_prev_valid && C.aca_prev_eps == C.eps_aca && C.aca_prev_kmax == C.k_max &&
                      C.aca_prev_esz == C.lr_esz &&
                      C.aca_prev_sig[0] == nb && C.aca_prev_sig[1] == sum_mn;
  const double prev_bytes = steady ? C.aca_prev_bytes : 0.0;   // deterministic ACA: the same factor bytes
  auto chunk_budget = [&]() {
    const auto tb0 = clk::now();
    struct Acc { double& t; clk::time_point a; ~Acc() { t += std::chrono::duration<double, std::milli>(clk::now() - a).count(); } };
    Acc acc_{C.times.aca_phase_ms[7], tb0};
    const double ws = 8.0 * (double)W.ws.n;
    const double free_b = std::max(0.0, (double)free0 - ((double)C.fpool.mapped - mapped0) - (ws - ws0));
    const double slack = std::max(0.0, (double)C.fpool.mapped - (double)C.fpool.used);
    const double room = std::max(0.0, free_b + ws - kAcaReserve);   // keep room for the solve's Krylov basis
    double b = std::min(C.aca_chunk_mb * 1048576.0, 0.9 * room);
    if (b - slack > room - b) b = 0.5 * (room + slack);
    b = std::max(std::min(b, 0.9 * room), 64.0 * 1048576.0);
    if (ws > 0) {
      // Reuse the allocated workspace (freeing / allocating tens of GB costs ~1 s each): chunks
      // of at most its size, provided their factor growth still fits in free memory beside it.
      // Only a too-small buffer (< 1/4 of the budget) is regrown, and it is released only when
      // the pool cannot grow otherwise.
      const double bu = std::min(b, ws);
      // factor growth still to be mapped: known exactly when this tree was set up before with
      // the same options (ACA is deterministic), else bounded by the chunk's workspace bytes
      const double growth = steady ? std::max(0.0, prev_bytes - (double)C.fpool.mapped) : bu - slack;
      if (growth <= free_b) {
        if (ws >= 0.25 * b) b = bu;
      } else {
        W.ws.release();
        C.aca_releases++;
      }
    }
    return b;
  };
  double budget = chunk_budget();
  std::vector<int32_t>& ids = W.h_ids;
  std::vector<int32_t> overflow;
  ids.clear();
  C.times.aca_phase_ms[4] = ms_since(t0);
  double used = 0;
  for (int64_t b = 0; b <= nb; ++b) {
    double need = 0;
    if (b < nb) {
      const Quad& q = C.h_adm[C.adm_begin + b];
      need = 8.0 * kws * ((q.rhi - q.rlo) + (q.chi - q.clo)) + 64.0;
    }
    if (b == nb || (!ids.empty() && used + need > budget)) {
      if (!ids.empty()) {
        run_chunk(C, W, ids, kws, overflow, rec ? &pivots : nullptr);
        C.aca_chunks++;
        budget = chunk_budget();
      }
      ids.clear();
      used = 0;
    }
    if (b < nb) { ids.push_back((int32_t)b); used += need; }
  }
  C.aca_overflow = (int)overflow.size();
  // re-run blocks that filled the workspace from scratch (ACA is deterministic: same pivots,
  // same factors) with twice the columns, until the full rank budget k_max; a smaller
  // workspace per block keeps the re-run chunks few (C6: 203k blocks overflow 12 columns,
  // none 24)
  for (int kw = std::min(C.k_max, 2 * kws); !overflow.empty(); kw = std::min(C.k_max, 2 * kw)) {
    std::vector<int32_t> again, part;
    double u2 = 0;
    for (size_t x = 0; x <= overflow.size(); ++x) {
      double need = 0;
      if (x < overflow.size()) {
        const Quad& q = C.h_adm[C.adm_begin + overflow[x]];
        need = 8.0 * kw * ((q.rhi - q.rlo) + (q.chi - q.clo)) + 64.0;
      }
      if (x == overflow.size() || (!part.empty() && u2 + need > budget)) {
        if (!part.empty()) { run_chunk(C, W, part, kw, again, rec ? &pivots : nullptr); budget = chunk_budget(); }
        part.clear();
        u2 = 0;
      }
      if (x < overflow.size()) { part.push_back(overflow[x]); u2 += need; }
    }
    if (!again.empty() && kw >= C.k_max) fail(HM_ERR_CUDA, "ACA overflow re-run did not converge within k_max");
    overflow.swap(again);
  }
  const auto t5 = clk::now();
  C.h_rank.resize(nb);
  C.h_foff.resize(nb);
  HM_CUDA(cudaMemcpyAsync(C.h_rank.data(), C.frank.get(), nb * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  HM_CUDA(cudaMemcpyAsync(C.h_foff.data(), C.foff.get(), nb * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HM_CUDA(cudaStreamSynchronize(st));
  unsigned long long hev = 0;
  int32_t hbad = INT_MAX;
  HM_CUDA(cudaMemcpyAsync(&hev, W.ev.get(), sizeof(hev), cudaMemcpyDeviceToHost, st));
  HM_CUDA(cudaMemcpyAsync(&hbad, W.bad.get(), sizeof(hbad), cudaMemcpyDeviceToHost, st));
  HM_CUDA(cudaStreamSynchronize(st));
  if (hbad != INT_MAX) {
    const Quad& q = C.h_adm[C.adm_begin + hbad];
    fail(HM_ERR_NUMERIC, "hm_setup: non-finite ACA factor entry in admissible leaf " +
                             std::to_string(C.adm_begin + hbad) + " (rows [" + std::to_string(q.rlo) + "," +
                             std::to_string(q.rhi) + ") x cols [" + std::to_string(q.clo) + "," +
                             std::to_string(q.chi) + "), internal order)");
  }
  C.evals_aca = (double)hev;
  C.factor_doubles = (int64_t)(C.fpool.used / C.lr_esz);       // factor entries (stored as lr_esz bytes)
  C.aca_prev_valid = true;
  C.aca_prev_sig[0] = nb;
  C.aca_prev_sig[1] = sum_mn;
  C.aca_prev_bytes = (double)C.fpool.used;
  C.aca_prev_eps = C.eps_aca;
  C.aca_prev_kmax = C.k_max;
  C.aca_prev_esz = C.lr_esz;
  C.times.aca_phase_ms[5] = ms_since(t5);
}

}  // namespace hm
