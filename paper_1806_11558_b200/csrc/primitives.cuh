// primitives.cuh — hand-written device-wide exclusive scan and stable LSD radix sort (pairs)
// for the tree build (Morton sort; canonical leaf order, A10), the near-field
// offsets and the per-step ACA compaction.  Replaces the CUB stopgap of round 1.
//
//   exclusive_scan(in, out, n)   out[i] = sum_{j < i} in[j]; three phases: per-tile sums,
//                                a scan of the tile sums (recursively), per-tile scan + offset
//   radix_sort_pairs(...)        stable LSD sort on bits [begin_bit, end_bit) of the keys, 8-bit
//                                digits; per pass: per-tile digit histograms (digit-major), one
//                                exclusive scan over them, a stable scatter (every warp ranks
//                                its 32 x kItems keys in index order with __match_any_sync,
//                                warps of a tile in order, tiles in order)
#pragma once
#include <cstdint>

#include "hm_internal.cuh"

namespace hm {
namespace prim {

constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

template <class T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* sh, T& total) {
  // warp inclusive scan, then warp totals, all exclusive in the end
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    T s = lane < (int)(blockDim.x >> 5) ? sh[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < (int)(blockDim.x >> 5)) sh[lane] = s;      // inclusive warp-total prefix
  }
  __syncthreads();
  total = sh[(blockDim.x >> 5) - 1];
  const T before = w > 0 ? sh[w - 1] : T(0);
  __syncthreads();
  return before + x - v;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_sums(const T* __restrict__ in, int64_t n, T* __restrict__ sums) {
  __shared__ T sh[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) s += in[base + i];
  T tot;
  block_exclusive_scan(s, sh, tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const T* in, int64_t n, const T* __restrict__ offs,
                                                            T* out) {   // in-place allowed
  __shared__ T sh[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? in[base + i] : T(0);
    s += v[i];
  }
  T tot;
  T run = block_exclusive_scan(s, sh, tot) + (offs ? offs[blockIdx.x] : T(0));
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
}

// scratch: sum over levels of ceil(n / tile) elements
template <class T>
inline size_t scan_scratch_elems(int64_t n) {
  size_t e = 0;
  while (n > kScanTile) {
    n = (n + kScanTile - 1) / kScanTile;
    e += (size_t)n + 1;
  }
  return e + 1;
}

// out may alias in; scratch: scan_scratch_elems<T>(n) elements
template <class T>
void exclusive_scan_raw(const T* in, T* out, int64_t n, T* scratch, cudaStream_t st) {
  if (n <= 0) return;
  if (n <= kScanTile) {
    k_tile_scan<T><<<1, kScanThreads, 0, st>>>(in, n, nullptr, out);
    HM_CHECK_LAUNCH();
    return;
  }
  // tile sums -> their exclusive scan (recursively, in the scratch) -> per-tile scan + offsets
  const int64_t nt = (n + kScanTile - 1) / kScanTile;
  T* sums = scratch;
  k_tile_sums<T><<<(unsigned)nt, kScanThreads, 0, st>>>(in, n, sums);
  HM_CHECK_LAUNCH();
  exclusive_scan_raw<T>(sums, sums, nt, scratch + nt + 1, st);
  k_tile_scan<T><<<(unsigned)nt, kScanThreads, 0, st>>>(in, n, sums, out);
  HM_CHECK_LAUNCH();
}

template <class T>
void exclusive_scan(const T* in, T* out, int64_t n, DBuf<char>& tmp, cudaStream_t st) {
  if (n <= 0) return;
  tmp.alloc(scan_scratch_elems<T>(n) * sizeof(T) + 64);
  exclusive_scan_raw<T>(in, out, n, reinterpret_cast<T*>(tmp.get()), st);
}

// ---- radix sort -------------------------------------------------------------------------------
constexpr int kSortThreads = 256, kSortItems = 8, kSortTile = kSortThreads * kSortItems, kRadix = 256;

template <class K>
__device__ __forceinline__ int digit_of(K k, int shift, int mask) { return (int)((k >> shift) & (K)mask); }

// hist[d * ntiles + tile] = count of digit d in the tile
template <class K>
__global__ void __launch_bounds__(kSortThreads) k_radix_hist(const K* __restrict__ keys, int64_t n, int shift, int mask,
                                                             int64_t ntiles, int64_t* __restrict__ hist) {
  __shared__ int cnt[kRadix];
  for (int d = threadIdx.x; d < kRadix; d += blockDim.x) cnt[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int i = threadIdx.x; i < kSortTile; i += blockDim.x)
    if (base + i < n) atomicAdd(&cnt[digit_of(keys[base + i], shift, mask)], 1);
  __syncthreads();
  for (int d = threadIdx.x; d < kRadix; d += blockDim.x) hist[(int64_t)d * ntiles + blockIdx.x] = cnt[d];
}

// Stable scatter: warp w of the tile owns keys [base + w 32 kSortItems, +32 kSortItems) in index
// order; round r covers 32 consecutive keys, lane order = index order.
template <class K, class V>
__global__ void __launch_bounds__(kSortThreads) k_radix_scatter(const K* __restrict__ kin, K* __restrict__ kout,
                                                                const V* __restrict__ vin, V* __restrict__ vout,
                                                                int64_t n, int shift, int mask, int64_t ntiles,
                                                                const int64_t* __restrict__ goff) {
  constexpr int NW = kSortThreads / 32;
  __shared__ int cnt[NW][kRadix];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = lane; d < kRadix; d += 32) cnt[w][d] = 0;
  __syncwarp();
  const int64_t base = (int64_t)blockIdx.x * kSortTile + (int64_t)w * 32 * kSortItems;
  const unsigned lt = (1u << lane) - 1u;
  int rank[kSortItems], dig[kSortItems];
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const int64_t i = base + r * 32 + lane;
    const bool valid = i < n;
    const int d = valid ? digit_of(kin[i], shift, mask) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int before = __popc(peers & lt);
    int c = 0;
    if (valid) c = cnt[w][d];
    __syncwarp();
    if (valid && before == 0) cnt[w][d] = c + __popc(peers);
    __syncwarp();
    rank[r] = c + before;
    dig[r] = d;
  }
  __syncthreads();
  // per digit: exclusive prefix over the warps of the tile (warp order = index order)
  for (int d = threadIdx.x; d < kRadix; d += blockDim.x) {
    int run = 0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) {
      const int t = cnt[ww][d];
      cnt[ww][d] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const int64_t i = base + r * 32 + lane;
    if (i < n) {
      const int d = dig[r];
      const int64_t dst = goff[(int64_t)d * ntiles + blockIdx.x] + cnt[w][d] + rank[r];
      kout[dst] = kin[i];
      vout[dst] = vin[i];
    }
  }
}

// Sort (keys, values) by bits [begin_bit, end_bit) of the keys, stable (equal keys keep their
// input order), kin / vin -> kout / vout (inputs untouched).  tmp holds the per-pass histograms,
// their scan scratch and one ping-pong copy of keys and values.
template <class K, class V>
void radix_sort_pairs(const K* kin, K* kout, const V* vin, V* vout, int64_t n, int begin_bit, int end_bit,
                      DBuf<char>& tmp, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
  const int64_t nh = kRadix * ntiles;
  auto up16 = [](size_t b) { return (b + 15) & ~size_t(15); };
  const size_t hb = up16((nh + scan_scratch_elems<int64_t>(nh) + 8) * sizeof(int64_t));
  const size_t kb = up16(n * sizeof(K)), vb = up16(n * sizeof(V));
  tmp.alloc(hb + kb + vb);
  int64_t* hist = reinterpret_cast<int64_t*>(tmp.get());
  int64_t* scratch = hist + nh;
  K* kalt = reinterpret_cast<K*>(tmp.get() + hb);
  V* valt = reinterpret_cast<V*>(tmp.get() + hb + kb);
  const int passes = (end_bit - begin_bit + 7) / 8;
  const K* ks = kin;
  const V* vs = vin;
  for (int p = 0; p < passes; ++p) {
    const int shift = begin_bit + 8 * p;
    const int bits = end_bit - shift < 8 ? end_bit - shift : 8;
    const int mask = (1 << bits) - 1;
    // the last pass writes kout / vout, the ones before alternate with kalt / valt
    K* kd = ((passes - 1 - p) % 2 == 0) ? kout : kalt;
    V* vd = ((passes - 1 - p) % 2 == 0) ? vout : valt;
    k_radix_hist<K><<<(unsigned)ntiles, kSortThreads, 0, st>>>(ks, n, shift, mask, ntiles, hist);
    HM_CHECK_LAUNCH();
    exclusive_scan_raw<int64_t>(hist, hist, nh, scratch, st);
    k_radix_scatter<K, V><<<(unsigned)ntiles, kSortThreads, 0, st>>>(ks, kd, vs, vd, n, shift, mask, ntiles, hist);
    HM_CHECK_LAUNCH();
    ks = kd;
    vs = vd;
  }
}

}  // namespace prim
}  // namespace hm
