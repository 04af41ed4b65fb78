// matvec.cu — batched H-matrix-vector product: non-admissible leaves apply their
// stored dense block, admissible leaves apply U (V^T x) ("two matrix-vector products
// of skinny matrices"); application<->internal permutations at entry and exit.
//
// Memory-bound (0.25 flop/B).  Storage is streamed once per product in storage order:
//   dense leaves   one warp per leaf; s lanes per row (s = pow2 ~ n/4) so each load
//                  instruction touches whole 32-B sectors; per-row shuffle reduction, one
//                  FP64 atomic per row into the L2-resident y.
//   low-rank       [U m x k | V n x k] col-major, contiguous per block: t = V^T x_sigma as k
//                  coalesced dot products, then y_tau += U t with lanes over rows (coalesced
//                  along each u_l), one atomic per row.  Warp per block when m+n <= 1024,
//                  CTA (256 threads) per block above.
#include <cub/cub.cuh>

#include "entry.cuh"

namespace hm {

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

template <int S>
__device__ __forceinline__ void dense_rows(const double* __restrict__ B, int m, int n, const double* __restrict__ x,
                                           double* __restrict__ y, int lane) {
  constexpr int RPP = 32 / S;               // rows per pass
  const int sub = lane % S, rr = lane / S;
  for (int r0 = 0; r0 < m; r0 += RPP) {
    const int r = r0 + rr;
    double acc = 0.0;
    if (r < m) {
      const double* row = B + (int64_t)r * n;
      for (int c = sub; c < n; c += S) acc += __ldg(row + c) * __ldg(x + c);
    }
#pragma unroll
    for (int o = S / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (sub == 0 && r < m) atomicAdd(y + r, acc);
  }
}

__global__ void k_mv_dense(const Quad* __restrict__ q, const int64_t* __restrict__ off, int64_t nb,
                           const double* __restrict__ store, const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = w0; b < nb; b += nw) {
    const Quad Q = q[b];
    const int m = Q.rhi - Q.rlo, n = Q.chi - Q.clo;
    const double* B = store + off[b];
    if (n <= 8) dense_rows<2>(B, m, n, x + Q.clo, y + Q.rlo, lane);
    else if (n <= 16) dense_rows<4>(B, m, n, x + Q.clo, y + Q.rlo, lane);
    else if (n <= 48) dense_rows<8>(B, m, n, x + Q.clo, y + Q.rlo, lane);
    else if (n <= 96) dense_rows<16>(B, m, n, x + Q.clo, y + Q.rlo, lane);
    else dense_rows<32>(B, m, n, x + Q.clo, y + Q.rlo, lane);
  }
}

// warp per low-rank block (m + n <= 1024)
__global__ void k_mv_lowrank_warp(const Quad* __restrict__ q, const int32_t* __restrict__ list, int64_t nl,
                                  const int64_t* __restrict__ foff, const int32_t* __restrict__ frank,
                                  const double* __restrict__ pool, const double* __restrict__ x,
                                  double* __restrict__ y) {
  __shared__ double tsh[8][64];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t a = w0; a < nl; a += nw) {
    const int b = list[a];
    const int k = frank[b];
    if (k <= 0) continue;
    const Quad Q = q[b];
    const int m = Q.rhi - Q.rlo, n = Q.chi - Q.clo;
    const double* U = pool + foff[b];
    const double* V = U + (int64_t)m * k;
    const double* xs = x + Q.clo;
    for (int l = 0; l < k; ++l) {
      const double* v = V + (int64_t)l * n;
      double acc = 0.0;
      for (int j = lane; j < n; j += 32) acc += __ldg(v + j) * __ldg(xs + j);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) tsh[wib][l] = acc;
    }
    __syncwarp();
    for (int t = lane; t < m; t += 32) {
      double acc = 0.0;
      for (int l = 0; l < k; ++l) acc += __ldg(U + t + (int64_t)l * m) * tsh[wib][l];
      atomicAdd(y + Q.rlo + t, acc);
    }
    __syncwarp();
  }
}

// CTA (256 threads) per large low-rank block
__global__ void k_mv_lowrank_cta(const Quad* __restrict__ q, const int32_t* __restrict__ list, int64_t nl,
                                 const int64_t* __restrict__ foff, const int32_t* __restrict__ frank,
                                 const double* __restrict__ pool, const double* __restrict__ x,
                                 double* __restrict__ y) {
  __shared__ double part[8][64];
  __shared__ double tsh[64];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (int64_t a = blockIdx.x; a < nl; a += gridDim.x) {
    const int b = list[a];
    const int k = frank[b];
    if (k <= 0) continue;
    const Quad Q = q[b];
    const int m = Q.rhi - Q.rlo, n = Q.chi - Q.clo;
    const double* U = pool + foff[b];
    const double* V = U + (int64_t)m * k;
    const double* xs = x + Q.clo;
    for (int l = 0; l < k; ++l) {
      const double* v = V + (int64_t)l * n;
      double acc = 0.0;
      for (int j = threadIdx.x; j < n; j += blockDim.x) acc += __ldg(v + j) * __ldg(xs + j);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) part[wib][l] = acc;
    }
    __syncthreads();
    if (threadIdx.x < k) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w][threadIdx.x];
      tsh[threadIdx.x] = s;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < m; t += blockDim.x) {
      double acc = 0.0;
      for (int l = 0; l < k; ++l) acc += __ldg(U + t + (int64_t)l * m) * tsh[l];
      atomicAdd(y + Q.rlo + t, acc);
    }
    __syncthreads();
  }
}

}  // namespace

void plan_matvec(Context& C) {
  const int64_t nb = C.adm_end - C.adm_begin;
  std::vector<int32_t> small, large;
  for (int64_t b = 0; b < nb; ++b) {
    const Quad& q = C.h_adm[C.adm_begin + b];
    if (C.h_rank[b] <= 0) continue;
    if ((q.rhi - q.rlo) + (q.chi - q.clo) <= 1024) small.push_back((int32_t)b);
    else large.push_back((int32_t)b);
  }
  C.n_lr_small = (int64_t)small.size();
  C.n_lr_large = (int64_t)large.size();
  C.lr_small.alloc_exact(C.n_lr_small);
  C.lr_large.alloc_exact(C.n_lr_large);
  if (C.n_lr_small)
    HM_CUDA(cudaMemcpyAsync(C.lr_small.get(), small.data(), small.size() * 4, cudaMemcpyHostToDevice, C.stream));
  if (C.n_lr_large)
    HM_CUDA(cudaMemcpyAsync(C.lr_large.get(), large.data(), large.size() * 4, cudaMemcpyHostToDevice, C.stream));
  HM_CUDA(cudaStreamSynchronize(C.stream));
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
  HM_CUDA(cudaMemsetAsync(y_int, 0, C.N * sizeof(double), st));
  const int64_t nd = C.dense_end - C.dense_begin;
  const int sms = 148;
  if (nd) {
    k_mv_dense<<<sms * 8, 256, 0, st>>>(C.dense.get() + C.dense_begin, C.doff.get(), nd, C.dstore.get(), x_int, y_int);
    HM_CHECK_LAUNCH();
  }
  const Quad* qa = C.adm.get() + C.adm_begin;
  if (C.n_lr_small) {
    k_mv_lowrank_warp<<<sms * 8, 256, 0, st>>>(qa, C.lr_small.get(), C.n_lr_small, C.foff.get(), C.frank.get(),
                                               (const double*)C.fpool.base, x_int, y_int);
    HM_CHECK_LAUNCH();
  }
  if (C.n_lr_large) {
    k_mv_lowrank_cta<<<sms * 4, 256, 0, st>>>(qa, C.lr_large.get(), C.n_lr_large, C.foff.get(), C.frank.get(),
                                              (const double*)C.fpool.base, x_int, y_int);
    HM_CHECK_LAUNCH();
  }
  if (C.world > 1) allreduce_sum(C, y_int, C.N);
}

}  // namespace hm
