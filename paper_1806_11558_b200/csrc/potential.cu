// potential.cu — single-layer potential of the solved density at evaluation points
// (u~(x) = int_Gamma G(x, y) u_h(y) dsigma_y; the paper's accuracy metric
// evaluates it inside the domain).  With u_h = sum_j alpha_j phi_j (A2):
//   u~(x) = (1/4pi) sum_j alpha_j int_{T_j} 1/|x - y| dy,
// each panel integral by the triangle rule of the regular entries (A14) on T_j alone,
// order n from rho^2 = |x - c_j|^2 / h_j^2 in the same bands (reading A23).  Direct sum
// over all panels (M points x N panels; a few hundred points cost milliseconds), every rank
// computes all points (collective-free; alpha is replicated).
//
// Grid: (panel tiles of 256) x (point tiles of kPts).  A thread owns one panel and keeps the
// kPts points' sums in registers; the CTA reduces them through shared memory and adds one
// FP64 atomic per point.
#include <algorithm>

#include "entry.cuh"

namespace hm {

namespace {

constexpr int kPts = 8;

// panels s < NP; the density of panel s is alpha_int[s >> qshift] (quads: both triangles of
// node s >> 1 carry alpha, A25)
__global__ void __launch_bounds__(256) k_potential(const Panel* __restrict__ P, const double* __restrict__ alpha_int,
                                                   int64_t N, int qshift, const double* __restrict__ X, int64_t M,
                                                   double* __restrict__ out) {
  __shared__ double sx[kPts][3];
  __shared__ double red[kPts][8];
  const int64_t p0 = (int64_t)blockIdx.y * kPts;
  if (threadIdx.x < kPts * 3) {
    const int64_t p = p0 + threadIdx.x / 3;
    sx[threadIdx.x / 3][threadIdx.x % 3] = p < M ? X[3 * p + threadIdx.x % 3] : 0.0;
  }
  __syncthreads();
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double acc[kPts];
#pragma unroll
  for (int q = 0; q < kPts; ++q) acc[q] = 0.0;
  if (s < N) {
    double V[9];
    load_panel_vertices(P, (int)s, V);
    const double cx = __ldg(&P[s].c[0]), cy = __ldg(&P[s].c[1]), cz = __ldg(&P[s].c[2]);
    const double h = __ldg(&P[s].h), h2 = dmul(h, h);
    const double a = __ldg(alpha_int + (s >> qshift)), two_area = dmul(2.0, __ldg(&P[s].area));
    const double e1x = dsub(V[3], V[0]), e1y = dsub(V[4], V[1]), e1z = dsub(V[5], V[2]);
    const double e2x = dsub(V[6], V[3]), e2y = dsub(V[7], V[4]), e2z = dsub(V[8], V[5]);
    for (int q = 0; q < kPts; ++q) {
      if (p0 + q >= M) break;
      const double x = sx[q][0], y = sx[q][1], z = sx[q][2];
      const double dx = dsub(x, cx), dy = dsub(y, cy), dz = dsub(z, cz);
      const double dc2 = dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
      const int n = dc2 < dmul(4.0, h2) ? 6 : dc2 < dmul(16.0, h2) ? 5 : dc2 < dmul(64.0, h2) ? 4 : 3;
      const double* S = c_rs[n - 3];
      const double* T = c_rt[n - 3];
      const double* W = c_rw[n - 3];
      double inner = 0.0;
      const int np = tri_rule_points(n);
      for (int k = 0; k < np; ++k) {
        const double px = dfma(T[k], e2x, dfma(S[k], e1x, V[0]));
        const double py = dfma(T[k], e2y, dfma(S[k], e1y, V[1]));
        const double pz = dfma(T[k], e2z, dfma(S[k], e1z, V[2]));
        const double ex = dsub(x, px), ey = dsub(y, py), ez = dsub(z, pz);
        inner = dadd(inner, qterm(W[k], dfma(ez, ez, dfma(ey, ey, dmul(ex, ex)))));
      }
      acc[q] = dmul(a, dmul(inner, two_area));
    }
  }
  // CTA reduction per point: warp butterflies, then the 8 warp sums in fixed order
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < kPts; ++q) {
    double v = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[q][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < kPts && p0 + threadIdx.x < M) {
    double v = 0.0;
    for (int g = 0; g < 8; ++g) v += red[threadIdx.x][g];
    atomicAdd(out + p0 + threadIdx.x, v);
  }
}

__global__ void k_scale_inplace(double* __restrict__ a, int64_t n, double f) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = dmul(a[i], f);
}

}  // namespace

void potential(Context& C, const double* alpha_app, int64_t M, const double* X_dev, double* out_dev) {
  cudaStream_t st = C.stream;
  C.xin.alloc(C.N);
  gather_perm(C, alpha_app, C.xin.get());
  HM_CUDA(cudaMemsetAsync(out_dev, 0, M * sizeof(double), st));
  if (M == 0) return;
  // point tiles on grid.y, at most 65535 per launch (gridDim.y limit): launches over point slices
  constexpr int64_t kMaxTilesY = 65535;
  for (int64_t p0 = 0; p0 < M; p0 += kMaxTilesY * kPts) {
    const int64_t m = std::min<int64_t>(M - p0, kMaxTilesY * kPts);
    const dim3 grid(grid_for(C.npanel, 256), (unsigned)((m + kPts - 1) / kPts));
    k_potential<<<grid, 256, 0, st>>>(C.panel.get(), C.xin.get(), C.npanel, C.quad ? 1 : 0, X_dev + 3 * p0, m,
                                      out_dev + p0);
    HM_CHECK_LAUNCH();
  }
  k_scale_inplace<<<grid_for(M, 256), 256, 0, st>>>(out_dev, M, kInv4Pi);
  HM_CHECK_LAUNCH();
}

}  // namespace hm
