// entry.cu — quadrature tables in constant memory, batched entry evaluation for arbitrary
// (i,j) lists (introspection / parity), and the right-hand side f_i = int_{T_i} f.
#include "entry.cuh"
#include "gauss_tables.h"

namespace hm {

__constant__ double c_rs[4][36];
__constant__ double c_rt[4][36];
__constant__ double c_rw[4][36];
__constant__ double c_qs[4][36];
__constant__ double c_qt[4][36];
__constant__ double c_qw[4][36];
__constant__ double c_g6[6];
__constant__ double c_w6[6];

void quadrature_table_host(int n, double* nodes, double* weights) {
  for (int k = 0; k < n; ++k) {
    nodes[k] = kGaussNodes01[n][k];
    weights[k] = kGaussWeights01[n][k];
  }
}

// collapsed Gauss on {0 <= eta2 <= eta1 <= 1}: s = xi, t = xi*zeta, w = (w_xi*w_zeta)*xi (A14)
void upload_quadrature_tables() {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && done[dev]) return;
  double rs[4][36] = {}, rt[4][36] = {}, rw[4][36] = {}, qs[4][36] = {}, qt[4][36] = {}, qw[4][36] = {};
  for (int n = 3; n <= 6; ++n) {
    const double* g = kGaussNodes01[n];
    const double* w = kGaussWeights01[n];
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b) {
        int q = a * n + b;
        if (n == 3) {            // triangles, order 3: Radon's 7-point rule (A14)
          if (q < 7) { rs[0][q] = kRadon7S[q]; rt[0][q] = kRadon7T[q]; rw[0][q] = kRadon7W[q]; }
        } else {
          rs[n - 3][q] = g[a];
          volatile double t = g[a] * g[b];
          rt[n - 3][q] = t;
          volatile double ww = w[a] * w[b];
          volatile double w3 = ww * g[a];
          rw[n - 3][q] = w3;
        }
        qs[n - 3][q] = g[a];              // unit square, tensor (A25)
        qt[n - 3][q] = g[b];
        volatile double wq = w[a] * w[b];
        qw[n - 3][q] = wq;
      }
  }
  HM_CUDA(cudaMemcpyToSymbol(c_rs, rs, sizeof(rs)));
  HM_CUDA(cudaMemcpyToSymbol(c_rt, rt, sizeof(rt)));
  HM_CUDA(cudaMemcpyToSymbol(c_rw, rw, sizeof(rw)));
  HM_CUDA(cudaMemcpyToSymbol(c_qs, qs, sizeof(qs)));
  HM_CUDA(cudaMemcpyToSymbol(c_qt, qt, sizeof(qt)));
  HM_CUDA(cudaMemcpyToSymbol(c_qw, qw, sizeof(qw)));
  HM_CUDA(cudaMemcpyToSymbol(c_g6, kGaussNodes01[6], 6 * sizeof(double)));
  HM_CUDA(cudaMemcpyToSymbol(c_w6, kGaussWeights01[6], 6 * sizeof(double)));
  if (dev < 64) done[dev] = true;
}

__global__ void k_eval_pairs(const Panel* __restrict__ P, const Panel* __restrict__ Pn, const int4* __restrict__ QV,
                             const int32_t* __restrict__ iperm, const int64_t* __restrict__ pairs, int64_t n,
                             double* __restrict__ out) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  int s = iperm[pairs[2 * e]], t = iperm[pairs[2 * e + 1]];
  unsigned long long ev = 0;
  out[e] = Pn ? quad_entry(Pn, P, QV, s, t, ev) : entry_st(P, s, t);
}

void eval_entries(Context& C, int64_t n, const int64_t* d_pairs, double* d_out) {
  if (n == 0) return;
  k_eval_pairs<<<grid_for(n, 128), 128, 0, C.stream>>>(C.panel.get(), C.quad ? C.qnode.get() : nullptr,
                                                        C.qv.get(), C.iperm.get(), d_pairs, n, d_out);
  HM_CHECK_LAUNCH();
}

// f_i = int_{T_i} f: kind 0 f = 1 -> |T_i|; kind 1 f = 4x^2-3y^2-z^2
// with the edge-midpoint rule (exact for quadratics on flat triangles, A16).
__device__ __forceinline__ double paper_f(double x, double y, double z) {
  return dsub(dsub(dmul(dmul(4.0, x), x), dmul(dmul(3.0, y), y)), dmul(z, z));
}

__device__ __forceinline__ double panel_rhs(const Panel& T, int kind) {
  double v;
  if (kind == 0) {
    v = T.area;
  } else {
    double m[3][3];
    for (int k = 0; k < 3; ++k) {
      m[0][k] = ddiv(dadd(T.v[k], T.v[3 + k]), 2.0);
      m[1][k] = ddiv(dadd(T.v[3 + k], T.v[6 + k]), 2.0);
      m[2][k] = ddiv(dadd(T.v[6 + k], T.v[k]), 2.0);
    }
    const double s3 = dadd(dadd(paper_f(m[0][0], m[0][1], m[0][2]), paper_f(m[1][0], m[1][1], m[1][2])),
                           paper_f(m[2][0], m[2][1], m[2][2]));
    v = dmul(ddiv(T.area, 3.0), s3);
  }
  return v;
}

// node s: triangles -> its panel; quads (A25) -> f_2i + f_2i+1 of its two triangles
__global__ void k_rhs(const Panel* __restrict__ P, int64_t N, int kind, bool quad, double* __restrict__ f_app) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= N) return;
  if (quad) f_app[P[2 * s].app >> 1] = dadd(panel_rhs(P[2 * s], kind), panel_rhs(P[2 * s + 1], kind));
  else f_app[P[s].app] = panel_rhs(P[s], kind);
}

void assemble_rhs(Context& C, int kind, double* f_app) {
  k_rhs<<<grid_for(C.N, 256), 256, 0, C.stream>>>(C.panel.get(), C.N, kind, C.quad, f_app);
  HM_CHECK_LAUNCH();
}

}  // namespace hm
