// solver.cu — Krylov solvers driving the batched H-matvec (A17):
//   CG (the paper's solver) and GMRES(m) with classical Gram-Schmidt + one
//   re-orthogonalisation (CGS2) and Givens rotations (BASELINE.json's solver).
// Vectors live in internal (Morton) order on the device.  One rank: full vectors.  p ranks:
// every Krylov vector is sharded by internal row range (rank r owns [r S, r S + n), S =
// ceil(N / p)); each matvec all-gathers x (ncclAllGather), applies the rank's leaves and
// reduce-scatters the partial y into the slices (ncclReduceScatter) — the volume of the
// paper's replicated vector + global sum; dot products are local fixed-grid tree
// reductions followed by an ncclAllReduce of the partials, so every rank sees bit-identical
// scalars and takes identical convergence decisions.  x0 = 0; stop at ||r|| <= tol ||b||.

#include <algorithm>
#include <cmath>

#include "entry.cuh"

namespace hm {

namespace {

constexpr int kRedBlocks = 296;
constexpr int kRedThreads = 256;

// partial dot products of w against nv vectors V[i] (stride ld), for i < nv; partial[b*nv + i];
// extra != nullptr: the last one (i = nv - 1) is extra^T w instead of V[nv-1]^T w
__global__ void k_mdot(const double* __restrict__ Vb, int64_t ld, int nv, const double* __restrict__ w, int64_t n,
                       double* __restrict__ partial, const double* __restrict__ extra) {
  __shared__ double sh[kRedThreads / 32][33];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (int i0 = 0; i0 < nv; i0 += 32) {
    const int cnt = min(32, nv - i0);
    double acc[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q] = 0.0;
    // the basis vectors of this pass; an extra vector (i = nv - 1, slot nb) is read from `extra`
    const int nb = (extra && i0 + cnt == nv) ? cnt - 1 : cnt;
    double accx = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
      const double wt = w[t];
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q < nb) acc[q] += Vb[(int64_t)(i0 + q) * ld + t] * wt;
      if (nb < cnt) accx += (extra == w ? wt : extra[t]) * wt;
    }
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      double a = (q == nb) ? accx : acc[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) sh[wib][q] = a;
    }
    __syncthreads();
    if (threadIdx.x < cnt) {
      double s = 0.0;
      for (int w2 = 0; w2 < kRedThreads / 32; ++w2) s += sh[w2][threadIdx.x];
      partial[(int64_t)blockIdx.x * nv + i0 + threadIdx.x] = s;
    }
    __syncthreads();
  }
}

__global__ void k_mdot_final(const double* __restrict__ partial, int nb, int nv, double* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += partial[(int64_t)b * nv + i];
  out[i] = s;
}

// w -= sum_i h[i] V[i]  (i ascending)
__global__ void k_msub(const double* __restrict__ Vb, int64_t ld, int nv, const double* __restrict__ h,
                       double* __restrict__ w, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double x = w[t];
    for (int i = 0; i < nv; ++i) x -= h[i] * Vb[(int64_t)i * ld + t];
    w[t] = x;
  }
}

// y += sum_i c[i] V[i]
__global__ void k_madd(const double* __restrict__ Vb, int64_t ld, int nv, const double* __restrict__ c,
                       double* __restrict__ y, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double x = y[t];
    for (int i = 0; i < nv; ++i) x += c[i] * Vb[(int64_t)i * ld + t];
    y[t] = x;
  }
}

__global__ void k_scale_to(const double* __restrict__ a, const double* __restrict__ s, bool recip,
                           double* __restrict__ out, int64_t n) {
  const double f = recip ? 1.0 / *s : *s;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = a[t] * f;
}

__global__ void k_sub(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = a[t] - b[t];
}

// CG update: x += a p; r -= a Ap
__global__ void k_cg_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                        const double* __restrict__ Ap, double a, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    x[t] += a * p[t];
    r[t] -= a * Ap[t];
  }
}

__global__ void k_cg_p(double* __restrict__ p, const double* __restrict__ r, double beta, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    p[t] = r[t] + beta * p[t];
}

// Krylov vector layout.  One rank: the full internal-order vector.  p ranks: rank r owns the
// slice [r S, r S + n) with S = ceil(N / p) (the last slice shorter); dot products are local
// sums all-reduced over NCCL, and the matvec all-gathers x into a p*S buffer whose first N
// entries are the internal-order x, applies the rank's leaves and reduce-scatters y back
// into slices (same NVLink volume as the replicated all-reduce, but the orthogonalisation
// work is split p ways).
struct Layout {
  int64_t n = 0, S = 0, off = 0;
  bool sharded = false;
};

struct Red {
  Context& C;
  const Layout& L;
  DBuf<double> part, out;
  Red(Context& c, const Layout& l) : C(c), L(l) {}
  // out[0..nv) = V[i]^T w (global) on the device; returns device pointer
  double* mdot(const double* Vb, int64_t ld, int nv, const double* w, const double* extra = nullptr) {
    part.alloc((size_t)kRedBlocks * nv);
    out.alloc(nv + 8);
    { KScope ks_(C, KF_KRYLOV);
    k_mdot<<<kRedBlocks, kRedThreads, 0, C.stream>>>(Vb, ld, nv, w, L.n, part.get(), extra);
    }
    { KScope ks_(C, KF_KRYLOV);
    k_mdot_final<<<(nv + 127) / 128, 128, 0, C.stream>>>(part.get(), kRedBlocks, nv, out.get());
    }
    HM_CHECK_LAUNCH();
    if (L.sharded) {
      if (p2p_on(C)) p2p_allreduce(C, out.get(), nv);
      else allreduce_sum(C, out.get(), nv);
    }
    return out.get();
  }
  double dot(const double* a, const double* b) {
    double* d = mdot(a, 0, 1, b);
    double h;
    HM_CUDA(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    HM_CUDA(cudaStreamSynchronize(C.stream));
    return h;
  }
};

unsigned vgrid(int64_t n) { return std::min<unsigned>(grid_for(n, 256), 148 * 16); }

// gathered: x was already published into every rank's gathered vector by the kernel that
// produced it (p2p_scale_publish), so the product starts without an all-gather
void apply(Context& C, const Layout& L, const double* x, double* y, bool gathered = false) {
  if (!L.sharded) { matvec_internal(C, x, y); return; }
  if (p2p_on(C)) {             // libhm's own collectives over NVLink peer memory (p2p.cu)
    if (!gathered) p2p_allgather(C, x, L.n, L.S);
    matvec_internal(C, p2p_xfull(C), p2p_ypart(C), /*reduce=*/false);
    p2p_reduce_scatter(C, y, L.n, L.S);
    return;
  }
  { KScope ks_(C, KF_COMM);
  HM_NCCL(ncclAllGather(x, C.sh_x.get(), (size_t)L.S, ncclDouble, C.comm, C.stream));
  }
  matvec_internal(C, C.sh_x.get(), C.sh_y.get(), /*reduce=*/false);
  { KScope ks_(C, KF_COMM);
  HM_NCCL(ncclReduceScatter(C.sh_y.get(), y, (size_t)L.S, ncclDouble, ncclSum, C.comm, C.stream));
  }
}

double true_relres(Context& C, const Layout& L, Red& R, const double* b, const double* x, double bn, double* tmp) {
  apply(C, L, x, tmp);
  { KScope ks_(C, KF_KRYLOV);
  k_sub<<<vgrid(L.n), 256, 0, C.stream>>>(b, tmp, tmp, L.n);
  }
  HM_CHECK_LAUNCH();
  double rr = R.dot(tmp, tmp);
  return bn > 0 ? std::sqrt(rr) / bn : 0.0;
}

void cg(Context& C, const Layout& L, const double* b, double* x, double tol, int* iters, double* relres) {
  const int64_t N = L.n;
  cudaStream_t st = C.stream;
  const int64_t ld = (L.S + 32) & ~int64_t(31);   // 256-B aligned vectors with slack (matvec x staging)
  C.krylov.alloc(3 * ld);
  double *r = C.krylov.get(), *p = r + ld, *Ap = p + ld;
  Red R(C, L);
  HM_CUDA(cudaMemsetAsync(x, 0, N * sizeof(double), st));
  HM_CUDA(cudaMemcpyAsync(r, b, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  HM_CUDA(cudaMemcpyAsync(p, b, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  const double bn = std::sqrt(R.dot(b, b));
  double rr = R.dot(r, r);
  int it = 0;
  if (bn == 0.0) { *iters = 0; *relres = 0.0; return; }
  while (it < C.max_iter && std::sqrt(rr) > tol * bn) {
    apply(C, L, p, Ap);
    const double pAp = R.dot(p, Ap);
    if (!(pAp > 0.0)) fail(HM_ERR_BREAKDOWN, "CG breakdown: p^T H p <= 0 at iteration " + std::to_string(it));
    const double alpha = rr / pAp;
    { KScope ks_(C, KF_KRYLOV);
    k_cg_xr<<<vgrid(N), 256, 0, st>>>(x, r, p, Ap, alpha, N);
    }
    HM_CHECK_LAUNCH();
    const double rr1 = R.dot(r, r);
    const double beta = rr1 / rr;
    rr = rr1;
    { KScope ks_(C, KF_KRYLOV);
    k_cg_p<<<vgrid(N), 256, 0, st>>>(p, r, beta, N);
    }
    HM_CHECK_LAUNCH();
    ++it;
  }
  *iters = it;
  *relres = true_relres(C, L, R, b, x, bn, Ap);
}

void gmres(Context& C, const Layout& L, const double* b, double* x, double tol, int* iters, double* relres) {
  const int64_t N = L.n;
  const int m = std::max(1, C.restart);
  cudaStream_t st = C.stream;
  const int64_t ld = (L.S + 32) & ~int64_t(31);   // 256-B aligned basis vectors with slack (matvec x staging)
  C.krylov.alloc((size_t)(m + 2) * ld);
  double* Vb = C.krylov.get();
  double* w = Vb + (int64_t)(m + 1) * ld;
  Red R(C, L);
  DBuf<double> hdev, hsum;
  hdev.alloc(m + 8);
  std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1), h(m + 1), h2(m + 2), y(m);
  HM_CUDA(cudaMemsetAsync(x, 0, N * sizeof(double), st));
  const double bn = std::sqrt(R.dot(b, b));
  int total = 0;
  if (bn == 0.0) { *iters = 0; *relres = 0.0; return; }
  bool x_zero = true;          // first cycle: x0 = 0, so r0 = b exactly (no product)
  for (;;) {
    if (x_zero) {
      HM_CUDA(cudaMemcpyAsync(w, b, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
    } else {
      apply(C, L, x, w);
      { KScope ks_(C, KF_KRYLOV);
      k_sub<<<vgrid(N), 256, 0, st>>>(b, w, w, N);
      }
      HM_CHECK_LAUNCH();
    }
    const double beta = std::sqrt(R.dot(w, w));
    if (beta <= tol * bn || total >= C.max_iter) break;
    HM_CUDA(cudaMemcpyAsync(hdev.get(), &beta, sizeof(double), cudaMemcpyHostToDevice, st));
    // sharded over P2P: the normalisation also publishes the next product's x (fused all-gather)
    const bool fused = L.sharded && p2p_on(C);
    if (fused) {
      p2p_scale_publish(C, w, hdev.get(), Vb, N, L.S);
    } else {
      { KScope ks_(C, KF_KRYLOV);
      k_scale_to<<<vgrid(N), 256, 0, st>>>(w, hdev.get(), true, Vb, N);
      }
      HM_CHECK_LAUNCH();
    }
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int jend = 0;
    bool conv = false;
    for (int j = 0; j < m; ++j) {
      apply(C, L, Vb + (int64_t)j * ld, w, fused);
      ++total;
      // CGS2
      double* d1 = R.mdot(Vb, ld, j + 1, w);
      { KScope ks_(C, KF_KRYLOV);
      k_msub<<<vgrid(N), 256, 0, st>>>(Vb, ld, j + 1, d1, w, N);
      }
      HM_CHECK_LAUNCH();
      HM_CUDA(cudaMemcpyAsync(h.data(), d1, (j + 1) * sizeof(double), cudaMemcpyDeviceToHost, st));
      // second projection and ||w'||^2 in one reduction (one all-reduce, one host sync per
      // iteration): ||w' - V h2||^2 = ||w'||^2 - ||h2||^2 for orthonormal V, and h2 is ~1e-8
      // ||w'|| after the first projection, so the difference does not cancel
      double* d2 = R.mdot(Vb, ld, j + 2, w, w);
      { KScope ks_(C, KF_KRYLOV);
      k_msub<<<vgrid(N), 256, 0, st>>>(Vb, ld, j + 1, d2, w, N);
      }
      HM_CHECK_LAUNCH();
      HM_CUDA(cudaMemcpyAsync(h2.data(), d2, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, st));
      HM_CUDA(cudaStreamSynchronize(st));
      double hh2 = 0.0;
      for (int i = 0; i <= j; ++i) { h[i] += h2[i]; hh2 += h2[i] * h2[i]; }
      const double hn = std::sqrt(std::max(0.0, h2[j + 1] - hh2));
      for (int i = 0; i < j; ++i) {
        const double t1 = cs[i] * h[i] + sn[i] * h[i + 1];
        const double t2 = -sn[i] * h[i] + cs[i] * h[i + 1];
        h[i] = t1; h[i + 1] = t2;
      }
      const double den = std::sqrt(h[j] * h[j] + hn * hn);
      if (den == 0.0) { cs[j] = 1.0; sn[j] = 0.0; }
      else { cs[j] = h[j] / den; sn[j] = hn / den; }
      h[j] = cs[j] * h[j] + sn[j] * hn;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      for (int i = 0; i <= j; ++i) H[i + (size_t)j * (m + 1)] = h[i];
      jend = j + 1;
      if (std::fabs(g[j + 1]) <= tol * bn || total >= C.max_iter || hn == 0.0) { conv = true; break; }
      HM_CUDA(cudaMemcpyAsync(hdev.get(), &hn, sizeof(double), cudaMemcpyHostToDevice, st));
      if (fused) {
        p2p_scale_publish(C, w, hdev.get(), Vb + (int64_t)(j + 1) * ld, N, L.S);
      } else {
        { KScope ks_(C, KF_KRYLOV);
        k_scale_to<<<vgrid(N), 256, 0, st>>>(w, hdev.get(), true, Vb + (int64_t)(j + 1) * ld, N);
        }
        HM_CHECK_LAUNCH();
      }
    }
    for (int i = jend - 1; i >= 0; --i) {
      double s = g[i];
      for (int l = i + 1; l < jend; ++l) s -= H[i + (size_t)l * (m + 1)] * y[l];
      y[i] = s / H[i + (size_t)i * (m + 1)];
    }
    HM_CUDA(cudaMemcpyAsync(hdev.get(), y.data(), jend * sizeof(double), cudaMemcpyHostToDevice, st));
    { KScope ks_(C, KF_KRYLOV);
    k_madd<<<vgrid(N), 256, 0, st>>>(Vb, ld, jend, hdev.get(), x, N);
    }
    HM_CHECK_LAUNCH();
    x_zero = false;
    HM_CUDA(cudaStreamSynchronize(st));
    if (conv && (std::fabs(g[jend]) <= tol * bn || total >= C.max_iter)) break;
    if (total >= C.max_iter) break;
  }
  *iters = total;
  *relres = true_relres(C, L, R, b, x, bn, w);
}

}  // namespace

void solve(Context& C, const double* rhs_int, double* sol_int, double tol, int* iters, double* relres) {
  Layout L;
  if (C.world == 1) {
    L.n = L.S = C.N;
    if (C.solver == 1) cg(C, L, rhs_int, sol_int, tol, iters, relres);
    else gmres(C, L, rhs_int, sol_int, tol, iters, relres);
    return;
  }
  // p ranks: sharded Krylov vectors (Layout), the replicated rhs is read in place
  L.sharded = true;
  L.S = (C.N + C.world - 1) / C.world;
  L.off = std::min<int64_t>((int64_t)C.rank * L.S, C.N);
  L.n = std::min<int64_t>(L.S, C.N - L.off);
  const int64_t full = L.S * C.world;
  if (C.sh_x.n < (size_t)full + 32) {
    C.sh_x.alloc(full + 32);
    C.sh_y.alloc(full + 32);
    HM_CUDA(cudaMemsetAsync(C.sh_x.get(), 0, (full + 32) * sizeof(double), C.stream));
    HM_CUDA(cudaMemsetAsync(C.sh_y.get(), 0, (full + 32) * sizeof(double), C.stream));   // padding stays 0
  }
  C.sh_sol.alloc(L.S + 32);
  HM_CUDA(cudaMemsetAsync(C.sh_sol.get(), 0, (L.S + 32) * sizeof(double), C.stream));
  const bool p2p = p2p_on(C);
  if (p2p) {
    // entries past N of the gathered x stay 0 (the staged x ranges may read one past N);
    // no peer writes there
    p2p_check_capacity(C, L.S);
    HM_CUDA(cudaMemsetAsync(p2p_xfull(C) + C.N, 0, (C.p2p.F - C.N) * sizeof(double), C.stream));
  }
  if (C.solver == 1) cg(C, L, rhs_int + L.off, C.sh_sol.get(), tol, iters, relres);
  else gmres(C, L, rhs_int + L.off, C.sh_sol.get(), tol, iters, relres);
  // the full solution on every rank
  if (p2p) {
    p2p_allgather(C, C.sh_sol.get(), L.n, L.S, /*into_ypart=*/true);
    HM_CUDA(cudaMemcpyAsync(sol_int, p2p_ypart(C), C.N * sizeof(double), cudaMemcpyDeviceToDevice, C.stream));
  } else {
    { KScope ks_(C, KF_COMM);
    HM_NCCL(ncclAllGather(C.sh_sol.get(), C.sh_x.get(), (size_t)L.S, ncclDouble, C.comm, C.stream));
    }
    HM_CUDA(cudaMemcpyAsync(sol_int, C.sh_x.get(), C.N * sizeof(double), cudaMemcpyDeviceToDevice, C.stream));
  }
  HM_CUDA(cudaStreamSynchronize(C.stream));
}

}  // namespace hm
