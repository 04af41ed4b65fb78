// tree.cu — hm_build_tree on the device:
//   a1 panel geometry, a2 Morton codes + stable radix sort, a3 cardinality-based cluster
//   tree + bounding boxes (level-wise), a4 level-wise block-cluster-tree traversal with
//   admissibility (Algorithm 1) and canonical DFS leaf order, plus the leaf partition
//   (A18).
// All floating-point decisions use explicitly rounded intrinsics so that codes, clusters and
// leaf lists are bit-identical to the definition (A4-A10).

#include "entry.cuh"
#include "primitives.cuh"

namespace hm {

namespace {


__global__ void k_geometry(const double* __restrict__ V, const int32_t* __restrict__ T, int64_t N,
                           int64_t nv, double* __restrict__ cen, double* __restrict__ area,
                           double* __restrict__ hh, unsigned int* bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  int32_t a = T[3 * i], b = T[3 * i + 1], c = T[3 * i + 2];
  if (a < 0 || b < 0 || c < 0 || a >= nv || b >= nv || c >= nv) { atomicOr(bad, 1u); return; }
  double v0[3], v1[3], v2[3];
  for (int k = 0; k < 3; ++k) { v0[k] = V[3 * (int64_t)a + k]; v1[k] = V[3 * (int64_t)b + k]; v2[k] = V[3 * (int64_t)c + k]; }
  for (int k = 0; k < 3; ++k) cen[3 * i + k] = ddiv(dadd(dadd(v0[k], v1[k]), v2[k]), 3.0);
  double e01[3], e02[3];
  for (int k = 0; k < 3; ++k) { e01[k] = dsub(v1[k], v0[k]); e02[k] = dsub(v2[k], v0[k]); }
  const double cx = dsub(dmul(e01[1], e02[2]), dmul(e01[2], e02[1]));
  const double cy = dsub(dmul(e01[2], e02[0]), dmul(e01[0], e02[2]));
  const double cz = dsub(dmul(e01[0], e02[1]), dmul(e01[1], e02[0]));
  const double ar = dmul(0.5, __dsqrt_rn(dadd(dadd(dmul(cx, cx), dmul(cy, cy)), dmul(cz, cz))));
  area[i] = ar;
  if (!(ar > 0.0)) atomicOr(bad, 2u);
  const double l0 = edge_length(v0, v1), l1 = edge_length(v1, v2), l2 = edge_length(v2, v0);
  const double m = l0 > l1 ? l0 : l1;
  hh[i] = m > l2 ? m : l2;
}

// Quadrilateral panels (A25): quad i = (q0,q1,q2,q3) -> triangles 2i = (q0,q1,q2), 2i+1 =
// (q0,q2,q3) with the triangle geometry of k_geometry (same operation order); node =
// ((q0 + q1) + (q2 + q3)) * 0.25, |Q| = |T_2i| + |T_2i+1|, h = max(h_2i, h_2i+1).
__global__ void k_geometry_quad(const double* __restrict__ V, const int32_t* __restrict__ Qv, int64_t N,
                                int64_t nv, double* __restrict__ cen, double* __restrict__ area,
                                double* __restrict__ hh, double* __restrict__ tcen, double* __restrict__ tarea,
                                double* __restrict__ th, unsigned int* bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  int32_t id[4];
  for (int r = 0; r < 4; ++r) {
    id[r] = Qv[4 * i + r];
    if (id[r] < 0 || id[r] >= nv) { atomicOr(bad, 1u); return; }
  }
  double q[4][3];
  for (int r = 0; r < 4; ++r)
    for (int k = 0; k < 3; ++k) q[r][k] = V[3 * (int64_t)id[r] + k];
  const int tv[2][3] = {{0, 1, 2}, {0, 2, 3}};
  for (int a = 0; a < 2; ++a) {
    const double* v0 = q[tv[a][0]];
    const double* v1 = q[tv[a][1]];
    const double* v2 = q[tv[a][2]];
    const int64_t t = 2 * i + a;
    for (int k = 0; k < 3; ++k) tcen[3 * t + k] = ddiv(dadd(dadd(v0[k], v1[k]), v2[k]), 3.0);
    double e01[3], e02[3];
    for (int k = 0; k < 3; ++k) { e01[k] = dsub(v1[k], v0[k]); e02[k] = dsub(v2[k], v0[k]); }
    const double cx = dsub(dmul(e01[1], e02[2]), dmul(e01[2], e02[1]));
    const double cy = dsub(dmul(e01[2], e02[0]), dmul(e01[0], e02[2]));
    const double cz = dsub(dmul(e01[0], e02[1]), dmul(e01[1], e02[0]));
    const double ar = dmul(0.5, __dsqrt_rn(dadd(dadd(dmul(cx, cx), dmul(cy, cy)), dmul(cz, cz))));
    tarea[t] = ar;
    if (!(ar > 0.0)) atomicOr(bad, 2u);
    const double l0 = edge_length(v0, v1), l1 = edge_length(v1, v2), l2 = edge_length(v2, v0);
    const double m = l0 > l1 ? l0 : l1;
    th[t] = m > l2 ? m : l2;
  }
  for (int k = 0; k < 3; ++k) cen[3 * i + k] = dmul(dadd(dadd(q[0][k], q[1][k]), dadd(q[2][k], q[3][k])), 0.25);
  area[i] = dadd(tarea[2 * i], tarea[2 * i + 1]);
  hh[i] = th[2 * i] > th[2 * i + 1] ? th[2 * i] : th[2 * i + 1];
}

// global centroid box: per-block partial min/max, then one block finishes
__global__ void k_minmax(const double* __restrict__ cen, int64_t N, double* __restrict__ part) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < 3; ++k) {
      double x = cen[3 * i + k];
      if (x < lo[k]) lo[k] = x;
      if (x > hi[k]) hi[k] = x;
    }
  __shared__ double s[6][256];
  for (int k = 0; k < 3; ++k) { s[k][threadIdx.x] = lo[k]; s[3 + k][threadIdx.x] = hi[k]; }
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int k = 0; k < 3; ++k) {
        double a = s[k][threadIdx.x + w], b = s[3 + k][threadIdx.x + w];
        if (a < s[k][threadIdx.x]) s[k][threadIdx.x] = a;
        if (b > s[3 + k][threadIdx.x]) s[3 + k][threadIdx.x] = b;
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[6 * blockIdx.x + threadIdx.x] = s[threadIdx.x][0];
}

__global__ void k_minmax_final(const double* __restrict__ part, int nb, double* __restrict__ box) {
  if (threadIdx.x >= 6) return;
  int k = threadIdx.x;
  double v = part[k];
  for (int b = 1; b < nb; ++b) {
    double x = part[6 * b + k];
    if (k < 3 ? x < v : x > v) v = x;
  }
  box[k] = v;
}

__device__ __forceinline__ uint64_t quantise(double c, double lo, double hi) {
  if (!(hi > lo)) return 0;
  const double s = dmul(ddiv(dsub(c, lo), dsub(hi, lo)), 2097152.0);
  uint64_t q = (uint64_t)floor(s);
  return q > 2097151ull ? 2097151ull : q;
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {   // 21 bits -> every third bit
  x &= 0x1fffffull;
  x = (x | (x << 32)) & 0x1f00000000ffffull;
  x = (x | (x << 16)) & 0x1f0000ff0000ffull;
  x = (x | (x << 8)) & 0x100f00f00f00f00full;
  x = (x | (x << 4)) & 0x10c30c30c30c30c3ull;
  x = (x | (x << 2)) & 0x1249249249249249ull;
  return x;
}

__global__ void k_morton(const double* __restrict__ cen, int64_t N, const double* __restrict__ box,
                         uint64_t* __restrict__ code, int32_t* __restrict__ idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  uint64_t q[3];
  for (int k = 0; k < 3; ++k) q[k] = quantise(cen[3 * i + k], box[k], box[3 + k]);
  code[i] = (spread3(q[0]) << 2) | (spread3(q[1]) << 1) | spread3(q[2]);
  idx[i] = (int32_t)i;
}

__global__ void k_gather_panels(const double* __restrict__ V, const int32_t* __restrict__ T,
                                const double* __restrict__ cen, const double* __restrict__ area,
                                const double* __restrict__ hh, const int32_t* __restrict__ perm,
                                int64_t N, Panel* __restrict__ P, int32_t* __restrict__ iperm) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= N) return;
  int32_t i = perm[s];
  Panel p;
  for (int r = 0; r < 3; ++r) {
    int32_t vid = T[3 * (int64_t)i + r];
    p.vid[r] = vid;
    for (int k = 0; k < 3; ++k) p.v[3 * r + k] = V[3 * (int64_t)vid + k];
  }
  for (int k = 0; k < 3; ++k) p.c[k] = cen[3 * (int64_t)i + k];
  p.area = area[i];
  p.h = hh[i];
  p.app = i;
  P[s] = p;
  iperm[i] = (int32_t)s;
}

// quads: panel p = 2s + a is triangle a of the quad at internal position s (application
// triangle 2 perm[s] + a); node centroids in internal order for the cluster boxes
__global__ void k_gather_panels_quad(const double* __restrict__ V, const int32_t* __restrict__ Qv,
                                     const double* __restrict__ cen, const double* __restrict__ tcen,
                                     const double* __restrict__ tarea, const double* __restrict__ th,
                                     const double* __restrict__ area, const double* __restrict__ hh,
                                     const int32_t* __restrict__ perm, int64_t N, Panel* __restrict__ P,
                                     int32_t* __restrict__ iperm, Panel* __restrict__ Pn, int4* __restrict__ QV) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= 2 * N) return;
  const int64_t s = p >> 1;
  const int a = (int)(p & 1);
  const int32_t i = perm[s];
  const int tv[2][3] = {{0, 1, 2}, {0, 2, 3}};
  const int64_t t = 2 * (int64_t)i + a;
  Panel pn;
  for (int r = 0; r < 3; ++r) {
    const int32_t vid = Qv[4 * (int64_t)i + tv[a][r]];
    pn.vid[r] = vid;
    for (int k = 0; k < 3; ++k) pn.v[3 * r + k] = V[3 * (int64_t)vid + k];
  }
  for (int k = 0; k < 3; ++k) pn.c[k] = tcen[3 * t + k];
  pn.area = tarea[t];
  pn.h = th[t];
  pn.app = (int32_t)t;
  P[p] = pn;
  if (a == 0) {
    iperm[i] = (int32_t)s;
    const int4 q = reinterpret_cast<const int4*>(Qv)[i];
    QV[s] = q;
    Panel nd;
    const int32_t ids[3] = {q.x, q.y, q.z};
    for (int r = 0; r < 3; ++r) {
      nd.vid[r] = ids[r];
      for (int k = 0; k < 3; ++k) nd.v[3 * r + k] = V[3 * (int64_t)ids[r] + k];
    }
    for (int k = 0; k < 3; ++k) nd.c[k] = cen[3 * (int64_t)i + k];
    nd.area = area[i];
    nd.h = hh[i];
    nd.app = i;
    Pn[s] = nd;
  }
}

// ---- cluster tree (level order): node c at level l splits iff |c| > C_leaf ------------
__global__ void k_split_flags(const int32_t* __restrict__ lo, const int32_t* __restrict__ hi, int64_t b,
                              int64_t e, int leaf, int32_t* __restrict__ flag) {
  int64_t c = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= e) return;
  flag[c - b] = (hi[c] - lo[c]) > leaf ? 1 : 0;
}

__global__ void k_split_emit(int32_t* __restrict__ lo, int32_t* __restrict__ hi, int32_t* __restrict__ child,
                             int32_t* __restrict__ depth, int64_t b, int64_t e, const int32_t* __restrict__ flag,
                             const int32_t* __restrict__ scan, int32_t level) {
  int64_t c = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= e) return;
  if (!flag[c - b]) { child[c] = -1; return; }
  int64_t k = e + 2 * (int64_t)scan[c - b];
  int32_t l = lo[c], h = hi[c], n = h - l;
  int32_t mid = l + (n + 1) / 2;          // |tau_1| = ceil(|tau|/2) (A8)
  child[c] = (int32_t)k;
  lo[k] = l; hi[k] = mid; lo[k + 1] = mid; hi[k + 1] = h;
  depth[k] = depth[k + 1] = level + 1;
}

// boxes bottom-up: leaves from their points, inner nodes from their two children (exact)
// node centroid of internal position s: cb[cstride * s + k] (triangles: the panels' c,
// quads: the node array)
__global__ void k_boxes(const double* __restrict__ cb, int cstride, const int32_t* __restrict__ lo,
                        const int32_t* __restrict__ hi, const int32_t* __restrict__ child, int64_t b, int64_t e,
                        double* __restrict__ box, double* __restrict__ diam2) {
  int64_t c = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= e) return;
  double m[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  if (child[c] < 0) {
    for (int32_t s = lo[c]; s < hi[c]; ++s)
      for (int k = 0; k < 3; ++k) {
        double x = cb[(int64_t)cstride * s + k];
        if (x < m[k]) m[k] = x;
        if (x > m[3 + k]) m[3 + k] = x;
      }
  } else {
    for (int ch = 0; ch < 2; ++ch) {
      const double* cb = box + 6 * (int64_t)(child[c] + ch);
      for (int k = 0; k < 3; ++k) {
        if (cb[k] < m[k]) m[k] = cb[k];
        if (cb[3 + k] > m[3 + k]) m[3 + k] = cb[3 + k];
      }
    }
  }
  for (int k = 0; k < 6; ++k) box[6 * c + k] = m[k];
  const double dx = dsub(m[3], m[0]), dy = dsub(m[4], m[1]), dz = dsub(m[5], m[2]);
  diam2[c] = dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
}

// ---- block cluster tree, one level of Algorithm 1 per launch --------------------------
// adm(t,s) <=> min(D_t, D_s) <= (eta*eta) * G, G = squared box gap (A5)
__device__ __forceinline__ bool admissible(const double* bt, const double* bs, double Dt, double Ds, double eta) {
  double g[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double g1 = dsub(bs[a], bt[3 + a]), g2 = dsub(bt[a], bs[3 + a]);
    const double m = g1 > g2 ? g1 : g2;
    g[a] = m > 0.0 ? m : 0.0;
  }
  const double G = dadd(dadd(dmul(g[0], g[0]), dmul(g[1], g[1])), dmul(g[2], g[2]));
  const double Dmin = Dt < Ds ? Dt : Ds;
  return Dmin <= dmul(dmul(eta, eta), G);
}

__device__ __forceinline__ int64_t warp_aggregated_add(unsigned long long* ctr, int amount, bool pred) {
  unsigned mask = __activemask();
  unsigned take = __ballot_sync(mask, pred);
  int lane = threadIdx.x & 31;
  int leader = __ffs(take) - 1;
  unsigned long long base = 0;
  int cnt = __popc(take) * amount;
  if (take && lane == leader) base = atomicAdd(ctr, (unsigned long long)cnt);
  base = __shfl_sync(mask, base, leader < 0 ? 0 : leader);
  int rank = __popc(take & ((1u << lane) - 1));
  return (int64_t)base + (int64_t)rank * amount;
}

__global__ void k_block_level(const int2* __restrict__ fr, const uint64_t* __restrict__ fkey, int64_t n_in,
                              int level, const int32_t* __restrict__ lo, const int32_t* __restrict__ hi,
                              const int32_t* __restrict__ child, const double* __restrict__ box,
                              const double* __restrict__ diam2, double eta, int leaf,
                              int2* __restrict__ fr_out, uint64_t* __restrict__ fkey_out,
                              Quad* __restrict__ adm, uint64_t* __restrict__ adm_key,
                              Quad* __restrict__ dense, uint64_t* __restrict__ dense_key,
                              unsigned long long* __restrict__ ctr /* [next, adm, dense] */) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool valid = e < n_in;
  int2 ts = valid ? fr[e] : make_int2(0, 0);
  uint64_t key = valid ? fkey[e] : 0;
  int t = ts.x, s = ts.y;
  bool a = false, split = false;
  if (valid) {
    a = admissible(box + 6 * (int64_t)t, box + 6 * (int64_t)s, diam2[t], diam2[s], eta);
    int nt = hi[t] - lo[t], ns = hi[s] - lo[s];
    split = !a && nt > leaf && ns > leaf;
  }
  int64_t pos = warp_aggregated_add(&ctr[0], 4, valid && split);
  if (valid && split) {
    int shift = 64 - 2 * (level + 1);
    int t0 = child[t], s0 = child[s];
    for (int c = 0; c < 4; ++c) {
      fr_out[pos + c] = make_int2(t0 + (c >> 1), s0 + (c & 1));
      fkey_out[pos + c] = key | ((uint64_t)c << shift);
    }
  }
  int64_t pa = warp_aggregated_add(&ctr[1], 1, valid && !split && a);
  if (valid && !split && a) {
    adm[pa] = Quad{lo[t], hi[t], lo[s], hi[s]};
    adm_key[pa] = key;
  }
  int64_t pd = warp_aggregated_add(&ctr[2], 1, valid && !split && !a);
  if (valid && !split && !a) {
    dense[pd] = Quad{lo[t], hi[t], lo[s], hi[s]};
    dense_key[pd] = key;
  }
}

// Per-leaf setup cost for the partition (A18).  model 0 (round 1): dense |t||s|, admissible
// (|t|+|s|) 10.  model 1 (default): the evaluations the leaf will cost —
//   dense: |t||s| x (mean rule evaluations per entry of its kind, measured at C4 on 400
//          leaves each: diagonal t = s 1542, boxes touching 360, separated 140 -> weights
//          110 / 26 / 10; boxes over the node centroids, the same boxes as admissibility)
//   admissible: (|t|+|s|) x 10 k^, k^ = 8.2 + 0.3 log2((|t|+|s|)/40): the mean ACA rank at
//          eps 1e-6 grows slowly with the block size (sampled at C3: 8.2 at m+n = 40 ... 10.0 at
//          ~5900)
// model 2: the dense weights of model 1, admissible (|t|+|s| + 21) x 10: a fixed per-block
//          cost (the per-step pivot / update / bookkeeping of a block, fitted on the one-GPU
//          emulation of 4- and 8-rank partitions at C4, profiles/r02_partition_emulate_c4.jsonl:
//          per rank ~21.7 us per block vs 1.0 us per unit of m + n)
__global__ void k_leaf_cost(const Quad* __restrict__ q, int64_t n, int kind, int model, const double* __restrict__ cen,
                            int cstride, int64_t* __restrict__ cost) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= n) return;
  const Quad Q = q[b];
  const int64_t m = Q.rhi - Q.rlo, nn = Q.chi - Q.clo;
  if (model == 0) { cost[b] = kind == 1 ? m * nn : (m + nn) * 10; return; }
  if (kind == 0) {
    if (model == 2) { cost[b] = (m + nn + 21) * 10; return; }
    const double kh = 8.2 + 0.3 * log2((double)(m + nn) / 40.0);
    cost[b] = (m + nn) * (int64_t)llrint(10.0 * fmax(kh, 7.0));
    return;
  }
  int64_t w = 10;
  if (Q.rlo == Q.clo && Q.rhi == Q.chi) {
    w = 110;
  } else {
    double bt[6], bs[6];
    for (int a = 0; a < 3; ++a) { bt[a] = bs[a] = 1e300; bt[3 + a] = bs[3 + a] = -1e300; }
    for (int s = Q.rlo; s < Q.rhi; ++s)
      for (int a = 0; a < 3; ++a) { const double c = cen[(int64_t)s * cstride + a]; bt[a] = fmin(bt[a], c); bt[3 + a] = fmax(bt[3 + a], c); }
    for (int s = Q.clo; s < Q.chi; ++s)
      for (int a = 0; a < 3; ++a) { const double c = cen[(int64_t)s * cstride + a]; bs[a] = fmin(bs[a], c); bs[3 + a] = fmax(bs[3 + a], c); }
    bool touch = true;
    for (int a = 0; a < 3; ++a) touch &= bs[a] <= bt[3 + a] && bt[a] <= bs[3 + a];
    if (touch) w = 26;
  }
  cost[b] = m * nn * w;
}

void grow_copy(DBuf<Quad>& q, DBuf<uint64_t>& k, int64_t used, int64_t need, cudaStream_t st) {
  if ((int64_t)q.n >= need) return;
  int64_t cap = std::max<int64_t>(need, 2 * (int64_t)q.n);
  Quad* nq = nullptr;
  uint64_t* nk = nullptr;
  HM_CUDA(cudaMalloc(&nq, cap * sizeof(Quad) + 16));
  HM_CUDA(cudaMalloc(&nk, cap * sizeof(uint64_t) + 16));
  if (used > 0) {
    HM_CUDA(cudaMemcpyAsync(nq, q.p, used * sizeof(Quad), cudaMemcpyDeviceToDevice, st));
    HM_CUDA(cudaMemcpyAsync(nk, k.p, used * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  }
  HM_CUDA(cudaStreamSynchronize(st));
  q.release(); k.release();
  q.p = nq; q.n = cap; k.p = nk; k.n = cap;
}

// first leaf whose exclusive cost prefix is >= bound[b] (lower_bound on the non-decreasing
// prefix), for the two bounds of this rank; out preset to n
__global__ void k_prefix_bounds(const int64_t* __restrict__ pref, int64_t n, const int64_t* __restrict__ bound,
                                unsigned long long* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int b = 0; b < 2; ++b)
    if (pref[i] >= bound[b] && (i == 0 || pref[i - 1] < bound[b])) atomicMin(&out[b], (unsigned long long)i);
}

void partition_list(Context& C, const DBuf<Quad>& q, int64_t n, int kind, int64_t& begin, int64_t& end,
                    DBuf<char>& tmp) {
  // diagnostic options part_ranks / part_rank (one process, world 1): take rank r's share of a
  // p-way partition, to measure every rank's setup of a p-GPU run one after the other on one GPU
  const int P = C.world > 1 ? C.world : C.part_ranks, R = C.world > 1 ? C.rank : C.part_rank;
  if (P <= 1 || n == 0) { begin = 0; end = n; return; }
  DBuf<int64_t>& cost = C.tws.cost; DBuf<int64_t>& pref = C.tws.pref;
  cost.alloc(n); pref.alloc(n);
  const Panel* nodes = C.quad ? C.qnode.get() : C.panel.get();
  const double* cen = reinterpret_cast<const double*>(reinterpret_cast<const char*>(nodes) + offsetof(Panel, c));
  k_leaf_cost<<<grid_for(n, 256), 256, 0, C.stream>>>(q.get(), n, kind, C.cost_model, cen,
                                                       (int)(sizeof(Panel) / sizeof(double)), cost.get());
  HM_CHECK_LAUNCH();
  prim::exclusive_scan<int64_t>(cost.get(), pref.get(), n, tmp, C.stream);
  int64_t h[2];
  HM_CUDA(cudaMemcpyAsync(&h[0], pref.get() + (n - 1), sizeof(int64_t), cudaMemcpyDeviceToHost, C.stream));
  HM_CUDA(cudaMemcpyAsync(&h[1], cost.get() + (n - 1), sizeof(int64_t), cudaMemcpyDeviceToHost, C.stream));
  HM_CUDA(cudaStreamSynchronize(C.stream));
  const int64_t total = h[0] + h[1];
  auto bound_of = [&](int r) -> int64_t { return (int64_t)(((__int128)r * total) / P); };
  // rank r owns the leaves whose exclusive prefix lies in [floor(rC/p), floor((r+1)C/p)) (A18)
  int64_t hb[2] = {bound_of(R), bound_of(R + 1)};
  unsigned long long ho[2] = {(unsigned long long)n, (unsigned long long)n};
  C.tws.bounds.alloc(2);
  C.tws.bout.alloc(2);
  HM_CUDA(cudaMemcpyAsync(C.tws.bounds.get(), hb, sizeof(hb), cudaMemcpyHostToDevice, C.stream));
  HM_CUDA(cudaMemcpyAsync(C.tws.bout.get(), ho, sizeof(ho), cudaMemcpyHostToDevice, C.stream));
  k_prefix_bounds<<<grid_for(n, 256), 256, 0, C.stream>>>(pref.get(), n, C.tws.bounds.get(), C.tws.bout.get());
  HM_CHECK_LAUNCH();
  HM_CUDA(cudaMemcpyAsync(ho, C.tws.bout.get(), sizeof(ho), cudaMemcpyDeviceToHost, C.stream));
  HM_CUDA(cudaStreamSynchronize(C.stream));
  begin = R == 0 ? 0 : (int64_t)ho[0];
  end = R + 1 >= P ? n : (int64_t)ho[1];
}

}  // namespace

void build_tree(Context& C, const hm_mesh& mesh, int leaf_size, double eta) {
  plan_dense_abort(C);   // a planner thread of a failed hm_setup must not see the new tree
  cudaStream_t st = C.stream;
  cudaEvent_t ev[7];
  for (auto& e : ev) HM_CUDA(cudaEventCreate(&e));
  HM_CUDA(cudaEventRecord(ev[0], st));
  const int64_t N = mesh.n_triangles, nv = mesh.n_vertices;
  C.have_tree = C.have_setup = false;
  C.N = N; C.nv = nv; C.leaf_size = leaf_size; C.eta = eta;
  upload_quadrature_tables();
  // ---- a1: mesh upload + panel geometry
  C.vert.alloc(nv * 3);
  C.quad = mesh.panel_vertices == 4;
  const int pv = C.quad ? 4 : 3;
  C.npanel = C.quad ? 2 * N : N;
  C.tri.alloc(N * pv);
  cudaMemcpyKind kind = mesh.memory ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  HM_CUDA(cudaMemcpyAsync(C.vert.get(), mesh.vertices, nv * 3 * sizeof(double), kind, st));
  HM_CUDA(cudaMemcpyAsync(C.tri.get(), mesh.triangles, N * pv * sizeof(int32_t), kind, st));
  TreeWs& ws = C.tws;
  DBuf<double>& cen = ws.cen; DBuf<double>& area = ws.area; DBuf<double>& hh = ws.hh;
  cen.alloc(N * 3); area.alloc(N); hh.alloc(N);
  DBuf<unsigned int>& bad = ws.bad;
  bad.alloc(1);
  HM_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(unsigned int), st));
  if (C.quad) {
    ws.tcen.alloc(2 * N * 3); ws.tarea.alloc(2 * N); ws.th.alloc(2 * N);
    k_geometry_quad<<<grid_for(N, 256), 256, 0, st>>>(C.vert.get(), C.tri.get(), N, nv, cen.get(), area.get(),
                                                        hh.get(), ws.tcen.get(), ws.tarea.get(), ws.th.get(),
                                                        bad.get());
  } else {
    k_geometry<<<grid_for(N, 256), 256, 0, st>>>(C.vert.get(), C.tri.get(), N, nv, cen.get(), area.get(),
                                                   hh.get(), bad.get());
  }
  HM_CHECK_LAUNCH();
  unsigned int hbad = 0;
  HM_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
  HM_CUDA(cudaEventRecord(ev[1], st));
  // ---- a2: Morton codes + stable sort
  const int nb = 148;
  DBuf<double>& part = ws.part; DBuf<double>& gbox = ws.gbox;
  part.alloc(6 * nb); gbox.alloc(6);
  k_minmax<<<nb, 256, 0, st>>>(cen.get(), N, part.get());
  k_minmax_final<<<1, 32, 0, st>>>(part.get(), nb, gbox.get());
  HM_CHECK_LAUNCH();
  HM_CUDA(cudaStreamSynchronize(st));
  if (hbad & 1u) fail(HM_ERR_ARG, "hm_build_tree: a panel references a vertex id out of range");
  if (hbad & 2u) fail(HM_ERR_ARG, "hm_build_tree: a panel (or half of a quad) has zero area (degenerate)");
  DBuf<uint64_t>& code_sorted = ws.code_sorted;
  DBuf<int32_t>& idx = ws.idx;
  C.codes_app.alloc(N);
  code_sorted.alloc(N); idx.alloc(N);
  C.perm.alloc(N); C.iperm.alloc(N);
  k_morton<<<grid_for(N, 256), 256, 0, st>>>(cen.get(), N, gbox.get(), C.codes_app.get(), idx.get());
  HM_CHECK_LAUNCH();
  DBuf<char>& tmp = ws.tmp;
  // LSD radix sort: stable, ties keep ascending index (A7)
  prim::radix_sort_pairs<uint64_t, int32_t>(C.codes_app.get(), code_sorted.get(), idx.get(), C.perm.get(), N, 0, 63,
                                            tmp, st);
  C.panel.alloc(C.npanel);
  if (C.quad) {
    C.qnode.alloc(N);
    C.qv.alloc(N);
    k_gather_panels_quad<<<grid_for(2 * N, 256), 256, 0, st>>>(C.vert.get(), C.tri.get(), cen.get(), ws.tcen.get(),
                                                                 ws.tarea.get(), ws.th.get(), area.get(), hh.get(),
                                                                 C.perm.get(), N, C.panel.get(), C.iperm.get(),
                                                                 C.qnode.get(), C.qv.get());
  } else {
    k_gather_panels<<<grid_for(N, 256), 256, 0, st>>>(C.vert.get(), C.tri.get(), cen.get(), area.get(), hh.get(),
                                                       C.perm.get(), N, C.panel.get(), C.iperm.get());
  }
  HM_CHECK_LAUNCH();
  HM_CUDA(cudaEventRecord(ev[2], st));
  // ---- a3: cluster tree, level order
  int64_t leaf_min = std::max<int64_t>(1, (leaf_size + 1) / 2);
  int64_t cap = 2 * (N / leaf_min + 2) + 4;
  C.cl_lo.alloc(cap); C.cl_hi.alloc(cap); C.cl_child.alloc(cap); C.cl_depth.alloc(cap);
  int32_t root[2] = {0, (int32_t)N}, zero = 0;
  HM_CUDA(cudaMemcpyAsync(C.cl_lo.get(), &root[0], sizeof(int32_t), cudaMemcpyHostToDevice, st));
  HM_CUDA(cudaMemcpyAsync(C.cl_hi.get(), &root[1], sizeof(int32_t), cudaMemcpyHostToDevice, st));
  HM_CUDA(cudaMemcpyAsync(C.cl_depth.get(), &zero, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  std::vector<int64_t> lev = {0, 1};
  DBuf<int32_t>& flag = ws.flag; DBuf<int32_t>& scan = ws.scan;
  flag.alloc(cap); scan.alloc(cap);
  for (int level = 0;; ++level) {
    int64_t b = lev[level], e = lev[level + 1], n = e - b;
    k_split_flags<<<grid_for(n, 256), 256, 0, st>>>(C.cl_lo.get(), C.cl_hi.get(), b, e, leaf_size, flag.get());
    HM_CHECK_LAUNCH();
    prim::exclusive_scan<int32_t>(flag.get(), scan.get(), n, tmp, st);
    k_split_emit<<<grid_for(n, 256), 256, 0, st>>>(C.cl_lo.get(), C.cl_hi.get(), C.cl_child.get(),
                                                    C.cl_depth.get(), b, e, flag.get(), scan.get(), level);
    HM_CHECK_LAUNCH();
    int32_t hs[2];
    HM_CUDA(cudaMemcpyAsync(&hs[0], scan.get() + (n - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HM_CUDA(cudaMemcpyAsync(&hs[1], flag.get() + (n - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HM_CUDA(cudaStreamSynchronize(st));
    int64_t nsplit = hs[0] + hs[1];
    if (nsplit == 0) break;
    if (e + 2 * nsplit > cap) fail(HM_ERR_CUDA, "cluster tree capacity exceeded");
    lev.push_back(e + 2 * nsplit);
  }
  C.ncl = lev.back();
  int nlev = (int)lev.size() - 1;
  C.cl_box.alloc(6 * C.ncl); C.cl_diam2.alloc(C.ncl);
  for (int level = nlev - 1; level >= 0; --level) {
    int64_t b = lev[level], e = lev[level + 1];
    const Panel* nodes = C.quad ? C.qnode.get() : C.panel.get();
    const double* cb = reinterpret_cast<const double*>(reinterpret_cast<const char*>(nodes) + offsetof(Panel, c));
    const int cstride = (int)(sizeof(Panel) / sizeof(double));
    k_boxes<<<grid_for(e - b, 128), 128, 0, st>>>(cb, cstride, C.cl_lo.get(), C.cl_hi.get(), C.cl_child.get(),
                                                   b, e, C.cl_box.get(), C.cl_diam2.get());
    HM_CHECK_LAUNCH();
  }
  HM_CUDA(cudaEventRecord(ev[3], st));
  // ---- a4: block cluster tree, level-wise
  DBuf<int2>* fr = ws.fr;
  DBuf<uint64_t>* fk = ws.fk;
  fr[0].alloc(1024); fk[0].alloc(1024);
  int2 r2 = make_int2(0, 0);
  uint64_t k0 = 0;
  HM_CUDA(cudaMemcpyAsync(fr[0].get(), &r2, sizeof(int2), cudaMemcpyHostToDevice, st));
  HM_CUDA(cudaMemcpyAsync(fk[0].get(), &k0, sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  DBuf<Quad>& admq = ws.admq; DBuf<Quad>& denq = ws.denq;
  DBuf<uint64_t>& admk = ws.admk; DBuf<uint64_t>& denk = ws.denk;
  DBuf<unsigned long long>& ctr = ws.ctr;
  ctr.alloc(3);
  int64_t n_in = 1, nadm = 0, nden = 0;
  int cur = 0;
  for (int level = 0; n_in > 0; ++level) {
    fr[1 - cur].alloc(4 * n_in); fk[1 - cur].alloc(4 * n_in);
    grow_copy(admq, admk, nadm, nadm + n_in, st);
    grow_copy(denq, denk, nden, nden + n_in, st);
    unsigned long long hc[3] = {0, (unsigned long long)nadm, (unsigned long long)nden};
    HM_CUDA(cudaMemcpyAsync(ctr.get(), hc, sizeof(hc), cudaMemcpyHostToDevice, st));
    k_block_level<<<grid_for(n_in, 256), 256, 0, st>>>(
        fr[cur].get(), fk[cur].get(), n_in, level, C.cl_lo.get(), C.cl_hi.get(), C.cl_child.get(), C.cl_box.get(),
        C.cl_diam2.get(), eta, leaf_size, fr[1 - cur].get(), fk[1 - cur].get(), admq.get(), admk.get(),
        denq.get(), denk.get(), ctr.get());
    HM_CHECK_LAUNCH();
    HM_CUDA(cudaMemcpyAsync(hc, ctr.get(), sizeof(hc), cudaMemcpyDeviceToHost, st));
    HM_CUDA(cudaStreamSynchronize(st));
    n_in = (int64_t)hc[0]; nadm = (int64_t)hc[1]; nden = (int64_t)hc[2];
    cur = 1 - cur;
    if (level > 62) fail(HM_ERR_ARG, "block tree deeper than 31 levels");
  }
  HM_CUDA(cudaEventRecord(ev[4], st));
  // canonical DFS order = ascending left-aligned path key (A10)
  C.nadm = nadm; C.ndense = nden;
  C.adm.alloc(nadm); C.dense.alloc(nden);
  DBuf<uint64_t>& ksorted = ws.ksorted;
  ksorted.alloc(std::max(nadm, nden));
  if (nadm) prim::radix_sort_pairs<uint64_t, Quad>(admk.get(), ksorted.get(), admq.get(), C.adm.get(), nadm, 0, 64, tmp, st);
  if (nden) prim::radix_sort_pairs<uint64_t, Quad>(denk.get(), ksorted.get(), denq.get(), C.dense.get(), nden, 0, 64, tmp, st);
  HM_CUDA(cudaEventRecord(ev[5], st));
  // ---- leaf partition over ranks (A18)
  partition_list(C, C.adm, nadm, 0, C.adm_begin, C.adm_end, tmp);
  partition_list(C, C.dense, nden, 1, C.dense_begin, C.dense_end, tmp);
  HM_CUDA(cudaEventRecord(ev[6], st));
  HM_CUDA(cudaStreamSynchronize(st));
  for (int k = 0; k < 6; ++k) {
    float ms = 0;
    HM_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
    C.times.tree_phase_ms[k] = ms;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  C.h_adm.clear(); C.h_dense.clear();
  C.have_tree = true;
}

}  // namespace hm
