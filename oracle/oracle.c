/*
 * oracle.c — plain, slow CPU oracle of the H-matrix BEM hot path of
 * Harbrecht & Zaspel, arXiv 1806.11558.  TEST INFRASTRUCTURE ONLY (see oracle.h):
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference legs
 * may load it; the product path never does.  It shares no code with the CUDA path.
 *
 * Structure follows the paper's definitions, in the paper's order:
 *   geometry      P:200-211, P:641-642 (nodes = element centres)
 *   Morton + sort P:400-411, S:118-126 (A6, A7)
 *   CBC tree      P:268-280, S:131 (A8)             recursion
 *   bbox / adm    P:256-266 (A4, A5)
 *   Alg. 1        P:283-306 (A9, A10)               recursion, DFS order
 *   entries a_ij  P:224-228 read per A1, rules A14, arithmetic A15
 *   ACA           P:318-321, A11-A12     one block at a time
 *   H-matvec      P:328-332                         loop over leaves
 *   CG / GMRES    P:646, A17
 *   partition     P:563-568, A18
 *   RHS           P:230-231, A16
 *   potential     P:176-177, A23           direct sum over panels
 *   fixed rank    P:776, A24 (ACA with eps = 0)
 *   quad panels   P:700, A25 (parallelograms: tensor Gauss when separated,
 *                 the two-triangle split when touching)
 *
 * Pins (tests/test_oracle_*.py, all -m "not gpu"):
 *   Morton/sort/CBC   SPEC worked examples S:124-126; invariants (C1)-(C4)
 *   bbox/adm          S:144-146, S:205-207 worked examples
 *   block tree        brute-force N x N tiling; adm/dense invariants; N<=C_leaf; eta=0
 *   Gauss-Legendre    50-digit decimal Newton in the test (independent)
 *   regular rule      far-field asymptotics; analytic triangle potential + outer quadrature
 *   self term         semi-analytic (analytic inner potential, subdivided outer Gauss)
 *   Sauter-Schwab     exact monomial integrals over T^xT^ (measure preservation),
 *                     identical map vs closed form, edge/vertex vs semi-analytic
 *   all entries       unit-sphere row sums (V1 = 1), symmetry, SPD (Cholesky)
 *   ACA               exact rank-r matrices; zero block; interpolation property
 *   matvec            eta = 0 / N = 320 -> H = A exactly; ||Hx-Ax|| <= 10 eps vs dense
 *   solvers           identity/diag cases; V u = 1 on the sphere -> u ~ 1; vs Cholesky
 *   partition         union/disjoint/bound invariants
 *   fixed-rank ACA    exactly K terms, interpolation at the pivots, error decreasing in K
 *   potential         closed-form triangle potential per band; sphere interior u = 1 / u = f
 *   quad panels       unit-square self integral (closed form); square pairs vs the exact
 *                     rectangle potential + graded outer rule; exact f integrals; cube
 *                     interior u = f at the paper's convergence rate N^-1.3
 * No function here is "parity unpinned".
 */
#include "oracle.h"

#include <float.h>
#include <quadmath.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define INV4PI 0.07957747154594767 /* 1/(4 pi), correctly rounded binary64 */
#define NQ_SINGULAR 6              /* Gauss points per coordinate, Sauter-Schwab (A14) */

/* ------------------------------------------------------------------ */
/* problem state                                                       */
/* ------------------------------------------------------------------ */
typedef struct {
  int32_t lo, hi, child0, child1, depth;
  double box[6];
} cluster_t;

typedef struct {
  int32_t rlo, rhi, clo, chi;
} quad_t;

struct or_problem {
  int64_t N, nv;
  double* V;          /* nv*3 */
  int32_t* T;         /* N*3  */
  double* cen;        /* N*3, application order */
  double* area;       /* N */
  double* h;          /* N */
  uint64_t* code;     /* N, application order */
  int32_t* perm;      /* internal -> application */
  int leaf_size;
  double eta;
  cluster_t* cl;
  int64_t ncl, capcl;
  quad_t* adm;
  int64_t nadm, capadm;
  quad_t* dense;
  int64_t ndense, capdense;
  /* assembled H */
  double** dblk;      /* per dense leaf, row-major, NULL if not owned */
  double** U;         /* per adm leaf, m x k col-major */
  double** Vf;        /* per adm leaf, n x k col-major */
  int32_t** piv;      /* per adm leaf, 2k */
  int* rank;          /* per adm leaf, -1 if not owned */
  double counters[4];
  /* quadrilateral meshes (A25): Q = N*4 vertex ids; tri = the split triangle problem
   * (2N triangles, quad i -> triangles 2i = (q0,q1,q2) and 2i+1 = (q0,q2,q3)) that
   * evaluates the entries, right-hand side and potential; NULL for triangle meshes */
  int32_t* Q;
  or_problem* tri;
};

/* ------------------------------------------------------------------ */
/* geometry                                     */
/* ------------------------------------------------------------------ */
static double edge_len(const double* a, const double* b) {
  double dx = b[0] - a[0], dy = b[1] - a[1], dz = b[2] - a[2];
  return sqrt((dx * dx + dy * dy) + dz * dz);
}

static void panel_geometry(const double* v0, const double* v1, const double* v2,
                           double* c, double* area, double* h) {
  for (int a = 0; a < 3; ++a) c[a] = ((v0[a] + v1[a]) + v2[a]) / 3.0;
  double e01[3], e02[3];
  for (int a = 0; a < 3; ++a) { e01[a] = v1[a] - v0[a]; e02[a] = v2[a] - v0[a]; }
  double cx = e01[1] * e02[2] - e01[2] * e02[1];
  double cy = e01[2] * e02[0] - e01[0] * e02[2];
  double cz = e01[0] * e02[1] - e01[1] * e02[0];
  *area = 0.5 * sqrt((cx * cx + cy * cy) + cz * cz);
  double l0 = edge_len(v0, v1), l1 = edge_len(v1, v2), l2 = edge_len(v2, v0);
  double m = l0 > l1 ? l0 : l1;
  *h = m > l2 ? m : l2;
}

static const double* vtx(const or_problem* P, int64_t tri, int k) {
  return P->V + 3 * (int64_t)P->T[3 * tri + k];
}

/* ------------------------------------------------------------------ */
/* Morton code (A6)                              */
/* ------------------------------------------------------------------ */
static uint64_t quantise(double c, double lo, double hi) {
  if (!(hi > lo)) return 0;
  double s = ((c - lo) / (hi - lo)) * 2097152.0;
  double f = floor(s);
  uint64_t q = (uint64_t)f;
  return q > 2097151u ? 2097151u : q;
}

static uint64_t interleave3(uint64_t qx, uint64_t qy, uint64_t qz) {
  uint64_t code = 0;
  for (int b = 20; b >= 0; --b) {
    code |= ((qx >> b) & 1u) << (3 * b + 2);
    code |= ((qy >> b) & 1u) << (3 * b + 1);
    code |= ((qz >> b) & 1u) << (3 * b);
  }
  return code;
}

/* stable sort by code: merge sort on (code, index) (A7) */
static void merge_sort(int32_t* idx, int32_t* tmp, const uint64_t* key, int64_t n) {
  if (n < 2) return;
  int64_t h = n / 2;
  merge_sort(idx, tmp, key, h);
  merge_sort(idx + h, tmp, key, n - h);
  int64_t a = 0, b = h, o = 0;
  while (a < h && b < n) {
    if (key[idx[b]] < key[idx[a]]) tmp[o++] = idx[b++];
    else tmp[o++] = idx[a++];
  }
  while (a < h) tmp[o++] = idx[a++];
  while (b < n) tmp[o++] = idx[b++];
  memcpy(idx, tmp, (size_t)n * sizeof(int32_t));
}

/* ------------------------------------------------------------------ */
/* cluster tree: cardinality-based clustering (A8)           */
/* ------------------------------------------------------------------ */
static int32_t build_cluster(or_problem* P, int32_t lo, int32_t hi, int32_t depth) {
  if (P->ncl == P->capcl) {
    P->capcl = P->capcl ? 2 * P->capcl : 64;
    P->cl = (cluster_t*)realloc(P->cl, (size_t)P->capcl * sizeof(cluster_t));
  }
  int32_t id = (int32_t)P->ncl++;
  cluster_t* c = &P->cl[id];
  c->lo = lo; c->hi = hi; c->depth = depth; c->child0 = -1; c->child1 = -1;
  /* Q_tau = prod [min, max] of node coordinates */
  for (int a = 0; a < 3; ++a) { c->box[a] = INFINITY; c->box[3 + a] = -INFINITY; }
  for (int32_t s = lo; s < hi; ++s) {
    const double* x = P->cen + 3 * (int64_t)P->perm[s];
    for (int a = 0; a < 3; ++a) {
      if (x[a] < c->box[a]) c->box[a] = x[a];
      if (x[a] > c->box[3 + a]) c->box[3 + a] = x[a];
    }
  }
  int32_t n = hi - lo;
  if (n > P->leaf_size) {                        /* (C3): leaf iff |tau| <= C_leaf */
    int32_t mid = lo + (n + 1) / 2;              /* |tau_1| = ceil(|tau|/2) */
    int32_t c0 = build_cluster(P, lo, mid, depth + 1);
    int32_t c1 = build_cluster(P, mid, hi, depth + 1);
    P->cl[id].child0 = c0;
    P->cl[id].child1 = c1;
  }
  return id;
}

/* ------------------------------------------------------------------ */
/* admissibility, squared form of, reading A4/A5            */
/* ------------------------------------------------------------------ */
int or_admissible(const double* bt, const double* bs, double eta) {
  double dx = bt[3] - bt[0], dy = bt[4] - bt[1], dz = bt[5] - bt[2];
  double Dt = (dx * dx + dy * dy) + dz * dz;
  dx = bs[3] - bs[0]; dy = bs[4] - bs[1]; dz = bs[5] - bs[2];
  double Ds = (dx * dx + dy * dy) + dz * dz;
  double g[3];
  for (int a = 0; a < 3; ++a) {
    double g1 = bs[a] - bt[3 + a], g2 = bt[a] - bs[3 + a];
    double m = g1 > g2 ? g1 : g2;
    g[a] = m > 0.0 ? m : 0.0;
  }
  double G = (g[0] * g[0] + g[1] * g[1]) + g[2] * g[2];
  double Dmin = Dt < Ds ? Dt : Ds;
  return Dmin <= (eta * eta) * G;
}

static void push_leaf(quad_t** arr, int64_t* n, int64_t* cap, const cluster_t* t, const cluster_t* s) {
  if (*n == *cap) {
    *cap = *cap ? 2 * *cap : 256;
    *arr = (quad_t*)realloc(*arr, (size_t)*cap * sizeof(quad_t));
  }
  quad_t q = {t->lo, t->hi, s->lo, s->hi};
  (*arr)[(*n)++] = q;
}

/* Algorithm 1 build_block_cluster_tree; leaves emitted in DFS
 * pre-order with children (t1s1, t1s2, t2s1, t2s2) (A10). */
static void build_block(or_problem* P, int32_t t, int32_t s) {
  const cluster_t* ct = &P->cl[t];
  const cluster_t* cs = &P->cl[s];
  int adm = or_admissible(ct->box, cs->box, P->eta);
  int nt = ct->hi - ct->lo, ns = cs->hi - cs->lo;
  if (!adm && nt > P->leaf_size && ns > P->leaf_size) {
    int32_t tc[2] = {ct->child0, ct->child1};
    int32_t sc[2] = {cs->child0, cs->child1};
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) build_block(P, tc[a], sc[b]);
  } else if (adm) {
    push_leaf(&P->adm, &P->nadm, &P->capadm, ct, cs);
  } else {
    push_leaf(&P->dense, &P->ndense, &P->capdense, ct, cs);
  }
}

static or_problem* alloc_problem(const double* V, int64_t n_v, int64_t N, int leaf_size, double eta) {
  or_problem* P = (or_problem*)calloc(1, sizeof(or_problem));
  P->N = N; P->nv = n_v; P->leaf_size = leaf_size; P->eta = eta;
  P->V = (double*)malloc((size_t)(n_v > 0 ? n_v : 1) * 3 * sizeof(double));
  memcpy(P->V, V, (size_t)n_v * 3 * sizeof(double));
  P->cen = (double*)malloc((size_t)(N > 0 ? N : 1) * 3 * sizeof(double));
  P->area = (double*)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
  P->h = (double*)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
  P->code = (uint64_t*)malloc((size_t)(N > 0 ? N : 1) * sizeof(uint64_t));
  P->perm = (int32_t*)malloc((size_t)(N > 0 ? N : 1) * sizeof(int32_t));
  return P;
}

static void order_and_trees(or_problem* P, int build_trees);

or_problem* or_create(const double* V, int64_t n_v, const int32_t* T, int64_t N,
                      int leaf_size, double eta) {
  or_problem* P = alloc_problem(V, n_v, N, leaf_size, eta);
  P->T = (int32_t*)malloc((size_t)(N > 0 ? N : 1) * 3 * sizeof(int32_t));
  if (N > 0) memcpy(P->T, T, (size_t)N * 3 * sizeof(int32_t));
  for (int64_t i = 0; i < N; ++i)
    panel_geometry(vtx(P, i, 0), vtx(P, i, 1), vtx(P, i, 2), P->cen + 3 * i, P->area + i, P->h + i);
  order_and_trees(P, 1);
  return P;
}

/* Quadrilateral panels (A25; the paper's model case): each quad
 * (q0,q1,q2,q3), vertices in cyclic order, is the union of the triangles (q0,q1,q2) and
 * (q0,q2,q3).  Node = the vertex average ((q0 + q1) + (q2 + q3)) * 0.25,
 * |Q_i| = |T_2i| + |T_2i+1|, h_i = max(h_2i, h_2i+1).  The piecewise-constant basis
 * function of Q_i is the sum of those of its two triangles, so every Galerkin integral over
 * Q_i x Q_j is the sum of the four triangle-pair integrals. */
or_problem* or_create_quads(const double* V, int64_t n_v, const int32_t* Qv, int64_t N,
                            int leaf_size, double eta) {
  or_problem* P = alloc_problem(V, n_v, N, leaf_size, eta);
  P->Q = (int32_t*)malloc((size_t)(N > 0 ? N : 1) * 4 * sizeof(int32_t));
  if (N > 0) memcpy(P->Q, Qv, (size_t)N * 4 * sizeof(int32_t));
  int32_t* T2 = (int32_t*)malloc((size_t)(N > 0 ? N : 1) * 6 * sizeof(int32_t));
  for (int64_t i = 0; i < N; ++i) {
    const int32_t* q = Qv + 4 * i;
    T2[6 * i + 0] = q[0]; T2[6 * i + 1] = q[1]; T2[6 * i + 2] = q[2];
    T2[6 * i + 3] = q[0]; T2[6 * i + 4] = q[2]; T2[6 * i + 5] = q[3];
  }
  P->tri = alloc_problem(V, n_v, 2 * N, leaf_size, eta);
  P->tri->T = T2;
  for (int64_t t = 0; t < 2 * N; ++t)
    panel_geometry(vtx(P->tri, t, 0), vtx(P->tri, t, 1), vtx(P->tri, t, 2), P->tri->cen + 3 * t,
                   P->tri->area + t, P->tri->h + t);
  order_and_trees(P->tri, 0);
  for (int64_t i = 0; i < N; ++i) {
    const double *a = P->V + 3 * (int64_t)Qv[4 * i], *b = P->V + 3 * (int64_t)Qv[4 * i + 1];
    const double *c = P->V + 3 * (int64_t)Qv[4 * i + 2], *d = P->V + 3 * (int64_t)Qv[4 * i + 3];
    for (int k = 0; k < 3; ++k) P->cen[3 * i + k] = ((a[k] + b[k]) + (c[k] + d[k])) * 0.25;
    P->area[i] = P->tri->area[2 * i] + P->tri->area[2 * i + 1];
    P->h[i] = P->tri->h[2 * i] > P->tri->h[2 * i + 1] ? P->tri->h[2 * i] : P->tri->h[2 * i + 1];
  }
  order_and_trees(P, 1);
  return P;
}

static void order_and_trees(or_problem* P, int build_trees) {
  const int64_t N = P->N;
  /* global centroid bounding box and Morton codes */
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < N; ++i)
    for (int a = 0; a < 3; ++a) {
      if (P->cen[3 * i + a] < lo[a]) lo[a] = P->cen[3 * i + a];
      if (P->cen[3 * i + a] > hi[a]) hi[a] = P->cen[3 * i + a];
    }
  for (int64_t i = 0; i < N; ++i) {
    const double* c = P->cen + 3 * i;
    P->code[i] = interleave3(quantise(c[0], lo[0], hi[0]), quantise(c[1], lo[1], hi[1]),
                             quantise(c[2], lo[2], hi[2]));
    P->perm[i] = (int32_t)i;
  }
  int32_t* tmp = (int32_t*)malloc((size_t)(N > 0 ? N : 1) * sizeof(int32_t));
  merge_sort(P->perm, tmp, P->code, N);
  free(tmp);
  if (N > 0 && build_trees) {
    build_cluster(P, 0, (int32_t)N, 0);
    build_block(P, 0, 0);
  }
  P->dblk = (double**)calloc((size_t)(P->ndense + 1), sizeof(double*));
  P->U = (double**)calloc((size_t)(P->nadm + 1), sizeof(double*));
  P->Vf = (double**)calloc((size_t)(P->nadm + 1), sizeof(double*));
  P->piv = (int32_t**)calloc((size_t)(P->nadm + 1), sizeof(int32_t*));
  P->rank = (int*)malloc((size_t)(P->nadm + 1) * sizeof(int));
  for (int64_t b = 0; b < P->nadm; ++b) P->rank[b] = -1;
}

static void free_assembly(or_problem* P) {
  for (int64_t b = 0; b < P->ndense; ++b) { free(P->dblk[b]); P->dblk[b] = NULL; }
  for (int64_t b = 0; b < P->nadm; ++b) {
    free(P->U[b]); free(P->Vf[b]); free(P->piv[b]);
    P->U[b] = P->Vf[b] = NULL; P->piv[b] = NULL; P->rank[b] = -1;
  }
}

/* Release the stored blocks of the last or_assemble (bookkeeping only, no arithmetic):
 * lets a caller that times or_assemble keep the frees of a previous assembly out of it. */
void or_release(or_problem* P) { free_assembly(P); }

void or_destroy(or_problem* P) {
  if (!P) return;
  free_assembly(P);
  free(P->dblk); free(P->U); free(P->Vf); free(P->piv); free(P->rank);
  free(P->V); free(P->T); free(P->cen); free(P->area); free(P->h); free(P->code);
  free(P->perm); free(P->cl); free(P->adm); free(P->dense);
  free(P->Q);
  or_destroy(P->tri);
  free(P);
}

int64_t or_n(const or_problem* P) { return P->N; }
void or_get_perm(const or_problem* P, int32_t* perm) { memcpy(perm, P->perm, (size_t)P->N * sizeof(int32_t)); }
void or_get_codes(const or_problem* P, uint64_t* codes) { memcpy(codes, P->code, (size_t)P->N * sizeof(uint64_t)); }
void or_get_geometry(const or_problem* P, double* c, double* area, double* h) {
  memcpy(c, P->cen, (size_t)P->N * 3 * sizeof(double));
  memcpy(area, P->area, (size_t)P->N * sizeof(double));
  memcpy(h, P->h, (size_t)P->N * sizeof(double));
}
int64_t or_num_clusters(const or_problem* P) { return P->ncl; }
void or_get_clusters(const or_problem* P, int32_t* lo, int32_t* hi, int32_t* child0,
                     int32_t* depth, double* bbox) {
  for (int64_t c = 0; c < P->ncl; ++c) {
    lo[c] = P->cl[c].lo; hi[c] = P->cl[c].hi; child0[c] = P->cl[c].child0; depth[c] = P->cl[c].depth;
    memcpy(bbox + 6 * c, P->cl[c].box, 6 * sizeof(double));
  }
}
int64_t or_num_leaves(const or_problem* P, int kind) { return kind == 0 ? P->nadm : P->ndense; }
void or_get_leaves(const or_problem* P, int kind, int32_t* quads) {
  const quad_t* q = kind == 0 ? P->adm : P->dense;
  int64_t n = kind == 0 ? P->nadm : P->ndense;
  memcpy(quads, q, (size_t)n * sizeof(quad_t));
}

/* ------------------------------------------------------------------ */
/* Gauss-Legendre on [0,1] (A14): Newton on the three-term recurrence in  */
/* long double, rounded once to binary64.                                 */
/* ------------------------------------------------------------------ */
void or_gauss_legendre01(int n, double* x, double* w) {
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int k = 0; k < n; ++k) {
    long double t = cosl(pi * ((long double)k + 0.75L) / ((long double)n + 0.5L));
    long double p0 = 1, p1 = t, dp = 1;
    for (int it = 0; it < 100; ++it) {
      p0 = 1.0L; p1 = t;
      for (int m = 2; m <= n; ++m) {
        long double p2 = ((2.0L * m - 1.0L) * t * p1 - (m - 1.0L) * p0) / (long double)m;
        p0 = p1; p1 = p2;
      }
      if (n == 1) { p0 = 1.0L; p1 = t; }
      dp = (long double)n * (t * p1 - p0) / (t * t - 1.0L);
      long double dt = p1 / dp;
      t -= dt;
      if (fabsl(dt) <= 1e-21L * fabsl(t) + 1e-30L) break;
    }
    p0 = 1.0L; p1 = t;
    for (int m = 2; m <= n; ++m) {
      long double p2 = ((2.0L * m - 1.0L) * t * p1 - (m - 1.0L) * p0) / (long double)m;
      p0 = p1; p1 = p2;
    }
    dp = (long double)n * (t * p1 - p0) / (t * t - 1.0L);
    /* t_k descends with k, so (1 - t)/2 ascends */
    x[k] = (double)((1.0L - t) / 2.0L);
    w[k] = (double)(1.0L / ((1.0L - t * t) * dp * dp));  /* = (2/((1-t^2)P'^2)) / 2 */
  }
}

/* ------------------------------------------------------------------ */
/* quadrature rules (A14), arithmetic (A15)                            */
/* ------------------------------------------------------------------ */
typedef struct { double v0[3], e1[3], e2[3]; } tri_t;   /* chi(s,t) = v0 + s e1 + t e2 */

static tri_t make_tri(const double* v0, const double* v1, const double* v2) {
  tri_t T;
  for (int a = 0; a < 3; ++a) { T.v0[a] = v0[a]; T.e1[a] = v1[a] - v0[a]; T.e2[a] = v2[a] - v1[a]; }
  return T;
}

/* collapsed-Gauss reference table of order n: s = xi, t = xi*zeta, w = (w_xi*w_zeta)*xi */
typedef struct { int n, np; double s[64], t[64], w[64]; } reftab_t;   /* np points */

static reftab_t make_reftab(int n) {
  reftab_t R;
  double g[32], gw[32];
  or_gauss_legendre01(n, g, gw);
  R.n = n;
  R.np = n * n;
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) {
      int q = a * n + b;
      R.s[q] = g[a];
      R.t[q] = g[a] * g[b];
      R.w[q] = (gw[a] * gw[b]) * g[a];
    }
  return R;
}

/* Radon's 7-point rule, exact to degree 5 (Radon 1948; Stroud T2:5-1), the A14 rule of the
 * rho >= 8 band: barycentric (1/3,1/3,1/3) weight 9/40; the three permutations of
 * (a, a, 1-2a), a = (6 - sqrt15)/21, weight (155 - sqrt15)/1200; of (b, b, 1-2b),
 * b = (6 + sqrt15)/21, weight (155 + sqrt15)/1200.  In the (s, t) form of chi with
 * lambda = (1 - s, s - t, t): s = 1 - lambda0, t = lambda2; weights halved (reference area
 * 1/2, like the collapsed rule).  Order: centre, (a,a,c), (a,c,a), (c,a,a), then b.
 * Values in binary128 (libquadmath), rounded once to binary64. */
static reftab_t make_reftab_radon(void) {
  reftab_t R;
  R.n = 3;
  R.np = 7;
  const __float128 r15 = sqrtq((__float128)15);
  const __float128 abc[2] = {(6 - r15) / 21, (6 + r15) / 21};
  const __float128 wab[2] = {(155 - r15) / 2400, (155 + r15) / 2400};
  const __float128 third = (__float128)1 / 3;
  R.s[0] = (double)(1 - third); R.t[0] = (double)third; R.w[0] = (double)((__float128)9 / 80);
  for (int g = 0; g < 2; ++g) {
    const __float128 a = abc[g], c = 1 - 2 * a;
    const __float128 lam[3][3] = {{a, a, c}, {a, c, a}, {c, a, a}};
    for (int k = 0; k < 3; ++k) {
      const int q = 1 + 3 * g + k;
      R.s[q] = (double)(1 - lam[k][0]);
      R.t[q] = (double)lam[k][2];
      R.w[q] = (double)wab[g];
    }
  }
  return R;
}

/* number of points of the A14 rule of regular order n on one triangle */
static int rule_points(const reftab_t* R) { return R->np; }

/* the A14 rule table of regular order n: Radon for n = 3, collapsed Gauss n x n otherwise */
static reftab_t rule_table(int n) { return n == 3 ? make_reftab_radon() : make_reftab(n); }

int or_rule_table(int n, double* s, double* t, double* w) {
  reftab_t R = rule_table(n);
  for (int q = 0; q < R.np; ++q) { s[q] = R.s[q]; t[q] = R.t[q]; w[q] = R.w[q]; }
  return R.np;
}

static void tri_point(const tri_t* T, double s, double t, double* x) {
  for (int a = 0; a < 3; ++a) x[a] = fma(t, T->e2[a], fma(s, T->e1[a], T->v0[a]));
}

/* regular rule: I = sum_p w_p sum_q w_q / |x_p - y_q|  (unscaled by Jacobians) */
static double regular_sum(const tri_t* X, const tri_t* Y, const reftab_t* R) {
  int nq = rule_points(R);
  double I = 0.0;
  for (int p = 0; p < nq; ++p) {
    double xp[3];
    tri_point(X, R->s[p], R->t[p], xp);
    double inner = 0.0;
    for (int q = 0; q < nq; ++q) {
      double yq[3];
      tri_point(Y, R->s[q], R->t[q], yq);
      double dx = xp[0] - yq[0], dy = xp[1] - yq[1], dz = xp[2] - yq[2];
      double d2 = fma(dz, dz, fma(dy, dy, dx * dx));
      inner = inner + R->w[q] / sqrt(d2);
    }
    I = I + R->w[p] * inner;
  }
  return I;
}

double or_regular_rule(const double* tx, const double* ty, int n) {
  tri_t X = make_tri(tx, tx + 3, tx + 6), Y = make_tri(ty, ty + 3, ty + 6);
  reftab_t R = rule_table(n);
  double c[3], ax, ay, h;
  panel_geometry(tx, tx + 3, tx + 6, c, &ax, &h);
  panel_geometry(ty, ty + 3, ty + 6, c, &ay, &h);
  return regular_sum(&X, &Y, &R) * ((2.0 * ax) * (2.0 * ay));
}

/* closed-form self integral int_T int_T 1/|x-y| = (4|T|^2/3) sum_e ln(p/(p-2 l_e))/l_e (A14) */
double or_selfterm_closed(const double* v0, const double* v1, const double* v2) {
  double c[3], area, h;
  panel_geometry(v0, v1, v2, c, &area, &h);
  double l0 = edge_len(v0, v1), l1 = edge_len(v1, v2), l2 = edge_len(v2, v0);
  double p = (l0 + l1) + l2;
  double S = log(p / (p - 2.0 * l0)) / l0;
  S = S + log(p / (p - 2.0 * l1)) / l1;
  S = S + log(p / (p - 2.0 * l2)) / l2;
  return ((4.0 * area * area) / 3.0) * S;
}

/* Sauter-Schwab reference maps (Sauter & Schwab 2011 §5.2, cited as [Sauter1997] at P:644).
 * Reference triangle {0 <= x2 <= x1 <= 1}, chi(x) = A + x1 (B - A) + x2 (C - B).
 * Returns the region count; fills x1[r],x2[r],y1[r],y2[r],wr[r] (region weight incl. Jacobian). */
static int ss_regions(int kind, double xi, double e1, double e2, double e3,
                      double* x1, double* x2, double* y1, double* y2, double* wr) {
  if (kind == 0) {           /* identical panels: 6 regions, weight xi^3 e1^2 e2 */
    double w = xi * xi * xi * e1 * e1 * e2;
    x1[0] = xi;                       x2[0] = xi * (1.0 - e1 + e1 * e2);
    y1[0] = xi * (1.0 - e1 * e2 * e3); y2[0] = xi * (1.0 - e1);
    x1[1] = y1[0]; x2[1] = y2[0]; y1[1] = x1[0]; y2[1] = x2[0];
    x1[2] = xi;                       x2[2] = xi * e1 * (1.0 - e2 + e2 * e3);
    y1[2] = xi * (1.0 - e1 * e2);     y2[2] = xi * e1 * (1.0 - e2);
    x1[3] = y1[2]; x2[3] = y2[2]; y1[3] = x1[2]; y2[3] = x2[2];
    x1[4] = xi * (1.0 - e1 * e2 * e3); x2[4] = xi * e1 * (1.0 - e2 * e3);
    y1[4] = xi;                       y2[4] = xi * e1 * (1.0 - e2);
    x1[5] = y1[4]; x2[5] = y2[4]; y1[5] = x1[4]; y2[5] = x2[4];
    for (int r = 0; r < 6; ++r) wr[r] = w;
    return 6;
  } else if (kind == 1) {    /* common edge (A,B): 5 regions */
    double w = xi * xi * xi * e1 * e1;
    x1[0] = xi;                       x2[0] = xi * e1 * e3;
    y1[0] = xi * (1.0 - e1 * e2);     y2[0] = xi * e1 * (1.0 - e2);
    x1[1] = xi;                       x2[1] = xi * e1;
    y1[1] = xi * (1.0 - e1 * e2 * e3); y2[1] = xi * e1 * e2 * (1.0 - e3);
    x1[2] = xi * (1.0 - e1 * e2);     x2[2] = xi * e1 * (1.0 - e2);
    y1[2] = xi;                       y2[2] = xi * e1 * e2 * e3;
    x1[3] = xi * (1.0 - e1 * e2 * e3); x2[3] = xi * e1 * e2 * (1.0 - e3);
    y1[3] = xi;                       y2[3] = xi * e1;
    x1[4] = xi * (1.0 - e1 * e2 * e3); x2[4] = xi * e1 * (1.0 - e2 * e3);
    y1[4] = xi;                       y2[4] = xi * e1 * e2;
    wr[0] = w;
    for (int r = 1; r < 5; ++r) wr[r] = w * e2;
    return 5;
  } else {                   /* common vertex A: 2 regions, weight xi^3 e2 */
    double w = xi * xi * xi * e2;
    x1[0] = xi;       x2[0] = xi * e1;
    y1[0] = xi * e2;  y2[0] = xi * e2 * e3;
    x1[1] = y1[0]; x2[1] = y2[0]; y1[1] = x1[0]; y2[1] = x2[0];
    wr[0] = w; wr[1] = w;
    return 2;
  }
}

/* int_{Tx} int_{Ty} 1/|x-y| for panels sharing vertex A (= tx[0..2] = ty[0..2]):
 * the difference x - y = (x1 E1x + x2 E2x) - (y1 E1y + y2 E2y) (A cancels exactly). */
static double ss_sum(int kind, const tri_t* X, const tri_t* Y, int nq) {
  double g[32], gw[32];
  or_gauss_legendre01(nq, g, gw);
  double I = 0.0;
  for (int a = 0; a < nq; ++a)
    for (int b = 0; b < nq; ++b)
      for (int c = 0; c < nq; ++c)
        for (int d = 0; d < nq; ++d) {
          double x1[6], x2[6], y1[6], y2[6], wr[6];
          int R = ss_regions(kind, g[a], g[b], g[c], g[d], x1, x2, y1, y2, wr);
          double s = 0.0;
          for (int r = 0; r < R; ++r) {
            double dv[3];
            for (int k = 0; k < 3; ++k)
              dv[k] = fma(x2[r], X->e2[k], x1[r] * X->e1[k]) - fma(y2[r], Y->e2[k], y1[r] * Y->e1[k]);
            double d2 = fma(dv[2], dv[2], fma(dv[1], dv[1], dv[0] * dv[0]));
            s = s + wr[r] / sqrt(d2);
          }
          I = I + (((gw[a] * gw[b]) * (gw[c] * gw[d])) * s);
        }
  return I;
}

double or_sauter_schwab(int kind, const double* tx, const double* ty, int nq) {
  tri_t X = make_tri(tx, tx + 3, tx + 6), Y = make_tri(ty, ty + 3, ty + 6);
  double c[3], ax, ay, h;
  panel_geometry(tx, tx + 3, tx + 6, c, &ax, &h);
  panel_geometry(ty, ty + 3, ty + 6, c, &ay, &h);
  return ss_sum(kind, &X, &Y, nq) * ((2.0 * ax) * (2.0 * ay));
}

double or_ss_reference_monomial(int kind, int nq, int pa, int pb, int pc, int pd) {
  double g[32], gw[32];
  or_gauss_legendre01(nq, g, gw);
  double I = 0.0;
  for (int a = 0; a < nq; ++a)
    for (int b = 0; b < nq; ++b)
      for (int c = 0; c < nq; ++c)
        for (int d = 0; d < nq; ++d) {
          double x1[6], x2[6], y1[6], y2[6], wr[6];
          int R = ss_regions(kind, g[a], g[b], g[c], g[d], x1, x2, y1, y2, wr);
          double s = 0.0;
          for (int r = 0; r < R; ++r)
            s += wr[r] * pow(x1[r], pa) * pow(x2[r], pb) * pow(y1[r], pc) * pow(y2[r], pd);
          I += gw[a] * gw[b] * gw[c] * gw[d] * s;
        }
  return I;
}

/* ------------------------------------------------------------------ */
/* Galerkin entry a_ij (P:224-228 per A1; classification A14)          */
/* ------------------------------------------------------------------ */
/* tensor-Gauss table of order n on the unit square (quads, A25): s = g_a, t = g_b,
 * w = w_a * w_b, q = a*n + b */
static reftab_t make_reftab_square(int n) {
  reftab_t R;
  double g[32], gw[32];
  or_gauss_legendre01(n, g, gw);
  R.n = n;
  R.np = n * n;
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) {
      int q = a * n + b;
      R.s[q] = g[a];
      R.t[q] = g[b];
      R.w[q] = gw[a] * gw[b];
    }
  return R;
}

static reftab_t g_tab[7], g_qtab[7];
static int g_tab_init = 0;
static void init_tables(void) {
  if (g_tab_init) return;
  for (int n = 3; n <= 6; ++n) { g_tab[n] = rule_table(n); g_qtab[n] = make_reftab_square(n); }
  g_tab_init = 1;
}

/* returns 0 identical, 1 edge, 2 vertex, else regular order n in {3,4,5,6} */
static int classify(const or_problem* P, int64_t i, int64_t j) {
  const int32_t* ti = P->T + 3 * i;
  const int32_t* tj = P->T + 3 * j;
  int shared = 0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) shared += (ti[a] == tj[b]);
  if (shared >= 3) return 0;
  if (shared == 2) return 1;
  if (shared == 1) return 2;
  const double* ci = P->cen + 3 * i;
  const double* cj = P->cen + 3 * j;
  double dx = ci[0] - cj[0], dy = ci[1] - cj[1], dz = ci[2] - cj[2];
  double dc2 = (dx * dx + dy * dy) + dz * dz;
  double hm = P->h[i] > P->h[j] ? P->h[i] : P->h[j];
  double hm2 = hm * hm;
  if (dc2 < 4.0 * hm2) return 6;
  if (dc2 < 16.0 * hm2) return 5;
  if (dc2 < 64.0 * hm2) return 4;
  return 3;
}

int or_entry_class(const or_problem* P, int64_t i, int64_t j) { return P->tri ? -1 : classify(P, i, j); }

static const int64_t ss_evals[3] = {0, 5 * 1296, 2 * 1296};

static double entry_app(const or_problem* P, int64_t i, int64_t j, double* evals) {
  int64_t x = i < j ? i : j, y = i < j ? j : i;    /* canonical: lower application index outer */
  if (P->tri) {                                    /* quadrilaterals (A25) */
    const int32_t* qx = P->Q + 4 * x;
    const int32_t* qy = P->Q + 4 * y;
    int shared = 0;
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) shared += (qx[a] == qy[b]);
    if (shared) {                                  /* touching: four triangle pairs, fixed order */
      double e00 = entry_app(P->tri, 2 * x, 2 * y, evals), e01 = entry_app(P->tri, 2 * x, 2 * y + 1, evals);
      double e10 = entry_app(P->tri, 2 * x + 1, 2 * y, evals), e11 = entry_app(P->tri, 2 * x + 1, 2 * y + 1, evals);
      return ((e00 + e01) + e10) + e11;
    }
    /* separated: tensor Gauss n x n on each parallelogram, chi(s,t) = q0 + s(q1-q0) + t(q2-q1),
     * n from the node distance in the bands of A14 with h = max of the two triangles' h */
    const double* ci = P->cen + 3 * x;
    const double* cj = P->cen + 3 * y;
    double dx = ci[0] - cj[0], dy = ci[1] - cj[1], dz = ci[2] - cj[2];
    double dc2 = (dx * dx + dy * dy) + dz * dz;
    double hm = P->h[x] > P->h[y] ? P->h[x] : P->h[y];
    double hm2 = hm * hm;
    int n = dc2 < 4.0 * hm2 ? 6 : dc2 < 16.0 * hm2 ? 5 : dc2 < 64.0 * hm2 ? 4 : 3;
    tri_t X = make_tri(P->V + 3 * qx[0], P->V + 3 * qx[1], P->V + 3 * qx[2]);
    tri_t Y = make_tri(P->V + 3 * qy[0], P->V + 3 * qy[1], P->V + 3 * qy[2]);
    if (evals) *evals += (double)(n * n * n * n);
    double I = regular_sum(&X, &Y, &g_qtab[n]);
    return (I * (P->area[x] * P->area[y])) * INV4PI;
  }
  int cls = classify(P, x, y);
  if (cls == 0) {
    if (evals) *evals += 0;
    return or_selfterm_closed(vtx(P, x, 0), vtx(P, x, 1), vtx(P, x, 2)) * INV4PI;
  }
  if (cls == 1 || cls == 2) {
    const int32_t* tx = P->T + 3 * x;
    const int32_t* ty = P->T + 3 * y;
    int32_t A, Bx, Cx, By, Cy;
    if (cls == 1) {
      int32_t s[2], ns = 0, ox = -1, oy = -1;
      for (int a = 0; a < 3; ++a) {
        int in = (tx[a] == ty[0]) || (tx[a] == ty[1]) || (tx[a] == ty[2]);
        if (in) s[ns++] = tx[a]; else ox = tx[a];
      }
      for (int b = 0; b < 3; ++b)
        if (ty[b] != s[0] && ty[b] != s[1]) oy = ty[b];
      A = s[0] < s[1] ? s[0] : s[1];                  /* lower vertex id first */
      Bx = By = s[0] < s[1] ? s[1] : s[0];
      Cx = ox; Cy = oy;
    } else {
      int ax = 0, ay = 0;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          if (tx[a] == ty[b]) { ax = a; ay = b; }
      A = tx[ax];
      Bx = tx[(ax + 1) % 3]; Cx = tx[(ax + 2) % 3];  /* cyclic order after the shared vertex */
      By = ty[(ay + 1) % 3]; Cy = ty[(ay + 2) % 3];
    }
    tri_t X = make_tri(P->V + 3 * A, P->V + 3 * Bx, P->V + 3 * Cx);
    tri_t Y = make_tri(P->V + 3 * A, P->V + 3 * By, P->V + 3 * Cy);
    if (evals) *evals += (double)ss_evals[cls];
    double I = ss_sum(cls, &X, &Y, NQ_SINGULAR);
    return (I * ((2.0 * P->area[x]) * (2.0 * P->area[y]))) * INV4PI;
  }
  tri_t X = make_tri(vtx(P, x, 0), vtx(P, x, 1), vtx(P, x, 2));
  tri_t Y = make_tri(vtx(P, y, 0), vtx(P, y, 1), vtx(P, y, 2));
  const reftab_t* R = &g_tab[cls];
  if (evals) *evals += (double)(R->np * R->np);
  double I = regular_sum(&X, &Y, R);
  return (I * ((2.0 * P->area[x]) * (2.0 * P->area[y]))) * INV4PI;
}

void or_entries(const or_problem* P, int64_t n, const int64_t* pairs, double* out) {
  init_tables();
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t e = 0; e < n; ++e) out[e] = entry_app(P, pairs[2 * e], pairs[2 * e + 1], NULL);
}

void or_dense_rows(const or_problem* P, int64_t nrows, const int64_t* rows, double* out) {
  init_tables();
  int64_t N = P->N;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t e = 0; e < nrows * N; ++e) out[e] = entry_app(P, rows[e / N], e % N, NULL);
}

/* ------------------------------------------------------------------ */
/* ACA with partial pivoting (A11, A12)           */
/* ------------------------------------------------------------------ */
typedef double (*entry_fn)(const void* ctx, int t, int j);

static int aca_core(entry_fn a, const void* ctx, int m, int n, double eps, int kcap,
                    double* U, double* V, int32_t* pivots) {
  if (m <= 0 || n <= 0) return 0;
  int kmax = m < n ? m : n;
  if (kcap < kmax) kmax = kcap;
  char* used = (char*)calloc((size_t)m, 1);
  double* r = (double*)malloc((size_t)n * sizeof(double));
  double* u = (double*)malloc((size_t)m * sizeof(double));
  int k = 0, i = 0;
  double S2 = 0.0;
  while (k < kmax) {
    /* 1. residual row r_j = a(i,j) - sum_{l<k} U[i][l] V[j][l], l ascending */
    for (int j = 0; j < n; ++j) {
      double rj = a(ctx, i, j);
      for (int l = 0; l < k; ++l) rj = rj - U[i + (int64_t)l * m] * V[j + (int64_t)l * n];
      r[j] = rj;
    }
    used[i] = 1;
    /* 2. column pivot: argmax |r_j|, lowest index on ties */
    int js = 0;
    double best = fabs(r[0]);
    for (int j = 1; j < n; ++j)
      if (fabs(r[j]) > best) { best = fabs(r[j]); js = j; }
    /* 3. zero residual row: next unused row */
    if (r[js] == 0.0) {
      int nx = -1;
      for (int t = 0; t < m; ++t) if (!used[t]) { nx = t; break; }
      if (nx < 0) break;
      i = nx;
      continue;
    }
    /* 4. v = r / r_js */
    double piv = r[js];
    double* vk = V + (int64_t)k * n;
    for (int j = 0; j < n; ++j) vk[j] = r[j] / piv;
    /* 5. residual column u_t = a(t,js) - sum_{l<k} U[t][l] V[js][l] */
    for (int t = 0; t < m; ++t) {
      double ut = a(ctx, t, js);
      for (int l = 0; l < k; ++l) ut = ut - U[t + (int64_t)l * m] * V[js + (int64_t)l * n];
      u[t] = ut;
    }
    /* 6. Frobenius norm update ||S_k||^2 (Bebendorf) */
    double uu = 0.0, vv = 0.0, cross = 0.0;
    for (int t = 0; t < m; ++t) uu = uu + u[t] * u[t];
    for (int j = 0; j < n; ++j) vv = vv + vk[j] * vk[j];
    for (int l = 0; l < k; ++l) {
      double du = 0.0, dv = 0.0;
      for (int t = 0; t < m; ++t) du = du + u[t] * U[t + (int64_t)l * m];
      for (int j = 0; j < n; ++j) dv = dv + V[j + (int64_t)l * n] * vk[j];
      cross = cross + du * dv;
    }
    S2 = (S2 + 2.0 * cross) + uu * vv;
    memcpy(U + (int64_t)k * m, u, (size_t)m * sizeof(double));
    if (pivots) { pivots[2 * k] = i; pivots[2 * k + 1] = js; }
    k += 1;
    /* 7. stop test ||u_k|| ||v_k|| <= eps ||S_k||_F */
    if (sqrt(uu) * sqrt(vv) <= eps * sqrt(S2)) break;
    /* 8. rank budget */
    if (k >= kmax) break;
    /* 9. next row: argmax over unused rows of |u_t|, lowest index on ties */
    int nx = -1;
    double bu = -1.0;
    for (int t = 0; t < m; ++t)
      if (!used[t] && fabs(u[t]) > bu) { bu = fabs(u[t]); nx = t; }
    if (nx < 0) break;
    i = nx;
  }
  free(used); free(r); free(u);
  return k;
}

typedef struct { const or_problem* P; int32_t rlo, clo; double evals; } blk_ctx;
static double blk_entry(const void* c, int t, int j) {
  blk_ctx* b = (blk_ctx*)c;
  return entry_app(b->P, b->P->perm[b->rlo + t], b->P->perm[b->clo + j], &b->evals);
}
typedef struct { const double* A; int n; } mat_ctx;
static double mat_entry(const void* c, int t, int j) {
  const mat_ctx* M = (const mat_ctx*)c;
  return M->A[(int64_t)t * M->n + j];
}

int or_aca_block(const or_problem* P, int32_t rlo, int32_t rhi, int32_t clo, int32_t chi,
                 double eps, int kcap, double* U, double* V, int32_t* pivots) {
  init_tables();
  blk_ctx c = {P, rlo, clo, 0.0};
  return aca_core(blk_entry, &c, rhi - rlo, chi - clo, eps, kcap, U, V, pivots);
}

int or_aca_matrix(const double* A, int m, int n, double eps, int kcap,
                  double* U, double* V, int32_t* pivots) {
  mat_ctx c = {A, n};
  return aca_core(mat_entry, &c, m, n, eps, kcap, U, V, pivots);
}

/* ------------------------------------------------------------------ */
/* assembly: near-field blocks + ACA blocks     */
/* ------------------------------------------------------------------ */
static void assemble_dense_leaf(or_problem* P, int64_t b, double* ev) {
  const quad_t* q = &P->dense[b];
  int m = q->rhi - q->rlo, n = q->chi - q->clo;
  double* B = (double*)malloc((size_t)m * n * sizeof(double));
  for (int a = 0; a < m; ++a)
    for (int c = 0; c < n; ++c)
      B[(int64_t)a * n + c] = entry_app(P, P->perm[q->rlo + a], P->perm[q->clo + c], ev);
  P->dblk[b] = B;
}

static void assemble_adm_leaf(or_problem* P, int64_t b, double eps, int kcap, double* ev) {
  const quad_t* q = &P->adm[b];
  int m = q->rhi - q->rlo, n = q->chi - q->clo;
  int kmax = m < n ? m : n;
  if (kcap < kmax) kmax = kcap;
  double* U = (double*)malloc((size_t)m * kmax * sizeof(double));
  double* V = (double*)malloc((size_t)n * kmax * sizeof(double));
  int32_t* pv = (int32_t*)malloc((size_t)(2 * kmax + 2) * sizeof(int32_t));
  blk_ctx c = {P, q->rlo, q->clo, 0.0};
  int k = aca_core(blk_entry, &c, m, n, eps, kcap, U, V, pv);
  P->U[b] = U; P->Vf[b] = V; P->piv[b] = pv; P->rank[b] = k;
  *ev += c.evals;
}

int or_assemble(or_problem* P, double eps, int kcap, int64_t d0, int64_t d1, int64_t a0, int64_t a1) {
  init_tables();
  free_assembly(P);
  double ev_near = 0, ev_aca = 0, en_near = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : ev_near, en_near)
  for (int64_t b = d0; b < d1; ++b) {
    double ev = 0;
    assemble_dense_leaf(P, b, &ev);
    ev_near += ev;
    en_near += (double)(P->dense[b].rhi - P->dense[b].rlo) * (P->dense[b].chi - P->dense[b].clo);
  }
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : ev_aca)
  for (int64_t b = a0; b < a1; ++b) {
    double ev = 0;
    assemble_adm_leaf(P, b, eps, kcap, &ev);
    ev_aca += ev;
  }
  P->counters[0] = ev_near; P->counters[1] = ev_aca;
  P->counters[2] = en_near; P->counters[3] = 0;
  return 0;
}

/* The same for explicit (ascending) lists of leaf indices: lets a timing harness assemble a
 * sample of leaves spread over the whole lists (bookkeeping only; same per-leaf code). */
int or_assemble_list(or_problem* P, double eps, int kcap, int64_t nd, const int64_t* dl, int64_t na,
                     const int64_t* al) {
  init_tables();
  free_assembly(P);
  double ev_near = 0, ev_aca = 0, en_near = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : ev_near, en_near)
  for (int64_t x = 0; x < nd; ++x) {
    double ev = 0;
    const int64_t b = dl[x];
    assemble_dense_leaf(P, b, &ev);
    ev_near += ev;
    en_near += (double)(P->dense[b].rhi - P->dense[b].rlo) * (P->dense[b].chi - P->dense[b].clo);
  }
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : ev_aca)
  for (int64_t x = 0; x < na; ++x) {
    double ev = 0;
    assemble_adm_leaf(P, al[x], eps, kcap, &ev);
    ev_aca += ev;
  }
  P->counters[0] = ev_near; P->counters[1] = ev_aca;
  P->counters[2] = en_near; P->counters[3] = 0;
  return 0;
}

void or_counters(const or_problem* P, double* out) { memcpy(out, P->counters, 4 * sizeof(double)); }

int64_t or_stored_doubles(const or_problem* P) {
  int64_t s = 0;
  for (int64_t b = 0; b < P->ndense; ++b)
    if (P->dblk[b]) s += (int64_t)(P->dense[b].rhi - P->dense[b].rlo) * (P->dense[b].chi - P->dense[b].clo);
  for (int64_t b = 0; b < P->nadm; ++b)
    if (P->rank[b] >= 0) s += (int64_t)P->rank[b] * ((P->adm[b].rhi - P->adm[b].rlo) + (P->adm[b].chi - P->adm[b].clo));
  return s;
}
int or_get_rank(const or_problem* P, int64_t b) { return P->rank[b]; }
void or_get_factors(const or_problem* P, int64_t b, double* U, double* V) {
  int m = P->adm[b].rhi - P->adm[b].rlo, n = P->adm[b].chi - P->adm[b].clo, k = P->rank[b];
  if (k <= 0) return;
  memcpy(U, P->U[b], (size_t)m * k * sizeof(double));
  memcpy(V, P->Vf[b], (size_t)n * k * sizeof(double));
}
void or_get_pivots(const or_problem* P, int64_t b, int32_t* pv) {
  if (P->rank[b] > 0) memcpy(pv, P->piv[b], (size_t)2 * P->rank[b] * sizeof(int32_t));
}
void or_get_dense_block(const or_problem* P, int64_t b, double* B) {
  int m = P->dense[b].rhi - P->dense[b].rlo, n = P->dense[b].chi - P->dense[b].clo;
  if (P->dblk[b]) memcpy(B, P->dblk[b], (size_t)m * n * sizeof(double));
}

/* ------------------------------------------------------------------ */
/* H-matvec: dense leaves apply the full block, admissible  */
/* leaves apply U (V^T x).  Per-thread partial sums over a static split */
/* of the leaf lists, summed in thread order.                           */
/* ------------------------------------------------------------------ */
void or_matvec(const or_problem* P, const double* x, double* y) {
  int64_t N = P->N;
  double* xi = (double*)malloc((size_t)(N + 1) * sizeof(double));
  for (int64_t s = 0; s < N; ++s) xi[s] = x[P->perm[s]];
  int nth = 1;
#ifdef _OPENMP
  nth = omp_get_max_threads();
#endif
  double* part = (double*)calloc((size_t)nth * (N + 1), sizeof(double));
#pragma omp parallel num_threads(nth)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    double* yi = part + (int64_t)tid * (N + 1);
#pragma omp for schedule(static)
    for (int64_t b = 0; b < P->ndense; ++b) {
      if (!P->dblk[b]) continue;
      const quad_t* q = &P->dense[b];
      int m = q->rhi - q->rlo, n = q->chi - q->clo;
      const double* B = P->dblk[b];
      for (int a = 0; a < m; ++a) {
        double s = 0.0;
        for (int c = 0; c < n; ++c) s += B[(int64_t)a * n + c] * xi[q->clo + c];
        yi[q->rlo + a] += s;
      }
    }
#pragma omp for schedule(static)
    for (int64_t b = 0; b < P->nadm; ++b) {
      int k = P->rank[b];
      if (k <= 0) continue;
      const quad_t* q = &P->adm[b];
      int m = q->rhi - q->rlo, n = q->chi - q->clo;
      double t[128];
      double* tt = k <= 128 ? t : (double*)malloc((size_t)k * sizeof(double));
      for (int l = 0; l < k; ++l) {
        double s = 0.0;
        for (int c = 0; c < n; ++c) s += P->Vf[b][c + (int64_t)l * n] * xi[q->clo + c];
        tt[l] = s;
      }
      for (int a = 0; a < m; ++a) {
        double s = 0.0;
        for (int l = 0; l < k; ++l) s += P->U[b][a + (int64_t)l * m] * tt[l];
        yi[q->rlo + a] += s;
      }
      if (tt != t) free(tt);
    }
  }
  for (int64_t s = 0; s < N; ++s) {
    double acc = 0.0;
    for (int th = 0; th < nth; ++th) acc += part[(int64_t)th * (N + 1) + s];
    y[P->perm[s]] = acc;
  }
  free(part); free(xi);
}

/* ------------------------------------------------------------------ */
/* right-hand side f_i = int_{T_i} f (A16)                   */
/* ------------------------------------------------------------------ */
static double paper_f(const double* x) { return (4.0 * x[0] * x[0] - 3.0 * x[1] * x[1]) - x[2] * x[2]; }

void or_rhs(const or_problem* P, int kind, double* f) {
  if (P->tri) {                                    /* quads (A25): f_i = f_2i + f_2i+1 */
    double* f2 = (double*)malloc((size_t)(2 * P->N > 0 ? 2 * P->N : 1) * sizeof(double));
    or_rhs(P->tri, kind, f2);
    for (int64_t i = 0; i < P->N; ++i) f[i] = f2[2 * i] + f2[2 * i + 1];
    free(f2);
    return;
  }
  for (int64_t i = 0; i < P->N; ++i) {
    if (kind == 0) { f[i] = P->area[i]; continue; }
    const double *a = vtx(P, i, 0), *b = vtx(P, i, 1), *c = vtx(P, i, 2);
    double m01[3], m12[3], m20[3];
    for (int k = 0; k < 3; ++k) {
      m01[k] = (a[k] + b[k]) / 2.0; m12[k] = (b[k] + c[k]) / 2.0; m20[k] = (c[k] + a[k]) / 2.0;
    }
    f[i] = (P->area[i] / 3.0) * ((paper_f(m01) + paper_f(m12)) + paper_f(m20));
  }
}

/* ------------------------------------------------------------------ */
/* Krylov solvers (A17)                              */
/* ------------------------------------------------------------------ */
static double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

static double true_relres(const or_problem* P, const double* b, const double* x, double bn) {
  int64_t N = P->N;
  double* r = (double*)malloc((size_t)N * sizeof(double));
  or_matvec(P, x, r);
  for (int64_t i = 0; i < N; ++i) r[i] = b[i] - r[i];
  double rn = sqrt(dot(r, r, N));
  free(r);
  return bn > 0 ? rn / bn : 0.0;
}

int or_cg(const or_problem* P, const double* b, double* x, double tol, int maxit,
          double* relres, int* status) {
  int64_t N = P->N;
  double* r = (double*)malloc((size_t)N * sizeof(double));
  double* p = (double*)malloc((size_t)N * sizeof(double));
  double* Ap = (double*)malloc((size_t)N * sizeof(double));
  for (int64_t i = 0; i < N; ++i) { x[i] = 0.0; r[i] = b[i]; p[i] = b[i]; }
  double bn = sqrt(dot(b, b, N));
  double rr = dot(r, r, N);
  int it = 0;
  *status = 0;
  if (bn == 0.0) { *relres = 0.0; free(r); free(p); free(Ap); return 0; }
  while (it < maxit && sqrt(rr) > tol * bn) {
    or_matvec(P, p, Ap);
    double pAp = dot(p, Ap, N);
    if (!(pAp > 0.0)) { *status = 7; break; }
    double alpha = rr / pAp;
    for (int64_t i = 0; i < N; ++i) { x[i] += alpha * p[i]; r[i] -= alpha * Ap[i]; }
    double rr1 = dot(r, r, N);
    double beta = rr1 / rr;
    rr = rr1;
    for (int64_t i = 0; i < N; ++i) p[i] = r[i] + beta * p[i];
    ++it;
  }
  *relres = true_relres(P, b, x, bn);
  free(r); free(p); free(Ap);
  return it;
}

int or_gmres(const or_problem* P, const double* b, double* x, double tol, int restart,
             int maxit, double* relres, int* status) {
  int64_t N = P->N;
  int m = restart;
  double* Vb = (double*)malloc((size_t)(m + 1) * N * sizeof(double));
  double* H = (double*)calloc((size_t)(m + 1) * m, sizeof(double));  /* H[i + j*(m+1)] */
  double* cs = (double*)malloc((size_t)m * sizeof(double));
  double* sn = (double*)malloc((size_t)m * sizeof(double));
  double* g = (double*)malloc((size_t)(m + 1) * sizeof(double));
  double* h = (double*)malloc((size_t)(m + 1) * sizeof(double));
  double* h2 = (double*)malloc((size_t)(m + 1) * sizeof(double));
  double* w = (double*)malloc((size_t)N * sizeof(double));
  double* yv = (double*)malloc((size_t)m * sizeof(double));
  for (int64_t i = 0; i < N; ++i) x[i] = 0.0;
  double bn = sqrt(dot(b, b, N));
  int total = 0;
  *status = 0;
  if (bn == 0.0) { *relres = 0.0; goto done; }
  for (;;) {
    /* r = b - A x */
    or_matvec(P, x, w);
    for (int64_t i = 0; i < N; ++i) w[i] = b[i] - w[i];
    double beta = sqrt(dot(w, w, N));
    if (beta <= tol * bn || total >= maxit) break;
    for (int64_t i = 0; i < N; ++i) Vb[i] = w[i] / beta;
    for (int i = 0; i <= m; ++i) g[i] = 0.0;
    g[0] = beta;
    int jend = 0;
    int conv = 0;
    for (int j = 0; j < m; ++j) {
      double* vj = Vb + (int64_t)j * N;
      or_matvec(P, vj, w);
      ++total;
      /* classical Gram-Schmidt with one re-orthogonalisation (CGS2) */
      for (int i = 0; i <= j; ++i) h[i] = dot(Vb + (int64_t)i * N, w, N);
      for (int i = 0; i <= j; ++i) { const double* vi = Vb + (int64_t)i * N; for (int64_t t = 0; t < N; ++t) w[t] -= h[i] * vi[t]; }
      for (int i = 0; i <= j; ++i) h2[i] = dot(Vb + (int64_t)i * N, w, N);
      for (int i = 0; i <= j; ++i) { const double* vi = Vb + (int64_t)i * N; for (int64_t t = 0; t < N; ++t) w[t] -= h2[i] * vi[t]; }
      for (int i = 0; i <= j; ++i) h[i] += h2[i];
      double hn = sqrt(dot(w, w, N));
      /* apply previous Givens rotations */
      for (int i = 0; i < j; ++i) {
        double t1 = cs[i] * h[i] + sn[i] * h[i + 1];
        double t2 = -sn[i] * h[i] + cs[i] * h[i + 1];
        h[i] = t1; h[i + 1] = t2;
      }
      double den = sqrt(h[j] * h[j] + hn * hn);
      if (den == 0.0) { cs[j] = 1.0; sn[j] = 0.0; }
      else { cs[j] = h[j] / den; sn[j] = hn / den; }
      h[j] = cs[j] * h[j] + sn[j] * hn;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      for (int i = 0; i <= j; ++i) H[i + (int64_t)j * (m + 1)] = h[i];
      jend = j + 1;
      if (fabs(g[j + 1]) <= tol * bn || total >= maxit || hn == 0.0) { conv = 1; break; }
      double* vn = Vb + (int64_t)(j + 1) * N;
      for (int64_t t = 0; t < N; ++t) vn[t] = w[t] / hn;
    }
    /* back substitution H y = g */
    for (int i = jend - 1; i >= 0; --i) {
      double s = g[i];
      for (int l = i + 1; l < jend; ++l) s -= H[i + (int64_t)l * (m + 1)] * yv[l];
      yv[i] = s / H[i + (int64_t)i * (m + 1)];
    }
    for (int i = 0; i < jend; ++i) {
      const double* vi = Vb + (int64_t)i * N;
      for (int64_t t = 0; t < N; ++t) x[t] += yv[i] * vi[t];
    }
    if (conv && (fabs(g[jend]) <= tol * bn || total >= maxit)) break;
    if (total >= maxit) break;
  }
  *relres = true_relres(P, b, x, bn);
done:
  free(Vb); free(H); free(cs); free(sn); free(g); free(h); free(h2); free(w); free(yv);
  return total;
}

/* ------------------------------------------------------------------ */
/* partition (A18)                               */
/* ------------------------------------------------------------------ */
void or_partition(const int64_t* cost, int64_t n, int p, int64_t* out) {
  int64_t C = 0;
  for (int64_t i = 0; i < n; ++i) C += cost[i];
  out[0] = 0;
  int r = 1;
  int64_t pref = 0;
  for (int64_t i = 0; i < n && r < p; ++i) {
    /* leaf i belongs to the rank whose [floor(rC/p), floor((r+1)C/p)) holds its prefix */
    while (r < p && pref >= (int64_t)(((__int128)r * C) / p)) out[r++] = i;
    pref += cost[i];
  }
  while (r < p) out[r++] = n;
  out[p] = n;
}

/* ---- single-layer potential at evaluation points (reading A23) ------
 * u(x) = (1/4pi) sum_j alpha_j int_{T_j} 1/|x - y| dy, alpha in application order.  Panel
 * integral: the A14 rule of order n on T_j (the regular rule's panel factor), n by the ratio
 * rho^2 = |x - c_j|^2 / h_j^2 in the bands of A14 (< 4: 6, < 16: 5, < 64: 4, else 3):
 *   I_j(x) = (2 |T_j|) * sum_q w_q / sqrt(d2_q),  d2 = fma(dz,dz, fma(dy,dy, dx*dx)).
 * Points must lie off the surface (the rule is not singular-aware). */
double or_panel_potential(const double* x, const double* tri, int n) {
  tri_t T = make_tri(tri, tri + 3, tri + 6);
  reftab_t R = rule_table(n);
  double c[3], area, h;
  panel_geometry(tri, tri + 3, tri + 6, c, &area, &h);
  double inner = 0.0;
  for (int q = 0; q < R.np; ++q) {
    double y[3];
    tri_point(&T, R.s[q], R.t[q], y);
    double dx = x[0] - y[0], dy = x[1] - y[1], dz = x[2] - y[2];
    double d2 = fma(dz, dz, fma(dy, dy, dx * dx));
    inner = inner + R.w[q] / sqrt(d2);
  }
  return inner * (2.0 * area);
}

void or_potential(const or_problem* P, const double* alpha, int64_t M, const double* X, double* out) {
  if (P->tri) {                                    /* quads (A25): both triangles carry alpha_i */
    double* a2 = (double*)malloc((size_t)(2 * P->N > 0 ? 2 * P->N : 1) * sizeof(double));
    for (int64_t i = 0; i < P->N; ++i) a2[2 * i] = a2[2 * i + 1] = alpha[i];
    or_potential(P->tri, a2, M, X, out);
    free(a2);
    return;
  }
  reftab_t R[4];
  for (int n = 3; n <= 6; ++n) R[n - 3] = rule_table(n);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t p = 0; p < M; ++p) {
    const double* x = X + 3 * p;
    double u = 0.0;
    for (int64_t j = 0; j < P->N; ++j) {
      const double* c = P->cen + 3 * j;
      double dx = x[0] - c[0], dy = x[1] - c[1], dz = x[2] - c[2];
      double dc2 = (dx * dx + dy * dy) + dz * dz;
      double h2 = P->h[j] * P->h[j];
      int n = dc2 < 4.0 * h2 ? 6 : dc2 < 16.0 * h2 ? 5 : dc2 < 64.0 * h2 ? 4 : 3;
      const int32_t* t = P->T + 3 * j;
      tri_t T = make_tri(P->V + 3 * t[0], P->V + 3 * t[1], P->V + 3 * t[2]);
      const reftab_t* Rn = &R[n - 3];
      double inner = 0.0;
      for (int q = 0; q < Rn->np; ++q) {
        double y[3];
        tri_point(&T, Rn->s[q], Rn->t[q], y);
        double ex = x[0] - y[0], ey = x[1] - y[1], ez = x[2] - y[2];
        double d2 = fma(ez, ez, fma(ey, ey, ex * ex));
        inner = inner + Rn->w[q] / sqrt(d2);
      }
      u = u + alpha[j] * (inner * (2.0 * P->area[j]));
    }
    out[p] = u * 0.07957747154594767;
  }
}
