/*
 * oracle.h — plain, slow CPU oracle of the H-matrix BEM hot path of
 * Harbrecht & Zaspel, arXiv 1806.11558 ("the paper", /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1806_11558_b200/) never links, imports or calls it,
 * and the two share no source, header, table or constant generator.
 *
 * Every function follows the paper's definitions step by step (citations
 * "P:n" = PAPER.md line n, "S:n" = SPEC.md line n, "A#" = a reading listed
 * in DESIGN.md §3).  Arithmetic is IEEE binary64, round-to-nearest, built
 * with -ffp-contract=off; fused multiply-adds appear only where the reading
 * writes fma() explicitly (A15).  Indices are 0-based.  "internal" index s
 * means Morton-sorted position; perm[s] is the application (triangle) index.
 *
 * Parity status per function: see the header comment of oracle.c.
 */
#ifndef HM_ORACLE_H
#define HM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_problem or_problem;

/* Build mesh geometry, Morton order, cluster tree and block cluster tree
 * (P:256-306).  V: n_v*3 doubles, T: N*3 int32.  Copies inputs. */
or_problem* or_create(const double* V, int64_t n_v, const int32_t* T, int64_t N,
                      int leaf_size, double eta);
/* Quadrilateral panels (A25): Q = N*4 int32 vertex ids in cyclic order, planar
 * parallelograms; quad i is the union of triangles (q0,q1,q2), (q0,q2,q3).  Entries of
 * quads sharing a vertex are the sums over the four triangle pairs; separated quads use a
 * tensor Gauss rule on each parallelogram (A14 bands).  Right-hand side and potential are
 * sums over the two triangles.  or_entry_class returns -1 for quad problems. */
or_problem* or_create_quads(const double* V, int64_t n_v, const int32_t* Q, int64_t N,
                            int leaf_size, double eta);
void or_destroy(or_problem* P);

int64_t or_n(const or_problem* P);
void or_get_perm(const or_problem* P, int32_t* perm);
void or_get_codes(const or_problem* P, uint64_t* codes);          /* application order */
void or_get_geometry(const or_problem* P, double* centroid, double* area, double* h);
int64_t or_num_clusters(const or_problem* P);
/* clusters in pre-order: lo, hi, child0 (-1 for leaves), depth, bbox[6] (minx,miny,minz,maxx,maxy,maxz) */
void or_get_clusters(const or_problem* P, int32_t* lo, int32_t* hi, int32_t* child0,
                     int32_t* depth, double* bbox);
int64_t or_num_leaves(const or_problem* P, int kind /*0 adm, 1 dense*/);
void or_get_leaves(const or_problem* P, int kind, int32_t* quads /*4 per leaf*/);

/* Admissibility of two explicit boxes, squared form (A5). */
int or_admissible(const double* box_t, const double* box_s, double eta);

/* Gauss-Legendre rule on [0,1], n points ascending (long double Newton). */
void or_gauss_legendre01(int n, double* x, double* w);

/* Galerkin entries a_ij for application index pairs (P:224-228 read per A1,
 * rule set A14, arithmetic A15).  pairs: 2*n int64. */
void or_entries(const or_problem* P, int64_t n, const int64_t* pairs, double* out);
/* entry class: 0 identical, 1 common edge, 2 common vertex, 3+ regular with order (cls-3)?
 * returns: 0 identical, 1 edge, 2 vertex, 6/5/4/3 = regular Gauss order */
int or_entry_class(const or_problem* P, int64_t i, int64_t j);
/* Individual rules for explicit triangles (tests): */
double or_selfterm_closed(const double* v0, const double* v1, const double* v2);
/* Sauter-Schwab integral of 1/|x-y| over Tx x Ty, kind 0 identical (Tx==Ty),
 * 1 common edge (Tx=(A,B,Cx), Ty=(A,B,Cy)), 2 common vertex (Tx=(A,Bx,Cx), Ty=(A,By,Cy)). */
double or_sauter_schwab(int kind, const double* tx, const double* ty, int nq);
/* Sauter-Schwab on the reference pair with a user integrand g(x1,x2,y1,y2) = polynomial
 * prod  x1^a x2^b y1^c y2^d  (tests the measure preservation of the maps). */
double or_ss_reference_monomial(int kind, int nq, int a, int b, int c, int d);
/* Regular rule of order n of A14 (Radon's 7-point rule for n = 3, collapsed Gauss n x n
 * otherwise) for 1/|x-y| over two triangles (9 doubles each). */
double or_regular_rule(const double* tx, const double* ty, int n);
/* The per-triangle table of that rule in the (s, t) form of chi (reference area 1/2):
 * writes np <= 36 points and returns np. */
int or_rule_table(int n, double* s, double* t, double* w);

/* Dense rows of A (application indices) -> out[nrows*N]. */
void or_dense_rows(const or_problem* P, int64_t nrows, const int64_t* rows, double* out);

/* ACA with partial pivoting on block rows [rlo,rhi) x cols [clo,chi) (internal
 * indices), Frobenius stop (A11-A12).  U: m*kcap col-major, V: n*kcap col-major.
 * pivots: 2*kcap (row, col) local indices.  Returns k. */
int or_aca_block(const or_problem* P, int32_t rlo, int32_t rhi, int32_t clo, int32_t chi,
                 double eps, int kcap, double* U, double* V, int32_t* pivots);
/* ACA on an explicit matrix (tests: exact low rank). A row-major m x n. */
int or_aca_matrix(const double* A, int m, int n, double eps, int kcap,
                  double* U, double* V, int32_t* pivots);

/* Assemble the H-matrix for dense leaves [d0,d1) and admissible leaves [a0,a1)
 * (ranges of the canonical lists; a rank's sub-lists).
 * Returns 0 on success. */
int or_assemble(or_problem* P, double eps, int kcap, int64_t d0, int64_t d1,
                int64_t a0, int64_t a1);
/* The same for explicit ascending lists of dense / admissible leaf indices (timing samples
 * spread over the whole lists). */
int or_assemble_list(or_problem* P, double eps, int kcap, int64_t nd, const int64_t* dense_leaves,
                     int64_t na, const int64_t* adm_leaves);
/* Free the blocks of the last or_assemble (or_assemble itself frees them first). */
void or_release(or_problem* P);
int64_t or_stored_doubles(const or_problem* P);                /* dense + factor doubles */
int or_get_rank(const or_problem* P, int64_t adm_leaf);         /* -1 if not assembled */
void or_get_factors(const or_problem* P, int64_t adm_leaf, double* U, double* V);
void or_get_pivots(const or_problem* P, int64_t adm_leaf, int32_t* pivots);
void or_get_dense_block(const or_problem* P, int64_t dense_leaf, double* B);

/* H-matvec over the assembled leaves, application order. */
void or_matvec(const or_problem* P, const double* x, double* y);

/* Right-hand side f_i = int_{T_i} f (A16). kind 0: f = 1, kind 1: f = 4x^2-3y^2-z^2. */
void or_rhs(const or_problem* P, int kind, double* f);

/* Krylov solvers on or_matvec, x0 = 0 (A17).  Return iterations;
 * *relres = final true relative residual; *status 0 ok, 7 breakdown. */
int or_cg(const or_problem* P, const double* b, double* x, double tol, int maxit,
          double* relres, int* status);
int or_gmres(const or_problem* P, const double* b, double* x, double tol, int restart,
             int maxit, double* relres, int* status);

/* Leaf partition (A18): rank r of p owns leaves [out[r], out[r+1]). */
void or_partition(const int64_t* cost, int64_t n, int p, int64_t* out);

/* Single-layer potential (1/4pi) sum_j alpha_j int_{T_j} 1/|x-y| at M points X (M*3), alpha
 * in application order (A23); and one panel's integral with order n. */
void or_potential(const or_problem* P, const double* alpha, int64_t M, const double* X, double* out);
double or_panel_potential(const double* x, const double* tri, int n);

/* Work counters of the last or_assemble (kernel evaluations, entries). */
void or_counters(const or_problem* P, double* out /* [evals_near, evals_aca, entries_near, entries_aca] */);

#ifdef __cplusplus
}
#endif
#endif
