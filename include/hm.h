/*
 * hm.h — C ABI of libhm, a B200-native (sm_100a) implementation of the data-parallel
 * hot path of Harbrecht & Zaspel, "A scalable H-matrix approach for the solution of
 * boundary integral equations on multi-GPU clusters", arXiv 1806.11558.
 *
 * Citations: "P:n" = line n of the paper text (/root/reference/PAPER.md at build time);
 * "A#" = a reading of an ambiguous passage, listed in DESIGN.md §3.
 *
 * The path:
 *   hm_build_tree  panel geometry, Morton codes + stable sort, cardinality-based cluster
 *                  tree, bounding boxes, level-wise block-cluster-tree traversal
 *                  (Algorithm 1), leaf partition
 *   hm_setup       batched near-field Galerkin assembly and batched
 *                  adaptive cross approximation of the rank's leaves
 *   hm_matvec      batched H-matrix-vector product + global sum
 *   hm_solve       CG or GMRES(m) driving hm_matvec
 *
 * Conventions shared by every entry point
 *   - Return value: hm_status.  On any non-HM_OK return, hm_last_error(ctx) holds a
 *     one-line message; the context stays valid unless the status is HM_ERR_CUDA
 *     (a sticky device error), after which only hm_destroy is meaningful.
 *   - Ordering: unknown i is triangle i of the mesh passed to hm_build_tree
 *     ("application order").  The library's internal Morton order is visible
 *     only through hm_get_perm and the leaf quadruples of hm_get_leaves.
 *   - Pointers: every vector argument (x, y, rhs, sol, f) may be a DEVICE pointer on the
 *     context's device or a HOST pointer (pageable or pinned); the library detects which
 *     with cudaPointerGetAttributes.  Host vectors are staged through library-owned
 *     device buffers and the call returns only after the result is back in host memory.
 *     Device vectors are read/written in stream order on the context stream.
 *   - Ownership: all inputs are caller-owned and never retained after return; all tree,
 *     leaf, factor and workspace storage is library-owned and released by hm_destroy.
 *   - Precision: IEEE binary64 throughout (the paper states none; BASELINE.json fixes FP64).
 *   - Multi-GPU: one context per process per GPU.  Calls marked COLLECTIVE
 *     must be made by every rank of the communicator, in the same order, with identical
 *     arguments (except the rank's own device buffers).
 */
#ifndef HM_H
#define HM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hm_ctx_s* hm_ctx;

typedef enum {
  HM_OK = 0,
  HM_ERR_ARG = 1,        /* invalid argument (see each function) */
  HM_ERR_STATE = 2,      /* call out of order (e.g. hm_setup before hm_build_tree) */
  HM_ERR_OOM = 3,        /* device or host allocation failed */
  HM_ERR_CUDA = 4,       /* CUDA runtime/driver error (sticky) */
  HM_ERR_NCCL = 5,       /* NCCL error */
  HM_ERR_NUMERIC = 6,    /* non-finite matrix entry or vector value */
  HM_ERR_BREAKDOWN = 7   /* Krylov breakdown (CG: p^T H p <= 0) */
} hm_status;

#define HM_NCCL_UNIQUE_ID_BYTES 128
#define HM_P2P_HANDLE_BYTES 64   /* a CUDA IPC memory handle */

/* Surface mesh of flat panels (nodes = element centres).
 * vertices: n_vertices*3 doubles, xyz row-major.  triangles: n_triangles*panel_vertices
 * int32, 0-based vertex ids; vertices must be deduplicated (singular-entry classification
 * compares ids).  panel_vertices: 3 (or 0) = triangles; 4 = planar quadrilaterals in cyclic
 * vertex order (the paper's cube), each evaluated as the triangles (q0,q1,q2) and
 * (q0,q2,q3) (A25); N = n_triangles panels either way.
 * memory: 0 = both arrays in host memory, 1 = both in device memory on the ctx device. */
typedef struct {
  const double* vertices;
  int64_t n_vertices;
  const int32_t* triangles;
  int64_t n_triangles;
  int memory;
  int panel_vertices;
} hm_mesh;

/* Create a context on CUDA device `device` for rank `rank` of `world_size` ranks.
 * nccl_unique_id: HM_NCCL_UNIQUE_ID_BYTES bytes of an ncclUniqueId made by
 * hm_nccl_unique_id on rank 0 and broadcast by the caller; NULL iff world_size == 1.
 * cuda_stream: a cudaStream_t on `device`, or NULL for a library-owned blocking stream (it
 * orders with the legacy default stream, so plain torch/cudaMemcpy users need no extra sync).
 * Errors: HM_ERR_ARG (rank/world/device out of range, id NULL with world_size > 1),
 * HM_ERR_CUDA, HM_ERR_NCCL.  COLLECTIVE when world_size > 1. */
hm_status hm_create(hm_ctx* out, int device, int rank, int world_size,
                    const void* nccl_unique_id, void* cuda_stream);
/* Fill `id_out` (HM_NCCL_UNIQUE_ID_BYTES bytes) with a fresh ncclUniqueId. */
hm_status hm_nccl_unique_id(void* id_out);
/* Release everything owned by the context.  Safe on NULL. */
hm_status hm_destroy(hm_ctx ctx);
/* Message of the last failing call on ctx (valid until the next call on ctx). */
const char* hm_last_error(hm_ctx ctx);

/* Options (hm_set_option / hm_get_option), numeric values:
 *   "k_max"        ACA rank cap per block (A11), default 64, 1..256; the fixed rank when
 *                  eps_aca = 0
 *   "solver"       0 = GMRES(restart) (BASELINE.json), 1 = CG; default 0
 *   "restart"      GMRES restart length m, default 100
 *   "max_iter"     Krylov iteration cap (total matvecs), default 10000
 *   "aca_chunk_mb" ACA workspace budget per chunk in MiB, default 32768, capped before every
 *                  chunk at 0.45 x (free device memory + current workspace)
 *   "aca_kws"      ACA workspace columns per block before the overflow re-run (blocks that
 *                  fill it restart with twice the columns, up to k_max), default 16
 *   "record_pivots" keep each block's ACA pivot sequence for hm_get_lowrank: 1 on, 0 off,
 *                  -1 (default) on iff N <= 25000
 *   "kernel_timing" 1: record CUDA events on the context stream around every launch of
 *                  each kernel family (near-field evaluation, ACA evaluation, other ACA,
 *                  matvec, Krylov BLAS-1); totals in hm_get_stats "kt"; setting it resets them
 *   "mv_kernel"    small-leaf matvec pipeline: 0 (default) two CTA rings per SM, 2 x 48 KiB
 *                  stages each; 1 one ring of 4 x 48 KiB stages; 2 two rings of 3 x 36 KiB;
 *                  3 two rings of 2 x 56 KiB; 4 two rings of 4 x 24 KiB; 5 two rings of
 *                  3 x 32 KiB.  Re-plans the matvec if set up.
 *   "mv_small_max" low-rank leaves up to this many bytes (default 16384) go through the
 *                  shared-memory pipeline, larger ones through the large-block kernels
 *   "mv_profile"   1: accumulate producer/consumer wait and work cycles of the CTA-ring
 *                  matvec (hm_get_stats "mv_prof_cycles"); diagnostic
 *   "mv_scramble"  1: DIAGNOSTIC ONLY, wrong products: spread the row bases of the CTA-ring
 *                  matvec's y atomics over y (measures same-address atomic contention)
 *   "mv_concurrent" 1 (default): the large low-rank matvec kernels run on a library side
 *                  stream beside the small-leaf pipeline (joined before hm_matvec returns its
 *                  stream order); 0: one stream
 *   "cost_model"   leaf cost of the partition over ranks (A18): 0 (default) dense leaves
 *                  |t||s|, admissible leaves (|t|+|s|) x 10 (~ stored bytes: balances the
 *                  matvec and, with the near field beside ACA, the setup); 2 dense leaves
 *                  weighted by kind (t = s 110, boxes touching 26, separated 10), admissible
 *                  leaves (|t|+|s| + 21) x 10 (best for a serial setup); 1 a size-dependent
 *                  rank estimate for admissible leaves.  Takes effect at hm_build_tree.
 *   "part_ranks", "part_rank"  DIAGNOSTIC (world_size 1 only): build rank part_rank's share of a
 *                  part_ranks-way partition (no collectives), to measure every rank's setup of
 *                  a p-GPU run on one GPU.  Takes effect at hm_build_tree.
 *   "aca_upd_occ"  CTAs per SM of the warp-per-block Frobenius-update kernel: 0 = 16 (64 registers),
 *                  1 = 24 (default, 40 registers), 2 = 32 (32 registers)
 *   "lr_f32"       1: hm_setup stores the ACA factors U, V in binary32 (each entry rounded once;
 *                  dense blocks, ACA itself and all matvec / Krylov arithmetic stay FP64: the
 *                  matvec widens the factors exactly before every FMA).  Halves the low-rank bytes
 *                  the matvec streams.  0 (default): FP64 factors.
 *                  Takes effect at the next hm_setup; hm_get_lowrank returns the widened values.
 *   "near_perf"    1 (default): near-field (dense-leaf) entries in perf mode: each
 *                  term w / |x - y| as w * rsqrt(d2), the hardware seed refined by one cubic
 *                  step, accumulated by FMA — within 1e-13 relative of the oracle's entries
 *                  (measured <= 8.1e-16); 0: parity mode (IEEE sqrt then IEEE division, no FMA in
 *                  the sums, as for the admissible entries, whose residuals steer the ACA pivots
 *                  and therefore always use parity mode).  Takes effect at the next hm_setup.
 *   "aca_perf"     1: the ACA row / column entries of orders 3 and 4 in the same perf mode —
 *                  NOT reading A15 (which keeps admissible entries bit-identical to the oracle so
 *                  that the ACA pivots coincide): measured identical rank and pivots on 99.9991%
 *                  (C2) / 99.9997% (C3) of the blocks, solutions within 6.3e-9 / 1.5e-9 of the
 *                  oracle's, C4 ACA evaluation -19%.  0 (default): parity mode.  Triangles only.
 *   "solve_comm"   sharded solve collectives: 0 NCCL (default), 1 libhm P2P kernels (requires
 *                  hm_p2p_import, which selects it).
 *   "setup_overlap" 1: hm_setup evaluates the near field on a least-priority stream from a
 *                  second host thread while ACA runs on a greatest-priority stream (results
 *                  bit-identical; 10-12% shorter setup at N = 1.57M), the default; 0: serial.  With
 *                  kernel timing on, "kt" "eval_union_ms" is the union of the two evaluation
 *                  families' intervals (their sum when serial)
 * Errors: HM_ERR_ARG for an unknown key or an out-of-range value. */
hm_status hm_set_option(hm_ctx ctx, const char* key, double value);
hm_status hm_get_option(hm_ctx ctx, const char* key, double* value);

/* Build the cluster tree and block cluster tree for `mesh` with
 * C_leaf = leaf_size and admissibility parameter eta (defaults of the paper:
 * 32 and 1.0), then split both leaf lists into world_size contiguous
 * cost-balanced sub-lists (A18).  The mesh is copied; the caller
 * may free it after return.  Replicated on every rank; no communication.
 * Re-calling invalidates a previous hm_setup.  Synchronous.
 * Errors: HM_ERR_ARG (leaf_size < 1, eta < 0 or not finite, n_triangles < 1 or > 2^30,
 * a vertex id out of range, a triangle of zero area), HM_ERR_OOM, HM_ERR_CUDA. */
hm_status hm_build_tree(hm_ctx ctx, const hm_mesh* mesh, int leaf_size, double eta);

/* Assemble this rank's part of the H-matrix: every owned non-admissible leaf is evaluated
 * densely, every owned admissible leaf is compressed by ACA with partial
 * pivoting and the relative Frobenius stop ||u_k|| ||v_k|| <= eps_aca ||S_k||_F (A11-A12).
 * eps_aca = 0 selects the paper's fixed-rank mode ("k" of P:447): no stop test,
 * every block runs to k = min(m, n, option k_max) unless its residual is exactly zero.
 * No communication.  Synchronous.
 * Errors: HM_ERR_STATE (no tree), HM_ERR_ARG (eps_aca < 0 or not finite), HM_ERR_OOM,
 * HM_ERR_NUMERIC (a non-finite stored value: the message names the first offending dense
 * leaf with the entry's internal row and column, or the first admissible leaf with a
 * non-finite ACA factor entry; every stored near-field entry and factor entry is checked),
 * HM_ERR_CUDA. */
hm_status hm_setup(hm_ctx ctx, double eps_aca);

/* y = H x, x and y of length N in application order (host or device pointers).
 * Each rank applies its own leaves; partial products are summed over all ranks
 * (ncclAllReduce), so every rank receives the full y.  COLLECTIVE.
 * Stream-ordered for device pointers; synchronous for host pointers.
 * Errors: HM_ERR_STATE (no setup), HM_ERR_ARG (NULL pointer or x == y), HM_ERR_CUDA,
 * HM_ERR_NCCL. */
hm_status hm_matvec(hm_ctx ctx, const double* x, double* y);

/* Solve H sol = rhs with x0 = 0, stopping at ||r||_2 <= tol ||rhs||_2 or after
 * "max_iter" matvecs.  Solver chosen by option "solver".  With world_size > 1 the Krylov
 * vectors are sharded by internal row range (rank r owns rows [r S, r S + n), S = ceil(N/p));
 * each matvec all-gathers x (ncclAllGather) and reduce-scatters the partial products
 * (ncclReduceScatter) — the volume of the paper's replicated vector + global sum, P:578-587 —
 * and dot products are all-reduced (ncclAllReduce), so all ranks take identical decisions;
 * rhs and sol are full-length on every rank (sol is all-gathered at the end).  After
 * hm_p2p_import (option "solve_comm" 1) the three collectives run as libhm kernels over NVLink
 * peer memory instead of NCCL (sums in rank order: identical scalars on all ranks).
 * COLLECTIVE.  Synchronous.
 * iters_out: matvecs performed (may be NULL); rel_residual_out: true relative residual
 * ||rhs - H sol|| / ||rhs|| after the last iteration (may be NULL).
 * Non-convergence within max_iter is NOT an error: HM_OK with *rel_residual_out > tol.
 * Errors: HM_ERR_STATE, HM_ERR_ARG (tol <= 0), HM_ERR_BREAKDOWN (CG), HM_ERR_CUDA,
 * HM_ERR_NCCL. */
hm_status hm_solve(hm_ctx ctx, const double* rhs, double* sol, double tol,
                   int* iters_out, double* rel_residual_out);

/* Peer-memory collectives for the sharded solve (the paper's per-product
 * global sum, and the solver's dot-product reductions).
 * hm_p2p_export: allocates this rank's exchange buffer (gathered x, partial y, dot-product
 * slots and flags; ~16 n_max bytes) for solves of up to n_max unknowns and writes its CUDA
 * IPC handle (HM_P2P_HANDLE_BYTES) to handle_out (host memory, caller-owned).  Once per
 * context.  Errors: HM_ERR_STATE (world_size < 2 or > 8, or already exported), HM_ERR_ARG
 * (n_max < 1 or NULL handle_out), HM_ERR_OOM, HM_ERR_CUDA.
 * hm_p2p_import: handles = world_size consecutive handles in rank order (host memory, as
 * exported by every rank and gathered by the caller, e.g. over the torch process group);
 * maps every peer's buffer (cudaIpcOpenMemHandle) and sets option "solve_comm" to 1: from now
 * on hm_solve's x all-gather, y reduce-scatter and dot-product all-reduce are libhm kernels
 * (P2P stores / loads over NVLink, flags with system-scope release / acquire) instead of
 * NCCL calls.  COLLECTIVE in the sense that every rank must import before any rank solves.
 * A solve with N > n_max fails with HM_ERR_STATE.  The buffers are unmapped / freed by
 * hm_destroy.  Errors: HM_ERR_STATE (not exported, or already imported), HM_ERR_ARG (NULL),
 * HM_ERR_CUDA (a peer buffer could not be mapped). */
hm_status hm_p2p_export(hm_ctx ctx, int64_t n_max, void* handle_out);
hm_status hm_p2p_import(hm_ctx ctx, const void* handles);

/* Right-hand side f_i = int_{T_i} f: kind 0 -> f = 1 (f_i = |T_i|);
 * kind 1 -> the paper's f(x) = 4x1^2 - 3x2^2 - x3^2, edge-midpoint rule (exact for
 * quadratics on flat triangles, A16).  f: length N, application order, host or device.
 * Errors: HM_ERR_STATE (no tree), HM_ERR_ARG. */
hm_status hm_assemble_rhs(hm_ctx ctx, int kind, double* f);

/* Single-layer potential of the density sol at m evaluation points (the paper's
 * accuracy metric evaluates it inside the domain):
 *   out[p] = (1/4pi) sum_j sol_j int_{T_j} 1/|x_p - y| dy,
 * each panel integral by the triangle rule of the regular entries on T_j alone (A14: Radon's
 * 7-point degree-5 rule for order 3, collapsed Gauss n x n for orders 4..6) with its order
 * from rho = |x_p - c_j| / h_j in the bands of A14 (reading A23); points must lie off the
 * surface.  Any m >= 0 (point tiles are launched in slices of at most 65535 x 8 points).  Direct sum over all N panels on every rank (collective-free).
 * sol: length N, application order; points: m*3 xyz row-major; out: length m; each host or
 * device.  Synchronous.  Errors: HM_ERR_STATE (no tree), HM_ERR_ARG. */
hm_status hm_potential(hm_ctx ctx, const double* sol, int64_t m, const double* points, double* out);

/* ---- introspection (host buffers) ---- */
/* perm[s] = application index of internal position s (length N). */
hm_status hm_get_perm(hm_ctx ctx, int32_t* perm);
/* kind 0 = admissible leaves, 1 = dense leaves, in canonical DFS order (A10).
 * *count = number of leaves; if quads != NULL it receives 4*count int32
 * (row_lo, row_hi, col_lo, col_hi) in internal indices, half-open.  owned_begin/end
 * (may be NULL): this rank's sub-list [begin, end). */
hm_status hm_get_leaves(hm_ctx ctx, int kind, int64_t* count, int32_t* quads,
                        int64_t* owned_begin, int64_t* owned_end);
/* Cluster tree: *count clusters; arrays (may be NULL) lo, hi (internal, half-open),
 * depth, bbox (6 doubles: min xyz, max xyz). */
hm_status hm_get_clusters(hm_ctx ctx, int64_t* count, int32_t* lo, int32_t* hi,
                          int32_t* depth, double* bbox);
/* Morton codes (application order, length N). */
hm_status hm_get_codes(hm_ctx ctx, uint64_t* codes);
/* Galerkin entries a_ij for n application-index pairs (2n int64, host) -> out (n, host),
 * evaluated by the same device code as setup.  Errors: HM_ERR_STATE, HM_ERR_ARG. */
hm_status hm_eval_entries(hm_ctx ctx, int64_t n, const int64_t* pairs, double* out);
/* Stored dense block of owned dense leaf `leaf` (m*n doubles, row-major). */
hm_status hm_get_dense_block(hm_ctx ctx, int64_t leaf, double* block);
/* Rank k of owned admissible leaf `leaf`; if U/V non-NULL they receive U (m*k) and
 * V (n*k), column-major (R = U V^T); if pivots non-NULL, 2k int32 (row, col)
 * local pivot indices in the order chosen. */
hm_status hm_get_lowrank(hm_ctx ctx, int64_t leaf, int32_t* k, double* U, double* V,
                         int32_t* pivots);
/* Gauss-Legendre table on [0,1] used by the device rules (n in 1..8). */
hm_status hm_quadrature_table(int n, double* nodes, double* weights);
/* JSON object with counts, bytes, per-phase device times (ms), kernel-evaluation counts,
 * rank histogram, partition bounds.  Writes at most buf_len bytes incl. the NUL.
 * Errors: HM_ERR_ARG if buf_len is too small (the message gives the needed size). */
hm_status hm_get_stats(hm_ctx ctx, char* json_buf, int64_t buf_len);

#ifdef __cplusplus
}
#endif
#endif /* HM_H */
