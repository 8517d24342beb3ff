/*
 * rrq.h -- C ABI of the B200 (sm_100a) recursive-reduction-quadrature near-correction builder.
 *
 * The library builds the sparse quadrature-correction matrix D_RRQ = D_near - D_smooth(near)
 * (eq dlpsplitting) for the Laplace layer potentials S, D, S', D'
 * (eqs slpdef..dprimelpdef) on a surface of curved triangular patches, by the scheme of
 * PAPER.md §4 (Steps 1-8) in matrix mode, with S / S' / D' per
 * P:L1527-1537.  The silent / garbled points of the paper are resolved as listed in DESIGN.md §2
 * (readings G1-G5, A1-A15); every kernel follows them.
 *
 * Conventions (all entry points):
 *  - Every array argument is a DEVICE pointer (cudaMalloc'd, e.g. a torch CUDA tensor) unless the
 *    comment says "host".  Arrays are caller-owned; the library never allocates caller-visible memory
 *    (it owns constant tables and internal scratch only, inside rrq_ctx).
 *  - Floating point is IEEE fp64; points/vectors are AoS xyz, row-major, C-contiguous.
 *  - Calls are asynchronous on the caller's cudaStream_t (0 = legacy default stream) unless stated.
 *  - Argument validation is synchronous and returns RRQ_ERR_INVALID_ARG with a message in
 *    rrq_last_error(); nothing throws across the ABI.  Kernel faults surface as RRQ_ERR_CUDA at the
 *    next call that synchronises.  Numerical trouble never aborts a batch: it is flagged per pair /
 *    per patch (status arrays) with the deterministic fallbacks of DESIGN.md §2.
 *  - Thread safety: one rrq_ctx per host thread (scratch is per context).
 */
#ifndef RRQ_H_
#define RRQ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *rrq_stream_t; /* == cudaStream_t */

typedef enum {
  RRQ_OK = 0,
  RRQ_ERR_INVALID_ARG = 1,
  RRQ_ERR_CUDA = 2,
  RRQ_ERR_CAPACITY = 3,
  RRQ_ERR_NOT_IMPLEMENTED = 4
} rrq_status;

/* kernel mask bits and flags */
enum { RRQ_S = 1, RRQ_D = 2, RRQ_SP = 4, RRQ_DP = 8, RRQ_ALL = 15, RRQ_RAW = 16 };

/* Discrete choices of the scheme:
 *  p        harmonic order; supported: 4, 6, 8, 10.
 *  n_nodes  nodes per patch, must be p*p (collapsed Gauss-Legendre, reading A1).
 *  p_edge   Gauss-Legendre nodes per edge p~; must be 2p (reading A4).
 *  n_omega  Gauss-Legendre nodes per side of the sinh-split Omega_0 rule (reading A9); 32.
 *  eta      near criterion |t - c_P| <= R_P + eta h_P (reading A6).
 *  rho_swap Bernstein-ellipse threshold rho0 of the swap regime (reading A5); 3.
 *  all_pairs if nonzero every (target, patch) pair is near (config 5). */
typedef struct {
  int32_t p, n_nodes, p_edge, n_omega;
  double eta, rho_swap;
  int32_t all_pairs;
} rrq_params;

typedef struct rrq_ctx_s *rrq_ctx;

/* Host call.  Builds the constant tables (Gauss-Legendre nodes, U = V^{-1} of P:L1239-1241 in
 * quad precision, sqrt-binomials of T_{jk,lm} P:L368-370) and uploads them.  Returns
 * RRQ_ERR_NOT_IMPLEMENTED for unsupported (p, p_edge).  *out is NULL on failure. */
rrq_status rrq_create(const rrq_params *params, rrq_ctx *out);
void rrq_destroy(rrq_ctx ctx);
/* Last error message of this context (or of the last failed rrq_create if ctx == NULL). */
const char *rrq_last_error(rrq_ctx ctx);

/* The discretised surface S = union of P patches ("Input/output").
 *  nodes   [P][n][3]   collocation / smooth-quadrature nodes of every patch
 *  normals [P][n][3]   unit outward normals at the nodes
 *  weights [P][n]      smooth quadrature weights including the Jacobian
 *  verts   [P][3][3]   patch vertices, counter-clockwise about the outward normal
 *  edge_x  [P][3][q][3] samples of edge e (verts[e] -> verts[(e+1)%3]) at the q Gauss-Legendre
 *                       parameters t_k in (-1,1) (ascending), q = p_edge
 *  edge_dx [P][3][q][3] d x / d t at the same parameters */
typedef struct {
  int64_t n_patches;
  const double *nodes, *normals, *weights, *verts, *edge_x, *edge_dx;
} rrq_surface;

/* Targets r'.
 *  x         [T][3]
 *  normal    [T][3] target normal nu' (needed for S', D'), or NULL (then S'/D' are invalid)
 *  self_node [T] global node id (patch*n + local) if the target IS that node, else -1; or NULL
 *  side      [T] +1 exterior (+nu side), -1 interior, 0 on-surface; or NULL (inferred, A8) */
typedef struct {
  int64_t n_targets;
  const double *x, *normal;
  const int64_t *self_node;
  const int8_t *side;
} rrq_targets;

/* Near list (reading A6): pairs (t, P) with |x_t - c_P| <= R_P + eta h_P, plus the
 * self patch, in target order with patches ascending.  Two-phase: with pair_patch == NULL the call
 * writes the exclusive-scanned counts to pair_ptr[0..T] (device) and the total to *n_pairs (host;
 * the call synchronises the stream); with pair_patch != NULL (capacity *n_pairs) it fills the
 * patch ids.  pair_ptr int64 [T+1], pair_patch int32 [n_pairs]. */
rrq_status rrq_near_list(rrq_ctx ctx, const rrq_surface *surf, const rrq_targets *tgt, int64_t *pair_ptr,
                         int32_t *pair_patch, int64_t *n_pairs, rrq_stream_t stream);

/* Bytes of the per-patch block written by rrq_patch_fit (frame, edge geometry, Step-3 edge
 * tables, fit operators P_D, P_Sp, P_Sd, P_Sg), for n_patches patches. */
size_t rrq_fit_bytes(rrq_ctx ctx, int64_t n_patches);

/* Steps 1-3 per patch in matrix mode (reading A1): local frame (A2),
 * harmonic gradients at the nodes, least-squares pseudo-inverse of the 4n x 4n_p quaternion system
 * and of the n x n_p scalar system by Householder QR, the S fit
 * P_Sg = P_D Hm P_Sd, the S' operator, and the edge tables
 * Hess S^{(j,k)} tau, grad S^{(j,k)} x tau at the 3 p_edge edge nodes.  fit: device buffer of
 * rrq_fit_bytes() bytes.  patch_status [P] (or NULL): 0 ok, 1 rank-deficient fit. */
rrq_status rrq_patch_fit(rrq_ctx ctx, const rrq_surface *surf, void *fit, int32_t *patch_status,
                         rrq_stream_t stream);

/* Steps 4-8 for every pair of rows [row_begin, row_end) (row chunking), P:L1448-1509 for S, D, S',
 * D' per kernel_mask (RRQ_S|RRQ_D|RRQ_SP|RRQ_DP; RRQ_RAW skips the smooth-rule subtraction of
 * reading A14 and returns the near rows themselves).  Outputs are CSR restricted to the chunk:
 * with base = pair_ptr[row_begin] (read from device; the call synchronises once to read it),
 *   row_ptr [row_end-row_begin+1]  int64   row_ptr[i] = (pair_ptr[row_begin+i] - base) * n
 *   col_idx [(pair_ptr[row_end]-base) * n] int32  global node id patch*n + local (or NULL)
 *   vals[k] same length, fp64, k = 0..3 for S, D, S', D' (NULL entries are skipped)
 *   pair_status [pairs of the chunk] int32 or NULL: bit0 Newton fallback on some edge, bit1
 *               nonfinite weight.
 * fit is the buffer written by rrq_patch_fit.  Nodes of a row are in patch-local order, patches
 * ascending.  Weights are in global units (S rows scale with h_P, D' rows with 1/h_P).
 * Alignment: surf->nodes, normals, weights and vals[k] 16-byte aligned, col_idx 8-byte aligned
 * (RRQ_ERR_INVALID_ARG otherwise); cudaMalloc / torch allocations satisfy this. */
rrq_status rrq_build_correction(rrq_ctx ctx, const rrq_surface *surf, const rrq_targets *tgt,
                                const int64_t *pair_ptr, const int32_t *pair_patch, int64_t n_pairs,
                                int64_t row_begin, int64_t row_end, const void *fit, uint32_t kernel_mask,
                                int64_t *row_ptr, int32_t *col_idx, double *const vals[4], int32_t *pair_status,
                                rrq_stream_t stream);

/* y[i] += sum_k vals[k] * density[col_idx[k]] over row i's entries (CSR SpMV).
 * row_ptr [n_rows+1] int64, col_idx int32, vals fp64, density [N_nodes], y [n_rows]. */
rrq_status rrq_apply_correction(rrq_ctx ctx, int64_t n_rows, const int64_t *row_ptr, const int32_t *col_idx,
                                const double *vals, const double *density, double *y, rrq_stream_t stream);

/* y[t] += alpha S_smooth[density](x_t) + beta D_smooth[density](x_t): the smooth rule of the splitting
 * over all surface nodes j except self_node[t] (reading A14),
 *   S_smooth = sum_j w_j density_j / (4 pi |x_t - x_j|),  D_smooth = sum_j w_j density_j (x_t - x_j).n_j / (4 pi |x_t - x_j|^3),
 * so that smooth + correction (rrq_apply_correction) is the discretised operator (used by the
 * combined-field solve).  Direct sum, O(n_targets x nodes) (no FMM).  tx [n_targets][3] and
 * self_node [n_targets] (or NULL) device arrays; density [nodes], y [n_targets] device fp64 (y accumulated). */
rrq_status rrq_apply_smooth(rrq_ctx ctx, int64_t n_targets, const double *tx, const int64_t *self_node,
                            const rrq_surface *surf, double alpha, double beta, const double *density, double *y,
                            rrq_stream_t stream);

/* Test hook: copy the host-built constant tables (GL nodes t[q], weights w[q], U[q][q] row-major)
 * into HOST arrays.  Lets tests check they are bit-identical to the oracle's. */
rrq_status rrq_get_tables(rrq_ctx ctx, double *t, double *w, double *U);

/* Number of kernel launches issued by this context since creation (host counter). */
int64_t rrq_launch_count(rrq_ctx ctx);

/* Device-time accounting.  When enabled, every launch of the build is bracketed by CUDA events
 * recorded on the stream it runs on; rrq_get_timing returns the accumulated milliseconds and launch
 * counts per stage: [0] near list, [1] patch fit (geometry, edge tables, QR), [2] k_pair_setup +
 * k_newton + k_edge_lines + k_target_gamma (Steps 4-5, scalar line integrals, I[gamma]; [8], [9], [10] = the
 * shares of k_newton, k_edge_lines, k_target_gamma), [3] k_qmap (Step 6 line-integral maps,
 * DMMA GEMM), [4] k_translate (Step 7), [5] k_contract (Step 8 DMMA GEMMs + smooth subtraction +
 * store), [6] build plumbing (pair permutation, work items), [7] whole rrq_build_correction calls
 * (caller's stream).  rrq_build_correction runs stage [2] of sub-chunk i+1 on an internal stream
 * concurrently with stages [3]-[5] of sub-chunk i (unless the environment sets RRQ_NO_OVERLAP=1),
 * so stages [2]-[6] may overlap; [7] is the build's device time.  The build works in sub-chunks of
 * whole patches (or tile ranges of one patch) within a scratch budget of 24 GB (RRQ_SCRATCH_BYTES
 * overrides it; a test hook).  stats[0] = pairs built, stats[1] =
 * swap-regime edges (reading A5).  The build synchronises the stream before the events are read. */
#define RRQ_NSTAGES 11
rrq_status rrq_set_timing(rrq_ctx ctx, int enable);
rrq_status rrq_get_timing(rrq_ctx ctx, double ms[RRQ_NSTAGES], int64_t launches[RRQ_NSTAGES], int64_t stats[2]);
rrq_status rrq_reset_timing(rrq_ctx ctx);

/* Producer/consumer overlap of rrq_build_correction (see above) on (1, the default unless the environment
 * sets RRQ_NO_OVERLAP=1) or off (0: every kernel on the caller's stream, so stages [2]-[5] are the
 * kernels' own device times).  Results are bit-identical either way. */
rrq_status rrq_set_overlap(rrq_ctx ctx, int enable);

/* Test hook: copy the internal per-pair contraction vectors of the LAST build sub-chunk to HOST
 * arrays: perm[i] = global pair id of row i, Z[i][13 n_p] = (Theta, zeta(W), zeta(dW), zeta_S) in
 * c-layout.  At most max_pairs rows; returns the row count in *n_out. */
rrq_status rrq_debug_zeta(rrq_ctx ctx, int64_t max_pairs, int64_t *perm, double *Z, int64_t *n_out);

/* Host-only self-test (no device needed): decodes k_translate's packed schedule for order p (4..14, even) the way
 * the kernel does and checks that every output W^{(l,m)} receives exactly the terms Q^{(j,k)} S'^{(l-j,m-k)} of the
 * direct translation (reading G4), each once, with the conjugate-symmetry sign flags.  Returns 0 when
 * the schedule is correct, a positive code naming the failed check otherwise, -1 for an unsupported p. */
int rrq_selftest_translate_schedule(int p);

/* Profiling hook: SM cycles spent by k_edge_lines in each of its steps ([0] pair load + swap-edge list,
 * [1] model integrals + Omega_0 sinh rule, [2] weights), summed over CTAs, into HOST out[8]; reset if set. */
rrq_status rrq_debug_phase_cycles(rrq_ctx ctx, uint64_t out[8], int reset);

/* Profiling hook: SM cycles spent by k_patch_fit_q in its phases (node tables, quaternion QR, Q^H e_c,
 * quaternion back substitution, real QR, Q_B^T e_c, real back substitution, P_Sg), summed over CTAs,
 * into HOST out[8]; reset if set. */
rrq_status rrq_debug_fit_cycles(rrq_ctx ctx, uint64_t out[8], int reset);

#ifdef __cplusplus
}
#endif
#endif /* RRQ_H_ */
