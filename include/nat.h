/*
 * nat.h — C ABI of libnat: the Helmholtz boundary-integral hot path of NAT
 * (arXiv 2506.06190) on NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = line n of the paper's LaTeX source; readings R-* are
 * listed in DESIGN.md §3.
 *
 * Conventions (every call):
 *  - Pointers are CUDA DEVICE pointers on the current device unless marked [host].
 *    Passing a host pointer where a device pointer is required -> NAT_ERR_INVALID_ARG.
 *  - Every buffer is caller-owned (torch tensors, contiguous).  The library never
 *    allocates device memory: calls that need scratch take (ws, ws_bytes) and have a
 *    *_workspace() size query; ws must be 256-byte aligned.
 *  - Layouts: coordinates are structure-of-arrays [3][n] float64 (x row, y row, z row);
 *    complex values are interleaved (re, im) pairs = torch complex128 ("c128") or
 *    complex64 ("c64").  Vectors handed to / returned by the library are c128; only
 *    stored matrices use the precision `nat_prec` selects.
 *  - Calls marked (async) only enqueue work on `stream`; calls marked (sync) return
 *    host-visible results and synchronise the stream.
 *  - Errors: negative status = no valid output, message in nat_last_error()
 *    (thread-local, valid until the next nat_* call on that thread).  There is no CPU
 *    fallback and no sign flipping at run time.
 *  - Not reentrant on the same stream for the same workspace; reentrant otherwise.
 */
#ifndef NAT_H
#define NAT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NAT_ABI_VERSION 2  /* 2: nat_bem_assemble takes nnz; nat_bem_mf.nnz */

typedef struct CUstream_st* nat_stream_t; /* == cudaStream_t (torch.cuda.Stream.cuda_stream) */

typedef enum {
  NAT_OK = 0,
  NAT_WARN_NOT_CONVERGED = 1, /* GMRES hit max_iter: best iterate written, converged = 0 */
  NAT_ERR_INVALID_ARG = -1,   /* null/host pointer, bad size/range, k < 0 or non-finite          */
  NAT_ERR_CUDA = -2,          /* CUDA runtime or launch error                                    */
  NAT_ERR_NCCL = -3,          /* NCCL error                                                      */
  NAT_ERR_SINGULAR = -4,      /* zero-area triangle, inward mesh, coincident MC samples          */
  NAT_ERR_NUMERIC = -5,       /* NaN/Inf in a residual norm                              */
  NAT_ERR_WORKSPACE = -6      /* ws_bytes smaller than the matching *_workspace() query          */
} nat_status;

typedef enum {
  NAT_FP32 = 0, /* fp32 kernel arithmetic, c64 stored matrices, fp64 tile/Krylov sums (R-prec) */
  NAT_FP64 = 1  /* fp64 arithmetic, c128 stored matrices                                      */
} nat_prec;

int nat_abi_version(void);
const char* nat_last_error(void);

/* Diagnostics (bench.py's roofline pass): CUDA events on the launching stream around the
 * main kernel of each category — 0: MC operator (a10), 1: MC right-hand side (a9),
 * 2: radiation (a11), 3: far assembly (a4), 4: the neural field's tensor-core products
 * (NEXT-4; "pairs" = flops 2 M N K).  Off by default (no events, no overhead).
 * nat_kernel_timer_enable resets the totals and switches the timer on/off;
 * nat_kernel_timer_read synchronises the recorded events and returns, for one category,
 * the summed kernel time, the algorithmic pair-evaluations of those launches and their
 * count (launches that returned at once because GMRES had already converged are not
 * counted).  Pairs are pair-evaluations x wavenumbers.  nat_kernel_timer_read_modes returns
 * the same totals restricted to the launches that evaluated n_modes wavenumbers per pair
 * (1..64; 0 = every launch, = nat_kernel_timer_read), for per-launch rooflines whose
 * shared work (r, 1/r, d.n) is amortised over n_modes.  [host] outputs;
 * NAT_ERR_INVALID_ARG for a category or n_modes out of range. */
void nat_kernel_timer_enable(int on);
nat_status nat_kernel_timer_read(int category, double* seconds, double* pairs, int64_t* launches);
nat_status nat_kernel_timer_read_modes(int category, int n_modes, double* seconds, double* pairs,
                                       int64_t* launches);

/* ---------------------------------------------------------------------------------
 * a1 — mesh preparation ("construct the scene and obtain its surface triangle
 * mesh"; reading R-geom).  Per triangle t with vertices (v1, v2, v3):
 *   e = (v2-v1) x (v3-v1);  area = |e|/2;  normal = e/|e|;  centroid = ((v1+v2)+v3)/3;
 *   diam = longest edge;  area_cdf = sequential fp64 prefix sum of area (no FMA
 *   contraction anywhere: these values decide integer results bit for bit).
 * Host scalars: total_area = area_cdf[n-1]; center = sum A_t c_t / total_area;
 * bound_radius = max over vertices |v - center|.
 * Errors: NAT_ERR_SINGULAR for a zero-area triangle or signed volume <= 0.
 * ------------------------------------------------------------------------------- */
typedef struct {
  int64_t n_vert, n_tri;
  const double* vxyz; /* [3][n_vert] metres                                           */
  const int32_t* tri; /* [3][n_tri] 0-based; CCW seen from outside => outward normals */
} nat_mesh;

typedef struct {
  int64_t n_tri;
  double* centroid; /* [3][n_tri] out */
  double* normal;   /* [3][n_tri] out */
  double* area;     /* [n_tri] out    */
  double* diam;     /* [n_tri] out    */
  double* area_cdf; /* [n_tri] out    */
  double total_area, center[3], bound_radius, volume; /* [host] out */
} nat_geom;

size_t nat_mesh_prepare_workspace(int64_t n_vert, int64_t n_tri);
nat_status nat_mesh_prepare(const nat_mesh* mesh, nat_geom* geom, void* ws, size_t ws_bytes,
                            nat_stream_t stream); /* (sync) */

/* ---------------------------------------------------------------------------------
 * Quadrature options (reading R-colloc / R-self).  All-zero fields => defaults.
 * ------------------------------------------------------------------------------- */
typedef struct {
  int far_pts;        /* 1 | 3 | 6 | 7 points on far pairs, default 3                       */
  int near_levels_S;  /* midpoint-subdivision levels x 7-pt rule, vertex-sharing pairs, def 3 */
  int near_levels_N;  /* same for close pairs, default 1                                     */
  double near_eta;    /* class N: |c_i - c_j| < near_eta * diam_j, default 4                 */
  int self_theta_pts; /* Gauss-Legendre points per edge of the polar self term, default 16   */
  int burton_miller;  /* NEXT-1: 0 = the CBIE (beta = 0, default); 1 = Eq. BM as printed with    */
                      /* beta = i/k (reading R-bm): A = 1/2 I - K - beta W,            */
                      /* b = -(V + beta K') g - (beta/2) g; needs k > 0                            */
  int galerkin;       /* NEXT-2: 0 = P0 centroid collocation (default); 1 = P0 Galerkin of the CBIE */
                      /* (reading R-galerkin): A_ij = 1/2 |T_i| delta_ij - int_Ti int_Tj  */
                      /* dG/dn_y, b_i = -sum_j int_Ti int_Tj G g_j; far pairs far_pts x far_pts     */
                      /* tensor points, class N (R7 x near_levels_N)^2 tensor points, class S and   */
                      /* self Sauter-Schwab (common vertex / edge / identical); near_levels_S and    */
                      /* self_theta_pts unused; not with burton_miller or the matrix-free operator  */
  int ss_order;       /* Gauss-Legendre points per cube dimension of Sauter-Schwab, default 4 (1..8) */
} nat_quad_opts;

/* ---------------------------------------------------------------------------------
 * a2 — near list ("adjacent or identical elements"; reading R-near) for rows
 * [row_begin, row_end).  Class 1 (S): shares a vertex index; class 2 (N): otherwise
 * |c_i - c_j| < eta diam_j (fp64, strict).  CSR, columns ascending.
 * nat_bem_near_count fills row_ptr[rows+1] (exclusive scan) and returns nnz; it
 * synchronises.  nat_bem_near_build then fills col[nnz], cls[nnz] (async).  Both take a
 * caller-owned device workspace of nat_bem_near_workspace(n_tri) bytes (tile bounding
 * boxes used to skip far source tiles); NAT_ERR_WORKSPACE when ws_bytes is smaller.
 * ------------------------------------------------------------------------------- */
size_t nat_bem_near_workspace(int64_t n_tri); /* bytes of ws for count / build (per-tile boxes) */
nat_status nat_bem_near_count(const nat_mesh* mesh, const nat_geom* geom, const nat_quad_opts* opts,
                              int64_t row_begin, int64_t row_end, int64_t* row_ptr,
                              int64_t* nnz /* [host] */, void* ws, size_t ws_bytes,
                              nat_stream_t stream); /* (sync) */
nat_status nat_bem_near_build(const nat_mesh* mesh, const nat_geom* geom, const nat_quad_opts* opts,
                              int64_t row_begin, int64_t row_end, const int64_t* row_ptr,
                              int32_t* col, uint8_t* cls, void* ws, size_t ws_bytes,
                              nat_stream_t stream); /* (async) */

/* ---------------------------------------------------------------------------------
 * a4 + a5 — dense collocation assembly of the conventional BIE (Eq. BM with beta = 0,
 * P:174-180; readings R-sign, R-colloc, R-self) for rows [row_begin, row_end):
 *   A[r][j] = 1/2 delta_ij - K_ij,   rhs[q][r] = - sum_j V_ij g[q][j],
 *   K_ij = int_{T_j} dG/dn_y(c_i, y) dS,  V_ij = int_{T_j} G(c_i, y) dS,  i = row_begin + r.
 * Far pairs use the far rule; pairs in the near list (rows of the CSR built for the
 * same row range) and the self pair are overwritten with the near/self rules and the
 * right-hand side is corrected in a fixed order (deterministic).
 * A: row-major [rows][lda], c64 (NAT_FP32) or c128 (NAT_FP64).  g: c128 [n_rhs][n_tri]
 * (may be NULL iff n_rhs == 0).  rhs: c128 [n_rhs][rows].  k >= 0 finite.
 * ------------------------------------------------------------------------------- */
/* nnz: the host value nat_bem_near_count returned (= near_row_ptr[rows]); the call never
 * reads the device copy back, so it is fully asynchronous (a wrong nnz is not detected).
 * The rule tables reach the workspace by one asynchronous copy from pinned host memory. */
size_t nat_bem_assemble_workspace(int64_t n_tri, int64_t rows, int64_t nnz, int n_rhs); /* nnz from near_count */
nat_status nat_bem_assemble(const nat_mesh* mesh, const nat_geom* geom, const nat_quad_opts* opts,
                            const int64_t* near_row_ptr, const int32_t* near_col,
                            const uint8_t* near_cls, int64_t nnz, double k, nat_prec prec, int64_t row_begin,
                            int64_t row_end, int n_rhs, const void* g, void* A, int64_t lda,
                            void* rhs, void* ws, size_t ws_bytes, nat_stream_t stream); /* (async) */

/* a4 + a5 for n_k wavenumbers on the same mesh and rows in one call (round 2): A[q] (host
 * array of n_k device matrices, [rows][lda] each) and rhs c128 [n_k][n_rhs][rows] are those
 * nat_bem_assemble writes for k[q].  NAT_FP32 collocation of the conventional BIE with
 * n_rhs <= 1 runs ONE far pass for all wavenumbers (shared geometry, rsqrt and d.n per
 * quadrature point; per wavenumber kr, sincos, the V / K sums and the store); other variants
 * loop over the wavenumbers.  1 <= n_k <= 4.  Workspace nat_bem_assemble_multi_workspace.  (async) */
size_t nat_bem_assemble_multi_workspace(int64_t n_tri, int64_t rows, int64_t nnz, int n_rhs, int n_k);
nat_status nat_bem_assemble_multi(const nat_mesh* mesh, const nat_geom* geom, const nat_quad_opts* opts,
                                  const int64_t* near_row_ptr, const int32_t* near_col, const uint8_t* near_cls,
                                  int64_t nnz, int n_k, const double* k /* [host] */, nat_prec prec, int64_t row_begin,
                                  int64_t row_end, int n_rhs, const void* g, void* const* A /* [host][n_k] */,
                                  int64_t lda, void* rhs, void* ws, size_t ws_bytes, nat_stream_t stream);

/* a6 — y = A x, A [rows][lda] in `prec`, x c128 [n], y c128 [rows]; fp64 accumulation
 * in a fixed per-row order (independent of the number of GPUs).                       */
nat_status nat_bem_matvec(nat_prec prec, int64_t rows, int64_t n, const void* A, int64_t lda,
                          const void* x, void* y, nat_stream_t stream); /* (async) */

/* ---------------------------------------------------------------------------------
 * Communicator for the row-sharded solve (NCCL over NVLink / NVSwitch).  Rank 0 calls
 * nat_comm_unique_id and broadcasts the 128 bytes (torch.distributed); every rank
 * then calls nat_comm_create_from_id.  A NULL communicator means world size 1.
 * ------------------------------------------------------------------------------- */
typedef struct nat_comm nat_comm;
nat_status nat_comm_unique_id(uint8_t* id /* [host] 128 B */);
nat_status nat_comm_create_from_id(nat_comm** comm, const uint8_t* id /* [host] 128 B */, int rank,
                                   int world);
/* Wraps a caller-owned ncclComm_t (void* to keep NCCL out of this header; e.g. the
 * communicator of torch.distributed's NCCL backend): its rank / size must equal
 * rank / world (checked, NAT_ERR_INVALID_ARG otherwise); NULL with world == 1 is a
 * single-rank communicator.  nat_comm_destroy never destroys a borrowed ncclComm_t. */
nat_status nat_comm_create(nat_comm** comm, void* nccl_comm /* borrowed ncclComm_t or NULL */, int rank,
                           int world);
nat_status nat_comm_destroy(nat_comm* comm); /* destroys the ncclComm_t only if the library made it */
/* Host-staged communicator (test backend, e.g. world > 1 on one GPU over a gloo group): each
 * in-place all-gather copies this rank's block (count doubles at buf + rank*count) to a
 * pinned host buffer owned by the communicator, synchronises the stream, calls
 * fn(user, host_buf, count, rank, world) — which must fill every rank's block of host_buf
 * (count * world doubles) and return 0 — and copies the buffer back (asynchronously).
 * No kernel waits on another rank.  Nonzero fn return -> NAT_ERR_NCCL. */
typedef int (*nat_allgather_fn)(void* user, double* host_buf, size_t count, int rank, int world);
nat_status nat_comm_create_host(nat_comm** comm, int rank, int world, nat_allgather_fn fn, void* user);

/* ---------------------------------------------------------------------------------
 * a7 — unrestarted GMRES (tol 1e-6, max 200; reading R-gmres) on the
 * row-sharded system: this rank owns rows [row_begin, row_end) of A (A_local, b_local);
 * each iteration = local matvec -> all-gather of the iterate (NCCL) -> replicated
 * Arnoldi (CGS2, deterministic reductions).  x0 = 0.  Row ownership is fixed:
 * rows_per_rank = ceil(n / world), row_begin = rank * rows_per_rank,
 * row_end = min(n, row_begin + rows_per_rank); comm == NULL means world = 1.  x: c128 [n] out, identical on
 * all ranks.  tol <= 0 => 1e-6, max_iter <= 0 => 200.  Returns NAT_OK or
 * NAT_WARN_NOT_CONVERGED; info->rel_residual is the true ||b - A x|| / ||b||.
 * ------------------------------------------------------------------------------- */
typedef struct {
  int iters, converged;
  double rel_residual; /* true ||b - A x|| / ||b||, formed by linearity from the operator
                          products saved during the iteration (b - sum_k y_k (A v_k); no extra
                          operator application; reading R-gmres)                               */
  double t_total_s;  /* host wall time of the call                                         */
  double t_matvec_s; /* device time (CUDA events) of the operator applications: matvec and,
                        on > 1 rank, the all-gather (bem_solve) / MC operator (mc)          */
  double t_comm_s;   /* host-side time spent enqueueing the all-gathers (info only)        */
} nat_solve_info;

size_t nat_bem_solve_workspace(nat_prec prec, int64_t n, int64_t rows_local, int max_iter);
nat_status nat_bem_solve(nat_comm* comm, nat_prec prec, int64_t n, int64_t row_begin, int64_t row_end,
                         const void* A_local, int64_t lda, const void* b_local, void* x, double tol,
                         int max_iter, void* ws, size_t ws_bytes, nat_solve_info* info /* [host] */,
                         nat_stream_t stream); /* (sync) */

/* ---------------------------------------------------------------------------------
 * NEXT-3 — matrix-free dense BEM operator for meshes whose stored matrix
 * does not fit (C5 on 1-2 GPUs: 199,692^2 x 16 B = 638 GB).  The operator is the same
 * A as nat_bem_assemble (P:174-191 with the rules of reading R-colloc), applied as
 *   (A x)_i = sum_j A^far_ij x_j + sum_{e in near(i)} delta_e x_col[e] + diag_i x_i,
 * where A^far_ij = -K^far_ij is the far rule on EVERY pair (re-evaluated per product,
 * nothing stored), delta_e = A_ij - A^far_ij on the near list and diag_i = A_ii -
 * A^far_ii.  Rows [row_begin, row_end) of one rank; the near list is the one
 * nat_bem_near_build made for the same rows and opts.  Burton-Miller is not supported.
 * near_delta: c128 [nnz], diag_delta: c128 [rows], caller-owned, written by
 * nat_bem_mf_prepare (which also forms rhs = -V g as nat_bem_assemble does, when
 * n_rhs > 0).  x: c128 [n_tri]; y: c128 [rows].  The far sums run in `prec` (fp32:
 * packed FP32x2 with per-CTA fp64 reductions; fp64), the partial sums and corrections
 * in fp64 in a fixed order (deterministic, independent of the row split).
 * Workspace: nat_bem_mf_workspace(op, nnz, n_rhs) bytes for prepare / matvec;
 * nat_bem_mf_solve_workspace(op, max_iter, world) for the solve.
 * ------------------------------------------------------------------------------- */
typedef struct {
  const nat_mesh* mesh;
  const nat_geom* geom;
  const nat_quad_opts* opts;   /* NULL => defaults; burton_miller must be 0         */
  double k;
  nat_prec prec;
  int64_t row_begin, row_end;
  const int64_t* near_row_ptr; /* [rows + 1]                                        */
  const int32_t* near_col;     /* [nnz]                                             */
  const uint8_t* near_cls;     /* [nnz]                                             */
  int64_t nnz;                 /* [host] near_row_ptr[rows] (nat_bem_near_count)    */
  void* near_delta;            /* [nnz] c128 (prepare writes, matvec reads)          */
  void* diag_delta;            /* [rows] c128                                        */
} nat_bem_mf;
size_t nat_bem_mf_workspace(const nat_bem_mf* op, int64_t nnz, int n_rhs);
nat_status nat_bem_mf_prepare(const nat_bem_mf* op, int n_rhs, const void* g, void* rhs, void* ws,
                              size_t ws_bytes, nat_stream_t stream); /* (async) */
nat_status nat_bem_mf_matvec(const nat_bem_mf* op, const void* x, void* y, void* ws, size_t ws_bytes,
                             nat_stream_t stream); /* (async) */
/* GMRES (as nat_bem_solve: same row ownership, all-gather, tolerances and info) over the
 * matrix-free operator; x c128 [n_tri] identical on all ranks.  (sync)                  */
size_t nat_bem_mf_solve_workspace(const nat_bem_mf* op, int max_iter, int world);
nat_status nat_bem_mf_solve(nat_comm* comm, const nat_bem_mf* op, const void* b_local, void* x, double tol,
                            int max_iter, void* ws, size_t ws_bytes, nat_solve_info* info /* [host] */,
                            nat_stream_t stream);

/* ---------------------------------------------------------------------------------
 * (b) Monte-Carlo BEM (Eq. BIE / SYS; disk terms P:215-236; readings
 * R-mc-sample, R-eps, R-weight, R-disk).
 *
 * a8  nat_mc_sample: sample j = Philox4x32-10(ctr (j, 0, stream_lo, stream_hi),
 *     key seed) -> triangle by area CDF (upper bound) -> uniform barycentric point;
 *     samples [6][M] float64 = (x, y, z, nx, ny, nz) rows; sample_tri [M] int32.
 *     Bit-identical with the oracle.  (async)
 * a9  nat_mc_rhs: b[m][i] = -w sum_{j != i} G_m(y_i, y_j) g[m][j] - (eps/2) g[m][i].
 * a10 nat_mc_apply: out[m][i] = 1/2 p[m][i] - w sum_{j != i} dG_m/dn_y(y_i, y_j) p[m][j].
 *     The library derives eps and w from total_area = |Gamma| (nat_mesh_prepare) and M:
 *     eps = sqrt(|Gamma| / (pi M)) unless eps > 0 is given (R-eps), and
 *     w = (|Gamma| - pi eps^2)/(M - 1) (R-weight; w = 0 for M = 1);
 *     NAT_ERR_INVALID_ARG for total_area <= 0 or pi eps^2 > |Gamma|.
 *     k [host][n_sys];  g, p, b, out c128 [n_sys][M].
 *     NAT_FP32: sample pairs closer than 2 eps (the disk diameter) are evaluated in fp64
 *     (their fp32 coordinates cannot resolve d.n); all other pairs in fp32.
 * nat_mc_surface_pressure: a8 (or caller samples) -> a9 -> batched GMRES over a10
 *     for all n_sys wavenumbers sharing one sample set; g_tri c128 [n_sys][n_tri].
 *     Errors: NAT_ERR_SINGULAR on coincident samples (|y_i - y_j| < 1e-12).
 * ------------------------------------------------------------------------------- */
typedef struct {
  int64_t M;
  uint64_t seed, stream_id;
  double eps;                 /* <= 0 => sqrt(|Gamma| / (pi M))        */
  const double* samples_in;   /* optional [6][M] (e.g. a host Poisson-disk set) */
  const int32_t* sample_tri_in; /* required with samples_in                     */
} nat_mc_opts;

nat_status nat_mc_sample(const nat_mesh* mesh, const nat_geom* geom, int64_t M, uint64_t seed,
                         uint64_t stream_id, double* samples, int32_t* sample_tri,
                         nat_stream_t stream); /* (async) */
size_t nat_mc_op_workspace(nat_prec prec, int64_t M, int n_sys);
nat_status nat_mc_rhs(nat_prec prec, int64_t M, const double* samples, int n_sys, const double* k,
                      const void* g, double total_area, double eps, void* b, void* ws, size_t ws_bytes,
                      nat_stream_t stream); /* (sync: builds the close-pair list) */
nat_status nat_mc_apply(nat_prec prec, int64_t M, const double* samples, int n_sys, const double* k,
                        const void* p, double total_area, double eps, void* out, void* ws, size_t ws_bytes,
                        nat_stream_t stream); /* (sync: builds the close-pair list) */
/* g_out[m][j] = g_tri[m][sample_tri[j]] (piecewise-constant Neumann data at the samples,
 * P:164; c128 [n_sys][n_tri] -> c128 [n_sys][M]).  (async)                              */
nat_status nat_mc_gather_neumann(int n_sys, int64_t M, int64_t n_tri, const void* g_tri,
                                 const int32_t* sample_tri, void* g_out, nat_stream_t stream);
nat_status nat_mc_check_coincident(int64_t M, const double* samples, int64_t* pair /* [host] 2 */,
                                   void* ws, size_t ws_bytes, nat_stream_t stream); /* (sync) */

size_t nat_mc_workspace(nat_prec prec, int64_t M, int n_sys, int max_iter);
/* Solve groups of nat_mc_surface_pressure (process-wide; default NAT_MC_GROUPS or 2): the
 * systems of each batch of <= 64 are split into `groups` contiguous groups whose GMRES
 * iterations run concurrently on their own streams from persistent library threads, so one
 * group's Krylov steps overlap another's operator application.  Each system's iteration is
 * the same arithmetic in any group (results agree to the launch shapes' rounding; the tests
 * compare group counts 1, 2, 4).  nat_mc_workspace covers every group count.  groups in
 * [1, 4], else NAT_ERR_INVALID_ARG. */
nat_status nat_mc_set_groups(int groups);
/* Shape of the fused Arnoldi step of the batched GMRES (a7; process-wide, applies to the
 * solves that start afterwards): cluster_ctas CTAs per system (2, 4, 8; 2 only with the
 * fp32 basis, else 4), threads per CTA (256 — fp32 basis only —, 512, 768) and the
 * shared-memory residency cap in KB (0 = none; default 120 = one CTA per SM).  Defaults:
 * NAT_FUSED_CL / NAT_FUSED_NTH / NAT_FUSED_SMEM_KB, else (4, 512, 120).  The narrow shapes
 * let the step's clusters co-reside with other streams' kernels (the C4 sweep); the wide
 * default is fastest for one solve alone.  Invalid values: NAT_ERR_INVALID_ARG.        */
nat_status nat_krylov_config(int cluster_ctas, int threads, int smem_cap_kb);
nat_status nat_mc_surface_pressure(const nat_mesh* mesh, const nat_geom* geom, int n_sys,
                                   const double* k /* [host] */, const void* g_tri, const nat_mc_opts* opts,
                                   nat_prec prec, double tol, int max_iter, double* samples_out,
                                   int32_t* sample_tri_out, void* p_out, void* ws, size_t ws_bytes,
                                   nat_solve_info* info /* [host][n_sys] */,
                                   nat_stream_t stream); /* (sync) */

/* Rows [row_begin, row_end) of the a10 operator (row sharding; SURVEY §8(e) "MC, one large
 * system"), eps and w derived as for nat_mc_apply:
 * out[m][r] = 1/2 p[m][i] - w sum_{j != i} dG_m/dn_y(y_i, y_j) p[m][j],
 * i = row_begin + r; p c128 [n_sys][M] (all rows), out c128 [n_sys][rows]; n_sys <= 64.
 * Workspace nat_mc_rows_workspace(prec, M, n_sys, rows).  (sync: builds the close-pair list) */
size_t nat_mc_rows_workspace(nat_prec prec, int64_t M, int n_sys, int64_t rows);
nat_status nat_mc_apply_rows(nat_prec prec, int64_t M, const double* samples, int n_sys, const double* k /* [host] */,
                             const void* p, double total_area, double eps, int64_t row_begin, int64_t row_end,
                             void* out, void* ws, size_t ws_bytes, nat_stream_t stream);
/* nat_mc_surface_pressure row-sharded across the ranks of `comm` (NULL => world 1): rank r
 * owns sample rows [r ceil(M/world), ...) of the RHS and the operator; every operator
 * application is followed by an in-place NCCL all-gather of each system's iterate and the
 * Arnoldi process is replicated (identical on all ranks).  Every rank regenerates the same
 * Philox sample set.  Outputs (samples, p_out [n_sys][M], info) identical on all ranks.
 * M >= 2.  Workspace nat_mc_sharded_workspace(prec, M, n_sys, max_iter, world).  (sync) */
size_t nat_mc_sharded_workspace(nat_prec prec, int64_t M, int n_sys, int max_iter, int world);
nat_status nat_mc_surface_pressure_sharded(nat_comm* comm, const nat_mesh* mesh, const nat_geom* geom, int n_sys,
                                           const double* k /* [host] */, const void* g_tri,
                                           const nat_mc_opts* opts, nat_prec prec, double tol, int max_iter,
                                           double* samples_out, int32_t* sample_tri_out, void* p_out, void* ws,
                                           size_t ws_bytes, nat_solve_info* info /* [host][n_sys] */,
                                           nat_stream_t stream);

/* ---------------------------------------------------------------------------------
 * (c) radiation to listeners (reading R-ext):
 *   p[m][l] = sum_s w_s [ p[m][s] dG_m/dn_y(x_l, y_s) - g[m][s] G_m(x_l, y_s) ].
 * ------------------------------------------------------------------------------- */
typedef struct {
  int64_t n_src;
  const double* xyz; /* [3][n_src]                       */
  const double* nrm; /* [3][n_src] unit normals          */
  const double* w;   /* [n_src] quadrature / MC weights  */
  int n_modes;
  const void* p;     /* c128 [n_modes][n_src] Dirichlet  */
  const void* g;     /* c128 [n_modes][n_src] Neumann    */
  double center[3];  /* [host] coordinate origin used for the fp32 cast (mesh centre) */
} nat_sources;

/* BEM solution -> sources: the q_rad (1|3|6|7) rule points of every triangle,
 * w = omega_q A_t, normal n_t, values p_t, g_t (c128 [n_modes][n_tri] in,
 * [n_modes][n_tri*q_rad] out; point index t*q_rad + q).                                */
nat_status nat_bem_sources(const nat_mesh* mesh, const nat_geom* geom, int q_rad, int n_modes,
                           const void* p_tri, const void* g_tri, double* xyz, double* nrm, double* w,
                           void* p_src, void* g_src, nat_stream_t stream); /* (async) */
/* MC solution -> sources: xyz/nrm rows of samples, w = total_area / M.               */
nat_status nat_mc_sources(int64_t M, const double* samples, double total_area, double* xyz,
                          double* nrm, double* w, nat_stream_t stream); /* (async) */

size_t nat_radiate_workspace(nat_prec prec, int64_t n_src, int n_modes, int64_t n_lis);
nat_status nat_radiate_field(const nat_sources* src, nat_prec prec, const double* k /* [host][n_modes] */,
                             int64_t n_lis, const double* lis_xyz /* [3][n_lis] */,
                             void* p_out /* c128 [n_modes][n_lis] */, void* ws, size_t ws_bytes,
                             nat_stream_t stream); /* (async) */

/* ---------------------------------------------------------------------------------
 * a12 — listener shell grid (reading R-listen): point ((w n_phi)+v) n_theta + u,
 *   theta_u = -pi + (u+1/2) 2pi/n_theta, phi_v = (v+1/2) pi/n_phi,
 *   r_w = R (r_lo + (r_hi - r_lo)(w+1/2)/n_r), x = center + r (sin phi cos theta,
 *   sin phi sin theta, cos phi).  out: [3][n_theta n_phi n_r] float64.
 * ------------------------------------------------------------------------------- */
nat_status nat_listener_grid(const double* center /* [host] 3 */, double R, int n_theta, int n_phi,
                             int n_r, double r_lo, double r_hi, double* out,
                             nat_stream_t stream); /* (async) */

/* NEXT-3 — Poisson-disk boundary samples ("parallel Poisson disk sampling";
 * reading R-poisson): phase-group dart throwing over 30 M_target candidates (the a8
 * construction with Philox tag 2), minimum distance r (r <= 0 => 0.7 sqrt(|Gamma| / M_target)),
 * cells of size r / sqrt(3) over geom->center +- geom->bound_radius.  Writes M samples,
 * ascending by candidate index, to samples_out [6][M] (xyz, normal; stride M) and
 * sample_tri_out [M]; *M_out = M, *r_out = r (optional).  Synchronous (M is a host output).
 * NAT_ERR_WORKSPACE when ws_bytes < nat_mc_poisson_workspace(...) or M > cap (M_out is
 * still set); NAT_ERR_INVALID_ARG for M_target < 1, a grid over 1280^3 cells or bad
 * pointers.  The samples feed nat_mc_surface_pressure through opts->samples_in.           */
size_t nat_mc_poisson_workspace(const nat_geom* geom, int64_t M_target, double r);
nat_status nat_mc_poisson_sample(const nat_mesh* mesh, const nat_geom* geom, int64_t M_target, double r,
                                 uint64_t seed, uint64_t stream_id, double* samples_out, int32_t* sample_tri_out,
                                 int64_t cap, int64_t* M_out /* [host] */, double* r_out /* [host] or NULL */,
                                 void* ws, size_t ws_bytes, nat_stream_t stream); /* (sync) */

/* a12 (optional form, "randomly sample theta, phi, and r within an enclosing
 * sphere"; reading R-listen-rand): n points uniform in the volume of the shell
 * R r_lo <= |x - center| <= R r_hi.  Point t: Philox4x32-10 counter (t, 1, stream_lo,
 * stream_hi), key = seed, u_a = (o_a + 1/2) 2^-32; cos(phi) = 1 - 2 u0,
 * sin(phi) = 2 sqrt(u0 (1 - u0)), theta = -pi + 2 pi u1, r = R cbrt(r_lo^3 + u2 (r_hi^3 - r_lo^3)).
 * out: [3][n] fp64 SoA (caller-owned device buffer).  Async.  NAT_ERR_INVALID_ARG for
 * n < 1, R <= 0, r_lo <= 0, r_hi < r_lo or a host / null out.                            */
nat_status nat_listener_random_shell(const double* center /* [host] 3 */, double R, int64_t n, double r_lo,
                                     double r_hi, uint64_t seed, uint64_t stream_id, double* out,
                                     nat_stream_t stream); /* (async) */

/* ---------------------------------------------------------------------------------
 * NEXT-4 — the NAT neural acoustic transfer field (reading R-nf):
 *   Phi(x, v) = MLP[ G(x) ; P(v) ],  x = (theta^, phi^, r^) in [0,1]^3, v in [0,1]^n_v;
 *   G: 4 feature lattices over x, resolutions 8, 16, 32, 64, 4 features per vertex,
 *      trilinear interpolation (dense tables: (N+1)^3 <= 2^19 rows; instant-NGP hash above);
 *   P: sin / cos(2^k pi v_d), k = 0..5;  input = [G (16) ; P (12 n_v) ; 0] padded to 64;
 *   MLP 64 -> 128 -> 128 -> 128 -> 128 -> n_out, ReLU after the hidden layers;
 *   loss = mean squared error (l.124); Adam (beta 0.9 / 0.999, eps 1e-8, bias-corrected).
 * Parameters: one fp32 vector in the order grid0..grid3 [rows][4], then per layer W [out][in]
 * (row-major) and b [out].  Every layer product runs on the tcgen05 tensor cores with bf16
 * operands (activations, weights, gradients) and fp32 accumulation; everything else fp32.
 * inputs: fp32 [n][3 + n_v]; targets, out: fp32 [n][n_out].  n_v <= 4, 1 <= n_out <= 16.
 * ------------------------------------------------------------------------------- */
typedef struct {
  int n_v;    /* condition variables (C4: height, size, material = 3) */
  int n_out;  /* outputs (C4: |p| of the 8 modes)                      */
} nat_nf_config;
int64_t nat_nf_param_count(const nat_nf_config* cfg);     /* -1 for an invalid cfg        */
size_t nat_nf_workspace(const nat_nf_config* cfg, int64_t n);
nat_status nat_nf_forward(const nat_nf_config* cfg, const float* params, int64_t n, const float* inputs,
                          float* out, void* ws, size_t ws_bytes, nat_stream_t stream); /* (async) */
/* forward, MSE, backward, Adam (in place on params, adam_m, adam_v; step >= 1 counts Adam
 * steps); loss: device fp32 [1] (the loss before the update); grad_out: optional device
 * fp32 [param_count] (the gradient).  (async) */
nat_status nat_nf_train_step(const nat_nf_config* cfg, float* params, float* adam_m, float* adam_v, int step,
                             float lr, int64_t n, const float* inputs, const float* targets, float* loss,
                             float* grad_out, void* ws, size_t ws_bytes, nat_stream_t stream);
/* The layers' tensor-core product alone: C (fp32 [M][ldc]) = A B^T with A bf16 [M][K]
 * (a_mn = 0) or [K][M] (a_mn = 1), B bf16 [N][K] (b_mn = 0) or [K][N] (b_mn = 1);
 * N in {16, 32, 64, 128}; lda, ldb multiples of 8.  (async) */
nat_status nat_nf_gemm_bf16(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int a_mn, const void* B,
                            int64_t ldb, int b_mn, float* C, int64_t ldc, nat_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* NAT_H */
