/*
 * emhd.h — C ABI of the B200-native EpiRK/Krylov hot path (libemhd.so).
 *
 * The reference (arxiv/paper_1604_02614, package `expmhd`) is pure Python:
 * its "plugin boundary" for this path is the set of Python callables the
 * EpiRK integrator hands to the Krylov layer.  Each entry point below
 * replaces one of them; the reference file:line it stands in for is cited
 * on the declaration.  A Python mirror with the reference's own names and
 * signatures (paper_1604_02614_b200/) binds these through ctypes — see
 * INTEGRATION.md for the binding a maintainer of `expmhd` would add.
 *
 * Conventions
 *  - every vector pointer is a DEVICE pointer (fp64, caller-owned);
 *  - calls are asynchronous and ordered on the context's CUDA stream
 *    (emhd_set_stream); only emhd_status_read synchronises;
 *  - state layout is the reference's (8, nx, ny) C order, y fastest
 *    (mhd.py:99-103); a rank of a slab decomposition holds nx local rows;
 *  - halos: optional [2 sides][8 fields][2 rows][ny] buffers holding the two
 *    rows below row 0 and above row nx-1 (bc EMHD_BC_EXTERNAL sides only);
 *  - return 0 on success, an EMHD_ERR_* code otherwise; numerical failures
 *    (admissibility, non-finite Jv, dense overflow) are reported through the
 *    device status word and mapped by the host to the reference's exception
 *    types (AdmissibilityError, FloatingPointError).
 *  - a context is not thread-safe; one host thread per GPU.
 */
#ifndef EMHD_H
#define EMHD_H

#ifdef __cplusplus
extern "C" {
#endif

#define EMHD_OK 0
#define EMHD_ERR_DENSITY 1
#define EMHD_ERR_PRESSURE 2
#define EMHD_ERR_NONFINITE 3
#define EMHD_ERR_CUDA 4
/* 5: EMHD_ERR_NCCL (below) */
#define EMHD_ERR_ARG 6
#define EMHD_ERR_DENSE 7

#define EMHD_BC_PERIODIC 0
#define EMHD_BC_REFLECT 1
#define EMHD_BC_ZEROGRAD 2
#define EMHD_BC_EXTERNAL 3

/* status flag bits */
#define EMHD_ST_RHO 1
#define EMHD_ST_PRESSURE 2
#define EMHD_ST_NONFINITE 4
#define EMHD_ST_BREAKDOWN 8
#define EMHD_ST_DENSE 16

typedef struct emhd_ctx emhd_ctx;

/* Grid2D (mhd.py:31-64) + BoundaryPolicy (mhd.py:84-96) + slab placement */
typedef struct emhd_geometry {
  int nx, ny;              /* local rows (x), columns (y) */
  int nx_global;           /* global rows */
  int x_offset;            /* global index of local row 0 */
  double hx, hy;           /* (x_hi - x_lo)/nx_global, (y_hi - y_lo)/ny */
  int bc_x_lo, bc_x_hi;    /* EMHD_BC_*; EXTERNAL = rows come from a halo buffer */
  int bc_y;                /* EMHD_BC_PERIODIC / REFLECT / ZEROGRAD */
} emhd_geometry;

/* MhdParams (mhd.py:67-81) + make_rhs(check=) (mhd.py:280) */
typedef struct emhd_physics {
  double mu, eta, kappa, gamma;
  int b_half;
  int check;
} emhd_physics;

typedef struct emhd_status {
  int flags;                           /* EMHD_ST_* bits seen since the last reset */
  int rhs_evals;                       /* stencil evaluations executed (device-counted) */
  unsigned long long first_nonfinite;  /* flat index of the first non-finite F(a+sigma v) */
  int breakdown;                       /* Arnoldi lucky breakdown seen */
  int fail_iter;                       /* epoch (emhd_set_epoch) of the first flagging stencil */
  int rhs_evals_mark;                  /* rhs_evals at the last emhd_evals_mark (stream-ordered) */
} emhd_status;

/* ---- context -------------------------------------------------------- */
const char* emhd_version(void);
const char* emhd_error_string(int code);
int emhd_ctx_create(emhd_ctx** ctx, const emhd_geometry* g, const emhd_physics* p, int max_vectors);
int emhd_ctx_destroy(emhd_ctx* ctx);
int emhd_set_stream(emhd_ctx* ctx, void* cuda_stream);
int emhd_num_sms(emhd_ctx* ctx);
/* tag recorded (atomic min) in emhd_status.fail_iter by stencil launches that flag an error;
 * -1 (the default) for launches outside the Arnoldi driver, whose iterations carry their index */
int emhd_set_epoch(emhd_ctx* ctx, int epoch);
/* synchronous read of the device status word (stream-ordered) */
int emhd_status_read(emhd_ctx* ctx, emhd_status* out);
int emhd_status_reset(emhd_ctx* ctx);
/* stream-ordered snapshot of rhs_evals into rhs_evals_mark (no sync): a step's RHS count is
 * then read in the step's one final status read instead of a read at its start */
int emhd_evals_mark(emhd_ctx* ctx);
/* stream-ordered: clear RHO/PRESSURE/NONFINITE flags whose fail_iter >= epoch_min (discarded
 * speculative Arnoldi iterations; no reference counterpart — they never run there) */
int emhd_status_scrub(emhd_ctx* ctx, int epoch_min);
/* stream-ordered: clear every error flag and first-failure record, keep rhs_evals (and its mark) */
int emhd_status_clear_errors(emhd_ctx* ctx);

/* ---- stencil launch selection (per context) ------------------------- */
/* Which kernel variant evaluates the fused RHS / Jv stencil.  All variants issue the same
 * operations in the same order (bit-identical outputs); the selection only moves performance.
 * Defaults come from the environment at context creation (EMHD_STENCIL_TY, EMHD_STENCIL_TMA,
 * EMHD_MIN_ROWS, EMHD_STENCIL_TILE_ROWS).  No reference counterpart (tuning / test hook). */
#define EMHD_STENCIL_AUTO 0      /* marching strips, 2D tiles when a strip CTA gets < tile_rows rows */
#define EMHD_STENCIL_MARCHING 1  /* row-marching strips of `strip` columns, rows_per_cta rows each */
#define EMHD_STENCIL_TILE 2      /* 8 x 32 output tiles, three barrier-separated phases */
typedef struct emhd_stencil_path {
  int kernel;        /* EMHD_STENCIL_* */
  int rows_per_cta;  /* marching: rows per CTA; 0 = one wave of resident CTAs (>= min_rows) */
  int strip;         /* marching: 32 / 64 / 128 columns per CTA; 0 = by ny and raw_rows (64 with two
                      * staged rows, 4 CTAs/SM; 128 with one) */
  int bulk;          /* marching: interior strips stage rows with bulk async copies (TMA engine)
                        when 16-byte aligned; 0 = per-thread cp.async everywhere */
  int min_rows;      /* >= 1 */
  int tile_rows;
  int raw_rows;      /* marching: input rows staged ahead, 1 or 2 (0 = auto: 2 with the halo warp for
                      * Jv / normalised Jv, 1 for the RHS) */
} emhd_stencil_path;
int emhd_set_stencil_path(emhd_ctx* ctx, const emhd_stencil_path* sel);
int emhd_get_stencil_path(emhd_ctx* ctx, emhd_stencil_path* out);
/* Small grids (every CTA of the streaming kernels co-resident: up to ~128^2 cells x 8 fields):
 * emhd_arnoldi_iter runs the orthogonalisation of krylov.py:151-166 — dots, update, the
 * selective re-orthogonalisation decision and, when needed, the second pass — as ONE launch
 * with grid barriers instead of four, bit-identical to the separate launches.  on = 0 turns it
 * off for this context (default: EMHD_FUSED_ORTH, 1). */
int emhd_set_fused_orth(emhd_ctx* ctx, int on);
/* what the last stencil launch on ctx ran: kernel (1 marching / 2 tile), rows_per_cta and strip
 * of a marching launch, bulk = 1 when some interior strip staged its rows by bulk copies */
int emhd_last_stencil(emhd_ctx* ctx, emhd_stencil_path* out);

/* ---- (a) right-hand side ------------------------------------------- */
/* F = rhs(u)   — replaces make_rhs(...)(y) / rhs(U, params, grid, bc)  mhd.py:269-285 */
int emhd_rhs(emhd_ctx* ctx, const double* u, const double* u_halo, double* F);

/* ---- (b) finite-difference Jacobian action ------------------------- */
/* out = (F(a + sigma v) - F(a)) / sigma, sigma from *d_vnorm = ||v||_inf on device;
 * ||v||_inf == 0 -> zeros, no RHS evaluation.
 * Replaces FdJacobianOperator._apply  fdjac.py:38-49 */
int emhd_jv(emhd_ctx* ctx, const double* a, const double* a_halo, const double* fa,
            const double* v, const double* v_halo, const double* d_vnorm, double* out);

/* Augmented apply of phi_comb (krylov.py:268-273): top = ch*J u + sum_k bcol[k]*q[bidx[k]],
 * bottom = upshift(q); x = [u; q] with q = d_q (length p).  nb <= 5, p <= 5. */
int emhd_jv_aug(emhd_ctx* ctx, const double* a, const double* a_halo, const double* fa,
                const double* u, const double* u_halo, const double* d_vnorm, const double* d_q,
                int p, double ch, int nb, const double* const* bcol, const int* bidx, double* out);

/* Fused Arnoldi operator step: v_j = w/h (written to v_out, incl. the p-entry tail),
 * out = J v_j (plain, or augmented when p > 0).  d_scal = {h_next, max|w_top|}.
 * Replaces V[:, j+1] = w / hnext (krylov.py:167) followed by apply(V[:, j]) (:149). */
int emhd_jv_normalized(emhd_ctx* ctx, const double* a, const double* a_halo, const double* fa,
                       const double* w, const double* w_halo, const double* d_scal, double* v_out,
                       int p, double ch, int nb, const double* const* bcol, const int* bidx,
                       double* out);

/* ---- (c) Arnoldi step pieces (krylov.py:144-168) ------------------- */
/* out[i] = <w, V_i> for i < nvec over len_dot; self: out[nvec] = <w, w> */
int emhd_multidot(emhd_ctx* ctx, const double* w, const double* V, long long ldv, int nvec,
                  long long len_dot, int self, double* out);
/* w[:len_upd] -= sum_i h[i] V_i; mode 0: out[i] = <w, V_i> (len_dot);
 * mode 1: out = {sum w^2 over len_dot, max|w| over len_max} */
int emhd_update(emhd_ctx* ctx, double* w, const double* V, long long ldv, int nvec, const double* h,
                long long len_upd, long long len_dot, long long len_max, int mode, double* out);
/* mode 0 writes nvec + 2 values: V^T w_new, then ||w_new||^2 (over len_dot) and max|w_new|
 * (over len_max) — the inputs of the selective re-orthogonalisation test below. */
/* Selective (DGKS) re-orthogonalisation after pass 1 (r = emhd_update mode-0 output,
 * all-reduced on slab ranks): when ||w1|| >= eta ||w|| (||w||^2 = *selfdot) set *gate = 1 and
 * finish column j with h1 alone (H, hnext = ||w1||, breakdown test, scal), else *gate = 0.
 * The reference always runs the second pass (krylov.py:156-160); skipping it when the first
 * left w1 orthogonal to working precision changes H and V at round-off level only. */
int emhd_reorth_decide(emhd_ctx* ctx, const double* h1, const double* r, int nvec,
                       const double* selfdot, int j, double* H, long long ldh, double* scal,
                       double* brk_hist, double eta, double* gate);
/* the next pass-2 launch on ctx (emhd_update mode 1, emhd_update_finish, emhd_update_push,
 * emhd_arnoldi_finish) does no work when *gate != 0 (device-side test) */
int emhd_skip_next(emhd_ctx* ctx, const double* gate);
/* slab ranks: rows {0,1} / {nx-2,nx-1} of w into the lo / hi neighbours' halo buffers (peer
 * pointers, NULL = none) when *gate != 0 (gate NULL: always) — the halo push of an iteration
 * whose second pass was skipped (emhd_update_push does it otherwise) */
int emhd_push_edges(emhd_ctx* ctx, const double* w, double* lo_halo, double* hi_halo, const double* gate);
/* emhd_update(mode 1) + emhd_arnoldi_finish in one launch (single rank: the norms need no
 * all-reduce before the column bookkeeping). */
int emhd_update_finish(emhd_ctx* ctx, double* w, const double* V, long long ldv, int nvec,
                       const double* h2, long long len_upd, long long len_dot, long long len_max,
                       double* nrm, const double* h1, const double* selfdot, int j, double* H,
                       long long ldh, double* scal, double* brk_hist);
/* out = {sum x^2 over len_sum, max|x| over len_max} */
int emhd_norms(emhd_ctx* ctx, const double* x, long long len_sum, long long len_max, double* out);
/* H[:j+1, j] = h1 + h2; hnext = sqrt(nrm[0]); breakdown if hnext <= 1e-12 max(sqrt(selfdot), 1);
 * scal = {hnext, nrm[1], breakdown}; brk_hist (optional) [j] = breakdown flag of iteration j.
 * Once scal[2] != 0 the next emhd_jv_normalized launch does no work (lets a caller queue
 * iterations ahead of its breakdown check). */
int emhd_arnoldi_finish(emhd_ctx* ctx, const double* h1, const double* h2, const double* nrm,
                        const double* selfdot, int j, double* H, long long ldh, double* scal,
                        double* brk_hist);
/* out = x / d (d = sqrt(*d) when take_sqrt); d_out receives d.  (krylov.py:137, :167) */
int emhd_div_scalar(emhd_ctx* ctx, const double* x, const double* d, int take_sqrt, double* out,
                    double* d_out, long long n);

/* ---- small dense phi (phifuncs.py:65-107, krylov.py:209-238,378-383) */
/* For s < S: y_s = beta * phi_order(scales[s] * H_m) e_1, res[s] = |h_next| |y_s[m-1]| / ||y_s||
 * * res_scale[s]; scales/res_scale/scal/beta/Y/res are device pointers. */
int emhd_phi_small(emhd_ctx* ctx, const double* H, long long ldh, int m, int order, int S,
                   const double* scales, const double* res_scale, const double* scal,
                   const double* beta, double* Y, double* res);

/* As emhd_phi_small with the S scales passed as a HOST array (copied into the launch) and
 * res[s] unscaled.  Saves the device scratch and its host-to-device copy per residual check. */
int emhd_phi_small_h(emhd_ctx* ctx, const double* H, long long ldh, int m, int order, int S,
                     const double* host_scales, const double* scal, const double* beta, double* Y,
                     double* res);

/* Speculative batch of residual checks on one factorisation: CTA s uses basis size ms[s] (host
 * int array), scale host_scales[s]; h_{m+1,m} from H (0 when brk_hist[m-1] != 0); Y rows of
 * stride ldy; res[s] unscaled.  S <= 8. */
int emhd_phi_small_batch(emhd_ctx* ctx, const double* H, long long ldh, const int* ms, int order, int S,
                         const double* host_scales, const double* brk_hist, const double* beta,
                         double* Y, long long ldy, double* res);

/* Small dense exponentials of dimension >= n run on a thread-block cluster of 8 CTAs (products,
 * norms and ell split by row blocks; 0 = never, every one on one CTA); process-wide; returns
 * the previous threshold (default: EMHD_DENSE_CLUSTER_N, else 56). */
int emhd_set_dense_cluster(int n);

/* The (V - U) X = (V + U) solve of the Pade approximant (scipy.linalg.expm's LAPACK solve behind
 * phifuncs.py:65-107): blocked Gauss-Jordan with partial pivoting, eight pivot columns per step,
 * for 24 <= n <= 128 (on != 0, default), or the unblocked solve for every n; process-wide;
 * returns the previous setting (default: EMHD_DENSE_GJ_BLOCKED, else 1). */
int emhd_set_dense_gj_blocked(int on);

/* E = expm(A), n x n row-major device matrices; work: device scratch of n + 4 doubles.
 * Synchronous.  (scipy.linalg.expm as called by phi_dense, phifuncs.py:97,104) */
int emhd_expm(emhd_ctx* ctx, const double* A, int n, double* E, double* work);

/* ---- (d) combinations ---------------------------------------------- */
/* outs[s] = base[s] + coef[s] * (V_m Y[s]) (base[s] may be NULL: outs[s] = V_m Y[s]); S <= 4.
 * Replaces Vm @ y (krylov.py:316, 374) fused with the stage axpys (epirk.py:207, 251-252). */
int emhd_combine(emhd_ctx* ctx, const double* V, long long ldv, int m, const double* Y, int S,
                 const double* const* base, const double* coef, double* const* outs, long long len);
/* out = post * (t_0 + t_1 + ...), t_k = c_k x_k (has_c[k]) or x_k, left to right, no FMA;
 * max_out (optional): max|out| over the first len_max entries.  (epirk.py stage algebra) */
int emhd_lincomb(emhd_ctx* ctx, int nterms, const double* const* x, const double* c, const int* has_c,
                 double post, int has_post, double* out, long long n, long long len_max,
                 double* max_out);
/* out[0] = sum_e (err_e / (tol + tol |y_e|))^2  (StepController.error_norm, epirk.py:156-158) */
int emhd_wrms(emhd_ctx* ctx, const double* err, const double* y, double tol, long long n, double* out);

/* ---- diagnostics --------------------------------------------------- */
/* Synchronous error-path report of the state a stencil call in `mode` (0 RHS, 1 Jv, 2 normalised
 * Jv) evaluated: report = {int which (1 density, 2 pressure, 0 none), int i, int j, int pad,
 * double value}, (i, j) the first minimising cell of the ghost-padded field, as the reference's
 * AdmissibilityError names it (mhd.py:111-131). */
int emhd_admissibility_report(emhd_ctx* ctx, int mode, const double* a, const double* a_halo,
                              const double* v, const double* v_halo, const double* scal,
                              void* report);

/* ---- diagnostics --------------------------------------- */
/* d = centred div B (mhd.py:288-296), *dmax = max |d| over this rank (device scalar) */
int emhd_div_b(emhd_ctx* ctx, const double* U, const double* U_halo, double* d, double* dmax);
/* J = curl B, (3, nx, ny) (mhd.py:299-309) */
int emhd_current_j(emhd_ctx* ctx, const double* U, const double* U_halo, double* J);

/* ---- single-rank Arnoldi driver ------------------------------------ */
/* args: a plain struct of device pointers and sizes (layout in paper_1604_02614_b200/_native.py,
 * ArnoldiArgs): a, F(a), V, ldv, H, ldh, w0, w1, d1, d2, nrm, vn, scal, brk, n_top, len_dot,
 * len_upd, p, nb, ch, bcol[5], bidx[5].  Launches iteration j of _ArnoldiProcess.extend
 * (krylov.py:144-168) — (normalise +) Jv, multi-dot, update + re-dot, update + norms +
 * column bookkeeping — as one stream-ordered call. */
int emhd_arnoldi_iter(emhd_ctx* ctx, const void* args, int j);
/* emhd_arnoldi_iter for j = j_begin .. j_end-1 (one call for a burst of iterations) */
int emhd_arnoldi_run(emhd_ctx* ctx, const void* args, int j_begin, int j_end);
/* emhd_arnoldi_run for look-ahead iterations queued while the residual checks of earlier ones
 * run on another stream: each iteration is gated on the context's cancel word (j >= 1).
 * No reference counterpart — the reference checks every residual before extending. */
int emhd_arnoldi_lookahead(emhd_ctx* ctx, const void* args, int j_begin, int j_end);
/* cancel the look-ahead iterations j >= epoch_min of process generation gen that have not
 * started (async 8-byte copy on the context's stream) */
int emhd_arnoldi_cancel(emhd_ctx* ctx, int gen, int epoch_min);
/* status.rhs_evals -= sum(evals[0:count]): RHS evaluations of discarded speculative
 * iterations (evals written per iteration by emhd_arnoldi_iter when args.evals is set) */
int emhd_evals_discount(emhd_ctx* ctx, const double* evals, int count);

/* Persisting-L2 window over [base, base + bytes) on the context's stream (bytes = 0: none);
 * B200-specific residency control for small Krylov bases, no reference counterpart. */
int emhd_l2_window(emhd_ctx* ctx, const void* base, long long bytes);

/* ---- per-launch profiling (benchmarks) ------------------------------ */
enum { EMHD_K_JV = 0, EMHD_K_JV_NORMALIZED = 1, EMHD_K_MULTIDOT = 2, EMHD_K_UPDATE = 3,
       EMHD_K_MULTIDOT2 = 4, EMHD_K_UPDATE_FINISH = 5, EMHD_K_NORMS = 6, EMHD_K_DIV_SCALAR = 7,
       EMHD_K_GATE = 8 };
/* enable != 0: clear and start recording CUDA events around every launch of emhd_arnoldi_*
 * (and emhd_jv / emhd_norms / emhd_div_scalar); 0: stop */
int emhd_profile(emhd_ctx* ctx, int enable);
/* sync, then copy out (kind, ms, algorithmic bytes; 0 bytes for a launch a device gate made a
 * no-op) of up to max_n records and clear them; returns the count (negative: -error) */
int emhd_profile_read(emhd_ctx* ctx, int max_n, int* kinds, double* ms, double* bytes);
/* Copy brk[0:nbrk] and res[0:nres] into host_out (pinned), then read the status word: the one
 * host synchronisation of a residual check. */
int emhd_readback(emhd_ctx* ctx, const double* brk, int nbrk, const double* res, int nres,
                  double* host_out, emhd_status* st);

/* ---- slab-rank collectives (x-slab decomposition, one process per GPU) ---- */
/* A context placed on an x-slab (EXTERNAL x sides) owns a communicator: the Arnoldi driver
 * (emhd_arnoldi_iter) then all-reduces its dot products and norms from C (stream-ordered, no
 * host sync) and every stencil entry point called with a NULL halo for the array it perturbs
 * exchanges that halo itself, on a second stream, while the interior rows [2, nx-2) run; the
 * edge rows follow when the halo has landed.  The reference is single-process; these replace
 * the distributed form of its sums (krylov.py:151,153,158,161) and ghosts (mhd.py:144-165). */
#define EMHD_ERR_NCCL 5
#define EMHD_OP_SUM 0
#define EMHD_OP_MAX 2
#define EMHD_OP_MIN 3
/* 128-byte NCCL unique id (rank 0 creates two: reduce and halo communicators) */
int emhd_nccl_unique_id(void* out128);
/* NCCL transport; lo / hi: neighbour ranks of the EXTERNAL x sides (-1: none, must match the
 * geometry's bc_x_lo / bc_x_hi); a rank may be its own neighbour (periodic ring of one) */
int emhd_comm_init_nccl(emhd_ctx* ctx, int nranks, int rank, int lo, int hi, const void* uid_reduce,
                        const void* uid_halo);
/* Host-callback transport (tests: ranks sharing one GPU over a CPU channel): ar(user, buf, n, op)
 * reduces n host doubles in place across ranks; ex(user, send, recv, n_side) delivers send[2][n_side]
 * (rows {0,1}, rows {nx-2,nx-1}) and fills recv[2][n_side] (lo neighbour's top rows, hi neighbour's
 * bottom rows).  Both return 0 on success.  Collectives synchronise the context's stream. */
typedef int (*emhd_host_allreduce_fn)(void* user, double* buf, int n, int op);
typedef int (*emhd_host_exchange_fn)(void* user, const double* send, double* recv, long long n_side);
int emhd_comm_init_host(emhd_ctx* ctx, int nranks, int rank, int lo, int hi, emhd_host_allreduce_fn ar,
                        emhd_host_exchange_fn ex, void* user);
/* in-place all-reduce of n device doubles (EMHD_OP_*) across the context's ranks (no comm: no-op) */
int emhd_allreduce(emhd_ctx* ctx, double* buf, int n, int op);
/* halo[2][8][2][ny] = x-halo of x (pack + exchange, ordered on the context's stream) */
int emhd_halo_exchange(emhd_ctx* ctx, const double* x, double* halo);

/* ---- slab halos ------------------------------------------------------ */
/* sendbuf[2][8][2][ny] = rows {0,1} and {nx-2, nx-1} of every field of x */
int emhd_pack_edges(emhd_ctx* ctx, const double* x, double* sendbuf);
/* emhd_update mode 1 (w -= V h; out = {sum w^2, max|w_top|}) that also stores the final w's
 * rows {0,1} into lo_halo side 1 and rows {nx-2,nx-1} into hi_halo side 0 (the neighbours'
 * [2][8][2][ny] halo buffers, peer pointers; NULL = no neighbour): the halo exchange of the next
 * normalised Jv (krylov.py:167,149) fused into the producing pass; the norm all-reduce that
 * follows orders the stores before the neighbours' stencil. */
int emhd_update_push(emhd_ctx* ctx, double* w, const double* V, long long ldv, int nvec, const double* h,
                     long long len_upd, long long len_dot, long long len_max, double* out,
                     double* lo_halo, double* hi_halo);
/* Arnoldi norms across slabs with ONE sum all-reduce (krylov.py:151,161 and the next sigma):
 * slots[0] = nrm[0], slots[1 + rank] = nrm[1], other slots 0; after the SUM all-reduce of the
 * 1 + nranks slots, emhd_unslot_norms gives nrm = {global sum, max over ranks}. */
int emhd_slot_norms(emhd_ctx* ctx, const double* nrm, int rank, int nranks, double* slots);
int emhd_unslot_norms(emhd_ctx* ctx, const double* slots, int nranks, double* nrm);

/* ---- output side: snapshots and the explicit-RK4 harness ---- */
/* cells[(c * 8) + f] = U[f * ncell + c]: the cell-major data block of a .mhd25 snapshot
 * (replaces np.moveaxis(U, 0, -1) in write_snapshot, snapshot.py:53-57); a slab's block is a
 * contiguous byte range of the file at offset 96 + 64 * x_offset * ny. */
int emhd_cells_pack(emhd_ctx* ctx, const double* U, long long ncell, double* cells);
/* inverse of emhd_cells_pack (read_snapshot, snapshot.py:77) */
int emhd_cells_unpack(emhd_ctx* ctx, const double* cells, long long ncell, double* U);
/* *cmax (device) = max over this rank's cells of sqrt((gamma p + |B|^2)/rho) + sqrt(|m|^2/rho^2),
 * bitwise the reference's (harness.py:166-174, pressure mhd.py:116-131); non-positive density or
 * pressure raises the status flags. */
int emhd_max_signal_speed(emhd_ctx* ctx, const double* U, double* cmax);
/* out[f] (device, 8) = sum over this rank's cells of (U_f - R_f)^2 (error_norm, harness.py:153-163) */
int emhd_field_sqdiff(emhd_ctx* ctx, const double* U, const double* R, double* out);
/* out = base + post (x) (t_0 + ...) with lincomb's term rules (harness.py:194, RK4 update) */
int emhd_lincomb_onto(emhd_ctx* ctx, const double* base, int nterms, const double* const* x, const double* c,
                      const int* has_c, double post, int has_post, double* out, long long n);

#ifdef __cplusplus
}
#endif
#endif /* EMHD_H */
