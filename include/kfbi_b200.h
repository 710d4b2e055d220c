/*
 * kfbi_b200.h — C ABI of the B200-native KFBI hot path.
 *
 * The reference (`/root/reference/pkg/src/kfbi`, pure Python) has no native
 * boundary of its own: every sweep goes through `Backend.dispatch(spec,
 * item_fn)` (engine.py:84-95) with numpy closures, which a GPU cannot plug
 * into.  The boundary therefore sits one level up, at the solver objects.
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions
 *   - All device pointers are caller-owned device memory (the Python host
 *     passes torch tensor data pointers); the plan owns only its scratch.
 *   - Grid fields are (M+1) x (M+1) row-major, flat index i + j*(M+1)
 *     (grid.py:4-6, grid.py:44-52).  Complex values are interleaved
 *     (re, im) doubles, i.e. numpy/torch complex128.
 *   - `dtype` is KFBI_F64 or KFBI_C128; real-kappa/real-data solves run the
 *     f64 path, anything complex runs the c128 path (boxsolve.py:56).
 *   - Every function returns a kfbi_status; on failure the message is in
 *     kfbi_last_error() (thread-local).  The Python host maps the codes onto
 *     the reference exception classes (errors.py:8-56).
 *   - A plan is bound to one device and is not thread-safe; distinct plans
 *     may be used concurrently.  Work is enqueued on the
 *     caller's stream; the only host syncs are the documented ones.
 */
#ifndef KFBI_B200_H
#define KFBI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KFBI_OK = 0,
  KFBI_E_CONFIG = 1,       /* -> ConfigError      (errors.py:12)          */
  KFBI_E_GRID = 2,         /* -> GridError        (errors.py:20)          */
  KFBI_E_NOCONV = 3,       /* -> ConvergenceError (errors.py:36-42)       */
  KFBI_E_INSTABILITY = 4,  /* -> InstabilityError (errors.py:45-56)       */
  KFBI_E_CUDA = 5          /* -> DispatchError(kernel_name) (errors.py:28) */
} kfbi_status;

typedef enum { KFBI_F64 = 0, KFBI_C128 = 1 } kfbi_dtype;
typedef enum { KFBI_DIRICHLET_ZERO = 0, KFBI_NEUMANN_ZERO = 1 } kfbi_box_bc;

/* The nine dispatch names of the reference engine (engine.py:23-35), used as
 * indices into the per-kernel timing arrays. */
enum {
  KFBI_K_CLASSIFY = 0,
  KFBI_K_EDGES = 1,
  KFBI_K_JUMPS = 2,          /* "jumps-and-corrections" */
  KFBI_K_ROWS = 3,           /* "transform-rows"        */
  KFBI_K_COLS = 4,           /* "transform-cols"        */
  KFBI_K_SCALE = 5,          /* "diagonal-scale"        */
  KFBI_K_EXTRACT = 6,        /* "extract-traces"        */
  KFBI_K_DENSITY = 7,        /* "density-update"        */
  KFBI_K_RHS = 8,            /* "rhs-update"            */
  KFBI_N_KERNEL_NAMES = 9
};

typedef struct kfbi_plan kfbi_plan;

/* CartesianGrid (grid.py:25-52) + the BoxSolver eigenvalue tables
 * (boxsolve.py:38-44).  m must be a power of two, 16 <= m <= 16384. */
typedef struct {
  int32_t m;
  double h;
  int32_t device;
} kfbi_grid_desc;

/* Host-side geometry tables, uploaded once (InterfaceWorkspace.__init__,
 * interface.py:137-162; TraceExtractor.__init__, bvp.py:37-86; records,
 * grid.py:71-101).  All pointers are HOST pointers, copied by the call. */
typedef struct {
  int32_t n_ctl;              /* control points                          */
  int32_t n_edges;            /* unique sign-change edges (2 records each) */
  int32_t n_rec;              /* intersection records                    */
  int32_t n_groups;           /* owning irregular nodes                  */
  const double *w_edges;      /* [n_edges][n_ctl] trig-interp rows, or NULL */
  const int8_t *edge_axis;    /* [n_edges] 0 = horizontal, 1 = vertical  */
  const int32_t *rec_edge;    /* [n_rec] edge of each record             */
  const double *rec_d;        /* [n_rec] neighbour-minus-crossing offset */
  const double *rec_sigma;    /* [n_rec] -1/h^2 interior, +1/h^2 exterior */
  const int32_t *group_start; /* [n_groups+1] CSR over records           */
  const int32_t *group_node;  /* [n_groups] owner flat index i + j(M+1)  */
  const int32_t *row_group;   /* [m+2] CSR of groups per grid row j      */
  const double *deriv_col;    /* [n_ctl] first column of d/dtheta        */
  const double *speed;        /* [n_ctl] |x'(theta)|                     */
  const double *tangent;      /* [n_ctl][2]                              */
  const double *normal;       /* [n_ctl][2]                              */
  const double *dtan_ds;      /* [n_ctl][2]                              */
  const double *inv3;         /* [n_ctl][3][3]                           */
  const int32_t *stencil;     /* [n_ctl][6] flat node indices            */
  const double *ainv_rows;    /* [n_ctl][3][6] rows 0..2 of the 6x6 inverse */
  const double *jcoef;        /* [n_ctl][6][6] jump-shift coefficients   */
  /* w_edges == NULL: build W on the device (trigonometric rows, even n_ctl
   * >= 32, interface.py:38-52) from these parameters instead */
  const double *edge_theta;   /* [n_edges] crossing parameter per edge   */
  const double *ctl_theta;    /* [n_ctl] control parameters              */
} kfbi_geometry;

/* One Dirichlet or Neumann BVP solve by Richardson iteration (BvpProblem,
 * bvp.py:231-262; richardson_solve, bvp.py:276-351).  Device pointers. */
typedef struct {
  int32_t dtype;
  double kappa_re, kappa_im;
  const void *F;          /* (M+1)^2 grid source                          */
  double F_sign;          /* +1 or -1 (timestepping.py:182 negates F)     */
  const void *f_gamma;    /* [n_ctl]                                      */
  double f_gamma_sign;
  const void *g;          /* [n_ctl] boundary values                      */
  void *density;          /* [n_ctl] in: initial density, out: final      */
  double gamma, tol;
  int32_t max_iter;
  int32_t sweeps_hint;    /* sweeps to enqueue before the first check     */
  void *u;                /* out (M+1)^2 field of the final sweep         */
  void *trace_u;          /* out [n_ctl]                                  */
  void *trace_un;         /* out [n_ctl]                                  */
  int32_t use_operator;   /* 1: sweeps >= 2 use the plan's trace operator */
  int32_t log_slot;       /* >= 0 (operator form only): fully asynchronous;
                             iterations / status land in the plan's step log
                             (kfbi_log_fetch), result fields are -1 (pending) */
  int32_t bc_kind;        /* 0 Dirichlet (density = phi, trace u+), 1 Neumann
                             (density = psi, trace d_n u+, one-sided
                             extraction; bvp.py:313-323) */
  int32_t box_bc;         /* kfbi_box_bc closure of the box solves          */
  int32_t field_chunks;   /* 1: the caller reads the returned field only at
                             the nodes covered by kfbi_plan_set_field_chunks
                             (the steppers mask it); the FACR odd rows of the
                             final sweep are solved only there               */
} kfbi_bvp;

/* One entry of the plan's device-side step log (asynchronous stepping). */
typedef struct {
  int32_t iterations;
  int32_t status;         /* 1 converged, 2 max_iter reached */
  double residual;        /* last density update max-norm */
  double norm;            /* blow-up norm of the step (kfbi_log_norm, which=0) */
  double newton;          /* worst pointwise Newton residual (which=1)      */
} kfbi_step_log;

typedef struct {
  int32_t iterations;
  int32_t converged;
  double residual;
  double *history;        /* host buffer [max_iter], filled on return     */
} kfbi_bvp_result;

const char *kfbi_last_error(void);
const char *kfbi_version(void);

kfbi_status kfbi_plan_create(const kfbi_grid_desc *desc, kfbi_plan **out);
kfbi_status kfbi_plan_destroy(kfbi_plan *plan);

/* BoxSolver.solve (boxsolve.py:46-94): (Delta_h - kappa) u = rhs with the
 * dirichlet-zero closure; returns u with an exact zero ring. */
kfbi_status kfbi_box_solve(kfbi_plan *plan, int32_t dtype, double kappa_re,
                           double kappa_im, const void *rhs, void *u,
                           void *stream);

/* BoxSolver.solve with either closure (boxsolve.py:46-94): dirichlet-zero
 * (DST-I, zero ring) or neumann-zero (DCT-I, mirror ghost, rhs read on the
 * whole grid; kappa = 0 rejected as singular, boxsolve.py:32-33). */
kfbi_status kfbi_box_solve_bc(kfbi_plan *plan, int32_t dtype, int32_t box_bc,
                              double kappa_re, double kappa_im, const void *rhs,
                              void *u, void *stream);

kfbi_status kfbi_plan_set_geometry(kfbi_plan *plan, const kfbi_geometry *geo);

/* classify (grid.py:122-155): interior[j*(m+1)+i] = level(x[i], y[j]) <= tol
 * on the device (host in/out arrays).  kind 0 circle (params cx, cy, r),
 * 1 ellipse (cx, cy, a, b), 2 star (cx, cy, scale, c, lobes).  Circle and
 * ellipse levels are evaluated exactly as numpy does (no contraction); for
 * the star the flat indices of nodes with |level - tol| <= 1e-12 are
 * returned in ambiguous[0 .. min(*n_ambiguous, cap)) for the caller to
 * re-evaluate with the reference formula. */
kfbi_status kfbi_classify_nodes(int32_t device, int32_t kind, const double *params,
                                const double *x, const double *y, int32_t m, double tol,
                                uint8_t *interior, int32_t *n_ambiguous, int64_t *ambiguous,
                                int32_t cap);

/* Column stage of the dirichlet-zero box solve (the scipy dst / idst pair
 * along axis 0 of boxsolve.py:70-82 with the spectral division between).
 * Mode 1 solves the equivalent constant-coefficient tridiagonal system of
 * every spectral column by a factored recurrence (O(M) per column,
 * box_tri.cuh); mode 2 runs DST-I -> divide -> DST-I on the FFT engine with
 * the reference's eigenvalue table; mode 0 (default, auto) uses the
 * recurrences when their deviation bound from the reference's rounded
 * eigenvalues, E = (4.4e-16 / h^2) / min |lam_p + lam_q - kappa|, is
 * <= 1e-11 (every time-stepping kappa), the DST-I engine otherwise.  The
 * neumann-zero closure always uses the DCT-I engine.
 * kfbi_plan_colsolver_for reports the choice and E for one kappa. */
kfbi_status kfbi_plan_set_colsolver(kfbi_plan *plan, int32_t mode);
kfbi_status kfbi_plan_get_colsolver(kfbi_plan *plan, int32_t *mode);
/* Operator form, Dirichlet, 512 <= M <= 8192: sweep 1 forms only its trace
 * (the inverse row transform evaluated at the six-point stencil nodes,
 * box_tri.cuh stencil_eval_kernel) instead of the whole field.  Opt-in
 * (default off): the direct evaluation reads the needed rows as scattered
 * 32-64 byte sectors of the strip layout and measured 98-169 us against
 * 100-200 us for the full inverse row pass.  The returned field
 * is the final pipeline's either way. */
kfbi_status kfbi_plan_set_trace_sweep(kfbi_plan *plan, int32_t on);
/* Dirichlet box solves on one slab, 64 <= M <= 8192, tridiagonal-eligible
 * kappa: one level of cyclic reduction in y (box_facr.cuh) — the even rows
 * by DST-I x tridiagonal recurrences with root r^2 on M/2 rows, the odd rows
 * by recurrences along x — half the row transforms, 5 instead of 6 field
 * sweeps of HBM.  Default on (environment KFBI_FACR=0 at plan creation: off);
 * 0 restores the three-pass solve. */
kfbi_status kfbi_plan_set_facr(kfbi_plan *plan, int32_t on);
/* 1 when a single-slab dirichlet box solve with this kappa uses FACR(1). */
kfbi_status kfbi_plan_facr_for(kfbi_plan *plan, double kappa_re, double kappa_im, int32_t *on);
kfbi_status kfbi_plan_colsolver_for(kfbi_plan *plan, double kappa_re, double kappa_im,
                                    int32_t *tridiagonal, double *bound);

/* Rows [row0, row0 + nrows) of the plan's W (n_ctl values each) to host. */
/* Edge values jv = W . JM (interface.py:206-238): the matrix-free spectral
 * form applies when the controls are the reference's theta_j = 2 pi j / n
 * with n even >= 32 (the trig branch of interp_rows, interface.py:38-52,
 * 70-75).  Mode 0 (default) uses it when the W rows it replaces would exceed
 * 192 MB and streams W rows (built on the device on first use) otherwise;
 * 1 forces the W rows, 2 the spectral form.
 * kfbi_plan_get_interp reports 1 when the spectral form is in use. */
kfbi_status kfbi_plan_set_interp(kfbi_plan *plan, int32_t mode);
kfbi_status kfbi_plan_get_interp(kfbi_plan *plan, int32_t *spectral);
kfbi_status kfbi_plan_copy_w(kfbi_plan *plan, int32_t row0, int32_t nrows, double *out);

/* OneSidedExtractor tables (bvp.py:115-212), host pointers: stencil7
 * [n_ctl][7] flat node indices, rows [n_ctl][3][7] (rows 0..2 of inv(A)),
 * fallback [n_ctl] (1: the point uses the six-point straddling stencil). */
kfbi_status kfbi_plan_set_onesided(kfbi_plan *plan, int32_t n_ctl, const int32_t *stencil7,
                                   const double *rows, const uint8_t *fallback);

/* OneSidedExtractor.extract (bvp.py:214-228): out [3][n_ctl]. */
kfbi_status kfbi_extract_onesided(kfbi_plan *plan, int32_t dtype, const void *u,
                                  const void *jm, void *out, void *stream);

/* compute_jumps (interface.py:171-203): jm out is SoA [6][n_ctl]
 * (u, ux, uy, uxx, uxy, uyy).  psi may be NULL (zero). */
kfbi_status kfbi_jumps(kfbi_plan *plan, int32_t dtype, double kappa_re,
                       double kappa_im, const void *phi, const void *psi,
                       const void *f_gamma, double f_gamma_sign, void *jm,
                       void *stream);

/* corrections (interface.py:206-238): c out is a full (M+1)^2 field. */
kfbi_status kfbi_corrections(kfbi_plan *plan, int32_t dtype, const void *jm,
                             void *c, void *stream);

/* solve_interface (interface.py:250-261): u = BoxSolver(F + corrections). */
kfbi_status kfbi_interface_solve(kfbi_plan *plan, int32_t dtype,
                                 double kappa_re, double kappa_im,
                                 const void *F, const void *jm, void *u,
                                 void *stream);
kfbi_status kfbi_interface_solve_bc(kfbi_plan *plan, int32_t dtype, int32_t box_bc,
                                    double kappa_re, double kappa_im,
                                    const void *F, const void *jm, void *u,
                                    void *stream);

/* TraceExtractor.extract (bvp.py:88-104): out [3][n_ctl] = (u+, ux+, uy+). */
kfbi_status kfbi_extract(kfbi_plan *plan, int32_t dtype, const void *u,
                         const void *jm, void *out, void *stream);

/* ---- slab-decomposed box solve (multi-GPU) ----
 * Rank `rank` of `nranks` (a power of two) owns grid rows
 * [rank*m/nranks, (rank+1)*m/nranks); its rhs / u arrays hold exactly those
 * rows, (m+1) values each (row 0 is the zero ring, row m is not stored).
 * One solve is
 *   kfbi_slab_rows_fwd -> all-to-all -> kfbi_slab_cols -> all-to-all ->
 *   kfbi_slab_rows_inv
 * where both all-to-alls exchange equal contiguous chunks of the panel
 * buffer (kfbi_slab_panel_bytes bytes per rank; nranks chunks, chunk g goes
 * to rank g), e.g. torch.distributed.all_to_all_single over NCCL.  With
 * nranks = 1 the two exchanges are identities and the result equals
 * kfbi_box_solve.  jv != NULL fuses the jump corrections of the plan's
 * geometry (rows of this slab) like the Richardson sweep does. */
typedef struct {
  int32_t nranks;
  int32_t rank;
} kfbi_slab;

kfbi_status kfbi_slab_panel_bytes(kfbi_plan *plan, int32_t dtype, int32_t nranks,
                                  int64_t *bytes);

/* Transpose-free column stage of the slab-decomposed dirichlet box solve
 * (tridiagonal recurrences, box_tri.cuh cols_tri_dist).  Rank g keeps its
 * rows of every spectral column in the row pass's own buffer ([panel][R][w],
 * kfbi_slab_rows_fwd with no exchange), solves them with zero carries at the
 * slab ends, and exchanges three values per column with every rank over peer
 * memory INSIDE the kernel (pushes into agg[h] / flags[h] of every rank h,
 * waits on its own flags for `epoch`); then kfbi_slab_rows_inv reads the same
 * buffer.  Replaces both all-to-alls: 3 P values per column cross NVLink
 * instead of 2 M^2 s / P bytes per rank.  Equal to the one-GPU solve to
 * rounding (the carries are combined in a different order).
 * virt = 1: all ranks in ONE launch on one device (panels[h] = every rank's
 * buffer), for tests.  Buffer sizes from kfbi_slab_tri_bytes. */
typedef struct {
  int32_t nranks, rank, virt;
  int32_t pad;
  uint64_t epoch;              /* > every earlier epoch on these flags          */
  int64_t max_spins;           /* bounded wait; a missing peer sets *timed_out */
  int32_t *timed_out;          /* device int, may be NULL                      */
  void *panels[8];             /* virt: every rank's panel buffer              */
  void *agg[8];                /* every rank's aggregate buffer, as mapped here */
  void *flags[8];              /* every rank's flag buffer (zeroed once)       */
} kfbi_tri_dist;

kfbi_status kfbi_slab_tri_bytes(kfbi_plan *plan, int32_t dtype, int32_t nranks,
                                int64_t *agg_bytes, int64_t *flag_bytes);
kfbi_status kfbi_slab_cols_tri(kfbi_plan *plan, int32_t dtype, int32_t nranks, int32_t rank,
                               double kappa_re, double kappa_im, void *panels,
                               const kfbi_tri_dist *dist, void *stream);
kfbi_status kfbi_slab_rows_fwd(kfbi_plan *plan, int32_t dtype, const kfbi_slab *slab,
                               const void *rhs, double sign, const void *jv,
                               void *panels, void *stream);
kfbi_status kfbi_slab_cols(kfbi_plan *plan, int32_t dtype, const kfbi_slab *slab,
                           double kappa_re, double kappa_im, void *panels, void *stream);
kfbi_status kfbi_slab_rows_inv(kfbi_plan *plan, int32_t dtype, const kfbi_slab *slab,
                               const void *panels, void *u, void *stream);

/* ---- slab passes with the all-to-all fused into the stores ----
 * Each rank holds two panel buffers in peer-addressable device memory
 * (kfbi_ipc_alloc; the handles are exchanged once and opened with
 * kfbi_ipc_open, or plain pointers of one device for virtual ranks):
 * A (column-pass input) and B (row-pass input).  One solve is
 *   kfbi_slab_rows_fwd_p2p(peer_panels = every rank's A)  -> barrier ->
 *   kfbi_slab_cols_p2p(panels = own A, peer_panels = every rank's B) ->
 *   barrier -> kfbi_slab_rows_inv(panels = own B)
 * The forward row pass writes panel chunk h of its rows directly into rank
 * h's A at the offset the all-to-all would have put it, and the column pass
 * writes row chunk h of its panels into rank h's B: the exchange overlaps
 * the transforms tile by tile and no separate collective runs.  The barrier
 * is kfbi_p2p_barrier over per-rank flag arrays (KFBI_MAX_PEERS uint64 each,
 * zero-initialised, epochs strictly increasing per call) or any stream-
 * ordered collective.  Results are bit-identical to the all-to-all form. */
#define KFBI_MAX_PEERS 8
#define KFBI_IPC_HANDLE_BYTES 64

kfbi_status kfbi_slab_rows_fwd_p2p(kfbi_plan *plan, int32_t dtype, const kfbi_slab *slab,
                                   const void *rhs, double sign, const void *jv,
                                   void *const *peer_panels, void *stream);
kfbi_status kfbi_slab_cols_p2p(kfbi_plan *plan, int32_t dtype, const kfbi_slab *slab,
                               double kappa_re, double kappa_im, const void *panels,
                               void *const *peer_panels, void *stream);
/* cudaMalloc'd, zeroed buffer + its IPC handle (KFBI_IPC_HANDLE_BYTES). */
kfbi_status kfbi_ipc_alloc(int64_t bytes, void **ptr, void *handle);
kfbi_status kfbi_ipc_free(void *ptr);
kfbi_status kfbi_ipc_open(const void *handle, void **ptr);
kfbi_status kfbi_ipc_close(void *ptr);
/* Stream-ordered barrier of `nranks` ranks over peer flag arrays; after
 * max_spins polls (<= 0: 2^28, tens of seconds) without every peer it gives
 * up and sets *timed_out (device int, may be NULL) to 1 instead of hanging. */
kfbi_status kfbi_p2p_barrier(void *const *peer_flags, int32_t nranks, int32_t rank,
                             int64_t epoch, int64_t max_spins, int32_t *timed_out,
                             void *stream);

/* ---- slab-decomposed Richardson sweep (dist.py SlabRichardson) ----
 * Per sweep on every rank: kfbi_jumps (replicated, O(n_ctl)) ->
 * kfbi_edge_values (jv = W . JM, replicated) -> kfbi_slab_rows_fwd (with jv:
 * the corrections of this slab's rows) -> all-to-all -> kfbi_slab_cols ->
 * all-to-all -> kfbi_slab_rows_inv -> kfbi_slab_stencil_values (u at the
 * extraction stencil nodes in this slab's rows, zero elsewhere;
 * [n_ctl][13]) -> all-reduce(sum) of the values -> kfbi_slab_update
 * (extraction + density update + residual, replicated, identical on every
 * rank); kfbi_rich_begin / kfbi_rich_state open the solve and read its
 * state (iterations, status 1 converged / 2 max_iter, residual, history). */
kfbi_status kfbi_edge_values(kfbi_plan *plan, int32_t dtype, const void *jm, void *jv,
                             void *stream);
kfbi_status kfbi_slab_stencil_values(kfbi_plan *plan, int32_t dtype, int32_t bc_kind,
                                     const kfbi_slab *slab, const void *u_slab, void *vals,
                                     void *stream);
kfbi_status kfbi_rich_begin(kfbi_plan *plan, int32_t max_iter, double tol, void *stream);
kfbi_status kfbi_slab_update(kfbi_plan *plan, int32_t dtype, int32_t bc_kind, const void *vals,
                             const void *jm, const void *g, void *density, void *trace_u,
                             void *trace_un, double gamma, void *stream);
kfbi_status kfbi_rich_state(kfbi_plan *plan, int32_t *iterations, int32_t *done,
                            double *residual, double *history, void *stream);

/* Opt-in restarted GMRES(restart) on the same boundary integral equation
 * (PAPER.md:768, SPEC.md:349 name Krylov solvers as the follow-up to the
 * reference's Richardson iteration): solves T phi = g - t_F for the density,
 * where trace(phi) = t_F + T phi is the affine sweep map of bvp.py:312-323.
 * Krylov vectors come from the pipeline with F = 0, f_gamma = 0, or from the
 * plan's trace operator when use_operator = 1; stopping rule
 * gamma ||g - trace(phi)||_2 <= tol (implies the reference's max-norm rule).
 * Same kfbi_bvp fields as kfbi_richardson (gamma only scales the stopping
 * test); u / traces are the field of the final density; iterations counts
 * matvecs plus full sweeps.  Results differ from Richardson's at the level
 * of tol (a different iterate converging to the same fixed point). */
kfbi_status kfbi_gmres(kfbi_plan *plan, const kfbi_bvp *bvp, int32_t restart,
                       kfbi_bvp_result *result, void *stream);

/* Largest n_ctl the on-chip operator sweeps support on the plan's device
 * (32 rows of T per SM); kfbi_build_trace_operator[_bc] rejects more with
 * KFBI_E_CONFIG and callers use the pipeline form. */
kfbi_status kfbi_operator_max_controls(kfbi_plan *plan, int32_t *n_max);

/* richardson_solve (bvp.py:276-351), device resident: one host sync per
 * batch of sweeps; history copied to result->history. */
kfbi_status kfbi_richardson(kfbi_plan *plan, const kfbi_bvp *bvp,
                            kfbi_bvp_result *result, void *stream);

/* Build the trace operator T (n_ctl x n_ctl, column-major) of the plan's
 * geometry for one kappa: column p is the sweep pipeline (jumps ->
 * corrections -> box solve -> extraction) applied to the unit density e_p
 * with F = 0, f_gamma = 0.  With kfbi_bvp.use_operator = 1, Richardson
 * sweeps k >= 2 evaluate trace_k = trace_1 + T (phi_k - phi_0): the same
 * affine map as the pipeline (bvp.py:313-323), identical iterates up to
 * rounding; sweep 1 and the returned field still run the full pipeline.
 * Costs n_ctl pipeline evaluations once per (geometry, kappa).
 * n_ctl is limited to kfbi_operator_max_controls (KFBI_E_CONFIG beyond). */
kfbi_status kfbi_build_trace_operator(kfbi_plan *plan, int32_t dtype,
                                      double kappa_re, double kappa_im,
                                      void *stream);
/* ... for a Dirichlet (bc_kind 0, T: phi -> u+) or Neumann (bc_kind 1,
 * T: psi -> d_n u+) BVP with the given box closure. */
kfbi_status kfbi_build_trace_operator_bc(kfbi_plan *plan, int32_t dtype, int32_t bc_kind,
                                         int32_t box_bc, double kappa_re,
                                         double kappa_im, void *stream);

/* Time-stepping right-hand sides (timestepping.py), element-wise over n
 * values: the (M+1)^2 grid with the uint8 interior mask, or the n_ctl control
 * points with mask == NULL.  Where a norm pointer is given, max|u_next| (the
 * blow-up norm of StepContext.check_stable, timestepping.py:172-175) is
 * returned after a stream sync. */

/* heat_step (timestepping.py:218-231): u <- mask*u; F_new = a*u - F_old
 * (F_new may alias F_old). */
kfbi_status kfbi_heat_rhs(kfbi_plan *plan, int64_t n, const uint8_t *mask, void *u,
                          const void *F_old, void *F_new, double a,
                          double *norm_out, void *stream);

/* wave_step (timestepping.py:284-302): u_next <- mask*u_next;
 * F_new = (2un - uc) kw + coef (kw un - fc) + (kw uc - fp). */
kfbi_status kfbi_wave_rhs(kfbi_plan *plan, int64_t n, const uint8_t *mask,
                          void *u_next, const void *u_curr, const void *F_curr,
                          const void *F_prev, void *F_new, double kw, double coef,
                          double *norm_out, void *stream);

/* Strang u* (timestepping.py:410-418), complex: mode 0 out = u - 0.5i tau
 * other (other = lap u0); mode 1 out = 2u - other (other = previous u**). */
kfbi_status kfbi_schr_ustar(kfbi_plan *plan, int64_t n, int32_t mode,
                            const void *u, const void *other, double tau,
                            void *out, void *stream);

/* nonlinear_phase_step (timestepping.py:317-368) per node, then the mask
 * (timestepping.py:391) and, when F != NULL, F = kappa * out
 * (timestepping.py:395).  Returns KFBI_E_NOCONV when a node stalls; with
 * max_res == NULL it does not wait and the caller logs the residual
 * (kfbi_log_norm(..., which = 1)). */
kfbi_status kfbi_nonlinear_phase(kfbi_plan *plan, int64_t n, const void *ustar,
                                 const double *v, double w, double half_tau,
                                 const uint8_t *mask, void *out, double kappa_re,
                                 double kappa_im, void *F, double *max_res,
                                 void *stream);

/* Strang B-phase of one step with u* formed inline: u* = u - (i tau/2) other
 * (mode 0, first step, other = lap u0) or 2u - other (mode 1, other = u** of
 * the previous step) (timestepping.py:410-418), then the pointwise Newton of
 * kfbi_nonlinear_phase on u*.  Same results as kfbi_schr_ustar followed by
 * kfbi_nonlinear_phase, without the full-grid u* round trip. */
kfbi_status kfbi_strang_phase(kfbi_plan *plan, int64_t n, int32_t mode, const void *u,
                              const void *other, double tau, const double *v, double w,
                              double half_tau, const uint8_t *mask, void *out,
                              double kappa_re, double kappa_im, void *F,
                              double *max_res, void *stream);

/* dst[i] = src[idx[i]], i < n (device pointers): packs the interior nodes
 * of a masked field (whose exterior is zero by construction) for a compact
 * device -> host copy of a step's result. */
kfbi_status kfbi_gather(kfbi_plan *plan, int32_t dtype, int64_t n, const int32_t *idx,
                        const void *src, void *dst, void *stream);

/* u <- mask*u and max|u| (np.where(ctx.mask, sol.u, 0) + check_stable). */
kfbi_status kfbi_mask_norm(kfbi_plan *plan, int32_t dtype, int64_t n,
                           const uint8_t *mask, void *u, double *norm_out,
                           void *stream);

/* Step log of asynchronous stepping: capacity, the norm of the last
 * *_rhs / mask_norm reduction into a slot, and a synchronous read-back. */
kfbi_status kfbi_log_reserve(kfbi_plan *plan, int32_t count);
kfbi_status kfbi_log_norm(kfbi_plan *plan, int32_t slot, int32_t which, void *stream);
kfbi_status kfbi_log_fetch(kfbi_plan *plan, int32_t first, int32_t count,
                           kfbi_step_log *out, void *stream);
/* Stream-ordered log maintenance for CUDA-graph replays of a step (the
 * graph logs into a fixed slot): zero `count` entries from `slot`, copy
 * `count` entries from `src` to `dst`. */
kfbi_status kfbi_log_clear(kfbi_plan *plan, int32_t slot, int32_t count, void *stream);
/* The caller guarantees that the F_new / out / F buffers it passes with a
 * mask to kfbi_heat_rhs, kfbi_wave_rhs, kfbi_nonlinear_phase and
 * kfbi_strang_phase already hold zeros outside the mask (the stepper's
 * zero-initialised buffer rings): the kernels then skip those stores. */
kfbi_status kfbi_plan_set_exterior_zero(kfbi_plan *plan, int32_t on);
/* The mask's interior nodes (increasing flat indices, caller-owned device
 * array that must outlive its use): with the exterior-zero promise the
 * masked Newton passes (kfbi_nonlinear_phase, kfbi_strang_phase) then visit
 * only these nodes.  idx = NULL clears it. */
kfbi_status kfbi_plan_set_interior_list(kfbi_plan *plan, const int32_t *idx, int64_t count);
/* (odd grid row, 16-node chunk) pairs, host int32[2 * count], covering every
 * node the caller reads of a field returned with kfbi_bvp.field_chunks = 1
 * (interior nodes and six-point stencil nodes); each chunk's windows must
 * lie inside the box (16 chunk >= 64, 16 chunk + 48 <= M - 1). */
kfbi_status kfbi_plan_set_field_chunks(kfbi_plan *plan, const int32_t *pairs, int64_t count);
/* Fractions of the FACR work the reduced solves still do (for roofline
 * accounting): out[0] / out[1] even rows inverse-transformed by a trace-only
 * first sweep / a masked final sweep, out[2] / out[3] odd-row chunks solved
 * by each (1 where the reduction does not apply). */
kfbi_status kfbi_plan_work_fractions(kfbi_plan *plan, double *out);
kfbi_status kfbi_log_copy(kfbi_plan *plan, int32_t src, int32_t dst, int32_t count, void *stream);

/* Per-kernel-name device time (ms) and call counts since the last reset
 * (Backend.timings / calls, engine.py:84-95).  Syncs the plan's events. */
kfbi_status kfbi_kernel_times(kfbi_plan *plan, double *ms, int64_t *calls);
kfbi_status kfbi_reset_kernel_times(kfbi_plan *plan);
kfbi_status kfbi_set_timing(kfbi_plan *plan, int32_t enabled);

/* Launch accounting for bench.py: kernels enqueued since the last reset. */
int64_t kfbi_launch_count(kfbi_plan *plan);

#ifdef __cplusplus
}
#endif

#endif /* KFBI_B200_H */
