/*
 * ig.h -- C ABI of libig.so: B200 (sm_100a) initial guesses for sequences of linear systems
 *         A x_n = b_n, after arXiv 2009.10863 ("PAPER.md" below = /root/reference/PAPER.md).
 *
 * Methods (all fp64):
 *   IG_PROJ_QR       Fischer right-hand-side projection with rolling-QR history updates,
 *                    Algorithm 2 "Rolling QR" (§2).  QR(M).
 *   IG_EXTRAP_LS     Stabilized least-squares polynomial extrapolation, Eq. EXTRAPEXPN
 *                     with weights Eq. LSQRCOEFFS (§3.2).
 *                    EXTRAP(degree, M).
 *   IG_PROJ_CLASSIC  Algorithm 1 "Classic": restart when d >= M.  CLASSIC(M).
 *   IG_EXTRAP_SPARSE Sparse (column-pivoted QR) extrapolation, Eq. CPQRCOEFFS (§3.3).
 *
 * Conventions (every function):
 *   - Vectors are DEVICE pointers to fp64[N] (N = this rank's local length), caller-owned,
 *     unless the name ends in _host (then pinned or pageable HOST pointers).
 *   - Calls enqueue work on the handle's CUDA stream and return without synchronising, except
 *     where stated ("syncs").  Asynchronous CUDA faults surface as IG_E_CUDA at a later call.
 *   - History storage (B~, X~, the solution ring, R) is owned by the library.
 *   - Return value: IG_OK (0) or an ig_status code; ig_last_error() gives a thread-local message.
 *   - A handle is used by one host thread at a time.  Handles are independent (one per field,
 *     PAPER.md:903-907).
 *   - Multi-GPU: every rank calls the same sequence with its contiguous DOF slice.  The
 *     projection's global sums are exchanged either inside the persistent kernels over NVLink
 *     peer memory (ig_attach_peers) or between kernels by an all-gather (ig_attach_comm: NCCL,
 *     or ig_comm_create_local for ranks that are threads of one process); either way the
 *     per-rank partial sums are summed in rank order: bitwise-identical decisions on all ranks.
 *     Extrapolation never communicates.
 */
#ifndef IG_H
#define IG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IG_MAX_HISTORY 32 /* M <= 32 */

typedef struct ig_ctx *ig_t;
typedef struct ig_comm_ctx *ig_comm_t;

enum ig_method {
    IG_PROJ_QR = 1,
    IG_EXTRAP_LS = 2,
    IG_PROJ_CLASSIC = 3,
    IG_EXTRAP_SPARSE = 4
};

enum ig_status {
    IG_OK = 0,
    IG_E_ARG = 1,   /* invalid argument (sizes, method, NULL pointer, misuse)              */
    IG_E_OOM = 2,   /* device allocation failed                                           */
    IG_E_CUDA = 3,  /* CUDA runtime error (also asynchronous faults of earlier calls)      */
    IG_E_NCCL = 4,  /* NCCL could not be loaded or a collective failed                     */
    IG_E_STATE = 5  /* call not valid in the handle's current state                       */
};

/* ---------------------------------------------------------------- lifecycle */

/* Create a handle for vectors of local length N.
 *   method : enum ig_method.
 *   m      : history capacity M (paper's M; BASELINE "m"), 1 <= m <= IG_MAX_HISTORY.
 *   degree : extrapolation degree (paper's m); 0 <= degree <= m-1 (M >= m+1).
 *            Ignored for the projection methods.
 * Allocates the history slabs on the current CUDA device: projection 2*m*N doubles (B~, X~,
 * PAPER.md:310-315), extrapolation m*N doubles (the solution window).  Extrapolation weights
 * (incl. the warm-up table for f < M stored solutions) are built here, on the host, once.
 * Returns NULL on error (see ig_last_error()). */
ig_t ig_create(int64_t N, int method, int m, int degree);

/* As ig_create, but the history slabs live in caller-provided device memory `storage` of
 * `bytes` >= ig_storage_bytes(N, method, m) bytes, 256-byte aligned (e.g. a torch tensor). */
ig_t ig_create_ext(int64_t N, int method, int m, int degree, void *storage, size_t bytes);
size_t ig_storage_bytes(int64_t N, int method, int m);

/* Release the handle (syncs its stream first).  NULL is a no-op. */
void ig_destroy(ig_t h);

/* Forget all history (d = 0 / empty window).  Enqueued on the stream. */
int ig_reset(ig_t h);

const char *ig_last_error(void);

/* Stream all subsequent work of h is enqueued on (a cudaStream_t; NULL = legacy default). */
int ig_set_stream(ig_t h, void *cuda_stream);

/* Projection admission tolerance (AMB-3 reading of PAPER.md:209-215, 246, 302): the new pair is
 * admitted iff ||b~|| > eps_rel * ||A x|| after the two Gram-Schmidt passes.  Default 1e-10
 * (relative).  This deliberately differs from SPEC.md's solver-tied absolute default
 * 10*eps_solver*max(||b~||, 1) (about 1e-7 relative for eps_solver = 1e-8): the paper only says
 * the value "will depend on ... the stopping criterion", and with a CG
 * tolerance of 1e-8 the measured ||b~||/||A x|| floor is 2e-9..5e-8, so the SPEC default rejects
 * most pairs and tripled QR(8)'s CG iterations.  Callers that want the
 * solver-tied rule pass eps_rel = 10 * eps_solver here. */
int ig_set_admit_tol(ig_t h, double eps_rel);

/* Projection kernel schedule.  fused = 1 (default): on a single rank (or with the in-kernel peer
 * exchange, ig_attach_peers) each ig_form_guess / ig_update is ONE persistent kernel whose passes
 * are separated by software grid barriers, so its grid (SMs x occupancy, or ig_set_grid_limit)
 * must be resident at once -- see ig_set_launch.  A barrier that cannot complete gives up after
 * the watchdog time (ig_set_watchdog) and reports IG_E_STATE.  fused = 0, or a handle with an NCCL communicator (ig_attach_comm): one kernel per
 * pass with the NCCL exchange of partial sums between them.  Same arithmetic.  A handle with
 * peers attached (ig_attach_peers) always runs the fused kernels (only they read the exchange
 * windows): ig_set_schedule(h, 0) then returns IG_E_STATE and changes nothing. */
int ig_set_schedule(ig_t h, int fused);

/* Launch mode of the persistent projection kernels.
 *   cooperative = 1 (DEFAULT): cooperative launch (PDL-chained as well).  The driver starts the
 *     grid only when all of its CTAs can be resident, so kernels of OTHER streams that hold SMs
 *     (the solver, a halo exchange, NCCL) delay the launch instead of stalling a grid barrier:
 *     safe next to any concurrent work.
 *   cooperative = 0: ordinary launch.  Correct only while no kernel on another stream holds SMs
 *     until this one finishes (e.g. the GPU is dedicated to this stream); otherwise the barrier
 *     waits for the missing CTAs, up to the watchdog time.  The library orders its own plain
 *     persistent launches across streams of one device (a launch from a different stream than
 *     the previous one first waits for that stream's work).
 *   cooperative = -1: the process default (env IG_LAUNCH: "plain" / "coop", plus "pdl"/"nopdl").
 * Handles with a grid limit (ig_set_grid_limit: virtual ranks sharing one GPU, whose grids are
 * sized to run side by side) default to the ordinary launch.  Results are bitwise identical in
 * every mode (same grid, same reduction order). */
int ig_set_launch(ig_t h, int cooperative);

/* ---------------------------------------------------------------- the hot path */

/* Form the initial guess for A x = b.
 *   Projection (Alg. 2 line 1): if d > 0, x0 <- X~ (B~_{:,1:d}^T b); if d == 0,
 *     x0 is left untouched (it is the caller's "arbitrary input").
 *   Extrapolation (Eq. EXTRAPEXPN): x0 <- sum_i beta_i x_{n-f+i} over the f = min(fill, M) stored
 *     solutions, oldest first; fill == 0 leaves x0 untouched.  b is ignored (may be NULL).
 * x0 may alias b.  x0 may alias ig_next_slot(h) (extrapolation).  Neither may alias other
 * history storage. */
int ig_form_guess(ig_t h, const double *b, double *x0);

/* Update the history with the solution x of the system just solved.
 *   Projection (Alg. 2 after the solve): Ax must be A*x (an explicit operator
 *     apply).  If d == M the oldest pair is dropped by a Givens QR downdate; then
 *     (x, Ax) is orthogonalised by twice-iterated classical Gram-Schmidt and admitted iff
 *     ||b~|| > eps*||Ax|| (d == 0: admitted iff ||Ax|| > 0).
 *     A zero Ax is skipped (d == 0; CLASSIC also at d >= M: no restart).  The sums (||Ax||^2,
 *     the Gram-Schmidt coefficients) are plain fp64 without scaling: ||A x||^2 must stay finite
 *     (entries below ~1e150 in magnitude); NaN/Inf sums leave the pair unadmitted and are
 *     reported as IG_E_STATE by the next synchronising call.
 *   Extrapolation: x is pushed into the solution window (Ax ignored, may be NULL).  If
 *     x == ig_next_slot(h) nothing is copied; otherwise one copy. */
int ig_update(ig_t h, const double *x, const double *Ax);

/* Multi-field batch (one history space per field): handles[i] with b[i], x0[i].
 * Consecutive extrapolation handles on the same device and stream (up to 4) share ONE kernel
 * launch; projection handles run their own persistent kernel.  bs may be NULL if all handles are
 * extrapolation; Axs may be NULL if no handle is a projection.  Same semantics per field as the
 * single-handle calls. */
int ig_form_guess_batch(int n, ig_t *handles, const double *const *bs, double *const *x0s);
int ig_update_batch(int n, ig_t *handles, const double *const *xs, const double *const *Axs);

/* Host-buffer variants (end-to-end path): inputs are copied host->device into handle-owned
 * staging buffers on the stream, the result device->host; these SYNC before returning.
 *   ig_form_guess_host: x0 (in: fallback, out: guess) and b are host arrays of N doubles.
 *   ig_update_host    : x, Ax host arrays (Ax may be NULL for extrapolation). */
int ig_form_guess_host(ig_t h, const double *b, double *x0);
int ig_update_host(ig_t h, const double *x, const double *Ax);

/* Host-buffer batch (several fields of one time step; arguments as in
 * ig_form_guess_batch / ig_update_batch, but host arrays; pinned memory gives the overlap):
 * one synchronisation per call, and the transfers of different fields overlap each other and the
 * kernels -- the extrapolation guesses travel device->host while the projection right-hand sides
 * travel host->device; the extrapolation uploads run while the projection update kernels run.
 * Each handle gets a second (copy) stream on first use.  Same results as the single calls. */
int ig_form_guess_batch_host(int n, ig_t *handles, const double *const *bs, double *const *x0s);
int ig_update_batch_host(int n, ig_t *handles, const double *const *xs, const double *const *Axs);

/* Extrapolation zero-copy slot: the device vector the next ig_update(h, slot, NULL) will push
 * without a copy.  The caller may solve directly into it (it may also be the x0 of
 * ig_form_guess).  NULL for projection methods. */
double *ig_next_slot(ig_t h);

/* ---------------------------------------------------------------- captured time steps */

/* Device-resident extrapolation window (the per-field history spaces of
 * PAPER.md:903-907, the zero-cost push of PAPER.md:1817-1819).  By default the window position
 * (head, fill) lives on the host and every ig_form_guess passes the weights and the solution
 * pointers of the current fill by value -- the fastest form for eager calls, but a captured CUDA
 * graph would replay the pointers of the capture step.  on = 1 moves the position into device
 * memory (a push counter): the extrapolation kernel reads f = min(pushes, M), picks the f stored
 * solutions and the warm-up weights of that f (Eq. LSQRCOEFFS table, nonzero weights only) on
 * the device, and the push kernel writes the solution into slot (pushes mod M) and advances the
 * counter -- no host state per call, so ig_form_guess / ig_update (single or batched) may be
 * captured once and replayed every time step.  Same arithmetic and summation order as the host
 * window (bitwise-identical guesses).  The push copies x unless x already IS the next slot
 * (zero-copy, e.g. x from ig_next_slot).  Switching either way keeps the history (any time).
 * Calls that read the window position on the host (ig_next_slot, ig_history_dim, ig_get_stats,
 * ig_bytes -- which then reports the form at the CURRENT window --, the *_host variants,
 * ig_save_state) sync the stream while on = 1.  Projection handles need nothing: their state is
 * always on the device.  IG_E_ARG for a projection handle; IG_E_OOM if the 33 KB table cannot
 * be allocated.  Capturing an extrapolation call of a handle with a host window returns
 * IG_E_STATE (it would replay stale pointers). */
int ig_set_device_ring(ig_t h, int on);

/* Stream capture of a whole time step (all fields' ig_form_guess... / ig_update... calls, and any
 * other work the caller enqueues on the same stream) into a CUDA graph, replayed with ONE launch
 * per step: removes the host's per-kernel launch cost, which dominates below ~1e6 DOFs.
 *   ig_capture_begin(stream): cudaStreamBeginCapture (thread-local mode) on a NON-default stream;
 *     every handle used in the captured calls must have ig_set_stream(h, stream).
 *   ig_capture_end(stream, &g): ends the capture and instantiates it; *g = NULL on error.
 *   ig_graph_launch(g, stream): one replay (asynchronous on `stream`).
 *   ig_graph_destroy(g): releases it (NULL: no-op).
 * The captured calls bind the device pointers passed at capture time: each step the caller
 * writes its new b / x / Ax into those buffers (or solves into them) before the replay.  A graph
 * refers to its handles' history storage: destroy it before the handles.  Calls that synchronise
 * (ig_history_dim, ig_get_stats, ig_bytes, ig_next_slot of a device window, the *_host variants,
 * checkpoint calls, ig_set_device_ring) must not be issued while capturing (IG_E_STATE or a
 * CUDA capture error).  Begin and end a capture on the same host thread.
 * ig_total_launches() counts the captured libig kernels once per replay, not at capture. */
typedef struct ig_graph_ctx *ig_graph_t;
int ig_capture_begin(void *cuda_stream);
int ig_capture_end(void *cuda_stream, ig_graph_t *out);
int ig_graph_launch(ig_graph_t g, void *cuda_stream);
void ig_graph_destroy(ig_graph_t g);

/* ---------------------------------------------------------------- checkpoint / resume */

/* Host-memory image of one history space (B~, X~, R and the device control block for
 * projection; the solution window, its order and fill for extrapolation) for restarting a long
 * run.  ig_save_state / ig_load_state sync the handle's stream; the image is only valid for a
 * handle created with the same (N, method, m, degree) on any device.  Multi-rank handles save
 * their local shard; all ranks must load images saved at the same step.  Loading restores the
 * history, d / ring position and the admission tolerance saved with it; the handle's own launch
 * and peer-exchange epochs are kept (they only move forward).  A header that does not match the
 * handle, or ring/dimension fields out of range, give IG_E_ARG and leave the handle unchanged.
 * (Checkpoint/resume is an auxiliary subsystem, outside the hot-path scope of SURVEY.md §8.) */
size_t ig_state_bytes(ig_t h);
int ig_save_state(ig_t h, void *host_buf, size_t bytes);
int ig_load_state(ig_t h, const void *host_buf, size_t bytes);

/* ---------------------------------------------------------------- multi-GPU */

/* Write a fresh NCCL unique id (128 bytes) into out (call on one rank, broadcast the bytes). */
int ig_comm_unique_id(void *out128);
/* Create a communicator over nranks processes (one GPU each; current device).  NCCL is loaded
 * at run time (dlopen "libnccl.so.2"); IG_E_NCCL if unavailable. */
int ig_comm_create(int nranks, int rank, const void *id128, ig_comm_t *out);
void ig_comm_destroy(ig_comm_t c);
/* Attach a communicator to a handle (projection: global sums over all ranks).  The handle's
 * N is then the LOCAL slice length; ranks may have different N. */
int ig_attach_comm(ig_t h, ig_comm_t c);

/* In-process communicator: ranks that are threads of ONE process (e.g. several ranks sharing one
 * GPU, where NCCL refuses duplicate devices).  Same all-gather semantics and layout as the NCCL
 * communicator -- each exchange records an event on the calling handle's stream, meets the other
 * ranks at a host barrier, and copies every rank's partial sums (device to device, after that
 * rank's event) into the handle's gather buffer -- so the multi-rank schedule runs unchanged.
 * Every rank must call from its own host thread, the same sequence of calls as the others.
 * ig_local_group_create returns NULL on bad arguments; destroy the group after its comms. */
void *ig_local_group_create(int nranks);
void ig_local_group_destroy(void *group);
int ig_comm_create_local(void *group, int rank, ig_comm_t *out);

/* In-kernel exchange over NVLink peer memory (fused compute + collective):
 * each projection handle owns a small exchange window (ig_xwin_bytes(), < 40 KB); after every
 * reduction pass the persistent kernel's CTA 0 stores the rank-local partial sums into EVERY
 * rank's window and releases an epoch flag (system scope); every CTA acquires the G flags and
 * sums the G contributions in rank order (bitwise-identical on all ranks).  No NCCL launch and
 * no host involvement per step.  Collective setup, all ranks (one handle each):
 *   ig_xwin_export(h, handle64)  -> CUDA IPC handle of this rank's window (64 bytes);
 *   exchange the handles (e.g. torch.distributed all-gather), then
 *   ig_attach_peers(h, nranks, rank, handles (nranks*64 bytes), NULL).
 * Ranks inside ONE process on the same GPU (virtual ranks, used by the single-GPU tests) pass
 * peer_ptrs[r] = ig_xwin_ptr(h_r) instead of IPC handles; such ranks must run on different
 * streams with grids that fit together (ig_set_grid_limit).  nranks <= 8.  All ranks must issue
 * the same sequence of ig_form_guess / ig_update / ig_reset calls. */
size_t ig_xwin_bytes(void);
int ig_xwin_export(ig_t h, void *ipc_handle_out);
void *ig_xwin_ptr(ig_t h);
int ig_attach_peers(ig_t h, int nranks, int rank, const void *ipc_handles, void *const *peer_ptrs);
/* Cap the grid of the persistent kernels (0 = SMs x occupancy). */
int ig_set_grid_limit(ig_t h, int max_blocks);
/* Failure detection: a grid barrier or peer-exchange wait longer than `seconds` (default 10) gives
 * up instead of hanging the GPU and records the event; the next ig_get_stats / ig_history_dim
 * returns IG_E_STATE (the history is then invalid: ig_reset every rank). */
int ig_set_watchdog(ig_t h, double seconds);

/* ---------------------------------------------------------------- introspection (tests/bench) */

/* Current history dimension d (projection) or fill (extrapolation).  Syncs. */
int ig_history_dim(ig_t h, int *d);

/* Extrapolation: the weights used with f stored solutions (1 <= f <= M), oldest first;
 * *len receives f.  f == 0 means the steady-state scheme (f = M). */
int ig_weights(ig_t h, int f, double *beta, int *len);

/* Algorithmic bytes (8 bytes per fp64 value loaded or stored) of the last ig_form_guess and
 * the last ig_update, per the fused schedule in DESIGN.md §7.  Extrapolation counts the solutions
 * actually streamed (nonzero weights) + the x0 write.  Syncs (reads d). */
int ig_bytes(ig_t h, int64_t *form_bytes, int64_t *update_bytes);

typedef struct ig_stats {
    int d;            /* history dimension / fill after the last call                     */
    int admitted;     /* projection: last update admitted its pair (1) or not (0)         */
    double rho;       /* projection: ||b~||/||A x|| of the last update                    */
    double norm_Ax;   /* projection: ||A x|| of the last update                            */
    double norm_bt;   /* projection: ||b~|| after the two Gram-Schmidt passes              */
    int64_t launches; /* kernels this handle has launched since creation                   */
} ig_stats_t;
int ig_get_stats(ig_t h, ig_stats_t *out); /* syncs */

/* Copy the projection state out (syncs).  Bt_dst/Xt_dst: DEVICE buffers of m columns of length
 * ld_dst (column k at +k*ld_dst); R_host: HOST m*m, column-major.  Any pointer may be NULL. */
int ig_copy_history(ig_t h, double *Bt_dst, double *Xt_dst, int64_t ld_dst, double *R_host);

/* Number of CUDA kernels launched by this process through libig (all handles). */
int64_t ig_total_launches(void);

/* Per-kernel timing with CUDA events recorded on the handle's stream around every launch
 * (tracing aid for bench.py's roofline; off by default).  ig_profile(h, 1) clears the counters
 * and turns it on, ig_profile(h, 0) turns it off.  ig_profile_read syncs and returns the summed
 * event time and launch count of one kernel since the last ig_profile call. */
enum ig_kernel {
    IG_K_FORM_DOT = 0,     /* alpha = B~^T b            (paper: rhsProject)               */
    IG_K_FORM_COMBINE = 1, /* x0 = X~ alpha             (paper: rhsReconstruct)           */
    IG_K_U1 = 2,           /* B~ Givens downdate + c1   (paper: rhsQRUpdate + rhsProject) */
    IG_K_U2 = 3,           /* CGS pass 2 dots           (paper: rhsReconstruct+rhsProject)*/
    IG_K_U3 = 4,           /* X~ downdate + store       (paper: rhsUpdateSpace, ...)      */
    IG_K_EXTRAP = 5,       /* x0 = sum beta_i x_i       (paper: extrapKernel)             */
    IG_K_COPY = 6,         /* window push by copy                                        */
    IG_K_FORM_FUSED = 7,   /* persistent form: dots -> grid barrier -> combine           */
    IG_K_UPDATE_FUSED = 8, /* persistent update: U1 -> barrier -> U2 -> barrier -> U3    */
    IG_NKERNELS = 9
};
int ig_profile(ig_t h, int enable);
int ig_profile_read(ig_t h, int kernel, double *total_ms, int64_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* IG_H */
