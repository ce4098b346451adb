// ig_internal.h -- device control block and kernel-launch interface shared by the libig sources.
// Product code only (never includes or is included by oracle/).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace ig {

constexpr int MAXM = 32;       // IG_MAX_HISTORY
constexpr int PS = MAXM + 1;   // partial-sum slots: coefficients 0..MAXM-1, norm^2 at slot MAXM
constexpr int NORM = MAXM;     // slot index of the squared norm
constexpr int MAXB = 1024;     // max blocks of a reduction kernel (block-partial buffer rows)
constexpr int THREADS = 256;   // threads per block of every streaming kernel

enum Stage { ST_FORM = 0, ST_U1 = 1, ST_U2 = 2, ST_U3 = 3, NSTAGE = 4 };
constexpr int MAXG = 8;        // ranks of an in-kernel peer-memory exchange (one NVLink node)
constexpr unsigned long long WATCHDOG_NS = 10ull * 1000 * 1000 * 1000;  // spin-wait limit (10 s)

// Exchange window of one rank, written by every rank over NVLink peer memory (or, for ranks in
// one process, ordinary device memory): data[stage][epoch parity][sender][slot] and a monotonic
// epoch flag per (stage, sender).  Parity double-buffering lets a fast rank publish epoch e+1
// while a slow rank may still be reading epoch e.
struct XWin {
    double data[NSTAGE][2][MAXG][PS];
    unsigned long long flag[NSTAGE][MAXG];
};
struct Exchange {
    XWin *peer[MAXG];  // every rank's window, indexed by rank (peer[rank] == own window)
    int G;             // ranks (0: no peer exchange)
    int rank;
};
enum Method { M_PROJ_QR = 1, M_EXTRAP_LS = 2, M_PROJ_CLASSIC = 3, M_EXTRAP_SPARSE = 4 };

// Device-resident state of one projection handle.  Every control decision (d, downdate,
// admission) is taken on the device from bitwise-identical (rank-ordered) sums, so the host
// never synchronises on the hot path and all ranks agree.
struct Ctrl {
    int d;          // current history dimension
    int pending;    // a QR downdate is due at the next update (d == M after an admission)
    int rotX;       // this update applied the downdate to B~ (U1): U3 must rotate X~
    int deff;       // dimension the Gram-Schmidt passes of the current update use
    int admitted;   // last update admitted its pair
    int last_rot;   // the last update applied a downdate (bytes accounting)
    int err;        // failure detection: 0 ok, 1 grid-barrier / 2 peer-exchange timeout, 3 non-finite sums
    int d_in;       // d at the start of the current update (split schedule: u1 overwrites d)
    unsigned ticket[NSTAGE];
    // Persistent fused kernels: launch epoch e (bumped once per launch that uses a grid barrier);
    // launch e uses the barrier and work-claim counters of parity e & 1 and zeroes those of parity
    // (e + 1) & 1 for the next launch, so no CTA has to wait for the others at exit.
    unsigned epoch;
    unsigned bar[2];               // grid-barrier arrival counters
    unsigned dyn3[2];              // work-claim counters of the dynamically balanced pass-3 tail
    unsigned long long xepoch[NSTAGE];  // completed peer exchanges per stage (all ranks agree)
    double rho, nAx, nb;
    double gc[MAXM], gs[MAXM];      // Givens (c_i, s_i) of the pending downdate
    double R[MAXM * MAXM];          // R, column-major R(i,j) = R[i + j*MAXM]
    double Rdn[MAXM * MAXM];        // R after the pending downdate
};

struct ProjArgs {
    Ctrl *ctrl;
    double *Bt;            // B~ slabs: column k at Bt + k*ld
    double *Xt;            // X~ slabs
    int64_t ld;            // slab stride (doubles), multiple of 32
    int64_t N;             // local vector length
    int M;                 // capacity
    int method;            // M_PROJ_QR or M_PROJ_CLASSIC
    double eps;            // relative admission tolerance
    double *blk;           // block partials [PS][MAXB]
    double *part;          // this rank's partial sums [NSTAGE][PS]
    const double *gath;    // gathered partials [NSTAGE][G][PS] (== part when G == 1)
    int G;                 // ranks
    const double *b;       // form: right-hand side
    double *x0;            // form: guess (out)
    const double *x;       // update: solution
    const double *Ax;      // update: A x
    int max_grid;          // cap on the persistent kernels' grid (0: SMs x occupancy)
    unsigned long long watchdog_ns;  // spin-wait limit of grid barriers / peer exchange
    Exchange xc;           // in-kernel peer exchange (xc.G > 1) for the fused kernels
    int coop;              // persistent kernels: 1 cooperative launch, 0 plain launch (host side only)
};

struct ExtrapArgs {
    const double *src[MAXM];  // stored solutions, oldest first
    double beta[MAXM];        // weights, oldest first
    int f;                    // number of terms
    int pad_;
    int64_t N;
    double *x0;
};

constexpr int MAXF = 4;  // fields per batched extrapolation launch (u_x, u_y, u_z, p)
struct ExtrapBatch {
    ExtrapArgs f[MAXF];
    int nf;
};

// Device-resident solution window (ig_set_device_ring): the push counter lives in device memory
// and the kernels derive the window from it, so form/push calls carry no host-side state and can
// be captured once into a CUDA graph and replayed every time step.
//   cnt = solutions pushed so far; f = min(cnt, M) stored; the j-th oldest (j = 0..f-1) is in
//   slot (cnt - f + j) mod M; the next push goes to slot cnt mod M (the same window as the host
//   ring's head/fill: head = cnt mod M once full).
struct DevRing {
    unsigned long long cnt;
    unsigned ticket;  // CTAs of the running push that have read cnt (the last one advances it)
    unsigned pad_;
};
struct RingTab {      // per fill f = 1..M (row f-1): the nonzero weights, oldest first
    int nnz[MAXM];
    int jidx[MAXM][MAXM];
    double beta[MAXM][MAXM];
};
struct RingArgs {
    DevRing *ring;
    const RingTab *tab;
    double *base;      // slot k at base + k*ld
    int64_t ld;
    int64_t N;
    int M;
    int pad_;
    double *x0;        // form: guess (out)
    const double *x;   // push: solution (in)
};
struct RingBatch {
    RingArgs f[MAXF];
    int nf;
};

// ----------------------------------------------------------------------------- launch policy
// Process-wide launch defaults (env IG_LAUNCH, comma list of "coop", "plain", "pdl", "nopdl";
// default coop + pdl; a handle overrides the coop choice with ig_set_launch):
//   coop: persistent fused kernels use cooperative launch: the driver only starts the grid when
//         all of its CTAs can be resident, so a kernel of another stream (a halo exchange, NCCL,
//         the solver) holding SMs delays the launch instead of stalling a grid barrier.
//   plain: ordinary launch; relies on grid = SMs x occupancy being resident at once, which holds
//         whenever no other stream pins SMs (ig_set_launch documents the trade).
//   pdl : programmatic dependent launch: every libig kernel may be launched while its stream
//         predecessor is finishing; each kernel executes griddepcontrol.wait (waits for the full
//         completion + memory flush of the predecessor) before touching memory, and triggers its
//         dependents once its streaming passes are done (C2: 232.2 -> 224.3 us/step).
struct LaunchFlags {
    bool coop = true;
    bool pdl = true;
};
LaunchFlags launch_flags();

#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... Exp, typename... Act>
static cudaError_t launch_ex(void (*kern)(Exp...), int grid, cudaStream_t s, bool coop, Act &&...args) {
    const LaunchFlags f = launch_flags();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (coop) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na].val.cooperative = 1;
        ++na;
    }
    if (f.pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
}
#endif

// Launchers (kern_proj.cu / kern_extrap.cu).  `vec` = 2 when every vector is 16-byte aligned.
// Return the cudaError_t of the launch.  *blocks receives the grid size used.
cudaError_t launch_form_dot(const ProjArgs &a, int vec, int nsm, cudaStream_t s);
cudaError_t launch_form_combine(const ProjArgs &a, int vec, int nsm, cudaStream_t s);
cudaError_t launch_u1(const ProjArgs &a, int vec, int nsm, cudaStream_t s);
cudaError_t launch_u2(const ProjArgs &a, int vec, int nsm, cudaStream_t s);
cudaError_t launch_u3(const ProjArgs &a, int vec, int nsm, cudaStream_t s);
// Persistent fused kernels (single GPU / peer exchange): one launch per call (see launch policy).
cudaError_t launch_form_fused(const ProjArgs &a, int vec, int nsm, cudaStream_t s);
cudaError_t launch_update_fused(const ProjArgs &a, int vec, int nsm, cudaStream_t s);
cudaError_t launch_extrap(const ExtrapArgs &a, int vec, int nsm, cudaStream_t s);
cudaError_t launch_extrap_batch(const ExtrapBatch &b, int vec, int nsm, cudaStream_t s);
cudaError_t launch_copy(double *dst, const double *src, int64_t N, int vec, int nsm, cudaStream_t s);
// Device-ring extrapolation (one launch for up to MAXF fields; fc = max nonzero weights over all
// fills of all fields, so the launch never depends on the current fill).
cudaError_t launch_extrap_ring(const RingBatch &b, int fc, int vec, int nsm, cudaStream_t s);
cudaError_t launch_push_ring(const RingBatch &b, int vec, int nsm, cudaStream_t s);

// Cached cudaOccupancyMaxActiveBlocksPerMultiprocessor(kernel, THREADS) (api.cpp); the query is
// ~microseconds of host time, paid once per kernel instantiation instead of per launch.
int cached_occupancy(const void *kernel);

// Host weight builders (coeffs.cpp).
// EXTRAP(m, M) least-squares weights, oldest first (Householder QR of the Legendre Vandermonde).
int build_ls_weights(int m, int M, double *beta);
// Theorem 3.1 naive weights (exact binomials).
void build_naive_weights(int M, double *beta);
// Sparse CPQR weights (Eq. CPQRCOEFFS); returns nonzero count or -1.
int build_sparse_weights(int m, int M, double *beta);

}  // namespace ig
