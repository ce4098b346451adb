// api.cpp -- libig C ABI (include/ig.h): handles, history storage, stream-ordered launch
// sequence of the hot path, NCCL exchange of the projection's partial sums, host staging.
//
// Per-step launch sequence (all asynchronous on the handle's stream, no host sync):
//   PROJ  form   : k_form_dot -> [all-gather alpha partials] -> k_form_combine
//         update : k_u1 -> [all-gather] -> k_u2 -> [all-gather] -> k_u3
//   EXTRAP form  : k_extrap (weights + slot pointers by value)
//          update: ring bump (0 bytes) or k_copy
#include <dlfcn.h>

#include <atomic>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "ig.h"
#include "ig_internal.h"

using namespace ig;

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

static int set_err(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_OK(expr)                                                                          \
    do {                                                                                       \
        cudaError_t e_ = (expr);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            return set_err(IG_E_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

ig::LaunchFlags ig::launch_flags() {
    static LaunchFlags f = [] {
        LaunchFlags r;
        const char *e = getenv("IG_LAUNCH");
        if (e) {
            std::string v(e);
            if (v.find("coop") != std::string::npos) r.coop = true;
            if (v.find("plain") != std::string::npos || v == "none" || v == "pdl") r.coop = false;
            r.pdl = v.find("pdl") != std::string::npos && v.find("nopdl") == std::string::npos;
        }
        return r;
    }();
    return f;
}

int ig::cached_occupancy(const void *kernel) {
    static std::mutex mu;
    static std::unordered_map<const void *, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(kernel);
    if (it != cache.end()) return it->second;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, THREADS, 0) != cudaSuccess) {
        cudaGetLastError();
        occ = 0;
    }
    cache[kernel] = occ;
    return occ;
}

// ----------------------------------------------------------------------------- NCCL (dlopen)
namespace {
typedef int ncclResult_t;
typedef void *ncclComm_t;
struct ncclUniqueId {
    char internal[128];
};
const int ncclFloat64 = 8;  // nccl.h: ncclFloat64 = 8

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char *(*errStr)(ncclResult_t) = nullptr;
};

NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *env = getenv("IG_NCCL_PATH");
        void *lib = nullptr;
        if (env && *env) lib = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            api.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return;
        }
        api.getUniqueId = (decltype(api.getUniqueId))dlsym(lib, "ncclGetUniqueId");
        api.commInitRank = (decltype(api.commInitRank))dlsym(lib, "ncclCommInitRank");
        api.allGather = (decltype(api.allGather))dlsym(lib, "ncclAllGather");
        api.commDestroy = (decltype(api.commDestroy))dlsym(lib, "ncclCommDestroy");
        api.errStr = (decltype(api.errStr))dlsym(lib, "ncclGetErrorString");
        api.ok = api.getUniqueId && api.commInitRank && api.allGather && api.commDestroy && api.errStr;
        if (!api.ok) api.why = "libnccl.so.2 lacks required symbols";
    });
    return api;
}
}  // namespace

// In-process rank group (ig_local_group_create): a host barrier plus the per-rank "partials
// ready" events and source pointers of the exchange in progress.
struct LocalGroup {
    int n = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    std::vector<cudaEvent_t> ready;
    std::vector<const double *> src;
    explicit LocalGroup(int n_) : n(n_), ready(n_, nullptr), src(n_, nullptr) {
        for (auto &e : ready) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    ~LocalGroup() {
        for (auto e : ready)
            if (e) cudaEventDestroy(e);
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const unsigned long long g = gen;
        if (++arrived == n) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct ig_comm_ctx {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    LocalGroup *local = nullptr;  // in-process group instead of NCCL
};

// ----------------------------------------------------------------------------- handle
struct ig_ctx {
    int64_t N = 0, ld = 0;
    int method = 0, M = 0, degree = 0;
    double eps = 1e-10;
    cudaStream_t stream = nullptr;
    int dev = 0, nsm = 148;
    double *slab = nullptr;
    size_t slab_bytes = 0;
    bool own_slab = false;
    // projection
    double *Bt = nullptr, *Xt = nullptr;
    Ctrl *ctrl = nullptr;
    double *blk = nullptr, *part = nullptr, *gath = nullptr;
    int G = 1;
    bool fused = true;  // persistent fused kernels when G == 1 (ig_set_schedule)
    ig_comm_ctx *comm = nullptr;
    int max_grid = 0;   // ig_set_grid_limit
    int coop = -1;      // ig_set_launch: 1 cooperative, 0 plain, -1 process default (IG_LAUNCH)
    unsigned long long watchdog_ns = WATCHDOG_NS;  // ig_set_watchdog
    // in-kernel peer exchange (ig_attach_peers)
    XWin *xwin = nullptr;
    Exchange xc = {};
    std::vector<void *> ipc_opened;
    // extrapolation
    std::vector<std::vector<double>> table;  // table[f-1]: weights for f stored solutions
    std::vector<double *> slots;
    int head = 0, fill = 0;     // host window (ignored while dring: the device counter rules)
    bool last_copy = false;
    // device-resident window (ig_set_device_ring): graph-capturable form / push
    bool dring = false;
    DevRing *ring = nullptr;
    RingTab *rtab = nullptr;
    int ring_fc = 0;            // max nonzero weights over every fill (kernel bucket)
    RingTab rtab_host;
    int last_form_f = 0;
    // host staging (end-to-end path)
    double *stage[4] = {nullptr, nullptr, nullptr, nullptr};
    int known_d = 0;  // projection d as of the last synchronising host-buffer call (-1: unknown)
    cudaStream_t cstream = nullptr;  // batch host calls: copies that overlap the handle's stream
    cudaEvent_t cev[2] = {nullptr, nullptr};
    int *pin_ctrl = nullptr;         // pinned copy of the control block's leading ints (d ... err)
    int64_t launches = 0;
    // per-kernel CUDA-event timing (ig_profile)
    bool profiling = false;
    std::vector<cudaEvent_t> ev_pool;
    struct Rec { int kid; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    double prof_ms[IG_NKERNELS] = {0};
    int64_t prof_n[IG_NKERNELS] = {0};
};

namespace {
bool is_proj(int m) { return m == IG_PROJ_QR || m == IG_PROJ_CLASSIC; }
bool is_extrap(int m) { return m == IG_EXTRAP_LS || m == IG_EXTRAP_SPARSE; }
int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }
bool al16(const void *p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

void count(ig_t h, int n) {
    h->launches += n;
    g_launches += n;
}

cudaEvent_t pool_get(ig_t h) {
    if (!h->ev_pool.empty()) {
        cudaEvent_t e = h->ev_pool.back();
        h->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Brackets one kernel launch with CUDA events on the handle's stream when profiling is on.
struct Prof {
    ig_t h;
    int kid;
    cudaEvent_t a = nullptr;
    Prof(ig_t h_, int kid_) : h(h_), kid(kid_) {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        if (h->profiling && cudaStreamIsCapturing(h->stream, &cap) != cudaSuccess) cudaGetLastError();
        if (h->profiling && cap == cudaStreamCaptureStatusNone) {  // events cannot time a capture
            a = pool_get(h);
            cudaEventRecord(a, h->stream);
        }
    }
    ~Prof() {
        if (a) {
            cudaEvent_t b = pool_get(h);
            cudaEventRecord(b, h->stream);
            h->recs.push_back({kid, a, b});
        }
    }
};

void prof_drain(ig_t h) {
    for (auto &r : h->recs) {
        float ms = 0.f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&ms, r.a, r.b);
        h->prof_ms[r.kid] += ms;
        h->prof_n[r.kid] += 1;
        h->ev_pool.push_back(r.a);
        h->ev_pool.push_back(r.b);
    }
    h->recs.clear();
}

ProjArgs proj_args(ig_t h) {
    ProjArgs a;
    memset(&a, 0, sizeof a);
    a.ctrl = h->ctrl;
    a.Bt = h->Bt;
    a.Xt = h->Xt;
    a.ld = h->ld;
    a.N = h->N;
    a.M = h->M;
    a.method = h->method == IG_PROJ_QR ? M_PROJ_QR : M_PROJ_CLASSIC;
    a.eps = h->eps;
    a.blk = h->blk;
    a.part = h->part;
    a.gath = h->gath;
    a.G = h->G;
    a.max_grid = h->max_grid;
    a.watchdog_ns = h->watchdog_ns;
    a.xc = h->xc;
    // default: cooperative, except grid-limited handles (ranks sharing one GPU, ig_set_grid_limit),
    // whose grids are sized to be co-resident with their peers' grids and must run concurrently
    a.coop = h->coop >= 0 ? h->coop : ((launch_flags().coop && h->max_grid == 0) ? 1 : 0);
    return a;
}

// Fused persistent kernels are used on one rank and with the in-kernel peer exchange; a NCCL
// communicator without peer windows uses one kernel per pass with NCCL between them.
// Peers attached (ig_attach_peers) always use the fused kernels: only they read the exchange
// windows (the split kernels would sum this rank's partials alone).
bool use_fused(ig_t h) { return h->xc.G > 1 || (h->fused && h->G == 1); }

// Plain-launched (ig_set_launch(h, 0)) full-grid persistent kernels of DIFFERENT streams on one
// device must not overlap: each needs its whole grid resident at once, and two grids whose
// CTAs interleave could each wait at a barrier for CTAs the other one holds.  Handles sharing a
// stream are ordered by the stream (the common case: nothing to do); a persistent launch from a
// different stream than the previous one on this device first waits for everything enqueued on
// that stream (one event).  Handles with a grid limit (ig_set_grid_limit: ranks sharing a GPU)
// are exempt -- their grids are sized to be co-resident.  The lock spans the launch, so two host
// threads cannot slip their kernels in between.
struct PersistOrder {
    std::mutex mu;
    cudaStream_t last = nullptr;
    bool any = false;
    cudaEvent_t ev = nullptr;
};
PersistOrder &persist_order(int dev) {
    static PersistOrder po[64];
    return po[dev & 63];
}
template <class F> int persistent_launch(ig_t h, F &&launch) {
    if (h->max_grid > 0) return launch();
    if (proj_args(h).coop) return launch();  // cooperative: the driver guarantees co-residency
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(h->stream, &cap) != cudaSuccess) cudaGetLastError();
    if (cap != cudaStreamCaptureStatusNone) return launch();  // graph capture: replays order themselves
    PersistOrder &p = persist_order(h->dev);
    std::lock_guard<std::mutex> lk(p.mu);
    if (p.any && p.last != h->stream) {
        if (!p.ev) CUDA_OK(cudaEventCreateWithFlags(&p.ev, cudaEventDisableTiming));
        if (cudaEventRecord(p.ev, p.last) == cudaSuccess) CUDA_OK(cudaStreamWaitEvent(h->stream, p.ev, 0));
        else cudaGetLastError();  // that stream no longer exists: its work was submitted before ours
    }
    p.last = h->stream;
    p.any = true;
    return launch();
}

int exchange(ig_t h, int stage) {
    if (h->G <= 1) return IG_OK;
    if (LocalGroup *g = h->comm->local) {  // all-gather among the threads of this process
        const int r = h->comm->rank;
        CUDA_OK(cudaEventRecord(g->ready[r], h->stream));
        g->src[r] = h->part + stage * PS;
        g->barrier();  // every rank's partials are enqueued, pointers published
        for (int q = 0; q < g->n; ++q) {
            CUDA_OK(cudaStreamWaitEvent(h->stream, g->ready[q], 0));
            CUDA_OK(cudaMemcpyAsync(h->gath + ((size_t)stage * h->G + q) * PS, g->src[q], sizeof(double) * PS,
                                    cudaMemcpyDeviceToDevice, h->stream));
        }
        g->barrier();  // every rank has enqueued its waits: the events / pointers may be reused
        return IG_OK;
    }
    NcclApi &api = nccl();
    ncclResult_t r = api.allGather(h->part + stage * PS, h->gath + (size_t)stage * h->G * PS, PS, ncclFloat64,
                                   h->comm->comm, h->stream);
    if (r != 0) return set_err(IG_E_NCCL, "ncclAllGather: %s", api.errStr(r));
    return IG_OK;
}

int slot_index(ig_t h, int j) { return (h->head + j) % h->M; }  // j-th oldest stored solution

// Extrapolation kernel arguments for the current fill; false when there is nothing to do.
// Only nonzero weights are streamed (exact zeros contribute exactly nothing): SPEXTRAP reads its
// m+1 selected solutions (Table 1: (m+2)N), LS skips e.g. beta_4 = 0 of EXTRAP(3,8).
bool extrap_args(ig_t h, double *x0, ExtrapArgs &a, bool &aligned) {
    const int f = h->fill < h->M ? h->fill : h->M;
    h->last_form_f = 0;
    if (f == 0) return false;
    memset(&a, 0, sizeof a);
    a.N = h->N;
    a.x0 = x0;
    aligned = al16(x0);
    int nz = 0;
    for (int j = 0; j < f; ++j) {
        const double bj = h->table[f - 1][j];
        if (bj == 0.0) continue;
        a.src[nz] = h->slots[slot_index(h, j)];
        a.beta[nz] = bj;
        aligned = aligned && al16(a.src[nz]);
        ++nz;
    }
    a.f = nz;
    h->last_form_f = nz;
    return true;
}
double *next_slot_ptr(ig_t h) { return h->fill < h->M ? h->slots[slot_index(h, h->fill)] : h->slots[h->head]; }

bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return cap != cudaStreamCaptureStatusNone;
}

// Device window <-> host window: cnt = fill while filling, M + head once full (cnt mod M = head).
unsigned long long ring_cnt_of(ig_t h) { return h->fill < h->M ? (unsigned long long)h->fill : (unsigned long long)(h->M + h->head); }
void ring_set_host(ig_t h, unsigned long long cnt) {
    h->fill = cnt < (unsigned long long)h->M ? (int)cnt : h->M;
    h->head = cnt < (unsigned long long)h->M ? 0 : (int)(cnt % (unsigned long long)h->M);
}
// Host mirror of a device window (syncs the stream): for the introspection / checkpoint calls.
int ring_pull(ig_t h) {
    if (!h->dring) return IG_OK;
    if (capturing(h->stream))  // a synchronising read would invalidate the caller's capture
        return set_err(IG_E_STATE, "the device window position cannot be read while the stream is being captured");
    DevRing r;
    CUDA_OK(cudaMemcpyAsync(&r, h->ring, sizeof r, cudaMemcpyDeviceToHost, h->stream));
    CUDA_OK(cudaStreamSynchronize(h->stream));
    ring_set_host(h, r.cnt);
    return IG_OK;
}
int ring_push_host(ig_t h) {  // host window -> device counter (enqueued; syncs: r is a stack object)
    if (!h->dring) return IG_OK;
    if (capturing(h->stream))
        return set_err(IG_E_STATE, "the device window cannot be (re)positioned while the stream is being captured");
    DevRing r = {ring_cnt_of(h), 0u, 0u};
    CUDA_OK(cudaMemcpyAsync(h->ring, &r, sizeof r, cudaMemcpyHostToDevice, h->stream));
    CUDA_OK(cudaStreamSynchronize(h->stream));
    return IG_OK;
}
bool in_slab(ig_t h, const double *p) { return p >= h->slab && p < h->slab + (size_t)h->M * h->ld; }
RingArgs ring_args(ig_t h) {
    RingArgs r;
    memset(&r, 0, sizeof r);
    r.ring = h->ring;
    r.tab = h->rtab;
    r.base = h->slab;
    r.ld = h->ld;
    r.N = h->N;
    r.M = h->M;
    return r;
}

ig_t create_impl(int64_t N, int method, int m, int degree, void *storage, size_t bytes) {
    if (N < 1) return set_err(IG_E_ARG, "N must be >= 1 (got %lld)", (long long)N), nullptr;
    if (!is_proj(method) && !is_extrap(method)) return set_err(IG_E_ARG, "unknown method %d", method), nullptr;
    if (m < 1 || m > IG_MAX_HISTORY)
        return set_err(IG_E_ARG, "history size m must be in [1, %d] (got %d)", IG_MAX_HISTORY, m), nullptr;
    if (is_extrap(method) && (degree < 0 || degree > m - 1))
        return set_err(IG_E_ARG, "degree must satisfy 0 <= degree <= m-1 (PAPER.md:416; got %d, m=%d)", degree, m),
               nullptr;
    ig_t h = new ig_ctx;
    h->N = N;
    h->method = method;
    h->M = m;
    h->degree = is_extrap(method) ? degree : 0;
    h->ld = round_up(N, 32);
    if (cudaGetDevice(&h->dev) != cudaSuccess) {
        set_err(IG_E_CUDA, "no CUDA device");
        delete h;
        return nullptr;
    }
    cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, h->dev);
    const size_t need = ig_storage_bytes(N, method, m);
    if (storage) {
        if (bytes < need || (reinterpret_cast<uintptr_t>(storage) & 255)) {
            set_err(IG_E_ARG, "storage too small (%zu < %zu) or not 256-byte aligned", bytes, need);
            delete h;
            return nullptr;
        }
        h->slab = static_cast<double *>(storage);
    } else {
        if (cudaMalloc(&h->slab, need) != cudaSuccess) {
            cudaGetLastError();
            set_err(IG_E_OOM, "cudaMalloc(%zu) for the history slabs failed", need);
            delete h;
            return nullptr;
        }
        h->own_slab = true;
    }
    h->slab_bytes = need;
    if (is_proj(method)) {
        h->Bt = h->slab;
        h->Xt = h->slab + (size_t)m * h->ld;
        bool ok = cudaMalloc(&h->ctrl, sizeof(Ctrl)) == cudaSuccess &&
                  cudaMalloc(&h->blk, 2 * sizeof(double) * PS * MAXB) == cudaSuccess &&
                  cudaMalloc(&h->part, sizeof(double) * PS * NSTAGE) == cudaSuccess;
        if (!ok || cudaMemset(h->ctrl, 0, sizeof(Ctrl)) != cudaSuccess ||
            cudaMemset(h->part, 0, sizeof(double) * PS * NSTAGE) != cudaSuccess) {
            cudaGetLastError();
            set_err(IG_E_OOM, "control-block allocation failed");
            ig_destroy(h);
            return nullptr;
        }
        h->gath = h->part;  // G == 1: [NSTAGE][1][PS] == [NSTAGE][PS]
    } else {
        for (int k = 0; k < m; ++k) h->slots.push_back(h->slab + (size_t)k * h->ld);
        h->table.resize(m);
        for (int f = 1; f <= m; ++f) {
            const int q = degree < f - 1 ? degree : f - 1;  // warm-up rule (AMB-13)
            h->table[f - 1].assign(f, 0.0);
            const int rc = method == IG_EXTRAP_LS ? build_ls_weights(q, f, h->table[f - 1].data())
                                                  : build_sparse_weights(q, f, h->table[f - 1].data());
            if (rc < 0) {
                set_err(IG_E_ARG, "weight builder failed for (%d, %d)", q, f);
                ig_destroy(h);
                return nullptr;
            }
        }
    }
    g_err.clear();
    return h;
}
}  // namespace

extern "C" {

size_t ig_storage_bytes(int64_t N, int method, int m) {
    if (N < 1 || m < 1) return 0;
    const size_t vec = sizeof(double) * (size_t)round_up(N, 32);
    return (is_proj(method) ? 2u : 1u) * (size_t)m * vec;
}

ig_t ig_create(int64_t N, int method, int m, int degree) { return create_impl(N, method, m, degree, nullptr, 0); }

ig_t ig_create_ext(int64_t N, int method, int m, int degree, void *storage, size_t bytes) {
    if (!storage) return set_err(IG_E_ARG, "storage is NULL"), nullptr;
    return create_impl(N, method, m, degree, storage, bytes);
}

void ig_destroy(ig_t h) {
    if (!h) return;
    DevGuard g(h->dev);
    if (h->stream) cudaStreamSynchronize(h->stream);
    else cudaDeviceSynchronize();
    if (h->own_slab) cudaFree(h->slab);
    cudaFree(h->ring);
    cudaFree(h->rtab);
    cudaFree(h->ctrl);
    cudaFree(h->blk);
    if (h->gath != h->part) cudaFree(h->gath);
    cudaFree(h->part);
    for (auto &s : h->stage) cudaFree(s);
    for (auto e : h->cev)
        if (e) cudaEventDestroy(e);
    if (h->cstream) cudaStreamDestroy(h->cstream);
    if (h->pin_ctrl) cudaFreeHost(h->pin_ctrl);
    for (void *p : h->ipc_opened) cudaIpcCloseMemHandle(p);
    cudaFree(h->xwin);
    prof_drain(h);
    for (auto e : h->ev_pool) cudaEventDestroy(e);
    delete h;
}

const char *ig_last_error(void) { return g_err.c_str(); }

int ig_set_stream(ig_t h, void *s) {
    if (!h) return set_err(IG_E_ARG, "NULL handle");
    h->stream = static_cast<cudaStream_t>(s);
    return IG_OK;
}

int ig_set_schedule(ig_t h, int fused) {
    if (!h) return set_err(IG_E_ARG, "NULL handle");
    if (!fused && h->xc.G > 1)
        return set_err(IG_E_STATE, "peers are attached: the in-kernel exchange needs the fused schedule");
    h->fused = fused != 0;
    return IG_OK;
}

int ig_set_admit_tol(ig_t h, double eps) {
    if (!h || !(eps >= 0.0)) return set_err(IG_E_ARG, "bad handle or eps");
    h->eps = eps;
    return IG_OK;
}

int ig_reset(ig_t h) {
    if (!h) return set_err(IG_E_ARG, "NULL handle");
    DevGuard g(h->dev);
    if (is_proj(h->method)) {
        // everything but the peer-exchange epochs, which stay monotonic across resets (every
        // rank resets at the same point of the call sequence)
        CUDA_OK(cudaMemsetAsync(h->ctrl, 0, offsetof(Ctrl, xepoch), h->stream));
        const size_t tail = offsetof(Ctrl, xepoch) + sizeof(((Ctrl *)0)->xepoch);
        CUDA_OK(cudaMemsetAsync(reinterpret_cast<char *>(h->ctrl) + tail, 0, sizeof(Ctrl) - tail, h->stream));
    }
    h->head = h->fill = 0;
    h->known_d = 0;
    if (h->dring) CUDA_OK(cudaMemsetAsync(h->ring, 0, sizeof(DevRing), h->stream));
    return IG_OK;
}

namespace {
struct StateHeader {
    uint64_t magic;  // "IGSTATE1"
    int32_t method, M, degree, head;
    int64_t N;
    int32_t fill, nslab;
    double eps;
};
const uint64_t STATE_MAGIC = 0x3145544154534749ull;  // "IGSTATE1" little-endian
int nslabs(ig_t h) { return is_proj(h->method) ? 2 * h->M : h->M; }
}  // namespace

size_t ig_state_bytes(ig_t h) {
    if (!h) return 0;
    return sizeof(StateHeader) + (is_proj(h->method) ? sizeof(Ctrl) : 0) +
           sizeof(double) * (size_t)nslabs(h) * (size_t)h->N;
}

int ig_save_state(ig_t h, void *host_buf, size_t bytes) {
    if (!h || !host_buf || bytes < ig_state_bytes(h)) return set_err(IG_E_ARG, "bad handle or buffer too small");
    DevGuard g(h->dev);
    int rc = ring_pull(h);
    if (rc) return rc;
    char *p = static_cast<char *>(host_buf);
    StateHeader hd = {STATE_MAGIC, h->method, h->M, h->degree, h->head, h->N, h->fill, nslabs(h), h->eps};
    memcpy(p, &hd, sizeof hd);
    p += sizeof hd;
    if (is_proj(h->method)) {
        CUDA_OK(cudaMemcpyAsync(p, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, h->stream));
        p += sizeof(Ctrl);
    }
    const size_t w = sizeof(double) * (size_t)h->N;
    CUDA_OK(cudaMemcpy2DAsync(p, w, h->slab, sizeof(double) * h->ld, w, nslabs(h), cudaMemcpyDeviceToHost,
                              h->stream));
    CUDA_OK(cudaStreamSynchronize(h->stream));
    return IG_OK;
}

int ig_load_state(ig_t h, const void *host_buf, size_t bytes) {
    if (!h || !host_buf || bytes < sizeof(StateHeader)) return set_err(IG_E_ARG, "bad handle or buffer");
    DevGuard g(h->dev);
    const char *p = static_cast<const char *>(host_buf);
    StateHeader hd;
    memcpy(&hd, p, sizeof hd);
    if (hd.magic != STATE_MAGIC) return set_err(IG_E_ARG, "not an ig state image");
    if (hd.method != h->method || hd.M != h->M || hd.degree != h->degree || hd.N != h->N)
        return set_err(IG_E_ARG, "state image is for (method %d, N %lld, m %d, degree %d)", hd.method,
                       (long long)hd.N, hd.M, hd.degree);
    if (bytes < ig_state_bytes(h)) return set_err(IG_E_ARG, "state image truncated");
    if (hd.nslab != nslabs(h) || hd.head < 0 || hd.head >= h->M || hd.fill < 0 || hd.fill > h->M ||
        !(hd.eps >= 0.0))
        return set_err(IG_E_ARG, "corrupt state image (nslab %d, head %d, fill %d)", hd.nslab, hd.head, hd.fill);
    p += sizeof hd;
    if (is_proj(h->method)) {
        Ctrl c;
        memcpy(&c, p, sizeof c);
        if (c.d < 0 || c.d > h->M || c.deff < 0 || c.deff > h->M)
            return set_err(IG_E_ARG, "corrupt state image (d %d)", c.d);
        for (unsigned &t : c.ticket) t = 0;  // transient launch state is never part of a checkpoint
        c.bar[0] = c.bar[1] = c.dyn3[0] = c.dyn3[1] = 0;
        c.err = 0;
        // the live handle's launch epoch and peer-exchange epochs stay: every rank's window flags
        // only move forward (an older image's epochs would let the next exchange pass on stale
        // flags), and the barrier counters zeroed above belong to the live epoch's parities
        Ctrl live;
        CUDA_OK(cudaMemcpyAsync(&live, h->ctrl, sizeof live, cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        c.epoch = live.epoch;
        memcpy(c.xepoch, live.xepoch, sizeof c.xepoch);
        CUDA_OK(cudaMemcpyAsync(h->ctrl, &c, sizeof c, cudaMemcpyHostToDevice, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));  // c is a stack object
        p += sizeof(Ctrl);
        h->known_d = -1;
    }
    const size_t w = sizeof(double) * (size_t)h->N;
    CUDA_OK(cudaMemcpy2DAsync(h->slab, sizeof(double) * h->ld, p, w, w, nslabs(h), cudaMemcpyHostToDevice,
                              h->stream));
    CUDA_OK(cudaStreamSynchronize(h->stream));
    h->head = hd.head;
    h->fill = hd.fill;
    h->eps = hd.eps;
    return ring_push_host(h);
}

int ig_form_guess(ig_t h, const double *b, double *x0) {
    if (!h) return set_err(IG_E_ARG, "NULL handle");
    if (!x0) return set_err(IG_E_ARG, "x0 is NULL");
    DevGuard g(h->dev);
    if (is_proj(h->method)) {
        if (!b) return set_err(IG_E_ARG, "b is NULL");
        ProjArgs a = proj_args(h);
        a.b = b;
        a.x0 = x0;
        const int vec = (al16(b) && al16(x0)) ? 2 : 1;
        if (use_fused(h)) {
            int rc = persistent_launch(h, [&]() -> int {
                Prof p(h, IG_K_FORM_FUSED);
                CUDA_OK(launch_form_fused(a, vec, h->nsm, h->stream));
                return IG_OK;
            });
            if (rc) return rc;
            count(h, 1);
            return IG_OK;
        }
        {
            Prof p(h, IG_K_FORM_DOT);
            CUDA_OK(launch_form_dot(a, vec, h->nsm, h->stream));
        }
        int rc = exchange(h, ST_FORM);
        if (rc) return rc;
        {
            Prof p(h, IG_K_FORM_COMBINE);
            CUDA_OK(launch_form_combine(a, vec, h->nsm, h->stream));
        }
        count(h, 2);
        return IG_OK;
    }
    if (h->dring) {  // device window: f, slots and weights are read on the device
        RingBatch rb;
        memset(&rb, 0, sizeof rb);
        rb.f[0] = ring_args(h);
        rb.f[0].x0 = x0;
        rb.nf = 1;
        Prof p(h, IG_K_EXTRAP);
        CUDA_OK(launch_extrap_ring(rb, h->ring_fc, al16(x0) ? 2 : 1, h->nsm, h->stream));
        count(h, 1);
        return IG_OK;
    }
    if (capturing(h->stream))
        return set_err(IG_E_STATE, "extrapolation window is host-side: ig_set_device_ring(h, 1) before capturing");
    ExtrapArgs a;
    bool aligned = true;
    if (!extrap_args(h, x0, a, aligned)) return IG_OK;  // fill == 0: x0 untouched (AMB-13)
    {
        Prof p(h, IG_K_EXTRAP);
        CUDA_OK(launch_extrap(a, aligned ? 2 : 1, h->nsm, h->stream));
    }
    count(h, 1);
    return IG_OK;
}

int ig_update(ig_t h, const double *x, const double *Ax) {
    if (!h) return set_err(IG_E_ARG, "NULL handle");
    if (!x) return set_err(IG_E_ARG, "x is NULL");
    DevGuard g(h->dev);
    if (is_proj(h->method)) {
        if (!Ax) return set_err(IG_E_ARG, "Ax is NULL (projection needs A x, PAPER.md:237)");
        ProjArgs a = proj_args(h);
        a.x = x;
        a.Ax = Ax;
        h->known_d = -1;  // d is decided on the device
        const int vec = (al16(x) && al16(Ax)) ? 2 : 1;
        if (use_fused(h)) {
            int rc = persistent_launch(h, [&]() -> int {
                Prof p(h, IG_K_UPDATE_FUSED);
                CUDA_OK(launch_update_fused(a, vec, h->nsm, h->stream));
                return IG_OK;
            });
            if (rc) return rc;
            count(h, 1);
            return IG_OK;
        }
        {
            Prof p(h, IG_K_U1);
            CUDA_OK(launch_u1(a, vec, h->nsm, h->stream));
        }
        int rc = exchange(h, ST_U1);
        if (rc) return rc;
        {
            Prof p(h, IG_K_U2);
            CUDA_OK(launch_u2(a, vec, h->nsm, h->stream));
        }
        rc = exchange(h, ST_U2);
        if (rc) return rc;
        {
            Prof p(h, IG_K_U3);
            CUDA_OK(launch_u3(a, vec, h->nsm, h->stream));
        }
        count(h, 3);
        return IG_OK;
    }
    if (h->dring) {  // device window: the push kernel picks the slot and advances the counter
        RingBatch rb;
        memset(&rb, 0, sizeof rb);
        rb.f[0] = ring_args(h);
        rb.f[0].x = x;
        rb.nf = 1;
        h->last_copy = !in_slab(h, x);
        Prof p(h, IG_K_COPY);
        CUDA_OK(launch_push_ring(rb, al16(x) ? 2 : 1, h->nsm, h->stream));
        count(h, 1);
        return IG_OK;
    }
    if (capturing(h->stream))
        return set_err(IG_E_STATE, "extrapolation window is host-side: ig_set_device_ring(h, 1) before capturing");
    double *slot = next_slot_ptr(h);
    h->last_copy = (x != slot);
    if (h->last_copy) {
        Prof p(h, IG_K_COPY);
        CUDA_OK(launch_copy(slot, x, h->N, (al16(x) && al16(slot)) ? 2 : 1, h->nsm, h->stream));
        count(h, 1);
    }
    if (h->fill < h->M) ++h->fill;
    else h->head = (h->head + 1) % h->M;
    return IG_OK;
}

int ig_form_guess_batch(int n, ig_t *hs, const double *const *bs, double *const *x0s) {
    if (n < 0 || (n > 0 && (!hs || !x0s))) return set_err(IG_E_ARG, "bad batch arguments");
    int i = 0;
    while (i < n) {
        ig_t h = hs[i];
        if (!h) return set_err(IG_E_ARG, "NULL handle in batch");
        if (!is_extrap(h->method)) {  // projection: its own persistent kernel
            int rc = ig_form_guess(h, bs ? bs[i] : nullptr, x0s[i]);
            if (rc) return rc;
            ++i;
            continue;
        }
        if (h->dring) {  // consecutive device-window handles on the same device and stream: one launch
            RingBatch rb;
            memset(&rb, 0, sizeof rb);
            int fc = 0;
            bool aligned = true;
            int j = i;
            for (; j < n && rb.nf < MAXF; ++j) {
                ig_t q = hs[j];
                if (!q || !is_extrap(q->method) || !q->dring || q->dev != h->dev || q->stream != h->stream) break;
                if (!x0s[j]) return set_err(IG_E_ARG, "x0 is NULL");
                rb.f[rb.nf] = ring_args(q);
                rb.f[rb.nf].x0 = x0s[j];
                aligned = aligned && al16(x0s[j]);
                fc = q->ring_fc > fc ? q->ring_fc : fc;
                ++rb.nf;
            }
            DevGuard g(h->dev);
            Prof p(h, IG_K_EXTRAP);
            CUDA_OK(launch_extrap_ring(rb, fc, aligned ? 2 : 1, h->nsm, h->stream));
            count(h, 1);
            i = j;
            continue;
        }
        if (capturing(h->stream))
            return set_err(IG_E_STATE, "extrapolation window is host-side: ig_set_device_ring(h, 1) before capturing");
        // group consecutive extrapolation handles on the same device and stream
        ExtrapBatch b;
        memset(&b, 0, sizeof b);
        bool aligned = true;
        int j = i;
        for (; j < n && b.nf < MAXF; ++j) {
            ig_t q = hs[j];
            if (!q || !is_extrap(q->method) || q->dring || q->dev != h->dev || q->stream != h->stream) break;
            if (!x0s[j]) return set_err(IG_E_ARG, "x0 is NULL");
            bool al = true;
            if (extrap_args(q, x0s[j], b.f[b.nf], al)) {
                aligned = aligned && al;
                ++b.nf;
            }
        }
        if (b.nf > 0) {
            DevGuard g(h->dev);
            Prof p(h, IG_K_EXTRAP);
            CUDA_OK(launch_extrap_batch(b, aligned ? 2 : 1, h->nsm, h->stream));
            count(h, 1);
        }
        i = j;
    }
    return IG_OK;
}

int ig_update_batch(int n, ig_t *hs, const double *const *xs, const double *const *Axs) {
    if (n < 0 || (n > 0 && (!hs || !xs))) return set_err(IG_E_ARG, "bad batch arguments");
    int i = 0;
    while (i < n) {
        ig_t h = hs[i];
        if (!h) return set_err(IG_E_ARG, "NULL handle in batch");
        if (!is_extrap(h->method) || !h->dring) {
            int rc = ig_update(h, xs[i], Axs ? Axs[i] : nullptr);
            if (rc) return rc;
            ++i;
            continue;
        }
        // consecutive device-window extrapolation handles (same device and stream): one push launch
        RingBatch rb;
        memset(&rb, 0, sizeof rb);
        bool aligned = true;
        int j = i;
        for (; j < n && rb.nf < MAXF; ++j) {
            ig_t q = hs[j];
            if (!q || !is_extrap(q->method) || !q->dring || q->dev != h->dev || q->stream != h->stream) break;
            if (!xs[j]) return set_err(IG_E_ARG, "x is NULL");
            rb.f[rb.nf] = ring_args(q);
            rb.f[rb.nf].x = xs[j];
            q->last_copy = !in_slab(q, xs[j]);
            aligned = aligned && al16(xs[j]);
            ++rb.nf;
        }
        DevGuard g(h->dev);
        Prof p(h, IG_K_COPY);
        CUDA_OK(launch_push_ring(rb, aligned ? 2 : 1, h->nsm, h->stream));
        count(h, 1);
        i = j;
    }
    return IG_OK;
}

static int watchdog_error(int err);

static int ensure_stage(ig_t h) {
    for (auto &s : h->stage)
        if (!s && cudaMalloc(&s, sizeof(double) * (size_t)h->ld) != cudaSuccess) {
            cudaGetLastError();
            return set_err(IG_E_OOM, "staging buffer allocation failed");
        }
    if (is_proj(h->method) && !h->pin_ctrl && cudaMallocHost(&h->pin_ctrl, offsetof(Ctrl, ticket)) != cudaSuccess) {
        cudaGetLastError();
        return set_err(IG_E_OOM, "pinned control readback allocation failed");
    }
    return IG_OK;
}

// Second stream + events for the batch host calls (copies overlapping the handle's stream).
static int ensure_cstream(ig_t h) {
    if (h->cstream) return IG_OK;
    CUDA_OK(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
    for (auto &e : h->cev) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return IG_OK;
}

// Projection: the update's d / watchdog flag travel back with the call's own synchronisation
// (4 x int32 D2H enqueued after the kernel), so the next ig_form_guess_host knows whether the
// fallback x0 is needed (d == 0) without another stream round trip.
static int ctrl_readback(ig_t h) { CUDA_OK(cudaMemcpyAsync(h->pin_ctrl, h->ctrl, offsetof(Ctrl, ticket), cudaMemcpyDeviceToHost, h->stream)); return IG_OK; }
static int ctrl_consume(ig_t h) {
    Ctrl c;
    memcpy(&c, h->pin_ctrl, offsetof(Ctrl, ticket));
    h->known_d = c.d;
    return watchdog_error(c.err);
}
static int known_dim(ig_t h) {
    if (h->known_d >= 0) return IG_OK;
    int d = 0;
    int rc = ig_history_dim(h, &d);
    if (rc) return rc;
    h->known_d = d;
    return IG_OK;
}

int ig_form_guess_host(ig_t h, const double *b, double *x0) {
    if (!h || !x0) return set_err(IG_E_ARG, "NULL handle or x0");
    DevGuard g(h->dev);
    int rc = ensure_stage(h);
    if (rc) return rc;
    const size_t nb = sizeof(double) * (size_t)h->N;
    if (is_proj(h->method)) {
        if (!b) return set_err(IG_E_ARG, "b is NULL");
        rc = known_dim(h);
        if (rc) return rc;
        CUDA_OK(cudaMemcpyAsync(h->stage[0], b, nb, cudaMemcpyHostToDevice, h->stream));
        // the fallback x0 is only read when d == 0: skip its upload otherwise
        if (h->known_d == 0) CUDA_OK(cudaMemcpyAsync(h->stage[1], x0, nb, cudaMemcpyHostToDevice, h->stream));
        rc = ig_form_guess(h, h->stage[0], h->stage[1]);
        if (rc) return rc;
    } else {
        rc = ring_pull(h);
        if (rc) return rc;
        if (h->fill == 0) return IG_OK;  // x0 untouched, nothing to move
        rc = ig_form_guess(h, nullptr, h->stage[1]);
        if (rc) return rc;
    }
    CUDA_OK(cudaMemcpyAsync(x0, h->stage[1], nb, cudaMemcpyDeviceToHost, h->stream));
    CUDA_OK(cudaStreamSynchronize(h->stream));
    return IG_OK;
}

int ig_update_host(ig_t h, const double *x, const double *Ax) {
    if (!h || !x) return set_err(IG_E_ARG, "NULL handle or x");
    DevGuard g(h->dev);
    const size_t nb = sizeof(double) * (size_t)h->N;
    if (is_proj(h->method)) {
        if (!Ax) return set_err(IG_E_ARG, "Ax is NULL");
        int rc = ensure_stage(h);
        if (rc) return rc;
        CUDA_OK(cudaMemcpyAsync(h->stage[2], x, nb, cudaMemcpyHostToDevice, h->stream));
        CUDA_OK(cudaMemcpyAsync(h->stage[3], Ax, nb, cudaMemcpyHostToDevice, h->stream));
        rc = ig_update(h, h->stage[2], h->stage[3]);
        if (rc) return rc;
        rc = ctrl_readback(h);
        if (rc) return rc;
        CUDA_OK(cudaStreamSynchronize(h->stream));
        return ctrl_consume(h);
    }
    int rc0 = ring_pull(h);
    if (rc0) return rc0;
    double *slot = next_slot_ptr(h);  // copy straight into the ring slot: zero-copy push
    CUDA_OK(cudaMemcpyAsync(slot, x, nb, cudaMemcpyHostToDevice, h->stream));
    int rc = ig_update(h, slot, nullptr);
    if (rc) return rc;
    CUDA_OK(cudaStreamSynchronize(h->stream));
    return IG_OK;
}

// Batch host calls (several fields, one synchronisation): the PCIe transfers of different fields
// overlap each other and the kernels (pinned host memory; H2D and D2H run on separate engines).
int ig_form_guess_batch_host(int n, ig_t *hs, const double *const *bs, double *const *x0s) {
    if (n < 0 || (n > 0 && (!hs || !x0s))) return set_err(IG_E_ARG, "bad batch arguments");
    for (int i = 0; i < n; ++i) {
        if (!hs[i] || !x0s[i]) return set_err(IG_E_ARG, "NULL handle or x0 in batch");
        if (is_proj(hs[i]->method) && (!bs || !bs[i])) return set_err(IG_E_ARG, "b is NULL");
        DevGuard g(hs[i]->dev);
        int rc = ensure_stage(hs[i]);
        if (!rc) rc = ensure_cstream(hs[i]);
        if (!rc && is_proj(hs[i]->method)) rc = known_dim(hs[i]);
        if (!rc) rc = ring_pull(hs[i]);
        if (rc) return rc;
    }
    // 1) extrapolation fields first (no inputs): kernel on the handle's stream, D2H of the guess on
    //    the handle's copy stream, so it overlaps the projection fields' H2D of b
    for (int i = 0; i < n; ++i) {
        ig_t q = hs[i];
        if (!is_extrap(q->method) || q->fill == 0) continue;  // fill == 0: x0 untouched
        DevGuard g(q->dev);
        int rc = ig_form_guess(q, nullptr, q->stage[1]);
        if (rc) return rc;
        CUDA_OK(cudaEventRecord(q->cev[0], q->stream));
        CUDA_OK(cudaStreamWaitEvent(q->cstream, q->cev[0], 0));
        CUDA_OK(cudaMemcpyAsync(x0s[i], q->stage[1], sizeof(double) * (size_t)q->N, cudaMemcpyDeviceToHost,
                                q->cstream));
    }
    // 2) projection fields: H2D b (and the fallback x0 iff d == 0), kernel, D2H of the guess
    for (int i = 0; i < n; ++i) {
        ig_t h = hs[i];
        if (!is_proj(h->method)) continue;
        DevGuard g(h->dev);
        const size_t nb = sizeof(double) * (size_t)h->N;
        CUDA_OK(cudaMemcpyAsync(h->stage[0], bs[i], nb, cudaMemcpyHostToDevice, h->stream));
        if (h->known_d == 0) CUDA_OK(cudaMemcpyAsync(h->stage[1], x0s[i], nb, cudaMemcpyHostToDevice, h->stream));
        int rc = ig_form_guess(h, h->stage[0], h->stage[1]);
        if (rc) return rc;
        CUDA_OK(cudaMemcpyAsync(x0s[i], h->stage[1], nb, cudaMemcpyDeviceToHost, h->stream));
    }
    for (int i = 0; i < n; ++i) {
        DevGuard g(hs[i]->dev);
        CUDA_OK(cudaStreamSynchronize(hs[i]->stream));
        CUDA_OK(cudaStreamSynchronize(hs[i]->cstream));
    }
    return IG_OK;
}

int ig_update_batch_host(int n, ig_t *hs, const double *const *xs, const double *const *Axs) {
    if (n < 0 || (n > 0 && (!hs || !xs))) return set_err(IG_E_ARG, "bad batch arguments");
    for (int i = 0; i < n; ++i) {
        if (!hs[i] || !xs[i]) return set_err(IG_E_ARG, "NULL handle or x in batch");
        if (is_proj(hs[i]->method) && (!Axs || !Axs[i])) return set_err(IG_E_ARG, "Ax is NULL");
        DevGuard g(hs[i]->dev);
        int rc = ensure_stage(hs[i]);
        if (!rc) rc = ensure_cstream(hs[i]);
        if (!rc) rc = ring_pull(hs[i]);
        if (rc) return rc;
    }
    // 1) projection fields: H2D x, Ax, then the update kernel
    ig_t last_proj = nullptr;
    for (int i = 0; i < n; ++i) {
        ig_t h = hs[i];
        if (!is_proj(h->method)) continue;
        DevGuard g(h->dev);
        const size_t nb = sizeof(double) * (size_t)h->N;
        CUDA_OK(cudaMemcpyAsync(h->stage[2], xs[i], nb, cudaMemcpyHostToDevice, h->stream));
        CUDA_OK(cudaMemcpyAsync(h->stage[3], Axs[i], nb, cudaMemcpyHostToDevice, h->stream));
        CUDA_OK(cudaEventRecord(h->cev[1], h->stream));  // uploads done (the kernel follows)
        int rc = ig_update(h, h->stage[2], h->stage[3]);
        if (!rc) rc = ctrl_readback(h);
        if (rc) return rc;
        last_proj = h;
    }
    // 2) extrapolation fields: H2D of x straight into the ring slot on the copy stream, after the
    //    projection uploads (PCIe is shared) so it overlaps the projection update kernels; the
    //    handle's stream then waits for it (later kernels read the slot)
    for (int i = 0; i < n; ++i) {
        ig_t q = hs[i];
        if (!is_extrap(q->method)) continue;
        DevGuard g(q->dev);
        double *slot = next_slot_ptr(q);
        CUDA_OK(cudaEventRecord(q->cev[0], q->stream));  // readers of the slot's old solution
        CUDA_OK(cudaStreamWaitEvent(q->cstream, q->cev[0], 0));
        if (last_proj && last_proj->dev == q->dev) CUDA_OK(cudaStreamWaitEvent(q->cstream, last_proj->cev[1], 0));
        CUDA_OK(cudaMemcpyAsync(slot, xs[i], sizeof(double) * (size_t)q->N, cudaMemcpyHostToDevice, q->cstream));
        CUDA_OK(cudaEventRecord(q->cev[1], q->cstream));
        CUDA_OK(cudaStreamWaitEvent(q->stream, q->cev[1], 0));
        int rc = ig_update(q, slot, nullptr);  // zero-copy push
        if (rc) return rc;
    }
    int first_err = IG_OK;
    for (int i = 0; i < n; ++i) {
        DevGuard g(hs[i]->dev);
        CUDA_OK(cudaStreamSynchronize(hs[i]->stream));
        CUDA_OK(cudaStreamSynchronize(hs[i]->cstream));
        if (is_proj(hs[i]->method)) {
            int rc = ctrl_consume(hs[i]);
            if (rc && !first_err) first_err = rc;
        }
    }
    return first_err;
}

double *ig_next_slot(ig_t h) {
    if (!h || !is_extrap(h->method)) return nullptr;
    if (h->dring) {
        DevGuard g(h->dev);
        if (ring_pull(h)) return nullptr;
    }
    return next_slot_ptr(h);
}

int ig_comm_unique_id(void *out128) {
    if (!out128) return set_err(IG_E_ARG, "NULL out");
    NcclApi &api = nccl();
    if (!api.ok) return set_err(IG_E_NCCL, "%s", api.why.c_str());
    ncclUniqueId id;
    ncclResult_t r = api.getUniqueId(&id);
    if (r) return set_err(IG_E_NCCL, "ncclGetUniqueId: %s", api.errStr(r));
    memcpy(out128, id.internal, 128);
    return IG_OK;
}

int ig_comm_create(int nranks, int rank, const void *id128, ig_comm_t *out) {
    if (!out || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return set_err(IG_E_ARG, "bad comm arguments");
    NcclApi &api = nccl();
    if (!api.ok) return set_err(IG_E_NCCL, "%s", api.why.c_str());
    ncclUniqueId id;
    memcpy(id.internal, id128, 128);
    auto *c = new ig_comm_ctx;
    c->nranks = nranks;
    c->rank = rank;
    ncclResult_t r = api.commInitRank(&c->comm, nranks, id, rank);
    if (r) {
        delete c;
        return set_err(IG_E_NCCL, "ncclCommInitRank: %s", api.errStr(r));
    }
    *out = c;
    return IG_OK;
}

void ig_comm_destroy(ig_comm_t c) {
    if (!c) return;
    if (c->comm && nccl().ok) nccl().commDestroy(c->comm);
    delete c;
}

void *ig_local_group_create(int nranks) {
    if (nranks < 1) return set_err(IG_E_ARG, "nranks must be >= 1"), nullptr;
    return new LocalGroup(nranks);
}

void ig_local_group_destroy(void *group) { delete static_cast<LocalGroup *>(group); }

int ig_comm_create_local(void *group, int rank, ig_comm_t *out) {
    LocalGroup *g = static_cast<LocalGroup *>(group);
    if (!g || !out || rank < 0 || rank >= g->n) return set_err(IG_E_ARG, "bad local comm arguments");
    auto *c = new ig_comm_ctx;
    c->nranks = g->n;
    c->rank = rank;
    c->local = g;
    *out = c;
    return IG_OK;
}

int ig_attach_comm(ig_t h, ig_comm_t c) {
    if (!h || !c) return set_err(IG_E_ARG, "NULL handle or comm");
    DevGuard g(h->dev);
    h->comm = c;
    if (!is_proj(h->method) || c->nranks == 1) return IG_OK;  // extrapolation never communicates
    if (h->gath != h->part) cudaFree(h->gath);
    double *gb = nullptr;
    if (cudaMalloc(&gb, sizeof(double) * PS * NSTAGE * c->nranks) != cudaSuccess) {
        cudaGetLastError();
        return set_err(IG_E_OOM, "gather buffer allocation failed");
    }
    CUDA_OK(cudaMemset(gb, 0, sizeof(double) * PS * NSTAGE * c->nranks));
    h->gath = gb;
    h->G = c->nranks;
    return IG_OK;
}

int ig_set_launch(ig_t h, int cooperative) {
    if (!h || cooperative < -1 || cooperative > 1) return set_err(IG_E_ARG, "bad handle or launch mode");
    h->coop = cooperative;
    return IG_OK;
}

int ig_set_watchdog(ig_t h, double seconds) {
    if (!h || !(seconds > 0.0)) return set_err(IG_E_ARG, "bad handle or watchdog time");
    h->watchdog_ns = (unsigned long long)(seconds * 1e9);
    return IG_OK;
}

int ig_set_grid_limit(ig_t h, int max_blocks) {
    if (!h || max_blocks < 0) return set_err(IG_E_ARG, "bad handle or grid limit");
    h->max_grid = max_blocks;
    return IG_OK;
}

static int ensure_xwin(ig_t h) {
    if (!is_proj(h->method)) return set_err(IG_E_ARG, "peer exchange is for projection handles");
    if (h->xwin) return IG_OK;
    if (cudaMalloc(&h->xwin, sizeof(XWin)) != cudaSuccess) {
        cudaGetLastError();
        h->xwin = nullptr;
        return set_err(IG_E_OOM, "exchange window allocation failed");
    }
    CUDA_OK(cudaMemset(h->xwin, 0, sizeof(XWin)));
    return IG_OK;
}

size_t ig_xwin_bytes(void) { return sizeof(XWin); }

int ig_xwin_export(ig_t h, void *ipc_handle_out) {
    if (!h || !ipc_handle_out) return set_err(IG_E_ARG, "NULL argument");
    DevGuard g(h->dev);
    int rc = ensure_xwin(h);
    if (rc) return rc;
    cudaIpcMemHandle_t mh;
    CUDA_OK(cudaIpcGetMemHandle(&mh, h->xwin));
    static_assert(sizeof(mh) == 64, "CUDA IPC handle is 64 bytes");
    memcpy(ipc_handle_out, &mh, 64);
    return IG_OK;
}

void *ig_xwin_ptr(ig_t h) {
    if (!h) return nullptr;
    DevGuard g(h->dev);
    if (ensure_xwin(h)) return nullptr;
    return h->xwin;
}

int ig_attach_peers(ig_t h, int nranks, int rank, const void *ipc_handles, void *const *peer_ptrs) {
    if (!h || nranks < 1 || nranks > MAXG || rank < 0 || rank >= nranks)
        return set_err(IG_E_ARG, "bad peer arguments (1 <= nranks <= %d)", MAXG);
    DevGuard g(h->dev);
    int rc = ensure_xwin(h);
    if (rc) return rc;
    Exchange xc = {};
    xc.G = nranks;
    xc.rank = rank;
    for (int r = 0; r < nranks; ++r) {
        if (r == rank) {
            xc.peer[r] = h->xwin;
        } else if (peer_ptrs && peer_ptrs[r]) {
            xc.peer[r] = static_cast<XWin *>(peer_ptrs[r]);  // same process (virtual ranks)
        } else {
            if (!ipc_handles) return set_err(IG_E_ARG, "rank %d: neither a pointer nor an IPC handle", r);
            cudaIpcMemHandle_t mh;
            memcpy(&mh, static_cast<const char *>(ipc_handles) + 64 * r, 64);
            void *p = nullptr;
            CUDA_OK(cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess));
            h->ipc_opened.push_back(p);
            xc.peer[r] = static_cast<XWin *>(p);
        }
    }
    h->xc = nranks > 1 ? xc : Exchange{};
    return IG_OK;
}

static int watchdog_error(int err) {
    if (err == 1)
        return set_err(IG_E_STATE, "device watchdog: a grid barrier timed out (persistent grid not co-resident?); "
                                   "the history is invalid, ig_reset the handle");
    if (err == 2)
        return set_err(IG_E_STATE, "device watchdog: the peer exchange timed out (a rank stopped calling?); "
                                   "the history is invalid, ig_reset every rank");
    if (err == 3)
        return set_err(IG_E_STATE, "non-finite projection sums (NaN/Inf in b, x or A x?); the pair was not "
                                   "admitted -- check the inputs");
    return IG_OK;
}

int ig_set_device_ring(ig_t h, int on) {
    if (!h || !is_extrap(h->method)) return set_err(IG_E_ARG, "extrapolation handle required");
    DevGuard g(h->dev);
    if (on && !h->dring) {
        if (!h->ring) {
            RingTab &t = h->rtab_host;
            memset(&t, 0, sizeof t);
            int fc = 0;
            for (int f = 1; f <= h->M; ++f) {
                int nz = 0;
                for (int j = 0; j < f; ++j) {
                    const double bj = h->table[f - 1][j];
                    if (bj == 0.0) continue;  // zero weights are not streamed (as extrap_args)
                    t.jidx[f - 1][nz] = j;
                    t.beta[f - 1][nz] = bj;
                    ++nz;
                }
                t.nnz[f - 1] = nz;
                fc = nz > fc ? nz : fc;
            }
            h->ring_fc = fc;
            if (cudaMalloc(&h->ring, sizeof(DevRing)) != cudaSuccess || cudaMalloc(&h->rtab, sizeof(RingTab)) != cudaSuccess) {
                cudaGetLastError();
                cudaFree(h->ring);
                h->ring = nullptr;
                return set_err(IG_E_OOM, "device window allocation failed");
            }
            CUDA_OK(cudaMemcpyAsync(h->rtab, &t, sizeof t, cudaMemcpyHostToDevice, h->stream));
        }
        h->dring = true;
        return ring_push_host(h);  // the device counter continues the host window
    }
    if (!on && h->dring) {
        int rc = ring_pull(h);
        if (rc) return rc;
        h->dring = false;
    }
    return IG_OK;
}

struct ig_graph_ctx {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;  // libig kernels per replay
};
static thread_local int64_t g_capture_launches0 = 0;

int ig_capture_begin(void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!s) return set_err(IG_E_ARG, "capture needs a non-default stream");
    CUDA_OK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    g_capture_launches0 = g_launches.load();
    return IG_OK;
}

int ig_capture_end(void *stream, ig_graph_t *out) {
    if (!out) return set_err(IG_E_ARG, "NULL out");
    *out = nullptr;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaGraph_t graph = nullptr;
    CUDA_OK(cudaStreamEndCapture(s, &graph));
    ig_graph_ctx *g = new ig_graph_ctx;
    g->graph = graph;
    // the captured calls counted their launches; they run at every replay instead
    g->launches = g_launches.load() - g_capture_launches0;
    g_launches -= g->launches;
    if (cudaGraphInstantiateWithFlags(&g->exec, graph, 0) != cudaSuccess) {
        cudaError_t e = cudaGetLastError();
        cudaGraphDestroy(graph);
        delete g;
        return set_err(IG_E_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e));
    }
    *out = g;
    return IG_OK;
}

int ig_graph_launch(ig_graph_t g, void *stream) {
    if (!g) return set_err(IG_E_ARG, "NULL graph");
    CUDA_OK(cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream)));
    g_launches += g->launches;
    return IG_OK;
}

void ig_graph_destroy(ig_graph_t g) {
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
}

int ig_history_dim(ig_t h, int *d) {
    if (!h || !d) return set_err(IG_E_ARG, "NULL argument");
    DevGuard g(h->dev);
    if (is_proj(h->method)) {
        Ctrl c;  // the leading ints (d ... err)
        CUDA_OK(cudaMemcpyAsync(&c, h->ctrl, offsetof(Ctrl, ticket), cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        *d = c.d;
        return watchdog_error(c.err);
    } else {
        int rc = ring_pull(h);
        if (rc) return rc;
        *d = h->fill;
    }
    return IG_OK;
}

int ig_weights(ig_t h, int f, double *beta, int *len) {
    if (!h || !beta || !len || !is_extrap(h->method)) return set_err(IG_E_ARG, "bad arguments");
    if (f == 0) f = h->M;
    if (f < 1 || f > h->M) return set_err(IG_E_ARG, "f must be in [0, M]");
    for (int j = 0; j < f; ++j) beta[j] = h->table[f - 1][j];
    *len = f;
    return IG_OK;
}

int ig_get_stats(ig_t h, ig_stats_t *out) {
    if (!h || !out) return set_err(IG_E_ARG, "NULL argument");
    DevGuard g(h->dev);
    memset(out, 0, sizeof *out);
    out->launches = h->launches;
    if (is_proj(h->method)) {
        Ctrl c;
        CUDA_OK(cudaMemcpyAsync(&c, h->ctrl, offsetof(Ctrl, gc), cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        out->d = c.d;
        out->admitted = c.admitted;
        out->rho = c.rho;
        out->norm_Ax = c.nAx;
        out->norm_bt = c.nb;
        if (c.err) return watchdog_error(c.err);
    } else {
        int rc = ring_pull(h);
        if (rc) return rc;
        out->d = h->fill;
        out->admitted = 1;
    }
    return IG_OK;
}

int ig_bytes(ig_t h, int64_t *form_bytes, int64_t *update_bytes) {
    if (!h || !form_bytes || !update_bytes) return set_err(IG_E_ARG, "NULL argument");
    DevGuard g(h->dev);
    const int64_t vb = 8 * h->N;
    if (is_extrap(h->method)) {
        if (h->dring) {  // device window: the form at the current window (the host never saw f)
            int rc = ring_pull(h);
            if (rc) return rc;
            h->last_form_f = h->fill > 0 ? h->rtab_host.nnz[h->fill - 1] : 0;
        }
        *form_bytes = h->last_form_f ? (h->last_form_f + 1) * vb : 0;
        *update_bytes = h->last_copy ? 2 * vb : 0;
        return IG_OK;
    }
    Ctrl c;
    CUDA_OK(cudaMemcpyAsync(&c, h->ctrl, offsetof(Ctrl, gc), cudaMemcpyDeviceToHost, h->stream));
    CUDA_OK(cudaStreamSynchronize(h->stream));
    const int M = h->M, de = c.deff, rot = c.last_rot, adm = c.admitted;
    // form at the current d: (d+1) reads for the dots, d reads + 1 write for the combine
    *form_bytes = c.d > 0 ? 2 * (int64_t)(c.d + 1) * vb : 0;
    int64_t v = rot ? (M + 1 + (M - 1)) : (de + 1);  // U1: [B~ rotation] + dots against Ax
    v += de > 0 ? de + 1 : 0;                          // U2
    if (adm) v += 1 + de + 1 + 2;                      // U3: Ax, B~, x, two new columns
    if (rot) v += M + (M - 1);                         // U3: X~ rotation
    else if (adm) v += de;                             // U3: X~ reads
    *update_bytes = v * vb;
    return IG_OK;
}

int ig_copy_history(ig_t h, double *Bt_dst, double *Xt_dst, int64_t ld_dst, double *R_host) {
    if (!h || !is_proj(h->method)) return set_err(IG_E_ARG, "projection handle required");
    DevGuard g(h->dev);
    const size_t w = sizeof(double) * (size_t)h->N;
    if (Bt_dst)
        CUDA_OK(cudaMemcpy2DAsync(Bt_dst, sizeof(double) * ld_dst, h->Bt, sizeof(double) * h->ld, w, h->M,
                                  cudaMemcpyDeviceToDevice, h->stream));
    if (Xt_dst)
        CUDA_OK(cudaMemcpy2DAsync(Xt_dst, sizeof(double) * ld_dst, h->Xt, sizeof(double) * h->ld, w, h->M,
                                  cudaMemcpyDeviceToDevice, h->stream));
    if (R_host) {
        std::vector<double> R(MAXM * MAXM);
        CUDA_OK(cudaMemcpyAsync(R.data(), h->ctrl->R, sizeof(double) * MAXM * MAXM, cudaMemcpyDeviceToHost,
                                h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        for (int j = 0; j < h->M; ++j)
            for (int i = 0; i < h->M; ++i) R_host[i + j * h->M] = R[i + j * MAXM];
    }
    CUDA_OK(cudaStreamSynchronize(h->stream));
    return IG_OK;
}

int64_t ig_total_launches(void) { return g_launches.load(); }

int ig_profile(ig_t h, int enable) {
    if (!h) return set_err(IG_E_ARG, "NULL handle");
    DevGuard g(h->dev);
    prof_drain(h);
    for (int k = 0; k < IG_NKERNELS; ++k) {
        h->prof_ms[k] = 0.0;
        h->prof_n[k] = 0;
    }
    h->profiling = enable != 0;
    return IG_OK;
}

int ig_profile_read(ig_t h, int kernel, double *total_ms, int64_t *launches) {
    if (!h || !total_ms || !launches || kernel < 0 || kernel >= IG_NKERNELS) return set_err(IG_E_ARG, "bad arguments");
    DevGuard g(h->dev);
    prof_drain(h);
    *total_ms = h->prof_ms[kernel];
    *launches = h->prof_n[kernel];
    return IG_OK;
}

}  // extern "C"
