// kern_fused.cu -- persistent projection kernels (one launch per call) for a single GPU and for
// the in-kernel peer exchange; launched as ordinary PDL-chained kernels by default (IG_LAUNCH).
//
// One launch per library call instead of one per pass: the passes of Alg. 2
// are separated by software grid barriers, and after each reduction EVERY CTA sums the block
// partials in the same fixed order (bitwise-identical coefficients in all CTAs, no serial
// last-block finish, no fp64 atomics).  This removes the per-kernel ramp-up/drain and launch
// gaps that dominate at the C2 size (2M DOFs, ~25-70 us per pass).
//
//   k_form_fused   : [alpha = B~^T b] --barrier--> [x0 = X~ alpha]
//   k_update_fused : [B~ downdate + c1, ||Ax||^2] --barrier--> [c2, ||b1||^2] --barrier-->
//                    [X~ downdate + x~, b~, admission, new columns]
//                    --> CTA 0 writes the control block (no exit barrier); the planner CTA
//                    (the last one, QR) computes R and the next downdate's Givens plan
//                    alongside (its prefix during passes 1-2, its suffix after barrier 2)
// Every kernel is instantiated per history bucket MC (mcb(): 1, 2, 4, 5, 6, 8, 10, ..., 32); the
// large buckets use the rolling prefetch (u1_roll / u2_roll / u3_roll, RF form) and, below 2^24
// DOFs, the one-copy pass-3 loop (OC) -- separate instantiations chosen by the launchers.
// Barrier and claim counters are double-buffered by a launch epoch in the control block.  The
// element arithmetic is the same device code as the one-kernel-per-pass path (proj_common.cuh),
// which stays in use when partial sums cross ranks through an all-gather (ig_attach_comm); with
// the in-kernel peer exchange (ig_attach_peers) these kernels are used for G > 1 as well.
#include <cstdlib>
#include <type_traits>

#include "proj_common.cuh"

// Phase timestamps per CTA (debug builds with -DIG_TRACE=1; IG_TRACE_PTR = device buffer address
// passed through the environment at launch): [cta][slot] = %globaltimer.
#ifdef IG_TRACE
__device__ unsigned long long g_trace[1024 * 16];
__device__ unsigned long long g_trace_form[1024 * 16];
#define TRACE(slot) do { if (threadIdx.x == 0) g_trace[blockIdx.x * 16 + (slot)] = globaltimer_ns(); } while (0)
#define TRACE_F(slot) do { if (threadIdx.x == 0) g_trace_form[blockIdx.x * 16 + (slot)] = globaltimer_ns(); } while (0)
extern "C" int ig_debug_trace_read(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * n);
}
extern "C" int ig_debug_trace_read_form(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_trace_form, sizeof(unsigned long long) * n);
}
#else
#define TRACE(slot) do { } while (0)
#define TRACE_F(slot) do { } while (0)
#endif

namespace ig {

// Second block-partial buffer so that a fast CTA's pass-2 partials never overwrite pass-1
// partials a slow CTA is still reading.
constexpr int BLK2 = PS * MAXB;

// Smallest bucket whose one-copy (OC) update kernel uses the rolling prefetch in passes 1 and 2
// (u1_roll / u2_roll; bitwise-identical results; A/B on one box, profiles/r3_roll_ab.md: N = 3e5
// QR(16) 49.5 -> 48.0, 1e6 QR(12) 137.0 -> 134.0, QR(24) 281.2 -> 275.3, QR(30) 339 -> 336,
// 3e6 QR(16) 510 -> 505, 1e7 QR(16) 1615 -> 1601 us/step).  -DIG_ROLL_MIN=64 turns it off.
#ifndef IG_ROLL_MIN
#define IG_ROLL_MIN 9
#endif
// The same for the large-vector (two-copy) kernels: the M = 17..32 bucket only (the M = 16
// kernel's register allocation is fragile); profiles/r3_roll_ab.md, with the rolling
// form kernel: N = 2e7 QR(17) 3956 -> 3710, QR(30) 5988 -> 5896; 2^27 QR(24) 33564 -> 32948,
// QR(30) 40394 -> 39937 us/step.
#ifndef IG_ROLL_BIG_MIN
#define IG_ROLL_BIG_MIN 17
#endif
// Buckets [IG_ROLL3_MIN, IG_ROLL3_MAX] of the one-copy update kernel run pass 3 with rolling
// register sets (u3_roll; the buckets whose B~ and X~ columns fit in registers together;
// bitwise-identical; profiles/r3_roll_ab.md: N = 1e6 QR(16) 171.9 -> 169.5, QR(12) 133.2 ->
// 131.8, QR(9) 109.3 -> 108.3 us/step; 1e7 QR(16) 1602 -> 1609; MC = 20 spills and was slower
// at 3e6-1e7).  -DIG_ROLL3_MIN=64 turns it off.
#ifndef IG_ROLL3_MIN
#define IG_ROLL3_MIN 9
#endif
#ifndef IG_ROLL3_MAX
#define IG_ROLL3_MAX 16
#endif

// RF: rolling prefetch in both passes (one element per trip, u1_roll-style: the next element's
// load of a column is issued as soon as this element has consumed it); a separate instantiation
// chosen by the launcher for the M = 17..32 bucket (bitwise-identical results).
template <int MC, int VEC, bool RF = false>
__global__ void __launch_bounds__(THREADS, 1) k_form_fused(const __grid_constant__ ProjArgs a) {
    typedef typename VT<VEC>::T V;
    constexpr int U = FusedUnroll<MC>::U;
    __shared__ double sh[(THREADS / 32) * (MC + 1)];
    __shared__ double s_red[PS];
    TRACE_F(8);
    pdl_wait();  // stream predecessor complete and visible (programmatic dependent launch)
    TRACE_F(0);
#ifdef IG_TRACE
    if (threadIdx.x == 0) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_trace_form[blockIdx.x * 16 + 12] = sm;
    }
#endif
    Ctrl *c = a.ctrl;
    const int d = c->d;
    if (d == 0) return;  // uniform: x0 stays the caller's fallback
    const unsigned e = launch_epoch(c);
    const unsigned long long ep = c->xepoch[ST_FORM] + 1;
    // All form traffic is single-use within the call (the caller's solve runs next): evict_first,
    // so the guess does not push the solver's working set out of L2.
    const unsigned long long ps = make_l2pol().stream;
    const int64_t nv = a.N / VEC;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i_first = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // ---- pass 1: alpha = B~^T b (UP strided elements per trip: read-only, more bytes in flight)
    constexpr int UP = FusedUnroll<MC>::FORM_P1;
    double v[MC + 1];
#pragma unroll
    for (int k = 0; k <= MC; ++k) v[k] = 0.0;
    constexpr int64_t W = VEC;
    if constexpr (RF) {
        static_assert(UP == 1 && FusedUnroll<MC>::FORM_P2 == 1 && FusedUnroll<MC>::FORM_PF == 1, "RF: one element per trip");
        V bv = vzero(V()), col[MC];
        {
            const bool ok = i_first < nv;
            const double *p = a.Bt + i_first * W;
            if (ok) bv = ldp<V>(a.b, i_first, ps);
#pragma unroll
            for (int k = 0; k < MC; ++k) {
                col[k] = (ok && k < d) ? ldp<V>(p, 0, ps) : vzero(V());
                p += a.ld;
            }
        }
        for (int64_t i = i_first; i < nv; i += stride) {
            const int64_t in = i + stride;
            const bool okn = in < nv;
            const V bc = bv;
            bv = okn ? ldp<V>(a.b, in, ps) : vzero(V());
            const double *p = a.Bt + in * W;
#pragma unroll
            for (int k = 0; k < MC; ++k) {
                v[k] = vdot(col[k], bc, v[k]);
                col[k] = (okn && k < d) ? ldp<V>(p, 0, ps) : vzero(V());
                p += a.ld;
            }
        }
    } else
    for (int64_t i0 = i_first; i0 < nv; i0 += UP * stride) {
        V bv[UP], col[UP][MC];
#pragma unroll
        for (int u = 0; u < UP; ++u) {
            const int64_t i = i0 + u * stride;
            const bool ok = i < nv;
            bv[u] = ok ? ldp<V>(a.b, i, ps) : vzero(V());
#pragma unroll
            for (int k = 0; k < MC; ++k) col[u][k] = (ok && k < d) ? ldp<V>(a.Bt + k * a.ld, i, ps) : vzero(V());
        }
#pragma unroll
        for (int u = 0; u < UP; ++u)
#pragma unroll
            for (int k = 0; k < MC; ++k) v[k] = vdot(col[u][k], bv[u], v[k]);
    }
    if (VEC == 2 && (a.N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t i = a.N - 1;
        const double bv = a.b[i];
#pragma unroll
        for (int k = 0; k < MC; ++k)
            if (k < d) v[k] = fma(a.Bt[k * a.ld + i], bv, v[k]);
    }
    // the first FP trips of pass 2 are in flight across the barrier (the bubble is ~2-4 us: one
    // trip of 1 CTA/SM covers ~1.5 us of the SM's bandwidth share)
    constexpr int FP = FusedUnroll<MC>::FORM_PF;
    constexpr int UX = FusedUnroll<MC>::FORM_P2;
    XTrip<MC, UX, V> pre[FP];
#pragma unroll
    for (int f = 0; f < FP; ++f) xtrip_load(pre[f], a, i_first + f * UX * stride, stride, nv, d, ps);
    block_partials_store<MC + 1>(v, d, false, a.blk, sh);
    TRACE_F(1);
    grid_barrier(&c->bar[e & 1], 1, &c->err, a.watchdog_ns);
    advance_epoch(c, e);
    TRACE_F(2);
    reduce_all_blocks<MC>(d, false, a.blk, s_red);
    TRACE_F(3);
    if (a.xc.G > 1) peer_allreduce(a.xc, ST_FORM, d, false, s_red, ep, &c->err, a.watchdog_ns);
    double al[MC];
#pragma unroll
    for (int k = 0; k < MC; ++k) al[k] = (k < d) ? s_red[k] : 0.0;
    // ---- pass 2: x0 = X~ alpha (b fully consumed before the barrier: x0 may alias b)
    if constexpr (RF) {
        XTrip<MC, UX, V> &r = pre[0];  // element i_first, loaded before the barrier
        for (int64_t i = i_first; i < nv; i += stride) {
            const int64_t in = i + stride;
            const bool okn = in < nv;
            const double *p = a.Xt + in * W;
            V acc = vzero(V());
#pragma unroll
            for (int k = 0; k < MC; ++k) {
                acc = vaxpy(al[k], r.col[0][k], acc);
                r.col[0][k] = (okn && k < d) ? ldp<V>(p, 0, ps) : vzero(V());
                p += a.ld;
            }
            stv<V>(a.x0, i, acc);
        }
    } else {
#pragma unroll
        for (int f = 0; f < FP; ++f) xtrip_store(pre[f], a, i_first + f * UX * stride, stride, nv, al);
        for (int64_t i0 = i_first + FP * UX * stride; i0 < nv; i0 += UX * stride) {
            XTrip<MC, UX, V> r;
            xtrip_load(r, a, i0, stride, nv, d, ps);
            xtrip_store(r, a, i0, stride, nv, al);
        }
    }
    if (VEC == 2 && (a.N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t i = a.N - 1;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < MC; ++k)
            if (k < d) acc = fma(al[k], a.Xt[k * a.ld + i], acc);
        a.x0[i] = acc;
    }
    TRACE_F(4);
    pdl_trigger();
    // epilogue: every CTA holds the same sums, so CTA 0 writes the control block without waiting
    // for the others (the next kernel sees it after this grid completes)
    if (blockIdx.x == 0) {
        if (threadIdx.x < d) a.part[ST_FORM * PS + threadIdx.x] = s_red[threadIdx.x];
        if (threadIdx.x < d && !isfinite(s_red[threadIdx.x])) watchdog_trip(&c->err, 3);
        if (threadIdx.x == 0 && a.xc.G > 1) c->xepoch[ST_FORM] = ep;
    }
    TRACE_F(7);
}

// Admission of the update's pair (thread 0; AMB-3 / AMB-6 / AMB-8): ||b~2||^2 = ||b~1||^2 - ||c2||^2
// (B~ orthonormal), relative test; a non-finite sum never admits (the history stays unchanged).
__device__ __forceinline__ void admission(const double *r1, const double *r2, int deff, double eps, double &nb,
                                          double &nAx, int &adm) {
    const double nAx2 = r1[NORM];
    double nb2;
    if (deff > 0) {
        double c2sq = 0.0;
        for (int k = 0; k < deff; ++k) c2sq = fma(r2[k], r2[k], c2sq);
        nb2 = r2[NORM] - c2sq;
    } else {
        nb2 = nAx2;  // d = 0: b~ = Ax
    }
    nb = sqrt(fmax(nb2, 0.0));
    nAx = sqrt(nAx2);
    const bool fin = isfinite(nAx2) && (deff == 0 || isfinite(nb2));
    adm = fin && ((deff > 0) ? (nb > eps * nAx) : (nAx > 0.0));
}

// The update's serial work -- R after this update and the Givens plan of the next downdate
// (Alg. 2) -- runs in a dedicated PLANNER CTA (the last CTA of a QR grid), which streams
// nothing.  At its start it stages the R the plan will act on (the downdated R if this update
// downdates, else R) in shared memory and, if this update can end with d = M, runs the plan's
// prefix (rotations 0..M-3, independent of this update's sums: proj_common.cuh) while the
// streaming CTAs run passes 1 and 2; after barrier 2 it reduces the same block partials in the
// same order as every other CTA (bitwise-identical sums and decisions), adds the new R column and
// runs the plan's suffix (one column, one rotation).  The serial chain (L2-latency-bound R assembly
// ~12 us and ~0.4 us per rotation at M = 30) is off the critical path at every N.  It arrives once
// at the barrier counter at its start (so CTA 0 advances the launch epoch only after every CTA,
// planner included, has read it) and never waits at a barrier: barrier p of the streaming CTAs
// waits for p * ns + 1 arrivals.
template <int MC>
__device__ __noinline__ void planner_cta(const ProjArgs &a, unsigned ns) {
    // its own shared arrays and control-block reads: a small call interface keeps the streaming
    // CTAs' register allocation independent of this code, which is also laid out away from the
    // streaming passes (their cold code per launch is fetched from L2 under full HBM load)
    __shared__ double sR[MAXM * MAXM], sW[MAXM * 32], s_r1[PS], s_r2[PS], pgc[MAXM], pgs[MAXM];
    __shared__ double s_nb, s_nAx;
    __shared__ int s_adm;
    Ctrl *c = a.ctrl;
    const int M = a.M;
    const unsigned e = *(volatile unsigned *)&c->epoch;
    const int d = c->d;
    const bool pend = c->pending != 0;
    const int deff = pend ? M - 1 : d;
    const unsigned long long ep1 = c->xepoch[ST_U1] + 1, ep2 = c->xepoch[ST_U2] + 1;
    __syncthreads();  // every thread has read the control block
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(&c->bar[e & 1], 1u);
    }
    TRACE(10);
    const double *Rsrc = pend ? c->Rdn : c->R;  // the R this update starts from (after its downdate)
    for (int idx = threadIdx.x; idx < MAXM * MAXM; idx += blockDim.x) sR[idx] = Rsrc[idx];
    __syncthreads();
    const bool could_plan = deff == M - 1;  // admitted -> d = M -> the next update downdates
    if (could_plan && threadIdx.x < 32) plan_prefix(M, sR, sW, pgc, pgs, c->Rdn);
    TRACE(14);
    grid_wait(&c->bar[e & 1], 2 * ns + 1, &c->err, a.watchdog_ns);  // the streaming CTAs' pass 2 partials
    TRACE(13);
    reduce_all_blocks<MC>(deff, true, a.blk, s_r1, (int)ns);
    if (a.xc.G > 1) peer_allreduce(a.xc, ST_U1, deff, true, s_r1, ep1, &c->err, a.watchdog_ns);
    if (deff > 0) reduce_all_blocks<MC>(deff, true, a.blk + BLK2, s_r2, (int)ns);
    if (deff > 0 && a.xc.G > 1) peer_allreduce(a.xc, ST_U2, deff, true, s_r2, ep2, &c->err, a.watchdog_ns);
    if (threadIdx.x == 0) {
        double nb, nAx;
        int adm;
        admission(s_r1, s_r2, deff, a.eps, nb, nAx, adm);
        s_nb = nb;
        s_nAx = nAx;
        s_adm = adm;
    }
    __syncthreads();
    const bool adm = s_adm != 0;
    const int dnew = deff + (adm ? 1 : 0);
    if (threadIdx.x < 32) {
        r_update(c, M, deff, pend, adm, s_r1, s_r2, s_nb, sR);
        if (dnew == M) {  // the next update downdates
            plan_suffix(M, sR, sW, pgc, pgs, c->Rdn);
            plan_publish(c, M, pgc, pgs);
        }
    }
    TRACE(11);
}

// OC: the one-copy pass-3 loop (see pass 3); a separate instantiation, chosen by the launcher for the
// M > 8 buckets below 2^24 DOFs, so the large-vector kernels keep their exact code and registers.
template <int MC, int VEC, bool OC = false>
__global__ void __launch_bounds__(THREADS, 1) k_update_fused(const __grid_constant__ ProjArgs a) {
    typedef typename VT<VEC>::T V;
    constexpr int U = FusedUnroll<MC>::U;
    __shared__ double sh[(THREADS / 32) * (MC + 1)];
    __shared__ double s_r1[PS], s_r2[PS];
    __shared__ double s_gc[MAXM], s_gs[MAXM], s_c1[MAXM], s_c2[MAXM];
    constexpr bool SMC = FusedUnroll<MC>::SMEM_COEF;
    constexpr int U3 = FusedUnroll<MC>::U3;
    __shared__ double s_nb, s_nAx;
    __shared__ int s_adm;
    __shared__ double s_R[MAXM * MAXM], s_W[MAXM * 32];
    TRACE(8);
    pdl_wait();  // stream predecessor complete and visible (programmatic dependent launch)
#ifdef IG_TRACE
    if (threadIdx.x == 0) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_trace[blockIdx.x * 16 + 12] = sm;
    }
#endif
    Ctrl *c = a.ctrl;
    const unsigned e = launch_epoch(c);
    const int d = c->d, M = a.M;
    const bool pend = c->pending != 0;
    const bool restart = (a.method == M_PROJ_CLASSIC) && (d >= M);  // Alg. 1 restart
    const int deff = pend ? M - 1 : (restart ? 0 : d);
    const unsigned long long ep1 = c->xepoch[ST_U1] + 1, ep2 = c->xepoch[ST_U2] + 1;
    // QR grids of >= 2 CTAs: the last CTA is the planner, the others stream (ns of them)
    const bool has_planner = a.method == M_PROJ_QR && gridDim.x >= 2;
    const unsigned ns = gridDim.x - (has_planner ? 1u : 0u);
    const unsigned bt = has_planner ? 1u : 0u;  // the planner's single arrival
    if (has_planner && blockIdx.x == ns) {
        planner_cta<MC>(a, ns);
        return;
    }
    const L2Pol pol = make_l2pol();
    TRACE(0);
    if (threadIdx.x < MAXM) {
        const bool rot = pend && threadIdx.x < M - 1;
        s_gc[threadIdx.x] = rot ? c->gc[threadIdx.x] : 1.0;
        s_gs[threadIdx.x] = rot ? c->gs[threadIdx.x] : 0.0;
    }
    __syncthreads();
    double gcr[SMC ? 1 : MC], gsr[SMC ? 1 : MC], c1r[SMC ? 1 : MC], c2r[SMC ? 1 : MC];
    if constexpr (!SMC) {
#pragma unroll
        for (int k = 0; k < MC; ++k) {
            gcr[k] = s_gc[k];
            gsr[k] = s_gs[k];
        }
    }
    typedef typename std::conditional<SMC, const volatile double *, const double *>::type CP;
    const CP gc = SMC ? (CP)s_gc : (CP)gcr;
    const CP gs = SMC ? (CP)s_gs : (CP)gsr;
    const CP c1 = SMC ? (CP)s_c1 : (CP)c1r;
    const CP c2 = SMC ? (CP)s_c2 : (CP)c2r;
    const int64_t nv = a.N / VEC;
    const int64_t stride = (int64_t)ns * blockDim.x;
    const int64_t i_first = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool tail = VEC == 2 && (a.N & 1) && blockIdx.x == 0 && threadIdx.x == 0;
    // ---- pass 1: [Givens rotation of B~] + c1 = B~^T Ax, ||Ax||^2
    double v[MC + 1];
#pragma unroll
    for (int k = 0; k <= MC; ++k) v[k] = 0.0;
    constexpr int UU1 = U;  // pass-1 elements per trip
    // ROLL: rolling prefetch in passes 1 and 2 (one element per trip; u1_roll / u2_roll)
    constexpr bool ROLL = (OC ? MC >= IG_ROLL_MIN : MC >= IG_ROLL_BIG_MIN) && U == 1 && FusedUnroll<MC>::U2 == 1;
    if constexpr (ROLL) {
        U2Trip<MC, 1, V> r1;
        const int nload = pend ? M : deff;
        if (i_first < nv) u2trip_load(r1, a, i_first, stride, nv, nload, pol.keep);
        if (pend) {
            for (int64_t i = i_first; i < nv; i += stride)
                u1_roll<MC, true>(r1, a, i, i + stride, i + stride < nv, nload, gc, gs, v, pol.keep);
        } else {
            for (int64_t i = i_first; i < nv; i += stride)
                u1_roll<MC, false>(r1, a, i, i + stride, i + stride < nv, nload, gc, gs, v, pol.keep);
        }
    } else {
        for (int64_t i0 = i_first; i0 < nv; i0 += UU1 * stride) u1_trip<MC, UU1, V>(a, i0, stride, nv, pend, deff, gc, gs, v, pol.keep);
    }
    if (tail) u1_trip<MC, 1, double>(a, a.N - 1, 1, a.N, pend, deff, gc, gs, v, pol.keep);
    // Serpentine order: pass 2 walks the vectors BACKWARDS, so it starts on the B~/Ax lines pass 1
    // touched last (still in the 126 MB L2); pass 3 walks forwards again and starts on what pass 2
    // touched last.  Same arithmetic per element, fewer HBM bytes per step.
    constexpr int UB = FusedUnroll<MC>::U2;
    const int64_t ntrip2 = (i_first < nv) ? (nv - i_first + UB * stride - 1) / (UB * stride) : 0;
    U2Trip<MC, UB, V> pre2;
    if (deff > 0 && ntrip2 > 0) u2trip_load(pre2, a, i_first + (ntrip2 - 1) * UB * stride, stride, nv, deff, pol.keep);
    block_partials_store<MC + 1>(v, deff, true, a.blk, sh);
    TRACE(1);
    grid_barrier(&c->bar[e & 1], 1, &c->err, a.watchdog_ns, ns + bt);
    advance_epoch(c, e);
    TRACE(2);
    reduce_all_blocks<MC>(deff, true, a.blk, s_r1, (int)ns);
    TRACE(3);
    if (a.xc.G > 1) peer_allreduce(a.xc, ST_U1, deff, true, s_r1, ep1, &c->err, a.watchdog_ns);
    if (threadIdx.x < MAXM) s_c1[threadIdx.x] = (threadIdx.x < deff) ? s_r1[threadIdx.x] : 0.0;
    __syncthreads();
    if constexpr (!SMC) {
#pragma unroll
        for (int k = 0; k < MC; ++k) c1r[k] = s_c1[k];
    }
    // ---- pass 2: b1 = Ax - B~ c1 (registers), c2 = B~^T b1, ||b1||^2
    if (deff > 0) {
#pragma unroll
        for (int k = 0; k <= MC; ++k) v[k] = 0.0;
        if constexpr (ROLL) {
            for (int64_t t = ntrip2 - 1; t >= 0; --t) u2_roll(pre2, a, i_first + (t - 1) * stride, t > 0, deff, c1, v, pol.keep);
        } else {
            for (int64_t t = ntrip2 - 1; t >= 0; --t) {  // one copy of the trip code (pre2 = the first)
                if (t < ntrip2 - 1) u2trip_load(pre2, a, i_first + t * UB * stride, stride, nv, deff, pol.keep);
                u2trip_compute(pre2, c1, v);
            }
        }
        if (tail) {
            U2Trip<MC, 1, double> r;
            u2trip_load(r, a, a.N - 1, 1, a.N, deff, pol.keep);
            u2trip_compute(r, c1, v);
        }
    }
    // first trip of pass 3, in flight across barrier 2 (ROLL3: the B~ part of the first element)
    constexpr bool ROLL3 = OC && MC >= IG_ROLL3_MIN && MC <= IG_ROLL3_MAX && U3 == 1;
    U3Trip<MC, U3, V> pre3;
    R3<MC, V> r3;
    if constexpr (ROLL3)
        r3_load(r3, a, i_first, i_first < nv, deff, pend, true, pol.stream);
    else
        u3trip_load(pre3, a, i_first, stride, nv, deff, pend, true, pol.stream);
    if (deff > 0) block_partials_store<MC + 1>(v, deff, true, a.blk + BLK2, sh);
    TRACE(4);
    grid_barrier(&c->bar[e & 1], 2, &c->err, a.watchdog_ns, 2 * ns + bt);
    TRACE(5);
    if (deff > 0) reduce_all_blocks<MC>(deff, true, a.blk + BLK2, s_r2, (int)ns);
    if (deff > 0 && a.xc.G > 1) peer_allreduce(a.xc, ST_U2, deff, true, s_r2, ep2, &c->err, a.watchdog_ns);
    if (threadIdx.x == 0) {
        double nb, nAx;
        int adm;
        admission(s_r1, s_r2, deff, a.eps, nb, nAx, adm);
        s_nb = nb;
        s_nAx = nAx;
        s_adm = adm;
    }
    __syncthreads();
    const bool adm = s_adm != 0;
    const double inv = adm ? 1.0 / s_nb : 0.0;
    if (threadIdx.x < MAXM) s_c2[threadIdx.x] = (deff > 0 && threadIdx.x < deff) ? s_r2[threadIdx.x] : 0.0;
    __syncthreads();
    if constexpr (!SMC) {
#pragma unroll
        for (int k = 0; k < MC; ++k) c2r[k] = s_c2[k];
    }
    // a zero A x is skipped (AMB-6); for CLASSIC at d >= M that includes the restart:
    // the full history is kept (Alg. 1's restart branch divides by ||b~||)
    const int dnew = (restart && !adm) ? d : deff + (adm ? 1 : 0);
    const bool plan = a.method == M_PROJ_QR && dnew == M;  // the next update downdates
    // ---- pass 3: [Givens rotation of X~] + store the admitted pair
    if (adm || pend) {
        // ~7/8 of the trips in the static grid-stride order (trip 0 is the prefetched pre3), the
        // last ~1/8 of the rows handed out to warps on demand (32*U3-row chunks, atomic claim):
        // CTAs on slower SMs take fewer tail chunks, so all CTAs reach the exit together.
        const int64_t chunk = (int64_t)U3 * stride;
        const int64_t trips = (nv + chunk - 1) / chunk;
        // (1/4 and 1/16 of the rows measured no better: profiles/r2_planner_ab.md)
        const int64_t Ts = trips < 4 ? trips : trips - (trips + 7) / 8;
        // dynamic claims: the tail rows [S, nv) in 32*U3-row chunks
        // OC (M > 8 buckets below 2^24 DOFs): ONE copy of the large trip code (~900 / ~1900
        // instructions at M = 16 / 32) serves the static trips and the claims, loading at the end of
        // each iteration for the next item -- the pass's hot code is half the size, which pays once
        // it no longer fits the instruction cache and the pass is short (profiles/r2_onecopy_ab.md:
        // N = 1e6 QR(12) 145.6 -> 138.1, QR(17) 255 -> 230, QR(30) 357 -> 339 us); at 2^27 the
        // two-copy form is as fast or faster, so large vectors use the OC = false kernel.
        if constexpr (ROLL3) {
            // as the OC loop below, with the rolling register set: the next item (static trip or
            // claim) is known before the current one is processed
            const int64_t S = Ts * chunk, WCH = 32;
            const int64_t nq = nv > S ? (nv - S + WCH - 1) / WCH : 0;
            const int lane = threadIdx.x & 31;
            if (Ts > 0) {
                int64_t t = 0, i0 = i_first;
                unsigned qn = 0xffffffffu;
                while (true) {
                    if (nq > 0 && t >= Ts - 1) {  // the next item is a claim: take its ticket now
                        unsigned v = (lane == 0) ? atomicAdd(&c->dyn3[e & 1], 1u) : 0u;
                        qn = __shfl_sync(0xffffffffu, v, 0);
                    }
                    const bool has = (t + 1 < Ts) || ((int64_t)qn < nq);  // also nq == 0 (qn stays ~0)
                    const int64_t in = (t + 1 < Ts) ? i_first + (t + 1) * chunk : S + (int64_t)qn * WCH + lane;
                    u3_roll(r3, a, i0, i0 < nv, in, has && in < nv, deff, pend, adm, inv, c1, c2, gc, gs, pol.stream);
                    if (!has) break;
                    t = (t + 1 < Ts) ? t + 1 : Ts;
                    i0 = in;
                }
            }
        } else if constexpr (OC) {
            const int64_t S = Ts * chunk, WCH = 32 * U3;
            const int64_t nq = nv > S ? (nv - S + WCH - 1) / WCH : 0;
            const int lane = threadIdx.x & 31;
            // ONE copy of the (large: ~1900 instructions at M = 32) trip code for the static trips
            // and the claims, loads at the end of each iteration for the next item: the pass's hot
            // code is half the size, which matters once it no longer fits the instruction cache
            if (Ts > 0) {
                int64_t t = 0, i0 = i_first, st = stride;
                unsigned qn = 0xffffffffu;
                while (true) {
                    if (nq > 0 && t >= Ts - 1) {  // the next item is a claim: take its ticket now
                        unsigned v = (lane == 0) ? atomicAdd(&c->dyn3[e & 1], 1u) : 0u;
                        qn = __shfl_sync(0xffffffffu, v, 0);
                    }
                    u3trip_store(pre3, a, i0, st, nv, deff, pend, adm, inv, c1, c2, gc, gs, pol.stream);
                    if (t + 1 < Ts) {
                        ++t;
                        i0 = i_first + t * chunk;
                        st = stride;
                    } else {
                        t = Ts;
                        if ((int64_t)qn >= nq) break;  // also nq == 0 (qn stays ~0)
                        i0 = S + (int64_t)qn * WCH + lane;
                        st = 32;
                    }
                    u3trip_load(pre3, a, i0, st, nv, deff, pend, adm, pol.stream);
                }
            }
        } else {
            if (Ts > 0) u3trip_store(pre3, a, i_first, stride, nv, deff, pend, adm, inv, c1, c2, gc, gs, pol.stream);
            for (int64_t t = 1; t < Ts; ++t) {
                const int64_t i0 = i_first + t * chunk;
                U3Trip<MC, U3, V> r;
                u3trip_load(r, a, i0, stride, nv, deff, pend, adm, pol.stream);
                u3trip_store(r, a, i0, stride, nv, deff, pend, adm, inv, c1, c2, gc, gs, pol.stream);
            }
            const int64_t S = Ts * chunk, WCH = 32 * U3;
            const int64_t nq = nv > S ? (nv - S + WCH - 1) / WCH : 0;
            if (nq > 0) {
                const int lane = threadIdx.x & 31;
                unsigned q = (lane == 0) ? atomicAdd(&c->dyn3[e & 1], 1u) : 0u;
                q = __shfl_sync(0xffffffffu, q, 0);
                while ((int64_t)q < nq) {
                    unsigned qn = (lane == 0) ? atomicAdd(&c->dyn3[e & 1], 1u) : 0u;  // claim the next one early
                    U3Trip<MC, U3, V> r;
                    const int64_t i0 = S + (int64_t)q * WCH + lane;
                    u3trip_load(r, a, i0, 32, nv, deff, pend, adm, pol.stream);
                    u3trip_store(r, a, i0, 32, nv, deff, pend, adm, inv, c1, c2, gc, gs, pol.stream);
                    q = __shfl_sync(0xffffffffu, qn, 0);
                }
            }
        }
        if (tail) {
            U3Trip<MC, 1, double> r;
            u3trip_load(r, a, a.N - 1, 1, a.N, deff, pend, adm, pol.stream);
            u3trip_store(r, a, a.N - 1, 1, a.N, deff, pend, adm, inv, c1, c2, gc, gs, pol.stream);
        }
    }
    TRACE(6);
    pdl_trigger();
    // ---- epilogue: every CTA holds the same sums and decisions, so CTA 0 writes the control
    // block without waiting for the others (every CTA read it before barrier 1; the next kernel
    // sees it after this grid completes).  No exit barrier, no fence drain on the critical path.
    if (blockIdx.x != 0) {
        TRACE(7);
        return;
    }
    TRACE(9);
    if (!has_planner && a.method == M_PROJ_QR && threadIdx.x < 32) {
        // single-CTA grid: R update and plan here, serially (CTA 0 read c->gc at its start)
        const bool newcol = adm;
        const double *Rsrc = pend ? c->Rdn : c->R;
        for (int idx = threadIdx.x; idx < MAXM * MAXM; idx += 32) s_R[idx] = Rsrc[idx];
        __syncwarp();
        r_update(c, M, deff, pend, newcol, s_r1, s_r2, s_nb, s_R);
        if (plan) givens_plan(c, M, s_R, s_W, s_c1, s_c2);  // s_c1/s_c2 are free after pass 3
    }
    if (threadIdx.x < PS) {
        a.part[ST_U1 * PS + threadIdx.x] = s_r1[threadIdx.x];
        a.part[ST_U2 * PS + threadIdx.x] = (deff > 0) ? s_r2[threadIdx.x] : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // failure detection: non-finite inputs poison the sums (the pair is then not admitted)
        bool fin = isfinite(s_r1[NORM]) && (deff == 0 || isfinite(s_r2[NORM]));
        for (int k = 0; k < deff; ++k) fin = fin && isfinite(s_r1[k]) && isfinite(s_r2[k]);
        if (!fin) watchdog_trip(&c->err, 3);
        c->d = dnew;
        c->deff = deff;
        c->pending = plan ? 1 : 0;
        c->admitted = adm ? 1 : 0;
        c->nb = s_nb;
        c->nAx = s_nAx;
        c->rho = (s_nAx > 0.0) ? s_nb / s_nAx : 0.0;
        c->last_rot = pend ? 1 : 0;
        c->rotX = 0;
        if (a.xc.G > 1) {
            c->xepoch[ST_U1] = ep1;
            if (deff > 0) c->xepoch[ST_U2] = ep2;
        }
    }
    __syncthreads();
    TRACE(7);
}

// ------------------------------------------------------------------ launchers (cooperative unless the handle asks for plain)
template <class K> static cudaError_t coop_launch(K kern, const ProjArgs &a, int nsm, cudaStream_t s) {
    static_assert(sizeof(ProjArgs) < 4096, "kernel parameters");
    int occ = cached_occupancy((const void *)kern);
    if (occ < 1) return cudaErrorInvalidConfiguration;
    if (occ > 4) occ = 4;
    int grid = nsm * occ;
    if (a.max_grid > 0 && grid > a.max_grid) grid = a.max_grid;
    if (grid > MAXB) grid = MAXB;
    return launch_ex(kern, grid, s, a.coop != 0, a);
}

// History-size buckets of the fused kernels.  Columns beyond M are predicated off but still cost
// issue slots and registers, and at one CTA of 8 warps per SM the first M of a coarse bucket was
// issue-bound (2^27 DOFs, buckets 1/2/4/8/12/16/24/32: QR(5) 0.92, QR(9) 0.91, QR(13) 0.95,
// QR(17) 0.95 of copy; profiles/r3_roll_ab.md).  IG_FINE_BUCKETS=0 restores those buckets.
#ifndef IG_FINE_BUCKETS
#define IG_FINE_BUCKETS 1
#endif
static int mcb(int M) {
    if (M <= 4) return M <= 1 ? 1 : M <= 2 ? 2 : 4;
#ifndef IG_MC5
#define IG_MC5 1
#endif
    if (IG_FINE_BUCKETS) return (IG_MC5 && M == 5) ? 5 : M <= 6 ? 6 : M <= 8 ? 8 : M <= 10 ? 10 : M <= 12 ? 12 : M <= 14 ? 14 : M <= 16 ? 16
                              : M <= 20 ? 20 : M <= 24 ? 24 : M <= 28 ? 28 : 32;
    return M <= 8 ? 8 : M <= 12 ? 12 : M <= 16 ? 16 : M <= 24 ? 24 : 32;
}

#define IG_FUSED_DISPATCH(KERNEL, ARGS, VEC_IN, NSM, STREAM)                                        \
    do {                                                                                            \
        const int mc = mcb((ARGS).M);                                                               \
        const bool v2 = ((VEC_IN) == 2);                                                            \
        switch (mc) {                                                                               \
        case 1: return v2 ? coop_launch(KERNEL<1, 2>, ARGS, NSM, STREAM)                            \
                          : coop_launch(KERNEL<1, 1>, ARGS, NSM, STREAM);                           \
        case 2: return v2 ? coop_launch(KERNEL<2, 2>, ARGS, NSM, STREAM)                            \
                          : coop_launch(KERNEL<2, 1>, ARGS, NSM, STREAM);                           \
        case 4: return v2 ? coop_launch(KERNEL<4, 2>, ARGS, NSM, STREAM)                            \
                          : coop_launch(KERNEL<4, 1>, ARGS, NSM, STREAM);                           \
        case 5: return v2 ? coop_launch(KERNEL<5, 2>, ARGS, NSM, STREAM)                            \
                          : coop_launch(KERNEL<5, 1>, ARGS, NSM, STREAM);                           \
        case 6: return v2 ? coop_launch(KERNEL<6, 2>, ARGS, NSM, STREAM)                            \
                          : coop_launch(KERNEL<6, 1>, ARGS, NSM, STREAM);                           \
        case 8: return v2 ? coop_launch(KERNEL<8, 2>, ARGS, NSM, STREAM)                            \
                          : coop_launch(KERNEL<8, 1>, ARGS, NSM, STREAM);                           \
        case 10: return v2 ? coop_launch(KERNEL<10, 2>, ARGS, NSM, STREAM)                          \
                           : coop_launch(KERNEL<10, 1>, ARGS, NSM, STREAM);                         \
        case 12: return v2 ? coop_launch(KERNEL<12, 2>, ARGS, NSM, STREAM)                          \
                           : coop_launch(KERNEL<12, 1>, ARGS, NSM, STREAM);                         \
        case 14: return v2 ? coop_launch(KERNEL<14, 2>, ARGS, NSM, STREAM)                          \
                           : coop_launch(KERNEL<14, 1>, ARGS, NSM, STREAM);                         \
        case 16: return v2 ? coop_launch(KERNEL<16, 2>, ARGS, NSM, STREAM)                          \
                           : coop_launch(KERNEL<16, 1>, ARGS, NSM, STREAM);                         \
        case 20: return v2 ? coop_launch(KERNEL<20, 2>, ARGS, NSM, STREAM)                          \
                           : coop_launch(KERNEL<20, 1>, ARGS, NSM, STREAM);                         \
        case 24: return v2 ? coop_launch(KERNEL<24, 2>, ARGS, NSM, STREAM)                          \
                           : coop_launch(KERNEL<24, 1>, ARGS, NSM, STREAM);                         \
        case 28: return v2 ? coop_launch(KERNEL<28, 2>, ARGS, NSM, STREAM)                          \
                           : coop_launch(KERNEL<28, 1>, ARGS, NSM, STREAM);                         \
        default: return v2 ? coop_launch(KERNEL<32, 2>, ARGS, NSM, STREAM)                          \
                           : coop_launch(KERNEL<32, 1>, ARGS, NSM, STREAM);                         \
        }                                                                                           \
    } while (0)

// Rolling form kernel for M = 17..32 at every N (A/B, profiles/r3_roll_ab.md: N = 1e6 QR(30)
// 335.5 -> 330.8, 1e7 QR(30) 3024 -> 2987 us/step; neutral at M = 16 and 0.8 us slower at 3e5
// QR(12), so the M <= 16 buckets keep the unrolled form).  -DIG_FORM_RF=0 turns it off.
#ifndef IG_FORM_RF
#define IG_FORM_RF 1
#endif
cudaError_t launch_form_fused(const ProjArgs &a, int vec, int nsm, cudaStream_t s) {
    if (IG_FORM_RF && vec == 2 && mcb(a.M) > 16) switch (mcb(a.M)) {
        case 20: return coop_launch(k_form_fused<20, 2, true>, a, nsm, s);
        case 24: return coop_launch(k_form_fused<24, 2, true>, a, nsm, s);
        case 28: return coop_launch(k_form_fused<28, 2, true>, a, nsm, s);
        default: return coop_launch(k_form_fused<32, 2, true>, a, nsm, s);
        }
    IG_FUSED_DISPATCH(k_form_fused, a, vec, nsm, s);
}
cudaError_t launch_update_fused(const ProjArgs &a, int vec, int nsm, cudaStream_t s) {
    const int mc = mcb(a.M);
    if (vec == 2 && mc > 8 && a.N < (int64_t(1) << 24)) switch (mc) {
        case 10: return coop_launch(k_update_fused<10, 2, true>, a, nsm, s);
        case 12: return coop_launch(k_update_fused<12, 2, true>, a, nsm, s);
        case 14: return coop_launch(k_update_fused<14, 2, true>, a, nsm, s);
        case 16: return coop_launch(k_update_fused<16, 2, true>, a, nsm, s);
        case 20: return coop_launch(k_update_fused<20, 2, true>, a, nsm, s);
        case 24: return coop_launch(k_update_fused<24, 2, true>, a, nsm, s);
        case 28: return coop_launch(k_update_fused<28, 2, true>, a, nsm, s);
        default: return coop_launch(k_update_fused<32, 2, true>, a, nsm, s);
        }
    IG_FUSED_DISPATCH(k_update_fused, a, vec, nsm, s);
}

}  // namespace ig
