// proj_common.cuh -- device helpers shared by the projection kernels (kern_proj.cu: one kernel per
// pass, used with G > 1 ranks; kern_fused.cu: persistent fused kernels, single GPU).
#pragma once
#include <type_traits>

#include "ig_internal.h"

namespace ig {

template <int VEC> struct VT;
template <> struct VT<1> { typedef double T; };
template <> struct VT<2> { typedef double2 T; };

__device__ __forceinline__ double vzero(double) { return 0.0; }
__device__ __forceinline__ double2 vzero(double2) { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double vdot(double a, double b, double acc) { return fma(a, b, acc); }
__device__ __forceinline__ double vdot(double2 a, double2 b, double acc) {
    return fma(a.y, b.y, fma(a.x, b.x, acc));
}
// y + s*a
__device__ __forceinline__ double vaxpy(double s, double a, double y) { return fma(s, a, y); }
__device__ __forceinline__ double2 vaxpy(double s, double2 a, double2 y) {
    return make_double2(fma(s, a.x, y.x), fma(s, a.y, y.y));
}
__device__ __forceinline__ double vscale(double s, double a) { return s * a; }
__device__ __forceinline__ double2 vscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
// (out, t) <- (c t + s n, -s t + c n): one Givens rotation of a column pair
__device__ __forceinline__ void vrot(double c, double s, double &t, double n, double &out) {
    out = c * t + s * n;
    t = -s * t + c * n;
}
__device__ __forceinline__ void vrot(double c, double s, double2 &t, double2 n, double2 &out) {
    vrot(c, s, t.x, n.x, out.x);
    vrot(c, s, t.y, n.y, out.y);
}

template <class V> __device__ __forceinline__ V ldro(const double *base, int64_t i) {
    return __ldg(reinterpret_cast<const V *>(base) + i);
}
template <class V> __device__ __forceinline__ V ldrw(const double *base, int64_t i) {
    return reinterpret_cast<const V *>(base)[i];
}
template <class V> __device__ __forceinline__ void stv(double *base, int64_t i, V v) {
    reinterpret_cast<V *>(base)[i] = v;
}

// L2 eviction-priority policies (createpolicy + .L2::cache_hint).  The update call marks the B~/Ax
// lines that later passes of the SAME call re-read as evict_last and its single-use traffic as
// evict_first, so the serpentine pass order finds more of its re-reads in the 126 MB L2.
struct L2Pol {
    unsigned long long keep, stream;
};
__device__ __forceinline__ L2Pol make_l2pol() {
    L2Pol p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p.keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p.stream));
    return p;
}
template <class V> __device__ __forceinline__ V ldp(const double *base, int64_t i, unsigned long long pol);
template <> __device__ __forceinline__ double2 ldp<double2>(const double *base, int64_t i, unsigned long long pol) {
    double2 r;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(reinterpret_cast<const double2 *>(base) + i), "l"(pol));
    return r;
}
template <> __device__ __forceinline__ double ldp<double>(const double *base, int64_t i, unsigned long long pol) {
    double r;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(base + i), "l"(pol));
    return r;
}
template <class V> __device__ __forceinline__ void stp(double *base, int64_t i, V v, unsigned long long pol);
template <> __device__ __forceinline__ void stp<double2>(double *base, int64_t i, double2 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(reinterpret_cast<double2 *>(base) + i),
                 "d"(v.x), "d"(v.y), "l"(pol)
                 : "memory");
}
template <> __device__ __forceinline__ void stp<double>(double *base, int64_t i, double v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(base + i), "d"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Warp sums of the MC coefficient values by a butterfly reduce-scatter: at xor offset o a lane
// keeps one half of the values it still holds and receives the partner's partial sums of that
// half (K/2 shuffles), so MC values cost MC-1 shuffles instead of 5*MC.  Lane l ends up holding
// the warp sum of value index l / (32/K0) (K0 = MC rounded up to a power of two, K0 <= 32); the
// fixed xor pattern makes the summation order deterministic.  The norm (value MC) is a plain
// xor-tree sum.  Inactive values are exact zeros, so they are reduced like the others and only
// the stores are conditional (no divergent shuffles).
template <int MC> struct Pow2 {
    static constexpr int K0 = MC <= 1 ? 1 : MC <= 2 ? 2 : MC <= 4 ? 4 : MC <= 8 ? 8 : MC <= 16 ? 16 : 32;
};
// Works in place: v[0..MC-1] are clobbered (the callers' accumulators are dead afterwards).
template <int MC>
__device__ __forceinline__ void warp_reduce_scatter(double (&v)[MC + 1], double &mine, double &norm) {
    constexpr int K0 = Pow2<MC>::K0;
    const int lane = threadIdx.x & 31;
    norm = warp_sum(v[MC]);
    double *w = v;  // K0 <= MC whenever K0 > 1 is padded below: use a zero pad slot for MC < K0
    double pad[K0 > MC ? K0 - MC : 1];
#pragma unroll
    for (int k = 0; k < (K0 > MC ? K0 - MC : 1); ++k) pad[k] = 0.0;
#pragma unroll
    for (int L = 0; L < 5; ++L) {
        const int o = 16 >> L;
        const int K = K0 >> L;  // values still held before this step (compile-time after unrolling)
        if (K > 1) {
            const int h = K / 2;
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int j = 0; j < h; ++j) {
                const double hi = (j + h < MC) ? w[j + h] : pad[(j + h - MC) < 0 ? 0 : (j + h - MC)];
                const double send = up ? w[j] : hi;
                const double keep = up ? hi : w[j];
                w[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        } else {
            w[0] += __shfl_xor_sync(0xffffffffu, w[0], o);
        }
    }
    mine = w[0];
}
// Index of the value lane `lane` holds after warp_reduce_scatter<MC>.
template <int MC> __device__ __forceinline__ int scatter_index(int lane) { return lane / (32 / Pow2<MC>::K0); }

// Block-reduce NV = MC+1 per-thread values (value MC is a squared norm, slot NORM) into this
// block's partials blk[slot*MAXB + blockIdx] (warp sums in shared memory, then warp-ordered sums).
template <int NV>
__device__ __forceinline__ void block_partials_store(double (&v)[NV], int nc, bool norm, double *blk, double *sh) {
    constexpr int MC = NV - 1;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double mine, nrm;
    warp_reduce_scatter<MC>(v, mine, nrm);
    const int k = scatter_index<MC>(lane);
    if (k < MC && (lane % (32 / Pow2<MC>::K0)) == 0) sh[w * NV + k] = mine;
    if (lane == 0) sh[w * NV + MC] = nrm;
    __syncthreads();
    for (int q = threadIdx.x; q < NV; q += blockDim.x) {
        const bool act = (q < NV - 1) ? (q < nc) : norm;
        if (act) {
            double s = 0.0;
            for (int j = 0; j < nw; ++j) s += sh[j * NV + q];
            blk[((q < NV - 1) ? q : NORM) * MAXB + blockIdx.x] = s;
        }
    }
}

// As block_partials_store, then take a ticket (one-kernel-per-pass schedule).  Returns true in the
// block that arrived last (it then owns the final, block-ordered reduction).
template <int NV>
__device__ __forceinline__ bool block_partials_ticket(double (&v)[NV], int nc, bool norm, double *blk,
                                                      unsigned *ticket, double *sh) {
    block_partials_store<NV>(v, nc, norm, blk, sh);
    __threadfence();
    __syncthreads();
    __shared__ unsigned s_ticket;
    if (threadIdx.x == 0) s_ticket = atomicAdd(ticket, 1u);
    __syncthreads();
    const bool last = (s_ticket == gridDim.x - 1);
    if (last) __threadfence();
    return last;
}

// out[slot] = sum over the gridDim.x block partials of that slot, in a fixed order.  Two stages:
// TPS = THREADS/(MC+1) threads per slot each sum the blocks r, r+TPS, ... (all loads of a chunk in
// flight: one L2 round trip for <= CHK*TPS blocks), then one thread per slot sums the TPS partials
// in order (shared memory).  Few registers, so the trip prefetched across a barrier stays resident
// even at M = 32.  Deterministic for a given grid.  Every thread of the block must call it.
template <int MC>
__device__ __forceinline__ void final_reduce(int nc, bool norm, const double *blk, double *out, int nblk = -1) {
    constexpr int NS = MC + 1;
    constexpr int TPS = THREADS / NS;
    constexpr int CHK = NS > 17 ? 24 : 12;
    __shared__ double s_part[NS * TPS];
    const int t = threadIdx.x, q = t / TPS, r = t % TPS;
    const int nb = nblk > 0 ? nblk : (int)gridDim.x;  // blocks that stored partials
    if (q < NS) {
        const bool act = (q < MC) ? (q < nc) : norm;
        double acc = 0.0;
        if (act) {
            const double *src = blk + ((q < MC) ? q : NORM) * MAXB;
            for (int b0 = r; b0 < nb; b0 += CHK * TPS) {
                double tv[CHK];
#pragma unroll
                for (int u = 0; u < CHK; ++u) tv[u] = (b0 + u * TPS < nb) ? __ldcg(src + b0 + u * TPS) : 0.0;
#pragma unroll
                for (int u = 0; u < CHK; ++u) acc += tv[u];
            }
        }
        s_part[t] = acc;
    }
    __syncthreads();
    if (t < NS) {
        const bool act = (t < MC) ? (t < nc) : norm;
        if (act) {
            double s = s_part[t * TPS];
            for (int j = 1; j < TPS; ++j) s += s_part[t * TPS + j];
            out[(t < MC) ? t : NORM] = s;
        }
    }
}

// ------------------------------------------------------------------ persistent-kernel helpers
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Software grid barrier for a co-resident grid.  `ctr` (the launch epoch's parity counter,
// zeroed by the previous launch, see Ctrl::epoch) counts arrivals monotonically within one launch;
// barrier number `phase` (1, 2, ...) waits for phase*gridDim arrivals.  Safe under CUDA-graph
// replay: the epoch lives in device memory.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Failure detection: a spin that exceeds WATCHDOG_NS (grid not co-resident, a peer rank that
// stopped calling) records a code in the control block and gives up instead of hanging the GPU;
// the host reports IG_E_STATE at the next synchronising call (ig_get_stats / ig_history_dim).
__device__ __forceinline__ void watchdog_trip(int *err, int code) { atomicCAS(err, 0, code); }

// The wait ends at `target` arrivals (default phase * gridDim.x; k_update_fused's planner CTA
// arrives once at its start and never waits at a barrier, see there).
__device__ __forceinline__ void grid_wait(unsigned *ctr, unsigned target, int *err, unsigned long long limit) {
    if (threadIdx.x == 0) {
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_u32(ctr) < target) {
            __nanosleep(20);
            if (globaltimer_ns() - t0 > limit) {
                watchdog_trip(err, 1);
                break;
            }
        }
        __threadfence();
    }
    __syncthreads();
}
__device__ __forceinline__ void grid_barrier(unsigned *ctr, unsigned phase, int *err, unsigned long long limit,
                                             unsigned target = 0) {
    __syncthreads();
    if (threadIdx.x == 0) {
        if (target == 0) target = phase * gridDim.x;
        // arrival: a release-add (bar.sync above made the CTA's writes -- block partials, stored
        // columns -- visible to thread 0, and the release carries them to every acquirer); wait:
        // an acquire spin (orders the other CTAs' writes before this CTA's later reads).  Round 1
        // used fence + atomicAdd + nanosleep polling + fence: N = 1e5 QR(8) 24.8 -> 22.9 us/step
        // with this form, C2 210.0 -> 209.3 (profiles/r2_onecopy_ab.md)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_u32(ctr) < target) {
            if (globaltimer_ns() - t0 > limit) {
                watchdog_trip(err, 1);
                break;
            }
        }
    }
    __syncthreads();
}

// Launch epoch of a persistent fused kernel (call after pdl_wait, before the first barrier, in
// every CTA): CTA 0 zeroes the counters of the NEXT epoch's parity (the launch that used them
// last has completed: stream order).  Returns this launch's epoch.
__device__ __forceinline__ unsigned launch_epoch(Ctrl *c) {
    const unsigned e = *(volatile unsigned *)&c->epoch;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c->bar[(e + 1) & 1] = 0;
        c->dyn3[(e + 1) & 1] = 0;
    }
    return e;
}
// After the first barrier every CTA has read the epoch: CTA 0 advances it for the next launch.
__device__ __forceinline__ void advance_epoch(Ctrl *c, unsigned e) {
    if (blockIdx.x == 0 && threadIdx.x == 0) c->epoch = e + 1;
}

// Every CTA reduces all block partials of a stage in the same fixed order (so all CTAs hold
// bitwise-identical sums) into out[slot] (shared memory).  Ends with __syncthreads().
template <int MC>
__device__ __forceinline__ void reduce_all_blocks(int nc, bool norm, const double *blk, double *out, int nblk = -1) {
    final_reduce<MC>(nc, norm, blk, out, nblk);
    __syncthreads();
}

// ------------------------------------------------------------------ in-kernel peer exchange
__device__ __forceinline__ void st_release_sys_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double ld_relaxed_sys_f64(const double *p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

// Cross-rank sum of one reduction pass inside the persistent kernel, over NVLink peer memory
// (fused compute + collective, replacing the host-launched NCCL all-gather of the split path).
// Every CTA holds the rank-local sums in shared `buf`; CTA 0 stores them into EVERY rank's window
// (remote stores), fences at system scope and releases a per-(stage, sender) epoch flag; every CTA
// acquires all G flags and sums the G contributions in RANK ORDER, so all ranks (and all CTAs)
// get bitwise-identical results.  `buf` is overwritten with the global sums.
__device__ __forceinline__ void peer_allreduce(const Exchange &xc, int stage, int nc, bool norm, double *buf,
                                               unsigned long long epoch, int *err, unsigned long long limit) {
    const int par = (int)(epoch & 1ull);
    const int G = xc.G, me = xc.rank;
    if (blockIdx.x == 0) {
        for (int idx = threadIdx.x; idx < G * PS; idx += blockDim.x) {
            const int r = idx / PS, k = idx % PS;
            const bool act = (k < MAXM) ? (k < nc) : norm;
            if (act) xc.peer[r]->data[stage][par][me][k] = buf[k];
        }
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x < G) st_release_sys_u64(&xc.peer[threadIdx.x]->flag[stage][me], epoch);
    }
    if (threadIdx.x == 0) {
        const XWin *w = xc.peer[me];
        const unsigned long long t0 = globaltimer_ns();
        for (int r = 0; r < G; ++r)
            while (ld_acquire_sys_u64(&w->flag[stage][r]) < epoch) {
                __nanosleep(32);
                if (globaltimer_ns() - t0 > limit) {
                    watchdog_trip(err, 2);
                    break;
                }
            }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < PS; k += blockDim.x) {
        const bool act = (k < MAXM) ? (k < nc) : norm;
        if (!act) continue;
        const XWin *w = xc.peer[me];
        double s = ld_relaxed_sys_f64(&w->data[stage][par][0][k]);
        for (int r = 1; r < G; ++r) s += ld_relaxed_sys_f64(&w->data[stage][par][r][k]);
        buf[k] = s;
    }
    __syncthreads();
}

// Rank-ordered sum of the gathered partials of one stage.
__device__ __forceinline__ double rank_sum(const double *g, int G, int k) {
    double s = g[k];
    for (int r = 1; r < G; ++r) s += g[r * PS + k];
    return s;
}

// All streaming loops follow one pattern: every load of a trip is issued before any
// arithmetic consumes it (`col[]` arrays), and the kernels are compiled with
// __launch_bounds__(THREADS, 1) so ptxas keeps them grouped instead of interleaving loads with
// their DFMAs to save registers (which cut memory-level parallelism to ~2 loads per thread).
// Streams with few vectors process U strided elements per trip for more bytes in flight.
template <int MC> struct Unroll {
    static constexpr int U = MC <= 2 ? 4 : (MC <= 4 ? 2 : 1);
};

template <int MC, int U, class V, class CP>
__device__ __forceinline__ void u1_trip(const ProjArgs &a, int64_t i0, int64_t stride, int64_t nv, bool pend,
                                        int deff, CP gc, CP gs, double (&v)[MC + 1], unsigned long long pk) {
    const int nload = pend ? a.M : deff;
    V col[U][MC], ax[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * stride;
        const bool ok = i < nv;
        ax[u] = ok ? ldp<V>(a.Ax, i, pk) : vzero(V());
#pragma unroll
        for (int k = 0; k < MC; ++k) col[u][k] = (ok && k < nload) ? ldp<V>(a.Bt + k * a.ld, i, pk) : vzero(V());
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * stride;
        v[MC] = vdot(ax[u], ax[u], v[MC]);
        if (pend) {
            V t = col[u][0];
#pragma unroll
            for (int k = 0; k < MC - 1; ++k) {
                if (k < a.M - 1) {
                    V nk;
                    vrot(gc[k], gs[k], t, col[u][k + 1], nk);
                    if (i < nv) stp<V>(a.Bt + k * a.ld, i, nk, pk);
                    v[k] = vdot(nk, ax[u], v[k]);
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < MC; ++k) v[k] = vdot(col[u][k], ax[u], v[k]);
        }
    }
}

template <int MC, int U, class V>
__device__ __forceinline__ void u2_trip(const ProjArgs &a, int64_t i0, int64_t stride, int64_t nv, int deff,
                                        const double *c1, double (&v)[MC + 1]) {
    V col[U][MC], ax[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * stride;
        const bool ok = i < nv;
        ax[u] = ok ? ldro<V>(a.Ax, i) : vzero(V());
#pragma unroll
        for (int k = 0; k < MC; ++k) col[u][k] = (ok && k < deff) ? ldro<V>(a.Bt + k * a.ld, i) : vzero(V());
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        V b1 = ax[u];
#pragma unroll
        for (int k = 0; k < MC; ++k) b1 = vaxpy(-c1[k], col[u][k], b1);
#pragma unroll
        for (int k = 0; k < MC; ++k) v[k] = vdot(col[u][k], b1, v[k]);
        v[MC] = vdot(b1, b1, v[MC]);
    }
}

// Per-column coefficient access: registers for MC <= 8, shared memory (re-read at each use) for
// larger buckets.  Fills `reg` from `smem` when registers are used and returns the pointer type
// the trip functions index.
template <int MC> struct Coef {
    static constexpr bool SMEM = MC > 8;
    typedef typename std::conditional<SMEM, const volatile double *, const double *>::type P;
    double reg[SMEM ? 1 : MC];
    __device__ __forceinline__ P bind(const double *smem) {
        if constexpr (SMEM) {
            return (P)smem;
        } else {
#pragma unroll
            for (int k = 0; k < MC; ++k) reg[k] = smem[k];
            return (P)reg;
        }
    }
};

// Per-bucket tuning of the fused kernels (elements per trip = bytes in flight per thread; the
// M = 8 entries were A/B-measured on the C2 bench):
//   FORM_P1  form pass 1 (alpha = B~^T b)        M=8: 2 -> 208.1, 3 -> 207.8, 4 -> 208.0 us/step
//   FORM_P2  form pass 2 (x0 = X~ alpha)         M=8: 2x2 prefetched 207.4, 3x1 207.2, 4x1 207.8
//   FORM_PF  form pass-2 trips prefetched across the grid barrier
//   U        update pass 1 (B~ rotation + c1)    M=8: 2 -> 208.5, 3 -> 210.7
//   U2       update pass 2 (mostly L2 hits)      M=8: 1 -> 214.2, 2 -> 208.5, 3 -> 209.1
//   U3       update pass 3 (X~ pass, 2d+2 streams)
// Elements per trip by bucket for MC <= 4 (U: update pass 1, U2: pass 2, U3: pass 3, P1/P2: form
// passes): few streams need more rows per trip for enough bytes in flight (A/B at N = 2^27:
// QR(1) 1.028 -> 1.094, QR(2) 0.967 -> 1.047, QR(4) 1.040 -> 1.052 of the copy roofline; N = 1e7:
// QR(2) 0.923 -> 0.995).  Experiment builds override single entries with -DIG_T_<FIELD>_<MC>=v
// (scripts/build_variants.py); the default build uses these values.
#define IG_T(F, MC, V) (MC == 1 ? IG_T_##F##_1 : MC == 2 ? IG_T_##F##_2 : MC == 4 ? IG_T_##F##_4 : V)
#ifndef IG_T_U_1
#define IG_T_U_1 8
#endif
#ifndef IG_T_U_2
#define IG_T_U_2 6
#endif
#ifndef IG_T_U_4
#define IG_T_U_4 4
#endif
#ifndef IG_T_U2_1
#define IG_T_U2_1 4
#endif
#ifndef IG_T_U2_2
#define IG_T_U2_2 8
#endif
#ifndef IG_T_U2_4
#define IG_T_U2_4 6
#endif
#ifndef IG_T_U3_1
#define IG_T_U3_1 6
#endif
#ifndef IG_T_U3_2
#define IG_T_U3_2 4
#endif
#ifndef IG_T_U3_4
#define IG_T_U3_4 2
#endif
#ifndef IG_T_P1_1
#define IG_T_P1_1 8
#endif
#ifndef IG_T_P1_2
#define IG_T_P1_2 6
#endif
#ifndef IG_T_P1_4
#define IG_T_P1_4 4
#endif
#ifndef IG_T_P2_1
#define IG_T_P2_1 8
#endif
#ifndef IG_T_P2_2
#define IG_T_P2_2 8
#endif
#ifndef IG_T_P2_4
#define IG_T_P2_4 6
#endif
// Buckets above IG_SMEM_COEF_MIN read the per-column coefficients from shared memory; up to it they
// live in registers (A/B, profiles/r3_roll_ab.md: registers for MC = 10/12 2^27 QR(9) 0.934 ->
// 0.950, QR(12) 0.962 -> 0.988, bitwise-identical; for MC = 14 they spill and run 2-3 % slower).
#ifndef IG_SMEM_COEF_MIN
#define IG_SMEM_COEF_MIN 12
#endif
template <int MC> struct FusedUnroll {
    static constexpr int U = IG_T(U, MC, (MC <= 8 ? 2 : 1));
    static constexpr int U3 = IG_T(U3, MC, 1);
    static constexpr int U2 = IG_T(U2, MC, (MC <= 8 ? 2 : 1));
    static constexpr int FORM_P1 = IG_T(P1, MC, ((MC > 4 && MC <= 8) ? 3 : 1));
    static constexpr int FORM_P2 = IG_T(P2, MC, ((MC > 4 && MC <= 8) ? 3 : 1));
    static constexpr int FORM_PF = (MC > 4 && MC <= 8) ? 1 : (MC < 8 ? 2 : 1);
    // For MC > IG_SMEM_COEF_MIN the per-column coefficients (c1, c2, Givens c/s) are read from shared memory
    // at each use instead of living in 4*MC registers, which the column loads need.
    static constexpr bool SMEM_COEF = MC > IG_SMEM_COEF_MIN;
};

// ------------------------------------------------------------------ trip = loads, then arithmetic
// The first trip of the pass AFTER a grid barrier is loaded BEFORE the barrier (the addresses do
// not depend on the reduction; each thread only reads rows it wrote itself in earlier passes), so
// the barrier + all-CTA reduction bubble overlaps useful HBM traffic.

template <int MC, int U, class V> struct XTrip {  // form pass 2: U strided elements of d X~ columns
    V col[U][MC];
};
template <int MC, int U, class V>
__device__ __forceinline__ void xtrip_load(XTrip<MC, U, V> &r, const ProjArgs &a, int64_t i0, int64_t stride,
                                           int64_t nv, int d, unsigned long long ps) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * stride;
#pragma unroll
        for (int k = 0; k < MC; ++k) r.col[u][k] = (i < nv && k < d) ? ldp<V>(a.Xt + k * a.ld, i, ps) : vzero(V());
    }
}
template <int MC, int U, class V>
__device__ __forceinline__ void xtrip_store(const XTrip<MC, U, V> &r, const ProjArgs &a, int64_t i0, int64_t stride,
                                            int64_t nv, const double *al) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * stride;
        V acc = vzero(V());
#pragma unroll
        for (int k = 0; k < MC; ++k) acc = vaxpy(al[k], r.col[u][k], acc);
        if (i < nv) stv<V>(a.x0, i, acc);
    }
}

template <int MC, int U, class V> struct U2Trip {  // update pass 2
    V ax[U];
    V col[U][MC];
};
template <int MC, int U, class V>
__device__ __forceinline__ void u2trip_load(U2Trip<MC, U, V> &r, const ProjArgs &a, int64_t i0, int64_t stride,
                                            int64_t nv, int deff, unsigned long long pk) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * stride;
        const bool ok = i < nv;
        r.ax[u] = ok ? ldp<V>(a.Ax, i, pk) : vzero(V());
#pragma unroll
        for (int k = 0; k < MC; ++k) r.col[u][k] = (ok && k < deff) ? ldp<V>(a.Bt + k * a.ld, i, pk) : vzero(V());
    }
}
template <int MC, int U, class V, class CP>
__device__ __forceinline__ void u2trip_compute(const U2Trip<MC, U, V> &r, CP c1, double (&v)[MC + 1]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        V b1 = r.ax[u];  // b1 = Ax - B~ c1 (registers only)
#pragma unroll
        for (int k = 0; k < MC; ++k) b1 = vaxpy(-c1[k], r.col[u][k], b1);
#pragma unroll
        for (int k = 0; k < MC; ++k) v[k] = vdot(r.col[u][k], b1, v[k]);
        v[MC] = vdot(b1, b1, v[MC]);
    }
}

// Rolling prefetch for the one-element-per-trip passes 1 and 2 of the large buckets (RollTrip =
// the U2Trip<MC, 1, V> layout: Ax and the B~ columns of one element): the next trip's load of a
// column is issued as soon as this trip has consumed that column, so about one trip of 16-byte
// loads stays in flight per thread through the arithmetic -- the loads of a warp no longer come
// in bursts separated by its compute, and the SM's bytes in flight stop depending on whether its
// eight warps happen to run in phase.  Same rows, same per-thread accumulation order as
// u1_trip / u2trip_compute (bitwise-identical sums).
// Column addresses of the next element advance by one running pointer (one add per column): with
// 32 columns, base + k*ld per column made ptxas keep 32 hoisted 64-bit column pointers live.
template <int MC, bool pend, class V, class CP>
__device__ __forceinline__ void u1_roll(U2Trip<MC, 1, V> &r, const ProjArgs &a, int64_t i, int64_t inext, bool okn,
                                        int nload, CP gc, CP gs, double (&v)[MC + 1], unsigned long long pk) {
    const V ax = r.ax[0];
    r.ax[0] = okn ? ldp<V>(a.Ax, inext, pk) : vzero(V());
    v[MC] = vdot(ax, ax, v[MC]);
    const double *pn = a.Bt + inext * (int64_t)(sizeof(V) / sizeof(double));  // column 0, next element
    double *ps = a.Bt + i * (int64_t)(sizeof(V) / sizeof(double));            // column 0, this element
    if constexpr (pend) {
        V t = r.col[0][0];
        r.col[0][0] = (okn && 0 < nload) ? ldp<V>(pn, 0, pk) : vzero(V());
#pragma unroll
        for (int k = 0; k < MC - 1; ++k) {
            if (k < a.M - 1) {
                V nk;
                pn += a.ld;
                vrot(gc[k], gs[k], t, r.col[0][k + 1], nk);
                r.col[0][k + 1] = (okn && k + 1 < nload) ? ldp<V>(pn, 0, pk) : vzero(V());
                stp<V>(ps, 0, nk, pk);
                ps += a.ld;
                v[k] = vdot(nk, ax, v[k]);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < MC; ++k) {
            v[k] = vdot(r.col[0][k], ax, v[k]);
            r.col[0][k] = (okn && k < nload) ? ldp<V>(pn, 0, pk) : vzero(V());
            pn += a.ld;
        }
    }
}
template <int MC, class V, class CP>
__device__ __forceinline__ void u2_roll(U2Trip<MC, 1, V> &r, const ProjArgs &a, int64_t inext, bool okn, int deff,
                                        CP c1, double (&v)[MC + 1], unsigned long long pk) {
    V b1 = r.ax[0];  // b1 = Ax - B~ c1 (registers only)
    r.ax[0] = okn ? ldp<V>(a.Ax, inext, pk) : vzero(V());
#pragma unroll
    for (int k = 0; k < MC; ++k) b1 = vaxpy(-c1[k], r.col[0][k], b1);
    const double *pn = a.Bt + inext * (int64_t)(sizeof(V) / sizeof(double));
#pragma unroll
    for (int k = 0; k < MC; ++k) {
        v[k] = vdot(r.col[0][k], b1, v[k]);
        r.col[0][k] = (okn && k < deff) ? ldp<V>(pn, 0, pk) : vzero(V());
        pn += a.ld;
    }
    v[MC] = vdot(b1, b1, v[MC]);
}

// For MC > 16 (SPLIT) a trip holds only Ax, x and the B~ columns; the X~ columns are loaded
// (all at once) after the B~ part is finished, so the two 32-column register sets are never live
// together and the pass can use 16-byte loads (VEC = 2) within the register file.
template <int MC, int U, class V> struct U3Trip {  // update pass 3: U strided elements
    static constexpr bool SPLIT = MC > 16;
    V ax[U], xv[U];
    V bc[U][MC];
    V xc[U][SPLIT ? 1 : MC];
};
template <int MC, class V>
__device__ __forceinline__ void u3_load_x(V (&xc)[MC], const ProjArgs &a, int64_t i, bool ok, int nX,
                                          unsigned long long ps) {
#pragma unroll
    for (int k = 0; k < MC; ++k) xc[k] = (ok && k < nX) ? ldp<V>(a.Xt + k * a.ld, i, ps) : vzero(V());
}
// Loads assume the pair is admitted (the common case); if it is not, the prefetched B~/Ax/x
// values of that one trip are simply unused.
template <int MC, int U, class V>
__device__ __forceinline__ void u3trip_load(U3Trip<MC, U, V> &r, const ProjArgs &a, int64_t i0, int64_t stride,
                                            int64_t nv, int deff, bool rotX, bool adm, unsigned long long ps) {
    const int nB = adm ? deff : 0;
    const int nX = rotX ? a.M : nB;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * stride;
        const bool ok = i < nv;
        r.ax[u] = (ok && adm) ? ldp<V>(a.Ax, i, ps) : vzero(V());
        r.xv[u] = (ok && adm) ? ldp<V>(a.x, i, ps) : vzero(V());
#pragma unroll
        for (int k = 0; k < MC; ++k) r.bc[u][k] = (ok && k < nB) ? ldp<V>(a.Bt + k * a.ld, i, ps) : vzero(V());
        if constexpr (!U3Trip<MC, U, V>::SPLIT) u3_load_x<MC, V>(r.xc[u], a, i, ok, nX, ps);
    }
}
template <int MC, class V, class CP>
__device__ __forceinline__ void u3_x_part(const V (&xc)[MC], const ProjArgs &a, int64_t i, bool rotX, V &xt, V &t2,
                                          CP c1, CP c2, CP gc, CP gs, unsigned long long ps) {
    if (rotX) {
        V t = xc[0];
#pragma unroll
        for (int k = 0; k < MC - 1; ++k) {
            if (k < a.M - 1) {
                V nk;
                vrot(gc[k], gs[k], t, xc[k + 1], nk);
                stp<V>(a.Xt + k * a.ld, i, nk, ps);
                xt = vaxpy(-c1[k], nk, xt);
                t2 = vaxpy(c2[k], nk, t2);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < MC; ++k) {
            xt = vaxpy(-c1[k], xc[k], xt);
            t2 = vaxpy(c2[k], xc[k], t2);
        }
    }
}
template <int MC, int U, class V, class CP>
__device__ __forceinline__ void u3trip_store(const U3Trip<MC, U, V> &r, const ProjArgs &a, int64_t i0,
                                             int64_t stride, int64_t nv, int deff, bool rotX, bool adm, double inv,
                                             CP c1, CP c2, CP gc, CP gs, unsigned long long ps) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * stride;
        if (i >= nv) break;
        // b~ = (Ax - B~ c1) - B~ c2 ; x~ = (x - X~ c1) - X~ c2 (separate corrections, DESIGN.md AMB-7)
        V b1 = r.ax[u], s2 = vzero(V());
#pragma unroll
        for (int k = 0; k < MC; ++k) b1 = vaxpy(-c1[k], r.bc[u][k], b1);
#pragma unroll
        for (int k = 0; k < MC; ++k) s2 = vaxpy(c2[k], r.bc[u][k], s2);
        if (adm) stp<V>(a.Bt + deff * a.ld, i, vscale(inv, vaxpy(-1.0, s2, b1)), ps);
        V xt = r.xv[u], t2 = vzero(V());
        if constexpr (U3Trip<MC, U, V>::SPLIT) {
            V xc[MC];
            u3_load_x<MC, V>(xc, a, i, true, rotX ? a.M : (adm ? deff : 0), ps);
            u3_x_part<MC, V>(xc, a, i, rotX, xt, t2, c1, c2, gc, gs, ps);
        } else {
            u3_x_part<MC, V>(r.xc[u], a, i, rotX, xt, t2, c1, c2, gc, gs, ps);
        }
        if (adm) stp<V>(a.Xt + deff * a.ld, i, vscale(inv, vaxpy(-1.0, t2, xt)), ps);
    }
}

// Pass 3 with rolling register sets (one element per trip, the one-copy kernels, buckets whose
// B~ and X~ columns fit in registers together): slot k of the B~ set is consumed by the two
// Gram-Schmidt sums of element i and then receives B~ column k of the NEXT element; slot k of
// the X~ set is consumed by the X~ part (rotation / combine) and receives X~ column k of the next
// element.  Every load is issued a whole element ahead of its use, so about 2M 16-byte loads per
// thread stay in flight through the arithmetic (the unrolled form issues them in one burst after
// the element's stores and then waits).  Same expressions in the same order as u3trip_store
// (bitwise-identical results).  (A single rolling set -- X~ of element i loaded into the B~
// slots right after the sums -- waits a full memory latency per element: 1.3-1.4x slower.)
template <int MC, class V> struct R3 {
    V ax, xv;
    V bs[MC], xs[MC];
};
template <int MC, class V>
__device__ __forceinline__ void r3_load(R3<MC, V> &r, const ProjArgs &a, int64_t i, bool ok, int deff, bool rotX,
                                        bool adm, unsigned long long ps) {
    const int nB = adm ? deff : 0;
    const int nX = rotX ? a.M : nB;
    r.ax = (ok && adm) ? ldp<V>(a.Ax, i, ps) : vzero(V());
    r.xv = (ok && adm) ? ldp<V>(a.x, i, ps) : vzero(V());
    const double *pb = a.Bt + i * (int64_t)(sizeof(V) / sizeof(double));
    const double *px = a.Xt + i * (int64_t)(sizeof(V) / sizeof(double));
#pragma unroll
    for (int k = 0; k < MC; ++k) {
        r.bs[k] = (ok && k < nB) ? ldp<V>(pb, 0, ps) : vzero(V());
        r.xs[k] = (ok && k < nX) ? ldp<V>(px, 0, ps) : vzero(V());
        pb += a.ld;
        px += a.ld;
    }
}
// Element i (valid iff ok) from r; loads element inext (iff okn) into r on the way.
template <int MC, class V, class CP>
__device__ __forceinline__ void u3_roll(R3<MC, V> &r, const ProjArgs &a, int64_t i, bool ok, int64_t inext, bool okn,
                                        int deff, bool rotX, bool adm, double inv, CP c1, CP c2, CP gc, CP gs,
                                        unsigned long long ps) {
    constexpr int64_t W = sizeof(V) / sizeof(double);
    const int nB = adm ? deff : 0;
    const int nX = rotX ? a.M : nB;
    // b~ = (Ax - B~ c1) - B~ c2 ; x~ = (x - X~ c1) - X~ c2 (separate corrections, DESIGN.md AMB-7)
    V b1 = r.ax, s2 = vzero(V());
    r.ax = (okn && adm) ? ldp<V>(a.Ax, inext, ps) : vzero(V());
#pragma unroll
    for (int k = 0; k < MC; ++k) b1 = vaxpy(-c1[k], r.bs[k], b1);
    const double *pb = a.Bt + inext * W;
#pragma unroll
    for (int k = 0; k < MC; ++k) {
        s2 = vaxpy(c2[k], r.bs[k], s2);
        r.bs[k] = (okn && k < nB) ? ldp<V>(pb, 0, ps) : vzero(V());
        pb += a.ld;
    }
    if (adm && ok) stp<V>(a.Bt + deff * a.ld, i, vscale(inv, vaxpy(-1.0, s2, b1)), ps);
    V xt = r.xv, t2 = vzero(V());
    r.xv = (okn && adm) ? ldp<V>(a.x, inext, ps) : vzero(V());
    const double *pn = a.Xt + inext * W;
    if (rotX) {
        double *pxs = a.Xt + i * W;
        V t = r.xs[0];
        r.xs[0] = (okn && 0 < nX) ? ldp<V>(pn, 0, ps) : vzero(V());
#pragma unroll
        for (int k = 0; k < MC - 1; ++k) {
            if (k < a.M - 1) {
                V nk;
                pn += a.ld;
                vrot(gc[k], gs[k], t, r.xs[k + 1], nk);
                r.xs[k + 1] = (okn && k + 1 < nX) ? ldp<V>(pn, 0, ps) : vzero(V());
                if (ok) stp<V>(pxs, 0, nk, ps);
                pxs += a.ld;
                xt = vaxpy(-c1[k], nk, xt);
                t2 = vaxpy(c2[k], nk, t2);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < MC; ++k) {
            xt = vaxpy(-c1[k], r.xs[k], xt);
            t2 = vaxpy(c2[k], r.xs[k], t2);
            r.xs[k] = (okn && k < nX) ? ldp<V>(pn, 0, ps) : vzero(V());
            pn += a.ld;
        }
    }
    if (adm && ok) stp<V>(a.Xt + deff * a.ld, i, vscale(inv, vaxpy(-1.0, t2, xt)), ps);
}

// Givens plan of the next downdate (AMB-2 reading of P:279-290): H = R_{:,2:M} (upper
// Hessenberg, H_ij = R_{i,j+1}); rotation i = 0..M-2 takes a = H_ii (after rotations < i),
// b = H_{i+1,i} = R_{i+1,i+1}, r = hypot(a, b), c = a/r, s = b/r and rotates rows (i, i+1) of H;
// row i of the downdated R is final after rotation i.  One warp; lane j owns H column j (its
// entry of the row carried down in `t`, the rows below in W[i*32 + j], shared).
// Rotation i reads only H columns <= i, i.e. R columns <= i+1, so rotations 0..M-3 need R columns
// 0..M-2 only -- which an update does not change: the column it may add (R column M-1 = H column
// M-2) enters the last rotation alone.  The plan is therefore split:
//   plan_prefix: rotations 0..M-3 on H columns 0..M-3 (lanes j <= M-3): Rdn columns 0..M-3 and
//                (c_i, s_i), i <= M-3 -- computable before the update's sums are known;
//   plan_suffix: H column M-2 through rotations 0..M-3, then rotation M-2 (Rdn column M-2, the zero
//                fill of the leading block, (c, s) of M-2).
// R: the R the downdate acts on (leading M x M block, column-major, stride MAXM; shared or global);
// Rdn: global; pgc/pgs: shared; W: shared [MAXM*32].  Explicit fma() pins the rounding, so the
// split and the one-piece plan (givens_plan) give bitwise-identical results.  The loops stay rolled:
// this code runs once per call, cold in the instruction cache.
static __device__ __noinline__ void plan_prefix(int M, const double *R, double *W, double *pgc, double *pgs,
                                                double *Rdn) {
    const int j = threadIdx.x & 31;
#pragma unroll 1
    for (int i = 0; i < M; ++i) W[i * 32 + j] = (j < M - 2) ? R[i + (j + 1) * MAXM] : 0.0;  // H_ij, j <= M-3
    __syncwarp();
    double t = W[j];
#pragma unroll 1
    for (int i = 0; i < M - 2; ++i) {
        const double aa = __shfl_sync(0xffffffffu, t, i);
        const double bb = R[(i + 1) + (i + 1) * MAXM];
        const double r = hypot(aa, bb);
        const double cs = (r == 0.0) ? 1.0 : aa / r;
        const double sn = (r == 0.0) ? 0.0 : bb / r;
        if (j == i) {
            pgc[i] = cs;
            pgs[i] = sn;
        }
        if (j >= i && j < M - 2) {
            const double hi1 = W[(i + 1) * 32 + j];
            Rdn[i + j * MAXM] = fma(cs, t, sn * hi1);
            t = fma(cs, hi1, -(sn * t));
        }
    }
    __syncwarp();
}
static __device__ __noinline__ void plan_suffix(int M, const double *R, double *W, double *pgc, double *pgs,
                                                double *Rdn) {
    const int j = threadIdx.x & 31;
    if (M >= 2) {
        if (j < M) W[j * 32 + (M - 2)] = R[j + (M - 1) * MAXM];  // H column M-2 = R column M-1
        __syncwarp();
        if (j == M - 2) {
            double t = W[M - 2];
#pragma unroll 1
            for (int i = 0; i < M - 2; ++i) {
                const double cs = pgc[i], sn = pgs[i], hi1 = W[(i + 1) * 32 + j];
                Rdn[i + j * MAXM] = fma(cs, t, sn * hi1);
                t = fma(cs, hi1, -(sn * t));
            }
            const int i = M - 2;
            const double bb = R[(i + 1) + (i + 1) * MAXM];
            const double r = hypot(t, bb);
            const double cs = (r == 0.0) ? 1.0 : t / r;
            const double sn = (r == 0.0) ? 0.0 : bb / r;
            pgc[i] = cs;
            pgs[i] = sn;
            Rdn[i + j * MAXM] = fma(cs, t, sn * W[(i + 1) * 32 + j]);
        }
    }
    if (j < M)  // the rest of the leading block of the downdated R is zero
#pragma unroll 1
        for (int i = 0; i < M; ++i)
            if (!(i < M - 1 && j < M - 1 && i <= j)) Rdn[i + j * MAXM] = 0.0;
    __syncwarp();
}
// Publish the plan: (c_i, s_i) for the next update's B~/X~ rotations, pending downdate.
static __device__ __forceinline__ void plan_publish(Ctrl *c, int M, const double *pgc, const double *pgs) {
    const int j = threadIdx.x & 31;
    if (j < M - 1) {
        c->gc[j] = pgc[j];
        c->gs[j] = pgs[j];
    }
    __syncwarp();
    if (j == 0) c->pending = 1;
}
// One-piece plan (split schedule, single-CTA grids): prefix + suffix + publish.
static __device__ __noinline__ void givens_plan(Ctrl *c, int M, const double *R, double *W, double *pgc,
                                                double *pgs) {
    plan_prefix(M, R, W, pgc, pgs, c->Rdn);
    plan_suffix(M, R, W, pgc, pgs, c->Rdn);
    plan_publish(c, M, pgc, pgs);
}

// One warp: R after this update, in place in sR (which holds the R it started from: the downdated
// R if a downdate ran, else R) -- plus, if the pair was admitted, the new column (c1 + c2; ||b~||)
// (Alg. 2) -- and to c->R.
static __device__ __noinline__ void r_update(Ctrl *c, int M, int deff, bool pend, bool newcol, const double *r1,
                                             const double *r2, double nb, double *sR) {
    const int lane = threadIdx.x & 31;
#pragma unroll 1
    for (int idx = lane; idx < M * M; idx += 32) {
        const int i = idx % M, j = idx / M;
        double v = sR[i + j * MAXM];
        if (newcol && j == deff) v = (i < deff) ? r1[i] + r2[i] : (i == deff ? nb : 0.0);
        sR[i + j * MAXM] = v;
        if (pend || (newcol && j == deff)) c->R[i + j * MAXM] = v;
    }
    if (newcol)
        for (int k = M + lane; k < MAXM; k += 32) c->R[k + deff * MAXM] = 0.0;
    __syncwarp();  // sR complete
}

}  // namespace ig
