// kern_extrap.cu -- sm_100a kernels of the extrapolation hot path (arXiv 2009.10863 §3).
//
//   k_extrap  x0 = sum_{i=1}^{f} beta_i x_{n-f+i}   (Eq. EXTRAPEXPN, PAPER.md:335-347;
//             paper kernel extrapKernel).  beta and the f slot pointers (oldest
//             first) travel BY VALUE in the kernel-parameter constant bank: every thread reads
//             them as uniform constants, no global state shared between handles.
//   k_copy    push of a solution that was not solved in place (2 values/element).
// Both are pure streams: (f+1) and 2 fp64 values per element.
#include <type_traits>

#include "ig_internal.h"

namespace ig {

template <int FC, int VEC, int UNROLL>
__device__ __forceinline__ void extrap_body(const ExtrapArgs &a) {
    // All loads of a trip are issued before the FMAs consume them (see kern_proj.cu); the
    // accumulation order is oldest -> newest, like Eq. EXTRAPEXPN.
    typedef typename std::conditional<VEC == 2, double2, double>::type V;
    // (an L2 evict_first hint on these single-use loads measured 8% SLOWER at N = 2^27: not used)
    const int f = a.f;
    const int64_t nv = a.N / VEC;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += UNROLL * stride) {
        V col[UNROLL][FC];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const int64_t i = i0 + u * stride;
#pragma unroll
            for (int j = 0; j < FC; ++j)
                col[u][j] = (i < nv && j < f) ? __ldg(reinterpret_cast<const V *>(a.src[j]) + i) : V{};
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const int64_t i = i0 + u * stride;
            V acc{};
#pragma unroll
            for (int j = 0; j < FC; ++j) {
                if (VEC == 2) {
                    double *pa = reinterpret_cast<double *>(&acc);
                    const double *pc = reinterpret_cast<const double *>(&col[u][j]);
                    pa[0] = fma(a.beta[j], pc[0], pa[0]);
                    pa[1] = fma(a.beta[j], pc[1], pa[1]);
                } else {
                    double *pa = reinterpret_cast<double *>(&acc);
                    pa[0] = fma(a.beta[j], *reinterpret_cast<const double *>(&col[u][j]), pa[0]);
                }
            }
            if (i < nv) reinterpret_cast<V *>(a.x0)[i] = acc;
        }
    }
    if (VEC == 2 && (a.N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t e = a.N - 1;
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < FC; ++j)
            if (j < f) acc = fma(a.beta[j], a.src[j][e], acc);
        a.x0[e] = acc;
    }
}

template <int FC, int VEC, int UNROLL>
__global__ void __launch_bounds__(THREADS, 1) k_extrap(const __grid_constant__ ExtrapArgs a) {
    pdl_wait();
    extrap_body<FC, VEC, UNROLL>(a);
    pdl_trigger();
}

// Multi-field batch (one history space per field): blockIdx.y
// selects the field, so the guesses of up to MAXF fields cost one launch.
template <int FC, int VEC, int UNROLL>
__global__ void __launch_bounds__(THREADS, 1) k_extrap_batch(const __grid_constant__ ExtrapBatch b) {
    pdl_wait();
    extrap_body<FC, VEC, UNROLL>(b.f[blockIdx.y]);
    pdl_trigger();
}

template <int VEC, int U>
__device__ __forceinline__ void copy_body(double *__restrict__ dst, const double *__restrict__ src, int64_t N) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (VEC == 2) {  // U strided 16-byte loads in flight per thread, then the U stores
        const int64_t nv = N >> 1;
        const double2 *s2 = reinterpret_cast<const double2 *>(src);
        double2 *d2 = reinterpret_cast<double2 *>(dst);
        for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += U * stride) {
            double2 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = (i0 + u * stride < nv) ? __ldg(s2 + i0 + u * stride) : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i0 + u * stride < nv) d2[i0 + u * stride] = r[u];
        }
        if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) dst[N - 1] = src[N - 1];
    } else {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) dst[i] = src[i];
    }
}

template <int VEC, int U>
__global__ void __launch_bounds__(THREADS, 1) k_copy(double *__restrict__ dst, const double *__restrict__ src, int64_t N) {
    pdl_wait();
    copy_body<VEC, U>(dst, src, N);
}

// ----------------------------------------------------------------------------- device ring
// Same arithmetic as k_extrap / k_copy; the window (f, slot pointers, weights) is derived on the
// device from the push counter (DevRing), so a captured graph replays correctly at every fill.
template <int FC, int VEC, int UNROLL>
__global__ void __launch_bounds__(THREADS, 1) k_extrap_ring(const __grid_constant__ RingBatch b) {
    pdl_wait();
    __shared__ ExtrapArgs sa;
    const RingArgs &r = b.f[blockIdx.y];
    if (threadIdx.x < 32) {
        const unsigned long long cnt = *reinterpret_cast<volatile unsigned long long *>(&r.ring->cnt);
        const int f = cnt < (unsigned long long)r.M ? (int)cnt : r.M;
        const int nz = f > 0 ? r.tab->nnz[f - 1] : 0;
        const int lane = threadIdx.x;
        if (lane < nz) {
            const int j = r.tab->jidx[f - 1][lane];
            const int64_t slot = (int64_t)((cnt - (unsigned long long)f + (unsigned long long)j) % (unsigned long long)r.M);
            sa.src[lane] = r.base + slot * r.ld;
            sa.beta[lane] = r.tab->beta[f - 1][lane];
        }
        if (lane == 0) {
            sa.f = nz;
            sa.N = r.N;
            sa.x0 = r.x0;
        }
    }
    __syncthreads();
    if (sa.f > 0) extrap_body<FC, VEC, UNROLL>(sa);  // f == 0: x0 untouched (AMB-13)
    pdl_trigger();
}

template <int VEC, int U>
__global__ void __launch_bounds__(THREADS, 1) k_push_ring(const __grid_constant__ RingBatch b) {
    pdl_wait();
    const RingArgs &r = b.f[blockIdx.y];
    __shared__ unsigned long long cnt_s;
    if (threadIdx.x == 0) cnt_s = *reinterpret_cast<volatile unsigned long long *>(&r.ring->cnt);
    __syncthreads();
    const unsigned long long cnt = cnt_s;
    double *dst = r.base + (int64_t)(cnt % (unsigned long long)r.M) * r.ld;
    if (dst != r.x) copy_body<VEC, U>(dst, r.x, r.N);  // solved in place: 0 bytes
    pdl_trigger();
    if (threadIdx.x == 0) {
        // every CTA has read cnt before it takes a ticket: the last one advances the window
        const unsigned t = atomicAdd(&r.ring->ticket, 1u);
        if (t == gridDim.x - 1) {
            r.ring->ticket = 0;
            r.ring->cnt = cnt + 1;
        }
    }
}

template <class K> static int grid_for_x(K kern, int64_t nv, int nsm) {
    int occ = cached_occupancy((const void *)kern);
    if (occ < 1) occ = 1;
    if (occ > 8) occ = 8;
    int64_t want = (nv + THREADS - 1) / THREADS;
    int64_t g = (int64_t)nsm * occ;
    if (want < g) g = want;
    if (g < 1) g = 1;
    return (int)g;
}

// Elements per trip of the combine (bytes in flight per thread), by term bucket; the 8-term value
// was A/B-measured on C2 (1 -> 207.8, 2 -> 207.4 us/step).
template <int FC> struct ExtrapTune {
    static constexpr int U = FC <= 2 ? 4 : (FC <= 4 ? 2 : (FC == 8 ? 2 : 1));
};
template <int FC>
static void launch_fc(const ExtrapArgs &a, int vec, int nsm, cudaStream_t s) {
    if (vec == 2) {
        constexpr int U = ExtrapTune<FC>::U;
        auto k = k_extrap<FC, 2, U>;  // U strided elements per trip when few streams
        launch_ex(k, grid_for_x(k, a.N / 2, nsm), s, false, a);
    } else {
        constexpr int U = FC <= 2 ? 4 : (FC <= 4 ? 2 : 1);
        auto k = k_extrap<FC, 1, U>;
        launch_ex(k, grid_for_x(k, a.N, nsm), s, false, a);
    }
}

cudaError_t launch_extrap(const ExtrapArgs &a, int vec, int nsm, cudaStream_t s) {
    const int f = a.f;
    if (f <= 1) launch_fc<1>(a, vec, nsm, s);
    else if (f <= 2) launch_fc<2>(a, vec, nsm, s);
    else if (f <= 4) launch_fc<4>(a, vec, nsm, s);
    else if (f <= 8) launch_fc<8>(a, vec, nsm, s);
    else if (f <= 16) launch_fc<16>(a, vec, nsm, s);
    else launch_fc<32>(a, vec, nsm, s);
    return cudaGetLastError();
}

template <int FC>
static void launch_fc_batch(const ExtrapBatch &b, int vec, int nsm, cudaStream_t s) {
    int64_t nmax = 0;
    for (int j = 0; j < b.nf; ++j) nmax = b.f[j].N > nmax ? b.f[j].N : nmax;
    constexpr int U = FC <= 2 ? 4 : (FC <= 4 ? 2 : 1);
    const LaunchFlags fl = launch_flags();
    auto go = [&](auto kern, int64_t nv) {
        cudaLaunchConfig_t cfg = {};
        int gx = grid_for_x(kern, nv, nsm);
        gx = (gx + b.nf - 1) / b.nf;  // the fields share the SMs
        cfg.gridDim = dim3(gx < 1 ? 1 : gx, b.nf);
        cfg.blockDim = dim3(THREADS);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = fl.pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, kern, b);
    };
    if (vec == 2) go(k_extrap_batch<FC, 2, U>, nmax / 2);
    else go(k_extrap_batch<FC, 1, U>, nmax);
}

cudaError_t launch_extrap_batch(const ExtrapBatch &b, int vec, int nsm, cudaStream_t s) {
    int f = 0;
    for (int j = 0; j < b.nf; ++j) f = b.f[j].f > f ? b.f[j].f : f;
    if (f <= 1) launch_fc_batch<1>(b, vec, nsm, s);
    else if (f <= 2) launch_fc_batch<2>(b, vec, nsm, s);
    else if (f <= 4) launch_fc_batch<4>(b, vec, nsm, s);
    else if (f <= 8) launch_fc_batch<8>(b, vec, nsm, s);
    else if (f <= 16) launch_fc_batch<16>(b, vec, nsm, s);
    else launch_fc_batch<32>(b, vec, nsm, s);
    return cudaGetLastError();
}

cudaError_t launch_copy(double *dst, const double *src, int64_t N, int vec, int nsm, cudaStream_t s) {
    if (vec == 2) {
        // large vectors: 4 loads in flight per thread (C3: 6.06 -> 6.48 TB/s); short ones: one
        // per thread on a grid 4x wider, which ramps up faster (C2: 7.2 -> 6.8 us per push)
        if (N >= (int64_t(1) << 24)) {
            auto k = k_copy<2, 4>;
            launch_ex(k, grid_for_x(k, N / 2, nsm), s, false, dst, src, N);
        } else {
            auto k = k_copy<2, 1>;
            launch_ex(k, grid_for_x(k, N / 2, nsm), s, false, dst, src, N);
        }
    } else {
        auto k = k_copy<1, 1>;
        launch_ex(k, grid_for_x(k, N, nsm), s, false, dst, src, N);
    }
    return cudaGetLastError();
}

template <class K> static void launch_ring(K kern, const RingBatch &b, int64_t nv, int nsm, cudaStream_t s) {
    const LaunchFlags fl = launch_flags();
    cudaLaunchConfig_t cfg = {};
    int gx = grid_for_x(kern, nv, nsm);
    gx = (gx + b.nf - 1) / b.nf;  // the fields share the SMs
    cfg.gridDim = dim3(gx < 1 ? 1 : gx, b.nf);
    cfg.blockDim = dim3(THREADS);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = fl.pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, b);
}

static int64_t ring_nmax(const RingBatch &b) {
    int64_t nmax = 0;
    for (int j = 0; j < b.nf; ++j) nmax = b.f[j].N > nmax ? b.f[j].N : nmax;
    return nmax;
}

template <int FC>
static void launch_ring_fc(const RingBatch &b, int vec, int nsm, cudaStream_t s) {
    const int64_t nmax = ring_nmax(b);
    if (vec == 2) launch_ring(k_extrap_ring<FC, 2, ExtrapTune<FC>::U>, b, nmax / 2, nsm, s);
    else launch_ring(k_extrap_ring<FC, 1, (FC <= 2 ? 4 : (FC <= 4 ? 2 : 1))>, b, nmax, nsm, s);
}

cudaError_t launch_extrap_ring(const RingBatch &b, int fc, int vec, int nsm, cudaStream_t s) {
    if (fc <= 1) launch_ring_fc<1>(b, vec, nsm, s);
    else if (fc <= 2) launch_ring_fc<2>(b, vec, nsm, s);
    else if (fc <= 4) launch_ring_fc<4>(b, vec, nsm, s);
    else if (fc <= 8) launch_ring_fc<8>(b, vec, nsm, s);
    else if (fc <= 16) launch_ring_fc<16>(b, vec, nsm, s);
    else launch_ring_fc<32>(b, vec, nsm, s);
    return cudaGetLastError();
}

cudaError_t launch_push_ring(const RingBatch &b, int vec, int nsm, cudaStream_t s) {
    const int64_t nmax = ring_nmax(b);
    if (vec == 2) {
        if (nmax >= (int64_t(1) << 24)) launch_ring(k_push_ring<2, 4>, b, nmax / 2, nsm, s);
        else launch_ring(k_push_ring<2, 1>, b, nmax / 2, nsm, s);
    } else {
        launch_ring(k_push_ring<1, 1>, b, nmax, nsm, s);
    }
    return cudaGetLastError();
}

}  // namespace ig
