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
__global__ void __launch_bounds__(THREADS, 1) k_extrap(const __grid_constant__ ExtrapArgs a) {
    // All loads of a trip are issued before the FMAs consume them (see kern_proj.cu); the
    // accumulation order is oldest -> newest, like Eq. EXTRAPEXPN.
    typedef typename std::conditional<VEC == 2, double2, double>::type V;
    pdl_wait();
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
    pdl_trigger();
}

template <int VEC>
__global__ void __launch_bounds__(THREADS, 1) k_copy(double *__restrict__ dst, const double *__restrict__ src, int64_t N) {
    pdl_wait();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (VEC == 2) {
        const int64_t nv = N >> 1;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride)
            reinterpret_cast<double2 *>(dst)[i] = __ldg(reinterpret_cast<const double2 *>(src) + i);
        if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) dst[N - 1] = src[N - 1];
    } else {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) dst[i] = src[i];
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

template <int FC>
static void launch_fc(const ExtrapArgs &a, int vec, int nsm, cudaStream_t s) {
    if (vec == 2) {
        constexpr int U = FC <= 2 ? 4 : (FC <= 4 ? 2 : 1);
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

cudaError_t launch_copy(double *dst, const double *src, int64_t N, int vec, int nsm, cudaStream_t s) {
    if (vec == 2) {
        auto k = k_copy<2>;
        launch_ex(k, grid_for_x(k, N / 2, nsm), s, false, dst, src, N);
    } else {
        auto k = k_copy<1>;
        launch_ex(k, grid_for_x(k, N, nsm), s, false, dst, src, N);
    }
    return cudaGetLastError();
}

}  // namespace ig
