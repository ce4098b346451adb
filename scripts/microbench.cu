// microbench.cu -- B200 streaming ceilings for the initial-guess access patterns (K read streams of
// fp64, one reduction or one write stream).  Not part of the library; used to size the kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int K, int U>
__global__ void __launch_bounds__(256, 1) rd_ldg(const double *__restrict__ base, int64_t ld, int64_t nv, double *out) {
    double acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += U * stride) {
        double2 c[U][K];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < K; ++k) {
                int64_t i = i0 + u * stride;
                c[u][k] = i < nv ? __ldg(reinterpret_cast<const double2 *>(base + k * ld) + i) : make_double2(0, 0);
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < K; ++k) acc += c[u][k].x * (k + 1) + c[u][k].y;
    }
    if (acc == 1234.5) out[0] = acc;
}

template <int K, int U>
__global__ void __launch_bounds__(256, 1) comb_ldg(const double *__restrict__ base, int64_t ld, int64_t nv, double *out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += U * stride) {
        double2 c[U][K];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < K; ++k) {
                int64_t i = i0 + u * stride;
                c[u][k] = i < nv ? __ldg(reinterpret_cast<const double2 *>(base + k * ld) + i) : make_double2(0, 0);
            }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double2 a = make_double2(0, 0);
#pragma unroll
            for (int k = 0; k < K; ++k) { a.x += c[u][k].x * (k + 1); a.y += c[u][k].y * (k + 1); }
            int64_t i = i0 + u * stride;
            if (i < nv) reinterpret_cast<double2 *>(out)[i] = a;
        }
    }
}

// TMA-style 1D bulk copies into a multi-stage shared-memory ring, one producer thread.
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(b)),
        "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}

template <int K, int TILE, int STAGES>
__global__ void __launch_bounds__(256, 1) rd_tma(const double *__restrict__ base, int64_t ld, int64_t n, double *out) {
    extern __shared__ __align__(128) double smem[];  // [STAGES][K][TILE]
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    const int nw = blockDim.x / 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nw); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t ntiles = n / TILE;
    double acc = 0;
    // tiles t = blockIdx.x + j*gridDim.x
    int64_t jmax = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    if (threadIdx.x == 0) {
        for (int64_t j = 0; j < jmax && j < STAGES; ++j) {
            int s = j % STAGES;
            mbar_expect_tx(&full[s], K * TILE * 8);
            int64_t t = blockIdx.x + j * gridDim.x;
            for (int k = 0; k < K; ++k) bulk_g2s(smem + (s * K + k) * TILE, base + k * ld + t * TILE, TILE * 8, &full[s]);
        }
    }
    for (int64_t j = 0; j < jmax; ++j) {
        int s = j % STAGES;
        unsigned ph = (j / STAGES) & 1;
        mbar_wait(&full[s], ph);
        const double *tl = smem + s * K * TILE;
        for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
#pragma unroll
            for (int k = 0; k < K; ++k) acc += tl[k * TILE + e] * (k + 1);
        }
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
        if (threadIdx.x == 0 && j + STAGES < jmax) {
            mbar_wait(&empty[s], ph);
            mbar_expect_tx(&full[s], K * TILE * 8);
            int64_t t = blockIdx.x + (j + STAGES) * gridDim.x;
            for (int k = 0; k < K; ++k) bulk_g2s(smem + (s * K + k) * TILE, base + k * ld + t * TILE, TILE * 8, &full[s]);
        }
    }
    if (acc == 1234.5) out[0] = acc;
}

__global__ void copyk(const double2 *__restrict__ a, double2 *__restrict__ b, int64_t nv) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) b[i] = a[i];
}

template <class F> float timeit(F f, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main(int argc, char **argv) {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    std::vector<int64_t> sizes = {1 << 21, 1 << 24};
    const int K = 9;
    double *buf, *out;
    int64_t nmax = 1 << 24;
    CK(cudaMalloc(&buf, sizeof(double) * nmax * (K + 1)));
    CK(cudaMalloc(&out, sizeof(double) * nmax));
    CK(cudaMemset(buf, 0, sizeof(double) * nmax * (K + 1)));
    // flush buffer
    double *flush;
    CK(cudaMalloc(&flush, 512 << 20));
    for (int64_t n : sizes) {
        int64_t ld = nmax;
        double rbytes = 8.0 * K * n;
        printf("== n = %lld doubles per stream, %d streams (%.0f MB read)\n", (long long)n, K, rbytes / 1e6);
        auto flushf = [&] { cudaMemsetAsync(flush, 1, 512 << 20); };
        for (int bps : {1, 2, 4}) {
            int g = nsm * bps;
            float ms = timeit([&] { flushf(); rd_ldg<K, 1><<<g, 256>>>(buf, ld, n / 2, out); }, 10);
            float msf = timeit([&] { flushf(); }, 10);
            printf("rd_ldg U1 grid %d: %.1f us  %.0f GB/s\n", g, (ms - msf) * 1e3, rbytes / ((ms - msf) * 1e-3) / 1e9);
            ms = timeit([&] { flushf(); rd_ldg<K, 2><<<g, 256>>>(buf, ld, n / 2, out); }, 10);
            printf("rd_ldg U2 grid %d: %.1f us  %.0f GB/s\n", g, (ms - msf) * 1e3, rbytes / ((ms - msf) * 1e-3) / 1e9);
            ms = timeit([&] { flushf(); comb_ldg<K - 1, 1><<<g, 256>>>(buf, ld, n / 2, out); }, 10);
            printf("comb_ldg(8->1) U1 grid %d: %.1f us  %.0f GB/s\n", g, (ms - msf) * 1e3, rbytes / ((ms - msf) * 1e-3) / 1e9);
        }
        {
            constexpr int TILE = 512, ST = 4;
            size_t sm = sizeof(double) * K * TILE * ST;
            cudaFuncSetAttribute(rd_tma<K, TILE, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            float msf = timeit([&] { flushf(); }, 10);
            float ms = timeit([&] { flushf(); rd_tma<K, TILE, ST><<<nsm, 256, sm>>>(buf, ld, n, out); }, 10);
            printf("rd_tma tile %d stages %d grid %d: %.1f us  %.0f GB/s  (err %s)\n", TILE, ST, nsm, (ms - msf) * 1e3,
                   rbytes / ((ms - msf) * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
        {
            constexpr int TILE = 256, ST = 8;
            size_t sm = sizeof(double) * K * TILE * ST;
            cudaFuncSetAttribute(rd_tma<K, TILE, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            float msf = timeit([&] { flushf(); }, 10);
            float ms = timeit([&] { flushf(); rd_tma<K, TILE, ST><<<nsm, 256, sm>>>(buf, ld, n, out); }, 10);
            printf("rd_tma tile %d stages %d grid %d: %.1f us  %.0f GB/s  (err %s)\n", TILE, ST, nsm, (ms - msf) * 1e3,
                   rbytes / ((ms - msf) * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
        {
            float msf = timeit([&] { flushf(); }, 10);
            int64_t nc = n * K / 2;  // same bytes moved: K/2 vectors read + written
            float ms = timeit([&] { flushf(); copyk<<<nsm * 8, 256>>>((const double2 *)buf, (double2 *)(buf + nc), nc / 2); }, 10);
            printf("copy %.0f MB: %.1f us  %.0f GB/s (read+write)\n", 16.0 * nc / 1e6, (ms - msf) * 1e3, 16.0 * nc / ((ms - msf) * 1e-3) / 1e9);
        }
    }
    return 0;
}
