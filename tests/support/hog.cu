// Test support only (not part of libig): a "foreign" kernel that holds SMs for a fixed time, as a
// solver kernel, halo exchange or NCCL kernel on another stream would.  Each CTA takes `smem`
// bytes of dynamic shared memory (up to the 227 KB per-CTA maximum, so no other CTA fits beside
// it on its SM) and spins on %globaltimer for `ns` nanoseconds.
#include <cuda_runtime.h>

__global__ void hog_kernel(unsigned long long ns, unsigned long long *started) {
    extern __shared__ char smem[];
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0) {
        smem[0] = 1;
        atomicAdd(started, 1ull);
    }
    unsigned long long t = t0;
    while (t - t0 < ns) {
        __nanosleep(1000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    }
}

extern "C" int hog_launch(int blocks, int smem, unsigned long long ns, unsigned long long *started, void *stream) {
    cudaError_t e = cudaFuncSetAttribute(hog_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return (int)e;
    hog_kernel<<<blocks, 32, smem, (cudaStream_t)stream>>>(ns, started);
    return (int)cudaGetLastError();
}
