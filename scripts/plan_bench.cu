// Microbenchmark of the serial Givens plan (proj_common.cuh::givens_plan) on one warp, warm and
// cold, for M = 8, 16, 30: is its cost the math chain or the memory/instruction path?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2009_10863_b200/csrc \
//        scripts/plan_bench.cu -o /tmp/plan_bench && /tmp/plan_bench
#include <cstdio>
#include <vector>

#include "proj_common.cuh"

using namespace ig;

__global__ void plan_kernel(Ctrl *c, int M, int reps, unsigned long long *t) {
    __shared__ double sR[MAXM * MAXM], sW[MAXM * 32];
    for (int i = threadIdx.x; i < MAXM * MAXM; i += blockDim.x) sR[i] = c->R[i];
    __syncwarp();
    for (int r = 0; r < reps; ++r) {
        const unsigned long long t0 = globaltimer_ns();
        givens_plan(c, M, sR, sW);
        __syncwarp();
        const unsigned long long t1 = globaltimer_ns();
        if (threadIdx.x == 0) t[r] = t1 - t0;
    }
}

int main() {
    Ctrl *c;
    unsigned long long *t;
    cudaMalloc(&c, sizeof(Ctrl));
    cudaMalloc(&t, 8 * 16);
    for (int M : {8, 16, 30}) {
        Ctrl h = {};
        for (int j = 0; j < M; ++j)  // a well-conditioned upper-triangular R
            for (int i = 0; i <= j; ++i) h.R[i + j * MAXM] = (i == j) ? 2.0 + j : 0.1 * (i + 1) / (j + 1);
        cudaMemcpy(c, &h, sizeof h, cudaMemcpyHostToDevice);
        plan_kernel<<<1, 32>>>(c, M, 4, t);
        unsigned long long ht[4];
        cudaMemcpy(ht, t, sizeof ht, cudaMemcpyDeviceToHost);
        printf("M = %2d: plan %.2f us (first, cold) then %.2f %.2f %.2f us (warm); %.3f us per rotation warm\n", M,
               ht[0] / 1e3, ht[1] / 1e3, ht[2] / 1e3, ht[3] / 1e3, ht[3] / 1e3 / (M - 1));
    }
    return 0;
}
