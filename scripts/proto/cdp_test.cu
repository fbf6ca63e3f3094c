// Feasibility probe: device-side scheduling loop with CDP2 tail launches.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void child(int* c, int n) { if (threadIdx.x == 0) atomicAdd(c, n); }
__global__ void sched(int* c, int* iters, int max_it, int grid) {
    int it = atomicAdd(iters, 1);
    if (it < max_it) {
        child<<<grid, 128, 0, cudaStreamTailLaunch>>>(c, 1);
        child<<<grid, 128, 0, cudaStreamTailLaunch>>>(c, 2);
        child<<<grid, 128, 0, cudaStreamTailLaunch>>>(c, 4);
        sched<<<1, 1, 0, cudaStreamTailLaunch>>>(c, iters, max_it, grid);
    }
}
int main() {
    int *c, *it;
    cudaMalloc(&c, 4); cudaMalloc(&it, 4);
    for (int grid : {1, 148, 1000}) {
        cudaMemset(c, 0, 4); cudaMemset(it, 0, 4);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        int N = 2000;
        cudaEventRecord(a);
        sched<<<1, 1>>>(c, it, N, grid);
        cudaEventRecord(b);
        cudaError_t e = cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        int hc; cudaMemcpy(&hc, c, 4, cudaMemcpyDeviceToHost);
        printf("grid %d: %s c=%d (expect %d) %.2f us per iteration (4 launches)\n", grid, cudaGetErrorString(e), hc, N * 7 * grid, 1000 * ms / N);
    }
    // host-driven reference: 3 launches + memcpy + sync per iteration
    {
        cudaStream_t s; cudaStreamCreate(&s);
        int* h; cudaMallocHost(&h, 4);
        auto t0 = clock();
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a, s);
        for (int i = 0; i < 2000; ++i) {
            child<<<148, 128, 0, s>>>(c, 1); child<<<148, 128, 0, s>>>(c, 2); child<<<148, 128, 0, s>>>(c, 4);
            cudaMemcpyAsync(h, c, 4, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s);
        }
        cudaEventRecord(b, s); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("host-driven: %.2f us per iteration (3 launches + D2H + sync)\n", 1000 * ms / 2000);
    }
    return 0;
}
