// Feasibility probe: device-driven scheduling loop as a CUDA graph with a
// conditional WHILE node whose body is [scheduler kernel -> SWITCH node over
// three event kernels]. Compares the per-iteration cost with the host-driven
// loop (launch + D2H + sync) and CDP2 tail launches (cdp_test.cu).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void child(int* c, int n, const int* dn) {
    // grid-stride over a device-resident length (graph kernels have fixed grids)
    int len = *dn;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x)
        if ((i & 1023) == 0) atomicAdd(c, n);
}
__global__ void sched(int* iters, int max_it, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hs) {
    int it = *iters;
    *iters = it + 1;
    cudaGraphSetConditional(hs, (unsigned)(it % 3));
    cudaGraphSetConditional(hw, it + 1 < max_it ? 1u : 0u);
}

int main() {
    int *c, *it, *dn;
    CK(cudaMalloc(&c, 4)); CK(cudaMalloc(&it, 4)); CK(cudaMalloc(&dn, 4));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    for (int len : {0, 1 << 16, 1 << 20}) {
        for (int grid : {148, 1184}) {
            CK(cudaMemcpy(dn, &len, 4, cudaMemcpyHostToDevice));
            cudaGraph_t g;
            CK(cudaGraphCreate(&g, 0));
            cudaGraphConditionalHandle hw, hs;
            CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
            CK(cudaGraphConditionalHandleCreate(&hs, g, 0, 0));
            cudaGraphNodeParams wp = {};
            wp.type = cudaGraphNodeTypeConditional;
            wp.conditional.handle = hw;
            wp.conditional.type = cudaGraphCondTypeWhile;
            wp.conditional.size = 1;
            cudaGraphNode_t wn;
            CK(cudaGraphAddNode(&wn, g, nullptr, 0, &wp));
            cudaGraph_t body = wp.conditional.phGraph_out[0];
            const int N = 3000;
            void* sa[] = {&it, (void*)&N, &hw, &hs};
            cudaKernelNodeParams kp = {};
            kp.func = (void*)sched; kp.gridDim = dim3(1); kp.blockDim = dim3(1); kp.kernelParams = sa;
            cudaGraphNode_t sn;
            CK(cudaGraphAddKernelNode(&sn, body, nullptr, 0, &kp));
            cudaGraphNodeParams sp = {};
            sp.type = cudaGraphNodeTypeConditional;
            sp.conditional.handle = hs;
            sp.conditional.type = cudaGraphCondTypeSwitch;
            sp.conditional.size = 3;
            cudaGraphNode_t swn;
            CK(cudaGraphAddNode(&swn, body, &sn, 1, &sp));
            int vals[3] = {1, 2, 4};
            for (int k = 0; k < 3; ++k) {
                void* ca[] = {&c, &vals[k], &dn};
                cudaKernelNodeParams cp = {};
                cp.func = (void*)child; cp.gridDim = dim3(grid); cp.blockDim = dim3(128); cp.kernelParams = ca;
                cudaGraphNode_t cn;
                CK(cudaGraphAddKernelNode(&cn, sp.conditional.phGraph_out[k], nullptr, 0, &cp));
            }
            cudaGraphExec_t ge;
            CK(cudaGraphInstantiate(&ge, g, 0));
            for (int rep = 0; rep < 2; ++rep) {
                CK(cudaMemset(c, 0, 4)); CK(cudaMemset(it, 0, 4));
                cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
                cudaEventRecord(a, s);
                CK(cudaGraphLaunch(ge, s));
                cudaEventRecord(b, s);
                CK(cudaEventSynchronize(b));
                float ms; cudaEventElapsedTime(&ms, a, b);
                int hit; cudaMemcpy(&hit, it, 4, cudaMemcpyDeviceToHost);
                if (rep) printf("graph while+switch len %7d grid %4d: iterations %d, %.2f us per iteration (sched + 1 kernel)\n",
                                len, grid, hit, 1000 * ms / hit);
            }
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
        // host-driven reference: 1 launch + D2H + sync per iteration
        int* h; CK(cudaMallocHost(&h, 4));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a, s);
        for (int i = 0; i < 3000; ++i) {
            child<<<1184, 128, 0, s>>>(c, 1, dn);
            cudaMemcpyAsync(h, c, 4, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s);
        }
        cudaEventRecord(b, s); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("host-driven       len %7d grid 1184: %.2f us per iteration (1 kernel + D2H + sync)\n", len, 1000 * ms / 3000);
        cudaEventRecord(a, s);
        for (int i = 0; i < 3000; ++i) child<<<1184, 128, 0, s>>>(c, 1, dn);
        cudaEventRecord(b, s); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("stream back2back  len %7d grid 1184: %.2f us per kernel\n", len, 1000 * ms / 3000);
    }
    return 0;
}
