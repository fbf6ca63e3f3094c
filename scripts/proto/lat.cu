// Dependent-chain latencies on this GPU (one thread, clock64): fp64 / fp32 / int ops,
// division, sqrt, and global-load latency at L1 / L2 / HBM distance.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double* out, long long* cyc, const int* chase, int nchase) {
    double a = out[0], b = out[1], c = out[2];
    float fa = (float)a, fb = (float)b;
    long long t0, t1;
    const int N = 1024;
    t0 = clock64();
    for (int i = 0; i < N; ++i) a = fma(a, b, c);
    t1 = clock64(); cyc[0] = (t1 - t0); out[3] = a;
    t0 = clock64();
    for (int i = 0; i < N; ++i) a = a + b;
    t1 = clock64(); cyc[1] = (t1 - t0); out[4] = a;
    t0 = clock64();
    for (int i = 0; i < N; ++i) fa = fmaf(fa, fb, 1.0f);
    t1 = clock64(); cyc[2] = (t1 - t0); out[5] = fa;
    t0 = clock64();
    for (int i = 0; i < 256; ++i) a = c / a;
    t1 = clock64(); cyc[3] = (t1 - t0) * 4; out[6] = a;
    t0 = clock64();
    for (int i = 0; i < 256; ++i) a = sqrt(a) + c;
    t1 = clock64(); cyc[4] = (t1 - t0) * 4; out[7] = a;
    int idx = 0;
    // pointer chase: nchase hops
    t0 = clock64();
    for (int i = 0; i < nchase; ++i) idx = chase[idx];
    t1 = clock64(); cyc[5] = (t1 - t0) * N / nchase; out[8] = idx;
    unsigned long long x = (unsigned long long)idx + 1;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = x * 6364136223846793005ULL + 1442695040888963407ULL;
    t1 = clock64(); cyc[6] = (t1 - t0); out[9] = (double)x;
}
int main() {
    double* d; long long* c; int* ch;
    cudaMalloc(&d, 16 * sizeof(double)); cudaMalloc(&c, 16 * sizeof(long long));
    double h[3] = {1.0000001, 0.9999999, 1e-9};
    cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    const char* nm[7] = {"DFMA", "DADD", "FFMA", "fp64 div", "fp64 sqrt+add", "LDG chase", "IMAD64 (LCG)"};
    for (long long span : {1LL << 12, 1LL << 20, 1LL << 26}) {  // 16 KB (L1), 4 MB (L2), 256 MB (HBM) of int
        int n = (int)span;
        int* hc = new int[n];
        for (int i = 0; i < n; ++i) hc[i] = (int)(((long long)i * 40503 + 4099) % n);  // stride permutation
        cudaMalloc(&ch, sizeof(int) * n);
        cudaMemcpy(ch, hc, sizeof(int) * n, cudaMemcpyHostToDevice);
        k_lat<<<1, 1>>>(d, c, ch, 512);  // warm
        k_lat<<<1, 1>>>(d, c, ch, 512);
        long long hcyc[7];
        cudaMemcpy(hcyc, c, sizeof hcyc, cudaMemcpyDeviceToHost);
        std::printf("span %lld ints:\n", span);
        for (int k = 0; k < 7; ++k) std::printf("  %-14s %6.1f cycles / op\n", nm[k], hcyc[k] / 1024.0);
        cudaFree(ch); delete[] hc;
    }
    return 0;
}
