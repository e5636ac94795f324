// fp64 dependent-chain latency and issue throughput on this GPU (diagnostic).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, double a, int iters, long long* cyc) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < iters; ++i) x = x + a;  // dependent DADD chain
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

template <int ILP>
__global__ void thr(double* out, double a, int iters) {
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = a + threadIdx.x + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = x[k] + a;
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 64 * sizeof(double));
    cudaMalloc(&cyc, 1024 * sizeof(long long));
    const int iters = 1 << 14;
    chain<<<1, 32>>>(out, 1e-9, iters, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.2f cycles\n", (double)c / iters);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    for (int warps : {4, 8, 16, 32}) {
        const int blocks = 148 * 4, threads = warps * 32 / 4;
        thr<8><<<blocks, threads>>>(out, 1e-9, 1024);
        cudaEventRecord(e0);
        thr<8><<<blocks, threads>>>(out, 1e-9, 4096);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)blocks * threads * 4096 * 8;
        printf("warps/SM %2d ILP 8: %.2f Tdadd/s (%.1f per SM per clk at %d MHz)\n", warps, ops / ms / 1e9,
               ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
    }
    for (int warps : {8, 16, 32}) {
        const int blocks = 148 * 4, threads = warps * 32 / 4;
        thr<1><<<blocks, threads>>>(out, 1e-9, 1024);
        cudaEventRecord(e0);
        thr<1><<<blocks, threads>>>(out, 1e-9, 16384);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)blocks * threads * 16384;
        printf("warps/SM %2d ILP 1: %.2f Tdadd/s\n", warps, ops / ms / 1e9);
    }
    return 0;
}
