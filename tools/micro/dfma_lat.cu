// Microbenchmark: DFMA dependent-chain latency and per-SM throughput on the local GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double *out, double a, double b, int iters, long long *cyc) {
    double x = threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) x = fma(x, a, b);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
template <int ILP>
__global__ void thru(double *out, double a, double b, int iters) {
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x * 1e-9 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void fchain(float *out, float a, float b, int iters, long long *cyc) {
    float x = threadIdx.x * 1e-9f;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) x = fmaf(x, a, b);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
int main() {
    double *d; float *f; long long *c;
    cudaMalloc(&d, 1 << 26); cudaMalloc(&f, 1 << 26); cudaMalloc(&c, 8 * 1024);
    int iters = 4096;
    long long h;
    chain<<<1, 32>>>(d, 0.999, 1e-3, iters, c); cudaDeviceSynchronize();
    chain<<<1, 32>>>(d, 0.999, 1e-3, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", (double)h / (iters * 16));
    fchain<<<1, 32>>>(f, 0.999f, 1e-3f, iters, c); cudaDeviceSynchronize();
    fchain<<<1, 32>>>(f, 0.999f, 1e-3f, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("FFMA dependent latency: %.2f cycles\n", (double)h / (iters * 16));
    int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        int blocks = p.multiProcessorCount, thr = warps * 32;
        thru<8><<<blocks, thr>>>(d, 0.999, 1e-3, 256); cudaDeviceSynchronize();
        cudaEventRecord(e0);
        thru<8><<<blocks, thr>>>(d, 0.999, 1e-3, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8 * iters * (double)blocks * thr;
        printf("DFMA throughput, %2d warps/SM, ILP 8: %.2f TFLOP/s  (%.1f DFMA/clk/SM at %d MHz)\n", warps, fl / ms / 1e9,
               fl / 2 / (ms * 1e-3) / blocks / (p.clockRate * 1e3), p.clockRate / 1000);
    }
    return 0;
}
