// Probe: cudaOccupancyMaxActiveClusters for cluster sizes 2..16 at the fused kernel's footprint.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(double *p) { extern __shared__ double s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (size_t smem : {100 * 1024, 110 * 1024, 200 * 1024}) {
        cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int thr : {256, 512}) {
            printf("smem %zu KB, %d threads:", smem / 1024, thr);
            for (int c = 2; c <= 16; ++c) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(c, 64, 1);
                cfg.blockDim = dim3(thr);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute a[1];
                a[0].id = cudaLaunchAttributeClusterDimension;
                a[0].val.clusterDim.x = c; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
                cfg.attrs = a; cfg.numAttrs = 1;
                int n = -1;
                cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
                printf(" C=%d:%d(%d)", c, e == cudaSuccess ? n : -1, e == cudaSuccess ? n * c : -1);
            }
            printf("  [SMs %d]\n", sms);
        }
    }
    return 0;
}
