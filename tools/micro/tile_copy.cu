// Microbenchmark: achievable HBM bandwidth of the step kernel's access pattern, without the solve.
// A slab [rows][nx] fp64 is read tile by tile through TMA boxes of (W + 4) x 32 doubles (the x-halo
// of the fused kernel, start 2 columns left of the tile) by 8 warps per CTA (one box per warp =
// 32 rows x (W+4) columns), and the W columns are written back with coalesced st.global into a
// second slab.  Persistent CTAs walk the tiles (W columns x 256 rows), double-buffered per warp.
//   ./tile_copy            prints GB/s (read W + write W per element) for W = 32, 64, 128
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t *b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b))); }
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                     su32(b)), "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void tma2d(void *dst, const CUtensorMap *m, int x, int y, uint64_t *b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(su32(b))
        : "memory");
}

template <int W, int RB, int HX = 4, int HL = 2>
__global__ void __launch_bounds__(256, 1) tile_copy(const __grid_constant__ CUtensorMap map, double *out, int nx, int rows,
                                                    int ntiles_x, int ntiles_y, int sweeps) {
    constexpr int BW = W + HX;
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t bar[2][8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *slot[2] = {sm + warp * RB * BW, sm + (8 + warp) * RB * BW};
    if (lane == 0) {
        mbar_init(&bar[0][warp]);
        mbar_init(&bar[1][warp]);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int total = ntiles_x * ntiles_y;
    const int per = (total - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int J = per * sweeps;
    auto tile_of = [&](int j, int &tx, int &ty) {
        const int g = blockIdx.x + (j % per) * gridDim.x;
        tx = g % ntiles_x;
        ty = g / ntiles_x;
    };
    const uint32_t bytes = BW * RB * 8;
    auto issue = [&](int j) {
        if (j >= J || lane != 0) return;
        int tx, ty;
        tile_of(j, tx, ty);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect(&bar[j & 1][warp], bytes);
        tma2d(slot[j & 1], &map, tx * W - HL, ty * 8 * RB + warp * RB, &bar[j & 1][warp]);
    };
    issue(0);
    issue(1);
    uint32_t ph = 0;
    for (int j = 0; j < J; ++j) {
        int tx, ty;
        tile_of(j, tx, ty);
        mbar_wait(&bar[j & 1][warp], (ph >> (j & 1)) & 1);
        ph ^= 1u << (j & 1);
        double v[RB][W / 32];
#pragma unroll
        for (int l = 0; l < RB; ++l)
#pragma unroll
            for (int c = 0; c < W / 32; ++c) v[l][c] = slot[j & 1][l * BW + HL + c * 32 + lane];
        __syncwarp();
        issue(j + 2);
        double *dst = out + static_cast<size_t>(ty * 8 * RB + warp * RB) * nx + tx * W + lane;
#pragma unroll
        for (int l = 0; l < RB; ++l)
#pragma unroll
            for (int c = 0; c < W / 32; ++c) dst[static_cast<size_t>(l) * nx + c * 32] = v[l][c] * 1.000001;
    }
}

// plain streaming copy (reference ceiling): float4-free, double2 coalesced
__global__ void plain_copy(const double2 *__restrict__ a, double2 *__restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
    const int nx = 4096, rows = 4096;  // two c2 subdomain slabs (2 x 2048 rows)
    double *a, *b;
    cudaMalloc(&a, sizeof(double) * nx * rows);
    cudaMalloc(&b, sizeof(double) * nx * rows);
    cudaMemset(a, 0, sizeof(double) * nx * rows);
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int sweeps = 10;
    {
        const size_t n = (size_t)nx * rows / 2;
        plain_copy<<<sms * 8, 256>>>((double2 *)a, (double2 *)b, n);
        cudaEventRecord(e0);
        for (int s = 0; s < sweeps; ++s) plain_copy<<<sms * 8, 256>>>((double2 *)a, (double2 *)b, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("plain copy: %.0f GB/s\n", 16.0 * nx * rows * sweeps / ms / 1e6);
    }
    auto run = [&](auto kern, int W, int RB, int ctas_per_sm, int HX = 4, int prom = 2) {
        CUtensorMap map;
        cuuint64_t dims[2] = {(cuuint64_t)nx, (cuuint64_t)rows};
        cuuint64_t str[1] = {(cuuint64_t)nx * 8};
        cuuint32_t box[2] = {(cuuint32_t)(W + HX), (cuuint32_t)RB};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("encode failed %d\n", (int)r);
            return;
        }
        const size_t smem = 2 * 8 * RB * (W + HX) * 8;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int grid = sms * ctas_per_sm;
        kern<<<grid, 256, smem>>>(map, b, nx, rows, nx / W, rows / (8 * RB), 1);
        cudaEventRecord(e0);
        kern<<<grid, 256, smem>>>(map, b, nx, rows, nx / W, rows / (8 * RB), sweeps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        printf("TMA tile copy W=%3d (box %d x %d), prom %d, %d CTA/SM, smem %zu: %.0f GB/s (alg. 16 B/elem)  %s\n", W, W + HX, RB,
               prom, ctas_per_sm, smem, 16.0 * nx * rows * sweeps / ms / 1e6, cudaGetErrorString(err));
    };
    for (int prom = 0; prom < 4; ++prom) run(tile_copy<32, 32>, 32, 32, 1, 4, prom);
    run(tile_copy<32, 32, 2, 0>, 32, 32, 1, 2, 2);
    run(tile_copy<32, 32, 0, 0>, 32, 32, 1, 0, 2);
    run(tile_copy<32, 16>, 32, 16, 2, 4, 2);
    run(tile_copy<32, 16, 2, 0>, 32, 16, 2, 2, 2);
    run(tile_copy<64, 16>, 64, 16, 1, 4, 2);
    run(tile_copy<128, 8>, 128, 8, 1, 4, 2);
    return 0;
}
