// Microbenchmark: streaming a [rows][nx] fp64 slab in NARROW column tiles (W = 8 or 16 columns x
// all rows) -- the access pattern of a cluster-free column-tile solver.  Each CTA (16 warps) walks
// tiles; per tile every warp loads a W x RB box (TMA, or cp.async 16 B per thread), then writes the
// tile back with coalesced stores.  Double-buffered.  Prints GB/s (16 B per element).
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

// MODE 0: TMA box W x RB per warp; MODE 1: cp.async 16 B per thread (W*RB*8/16 chunks per warp)
template <int W, int RB, int MODE>
__global__ void __launch_bounds__(512, 1) narrow(const __grid_constant__ CUtensorMap map, const double *in, double *out,
                                                 int nx, int rows, int sweeps) {
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t bar[2][16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kSlot = W * RB;  // doubles per warp per slot
    double *slot[2] = {sm + warp * kSlot, sm + (16 + warp) * kSlot};
    if (lane == 0) {
        mbar_init(&bar[0][warp]);
        mbar_init(&bar[1][warp]);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int ntx = nx / W, nty = rows / (16 * RB);
    const int total = ntx * nty;
    const int per = (total - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int J = per * sweeps;
    auto tile_of = [&](int j, int &tx, int &ty) {
        const int g = blockIdx.x + (j % per) * gridDim.x;
        tx = g % ntx;
        ty = g / ntx;
    };
    auto issue = [&](int j) {
        if (j >= J) return;
        int tx, ty;
        tile_of(j, tx, ty);
        const int r0 = ty * 16 * RB + warp * RB;
        if (MODE == 0) {
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect(&bar[j & 1][warp], kSlot * 8);
                tma2d(slot[j & 1], &map, tx * W, r0, &bar[j & 1][warp]);
            }
        } else {
            constexpr int kChunks = kSlot * 8 / 16;  // 16-B pieces per warp
            for (int i = lane; i < kChunks; i += 32) {
                const int row = i / (W / 2), c2 = i % (W / 2);
                const double *src = in + static_cast<size_t>(r0 + row) * nx + tx * W + 2 * c2;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(slot[j & 1] + row * W + 2 * c2)), "l"(src)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    };
    issue(0);
    issue(1);
    uint32_t ph = 0;
    for (int j = 0; j < J; ++j) {
        int tx, ty;
        tile_of(j, tx, ty);
        if (MODE == 0) {
            mbar_wait(&bar[j & 1][warp], (ph >> (j & 1)) & 1);
            ph ^= 1u << (j & 1);
        } else {
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            __syncwarp();
        }
        // lane = (column c = lane % W, row group g = lane / W); rows g, g + 32/W, ...
        constexpr int G = 32 / W;
        double v[RB / G];
#pragma unroll
        for (int i = 0; i < RB / G; ++i) v[i] = slot[j & 1][(i * G + lane / W) * W + lane % W];
        __syncwarp();
        if (MODE == 1) {  // keep the group accounting uniform: issue (possibly empty) group
        }
        issue(j + 2);
        const int r0 = ty * 16 * RB + warp * RB;
        double *dst = out + static_cast<size_t>(r0 + lane / W) * nx + tx * W + lane % W;
#pragma unroll
        for (int i = 0; i < RB / G; ++i) dst[static_cast<size_t>(i * G) * nx] = v[i] * 1.000001;
    }
}

int main() {
    const int nx = 4096, rows = 4096;
    double *a, *b;
    cudaMalloc(&a, sizeof(double) * nx * rows);
    cudaMalloc(&b, sizeof(double) * nx * rows);
    cudaMemset(a, 0, sizeof(double) * nx * rows);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int sweeps = 10;
    auto run = [&](auto kern, int W, int RB, int mode) {
        CUtensorMap map;
        cuuint64_t dims[2] = {(cuuint64_t)nx, (cuuint64_t)rows};
        cuuint64_t str[1] = {(cuuint64_t)nx * 8};
        cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)RB};
        cuuint32_t es[2] = {1, 1};
        enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const size_t smem = 2 * 16 * W * RB * 8;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<sms, 512, smem>>>(map, a, b, nx, rows, 1);
        cudaEventRecord(e0);
        kern<<<sms, 512, smem>>>(map, a, b, nx, rows, sweeps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("narrow %s W=%2d RB=%3d (tile %d x %d), smem %zu: %.0f GB/s  %s\n", mode ? "cp.async" : "TMA     ", W, RB, W,
               16 * RB, smem, 16.0 * nx * rows * sweeps / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    run(narrow<8, 32, 0>, 8, 32, 0);
    run(narrow<8, 64, 0>, 8, 64, 0);
    run(narrow<16, 32, 0>, 16, 32, 0);
    run(narrow<32, 16, 0>, 32, 16, 0);
    run(narrow<8, 32, 1>, 8, 32, 1);
    run(narrow<8, 64, 1>, 8, 64, 1);
    run(narrow<16, 32, 1>, 16, 32, 1);
    run(narrow<32, 16, 1>, 32, 16, 1);
    return 0;
}
