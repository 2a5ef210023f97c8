// tools/tma_bench.cu — TMA (cp.async.bulk.tensor) ring throughput per SM, no MMA: one producer
// thread refills S stages of 2 x (128 rows x 128 B, SWIZZLE_128B) boxes; one consumer thread waits
// on each full barrier and immediately releases the stage (plain mbarrier arrive or tcgen05.commit).
// Experiments only.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bench tools/tma_bench.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../paper_2412_19437_b200/csrc/sm100.cuh"

using namespace fp8bs;

template <int S, int RELEASE>   // RELEASE 0: mbarrier.arrive, 1: tcgen05.commit
__global__ void __launch_bounds__(64, 1) k_tma(const __grid_constant__ CUtensorMap tm, int iters, int rows_total,
                                               unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[16], empty[16];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { mbar_init(smem_u32(&full[i]), 1); mbar_init(smem_u32(&empty[i]), 1); }
        fence_mbar_init();
    }
    if (RELEASE == 1 && warp == 1) tmem_alloc<32>(smem_u32(&slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t sb = smem_u32(smem);
    if (warp == 0 && lane == 0) {
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            mbar_wait(smem_u32(&empty[s]), ((it / S) & 1) ^ 1);
            mbar_arrive_expect_tx(smem_u32(&full[s]), 32768);
            const int row = ((blockIdx.x * 131 + it) * 256) % rows_total;
            tma_load_2d(sb + s * 32768, &tm, smem_u32(&full[s]), 0, row);
            tma_load_2d(sb + s * 32768 + 16384, &tm, smem_u32(&full[s]), 128, row + 128);
        }
        unsigned long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    } else if (warp == 1 && lane == 0) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            mbar_wait(smem_u32(&full[s]), (it / S) & 1);
            if (RELEASE == 0) mbar_arrive(smem_u32(&empty[s]));
            else mma_commit(smem_u32(&empty[s]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (RELEASE == 1 && warp == 1) { tc_fence_after(); tmem_dealloc<32>(slot); }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;

template <int S, int RELEASE>
static void run(const char* name, void* buf, int rows, int grid) {
    CUtensorMap tm;
    uint64_t dims[2] = {7168, (uint64_t)rows};
    uint64_t str[1] = {7168};
    uint32_t box[2] = {128, 128}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    auto kern = k_tma<S, RELEASE>;
    const int smem = S * 32768 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* dcyc;
    cudaMalloc(&dcyc, 148 * 8);
    const int iters = 4000;
    kern<<<grid, 64, smem>>>(tm, iters, rows - 256, dcyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<grid, 64, smem>>>(tm, iters, rows - 256, dcyc);
    cudaEventRecord(b);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s failed\n", name); return; }
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[148];
    cudaMemcpy(h, dcyc, grid * 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < grid; ++i) avg += h[i]; avg /= grid;
    printf("%-34s S=%d grid=%3d rows=%6d: %6.0f cyc/stage  %5.1f B/clk/SM  %6.1f TB/s total\n", name, S, grid, rows,
           avg / iters, 32768.0 * iters / avg, 32768.0 * iters * grid / (ms * 1e-3) / 1e12);
    fflush(stdout);
    cudaFree(dcyc);
}

int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    void *big, *small;
    cudaMalloc(&big, (size_t)7168 * 65536);      // 470 MB: DRAM-resident
    cudaMalloc(&small, (size_t)7168 * 2048);     // 14.7 MB: L2-resident
    cudaMemset(big, 0x38, (size_t)7168 * 65536);
    cudaMemset(small, 0x38, (size_t)7168 * 2048);
    run<6, 0>("L2 arrive-release", small, 2048, 148);
    run<6, 1>("L2 commit-release", small, 2048, 148);
    run<2, 0>("L2 arrive-release", small, 2048, 148);
    run<4, 0>("L2 arrive-release", small, 2048, 148);
    run<6, 0>("L2 arrive-release 1 SM", small, 2048, 1);
    run<6, 0>("L2 arrive-release 16 SM", small, 2048, 16);
    run<6, 0>("DRAM arrive-release", big, 65536, 148);
    run<6, 1>("DRAM commit-release", big, 65536, 148);
    return 0;
}
