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

template <int S, int RELEASE, bool PAIR = false, int GEMMLIKE = 0>   // RELEASE 0: mbarrier.arrive, 1: tcgen05.commit
__global__ void __launch_bounds__(64, 1) k_tma(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm2, const __grid_constant__ CUtensorMap tm2h, int iters, int rows_total,
                                               unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[16], empty[16], extra[2];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { mbar_init(smem_u32(&full[i]), 1); mbar_init(smem_u32(&empty[i]), GEMMLIKE == 3 ? 2 : 1); }
        mbar_init(smem_u32(&extra[0]), 1); mbar_init(smem_u32(&extra[1]), 1);
        fence_mbar_init();
    }
    const uint32_t rank = (PAIR || GEMMLIKE == 3) ? cluster_ctarank() : 0;
    if (RELEASE >= 1 && warp == 1) {
        if (PAIR) tmem_alloc_pair<32>(smem_u32(&slot)); else tmem_alloc<32>(smem_u32(&slot));
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR || GEMMLIKE == 3) cluster_sync();
    tc_fence_after();
    const uint32_t sb = smem_u32(smem);
    if (warp == 0 && lane == 0) {
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            mbar_wait(smem_u32(&empty[s]), ((it / S) & 1) ^ 1);
            const int row = ((blockIdx.x * 131 + it) * 256) % rows_total;
            if (GEMMLIKE == 3) {
                // cluster of 2 CTAs sharing the B tile: each loads its own A, half of B multicast to both
                const int tile = (blockIdx.x >> 1) + (it / 56) * (gridDim.x >> 1), kb = it % 56;
                const int arow = ((tile % 16) * 2 + (int)rank) * 128, brow = ((tile / 16) % 72) * 256;
                mbar_arrive_expect_tx(smem_u32(&full[s]), 16384 + 32768);
                tma_load_2d(sb + s * 49152, &tm, smem_u32(&full[s]), kb * 128, arow);
                tma_load_2d_mc(sb + s * 49152 + 16384 + rank * 16384, &tm2h, smem_u32(&full[s]), kb * 128, brow + rank * 128, 3);
            } else if (GEMMLIKE) {
                // A: tile rows fixed for 56 K-blocks, B: another tensor; K columns advance by 128
                const int tile = blockIdx.x + (it / 56) * gridDim.x, kb = it % 56;
                const int arow = (tile % 32) * 128, brow = ((tile / 32) % 72) * 256;
                mbar_arrive_expect_tx(smem_u32(&full[s]), 16384 + (GEMMLIKE == 2 ? 16384 : 32768));
                tma_load_2d(sb + s * 49152, &tm, smem_u32(&full[s]), kb * 128, arow);
                if (GEMMLIKE == 2) tma_load_2d(sb + s * 49152 + 16384, &tm, smem_u32(&full[s]), kb * 128, brow % 4096);
                else tma_load_2d(sb + s * 49152 + 16384, &tm2, smem_u32(&full[s]), kb * 128, brow);
            } else if (PAIR) {
                if (rank == 0) mbar_arrive_expect_tx(smem_u32(&full[s]), 65536);
                tma_load_2d_pair(sb + s * 32768, &tm, smem_u32(&full[s]), 0, row);
                tma_load_2d_pair(sb + s * 32768 + 16384, &tm, smem_u32(&full[s]), 128, row + 128);
            } else {
                mbar_arrive_expect_tx(smem_u32(&full[s]), 32768);
                tma_load_2d(sb + s * 32768, &tm, smem_u32(&full[s]), 0, row);
                tma_load_2d(sb + s * 32768 + 16384, &tm, smem_u32(&full[s]), 128, row + 128);
            }
        }
        unsigned long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    } else if (GEMMLIKE == 3 && warp == 1 && lane == 0) {
        // both CTAs' consumers must release a stage before either producer refills it (multicast)
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            mbar_wait(smem_u32(&full[s]), (it / S) & 1);
            mbar_arrive(smem_u32(&empty[s]));
            mbar_arrive_cluster(mapa_shared(smem_u32(&empty[s]), rank ^ 1));
        }
    } else if (warp == 1 && lane == 0 && rank == 0) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            mbar_wait(smem_u32(&full[s]), (it / S) & 1);
            if (PAIR) mma_commit_pair(smem_u32(&empty[s]), 3);
            else if (RELEASE == 0) mbar_arrive(smem_u32(&empty[s]));
            else mma_commit(smem_u32(&empty[s]));
            if (RELEASE == 2) mma_commit(smem_u32(&extra[it & 1]));   // second commit per stage (GEMM: pfull)
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR || GEMMLIKE == 3) cluster_sync();
    if (RELEASE >= 1 && warp == 1) {
        tc_fence_after();
        if (PAIR) tmem_dealloc_pair<32>(slot); else tmem_dealloc<32>(slot);
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;

template <int S, int RELEASE, bool PAIR = false, int GEMMLIKE = 0>
static void run(const char* name, void* buf, int rows, int grid, void* buf2 = nullptr) {
    CUtensorMap tm, tm2, tm2h;
    uint64_t dims[2] = {7168, (uint64_t)rows};
    uint64_t str[1] = {7168};
    uint32_t box[2] = {128, 128}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    {
        uint64_t dims2[2] = {7168, 18432};
        uint32_t box2[2] = {128, 256};
        enc(&tm2, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf2 ? buf2 : buf, dims2, str, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        uint32_t box3[2] = {128, 128};
        enc(&tm2h, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf2 ? buf2 : buf, dims2, str, box3, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    auto kern = k_tma<S, RELEASE, PAIR, GEMMLIKE>;
    const int smem = S * (GEMMLIKE ? 49152 : 32768) + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* dcyc;
    cudaMalloc(&dcyc, 148 * 8);
    const int iters = 4000;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(64); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (PAIR || GEMMLIKE == 3) ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    const int rt = rows - 256;
    cudaLaunchKernelEx(&cfg, kern, tm, tm2, tm2h, iters, rt, dcyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, kern, tm, tm2, tm2h, iters, rt, dcyc);
    cudaEventRecord(b);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s failed\n", name); return; }
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[148];
    cudaMemcpy(h, dcyc, grid * 8, cudaMemcpyDeviceToHost);
    double avg = 0; int cnt = 0; for (int i = 0; i < grid; i += (PAIR ? 2 : 1)) { if (h[i]) { avg += h[i]; ++cnt; } } avg /= cnt;
    const double sb = (GEMMLIKE == 1 || GEMMLIKE == 3) ? 49152.0 : 32768.0;
    printf("%-34s S=%d grid=%3d rows=%6d: %6.0f cyc/stage  %5.1f B/clk/SM  %6.1f TB/s total\n", name, S, grid, rows,
           avg / iters, sb * iters / avg, sb * iters * grid / (ms * 1e-3) / 1e12);
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
    void* wbig;
    cudaMalloc(&wbig, (size_t)7168 * 18432);
    cudaMemset(wbig, 0x38, (size_t)7168 * 18432);
    run<6, 1>("L2 commit-release", small, 2048, 148);
    run<6, 2>("L2 commit-release + 2nd commit", small, 2048, 148);
    run<4, 1, false, 1>("GEMM-like A(4096)+B(18432) 48KB", big, 4096, 148, wbig);
    run<4, 2, false, 1>("GEMM-like 48KB + 2nd commit", big, 4096, 148, wbig);
    return 0;
}
