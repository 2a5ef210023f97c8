// tools/l2_bench.cu — L2 -> SM delivery of a GEMM-like TMA pattern, no MMA (experiments only).
// Cluster of CS CTAs = P pairs stacked along M that share one N-tile (Fprop C1 shapes: A [4096,7168],
// B [18432,7168] uint8).  Per K-block each CTA needs its own 128 rows of A (16 KB, unicast) and the
// 128-row half of the B tile of its pair rank (16 KB).  With MC=1 the B half is split into P slices;
// CTA p of each rank loads slice p and multicasts it to the P CTAs of that rank, so each SM requests
// 16 + 16/P KB from L2 but receives 32 KB.  One consumer thread per CTA releases a stage to every CTA
// that writes into it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_bench tools/l2_bench.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../paper_2412_19437_b200/csrc/sm100.cuh"

using namespace fp8bs;

template <int CS, bool MC, int S>
__global__ void __launch_bounds__(64, 1) k_l2(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                                              int iters, int num_m, int num_n, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[8], empty[8];
    constexpr int P = CS / 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = CS > 1 ? cluster_ctarank() : 0;
    const int p = crank >> 1, r = crank & 1;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { mbar_init(smem_u32(&full[i]), 1); mbar_init(smem_u32(&empty[i]), MC ? P : 1); }
        fence_mbar_init();
    }
    __syncthreads();
    if (CS > 1) cluster_sync();
    const uint32_t sb = smem_u32(smem);
    const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;
    if (warp == 0 && lane == 0) {
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            mbar_wait(smem_u32(&empty[s]), ((it / S) & 1) ^ 1);
            const int tile = cid + (it / 56) * ncl, kb = it % 56;
            const int mt = tile % num_m, nt = (tile / num_m) % num_n;
            const int arow = (mt * P + p) * 256 + r * 128;      // this CTA's A rows
            const int brow = nt * 256 + r * 128;                 // this rank's B half
            const uint32_t dst = sb + s * 32768;
            mbar_arrive_expect_tx(smem_u32(&full[s]), 32768);
            tma_load_2d(dst, &tA, smem_u32(&full[s]), kb * 128, arow);
            if (MC && P > 1) {
                constexpr int SL = 128 / P;
                uint16_t mask = 0;
                for (int q = 0; q < P; ++q) mask |= (uint16_t)(1u << (2 * q + r));
                tma_load_2d_mc(dst + 16384 + p * SL * 128, &tB, smem_u32(&full[s]), kb * 128, brow + p * SL, mask);
            } else {
                tma_load_2d(dst + 16384, &tB, smem_u32(&full[s]), kb * 128, brow);
            }
        }
        cyc[blockIdx.x] = clock64() - t0;
    } else if (warp == 1 && lane == 0) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            mbar_wait(smem_u32(&full[s]), (it / S) & 1);
            if (MC && P > 1) {
                for (int q = 0; q < P; ++q) mbar_arrive_cluster(mapa_shared(smem_u32(&empty[s]), 2 * q + r));
            } else {
                mbar_arrive(smem_u32(&empty[s]));
            }
        }
    }
    __syncthreads();
    if (CS > 1) cluster_sync();
}

// Pair modes (cluster of 2, cta_group::2 TMA completing on the leader's barrier, like the GEMM):
// REL 0: the leader's consumer thread releases both CTAs' stages with mbarrier arrives;
// REL 1: with tcgen05.commit.cta_group::2 multicast (the GEMM's MMA warp, here with no MMAs).
// SPLITB: B half loaded as two 64-row boxes (the N = 128-half GEMM layout).
template <int REL, bool SPLITB, int S>
__global__ void __launch_bounds__(128, 1) k_pair(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                                                 const __grid_constant__ CUtensorMap tB64, int iters, int num_m, int num_n,
                                                 unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[8], empty[8];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t r = cluster_ctarank();
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { mbar_init(smem_u32(&full[i]), 1); mbar_init(smem_u32(&empty[i]), 1); }
        fence_mbar_init();
    }
    if (REL == 1 && warp == 2) tmem_alloc_pair<32>(smem_u32(&slot));
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t sb = smem_u32(smem);
    const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
    if (warp == 0) {
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            mbar_wait(smem_u32(&empty[s]), ((it / S) & 1) ^ 1);
            const int tile = cid + (it / 56) * ncl, kb = it % 56;
            const int mt = tile % num_m, nt = (tile / num_m) % num_n;
            const int arow = mt * 256 + r * 128;
            const uint32_t dst = sb + s * 32768;
            if (elect_one()) {
                if (r == 0) mbar_arrive_expect_tx(smem_u32(&full[s]), 65536);
                tma_load_2d_pair(dst, &tA, smem_u32(&full[s]), kb * 128, arow);
                if (SPLITB) {
                    tma_load_2d_pair(dst + 16384, &tB64, smem_u32(&full[s]), kb * 128, nt * 256 + r * 64);
                    tma_load_2d_pair(dst + 16384 + 8192, &tB64, smem_u32(&full[s]), kb * 128, nt * 256 + 128 + r * 64);
                } else {
                    tma_load_2d_pair(dst + 16384, &tB, smem_u32(&full[s]), kb * 128, nt * 256 + r * 128);
                }
            }
            __syncwarp();
        }
        if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
    } else if (warp == 1 && r == 0) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            mbar_wait(smem_u32(&full[s]), (it / S) & 1);
            tc_fence_after();
            if (elect_one()) {
                if (REL == 1) {
                    mma_commit_pair(smem_u32(&empty[s]), 3);
                } else {
                    mbar_arrive(smem_u32(&empty[s]));
                    mbar_arrive_cluster(mapa_shared(smem_u32(&empty[s]), 1));
                }
            }
            __syncwarp();
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (REL == 1 && warp == 2) { tc_fence_after(); tmem_dealloc_pair<32>(slot); }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;

template <int REL, bool SPLITB, int S>
static void run_pair(const char* name, void* A, void* B) {
    CUtensorMap tA, tB, tB64;
    uint32_t es[2] = {1, 1};
    uint64_t dA[2] = {7168, 4096}, dB[2] = {7168, 18432}, str[1] = {7168};
    uint32_t box[2] = {128, 128}, box64[2] = {128, 64};
    enc(&tA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, A, dA, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, B, dB, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tB64, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, B, dB, str, box64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    auto kern = k_pair<REL, SPLITB, S>;
    const int smem = S * 32768 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* dcyc;
    cudaMalloc(&dcyc, 148 * 8);
    const int iters = 56 * 16;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, tA, tB, tB64, iters, 16, 72, dcyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) cudaLaunchKernelEx(&cfg, kern, tA, tB, tB64, iters, 16, 72, dcyc);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s failed: %s\n", name, cudaGetErrorString(e)); return; }
    float ms; cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    unsigned long long h[148];
    cudaMemcpy(h, dcyc, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("%-40s S=%d: %6.0f cyc/kb  delivered %5.1f B/clk/SM  %5.1f TB/s  (%.1f us for 16 tiles)\n", name, S, avg / iters,
           32768.0 * iters / avg, 32768.0 * iters * 148 / (ms * 1e-3) / 1e12, ms * 1e3);
    fflush(stdout);
    cudaFree(dcyc);
}

template <int CS, bool MC, int S>
static void run(const char* name, void* A, void* B) {
    constexpr int P = CS / 2 > 0 ? CS / 2 : 1;
    CUtensorMap tA, tB;
    uint32_t es[2] = {1, 1};
    {
        uint64_t dims[2] = {7168, 4096}, str[1] = {7168};
        uint32_t box[2] = {128, 128};
        enc(&tA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    {
        uint64_t dims[2] = {7168, 18432}, str[1] = {7168};
        uint32_t box[2] = {128, (uint32_t)(MC ? 128 / P : 128)};
        enc(&tB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, B, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    auto kern = k_l2<CS, MC, S>;
    const int smem = S * 32768 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (CS > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    unsigned long long* dcyc;
    cudaMalloc(&dcyc, 148 * 8);
    const int grid = (148 / (CS > 1 ? CS : 1)) * (CS > 1 ? CS : 1);
    const int iters = 56 * 8;
    const int num_m = 4096 / (256 * P), num_n = 72;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(64); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS > 1 ? CS : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, tA, tB, iters, num_m, num_n, dcyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) cudaLaunchKernelEx(&cfg, kern, tA, tB, iters, num_m, num_n, dcyc);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s failed: %s\n", name, cudaGetErrorString(e)); return; }
    float ms; cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    unsigned long long h[148];
    cudaMemcpy(h, dcyc, grid * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < grid; ++i) avg += h[i];
    avg /= grid;
    const double req = 16384.0 + (MC ? 16384.0 / P : 16384.0);
    printf("%-30s CS=%d grid=%3d: %6.0f cyc/kb  delivered %5.1f B/clk/SM  requested %5.1f B/clk/SM  %5.1f TB/s delivered\n",
           name, CS, grid, avg / iters, 32768.0 * iters / avg, req * iters / avg, 32768.0 * iters * grid / (ms * 1e-3) / 1e12);
    fflush(stdout);
    cudaFree(dcyc);
}

int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    void *A, *B;
    cudaMalloc(&A, (size_t)7168 * 4096);
    cudaMalloc(&B, (size_t)7168 * 18432);
    cudaMemset(A, 0x38, (size_t)7168 * 4096);
    cudaMemset(B, 0x38, (size_t)7168 * 18432);
    run<2, false, 6>("pair, unicast, per-CTA barriers", A, B);
    run_pair<0, false, 6>("pair TMA, leader bar, mbarrier release", A, B);
    run_pair<1, false, 6>("pair TMA, leader bar, commit release", A, B);
    run_pair<0, true, 6>("pair TMA split B, mbarrier release", A, B);
    run_pair<1, true, 6>("pair TMA split B, commit release", A, B);
    run_pair<1, false, 4>("pair TMA, commit release", A, B);
    run_pair<1, false, 3>("pair TMA, commit release", A, B);
    return 0;
}
