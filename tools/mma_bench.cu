// tools/mma_bench.cu — tcgen05.mma kind::f8f6f4 peak throughput with operands resident in smem
// (no TMA), for 1-CTA (M=128) and CTA-pair (M=256) shapes.  Experiments only, not product code.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../paper_2412_19437_b200/csrc/sm100.cuh"
#define LD32X(taddr, r) FP8BS_TMEM_LD32(taddr, r)

using namespace fp8bs;
__device__ int tma_count[148];
static CUtensorMap g_tmx;

// iters K-blocks of 4 MMAs each; buffers alternate between TMEM columns [0,N) and [N,2N);
// commit every kb to an mbarrier; the issuing thread waits on the commit of kb-depth (depth in-flight).
template <int N, bool kPair, int DEPTH, int MP = 256, int MODE = 0>
__global__ void __launch_bounds__(640, 1) k_mma(int iters, unsigned long long* cyc, const __grid_constant__ CUtensorMap tmx) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bars[8];
    __shared__ uint32_t slot;
    __shared__ volatile int stop;
    __shared__ uint64_t tbar[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = kPair ? cluster_ctarank() : 0;
    const uint32_t sa = smem_u32(smem);
    const uint32_t sb = sa + 16384;
    for (int i = threadIdx.x; i < (16384 + N * 128 / (kPair ? 2 : 1)) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = (MODE & 8) ? ((uint32_t)(i * 2654435761u + blockIdx.x * 40503u) & 0x77777777u) : 0x38383838u;   // MODE 3: random codes
    if (threadIdx.x == 0) {
        stop = 0;
        for (int i = 0; i < 8; ++i) mbar_init(smem_u32(&bars[i]), 1);
        for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&tbar[i]), 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        if constexpr (kPair) tmem_alloc_pair<512>(smem_u32(&slot));
        else tmem_alloc<512>(smem_u32(&slot));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    if constexpr (kPair) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = slot;
    if ((MODE & 16) && (warp == 0 || warp == 3) && rank == 0) {
        // two issuing warps: warp 0 issues into even buffers, warp 3 into odd ones (each commits its own)
        constexpr uint32_t idesc = idesc_e4m3_f32(kPair ? MP : 128, N);
        const uint64_t ad = sdesc_k_sw128(sa), bd = sdesc_k_sw128(sb);
        const int w = warp == 0 ? 0 : 1;
        unsigned long long t0 = clock64();
        for (int kb = w; kb < iters; kb += 2) {
            if (kb >= DEPTH) mbar_wait(smem_u32(&bars[(kb - DEPTH) & 7]), ((kb - DEPTH) >> 3) & 1);
            const uint32_t d = tmem + ((kb % (512 / N)) * N);
            if (elect_one()) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if constexpr (kPair) mma_f8f6f4_pair(d, ad + 2 * k, bd + 2 * k, idesc, k > 0);
                    else mma_f8f6f4(d, ad + 2 * k, bd + 2 * k, idesc, k > 0);
                }
                if constexpr (kPair) mma_commit_pair(smem_u32(&bars[kb & 7]), 1);
                else mma_commit(smem_u32(&bars[kb & 7]));
            }
            __syncwarp();
        }
        for (int kb = iters - DEPTH > 0 ? iters - DEPTH : 0; kb < iters; ++kb)
            if ((kb & 1) == w) mbar_wait(smem_u32(&bars[kb & 7]), (kb >> 3) & 1);
        unsigned long long t1 = clock64();
        if (lane == 0 && w == 0) cyc[blockIdx.x / (kPair ? 2 : 1)] = t1 - t0;
    } else if (warp == 0 && rank == 0) {
        // whole warp runs the loop; one elected lane issues (a lane-0-only loop makes ptxas wrap
        // every tcgen05.mma in an ELECT/R2UR waterfall, ~100 cycles per instruction)
        constexpr uint32_t idesc = idesc_e4m3_f32(kPair ? MP : 128, N);
        const uint64_t ad = sdesc_k_sw128(sa), bd = sdesc_k_sw128(sb);
        unsigned long long t0 = clock64();
        for (int kb = 0; kb < iters; ++kb) {
            if (kb >= DEPTH) mbar_wait(smem_u32(&bars[(kb - DEPTH) & 7]), ((kb - DEPTH) >> 3) & 1);
            const uint32_t d = tmem + ((kb % (512 / N)) * N);
            if (elect_one()) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if constexpr (kPair) mma_f8f6f4_pair(d, ad + 2 * k, bd + 2 * k, idesc, k > 0);
                    else mma_f8f6f4(d, ad + 2 * k, bd + 2 * k, idesc, k > 0);
                }
                if constexpr (kPair) mma_commit_pair(smem_u32(&bars[kb & 7]), 1);
                else mma_commit(smem_u32(&bars[kb & 7]));
            }
            __syncwarp();
        }
        for (int kb = iters - DEPTH > 0 ? iters - DEPTH : 0; kb < iters; ++kb)
            mbar_wait(smem_u32(&bars[kb & 7]), (kb >> 3) & 1);
        unsigned long long t1 = clock64();
        if (lane == 0) cyc[blockIdx.x / (kPair ? 2 : 1)] = t1 - t0;
        if (lane == 0) {
            stop = 1;
            if (kPair) asm volatile("st.shared::cluster.u32 [%0], %1;" :: "r"(mapa_shared(smem_u32((const void*)&stop), 1)), "r"(1) : "memory");
        }
    } else if ((MODE & 4) && warp == 2 && lane == 0) {
        // interference: a TMA stream into a 4 x 32 KB ring (immediately re-armed), ~rate of a GEMM feed
        const uint32_t ring = smem_u32(smem) + 65536;
        uint32_t bars = smem_u32(&tbar[0]);
        int it = 0;
        while (!stop) {
            const int s = it & 3;
            if (it >= 4) mbar_wait(bars + 8 * s, ((it >> 2) - 1) & 1);
            mbar_arrive_expect_tx(bars + 8 * s, 32768);
            tma_load_2d(ring + s * 32768, &tmx, bars + 8 * s, 0, (it * 256 + blockIdx.x * 128) % 3840);
            tma_load_2d(ring + s * 32768 + 16384, &tmx, bars + 8 * s, 128, (it * 256 + blockIdx.x * 128) % 3840);
            ++it;
        }
        for (int j = it - 4 < 0 ? 0 : it - 4; j < it; ++j) mbar_wait(bars + 8 * (j & 3), (j >> 2) & 1);
        tma_count[blockIdx.x] = it;
    } else if ((MODE & 1) && warp >= 4) {
        // interference: continuous tcgen05.ld of 64 columns per thread (TMEM read traffic)
        const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((warp >> 2) - 1) * 64;
        uint32_t acc = 0;
        int n = 0;
        while (!stop) {
            uint32_t r[32];
            LD32X(base, r); asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int j = 0; j < 32; ++j) acc += r[j];
            ++n;
        }
        if (acc == 12345) cyc[200] = acc;
        if (lane == 0 && warp == 4) tma_count[blockIdx.x] = n;
    } else if ((MODE & 2) && warp >= 4 && warp < 12) {
        // interference: continuous 16-byte smem stores into a scratch region (like TMA writes)
        uint32_t a = smem_u32(smem) + 65536 + (threadIdx.x % 256) * 16;
        uint32_t v = threadIdx.x;
        while (!stop) {
            for (int i = 0; i < 16; ++i)
                asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" :: "r"(a + (i % 8) * 4096), "r"(v) : "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (kPair) cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        if constexpr (kPair) tmem_dealloc_pair<512>(tmem);
        else tmem_dealloc<512>(tmem);
    }
}

template <int N, bool kPair, int DEPTH, int MP = 256, int MODE = 0>
static void run(const char* name, int iters) {
    auto kern = k_mma<N, kPair, DEPTH, MP, MODE>;
    const int smem = 1024 + 65536 + 131072 + 4096;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* dcyc;
    cudaMalloc(&dcyc, 256 * 8);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3((MODE & 3) ? 640 : 128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kPair ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, kern, iters, dcyc, g_tmx);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, kern, iters, dcyc, g_tmx);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[148];
    cudaMemcpy(h, dcyc, sizeof h, cudaMemcpyDeviceToHost);
    const int nunits = kPair ? 74 : 148;
    double avg = 0; for (int i = 0; i < nunits; ++i) avg += h[i]; avg /= nunits;
    const double macs_per_kb_per_sm = (kPair ? MP / 2.0 : 128.0) * N * 128;    // per SM (pair: each SM does 128 rows)
    const double flops = 2.0 * macs_per_kb_per_sm * iters * 148;
    printf("%-28s N=%3d depth=%d: %7.1f cyc/kb  (ideal %d)  %6.0f MAC/clk/SM  %7.1f TFLOP/s (events)\n", name, N, DEPTH,
           avg / iters, (int)(macs_per_kb_per_sm / 8192), macs_per_kb_per_sm * iters / avg, flops / (ms * 1e-3) / 1e12);
    if (MODE & 4) { int tc[148]; cudaMemcpyFromSymbol(tc, tma_count, sizeof tc); printf("    concurrent TMA: %.1f B/clk/SM\n", 32768.0 * tc[0] / h[0]); }
    else if (MODE & 1) { int tc[148]; cudaMemcpyFromSymbol(tc, tma_count, sizeof tc); printf("    concurrent TMEM reads: %.1f B/clk/SM\n", 16.0 * 32768.0 * tc[0] / h[0]); }
    fflush(stdout);
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    void* buf; cudaMalloc(&buf, (size_t)7168 * 4096); cudaMemset(buf, 0x38, (size_t)7168 * 4096);
    uint64_t dims[2] = {7168, 4096}, str[1] = {7168}; uint32_t box[2] = {128, 128}, es[2] = {1, 1};
    enc(&g_tmx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int it = 20000;
    run<256, true, 2, 256, 0>("pair N=256 alone d2", it);
    run<128, true, 4, 256, 0>("pair N=128 d4", it);
    run<64, true, 8, 256, 0>("pair N=64 d8", it);
    run<32, true, 8, 256, 0>("pair N=32 d8", it);
    run<128, false, 4, 256, 0>("1-CTA N=128 d4", it);
    run<64, false, 8, 256, 0>("1-CTA N=64 d8", it);
    run<64, true, 8, 256, 16>("pair N=64 d8 two issuers", it);
    run<32, true, 8, 256, 16>("pair N=32 d8 two issuers", it);
    run<64, false, 8, 256, 16>("1-CTA N=64 d8 two issuers", it);
    return 0;
}
