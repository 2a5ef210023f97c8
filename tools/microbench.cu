// tools/microbench.cu — B200 microbenchmarks that size the GEMM promotion step (not product code).
//   tmem   : tcgen05.ld throughput (bytes/clk/SM) vs load width and warp count
//   fma    : FFMA vs FFMA2 throughput for the promotion pattern acc[j] += p[j] * f
//   promo  : tcgen05.ld + FFMA2 together (the promotion inner loop without the MMA)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void tmem_alloc512(uint32_t dst) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(dst) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc512(uint32_t t) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t) : "memory");
}

#define LD32(taddr, r) asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" \
  : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]), \
    "=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(taddr))
#define LD16(taddr, r) asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
  : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]) : "r"(taddr))
__device__ __forceinline__ void ldwait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- TMEM load throughput ----
template <int W, int NLD>   // W = 16 or 32 columns per ld; NLD loads in flight before wait
__global__ void k_tmem(int iters, unsigned long long* cyc, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc512((uint32_t)__cvta_generic_to_shared(&slot));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
    // warps sharing a quadrant read different column ranges
    const uint32_t col0 = (warp >> 2) * 128;
    uint32_t acc = 0;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int l = 0; l < NLD; ++l) {
            uint32_t r[32];
            if (W == 32) LD32(base + ((col0 + l * W) & 511), r); else LD16(base + ((col0 + l * W) & 511), r);
            ldwait();
#pragma unroll
            for (int j = 0; j < W; ++j) acc ^= r[j];
        }
    }
    unsigned long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) tmem_dealloc512(slot);
}

// LD without per-load wait: NLD loads then one wait (max memory parallelism)
template <int NLD>
__global__ void k_tmem_batch(int iters, unsigned long long* cyc, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc512((uint32_t)__cvta_generic_to_shared(&slot));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
    uint32_t acc = 0;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[NLD][32];
#pragma unroll
        for (int l = 0; l < NLD; ++l) LD32(base + l * 32, r[l]);
        ldwait();
#pragma unroll
        for (int l = 0; l < NLD; ++l)
#pragma unroll
            for (int j = 0; j < 32; ++j) acc += r[l][j];
    }
    unsigned long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) tmem_dealloc512(slot);
}

// ---------------------------------------------------------------- FMA throughput ----
template <bool kPacked>
__global__ void k_fma(int iters, float f, unsigned long long* cyc, float* sink) {
    float acc[64], p[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) { acc[j] = 0.f; p[j] = threadIdx.x * 0.001f + j; }
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if constexpr (kPacked) {
            const float2 ff = make_float2(f, f);
#pragma unroll
            for (int j = 0; j < 64; j += 2) {
                float2 a = make_float2(acc[j], acc[j + 1]);
                a = __ffma2_rn(make_float2(p[j], p[j + 1]), ff, a);
                acc[j] = a.x; acc[j + 1] = a.y;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 64; ++j) acc[j] = __fmaf_rn(p[j], f, acc[j]);
        }
#pragma unroll
        for (int j = 0; j < 64; ++j) p[j] = __int_as_float(__float_as_int(p[j]) ^ it);  // keep p live
    }
    unsigned long long t1 = clock64();
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 64; ++j) s += acc[j];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// pure FMA chain without the xor (to isolate FMA rate)
template <bool kPacked>
__global__ void k_fma_pure(int iters, float f, unsigned long long* cyc, float* sink) {
    float acc[64], p[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) { acc[j] = 0.f; p[j] = threadIdx.x * 0.001f + j; }
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if constexpr (kPacked) {
            const float2 ff = make_float2(f, f);
#pragma unroll
            for (int j = 0; j < 64; j += 2) {
                float2 a = make_float2(acc[j], acc[j + 1]);
                a = __ffma2_rn(make_float2(p[j], p[j + 1]), ff, a);
                acc[j] = a.x; acc[j + 1] = a.y;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 64; ++j) acc[j] = __fmaf_rn(p[j], f, acc[j]);
        }
    }
    unsigned long long t1 = clock64();
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 64; ++j) s += acc[j];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// ---------------------------------------------------------------- promotion loop ----
// 8 warps; each warp: per "kb", load 128 columns (4 x LD32) of its quadrant and FMA into 128 acc.
template <bool kPacked>
__global__ void __launch_bounds__(256, 1) k_promo(int iters, float f, unsigned long long* cyc, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc512((uint32_t)__cvta_generic_to_shared(&slot));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
    float acc[128];
#pragma unroll
    for (int j = 0; j < 128; ++j) acc[j] = 0.f;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const uint32_t b = base + (it & 1) * 256;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            LD32(b + c * 32, r);
            ldwait();
            if constexpr (kPacked) {
                const float2 ff = make_float2(f, f);
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    float2 a = make_float2(acc[c * 32 + j], acc[c * 32 + j + 1]);
                    a = __ffma2_rn(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), ff, a);
                    acc[c * 32 + j] = a.x; acc[c * 32 + j + 1] = a.y;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[c * 32 + j] = __fmaf_rn(__uint_as_float(r[j]), f, acc[c * 32 + j]);
            }
        }
    }
    unsigned long long t1 = clock64();
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 128; ++j) s += acc[j];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) tmem_dealloc512(slot);
}

template <typename K>
static double run(K kern, int warps, int iters, const char* name, double bytes_or_ops_per_iter_per_warp, const char* unit,
                  unsigned long long* dcyc, void* dsink, float f = 1.0f, bool is_fma = false) {
    const int blocks = 148;
    if (is_fma) ((void (*)(int, float, unsigned long long*, float*))kern)<<<blocks, warps * 32>>>(iters, f, dcyc, (float*)dsink);
    else ((void (*)(int, unsigned long long*, uint32_t*))kern)<<<blocks, warps * 32>>>(iters, dcyc, (uint32_t*)dsink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return -1; }
    unsigned long long h[148];
    cudaMemcpy(h, dcyc, sizeof h, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < blocks; ++i) avg += h[i];
    avg /= blocks;
    double per_clk = bytes_or_ops_per_iter_per_warp * warps * iters / avg;
    printf("%-40s warps=%2d  %8.1f %s per clk per SM   (%.0f cyc)\n", name, warps, per_clk, unit, avg);
    return per_clk;
}

int main() {
    unsigned long long* dcyc;
    void* dsink;
    CK(cudaMalloc(&dcyc, 148 * sizeof(unsigned long long)));
    CK(cudaMalloc(&dsink, 148 * 1024 * 4));
    const int it = 2000;
    for (int w : {4, 8, 16}) {
        run(k_tmem<32, 4>, w, it, "tmem ld x32 (wait each)", 4 * 32 * 32 * 4.0, "B", dcyc, dsink);
        run(k_tmem<16, 8>, w, it, "tmem ld x16 (wait each)", 8 * 16 * 32 * 4.0, "B", dcyc, dsink);
        run(k_tmem_batch<2>, w, it, "tmem ld 2 x x32 then wait", 2 * 32 * 32 * 4.0, "B", dcyc, dsink);
        run(k_tmem_batch<4>, w, it, "tmem ld 4 x x32 then wait", 4 * 32 * 32 * 4.0, "B", dcyc, dsink);
    }
    for (int w : {4, 8, 16}) {
        run(k_fma_pure<false>, w, it, "FFMA  acc[j]+=p[j]*f (64 indep)", 64 * 32.0, "FMA", dcyc, dsink, 1.0001f, true);
        run(k_fma_pure<true>, w, it, "FFMA2 acc[j]+=p[j]*f (64 indep)", 64 * 32.0, "FMA", dcyc, dsink, 1.0001f, true);
    }
    for (int w : {8}) {
        run(k_promo<false>, w, it, "promo: 4xLD32 + FFMA (128 col)", 128 * 32.0, "elem", dcyc, dsink, 1.0001f, true);
        run(k_promo<true>, w, it, "promo: 4xLD32 + FFMA2 (128 col)", 128 * 32.0, "elem", dcyc, dsink, 1.0001f, true);
    }
    return 0;
}
