// ep.cu — the exchange steps around the expert GEMM in expert parallelism (NEXT-3; §3.3.4
// "we quantize the activation before MoE up-projections into FP8 and then apply dispatch
// components ... the combine components ... retained in BF16"), over NVLink peer memory.
//
// The caller maps every rank's receive buffers into this process (peer pointers, e.g. torch symmetric
// memory or CUDA IPC) and passes them as a DEVICE array indexed by rank; the kernels then write the
// rows straight into the destination GPU's memory (NVLink/NVSwitch stores, fire-and-forget), one warp
// per row.  Ordering across GPUs (the receiver may read only after every sender's kernel finished) is
// the caller's barrier.
#include <cuda_bf16.h>

#include "sm100.cuh"
#include "internal.h"

namespace fp8bs {

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// Dispatch: slot i = (local token i / top_k, its (i % top_k)-th expert) goes to rank dst_rank[i] (< 0: not
// sent), receive row dst_row[i]: the token's K E4M3 codes (16-byte vectors, a 512-byte warp store per
// step) and its K/128 1x128 scales (row-major: recv_s[r][row * KB + kb], so a row's scales are one
// contiguous 4*KB-byte run over the link rather than KB scattered 4-byte writes).
__global__ void __launch_bounds__(256) k_dispatch_fp8(int64_t n, int top_k, int64_t K, int64_t KB, const uint8_t* __restrict__ xq,
                                                      int64_t ldxq, const float* __restrict__ xs, int64_t ldxs,
                                                      const int32_t* __restrict__ dst_rank, const int64_t* __restrict__ dst_row,
                                                      uint8_t* const* __restrict__ recv_q, int64_t ld_rq,
                                                      float* const* __restrict__ recv_s) {
    griddep_wait();
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * 8;
    for (int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); i < n; i += nw) {
        const int r = dst_rank[i];
        if (r < 0) continue;
        const int64_t row = dst_row[i], t = i / top_k;
        const uint8_t* src = xq + t * ldxq;
        uint8_t* dst = recv_q[r] + row * ld_rq;
        for (int64_t c = (int64_t)lane * 16; c < K; c += 512)
            *reinterpret_cast<uint4*>(dst + c) = ldg_nc_v4(src + c);
        float* ds = recv_s[r] + row * KB;
        for (int64_t kb = lane; kb < KB; kb += 32) ds[kb] = xs[kb * ldxs + t];
    }
}

// Row-major [R][KB] scales -> the GEMM's contraction-block-major [KB][ldd] layout (32 x 32 tiles through
// shared memory: both sides coalesced).
__global__ void __launch_bounds__(256) k_rows_to_blocks(int64_t R, int64_t KB, const float* __restrict__ src,
                                                        float* __restrict__ dst, int64_t ldd) {
    __shared__ float tile[32][33];
    griddep_wait();
    griddep_launch_dependents();
    const int64_t r0 = (int64_t)blockIdx.x * 32, k0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    for (int j = ty; j < 32; j += 8) {
        const int64_t r = r0 + j, k = k0 + tx;
        if (r < R && k < KB) tile[j][tx] = src[r * KB + k];
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
        const int64_t k = k0 + j, r = r0 + tx;
        if (r < R && k < KB) dst[k * ldd + r] = tile[tx][j];
    }
}

// Combine push: local expert output row i (BF16 [R, N]) -> rank dst_rank[i]'s combine buffer, row
// dst_slot[i] (= token * top_k + k on that rank).
__global__ void __launch_bounds__(256) k_combine_push(int64_t R, int64_t nbytes, const uint8_t* __restrict__ y, int64_t ldy_b,
                                                      const int32_t* __restrict__ dst_rank, const int64_t* __restrict__ dst_slot,
                                                      uint8_t* const* __restrict__ recv_y, int64_t ldr_b) {
    griddep_wait();
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * 8;
    for (int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); i < R; i += nw) {
        const int r = dst_rank[i];
        if (r < 0) continue;
        const uint8_t* src = y + i * ldy_b;
        uint8_t* dst = recv_y[r] + dst_slot[i] * ldr_b;
        for (int64_t c = (int64_t)lane * 16; c < nbytes; c += 512)
            *reinterpret_cast<uint4*>(dst + c) = ldg_nc_v4(src + c);
    }
}

// Combine reduce (reading R28): out[t][n] = BF16_RNE(acc), acc = fma(g[t][k], y[t*top_k+k][n], acc)
// from 0 in k order; one thread per 8 columns.
__global__ void __launch_bounds__(256) k_combine_reduce(int64_t T, int top_k, int64_t N, const __nv_bfloat16* __restrict__ buf,
                                                        int64_t ldb, const float* __restrict__ g,
                                                        __nv_bfloat16* __restrict__ out, int64_t ldo) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t per_row = N / 8;
    const int64_t total = T * per_row;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < total; u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = u / per_row, c = (u - t * per_row) * 8;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int k = 0; k < top_k; ++k) {
            const float gk = g[t * top_k + k];
            const uint4 v = ldg_nc_v4(buf + (t * top_k + k) * ldb + c);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                acc[2 * j] = __fmaf_rn(gk, __uint_as_float(w[j] << 16), acc[2 * j]);
                acc[2 * j + 1] = __fmaf_rn(gk, __uint_as_float(w[j] & 0xFFFF0000u), acc[2 * j + 1]);
            }
        }
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * j], acc[2 * j + 1]);
            o[j] = *reinterpret_cast<uint32_t*>(&b);
        }
        *reinterpret_cast<uint4*>(out + t * ldo + c) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

static int rows_grid(int64_t rows) {   // one warp per row, 8 per CTA, at most 8 CTAs per SM
    const int64_t ctas = (rows + 7) / 8, cap = (int64_t)num_sms() * 8;
    return (int)(ctas < 1 ? 1 : (ctas > cap ? cap : ctas));
}

cudaError_t launch_dispatch_fp8(int64_t n, int top_k, int64_t K, const uint8_t* xq, int64_t ldxq, const float* xs,
                                int64_t ldxs, const int32_t* dst_rank, const int64_t* dst_row, uint8_t* const* recv_q,
                                int64_t ld_rq, float* const* recv_s, cudaStream_t st) {
    return launch_pdl(k_dispatch_fp8, dim3(rows_grid(n)), dim3(256), 0, st, n, top_k, K, K / 128, xq, ldxq, xs, ldxs,
                      dst_rank, dst_row, recv_q, ld_rq, recv_s);
}
cudaError_t launch_rows_to_blocks(int64_t R, int64_t KB, const float* src, float* dst, int64_t ldd, cudaStream_t st) {
    return launch_pdl(k_rows_to_blocks, dim3((unsigned)((R + 31) / 32), (unsigned)((KB + 31) / 32)), dim3(256), 0, st,
                      R, KB, src, dst, ldd);
}
cudaError_t launch_combine_push(int64_t R, int64_t N, const void* y, int64_t ldy, const int32_t* dst_rank,
                                const int64_t* dst_slot, void* const* recv_y, int64_t ld_recv_y, cudaStream_t st) {
    return launch_pdl(k_combine_push, dim3(rows_grid(R)), dim3(256), 0, st, R, N * 2, reinterpret_cast<const uint8_t*>(y),
                      ldy * 2, dst_rank, dst_slot, reinterpret_cast<uint8_t* const*>(recv_y), ld_recv_y * 2);
}
cudaError_t launch_combine_reduce(int64_t T, int top_k, int64_t N, const void* buf, int64_t ldb, const float* g, void* out,
                                  int64_t ldo, cudaStream_t st) {
    const int64_t total = T * (N / 8);
    const int64_t ctas = (total + 255) / 256, cap = (int64_t)num_sms() * 8;
    return launch_pdl(k_combine_reduce, dim3((unsigned)(ctas < 1 ? 1 : (ctas > cap ? cap : ctas))), dim3(256), 0, st, T,
                      top_k, N, reinterpret_cast<const __nv_bfloat16*>(buf), ldb, g, reinterpret_cast<__nv_bfloat16*>(out), ldo);
}

}  // namespace fp8bs
