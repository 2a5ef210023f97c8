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

// Streamed dispatch (overlapped with the expert GEMM on the receivers): the sender's slots come as a
// SEND LIST sorted by (chunk, destination rank, destination row); chunk c of a receiver is the rows of
// its local expert groups g with g * C / G == c, so every receiver's GEMM can start on chunk c as soon as
// all senders have delivered it.  Per entry: the token's K codes (a warp per row, 16-byte stores) and its
// KB scales written straight into the receiver's [KB][ld_rs] GEMM layout (lane = entry: 32 consecutive
// destination rows give 128-byte stores per contraction block).  After its part of chunk c every CTA
// fences (system scope) and counts itself on local_done[c]; the CTA that completes the count publishes the
// chunk with one release-add on every receiver's flag[c].  local_done is zeroed on the stream before every
// call; the flags are monotonic: after call number `epoch` (1, 2, ...) each flag[c] = world * epoch.
__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// The codes of a row travel by TMA bulk copies (global -> shared -> peer global, one elected lane per
// warp driving a per-warp ring of kDsStages row buffers): a warp then keeps several rows in flight with a
// handful of instructions, so a dispatch confined to a few SMs still fills the link (per-lane 16-byte
// peer stores reached ~15-20 GB/s per SM, i.e. ~40 SMs taken from the concurrent GEMM).
// Measured (C4, 2 GPUs, the dispatch alone): ~18-30 GB/s per SM whatever the ring shape (4 warps x 4
// stages, 3 loads ahead: 6.7 ms on 8 SMs, 2.1 ms on 32, 1.6 ms on 128; 2 warps x 8 stages, 2 ahead: 12.4 ms
// on 8 SMs), like per-lane 16-byte peer stores: a dispatch confined to few SMs cannot fill the link.
constexpr int kDsWarps = 4, kDsStages = 4, kDsAhead = 3;

__global__ void __launch_bounds__(32 * kDsWarps) k_dispatch_stream(int C, const int64_t* __restrict__ chunk_off,
                                                         const int64_t* __restrict__ send_tok, const int32_t* __restrict__ send_rank,
                                                         const int64_t* __restrict__ send_row, int64_t K, int64_t KB,
                                                         const uint8_t* __restrict__ xq, int64_t ldxq,
                                                         const float* __restrict__ xs, int64_t ldxs,
                                                         uint8_t* const* __restrict__ recv_q, int64_t ld_rq,
                                                         float* const* __restrict__ recv_s, int64_t ld_rs,
                                                         uint32_t* __restrict__ local_done, uint32_t* const* __restrict__ flags,
                                                         int world, uint32_t epoch) {
    extern __shared__ __align__(128) uint8_t dsmem[];
    griddep_wait();
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t rowb = (uint32_t)((K + 127) / 128 * 128);           // one staged row, 128-byte aligned
    const uint32_t ring = smem_u32(dsmem) + (uint32_t)warp * kDsStages * rowb;
    const uint32_t bar0 = smem_u32(dsmem) + (uint32_t)kDsWarps * kDsStages * rowb + (uint32_t)warp * kDsStages * 8;
    if (lane == 0) {
        for (int i = 0; i < kDsStages; ++i) mbar_init(bar0 + 8 * i, 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t nload = 0;                                                // rows loaded by this warp so far (ring position)
    for (int c = 0; c < C; ++c) {
        const int64_t s0 = chunk_off[c], s1 = chunk_off[c + 1];
        const int64_t nb = (s1 - s0 + 31) / 32;
        for (int64_t b = (int64_t)blockIdx.x * kDsWarps + warp; b < nb; b += (int64_t)gridDim.x * kDsWarps) {
            const int64_t e0 = s0 + b * 32;
            const int n = (int)min((int64_t)32, s1 - e0);
            int64_t tok = 0, row = 0;
            int rk = 0;
            if (lane < n) { tok = send_tok[e0 + lane]; rk = send_rank[e0 + lane]; row = send_row[e0 + lane]; }
            // codes: lane 0 streams the n rows through the ring, loads kDsAhead rows ahead of the stores.
            // Step j: store row j - kDsAhead from its stage, then load row j into stage (j mod S) once the
            // store of row j - S (issued at step j - S + kDsAhead, followed by S - kDsAhead newer store
            // groups) has read it.
            const uint32_t base = nload;
            for (int j = 0; j < n + kDsAhead; ++j) {
                const int jj = j - kDsAhead;
                const int64_t tj = __shfl_sync(0xffffffffu, tok, j < n ? j : 0);
                const int64_t rwj = __shfl_sync(0xffffffffu, row, jj >= 0 ? jj : 0);
                const int rkj = __shfl_sync(0xffffffffu, rk, jj >= 0 ? jj : 0);
                if (lane == 0) {
                    if (jj >= 0) {
                        const uint32_t q = (base + (uint32_t)jj) % kDsStages;
                        mbar_wait(bar0 + 8 * q, ((base + (uint32_t)jj) / kDsStages) & 1u);
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                                     :: "l"(recv_q[rkj] + rwj * ld_rq), "r"(ring + q * rowb), "r"((uint32_t)K) : "memory");
                        bulk_commit_group();
                    }
                    if (j < n) {
                        const uint32_t q = (base + (uint32_t)j) % kDsStages;
                        bulk_wait_group_read<kDsStages - kDsAhead>();
                        mbar_arrive_expect_tx(bar0 + 8 * q, (uint32_t)K);
                        bulk_load(ring + q * rowb, xq + tj * ldxq, (uint32_t)K, bar0 + 8 * q);
                    }
                }
            }
            nload = base + (uint32_t)n;
            if (lane < n) {                             // scales: lane = entry, one store per contraction block
                float* ds = recv_s[rk] + row;
                for (int64_t kb = 0; kb < KB; ++kb) ds[kb * ld_rs] = xs[kb * ldxs + tok];
            }
        }
        // chunk c: this warp's bulk stores complete (written at the destination), then ordered before
        // the count with the generic proxy at system scope
        if (lane == 0) bulk_wait_group<0>();
        __syncwarp();
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t old = atomicAdd(local_done + c, 1u);
            if (old == gridDim.x - 1u) {                // the last CTA of this rank to finish chunk c
                __threadfence_system();
                for (int o = 0; o < world; ++o) red_release_sys_add(flags[o] + c, 1u);
            }
        }
    }
}

// Token-once dispatch: send entry i = local token tok[i] -> rank dst_rank[i], token-buffer row dst_row[i]
// (codes + row-major scales, as k_dispatch_fp8); each (token, destination rank) pair is sent once.
__global__ void __launch_bounds__(256) k_send_rows(int64_t n, const int64_t* __restrict__ tok, int64_t K, int64_t KB,
                                                   const uint8_t* __restrict__ xq, int64_t ldxq,
                                                   const float* __restrict__ xs, int64_t ldxs,
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
        const int64_t row = dst_row[i], t = tok[i];
        const uint8_t* src = xq + t * ldxq;
        uint8_t* dst = recv_q[r] + row * ld_rq;
        for (int64_t c = (int64_t)lane * 16; c < K; c += 512)
            *reinterpret_cast<uint4*>(dst + c) = ldg_nc_v4(src + c);
        float* ds = recv_s[r] + row * KB;
        for (int64_t kb = lane; kb < KB; kb += 32) ds[kb] = xs[kb * ldxs + t];
    }
}

// Receiver side of the token-once dispatch: expert row i <- token-buffer row idx[i]: the codes (a warp per
// row, 16-byte vectors) and the scales, transposed into the GEMM's [KB][ldsA] layout (lane = row of a
// batch of 32 consecutive rows: 128-byte stores per contraction block).
__global__ void __launch_bounds__(256) k_expand_rows(int64_t R, const int64_t* __restrict__ idx, int64_t K, int64_t KB,
                                                     const uint8_t* __restrict__ tq, int64_t ldtq,
                                                     const float* __restrict__ ts, int64_t ts_rs, int64_t ts_ks,
                                                     uint8_t* __restrict__ A, int64_t lda,
                                                     float* __restrict__ sA, int64_t ldsA) {
    griddep_wait();
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t nb = (R + 31) / 32, nw = (int64_t)gridDim.x * 8;
    for (int64_t b = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); b < nb; b += nw) {
        const int64_t i0 = b * 32;
        const int n = (int)min((int64_t)32, R - i0);
        const int64_t my = lane < n ? idx[i0 + lane] : 0;
        for (int j = 0; j < n; ++j) {
            const int64_t src_row = __shfl_sync(0xffffffffu, my, j);
            const uint8_t* src = tq + src_row * ldtq;
            uint8_t* dst = A + (i0 + j) * lda;
            for (int64_t c = (int64_t)lane * 16; c < K; c += 512)
                *reinterpret_cast<uint4*>(dst + c) = ldg_nc_v4(src + c);
        }
        if (lane < n) {
            const float* s = ts + my * ts_rs;
            for (int64_t kb = 0; kb < KB; ++kb) sA[kb * ldsA + i0 + lane] = s[kb * ts_ks];
        }
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
cudaError_t launch_dispatch_stream(int C, const int64_t* chunk_off, const int64_t* send_tok, const int32_t* send_rank,
                                  const int64_t* send_row, int64_t K, const uint8_t* xq, int64_t ldxq, const float* xs,
                                  int64_t ldxs, uint8_t* const* recv_q, int64_t ld_rq, float* const* recv_s, int64_t ld_rs,
                                  uint32_t* local_done, uint32_t* const* flags, int world, uint32_t epoch, int ctas,
                                  cudaStream_t st) {
    // plain launch (no PDL attribute): it runs concurrently with the GEMM on another stream
    const size_t rowb = (size_t)((K + 127) / 128 * 128);
    const size_t smem = (size_t)kDsWarps * kDsStages * (rowb + 8);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_dispatch_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    // the per-chunk CTA counts start from zero every call (the flags are the monotonic counters)
    cudaError_t e0 = cudaMemsetAsync(local_done, 0, (size_t)C * sizeof(uint32_t), st);
    if (e0 != cudaSuccess) return e0;
    k_dispatch_stream<<<ctas, 32 * kDsWarps, smem, st>>>(C, chunk_off, send_tok, send_rank, send_row, K, K / 128, xq, ldxq,
                                                         xs, ldxs, recv_q, ld_rq, recv_s, ld_rs, local_done, flags, world,
                                                         epoch);
    return cudaPeekAtLastError();
}
cudaError_t launch_send_rows(int64_t n, const int64_t* tok, int64_t K, const uint8_t* xq, int64_t ldxq, const float* xs,
                             int64_t ldxs, const int32_t* dst_rank, const int64_t* dst_row, uint8_t* const* recv_q,
                             int64_t ld_rq, float* const* recv_s, cudaStream_t st) {
    return launch_pdl(k_send_rows, dim3(rows_grid(n)), dim3(256), 0, st, n, tok, K, K / 128, xq, ldxq, xs, ldxs, dst_rank,
                      dst_row, recv_q, ld_rq, recv_s);
}
cudaError_t launch_expand_rows(int64_t R, const int64_t* idx, int64_t K, const uint8_t* tq, int64_t ldtq, const float* ts,
                               int64_t ts_rs, int64_t ts_ks, uint8_t* A, int64_t lda, float* sA, int64_t ldsA,
                               cudaStream_t st) {
    return launch_pdl(k_expand_rows, dim3(rows_grid((R + 31) / 32)), dim3(256), 0, st, R, idx, K, K / 128, tq, ldtq, ts,
                      ts_rs, ts_ks, A, lda, sA, ldsA);
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
