// gemm_mx.cu — block-scaled FP8 GEMM for POWER-OF-TWO scales on the tensor core's own block scaling
// (PAPER.md P:558 / P:565 "integral power of 2" scales, P:659-660 where the
// paper asks hardware to take the scaling into the MMA).
//
//   D[i,j] (+)= sum_kb sA(kb,i) * sB(kb,j) * sum_{c in kb} dec(A[i,c]) dec(B[j,c])
//
// with every sA, sB an exact power of two in [2^-127, 2^127] (fp8bs_quantize_act_1x128_pow2, the pow2
// requantization, or any caller-made pow2 scales).  A power of two is exactly a UE8M0 scale factor
// (the FP32 biased exponent), so tcgen05.mma.kind::mxf8f6f4.block_scale applies sA * sB inside the
// tensor core (one scale byte per row / column per 32-element K-step, our per-128 scale repeated 4x)
// and the FP32 accumulator stays in TMEM for the whole K loop: there is no promotion step.
//
// One CTA per 128 x 224 output tile (persistent):
//   w0  TMA producer: A (128 x 128 B) and B (224 x 128 B) K-blocks into a 4-stage ring;
//   w1, w3, w8, w9  scale-factor producers, one per ring stage (a warp's K-blocks are a ring cycle
//       apart, so its parity waits never alias and its global scale loads, issued before the wait,
//       have a whole cycle to land): per K-block the UE8M0 atoms in the stage (SFA: 32 lanes x 16 B,
//       byte [r1][t] = row l + 32 r1; SFB the same for columns, two atoms) from the FP32 scales;
//   w2  MMA issuer: tcgen05.cp.32x128b.warpx4 of the three atoms into TMEM, then 4 block-scaled MMAs
//       (K = 32, sf_id = K-step) into one of two 224-column accumulators; commits release the stage
//       and, after the last K-block, hand the accumulator to the epilogue (tools/mx_probe.cu pins the
//       scale-factor TMEM layout: row l + 32 r1 -> lane l of every quadrant, column + r1, byte t);
//   w4..w7 epilogue: each drains its lane quadrant (32 rows x 224 columns) in 32-column chunks through
//       a staging buffer and TMA stores (reduce-add for Wgrad accumulate), then frees the accumulator.
// TMEM: 2 x 224 accumulator columns + 12 scale-factor columns (512 allocated).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "sm100.cuh"
#include "internal.h"

namespace fp8bs {
namespace mx {

constexpr int BM = 128, BN = 224, BK = 128;
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK;                 // 16 KB
constexpr int B_BYTES = BN * BK;                 // 28 KB
constexpr int SF_BYTES = 3 * 512;                // SFA atom + 2 SFB atoms
constexpr int STAGE = ((A_BYTES + B_BYTES + SF_BYTES + 1023) / 1024) * 1024;
constexpr int EPI_WARP = 2 * 32 * 128;           // two 32 rows x 128 B staging buffers per epilogue warp
constexpr int OFF_EPI = STAGES * STAGE;
constexpr int OFF_BAR = OFF_EPI + 4 * EPI_WARP;
constexpr int NBAR = 2 * STAGES + 4;             // full, empty, accfull[2], accempty[2]
constexpr int SMEM = 1024 + OFF_BAR + NBAR * 8 + 16;
constexpr int NSF = STAGES;                      // scale-factor warps 1, 3, 8, 9: warp k owns stage k
constexpr int THREADS = 32 * 10;
constexpr uint32_t ACC_COLS = 256;               // accumulator b at columns [256 b, 256 b + 224)
constexpr uint32_t SF_COL = 480;                 // SFA [480, 484), SFB [484, 492)

struct Params {
    int M, N, K, KB, num_m, num_n, layout, n_fast;
    const float* sA; int64_t ldsA;
    const float* sB; int64_t ldsB;
    int accumulate;
};

// Tile order: the operand with fewer rows stays L2-resident while the other streams once (m fastest
// when M <= N; n fastest otherwise, e.g. Wgrad's 18432 x 7168).
__device__ __forceinline__ int tile_m(const Params& p, int t) { return p.n_fast ? t / p.num_n : t % p.num_m; }
__device__ __forceinline__ int tile_n(const Params& p, int t) { return p.n_fast ? t % p.num_n : t / p.num_m; }

__device__ __forceinline__ uint32_t ue8m0(float s) { return (__float_as_uint(s) >> 23) & 0xFFu; }

__device__ __forceinline__ float scale_b(const Params& p, int kb, int j) {
    if (p.layout == 0) return __ldg(p.sB + (int64_t)(j >> 7) * p.ldsB + kb);     // FPROP: [N/128][K/128]
    if (p.layout == 1) return __ldg(p.sB + (int64_t)kb * p.ldsB + (j >> 7));     // DGRAD: [K/128][N/128]
    return __ldg(p.sB + (int64_t)kb * p.ldsB + j);                               // WGRAD: [K/128][N]
}

// tcgen05.cp source descriptor: 32 rows x 16 B atom, no swizzle, 8-row core matrices 128 B apart
__device__ __forceinline__ uint64_t cp_desc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void tmem_cp_atom(uint32_t taddr, uint64_t desc) {
    asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" :: "r"(taddr), "l"(desc) : "memory");
}
// block-scaled instruction descriptor (E4M3 x E4M3, FP32 accumulate, UE8M0 scales)
__host__ __device__ constexpr uint32_t idesc_mx(uint32_t m, uint32_t n, uint32_t sf_id) {
    return (sf_id << 4) | ((n >> 3) << 17) | (1u << 23) | ((m >> 4) << 24) | (sf_id << 29);
}
__device__ __forceinline__ void mma_mx(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa, uint32_t sfb, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
                 :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}

template <bool kOutF32>
__global__ void __launch_bounds__(THREADS, 1)
k_gemm_mx(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
          const __grid_constant__ CUtensorMap tmD, const Params p) {
    extern __shared__ uint8_t smem_raw[];
    griddep_wait();                 // PDL: previous grid complete, its writes visible
    griddep_launch_dependents();
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + OFF_BAR;
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
    auto accfull_bar = [&](int b) { return bar0 + 8u * (2 * STAGES + b); };
    auto accempty_bar = [&](int b) { return bar0 + 8u * (2 * STAGES + 2 + b); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + NBAR * 8);
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(full_bar(s), 2); mbar_init(empty_bar(s), 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(accfull_bar(b), 1); mbar_init(accempty_bar(b), 4); }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<512>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int ntiles = p.num_m * p.num_n;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); tma_prefetch_desc(&tmD); }
        int it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int m0 = tile_m(p, t) * BM, n0 = tile_n(p, t) * BN;
            for (int kb = 0; kb < p.KB; ++kb, ++it) {
                const int s = it % STAGES;
                mbar_wait(empty_bar(s), ((it / STAGES) & 1) ^ 1);
                if (elect_one()) {
                    const uint32_t st = sbase + s * STAGE;
                    mbar_arrive_expect_tx(full_bar(s), A_BYTES + B_BYTES);
                    tma_load_2d(st, &tmA, full_bar(s), kb * BK, m0);
                    tma_load_2d(st + A_BYTES, &tmB, full_bar(s), kb * BK, n0);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1 || warp == 3 || warp >= 8) {
        // ---------------- scale-factor atoms ----------------
        const int slot = warp == 1 ? 0 : warp == 3 ? 1 : warp - 6;
        // this warp's K-blocks: global iteration it = slot, slot + NSF, ... (tile it / KB of this CTA's
        // sequence, K-block it % KB); the scale values of the next one are loaded while the current
        // one waits for its stage, so each load has two ring cycles to land
        auto load = [&](int it, uint32_t* wa, uint32_t* wb) -> bool {
            const int t = blockIdx.x + (it / p.KB) * gridDim.x, kb = it % p.KB;
            if (t >= ntiles) return false;
            const int m0 = tile_m(p, t) * BM, n0 = tile_n(p, t) * BN;
#pragma unroll
            for (int r1 = 0; r1 < 4; ++r1) {
                const int i = m0 + lane + 32 * r1;
                wa[r1] = i < p.M ? ue8m0(__ldg(p.sA + (int64_t)kb * p.ldsA + i)) * 0x01010101u : 127u * 0x01010101u;
            }
#pragma unroll
            for (int r1 = 0; r1 < 8; ++r1) {
                const int j = n0 + lane + 32 * r1;
                wb[r1] = (r1 < BN / 32 && j < p.N) ? ue8m0(scale_b(p, kb, j)) * 0x01010101u : 127u * 0x01010101u;
            }
            return true;
        };
        uint32_t wa[4], wb[8], na[4], nb[8];
        bool have = load(slot, wa, wb);
        for (int it = slot; have; it += NSF) {
            const bool more = load(it + NSF, na, nb);          // in flight during the wait below
            const int s = it % STAGES;
            uint8_t* sf = smem + s * STAGE + A_BYTES + B_BYTES;
            mbar_wait(empty_bar(s), ((it / STAGES) & 1) ^ 1);
            *reinterpret_cast<uint4*>(sf + lane * 16) = make_uint4(wa[0], wa[1], wa[2], wa[3]);
            *reinterpret_cast<uint4*>(sf + 512 + lane * 16) = make_uint4(wb[0], wb[1], wb[2], wb[3]);
            *reinterpret_cast<uint4*>(sf + 1024 + lane * 16) = make_uint4(wb[4], wb[5], wb[6], wb[7]);
            fence_proxy_async_smem();                       // generic writes -> the async proxy (tcgen05.cp)
            __syncwarp();
            if (lane == 0) mbar_arrive(full_bar(s));
#pragma unroll
            for (int r = 0; r < 4; ++r) wa[r] = na[r];
#pragma unroll
            for (int r = 0; r < 8; ++r) wb[r] = nb[r];
            have = more;
        }
    } else if (warp == 2) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc0 = idesc_mx(BM, BN, 0);
        int it = 0, tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            const int b = tl & 1;
            mbar_wait(accempty_bar(b), ((tl >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d = tmem_base + ACC_COLS * b;
            for (int kb = 0; kb < p.KB; ++kb, ++it) {
                const int s = it % STAGES;
                mbar_wait(full_bar(s), (it / STAGES) & 1);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t st = sbase + s * STAGE;
                    const uint32_t sf = st + A_BYTES + B_BYTES;
                    tmem_cp_atom(tmem_base + SF_COL, cp_desc(sf));
                    tmem_cp_atom(tmem_base + SF_COL + 4, cp_desc(sf + 512));
                    tmem_cp_atom(tmem_base + SF_COL + 8, cp_desc(sf + 1024));
                    const uint64_t ad = sdesc_k_sw128(st), bd = sdesc_k_sw128(st + A_BYTES);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t id = idesc0 | ((uint32_t)k << 4) | ((uint32_t)k << 29);
                        mma_mx(d, ad + 2 * k, bd + 2 * k, id, tmem_base + SF_COL + ((uint32_t)k << 30),
                               tmem_base + SF_COL + 4 + ((uint32_t)k << 30), (kb > 0 || k > 0) ? 1u : 0u);
                    }
                    mma_commit(empty_bar(s));
                    if (kb == p.KB - 1) mma_commit(accfull_bar(b));
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue ----------------
        const int quad = warp & 3;
        const uint32_t ebuf0 = sbase + OFF_EPI + (warp - 4) * EPI_WARP;
        int chunk = 0;                                  // running chunk count: alternates the two buffers
        int tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            const int b = tl & 1;
            const int m0 = tile_m(p, t) * BM, n0 = tile_n(p, t) * BN;
            mbar_wait(accfull_bar(b), (tl >> 1) & 1);
            tc_fence_after();
            const uint32_t ta = tmem_base + ((uint32_t)(quad * 32) << 16) + ACC_COLS * b;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c, ++chunk) {
                const uint32_t ebuf = ebuf0 + (chunk & 1) * (32 * 128);
                uint32_t v[32];
                FP8BS_TMEM_LD32(ta + 32 * c, v);
                tmem_ld_wait();
                if (c == BN / 32 - 1) {              // the accumulator is in registers: free it
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(accempty_bar(b));
                }
                if (lane == 0) bulk_wait_group_read<1>();   // the store that last used this buffer has read it
                __syncwarp();
                if constexpr (kOutF32) {
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        sts_u32x4(ebuf + lane * 128 + ((u ^ (lane & 7)) << 4), v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        uint32_t w[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(v[8 * u + 2 * q]), __uint_as_float(v[8 * u + 2 * q + 1]));
                            w[q] = *reinterpret_cast<uint32_t*>(&b2);
                        }
                        sts_u32x4(ebuf + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4), w[0], w[1], w[2], w[3]);
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    const int col = n0 + 32 * c, row = m0 + quad * 32;
                    if (col < p.N && row < p.M) {
                        if (kOutF32 && p.accumulate) tma_reduce_add_2d(&tmD, ebuf, col, row);
                        else tma_store_2d(&tmD, ebuf, col, row);
                    }
                    bulk_commit_group();
                }
            }
        }
        if (lane == 0) bulk_wait_group<0>();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

}  // namespace mx

cudaError_t launch_gemm_mx(const GemmArgs& a, cudaStream_t st, const char** detail) {
    using namespace mx;
    const int KB = (int)(a.K / BK);
    CUtensorMap tA, tB, tD;
    {
        const uint64_t dims[2] = {(uint64_t)a.K, (uint64_t)a.M};
        const uint64_t str[1] = {(uint64_t)a.lda};
        const uint32_t box[2] = {BK, BM};
        if (!make_tmap(&tA, TMAP_U8, 2, a.A, dims, str, box, 128)) { *detail = "tensor map A"; return cudaErrorInvalidValue; }
    }
    {
        const uint64_t dims[2] = {(uint64_t)a.K, (uint64_t)a.N};
        const uint64_t str[1] = {(uint64_t)a.ldb};
        const uint32_t box[2] = {BK, BN};
        if (!make_tmap(&tB, TMAP_U8, 2, a.B, dims, str, box, 128)) { *detail = "tensor map B"; return cudaErrorInvalidValue; }
    }
    {
        // 32 rows x 32 columns per store: FP32 128 B (SWIZZLE_128B staging), BF16 64 B (SWIZZLE_64B)
        const uint64_t esz = a.out_f32 ? 4 : 2;
        const uint64_t dims[2] = {(uint64_t)a.N, (uint64_t)a.M};
        const uint64_t str[1] = {(uint64_t)a.ldd * esz};
        const uint32_t box[2] = {32, 32};
        if (!make_tmap(&tD, a.out_f32 ? TMAP_F32 : TMAP_BF16, 2, a.D, dims, str, box, a.out_f32 ? 128 : 64)) {
            *detail = "tensor map D"; return cudaErrorInvalidValue;
        }
    }
    Params p{};
    p.M = (int)a.M; p.N = (int)a.N; p.K = (int)a.K; p.KB = KB;
    p.num_m = (int)((a.M + BM - 1) / BM); p.num_n = (int)((a.N + BN - 1) / BN);
    p.n_fast = 0;   // m fastest for every shape: n-fastest measured slower for Wgrad (1156 vs 1216 TFLOP/s)
    p.layout = a.layout; p.sA = a.sA; p.ldsA = a.ldsA; p.sB = a.sB; p.ldsB = a.ldsB; p.accumulate = a.accumulate;
    const int64_t tiles = (int64_t)p.num_m * p.num_n;
    const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    auto kern = a.out_f32 ? k_gemm_mx<true> : k_gemm_mx<false>;
    static bool attr[2][64] = {{false}};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[a.out_f32 ? 1 : 0][dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) attr[a.out_f32 ? 1 : 0][dev] = true;
    }
    return launch_pdl(kern, dim3(grid), dim3(THREADS), SMEM, st, tA, tB, tD, p);
}

}  // namespace fp8bs
