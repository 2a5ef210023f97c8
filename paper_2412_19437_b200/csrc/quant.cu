// quant.cu — online fine-grained FP8 quantizers (§3.3.2):
//   1x128 tiles for activations, 128x1 (transposed) tiles for Wgrad operands,
//   128x128 blocks for weights.  All are HBM-bound: one read of the input, one write of the codes
//   (+ 1/128 or 1/16384 of scales).  Per group: amax (maxNum over |x|, warp shuffles), s = amax/448
//   (IEEE division), then per element RN32(x/s) (Markstein sequence) and cvt.rn.satfinite.e4m3x2.
#include <cuda.h>

#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "sm100.cuh"
#include "internal.h"

namespace fp8bs {

template <typename T> struct Vec;
template <> struct Vec<__nv_bfloat16> {
    static constexpr int E = 8;   // elements per 16-byte chunk
    __device__ static void unpack(const uint4& v, float* f) {
        f[0] = bf16_lo(v.x); f[1] = bf16_hi(v.x); f[2] = bf16_lo(v.y); f[3] = bf16_hi(v.y);
        f[4] = bf16_lo(v.z); f[5] = bf16_hi(v.z); f[6] = bf16_lo(v.w); f[7] = bf16_hi(v.w);
    }
};
template <> struct Vec<float> {
    static constexpr int E = 4;
    __device__ static void unpack(const uint4& v, float* f) {
        f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
        f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
    }
};

__device__ __forceinline__ uint4 ld_stream16(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <typename T>
__device__ __forceinline__ float load_scalar(const T* p) {
    if constexpr (sizeof(T) == 2) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
    else return *reinterpret_cast<const float*>(p);
}

// E codes of one 16-byte chunk, packed little-endian (element 0 in the lowest byte).  `fast` is
// uniform per group, so the branch is taken once per chunk (not per element): the fast path is
// the packed Markstein quotient, the slow path (tiny / huge scales, reading R2) IEEE division.
template <int E>
__device__ __forceinline__ void encode_chunk(const float* f, float sc, float r, bool fast, uint32_t* w) {
    if (fast) {
        const float2 r2 = make_float2(r, r), ns2 = make_float2(-sc, -sc);
#pragma unroll
        for (int i = 0; i < E / 4; ++i) {
            const float2 a = div_scale2_fast(make_float2(f[4 * i + 0], f[4 * i + 1]), r2, ns2);
            const float2 b = div_scale2_fast(make_float2(f[4 * i + 2], f[4 * i + 3]), r2, ns2);
            w[i] = cvt_e4m3x2(a.x, a.y) | (cvt_e4m3x2(b.x, b.y) << 16);
        }
    } else {
#pragma unroll
        for (int i = 0; i < E / 4; ++i) {
            const uint32_t lo = cvt_e4m3x2(__fdiv_rn(f[4 * i + 0], sc), __fdiv_rn(f[4 * i + 1], sc));
            const uint32_t hi = cvt_e4m3x2(__fdiv_rn(f[4 * i + 2], sc), __fdiv_rn(f[4 * i + 3], sc));
            w[i] = lo | (hi << 16);
        }
    }
}

// ===========================================================================================
// 1x128: a group of L = 128/E lanes owns one tile (16 lanes x 8 BF16, or 32 lanes x 4 FP32).
// Work unit = (row m, chunk of TPW*U consecutive tiles); units are row-major so consecutive
// warps stream consecutive bytes.  U independent 16-byte loads per lane are in flight.
// ===========================================================================================
template <typename T, int U>
__global__ void __launch_bounds__(256)
k_quant_act_1x128(const T* __restrict__ x, int64_t M, int64_t K, int64_t ldx,
                  uint8_t* __restrict__ q, int64_t ldq, float* __restrict__ s, int64_t lds) {
    constexpr int E = Vec<T>::E;
    constexpr int L = 128 / E;
    constexpr int TPW = 32 / L;
    constexpr int TPU = TPW * U;                       // tiles per unit
    const int lane = threadIdx.x & 31;
    const int sub = lane / L, li = lane % L;
    const int64_t KB = (K + 127) >> 7;
    const int64_t CPR = (KB + TPU - 1) / TPU;          // units per row
    const int64_t nunits = M * CPR;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); u < nunits; u += nwarps) {
        const int64_t m = u / CPR;
        const int64_t kbase = (u - m * CPR) * TPU;
        const T* xr = x + m * ldx;
        uint4 v[U];
        bool ok[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int64_t kb = kbase + j * TPW + sub;
            const int64_t col = kb * 128 + li * E;
            ok[j] = (kb < KB) && (col < K);
            v[j] = ok[j] ? ld_stream16(xr + col) : make_uint4(0, 0, 0, 0);
        }
        // all shuffle reductions first (convergent), then the per-tile encode
        float sc[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            float f[E];
            Vec<T>::unpack(v[j], f);
            float amax = 0.0f;
#pragma unroll
            for (int e = 0; e < E; ++e) amax = fmaxf(amax, fabsf(f[e]));
#pragma unroll
            for (int o = L / 2; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            sc[j] = group_scale(amax);
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            float f[E];
            Vec<T>::unpack(v[j], f);
            const float r = __frcp_rn(sc[j]);
            uint32_t w[E / 4];
            encode_chunk<E>(f, sc[j], r, fast_div_ok(sc[j]), w);
            const int64_t kb = kbase + j * TPW + sub;
            if (ok[j]) {
                uint8_t* dst = q + m * ldq + kb * 128 + li * E;
                if constexpr (E == 8) *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
                else *reinterpret_cast<uint32_t*>(dst) = w[0];
                if (li == 0) s[kb * lds + m] = sc[j];
            }
        }
    }
}

// ===========================================================================================
// 1x128, streamed with TMA bulk copies (fast path: contiguous rows, K % 128 == 0, ldq == K).
// The input is then a flat sequence of T = M*KB tiles.  One producer warp streams 16 KB chunks
// of tiles with cp.async.bulk into a 6-stage shared-memory ring (mbarrier full/empty); 8
// consumer warps encode from shared memory and store codes/scales directly.  Memory traffic is
// decoupled from the encode arithmetic, so up to 192 KB per SM stays in flight.
// ===========================================================================================
#ifndef FP8BS_Q1_EL
#define FP8BS_Q1_EL 32   // BF16 elements per consumer lane (16: 8 lanes per tile)
#endif
template <typename T>
struct Q1Cfg {
    // elements per lane: BF16 32 (4 lanes per tile: the per-group scale work — shuffles, the scale
    // division, its reciprocal — is shared by 32 elements, which keeps the kernel HBM-bound at the
    // ~1.4 GHz a preceding GEMM leaves the SMs at); FP32 16
    static constexpr int EL = sizeof(T) == 2 ? FP8BS_Q1_EL : 16;
    static constexpr int L = 128 / EL;
    static constexpr int VEC = EL * (int)sizeof(T) / 16;    // 16-byte smem loads per lane: 4 / 4
    static constexpr int TILE_BYTES = 128 * (int)sizeof(T);
#ifndef FP8BS_Q1_WARPS
#define FP8BS_Q1_WARPS 16
#endif
    // 16 consumer warps (BF16, 32 per lane: 128 tiles = 32 KB per stage, 3 stages).  Measured on C4's
    // 65536 x 7168 (tools/quant_instep.py, same box, GB/s alone at 1965 MHz / right after the grouped
    // GEMM at its power-capped clock): 16 per lane x 16 warps 6035 / 4189-4375; 32 per lane x 16 warps
    // 5461 / 4969-5230; 32 x 8 warps 5297 / 4636-4725; 32 contiguous x 8 warps 6195 / 4113-4165.  The
    // step's quantizer runs right after the GEMM, so the second column decides.
    static constexpr int CONSUMERS = FP8BS_Q1_WARPS;
    // BF16, 32 per lane: lane li of a tile takes the 16-byte chunks li, li + L, ... (2-way shared-memory
    // bank conflicts like the 16-per-lane contiguous split; contiguous 64-byte runs would be 4-way)
#ifndef FP8BS_Q1_INTERLEAVE
#define FP8BS_Q1_INTERLEAVE 1
#endif
    static constexpr bool INTERLEAVED = FP8BS_Q1_INTERLEAVE && sizeof(T) == 2 && EL == 32;
    static constexpr int TILES_PER_PASS = CONSUMERS * (32 / L);    // 64
    static constexpr int PASSES = 1;
    static constexpr int CHUNK_TILES = TILES_PER_PASS * PASSES;
    static constexpr int CHUNK_BYTES = CHUNK_TILES * TILE_BYTES;   // 16 KB (BF16) / 32 KB (FP32)
    static constexpr int STAGES = 98304 / CHUNK_BYTES;             // 96 KB ring: 2 CTAs per SM
    static constexpr int THREADS = 32 * (CONSUMERS + 1);
    static constexpr int SMEM = STAGES * CHUNK_BYTES + 2 * STAGES * 8;
};

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

template <typename T, bool kPow2 = false>
__global__ void __launch_bounds__(Q1Cfg<T>::THREADS)
k_quant_act_1x128_tma(const T* __restrict__ x, int64_t M, int64_t K, uint8_t* __restrict__ q,
                      float* __restrict__ s, int64_t lds) {
    using C = Q1Cfg<T>;
    extern __shared__ __align__(128) uint8_t smem[];
    griddep_wait();                 // PDL: previous grid complete, its writes visible
    griddep_launch_dependents();
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + C::STAGES * C::CHUNK_BYTES;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < C::STAGES; ++i) { mbar_init(bar0 + 8 * i, 1); mbar_init(bar0 + 8 * (C::STAGES + i), C::CONSUMERS); }
        fence_mbar_init();
    }
    __syncthreads();
    const int KB = (int)(K >> 7);
    const int NT = (int)(M * KB);                            // < 2^31 (host-checked)
    const int nchunks = (NT + C::CHUNK_TILES - 1) / C::CHUNK_TILES;
    if (warp == C::CONSUMERS) {
        // ---------------- producer ----------------
        if (lane == 0) {
            int it = 0;
            for (int c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
                const int st = it % C::STAGES;
                mbar_wait(bar0 + 8 * (C::STAGES + st), ((it / C::STAGES) & 1) ^ 1);
                const int t0 = c * C::CHUNK_TILES;
                const uint32_t bytes = (uint32_t)min(C::CHUNK_TILES, NT - t0) * C::TILE_BYTES;
                mbar_arrive_expect_tx(bar0 + 8 * st, bytes);
                bulk_load(sbase + st * C::CHUNK_BYTES, reinterpret_cast<const uint8_t*>(x) + (int64_t)t0 * C::TILE_BYTES,
                          bytes, bar0 + 8 * st);
            }
        }
        return;
    }
    // ---------------- consumers: lane = (tile slot, 16-element slice) ----------------
    const int sub = lane / C::L, li = lane % C::L;
    int it = 0;
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int st = it % C::STAGES;
        mbar_wait(bar0 + 8 * st, (it / C::STAGES) & 1);
        const int t0 = c * C::CHUNK_TILES;
        const int ntl = min(C::CHUNK_TILES, NT - t0);
#pragma unroll
        for (int pass = 0; pass < C::PASSES; ++pass) {
            const int d = pass * C::TILES_PER_PASS + warp * (32 / C::L) + sub;   // tile within the chunk
            const bool ok = d < ntl;
            float f[C::EL];
#pragma unroll
            for (int v = 0; v < C::VEC; ++v) {
                const int cb = C::INTERLEAVED ? (li + C::L * v) * 16 : li * (C::EL * (int)sizeof(T)) + v * 16;
                const uint4 u = ok ? lds128(sbase + st * C::CHUNK_BYTES + d * C::TILE_BYTES + cb)
                                   : make_uint4(0, 0, 0, 0);
                Vec<T>::unpack(u, f + v * Vec<T>::E);
            }
            float amax = 0.0f;
#pragma unroll
            for (int e = 0; e < C::EL; ++e) amax = fmaxf(amax, fabsf(f[e]));
#pragma unroll
            for (int o = C::L / 2; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            const float sc = group_scale_t<kPow2>(amax);
            const float r = __frcp_rn(sc);
            uint32_t w[C::EL / 4];
            if (__all_sync(0xffffffffu, fast_div_ok(sc))) {                                     // warp-uniform
#pragma unroll
                for (int hh = 0; hh < C::EL / 16; ++hh) encode_chunk<16>(f + 16 * hh, sc, r, true, w + 4 * hh);
            } else {
#pragma unroll
                for (int hh = 0; hh < C::EL / 16; ++hh) encode_chunk<16>(f + 16 * hh, sc, r, false, w + 4 * hh);
            }
            if (ok) {
                const int t = t0 + d;
                if constexpr (C::INTERLEAVED) {             // chunk li + L*v: 8 codes at (li + L*v) * 8
#pragma unroll
                    for (int v = 0; v < C::VEC; ++v)
                        *reinterpret_cast<uint2*>(q + (int64_t)t * 128 + (li + C::L * v) * 8) = make_uint2(w[2 * v], w[2 * v + 1]);
                } else {
#pragma unroll
                    for (int hh = 0; hh < C::EL / 16; ++hh)
                        *reinterpret_cast<uint4*>(q + (int64_t)t * 128 + li * C::EL + 16 * hh) =
                            make_uint4(w[4 * hh], w[4 * hh + 1], w[4 * hh + 2], w[4 * hh + 3]);
                }
                if (li == 0) {
                    const int m = t / KB, kb = t - m * KB;
                    s[(int64_t)kb * lds + m] = sc;
                }
            }
        }
        // the stage was written by TMA (async proxy) and read with ld.shared (generic proxy): a proxy
        // fence keeps the producer's next TMA into it behind these reads (an mbarrier arrive alone
        // does not; see gemm.cu release_scales)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar0 + 8 * (C::STAGES + st));
    }
}

// ===========================================================================================
// 128x1 transpose-quantize.  CTA tile = 128 tokens x CH channels (CH*sizeof(T) = 256 B per row).
// Phase 1: coalesced 16-byte loads into smem.  Phase 2: TPC threads per channel reduce the
// column amax and encode their rows, staging codes per channel in smem.  Phase 3: each
// channel's 128 codes are written as one contiguous 128-byte row of qT.
// ===========================================================================================
template <typename T>
struct T128x1 {
    static constexpr int E = Vec<T>::E;
    static constexpr int CH = 256 / sizeof(T);          // 128 BF16 / 64 FP32 channels
    static constexpr int CPR = CH / E;                  // 16-byte chunks per row = 16
    static constexpr int TPC = 256 / CH;                // threads per channel: 2 / 4
    static constexpr int RPT = 128 / TPC;               // rows per thread: 64 / 32
    static constexpr int QSTR = 144;                    // staged code row stride (conflict-free v4)
    static constexpr size_t SMEM = 128 * 256 + CH * QSTR + TPC * CH * 4;
};

template <typename T>
__global__ void __launch_bounds__(256)
k_quant_act_128x1(const T* __restrict__ x, int64_t M, int64_t C, int64_t ldx,
                  uint8_t* __restrict__ qT, int64_t ldq, float* __restrict__ sT, int64_t lds) {
    using P = T128x1<T>;
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* xs = smem;                                  // [128][256 B]
    uint8_t* qs = smem + 128 * 256;                      // [CH][QSTR]
    float* red = reinterpret_cast<float*>(qs + P::CH * P::QSTR);   // [TPC][CH]
    const int tid = threadIdx.x;
    const int64_t MB = (M + 127) >> 7, NCB = (C + P::CH - 1) / P::CH;
    const int64_t ntiles = MB * NCB;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t mb = t / NCB, cb = t - mb * NCB;
        const int64_t m0 = mb * 128, c0 = cb * P::CH;
        // phase 1
        uint4 v[128 * P::CPR / 256];
#pragma unroll
        for (int i = 0; i < 128 * P::CPR / 256; ++i) {
            const int idx = i * 256 + tid, r = idx / P::CPR, ck = idx % P::CPR;
            const int64_t col = c0 + ck * P::E;
            const bool ok = (m0 + r < M) && (col < C);
            v[i] = ok ? ld_stream16(x + (m0 + r) * ldx + col) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < 128 * P::CPR / 256; ++i) {
            const int idx = i * 256 + tid, r = idx / P::CPR, ck = idx % P::CPR;
            *reinterpret_cast<uint4*>(xs + r * 256 + ck * 16) = v[i];
        }
        __syncthreads();
        // phase 2
        const int ch = tid % P::CH, part = tid / P::CH;
        const int r0 = part * P::RPT;
        float amax = 0.0f;
#pragma unroll 8
        for (int r = r0; r < r0 + P::RPT; ++r)
            amax = fmaxf(amax, fabsf(load_scalar<T>(reinterpret_cast<const T*>(xs + r * 256) + ch)));
        red[part * P::CH + ch] = amax;
        __syncthreads();
#pragma unroll
        for (int p = 0; p < P::TPC; ++p) amax = fmaxf(amax, red[p * P::CH + ch]);
        const float sc = group_scale(amax);
        const float rc = __frcp_rn(sc);
        const bool fast = fast_div_ok(sc);
#pragma unroll
        for (int r = r0; r < r0 + P::RPT; r += 16) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                float f[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) f[e] = load_scalar<T>(reinterpret_cast<const T*>(xs + (r + 4 * i + e) * 256) + ch);
                encode_chunk<4>(f, sc, rc, fast, &w[i]);
            }
            *reinterpret_cast<uint4*>(qs + ch * P::QSTR + r) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        if (part == 0 && c0 + ch < C) sT[mb * lds + c0 + ch] = sc;
        __syncthreads();
        // phase 3
#pragma unroll
        for (int i = 0; i < P::CH * 8 / 256; ++i) {
            const int idx = i * 256 + tid, chl = idx >> 3, pk = idx & 7;
            const int64_t c = c0 + chl, m = m0 + pk * 16;
            if (c < C && m < M) {
                const uint4 val = *reinterpret_cast<const uint4*>(qs + chl * P::QSTR + pk * 16);
                uint8_t* dst = qT + c * ldq + m;
                if (m + 16 <= M) {
                    *reinterpret_cast<uint4*>(dst) = val;
                } else {
                    const uint8_t* b = reinterpret_cast<const uint8_t*>(&val);
                    for (int e = 0; e < 16 && m + e < M; ++e) dst[e] = b[e];
                }
            }
        }
        __syncthreads();
    }
}

// ===========================================================================================
// 128x1, TMA-streamed (fast path): a producer warp loads 128-token x 256-byte tiles of x with a
// 2-D tensor map into a 3-stage ring (OOB rows/channels zero-filled); 8 consumer warps own one
// 32-bit word column (2 BF16 / 1 FP32 channels) x 32 rows each: column amax via smem across the 4
// row groups, packed Markstein encode of row pairs (cvt of rows r, r+1 gives adjacent code bytes of
// the transposed row directly), codes staged per channel and written as 128-byte rows of qT.
// ===========================================================================================
#ifndef FP8BS_DUAL_UNROLL
#define FP8BS_DUAL_UNROLL 1
#endif
#ifndef FP8BS_DUAL_ROW32
#define FP8BS_DUAL_ROW32 0   // experiment: dual quantizer row pass with 32 elements per lane (C1: X 35.6 -> 36.7 us, dY 75.9 -> 77.2 us: slower)
#endif
constexpr int kDualUnroll = FP8BS_DUAL_UNROLL;   // row passes of the dual quantizer in flight (experiments)
template <typename T>
struct QTCfg {
    static constexpr int CH = 256 / (int)sizeof(T);         // channels per tile: 128 BF16 / 64 FP32
    static constexpr int CPW = 4 / (int)sizeof(T);          // channels per 32-bit word
    static constexpr int TILE_BYTES = 128 * 256;
    static constexpr int STAGES = 2;                        // 84 KB per CTA: two CTAs (16 consumer warps) per SM
    static constexpr int CONSUMERS = 8;
    static constexpr int THREADS = 32 * (CONSUMERS + 1);
    static constexpr int QSTR = 144;
    static constexpr int OFF_Q = STAGES * TILE_BYTES;       // code staging [CH][QSTR]
    static constexpr int OFF_RED = OFF_Q + CH * QSTR;       // partial amax [4][CH]
    static constexpr int OFF_BAR = OFF_RED + 4 * CH * 4;
    static constexpr int SMEM = OFF_BAR + 2 * STAGES * 8;
};

// The dual quantizer's stages: three 32 KB tiles in flight per CTA (two CTAs per SM), the 128x1
// codes staged in the first 18 KB of the tile's own stage once its columns are in registers (the
// stage is released after the copy-out) instead of a separate buffer — measured: with two stages
// plus a separate 18 KB buffer the kernel waited on DRAM latency (4 tiles in flight per SM).
#ifndef FP8BS_DUAL_STAGES
#define FP8BS_DUAL_STAGES 3
#endif
struct QDCfg {
    static constexpr int CH = 128, CPW = 2;                 // BF16: channels per tile, per 32-bit word
    static constexpr int TILE_BYTES = 128 * 256;
    static constexpr int STAGES = FP8BS_DUAL_STAGES;
    static constexpr int CONSUMERS = 8;
    static constexpr int THREADS = 32 * (CONSUMERS + 1);
    static constexpr int QSTR = 144;                        // code staging [CH][QSTR] inside the stage
    static_assert(CH * QSTR <= TILE_BYTES, "codes staged inside the stage");
    static constexpr int OFF_RED = STAGES * TILE_BYTES;     // partial amax [4][CH]
    static constexpr int OFF_BAR = OFF_RED + 4 * CH * 4;
    static constexpr int SMEM = OFF_BAR + 2 * STAGES * 8;
};

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" :: "r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
template <typename T>
__device__ __forceinline__ float word_elem(uint32_t w, int j) {
    if constexpr (sizeof(T) == 2) return j == 0 ? bf16_lo(w) : bf16_hi(w);
    else return __uint_as_float(w);
}


// Column amax of 32 rows x one 32-bit word (2 BF16 channels or 1 FP32 channel) for the 128x1 paths:
// red[j] = maxNum over rows of |x(row, channel j)|.  BF16: packed 3-input max and min over the raw
// words (VHMNMX.BF16_V2, 2 words per instruction; BF16 selection is exact, maxNum ignores NaN like
// fmaxf), then |.| of the two extremes: 0.5 instructions per element instead of an unpack plus a max.
template <typename T>
__device__ __forceinline__ void column_amax(const uint32_t* w, float* red) {
    if constexpr (sizeof(T) == 2) {
        __nv_bfloat162 mx = __floats2bfloat162_rn(0.0f, 0.0f), mn = mx;
#pragma unroll
        for (int r = 0; r < 32; r += 2) {
            const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&w[r]);
            const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&w[r + 1]);
            mx = __hmax2(mx, __hmax2(a, b));
            mn = __hmin2(mn, __hmin2(a, b));
        }
        red[0] = fmaxf(fabsf(__low2float(mx)), fabsf(__low2float(mn)));
        red[1] = fmaxf(fabsf(__high2float(mx)), fabsf(__high2float(mn)));
    } else {
        float a = 0.0f;
#pragma unroll
        for (int r = 0; r < 32; ++r) a = fmaxf(a, fabsf(__uint_as_float(w[r])));
        red[0] = a;
    }
}

// Token-block maps of the 128x1 quantizer: which source rows feed output token block mb.
// Dense: rows [128 mb, 128 mb + 128) (TMA zero-fills past M).  Grouped (expert-aligned layout, R25):
// output block mb lies in expert e's padded range [pad[e], pad[e+1]); its rows start at
// off[e] + 128 mb - pad[e] and only cnt = min(128, off[e+1] - src) of them belong to e (the rest are
// masked to +0, which gives amax-neutral zeros and code 0 in the padding).
struct DenseRows {
    __device__ __forceinline__ void at(int mb, int64_t, int64_t& src, int& cnt) const { src = (int64_t)mb * 128; cnt = 128; }
};
struct GroupRows {
    static constexpr int MAXG = 1024;
    int G;
    int off[MAXG + 1];
    int pad[MAXG + 1];
    __device__ __forceinline__ void at(int mb, int64_t, int64_t& src, int& cnt) const {
        const int m0 = mb * 128;
        int lo = 0, hi = G - 1;               // last e with pad[e] <= m0 (empty experts have pad[e] == pad[e+1])
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pad[mid] <= m0) lo = mid; else hi = mid - 1;
        }
        // lo is non-empty: an empty lo < G-1 has pad[lo+1] == pad[lo] <= m0, so lo+1 would have been chosen
        src = (int64_t)off[lo] + (m0 - pad[lo]);
        const int64_t left = (int64_t)off[lo + 1] - src;
        cnt = left < 128 ? (int)left : 128;
    }
};

template <typename T, class Rows>
__global__ void __launch_bounds__(QTCfg<T>::THREADS, 2)   // 2 CTAs/SM: <= 112 registers
k_quant_act_128x1_tma(const __grid_constant__ CUtensorMap tmX, int64_t M, int64_t C, uint8_t* __restrict__ qT,
                      int64_t ldq, float* __restrict__ sT, int64_t lds, const __grid_constant__ Rows rows) {
    using P = QTCfg<T>;
    extern __shared__ __align__(128) uint8_t smem[];
    griddep_wait();                 // PDL: previous grid complete, its writes visible
    griddep_launch_dependents();
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + P::OFF_BAR;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < P::STAGES; ++i) { mbar_init(bar0 + 8 * i, 1); mbar_init(bar0 + 8 * (P::STAGES + i), P::CONSUMERS); }
        fence_mbar_init();
    }
    __syncthreads();
    const int MB = (int)((M + 127) >> 7), NCB = (int)((C + P::CH - 1) / P::CH);
    const int ntiles = MB * NCB;
    if (warp == P::CONSUMERS) {
        if (lane == 0) {
            tma_prefetch_desc(&tmX);
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const int st = it % P::STAGES;
                mbar_wait(bar0 + 8 * (P::STAGES + st), ((it / P::STAGES) & 1) ^ 1);
                mbar_arrive_expect_tx(bar0 + 8 * st, P::TILE_BYTES);
                int64_t src;
                int cnt;
                rows.at(t / NCB, M, src, cnt);
                tma_load_2d(sbase + st * P::TILE_BYTES, &tmX, bar0 + 8 * st, (t % NCB) * P::CH, (int)src);
            }
        }
        return;
    }
    const int tid = threadIdx.x, wc = tid & 63, rg = tid >> 6;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = it % P::STAGES;
        const int mb = t / NCB, cb = t - mb * NCB;
        const int64_t m0 = (int64_t)mb * 128, c0 = (int64_t)cb * P::CH;
        mbar_wait(bar0 + 8 * st, (it / P::STAGES) & 1);
        uint32_t w[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) w[r] = lds32(sbase + st * P::TILE_BYTES + (rg * 32 + r) * 256 + wc * 4);
        if constexpr (!std::is_same<Rows, DenseRows>::value) {   // rows of the next expert -> +0
            int64_t src;
            int cnt;
            rows.at(mb, M, src, cnt);
#pragma unroll
            for (int r = 0; r < 32; ++r)
                if (rg * 32 + r >= cnt) w[r] = 0u;
        }
        // the stage was written by TMA (async proxy) and read with ld.shared (generic proxy): a proxy
        // fence keeps the producer's next TMA into it behind these reads (an mbarrier arrive alone
        // does not; see gemm.cu release_scales)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar0 + 8 * (P::STAGES + st));     // stage consumed
        float sc[P::CPW];
        column_amax<T>(w, reinterpret_cast<float*>(smem + P::OFF_RED) + rg * P::CH + wc * P::CPW);
        named_bar_sync(1, 32 * P::CONSUMERS);
        bool fast = true;
#pragma unroll
        for (int j = 0; j < P::CPW; ++j) {
            const int ch = wc * P::CPW + j;
            const float* red = reinterpret_cast<const float*>(smem + P::OFF_RED);
            const float a = fmaxf(fmaxf(red[ch], red[P::CH + ch]), fmaxf(red[2 * P::CH + ch], red[3 * P::CH + ch]));
            sc[j] = group_scale(a);
            fast = fast && fast_div_ok(sc[j]);
            if (rg == 0 && c0 + ch < C) sT[(int64_t)mb * lds + c0 + ch] = sc[j];
        }
        fast = __all_sync(0xffffffffu, fast);
#pragma unroll
        for (int j = 0; j < P::CPW; ++j) {
            const float r = __frcp_rn(sc[j]);
            uint32_t code[8];
            if (fast) {
                const float2 r2 = make_float2(r, r), ns2 = make_float2(-sc[j], -sc[j]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float2 a = div_scale2_fast(make_float2(word_elem<T>(w[4 * k], j), word_elem<T>(w[4 * k + 1], j)), r2, ns2);
                    const float2 b = div_scale2_fast(make_float2(word_elem<T>(w[4 * k + 2], j), word_elem<T>(w[4 * k + 3], j)), r2, ns2);
                    code[k] = cvt_e4m3x2(a.x, a.y) | (cvt_e4m3x2(b.x, b.y) << 16);
                }
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    code[k] = cvt_e4m3x2(__fdiv_rn(word_elem<T>(w[4 * k], j), sc[j]), __fdiv_rn(word_elem<T>(w[4 * k + 1], j), sc[j])) |
                              (cvt_e4m3x2(__fdiv_rn(word_elem<T>(w[4 * k + 2], j), sc[j]), __fdiv_rn(word_elem<T>(w[4 * k + 3], j), sc[j])) << 16);
                }
            }
            const uint32_t qa = sbase + P::OFF_Q + (wc * P::CPW + j) * P::QSTR + rg * 32;
            sts128(qa, make_uint4(code[0], code[1], code[2], code[3]));
            sts128(qa + 16, make_uint4(code[4], code[5], code[6], code[7]));
        }
        named_bar_sync(1, 32 * P::CONSUMERS);
#pragma unroll
        for (int i = 0; i < P::CH * 8 / (32 * P::CONSUMERS); ++i) {
            const int idx = i * 32 * P::CONSUMERS + tid, chl = idx >> 3, pk = idx & 7;
            const int64_t c = c0 + chl, m = m0 + pk * 16;
            if (c < C && m < M) {
                const uint4 val = lds128(sbase + P::OFF_Q + chl * P::QSTR + pk * 16);
                uint8_t* dst = qT + c * ldq + m;
                if (m + 16 <= M) {
                    *reinterpret_cast<uint4*>(dst) = val;
                } else {
                    const uint8_t* b = reinterpret_cast<const uint8_t*>(&val);
                    for (int e = 0; e < 16 && m + e < M; ++e) dst[e] = b[e];
                }
            }
        }
    }
}

// ===========================================================================================
// Dual 1x128 + 128x1 activation quantization from ONE read of a BF16 tile (the paper, §3.5.2
// P:672-673, asks for the FP8 cast to be fused with the memory access; a training step needs both
// groupings of X and of dY).  Same TMA ring and 128x1 column path as k_quant_act_128x1_tma; before a
// stage is released the 8 consumer warps also quantize its 128 rows along the channels (a BF16 tile
// is exactly one 128-wide K group per row): 8 lanes per row, 16 elements per lane, shuffle amax,
// 16-byte code stores (128-byte row segments) and one coalesced 512-byte scale vector per tile.
// Outputs are bit-identical to the two separate kernels.
// ===========================================================================================
template <bool kPow2 = false>
__global__ void __launch_bounds__(QDCfg::THREADS, 2)   // 2 CTAs/SM: <= 112 registers
k_quant_act_dual_tma(const __grid_constant__ CUtensorMap tmX, int64_t M, int64_t C,
                     uint8_t* __restrict__ q, int64_t ldq, float* __restrict__ s, int64_t lds,
                     uint8_t* __restrict__ qT, int64_t ldqT, float* __restrict__ sT, int64_t ldsT) {
    using T = __nv_bfloat16;
    using P = QDCfg;
    extern __shared__ __align__(128) uint8_t smem[];
    griddep_wait();                 // PDL: previous grid complete, its writes visible
    griddep_launch_dependents();
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + P::OFF_BAR;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < P::STAGES; ++i) { mbar_init(bar0 + 8 * i, 1); mbar_init(bar0 + 8 * (P::STAGES + i), P::CONSUMERS); }
        fence_mbar_init();
    }
    __syncthreads();
    const int MB = (int)((M + 127) >> 7), NCB = (int)((C + P::CH - 1) / P::CH);
    const int ntiles = MB * NCB;
    if (warp == P::CONSUMERS) {
        if (lane == 0) {
            tma_prefetch_desc(&tmX);
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const int st = it % P::STAGES;
                mbar_wait(bar0 + 8 * (P::STAGES + st), ((it / P::STAGES) & 1) ^ 1);
                mbar_arrive_expect_tx(bar0 + 8 * st, P::TILE_BYTES);
                tma_load_2d(sbase + st * P::TILE_BYTES, &tmX, bar0 + 8 * st, (t % NCB) * P::CH, (t / NCB) * 128);
            }
        }
        return;
    }
    const int tid = threadIdx.x, wc = tid & 63, rg = tid >> 6;
#if FP8BS_DUAL_ROW32
    // row phase: 8 rows per warp pass, 4 lanes per row, 32 elements per lane (the per-row scale work
    // shared by twice the elements, as in k_quant_act_1x128_tma); lane li takes the 16-byte chunks li,
    // li + 4, ... of its row (2-way shared-memory conflicts, like the 8-lane split)
    const int sub = lane >> 2, li = lane & 3;
#else
    const int sub = lane >> 3, li = lane & 7;          // row phase: 4 rows per warp pass, 8 lanes per row
#endif
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = it % P::STAGES;
        const int mb = t / NCB, cb = t - mb * NCB;
        const int64_t m0 = (int64_t)mb * 128, c0 = (int64_t)cb * P::CH;
        const uint32_t tile = sbase + st * P::TILE_BYTES;
        mbar_wait(bar0 + 8 * st, (it / P::STAGES) & 1);
        // Interior tile (all tiles of M, C multiples of 128): stores through per-thread base pointers
        // advanced by constant strides, without per-store bounds arithmetic.
        const bool full = (m0 + 128 <= M) && (c0 + P::CH <= C);
#if FP8BS_DUAL_ROW32
        constexpr int RPW = 8;                                               // rows per warp per pass
#else
        constexpr int RPW = 4;
#endif
        uint8_t* qrow = q + (m0 + warp * RPW + sub) * ldq + c0;              // + pass * 8 * RPW rows
        float* srow = s + (int64_t)cb * lds + m0 + warp * RPW + sub;
        // ---- 1x128 along the channels: rows of the tile ----
#pragma unroll kDualUnroll
        for (int pass = 0; pass < 128 / (RPW * P::CONSUMERS); ++pass) {
            const int row = pass * RPW * P::CONSUMERS + warp * RPW + sub;
#if FP8BS_DUAL_ROW32
            float f[32];
#pragma unroll
            for (int v = 0; v < 4; ++v) Vec<T>::unpack(lds128(tile + row * 256 + (li + 4 * v) * 16), f + 8 * v);
            float amax = 0.0f;
#pragma unroll
            for (int e = 0; e < 32; ++e) amax = fmaxf(amax, fabsf(f[e]));
#pragma unroll
            for (int o = 2; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            const float sc = group_scale_t<kPow2>(amax);
            const float r = __frcp_rn(sc);
            uint32_t w8[8];
            if (__all_sync(0xffffffffu, fast_div_ok(sc))) {                    // warp-uniform
                encode_chunk<16>(f, sc, r, true, w8);
                encode_chunk<16>(f + 16, sc, r, true, w8 + 4);
            } else {
                encode_chunk<16>(f, sc, r, false, w8);
                encode_chunk<16>(f + 16, sc, r, false, w8 + 4);
            }
            if (full) {
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    *reinterpret_cast<uint2*>(qrow + pass * RPW * P::CONSUMERS * ldq + (li + 4 * v) * 8) = make_uint2(w8[2 * v], w8[2 * v + 1]);
                if (li == 0) srow[pass * RPW * P::CONSUMERS] = sc;
            } else {
                const int64_t m = m0 + row;
                if (m < M) {
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const int64_t c = c0 + (li + 4 * v) * 8;
                        if (c < C) *reinterpret_cast<uint2*>(q + m * ldq + c) = make_uint2(w8[2 * v], w8[2 * v + 1]);
                    }
                    if (li == 0) s[(int64_t)cb * lds + m] = sc;
                }
            }
#else
            float f[16];
            Vec<T>::unpack(lds128(tile + row * 256 + li * 32), f);
            Vec<T>::unpack(lds128(tile + row * 256 + li * 32 + 16), f + 8);
            float amax = 0.0f;
#pragma unroll
            for (int e = 0; e < 16; ++e) amax = fmaxf(amax, fabsf(f[e]));
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            const float sc = group_scale_t<kPow2>(amax);
            const float r = __frcp_rn(sc);
            uint32_t w4[4];
            if (__all_sync(0xffffffffu, fast_div_ok(sc))) encode_chunk<16>(f, sc, r, true, w4);   // warp-uniform
            else encode_chunk<16>(f, sc, r, false, w4);
            if (full) {
                *reinterpret_cast<uint4*>(qrow + pass * 32 * ldq + li * 16) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                if (li == 0) srow[pass * 32] = sc;
            } else {
                const int64_t m = m0 + row, c = c0 + li * 16;
                if (m < M) {
                    if (c < C) *reinterpret_cast<uint4*>(q + m * ldq + c) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                    if (li == 0) s[(int64_t)cb * lds + m] = sc;
                }
            }
#endif
        }
        // ---- 128x1 along the tokens: columns of the tile (as k_quant_act_128x1_tma) ----
        uint32_t w[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) w[r] = lds32(tile + (rg * 32 + r) * 256 + wc * 4);
        // (the stage stays held: its first 18 KB stage the 128x1 codes below, after the barrier that
        // follows every thread's column loads; it is released after the copy-out)
        float sc[P::CPW];
        column_amax<T>(w, reinterpret_cast<float*>(smem + P::OFF_RED) + rg * P::CH + wc * P::CPW);
        named_bar_sync(1, 32 * P::CONSUMERS);
        bool fast = true;
#pragma unroll
        for (int j = 0; j < P::CPW; ++j) {
            const int ch = wc * P::CPW + j;
            const float* red = reinterpret_cast<const float*>(smem + P::OFF_RED);
            const float a = fmaxf(fmaxf(red[ch], red[P::CH + ch]), fmaxf(red[2 * P::CH + ch], red[3 * P::CH + ch]));
            sc[j] = group_scale_t<kPow2>(a);
            fast = fast && fast_div_ok(sc[j]);
            if (rg == 0 && (full || c0 + ch < C)) sT[(int64_t)mb * ldsT + c0 + ch] = sc[j];
        }
        fast = __all_sync(0xffffffffu, fast);
#pragma unroll
        for (int j = 0; j < P::CPW; ++j) {
            const float r = __frcp_rn(sc[j]);
            uint32_t code[8];
            if (fast) {
                const float2 r2 = make_float2(r, r), ns2 = make_float2(-sc[j], -sc[j]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float2 a = div_scale2_fast(make_float2(word_elem<T>(w[4 * k], j), word_elem<T>(w[4 * k + 1], j)), r2, ns2);
                    const float2 b = div_scale2_fast(make_float2(word_elem<T>(w[4 * k + 2], j), word_elem<T>(w[4 * k + 3], j)), r2, ns2);
                    code[k] = cvt_e4m3x2(a.x, a.y) | (cvt_e4m3x2(b.x, b.y) << 16);
                }
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    code[k] = cvt_e4m3x2(__fdiv_rn(word_elem<T>(w[4 * k], j), sc[j]), __fdiv_rn(word_elem<T>(w[4 * k + 1], j), sc[j])) |
                              (cvt_e4m3x2(__fdiv_rn(word_elem<T>(w[4 * k + 2], j), sc[j]), __fdiv_rn(word_elem<T>(w[4 * k + 3], j), sc[j])) << 16);
                }
            }
            const uint32_t qa = tile + (wc * P::CPW + j) * P::QSTR + rg * 32;
            sts128(qa, make_uint4(code[0], code[1], code[2], code[3]));
            sts128(qa + 16, make_uint4(code[4], code[5], code[6], code[7]));
        }
        named_bar_sync(1, 32 * P::CONSUMERS);
        if (full) {
            // thread -> channel i * 32 + tid / 8, tokens (tid & 7) * 16 .. + 16 of the tile
            uint8_t* tb = qT + (c0 + (tid >> 3)) * ldqT + m0 + (tid & 7) * 16;
            const uint32_t qs = tile + (tid >> 3) * P::QSTR + (tid & 7) * 16;
#pragma unroll
            for (int i = 0; i < P::CH * 8 / (32 * P::CONSUMERS); ++i)
                *reinterpret_cast<uint4*>(tb + (int64_t)(i * 32) * ldqT) = lds128(qs + i * 32 * P::QSTR);
            // the stage was written by TMA (async proxy) and read with ld.shared (generic proxy): a
            // proxy fence keeps the producer's next TMA into it behind these reads (an mbarrier
            // arrive alone does not; see gemm.cu release_scales)
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar0 + 8 * (P::STAGES + st));     // stage consumed
            continue;
        }
#pragma unroll
        for (int i = 0; i < P::CH * 8 / (32 * P::CONSUMERS); ++i) {
            const int idx = i * 32 * P::CONSUMERS + tid, chl = idx >> 3, pk = idx & 7;
            const int64_t c = c0 + chl, m = m0 + pk * 16;
            if (c < C && m < M) {
                const uint4 val = lds128(tile + chl * P::QSTR + pk * 16);
                uint8_t* dst = qT + c * ldqT + m;
                if (m + 16 <= M) {
                    *reinterpret_cast<uint4*>(dst) = val;
                } else {
                    const uint8_t* b = reinterpret_cast<const uint8_t*>(&val);
                    for (int e = 0; e < 16 && m + e < M; ++e) dst[e] = b[e];
                }
            }
        }
        // the stage was written by TMA (async proxy) and read with ld.shared (generic proxy): a
        // proxy fence keeps the producer's next TMA into it behind these reads (an mbarrier
        // arrive alone does not; see gemm.cu release_scales)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar0 + 8 * (P::STAGES + st));     // stage consumed
    }
}

// ===========================================================================================
// 128x128 weights, TMA-streamed (fast path): one 128x128 block per stage (64 KB FP32 / 32 KB BF16)
// loaded by a producer warp; 16 consumer warps read 16-byte chunks (lane-contiguous, conflict-free),
// block amax via shuffles + smem, codes written row-major straight to global (coalesced 128-byte
// rows); the transposed copy goes through a row-major code tile in smem and 4-row byte gathers.
// ===========================================================================================
template <typename T>
struct QWCfg {
    static constexpr int E = Vec<T>::E;                     // elements per 16-byte chunk
    static constexpr int CPR = 128 / E;                     // chunks per block row
    static constexpr int BLOCK_BYTES = 128 * 128 * (int)sizeof(T);
    static constexpr int STAGES = sizeof(T) == 4 ? 3 : 4;
    static constexpr int CONSUMERS = 16;
    static constexpr int THREADS = 32 * (CONSUMERS + 1);
    static constexpr int NCH = 128 * CPR / (32 * CONSUMERS); // chunks per consumer thread: 8 / 4
    static constexpr int OFF_C = STAGES * BLOCK_BYTES;      // code tile [128][128]
    static constexpr int OFF_RED = OFF_C + 128 * 128;
    static constexpr int OFF_BAR = OFF_RED + 2 * CONSUMERS * 4;   // per-warp amax, double-buffered by block parity
    static constexpr int SMEM = OFF_BAR + 2 * STAGES * 8;
};

template <typename T, bool kPow2 = false>
__global__ void __launch_bounds__(QWCfg<T>::THREADS)
k_quant_weight_tma(const __grid_constant__ CUtensorMap tmW, int64_t N, int64_t K, uint8_t* __restrict__ q, int64_t ldq,
                   float* __restrict__ s, int64_t ldsw, uint8_t* __restrict__ qT, int64_t ldqT) {
    using P = QWCfg<T>;
    extern __shared__ __align__(128) uint8_t smem[];
    griddep_wait();                 // PDL: previous grid complete, its writes visible
    griddep_launch_dependents();
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + P::OFF_BAR;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < P::STAGES; ++i) { mbar_init(bar0 + 8 * i, 1); mbar_init(bar0 + 8 * (P::STAGES + i), P::CONSUMERS); }
        fence_mbar_init();
    }
    __syncthreads();
    const int NB = (int)((N + 127) >> 7), KB = (int)((K + 127) >> 7);
    const int nblocks = NB * KB;
    if (warp == P::CONSUMERS) {
        if (lane == 0) {
            tma_prefetch_desc(&tmW);
            int it = 0;
            for (int b = blockIdx.x; b < nblocks; b += gridDim.x, ++it) {
                const int st = it % P::STAGES;
                mbar_wait(bar0 + 8 * (P::STAGES + st), ((it / P::STAGES) & 1) ^ 1);
                mbar_arrive_expect_tx(bar0 + 8 * st, P::BLOCK_BYTES);
                tma_load_2d(sbase + st * P::BLOCK_BYTES, &tmW, bar0 + 8 * st, (b % KB) * 128, (b / KB) * 128);
            }
        }
        return;
    }
    const int tid = threadIdx.x;
    float* red = reinterpret_cast<float*>(smem + P::OFF_RED);
    int it = 0;
    for (int b = blockIdx.x; b < nblocks; b += gridDim.x, ++it) {
        const int st = it % P::STAGES;
        const int nb = b / KB, kb = b - nb * KB;
        const int64_t n0 = (int64_t)nb * 128, k0 = (int64_t)kb * 128;
        mbar_wait(bar0 + 8 * st, (it / P::STAGES) & 1);
        uint4 v[P::NCH];
#pragma unroll
        for (int i = 0; i < P::NCH; ++i) v[i] = lds128(sbase + st * P::BLOCK_BYTES + (i * 32 * P::CONSUMERS + tid) * 16);
        // the stage was written by TMA (async proxy) and read with ld.shared (generic proxy): a proxy
        // fence keeps the producer's next TMA into it behind these reads (an mbarrier arrive alone
        // does not; see gemm.cu release_scales)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar0 + 8 * (P::STAGES + st));
        float amax = 0.0f;
#pragma unroll
        for (int i = 0; i < P::NCH; ++i) {
            float f[P::E];
            Vec<T>::unpack(v[i], f);
#pragma unroll
            for (int e = 0; e < P::E; ++e) amax = fmaxf(amax, fabsf(f[e]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        // per-block parity: without the transposed copy there is no second barrier, and a fast warp
        // would otherwise overwrite its slot for the next block while a slow one still reads this one
        float* rb = red + (it & 1) * P::CONSUMERS;
        if (lane == 0) rb[warp] = amax;
        named_bar_sync(1, 32 * P::CONSUMERS);
        amax = rb[0];
#pragma unroll
        for (int i = 1; i < P::CONSUMERS; ++i) amax = fmaxf(amax, rb[i]);
        const float sc = group_scale_t<kPow2>(amax);
        const float rc = __frcp_rn(sc);
        const bool fast = fast_div_ok(sc);                  // block-uniform
        // Interior block (every block of the C1/C2 weights): branch-free stores from one base pointer
        // per thread; the integer bounds arithmetic of the general path below was most of this
        // kernel's instructions (ncu: ~22 instructions per element).
        const bool full = (n0 + 128 <= N) && (k0 + 128 <= K);
        if (full && fast) {
            constexpr int RSTEP = 32 * P::CONSUMERS / P::CPR;             // rows between a thread's chunks
            const int row0 = tid / P::CPR, col = (tid % P::CPR) * P::E;
            uint8_t* qb = q + (n0 + row0) * ldq + k0 + col;
            const int64_t qstep = (int64_t)RSTEP * ldq;
            const uint32_t cbase = sbase + P::OFF_C;
#pragma unroll
            for (int i = 0; i < P::NCH; ++i) {
                float f[P::E];
                Vec<T>::unpack(v[i], f);
                uint32_t wd[P::E / 4];
                encode_chunk<P::E>(f, sc, rc, true, wd);
                if constexpr (P::E == 8) *reinterpret_cast<uint2*>(qb + i * qstep) = make_uint2(wd[0], wd[1]);
                else *reinterpret_cast<uint32_t*>(qb + i * qstep) = wd[0];
                if (qT) {
                    const int row = row0 + i * RSTEP;
#pragma unroll
                    for (int e = 0; e < P::E / 4; ++e) {
                        const int kw = col / 4 + e;
                        asm volatile("st.shared.u32 [%0], %1;" :: "r"(cbase + row * 128 + 4 * (kw ^ ((row >> 2) & 31))),
                                     "r"(wd[e]) : "memory");
                    }
                }
            }
            if (tid == 0) s[(int64_t)nb * ldsw + kb] = sc;
            if (qT) {
                named_bar_sync(1, 32 * P::CONSUMERS);
                const int l = tid & 31;
                uint8_t* tb = qT + k0 * ldqT + n0 + 4 * l;
#pragma unroll
                for (int i = 0; i < 32 * 32 / (32 * P::CONSUMERS); ++i) {
                    const int kw = (i * 32 * P::CONSUMERS + tid) >> 5;          // rows 4l..4l+3, k 4kw..4kw+3
                    uint32_t a[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) a[j] = lds32(cbase + (4 * l + j) * 128 + 4 * (kw ^ l));
                    const uint32_t t0 = __byte_perm(a[0], a[1], 0x5140), t1 = __byte_perm(a[0], a[1], 0x7362);
                    const uint32_t t2 = __byte_perm(a[2], a[3], 0x5140), t3 = __byte_perm(a[2], a[3], 0x7362);
                    const uint32_t b4[4] = {__byte_perm(t0, t2, 0x5410), __byte_perm(t0, t2, 0x7632),
                                            __byte_perm(t1, t3, 0x5410), __byte_perm(t1, t3, 0x7632)};
                    uint8_t* d = tb + (int64_t)(4 * kw) * ldqT;
#pragma unroll
                    for (int e = 0; e < 4; ++e) *reinterpret_cast<uint32_t*>(d + e * ldqT) = b4[e];
                }
            }
            continue;
        }
#pragma unroll
        for (int i = 0; i < P::NCH; ++i) {
            const int idx = i * 32 * P::CONSUMERS + tid, row = idx / P::CPR, col = (idx % P::CPR) * P::E;
            float f[P::E];
            Vec<T>::unpack(v[i], f);
            uint32_t wd[P::E / 4];
            encode_chunk<P::E>(f, sc, rc, fast, wd);
            if (n0 + row < N && k0 + col < K) {
                uint8_t* dst = q + (n0 + row) * ldq + k0 + col;
                if constexpr (P::E == 8) *reinterpret_cast<uint2*>(dst) = make_uint2(wd[0], wd[1]);
                else *reinterpret_cast<uint32_t*>(dst) = wd[0];
            }
            if (qT) {   // code tile word (row, kw) lives at row*128 + 4*(kw ^ (row/4 % 32)): conflict-free both ways
#pragma unroll
                for (int e = 0; e < P::E / 4; ++e) {
                    const int kw = col / 4 + e;
                    asm volatile("st.shared.u32 [%0], %1;" :: "r"(sbase + P::OFF_C + row * 128 + 4 * (kw ^ ((row >> 2) & 31))),
                                 "r"(wd[e]) : "memory");
                }
            }
        }
        if (tid == 0) s[(int64_t)nb * ldsw + kb] = sc;
        if (qT) {
            named_bar_sync(1, 32 * P::CONSUMERS);
#pragma unroll
            for (int i = 0; i < 32 * 32 / (32 * P::CONSUMERS); ++i) {
                const int idx = i * 32 * P::CONSUMERS + tid, kw = idx >> 5, l = idx & 31;   // rows 4l..4l+3, k 4kw..4kw+3
                uint32_t a[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) a[j] = lds32(sbase + P::OFF_C + (4 * l + j) * 128 + 4 * (kw ^ l));
                // 4x4 byte transpose: b[e] = bytes e of a[0..3]
                const uint32_t t0 = __byte_perm(a[0], a[1], 0x5140), t1 = __byte_perm(a[0], a[1], 0x7362);
                const uint32_t t2 = __byte_perm(a[2], a[3], 0x5140), t3 = __byte_perm(a[2], a[3], 0x7362);
                const uint32_t b[4] = {__byte_perm(t0, t2, 0x5410), __byte_perm(t0, t2, 0x7632),
                                       __byte_perm(t1, t3, 0x5410), __byte_perm(t1, t3, 0x7632)};
                const int64_t n = n0 + 4 * l;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int64_t kk = k0 + 4 * kw + e;
                    if (kk < K && n < N) {
                        uint8_t* dst = qT + kk * ldqT + n;
                        if (n + 4 <= N) *reinterpret_cast<uint32_t*>(dst) = b[e];
                        else for (int x = 0; x < 4 && n + x < N; ++x) dst[x] = (uint8_t)(b[e] >> (8 * x));
                    }
                }
            }
        }
    }
}

// ===========================================================================================
// 128x128 weight blocks.  CTA per block: 16-byte loads held in registers, block amax via warp
// shuffles + smem, codes written row-major; the optional transposed copy is staged in smem
// ([k][n], 132-byte rows) and written as contiguous 128-byte rows of qT.
// ===========================================================================================
template <typename T>
struct TW {
    static constexpr int E = Vec<T>::E;
    static constexpr int CPR = 128 / E;                 // chunks per block row: 32 FP32 / 16 BF16
    static constexpr int NCH = 128 * CPR / 256;         // chunks per thread: 16 / 8
    static constexpr int TSTR = 132;
};

template <typename T>
__global__ void __launch_bounds__(256)
k_quant_weight_128x128(const T* __restrict__ w, int64_t N, int64_t K, int64_t ldw,
                       uint8_t* __restrict__ q, int64_t ldq, float* __restrict__ s, int64_t ldsw,
                       uint8_t* __restrict__ qT, int64_t ldqT) {
    using P = TW<T>;
    __shared__ __align__(16) uint8_t ts[128 * P::TSTR];
    __shared__ float red[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t NB = (N + 127) >> 7, KB = (K + 127) >> 7;
    for (int64_t t = blockIdx.x; t < NB * KB; t += gridDim.x) {
        const int64_t nb = t / KB, kb = t - nb * KB;
        const int64_t n0 = nb * 128, k0 = kb * 128;
        uint4 v[P::NCH];
#pragma unroll
        for (int i = 0; i < P::NCH; ++i) {
            const int idx = i * 256 + tid, r = idx / P::CPR, ck = idx % P::CPR;
            const int64_t col = k0 + ck * P::E;
            const bool ok = (n0 + r < N) && (col < K);
            v[i] = ok ? ld_stream16(w + (n0 + r) * ldw + col) : make_uint4(0, 0, 0, 0);
        }
        float amax = 0.0f;
#pragma unroll
        for (int i = 0; i < P::NCH; ++i) {
            float f[P::E];
            Vec<T>::unpack(v[i], f);
#pragma unroll
            for (int e = 0; e < P::E; ++e) amax = fmaxf(amax, fabsf(f[e]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        if (lane == 0) red[warp] = amax;
        __syncthreads();
        amax = red[0];
#pragma unroll
        for (int i = 1; i < 8; ++i) amax = fmaxf(amax, red[i]);
        const float sc = group_scale(amax);
        const float rc = __frcp_rn(sc);
        const bool fast = fast_div_ok(sc);
#pragma unroll
        for (int i = 0; i < P::NCH; ++i) {
            const int idx = i * 256 + tid, r = idx / P::CPR, ck = idx % P::CPR;
            float f[P::E];
            Vec<T>::unpack(v[i], f);
            uint32_t wd[P::E / 4];
            encode_chunk<P::E>(f, sc, rc, fast, wd);
            const int64_t col = k0 + ck * P::E;
            if ((n0 + r < N) && (col < K)) {
                uint8_t* dst = q + (n0 + r) * ldq + col;
                if constexpr (P::E == 8) *reinterpret_cast<uint2*>(dst) = make_uint2(wd[0], wd[1]);
                else *reinterpret_cast<uint32_t*>(dst) = wd[0];
            }
            if (qT) {
#pragma unroll
                for (int e = 0; e < P::E; ++e) ts[(ck * P::E + e) * P::TSTR + r] = (uint8_t)(wd[e >> 2] >> (8 * (e & 3)));
            }
        }
        if (tid == 0) s[nb * ldsw + kb] = sc;
        if (qT) {
            __syncthreads();
#pragma unroll 4
            for (int i = 0; i < 16; ++i) {
                const int idx = i * 256 + tid, k = idx >> 5, wj = idx & 31;
                const int64_t kk = k0 + k, n = n0 + wj * 4;
                if (kk < K && n < N) {
                    const uint32_t val = *reinterpret_cast<const uint32_t*>(ts + k * P::TSTR + wj * 4);
                    uint8_t* dst = qT + kk * ldqT + n;
                    if (n + 4 <= N) *reinterpret_cast<uint32_t*>(dst) = val;
                    else for (int e = 0; e < 4 && n + e < N; ++e) dst[e] = (uint8_t)(val >> (8 * e));
                }
            }
        }
        __syncthreads();
    }
}

// ===========================================================================================
// Generic (any alignment / shape) group quantizer: one CTA of 128 threads per group.
// Element (r, c) of the input is x[r*xr + c*xc]; group g = (gi, gj) covers rows
// [gi*gr, +gr) x cols [gj*gc, +gc); codes go to q[r*qr + c*qc] (and q2[r*q2r + c*q2c] if q2),
// the scale to s[gi*sr + gj*sc].
// ===========================================================================================
template <typename T, bool kPow2 = false>
__global__ void __launch_bounds__(128)
k_quant_generic(const T* __restrict__ x, int64_t R, int64_t Cn, int64_t xr, int64_t xc, int gr, int gc,
                uint8_t* __restrict__ q, int64_t qr, int64_t qc, uint8_t* __restrict__ q2, int64_t q2r, int64_t q2c,
                float* __restrict__ s, int64_t sr, int64_t sc_) {
    __shared__ float red[4];
    const int64_t GI = (R + gr - 1) / gr, GJ = (Cn + gc - 1) / gc;
    for (int64_t g = blockIdx.x; g < GI * GJ; g += gridDim.x) {
        const int64_t gi = g / GJ, gj = g - gi * GJ;
        const int64_t r0 = gi * gr, c0 = gj * gc;
        const int64_t nr = min((int64_t)gr, R - r0), nc = min((int64_t)gc, Cn - c0);
        const int64_t n = nr * nc;
        float amax = 0.0f;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const int64_t r = r0 + i / nc, c = c0 + i % nc;
            amax = fmaxf(amax, fabsf(load_scalar<T>(x + r * xr + c * xc)));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
        __syncthreads();
        amax = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
        const float scl = group_scale_t<kPow2>(amax);
        const float rc = __frcp_rn(scl);
        const bool fast = fast_div_ok(scl);
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const int64_t r = r0 + i / nc, c = c0 + i % nc;
            const float v = div_scale(load_scalar<T>(x + r * xr + c * xc), scl, rc, fast);
            const uint8_t code = (uint8_t)(cvt_e4m3x2(v, 0.0f) & 0xFF);
            q[r * qr + c * qc] = code;
            if (q2) q2[r * q2r + c * q2c] = code;
        }
        if (threadIdx.x == 0) s[gi * sr + gj * sc_] = scl;
        __syncthreads();
    }
}

// ===========================================================================================
// launchers
// ===========================================================================================
static int grid_for(int64_t work, int per_sm, int max_ctas_per_sm = 8) {
    int64_t g = work;
    int64_t cap = (int64_t)num_sms() * max_ctas_per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    (void)per_sm;
    return (int)g;
}

template <typename T>
static cudaError_t launch_1x128_t(const void* x, int64_t M, int64_t K, int64_t ldx, uint8_t* q, int64_t ldq,
                                  float* s, int64_t lds, cudaStream_t st) {
    constexpr int E = Vec<T>::E;
    const bool fast = aligned16(x) && ((ldx * (int64_t)sizeof(T)) % 16 == 0) && (K % E == 0) &&
                      (reinterpret_cast<uintptr_t>(q) % E == 0) && (ldq % E == 0);
    const bool flat = fast && (ldx == K) && (K % 128 == 0) && (ldq == K) && aligned16(q) && (M * (K / 128) < (1ll << 31));
    if (flat) {
        using C = Q1Cfg<T>;
        static bool attr_set[64] = {false};   // per device
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || !attr_set[dev]) {
            cudaFuncSetAttribute(k_quant_act_1x128_tma<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
            if (dev >= 0 && dev < 64) attr_set[dev] = true;
        }
        const int64_t chunks = (M * (K / 128) + C::CHUNK_TILES - 1) / C::CHUNK_TILES;
        return launch_pdl(k_quant_act_1x128_tma<T>, grid_for(chunks, 2, 2), C::THREADS, C::SMEM, st, 
            reinterpret_cast<const T*>(x), M, K, q, s, lds);
    } else if (fast) {
        constexpr int U = 4;
        constexpr int TPU = (32 / (128 / E)) * U;
        const int64_t KB = (K + 127) / 128;
        const int64_t units = M * ((KB + TPU - 1) / TPU);
        k_quant_act_1x128<T, U><<<grid_for((units + 7) / 8, 8), 256, 0, st>>>(
            reinterpret_cast<const T*>(x), M, K, ldx, q, ldq, s, lds);
    } else {
        const int64_t groups = M * ((K + 127) / 128);
        k_quant_generic<T><<<grid_for(groups, 16, 16), 128, 0, st>>>(
            reinterpret_cast<const T*>(x), M, K, ldx, 1, 1, 128, q, ldq, 1, nullptr, 0, 0, s, 1, lds);
    }
    return cudaPeekAtLastError();
}

// Power-of-two scales (fp8bs_quantize_act_1x128_pow2): the TMA kernel for flat aligned inputs, the
// generic kernel otherwise.
template <typename T>
static cudaError_t launch_1x128_pow2_t(const void* x, int64_t M, int64_t K, int64_t ldx, uint8_t* q, int64_t ldq,
                                       float* s, int64_t lds, cudaStream_t st) {
    constexpr int E = Vec<T>::E;
    const bool flat = aligned16(x) && ((ldx * (int64_t)sizeof(T)) % 16 == 0) && (K % E == 0) && (ldx == K) &&
                      (K % 128 == 0) && (ldq == K) && aligned16(q) && (M * (K / 128) < (1ll << 31));
    if (flat) {
        using C = Q1Cfg<T>;
        static bool attr_set[64] = {false};   // per device
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || !attr_set[dev]) {
            cudaFuncSetAttribute(k_quant_act_1x128_tma<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
            if (dev >= 0 && dev < 64) attr_set[dev] = true;
        }
        const int64_t chunks = (M * (K / 128) + C::CHUNK_TILES - 1) / C::CHUNK_TILES;
        return launch_pdl(k_quant_act_1x128_tma<T, true>, grid_for(chunks, 2, 2), C::THREADS, C::SMEM, st,
                          reinterpret_cast<const T*>(x), M, K, q, s, lds);
    }
    const int64_t groups = M * ((K + 127) / 128);
    k_quant_generic<T, true><<<grid_for(groups, 16, 16), 128, 0, st>>>(
        reinterpret_cast<const T*>(x), M, K, ldx, 1, 1, 128, q, ldq, 1, nullptr, 0, 0, s, 1, lds);
    return cudaPeekAtLastError();
}

cudaError_t launch_quant_act_1x128_pow2(const void* x, int xdt, int64_t M, int64_t K, int64_t ldx, uint8_t* q,
                                        int64_t ldq, float* s, int64_t lds, cudaStream_t st) {
    if (xdt == 0) return launch_1x128_pow2_t<__nv_bfloat16>(x, M, K, ldx, q, ldq, s, lds, st);
    return launch_1x128_pow2_t<float>(x, M, K, ldx, q, ldq, s, lds, st);
}

cudaError_t launch_quant_act_1x128(const void* x, int xdt, int64_t M, int64_t K, int64_t ldx, uint8_t* q,
                                   int64_t ldq, float* s, int64_t lds, cudaStream_t st) {
    if (xdt == 0) return launch_1x128_t<__nv_bfloat16>(x, M, K, ldx, q, ldq, s, lds, st);
    return launch_1x128_t<float>(x, M, K, ldx, q, ldq, s, lds, st);
}

template <typename T>
static cudaError_t launch_128x1_t(const void* x, int64_t M, int64_t C, int64_t ldx, uint8_t* qT, int64_t ldq,
                                  float* sT, int64_t lds, cudaStream_t st) {
    using P = T128x1<T>;
    const bool fast = aligned16(x) && ((ldx * (int64_t)sizeof(T)) % 16 == 0) && (C % P::E == 0) &&
                      aligned16(qT) && (ldq % 16 == 0);
    alignas(64) CUtensorMap tm;
    bool tma = fast && (M * ((C + P::CH - 1) / P::CH) / 128 < (1ll << 31));
    if (tma) {
        const uint64_t dims[2] = {(uint64_t)C, (uint64_t)M};
        const uint64_t str[1] = {(uint64_t)ldx * sizeof(T)};
        const uint32_t box[2] = {(uint32_t)P::CH, 128};
        tma = make_tmap(&tm, sizeof(T) == 2 ? TMAP_BF16 : TMAP_F32, 2, x, dims, str, box, 0);
    }
    if (tma) {
        using Q = QTCfg<T>;
        static bool attr_tma[64] = {false};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || !attr_tma[dev]) {
            cudaFuncSetAttribute(k_quant_act_128x1_tma<T, DenseRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, Q::SMEM);
            if (dev >= 0 && dev < 64) attr_tma[dev] = true;
        }
        const int64_t tiles = ((M + 127) / 128) * ((C + Q::CH - 1) / Q::CH);
        return launch_pdl(k_quant_act_128x1_tma<T, DenseRows>, grid_for(tiles, 2, 2), Q::THREADS, Q::SMEM, st, tm, M, C, qT, ldq,
                          sT, lds, DenseRows{});
    } else if (fast) {
        static bool attr_set[64] = {false};   // per device; idempotent, benign race
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || !attr_set[dev]) {
            cudaFuncSetAttribute(k_quant_act_128x1<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
            if (dev >= 0 && dev < 64) attr_set[dev] = true;
        }
        const int64_t tiles = ((M + 127) / 128) * ((C + P::CH - 1) / P::CH);
        k_quant_act_128x1<T><<<grid_for(tiles, 4, 4), 256, P::SMEM, st>>>(
            reinterpret_cast<const T*>(x), M, C, ldx, qT, ldq, sT, lds);
    } else {
        const int64_t groups = ((M + 127) / 128) * C;
        k_quant_generic<T><<<grid_for(groups, 16, 16), 128, 0, st>>>(
            reinterpret_cast<const T*>(x), M, C, ldx, 1, 128, 1, qT, 1, ldq, nullptr, 0, 0, sT, lds, 1);
    }
    return cudaPeekAtLastError();
}

cudaError_t launch_quant_act_128x1(const void* x, int xdt, int64_t M, int64_t C, int64_t ldx, uint8_t* qT,
                                   int64_t ldq, float* sT, int64_t lds, cudaStream_t st) {
    if (xdt == 0) return launch_128x1_t<__nv_bfloat16>(x, M, C, ldx, qT, ldq, sT, lds, st);
    return launch_128x1_t<float>(x, M, C, ldx, qT, ldq, sT, lds, st);
}

// Grouped 128x1 (expert-aligned layout, R25): one launch over all experts' token blocks (BF16 or FP32).
// Returns cudaErrorNotSupported when the TMA path does not apply (the caller then loops per expert).
template <typename T>
static cudaError_t launch_128x1_grouped_t(const void* x, int32_t G, const int64_t* off, const int64_t* pad, int64_t C,
                                          int64_t ldx, uint8_t* qT, int64_t ldq, float* sT, int64_t lds, cudaStream_t st) {
    using Q = QTCfg<T>;
    using P = T128x1<T>;
    const int64_t R = off[G], Mp = pad[G];
    if (!(aligned16(x) && ((ldx * (int64_t)sizeof(T)) % 16 == 0) && (C % P::E == 0) && aligned16(qT) && (ldq % 16 == 0)) ||
        R == 0)
        return cudaErrorNotSupported;
    alignas(64) CUtensorMap tm;
    const uint64_t dims[2] = {(uint64_t)C, (uint64_t)R};
    const uint64_t str[1] = {(uint64_t)ldx * sizeof(T)};
    const uint32_t box[2] = {(uint32_t)Q::CH, 128};
    if (!make_tmap(&tm, sizeof(T) == 2 ? TMAP_BF16 : TMAP_F32, 2, x, dims, str, box, 0)) return cudaErrorNotSupported;
    static thread_local GroupRows* rp = nullptr;   // host staging of the 8 KB kernel parameter
    if (!rp) rp = new GroupRows();
    rp->G = G;
    for (int e = 0; e <= G; ++e) { rp->off[e] = (int)off[e]; rp->pad[e] = (int)pad[e]; }
    static bool attr[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[dev]) {
        cudaFuncSetAttribute(k_quant_act_128x1_tma<T, GroupRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, Q::SMEM);
        if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    const int64_t tiles = (Mp / 128) * ((C + Q::CH - 1) / Q::CH);
    return launch_pdl(k_quant_act_128x1_tma<T, GroupRows>, grid_for(tiles, 2, 2), Q::THREADS, Q::SMEM, st, tm,
                      Mp, C, qT, ldq, sT, lds, *rp);
}

cudaError_t launch_quant_act_128x1_grouped(const void* x, int xdt, int32_t G, const int64_t* off, const int64_t* pad,
                                           int64_t C, int64_t ldx, uint8_t* qT, int64_t ldq, float* sT, int64_t lds,
                                           cudaStream_t st) {
    if (G > GroupRows::MAXG || off[G] >= (1ll << 31) || pad[G] >= (1ll << 31)) return cudaErrorNotSupported;
    if (xdt == 0) return launch_128x1_grouped_t<__nv_bfloat16>(x, G, off, pad, C, ldx, qT, ldq, sT, lds, st);
    return launch_128x1_grouped_t<float>(x, G, off, pad, C, ldx, qT, ldq, sT, lds, st);
}

cudaError_t launch_quant_act_dual(const void* x, int xdt, int64_t M, int64_t K, int64_t ldx, uint8_t* q, int64_t ldq,
                                  float* s, int64_t lds, uint8_t* qT, int64_t ldqT, float* sT, int64_t ldsT,
                                  int pow2, cudaStream_t st) {
    using Q = QDCfg;
    // fused path: BF16 (a 128-channel tile row is one 1x128 group), 16-byte aligned rows and codes
    bool fused = xdt == 0 && aligned16(x) && ((ldx * 2) % 16 == 0) && (K % 16 == 0) && aligned16(q) && (ldq % 16 == 0) &&
                 aligned16(qT) && (ldqT % 16 == 0) && (M * ((K + Q::CH - 1) / Q::CH) / 128 < (1ll << 31));
    alignas(64) CUtensorMap tm;
    if (fused) {
        const uint64_t dims[2] = {(uint64_t)K, (uint64_t)M};
        const uint64_t str[1] = {(uint64_t)ldx * 2};
        const uint32_t box[2] = {(uint32_t)Q::CH, 128};
        fused = make_tmap(&tm, TMAP_BF16, 2, x, dims, str, box, 0);
    }
    if (!fused && pow2) {   // two passes over x, generic kernel (power-of-two scales)
        const int64_t g1 = M * ((K + 127) / 128), g2 = ((M + 127) / 128) * K;
        if (xdt == 0) {
            const auto* xb = reinterpret_cast<const __nv_bfloat16*>(x);
            k_quant_generic<__nv_bfloat16, true><<<grid_for(g1, 16, 16), 128, 0, st>>>(xb, M, K, ldx, 1, 1, 128, q, ldq, 1, nullptr, 0, 0, s, 1, lds);
            k_quant_generic<__nv_bfloat16, true><<<grid_for(g2, 16, 16), 128, 0, st>>>(xb, M, K, ldx, 1, 128, 1, qT, 1, ldqT, nullptr, 0, 0, sT, ldsT, 1);
        } else {
            const auto* xf = reinterpret_cast<const float*>(x);
            k_quant_generic<float, true><<<grid_for(g1, 16, 16), 128, 0, st>>>(xf, M, K, ldx, 1, 1, 128, q, ldq, 1, nullptr, 0, 0, s, 1, lds);
            k_quant_generic<float, true><<<grid_for(g2, 16, 16), 128, 0, st>>>(xf, M, K, ldx, 1, 128, 1, qT, 1, ldqT, nullptr, 0, 0, sT, ldsT, 1);
        }
        return cudaPeekAtLastError();
    }
    if (!fused) {   // two passes over x
        cudaError_t e = launch_quant_act_1x128(x, xdt, M, K, ldx, q, ldq, s, lds, st);
        if (e != cudaSuccess) return e;
        return launch_quant_act_128x1(x, xdt, M, K, ldx, qT, ldqT, sT, ldsT, st);
    }
    auto kern = pow2 ? k_quant_act_dual_tma<true> : k_quant_act_dual_tma<false>;
    static bool attr[2][64] = {{false}};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[pow2 ? 1 : 0][dev]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Q::SMEM);
        if (dev >= 0 && dev < 64) attr[pow2 ? 1 : 0][dev] = true;
    }
    const int64_t tiles = ((M + 127) / 128) * ((K + Q::CH - 1) / Q::CH);
    return launch_pdl(kern, grid_for(tiles, 2, 2), Q::THREADS, Q::SMEM, st, tm, M, K, q, ldq, s, lds, qT, ldqT, sT, ldsT);
}

template <typename T>
static cudaError_t launch_w_t(const void* w, int64_t N, int64_t K, int64_t ldw, uint8_t* q, int64_t ldq,
                              float* s, int64_t ldsw, uint8_t* qT, int64_t ldqT, int pow2, cudaStream_t st) {
    using P = TW<T>;
    const bool fast = aligned16(w) && ((ldw * (int64_t)sizeof(T)) % 16 == 0) && (K % P::E == 0) &&
                      (reinterpret_cast<uintptr_t>(q) % P::E == 0) && (ldq % P::E == 0) &&
                      (qT == nullptr || ((reinterpret_cast<uintptr_t>(qT) % 4 == 0) && (ldqT % 4 == 0)));
    const int64_t blocks = ((N + 127) / 128) * ((K + 127) / 128);
    alignas(64) CUtensorMap tm;
    bool tma = fast && blocks < (1ll << 31);
    if (tma) {
        const uint64_t dims[2] = {(uint64_t)K, (uint64_t)N};
        const uint64_t str[1] = {(uint64_t)ldw * sizeof(T)};
        const uint32_t box[2] = {128, 128};
        tma = make_tmap(&tm, sizeof(T) == 2 ? TMAP_BF16 : TMAP_F32, 2, w, dims, str, box, 0);
    }
    if (tma) {
        using Q = QWCfg<T>;
        auto kern = pow2 ? k_quant_weight_tma<T, true> : k_quant_weight_tma<T, false>;
        static bool attr_tma[2][64] = {{false}};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || !attr_tma[pow2 ? 1 : 0][dev]) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Q::SMEM);
            if (dev >= 0 && dev < 64) attr_tma[pow2 ? 1 : 0][dev] = true;
        }
        return launch_pdl(kern, grid_for(blocks, 1, 1), Q::THREADS, Q::SMEM, st, tm, N, K, q, ldq, s, ldsw, qT, ldqT);
    } else if (pow2) {
        k_quant_generic<T, true><<<grid_for(blocks, 16, 16), 128, 0, st>>>(
            reinterpret_cast<const T*>(w), N, K, ldw, 1, 128, 128, q, ldq, 1, qT, 1, ldqT, s, ldsw, 1);
    } else if (fast) {
        k_quant_weight_128x128<T><<<grid_for(blocks, 4, 4), 256, 0, st>>>(
            reinterpret_cast<const T*>(w), N, K, ldw, q, ldq, s, ldsw, qT, ldqT);
    } else {
        k_quant_generic<T><<<grid_for(blocks, 16, 16), 128, 0, st>>>(
            reinterpret_cast<const T*>(w), N, K, ldw, 1, 128, 128, q, ldq, 1, qT, 1, ldqT, s, ldsw, 1);
    }
    return cudaPeekAtLastError();
}

cudaError_t launch_quant_weight_128x128(const void* w, int wdt, int64_t N, int64_t K, int64_t ldw, uint8_t* q,
                                        int64_t ldq, float* s, int64_t ldsw, uint8_t* qT, int64_t ldqT,
                                        int pow2, cudaStream_t st) {
    if (wdt == 0) return launch_w_t<__nv_bfloat16>(w, N, K, ldw, q, ldq, s, ldsw, qT, ldqT, pow2, st);
    return launch_w_t<float>(w, N, K, ldw, q, ldq, s, ldsw, qT, ldqT, pow2, st);
}

}  // namespace fp8bs

// ===========================================================================================
// FP8 -> FP8 re-quantization of a cached activation: 1x128 codes + scales -> dequantize -> 128x1
// (§3.3.3, §3.5.2: the forward's FP8 activations are "read out,
// dequantized, transposed, re-quantized into 128x1 tiles" for the backward pass).
// Work unit: a 128-token x 128-channel tile (exactly one 1x128 scale group per row).  Dequantized
// value xhat = RN32(dec(q) * s) (E4M3 -> FP16 -> FP32 is exact, one rounded FP32 multiply).
// ===========================================================================================
namespace fp8bs {
// Persistent, TMA-fed: lane 0 of warp 0 streams 128-token x 128-channel code tiles (16 KB, SWIZZLE_128B)
// into a 4-stage ring.  Each of the 8 warps owns 16 channels (one 16-byte chunk of every
// row) over all 128 tokens, so a channel's 128x1 amax is a warp reduction and the consumers never
// wait on each other (the previous form, 16 tokens x 4 channels per thread with a shared-memory
// reduction, paid three CTA barriers per tile).  Lane (cg = lane & 3, tg = lane >> 2): channels
// 16w + 4cg + [0, 4) of tokens 16tg + [0, 16).  A lane walks its 16 tokens rotated by tg (token
// 16tg + ((r + tg) & 15) at step r), so the 8 token groups of one ld.shared hit 8 different swizzled
// 16-byte chunks (no bank conflicts); the channel's 16 codes, packed in that rotated order, are
// rotated back by tg bytes and stored as one 16-byte run of qT (a warp store covers 4 channels x
// 128 tokens).  2 CTAs per SM.
struct RQCfg {
    // no separate producer warp: with 288 threads ncu reported a register block limit of one CTA per
    // SM (even at 104 registers); lane 0 of warp 0 issues the TMA loads, STAGES - 1 tiles ahead
    static constexpr int STAGES = 4, CONSUMERS = 8, THREADS = 32 * CONSUMERS;
    static constexpr int TILE_BYTES = 128 * 128;
    static constexpr int OFF_BAR = STAGES * TILE_BYTES;
    static constexpr int SMEM = 1024 + OFF_BAR + 2 * STAGES * 8;   // + alignment slack (SWIZZLE_128B)
};

template <bool kPow2>
__global__ void __launch_bounds__(RQCfg::THREADS, 2)
k_requant_1x128_to_128x1(const __grid_constant__ CUtensorMap tmQ, const float* __restrict__ s, int64_t lds,
                         int64_t M, int64_t K, uint8_t* __restrict__ qT, int64_t ldqT, float* __restrict__ sT, int64_t ldsT) {
    using P = RQCfg;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    griddep_wait();                 // PDL: previous grid complete, its writes visible
    griddep_launch_dependents();
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + P::OFF_BAR;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < P::STAGES; ++i) { mbar_init(bar0 + 8 * i, 1); mbar_init(bar0 + 8 * (P::STAGES + i), P::CONSUMERS); }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t KB = (K + 127) / 128, MB = (M + 127) / 128;
    const int64_t ntiles = MB * KB;
    const bool issuer = warp == 0 && lane == 0;
    auto issue = [&](int64_t tt, int st) {
        mbar_arrive_expect_tx(bar0 + 8 * st, P::TILE_BYTES);
        tma_load_2d(sbase + st * P::TILE_BYTES, &tmQ, bar0 + 8 * st, (int)((tt % KB) * 128), (int)((tt / KB) * 128));
    };
    if (issuer) {
        tma_prefetch_desc(&tmQ);
        for (int i = 0; i < P::STAGES - 1 && blockIdx.x + (int64_t)i * gridDim.x < ntiles; ++i) issue(blockIdx.x + (int64_t)i * gridDim.x, i);
    }
    const int cg = lane & 3, tg = lane >> 2;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = it % P::STAGES;
        if (issuer) {
            // tile #it + STAGES - 1 into the stage tile #it - 1 used (released by every warp by now, usually)
            const int64_t tn = t + (int64_t)(P::STAGES - 1) * gridDim.x;
            if (tn < ntiles) {
                const int sn = (it + P::STAGES - 1) % P::STAGES;
                if (it >= 1) mbar_wait(bar0 + 8 * (P::STAGES + sn), ((it - 1) / P::STAGES) & 1);
                issue(tn, sn);
            }
        }
        const int64_t mb = t / KB, kb = t - mb * KB;
        const int64_t m0 = mb * 128 + 16 * tg;           // this lane's first token
        // row scales of the lane's tokens in its rotated order (issued before the stage wait)
        const float* srow = s + kb * lds + m0;
        float sr[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int k = (r + tg) & 15;
            sr[r] = (m0 + k < M) ? __ldg(srow + k) : 0.0f;
        }
        mbar_wait(bar0 + 8 * st, (it / P::STAGES) & 1);
        const uint32_t tile = sbase + st * P::TILE_BYTES;
        uint32_t w[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int row = 16 * tg + ((r + tg) & 15);
            w[r] = lds32(tile + row * 128 + ((warp ^ (row & 7)) << 4) + 4 * cg);
        }
        // TMA-written stage read with ld.shared: proxy fence before the release (gemm.cu release_scales)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar0 + 8 * (P::STAGES + st));
        // xhat = RN32(dec(q) * s): recomputed in the encode pass below rather than kept (64 registers
        // more would leave one CTA per SM)
        auto dequant = [&](int r, float* d) __attribute__((always_inline)) {
            const __half2_raw lo = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(w[r] & 0xFFFFu), __NV_E4M3);
            const __half2_raw hi = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(w[r] >> 16), __NV_E4M3);
            const float2 d01 = __half22float2(*reinterpret_cast<const __half2*>(&lo));
            const float2 d23 = __half22float2(*reinterpret_cast<const __half2*>(&hi));
            d[0] = __fmul_rn(d01.x, sr[r]); d[1] = __fmul_rn(d01.y, sr[r]);   // TMA zero-fills codes past M / K
            d[2] = __fmul_rn(d23.x, sr[r]); d[3] = __fmul_rn(d23.y, sr[r]);
        };
        float a4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            float d[4];
            dequant(r, d);
#pragma unroll
            for (int j = 0; j < 4; ++j) a4[j] = fmaxf(a4[j], fabsf(d[j]));
        }
        // the channel's amax over the tile's 128 tokens: the warp's 8 token groups
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) a4[j] = fmaxf(a4[j], __shfl_xor_sync(0xffffffffu, a4[j], o));
        }
        const int64_t c0 = kb * 128 + 16 * warp + 4 * cg;   // this lane's first channel
        float sc[4], rc[4];
        bool fast = true;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            sc[j] = group_scale_t<kPow2>(a4[j]);
            rc[j] = __frcp_rn(sc[j]);
            fast = fast && fast_div_ok(sc[j]);
            if (tg == 0 && c0 + j < K) sT[mb * ldsT + c0 + j] = sc[j];
        }
        fast = __all_sync(0xffffffffu, fast);               // warp-uniform branch below
        const uint32_t rot = 8u * (tg & 3);
        const bool wrot = tg >= 4;
        uint32_t code[4][4];                                 // [channel][4-token group]
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float x[4][4];                                   // [token][channel]
#pragma unroll
            for (int i = 0; i < 4; ++i) dequant(4 * u + i, x[i]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float y[4];
                if (fast) {
                    const float2 r2 = make_float2(rc[j], rc[j]), ns2 = make_float2(-sc[j], -sc[j]);
                    const float2 a = div_scale2_fast(make_float2(x[0][j], x[1][j]), r2, ns2);
                    const float2 b = div_scale2_fast(make_float2(x[2][j], x[3][j]), r2, ns2);
                    y[0] = a.x; y[1] = a.y; y[2] = b.x; y[3] = b.y;
                } else {
                    const bool f = fast_div_ok(sc[j]);
#pragma unroll
                    for (int e = 0; e < 4; ++e) y[e] = div_scale(x[e][j], sc[j], rc[j], f);
                }
                code[j][u] = cvt_e4m3x2(y[0], y[1]) | (cvt_e4m3x2(y[2], y[3]) << 16);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t* c = code[j];
            // byte r of c is token 16tg + ((r + tg) & 15): rotate the 16 bytes left by tg so that byte
            // k is token 16tg + k (a whole word for tg >= 4, then tg & 3 bytes)
            uint32_t d[4], e[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) d[i] = wrot ? c[(i + 3) & 3] : c[i];
#pragma unroll
            for (int i = 0; i < 4; ++i) e[i] = __funnelshift_l(d[(i + 3) & 3], d[i], rot);
            const int64_t ch = c0 + j;
            if (ch < K && m0 < M) {
                uint8_t* dst = qT + ch * ldqT + m0;
                if (m0 + 16 <= M) {
                    *reinterpret_cast<uint4*>(dst) = make_uint4(e[0], e[1], e[2], e[3]);
                } else {
                    for (int b = 0; b < 16 && m0 + b < M; ++b) dst[b] = (uint8_t)(e[b >> 2] >> (8 * (b & 3)));
                }
            }
        }
    }
}

cudaError_t launch_requant_1x128_to_128x1(const uint8_t* q, int64_t ldq, const float* s, int64_t lds, int64_t M, int64_t K,
                                          uint8_t* qT, int64_t ldqT, float* sT, int64_t ldsT, int pow2, cudaStream_t st) {
    using P = RQCfg;
    alignas(64) CUtensorMap tm;
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)M};
    const uint64_t str[1] = {(uint64_t)ldq};
    const uint32_t box[2] = {128, 128};
    if (!make_tmap(&tm, TMAP_U8, 2, q, dims, str, box, 128)) return cudaErrorInvalidValue;   // SWIZZLE_128B
    static bool attr[2][64] = {{false}};   // per instantiation and device
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = pow2 ? k_requant_1x128_to_128x1<true> : k_requant_1x128_to_128x1<false>;
    if (dev < 0 || dev >= 64 || !attr[pow2 ? 1 : 0][dev]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM);
        if (dev >= 0 && dev < 64) attr[pow2 ? 1 : 0][dev] = true;
    }
    const int64_t tiles = ((M + 127) / 128) * ((K + 127) / 128);
    return launch_pdl(kern, grid_for(tiles, 2, 2), P::THREADS, P::SMEM, st, tm, s, lds, M, K, qT, ldqT, sT, ldsT);
}
}  // namespace fp8bs
