// gemm.cu — block-scaled FP8 GEMM with FP32 promotion for B200 (sm_100a).
//
// What it computes (§3.3.2; include/fp8bs.h):
//   D[i,j] (+)= sum_kb  sA(kb,i) * sB(kb,j) * P_kb[i,j],   P_kb = sum_{c in kb} dec(A[i,c]) dec(B[j,c])
// with one scale per N_C = 128 contraction elements.  The paper (H800) promotes WGMMA partials
// to CUDA-core registers every 128 elements; here the promotion interval is the same (forced by
// the per-128 scales) but the machinery is Blackwell's:
//   * TMA (SWIZZLE_128B) stages A and B K-blocks (128 wide) into a shared-memory ring;
//   * one thread issues 4x tcgen05.mma.kind::f8f6f4 (K = 32 each) per K-block into a FRESH
//     TMEM buffer P (FP32; double-buffered so the tensor core runs ahead of the promotion);
//   * 16 promotion warps per CTA read P with tcgen05.ld, multiply by sA(kb,i)*sB(kb,j) and
//     accumulate in registers with packed FFMA2, then write BF16 (RNE) or FP32 (+= for Wgrad);
//   * a scale warp streams sA (and Wgrad's per-column sB) with TMA into its own ring.
// kPair = true: a cluster of 2 CTAs on a TPC runs tcgen05.mma.cta_group::2 with M = 256 (128 rows
// per CTA) and N = BN: each CTA stages its own 128 rows of A and BN/2 rows of B, so per-SM
// shared-memory traffic per MAC halves versus one CTA (the 1-CTA 128x256 tile measured ~53%
// tensor-pipe activity, shared-memory-bandwidth bound).  The leader CTA
// issues the MMAs; both CTAs' TMA loads complete on the leader's barrier; commits multicast to
// both CTAs; promotion warps release a TMEM buffer by arriving on the leader's barrier.
// Warp roles (640 threads): w0 TMA A/B producer, w1 MMA issuer, w2 TMEM allocator, w3 scale
// producer, w4..w19 promotion + epilogue (warpgroup h owns columns [h*BN/4, (h+1)*BN/4)).
// Persistent clusters walk a static tile schedule; the grouped (MoE) variant maps tiles to
// (expert, m-tile, n-tile) from device-side offsets with no host synchronisation.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "sm100.cuh"
#include "internal.h"

namespace fp8bs {

constexpr int BM = 128, BK = 128;     // rows per CTA, K-block (= N_C)
constexpr int kMaxGroups = 1024;

template <int BN, bool kPair>
struct Cfg {
    static constexpr int CS = kPair ? 2 : 1;                // CTAs per cluster
    static constexpr int ROWS = BM * CS;                    // rows per cluster tile
    static constexpr int BROWS = kPair ? BN / 2 : BN;       // B rows staged per CTA
    static constexpr int A_BYTES = BM * BK;
    static constexpr int B_BYTES = BROWS * BK;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int kStages = (196608 / STAGE) > 8 ? 8 : (196608 / STAGE);
    static constexpr int kSStages = 8;
    // TMEM partial buffers: as many BN-column buffers as fit in 512 columns.  The promotion's
    // release of buffer kb gates MMA(kb + NBUF); with N=256 only 2 fit and the release chain
    // (commit -> wake -> TMEM read -> arrive -> wake) exceeds one 512-cycle MMA block, so N=160
    // with 3 buffers is the default dense tile.
    static constexpr int NBUF = 512 / BN;
    static constexpr int TMEM_COLS = 512;
    // sA box: BM + 4 floats starting at the 4-aligned row at or below the CTA's first row (a TMA
    // box must start 16-byte aligned in its inner dimension; grouped tiles start at any row).
    static constexpr int SA_BOX = BM + 4;
    static constexpr int SA_BYTES = 640;                    // >= SA_BOX * 4, multiple of 128
    // per-column sB of the tile for this K-block (Wgrad: TMA; Fprop/Dgrad: expanded from the
    // 128-column block scalars by the scale warp); TMA destinations must be 128-byte aligned
    static constexpr int SB_BYTES = (BN * 4 + 127) / 128 * 128;
    static constexpr int SSTAGE = SA_BYTES + SB_BYTES;
    static_assert(SSTAGE % 128 == 0 && STAGE % 1024 == 0, "TMA smem destinations need 128 B (1024 B swizzled) alignment");
    // 4 promotion warpgroups (16 warps): TMEM->register bandwidth and FFMA2 issue both scale with
    // the number of warps (tools/microbench.cu: 322 B/clk at 8 warps, ~470 at 16).
    static constexpr int NWG = 4;
    static constexpr int THREADS = 128 * (1 + NWG);
    static constexpr int NC = BN / NWG;                     // columns per promotion thread
    static_assert(NC % 8 == 0, "promotion slices are multiples of 8 columns");
    static constexpr bool kOneShot = NC <= 40;              // load the whole slice, then one wait
    static constexpr int REG_OTHER = 40, REG_PROMO = 104;   // setmaxnreg split of the 96 x 640 pool
    static constexpr int OFF_SS = kStages * STAGE;
    static constexpr int OFF_BAR = OFF_SS + kSStages * SSTAGE;
    static constexpr int NBAR = 2 * kStages + 2 * kSStages + 2 * NBUF;
    static constexpr int OFF_GRP = OFF_BAR + NBAR * 8 + 16;
    static constexpr int SMEM_DENSE = 1024 + OFF_GRP;
    static constexpr int SMEM_GROUPED = 1024 + OFF_GRP + 2 * (kMaxGroups + 1) * 4;
};

struct KParams {
    int M, N, K, KB;
    int num_m, num_n;
    const float* sB;              // FPROP/DGRAD/grouped block scalars
    int64_t sb_nb_stride, sb_kb_stride, sb_expert_stride;
    int NB;                       // ceil(N/128)
    void* D; int64_t ldd; int accumulate;
    int G; const int64_t* offsets;
    int gm;                       // raster band height in m-tiles (dense)
    int debug;                    // experiments only (FP8BS_GEMM_DEBUG): 1 skip promotion math,
                                  // 2 skip MMAs, 4 TMA always re-reads K-block 0 (L2-resident),
                                  // 8 load A only, 16 record clock64 timestamps of CTA 0
    unsigned long long* ts;       // [8][kTsN] timestamps (debug & 16)
};
constexpr int kTsN = 512;
constexpr int kTsSlots = 12;
#define FP8BS_TS(slot, kb) do { if ((p.debug & 16) && blockIdx.x == 0 && (kb) < kTsN) p.ts[(slot) * kTsN + (kb)] = clock64(); } while (0)

struct Tile { int row0, row_end, n0, e; };   // row0: first row of the CLUSTER tile

template <int ROWS>
__device__ __forceinline__ bool get_tile_dense(const KParams& p, int t, Tile& tl) {
    if (t >= p.num_m * p.num_n) return false;
    // banded raster: m-fastest inside bands of gm m-tiles whose A rows fit in L2, so A is read from
    // DRAM once per band instead of once per group of concurrent n-tiles (ncu: Dgrad read 627 MB,
    // Wgrad 1.05 GB of DRAM with plain m-fastest order)
    const int band = t / (p.gm * p.num_n);
    const int gmb = min(p.gm, p.num_m - band * p.gm);
    const int local = t - band * p.gm * p.num_n;
    const int m = band * p.gm + local % gmb, n = local / gmb;
    tl.row0 = m * ROWS; tl.row_end = p.M; tl.n0 = n; tl.e = 0;   // n0 is scaled by BN by the caller
    return true;
}

// cum[e] = number of tiles of experts < e; off[e] = first row of expert e.
template <int ROWS>
__device__ __forceinline__ bool get_tile_grouped(const KParams& p, const int* cum, const int* off, int t, Tile& tl) {
    if (t >= cum[p.G]) return false;
    int lo = 0, hi = p.G;                       // find e: cum[e] <= t < cum[e+1]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (cum[mid] <= t) lo = mid; else hi = mid;
    }
    const int e = lo;
    const int seg = off[e + 1] - off[e];
    const int mt = (seg + ROWS - 1) / ROWS;
    const int local = t - cum[e];
    const int m = local % mt, n = local / mt;
    tl.row0 = off[e] + m * ROWS; tl.row_end = off[e + 1]; tl.n0 = n; tl.e = e;
    return true;
}

template <int BN, bool kWgrad, bool kOutF32, bool kGrouped, bool kPair>
__global__ void __launch_bounds__(Cfg<BN, kPair>::THREADS, 1)
k_gemm_bs(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
          const __grid_constant__ CUtensorMap tmSA, const __grid_constant__ CUtensorMap tmSB,
          const KParams p) {
    using C = Cfg<BN, kPair>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + C::OFF_BAR;
    auto full_bar   = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar  = [&](int s) { return bar0 + 8u * (C::kStages + s); };
    auto sfull_bar  = [&](int s) { return bar0 + 8u * (2 * C::kStages + s); };
    auto sempty_bar = [&](int s) { return bar0 + 8u * (2 * C::kStages + C::kSStages + s); };
    auto pfull_bar  = [&](int b) { return bar0 + 8u * (2 * C::kStages + 2 * C::kSStages + b); };
    auto pempty_bar = [&](int b) { return bar0 + 8u * (2 * C::kStages + 2 * C::kSStages + C::NBUF + b); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_BAR + C::NBAR * 8);
    int* cum = reinterpret_cast<int*>(smem + C::OFF_GRP);
    int* off = cum + (kMaxGroups + 1);

    // warp index broadcast from lane 0 so the compiler knows role branches are warp-uniform
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const uint32_t rank = kPair ? cluster_ctarank() : 0u;
    const int cid = blockIdx.x / C::CS, ncl = gridDim.x / C::CS;

    if (threadIdx.x == 32) {
        for (int s = 0; s < C::kStages; ++s) { mbar_init(full_bar(s), 1); mbar_init(empty_bar(s), 1); }
        for (int s = 0; s < C::kSStages; ++s) { mbar_init(sfull_bar(s), 1); mbar_init(sempty_bar(s), 4 * C::NWG); }
        for (int b = 0; b < C::NBUF; ++b) { mbar_init(pfull_bar(b), 1); mbar_init(pempty_bar(b), 4 * C::NWG * C::CS); }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); tma_prefetch_desc(&tmSA);
        if (kWgrad) tma_prefetch_desc(&tmSB);
    }
    if (warp == 2) {
        if constexpr (kPair) tmem_alloc_pair<C::TMEM_COLS>(smem_u32(tmem_slot));
        else tmem_alloc<C::TMEM_COLS>(smem_u32(tmem_slot));
    }
    if constexpr (kGrouped) {
        if (warp == 4) {
            // tile prefix over experts: cum[e+1] = cum[e] + ceil(M_e/ROWS) * num_n
            const int G = p.G;
            const int per = (G + 31) / 32;
            const int e0 = lane * per, e1 = min(G, e0 + per);
            int local = 0;
            for (int e = e0; e < e1; ++e) {
                const int64_t a = p.offsets[e], b = p.offsets[e + 1];
                const int seg = b > a ? (int)(b - a) : 0;
                off[e] = (int)a;
                local += ((seg + C::ROWS - 1) / C::ROWS) * p.num_n;
            }
            int incl = local;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            int run = incl - local;
            for (int e = e0; e < e1; ++e) {
                cum[e] = run;
                const int a = off[e];
                const int64_t b = p.offsets[e + 1];
                const int seg = b > a ? (int)(b - a) : 0;
                run += ((seg + C::ROWS - 1) / C::ROWS) * p.num_n;
            }
            if (lane == 31) { cum[G] = incl; off[G] = (int)p.offsets[G]; }
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (kPair) cluster_sync();        // peer barriers initialised before any remote arrive / TMA
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto next_tile = [&](int t, Tile& tl) -> bool {
        bool ok;
        if constexpr (kGrouped) ok = get_tile_grouped<C::ROWS>(p, cum, off, t, tl);
        else ok = get_tile_dense<C::ROWS>(p, t, tl);
        tl.n0 *= BN;
        return ok;
    };

    if (warp < 4) {
        setmaxnreg_dec<C::REG_OTHER>();
        // Producer and MMA roles run on the WHOLE warp (all lanes keep identical, provably uniform
        // values) and only the issuing instructions are under elect.sync.  With the loops on lane 0
        // alone, ptxas wrapped every tcgen05.mma in an ELECT / R2UR.BROADCAST waterfall loop:
        // ~100 cycles per MMA instruction and ~600 per K-block of issue (measured with clock64).
        if (warp == 0) {
            // ---------------- TMA producer: A and B K-blocks (this CTA's halves) ----------------
            int it = 0;
            Tile tl;
            for (int t = cid; next_tile(t, tl); t += ncl) {
                const int arow = tl.row0 + (int)rank * BM;
                const int brow = tl.n0 + (int)rank * C::BROWS;
                for (int kb = 0; kb < p.KB; ++kb, ++it) {
                    const int s = it % C::kStages;
                    const uint32_t ph = (it / C::kStages) & 1;
                    mbar_wait(empty_bar(s), ph ^ 1);
                    const uint32_t sa = sbase + s * C::STAGE;
                    const int kc = kb * BK;
                    if (elect_one()) {
                        if constexpr (kPair) {
                            if (rank == 0) mbar_arrive_expect_tx(full_bar(s), 2 * C::STAGE);
                            tma_load_2d_pair(sa, &tmA, full_bar(s), kc, arow);
                            if constexpr (kGrouped) tma_load_3d_pair(sa + C::A_BYTES, &tmB, full_bar(s), kc, brow, tl.e);
                            else tma_load_2d_pair(sa + C::A_BYTES, &tmB, full_bar(s), kc, brow);
                        } else {
                            mbar_arrive_expect_tx(full_bar(s), C::STAGE);
                            tma_load_2d(sa, &tmA, full_bar(s), kc, arow);
                            if constexpr (kGrouped) tma_load_3d(sa + C::A_BYTES, &tmB, full_bar(s), kc, brow, tl.e);
                            else tma_load_2d(sa + C::A_BYTES, &tmB, full_bar(s), kc, brow);
                        }
                    }
                    __syncwarp();
                }
            }
        } else if (warp == 1) {
          if (rank == 0) {
            // ---------------- MMA issuer (leader CTA) ----------------
            constexpr uint32_t idesc = idesc_e4m3_f32(C::ROWS, BN);
            int it = 0, pit = 0;
            Tile tl;
            for (int t = cid; next_tile(t, tl); t += ncl) {
                for (int kb = 0; kb < p.KB; ++kb, ++it, ++pit) {
                    const int s = it % C::kStages;
                    const uint32_t ph = (it / C::kStages) & 1;
                    const int pb = pit % C::NBUF;
                    const uint32_t pph = (pit / C::NBUF) & 1;
                    if (!(p.debug & 64)) mbar_wait(pempty_bar(pb), pph ^ 1);
                    FP8BS_TS(0, pit);
                    mbar_wait(full_bar(s), ph);
                    FP8BS_TS(1, pit);
                    tc_fence_after();
                    const uint32_t sa = sbase + s * C::STAGE;
                    const uint64_t ad = sdesc_k_sw128(sa), bd = sdesc_k_sw128(sa + C::A_BYTES);
                    const uint32_t d = tmem_base + pb * BN;
                    if (elect_one()) {
                        if (!(p.debug & 2)) {
#pragma unroll
                            for (int k = 0; k < BK / 32; ++k) {
                                if constexpr (kPair) mma_f8f6f4_pair(d, ad + 2 * k, bd + 2 * k, idesc, k > 0 ? 1u : 0u);
                                else mma_f8f6f4(d, ad + 2 * k, bd + 2 * k, idesc, k > 0 ? 1u : 0u);
                                FP8BS_TS(8 + k, pit);
                            }
                        }
                        if constexpr (kPair) {
                            mma_commit_pair(empty_bar(s), 3);
                            mma_commit_pair(pfull_bar(pb), 3);
                        } else {
                            mma_commit(empty_bar(s));
                            mma_commit(pfull_bar(pb));
                        }
                        FP8BS_TS(2, pit);
                    }
                    __syncwarp();
                }
            }
          }
        } else if (warp == 3) {
            // ---------------- scale producer (this CTA's rows; the tile's per-column sB) ----------------
            int sit = 0;
            if (p.debug & 512) return;   // experiment: no scale ring traffic (promotion uses stale scales)
            Tile tl;
            for (int t = cid; next_tile(t, tl); t += ncl) {
                const float* sbp = p.sB;
                if constexpr (kGrouped) sbp += (int64_t)tl.e * p.sb_expert_stride;
                const int arow = tl.row0 + (int)rank * BM;
                const int nb0 = tl.n0 / 128;
                for (int kb0 = 0; kb0 < p.KB; kb0 += 32) {
                    // lane j holds the <= 3 block scalars the tile's columns need at K-block kb0 + j
                    float v[3] = {0.0f, 0.0f, 0.0f};
                    if constexpr (!kWgrad) {
                        const int kb = kb0 + lane;
                        if (kb < p.KB) {
#pragma unroll
                            for (int b = 0; b < 3; ++b)
                                if (nb0 + b < p.NB && b * 128 < (tl.n0 % 128) + BN)
                                    v[b] = __ldg(sbp + (nb0 + b) * p.sb_nb_stride + kb * p.sb_kb_stride);
                        }
                    }
                    const int nk = min(32, p.KB - kb0);
                    for (int j = 0; j < nk; ++j, ++sit) {
                        const int ss = sit % C::kSStages;
                        const uint32_t sph = (sit / C::kSStages) & 1;
                        mbar_wait(sempty_bar(ss), sph ^ 1);          // whole warp: shuffles stay convergent
                        const uint32_t sst = sbase + C::OFF_SS + ss * C::SSTAGE;
                        // Fprop/Dgrad: the <= 3 block scalars of the tile's 128-column weight blocks
                        const float b0 = __shfl_sync(0xffffffffu, v[0], j);
                        const float b1 = __shfl_sync(0xffffffffu, v[1], j);
                        const float b2 = __shfl_sync(0xffffffffu, v[2], j);
                        if (lane == 0) {
                            if constexpr (!kWgrad) {
                                float* sbs = reinterpret_cast<float*>(smem + C::OFF_SS + ss * C::SSTAGE + C::SA_BYTES);
                                sbs[0] = b0; sbs[1] = b1; sbs[2] = b2;
                            }
                            mbar_arrive_expect_tx(sfull_bar(ss), C::SA_BOX * 4 + (kWgrad ? BN * 4 : 0));
                            tma_load_2d(sst, &tmSA, sfull_bar(ss), arow & ~3, kb0 + j);
                            if constexpr (kWgrad) tma_load_2d(sst + C::SA_BYTES, &tmSB, sfull_bar(ss), tl.n0, kb0 + j);
                        }
                        __syncwarp();
                    }
                }
            }
        }
        __syncwarp();
    } else {
        setmaxnreg_inc<C::REG_PROMO>();
        // ---------------- promotion + epilogue ----------------
        const int h = (warp - 4) >> 2;                  // promotion warpgroup = column slice
        const int quad = warp & 3;                      // TMEM lane quadrant
        const int row = quad * 32 + lane;               // row within this CTA's 128
        constexpr int NC = C::NC;
        const uint32_t pempty_addr0 = kPair ? mapa_shared(pempty_bar(0), 0) : pempty_bar(0);
        float acc[NC];
        int sit = 0, pit = 0;
        Tile tl;
        for (int t = cid; next_tile(t, tl); t += ncl) {
            const int arow = tl.row0 + (int)rank * BM;
            // weight block (relative to the tile's first) of this slice's first column, and the number
            // of 8-column groups of the slice that lie in that block
            const int c_first = tl.n0 + h * NC;
            const int blo = c_first / 128 - tl.n0 / 128;
            const int gsplit = (((c_first / 128) + 1) * 128 - c_first) / 8;
#pragma unroll
            for (int i = 0; i < NC; ++i) acc[i] = 0.0f;
            for (int kb = 0; kb < p.KB; ++kb, ++sit, ++pit) {
                const int ss = sit % C::kSStages;
                const uint32_t sph = (sit / C::kSStages) & 1;
                if (!(p.debug & 512)) mbar_wait(sfull_bar(ss), sph);
                const uint32_t sst = sbase + C::OFF_SS + ss * C::SSTAGE;
                const float sa = lds_f32(sst + 4u * ((arow & 3) + row));
                const float2 sa2 = make_float2(sa, sa);
                const uint32_t sbv = sst + C::SA_BYTES + 4u * (h * NC);   // Wgrad: this slice's per-column sB
                // Fprop/Dgrad: the slice spans <= 2 weight blocks; groups of 8 columns before gsplit use
                // f_lo = sA*sB(blo), the rest f_hi = sA*sB(blo+1) (block edges fall on multiples of 8
                // columns: n0 is a multiple of 32 and slices of NC are multiples of 8)
                float f_lo = 0.0f, f_hi = 0.0f;
                if constexpr (!kWgrad) {
                    f_lo = __fmul_rn(sa, lds_f32(sst + C::SA_BYTES + 4u * blo));
                    f_hi = __fmul_rn(sa, lds_f32(sst + C::SA_BYTES + 4u * (blo + 1)));
                }
                const int pb = pit % C::NBUF;
                const uint32_t pph = (pit / C::NBUF) & 1;
                if (lane == 0 && (warp == 4 || warp == C::THREADS / 32 - 1)) FP8BS_TS(warp == 4 ? 3 : 5, pit);
                mbar_wait(pfull_bar(pb), pph);
                if (lane == 0 && (warp == 4 || warp == C::THREADS / 32 - 1)) FP8BS_TS(warp == 4 ? 4 : 6, pit);
                tc_fence_after();
                const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + pb * BN + h * NC;
                auto release_p = [&]() {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (kPair) mbar_arrive_cluster(pempty_addr0 + 8u * pb);
                        else mbar_arrive(pempty_bar(pb));
                        if (warp == C::THREADS / 32 - 1) FP8BS_TS(7, pit);
                    }
                };
                // acc[c0 + j] += P[j] * (sA(kb,row) * sB(kb, col)) for a chunk of W columns:
                // Fprop/Dgrad one FFMA2 per column pair; Wgrad FMUL2 + FFMA2 (outer-product scales)
                auto fma_chunk = [&](const uint32_t* r, int c0, int W) {
                    if constexpr (!kWgrad) {
#pragma unroll
                        for (int g = 0; g < W / 8; ++g) {
                            const float f = ((c0 >> 3) + g < gsplit) ? f_lo : f_hi;
                            const float2 f2 = make_float2(f, f);
#pragma unroll
                            for (int j = 8 * g; j < 8 * g + 8; j += 2) {
                                const float2 a = __ffma2_rn(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), f2,
                                                            make_float2(acc[c0 + j], acc[c0 + j + 1]));
                                acc[c0 + j] = a.x; acc[c0 + j + 1] = a.y;
                            }
                        }
                        return;
                    }
#pragma unroll
                    for (int j4 = 0; j4 < W / 4; ++j4) {
                        const float4 b = lds_f32x4(sbv + 4u * (c0 + j4 * 4));
                        const int j = c0 + j4 * 4;
                        const float2 fa = __fmul2_rn(sa2, make_float2(b.x, b.y));
                        const float2 fb = __fmul2_rn(sa2, make_float2(b.z, b.w));
                        const float2 a0 = __ffma2_rn(make_float2(__uint_as_float(r[j4 * 4 + 0]), __uint_as_float(r[j4 * 4 + 1])), fa,
                                                     make_float2(acc[j + 0], acc[j + 1]));
                        const float2 a1 = __ffma2_rn(make_float2(__uint_as_float(r[j4 * 4 + 2]), __uint_as_float(r[j4 * 4 + 3])), fb,
                                                     make_float2(acc[j + 2], acc[j + 3]));
                        acc[j + 0] = a0.x; acc[j + 1] = a0.y; acc[j + 2] = a1.x; acc[j + 3] = a1.y;
                    }
                };
                if (p.debug & 1) {
                    release_p();
                } else if constexpr (C::kOneShot) {
                    // whole slice in flight at once, one wait, release the buffer, then the math
                    uint32_t r[NC];
#pragma unroll
                    for (int c = 0; c + 32 <= NC; c += 32) FP8BS_TMEM_LD32(taddr + c, (r + c));
                    if constexpr (NC % 32 >= 16) FP8BS_TMEM_LD16(taddr + NC / 32 * 32, (r + NC / 32 * 32));
                    if constexpr (NC % 16 == 8) FP8BS_TMEM_LD8(taddr + NC - 8, (r + NC - 8));
                    tmem_ld_wait();
                    release_p();
                    fma_chunk(r, 0, NC);
                } else {
                    constexpr int CW = 16;
#pragma unroll
                    for (int c = 0; c < NC / CW; ++c) {
                        uint32_t r[CW];
                        FP8BS_TMEM_LD16(taddr + c * CW, r);
                        tmem_ld_wait();
                        if (c == NC / CW - 1) release_p();
                        fma_chunk(r, c * CW, CW);
                    }
                }
                __syncwarp();
                if (lane == 0 && !(p.debug & 512)) mbar_arrive(sempty_bar(ss));
            }
            // ---------------- epilogue ----------------
            const int grow = arow + row;
            if (grow < tl.row_end) {
                const int col0 = tl.n0 + h * NC;
                if constexpr (kOutF32) {
                    float* drow = reinterpret_cast<float*>(p.D) + (int64_t)grow * p.ldd + col0;
#pragma unroll
                    for (int i = 0; i < NC / 4; ++i) {
                        if (col0 + 4 * i < p.N) {
                            float4 v = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
                            if (p.accumulate) {
                                const float4 o = *reinterpret_cast<const float4*>(drow + 4 * i);
                                v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
                            }
                            *reinterpret_cast<float4*>(drow + 4 * i) = v;
                        }
                    }
                } else {
                    __nv_bfloat16* drow = reinterpret_cast<__nv_bfloat16*>(p.D) + (int64_t)grow * p.ldd + col0;
#pragma unroll
                    for (int i = 0; i < NC / 8; ++i) {
                        if (col0 + 8 * i < p.N) {
                            uint32_t w[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                __nv_bfloat162 b2 = __floats2bfloat162_rn(acc[8 * i + 2 * k], acc[8 * i + 2 * k + 1]);
                                w[k] = *reinterpret_cast<uint32_t*>(&b2);
                            }
                            *reinterpret_cast<uint4*>(drow + 8 * i) = make_uint4(w[0], w[1], w[2], w[3]);
                        }
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (kPair) cluster_sync();        // no CTA leaves while its peer may still arrive on it
    if (warp == 2) {
        tc_fence_after();
        if constexpr (kPair) tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
        else tmem_dealloc<C::TMEM_COLS>(tmem_base);
    }
}

// ===========================================================================================
// host side: tensor maps + launch
// ===========================================================================================
static bool make_map(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base, const uint64_t* dims,
                     const uint64_t* strides_bytes /* rank-1 */, const uint32_t* box, CUtensorMapSwizzle sw) {
    const int d = dt == CU_TENSOR_MAP_DATA_TYPE_UINT8 ? TMAP_U8 : TMAP_F32;
    return make_tmap(m, d, rank, base, dims, strides_bytes, box, sw == CU_TENSOR_MAP_SWIZZLE_128B ? 128 : 0);
}

static unsigned long long* g_ts = nullptr;   // debug timestamps (FP8BS_GEMM_DEBUG & 16)

template <int BN, bool kWgrad, bool kOutF32, bool kGrouped, bool kPair>
static cudaError_t launch_cfg(const GemmArgs& a, cudaStream_t st, const char** detail) {
    using C = Cfg<BN, kPair>;
    const int KB = (int)(a.K / BK);
    const int64_t rows = a.M;   // total rows of A (total_M for grouped)
    CUtensorMap tA, tB, tSA, tSB;
    {
        uint64_t dims[2] = {(uint64_t)a.K, (uint64_t)rows};
        uint64_t str[1] = {(uint64_t)a.lda};
        uint32_t box[2] = {BK, BM};
        if (!make_map(&tA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, a.A, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) {
            *detail = "cuTensorMapEncodeTiled failed for A"; return cudaErrorInvalidValue;
        }
    }
    if (kGrouped) {
        uint64_t dims[3] = {(uint64_t)a.K, (uint64_t)a.N, (uint64_t)a.G};
        uint64_t str[2] = {(uint64_t)a.K, (uint64_t)a.K * (uint64_t)a.N};
        uint32_t box[3] = {BK, (uint32_t)C::BROWS, 1};
        if (!make_map(&tB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, a.B, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) {
            *detail = "cuTensorMapEncodeTiled failed for B (grouped)"; return cudaErrorInvalidValue;
        }
    } else {
        uint64_t dims[2] = {(uint64_t)a.K, (uint64_t)a.N};
        uint64_t str[1] = {(uint64_t)a.ldb};
        uint32_t box[2] = {BK, (uint32_t)C::BROWS};
        if (!make_map(&tB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, a.B, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) {
            *detail = "cuTensorMapEncodeTiled failed for B"; return cudaErrorInvalidValue;
        }
    }
    {
        uint64_t dims[2] = {(uint64_t)rows, (uint64_t)KB};
        uint64_t str[1] = {(uint64_t)a.ldsA * 4};
        uint32_t box[2] = {C::SA_BOX, 1};
        if (!make_map(&tSA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a.sA, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE)) {
            *detail = "cuTensorMapEncodeTiled failed for sA"; return cudaErrorInvalidValue;
        }
    }
    if (kWgrad) {
        uint64_t dims[2] = {(uint64_t)a.N, (uint64_t)KB};
        uint64_t str[1] = {(uint64_t)a.ldsB * 4};
        uint32_t box[2] = {(uint32_t)BN, 1};
        if (!make_map(&tSB, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a.sB, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE)) {
            *detail = "cuTensorMapEncodeTiled failed for sB"; return cudaErrorInvalidValue;
        }
    } else {
        tSB = tSA;
    }
    KParams p{};
    p.M = (int)a.M; p.N = (int)a.N; p.K = (int)a.K; p.KB = KB;
    p.num_m = (int)((a.M + C::ROWS - 1) / C::ROWS); p.num_n = (int)((a.N + BN - 1) / BN);
    p.NB = (int)((a.N + 127) / 128);
    p.sB = a.sB;
    if (kGrouped) { p.sb_nb_stride = KB; p.sb_kb_stride = 1; p.sb_expert_stride = (int64_t)p.NB * KB; }
    else if (a.layout == 0) { p.sb_nb_stride = a.ldsB; p.sb_kb_stride = 1; p.sb_expert_stride = 0; }
    else { p.sb_nb_stride = 1; p.sb_kb_stride = a.ldsB; p.sb_expert_stride = 0; }
    p.D = a.D; p.ldd = a.ldd; p.accumulate = a.accumulate;
    p.G = a.G; p.offsets = a.offsets;
    {
        // band only when the K extent is long (Dgrad-like: measured -2%); Wgrad-like shapes keep
        // plain m-fastest order (banding measured +4% there)
        const int64_t band_bytes = a.K > 8192 ? (48ll << 20) : (int64_t)1 << 62;   // A rows kept L2-resident per band
        int64_t gm = band_bytes / ((int64_t)C::ROWS * a.K);
        p.gm = (int)(gm < 1 ? 1 : (gm > p.num_m ? p.num_m : gm));
    }
    {
        static int dbg = -1;
        if (dbg < 0) { const char* e = getenv("FP8BS_GEMM_DEBUG"); dbg = e ? atoi(e) : 0; }
        p.debug = dbg;
        if (dbg & 16) {
            if (!g_ts) cudaMalloc(&g_ts, kTsSlots * kTsN * sizeof(unsigned long long));
            cudaMemsetAsync(g_ts, 0, kTsSlots * kTsN * sizeof(unsigned long long), st);
            p.ts = g_ts;
        }
    }

    int64_t tiles_ub;
    if (kGrouped) tiles_ub = ((a.M + C::ROWS - 1) / C::ROWS + a.G) * (int64_t)p.num_n;
    else tiles_ub = (int64_t)p.num_m * p.num_n;
    const int64_t max_clusters = num_sms() / C::CS;
    int clusters = (int)(tiles_ub < max_clusters ? tiles_ub : max_clusters);
    if (clusters < 1) clusters = 1;
    const int smem = kGrouped ? C::SMEM_GROUPED : C::SMEM_DENSE;
    auto kern = k_gemm_bs<BN, kWgrad, kOutF32, kGrouped, kPair>;
    static bool attr[64] = {false};   // per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(clusters * C::CS);
    cfg.blockDim = dim3(C::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C::CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tA, tB, tSA, tSB, p);
    if (e != cudaSuccess) return e;
    return cudaPeekAtLastError();
}

int gemm_variant_override = 0;   // test hook (also FP8BS_GEMM_VARIANT): see launch_gemm

template <int BN, bool kPair>
static cudaError_t launch_v(const GemmArgs& a, cudaStream_t st, const char** detail) {
    if (a.grouped) {
        return a.out_f32 ? launch_cfg<BN, false, true, true, kPair>(a, st, detail)
                         : launch_cfg<BN, false, false, true, kPair>(a, st, detail);
    }
    if (a.layout == 2) return launch_cfg<BN, true, true, false, kPair>(a, st, detail);
    return a.out_f32 ? launch_cfg<BN, false, true, false, kPair>(a, st, detail)
                     : launch_cfg<BN, false, false, false, kPair>(a, st, detail);
}

// Variants: 1 = 1-CTA N=128 (4 TMEM buffers), 2 = 1-CTA N=256 (2), 3 = CTA pair N=256 (2),
//           4 = CTA pair N=160 (3), 5 = 1-CTA N=160 (3).
cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t st, const char** detail) {
    static int env_variant = -1;   // FP8BS_GEMM_VARIANT (experiments only; read once)
    if (env_variant < 0) {
        const char* e = getenv("FP8BS_GEMM_VARIANT");
        env_variant = e ? atoi(e) : 0;
    }
    int v = env_variant ? env_variant : gemm_variant_override;
    if (v < 1 || v > 5) {
        // measured on B200 (tools/gemm_perf.py, C1 shapes): pair N=256 is fastest for large M;
        // ~128-row experts / small M waste half of a 256-row pair tile -> 1-CTA N=256.
        if (a.N <= 128) v = 1;
        else if (a.grouped) v = (a.M / (a.G > 0 ? a.G : 1) >= 256) ? 3 : 2;
        else v = (a.M <= 128) ? 2 : 3;
    }
    switch (v) {
        case 1: return launch_v<128, false>(a, st, detail);
        case 2: return launch_v<256, false>(a, st, detail);
        case 3: return launch_v<256, true>(a, st, detail);
        case 5: return launch_v<160, false>(a, st, detail);
        default: return launch_v<160, true>(a, st, detail);
    }
}

}  // namespace fp8bs

// Experiments only (not in include/fp8bs.h): copy the debug timestamps of the last GEMM launch.
extern "C" __attribute__((visibility("default"))) int fp8bs_internal_debug_timestamps(unsigned long long* host, int n) {
    if (!fp8bs::g_ts) return 0;
    if (n > fp8bs::kTsSlots * fp8bs::kTsN) n = fp8bs::kTsSlots * fp8bs::kTsN;
    cudaDeviceSynchronize();
    cudaMemcpy(host, fp8bs::g_ts, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    return n;
}
