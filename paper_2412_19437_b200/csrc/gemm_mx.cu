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
// One CTA per 128 x 224 output tile (persistent); CTAs run in clusters of two on m tiles 2u, 2u + 1 of
// the same n tile, each loading half of the shared B tile and multicasting it into both (L2 -> SM
// operand traffic 44 -> 30 KB per K-block per SM):
//   w0  TMA producer: A (128 x 128 B) and its B half (112 x 128 B, multicast) into a 4-stage ring; a
//       stage is refilled only when both CTAs' MMAs have read it;
//   w1, w3, w8, w9  scale-factor producers, one per ring stage (a warp's K-blocks are a ring cycle
//       apart, so its parity waits never alias): per K-block the UE8M0 atoms in the stage (SFA: 32
//       lanes x 16 B, byte [r1][t] = row l + 32 r1; SFB the same for columns, two atoms) from FP32
//       scales loaded a ring cycle ahead and converted only after the wait;
//   w2  MMA issuer: tcgen05.cp.32x128b.warpx4 of the three atoms into TMEM, then 4 block-scaled MMAs
//       (K = 32, sf_id = K-step) into one of two 224-column accumulators; commits release the stage
//       in both CTAs and, after the last K-block, hand the accumulator to the epilogue
//       (tools/mx_probe.cu pins the scale-factor TMEM layout: row l + 32 r1 -> lane l of every
//       quadrant, column + r1, byte t);
//   w4..w7 epilogue: each drains its lane quadrant (32 rows x 224 columns) in 32-column chunks through
//       a staging buffer and TMA stores (reduce-add for Wgrad accumulate), then frees the accumulator.
// TMEM: 2 x 224 accumulator columns + 12 scale-factor columns (512 allocated).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "sm100.cuh"
#include "internal.h"

#ifndef FP8BS_MX_PF
#define FP8BS_MX_PF 1    // owned K-blocks whose scales are in flight ahead of the one being written (2, 3: same speed)
#endif
#ifndef FP8BS_MX_NFAST
#define FP8BS_MX_NFAST 2 // tile order: 0 m fastest, 1 n fastest, 2 n fastest when M > N (the smaller operand re-streams from L2)
#endif
#ifndef FP8BS_MX_MC
#define FP8BS_MX_MC 1    // CTA pairs along M sharing each B tile by TMA multicast (0: independent CTAs)
#endif
#ifndef FP8BS_MX_GPAIR_ROWS
// grouped Fprop/Dgrad: CTA pairs from this many rows per expert on average.  Uniform top-8 routing, 256
// experts, K = 7168, N = 2048 (tools/grouped_mx_sweep.py, r02; one CTA / pair, ms): 128 rows 0.835 /
// 0.994, 160: 1.041 / 0.994, 192: 1.047 / 1.000, 224: 1.068 / 1.021
#define FP8BS_MX_GPAIR_ROWS 144
#endif
#ifndef FP8BS_MX_2CTA
#define FP8BS_MX_2CTA 1  // the CTA pairs run tcgen05.mma.cta_group::2 (M = 256, each CTA stages half of B) instead of
                         // two cta_group::1 MMAs over a multicast full B
#endif
#ifndef FP8BS_MX_2CTA_RELCL
#define FP8BS_MX_2CTA_RELCL 0   // cluster-scope release/acquire on the SF atoms' handoff (a MEMBAR per K-block)
#endif
#ifndef FP8BS_MX_DBG
#define FP8BS_MX_DBG 0   // experiments (tools/): 1 = skip the output stores, 2 = constant scale atoms (no loads)
#endif

#ifndef FP8BS_BAND_MB
#define FP8BS_BAND_MB 48   // L2 budget of the resident operand's band (raster)
#endif

namespace fp8bs {
namespace mx {

constexpr int BM = 128, BN = 224, BK = 128;
#ifndef FP8BS_MX_STAGES
#define FP8BS_MX_STAGES 4
#endif
#ifndef FP8BS_MX_EPIBUF
#define FP8BS_MX_EPIBUF 2
#endif
constexpr int STAGES = FP8BS_MX_STAGES;           // 3 or 4
constexpr int EPIBUF = FP8BS_MX_EPIBUF;           // staging buffers per epilogue warp (2 or 4)
constexpr int A_BYTES = BM * BK;                 // 16 KB
constexpr int B_BYTES = BN * BK;                 // 28 KB
constexpr int SF_BYTES = 3 * 512;                // SFA atom + 2 SFB atoms
constexpr int STAGE = ((A_BYTES + B_BYTES + SF_BYTES + 1023) / 1024) * 1024;
constexpr int EPI_WARP = EPIBUF * 32 * 128;      // 32 rows x 128 B staging buffers per epilogue warp
constexpr int OFF_EPI = STAGES * STAGE;
constexpr int OFF_BAR = OFF_EPI + 4 * EPI_WARP;
constexpr int kTQ = 4;                           // grouped: ring of dynamically claimed tile indices
constexpr int NBAR = 2 * STAGES + 4 + 2 * kTQ;   // full, empty, accfull[2], accempty[2], tqfull, tqempty
constexpr int OFF_TQ = OFF_BAR + NBAR * 8 + 16;  // (after the barriers and the TMEM address)
constexpr int SMEM = 1024 + OFF_TQ + kTQ * 4;
constexpr int MAX_G = 1024;                       // grouped: cum[G + 1], off[G + 1] after the ring
constexpr int OFF_GRP = OFF_TQ + 16;
constexpr int SMEM_G = 1024 + OFF_GRP + 2 * (MAX_G + 1) * 4;
static_assert(SMEM_G <= 232448, "shared memory");
constexpr int NSF = STAGES;                      // scale-factor warps 1, 3, 8, 9: warp k owns stage k
constexpr int THREADS = 32 * 10;
constexpr int MX_PF = FP8BS_MX_PF;
constexpr uint32_t ACC_COLS = 256;               // accumulator b at columns [256 b, 256 b + 224)
constexpr uint32_t SF_COL = 480;                 // SFA [480, 484), SFB [484, 492)

struct Params {
    int M, N, K, KB, num_m, num_n, layout, rast_n, gm;
    const float* sA; int64_t ldsA;
    const float* sB; int64_t ldsB;
    int accumulate;
    // grouped (MoE expert Fprop): rows [offsets[e], offsets[e+1]) of A use B[e], sB + e * sb_expert_stride
    int G; const int64_t* offsets; int64_t sb_expert_stride;
    void* D; int64_t ldd;                       // rows crossing an expert's end are stored directly
    int* claim;                                 // grouped: the tile claim counter (caller's workspace, zeroed per launch)
};

// Tile order (as the promotion kernel's banded raster, gemm.cu get_tile_dense): the operand with fewer
// rows stays L2-resident, in bands of gm tiles when it is larger than ~48 MB; inside a band consecutive
// tiles walk the resident operand fastest so concurrent CTAs share each streamed tile through L2.
// (m fastest for Wgrad's 18432 x 7168 read 1.23 GB of DRAM for 104 MB of operands: 2124 TFLOP/s;
// n fastest 2421.)
__device__ __forceinline__ void tile_mn(const Params& p, int t, int& m, int& n) {
    const int nres = p.rast_n ? p.num_n : p.num_m, nstr = p.rast_n ? p.num_m : p.num_n;
    const int band = t / (p.gm * nstr);
    const int gb = min(p.gm, nres - band * p.gm);
    const int local = t - band * p.gm * nstr;
    const int ires = band * p.gm + local % gb, istr = local / gb;
    m = p.rast_n ? istr : ires;
    n = p.rast_n ? ires : istr;
}

__device__ __forceinline__ uint32_t ue8m0(float s) { return (__float_as_uint(s) >> 23) & 0xFFu; }

__device__ __forceinline__ float scale_b(const Params& p, int kb, int j, int e) {
    if (p.layout == 0) return __ldg(p.sB + (int64_t)e * p.sb_expert_stride + (int64_t)(j >> 7) * p.ldsB + kb);   // FPROP: [(G,) N/128][K/128]
    if (p.layout == 1) return __ldg(p.sB + (int64_t)e * p.sb_expert_stride + (int64_t)kb * p.ldsB + (j >> 7));   // DGRAD: [(G,) K/128][N/128]
    return __ldg(p.sB + (int64_t)kb * p.ldsB + j);                               // WGRAD: [K/128][N]
}

// tcgen05.cp source descriptor: 32 rows x 16 B atom, no swizzle, 8-row core matrices 128 B apart
__device__ __forceinline__ uint64_t cp_desc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void tmem_cp_atom(uint32_t taddr, uint64_t desc) {
    asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" :: "r"(taddr), "l"(desc) : "memory");
}
// cta_group::2 (issued by the pair's leader): each CTA's atom at the same shared-memory offset into the
// same TMEM columns of that CTA
__device__ __forceinline__ void tmem_cp_atom_pair(uint32_t taddr, uint64_t desc) {
    asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" :: "r"(taddr), "l"(desc) : "memory");
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

// Issued by the pair's leader: D (both CTAs' TMEM, 128 lanes each) (+)= A (128 rows per CTA) x B (N/2 rows per
// CTA), block-scaled with each CTA's SFA (its rows) and SFB (all N columns, duplicated in both CTAs)
__device__ __forceinline__ void mma_mx_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa, uint32_t sfb, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
                 :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}

__device__ __forceinline__ void tma_load_3d_mc(uint32_t dst, const void* tmap, uint32_t bar, int32_t c0, int32_t c1, int32_t c2, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;"
        :: "r"(dst), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "h"(mask) : "memory");
}

struct MxTile { int m0, n0, e, row_end, kb0, kbn; };

// Grouped Wgrad (one launch over every expert): expert e's 128-token blocks in the padded layout, .x =
// first block, .y = blocks (0 for an expert without tokens).  Kernel parameter space (8 KB at 1024).
template <int kG>
struct GWs { int2 e[kG]; };
constexpr int kGWMax = 1024;

// Arrive once on the barrier at this offset in both CTAs of the pair when the MMAs complete.
__device__ __forceinline__ void mma_commit_mc(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(bar), "h"((uint16_t)3) : "memory");
}

// kGW: grouped Wgrad — tiles (expert, m, n) with m fastest inside an expert, each contracting over its
// expert's own token blocks gw.e[e]; output rows of expert e at e * M (D = [G x M, N]).
template <bool kOutF32, bool kMc, bool kGrouped, bool kGW>
__global__ void __launch_bounds__(THREADS, 1)
k_gemm_mx(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
          const __grid_constant__ CUtensorMap tmD, const Params p, const __grid_constant__ GWs<kGW ? kGWMax : 1> gw) {
    static_assert(!(kGW && kGrouped), "grouped Wgrad has its own tile map");
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
    auto tqfull_bar = [&](int q) { return bar0 + 8u * (2 * STAGES + 4 + q); };
    auto tqempty_bar = [&](int q) { return bar0 + 8u * (2 * STAGES + 4 + kTQ + q); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + NBAR * 8);
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    // kMc: the two CTAs of a cluster take m tiles 2u and 2u + 1 of the same n tile; each loads its
    // half of the B tile and multicasts it into both, so a stage is free only when BOTH CTAs' MMAs
    // have read it (each commit arrives on the empty barrier of both CTAs: count 2)
    constexpr int MC = kMc ? 2 : 1;
    // k2: the pair runs 2-CTA MMAs issued by the leader: each CTA stages its A rows and HALF of the B tile
    // (TMA completing on the leader's full barrier), its SF atoms (own rows' SFA, all columns' SFB), and
    // the leader's commits free both CTAs' stages and hand both CTAs their accumulator rows
    constexpr bool k2 = kMc && FP8BS_MX_2CTA;
    const uint32_t rank = kMc ? cluster_ctarank() : 0;
    const int cid = kMc ? (int)(blockIdx.x >> 1) : (int)blockIdx.x, ncl = kMc ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    if (threadIdx.x == 0) {
        // k2 (the leader's barriers count): full = its producer + both CTAs' SF warps; empty = the leader's
        // multicast commit; accempty = both CTAs' 4 epilogue warps
        for (int s = 0; s < STAGES; ++s) { mbar_init(full_bar(s), k2 ? 3 : 2); mbar_init(empty_bar(s), k2 ? 1 : MC); }
        for (int b = 0; b < 2; ++b) { mbar_init(accfull_bar(b), 1); mbar_init(accempty_bar(b), k2 ? 8 : 4); }
        // grouped: each claimed index is read by 4 SF + 4 epilogue warps per CTA, the leader's MMA warp
        // and the peer's producer (the leader's producer claims)
        for (int q = 0; q < kTQ; ++q) { mbar_init(tqfull_bar(q), 1); mbar_init(tqempty_bar(q), kMc ? 18 : 9); }
        fence_mbar_init();
    }
    if (warp == 2) {
        if constexpr (k2) tmem_alloc_pair<512>(smem_u32(tmem_slot));
        else tmem_alloc<512>(smem_u32(tmem_slot));
    }
    int* cum = reinterpret_cast<int*>(smem + OFF_GRP);    // grouped: units of experts < e
    int* off = cum + (MAX_G + 1);                         // grouped: first row of expert e
    if constexpr (kGrouped) {
        if (warp == 4) {
            // unit prefix over experts: cum[e+1] = cum[e] + ceil(M_e / (MC * BM)) * num_n
            const int G = p.G, per = (G + 31) / 32;
            const int e0 = lane * per, e1 = min(G, e0 + per);
            int local = 0;
            for (int e = e0; e < e1; ++e) {
                const int64_t a = p.offsets[e], b = p.offsets[e + 1];
                off[e] = (int)a;
                local += (int)((b > a ? b - a : 0) + MC * BM - 1) / (MC * BM) * p.num_n;
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
                const int64_t b = p.offsets[e + 1];
                run += (int)((b > off[e] ? b - off[e] : 0) + MC * BM - 1) / (MC * BM) * p.num_n;
            }
            if (lane == 31) { cum[G] = incl; off[G] = (int)p.offsets[G]; }
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (kMc) cluster_sync();              // the peer's barriers exist before any multicast
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int ntiles = kGrouped ? cum[p.G] : kGW ? p.G * p.num_m * p.num_n : p.num_m * p.num_n;
    // Grouped: tiles are claimed dynamically, as in the promotion kernel (gemm.cu): the leader's producer
    // claims the next unit index with an atomic, one ahead, and hands it to every role of both CTAs
    // through a kTQ-entry ring (a static schedule let the persistent clusters drift apart and re-read
    // A from DRAM: 24.2 GB per C4 launch against 7.6).  Every role reads index #j in order and
    // releases the entry at once.  Dense / grouped Wgrad: the static schedule cid, cid + ncl, ...
    uint32_t* tqv = reinterpret_cast<uint32_t*>(smem + OFF_TQ);
    auto tq_publish = [&](int j) -> int {            // leader producer, one lane
        const int q = j % kTQ;
        mbar_wait(tqempty_bar(q), ((j / kTQ) & 1) ^ 1);
        const int t = atomicAdd(p.claim, 1);
        const uint32_t a = smem_u32(tqv + q);
        asm volatile("st.shared.u32 [%0], %1;" :: "r"(a), "r"(t) : "memory");
        mbar_arrive(tqfull_bar(q));
        if constexpr (kMc) {
            st_shared_cluster_u32(mapa_shared(a, 1), (uint32_t)t);
            mbar_arrive_release_cluster(mapa_shared(tqfull_bar(q), 1));
        }
        return t;
    };
    auto tq_take = [&](int j) -> int {               // every other role, whole warp
        const int q = j % kTQ;
        mbar_wait_acquire_cluster(tqfull_bar(q), (j / kTQ) & 1);
        const int t = (int)lds_u32(smem_u32(tqv + q));
        __syncwarp();
        if (elect_one()) {
            if (kMc && rank != 0) mbar_arrive_release_cluster(tqempty_bar(q) & kPeerBitMask);
            else mbar_arrive(tqempty_bar(q));
        }
        __syncwarp();
        return t;
    };
    int t_next = 0;
    auto tile_at = [&](int j) -> int {               // this role's tile #j (>= ntiles: none left)
        if constexpr (!kGrouped) return cid + j * ncl;
        else return tq_take(j);
    };
    auto tile_at_claim = [&](int j) -> int {         // the leader's producer: claims #j + 1 ahead
        if constexpr (!kGrouped) return cid + j * ncl;
        else {
            int t = 0;
            if (lane == 0) {
                t = j == 0 ? tq_publish(0) : t_next;
                if (t < ntiles) t_next = tq_publish(j + 1);
            }
            return __shfl_sync(0xffffffffu, t, 0);
        }
    };
    // unit t -> this CTA's tile: rows [m0, m0 + BM) (clipped at row_end), columns [n0, n0 + BN)
    auto decode = [&](int t, MxTile& tl) {
        if constexpr (kGrouped) {
            int lo = 0, hi = p.G;                       // e: cum[e] <= t < cum[e + 1]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (cum[mid] <= t) lo = mid; else hi = mid;
            }
            const int seg = off[lo + 1] - off[lo];
            const int mt = (seg + MC * BM - 1) / (MC * BM), local = t - cum[lo];
            const bool nfast = seg > p.N;                // as the promotion kernel: smaller operand resident
            const int pm = nfast ? local / p.num_n : local % mt, n = nfast ? local % p.num_n : local / mt;
            tl.m0 = off[lo] + (pm * MC + (int)rank) * BM; tl.n0 = n * BN; tl.e = lo; tl.row_end = off[lo + 1];
            tl.kb0 = 0; tl.kbn = p.KB;
        } else if constexpr (kGW) {
            const int per = p.num_m * p.num_n, e = t / per, l = t - e * per;
            const int pm = l % p.num_m, n = l / p.num_m;
            tl.m0 = (pm * MC + (int)rank) * BM; tl.n0 = n * BN; tl.e = e; tl.row_end = p.M;
            const int2 k = gw.e[e];
            tl.kb0 = k.x; tl.kbn = k.y;
        } else {
            int tm, tn;
            tile_mn(p, t, tm, tn);
            tl.m0 = (tm * MC + (int)rank) * BM; tl.n0 = tn * BN; tl.e = 0; tl.row_end = p.M;
            tl.kb0 = 0; tl.kbn = p.KB;
        }
    };

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); tma_prefetch_desc(&tmD); }
        int it = 0;
        int jj = 0;
        for (int t = rank == 0 ? tile_at_claim(0) : tile_at(0); t < ntiles; ++jj, t = rank == 0 ? tile_at_claim(jj) : tile_at(jj)) {
            MxTile tl;
            decode(t, tl);
            const int m0 = tl.m0, n0 = tl.n0;
            for (int kb = 0; kb < tl.kbn; ++kb, ++it) {
                const int s = it % STAGES;
                mbar_wait(empty_bar(s), ((it / STAGES) & 1) ^ 1);
                if (elect_one()) {
                    const uint32_t st = sbase + s * STAGE;
                    const int kc = (tl.kb0 + kb) * BK;
                    if constexpr (k2) {
                        if (rank == 0) mbar_arrive_expect_tx(full_bar(s), 2 * (A_BYTES + B_BYTES / 2));
                        tma_load_2d_pair(st, &tmA, full_bar(s), kc, m0);
                        if constexpr (kGrouped)
                            tma_load_3d_pair(st + A_BYTES, &tmB, full_bar(s), kc, n0 + (int)rank * (BN / 2), tl.e);
                        else
                            tma_load_2d_pair(st + A_BYTES, &tmB, full_bar(s), kc, n0 + (int)rank * (BN / 2));
                    } else {
                    mbar_arrive_expect_tx(full_bar(s), A_BYTES + B_BYTES);
                    tma_load_2d(st, &tmA, full_bar(s), kc, m0);
                    if constexpr (kMc && kGrouped)
                        tma_load_3d_mc(st + A_BYTES + rank * (B_BYTES / 2), &tmB, full_bar(s), kc, n0 + (int)rank * (BN / 2), tl.e, 3);
                    else if constexpr (kMc)
                        tma_load_2d_mc(st + A_BYTES + rank * (B_BYTES / 2), &tmB, full_bar(s), kc, n0 + (int)rank * (BN / 2), 3);
                    else if constexpr (kGrouped)
                        tma_load_3d(st + A_BYTES, &tmB, full_bar(s), kc, n0, tl.e);
                    else
                        tma_load_2d(st + A_BYTES, &tmB, full_bar(s), kc, n0);
                    }
                }
                __syncwarp();
            }
        }
        if constexpr (kMc) {
            // the peer's last commits arrive on this CTA's empty barriers: wait for them before exit
            for (int i = 0; i < STAGES; ++i, ++it) mbar_wait(empty_bar(it % STAGES), ((it / STAGES) & 1) ^ 1);
        }
    } else if (warp == 1 || warp == 3 || warp >= 8) {
        // ---------------- scale-factor atoms ----------------
        const int slot = warp == 1 ? 0 : warp == 3 ? 1 : warp - 6;
        if (slot >= NSF) goto done;                     // (3 stages: warp 9 idles)
        // this warp's K-blocks: global iteration it = slot, slot + NSF, ... (tile it / KB of this CTA's
        // sequence, K-block it % KB).  The raw FP32 scales of the next MX_PF owned K-blocks are in flight
        // while the current one waits for its stage: they are converted only after the wait, so no
        // load is consumed at issue (converting at load time stalled each warp on its loads: Wgrad's
        // 1187 TFLOP/s became 2254 with constant atoms)
        // kGW: tiles have different K-block counts, so the CTA's global iteration `it` is mapped to
        // (tile, K-block) with a cursor that only moves forward (load() is called with increasing it)
        int cur_t = kGW ? cid : -1, cur_base = 0;
        MxTile cur_tl;
        int sf_j = -1, sf_t = 0;                       // grouped: the last claimed index this warp read
        auto load = [&](int it, float* fa, float* fb) -> bool {
            int t, kb;
            MxTile tl;
            if constexpr (kGW) {
                for (;;) {
                    if (cur_t >= ntiles) return false;
                    decode(cur_t, tl);
                    if (it < cur_base + tl.kbn) break;
                    cur_base += tl.kbn;
                    cur_t += ncl;
                }
                t = cur_t;
                kb = tl.kb0 + (it - cur_base);
            } else {
                kb = it % p.KB;
                if constexpr (kGrouped) {
                    // walk the claimed indices in order up to tile #(it / KB) (every entry read once)
                    const int jt = it / p.KB;
                    while (sf_j < jt) {
                        if (sf_t >= ntiles) return false;
                        ++sf_j;
                        sf_t = tq_take(sf_j);
                    }
                    t = sf_t;
                } else {
                    t = cid + (it / p.KB) * ncl;
                }
                if (t >= ntiles) return false;
                // the tile changes every KB K-blocks: decode it once (the grouped decode is a binary
                // search over the experts in shared memory)
                if (t != cur_t) { decode(t, cur_tl); cur_t = t; }
                tl = cur_tl;
            }
            (void)t;
            const int m0 = tl.m0, n0 = tl.n0;
#pragma unroll
            for (int r1 = 0; r1 < 4; ++r1) {
                const int i = m0 + lane + 32 * r1;
                fa[r1] = ((FP8BS_MX_DBG & 2) || i >= p.M) ? 1.0f : __ldg(p.sA + (int64_t)kb * p.ldsA + i);
            }
#pragma unroll
            for (int r1 = 0; r1 < 7; ++r1) {
                const int j = n0 + lane + 32 * r1;
                fb[r1] = ((FP8BS_MX_DBG & 2) || j >= p.N) ? 1.0f : scale_b(p, kb, j, tl.e);
            }
            return true;
        };
        constexpr int PF = MX_PF;
        float fa[PF + 1][4], fb[PF + 1][7];
        bool have[PF + 1];
#pragma unroll
        for (int d = 0; d < PF; ++d) have[d] = load(slot + d * NSF, fa[d], fb[d]);
        for (int it = slot; have[0]; it += NSF) {
            have[PF] = load(it + PF * NSF, fa[PF], fb[PF]);    // in flight during the wait below
            const int s = it % STAGES;
            uint8_t* sf = smem + s * STAGE + A_BYTES + B_BYTES;
            uint32_t wa[4], wb[8];
#pragma unroll
            for (int r = 0; r < 4; ++r) wa[r] = ue8m0(fa[0][r]) * 0x01010101u;
#pragma unroll
            for (int r = 0; r < 7; ++r) wb[r] = ue8m0(fb[0][r]) * 0x01010101u;
            wb[7] = 127u * 0x01010101u;                        // columns 224..255 of the atom: unused
            mbar_wait(empty_bar(s), ((it / STAGES) & 1) ^ 1);
            *reinterpret_cast<uint4*>(sf + lane * 16) = make_uint4(wa[0], wa[1], wa[2], wa[3]);
            *reinterpret_cast<uint4*>(sf + 512 + lane * 16) = make_uint4(wb[0], wb[1], wb[2], wb[3]);
            *reinterpret_cast<uint4*>(sf + 1024 + lane * 16) = make_uint4(wb[4], wb[5], wb[6], wb[7]);
            // generic writes -> the async proxy (tcgen05.cp).  k2: the leader's tcgen05.cp.cta_group::2 reads
            // this CTA's atoms, handed over through the leader's mbarrier: the cluster-wide proxy release
            // fence for mbarrier-synchronised handoffs (a CTA-scope MEMBAR; a release.cluster arrive costs a
            // GPU-scope MEMBAR per K-block: 2238 against 2958 TFLOP/s on C1 Fprop)
            if constexpr (k2) asm volatile("fence.proxy.async::generic.release.sync_restrict::shared::cta.cluster;" ::: "memory");
            else fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
#if FP8BS_MX_2CTA_RELCL
                if constexpr (k2) mbar_arrive_release_cluster(mapa_shared(full_bar(s), 0));
#else
                if constexpr (k2) mbar_arrive_cluster(full_bar(s) & kPeerBitMask);
#endif
                else mbar_arrive(full_bar(s));
            }
#pragma unroll
            for (int d = 0; d < PF; ++d) {
                have[d] = have[d + 1];
#pragma unroll
                for (int r = 0; r < 4; ++r) fa[d][r] = fa[d + 1][r];
#pragma unroll
                for (int r = 0; r < 7; ++r) fb[d][r] = fb[d + 1][r];
            }
        }
    } else if (warp == 2) {
        // ---------------- MMA issuer ----------------
        if (k2 && rank != 0) goto done;                 // k2: the leader issues for the pair
        constexpr uint32_t idesc0 = idesc_mx(k2 ? 2 * BM : BM, BN, 0);
        int it = 0, tl = 0;
        for (int t = tile_at(0); t < ntiles; t = tile_at(++tl)) {
            const int b = tl & 1;
            int kbn = p.KB;
            if constexpr (kGW) { MxTile ti; decode(t, ti); kbn = ti.kbn; }
            mbar_wait(accempty_bar(b), ((tl >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d = tmem_base + ACC_COLS * b;
            if (kGW && kbn == 0) {                      // expert without tokens: no MMAs; the epilogue writes 0
                if (elect_one()) {
                    if constexpr (k2) mma_commit_pair(accfull_bar(b), 3);
                    else mma_commit(accfull_bar(b));
                }
                __syncwarp();
                continue;
            }
            for (int kb = 0; kb < kbn; ++kb, ++it) {
                const int s = it % STAGES;
#if FP8BS_MX_2CTA_RELCL
                if constexpr (k2) mbar_wait_acquire_cluster(full_bar(s), (it / STAGES) & 1);
                else
#endif
                mbar_wait(full_bar(s), (it / STAGES) & 1);
                if constexpr (k2) asm volatile("fence.proxy.async::generic.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t st = sbase + s * STAGE;
                    const uint32_t sf = st + A_BYTES + B_BYTES;
                    if constexpr (k2) {
                        tmem_cp_atom_pair(tmem_base + SF_COL, cp_desc(sf));
                        tmem_cp_atom_pair(tmem_base + SF_COL + 4, cp_desc(sf + 512));
                        tmem_cp_atom_pair(tmem_base + SF_COL + 8, cp_desc(sf + 1024));
                    } else {
                        tmem_cp_atom(tmem_base + SF_COL, cp_desc(sf));
                        tmem_cp_atom(tmem_base + SF_COL + 4, cp_desc(sf + 512));
                        tmem_cp_atom(tmem_base + SF_COL + 8, cp_desc(sf + 1024));
                    }
                    const uint64_t ad = sdesc_k_sw128(st), bd = sdesc_k_sw128(st + A_BYTES);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t id = idesc0 | ((uint32_t)k << 4) | ((uint32_t)k << 29);
                        if constexpr (k2)
                            mma_mx_pair(d, ad + 2 * k, bd + 2 * k, id, tmem_base + SF_COL + ((uint32_t)k << 30),
                                        tmem_base + SF_COL + 4 + ((uint32_t)k << 30), (kb > 0 || k > 0) ? 1u : 0u);
                        else
                            mma_mx(d, ad + 2 * k, bd + 2 * k, id, tmem_base + SF_COL + ((uint32_t)k << 30),
                                   tmem_base + SF_COL + 4 + ((uint32_t)k << 30), (kb > 0 || k > 0) ? 1u : 0u);
                    }
                    if constexpr (k2) mma_commit_pair(empty_bar(s), 3);
                    else if constexpr (kMc) mma_commit_mc(empty_bar(s));
                    else mma_commit(empty_bar(s));
                    if (kb == kbn - 1) {
                        if constexpr (k2) mma_commit_pair(accfull_bar(b), 3);
                        else mma_commit(accfull_bar(b));
                    }
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
        for (int t = tile_at(0); t < ntiles; t = tile_at(++tl)) {
            const int b = tl & 1;
            MxTile ti;
            decode(t, ti);
            const int m0 = ti.m0, n0 = ti.n0;
            const int rows_here = ti.row_end - (m0 + quad * 32);     // rows of this warp's 32 in range
            const int orow = kGW ? ti.e * p.M : 0;                   // grouped Wgrad: expert e's output rows
            const bool zero = kGW && ti.kbn == 0;                     // expert without tokens
            mbar_wait(accfull_bar(b), (tl >> 1) & 1);
            tc_fence_after();
            const uint32_t ta = tmem_base + ((uint32_t)(quad * 32) << 16) + ACC_COLS * b;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c, ++chunk) {
                const uint32_t ebuf = ebuf0 + (chunk & (EPIBUF - 1)) * (32 * 128);
                uint32_t v[32];
                FP8BS_TMEM_LD32(ta + 32 * c, v);
                tmem_ld_wait();
                if (c == BN / 32 - 1) {              // the accumulator is in registers: free it
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (k2 && rank != 0) mbar_arrive_cluster(accempty_bar(b) & kPeerBitMask);   // the leader's
                        else mbar_arrive(accempty_bar(b));
                    }
                }
                if (zero) {
                    if (p.accumulate) continue;      // D += 0
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = 0u;
                }
                if ((kGrouped || kGW) && rows_here < 32) {
                    // the expert ends inside this warp's 32 rows (rows past it belong to the next
                    // expert): each lane stores its own row directly
                    const int col = n0 + 32 * c;
                    if (lane < rows_here && col < p.N && !(FP8BS_MX_DBG & 1)) {
                        const int64_t grow = (int64_t)orow + m0 + quad * 32 + lane;
                        const int ncol = min(32, p.N - col);
                        if constexpr (kOutF32) {
                            float* d = reinterpret_cast<float*>(p.D) + grow * p.ldd + col;
                            if (p.accumulate) for (int j = 0; j < ncol; ++j) d[j] += __uint_as_float(v[j]);
                            else for (int j = 0; j < ncol; ++j) d[j] = __uint_as_float(v[j]);
                        } else {
                            __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(p.D) + grow * p.ldd + col;
                            for (int j = 0; j < ncol; ++j) d[j] = __float2bfloat16_rn(__uint_as_float(v[j]));
                        }
                    }
                    continue;
                }
                if (lane == 0) bulk_wait_group_read<EPIBUF - 1>();   // the store that last used this buffer has read it
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
                    if (col < p.N && row < p.M && !(FP8BS_MX_DBG & 1)) {
                        const int srow = orow + row;
                        if (kOutF32 && p.accumulate) tma_reduce_add_2d(&tmD, ebuf, col, srow);
                        else tma_store_2d(&tmD, ebuf, col, srow);
                    }
                    bulk_commit_group();
                }
            }
        }
        if (lane == 0) bulk_wait_group<0>();
    }
done:
    tc_fence_before();
    __syncthreads();
    if constexpr (k2) cluster_sync();           // no CTA leaves while the pair may still arrive on it / use its TMEM
    if (warp == 2) {
        tc_fence_after();
        if constexpr (k2) tmem_dealloc_pair<512>(tmem_base);
        else tmem_dealloc<512>(tmem_base);
    }
}

}  // namespace mx

cudaError_t launch_gemm_mx(const GemmArgs& a, cudaStream_t st, const char** detail) {
    using namespace mx;
    const int KB = (int)(a.K / BK);
    const bool gw = a.grouped && a.layout == 2;   // grouped Wgrad: dense-shaped operands, per-expert K ranges
    CUtensorMap tA, tB, tD;
    {
        const uint64_t dims[2] = {(uint64_t)a.K, (uint64_t)a.M};
        const uint64_t str[1] = {(uint64_t)a.lda};
        const uint32_t box[2] = {BK, BM};
        if (!make_tmap(&tA, TMAP_U8, 2, a.A, dims, str, box, 128)) { *detail = "tensor map A"; return cudaErrorInvalidValue; }
    }
    // grouped (Fprop / Dgrad): CTA pairs (2-CTA MMAs over 256-row units of one expert) when the experts
    // average at least 256 rows (C4); otherwise unpaired: a pair shares one expert's n tile over 2 x 128
    // rows, and at the small-expert MoE shapes that left the second CTA idle (C2: 810 vs 1234 TFLOP/s)
    const bool gpair = a.grouped && !gw && FP8BS_MX_MC && FP8BS_MX_2CTA && a.M / (a.G > 0 ? a.G : 1) >= FP8BS_MX_GPAIR_ROWS;
    if (a.grouped && !gw) {   // B [G][N][K], contiguous
        const uint64_t dims[3] = {(uint64_t)a.K, (uint64_t)a.N, (uint64_t)a.G};
        const uint64_t str[2] = {(uint64_t)a.K, (uint64_t)a.K * (uint64_t)a.N};
        const uint32_t box[3] = {BK, gpair ? BN / 2 : BN, 1};
        if (!make_tmap(&tB, TMAP_U8, 3, a.B, dims, str, box, 128)) { *detail = "tensor map B (grouped)"; return cudaErrorInvalidValue; }
    } else {
        const uint64_t dims[2] = {(uint64_t)a.K, (uint64_t)a.N};
        const uint64_t str[1] = {(uint64_t)a.ldb};
        const uint32_t box[2] = {BK, FP8BS_MX_MC ? BN / 2 : BN};
        if (!make_tmap(&tB, TMAP_U8, 2, a.B, dims, str, box, 128)) { *detail = "tensor map B"; return cudaErrorInvalidValue; }
    }
    {
        // 32 rows x 32 columns per store: FP32 128 B (SWIZZLE_128B staging), BF16 64 B (SWIZZLE_64B)
        const uint64_t esz = a.out_f32 ? 4 : 2;
        const uint64_t dims[2] = {(uint64_t)a.N, (uint64_t)(gw ? a.M * a.G : a.M)};   // grouped Wgrad: experts stacked
        const uint64_t str[1] = {(uint64_t)a.ldd * esz};
        const uint32_t box[2] = {32, 32};
        if (!make_tmap(&tD, a.out_f32 ? TMAP_F32 : TMAP_BF16, 2, a.D, dims, str, box, a.out_f32 ? 128 : 64)) {
            *detail = "tensor map D"; return cudaErrorInvalidValue;
        }
    }
    Params p{};
    p.M = (int)a.M; p.N = (int)a.N; p.K = (int)a.K; p.KB = KB;
    // Grouped runs without CTA pairs: a pair shares one expert's n tile over 2 x 128 rows, and at the
    // MoE shapes most experts have <= 128 rows, which left the second CTA idle (C2: 810 vs 1234
    // TFLOP/s unpaired).
    const int MC = (FP8BS_MX_MC && (!a.grouped || gw || gpair)) ? 2 : 1;
    p.num_m = (int)((a.M + BM * MC - 1) / (BM * MC)); p.num_n = (int)((a.N + BN - 1) / BN);   // m units of MC tiles
    p.rast_n = FP8BS_MX_NFAST == 2 ? (a.M > a.N ? 1 : 0) : FP8BS_MX_NFAST;
    {
        const int64_t res_rows = p.rast_n ? BN : BM * MC, nres = p.rast_n ? p.num_n : p.num_m;
        const int64_t gb = ((int64_t)FP8BS_BAND_MB << 20) / (res_rows * a.K);
        p.gm = (int)(gb < 1 ? 1 : (gb > nres ? nres : gb));
    }
    p.layout = a.layout; p.sA = a.sA; p.ldsA = a.ldsA; p.sB = a.sB; p.ldsB = a.ldsB; p.accumulate = a.accumulate;
    p.G = a.grouped ? a.G : 0; p.offsets = a.offsets; p.sb_expert_stride = (int64_t)((a.N + 127) / 128) * KB;
    if (gw) p.rast_n = 0;   // m fastest inside an expert (decode): its dYqT_e stays in L2 while XqT_e streams
    p.D = a.D; p.ldd = a.ldd;
    p.claim = static_cast<int*>(a.workspace);
    if (a.grouped && !gw) {                       // the claim counter starts at 0 every launch
        if (!a.workspace) { *detail = "grouped UE8M0 GEMM without a workspace"; return cudaErrorInvalidValue; }
        cudaError_t e0 = cudaMemsetAsync(a.workspace, 0, sizeof(int), st);
        if (e0 != cudaSuccess) return e0;
    }
    // grouped: an upper bound on the units (each expert adds at most one partial m unit per n tile)
    const int64_t units = gw ? (int64_t)a.G * p.num_m * p.num_n
                        : a.grouped ? (int64_t)(p.num_m + a.G) * p.num_n : (int64_t)p.num_m * p.num_n;
    const int64_t max_units = num_sms() / MC;
    const int grid = (int)(units < max_units ? units : max_units) * MC;
    constexpr bool kMc = FP8BS_MX_MC != 0;
    if (gw) {
        GWs<kGWMax> g;
        for (int e = 0; e < a.G; ++e) g.e[e] = make_int2(a.gw_kb[2 * e], a.gw_kb[2 * e + 1]);
        auto kern = k_gemm_mx<true, kMc, false, true>;
        static bool attr_gw[64] = {false};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || !attr_gw[dev]) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
            if (e != cudaSuccess) return e;
            if (dev >= 0 && dev < 64) attr_gw[dev] = true;
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(THREADS);
        cfg.dynamicSmemBytes = SMEM;
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = MC; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tA, tB, tD, p, g);
        if (e != cudaSuccess) return e;
        return cudaPeekAtLastError();
    }
    auto kern = a.grouped ? (gpair ? (a.out_f32 ? k_gemm_mx<true, kMc, true, false> : k_gemm_mx<false, kMc, true, false>)
                                   : (a.out_f32 ? k_gemm_mx<true, false, true, false> : k_gemm_mx<false, false, true, false>))
                          : (a.out_f32 ? k_gemm_mx<true, kMc, false, false> : k_gemm_mx<false, kMc, false, false>);
    const int smem = a.grouped ? SMEM_G : SMEM;
    static bool attr[6][64] = {{false}};
    const int ki = (a.out_f32 ? 1 : 0) + (a.grouped ? (gpair ? 4 : 2) : 0);
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[ki][dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) attr[ki][dev] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (internal.h launch_pdl)
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = MC; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    GWs<1> g0;
    g0.e[0] = make_int2(0, 0);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tA, tB, tD, p, g0);
    if (e != cudaSuccess) return e;
    return cudaPeekAtLastError();
}

}  // namespace fp8bs
