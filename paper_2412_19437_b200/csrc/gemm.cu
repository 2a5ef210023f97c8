// gemm.cu — block-scaled FP8 GEMM with FP32 promotion for B200 (sm_100a).
//
// What it computes (§3.3.2; include/fp8bs.h):
//   D[i,j] (+)= sum_kb  sA(kb,i) * sB(kb,j) * P_kb[i,j],   P_kb = sum_{c in kb} dec(A[i,c]) dec(B[j,c])
// with one scale per N_C = 128 contraction elements.  The paper (H800) promotes WGMMA partials
// to CUDA-core registers every 128 elements; here the promotion interval is the same (forced by
// the per-128 scales) but the machinery is Blackwell's:
//   * TMA (SWIZZLE_128B) stages A and B K-blocks (128 wide) into a shared-memory ring;
//   * a 256-column tile is computed as two N = 128 halves, each with its own MMA-issuing warp
//     (one thread issues a tcgen05.mma only every ~70 cycles) and its own two TMEM slots: per
//     K-block each issuer runs 4x tcgen05.mma.kind::f8f6f4 (K = 32) into a fresh FP32 slot P;
//   * 8 promotion warps (FP8BS_NPW) read each P with four tcgen05.ld.32x32b.x32 (a warp owns one
//     TMEM lane quadrant = 32 rows x 128 columns of a half), release the slot, and accumulate
//     P * sA(kb,i) * sB(kb,j) in 128 registers with packed FFMA2 (Wgrad: FMUL2 + FFMA2), finally
//     writing BF16 (RNE) or FP32 (+= for Wgrad) through TMA stores.  A slot is reused two K-blocks
//     later, so its release has three other N = 128 MMA groups (768 cycles at peak) to land;
//   * a scale warp streams sA (and Wgrad's per-column sB) with TMA into its own 8-stage ring; every
//     release of a TMA-filled stage read with ld.shared is preceded by a proxy fence (release_scales).
// kPair = true: a cluster of 2 CTAs on a TPC runs tcgen05.mma.cta_group::2 with M = 256 (128 rows
// per CTA): each CTA stages its own 128 rows of A and 64 rows of each B half, so per-SM L2->SMEM
// traffic per MAC is that of a 256 x 256 tile.  The leader CTA issues the MMAs; both CTAs' TMA loads
// complete on the leader's barrier; commits multicast to both CTAs; promotion warps release a TMEM
// slot by arriving on the leader's barrier.
// Warp roles (384 threads): w0 TMA A/B producer, w1/w2 MMA issuers (half 0/1; w2 also allocates
// TMEM), w3 scale producer, w4..w11 promotion + epilogue (w4..w7 half 0, w8..w11 half 1; lane
// quadrant = warp % 4).  Persistent clusters walk a static tile schedule; the grouped (MoE) variant
// maps tiles to (expert, m-tile, n-tile) from device-side offsets with no host synchronisation.
// DESIGN.md §5 has the measurements behind these choices.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstddef>
#include <type_traits>
#include <cstdlib>

#include "sm100.cuh"
#include "internal.h"

#ifndef FP8BS_BAND_MB
#define FP8BS_BAND_MB 48   // L2 budget of the resident operand's band (raster)
#endif

namespace fp8bs {

constexpr int BM = 128, BK = 128;     // rows per CTA, K-block (= N_C)
constexpr int BN = 256;               // tile columns, issued as two N = 128 MMA halves
constexpr int HN = 128;               // columns per half (= one TMEM slot, = one weight block)
constexpr int kMaxGroups = 1024;   // experts per grouped launch (one scheduler thread each)

#ifndef FP8BS_NPW
#define FP8BS_NPW 8
#endif
#ifndef FP8BS_EPI_BUFS
#define FP8BS_EPI_BUFS 1   // 2 measured no faster (one fewer operand stage; Wgrad -2%)
#endif

template <bool kPair, bool kWgrad>
struct Cfg {
    static constexpr int CS = kPair ? 2 : 1;                // CTAs per cluster
    static constexpr int ROWS = BM * CS;                    // rows per cluster tile
    // B rows staged per CTA per half: a CTA pair splits each N = 128 half into 2 x 64 rows
    static constexpr int BH_ROWS = kPair ? HN / 2 : HN;
    static constexpr int BH_BYTES = BH_ROWS * BK;
    static constexpr int A_BYTES = BM * BK;
    static constexpr int STAGE = A_BYTES + 2 * BH_BYTES;
    static constexpr int kSStages = 8;                     // power of two (promotion indexes with a mask)
    // TMEM: 4 slots of 128 FP32 columns; half h of a K-block alternates between slots 2h and 2h + 1,
    // so a slot's promotion overlaps three other N = 128 MMA groups (768 cycles at peak) before the
    // MMA that reuses it (a 2 x 256-column double buffer gave 512).
    static constexpr int NSLOT = 4;
    static constexpr int TMEM_COLS = 512;
    // sA box: BM + 4 floats starting at the 4-aligned row at or below the CTA's first row (a TMA
    // box must start 16-byte aligned in its inner dimension; grouped tiles start at any row).
    static constexpr int SA_BOX = BM + 4;
    static constexpr int SA_BYTES = 640;                    // >= SA_BOX * 4, multiple of 128
    // Wgrad: per-column sB of the tile for this K-block (TMA); Fprop/Dgrad: the two 128-column
    // weight-block scalars of the tile.  TMA destinations must be 128-byte aligned.
    static constexpr int SB_BYTES = kWgrad ? BN * 4 : 128;
    static constexpr int SSTAGE = SA_BYTES + SB_BYTES;
    static_assert(SSTAGE % 128 == 0 && STAGE % 1024 == 0, "TMA smem destinations need 128 B (1024 B swizzled) alignment");
    // Epilogue: each promotion warp stages 32 rows x 128 bytes (SWIZZLE_128B) for a TMA store.
    static constexpr int EPI_BUFS = FP8BS_EPI_BUFS;          // staging buffers per warp (2: chunk c+1 is staged while chunk c's TMA store reads)
    static constexpr int EPI_WARP_BYTES = 32 * 128 * EPI_BUFS;
    // Operand stages fill the dynamic shared memory left after the static scale ring, the epilogue
    // buffers and the barriers (227 KB per CTA, 1 KB of alignment slack).
    static constexpr int SCAT_BYTES = 32 * 8;               // scatter epilogue: a warp's 32 row destinations
    static constexpr int SMEM_FREE = 227 * 1024 - 2048 - kSStages * SSTAGE - FP8BS_NPW * (EPI_WARP_BYTES + SCAT_BYTES);
    static constexpr int kStages = SMEM_FREE / STAGE > 8 ? 8 : SMEM_FREE / STAGE;
    // Promotion warps (FP8BS_NPW, 8 or 16): warp (h, gg, quad) owns rows [32 quad, 32 quad + 32) x
    // NC = 128 * 8 / NPW columns (group gg) of half h.  8 wide warps pay the per-K-block barrier and
    // scale overhead once per 128 columns; 16 narrower warps halve each warp's FFMA2 chain.
    static constexpr int NPW = FP8BS_NPW;
    static_assert(NPW == 8 || NPW == 16, "8 or 16 promotion warps");
    static constexpr int THREADS = 128 + 32 * NPW;          // 384 / 640
    static constexpr int NC = HN * 8 / NPW;                 // columns per promotion thread (128 / 64)
    static constexpr int REG_LAUNCH = NPW == 8 ? 168 : 96;  // 65536 / THREADS rounded down to 8
    static constexpr int REG_OTHER = 24, REG_PROMO = NPW == 8 ? 240 : 112;   // setmaxnreg split of the launch pool
    static_assert((REG_LAUNCH - REG_OTHER) * 128 >= (REG_PROMO - REG_LAUNCH) * 32 * NPW, "setmaxnreg.inc would wait forever: the CTA's pool is fixed at launch");
    // grouped: a 4-entry ring of dynamically claimed tile indices (full / empty barrier per entry)
    static constexpr int kTQ = 4;
    // warps that take each claimed tile from the ring: leader CTA w1, w2 (issuers), w3, the NPW
    // promotion warps; the peer CTA w0 (its A/B producer), w3, the promotion warps
    static constexpr int TQ_CONSUMERS = kPair ? (3 + NPW) + (2 + NPW) : 3 + NPW;
    static constexpr int NBAR = 2 * kStages + 2 * kSStages + 2 * NSLOT + 2 * kTQ;
    static constexpr int OFF_EPI = kStages * STAGE;
    static constexpr int OFF_SCAT = OFF_EPI + NPW * EPI_WARP_BYTES;
    static constexpr int SMEM_DENSE = 1024 + OFF_SCAT + NPW * SCAT_BYTES;
};

struct KParams {
    int M, N, K, KB;
    int num_m, num_n;
    const float* sB;              // FPROP/DGRAD/grouped block scalars
    int64_t sb_nb_stride, sb_kb_stride, sb_expert_stride;
    int NB;                       // ceil(N/128)
    void* D; int64_t ldd; int accumulate;
    // SwiGLU epilogue (kOutSwiglu): D = qy codes [M, N/2] (ldd), sy [N/256][ldsy]; qh codes [M, N]
    // (ldqh) and sh [N/128][ldsh] — the FP8 cache of H — when qh != nullptr
    float* sy; int64_t ldsy; uint8_t* qh; int64_t ldqh; float* sh; int64_t ldsh;
    int G; const int64_t* offsets;
    void* tiles;                  // grouped: TileTable in the caller's workspace
    int gm;                       // raster band width (dense): tiles of the resident operand per band
    int rast_n;                   // 1: n-fastest (B resident, A streamed), 0: m-fastest
    int tile_end;                 // dense: tiles [0, tile_end) of the raster belong to this launch
    // kOutScatter: row r of the output goes to sc_base[sc_rank[r]] + sc_row[r] * ldd (BF16 elements)
    void* const* sc_base; const int32_t* sc_rank; const int64_t* sc_row;
    // grouped, streamed operands (a dispatch still writing A / sA): the rows of local group e may be
    // read once ready[e * ready_chunks / G] >= ready_target (wrap-safe); ready == nullptr: no waits
    const uint32_t* ready; uint32_t ready_target; int ready_chunks;
    // grouped: expert weights [G][N][K] (the claimer prefetches the next expert's into L2)
    const uint8_t* Bp; int64_t b_expert_bytes; int b_pf_chunk; int b_pf_last_or_chunk[2];
    // split-K tail (kOutSplit): units u < split_units are (tile split_t0 + u / split_s, K-chunk u % split_s);
    // unit u writes its FP32 partial tile to rows [u * ROWS, (u + 1) * ROWS) of the workspace (BN columns)
    int split_t0, split_s, split_units;
    int debug;                    // unused (debug bits are compile-time: FP8BS_GEMM_DEBUG_BITS): 1 skip promotion math,
                                  // 2 skip MMAs, 4 TMA always re-reads K-block 0 (L2-resident),
                                  // 16 record clock64 timestamps of CTA 0, 64 MMA ignores slot release,
                                  // 128 promotion ignores slot completion (with 64: free-running
                                  // TMA + MMA pipeline), 256 issuers pace on their own commits (with 128: MMA + TMA only),
                                  // 1024 no epilogue stores,
                                  // 512 no scale ring
    unsigned long long* ts;       // [kTsSlots][kTsN] timestamps (debug & 16)
};
constexpr int kTsN = 512;
constexpr int kTsSlots = 12;
#ifndef FP8BS_PROMO_POLL
// promotion warps busy-poll (test_wait) the TMEM slot's full barrier instead of try_wait: 0 never, 1 always,
// 2 grouped CTA-pair kernels only (in the one-CTA grouped kernels it made ptxas spill ~330 bytes).  Same-box A/B (r02): C4 grouped +1% with idle gaps (2315 -> 2338 TFLOP/s) and
// +0.4-2% in 40 power-capped bench steps; the dense C1 GEMMs within noise.
#define FP8BS_PROMO_POLL 2
#endif
#ifndef FP8BS_ISSUER_POLL
#define FP8BS_ISSUER_POLL 0
#endif
#ifndef FP8BS_WG_NOSB
#define FP8BS_WG_NOSB 0
#endif
#ifndef FP8BS_B_PREFETCH
#define FP8BS_B_PREFETCH 0   // experiment: prefetch the next expert's weights into L2 at an expert's first tile (C4: -0.5%)
#endif
#ifndef FP8BS_FOLD
#define FP8BS_FOLD 1           // grouped pair tiles whose expert ends in the first 128 rows run folded (M = 128)
#endif
#ifndef FP8BS_STATIC_SCHED
#define FP8BS_STATIC_SCHED 0   // experiments: 1 = grouped tiles on the static schedule too (A/B builds)
#endif
#ifndef FP8BS_GEMM_DEBUG_BITS
#define FP8BS_GEMM_DEBUG_BITS 0
#endif
// Experiments (tools/build_rev.sh WORKTREE <name> -DFP8BS_GEMM_DEBUG_BITS=<bits>): the debug bits are
// compile-time, so the product kernel (bits 0) carries none of their instructions.
constexpr int kDbg = FP8BS_GEMM_DEBUG_BITS;
constexpr bool kTrace = kDbg != 0;
#define FP8BS_TS(slot, kb) do { if ((kDbg & 16) && blockIdx.x == 0 && (kb) < kTsN) p.ts[(slot) * kTsN + (kb)] = clock64(); } while (0)

// row0: first row of A of the CLUSTER tile; nh: halves in range.  Grouped Wgrad only: orow0 / row_end
// are rows of the stacked [G x M, N] output, kb0 / kbn the tile's contraction blocks (its expert's).
struct Tile { int row0, row_end, n0, e, nh; int orow0, kb0, kbn; };

// Grouped Wgrad (one launch over all experts): expert e's token blocks in the padded layout —
// .x = first 128-token block, .y = number of blocks (0 for an expert without tokens).  Passed by value
// (kernel parameter space, 8 KB at 1024 experts).
template <int kG>
struct GWSched { int2 e[kG]; };
constexpr int kGWMax = 1024;

template <int ROWS>
__host__ __device__ __forceinline__ void decode_dense(const KParams& p, int t, Tile& tl) {
    // Banded raster.  The operand with fewer bytes stays L2-resident and the other streams from
    // DRAM once: inside a band of gm tiles of the resident operand, consecutive tiles walk the
    // resident operand fastest, so the concurrent clusters share each streamed tile through L2.
    // (ncu, m-fastest only: Wgrad C1 read 1.05 GB of DRAM for 104 MB of operands.)
    const int nres = p.rast_n ? p.num_n : p.num_m, nstr = p.rast_n ? p.num_m : p.num_n;
    const int band = t / (p.gm * nstr);
    const int gb = min(p.gm, nres - band * p.gm);
    const int local = t - band * p.gm * nstr;
    const int ires = band * p.gm + local % gb, istr = local / gb;
    const int m = p.rast_n ? istr : ires, n = p.rast_n ? ires : istr;
    tl.row0 = m * ROWS; tl.row_end = p.M; tl.n0 = n * BN; tl.e = 0;
    tl.nh = (p.N - tl.n0 > HN) ? 2 : 1;
}

template <int ROWS>
__device__ __forceinline__ bool get_tile_dense(const KParams& p, int t, Tile& tl) {
    if (t >= p.tile_end) return false;
    decode_dense<ROWS>(p, t, tl);
    return true;
}

// Split-K tail (reading R30): when the last wave of a dense GEMM would leave most
// clusters idle, its tiles are cut along K into split_s chunks of consecutive K-blocks; unit u is
// chunk u % split_s of tail tile u / split_s and writes its FP32 partial (promoted exactly as a whole
// tile would be, over its own K-blocks) into its own workspace slab; k_splitk_reduce sums the chunks
// in chunk order and writes D.
template <int ROWS>
__device__ __forceinline__ bool get_tile_split(const KParams& p, int u, Tile& tl) {
    if (u >= p.split_units) return false;
    const int i = u / p.split_s, c = u - i * p.split_s;
    decode_dense<ROWS>(p, p.split_t0 + i, tl);
    tl.kb0 = c * p.KB / p.split_s;
    tl.kbn = (c + 1) * p.KB / p.split_s - tl.kb0;
    tl.orow0 = u * ROWS; tl.row_end = tl.orow0 + ROWS;
    return true;
}

// Streamed operands: spin (acquire, system scope: the writers are other GPUs' dispatch kernels) until the
// tile's chunk is published, then order those generic-proxy writes before this thread's TMA reads.
__device__ __forceinline__ void wait_chunk_ready(const KParams& p, int e) {
    const uint32_t* f = p.ready + (e * p.ready_chunks) / p.G;
    uint32_t v;
    for (;;) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if ((int32_t)(v - p.ready_target) >= 0) break;
        __nanosleep(256);
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Grouped Wgrad tiles: expert-major, m fastest inside an expert (the smaller operand dYqT_e stays in
// L2 while the n-tiles of XqT_e stream past it); every expert has num_m x num_n tiles, an expert without
// tokens included (its tiles write zeros, or add nothing when accumulating).
template <int ROWS, int kG>
__device__ __forceinline__ bool get_tile_gw(const KParams& p, const GWSched<kG>& gw, int t, Tile& tl) {
    const int per = p.num_m * p.num_n;
    if (t >= p.G * per) return false;
    const int e = t / per, l = t - e * per;
    const int m = l % p.num_m, n = l / p.num_m;
    tl.row0 = m * ROWS; tl.n0 = n * BN; tl.e = e;
    tl.orow0 = e * p.M + tl.row0; tl.row_end = e * p.M + p.M;
    tl.nh = (p.N - tl.n0 > HN) ? 2 : 1;
    const int2 k = gw.e[e];
    tl.kb0 = k.x; tl.kbn = k.y;
    return true;
}

// Grouped (MoE) tile table, written by k_grouped_schedule into the caller's workspace before the GEMM
// runs (same stream, PDL): tiles[t] = {first row of the cluster tile, (rows of its expert left in the
// tile, capped at 2 x rows) << 22 | (expert & 63) << 16 | n-tile, expert >> 6, 0}; ntiles = number of
// entries (n-tiles < 65536, experts <= 1024).  Every role decodes tile t with one 16-byte L2 load, so the
// GEMM kernel itself holds no per-expert state: the in-kernel prefix scan it replaced made ptxas
// spill promotion accumulators.
struct TileTable { int ntiles; int next; int pad[2]; int4 t[1]; };   // next: the dynamic claim counter

__device__ __forceinline__ void decode_table_entry(const int4 v, int N, Tile& tl) {
    tl.row0 = v.x;
    tl.row_end = v.x + (int)((uint32_t)v.y >> 22);     // rows of the expert left in the tile (<= 512)
    tl.n0 = (v.y & 0xFFFF) * BN;
    tl.e = ((v.y >> 16) & 0x3F) | (v.z << 6);          // low 6 bits of the expert; the rest in .z
    tl.nh = (N - tl.n0 > HN) ? 2 : 1;
}

__device__ __forceinline__ bool get_tile_table(const TileTable* tt, int N, int t, Tile& tl) {
    // static-schedule experiments (FP8BS_STATIC_SCHED): the count and the entry re-read per tile (L2)
    if (t >= __ldcg(&tt->ntiles)) return false;
    decode_table_entry(__ldcg(&tt->t[t]), N, tl);      // L2 only: written by the previous grid
    return true;
}

// CTAs of 1024 threads (G <= 1024): in each, thread e counts expert e's tiles, ceil(M_e/rows) x num_n,
// a block scan places them expert by expert, then the threads write the CTA's share of the entries
// (tile t's expert by binary search over the scanned starts).  Inside an expert the smaller operand stays L2-resident:
// more rows than N walks the n-tiles fastest (A rows read once, B_e resident), fewer walks m fastest.
#ifndef FP8BS_GROUPED_ORDER
#define FP8BS_GROUPED_ORDER 0   // experiments: 1 always m-fastest, 2 always n-fastest
#endif
__global__ void __launch_bounds__(1024) k_grouped_schedule(const int64_t* __restrict__ offsets, int G, int rows,
                                                           int num_n, int N, TileTable* tt) {
    griddep_wait();
    griddep_launch_dependents();
    __shared__ int warp_sum[32];
    __shared__ int start[kMaxGroups + 1];      // first tile of expert e; start[G] = total
    __shared__ int row0[kMaxGroups + 1];
    const int e = threadIdx.x, lane = e & 31, w = e >> 5;
    int64_t a = 0, b = 0;
    if (e < G) { a = offsets[e]; b = offsets[e + 1]; }
    const int seg = b > a ? (int)(b - a) : 0;
    const int cnt = ((seg + rows - 1) / rows) * num_n;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_sum[w] = incl;
    __syncthreads();
    if (w == 0) {
        int v = warp_sum[lane], x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += u;
        }
        warp_sum[lane] = x - v;                            // exclusive prefix of the warp sums
    }
    __syncthreads();
    if (e < G) { start[e] = warp_sum[w] + incl - cnt; row0[e] = (int)a; }
    if (e == G - 1) {
        start[G] = warp_sum[w] + incl; row0[G] = (int)b;
        if (blockIdx.x == 0) { tt->ntiles = start[G]; tt->next = 0; }
    }
    __syncthreads();
    const int total = start[G];
    // every CTA redoes the (cheap) scan and fills its share of the entries: one CTA took ~18 us at C4
    for (int t = blockIdx.x * blockDim.x + e; t < total; t += gridDim.x * blockDim.x) {
        int lo = 0, hi = G;                                // expert x: start[x] <= t < start[x + 1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (start[mid] <= t) lo = mid; else hi = mid;
        }
        const int x = lo, l = t - start[x];
        const int sg = row0[x + 1] - row0[x], mt = (sg + rows - 1) / rows;
        const bool nfast = FP8BS_GROUPED_ORDER == 1 ? false : FP8BS_GROUPED_ORDER == 2 ? true : sg > N;
        const int m = nfast ? l / num_n : l % mt, n = nfast ? l % num_n : l / mt;
        const int r0 = row0[x] + m * rows;
        const int left = min(row0[x + 1] - r0, 2 * rows);  // only < rows (a crossing tile) matters
        tt->t[t] = make_int4(r0, (left << 22) | ((x & 0x3F) << 16) | n, x >> 6, l == 0 ? 1 : 0);   // .w: expert's first tile
    }
}

// ------------------------------------------------------------------------------------------
// SwiGLU FP8 epilogue (NEXT-2; reading R27).  The up-projection's columns come in
// (gate, up) pairs of 128: a 256-column tile is exactly gate block j (half 0) and up block j (half
// 1), so the promotion warps of a (gate, up) pair — same TMEM lane quadrant, hence the same 32 rows —
// hold matching values, and one thread holds one row of a 1x128 group in its 128 accumulators.
// ------------------------------------------------------------------------------------------
// exp, 1/d and SwiGLU in binary32 by the fixed, branch-free sequences of reading R27 — operation
// for operation oracle_exp32 / oracle_rcp32 / oracle_swiglu32 (fused multiply-adds are correctly
// rounded on both sides), evaluated two elements at a time with the packed FP32 instructions, so the
// epilogue is bit-reproducible against the oracle:
//   x = clamp(-g, -86, 86); th = RN(x L2E), tl = fma(x, L2E_LO, fma(x, L2E, -th)); k = RNE(th);
//   f = RN(RN(th - k) + tl); 2^f by a degree-7 Taylor polynomial (Horner, FMA); e = 2^f * 2^k via the
//   exponent field; d = RN(1 + e); r = 0x7EF311C3 - bits(d), then three r = fma(r, fma(-d, r, 1), r);
//   y = RN(RN(g r) u).
__device__ __forceinline__ float2 swiglu32x2(const float2 g, const float2 u) {
    const float2 x = make_float2(fminf(fmaxf(-g.x, -86.0f), 86.0f), fminf(fmaxf(-g.y, -86.0f), 86.0f));
    const float2 L2E = make_float2(1.44269502162933349609375f, 1.44269502162933349609375f);
    const float2 L2E_LO = make_float2(1.925963033500011079013347625732421875e-08f, 1.925963033500011079013347625732421875e-08f);
    const float2 th = __fmul2_rn(x, L2E);
    const float2 tl = __ffma2_rn(x, L2E_LO, __ffma2_rn(x, L2E, make_float2(-th.x, -th.y)));
    const float2 k = make_float2(rintf(th.x), rintf(th.y));
    const float2 f = __fadd2_rn(__fadd2_rn(th, make_float2(-k.x, -k.y)), tl);
    float2 q = make_float2(1.5252733804059840e-5f, 1.5252733804059840e-5f);
    q = __ffma2_rn(q, f, make_float2(1.5403530393381608e-4f, 1.5403530393381608e-4f));
    q = __ffma2_rn(q, f, make_float2(1.3333558146428443e-3f, 1.3333558146428443e-3f));
    q = __ffma2_rn(q, f, make_float2(9.6181291076284772e-3f, 9.6181291076284772e-3f));
    q = __ffma2_rn(q, f, make_float2(5.5504108664821580e-2f, 5.5504108664821580e-2f));
    q = __ffma2_rn(q, f, make_float2(2.4022650695910071e-1f, 2.4022650695910071e-1f));
    q = __ffma2_rn(q, f, make_float2(6.9314718055994531e-1f, 6.9314718055994531e-1f));
    q = __ffma2_rn(q, f, make_float2(1.0f, 1.0f));
    const float2 e = make_float2(__uint_as_float(__float_as_uint(q.x) + ((uint32_t)(int32_t)k.x << 23)),
                                 __uint_as_float(__float_as_uint(q.y) + ((uint32_t)(int32_t)k.y << 23)));
    const float2 d = __fadd2_rn(make_float2(1.0f, 1.0f), e);
    float2 r = make_float2(__uint_as_float(0x7EF311C3u - __float_as_uint(d.x)), __uint_as_float(0x7EF311C3u - __float_as_uint(d.y)));
    const float2 nd = make_float2(-d.x, -d.y), one = make_float2(1.0f, 1.0f);
#pragma unroll
    for (int i = 0; i < 3; ++i) r = __ffma2_rn(r, __ffma2_rn(nd, r, one), r);
    return __fmul2_rn(__fmul2_rn(g, r), u);
}

// One thread's row of a 1x128 group in registers: v[0 .. 16 U) quantized with scale sc (RN32 of the
// quotient, then RNE to E4M3 saturating: the quantizers' exact contract) and written as U 16-byte
// stores to dst (the row's codes; rows are the lanes, so a warp's store touches 32 rows: the code rows
// are short — 64 or 128 bytes — and staging them through shared memory for a TMA store cost a wait
// on the TMA engine, which the producer's loads keep busy, on every tile).
template <int U>
__device__ __forceinline__ void encode_row_store(const float* v, float sc, uint8_t* dst, bool store) {
    const float r = __frcp_rn(sc);
    // warp-uniform choice (as the quantizer kernels): a per-lane branch around the IEEE-division
    // slow path cost the epilogue ~40% of the GEMM's time
    if (__all_sync(0xffffffffu, fast_div_ok(sc))) {
        const float2 r2 = make_float2(r, r), ns2 = make_float2(-sc, -sc);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float* f = v + 16 * u + 4 * i;
                const float2 a = div_scale2_fast(make_float2(f[0], f[1]), r2, ns2);
                const float2 b = div_scale2_fast(make_float2(f[2], f[3]), r2, ns2);
                w[i] = cvt_e4m3x2(a.x, a.y) | (cvt_e4m3x2(b.x, b.y) << 16);
            }
            if (store) *reinterpret_cast<uint4*>(dst + 16 * u) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        return;
    }
    const bool fast = false;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float* f = v + 16 * u + 4 * i;
            if (fast) {
                const float2 r2 = make_float2(r, r), ns2 = make_float2(-sc, -sc);
                const float2 a = div_scale2_fast(make_float2(f[0], f[1]), r2, ns2);
                const float2 b = div_scale2_fast(make_float2(f[2], f[3]), r2, ns2);
                w[i] = cvt_e4m3x2(a.x, a.y) | (cvt_e4m3x2(b.x, b.y) << 16);
            } else {
                w[i] = cvt_e4m3x2(__fdiv_rn(f[0], sc), __fdiv_rn(f[1], sc)) |
                       (cvt_e4m3x2(__fdiv_rn(f[2], sc), __fdiv_rn(f[3], sc)) << 16);
            }
        }
        if (store) *reinterpret_cast<uint4*>(dst + 16 * u) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}
// maxNum of |v[0 .. n)| (the quantizers' amax)
template <int N>
__device__ __forceinline__ float row_amax(const float* v) {
    float a = 0.0f;
#pragma unroll
    for (int j = 0; j < N; ++j) a = fmaxf(a, fabsf(v[j]));
    return a;
}

template <int kH>
__device__ __forceinline__ void swiglu_exchange(float (&acc)[128], int lane, uint32_t ebuf, uint32_t pbuf,
                                                uint32_t pair_bar) {
    constexpr int mine = kH == 0 ? 0 : 64, theirs = 64 - mine;
#pragma unroll
    for (int rd = 0; rd < 2; ++rd) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float* v = acc + theirs + 32 * rd + 4 * u;
            sts_u32x4(ebuf + lane * 128 + ((u ^ (lane & 7)) << 4), __float_as_uint(v[0]), __float_as_uint(v[1]),
                      __float_as_uint(v[2]), __float_as_uint(v[3]));
        }
        named_bar_sync(pair_bar, 64);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint4 w = lds_u32x4(pbuf + lane * 128 + ((u ^ (lane & 7)) << 4));
            float* a = acc + mine + 32 * rd + 4 * u;
            const float2 o0 = make_float2(__uint_as_float(w.x), __uint_as_float(w.y));
            const float2 o1 = make_float2(__uint_as_float(w.z), __uint_as_float(w.w));
            const float2 m0 = make_float2(a[0], a[1]), m1 = make_float2(a[2], a[3]);
            const float2 y0 = kH == 0 ? swiglu32x2(m0, o0) : swiglu32x2(o0, m0);
            const float2 y1 = kH == 0 ? swiglu32x2(m1, o1) : swiglu32x2(o1, m1);
            a[0] = y0.x; a[1] = y0.y; a[2] = y1.x; a[3] = y1.y;
        }
        named_bar_sync(pair_bar, 64);
    }
}

// The epilogue of one (gate, up) warp pair (h = 0 gate, 1 up; ebuf = this warp's 4 KB staging buffer,
// pbuf = the partner's); lane = one row (row < rows_here of the tile's expert: the rest belong to
// the next expert and are not written):
//   1. (p.qh) each warp quantizes its own 128 columns 1x128 — the FP8 cache of the SwiGLU inputs;
//   2. the warps split the SwiGLU: the gate warp forms output columns [0, 64), the up warp [64, 128),
//      each receiving the partner's operand through the partner's staging buffer (32 columns per
//      round, two rounds, between pair barriers);
//   3. the row amax of y meets through the up warp's buffer; each warp writes its 64 codes, the gate
//      warp the row's scale.
__device__ __forceinline__ void swiglu_epilogue(float (&acc)[128], int h, int quad, int lane, const Tile& tl,
                                                int grow0, int rows_here, const KParams& p, uint32_t ebuf,
                                                uint32_t pbuf) {
    const uint32_t pair_bar = 1 + quad;   // named barrier of the (gate, up) pair: 64 threads
    const bool row_ok = lane < rows_here;
    const int64_t grow = grow0 + lane;
    if (p.qh) {
        const float sc = group_scale(row_amax<128>(acc));
        const int col = tl.n0 + h * HN;
        encode_row_store<8>(acc, sc, p.qh + grow * p.ldqh + col, row_ok);   // (whole warp: warp-uniform branch inside)
        if (row_ok) p.sh[(int64_t)(col / 128) * p.ldsh + grow] = sc;
    }
    // 2. (h is a template argument: a runtime offset into acc would move it to local memory)
    if (h == 0) swiglu_exchange<0>(acc, lane, ebuf, pbuf, pair_bar);
    else swiglu_exchange<1>(acc, lane, ebuf, pbuf, pair_bar);
    // 3. row amax over both halves (slots in the up warp's buffer, free after the exchange's last barrier)
    const uint32_t up_buf = h == 0 ? pbuf : ebuf;
    const float am = h == 0 ? row_amax<64>(acc) : row_amax<64>(acc + 64);
    asm volatile("st.shared.f32 [%0], %1;" :: "r"(up_buf + 128u * h + 4u * lane), "f"(am) : "memory");
    named_bar_sync(pair_bar, 64);
    const float sc = group_scale(fmaxf(am, lds_f32(up_buf + 128u * (h ^ 1) + 4u * lane)));
    named_bar_sync(pair_bar, 64);                // the slots are read before the next tile's exchange
    const int col = tl.n0 / 2;                   // output channels of this tile: [n0 / 2, n0 / 2 + 128)
    uint8_t* dst = reinterpret_cast<uint8_t*>(p.D) + grow * p.ldd + col;
    if (h == 0) {
        encode_row_store<4>(acc, sc, dst, row_ok);
        if (row_ok) p.sy[(int64_t)(col / 128) * p.ldsy + grow] = sc;
    } else {
        encode_row_store<4>(acc + 64, sc, dst + 64, row_ok);
    }
}

// kOut: 0 BF16 output, 1 FP32 output, 2 the SwiGLU FP8 epilogue (kOutSwiglu).
// kOutSplit: FP32 partials of the split-K tail; kOutScatter: BF16 rows scattered to (rank, row) destinations
// through a pointer table (the MoE combine's send fused into the grouped epilogue, NVLink peer stores)
constexpr int kOutBF16 = 0, kOutFP32 = 1, kOutSwiglu = 2, kOutSplit = 3, kOutScatter = 4;
template <bool kWgrad, int kOut, bool kGrouped, bool kPair>
__global__ void __launch_bounds__(Cfg<kPair, kWgrad>::THREADS, 1)
k_gemm_bs(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
          const __grid_constant__ CUtensorMap tmSA, const __grid_constant__ CUtensorMap tmSB,
          const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmD2, const KParams p,
          const __grid_constant__ GWSched<(kWgrad && kGrouped) ? kGWMax : 1> gw) {
    using C = Cfg<kPair, kWgrad>;
    // grouped Wgrad: one launch over every expert, each tile with its expert's contraction blocks
    constexpr bool kGW = kWgrad && kGrouped;
    constexpr bool kSplit = kOut == kOutSplit;
    static_assert(!(kSplit && kGrouped), "the split-K tail is for dense launches");
    constexpr bool kOutF32 = kOut == kOutFP32 || kSplit;
    constexpr bool kSwiglu = kOut == kOutSwiglu;
    constexpr bool kScatter = kOut == kOutScatter;
    static_assert(!kScatter || (kGrouped && !kWgrad), "the scatter epilogue is the grouped Fprop's");
    constexpr bool kKR = kGW || kSplit;   // tiles carry their own contraction-block range
    extern __shared__ uint8_t smem_raw[];
    griddep_wait();                 // PDL: previous grid complete, its writes visible
    griddep_launch_dependents();
    // barriers and the scale ring live in static shared memory: their addresses are constants, so
    // the promotion loop does not re-derive the aligned dynamic base every K-block
    // one static block (scale ring, barriers, TMEM address): every static shared address is a
    // constant offset from one pinned base register
    struct __align__(1024) StaticSmem {
        uint8_t scale[C::kSStages * C::SSTAGE];
        uint64_t bar[C::NBAR];
        uint32_t tmem;
        int4 tq[C::kTQ];           // grouped: claimed tiles' table entries (.w = tile index, -1: none left)
    };
    __shared__ StaticSmem s_static;
    uint8_t* s_scale = s_static.scale;
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    // Wgrad: pinned (ptxas otherwise re-derives the base with S2UR SR_CgaCtaId at every use in the
    // promotion loop: 292 -> 259 instructions per K-block).  Fprop/Dgrad: the pinned base costs the
    // register that makes ptxas spill accumulators, so the base stays rematerializable there.
    const uint32_t sring = kWgrad ? smem_u32_pinned(&s_static) : smem_u32(&s_static);
    const uint32_t bar0 = sring + (uint32_t)offsetof(StaticSmem, bar);
    auto full_bar   = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar  = [&](int s) { return bar0 + 8u * (C::kStages + s); };
    auto sfull_bar  = [&](int s) { return bar0 + 8u * (2 * C::kStages + s); };
    auto sempty_bar = [&](int s) { return bar0 + 8u * (2 * C::kStages + C::kSStages + s); };
    auto pfull_bar  = [&](int b) { return bar0 + 8u * (2 * C::kStages + 2 * C::kSStages + b); };
    auto pempty_bar = [&](int b) { return bar0 + 8u * (2 * C::kStages + 2 * C::kSStages + C::NSLOT + b); };
    auto tqfull_bar  = [&](int q) { return bar0 + 8u * (2 * C::kStages + 2 * C::kSStages + 2 * C::NSLOT + q); };
    auto tqempty_bar = [&](int q) { return bar0 + 8u * (2 * C::kStages + 2 * C::kSStages + 2 * C::NSLOT + C::kTQ + q); };
    uint32_t* tmem_slot = &s_static.tmem;
    uint8_t* s_epi = smem + C::OFF_EPI;                // epilogue staging (1024-aligned, dynamic)

    // warp index broadcast from lane 0 so the compiler knows role branches are warp-uniform
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const uint32_t rank = kPair ? cluster_ctarank() : 0u;
    const int cid = blockIdx.x / C::CS, ncl = gridDim.x / C::CS;

    if (threadIdx.x == 32) {
        for (int s = 0; s < C::kStages; ++s) { mbar_init(full_bar(s), 1); mbar_init(empty_bar(s), 2); }
        for (int s = 0; s < C::kSStages; ++s) { mbar_init(sfull_bar(s), 1); mbar_init(sempty_bar(s), C::NPW); }
        for (int b = 0; b < C::NSLOT; ++b) { mbar_init(pfull_bar(b), 1); mbar_init(pempty_bar(b), (C::NPW / 2) * C::CS); }
        for (int q = 0; q < C::kTQ; ++q) { mbar_init(tqfull_bar(q), 1); mbar_init(tqempty_bar(q), C::TQ_CONSUMERS); }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); tma_prefetch_desc(&tmSA); tma_prefetch_desc(&tmD);
        if (kWgrad || (kGrouped && kPair)) tma_prefetch_desc(&tmSB);
    }
    if (warp == 2) {
        if constexpr (kPair) tmem_alloc_pair<C::TMEM_COLS>(smem_u32(tmem_slot));
        else tmem_alloc<C::TMEM_COLS>(smem_u32(tmem_slot));
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (kPair) cluster_sync();        // peer barriers initialised before any remote arrive / TMA
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // A tile reference: its index (static schedules) or, for the dynamically claimed grouped tiles, the
    // table entry the claimer shipped through the tq ring (decoded here with no memory access).
    constexpr bool kDyn = kGrouped && !kGW && !FP8BS_STATIC_SCHED;
    using TileRef = typename std::conditional<kDyn, int4, int>::type;
    auto next_tile = [&](const TileRef t, Tile& tl) -> bool {
        if constexpr (kDyn) {
            if (t.w < 0) return false;
            decode_table_entry(t, p.N, tl);
            return true;
        } else if constexpr (kGW) return get_tile_gw<C::ROWS>(p, gw, t, tl);
        else if constexpr (kSplit) return get_tile_split<C::ROWS>(p, t, tl);
        else if constexpr (kGrouped) return get_tile_table(reinterpret_cast<const TileTable*>(p.tiles), p.N, t, tl);
        else return get_tile_dense<C::ROWS>(p, t, tl);
    };
    // contraction blocks of a tile and their first block (grouped Wgrad and split-K tiles differ)
    auto nkb = [&](const Tile& tl) -> int { if constexpr (kKR) return tl.kbn; else return p.KB; };
    auto kbase = [&](const Tile& tl) -> int { if constexpr (kKR) return tl.kb0; else return 0; };
    // Folded tiles (grouped Fprop/Dgrad on CTA pairs): a tile whose expert ends within its first 128
    // rows is issued as tcgen05.mma.cta_group::2 with M = 128 (64 rows per CTA) instead of M = 256,
    // which halves its MMA work and its promotion.  Each CTA's 64 x 128 accumulator of a half then lies
    // folded over the 128 TMEM lanes in 64 columns: columns [0, 64) of the half in lanes 0..63,
    // columns [64, 128) in lanes 64..127 (CUTLASS cute/atom/mma_traits_sm100.hpp, tmem_frg, the
    // N_SM = 2, M_MMA = 64 "2x2" atom), so the warp of lane quadrant q promotes rows 32 (q & 1) + lane
    // of the CTA's 64 and columns 64 (q >> 1) + [0, 64) of the half.
    constexpr bool kFold = FP8BS_FOLD && kGrouped && kPair && !kWgrad && !kSwiglu && C::NC == 128;
    auto folded = [&](const Tile& tl) -> bool { if constexpr (kFold) return tl.row_end - tl.row0 <= BM; else return false; };
    auto cta_row0 = [&](const Tile& tl) -> int { return tl.row0 + (int)rank * (folded(tl) ? BM / 2 : BM); };

    // Tile order.  Dense: static, cluster c takes tiles c, c + ncl, ...  Grouped: dynamic — the
    // leader's producer thread claims the next tile index with an atomic on the workspace counter
    // and hands it to every role of both CTAs through the tq ring, so the tiles in flight at any time
    // are consecutive in the table (a static schedule let clusters drift apart over the ~220 tiles
    // each runs at C4 and lose the L2 sharing of A rows between the n-tiles of an m-tile: DRAM read
    // 4.5x the operands).  The claimer runs one tile ahead so the atomic's latency is off the path.
    TileTable* ttw = reinterpret_cast<TileTable*>(p.tiles);
    // The claimer ships the claimed tile's 16-byte table entry itself (it loads it off the critical path,
    // one tile ahead): the other roles decode the tile from shared memory instead of waiting on an L2
    // load at every tile boundary.
    auto tq_publish = [&](int j) -> int {            // leader w0, one lane: claim tile #j of this cluster
        const int q = j % C::kTQ;
        mbar_wait(tqempty_bar(q), ((j / C::kTQ) & 1) ^ 1);
        const int t = atomicAdd(&ttw->next, 1);
        int4 e = make_int4(0, 0, 0, -1);
        if (t < __ldcg(&ttw->ntiles)) {
            e = __ldcg(&ttw->t[t]);
#if FP8BS_B_PREFETCH
            // the first tile of expert x: start pulling expert x + 1's weights into L2, so its first
            // tiles (claimed about a wave later) do not wait on DRAM
            const int x = ((e.y >> 16) & 0x3F) | (e.z << 6);
            if (e.w && x + 1 < p.G) {
                const uint8_t* nb = p.Bp + (int64_t)(x + 1) * p.b_expert_bytes;
#pragma unroll 1
                for (int c = 0; c < 16; ++c)             // 16 bulk prefetches of b_pf_chunk bytes (the last clipped)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                                 :: "l"(nb + (int64_t)c * p.b_pf_chunk), "r"((uint32_t)p.b_pf_last_or_chunk[c == 15]) : "memory");
            }
#endif
            e.w = t;
        }
        const uint32_t a = smem_u32(&s_static.tq[q]);
        sts_u32x4(a, (uint32_t)e.x, (uint32_t)e.y, (uint32_t)e.z, (uint32_t)e.w);
        mbar_arrive(tqfull_bar(q));
        if constexpr (kPair) {
            st_shared_cluster_u32x4(mapa_shared(a, 1), (uint32_t)e.x, (uint32_t)e.y, (uint32_t)e.z, (uint32_t)e.w);
            mbar_arrive_release_cluster(mapa_shared(tqfull_bar(q), 1));
        }
        return e.w;
    };
    auto tq_entry = [&](int q) -> int4 {
        const uint4 v = lds_u32x4(opaque_u32(sring) + (uint32_t)offsetof(StaticSmem, tq) + 16u * q);
        return make_int4((int)v.x, (int)v.y, (int)v.z, (int)v.w);
    };
    auto tq_take = [&](int j) -> int4 {              // every other role, whole warp: tile #j
        // addresses rebuilt from an opaque base at each call: hoisted out of the tile loop they
        // would stay live across the K loop and push the promotion warps' accumulators into spills
        const int q = j % C::kTQ;
        const uint32_t b = opaque_u32(bar0) + 8u * (2 * C::kStages + 2 * C::kSStages + 2 * C::NSLOT + q);
        mbar_wait_acquire_cluster(b, (j / C::kTQ) & 1);
        const int4 t = tq_entry(q);
        __syncwarp();
        if (elect_one()) {
            const uint32_t e = b + 8u * C::kTQ;
            if (kPair && cluster_ctarank() != 0) {
                // The leader overwrites this slot (remotely) once every consumer has arrived, so the read
                // above must be complete before the arrive.  A release.cluster arrive costs a GPU-scope
                // MEMBAR per tile per warp (measured: C4 2157-2175 vs 2205-2211 TFLOP/s); instead the
                // arrive's address depends on the loaded value (z is always 0: row0 is never ~0u), so
                // it cannot issue before the load has returned.
                uint32_t z;
                asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, 0xFFFFFFFF;\n\tselp.u32 %0, 8, 0, p;\n\t}"
                             : "=r"(z) : "r"((uint32_t)t.x));
                mbar_arrive_cluster((e + z) & kPeerBitMask);
            } else {
                mbar_arrive(e);
            }
        }
        __syncwarp();
        return t;
    };
    int t_next = 0;                                  // claimer: tile #j+1, claimed ahead (-1: none left)
    // the leader's producer warp (lane 0 claims, the warp reads the entry back from its own ring slot:
    // the slot of tile #j is republished only at claim #j + kTQ, after this read)
    auto tile_index_claim = [&](int j) -> TileRef {
        if constexpr (!kDyn) return cid + j * ncl;
        else {
            if (lane == 0) {
                const int t = j == 0 ? tq_publish(0) : t_next;
                if (t >= 0) t_next = tq_publish(j + 1);
            }
            __syncwarp();
            return tq_entry(j % C::kTQ);
        }
    };
    // every other role
    auto tile_index = [&](int j) -> TileRef {
        if constexpr (!kDyn) return cid + j * ncl;
        else return tq_take(j);
    };

    if (warp < 4) {
        setmaxnreg_dec<C::REG_OTHER>();
        // Producer and MMA roles run on the WHOLE warp (all lanes keep identical, provably uniform
        // values) and only the issuing instructions are under elect.sync.  With the loops on lane 0
        // alone, ptxas wrapped every tcgen05.mma in an ELECT / R2UR.BROADCAST waterfall loop:
        // ~100 cycles per MMA instruction (measured with clock64; tools/mma_bench.cu).
        if (warp == 0) {
            // ---------------- TMA producer: A and the two B halves (this CTA's rows) ----------------
            int it = 0;
            Tile tl;
            auto tix = [&](int j) { return rank == 0 ? tile_index_claim(j) : tile_index(j); };
            int j = 0;
            for (TileRef t = tix(0); next_tile(t, tl); t = tix(++j)) {
                if constexpr (kGrouped && !kWgrad) { if (p.ready) wait_chunk_ready(p, tl.e); }
                const int arow = cta_row0(tl);
                const int brow = tl.n0 + (int)rank * C::BH_ROWS;
                // folded tiles load 64 rows of A per CTA, through the 64-row map the grouped launch passes
                // in tmSB's place (the grouped Fprop/Dgrad has no per-column sB map)
                const bool fold = folded(tl);
                for (int kb = 0; kb < nkb(tl); ++kb, ++it) {
                    const int s = it % C::kStages;
                    const uint32_t ph = (it / C::kStages) & 1;
                    mbar_wait(empty_bar(s), ph ^ 1);
                    const uint32_t sa = sbase + s * C::STAGE;
                    const int kc = ((kDbg & 4)) ? 0 : (kbase(tl) + kb) * BK;
                    if (elect_one()) {
                        if constexpr (kPair) {
                            if (rank == 0) mbar_arrive_expect_tx(full_bar(s), 2 * ((fold ? C::A_BYTES / 2 : C::A_BYTES) + tl.nh * C::BH_BYTES));
                            if (fold) tma_load_2d_pair(sa, &tmSB, full_bar(s), kc, arow);
                            else tma_load_2d_pair(sa, &tmA, full_bar(s), kc, arow);
                            for (int h = 0; h < tl.nh; ++h) {
                                if constexpr (kGrouped && !kWgrad) tma_load_3d_pair(sa + C::A_BYTES + h * C::BH_BYTES, &tmB, full_bar(s), kc, brow + h * HN, tl.e);
                                else tma_load_2d_pair(sa + C::A_BYTES + h * C::BH_BYTES, &tmB, full_bar(s), kc, brow + h * HN);
                            }
                        } else {
                            mbar_arrive_expect_tx(full_bar(s), C::A_BYTES + tl.nh * C::BH_BYTES);
                            tma_load_2d(sa, &tmA, full_bar(s), kc, arow);
                            for (int h = 0; h < tl.nh; ++h) {
                                if constexpr (kGrouped && !kWgrad) tma_load_3d(sa + C::A_BYTES + h * C::BH_BYTES, &tmB, full_bar(s), kc, brow + h * HN, tl.e);
                                else tma_load_2d(sa + C::A_BYTES + h * C::BH_BYTES, &tmB, full_bar(s), kc, brow + h * HN);
                            }
                        }
                    }
                    __syncwarp();
                }
            }
        } else if (warp == 1 || warp == 2) {
          if (rank == 0) {
            // ---------------- MMA issuers (leader CTA): warp 1 half 0, warp 2 half 1 ----------------
            // One thread issues a tcgen05.mma about every 70 cycles (tools/mma_bench.cu), so the 8
            // N = 128 MMAs of a K-block (512 cycles at peak) need two issuers.  Each half has its own
            // two TMEM slots (2h, 2h + 1); a stage is released by one commit per half.
            const int h = warp - 1;
            constexpr uint32_t idesc_full = idesc_e4m3_f32(C::ROWS, HN);
            int it = 0, qh = 0;
            Tile tl;
            int j = 0;
            for (TileRef t = tile_index(0); next_tile(t, tl); t = tile_index(++j)) {
                if (h >= tl.nh) {
                    // This half lies past N (last column tile): no MMAs, but the issuer still walks
                    // the ring in step and releases each stage with its own (empty) commit.  Jumping
                    // ahead by KB instead let a later parity wait on full_bar pass one or more phases
                    // early (an mbarrier parity wait only tells apart adjacent phases), so the next
                    // tile's MMAs read stages still being filled.
                    for (int kb = 0; kb < nkb(tl); ++kb, ++it) {
                        const int s = it % C::kStages;
                        mbar_wait(full_bar(s), (it / C::kStages) & 1);
                        if (elect_one()) {
                            if constexpr (kPair) mma_commit_pair(empty_bar(s), 3);
                            else mma_commit(empty_bar(s));
                        }
                        __syncwarp();
                    }
                    continue;
                }
                const uint32_t idesc = folded(tl) ? idesc_e4m3_f32(C::ROWS / 2, HN) : idesc_full;
                for (int kb = 0; kb < nkb(tl); ++kb, ++it, ++qh) {
                    const int s = it % C::kStages;
                    const uint32_t ph = (it / C::kStages) & 1;
                    const int pb = 2 * h + (qh & 1);
                    const uint32_t pph = (qh >> 1) & 1;
                    if ((kDbg & 256)) { if (qh >= 2) mbar_wait(pfull_bar(pb), pph ^ 1); }   // self-paced
                    else if (!((kDbg & 64))) {
#if FP8BS_ISSUER_POLL
                        mbar_wait_poll(pempty_bar(pb), pph ^ 1);
#else
                        mbar_wait(pempty_bar(pb), pph ^ 1);
#endif
                    }
                    if (h == 0) FP8BS_TS(0, it);
                    mbar_wait(full_bar(s), ph);
                    if (h == 0) FP8BS_TS(1, it);
                    tc_fence_after();
                    const uint32_t sa = sbase + s * C::STAGE;
                    const uint64_t ad = sdesc_k_sw128(sa);
                    const uint64_t bd = sdesc_k_sw128(sa + C::A_BYTES + h * C::BH_BYTES);
                    const uint32_t d = tmem_base + pb * HN;
                    if (elect_one()) {
                        if (!((kDbg & 2))) {
#pragma unroll
                            for (int k = 0; k < BK / 32; ++k) {
                                if constexpr (kPair) mma_f8f6f4_pair(d, ad + 2 * k, bd + 2 * k, idesc, k > 0 ? 1u : 0u);
                                else mma_f8f6f4(d, ad + 2 * k, bd + 2 * k, idesc, k > 0 ? 1u : 0u);
                            }
                        }
                        if constexpr (kPair) mma_commit_pair(pfull_bar(pb), 3);
                        else mma_commit(pfull_bar(pb));
                        // release the smem stage once this half's MMAs have read it (the barrier
                        // counts one commit per half; an inactive half commits without MMAs)
                        if constexpr (kPair) mma_commit_pair(empty_bar(s), 3);
                        else mma_commit(empty_bar(s));
                    }
                    __syncwarp();
                    if (h == 0) FP8BS_TS(2, it);
                }
            }
          }
        } else if (warp == 3) {
            // ---------------- scale producer (this CTA's rows; the tile's sB) ----------------
            int sit = 0;
            if ((kDbg & 512)) return;   // experiment: no scale ring traffic (promotion uses stale scales)
            Tile tl;
            int j = 0;
            for (TileRef t = tile_index(0); next_tile(t, tl); t = tile_index(++j)) {
                if constexpr (kGrouped && !kWgrad) { if (p.ready) wait_chunk_ready(p, tl.e); }
                const float* sbp = p.sB;
                if constexpr (kGrouped) sbp += (int64_t)tl.e * p.sb_expert_stride;
                const int arow = cta_row0(tl);
                const int nb0 = tl.n0 / 128;
                for (int kb0 = 0; kb0 < nkb(tl); kb0 += 32) {
                    // lane j holds the 2 block scalars the tile's columns need at K-block kb0 + j
                    float v0 = 0.0f, v1 = 0.0f;
                    if constexpr (!kWgrad) {
                        const int kb = kbase(tl) + kb0 + lane;
                        if (kb < kbase(tl) + nkb(tl)) {
                            v0 = __ldg(sbp + nb0 * p.sb_nb_stride + kb * p.sb_kb_stride);
                            if (nb0 + 1 < p.NB) v1 = __ldg(sbp + (nb0 + 1) * p.sb_nb_stride + kb * p.sb_kb_stride);
                        }
                    }
                    const int nk = min(32, nkb(tl) - kb0);
                    for (int j = 0; j < nk; ++j, ++sit) {
                        const int ss = sit % C::kSStages;
                        const uint32_t sph = (sit / C::kSStages) & 1;
                        mbar_wait(sempty_bar(ss), sph ^ 1);          // whole warp: shuffles stay convergent
                        const uint32_t sst = sring + ss * C::SSTAGE;
                        const float b0 = __shfl_sync(0xffffffffu, v0, j);
                        const float b1 = __shfl_sync(0xffffffffu, v1, j);
                        if (lane == 0) {
                            if constexpr (!kWgrad) {
                                float* sbs = reinterpret_cast<float*>(s_scale + ss * C::SSTAGE + C::SA_BYTES);
                                sbs[0] = b0; sbs[1] = b1;
                            }
                            mbar_arrive_expect_tx(sfull_bar(ss), C::SA_BOX * 4 + (kWgrad ? BN * 4 : 0));
                            tma_load_2d(sst, &tmSA, sfull_bar(ss), arow & ~3, kbase(tl) + kb0 + j);
                            if constexpr (kWgrad) tma_load_2d(sst + C::SA_BYTES, &tmSB, sfull_bar(ss), tl.n0, kbase(tl) + kb0 + j);
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
        // Warps 4..7 promote half 0, warps 8..11 half 1 (each SMSP runs one warp of each half).
        const int h = (warp - 4) / (C::NPW / 2);        // half
        const int gg = ((warp - 4) >> 2) % (C::NPW / 8); // column group within the half
        const int quad = warp & 3;                      // TMEM lane quadrant
        const int row = quad * 32 + lane;               // row within this CTA's 128
        constexpr int NC = C::NC;                       // 128 / 64
        float acc[NC];
        const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + gg * NC;
        const uint32_t sb_off = C::SA_BYTES + 4u * (kWgrad ? h * HN + gg * NC : h);
        int sit = 0, qh = 0;                            // K-block, slot uses of this half
        Tile tl;
        // every tile advances sit by exactly KB, so the tile's sequence number is sit / KB (one
        // register fewer than a counter: the accumulators are at the edge of the 240-register budget)
        int jt = 0;                                     // grouped Wgrad: tiles walked (KB varies per tile)
        auto next_j = [&]() -> int { if constexpr (kKR) return ++jt; else return sit / p.KB; };
        for (TileRef t = tile_index(0); next_tile(t, tl); t = tile_index(next_j())) {
            const bool fold = folded(tl);
            // this row's sA in a stage (folded: row 32 (quad & 1) + lane of the CTA's 64)
            const uint32_t sa_off = 4u * ((cta_row0(tl) & 3) + (fold ? (quad & 1) * 32 + lane : row));
            const bool active = h < tl.nh;
            if (!active) {
                // this half lies past N (last column tile): only keep the scale ring moving (the
                // issuer skips its MMAs and slot uses too)
                for (int kb = 0; kb < nkb(tl); ++kb, ++sit) {
                    if (!(kDbg & 512)) {
                        mbar_wait(sfull_bar(sit & (C::kSStages - 1)), (sit / C::kSStages) & 1);
                        if (elect_one()) mbar_arrive(sempty_bar(sit & (C::kSStages - 1)));
                    }
                }
                continue;
            }
#pragma unroll
            for (int i = 0; i < NC; ++i) acc[i] = 0.0f;
            // One K-block of promotion for this warp: wait for the scale stage and the TMEM slot, read
            // the slot, release it, accumulate.  ss/pb/pph are compile-time in the unrolled loop below.
            auto promote_kb = [&](const int ss, const uint32_t sph, const int pb, const uint32_t pph, const int sit) __attribute__((always_inline)) {
                if (!(kDbg & 512)) mbar_wait(sfull_bar(ss), sph);
                if (kTrace && lane == 0 && warp == C::THREADS / 32 - 1) FP8BS_TS(11, sit);
                const uint32_t sst = sring + ss * C::SSTAGE;
                const float sa = lds_f32(sst + sa_off);
                // Fprop/Dgrad: half h is exactly weight block n0/128 + h (n0 is a multiple of 256),
                // so one factor sA(kb,row) * sB(kb, block) per warp: one FFMA per element.
                float f = 0.0f;
                if constexpr (!kWgrad) f = __fmul_rn(sa, lds_f32(sst + sb_off));

                if (kTrace && lane == 0 && (warp == 4 || warp == 7)) FP8BS_TS(warp == 4 ? 3 : 5, sit);
                if (kTrace && lane == 0 && warp == C::THREADS / 32 - 1) FP8BS_TS(8, sit);
                if (!((kDbg & 128))) {
                    if constexpr (FP8BS_PROMO_POLL == 1 || (FP8BS_PROMO_POLL == 2 && kGrouped && kPair)) mbar_wait_poll(pfull_bar(pb), pph);
                    else mbar_wait(pfull_bar(pb), pph);
                }
                if (kTrace && lane == 0 && warp == C::THREADS / 32 - 1) FP8BS_TS(9, sit);
                if (kTrace && lane == 0 && (warp == 4 || warp == 7)) FP8BS_TS(warp == 4 ? 4 : 6, sit);
                tc_fence_after();
                // acc[c0 + j] += P[j] * sA(kb,row) * sB(kb, col): Fprop/Dgrad one FFMA2 per column
                // pair; Wgrad FMUL2 + FFMA2 (outer-product scales)
                auto fma32 = [&](const uint32_t* r, int c0) {
                    if ((kDbg & 1)) {   // experiment: loads only
                        if (r[0] == 0x7fffffffu) acc[c0] += 1.0f;
                        return;
                    }
                    if constexpr (!kWgrad) {
                        const float2 f2 = make_float2(f, f);
#pragma unroll
                        for (int j = 0; j < ((kDbg & 4096) ? 16 : 32); j += 2) {   // 4096: half the math (experiment)
                            const float2 a = __ffma2_rn(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), f2,
                                                        make_float2(acc[c0 + j], acc[c0 + j + 1]));
                            acc[c0 + j] = a.x; acc[c0 + j + 1] = a.y;
                        }
                    } else {
                        const float2 sa2 = make_float2(sa, sa);
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
#if FP8BS_WG_NOSB   // experiment: no per-column scale loads (wrong results; timing only)
                            const float4 b = make_float4(sa, sa, sa, sa);
#else
                            const float4 b = lds_f32x4(sst + sb_off + 4u * (c0 + j));
#endif
                            const float2 fa = __fmul2_rn(sa2, make_float2(b.x, b.y));
                            const float2 fb = __fmul2_rn(sa2, make_float2(b.z, b.w));
                            const float2 a0 = __ffma2_rn(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), fa,
                                                         make_float2(acc[c0 + j], acc[c0 + j + 1]));
                            const float2 a1 = __ffma2_rn(make_float2(__uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])), fb,
                                                         make_float2(acc[c0 + j + 2], acc[c0 + j + 3]));
                            acc[c0 + j] = a0.x; acc[c0 + j + 1] = a0.y; acc[c0 + j + 2] = a1.x; acc[c0 + j + 3] = a1.y;
                        }
                    }
                };
                const uint32_t ta = tbase + pb * HN;   // folded: the lane quadrant's 64 columns start here too
                if ((kDbg & 8)) {     // experiment: no TMEM reads, no math
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (kPair) mbar_arrive_cluster(pempty_bar(pb) & kPeerBitMask);
                        else mbar_arrive(pempty_bar(pb));
                    }
                    return;
                }
                uint32_t r0[32], r1[32];
                if constexpr (NC == 128) {
                    // two 64-column rounds: two tcgen05.ld in flight per wait; the slot is released as
                    // soon as the second round has landed (32 FFMA2 after the first wait).  Folded: one
                    // round, the slot released before its math.
                    FP8BS_TMEM_LD32(ta, r0);
                    FP8BS_TMEM_LD32(ta + 32, r1);
                    tmem_ld_wait();
                    if (!fold) {
                        fma32(r0, 0);
                        fma32(r1, 32);
#pragma unroll
                        for (int j = 0; j < 64; ++j) asm volatile("" : "+f"(acc[j]));
                        FP8BS_TMEM_LD32(ta + 64, r0);
                        FP8BS_TMEM_LD32(ta + 96, r1);
                        tmem_ld_wait();
                    }
                } else {
                    // 64 columns: one 32-column round, its math, then the second round
                    FP8BS_TMEM_LD32(ta, r0);
                    tmem_ld_wait();
                    fma32(r0, 0);
#pragma unroll
                    for (int j = 0; j < 32; ++j) asm volatile("" : "+f"(acc[j]));
                    FP8BS_TMEM_LD32(ta + 32, r1);
                    tmem_ld_wait();
                }
                // release the slot before the last math: the registers hold this warp's part now.
                // tcgen05.wait::ld is warp-collective, so one elected lane may arrive; ptxas schedules
                // Wgrad better with elect.sync and Fprop/Dgrad better with lane 0 after __syncwarp
                // (measured: Wgrad +8% / Fprop -13% with elect)
                tc_fence_before();
                bool rel_lane;
                if constexpr (kWgrad) {
                    rel_lane = elect_one();
                } else {
                    __syncwarp();
                    rel_lane = lane == 0;
                }
                if (rel_lane) {
                    // the leader's barrier: clear the CTA-rank bit of the shared address (a mapa'd address held
                    // across the loop made ptxas spill ~30 accumulators)
                    if constexpr (kPair) mbar_arrive_cluster(pempty_bar(pb) & kPeerBitMask);
                    else mbar_arrive(pempty_bar(pb));
                    if (kTrace && warp == C::THREADS / 32 - 1) FP8BS_TS(10, sit);
                    if (kTrace && warp == 7) FP8BS_TS(7, sit);
                }
                if constexpr (NC == 128) {
                    if (fold) {
                        fma32(r0, 0);
                        fma32(r1, 32);
                    } else {
                        fma32(r0, 64);
                        fma32(r1, 96);
                    }
                } else {
                    fma32(r1, 32);
                }
            };
            auto release_scales = [&](const int ss) __attribute__((always_inline)) {
                // The stage was written by TMA (async proxy) and read here with ld.shared (generic
                // proxy); the producer's next TMA into it must not overtake those reads, so a proxy
                // fence precedes the arrive.  Without it Wgrad's late per-column scale reads saw the
                // refilled stage, nondeterministically (tools/dbg_race.py: columns 96..127 of a half).
                if (!(kDbg & 512)) fence_proxy_async_smem();
                if (elect_one() && !((kDbg & 512))) mbar_arrive(sempty_bar(ss));
            };
            bool unrolled = false;
            // Fprop/Dgrad, dense and grouped (K-blocks a multiple of 8): in the Wgrad kernel the unrolled
            // body makes ptxas spill loop state into local memory (measured: Wgrad -7%); the split-K
            // units cover arbitrary K-block ranges
            if constexpr (!kWgrad && !kSplit) unrolled = p.KB % C::kSStages == 0;
            if (unrolled) {
                // K-blocks in groups of kSStages (8): the scale stage is the index in the group, the TMEM
                // slot alternates 2h, 2h + 1 and its phase flips every 2 K-blocks (sit and qh are
                // multiples of 8 at every tile start), so only the scale phase is a runtime value.
                for (int kb0 = 0; kb0 < p.KB; kb0 += C::kSStages, sit += C::kSStages, qh += C::kSStages) {
                    const uint32_t sph = (sit / C::kSStages) & 1;
#pragma unroll
                    for (int i = 0; i < C::kSStages; ++i) {
                        promote_kb(i, sph, 2 * h + (i & 1), (i >> 1) & 1, sit + i);
                        release_scales(i);
                    }
                }
            } else {
                for (int kb = 0; kb < nkb(tl); ++kb, ++sit, ++qh) {
                    promote_kb(sit & (C::kSStages - 1), (sit / C::kSStages) & 1, 2 * h + (qh & 1), (qh >> 1) & 1, sit);
                    release_scales(sit & (C::kSStages - 1));
                }
            }
            // ---------------- epilogue ----------------
            const int arow = kKR ? tl.orow0 + (int)rank * BM : cta_row0(tl);   // output rows
            // Each warp owns 32 rows x 128 columns.  It stages 128-byte-wide column chunks (32 FP32 or
            // 64 BF16 columns) in its own SWIZZLE_128B buffer and writes them with asynchronous TMA
            // stores (reduce-add for Wgrad's D += acc): a warp store used to touch 32 rows at once.
            // TMA clips rows >= M and columns >= N; a grouped warp whose 32 rows cross the expert's
            // end stores its rows directly (rows past row_end belong to the next expert).
            const int grow0 = arow + (fold ? (quad & 1) : quad) * 32;
            const int rows_here = tl.row_end - grow0;
            if constexpr (kSwiglu) {
                static_assert(NC == 128 && C::EPI_BUFS == 1, "SwiGLU epilogue: 8 promotion warps, one staging buffer each");
                // both warps of a (gate, up) pair share quad, hence rows_here
                if (rows_here > 0) swiglu_epilogue(acc, h, quad, lane, tl, grow0, rows_here, p,
                                                   smem_u32(s_epi) + (warp - 4) * C::EPI_WARP_BYTES,
                                                   smem_u32(s_epi) + (warp - 4 + (h == 0 ? 4 : -4)) * C::EPI_WARP_BYTES);
            } else
            if ((kDbg & 2048) && active) {       // experiment: keep the math, skip the stores
                float x = 0.0f;
#pragma unroll
                for (int i = 0; i < NC; ++i) x += acc[i];
                if (x == 1.2345e-30f) reinterpret_cast<float*>(p.D)[row] = x;
            } else if (active && rows_here > 0 && !(kDbg & 1024)) {
                constexpr int ESZ = kOutF32 ? 4 : 2;
                constexpr int CW = 128 / ESZ;                   // columns per 128-byte chunk
                // every warp stages its chunk the same way (one code path over acc); only the store
                // differs: a whole 32-row block goes out as one TMA store, the rows of a grouped warp
                // that crosses its expert's end are copied out of the staging buffer by the lanes
                const bool full = !kGrouped || (!kScatter && rows_here >= 32);
                const uint32_t ebuf0 = smem_u32(s_epi) + (warp - 4) * C::EPI_WARP_BYTES;
                // scatter: lane l resolves row l's destination once per tile into shared memory (the
                // chunks below read it back instead of the rank, slot and pointer table per store)
                const uint32_t sdst = smem_u32(smem + C::OFF_SCAT) + (warp - 4) * C::SCAT_BYTES;
                if constexpr (kScatter) {
                    const int64_t gr = grow0 + lane;
                    if (lane < rows_here) {
                        const uint64_t d = reinterpret_cast<uint64_t>(p.sc_base[__ldg(p.sc_rank + gr)]) +
                                           (uint64_t)(__ldg(p.sc_row + gr) * p.ldd) * ESZ;
                        asm volatile("st.shared.u64 [%0], %1;" :: "r"(sdst + 8u * lane), "l"(d) : "memory");
                    }
                    __syncwarp();
                }
#pragma unroll
                for (int c = 0; c < NC / CW; ++c) {
                    if (fold && c >= NC / CW / 2) break;         // folded: 64 columns per warp
                    const uint32_t ebuf = ebuf0 + (c % C::EPI_BUFS) * (32 * 128);
                    // the store that last used this buffer has read it
                    if (lane == 0) bulk_wait_group_read<C::EPI_BUFS - 1>();
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < 8; ++u) {                   // 16-byte units of this lane's row
                        uint32_t w[4];
                        if constexpr (kOutF32) {
#pragma unroll
                            for (int k = 0; k < 4; ++k) w[k] = __float_as_uint(acc[c * CW + 4 * u + k]);
                        } else {
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                __nv_bfloat162 b2 = __floats2bfloat162_rn(acc[c * CW + 8 * u + 2 * k], acc[c * CW + 8 * u + 2 * k + 1]);
                                w[k] = *reinterpret_cast<uint32_t*>(&b2);
                            }
                        }
                        sts_u32x4(ebuf + lane * 128 + ((u ^ (lane & 7)) << 4), w[0], w[1], w[2], w[3]);
                    }
                    const int col = (kSplit ? 0 : tl.n0) + h * HN + gg * NC + (fold ? (quad >> 1) * 64 : 0) + c * CW;   // split: the unit's slab
                    if (kGrouped && !full) {
                        __syncwarp();
                        const int nr = rows_here < 32 ? rows_here : 32;
                        for (int i = lane; i < nr * 8; i += 32) {
                            const int r = i >> 3, u = i & 7;
                            if (col + u * (16 / ESZ) < p.N) {
                                const uint4 v = lds_u32x4(ebuf + r * 128 + ((u ^ (r & 7)) << 4));
                                uint8_t* dst;
                                if constexpr (kScatter) {   // 8 lanes write one row's 128 bytes to its owner
                                    uint64_t d;
                                    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(d) : "r"(sdst + 8u * r));
                                    dst = reinterpret_cast<uint8_t*>(d) + (int64_t)col * ESZ + u * 16;
                                } else {
                                    dst = reinterpret_cast<uint8_t*>(p.D) + ((int64_t)(grow0 + r) * p.ldd + col) * ESZ + u * 16;
                                }
                                if (kOutF32 && p.accumulate) {          // Wgrad D += dW: this lane owns these 4 floats
                                    float4 o = *reinterpret_cast<const float4*>(dst);
                                    o.x += __uint_as_float(v.x); o.y += __uint_as_float(v.y);
                                    o.z += __uint_as_float(v.z); o.w += __uint_as_float(v.w);
                                    *reinterpret_cast<float4*>(dst) = o;
                                } else {
                                    *reinterpret_cast<uint4*>(dst) = v;
                                }
                            }
                        }
                        __syncwarp();                               // buffer reads done before its reuse
                        continue;
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (kOutF32 && p.accumulate) tma_reduce_add_2d(&tmD, ebuf, col, grow0);
                        else tma_store_2d(&tmD, ebuf, col, grow0);
                        bulk_commit_group();
                    }
                }
            }
        }
        if (lane == 0) bulk_wait_group<0>();           // all TMA stores of this warp complete
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

// Split-K tail, second step: D tile (+)= sum over chunks c = 0..S-1, in that order, of the FP32
// partials.  One thread per 4 columns of a row; block (x, i): rows 4x..4x+3 of tail tile i.
template <int ROWS>
__global__ void __launch_bounds__(256) k_splitk_reduce(const float* __restrict__ part, const KParams p,
                                                      void* D, int64_t ldd, int out_f32, int accumulate) {
    griddep_wait();
    griddep_launch_dependents();
    const int i = blockIdx.y;
    const int r = blockIdx.x * 4 + (threadIdx.x >> 6);
    const int c4 = threadIdx.x & 63;
    Tile tl;
    decode_dense<ROWS>(p, p.split_t0 + i, tl);
    const int row = tl.row0 + r, col = tl.n0 + 4 * c4;
    if (row >= p.M || col >= p.N) return;
    const float4* src = reinterpret_cast<const float4*>(part) + ((int64_t)i * p.split_s * ROWS + r) * (BN / 4) + c4;
    float4 acc = __ldcg(src);
    for (int c = 1; c < p.split_s; ++c) {
        const float4 v = __ldcg(src + (int64_t)c * ROWS * (BN / 4));
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (out_f32) {
        float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(D) + (int64_t)row * ldd + col);
        if (accumulate) {
            const float4 o = *d;
            acc.x = o.x + acc.x; acc.y = o.y + acc.y; acc.z = o.z + acc.z; acc.w = o.w + acc.w;
        }
        *d = acc;
    } else {
        __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&lo); w.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(D) + (int64_t)row * ldd + col) = w;
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

// Split-K tail plan of a dense launch (get_tile_split): tiles [t0, t0 + units / S) of the raster, each
// cut into S chunks along K.  Used when the last wave would fill at most half of the clusters: S =
// clusters / tail tiles (so the units fill one wave), and only when it saves at least kSplitMinSaved
// K-blocks of the tail tile's time: the second launch and the reduce cost ~20 us, about 40 K-blocks of a
// wave (measured: C1 Dgrad saves 136 and gains 10%; C1 Wgrad would save 24 and lost 4 us net).
struct SplitPlan { int t0 = 0, S = 0, units = 0; };
constexpr int kSplitMinKB = 4, kSplitMinSaved = 40;

static SplitPlan split_plan(int64_t M, int64_t N, int64_t K, int rows, int clusters) {
    SplitPlan sp;
    const int64_t tiles = ((M + rows - 1) / rows) * ((N + BN - 1) / BN);
    const int KB = (int)(K / BK);
    if (clusters < 2 || tiles <= 0) return sp;
    const int64_t rem = tiles % clusters;
    if (rem == 0) return sp;
    int S = (int)(clusters / rem);
    if (S > KB / kSplitMinKB) S = KB / kSplitMinKB;
    if (S < 2 || KB - KB / S < kSplitMinSaved) return sp;
    sp.t0 = (int)(tiles - rem); sp.S = S; sp.units = (int)rem * S;
    return sp;
}
static size_t split_bytes(const SplitPlan& sp, int rows) { return (size_t)sp.units * rows * BN * 4; }

// dense raster parameters (shared by the GEMM launches and the split-K reduce)
static void dense_raster(const GemmArgs& a, int rows, KParams& p) {
    p.num_m = (int)((a.M + rows - 1) / rows); p.num_n = (int)((a.N + BN - 1) / BN);
    // keep the smaller operand resident; band it to ~48 MB of L2 when it is larger than that
    p.rast_n = a.M > a.N ? 1 : 0;
    const int64_t res_rows = p.rast_n ? (int64_t)BN : (int64_t)rows;   // rows per resident tile
    const int nres = p.rast_n ? p.num_n : p.num_m;
    int64_t gb = ((int64_t)FP8BS_BAND_MB << 20) / (res_rows * a.K);
    p.gm = (int)(gb < 1 ? 1 : (gb > nres ? nres : gb));
}

template <bool kWgrad, int kOut, bool kGrouped, bool kPair>
static cudaError_t launch_cfg(const GemmArgs& a, cudaStream_t st, const char** detail, const SplitPlan* sp = nullptr) {
    using C = Cfg<kPair, kWgrad>;
    constexpr bool kSplit = kOut == kOutSplit, kScatter = kOut == kOutScatter;
    constexpr bool kOutF32 = kOut == kOutFP32 || kSplit, kSwiglu = kOut == kOutSwiglu;
    const int KB = (int)(a.K / BK);
    constexpr bool kGW = kWgrad && kGrouped;   // grouped Wgrad: A = dYqT [M, Mp], D = [G x M, N]
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
    if (kGrouped && !kWgrad) {
        uint64_t dims[3] = {(uint64_t)a.K, (uint64_t)a.N, (uint64_t)a.G};
        uint64_t str[2] = {(uint64_t)a.K, (uint64_t)a.K * (uint64_t)a.N};
        uint32_t box[3] = {BK, (uint32_t)C::BH_ROWS, 1};
        if (!make_map(&tB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, a.B, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) {
            *detail = "cuTensorMapEncodeTiled failed for B (grouped)"; return cudaErrorInvalidValue;
        }
    } else {
        uint64_t dims[2] = {(uint64_t)a.K, (uint64_t)a.N};
        uint64_t str[1] = {(uint64_t)a.ldb};
        uint32_t box[2] = {BK, (uint32_t)C::BH_ROWS};
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
    } else if (kGrouped && kPair) {
        // folded tiles (M = 128 over the pair): A with a 64-row box, passed in tmSB's place
        uint64_t dims[2] = {(uint64_t)a.K, (uint64_t)rows};
        uint64_t str[1] = {(uint64_t)a.lda};
        uint32_t box[2] = {BK, BM / 2};
        if (!make_map(&tSB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, a.A, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) {
            *detail = "cuTensorMapEncodeTiled failed for A (64-row box)"; return cudaErrorInvalidValue;
        }
    } else {
        tSB = tSA;
    }
    CUtensorMap tD, tD2;
    if constexpr (kSwiglu) {
        // codes: y [M, N/2] (D) and the H cache [M, N] (qh), 32 rows x 128 bytes per store
        uint64_t dims[2] = {(uint64_t)(a.N / 2), (uint64_t)rows};
        uint64_t str[1] = {(uint64_t)a.ldd};
        uint32_t box[2] = {128, 32};
        if (!make_tmap(&tD, TMAP_U8, 2, a.D, dims, str, box, 128)) {
            *detail = "cuTensorMapEncodeTiled failed for the SwiGLU codes"; return cudaErrorInvalidValue;
        }
        tD2 = tD;
        if (a.qh) {
            uint64_t dh[2] = {(uint64_t)a.N, (uint64_t)rows};
            uint64_t sh[1] = {(uint64_t)a.ldqh};
            if (!make_tmap(&tD2, TMAP_U8, 2, a.qh, dh, sh, box, 128)) {
                *detail = "cuTensorMapEncodeTiled failed for the SwiGLU input cache"; return cudaErrorInvalidValue;
            }
        }
    } else if constexpr (kScatter) {
        tD = tA; tD2 = tA;                 // no D tensor: rows are stored through the pointer table
    } else if constexpr (kSplit) {
        // the units' FP32 partial slabs: [units x ROWS, BN] in the caller's workspace
        uint64_t dims[2] = {(uint64_t)BN, (uint64_t)sp->units * C::ROWS};
        uint64_t str[1] = {(uint64_t)BN * 4};
        uint32_t box[2] = {32, 32};
        if (!make_tmap(&tD, TMAP_F32, 2, a.split_ws, dims, str, box, 128)) {
            *detail = "cuTensorMapEncodeTiled failed for the split-K workspace"; return cudaErrorInvalidValue;
        }
        tD2 = tD;
    } else {
        const uint64_t esz = kOutF32 ? 4 : 2;
        uint64_t dims[2] = {(uint64_t)a.N, (uint64_t)(kGW ? rows * a.G : rows)};   // grouped Wgrad: experts stacked
        uint64_t str[1] = {(uint64_t)a.ldd * esz};
        uint32_t box[2] = {(uint32_t)(128 / esz), 32};
        if (!make_tmap(&tD, kOutF32 ? TMAP_F32 : TMAP_BF16, 2, a.D, dims, str, box, 128)) {
            *detail = "cuTensorMapEncodeTiled failed for D"; return cudaErrorInvalidValue;
        }
        tD2 = tD;
    }
    KParams p{};
    p.M = (int)a.M; p.N = (int)a.N; p.K = (int)a.K; p.KB = KB;
    p.sy = a.sy; p.ldsy = a.ldsy; p.qh = a.qh; p.ldqh = a.ldqh; p.sh = a.sh; p.ldsh = a.ldsh;
    dense_raster(a, C::ROWS, p);
    p.NB = (int)((a.N + 127) / 128);
    p.sB = a.sB;
    if (kGrouped && a.layout == 1) { p.sb_nb_stride = 1; p.sb_kb_stride = p.NB; p.sb_expert_stride = (int64_t)p.NB * KB; }   // grouped Dgrad
    else if (kGrouped) { p.sb_nb_stride = KB; p.sb_kb_stride = 1; p.sb_expert_stride = (int64_t)p.NB * KB; }
    else if (a.layout == 0) { p.sb_nb_stride = a.ldsB; p.sb_kb_stride = 1; p.sb_expert_stride = 0; }
    else { p.sb_nb_stride = 1; p.sb_kb_stride = a.ldsB; p.sb_expert_stride = 0; }
    p.D = a.D; p.ldd = a.ldd; p.accumulate = a.accumulate;
    p.sc_base = a.sc_base; p.sc_rank = a.sc_rank; p.sc_row = a.sc_row;
    p.Bp = a.B; p.b_expert_bytes = (int64_t)a.N * a.K;
    p.b_pf_chunk = (int)(((p.b_expert_bytes + 15) / 16 + 15) / 16 * 16);     // 16 chunks, multiples of 16 bytes
    p.b_pf_last_or_chunk[0] = p.b_pf_chunk;
    p.b_pf_last_or_chunk[1] = (int)max((int64_t)16, p.b_expert_bytes - 15 * (int64_t)p.b_pf_chunk);
    p.ready = a.ready; p.ready_target = a.ready_target; p.ready_chunks = a.ready_chunks;
    p.G = a.G; p.offsets = a.offsets; p.tiles = a.workspace;
    p.tile_end = sp ? sp->t0 : p.num_m * p.num_n;
    if constexpr (kSplit) {
        p.split_t0 = sp->t0; p.split_s = sp->S; p.split_units = sp->units;
        p.accumulate = 0;                      // the reduce adds into D
    }
    {
        if (kDbg & 16) {
            if (!g_ts) cudaMalloc(&g_ts, kTsSlots * kTsN * sizeof(unsigned long long));
            cudaMemsetAsync(g_ts, 0, kTsSlots * kTsN * sizeof(unsigned long long), st);
            p.ts = g_ts;
        }
    }

    int64_t tiles_ub;
    if (kGW) tiles_ub = (int64_t)a.G * p.num_m * p.num_n;
    else if (kGrouped) tiles_ub = ((a.M + C::ROWS - 1) / C::ROWS + a.G) * (int64_t)p.num_n;
    else if (kSplit) tiles_ub = sp->units;
    else tiles_ub = p.tile_end;
    int64_t max_clusters = num_sms() / C::CS;
    if (a.max_sms > 0 && a.max_sms / C::CS < max_clusters) max_clusters = a.max_sms / C::CS;   // SMs left to a concurrent kernel
    int clusters = (int)(tiles_ub < max_clusters ? tiles_ub : max_clusters);
    if (clusters < 1) clusters = 1;
    const int smem = C::SMEM_DENSE;
    if (kGrouped && !kWgrad) {
        // the tile table for this launch (k_grouped_schedule), then the GEMM; both PDL
        const int64_t ub = ((a.M + C::ROWS - 1) / C::ROWS + a.G) * (int64_t)p.num_n;   // tiles, upper bound
        int64_t sg = (ub + 4 * kMaxGroups - 1) / (4 * kMaxGroups);                    // ~4 entries per thread
        sg = sg < 1 ? 1 : (sg > num_sms() ? num_sms() : sg);
        cudaError_t e = launch_pdl(k_grouped_schedule, dim3((unsigned)sg), dim3(kMaxGroups), 0, st, a.offsets, a.G,
                                   C::ROWS, p.num_n, p.N, reinterpret_cast<TileTable*>(a.workspace));
        if (e != cudaSuccess) return e;
    }
    auto kern = k_gemm_bs<kWgrad, kOut, kGrouped, kPair>;
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
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C::CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (internal.h launch_pdl)
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    GWSched<kGW ? kGWMax : 1> gw;
    if constexpr (kGW) {
        for (int e = 0; e < a.G; ++e) gw.e[e] = make_int2(a.gw_kb[2 * e], a.gw_kb[2 * e + 1]);
    } else {
        gw.e[0] = make_int2(0, 0);
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tA, tB, tSA, tSB, tD, tD2, p, gw);
    if (e != cudaSuccess) return e;
    return cudaPeekAtLastError();
}

#if FP8BS_TEST_HOOKS
// Test-only build (libfp8bs_testhooks.so): tests force the tile variant through an exported hook.
// The product library has no such state: the variant follows from the problem shape alone.
static int g_forced_variant = 0;
#endif

// A dense launch, with the split-K tail when the caller passed a workspace and the shape has one:
// the full waves (if any), the tail units, then the reduce — three kernels on `st`, chained by PDL.
template <bool kWgrad, int kOut, bool kPair>
static cudaError_t launch_dense(const GemmArgs& a, cudaStream_t st, const char** detail) {
    using C = Cfg<kPair, kWgrad>;
    const SplitPlan sp = split_plan(a.M, a.N, a.K, C::ROWS, num_sms() / C::CS);
    if (sp.S < 2 || !a.split_ws || a.split_ws_bytes < split_bytes(sp, C::ROWS))
        return launch_cfg<kWgrad, kOut, false, kPair>(a, st, detail);
    cudaError_t e;
    if (sp.t0 > 0 && (e = launch_cfg<kWgrad, kOut, false, kPair>(a, st, detail, &sp)) != cudaSuccess) return e;
    if ((e = launch_cfg<kWgrad, kOutSplit, false, kPair>(a, st, detail, &sp)) != cudaSuccess) return e;
    KParams p{};
    p.M = (int)a.M; p.N = (int)a.N; p.K = (int)a.K; p.KB = (int)(a.K / BK);
    dense_raster(a, C::ROWS, p);
    p.split_t0 = sp.t0; p.split_s = sp.S; p.split_units = sp.units;
    e = launch_pdl(k_splitk_reduce<C::ROWS>, dim3(C::ROWS / 4, sp.units / sp.S), dim3(256), 0, st,
                   static_cast<const float*>(a.split_ws), p, a.D, a.ldd, a.out_f32, a.accumulate);
    if (e != cudaSuccess) return e;
    return cudaPeekAtLastError();
}

size_t split_workspace_bytes(int64_t M, int64_t N, int64_t K) {
    // either tile variant (the test build can force one): the larger of the two plans
    size_t b = 0;
    const SplitPlan s1 = split_plan(M, N, K, BM, num_sms()), s2 = split_plan(M, N, K, 2 * BM, num_sms() / 2);
    if (s1.S >= 2) b = split_bytes(s1, BM);
    if (s2.S >= 2 && split_bytes(s2, 2 * BM) > b) b = split_bytes(s2, 2 * BM);
    return b;
}

template <bool kPair>
static cudaError_t launch_v(const GemmArgs& a, cudaStream_t st, const char** detail) {
    if (a.grouped && a.layout == 2) return launch_cfg<true, kOutFP32, true, kPair>(a, st, detail);
    if (a.swiglu) {
        return a.grouped ? launch_cfg<false, kOutSwiglu, true, kPair>(a, st, detail)
                         : launch_cfg<false, kOutSwiglu, false, kPair>(a, st, detail);
    }
    if (a.grouped) {
        if (a.sc_base) return launch_cfg<false, kOutScatter, true, kPair>(a, st, detail);
        return a.out_f32 ? launch_cfg<false, kOutFP32, true, kPair>(a, st, detail)
                         : launch_cfg<false, kOutBF16, true, kPair>(a, st, detail);
    }
    if (a.layout == 2) return launch_dense<true, kOutFP32, kPair>(a, st, detail);
    return a.out_f32 ? launch_dense<false, kOutFP32, kPair>(a, st, detail)
                     : launch_dense<false, kOutBF16, kPair>(a, st, detail);
}

size_t grouped_workspace_bytes(int32_t G, int64_t total_M, int64_t N) {
    // TileTable header + one int4 per tile; 128-row tiles bound both variants
    const int64_t tiles = ((total_M + BM - 1) / BM + G) * ((N + BN - 1) / BN);
    return (size_t)(16 + 16 * (tiles > 0 ? tiles : 1));
}

// Variants: 1 = one CTA per 128 x 256 tile, 2 = CTA pair (cta_group::2) per 256 x 256 tile.
cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t st, const char** detail) {
    int v = 0;
#if FP8BS_TEST_HOOKS
    v = g_forced_variant;
#endif
    if (v < 1 || v > 2) {
        // grouped Fprop/Dgrad: pairs from 128 rows per expert on average (an expert ending within a
        // pair tile's first 128 rows runs it folded, at half the MMA work).  Measured with uniform top-8
        // routing over 256 experts, K = 7168, N = 2048 (tools/gemm_matrix.py, r02; one CTA / pair, us):
        // 112 rows per expert 669-687 / 727-746; 128: 815-966 / 788-845 (box to box); 144: 988-1200 /
        // 922; 160: 1128-1242 / 943; 192: 1268-1370 / 893-936; 224: 1286-1383 / 898-1012; 256:
        // 1295-1314 / 1157-1166.  The grouped SwiGLU epilogue has no folded tiles: pairs from 256 rows
        // (tools/swiglu_bench.py SWIGLU_SWEEP, r02, one CTA / pair, ms: 256 rows 2.574 / 2.580, 384:
        // 3.463 / 3.310, 512: 4.256 / 4.106, 2048: 14.29 / 13.07; before the promotion's busy-poll the
        // pair kernel spilled ~300 bytes and lost at every size).  (Grouped Wgrad: a.M is one expert's
        // output rows — the dense per-expert choice.)
        if (a.grouped && a.layout != 2) v = (a.M / (a.G > 0 ? a.G : 1) >= (a.swiglu ? 256 : 128)) ? 2 : 1;
        else v = (a.M <= 128) ? 1 : 2;
    }
    return v == 1 ? launch_v<false>(a, st, detail) : launch_v<true>(a, st, detail);
}

}  // namespace fp8bs

#if FP8BS_TEST_HOOKS
// Test-only build (not in include/fp8bs.h, not in libfp8bs.so): copy the debug timestamps of the last
// GEMM launch (experiment builds with FP8BS_GEMM_DEBUG_BITS & 16), and force the tile variant
// (1: one CTA per 128-row tile, 2: CTA pair per 256-row tile, 0: by shape) for later launches.
extern "C" __attribute__((visibility("default"))) int fp8bs_internal_debug_timestamps(unsigned long long* host, int n) {
    if (!fp8bs::g_ts) return 0;
    if (n > fp8bs::kTsSlots * fp8bs::kTsN) n = fp8bs::kTsSlots * fp8bs::kTsN;
    cudaDeviceSynchronize();
    cudaMemcpy(host, fp8bs::g_ts, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    return n;
}
extern "C" __attribute__((visibility("default"))) void fp8bs_internal_set_gemm_variant(int v) { fp8bs::g_forced_variant = v; }
#endif
