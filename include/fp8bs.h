/* include/fp8bs.h — C-ABI of libfp8bs.so: DeepSeek-V3 fine-grained FP8 quantization and
 * block-scaled FP8 GEMMs with FP32 accumulation, hand-written for B200 (sm_100a).
 *
 * Paper: arXiv 2412.19437 (DeepSeek-V3), §3.3 "FP8 Training", /root/reference/PAPER.md:
 *   P:503-510  fine-grained quantization: 1x128 tiles for activations ("per token per 128
 *              channels"), 128x128 blocks for weights;
 *   P:512-514  per-group scaling factors along the GEMM inner dimension K;
 *   P:526-534  FP32 promotion of tensor-core partial sums every N_C = 128 elements, where
 *              the per-group scales are multiplied in;
 *   P:536-539  E4M3 on all tensors;  P:541-544  online max-abs scaling;
 *   P:476-481  Fprop / Dgrad / Wgrad GEMMs all in FP8, outputs BF16 or FP32;
 *   P:558, P:672-673, P:1568-1571  128x1 tiles for the backward (Wgrad) operands.
 * Numerical contract (readings R1-R8): s = RN32(amax / 448.0f) (1 if 0),
 * q = E4M3_RNE_SATFINITE(RN32(x / s)); quantizer outputs are bit-exact vs the CPU oracle.
 *
 * CONVENTIONS (all functions)
 *   - Every tensor pointer is a DEVICE pointer (cudaMalloc / torch CUDA memory) on the
 *     current device; all matrices are row-major with explicit leading dimensions `ld*`
 *     counted in ELEMENTS.  E4M3 codes are stored as uint8_t.
 *   - Ownership: the caller allocates and frees every buffer.  The library never
 *     allocates, frees or retains device memory and keeps no state across calls (except a
 *     once-only lookup of the driver entry point cuTensorMapEncodeTiled).
 *   - Asynchrony: compute calls validate their arguments on the host, enqueue kernels on
 *     `stream` and return; there is no implicit synchronisation and no device->host read.
 *   - Errors: validation happens before any launch; a failing call has no side effects and
 *     returns a non-zero fp8bs_status.  fp8bs_last_error_detail() (thread-local) explains
 *     the last failure.  Kernel launch failures are reported as FP8BS_ERR_CUDA.
 *   - Thread safety: reentrant; concurrent calls on different streams / devices are safe.
 */
#ifndef FP8BS_H
#define FP8BS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FP8BS_ABI_VERSION 3   /* 2: fp8bs_grouped_gemm{,_dgrad} require their workspace; 3: so do the _mx forms */

#if defined(__GNUC__)
#define FP8BS_API __attribute__((visibility("default")))
#else
#define FP8BS_API
#endif

typedef struct CUstream_st* fp8bs_stream_t;   /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    FP8BS_OK = 0,
    FP8BS_ERR_INVALID_ARG = 1,   /* NULL pointer, negative size, bad enum */
    FP8BS_ERR_SHAPE = 2,         /* inconsistent sizes / leading dimensions, K % 128 != 0 */
    FP8BS_ERR_ALIGN = 3,         /* pointer or row pitch not 16-byte aligned (TMA) */
    FP8BS_ERR_UNSUPPORTED = 4,   /* valid but unsupported combination (e.g. BF16 + accumulate) */
    FP8BS_ERR_DEVICE = 5,        /* no CUDA device, or not compute capability 10.0 (sm_100) */
    FP8BS_ERR_CUDA = 6           /* CUDA runtime / driver error during launch */
} fp8bs_status;

typedef enum { FP8BS_BF16 = 0, FP8BS_FP32 = 1 } fp8bs_dtype;

/* GEMM layouts of a Linear with weight W [out, in] over T tokens.  In every layout
 * D[i,j] (+)= sum_c deq(A)[i,c] * deq(B)[j,c]; A [M,K] and B [N,K] are both K-major.
 *   FPROP: A = Xq [T, in]     (1x128),      B = Wq  [out, in] (128x128) -> D = Y  [T, out]
 *   DGRAD: A = dYq [T, out]   (1x128),      B = WqT [in, out] (128x128) -> D = dX [T, in]
 *   WGRAD: A = dYqT [out, T]  (128x1),      B = XqT [in, T]   (128x1)   -> D = dW [out, in] FP32 */
typedef enum { FP8BS_FPROP = 0, FP8BS_DGRAD = 1, FP8BS_WGRAD = 2 } fp8bs_layout;

FP8BS_API int          fp8bs_abi_version(void);                  /* returns FP8BS_ABI_VERSION */
FP8BS_API const char*  fp8bs_status_string(fp8bs_status status); /* static string; never NULL */
FP8BS_API const char*  fp8bs_last_error_detail(void);            /* thread-local; "" if none */
FP8BS_API fp8bs_status fp8bs_device_supported(int device);       /* FP8BS_OK iff CC 10.0 (sm_100) */

/* ---- quantize_act_1x128 ("per token per 128 channels", P:541-544 online) ----------
 * x   : [M, K] activations, dtype xdt (BF16 or FP32), leading dimension ldx >= K.
 * q   : [M, K] uint8 E4M3 codes, ldq >= K:   q[m*ldq + k] = E4M3(x[m,k] / s[kb][m]).
 * s   : [ceil(K/128), lds] FP32 scales, lds >= M ("contraction-block-major", so a GEMM can load
 *       one contiguous vector of 128 row scales per K block):  s[kb*lds + m] = amax/448 (1 if 0),
 *       amax = max |x[m, kb*128 .. kb*128+127]| (NaN ignored; a short last group uses the
 *       elements that exist).
 * Any M, K >= 0 (M == 0 or K == 0 is a no-op).  No alignment requirement (unaligned or odd
 * shapes take a slower generic kernel). */
FP8BS_API fp8bs_status fp8bs_quantize_act_1x128(const void* x, fp8bs_dtype xdt, int64_t M, int64_t K, int64_t ldx,
                                      uint8_t* q, int64_t ldq, float* s, int64_t lds,
                                      fp8bs_stream_t stream);

/* ---- quantize_act_1x128_pow2: 1x128 tiles with power-of-two scales --------------------------
 * P:558 ("integral power of 2" scaling factors for the inputs of the Linear after attention) and
 * P:565 (the activations quantized before MoE dispatch).  As fp8bs_quantize_act_1x128 except
 * s = 2^e, the smallest power of two with 448 * 2^e >= amax (reading R23: rounded up from the exact
 * quotient, so nothing saturates; amax 3.0 -> s = 2^-7, 3.0 / s = 384), e >= -127
 * (reading R26: the smallest UE8M0 value, so the scales are exact inputs of fp8bs_gemm_mx), 1 for an
 * all-zero tile.  The quotient x / s is then exact before the E4M3 rounding.  Same layouts,
 * ownership and errors as fp8bs_quantize_act_1x128; the scales feed fp8bs_gemm unchanged. */
FP8BS_API fp8bs_status fp8bs_quantize_act_1x128_pow2(const void* x, fp8bs_dtype xdt, int64_t M, int64_t K, int64_t ldx,
                                           uint8_t* q, int64_t ldq, float* s, int64_t lds, fp8bs_stream_t stream);

/* ---- quantize_act_128x1: transpose-quantize for Wgrad operands --------
 * x   : [M, C] activations (M tokens, C channels), ldx >= C.
 * qT  : [C, M] uint8 codes, ldq >= M:  qT[c*ldq + m] = E4M3(x[m,c] / sT[mb][c]), mb = m/128.
 * sT  : [ceil(M/128), lds] FP32, lds >= C:  sT[mb*lds + c] = amax over x[mb*128 .. +127, c] / 448.
 * Built from BF16/FP32 (single rounding; reading R10).  Any M, C >= 0. */
FP8BS_API fp8bs_status fp8bs_quantize_act_128x1(const void* x, fp8bs_dtype xdt, int64_t M, int64_t C, int64_t ldx,
                                      uint8_t* qT, int64_t ldq, float* sT, int64_t lds,
                                      fp8bs_stream_t stream);

/* ---- quantize_act_dual: 1x128 AND 128x1 groupings of one activation from a single read -------
 * The same outputs as fp8bs_quantize_act_1x128(x -> q, s) followed by
 * fp8bs_quantize_act_128x1(x -> qT, sT), bit for bit (P:508 groupings, P:558 / P:1568-1569 128x1
 * tiles for Wgrad).  A training step needs both groupings of X (Fprop, Wgrad) and of dY (Dgrad,
 * Wgrad); reading x once follows the paper's call to fuse the FP8 cast with the memory access
 * (§3.5.2).  Fused for BF16 x with 16-byte aligned rows and K % 16 == 0; otherwise it
 * runs the two single-grouping kernels.  Layouts, ownership and errors as the two calls above
 * (ldx >= K, ldq >= K, lds >= M, ldqT >= M, ldsT >= K). */
FP8BS_API fp8bs_status fp8bs_quantize_act_dual(const void* x, fp8bs_dtype xdt, int64_t M, int64_t K, int64_t ldx,
                                     uint8_t* q, int64_t ldq, float* s, int64_t lds,
                                     uint8_t* qT, int64_t ldqT, float* sT, int64_t ldsT,
                                     fp8bs_stream_t stream);

/* ---- quantize_act_dual_pow2: the dual quantizer with power-of-two scales --------------------
 * As fp8bs_quantize_act_dual, every scale (both groupings) the smallest 2^e with 448 * 2^e >= amax
 * (reading R23, see fp8bs_quantize_act_1x128_pow2).  The outputs feed fp8bs_gemm_mx
 * (UE8M0 block scaling) or fp8bs_gemm.  Same layouts, ownership and errors; fused for BF16 x with
 * 16-byte aligned rows and K % 16 == 0, a generic two-pass kernel otherwise. */
FP8BS_API fp8bs_status fp8bs_quantize_act_dual_pow2(const void* x, fp8bs_dtype xdt, int64_t M, int64_t K, int64_t ldx,
                                          uint8_t* q, int64_t ldq, float* s, int64_t lds,
                                          uint8_t* qT, int64_t ldqT, float* sT, int64_t ldsT,
                                          fp8bs_stream_t stream);

/* ---- requantize_1x128_to_128x1: FP8 -> FP8 re-quantization of a cached activation ---------
 * P:558 (§3.3.3) and P:672-673 (§3.5.2): the FP8 activations kept from the forward pass are "read
 * out, dequantized, transposed, re-quantized into 128x1 tiles" for the Wgrad GEMM.
 * q   : [M, K] uint8 codes in 1x128 tiles (fp8bs_quantize_act_1x128 output), ldq >= K.
 * s   : [ceil(K/128), lds] FP32, lds >= M: s[(k/128)*lds + m].
 * Dequantized value xhat[m,k] = RN32(dec(q[m,k]) * s[(k/128)*lds + m]) (FP32), then the 128x1
 * quantization of xhat exactly as fp8bs_quantize_act_128x1 (same contract, same outputs):
 * qT  : [K, M] uint8, ldqT >= M: qT[k*ldqT + m].    sT : [ceil(M/128), ldsT] FP32, ldsT >= K.
 * pow2 != 0: the output scales are powers of two (the paper's choice for this conversion, P:558:
 *   s = the smallest 2^e with 448 * 2^e >= amax, see fp8bs_quantize_act_1x128_pow2).  With pow2
 *   input scales too, every re-quantized code is the input code shifted by a power of two: no extra
 *   rounding unless it falls below E4M3's normal range (the paper's rationale).
 * Alignment: q, qT 16-byte aligned, ldq and ldqT multiples of 16 (else FP8BS_ERR_ALIGN).
 * Any M, K >= 0 (short last groups on both axes).  Bit-exact vs the CPU oracle. */
FP8BS_API fp8bs_status fp8bs_requantize_1x128_to_128x1(const uint8_t* q, int64_t ldq, const float* s, int64_t lds,
                                             int64_t M, int64_t K, uint8_t* qT, int64_t ldqT,
                                             float* sT, int64_t ldsT, int pow2, fp8bs_stream_t stream);

/* ---- quantize_weight_128x128 ("per 128 input channels per 128 output channels") ----
 * w   : [N, K] weights (FP32 master weights, or BF16), ldw >= K.
 * q   : [N, K] uint8 codes, ldq >= K.
 * s   : [ceil(N/128), ldsw] FP32, ldsw >= ceil(K/128):  s[nb*ldsw + kb] = block amax / 448.
 * qT  : optional [K, N] transposed copy of q (qT[k*ldqT + n] == q[n*ldq + k]), ldqT >= N, used as
 *       the Dgrad B operand; pass NULL to skip.  Any N, K >= 0. */
FP8BS_API fp8bs_status fp8bs_quantize_weight_128x128(const void* w, fp8bs_dtype wdt, int64_t N, int64_t K, int64_t ldw,
                                           uint8_t* q, int64_t ldq, float* s, int64_t ldsw,
                                           uint8_t* qT, int64_t ldqT, fp8bs_stream_t stream);

/* ---- quantize_weight_128x128_pow2: 128x128 blocks with power-of-two scales -------------------
 * As fp8bs_quantize_weight_128x128, s[nb*ldsw + kb] = the smallest 2^e with 448 * 2^e >= block amax
 * (the power-of-two option of P:558 / P:565 applied to the weights so that a whole layer runs on
 * UE8M0 scales, fp8bs_gemm_mx).  Same layouts, ownership and errors. */
FP8BS_API fp8bs_status fp8bs_quantize_weight_128x128_pow2(const void* w, fp8bs_dtype wdt, int64_t N, int64_t K, int64_t ldw,
                                                uint8_t* q, int64_t ldq, float* s, int64_t ldsw,
                                                uint8_t* qT, int64_t ldqT, fp8bs_stream_t stream);

/* ---- gemm: block-scaled FP8 GEMM, FP32 accumulation -----
 * D[i,j] (+)= sum_kb sA(kb,i) * sB(kb,j) * sum_{c in kb} dec(A[i,c]) * dec(B[j,c])
 *   i < M, j < N, contraction K with K % 128 == 0 ("misaligned groups" otherwise).
 * A   : [M, K] uint8 codes, lda >= K.          sA : [K/128, ldsA], ldsA >= M: sA(kb,i) = sA[kb*ldsA + i].
 * B   : [N, K] uint8 codes, ldb >= K.
 * sB  : FPROP  [ceil(N/128), ldsB], ldsB >= K/128 : sB(kb,j) = sB[(j/128)*ldsB + kb]
 *       DGRAD  [K/128, ldsB], ldsB >= ceil(N/128) : sB(kb,j) = sB[kb*ldsB + j/128]
 *                (the SAME sW array quantize_weight_128x128 wrote, read as [out-block][in-block])
 *       WGRAD  [K/128, ldsB], ldsB >= N            : sB(kb,j) = sB[kb*ldsB + j]   (128x1 scales)
 * D   : [M, N] of dtype ddt, ldd >= N.  FPROP/DGRAD: BF16 (round-to-nearest-even) or FP32.
 *       WGRAD: FP32 only; accumulate != 0 adds into D (gradient accumulation).
 *       accumulate with BF16 output -> FP8BS_ERR_UNSUPPORTED.
 * Alignment: A, B, D 16-byte aligned; lda, ldb multiples of 16; sA, sB 16-byte aligned with ldsA
 * (and WGRAD ldsB) multiples of 4; ldd*sizeof(ddt) a multiple of 16; N a multiple of 8 (BF16)
 * or 4 (FP32) -> else FP8BS_ERR_ALIGN.  M, N, K <= 2^31 - 1.  M == 0 or N == 0 is a no-op. */
FP8BS_API fp8bs_status fp8bs_gemm(fp8bs_layout layout, int64_t M, int64_t N, int64_t K,
                        const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                        const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                        void* D, fp8bs_dtype ddt, int64_t ldd, int accumulate,
                        fp8bs_stream_t stream);

/* ---- gemm_ws: fp8bs_gemm with a workspace for the split-K tail --------------------------------
 * Same arguments, layouts, validation and result definition as fp8bs_gemm, plus
 * workspace : DEVICE scratch, 16-byte aligned, owned by the caller, of at least
 *             fp8bs_gemm_workspace_size(layout, M, N, K) bytes (<= 19.4 MB on a 148-SM B200), or NULL.
 * When the last wave of output tiles would fill at most half of the SMs (C1's Dgrad: 448 tiles on 74
 * CTA pairs = 6 waves + 4 tiles), those tail tiles are cut along K into S chunks of consecutive
 * K-blocks (S = clusters / tail tiles, >= 4 K-blocks each); every chunk is promoted exactly like a whole
 * tile over its own K-blocks into an FP32 partial in the workspace, and a reduce kernel
 * adds the S partials in chunk order in FP32 and writes D (BF16 RNE or FP32; WGRAD accumulate:
 * D + sum).  Only the FP32 summation order of the tail tiles differs from fp8bs_gemm (R30):
 * deterministic, and the same error bound.  Three kernels on `stream` instead of one; the workspace
 * must not be reused until they have run.  workspace == NULL, or a shape without such a tail
 * (fp8bs_gemm_workspace_size == 0): identical to fp8bs_gemm.  workspace_bytes below the required size:
 * FP8BS_ERR_INVALID_ARG; misaligned: FP8BS_ERR_ALIGN (both before any launch). */
FP8BS_API fp8bs_status fp8bs_gemm_ws(fp8bs_layout layout, int64_t M, int64_t N, int64_t K,
                           const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                           const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                           void* D, fp8bs_dtype ddt, int64_t ldd, int accumulate,
                           void* workspace, size_t workspace_bytes, fp8bs_stream_t stream);
/* Bytes fp8bs_gemm_ws needs for this shape on the CURRENT device (its SM count decides the waves); 0
 * when there is no split-K tail or the arguments are invalid. */
FP8BS_API size_t fp8bs_gemm_workspace_size(fp8bs_layout layout, int64_t M, int64_t N, int64_t K);

/* ---- gemm_mx: the same GEMM for POWER-OF-TWO scales on the tensor core's block scaling ----------
 * NEXT-1 (P:558, P:565 power-of-two scales; scaling inside the MMA).  Identical arguments,
 * layouts and validation as fp8bs_gemm, with one precondition: every sA and sB value is an exact power
 * of two in [2^-127, 2^127] (e.g. from fp8bs_quantize_act_1x128_pow2).  Each scale is passed to
 * tcgen05.mma.kind::mxf8f6f4.block_scale as its UE8M0 exponent, so there is no FP32 promotion step;
 * a scale that is not a power of two is silently truncated to its exponent (undefined results). */
FP8BS_API fp8bs_status fp8bs_gemm_mx(fp8bs_layout layout, int64_t M, int64_t N, int64_t K,
                           const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                           const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                           void* D, fp8bs_dtype ddt, int64_t ldd, int accumulate,
                           fp8bs_stream_t stream);

/* ---- grouped_gemm: MoE expert Fprop over token rows grouped by expert
 * offsets : DEVICE int64 [G+1], offsets[0] = 0, non-decreasing, offsets[G] = total_M; rows
 *           [offsets[e], offsets[e+1]) of A belong to expert e.  Any M_e >= 0 (no token
 *           dropping, no capacity padding).  Never read by the host (no device->host sync).
 *           Violations (decreasing offsets) are undefined behaviour (clamped, no trap).
 * A   : [total_M, K] uint8 codes, lda >= K;  sA : [K/128, ldsA], ldsA >= total_M (1x128 scales).
 * B   : [G, N, K] uint8 codes, contiguous (expert stride N*K);
 * sB  : [G, ceil(N/128), K/128] FP32, contiguous (FPROP 128x128 scales per expert).
 * D   : [total_M, N], BF16 or FP32, ldd >= N.
 * workspace : DEVICE scratch, 16-byte aligned, of at least fp8bs_grouped_gemm_workspace_size(G,
 *           total_M, N, K) bytes (16 bytes per 128 x 256 output tile + 16; ~0.3 MB at C4), owned by
 *           the caller and not read by the host.  The call first launches a one-CTA scheduler that
 *           writes this launch's tile table there (the (expert, m-tile, n-tile) order, from offsets on
 *           the device), then the GEMM, both on `stream`: the workspace must not be reused by
 *           another call until this one has run.  NULL or too small: FP8BS_ERR_INVALID_ARG.
 * 1 <= G <= 1024.  K a multiple of 128.  Same alignment rules as fp8bs_gemm. */
FP8BS_API fp8bs_status fp8bs_grouped_gemm(int32_t G, int64_t total_M, int64_t N, int64_t K, const int64_t* offsets,
                                const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                const uint8_t* B, const float* sB,
                                void* D, fp8bs_dtype ddt, int64_t ldd,
                                void* workspace, size_t workspace_bytes, fp8bs_stream_t stream);

/* ---- grouped_gemm_mx: the MoE expert Fprop on UE8M0 block scaling (NEXT-1) -----
 * fp8bs_grouped_gemm's arguments, layouts, validation and workspace (ABI 3: at least
 * fp8bs_grouped_gemm_workspace_size bytes; the call zeroes its first 4 bytes on `stream` and uses them
 * as the tile claim counter), with fp8bs_gemm_mx's precondition: every sA and sB value is an exact
 * power of two in [2^-127, 2^127] (e.g. from fp8bs_quantize_act_dual_pow2 /
 * fp8bs_quantize_weight_128x128_pow2).  No promotion step; experts averaging >= 256 rows run on CTA
 * pairs with 2-CTA block-scaled MMAs. */
FP8BS_API fp8bs_status fp8bs_grouped_gemm_mx(int32_t G, int64_t total_M, int64_t N, int64_t K, const int64_t* offsets,
                                   const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                   const uint8_t* B, const float* sB,
                                   void* D, fp8bs_dtype ddt, int64_t ldd,
                                   void* workspace, size_t workspace_bytes, fp8bs_stream_t stream);
FP8BS_API size_t fp8bs_grouped_gemm_workspace_size(int32_t G, int64_t total_M, int64_t N, int64_t K);

/* ---- grouped_gemm_scatter: the MoE expert Fprop with the combine's send fused into its epilogue ----
 * (NEXT-3; "combine components ... retained in BF16").  Computes exactly fp8bs_grouped_gemm's
 * BF16 output (same arguments, validation, workspace and result bits), but row r of it is written to
 *   dst_base[dst_rank[r]] + dst_row[r] * ldd   (BF16 elements, row of N values)
 * instead of D: dst_base is a DEVICE array of destination base pointers (e.g. every rank's symmetric-
 * memory combine buffer, written over NVLink by the epilogue's stores), dst_rank DEVICE int32 [total_M]
 * indexes it, dst_row DEVICE int64 [total_M] is the row there.  Destinations must be 16-byte aligned,
 * ldd*2 a multiple of 16, N a multiple of 8; rows must not overlap (undefined otherwise).  The stores
 * are complete and visible to the peers when the kernel completes (order them with the peers before
 * reading, e.g. a symmetric-memory barrier).  NULL table / rank / row: FP8BS_ERR_INVALID_ARG.
 * Streamed operands (overlap with fp8bs_dispatch_fp8_stream): ready != NULL is a DEVICE uint32 array
 * [ready_chunks]; the rows (and scales) of local expert group e are read only once
 * ready[e * ready_chunks / G] >= ready_target (wrap-safe compare, acquire at system scope), so a
 * dispatch still writing A / sA from other GPUs can run concurrently.  max_sms > 0 caps the GEMM's
 * persistent grid at that many SMs (required with ready: the SMs left run the dispatch it waits for,
 * otherwise the two could deadlock); ready_chunks >= 1.  ready == NULL, max_sms == 0: the plain
 * grouped Fprop with the scatter epilogue. */
FP8BS_API fp8bs_status fp8bs_grouped_gemm_scatter(int32_t G, int64_t total_M, int64_t N, int64_t K, const int64_t* offsets,
                                        const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                        const uint8_t* B, const float* sB,
                                        void* const* dst_base, const int32_t* dst_rank, const int64_t* dst_row,
                                        int64_t ldd, const uint32_t* ready, uint32_t ready_target, int32_t ready_chunks,
                                        int32_t max_sms, void* workspace, size_t workspace_bytes, fp8bs_stream_t stream);

/* ---- grouped_gemm_dgrad: MoE expert Dgrad (NEXT-3; the backward of the grouped Fprop above) ----
 * dX rows of expert e = dY rows of e (1x128 along the expert's output channels) x W_e:
 * offsets, A = dYq [total_M, K] (K = the experts' output width, the contraction), sA [K/128, ldsA],
 * D [total_M, N] (N = the experts' input width) as in fp8bs_grouped_gemm;
 * B   : [G, N, K] uint8, contiguous: per expert the transposed weight codes WqT_e [in, out] (the qT
 *       output of fp8bs_quantize_weight_128x128 on W_e [out, in]);
 * sB  : [G, K/128, ceil(N/128)] FP32, contiguous: per expert the SAME sW_e array the weight quantizer
 *       wrote ([out-block][in-block]), i.e. sB(e, kb, j) = sB[(e*(K/128) + kb)*ceil(N/128) + j/128].
 * Same sizes, alignment and workspace rules as fp8bs_grouped_gemm. */
FP8BS_API fp8bs_status fp8bs_grouped_gemm_dgrad(int32_t G, int64_t total_M, int64_t N, int64_t K, const int64_t* offsets,
                                      const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                      const uint8_t* B, const float* sB,
                                      void* D, fp8bs_dtype ddt, int64_t ldd,
                                      void* workspace, size_t workspace_bytes, fp8bs_stream_t stream);

/* ---- Expert-parallel exchange over NVLink (NEXT-3; §3.3.4) ---------------------------
 * "we quantize the activation before MoE up-projections into FP8 and then apply dispatch components
 * ... the combine components ... retained in BF16".  The expert GEMM's rows live on the
 * rank that owns the expert; these calls move them there and back with the kernels WRITING straight
 * into the destination GPU's memory over NVLink / NVSwitch (one warp per row, 16-byte stores).
 * recv_* are DEVICE arrays indexed by rank of pointers into each rank's receive buffer, mapped into the
 * calling process (peer pointers: torch symmetric memory, CUDA IPC; the caller's own entry may point to
 * local memory).  The calls only enqueue on `stream`: the caller orders them across GPUs (a barrier
 * after the senders' kernels, before the receiver reads).  Rows with dst_rank < 0 are not sent.
 *
 * dispatch_fp8: token slot i (token i / top_k, its (i % top_k)-th expert; n_slots = tokens * top_k)
 *   -> rank dst_rank[i], receive row dst_row[i]: the token's K codes xq [tokens, ldxq] to recv_q[r] +
 *   row * ld_recv_q, and its K/128 scales xs [K/128, ldxs] (the 1x128 quantizer's layout) to
 *   recv_s[r] + row * (K/128) (row-major: one contiguous run per row over the link).  K % 128 == 0.
 * scales_rows_to_blocks: the received row-major [R][KB] scales -> the GEMM's [KB][ldd >= R].
 * combine_push_bf16: expert output row i (BF16 y [R, ldy]) -> rank dst_rank[i]'s combine buffer row
 *   dst_slot[i] (= token * top_k + k there), recv_y[r] + dst_slot[i] * ld_recv_y.  N % 8 == 0.
 * combine_reduce_bf16: out[t] = BF16_RNE(sum_k gates[t][k] buf[t * top_k + k]) with the sum an FP32
 *   fused multiply-add chain in k order from 0 (reading R28); buf, out BF16, gates FP32 [T, top_k]. */
FP8BS_API fp8bs_status fp8bs_dispatch_fp8(int64_t n_slots, int32_t top_k, int64_t K, const uint8_t* xq, int64_t ldxq,
                                const float* xs, int64_t ldxs, const int32_t* dst_rank, const int64_t* dst_row,
                                uint8_t* const* recv_q, int64_t ld_recv_q, float* const* recv_s, fp8bs_stream_t stream);
/* dispatch_fp8_stream: the dispatch of fp8bs_dispatch_fp8 restructured so the receivers' grouped GEMM
 * can run concurrently (fp8bs_grouped_gemm_scatter with ready flags).  The sender's slots come as a
 * DEVICE send list sorted by (chunk, destination rank, destination row): entry j sends local token
 * send_tok[j] (its K codes of xq and its K/128 scales xs[kb * ldxs + token]) to rank send_rank[j], row
 * send_row[j]; chunk_off DEVICE int64 [chunks + 1] delimits the chunks in the list (chunk c of a receiver
 * = the rows of its local groups e with e * chunks / G == c).  Codes go to recv_q[rank] + row * ld_recv_q;
 * scales go straight into the receiver's GEMM layout recv_s[rank][kb * ld_recv_s + row] (no
 * fp8bs_scales_rows_to_blocks).  When every CTA of this call has finished chunk c (counted in
 * local_done[c], DEVICE uint32 [chunks] scratch of this rank, zeroed on `stream` by the call), one
 * release-add (system scope) increments flags[o][c] on every rank o (flags: DEVICE array of world
 * pointers to uint32 [chunks] in each rank's memory).  The flags are monotonic: zero them once, then call
 * with epoch = 1, 2, ... (one per forward, every rank); a receiver's chunk c is complete when its
 * flags[c] reaches world * epoch.  ctas CTAs of 128 threads, one per SM (114 KB of shared memory each
 * for the bulk-copy rings; a plain launch meant to run concurrently with the GEMM on another stream). */
FP8BS_API fp8bs_status fp8bs_dispatch_fp8_stream(int32_t chunks, const int64_t* chunk_off, const int64_t* send_tok,
                                       const int32_t* send_rank, const int64_t* send_row, int64_t K,
                                       const uint8_t* xq, int64_t ldxq, const float* xs, int64_t ldxs,
                                       uint8_t* const* recv_q, int64_t ld_recv_q, float* const* recv_s, int64_t ld_recv_s,
                                       uint32_t* local_done, uint32_t* const* flags, int32_t world, uint32_t epoch,
                                       int32_t ctas, fp8bs_stream_t stream);
/* send_rows / expand_rows: the token-once dispatch.  A token routed to several experts on one rank
 * crosses the link once (top-8 over 4 ranks: ~3.6 distinct ranks per token, 45% of the per-slot rows).
 * send_rows: entry i sends local token tok[i] (DEVICE int64 [n]) — its K codes of xq and K/128 scales
 *   xs[kb * ldxs + token] — to rank dst_rank[i], row dst_row[i] of that rank's TOKEN buffer (codes at
 *   recv_q[r] + row * ld_recv_q, scales row-major at recv_s[r] + row * (K/128)); dst_rank < 0: skipped.
 * expand_rows (local): expert row i of A [R, lda] <- token-buffer row idx[i] (DEVICE int64 [R]) of
 *   tq [*, ld_tq] (codes) and the scales of that token at ts[t * ts_row_stride + kb * ts_kb_stride]
 *   (row-major token buffer: (K/128, 1); the 1x128 quantizer's own [K/128][lds] layout: (1, lds)),
 *   written transposed into the GEMM's layout sA[kb * ldsA + i] (ldsA >= R).  Both K % 128 == 0,
 *   16-byte aligned code rows. */
FP8BS_API fp8bs_status fp8bs_send_rows(int64_t n, const int64_t* tok, int64_t K, const uint8_t* xq, int64_t ldxq, const float* xs,
                             int64_t ldxs, const int32_t* dst_rank, const int64_t* dst_row, uint8_t* const* recv_q,
                             int64_t ld_recv_q, float* const* recv_s, fp8bs_stream_t stream);
FP8BS_API fp8bs_status fp8bs_expand_rows(int64_t R, const int64_t* idx, int64_t K, const uint8_t* tq, int64_t ld_tq, const float* ts,
                               int64_t ts_row_stride, int64_t ts_kb_stride, uint8_t* A, int64_t lda, float* sA, int64_t ldsA,
                               fp8bs_stream_t stream);
FP8BS_API fp8bs_status fp8bs_scales_rows_to_blocks(int64_t R, int64_t KB, const float* src, float* dst, int64_t ldd,
                                         fp8bs_stream_t stream);
FP8BS_API fp8bs_status fp8bs_combine_push_bf16(int64_t R, int64_t N, const void* y, int64_t ldy, const int32_t* dst_rank,
                                     const int64_t* dst_slot, void* const* recv_y, int64_t ld_recv_y,
                                     fp8bs_stream_t stream);
FP8BS_API fp8bs_status fp8bs_combine_reduce_bf16(int64_t T, int32_t top_k, int64_t N, const void* buf, int64_t ldb,
                                       const float* gates, void* out, int64_t ldo, fp8bs_stream_t stream);

/* ---- gemm_swiglu: the up-projection with its SwiGLU FP8 epilogue (NEXT-2) ---------------------
 * "we cache the inputs of the SwiGLU operator and recompute its output in the backward pass.
 * These activations are also stored in FP8 with our fine-grained quantization method"; and every
 * Fprop input is FP8 (Fig. fp8_framework), so the down-projection consumes the SwiGLU
 * output quantized 1x128.  One FPROP GEMM (operands, layouts, alignment and errors as fp8bs_gemm
 * FPROP) whose epilogue, instead of writing H = A x B^T, writes from H's FP32 accumulators:
 *   y  [M, I] E4M3 codes (qy, ldqy >= I, 16-byte aligned rows) and sy [I/128, ldsy >= M] FP32: the
 *      1x128 quantization (the fp8bs_quantize_act_1x128 contract) of y = swiglu32(gate, up);
 *   qh [M, N] codes + sh [N/128, ldsh >= M] (optional, both NULL to skip): H itself quantized 1x128,
 *      the FP8 cache of the SwiGLU inputs.
 * N = 2I, a multiple of 256: B's rows come in (gate, up) blocks of 128 — output channels
 * [128 j, 128 j + 128) take gate = H columns [256 j, 256 j + 128) and up = [256 j + 128, 256 j + 256).
 * swiglu32(g, u) = RN(RN(g / RN(1 + exp32(-g))) * u) in binary32 with exp32 the fixed Cody-Waite /
 * degree-7 sequence of DESIGN.md reading R27 (so the codes are reproducible bit for bit).  No BF16
 * (or FP32) H ever reaches memory. */
FP8BS_API fp8bs_status fp8bs_gemm_swiglu(int64_t M, int64_t N, int64_t K,
                               const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                               const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                               uint8_t* qy, int64_t ldqy, float* sy, int64_t ldsy,
                               uint8_t* qh, int64_t ldqh, float* sh, int64_t ldsh, fp8bs_stream_t stream);
/* The same epilogue on the grouped (MoE) expert up-projection: fp8bs_grouped_gemm's arguments, layouts,
 * workspace and validation, with the outputs of fp8bs_gemm_swiglu over the total_M expert rows. */
FP8BS_API fp8bs_status fp8bs_grouped_gemm_swiglu(int32_t G, int64_t total_M, int64_t N, int64_t K, const int64_t* offsets,
                                       const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                       const uint8_t* B, const float* sB,
                                       uint8_t* qy, int64_t ldqy, float* sy, int64_t ldsy,
                                       uint8_t* qh, int64_t ldqh, float* sh, int64_t ldsh,
                                       void* workspace, size_t workspace_bytes, fp8bs_stream_t stream);

/* ---- grouped_gemm_dgrad_mx: the MoE expert Dgrad on UE8M0 block scaling (NEXT-1) ----------------
 * fp8bs_grouped_gemm_dgrad's arguments, layouts and workspace (as fp8bs_grouped_gemm_mx), with
 * fp8bs_gemm_mx's precondition: every sA and sB value an exact power of two in [2^-127, 2^127]. */
FP8BS_API fp8bs_status fp8bs_grouped_gemm_dgrad_mx(int32_t G, int64_t total_M, int64_t N, int64_t K, const int64_t* offsets,
                                         const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                         const uint8_t* B, const float* sB,
                                         void* D, fp8bs_dtype ddt, int64_t ldd,
                                         void* workspace, size_t workspace_bytes, fp8bs_stream_t stream);

/* ---- Grouped MoE expert Wgrad (NEXT-3) ------------------------------------------
 * dW_e [N, K] = sum over expert e's tokens t of dY[t, :]^T X[t, :]   (P:476-481 applied per expert;
 * Wgrad operands in 128x1 tiles along the tokens).  The contraction is each
 * expert's own token segment, and its 128x1 groups restart at the expert's first token: a group never
 * straddles two experts (reading R25).
 *
 * Expert-aligned token layout ("padded tokens"): expert e's M_e = offsets[e+1] - offsets[e] tokens
 * occupy columns [P_e, P_e + M_e) of the transposed operands, P_e = sum_{f<e} roundup(M_f, 128), and
 * columns [P_e + M_e, P_{e+1}) hold code 0 (which contributes exactly 0).  Mp = P_G.  Group g of the
 * padded layout is scale row g; every group starts at a multiple of 128, so the Wgrad GEMM of one
 * expert is a dense WGRAD over K_e = roundup(M_e, 128) columns at an aligned offset.
 *
 * offsets are HOST int64 [G+1] (non-decreasing, offsets[0] = 0): the expert counts are known on the
 * host when the dispatch is planned (no device sync).  fp8bs_grouped_gemm_wgrad is ONE persistent
 * launch over every expert's (m, n) tiles, each contracting over its own expert's token blocks; the
 * expert blocks travel in the kernel's parameters (G <= 1024).  Every argument is validated before
 * the launch.  Errors as the dense calls; FP8BS_ERR_INVALID_ARG on bad offsets. */

/* Mp for the given host offsets (0 if offsets are invalid). */
FP8BS_API int64_t fp8bs_padded_tokens(int32_t G, const int64_t* offsets);

/* x [offsets[G], C] rows grouped by expert (ldx >= C) -> qT [C, ldq >= Mp] codes in the padded layout
 * (padding columns written 0), sT [Mp/128, lds >= C] FP32: the 128x1 quantization of each expert's
 * segment (fp8bs_quantize_act_128x1's contract per segment). */
FP8BS_API fp8bs_status fp8bs_quantize_act_128x1_grouped(const void* x, fp8bs_dtype xdt, int32_t G,
                                              const int64_t* offsets, int64_t C, int64_t ldx,
                                              uint8_t* qT, int64_t ldq, float* sT, int64_t lds,
                                              fp8bs_stream_t stream);

/* A = dYqT [N, lda >= Mp], sA [Mp/128, ldsA >= N]; B = XqT [K, ldb >= Mp], sB [Mp/128, ldsB >= K], both in
 * the padded layout.  D [G, N, K] FP32, expert e at D + e*N*ldd (ldd >= K):  D_e (+)= the WGRAD of
 * expert e (fp8bs_gemm(FP8BS_WGRAD, N, K, roundup(M_e,128), ...) on its columns).  An expert with no
 * tokens gets D_e = 0 (accumulate = 0) or keeps D_e (accumulate = 1). */
FP8BS_API fp8bs_status fp8bs_grouped_gemm_wgrad(int32_t G, const int64_t* offsets, int64_t N, int64_t K,
                                      const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                      const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                                      float* D, int64_t ldd, int accumulate, fp8bs_stream_t stream);

/* ---- grouped_gemm_wgrad_mx: the grouped expert Wgrad on UE8M0 block scaling (NEXT-1) --
 * Identical arguments, layouts, validation and result definition as fp8bs_grouped_gemm_wgrad, with the
 * fp8bs_gemm_mx precondition: every sA and sB value is an exact power of two in [2^-127, 2^127] (e.g.
 * the pow2 128x1 quantization of each expert's tokens), applied inside tcgen05.mma.kind::mxf8f6f4 with
 * no promotion step.  One persistent launch over every expert's (m, n) tiles (CTA pairs along m sharing
 * the B tile by multicast); an expert without tokens gets D_e = 0 (accumulate: D_e unchanged). */
FP8BS_API fp8bs_status fp8bs_grouped_gemm_wgrad_mx(int32_t G, const int64_t* offsets, int64_t N, int64_t K,
                                         const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                         const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                                         float* D, int64_t ldd, int accumulate, fp8bs_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* FP8BS_H */
