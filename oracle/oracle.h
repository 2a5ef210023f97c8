/* oracle/oracle.h — CPU oracle for DeepSeek-V3 fine-grained FP8 quantization + block-scaled GEMM.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2412_19437_b200, include/fp8bs.h) never includes, links or calls it, and
 * this file shares no code, header, table or constant generator with csrc/.
 *
 * Host pointers only, no state.  Layouts mirror include/fp8bs.h so buffers
 * compare with memcmp:
 *   activations 1x128   q[m*ldq + k],  s[(k/128)*lds + m]
 *   activations 128x1   qT[c*ldq + m], sT[(m/128)*lds + c]
 *   weights 128x128     q[n*ldq + k],  s[(n/128)*ldsw + k/128], optional qT[k*ldqT + n]
 * Citations: PAPER.md P:503-510 (groupings), P:541-544 (online amax -> scale -> cast),
 * P:536-539 (E4M3 everywhere), P:512-514 + P:529-531 (per-group scales along K,
 * FP32-promoted partial sums every N_C = 128), P:477 + P:487 (BF16/FP32 outputs).
 */
#ifndef FP8_ORACLE_H
#define FP8_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_BF16 0
#define ORACLE_FP32 1

#define ORACLE_FPROP 0
#define ORACLE_DGRAD 1
#define ORACLE_WGRAD 2

/* E4M3 ("fn": bias 7, no Inf, NaN = S.1111.111, max 448) */
double  oracle_e4m3_decode(uint8_t code);          /* NaN for 0x7F / 0xFF */
uint8_t oracle_e4m3_encode(float y);               /* RNE, saturate-to-finite, NaN -> 0x7F */
void    oracle_e4m3_encode_array(const float* y, int64_t n, uint8_t* out);
float   oracle_bf16_to_float(uint16_t bits);

void oracle_quantize_act_1x128(const void* x, int xdt, int64_t M, int64_t K, int64_t ldx,
                               uint8_t* q, int64_t ldq, float* s, int64_t lds);
/* 1x128 with power-of-two scales: s = smallest 2^e with 448*2^e >= amax (e >= -127, R26; 1 if amax == 0) */
void oracle_quantize_act_1x128_pow2(const void* x, int xdt, int64_t M, int64_t K, int64_t ldx,
                                    uint8_t* q, int64_t ldq, float* s, int64_t lds);
void oracle_quantize_act_128x1(const void* x, int xdt, int64_t M, int64_t C, int64_t ldx,
                               uint8_t* qT, int64_t ldq, float* sT, int64_t lds);
void oracle_quantize_weight_128x128(const void* w, int wdt, int64_t N, int64_t K, int64_t ldw,
                                    uint8_t* q, int64_t ldq, float* s, int64_t ldsw,
                                    uint8_t* qT, int64_t ldqT);
/* power-of-two scale variants of the two above (same scale rule as oracle_quantize_act_1x128_pow2) */
void oracle_quantize_act_128x1_pow2(const void* x, int xdt, int64_t M, int64_t C, int64_t ldx,
                                    uint8_t* qT, int64_t ldq, float* sT, int64_t lds);
void oracle_quantize_weight_128x128_pow2(const void* w, int wdt, int64_t N, int64_t K, int64_t ldw,
                                         uint8_t* q, int64_t ldq, float* s, int64_t ldsw,
                                         uint8_t* qT, int64_t ldqT);

/* FP8 1x128 (q[m*ldq+k], s[(k/128)*lds+m]) -> dequantize to FP32 -> 128x1 (qT[k*ldqT+m],
 * sT[(m/128)*ldsT+k]).  P:558. */
void oracle_requantize_1x128_to_128x1(const uint8_t* q, int64_t ldq, const float* s, int64_t lds,
                                      int64_t M, int64_t K, uint8_t* qT, int64_t ldqT, float* sT, int64_t ldsT,
                                      int pow2);   /* pow2 != 0: power-of-two output scales */

/* O[r*N + j] = sum_kb sA(kb,i)*sB(kb,j) * sum_{c in kb} dec(A[i,c])*dec(B[j,c]),  FP64.
 * i = rows[r] (rows == NULL -> i = r, nrows = M).  Contraction K % 128 == 0.
 * sA(kb,i) = sA[kb*ldsA + i]
 * sB(kb,j) = FPROP: sB[(j/128)*ldsB + kb]; DGRAD: sB[kb*ldsB + j/128]; WGRAD: sB[kb*ldsB + j]
 * threads <= 0 -> all available cores. */
void oracle_gemm(int layout, int64_t M, int64_t N, int64_t K,
                 const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                 const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                 const int64_t* rows, int64_t nrows, double* O, int threads);

/* Grouped FPROP over expert segments [offsets[e], offsets[e+1]) of A's rows.
 * B is [G][N][K] (ld K), sB is [G][ceil(N/128)][K/128].  Rows as in oracle_gemm. */
void oracle_grouped_gemm(int32_t G, const int64_t* offsets, int64_t N, int64_t K,
                         const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                         const uint8_t* B, const float* sB,
                         const int64_t* rows, int64_t nrows, double* O, int threads);

/* SwiGLU FP8 epilogue of an up-projection (NEXT-2; R27).  exp32 / rcp32: the fixed
 * binary32 sequences; swiglu32: RN(RN(g * rcp32(RN(1 + exp32(-g)))) * u).  H [M, 2I] FP32 with gate/up interleaved
 * per 128 channels -> y [M, I] quantized 1x128 (qy, sy[(c/128)*ldsy + m]); qh/sh (optional, NULL to
 * skip): H itself quantized 1x128 (the FP8 cache of the SwiGLU inputs). */
float oracle_exp32(float x);
float oracle_rcp32(float d);
float oracle_swiglu32(float g, float u);
void oracle_swiglu_quant_1x128(const float* H, int64_t M, int64_t I, int64_t ldh,
                               uint8_t* qy, int64_t ldqy, float* sy, int64_t ldsy,
                               uint8_t* qh, int64_t ldqh, float* sh, int64_t ldsh);

/* MoE combine (NEXT-3; R28): out[t] = BF16_RNE(sum_k g[t][k] y[t*top_k+k])
 * accumulated with fmaf in k order from 0.0f; y, out BF16 bits. */
uint16_t oracle_float_to_bf16(float f);
void oracle_combine_bf16(int64_t T, int top_k, int64_t N, const uint16_t* y, const float* g, uint16_t* out);

/* Hopper limited-precision accumulation emulation (context only; R24).
 * A [M,K] codes (ld lda), B [N,K] codes (ld ldb); per-row scales with the WGRAD layout:
 * sA(kb,i) = sA[kb*ldsA + i], sB(kb,j) = sB[kb*ldsB + j].  bits = retained bits (14 on
 * H800), chunk = products per accumulation step (32 = one MMA K-step, <= 256),
 * nc = promotion interval (0 = none: scales of block 0 applied once at the end);
 * toward_zero = 0: sign-fill shift (floor), 1: truncation toward zero.
 * O [M,N] FP64. */
void oracle_gemm_limited_accum(int64_t M, int64_t N, int64_t K,
                               const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                               const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                               int bits, int chunk, int nc, int toward_zero, double* O, int threads);

/* max_ij |D - O| / max_ij |O|  (reading R14) */
double oracle_rel_err_normwise(const double* D, const double* O, int64_t n);

int oracle_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
