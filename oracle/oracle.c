/* oracle/oracle.c — plain, slow, obviously-correct CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py.  Never part of the product path.
 * Shares no code with paper_2412_19437_b200/csrc (different language, no common
 * header, table or generator).
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -fPIC -shared
 * (IEEE binary32/binary64 arithmetic, no FMA contraction, no flush-to-zero).
 *
 * Every function follows the paper's definition in the paper's order:
 *   - fine-grained groupings 1x128 (activations, per token per 128 channels) and
 *     128x128 (weights), PAPER.md P:503-510;
 *   - online quantization: max-abs of the group -> scaling factor -> cast to FP8,
 *     P:541-544; the scale maps amax onto the maximum representable E4M3 value
 *     ("scaling the maximum absolute value ... to the maximum representable
 *     value of FP8"), i.e. s = amax / 448 (readings R1, R2);
 *   - E4M3 on all tensors, P:536-539;
 *   - GEMM with per-group scales along K, partial sums over each N_C = 128 interval
 *     multiplied by the scaling factors and added into a high-precision accumulator,
 *     P:512-514, P:529-531 (here FP64);
 *   - 128x1 tiles for the Wgrad operands, P:558, P:672-673 (reading R10).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- E4M3 ---- */
/* Bit definition: sign(1) | exponent(4, bias 7) | mantissa(3).
 * exponent 0: subnormal, value = m * 2^-9.  exponent 15 with mantissa 7: NaN (no Inf).
 * Otherwise value = (1 + m/8) * 2^(e-7).  Max finite = 1.75 * 2^8 = 448. */
double oracle_e4m3_decode(uint8_t code) {
    int sign = code >> 7;
    int e = (code >> 3) & 0xF;
    int m = code & 0x7;
    double v;
    if (e == 0xF && m == 0x7) return NAN;
    if (e == 0) v = ldexp((double)m, -9);
    else v = ldexp(1.0 + m / 8.0, e - 7);
    return sign ? -v : v;
}

/* Round-to-nearest-even onto the E4M3 grid, saturating to +-448 (R3):
 * the value is written as n * quantum with quantum the grid spacing of |y|'s binade
 * (2^-9 below the smallest normal 2^-6), n rounded to the nearest integer with ties
 * to even (an even n is an even mantissa), and the result re-encoded from the bit
 * definition above.  NaN -> canonical 0x7F (R6). */
uint8_t oracle_e4m3_encode(float y) {
    if (isnan(y)) return 0x7F;
    uint8_t sign = signbit(y) ? 0x80 : 0x00;
    double a = fabs((double)y);                   /* exact */
    if (a >= 448.0) return sign | 0x7E;           /* saturate (includes +-Inf) */
    double quantum;
    if (a < ldexp(1.0, -6)) {
        quantum = ldexp(1.0, -9);                 /* subnormal grid */
    } else {
        int ex;
        frexp(a, &ex);                            /* a = f * 2^ex, f in [0.5, 1) */
        quantum = ldexp(1.0, (ex - 1) - 3);       /* 3 mantissa bits in binade 2^(ex-1) */
    }
    double n = a / quantum;                       /* exact: power-of-two division */
    double r = nearbyint(n);                      /* default mode = round half to even */
    double v = r * quantum;                       /* exact */
    if (v == 0.0) return sign;
    if (v < ldexp(1.0, -6)) return sign | (uint8_t)r;   /* subnormal code = multiple of 2^-9 */
    int ex;
    double f = frexp(v, &ex);                     /* v = f * 2^ex, f in [0.5,1) */
    int e = (ex - 1) + 7;                         /* biased exponent */
    int m = (int)((2.0 * f - 1.0) * 8.0);         /* exact: v is on the grid */
    if (e > 15 || (e == 15 && m == 7)) return sign | 0x7E;  /* cannot happen below 448 */
    return sign | (uint8_t)((e << 3) | m);
}

void oracle_e4m3_encode_array(const float* y, int64_t n, uint8_t* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_e4m3_encode(y[i]);
}

float oracle_bf16_to_float(uint16_t bits) {
    uint32_t u = ((uint32_t)bits) << 16;         /* BF16 is the top half of binary32 */
    float f;
    memcpy(&f, &u, sizeof f);
    return f;
}

static float load_elem(const void* x, int dt, int64_t idx) {
    if (dt == ORACLE_BF16) return oracle_bf16_to_float(((const uint16_t*)x)[idx]);
    return ((const float*)x)[idx];
}

/* scale of a group from its max-abs: s = amax / 448 in binary32 (IEEE division);
 * an all-zero group (or one whose quotient underflows to 0) takes s = 1
 * (R4). */
static float group_scale(float amax) {
    float s = amax / 448.0f;
    if (s == 0.0f) s = 1.0f;
    return s;
}

/* power-of-two scale ("integral power of 2"; SPEC S:374 / S:417 round UP): the
 * smallest s = 2^e with 448 * s >= amax, computed on exact values (448 * 2^e is exact in double);
 * e >= -127, the smallest UE8M0 value, so every pow2 scale is representable by the tensor core's
 * block-scale format (reading R26; an amax below 448 * 2^-127 then still fits without saturating);
 * 1 for an all-zero group; a non-finite amax passes through (as amax / 448 does in group_scale). */
static float group_scale_pow2(float amax) {
    if (amax == 0.0f) return 1.0f;
    if (!isfinite(amax)) return amax;
    int e = -160;
    while (ldexp(448.0, e) < (double)amax) ++e;    /* plain linear search from below */
    if (e < -127) e = -127;
    return ldexpf(1.0f, e);
}

/* ------------------------------------------------------ quantizers ---- */
/* 1x128 tiles: per token m, per 128 channels kb ("per token per 128 channels"). */
static void quantize_1x128(const void* x, int xdt, int64_t M, int64_t K, int64_t ldx,
                           uint8_t* q, int64_t ldq, float* s, int64_t lds, float (*scale)(float));
void oracle_quantize_act_1x128(const void* x, int xdt, int64_t M, int64_t K, int64_t ldx,
                               uint8_t* q, int64_t ldq, float* s, int64_t lds) {
    quantize_1x128(x, xdt, M, K, ldx, q, ldq, s, lds, group_scale);
}
/* the same tiles with power-of-two scales */
void oracle_quantize_act_1x128_pow2(const void* x, int xdt, int64_t M, int64_t K, int64_t ldx,
                                    uint8_t* q, int64_t ldq, float* s, int64_t lds) {
    quantize_1x128(x, xdt, M, K, ldx, q, ldq, s, lds, group_scale_pow2);
}
static void quantize_1x128(const void* x, int xdt, int64_t M, int64_t K, int64_t ldx,
                           uint8_t* q, int64_t ldq, float* s, int64_t lds, float (*scale)(float)) {
    int64_t KB = (K + 127) / 128;
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t kb = 0; kb < KB; ++kb) {
            int64_t k0 = kb * 128, k1 = k0 + 128 < K ? k0 + 128 : K;   /* short last group */
            float amax = 0.0f;
            for (int64_t k = k0; k < k1; ++k) amax = fmaxf(amax, fabsf(load_elem(x, xdt, m * ldx + k)));
            float sc = scale(amax);
            s[kb * lds + m] = sc;
            for (int64_t k = k0; k < k1; ++k) q[m * ldq + k] = oracle_e4m3_encode(load_elem(x, xdt, m * ldx + k) / sc);
        }
    }
}

/* 128x1 tiles: per channel c, per 128 tokens mb; stored transposed (qT[c][m]) so the
 * Wgrad contraction (tokens) is contiguous. */
static void quantize_128x1(const void* x, int xdt, int64_t M, int64_t C, int64_t ldx,
                           uint8_t* qT, int64_t ldq, float* sT, int64_t lds, float (*scale)(float));
void oracle_quantize_act_128x1(const void* x, int xdt, int64_t M, int64_t C, int64_t ldx,
                               uint8_t* qT, int64_t ldq, float* sT, int64_t lds) {
    quantize_128x1(x, xdt, M, C, ldx, qT, ldq, sT, lds, group_scale);
}
/* 128x1 with power-of-two scales */
void oracle_quantize_act_128x1_pow2(const void* x, int xdt, int64_t M, int64_t C, int64_t ldx,
                                    uint8_t* qT, int64_t ldq, float* sT, int64_t lds) {
    quantize_128x1(x, xdt, M, C, ldx, qT, ldq, sT, lds, group_scale_pow2);
}
static void quantize_128x1(const void* x, int xdt, int64_t M, int64_t C, int64_t ldx,
                           uint8_t* qT, int64_t ldq, float* sT, int64_t lds, float (*scale)(float)) {
    int64_t MB = (M + 127) / 128;
    for (int64_t c = 0; c < C; ++c) {
        for (int64_t mb = 0; mb < MB; ++mb) {
            int64_t m0 = mb * 128, m1 = m0 + 128 < M ? m0 + 128 : M;
            float amax = 0.0f;
            for (int64_t m = m0; m < m1; ++m) amax = fmaxf(amax, fabsf(load_elem(x, xdt, m * ldx + c)));
            float sc = scale(amax);
            sT[mb * lds + c] = sc;
            for (int64_t m = m0; m < m1; ++m) qT[c * ldq + m] = oracle_e4m3_encode(load_elem(x, xdt, m * ldx + c) / sc);
        }
    }
}

/* 128x128 blocks: per 128 output channels nb, per 128 input channels kb. */
static void quantize_weight(const void* w, int wdt, int64_t N, int64_t K, int64_t ldw,
                            uint8_t* q, int64_t ldq, float* s, int64_t ldsw,
                            uint8_t* qT, int64_t ldqT, float (*scale)(float));
void oracle_quantize_weight_128x128(const void* w, int wdt, int64_t N, int64_t K, int64_t ldw,
                                    uint8_t* q, int64_t ldq, float* s, int64_t ldsw,
                                    uint8_t* qT, int64_t ldqT) {
    quantize_weight(w, wdt, N, K, ldw, q, ldq, s, ldsw, qT, ldqT, group_scale);
}
/* 128x128 with power-of-two scales (the P:558 / P:565 option applied to the weights) */
void oracle_quantize_weight_128x128_pow2(const void* w, int wdt, int64_t N, int64_t K, int64_t ldw,
                                         uint8_t* q, int64_t ldq, float* s, int64_t ldsw,
                                         uint8_t* qT, int64_t ldqT) {
    quantize_weight(w, wdt, N, K, ldw, q, ldq, s, ldsw, qT, ldqT, group_scale_pow2);
}
static void quantize_weight(const void* w, int wdt, int64_t N, int64_t K, int64_t ldw,
                            uint8_t* q, int64_t ldq, float* s, int64_t ldsw,
                            uint8_t* qT, int64_t ldqT, float (*scale)(float)) {
    int64_t NB = (N + 127) / 128, KB = (K + 127) / 128;
    for (int64_t nb = 0; nb < NB; ++nb) {
        int64_t n0 = nb * 128, n1 = n0 + 128 < N ? n0 + 128 : N;
        for (int64_t kb = 0; kb < KB; ++kb) {
            int64_t k0 = kb * 128, k1 = k0 + 128 < K ? k0 + 128 : K;
            float amax = 0.0f;
            for (int64_t n = n0; n < n1; ++n)
                for (int64_t k = k0; k < k1; ++k) amax = fmaxf(amax, fabsf(load_elem(w, wdt, n * ldw + k)));
            float sc = scale(amax);
            s[nb * ldsw + kb] = sc;
            for (int64_t n = n0; n < n1; ++n)
                for (int64_t k = k0; k < k1; ++k) {
                    uint8_t c = oracle_e4m3_encode(load_elem(w, wdt, n * ldw + k) / sc);
                    q[n * ldq + k] = c;
                    if (qT) qT[k * ldqT + n] = c;
                }
        }
    }
}

/* FP8 -> FP8 re-quantization of a cached activation (§3.5.2: the FP8 activations
 * of the forward pass "need to be read out, dequantized, transposed, re-quantized into 128x1
 * tiles").  Step 1, dequantize: xhat[m,k] = RN32(dec(q[m,k]) * s(k/128, m)), the product taken
 * exactly in FP64 (4 x 24 significant bits) and rounded once to FP32 (reading R19: the
 * dequantized tensor is FP32).  Step 2: the 128x1 quantization of xhat (the function above). */
void oracle_requantize_1x128_to_128x1(const uint8_t* q, int64_t ldq, const float* s, int64_t lds,
                                      int64_t M, int64_t K, uint8_t* qT, int64_t ldqT, float* sT, int64_t ldsT,
                                      int pow2) {
    float* xhat = (float*)malloc((size_t)(M > 0 ? M : 1) * (size_t)(K > 0 ? K : 1) * sizeof(float));
    if (!xhat) return;
    for (int64_t m = 0; m < M; ++m)
        for (int64_t k = 0; k < K; ++k)
            xhat[m * K + k] = (float)(oracle_e4m3_decode(q[m * ldq + k]) * (double)s[(k / 128) * lds + m]);
    quantize_128x1(xhat, 1, M, K, K, qT, ldqT, sT, ldsT, pow2 ? group_scale_pow2 : group_scale);
    free(xhat);
}

/* ------------------------------------------------------------ GEMM ---- */
static double g_dec[256];
static int g_dec_ready = 0;
static void dec_table_init(void) {
    if (g_dec_ready) return;
    for (int c = 0; c < 256; ++c) g_dec[c] = oracle_e4m3_decode((uint8_t)c);
    g_dec_ready = 1;
}

static double scale_b(int layout, const float* sB, int64_t ldsB, int64_t kb, int64_t j) {
    if (layout == ORACLE_FPROP) return sB[(j / 128) * ldsB + kb];
    if (layout == ORACLE_DGRAD) return sB[kb * ldsB + j / 128];
    return sB[kb * ldsB + j];                                  /* WGRAD: per row of B */
}

/* One output row.  For each N_C = 128 interval kb: the partial sum P_kb of exact
 * FP8 x FP8 products, multiplied by the two group scales and added into the FP64
 * accumulator.  Every product dec(a)*dec(b) is exact in binary64 and each
 * 128-term P_kb is exact too (products are multiples of 2^-18 below 2^18), so FP64
 * rounding enters only through the scale multiply and the kb sum. */
static void gemm_row(int layout, int64_t i, int64_t N, int64_t K,
                     const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                     const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB, double* out) {
    int64_t KB = K / 128;
    const uint8_t* a = A + i * lda;
    for (int64_t j = 0; j < N; ++j) {
        const uint8_t* b = B + j * ldb;
        double acc = 0.0;
        for (int64_t kb = 0; kb < KB; ++kb) {
            double p = 0.0;
            for (int64_t c = kb * 128; c < kb * 128 + 128; ++c) p += g_dec[a[c]] * g_dec[b[c]];
            double sa = sA[kb * ldsA + i];
            double sb = scale_b(layout, sB, ldsB, kb, j);
            acc += (sa * sb) * p;
        }
        out[j] = acc;
    }
}

void oracle_gemm(int layout, int64_t M, int64_t N, int64_t K,
                 const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                 const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                 const int64_t* rows, int64_t nrows, double* O, int threads) {
    dec_table_init();
    if (!rows) nrows = M;
#ifdef _OPENMP
    int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
#endif
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = rows ? rows[r] : r;
        gemm_row(layout, i, N, K, A, lda, sA, ldsA, B, ldb, sB, ldsB, O + r * N);
    }
    (void)threads;
}

void oracle_grouped_gemm(int32_t G, const int64_t* offsets, int64_t N, int64_t K,
                         const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                         const uint8_t* B, const float* sB,
                         const int64_t* rows, int64_t nrows, double* O, int threads) {
    dec_table_init();
    int64_t total = offsets[G];
    if (!rows) nrows = total;
    int64_t NB = (N + 127) / 128, KB = K / 128;
#ifdef _OPENMP
    int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
#endif
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = rows ? rows[r] : r;
        int32_t e = 0;                                  /* the expert segment holding row i */
        while (e < G && !(offsets[e] <= i && i < offsets[e + 1])) ++e;
        if (e == G) { for (int64_t j = 0; j < N; ++j) O[r * N + j] = NAN; continue; }
        gemm_row(ORACLE_FPROP, i, N, K, A, lda, sA, ldsA,
                 B + (int64_t)e * N * K, K, sB + (int64_t)e * NB * KB, KB, O + r * N);
    }
    (void)threads;
}

/* ------------------------------------------- limited accumulation (NEXT-4) ---- */
/* Emulation of the Hopper tensor-core accumulator the paper measured (context only,
 * DESIGN.md reading R24):
 *   "FP8 GEMM employs fixed-point accumulation, aligning the mantissa products by
 *    right-shifting based on the maximum exponent before addition. ... it only uses the
 *    highest 14 bits of each mantissa product after sign-fill right shifting, and
 *    truncates bits exceeding this range";
 *   "to achieve precise FP32 results from the accumulation of 32 FP8xFP8
 *    multiplications, at least 34-bit precision is required", i.e. one MMA step
 *    adds `chunk` products into the accumulator;
 *   promotion: "Once an interval of N_C is reached, these partial results will be copied
 *    to FP32 registers on CUDA Cores, where full-precision FP32 accumulation is
 *    performed" and the group scales are multiplied there.
 * One accumulation step over terms t_0 = acc, t_1..t_chunk = the chunk's exact products:
 *   E = max_i floor(log2|t_i|) (nonzero t_i);  q = 2^(E - bits + 1);
 *   each t_i -> floor(t_i / q) * q   (sign-fill right shift = floor, two's complement);
 *   acc = RN32(sum of the shifted terms)   (the sum itself is exact in binary64 here).
 * toward_zero = 1 replaces the floor by truncation toward zero (a sign-magnitude shift):
 * not the paper's words, kept to bracket its "nearly 2%" figure (R24).
 * nc = 0: no promotion, the limited accumulator runs over all of K and the scales of
 * block 0 are applied once at the end (tensor-wise scaling: pass one scale per row/col).
 * nc > 0 (a multiple of chunk dividing 128): the limited accumulator is
 * restarted every nc elements, multiplied by the group scales of its 128-block and added
 * into an FP64 accumulator (the oracle's promotion precision, see oracle_gemm). */
static double shift_floor(double t, double q, int toward_zero) {
    return (toward_zero ? trunc(t / q) : floor(t / q)) * q;
}

static double limited_step(double acc, const double* p, int n, int bits, int toward_zero) {
    int E = INT32_MIN;
    int e;
    if (acc != 0.0) { frexp(acc, &e); E = e - 1; }
    for (int i = 0; i < n; ++i)
        if (p[i] != 0.0) { frexp(p[i], &e); if (e - 1 > E) E = e - 1; }
    if (E == INT32_MIN) return 0.0;
    double q = ldexp(1.0, E - bits + 1);
    double sum = shift_floor(acc, q, toward_zero);
    for (int i = 0; i < n; ++i) sum += shift_floor(p[i], q, toward_zero);
    return (double)(float)sum;
}

void oracle_gemm_limited_accum(int64_t M, int64_t N, int64_t K,
                               const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                               const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                               int bits, int chunk, int nc, int toward_zero, double* O, int threads) {
    dec_table_init();
#ifdef _OPENMP
    int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
#endif
    for (int64_t i = 0; i < M; ++i) {
        double p[256];
        for (int64_t j = 0; j < N; ++j) {
            const uint8_t* a = A + i * lda;
            const uint8_t* b = B + j * ldb;
            double hi = 0.0, acc = 0.0;
            for (int64_t c0 = 0; c0 < K; c0 += chunk) {
                int n = (int)(K - c0 < chunk ? K - c0 : chunk);
                for (int t = 0; t < n; ++t) p[t] = g_dec[a[c0 + t]] * g_dec[b[c0 + t]];
                acc = limited_step(acc, p, n, bits, toward_zero);
                int64_t done = c0 + n;
                if (nc > 0 && (done % nc == 0 || done == K)) {
                    int64_t kb = (done - 1) / 128;
                    hi += ((double)sA[kb * ldsA + i] * (double)sB[kb * ldsB + j]) * acc;
                    acc = 0.0;
                }
            }
            if (nc == 0) hi = ((double)sA[i] * (double)sB[j]) * acc;
            O[i * N + j] = hi;
        }
    }
    (void)threads;
}

double oracle_rel_err_normwise(const double* D, const double* O, int64_t n) {
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double d = fabs(D[i] - O[i]);
        if (d > num || isnan(d)) num = isnan(d) ? INFINITY : (d > num ? d : num);
        if (fabs(O[i]) > den) den = fabs(O[i]);
    }
    if (den == 0.0) return num == 0.0 ? 0.0 : INFINITY;
    return num / den;
}

/* ------------------------------------------------- SwiGLU epilogue (NEXT-2) ---- */
/* exp(x) in binary32 by ONE fixed, branch-free sequence of IEEE round-to-nearest operations (reading
 * R27), so that a GPU epilogue evaluating the same sequence (fmaf = correctly rounded fused
 * multiply-add) reproduces it bit for bit:
 *   x is clamped to [-86, 86] (NaN becomes -86: callers carry NaN through their own operands);
 *   t = x log2(e) as an unevaluated pair th + tl (th = RN(x L2E), tl = the FMA residual of that
 *   product + x L2E_LO); k = RNE(th); f = RN((th - k) + tl) (th - k is exact);
 *   2^f by the degree-7 Taylor polynomial of exp(f ln 2) in Horner form (|f| <= 0.5: truncation
 *   < 6e-9 relative), then times 2^k by adding k to the exponent field (the result is normal for
 *   |x| <= 86).  Accuracy vs the C library's exp: <= 2 ulp (tests/test_oracle.py). */
static float bits_f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t f_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
float oracle_exp32(float x) {
    x = fminf(fmaxf(x, -86.0f), 86.0f);
    const float L2E = 1.44269502162933349609375f, L2E_LO = 1.925963033500011079013347625732421875e-08f;
    const float th = x * L2E;
    const float tl = fmaf(x, L2E_LO, fmaf(x, L2E, -th));
    const float k = rintf(th);
    const float f = (th - k) + tl;
    float p = 1.5252733804059840e-5f;                        /* ln2^7 / 7! */
    p = fmaf(p, f, 1.5403530393381608e-4f);                  /* ln2^6 / 6! */
    p = fmaf(p, f, 1.3333558146428443e-3f);                  /* ln2^5 / 5! */
    p = fmaf(p, f, 9.6181291076284772e-3f);                  /* ln2^4 / 4! */
    p = fmaf(p, f, 5.5504108664821580e-2f);                  /* ln2^3 / 3! */
    p = fmaf(p, f, 2.4022650695910071e-1f);                  /* ln2^2 / 2! */
    p = fmaf(p, f, 6.9314718055994531e-1f);                  /* ln2 */
    p = fmaf(p, f, 1.0f);
    return bits_f(f_bits(p) + ((uint32_t)(int32_t)k << 23));
}

/* 1/d for d in [1, 2^125) by a fixed sequence (reading R27): the bit-level first guess
 * 0x7EF311C3 - bits(d) and three Newton steps r += r (1 - d r), each residual by one FMA. */
float oracle_rcp32(float d) {
    float r = bits_f(0x7EF311C3u - f_bits(d));
    for (int i = 0; i < 3; ++i) r = fmaf(r, fmaf(-d, r, 1.0f), r);
    return r;
}

/* SwiGLU (SiLU-gated linear unit: silu(g) * u, silu(g) = g * sigmoid(g) = g / (1 + exp(-g))) of
 * one (gate, up) pair in binary32, in this order (reading R27):
 *   e = exp32(-g);  d = RN(1 + e);  s = RN(g * rcp32(d));  y = RN(s * u). */
float oracle_swiglu32(float g, float u) {
    const float d = 1.0f + oracle_exp32(-g);
    const float sg = g * oracle_rcp32(d);
    return sg * u;
}

/* The FP8 epilogue of an expert up-projection (NEXT-2; "we cache the inputs of the SwiGLU
 * operator ... stored in FP8 with our fine-grained quantization method", and every Fprop input is FP8,
 * Fig. fp8_framework P:453-460 — so the down-projection's input is the 1x128-quantized SwiGLU output).
 * H [M, 2I] (ld ldh) is the up-projection's binary32 output with gate and up interleaved per 128
 * channels: output block j (channels [128 j, 128 j + 128)) has gate = columns [256 j, 256 j + 128) and
 * up = columns [256 j + 128, 256 j + 256) (reading R27).  I % 128 == 0.
 *   y[m][128 j + c] = swiglu32(H[m][256 j + c], H[m][256 j + 128 + c]);
 *   (qy, sy) = 1x128 quantization of y (the same contract as oracle_quantize_act_1x128);
 *   (qh, sh) = 1x128 quantization of H itself — the FP8 cache of the SwiGLU inputs; skipped
 *   when qh == NULL. */
void oracle_swiglu_quant_1x128(const float* H, int64_t M, int64_t I, int64_t ldh,
                               uint8_t* qy, int64_t ldqy, float* sy, int64_t ldsy,
                               uint8_t* qh, int64_t ldqh, float* sh, int64_t ldsh) {
    float* y = (float*)malloc((size_t)(M > 0 ? M : 1) * (size_t)(I > 0 ? I : 1) * sizeof(float));
    for (int64_t m = 0; m < M; ++m)
        for (int64_t c = 0; c < I; ++c) {
            const int64_t j = c / 128, cc = c % 128;
            y[m * I + c] = oracle_swiglu32(H[m * ldh + 256 * j + cc], H[m * ldh + 256 * j + 128 + cc]);
        }
    quantize_1x128(y, 1 /* FP32 */, M, I, I, qy, ldqy, sy, ldsy, group_scale);
    if (qh) quantize_1x128(H, 1, M, 2 * I, ldh, qh, ldqh, sh, ldsh, group_scale);
    free(y);
}

/* ------------------------------------------------ MoE combine (NEXT-3) ---- */
/* binary32 -> BF16 bits, round to nearest even (NaN -> a quiet NaN of the same sign). */
uint16_t oracle_float_to_bf16(float f) {
    uint32_t u = f_bits(f);
    if (isnan(f)) return (uint16_t)((u >> 16) | 0x40);
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;                         /* ties to even on the 16 dropped bits */
    return (uint16_t)(u >> 16);
}

/* The BF16 combine of routed-expert outputs (h'_t = u_t + sum_i g_{i,t} FFN_i(u_t); P:565-567:
 * the combine runs in BF16): y holds, for token t, its top_k expert outputs at rows t * top_k + k
 * (BF16 [T * top_k, N]); g [T, top_k] FP32 gates.  out[t][n] = BF16_RNE(acc), acc = 0.0f and
 * acc = fmaf(g[t][k], y[t*top_k + k][n], acc) for k = 0 .. top_k - 1 (reading R28). */
void oracle_combine_bf16(int64_t T, int top_k, int64_t N, const uint16_t* y, const float* g, uint16_t* out) {
    for (int64_t t = 0; t < T; ++t)
        for (int64_t n = 0; n < N; ++n) {
            float acc = 0.0f;
            for (int k = 0; k < top_k; ++k)
                acc = fmaf(g[t * top_k + k], oracle_bf16_to_float(y[(t * top_k + k) * N + n]), acc);
            out[t * N + n] = oracle_float_to_bf16(acc);
        }
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
