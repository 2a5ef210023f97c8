// api.cu — C-ABI entry points of libfp8bs.so (include/fp8bs.h): argument validation, device
// check, then kernel launch on the caller's stream.  Validation runs before any CUDA call so a
// failing call has no side effects (and the validation paths are testable without a GPU).
#include <cstdlib>
#include <vector>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/fp8bs.h"
#include "internal.h"

namespace fp8bs {

static thread_local char g_detail[512] = "";

static fp8bs_status fail(fp8bs_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_detail, sizeof g_detail, fmt, ap);
    va_end(ap);
    return st;
}
static fp8bs_status ok() { g_detail[0] = 0; return FP8BS_OK; }

int num_sms() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (cache[dev] == 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cache[dev] = n;
    }
    return cache[dev];
}

static fp8bs_status check_device() {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) { cudaGetLastError(); return fail(FP8BS_ERR_DEVICE, "no CUDA device: %s", cudaGetErrorString(e)); }
    static int verdict[64] = {0};   // 0 unknown, 1 ok, 2 bad
    if (dev >= 0 && dev < 64 && verdict[dev] == 1) return FP8BS_OK;
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0) {
        if (dev >= 0 && dev < 64) verdict[dev] = 2;
        return fail(FP8BS_ERR_DEVICE, "device %d is compute capability %d.%d; libfp8bs is built for sm_100a (10.0)", dev, major, minor);
    }
    if (dev >= 0 && dev < 64) verdict[dev] = 1;
    return FP8BS_OK;
}

static fp8bs_status from_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return ok();
    return fail(FP8BS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

static bool valid_dtype(int d) { return d == FP8BS_BF16 || d == FP8BS_FP32; }

}  // namespace fp8bs

using namespace fp8bs;

extern "C" {

int fp8bs_abi_version(void) { return FP8BS_ABI_VERSION; }

const char* fp8bs_status_string(fp8bs_status s) {
    switch (s) {
        case FP8BS_OK: return "FP8BS_OK";
        case FP8BS_ERR_INVALID_ARG: return "FP8BS_ERR_INVALID_ARG: null pointer, negative size or bad enum";
        case FP8BS_ERR_SHAPE: return "FP8BS_ERR_SHAPE: inconsistent sizes or leading dimensions";
        case FP8BS_ERR_ALIGN: return "FP8BS_ERR_ALIGN: pointer or pitch not aligned as required";
        case FP8BS_ERR_UNSUPPORTED: return "FP8BS_ERR_UNSUPPORTED: unsupported combination";
        case FP8BS_ERR_DEVICE: return "FP8BS_ERR_DEVICE: no sm_100 device";
        case FP8BS_ERR_CUDA: return "FP8BS_ERR_CUDA: CUDA error";
    }
    return "FP8BS_ERR_UNKNOWN";
}

const char* fp8bs_last_error_detail(void) { return g_detail; }

fp8bs_status fp8bs_device_supported(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) { cudaGetLastError(); return fail(FP8BS_ERR_DEVICE, "cudaGetDeviceCount: %s", cudaGetErrorString(e)); }
    if (device < 0 || device >= n) return fail(FP8BS_ERR_DEVICE, "device %d out of range (%d devices)", device, n);
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    if (major != 10 || minor != 0) return fail(FP8BS_ERR_DEVICE, "compute capability %d.%d is not 10.0", major, minor);
    return ok();
}

fp8bs_status fp8bs_quantize_act_1x128(const void* x, fp8bs_dtype xdt, int64_t M, int64_t K, int64_t ldx,
                                      uint8_t* q, int64_t ldq, float* s, int64_t lds, fp8bs_stream_t stream) {
    if (!valid_dtype(xdt)) return fail(FP8BS_ERR_INVALID_ARG, "xdt=%d", (int)xdt);
    if (M < 0 || K < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative size M=%lld K=%lld", (long long)M, (long long)K);
    if (M == 0 || K == 0) return ok();
    if (!x || !q || !s) return fail(FP8BS_ERR_INVALID_ARG, "null pointer (x=%p q=%p s=%p)", x, (void*)q, (void*)s);
    if (ldx < K || ldq < K || lds < M) return fail(FP8BS_ERR_SHAPE, "need ldx>=K, ldq>=K, lds>=M (ldx=%lld ldq=%lld lds=%lld)",
                                                   (long long)ldx, (long long)ldq, (long long)lds);
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_quant_act_1x128(x, (int)xdt, M, K, ldx, q, ldq, s, lds, (cudaStream_t)stream),
                     "quantize_act_1x128 launch");
}

fp8bs_status fp8bs_quantize_act_1x128_pow2(const void* x, fp8bs_dtype xdt, int64_t M, int64_t K, int64_t ldx,
                                           uint8_t* q, int64_t ldq, float* s, int64_t lds, fp8bs_stream_t stream) {
    if (!valid_dtype(xdt)) return fail(FP8BS_ERR_INVALID_ARG, "xdt=%d", (int)xdt);
    if (M < 0 || K < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative size M=%lld K=%lld", (long long)M, (long long)K);
    if (M == 0 || K == 0) return ok();
    if (!x || !q || !s) return fail(FP8BS_ERR_INVALID_ARG, "null pointer (x=%p q=%p s=%p)", x, (void*)q, (void*)s);
    if (ldx < K || ldq < K || lds < M) return fail(FP8BS_ERR_SHAPE, "need ldx>=K, ldq>=K, lds>=M (ldx=%lld ldq=%lld lds=%lld)",
                                                   (long long)ldx, (long long)ldq, (long long)lds);
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_quant_act_1x128_pow2(x, (int)xdt, M, K, ldx, q, ldq, s, lds, (cudaStream_t)stream),
                     "quantize_act_1x128_pow2 launch");
}

fp8bs_status fp8bs_quantize_act_128x1(const void* x, fp8bs_dtype xdt, int64_t M, int64_t C, int64_t ldx,
                                      uint8_t* qT, int64_t ldq, float* sT, int64_t lds, fp8bs_stream_t stream) {
    if (!valid_dtype(xdt)) return fail(FP8BS_ERR_INVALID_ARG, "xdt=%d", (int)xdt);
    if (M < 0 || C < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative size M=%lld C=%lld", (long long)M, (long long)C);
    if (M == 0 || C == 0) return ok();
    if (!x || !qT || !sT) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ldx < C || ldq < M || lds < C) return fail(FP8BS_ERR_SHAPE, "need ldx>=C, ldq>=M, lds>=C");
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_quant_act_128x1(x, (int)xdt, M, C, ldx, qT, ldq, sT, lds, (cudaStream_t)stream),
                     "quantize_act_128x1 launch");
}

static fp8bs_status quantize_act_dual_impl(const void* x, fp8bs_dtype xdt, int64_t M, int64_t K, int64_t ldx,
                                           uint8_t* q, int64_t ldq, float* s, int64_t lds,
                                           uint8_t* qT, int64_t ldqT, float* sT, int64_t ldsT, int pow2,
                                           fp8bs_stream_t stream) {
    if (!valid_dtype(xdt)) return fail(FP8BS_ERR_INVALID_ARG, "xdt=%d", (int)xdt);
    if (M < 0 || K < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative size M=%lld K=%lld", (long long)M, (long long)K);
    if (M == 0 || K == 0) return ok();
    if (!x || !q || !s || !qT || !sT) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ldx < K || ldq < K || lds < M || ldqT < M || ldsT < K)
        return fail(FP8BS_ERR_SHAPE, "need ldx>=K, ldq>=K, lds>=M, ldqT>=M, ldsT>=K");
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_quant_act_dual(x, (int)xdt, M, K, ldx, q, ldq, s, lds, qT, ldqT, sT, ldsT, pow2, (cudaStream_t)stream),
                     pow2 ? "quantize_act_dual_pow2 launch" : "quantize_act_dual launch");
}

fp8bs_status fp8bs_quantize_act_dual(const void* x, fp8bs_dtype xdt, int64_t M, int64_t K, int64_t ldx,
                                    uint8_t* q, int64_t ldq, float* s, int64_t lds,
                                    uint8_t* qT, int64_t ldqT, float* sT, int64_t ldsT, fp8bs_stream_t stream) {
    return quantize_act_dual_impl(x, xdt, M, K, ldx, q, ldq, s, lds, qT, ldqT, sT, ldsT, 0, stream);
}

fp8bs_status fp8bs_quantize_act_dual_pow2(const void* x, fp8bs_dtype xdt, int64_t M, int64_t K, int64_t ldx,
                                         uint8_t* q, int64_t ldq, float* s, int64_t lds,
                                         uint8_t* qT, int64_t ldqT, float* sT, int64_t ldsT, fp8bs_stream_t stream) {
    return quantize_act_dual_impl(x, xdt, M, K, ldx, q, ldq, s, lds, qT, ldqT, sT, ldsT, 1, stream);
}

fp8bs_status fp8bs_requantize_1x128_to_128x1(const uint8_t* q, int64_t ldq, const float* s, int64_t lds,
                                             int64_t M, int64_t K, uint8_t* qT, int64_t ldqT,
                                             float* sT, int64_t ldsT, int pow2, fp8bs_stream_t stream) {
    if (M < 0 || K < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative size M=%lld K=%lld", (long long)M, (long long)K);
    if (M == 0 || K == 0) return ok();
    if (!q || !s || !qT || !sT) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ldq < K || lds < M || ldqT < M || ldsT < K) return fail(FP8BS_ERR_SHAPE, "need ldq>=K, lds>=M, ldqT>=M, ldsT>=K");
    if (!aligned16(q) || !aligned16(qT) || ldq % 16 || ldqT % 16)
        return fail(FP8BS_ERR_ALIGN, "q, qT must be 16-byte aligned with ldq, ldqT multiples of 16");
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_requant_1x128_to_128x1(q, ldq, s, lds, M, K, qT, ldqT, sT, ldsT, pow2 != 0, (cudaStream_t)stream),
                     "requantize_1x128_to_128x1 launch");
}

static fp8bs_status quantize_weight_impl(const void* w, fp8bs_dtype wdt, int64_t N, int64_t K, int64_t ldw,
                                         uint8_t* q, int64_t ldq, float* s, int64_t ldsw,
                                         uint8_t* qT, int64_t ldqT, int pow2, fp8bs_stream_t stream) {
    if (!valid_dtype(wdt)) return fail(FP8BS_ERR_INVALID_ARG, "wdt=%d", (int)wdt);
    if (N < 0 || K < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative size");
    if (N == 0 || K == 0) return ok();
    if (!w || !q || !s) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ldw < K || ldq < K || ldsw < (K + 127) / 128) return fail(FP8BS_ERR_SHAPE, "need ldw>=K, ldq>=K, ldsw>=ceil(K/128)");
    if (qT && ldqT < N) return fail(FP8BS_ERR_SHAPE, "need ldqT>=N");
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_quant_weight_128x128(w, (int)wdt, N, K, ldw, q, ldq, s, ldsw, qT, ldqT, pow2, (cudaStream_t)stream),
                     pow2 ? "quantize_weight_128x128_pow2 launch" : "quantize_weight_128x128 launch");
}

fp8bs_status fp8bs_quantize_weight_128x128(const void* w, fp8bs_dtype wdt, int64_t N, int64_t K, int64_t ldw,
                                           uint8_t* q, int64_t ldq, float* s, int64_t ldsw,
                                           uint8_t* qT, int64_t ldqT, fp8bs_stream_t stream) {
    return quantize_weight_impl(w, wdt, N, K, ldw, q, ldq, s, ldsw, qT, ldqT, 0, stream);
}

fp8bs_status fp8bs_quantize_weight_128x128_pow2(const void* w, fp8bs_dtype wdt, int64_t N, int64_t K, int64_t ldw,
                                                uint8_t* q, int64_t ldq, float* s, int64_t ldsw,
                                                uint8_t* qT, int64_t ldqT, fp8bs_stream_t stream) {
    return quantize_weight_impl(w, wdt, N, K, ldw, q, ldq, s, ldsw, qT, ldqT, 1, stream);
}

static fp8bs_status check_gemm_common(int64_t M, int64_t N, int64_t K, const uint8_t* A, int64_t lda, const float* sA,
                                      int64_t ldsA, const uint8_t* B, int64_t ldb, const float* sB, void* D,
                                      fp8bs_dtype ddt, int64_t ldd) {
    if (!valid_dtype(ddt)) return fail(FP8BS_ERR_INVALID_ARG, "ddt=%d", (int)ddt);
    if (M < 0 || N < 0 || K < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative size");
    if (M > 0x7fffffff || N > 0x7fffffff || K > 0x7fffffff) return fail(FP8BS_ERR_SHAPE, "sizes must be < 2^31");
    if (M == 0 || N == 0) return FP8BS_OK;
    if (K == 0 || K % 128) return fail(FP8BS_ERR_SHAPE, "misaligned groups: contraction K=%lld must be a positive multiple of 128", (long long)K);
    if (!A || !sA || !B || !sB || !D) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (lda < K || ldb < K || ldd < N || ldsA < M) return fail(FP8BS_ERR_SHAPE, "need lda>=K, ldb>=K, ldd>=N, ldsA>=M");
    if (!aligned16(A) || !aligned16(B) || !aligned16(D) || !aligned16(sA) || !aligned16(sB))
        return fail(FP8BS_ERR_ALIGN, "A, B, D, sA, sB must be 16-byte aligned");
    if (lda % 16 || ldb % 16 || ldsA % 4) return fail(FP8BS_ERR_ALIGN, "lda, ldb must be multiples of 16 and ldsA of 4");
    const int64_t esz = ddt == FP8BS_BF16 ? 2 : 4;
    if ((ldd * esz) % 16) return fail(FP8BS_ERR_ALIGN, "ldd*sizeof(D) must be a multiple of 16");
    if (N % (ddt == FP8BS_BF16 ? 8 : 4)) return fail(FP8BS_ERR_ALIGN, "N must be a multiple of 8 (BF16 out) or 4 (FP32 out)");
    return FP8BS_OK;
}

static fp8bs_status gemm_impl(int mx, fp8bs_layout layout, int64_t M, int64_t N, int64_t K,
                              const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                              const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                              void* D, fp8bs_dtype ddt, int64_t ldd, int accumulate, fp8bs_stream_t stream,
                              void* workspace = nullptr, size_t workspace_bytes = 0);

fp8bs_status fp8bs_gemm(fp8bs_layout layout, int64_t M, int64_t N, int64_t K,
                        const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                        const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                        void* D, fp8bs_dtype ddt, int64_t ldd, int accumulate, fp8bs_stream_t stream) {
    return gemm_impl(0, layout, M, N, K, A, lda, sA, ldsA, B, ldb, sB, ldsB, D, ddt, ldd, accumulate, stream);
}

size_t fp8bs_gemm_workspace_size(fp8bs_layout layout, int64_t M, int64_t N, int64_t K) {
    if (layout != FP8BS_FPROP && layout != FP8BS_DGRAD && layout != FP8BS_WGRAD) return 0;
    if (M <= 0 || N <= 0 || K <= 0 || K % 128 || M > 0x7fffffff || N > 0x7fffffff || K > 0x7fffffff) return 0;
    return split_workspace_bytes(M, N, K);
}

fp8bs_status fp8bs_gemm_ws(fp8bs_layout layout, int64_t M, int64_t N, int64_t K,
                           const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                           const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                           void* D, fp8bs_dtype ddt, int64_t ldd, int accumulate,
                           void* workspace, size_t workspace_bytes, fp8bs_stream_t stream) {
    return gemm_impl(0, layout, M, N, K, A, lda, sA, ldsA, B, ldb, sB, ldsB, D, ddt, ldd, accumulate, stream,
                     workspace, workspace_bytes);
}

fp8bs_status fp8bs_gemm_mx(fp8bs_layout layout, int64_t M, int64_t N, int64_t K,
                           const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                           const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                           void* D, fp8bs_dtype ddt, int64_t ldd, int accumulate, fp8bs_stream_t stream) {
    return gemm_impl(1, layout, M, N, K, A, lda, sA, ldsA, B, ldb, sB, ldsB, D, ddt, ldd, accumulate, stream);
}

static fp8bs_status gemm_impl(int mx, fp8bs_layout layout, int64_t M, int64_t N, int64_t K,
                              const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                              const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                              void* D, fp8bs_dtype ddt, int64_t ldd, int accumulate, fp8bs_stream_t stream,
                              void* workspace, size_t workspace_bytes) {
    if (layout != FP8BS_FPROP && layout != FP8BS_DGRAD && layout != FP8BS_WGRAD)
        return fail(FP8BS_ERR_INVALID_ARG, "layout=%d", (int)layout);
    fp8bs_status c = check_gemm_common(M, N, K, A, lda, sA, ldsA, B, ldb, sB, D, ddt, ldd);
    if (c != FP8BS_OK) return c;
    if (M == 0 || N == 0) return ok();
    const int64_t KB = K / 128, NB = (N + 127) / 128;
    if (layout == FP8BS_FPROP && ldsB < KB) return fail(FP8BS_ERR_SHAPE, "FPROP needs ldsB >= K/128");
    if (layout == FP8BS_DGRAD && ldsB < NB) return fail(FP8BS_ERR_SHAPE, "DGRAD needs ldsB >= ceil(N/128)");
    if (layout == FP8BS_WGRAD) {
        if (ldsB < N) return fail(FP8BS_ERR_SHAPE, "WGRAD needs ldsB >= N");
        if (ldsB % 4) return fail(FP8BS_ERR_ALIGN, "WGRAD needs ldsB % 4 == 0");
        if (ddt != FP8BS_FP32) return fail(FP8BS_ERR_UNSUPPORTED, "WGRAD writes FP32 weight gradients (P:487, P:551)");
    }
    if (accumulate && ddt != FP8BS_FP32) return fail(FP8BS_ERR_UNSUPPORTED, "accumulate requires FP32 output");
    if (accumulate && layout != FP8BS_WGRAD) return fail(FP8BS_ERR_UNSUPPORTED, "accumulate is supported for WGRAD only");
    if (workspace) {
        if (!aligned16(workspace)) return fail(FP8BS_ERR_ALIGN, "workspace must be 16-byte aligned");
        const size_t need = split_workspace_bytes(M, N, K);
        if (workspace_bytes < need)
            return fail(FP8BS_ERR_INVALID_ARG, "workspace of %zu bytes < fp8bs_gemm_workspace_size = %zu", workspace_bytes, need);
    }
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    GemmArgs a{};
    a.layout = (int)layout; a.M = M; a.N = N; a.K = K;
    a.A = A; a.lda = lda; a.sA = sA; a.ldsA = ldsA; a.B = B; a.ldb = ldb; a.sB = sB; a.ldsB = ldsB;
    a.D = D; a.out_f32 = ddt == FP8BS_FP32; a.ldd = ldd; a.accumulate = accumulate ? 1 : 0;
    a.grouped = 0; a.G = 0; a.offsets = nullptr;
    if (workspace) { a.split_ws = workspace; a.split_ws_bytes = workspace_bytes; }
    const char* detail = nullptr;
    cudaError_t e = mx ? launch_gemm_mx(a, (cudaStream_t)stream, &detail) : launch_gemm(a, (cudaStream_t)stream, &detail);
    if (e != cudaSuccess && detail) return fail(FP8BS_ERR_CUDA, "%s", detail);
    return from_cuda(e, mx ? "gemm_mx launch" : "gemm launch");
}

size_t fp8bs_grouped_gemm_workspace_size(int32_t G, int64_t total_M, int64_t N, int64_t K) {
    (void)K;
    if (G < 1 || total_M < 0 || N < 0) return 0;
    return grouped_workspace_bytes(G, total_M, N);
}

// streamed-operand arguments of fp8bs_grouped_gemm_scatter (internal.h GemmArgs::ready / max_sms)
struct StreamArgs { const uint32_t* ready; uint32_t target; int32_t chunks; int32_t max_sms; };

static fp8bs_status grouped_gemm_layout(int layout, int32_t G, int64_t total_M, int64_t N, int64_t K,
                                        const int64_t* offsets, const uint8_t* A, int64_t lda, const float* sA,
                                        int64_t ldsA, const uint8_t* B, const float* sB, void* D, fp8bs_dtype ddt,
                                        int64_t ldd, fp8bs_stream_t stream, int mx = 0, void* workspace = nullptr,
                                        size_t workspace_bytes = 0, void* const* sc_base = nullptr,
                                        const int32_t* sc_rank = nullptr, const int64_t* sc_row = nullptr,
                                        const StreamArgs* sa_stream = nullptr);

fp8bs_status fp8bs_grouped_gemm(int32_t G, int64_t total_M, int64_t N, int64_t K, const int64_t* offsets,
                                const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                const uint8_t* B, const float* sB,
                                void* D, fp8bs_dtype ddt, int64_t ldd,
                                void* workspace, size_t workspace_bytes, fp8bs_stream_t stream) {
    return grouped_gemm_layout(FP8BS_FPROP, G, total_M, N, K, offsets, A, lda, sA, ldsA, B, sB, D, ddt, ldd, stream, 0,
                               workspace, workspace_bytes);
}

fp8bs_status fp8bs_grouped_gemm_mx(int32_t G, int64_t total_M, int64_t N, int64_t K, const int64_t* offsets,
                                   const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                   const uint8_t* B, const float* sB,
                                   void* D, fp8bs_dtype ddt, int64_t ldd,
                                   void* workspace, size_t workspace_bytes, fp8bs_stream_t stream) {
    return grouped_gemm_layout(FP8BS_FPROP, G, total_M, N, K, offsets, A, lda, sA, ldsA, B, sB, D, ddt, ldd, stream, 1,
                               workspace, workspace_bytes);
}

fp8bs_status fp8bs_grouped_gemm_dgrad_mx(int32_t G, int64_t total_M, int64_t N, int64_t K, const int64_t* offsets,
                                         const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                         const uint8_t* B, const float* sB,
                                         void* D, fp8bs_dtype ddt, int64_t ldd,
                                         void* workspace, size_t workspace_bytes, fp8bs_stream_t stream) {
    return grouped_gemm_layout(FP8BS_DGRAD, G, total_M, N, K, offsets, A, lda, sA, ldsA, B, sB, D, ddt, ldd, stream, 1,
                               workspace, workspace_bytes);
}

fp8bs_status fp8bs_grouped_gemm_dgrad(int32_t G, int64_t total_M, int64_t N, int64_t K, const int64_t* offsets,
                                      const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                      const uint8_t* B, const float* sB,
                                      void* D, fp8bs_dtype ddt, int64_t ldd,
                                      void* workspace, size_t workspace_bytes, fp8bs_stream_t stream) {
    return grouped_gemm_layout(FP8BS_DGRAD, G, total_M, N, K, offsets, A, lda, sA, ldsA, B, sB, D, ddt, ldd, stream, 0,
                               workspace, workspace_bytes);
}

fp8bs_status fp8bs_grouped_gemm_scatter(int32_t G, int64_t total_M, int64_t N, int64_t K, const int64_t* offsets,
                                        const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                        const uint8_t* B, const float* sB,
                                        void* const* dst_base, const int32_t* dst_rank, const int64_t* dst_row,
                                        int64_t ldd, const uint32_t* ready, uint32_t ready_target, int32_t ready_chunks,
                                        int32_t max_sms, void* workspace, size_t workspace_bytes, fp8bs_stream_t stream) {
    if (!dst_base || !dst_rank || !dst_row) return fail(FP8BS_ERR_INVALID_ARG, "null destination table");
    if (ready && ready_chunks < 1) return fail(FP8BS_ERR_INVALID_ARG, "ready_chunks=%d must be >= 1", (int)ready_chunks);
    if (max_sms < 0) return fail(FP8BS_ERR_INVALID_ARG, "max_sms=%d < 0", (int)max_sms);
    if (ready && max_sms == 0)
        return fail(FP8BS_ERR_INVALID_ARG, "streamed operands need max_sms > 0 (SMs left for the dispatch it waits for)");
    const StreamArgs sa{ready, ready_target, ready_chunks, max_sms};
    /* no D: the common checks see A in its place (validated there); the rows go through the table */
    return grouped_gemm_layout(FP8BS_FPROP, G, total_M, N, K, offsets, A, lda, sA, ldsA, B, sB, (void*)A,
                               FP8BS_BF16, ldd, stream, 0, workspace, workspace_bytes, dst_base, dst_rank, dst_row, &sa);
}

static fp8bs_status grouped_gemm_layout(int layout, int32_t G, int64_t total_M, int64_t N, int64_t K,
                                        const int64_t* offsets, const uint8_t* A, int64_t lda, const float* sA,
                                        int64_t ldsA, const uint8_t* B, const float* sB, void* D, fp8bs_dtype ddt,
                                        int64_t ldd, fp8bs_stream_t stream, int mx, void* workspace,
                                        size_t workspace_bytes, void* const* sc_base, const int32_t* sc_rank,
                                        const int64_t* sc_row, const StreamArgs* sa_stream) {
    if (G < 1 || G > 1024) return fail(FP8BS_ERR_INVALID_ARG, "G=%d must be in [1, 1024]", (int)G);
    if (!offsets) return fail(FP8BS_ERR_INVALID_ARG, "offsets is NULL");
    fp8bs_status c = check_gemm_common(total_M, N, K, A, lda, sA, ldsA, B, K, sB, D, ddt, ldd);
    if (c != FP8BS_OK) return c;
    if (total_M == 0 || N == 0) return ok();
    if (K % 16) return fail(FP8BS_ERR_ALIGN, "K must be a multiple of 16");
    {   /* the tile table (promotion kernel) or the tile claim counter (UE8M0 kernel) */
        const size_t need = grouped_workspace_bytes(G, total_M, N);
        if (!workspace || workspace_bytes < need)
            return fail(FP8BS_ERR_INVALID_ARG, "workspace of %zu bytes needed (fp8bs_grouped_gemm_workspace_size), got %zu%s",
                        need, workspace_bytes, workspace ? "" : " (NULL)");
        if (!aligned16(workspace)) return fail(FP8BS_ERR_ALIGN, "workspace must be 16-byte aligned");
    }
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    GemmArgs a{};
    a.layout = layout; a.M = total_M; a.N = N; a.K = K;
    a.A = A; a.lda = lda; a.sA = sA; a.ldsA = ldsA; a.B = B; a.ldb = K; a.sB = sB;
    a.ldsB = layout == FP8BS_DGRAD ? (N + 127) / 128 : K / 128;
    a.D = D; a.out_f32 = ddt == FP8BS_FP32; a.ldd = ldd; a.accumulate = 0;
    a.grouped = 1; a.G = G; a.offsets = offsets; a.workspace = workspace;
    a.sc_base = sc_base; a.sc_rank = sc_rank; a.sc_row = sc_row;
    if (sa_stream) { a.ready = sa_stream->ready; a.ready_target = sa_stream->target; a.ready_chunks = sa_stream->chunks; a.max_sms = sa_stream->max_sms; }
    const char* detail = nullptr;
    cudaError_t e = mx ? launch_gemm_mx(a, (cudaStream_t)stream, &detail) : launch_gemm(a, (cudaStream_t)stream, &detail);
    if (e != cudaSuccess && detail) return fail(FP8BS_ERR_CUDA, "%s", detail);
    return from_cuda(e, mx ? "grouped_gemm_mx launch" : "grouped_gemm launch");
}

/* ---- expert-parallel exchange over NVLink peer memory (NEXT-3) ---- */
fp8bs_status fp8bs_dispatch_fp8(int64_t n_slots, int32_t top_k, int64_t K, const uint8_t* xq, int64_t ldxq,
                                const float* xs, int64_t ldxs, const int32_t* dst_rank, const int64_t* dst_row,
                                uint8_t* const* recv_q, int64_t ld_recv_q, float* const* recv_s, fp8bs_stream_t stream) {
    if (n_slots < 0 || K < 0 || top_k < 1) return fail(FP8BS_ERR_INVALID_ARG, "negative size or top_k < 1");
    if (n_slots == 0 || K == 0) return ok();
    if (n_slots % top_k) return fail(FP8BS_ERR_SHAPE, "n_slots must be a multiple of top_k (slots of whole tokens)");
    if (K % 128) return fail(FP8BS_ERR_SHAPE, "K must be a multiple of 128 (whole 1x128 groups)");
    if (!xq || !xs || !dst_rank || !dst_row || !recv_q || !recv_s) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ldxq < K || ld_recv_q < K || ldxs < n_slots / top_k) return fail(FP8BS_ERR_SHAPE, "need ldxq, ld_recv_q >= K, ldxs >= tokens");
    if (!aligned16(xq) || ldxq % 16 || ld_recv_q % 16) return fail(FP8BS_ERR_ALIGN, "xq 16-byte aligned, ldxq and ld_recv_q multiples of 16");
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_dispatch_fp8(n_slots, top_k, K, xq, ldxq, xs, ldxs, dst_rank, dst_row, recv_q, ld_recv_q, recv_s,
                                         (cudaStream_t)stream), "dispatch_fp8 launch");
}

fp8bs_status fp8bs_dispatch_fp8_stream(int32_t chunks, const int64_t* chunk_off, const int64_t* send_tok,
                                       const int32_t* send_rank, const int64_t* send_row, int64_t K,
                                       const uint8_t* xq, int64_t ldxq, const float* xs, int64_t ldxs,
                                       uint8_t* const* recv_q, int64_t ld_recv_q, float* const* recv_s, int64_t ld_recv_s,
                                       uint32_t* local_done, uint32_t* const* flags, int32_t world, uint32_t epoch,
                                       int32_t ctas, fp8bs_stream_t stream) {
    if (chunks < 1 || chunks > 1024) return fail(FP8BS_ERR_INVALID_ARG, "chunks=%d must be in [1, 1024]", (int)chunks);
    if (world < 1 || ctas < 1 || epoch == 0) return fail(FP8BS_ERR_INVALID_ARG, "need world >= 1, ctas >= 1, epoch >= 1");
    if (K <= 0 || K % 128) return fail(FP8BS_ERR_SHAPE, "K must be a positive multiple of 128 (whole 1x128 groups)");
    if (!chunk_off || !send_tok || !send_rank || !send_row || !xq || !xs || !recv_q || !recv_s || !local_done || !flags)
        return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ldxq < K || ld_recv_q < K || ldxs < 0 || ld_recv_s < 0) return fail(FP8BS_ERR_SHAPE, "need ldxq, ld_recv_q >= K");
    if (!aligned16(xq) || ldxq % 16 || ld_recv_q % 16) return fail(FP8BS_ERR_ALIGN, "xq 16-byte aligned, ldxq and ld_recv_q multiples of 16");
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_dispatch_stream(chunks, chunk_off, send_tok, send_rank, send_row, K, xq, ldxq, xs, ldxs, recv_q,
                                            ld_recv_q, recv_s, ld_recv_s, local_done, flags, world, epoch, ctas,
                                            (cudaStream_t)stream), "dispatch_fp8_stream launch");
}

fp8bs_status fp8bs_send_rows(int64_t n, const int64_t* tok, int64_t K, const uint8_t* xq, int64_t ldxq, const float* xs,
                             int64_t ldxs, const int32_t* dst_rank, const int64_t* dst_row, uint8_t* const* recv_q,
                             int64_t ld_recv_q, float* const* recv_s, fp8bs_stream_t stream) {
    if (n < 0 || K < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative size");
    if (n == 0 || K == 0) return ok();
    if (K % 128) return fail(FP8BS_ERR_SHAPE, "K must be a multiple of 128 (whole 1x128 groups)");
    if (!tok || !xq || !xs || !dst_rank || !dst_row || !recv_q || !recv_s) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ldxq < K || ld_recv_q < K || ldxs < 1) return fail(FP8BS_ERR_SHAPE, "need ldxq, ld_recv_q >= K");
    if (!aligned16(xq) || ldxq % 16 || ld_recv_q % 16) return fail(FP8BS_ERR_ALIGN, "xq 16-byte aligned, ldxq and ld_recv_q multiples of 16");
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_send_rows(n, tok, K, xq, ldxq, xs, ldxs, dst_rank, dst_row, recv_q, ld_recv_q, recv_s,
                                      (cudaStream_t)stream), "send_rows launch");
}

fp8bs_status fp8bs_expand_rows(int64_t R, const int64_t* idx, int64_t K, const uint8_t* tq, int64_t ld_tq, const float* ts,
                               int64_t ts_row_stride, int64_t ts_kb_stride, uint8_t* A, int64_t lda, float* sA, int64_t ldsA,
                               fp8bs_stream_t stream) {
    if (R < 0 || K < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative size");
    if (R == 0 || K == 0) return ok();
    if (K % 128) return fail(FP8BS_ERR_SHAPE, "K must be a multiple of 128 (whole 1x128 groups)");
    if (!idx || !tq || !ts || !A || !sA) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ld_tq < K || lda < K || ldsA < R) return fail(FP8BS_ERR_SHAPE, "need ld_tq, lda >= K and ldsA >= R");
    if (ts_row_stride < 0 || ts_kb_stride < 0) return fail(FP8BS_ERR_SHAPE, "negative scale strides");
    if (!aligned16(tq) || !aligned16(A) || ld_tq % 16 || lda % 16)
        return fail(FP8BS_ERR_ALIGN, "tq, A 16-byte aligned, ld_tq and lda multiples of 16");
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_expand_rows(R, idx, K, tq, ld_tq, ts, ts_row_stride, ts_kb_stride, A, lda, sA, ldsA,
                                        (cudaStream_t)stream), "expand_rows launch");
}

fp8bs_status fp8bs_scales_rows_to_blocks(int64_t R, int64_t KB, const float* src, float* dst, int64_t ldd,
                                         fp8bs_stream_t stream) {
    if (R < 0 || KB < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative size");
    if (R == 0 || KB == 0) return ok();
    if (!src || !dst) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ldd < R) return fail(FP8BS_ERR_SHAPE, "need ldd >= R");
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_rows_to_blocks(R, KB, src, dst, ldd, (cudaStream_t)stream), "scales_rows_to_blocks launch");
}

fp8bs_status fp8bs_combine_push_bf16(int64_t R, int64_t N, const void* y, int64_t ldy, const int32_t* dst_rank,
                                     const int64_t* dst_slot, void* const* recv_y, int64_t ld_recv_y,
                                     fp8bs_stream_t stream) {
    if (R < 0 || N < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative size");
    if (R == 0 || N == 0) return ok();
    if (!y || !dst_rank || !dst_slot || !recv_y) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ldy < N || ld_recv_y < N) return fail(FP8BS_ERR_SHAPE, "need ldy, ld_recv_y >= N");
    if (!aligned16(y) || N % 8 || ldy % 8 || ld_recv_y % 8) return fail(FP8BS_ERR_ALIGN, "y 16-byte aligned; N, ldy, ld_recv_y multiples of 8");
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_combine_push(R, N, y, ldy, dst_rank, dst_slot, recv_y, ld_recv_y, (cudaStream_t)stream),
                     "combine_push_bf16 launch");
}

fp8bs_status fp8bs_combine_reduce_bf16(int64_t T, int32_t top_k, int64_t N, const void* buf, int64_t ldb,
                                       const float* gates, void* out, int64_t ldo, fp8bs_stream_t stream) {
    if (T < 0 || N < 0 || top_k < 1) return fail(FP8BS_ERR_INVALID_ARG, "negative size or top_k < 1");
    if (T == 0 || N == 0) return ok();
    if (!buf || !gates || !out) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ldb < N || ldo < N) return fail(FP8BS_ERR_SHAPE, "need ldb, ldo >= N");
    if (!aligned16(buf) || !aligned16(out) || N % 8 || ldb % 8 || ldo % 8)
        return fail(FP8BS_ERR_ALIGN, "buf, out 16-byte aligned; N, ldb, ldo multiples of 8");
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    return from_cuda(launch_combine_reduce(T, top_k, N, buf, ldb, gates, out, ldo, (cudaStream_t)stream),
                     "combine_reduce_bf16 launch");
}

/* ---- SwiGLU FP8 epilogue of an up-projection (NEXT-2; reading R27) ---- */
static fp8bs_status check_swiglu_out(int64_t M, int64_t N2, uint8_t* qy, int64_t ldqy, float* sy, int64_t ldsy,
                                     uint8_t* qh, int64_t ldqh, float* sh, int64_t ldsh) {
    if (N2 % 256) return fail(FP8BS_ERR_SHAPE, "N = 2I must be a multiple of 256 (gate/up blocks of 128)");
    if (!qy || !sy) return fail(FP8BS_ERR_INVALID_ARG, "null pointer (qy, sy)");
    if ((qh == nullptr) != (sh == nullptr)) return fail(FP8BS_ERR_INVALID_ARG, "qh and sh: both or neither");
    if (ldqy < N2 / 2 || ldsy < M) return fail(FP8BS_ERR_SHAPE, "need ldqy >= N/2, ldsy >= M");
    if (!aligned16(qy) || ldqy % 16) return fail(FP8BS_ERR_ALIGN, "qy must be 16-byte aligned, ldqy a multiple of 16");
    if (reinterpret_cast<uintptr_t>(sy) % 4) return fail(FP8BS_ERR_ALIGN, "sy must be 4-byte aligned");
    if (qh) {
        if (ldqh < N2 || ldsh < M) return fail(FP8BS_ERR_SHAPE, "need ldqh >= N, ldsh >= M");
        if (!aligned16(qh) || ldqh % 16) return fail(FP8BS_ERR_ALIGN, "qh must be 16-byte aligned, ldqh a multiple of 16");
        if (reinterpret_cast<uintptr_t>(sh) % 4) return fail(FP8BS_ERR_ALIGN, "sh must be 4-byte aligned");
    }
    return FP8BS_OK;
}

fp8bs_status fp8bs_gemm_swiglu(int64_t M, int64_t N, int64_t K,
                               const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                               const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                               uint8_t* qy, int64_t ldqy, float* sy, int64_t ldsy,
                               uint8_t* qh, int64_t ldqh, float* sh, int64_t ldsh, fp8bs_stream_t stream) {
    /* the GEMM operands as an FPROP with BF16 output (the output pointer is qy, checked below) */
    fp8bs_status c = check_gemm_common(M, N, K, A, lda, sA, ldsA, B, ldb, sB, qy, FP8BS_BF16, N);
    if (c != FP8BS_OK) return c;
    if (M == 0 || N == 0) return ok();
    if (ldsB < K / 128) return fail(FP8BS_ERR_SHAPE, "FPROP needs ldsB >= K/128");
    c = check_swiglu_out(M, N, qy, ldqy, sy, ldsy, qh, ldqh, sh, ldsh);
    if (c != FP8BS_OK) return c;
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    GemmArgs a{};
    a.layout = FP8BS_FPROP; a.M = M; a.N = N; a.K = K;
    a.A = A; a.lda = lda; a.sA = sA; a.ldsA = ldsA; a.B = B; a.ldb = ldb; a.sB = sB; a.ldsB = ldsB;
    a.D = qy; a.out_f32 = 0; a.ldd = ldqy; a.accumulate = 0;
    a.swiglu = 1; a.sy = sy; a.ldsy = ldsy; a.qh = qh; a.ldqh = ldqh; a.sh = sh; a.ldsh = ldsh;
    const char* detail = nullptr;
    cudaError_t e = launch_gemm(a, (cudaStream_t)stream, &detail);
    if (e != cudaSuccess && detail) return fail(FP8BS_ERR_CUDA, "%s", detail);
    return from_cuda(e, "gemm_swiglu launch");
}

fp8bs_status fp8bs_grouped_gemm_swiglu(int32_t G, int64_t total_M, int64_t N, int64_t K, const int64_t* offsets,
                                       const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                       const uint8_t* B, const float* sB,
                                       uint8_t* qy, int64_t ldqy, float* sy, int64_t ldsy,
                                       uint8_t* qh, int64_t ldqh, float* sh, int64_t ldsh,
                                       void* workspace, size_t workspace_bytes, fp8bs_stream_t stream) {
    if (G < 1 || G > 1024) return fail(FP8BS_ERR_INVALID_ARG, "G=%d must be in [1, 1024]", (int)G);
    if (!offsets) return fail(FP8BS_ERR_INVALID_ARG, "offsets is NULL");
    fp8bs_status c = check_gemm_common(total_M, N, K, A, lda, sA, ldsA, B, K, sB, qy, FP8BS_BF16, N);
    if (c != FP8BS_OK) return c;
    if (total_M == 0 || N == 0) return ok();
    c = check_swiglu_out(total_M, N, qy, ldqy, sy, ldsy, qh, ldqh, sh, ldsh);
    if (c != FP8BS_OK) return c;
    const size_t need = grouped_workspace_bytes(G, total_M, N);
    if (!workspace || workspace_bytes < need)
        return fail(FP8BS_ERR_INVALID_ARG, "workspace of %zu bytes needed (fp8bs_grouped_gemm_workspace_size), got %zu",
                    need, workspace_bytes);
    if (!aligned16(workspace)) return fail(FP8BS_ERR_ALIGN, "workspace must be 16-byte aligned");
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    GemmArgs a{};
    a.layout = FP8BS_FPROP; a.M = total_M; a.N = N; a.K = K;
    a.A = A; a.lda = lda; a.sA = sA; a.ldsA = ldsA; a.B = B; a.ldb = K; a.sB = sB; a.ldsB = K / 128;
    a.D = qy; a.out_f32 = 0; a.ldd = ldqy; a.accumulate = 0;
    a.grouped = 1; a.G = G; a.offsets = offsets; a.workspace = workspace;
    a.swiglu = 1; a.sy = sy; a.ldsy = ldsy; a.qh = qh; a.ldqh = ldqh; a.sh = sh; a.ldsh = ldsh;
    const char* detail = nullptr;
    cudaError_t e = launch_gemm(a, (cudaStream_t)stream, &detail);
    if (e != cudaSuccess && detail) return fail(FP8BS_ERR_CUDA, "%s", detail);
    return from_cuda(e, "grouped_gemm_swiglu launch");
}

/* ---- grouped MoE expert Wgrad on the expert-aligned (padded) token layout (NEXT-3) ---- */
static int64_t padded_tokens(int32_t G, const int64_t* off) {
    if (G < 0 || !off || off[0] != 0) return -1;
    int64_t p = 0;
    for (int32_t e = 0; e < G; ++e) {
        int64_t m = off[e + 1] - off[e];
        if (m < 0) return -1;
        p += (m + 127) / 128 * 128;
    }
    return p;
}

int64_t fp8bs_padded_tokens(int32_t G, const int64_t* offsets) {
    int64_t p = padded_tokens(G, offsets);
    return p < 0 ? 0 : p;
}

fp8bs_status fp8bs_quantize_act_128x1_grouped(const void* x, fp8bs_dtype xdt, int32_t G, const int64_t* offsets,
                                              int64_t C, int64_t ldx, uint8_t* qT, int64_t ldq, float* sT,
                                              int64_t lds, fp8bs_stream_t stream) {
    if (!valid_dtype(xdt)) return fail(FP8BS_ERR_INVALID_ARG, "xdt=%d", (int)xdt);
    const int64_t Mp = padded_tokens(G, offsets);
    if (Mp < 0) return fail(FP8BS_ERR_INVALID_ARG, "offsets must be host int64 [G+1], offsets[0]=0, non-decreasing");
    if (C < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative C");
    if (Mp == 0 || C == 0) return ok();
    if (!x || !qT || !sT) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ldx < C || ldq < Mp || lds < C) return fail(FP8BS_ERR_SHAPE, "need ldx>=C, ldq>=Mp=%lld, lds>=C", (long long)Mp);
    fp8bs_status d = check_device();
    if (d != FP8BS_OK) return d;
    const size_t esz = xdt == FP8BS_BF16 ? 2 : 4;
    cudaStream_t st = (cudaStream_t)stream;
    {   /* one launch over every expert's token blocks (16-byte aligned rows); else a loop per expert */
        std::vector<int64_t> pad(G + 1, 0);
        for (int32_t e = 0; e < G; ++e) pad[e + 1] = pad[e] + (offsets[e + 1] - offsets[e] + 127) / 128 * 128;
        cudaError_t err = launch_quant_act_128x1_grouped(x, (int)xdt, G, offsets, pad.data(), C, ldx, qT, ldq, sT, lds, st);
        if (err == cudaSuccess) return ok();
        if (err != cudaErrorNotSupported) return from_cuda(err, "quantize_act_128x1_grouped launch");
        (void)cudaGetLastError();
    }
    int64_t p = 0;
    for (int32_t e = 0; e < G; ++e) {
        const int64_t m = offsets[e + 1] - offsets[e], mp = (m + 127) / 128 * 128;
        if (m == 0) continue;
        cudaError_t err = launch_quant_act_128x1((const char*)x + (size_t)offsets[e] * ldx * esz, (int)xdt, m, C, ldx,
                                                 qT + p, ldq, sT + (p / 128) * lds, lds, st);
        if (err != cudaSuccess) return from_cuda(err, "quantize_act_128x1_grouped launch");
        if (mp > m) {   /* zero codes in the padding columns: they add exactly 0 to the Wgrad */
            err = cudaMemset2DAsync(qT + p + m, (size_t)ldq, 0, (size_t)(mp - m), (size_t)C, st);
            if (err != cudaSuccess) return from_cuda(err, "quantize_act_128x1_grouped padding");
        }
        p += mp;
    }
    return ok();
}

static fp8bs_status grouped_wgrad_impl(int mx, int32_t G, const int64_t* offsets, int64_t N, int64_t K,
                                       const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                       const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                                       float* D, int64_t ldd, int accumulate, fp8bs_stream_t stream);

fp8bs_status fp8bs_grouped_gemm_wgrad(int32_t G, const int64_t* offsets, int64_t N, int64_t K,
                                      const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                      const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                                      float* D, int64_t ldd, int accumulate, fp8bs_stream_t stream) {
    return grouped_wgrad_impl(0, G, offsets, N, K, A, lda, sA, ldsA, B, ldb, sB, ldsB, D, ldd, accumulate, stream);
}

fp8bs_status fp8bs_grouped_gemm_wgrad_mx(int32_t G, const int64_t* offsets, int64_t N, int64_t K,
                                         const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                         const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                                         float* D, int64_t ldd, int accumulate, fp8bs_stream_t stream) {
    return grouped_wgrad_impl(1, G, offsets, N, K, A, lda, sA, ldsA, B, ldb, sB, ldsB, D, ldd, accumulate, stream);
}

static fp8bs_status grouped_wgrad_impl(int mx, int32_t G, const int64_t* offsets, int64_t N, int64_t K,
                                       const uint8_t* A, int64_t lda, const float* sA, int64_t ldsA,
                                       const uint8_t* B, int64_t ldb, const float* sB, int64_t ldsB,
                                       float* D, int64_t ldd, int accumulate, fp8bs_stream_t stream) {
    /* every argument is checked here, before the single launch: a failing call enqueues nothing */
    if (G < 0 || G > 1024) return fail(FP8BS_ERR_INVALID_ARG, "G=%d must be in [0, 1024]", (int)G);
    const int64_t Mp = padded_tokens(G, offsets);
    if (Mp < 0) return fail(FP8BS_ERR_INVALID_ARG, "offsets must be host int64 [G+1], offsets[0]=0, non-decreasing");
    if (N < 0 || K < 0) return fail(FP8BS_ERR_INVALID_ARG, "negative size");
    if (G == 0 || N == 0 || K == 0) return ok();
    if (N > 0x7fffffff / G || K > 0x7fffffff || Mp > 0x7fffffff) return fail(FP8BS_ERR_SHAPE, "sizes must be < 2^31");
    if (!D) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
    if (ldd < K) return fail(FP8BS_ERR_SHAPE, "need ldd >= K");
    if (!aligned16(D) || (ldd * 4) % 16 || K % 4) return fail(FP8BS_ERR_ALIGN, "D must be 16-byte aligned, ldd and K multiples of 4");
    if (Mp > 0) {
        if (!A || !sA || !B || !sB) return fail(FP8BS_ERR_INVALID_ARG, "null pointer");
        if (lda < Mp || ldb < Mp) return fail(FP8BS_ERR_SHAPE, "need lda, ldb >= Mp=%lld", (long long)Mp);
        if (ldsA < N || ldsB < K) return fail(FP8BS_ERR_SHAPE, "need ldsA >= N, ldsB >= K");
        if (!aligned16(A) || !aligned16(B) || !aligned16(sA) || !aligned16(sB))
            return fail(FP8BS_ERR_ALIGN, "A, B, sA, sB must be 16-byte aligned");
        if (lda % 16 || ldb % 16 || ldsA % 4 || ldsB % 4)
            return fail(FP8BS_ERR_ALIGN, "lda, ldb must be multiples of 16 and ldsA, ldsB of 4");
    }
    fp8bs_status dv = check_device();
    if (dv != FP8BS_OK) return dv;
    /* One persistent launch over (expert, n-tile, m-tile) tiles; tile of expert e contracts over its
     * own token blocks [P_e/128, P_e/128 + roundup(M_e,128)/128) — none for an expert without tokens,
     * whose tiles then write zeros (or add nothing when accumulating).  No side streams, no state. */
    std::vector<int> kb(2 * (size_t)G);
    int64_t p = 0;
    for (int32_t e = 0; e < G; ++e) {
        const int64_t mp = (offsets[e + 1] - offsets[e] + 127) / 128 * 128;
        kb[2 * e] = (int)(p / 128);
        kb[2 * e + 1] = (int)(mp / 128);
        p += mp;
    }
    GemmArgs a{};
    a.layout = FP8BS_WGRAD; a.M = N; a.N = K; a.K = Mp > 0 ? Mp : 128;
    a.A = A; a.lda = lda; a.sA = sA; a.ldsA = ldsA; a.B = B; a.ldb = ldb; a.sB = sB; a.ldsB = ldsB;
    a.D = D; a.out_f32 = 1; a.ldd = ldd; a.accumulate = accumulate ? 1 : 0;
    a.grouped = 1; a.G = G; a.offsets = nullptr; a.workspace = nullptr; a.gw_kb = kb.data();
    if (Mp == 0) {   /* no tokens at all: the tensor maps still need valid (never read) operands */
        if (accumulate) return ok();
        cudaError_t err = cudaMemset2DAsync(D, (size_t)ldd * 4, 0, (size_t)K * 4, (size_t)(N * G), (cudaStream_t)stream);
        return from_cuda(err, "grouped_gemm_wgrad zero fill");
    }
    const char* detail = nullptr;
    cudaError_t e = mx ? launch_gemm_mx(a, (cudaStream_t)stream, &detail) : launch_gemm(a, (cudaStream_t)stream, &detail);
    if (e != cudaSuccess && detail) return fail(FP8BS_ERR_CUDA, "%s", detail);
    return from_cuda(e, mx ? "grouped_gemm_wgrad_mx launch" : "grouped_gemm_wgrad launch");
}

}  // extern "C"
