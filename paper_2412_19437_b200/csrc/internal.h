// internal.h — declarations shared between the C-ABI layer (api.cu) and the kernel files.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef FP8BS_TEST_HOOKS
#define FP8BS_TEST_HOOKS 0   // 1 only in libfp8bs_testhooks.so (build.py): exported test hooks
#endif

namespace fp8bs {

int num_sms();                                   // SM count of the current device (cached per device)
// TMA tensor map (a CUtensorMap, 64-byte aligned, 128 bytes) — tmap.cu
enum { TMAP_U8 = 0, TMAP_BF16 = 1, TMAP_F32 = 2 };
bool make_tmap(void* map, int dtype, int rank, const void* base, const uint64_t* dims,
               const uint64_t* strides_bytes /* rank-1 */, const uint32_t* box, int swizzle /* 0, 64, 128 bytes */);
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

cudaError_t launch_quant_act_1x128(const void* x, int xdt, int64_t M, int64_t K, int64_t ldx, uint8_t* q,
                                   int64_t ldq, float* s, int64_t lds, cudaStream_t st);
cudaError_t launch_quant_act_128x1_grouped(const void* x, int xdt, int32_t G, const int64_t* off, const int64_t* pad,
                                           int64_t C, int64_t ldx, uint8_t* qT, int64_t ldq, float* sT, int64_t lds,
                                           cudaStream_t st);
cudaError_t launch_quant_act_128x1(const void* x, int xdt, int64_t M, int64_t C, int64_t ldx, uint8_t* qT,
                                   int64_t ldq, float* sT, int64_t lds, cudaStream_t st);
cudaError_t launch_quant_act_dual(const void* x, int xdt, int64_t M, int64_t K, int64_t ldx, uint8_t* q, int64_t ldq,
                                  float* s, int64_t lds, uint8_t* qT, int64_t ldqT, float* sT, int64_t ldsT,
                                  int pow2, cudaStream_t st);
cudaError_t launch_quant_weight_128x128(const void* w, int wdt, int64_t N, int64_t K, int64_t ldw, uint8_t* q,
                                        int64_t ldq, float* s, int64_t ldsw, uint8_t* qT, int64_t ldqT,
                                        int pow2, cudaStream_t st);

cudaError_t launch_requant_1x128_to_128x1(const uint8_t* q, int64_t ldq, const float* s, int64_t lds, int64_t M, int64_t K,
                                          uint8_t* qT, int64_t ldqT, float* sT, int64_t ldsT, int pow2, cudaStream_t st);
cudaError_t launch_quant_act_1x128_pow2(const void* x, int xdt, int64_t M, int64_t K, int64_t ldx, uint8_t* q,
                                        int64_t ldq, float* s, int64_t lds, cudaStream_t st);

// Programmatic dependent launch (PDL): the kernel is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so its CTAs may be scheduled while the
// previous kernel in the stream drains; every PDL kernel executes griddepcontrol.wait (sm100.cuh
// griddep_wait) before its first global-memory access, which waits for the previous grid to
// complete and its writes to be visible.  This hides the launch gap between the step's kernels.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// expert-parallel exchange (ep.cu)
cudaError_t launch_dispatch_fp8(int64_t n, int top_k, int64_t K, const uint8_t* xq, int64_t ldxq, const float* xs,
                                int64_t ldxs, const int32_t* dst_rank, const int64_t* dst_row, uint8_t* const* recv_q,
                                int64_t ld_rq, float* const* recv_s, cudaStream_t st);
cudaError_t launch_dispatch_stream(int C, const int64_t* chunk_off, const int64_t* send_tok, const int32_t* send_rank,
                                  const int64_t* send_row, int64_t K, const uint8_t* xq, int64_t ldxq, const float* xs,
                                  int64_t ldxs, uint8_t* const* recv_q, int64_t ld_rq, float* const* recv_s, int64_t ld_rs,
                                  uint32_t* local_done, uint32_t* const* flags, int world, uint32_t epoch, int ctas,
                                  cudaStream_t st);
cudaError_t launch_send_rows(int64_t n, const int64_t* tok, int64_t K, const uint8_t* xq, int64_t ldxq, const float* xs,
                             int64_t ldxs, const int32_t* dst_rank, const int64_t* dst_row, uint8_t* const* recv_q,
                             int64_t ld_rq, float* const* recv_s, cudaStream_t st);
cudaError_t launch_expand_rows(int64_t R, const int64_t* idx, int64_t K, const uint8_t* tq, int64_t ldtq, const float* ts,
                               int64_t ts_rs, int64_t ts_ks, uint8_t* A, int64_t lda, float* sA, int64_t ldsA,
                               cudaStream_t st);
cudaError_t launch_rows_to_blocks(int64_t R, int64_t KB, const float* src, float* dst, int64_t ldd, cudaStream_t st);
cudaError_t launch_combine_push(int64_t R, int64_t N, const void* y, int64_t ldy, const int32_t* dst_rank,
                                const int64_t* dst_slot, void* const* recv_y, int64_t ld_recv_y, cudaStream_t st);
cudaError_t launch_combine_reduce(int64_t T, int top_k, int64_t N, const void* buf, int64_t ldb, const float* g, void* out,
                                  int64_t ldo, cudaStream_t st);

struct GemmArgs {
    int layout;              // 0 FPROP, 1 DGRAD, 2 WGRAD
    int64_t M, N, K;
    const uint8_t* A; int64_t lda;
    const float* sA; int64_t ldsA;
    const uint8_t* B; int64_t ldb;
    const float* sB; int64_t ldsB;
    void* D; int out_f32; int64_t ldd; int accumulate;
    // grouped
    int grouped; int32_t G; const int64_t* offsets;
    void* workspace;         // grouped: >= grouped_workspace_bytes(G, M, N) of device memory (tile table)
    const int* gw_kb;        // grouped Wgrad (layout 2): host [G][2] = {first 128-token block, blocks} per expert
    // SwiGLU FP8 epilogue (FPROP; N = 2I, gate / up interleaved per 128 columns): D = y codes [M, I]
    // (ldd), sy [I/128][ldsy]; optional FP8 cache of H: qh [M, N] (ldqh), sh [N/128][ldsh]
    int swiglu; float* sy; int64_t ldsy; uint8_t* qh; int64_t ldqh; float* sh; int64_t ldsh;
    // dense: optional split-K tail workspace (>= split_workspace_bytes(M, N, K)), nullptr = unsplit
    void* split_ws; size_t split_ws_bytes;
    // grouped Fprop, BF16: row r stored at sc_base[sc_rank[r]] + sc_row[r] * ldd instead of D (nullptr: D)
    void* const* sc_base; const int32_t* sc_rank; const int64_t* sc_row;
    // grouped, streamed A / sA: wait for ready[e * ready_chunks / G] >= ready_target (nullptr: no waits);
    // max_sms > 0 caps the persistent grid (the SMs left run the concurrent dispatch)
    const uint32_t* ready; uint32_t ready_target; int ready_chunks; int max_sms;
};
size_t grouped_workspace_bytes(int32_t G, int64_t total_M, int64_t N);
size_t split_workspace_bytes(int64_t M, int64_t N, int64_t K);   // 0: no split-K tail for this shape

// Returns cudaSuccess or the launch error; *detail gets a static message on host-side failures
// (tensor-map encoding).
cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t st, const char** detail);
// power-of-two scales on the tensor core's UE8M0 block scaling (gemm_mx.cu)
cudaError_t launch_gemm_mx(const GemmArgs& a, cudaStream_t st, const char** detail);

}  // namespace fp8bs
