// tmap.cu — host-side TMA tensor-map encoding (cuTensorMapEncodeTiled through the runtime's
// driver entry point, so libfp8bs.so needs no link-time libcuda and loads on GPU-less hosts).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "internal.h"

namespace fp8bs {

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

bool make_tmap(void* map, int dtype, int rank, const void* base, const uint64_t* dims,
               const uint64_t* strides_bytes, const uint32_t* box, int swizzle) {
    auto enc = get_encode();
    if (!enc) return false;
    const CUtensorMapDataType dt = dtype == TMAP_U8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : dtype == TMAP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                      : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    uint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(reinterpret_cast<CUtensorMap*>(map), dt, (cuuint32_t)rank, const_cast<void*>(base),
                     (const cuuint64_t*)dims, (const cuuint64_t*)strides_bytes, (const cuuint32_t*)box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swizzle == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                     : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace fp8bs
