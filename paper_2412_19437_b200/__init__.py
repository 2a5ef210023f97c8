"""paper_2412_19437_b200 — B200-native (sm_100a) FP8 fine-grained quantization and block-scaled
FP8 GEMMs with FP32 accumulation: the data-parallel hot path of DeepSeek-V3's FP8 training
framework (arXiv 2412.19437 §3.3).

All compute runs in ``libfp8bs.so`` (hand-written CUDA for sm_100a behind the C-ABI in
``include/fp8bs.h``); this package is the thin Python binding plus the expert-parallel sharding
layer (``ep``).  PyTorch supplies device memory, streams and process groups only.
"""
from ._lib import (BF16, DGRAD, FP32, FPROP, WGRAD, Fp8bsError, abi_version, device_supported, forced_variant, gemm, gemm_workspace_size, testhooks_lib,  # noqa: F401
                   grouped_gemm, grouped_gemm_scatter, grouped_gemm_swiglu, dispatch_fp8, dispatch_fp8_stream, send_rows, expand_rows, scales_rows_to_blocks, combine_push_bf16, combine_reduce_bf16, grouped_gemm_wgrad, gemm_swiglu, header_symbols, last_error_detail, lib, quantize_act_1x128, quantize_act_1x128_pow2, quantize_act_128x1, quantize_act_128x1_grouped, quantize_act_dual,
                   padded_tokens, quantize_weight_128x128, requantize_1x128_to_128x1, status_string)

__all__ = ["quantize_act_1x128", "quantize_act_1x128_pow2", "quantize_act_128x1", "quantize_act_dual", "quantize_weight_128x128", "requantize_1x128_to_128x1", "gemm", "grouped_gemm", "grouped_gemm_wgrad", "quantize_act_128x1_grouped", "padded_tokens",
           "FPROP", "DGRAD", "WGRAD", "Fp8bsError", "abi_version", "device_supported", "lib"]
