"""ctypes binding of libfp8bs.so (include/fp8bs.h) — argument marshalling only.

Every step of the path runs in the CUDA kernels behind the C-ABI; this module only turns torch
tensors into (device pointer, size, leading dimension) tuples, allocates outputs with torch's
CUDA allocator, and passes torch's current CUDA stream.  There is no CPU fallback: if the
shared library is missing or fails to load, importing the functions raises.
"""
from __future__ import annotations

import ctypes
import os
import re

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FP8BS_LIB") or os.path.join(_PKG, "libfp8bs.so")   # FP8BS_LIB: A/B experiments
# Test-only build of the same sources (-DFP8BS_TEST_HOOKS=1, build.py): adds fp8bs_internal_* hooks.
TESTHOOKS_PATH = os.path.join(_PKG, "libfp8bs_testhooks.so")
HEADER = os.path.join(os.path.dirname(_PKG), "include", "fp8bs.h")

OK, ERR_INVALID_ARG, ERR_SHAPE, ERR_ALIGN, ERR_UNSUPPORTED, ERR_DEVICE, ERR_CUDA = range(7)
BF16, FP32 = 0, 1
FPROP, DGRAD, WGRAD = 0, 1, 2

_lib = None
_test_lib = None


class Fp8bsError(RuntimeError):
    def __init__(self, status: int, fn: str, detail: str):
        self.status = status
        super().__init__(f"{fn} -> {status_string(status)} ({detail})")


def lib() -> ctypes.CDLL:
    """Load libfp8bs.so (raises if it was not built: there is no fallback path)."""
    global _lib
    if _lib is None:
        _lib = _load(LIB_PATH)
    return _lib


def testhooks_lib() -> ctypes.CDLL:
    """The test-only build (tests/ and tools/ only): the same kernels plus fp8bs_internal_* hooks."""
    global _test_lib
    if _test_lib is None:
        _test_lib = _load(TESTHOOKS_PATH)
        _test_lib.fp8bs_internal_set_gemm_variant.argtypes = [ctypes.c_int]
        _test_lib.fp8bs_internal_debug_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
        _test_lib.fp8bs_internal_debug_timestamps.restype = ctypes.c_int
    return _test_lib


class forced_variant:
    """Context manager for tests: route every binding call through the test-hooks build with the GEMM
    tile variant forced (1: one CTA per 128-row tile, 2: CTA pair per 256-row tile)."""

    def __init__(self, v: int):
        self.v = v

    def __enter__(self):
        global _lib
        self.saved = lib()
        T = testhooks_lib()
        T.fp8bs_internal_set_gemm_variant(self.v)
        _lib = T
        return self

    def __exit__(self, *exc):
        global _lib
        _lib.fp8bs_internal_set_gemm_variant(0)
        _lib = self.saved
        return False


def _load(path: str) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -m paper_2412_19437_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    i64, vp, i32, st = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int
    L.fp8bs_abi_version.restype = ctypes.c_int
    L.fp8bs_status_string.restype = ctypes.c_char_p
    L.fp8bs_status_string.argtypes = [st]
    L.fp8bs_last_error_detail.restype = ctypes.c_char_p
    L.fp8bs_device_supported.restype = st
    L.fp8bs_device_supported.argtypes = [i32]
    L.fp8bs_quantize_act_1x128.restype = st
    L.fp8bs_quantize_act_1x128.argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64, vp]
    L.fp8bs_quantize_act_128x1.restype = st
    L.fp8bs_quantize_act_128x1.argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64, vp]
    L.fp8bs_quantize_weight_128x128.restype = st
    if hasattr(L, "fp8bs_quantize_act_dual"):   # (older builds, loaded via FP8BS_LIB for A/B runs, lack it)
        L.fp8bs_quantize_act_dual.argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp]
        L.fp8bs_quantize_act_dual.restype = st
    L.fp8bs_quantize_weight_128x128.argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp]
    if hasattr(L, "fp8bs_requantize_1x128_to_128x1"):
        L.fp8bs_requantize_1x128_to_128x1.restype = st
        L.fp8bs_requantize_1x128_to_128x1.argtypes = [vp, i64, vp, i64, i64, i64, vp, i64, vp, i64, i32, vp]
    if hasattr(L, "fp8bs_quantize_act_1x128_pow2"):
        L.fp8bs_quantize_act_1x128_pow2.restype = st
        L.fp8bs_quantize_act_1x128_pow2.argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64, vp]
    for name in ("fp8bs_quantize_act_dual_pow2",):
        if hasattr(L, name):
            getattr(L, name).argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp]
            getattr(L, name).restype = st
    if hasattr(L, "fp8bs_quantize_weight_128x128_pow2"):
        L.fp8bs_quantize_weight_128x128_pow2.argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp]
        L.fp8bs_quantize_weight_128x128_pow2.restype = st
    if hasattr(L, "fp8bs_grouped_gemm_mx"):
        L.fp8bs_grouped_gemm_mx.restype = st
        L.fp8bs_grouped_gemm_mx.argtypes = [ctypes.c_int32, i64, i64, i64, vp, vp, i64, vp, i64, vp, vp, vp, i32,
                                            i64, vp, ctypes.c_size_t, vp]
    if hasattr(L, "fp8bs_grouped_gemm_dgrad_mx"):
        L.fp8bs_grouped_gemm_dgrad_mx.restype = st
        L.fp8bs_grouped_gemm_dgrad_mx.argtypes = L.fp8bs_grouped_gemm_mx.argtypes
    if hasattr(L, "fp8bs_gemm_mx"):
        L.fp8bs_gemm_mx.restype = st
        L.fp8bs_gemm_mx.argtypes = [i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp, i32, i64, i32, vp]
    L.fp8bs_gemm.restype = st
    L.fp8bs_gemm.argtypes = [i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp, i32, i64, i32, vp]
    if hasattr(L, "fp8bs_gemm_ws"):
        L.fp8bs_gemm_ws.restype = st
        L.fp8bs_gemm_ws.argtypes = [i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp, i32, i64, i32, vp,
                                    ctypes.c_size_t, vp]
        L.fp8bs_gemm_workspace_size.restype = ctypes.c_size_t
        L.fp8bs_gemm_workspace_size.argtypes = [i32, i64, i64, i64]
    L.fp8bs_grouped_gemm.restype = st
    L.fp8bs_grouped_gemm.argtypes = [ctypes.c_int32, i64, i64, i64, vp, vp, i64, vp, i64, vp, vp, vp, i32, i64,
                                     vp, ctypes.c_size_t, vp]
    if hasattr(L, "fp8bs_grouped_gemm_scatter"):
        L.fp8bs_grouped_gemm_scatter.restype = st
        L.fp8bs_grouped_gemm_scatter.argtypes = [ctypes.c_int32, i64, i64, i64, vp, vp, i64, vp, i64, vp, vp, vp, vp,
                                                 vp, i64, vp, ctypes.c_uint32, ctypes.c_int32, ctypes.c_int32, vp,
                                                 ctypes.c_size_t, vp]
    if hasattr(L, "fp8bs_grouped_gemm_dgrad"):
        L.fp8bs_grouped_gemm_dgrad.restype = st
        L.fp8bs_grouped_gemm_dgrad.argtypes = L.fp8bs_grouped_gemm.argtypes
    if hasattr(L, "fp8bs_grouped_gemm_wgrad"):
        L.fp8bs_padded_tokens.restype = i64
        L.fp8bs_padded_tokens.argtypes = [ctypes.c_int32, vp]
        L.fp8bs_quantize_act_128x1_grouped.restype = st
        L.fp8bs_quantize_act_128x1_grouped.argtypes = [vp, i32, ctypes.c_int32, vp, i64, i64, vp, i64, vp, i64, vp]
        L.fp8bs_grouped_gemm_wgrad.restype = st
        L.fp8bs_grouped_gemm_wgrad.argtypes = [ctypes.c_int32, vp, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64,
                                               vp, i64, i32, vp]
        if hasattr(L, "fp8bs_grouped_gemm_wgrad_mx"):
            L.fp8bs_grouped_gemm_wgrad_mx.restype = st
            L.fp8bs_grouped_gemm_wgrad_mx.argtypes = L.fp8bs_grouped_gemm_wgrad.argtypes
    if hasattr(L, "fp8bs_dispatch_fp8_stream"):
        L.fp8bs_dispatch_fp8_stream.restype = st
        L.fp8bs_dispatch_fp8_stream.argtypes = [ctypes.c_int32, vp, vp, vp, vp, i64, vp, i64, vp, i64, vp, i64, vp, i64,
                                                vp, vp, ctypes.c_int32, ctypes.c_uint32, ctypes.c_int32, vp]
    if hasattr(L, "fp8bs_send_rows"):
        L.fp8bs_send_rows.restype = st
        L.fp8bs_send_rows.argtypes = [i64, vp, i64, vp, i64, vp, i64, vp, vp, vp, i64, vp, vp]
        L.fp8bs_expand_rows.restype = st
        L.fp8bs_expand_rows.argtypes = [i64, vp, i64, vp, i64, vp, i64, i64, vp, i64, vp, i64, vp]
    if hasattr(L, "fp8bs_dispatch_fp8"):
        L.fp8bs_dispatch_fp8.restype = st
        L.fp8bs_dispatch_fp8.argtypes = [i64, ctypes.c_int32, i64, vp, i64, vp, i64, vp, vp, vp, i64, vp, vp]
        L.fp8bs_scales_rows_to_blocks.restype = st
        L.fp8bs_scales_rows_to_blocks.argtypes = [i64, i64, vp, vp, i64, vp]
        L.fp8bs_combine_push_bf16.restype = st
        L.fp8bs_combine_push_bf16.argtypes = [i64, i64, vp, i64, vp, vp, vp, i64, vp]
        L.fp8bs_combine_reduce_bf16.restype = st
        L.fp8bs_combine_reduce_bf16.argtypes = [i64, ctypes.c_int32, i64, vp, i64, vp, vp, i64, vp]
    if hasattr(L, "fp8bs_gemm_swiglu"):
        L.fp8bs_gemm_swiglu.restype = st
        L.fp8bs_gemm_swiglu.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp, i64,
                                        vp, i64, vp]
        L.fp8bs_grouped_gemm_swiglu.restype = st
        L.fp8bs_grouped_gemm_swiglu.argtypes = [ctypes.c_int32, i64, i64, i64, vp, vp, i64, vp, i64, vp, vp, vp, i64,
                                                vp, i64, vp, i64, vp, i64, vp, ctypes.c_size_t, vp]
    L.fp8bs_grouped_gemm_workspace_size.restype = ctypes.c_size_t
    L.fp8bs_grouped_gemm_workspace_size.argtypes = [ctypes.c_int32, i64, i64, i64]
    return L


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fp8bs_[a-z0-9_]+)\s*\(", txt)))


def status_string(status: int) -> str:
    return lib().fp8bs_status_string(status).decode()


def last_error_detail() -> str:
    return lib().fp8bs_last_error_detail().decode()


def abi_version() -> int:
    return lib().fp8bs_abi_version()


def device_supported(device: int = 0) -> bool:
    return lib().fp8bs_device_supported(device) == OK


def _check(status: int, fn: str):
    if status != OK:
        raise Fp8bsError(status, fn, last_error_detail())


def _p(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(t: torch.Tensor):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return FP32
    raise TypeError(f"unsupported dtype {t.dtype} (BF16 or FP32)")


def _pad4(n: int) -> int:
    return (n + 3) // 4 * 4


def _cuda2d(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError(f"{name} must be 2-D with unit column stride")


# ------------------------------------------------------------------ quantizers ----
def quantize_act_1x128(x: torch.Tensor, q: torch.Tensor | None = None, s: torch.Tensor | None = None):
    """x [M,K] BF16/FP32 -> (q uint8 [M,K], s fp32 [ceil(K/128), M])  (include/fp8bs.h)."""
    _cuda2d(x, "x")
    M, K = x.shape
    if q is None:
        q = torch.empty(M, K, dtype=torch.uint8, device=x.device)
    if s is None:   # leading dimension padded to a multiple of 4 (16 B rows for the GEMM's TMA)
        s = torch.empty((K + 127) // 128, _pad4(M), dtype=torch.float32, device=x.device)[:, :M]
    _check(lib().fp8bs_quantize_act_1x128(_p(x), _dt(x), M, K, x.stride(0), _p(q), q.stride(0), _p(s), s.stride(0),
                                          _stream(x)), "fp8bs_quantize_act_1x128")
    return q, s


def quantize_act_1x128_pow2(x: torch.Tensor, q: torch.Tensor | None = None, s: torch.Tensor | None = None):
    """x [M,K] -> (q uint8 [M,K], s fp32 [ceil(K/128), M]) with power-of-two scales."""
    _cuda2d(x, "x")
    M, K = x.shape
    if q is None:
        q = torch.empty(M, K, dtype=torch.uint8, device=x.device)
    if s is None:
        s = torch.empty((K + 127) // 128, _pad4(M), dtype=torch.float32, device=x.device)[:, :M]
    _check(lib().fp8bs_quantize_act_1x128_pow2(_p(x), _dt(x), M, K, x.stride(0), _p(q), q.stride(0), _p(s), s.stride(0),
                                               _stream(x)), "fp8bs_quantize_act_1x128_pow2")
    return q, s


def quantize_act_128x1(x: torch.Tensor, qT: torch.Tensor | None = None, sT: torch.Tensor | None = None):
    """x [M,C] -> (qT uint8 [C,M], sT fp32 [ceil(M/128), C])."""
    _cuda2d(x, "x")
    M, C = x.shape
    if qT is None:
        qT = torch.empty(C, M, dtype=torch.uint8, device=x.device)
    if sT is None:
        sT = torch.empty((M + 127) // 128, _pad4(C), dtype=torch.float32, device=x.device)[:, :C]
    _check(lib().fp8bs_quantize_act_128x1(_p(x), _dt(x), M, C, x.stride(0), _p(qT), qT.stride(0), _p(sT),
                                          sT.stride(0), _stream(x)), "fp8bs_quantize_act_128x1")
    return qT, sT


def _host_offsets(offsets) -> torch.Tensor:
    """Expert offsets as a contiguous CPU int64 tensor (the grouped Wgrad calls take HOST offsets)."""
    off = torch.as_tensor(offsets, dtype=torch.int64).cpu().contiguous()
    if off.dim() != 1 or off.numel() < 1:
        raise ValueError("offsets must be int64 [G+1]")
    return off


def padded_tokens(offsets) -> int:
    """Mp = sum_e roundup(M_e, 128): token columns of the expert-aligned layout (include/fp8bs.h)."""
    off = _host_offsets(offsets)
    return int(lib().fp8bs_padded_tokens(off.numel() - 1, off.data_ptr()))


def quantize_act_128x1_grouped(x: torch.Tensor, offsets, qT: torch.Tensor | None = None,
                               sT: torch.Tensor | None = None):
    """x [R,C] rows grouped by expert (host offsets [G+1]) -> (qT uint8 [C,Mp], sT fp32 [Mp/128, C]) in
    the expert-aligned layout: 128x1 groups restart at each expert (fp8bs_quantize_act_128x1_grouped)."""
    _cuda2d(x, "x")
    off = _host_offsets(offsets)
    G, C = off.numel() - 1, x.shape[1]
    if int(off[0]) != 0 or int(off[-1]) != x.shape[0] or bool((off[1:] < off[:-1]).any()):
        raise ValueError(f"offsets must rise from 0 to x.shape[0] = {x.shape[0]} (got {off[0]}..{off[-1]})")
    Mp = padded_tokens(off)
    if qT is None:
        qT = torch.empty(C, Mp, dtype=torch.uint8, device=x.device)
    if sT is None:
        sT = torch.empty(Mp // 128, _pad4(C), dtype=torch.float32, device=x.device)[:, :C]
    if qT.dtype != torch.uint8 or qT.shape[0] < C or qT.shape[1] < Mp:
        raise ValueError(f"qT must be uint8 of at least [{C}, {Mp}]")
    if sT.dtype != torch.float32 or sT.shape[0] < Mp // 128 or sT.shape[1] < C:
        raise ValueError(f"sT must be float32 of at least [{Mp // 128}, {C}]")
    _check(lib().fp8bs_quantize_act_128x1_grouped(_p(x), _dt(x), G, off.data_ptr(), C, x.stride(0), _p(qT),
                                                  qT.stride(0), _p(sT), sT.stride(0), _stream(x)),
           "fp8bs_quantize_act_128x1_grouped")
    return qT, sT


def grouped_gemm_wgrad(offsets, A: torch.Tensor, sA: torch.Tensor, B: torch.Tensor, sB: torch.Tensor,
                       out: torch.Tensor | None = None, accumulate: bool = False, mx: bool = False):
    """Per-expert dW_e [N,K] (+)= WGRAD over expert e's tokens: A = dYqT [N,Mp], B = XqT [K,Mp], sA [Mp/128,N],
    sB [Mp/128,K] in the expert-aligned layout; out FP32 [G,N,K] (fp8bs_grouped_gemm_wgrad).  mx=True:
    power-of-two scales on UE8M0 block scaling (fp8bs_grouped_gemm_wgrad_mx)."""
    for t, n in ((A, "A"), (B, "B"), (sA, "sA"), (sB, "sB")):
        _cuda2d(t, n)
    off = _host_offsets(offsets)
    G, N, K = off.numel() - 1, A.shape[0], B.shape[0]
    if out is None:
        out = torch.empty(G, N, K, dtype=torch.float32, device=A.device)
    if out.dtype != torch.float32 or not out.is_cuda or out.stride(2) != 1 or out.stride(0) != N * out.stride(1):
        raise ValueError("out must be a CUDA float32 [G,N,K] tensor with unit column stride and stacked experts")
    fn, name = ((lib().fp8bs_grouped_gemm_wgrad_mx, "fp8bs_grouped_gemm_wgrad_mx") if mx
                else (lib().fp8bs_grouped_gemm_wgrad, "fp8bs_grouped_gemm_wgrad"))
    _check(fn(G, off.data_ptr(), N, K, _p(A), A.stride(0), _p(sA), sA.stride(0), _p(B), B.stride(0), _p(sB), sB.stride(0),
              _p(out), out.stride(1), 1 if accumulate else 0, _stream(A)), name)
    return out


def requantize_1x128_to_128x1(q: torch.Tensor, s: torch.Tensor, qT: torch.Tensor | None = None,
                              sT: torch.Tensor | None = None, pow2: bool = False):
    """Cached FP8 activation q [M,K] (1x128 codes) + s [ceil(K/128), M] -> dequantize -> 128x1:
    (qT uint8 [K,M], sT fp32 [ceil(M/128), K])  (include/fp8bs.h)."""
    _cuda2d(q, "q")
    M, K = q.shape
    if qT is None:   # row pitch padded to 16 bytes (16-byte code stores)
        qT = torch.empty(K, (M + 15) // 16 * 16, dtype=torch.uint8, device=q.device)[:, :M]
    if sT is None:
        sT = torch.empty((M + 127) // 128, _pad4(K), dtype=torch.float32, device=q.device)[:, :K]
    _check(lib().fp8bs_requantize_1x128_to_128x1(_p(q), q.stride(0), _p(s), s.stride(0), M, K, _p(qT), qT.stride(0),
                                                 _p(sT), sT.stride(0), int(pow2), _stream(q)), "fp8bs_requantize_1x128_to_128x1")
    return qT, sT


def quantize_act_dual(x: torch.Tensor, q=None, s=None, qT=None, sT=None, pow2: bool = False):
    """x [M,K] -> (q [M,K], s [ceil(K/128), M], qT [K,M], sT [ceil(M/128), K]): both groupings from one
    read of x (bit-identical to quantize_act_1x128 + quantize_act_128x1).  pow2: power-of-two scales
    (fp8bs_quantize_act_dual_pow2)."""
    _cuda2d(x, "x")
    M, K = x.shape
    if q is None:
        q = torch.empty(M, K, dtype=torch.uint8, device=x.device)
    if s is None:
        s = torch.empty((K + 127) // 128, _pad4(M), dtype=torch.float32, device=x.device)[:, :M]
    if qT is None:
        qT = torch.empty(K, M, dtype=torch.uint8, device=x.device)
    if sT is None:
        sT = torch.empty((M + 127) // 128, _pad4(K), dtype=torch.float32, device=x.device)[:, :K]
    name = "fp8bs_quantize_act_dual_pow2" if pow2 else "fp8bs_quantize_act_dual"
    _check(getattr(lib(), name)(_p(x), _dt(x), M, K, x.stride(0), _p(q), q.stride(0), _p(s), s.stride(0),
                                _p(qT), qT.stride(0), _p(sT), sT.stride(0), _stream(x)), name)
    return q, s, qT, sT


def quantize_weight_128x128(w: torch.Tensor, want_t: bool = True, q=None, s=None, qT=None, pow2: bool = False):
    """w [N,K] FP32/BF16 -> (q uint8 [N,K], s fp32 [ceil(N/128), ceil(K/128)], qT uint8 [K,N] or None).
    pow2: power-of-two scales (fp8bs_quantize_weight_128x128_pow2)."""
    _cuda2d(w, "w")
    N, K = w.shape
    if q is None:
        q = torch.empty(N, K, dtype=torch.uint8, device=w.device)
    if s is None:
        s = torch.empty((N + 127) // 128, (K + 127) // 128, dtype=torch.float32, device=w.device)
    if want_t and qT is None:
        qT = torch.empty(K, N, dtype=torch.uint8, device=w.device)
    name = "fp8bs_quantize_weight_128x128_pow2" if pow2 else "fp8bs_quantize_weight_128x128"
    _check(getattr(lib(), name)(_p(w), _dt(w), N, K, w.stride(0), _p(q), q.stride(0), _p(s),
                                s.stride(0), _p(qT) if want_t else None,
                                qT.stride(0) if want_t else 0, _stream(w)), name)
    return q, s, (qT if want_t else None)


# ------------------------------------------------------------------------ GEMM ----
def gemm_workspace_size(layout: int, M: int, N: int, K: int) -> int:
    """fp8bs_gemm_workspace_size: bytes of the split-K tail workspace for this shape (0: none)."""
    return int(lib().fp8bs_gemm_workspace_size(layout, M, N, K))


def gemm(layout: int, A: torch.Tensor, sA: torch.Tensor, B: torch.Tensor, sB: torch.Tensor,
         out_dtype: torch.dtype = torch.bfloat16, out: torch.Tensor | None = None, accumulate: bool = False,
         mx: bool = False, workspace="auto"):
    """D [M,N] (+)= block-scaled A [M,K] x B [N,K]^T (see include/fp8bs.h for the sB layout per
    layout).  mx=True: fp8bs_gemm_mx (all scales exact powers of two; UE8M0 block scaling in the
    tensor core, no promotion).  workspace: "auto" (default) allocates the split-K tail workspace when
    the shape has one (fp8bs_gemm_ws), a device uint8 tensor is used as that workspace, None runs
    fp8bs_gemm (every tile promoted over all of K in order).  Returns D."""
    for t, n in ((A, "A"), (B, "B"), (sA, "sA"), (sB, "sB")):
        _cuda2d(t, n)
    M, K = A.shape
    N = B.shape[0]
    if B.shape[1] != K:
        raise ValueError("A and B contraction sizes differ")
    if out is None:
        out = torch.empty(M, N, dtype=out_dtype, device=A.device)
    _cuda2d(out, "out")
    args = (layout, M, N, K, _p(A), A.stride(0), _p(sA), sA.stride(0), _p(B), B.stride(0), _p(sB),
            sB.stride(0), _p(out), _dt(out), out.stride(0), 1 if accumulate else 0)
    if mx:
        _check(lib().fp8bs_gemm_mx(*args, _stream(A)), "fp8bs_gemm_mx")
        return out
    if isinstance(workspace, str):
        if workspace != "auto":
            raise ValueError("workspace: 'auto', None or a device uint8 tensor")
        wsb = gemm_workspace_size(layout, M, N, K) if M > 0 and N > 0 else 0
        workspace = torch.empty(wsb, dtype=torch.uint8, device=A.device) if wsb > 0 else None
    if workspace is None:
        _check(lib().fp8bs_gemm(*args, _stream(A)), "fp8bs_gemm")
    else:
        if not workspace.is_cuda:
            raise ValueError("workspace must be a CUDA tensor")
        _check(lib().fp8bs_gemm_ws(*args, _p(workspace), workspace.numel() * workspace.element_size(), _stream(A)),
               "fp8bs_gemm_ws")
    return out


def grouped_gemm(offsets: torch.Tensor, A: torch.Tensor, sA: torch.Tensor, B: torch.Tensor, sB: torch.Tensor,
                 out_dtype: torch.dtype = torch.bfloat16, out: torch.Tensor | None = None, layout: int = FPROP,
                 mx: bool = False, workspace: torch.Tensor | None = None):
    """MoE expert GEMM over token rows grouped by expert: offsets int64 [G+1] (device), A [R,K],
    sA [K/128, R], B [G,N,K].  FPROP: sB [G,ceil(N/128),K/128] (fp8bs_grouped_gemm).  DGRAD: B holds
    each expert's WqT [in, out], sB [G,K/128,ceil(N/128)] each expert's sW (fp8bs_grouped_gemm_dgrad).
    workspace: device uint8 of fp8bs_grouped_gemm_workspace_size bytes (allocated per call if None)."""
    _cuda2d(A, "A")
    _cuda2d(sA, "sA")
    if offsets.dtype != torch.int64 or not offsets.is_cuda:
        raise ValueError("offsets must be a CUDA int64 tensor")
    if not (B.is_cuda and B.is_contiguous() and sB.is_cuda and sB.is_contiguous()):
        raise ValueError("B and sB must be contiguous CUDA tensors")
    G, N, K = B.shape
    R = A.shape[0]
    if out is None:
        out = torch.empty(R, N, dtype=out_dtype, device=A.device)
    if layout not in (FPROP, DGRAD):
        raise ValueError("grouped layouts: FPROP, DGRAD")
    if workspace is None:   # the tile table / claim counter (torch's caching allocator makes this cheap per call)
        wsb = int(lib().fp8bs_grouped_gemm_workspace_size(G, R, N, K))
        workspace = torch.empty((wsb + 15) // 16 * 16, dtype=torch.uint8, device=A.device)
    if mx:   # power-of-two scales on UE8M0 block scaling (fp8bs_grouped_gemm_mx / _dgrad_mx)
        fn, name = ((lib().fp8bs_grouped_gemm_mx, "fp8bs_grouped_gemm_mx") if layout == FPROP
                    else (lib().fp8bs_grouped_gemm_dgrad_mx, "fp8bs_grouped_gemm_dgrad_mx"))
    else:
        fn, name = ((lib().fp8bs_grouped_gemm, "fp8bs_grouped_gemm") if layout == FPROP
                    else (lib().fp8bs_grouped_gemm_dgrad, "fp8bs_grouped_gemm_dgrad"))
    _check(fn(G, R, N, K, _p(offsets), _p(A), A.stride(0), _p(sA), sA.stride(0), _p(B), _p(sB),
              _p(out), _dt(out), out.stride(0), _p(workspace), workspace.numel(), _stream(A)), name)
    return out


def grouped_gemm_scatter(offsets: torch.Tensor, A: torch.Tensor, sA: torch.Tensor, B: torch.Tensor, sB: torch.Tensor,
                         dst_ptrs: int, dst_rank: torch.Tensor, dst_row: torch.Tensor, ldd: int,
                         workspace: torch.Tensor | None = None, ready: torch.Tensor | None = None,
                         ready_target: int = 0, ready_chunks: int = 0, max_sms: int = 0):
    """fp8bs_grouped_gemm_scatter: the grouped expert Fprop (BF16) whose output row r is stored at
    dst_ptrs[dst_rank[r]] + dst_row[r] * ldd — dst_ptrs a device address of a pointer table (e.g. a
    symmetric-memory handle's buffer_ptrs_dev), dst_rank int32 / dst_row int64 device [R].  ready (device
    int32/uint32 [ready_chunks]), ready_target, max_sms: streamed operands (include/fp8bs.h)."""
    _cuda2d(A, "A")
    _cuda2d(sA, "sA")
    if offsets.dtype != torch.int64 or not offsets.is_cuda:
        raise ValueError("offsets must be a CUDA int64 tensor")
    if not (B.is_cuda and B.is_contiguous() and sB.is_cuda and sB.is_contiguous()):
        raise ValueError("B and sB must be contiguous CUDA tensors")
    if dst_rank.dtype != torch.int32 or dst_row.dtype != torch.int64 or not (dst_rank.is_cuda and dst_row.is_cuda):
        raise ValueError("dst_rank must be CUDA int32 and dst_row CUDA int64")
    G, N, K = B.shape
    R = A.shape[0]
    if dst_rank.numel() < R or dst_row.numel() < R:
        raise ValueError("dst_rank / dst_row need one entry per row of A")
    if workspace is None:
        wsb = int(lib().fp8bs_grouped_gemm_workspace_size(G, R, N, K))
        workspace = torch.empty((wsb + 15) // 16 * 16, dtype=torch.uint8, device=A.device)
    _check(lib().fp8bs_grouped_gemm_scatter(G, R, N, K, _p(offsets), _p(A), A.stride(0), _p(sA), sA.stride(0), _p(B),
                                            _p(sB), ctypes.c_void_p(dst_ptrs), _p(dst_rank), _p(dst_row), ldd,
                                            _p(ready), ready_target & 0xFFFFFFFF, ready_chunks, max_sms,
                                            _p(workspace), workspace.numel(), _stream(A)), "fp8bs_grouped_gemm_scatter")


def send_rows(tok: torch.Tensor, xq: torch.Tensor, xs: torch.Tensor, dst_rank: torch.Tensor, dst_row: torch.Tensor,
              recv_q_ptrs: int, ld_recv_q: int, recv_s_ptrs: int):
    """fp8bs_send_rows: each (token, destination rank) pair once into the receivers' token buffers."""
    _cuda2d(xq, "xq")
    _check(lib().fp8bs_send_rows(tok.numel(), _p(tok), xq.shape[1], _p(xq), xq.stride(0), _p(xs), xs.stride(0),
                                 _p(dst_rank), _p(dst_row), ctypes.c_void_p(recv_q_ptrs), ld_recv_q,
                                 ctypes.c_void_p(recv_s_ptrs), _stream(xq)), "fp8bs_send_rows")


def expand_rows(idx: torch.Tensor, tq: torch.Tensor, ts: torch.Tensor, A: torch.Tensor | None = None,
                sA: torch.Tensor | None = None, ts_layout: str = "rows"):
    """fp8bs_expand_rows: expert rows A [R, K] and sA [K/128, R] from the token codes tq and scales ts —
    ts_layout "rows": a row-major token buffer [tokens, K/128]; "blocks": the 1x128 quantizer's [K/128, lds]."""
    _cuda2d(tq, "tq")
    R, K = idx.numel(), tq.shape[1]
    if A is None:
        A = torch.empty(R, K, dtype=torch.uint8, device=tq.device)
    if sA is None:
        sA = torch.empty(K // 128, _pad4(R), dtype=torch.float32, device=tq.device)[:, :R]
    if A.shape[0] < R or A.shape[1] < K or A.dtype != torch.uint8 or sA.shape[0] < K // 128 or sA.shape[1] < R:
        raise ValueError("A must be uint8 [>= R, >= K] and sA [>= K/128, >= R]")
    if not (idx.is_cuda and idx.dtype == torch.int64):
        raise ValueError("idx must be a CUDA int64 tensor")
    rs, ks = (ts.stride(0), ts.stride(1)) if ts_layout == "rows" else (ts.stride(1), ts.stride(0))
    _check(lib().fp8bs_expand_rows(R, _p(idx), K, _p(tq), tq.stride(0), _p(ts), rs, ks, _p(A), A.stride(0), _p(sA),
                                   sA.stride(0), _stream(tq)), "fp8bs_expand_rows")
    return A, sA


def dispatch_fp8_stream(chunk_off: torch.Tensor, send_tok: torch.Tensor, send_rank: torch.Tensor, send_row: torch.Tensor,
                        xq: torch.Tensor, xs: torch.Tensor, recv_q_ptrs: int, ld_recv_q: int, recv_s_ptrs: int,
                        ld_recv_s: int, local_done: torch.Tensor, flag_ptrs: int, world: int, epoch: int, ctas: int = 32):
    """fp8bs_dispatch_fp8_stream (include/fp8bs.h): the chunked dispatch a concurrent grouped GEMM waits on."""
    _cuda2d(xq, "xq")
    K = xq.shape[1]
    _check(lib().fp8bs_dispatch_fp8_stream(chunk_off.numel() - 1, _p(chunk_off), _p(send_tok), _p(send_rank), _p(send_row),
                                           K, _p(xq), xq.stride(0), _p(xs), xs.stride(0), ctypes.c_void_p(recv_q_ptrs),
                                           ld_recv_q, ctypes.c_void_p(recv_s_ptrs), ld_recv_s, _p(local_done),
                                           ctypes.c_void_p(flag_ptrs), world, epoch & 0xFFFFFFFF, ctas, _stream(xq)),
           "fp8bs_dispatch_fp8_stream")


def _swiglu_outputs(R: int, N2: int, dev, cache: bool, qy, sy, qh, sh):
    I = N2 // 2
    if qy is None:
        qy = torch.empty(R, I, dtype=torch.uint8, device=dev)
    if sy is None:
        sy = torch.empty(I // 128, _pad4(R), dtype=torch.float32, device=dev)[:, :R]
    if cache and qh is None:
        qh = torch.empty(R, N2, dtype=torch.uint8, device=dev)
    if cache and sh is None:
        sh = torch.empty(N2 // 128, _pad4(R), dtype=torch.float32, device=dev)[:, :R]
    return qy, sy, qh, sh


def gemm_swiglu(A: torch.Tensor, sA: torch.Tensor, B: torch.Tensor, sB: torch.Tensor, cache: bool = True,
                qy=None, sy=None, qh=None, sh=None):
    """Up-projection with the SwiGLU FP8 epilogue (fp8bs_gemm_swiglu): A [M,K] codes, sA [K/128, M],
    B [2I, K] codes with (gate, up) row blocks of 128, sB [2I/128, K/128].  Returns (qy [M, I] codes,
    sy [I/128, M], qh [M, 2I] codes or None, sh [2I/128, M] or None)."""
    for t, n in ((A, "A"), (B, "B"), (sA, "sA"), (sB, "sB")):
        _cuda2d(t, n)
    M, K = A.shape
    N2 = B.shape[0]
    qy, sy, qh, sh = _swiglu_outputs(M, N2, A.device, cache, qy, sy, qh, sh)
    _check(lib().fp8bs_gemm_swiglu(M, N2, K, _p(A), A.stride(0), _p(sA), sA.stride(0), _p(B), B.stride(0), _p(sB),
                                   sB.stride(0), _p(qy), qy.stride(0), _p(sy), sy.stride(0), _p(qh),
                                   qh.stride(0) if qh is not None else 0, _p(sh), sh.stride(0) if sh is not None else 0,
                                   _stream(A)), "fp8bs_gemm_swiglu")
    return qy, sy, qh, sh


def grouped_gemm_swiglu(offsets: torch.Tensor, A: torch.Tensor, sA: torch.Tensor, B: torch.Tensor, sB: torch.Tensor,
                        cache: bool = True, qy=None, sy=None, qh=None, sh=None, workspace: torch.Tensor | None = None):
    """The grouped (MoE) expert up-projection with the SwiGLU FP8 epilogue (fp8bs_grouped_gemm_swiglu):
    offsets int64 [G+1] (device), A [R,K], sA [K/128, R], B [G, 2I, K], sB [G, 2I/128, K/128]."""
    _cuda2d(A, "A")
    _cuda2d(sA, "sA")
    if offsets.dtype != torch.int64 or not offsets.is_cuda:
        raise ValueError("offsets must be a CUDA int64 tensor")
    if not (B.is_cuda and B.is_contiguous() and sB.is_cuda and sB.is_contiguous()):
        raise ValueError("B and sB must be contiguous CUDA tensors")
    G, N2, K = B.shape
    R = A.shape[0]
    qy, sy, qh, sh = _swiglu_outputs(R, N2, A.device, cache, qy, sy, qh, sh)
    if workspace is None:
        wsb = int(lib().fp8bs_grouped_gemm_workspace_size(G, R, N2, K))
        workspace = torch.empty((wsb + 15) // 16 * 16, dtype=torch.uint8, device=A.device)
    _check(lib().fp8bs_grouped_gemm_swiglu(G, R, N2, K, _p(offsets), _p(A), A.stride(0), _p(sA), sA.stride(0), _p(B),
                                           _p(sB), _p(qy), qy.stride(0), _p(sy), sy.stride(0), _p(qh),
                                           qh.stride(0) if qh is not None else 0, _p(sh),
                                           sh.stride(0) if sh is not None else 0, _p(workspace), workspace.numel(),
                                           _stream(A)), "fp8bs_grouped_gemm_swiglu")
    return qy, sy, qh, sh


# --------------------------------------------------------- expert-parallel exchange ----
def dispatch_fp8(xq: torch.Tensor, xs: torch.Tensor, top_k: int, dst_rank: torch.Tensor, dst_row: torch.Tensor,
                 recv_q_ptrs: int, ld_recv_q: int, recv_s_ptrs: int):
    """fp8bs_dispatch_fp8: the local tokens' 1x128 codes xq [T, K] and scales xs [K/128, T] to every
    (token, k) slot's destination rank / row.  recv_*_ptrs: device addresses of [world] pointer arrays
    (peer pointers, e.g. torch symmetric memory's buffer_ptrs_dev)."""
    _cuda2d(xq, "xq")
    _cuda2d(xs, "xs")
    T, K = xq.shape
    if dst_rank.dtype != torch.int32 or dst_row.dtype != torch.int64 or dst_rank.numel() != T * top_k \
            or dst_row.numel() != T * top_k or not (dst_rank.is_cuda and dst_row.is_cuda):
        raise ValueError("dst_rank int32 / dst_row int64 CUDA tensors of T * top_k slots")
    _check(lib().fp8bs_dispatch_fp8(T * top_k, top_k, K, _p(xq), xq.stride(0), _p(xs), xs.stride(0), _p(dst_rank),
                                    _p(dst_row), ctypes.c_void_p(recv_q_ptrs), ld_recv_q, ctypes.c_void_p(recv_s_ptrs),
                                    _stream(xq)), "fp8bs_dispatch_fp8")


def scales_rows_to_blocks(src: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Row-major [R, KB] scales -> [KB, R] (row pitch padded to a multiple of 4) (fp8bs_scales_rows_to_blocks)."""
    _cuda2d(src, "src")
    R, KB = src.shape
    if out is None:
        out = torch.empty(KB, _pad4(R), dtype=torch.float32, device=src.device)[:, :R]
    _check(lib().fp8bs_scales_rows_to_blocks(R, KB, _p(src), _p(out), out.stride(0), _stream(src)),
           "fp8bs_scales_rows_to_blocks")
    return out


def combine_push_bf16(y: torch.Tensor, dst_rank: torch.Tensor, dst_slot: torch.Tensor, recv_y_ptrs: int, ld_recv_y: int):
    """fp8bs_combine_push_bf16: expert output rows y [R, N] BF16 to their token owners' combine buffers."""
    _cuda2d(y, "y")
    R, N = y.shape
    _check(lib().fp8bs_combine_push_bf16(R, N, _p(y), y.stride(0), _p(dst_rank), _p(dst_slot),
                                         ctypes.c_void_p(recv_y_ptrs), ld_recv_y, _stream(y)), "fp8bs_combine_push_bf16")


def combine_reduce_bf16(buf: torch.Tensor, gates: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[t] = BF16(sum_k gates[t, k] * buf[t * top_k + k]) (fp8bs_combine_reduce_bf16; R28)."""
    _cuda2d(buf, "buf")
    T, top_k = gates.shape
    N = buf.shape[1]
    if out is None:
        out = torch.empty(T, N, dtype=torch.bfloat16, device=buf.device)
    _check(lib().fp8bs_combine_reduce_bf16(T, top_k, N, _p(buf), buf.stride(0), _p(gates.contiguous()), _p(out),
                                           out.stride(0), _stream(buf)), "fp8bs_combine_reduce_bf16")
    return out
