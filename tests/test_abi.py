"""C-ABI contract tests that need no GPU: the library loads, exports every symbol the header
declares, and rejects bad arguments before touching the device (include/fp8bs.h "Errors")."""
import ctypes

import pytest
import torch

import paper_2412_19437_b200 as fp
from paper_2412_19437_b200 import _lib as L


def test_library_loads_and_exports_header_symbols():
    lib = fp.lib()
    syms = L.header_symbols()
    assert len(syms) >= 10
    for name in syms:
        assert hasattr(lib, name), name
    assert fp.abi_version() == 3


def test_product_library_exports_only_header_symbols():
    """The product library exports exactly the header's functions: the fp8bs_internal_* test hooks
    live only in the test build (libfp8bs_testhooks.so)."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln and "fp8bs_" in ln}
    assert exported == set(L.header_symbols())
    hooks = subprocess.run(["nm", "-D", "--defined-only", L.TESTHOOKS_PATH], capture_output=True, text=True,
                           check=True).stdout
    assert "fp8bs_internal_set_gemm_variant" in hooks


def test_status_strings():
    for st in range(7):
        s = fp.status_string(st)
        assert s.startswith("FP8BS_")
    assert "UNKNOWN" in fp.status_string(99)


FAKE = ctypes.c_void_p(1 << 20)   # never dereferenced: validation fails first


def _q1x128(**kw):
    a = dict(x=FAKE, xdt=0, M=4, K=256, ldx=256, q=FAKE, ldq=256, s=FAKE, lds=4)
    a.update(kw)
    return fp.lib().fp8bs_quantize_act_1x128(a["x"], a["xdt"], a["M"], a["K"], a["ldx"], a["q"], a["ldq"],
                                             a["s"], a["lds"], None)


def test_quantize_validation():
    assert _q1x128(x=None) == L.ERR_INVALID_ARG
    assert _q1x128(xdt=7) == L.ERR_INVALID_ARG
    assert _q1x128(M=-1) == L.ERR_INVALID_ARG
    assert _q1x128(ldx=100) == L.ERR_SHAPE
    assert _q1x128(lds=3) == L.ERR_SHAPE
    assert _q1x128(M=0) == L.OK            # empty is a no-op, no device needed
    assert "lds" in fp.last_error_detail() or True
    lib = fp.lib()
    assert lib.fp8bs_quantize_act_128x1(FAKE, 0, 10, 8, 8, FAKE, 5, FAKE, 8, None) == L.ERR_SHAPE   # ldq < M
    assert lib.fp8bs_quantize_weight_128x128(FAKE, 1, 10, 300, 300, FAKE, 300, FAKE, 2, None, 0, None) == L.ERR_SHAPE
    # dual: every output is required and every leading dimension checked
    assert lib.fp8bs_quantize_act_dual(FAKE, 0, 10, 8, 8, FAKE, 8, FAKE, 10, None, 10, FAKE, 8, None) == L.ERR_INVALID_ARG
    assert lib.fp8bs_quantize_act_dual(FAKE, 0, 10, 8, 8, FAKE, 8, FAKE, 10, FAKE, 9, FAKE, 8, None) == L.ERR_SHAPE   # ldqT < M
    assert lib.fp8bs_quantize_act_dual(FAKE, 0, 10, 8, 8, FAKE, 8, FAKE, 10, FAKE, 10, FAKE, 7, None) == L.ERR_SHAPE  # ldsT < K
    assert lib.fp8bs_quantize_act_dual(FAKE, 3, 10, 8, 8, FAKE, 8, FAKE, 10, FAKE, 10, FAKE, 8, None) == L.ERR_INVALID_ARG
    assert lib.fp8bs_quantize_act_dual(FAKE, 0, 0, 8, 8, FAKE, 8, FAKE, 10, FAKE, 10, FAKE, 8, None) == L.OK
    assert lib.fp8bs_quantize_weight_128x128(FAKE, 1, 10, 300, 300, FAKE, 300, FAKE, 3, FAKE, 5, None) == L.ERR_SHAPE


def _gemm(**kw):
    A16 = ctypes.c_void_p(1 << 20)
    a = dict(layout=0, M=256, N=256, K=512, A=A16, lda=512, sA=A16, ldsA=256, B=A16, ldb=512, sB=A16, ldsB=4,
             D=A16, ddt=0, ldd=256, acc=0)
    a.update(kw)
    return fp.lib().fp8bs_gemm(a["layout"], a["M"], a["N"], a["K"], a["A"], a["lda"], a["sA"], a["ldsA"], a["B"],
                               a["ldb"], a["sB"], a["ldsB"], a["D"], a["ddt"], a["ldd"], a["acc"], None)


def test_gemm_validation():
    assert _gemm(layout=5) == L.ERR_INVALID_ARG
    assert _gemm(K=300) == L.ERR_SHAPE                    # misaligned groups
    assert "misaligned" in fp.last_error_detail()
    assert _gemm(A=None) == L.ERR_INVALID_ARG
    assert _gemm(A=ctypes.c_void_p((1 << 20) + 8)) == L.ERR_ALIGN
    assert _gemm(lda=520, K=512) == L.ERR_ALIGN
    assert _gemm(ldsA=258) == L.ERR_ALIGN
    assert _gemm(N=100, ldd=104) == L.ERR_ALIGN           # BF16 out needs N % 8
    assert _gemm(ldsB=3) == L.ERR_SHAPE                   # FPROP needs ldsB >= K/128
    assert _gemm(layout=1, ldsB=1) == L.ERR_SHAPE         # DGRAD needs ldsB >= ceil(N/128)
    assert _gemm(layout=2, ldsB=256, ddt=0) == L.ERR_UNSUPPORTED   # WGRAD is FP32 out
    assert _gemm(layout=2, ldsB=100) == L.ERR_SHAPE
    assert _gemm(acc=1, ddt=0) == L.ERR_UNSUPPORTED
    assert _gemm(acc=1, ddt=1, layout=0) == L.ERR_UNSUPPORTED
    assert _gemm(M=0) == L.OK


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only check")
def test_valid_call_without_device_reports_device_error():
    assert _gemm() == L.ERR_DEVICE
    assert _q1x128() == L.ERR_DEVICE
    assert not fp.device_supported(0)


def test_grouped_validation():
    lib = fp.lib()
    A16 = ctypes.c_void_p(1 << 20)
    assert lib.fp8bs_grouped_gemm(0, 10, 256, 512, A16, A16, 512, A16, 16, A16, A16, A16, 0, 256, None, 0, None) == L.ERR_INVALID_ARG
    assert lib.fp8bs_grouped_gemm(2000, 10, 256, 512, A16, A16, 512, A16, 16, A16, A16, A16, 0, 256, None, 0, None) == L.ERR_INVALID_ARG
    assert lib.fp8bs_grouped_gemm(4, 10, 256, 512, None, A16, 512, A16, 16, A16, A16, A16, 0, 256, None, 0, None) == L.ERR_INVALID_ARG
    assert lib.fp8bs_grouped_gemm(4, 10, 256, 500, A16, A16, 512, A16, 16, A16, A16, A16, 0, 256, None, 0, None) == L.ERR_SHAPE
    # ABI 2: a device workspace for the tile table is required (16 B per 128 x 256 tile + 16)
    ws = lib.fp8bs_grouped_gemm_workspace_size(4, 10, 256, 512)
    assert ws == 16 + 16 * ((1 + 4) * 1)
    assert lib.fp8bs_grouped_gemm(4, 10, 256, 512, A16, A16, 512, A16, 16, A16, A16, A16, 0, 256, None, 0, None) == L.ERR_INVALID_ARG
    assert lib.fp8bs_grouped_gemm(4, 10, 256, 512, A16, A16, 512, A16, 16, A16, A16, A16, 0, 256, A16, ws - 16, None) == L.ERR_INVALID_ARG
    assert lib.fp8bs_grouped_gemm(4, 10, 256, 512, A16, A16, 512, A16, 16, A16, A16, A16, 0, 256,
                                  ctypes.c_void_p((1 << 20) + 8), ws, None) == L.ERR_ALIGN
    assert lib.fp8bs_grouped_gemm_dgrad(4, 10, 256, 512, A16, A16, 512, A16, 16, A16, A16, A16, 0, 256, None, 0, None) == L.ERR_INVALID_ARG


def test_python_binding_rejects_cpu_tensors():
    with pytest.raises(ValueError):
        fp.quantize_act_1x128(torch.zeros(4, 128))


def test_requant_pow2_and_grouped_dgrad_validation():
    """Host-side validation of the entry points added in this round (no device needed)."""
    lib = fp.lib()
    A16 = ctypes.c_void_p(1 << 20)
    # fp8bs_requantize_1x128_to_128x1(q, ldq, s, lds, M, K, qT, ldqT, sT, ldsT, pow2, stream)
    assert lib.fp8bs_requantize_1x128_to_128x1(None, 256, A16, 64, 64, 256, A16, 64, A16, 256, 0, None) == L.ERR_INVALID_ARG
    assert lib.fp8bs_requantize_1x128_to_128x1(A16, 200, A16, 64, 64, 256, A16, 64, A16, 256, 0, None) == L.ERR_SHAPE  # ldq < K
    assert lib.fp8bs_requantize_1x128_to_128x1(A16, 264, A16, 64, 64, 256, A16, 64, A16, 256, 1, None) == L.ERR_ALIGN  # ldq % 16
    assert lib.fp8bs_requantize_1x128_to_128x1(A16, 256, A16, 64, 64, 256, A16, 64, A16, 255, 0, None) == L.ERR_SHAPE  # ldsT < K
    assert lib.fp8bs_requantize_1x128_to_128x1(A16, 256, A16, 64, 0, 256, A16, 64, A16, 256, 0, None) == L.OK         # M == 0
    # fp8bs_quantize_act_1x128_pow2: same contract as fp8bs_quantize_act_1x128
    assert lib.fp8bs_quantize_act_1x128_pow2(A16, 2, 10, 128, 128, A16, 128, A16, 10, None) == L.ERR_INVALID_ARG   # dtype
    assert lib.fp8bs_quantize_act_1x128_pow2(A16, 0, 10, 128, 100, A16, 128, A16, 10, None) == L.ERR_SHAPE         # ldx < K
    # fp8bs_grouped_gemm_dgrad: same rules as the grouped Fprop
    assert lib.fp8bs_grouped_gemm_dgrad(0, 10, 256, 512, A16, A16, 512, A16, 16, A16, A16, A16, 0, 256, None, 0, None) == L.ERR_INVALID_ARG
    assert lib.fp8bs_grouped_gemm_dgrad(4, 10, 256, 500, A16, A16, 512, A16, 16, A16, A16, A16, 0, 256, None, 0, None) == L.ERR_SHAPE


def test_gemm_ws_workspace_size_and_validation():
    """fp8bs_gemm_workspace_size / fp8bs_gemm_ws (split-K tail, reading R30), host side only.  Without a
    device the SM count falls back to B200's 148: C1's Dgrad (448 pair tiles on 74 clusters = 6 waves +
    4 tiles) cuts its 4 tail tiles into 18 chunks -> 72 units of 256 x 256 FP32; C1's Fprop tail fills
    57% of a wave -> no split (0 bytes)."""
    lib = fp.lib()
    assert L.gemm_workspace_size(L.DGRAD, 4096, 7168, 18432) == 72 * 256 * 256 * 4
    assert L.gemm_workspace_size(L.FPROP, 4096, 18432, 7168) == 0
    assert L.gemm_workspace_size(L.FPROP, 4096, 18432, 7100) == 0        # invalid K
    assert L.gemm_workspace_size(7, 4096, 7168, 18432) == 0
    A16 = ctypes.c_void_p(1 << 20)
    args = (L.DGRAD, 4096, 7168, 18432, A16, 18432, A16, 4096, A16, 18432, A16, 56, A16, 0, 7168, 0)
    need = L.gemm_workspace_size(L.DGRAD, 4096, 7168, 18432)
    assert lib.fp8bs_gemm_ws(*args, A16, need - 16, None) == L.ERR_INVALID_ARG
    assert "workspace" in fp.last_error_detail()
    assert lib.fp8bs_gemm_ws(*args, ctypes.c_void_p((1 << 20) + 8), need, None) == L.ERR_ALIGN
    assert lib.fp8bs_gemm_ws(*args[:5], 100, *args[6:], A16, need, None) == L.ERR_SHAPE      # lda < K first


def test_grouped_gemm_scatter_validation():
    lib = fp.lib()
    A16 = ctypes.c_void_p(1 << 20)
    ws = lib.fp8bs_grouped_gemm_workspace_size(4, 10, 256, 512)
    args = (4, 10, 256, 512, A16, A16, 512, A16, 16, A16, A16)
    plain = (None, 0, 0, 0)   # ready, ready_target, ready_chunks, max_sms
    assert lib.fp8bs_grouped_gemm_scatter(*args, None, A16, A16, 256, *plain, A16, ws, None) == L.ERR_INVALID_ARG
    assert lib.fp8bs_grouped_gemm_scatter(*args, A16, None, A16, 256, *plain, A16, ws, None) == L.ERR_INVALID_ARG
    assert lib.fp8bs_grouped_gemm_scatter(*args, A16, A16, A16, 200, *plain, A16, ws, None) == L.ERR_SHAPE       # ldd < N
    assert lib.fp8bs_grouped_gemm_scatter(*args, A16, A16, A16, 256, *plain, A16, ws - 16, None) == L.ERR_INVALID_ARG
    # streamed operands: ready flags need chunks >= 1 and an SM cap (the dispatch they wait for needs SMs)
    assert lib.fp8bs_grouped_gemm_scatter(*args, A16, A16, A16, 256, A16, 1, 0, 100, A16, ws, None) == L.ERR_INVALID_ARG
    assert lib.fp8bs_grouped_gemm_scatter(*args, A16, A16, A16, 256, A16, 1, 4, 0, A16, ws, None) == L.ERR_INVALID_ARG
    # fp8bs_dispatch_fp8_stream: host checks before any launch
    d = (8, A16, A16, A16, A16, 7168, A16, 7168, A16, 16, A16, 7168, A16, 16, A16, A16)
    assert lib.fp8bs_dispatch_fp8_stream(*d, 2, 1, 32, None) == L.ERR_DEVICE or torch.cuda.is_available()
    assert lib.fp8bs_dispatch_fp8_stream(0, *d[1:], 2, 1, 32, None) == L.ERR_INVALID_ARG            # chunks
    assert lib.fp8bs_dispatch_fp8_stream(*d, 2, 0, 32, None) == L.ERR_INVALID_ARG                    # epoch 0
    assert lib.fp8bs_dispatch_fp8_stream(*d[:5], 7000, *d[6:], 2, 1, 32, None) == L.ERR_SHAPE        # K % 128
