"""CPU oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2412_19437_b200`` never imports it and shares no code with it.

Thin ctypes wrappers around ``oracle/liboracle.so`` (built from ``oracle/oracle.c`` by
``__graft_entry__.build()``), taking/returning CPU torch tensors.  Every function
follows the paper's definition; see ``oracle/oracle.c`` for the citations.

Pins (tests/test_oracle.py): E4M3 table invariants + torch float8 decode; encoder vs
an independent brute-force nearest search and vs torch's cast in the non-saturating
range; SPEC/worked-example goldens (tests/golden/); quantizer closed forms and
transpose/permutation invariants; GEMM closed form (exact integer arithmetic) and vs
numpy float64 matmul of dequantized operands.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
SRC_PATH = os.path.join(_HERE, "oracle.c")

BF16, FP32 = 0, 1
FPROP, DGRAD, WGRAD = 0, 1, 2

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with IEEE-strict flags."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(SRC_PATH), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC",
               "-shared", "-std=c11", "-Wall", "-o", LIB_PATH, SRC_PATH, "-lm"]
        subprocess.check_call(cmd)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        i64, vp, i32 = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        L.oracle_e4m3_decode.restype = ctypes.c_double
        L.oracle_e4m3_decode.argtypes = [ctypes.c_uint8]
        L.oracle_e4m3_encode.restype = ctypes.c_uint8
        L.oracle_e4m3_encode.argtypes = [ctypes.c_float]
        L.oracle_e4m3_encode_array.argtypes = [vp, i64, vp]
        L.oracle_quantize_act_1x128.argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64]
        L.oracle_quantize_act_128x1.argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64]
        L.oracle_quantize_weight_128x128.argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64]
        L.oracle_requantize_1x128_to_128x1.argtypes = [vp, i64, vp, i64, i64, i64, vp, i64, vp, i64, i32]
        L.oracle_quantize_act_1x128_pow2.argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64]
        L.oracle_quantize_act_128x1_pow2.argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64]
        L.oracle_quantize_weight_128x128_pow2.argtypes = [vp, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64]
        L.oracle_gemm.argtypes = [i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp, i32]
        L.oracle_grouped_gemm.argtypes = [ctypes.c_int32, vp, i64, i64, vp, i64, vp, i64, vp, vp, vp, i64, vp, i32]
        L.oracle_gemm_limited_accum.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64,
                                                i32, i32, i32, i32, vp, i32]
        L.oracle_rel_err_normwise.restype = ctypes.c_double
        L.oracle_rel_err_normwise.argtypes = [vp, vp, i64]
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_exp32.restype = ctypes.c_float
        L.oracle_exp32.argtypes = [ctypes.c_float]
        L.oracle_rcp32.restype = ctypes.c_float
        L.oracle_rcp32.argtypes = [ctypes.c_float]
        L.oracle_swiglu32.restype = ctypes.c_float
        L.oracle_swiglu32.argtypes = [ctypes.c_float, ctypes.c_float]
        L.oracle_swiglu_quant_1x128.argtypes = [vp, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64]
        L.oracle_float_to_bf16.restype = ctypes.c_uint16
        L.oracle_float_to_bf16.argtypes = [ctypes.c_float]
        L.oracle_combine_bf16.argtypes = [i64, i32, i64, vp, vp, vp]
        _lib = L
    return _lib


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    assert t.device.type == "cpu" and t.is_contiguous()
    return ctypes.c_void_p(t.data_ptr())


def _dt(x: torch.Tensor) -> int:
    if x.dtype == torch.bfloat16:
        return BF16
    if x.dtype == torch.float32:
        return FP32
    raise TypeError(f"unsupported dtype {x.dtype}")


def e4m3_decode(code: int) -> float:
    return lib().oracle_e4m3_decode(code)


def e4m3_encode(y: float) -> int:
    return lib().oracle_e4m3_encode(y)


def decode_table() -> torch.Tensor:
    """float64 [256] values of every E4M3 code (NaN at 0x7F/0xFF)."""
    return torch.tensor([e4m3_decode(c) for c in range(256)], dtype=torch.float64)


def encode_tensor(y: torch.Tensor) -> torch.Tensor:
    """Element-wise E4M3 encode of a float32 tensor."""
    flat = y.to(torch.float32).contiguous().reshape(-1)
    out = torch.empty(flat.numel(), dtype=torch.uint8)
    lib().oracle_e4m3_encode_array(_ptr(flat), flat.numel(), _ptr(out))
    return out.reshape(y.shape)


def quantize_act_1x128(x: torch.Tensor):
    """x [M,K] bf16/fp32 -> (q uint8 [M,K], s fp32 [ceil(K/128), M])."""
    x = x.contiguous()
    M, K = x.shape
    q = torch.empty(M, K, dtype=torch.uint8)
    s = torch.empty((K + 127) // 128, M, dtype=torch.float32)
    lib().oracle_quantize_act_1x128(_ptr(x), _dt(x), M, K, K, _ptr(q), K, _ptr(s), M)
    return q, s


def quantize_act_1x128_pow2(x: torch.Tensor):
    """1x128 tiles with power-of-two scales: x [M,K] -> (q [M,K], s [ceil(K/128), M])."""
    x = x.contiguous()
    M, K = x.shape
    q = torch.empty(M, K, dtype=torch.uint8)
    s = torch.empty((K + 127) // 128, M, dtype=torch.float32)
    lib().oracle_quantize_act_1x128_pow2(_ptr(x), _dt(x), M, K, K, _ptr(q), K, _ptr(s), M)
    return q, s


def quantize_act_128x1(x: torch.Tensor, pow2: bool = False):
    """x [M,C] -> (qT uint8 [C,M], sT fp32 [ceil(M/128), C]).  pow2: power-of-two scales."""
    x = x.contiguous()
    M, C = x.shape
    qT = torch.empty(C, M, dtype=torch.uint8)
    sT = torch.empty((M + 127) // 128, C, dtype=torch.float32)
    fn = lib().oracle_quantize_act_128x1_pow2 if pow2 else lib().oracle_quantize_act_128x1
    fn(_ptr(x), _dt(x), M, C, C, _ptr(qT), M, _ptr(sT), C)
    return qT, sT


def quantize_weight_128x128(w: torch.Tensor, want_t: bool = True, pow2: bool = False):
    """w [N,K] -> (q uint8 [N,K], s fp32 [ceil(N/128), ceil(K/128)], qT uint8 [K,N] or None).
    pow2: power-of-two scales."""
    w = w.contiguous()
    N, K = w.shape
    KB = (K + 127) // 128
    q = torch.empty(N, K, dtype=torch.uint8)
    s = torch.empty((N + 127) // 128, KB, dtype=torch.float32)
    qT = torch.empty(K, N, dtype=torch.uint8) if want_t else None
    fn = lib().oracle_quantize_weight_128x128_pow2 if pow2 else lib().oracle_quantize_weight_128x128
    fn(_ptr(w), _dt(w), N, K, K, _ptr(q), K, _ptr(s), KB, _ptr(qT), N)
    return q, s, qT


def exp32(x: float) -> float:
    """The fixed binary32 exp sequence of reading R27 (oracle.c oracle_exp32)."""
    return lib().oracle_exp32(x)


def rcp32(d: float) -> float:
    """The fixed binary32 reciprocal sequence of reading R27 (d in [1, 2^125))."""
    return lib().oracle_rcp32(d)


def swiglu32(g: float, u: float) -> float:
    """RN(RN(g * rcp32(RN(1 + exp32(-g)))) * u) (reading R27)."""
    return lib().oracle_swiglu32(g, u)


def swiglu_quant_1x128(H: torch.Tensor, cache: bool = True):
    """Up-projection output H float32 [M, 2I] (gate / up interleaved per 128 channels, R27) ->
    (qy uint8 [M, I], sy fp32 [I/128, M], qh uint8 [M, 2I] or None, sh fp32 [2I/128, M] or None):
    the 1x128-quantized SwiGLU output and (cache=True) the 1x128-quantized H."""
    H = H.to(torch.float32).contiguous()
    M, N2 = H.shape
    I = N2 // 2
    qy = torch.empty(M, I, dtype=torch.uint8)
    sy = torch.empty(I // 128, M, dtype=torch.float32)
    qh = torch.empty(M, N2, dtype=torch.uint8) if cache else None
    sh = torch.empty(N2 // 128, M, dtype=torch.float32) if cache else None
    lib().oracle_swiglu_quant_1x128(_ptr(H), M, I, N2, _ptr(qy), I, _ptr(sy), M, _ptr(qh), N2, _ptr(sh), M)
    return qy, sy, qh, sh


def combine_bf16(y: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    """MoE combine (R28): y BF16 [T * top_k, N] (token t's k-th expert output at row
    t * top_k + k), g FP32 [T, top_k] -> BF16 [T, N], fmaf-accumulated in k order from 0."""
    T, top_k = g.shape
    N = y.shape[1]
    y = y.to(torch.bfloat16).contiguous()
    g = g.to(torch.float32).contiguous()
    out = torch.empty(T, N, dtype=torch.bfloat16)
    lib().oracle_combine_bf16(T, top_k, N, _ptr(y), _ptr(g), _ptr(out))
    return out


def requantize_1x128_to_128x1(q: torch.Tensor, s: torch.Tensor, pow2: bool = False):
    """FP8 1x128 codes q [M,K] + scales s [ceil(K/128), M] -> dequantize (FP32) -> 128x1:
    (qT uint8 [K,M], sT fp32 [ceil(M/128), K]).  P:558."""
    q, s = q.contiguous(), s.contiguous()
    M, K = q.shape
    qT = torch.empty(K, M, dtype=torch.uint8)
    sT = torch.empty((M + 127) // 128, K, dtype=torch.float32)
    lib().oracle_requantize_1x128_to_128x1(_ptr(q), K, _ptr(s), s.shape[1], M, K, _ptr(qT), M, _ptr(sT), K, int(pow2))
    return qT, sT


def gemm(layout: int, A: torch.Tensor, sA: torch.Tensor, B: torch.Tensor, sB: torch.Tensor,
         rows: torch.Tensor | None = None, threads: int = 0) -> torch.Tensor:
    """FP64 block-scaled GEMM.  A [M,K] codes, sA [K/128, M]; B [N,K] codes;
    sB: FPROP [ceil(N/128), K/128], DGRAD [K/128, ceil(N/128)], WGRAD [K/128, N].
    Returns O float64 [len(rows) or M, N]."""
    A, B, sA, sB = A.contiguous(), B.contiguous(), sA.contiguous(), sB.contiguous()
    M, K = A.shape
    N = B.shape[0]
    assert K % 128 == 0 and B.shape[1] == K
    if rows is not None:
        rows = rows.to(torch.int64).contiguous()
    nr = M if rows is None else rows.numel()
    O = torch.empty(nr, N, dtype=torch.float64)
    lib().oracle_gemm(layout, M, N, K, _ptr(A), K, _ptr(sA), sA.shape[1], _ptr(B), K, _ptr(sB),
                      sB.shape[1], _ptr(rows), nr, _ptr(O), threads)
    return O


def grouped_gemm(offsets: torch.Tensor, A: torch.Tensor, sA: torch.Tensor, B: torch.Tensor,
                 sB: torch.Tensor, rows: torch.Tensor | None = None, threads: int = 0) -> torch.Tensor:
    """Grouped FPROP.  offsets int64 [G+1]; A [R,K]; sA [K/128, R]; B [G,N,K]; sB [G,ceil(N/128),K/128]."""
    offsets = offsets.to(torch.int64).contiguous()
    A, B, sA, sB = A.contiguous(), B.contiguous(), sA.contiguous(), sB.contiguous()
    G, N, K = B.shape
    R = A.shape[0]
    if rows is not None:
        rows = rows.to(torch.int64).contiguous()
    nr = R if rows is None else rows.numel()
    O = torch.empty(nr, N, dtype=torch.float64)
    lib().oracle_grouped_gemm(G, _ptr(offsets), N, K, _ptr(A), K, _ptr(sA), sA.shape[1], _ptr(B),
                              _ptr(sB), _ptr(rows), nr, _ptr(O), threads)
    return O


def gemm_limited_accum(A: torch.Tensor, sA: torch.Tensor, B: torch.Tensor, sB: torch.Tensor,
                       bits: int = 14, chunk: int = 32, nc: int = 0, toward_zero: bool = False,
                       threads: int = 0) -> torch.Tensor:
    """Hopper limited-accumulation emulation (R24), context only.
    A [M,K], B [N,K] codes; sA [K/128, M], sB [K/128, N] per-row scales (nc = 0 uses row 0 of
    each as one tensor-wise scale per row/column).  Returns O float64 [M,N]."""
    A, B, sA, sB = A.contiguous(), B.contiguous(), sA.contiguous(), sB.contiguous()
    M, K = A.shape
    N = B.shape[0]
    assert B.shape[1] == K and 0 < chunk <= 256
    assert nc == 0 or (nc % chunk == 0 and 128 % nc == 0)
    O = torch.empty(M, N, dtype=torch.float64)
    lib().oracle_gemm_limited_accum(M, N, K, _ptr(A), K, _ptr(sA), sA.shape[1], _ptr(B), K, _ptr(sB),
                                    sB.shape[1], bits, chunk, nc, int(toward_zero), _ptr(O), threads)
    return O


def padded_offsets(offsets: torch.Tensor) -> torch.Tensor:
    """P_e = sum_{f<e} roundup(M_f, 128): the expert-aligned token layout (reading R25)."""
    m = offsets[1:] - offsets[:-1]
    P = torch.zeros(offsets.numel(), dtype=torch.int64)
    P[1:] = torch.cumsum((m + 127) // 128 * 128, 0)
    return P


def quantize_act_128x1_grouped(x: torch.Tensor, offsets: torch.Tensor):
    """128x1 groups that restart at each expert's first token (R25): expert e's rows
    x[offsets[e]:offsets[e+1]] quantized alone with quantize_act_128x1 and placed at columns
    [P_e, P_e + M_e) of qT [C, Mp]; padding codes 0, scale rows g = P_e/128 .. P_{e+1}/128 - 1."""
    offsets = offsets.to(torch.int64)
    P = padded_offsets(offsets)
    C, Mp = x.shape[1], int(P[-1])
    qT = torch.zeros(C, Mp, dtype=torch.uint8)
    sT = torch.zeros(Mp // 128, C, dtype=torch.float32)
    for e in range(offsets.numel() - 1):
        a, b, p = int(offsets[e]), int(offsets[e + 1]), int(P[e])
        if b == a:
            continue
        q, s_ = quantize_act_128x1(x[a:b])
        qT[:, p:p + b - a] = q
        sT[p // 128:p // 128 + s_.shape[0]] = s_
    return qT, sT


def grouped_gemm_wgrad(offsets: torch.Tensor, A: torch.Tensor, sA: torch.Tensor, B: torch.Tensor,
                       sB: torch.Tensor, threads: int = 0) -> torch.Tensor:
    """dW_e = WGRAD over expert e's token columns [P_e, P_e + roundup(M_e,128)) of the expert-aligned
    layout: A = dYqT [N, Mp], sA [Mp/128, N]; B = XqT [K, Mp], sB [Mp/128, K].  Returns [G, N, K] FP64;
    an expert without tokens gets zeros."""
    offsets = offsets.to(torch.int64)
    P = padded_offsets(offsets)
    G, N, K = offsets.numel() - 1, A.shape[0], B.shape[0]
    O = torch.zeros(G, N, K, dtype=torch.float64)
    for e in range(G):
        p, q = int(P[e]), int(P[e + 1])
        if q == p:
            continue
        O[e] = gemm(2, A[:, p:q], sA[p // 128:q // 128], B[:, p:q], sB[p // 128:q // 128], threads=threads)
    return O


def rel_err_normwise(D: torch.Tensor, O: torch.Tensor) -> float:
    D = D.to(torch.float64).contiguous()
    O = O.to(torch.float64).contiguous()
    return lib().oracle_rel_err_normwise(_ptr(D), _ptr(O), O.numel())


def max_threads() -> int:
    return lib().oracle_max_threads()
