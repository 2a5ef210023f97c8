"""Accumulation precision: the paper's 14-bit Hopper accumulator, emulated in
the oracle, and the B200 tensor core's accumulator, characterized through the C-ABI.

PAPER.md §3.3.2: "the accumulation precision of FP8 GEMM on NVIDIA H800 GPUs is limited to
retaining around 14 bits"; for K = 4096 random matrices "a maximum relative error of nearly 2%"; fixed
by promotion to FP32 every N_C = 128 elements.  §3.5.2 gives the mechanism: fixed-point
accumulation aligned to the maximum exponent, "the highest 14 bits of each mantissa product after
sign-fill right shifting".  oracle.gemm_limited_accum emulates it (reading R24).

CPU tests pin the emulation with hand-computed cases (each value worked out below), the wide-accumulator
limit (which must reproduce the FP64 oracle GEMM), and the ladder full <= promoted <= limited at
K = 4096.  The paper's 2% is context (R18): the test checks that the two shift readings bracket it.

GPU tests (characterization, T4): the same K = 4096 problem through fp8bs_gemm_mx (the whole K in one
TMEM accumulator, no promotion) and fp8bs_gemm (promotion every 128), and a probe of how many bits of
a small addend survive next to a large one inside and across tcgen05.mma K-steps.  Measured numbers
are written to $FP8BS_ACCUM_REPORT when set (DESIGN.md quotes them).
"""
import json
import os

import pytest
import torch

import oracle

K4096 = 4096


def _code(v: float) -> int:
    return oracle.e4m3_encode(v)


def _hand(a_vals, b_vals, bits, nc=0, toward_zero=False, sa=1.0, sb=1.0, chunk=32):
    """One output element D[0,0] of the emulation for sparse rows {k: value} of A and B (K = 128)."""
    A = torch.zeros(1, 128, dtype=torch.uint8)
    B = torch.zeros(1, 128, dtype=torch.uint8)
    for k, v in a_vals.items():
        A[0, k] = _code(v)
    for k, v in b_vals.items():
        B[0, k] = _code(v)
    sA = torch.full((1, 1), sa)
    sB = torch.full((1, 1), sb)
    return float(oracle.gemm_limited_accum(A, sA, B, sB, bits=bits, chunk=chunk, nc=nc,
                                           toward_zero=toward_zero)[0, 0])


def test_limited_accum_hand_cases():
    """Terms 1 and +-2^-14 (= 2^-7 * 2^-7, E4M3 subnormals).  Max exponent 0, so with 14 retained bits
    the quantum is 2^-13: +2^-14 shifts out (floor -> 0); -2^-14 floors to -2^-13 (sign fill: the
    two's-complement shift rounds toward -inf), truncation toward zero drops it.  15 bits keep it."""
    one, small = {0: 1.0, 1: 2.0 ** -7}, {0: 1.0, 1: 2.0 ** -7}
    neg = {0: 1.0, 1: -(2.0 ** -7)}
    assert _hand(one, small, bits=14) == 1.0
    assert _hand(one, small, bits=15) == 1.0 + 2.0 ** -14
    assert _hand(neg, small, bits=14) == 1.0 - 2.0 ** -13
    assert _hand(neg, small, bits=14, toward_zero=True) == 1.0
    assert _hand(neg, small, bits=15) == 1.0 - 2.0 ** -14
    # the small term in a later MMA step (k = 64): aligned against the accumulator's exponent, same result
    late_a, late_b = {0: 1.0, 64: -(2.0 ** -7)}, {0: 1.0, 64: 2.0 ** -7}
    assert _hand(late_a, late_b, bits=14) == 1.0 - 2.0 ** -13
    # promotion every 32 products: the small term sits alone in its step and reaches FP64 intact
    assert _hand(late_a, late_b, bits=14, nc=32) == 1.0 - 2.0 ** -14
    # ... but not when it shares a step with the large one
    assert _hand(neg, small, bits=14, nc=32) == 1.0 - 2.0 ** -13
    # the scales multiply the promoted partial: 2 * 4 * (1 + 2^-14)
    assert _hand(one, small, bits=15, nc=128, sa=2.0, sb=4.0) == 8.0 * (1.0 + 2.0 ** -14)
    # the accumulator is shifted too: step 1 leaves 1 + 2^-13 (exact at E = 0); step 2 adds 1, E = 1,
    # quantum 2^-12, so the accumulator's 2^-13 bit shifts out
    assert _hand({0: 1.0, 1: 2.0 ** -7, 64: 1.0}, {0: 1.0, 1: 2.0 ** -6, 64: 1.0}, bits=14) == 2.0
    assert _hand({0: 1.0, 1: 2.0 ** -7, 64: 1.0}, {0: 1.0, 1: 2.0 ** -6, 64: 1.0}, bits=15) == 2.0 + 2.0 ** -13
    # all terms below the quantum: zero partial -> zero, exactly
    assert _hand({5: 2.0 ** -9}, {5: 2.0 ** -9}, bits=14) == 2.0 ** -18   # alone: its own exponent
    assert _hand({}, {}, bits=14) == 0.0


def _tensorwise(x: torch.Tensor):
    """Tensor-wise power-of-two scale (one scale for the whole matrix, the paper's K=4096 test setup):
    x/s is exact, so the codes are E4M3(x/s) with a single rounding."""
    amax = float(x.abs().max())
    s = 2.0 ** torch.tensor(amax / 448.0).log2().ceil().item()
    return oracle.encode_tensor((x / s).float()), s


def _k4096_problem(seed, M=64, N=64):
    g = torch.Generator().manual_seed(seed)
    X = torch.randn(M, K4096, generator=g)
    Wm = torch.randn(N, K4096, generator=g)
    qa, sa = _tensorwise(X)
    qb, sb = _tensorwise(Wm)
    KB = K4096 // 128
    return qa, torch.full((KB, M), sa), qb, torch.full((KB, N), sb)


def test_limited_accum_wide_equals_oracle_gemm():
    """With 60 retained bits no shift drops anything; what remains is the FP32 rounding of each
    step's accumulator, so the result matches the FP64 oracle GEMM to FP32 precision."""
    qa, sA, qb, sB = _k4096_problem(seed=11, M=32, N=48)
    g = torch.Generator().manual_seed(12)
    sA = sA * (1.0 + torch.randint(0, 4, sA.shape, generator=g).float())   # per-block scales too
    O = oracle.gemm(2, qa, sA, qb, sB)
    for nc in (32, 128):
        L = oracle.gemm_limited_accum(qa, sA, qb, sB, bits=60, chunk=32, nc=nc)
        assert oracle.rel_err_normwise(L, O) <= 1e-6


def test_accumulation_ladder_k4096():
    """at K = 4096, 14-bit accumulation without promotion is far worse than with
    promotion every N_C = 128, which is far worse than a wide accumulator; per seed.  The paper's
    'nearly 2%' (metric unstated, R18) lies between the floor (sign-fill) and truncate-to-zero readings."""
    for seed in range(4):
        qa, sA, qb, sB = _k4096_problem(seed)
        O = oracle.gemm(2, qa, sA, qb, sB)
        err = lambda **kw: oracle.rel_err_normwise(
            oracle.gemm_limited_accum(qa, sA, qb, sB, chunk=32, **kw), O)
        full = err(bits=60, nc=0)
        promoted = err(bits=14, nc=128)
        limited = err(bits=14, nc=0)
        limited_tz = err(bits=14, nc=0, toward_zero=True)
        assert full < 1e-6 < promoted < limited
        assert promoted < 2.5e-3            # SPEC's "promoted < 0.25%" acceptance line
        assert limited_tz < 0.02 < limited


# ------------------------------------------------------------------------------- GPU (T4) ----
def _report(key, value):
    path = os.environ.get("FP8BS_ACCUM_REPORT")
    if not path:
        return
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[key] = value
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    json.dump(data, open(path, "w"), indent=1)


@pytest.mark.gpu
def test_b200_accumulator_k4096():
    """The paper's K = 4096 experiment on B200: the MX kernel keeps all 4096 products in one TMEM
    FP32 accumulator (no promotion, unit UE8M0 scales inside the MMA); the promotion kernel adds every
    128-product partial in FP32 registers.  Both must be far below the 14-bit emulation."""
    import paper_2412_19437_b200 as fp
    out = {}
    for seed in range(2):
        qa, sA, qb, sB = _k4096_problem(seed, M=256, N=448)
        O = oracle.gemm(2, qa, sA, qb, sB)
        M, N = qa.shape[0], qb.shape[0]
        # Fprop layout with the tensor-wise scales moved onto per-row / per-block scales
        sA_d = sA.cuda()
        sB_blk = torch.full((N // 128 + (N % 128 > 0), K4096 // 128), float(sB[0, 0]), device="cuda")
        D_mx = fp.gemm(fp.FPROP, qa.cuda(), sA_d, qb.cuda(), sB_blk, out_dtype=torch.float32, mx=True)
        D_pr = fp.gemm(fp.FPROP, qa.cuda(), sA_d, qb.cuda(), sB_blk, out_dtype=torch.float32)
        torch.cuda.synchronize()
        e_mx = oracle.rel_err_normwise(D_mx.cpu().double(), O)
        e_pr = oracle.rel_err_normwise(D_pr.cpu().double(), O)
        e_14 = oracle.rel_err_normwise(oracle.gemm_limited_accum(qa, sA, qb, sB, bits=14, nc=0), O)
        out[f"seed{seed}"] = {"mx_no_promotion": e_mx, "promotion_128": e_pr, "emulated_h800_14bit": e_14}
        assert e_mx <= 1e-4 and e_pr <= 1e-4
        assert e_14 > 100 * max(e_mx, e_pr)
    _report("k4096_normwise", out)


@pytest.mark.gpu
def test_b200_accumulator_bit_probe():
    """How many bits of a small product survive next to 256 = 16 * 16 (row A[i]: 16 at k=0 and +-v at
    k = 1 (same K=32 MMA step) or k = 64 (a later step, the accumulator already holds 256); column
    B[j]: 16 at k=0 and 2^-j at k = 1 and 64).  The addend is v * 2^-j, from 2^-0 down to 2^-18, i.e.
    2^-8 .. 2^-26 relative to 256.  At least as precise as H800's 14 bits (error < 2^(8-13)), and the
    measured pattern pinned exactly."""
    import paper_2412_19437_b200 as fp
    rows = [(pos, sgn, v) for v in (1.0, 2.0 ** -9) for pos in (1, 64) for sgn in (1.0, -1.0)]
    M, N, K = 128, 128, 256
    A = torch.zeros(M, K, dtype=torch.uint8)
    B = torch.zeros(N, K, dtype=torch.uint8)
    for i, (pos, sgn, v) in enumerate(rows):
        A[i, 0] = _code(16.0)
        A[i, pos] = _code(sgn * v)
    for j in range(10):
        B[j, 0] = _code(16.0)
        B[j, 1] = B[j, 64] = _code(2.0 ** -j)
    sA = torch.ones(K // 128, M)
    sB = torch.ones(1, K // 128)
    O = oracle.gemm(fp.FPROP, A, sA, B, sB)
    res = {}
    for name, mx in (("mx", True), ("promotion", False)):
        D = fp.gemm(fp.FPROP, A.cuda(), sA.cuda(), B.cuda(), sB.cuda(), out_dtype=torch.float32, mx=mx).cpu()
        torch.cuda.synchronize()
        for i, (pos, sgn, v) in enumerate(rows):
            for j in range(10):
                exact = float(O[i, j])
                got = float(D[i, j])
                assert abs(got - exact) < 2.0 ** (8 - 13), (name, pos, sgn, v, j, got, exact)
                fp32 = float(torch.tensor(exact, dtype=torch.float64).float())
                # measured on B200: every addend FP32 can hold next to 256 survives, in
                # the same MMA step or a later one; the one tie, 256 - 2^-17, comes out 256 - 2^-16
                # (rounded toward zero, not to even), and 256 - 2^-18 comes out 256
                want = 256.0 - 2.0 ** -16 if exact == 256.0 - 2.0 ** -17 else fp32
                assert got == want, (name, pos, sgn * v * 2.0 ** -j, got - 256.0, want - 256.0)
                res.setdefault(name, []).append({"pos": pos, "addend": sgn * v * 2.0 ** -j,
                                                 "got_minus_256": got - 256.0,
                                                 "fp32_of_exact_minus_256": fp32 - 256.0})
    _report("bit_probe", res)
