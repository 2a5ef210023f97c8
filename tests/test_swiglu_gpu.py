"""GPU parity of the SwiGLU FP8 epilogue (NEXT-2; reading R27): the up-projection
writes the 1x128-quantized SwiGLU output (the down-projection's FP8 input) and the 1x128-quantized
SwiGLU inputs (the FP8 cache) straight from its FP32 accumulators.

Closed-form operands (codes in {0, +-1, +-2}, power-of-two scales) make every accumulator an exact
binary32 value, so the oracle's H — its FP64 GEMM, exactly representable — is the kernel's own
accumulator, and codes and scales must match oracle.swiglu_quant_1x128(H) bit for bit.  Realistic
operands (quantized Gaussian activations and N(0, 0.006^2) weights) are checked against the FP64
oracle on the dequantized output.
"""
import pytest
import torch

import oracle
import paper_2412_19437_b200 as fp
import workloads as W

pytestmark = pytest.mark.gpu
DEV = "cuda"


def dev(t):
    return t.to(DEV)


def dev_scales(s):
    """[KB, n] scales on the device with the row pitch padded to a multiple of 4 (the GEMM's TMA rule)."""
    kb, n = s.shape
    buf = torch.zeros(kb, (n + 3) // 4 * 4, dtype=s.dtype, device=DEV)
    buf[:, :n] = s.to(DEV)
    return buf[:, :n]


def closed_form(M, N2, K, seed):
    A = W.codes_small(M, K, seed=seed)
    B = W.codes_small(N2, K, seed=seed + 1)
    # scales 2^-6 .. 2^-4: accumulators of a few units, where silu is far from linear
    sA = W.scales_pow2(K // 128, M, seed=seed + 2) * 2.0 ** -6
    sB = W.scales_pow2(N2 // 128, K // 128, seed=seed + 3) * 2.0 ** -4
    H = oracle.gemm(fp.FPROP, A, sA, B, sB)            # FP64, exact, binary32-representable
    H32 = H.to(torch.float32)
    assert torch.equal(H32.double(), H)
    return A, sA, B, sB, H32


def assert_bits(got, want, what):
    got, want = got.cpu(), want.cpu()
    if got.dtype == torch.float32:
        got, want = got.view(torch.int32), want.view(torch.int32)
    bad = (got != want).nonzero()
    assert bad.numel() == 0, f"{what}: {bad.shape[0]} mismatches, first {bad[:4].tolist()}"


@pytest.fixture(params=[1, 2], ids=["cta1", "pair"])
def variant(request):
    with fp.forced_variant(request.param):
        yield request.param


@pytest.mark.parametrize("M,I,K", [(256, 128, 512), (300, 256, 384), (1000, 384, 256)])
def test_swiglu_closed_form_bitexact(M, I, K, variant):
    A, sA, B, sB, H = closed_form(M, 2 * I, K, seed=M + I)
    qy, sy, qh, sh = fp.gemm_swiglu(dev(A), dev_scales(sA), dev(B), dev(sB))
    ry, rsy, rh, rsh = oracle.swiglu_quant_1x128(H)
    torch.cuda.synchronize()
    assert_bits(qy, ry, "y codes")
    assert_bits(sy, rsy, "y scales")
    assert_bits(qh, rh, "H cache codes")
    assert_bits(sh, rsh, "H cache scales")
    # the accumulators actually exercise silu's curved part
    assert (H.abs() < 8).float().mean() > 0.5


def test_swiglu_without_cache():
    A, sA, B, sB, H = closed_form(384, 512, 256, seed=3)
    qy, sy, qh, sh = fp.gemm_swiglu(dev(A), dev(sA), dev(B), dev(sB), cache=False)
    assert qh is None and sh is None
    ry, rsy, _, _ = oracle.swiglu_quant_1x128(H, cache=False)
    assert_bits(qy, ry, "y codes")
    assert_bits(sy, rsy, "y scales")


@pytest.mark.parametrize("counts", [[0, 1, 300, 128, 257, 0, 700, 40], [1000], [0, 0, 513]],
                         ids=["ragged8", "one", "empties"])
def test_grouped_swiglu_closed_form_bitexact(counts, variant):
    """MoE experts with ragged row counts: tiles cross expert ends (the lanes copy those rows out),
    empty experts, a 1-row expert."""
    G, I, K = len(counts), 256, 384
    off = torch.zeros(G + 1, dtype=torch.int64)
    off[1:] = torch.cumsum(torch.tensor(counts), 0)
    R = int(off[-1])
    A = W.codes_small(R, K, seed=11)
    sA = W.scales_pow2(K // 128, R, seed=12) * 2.0 ** -6
    B = torch.stack([W.codes_small(2 * I, K, seed=20 + e) for e in range(G)])
    sB = torch.stack([W.scales_pow2(2 * I // 128, K // 128, seed=40 + e) for e in range(G)]) * 2.0 ** -4
    H = torch.empty(R, 2 * I, dtype=torch.float32)
    for e in range(G):
        a, b = int(off[e]), int(off[e + 1])
        if b > a:
            H[a:b] = oracle.gemm(fp.FPROP, A[a:b], sA[:, a:b].contiguous(), B[e], sB[e]).to(torch.float32)
    qy, sy, qh, sh = fp.grouped_gemm_swiglu(dev(off), dev(A), dev_scales(sA), dev(B), dev(sB))
    ry, rsy, rh, rsh = oracle.swiglu_quant_1x128(H)
    torch.cuda.synchronize()
    assert_bits(qy, ry, "y codes")
    assert_bits(sy, rsy, "y scales")
    assert_bits(qh, rh, "H cache codes")
    assert_bits(sh, rsh, "H cache scales")


def test_swiglu_realistic_vs_fp64_oracle():
    """Quantized Gaussian activations x N(0, 0.006^2) weights (the expert up-projection's value
    ranges, K = 7168): the dequantized FP8 output within the E4M3 quantization error of the FP64
    SwiGLU of the FP64 GEMM, and bit-equal codes wherever the kernel's FP32 accumulators round to the
    oracle's (all but a handful of near-tie elements)."""
    M, I, K = 512, 256, 7168
    qx, sx = oracle.quantize_act_1x128(W.gaussian_act(M, K, seed=0))
    qw, sw, _ = oracle.quantize_weight_128x128(W.master_weight(2 * I, K, seed=1) * 20, want_t=False)
    H64 = oracle.gemm(fp.FPROP, qx, sx, qw, sw)
    qy, sy, _, _ = fp.gemm_swiglu(dev(qx), dev(sx), dev(qw), dev(sw), cache=False)
    ry, rsy, _, _ = oracle.swiglu_quant_1x128(H64.to(torch.float32), cache=False)
    qy, sy = qy.cpu(), sy.cpu()
    # the scales: within a few ulp (the kernel's amax comes from its own FP32 accumulators)
    assert torch.allclose(sy, rsy, rtol=1e-5, atol=0)
    assert (qy != ry).float().mean() < 0.01
    # dequantized output vs the FP64 SwiGLU
    g, u = H64.reshape(M, I // 128, 2, 128)[:, :, 0], H64.reshape(M, I // 128, 2, 128)[:, :, 1]
    y64 = (g * torch.sigmoid(g) * u).reshape(M, I)
    dq = oracle.decode_table()[qy.long()] * sy.t().repeat_interleave(128, dim=1).double()
    err = oracle.rel_err_normwise(dq, y64)
    assert err < 0.05, err            # E4M3 (3 mantissa bits) quantization error, normwise
