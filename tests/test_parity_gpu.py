"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle on the same seeded inputs.

Bars:
  * quantizers: codes and scales BIT-EXACT;
  * GEMM, FP32 output: normwise max|D-O|/max|O| <= 1e-3 (north_star), and BIT-EXACT on the
    closed-form operands (small-integer codes, power-of-two scales: every partial sum is exact);
  * GEMM, BF16 output: D_bf16 == RNE_bf16(D_fp32) bitwise (same accumulator) and within 1 BF16
    ulp of RNE_bf16(oracle);
  * grouped: bitwise equal to per-expert dense GEMMs, and vs the oracle as above.
"""
import pytest
import torch

import oracle
import paper_2412_19437_b200 as fp
import workloads as W

pytestmark = pytest.mark.gpu
DEV = "cuda"
TOL = 1e-3


def dev(t):
    return t.to(DEV)


def dev_scales(s):
    """Device copy of a [KB, n] scale matrix with its leading dimension padded to a multiple
    of 4 (the GEMM loads 128-row scale vectors with TMA: 16-byte row pitch)."""
    kb, n = s.shape
    buf = torch.zeros(kb, (n + 3) // 4 * 4, dtype=s.dtype, device=DEV)
    buf[:, :n] = s.to(DEV)
    return buf[:, :n]


@pytest.fixture(params=[1, 2], ids=["cta1", "pair"])
def variant(request):
    """Force the GEMM tile variant (1: one CTA per 128x256 tile, 2: CTA pair per 256x256 tile) through
    the test-hooks build of the same sources, so both paths are covered at every shape."""
    with fp.forced_variant(request.param):
        yield request.param


def assert_bits_equal(got: torch.Tensor, want: torch.Tensor, what: str):
    got, want = got.cpu(), want.cpu()
    if got.dtype == torch.float32:
        got, want = got.view(torch.int32), want.view(torch.int32)
    bad = (got != want).nonzero()
    assert bad.numel() == 0, f"{what}: {bad.shape[0]} mismatches, first at {bad[:5].tolist()}"


# ------------------------------------------------------------------------ quantizers ----
ACT_CASES = [
    ("tiny_C0", 128, 256, "gauss", torch.bfloat16),
    ("ragged_tail", 300, 1096, "outlier", torch.bfloat16),     # K % 128 != 0 (short last group)
    ("odd_K_generic", 37, 1001, "gauss", torch.bfloat16),      # K % 8 != 0 -> generic kernel
    ("fp32_in", 130, 384, "outlier", torch.float32),
    ("specials", 64, 640, "special", torch.float32),
    ("C1_X", 4096, 7168, "gauss", torch.bfloat16),
    ("C3_X_outlier", 2048, 7168, "outlier", torch.bfloat16),
]


def make_act(kind, M, K, dtype, seed=0):
    if kind == "gauss":
        return W.gaussian_act(M, K, seed=seed, dtype=dtype)
    if kind == "outlier":
        return W.outlier_act(M, K, seed=seed, dtype=dtype)
    return W.special_values_act(M, K, seed=seed).to(dtype)


@pytest.mark.parametrize("name,M,K,kind,dtype", ACT_CASES, ids=[c[0] for c in ACT_CASES])
def test_quantize_act_1x128_bitexact(name, M, K, kind, dtype):
    x = make_act(kind, M, K, dtype)
    q_ref, s_ref = oracle.quantize_act_1x128(x)
    q, s = fp.quantize_act_1x128(dev(x))
    torch.cuda.synchronize()
    assert_bits_equal(s, s_ref, "scales")
    assert_bits_equal(q, q_ref, "codes")


def test_quantize_act_1x128_strided_input_and_outputs():
    x = W.outlier_act(200, 1024, seed=3)
    big = torch.zeros(200, 1024 + 64, dtype=torch.bfloat16)
    big[:, :1024] = x
    xd = dev(big)[:, :1024]
    q = torch.full((200, 1024 + 32), 0xAA, dtype=torch.uint8, device=DEV)
    s = torch.zeros(8, 256, device=DEV)
    fp.quantize_act_1x128(xd, q[:, :1024], s[:, :200])
    q_ref, s_ref = oracle.quantize_act_1x128(x)
    assert_bits_equal(q[:, :1024], q_ref, "codes")
    assert torch.all(q[:, 1024:] == 0xAA)
    assert_bits_equal(s[:, :200], s_ref, "scales")


T_CASES = [
    ("tiny", 256, 384, "gauss", torch.bfloat16),
    ("ragged_M", 300, 136, "outlier", torch.bfloat16),         # M % 128 != 0
    ("fp32_in", 260, 200, "gauss", torch.float32),
    ("odd_C_generic", 130, 37, "gauss", torch.bfloat16),
    ("C1_X", 4096, 7168, "gauss", torch.bfloat16),
]


@pytest.mark.parametrize("name,M,C,kind,dtype", T_CASES, ids=[c[0] for c in T_CASES])
def test_quantize_act_128x1_bitexact(name, M, C, kind, dtype):
    x = make_act(kind, M, C, dtype, seed=2)
    q_ref, s_ref = oracle.quantize_act_128x1(x)
    q, s = fp.quantize_act_128x1(dev(x))
    torch.cuda.synchronize()
    assert_bits_equal(s, s_ref, "scales")
    assert_bits_equal(q, q_ref, "codes")


DUAL_CASES = [
    ("tiny_C0", 128, 256, "gauss", torch.bfloat16),
    ("ragged_fused", 300, 1104, "outlier", torch.bfloat16),    # M % 128, K % 128 != 0, K % 16 == 0: fused
    ("specials_fused", 64, 640, "special", torch.bfloat16),
    ("odd_K_fallback", 37, 1001, "gauss", torch.bfloat16),     # K % 16 != 0: two-kernel fallback
    ("fp32_fallback", 130, 384, "outlier", torch.float32),
    ("C1_dY", 4096, 18432, "gauss", torch.bfloat16),
    ("C3_X_outlier", 2048, 7168, "outlier", torch.bfloat16),
]


@pytest.mark.parametrize("name,M,K,kind,dtype", DUAL_CASES, ids=[c[0] for c in DUAL_CASES])
def test_quantize_act_dual_bitexact(name, M, K, kind, dtype):
    """Both groupings from one read: bit-exact vs the oracle's 1x128 and 128x1 quantizers."""
    x = make_act(kind, M, K, dtype, seed=4)
    q_ref, s_ref = oracle.quantize_act_1x128(x)
    qT_ref, sT_ref = oracle.quantize_act_128x1(x)
    q, s, qT, sT = fp.quantize_act_dual(dev(x))
    torch.cuda.synchronize()
    assert_bits_equal(s, s_ref, "1x128 scales")
    assert_bits_equal(q, q_ref, "1x128 codes")
    assert_bits_equal(sT, sT_ref, "128x1 scales")
    assert_bits_equal(qT, qT_ref, "128x1 codes")


W_CASES = [
    ("C0", 128, 256, torch.float32),
    ("ragged", 300, 200, torch.float32),
    ("C3_kv_576", 576, 7168, torch.float32),
    ("bf16", 256, 384, torch.bfloat16),
    ("odd_generic", 130, 101, torch.float32),
]


REQ_CASES = [
    ("tiny_C0", 128, 256, "gauss"),
    ("ragged_M_and_K", 300, 1104, "outlier"),      # short last groups on both axes
    ("C1_X", 4096, 7168, "gauss"),                  # the bench's X: the Wgrad operand from cached FP8
    ("special", 256, 384, "special"),               # signed zeros, subnormals, 448 boundary, huge/tiny rows
    ("short_rows", 5, 144, "outlier"),              # fewer tokens than one lane's 16-token run
]


@pytest.mark.parametrize("name,M,K,kind", REQ_CASES, ids=[c[0] for c in REQ_CASES])
def test_requantize_1x128_to_128x1_bitexact(name, M, K, kind):
    """FP8 -> FP8 re-quantization of a cached 1x128 activation into 128x1 tiles:
    the CUDA path through the C-ABI vs the oracle, codes and scales bit-exact."""
    x = {"gauss": W.gaussian_act, "outlier": W.outlier_act, "special": W.special_values_act}[kind](M, K, seed=3)
    q, s = oracle.quantize_act_1x128(x)
    qT, sT = fp.requantize_1x128_to_128x1(dev(q), dev_scales(s))
    rqT, rsT = oracle.requantize_1x128_to_128x1(q, s)
    assert_bits_equal(qT, rqT, "requant codes")
    assert_bits_equal(sT, rsT, "requant scales")


POW2_CASES = [
    ("flat_tma", 256, 1024, "outlier", torch.bfloat16),    # the TMA 1x128 kernel
    ("ragged_generic", 300, 1100, "gauss", torch.bfloat16),  # K % 128 != 0 -> generic kernel
    ("special_fp32", 64, 384, "special", torch.float32),    # subnormal / huge groups, FP32 input
]


@pytest.mark.parametrize("name,M,K,kind,dtype", POW2_CASES, ids=[c[0] for c in POW2_CASES])
def test_quantize_act_1x128_pow2_bitexact(name, M, K, kind, dtype):
    """Power-of-two 1x128 scales: codes and scales bit-exact vs the oracle."""
    x = {"gauss": W.gaussian_act, "outlier": W.outlier_act, "special": W.special_values_act}[kind](M, K, seed=14).to(dtype)
    q, s = fp.quantize_act_1x128_pow2(dev(x))
    rq, rs = oracle.quantize_act_1x128_pow2(x)
    assert_bits_equal(q, rq, "pow2 codes")
    assert_bits_equal(s, rs, "pow2 scales")


@pytest.mark.parametrize("name,M,K,kind", REQ_CASES, ids=[c[0] for c in REQ_CASES])
def test_requantize_pow2_bitexact(name, M, K, kind):
    """The paper's re-quantization with power-of-two scales on both sides: bit-exact."""
    x = {"gauss": W.gaussian_act, "outlier": W.outlier_act, "special": W.special_values_act}[kind](M, K, seed=15)
    q, s = oracle.quantize_act_1x128_pow2(x)
    qT, sT = fp.requantize_1x128_to_128x1(dev(q), dev_scales(s), pow2=True)
    rqT, rsT = oracle.requantize_1x128_to_128x1(q, s, pow2=True)
    assert_bits_equal(qT, rqT, "pow2 requant codes")
    assert_bits_equal(sT, rsT, "pow2 requant scales")


def test_gemm_with_pow2_scales_vs_oracle():
    """Power-of-two scales feed the same block-scaled GEMM (scales are arbitrary FP32 there)."""
    M, N, K = 256, 512, 1024
    qa, sa = oracle.quantize_act_1x128_pow2(W.outlier_act(M, K, seed=16))
    qb, sb, _ = oracle.quantize_weight_128x128(W.master_weight(N, K, seed=17))
    D = fp.gemm(fp.FPROP, dev(qa), dev_scales(sa), dev(qb), dev(sb), out_dtype=torch.float32)
    O = oracle.gemm(oracle.FPROP, qa, sa, qb, sb)
    assert oracle.rel_err_normwise(D.cpu().double(), O) <= TOL


def test_requantize_matches_direct_128x1_on_exact_inputs():
    """When the 1x128 quantization is lossless (E4M3 grid values times a power of two with a 448 in
    every row group), the re-quantized tiles equal the direct 128x1 quantization of the BF16 input."""
    g = torch.Generator().manual_seed(6)
    dec = torch.arange(127, dtype=torch.uint8).view(torch.float8_e4m3fn).float()
    M, K = 256, 512
    v = dec[torch.randint(0, 127, (M, K), generator=g)] * (torch.randint(0, 2, (M, K), generator=g) * 2 - 1)
    v[:, ::128] = 448.0
    x = (v * 2.0 ** -5).to(torch.bfloat16)
    q, s = fp.quantize_act_1x128(dev(x))
    qT, sT = fp.requantize_1x128_to_128x1(q, s)
    dqT, dsT = fp.quantize_act_128x1(dev(x))
    assert_bits_equal(qT, dqT.cpu(), "requant vs direct codes")
    assert_bits_equal(sT, dsT.cpu(), "requant vs direct scales")


@pytest.mark.parametrize("name,N,K,dtype", W_CASES, ids=[c[0] for c in W_CASES])
def test_quantize_weight_bitexact(name, N, K, dtype):
    w = W.master_weight(N, K, seed=1, dtype=dtype)
    q_ref, s_ref, qT_ref = oracle.quantize_weight_128x128(w)
    q, s, qT = fp.quantize_weight_128x128(dev(w))
    torch.cuda.synchronize()
    assert_bits_equal(s, s_ref, "scales")
    assert_bits_equal(q, q_ref, "codes")
    assert_bits_equal(qT, qT_ref, "transposed codes")


# ------------------------------------------------------------------------------- GEMM ----
def scale_b_shape(layout, N, K):
    KB, NB = K // 128, (N + 127) // 128
    return {fp.FPROP: (NB, KB), fp.DGRAD: (KB, NB), fp.WGRAD: (KB, N)}[layout]


GEMM_SHAPES = [(128, 128, 256), (256, 512, 512), (200, 136, 384), (300, 520, 1024), (1000, 264, 256), (520, 1160, 640)]


@pytest.mark.parametrize("layout", [fp.FPROP, fp.DGRAD, fp.WGRAD], ids=["fprop", "dgrad", "wgrad"])
@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_closed_form_bitexact(layout, M, N, K, variant):
    A = W.codes_small(M, K, seed=M)
    B = W.codes_small(N, K, seed=N + 1)
    sA = W.scales_pow2(K // 128, M, seed=3)
    sB = W.scales_pow2(*scale_b_shape(layout, N, K), seed=4)
    O = oracle.gemm(layout, A, sA, B, sB)
    D = fp.gemm(layout, dev(A), dev(sA), dev(B), dev(sB), out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert_bits_equal(D, O.to(torch.float32), "closed-form GEMM")


@pytest.mark.parametrize("layout", [fp.FPROP, fp.DGRAD, fp.WGRAD], ids=["fprop", "dgrad", "wgrad"])
@pytest.mark.parametrize("N", [320, 576], ids=["n320", "n576"])
def test_gemm_half_tiles_with_several_tiles_per_cta(layout, N, variant):
    """Regression: a last column tile with one active N = 128 half (N % 256 in (0, 128]) inside a
    persistent CTA's walk over SEVERAL tiles.  The inactive half's issuer used to jump KB stages
    ahead and then pass a full-barrier parity wait a phase early (C3 kv-lora, N = 576, crashed).
    8192 rows give 192 single-CTA tiles / 96 pair tiles: more than one per CTA (cluster)."""
    M, K = 8192, 512
    A = W.codes_small(M, K, seed=N)
    B = W.codes_small(N, K, seed=N + 1)
    sA = W.scales_pow2(K // 128, M, seed=5)
    sB = W.scales_pow2(*scale_b_shape(layout, N, K), seed=6)
    D = fp.gemm(layout, dev(A), dev(sA), dev(B), dev(sB), out_dtype=torch.float32)
    O = oracle.gemm(layout, A, sA, B, sB)
    assert_bits_equal(D, O.to(torch.float32), "closed-form GEMM, half tiles")


def quantized_operands(layout, M, N, K, seed=0):
    """Operands as the Linear layer produces them (quantized by the ORACLE, so the GEMM parity
    does not depend on the GPU quantizers)."""
    if layout == fp.FPROP:
        qa, sa = oracle.quantize_act_1x128(W.outlier_act(M, K, seed=seed))
        qb, sb, _ = oracle.quantize_weight_128x128(W.master_weight(N, K, seed=seed + 1))
    elif layout == fp.DGRAD:
        qa, sa = oracle.quantize_act_1x128(W.grad_out(M, K, seed=seed))
        _, sw, qt = oracle.quantize_weight_128x128(W.master_weight(K, N, seed=seed + 1))   # W [out=K, in=N]
        qb, sb = qt, sw
    else:
        qa, sa = oracle.quantize_act_128x1(W.grad_out(K, M, seed=seed))        # dY [T=K, out=M]
        qb, sb = oracle.quantize_act_128x1(W.gaussian_act(K, N, seed=seed + 1))  # X [T=K, in=N]
    return qa, sa, qb, sb


@pytest.mark.parametrize("layout", [fp.FPROP, fp.DGRAD, fp.WGRAD], ids=["fprop", "dgrad", "wgrad"])
@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_vs_oracle_fp32(layout, M, N, K, variant):
    qa, sa, qb, sb = quantized_operands(layout, M, N, K)
    O = oracle.gemm(layout, qa, sa, qb, sb)
    D = fp.gemm(layout, dev(qa), dev(sa), dev(qb), dev(sb), out_dtype=torch.float32)
    err = oracle.rel_err_normwise(D.cpu().double(), O)
    assert err <= TOL, err


@pytest.mark.parametrize("layout", [fp.FPROP, fp.DGRAD], ids=["fprop", "dgrad"])
def test_gemm_bf16_output(layout):
    M, N, K = 300, 520, 1024
    qa, sa, qb, sb = quantized_operands(layout, M, N, K, seed=5)
    args = (layout, dev(qa), dev(sa), dev(qb), dev(sb))
    D32 = fp.gemm(*args, out_dtype=torch.float32)
    D16 = fp.gemm(*args, out_dtype=torch.bfloat16)
    assert_bits_equal(D16.view(torch.int16), D32.cpu().to(torch.bfloat16).view(torch.int16), "bf16 == RNE(fp32)")
    O = oracle.gemm(layout, qa, sa, qb, sb)
    ref = O.to(torch.bfloat16).float()
    got = D16.cpu().float()
    ulp = torch.abs(ref) * 2.0 ** -7 + 1e-30      # one BF16 ulp (8 significant bits) bound
    assert torch.all(torch.abs(got - ref) <= ulp + 1e-6 * O.abs().max().item())


def test_wgrad_accumulate():
    M, N, K = 256, 264, 512
    qa, sa, qb, sb = quantized_operands(fp.WGRAD, M, N, K, seed=9)
    D0 = torch.randn(M, N, generator=torch.Generator().manual_seed(1))
    D = dev(D0.clone())
    fp.gemm(fp.WGRAD, dev(qa), dev(sa), dev(qb), dev(sb), out=D, accumulate=True)
    O = oracle.gemm(fp.WGRAD, qa, sa, qb, sb) + D0.double()
    assert oracle.rel_err_normwise(D.cpu().double(), O) <= TOL


def test_gemm_identity_gives_dequant():
    # identity x X = dequant(quant(X)) exactly (codes 1.0 on the diagonal, scale 1).
    x = W.outlier_act(256, 512, seed=2)
    q, s = oracle.quantize_act_1x128(x)
    I = torch.zeros(512, 512, dtype=torch.uint8)
    I[torch.arange(512), torch.arange(512)] = 0x38
    sI = torch.ones(4, 4)
    D = fp.gemm(fp.FPROP, dev(q), dev(s), dev(I), dev(sI), out_dtype=torch.float32)
    O = oracle.gemm(fp.FPROP, q, s, I, sI)
    assert_bits_equal(D, O.to(torch.float32), "identity")


@pytest.mark.parametrize("layout", [fp.FPROP, fp.DGRAD, fp.WGRAD], ids=["fprop", "dgrad", "wgrad"])
def test_gemm_C1_full_size_sampled_rows(layout):
    """BASELINE configs[1] at full size, in the launch configuration bench.py times; the oracle
    computes a sample of rows (first / last tile rows and random rows)."""
    T, IN, OUT = 4096, 7168, 18432
    M, N, K = {fp.FPROP: (T, OUT, IN), fp.DGRAD: (T, IN, OUT), fp.WGRAD: (OUT, IN, T)}[layout]
    qa, sa, qb, sb = quantized_operands(layout, M, N, K, seed=11)
    D = fp.gemm(layout, dev(qa), dev(sa), dev(qb), dev(sb), out_dtype=torch.float32).cpu()
    rows = torch.cat([torch.tensor([0, 127, 128, M - 1]),
                      torch.randint(0, M, (8,), generator=torch.Generator().manual_seed(0))])
    O = oracle.gemm(layout, qa, sa, qb, sb, rows=rows)
    assert oracle.rel_err_normwise(D[rows].double(), O) <= TOL


# ---------------------------------------------------------------------------- grouped ----
def grouped_case(counts, N, K, seed=0):
    offsets = torch.zeros(len(counts) + 1, dtype=torch.int64)
    offsets[1:] = torch.cumsum(torch.tensor(counts, dtype=torch.int64), 0)
    R = int(offsets[-1])
    qa, sa = oracle.quantize_act_1x128(W.gaussian_act(R, K, seed=seed))
    G = len(counts)
    w = W.expert_weights(G, N, K, seed=seed + 1, dtype=torch.float32)
    qb = torch.empty(G, N, K, dtype=torch.uint8)
    sb = torch.empty(G, (N + 127) // 128, K // 128)
    for e in range(G):
        qb[e], sb[e], _ = oracle.quantize_weight_128x128(w[e], want_t=False)
    return offsets, qa, sa, qb, sb


# "fold": expert ends on both sides of the folded-tile boundary (a CTA-pair tile whose expert ends within
# its first 128 rows runs as an M = 128 MMA, 64 rows per CTA; gemm.cu kFold)
GROUPED_COUNTS = [[0, 7, 130, 1, 64, 0, 300], [128, 128, 128], [5], [0, 0, 257], [127, 128, 129, 255, 320, 384, 385]]


@pytest.mark.parametrize("counts", GROUPED_COUNTS, ids=["mixed", "three128", "five", "lead0", "fold"])
def test_grouped_vs_dense_bitwise_and_oracle(counts, variant):
    N, K = 264, 512
    offsets, qa, sa, qb, sb = grouped_case(counts, N, K)
    D = fp.grouped_gemm(dev(offsets), dev(qa), dev_scales(sa), dev(qb), dev(sb), out_dtype=torch.float32)
    torch.cuda.synchronize()
    for e in range(len(counts)):
        a, b = int(offsets[e]), int(offsets[e + 1])
        if a == b:
            continue
        De = fp.gemm(fp.FPROP, dev(qa[a:b].contiguous()), dev_scales(sa[:, a:b].contiguous()), dev(qb[e]), dev(sb[e]),
                     out_dtype=torch.float32)
        assert_bits_equal(D[a:b], De.cpu(), f"expert {e}")
    O = oracle.grouped_gemm(offsets, qa, sa, qb, sb)
    assert oracle.rel_err_normwise(D.cpu().double(), O) <= TOL
    # BF16 output (the bench's) is the RNE of the FP32 output, folded tiles included
    Db = fp.grouped_gemm(dev(offsets), dev(qa), dev_scales(sa), dev(qb), dev(sb), out_dtype=torch.bfloat16)
    assert_bits_equal(Db, D.to(torch.bfloat16), "bf16 == RNE(fp32)")


@pytest.mark.parametrize("counts", [[0, 7, 130, 1, 64, 0, 300], [256, 256], [3], [127, 128, 129, 255, 320, 384, 385]],
                         ids=["mixed", "two256", "three", "fold"])
def test_grouped_dgrad_vs_dense_bitwise_and_oracle(counts, variant):
    """MoE expert Dgrad (fp8bs_grouped_gemm_dgrad): per expert, dX_e = dY_e (1x128 along the expert's
    output channels) x W_e through WqT_e and the expert's sW read [out-block][in-block]; bitwise equal to
    the dense DGRAD GEMM on each segment, and within 1e-3 of the oracle."""
    G, out_c, in_c = len(counts), 384, 264           # expert W_e [out, in]; contraction = out
    offsets = torch.zeros(G + 1, dtype=torch.int64)
    offsets[1:] = torch.cumsum(torch.tensor(counts, dtype=torch.int64), 0)
    R = int(offsets[-1])
    qa, sa = oracle.quantize_act_1x128(W.grad_out(R, out_c, seed=9))
    w = W.expert_weights(G, out_c, in_c, seed=10, dtype=torch.float32)
    qbT = torch.empty(G, in_c, out_c, dtype=torch.uint8)
    sb = torch.empty(G, out_c // 128, (in_c + 127) // 128)
    for e in range(G):
        _, sb[e], qbT[e] = oracle.quantize_weight_128x128(w[e])
    D = fp.grouped_gemm(dev(offsets), dev(qa), dev_scales(sa), dev(qbT), dev(sb), out_dtype=torch.float32,
                        layout=fp.DGRAD)
    torch.cuda.synchronize()
    for e in range(G):
        a, b = int(offsets[e]), int(offsets[e + 1])
        if a == b:
            continue
        De = fp.gemm(fp.DGRAD, dev(qa[a:b].contiguous()), dev_scales(sa[:, a:b].contiguous()), dev(qbT[e]), dev(sb[e]),
                     out_dtype=torch.float32)
        assert_bits_equal(D[a:b], De.cpu(), f"expert {e}")
        O = oracle.gemm(oracle.DGRAD, qa[a:b].contiguous(), sa[:, a:b].contiguous(), qbT[e], sb[e])
        assert oracle.rel_err_normwise(D[a:b].cpu().double(), O) <= TOL


def test_grouped_C2_shape_sampled():
    """BASELINE configs[2] per-expert shape (K=7168, N=2048, ~128 rows/expert, top-8 uniform
    routing) over 32 experts so the CPU oracle stays within seconds; bench.py runs all 256."""
    T, E, topk, N, K = 512, 32, 8, 2048, 7168
    routes = W.route_uniform(T, E, topk, seed=3)
    tok, offsets = W.group_rows(routes, E)
    x = W.gaussian_act(T, K, seed=0)
    qx, sx = oracle.quantize_act_1x128(x)
    qa = qx[tok].contiguous()                       # dispatch of FP8 rows (bit-exact: scales are per row)
    sa = sx[:, tok].contiguous()
    w = W.expert_weights(E, N, K, seed=1, dtype=torch.bfloat16)
    qb = torch.empty(E, N, K, dtype=torch.uint8)
    sb = torch.empty(E, N // 128, K // 128)
    for e in range(E):
        qb[e], sb[e], _ = oracle.quantize_weight_128x128(w[e], want_t=False)
    D = fp.grouped_gemm(dev(offsets), dev(qa), dev_scales(sa), dev(qb), dev(sb), out_dtype=torch.float32).cpu()
    R = int(offsets[-1])
    rows = torch.cat([offsets[:-1][:8], torch.randint(0, R, (8,), generator=torch.Generator().manual_seed(1))])
    O = oracle.grouped_gemm(offsets, qa, sa, qb, sb, rows=rows)
    assert oracle.rel_err_normwise(D[rows].double(), O) <= TOL


@pytest.mark.parametrize("layout", [fp.FPROP, fp.DGRAD, fp.WGRAD], ids=["fprop", "dgrad", "wgrad"])
def test_gemm_C1_full_size_deterministic(layout):
    """Repeated launches at the bench's full C1 size are bitwise identical.  This is the check that
    caught a scale-ring race (a stage refilled by TMA before the last ld.shared of its per-column
    Wgrad scales completed; fixed with a proxy fence before the release, gemm.cu release_scales):
    the outputs stayed within tolerance in most runs but differed between runs."""
    T, IN, OUT = 4096, 7168, 18432
    M, N, K = {fp.FPROP: (T, OUT, IN), fp.DGRAD: (T, IN, OUT), fp.WGRAD: (OUT, IN, T)}[layout]
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device="cuda", generator=g)
    B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device="cuda", generator=g)
    sA = torch.rand(K // 128, M, device="cuda", generator=g) + 0.5
    sB = {fp.FPROP: (N // 128, K // 128), fp.DGRAD: (K // 128, N // 128), fp.WGRAD: (K // 128, N)}[layout]
    sB = torch.rand(*sB, device="cuda", generator=g) + 0.5
    ref = fp.gemm(layout, A, sA, B, sB, out_dtype=torch.float32)
    for _ in range(4):
        D = fp.gemm(layout, A, sA, B, sB, out_dtype=torch.float32)
        assert torch.equal(D.view(torch.int32), ref.view(torch.int32)), "nondeterministic GEMM output"


# ------------------------------------------- power-of-two scales on the MMA's block scaling ----
@pytest.mark.parametrize("layout", [fp.FPROP, fp.DGRAD, fp.WGRAD], ids=["fprop", "dgrad", "wgrad"])
@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_mx_closed_form_bitexact(layout, M, N, K):
    """fp8bs_gemm_mx (UE8M0 block-scaled tcgen05.mma, no promotion) on the closed-form operands:
    small-integer codes and power-of-two scales make every partial sum exact, so the FP32 output
    equals the oracle bit for bit; ragged M and N (partial 128 x 224 tiles)."""
    A = W.codes_small(M, K, seed=M)
    B = W.codes_small(N, K, seed=N + 1)
    sA = W.scales_pow2(K // 128, M, seed=3)
    sB = W.scales_pow2(*scale_b_shape(layout, N, K), seed=4)
    O = oracle.gemm(layout, A, sA, B, sB)
    D = fp.gemm(layout, dev(A), dev_scales(sA), dev(B), dev(sB), out_dtype=torch.float32, mx=True)
    torch.cuda.synchronize()
    assert_bits_equal(D, O.to(torch.float32), "closed-form MX GEMM")


@pytest.mark.parametrize("layout", [fp.FPROP, fp.DGRAD], ids=["fprop", "dgrad"])
def test_gemm_mx_pow2_quantized_vs_oracle_and_bf16(layout):
    """Activations quantized with power-of-two 1x128 scales and pow2 weight scales:
    within 1e-3 of the FP64 oracle; the BF16 output is the RNE of the same kernel's FP32 output."""
    M, N, K = 640, 1000, 1536
    qa, sa = oracle.quantize_act_1x128_pow2(W.outlier_act(M, K, seed=21))
    qb = W.codes_small(N, K, seed=22)
    sb = W.scales_pow2(*scale_b_shape(layout, N, K), seed=23) * 2.0 ** -9
    O = oracle.gemm(layout, qa, sa, qb, sb)
    D = fp.gemm(layout, dev(qa), dev_scales(sa), dev(qb), dev(sb), out_dtype=torch.float32, mx=True)
    Db = fp.gemm(layout, dev(qa), dev_scales(sa), dev(qb), dev(sb), out_dtype=torch.bfloat16, mx=True)
    torch.cuda.synchronize()
    assert oracle.rel_err_normwise(D.cpu().double(), O) <= TOL
    assert torch.equal(Db.cpu().view(torch.int16), D.cpu().to(torch.bfloat16).view(torch.int16))


def test_gemm_mx_wgrad_accumulate():
    M, N, K = 384, 448, 512
    A = W.codes_small(M, K, seed=31)
    B = W.codes_small(N, K, seed=32)
    sA = W.scales_pow2(K // 128, M, seed=33)
    sB = W.scales_pow2(K // 128, N, seed=34)
    O = oracle.gemm(fp.WGRAD, A, sA, B, sB)
    D = torch.full((M, N), 3.0, device=DEV)
    fp.gemm(fp.WGRAD, dev(A), dev_scales(sA), dev(B), dev_scales(sB), out=D, accumulate=True, mx=True)
    torch.cuda.synchronize()
    assert_bits_equal(D, (O + 3.0).to(torch.float32), "MX Wgrad accumulate")


# --------------------------------------------- power-of-two recipe, whole layer (NEXT-1) ----
@pytest.mark.parametrize("name,M,K,kind,dtype", DUAL_CASES[:5], ids=[c[0] for c in DUAL_CASES[:5]])
def test_quantize_act_dual_pow2_bitexact(name, M, K, kind, dtype):
    """Both groupings with power-of-two scales: bit-exact vs the oracle's pow2 1x128
    and 128x1 quantizers, fused kernel and two-pass fallback."""
    x = make_act(kind, M, K, dtype, seed=5)
    q_ref, s_ref = oracle.quantize_act_1x128_pow2(x)
    qT_ref, sT_ref = oracle.quantize_act_128x1(x, pow2=True)
    q, s, qT, sT = fp.quantize_act_dual(dev(x), pow2=True)
    torch.cuda.synchronize()
    assert_bits_equal(s, s_ref, "pow2 1x128 scales")
    assert_bits_equal(q, q_ref, "pow2 1x128 codes")
    assert_bits_equal(sT, sT_ref, "pow2 128x1 scales")
    assert_bits_equal(qT, qT_ref, "pow2 128x1 codes")


@pytest.mark.parametrize("name,N,K,dtype", W_CASES, ids=[c[0] for c in W_CASES])
def test_quantize_weight_pow2_bitexact(name, N, K, dtype):
    w = W.master_weight(N, K, seed=2, dtype=dtype)
    q_ref, s_ref, qT_ref = oracle.quantize_weight_128x128(w, pow2=True)
    q, s, qT = fp.quantize_weight_128x128(dev(w), pow2=True)
    torch.cuda.synchronize()
    assert_bits_equal(s, s_ref, "pow2 scales")
    assert_bits_equal(q, q_ref, "pow2 codes")
    assert_bits_equal(qT, qT_ref, "pow2 transposed codes")


@pytest.mark.parametrize("T,IN,OUT", [(256, 384, 640), (384, 1152, 520)])
def test_pow2_training_step_through_mx(T, IN, OUT):
    """One FP8 Linear training step on the power-of-two recipe, every step on the GPU: dual pow2
    quantization of X and dY, pow2 weight quantization, Fprop / Dgrad / Wgrad on the UE8M0 GEMM.
    Quantized operands bit-exact vs the oracle; each GEMM within 1e-3 of the oracle's FP64 GEMM on the
    oracle's codes."""
    x = W.outlier_act(T, IN, seed=41)
    dy = W.gaussian_act(T, OUT, seed=42)
    w = W.master_weight(OUT, IN, seed=43)
    xq, xs, xqT, xsT = fp.quantize_act_dual(dev(x), pow2=True)
    dq, ds, dqT, dsT = fp.quantize_act_dual(dev(dy), pow2=True)
    wq, ws, wqT = fp.quantize_weight_128x128(dev(w), pow2=True)
    y = fp.gemm(fp.FPROP, xq, xs, wq, ws, out_dtype=torch.float32, mx=True)
    dx = fp.gemm(fp.DGRAD, dq, ds, wqT, ws, out_dtype=torch.float32, mx=True) if OUT % 128 == 0 else None
    dw = fp.gemm(fp.WGRAD, dqT, dsT, xqT, xsT, out_dtype=torch.float32, mx=True) if T % 128 == 0 else None
    torch.cuda.synchronize()
    rxq, rxs = oracle.quantize_act_1x128_pow2(x)
    rwq, rws, rwqT = oracle.quantize_weight_128x128(w, pow2=True)
    assert_bits_equal(xq, rxq, "X codes")
    assert_bits_equal(wq, rwq, "W codes")
    assert oracle.rel_err_normwise(y.cpu().double(), oracle.gemm(fp.FPROP, rxq, rxs, rwq, rws)) <= TOL
    if dx is not None:
        rdq, rds = oracle.quantize_act_1x128_pow2(dy)
        assert_bits_equal(dq, rdq, "dY codes")
        O = oracle.gemm(fp.DGRAD, rdq, rds, rwqT, rws)
        assert oracle.rel_err_normwise(dx.cpu().double(), O) <= TOL
    if dw is not None:
        rdqT, rdsT = oracle.quantize_act_128x1(dy, pow2=True)
        rxqT, rxsT = oracle.quantize_act_128x1(x, pow2=True)
        assert_bits_equal(dqT, rdqT, "dY^T codes")
        O = oracle.gemm(fp.WGRAD, rdqT, rdsT, rxqT, rxsT)
        assert oracle.rel_err_normwise(dw.cpu().double(), O) <= TOL


def grouped_case_pow2(counts, N, K, seed=0):
    offsets = torch.zeros(len(counts) + 1, dtype=torch.int64)
    offsets[1:] = torch.cumsum(torch.tensor(counts, dtype=torch.int64), 0)
    R = int(offsets[-1])
    qa, sa = oracle.quantize_act_1x128_pow2(W.outlier_act(R, K, seed=seed))
    G = len(counts)
    w = W.expert_weights(G, N, K, seed=seed + 1, dtype=torch.float32)
    qb = torch.empty(G, N, K, dtype=torch.uint8)
    sb = torch.empty(G, (N + 127) // 128, K // 128)
    for e in range(G):
        qb[e], sb[e], _ = oracle.quantize_weight_128x128(w[e], want_t=False, pow2=True)
    return offsets, qa, sa, qb, sb


# experts averaging >= 256 rows run on CTA pairs with 2-CTA block-scaled MMAs ("two256", "big-ragged")
GROUPED_MX_COUNTS = [[0, 7, 130, 1, 64, 0, 300], [256, 256], [3], [0, 0, 257],
                     [int(c) for c in torch.randint(0, 200, (40,), generator=torch.Generator().manual_seed(5))],
                     [300, 700, 0, 513, 1024, 33]]


@pytest.mark.parametrize("counts", GROUPED_MX_COUNTS, ids=["mixed", "two256", "three", "lead0", "e40", "big-ragged"])
def test_grouped_mx_vs_dense_mx_bitwise_and_oracle(counts):
    """MoE expert Fprop on UE8M0 block scaling (fp8bs_grouped_gemm_mx), power-of-two scales: per
    expert bitwise equal to the dense fp8bs_gemm_mx on its segment (experts ending inside a 32-row
    store block included), within 1e-3 of the oracle, BF16 = RNE of the FP32 output."""
    N, K = 264, 512
    offsets, qa, sa, qb, sb = grouped_case_pow2(counts, N, K, seed=7)
    D = fp.grouped_gemm(dev(offsets), dev(qa), dev_scales(sa), dev(qb), dev(sb), out_dtype=torch.float32, mx=True)
    Db = fp.grouped_gemm(dev(offsets), dev(qa), dev_scales(sa), dev(qb), dev(sb), out_dtype=torch.bfloat16, mx=True)
    torch.cuda.synchronize()
    for e in range(len(counts)):
        a, b = int(offsets[e]), int(offsets[e + 1])
        if a == b:
            continue
        De = fp.gemm(fp.FPROP, dev(qa[a:b].contiguous()), dev_scales(sa[:, a:b].contiguous()), dev(qb[e]), dev(sb[e]),
                     out_dtype=torch.float32, mx=True)
        assert_bits_equal(D[a:b], De.cpu(), f"expert {e}")
    O = oracle.grouped_gemm(offsets, qa, sa, qb, sb)
    assert oracle.rel_err_normwise(D.cpu().double(), O) <= TOL
    assert torch.equal(Db.cpu().view(torch.int16), D.cpu().to(torch.bfloat16).view(torch.int16))


@pytest.mark.parametrize("counts", [[0, 1, 300, 128, 257, 0, 40], [700], [600, 0, 257, 1300]], ids=["ragged", "one", "big-pairs"])
def test_grouped_dgrad_mx_closed_form_bitexact(counts):
    """MoE expert Dgrad on UE8M0 block scaling (fp8bs_grouped_gemm_dgrad_mx, NEXT-1): closed-form
    operands (codes {0, +-1, +-2}, power-of-two scales) keep every product and sum exact, so each
    expert's rows equal the oracle's DGRAD on its segment bit for bit, and the dense fp8bs_gemm_mx
    DGRAD on the segment."""
    G, out_c, in_c = len(counts), 384, 264                # contraction = out
    offsets = torch.zeros(G + 1, dtype=torch.int64)
    offsets[1:] = torch.cumsum(torch.tensor(counts, dtype=torch.int64), 0)
    R = int(offsets[-1])
    qa = W.codes_small(R, out_c, seed=3)
    sa = W.scales_pow2(out_c // 128, R, seed=4)
    qbT = torch.stack([W.codes_small(in_c, out_c, seed=10 + e) for e in range(G)])
    sb = torch.stack([W.scales_pow2(out_c // 128, (in_c + 127) // 128, seed=30 + e) for e in range(G)])
    D = fp.grouped_gemm(dev(offsets), dev(qa), dev_scales(sa), dev(qbT), dev(sb), out_dtype=torch.float32,
                        layout=fp.DGRAD, mx=True)
    torch.cuda.synchronize()
    for e in range(G):
        a, b = int(offsets[e]), int(offsets[e + 1])
        if a == b:
            continue
        O = oracle.gemm(oracle.DGRAD, qa[a:b].contiguous(), sa[:, a:b].contiguous(), qbT[e], sb[e])
        assert_bits_equal(D[a:b], O.to(torch.float32), f"expert {e} vs oracle")
        De = fp.gemm(fp.DGRAD, dev(qa[a:b].contiguous()), dev_scales(sa[:, a:b].contiguous()), dev(qbT[e]), dev(sb[e]),
                     out_dtype=torch.float32, mx=True)
        assert_bits_equal(D[a:b], De.cpu(), f"expert {e} vs dense mx")
