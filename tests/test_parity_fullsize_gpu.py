"""GPU parity at the configs the bench times (BASELINE configs[1], [3], [4]) and on non-finite inputs.

The CUDA path (through the C-ABI) against the CPU oracle on the same seeded inputs:
  * C1 (dense FFN up-projection, 4096 x 7168 -> 18432), all three layouts, both tile variants, at the
    real contraction lengths (7168, 18432, 4096): the closed-form operands (codes of {0, +-1, +-2},
    scales in {1, 2, 4}) keep every partial and promoted sum an integer below 2^24, so the FP32 output
    must equal the oracle BIT FOR BIT on sampled rows that cover every 128-row block;
  * C1 BF16 output: the whole D_bf16 == RNE(D_fp32) of the same kernel, and <= 1 BF16 ulp of
    RNE(oracle) on sampled rows (R14);
  * C3 (MLA q-lora / kv-lora projections, heavy-outlier X): within 1e-3 on sampled rows;
  * C4 (256 experts, K = 7168, N = 2048, 65536 tokens x top-8, skewed routing, 524288 rows) in the
    launch configuration bench.py times: sampled rows of every 16th expert within 1e-3 of the oracle,
    bitwise equal to the dense GEMM on single experts, and the expert-parallel split (G = 2, 4, 8
    contiguous expert shards, each its own grouped launch) bitwise equal to G = 1;
  * NaN and +-Inf inputs (reading R6) through every quantizer path, bit-exact.
"""
import pytest
import torch

import oracle
import paper_2412_19437_b200 as fp
import workloads as W

pytestmark = pytest.mark.gpu
DEV = "cuda"
TOL = 1e-3
T, IN, OUT = 4096, 7168, 18432


def dev(t):
    return t.to(DEV)


def dev_scales(s):
    kb, n = s.shape
    buf = torch.zeros(kb, (n + 3) // 4 * 4, dtype=s.dtype, device=DEV)
    buf[:, :n] = s.to(DEV)
    return buf[:, :n]


def assert_bits_equal(got, want, what):
    got, want = got.cpu(), want.cpu()
    if got.dtype == torch.float32:
        got, want = got.view(torch.int32), want.view(torch.int32)
    elif got.dtype == torch.bfloat16:
        got, want = got.view(torch.int16), want.view(torch.int16)
    bad = (got != want).nonzero()
    assert bad.numel() == 0, f"{what}: {bad.shape[0]} mismatches, first at {bad[:5].tolist()}"


@pytest.fixture(params=[1, 2], ids=["cta1", "pair"])
def variant(request):
    """Force the GEMM tile variant (1: one CTA per 128x256 tile, 2: CTA pair per 256x256 tile) through
    the test-hooks build of the same sources, so both paths are covered at every shape."""
    with fp.forced_variant(request.param):
        yield request.param


def block_rows(M, seed, per_block=2):
    """Two random rows in every 128-row block, plus the first and last row."""
    g = torch.Generator().manual_seed(seed)
    nb = (M + 127) // 128
    r = [torch.tensor([0, M - 1])]
    for b in range(nb):
        lo, hi = b * 128, min(M, b * 128 + 128)
        r.append(torch.randint(lo, hi, (per_block,), generator=g))
    return torch.unique(torch.cat(r))


C1_SHAPES = {fp.FPROP: (T, OUT, IN), fp.DGRAD: (T, IN, OUT), fp.WGRAD: (OUT, IN, T)}


def scale_b_shape(layout, N, K):
    KB, NB = K // 128, (N + 127) // 128
    return {fp.FPROP: (NB, KB), fp.DGRAD: (KB, NB), fp.WGRAD: (KB, N)}[layout]


# ------------------------------------------------------------------------------ C1 ----
@pytest.mark.parametrize("layout", [fp.FPROP, fp.DGRAD, fp.WGRAD], ids=["fprop", "dgrad", "wgrad"])
def test_C1_closed_form_bitexact_full_contraction(layout, variant):
    M, N, K = C1_SHAPES[layout]
    A = W.codes_small(M, K, seed=101)
    B = W.codes_small(N, K, seed=102)
    sA = W.scales_pow2(K // 128, M, seed=103)
    sB = W.scales_pow2(*scale_b_shape(layout, N, K), seed=104)
    D = fp.gemm(layout, dev(A), dev_scales(sA), dev(B), dev_scales(sB), out_dtype=torch.float32)
    rows = block_rows(M, seed=layout)
    Dr = D[dev(rows)].cpu()
    del D
    O = oracle.gemm(layout, A, sA, B, sB, rows=rows)
    assert_bits_equal(Dr, O.to(torch.float32), f"C1 closed form layout {layout}")


@pytest.mark.parametrize("layout", [fp.FPROP, fp.DGRAD], ids=["fprop", "dgrad"])
def test_C1_bf16_output_full_size(layout):
    """The benched BF16 output at full C1 size: every element RNE of the same kernel's FP32 output;
    sampled rows within one BF16 ulp of RNE(oracle)."""
    M, N, K = C1_SHAPES[layout]
    if layout == fp.FPROP:
        qa, sa = oracle.quantize_act_1x128(W.gaussian_act(M, K, seed=0))
        qb, sb, _ = oracle.quantize_weight_128x128(W.master_weight(N, K, seed=1), want_t=False)
    else:
        qa, sa = oracle.quantize_act_1x128(W.grad_out(M, K, seed=2))
        _, sb, qb = oracle.quantize_weight_128x128(W.master_weight(K, N, seed=1))
    args = (layout, dev(qa), dev_scales(sa), dev(qb), dev(sb))
    D32 = fp.gemm(*args, out_dtype=torch.float32)
    D16 = fp.gemm(*args, out_dtype=torch.bfloat16)
    assert torch.equal(D16.view(torch.int16), D32.to(torch.bfloat16).view(torch.int16)), "bf16 != RNE(fp32)"
    rows = block_rows(M, seed=7, per_block=1)
    got = D16[dev(rows)].cpu().float()
    del D32, D16
    O = oracle.gemm(layout, qa, sa, qb, sb, rows=rows)
    ref = O.to(torch.bfloat16).float()
    ulp = torch.abs(ref) * 2.0 ** -7 + 1e-30
    assert torch.all(torch.abs(got - ref) <= ulp + 1e-6 * O.abs().max().item())


# ------------------------------------------------------------------------------ C3 ----
@pytest.mark.parametrize("N", [1536, 576], ids=["q_lora", "kv_lora"])
def test_C3_mla_projection_sampled_rows(N, variant):
    """BASELINE configs[3]: 16384 heavy-outlier tokens x 7168 -> 1536 / 576 (N = 576 ends in a 64-row
    weight block)."""
    M, K = 16384, 7168
    qa, sa = oracle.quantize_act_1x128(W.outlier_act(M, K, seed=0))
    qb, sb, _ = oracle.quantize_weight_128x128(W.master_weight(N, K, seed=1), want_t=False)
    D = fp.gemm(fp.FPROP, dev(qa), dev_scales(sa), dev(qb), dev(sb), out_dtype=torch.float32)
    rows = block_rows(M, seed=3, per_block=1)
    Dr = D[dev(rows)].cpu().double()
    O = oracle.gemm(fp.FPROP, qa, sa, qb, sb, rows=rows)
    assert oracle.rel_err_normwise(Dr, O) <= TOL
    # BF16 output (the benched dtype) is the RNE of the FP32 output
    D16 = fp.gemm(fp.FPROP, dev(qa), dev_scales(sa), dev(qb), dev(sb), out_dtype=torch.bfloat16)
    assert torch.equal(D16.view(torch.int16), D.to(torch.bfloat16).view(torch.int16))


# ------------------------------------------------------------------------------ C4 ----
C4 = dict(tokens=65536, experts=256, top_k=8, K=7168, N=2048)


@pytest.fixture(scope="module")
def c4():
    """The C4 problem in bench.py's layout: tokens quantized 1x128 ONCE by the oracle, FP8 rows and
    per-row scales gathered by expert (exact: the scales are per row), expert weights as random
    finite E4M3 codes with log-uniform block scales (quantizing 256 x 2048 x 7168 with the oracle
    would take minutes)."""
    routes = W.route_skewed(C4["tokens"], C4["experts"], C4["top_k"], alpha=0.5, seed=3)
    tok, offsets = W.group_rows(routes, C4["experts"])
    qx, sx = oracle.quantize_act_1x128(W.gaussian_act(C4["tokens"], C4["K"], seed=0))
    A = qx.index_select(0, tok)
    sA = sx.index_select(1, tok).contiguous()
    del qx, sx
    E, N, K = C4["experts"], C4["N"], C4["K"]
    B = W.random_codes(E * N, K, seed=5).reshape(E, N, K)
    sB = W.random_scales(E, N // 128, K // 128, seed=6)
    d = dict(offsets=offsets, A=A, sA=sA, B=B, sB=sB)
    d["dA"], d["dsA"], d["dB"], d["dsB"] = dev(A), dev_scales(sA), dev(B), dev(sB)
    d["doff"] = dev(offsets)
    d["D"] = fp.grouped_gemm(d["doff"], d["dA"], d["dsA"], d["dB"], d["dsB"], out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    yield d
    d.clear()
    torch.cuda.empty_cache()


def test_C4_grouped_vs_oracle_every_16th_expert(c4):
    """Sampled rows (first, last, 2 random) of every 16th expert, FP32 output, within 1e-3 of the
    oracle; the benched BF16 output is RNE of the FP32 output on every row."""
    off = c4["offsets"]
    D32 = fp.grouped_gemm(c4["doff"], c4["dA"], c4["dsA"], c4["dB"], c4["dsB"], out_dtype=torch.float32)
    assert torch.equal(c4["D"].view(torch.int16), D32.to(torch.bfloat16).view(torch.int16))
    g = torch.Generator().manual_seed(4)
    rows = []
    for e in range(0, C4["experts"], 16):
        a, b = int(off[e]), int(off[e + 1])
        if b > a:
            rows += [a, b - 1] + torch.randint(a, b, (2,), generator=g).tolist()
    rows = torch.tensor(sorted(set(rows)), dtype=torch.int64)
    Dr = D32[dev(rows)].cpu().double()
    del D32
    O = oracle.grouped_gemm(off, c4["A"], c4["sA"], c4["B"], c4["sB"], rows=rows)
    assert oracle.rel_err_normwise(Dr, O) <= TOL


def test_C4_grouped_bitwise_equal_dense_per_expert(c4):
    off = c4["offsets"]
    m = off[1:] - off[:-1]
    for e in {int(torch.argmin(m)), int(torch.argmax(m)), 128}:
        a, b = int(off[e]), int(off[e + 1])
        De = fp.gemm(fp.FPROP, c4["dA"][a:b], dev_scales(c4["sA"][:, a:b].contiguous()), c4["dB"][e], c4["dsB"][e])
        assert_bits_equal(c4["D"][a:b], De, f"expert {e} ({b - a} rows)")


@pytest.mark.parametrize("G", [2, 4, 8])
def test_C4_expert_parallel_split_bitwise_equal_G1(c4, G):
    """The expert-parallel partition bench.py times at N GPUs, run on one GPU: G contiguous expert
    shards (ep.shard_range), each its own grouped launch on its own rows, concatenated == G = 1."""
    from paper_2412_19437_b200 import ep
    off = c4["offsets"]
    parts = []
    for r in range(G):
        e0, e1 = ep.shard_range(C4["experts"], G, r)
        a, b = int(off[e0]), int(off[e1])
        loff = dev(off[e0:e1 + 1] - off[e0])
        sa = dev_scales(c4["sA"][:, a:b].contiguous())
        parts.append(fp.grouped_gemm(loff, c4["dA"][a:b], sa, c4["dB"][e0:e1], c4["dsB"][e0:e1]))
    assert_bits_equal(torch.cat(parts), c4["D"], f"G={G} vs G=1")


@pytest.mark.parametrize("G", [2, 4, 8])
def test_C4_balanced_redundant_placement_bitwise_equal_G1(c4, G):
    """The load-aware placement bench.py uses at N GPUs (LPT over a previous batch's loads,
    one redundant expert per rank whose copies split the expert's rows), run on one GPU: each rank's
    grouped launch over its own (expert, share) groups, scattered back to global row order == G = 1."""
    from paper_2412_19437_b200 import ep
    cfg = ep.EPConfig()
    pl = ep.make_placement(cfg, G, "balanced")
    assert pl.redundant == G
    off = c4["offsets"]
    got = torch.zeros_like(c4["D"])
    for r in range(G):
        rows, loff, exps = ep.placement_rows(off, pl, r)
        rd = dev(rows)
        sa = dev_scales(c4["sA"][:, rows].contiguous())
        ed = dev(exps)
        y = fp.grouped_gemm(dev(loff), c4["dA"].index_select(0, rd), sa, c4["dB"].index_select(0, ed).contiguous(),
                            c4["dsB"].index_select(0, ed).contiguous())
        got.index_copy_(0, rd, y)
    assert_bits_equal(got, c4["D"], f"balanced G={G} vs G=1")


# ------------------------------------------------------------------- non-finite inputs ----
NF_SHAPES = [("flat_tma", 256, 1024, 0), ("strided", 200, 1024, 64), ("generic", 130, 1001, 0)]


def _nf_input(M, K, pad, dtype):
    x = W.nonfinite_act(M, K, seed=M + K).to(dtype)
    if not pad:
        return x, dev(x)
    big = torch.zeros(M, K + pad, dtype=dtype)
    big[:, :K] = x
    return x, dev(big)[:, :K]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "fp32"])
@pytest.mark.parametrize("name,M,K,pad", NF_SHAPES, ids=[c[0] for c in NF_SHAPES])
def test_nonfinite_every_quantizer_bitexact(name, M, K, pad, dtype):
    """NaN / +-Inf elements (reading R6: maxNum amax, Inf scale, NaN -> 0x7F, Inf saturates) through
    the 1x128 (TMA / strided / generic), 128x1 (TMA with the packed-BF16 column amax / generic), fused
    dual, weight 128x128 and power-of-two kernels: codes and scales bit-exact vs the oracle."""
    x, xd = _nf_input(M, K, pad, dtype)
    checks = []
    checks.append(("1x128", fp.quantize_act_1x128(xd), oracle.quantize_act_1x128(x)))
    checks.append(("1x128 pow2", fp.quantize_act_1x128_pow2(xd), oracle.quantize_act_1x128_pow2(x)))
    checks.append(("128x1", fp.quantize_act_128x1(xd), oracle.quantize_act_128x1(x)))
    q, s, qT, sT = fp.quantize_act_dual(xd)
    checks.append(("dual", (q, s, qT, sT), oracle.quantize_act_1x128(x) + oracle.quantize_act_128x1(x)))
    q, s, qT, sT = fp.quantize_act_dual(xd, pow2=True)
    checks.append(("dual pow2", (q, s, qT, sT),
                   oracle.quantize_act_1x128_pow2(x) + oracle.quantize_act_128x1(x, pow2=True)))
    checks.append(("weight", fp.quantize_weight_128x128(xd), oracle.quantize_weight_128x128(x)))
    checks.append(("weight pow2", fp.quantize_weight_128x128(xd, pow2=True), oracle.quantize_weight_128x128(x, pow2=True)))
    torch.cuda.synchronize()
    for what, got, want in checks:
        for i, (g, w) in enumerate(zip(got, want)):
            assert_bits_equal(g, w, f"{what} output {i}")


def test_nonfinite_grouped_128x1_and_requant_bitexact():
    """The grouped (expert-aligned) 128x1 quantizer and the FP8 -> FP8 re-quantization of a cached
    activation holding NaN codes (0x7F) and Inf-scaled groups."""
    x = W.nonfinite_act(700, 384, seed=9).to(torch.bfloat16)
    offsets = torch.tensor([0, 3, 130, 130, 400, 700], dtype=torch.int64)
    qT, sT = fp.quantize_act_128x1_grouped(dev(x), offsets)
    rqT, rsT = oracle.quantize_act_128x1_grouped(x, offsets)
    assert_bits_equal(qT, rqT, "grouped codes")
    assert_bits_equal(sT, rsT, "grouped scales")
    q, s = oracle.quantize_act_1x128(x)
    for pow2 in (False, True):
        gq, gs = fp.requantize_1x128_to_128x1(dev(q), dev_scales(s), pow2=pow2)
        rq, rs = oracle.requantize_1x128_to_128x1(q, s, pow2=pow2)
        assert_bits_equal(gq, rq, f"requant codes pow2={pow2}")
        assert_bits_equal(gs, rs, f"requant scales pow2={pow2}")


# --------------------------------------------------------------- tiny pow2 scales (R26) ----
def test_pow2_tiny_groups_feed_the_mx_gemm_exactly():
    """Groups with amax below 448 * 2^-127 get the smallest UE8M0 scale 2^-127 (reading R26), and the
    UE8M0 GEMM applies exactly that scale: within 1e-3 of the oracle on the oracle's codes/scales."""
    M, N, K = 256, 256, 512
    x = W.gaussian_act(M, K, seed=30, dtype=torch.float32)
    x[:64] *= 2.0 ** -135                  # rows whose groups need a scale below 2^-127
    x[64:128] *= 2.0 ** -120
    q, s = fp.quantize_act_1x128_pow2(dev(x))
    rq, rs = oracle.quantize_act_1x128_pow2(x)
    assert_bits_equal(q, rq, "tiny pow2 codes")
    assert_bits_equal(s, rs, "tiny pow2 scales")
    assert float(rs[:, :64].min()) == 2.0 ** -127
    qb = W.codes_small(N, K, seed=31)
    sb = W.scales_pow2(N // 128, K // 128, seed=32)
    D = fp.gemm(fp.FPROP, dev(rq), dev_scales(rs), dev(qb), dev(sb), out_dtype=torch.float32, mx=True)
    O = oracle.gemm(fp.FPROP, rq, rs, qb, sb)
    for lo, hi in ((0, 64), (64, 128), (128, 256)):
        assert oracle.rel_err_normwise(D[lo:hi].cpu().double(), O[lo:hi]) <= TOL
