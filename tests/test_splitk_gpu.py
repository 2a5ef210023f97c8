"""GPU parity of the split-K tail (fp8bs_gemm_ws; include/fp8bs.h, reading R30).

When a dense GEMM's last wave of output tiles would fill at most half of the clusters, those tiles are
cut along K into S chunks; each chunk is promoted like a whole tile over its own K-blocks into an FP32
partial and a reduce kernel sums the chunks in order.  Checked through the C-ABI, both tile variants:
  * closed-form operands (codes {0, +-1, +-2}, power-of-two scales): every partial and every sum is an
    exact integer below 2^24, so the result must equal the oracle BIT FOR BIT whatever the order;
  * quantized Gaussian / outlier operands: within 1e-3 of the FP64 oracle on sampled rows, and within
    FP32 rounding of the unsplit kernel (fp8bs_gemm) everywhere;
  * BF16 output == RNE of the split FP32 output; WGRAD accumulate == D0 + the split result;
  * repeated launches bitwise identical (deterministic reduction order);
  * a workspace below fp8bs_gemm_workspace_size is rejected before any launch.
"""
import pytest
import torch

import oracle
import paper_2412_19437_b200 as fp
import workloads as W

pytestmark = pytest.mark.gpu
DEV = "cuda"

# (M, N, K): a few tiles (no full wave); 78 pair / 156 single-CTA tiles = one wave + a small tail;
# a ragged WGRAD-like shape.  Every one has a split-K tail on a 148-SM B200 (asserted below).
SHAPES = [(300, 512, 8192), (3300, 1400, 8192), (1000, 776, 8192)]


@pytest.fixture(params=[1, 2], ids=["cta1", "pair"])
def variant(request):
    with fp.forced_variant(request.param):
        yield request.param


def dev(t):
    return t.to(DEV)


def scale_b_shape(layout, N, K):
    KB, NB = K // 128, (N + 127) // 128
    return {fp.FPROP: (NB, KB), fp.DGRAD: (KB, NB), fp.WGRAD: (KB, N)}[layout]


def sample_rows(M, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.unique(torch.cat([torch.tensor([0, M - 1]), torch.randint(0, M, (48,), generator=g)]))


def assert_bits_equal(got, want, what):
    got, want = got.cpu().contiguous(), want.cpu().contiguous()
    iv = torch.int32 if got.dtype == torch.float32 else torch.int16
    bad = (got.view(iv) != want.view(iv)).nonzero()
    assert bad.numel() == 0, f"{what}: {bad.shape[0]} mismatches, first at {bad[:5].tolist()}"


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_shapes_have_a_split_tail(M, N, K):
    torch.cuda.init()
    for layout in (fp.FPROP, fp.DGRAD, fp.WGRAD):
        assert fp.gemm_workspace_size(layout, M, N, K) > 0, (layout, M, N, K)


@pytest.mark.parametrize("layout", [fp.FPROP, fp.DGRAD, fp.WGRAD], ids=["fprop", "dgrad", "wgrad"])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_split_closed_form_bitexact(layout, M, N, K, variant):
    A = W.codes_small(M, K, seed=M + 7)
    B = W.codes_small(N, K, seed=N + 8)
    sA = W.scales_pow2(K // 128, M, seed=9)
    sB = W.scales_pow2(*scale_b_shape(layout, N, K), seed=10)
    D = fp.gemm(layout, dev(A), dev(sA), dev(B), dev(sB), out_dtype=torch.float32)          # workspace "auto"
    rows = sample_rows(M, seed=layout)
    O = oracle.gemm(layout, A, sA, B, sB, rows=rows)
    assert_bits_equal(D[dev(rows)], O.to(torch.float32), "split-K closed form")


def operands(layout, M, N, K, seed=0):
    if layout == fp.FPROP:
        qa, sa = oracle.quantize_act_1x128(W.outlier_act(M, K, seed=seed))
        qb, sb, _ = oracle.quantize_weight_128x128(W.master_weight(N, K, seed=seed + 1), want_t=False)
    elif layout == fp.DGRAD:
        qa, sa = oracle.quantize_act_1x128(W.grad_out(M, K, seed=seed))
        _, sb, qb = oracle.quantize_weight_128x128(W.master_weight(K, N, seed=seed + 1))
    else:
        qa, sa = oracle.quantize_act_128x1(W.grad_out(K, M, seed=seed))
        qb, sb = oracle.quantize_act_128x1(W.gaussian_act(K, N, seed=seed + 1))
    return qa, sa, qb, sb


@pytest.mark.parametrize("layout", [fp.FPROP, fp.DGRAD, fp.WGRAD], ids=["fprop", "dgrad", "wgrad"])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_split_vs_oracle_and_unsplit(layout, M, N, K, variant):
    qa, sa, qb, sb = operands(layout, M, N, K)
    args = (layout, dev(qa), dev(sa), dev(qb), dev(sb))
    Ds = fp.gemm(*args, out_dtype=torch.float32)                    # split tail
    Du = fp.gemm(*args, out_dtype=torch.float32, workspace=None)    # every tile over all of K
    rows = sample_rows(M, seed=layout + 3)
    O = oracle.gemm(layout, qa, sa, qb, sb, rows=rows)
    assert oracle.rel_err_normwise(Ds[dev(rows)].cpu().double(), O) <= 1e-3
    # the two summation orders differ by FP32 rounding only
    scale = Du.abs().max().item()
    assert torch.allclose(Ds, Du, rtol=1e-5, atol=1e-6 * scale)
    assert not torch.equal(Ds, torch.zeros_like(Ds))
    # BF16 output is the RNE of the split FP32 output (layout permitting)
    if layout != fp.WGRAD:
        D16 = fp.gemm(*args, out_dtype=torch.bfloat16)
        assert_bits_equal(D16, Ds.to(torch.bfloat16), "bf16 == RNE(split fp32)")
    # deterministic: a second launch is bitwise identical
    assert_bits_equal(fp.gemm(*args, out_dtype=torch.float32), Ds, "repeat")


def test_split_wgrad_accumulate(variant):
    M, N, K = 1000, 776, 8192
    qa, sa, qb, sb = operands(fp.WGRAD, M, N, K, seed=5)
    args = (fp.WGRAD, dev(qa), dev(sa), dev(qb), dev(sb))
    D0 = torch.randn(M, N, generator=torch.Generator().manual_seed(1)).to(DEV)
    S = fp.gemm(*args, out_dtype=torch.float32)
    D = D0.clone()
    fp.gemm(*args, out=D, accumulate=True)
    assert_bits_equal(D, D0 + S, "D0 + split")


def test_split_workspace_too_small_is_rejected():
    M, N, K = 300, 512, 8192
    qa, sa, qb, sb = operands(fp.FPROP, M, N, K)
    need = fp.gemm_workspace_size(fp.FPROP, M, N, K)
    ws = torch.empty(need - 16, dtype=torch.uint8, device=DEV)
    with pytest.raises(fp.Fp8bsError):
        fp.gemm(fp.FPROP, dev(qa), dev(sa), dev(qb), dev(sb), workspace=ws)
    # exactly the required size works and equals the auto-allocated call
    ws = torch.empty(need, dtype=torch.uint8, device=DEV)
    a = fp.gemm(fp.FPROP, dev(qa), dev(sa), dev(qb), dev(sb), out_dtype=torch.float32, workspace=ws)
    b = fp.gemm(fp.FPROP, dev(qa), dev(sa), dev(qb), dev(sb), out_dtype=torch.float32)
    assert_bits_equal(a, b, "explicit workspace == auto")


def test_split_graph_capture():
    """The three launches (full waves, tail units, reduce) capture into a CUDA graph and replay."""
    M, N, K = 3300, 1400, 8192
    qa, sa, qb, sb = operands(fp.DGRAD, M, N, K, seed=2)
    args = (fp.DGRAD, dev(qa), dev(sa), dev(qb), dev(sb))
    ref = fp.gemm(*args, out_dtype=torch.float32)
    out = torch.empty_like(ref)
    ws = torch.empty(fp.gemm_workspace_size(fp.DGRAD, M, N, K), dtype=torch.uint8, device=DEV)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fp.gemm(*args, out=out, workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    out.zero_()
    with torch.cuda.graph(g, stream=s):
        fp.gemm(*args, out=out, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    assert_bits_equal(out, ref, "graph replay")
