"""Grouped MoE expert Wgrad: dW_e = dY_e^T X_e over each expert's own tokens, with
the Wgrad operands in 128x1 tiles along the tokens whose groups restart at each
expert's first token (reading R25), on the expert-aligned ("padded") token layout of
include/fp8bs.h.

CPU: the oracle's grouped functions pinned by properties the definition fixes (segment = dense
quantization of that expert alone, invariance under reordering the experts, the one-expert case equals
the dense path, padding adds nothing, the dequantized product is close to the unquantized one) and the
host-side validation of the C-ABI.  GPU: the CUDA path through the C-ABI vs the oracle (codes and scales
bit-exact; dW within 1e-3 normwise per expert; bitwise equal to per-expert dense fp8bs_gemm WGRAD calls).
"""
import pytest
import torch

import oracle
import workloads as W

TOL = 1e-3
# expert token counts: empty experts, a 1-token expert, exact multiples of 128, ragged tails
COUNTS = [[0, 5, 128, 200, 0, 300, 1, 256], [130], [0, 0, 77]]


def _offsets(counts):
    off = torch.zeros(len(counts) + 1, dtype=torch.int64)
    off[1:] = torch.cumsum(torch.tensor(counts, dtype=torch.int64), 0)
    return off


def _problem(counts, C_in=256, N_out=384, seed=0):
    off = _offsets(counts)
    R = int(off[-1])
    x = W.gaussian_act(R, C_in, seed=seed)
    dy = W.grad_out(R, N_out, seed=seed + 1)
    return off, x, dy


def test_grouped_128x1_is_per_expert_dense():
    off, x, _ = _problem(COUNTS[0])
    qT, sT = oracle.quantize_act_128x1_grouped(x, off)
    P = oracle.padded_offsets(off)
    assert int(P[-1]) == sum((c + 127) // 128 * 128 for c in COUNTS[0])
    for e in range(len(COUNTS[0])):
        a, b, p, q = int(off[e]), int(off[e + 1]), int(P[e]), int(P[e + 1])
        if a == b:
            assert p == q
            continue
        qd, sd = oracle.quantize_act_128x1(x[a:b])
        assert torch.equal(qT[:, p:p + b - a], qd)
        assert torch.equal(qT[:, p + b - a:q], torch.zeros_like(qT[:, p + b - a:q]))   # padding codes 0
        assert torch.equal(sT[p // 128:q // 128], sd)


def test_groups_never_straddle_experts():
    """Expert e's rows scaled by 10^e: every scale row must see one expert's magnitude only."""
    counts = [70, 90, 60]
    off, x, _ = _problem(counts)
    x = x.float()
    for e in range(3):
        x[int(off[e]):int(off[e + 1])] *= 10.0 ** (2 * e)
    _, sT = oracle.quantize_act_128x1_grouped(x, off)
    amax = [x[int(off[e]):int(off[e + 1])].abs().amax(0) for e in range(3)]
    for e in range(3):
        assert torch.equal(sT[e], (amax[e] / 448.0).float())     # one 128-group per expert here


def test_grouped_wgrad_oracle_properties():
    counts = COUNTS[0]
    off, x, dy = _problem(counts)
    XqT, sX = oracle.quantize_act_128x1_grouped(x, off)
    DqT, sD = oracle.quantize_act_128x1_grouped(dy, off)
    O = oracle.grouped_gemm_wgrad(off, DqT, sD, XqT, sX)
    G = len(counts)
    # (1) permuting the experts permutes the result
    perm = [3, 0, 7, 2, 5, 1, 6, 4]
    segs = [(int(off[e]), int(off[e + 1])) for e in range(G)]
    xp = torch.cat([x[a:b] for a, b in (segs[e] for e in perm)])
    dyp = torch.cat([dy[a:b] for a, b in (segs[e] for e in perm)])
    offp = _offsets([counts[e] for e in perm])
    XqTp, sXp = oracle.quantize_act_128x1_grouped(xp, offp)
    DqTp, sDp = oracle.quantize_act_128x1_grouped(dyp, offp)
    Op = oracle.grouped_gemm_wgrad(offp, DqTp, sDp, XqTp, sXp)
    for i, e in enumerate(perm):
        assert torch.equal(Op[i], O[e])
    # (2) empty experts are zero; (3) close to the unquantized per-expert product (E4M3: ~4e-2, §3)
    for e, (a, b) in enumerate(segs):
        if a == b:
            assert not O[e].any()
            continue
        exact = dy[a:b].double().T @ x[a:b].double()
        assert oracle.rel_err_normwise(O[e], exact) < 0.15
    # (4) one expert with a multiple of 128 tokens: the dense 128x1 + WGRAD path
    off1, x1, dy1 = _problem([256])
    XqT1, sX1 = oracle.quantize_act_128x1_grouped(x1, off1)
    DqT1, sD1 = oracle.quantize_act_128x1_grouped(dy1, off1)
    qx, sx = oracle.quantize_act_128x1(x1)
    qd, sd = oracle.quantize_act_128x1(dy1)
    assert torch.equal(oracle.grouped_gemm_wgrad(off1, DqT1, sD1, XqT1, sX1)[0], oracle.gemm(2, qd, sd, qx, sx))


def test_grouped_wgrad_abi_validation():
    """Host-side argument checks of the grouped Wgrad entry points (no GPU needed: offsets are checked
    before the device)."""
    import ctypes

    import paper_2412_19437_b200 as fp
    L = fp.lib()
    bad = torch.tensor([0, 5, 3], dtype=torch.int64)          # decreasing
    nz = torch.tensor([1, 5], dtype=torch.int64)              # offsets[0] != 0
    for off in (bad, nz):
        st = L.fp8bs_quantize_act_128x1_grouped(ctypes.c_void_p(16), 0, off.numel() - 1, off.data_ptr(), 128, 128,
                                                ctypes.c_void_p(16), 4096, ctypes.c_void_p(16), 128, None)
        assert st == 1, fp.last_error_detail()
        st = L.fp8bs_grouped_gemm_wgrad(off.numel() - 1, off.data_ptr(), 128, 128, None, 4096, None, 128, None, 4096,
                                        None, 128, None, 128, 0, None)
        assert st == 1
        assert L.fp8bs_padded_tokens(off.numel() - 1, off.data_ptr()) == 0
    assert fp.padded_tokens([0, 5, 5, 300]) == 128 + 0 + 384


# ----------------------------------------------------------------------------------- GPU ----
@pytest.mark.gpu
@pytest.mark.parametrize("dtype,aligned", [(torch.bfloat16, True), (torch.float32, True), (torch.bfloat16, False)],
                         ids=["bf16_one_launch", "fp32_one_launch", "bf16_unaligned_per_expert"])
@pytest.mark.parametrize("counts", COUNTS, ids=["mixed8", "one", "empties"])
def test_grouped_128x1_gpu_bitexact(counts, dtype, aligned):
    """Aligned rows take the single-launch kernel (token-block map over all experts); rows whose pitch
    is not a multiple of 16 bytes take the per-expert loop of the generic kernel."""
    import paper_2412_19437_b200 as fp
    off, x, _ = _problem(counts)
    x = x.to(dtype)
    qT_ref, sT_ref = oracle.quantize_act_128x1_grouped(x, off)
    qT = torch.full((x.shape[1], int(oracle.padded_offsets(off)[-1])), 0x55, dtype=torch.uint8, device="cuda")
    xd = x.cuda()
    if not aligned:   # row pitch C + 1 elements
        wide = torch.zeros(x.shape[0], x.shape[1] + 1, dtype=dtype, device="cuda")
        wide[:, :x.shape[1]] = xd
        xd = wide[:, :x.shape[1]]
    qT, sT = fp.quantize_act_128x1_grouped(xd, off, qT=qT)
    torch.cuda.synchronize()
    assert torch.equal(qT.cpu(), qT_ref)          # padding overwritten with 0
    assert torch.equal(sT.cpu().view(torch.int32), sT_ref.view(torch.int32))


@pytest.mark.gpu
@pytest.mark.parametrize("counts", COUNTS, ids=["mixed8", "one", "empties"])
def test_grouped_wgrad_gpu_vs_oracle_and_dense(counts):
    import paper_2412_19437_b200 as fp
    off, x, dy = _problem(counts, C_in=448, N_out=640)
    XqT, sX = oracle.quantize_act_128x1_grouped(x, off)
    DqT, sD = oracle.quantize_act_128x1_grouped(dy, off)
    O = oracle.grouped_gemm_wgrad(off, DqT, sD, XqT, sX)
    XqT_d, sX_d = fp.quantize_act_128x1_grouped(x.cuda(), off)
    DqT_d, sD_d = fp.quantize_act_128x1_grouped(dy.cuda(), off)
    G, N, K = len(counts), dy.shape[1], x.shape[1]
    D = torch.full((G, N, K), float("nan"), device="cuda")
    fp.grouped_gemm_wgrad(off, DqT_d, sD_d, XqT_d, sX_d, out=D)
    torch.cuda.synchronize()
    P = oracle.padded_offsets(off)
    for e in range(G):
        p, q = int(P[e]), int(P[e + 1])
        if p == q:
            assert not D[e].any(), "expert without tokens must get dW = 0"
            continue
        assert oracle.rel_err_normwise(D[e].cpu().double(), O[e]) <= TOL
        De = fp.gemm(fp.WGRAD, DqT_d[:, p:q], sD_d[p // 128:q // 128], XqT_d[:, p:q], sX_d[p // 128:q // 128],
                     out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert torch.equal(D[e].view(torch.int32), De.view(torch.int32))
    # accumulate: D += dW (experts without tokens keep D)
    D2 = torch.ones(G, N, K, device="cuda")
    fp.grouped_gemm_wgrad(off, DqT_d, sD_d, XqT_d, sX_d, out=D2, accumulate=True)
    torch.cuda.synchronize()
    for e in range(G):
        assert oracle.rel_err_normwise(D2[e].cpu().double(), O[e] + 1.0) <= TOL


@pytest.mark.gpu
def test_grouped_wgrad_c4_full_size_sampled():
    """C4's expert shape at the size tools/grouped_wgrad_bench.py times (256 experts, 8192 tokens x
    top-8 = 65536 rows, skewed routing R16, 7168 -> 2048): GPU quantizer + grouped Wgrad, checked on
    sampled dW rows of the smallest, the largest and two other experts against the oracle GEMM on the
    same codes (the oracle quantizer checks the sampled experts' codes bit for bit)."""
    import paper_2412_19437_b200 as fp
    G, T, N, K = 256, 8192, 2048, 7168
    routes = W.route_skewed(T, G, 8, seed=3)
    _, off = W.group_rows(routes, G)
    R = int(off[-1])
    x = W.gaussian_act(R, K, seed=0)
    dy = W.grad_out(R, N, seed=1)
    XqT, sX = fp.quantize_act_128x1_grouped(x.cuda(), off)
    DqT, sD = fp.quantize_act_128x1_grouped(dy.cuda(), off)
    D = fp.grouped_gemm_wgrad(off, DqT, sD, XqT, sX)
    torch.cuda.synchronize()
    m = off[1:] - off[:-1]
    P = oracle.padded_offsets(off)
    experts = sorted({int(m.argmin()), int(m.argmax()), 17, 200})
    g = torch.Generator().manual_seed(4)
    for e in experts:
        a, b, p, q = int(off[e]), int(off[e + 1]), int(P[e]), int(P[e + 1])
        qx, sx = oracle.quantize_act_128x1(x[a:b])
        qd, sd = oracle.quantize_act_128x1(dy[a:b])
        assert torch.equal(XqT[:, p:p + b - a].cpu(), qx) and torch.equal(DqT[:, p:p + b - a].cpu(), qd)
        assert torch.equal(sX[p // 128:q // 128].cpu().view(torch.int32), sx.view(torch.int32))
        rows = torch.cat([torch.tensor([0, N - 1]), torch.randint(0, N, (6,), generator=g)])
        pad = lambda c: torch.nn.functional.pad(c, (0, (q - p) - (b - a)))   # zero codes up to roundup(M_e,128)
        O = oracle.gemm(2, pad(qd), sd, pad(qx), sx, rows=rows)
        assert oracle.rel_err_normwise(D[e][rows.cuda()].cpu().double(), O) <= TOL


@pytest.mark.gpu
def test_grouped_calls_capture_in_a_cuda_graph():
    """The grouped Wgrad is one launch and the grouped Fprop two (tile scheduler + GEMM), with no host
    synchronisation and no library state: both capture into a CUDA graph, and a replay is bitwise equal
    to the eager call (the side-stream fork it replaced had no such test)."""
    import paper_2412_19437_b200 as fp
    counts = [0, 1, 300, 128, 257, 0, 700]
    off, x, dy = _problem(counts, C_in=384, N_out=256)
    XqT, sX = fp.quantize_act_128x1_grouped(x.cuda(), off)
    DqT, sD = fp.quantize_act_128x1_grouped(dy.cuda(), off)
    G, N, K = len(counts), dy.shape[1], x.shape[1]
    eager = fp.grouped_gemm_wgrad(off, DqT, sD, XqT, sX)
    qx, sx = fp.quantize_act_1x128(x.cuda())
    Bq = torch.randint(0, 0x7E, (G, N, K), dtype=torch.uint8, device="cuda")
    sB = torch.rand(G, N // 128, K // 128, device="cuda") * 1e-3
    doff = off.cuda()
    ws = torch.empty(int(fp.lib().fp8bs_grouped_gemm_workspace_size(G, x.shape[0], N, K)), dtype=torch.uint8,
                     device="cuda")
    eager_f = fp.grouped_gemm(doff, qx, sx, Bq, sB, workspace=ws)
    torch.cuda.synchronize()
    out_w = torch.full_like(eager, float("nan"))
    out_f = torch.empty_like(eager_f)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fp.grouped_gemm_wgrad(off, DqT, sD, XqT, sX, out=out_w)
            fp.grouped_gemm(doff, qx, sx, Bq, sB, out=out_f, workspace=ws)
    for _ in range(2):
        out_w.fill_(float("nan"))
        out_f.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out_w.view(torch.int32), eager.view(torch.int32))
        assert torch.equal(out_f.view(torch.int16), eager_f.view(torch.int16))


# ----------------------------------------------------------- grouped Wgrad on UE8M0 (NEXT-1) ----
def _grouped_pow2_128x1(x, off):
    """The expert-aligned 128x1 layout with POWER-OF-TWO scales (R23): each expert's tokens quantized
    alone by the oracle's pow2 128x1 function (the grouped definition: segment = dense quantization of
    that expert, pinned above), codes 0 in the padding."""
    P = oracle.padded_offsets(off)
    C, Mp = x.shape[1], int(P[-1])
    qT = torch.zeros(C, Mp, dtype=torch.uint8)
    sT = torch.zeros(Mp // 128, C, dtype=torch.float32)
    for e in range(off.numel() - 1):
        a, b, p = int(off[e]), int(off[e + 1]), int(P[e])
        if a == b:
            continue
        q, s = oracle.quantize_act_128x1(x[a:b], pow2=True)
        qT[:, p:p + b - a] = q
        sT[p // 128:p // 128 + s.shape[0]] = s
    return qT, sT


def _dev_rows(t):
    """Device copy with the row pitch padded to 16 bytes (the GEMM's alignment rule)."""
    r, c = t.shape
    align = 16 // t.element_size()
    buf = torch.zeros(r, (c + align - 1) // align * align, dtype=t.dtype, device="cuda")
    buf[:, :c] = t.cuda()
    return buf[:, :c]


@pytest.mark.gpu
@pytest.mark.parametrize("counts", COUNTS + [[300, 0, 1000, 129]], ids=["mixed8", "one", "empties", "wide"])
def test_grouped_wgrad_mx_vs_oracle_and_dense_mx(counts):
    """fp8bs_grouped_gemm_wgrad_mx: within 1e-3 of the oracle per expert, bitwise equal to the dense
    UE8M0 WGRAD (fp8bs_gemm_mx) on each expert's own columns, zero for experts without tokens, and
    D += dW when accumulating."""
    import paper_2412_19437_b200 as fp
    off, x, dy = _problem(counts, C_in=448, N_out=640)
    XqT, sX = _grouped_pow2_128x1(x, off)
    DqT, sD = _grouped_pow2_128x1(dy, off)
    O = oracle.grouped_gemm_wgrad(off, DqT, sD, XqT, sX)
    XqT_d, sX_d, DqT_d, sD_d = _dev_rows(XqT), _dev_rows(sX), _dev_rows(DqT), _dev_rows(sD)
    G, N, K = len(counts), dy.shape[1], x.shape[1]
    D = torch.full((G, N, K), float("nan"), device="cuda")
    fp.grouped_gemm_wgrad(off, DqT_d, sD_d, XqT_d, sX_d, out=D, mx=True)
    torch.cuda.synchronize()
    P = oracle.padded_offsets(off)
    for e in range(G):
        p, q = int(P[e]), int(P[e + 1])
        if p == q:
            assert not D[e].any(), "expert without tokens must get dW = 0"
            continue
        assert oracle.rel_err_normwise(D[e].cpu().double(), O[e]) <= TOL
        De = fp.gemm(fp.WGRAD, DqT_d[:, p:q], sD_d[p // 128:q // 128], XqT_d[:, p:q], sX_d[p // 128:q // 128],
                     out_dtype=torch.float32, mx=True)
        torch.cuda.synchronize()
        assert torch.equal(D[e].view(torch.int32), De.view(torch.int32)), f"expert {e}"
    D2 = torch.ones(G, N, K, device="cuda")
    fp.grouped_gemm_wgrad(off, DqT_d, sD_d, XqT_d, sX_d, out=D2, accumulate=True, mx=True)
    torch.cuda.synchronize()
    for e in range(G):
        assert torch.equal(D2[e].view(torch.int32), (D[e] + 1.0).view(torch.int32)) if int(P[e]) < int(P[e + 1]) \
            else bool((D2[e] == 1.0).all())


@pytest.mark.gpu
def test_grouped_wgrad_mx_closed_form_bitexact():
    """Codes of {0, +-1, +-2} with power-of-two scales: every product and sum is exact, so the grouped
    UE8M0 Wgrad must equal the oracle bit for bit on every expert (ragged experts included)."""
    import paper_2412_19437_b200 as fp
    counts = [130, 0, 384, 7, 1000]
    off = _offsets(counts)
    P = oracle.padded_offsets(off)
    Mp, N, K = int(P[-1]), 384, 704
    A = W.codes_small(N, Mp, seed=21)
    B = W.codes_small(K, Mp, seed=22)
    for e in range(len(counts)):       # padding columns hold code 0 (as the grouped quantizer writes)
        a, b, p, q = int(off[e]), int(off[e + 1]), int(P[e]), int(P[e + 1])
        A[:, p + b - a:q] = 0
        B[:, p + b - a:q] = 0
    sA = W.scales_pow2(Mp // 128, N, seed=23)
    sB = W.scales_pow2(Mp // 128, K, seed=24)
    O = oracle.grouped_gemm_wgrad(off, A, sA, B, sB)
    D = fp.grouped_gemm_wgrad(off, _dev_rows(A), _dev_rows(sA), _dev_rows(B), _dev_rows(sB), mx=True)
    torch.cuda.synchronize()
    assert torch.equal(D.cpu().view(torch.int32), O.to(torch.float32).view(torch.int32))
