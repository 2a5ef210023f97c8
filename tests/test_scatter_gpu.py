"""fp8bs_grouped_gemm_scatter on one GPU (NEXT-3, the combine's send fused into the grouped Fprop's
epilogue): with a pointer table of two local buffers standing in for two ranks' combine buffers, every
output row must land at (dst_rank[r], dst_row[r]) with exactly the bits fp8bs_grouped_gemm writes for
row r, and nothing else may be written.  Both tile variants; ragged and empty experts."""
import pytest
import torch

import paper_2412_19437_b200 as fp
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[1, 2], ids=["cta1", "pair"])
def variant(request):
    with fp.forced_variant(request.param):
        yield request.param


@pytest.mark.parametrize("counts", [[0, 7, 130, 1, 64, 0, 300], [512, 256], [3]])
def test_scatter_equals_grouped_rows(counts, variant):
    N, K = 264, 512
    off = torch.zeros(len(counts) + 1, dtype=torch.int64)
    off[1:] = torch.cumsum(torch.tensor(counts), 0)
    R, G = int(off[-1]), len(counts)
    A = W.codes_small(R, K, seed=1).cuda()
    sA = torch.zeros(K // 128, (R + 3) // 4 * 4, device="cuda")[:, :R]
    sA.copy_(W.scales_pow2(K // 128, R, seed=2).cuda())
    B = W.random_codes(G * N, K, seed=3).reshape(G, N, K).cuda()
    sB = W.random_scales(G, (N + 127) // 128, K // 128, seed=4).cuda()
    doff = off.cuda()
    ref = fp.grouped_gemm(doff, A, sA, B, sB)
    # two destination "ranks", rows permuted, a 16-byte aligned pitch wider than N
    g = torch.Generator().manual_seed(5)
    rank = torch.randint(0, 2, (R,), generator=g, dtype=torch.int32)
    row = torch.empty(R, dtype=torch.int64)
    for r in (0, 1):
        idx = (rank == r).nonzero().flatten()
        row[idx] = torch.randperm(idx.numel(), generator=g)
    ld = N + 8
    bufs = [torch.full((R, ld), -7.0, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    table = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    fp.grouped_gemm_scatter(doff, A, sA, B, sB, table.data_ptr(), rank.cuda(), row.cuda(), ld)
    torch.cuda.synchronize()
    for r in (0, 1):
        idx = (rank == r).nonzero().flatten()
        got = bufs[r][row[idx].cuda()]
        assert torch.equal(got[:, :N].view(torch.int16), ref[idx.cuda()].view(torch.int16))
        assert bool((got[:, N:] == -7.0).all()), "pitch padding must stay untouched"
        unused = torch.ones(R, dtype=torch.bool)
        unused[row[idx]] = False
        assert bool((bufs[r][unused.cuda()] == -7.0).all()), "rows no expert row maps to must stay untouched"


@pytest.mark.parametrize("layout", ["rows", "blocks"])
def test_expand_rows_gathers_codes_and_transposes_scales(layout):
    """fp8bs_expand_rows (the receiver side of the token-once dispatch, and bench.py's C4 e2e gather):
    A[i] == tq[idx[i]] and sA[:, i] == the scales of token idx[i], bit for bit, from a row-major token
    buffer or from the 1x128 quantizer's [K/128, lds] layout; ragged R (not a multiple of 32)."""
    U, K, R = 300, 1024, 1000
    KB = K // 128
    g = torch.Generator().manual_seed(3)
    tq = torch.randint(0, 256, (U, K), generator=g, dtype=torch.uint8).cuda()
    ts_rows = torch.rand(U, KB, generator=g).cuda()
    idx = torch.randint(0, U, (R,), generator=g).cuda()
    if layout == "rows":
        ts = ts_rows
    else:
        ts = torch.zeros(KB, (U + 3) // 4 * 4, device="cuda")[:, :U]
        ts.copy_(ts_rows.T)
    A, sA = fp.expand_rows(idx, tq, ts, ts_layout=layout)
    torch.cuda.synchronize()
    assert torch.equal(A, tq[idx])
    assert torch.equal(sA.view(torch.int32), ts_rows[idx].T.contiguous().view(torch.int32))
