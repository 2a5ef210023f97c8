"""Accuracy study on the CPU oracle: why the activation gradient is quantized
tile-wise, not block-wise.

PAPER.md App. B.2: quantizing the tensors of Dgrad per 128x128 block "leads to model
divergence"; the paper attributes it to activation gradients being "highly imbalanced among tokens,
resulting in token-correlated outliers" that block-wise quantization cannot manage.  The oracle lets us
measure the GEMM-level effect on synthetic gradients with exactly that structure (workloads.grad_out:
N(0,1)*1e-2 with 1% of the tokens x100):

    dX = dY . W   (Dgrad; contraction over the output channels)

  * tile-wise  (the paper's recipe): dY in 1x128 tiles along the contraction (one scale per token per
    128 channels), W in 128x128 blocks;
  * block-wise (the rejected one):   dY in 128x128 blocks (one scale per 128 tokens x 128 channels).

Both go through the same FP64 oracle GEMM (a block scale is a per-row scale repeated over the block's
128 rows), and are compared with the unquantized product of the same BF16/FP32 inputs, for a range of
outlier factors.  Measured: at x100 (the bench's dY recipe) block-wise is no worse, because
E4M3 with an FP32 scale spans ~2^15 of normal range; the ordinary tokens only lose precision once the
token imbalance pushes them below E4M3's normal range.  The test pins that shape.
"""
import torch

import oracle
import workloads as W


def _grad_out(T, out, factor, seed):
    """workloads.grad_out's recipe with a chosen outlier factor: N(0,1)*1e-2, 1% of tokens x factor."""
    g = torch.Generator().manual_seed(seed)
    dy = torch.randn(T, out, generator=g) * 1e-2
    tok = torch.randperm(T, generator=g)[:max(1, T // 100)]
    dy[tok] *= factor
    return dy.to(torch.bfloat16), tok


def _dgrad_errors(factor, T=512, out=1024, inn=512, seed=2):
    dy, tok = _grad_out(T, out, factor, seed)
    w = W.master_weight(out, inn, seed=seed + 1)                # FP32 master weight [out, in]
    exact = dy.double() @ w.double()                            # [T, in]
    # W as the Dgrad B operand: WqT [in, out] with the 128x128 block scales read as [K/128][N/128]
    qw, sw, qwT = oracle.quantize_weight_128x128(w)
    # tile-wise dY: 1x128 along the contraction (out)
    qt, st = oracle.quantize_act_1x128(dy)                      # st [out/128, T]
    tile = oracle.gemm(oracle.DGRAD, qt, st, qwT, sw)
    # block-wise dY: 128x128 blocks, each block's scale repeated over its 128 token rows
    qb, sb, _ = oracle.quantize_weight_128x128(dy, want_t=False)   # sb [T/128, out/128]
    sb_rows = sb.t().repeat_interleave(128, dim=1)[:, :T].contiguous()  # [out/128, T]
    block = oracle.gemm(oracle.DGRAD, qb, sb_rows, qwT, sw)
    plain = torch.ones(T, dtype=torch.bool)
    plain[tok] = False

    def nerr(D, rows):   # normwise over a token group: max |err| / max |exact|
        return float((D[rows] - exact[rows]).abs().max() / exact[rows].abs().max())
    return {"tile_plain": nerr(tile, plain), "block_plain": nerr(block, plain),
            "tile_outlier": nerr(tile, ~plain), "block_outlier": nerr(block, ~plain)}


def test_blockwise_dgrad_error_vs_token_imbalance():
    """Tile-wise error is flat in the imbalance; block-wise error on the ordinary tokens is flat while
    the outlier/ordinary ratio stays inside E4M3's normal range (2^-6..448, ~2^15) and blows up
    beyond it, when the ordinary tokens of an outlier's block fall into subnormals or to zero."""
    rows = {f: _dgrad_errors(f) for f in (1e2, 1e3, 1e4, 1e5, 1e6)}
    for f, e in rows.items():
        print(f"outlier x{f:.0e}: " + ", ".join(f"{k} {v:.3e}" for k, v in e.items()))
    for e in rows.values():
        assert e["tile_plain"] < 0.06 and e["tile_outlier"] < 0.06     # E4M3: a few 1e-2, any imbalance
    assert rows[1e2]["block_plain"] < 2 * rows[1e2]["tile_plain"]      # within the normal range: no harm
    assert rows[1e5]["block_plain"] > 5 * rows[1e5]["tile_plain"]      # beyond it: the block scale wipes them
    assert rows[1e6]["block_plain"] > 0.5                               # mostly flushed to zero
