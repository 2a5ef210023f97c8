"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the method (no amax, no scale, no E4M3
rounding, no GEMM).  It only draws random tensors with the shapes and value
distributions of DeepSeek-V3's FP8 Linear / MoE workloads, on the CPU, with a
fixed torch generator per tensor, so that the oracle side (``oracle/``) and the
product side (``paper_2412_19437_b200``) see bit-identical inputs.

Recipes:

* ``gaussian_act``   X ~ N(0,1) -> BF16                         (seed 0)
* ``outlier_act``    N(0,1); a fixed 0.5% of channels x64; one random element
                     per row x1000; -> BF16          (seeds 0 / 10)
* ``master_weight``  W ~ N(0, 0.006^2) FP32 (init std) (seed 1)
* ``grad_out``       dY ~ N(0,1)*1e-2, 1% of tokens x100 (token-correlated
                     outliers) -> BF16                   (seed 2)
* ``route_uniform``  every token picks top_k distinct experts uniformly
                     (Gumbel-top-k)                              (seed 3)
* ``route_skewed``   expert weight ~ (rank+1)^-alpha over a random expert
                     permutation, top_k distinct per token (Gumbel-top-k) (seed 3)
* ``codes_small`` / ``scales_pow2``  exact-arithmetic GEMM operands: E4M3
                     codes of {0, +-1, +-2} and scales in {1, 2, 4}
                     (SURVEY.md §8(c) "GEMM closed form")
"""
from __future__ import annotations

import torch

# E4M3 codes of the values 0, +1, -1, +2, -2 (bit layout: sign | exp(4, bias 7) | man(3)).
# These are bit patterns chosen for the closed-form GEMM test, not a rounding rule.
E4M3_SMALL_CODES = (0x00, 0x38, 0xB8, 0x40, 0xC0)


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def gaussian_act(M: int, K: int, seed: int = 0, dtype=torch.bfloat16) -> torch.Tensor:
    """X ~ N(0,1), [M, K] row-major, cast to ``dtype`` (BF16 by default)."""
    return torch.randn(M, K, generator=_gen(seed), dtype=torch.float32).to(dtype)


def outlier_act(M: int, K: int, seed: int = 0, dtype=torch.bfloat16) -> torch.Tensor:
    """Heavy-outlier activations: N(0,1), 0.5% of channels x64,
    one random element per row x1000."""
    g = _gen(seed)
    x = torch.randn(M, K, generator=g, dtype=torch.float32)
    n_ch = max(1, (K * 5) // 1000)
    ch = torch.randperm(K, generator=g)[:n_ch]
    x[:, ch] *= 64.0
    g2 = _gen(seed + 10)
    pos = torch.randint(0, K, (M,), generator=g2)
    x[torch.arange(M), pos] *= 1000.0
    return x.to(dtype)


def master_weight(N: int, K: int, seed: int = 1, dtype=torch.float32) -> torch.Tensor:
    """W ~ N(0, 0.006^2) FP32 master weight [N(out), K(in)] (P:705 init std)."""
    return (torch.randn(N, K, generator=_gen(seed), dtype=torch.float32) * 0.006).to(dtype)


def expert_weights(E: int, N: int, K: int, seed: int = 1, dtype=torch.bfloat16,
                   first_expert: int = 0) -> torch.Tensor:
    """[E, N, K] expert weights; expert e (global id first_expert+e) uses seed+id so that
    an expert-parallel shard regenerates exactly the same weights as the global tensor."""
    out = torch.empty(E, N, K, dtype=dtype)
    for e in range(E):
        gid = first_expert + e
        out[e] = (torch.randn(N, K, generator=_gen(seed + 1000 + gid), dtype=torch.float32)
                  * 0.006).to(dtype)
    return out


def grad_out(M: int, N: int, seed: int = 2, dtype=torch.bfloat16) -> torch.Tensor:
    """dY ~ N(0,1)*1e-2 with 1% of tokens x100 (token-correlated outliers)."""
    g = _gen(seed)
    dy = torch.randn(M, N, generator=g, dtype=torch.float32) * 1e-2
    n_tok = max(1, M // 100)
    tok = torch.randperm(M, generator=g)[:n_tok]
    dy[tok] *= 100.0
    return dy.to(dtype)


def _gumbel_topk(logw: torch.Tensor, T: int, top_k: int, g: torch.Generator) -> torch.Tensor:
    """T tokens each draw top_k DISTINCT experts with probability ~ exp(logw) (Gumbel-top-k)."""
    E = logw.numel()
    u = torch.rand(T, E, generator=g, dtype=torch.float64).clamp_(1e-300, 1.0)
    gumbel = -torch.log(-torch.log(u))
    return torch.topk(logw.to(torch.float64)[None, :] + gumbel, top_k, dim=1).indices


def route_uniform(T: int, E: int, top_k: int, seed: int = 3) -> torch.Tensor:
    """[T, top_k] expert ids, uniform distinct routing."""
    return _gumbel_topk(torch.zeros(E), T, top_k, _gen(seed))


def route_skewed(T: int, E: int, top_k: int, alpha: float = 0.5, seed: int = 3,
                 popularity_seed: int | None = None) -> torch.Tensor:
    """[T, top_k] expert ids with Zipf-like skew.  The popularity order of the
    experts is drawn from `seed` unless `popularity_seed` is given: two batches with the same
    popularity_seed and different seeds are independent draws of one routing distribution (the
    "observed statistics" of a previous batch)."""
    g = _gen(seed)
    perm = torch.randperm(E, generator=g)
    if popularity_seed is not None:
        perm = torch.randperm(E, generator=_gen(popularity_seed))
    rank = torch.empty(E, dtype=torch.float64)
    rank[perm] = torch.arange(E, dtype=torch.float64)
    logw = -alpha * torch.log(rank + 1.0)
    return _gumbel_topk(logw, T, top_k, g)


def group_rows(routes: torch.Tensor, E: int):
    """Sort the (token, slot) pairs by (expert, token).  Returns (token_index[R] int64,
    offsets[E+1] int64): rows of expert e are token_index[offsets[e]:offsets[e+1]].
    Pure bookkeeping (a stable sort); no arithmetic of the method."""
    T, k = routes.shape
    flat_e = routes.reshape(-1).to(torch.int64)
    flat_t = torch.arange(T, dtype=torch.int64).repeat_interleave(k)
    key = flat_e * T + flat_t
    order = torch.argsort(key, stable=True)
    counts = torch.bincount(flat_e, minlength=E)
    offsets = torch.zeros(E + 1, dtype=torch.int64)
    offsets[1:] = torch.cumsum(counts, 0)
    return flat_t[order], offsets


def codes_small(R: int, C: int, seed: int) -> torch.Tensor:
    """uint8 [R, C] E4M3 codes drawn from {0, +-1, +-2} (closed-form GEMM operands)."""
    idx = torch.randint(0, len(E4M3_SMALL_CODES), (R, C), generator=_gen(seed))
    return torch.tensor(E4M3_SMALL_CODES, dtype=torch.uint8)[idx]


def scales_pow2(*shape: int, seed: int) -> torch.Tensor:
    """float32 scales drawn from {1, 2, 4} (closed-form GEMM operands)."""
    idx = torch.randint(0, 3, shape, generator=_gen(seed))
    return torch.tensor([1.0, 2.0, 4.0], dtype=torch.float32)[idx]


def special_values_act(M: int, K: int, seed: int = 7) -> torch.Tensor:
    """FP32 edge-case activations: signed zeros, subnormals, tiny/huge magnitudes,
    the 448 boundary, exact E4M3 ties, all-zero tiles.  Finite only (non-finite
    inputs are a separate, explicitly-labelled test)."""
    g = _gen(seed)
    x = torch.randn(M, K, generator=g, dtype=torch.float32)
    mags = torch.tensor([0.0, -0.0, 1e-45, -1e-45, 1e-40, 2.0 ** -126, 1e-30, 1e-10,
                         448.0, 449.0, 464.0, 465.0, 3.0, 17.0, 19.0, 232.0, 248.0,
                         1e30, -1e30, 3.0e38, -3.0e38], dtype=torch.float32)
    sel = torch.randint(0, mags.numel(), (M, K), generator=g)
    use = torch.rand(M, K, generator=g) < 0.25
    # scale rows to stress scale ranges (gaussian part only, stays finite)
    row_scale = torch.tensor([1.0, 1e-38, 1e-20, 1e20, 2.0 ** -100, 1.0], dtype=torch.float32)
    rs = row_scale[torch.randint(0, row_scale.numel(), (M,), generator=g)]
    x = torch.where(use, mags[sel], x * rs[:, None])
    if K >= 128 and M >= 2:
        x[1, :128] = 0.0
        x[0, : min(K, 256)] = -0.0
    return x


def nonfinite_act(M: int, K: int, seed: int = 8) -> torch.Tensor:
    """FP32 activations with NaN and +-Inf elements (reading R6): N(0,1) with ~2% NaN,
    ~1% +Inf and ~1% -Inf scattered, plus whole groups of special content where the shape allows:
    row 0's first 128 channels all NaN; row 1's first 128 channels +Inf except one finite element;
    row 2's first 128 channels a single -Inf among zeros; the first 128 tokens of channel 3 hold a
    NaN and an Inf (a 128x1 group).  Cast to BF16 by the caller if wanted (NaN/Inf survive)."""
    g = _gen(seed)
    x = torch.randn(M, K, generator=g, dtype=torch.float32)
    u = torch.rand(M, K, generator=g)
    x = torch.where(u < 0.02, torch.full_like(x, float("nan")), x)
    x = torch.where((u >= 0.02) & (u < 0.03), torch.full_like(x, float("inf")), x)
    x = torch.where((u >= 0.03) & (u < 0.04), torch.full_like(x, float("-inf")), x)
    w = min(K, 128)
    if M >= 1:
        x[0, :w] = float("nan")
    if M >= 2:
        x[1, :w] = float("inf")
        x[1, 0] = 3.0
    if M >= 3:
        x[2, :w] = 0.0
        x[2, w - 1] = float("-inf")
    if K >= 4:
        h = min(M, 128)
        x[:h, 3] = torch.randn(h, generator=g)
        x[0, 3] = float("nan")
        if h > 1:
            x[h - 1, 3] = float("inf")
    return x


def random_codes(R: int, C: int, seed: int) -> torch.Tensor:
    """uint8 [R, C] uniformly random FINITE E4M3 codes: random bytes, with the two NaN patterns
    (0x7F, 0xFF) moved to the neighbouring +-448 codes (0x7E, 0xFE).  Bookkeeping on bit patterns
    only; used as GEMM operands at full size, where quantizing with the oracle would take minutes."""
    n = R * C
    words = torch.randint(-(2 ** 63), 2 ** 63 - 1, ((n + 7) // 8,), generator=_gen(seed), dtype=torch.int64)
    c = words.view(torch.uint8)[:n].reshape(R, C).clone()
    c[(c & 0x7F) == 0x7F] -= 1
    return c


def random_scales(*shape: int, seed: int, lo: float = 2.0 ** -12, hi: float = 2.0 ** -6) -> torch.Tensor:
    """float32 positive scales log-uniform in [lo, hi) (the range of amax/448 for the init-std
    weights of P:705 up to unit activations)."""
    u = torch.rand(*shape, generator=_gen(seed), dtype=torch.float64)
    return torch.exp(torch.log(torch.tensor(lo, dtype=torch.float64)) * (1 - u)
                     + torch.log(torch.tensor(hi, dtype=torch.float64)) * u).to(torch.float32)
