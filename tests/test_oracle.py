"""Pins for the CPU oracle (runs without a GPU).

The oracle is pinned to things other than itself:
  * the E4M3 bit definition's invariants and torch's float8_e4m3fn decoder;
  * an independent brute-force nearest-value search (numpy) and torch's own cast in
    the non-saturating range, for the encoder;
  * hand-derived goldens (tests/golden/e4m3_worked_example.txt);
  * closed forms for the quantizers (power-of-two scales -> exact recovery) and the
    GEMM (small-integer operands -> exact arithmetic in any order);
  * numpy float64 matmul of dequantized operands; a naive numpy re-implementation of
    the groupings on tiny tensors; transpose / permutation invariants.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle
import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "e4m3_worked_example.txt")


# ------------------------------------------------------------------ helpers ----
def torch_decode_table() -> np.ndarray:
    """E4M3 values of codes 0..255 from torch's float8_e4m3fn (independent decoder)."""
    return torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).to(torch.float64).numpy()


MAGS = torch_decode_table()[:127]          # codes 0x00..0x7E: 0 .. 448, ascending


def brute_encode(y: np.ndarray) -> np.ndarray:
    """Nearest finite E4M3 magnitude by exhaustive distance over all 127 non-negative
    finite values, ties -> even code (the mantissa LSB is the code LSB), the sign copied
    from y.  Inf saturates to 448 (satfinite); NaN -> 0x7F."""
    y = np.asarray(y, dtype=np.float32)
    out = np.empty(y.shape, dtype=np.uint8)
    flat = y.reshape(-1)
    res = out.reshape(-1)
    for s in range(0, flat.size, 1 << 15):
        v = flat[s:s + (1 << 15)]
        a = np.abs(v.astype(np.float64))
        finite = np.isfinite(a)
        # every candidate is <= 448, so for |y| >= 448 the distance ORDER does not depend
        # on |y|; clipping to 1024 keeps a - m exact in float64 (no false ties).
        a2 = np.minimum(np.where(finite, a, 0.0), 1024.0)
        d = np.abs(a2[:, None] - MAGS[None, :])              # [n, 127] brute force
        dmin = d.min(axis=1, keepdims=True)
        cand = d == dmin
        codes = np.arange(127)[None, :]
        # among equidistant candidates prefer the even code
        even = cand & (codes % 2 == 0)
        pick = np.where(even.any(axis=1), np.argmax(even, axis=1), np.argmax(cand, axis=1))
        pick = np.where(np.isinf(v), 126, pick)
        c = pick.astype(np.uint8) | np.where(np.signbit(v), 0x80, 0).astype(np.uint8)
        c = np.where(np.isnan(v), 0x7F, c)
        res[s:s + v.size] = c
    return out


def oracle_encode(y: np.ndarray) -> np.ndarray:
    return oracle.encode_tensor(torch.from_numpy(np.ascontiguousarray(y, dtype=np.float32))).numpy()


def naive_quant_groups(x: np.ndarray, groups):
    """Naive numpy grouping quantizer: for each group (list of flat indices) compute the
    float32 amax, s = f32(amax)/f32(448) (1 if 0), codes = brute_encode(f32(x)/s)."""
    x = x.astype(np.float32)
    q = np.zeros(x.shape, dtype=np.uint8)
    scales = []
    for idx in groups:
        v = x[idx]
        amax = np.float32(np.max(np.abs(v))) if v.size else np.float32(0)
        s = np.float32(amax) / np.float32(448.0)
        if s == 0:
            s = np.float32(1.0)
        q[idx] = brute_encode((v / s).astype(np.float32))
        scales.append(s)
    return q, scales


# ------------------------------------------------------------ E4M3 table ----
def test_decode_table_invariants():
    t = oracle.decode_table().numpy()
    assert np.isnan(t[0x7F]) and np.isnan(t[0xFF])
    assert np.isfinite(t).sum() == 254
    assert t[0x7E] == 448.0 and t[0xFE] == -448.0           # max finite
    assert t[0x08] == 2.0 ** -6                             # min normal
    assert t[0x01] == 2.0 ** -9                             # min subnormal
    assert t[0x00] == 0.0 and t[0x80] == 0.0 and math.copysign(1, t[0x80]) < 0
    pos = t[:127]
    assert np.all(np.diff(pos) > 0)                         # monotone in code
    assert np.all(t[128:255] == -pos)                       # sign symmetry
    assert ((pos > 0) & (pos < 2.0 ** -6)).sum() == 7       # 7 subnormals
    assert (pos >= 2.0 ** -6).sum() == 119                  # 119 normals


def test_decode_matches_torch_float8():
    t = oracle.decode_table().numpy()
    ref = torch_decode_table()
    fin = np.isfinite(ref)
    assert np.array_equal(np.isnan(t), np.isnan(ref))
    assert np.array_equal(t[fin], ref[fin])
    assert np.array_equal(np.signbit(t[fin]), np.signbit(ref[fin]))


def test_encode_decode_roundtrip_all_codes():
    t = oracle.decode_table().numpy()
    for c in range(256):
        if np.isnan(t[c]):
            continue
        assert oracle.e4m3_encode(float(t[c])) == c, hex(c)


def test_spec_codec_examples():
    # 0.0 <-> code 0; 1.0 exact; encode(449) saturates to 448.
    assert oracle.e4m3_encode(0.0) == 0x00
    assert oracle.e4m3_decode(oracle.e4m3_encode(1.0)) == 1.0
    assert oracle.e4m3_decode(oracle.e4m3_encode(449.0)) == 448.0
    assert oracle.e4m3_encode(float("inf")) == 0x7E and oracle.e4m3_encode(float("-inf")) == 0xFE
    assert oracle.e4m3_encode(float("nan")) == 0x7F


# ------------------------------------------------------------- encoder ----
def _encoder_probe_values() -> np.ndarray:
    rng = np.random.default_rng(1234)
    vals = [MAGS.astype(np.float32)]
    mids = ((MAGS[1:] + MAGS[:-1]) / 2).astype(np.float32)   # exact in binary32
    vals.append(mids)
    base = np.concatenate(vals)
    up = np.nextafter(base, np.float32(np.inf))
    dn = np.nextafter(base, np.float32(-np.inf))
    rand_bits = rng.integers(0, 2 ** 32, size=1 << 18, dtype=np.uint64).astype(np.uint32).view(np.float32)
    rand_bits = rand_bits[~np.isnan(rand_bits)]
    uni = rng.uniform(-520, 520, size=1 << 18).astype(np.float32)
    small = (rng.standard_normal(1 << 17) * 2.0 ** rng.integers(-14, 2, 1 << 17)).astype(np.float32)
    special = np.array([0.0, -0.0, np.inf, -np.inf, 1e-45, -1e-45, 448, 449, 463.99997, 464,
                        464.00003, 480, 1e38, 2.0 ** -10, 2.0 ** -11, 3 * 2.0 ** -11], dtype=np.float32)
    allv = np.concatenate([base, up, dn, rand_bits, uni, small, special])
    return np.concatenate([allv, -allv]).astype(np.float32)


def test_encoder_vs_bruteforce_nearest():
    v = _encoder_probe_values()
    got = oracle_encode(v)
    ref = brute_encode(v)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, [(float(v[i]), hex(got[i]), hex(ref[i])) for i in bad[:10]]


def test_encoder_vs_torch_cast_nonsaturating_range():
    # torch's cast is RNE but NON-saturating (|x| > 464 -> NaN, R3), so only
    # compare where both agree on semantics: |x| <= 448.
    rng = np.random.default_rng(7)
    v = np.concatenate([rng.uniform(-448, 448, 1 << 18),
                        rng.standard_normal(1 << 18) * 2.0 ** rng.integers(-16, 8, 1 << 18)]).astype(np.float32)
    v = v[np.abs(v) <= 448]
    ref = torch.from_numpy(v).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    got = oracle_encode(v)
    assert np.array_equal(got, ref)


def test_encoder_monotone():
    v = np.sort(np.random.default_rng(3).uniform(-500, 500, 1 << 16).astype(np.float32))
    dec = oracle.decode_table().numpy()[oracle_encode(v)]
    assert np.all(np.diff(dec) >= 0)


# ------------------------------------------------------------ goldens ----
def _read_golden():
    tiles = []
    for line in open(GOLDEN):
        line = line.split("#")[0].strip()
        if not line:
            continue
        f = line.split()
        if f[0] == "tile":
            tiles.append({"scale": float.fromhex(f[3]), "xs": [], "codes": []})
        else:
            x = float.fromhex(f[1]) if f[1].startswith(("0x", "-0x")) else float(f[1])
            tiles[-1]["xs"].append(x)
            tiles[-1]["codes"].append(int(f[3], 16))
    return tiles


def test_golden_worked_example():
    tiles = _read_golden()
    assert len(tiles) == 3
    x = torch.zeros(len(tiles), 128, dtype=torch.float32)
    for r, t in enumerate(tiles):
        x[r, :len(t["xs"])] = torch.tensor(t["xs"], dtype=torch.float32)
    q, s = oracle.quantize_act_1x128(x)
    # s = 3/448 for amax 3.0 (binary32 quotient, computed here by numpy).
    assert s[0, 0].item() == float(np.float32(3.0) / np.float32(448.0))
    for r, t in enumerate(tiles):
        assert s[0, r].item() == t["scale"], r
        n = len(t["xs"])
        assert q[r, :n].tolist() == t["codes"], (r, [hex(c) for c in q[r, :n].tolist()])
        assert torch.all(q[r, n:] == 0)


def test_spec_quantize_examples():
    # all-zero tile -> scale 1, codes 0.  S:378: amax 3.0 -> s ~= 0.0066964.
    q, s = oracle.quantize_act_1x128(torch.zeros(2, 256))
    assert torch.all(s == 1.0) and torch.all(q == 0)
    x = torch.zeros(1, 128)
    x[0, 5] = -3.0
    q, s = oracle.quantize_act_1x128(x)
    assert abs(s.item() - 0.0066964) < 1e-7
    assert q[0, 5].item() == 0xFE


# --------------------------------------------------------- quantizers ----
def _closed_form_tile(rng, n, s0):
    """A group whose scale is exactly s0 (power of two) and whose codes are recovered:
    values s0*e with e on the E4M3 grid, one element = 448*s0 (=amax)."""
    codes = rng.integers(0, 127, n).astype(np.uint8)
    codes = codes | (rng.integers(0, 2, n).astype(np.uint8) << 7)
    codes[rng.integers(0, n)] = 0x7E
    vals = torch_decode_table()[codes] * s0
    return codes, vals


@pytest.mark.parametrize("s0", [2.0 ** -20, 2.0 ** -3, 1.0, 2.0 ** 10])
def test_quant_1x128_closed_form_exact_recovery(s0):
    rng = np.random.default_rng(11)
    M, K = 3, 384
    x = np.zeros((M, K), np.float32)
    want = np.zeros((M, K), np.uint8)
    for m in range(M):
        for kb in range(K // 128):
            c, v = _closed_form_tile(rng, 128, s0)
            x[m, kb * 128:(kb + 1) * 128] = v
            want[m, kb * 128:(kb + 1) * 128] = c
    # -0 codes (0x80) decode to -0.0 and re-encode to 0x80; all recovered exactly.
    q, s = oracle.quantize_act_1x128(torch.from_numpy(x))
    assert torch.all(s == s0)
    assert np.array_equal(q.numpy(), want)


def test_quant_weight_closed_form_exact_recovery():
    rng = np.random.default_rng(12)
    N, K, s0 = 256, 256, 2.0 ** -7
    w = np.zeros((N, K), np.float32)
    want = np.zeros((N, K), np.uint8)
    for nb in range(2):
        for kb in range(2):
            c, v = _closed_form_tile(rng, 128 * 128, s0)
            w[nb * 128:(nb + 1) * 128, kb * 128:(kb + 1) * 128] = v.reshape(128, 128)
            want[nb * 128:(nb + 1) * 128, kb * 128:(kb + 1) * 128] = c.reshape(128, 128)
    q, s, qT = oracle.quantize_weight_128x128(torch.from_numpy(w))
    assert torch.all(s == s0)
    assert np.array_equal(q.numpy(), want)
    assert np.array_equal(qT.numpy(), want.T)


@pytest.mark.parametrize("M,K", [(3, 300), (2, 128), (1, 5)])
def test_quant_1x128_vs_naive_groups(M, K):
    x = W.special_values_act(M, K, seed=M * 1000 + K).numpy()
    x = np.where(np.isfinite(x), x, 0).astype(np.float32)
    groups = [np.ravel_multi_index((np.full(min(128, K - k0), m), np.arange(k0, min(K, k0 + 128))), (M, K))
              for m in range(M) for k0 in range(0, K, 128)]
    qn, sn = naive_quant_groups(x.reshape(-1), groups)
    q, s = oracle.quantize_act_1x128(torch.from_numpy(x))
    assert np.array_equal(q.numpy().reshape(-1), qn)
    KB = (K + 127) // 128
    assert np.array_equal(s.numpy(), np.array(sn, np.float32).reshape(M, KB).T)


@pytest.mark.parametrize("M,C", [(300, 3), (128, 2), (5, 4)])
def test_quant_128x1_vs_naive_groups(M, C):
    x = W.gaussian_act(M, C, seed=5).float().numpy() * np.float32(3.0)
    groups = [np.ravel_multi_index((np.arange(m0, min(M, m0 + 128)), np.full(min(128, M - m0), c)), (M, C))
              for c in range(C) for m0 in range(0, M, 128)]
    qn, sn = naive_quant_groups(x.reshape(-1), groups)
    qT, sT = oracle.quantize_act_128x1(torch.from_numpy(x))
    assert np.array_equal(qT.numpy(), qn.reshape(M, C).T)
    MB = (M + 127) // 128
    assert np.array_equal(sT.numpy(), np.array(sn, np.float32).reshape(C, MB).T)


@pytest.mark.parametrize("N,K", [(130, 200), (128, 128), (64, 300)])
def test_quant_weight_vs_naive_groups(N, K):
    w = W.master_weight(N, K, seed=9).numpy()
    groups, keys = [], []
    for n0 in range(0, N, 128):
        for k0 in range(0, K, 128):
            nn, kk = np.meshgrid(np.arange(n0, min(N, n0 + 128)), np.arange(k0, min(K, k0 + 128)), indexing="ij")
            groups.append(np.ravel_multi_index((nn.ravel(), kk.ravel()), (N, K)))
    qn, sn = naive_quant_groups(w.reshape(-1), groups)
    q, s, qT = oracle.quantize_weight_128x128(torch.from_numpy(w))
    assert np.array_equal(q.numpy().reshape(-1), qn)
    assert np.array_equal(qT.numpy(), q.numpy().T)
    assert np.array_equal(s.numpy().reshape(-1), np.array(sn, np.float32))


def test_quant_invariants_transpose_and_permutation():
    x = W.outlier_act(200, 260, seed=4)
    q1, s1 = oracle.quantize_act_1x128(x)
    qT, sT = oracle.quantize_act_128x1(x.t().contiguous())
    assert torch.equal(qT, q1) and torch.equal(sT, s1)      # 128x1(X^T) == 1x128(X)
    perm = torch.randperm(200, generator=torch.Generator().manual_seed(0))
    qp, sp = oracle.quantize_act_1x128(x[perm])
    assert torch.equal(qp, q1[perm]) and torch.equal(sp, s1[:, perm])   # dispatch commutes
    w = W.master_weight(300, 200, seed=3)
    qa, sa, _ = oracle.quantize_weight_128x128(w)
    qb, sb, _ = oracle.quantize_weight_128x128(w.t().contiguous())
    assert torch.equal(qb, qa.t()) and torch.equal(sb, sa.t())


def test_fine_grained_beats_tensorwise_on_outliers():
    # with one element x1000 per row, 1x128 error <= tensor-wise error.
    x = W.outlier_act(64, 1024, seed=1).float()
    q, s = oracle.quantize_act_1x128(x)
    dec = torch.from_numpy(torch_decode_table())
    deq = dec[q.long()] * s.t().repeat_interleave(128, dim=1)[:, :1024].double()
    err_tile = (deq - x.double()).abs().mean().item()
    amax = x.abs().max()
    st = (amax / 448.0).item()
    qt = oracle.encode_tensor(x / st)
    err_tensor = (dec[qt.long()] * st - x.double()).abs().mean().item()
    assert err_tile < err_tensor


# ---------------------------------------------------------------- GEMM ----
def _expand_scale_b(layout, sB, N, KB):
    """sB(kb, j) as a dense [KB, N] float64 matrix, from the layout's index rule."""
    j = torch.arange(N)
    if layout == oracle.FPROP:
        return sB.double()[j // 128, :].t()
    if layout == oracle.DGRAD:
        return sB.double()[:, j // 128]
    return sB.double()


def _exact_reference(layout, A, sA, B, sB):
    """Closed form for small-integer operands: P_kb = intA_kb @ intB_kb^T exactly (int64),
    then sum_kb sA*sB*P_kb with all terms integers < 2^53 (exact in float64)."""
    dec = torch.from_numpy(torch_decode_table())
    Ai = dec[A.long()].to(torch.int64)
    Bi = dec[B.long()].to(torch.int64)
    M, K = A.shape
    N = B.shape[0]
    KB = K // 128
    sBx = _expand_scale_b(layout, sB, N, KB)
    O = torch.zeros(M, N, dtype=torch.float64)
    for kb in range(KB):
        P = Ai[:, kb * 128:(kb + 1) * 128] @ Bi[:, kb * 128:(kb + 1) * 128].t()
        O += sA[kb].double()[:, None] * sBx[kb][None, :] * P.double()
    return O


@pytest.mark.parametrize("layout", [oracle.FPROP, oracle.DGRAD, oracle.WGRAD])
def test_gemm_closed_form_exact(layout):
    M, N, K = 96, 200, 384
    KB = K // 128
    A = W.codes_small(M, K, seed=1)
    B = W.codes_small(N, K, seed=2)
    sA = W.scales_pow2(KB, M, seed=3)
    NB = (N + 127) // 128
    sB = {oracle.FPROP: W.scales_pow2(NB, KB, seed=4), oracle.DGRAD: W.scales_pow2(KB, NB, seed=4),
          oracle.WGRAD: W.scales_pow2(KB, N, seed=4)}[layout]
    O = oracle.gemm(layout, A, sA, B, sB)
    ref = _exact_reference(layout, A, sA, B, sB)
    assert torch.equal(O, ref)


@pytest.mark.parametrize("layout", [oracle.FPROP, oracle.DGRAD, oracle.WGRAD])
def test_gemm_vs_numpy_dequantized_matmul(layout):
    g = torch.Generator().manual_seed(5)
    M, N, K = 64, 160, 512
    KB, NB = K // 128, (N + 127) // 128
    A = torch.randint(0, 256, (M, K), generator=g, dtype=torch.uint8)
    B = torch.randint(0, 256, (N, K), generator=g, dtype=torch.uint8)
    A[A & 0x7F == 0x7F] = 0x00   # no NaN codes
    B[B & 0x7F == 0x7F] = 0x00
    sA = torch.rand(KB, M, generator=g) + 0.01
    sB = {oracle.FPROP: torch.rand(NB, KB, generator=g), oracle.DGRAD: torch.rand(KB, NB, generator=g),
          oracle.WGRAD: torch.rand(KB, N, generator=g)}[layout] + 0.01
    dec = torch_decode_table()
    dA = dec[A.numpy()] * np.repeat(sA.double().numpy().T, 128, axis=1)
    dB = dec[B.numpy()] * np.repeat(_expand_scale_b(layout, sB, N, KB).numpy().T, 128, axis=1)
    ref = dA @ dB.T
    O = oracle.gemm(layout, A, sA, B, sB).numpy()
    assert np.max(np.abs(O - ref)) / np.max(np.abs(ref)) < 1e-13


def test_gemm_identity_gives_dequant():
    # identity (exactly representable) x X in full precision = dequant(quant(X)).
    x = W.outlier_act(40, 256, seed=2)
    q, s = oracle.quantize_act_1x128(x)
    I = torch.zeros(256, 256, dtype=torch.uint8)
    I[torch.arange(256), torch.arange(256)] = 0x38           # E4M3 1.0
    O = oracle.gemm(oracle.FPROP, q, s, I, torch.ones(2, 2))
    dec = torch.from_numpy(torch_decode_table())
    deq = dec[q.long()] * s.t().double().repeat_interleave(128, dim=1)
    assert torch.equal(O, deq)


def test_gemm_row_sampling_matches_full():
    A = W.codes_small(50, 256, seed=8)
    B = W.codes_small(30, 256, seed=9)
    sA = torch.rand(2, 50) + 0.5
    sB = torch.rand(1, 2) + 0.5
    full = oracle.gemm(oracle.FPROP, A, sA, B, sB)
    rows = torch.tensor([49, 0, 17])
    part = oracle.gemm(oracle.FPROP, A, sA, B, sB, rows=rows)
    assert torch.equal(part, full[rows])


def test_grouped_gemm_equals_per_expert_gemm():
    G, N, K = 5, 136, 256
    counts = [0, 7, 130, 1, 64]
    offsets = torch.tensor([0] + list(np.cumsum(counts)), dtype=torch.int64)
    R = int(offsets[-1])
    A = W.codes_small(R, K, seed=1)
    sA = torch.rand(K // 128, R) + 0.1
    B = torch.stack([W.codes_small(N, K, seed=10 + e) for e in range(G)])
    sB = torch.rand(G, (N + 127) // 128, K // 128) + 0.1
    O = oracle.grouped_gemm(offsets, A, sA, B, sB)
    for e in range(G):
        a, b = int(offsets[e]), int(offsets[e + 1])
        if a == b:
            continue
        ref = oracle.gemm(oracle.FPROP, A[a:b], sA[:, a:b], B[e], sB[e])
        assert torch.equal(O[a:b], ref)


def test_rel_err_normwise():
    O = torch.tensor([1.0, -2.0, 4.0], dtype=torch.float64)
    assert oracle.rel_err_normwise(O, O) == 0.0
    assert abs(oracle.rel_err_normwise(O * 1.01, O) - 0.01) < 1e-15


# ------------------------------------------------------- FP8 -> FP8 re-quantization ----
@pytest.mark.parametrize("M,K", [(300, 200), (128, 256), (5, 130)])
def test_requantize_vs_naive_dequant_then_groups(M, K):
    """requantize_1x128_to_128x1 == an independent composition: dequantize with
    torch's float8 decoder x float64 scale, round once to float32, then the naive 128x1 grouping
    quantizer (brute-force encoder); ragged M and K (short last groups on both axes)."""
    x = W.outlier_act(M, K, seed=4)
    q, s = oracle.quantize_act_1x128(x)
    dec = torch_decode_table()
    xhat = (dec[q.numpy()] * np.repeat(s.numpy().T.astype(np.float64), 128, axis=1)[:, :K]).astype(np.float32)
    groups = [np.ravel_multi_index((np.arange(m0, min(M, m0 + 128)), np.full(min(128, M - m0), c)), (M, K))
              for c in range(K) for m0 in range(0, M, 128)]
    qn, sn = naive_quant_groups(xhat.reshape(-1), groups)
    qT, sT = oracle.requantize_1x128_to_128x1(q, s)
    assert np.array_equal(qT.numpy(), qn.reshape(M, K).T)
    assert np.array_equal(sT.numpy(), np.array(sn, np.float32).reshape(K, (M + 127) // 128).T)


def test_requantize_closed_form_is_a_transpose():
    """Closed form: every value is an E4M3 grid value times one power of two 2^p, and every 1x128 row
    group and every 128x1 column group holds +-448*2^p (a diagonal of 448s in each 128x128 block).
    Both quantizations are then exact with s = 2^p, so the re-quantized codes are the transpose."""
    rng = np.random.default_rng(8)
    M, K, p = 256, 384, -7
    mags = torch_decode_table()[:127]
    v = rng.choice(mags, size=(M, K)) * rng.choice([-1.0, 1.0], size=(M, K))
    r, c = np.meshgrid(np.arange(M), np.arange(K), indexing="ij")
    v = np.where((r % 128) == (c % 128), 448.0, v)
    x = torch.from_numpy((v * 2.0 ** p).astype(np.float32))
    q, s = oracle.quantize_act_1x128(x)
    assert torch.all(s == 2.0 ** p)
    qT, sT = oracle.requantize_1x128_to_128x1(q, s)
    assert torch.all(sT == 2.0 ** p)
    assert torch.equal(qT, q.t().contiguous())


# ------------------------------------------------------------ power-of-two scales ----
def _pow2_scale_exact(amax: float) -> float:
    """Independent reading R23 with exact rationals: the smallest 2^e (e >= -127, R26) with 448 * 2^e >= amax."""
    from fractions import Fraction
    if amax == 0:
        return 1.0
    a = Fraction(amax)
    e = -127
    while Fraction(448) * Fraction(2) ** e < a:
        e += 1
    return float(Fraction(2) ** e)


def test_pow2_scale_spec_example():
    """tile amax 3.0 -> pow2 s = 2^-7 and 3.0 / s = 384 <= 448 (no overflow)."""
    x = torch.zeros(1, 128, dtype=torch.float32)
    x[0, 0], x[0, 1], x[0, 2] = 3.0, 1.0, -0.5
    q, s = oracle.quantize_act_1x128_pow2(x)
    assert float(s[0, 0]) == 2.0 ** -7
    assert oracle.e4m3_decode(int(q[0, 0])) == 384.0          # exact: 3 * 2^7
    assert oracle.e4m3_decode(int(q[0, 1])) == 128.0
    assert oracle.e4m3_decode(int(q[0, 2])) == -64.0


@pytest.mark.parametrize("kind", ["gauss", "outlier", "special"])
def test_pow2_quantizer_vs_exact_rationals_and_bruteforce(kind):
    """quantize_act_1x128_pow2 == an independent composition: exact-rational pow2 scale per group, the
    exact quotient x / s (a power-of-two division), brute-force nearest E4M3 code; and |x / s| <= 448
    everywhere (rounding UP never saturates)."""
    M, K = 24, 300
    x = {"gauss": W.gaussian_act, "outlier": W.outlier_act, "special": W.special_values_act}[kind](M, K, seed=12).float()
    q, s = oracle.quantize_act_1x128_pow2(x)
    xn = x.numpy()
    for m in range(M):
        for kb in range((K + 127) // 128):
            v = xn[m, kb * 128:(kb + 1) * 128]
            sc = _pow2_scale_exact(float(np.max(np.abs(v))))
            assert float(s[kb, m]) == np.float32(sc)
            quot = (v.astype(np.float64) / sc).astype(np.float32)     # exact unless below float's range
            assert np.all(np.abs(quot) <= 448.0)
            assert np.array_equal(q[m, kb * 128:(kb + 1) * 128].numpy(), brute_encode(quot))


@pytest.mark.parametrize("kind", ["gauss", "outlier", "special"])
def test_pow2_128x1_and_weight_vs_exact_rationals_and_bruteforce(kind):
    """The 128x1 and 128x128 power-of-two quantizers == the same independent composition as above over
    their groups: exact-rational pow2 scale per group (a 128-token column segment; a 128x128 block),
    the exact quotient, brute-force nearest E4M3 code; the weight's transposed copy is q's transpose."""
    M, C = 300, 260
    x = {"gauss": W.gaussian_act, "outlier": W.outlier_act, "special": W.special_values_act}[kind](M, C, seed=14).float()
    qT, sT = oracle.quantize_act_128x1(x, pow2=True)
    qw, sw, qwT = oracle.quantize_weight_128x128(x, pow2=True)
    xn = x.numpy()
    for mb in range((M + 127) // 128):
        for c in range(C):
            v = xn[mb * 128:(mb + 1) * 128, c]
            sc = _pow2_scale_exact(float(np.max(np.abs(v))))
            assert float(sT[mb, c]) == np.float32(sc)
            quot = (v.astype(np.float64) / sc).astype(np.float32)
            assert np.all(np.abs(quot) <= 448.0)
            assert np.array_equal(qT[c, mb * 128:(mb + 1) * 128].numpy(), brute_encode(quot))
    for nb in range((M + 127) // 128):
        for kb in range((C + 127) // 128):
            v = xn[nb * 128:(nb + 1) * 128, kb * 128:(kb + 1) * 128]
            sc = _pow2_scale_exact(float(np.max(np.abs(v))))
            assert float(sw[nb, kb]) == np.float32(sc)
            quot = (v.astype(np.float64) / sc).astype(np.float32)
            assert np.all(np.abs(quot) <= 448.0)
            assert np.array_equal(qw[nb * 128:(nb + 1) * 128, kb * 128:(kb + 1) * 128].numpy(),
                                  brute_encode(quot.reshape(-1)).reshape(quot.shape))
    assert torch.equal(qwT, qw.t().contiguous())


def test_requantize_pow2_loses_nothing():
    """P:558's rationale for power-of-two scales: re-quantizing pow2-scaled FP8 into 128x1 tiles with
    pow2 scales only shifts exponents, so every dequantized value whose new quotient stays in E4M3's
    normal range (>= 2^-6) is unchanged."""
    M, K = 256, 384
    x = W.gaussian_act(M, K, seed=13)
    q, s = oracle.quantize_act_1x128_pow2(x)
    qT, sT = oracle.requantize_1x128_to_128x1(q, s, pow2=True)
    dec = torch_decode_table()
    s_mk = np.repeat(s.numpy().T.astype(np.float64), 128, axis=1)[:, :K]      # s(k // 128, m) at [m, k]
    sT_mk = np.repeat(sT.numpy().astype(np.float64), 128, axis=0)[:M, :]      # sT(m // 128, k) at [m, k]
    before = dec[q.numpy()] * s_mk
    after = dec[qT.numpy()].T * sT_mk
    normal = np.abs(before) >= sT_mk * 2.0 ** -6
    assert normal.mean() > 0.9
    assert np.array_equal(before[normal], after[normal])


# ------------------------------------------------- input dtypes and non-finite inputs ----
def _quant_all(x):
    q, s = oracle.quantize_act_1x128(x)
    qT, sT = oracle.quantize_act_128x1(x)
    qw, sw, qwT = oracle.quantize_weight_128x128(x)
    p, ps = oracle.quantize_act_1x128_pow2(x)
    pT, psT = oracle.quantize_act_128x1(x, pow2=True)
    return q, s, qT, sT, qw, sw, qwT, p, ps, pT, psT


@pytest.mark.parametrize("kind", ["gauss", "outlier", "special", "nonfinite"])
def test_bf16_input_path_equals_fp32_of_the_same_values(kind):
    """The oracle's BF16 loader (oracle_bf16_to_float) is pinned to torch's BF16 -> FP32 conversion:
    every quantizer gives bit-identical codes and scales on x_bf16 and on x_bf16.float()."""
    M, K = 260, 300
    gen = {"gauss": W.gaussian_act, "outlier": W.outlier_act, "special": W.special_values_act,
           "nonfinite": W.nonfinite_act}[kind]
    xb = gen(M, K, seed=21).to(torch.bfloat16)
    for a, b in zip(_quant_all(xb), _quant_all(xb.float())):
        if a.dtype == torch.float32:
            a, b = a.view(torch.int32), b.view(torch.int32)
        assert torch.equal(a, b)


def naive_quant_groups_maxnum(x: np.ndarray, groups):
    """naive_quant_groups with reading R6 spelled out: the group amax ignores NaN (maxNum; an all-NaN
    group has amax 0, so s = 1); Inf elements give s = Inf; the quotient is IEEE float32 division
    (finite / Inf = +-0, Inf / Inf = NaN); NaN encodes to 0x7F, +-Inf saturates."""
    x = x.astype(np.float32)
    q = np.zeros(x.shape, dtype=np.uint8)
    scales = []
    for idx in groups:
        v = x[idx]
        a = np.abs(v[~np.isnan(v)])
        amax = np.float32(a.max()) if a.size else np.float32(0)
        with np.errstate(invalid="ignore", over="ignore"):
            s = np.float32(amax) / np.float32(448.0)
            if s == 0:
                s = np.float32(1.0)
            q[idx] = brute_encode((v / s).astype(np.float32))
        scales.append(s)
    return q, scales


def test_nonfinite_inputs_follow_reading_R6():
    """NaN / +-Inf inputs (reading R6) through the 1x128, 128x1 and 128x128 quantizers ==
    a naive numpy composition with maxNum amax, IEEE division and the brute-force encoder."""
    M, K = 140, 260
    x = W.nonfinite_act(M, K, seed=3)
    xn = x.numpy()
    rows = [np.ravel_multi_index((np.full(min(128, K - k0), m), np.arange(k0, min(K, k0 + 128))), (M, K))
            for m in range(M) for k0 in range(0, K, 128)]
    qn, sn = naive_quant_groups_maxnum(xn.reshape(-1), rows)
    q, s = oracle.quantize_act_1x128(x)
    assert np.array_equal(q.numpy().reshape(-1), qn)
    assert np.array_equal(s.numpy().view(np.int32), np.array(sn, np.float32).reshape(M, -1).T.view(np.int32))
    cols = [np.ravel_multi_index((np.arange(m0, min(M, m0 + 128)), np.full(min(128, M - m0), c)), (M, K))
            for c in range(K) for m0 in range(0, M, 128)]
    qn, sn = naive_quant_groups_maxnum(xn.reshape(-1), cols)
    qT, sT = oracle.quantize_act_128x1(x)
    assert np.array_equal(qT.numpy(), qn.reshape(M, K).T)
    assert np.array_equal(sT.numpy().view(np.int32), np.array(sn, np.float32).reshape(K, -1).T.view(np.int32))
    blocks = []
    for n0 in range(0, M, 128):
        for k0 in range(0, K, 128):
            nn, kk = np.meshgrid(np.arange(n0, min(M, n0 + 128)), np.arange(k0, min(K, k0 + 128)), indexing="ij")
            blocks.append(np.ravel_multi_index((nn.ravel(), kk.ravel()), (M, K)))
    qn, sn = naive_quant_groups_maxnum(xn.reshape(-1), blocks)
    qw, sw, _ = oracle.quantize_weight_128x128(x)
    assert np.array_equal(qw.numpy().reshape(-1), qn)
    assert np.array_equal(sw.numpy().reshape(-1).view(np.int32), np.array(sn, np.float32).view(np.int32))
    # the special groups of the recipe: all-NaN -> s = 1 and codes 0x7F; Inf group -> s = Inf
    assert float(s[0, 0]) == 1.0 and torch.all(q[0, :128] == 0x7F)
    assert math.isinf(float(s[0, 1]))
    inf = x[1, :128].isinf()
    assert torch.all(q[1, :128][inf] == 0x7F) and torch.all((q[1, :128][~inf] & 0x7F) == 0)


# ------------------------------------------------------ SwiGLU FP8 epilogue (NEXT-2, R27) ----
def _ulp_err(a: float, ref: float) -> float:
    """|a - ref| in units of the binary32 ulp at ref (normal range)."""
    if ref == 0:
        return abs(a)
    e = math.frexp(abs(ref))[1] - 1
    return abs(a - ref) / 2.0 ** (max(e, -126) - 23)


def test_exp32_accuracy_and_specials():
    """The fixed binary32 exp sequence of R27 stays within 2 ulp of the C library's double exp (rounded
    to binary32) over its whole domain [-86, 86]; exact at 0; arguments are clamped to [-86, 86] (NaN
    to -86); rcp32 is within 1 ulp of 1/d over [1, 1e37] and exact at 1."""
    g = torch.Generator().manual_seed(5)
    xs = (torch.rand(200000, generator=g, dtype=torch.float64) * 172.0 - 86.0).to(torch.float32).tolist()
    xs += [0.0, -0.0, 1.0, -1.0, 0.5, 0.3465735902799727, -0.3465735902799727, 86.0, -86.0]
    worst = 0.0
    for x in xs:
        worst = max(worst, _ulp_err(oracle.exp32(x), float(np.float32(math.exp(x)))))
    assert worst <= 2.0, worst
    assert oracle.exp32(0.0) == 1.0 and oracle.exp32(-0.0) == 1.0
    assert oracle.exp32(89.0) == oracle.exp32(86.0) == oracle.exp32(float("inf"))
    assert oracle.exp32(-110.0) == oracle.exp32(-86.0) == oracle.exp32(float("nan"))
    ds = (10.0 ** (torch.rand(50000, generator=g, dtype=torch.float64) * 37)).to(torch.float32).tolist()
    assert max(_ulp_err(oracle.rcp32(d), float(np.float32(1.0 / d))) for d in ds) <= 1.0
    assert oracle.rcp32(1.0) == 1.0 and oracle.rcp32(2.0) == 0.5


def test_swiglu32_matches_double_silu():
    """swiglu32(g, u) = RN(RN(g * rcp32(RN(1 + exp32(-g)))) * u) is within 4 ulp of the double-precision
    g * sigmoid(g) * u, and follows the closed forms: g = 0 -> 0; g >= 20 -> exactly RN(g * u)
    (exp(-g) < ulp(1)/2, so 1 + e rounds to 1 and rcp32(1) = 1); g <= -86 -> |y| < 1e-30 with the
    sign of g * u (the clamped exp keeps sigmoid at ~exp(-86))."""
    g = torch.Generator().manual_seed(6)
    gs = (torch.randn(20000, generator=g) * 4).tolist()
    us = (torch.randn(20000, generator=g) * 2).tolist()
    worst = 0.0
    for a, b in zip(gs, us):
        a, b = float(np.float32(a)), float(np.float32(b))
        ref = a / (1.0 + math.exp(-a)) * b
        worst = max(worst, _ulp_err(oracle.swiglu32(a, b), float(np.float32(ref))))
    assert worst <= 4.0, worst
    assert oracle.swiglu32(0.0, 3.0) == 0.0
    for a, b in ((20.0, 3.0), (32.0, -1.5), (100.0, 0.25), (1000.0, 7.0)):
        assert oracle.swiglu32(a, b) == float(np.float32(a * b))
    y = oracle.swiglu32(-200.0, 5.0)
    assert y < 0 and abs(y) < 1e-30


def test_swiglu_quant_is_the_composition():
    """oracle.swiglu_quant_1x128 = elementwise swiglu32 over the interleaved (gate, up) blocks,
    followed by the pinned 1x128 quantizer; the cache output is the 1x128 quantizer applied to H."""
    M, I = 37, 256
    H = W.gaussian_act(M, 2 * I, seed=12, dtype=torch.float32) * 3
    H[0, :128] = 0.0                    # gate 0 -> y = 0 for output block 0 of row 0 -> s = 1
    H[1, 256:384] = 25.0                # gate >= 20 -> y = RN(g * u) exactly
    qy, sy, qh, sh = oracle.swiglu_quant_1x128(H)
    y = torch.empty(M, I, dtype=torch.float32)
    Hl = H.tolist()
    for m in range(M):
        for c in range(I):
            j, cc = divmod(c, 128)
            y[m, c] = oracle.swiglu32(Hl[m][256 * j + cc], Hl[m][256 * j + 128 + cc])
    rq, rs = oracle.quantize_act_1x128(y)
    assert torch.equal(qy, rq) and torch.equal(sy.view(torch.int32), rs.view(torch.int32))
    hq, hs = oracle.quantize_act_1x128(H)
    assert torch.equal(qh, hq) and torch.equal(sh.view(torch.int32), hs.view(torch.int32))
    assert float(sy[0, 0]) == 1.0 and not (qy[0, :128] & 0x7F).any()
    assert torch.equal(y[1, 128:256], (25.0 * H[1, 384:512]).to(torch.float32))


# ------------------------------------------------------------------ MoE combine (NEXT-3, R28) ----
def test_float_to_bf16_is_torch_rne():
    """The oracle's binary32 -> BF16 rounding equals torch's (round to nearest even) on random, tie,
    subnormal and special values."""
    g = torch.Generator().manual_seed(9)
    x = torch.randn(20000, generator=g) * 10.0 ** torch.randint(-40, 38, (20000,), generator=g).float()
    ties = (torch.randint(0, 0x7F7F, (2000,), generator=g).to(torch.int32) << 16 | 0x8000).view(torch.float32)
    x = torch.cat([x, ties, torch.tensor([0.0, -0.0, float("inf"), -float("inf"), 1e-45, 3.4e38])])
    got = torch.tensor([oracle.lib().oracle_float_to_bf16(float(v)) for v in x.tolist()], dtype=torch.int32)
    want = x.to(torch.bfloat16).view(torch.int16).to(torch.int32) & 0xFFFF
    assert torch.equal(got, want)
    assert (oracle.lib().oracle_float_to_bf16(float("nan")) & 0x7FC0) == 0x7FC0


def test_combine_bf16_closed_form_and_numpy():
    """combine_bf16: one-hot gates select one expert row exactly; unit gates on exactly representable
    values give the exact sum; random gates agree with a float64 numpy composition within BF16's
    rounding (the fmaf chain stays within 2^-20 relative before the final BF16 rounding)."""
    T, k, N = 33, 8, 256
    g = torch.Generator().manual_seed(10)
    y = (torch.randn(T * k, N, generator=g) * 3).to(torch.bfloat16)
    onehot = torch.zeros(T, k)
    pick = torch.randint(0, k, (T,), generator=g)
    onehot[torch.arange(T), pick] = 1.0
    out = oracle.combine_bf16(y, onehot)
    assert torch.equal(out.view(torch.int16), y.view(T, k, N)[torch.arange(T), pick].view(torch.int16))
    yi = torch.randint(-8, 9, (T * k, N), generator=g).to(torch.bfloat16)
    out = oracle.combine_bf16(yi, torch.ones(T, k))
    assert torch.equal(out.float(), yi.float().view(T, k, N).sum(1))
    gates = torch.rand(T, k, generator=g)
    out = oracle.combine_bf16(y, gates)
    ref = (y.double().view(T, k, N) * gates.double()[:, :, None]).sum(1)
    assert torch.all((out.double() - ref).abs() <= ref.abs() * 2.0 ** -8 + 1e-30)
