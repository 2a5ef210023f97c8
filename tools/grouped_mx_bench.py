"""fp8bs_grouped_gemm_mx (UE8M0, power-of-two scales) vs fp8bs_grouped_gemm (FP32 promotion) at the
C4 expert shape (experiments only): 256 experts, K=7168, N=2048, 65536 rows (8192 tokens x top-8) with
skewed routing; and C2 (uniform ~128 rows per expert)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200 as fp


def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    dev = "cuda"
    g = torch.Generator(device="cpu").manual_seed(0)
    G, N, K = 256, 2048, 7168
    for name, R, skew in (("C4 skewed 524288 rows", 524288, True), ("C4 skewed 65536 rows", 65536, True),
                          ("C2 uniform 32768 rows", 32768, False)):
        w = torch.rand(G, generator=g) ** (3.0 if skew else 0.0) + 0.05
        counts = torch.floor(w / w.sum() * R).long()
        counts[0] += R - int(counts.sum())
        offsets = torch.zeros(G + 1, dtype=torch.int64)
        offsets[1:] = torch.cumsum(counts, 0)
        A = torch.randint(0, 120, (R, K), dtype=torch.uint8, device=dev)
        B = torch.randint(0, 120, (G, N, K), dtype=torch.uint8, device=dev)
        sA = 2.0 ** torch.randint(-10, -2, (K // 128, R), device=dev).float()
        sB = 2.0 ** torch.randint(-10, -2, (G, N // 128, K // 128), device=dev).float()
        off = offsets.to(dev)
        out = torch.empty(R, N, dtype=torch.bfloat16, device=dev)
        out2 = torch.empty(R, N, dtype=torch.bfloat16, device=dev)
        ms0 = timeit(lambda: fp.grouped_gemm(off, A, sA, B, sB, out=out))
        ms1 = timeit(lambda: fp.grouped_gemm(off, A, sA, B, sB, out=out2, mx=True))
        fl = 2.0 * R * N * K
        same = float((out.float() - out2.float()).abs().max() / out.float().abs().max())
        print(f"{name}: promotion {ms0 * 1e3:7.1f} us {fl / ms0 / 1e9:6.0f} TFLOP/s | mx {ms1 * 1e3:7.1f} us "
              f"{fl / ms1 / 1e9:6.0f} TFLOP/s | max rel diff {same:.2e}", flush=True)


if __name__ == "__main__":
    main()
