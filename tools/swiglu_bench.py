"""SwiGLU FP8 epilogue cost (experiments only): the expert up-projection (K = 7168 -> 2I = 4096, gate/up
interleaved) timed with BF16 output vs the fused SwiGLU FP8 epilogue (with / without the FP8 cache of
its inputs), dense over 16384 rows and grouped over C4's routing at 8192 tokens x top-8.
Median of N launches with ~10 ms idle between them."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200 as fp
import workloads as W


def med_ms(fn, iters=7):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        torch.cuda._sleep(20_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    dev = "cuda"
    K, N2 = 7168, 4096
    M = 16384
    A = torch.randint(0, 0x7E, (M, K), dtype=torch.uint8, device=dev)
    sA = torch.rand(K // 128, M, device=dev) * 1e-2
    B = torch.randint(0, 0x7E, (N2, K), dtype=torch.uint8, device=dev)
    sB = torch.rand(N2 // 128, K // 128, device=dev) * 1e-3
    out = torch.empty(M, N2, dtype=torch.bfloat16, device=dev)
    fl = 2.0 * M * N2 * K
    for name, fn in (("dense BF16 H", lambda: fp.gemm(fp.FPROP, A, sA, B, sB, out=out)),
                     ("dense SwiGLU FP8 + cache", lambda: fp.gemm_swiglu(A, sA, B, sB)),
                     ("dense SwiGLU FP8", lambda: fp.gemm_swiglu(A, sA, B, sB, cache=False))):
        ms = med_ms(fn)
        print(f"{name:36s} {ms:7.3f} ms {fl / ms / 1e9:6.0f} TFLOP/s", flush=True)
    E = 256
    _, off = W.group_rows(W.route_skewed(8192, E, 8, seed=3), E)
    R = int(off[-1])
    A4 = torch.randint(0, 0x7E, (R, K), dtype=torch.uint8, device=dev)
    sA4 = torch.rand(K // 128, (R + 3) // 4 * 4, device=dev)[:, :R] * 1e-2
    B4 = torch.randint(0, 0x7E, (E, N2, K), dtype=torch.uint8, device=dev)
    sB4 = torch.rand(E, N2 // 128, K // 128, device=dev) * 1e-3
    o4 = off.to(dev)
    out4 = torch.empty(R, N2, dtype=torch.bfloat16, device=dev)
    fl4 = 2.0 * R * N2 * K
    for name, fn in (("grouped BF16 H", lambda: fp.grouped_gemm(o4, A4, sA4, B4, sB4, out=out4)),
                     ("grouped SwiGLU FP8 + cache", lambda: fp.grouped_gemm_swiglu(o4, A4, sA4, B4, sB4)),
                     ("grouped SwiGLU FP8", lambda: fp.grouped_gemm_swiglu(o4, A4, sA4, B4, sB4, cache=False))):
        ms = med_ms(fn)
        print(f"{name:36s} {ms:7.3f} ms {fl4 / ms / 1e9:6.0f} TFLOP/s  ({R} rows)", flush=True)



def variant_sweep(tokens):
    """Grouped SwiGLU (no cache) under both tile variants (the test-hooks build), uniform top-8 routing
    over 256 experts: where CTA pairs start to pay without folded tiles."""
    dev = "cuda"
    K, N2, E = 7168, 4096, 256
    B4 = torch.randint(0, 0x7E, (E, N2, K), dtype=torch.uint8, device=dev)
    sB4 = torch.rand(E, N2 // 128, K // 128, device=dev) * 1e-3
    for T in tokens:
        _, off = W.group_rows(W.route_uniform(T, E, 8), E)
        R = int(off[-1])
        A4 = torch.randint(0, 0x7E, (R, K), dtype=torch.uint8, device=dev)
        sA4 = torch.rand(K // 128, (R + 3) // 4 * 4, device=dev)[:, :R] * 1e-2
        o4 = off.to(dev)
        for v in (1, 2):
            with fp.forced_variant(v):
                ms = med_ms(lambda: fp.grouped_gemm_swiglu(o4, A4, sA4, B4, sB4, cache=False))
            print(f"tokens {T:6d} ({R // E} rows/expert) variant {v}: {ms:7.3f} ms", flush=True)


if __name__ == "__main__":
    if os.environ.get("SWIGLU_SWEEP"):
        variant_sweep([int(t) for t in os.environ["SWIGLU_SWEEP"].split(",")])
    else:
        main()
