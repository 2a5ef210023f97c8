"""Where does the grouped kernel lose against the dense one? (experiments only)  Same Fprop shape
(K=7168, N=2048) as: dense GEMM; grouped with one expert; grouped with equal 2048-row experts;
grouped with the C4 skewed routing.  FP8BS_LIB selects another build."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200 as fp
import paper_2412_19437_b200._lib as _L
import workloads as W

if os.environ.get("FP8BS_LIB"):
    _L.LIB_PATH = os.environ["FP8BS_LIB"]


def timeit(fn, iters=10):
    for _ in range(2):
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
    N, K, R = 2048, 7168, 65536
    A = torch.randint(0, 120, (R, K), dtype=torch.uint8, device=dev)
    sA = torch.rand(K // 128, R, device=dev)
    for G in (1, 32):
        B = torch.randint(0, 120, (G, N, K), dtype=torch.uint8, device=dev)
        sB = torch.rand(G, N // 128, K // 128, device=dev)
        out = torch.empty(R, N, dtype=torch.bfloat16, device=dev)
        if G == 1:
            ms = timeit(lambda: fp.gemm(fp.FPROP, A, sA, B[0], sB[0], out=out))
            print(f"dense  M={R}            {ms * 1e3:8.1f} us {2 * R * N * K / ms / 1e9:6.0f} TFLOP/s", flush=True)
        offs = torch.arange(G + 1, dtype=torch.int64, device=dev) * (R // G)
        ms = timeit(lambda: fp.grouped_gemm(offs, A, sA, B, sB, out=out))
        print(f"grouped G={G:3d} x {R // G:6d} rows {ms * 1e3:8.1f} us {2 * R * N * K / ms / 1e9:6.0f} TFLOP/s", flush=True)
    E = 256
    _, offs4 = W.group_rows(W.route_skewed(8192, E, 8), E)   # the C4 routing at 1/8 of the tokens
    R4 = int(offs4[-1])
    B = torch.randint(0, 120, (E, N, K), dtype=torch.uint8, device=dev)
    sB = torch.rand(E, N // 128, K // 128, device=dev)
    A4, sA4 = A[:R4].contiguous(), sA[:, :R4].contiguous()
    out = torch.empty(R4, N, dtype=torch.bfloat16, device=dev)
    o4 = offs4.to(dev)
    ms = timeit(lambda: fp.grouped_gemm(o4, A4, sA4, B, sB, out=out))
    print(f"grouped C4 routing (8192 tok, {R4} rows) {ms * 1e3:8.1f} us {2 * R4 * N * K / ms / 1e9:6.0f} TFLOP/s", flush=True)
    # the matching expert Dgrad: dY [R4, 2048] x W_e -> dX [R4, 7168] (contraction over the 2048 outputs)
    Bd = torch.randint(0, 120, (E, K, N), dtype=torch.uint8, device=dev)        # WqT_e [in=7168, out=2048]
    sBd = torch.rand(E, N // 128, K // 128, device=dev)
    dYq = torch.randint(0, 120, (R4, N), dtype=torch.uint8, device=dev)
    sdY = torch.rand(N // 128, R4, device=dev)
    dX = torch.empty(R4, K, dtype=torch.bfloat16, device=dev)
    ms = timeit(lambda: fp.grouped_gemm(o4, dYq, sdY, Bd, sBd, out=dX, layout=fp.DGRAD))
    print(f"grouped Dgrad C4 routing ({R4} rows)      {ms * 1e3:8.1f} us {2 * R4 * N * K / ms / 1e9:6.0f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
