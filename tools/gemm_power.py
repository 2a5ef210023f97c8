"""Is the GEMM power-limited?  Time Fprop at the C1 shape with zero, constant and random operands
(experiments only).  FP8BS_LIB selects another build."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_19437_b200 as fp


def timeit(fn, iters=20):
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


T, IN, OUT = 4096, 7168, 18432
M, N, K = T, OUT, IN
dev = "cuda"
sA = torch.rand(K // 128, M, device=dev)
sB = torch.rand(N // 128, K // 128, device=dev)
out = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
for name, fill in (("zeros", lambda s: torch.zeros(s, dtype=torch.uint8, device=dev)),
                   ("const 0x38", lambda s: torch.full(s, 0x38, dtype=torch.uint8, device=dev)),
                   ("random", lambda s: torch.randint(0, 120, s, dtype=torch.uint8, device=dev)),
                   ("zeros again", lambda s: torch.zeros(s, dtype=torch.uint8, device=dev))):
    A, B = fill((M, K)), fill((N, K))
    ms = timeit(lambda: fp.gemm(fp.FPROP, A, sA, B, sB, out=out))
    print(f"{name:12s} {ms * 1e3:8.1f} us  {2 * M * N * K / ms / 1e9:7.0f} TFLOP/s", flush=True)
