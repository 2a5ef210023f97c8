"""One dense up-projection launch with the SwiGLU FP8 epilogue (+ cache) for ncu (experiments only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200 as fp

dev = "cuda"
M, K, N2 = 16384, 7168, 4096
A = torch.randint(0, 0x7E, (M, K), dtype=torch.uint8, device=dev)
sA = torch.rand(K // 128, M, device=dev) * 1e-2
B = torch.randint(0, 0x7E, (N2, K), dtype=torch.uint8, device=dev)
sB = torch.rand(N2 // 128, K // 128, device=dev) * 1e-3
cache = len(sys.argv) > 1 and sys.argv[1] == "cache"
for _ in range(3):
    fp.gemm_swiglu(A, sA, B, sB, cache=cache)
torch.cuda.synchronize()
