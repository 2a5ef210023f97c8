"""One C4-sized grouped UE8M0 launch (524288 rows, skewed) for ncu (tools/grouped_mx_bench.py's problem)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_19437_b200 as fp  # noqa: E402

dev = "cuda"
g = torch.Generator(device="cpu").manual_seed(0)
G, N, K, R = 256, 2048, 7168, 524288
w = torch.rand(G, generator=g) ** 3.0 + 0.05
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
for _ in range(3):
    fp.grouped_gemm(off, A, sA, B, sB, out=out, mx=True)
    fp.grouped_gemm(off, A, sA, B, sB, out=out)
torch.cuda.synchronize()
