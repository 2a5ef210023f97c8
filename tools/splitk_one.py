"""One C1 Dgrad (or --qlora) launch with and without the split-K tail, for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_19437_b200 as fp  # noqa: E402

dev = torch.device("cuda")
layout, M, N, K = (fp.FPROP, 16384, 1536, 7168) if "--qlora" in sys.argv else (fp.DGRAD, 4096, 7168, 18432)
A = torch.randint(0, 126, (M, K), dtype=torch.uint8, device=dev)
B = torch.randint(0, 126, (N, K), dtype=torch.uint8, device=dev)
sA = torch.rand(K // 128, M, device=dev) + 0.5
nb = (N + 127) // 128
sB = torch.rand(*((K // 128, nb) if layout == fp.DGRAD else (nb, K // 128)), device=dev) + 0.5
out = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
ws = torch.empty(fp.gemm_workspace_size(layout, M, N, K), dtype=torch.uint8, device=dev)
for _ in range(3):
    fp.gemm(layout, A, sA, B, sB, out=out, workspace=ws)
    fp.gemm(layout, A, sA, B, sB, out=out, workspace=None)
torch.cuda.synchronize()
