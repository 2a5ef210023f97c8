"""Experiment: DRAM bytes of the dense C4-shaped Fprop vs M (L2 reuse vs persistent-schedule drift)."""
import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2412_19437_b200 as fp
dev = 'cuda'
K, N = 7168, 2048
for M in (32768, 131072, 524288):
    A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev)
    sA = torch.rand(K // 128, M, device=dev)
    B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device=dev)
    sB = torch.rand(N // 128, K // 128, device=dev)
    out = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    fp.gemm(fp.FPROP, A, sA, B, sB, out=out)
    torch.cuda.synchronize()
    del A, out
