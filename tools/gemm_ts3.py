"""MMA issue timeline of CTA 0 (FP8BS_GEMM_DEBUG=16): per K-block, cycles from full_ok to each MMA issue."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2412_19437_b200 as fp
M, N, K = 4096, 18432, 7168
dev = "cuda"
A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev)
B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device=dev)
sA = torch.rand(K // 128, M, device=dev)
sB = torch.rand(N // 128, K // 128, device=dev)
out = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
for _ in range(3):
    fp.gemm(fp.FPROP, A, sA, B, sB, out=out)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (12 * 512))()
fp.lib().fp8bs_internal_debug_timestamps(buf, 12 * 512)
t = np.array(buf, dtype=np.int64).reshape(12, 512)
n = int((t[2] > 0).sum())
sl = slice(60, n - 2)
print("median (cycles):  pempty_ok->full_ok", np.median((t[1] - t[0])[sl]),
      " full_ok->mma0", np.median((t[8] - t[1])[sl]), " mma0->mma1", np.median((t[9] - t[8])[sl]),
      " mma1->mma2", np.median((t[10] - t[9])[sl]), " mma2->mma3", np.median((t[11] - t[10])[sl]),
      " mma3->committed", np.median((t[2] - t[11])[sl]))
print("median committed(kb) -> pempty_ok(kb+1):", np.median(t[0, 61:n - 1] - t[2, 60:n - 2]))
print("median pfull_ok(kb) on last promo warp - committed(kb):", np.median((t[6] - t[2])[sl]))
print("median promo: pfull_ok -> last arrive:", np.median((t[7] - t[6])[sl]))
for kb in range(100, 104):
    print(kb, [int(t[i, kb] - t[0, 100]) for i in (0, 1, 8, 9, 10, 11, 2, 5, 6, 7)])
