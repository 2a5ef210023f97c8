"""Timeline summary of one GEMM under FP8BS_GEMM_DEBUG (with the 16 bit set): per-K-block deltas."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2412_19437_b200 as fp
T, IN, OUT = 4096, 7168, 18432
M, N, K = T, OUT, IN
dev = "cuda"
A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev)
B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device=dev)
sA = torch.rand(K // 128, M, device=dev)
sB = torch.rand(N // 128, K // 128, device=dev)
out = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
for _ in range(3):
    fp.gemm(fp.FPROP, A, sA, B, sB, out=out)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (8 * 512))()
fp.lib().fp8bs_internal_debug_timestamps(buf, 8 * 512)
t = np.array(buf, dtype=np.int64).reshape(8, 512)
n = int((t[2] > 0).sum())
for name, row in (("mma_full_ok", 1), ("mma_committed", 2), ("promo_pfull_ok", 6)):
    d = np.diff(t[row, 60:n - 1])
    print(f"{name:16s} delta per kb: median {np.median(d):6.0f}  p10 {np.percentile(d,10):6.0f}  p90 {np.percentile(d,90):6.0f}")
print("first 12 full_ok deltas:", np.diff(t[1, :13]).tolist())
print("kb 56..70 full_ok deltas (tile boundary at 56):", np.diff(t[1, 54:70]).tolist())
