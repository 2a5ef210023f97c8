"""Run one GEMM with FP8BS_GEMM_DEBUG=16(+x) and print the per-K-block pipeline timeline of CTA 0."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2412_19437_b200 as fp

layout = sys.argv[1] if len(sys.argv) > 1 else "fprop"
T, IN, OUT = 4096, 7168, 18432
M, N, K = {"fprop": (T, OUT, IN), "dgrad": (T, IN, OUT), "wgrad": (OUT, IN, T)}[layout]
L = {"fprop": fp.FPROP, "dgrad": fp.DGRAD, "wgrad": fp.WGRAD}[layout]
dev = "cuda"
A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev)
B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device=dev)
sA = torch.rand(K // 128, M, device=dev)
sB = {fp.FPROP: torch.rand(N // 128, K // 128, device=dev), fp.DGRAD: torch.rand(K // 128, N // 128, device=dev),
      fp.WGRAD: torch.rand(K // 128, N, device=dev)}[L]
out = torch.empty(M, N, dtype=torch.float32 if L == fp.WGRAD else torch.bfloat16, device=dev)
for _ in range(3):
    fp.gemm(L, A, sA, B, sB, out=out)
torch.cuda.synchronize()
lib = fp.lib()
buf = (ctypes.c_ulonglong * (12 * 512))()
lib.fp8bs_internal_debug_timestamps(buf, 12 * 512)
t = np.array(buf, dtype=np.int64).reshape(12, 512)
names = ["i0_pempty_ok", "i0_full_ok", "i0_committed", "p4_wait0", "p4_ok0", "pL_wait0", "pL_ok0", "pL_rel0", "pL_wait1", "pL_ok1", "pL_rel1", "pL_sfull_ok"]
t0 = t[0, 0]
n = int((t[2] > 0).sum())
print(f"{layout} K-blocks recorded: {n}")
for kb in list(range(0, 12)) + list(range(100, 108)):
    print(kb, " ".join(f"{names[i]}={t[i, kb] - t0:>8d}" for i in range(12)))
d = np.diff(t[2, 60:n - 1])
print("median cycles per K-block (commit to commit, steady):", np.median(d))
print("median pfull-ok -> last-arrive (promotion of one kb):", np.median((t[7] - t[6])[60:n - 1]))
print("median commit(kb) -> pfull_ok(kb) on last warp:", np.median((t[6] - t[2])[60:n - 1]))
nb = int(os.environ.get("NBUF", "2")); m = min(n - 1 - nb, 400); print("median last-arrive(kb) -> mma pempty_ok(kb+nbuf):", np.median(t[0, 60 + nb:m + nb] - t[7, 60:m]))
print("median mma pempty_ok -> full_ok:", np.median((t[1] - t[0])[60:n - 1]), " full_ok -> committed:", np.median((t[2] - t[1])[60:n - 1]))
