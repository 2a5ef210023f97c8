"""Slot-turnaround timeline of the leader CTA of cluster 0 for the C1 Fprop GEMM (experiments only).
Needs a library built with -DFP8BS_GEMM_DEBUG_BITS=16 (clock64 stamps; see gemm.cu FP8BS_TS):
    tools/build_rev.sh WORKTREE ts -DFP8BS_GEMM_DEBUG_BITS=16
    FP8BS_LIB=tools/libfp8bs_ts.so python tools/gemm_trace.py [fprop|dgrad|wgrad]
Slots (K-block index = the CTA's running K-block count): 0 issuer h0 slot free, 1 issuer h0 stage full,
2 issuer h0 after commit, 3/4 warp 4 (half 0, quadrant 0) before/after the slot-full wait, 5/6 warp 7
(half 0, quadrant 3) before/after, 7 warp 7 slot release, 8/9/10 warp 11 (half 1) before/after/release,
11 warp 11 scale stage ready."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2412_19437_b200 as fp
import paper_2412_19437_b200._lib as _L

if os.environ.get("FP8BS_LIB"):
    _L.LIB_PATH = os.environ["FP8BS_LIB"]


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "fprop"
    T, IN, OUT = 4096, 7168, 18432
    L, (M, N, K) = {"fprop": (fp.FPROP, (T, OUT, IN)), "dgrad": (fp.DGRAD, (T, IN, OUT)),
                    "wgrad": (fp.WGRAD, (OUT, IN, T))}[which]
    dev = "cuda"
    A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev)
    B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device=dev)
    sA = torch.rand(K // 128, M, device=dev)
    sB = {fp.FPROP: torch.rand(N // 128, K // 128, device=dev), fp.DGRAD: torch.rand(K // 128, N // 128, device=dev),
          fp.WGRAD: torch.rand(K // 128, N, device=dev)}[L]
    out = torch.empty(M, N, dtype=torch.float32 if L == fp.WGRAD else torch.bfloat16, device=dev)
    with fp.forced_variant(0):   # route through the test-hooks build (its timestamps are read below)
        for _ in range(3):
            fp.gemm(L, A, sA, B, sB, out=out)
    torch.cuda.synchronize()
    lib = fp.testhooks_lib()   # built with -DFP8BS_TEST_HOOKS=1 (and the experiment's debug bits)
    buf = (ctypes.c_ulonglong * (12 * 512))()
    lib.fp8bs_internal_debug_timestamps(buf, 12 * 512)
    t = np.array(buf, dtype=np.int64).reshape(12, 512)
    n = int((t[2] > 0).sum())
    KB = K // 128
    # steady state: skip the first tile, stay 2 K-blocks away from tile boundaries
    ks = [k for k in range(KB, n - 3) if 2 <= k % KB < KB - 3]
    ks = np.array(ks)

    def med(x):
        return float(np.median(x))

    print(f"{which}: {n} K-blocks traced, KB={KB}, steady-state samples {len(ks)}")
    print(f"  period (issuer h0 slot-free to slot-free)      {med(t[0, ks + 1] - t[0, ks]):7.0f} cycles (512 at tensor peak)")
    print(f"  A issuer: slot free -> stage full (TMA wait)     {med(t[1, ks] - t[0, ks]):7.0f}")
    print(f"  B issuer: stage full -> commit issued (4 MMAs)  {med(t[2, ks] - t[1, ks]):7.0f}")
    print(f"  G issuer: commit(kb) -> slot free(kb+1)          {med(t[0, ks + 1] - t[2, ks]):7.0f}")
    print(f"  C commit issued(kb) -> warp4 sees slot full(kb)  {med(t[4, ks] - t[2, ks]):7.0f}  (MMA execution + queue)")
    print(f"  D warp4 slot-full wait                           {med(t[4, ks] - t[3, ks]):7.0f}")
    print(f"  E warp7 slot full -> release (promotion chain)   {med(t[7, ks] - t[6, ks]):7.0f}")
    print(f"  F warp7 release(kb) -> issuer slot free(kb+2)    {med(t[0, ks + 2] - t[7, ks]):7.0f}  (other warps, peer CTA, wake-up)")
    print(f"  warp7 kb-to-kb period                            {med(t[6, ks + 1] - t[6, ks]):7.0f}")
    print(f"  warp7 release(kb) -> next slot-full wait start   {med(t[5, ks + 1] - t[7, ks]):7.0f}  (math after release + next scale wait)")
    print(f"  warp11 scale ready -> slot full ok               {med(t[9, ks] - t[11, ks]):7.0f}")
    print(f"  warp11 release(kb) - warp7 release(kb)           {med(t[10, ks] - t[7, ks]):7.0f}")
    for k in ks[100:104]:
        print(k, [int(t[i, k] - t[0, ks[100]]) for i in range(12)])


if __name__ == "__main__":
    main()
