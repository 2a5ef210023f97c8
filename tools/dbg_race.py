"""Determinism check (experiments only): run one C1 GEMM layout repeatedly and compare every run bitwise
with the first; report where results differ (tile, rows, columns).  FP8BS_LIB selects another build.
    python tools/dbg_race.py [fprop|dgrad|wgrad] [runs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200 as fp
import paper_2412_19437_b200._lib as _L

if os.environ.get("FP8BS_LIB"):
    _L.LIB_PATH = os.environ["FP8BS_LIB"]


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "wgrad"
    runs = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    T, IN, OUT = 4096, 7168, 18432
    L, (M, N, K) = {"fprop": (fp.FPROP, (T, OUT, IN)), "dgrad": (fp.DGRAD, (T, IN, OUT)),
                    "wgrad": (fp.WGRAD, (OUT, IN, T))}[which]
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev, generator=g)
    B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device=dev, generator=g)
    sA = torch.rand(K // 128, M, device=dev, generator=g) + 0.5
    sB = {fp.FPROP: torch.rand(N // 128, K // 128, device=dev, generator=g), fp.DGRAD: torch.rand(K // 128, N // 128, device=dev, generator=g),
          fp.WGRAD: torch.rand(K // 128, N, device=dev, generator=g)}[L] + 0.5
    ref = fp.gemm(L, A, sA, B, sB, out_dtype=torch.float32)
    torch.cuda.synchronize()
    bad = 0
    for i in range(runs):
        D = fp.gemm(L, A, sA, B, sB, out_dtype=torch.float32)
        torch.cuda.synchronize()
        diff = (D.view(torch.int32) != ref.view(torch.int32))
        n = int(diff.sum())
        if n:
            bad += 1
            idx = diff.nonzero()
            r, c = idx[:, 0], idx[:, 1]
            tiles = torch.unique(torch.stack([r // 256, c // 256], 1), dim=0)
            rel = ((D - ref).abs().max() / ref.abs().max()).item()
            print(f"run {i}: {n} elements differ, rel {rel:.3e}, tiles (m,n) {tiles[:8].tolist()} ({len(tiles)} tiles); "
                  f"rows%256 {torch.unique(r % 256)[:8].tolist()}.. cols%256 min {int((c % 256).min())} max {int((c % 256).max())}", flush=True)
            for t in tiles[:3].tolist():
                m = (r // 256 == t[0]) & (c // 256 == t[1])
                rr, cc = r[m] % 256, c[m] % 256
                print(f"   tile {t}: rows {int(rr.min())}..{int(rr.max())} ({len(torch.unique(rr))} distinct), cols {int(cc.min())}..{int(cc.max())} ({len(torch.unique(cc))} distinct); "
                      f"ratio D/ref median {float((D[r[m], c[m]] / ref[r[m], c[m]]).median()):.4f}")
    print(f"{which}: {bad} of {runs} runs differ from the first")


if __name__ == "__main__":
    main()
