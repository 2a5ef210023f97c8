"""Grouped UE8M0 (MX) Fprop over uniform top-8 routing, 256 experts, K = 7168, N = 2048, at several token
counts (experiments only; A/B the pair threshold with FP8BS_LIB builds of -DFP8BS_MX_GPAIR_ROWS=<rows>).
    FP8BS_LIB=tools/libfp8bs_<name>.so python tools/grouped_mx_sweep.py 4096,8192,16384"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200 as fp
import paper_2412_19437_b200._lib as _L
import workloads as W

if os.environ.get("FP8BS_LIB"):
    _L.LIB_PATH = os.environ["FP8BS_LIB"]


def med_ms(fn, iters=7):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        torch.cuda._sleep(20_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    dev = "cuda"
    K, N, E = 7168, 2048, 256
    B = torch.randint(0, 0x7E, (E, N, K), dtype=torch.uint8, device=dev)
    sB = torch.exp2(torch.randint(-12, -4, (E, N // 128, K // 128), device=dev).float())
    for T in [int(t) for t in (sys.argv[1] if len(sys.argv) > 1 else "4096,8192,16384").split(",")]:
        _, off = W.group_rows(W.route_uniform(T, E, 8), E)
        R = int(off[-1])
        A = torch.randint(0, 0x7E, (R, K), dtype=torch.uint8, device=dev)
        sA = torch.exp2(torch.randint(-12, -4, (K // 128, (R + 3) // 4 * 4), device=dev).float())[:, :R]
        o = off.to(dev)
        out = torch.empty(R, N, dtype=torch.bfloat16, device=dev)
        ms = med_ms(lambda: fp.grouped_gemm(o, A, sA, B, sB, out=out, mx=True))
        print(f"tokens {T:6d} ({R // E:4d} rows/expert) {ms:7.3f} ms {2.0 * R * N * K / ms / 1e9:6.0f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
