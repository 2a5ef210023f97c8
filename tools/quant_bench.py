"""Quantizer timings at the C1 shapes (experiments only): each launch timed alone with CUDA events,
L2 flushed (256 MB write) before every launch; prints us and algorithmic GB/s.
FP8BS_LIB selects another build."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200 as fp
import paper_2412_19437_b200._lib as _L
import workloads as W

if os.environ.get("FP8BS_LIB"):
    _L.LIB_PATH = os.environ["FP8BS_LIB"]


def timed(fn, iters=20):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    dev = "cuda"
    T, IN, OUT = 4096, 7168, 18432
    p4 = lambda n: (n + 3) // 4 * 4  # noqa: E731
    e = lambda *s, dt=torch.uint8: torch.empty(*s, dtype=dt, device=dev)  # noqa: E731
    cases = []
    for name, (M, C) in (("dual(X)", (T, IN)), ("dual(dY)", (T, OUT)), ("dual(C3 X)", (16384, 7168))):
        x = W.gaussian_act(M, C, seed=0).to(dev)
        q, s = e(M, C), e(C // 128, p4(M), dt=torch.float32)[:, :M]
        qT, sT = e(C, M), e(M // 128, p4(C), dt=torch.float32)[:, :C]
        nbytes = 2 * M * C + 2 * M * C + 4 * M * (C // 128) + 4 * C * (M // 128)
        cases.append((name, nbytes, lambda x=x, q=q, s=s, qT=qT, sT=sT: fp.quantize_act_dual(x, q, s, qT, sT)))
        q1, s1 = e(M, C), e(C // 128, p4(M), dt=torch.float32)[:, :M]
        cases.append((name.replace("dual", "1x128"), 3 * M * C + 4 * M * (C // 128),
                      lambda x=x, q1=q1, s1=s1: fp.quantize_act_1x128(x, q1, s1)))
    # FP8 -> FP8 re-quantization of the cached X (1x128 -> 128x1), the Wgrad operand
    xq, xs = fp.quantize_act_1x128(W.gaussian_act(T, IN, seed=0).to(dev))
    rqT, rsT = e(IN, T), e(T // 128, p4(IN), dt=torch.float32)[:, :IN]
    cases.append(("requant(X)", T * IN * 2 + 4 * T * (IN // 128) + 4 * IN * (T // 128),
                  lambda: fp.requantize_1x128_to_128x1(xq, xs, rqT, rsT)))
    M3 = 16384                                  # C3's token count: the fixed per-launch cost amortised
    xq3, xs3 = fp.quantize_act_1x128(W.gaussian_act(M3, IN, seed=0).to(dev))
    rqT3, rsT3 = e(IN, M3), e(M3 // 128, p4(IN), dt=torch.float32)[:, :IN]
    cases.append(("requant(C3 X)", M3 * IN * 2 + 4 * M3 * (IN // 128) + 4 * IN * (M3 // 128),
                  lambda: fp.requantize_1x128_to_128x1(xq3, xs3, rqT3, rsT3)))
    w = W.master_weight(OUT, IN, seed=1).to(dev)
    wq, sw, wqT = e(OUT, IN), e(OUT // 128, IN // 128, dt=torch.float32), e(IN, OUT)
    cases.append(("weight(W)+T", 6 * OUT * IN + 4 * (OUT // 128) * (IN // 128),
                  lambda: fp.quantize_weight_128x128(w, True, wq, sw, wqT)))
    only = sys.argv[1].split(",") if len(sys.argv) > 1 else None
    for name, nbytes, fn in cases:
        if only and name not in only:
            continue
        ms = timed(fn)
        print(f"{name:14s} {ms * 1e3:8.1f} us  {nbytes / ms / 1e6:7.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
