"""Where the C4 grouped Fprop loses time (experiments only): the same 524288 x 7168 FP8 rows and
256 expert weights of bench.py's C4 problem, timed (median of N launches, each after ~10 ms idle)
as: dense Fprop with expert 0's weight over all rows; grouped with one expert; grouped with 256
equal 2048-row experts (no ragged tails); grouped with the C4 skewed routing (the bench's launch).
    FP8BS_LIB=... python tools/grouped_anatomy.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200 as fp
from paper_2412_19437_b200 import ep


def med_ms(fn, iters):
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
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 7
    dev = torch.device("cuda", 0)
    cfg = ep.EPConfig()
    pb = ep.build_rank_problem(cfg, 1, 0, dev)
    R, K = pb.A.shape
    N = cfg.inter
    fl = 2.0 * R * N * K
    out = pb.out
    cases = [("dense (expert 0's W over all rows)", lambda: fp.gemm(fp.FPROP, pb.A, pb.sA, pb.Bq[0], pb.sB[0], out=out))]
    o1 = torch.tensor([0, R], dtype=torch.int64, device=dev)
    cases.append(("grouped G=1", lambda: fp.grouped_gemm(o1, pb.A, pb.sA, pb.Bq[:1], pb.sB[:1], out=out)))
    oe = torch.arange(257, dtype=torch.int64, device=dev) * (R // 256)
    cases.append(("grouped 256 x 2048 equal", lambda: fp.grouped_gemm(oe, pb.A, pb.sA, pb.Bq, pb.sB, out=out)))
    cases.append(("grouped C4 skewed (bench)", lambda: ep.run_rank(pb)))
    for name, fn in cases:
        ms = med_ms(fn, iters)
        print(f"{name:40s} {ms:7.3f} ms {fl / ms / 1e9:7.0f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
