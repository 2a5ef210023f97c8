"""Time the C4 grouped Fprop (bench.py's launch) with the library in FP8BS_LIB (A/B of builds).
    FP8BS_LIB=tools/libfp8bs_<name>.so python tools/grouped_c4_time.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2412_19437_b200 import ep


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    dev = torch.device("cuda", 0)
    cfg = ep.EPConfig()
    pb = ep.build_rank_problem(cfg, 1, 0, dev)
    for _ in range(3):
        ep.run_rank(pb)
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ep.run_rank(pb)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
        torch.cuda.synchronize()
        torch.cuda._sleep(20_000_000)   # ~10 ms idle between launches: each launch starts cool
    ts.sort()
    med = ts[len(ts) // 2]
    print(f"{os.environ.get('FP8BS_LIB', 'in-tree')}: median {med:.3f} ms  {pb.flops / med / 1e9:.0f} TFLOP/s  min {ts[0]:.3f}")


if __name__ == "__main__":
    main()
