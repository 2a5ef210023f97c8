"""Is the in-step 1x128 quantizer slower because of the GEMM before it?  C4's token batch (65536 x 7168
BF16): the quantizer alone back to back, then alternating with the C4 grouped GEMM (as bench.py's
step), CUDA events around each quantizer launch; nvidia-smi SM clock sampled in each phase."""
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_19437_b200 as fp  # noqa: E402
from paper_2412_19437_b200 import ep  # noqa: E402


def clocks(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-i", "0"],
                           capture_output=True, text=True)
        try:
            out.append(int(r.stdout.strip().splitlines()[0]))
        except Exception:
            pass
        time.sleep(0.05)


def main():
    dev = torch.device("cuda")
    cfg = ep.EPConfig()
    pb = ep.build_rank_problem(cfg, 1, 0, dev, keep_tokens=True)
    torch.cuda.synchronize()
    byts = pb.x.numel() * 2 + pb.x.numel() + pb.x.shape[0] * (pb.x.shape[1] // 128) * 4

    def run(phase, with_gemm, n=30):
        ev = []
        stop, ck = threading.Event(), []
        th = threading.Thread(target=clocks, args=(stop, ck))
        th.start()
        for i in range(n):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ep.quantize_tokens(pb)
            b.record()
            ev.append((a, b))
            if with_gemm:
                ep.run_rank(pb)
        torch.cuda.synchronize()
        stop.set()
        th.join()
        t = sorted(a.elapsed_time(b) for a, b in ev[5:])
        med = t[len(t) // 2]
        ck.sort()
        print(f"{phase:28s} quant median {med * 1e3:6.1f} us = {byts / med / 1e6:5.0f} GB/s  (min {t[0] * 1e3:.1f})"
              f"  sm clock median {ck[len(ck) // 2] if ck else -1} MHz", flush=True)

    run("quantizer alone", False, 200)
    run("quantizer after grouped GEMM", True, 40)
    time.sleep(2)
    run("quantizer alone (again)", False, 200)


if __name__ == "__main__":
    main()
