"""C1 step time without per-kernel events (experiments only): the 6 launches back to back, K steps
between two events.  FP8BS_LIB selects another build."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200._lib as _L

if os.environ.get("FP8BS_LIB"):
    _L.LIB_PATH = os.environ["FP8BS_LIB"]
import bench  # noqa: E402


def main():
    st = bench.DenseStep(torch.device("cuda"))
    for _ in range(5):
        st.run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 30
    a.record()
    for _ in range(K):
        st.run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    print(f"step {ms * 1e3:7.1f} us  {st.flops / ms / 1e9:6.0f} TFLOP/s")


if __name__ == "__main__":
    main()
