"""GEMM throughput vs SM clock and power (experiments only): each C1 layout runs back to back for
~1.5 s while NVML samples SM clock, power and throttle reasons every 5 ms; prints TFLOP/s, median
clock under load, and the tensor-pipe fraction at that clock (8192 FP8 MAC/clk/SM x 148 SMs).
FP8BS_LIB selects another build."""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
import torch

import paper_2412_19437_b200 as fp
import paper_2412_19437_b200._lib as _L

if os.environ.get("FP8BS_LIB"):
    _L.LIB_PATH = os.environ["FP8BS_LIB"]

pynvml.nvmlInit()
H = pynvml.nvmlDeviceGetHandleByIndex(0)
REASONS = {pynvml.nvmlClocksEventReasonSwPowerCap: "sw_power_cap", pynvml.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
           pynvml.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal", pynvml.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal"}


def sample(stop, out):
    while not stop.is_set():
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(H)
        out.append((pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(H) / 1000.0,
                    [n for b, n in REASONS.items() if r & b]))
        time.sleep(0.005)


def run(name, fn, flop, seconds=1.5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        fn()
    b.record()
    torch.cuda.synchronize()
    n = max(5, int(seconds / (a.elapsed_time(b) / 5e3)))
    samples, stop = [], threading.Event()
    t = threading.Thread(target=sample, args=(stop, samples))
    t.start()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    stop.set()
    t.join()
    ms = a.elapsed_time(b) / n
    tf = flop / ms / 1e9
    load = samples[len(samples) // 5:]          # skip the ramp
    mhz = statistics.median(s[0] for s in load)
    pw = statistics.median(s[1] for s in load)
    reasons = sorted({r for s in load for r in s[2]})
    peak = 8192 * 2 * 148 * mhz * 1e6 / 1e12
    print(f"{name:8s} {ms * 1e3:8.1f} us {tf:7.0f} TFLOP/s  clock {mhz:5.0f} MHz  power {pw:6.0f} W  "
          f"tensor frac at clock {tf / peak:5.3f}  reasons {reasons}", flush=True)


def main():
    only = sys.argv[1].split(",") if len(sys.argv) > 1 else ["fprop", "dgrad", "wgrad"]
    T, IN, OUT = 4096, 7168, 18432
    dev = "cuda"
    for name, L, (M, N, K) in (("fprop", fp.FPROP, (T, OUT, IN)), ("dgrad", fp.DGRAD, (T, IN, OUT)),
                               ("wgrad", fp.WGRAD, (OUT, IN, T))):
        if name not in only:
            continue
        A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev)
        B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device=dev)
        sA = torch.rand(K // 128, M, device=dev)
        sB = {fp.FPROP: torch.rand(N // 128, K // 128, device=dev), fp.DGRAD: torch.rand(K // 128, N // 128, device=dev),
              fp.WGRAD: torch.rand(K // 128, N, device=dev)}[L]
        out = torch.empty(M, N, dtype=torch.float32 if L == fp.WGRAD else torch.bfloat16, device=dev)
        run(name, lambda: fp.gemm(L, A, sA, B, sB, out=out), 2.0 * M * N * K)


if __name__ == "__main__":
    main()
