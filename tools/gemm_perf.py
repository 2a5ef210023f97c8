"""Time one GEMM layout at the C1 shape with CUDA events (experiments; not the bench)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_19437_b200 as fp

def main():
    layout = {"fprop": fp.FPROP, "dgrad": fp.DGRAD, "wgrad": fp.WGRAD}[sys.argv[1]]
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    T, IN, OUT = 4096, 7168, 18432
    M, N, K = {fp.FPROP: (T, OUT, IN), fp.DGRAD: (T, IN, OUT), fp.WGRAD: (OUT, IN, T)}[layout]
    dev = "cuda"
    A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev)
    B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device=dev)
    sA = torch.rand(K // 128, M, device=dev)
    sB = {fp.FPROP: torch.rand(N // 128, K // 128, device=dev), fp.DGRAD: torch.rand(K // 128, N // 128, device=dev),
          fp.WGRAD: torch.rand(K // 128, N, device=dev)}[layout]
    out = torch.empty(M, N, dtype=torch.float32 if layout == fp.WGRAD else torch.bfloat16, device=dev)
    for _ in range(3):
        fp.gemm(layout, A, sA, B, sB, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fp.gemm(layout, A, sA, B, sB, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    print(f"{sys.argv[1]} variant={os.environ.get('FP8BS_GEMM_VARIANT','auto')} M={M} N={N} K={K}: {ms*1e3:.1f} us  {2*M*N*K/ms/1e9:.0f} TFLOP/s")

if __name__ == "__main__":
    main()
