"""fp8bs_gemm_mx (UE8M0 block scaling, power-of-two scales) vs fp8bs_gemm (FP32 promotion) at the C1
shapes (experiments only).  Same random codes; scales are powers of two for both."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200 as fp


def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def diag():
    """MX kernel only, Wgrad's slowness pulled apart: layout x shape x output type."""
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    p2 = lambda *s: 2.0 ** torch.randint(-10, -2, s, device=dev, generator=g).float()  # noqa: E731
    for name, L, (M, N, K), dt in (("fprop C1 bf16", fp.FPROP, (4096, 18432, 7168), torch.bfloat16),
                                   ("fprop C1 f32", fp.FPROP, (4096, 18432, 7168), torch.float32),
                                   ("fprop wgshape bf16", fp.FPROP, (18432, 7168, 4096), torch.bfloat16),
                                   ("fprop wgshape f32", fp.FPROP, (18432, 7168, 4096), torch.float32),
                                   ("fprop 4096x7168x18432 f32", fp.FPROP, (4096, 7168, 18432), torch.float32),
                                   ("wgrad f32", fp.WGRAD, (18432, 7168, 4096), torch.float32),
                                   ("wgrad K=8192 f32", fp.WGRAD, (18432, 7168, 8192), torch.float32)):
        A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev, generator=g)
        B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device=dev, generator=g)
        sA = p2(K // 128, M)
        sB = p2(N // 128, K // 128) if L == fp.FPROP else p2(K // 128, N)
        out = torch.empty(M, N, dtype=dt, device=dev)
        ms = timeit(lambda: fp.gemm(L, A, sA, B, sB, out=out, mx=True))
        print(f"{name:28s} {ms * 1e3:7.1f} us {2.0 * M * N * K / ms / 1e9:6.0f} TFLOP/s", flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "diag":
        return diag()
    dev = "cuda"
    T, IN, OUT = 4096, 7168, 18432
    g = torch.Generator(device=dev).manual_seed(0)
    for name, L, (M, N, K) in (("fprop", fp.FPROP, (T, OUT, IN)), ("dgrad", fp.DGRAD, (T, IN, OUT)),
                               ("wgrad", fp.WGRAD, (OUT, IN, T))):
        A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev, generator=g)
        B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device=dev, generator=g)
        p2 = lambda *s: 2.0 ** torch.randint(-10, -2, s, device=dev, generator=g).float()  # noqa: E731
        sA = p2(K // 128, M)
        sB = {fp.FPROP: p2(N // 128, K // 128), fp.DGRAD: p2(K // 128, N // 128), fp.WGRAD: p2(K // 128, N)}[L]
        dt = torch.float32 if L == fp.WGRAD else torch.bfloat16
        out = torch.empty(M, N, dtype=dt, device=dev)
        out2 = torch.empty(M, N, dtype=dt, device=dev)
        ms0 = timeit(lambda: fp.gemm(L, A, sA, B, sB, out=out))
        ms1 = timeit(lambda: fp.gemm(L, A, sA, B, sB, out=out2, mx=True))
        fl = 2.0 * M * N * K
        rel = float((out.float() - out2.float()).abs().max() / out.float().abs().max())
        print(f"{name}: promotion {ms0 * 1e3:7.1f} us {fl / ms0 / 1e9:6.0f} TFLOP/s | mx {ms1 * 1e3:7.1f} us "
              f"{fl / ms1 / 1e9:6.0f} TFLOP/s | max rel diff {rel:.2e}", flush=True)


if __name__ == "__main__":
    main()
