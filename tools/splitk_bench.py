"""Split-K tail A/B on one GPU (fp8bs_gemm_ws vs fp8bs_gemm), same process, alternating:
    python tools/splitk_bench.py [iters]
C1's three GEMMs and C3's q-lora projection, BF16 (FP32 for Wgrad) output, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_19437_b200 as fp  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    dev = torch.device("cuda")
    cases = [("C1 fprop", fp.FPROP, 4096, 18432, 7168), ("C1 dgrad", fp.DGRAD, 4096, 7168, 18432),
             ("C1 wgrad", fp.WGRAD, 18432, 7168, 4096), ("C3 q-lora", fp.FPROP, 16384, 1536, 7168)]
    for name, layout, M, N, K in cases:
        g = torch.Generator(device=dev).manual_seed(0)
        A = torch.randint(0, 126, (M, K), dtype=torch.uint8, device=dev, generator=g)
        B = torch.randint(0, 126, (N, K), dtype=torch.uint8, device=dev, generator=g)
        sA = torch.rand(K // 128, M, device=dev, generator=g) + 0.5
        nb = (N + 127) // 128
        sB = {fp.FPROP: (nb, K // 128), fp.DGRAD: (K // 128, nb), fp.WGRAD: (K // 128, N)}[layout]
        sB = torch.rand(*sB, device=dev, generator=g) + 0.5
        odt = torch.float32 if layout == fp.WGRAD else torch.bfloat16
        out = torch.empty(M, N, dtype=odt, device=dev)
        wsb = fp.gemm_workspace_size(layout, M, N, K)
        ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
        runs = {"split": lambda: fp.gemm(layout, A, sA, B, sB, out=out, workspace=ws),
                "unsplit": lambda: fp.gemm(layout, A, sA, B, sB, out=out, workspace=None)}
        res = {k: [] for k in runs}
        for _ in range(3):
            for fn in runs.values():
                fn()
        torch.cuda.synchronize()
        for _ in range(iters):
            for k, fn in runs.items():
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                res[k].append(a.elapsed_time(b))
        fl = 2.0 * M * N * K
        line = f"{name:10s} ws={wsb / 2**20:5.1f} MB"
        for k, v in res.items():
            v.sort()
            med = v[len(v) // 2]
            line += f" | {k} {med * 1e3:7.1f} us {fl / (med * 1e-3) / 1e12:6.0f} TF/s"
        print(line, flush=True)


if __name__ == "__main__":
    main()
