"""Grouped MoE expert Wgrad (fp8bs_quantize_act_128x1_grouped + fp8bs_grouped_gemm_wgrad, NEXT-3) at the
C4 / C2 expert shapes on one GPU (experiments only): 256 experts, up-projection in=7168 -> out=2048,
dW_e = dY_e^T X_e [2048, 7168] FP32 per expert.  Routing as workloads.route_skewed / route_uniform
(R15, R16).  Reports the grouped Wgrad TFLOP/s (algorithmic flops 2*R*N*K over the R real rows), the
dense-equivalent Wgrad over the same R rows for comparison, and the grouped quantizer's GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200 as fp
import workloads as W


def timeit(fn, iters=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    dev = "cuda"
    G, N, K = 256, 2048, 7168
    for name, T, skew in (("C4 skewed 65536 tokens x top-8", 65536, True), ("C4 skewed 8192 tokens x top-8", 8192, True),
                          ("C2 uniform 4096 tokens x top-8", 4096, False)):
        routes = W.route_skewed(T, G, 8, seed=3) if skew else W.route_uniform(T, G, 8, seed=3)
        _, offsets = W.group_rows(routes, G)
        R = int(offsets[-1])
        Mp = fp.padded_tokens(offsets)
        x = torch.randn(R, K, device=dev).to(torch.bfloat16)
        dy = (torch.randn(R, N, device=dev) * 1e-2).to(torch.bfloat16)
        XqT, sX = fp.quantize_act_128x1_grouped(x, offsets)
        DqT, sD = fp.quantize_act_128x1_grouped(dy, offsets)
        out = torch.empty(G, N, K, dtype=torch.float32, device=dev)
        ms_q = timeit(lambda: fp.quantize_act_128x1_grouped(x, offsets, qT=XqT, sT=sX))
        ms_w = timeit(lambda: fp.grouped_gemm_wgrad(offsets, DqT, sD, XqT, sX, out=out))
        # UE8M0 form (fp8bs_grouped_gemm_wgrad_mx) on power-of-two scales (the same codes; timing only)
        sDp, sXp = torch.exp2(torch.floor(torch.log2(sD))), torch.exp2(torch.floor(torch.log2(sX)))
        ms_mx = timeit(lambda: fp.grouped_gemm_wgrad(offsets, DqT, sDp, XqT, sXp, out=out, mx=True))
        # dense Wgrad over the same R rows (one expert), for comparison
        qx, sx = fp.quantize_act_128x1(x[: R // 128 * 128])
        qd, sd = fp.quantize_act_128x1(dy[: R // 128 * 128])
        dense_out = torch.empty(N, K, dtype=torch.float32, device=dev)
        ms_d = timeit(lambda: fp.gemm(fp.WGRAD, qd, sd, qx, sx, out=dense_out, out_dtype=torch.float32))
        fl = 2.0 * R * N * K
        fl_d = 2.0 * (R // 128 * 128) * N * K
        qbytes = R * K * 2 + Mp * K + Mp // 128 * K * 4
        m = offsets[1:] - offsets[:-1]
        print(f"{name}: R={R} Mp={Mp} M_e in [{int(m.min())},{int(m.max())}] | grouped wgrad {ms_w:.3f} ms "
              f"{fl / ms_w / 1e9:.0f} TFLOP/s (out {G * N * K * 4 / 1e9:.1f} GB FP32) | mx {ms_mx:.3f} ms {fl / ms_mx / 1e9:.0f} | dense same rows {ms_d:.3f} ms "
              f"{fl_d / ms_d / 1e9:.0f} TFLOP/s | grouped 128x1 quant X {ms_q * 1e3:.0f} us {qbytes / ms_q / 1e6:.0f} GB/s",
              flush=True)
        del XqT, DqT, out, x, dy, qx, qd
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
