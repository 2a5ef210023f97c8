"""Debug helper: run the grouped GEMM on synthetic ragged segments and compare with per-expert
dense GEMMs (bitwise) — isolates grouped-scheduler faults.  Usage:
    python tools/dbg_grouped.py G K N counts_mode[ragged|aligned] out[f32|bf16]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200 as fp
import workloads as W


def main():
    G, K, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    mode, out = sys.argv[4], sys.argv[5]
    g = torch.Generator().manual_seed(0)
    if mode == "aligned":
        counts = [128] * G
    elif mode == "ragged4":
        counts = (torch.randint(15, 50, (G,), generator=g) * 4).tolist()
    elif mode == "mult128":
        counts = (torch.randint(1, 3, (G,), generator=g) * 128).tolist()
    else:
        counts = torch.randint(60, 200, (G,), generator=g).tolist()
    offsets = torch.zeros(G + 1, dtype=torch.int64)
    offsets[1:] = torch.cumsum(torch.tensor(counts), 0)
    R = int(offsets[-1])
    dev = "cuda"
    A = W.codes_small(R, K, seed=1).to(dev)
    sA = torch.ones(K // 128, (R + 3) // 4 * 4, device=dev)[:, :R]
    B = W.codes_small(G * N, K, seed=2).reshape(G, N, K).to(dev)
    sB = torch.ones(G, (N + 127) // 128, K // 128, device=dev)
    od = torch.float32 if out == "f32" else torch.bfloat16
    D = fp.grouped_gemm(offsets.to(dev), A, sA, B, sB, out_dtype=od)
    torch.cuda.synchronize()
    bad = 0
    for e in range(G):
        a, b = int(offsets[e]), int(offsets[e + 1])
        De = fp.gemm(fp.FPROP, A[a:b].contiguous(), torch.ones(K // 128, (b - a + 3) // 4 * 4, device=dev)[:, :b - a],
                     B[e], sB[e], out_dtype=od)
        if not torch.equal(De, D[a:b]):
            bad += 1
    torch.cuda.synchronize()
    print(f"G={G} K={K} N={N} {mode} {out}: R={R} mismatching experts={bad}")


if __name__ == "__main__":
    main()
