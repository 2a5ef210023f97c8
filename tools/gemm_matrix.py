"""GEMM experiment matrix (experiments only; not the bench): time each layout at the C1 shapes and the
C2 grouped shape for several kernel variants and debug bits, all in one process.

    FP8BS_LIB=<other .so> python tools/gemm_matrix.py [variants=2,1] [debugs=0,1] [cases=fprop,dgrad,wgrad,grouped_C2]

Debug bits are compile-time (tools/build_rev.sh WORKTREE <name> -DFP8BS_GEMM_DEBUG_BITS=<bits>, see
gemm.cu): 1 skip promotion math, 2 skip MMAs, 4 TMA re-reads K-block 0 (L2-resident operands), 8 no TMEM
reads, 16 timestamps, 64 MMA issuer ignores TMEM-slot release, 128 promotion ignores slot completion,
256 issuers pace on their own commits, 512 no scale ring.  The debugs argument only labels the rows.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_19437_b200 as fp
import paper_2412_19437_b200._lib as _L
import workloads as W

if os.environ.get("FP8BS_LIB"):          # A/B experiments against another build of the library
    _L.LIB_PATH = os.environ["FP8BS_LIB"]


def timeit(fn, iters=10):
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
    variants = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "2,1").split(",")]
    debugs = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,1").split(",")]
    only = sys.argv[3].split(",") if len(sys.argv) > 3 else None
    dev = "cuda"
    T, IN, OUT = 4096, 7168, 18432
    cases = []
    for name, L, (M, N, K) in (("fprop", fp.FPROP, (T, OUT, IN)), ("dgrad", fp.DGRAD, (T, IN, OUT)),
                               ("wgrad", fp.WGRAD, (OUT, IN, T))):
        A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev)
        B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device=dev)
        sA = torch.rand(K // 128, M, device=dev)
        sB = {fp.FPROP: torch.rand(N // 128, K // 128, device=dev), fp.DGRAD: torch.rand(K // 128, N // 128, device=dev),
              fp.WGRAD: torch.rand(K // 128, N, device=dev)}[L]
        out = torch.empty(M, N, dtype=torch.float32 if L == fp.WGRAD else torch.bfloat16, device=dev)
        cases.append((name, 2.0 * M * N * K, (lambda L=L, A=A, sA=sA, B=B, sB=sB, out=out: fp.gemm(L, A, sA, B, sB, out=out))))
    # C3: MLA projections over 16384 tokens (q-lora 7168 -> 1536, kv-lora 7168 -> 576), Fprop BF16 out
    for name, (M, N, K) in (("C3_q", (16384, 1536, 7168)), ("C3_kv", (16384, 576, 7168))):
        if only and name not in only:
            continue
        A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev)
        B = torch.randint(0, 120, (N, K), dtype=torch.uint8, device=dev)
        sA = torch.rand(K // 128, M, device=dev)
        sB = torch.rand((N + 127) // 128, K // 128, device=dev)
        out = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
        cases.append((name, 2.0 * M * N * K, (lambda A=A, sA=sA, B=B, sB=sB, out=out: fp.gemm(fp.FPROP, A, sA, B, sB, out=out))))
    # C2: 256 experts, K=7168, N=2048, 4096 tokens x top-8 uniform
    E, N2, K2 = 256, 2048, 7168
    _, offs = W.group_rows(W.route_uniform(4096, E, 8), E)
    R = int(offs[-1])
    A2 = torch.randint(0, 120, (R, K2), dtype=torch.uint8, device=dev)
    sA2 = torch.rand(K2 // 128, R, device=dev)
    B2 = torch.randint(0, 120, (E, N2, K2), dtype=torch.uint8, device=dev)
    sB2 = torch.rand(E, N2 // 128, K2 // 128, device=dev)
    o2 = offs.to(dev)
    out2 = torch.empty(R, N2, dtype=torch.bfloat16, device=dev)
    cases.append(("grouped_C2", 2.0 * R * N2 * K2, lambda: fp.grouped_gemm(o2, A2, sA2, B2, sB2, out=out2)))
    for T2 in [int(t) for t in os.environ.get("GROUPED_T", "2048,8192").split(",")]:
        # ~64 and ~256 rows per expert (uniform): where the one-CTA / pair variant choice flips
        name = f"grouped_T{T2}"
        if only and name not in only:
            continue
        _, offsT = W.group_rows(W.route_uniform(T2, E, 8), E)
        RT = int(offsT[-1])
        AT = torch.randint(0, 120, (RT, K2), dtype=torch.uint8, device=dev)
        sAT = torch.rand(K2 // 128, RT, device=dev)
        oT = offsT.to(dev)
        outT = torch.empty(RT, N2, dtype=torch.bfloat16, device=dev)
        cases.append((name, 2.0 * RT * N2 * K2, (lambda oT=oT, AT=AT, sAT=sAT, outT=outT: fp.grouped_gemm(oT, AT, sAT, B2, sB2, out=outT))))
    if only and "grouped_C4" in only:
        # C4 at one GPU: 65536 tokens x top-8, skewed routing (alpha 0.5), all 256 experts
        _, offs4 = W.group_rows(W.route_skewed(65536, E, 8), E)
        R4 = int(offs4[-1])
        A4 = torch.randint(0, 120, (R4, K2), dtype=torch.uint8, device=dev)
        sA4 = torch.rand(K2 // 128, R4, device=dev)
        o4 = offs4.to(dev)
        out4 = torch.empty(R4, N2, dtype=torch.bfloat16, device=dev)
        cases.append(("grouped_C4", 2.0 * R4 * N2 * K2, lambda: fp.grouped_gemm(o4, A4, sA4, B2, sB2, out=out4)))
    for v in variants:
        with fp.forced_variant(v):   # the test-hooks build of the same sources
            for d in debugs:
                for name, flop, fn in cases:
                    if only and name not in only:
                        continue
                    ms = timeit(fn)
                    print(f"variant={v} debug={d:4d} {name:11s} {ms * 1e3:8.1f} us  {flop / ms / 1e9:7.0f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
