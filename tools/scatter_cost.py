"""Cost of the fused-combine epilogue on one GPU: the C4 grouped Fprop (bench.py's problem) writing D
contiguously (TMA stores) vs scattering its BF16 rows to (rank, slot) destinations through a pointer
table (fp8bs_grouped_gemm_scatter; here a 4-entry table of local buffers and the C4 routing's real
token-slot order at 4 ranks), CUDA events, alternating.  python tools/scatter_cost.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_19437_b200 as fp  # noqa: E402
from paper_2412_19437_b200 import ep  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    dev = torch.device("cuda")
    cfg = ep.EPConfig()
    routes = ep.routes_for(cfg)
    pb = ep.build_rank_problem(cfg, 1, 0, dev, routes)
    R, N = pb.A.shape[0], cfg.inter
    # destinations: the token owner (4 data-parallel shards) and its slot, as the 4-rank exchange writes
    tok = pb.tok
    T, k, W = cfg.tokens, cfg.top_k, 4
    shard = T // W
    rank = (tok // shard).to(torch.int32)
    slot = torch.empty(R, dtype=torch.int64)
    order = torch.argsort(routes.reshape(-1).to(torch.int64) * T + torch.arange(T).repeat_interleave(k), stable=True)
    slot_of_row = order                                   # global row -> flat slot (t * k + j)
    slot[:] = (slot_of_row // k - (slot_of_row // k // shard) * shard) * k + slot_of_row % k
    bufs = [torch.empty(shard * k, N, dtype=torch.bfloat16, device=dev) for _ in range(W)]
    table = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=dev)
    rk, sl = rank.to(dev), slot.to(dev)
    runs = {"grouped (TMA store to D)": lambda: ep.run_rank(pb),
            "grouped + scatter epilogue": lambda: fp.grouped_gemm_scatter(pb.offsets, pb.A, pb.sA, pb.Bq, pb.sB,
                                                                          table.data_ptr(), rk, sl, N, workspace=pb.ws)}
    res = {n: [] for n in runs}
    for _ in range(2):
        for f in runs.values():
            f()
    torch.cuda.synchronize()
    for _ in range(iters):
        for n, f in runs.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            torch.cuda.synchronize()
            res[n].append(a.elapsed_time(b))
            torch.cuda._sleep(20_000_000)
    for n, v in res.items():
        v.sort()
        med = v[len(v) // 2]
        print(f"{n:30s} median {med:.3f} ms  {pb.flops / med / 1e9:.0f} TFLOP/s", flush=True)
    # correctness: every row landed where the plain output says
    torch.cuda.synchronize()
    ok = all(torch.equal(bufs[r][sl[rk == r]].view(torch.int16), pb.out[rk == r].view(torch.int16)) for r in range(W))
    print("scatter rows bitwise equal to D rows:", ok)


if __name__ == "__main__":
    main()
