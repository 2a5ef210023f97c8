"""Expert-parallel sharding of the grouped MoE expert GEMM (BASELINE configs[4]).

DeepSeek-V3 trains with 64-way expert parallelism and no token dropping
(P:267-270).  Here the grouped expert Fprop is partitioned by expert: rank r owns the contiguous
expert block [r*E/W, (r+1)*E/W).  Experts are independent, so there is NO exchange step in the
computed path: every rank regenerates, from the shared seeds, the routing of all tokens, its own
experts' weights and the FP8 rows routed to them (the rows a dispatch would deliver — dispatch
itself, is out of scope), and runs one fp8bs_grouped_gemm.  NCCL (torch.distributed)
is used only to gather per-rank outputs for verification, outside any timed region.

Bookkeeping helpers are pure functions (unit-tested on CPU with world_size 2 over gloo);
`build_rank_problem` / `run_rank` touch the GPU only through the fp8bs C-ABI binding.
"""
from __future__ import annotations

import dataclasses
import time

import torch

import workloads as W


def shard_range(E: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous expert block of `rank` (E need not divide evenly: the first E % world ranks get
    one extra expert)."""
    base, extra = divmod(E, world)
    e0 = rank * base + min(rank, extra)
    return e0, e0 + base + (1 if rank < extra else 0)


def local_rows(routes: torch.Tensor, E: int, e0: int, e1: int):
    """Rows (token, slot) routed to experts [e0, e1), sorted by (expert, token).
    Returns (token_index int64 [R_local], offsets int64 [e1-e0+1])."""
    tok, offsets = W.group_rows(routes, E)
    a, b = int(offsets[e0]), int(offsets[e1])
    return tok[a:b].clone(), (offsets[e0:e1 + 1] - offsets[e0]).clone()


def imbalance(counts_per_rank) -> float:
    """max / mean rows per rank: the load-imbalance bound on expert-parallel scaling."""
    c = torch.tensor(counts_per_rank, dtype=torch.float64)
    return float(c.max() / c.mean()) if c.sum() > 0 else 1.0


def gather_rows(local: torch.Tensor, world: int, group=None) -> list[torch.Tensor]:
    """all_gather of variable-length row blocks (pad to the max, gather, trim).  Verification only."""
    import torch.distributed as dist
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    m = int(max(int(x.item()) for x in ns))
    pad = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    outs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return [o[:int(k.item())] for o, k in zip(outs, ns)]


@dataclasses.dataclass
class EPConfig:
    tokens: int = 65536
    experts: int = 256
    top_k: int = 8
    hidden: int = 7168          # K
    inter: int = 2048           # N (expert FFN dim)
    skew_alpha: float = 0.5     # 0 -> uniform routing
    seed: int = 3


def routes_for(cfg: EPConfig) -> torch.Tensor:
    if cfg.skew_alpha > 0:
        return W.route_skewed(cfg.tokens, cfg.experts, cfg.top_k, alpha=cfg.skew_alpha, seed=cfg.seed)
    return W.route_uniform(cfg.tokens, cfg.experts, cfg.top_k, seed=cfg.seed)


@dataclasses.dataclass
class RankProblem:
    e0: int
    e1: int
    offsets: torch.Tensor       # int64 [G_local + 1], device
    tok: torch.Tensor           # int64 [R_local], CPU
    A: torch.Tensor             # uint8 [R_local, K] FP8 rows (quantized per token, then gathered)
    sA: torch.Tensor            # f32 [K/128, R_local]
    Bq: torch.Tensor            # uint8 [G_local, N, K]
    sB: torch.Tensor            # f32 [G_local, N/128, K/128]
    out: torch.Tensor           # bf16 [R_local, N]
    flops: float


def build_rank_problem(cfg: EPConfig, world: int, rank: int, device, routes: torch.Tensor | None = None) -> RankProblem:
    """Everything rank `rank` needs, regenerated from the seeds (identical on every rank).
    Activations: N(0,1) BF16 from a seeded CUDA generator; quantized 1x128 ONCE per token (the
    paper quantizes before dispatch) and the FP8 rows + per-row scales are gathered —
    exact, because 1x128 scales are per row."""
    import paper_2412_19437_b200 as fp
    if routes is None:
        routes = routes_for(cfg)
    e0, e1 = shard_range(cfg.experts, world, rank)
    tok, offsets = local_rows(routes, cfg.experts, e0, e1)
    K, N = cfg.hidden, cfg.inter
    g = torch.Generator(device=device)
    g.manual_seed(cfg.seed + 100)
    x = torch.randn(cfg.tokens, K, generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    xq, xs = fp.quantize_act_1x128(x)
    del x
    tokd = tok.to(device)
    R = tok.numel()
    A = xq.index_select(0, tokd).contiguous()
    sA = torch.empty(K // 128, (R + 3) // 4 * 4 if R else 4, dtype=torch.float32, device=device)[:, :R]
    sA.copy_(xs.index_select(1, tokd))
    del xq, xs
    G = e1 - e0
    Bq = torch.empty(G, N, K, dtype=torch.uint8, device=device)
    sB = torch.empty(G, N // 128, K // 128, dtype=torch.float32, device=device)
    for i in range(G):
        ge = torch.Generator(device=device)
        ge.manual_seed(cfg.seed + 1000 + e0 + i)
        w = (torch.randn(N, K, generator=ge, device=device, dtype=torch.float32) * 0.006).to(torch.bfloat16)
        fp.quantize_weight_128x128(w, want_t=False, q=Bq[i], s=sB[i])
    out = torch.empty(R, N, dtype=torch.bfloat16, device=device)
    return RankProblem(e0, e1, offsets.to(device), tok, A, sA, Bq, sB, out, 2.0 * R * N * K)


def run_rank(pb: RankProblem):
    """The timed unit: one grouped GEMM over this rank's experts."""
    import paper_2412_19437_b200 as fp
    if pb.A.shape[0] == 0:
        return pb.out
    return fp.grouped_gemm(pb.offsets, pb.A, pb.sA, pb.Bq, pb.sB, out=pb.out)


def bench(args, world, rank, dev, barrier, max_over_ranks, ClockSampler, load_peaks):
    """bench.py --workload ep: time the per-rank grouped GEMM, report whole-job TFLOP/s."""
    cfg = EPConfig()
    routes = routes_for(cfg)
    pb = build_rank_problem(cfg, world, rank, dev, routes)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        run_rank(pb)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    with ClockSampler(dev.index or 0) as clk:
        a.record(stream)
        for _ in range(args.steps):
            run_rank(pb)
        b.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms_local = a.elapsed_time(b)
    ms = max_over_ranks(ms_local, world, dev)
    rows = [0] * world
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([pb.A.shape[0]], dtype=torch.int64, device=dev)
        lst = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(lst, t)
        rows = [int(x.item()) for x in lst]
    else:
        rows = [pb.A.shape[0]]
    total_flops = sum(2.0 * r * cfg.inter * cfg.hidden for r in rows)
    value = total_flops * args.steps / (ms * 1e-3) / 1e12
    peaks = load_peaks()
    local_tflops = pb.flops * args.steps / (ms_local * 1e-3) / 1e12
    peak = 2.0 * peaks["bf16_tflops"]
    return {"value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "e4m3", "data": "synthetic",
            "roofline": {"kernel": "grouped_gemm", "bound": "tensor", "achieved": local_tflops, "peak": peak,
                         "unit": "TFLOP/s", "frac": local_tflops / peak, "traffic": None,
                         "peak_src": f"{peaks['src']}: 2 x bf16_tflops (burst)"},
            "clocks": clk.summary(), "gpu_launches": args.steps,
            "ep": {"rows_per_rank": rows, "imbalance_max_over_mean": imbalance(rows),
                   "experts_per_rank": cfg.experts // world}}
