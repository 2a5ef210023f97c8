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
    t0: int = 0                 # this rank's data-parallel token shard [t0, t1) ...
    t1: int = 0
    x: torch.Tensor | None = None    # ... its BF16 activations [t1 - t0, K] (device)
    xq: torch.Tensor | None = None   # ... and the 1x128 codes / scales the step writes
    xs: torch.Tensor | None = None
    ws: torch.Tensor | None = None   # the grouped GEMM's workspace (tile table), allocated once


def token_shard(T: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous data-parallel token shard of `rank` (the tokens whose activations it quantizes
    before dispatch)."""
    return shard_range(T, world, rank)


def build_rank_problem(cfg: EPConfig, world: int, rank: int, device, routes: torch.Tensor | None = None,
                       keep_tokens: bool = False) -> RankProblem:
    """Everything rank `rank` needs, regenerated from the seeds (identical on every rank).
    Activations: N(0,1) BF16 from a seeded CUDA generator; quantized 1x128 ONCE per token (the
    paper quantizes before dispatch) and the FP8 rows + per-row scales are gathered —
    exact, because 1x128 scales are per row.  keep_tokens: also keep the rank's data-parallel token
    shard (BF16) and output buffers for its 1x128 codes / scales (bench.py's C4 step quantizes it)."""
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
    t0, t1 = token_shard(cfg.tokens, world, rank)
    xsh = x[t0:t1].clone() if keep_tokens else None
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
    pb = RankProblem(e0, e1, offsets.to(device), tok, A, sA, Bq, sB, out, 2.0 * R * N * K, t0, t1)
    wsb = int(fp.lib().fp8bs_grouped_gemm_workspace_size(G, R, N, K)) if G > 0 else 16
    pb.ws = torch.empty((wsb + 15) // 16 * 16, dtype=torch.uint8, device=device)
    if keep_tokens:
        Tl = t1 - t0
        pb.x = xsh
        pb.xq = torch.empty(Tl, K, dtype=torch.uint8, device=device)
        pb.xs = torch.empty(K // 128, (Tl + 3) // 4 * 4 if Tl else 4, dtype=torch.float32, device=device)[:, :Tl]
    return pb


def quantize_tokens(pb: RankProblem):
    """The C4 step's first launch: 1x128 quantization of this rank's token shard (a-1, a-2)."""
    import paper_2412_19437_b200 as fp
    if pb.x is not None and pb.x.shape[0] > 0:
        fp.quantize_act_1x128(pb.x, pb.xq, pb.xs)


def run_rank(pb: RankProblem):
    """The C4 step's GEMM: one grouped launch over this rank's experts."""
    import paper_2412_19437_b200 as fp
    if pb.A.shape[0] == 0:
        return pb.out
    return fp.grouped_gemm(pb.offsets, pb.A, pb.sA, pb.Bq, pb.sB, out=pb.out, workspace=pb.ws)


def split_equals_G1_on_one_gpu(pb: RankProblem, cfg: EPConfig, splits=(2, 4, 8)) -> dict:
    """On ONE GPU holding the whole (G = 1) problem: for each G in `splits`, run the G contiguous expert
    shards as separate grouped launches on their own rows and compare the concatenation with the
    G = 1 output bitwise (the partition bench.py times at N GPUs, without NCCL)."""
    import paper_2412_19437_b200 as fp
    off = pb.offsets.cpu()
    ref = run_rank(pb).clone()
    res = {}
    for G in splits:
        parts = []
        for r in range(G):
            e0, e1 = shard_range(cfg.experts, G, r)
            a, b = int(off[e0]), int(off[e1])
            sa = torch.empty(pb.sA.shape[0], (b - a + 3) // 4 * 4 if b > a else 4, dtype=torch.float32,
                             device=pb.A.device)[:, :b - a]
            sa.copy_(pb.sA[:, a:b])
            if b > a:
                parts.append(fp.grouped_gemm((pb.offsets[e0:e1 + 1] - off[e0]).contiguous(), pb.A[a:b], sa,
                                             pb.Bq[e0:e1], pb.sB[e0:e1]))
        got = torch.cat(parts)
        res[str(G)] = bool(torch.equal(got.view(torch.int16), ref.view(torch.int16)))
    return res


def gathered_equals_G1(pb: RankProblem, cfg: EPConfig, world: int, rank: int, device, routes) -> bool | None:
    """N > 1: NCCL all_gather of every rank's output rows (verification only, outside any timed
    region); rank 0 rebuilds the G = 1 problem on its own GPU and compares bitwise.  Returns the
    verdict on rank 0, None elsewhere."""
    parts = gather_rows(pb.out, world)
    if rank != 0:
        return None
    got = torch.cat(parts)
    del parts
    ref_pb = build_rank_problem(cfg, 1, 0, device, routes)
    ref = run_rank(ref_pb)
    torch.cuda.synchronize()
    ok = bool(torch.equal(got.view(torch.int16), ref.view(torch.int16)))
    del ref_pb, ref, got
    torch.cuda.empty_cache()
    return ok


# ------------------------------------------------------------------------------------------
# The exchange steps (NEXT-3): FP8 dispatch of each token's 1x128 codes to the ranks
# owning its experts, BF16 combine of the expert outputs back to the token's owner, both written
# by the sender straight into the receiver's memory over NVLink (fp8bs_dispatch_fp8 /
# fp8bs_combine_push_bf16 on torch symmetric-memory buffers).  Tokens are data-parallel: rank r
# owns tokens token_shard(T, world, r).
# ------------------------------------------------------------------------------------------
@dataclasses.dataclass
class ExchangePlan:
    """Where every slot goes (pure bookkeeping from the routes; identical on every rank)."""
    t0: int; t1: int                 # this rank's tokens
    e0: int; e1: int                 # this rank's experts
    dst_rank: torch.Tensor           # int32 [(t1 - t0) * top_k]: owner of slot (t, j)'s expert
    dst_row: torch.Tensor            # int64 [...]: its row in the owner's expert-grouped receive buffer
    offsets: torch.Tensor            # int64 [e1 - e0 + 1]: this rank's received rows per expert
    c_rank: torch.Tensor             # int32 [R_local]: token owner of each received row
    c_slot: torch.Tensor             # int64 [R_local]: its slot (t - t0(owner)) * top_k + j there
    rows: int                        # R_local


def exchange_plan(routes: torch.Tensor, E: int, world: int, rank: int) -> ExchangePlan:
    T, k = routes.shape
    flat_e = routes.reshape(-1).to(torch.int64)
    flat_t = torch.arange(T, dtype=torch.int64).repeat_interleave(k)
    order = torch.argsort(flat_e * T + flat_t, stable=True)          # global row -> flat slot (as group_rows)
    pos = torch.empty_like(order)
    pos[order] = torch.arange(order.numel(), dtype=torch.int64)      # flat slot -> global row
    counts = torch.bincount(flat_e, minlength=E)
    offsets = torch.zeros(E + 1, dtype=torch.int64)
    offsets[1:] = torch.cumsum(counts, 0)
    e_start = torch.tensor([shard_range(E, world, r)[0] for r in range(world)] + [E], dtype=torch.int64)
    owner_of_e = torch.searchsorted(e_start, torch.arange(E), right=True) - 1
    t_start = torch.tensor([token_shard(T, world, r)[0] for r in range(world)] + [T], dtype=torch.int64)
    t0, t1 = token_shard(T, world, rank)
    e0, e1 = shard_range(E, world, rank)
    sl = slice(t0 * k, t1 * k)
    owner = owner_of_e[flat_e[sl]]
    dst_row = pos[sl] - offsets[e_start[owner]]
    g0, g1 = int(offsets[e0]), int(offsets[e1])
    slots = order[g0:g1]                                              # flat slots of this rank's rows
    tok = slots // k
    tok_owner = torch.searchsorted(t_start, tok, right=True) - 1
    c_slot = (tok - t_start[tok_owner]) * k + slots % k
    return ExchangePlan(t0, t1, e0, e1, owner.to(torch.int32), dst_row, (offsets[e0:e1 + 1] - g0).clone(),
                        tok_owner.to(torch.int32), c_slot, g1 - g0)


class Exchange:
    """Symmetric-memory receive buffers of the exchange (rendezvous over `group`): FP8 codes + row-major
    scales for dispatch, BF16 expert outputs per token slot for combine."""

    def __init__(self, group, device, max_rows: int, max_slots: int, K: int, N: int):
        import torch.distributed._symmetric_memory as symm_mem
        self.K, self.N = K, N
        self.recv_q = symm_mem.empty(max_rows, K, dtype=torch.uint8, device=device)
        self.recv_s = symm_mem.empty(max_rows, K // 128, dtype=torch.float32, device=device)
        self.recv_y = symm_mem.empty(max_slots, N, dtype=torch.bfloat16, device=device)
        self.hq = symm_mem.rendezvous(self.recv_q, group)
        self.hs = symm_mem.rendezvous(self.recv_s, group)
        self.hy = symm_mem.rendezvous(self.recv_y, group)

    def barrier(self):
        """Every rank's kernels enqueued so far (their peer writes) complete before what follows."""
        self.hq.barrier(channel=0)


def moe_forward(ex: Exchange, plan: ExchangePlan, x_local: torch.Tensor, gates: torch.Tensor, top_k: int,
                Bq: torch.Tensor, sB: torch.Tensor, ws: torch.Tensor | None = None, keep: dict | None = None):
    """The expert layer's FP8 forward on this rank: 1x128 quantization of its tokens ->
    FP8 dispatch over NVLink -> grouped Fprop over the received rows -> BF16 combine over NVLink ->
    gate-weighted sum.  keep (optional dict) receives the intermediate tensors for verification."""
    import paper_2412_19437_b200 as fp
    xq, xs = fp.quantize_act_1x128(x_local)
    fp.dispatch_fp8(xq, xs, top_k, plan.dst_rank_dev, plan.dst_row_dev, ex.hq.buffer_ptrs_dev, ex.K, ex.hs.buffer_ptrs_dev)
    ex.barrier()
    R = plan.rows
    A = ex.recv_q[:R]
    sA = fp.scales_rows_to_blocks(ex.recv_s[:R])
    y = fp.grouped_gemm(plan.offsets_dev, A, sA, Bq, sB, workspace=ws)
    fp.combine_push_bf16(y, plan.c_rank_dev, plan.c_slot_dev, ex.hy.buffer_ptrs_dev, ex.N)
    ex.barrier()
    out = fp.combine_reduce_bf16(ex.recv_y[:(plan.t1 - plan.t0) * top_k], gates)
    if keep is not None:
        keep.update(xq=xq, xs=xs, A=A, sA=sA, y=y, out=out)
    return out


def plan_to_device(plan: ExchangePlan, device) -> ExchangePlan:
    plan.dst_rank_dev = plan.dst_rank.to(device)
    plan.dst_row_dev = plan.dst_row.to(device)
    plan.offsets_dev = plan.offsets.to(device)
    plan.c_rank_dev = plan.c_rank.to(device)
    plan.c_slot_dev = plan.c_slot.to(device)
    return plan
