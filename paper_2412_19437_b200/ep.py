"""Expert-parallel sharding of the grouped MoE expert GEMM (BASELINE configs[4]).

DeepSeek-V3 trains with 64-way expert parallelism and no token dropping
(P:267-270).  Here the grouped expert Fprop is partitioned by expert replica: a `Placement` says which
experts (or which share of a duplicated expert's rows) each rank computes.  Two placements:
  * contiguous: rank r owns the expert block [r*E/W, (r+1)*E/W) (the r01/r02a layout);
  * balanced: experts are rearranged among the GPUs by observed load so that every GPU
    processes about the same number of rows, optionally with redundant copies of the hottest experts
    (the paper deploys one extra expert per GPU for prefilling), each copy taking an equal
    share of that expert's rows.
Experts are independent, so the bench's timed path has NO exchange step: every rank regenerates, from
the shared seeds, the routing of all tokens, its experts' weights and the FP8 rows routed to them, and
runs one fp8bs_grouped_gemm.  The NVLink exchange (dispatch / combine) is the second half of
this module (`exchange_plan`, `Exchange`, `moe_forward`).  NCCL (torch.distributed) gathers per-rank
outputs for verification only, outside any timed region.

Bookkeeping helpers are pure functions (unit-tested on CPU, world_size 2 over gloo);
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


# ------------------------------------------------------------------------------------------
# Expert placement: which expert replicas each rank computes.
# ------------------------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Placement:
    """groups[r] = the (expert, part, parts) triples rank r computes, in its local (launch) order:
    the part-th of `parts` equal contiguous chunks of expert e's rows (rows in (expert, token) order,
    W.group_rows; chunk bounds floor(part * c / parts)).  parts > 1 means e is deployed redundantly
    on `parts` distinct ranks.  Every row of every expert belongs to exactly one (rank, group)."""
    world: int
    experts: int
    groups: tuple
    kind: str = "contiguous"
    redundant: int = 0

    def experts_of(self, rank: int) -> list[int]:
        return [e for e, _, _ in self.groups[rank]]


def contiguous_placement(E: int, world: int) -> Placement:
    """Rank r owns the contiguous expert block shard_range(E, world, r)."""
    return Placement(world, E, tuple(tuple((e, 0, 1) for e in range(*shard_range(E, world, r))) for r in range(world)))


def balanced_placement(load, world: int, redundant: int = 0) -> Placement:
    """Load-aware placement: "duplicates high-load experts and deploys them redundantly"
    and "rearrange[s] experts among GPUs ... based on the observed loads, striving to balance the load
    across GPUs".  The paper gives the goal, not the algorithm (reading R29):
      1. redundancy: `redundant` times, give one more copy to the expert with the largest load per
         copy (at most `world` copies: copies sit on distinct ranks); a copy's load is load / copies;
      2. rearrangement: longest-processing-time-first list scheduling — copies in decreasing load
         (ties by expert id) each go to the least-loaded rank (ties by rank id) that has room and does
         not already hold a copy of that expert.  Room: ceil((E + redundant) / world) copies per rank,
         i.e. the paper's "original 8 experts" plus "one additional redundant expert" when
         redundant == world.
    `load` is the OBSERVED per-expert row count (a previous batch's statistics): the placement
    is fixed before the batch it serves; each copy then takes an equal share of the batch's rows."""
    load = torch.as_tensor(load, dtype=torch.float64)
    E = load.numel()
    if not 0 <= redundant <= E * (world - 1):
        raise ValueError(f"redundant={redundant} outside [0, E*(world-1)]")
    copies = torch.ones(E, dtype=torch.int64)
    for _ in range(redundant):
        per = torch.where(copies < world, load / copies, torch.full_like(load, -1.0))
        copies[int(torch.argmax(per))] += 1            # argmax: first index among equals
    items = sorted(((float(load[e]) / int(copies[e]), e, p) for e in range(E) for p in range(int(copies[e]))),
                   key=lambda it: (-it[0], it[1], it[2]))
    cap = -(-len(items) // world)
    rank_load = [0.0] * world
    held = [[] for _ in range(world)]
    for w, e, p in items:
        cand = [r for r in range(world) if len(held[r]) < cap and all(x[0] != e for x in held[r])]
        if not cand:                                  # only reachable when the room is exhausted
            cand = [r for r in range(world) if all(x[0] != e for x in held[r])]
        r = min(cand, key=lambda r: (rank_load[r], r))
        held[r].append((e, p, int(copies[e])))
        rank_load[r] += w
    return Placement(world, E, tuple(tuple(sorted(h)) for h in held), "balanced", redundant)


def chunk_bounds(c: int, part: int, parts: int) -> tuple[int, int]:
    """Rows [lo, hi) of an expert's c rows that copy `part` of `parts` computes."""
    return part * c // parts, (part + 1) * c // parts


def placement_rows(offsets: torch.Tensor, placement: Placement, rank: int):
    """Rank `rank`'s rows under `placement`.  offsets: the global (expert, token) grouping's int64
    [E + 1] (W.group_rows).  Returns (global row indices int64 [R_r], local offsets int64 [G_r + 1],
    expert ids int64 [G_r]) — local group g is rows[loff[g]:loff[g+1]] of expert experts[g]."""
    idx, loff, exps = [], [0], []
    for e, part, parts in placement.groups[rank]:
        a = int(offsets[e])
        lo, hi = chunk_bounds(int(offsets[e + 1]) - a, part, parts)
        idx.append(torch.arange(a + lo, a + hi, dtype=torch.int64))
        loff.append(loff[-1] + hi - lo)
        exps.append(e)
    rows = torch.cat(idx) if idx else torch.zeros(0, dtype=torch.int64)
    return rows, torch.tensor(loff, dtype=torch.int64), torch.tensor(exps, dtype=torch.int64)


def rank_rows(offsets: torch.Tensor, placement: Placement) -> list[int]:
    """Rows each rank computes under `placement`."""
    out = []
    for r in range(placement.world):
        n = 0
        for e, part, parts in placement.groups[r]:
            lo, hi = chunk_bounds(int(offsets[e + 1] - offsets[e]), part, parts)
            n += hi - lo
        out.append(n)
    return out


def observed_load(cfg: "EPConfig") -> torch.Tensor:
    """Per-expert row counts of a PREVIOUS batch of cfg's routing distribution (same expert popularity,
    independent token draws, seed + 1): the statistics a balanced placement is built from."""
    if cfg.skew_alpha > 0:
        prev = W.route_skewed(cfg.tokens, cfg.experts, cfg.top_k, alpha=cfg.skew_alpha, seed=cfg.seed + 1,
                              popularity_seed=cfg.seed)
    else:
        prev = W.route_uniform(cfg.tokens, cfg.experts, cfg.top_k, seed=cfg.seed + 1)
    return torch.bincount(prev.reshape(-1).to(torch.int64), minlength=cfg.experts)


def make_placement(cfg: "EPConfig", world: int, kind: str = "balanced", redundant: int | None = None) -> Placement:
    """kind "contiguous" or "balanced"; balanced defaults to one redundant expert per rank at world > 1
     and takes its loads from observed_load(cfg)."""
    if kind == "contiguous" or world == 1:
        return contiguous_placement(cfg.experts, world)
    if kind != "balanced":
        raise ValueError(kind)
    return balanced_placement(observed_load(cfg), world, world if redundant is None else redundant)


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
    experts: list               # expert id of each local group (launch order)
    rows: torch.Tensor          # int64 [R_local], CPU: the global (expert, token)-order index of each row
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
    placement: Placement | None = None


def token_shard(T: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous data-parallel token shard of `rank` (the tokens whose activations it quantizes
    before dispatch)."""
    return shard_range(T, world, rank)


def build_rank_problem(cfg: EPConfig, world: int, rank: int, device, routes: torch.Tensor | None = None,
                       keep_tokens: bool = False, placement: Placement | None = None) -> RankProblem:
    """Everything rank `rank` needs under `placement` (default: contiguous), regenerated from the seeds
    (identical on every rank).  Activations: N(0,1) BF16 from a seeded CUDA generator; quantized 1x128
    ONCE per token (the paper quantizes before dispatch) and the FP8 rows + per-row scales
    are gathered — exact, because 1x128 scales are per row.  A redundant expert's weights are
    regenerated from the expert's own seed on every rank that holds a copy.  keep_tokens: also keep
    the rank's data-parallel token shard (BF16) and output buffers for its 1x128 codes / scales
    (bench.py's C4 step quantizes it)."""
    import paper_2412_19437_b200 as fp
    if routes is None:
        routes = routes_for(cfg)
    if placement is None:
        placement = contiguous_placement(cfg.experts, world)
    assert placement.world == world and placement.experts == cfg.experts
    tok_all, goff = W.group_rows(routes, cfg.experts)
    grows, offsets, exps = placement_rows(goff, placement, rank)
    tok = tok_all[grows]
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
    experts = [int(e) for e in exps]
    G = len(experts)
    Bq = torch.empty(G, N, K, dtype=torch.uint8, device=device)
    sB = torch.empty(G, N // 128, K // 128, dtype=torch.float32, device=device)
    for i, e in enumerate(experts):
        ge = torch.Generator(device=device)
        ge.manual_seed(cfg.seed + 1000 + e)
        w = (torch.randn(N, K, generator=ge, device=device, dtype=torch.float32) * 0.006).to(torch.bfloat16)
        fp.quantize_weight_128x128(w, want_t=False, q=Bq[i], s=sB[i])
    out = torch.empty(R, N, dtype=torch.bfloat16, device=device)
    pb = RankProblem(experts, grows, offsets.to(device), tok, A, sA, Bq, sB, out, 2.0 * R * N * K, t0, t1,
                     placement=placement)
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


def placement_equals_G1_on_one_gpu(pb: RankProblem, placement: Placement) -> bool:
    """On ONE GPU holding the whole (G = 1) problem `pb` (its rows in global order): run every rank of
    `placement` as its own grouped launch on its own rows and experts, scatter the outputs back to the
    global row order and compare with the G = 1 output bitwise (the partition bench.py times at
    N GPUs, without NCCL)."""
    import paper_2412_19437_b200 as fp
    assert pb.rows.numel() == 0 or bool(torch.equal(pb.rows, torch.arange(pb.rows.numel())))
    ref = run_rank(pb).clone()
    goff = pb.offsets.cpu()
    got = torch.zeros_like(ref)
    dev = pb.A.device
    for r in range(placement.world):
        rows, loff, exps = placement_rows(goff, placement, r)
        n = rows.numel()
        if n == 0:
            continue
        rd = rows.to(dev)
        sa = torch.empty(pb.sA.shape[0], (n + 3) // 4 * 4, dtype=torch.float32, device=dev)[:, :n]
        sa.copy_(pb.sA.index_select(1, rd))
        ed = exps.to(dev)
        y = fp.grouped_gemm(loff.to(dev), pb.A.index_select(0, rd), sa, pb.Bq.index_select(0, ed).contiguous(),
                            pb.sB.index_select(0, ed).contiguous())
        got.index_copy_(0, rd, y)
        del y, sa
    return bool(torch.equal(got.view(torch.int16), ref.view(torch.int16)))


def split_equals_G1_on_one_gpu(pb: RankProblem, cfg: EPConfig, splits=(2, 4, 8), kind: str = "contiguous") -> dict:
    """placement_equals_G1_on_one_gpu for the `kind` placement at each G in `splits`."""
    return {str(G): placement_equals_G1_on_one_gpu(pb, make_placement(cfg, G, kind)) for G in splits}


def gathered_equals_G1(pb: RankProblem, cfg: EPConfig, world: int, rank: int, device, routes) -> bool | None:
    """N > 1: NCCL all_gather of every rank's output rows (verification only, outside any timed
    region); rank 0 scatters them back to the global row order, rebuilds the G = 1 problem on its own
    GPU and compares bitwise.  Returns the verdict on rank 0, None elsewhere."""
    parts = gather_rows(pb.out, world)
    if rank != 0:
        return None
    _, goff = W.group_rows(routes, cfg.experts)
    got = torch.empty((int(goff[-1]), pb.out.shape[1]), dtype=pb.out.dtype, device=pb.out.device)
    for r, part in enumerate(parts):
        rows, _, _ = placement_rows(goff, pb.placement, r)
        got.index_copy_(0, rows.to(got.device), part)
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
    experts: list                    # expert id of each of this rank's local groups
    grows: torch.Tensor              # int64 [R_local]: global (expert, token)-order index of each received row
    dst_rank: torch.Tensor           # int32 [(t1 - t0) * top_k]: rank computing slot (t, j)'s row
    dst_row: torch.Tensor            # int64 [...]: its row in that rank's expert-grouped receive buffer
    offsets: torch.Tensor            # int64 [G_local + 1]: this rank's received rows per local group
    c_rank: torch.Tensor             # int32 [R_local]: token owner of each received row
    c_slot: torch.Tensor             # int64 [R_local]: its slot (t - t0(owner)) * top_k + j there
    rows: int                        # R_local
    # streamed dispatch (fp8bs_dispatch_fp8_stream): this rank's slots sorted by (chunk, dst rank, dst
    # row), chunk c of a receiver = the rows of its local groups g with g * chunks // G == c
    chunks: int = 8
    send_tok: torch.Tensor | None = None    # int64 [S]: local token (t - t0) of entry j
    send_rank: torch.Tensor | None = None   # int32 [S]
    send_row: torch.Tensor | None = None    # int64 [S]
    chunk_off: torch.Tensor | None = None   # int64 [chunks + 1]: entries of chunk c are [chunk_off[c], chunk_off[c+1])
    # token-once dispatch (fp8bs_send_rows + fp8bs_expand_rows): each (token, destination rank) pair is sent
    # once, into the receiver's token buffer (rows grouped by source rank, tokens in order); the receiver
    # expands them into its expert-grouped rows
    u_tok: torch.Tensor | None = None       # int64 [U]: local token (t - t0) of send entry j
    u_rank: torch.Tensor | None = None      # int32 [U]: destination rank
    u_row: torch.Tensor | None = None       # int64 [U]: row in the destination's token buffer
    x_idx: torch.Tensor | None = None       # int64 [R_local]: token-buffer row of each of this rank's expert rows
    tok_rows: int = 0                       # rows of this rank's token buffer


def exchange_plan(routes: torch.Tensor, E: int, world: int, rank: int,
                  placement: Placement | None = None, chunks: int = 8) -> ExchangePlan:
    """Dispatch / combine bookkeeping of `rank` under `placement` (default contiguous): slot (t, j) of
    a token goes to the rank computing its global row; with a redundant expert, the copy whose share
    of the expert's rows holds that row (chunk_bounds)."""
    if placement is None:
        placement = contiguous_placement(E, world)
    T, k = routes.shape
    flat_e = routes.reshape(-1).to(torch.int64)
    flat_t = torch.arange(T, dtype=torch.int64).repeat_interleave(k)
    order = torch.argsort(flat_e * T + flat_t, stable=True)          # global row -> flat slot (as group_rows)
    pos = torch.empty_like(order)
    pos[order] = torch.arange(order.numel(), dtype=torch.int64)      # flat slot -> global row
    counts = torch.bincount(flat_e, minlength=E)
    offsets = torch.zeros(E + 1, dtype=torch.int64)
    offsets[1:] = torch.cumsum(counts, 0)
    owner_of_row = torch.full((T * k,), -1, dtype=torch.int64)
    lrow_of_row = torch.full((T * k,), -1, dtype=torch.int64)
    chunk_of_row = torch.zeros(T * k, dtype=torch.int64)
    mine = None
    for r in range(world):
        rows_r, loff_r, exps_r = placement_rows(offsets, placement, r)
        owner_of_row[rows_r] = r
        lrow_of_row[rows_r] = torch.arange(rows_r.numel(), dtype=torch.int64)
        G_r = loff_r.numel() - 1
        if G_r > 0:
            grp = torch.repeat_interleave(torch.arange(G_r, dtype=torch.int64), loff_r[1:] - loff_r[:-1])
            chunk_of_row[rows_r] = grp * chunks // G_r
        if r == rank:
            mine = (rows_r, loff_r, exps_r)
    assert bool((owner_of_row >= 0).all()), "placement does not cover every row"
    t_start = torch.tensor([token_shard(T, world, r)[0] for r in range(world)] + [T], dtype=torch.int64)
    t0, t1 = token_shard(T, world, rank)
    sl = slice(t0 * k, t1 * k)
    g = pos[sl]
    rows_me, loff, exps = mine
    slots = order[rows_me]                                            # flat slots of this rank's rows
    tok = slots // k
    tok_owner = torch.searchsorted(t_start, tok, right=True) - 1
    c_slot = (tok - t_start[tok_owner]) * k + slots % k
    d_rank, d_row, d_chunk = owner_of_row[g], lrow_of_row[g], chunk_of_row[g]
    key = (d_chunk * world + d_rank) * (T * k) + d_row
    order_s = torch.argsort(key, stable=True)
    chunk_off = torch.zeros(chunks + 1, dtype=torch.int64)
    chunk_off[1:] = torch.cumsum(torch.bincount(d_chunk, minlength=chunks), 0)
    # token-once dispatch: the distinct (token, destination rank) pairs, sorted by token; a receiver's
    # token-buffer row of a pair is its index among the pairs with that receiver (source ranks own
    # contiguous token ranges, so the rows come grouped by source rank)
    slot_rank = owner_of_row[pos]                                     # [T * k] destination rank of every slot
    pair = torch.unique(flat_t * world + slot_rank)                   # sorted: by token, then rank
    p_tok, p_rank = pair // world, pair % world
    p_row = torch.empty_like(pair)
    for o in range(world):
        m = p_rank == o
        p_row[m] = torch.arange(int(m.sum()), dtype=torch.int64)
    mine_p = (p_tok >= t0) & (p_tok < t1)
    recv_p = p_rank == rank
    tb_row = torch.full((T,), -1, dtype=torch.int64)                  # token -> its row in MY token buffer
    tb_row[p_tok[recv_p]] = p_row[recv_p]
    x_idx = tb_row[tok]
    return ExchangePlan(t0, t1, [int(e) for e in exps], rows_me, d_rank.to(torch.int32), d_row,
                        loff, tok_owner.to(torch.int32), c_slot, int(rows_me.numel()), chunks,
                        order_s // k, d_rank[order_s].to(torch.int32), d_row[order_s], chunk_off,
                        p_tok[mine_p] - t0, p_rank[mine_p].to(torch.int32), p_row[mine_p], x_idx, int(recv_p.sum()))


class Exchange:
    """Symmetric-memory receive buffers of the exchange (rendezvous over `group`): FP8 codes + row-major
    scales for dispatch, BF16 expert outputs per token slot for combine; for the streamed dispatch also
    the scales in the GEMM's [K/128][ld] layout, the per-chunk ready flags (uint32, zeroed once) and two
    combine buffers used alternately (a peer's GEMM of forward n+1 may write while this rank still reads
    forward n's)."""

    def __init__(self, group, device, max_rows: int, max_slots: int, K: int, N: int, chunks: int = 8,
                 dispatch_ctas: int = 32):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        self.K, self.N, self.chunks, self.ctas = K, N, chunks, dispatch_ctas
        self.world = dist.get_world_size(group)
        self.recv_q = symm_mem.empty(max_rows, K, dtype=torch.uint8, device=device)
        self.recv_s = symm_mem.empty(max_rows, K // 128, dtype=torch.float32, device=device)
        self.ld_sb = max(4, (max_rows + 3) // 4 * 4)
        self.recv_sb = symm_mem.empty(K // 128, self.ld_sb, dtype=torch.float32, device=device)
        self.recv_y = symm_mem.empty(max_slots, N, dtype=torch.bfloat16, device=device)
        self.recv_y2 = symm_mem.empty(max_slots, N, dtype=torch.bfloat16, device=device)
        # token-once dispatch: token buffers (a token's row arrives once per rank; rows <= expert rows)
        self.tok_q = symm_mem.empty(max_rows, K, dtype=torch.uint8, device=device)
        self.tok_s = symm_mem.empty(max_rows, K // 128, dtype=torch.float32, device=device)
        self.flags = symm_mem.empty(chunks, dtype=torch.int32, device=device)
        self.flags.zero_()
        self.hq = symm_mem.rendezvous(self.recv_q, group)
        self.hs = symm_mem.rendezvous(self.recv_s, group)
        self.hsb = symm_mem.rendezvous(self.recv_sb, group)
        self.hy = symm_mem.rendezvous(self.recv_y, group)
        self.hy2 = symm_mem.rendezvous(self.recv_y2, group)
        self.hf = symm_mem.rendezvous(self.flags, group)
        self.htq = symm_mem.rendezvous(self.tok_q, group)
        self.hts = symm_mem.rendezvous(self.tok_s, group)
        self.local_done = torch.zeros(chunks, dtype=torch.int32, device=device)
        self.epoch = 0
        self.dstream = torch.cuda.Stream(device=device)
        self.num_sms = torch.cuda.get_device_properties(device).multi_processor_count
        torch.cuda.synchronize(device)
        self.hf.barrier(channel=0)          # every rank's flags are zero before anyone can signal them

    def barrier(self):
        """Every rank's kernels enqueued so far (their peer writes) complete before what follows."""
        self.hq.barrier(channel=0)


def moe_forward(ex: Exchange, plan: ExchangePlan, x_local: torch.Tensor, gates: torch.Tensor, top_k: int,
                Bq: torch.Tensor, sB: torch.Tensor, ws: torch.Tensor | None = None, keep: dict | None = None,
                fused: bool = True, streamed: bool = False, dedup: bool = True):
    """The expert layer's FP8 forward on this rank: 1x128 quantization of its tokens ->
    FP8 dispatch over NVLink -> grouped Fprop over the received rows -> BF16 combine over NVLink ->
    gate-weighted sum.  fused (default): the grouped Fprop's epilogue stores each BF16 output row
    straight into its token owner's combine buffer (fp8bs_grouped_gemm_scatter), so the combine's
    send overlaps the GEMM and y never exists in HBM; fused=False runs the GEMM into y and then
    fp8bs_combine_push_bf16.  streamed (implies fused): the dispatch runs on its own stream and SMs
    (fp8bs_dispatch_fp8_stream, chunk by chunk in the receivers' expert order, scales straight into the
    GEMM's layout) while the GEMM, on the remaining SMs, waits per chunk on the ready flags the senders
    publish: no barrier and no scale re-layout between dispatch and GEMM.  dedup (default; with fused,
    not streamed): each (token, destination rank) pair crosses the link once (fp8bs_send_rows into the
    receivers' token buffers), and each receiver expands its expert rows locally (fp8bs_expand_rows, the
    scales straight into the GEMM layout).  keep (optional dict) receives the intermediate tensors for
    verification."""
    import paper_2412_19437_b200 as fp
    xq, xs = fp.quantize_act_1x128(x_local)
    R = plan.rows
    y = None
    buf = ex.recv_y
    if streamed:
        ex.epoch += 1
        hy = ex.hy if ex.epoch % 2 else ex.hy2
        buf = ex.recv_y if ex.epoch % 2 else ex.recv_y2
        main = torch.cuda.current_stream()
        ex.dstream.wait_stream(main)
        with torch.cuda.stream(ex.dstream):
            fp.dispatch_fp8_stream(plan.chunk_off_dev, plan.send_tok_dev, plan.send_rank_dev, plan.send_row_dev, xq, xs,
                                   ex.hq.buffer_ptrs_dev, ex.K, ex.hsb.buffer_ptrs_dev, ex.ld_sb, ex.local_done,
                                   ex.hf.buffer_ptrs_dev, ex.world, ex.epoch, ex.ctas)
        A = ex.recv_q[:R]
        sA = ex.recv_sb[:, :R]
        if R > 0:
            fp.grouped_gemm_scatter(plan.offsets_dev, A, sA, Bq, sB, hy.buffer_ptrs_dev, plan.c_rank_dev, plan.c_slot_dev,
                                    ex.N, workspace=ws, ready=ex.flags, ready_target=ex.world * ex.epoch,
                                    ready_chunks=plan.chunks, max_sms=ex.num_sms - ex.ctas)
        main.wait_stream(ex.dstream)
        xq.record_stream(ex.dstream)
        xs.record_stream(ex.dstream)
    elif dedup and fused:
        fp.send_rows(plan.u_tok_dev, xq, xs, plan.u_rank_dev, plan.u_row_dev, ex.htq.buffer_ptrs_dev, ex.K,
                     ex.hts.buffer_ptrs_dev)
        ex.barrier()
        A, sA = ex.recv_q[:R], ex.recv_sb[:, :R]
        if R > 0:
            fp.expand_rows(plan.x_idx_dev, ex.tok_q[:plan.tok_rows], ex.tok_s[:plan.tok_rows], A=A, sA=sA)
            fp.grouped_gemm_scatter(plan.offsets_dev, A, sA, Bq, sB, ex.hy.buffer_ptrs_dev, plan.c_rank_dev,
                                    plan.c_slot_dev, ex.N, workspace=ws)
    else:
        fp.dispatch_fp8(xq, xs, top_k, plan.dst_rank_dev, plan.dst_row_dev, ex.hq.buffer_ptrs_dev, ex.K, ex.hs.buffer_ptrs_dev)
        ex.barrier()
        A = ex.recv_q[:R]
        sA = fp.scales_rows_to_blocks(ex.recv_s[:R])
        if fused:
            if R > 0:
                fp.grouped_gemm_scatter(plan.offsets_dev, A, sA, Bq, sB, ex.hy.buffer_ptrs_dev, plan.c_rank_dev,
                                        plan.c_slot_dev, ex.N, workspace=ws)
        else:
            y = fp.grouped_gemm(plan.offsets_dev, A, sA, Bq, sB, workspace=ws)
            fp.combine_push_bf16(y, plan.c_rank_dev, plan.c_slot_dev, ex.hy.buffer_ptrs_dev, ex.N)
    ex.barrier()
    out = fp.combine_reduce_bf16(buf[:(plan.t1 - plan.t0) * top_k], gates)
    if keep is not None:
        keep.update(xq=xq, xs=xs, A=A, sA=sA, y=y, out=out)
    return out


def plan_to_device(plan: ExchangePlan, device) -> ExchangePlan:
    plan.dst_rank_dev = plan.dst_rank.to(device)
    plan.dst_row_dev = plan.dst_row.to(device)
    plan.offsets_dev = plan.offsets.to(device)
    plan.c_rank_dev = plan.c_rank.to(device)
    plan.c_slot_dev = plan.c_slot.to(device)
    plan.send_tok_dev = plan.send_tok.to(device)
    plan.send_rank_dev = plan.send_rank.to(device)
    plan.send_row_dev = plan.send_row.to(device)
    plan.chunk_off_dev = plan.chunk_off.to(device)
    plan.u_tok_dev = plan.u_tok.to(device)
    plan.u_rank_dev = plan.u_rank.to(device)
    plan.u_row_dev = plan.u_row.to(device)
    plan.x_idx_dev = plan.x_idx.to(device)
    return plan
