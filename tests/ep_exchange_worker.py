"""Worker of tests/test_ep_exchange_gpu.py (torchrun, one process per GPU): the expert layer's FP8
forward with the NVLink exchange (ep.moe_forward) on a seeded problem, checked on every rank:
  * dispatch: the received FP8 rows and scales == a host gather of every rank's 1x128 codes (bitwise);
  * expert GEMM: == the grouped GEMM on the host-gathered rows (bitwise);
  * combine: == oracle.combine_bf16 of the gathered expert outputs with the rank's gates (bitwise).
Then times the two exchanges alone (CUDA events) and reports bytes moved over NVLink per second.
    torchrun --nproc-per-node 2 tests/ep_exchange_worker.py [tokens experts top_k K N [placement]] > result.json
placement: contiguous (default) or balanced (observed-load LPT with one redundant expert per rank)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import oracle
import paper_2412_19437_b200 as fp
import workloads as W
from paper_2412_19437_b200 import ep


def main():
    T, E, top_k, K, N = (int(a) for a in (sys.argv[1:6] if len(sys.argv) > 5 else (4096, 16, 4, 1024, 512)))
    kind = sys.argv[6] if len(sys.argv) > 6 else "contiguous"
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    routes = W.route_skewed(T, E, top_k, seed=3)
    tok, off = W.group_rows(routes, E)
    if kind == "balanced":   # loads observed on an independent batch of the same routing distribution
        prev = W.route_skewed(T, E, top_k, seed=4, popularity_seed=3)
        placement = ep.balanced_placement(torch.bincount(prev.reshape(-1).long(), minlength=E), world, world)
    else:
        placement = ep.contiguous_placement(E, world)
    plans = [ep.exchange_plan(routes, E, world, r, placement) for r in range(world)]
    plan = ep.plan_to_device(plans[rank], dev)
    x = W.gaussian_act(T, K, seed=0)
    B = W.random_codes(E * N, K, seed=5).reshape(E, N, K)
    sB = W.random_scales(E, N // 128, K // 128, seed=6)
    g = torch.rand(T, top_k, generator=torch.Generator().manual_seed(7))
    gates = g / g.sum(1, keepdim=True)
    t0, t1 = plan.t0, plan.t1
    x_local = x[t0:t1].to(dev)
    Bq, sBl = B[plan.experts].contiguous().to(dev), sB[plan.experts].contiguous().to(dev)
    gl = gates[t0:t1].contiguous().to(dev)
    ws = torch.empty(int(fp.lib().fp8bs_grouped_gemm_workspace_size(max(len(plan.experts), 1), max(plan.rows, 1), N, K)) + 16,
                     dtype=torch.uint8, device=dev)
    ex = ep.Exchange(dist.group.WORLD, dev, max(p.rows for p in plans), max((p.t1 - p.t0) * top_k for p in plans), K, N,
                     dispatch_ctas=int(os.environ.get("FP8BS_EP_CTAS", "32")))
    keep = {}
    out = ep.moe_forward(ex, plan, x_local, gl, top_k, Bq, sBl, ws=ws, keep=keep, fused=False)
    torch.cuda.synchronize()
    out = out.clone()
    # the fused form (combine's send in the grouped GEMM's epilogue) must give the same bits
    out_fused = ep.moe_forward(ex, plan, x_local, gl, top_k, Bq, sBl, ws=ws, fused=True, dedup=False).clone()
    torch.cuda.synchronize()
    # the streamed form (dispatch overlapped with the GEMM through per-chunk ready flags), twice: the
    # second call exercises the monotonic counters and the other combine buffer
    outs_streamed = [ep.moe_forward(ex, plan, x_local, gl, top_k, Bq, sBl, ws=ws, streamed=True).clone() for _ in range(3)]
    out_dedup = ep.moe_forward(ex, plan, x_local, gl, top_k, Bq, sBl, ws=ws, dedup=True).clone()
    torch.cuda.synchronize()
    # ---- verification (NCCL all_gather outside the measured calls) ----
    def gather_cat(t, dim=0):
        parts = ep.gather_rows(t.transpose(0, dim).contiguous() if dim else t.contiguous(), world)
        cat = torch.cat(parts)
        return cat.transpose(0, dim) if dim else cat
    xq_all = gather_cat(keep["xq"])                       # [T, K] in token order
    xs_all = gather_cat(keep["xs"], dim=1)                # [KB, T]
    rows = tok[plan.grows].to(dev)
    A_ref = xq_all.index_select(0, rows)
    sA_ref = xs_all.index_select(1, rows)
    res = {"rank": rank, "rows": plan.rows, "tokens": t1 - t0, "placement": kind, "experts": len(plan.experts)}
    res["dispatch_codes_bitwise"] = bool(torch.equal(keep["A"], A_ref))
    res["dispatch_scales_bitwise"] = bool(torch.equal(keep["sA"].contiguous().view(torch.int32), sA_ref.contiguous().view(torch.int32)))
    sa_pad = torch.empty(sA_ref.shape[0], (plan.rows + 3) // 4 * 4, dtype=torch.float32, device=dev)[:, :plan.rows]
    sa_pad.copy_(sA_ref)
    y_ref = fp.grouped_gemm(plan.offsets_dev, A_ref.contiguous(), sa_pad, Bq, sBl)
    res["expert_gemm_bitwise"] = bool(torch.equal(keep["y"].view(torch.int16), y_ref.view(torch.int16)))
    y_parts = ep.gather_rows(keep["y"].contiguous(), world)
    y_all = torch.empty(T * top_k, N, dtype=torch.bfloat16, device=dev)   # global expert-grouped order
    for r in range(world):
        y_all.index_copy_(0, plans[r].grows.to(dev), y_parts[r])
    order = torch.argsort(routes.reshape(-1).to(torch.int64) * T + torch.arange(T).repeat_interleave(top_k), stable=True)
    pos = torch.empty_like(order)
    pos[order] = torch.arange(order.numel())
    y_slots = y_all.cpu()[pos[t0 * top_k:t1 * top_k]]    # this rank's slots (t, j), t in [t0, t1)
    ref = oracle.combine_bf16(y_slots, gates[t0:t1])
    res["combine_bitwise_vs_oracle"] = bool(torch.equal(out.cpu().view(torch.int16), ref.view(torch.int16)))
    res["fused_scatter_bitwise_vs_unfused"] = bool(torch.equal(out_fused.view(torch.int16), out.view(torch.int16)))
    res["dedup_bitwise_vs_unfused"] = bool(torch.equal(out_dedup.view(torch.int16), out.view(torch.int16)))
    res["streamed_bitwise_vs_unfused"] = all(bool(torch.equal(o.view(torch.int16), out.view(torch.int16))) for o in outs_streamed)
    # ---- timing of the exchanges alone ----
    xq, xs = keep["xq"], keep["xs"]
    remote_slots = int((plan.dst_rank != rank).sum())
    remote_rows = int((plan.c_rank != rank).sum())

    def timeit(fn, iters=20):
        for _ in range(3):
            fn()
        ex.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / iters
    ms_d = timeit(lambda: fp.dispatch_fp8(xq, xs, top_k, plan.dst_rank_dev, plan.dst_row_dev, ex.hq.buffer_ptrs_dev, K,
                                          ex.hs.buffer_ptrs_dev))
    ms_c = timeit(lambda: fp.combine_push_bf16(keep["y"], plan.c_rank_dev, plan.c_slot_dev, ex.hy.buffer_ptrs_dev, N))
    res["dispatch_ms"] = ms_d
    res["dispatch_remote_GBps"] = remote_slots * (K + 4 * (K // 128)) / (ms_d * 1e-3) / 1e9
    res["dispatch_total_GBps"] = (t1 - t0) * top_k * (K + 4 * (K // 128)) / (ms_d * 1e-3) / 1e9
    res["combine_ms"] = ms_c
    res["combine_remote_GBps"] = remote_rows * N * 2 / (ms_c * 1e-3) / 1e9
    for c in (32,):                     # the streamed dispatch alone (no GEMM waiting on it)
        def ds():
            ex.epoch += 1
            fp.dispatch_fp8_stream(plan.chunk_off_dev, plan.send_tok_dev, plan.send_rank_dev, plan.send_row_dev, xq, xs,
                                   ex.hq.buffer_ptrs_dev, ex.K, ex.hsb.buffer_ptrs_dev, ex.ld_sb, ex.local_done,
                                   ex.hf.buffer_ptrs_dev, ex.world, ex.epoch, c)
        res[f"dispatch_stream_ms_ctas{c}"] = timeit(ds, 10)
    res["layer_ms_unfused"] = timeit(lambda: ep.moe_forward(ex, plan, x_local, gl, top_k, Bq, sBl, ws=ws, fused=False), 10)
    res["layer_ms_fused"] = timeit(lambda: ep.moe_forward(ex, plan, x_local, gl, top_k, Bq, sBl, ws=ws, fused=True, dedup=False), 10)
    res["layer_ms_dedup"] = timeit(lambda: ep.moe_forward(ex, plan, x_local, gl, top_k, Bq, sBl, ws=ws, dedup=True), 10)
    res["send_rows_ms"] = timeit(lambda: fp.send_rows(plan.u_tok_dev, xq, xs, plan.u_rank_dev, plan.u_row_dev,
                                                      ex.htq.buffer_ptrs_dev, K, ex.hts.buffer_ptrs_dev))
    res["layer_ms_streamed"] = timeit(lambda: ep.moe_forward(ex, plan, x_local, gl, top_k, Bq, sBl, ws=ws, streamed=True), 10)
    res["streamed_after_timing_bitwise"] = bool(torch.equal(
        ep.moe_forward(ex, plan, x_local, gl, top_k, Bq, sBl, ws=ws, streamed=True).view(torch.int16), out.view(torch.int16)))
    ex.barrier()
    torch.cuda.synchronize()
    allres = [None] * world
    dist.all_gather_object(allres, res)
    if rank == 0:
        print(json.dumps({"world": world, "T": T, "E": E, "top_k": top_k, "K": K, "N": N, "ranks": allres}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
