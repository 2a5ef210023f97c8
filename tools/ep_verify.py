"""Expert-parallel verification ("EP" pin): gathered outputs at G ranks are
bitwise equal to the G = 1 result, and per-rank row counts / imbalance are reported.

    torchrun --nproc-per-node G --master-addr 127.0.0.1 tools/ep_verify.py [tokens]

Rank 0 also recomputes all experts on its own GPU (the G = 1 problem) and compares.  NCCL is used
only here, to gather outputs (never inside a timed region)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_2412_19437_b200 import ep


def main():
    tokens = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl")
    cfg = ep.EPConfig(tokens=tokens)
    routes = ep.routes_for(cfg)
    pb = ep.build_rank_problem(cfg, world, rank, dev, routes)
    out = ep.run_rank(pb)
    torch.cuda.synchronize()
    parts = ep.gather_rows(out, world) if world > 1 else [out]
    if rank == 0:
        got = torch.cat(parts)
        ref_pb = ep.build_rank_problem(cfg, 1, 0, dev, routes)
        ref = ep.run_rank(ref_pb)
        torch.cuda.synchronize()
        rows = [p.shape[0] for p in parts]
        res = {"world": world, "tokens": tokens, "rows_per_rank": rows, "imbalance": ep.imbalance(rows),
               "bitwise_equal_to_G1": bool(torch.equal(got.view(torch.int16), ref.view(torch.int16))),
               "max_abs_diff": float((got.float() - ref.float()).abs().max())}
        print(json.dumps(res))
        assert res["bitwise_equal_to_G1"], res
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
