"""Run the C4 expert-parallel grouped GEMM (1 rank) a few times: for ncu captures (experiments only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_19437_b200 import ep

cfg = ep.EPConfig()
dev = torch.device("cuda", 0)
pb = ep.build_rank_problem(cfg, 1, 0, dev, ep.routes_for(cfg))
for _ in range(4):
    ep.run_rank(pb)
torch.cuda.synchronize()
print("rows", pb.A.shape[0])
