"""The README's grouped expert Wgrad example, checked against the unquantized per-expert product."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2412_19437_b200 as fp
offsets = [0, 300, 300, 1000]
xe = torch.randn(1000, 7168, device="cuda", dtype=torch.bfloat16)
dye = torch.randn(1000, 2048, device="cuda", dtype=torch.bfloat16)
XqT, sX = fp.quantize_act_128x1_grouped(xe, offsets)
DqT, sD = fp.quantize_act_128x1_grouped(dye, offsets)
dW = fp.grouped_gemm_wgrad(offsets, DqT, sD, XqT, sX)
torch.cuda.synchronize()
ref = [dye[0:300].float().T @ xe[0:300].float(), None, dye[300:].float().T @ xe[300:].float()]
print("shapes", tuple(XqT.shape), tuple(dW.shape), "dW[1] zero", bool((dW[1] == 0).all()))
for e in (0, 2):
    print("expert", e, "normwise vs unquantized", float((dW[e] - ref[e]).abs().max() / ref[e].abs().max()))
