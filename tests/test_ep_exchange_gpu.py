"""Expert-parallel NVLink exchange (NEXT-3) on 2 GPUs: runs tests/ep_exchange_worker.py under
torchrun and checks that dispatch, the expert GEMM and combine are bitwise equal to the host-gathered
references on every rank.  Skipped with fewer than 2 GPUs (the driver's GPU tier runs on one)."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("shape", [(4096, 16, 4, 1024, 512), (3000, 32, 8, 2048, 768),
                                   (3000, 32, 8, 2048, 768, "balanced")], ids=["small", "ragged", "ragged-balanced"])
def test_ep_exchange_two_gpus(shape):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr=127.0.0.1",
           "--master-port=29555", os.path.join(ROOT, "tests", "ep_exchange_worker.py"), *map(str, shape)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, start_new_session=True)
    assert p.returncode == 0, p.stderr[-3000:]
    res = json.loads(p.stdout.strip().splitlines()[-1])
    for r in res["ranks"]:
        for key in ("dispatch_codes_bitwise", "dispatch_scales_bitwise", "expert_gemm_bitwise", "combine_bitwise_vs_oracle",
                    "fused_scatter_bitwise_vs_unfused", "streamed_bitwise_vs_unfused", "streamed_after_timing_bitwise",
                    "dedup_bitwise_vs_unfused"):
            assert r[key], (key, r)
