#!/usr/bin/env python
"""bench.py — DeepSeek-V3 FP8 Linear training step on B200 (BASELINE.json configs[1]).

One STEP = the whole hot path for a Linear W [out=18432, in=7168]
over T=4096 tokens, synthetic seeded inputs (workloads.py):
    quantize_act_dual(X)  (1x128 for Fprop + 128x1 for Wgrad, one read of X)
    quantize_weight_128x128(W) (+ transposed copy for Dgrad)
    Fprop  Y  = Xq  . Wq^T          (BF16 out)
    quantize_act_dual(dY) (1x128 for Dgrad + 128x1 for Wgrad, one read of dY)
    Dgrad  dX = dYq . WqT^T         (BF16 out)
    Wgrad  dW = dYqT . XqT^T        (FP32 out)
value = 3 * 2*T*in*out GEMM FLOP per step / device time (TFLOP/s), whole job over all ranks.
Multi-GPU (torchrun): the dense step does not shard -> independent replicas, "scaling": "weak".
`--workload ep` times the expert-parallel grouped GEMM (BASELINE configs[4]) instead.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload dense|ep]

`--impl reference` times the CPU oracle (oracle/, as it stands) on a bounded sample of the same
workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "FP8 block-scaled GEMM TFLOPS (% of B200 FP8 peak); quantizer HBM GB/s"
T_TOK, D_IN, D_OUT = 4096, 7168, 18432
# CPU sample of the same step (cpu_baseline / --impl reference): 128 tokens x all 7168 inputs x
# the first CPU_OUT output channels.
CPU_TOK, CPU_OUT = 128, 2048


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "src": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}


# ------------------------------------------------------------------------ clocks ----
class ClockSampler:
    """NVML sampler of SM clock + throttle reasons while the timed region runs."""

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            pass

    def _run(self):
        nv = self.nv
        names = {getattr(nv, k, None): n for k, n in [
            ("nvmlClocksEventReasonSwPowerCap", "sw_power_cap"), ("nvmlClocksEventReasonHwSlowdown", "hw_slowdown"),
            ("nvmlClocksEventReasonHwThermalSlowdown", "hw_thermal_slowdown"),
            ("nvmlClocksEventReasonSwThermalSlowdown", "sw_thermal_slowdown"),
            ("nvmlClocksEventReasonHwPowerBrakeSlowdown", "hw_power_brake_slowdown")] if getattr(nv, k, None)}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, n in names.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self._ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------- dense step ----
class DenseStep:
    """Preallocated buffers + the 6 launches of one FP8 Linear training step.  pow2: the power-of-two
    scale recipe end to end: pow2 quantizers and the UE8M0 block-scaled GEMM."""

    def __init__(self, dev, T=T_TOK, IN=D_IN, OUT=D_OUT, seed=0, pow2=False):
        import paper_2412_19437_b200 as fp
        self.fp = fp
        self.pow2 = pow2
        self.T, self.IN, self.OUT = T, IN, OUT
        self.h_x = W.gaussian_act(T, IN, seed=seed)                 # BF16 activations
        self.h_w = W.master_weight(OUT, IN, seed=seed + 1)          # FP32 master weight
        self.h_dy = W.grad_out(T, OUT, seed=seed + 2)               # BF16 output gradient
        self.x, self.w, self.dy = self.h_x.to(dev), self.h_w.to(dev), self.h_dy.to(dev)
        u8, f32, bf = torch.uint8, torch.float32, torch.bfloat16
        e = lambda *s, dt=u8: torch.empty(*s, dtype=dt, device=dev)  # noqa: E731
        p4 = lambda n: (n + 3) // 4 * 4  # noqa: E731
        self.xq, self.sx = e(T, IN), e(IN // 128, p4(T), dt=f32)[:, :T]
        self.wq, self.sw, self.wqT = e(OUT, IN), e(OUT // 128, IN // 128, dt=f32), e(IN, OUT)
        self.y = e(T, OUT, dt=bf)
        self.dyq, self.sdy = e(T, OUT), e(OUT // 128, p4(T), dt=f32)[:, :T]
        self.dx = e(T, IN, dt=bf)
        self.dyqT, self.sdyT = e(OUT, T), e(T // 128, p4(OUT), dt=f32)[:, :OUT]
        self.xqT, self.sxT = e(IN, T), e(T // 128, p4(IN), dt=f32)[:, :IN]
        self.dw = e(OUT, IN, dt=f32)
        gf = 2.0 * T * IN * OUT
        # dual quantizer: bf16 in, codes of both groupings and both scale sets out
        BD = lambda m, k: 2 * m * k + 2 * m * k + 4 * m * ((k + 127) // 128) + 4 * k * ((m + 127) // 128)  # noqa: E731
        # name -> (callable, kind, algorithmic amount per launch: FLOP for gemm, bytes for quantizers)
        self.launches = [
            ("quant_act_dual(X)", self.q_x, "hbm", BD(T, IN)),
            ("quant_weight_128x128(W)+T", self.q_w, "hbm", 4 * OUT * IN + 2 * OUT * IN + 4 * (OUT // 128) * (IN // 128)),
            ("gemm_fprop", self.g_fprop, "tensor", gf),
            ("quant_act_dual(dY)", self.q_dy, "hbm", BD(T, OUT)),
            ("gemm_dgrad", self.g_dgrad, "tensor", gf),
            ("gemm_wgrad", self.g_wgrad, "tensor", gf),
        ]
        self.flops = 3 * gf
        self.h2d_bytes = self.h_x.numel() * 2 + self.h_w.numel() * 4 + self.h_dy.numel() * 2
        self.d2h_bytes = self.y.numel() * 2 + self.dx.numel() * 2 + self.dw.numel() * 4

    def q_x(self):
        self.fp.quantize_act_dual(self.x, self.xq, self.sx, self.xqT, self.sxT, pow2=self.pow2)

    def q_w(self):
        self.fp.quantize_weight_128x128(self.w, True, self.wq, self.sw, self.wqT, pow2=self.pow2)

    def g_fprop(self):
        self.fp.gemm(self.fp.FPROP, self.xq, self.sx, self.wq, self.sw, out=self.y, mx=self.pow2)

    def q_dy(self):
        self.fp.quantize_act_dual(self.dy, self.dyq, self.sdy, self.dyqT, self.sdyT, pow2=self.pow2)

    def g_dgrad(self):
        self.fp.gemm(self.fp.DGRAD, self.dyq, self.sdy, self.wqT, self.sw, out=self.dx, mx=self.pow2)

    def g_wgrad(self):
        self.fp.gemm(self.fp.WGRAD, self.dyqT, self.sdyT, self.xqT, self.sxT, out=self.dw, mx=self.pow2)

    def run(self):
        for _, fn, _, _ in self.launches:
            fn()


def cpu_sample_step():
    """The same step restricted to CPU_TOK tokens x CPU_OUT output channels, on the CPU oracle.
    Returns (seconds, GEMM FLOP)."""
    import oracle
    x = W.gaussian_act(T_TOK, D_IN, seed=0)[:CPU_TOK].contiguous()
    w = W.master_weight(CPU_OUT, D_IN, seed=1)
    dy = W.grad_out(CPU_TOK, CPU_OUT, seed=2)
    t0 = time.perf_counter()
    qx, sx = oracle.quantize_act_1x128(x)
    qw, sw, qwT = oracle.quantize_weight_128x128(w)
    oracle.gemm(oracle.FPROP, qx, sx, qw, sw)
    qdy, sdy = oracle.quantize_act_1x128(dy)
    oracle.gemm(oracle.DGRAD, qdy, sdy, qwT, sw)
    qdyT, sdyT = oracle.quantize_act_128x1(dy)
    qxT, sxT = oracle.quantize_act_128x1(x)
    oracle.gemm(oracle.WGRAD, qdyT, sdyT, qxT, sxT)
    return time.perf_counter() - t0, 3 * 2.0 * CPU_TOK * D_IN * CPU_OUT


def cpu_baseline_block(min_seconds=10.0):
    """Time the oracle on repeated samples until at least min_seconds of CPU work."""
    import oracle
    dt, fl = 0.0, 0.0
    while dt < min_seconds:
        d, f = cpu_sample_step()
        dt += d
        fl += f
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": oracle.max_threads(), "kind": "oracle",
            "sample": f"the C1 step restricted to {CPU_TOK} tokens x {D_IN} in x {CPU_OUT} out channels "
                      f"(all 8 stages: 3 quantizers + weight quantizer + Fprop/Dgrad/Wgrad FP64 oracle GEMMs), "
                      f"{fl / 1e9:.2f} GFLOP in {dt:.2f} s"}


# ------------------------------------------------------------------------ main ----
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if args.impl == "ours" else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v: float, world: int, dev) -> float:
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_reference(args, world, rank):
    if rank != 0:
        return
    # torchrun exports OMP_NUM_THREADS=1; rank 0 runs the oracle alone on the box's host cores
    torch.set_num_threads(len(os.sched_getaffinity(0)))   # the process's OpenMP pool (shared with the oracle)
    for _ in range(args.warmup):
        cpu_sample_step()
    t, f = 0.0, 0.0
    for _ in range(args.steps):
        d, fl = cpu_sample_step()
        t += d
        f += fl
    import oracle
    v = f / t / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_block(args, world),
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": oracle.max_threads(), "kind": "oracle",
                             "sample": f"each step: the C1 step restricted to {CPU_TOK} tokens x {D_IN} in x "
                                       f"{CPU_OUT} out channels on the CPU oracle"},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_block(args, world):
    if args.workload == "ep":
        return {"workload": "C4 expert-parallel grouped GEMM: 256 experts (K=7168, N=2048) sharded over ranks, "
                            "65536 tokens x top-8, skewed load", "parallelism": f"ep{world}",
                "l2": "inputs larger than L2"}
    return {"workload": "C1 dense FP8 Linear training step (quantize + Fprop/Dgrad/Wgrad), BASELINE configs[1]",
            "tokens": T_TOK, "in": D_IN, "out": D_OUT, "global_batch": T_TOK * world,
            "parallelism": "replicas" if world > 1 else "single",
            "l2": "inputs larger than L2 (738 MB read per step: X, W, dY)"}


def time_dense(args, world, rank, dev):
    peaks = load_peaks()
    st = DenseStep(dev)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        st.run()
    torch.cuda.synchronize()
    nL = len(st.launches)
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nL)]
          for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        start.record(stream)
        for k in range(args.steps):
            for i, (_, fn, _, _) in enumerate(st.launches):
                ev[k][i][0].record(stream)
                fn()
                ev[k][i][1].record(stream)
        stop.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms_local = start.elapsed_time(stop)
    ms = max_over_ranks(ms_local, world, dev)
    per = {}
    for i, (name, _, kind, amount) in enumerate(st.launches):
        d = statistics.mean(ev[k][i][0].elapsed_time(ev[k][i][1]) for k in range(args.steps))
        if kind == "tensor":
            ach = amount / (d * 1e-3) / 1e12
            peak = 2.0 * peaks["bf16_tflops"]       # FP8 = 2x BF16 (guide's nominal ratio)
            per[name] = {"ms": d, "achieved": ach, "unit": "TFLOP/s", "peak": peak, "frac": ach / peak}
        else:
            ach = amount / (d * 1e-3) / 1e9
            per[name] = {"ms": d, "achieved": ach, "unit": "GB/s", "peak": peaks["hbm_gbs"], "frac": ach / peaks["hbm_gbs"]}
    dom = max(per, key=lambda n: per[n]["ms"])
    dk = next(l for l in st.launches if l[0] == dom)
    traffic, traffic_src = None, None
    try:   # DRAM bytes per launch of this kernel from the committed ncu --set full capture
        tj = json.load(open(os.path.join(ROOT, "profiles", "r01", "traffic.json")))
        traffic = tj["dram_bytes_per_launch"].get(dom)
        traffic_src = tj["source"]
    except Exception:
        pass
    # Tensor-bound roofline kernel: the guide's sustained peak applies to a kernel timed inside a long
    # step; the timed region is taken as "long" when the clock sampler saw the power cap.  The burst
    # fraction is reported next to it.
    clocks = clk.summary()
    sustained = dk[2] == "tensor" and "sw_power_cap" in clocks.get("reasons", [])
    peak_t = 2.0 * (peaks["bf16_tflops_sustained"] if sustained else peaks["bf16_tflops"])
    roof_peak = peak_t if dk[2] == "tensor" else per[dom]["peak"]
    roof = {"kernel": dom, "bound": "tensor" if dk[2] == "tensor" else "hbm", "achieved": per[dom]["achieved"],
            "peak": roof_peak, "unit": per[dom]["unit"], "frac": per[dom]["achieved"] / roof_peak, "traffic": traffic,
            "traffic_unit": "bytes per launch", "traffic_src": traffic_src,
            "peak_src": f"{peaks['src']}: " + (("2 x bf16_tflops_sustained (timed region power-capped: sw_power_cap)" if sustained
                                                else "2 x bf16_tflops (burst)") + " of MEASURED_PEAKS.json" if dk[2] == "tensor"
                                               else "hbm_gbs of MEASURED_PEAKS.json"),
            "frac_vs_burst_peak": per[dom]["frac"],
            "share_of_step": per[dom]["ms"] * args.steps / (ms_local)}
    value = world * st.flops * args.steps / (ms * 1e-3) / 1e12
    gemm_ms = sum(per[n]["ms"] for n in per if n.startswith("gemm"))
    q_ms = sum(per[n]["ms"] for n in per if not n.startswith("gemm"))
    q_bytes = sum(l[3] for l in st.launches if l[2] == "hbm")
    result = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "e4m3", "data": "synthetic", "config": config_block(args, world),
        "roofline": roof, "clocks": clocks, "gpu_launches": nL * args.steps,
        "gemm_tflops": st.flops / (gemm_ms * 1e-3) / 1e12, "gemm_frac_fp8_peak_4500": st.flops / (gemm_ms * 1e-3) / 4.5e15,
        "quantizer_gbs": q_bytes / (q_ms * 1e-3) / 1e9, "quantizer_frac_hbm": q_bytes / (q_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
        "kernels": per,
    }
    if args.e2e:
        result["e2e"] = time_e2e(args, world, st, dev)
    if args.pow2:
        del st
        result["pow2_recipe"] = time_pow2_recipe(args, dev)
    return result


def time_pow2_recipe(args, dev):
    """Context line, not the headline: the same C1 step on the power-of-two scale recipe (
    pow2 dual / weight quantizers, UE8M0 block-scaled GEMM fp8bs_gemm_mx), timed like the main step
    on this rank's stream after it (per-launch CUDA events, inputs larger than L2)."""
    st = DenseStep(dev, pow2=True)
    stream = torch.cuda.current_stream()
    steps = min(args.steps, 50)
    for _ in range(args.warmup):
        st.run()
    torch.cuda.synchronize()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in st.launches]
          for _ in range(steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(steps):
        for i, (_, fn, _, _) in enumerate(st.launches):
            ev[k][i][0].record(stream)
            fn()
            ev[k][i][1].record(stream)
    stop.record(stream)
    torch.cuda.synchronize()
    ms = start.elapsed_time(stop)
    per = {}
    for i, (name, _, kind, amount) in enumerate(st.launches):
        d = statistics.mean(ev[k][i][0].elapsed_time(ev[k][i][1]) for k in range(steps))
        per[name] = {"ms": d, "achieved": amount / (d * 1e-3) / (1e12 if kind == "tensor" else 1e9),
                     "unit": "TFLOP/s" if kind == "tensor" else "GB/s"}
    return {"value": st.flops * steps / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms / steps,
            "steps": steps, "recipe": "power-of-two scales (P:558, P:565): fp8bs_quantize_act_dual_pow2, "
            "fp8bs_quantize_weight_128x128_pow2, fp8bs_gemm_mx (UE8M0 block scaling, no promotion step)",
            "kernels": per}


def time_e2e(args, world, st, dev):
    """Same metric through the public API with host buffers: every step copies X, W, dY from pinned
    host memory to the device, runs the 6 launches, and copies Y, dX, dW back to pinned host memory.
    Steps are pipelined over two buffer sets and three streams (H2D, compute, D2H): the copies of
    step k+1's inputs and step k-1's outputs overlap step k's kernels, and PCIe runs both directions
    at once.  Timed from the first H2D to the last D2H on the device."""
    n = max(4, args.steps // 4)
    hx = [st.h_x.pin_memory() for _ in range(2)]
    hw = [st.h_w.pin_memory() for _ in range(2)]
    hdy = [st.h_dy.pin_memory() for _ in range(2)]
    hy = [torch.empty(st.y.shape, dtype=st.y.dtype).pin_memory() for _ in range(2)]
    hdx = [torch.empty(st.dx.shape, dtype=st.dx.dtype).pin_memory() for _ in range(2)]
    hdw = [torch.empty(st.dw.shape, dtype=st.dw.dtype).pin_memory() for _ in range(2)]
    sets = [(st.x, st.w, st.dy, st.y, st.dx, st.dw),
            tuple(torch.empty_like(t) for t in (st.x, st.w, st.dy, st.y, st.dx, st.dw))]
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event(enable_timing=False)  # noqa: E731

    def run(nsteps, timed):
        h2d_done, comp_done, d2h_done = {}, {}, {}
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for k in range(nsteps):
            b = k % 2
            x, w, dy, y, dx, dw = sets[b]
            with torch.cuda.stream(s_in):
                if k >= 2:
                    s_in.wait_event(comp_done[k - 2])          # inputs of set b consumed
                if k == 0 and timed:
                    t0.record(s_in)
                x.copy_(hx[b], non_blocking=True)
                w.copy_(hw[b], non_blocking=True)
                dy.copy_(hdy[b], non_blocking=True)
                h2d_done[k] = ev()
                h2d_done[k].record(s_in)
            comp.wait_event(h2d_done[k])
            if k >= 2:
                comp.wait_event(d2h_done[k - 2])               # outputs of set b copied out
            st.x, st.w, st.dy, st.y, st.dx, st.dw = x, w, dy, y, dx, dw
            st.run()
            comp_done[k] = ev()
            comp_done[k].record(comp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(comp_done[k])
                hy[b].copy_(y, non_blocking=True)
                hdx[b].copy_(dx, non_blocking=True)
                hdw[b].copy_(dw, non_blocking=True)
                d2h_done[k] = ev()
                d2h_done[k].record(s_out)
        if timed:
            t1.record(s_out)
        torch.cuda.synchronize()
        return t0, t1

    run(max(2, args.warmup // 2), False)
    barrier(world)
    torch.cuda.synchronize()
    t0, t1 = run(n, True)
    barrier(world)
    st.x, st.w, st.dy, st.y, st.dx, st.dw = sets[0]
    ms = max_over_ranks(t0.elapsed_time(t1), world, dev)
    return {"value": world * st.flops * n / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "steps": n,
            "h2d_bytes_per_step": st.h2d_bytes, "d2h_bytes_per_step": st.d2h_bytes,
            "ms_per_step": ms / n, "pipelined": "2 buffer sets; H2D, compute and D2H streams overlap across steps"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="dense", choices=["dense", "ep"])
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu", dest="cpu", action="store_false")
    ap.add_argument("--no-pow2", dest="pow2", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if args.workload == "ep":
        from paper_2412_19437_b200 import ep
        result = ep.bench(args, world, rank, dev, barrier, max_over_ranks, ClockSampler, load_peaks)
        result["config"] = config_block(args, world)
        result["metric"] = METRIC
    else:
        result = time_dense(args, world, rank, dev)
    if rank == 0:
        if args.cpu and world == 1:
            result["cpu_baseline"] = cpu_baseline_block()
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
