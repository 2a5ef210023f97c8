#!/usr/bin/env python
"""bench.py — DeepSeek-V3 FP8 expert GEMM (BASELINE.json configs[4], the north_star target) on B200.

Headline (default `--workload c4`): the expert-parallel grouped expert GEMM of C4 — 256 routed
experts (K = 7168 hidden, N = 2048 expert FFN dim), 65536 tokens x top-8 with skewed
routing (524288 expert rows), experts sharded contiguously over the N ranks (ep.py).  One STEP on
rank r is the FP8 forward of its share of the expert layer:
    quantize_act_1x128(X[t0:t1])     the 1x128 cast of the rank's data-parallel token shard, the
                                     cast the paper applies before dispatch (a-1, a-2)
    grouped_gemm(offsets, A, sA, Bq, sB) -> BF16   Fprop over the FP8 rows its experts receive
                                     (a-5..a-8; the rows are the exact gather of the same 1x128
                                     codes — dispatch itself is out of scope)
value = sum over ranks of 2 * R_r * N * K GEMM FLOP per step / max-over-ranks step time (TFLOP/s);
the total problem is fixed ("scaling": "strong").  `roofline` is the grouped GEMM kernel's, from
CUDA events around each launch inside the timed region.  The C1 dense FP8 Linear training step
(quantizers + Fprop/Dgrad/Wgrad, BASELINE configs[1]) is timed after it on every rank and reported
as the sub-object `c1_step` (per-kernel TFLOP/s and GB/s; replicas at N > 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c4|c1]

`--impl reference` times the CPU oracle (oracle/, as it stands) on a bounded sample of the same C4
step on the host cores (rank 0 only; the other ranks exit without work).
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
# CPU sample of the C1 step (its cpu_baseline): 128 tokens x all 7168 inputs x the first CPU_OUT outputs
CPU_TOK, CPU_OUT = 128, 2048
# CPU sample of the C4 step: every CPU_EXPERT_STRIDE-th expert, CPU_ROWS rows each
CPU_EXPERT_STRIDE, CPU_ROWS = 16, 4
# A timed region at least this long is "a kernel timed inside a long step": its tensor roofline takes
# the measured SUSTAINED peak (MEASURED_PEAKS.json: 4 s back to back); shorter regions the burst one.
SUSTAINED_REGION_S = 1.0


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "src": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}


def fp8_peak(peaks, region_s: float):
    """Dense FP8 peak = 2 x the measured BF16 peak (the guide's nominal FP8:BF16 ratio): sustained
    for a timed region of >= SUSTAINED_REGION_S, burst otherwise.  Returns (peak, label)."""
    sustained = region_s >= SUSTAINED_REGION_S
    key = "bf16_tflops_sustained" if sustained else "bf16_tflops"
    return 2.0 * peaks[key], (f"{peaks['src']}: 2 x {key} of MEASURED_PEAKS.json "
                              f"({'sustained' if sustained else 'burst'}: timed region {region_s:.3f} s "
                              f"{'>=' if sustained else '<'} {SUSTAINED_REGION_S} s)")


def committed_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture (or None)."""
    for rnd in ("r02", "r01"):
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", rnd, "traffic.json")))
        except Exception:
            continue
        v = tj.get("dram_bytes_per_launch", {}).get(kernel)
        if v is not None:
            return v, tj.get("source")
    return None, None


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
        # split-K tail workspace (fp8bs_gemm_ws): one buffer for the three GEMMs (same stream); the
        # shapes with a tail (C1: Dgrad) run 3 kernels — full waves, tail units, reduce
        shapes = {fp.FPROP: (T, OUT, IN), fp.DGRAD: (T, IN, OUT), fp.WGRAD: (OUT, IN, T)}
        wsb = {l: (0 if pow2 else fp.gemm_workspace_size(l, *shp)) for l, shp in shapes.items()}
        self.ws = e(max(max(wsb.values()), 16))
        self.kernels = {l: (3 if wsb[l] > 0 else 1) for l in shapes}
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
        self.fp.gemm(self.fp.FPROP, self.xq, self.sx, self.wq, self.sw, out=self.y, mx=self.pow2, workspace=self.ws)

    def q_dy(self):
        self.fp.quantize_act_dual(self.dy, self.dyq, self.sdy, self.dyqT, self.sdyT, pow2=self.pow2)

    def g_dgrad(self):
        self.fp.gemm(self.fp.DGRAD, self.dyq, self.sdy, self.wqT, self.sw, out=self.dx, mx=self.pow2, workspace=self.ws)

    def g_wgrad(self):
        self.fp.gemm(self.fp.WGRAD, self.dyqT, self.sdyT, self.xqT, self.sxT, out=self.dw, mx=self.pow2, workspace=self.ws)

    def run(self):
        for _, fn, _, _ in self.launches:
            fn()

    def kernel_count(self) -> int:
        """Kernels one step launches: 3 quantizers + the GEMMs (3 kernels for a split-K tail)."""
        return 3 + sum(self.kernels.values())


# ------------------------------------------------------------------- timing helpers ----
def timed_launches(launches, steps, warmup, world, dev):
    """Run `warmup` untimed steps, then `steps` timed steps of the launch list [(name, fn), ...] on the
    current stream with a CUDA event pair around each launch, bracketed by barrier + synchronize.
    Returns (region ms on this rank, per-launch mean ms list, clock summary)."""
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        for _, fn in launches:
            fn()
    torch.cuda.synchronize()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in launches]
          for _ in range(steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        start.record(stream)
        for k in range(steps):
            for i, (_, fn) in enumerate(launches):
                ev[k][i][0].record(stream)
                fn()
                ev[k][i][1].record(stream)
        stop.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    per = [statistics.mean(ev[k][i][0].elapsed_time(ev[k][i][1]) for k in range(steps)) for i in range(len(launches))]
    return start.elapsed_time(stop), per, clk.summary()


# ------------------------------------------------------------------------ C1 step ----
def time_c1(args, world, rank, dev, e2e=False):
    """The C1 dense FP8 Linear training step (6 launches), replicas at N > 1 ("scaling": "weak")."""
    peaks = load_peaks()
    st = DenseStep(dev)
    ms_local, per_ms, clocks = timed_launches([(n, fn) for n, fn, _, _ in st.launches], args.steps, args.warmup,
                                              world, dev)
    ms = max_over_ranks(ms_local, world, dev)
    peak_t, peak_src = fp8_peak(peaks, ms_local * 1e-3)
    per = {}
    for (name, _, kind, amount), d in zip(st.launches, per_ms):
        if kind == "tensor":
            ach = amount / (d * 1e-3) / 1e12
            per[name] = {"ms": d, "achieved": ach, "unit": "TFLOP/s", "peak": peak_t, "frac": ach / peak_t}
        else:
            ach = amount / (d * 1e-3) / 1e9
            per[name] = {"ms": d, "achieved": ach, "unit": "GB/s", "peak": peaks["hbm_gbs"], "frac": ach / peaks["hbm_gbs"]}
    dom = max(per, key=lambda n: per[n]["ms"])
    dk = next(l for l in st.launches if l[0] == dom)
    traffic, traffic_src = committed_traffic(dom)
    tensor = dk[2] == "tensor"
    roof = {"kernel": dom, "bound": "tensor" if tensor else "hbm", "achieved": per[dom]["achieved"],
            "peak": per[dom]["peak"], "unit": per[dom]["unit"], "frac": per[dom]["frac"],
            "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
            "traffic_src": traffic_src, "algorithmic": dk[3],
            "peak_src": peak_src if tensor else f"{peaks['src']}: hbm_gbs of MEASURED_PEAKS.json",
            "share_of_step": per[dom]["ms"] * args.steps / ms_local}
    if tensor:
        sus = 2.0 * peaks["bf16_tflops_sustained"]
        roof["frac_vs_sustained_peak"] = per[dom]["achieved"] / sus
    gemm_ms = sum(per[n]["ms"] for n in per if n.startswith("gemm"))
    q_ms = sum(per[n]["ms"] for n in per if not n.startswith("gemm"))
    q_bytes = sum(l[3] for l in st.launches if l[2] == "hbm")
    res = {"workload": "C1 dense FP8 Linear training step (dual-quantize X, quantize W (+WqT), Fprop, dual-quantize dY, "
                       "Dgrad, Wgrad), BASELINE configs[1]", "tokens": T_TOK, "in": D_IN, "out": D_OUT,
           "parallelism": "replicas" if world > 1 else "single", "scaling": "weak",
           "value": world * st.flops * args.steps / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
           "ms_per_step": ms / args.steps, "steps": args.steps, "warmup": args.warmup, "dtype": "e4m3",
           "l2": "inputs larger than L2 (738 MB read per step: X, W, dY)",
           "roofline": roof, "clocks": clocks, "gpu_launches": st.kernel_count() * args.steps,
           "gemm_tflops": st.flops / (gemm_ms * 1e-3) / 1e12,
           "quantizer_gbs": q_bytes / (q_ms * 1e-3) / 1e9, "quantizer_frac_hbm": q_bytes / (q_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
           "kernels": per}
    if e2e:
        res["e2e"] = time_c1_e2e(args, world, st, dev)
    if args.pow2:
        del st
        res["pow2_recipe"] = time_pow2_recipe(args, world, dev)
    return res


def time_pow2_recipe(args, world, dev):
    """Context, not the headline: the same C1 step on the power-of-two scale recipe (
    pow2 dual / weight quantizers, UE8M0 block-scaled GEMM fp8bs_gemm_mx), timed like the C1 step."""
    st = DenseStep(dev, pow2=True)
    steps = min(args.steps, 50)
    ms, per_ms, _ = timed_launches([(n, fn) for n, fn, _, _ in st.launches], steps, args.warmup, world, dev)
    per = {name: {"ms": d, "achieved": amount / (d * 1e-3) / (1e12 if kind == "tensor" else 1e9),
                  "unit": "TFLOP/s" if kind == "tensor" else "GB/s"}
           for (name, _, kind, amount), d in zip(st.launches, per_ms)}
    return {"value": st.flops * steps / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms / steps,
            "steps": steps, "recipe": "power-of-two scales (P:558, P:565): fp8bs_quantize_act_dual_pow2, "
            "fp8bs_quantize_weight_128x128_pow2, fp8bs_gemm_mx (UE8M0 block scaling, no promotion step)",
            "kernels": per}


def pipelined_e2e(n, warmup, world, dev, h_in, d_sets, h_out_sets, run_compute):
    """Steps pipelined over two device buffer sets and three streams (H2D, compute, D2H): every step
    copies its inputs from pinned host memory (h_in: list of host tensors, one set) into its device
    set, runs the kernels, and copies its outputs back into pinned host memory (alternating sets).
    d_sets[b] = (inputs list, outputs list).  Timed on the device from the first H2D to the last D2H.
    Returns max-over-ranks ms for n steps."""
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event(enable_timing=False)  # noqa: E731

    def run(nsteps, timed):
        h2d_done, comp_done, d2h_done = {}, {}, {}
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for k in range(nsteps):
            b = k % 2
            d_in, d_out = d_sets[b]
            with torch.cuda.stream(s_in):
                if k >= 2:
                    s_in.wait_event(comp_done[k - 2])          # inputs of set b consumed
                if k == 0 and timed:
                    t0.record(s_in)
                for d, h in zip(d_in, h_in):
                    d.copy_(h, non_blocking=True)
                h2d_done[k] = ev()
                h2d_done[k].record(s_in)
            comp.wait_event(h2d_done[k])
            if k >= 2:
                comp.wait_event(d2h_done[k - 2])               # outputs of set b copied out
            run_compute(b)
            comp_done[k] = ev()
            comp_done[k].record(comp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(comp_done[k])
                for h, d in zip(h_out_sets[b], d_out):
                    h.copy_(d, non_blocking=True)
                d2h_done[k] = ev()
                d2h_done[k].record(s_out)
        if timed:
            t1.record(s_out)
        torch.cuda.synchronize()
        return t0, t1

    run(max(2, warmup), False)
    barrier(world)
    torch.cuda.synchronize()
    t0, t1 = run(n, True)
    barrier(world)
    return max_over_ranks(t0.elapsed_time(t1), world, dev)


def time_c1_e2e(args, world, st, dev):
    """C1 step through the public API with host buffers (X, W, dY in; Y, dX, dW out)."""
    n = max(4, args.steps // 4)
    h_in = [st.h_x.pin_memory(), st.h_w.pin_memory(), st.h_dy.pin_memory()]
    outs0 = [st.y, st.dx, st.dw]
    sets = [([st.x, st.w, st.dy], outs0),
            ([torch.empty_like(t) for t in (st.x, st.w, st.dy)], [torch.empty_like(t) for t in outs0])]
    h_out = [[torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in outs0] for _ in range(2)]

    def compute(b):
        (st.x, st.w, st.dy), (st.y, st.dx, st.dw) = sets[b]
        st.run()

    ms = pipelined_e2e(n, args.warmup, world, dev, h_in, sets, h_out, compute)
    (st.x, st.w, st.dy), (st.y, st.dx, st.dw) = sets[0]
    return {"value": world * st.flops * n / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "steps": n,
            "h2d_bytes_per_step": st.h2d_bytes, "d2h_bytes_per_step": st.d2h_bytes, "ms_per_step": ms / n,
            "pipelined": "2 buffer sets; H2D, compute and D2H streams overlap across steps"}


# ------------------------------------------------------------------------ C4 step ----
def c4_config(world, placement="balanced"):
    how = ("placed over ranks by a previous batch's observed loads (LPT, one redundant expert per rank at N > 1, "
           "P:584-589)" if placement == "balanced" else "sharded contiguously over ranks")
    return {"workload": "C4 expert-parallel grouped expert GEMM (BASELINE configs[4]): 256 routed experts (K=7168, "
                        f"N=2048) {how}, 65536 tokens x top-8 skewed routing (alpha 0.5, seed 3) "
                        "= 524288 expert rows; step = 1x128 quantize of the rank's token shard + grouped Fprop (BF16 out)",
            "experts": 256, "hidden": 7168, "expert_ffn": 2048, "tokens": 65536, "top_k": 8, "global_batch": 65536,
            "parallelism": f"ep{world}",
            "l2": "inputs larger than L2 (3.76 GB of FP8 rows + 3.76 GB of FP8 expert weights per step at N=1)"}


def time_c4(args, world, rank, dev):
    from paper_2412_19437_b200 import ep
    peaks = load_peaks()
    cfg = ep.EPConfig()
    routes = ep.routes_for(cfg)
    placement = ep.make_placement(cfg, world, args.placement, args.redundant)
    pb = ep.build_rank_problem(cfg, world, rank, dev, routes, keep_tokens=True, placement=placement)
    torch.cuda.synchronize()
    launches = [("quant_act_1x128(X shard)", lambda: ep.quantize_tokens(pb)), ("grouped_gemm_fprop", lambda: ep.run_rank(pb))]
    # our kernels per step: the quantizer, then k_grouped_schedule + k_gemm_bs (the grouped call also
    # zeroes its 4-byte claim counter with cudaMemsetAsync, not a kernel of ours)
    kernels_per_step = (1 if pb.x is not None and pb.x.shape[0] > 0 else 0) + (2 if pb.A.shape[0] > 0 else 0)
    ms_local, per_ms, clocks = timed_launches(launches, args.steps, args.warmup, world, dev)
    ms = max_over_ranks(ms_local, world, dev)
    K, N = cfg.hidden, cfg.inter
    R = pb.A.shape[0]
    rows = gather_ints([R], world, dev)
    ms_ranks = gather_floats([ms_local / args.steps], world, dev)
    total_flops = sum(2.0 * r * N * K for r in rows)
    Tl = pb.t1 - pb.t0
    q_bytes = Tl * K * 2 + Tl * K + 4 * Tl * (K // 128)          # BF16 in, codes + scales out
    q_ms, g_ms = per_ms
    g_ach = pb.flops / (g_ms * 1e-3) / 1e12
    peak_t, peak_src = fp8_peak(peaks, ms_local * 1e-3)
    traffic, traffic_src = committed_traffic("grouped_gemm_fprop")
    alg_bytes = R * K + len(pb.experts) * N * K + 4 * R * (K // 128) + 2 * R * N
    roof = {"kernel": "grouped_gemm_fprop (k_gemm_bs grouped)", "bound": "tensor", "achieved": g_ach, "peak": peak_t,
            "unit": "TFLOP/s", "frac": g_ach / peak_t, "peak_src": peak_src,
            "frac_vs_sustained_peak": g_ach / (2.0 * peaks["bf16_tflops_sustained"]),
            "algorithmic": pb.flops, "algorithmic_unit": "FLOP per launch (2 * R * N * K)",
            "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
            "traffic_src": traffic_src, "algorithmic_bytes": alg_bytes,
            "share_of_step": g_ms * args.steps / ms_local}
    kernels = {"quant_act_1x128(X shard)": {"ms": q_ms, "achieved": q_bytes / (q_ms * 1e-3) / 1e9, "unit": "GB/s",
                                            "peak": peaks["hbm_gbs"], "frac": q_bytes / (q_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                                            "bytes": q_bytes},
               "grouped_gemm_fprop": {"ms": g_ms, "achieved": g_ach, "unit": "TFLOP/s", "peak": peak_t, "frac": g_ach / peak_t,
                                      "flop": pb.flops}}
    _, goff = W.group_rows(routes, cfg.experts)
    ep_block = {"placement": placement.kind, "redundant_experts": placement.redundant,
                "rows_per_rank": rows, "experts_per_rank": [len(g) for g in placement.groups],
                "ms_per_step_per_rank": ms_ranks, "imbalance_max_over_mean": ep.imbalance(rows),
                "scaling_bound_from_imbalance": 1.0 / ep.imbalance(rows),
                "imbalance_if_contiguous": ep.imbalance(ep.rank_rows(goff, ep.contiguous_placement(cfg.experts, world))),
                "collective": "none in the timed path; NCCL all_gather of outputs for verification only"}
    result = {"metric": METRIC, "value": total_flops * args.steps / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
              "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
              "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "e4m3",
              "data": "synthetic (seeded Gaussian activations, N(0, 0.006^2) expert weights, skewed top-8 routing)",
              "config": c4_config(world, args.placement), "roofline": roof, "clocks": clocks, "gpu_launches": kernels_per_step * args.steps,
              "kernels": kernels, "ep": ep_block}
    # verification, outside the timed region
    if args.verify:
        if world > 1:
            ok = ep.gathered_equals_G1(pb, cfg, world, rank, dev, routes)
            ep_block["bitwise_equal_to_G1"] = ok
            ep_block["verify"] = "NCCL all_gather of every rank's output rows; rank 0 recomputes G=1 on its GPU"
        else:
            ep_block["split_bitwise_equal_to_G1_on_one_gpu"] = ep.split_equals_G1_on_one_gpu(pb, cfg)
            ep_block["balanced_split_bitwise_equal_to_G1_on_one_gpu"] = ep.split_equals_G1_on_one_gpu(pb, cfg, kind="balanced")
            ep_block["verify"] = ("G=2/4/8 contiguous and balanced (redundant) placements, each rank a separate launch "
                                  "on one GPU, scattered back to global row order vs the G=1 launch")
    if args.e2e:
        result["e2e"] = time_c4_e2e(args, world, pb, dev, rows, N, K)
    return result, pb


def time_c4_e2e(args, world, pb, dev, rows, N, K):
    """The C4 step through the public API with host buffers, as a user holding BF16 tokens and the router's
    output runs it: every step uploads, from pinned host memory, the BF16 rows of the distinct tokens this
    rank's expert rows use and the row -> token index, then runs 1x128 quantization of those tokens ->
    fp8bs_expand_rows (gather into expert-grouped FP8 rows, scales into the GEMM layout) -> the grouped
    Fprop, and downloads the BF16 expert outputs.  The expert weights stay resident, as model parameters
    do.  The output is checked bitwise against the device-timed step's (1x128 scales are per row, so
    quantizing the gathered tokens gives the same codes)."""
    import paper_2412_19437_b200 as fp
    from paper_2412_19437_b200 import ep
    cfg = ep.EPConfig()
    # as many steps as the device-timed region (<= 20): the pipeline's fill (the first upload) and drain
    # (the last download) are paid once per timed region, as in a serving loop
    n = max(3, min(20, args.steps))
    uniq, inv = torch.unique(pb.tok, return_inverse=True)
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed + 100)                      # the token batch of build_rank_problem
    x = torch.randn(cfg.tokens, K, generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    h_x = x.index_select(0, uniq.to(dev)).cpu().pin_memory()
    del x
    h_idx = inv.to(torch.int64).contiguous().pin_memory()
    U, R, KB = uniq.numel(), pb.A.shape[0], K // 128
    p4 = lambda m: (m + 3) // 4 * 4  # noqa: E731

    def dset():
        ins = [torch.empty(U, K, dtype=torch.bfloat16, device=dev), torch.empty(R, dtype=torch.int64, device=dev)]
        scratch = (torch.empty(U, K, dtype=torch.uint8, device=dev),
                   torch.empty(KB, p4(U), dtype=torch.float32, device=dev)[:, :U],
                   torch.empty(R, K, dtype=torch.uint8, device=dev),
                   torch.empty(KB, p4(R), dtype=torch.float32, device=dev)[:, :R])
        return ins, [torch.empty(R, N, dtype=torch.bfloat16, device=dev)], scratch
    d = [dset(), dset()]
    sets = [(d[0][0], d[0][1]), (d[1][0], d[1][1])]
    h_out = [[torch.empty(R, N, dtype=torch.bfloat16).pin_memory()] for _ in range(2)]

    def compute(b):
        (xb, idxb), (outb,), (xq, xs, A, sA) = d[b]
        if R == 0:
            return
        fp.quantize_act_1x128(xb, xq, xs)
        fp.expand_rows(idxb, xq, xs, A=A, sA=sA, ts_layout="blocks")
        fp.grouped_gemm(pb.offsets, A, sA, pb.Bq, pb.sB, out=outb, workspace=pb.ws)

    ms = pipelined_e2e(n, 2, world, dev, [h_x, h_idx], sets, h_out, compute)
    ep.run_rank(pb)
    torch.cuda.synchronize()
    same = bool(torch.equal(h_out[(n - 1) % 2][0].view(torch.int16), pb.out.cpu().view(torch.int16)))
    del d, sets
    torch.cuda.empty_cache()
    total = sum(2.0 * r * N * K for r in rows)
    h2d = h_x.numel() * 2 + h_idx.numel() * 8
    return {"value": total * n / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "steps": n, "ms_per_step": ms / n,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": R * N * 2,
            "inputs": f"BF16 rows of the {U} distinct tokens this rank's expert rows use + the row -> token index",
            "step": "1x128 quantize -> fp8bs_expand_rows (gather) -> grouped Fprop; BF16 expert outputs downloaded",
            "bitwise_equal_device_step": same,
            "pipelined": "2 device buffer sets; H2D, compute and D2H streams overlap across steps (PCIe-bound)"}


def time_moe_forward(args, world, rank, dev, pb):
    """N > 1, context (not the headline): the expert layer's whole FP8 forward with the NVLink exchange
    (ep.moe_forward, NEXT-3): 1x128 quantization of the rank's tokens -> FP8 dispatch written into the
    expert owners' memory -> grouped Fprop -> BF16 combine written back -> gate-weighted sum.  CUDA events
    around each phase, max over ranks; dispatch / combine GB/s count the bytes that cross NVLink."""
    import torch.distributed as dist
    from paper_2412_19437_b200 import ep
    import paper_2412_19437_b200 as fp
    cfg = ep.EPConfig()
    routes = ep.routes_for(cfg)
    T, E, k, K, N = cfg.tokens, cfg.experts, cfg.top_k, cfg.hidden, cfg.inter
    plans = [ep.exchange_plan(routes, E, world, r, pb.placement) for r in range(world)]
    plan = ep.plan_to_device(plans[rank], dev)
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed + 100)
    x = torch.randn(T, K, generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    x_local = x[plan.t0:plan.t1].contiguous()
    del x
    gg = torch.rand(plan.t1 - plan.t0, k, generator=g, device=dev)
    gates = (gg / gg.sum(1, keepdim=True)).contiguous()
    ex = ep.Exchange(dist.group.WORLD, dev, max(p.rows for p in plans), max((p.t1 - p.t0) * k for p in plans), K, N)
    ws = torch.empty(int(fp.lib().fp8bs_grouped_gemm_workspace_size(max(len(plan.experts), 1), max(plan.rows, 1), N, K)) + 16,
                     dtype=torch.uint8, device=dev)
    steps = min(args.steps, 10)
    stream = torch.cuda.current_stream()

    def layer_ms(**kw):
        for _ in range(args.warmup):
            ep.moe_forward(ex, plan, x_local, gates, k, pb.Bq, pb.sB, ws=ws, **kw)
        torch.cuda.synchronize()
        barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            ep.moe_forward(ex, plan, x_local, gates, k, pb.Bq, pb.sB, ws=ws, **kw)
        b.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(a.elapsed_time(b) / steps, world, dev)
    ms_unfused = layer_ms(fused=False)
    ms_fused = layer_ms(fused=True, dedup=False)
    ms = layer_ms(dedup=True)
    keep = {}
    ref_out = ep.moe_forward(ex, plan, x_local, gates, k, pb.Bq, pb.sB, ws=ws, keep=keep, fused=False).clone()
    fused_out = ep.moe_forward(ex, plan, x_local, gates, k, pb.Bq, pb.sB, ws=ws, fused=True, dedup=False).clone()
    dedup_out = ep.moe_forward(ex, plan, x_local, gates, k, pb.Bq, pb.sB, ws=ws, dedup=True)
    torch.cuda.synchronize()
    fused_ok = gather_ints([int(torch.equal(fused_out.view(torch.int16), ref_out.view(torch.int16)) and
                                torch.equal(dedup_out.view(torch.int16), ref_out.view(torch.int16)))], world, dev)
    xq, xs, y = keep["xq"], keep["xs"], keep["y"]

    def phase(fn, iters=10):
        fn()
        ex.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_time(e1) / iters, world, dev)
    ms_d = phase(lambda: fp.dispatch_fp8(xq, xs, k, plan.dst_rank_dev, plan.dst_row_dev, ex.hq.buffer_ptrs_dev, K,
                                         ex.hs.buffer_ptrs_dev))
    ms_c = phase(lambda: fp.combine_push_bf16(y, plan.c_rank_dev, plan.c_slot_dev, ex.hy.buffer_ptrs_dev, N))
    remote_d = gather_ints([int((plan.dst_rank != rank).sum())], world, dev)
    remote_c = gather_ints([int((plan.c_rank != rank).sum())], world, dev)
    rows = gather_ints([plan.rows], world, dev)
    fl = sum(2.0 * r * N * K for r in rows)
    ex.barrier()
    torch.cuda.synchronize()
    return {"what": "whole expert-layer FP8 forward per rank: quantize tokens -> NVLink FP8 dispatch, each (token, rank) "
                    "pair once -> local expansion to expert rows -> grouped Fprop whose epilogue stores each BF16 row into "
                    "its token owner's combine buffer (fused combine send) -> gate-weighted sum (ep.moe_forward(dedup=True); "
                    "symmetric-memory barriers between)",
            "ms_per_step": ms, "steps": steps, "value": fl / (ms * 1e-3) / 1e12, "unit": "TFLOP/s (expert GEMM flop / step)",
            "ms_per_step_unfused": ms_unfused, "ms_per_step_fused_per_slot_dispatch": ms_fused,
            "fused_bitwise_equal_unfused_all_ranks": all(bool(v) for v in fused_ok),
            "dispatch_ms": ms_d, "dispatch_remote_GBps_per_rank": max(remote_d) * (K + 4 * (K // 128)) / (ms_d * 1e-3) / 1e9,
            "combine_ms": ms_c, "combine_remote_GBps_per_rank": max(remote_c) * N * 2 / (ms_c * 1e-3) / 1e9,
            "nvlink_reference_GBps_per_direction": 770}


# ------------------------------------------------------------------- CPU oracle ----
def c4_cpu_sample():
    """The C4 step on the CPU oracle, restricted to CPU_ROWS rows of every CPU_EXPERT_STRIDE-th expert
    (16 experts x 4 rows x N=2048 x K=7168): 1x128 quantization of those rows' tokens and the grouped
    FP64 oracle GEMM.  Expert weights (N(0, 0.006^2), CPU generator) are quantized by the oracle outside
    the timing, as the GPU path holds its quantized weights.  Returns (seconds, GEMM FLOP, description)."""
    import oracle
    from paper_2412_19437_b200 import ep
    cfg = ep.EPConfig()
    if not hasattr(c4_cpu_sample, "cache"):
        experts = list(range(0, cfg.experts, CPU_EXPERT_STRIDE))
        Bq, sB = [], []
        for e in experts:
            w = W.master_weight(cfg.inter, cfg.hidden, seed=cfg.seed + 1000 + e)
            q, s, _ = oracle.quantize_weight_128x128(w, want_t=False)
            Bq.append(q)
            sB.append(s)
        x = W.gaussian_act(len(experts) * CPU_ROWS, cfg.hidden, seed=0)
        off = torch.arange(0, len(experts) + 1, dtype=torch.int64) * CPU_ROWS
        c4_cpu_sample.cache = (x, off, torch.stack(Bq), torch.stack(sB), len(experts))
    x, off, Bq, sB, ne = c4_cpu_sample.cache
    t0 = time.perf_counter()
    q, s = oracle.quantize_act_1x128(x)
    oracle.grouped_gemm(off, q, s, Bq, sB)
    dt = time.perf_counter() - t0
    return dt, 2.0 * x.shape[0] * cfg.inter * cfg.hidden, (
        f"C4 step restricted to {CPU_ROWS} rows of each of {ne} experts (every {CPU_EXPERT_STRIDE}th): 1x128 quantize of "
        f"those {x.shape[0]} token rows + FP64 grouped oracle GEMM (N=2048, K=7168)")


def cpu_baseline_block(min_seconds=10.0):
    """Time the oracle on repeated C4 samples until at least min_seconds of CPU work."""
    import oracle
    c4_cpu_sample()   # build the cached sample (weights quantized by the oracle) outside the timing
    dt, fl, n = 0.0, 0.0, 0
    desc = ""
    while dt < min_seconds:
        d, f, desc = c4_cpu_sample()
        dt += d
        fl += f
        n += 1
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": oracle.max_threads(), "kind": "oracle",
            "sample": f"{desc}; {n} repetitions, {fl / 1e9:.2f} GFLOP in {dt:.2f} s"}


# ------------------------------------------------------------------------ main ----
_OUT_FD = None   # the process's original stdout: the JSON line goes there and nothing else does


def keep_stdout_for_the_line():
    """Route everything else written to stdout (C libraries included: NCCL prints its version banner at
    communicator init) to stderr, so that stdout carries exactly the one JSON line."""
    global _OUT_FD
    sys.stdout.flush()
    _OUT_FD = os.dup(1)
    os.dup2(2, 1)


def emit(line: dict):
    data = (json.dumps(line) + "\n").encode()
    if _OUT_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        while data:                      # os.write may write fewer bytes than asked
            data = data[os.write(_OUT_FD, data):]


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


def gather_ints(v, world, dev):
    if world == 1:
        return list(v)
    import torch.distributed as dist
    t = torch.tensor(v, dtype=torch.int64, device=dev)
    lst = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(lst, t)
    return [int(x) for l in lst for x in l.tolist()]


def gather_floats(v, world, dev):
    if world == 1:
        return list(v)
    import torch.distributed as dist
    t = torch.tensor(v, dtype=torch.float64, device=dev)
    lst = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(lst, t)
    return [float(x) for l in lst for x in l.tolist()]


def run_reference(args, world, rank):
    """--impl reference: the CPU oracle as it stands, on a bounded sample of the C4 step, rank 0 only."""
    if rank != 0:
        return
    # torchrun exports OMP_NUM_THREADS=1; rank 0 runs the oracle alone on the box's host cores
    torch.set_num_threads(len(os.sched_getaffinity(0)))   # the process's OpenMP pool (shared with the oracle)
    c4_cpu_sample()   # sample setup (weights quantized by the oracle) outside the timing
    for _ in range(args.warmup):
        c4_cpu_sample()
    t, f, desc = 0.0, 0.0, ""
    for _ in range(args.steps):
        d, fl, desc = c4_cpu_sample()
        t += d
        f += fl
    import oracle
    v = f / t / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": c4_config(world, args.placement) if args.workload == "c4" else {"workload": "C1"},
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": oracle.max_threads(), "kind": "oracle",
                             "sample": f"each step: {desc}"},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c4", "c1"])
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu", dest="cpu", action="store_false")
    ap.add_argument("--no-pow2", dest="pow2", action="store_false")
    ap.add_argument("--no-c1", dest="c1", action="store_false")
    ap.add_argument("--no-verify", dest="verify", action="store_false")
    ap.add_argument("--no-exchange", dest="exchange", action="store_false")
    ap.add_argument("--placement", default="balanced", choices=["balanced", "contiguous"],
                    help="C4 expert placement over ranks (balanced: observed-load LPT + one redundant expert per "
                         "rank at N > 1, P:584-589)")
    ap.add_argument("--redundant", type=int, default=None, help="redundant expert copies (default: one per rank)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    keep_stdout_for_the_line()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if args.workload == "c4":
        result, pb = time_c4(args, world, rank, dev)
        if world > 1 and args.exchange:
            result["c4_moe_forward"] = time_moe_forward(args, world, rank, dev, pb)
        del pb
        torch.cuda.empty_cache()
        if args.c1:
            result["c1_step"] = time_c1(args, world, rank, dev)
    else:
        c1 = time_c1(args, world, rank, dev, e2e=args.e2e)
        result = {"metric": METRIC, "value": c1.pop("value"), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                  "warmup": args.warmup, "ms_per_step": c1.pop("ms_per_step"), "higher_is_better": True,
                  "scaling": c1.pop("scaling"), "vs_baseline": None, "dtype": "e4m3", "data": "synthetic",
                  "config": {"workload": c1.pop("workload"), "tokens": T_TOK, "in": D_IN, "out": D_OUT,
                             "global_batch": T_TOK * world, "parallelism": c1.pop("parallelism"), "l2": c1.pop("l2")},
                  **c1}
    if rank == 0:
        if args.cpu and world == 1:
            result["cpu_baseline"] = cpu_baseline_block()
        emit(result)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
