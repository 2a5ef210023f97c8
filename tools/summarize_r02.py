"""Summarize a tools/gpu_bench_profile.sh run (round 2 layout) into profiles/<round>/ (tracked):
  bench.json               the default bench line of that run (C4 headline + c1_step)
  ncu_launches_c4.csv      raw ncu launch list of the C4 step (gpu__time_duration, --clock-control none)
  ncu_launches_c1.csv      raw ncu launch list of the C1 step
  ncu_summary.md           per-launch shares (ncu vs the bench's CUDA events) and --set full metrics
  traffic.json             DRAM bytes per launch keyed by the bench's launch names
  sass_histogram.md        tcgen05 / TMA / packed-FP32 instruction counts per kernel (cuobjdump -sass)

    python tools/summarize_r02.py <tag> [round_dir=profiles/r02]
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
C1 = ["quant_act_dual(X)", "quant_weight_128x128(W)+T", "gemm_fprop", "quant_act_dual(dY)", "gemm_dgrad",
      "gemm_dgrad (split-K tail)", "gemm_dgrad (split-K reduce)", "gemm_wgrad"]
C1_GEMMS = ["gemm_fprop", "gemm_dgrad", "gemm_dgrad (split-K tail)", "gemm_dgrad (split-K reduce)", "gemm_wgrad"]
C4 = ["quant_act_1x128(X shard)", "k_grouped_schedule", "grouped_gemm_fprop"]
METRICS = [
    ("gpu__time_duration.sum", "time (us)", "us"),
    ("dram__bytes_read.sum", "DRAM read (MB)", "MB"),
    ("dram__bytes_write.sum", "DRAM write (MB)", "MB"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active (%)", ""),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active (%)", ""),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (%)", ""),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate (%)", ""),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (GHz)", "GHz"),
    ("launch__registers_per_thread", "registers/thread", ""),
    ("launch__grid_size", "grid", ""),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-3, "usecond": 1, "us": 1,
         "msecond": 1e3, "ms": 1e3, "Ghz": 1, "Mhz": 1e-3, "hz": 1e-9}


def conv(v, unit, want):
    x = float(v)
    if want == "MB":
        return x * SCALE.get(unit, 1) / 1e6
    if want in ("us", "GHz"):
        return x * SCALE.get(unit, 1)
    return x


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def launch_times(path):
    raw = open(path).read()
    lines = [l for l in raw.splitlines() if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    return raw, [(r["Kernel Name"], float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1)) for r in rows
                 if r["Metric Name"] == "gpu__time_duration.sum"]


def metrics_table(md, title, recs, units, names):
    md += ["", f"## {title}", "", "| metric | " + " | ".join(names) + " |", "|---|" + "---|" * len(names)]
    for key, label, want in METRICS:
        vals = []
        for r in recs[:len(names)]:
            try:
                v = conv(r.get(key, ""), units.get(key, ""), want)
                vals.append(f"{v:.3f}" if want == "GHz" else f"{v:.1f}")
            except ValueError:
                vals.append(r.get(key, ""))
        md.append(f"| {label} | " + " | ".join(vals) + " |")


def sass_histogram():
    lib = os.path.join(ROOT, "paper_2412_19437_b200", "libfp8bs.so")
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    pats = ["UTCQMMA", "UTCMMA", "UTCBAR", "UTCCP", "LDTM", "UTMALDG", "UTMASTG", "UTMAREDG", "UBLKCP", "FFMA2",
            "FMUL2", "FADD2", "F2FP.SATFINITE.E4M3", "SYNCS", "ELECT", "STL", "LDL"]
    counts = collections.OrderedDict()
    fn = None
    for l in out.splitlines():
        m = re.search(r"Function : (\S+)", l)
        if m:
            fn = m.group(1)
            counts[fn] = collections.Counter()
            continue
        if fn and re.search(r"/\*[0-9a-f]{4,}\*/", l):
            ins = l.split("*/", 1)[1].strip().split(" ;")[0]
            op = ins.split()[0] if not ins.startswith("@") else ins.split()[1]
            for p in pats:
                if op.startswith(p):
                    counts[fn][p] += 1
                    break
    md = ["# SASS instruction histogram of libfp8bs.so (cuobjdump -sass, static counts)", "",
          "Evidence that the GEMMs issue tcgen05 MMAs (`UTCQMMA*`: kind::f8f6f4 / mxf8f6f4), read TMEM "
          "(`LDTM`), move tiles with TMA (`UTMALDG` / `UTMASTG` / `UTMAREDG`), and promote with packed FP32 "
          "(`FFMA2` / `FMUL2`); `STL`/`LDL` are register spills.", "",
          "| kernel | " + " | ".join(pats) + " |", "|---|" + "---|" * len(pats)]
    def pretty(f):
        m = re.search(r"k_gemm_bsILb(\d)ELi(\d)ELb(\d)ELb(\d)E", f)
        if m:
            w, o, g, pr = m.groups()
            return (f"k_gemm_bs<{'wgrad' if w == '1' else 'fprop/dgrad'}, "
                    f"{['bf16', 'fp32', 'swiglu-fp8', 'split-K fp32 partial', 'scatter bf16'][int(o)]} out, "
                    f"{'grouped' if g == '1' else 'dense'}, {'cta pair' if pr == '1' else '1 cta'}>")
        m = re.search(r"k_gemm_mxILb(\d)ELb(\d)ELb(\d)E", f)
        if m:
            return f"k_gemm_mx<{m.group(1)},{m.group(2)},{m.group(3)}>"
        m = re.search(r"\d+(k_[a-z0-9_]+?)(I|E|P|v|$)", f)
        return (m.group(1) if m else f)[:60]
    for f, c in counts.items():
        short = pretty(f)
        md.append(f"| `{short}` | " + " | ".join(str(c.get(p, 0)) for p in pats) + " |")
    return "\n".join(md) + "\n"


def main():
    tag = sys.argv[1]
    rdir = os.path.join(ROOT, sys.argv[2] if len(sys.argv) > 2 else "profiles/r02")
    os.makedirs(rdir, exist_ok=True)
    bench = json.loads(open(os.path.join(OUT, f"bench_{tag}.json")).read().strip().splitlines()[-1])
    json.dump(bench, open(os.path.join(rdir, "bench.json"), "w"), indent=1)
    md = [f"# Profiles ({tag}) — B200 via gpurun, the committed build", "",
          f"Bench line: `bench.json` — C4 {bench['value']:.0f} {bench['unit']} ({bench['ms_per_step']:.3f} ms per step, "
          f"grouped GEMM {bench['roofline']['achieved']:.0f} TFLOP/s = {bench['roofline']['frac']:.3f} of "
          f"{bench['roofline']['peak']}); clocks {bench['clocks']}."]
    traffic = {}
    for name, steps, kb in (("c4", C4, bench["kernels"]), ("c1", C1, bench.get("c1_step", {}).get("kernels", {}))):
        path = os.path.join(OUT, f"launches_{name}_{tag}.csv")
        if not os.path.exists(path):
            continue
        raw, times = launch_times(path)
        open(os.path.join(rdir, f"ncu_launches_{name}.csv"), "w").write(raw)
        last = times[-len(steps):]
        tot = sum(t for _, t in last)
        ev = {n: kb[n]["ms"] for n in steps if n in kb}
        ev_tot = sum(ev.values())
        md += ["", f"## ncu launch list, {name.upper()}: the last step (gpu__time_duration, --clock-control none)", "",
               "| launch | kernel | ncu us (cold, serialised) | share (ncu) | share (bench CUDA events) |", "|---|---|---|---|---|"]
        for n, (k, t) in zip(steps, last):
            share = f"{100 * ev[n] / ev_tot:.1f}%" if n in ev and ev_tot else "(inside the GEMM call's events)"
            md.append(f"| {n} | `{k[:70]}` | {t:.1f} | {100 * t / tot:.1f}% | {share} |")
    for rep, names, title in ((f"prof_grouped_{tag}.ncu-rep", ["grouped_gemm_fprop"], "C4 grouped GEMM, `ncu --set full` (one launch)"),
                              (f"prof_gemm_{tag}.ncu-rep", C1_GEMMS, "C1 GEMMs, `ncu --set full`"),
                              (f"prof_quant_{tag}.ncu-rep", ["quant_act_dual(X)", "quant_weight_128x128(W)+T", "quant_act_dual(dY)"],
                               "C1 quantizers, `ncu --set full`")):
        path = os.path.join(OUT, rep)
        if not os.path.exists(path):
            continue
        recs, units = ncu_raw(path)
        metrics_table(md, title, recs, units, names)
        for n, r in zip(names, recs):
            traffic[n] = conv(r["dram__bytes_read.sum"], units["dram__bytes_read.sum"], "MB") * 1e6 + \
                conv(r["dram__bytes_write.sum"], units["dram__bytes_write.sum"], "MB") * 1e6
    json.dump({"source": f"{os.path.relpath(rdir, ROOT)} ncu --set full --clock-control none ({tag}; one launch per kernel)",
               "dram_bytes_per_launch": traffic}, open(os.path.join(rdir, "traffic.json"), "w"), indent=1)
    open(os.path.join(rdir, "ncu_summary.md"), "w").write("\n".join(md) + "\n")
    open(os.path.join(rdir, "sass_histogram.md"), "w").write(sass_histogram())
    print("\n".join(md))


if __name__ == "__main__":
    main()
