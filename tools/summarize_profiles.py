"""Summarize a tools/gpu_bench_profile.sh run into profiles/<round>/ (tracked):
  bench.json      the bench line of that run
  ncu_launches.csv the raw ncu launch list (gpu__time_duration per launch, --clock-control none)
  ncu_summary.md  per-launch times of the last complete step (cold, serialised) next to the bench's
                  CUDA-event shares, and the --set full metrics of each kernel
  traffic.json    DRAM bytes per launch (read + write) keyed by the bench's launch names

    python tools/summarize_profiles.py <tag> [round_dir=profiles/r01]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
STEP = ["quant_act_dual(X)", "quant_weight_128x128(W)+T", "gemm_fprop", "quant_act_dual(dY)", "gemm_dgrad", "gemm_wgrad"]
GEMMS = ["gemm_fprop", "gemm_dgrad", "gemm_wgrad"]
QUANTS = ["quant_act_dual(X)", "quant_weight_128x128(W)+T", "quant_act_dual(dY)"]
METRICS = [
    ("gpu__time_duration.sum", "time (us)"),
    ("dram__bytes_read.sum", "DRAM read (MB)"),
    ("dram__bytes_write.sum", "DRAM write (MB)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active (%)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active (%)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (%)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (GHz)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def to_unit(v, unit, want):
    x = float(v)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3,
             "ms": 1e3, "Ghz": 1, "Mhz": 1e-3, "hz": 1e-9}
    if want == "MB":
        return x * scale.get(unit, 1) / 1e6
    if want == "us":
        return x * scale.get(unit, 1)
    if want == "GHz":
        return x * scale.get(unit, 1)
    return x


def main():
    tag = sys.argv[1]
    rdir = os.path.join(ROOT, sys.argv[2] if len(sys.argv) > 2 else "profiles/r01")
    os.makedirs(rdir, exist_ok=True)
    bench = json.loads(open(os.path.join(OUT, f"bench_{tag}.json")).read().strip().splitlines()[-1])
    json.dump(bench, open(os.path.join(rdir, "bench.json"), "w"), indent=1)
    # launch list: keep the last complete step (6 launches)
    raw = open(os.path.join(OUT, f"launches_{tag}.csv")).read()
    open(os.path.join(rdir, "ncu_launches.csv"), "w").write(raw)
    lines = [l for l in raw.splitlines() if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    times = [(r["Kernel Name"], float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1)) for r in rows
             if r["Metric Name"] == "gpu__time_duration.sum"]
    last = times[-len(STEP):]
    tot = sum(t for _, t in last)
    kb = bench["kernels"]
    ev_tot = sum(kb[n]["ms"] for n in STEP)
    md = [f"# Profiles ({tag}) — B200, gpurun, committed build", "",
          f"Bench line: `bench.json` ({bench['value']:.0f} {bench['unit']}, {bench['ms_per_step']:.3f} ms per step).", "",
          "## ncu launch list: last step of `bench.py --steps 2 --warmup 3` (gpu__time_duration, --clock-control none)", "",
          "| launch | kernel | ncu us (cold, serialised) | share of step (ncu) | share of step (bench CUDA events) |",
          "|---|---|---|---|---|"]
    for name, (k, t) in zip(STEP, last):
        md.append(f"| {name} | `{k[:60]}` | {t:.1f} | {100 * t / tot:.1f}% | {100 * kb[name]['ms'] / ev_tot:.1f}% |")
    traffic = {}
    for rep, names in ((f"prof_gemm_{tag}.ncu-rep", GEMMS), (f"prof_quant_{tag}.ncu-rep", QUANTS)):
        path = os.path.join(OUT, rep)
        if not os.path.exists(path):
            continue
        recs, units = ncu_raw(path)
        md += ["", f"## `ncu --set full` ({rep}; one launch each, step 4)", "",
               "| metric | " + " | ".join(names) + " |", "|---|" + "---|" * len(names)]
        for key, label in METRICS:
            vals = []
            for r in recs[:len(names)]:
                v = r.get(key, "")
                u = units.get(key, "")
                try:
                    if "MB" in label:
                        vals.append(f"{to_unit(v, u, 'MB'):.1f}")
                    elif "us" in label:
                        vals.append(f"{to_unit(v, u, 'us'):.1f}")
                    elif "GHz" in label:
                        vals.append(f"{to_unit(v, u, 'GHz'):.3f}")
                    else:
                        vals.append(f"{float(v):.1f}")
                except ValueError:
                    vals.append(v)
            md.append(f"| {label} | " + " | ".join(vals) + " |")
        for n, r in zip(names, recs):
            traffic[n] = to_unit(r["dram__bytes_read.sum"], units["dram__bytes_read.sum"], "MB") * 1e6 + \
                to_unit(r["dram__bytes_write.sum"], units["dram__bytes_write.sum"], "MB") * 1e6
    json.dump({"source": f"{os.path.relpath(rdir, ROOT)} ncu --set full --clock-control none ({tag}; one launch per kernel "
                         "of bench.py step 4)", "dram_bytes_per_launch": traffic},
              open(os.path.join(rdir, "traffic.json"), "w"), indent=1)
    open(os.path.join(rdir, "ncu_summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
