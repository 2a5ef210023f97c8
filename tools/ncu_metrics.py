"""Print the key --set full metrics of every kernel in an .ncu-rep (read here, after gpurun):
    python tools/ncu_metrics.py gpurun_out/<file>.ncu-rep [extra_metric_substring ...]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_ltcfabric.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "smsp__sass_inst_executed_op_local_ld.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size"]


def main():
    rep = sys.argv[1]
    extra = sys.argv[2:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print("==", d.get("Kernel Name", "?")[:90])
        for i, h in enumerate(hdr):
            if h in KEYS or any(e in h for e in extra):
                print(f"  {h:70s} {d[h]:>16s} {units[i]}")


if __name__ == "__main__":
    main()
