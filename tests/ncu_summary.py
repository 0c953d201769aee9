"""Summarise ncu --set full reports (one launch each) into the text format of
profiles/r01_ncu_kernels.txt:  python tests/ncu_summary.py name=path.ncu-rep ...
Not collected by pytest (runs where ncu is installed)."""
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "dram__bytes_read.sum",
    "dram__bytes_write.sum",
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main():
    print("# ncu --set full --clock-control none --import-source on, one mid-solve launch per kernel")
    print("# command: ncu --profile-from-start off --set full --import-source on --clock-control "
          "none -k regex:<kernel> [-s 20] -c 1 -o ... python tests/profile_solve.py  (C3; "
          "k_correlate: tests/profile_plugin.py, the BenchWorkload plugin pass)")
    for arg in sys.argv[1:]:
        name, path = arg.split("=", 1)
        try:
            hdr, units, vals = raw(path)
        except (subprocess.CalledProcessError, IndexError, FileNotFoundError):
            print(f"== {name}\n  (no report at {path})")
            continue
        col = {h: i for i, h in enumerate(hdr)}
        print(f"== {name}")
        for m in METRICS:
            if m in col:
                print(f"{m:75s} {units[col[m]]:12s} {vals[col[m]]}")
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    v = float(vals[i])
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        for v, h in sorted(stalls, reverse=True):
            print(f"  stall {h:60s} {v:.6f}")


if __name__ == "__main__":
    main()
