"""Key counters of one kernel in an ncu --set full report (the numbers the
profiles/*.txt summaries quote): duration, occupancy, FP64 pipe, issue,
DRAM bytes, shared-memory bank conflicts, stall reasons per issued
instruction.  Usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.per_cycle_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        if pat and not pat.search(name):
            continue
        print(f"Kernel Name  {name}")
        for k in KEYS:
            if k in col:
                print(f"{k:72s} {units[col[k]]:>14s} {r[col[k]]}")
        print("# warp stall reasons (cycles per issued instruction)")
        for k in sorted(col):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[col[k]])
                except ValueError:
                    continue
                if v >= 0.05:
                    print(f"{k:88s} {v:.3f}")
        print()


if __name__ == "__main__":
    main()
