"""Condense `ncu --set full` reports into the JSON kept under profiles/.

    python tools/ncu_summary.py OUT.json name=report.ncu-rep [name=report.ncu-rep ...]
    python tools/ncu_summary.py OUT.json name=report.raw.csv ...      (the `ncu -i rep --page raw --csv` export)

For every report the first captured kernel's headline metrics are kept: duration, launch shape, registers,
pipe utilisation (the integer multiplier lives on the "fmaheavy" pipe), issue activity, warp-stall mix,
instruction-cache hit rate, shared-memory and DRAM traffic.  Runs here (no GPU needed): ncu only reads the file.
"""
import csv
import io
import json
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__icc_request_hit_rate.pct",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
]


def summarise(report: str) -> dict:
    if report.endswith(".csv"):
        text = open(report).read()
    else:
        text = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                              check=True).stdout
    rows = [r for r in csv.reader(io.StringIO(text)) if len(r) > 10]
    head, units, first = rows[0], rows[1], rows[2]
    out = {}
    for h, u, v in zip(head, units, first):
        if h == "Kernel Name" or h in KEEP:
            out[h] = {"unit": u, "value": v}
    out["kernels_in_report"] = len(rows) - 2
    return out


def main():
    dest, pairs = sys.argv[1], sys.argv[2:]
    result = {}
    for pair in pairs:
        name, path = pair.split("=", 1)
        result[name] = summarise(path)
    with open(dest, "w") as fh:
        json.dump(result, fh, indent=1)
    for name, s in result.items():
        print(name, s.get("Kernel Name", {}).get("value"), s.get("gpu__time_duration.sum", {}).get("value"), "ms",
              "fmaheavy", s.get("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", {}).get("value"))


if __name__ == "__main__":
    main()
