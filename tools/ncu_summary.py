"""Summarise an ncu report (details + raw) into markdown for profiles/ (run here, no GPU needed)."""
import csv
import subprocess
import sys

KEYS_DETAILS = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
                "Achieved Occupancy", "Registers Per Thread", "Executed Instructions", "L1/TEX Hit Rate",
                "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
                "Eligible Warps Per Scheduler", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
                "Static Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio"]


def run(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", "--print-kernel-base", "function"],
                         capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def main(rep):
    det = run(rep, "details")
    h = det[0]
    per = {}
    for row in det[1:]:
        d = dict(zip(h, row))
        k = (d["ID"], d["Kernel Name"])
        if d["Metric Name"] in KEYS_DETAILS:
            per.setdefault(k, {})[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    raw = run(rep, "raw")
    rh = raw[0]
    units = dict(zip(rh, raw[1]))
    rawv = {}
    for row in raw[2:]:
        d = dict(zip(rh, row))
        rawv[(d["ID"], d["Kernel Name"])] = {k: (f"{d[k]} {units.get(k, '')}".strip() if d.get(k) is not None
                                                 else None) for k in RAW}
    print(f"# ncu summary of `{rep}`\n")
    for k in sorted(per):
        print(f"## launch {k[0]}: `{k[1]}`\n")
        print("| metric | value |\n|---|---|")
        for m in KEYS_DETAILS:
            if m in per[k]:
                print(f"| {m} | {per[k][m]} |")
        for m, v in rawv.get(k, {}).items():
            if v is not None:
                print(f"| {m} | {v} |")
        print()


if __name__ == "__main__":
    main(sys.argv[1])
