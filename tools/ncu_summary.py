"""Summaries of `ncu --page raw --csv` exports for profiles/: python tools/ncu_summary.py OUT.json
SOURCE_NOTE CSV [CSV ...] -> {"_source": ..., "kernels": {name: {metric: "value unit"}}} (first
launch of each CSV; the CSV file stem names the entry), plus the C5 traffic figure when asked."""
import csv
import json
import os
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]


def rows_of(path):
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = r[i][:60] if k == "Kernel Name" else f"{r[i]} {u[i]}".strip()
        out.append(d)
    return out


if __name__ == "__main__":
    out_path, note, csvs = sys.argv[1], sys.argv[2], sys.argv[3:]
    res = {"_source": note, "kernels": {}}
    for p in csvs:
        stem = os.path.splitext(os.path.basename(p))[0]
        launches = rows_of(p)
        if len(launches) == 1:
            res["kernels"][stem] = launches[0]
        else:
            for i, d in enumerate(launches):
                res["kernels"][f"{stem}#{i}"] = d
    json.dump(res, open(out_path, "w"), indent=1)
    for k, d in res["kernels"].items():
        print(k, d.get("gpu__time_duration.sum"), d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum"),
              "dmma", d.get("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"))
