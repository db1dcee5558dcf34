"""Key metrics of ncu --set full reports -> JSON (profiles/).

    python tools/ncu_summary.py out.json name=report.ncu-rep [name=raw.csv ...]

The first argument is the OUTPUT file.  Inputs are reports, or the `--page raw --csv` export of
one (written on the GPU box, where the reports are too big to bring back).  Refuses to overwrite
an input."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "Cluster Size", "gpu__time_duration.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum"]


def summarize(rep):
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            d[k] = (vals[i] + (" " + units[i] if units[i] else "")).strip()
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                v = float(vals[i])
            except ValueError:
                continue
            if v >= 0.2:
                d["stall:" + k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
    return d


if __name__ == "__main__":
    if not sys.argv[1].endswith(".json") or "=" in sys.argv[1]:
        sys.exit("usage: ncu_summary.py out.json name=report [...] (the first argument is the output)")
    res = {}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        res[name] = summarize(rep)
    with open(sys.argv[1], "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1)[:3000])
