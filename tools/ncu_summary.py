"""Summarise an ncu --set full report: duration, issue/pipe utilisation,
stall reasons, DRAM traffic, registers/occupancy (reads gpurun_out/*.ncu-rep)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg.per_second", "smsp__cycles_active.avg"]


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {k: (x, uu) for k, uu, x in zip(h, u, v)}
    res = {"kernel": d.get("Kernel Name", ("?",))[0]}
    for k in KEYS:
        if k in d:
            res[k] = d[k][0] + " " + d[k][1]
    # every FP64 / XU (MUFU) pipe counter the capture holds: the ratio of
    # pipe cycles to instructions says what one FP64 instruction costs
    for k, (x, uu) in d.items():
        if ("fp64" in k or "pipe_xu" in k) and (k.endswith(".sum") or "pct_of_peak" in k) and k not in res:
            res[k] = x + " " + uu
    stalls = {}
    for k, (x, _) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                if float(x) > 0.03:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(x)
            except ValueError:
                pass
    res["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        r = summary(p)
        print(p)
        for k, v in r.items():
            print("  ", k, "=", v)
