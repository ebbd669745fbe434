#!/usr/bin/env python
"""Summarise ncu outputs into markdown for profiles/.

  ncu_summary.py launches <launches.csv> <steps_in_run>   per-kernel share of one step
  ncu_summary.py full <report.ncu-rep>                     key --set full metrics per launch
"""
import collections
import csv
import subprocess
import sys


def launches(path, steps):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    data = [dict(zip(hdr, r)) for r in rows[start + 1:] if len(r) == len(hdr)]
    # the timed steps are the last `steps` of (warmup + steps) identical steps; report per step averages
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches (all steps) | total ms | share |")
    print("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print("| `%s` | %d | %.3f | %.1f%% |" % (k[:70], v[0], v[1] / 1e6, 100 * v[1] / tot))
    print("\nTotal device time of all %d launches: %.3f ms (cold-cache, serialised)." % (len(data), tot / 1e6))


def full(path):
    metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
               "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__inst_executed.sum",
               "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
               "launch__registers_per_thread", "lts__t_sector_hit_rate.pct",
               "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    units = r[1]
    idx = [h.index("Kernel Name")] + [h.index(m) for m in metrics if m in h]
    print("| " + " | ".join(h[i] + (" (%s)" % units[i] if units[i] else "") for i in idx) + " | sectors/req |")
    print("|" + "---|" * (len(idx) + 1))
    for row in r[2:]:
        vals = [row[i] for i in idx]
        try:
            spr = float(row[h.index("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")].replace(",", "")) / max(
                1.0, float(row[h.index("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")].replace(",", "")))
        except Exception:
            spr = float("nan")
        vals[0] = "`" + vals[0].split("(")[0][:48] + "`"
        print("| " + " | ".join(vals) + " | %.2f |" % spr)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 1)
    else:
        full(sys.argv[2])
