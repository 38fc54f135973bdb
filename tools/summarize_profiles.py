"""Summaries of the ncu captures (tools/capture_profiles.sh) for profiles/."""
import collections
import csv
import json
import subprocess
import sys


def launch_table(path, skip_setup=True):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in data:
        k = r[ki].split("(")[0].replace("void ", "")
        agg.setdefault(k, []).append(float(r[vi].replace(",", "")))
    out = []
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k:45s} launches={len(v):5d} mean={sum(v)/len(v)/1e3:9.2f} us "
                   f"total={sum(v)/1e6:9.3f} ms share={sum(v)/tot:6.1%}")
    return "\n".join(out)


def full_metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                          "sm__throughput.avg.pct_of_peak_sustained_elapsed,"
                          "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,"
                          "launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,"
                          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,"
                          "sm__inst_executed_pipe_fp64.sum,smsp__inst_executed_op_dmma.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append(d)
    return res


if __name__ == "__main__":
    print(launch_table(sys.argv[1]))
