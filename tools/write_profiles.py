"""Write the profiles/ summaries from a tools/capture_profiles.sh run (gpurun_out/ by default).

  python tools/write_profiles.py [capture_dir] [round_tag]
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from summarize_profiles import launch_table  # noqa: E402

METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,"
           "sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,"
           "launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active,"
           "smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,"
           "sm__cycles_elapsed.avg.per_second")
UNITS = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def full(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", METRICS],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        o = {"kernel": d["Kernel Name"].split("(")[0].replace("void ", "")}
        for k in hdr:
            if "__" in k and d.get(k):
                o[k] = (d[k] + " " + units[hdr.index(k)]).strip()
        out.append(o)
    return out


def dram_bytes(o):
    v, u = o["dram__bytes_read.sum"].split()
    w, uw = o["dram__bytes_write.sum"].split()
    return float(v) * UNITS[u] + float(w) * UNITS[uw]


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
    tag = sys.argv[2] if len(sys.argv) > 2 else "r01"
    dst = os.path.join(ROOT, "profiles")
    commit = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"],
                            capture_output=True, text=True).stdout.strip()
    hdr = f"# commit {commit}; tools/capture_profiles.sh on one B200 (ncu, --clock-control none)\n"
    for name in ("c2", "c2_warm", "c5"):  # gpurun_out/launch_<name>.csv -> <tag>_<name>_launches.csv
        shutil.copy(f"{src}/launch_{name}.csv", f"{dst}/{tag}_{name}_launches.csv")
    notes = {
        "c2": "C2 bench.py --steps 1 --warmup 3 (gpu__time_duration.sum per launch, caches flushed between launches)",
        "c2_warm": "C2 tools/prof_solve.py --iters 80, --cache-control none (L2 kept between launches: closer to the in-graph durations)",
        "c5": "C5 tools/prof_batch.py --iters 20 --solves 1 (setup kernels generate the 128 problems)",
    }
    for k, note in notes.items():
        with open(f"{dst}/{tag}_{k}_launch_summary.txt", "w") as f:
            f.write(hdr + f"# {note}\n" + launch_table(f"{dst}/{tag}_{k}_launches.csv") + "\n")
    c2, c5 = full(f"{src}/full_c2.ncu-rep"), full(f"{src}/full_c5.ncu-rep")
    with open(f"{dst}/{tag}_c2_ncu_full_summary.txt", "w") as f:
        f.write(hdr + "# ncu --set full --import-source on, C2 tools/prof_solve.py --iters 60, one launch of each iteration kernel (skip 200 matching launches)\n")
        for o in c2:
            f.write(json.dumps(o) + "\n")
    with open(f"{dst}/{tag}_ncu_full_summary.txt", "w") as f:
        f.write(hdr + "# ncu --set full, C5 tools/prof_batch.py --iters 5: DMMA products, batched finishes, batched projection\n")
        for o in c5:
            f.write(json.dumps(o) + "\n")

    def first(lst, prefix):
        return [o for o in lst if o["kernel"].startswith(prefix)][0]
    tr = {"C2_adj": dram_bytes(first(c2, "adj_kernel")),
          "C2_fwd_sparse": dram_bytes(first(c2, "fwd_sparse")),
          "C5_bfwd": dram_bytes(first(c5, "bfwd")),
          "C5_badj": dram_bytes(first(c5, "badj")),
          "note": f"dram__bytes_read.sum + dram__bytes_write.sum per launch from the {tag} full "
                  f"captures (commit {commit}); the sparse forward traffic follows the support of "
                  "d at the captured iteration"}
    with open(f"{dst}/traffic.json", "w") as f:
        json.dump(tr, f, indent=1)
    shutil.copy(f"{src}/timeline_c2.txt", f"{dst}/{tag}_c2_timeline.txt")
    shutil.copy(f"{src}/proj_phases_c2.txt", f"{dst}/{tag}_c2_proj_phases.txt")
    print(json.dumps(tr))


if __name__ == "__main__":
    main()
