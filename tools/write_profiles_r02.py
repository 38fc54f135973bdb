"""Write the round-2 profiles/ files from a tools/evidence_r02.sh run (gpurun_out/).

  python tools/write_profiles_r02.py [capture_dir]
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from summarize_profiles import launch_table  # noqa: E402
from write_profiles import dram_bytes, full  # noqa: E402

TAG = "r02"


def last_json(path):
    lines = [ln for ln in open(path).read().splitlines() if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
    dst = os.path.join(ROOT, "profiles")
    commit = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"],
                            capture_output=True, text=True).stdout.strip()
    hdr = f"# commit {commit}; tools/evidence_r02.sh on one B200\n"
    for c in ("C1", "C2", "C3", "C4", "C5"):
        p = f"{src}/ev_bench_{c}.json"
        if os.path.exists(p) and last_json(p):
            with open(f"{dst}/{TAG}_bench_{c.lower()}.json", "w") as f:
                json.dump(last_json(p), f, indent=1)
    for name, note in [("phases_C2", "projection phases, C2, tools/prof_solve.py --profile"),
                       ("phases_C4", "projection phases, C4, tools/prof_solve.py --profile"),
                       ("timeline_C2", "in-graph kernel timeline (L1G_TIMELINE build), C2"),
                       ("timeline_C4", "in-graph kernel timeline (L1G_TIMELINE build), C4"),
                       ("crossover_C2", "forward density crossover, tools/fwd_crossover.py")]:
        p = f"{src}/ev_{name}.txt"
        if os.path.exists(p):
            with open(f"{dst}/{TAG}_{name.lower()}.txt", "w") as f:
                f.write(hdr + f"# {note}\n" + open(p).read())
    notes = {
        "c4": "C4 tools/prof_solve.py --iters 12 (bench default config; setup kernels generate K)",
        "c2": "C2 tools/prof_solve.py --iters 80",
        "c5": "C5 tools/prof_batch.py --iters 20 --solves 1 (setup kernels generate the 128 problems)",
    }
    for k, note in notes.items():
        p = f"{src}/launch_{k}.csv"
        if os.path.exists(p):
            shutil.copy(p, f"{dst}/{TAG}_{k}_launches.csv")
            with open(f"{dst}/{TAG}_{k}_launch_summary.txt", "w") as f:
                f.write(hdr + "# ncu --metrics gpu__time_duration.sum --clock-control none "
                        "(cold caches, serialised launches: compare shares)\n# " + note + "\n" +
                        launch_table(p) + "\n")
    tr = json.load(open(f"{dst}/traffic.json"))
    for k in ("c4", "c2", "c5"):
        p = f"{src}/full_{k}.ncu-rep"
        if not os.path.exists(p):
            continue
        rows = full(p)
        with open(f"{dst}/{TAG}_{k}_ncu_full_summary.txt", "w") as f:
            f.write(hdr + f"# ncu --set full --import-source on --clock-control none, {k.upper()}"
                    ": one launch of each hot kernel\n")
            for o in rows:
                f.write(json.dumps(o) + "\n")
        for o in rows:
            kn = o["kernel"].split("<")[0]
            key = {"adj_kernel": "adj", "fwd_sparse_kernel": "fwd_sparse", "fwd_kernel": "fwd",
                   "bfwd_wide_kernel": "bfwd", "badj_wide_kernel": "badj", "bfwd_kernel": "bfwd",
                   "badj_kernel": "badj", "bfwd_ws_kernel": "bfwd", "badj_ws_kernel": "badj"}.get(kn)
            if key:
                tr[f"{k.upper()}_{key}"] = dram_bytes(o)
                if key == "fwd_sparse":  # the bench's dominant-kernel key for the forward
                    tr[f"{k.upper()}_fwd"] = dram_bytes(o)
    tr["note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch from the {TAG} full "
                  f"captures (commit {commit}); the sparse forward traffic follows the support of "
                  "d at the captured iteration")
    with open(f"{dst}/traffic.json", "w") as f:
        json.dump(tr, f, indent=1)
    print(json.dumps(tr, indent=1))


if __name__ == "__main__":
    main()
