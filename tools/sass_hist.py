"""Per-kernel SASS instruction histogram of libl1g.so (cuobjdump -sass; no GPU needed).

  python tools/sass_hist.py [lib] > profiles/r02_sass_histogram.txt

Shows which data-movement and math units each hot kernel uses: UBLKCP (cp.async.bulk, the TMA
bulk-copy engine), SYNCS (mbarrier waits/arrives), LDGSTS (cp.async), DMMA (FP64 tensor core
mma.sync), DFMA / DMUL / DADD (FP64 pipe), LDG / STG / LDS / STS, and the cluster/DSMEM ops.
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UBLKCP", "UTMALDG", "SYNCS", "LDGSTS", "DMMA", "DFMA", "DMUL", "DADD", "LDG", "STG",
        "LDS", "STS", "LD", "ST", "ATOMS", "ATOM", "RED", "ATOMG", "UCGABAR", "CCTL", "MEMBAR", "BAR",
        "SHFL", "ACQBULK", "ELECT"]
HOT = ["adj_kernel", "fwd_kernel", "fwd_sparse_kernel", "fwd_finish_kernel", "adj_finish_kernel",
       "proj_kernel", "bfwd_kernel", "badj_kernel", "bfwd_wide_kernel", "badj_wide_kernel",
       "bfin_fwd_kernel", "bfin_adj_kernel", "brupdate_kernel"]


def demangle(name):
    out = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    return re.sub(r"\(.*\)$", "", out).replace("l1g::", "").replace("void ", "")


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_0902_4424_b200", "libl1g.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = demangle(m.group(1))
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if cur and m:
            op = m.group(1)
            op = "UCGABAR" if op.startswith("UCGABAR") else op  # _ARV / _WAIT: cluster barrier
            funcs[cur][op] += 1
            funcs[cur]["_total"] += 1
    commit = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"],
                            capture_output=True, text=True).stdout.strip()
    print(f"# cuobjdump -sass {os.path.relpath(lib, ROOT)} (commit {commit}, sm_100a); static "
          "instruction counts per kernel")
    print("# UBLKCP = cp.async.bulk (TMA bulk copy), SYNCS = mbarrier ops, LDGSTS = cp.async, "
          "DMMA = FP64 tensor-core MMA (mma.sync.m8n8k4.f64); no tcgen05 (sm_100a has no f64 kind)")
    cols = ["_total"] + KEYS
    print("kernel".ljust(34) + "".join(c.replace("_total", "total").rjust(8) for c in cols))
    for f, c in funcs.items():
        if not any(f.startswith(h) for h in HOT):
            continue
        print(f[:34].ljust(34) + "".join(str(c.get(k, 0)).rjust(8) for k in cols))


if __name__ == "__main__":
    main()
