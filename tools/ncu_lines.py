"""Top source lines of one kernel by warp-stall samples, from an ncu report (--import-source).

  python tools/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows, fname, hdr, seen = [], None, None, False
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            if seen and hdr:  # only the first launch in the report
                pass
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0].isdigit() and len(r) > 4 and r[2] == "-":
            d = dict(zip(hdr[2:], r[2:]))
            stalls = {k: float(v) for k, v in zip(hdr, r) if k.startswith("stall_") and
                      "Not Issued" not in k and v not in ("", "-") and float(v) > 0}
            rows.append((float(r[4] or 0), fname, int(r[0]), r[1].strip()[:90], stalls,
                         d.get("Instructions Executed", "")))
    tot = sum(x[0] for x in rows) or 1.0
    rows.sort(key=lambda x: -x[0])
    print(f"total samples {tot:.0f}")
    for s, f, ln, src, st, ie in rows[:top]:
        ss = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"{s / tot:6.1%} {f}:{ln:<5} {src:<90} " +
              " ".join(f"{k[6:]}={v:.0f}" for k, v in ss))


if __name__ == "__main__":
    main()
