"""Per-CUDA-source-line summary of an ncu --set full report (needs -lineinfo + --import-source on).

  python scripts/ncu_lines.py <report.ncu-rep> [top]
Aggregates the SASS rows of the interleaved cuda,sass source view by source line and prints
the lines with the most warp instructions executed and the most stall samples.
"""
import collections
import csv
import io
import os
import subprocess
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    num = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0
    ex = collections.Counter()
    st = collections.Counter()
    text = {}
    fname, line, h = "?", "?", None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            h = r
            i_ex = h.index("Instructions Executed")
            i_s = h.index("Warp Stall Sampling (All Samples)")
            continue
        if h is None or len(r) != len(h):
            continue
        if r[0]:
            line = r[0]
            text[(fname, line)] = r[1]
        if r[2] and r[2] != "...":
            ex[(fname, line)] += num(r[i_ex])
            st[(fname, line)] += num(r[i_s])
    tex, ts = sum(ex.values()), sum(st.values())
    print(f"total warp instructions executed {tex:.4g}, stall samples {ts:.0f}")
    for title, c in (("instructions executed", ex), ("stall samples", st)):
        print(f"-- by {title}")
        for k, _ in c.most_common(top):
            print(f"{k[0]}:{k[1]:>5s} {ex[k] / tex * 100:5.1f}% ex {st[k] / ts * 100:5.1f}% st  {text.get(k, '').strip()[:80]}")


if __name__ == "__main__":
    main()
