"""Per-instruction stall summary from an ncu --set full report (source page, SASS).

  python scripts/ncu_source.py <report.ncu-rep> [top]
Prints the instructions with the most warp-stall samples, with their stall breakdown.
"""
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    h = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(h)]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    i_src = h.index("Source")
    i_ex = h.index("Instructions Executed")
    stall_cols = [i for i, k in enumerate(h) if k.startswith("stall_") or k.endswith("(Stall)") ]
    seen = set()
    uniq = []
    for r in data:
        if r[0] in seen:
            continue
        seen.add(r[0])
        uniq.append(r)
    num = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0
    tot = sum(num(r[i_s]) for r in uniq)
    print(f"total stall samples {tot:.0f}, {len(uniq)} SASS instructions")
    for r in sorted(uniq, key=lambda r: -num(r[i_s]))[:top]:
        extra = ""
        if stall_cols:
            parts = sorted(((num(r[i]), h[i]) for i in stall_cols), reverse=True)[:3]
            extra = "  " + ", ".join(f"{k}={v:.0f}" for v, k in parts if v > 0)
        print(f"{r[0][-6:]} {num(r[i_s]) / tot * 100:5.1f}% ex={r[i_ex]:>9s}  {r[i_src].strip()[:70]}{extra}")


if __name__ == "__main__":
    main()
