"""Summaries of ncu output for profiles/.

  python scripts/ncu_summary.py launches <launches.csv> [steps]
      per-kernel launch count, total and mean device time, share of all launches
      (cold-cache, serialised: compare SHARES, not absolute times)
  python scripts/ncu_summary.py full <report.ncu-rep>
      key counters of every profiled launch in a --set full report
  python scripts/ncu_summary.py traffic <report.ncu-rep> <config> profiles/ncu_traffic.json
      dram read+write bytes per launch of the captured kernel (bench.py roofline.traffic)
"""
import csv
import collections
import io
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.avg.per_cycle_active",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tcgen05_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__average_warp_latency_issue_stalled_barrier",
]


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)          # drop the parameter list
    name = name.replace("void ", "").replace("snn::<unnamed>::", "")
    return name.strip()


def launches(path: str, steps: int = 0):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    agg = collections.OrderedDict()
    for r in rows:
        if r[12] != "gpu__time_duration.sum":
            continue
        k = short(r[4])
        ns = float(r[14].replace(",", ""))
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + ns)
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':64s} {'launches':>8s} {'total_us':>10s} {'mean_us':>10s} {'share':>7s}")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:64]:64s} {c:8d} {t / 1e3:10.1f} {t / c / 1e3:10.2f} {100 * t / tot:6.1f}%")
    print(f"{'TOTAL':64s} {sum(c for c, _ in agg.values()):8d} {tot / 1e3:10.1f}")


def full(path: str):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"== {short(d.get('Kernel Name', '?'))}  grid {d.get('Grid Size')} block {d.get('Block Size')}")
        for k in KEYS:
            if k in d and d[k] != "":
                print(f"   {k:80s} {d[k]:>16s} {units[hdr.index(k)]}")


def traffic(path: str, config: str, out_json: str):
    """Record dram read+write bytes per launch (mean over the captured launches) of the
    dominant kernel for bench.py's roofline.traffic."""
    import json
    import os
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    vals, name = [], None
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(d[k].replace(",", "")) * scale[units[hdr.index(k)]]
        vals.append(b)
        name = short(d.get("Kernel Name", "?"))
    db = json.load(open(out_json)) if os.path.exists(out_json) else {}
    db[config] = {"kernel": name, "dominant_kernel_dram_bytes_per_launch": sum(vals) / len(vals),
                  "launches_captured": len(vals), "source": os.path.basename(path)}
    json.dump(db, open(out_json, "w"), indent=1)
    print(config, db[config])


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)
    else:
        full(sys.argv[2])
