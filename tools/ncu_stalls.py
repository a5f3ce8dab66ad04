"""Per-kernel metrics + top stalled SASS instructions from an ncu report.
Usage: python tools/ncu_stalls.py <report.ncu-rep> [kernel-regex] [n_top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 25
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size"]


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(run("--page", "raw", "--csv", "-k", "regex:" + kre))))
hdr, units = rows[0], rows[1]
for d in rows[2:]:
    print("==", d[hdr.index("Kernel Name")][:80])
    for w in WANT:
        if w in hdr:
            print(f"  {w:60s} {d[hdr.index(w)]} {units[hdr.index(w)]}")
    st = [(h[len("smsp__average_warps_issue_stalled_"):], float(d[i] or 0))
          for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
          and h.endswith("_per_issue_active.ratio")]
    for k, v in sorted(st, key=lambda x: -x[1])[:6]:
        print(f"    stall {k:50s} {v:.2f}")
rows = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "-k", "regex:" + kre))))
his = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
for n, hi in enumerate(his):
    hdr = rows[hi]
    end = his[n + 1] - 1 if n + 1 < len(his) else len(rows)
    data = [r for r in rows[hi + 1:end] if len(r) == len(hdr)]
    iS, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    tot = sum(f(r[iS]) for r in data) or 1.0
    print(f"-- top stalled instructions ({tot:.0f} samples)")
    idx = sorted(range(len(data)), key=lambda i: -f(data[i][iS]))[:ntop]
    for i in idx:
        r = data[i]
        prev = " | ".join(data[j][iSrc].strip()[:40] for j in range(max(0, i - 2), i))
        print(f"  {f(r[iS]) / tot * 100:5.1f}% {r[0][-5:]} {r[iSrc].strip()[:60]:60s}  <- {prev}")
