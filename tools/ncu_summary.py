"""Summarize ncu outputs into markdown for profiles/.

  python tools/ncu_summary.py launches <launches.csv>        # per-kernel share of the step
  python tools/ncu_summary.py full <report.ncu-rep>          # key metrics per captured launch
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1tex %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "long-scoreboard stall/issue"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
              "msecond": 1e3}.get(unit, 1.0)
        name = d["Kernel Name"].split("(")[0].replace("void ", "").strip()
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total ms | mean us | share |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {t / 1e3:.3f} | {t / n:.1f} | {t / tot:.1%} |")
    out.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot / 1e3:.3f} | | |")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {m: hdr.index(m) for m, _ in FULL_METRICS if m in hdr}
    kn = hdr.index("Kernel Name")
    out = ["| kernel | " + " | ".join(lbl for m, lbl in FULL_METRICS if m in idx) + " |",
           "|---" * (1 + len(idx)) + "|"]
    for r in rows[2:]:
        name = r[kn].split("(")[0].replace("void ", "")
        vals = []
        for m, _ in FULL_METRICS:
            if m in idx:
                vals.append(f"{r[idx[m]]} {units[idx[m]]}".strip())
        out.append(f"| `{name}` | " + " | ".join(vals) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else full(path))
