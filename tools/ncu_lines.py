"""Instructions executed and stall samples aggregated per CUDA source line.
Usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> [n_top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
fname, hdr = None, None
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iI, iS = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].strip().isdigit():
        continue
    try:
        ie, ss = float(r[iI] or 0), float(r[iS] or 0)
    except ValueError:
        continue
    a = agg[(fname, int(r[0]))]
    a[0] += ie
    a[1] += ss
    a[2] = r[1].strip()[:80]
tot = sum(v[0] for v in agg.values()) or 1.0
tots = sum(v[1] for v in agg.values()) or 1.0
print(f"total warp instructions {tot:.0f}, stall samples {tots:.0f}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:ntop]:
    print(f"{v[0] / tot * 100:5.1f}% instr {v[1] / tots * 100:5.1f}% stall  {k[0]}:{k[1]}  {v[2]}")
