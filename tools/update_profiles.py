"""Copy the outputs of tools/measure_round.sh (gpurun_out/) into profiles/:
r1_bench.json, r1_bench_reference.json, r1_launches_bench.csv + r1_launches.md (table part),
traffic.json (warm per-term DRAM bytes of the term kernels).
Usage: python tools/update_profiles.py [round-tag, default r1]"""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PRO = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"

shutil.copy(os.path.join(OUT, "bench.json"), os.path.join(PRO, f"{tag}_bench.json"))
shutil.copy(os.path.join(OUT, "bench_ref.json"), os.path.join(PRO, f"{tag}_bench_reference.json"))
shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PRO, f"{tag}_launches_bench.csv"))

# launch table: replace the table inside r?_launches.md
table = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), "launches",
                        os.path.join(OUT, "launches.csv")], capture_output=True, text=True).stdout
md_path = os.path.join(PRO, f"{tag}_launches.md")
md = open(md_path).read()
md = re.sub(r"\| kernel \| launches \|.*?\*\*total\*\*[^\n]*\n", table, md, flags=re.S)
open(md_path, "w").write(md)

# warm per-term traffic
rows = list(csv.reader(open(os.path.join(OUT, "traffic.csv"))))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
         "msecond": 1e3, "ms": 1e3}
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    name = r[h.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").strip()
    m, u = r[h.index("Metric Name")], r[h.index("Metric Unit")]
    v = float(r[h.index("Metric Value")].replace(",", "")) * scale.get(u, 1)
    agg[name][m] += v
    if m == "gpu__time_duration.sum":
        cnt[name] += 1


def tot(k):
    return agg[k]["dram__bytes_read.sum"] + agg[k]["dram__bytes_write.sum"]


bench = json.load(open(os.path.join(OUT, "bench.json")))
t = {"n_obs": bench["config"]["n_obs"], "blocks": cnt["k_lm_reduce"],
     "per_term_bytes": {"k_cam_pipe": tot("k_cam_pipe") + tot("k_cam"), "k_cam": tot("k_cam"),
                        "k_lm_reduce": tot("k_lm_reduce")},
     "per_launch_bytes": {k: tot(k) / max(cnt[k], 1) for k in ("k_cam_pipe", "k_cam",
                                                              "k_lm_reduce")},
     "per_term_ncu_us": {k: agg[k]["gpu__time_duration.sum"] for k in ("k_cam_pipe", "k_cam",
                                                                       "k_lm_reduce")},
     "launches_per_term": dict(cnt),
     "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
               "--cache-control none --clock-control none over one steady-state term of "
               "tools/profile_terms.py vlarge 1 4 (tools/measure_round.sh); warm L2 (the blocked "
               "term keeps s and t in the persisting L2).  k_cam_pipe's per-term figure includes "
               "the term's k_cam epilogue launch (the camera pass of one term)."}
json.dump(t, open(os.path.join(PRO, "traffic.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in t.items() if k != "source"}, indent=1))
