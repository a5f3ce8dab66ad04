"""Turn the achieved-error log of the GPU parity tests (PV_PARITY_REPORT=<json> python -m
pytest tests -m gpu) into profiles/<tag>_parity.md: per test and quantity, the worst achieved
error next to its tolerance.  Usage: python tools/parity_table.py gpurun_out/parity.json [tag]"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1]
tag = sys.argv[2] if len(sys.argv) > 2 else "r2"
rows = json.load(open(src))
worst = collections.OrderedDict()
for r in rows:
    test = r["test"].split("::", 1)[-1] if "::" in r["test"] else r["test"]
    key = (r["test"].split("::")[0].split("/")[-1], test, r["quantity"], r["tol"])
    worst[key] = max(worst.get(key, 0.0), r["error"])
out = [f"# Round {tag[1:]} — achieved parity errors of the GPU tests (1 B200)", "",
       "`PV_PARITY_REPORT=gpurun_out/parity.json python -m pytest tests -m gpu` (every `check()` of",
       "`tests/_pvutil.py` logs the achieved error; worst case per test and quantity below).  Errors",
       "are relative (norm-wise over the whole output, SURVEY App. B.1) against fixtures produced by",
       "the real reference (`tests/golden/make_golden*.py`) unless the quantity says otherwise.", "",
       f"{len(rows)} checks, {len(worst)} distinct (test, quantity) pairs; largest error / tolerance "
       f"ratio {max(v / k[3] for k, v in worst.items() if k[3] > 0):.3f}.", "",
       "| file | test | quantity | achieved | tolerance |", "|---|---|---|---|---|"]
for (f, t, q, tol), e in worst.items():
    out.append(f"| {f} | {t} | {q} | {e:.2e} | {tol:.0e} |")
path = os.path.join(ROOT, "profiles", f"{tag}_parity.md")
open(path, "w").write("\n".join(out) + "\n")
print(path, len(rows), "checks")
