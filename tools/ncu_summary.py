"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("unnamed>::", "")
    try:
        v = float(d["Metric Value"].replace(",", "")) * (1e-3 if d["Metric Unit"] == "ns" else 1.0 if d["Metric Unit"] == "us" else 1e3)
    except ValueError:
        continue
    if v != v:  # nan (a replay ncu could not time)
        continue
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
step = {k: v for k, v in tot.items() if "bwd_fused" in k or "spmm" in k or "mse" in k or "sgd" in k or "job_reduce" in k}
print(f"{'kernel':60s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:10.1f} {tot[k]/cnt[k]:9.1f} {100*tot[k]/T:5.1f}%")
print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {T:10.1f}")
S = sum(step.values())
print(f"\nstep kernels only (excluding handle creation): {S:.1f} us")
for k in sorted(step, key=lambda k: -step[k]):
    print(f"  {k[:58]:58s} {100 * step[k] / S:5.1f}%")
