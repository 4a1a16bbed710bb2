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
    v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0 if d["Metric Unit"] == "us" else 1e3)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:10.1f} {tot[k]/cnt[k]:9.1f} {100*tot[k]/T:5.1f}%")
print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {T:10.1f}")
