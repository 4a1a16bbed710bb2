"""Per-kernel DRAM traffic per launch from an ncu --set full report -> profiles/*_kernel_traffic.json.

usage: python tools/ncu_traffic.py <report.ncu-rep> <out.json> <source note>"""
import csv
import json
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
ix = {h: i for i, h in enumerate(hdr)}


def val(r, name):
    v, u = float(r[ix[name]]), units[ix[name]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3}
    return v * scale.get(u, 1)


# bwd_fused_sk_kernel<RPW, NW, GATE, DWONLY>: DWONLY=1 is sp_linear_bwd_weight alone
classes = {"bwd_fused": r"bwd_fused(_sk_kernel<\d+, \d+, \d, 0[,>]|_kernel)",
           "sddmm_dw_only": r"bwd_fused_sk_kernel<\d+, \d+, \d, 1[,>]",
           "fwd_spmm": r"spmm_tiled|spmm_hyb"}
res = {"source": sys.argv[3], "kernels": {}}
for r in rows[2:]:
    name = re.sub(r"\(.*", "", r[ix["Kernel Name"]])
    for cls, pat in classes.items():
        if re.search(pat, name):
            d = res["kernels"].setdefault(cls, {"launches": []})
            d["launches"].append({"kernel": name, "dram_read_bytes": val(r, "dram__bytes_read.sum"),
                                  "dram_write_bytes": val(r, "dram__bytes_write.sum"),
                                  "duration_us": val(r, "gpu__time_duration.sum")})
for d in res["kernels"].values():
    L = d["launches"]
    d["traffic_bytes_per_launch_mean"] = sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in L) / len(L)
json.dump(res, open(sys.argv[2], "w"), indent=1)
print(json.dumps({k: (len(v["launches"]), v["traffic_bytes_per_launch_mean"]) for k, v in res["kernels"].items()}))
