#!/bin/bash
# Refresh profiles/r2_* from a tools/r2_measure.sh run's gpurun_out/${TAG}_* files.
cd "$(dirname "$0")/.."
T=${1:?tag}
grep "^{" gpurun_out/${T}_bench.log > profiles/r2_bench_cfg5.json
for k in cfg5 cfg2a cfg3 cfg4_uniform0.95 cfg4_zipf0.95 cfg4_uniform0.99; do
  cp gpurun_out/${T}_full_${k}_summary.txt profiles/r2_ncu_full_${k}.txt
done
cp gpurun_out/${T}_launches.csv profiles/r2_ncu_launches.csv
python tools/ncu_summary.py profiles/r2_ncu_launches.csv > profiles/r2_ncu_launches_summary.txt 2>&1
python - "$T" <<'PY'
import csv, glob, json, sys
T = sys.argv[1]
json.dump(json.load(open(f'gpurun_out/{T}_full_cfg5_traffic.json')), open('profiles/r2_kernel_traffic.json', 'w'), indent=1)
keys = ["gpu__time_duration.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
with open('profiles/r2_l2_traffic.txt', 'w') as out:
    out.write(f"# L2 -> SM traffic of every kernel in the round-2 --set full captures ({T}; tools/r2_measure.sh)\n")
    out.write("# columns: duration us | lts__throughput % of peak | L2->SM read MB (l1tex__m_xbar2l1tex_read_bytes) | "
              "the same, % of the xbar port peak | shared-memory wavefronts % | issue active %\n")
    out.write("config | kernel | us | L2 thr % | L2->SM MB | L2->SM % | smem wf % | issue %\n")
    for f in sorted(glob.glob(f'gpurun_out/{T}_full_*_raw.csv')):
        rows = list(csv.reader(open(f)))
        h, units = rows[0], rows[1]
        idx = [h.index(k) for k in keys]
        ik = h.index("Kernel Name")
        for r in rows[2:]:
            name = r[ik].split('(')[0].replace('void ', '').split('::')[-1]
            vals = []
            for i, k in zip(idx, keys):
                v = float(r[i]); u = units[i]
                if k == "gpu__time_duration.sum": v *= {"ns": 1e-3, "us": 1, "ms": 1e3}.get(u, 1)
                if k.endswith("read_bytes.sum"): v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)
                vals.append(f"{v:.1f}")
            out.write(f.split(f'{T}_full_')[1].replace('_raw.csv', '') + " | " + name + " | " + " | ".join(vals) + "\n")
PY
(python tools/ncu_sass_breakdown.py gpurun_out/${T}_full_cfg5.ncu-rep bwd_fused 1; echo;
 python tools/ncu_sass_breakdown.py gpurun_out/${T}_full_cfg5.ncu-rep spmm_hyb 0) > profiles/r2_sass_breakdown_cfg5.txt 2>&1
echo "profiles refreshed from $T"
