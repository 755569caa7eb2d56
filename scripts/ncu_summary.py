"""Writes a text summary of an ncu --set full report (+ optional launch list csv).

usage: python scripts/ncu_summary.py <report.ncu-rep> [launches.csv] > profiles/<name>.txt
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
print(f"# ncu --set full summary of {rep}")
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    print(f"\nkernel: {d['Kernel Name']}\ngrid {d.get('Grid Size')} block {d.get('Block Size')}")
    keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
            "smsp__sass_inst_executed_op_tmem_ldt.sum", "smsp__sass_inst_executed_op_tmem_stt.sum",
            "sm__sass_inst_executed_op_shared_ld.sum", "smsp__inst_executed_op_utcmma.sum"]
    for k in keys:
        if k in d:
            print(f"  {k:70s} {d[k]:>18s} {u.get(k, '')}")
    st = {k[len('smsp__pcsamp_warps_issue_stalled_'):]: float(d[k] or 0) for k in hdr
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(st.values()) or 1
    print("  warp-state samples (share):", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in
                                                 sorted(st.items(), key=lambda x: -x[1])[:10]))
if len(sys.argv) > 2:
    lines = open(sys.argv[2]).read().splitlines()
    i0 = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rr = list(csv.reader(lines[i0:]))
    h = rr[0]
    agg = collections.defaultdict(list)
    for r in rr[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            agg[d["Kernel Name"]].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    print(f"\n# launch list ({sys.argv[2]}): gpu__time_duration.sum per kernel (cold-cache, serialised)")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"  {len(v):4d} launches  avg {sum(v) / len(v) / 1e3:10.3f} us  share {sum(v) / tot * 100:5.1f}%  {k[:90]}")
