#!/usr/bin/env python
"""Summarise one measurement round into profiles/ (tracked):
  profiles/<tag>_bench.json        the bench line
  profiles/<tag>_launches.csv      ncu per-launch list (time, DRAM bytes)
  profiles/<tag>_ncu_summary.txt   key raw metrics + stall mix per captured kernel
  profiles/traffic.json            per-launch DRAM bytes of k_scatter (read by bench.py)
usage: make_profiles.py TAG"""
import csv, io, json, os, shutil, subprocess, sys
tag = sys.argv[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go, pr = os.path.join(root, "gpurun_out"), os.path.join(root, "profiles")
shutil.copy(os.path.join(go, f"{tag}_bench.json"), os.path.join(pr, f"{tag}_bench.json"))
shutil.copy(os.path.join(go, f"{tag}_launches.csv"), os.path.join(pr, f"{tag}_launches.csv"))
# traffic per k_scatter launch from the launch list
rows = list(csv.reader(open(os.path.join(go, f"{tag}_launches.csv"))))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]; ix = {k: i for i, k in enumerate(h)}
per = {}
for r in rows[hi + 1:]:
    if len(r) != len(h): continue
    k = (r[ix["ID"]], r[ix["Kernel Name"]])
    per.setdefault(k, {})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
bench = json.load(open(os.path.join(go, f"{tag}_bench.json")))
n = bench["config"]["n"]; case = bench["config"]["workload"].split(":")[0]
tj_path = os.path.join(pr, "traffic.json")
tj = json.load(open(tj_path)) if os.path.exists(tj_path) else {}
for fam in ["k_scatter<", "k_scatter_fh", "k_fused", "k_hist"]:
    sc = [v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for (i, nm), v in per.items()
          if fam in nm and v["gpu__time_duration.sum"] > 100000]
    if sc:
        tj[f"{case}:{n}:{fam.rstrip('<')}"] = sum(sc) / len(sc)
json.dump(tj, open(tj_path, "w"), indent=1)
# full-capture summary
rep = os.path.join(go, f"{tag}_full.ncu-rep")
out = []
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hh, uu = rr[0], rr[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "launch__grid_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed_op_shared_atom.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
            "smsp__inst_executed_op_global_red.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum"]
    for r in rr[2:]:
        out.append("---- " + r[hh.index("Kernel Name")])
        for w in want:
            if w in hh:
                i = hh.index(w)
                out.append(f"  {w:62s} {r[i]} {uu[i]}")
    for k in ("k_hist", "k_scatter", "k_scatter_fh", "k_fused"):
        s = subprocess.run([sys.executable, os.path.join(root, "tools", "ncu_regions.py"), rep, k],
                           capture_output=True, text=True).stdout.split("\n")[:2]
        out.append(f"==== stall mix {k}: " + " | ".join(s))
open(os.path.join(pr, f"{tag}_ncu_summary.txt"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
