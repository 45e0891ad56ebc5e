"""Summarize a profile capture (tools/profile_capture.sh) into profiles/:
the bench line, the aggregated launch list, key ncu metrics of the two fused
kernels, and the per-iteration DRAM traffic used as bench.py's `traffic`."""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = "gpurun_out"
dst = "profiles"
os.makedirs(dst, exist_ok=True)
bench = json.loads(open(f"{src}/{tag}_bench.json").read().strip().splitlines()[-1])
with open(f"{dst}/{tag}_bench.json", "w") as f:
    json.dump(bench, f, indent=1)

rows = [r for r in csv.reader(open(f"{src}/{tag}_launches.csv")) if len(r) > 10 and r[0].isdigit()]
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    name = r[4].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(r[-1]) / 1e3          # ns -> us
tot = sum(v[1] for v in agg.values())
launch_lines = [f"{k:48s} {n:5d} {t/1e3:9.2f} ms {100*t/tot:5.1f}%  avg {t/n:9.1f} us"
                for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]
with open(f"{dst}/{tag}_launches_c5.csv", "w") as f:
    f.write(open(f"{src}/{tag}_launches.csv").read())

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum"]
kern = {}
for k in ("k_update", "k_partition"):
    # exported on the GPU box (profile_capture.sh) when the report is too big
    # to travel; else read from the .ncu-rep here
    raw = f"{src}/{tag}_{k}_raw.csv"
    out = open(raw).read() if os.path.exists(raw) else subprocess.run(
        ["ncu", "-i", f"{src}/{tag}_{k}.ncu-rep", "--page", "raw", "--csv"],
        capture_output=True, text=True).stdout
    rr = list(csv.reader(out.splitlines()))
    h, u, v = rr[0], rr[1], rr[2]
    d = {}
    for m in METRICS:
        if m in h:
            i = h.index(m)
            d[m] = (v[i], u[i])
    kern[k] = d
    dpath = f"{src}/{tag}_{k}_details.txt"
    det = open(dpath).read() if os.path.exists(dpath) else subprocess.run(
        ["ncu", "-i", f"{src}/{tag}_{k}.ncu-rep", "--page", "details"],
        capture_output=True, text=True).stdout
    with open(f"{dst}/{tag}_ncu_{k}_details.txt", "w") as f:
        f.write(det)


def num(x):
    v, unit = x
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "msecond": 1e-3,
             "usecond": 1e-6, "nsecond": 1e-9}.get(unit, 1)
    return v * scale


traffic = {k: num(kern[k]["dram__bytes_read.sum"]) + num(kern[k]["dram__bytes_write.sum"])
           for k in kern}
size = int(bench["config"]["workload"].split()[1].split("x")[0])
with open(f"{dst}/traffic_latest.json", "w") as f:
    json.dump({"size": size, "bytes_per_iteration": sum(traffic.values()),
               "source": f"ncu --set full ({dst}/{tag}_ncu_*_details.txt): one steady-state "
                         "k_update + k_partition launch, C5, dense pass",
               "per_kernel": traffic}, f, indent=1)

r = bench["roofline"]
lines = [f"# Profile summary {tag} (B200, sm_100a)", "",
         "Bench line (`python bench.py`, defaults) — " + f"{dst}/{tag}_bench.json:", "",
         "| quantity | value |", "|---|---|",
         f"| dense C5 throughput (`value`) | **{bench['value']:.1f} Gpix-it/s** "
         f"({bench['ms_per_step']:.0f} ms per 500-iteration job) |",
         f"| canonical roofline (12 B/px-it vs {r['peak']} GB/s) | {r['achieved']:.0f} GB/s = "
         f"**{100*r['frac']:.1f} %** |",
         f"| actual-bytes roofline ({r['actual_bytes_per_px_it']:.2f} B/px-it) | "
         f"{r['achieved_actual_gbs']:.0f} GB/s = {100*r['frac_actual']:.1f} % |",
         f"| per iteration: update / partition+finalize | {r['update_ms']:.3f} ms / "
         f"{r['partition_ms']:.3f} ms |",
         f"| uniform-window skip (bit-identical) | {bench['uniform_skip']['value']:.1f} Gpix-it/s |",
         f"| end to end through the C ABI | {bench['e2e']['value']:.1f} Gpix-it/s |",
         f"| CPU baseline ({bench['cpu_baseline']['kind']}, {bench['cpu_baseline']['cores']} "
         f"threads) | {bench['cpu_baseline']['value']*1e3:.0f} Mpix-it/s |",
         f"| clocks | {bench['clocks']} |", ""]
oc = bench.get("other_configs") or {}
if oc:
    lines += ["Other BASELINE configs measured by the same run:", "",
              "| config | Gpix-it/s | note |", "|---|---|---|"]
    for k, v in oc.items():
        note = v.get("bound", "")
        if "roofline" in v:
            note = f"{100*v['roofline']['frac']:.1f} % of the {v['roofline']['algorithmic_bytes_per_px_it']:.0f} B/px-it roofline"
        lines.append(f"| {k} | {v['value']:.2f} | {v['workload']}; {note} |")
    lines.append("")
lines += [f"Launch list ({dst}/{tag}_launches_c5.csv: `ncu --metrics gpu__time_duration.sum "
          "--clock-control none -c 1200` of the bench command; cold-cache, serialised):", "",
          "```"] + launch_lines[:14] + ["```", "",
          "ncu --set full, one steady-state launch each (details in "
          f"{dst}/{tag}_ncu_*_details.txt):", "", "| metric | k_update | k_partition |",
          "|---|---|---|"]
for m in METRICS:
    a = kern["k_update"].get(m, ("-", ""))
    b = kern["k_partition"].get(m, ("-", ""))
    lines.append(f"| {m} | {a[0]} {a[1]} | {b[0]} {b[1]} |")
lines += ["", f"DRAM traffic per iteration: {sum(traffic.values())/1e9:.3f} GB "
          f"({sum(traffic.values())/size/size:.2f} B/px) vs canonical 12 B/px."]
open(f"{dst}/{tag}_summary.md", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
