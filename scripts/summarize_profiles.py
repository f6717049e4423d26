"""Summarize an ncu round into profiles/ (tracked): launch-list shares and the
key counters of each full capture.

usage: python scripts/summarize_profiles.py <tag> [gpurun_out dir] [config]
(config: the bench.py --config the captures ran, default c3; c3rw for the
roulette capture)
writes profiles/<tag>_launches.csv, profiles/<tag>_kernels.csv,
profiles/<tag>_hotlines.txt
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
config = sys.argv[3] if len(sys.argv) > 3 else "c3"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_dir = os.path.join(root, "profiles")
os.makedirs(out_dir, exist_ok=True)

# ---- launch list -------------------------------------------------------------
launch_path = os.path.join(src, f"launches_{tag}.csv")
rows = list(csv.reader(open(launch_path))) if os.path.exists(launch_path) else [["Kernel Name", "Metric Value"]]
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg, cnt = collections.OrderedDict(), collections.Counter()
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    agg[name] = agg.get(name, 0.0) + float(r[vi].replace(",", "")) / 1e3
    cnt[name] += 1
total = sum(agg.values()) or 1.0
with open(os.path.join(out_dir, f"{tag}_launches.csv"), "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["kernel", "launches", "total_us", "mean_us", "share"])
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        w.writerow([k, cnt[k], f"{v:.1f}", f"{v / cnt[k]:.1f}", f"{v / total:.4f}"])

# ---- full captures ----------------------------------------------------------------
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
]
reps = sorted(f for f in os.listdir(src) if f.startswith("prof_") and f.endswith(f"_{tag}.ncu-rep"))
kern_rows = []
hot = []
for rep in reps:
    path = os.path.join(src, rep)
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    if len(r) < 3:
        continue
    hh, uu, vv = r[0], r[1], r[2]
    rec = {"report": rep, "kernel": vv[hh.index("Kernel Name")].split("(")[0] if "Kernel Name" in hh else ""}
    for m in METRICS:
        if m in hh:
            rec[m] = f"{vv[hh.index(m)]} {uu[hh.index(m)]}".strip()
    kern_rows.append(rec)
    lines = subprocess.run([sys.executable, os.path.join(root, "scripts", "ncu_lines.py"), path, "12"],
                           capture_output=True, text=True).stdout
    hot.append(f"== {rep}\n{lines}")
with open(os.path.join(out_dir, f"{tag}_kernels.csv"), "w", newline="") as f:
    cols = ["report", "kernel"] + METRICS
    w = csv.DictWriter(f, fieldnames=cols)
    w.writeheader()
    for rec in kern_rows:
        w.writerow(rec)
# per-launch DRAM traffic of each captured kernel, read by bench.py for
# roofline.traffic (dram__bytes_read.sum + dram__bytes_write.sum)
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def _bytes(v):
    if not v:
        return None
    num, _, unit = v.partition(" ")
    return float(num.replace(",", "")) * UNITS.get(unit.strip(), 1)


traffic_path = os.path.join(out_dir, "traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
for rec in kern_rows:
    base = rec["kernel"].replace("void ", "").split("<")[0].split("::")[-1].strip()
    rd, wr = _bytes(rec.get("dram__bytes_read.sum")), _bytes(rec.get("dram__bytes_write.sum"))
    if rd is None or wr is None:
        continue
    cfg = "c3rw" if base == "k_construct_rw" else config  # scripts/profile_round.sh
    inst = rec.get("smsp__inst_executed.sum")
    traffic[f"{base}@{cfg}"] = {"config": cfg,
                     "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
                     "warp_instructions_per_launch": float(inst.split()[0].replace(",", "")) if inst else None,
                     "issue_active_pct": rec.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                     "duration": rec.get("gpu__time_duration.sum"), "l2_hit_rate": rec.get("lts__t_sector_hit_rate.pct"),
                     "capture": f"profiles/{tag}_kernels.csv ({rec['report']}, ncu --set full)"}
with open(traffic_path, "w") as f:
    json.dump(traffic, f, indent=1, sort_keys=True)
with open(os.path.join(out_dir, f"{tag}_hotlines.txt"), "w") as f:
    f.write("\n".join(hot))
print(open(os.path.join(out_dir, f"{tag}_launches.csv")).read())
for rec in kern_rows:
    print(rec["report"], rec.get("gpu__time_duration.sum"), rec.get("dram__bytes_read.sum"),
          rec.get("dram__bytes_write.sum"), rec.get("lts__t_sector_hit_rate.pct"),
          rec.get("smsp__issue_active.avg.pct_of_peak_sustained_active"))
