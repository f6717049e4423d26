"""Aggregate ncu source-page warp-stall samples per CUDA source line.

usage: python scripts/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
stats, cur_file, hdr = {}, "", None
total = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        samples = int(r[4]) if r[4] not in ("-", "") else 0
        inst = int(r[7]) if r[7] not in ("-", "") else 0
    except ValueError:
        continue
    key = (cur_file, r[0])
    s = stats.setdefault(key, [0, 0, r[1][:90]])
    s[0] += samples
    s[1] += inst
    total += samples
for (f, line), (smp, inst, src) in sorted(stats.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100.0 * smp / max(total, 1):5.1f}%  {f}:{line:>4}  inst={inst:>11}  {src}")
