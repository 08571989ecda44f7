"""Executed instruction mix (warp-level) by opcode for one launch of an ncu report.
usage: python tools/ncu_mix.py REPORT LAUNCH_INDEX"""
import csv, io, subprocess, sys
from collections import Counter
rep, idx = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", idx, "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
h0 = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[h0:]))))
hdr = rows[0]
ci = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[1:] if r and r[0].startswith("0x")]
half = len(data) // 2 if len(data) % 2 == 0 and data[:len(data)//2] == data[len(data)//2:] else len(data)
data = data[:half]
ex = ci["Instructions Executed"]
c = Counter()
for r in data:
    t = r[ci["Source"]].split()
    if not t:
        continue
    o = t[1] if t[0].startswith("@") else t[0]
    c[o.split(".")[0]] += float(r[ex] or 0)
tot = sum(c.values())
print(lines[0])
print(f"warp instructions {tot:.4g}")
print(", ".join(f"{k} {v/tot*100:.1f}%" for k, v in c.most_common(25)))

# executed FP64 thread instructions (DFMA/DMUL/DADD/DSETP/DMNMX...) per launch
pt = ci["Predicated-On Thread Instructions Executed"]
fp64 = 0.0
for r in data:
    t = r[ci["Source"]].split()
    if not t:
        continue
    o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    if o in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "DMMA"):
        fp64 += float(r[pt] or 0)
cells = float(sys.argv[3]) if len(sys.argv) > 3 else 0
print(f"fp64 thread instructions {fp64:.4g}" + (f" = {fp64 / cells:.1f} per cell" if cells else ""))
