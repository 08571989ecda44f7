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
