"""Stall-reason totals over an address range (or all) of one launch's SASS.
usage: python tools/ncu_stalls.py REPORT LAUNCH_INDEX [lo hi]  (lo/hi = SASS row indices)"""
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
if len(data) % 2 == 0 and data[:len(data) // 2] == data[len(data) // 2:]:
    data = data[:len(data) // 2]
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, len(data))
c = Counter()
for r in data[lo:hi]:
    for h in hdr:
        if h.startswith("stall_") and "Not Issued" not in h:
            c[h[6:]] += float(r[ci[h]] or 0)
tot = sum(c.values())
print(lines[0], f"rows {lo}-{hi}", f"samples {tot:.0f}")
print(", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in c.most_common(12)))
