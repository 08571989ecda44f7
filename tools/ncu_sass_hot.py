"""Top SASS instructions by warp-stall samples for one kernel of an ncu report.
usage: python tools/ncu_sass_hot.py REPORT LAUNCH_INDEX [N]"""
import csv, io, subprocess, sys
rep, idx = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", idx, "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
print(lines[0])
h0 = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[h0:]))))
hdr = rows[0]
data = [r for r in rows[1:] if r and r[0].startswith("0x")]
ci = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") or "Stall" in h and "Sampling" not in h]
samp = ci["Warp Stall Sampling (All Samples)"]
tot = sum(float(r[samp] or 0) for r in data)
print("total samples", tot, "instructions", len(data))
# opcode histogram of samples
from collections import Counter
op = Counter()
for r in data:
    o = r[ci["Source"]].split()[0] if r[ci["Source"]].split() else "?"
    if o.startswith("@"):
        o = r[ci["Source"]].split()[1]
    op[o.split(".")[0]] += float(r[samp] or 0)
print("samples by opcode:", ", ".join(f"{k} {v/tot*100:.1f}%" for k, v in op.most_common(14)))
order = sorted(range(len(data)), key=lambda i: -float(data[i][samp] or 0))
reason_cols = [h for h in hdr if h.lower().startswith("warp stall sampling (") is False and "stall" in h.lower()]
for i in order[:n]:
    r = data[i]
    reasons = []
    for h in hdr:
        if h.startswith("stall_") and "Not Issued" not in h:
            v = float(r[ci[h]] or 0)
            if v > 0:
                reasons.append((v, h))
    reasons.sort(reverse=True)
    print(f"{i:5d} {float(r[samp]):6.0f} {r[ci['Source']][:60]:60s}", " ".join(f"{h[6:]}:{v:.0f}" for v, h in reasons[:3]))
