"""Summarise an ncu report (from gpurun_out/) into profiles/<name>.json + .md.

usage: python tools/ncu_summary.py gpurun_out/prof_r01.ncu-rep profiles/r01_ncu [cells]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "time_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dfma": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "dmul": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "dadd": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "fp64_all": "smsp__sass_thread_inst_executed_op_fp64_pred_on.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_busy_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread",
    "warp_inst": "smsp__inst_executed.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "grid": "launch__grid_size",
}


def to_num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return s


def fp64_from_source(rep: str, idx: int):
    """Predicated-on thread instructions of FP64-pipe opcodes of launch idx."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True,
                         text=True).stdout.splitlines()
    try:
        h0 = next(i for i, ln in enumerate(out) if ln.startswith('"Address"'))
    except StopIteration:
        return None
    rows = list(csv.reader(io.StringIO("\n".join(out[h0:]))))
    ci = {h: i for i, h in enumerate(rows[0])}
    data = [r for r in rows[1:] if r and r[0].startswith("0x")]
    if len(data) % 2 == 0 and data[:len(data) // 2] == data[len(data) // 2:]:
        data = data[:len(data) // 2]
    tot = 0.0
    for r in data:
        t = r[ci["Source"]].split()
        if t and (t[1] if t[0].startswith("@") else t[0]).split(".")[0] in ("DFMA", "DMUL", "DADD", "DSETP",
                                                                          "DMNMX"):
            tot += float(r[ci["Predicated-On Thread Instructions Executed"]] or 0)
    return tot


def main():
    rep, out = sys.argv[1], sys.argv[2]
    cells = float(sys.argv[3]) if len(sys.argv) > 3 else 1048576.0
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, m in METRICS.items():
            if m in hdr:
                v = to_num(r[hdr.index(m)])
                u = units[hdr.index(m)]
                if k == "time_us" and u == "ns":
                    v = v / 1e3
                if k == "time_us" and u == "ms":
                    v = v * 1e3
                if k.startswith("dram_") and k != "dram_pct":
                    v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                d[k] = v
        if not isinstance(d.get("fp64_all"), float):  # not in --set full: count from the SASS page
            d["fp64_all"] = fp64_from_source(rep, len(res))
        if isinstance(d.get("fp64_all"), float):
            d["fp64_per_cell"] = d["fp64_all"] / cells
        if isinstance(d.get("dram_read"), float):
            d["dram_bytes_per_cell"] = (d["dram_read"] + d["dram_write"]) / cells
        res.append(d)
    json.dump({"report": rep, "cells": cells, "kernels": res}, open(out + ".json", "w"), indent=1)
    with open(out + ".md", "w") as f:
        f.write(f"# ncu summary: {rep}\n\ncells per launch: {cells:.0f}\n\n")
        f.write("| kernel | us | FP64 instr/cell | FP64 pipe % | warps active % | DRAM B/cell | "
                "DRAM % | L2 hit % | regs |\n|---|---|---|---|---|---|---|---|---|\n")
        for d in res:
            f.write("| {kernel} | {t:.1f} | {w:.0f} | {p:.1f} | {a:.1f} | {b:.0f} | {dp:.1f} | "
                    "{l2} | {regs} |\n".format(
                        kernel=d["kernel"][:40], t=d.get("time_us", 0), w=d.get("fp64_per_cell", 0),
                        p=d.get("fp64_pipe_pct", 0), a=d.get("warps_active_pct", 0),
                        b=d.get("dram_bytes_per_cell", 0), dp=d.get("dram_pct", 0),
                        l2=d.get("l2_hit_pct", "-"), regs=d.get("regs", "-")))
    print(open(out + ".md").read())


if __name__ == "__main__":
    main()
