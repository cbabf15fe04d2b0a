"""Summarise an ncu capture (--set full .ncu-rep) and a launch list (CSV of
gpu__time_duration.sum) into a markdown file under profiles/.

usage: python tools/ncu_summary.py <prof.ncu-rep> <launches.csv> <out.md> [title]
Also writes profiles/ncu_traffic.json (dram bytes per launch of the profiled
kernel) which bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__cluster_dim_x", "launch__shared_mem_per_block_dynamic",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
    "lts__t_bytes.sum", "smsp__average_warp_latency_issue_stalled_barrier", "sm__ctas_launched.sum",
    "l1tex__m_l1tex2xbar_write_bytes_mem_dshared.sum", "l1tex__m_l1tex2xbar_req_cycles_active_mem_dshared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            d[h] = (v, u)
        kernels.append(d)
    return kernels


def stall_summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = rows[2:]
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {c: sum(int(r[hdr.index(c)] or 0) for r in data) for c in cols}
    s = sum(tot.values()) or 1
    ex = defaultdict(int)
    iex = hdr.index("Instructions Executed")
    isrc = hdr.index("Source")
    for r in data:
        toks = r[isrc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        ex[op.split(".")[0]] += int(r[iex] or 0)
    etot = sum(ex.values()) or 1
    return ({k: v / s for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v},
            {k: v / etot for k, v in sorted(ex.items(), key=lambda kv: -kv[1])[:14]})


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    agg = defaultdict(list)
    for r in rows[1:]:
        try:
            agg[r[hdr.index("Kernel Name")]].append(float(r[hdr.index("Metric Value")].replace(",", "")))
        except ValueError:
            pass
    return agg


def main():
    rep, lcsv, out = sys.argv[1:4]
    title = sys.argv[4] if len(sys.argv) > 4 else os.path.basename(rep)
    ks = raw_metrics(rep)
    lines = [f"# {title}", "", f"source: `{os.path.basename(rep)}` (ncu --set full --clock-control none), "
             f"`{os.path.basename(lcsv)}` (gpu__time_duration.sum per launch)", ""]
    traffic = None
    for k in ks:
        name = k.get("Kernel Name", ("?", ""))[0]
        lines.append(f"## kernel `{name}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for key in KEYS:
            if key in k:
                v, u = k[key]
                lines.append(f"| {key} | {v} | {u} |")
        try:
            rd = float(k["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(k["dram__bytes_write.sum"][0].replace(",", ""))
            mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= mul.get(k["dram__bytes_read.sum"][1], 1)
            wr *= mul.get(k["dram__bytes_write.sum"][1], 1)
            traffic = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr, "kernel": name,
                       "source": os.path.join("profiles", os.path.basename(out))}
            lines.append(f"| dram read+write per launch | {rd + wr:.4g} | byte |")
        except Exception:
            pass
        lines.append("")
    stalls, mix = stall_summary(rep)
    lines += ["## warp-stall breakdown (source page, all samples)", "", "| reason | share |", "|---|---|"]
    lines += [f"| {k} | {100 * v:.1f}% |" for k, v in stalls.items()]
    lines += ["", "## executed instruction mix (top opcodes)", "", "| opcode | share |", "|---|---|"]
    lines += [f"| {k} | {100 * v:.1f}% |" for k, v in mix.items()]
    agg = launches(lcsv)
    tot = sum(sum(v) for v in agg.values()) or 1
    lines += ["", "## launch list (share of GPU time in the profiled command)", "",
              "| share | launches | avg us | kernel |", "|---|---|---|---|"]
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {100 * sum(v) / tot:.1f}% | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | `{name[:90]}` |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic:
        with open(os.path.join(os.path.dirname(out), "ncu_traffic.json"), "w") as f:
            json.dump(traffic, f, indent=1)
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()
