#!/usr/bin/env python3
"""Summarise ncu artefacts (from gpurun_out/) into profiles/.

    python scripts/summarize_ncu.py launches gpurun_out/launches.csv profiles/launches_r01.md
    python scripts/summarize_ncu.py report gpurun_out/prof_lfsr.ncu-rep profiles/ncu_lfsr_r01.md

`launches` also writes profiles/dram_traffic.json (DRAM bytes per launch of the
bench's kernels, the roofline "traffic" field bench.py reports).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

BENCH_KEYS = {
    "quant_elem_kernel<2, 0, 256>": "e5m2_rne",
    "quant_lfsr_staged_kernel<2>": "e5m2_sr_lfsr",
    "quant_elem_kernel<10, 1, 256>": "fp16_sr_counter",
}

KEY_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "gpc__cycles_elapsed.max", "lts__t_sector_hit_rate.pct",
]


def _short(name):
    name = name.replace("void ", "").replace("fp8b::", "").replace("(int)", "")
    return name.split("(")[0].strip()


def launches(csv_path, out_md):
    text = open(csv_path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = collections.defaultdict(lambda: {"n": 0, "us": [], "rd": [], "wr": []})
    order = []
    for r in rows:
        k = _short(r["Kernel Name"])
        if k not in per:
            order.append(k)
        m, v = r["Metric Name"], r["Metric Value"].replace(",", "")
        unit = r.get("Metric Unit", "")
        d = per[k]
        if m == "gpu__time_duration.sum":
            d["n"] += 1
            d["us"].append(float(v) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
                                       "ms": 1e3, "msecond": 1e3}.get(unit, 1.0))
        elif m == "dram__bytes_read.sum":
            d["rd"].append(float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1))
        elif m == "dram__bytes_write.sum":
            d["wr"].append(float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1))
    tot = sum(sum(d["us"]) for d in per.values())
    lines = ["# ncu launch list (cold cache, serialised; compare shares, not absolutes)", "",
             f"source: `{csv_path}`", "",
             "| kernel | launches | median us | share of kernel time | DRAM read MB/launch | DRAM write MB/launch |",
             "|---|---|---|---|---|---|"]
    traffic = {}
    for k in order:
        d = per[k]
        if not d["n"]:
            continue
        med = lambda a: sorted(a)[len(a) // 2] if a else 0.0
        mean = med(d["us"])  # median launch (the list mixes the 2^28 sweep with small e2e runs)
        rd = med(d["rd"])
        wr = med(d["wr"])
        lines.append(f"| `{k}` | {d['n']} | {mean:.1f} | {100 * sum(d['us']) / tot:.1f}% | "
                     f"{rd / 1e6:.1f} | {wr / 1e6:.1f} |")
        for pat, key in BENCH_KEYS.items():
            if k.startswith(pat.split("<")[0]) and k.replace(" ", "") == pat.replace(" ", ""):
                traffic[key] = round(rd + wr)
    open(out_md, "w").write("\n".join(lines) + "\n")
    tj = os.path.join(os.path.dirname(out_md), "dram_traffic.json")
    json.dump(traffic, open(tj, "w"), indent=1)
    print(open(out_md).read())
    print(traffic)


def report(rep, out_md):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units, vals = r[0], r[1], r[2]
    name = vals[h.index("Kernel Name")]
    lines = [f"# ncu --set full: `{_short(name)}`", "", f"report: `{rep}`", "",
             "| metric | value | unit |", "|---|---|---|"]
    for m in KEY_METRICS:
        if m in h:
            i = h.index(m)
            lines.append(f"| {m} | {vals[i]} | {units[i]} |")
    stalls = []
    for i, m in enumerate(h):
        if m.startswith("smsp__average_warps_issue_stalled") and m.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(vals[i]), m.replace("smsp__average_warps_issue_stalled_", "")
                               .replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    lines += ["", "Top warp stall reasons (per issue):", ""]
    for v, m in sorted(stalls, reverse=True)[:8]:
        lines.append(f"- {m}: {v:.3f}")
    open(out_md, "w").write("\n".join(lines) + "\n")
    print(open(out_md).read())


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2], sys.argv[3])
