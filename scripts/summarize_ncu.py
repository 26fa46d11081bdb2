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
    "quant_elem_kernel<2, 0, 256, 2, 0>": "e5m2_rne",
    "quant_elem_kernel<10, 1, 256, 2, 0>": "fp16_sr_counter",
    "quant_lfsr_warp_kernel<2>": "e5m2_sr_lfsr",
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
    """Per kernel, launches split into the full-size class (the bench's timed
    2^28-element sweep: DRAM bytes >= 1/2 of the kernel's largest launch) and
    the small rest (e2e chunks, warm-up of other sizes); the roofline traffic is
    the full-size median."""
    text = open(csv_path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per_launch = collections.OrderedDict()
    order = []
    scale_t = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    scale_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows:
        key = (r["ID"], _short(r["Kernel Name"]))
        if key[1] not in order:
            order.append(key[1])
        d = per_launch.setdefault(key, {"us": 0.0, "rd": 0.0, "wr": 0.0})
        m, v = r["Metric Name"], float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        if m == "gpu__time_duration.sum":
            d["us"] = v * scale_t.get(unit, 1.0)
        elif m == "dram__bytes_read.sum":
            d["rd"] = v * scale_b.get(unit, 1)
        elif m == "dram__bytes_write.sum":
            d["wr"] = v * scale_b.get(unit, 1)
    tot = sum(d["us"] for d in per_launch.values())
    med = lambda a: sorted(a)[len(a) // 2] if a else 0.0  # noqa: E731
    lines = ["# ncu launch list (cold cache, serialised; compare shares, not absolutes)", "",
             f"source: `{csv_path}`", "",
             "Per kernel: the full-size launches (DRAM bytes >= 1/2 of its largest launch: the",
             "timed 2^28-element sweep) and the small ones (e2e chunks) separately.", "",
             "| kernel | class | launches | median us | share of kernel time | DRAM read MB/launch | DRAM write MB/launch |",
             "|---|---|---|---|---|---|---|"]
    traffic = {}
    for k in order:
        ls = [d for (i, kk), d in per_launch.items() if kk == k]
        big = max(d["rd"] + d["wr"] for d in ls)
        for cls, group in (("full", [d for d in ls if d["rd"] + d["wr"] >= 0.5 * big]),
                           ("small", [d for d in ls if d["rd"] + d["wr"] < 0.5 * big])):
            if not group:
                continue
            us = med([d["us"] for d in group])
            rd, wr = med([d["rd"] for d in group]), med([d["wr"] for d in group])
            lines.append(f"| `{k}` | {cls} | {len(group)} | {us:.1f} | "
                         f"{100 * sum(d['us'] for d in group) / tot:.1f}% | {rd / 1e6:.1f} | {wr / 1e6:.1f} |")
            if cls == "full":
                for pat, key in BENCH_KEYS.items():
                    if k.replace(" ", "") == pat.replace(" ", ""):
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
