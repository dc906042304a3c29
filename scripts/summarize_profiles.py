#!/usr/bin/env python
"""Turn gpurun_out/ evidence (bench JSON lines, ncu launch lists, ncu --set full
reports) into the committed summaries under profiles/.

    python scripts/summarize_profiles.py <tag> <config> [<config> ...]

Writes profiles/<tag>_<config>.md (bench line, per-kernel launch shares, key
ncu counters, top stall reasons) and updates profiles/traffic.json (DRAM bytes
read + written per launch of the attention kernel, read by bench.py).
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def ncu_raw(rep: str) -> dict:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def to_bytes(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return x * scale


def launches(path: str):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in data:
        if len(r) > iv and r[iv]:
            v = float(r[iv].replace(",", ""))
            v = v / 1e3 if r[iu] == "ns" else (v * 1e3 if r[iu] == "ms" else v)   # -> us
            name = r[ik].split("(")[0].replace("void ", "").replace("hetis::<unnamed>::", "")
            agg[name].append(v)
    return agg


def main():
    tag, cfgs = sys.argv[1], sys.argv[2:]
    os.makedirs(PROF, exist_ok=True)
    tpath = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for c in cfgs:
        lines = [f"# {tag} / {c}\n"]
        bpath = os.path.join(OUT, f"bench_{tag}_{c}.log")
        if os.path.exists(bpath):
            js = [l for l in open(bpath).read().splitlines() if l.startswith("{")]
            if js:
                d = json.loads(js[-1])
                r = d["roofline"]
                lines += ["## bench.py line (not under a profiler)\n", "```json", json.dumps(d, indent=1), "```\n",
                          f"attention kernel: {r['achieved']:.0f} GB/s achieved = {100 * r['frac']:.1f}% of "
                          f"{r['peak']:.0f} GB/s ({r['peak_source']}); {100 * r['frac_of_8TBps_nominal']:.1f}% of "
                          f"8 TB/s nominal\n"]
        lpath = os.path.join(OUT, f"launches_{tag}_{c}.csv")
        if os.path.exists(lpath):
            agg = launches(lpath)
            tot = sum(sum(v) for v in agg.values())
            lines += ["## ncu launch list (cold-cache, serialised; compare shares)\n",
                      "| kernel | launches | mean us | share |", "|---|---|---|---|"]
            for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
                lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.2f} | {100 * sum(v) / tot:.1f}% |")
            lines.append("")
        rep = os.path.join(OUT, f"prof_{tag}_{c}.ncu-rep")
        if os.path.exists(rep):
            raw = ncu_raw(rep)
            lines += ["## ncu --set full, attention kernel (one launch)\n", "| metric | value | unit |", "|---|---|---|"]
            for k in KEYS:
                if k in raw:
                    lines.append(f"| {k} | {raw[k][0]} | {raw[k][1]} |")
            stalls = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", ""), float(v[0] or 0)) for h, v in raw.items()
                if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")),
                key=lambda x: -x[1])[:8]
            lines += ["", "top stall reasons (warps per issue-active cycle): " +
                      ", ".join(f"{n} {v:.2f}" for n, v in stalls), ""]
            if "dram__bytes_read.sum" in raw:
                rb = to_bytes(*raw["dram__bytes_read.sum"])
                wb = to_bytes(*raw["dram__bytes_write.sum"])
                traffic[f"{c}/N1"] = rb + wb
                lines.append(f"DRAM traffic per launch: {rb / 1e9:.4f} GB read + {wb / 1e6:.2f} MB written\n")
        with open(os.path.join(PROF, f"{tag}_{c}.md"), "w") as f:
            f.write("\n".join(lines) + "\n")
        print("wrote", os.path.join(PROF, f"{tag}_{c}.md"))
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
