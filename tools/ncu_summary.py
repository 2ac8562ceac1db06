"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/ncu_summary.py <tag> <launches.csv> <prof.ncu-rep> [...]

Writes profiles/<tag>_ncu_full.json (per captured kernel: duration, DRAM
bytes, throughput %, occupancy, stall mix), profiles/<tag>_launches.json
(share of device time per kernel over the launch list) and
profiles/traffic.json (DRAM bytes per launch keyed by bench timer name,
read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "warp_inst",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
}
STALLS = ["long_scoreboard", "barrier", "mio_throttle", "short_scoreboard", "wait", "selected",
          "not_selected", "math_pipe_throttle", "lg_throttle"]

# kernel name fragment -> bench.py timer name
# kernel-name pattern -> bench.py timer name (demangled with or without casts)
TIMER = [(r"k_scatter_tile(_fp)?<(\(int\))?3", "sl_scatter_sweep"),
         (r"k_gather_tile<(\(int\))?3, (\(bool\))?(0|false), (\(int\))?2>", "sl_inc_step"),
         (r"k_inc_u", "sl_inc_init"), (r"k_assemble", "sl_assemble"),
         (r"k_axis_d2<(\(int\))?\d+, (\(int\))?1>", "spec_axis1"),
         (r"k_axis_d2<(\(int\))?\d+, (\(int\))?2>", "spec_axis2"),
         (r"k_axis_d2<(\(int\))?\d+, (\(int\))?3>", "spec_axis3")]


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
            "msecond": 1e-3, "second": 1}.get(u, 1)


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for d in rows[2:]:
        k = {"kernel": d[hdr.index("Kernel Name")][:120]}
        for m, name in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    k[name] = float(d[i]) * unit_scale(units[i])
                except ValueError:
                    pass
        for s in STALLS:
            m = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if m in hdr:
                k[f"stall_{s}"] = float(d[hdr.index(m)] or 0)
        out.append(k)
    return out


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) < len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[hdr.index("Kernel Name")].split("(")[0][:80]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values()) or 1.0
    return {k: {"launches": cnt[k], "total_ns": tot[k], "share": tot[k] / s}
            for k in sorted(tot, key=lambda x: -tot[x])}


def main():
    tag, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    os.makedirs(PROF, exist_ok=True)
    f = [k for rep in reps for k in full(rep)]
    json.dump(f, open(os.path.join(PROF, f"{tag}_ncu_full.json"), "w"), indent=1)
    if os.path.exists(lcsv):
        json.dump(launches(lcsv), open(os.path.join(PROF, f"{tag}_launches.json"), "w"), indent=1)
    tpath = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for k in f:
        for pat, timer in TIMER:
            if re.search(pat, k["kernel"]) and "dram_read" in k:
                traffic[timer] = k["dram_read"] + k.get("dram_write", 0.0)
    json.dump(traffic, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    # shared-memory wavefronts per launch (the SL kernels' binding pipe)
    wpath = os.path.join(PROF, "smem_wavefronts.json")
    wf = json.load(open(wpath)) if os.path.exists(wpath) else {}
    for k in f:
        for pat, timer in TIMER:
            if re.search(pat, k["kernel"]) and "smem_wavefronts" in k:
                wf[timer] = k["smem_wavefronts"]
    json.dump(wf, open(wpath, "w"), indent=1)
    for k in f:
        print(k["kernel"][:60], {x: round(k[x], 1) for x in ("duration", "dram_read", "dram_write",
                                                           "dram_pct", "warps_active_pct",
                                                           "issue_active_pct")
                                 if x in k})


if __name__ == "__main__":
    main()
