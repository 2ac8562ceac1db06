"""One-line-per-capture summary of ncu raw CSV exports (profiles/r02)."""
import csv, json, sys
keys = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "lsu_pct",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "bank_conflicts",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
        "launch__registers_per_thread": "regs", "smsp__inst_executed.sum": "warp_inst"}
out = {}
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
    rec = {"kernel": d.get("Kernel Name", "")[:90]}
    for k, n in keys.items():
        if k in d:
            v = float(d[k].replace(",", ""))
            if k.startswith("dram__bytes"):
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[k], 1)
            if k == "gpu__time_duration.sum":
                v *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u[k], 1)
            rec[n] = v
    out[f.split("/")[-1].replace(".raw.csv", "")] = rec
print(json.dumps(out, indent=1))
