"""Summarise an ncu report: SOL, issue, occupancy, smem wavefronts/conflicts, DRAM bytes, stall reasons."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
hdr, vals = r[0], r[2:]
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "lts__t_bytes.sum"]
for v in vals:
    d = dict(zip(hdr, v))
    for k in keys:
        if k in d:
            print(f"{k:70s} {d[k]}")
    st = {k: float(d[k]) for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled") or k.startswith("smsp__pcsamp_warps_issue_stalled")
          if d.get(k, "").replace(".", "", 1).isdigit()}
    top = sorted(st.items(), key=lambda kv: -kv[1])[:10]
    for k, x in top:
        print(f"   {k:80s} {x}")
    print("-" * 40)
