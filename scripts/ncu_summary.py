"""Summarise an ncu report: per kernel, SOL %, DRAM bytes, pipe utilisation, top stalls."""
import csv, io, subprocess, sys, re
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]
idx = {n: h.index(n) for n in want if n in h}
stall = [i for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
for r in rows[2:]:
    print("=" * 100)
    for n, i in idx.items():
        v = r[i]
        if n == "Kernel Name":
            v = re.sub(r"\(.*", "", v)[:90]
        print(f"  {n:75s} {units[i]:10s} {v}")
    st = sorted(((float(r[i].replace(',', '') or 0), h[i].replace("smsp__pcsamp_warps_issue_stalled_", "")) for i in stall), reverse=True)
    tot = sum(s for s, _ in st) or 1
    print("  top stalls:", ", ".join(f"{n} {100*s/tot:.0f}%" for s, n in st[:6]))
