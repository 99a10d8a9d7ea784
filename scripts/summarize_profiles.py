"""Write profiles/<tag>_summary.md from gpurun_out/{launches_<tag>.csv, full_<tag>.ncu-rep, bench_<tag>.json}."""
import csv, io, json, os, re, subprocess, sys
from collections import defaultdict

tag = sys.argv[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go = os.path.join(root, "gpurun_out")
out = []

bench = os.path.join(go, f"bench_{tag}.json")
if os.path.exists(bench):
    line = open(bench).read().strip().splitlines()[-1]
    out.append("## bench line\n\n```json\n" + json.dumps(json.loads(line), indent=1) + "\n```\n")

lc = os.path.join(go, f"launches_{tag}.csv")
if os.path.exists(lc):
    txt = open(lc).read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    h = rows[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        name = re.sub(r"\(.*", "", r[ik]).replace("void ", "")
        v = float(r[iv].replace(",", ""))
        v = {"nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}.get(r[iu], 1.0) * v  # -> usecond
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    hot = ("k_ramp", "k_row_rdft", "k_rho_conv", "k_irdft_readout", "k_row_irdft", "k_readout")
    ours = {k: v for k, v in agg.items() if any(h in k for h in hot)}
    tot_ours = sum(v[1] for v in ours.values())
    out.append(f"## launch list (ncu gpu__time_duration, cold-cache serialised)\n\n"
               f"{sum(v[0] for v in agg.values())} launches, {tot:.0f} us total; hot-path kernels {tot_ours:.0f} us "
               "(input generation k_radon_ellipses and torch noise kernels are harness)\n\n"
               "| kernel | launches | total us | share of hot path |\n|---|---|---|---|\n")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share = f"{100 * t / tot_ours:.1f}%" if k in ours else "-"
        out.append(f"| {k[:70]} | {n} | {t:.0f} | {share} |\n")
    out.append("\n")

rep = os.path.join(go, f"full_{tag}.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    keys = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
            ("dram__bytes_write.sum", "DRAM write"),
            ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
            ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
            ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
            ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
            ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
            ("lts__t_sector_hit_rate.pct", "L2 hit %"),
            ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld conflicts"),
            ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st conflicts"),
            ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"), ("launch__block_size", "block")]
    stall = [i for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
    out.append("## ncu --set full (one launch per kernel, chunk of 32 slices 2048^2 FBP (bench default))\n\n")
    names = [re.sub(r"\(.*", "", r[h.index("Kernel Name")]).replace("void ", "") for r in rows[2:]]
    out.append("| metric | " + " | ".join(names) + " |\n|---|" + "---|" * len(names) + "\n")
    for k, label in keys:
        if k not in h:
            continue
        i = h.index(k)
        out.append(f"| {label} ({units[i]}) | " + " | ".join(r[i] for r in rows[2:]) + " |\n")
    tops = []
    for r in rows[2:]:
        st = sorted(((float(r[i].replace(',', '') or 0), h[i].replace("smsp__pcsamp_warps_issue_stalled_", "")) for i in stall), reverse=True)
        t = sum(s for s, _ in st) or 1
        tops.append(", ".join(f"{n} {100 * s / t:.0f}%" for s, n in st[:4]))
    out.append("| top stalls | " + " | ".join(tops) + " |\n")

dst = os.path.join(root, "profiles", f"{tag}_summary.md")
open(dst, "w").write(f"# profile summary {tag}\n\n" + "".join(out))
print(open(dst).read())
