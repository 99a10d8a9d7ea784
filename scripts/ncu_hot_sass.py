"""Top stalled SASS instructions of one kernel in an ncu report (needs --import-source / -lineinfo)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc, ist = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
iex = h.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ist]), r[ia], r[isrc].strip(), int(r[iex])))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print(f"total samples {tot}")
for s, a, src, ex in sorted(data, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}%  {a[-5:]}  {src[:70]:70s} exec={ex}")
# grouped by opcode
from collections import Counter
c = Counter()
for s, a, src, ex in data:
    c[src.split()[0] if not src.startswith('@') else src.split()[1]] += s
print("by opcode:", ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in c.most_common(12)))
