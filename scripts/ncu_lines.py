"""Attribute ncu warp-stall samples of one kernel to source lines (inline chain aware).

usage: python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX MANGLED_SUBSTR [SO] [TOP]

Joins the SASS page of the report (per-instruction samples, function-relative
offsets) with `nvdisasm -gi` line info of the same kernel from the cubin inside
the shared library, and prints samples per outermost-call-site chain, so the
phases of an inlined block_conv / block_fft (pass by pass) can be told apart.
Needs the library that was profiled (default paper_1608_03589_b200/liblpbp.so).
"""
import csv, io, os, re, subprocess, sys, tempfile
from collections import defaultdict

rep, kre, mangled = sys.argv[1], sys.argv[2], sys.argv[3]
rest = sys.argv[4:]
top = 40
if rest and rest[-1].isdigit():  # [SO] [TOP] in either form
    top = int(rest.pop())
so = rest[0] if rest else os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1608_03589_b200",
                                       "liblpbp.so")
NF = int(os.environ.get("NF", "2"))

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, ist, isrc = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
iex = h.index("Instructions Executed")
samples = {}
base = None
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except (ValueError, IndexError):
        continue
    if a in samples:  # the listing repeats itself
        break
    base = a if base is None else min(base, a)
    samples[a] = (int(r[ist] or 0), r[isrc].strip(), int(r[iex] or 0))

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
chain_of = {}
for cub in os.listdir(tmp):
    dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    infn, cur, prev_comment = False, "", False
    for line in dis.splitlines():
        if line.startswith("//----") and ".text." in line:
            infn = mangled in line
            continue
        if not infn:
            continue
        m = re.match(r"\s*//## File \"([^\"]+)\", line (\d+)", line)
        if m:
            # a group of consecutive comments lists the inline chain innermost -> outermost, one frame each
            here = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            cur = cur + " <- " + here if prev_comment else here
            prev_comment = True
            continue
        prev_comment = False
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
        if m:
            chain_of[int(m.group(1), 16)] = cur
    if chain_of:
        break

tot = sum(v[0] for v in samples.values()) or 1
tex = sum(v[2] for v in samples.values()) or 1
by_site = defaultdict(lambda: [0, 0])
for a, (s, src, ex) in samples.items():
    ch = chain_of.get(a - base, "?")
    parts = ch.split(" <- ")
    k = " <- ".join(parts[-NF:])
    by_site[k][0] += s
    by_site[k][1] += ex
print(f"total samples {tot}, warp-instructions executed {tex:.3g}, SASS lines {len(samples)}, "
      f"mapped {sum(1 for a in samples if a - base in chain_of)}")
print("-- by outer call site (last NF frames): % of stall samples, % of executed instructions")
for k, v in sorted(by_site.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}%  {100 * v[1] / tex:5.1f}%  {k}")
