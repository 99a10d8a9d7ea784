"""profiles/traffic.json from an ncu --set full capture of the pipeline kernels (8-slice launches):
per-slice dram__bytes_read.sum + dram__bytes_write.sum per kernel, tagged with the sha256 of the
kernel sources the capture was taken on (bench.py reports roofline.traffic only for that source)."""
import csv, io, json, os, re, subprocess, sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
from paper_1608_03589_b200 import roofline  # noqa: E402

rep, tag, engine = sys.argv[1], sys.argv[2], (sys.argv[3] if len(sys.argv) > 3 else "logpolar")
slices = int(sys.argv[4]) if len(sys.argv) > 4 else 32  # slices per captured launch (the bench chunk)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
names = {"k_ramp": "ramp_filter", "k_row_rdft": "row_rdft", "k_rho_conv": "rho_conv", "k_irdft_readout": "irdft_readout",
         "k_bst_radial": "bst_radial", "k_bst_grid_x": "bst_grid_x", "k_bst_grid_y": "bst_grid_y"}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
ik, ir, iw = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
per = {}
for r in rows[2:]:
    k = re.sub(r"\(.*", "", r[ik]).replace("void ", "").split("<")[0].split("::")[-1]
    stage = next((v for kk, v in names.items() if k.startswith(kk)), None)
    if stage:
        b = float(r[ir].replace(",", "")) * scale[units[ir]] + float(r[iw].replace(",", "")) * scale[units[iw]]
        per[stage] = b / slices
path = os.path.join(root, "profiles", "traffic.json")
t = json.load(open(path)) if os.path.exists(path) else {}
t[engine] = {"capture": f"profiles/{tag}_summary.md", "csrc_sha256": roofline.kernel_source_digest(), "per_slice": per}
json.dump(t, open(path, "w"), indent=1)
print(json.dumps(t[engine], indent=1))
