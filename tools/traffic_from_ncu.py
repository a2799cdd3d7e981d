"""Write profiles/<round>/traffic.json from an ncu --set full capture of
tools/profile_kernels.py (DRAM bytes read + written per frame of K1 and K2).

  python tools/traffic_from_ncu.py gpurun_out/prof.ncu-rep <frames> profiles/r1/traffic.json
"""
import csv
import io
import json
import subprocess
import sys

rep, frames, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
res = {}
for row in rows[2:]:
    name = row[hdr.index("Kernel Name")]
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[i]]
        tot += float(row[i].replace(",", "")) * scale
    key = "K1" if "analytic" in name else "K2" if "das_image" in name else \
        "RC" if "rowconv_tc1_kernel<0>" in name else None
    if key and key not in res:
        res[key] = tot if key == "RC" else tot / frames
out_d = {"das_pipeline_bytes_per_frame": res["K1"] + res["K2"], "K1_bytes_per_frame": res["K1"],
         "K2_bytes_per_frame": res["K2"], "frames_per_launch": frames,
         "source": f"{rep} (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum)"}
if "RC" in res:
    out_d.update(rowconv_cfg4_bytes_per_launch=res["RC"], rowconv_cfg4_algorithmic_bytes_per_launch=256 * 2048 * 1024 * 8,
                 rowconv_source=f"{rep}: rowconv_tc1_kernel<fwd>, 256 cfg4 maps")
try:  # keep the L2-sized-chunk record (tools/chunk_dram_summary.py) across refreshes
    old = json.load(open(out))
    if "l2_chunk" in old:
        out_d["l2_chunk"] = old["l2_chunk"]
except (OSError, ValueError):
    pass
open(out, "w").write(json.dumps(out_d, indent=1) + "\n")
print(out_d)
