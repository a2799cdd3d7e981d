"""DRAM bytes per frame of K1 / K2 per chunk size from the ncu csv of
  ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:"das_image|analytic" --csv --log-file X.csv python tools/das_chunk_sweep.py 16 32 ...
(cfg2: grid = 64 channel-pair CTAs (K1) / 64 CTAs (K2) per frame, so frames per launch = grid / 64)
  python tools/chunk_dram_summary.py X.csv [traffic.json chunk]   (adds the chunk's record as "l2_chunk")"""
import collections
import csv
import io
import json
import sys

ALG = 2621440
rows = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}
for r in csv.DictReader(io.StringIO("".join(rows))):
    frames = int(r["Grid Size"].strip("()").split(",")[0]) // 64
    k = (frames, "K1" if "analytic" in r["Kernel Name"] else "K2")
    agg[k][r["Metric Name"]] += float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1)
    cnt[k] += r["Metric Name"] == "gpu__time_duration.sum"
recs = {}
for frames in sorted({k[0] for k in agg}):
    rec = {"chunk_frames": frames}
    tot = 0.0
    for kern in ("K1", "K2"):
        a, n = agg[(frames, kern)], cnt[(frames, kern)] * frames
        rec[f"{kern}_read_MB"] = round(a["dram__bytes_read.sum"] / n / 1e6, 3)
        rec[f"{kern}_write_MB"] = round(a["dram__bytes_write.sum"] / n / 1e6, 3)
        rec[f"{kern}_us"] = round(a["gpu__time_duration.sum"] / n, 3)
        tot += (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / n
    rec["dram_MB_per_frame"] = round(tot / 1e6, 3)
    rec["x_algorithmic"] = round(tot / ALG, 3)
    recs[frames] = rec
    print(json.dumps(rec))
if len(sys.argv) > 3:
    path, chunk = sys.argv[2], int(sys.argv[3])
    d = json.load(open(path))
    d["l2_chunk"] = dict(recs[chunk], dram_bytes_per_frame=recs[chunk]["dram_MB_per_frame"] * 1e6,
                         source=f"{sys.argv[1]} (ncu --cache-control none: L2 contents kept between K1 and K2, "
                                "dram__bytes_read.sum + dram__bytes_write.sum averaged over the sweep's launches)")
    open(path, "w").write(json.dumps(d, indent=1) + "\n")
