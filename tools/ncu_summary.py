"""Summarise an .ncu-rep (run here, no GPU): per kernel duration, throughput,
occupancy, instruction mix, top stall reasons, shared-memory conflicts, DRAM bytes.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [kernel-substring]
"""
import csv
import io
import subprocess
import sys

import json
from pathlib import Path

_pk = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
HBM = float(json.loads(_pk.read_text())["hbm_gbs"]) if _pk.exists() else 6650.0
rep = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
KEYS = [("gpu__time_duration.sum", "duration"), ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %"),
        ("dram__bytes_read.sum", "dram rd"), ("dram__bytes_write.sum", "dram wr"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("launch__registers_per_thread", "regs"), ("smsp__inst_executed.sum", "warp inst"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lds conflicts"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "sts conflicts"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
        ("smsp__sass_inst_executed_op_shared_ld.sum", "LDS"), ("smsp__sass_inst_executed_op_shared_st.sum", "STS"),
        ("smsp__sass_inst_executed_op_local_ld.sum", "LDL"), ("smsp__sass_inst_executed_op_global_ld.sum", "LDG"),
        ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "ffma thr-inst")]
for row in rows[2:]:
    name = row[hdr.index("Kernel Name")]
    if flt not in name:
        continue
    print("==", name[:90])
    for k, lab in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"   {lab:16s} {row[i]} {units[i]}")
    # achieved bandwidths against the B200 peaks (MEASURED_PEAKS.json HBM copy
    # bandwidth; shared memory 128 B/clk/SM and L2 sectors at the captured clocks)
    def num(key):
        if key not in hdr:
            return None
        i = hdr.index(key)
        v = float(row[i].replace(",", "") or 0)
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                    "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
                    "hz": 1, "khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "MHz": 1e6, "GHz": 1e9,
                    "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "cycle/second": 1.0}.get(units[i], 1)
    dur = num("gpu__time_duration.sum")
    if dur:
        drb = (num("dram__bytes_read.sum") or 0) + (num("dram__bytes_write.sum") or 0)
        l2b = (num("lts__t_sectors.sum") or 0) * 32
        smw = (num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") or 0)
        clk = num("sm__cycles_elapsed.avg.per_second") or 1.965e9
        smpk = 128 * 148 * clk
        print(f"   dram GB/s        {drb / dur / 1e9:8.1f}  ({100 * drb / dur / 1e9 / HBM:.1f}% of {HBM:.0f} GB/s)")
        print(f"   L2 GB/s          {l2b / dur / 1e9:8.1f}  (lts__t_sectors x 32 B; lts throughput "
              f"{row[hdr.index('lts__throughput.avg.pct_of_peak_sustained_elapsed')] if 'lts__throughput.avg.pct_of_peak_sustained_elapsed' in hdr else '?'}% of peak)")
        print(f"   smem GB/s        {smw * 128 / dur / 1e9:8.1f}  ({100 * smw * 128 / dur / smpk:.1f}% of 128 B/clk/SM x 148 at "
              f"{clk / 1e6:.0f} MHz)")
    pipes = [(h, row[i]) for i, h in enumerate(hdr)
             if h.startswith("sm__inst_executed_pipe_") and h.endswith(".avg.pct_of_peak_sustained_active")]
    pipes = sorted(((float(v or 0), h.split("pipe_")[1].split(".")[0]) for h, v in pipes), reverse=True)[:6]
    print("   pipes          ", ", ".join(f"{n} {v:.0f}%" for v, n in pipes))
    st = [(h, row[i]) for i, h in enumerate(hdr)
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    tot = sum(float(v or 0) for _, v in st) or 1.0
    st = sorted(((float(v or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h, v in st), reverse=True)[:7]
    print("   stalls         ", ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in st))
