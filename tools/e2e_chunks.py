"""e2e (pinned host RF -> pinned host images) frames/s at cfg2 vs HostPipeline chunk size."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2507_15464_b200 as tb
from tests.setups import CFG2

c = CFG2
F, steps = 64, 20
x = np.linspace(*c["x"], c["nx"]); z = np.linspace(*c["z"], c["nz"])
plan = tb.plane_wave_plan(n_el=c["n_el"], pitch=c["pitch"], fs=c["fs"], c=c["c"], n_samples=c["n_samples"],
                          x=x, z=z, angles=[0.0], f_number=c["f_number"])
host_rf = torch.randn((F, 1, c["n_el"], c["n_samples"]), dtype=torch.float32).pin_memory()
host_img = torch.empty((F, c["nz"], c["nx"]), dtype=torch.float32).pin_memory()
cur = torch.cuda.current_stream()
for chunk in (8, 16, 32, 64):
    pipe = tb.HostPipeline(plan, chunk=chunk)
    for _ in range(3):
        pipe.run(host_rf, host_img)
    pipe.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    pipe.wait_for(cur)
    for _ in range(steps):
        pipe.run(host_rf, host_img)
    pipe.join(cur)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"chunk {chunk:3d}: {ms:.3f} ms/step  {F / ms * 1e3:.0f} frames/s  "
          f"(H2D {host_rf.numel() * 4 / ms / 1e6:.1f} GB/s)", flush=True)
# serial reference: copy in, compute, copy out on one stream
rf_dev = torch.empty(host_rf.shape, device="cuda"); img = torch.empty(host_img.shape, device="cuda")
ws = tb.DasWorkspace(plan)
def serial():
    rf_dev.copy_(host_rf, non_blocking=True); tb.das_image(rf_dev, plan, out=img, workspace=ws)
    host_img.copy_(img, non_blocking=True)
for _ in range(3): serial()
torch.cuda.synchronize()
e0.record(); [serial() for _ in range(steps)]; e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"serial: {ms:.3f} ms/step  {F / ms * 1e3:.0f} frames/s")
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); [rf_dev.copy_(host_rf, non_blocking=True) for _ in range(steps)]; t1.record(); torch.cuda.synchronize()
print(f"H2D alone: {host_rf.numel() * 4 * steps / t0.elapsed_time(t1) / 1e6:.1f} GB/s")
