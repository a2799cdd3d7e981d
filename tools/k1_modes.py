"""Time K1 (rf_analytic) per TIDAS_K1_MODE on 64 cfg2 frames (f32) and 16 cfg5-shaped
frames (int16, 192 x 8192), each mode in a fresh process; outputs are saved and
compared bitwise against mode 0."""
import os, subprocess, sys
code = r'''
import os, sys, torch
sys.path.insert(0, ".")
import paper_2507_15464_b200 as tb
from bench import CFG2, frame_scatterers
cfg = CFG2; F = 64
sx, sz, a = frame_scatterers(cfg, range(F))
rf = tb.synthesize_batch(sx, sz, a, angles=[0.0], n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"])
g = torch.Generator(device="cuda"); g.manual_seed(5)
rf5 = (torch.randn((16, 1, 192, 8192), device="cuda", generator=g) * 1000).round().clamp(-32768, 32767).to(torch.int16)
rf1 = torch.randn((256, 1, 64, 2048), device="cuda", generator=g, dtype=torch.float64)
res = {}
for name, x in (("cfg2_f32", rf), ("cfg5_i16", rf5), ("cfg1_f64", rf1)):
    an = torch.empty(x.shape, dtype=torch.complex64, device="cuda")
    for _ in range(3): tb.rf_analytic(x, "f32", out=an)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): tb.rf_analytic(x, "f32", out=an)
    e1.record(); torch.cuda.synchronize()
    res[name] = an.cpu()
    print(name, "K1 us/frame", round(e0.elapsed_time(e1) * 1e3 / 10 / x.shape[0], 3))
torch.save({"rf": rf.cpu(), **res}, f"/tmp/k1_mode_{os.environ['TIDAS_K1_MODE']}.pt")
'''
modes = sys.argv[1:] or ["0", "1"]
for m in modes:
    env = dict(os.environ, TIDAS_K1_MODE=m)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("mode", m, (out.stdout.strip() or out.stderr.strip()[-600:]))
import torch
ref = torch.load(f"/tmp/k1_mode_{modes[0]}.pt")
for m in modes[1:]:
    d = torch.load(f"/tmp/k1_mode_{m}.pt")
    # the cfg2 RF comes from an atomics-based simulator: compare only when the inputs match
    same_in = torch.equal(ref["rf"], d["rf"])
    rel = lambda a, b: float((a - b).abs().pow(2).sum().sqrt() / b.abs().pow(2).sum().sqrt())
    print("mode", m, "cfg5 bitwise equal to mode", modes[0], torch.equal(ref["cfg5_i16"], d["cfg5_i16"]),
          "rel_l2", rel(d["cfg5_i16"], ref["cfg5_i16"]),
          "| cfg2 inputs equal", same_in, "outputs equal", torch.equal(ref["cfg2_f32"], d["cfg2_f32"]) if same_in else None,
          "rel_l2", rel(d["cfg2_f32"], ref["cfg2_f32"]) if same_in else None)
